/*
 * fkde_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's naive O(n*m*d) oracle
 * (/root/reference/proj/core/src/oracle.cpp:36-118), its scalar kernels
 * (kernels.cpp:26-41), its portable RNG (rng.cpp:8-32, rng.hpp:52-75), the
 * mixture sampler (mixture.cpp:40-67) and the bandwidth rules
 * (bandwidth.cpp:9-58).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this library, and only as the checker or the
 * CPU baseline -- never as the product path.  The product path
 * (paper_2602_10378_b200/) never links or loads it.
 *
 * Parity is pinned (tests/test_oracle.py) against:
 *   - the reference's own known-answer constants (test_kernels.cpp:14-55,
 *     test_oracle.cpp:21-167), and
 *   - oracle/_ref/libfkde_ref.so, the reference's own oracle.cpp/kernels.cpp/
 *     rng.cpp/mixture.cpp/bandwidth.cpp/types.cpp compiled here from
 *     /root/reference by oracle/Makefile, bitwise on seeded inputs, and
 *   - tests/golden/*.npz fixtures produced by that library
 *     (tests/golden/make_golden.py).
 *
 * Arithmetic is fp64, evaluation order mirrors the reference expression by
 * expression, and the file is compiled with -ffp-contract=off exactly like
 * the reference oracle (core/CMakeLists.txt:25).
 */
#ifndef FKDE_ORACLE_H
#define FKDE_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes shared with the tests */
#define FKO_OK 0
#define FKO_INVALID_ARGUMENT 1
#define FKO_DIMENSION_MISMATCH 2
#define FKO_SCORE_UNDERFLOW 3

/* --- RNG (rng.cpp / rng.hpp) ------------------------------------------- */
uint64_t fko_mix64(uint64_t x);
/* train-style i.i.d. N(0, scale^2) fill, test_util.hpp:12-20 */
void fko_random_gaussian(size_t n, size_t d, uint64_t seed, double scale, double* out);
/* Rng(seed, stream).uniform01() sequence, for the h-draws in acceptance crit. 1 */
void fko_uniform01(uint64_t seed, uint64_t stream, size_t count, double* out);
/* mixture.cpp:40-67; means is k x d row-major */
void fko_sample_mixture(const double* weights, const double* means, const double* sigmas,
                        size_t k, size_t d, size_t n, uint64_t seed, double* out);

/* --- scalar kernels (kernels.cpp) ---------------------------------------- */
double fko_gaussian_norm_const(double h, size_t d);
double fko_gaussian_kernel(double r2, double h, size_t d);
double fko_laplace_corrected_kernel(double r2, double h, size_t d);

/* --- bandwidth rules (bandwidth.cpp) -------------------------------------- */
double fko_mean_stddev(const double* x, size_t n, size_t d);
double fko_silverman_prefactor(size_t d);
double fko_silverman_bandwidth(const double* x, size_t n, size_t d);
double fko_sdkde_bandwidth(const double* x, size_t n, size_t d, double c);

/* --- naive estimators (oracle.cpp) ---------------------------------------
 * eval rows [row_begin, row_end) only; the full call is [0, m).  Each row is
 * a pure function of its inputs, so sharded calls are bitwise identical to a
 * full call.  nthreads > 1 splits the row range into contiguous shards. */
int fko_kde_naive(const double* train, size_t n, const double* queries, size_t m, size_t d,
                  double h, size_t row_begin, size_t row_end, int nthreads, double* out);
int fko_laplace_naive(const double* train, size_t n, const double* queries, size_t m, size_t d,
                      double h, size_t row_begin, size_t row_end, int nthreads, double* out);
/* out is (row_end-row_begin) x d; *err_index receives the underflowing row */
int fko_score_naive(const double* train, size_t n, const double* eval, size_t m, size_t d,
                    double h_score, size_t row_begin, size_t row_end, int nthreads,
                    double* out, size_t* err_index);
/* full pipeline (oracle.cpp:87-101); debiased (n x d) may be NULL */
int fko_sdkde_naive(const double* train, size_t n, const double* queries, size_t m, size_t d,
                    double h, double h_score, int nthreads, double* out, double* debiased,
                    size_t* err_index);

#ifdef __cplusplus
}
#endif
#endif
