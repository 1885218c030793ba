/*
 * fkde_gpu.h -- C ABI of the B200-native Flash-SD-KDE engine
 * (paper_2602_10378_b200/libfkde_b200.so).
 *
 * This is the drop-in boundary for the reference's estimator hot path.  Each
 * entry point replaces one function of the reference's C++ engine
 * (/root/reference/proj/core/include/fkde/engine.hpp) behind the dispatcher
 * fkde::estimate() (estimator.hpp:9-10, estimator.cpp:22-48):
 *
 *   fkde_gpu_score             <- fkde::engine::score_flash        engine.hpp:63-64, engine.cpp:302-340
 *   fkde_gpu_score_accumulate  <- fkde::engine::score_accumulate   engine.hpp:58-59, engine.cpp:279-300
 *   fkde_gpu_kde               <- fkde::engine::kde_flash          engine.hpp:70-72, engine.cpp:342-387
 *   fkde_gpu_sdkde             <- fkde::engine::sdkde_flash        engine.hpp:74-76, engine.cpp:389-405
 *   fkde_gpu_pairwise_sq_dists <- fkde::engine::pairwise_sq_dists_block  engine.hpp:46-49, engine.cpp:261-277
 *   fkde_gpu_estimate          <- fkde::estimate                   estimator.hpp:9-10, estimator.cpp:52-60
 *
 * Conventions (mirroring the reference's value semantics):
 *   - inputs are caller-owned, row-major, fp64 (SampleSet::values layout,
 *     types.hpp:15-41); outputs are caller-allocated fp64 buffers;
 *   - no exception crosses the ABI: every call returns an fkde_status and
 *     fkde_gpu_last_error(ctx) holds the message; the C++ facade
 *     (include/fkde_b200/engine.hpp) maps statuses back onto the reference's
 *     exception types (errors.hpp:10-56);
 *   - validation matches the reference: n, d >= 1, finite entries, h > 0,
 *     train.d == queries.d (types.cpp:21-33, 65-79; engine.cpp:27-34);
 *   - the context owns the CUDA streams, cached device workspaces and (for
 *     more than one device) the NCCL communicator, and is reused across calls
 *     so that timing excludes initialisation;
 *   - results are bitwise deterministic for a fixed context configuration.
 *
 * Multi-GPU: fkde_gpu_create(devices, n) drives n devices from one process
 * (one host thread per device, ncclCommInitAll); fkde_gpu_create_rank() is the
 * one-process-per-GPU form (torchrun), with the ncclUniqueId produced by
 * fkde_gpu_nccl_unique_id() on rank 0 and broadcast by the caller.  NCCL is
 * dlopen'ed on first multi-rank use: libnccl.so.2, or the library named by the
 * FKDE_NCCL_LIB environment variable (a specific NCCL build, or the tests'
 * in-process transport, tests/cpp/nccl_emu.cpp).  Sample
 * rows are sharded for the score pass, the debiased samples are gathered with
 * one ncclAllGather, and queries are sharded for the density pass.
 */
#ifndef FKDE_GPU_H
#define FKDE_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum fkde_status {
    FKDE_OK = 0,
    FKDE_INVALID_ARGUMENT = 1,    /* fkde::InvalidArgumentError            */
    FKDE_DIMENSION_MISMATCH = 2,  /* fkde::DimensionMismatchError          */
    FKDE_SCORE_UNDERFLOW = 3,     /* fkde::ScoreUnderflowError(index)       */
    FKDE_NON_FINITE = 4,          /* fkde::InvalidArgumentError (non-finite input) */
    FKDE_CUDA_ERROR = 5,
    FKDE_NCCL_ERROR = 6,
    FKDE_UNSUPPORTED_D = 7,       /* d > 16 on the tensor-core path          */
    FKDE_NO_DEVICE = 8
} fkde_status;

/* KernelKind (types.hpp:45) */
enum { FKDE_KERNEL_GAUSSIAN = 0, FKDE_KERNEL_LAPLACE_CORRECTED = 1 };
/* Method (types.hpp:43) */
enum { FKDE_METHOD_KDE = 0, FKDE_METHOD_SDKDE = 1, FKDE_METHOD_LAPLACE = 2 };

/* options (fkde_gpu_set_option) */
enum {
    FKDE_OPT_ENGINE = 1,      /* FKDE_ENGINE_TC (the only engine; kept for ABI
                                 stability, any other value is rejected)         */
    FKDE_OPT_SPLITS = 2,      /* 0 = auto; >0 forces column splits per row tile  */
    FKDE_OPT_TIMING = 3,      /* 1 = record per-phase CUDA-event times            */
    FKDE_OPT_MAX_CTAS = 4,    /* 0 = all SMs; >0 caps the persistent grid        */
    FKDE_OPT_FLUSH_TILES = 5, /* score pass: drain the TMEM accumulator to the
                                 extended-precision register sums every k column
                                 tiles; k a power of two in [1, 2^20], or 0 for
                                 the default (~256 columns)                      */
    FKDE_OPT_TRACE_PTR = 6,   /* debug: device pointer (32*8*256 int64) receiving
                                 clock64 stamps of the score kernel's block 0   */
    FKDE_OPT_SPATIAL = 7,     /* score and density passes on a spatial (Morton /
                                 principal-axis) order of the points, skipping the
                                 tile pairs proven / checked to contribute nothing
                                 (score: exact zeros; density: < 2^-24 of a row's
                                 mass, else the row is recomputed directly):
                                 0 = auto (n >= 32768), 1 = always, 2 = never,
                                 3 = the order without skipping (tests: skipping
                                 must not change a score bit)                    */
    FKDE_OPT_PDL = 8          /* 1 (default) = launch the kernel chain with
                                 programmatic dependent launch; 0 = plain launches */
};
enum { FKDE_ENGINE_TC = 0 };

/* per-phase timings (fkde_gpu_last_timing), milliseconds, rank-local */
enum {
    FKDE_T_PREP = 0,      /* H2D + mean + operand packing         */
    FKDE_T_SCORE = 1,     /* score pass kernel                    */
    FKDE_T_FINALIZE = 2,  /* score finalize + SD shift            */
    FKDE_T_GATHER = 3,    /* allgather of the debiased samples    */
    FKDE_T_QUERY = 4,     /* density pass kernel(s)               */
    FKDE_T_REDUCE = 5,    /* density reduction + gather + D2H     */
    FKDE_T_TOTAL = 6,
    FKDE_T_COUNT = 7
};

typedef struct fkde_gpu_ctx fkde_gpu_ctx;

/* ---- lifecycle ---------------------------------------------------------- */
int fkde_gpu_device_count(int* count);
/* devices: ids in [0, device count), or NULL for 0..n_devices-1 */
int fkde_gpu_create(const int* devices, int n_devices, fkde_gpu_ctx** out);
int fkde_gpu_nccl_unique_id(unsigned char id[128]);
int fkde_gpu_create_rank(int device, int rank, int world, const unsigned char id[128],
                         fkde_gpu_ctx** out);
void fkde_gpu_destroy(fkde_gpu_ctx* ctx);
/* message of the calling thread's last call on ctx (or, if this thread made
 * none, a private copy of the context's most recent message); the pointer
 * stays valid until this thread's next call on ctx */
const char* fkde_gpu_last_error(const fkde_gpu_ctx* ctx);
int fkde_gpu_set_option(fkde_gpu_ctx* ctx, int key, int64_t value);
int fkde_gpu_world(const fkde_gpu_ctx* ctx, int* rank, int* world);
/* cudaStream_t of the (first) device, for callers timing on the device */
void* fkde_gpu_stream(fkde_gpu_ctx* ctx);
/* device timings of the last call (needs FKDE_OPT_TIMING=1); n <= FKDE_T_COUNT */
int fkde_gpu_last_timing(const fkde_gpu_ctx* ctx, float* ms, int n);
/* per-kernel device times of the last call (needs FKDE_OPT_TIMING=1): CUDA events
 * bracketing each tensor-core pass kernel on the engine's stream, ms, 0 where the
 * kernel did not run; n <= FKDE_KT_COUNT */
enum {
    FKDE_KT_SCORE = 0,    /* pairwise_tc_kernel<Score>                         */
    FKDE_KT_CHECK = 1,    /* pairwise_tc_kernel<Check> (score tile skipping)   */
    FKDE_KT_DENSITY = 2,  /* pairwise_tc_kernel<Gauss|Laplace> (last launch)   */
    FKDE_KT_COUNT = 3
};
int fkde_gpu_last_kernel_timing(const fkde_gpu_ctx* ctx, float* ms, int n);
/* number of kernels this library launched during the last call (this rank) */
int64_t fkde_gpu_last_launch_count(const fkde_gpu_ctx* ctx);
/* tile skipping of the last call on device 0 (synchronises); fills
 * min(n, FKDE_SKIP_STATS_COUNT) entries:
 *   [0] score pass: (row tile, column tile) pairs checked exactly
 *   [1] score pass: pairs skipped (every pair of points in them contributes
 *       exactly zero to the fp16 P sums)
 *   [2] score pass: pairs in the pass       [3] 1 if it ran on the spatial order
 *   [4] density pass: pairs skipped (box bound: every kernel value < 2^-44.5)
 *   [5] density pass: pairs in the pass     [6] 1 if it ran on the spatial order
 *   [7] density pass: query rows recomputed by direct differences
 *   [8] score pass: rows recomputed by direct differences */
#define FKDE_SKIP_STATS_COUNT 9
int fkde_gpu_last_skip_stats(fkde_gpu_ctx* ctx, uint64_t* out, size_t n);
/* device workspace currently held by the context (all devices), bytes: the
 * analogue of the reference's transient-allocation accounting
 * (alloc_stats, test_engine.cpp:218-243) -- linear in n + m, never n x m */
int fkde_gpu_workspace_bytes(const fkde_gpu_ctx* ctx, size_t* bytes);

/* Row partition used by every multi-GPU pass: rank r owns rows
 * [begin, begin + rows) of n, slices are `chunk` rows (chunk = ceil(n/world)
 * rounded up to `align`), so every allgather slice has the same size.  Pure
 * host arithmetic (no device needed). */
int fkde_gpu_shard_range(size_t n, int world, int rank, size_t align, size_t* begin,
                         size_t* rows, size_t* chunk);

/* ---- hot path (host fp64 buffers) --------------------------------------- */
/* scores: n x d.  On FKDE_SCORE_UNDERFLOW *err_index is the failing row. */
int fkde_gpu_score(fkde_gpu_ctx* ctx, const double* X, size_t n, size_t d, double h_score,
                   double* scores, size_t* err_index);
/* raw totals: phi_sum[n] = sum_j phi_ij (self term included), weighted n x d = sum_j phi_ij x_j */
int fkde_gpu_score_accumulate(fkde_gpu_ctx* ctx, const double* X, size_t n, size_t d,
                              double h_score, double* phi_sum, double* weighted);
/* densities at m queries; kernel = FKDE_KERNEL_*; fused only for Laplace */
int fkde_gpu_kde(fkde_gpu_ctx* ctx, const double* X, size_t n, const double* Y, size_t m,
                 size_t d, double h, int kernel, int fused, double* out);
/* score -> x + h^2/2 s -> Gaussian KDE; debiased (n x d) may be NULL */
int fkde_gpu_sdkde(fkde_gpu_ctx* ctx, const double* X, size_t n, const double* Y, size_t m,
                   size_t d, double h, double h_score, double* out, double* debiased,
                   size_t* err_index);
/* fkde::estimate: method = FKDE_METHOD_*; tile_m/tile_n validated (>= 1) for
 * error parity but the device schedule is the engine's own; negative_mass
 * (may be NULL) receives the Laplace diagnostic (estimator.cpp:14-20). */
int fkde_gpu_estimate(fkde_gpu_ctx* ctx, const double* X, size_t n, const double* Y, size_t m,
                      size_t d, int method, double h, double h_score, size_t tile_m,
                      size_t tile_n, int fused, double* out, double* debiased,
                      double* negative_mass, size_t* err_index);
/* na x nb squared distances, norm expansion with the 16-eps snap band (fp64) */
int fkde_gpu_pairwise_sq_dists(fkde_gpu_ctx* ctx, const double* A, size_t na, const double* B,
                               size_t nb, size_t d, double* out);

/* ---- device-resident variants (single-device contexts) -------------------
 * Pointers are device memory on the context's device; work is enqueued on
 * fkde_gpu_stream(ctx) and the call returns without synchronising.  A call
 * repeated with identical arguments and options is captured into a CUDA
 * graph on its second occurrence and replayed from the third on.
 * Host-side argument checks are the same as the host entry points (null
 * pointers, sizes, d, h, kernel kind); because nothing is read back, these
 * calls NEVER report FKDE_NON_FINITE (NaN/Inf inputs) or
 * FKDE_SCORE_UNDERFLOW -- use the host entry points when those diagnostics
 * matter. */
int fkde_gpu_sdkde_device(fkde_gpu_ctx* ctx, const double* dX, size_t n, const double* dY,
                          size_t m, size_t d, double h, double h_score, double* d_out);
/* scores (n x d) of device-resident samples; rows whose score denominator
 * underflows are not reported here (use fkde_gpu_score for the error index) */
int fkde_gpu_score_device(fkde_gpu_ctx* ctx, const double* dX, size_t n, size_t d, double h_score,
                          double* d_scores);
int fkde_gpu_kde_device(fkde_gpu_ctx* ctx, const double* dX, size_t n, const double* dY,
                        size_t m, size_t d, double h, int kernel, int fused, double* d_out);

/* ---- host-side input fixtures (bench / CLI), not on the device path -------
 * Bitwise reproductions of the reference's RNG (rng.cpp, mixture.cpp:40-67,
 * test_util.hpp:12-20) and bandwidth rules (bandwidth.cpp:9-58). */
uint64_t fkde_host_mix64(uint64_t x);
void fkde_host_random_gaussian(size_t n, size_t d, uint64_t seed, double scale, double* out);
int fkde_host_sample_mixture(const double* weights, const double* means, const double* sigmas,
                             size_t k, size_t d, size_t n, uint64_t seed, double* out);
double fkde_host_mean_stddev(const double* x, size_t n, size_t d);
double fkde_host_silverman_prefactor(size_t d);
double fkde_host_silverman_bandwidth(const double* x, size_t n, size_t d);
double fkde_host_sdkde_bandwidth(const double* x, size_t n, size_t d, double c);

#ifdef __cplusplus
}
#endif
#endif /* FKDE_GPU_H */
