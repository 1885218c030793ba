/*
 * fkde_oracle.c -- TEST INFRASTRUCTURE ONLY (see fkde_oracle.h).
 * CPU restatement of the reference oracle; every function cites the
 * reference line it follows.  Compile with -ffp-contract=off.
 */
#include "fkde_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* mt19937_64 (the engine std::mt19937_64 the reference wraps, rng.hpp:72)   */
/* ------------------------------------------------------------------------ */
typedef struct {
    uint64_t mt[312];
    int idx;
    double spare;
    int has_spare;
} fko_rng;

static void mt_seed(fko_rng* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < 312; ++i) {
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    }
    r->idx = 312;
    r->has_spare = 0;
    r->spare = 0.0;
}

static uint64_t mt_next(fko_rng* r) {
    if (r->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (r->mt[i] & 0xFFFFFFFF80000000ULL) | (r->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
        }
        r->idx = 0;
    }
    uint64_t y = r->mt[r->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

/* rng.cpp:8-13 */
uint64_t fko_mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

/* rng.hpp:54-55: Rng(seed, stream) seeds with mix64(seed ^ mix64(stream + 1)) */
static void rng_init(fko_rng* r, uint64_t seed, uint64_t stream) {
    mt_seed(r, fko_mix64(seed ^ fko_mix64(stream + 1)));
}

/* rng.hpp:60-62 */
static double rng_uniform01(fko_rng* r) { return (double)(mt_next(r) >> 11) * 0x1.0p-53; }

/* rng.cpp:15-32 (Box-Muller, caches the sine deviate) */
static double rng_normal(fko_rng* r) {
    if (r->has_spare) {
        r->has_spare = 0;
        return r->spare;
    }
    double u1;
    do {
        u1 = rng_uniform01(r);
    } while (u1 == 0.0);
    const double u2 = rng_uniform01(r);
    const double rr = sqrt(-2.0 * log(u1));
    const double theta = 2.0 * 3.141592653589793238462643383279502884 * u2;
    r->spare = rr * sin(theta);
    r->has_spare = 1;
    return rr * cos(theta);
}

/* test_util.hpp:12-20 */
void fko_random_gaussian(size_t n, size_t d, uint64_t seed, double scale, double* out) {
    fko_rng r;
    rng_init(&r, seed, 0);
    for (size_t i = 0; i < n * d; ++i) out[i] = scale * rng_normal(&r);
}

void fko_uniform01(uint64_t seed, uint64_t stream, size_t count, double* out) {
    fko_rng r;
    rng_init(&r, seed, stream);
    for (size_t i = 0; i < count; ++i) out[i] = rng_uniform01(&r);
}

/* mixture.cpp:40-67 */
void fko_sample_mixture(const double* weights, const double* means, const double* sigmas,
                        size_t k, size_t d, size_t n, uint64_t seed, double* out) {
    fko_rng r;
    rng_init(&r, seed, 0);
    for (size_t i = 0; i < n; ++i) {
        const double u = rng_uniform01(&r);
        size_t comp = k - 1;
        double cum = 0.0;
        for (size_t c = 0; c < k; ++c) {
            cum += weights[c];
            if (u < cum) {
                comp = c;
                break;
            }
        }
        for (size_t kk = 0; kk < d; ++kk) {
            out[i * d + kk] = means[comp * d + kk] + sigmas[comp] * rng_normal(&r);
        }
    }
}

/* ------------------------------------------------------------------------ */
/* kernels.cpp:26-41                                                         */
/* ------------------------------------------------------------------------ */
double fko_gaussian_norm_const(double h, size_t d) {
    const double dd = (double)d;
    return pow(2.0 * 3.141592653589793238462643383279502884, -0.5 * dd) * pow(h, -dd);
}

double fko_gaussian_kernel(double r2, double h, size_t d) {
    return fko_gaussian_norm_const(h, d) * exp(-r2 / (2.0 * h * h));
}

double fko_laplace_corrected_kernel(double r2, double h, size_t d) {
    const double u = r2 / (2.0 * h * h);
    return fko_gaussian_norm_const(h, d) * exp(-u) * (1.0 + 0.5 * (double)d - u);
}

/* ------------------------------------------------------------------------ */
/* bandwidth.cpp:9-58                                                        */
/* ------------------------------------------------------------------------ */
double fko_mean_stddev(const double* x, size_t n, size_t d) {
    double acc = 0.0;
    for (size_t j = 0; j < d; ++j) {
        double mean = 0.0;
        for (size_t i = 0; i < n; ++i) mean += x[i * d + j];
        mean /= (double)n;
        double ssq = 0.0;
        for (size_t i = 0; i < n; ++i) {
            const double diff = x[i * d + j] - mean;
            ssq += diff * diff;
        }
        acc += sqrt(ssq / (double)(n - 1));
    }
    return acc / (double)d;
}

double fko_silverman_prefactor(size_t d) {
    const double dd = (double)d;
    return pow(4.0 / (dd + 2.0), 1.0 / (dd + 4.0));
}

double fko_silverman_bandwidth(const double* x, size_t n, size_t d) {
    const double sigma = fko_mean_stddev(x, n, d);
    const double dd = (double)d;
    return sigma * fko_silverman_prefactor(d) * pow((double)n, -1.0 / (dd + 4.0));
}

double fko_sdkde_bandwidth(const double* x, size_t n, size_t d, double c) {
    const double sigma = fko_mean_stddev(x, n, d);
    const double dd = (double)d;
    return c * sigma * pow((double)n, -1.0 / (dd + 8.0));
}

/* ------------------------------------------------------------------------ */
/* oracle.cpp                                                                */
/* ------------------------------------------------------------------------ */
/* oracle.cpp:25-32 */
static double sq_dist(const double* a, const double* b, size_t d) {
    double r2 = 0.0;
    for (size_t k = 0; k < d; ++k) {
        const double diff = a[k] - b[k];
        r2 += diff * diff;
    }
    return r2;
}

static int valid_h(double h) { return h > 0.0 && isfinite(h); }

enum { JOB_KDE, JOB_LAPLACE, JOB_SCORE };

typedef struct {
    int kind;
    const double* train;
    size_t n;
    const double* eval;
    size_t d;
    double h;
    size_t begin, end, out_base;
    double* out;
    size_t err_index;
    int status;
} fko_job;

/* oracle.cpp:36-51 (kde) and 103-118 (laplace) for rows [begin, end) */
static void run_kde_rows(fko_job* j) {
    for (size_t q = j->begin; q < j->end; ++q) {
        const double* y = j->eval + q * j->d;
        double acc = 0.0;
        if (j->kind == JOB_KDE) {
            for (size_t i = 0; i < j->n; ++i)
                acc += fko_gaussian_kernel(sq_dist(y, j->train + i * j->d, j->d), j->h, j->d);
        } else {
            for (size_t i = 0; i < j->n; ++i)
                acc += fko_laplace_corrected_kernel(sq_dist(y, j->train + i * j->d, j->d), j->h,
                                                    j->d);
        }
        j->out[q - j->out_base] = acc / (double)j->n;
    }
}

/* oracle.cpp:53-85 for rows [begin, end) */
static void run_score_rows(fko_job* j) {
    const size_t d = j->d;
    const double h = j->h;
    const double inv_2h2 = 1.0 / (2.0 * h * h);
    double numer_stack[64];
    double* numer = d <= 64 ? numer_stack : (double*)malloc(d * sizeof(double));
    for (size_t q = j->begin; q < j->end; ++q) {
        const double* y = j->eval + q * d;
        for (size_t k = 0; k < d; ++k) numer[k] = 0.0;
        double denom = 0.0;
        for (size_t i = 0; i < j->n; ++i) {
            const double* x = j->train + i * d;
            const double phi = exp(-sq_dist(y, x, d) * inv_2h2);
            denom += phi;
            for (size_t k = 0; k < d; ++k) numer[k] += -(y[k] - x[k]) * phi;
        }
        if (denom == 0.0) {
            j->status = FKO_SCORE_UNDERFLOW;
            j->err_index = q;
            break;
        }
        const double scale = 1.0 / (h * h * denom);
        double* o = j->out + (q - j->out_base) * d;
        for (size_t k = 0; k < d; ++k) o[k] = numer[k] * scale;
    }
    if (numer != numer_stack) free(numer);
}

static void* job_main(void* p) {
    fko_job* j = (fko_job*)p;
    if (j->kind == JOB_SCORE)
        run_score_rows(j);
    else
        run_kde_rows(j);
    return NULL;
}

static int run_sharded(int kind, const double* train, size_t n, const double* eval, size_t d,
                       double h, size_t begin, size_t end, int nthreads, double* out,
                       size_t* err_index) {
    if (nthreads < 1) nthreads = 1;
    const size_t rows = end - begin;
    if ((size_t)nthreads > rows) nthreads = rows ? (int)rows : 1;
    fko_job* jobs = (fko_job*)calloc((size_t)nthreads, sizeof(fko_job));
    pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
    for (int t = 0; t < nthreads; ++t) {
        jobs[t].kind = kind;
        jobs[t].train = train;
        jobs[t].n = n;
        jobs[t].eval = eval;
        jobs[t].d = d;
        jobs[t].h = h;
        jobs[t].begin = begin + rows * (size_t)t / (size_t)nthreads;
        jobs[t].end = begin + rows * (size_t)(t + 1) / (size_t)nthreads;
        jobs[t].out_base = begin;
        jobs[t].out = out;
        jobs[t].status = FKO_OK;
    }
    if (nthreads == 1) {
        job_main(&jobs[0]);
    } else {
        for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, job_main, &jobs[t]);
        for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    }
    int status = FKO_OK;
    for (int t = 0; t < nthreads; ++t) {
        if (jobs[t].status != FKO_OK) { /* first failing row, like a serial loop */
            status = jobs[t].status;
            if (err_index) *err_index = jobs[t].err_index;
            break;
        }
    }
    free(jobs);
    free(th);
    return status;
}

static int check_common(size_t n, size_t m, size_t d, double h, size_t begin, size_t end) {
    if (n == 0 || m == 0 || d == 0) return FKO_INVALID_ARGUMENT;
    if (!valid_h(h)) return FKO_INVALID_ARGUMENT;
    if (begin > end || end > m) return FKO_INVALID_ARGUMENT;
    return FKO_OK;
}

int fko_kde_naive(const double* train, size_t n, const double* queries, size_t m, size_t d,
                  double h, size_t row_begin, size_t row_end, int nthreads, double* out) {
    int s = check_common(n, m, d, h, row_begin, row_end);
    if (s) return s;
    return run_sharded(JOB_KDE, train, n, queries, d, h, row_begin, row_end, nthreads, out, NULL);
}

int fko_laplace_naive(const double* train, size_t n, const double* queries, size_t m, size_t d,
                      double h, size_t row_begin, size_t row_end, int nthreads, double* out) {
    int s = check_common(n, m, d, h, row_begin, row_end);
    if (s) return s;
    return run_sharded(JOB_LAPLACE, train, n, queries, d, h, row_begin, row_end, nthreads, out,
                       NULL);
}

int fko_score_naive(const double* train, size_t n, const double* eval, size_t m, size_t d,
                    double h_score, size_t row_begin, size_t row_end, int nthreads, double* out,
                    size_t* err_index) {
    int s = check_common(n, m, d, h_score, row_begin, row_end);
    if (s) return s;
    return run_sharded(JOB_SCORE, train, n, eval, d, h_score, row_begin, row_end, nthreads, out,
                       err_index);
}

/* oracle.cpp:87-101 */
int fko_sdkde_naive(const double* train, size_t n, const double* queries, size_t m, size_t d,
                    double h, double h_score, int nthreads, double* out, double* debiased,
                    size_t* err_index) {
    if (!valid_h(h) || !valid_h(h_score)) return FKO_INVALID_ARGUMENT;
    int s = check_common(n, m, d, h, 0, m);
    if (s) return s;
    double* scores = (double*)malloc(n * d * sizeof(double));
    double* deb = (double*)malloc(n * d * sizeof(double));
    s = fko_score_naive(train, n, train, n, d, h_score, 0, n, nthreads, scores, err_index);
    if (s == FKO_OK) {
        const double shift = 0.5 * h * h;
        for (size_t i = 0; i < n * d; ++i) deb[i] = train[i] + shift * scores[i];
        s = fko_kde_naive(deb, n, queries, m, d, h, 0, m, nthreads, out);
        if (debiased) memcpy(debiased, deb, n * d * sizeof(double));
    }
    free(scores);
    free(deb);
    return s;
}
