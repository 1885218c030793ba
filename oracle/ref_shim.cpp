// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrappers around the reference's OWN oracle, RNG, mixture sampler
// and bandwidth rules, compiled here from the unmodified sources under
// /root/reference/proj/core/src by oracle/Makefile into
// oracle/_ref/libfkde_ref.so.  This file contains no estimator arithmetic; it
// only marshals plain pointers into fkde::SampleSet and back, so the tests can
// run the reference itself next to the C restatement (fkde_oracle.c) and
// next to the GPU engine.  Wrapped interfaces:
//   fkde::oracle::{kde_naive, score_naive, sdkde_naive, laplace_naive}  (oracle.hpp:10-25)
//   fkde::{gaussian_kernel, laplace_corrected_kernel, gaussian_norm_const} (kernels.hpp)
//   fkde::Rng / mix64 (rng.hpp), fkde::bench::sample_mixture (mixture.hpp:25)
//   fkde::{mean_stddev, silverman_bandwidth, sdkde_bandwidth, silverman_prefactor}
//   fkde::io::{write_samples_bin, write_samples_csv, write_values} (io.hpp) and
//   fkde::bench::{load_mixture, mixture_hash, mixture_pdf} (mixture.hpp),
//   fkde::perfmodel::{flops_nd, flops_1d, bytes_nd, bytes_1d, bytes_linear,
//   intensity_asymptotic} (perfmodel.hpp) -- the §8f rows' file formats and models,
//   fkde::bench::error_metrics (metrics.hpp:31-32, metrics.cpp:47-120) with the
//   estimator supplied by the caller (a C callback: the GPU engine or the oracle)
#include <cstring>
#include <exception>
#include <thread>
#include <vector>

#include "fkde/bandwidth.hpp"
#include "fkde/errors.hpp"
#include "fkde/io.hpp"
#include "fkde/perfmodel.hpp"
#include "fkde/kernels.hpp"
#include "fkde/metrics.hpp"
#include "fkde/mixture.hpp"
#include "fkde/oracle.hpp"
#include "fkde/rng.hpp"
#include "fkde/types.hpp"

using namespace fkde;

namespace {

SampleSet make_set(const double* p, std::size_t n, std::size_t d) {
    return SampleSet(std::vector<double>(p, p + n * d), n, d);
}

// 0 ok, 1 invalid argument, 2 dimension mismatch, 3 score underflow, 9 other
int map_exception(std::size_t* err_index) {
    try {
        throw;
    } catch (const ScoreUnderflowError& e) {
        if (err_index) *err_index = e.index();
        return 3;
    } catch (const DimensionMismatchError&) {
        return 2;
    } catch (const InvalidArgumentError&) {
        return 1;
    } catch (...) {
        return 9;
    }
}

// Evaluate rows [b, e) of `eval` by calling the reference function on that
// row block (each row is a pure function of its inputs, oracle.cpp:36-118),
// split into contiguous shards over `threads` std::threads.
template <typename F>
int sharded(const double* eval, std::size_t b, std::size_t e, std::size_t d, int threads,
            std::size_t out_stride, double* out, std::size_t* err_index, F&& fn) {
    if (threads < 1) threads = 1;
    const std::size_t rows = e - b;
    if (static_cast<std::size_t>(threads) > rows) threads = rows ? static_cast<int>(rows) : 1;
    std::vector<int> status(threads, 0);
    std::vector<std::size_t> idx(threads, 0);
    auto work = [&](int t) {
        const std::size_t lo = b + rows * t / threads, hi = b + rows * (t + 1) / threads;
        if (lo == hi) return;
        try {
            SampleSet block = make_set(eval + lo * d, hi - lo, d);
            std::vector<double> res = fn(block);
            std::memcpy(out + (lo - b) * out_stride, res.data(), res.size() * sizeof(double));
        } catch (...) {
            status[t] = map_exception(&idx[t]);
            idx[t] += lo;
        }
    };
    if (threads == 1) {
        work(0);
    } else {
        std::vector<std::thread> pool;
        for (int t = 0; t < threads; ++t) pool.emplace_back(work, t);
        for (auto& th : pool) th.join();
    }
    for (int t = 0; t < threads; ++t) {
        if (status[t]) {
            if (err_index) *err_index = idx[t];
            return status[t];
        }
    }
    return 0;
}

}  // namespace

extern "C" {

std::uint64_t fkr_mix64(std::uint64_t x) { return mix64(x); }

void fkr_random_gaussian(std::size_t n, std::size_t d, std::uint64_t seed, double scale,
                         double* out) {
    Rng rng(seed);
    for (std::size_t i = 0; i < n * d; ++i) out[i] = scale * rng.normal();
}

void fkr_uniform01(std::uint64_t seed, std::uint64_t stream, std::size_t count, double* out) {
    Rng rng(seed, stream);
    for (std::size_t i = 0; i < count; ++i) out[i] = rng.uniform01();
}

int fkr_sample_mixture(const double* weights, const double* means, const double* sigmas,
                       std::size_t k, std::size_t d, std::size_t n, std::uint64_t seed,
                       double* out) {
    try {
        bench::GaussianMixture mix;
        mix.weights.assign(weights, weights + k);
        mix.sigmas.assign(sigmas, sigmas + k);
        mix.means = make_set(means, k, d);
        SampleSet s = bench::sample_mixture(mix, n, seed);
        std::memcpy(out, s.data(), n * d * sizeof(double));
        return 0;
    } catch (...) {
        return map_exception(nullptr);
    }
}

double fkr_gaussian_norm_const(double h, std::size_t d) { return gaussian_norm_const(h, d); }
double fkr_gaussian_kernel(double r2, double h, std::size_t d) {
    return gaussian_kernel(r2, h, d);
}
double fkr_laplace_corrected_kernel(double r2, double h, std::size_t d) {
    return laplace_corrected_kernel(r2, h, d);
}

double fkr_mean_stddev(const double* x, std::size_t n, std::size_t d) {
    return mean_stddev(make_set(x, n, d));
}
double fkr_silverman_prefactor(std::size_t d) { return silverman_prefactor(d); }
double fkr_silverman_bandwidth(const double* x, std::size_t n, std::size_t d) {
    return silverman_bandwidth(make_set(x, n, d));
}
double fkr_sdkde_bandwidth(const double* x, std::size_t n, std::size_t d, double c) {
    return sdkde_bandwidth(make_set(x, n, d), c);
}

int fkr_kde_naive(const double* train, std::size_t n, const double* queries, std::size_t m,
                  std::size_t d, double h, std::size_t b, std::size_t e, int threads,
                  double* out) {
    try {
        const SampleSet tr = make_set(train, n, d);
        return sharded(queries, b, e, d, threads, 1, out, nullptr,
                       [&](const SampleSet& q) { return oracle::kde_naive(tr, q, h).values; });
    } catch (...) {
        return map_exception(nullptr);
    }
    (void)m;
}

int fkr_laplace_naive(const double* train, std::size_t n, const double* queries, std::size_t m,
                      std::size_t d, double h, std::size_t b, std::size_t e, int threads,
                      double* out) {
    try {
        const SampleSet tr = make_set(train, n, d);
        return sharded(queries, b, e, d, threads, 1, out, nullptr,
                       [&](const SampleSet& q) { return oracle::laplace_naive(tr, q, h).values; });
    } catch (...) {
        return map_exception(nullptr);
    }
    (void)m;
}

int fkr_score_naive(const double* train, std::size_t n, const double* eval, std::size_t m,
                    std::size_t d, double h_score, std::size_t b, std::size_t e, int threads,
                    double* out, std::size_t* err_index) {
    try {
        const SampleSet tr = make_set(train, n, d);
        return sharded(eval, b, e, d, threads, d, out, err_index, [&](const SampleSet& q) {
            return oracle::score_naive(tr, q, h_score).values;
        });
    } catch (...) {
        return map_exception(err_index);
    }
    (void)m;
}

// Single-threaded full pipeline, exactly oracle::sdkde_naive.
int fkr_sdkde_naive(const double* train, std::size_t n, const double* queries, std::size_t m,
                    std::size_t d, double h, double h_score, double* out, double* debiased,
                    std::size_t* err_index) {
    try {
        const auto r = oracle::sdkde_naive(make_set(train, n, d), make_set(queries, m, d),
                                           Bandwidth{h, h_score});
        std::memcpy(out, r.values.data(), m * sizeof(double));
        if (debiased) std::memcpy(debiased, r.debiased_samples->data(), n * d * sizeof(double));
        return 0;
    } catch (...) {
        return map_exception(err_index);
    }
}

// ---- §8f rows: file formats, mixture config, perf model ----------------------
int fkr_write_samples_bin(const char* path, const double* v, std::size_t n, std::size_t d) {
    try {
        io::write_samples_bin(make_set(v, n, d), path);
        return 0;
    } catch (...) {
        return map_exception(nullptr);
    }
}
int fkr_write_samples_csv(const char* path, const double* v, std::size_t n, std::size_t d) {
    try {
        io::write_samples_csv(make_set(v, n, d), path);
        return 0;
    } catch (...) {
        return map_exception(nullptr);
    }
}
int fkr_write_values(const char* path, const double* v, std::size_t m, const char* format) {
    try {
        io::write_values(std::vector<double>(v, v + m), path, format);
        return 0;
    } catch (...) {
        return map_exception(nullptr);
    }
}
// n, d of a sample file (0 on error); values copied when out != nullptr
int fkr_read_samples(const char* path, double* out, std::size_t cap, std::size_t* n, std::size_t* d) {
    try {
        const SampleSet s = io::read_samples(path);
        *n = s.n;
        *d = s.d;
        if (out && cap >= s.values.size()) std::memcpy(out, s.values.data(), s.values.size() * 8);
        return 0;
    } catch (const IoError&) {
        return 8;
    } catch (...) {
        return map_exception(nullptr);
    }
}
int fkr_read_values(const char* path, double* out, std::size_t cap, std::size_t* m) {
    try {
        const std::vector<double> v = io::read_values(path);
        *m = v.size();
        if (out && cap >= v.size()) std::memcpy(out, v.data(), v.size() * 8);
        return 0;
    } catch (const IoError&) {
        return 8;
    } catch (...) {
        return map_exception(nullptr);
    }
}
std::uint64_t fkr_mixture_hash(const char* config_path) {
    return bench::mixture_hash(bench::load_mixture(config_path));
}
int fkr_mixture_pdf(const char* config_path, const double* x, std::size_t n, double* out) {
    try {
        const auto mix = bench::load_mixture(config_path);
        const auto v = bench::mixture_pdf(mix, make_set(x, n, mix.dim()));
        std::memcpy(out, v.data(), n * 8);
        return 0;
    } catch (...) {
        return map_exception(nullptr);
    }
}
// error_metrics(estimate_at, mixture, mode, n_eval, seed): the estimator is
// the callback est(points, n, d, out, user) -> 0 on success.  out6 = {mise,
// mise_se, miae, miae_se, negative_mass, negative_mass_se}.
typedef int (*fkr_estimate_cb)(const double* pts, std::size_t n, std::size_t d, double* out,
                               void* user);
int fkr_error_metrics(const char* config_path, int grid, std::size_t n_eval, std::uint64_t seed,
                      fkr_estimate_cb est, void* user, double* out6) {
    try {
        const auto mix = bench::load_mixture(config_path);
        const bench::EstimateFn fn = [&](const SampleSet& pts) {
            std::vector<double> v(pts.n);
            if (est(pts.values.data(), pts.n, pts.d, v.data(), user) != 0)
                throw std::runtime_error("estimate callback failed");
            return v;
        };
        const auto r = bench::error_metrics(
            fn, mix, grid ? bench::ErrorMode::Grid1D : bench::ErrorMode::ImportanceMC, n_eval, seed);
        const double o[6] = {r.mise, r.mise_se, r.miae, r.miae_se, r.negative_mass,
                             r.negative_mass_se};
        std::memcpy(out6, o, sizeof(o));
        return 0;
    } catch (...) {
        return map_exception(nullptr);
    }
}
double fkr_flops_nd(std::size_t d, std::size_t k) { return perfmodel::flops_nd(d, k); }
double fkr_flops_1d(std::size_t k) { return perfmodel::flops_1d(k); }
double fkr_bytes_nd(std::size_t d, std::size_t k, std::size_t tm, std::size_t tn) {
    return perfmodel::bytes_nd(d, k, tm, tn);
}
double fkr_bytes_1d(std::size_t k) { return perfmodel::bytes_1d(k); }
double fkr_bytes_linear(std::size_t d, std::size_t k) { return perfmodel::bytes_linear(d, k); }
double fkr_intensity_asymptotic(std::size_t d) { return perfmodel::intensity_asymptotic(d); }

}  // extern "C"
