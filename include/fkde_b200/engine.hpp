// fkde_b200/engine.hpp -- header-only C++ facade over the C ABI (fkde_gpu.h)
// that mirrors the reference's engine API (proj/core/include/fkde/engine.hpp:
// 15-76, estimator.hpp:9-10) so the B200 engine drops into the reference's
// call sites:
//
//   fkde::gpu::score_accumulate / score_flash / kde_flash / sdkde_flash /
//   pairwise_sq_dists_block / estimate, and fkde::gpu::io (the io.hpp file formats)
//
// Same argument meaning, same validation order, same exception types
// (errors.hpp:10-56): the facade validates on the host exactly like the
// reference (SampleSet::validate, Bandwidth::validate, TilePlan::make,
// check_pair), calls the ABI, and maps fkde_status back onto
// InvalidArgumentError / DimensionMismatchError / ScoreUnderflowError.
//
// Types: inside the reference's build define FKDE_B200_USE_REFERENCE_TYPES
// (and put proj/core/include on the include path) to use fkde::SampleSet etc.
// from fkde/types.hpp.  Without it, this header declares API-compatible
// minimal versions of those types in namespace fkde (for standalone use and
// for this repository's own C++ tests).
#pragma once

#include <cmath>
#include <cstddef>
#include <memory>
#include <mutex>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "../fkde_gpu.h"
#include "../fkde_io.h"

#ifdef FKDE_B200_USE_REFERENCE_TYPES
#include "fkde/engine.hpp"
#include "fkde/errors.hpp"
#include "fkde/types.hpp"
#else
namespace fkde {

class InvalidArgumentError : public std::invalid_argument {
public:
    using std::invalid_argument::invalid_argument;
};
class DimensionMismatchError : public InvalidArgumentError {
public:
    using InvalidArgumentError::InvalidArgumentError;
};
class IoError : public std::runtime_error {  // errors.hpp:53
public:
    using std::runtime_error::runtime_error;
};
class ScoreUnderflowError : public std::runtime_error {
public:
    ScoreUnderflowError(std::size_t index, const std::string& what)
        : std::runtime_error(what), index_(index) {}
    std::size_t index() const noexcept { return index_; }

private:
    std::size_t index_;
};

struct SampleSet {
    std::vector<double> values;
    std::size_t n = 0;
    std::size_t d = 0;
    SampleSet() = default;
    SampleSet(std::vector<double> data, std::size_t n_rows, std::size_t n_cols)
        : values(std::move(data)), n(n_rows), d(n_cols) {
        validate();
    }
    static SampleSet zeros(std::size_t n_rows, std::size_t n_cols) {
        SampleSet s;
        s.values.assign(n_rows * n_cols, 0.0);
        s.n = n_rows;
        s.d = n_cols;
        return s;
    }
    const double* data() const noexcept { return values.data(); }
    double* data() noexcept { return values.data(); }
    void validate() const {  // types.cpp:21-33
        if (n == 0 || d == 0) throw InvalidArgumentError("SampleSet: n and d must be >= 1");
        if (values.size() != n * d)
            throw InvalidArgumentError("SampleSet: storage size does not match n*d");
        for (double v : values)
            if (!std::isfinite(v)) throw InvalidArgumentError("SampleSet: non-finite entry");
    }
};

enum class Method { Kde, Sdkde, LaplaceKde };
enum class EngineKind { Naive, Flash };
enum class KernelKind { Gaussian, LaplaceCorrected };

struct Bandwidth {
    double h = 1.0;
    double h_score = 1.0;
    static Bandwidth uniform(double h) { return {h, h}; }
    static Bandwidth half_variance_score(double h) { return {h, h / std::sqrt(2.0)}; }
    void validate() const {  // types.cpp:65-72
        if (!(h > 0.0) || !std::isfinite(h))
            throw InvalidArgumentError("Bandwidth: h must be positive and finite");
        if (!(h_score > 0.0) || !std::isfinite(h_score))
            throw InvalidArgumentError("Bandwidth: h_score must be positive and finite");
    }
};

struct EstimatorConfig {
    Method method = Method::Kde;
    Bandwidth bandwidth;
    EngineKind engine = EngineKind::Flash;
    std::size_t tile_m = 64;
    std::size_t tile_n = 1024;
    bool fused = true;
    std::size_t threads = 0;
    bool fast_accumulation = false;
    void validate() const {  // types.cpp:74-79
        bandwidth.validate();
        if (tile_m == 0 || tile_n == 0)
            throw InvalidArgumentError("EstimatorConfig: tile_m and tile_n must be >= 1");
    }
};

struct DensityResult {
    std::vector<double> values;
    std::optional<double> negative_mass_estimate;
    std::optional<SampleSet> debiased_samples;
};

namespace engine {
struct TilePlan {
    std::size_t tile_m = 64, tile_n = 1024, n_tiles_m = 0, n_tiles_n = 0;
    static TilePlan make(std::size_t n_queries, std::size_t n_train, std::size_t tile_m,
                         std::size_t tile_n) {  // engine.cpp:248-259
        if (tile_m == 0 || tile_n == 0) throw InvalidArgumentError("TilePlan: tile sizes must be >= 1");
        TilePlan p;
        p.tile_m = tile_m;
        p.tile_n = tile_n;
        p.n_tiles_m = n_queries == 0 ? 0 : (n_queries + tile_m - 1) / tile_m;
        p.n_tiles_n = n_train == 0 ? 0 : (n_train + tile_n - 1) / tile_n;
        return p;
    }
};
struct ScoreAccumulator {
    std::vector<double> phi_sum;
    SampleSet weighted_sum;
};
struct EngineOptions {
    std::size_t threads = 0;
    bool fast_accumulation = false;
};
}  // namespace engine
}  // namespace fkde
#endif

namespace fkde {
namespace gpu {

// RAII owner of an fkde_gpu_ctx (streams, device workspaces, NCCL comm).
class Context {
public:
    explicit Context(const std::vector<int>& devices = {0}) {
        const int rc = fkde_gpu_create(devices.data(), static_cast<int>(devices.size()), &ctx_);
        if (rc != FKDE_OK) throw std::runtime_error("fkde_gpu_create failed: status " + std::to_string(rc));
    }
    Context(int device, int rank, int world, const unsigned char nccl_id[128]) {
        const int rc = fkde_gpu_create_rank(device, rank, world, nccl_id, &ctx_);
        if (rc != FKDE_OK) throw std::runtime_error("fkde_gpu_create_rank failed: status " + std::to_string(rc));
    }
    ~Context() { fkde_gpu_destroy(ctx_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    fkde_gpu_ctx* get() const { return ctx_; }

    // process-wide default context on device 0 (created on first use, after the
    // host-side validation of the call that needs it)
    static Context& instance() {
        static std::once_flag once;
        static std::unique_ptr<Context> ctx;
        std::call_once(once, [] { ctx = std::make_unique<Context>(); });
        return *ctx;
    }

private:
    fkde_gpu_ctx* ctx_ = nullptr;
};

namespace detail {
inline void check(fkde_gpu_ctx* ctx, int rc, std::size_t err_index = 0) {
    if (rc == FKDE_OK) return;
    const std::string msg = fkde_gpu_last_error(ctx);
    switch (rc) {
        case FKDE_INVALID_ARGUMENT:
        case FKDE_NON_FINITE:
        case FKDE_UNSUPPORTED_D:
            throw InvalidArgumentError(msg);
        case FKDE_DIMENSION_MISMATCH:
            throw DimensionMismatchError(msg);
        case FKDE_SCORE_UNDERFLOW:
            throw ScoreUnderflowError(err_index, msg);
        default:
            throw std::runtime_error("fkde_gpu: status " + std::to_string(rc) + ": " + msg);
    }
}
// TilePlan::make's validation (engine.cpp:248-252), without needing the
// reference's engine.cpp (which requires Eigen) at link time
inline void check_plan(std::size_t tile_m, std::size_t tile_n) {
    if (tile_m == 0 || tile_n == 0) throw InvalidArgumentError("TilePlan: tile sizes must be >= 1");
}
inline void check_pair(const SampleSet& a, const SampleSet& b) {  // engine.cpp:27-34
    a.validate();
    b.validate();
    if (a.d != b.d)
        throw DimensionMismatchError("engine: train.d=" + std::to_string(a.d) +
                                     " != queries.d=" + std::to_string(b.d));
}
}  // namespace detail

// engine.hpp:46-49
inline SampleSet pairwise_sq_dists_block(const SampleSet& a, const SampleSet& b,
                                         Context* ctx_ = nullptr) {
    detail::check_pair(a, b);
    Context& ctx = ctx_ ? *ctx_ : Context::instance();
    SampleSet out = SampleSet::zeros(a.n, b.n);
    detail::check(ctx.get(), fkde_gpu_pairwise_sq_dists(ctx.get(), a.data(), a.n, b.data(), b.n,
                                                        a.d, out.data()));
    return out;
}

// engine.hpp:58-59
inline engine::ScoreAccumulator score_accumulate(const SampleSet& train, double h_score,
                                                 const engine::TilePlan& plan,
                                                 const engine::EngineOptions& = {},
                                                 Context* ctx_ = nullptr) {
    train.validate();
    Bandwidth{h_score, h_score}.validate();
    detail::check_plan(plan.tile_m, plan.tile_n);
    Context& ctx = ctx_ ? *ctx_ : Context::instance();
    engine::ScoreAccumulator acc;
    acc.phi_sum.assign(train.n, 0.0);
    acc.weighted_sum = SampleSet::zeros(train.n, train.d);
    detail::check(ctx.get(), fkde_gpu_score_accumulate(ctx.get(), train.data(), train.n, train.d,
                                                       h_score, acc.phi_sum.data(),
                                                       acc.weighted_sum.data()));
    return acc;
}

// engine.hpp:63-64
inline SampleSet score_flash(const SampleSet& train, double h_score, const engine::TilePlan& plan,
                             const engine::EngineOptions& = {}, Context* ctx_ = nullptr) {
    train.validate();
    Bandwidth{h_score, h_score}.validate();
    detail::check_plan(plan.tile_m, plan.tile_n);
    Context& ctx = ctx_ ? *ctx_ : Context::instance();
    SampleSet scores = SampleSet::zeros(train.n, train.d);
    std::size_t idx = 0;
    detail::check(ctx.get(), fkde_gpu_score(ctx.get(), train.data(), train.n, train.d, h_score,
                                            scores.data(), &idx),
                  idx);
    return scores;
}

// engine.hpp:70-72
inline DensityResult kde_flash(const SampleSet& train, const SampleSet& queries, double h,
                               KernelKind kernel, bool fused, const engine::TilePlan& plan,
                               const engine::EngineOptions& = {},
                               Context* ctx_ = nullptr) {
    detail::check_pair(train, queries);
    Bandwidth{h, h}.validate();
    detail::check_plan(plan.tile_m, plan.tile_n);
    Context& ctx = ctx_ ? *ctx_ : Context::instance();
    DensityResult r;
    r.values.assign(queries.n, 0.0);
    const int k = kernel == KernelKind::Gaussian ? FKDE_KERNEL_GAUSSIAN : FKDE_KERNEL_LAPLACE_CORRECTED;
    detail::check(ctx.get(), fkde_gpu_kde(ctx.get(), train.data(), train.n, queries.data(),
                                          queries.n, train.d, h, k, fused ? 1 : 0,
                                          r.values.data()));
    return r;
}

// engine.hpp:74-76
inline DensityResult sdkde_flash(const SampleSet& train, const SampleSet& queries,
                                 const Bandwidth& bw, const engine::TilePlan& plan,
                                 const engine::EngineOptions& = {},
                                 Context* ctx_ = nullptr) {
    detail::check_pair(train, queries);
    bw.validate();
    detail::check_plan(plan.tile_m, plan.tile_n);
    Context& ctx = ctx_ ? *ctx_ : Context::instance();
    DensityResult r;
    r.values.assign(queries.n, 0.0);
    SampleSet deb = SampleSet::zeros(train.n, train.d);
    std::size_t idx = 0;
    detail::check(ctx.get(), fkde_gpu_sdkde(ctx.get(), train.data(), train.n, queries.data(),
                                            queries.n, train.d, bw.h, bw.h_score,
                                            r.values.data(), deb.data(), &idx),
                  idx);
    r.debiased_samples = std::move(deb);
    return r;
}

// estimator.cpp:52-60 for the B200 engine (EngineKind::Flash -> GPU)
inline DensityResult estimate(const SampleSet& train, const SampleSet& queries,
                              const EstimatorConfig& config, Context* ctx_ = nullptr) {
    config.validate();
    detail::check_plan(config.tile_m, config.tile_n);
    const engine::TilePlan plan{config.tile_m, config.tile_n,
                                (queries.n + config.tile_m - 1) / config.tile_m,
                                (train.n + config.tile_n - 1) / config.tile_n};
    const engine::EngineOptions opts{config.threads, config.fast_accumulation};
    switch (config.method) {
        case Method::Kde:
            return kde_flash(train, queries, config.bandwidth.h, KernelKind::Gaussian, true, plan,
                             opts, ctx_);
        case Method::Sdkde:
            return sdkde_flash(train, queries, config.bandwidth, plan, opts, ctx_);
        case Method::LaplaceKde: {
            DensityResult r = kde_flash(train, queries, config.bandwidth.h,
                                        KernelKind::LaplaceCorrected, config.fused, plan, opts, ctx_);
            double acc = 0.0;  // estimator.cpp:14-20
            for (double v : r.values) acc += v < 0.0 ? -v : 0.0;
            r.negative_mass_estimate = acc / static_cast<double>(r.values.size());
            return r;
        }
    }
    throw InvalidArgumentError("estimate: unknown method");
}

// fkde::io (io.hpp:11-38) over fkde_io.h: same formats byte for byte, same
// exceptions; read_samples can stage the file through page-locked memory.
namespace io {
namespace detail {
inline void check(int rc) {
    if (rc == FKDE_IO_OK) return;
    const std::string msg = fkde_io_last_error();
    if (rc == FKDE_IO_INVALID_ARGUMENT) throw InvalidArgumentError(msg);
    throw IoError(msg);
}
}  // namespace detail

inline SampleSet read_samples(const std::string& path, bool pinned = false) {  // io.cpp:177-190
    double* p = nullptr;
    std::size_t n = 0, d = 0;
    int pin = pinned ? 1 : 0;
    detail::check(fkde_io_read_samples(path.c_str(), &p, &n, &d, &pin));
    std::vector<double> v(p, p + n * d);
    fkde_io_free(p, pin);
    return SampleSet(std::move(v), n, d);
}
inline void write_samples_bin(const SampleSet& s, const std::string& path) {
    detail::check(fkde_io_write_samples_bin(path.c_str(), s.values.data(), s.n, s.d));
}
inline void write_samples_csv(const SampleSet& s, const std::string& path) {
    detail::check(fkde_io_write_samples_csv(path.c_str(), s.values.data(), s.n, s.d));
}
inline void write_values(const std::vector<double>& values, const std::string& path,
                         const std::string& format) {
    detail::check(fkde_io_write_values(path.c_str(), values.data(), values.size(), format.c_str()));
}
inline std::vector<double> read_values(const std::string& path) {
    double* p = nullptr;
    std::size_t m = 0;
    detail::check(fkde_io_read_values(path.c_str(), &p, &m));
    std::vector<double> v(p, p + m);
    fkde_io_free(p, 0);
    return v;
}
}  // namespace io

}  // namespace gpu
}  // namespace fkde
