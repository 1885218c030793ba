// host_fixtures.cpp -- synthetic-input generators and bandwidth rules, host
// side, so the engine's bench/CLI produce exactly the reference's inputs
// (the reference's RNG contract is "bitwise reproducible for a fixed seed",
// rng.hpp:45-51, mixture.hpp:24-25).  Not on the device path.
//
//   fkde_host_mix64            <- fkde::mix64                 rng.cpp:8-13
//   fkde_host_random_gaussian  <- testutil::random_gaussian   test_util.hpp:12-20
//   fkde_host_sample_mixture   <- fkde::bench::sample_mixture mixture.cpp:40-67
//   fkde_host_mean_stddev / fkde_host_silverman_bandwidth / fkde_host_sdkde_bandwidth
//                              <- bandwidth.cpp:9-58
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <random>
#include <thread>
#include <vector>

namespace {

uint64_t mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

// mt19937_64 with the reference's hand-rolled uniform / Box-Muller draws
class Rng {
public:
    explicit Rng(uint64_t seed, uint64_t stream = 0) : gen_(mix64(seed ^ mix64(stream + 1))) {}
    double uniform01() { return static_cast<double>(gen_() >> 11) * 0x1.0p-53; }
    double normal() {
        if (has_spare_) {
            has_spare_ = false;
            return spare_;
        }
        double u1;
        do {
            u1 = uniform01();
        } while (u1 == 0.0);
        const double u2 = uniform01();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double theta = 2.0 * 3.141592653589793238462643383279502884 * u2;
        spare_ = r * std::sin(theta);
        has_spare_ = true;
        return r * std::cos(theta);
    }

private:
    std::mt19937_64 gen_;
    double spare_ = 0.0;
    bool has_spare_ = false;
};

// bandwidth.cpp:9-30, bitwise: each column is still summed in row order (the
// same rounding sequence), but all columns advance together in one row-major
// sweep -- the reference's column-at-a-time loop walks the n x d array d
// times with a stride of d doubles, which at n = 2^20 costs ~0.2 s of cache
// misses per call and sat inside every timed estimate of the runtime sweep
double mean_stddev(const double* x, size_t n, size_t d) {
    constexpr size_t kCols = 64;
    double acc = 0.0;
    for (size_t j0 = 0; j0 < d; j0 += kCols) {
        const size_t w = d - j0 < kCols ? d - j0 : kCols;
        double mean[kCols], ssq[kCols];
        for (size_t j = 0; j < w; ++j) mean[j] = ssq[j] = 0.0;
        for (size_t i = 0; i < n; ++i)
            for (size_t j = 0; j < w; ++j) mean[j] += x[i * d + j0 + j];
        for (size_t j = 0; j < w; ++j) mean[j] /= static_cast<double>(n);
        for (size_t i = 0; i < n; ++i)
            for (size_t j = 0; j < w; ++j) {
                const double diff = x[i * d + j0 + j] - mean[j];
                ssq[j] += diff * diff;
            }
        for (size_t j = 0; j < w; ++j) acc += std::sqrt(ssq[j] / static_cast<double>(n - 1));
    }
    return acc / static_cast<double>(d);
}

}  // namespace

extern "C" {

uint64_t fkde_host_mix64(uint64_t x) { return mix64(x); }

void fkde_host_random_gaussian(size_t n, size_t d, uint64_t seed, double scale, double* out) {
    Rng rng(seed);
    for (size_t i = 0; i < n * d; ++i) out[i] = scale * rng.normal();
}

int fkde_host_sample_mixture(const double* weights, const double* means, const double* sigmas,
                             size_t k, size_t d, size_t n, uint64_t seed, double* out) {
    if (k == 0 || d == 0 || n == 0) return 1;
    Rng rng(seed, 0);
    for (size_t i = 0; i < n; ++i) {
        const double u = rng.uniform01();
        size_t comp = k - 1;
        double cum = 0.0;
        for (size_t c = 0; c < k; ++c) {
            cum += weights[c];
            if (u < cum) {
                comp = c;
                break;
            }
        }
        for (size_t kk = 0; kk < d; ++kk)
            out[i * d + kk] = means[comp * d + kk] + sigmas[comp] * rng.normal();
    }
    return 0;
}

double fkde_host_mean_stddev(const double* x, size_t n, size_t d) { return mean_stddev(x, n, d); }

double fkde_host_silverman_prefactor(size_t d) {
    const double dd = static_cast<double>(d);
    return std::pow(4.0 / (dd + 2.0), 1.0 / (dd + 4.0));
}

double fkde_host_silverman_bandwidth(const double* x, size_t n, size_t d) {
    const double dd = static_cast<double>(d);
    return mean_stddev(x, n, d) * fkde_host_silverman_prefactor(d) *
           std::pow(static_cast<double>(n), -1.0 / (dd + 4.0));
}

double fkde_host_sdkde_bandwidth(const double* x, size_t n, size_t d, double c) {
    const double dd = static_cast<double>(d);
    return c * mean_stddev(x, n, d) * std::pow(static_cast<double>(n), -1.0 / (dd + 8.0));
}

}  // extern "C"
