// C++ drop-in test of include/fkde_b200/engine.hpp (the facade over the C ABI).
// Reads like the reference's own tests (proj/tests/test_engine.cpp,
// test_estimator.cpp): same calls, same exception types.
//   ./test_facade          host-side validation only (no device needed)
//   ./test_facade gpu      also runs the engine on cuda:0 against a direct
//                          fp64 double loop (the oracle's formulation)
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "fkde_b200/engine.hpp"

using namespace fkde;

static int failures = 0;
#define EXPECT(cond)                                                     \
    do {                                                                 \
        if (!(cond)) {                                                   \
            std::printf("FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond); \
            ++failures;                                                  \
        }                                                                \
    } while (0)

template <typename E, typename F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static SampleSet random_set(std::size_t n, std::size_t d, unsigned seed, double scale = 1.0) {
    std::mt19937_64 g(seed);
    std::normal_distribution<double> nd(0.0, scale);
    std::vector<double> v(n * d);
    for (auto& x : v) x = nd(g);
    return SampleSet(std::move(v), n, d);
}

int main(int argc, char** argv) {
    const bool gpu = argc > 1 && std::strcmp(argv[1], "gpu") == 0;
    // ---- fkde::gpu::io: reference file formats (test_io.cpp:31-102) ----
    {
        const auto s = random_set(33, 4, 9, 1e3);
        const std::string bin = "/tmp/fkde_facade_io.bin", csv = "/tmp/fkde_facade_io.csv",
                          val = "/tmp/fkde_facade_io_v.json";
        gpu::io::write_samples_bin(s, bin);
        gpu::io::write_samples_csv(s, csv);
        const auto r1 = gpu::io::read_samples(bin), r2 = gpu::io::read_samples(csv, true);
        EXPECT(r1.n == 33 && r1.d == 4 && r1.values == s.values);
        EXPECT(r2.values == s.values);
        gpu::io::write_values(s.values, val, "json");
        EXPECT(gpu::io::read_values(val) == s.values);
        EXPECT(throws<IoError>([&] { gpu::io::read_samples("/tmp/definitely_missing_fkde.bin"); }));
        EXPECT(throws<InvalidArgumentError>([&] { gpu::io::write_values({1.0}, val, "xml"); }));
        std::remove(bin.c_str());
        std::remove(csv.c_str());
        std::remove(val.c_str());
    }
    // ---- validation (types.cpp / engine.cpp semantics), no device touched ----
    const auto a = random_set(10, 2, 1), b = random_set(10, 3, 2);
    const engine::TilePlan plan{64, 1024, 1, 1};
    EXPECT(throws<DimensionMismatchError>([&] {
        gpu::kde_flash(a, b, 1.0, KernelKind::Gaussian, true, plan);
    }));
    EXPECT(throws<InvalidArgumentError>([&] { gpu::score_flash(a, -1.0, plan); }));
    EXPECT(throws<InvalidArgumentError>([&] {
        gpu::kde_flash(a, a, 1.0, KernelKind::Gaussian, true, engine::TilePlan{0, 4, 0, 0});
    }));
    EstimatorConfig cfg;
    cfg.bandwidth = Bandwidth::uniform(0.5);
    cfg.tile_m = 0;
    EXPECT(throws<InvalidArgumentError>([&] { gpu::estimate(a, a, cfg); }));
    EXPECT(throws<InvalidArgumentError>([&] { SampleSet(std::vector<double>{1.0, NAN}, 2, 1); }));

    if (gpu) {
        // SD-KDE against a direct double loop (oracle.cpp:53-101 formulation)
        const std::size_t n = 300, m = 40, d = 16;
        const double h = 1.1;
        const auto tr = random_set(n, d, 7), q = random_set(m, d, 8);
        const auto res = gpu::sdkde_flash(tr, q, Bandwidth::uniform(h), plan);
        std::vector<double> deb(tr.values);
        for (std::size_t i = 0; i < n; ++i) {
            double den = 0, num[16] = {0};
            for (std::size_t j = 0; j < n; ++j) {
                double r2 = 0;
                for (std::size_t k = 0; k < d; ++k) {
                    const double df = tr.values[i * d + k] - tr.values[j * d + k];
                    r2 += df * df;
                }
                const double phi = std::exp(-r2 / (2 * h * h));
                den += phi;
                for (std::size_t k = 0; k < d; ++k) num[k] += -(tr.values[i * d + k] - tr.values[j * d + k]) * phi;
            }
            for (std::size_t k = 0; k < d; ++k) deb[i * d + k] += 0.5 * h * h * num[k] / (h * h * den);
        }
        double worst = 0;
        const double norm = std::pow(2 * M_PI, -0.5 * d) * std::pow(h, -double(d)) / n;
        for (std::size_t j = 0; j < m; ++j) {
            double acc = 0;
            for (std::size_t i = 0; i < n; ++i) {
                double r2 = 0;
                for (std::size_t k = 0; k < d; ++k) {
                    const double df = q.values[j * d + k] - deb[i * d + k];
                    r2 += df * df;
                }
                acc += std::exp(-r2 / (2 * h * h));
            }
            const double ref = acc * norm;
            worst = std::fmax(worst, std::fabs(res.values[j] - ref) / ref);
        }
        std::printf("sdkde max rel err %.3e\n", worst);
        EXPECT(worst < 1e-4);
        EXPECT(res.debiased_samples.has_value());
        cfg.tile_m = 64;
        cfg.method = Method::LaplaceKde;
        const auto lap = gpu::estimate(tr, q, cfg);
        EXPECT(lap.negative_mass_estimate.has_value());
        const auto acc = gpu::score_accumulate(tr, 0.7, plan);
        for (double p : acc.phi_sum) EXPECT(p >= 0.99);
    }
    std::printf("%s (%d failures)\n", failures ? "FAIL" : "OK", failures);
    return failures ? 1 : 0;
}
