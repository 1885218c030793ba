// fkde-b200 -- command-line front end of the B200 engine, the drop-in for the
// reference's `fkde` tool (proj/tools/src/main.cpp) on the estimator path:
//
//   gen       draw mixture samples          main.cpp:87-108   (FKDE bin / CSV + .meta.json)
//   estimate  density at query points        main.cpp:110-152  (--engine gpu|flash: B200 engine)
//   compare   gate two value files           main.cpp:154-188
//   bench     runtime / error sweeps         main.cpp:225-320, sweep.cpp:105-241 (same CSV/JSON schema)
//   model     analytic FLOP/byte report      main.cpp:190-215, perfmodel.cpp (+ B200 presets)
//
// Same flags, same outputs, same exit codes (0 ok, 1 comparison/strict
// failure, 2 usage, 3 file I/O, 4 numeric or dimension error).  The CPU
// engines (naive, the Eigen flash engine) are not part of this build:
// `--engine flash` selects the B200 engine that replaces it, `naive` is a
// usage error.  Inputs are read into pinned host memory (fkde_io.h) and handed
// to the engine through the C ABI (fkde_gpu.h) without further copies.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <memory>
#include <numbers>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include <json.hpp>

#include "fkde_gpu.h"
#include "fkde_io.h"

namespace {

constexpr int kExitOk = 0, kExitFail = 1, kExitUsage = 2, kExitIo = 3, kExitNumeric = 4;

struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct IoError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct NumericError : std::runtime_error {  // InvalidArgument / DimensionMismatch / ScoreUnderflow
    using std::runtime_error::runtime_error;
};

// ---------------------------------------------------------------- arguments
struct Args {
    std::vector<std::string> pos;
    std::map<std::string, std::string> opt;
    std::vector<std::string> flags;

    bool has(const std::string& k) const { return opt.count(k) > 0; }
    bool flag(const std::string& k) const {
        return std::find(flags.begin(), flags.end(), k) != flags.end();
    }
    std::string str(const std::string& k, const std::string& def = "") const {
        auto it = opt.find(k);
        return it == opt.end() ? def : it->second;
    }
    std::string req(const std::string& k) const {
        if (!has(k)) throw UsageError(k + " is required");
        return opt.at(k);
    }
};

Args parse(int argc, char** argv, int first, const std::vector<std::string>& flag_names) {
    Args a;
    for (int i = first; i < argc; ++i) {
        std::string s = argv[i];
        if (s.rfind("--", 0) == 0) {
            std::string key = s, val;
            const auto eq = s.find('=');
            if (eq != std::string::npos) {
                key = s.substr(0, eq);
                val = s.substr(eq + 1);
                a.opt[key] = val;
                continue;
            }
            if (std::find(flag_names.begin(), flag_names.end(), key) != flag_names.end()) {
                a.flags.push_back(key);
                continue;
            }
            if (i + 1 >= argc) throw UsageError(key + " needs a value");
            a.opt[key] = argv[++i];
        } else {
            a.pos.push_back(s);
        }
    }
    return a;
}

double to_double(const std::string& s, const std::string& what) {
    try {
        size_t used = 0;
        const double v = std::stod(s, &used);
        if (used != s.size()) throw std::invalid_argument(s);
        return v;
    } catch (const std::exception&) {
        throw UsageError(what + ": not a number: " + s);
    }
}
uint64_t to_u64(const std::string& s, const std::string& what) {
    if (s.empty() || s[0] == '-') throw UsageError(what + ": not a non-negative integer: " + s);
    try {
        size_t used = 0;
        const unsigned long long v = std::stoull(s, &used);
        if (used != s.size()) throw std::invalid_argument(s);
        return v;
    } catch (const std::exception&) {
        throw UsageError(what + ": not a non-negative integer: " + s);
    }
}
size_t positive(const std::string& s, const std::string& what) {
    const uint64_t v = to_u64(s, what);
    if (v == 0) throw UsageError(what + " must be positive");
    return static_cast<size_t>(v);
}
std::vector<std::string> split_list(const std::string& s) {
    std::vector<std::string> out;
    std::string cur;
    for (char c : s) {
        if (c == ',') {
            out.push_back(cur);
            cur.clear();
        } else {
            cur.push_back(c);
        }
    }
    out.push_back(cur);
    return out;
}
void member(const std::string& v, const std::vector<std::string>& allowed, const std::string& what) {
    if (std::find(allowed.begin(), allowed.end(), v) == allowed.end())
        throw UsageError(what + ": '" + v + "' not in {" + [&] {
            std::string j;
            for (auto& x : allowed) j += (j.empty() ? "" : ", ") + x;
            return j;
        }() + "}");
}

// ---------------------------------------------------------------- samples
struct Samples {  // host buffer from fkde_io_read_samples / fkde_io_alloc (pinned when possible)
    double* p = nullptr;
    bool pinned = false;
    size_t n = 0, d = 0;
    Samples() = default;
    Samples(const Samples&) = delete;
    Samples& operator=(const Samples&) = delete;
    Samples(Samples&& o) noexcept { *this = std::move(o); }
    Samples& operator=(Samples&& o) noexcept {
        std::swap(p, o.p);
        std::swap(pinned, o.pinned);
        std::swap(n, o.n);
        std::swap(d, o.d);
        return *this;
    }
    ~Samples() { fkde_io_free(p, pinned ? 1 : 0); }
    const double* data() const { return p; }
};

Samples read_samples(const std::string& path) {
    Samples s;
    double* p = nullptr;
    int pinned = 1;
    const int rc = fkde_io_read_samples(path.c_str(), &p, &s.n, &s.d, &pinned);
    if (rc == FKDE_IO_INVALID_ARGUMENT) throw NumericError(fkde_io_last_error());
    if (rc != FKDE_IO_OK) throw IoError(fkde_io_last_error());
    s.p = p;
    s.pinned = pinned != 0;
    return s;
}

void io_check(int rc) {
    if (rc == FKDE_IO_INVALID_ARGUMENT) throw NumericError(fkde_io_last_error());
    if (rc != FKDE_IO_OK) throw IoError(fkde_io_last_error());
}

std::string fmt17(double v) {
    std::ostringstream os;
    os.precision(17);
    os << v;
    return os.str();
}

// ---------------------------------------------------------------- mixture (mixture.cpp)
struct Mixture {
    std::vector<double> weights, means, sigmas;
    size_t d = 0;
    size_t k() const { return weights.size(); }
    void validate() const {  // mixture.cpp:15-38
        if (weights.empty()) throw NumericError("mixture: needs at least one component");
        if (means.size() != weights.size() * d || sigmas.size() != weights.size() || d == 0)
            throw NumericError("mixture: weights/means/sigmas size mismatch");
        for (double m : means)
            if (!std::isfinite(m)) throw NumericError("SampleSet: non-finite entry");
        double total = 0.0;
        for (double w : weights) {
            if (!(w >= 0.0) || !std::isfinite(w)) throw NumericError("mixture: weights must be finite and >= 0");
            total += w;
        }
        if (std::abs(total - 1.0) > 1e-12) throw NumericError("mixture: weights must sum to 1 within 1e-12");
        for (double s : sigmas)
            if (!(s > 0.0) || !std::isfinite(s)) throw NumericError("mixture: sigmas must be positive");
    }
    nlohmann::json to_json() const {  // canonical form hashed by mixture_hash (mixture.cpp:133-146)
        nlohmann::json j;
        j["schema_version"] = 1;
        j["d"] = d;
        j["weights"] = weights;
        j["sigmas"] = sigmas;
        std::vector<std::vector<double>> rows(k());
        for (size_t c = 0; c < k(); ++c) rows[c].assign(means.begin() + c * d, means.begin() + (c + 1) * d);
        j["means"] = rows;
        return j;
    }
    uint64_t hash() const {  // FNV-1a 64, mixture.cpp:163-170
        const std::string canon = to_json().dump();
        uint64_t h = 0xcbf29ce484222325ULL;
        for (unsigned char ch : canon) {
            h ^= ch;
            h *= 0x100000001b3ULL;
        }
        return h;
    }
    // draws into page-locked memory (the engine's H2D copy is then one DMA)
    Samples sample(size_t n, uint64_t seed) const {
        Samples s;
        int pinned = 1;
        s.p = fkde_io_alloc(n * d, &pinned);
        if (!s.p) throw std::bad_alloc();
        s.pinned = pinned != 0;
        s.n = n;
        s.d = d;
        if (fkde_host_sample_mixture(weights.data(), means.data(), sigmas.data(), k(), d, n, seed, s.p) != 0)
            throw NumericError("sample_mixture: invalid mixture");
        return s;
    }
    std::vector<double> pdf(const double* x, size_t n) const {  // mixture.cpp:68-95
        std::vector<double> out(n, 0.0), norm(k());
        for (size_t c = 0; c < k(); ++c)
            norm[c] = weights[c] * std::pow(2.0 * std::numbers::pi * sigmas[c] * sigmas[c],
                                            -0.5 * static_cast<double>(d));
        for (size_t j = 0; j < n; ++j) {
            double acc = 0.0;
            for (size_t c = 0; c < k(); ++c) {
                double r2 = 0.0;
                for (size_t q = 0; q < d; ++q) {
                    const double diff = x[j * d + q] - means[c * d + q];
                    r2 += diff * diff;
                }
                acc += norm[c] * std::exp(-r2 / (2.0 * sigmas[c] * sigmas[c]));
            }
            out[j] = acc;
        }
        return out;
    }
};

Mixture load_mixture(const std::string& path) {  // mixture.cpp:97-127
    std::ifstream in(path);
    if (!in) throw IoError("cannot open mixture config: " + path);
    nlohmann::json j;
    try {
        in >> j;
    } catch (const nlohmann::json::exception& e) {
        throw IoError("mixture config parse error in " + path + ": " + e.what());
    }
    Mixture m;
    try {
        m.d = j.at("d").get<size_t>();
        m.weights = j.at("weights").get<std::vector<double>>();
        m.sigmas = j.at("sigmas").get<std::vector<double>>();
        for (const auto& r : j.at("means").get<std::vector<std::vector<double>>>()) {
            if (r.size() != m.d) throw NumericError("mixture config: mean row length != d");
            m.means.insert(m.means.end(), r.begin(), r.end());
        }
    } catch (const nlohmann::json::exception& e) {
        throw NumericError("mixture config missing field in " + path + ": " + e.what());
    }
    m.validate();
    return m;
}

uint64_t mix64(uint64_t x) { return fkde_host_mix64(x); }
uint64_t cell_data_seed(uint64_t seed, size_t n) {  // sweep.cpp:67-69
    return mix64(seed ^ mix64(static_cast<uint64_t>(n)));
}

// ---------------------------------------------------------------- bandwidth (sweep.cpp:31-61)
enum Method { kKde = 0, kSdkde = 1, kLaplace = 2 };
const char* method_name(Method m) { return m == kKde ? "kde" : m == kSdkde ? "sdkde" : "laplace"; }

struct MethodSpec {
    Method method = kKde;
    bool fused = true;
    static MethodSpec parse(const std::string& t) {  // sweep.cpp:17-22
        if (t == "laplace-nofuse") return {kLaplace, false};
        if (t == "kde") return {kKde, true};
        if (t == "sdkde") return {kSdkde, true};
        if (t == "laplace") return {kLaplace, true};
        throw NumericError("unknown method: " + t);
    }
    std::string label() const { return method == kLaplace && !fused ? "laplace-nofuse" : method_name(method); }
};

struct BandwidthPolicy {
    std::string rule = "auto";   // auto | silverman | sdkde | fixed
    double fixed_h = 0.0, sdkde_c = 0.0, fixed_h_score = 0.0;
    bool half = false;

    void attach(const Args& a) {  // BandwidthFlags, main.cpp:37-80
        if (a.has("--h-rule")) {
            rule = a.str("--h-rule");
            member(rule, {"auto", "silverman", "sdkde", "fixed"}, "--h-rule");
        }
        if (a.has("--h")) fixed_h = to_double(a.str("--h"), "--h");
        if (a.has("--h-score")) fixed_h_score = to_double(a.str("--h-score"), "--h-score");
        if (a.has("--sdkde-c")) sdkde_c = to_double(a.str("--sdkde-c"), "--sdkde-c");
        half = a.flag("--h-score-half");
        if (rule == "fixed" && !(fixed_h > 0.0)) throw UsageError("--h-rule fixed requires --h > 0");
        if (rule != "silverman" && rule != "sdkde" && fixed_h > 0.0) rule = "fixed";
    }
    bool data_dependent() const { return rule != "fixed"; }
    std::pair<double, double> resolve(const Samples& train, Method m) const {
        std::string eff = rule;
        if (eff == "auto") eff = m == kSdkde ? "sdkde" : "silverman";
        double h = 0.0;
        if (eff == "silverman") {
            h = fkde_host_silverman_bandwidth(train.data(), train.n, train.d);
        } else if (eff == "sdkde") {
            const double c = sdkde_c > 0.0 ? sdkde_c : fkde_host_silverman_prefactor(train.d);
            h = fkde_host_sdkde_bandwidth(train.data(), train.n, train.d, c);
        } else {
            if (!(fixed_h > 0.0)) throw NumericError("bandwidth policy: fixed rule needs h > 0");
            h = fixed_h;
        }
        if (!(h > 0.0) || !std::isfinite(h)) throw NumericError("bandwidth: degenerate data (h = 0)");
        double hs = half ? h / std::sqrt(2.0) : h;
        if (fixed_h_score > 0.0) hs = fixed_h_score;
        return {h, hs};
    }
};

// ---------------------------------------------------------------- engine
struct Engine {
    fkde_gpu_ctx* ctx = nullptr;
    // --threads maps onto devices (the reference's worker cap, engine.hpp:33-38):
    // 0 = every visible GPU (row / query shards + NCCL allgathers), k = the first k
    explicit Engine(size_t threads = 0) {
        int devs = 0;
        if (fkde_gpu_device_count(&devs) != 0 || devs < 1)
            throw std::runtime_error("no CUDA device for the B200 engine");
        const int use = threads == 0 ? devs : static_cast<int>(std::min<size_t>(threads, devs));
        std::vector<int> ids(use);
        for (int i = 0; i < use; ++i) ids[i] = i;
        const int rc = fkde_gpu_create(ids.data(), use, &ctx);
        if (rc != FKDE_OK) throw std::runtime_error("fkde_gpu_create on " + std::to_string(use) +
                                                    " device(s) failed (status " + std::to_string(rc) + ")");
    }
    ~Engine() { fkde_gpu_destroy(ctx); }
    void check(int rc) const {
        if (rc == FKDE_OK) return;
        const std::string msg = fkde_gpu_last_error(ctx);
        if (rc == FKDE_INVALID_ARGUMENT || rc == FKDE_DIMENSION_MISMATCH || rc == FKDE_SCORE_UNDERFLOW ||
            rc == FKDE_NON_FINITE || rc == FKDE_UNSUPPORTED_D)
            throw NumericError(msg);
        throw std::runtime_error(msg);
    }
    // fkde::estimate (estimator.cpp:14-60) on the B200 engine
    std::vector<double> estimate(const Samples& train, const double* q, size_t m, size_t d, Method method,
                                 std::pair<double, double> bw, size_t tile_m, size_t tile_n, bool fused,
                                 std::optional<double>* neg_mass) const {
        std::vector<double> out(m);
        double neg = 0.0;
        size_t err = 0;
        check(fkde_gpu_estimate(ctx, train.data(), train.n, q, m, d, method, bw.first, bw.second, tile_m,
                                tile_n, fused ? 1 : 0, out.data(), nullptr, &neg, &err));
        if (neg_mass && method == kLaplace) *neg_mass = neg;
        return out;
    }
};

void check_engine(const std::string& e) {
    if (e == "naive")
        throw UsageError("--engine naive: the CPU oracle engine is not part of the B200 build "
                         "(use the reference tool); engines here: gpu, flash (= gpu)");
    member(e, {"gpu", "flash"}, "--engine");
}

// ---------------------------------------------------------------- perf model (perfmodel.cpp)
struct HardwareSpec {
    std::string name;
    double peak_flops = 0.0, mem_bw = 0.0, exp_cost = 8.0;
};
HardwareSpec load_hw(const std::string& path) {  // perfmodel.cpp:16-52
    std::ifstream in(path);
    if (!in) throw IoError("cannot open hardware spec: " + path);
    HardwareSpec hw;
    std::string line;
    auto trim = [](std::string s) {
        const auto a = s.find_first_not_of(" \t\r");
        const auto b = s.find_last_not_of(" \t\r");
        return a == std::string::npos ? std::string{} : s.substr(a, b - a + 1);
    };
    while (std::getline(in, line)) {
        const auto hash = line.find('#');
        if (hash != std::string::npos) line.erase(hash);
        const auto eq = line.find('=');
        if (eq == std::string::npos) continue;
        const std::string key = trim(line.substr(0, eq)), value = trim(line.substr(eq + 1));
        try {
            if (key == "name") hw.name = value;
            else if (key == "peak_flops") hw.peak_flops = std::stod(value);
            else if (key == "mem_bw") hw.mem_bw = std::stod(value);
            else if (key == "exp_cost") hw.exp_cost = std::stod(value);
            else throw NumericError("hardware spec: unknown key '" + key + "' in " + path);
        } catch (const std::invalid_argument&) {
            throw NumericError("hardware spec: bad value for '" + key + "' in " + path);
        }
    }
    if (!(hw.peak_flops > 0.0) || !(hw.mem_bw > 0.0) || !(hw.exp_cost > 0.0))
        throw NumericError("HardwareSpec: peak_flops, mem_bw, exp_cost must be > 0");
    return hw;
}
double flops_nd(size_t d, size_t k) {  // perfmodel.cpp:62-67
    const double dd = static_cast<double>(d), kk = static_cast<double>(k);
    return (4.0 * dd + 12.0 + dd / 4.0 + 1.5) * kk * kk;
}
double flops_1d(size_t k) { return 17.75 * static_cast<double>(k) * static_cast<double>(k); }
double bytes_tile(size_t d, size_t tm, size_t tn) {
    return 4.0 * (2.0 * tm * static_cast<double>(d) + tn * static_cast<double>(d) + tm);
}
double bytes_nd(size_t d, size_t k, size_t tm, size_t tn) {
    return bytes_tile(d, tm, tn) * static_cast<double>((k + tm - 1) / tm) * static_cast<double>((k + tn - 1) / tn);
}
double bytes_linear(size_t d, size_t k) {
    return 4.0 * ((9.0 / 8.0) * d * static_cast<double>(k) + static_cast<double>(k) / 8.0);
}
double bytes_1d(size_t k) { return 5.0 * static_cast<double>(k); }
double intensity_asymptotic(size_t d) {
    const double dd = static_cast<double>(d);
    return ((17.0 / 4.0) * dd + 27.0 / 2.0) / (9.0 * dd / 2.0);
}
// sweep.cpp:74-90
double model_flops(const MethodSpec& s, size_t d, size_t n, size_t m) {
    const double dd = static_cast<double>(d), nn = static_cast<double>(n), mm = static_cast<double>(m);
    switch (s.method) {
        case kKde: return (2.0 * dd + 12.0) * nn * mm;
        case kSdkde: return (4.0 * dd + 12.0) * nn * nn + (2.0 * dd + 12.0) * nn * mm;
        case kLaplace: return s.fused ? (2.0 * dd + 14.0) * nn * mm : (4.0 * dd + 26.0) * nn * mm;
    }
    return 0.0;
}
// B200 view of the same call: exponentials (the MUFU roof)
double exp_count(const MethodSpec& s, size_t n, size_t m) {
    const double nn = static_cast<double>(n), mm = static_cast<double>(m);
    switch (s.method) {
        case kKde: return nn * mm;
        case kSdkde: return nn * nn + nn * mm;
        case kLaplace: return s.fused ? nn * mm : 2.0 * nn * mm;
    }
    return 0.0;
}

double median_of(std::vector<double> xs) {
    std::sort(xs.begin(), xs.end());
    const size_t m = xs.size() / 2;
    return xs.size() % 2 == 1 ? xs[m] : 0.5 * (xs[m - 1] + xs[m]);
}

void write_text(const std::string& path, const std::string& text) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw IoError("cannot open for writing: " + path);
    out << text;
    if (!out) throw IoError("short write: " + path);
}

std::string hex64(uint64_t v) {
    char buf[19];
    std::snprintf(buf, sizeof(buf), "0x%016llx", static_cast<unsigned long long>(v));
    return buf;
}

// ================================================================ subcommands
int run_gen(const Args& a) {
    const std::string config = a.req("--config");
    const size_t n = positive(a.req("--n"), "--n");
    const uint64_t seed = to_u64(a.req("--seed"), "--seed");
    const std::string out = a.req("--out"), format = a.str("--format", "bin");
    member(format, {"bin", "csv"}, "--format");
    const Mixture mix = load_mixture(config);
    const Samples s = mix.sample(n, seed);
    io_check(format == "bin" ? fkde_io_write_samples_bin(out.c_str(), s.data(), s.n, s.d)
                             : fkde_io_write_samples_csv(out.c_str(), s.data(), s.n, s.d));
    nlohmann::json meta;
    meta["n"] = s.n;
    meta["d"] = s.d;
    meta["seed"] = seed;
    meta["mixture_hash"] = hex64(mix.hash());
    meta["format"] = format;
    meta["format_version"] = 1;
    write_text(out + ".meta.json", meta.dump(2) + "\n");
    return kExitOk;
}

int run_estimate(const Args& a) {
    if (a.pos.size() != 2) throw UsageError("estimate needs <train> <query>");
    const std::string method_s = a.str("--method", "kde"), engine_s = a.str("--engine", "flash");
    member(method_s, {"kde", "sdkde", "laplace"}, "--method");
    check_engine(engine_s);
    BandwidthPolicy bw;
    bw.attach(a);
    const size_t tile_m = a.has("--tile-m") ? positive(a.str("--tile-m"), "--tile-m") : 64;
    const size_t tile_n = a.has("--tile-n") ? positive(a.str("--tile-n"), "--tile-n") : 1024;
    const bool no_fuse = a.flag("--no-fuse");
    const size_t threads = a.has("--threads") ? to_u64(a.str("--threads"), "--threads") : 0;
    const std::string out = a.req("--out"), format = a.str("--format", "csv");
    member(format, {"csv", "bin", "json"}, "--format");

    const Samples train = read_samples(a.pos[0]);
    const Samples queries = read_samples(a.pos[1]);
    const Method method = MethodSpec::parse(method_s).method;
    if (train.d != queries.d) throw NumericError("estimate: train and query dimensions differ");
    const auto h = bw.resolve(train, method);
    Engine eng(threads);
    const auto t0 = std::chrono::steady_clock::now();
    std::optional<double> neg;
    const std::vector<double> vals = eng.estimate(train, queries.data(), queries.n, train.d, method, h,
                                                  tile_m, tile_n, !no_fuse, &neg);
    const auto t1 = std::chrono::steady_clock::now();
    io_check(fkde_io_write_values(out.c_str(), vals.data(), vals.size(), format.c_str()));

    nlohmann::json s;   // main.cpp:133-150
    s["n_train"] = train.n;
    s["n_test"] = queries.n;
    s["d"] = train.d;
    s["method"] = method_s;
    s["engine"] = "gpu";
    s["h"] = h.first;
    s["h_score"] = h.second;
    s["tile_m"] = tile_m;
    s["tile_n"] = tile_n;
    s["fused"] = !no_fuse;
    s["wall_time_s"] = std::chrono::duration<double>(t1 - t0).count();
    if (neg) s["negative_mass"] = *neg;
    s["out"] = out;
    std::cout << s.dump() << "\n";
    return kExitOk;
}

int run_compare(const Args& a) {  // main.cpp:154-188
    if (a.pos.size() != 2) throw UsageError("compare needs <a> <b>");
    const double rtol = a.has("--rtol") ? to_double(a.str("--rtol"), "--rtol") : 1e-8;
    const bool per_component = a.flag("--per-component");
    auto load = [](const std::string& p) {
        double* v = nullptr;
        size_t m = 0;
        io_check(fkde_io_read_values(p.c_str(), &v, &m));
        std::vector<double> out(v, v + m);
        fkde_io_free(v, 0);
        return out;
    };
    const std::vector<double> x = load(a.pos[0]), y = load(a.pos[1]);
    if (x.size() != y.size()) throw NumericError("compare: value files have different lengths");
    double max_abs = 0.0, max_diff = 0.0, max_rel = 0.0;
    for (size_t i = 0; i < x.size(); ++i) max_abs = std::max(max_abs, std::max(std::abs(x[i]), std::abs(y[i])));
    for (size_t i = 0; i < x.size(); ++i) {
        const double diff = std::abs(x[i] - y[i]);
        max_diff = std::max(max_diff, diff);
        const double den = std::max(std::abs(x[i]), std::abs(y[i]));
        if (den > 0.0) max_rel = std::max(max_rel, diff / den);
        else if (diff > 0.0) max_rel = INFINITY;
    }
    const double normalized = max_abs > 0.0 ? max_diff / max_abs : (max_diff > 0.0 ? INFINITY : 0.0);
    const double gate = per_component ? max_rel : normalized;
    nlohmann::json o;
    o["count"] = x.size();
    o["max_abs_diff"] = max_diff;
    o["max_rel_vs_peak"] = normalized;
    o["max_rel_per_component"] = max_rel;
    o["rtol"] = rtol;
    o["pass"] = gate <= rtol;
    std::cout << o.dump() << "\n";
    return gate <= rtol ? kExitOk : kExitFail;
}

int run_model(const Args& a) {  // main.cpp:190-215
    const size_t d = positive(a.req("--d"), "--d");
    const size_t k = positive(a.req("--k"), "--k");
    const size_t tm = a.has("--tile-m") ? positive(a.str("--tile-m"), "--tile-m") : 64;
    const size_t tn = a.has("--tile-n") ? positive(a.str("--tile-n"), "--tile-n") : 1024;
    const HardwareSpec hw = load_hw(a.req("--hw"));
    const double flops = d == 1 ? flops_1d(k) : flops_nd(d, k);
    const double bytes = d == 1 ? bytes_1d(k) : bytes_nd(d, k, tm, tn);
    const double inten = flops / bytes, balance = hw.peak_flops / hw.mem_bw;
    nlohmann::json o;
    o["d"] = d;
    o["k"] = k;
    o["tile_m"] = tm;
    o["tile_n"] = tn;
    o["hw"] = hw.name;
    o["flops"] = flops;
    o["bytes"] = bytes;
    o["intensity"] = inten;
    o["machine_balance"] = balance;
    o["classification"] = inten >= balance ? "compute-bound" : "memory-bound";
    if (d > 1) {
        o["intensity_asymptotic_per_k"] = intensity_asymptotic(d);
        o["bytes_linear"] = bytes_linear(d, k);
    }
    // B200 roof of the same SD-KDE (n_train = k, n_test = k/8): one exp per pair
    const double exps = static_cast<double>(k) * k + static_cast<double>(k) * std::max<size_t>(1, k / 8);
    o["exp_count"] = exps;
    o["exp_bound_s"] = exps * hw.exp_cost / hw.peak_flops;
    std::cout << o.dump() << "\n";
    return kExitOk;
}

struct RuntimeRow {
    MethodSpec spec;
    size_t n = 0, m = 0, d = 0, tm = 0, tn = 0, repeats = 0;
    double median = 0.0, mflops = 0.0, exps = 0.0;
    std::optional<double> util;
    bool failed = false;
    std::string error;
};
struct ErrorRow {
    MethodSpec spec;
    size_t n = 0, d = 0;
    uint64_t seed = 0;
    double h = 0.0, hs = 0.0, mise = 0.0, mise_se = 0.0, miae = 0.0, miae_se = 0.0, neg = 0.0, neg_se = 0.0;
    bool failed = false;
    std::string error;
};

int run_bench(const Args& a) {
    const std::string mode = a.req("--mode");
    member(mode, {"runtime", "error"}, "--mode");
    const Mixture mix = load_mixture(a.req("--config"));
    std::vector<MethodSpec> methods;
    for (const auto& t : split_list(a.str("--methods", "kde,sdkde,laplace,laplace-nofuse"))) {
        member(t, {"kde", "sdkde", "laplace", "laplace-nofuse"}, "--methods");
        methods.push_back(MethodSpec::parse(t));
    }
    std::vector<size_t> n_grid;
    for (const auto& t : split_list(a.req("--n-grid"))) n_grid.push_back(positive(t, "--n-grid"));
    BandwidthPolicy bw;
    bw.attach(a);
    std::vector<size_t> tm_grid{64}, tn_grid{1024};
    if (a.has("--tile-m")) {
        tm_grid.clear();
        for (const auto& t : split_list(a.str("--tile-m"))) tm_grid.push_back(positive(t, "--tile-m"));
    }
    if (a.has("--tile-n")) {
        tn_grid.clear();
        for (const auto& t : split_list(a.str("--tile-n"))) tn_grid.push_back(positive(t, "--tile-n"));
    }
    const size_t repeats = a.has("--repeats") ? positive(a.str("--repeats"), "--repeats") : 5;
    const size_t threads = a.has("--threads") ? to_u64(a.str("--threads"), "--threads") : 0;
    const std::string out = a.req("--out"), format = a.str("--format", "csv");
    member(format, {"csv", "json"}, "--format");
    const bool strict = a.flag("--strict");
    size_t failed = 0, nrows = 0;
    std::string text;

    if (mode == "runtime") {
        // sweep.cpp:156-241: one warm-up then the median of `repeats` timed estimate()
        // calls per cell; data generation excluded, data-dependent bandwidth included
        if (!a.has("--seed")) throw UsageError("bench --mode runtime requires --seed");
        const uint64_t seed = to_u64(a.str("--seed"), "--seed");
        std::vector<std::string> engines = split_list(a.str("--engines", "gpu"));
        for (const auto& e : engines) check_engine(e);
        std::optional<HardwareSpec> hw;
        if (a.has("--hw")) hw = load_hw(a.str("--hw"));
        std::unique_ptr<Engine> eng;
        std::vector<RuntimeRow> rows;
        for (const auto& spec : methods)
            for (size_t ei = 0; ei < engines.size(); ++ei)
                for (size_t n : n_grid) {
                    const size_t m = std::max<size_t>(1, n / 8);
                    const Samples train = mix.sample(n, cell_data_seed(seed, n));
                    const Samples q = mix.sample(m, mix64(cell_data_seed(seed, n) ^ 0x71ULL));
                    for (size_t tm : tm_grid)
                        for (size_t tn : tn_grid) {
                            RuntimeRow r;
                            r.spec = spec;
                            r.n = n;
                            r.m = m;
                            r.d = mix.d;
                            r.tm = tm;
                            r.tn = tn;
                            r.repeats = repeats;
                            r.mflops = model_flops(spec, mix.d, n, m);
                            r.exps = exp_count(spec, n, m);
                            try {
                                if (!eng) eng = std::make_unique<Engine>(threads);
                                auto once = [&] {
                                    const auto h = bw.resolve(train, spec.method);
                                    eng->estimate(train, q.data(), m, mix.d, spec.method, h, tm, tn, spec.fused,
                                                  nullptr);
                                };
                                once();
                                std::vector<double> ts(repeats);
                                for (size_t i = 0; i < repeats; ++i) {
                                    const auto t0 = std::chrono::steady_clock::now();
                                    once();
                                    ts[i] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
                                }
                                r.median = median_of(ts);
                                if (hw) r.util = r.mflops / (r.median * hw->peak_flops);
                            } catch (const std::exception& e) {
                                r.failed = true;
                                r.error = e.what();
                            }
                            rows.push_back(r);
                        }
                }
        // sweep.cpp:281-322 schema (+ exp_count, the B200 roof's unit of work, last)
        if (format == "csv") {
            text = "schema_version,method,engine,n_train,n_test,d,tile_m,tile_n,repeats,"
                   "median_seconds,model_flops,utilization,failed,error,exp_count\n";
            for (const auto& r : rows)
                text += "1," + r.spec.label() + ",gpu," + std::to_string(r.n) + "," + std::to_string(r.m) + "," +
                        std::to_string(r.d) + "," + std::to_string(r.tm) + "," + std::to_string(r.tn) + "," +
                        std::to_string(r.repeats) + "," + fmt17(r.median) + "," + fmt17(r.mflops) + "," +
                        (r.util ? fmt17(*r.util) : "") + "," + (r.failed ? "1" : "0") + "," + r.error + "," +
                        fmt17(r.exps) + "\n";
        } else {
            nlohmann::json j;
            j["schema_version"] = 1;
            auto& arr = j["rows"] = nlohmann::json::array();
            for (const auto& r : rows) {
                nlohmann::json e;
                e["method"] = r.spec.label();
                e["engine"] = "gpu";
                e["n_train"] = r.n;
                e["n_test"] = r.m;
                e["d"] = r.d;
                e["tile_m"] = r.tm;
                e["tile_n"] = r.tn;
                e["repeats"] = r.repeats;
                e["median_seconds"] = r.median;
                e["model_flops"] = r.mflops;
                e["exp_count"] = r.exps;
                if (r.util) e["utilization"] = *r.util;
                e["failed"] = r.failed;
                if (r.failed) e["error"] = r.error;
                arr.push_back(e);
            }
            text = j.dump(2) + "\n";
        }
        for (const auto& r : rows) failed += r.failed;
        nrows = rows.size();
    } else {
        // sweep.cpp:105-154 + metrics.cpp:44-119
        const std::string engine_s = a.str("--engine", "flash");
        check_engine(engine_s);
        std::vector<uint64_t> seeds;
        for (const auto& t : split_list(a.str("--seeds", "0"))) seeds.push_back(to_u64(t, "--seeds"));
        const size_t n_eval = a.has("--n-eval") ? to_u64(a.str("--n-eval"), "--n-eval") : 2048;
        std::string metric = a.str("--metric", "auto");
        member(metric, {"auto", "grid", "mc"}, "--metric");
        const bool grid = metric == "grid" || (metric == "auto" && mix.d == 1);
        const size_t tm = tm_grid.front(), tn = tn_grid.front();
        std::unique_ptr<Engine> eng;
        std::vector<ErrorRow> rows;
        for (const auto& spec : methods)
            for (size_t n : n_grid)
                for (uint64_t seed : seeds) {
                    ErrorRow r;
                    r.spec = spec;
                    r.n = n;
                    r.seed = seed;
                    r.d = mix.d;
                    try {
                        const Samples train = mix.sample(n, cell_data_seed(seed, n));
                        const auto h = bw.resolve(train, spec.method);
                        r.h = h.first;
                        r.hs = h.second;
                        if (n_eval < 2) throw NumericError("error_metrics: n_eval must be >= 2");
                        if (!eng) eng = std::make_unique<Engine>(threads);
                        if (grid) {   // trapezoid on [min(mu - 6 sigma), max(mu + 6 sigma)]
                            if (mix.d != 1) throw NumericError("error_metrics: Grid1D requires d == 1");
                            double lo = mix.means[0] - 6.0 * mix.sigmas[0], hi = mix.means[0] + 6.0 * mix.sigmas[0];
                            for (size_t c = 1; c < mix.k(); ++c) {
                                lo = std::min(lo, mix.means[c] - 6.0 * mix.sigmas[c]);
                                hi = std::max(hi, mix.means[c] + 6.0 * mix.sigmas[c]);
                            }
                            std::vector<double> g(n_eval);
                            const double dx = (hi - lo) / static_cast<double>(n_eval - 1);
                            for (size_t i = 0; i < n_eval; ++i) g[i] = lo + dx * static_cast<double>(i);
                            const auto est = eng->estimate(train, g.data(), n_eval, 1, spec.method, h, tm, tn,
                                                           spec.fused, nullptr);
                            const auto truth = mix.pdf(g.data(), n_eval);
                            double mise = 0, miae = 0, neg = 0;
                            for (size_t i = 0; i < n_eval; ++i) {
                                if (!std::isfinite(est[i])) throw NumericError("estimate produced a non-finite value");
                                const double w = (i == 0 || i == n_eval - 1) ? 0.5 : 1.0;
                                const double diff = est[i] - truth[i];
                                mise += w * diff * diff;
                                miae += w * std::abs(diff);
                                neg += w * std::max(0.0, -est[i]);
                            }
                            r.mise = mise * dx;
                            r.miae = miae * dx;
                            r.neg = neg * dx;
                        } else {      // importance MC from the true mixture
                            const Samples z = mix.sample(n_eval, mix64(seed ^ 0x5eedULL));
                            const auto est = eng->estimate(train, z.data(), n_eval, mix.d, spec.method, h, tm, tn,
                                                           spec.fused, nullptr);
                            const auto truth = mix.pdf(z.data(), n_eval);
                            std::vector<double> sq(n_eval), ab(n_eval), ng(n_eval);
                            for (size_t i = 0; i < n_eval; ++i) {
                                if (!std::isfinite(est[i])) throw NumericError("estimate produced a non-finite value");
                                const double diff = est[i] - truth[i];
                                sq[i] = diff * diff / truth[i];
                                ab[i] = std::abs(diff) / truth[i];
                                ng[i] = std::max(0.0, -est[i]) / truth[i];
                            }
                            auto mse = [](const std::vector<double>& xs, double& mean, double& se) {
                                const double nn = static_cast<double>(xs.size());
                                mean = 0.0;
                                for (double x : xs) mean += x;
                                mean /= nn;
                                se = 0.0;
                                if (xs.size() < 2) return;
                                double ssq = 0.0;
                                for (double x : xs) ssq += (x - mean) * (x - mean);
                                se = std::sqrt(ssq / (nn - 1.0) / nn);
                            };
                            mse(sq, r.mise, r.mise_se);
                            mse(ab, r.miae, r.miae_se);
                            mse(ng, r.neg, r.neg_se);
                        }
                    } catch (const std::exception& e) {
                        r.failed = true;
                        r.error = e.what();
                    }
                    rows.push_back(r);
                }
        if (format == "csv") {   // sweep.cpp:243-260
            text = "schema_version,method,engine,n_train,seed,d,h,h_score,"
                   "mise,mise_se,miae,miae_se,negative_mass,negative_mass_se,failed,error\n";
            for (const auto& r : rows)
                text += "1," + r.spec.label() + ",gpu," + std::to_string(r.n) + "," + std::to_string(r.seed) + "," +
                        std::to_string(r.d) + "," + fmt17(r.h) + "," + fmt17(r.hs) + "," + fmt17(r.mise) + "," +
                        fmt17(r.mise_se) + "," + fmt17(r.miae) + "," + fmt17(r.miae_se) + "," + fmt17(r.neg) + "," +
                        fmt17(r.neg_se) + "," + (r.failed ? "1" : "0") + "," + r.error + "\n";
        } else {
            nlohmann::json j;
            j["schema_version"] = 1;
            auto& arr = j["rows"] = nlohmann::json::array();
            for (const auto& r : rows) {
                nlohmann::json e;
                e["method"] = r.spec.label();
                e["engine"] = "gpu";
                e["n_train"] = r.n;
                e["seed"] = r.seed;
                e["d"] = r.d;
                e["h"] = r.h;
                e["h_score"] = r.hs;
                e["mise"] = r.mise;
                e["mise_se"] = r.mise_se;
                e["miae"] = r.miae;
                e["miae_se"] = r.miae_se;
                e["negative_mass"] = r.neg;
                e["negative_mass_se"] = r.neg_se;
                e["failed"] = r.failed;
                if (r.failed) e["error"] = r.error;
                arr.push_back(e);
            }
            text = j.dump(2) + "\n";
        }
        for (const auto& r : rows) failed += r.failed;
        nrows = rows.size();
    }
    write_text(out, text);
    nlohmann::json s;
    s["rows"] = nrows;
    s["failed"] = failed;
    s["out"] = out;
    std::cout << s.dump() << "\n";
    return strict && failed ? kExitFail : kExitOk;
}

const char* kUsage =
    "fkde-b200 <gen|estimate|compare|bench|model> [options]\n"
    "  gen --config MIX.json --n N --seed S --out FILE [--format bin|csv]\n"
    "  estimate TRAIN QUERY --out FILE [--method kde|sdkde|laplace] [--engine gpu|flash]\n"
    "           [--h-rule auto|silverman|sdkde|fixed] [--h H] [--h-score HS] [--sdkde-c C]\n"
    "           [--h-score-half] [--tile-m M] [--tile-n N] [--no-fuse] [--format csv|bin|json]\n"
    "  compare A B [--rtol R] [--per-component]\n"
    "  bench --mode runtime|error --config MIX.json --n-grid N1,N2 --out FILE [--methods ...]\n"
    "        [--seed S] [--seeds S1,S2] [--engines gpu] [--tile-m ...] [--tile-n ...]\n"
    "        [--repeats R] [--metric auto|grid|mc] [--n-eval E] [--hw SPEC] [--format csv|json] [--strict]\n"
    "        [--threads K]   (estimate / bench: K GPUs, 0 = all visible)\n"
    "  model --d D --k K --hw SPEC [--tile-m M] [--tile-n N]\n";

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::cerr << kUsage;
        return kExitUsage;
    }
    const std::string cmd = argv[1];
    if (cmd == "--help" || cmd == "-h") {
        std::cout << kUsage;
        return kExitOk;
    }
    try {
        const std::vector<std::string> flags{"--h-score-half", "--no-fuse", "--fast", "--per-component",
                                             "--strict", "--help"};
        const Args a = parse(argc, argv, 2, flags);
        if (a.flag("--help")) {
            std::cout << kUsage;
            return kExitOk;
        }
        if (cmd == "gen") return run_gen(a);
        if (cmd == "estimate") return run_estimate(a);
        if (cmd == "compare") return run_compare(a);
        if (cmd == "bench") return run_bench(a);
        if (cmd == "model") return run_model(a);
        std::cerr << "unknown subcommand: " << cmd << "\n" << kUsage;
        return kExitUsage;
    } catch (const UsageError& e) {
        std::cerr << "usage error: " << e.what() << "\n";
        return kExitUsage;
    } catch (const IoError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return kExitIo;
    } catch (const NumericError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return kExitNumeric;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return kExitFail;
    }
}
