// host_io.cpp -- FKDE sample / value files for the B200 engine (include/fkde_io.h).
//
// Formats follow the reference byte for byte (proj/core/src/io.cpp):
//   binary samples  io.cpp:55-104   "FKDE" | u32 version=1 | u64 n | u64 d | n*d f64 LE
//   CSV samples     io.cpp:106-175  header x0..x{d-1}; rows of %.17g values
//   values          io.cpp:192-258  csv ("value" header) | bin (n x 1) | json array
// What differs is where the bytes land: fkde_io_read_samples can read the
// payload straight into pinned host memory (one read(2) into a
// cudaHostAlloc'ed buffer), which the engine then copies to HBM as a single
// DMA.  Host code only; no device work happens here.
#include <json.hpp>
#include <cuda_runtime.h>

#include <cerrno>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <system_error>
#include <vector>

#include "../../include/fkde_io.h"

static_assert(sizeof(double) == 8, "FKDE files hold IEEE-754 binary64");

namespace {

thread_local std::string g_err;

struct IoFail {
    int status;
    std::string msg;
};

[[noreturn]] void io_error(const std::string& m) { throw IoFail{FKDE_IO_ERROR, m}; }
[[noreturn]] void arg_error(const std::string& m) { throw IoFail{FKDE_IO_INVALID_ARGUMENT, m}; }

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return FKDE_IO_OK;
    } catch (const IoFail& e) {
        g_err = e.msg;
        return e.status;
    } catch (const std::bad_alloc&) {
        g_err = "out of host memory";
        return FKDE_IO_ERROR;
    }
}

constexpr char kMagic[4] = {'F', 'K', 'D', 'E'};
constexpr uint32_t kVersion = 1;

struct File {
    FILE* f = nullptr;
    File(const char* path, const char* mode) : f(std::fopen(path, mode)) {}
    ~File() {
        if (f) std::fclose(f);
    }
};

void check_finite(const double* v, size_t count, const char* what) {  // SampleSet::validate
    for (size_t i = 0; i < count; ++i)
        if (!std::isfinite(v[i])) arg_error(std::string(what) + ": non-finite entry");
}

std::string fmt17(double v) {  // ostream precision(17), default floatfield == %.17g
    char buf[40];
    std::snprintf(buf, sizeof(buf), "%.17g", v);
    return buf;
}

// CSV row of doubles separated by ',' (trailing '\r' / ' ' ignored), io.cpp:24-50
void parse_row(const char* p, const char* end, const std::string& path, std::vector<double>& out) {
    while (end > p && (end[-1] == '\r' || end[-1] == ' ')) --end;
    while (p < end) {
        double v = 0.0;
        const auto r = std::from_chars(p, end, v);
        if (r.ec != std::errc()) io_error("bad CSV number in " + path);
        out.push_back(v);
        p = r.ptr;
        if (p == end) break;
        if (*p != ',') io_error("bad CSV separator in " + path);
        ++p;
    }
}

bool read_line(FILE* f, std::string& line) {
    line.clear();
    int c;
    bool any = false;
    while ((c = std::fgetc(f)) != EOF) {
        any = true;
        if (c == '\n') return true;
        line.push_back(static_cast<char>(c));
    }
    return any;
}

// pinned: in = requested, out = granted (page-locked memory needs a CUDA
// driver; without one the buffer is ordinary heap memory)
double* alloc_values(size_t count, int* pinned) {
    const size_t bytes = (count ? count : 1) * sizeof(double);
    void* p = nullptr;
    if (*pinned && cudaHostAlloc(&p, bytes, cudaHostAllocPortable) != cudaSuccess) {
        cudaGetLastError();
        p = nullptr;
        *pinned = 0;
    }
    if (!*pinned) {
        p = std::malloc(bytes);
        if (!p) throw std::bad_alloc();
    }
    return static_cast<double*>(p);
}

void read_bin(const std::string& path, double** out, size_t* n_out, size_t* d_out, int* pinned) {
    File in(path.c_str(), "rb");
    if (!in.f) io_error("cannot open: " + path);
    char magic[4];
    if (std::fread(magic, 1, 4, in.f) != 4 || std::memcmp(magic, kMagic, 4) != 0)
        io_error("not a FKDE sample file: " + path);
    uint32_t version = 0;
    uint64_t n = 0, d = 0;
    const bool ok = std::fread(&version, 4, 1, in.f) == 1 && std::fread(&n, 8, 1, in.f) == 1 &&
                    std::fread(&d, 8, 1, in.f) == 1;
    if (!ok || version != kVersion) io_error("unsupported FKDE format version in " + path);
    if (n == 0 || d == 0 || n > (1ULL << 40) || d > (1ULL << 20))
        io_error("implausible header in " + path);
    double* v = alloc_values(n * d, pinned);
    if (std::fread(v, sizeof(double), n * d, in.f) != n * d) {
        fkde_io_free(v, *pinned);
        io_error("truncated FKDE sample file: " + path);
    }
    for (size_t i = 0; i < n * d; ++i)
        if (!std::isfinite(v[i])) {
            fkde_io_free(v, *pinned);
            arg_error("SampleSet: non-finite entry");
        }
    *out = v;
    *n_out = n;
    *d_out = d;
}

void read_csv(const std::string& path, double** out, size_t* n_out, size_t* d_out, int* pinned) {
    File in(path.c_str(), "rb");
    if (!in.f) io_error("cannot open: " + path);
    std::string header;
    if (!read_line(in.f, header)) io_error("empty CSV file: " + path);
    size_t d = 1;
    for (char c : header) d += c == ',';
    std::vector<double> vals, row;
    std::string line;
    size_t n = 0;
    while (read_line(in.f, line)) {
        if (line.empty()) continue;
        row.clear();
        parse_row(line.data(), line.data() + line.size(), path, row);
        if (row.size() != d) io_error("CSV row width mismatch in " + path);
        vals.insert(vals.end(), row.begin(), row.end());
        ++n;
    }
    if (n == 0) io_error("CSV file has no data rows: " + path);
    check_finite(vals.data(), vals.size(), "SampleSet");
    double* v = alloc_values(vals.size(), pinned);
    std::memcpy(v, vals.data(), vals.size() * sizeof(double));
    *out = v;
    *n_out = n;
    *d_out = d;
}

void write_bin(const char* path, const double* values, size_t n, size_t d) {
    if (n == 0 || d == 0) arg_error("SampleSet: n and d must be >= 1");
    check_finite(values, n * d, "SampleSet");
    File out(path, "wb");
    if (!out.f) io_error(std::string("cannot open for writing: ") + path);
    const uint64_t n64 = n, d64 = d;
    const bool ok = std::fwrite(kMagic, 1, 4, out.f) == 4 && std::fwrite(&kVersion, 4, 1, out.f) == 1 &&
                    std::fwrite(&n64, 8, 1, out.f) == 1 && std::fwrite(&d64, 8, 1, out.f) == 1 &&
                    std::fwrite(values, sizeof(double), n * d, out.f) == n * d;
    if (!ok || std::fflush(out.f) != 0) io_error(std::string("short write: ") + path);
}

}  // namespace

extern "C" {

int fkde_io_read_samples(const char* path, double** out, size_t* n, size_t* d, int* pinned) {
    return guarded([&] {
        if (!path || !out || !n || !d || !pinned) arg_error("fkde_io_read_samples: null argument");
        *pinned = *pinned ? 1 : 0;
        *out = nullptr;
        File probe(path, "rb");
        if (!probe.f) io_error(std::string("cannot open: ") + path);
        char magic[4] = {0, 0, 0, 0};
        const size_t got = std::fread(magic, 1, 4, probe.f);
        const bool bin = got == 4 && std::memcmp(magic, kMagic, 4) == 0;
        if (bin) read_bin(path, out, n, d, pinned);
        else read_csv(path, out, n, d, pinned);
    });
}

double* fkde_io_alloc(size_t count, int* pinned) {
    if (!pinned) return nullptr;
    *pinned = *pinned ? 1 : 0;
    try {
        return alloc_values(count, pinned);
    } catch (...) {
        return nullptr;
    }
}

void fkde_io_free(double* p, int pinned) {
    if (!p) return;
    if (pinned) cudaFreeHost(p);
    else std::free(p);
}

int fkde_io_write_samples_bin(const char* path, const double* values, size_t n, size_t d) {
    return guarded([&] {
        if (!path || (!values && n * d)) arg_error("fkde_io_write_samples_bin: null argument");
        write_bin(path, values, n, d);
    });
}

int fkde_io_write_samples_csv(const char* path, const double* values, size_t n, size_t d) {
    return guarded([&] {
        if (!path || (!values && n * d)) arg_error("fkde_io_write_samples_csv: null argument");
        if (n == 0 || d == 0) arg_error("SampleSet: n and d must be >= 1");
        check_finite(values, n * d, "SampleSet");
        std::string text;
        for (size_t k = 0; k < d; ++k) text += (k ? ",x" : "x") + std::to_string(k);
        text += '\n';
        for (size_t i = 0; i < n; ++i) {
            for (size_t k = 0; k < d; ++k) {
                if (k) text += ',';
                text += fmt17(values[i * d + k]);
            }
            text += '\n';
        }
        File out(path, "wb");
        if (!out.f) io_error(std::string("cannot open for writing: ") + path);
        if (std::fwrite(text.data(), 1, text.size(), out.f) != text.size() || std::fflush(out.f) != 0)
            io_error(std::string("short write: ") + path);
    });
}

int fkde_io_write_values(const char* path, const double* values, size_t m, const char* format) {
    return guarded([&] {
        if (!path || !format) arg_error("fkde_io_write_values: null argument");
        if (m == 0) arg_error("write_values: empty value vector");
        const std::string fmt = format;
        if (fmt == "bin") {
            write_bin(path, values, m, 1);
            return;
        }
        std::string text;
        if (fmt == "csv") {
            text = "value\n";
            for (size_t i = 0; i < m; ++i) text += fmt17(values[i]) + "\n";
        } else if (fmt == "json") {
            // nlohmann::json, like the reference's writer (io.cpp:203-206): the same
            // number formatting (grisu2 shortest form, "0.0" for integral values,
            // null for non-finite), so the files are byte-identical
            nlohmann::json j = std::vector<double>(values, values + m);
            text = j.dump() + "\n";
        } else {
            arg_error("write_values: unknown format '" + fmt + "'");
        }
        File out(path, "wb");
        if (!out.f) io_error(std::string("cannot open for writing: ") + path);
        if (std::fwrite(text.data(), 1, text.size(), out.f) != text.size() || std::fflush(out.f) != 0)
            io_error(std::string("short write: ") + path);
    });
}

int fkde_io_read_values(const char* path, double** out, size_t* m) {
    return guarded([&] {
        if (!path || !out || !m) arg_error("fkde_io_read_values: null argument");
        *out = nullptr;
        File in(path, "rb");
        if (!in.f) io_error(std::string("cannot open: ") + path);
        const int first = std::fgetc(in.f);
        if (first == 'F') {
            std::fclose(in.f);
            in.f = nullptr;
            size_t n = 0, d = 0;
            int heap = 0;
            read_bin(path, out, &n, &d, &heap);
            *m = n * d;
            return;
        }
        std::vector<double> vals;
        if (first == '[') {   // JSON array of numbers
            std::string text;
            int c;
            while ((c = std::fgetc(in.f)) != EOF) text.push_back(static_cast<char>(c));
            const char* p = text.data();
            const char* end = p + text.size();
            auto skip = [&] {
                while (p < end && (*p == ' ' || *p == '\n' || *p == '\r' || *p == '\t')) ++p;
            };
            skip();
            if (p < end && *p == ']') io_error(std::string("values file has no rows: ") + path);
            for (;;) {
                skip();
                double v = 0.0;
                const auto r = std::from_chars(p, end, v);
                if (r.ec != std::errc()) io_error(std::string("bad JSON values file ") + path);
                vals.push_back(v);
                p = r.ptr;
                skip();
                if (p < end && *p == ',') {
                    ++p;
                    continue;
                }
                if (p < end && *p == ']') break;
                io_error(std::string("bad JSON values file ") + path);
            }
        } else {
            std::string header;
            if (first != EOF) header.push_back(static_cast<char>(first));
            std::string rest;
            if (first != '\n' && first != EOF) {
                read_line(in.f, rest);
                header += rest;
            } else if (first == '\n') {
                header.clear();
            }
            while (!header.empty() && (header.back() == '\r' || header.back() == ' ')) header.pop_back();
            if (header != "value")
                io_error(std::string("not a values file (expected 'value' header): ") + path);
            std::string line;
            std::vector<double> row;
            while (read_line(in.f, line)) {
                if (line.empty()) continue;
                row.clear();
                parse_row(line.data(), line.data() + line.size(), path, row);
                if (row.empty()) io_error(std::string("bad CSV number in ") + path);
                vals.push_back(row[0]);
            }
        }
        if (vals.empty()) io_error(std::string("values file has no rows: ") + path);
        int heap = 0;
        double* v = alloc_values(vals.size(), &heap);
        std::memcpy(v, vals.data(), vals.size() * sizeof(double));
        *out = v;
        *m = vals.size();
    });
}

const char* fkde_io_last_error(void) { return g_err.c_str(); }

}  // extern "C"
