// fkde_gpu.cu -- runtime + C ABI of the B200-native Flash-SD-KDE engine.
//
// Implements include/fkde_gpu.h.  The estimator pipeline of the reference
// (fkde::engine::sdkde_flash, engine.cpp:389-405) runs per device as:
//
//   H2D -> column mean (centring) -> operand scale -> pack A/B tiles
//   -> pairwise_tc_kernel<Score>     (rows sharded across ranks)
//   -> finalize_score (s, x + h^2/2 s)
//   -> ncclAllGather(x_sd)           (only when world > 1)
//   -> pack -> pairwise_tc_kernel<Gauss|Laplace> (queries sharded)
//   -> reduce_density -> ncclAllGather(densities) -> D2H
//
// Single process: one host thread per device (ncclCommInitAll).  One process
// per GPU: fkde_gpu_create_rank (ncclCommInitRank with a caller-broadcast id).
// NCCL is loaded lazily with dlopen so that single-GPU use has no NCCL
// dependency and a process that already loaded torch's NCCL reuses it.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <numeric>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/fkde_gpu.h"
#include "layout.cuh"
#include "pairwise_tc.cuh"
#include "prep_kernels.cuh"
#include "direct_rows.cuh"
#include "spatial_order.cuh"

#include <cub/device/device_radix_sort.cuh>

using namespace fkde_b200;

namespace {

// --------------------------------------------------------------------------
// NCCL (dlopen)
// --------------------------------------------------------------------------
struct NcclApi {
    bool loaded = false;
    std::string err;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        // FKDE_NCCL_LIB: explicit NCCL (or NCCL-API-compatible) library path,
        // e.g. a specific NCCL build; tests use it for an in-process transport
        // that lets the multi-rank code path run on a single GPU
        const char* env = std::getenv("FKDE_NCCL_LIB");
        const char* names[] = {env && *env ? env : "libnccl.so.2", "libnccl.so.2", "libnccl.so"};
        void* h = nullptr;
        for (const char* nm : names) {
            h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
            if (h) break;
        }
        if (!h) {
            api.err = std::string("cannot dlopen libnccl.so.2: ") + dlerror();
            return;
        }
        api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
        api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
        api.CommInitAll = (decltype(api.CommInitAll))dlsym(h, "ncclCommInitAll");
        api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
        api.AllGather = (decltype(api.AllGather))dlsym(h, "ncclAllGather");
        api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
        api.loaded = api.GetUniqueId && api.CommInitRank && api.CommInitAll && api.CommDestroy &&
                     api.AllGather && api.GetErrorString;
        if (!api.loaded) api.err = "libnccl.so.2 lacks required symbols";
    });
    return api;
}

// --------------------------------------------------------------------------
// errors
// --------------------------------------------------------------------------
struct Status {
    int code = FKDE_OK;
    std::string msg;
    size_t index = 0;
    bool ok() const { return code == FKDE_OK; }
};

Status make_status(int code, const char* fmt, ...) {
    Status s;
    s.code = code;
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    s.msg = buf;
    return s;
}

#define CUDA_TRY(expr)                                                                         \
    do {                                                                                       \
        cudaError_t e__ = (expr);                                                              \
        if (e__ != cudaSuccess)                                                                \
            return make_status(FKDE_CUDA_ERROR, "%s failed: %s (%s:%d)", #expr,                \
                               cudaGetErrorString(e__), __FILE__, __LINE__);                   \
    } while (0)

#define NCCL_TRY(expr)                                                                         \
    do {                                                                                       \
        ncclResult_t r__ = (expr);                                                             \
        if (r__ != ncclSuccess)                                                                \
            return make_status(FKDE_NCCL_ERROR, "%s failed: %s", #expr,                        \
                               nccl().GetErrorString(r__));                                    \
    } while (0)

#define STATUS_TRY(expr)            \
    do {                            \
        Status s__ = (expr);        \
        if (!s__.ok()) return s__;  \
    } while (0)

// --------------------------------------------------------------------------
// device state
// --------------------------------------------------------------------------
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
};

// bumped on every workspace (re)allocation: a captured CUDA graph holds raw
// workspace pointers and is only replayed while this is unchanged
std::atomic<uint64_t> g_alloc_epoch{0};

Status ensure(DevBuf& b, size_t bytes) {
    if (bytes == 0) bytes = 16;
    if (b.bytes >= bytes) return {};
    g_alloc_epoch.fetch_add(1);
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.bytes = 0;
    const size_t want = round_up(bytes + bytes / 8, 1 << 20);  // grow with headroom
    CUDA_TRY(cudaMalloc(&b.p, want));
    b.bytes = want;
    return {};
}

// FKDE_PDL=0 in the environment switches programmatic dependent launch off by default
bool g_pdl_default = [] {
    const char* e = std::getenv("FKDE_PDL");
    return !(e && *e == '0');
}();

struct Options {
    int engine = FKDE_ENGINE_TC;
    int spatial = 0;       // FKDE_OPT_SPATIAL: 0 auto (n >= kSpatialMinN), 1 on, 2 off
    bool pdl = g_pdl_default;   // FKDE_OPT_PDL: programmatic dependent launch of the kernel chain
    int splits = 0;
    int timing = 0;
    int max_ctas = 0;
    int flush_tiles = 0;   // 0: ~256 columns (engine default)
    long long* trace = nullptr;   // debug: device buffer for pairwise_tc_kernel's clock trace
};

struct Device {
    int dev = 0;
    int rank = 0;
    int world = 1;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    cudaStream_t side = nullptr;       // host copies that overlap the next pass
    cudaEvent_t ev_side_in = nullptr, ev_side_out = nullptr;
    cudaEvent_t ev_y_in = nullptr, ev_y = nullptr;   // SD-KDE: query upload on the side stream
    // FKDE_OPT_TIMING: events bracketing each tensor-core pass kernel (FKDE_KT_*)
    cudaEvent_t kev[2 * FKDE_KT_COUNT] = {};
    bool kran[FKDE_KT_COUNT] = {};
    ncclComm_t comm = nullptr;
    bool attrs_set = false;
    DevBuf X, Y, opA, opB, opB2, part0, part1, xsd, out, aux0, aux1, colpart, scal, err, flags;
    DevBuf risk, dpart, ddone;   // direct_rows_kernel: spread flags, partials, counters
    DevBuf pdone;                // prep_stats / scale_two completion counters (self-resetting)
    DevBuf sched;                // pairwise kernels' unit schedulers, 2 per mode (self-resetting)
    DevBuf qmax;                 // scale_two per-block maxima
    // spatial order of the score pass (spatial_order.cuh): sorted points, permutation,
    // keys, CUB scratch, axes, tile centroids, skip statistics, un-permuted outputs
    DevBuf Xs, perm, keys, cubtmp, ordsc, cenA, cenB, boxA, boxB, skipstats, unperm0, unperm1, pmask, smask;
    // the density pass's tile masks: its own buffers, so that the score pass's skip mask
    // (read back by fkde_gpu_last_skip_stats) is not overwritten by the density pass
    DevBuf dpmask, dsmask;
    size_t mask_bytes = 0;       // skip mask of the last score pass (0: none)
    uint64_t tiles_total = 0;    // tile pairs of the last score pass
    bool ordered = false;        // last score pass ran on the spatial order
    // density pass on the spatial order: sorted queries, their permutation, keys + CUB
    // scratch, skipped tiles per query tile, densities back in the caller's order
    DevBuf Qs, qperm, qkeys, qcubtmp, qskip, qmass, qout;
    bool qordered = false;       // last density pass ran on the spatial order (D.qout)
    uint64_t dtiles_total = 0;   // tile pairs of the last density pass
    size_t dtiles_rows = 0;      // query tiles of the last skipping density pass (0: none)
    cudaEvent_t ev[FKDE_T_COUNT + 1] = {};
    int64_t launches = 0;
    // device-resident API: the call's whole device program as a CUDA graph,
    // replayed while the arguments and options repeat (small problems are
    // launch-bound: ~20 kernels per SD-KDE)
    std::string graph_key, graph_seen;
    cudaGraphExec_t graph = nullptr;
    int64_t graph_launches = 0;
    uint64_t graph_epoch = 0;   // g_alloc_epoch when the graph was captured
    float timing[FKDE_T_COUNT] = {};
    Status last;
    std::vector<DevBuf*> buffers() {   // every device workspace (free / size accounting)
        return {&X,     &Y,     &opA,  &opB,    &opB2,  &part0, &part1,     &xsd,     &out,
                &aux0,  &aux1,  &colpart, &scal, &err,  &flags, &risk,      &dpart,   &ddone,
                &pdone, &sched, &qmax,  &Xs,   &perm,   &keys,  &cubtmp, &ordsc,    &cenA,    &cenB,
                &boxA,  &boxB,  &skipstats, &unperm0, &unperm1, &pmask, &smask, &Qs, &qperm,
                &qkeys, &qcubtmp, &qskip, &qmass, &qout, &dpmask, &dsmask};
    }
};

}  // namespace

struct fkde_gpu_ctx {
    std::vector<Device> devs;
    int world = 1;
    bool per_rank = false;  // one process per GPU
    Options opt;
    std::mutex mu;          // serialises calls (device state, workspaces, graphs)
    std::mutex err_mu;      // guards err (written by every call's finish())
    std::string err;        // message of the most recent call on this context
};

namespace {

// Per-thread copy of the last message a thread produced (or read) for a
// context: fkde_gpu_last_error hands out a pointer that no other thread can
// invalidate, and a thread sees the outcome of its own last call even when
// other threads share the context.
struct ErrSlot {
    const fkde_gpu_ctx* ctx;
    std::string msg;
};
thread_local std::vector<ErrSlot> t_errors;

std::string& thread_error_slot(const fkde_gpu_ctx* ctx) {
    for (auto& e : t_errors)
        if (e.ctx == ctx) return e.msg;
    if (t_errors.size() >= 16) t_errors.erase(t_errors.begin());
    t_errors.push_back({ctx, std::string()});
    return t_errors.back().msg;
}


// shard [r*chunk, min(n,(r+1)*chunk)) with chunk = ceil(n/world): equal-size
// allgather slices (the tail slice is padding).
struct Shard {
    size_t chunk, begin, rows;
};
Shard shard_of(size_t n, int world, int rank, size_t align = 1) {
    Shard s;
    s.chunk = round_up((n + world - 1) / world, align);
    s.begin = std::min(n, s.chunk * rank);
    s.rows = std::min(n, s.begin + s.chunk) - s.begin;
    return s;
}

int choose_splits(const Options& o, size_t row_tiles, size_t col_tiles, int ctas) {
    if (o.splits > 0) return static_cast<int>(std::min<size_t>(o.splits, col_tiles));
    // Units run chunk-major, so one column chunk's B tiles are the L2 working
    // set: keep a chunk <= 32 MiB (2048 tiles) so the operand stream is read
    // from HBM about once.  Then minimise rounds * (tiles per unit + pipeline
    // fill) over S in [s_min, min(col_tiles, 64)].
    const size_t s_min = std::min<size_t>(col_tiles, (col_tiles + 2047) / 2048);
    double best = 1e300;
    int best_s = static_cast<int>(std::max<size_t>(s_min, 1));
    const size_t smax = std::max<size_t>(std::min<size_t>(col_tiles, 64), s_min);
    for (size_t s = std::max<size_t>(s_min, 1); s <= smax; ++s) {
        const size_t units = row_tiles * s;
        const size_t rounds = (units + ctas - 1) / ctas;
        const double per_unit = static_cast<double>((col_tiles + s - 1) / s) + 2.0;
        const double t = static_cast<double>(rounds) * per_unit;
        if (t < best * 0.999) {
            best = t;
            best_s = static_cast<int>(s);
        }
    }
    return best_s;
}

inline unsigned grid1(size_t n, unsigned bs) { return static_cast<unsigned>((n + bs - 1) / bs); }

double risk_half_norm() {   // (FKDE_RISK_HALF_NORM: debug override for accuracy probes)
    static const double v = [] {
        const char* e = std::getenv("FKDE_RISK_HALF_NORM");
        return e && *e ? std::atof(e) : kRiskHalfNorm;
    }();
    return v;
}

// Kernel-chain launch with programmatic dependent launch (layout.cuh: every chain
// kernel waits on griddepcontrol before touching global memory), so each kernel's
// launch and prologue (block scheduling, barrier init, TMEM allocation) overlap
// the tail of its predecessor.  FKDE_OPT_PDL = 0 launches them plainly.


template <typename... KArgs, typename... Args>
cudaError_t launch_chain(bool pdl, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                         cudaStream_t stream, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

template <int MODE>
Status launch_pairwise(Device& D, const Options& o, const PairArgs& a, size_t n_cols) {
    {
        using Cfg = TcConfig<MODE>;
        static thread_local int attr_done_dev[64] = {};
        if (!(attr_done_dev[D.dev & 63] & (1 << MODE))) {
            CUDA_TRY(cudaFuncSetAttribute(pairwise_tc_kernel<MODE>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          Cfg::kSmemBytes));
            attr_done_dev[D.dev & 63] |= 1 << MODE;
        }
        const int units = a.n_row_tiles * a.splits;
        if (units == 0) return {};   // (an empty shard)
        int grid = std::min(units, D.num_sms);
        if (o.max_ctas > 0) grid = std::min(grid, o.max_ctas);
        PairArgs b = a;
        b.sched = D.sched.as<unsigned int>() + 2 * MODE;   // (ensure_call_scratch)
        const int kt = MODE == kModeScore ? FKDE_KT_SCORE : (MODE == kModeCheck ? FKDE_KT_CHECK : FKDE_KT_DENSITY);
        if (o.timing) {
            if (!D.kev[0])
                for (auto& e : D.kev) CUDA_TRY(cudaEventCreate(&e));
            CUDA_TRY(cudaEventRecord(D.kev[2 * kt], D.stream));
        }
        CUDA_TRY(launch_chain(o.pdl, pairwise_tc_kernel<MODE>, dim3(grid), dim3(Cfg::kThreads),
                              Cfg::kSmemBytes, D.stream, b));
        if (o.timing) {
            CUDA_TRY(cudaEventRecord(D.kev[2 * kt + 1], D.stream));
            D.kran[kt] = true;
        }
    }
    ++D.launches;
    CUDA_TRY(cudaGetLastError());
    return {};
}



void record(Device& D, const Options& o, int idx) {
    if (o.timing) cudaEventRecord(D.ev[idx], D.stream);
}

// ---- building blocks ------------------------------------------------------------
// Per-call device scratch that the fused prologue kernels clear: flag lists (sized
// for either pass), the underflow row, the skip statistics and the completion
// counters.  Allocated before any kernel of the call is enqueued, so no buffer
// moves between the kernel that clears it and the ones that use it.
Status ensure_call_scratch(Device& D, size_t flag_rows) {
    STATUS_TRY(ensure(D.flags, (flag_rows + 1) * sizeof(unsigned int)));
    STATUS_TRY(ensure(D.err, sizeof(unsigned long long)));
    STATUS_TRY(ensure(D.skipstats, 4 * sizeof(unsigned long long)));
    if (!D.pdone.p) {   // counters start at zero and reset themselves
        STATUS_TRY(ensure(D.pdone, 4 * sizeof(unsigned int)));
        CUDA_TRY(cudaMemsetAsync(D.pdone.p, 0, D.pdone.bytes, D.stream));
    }
    if (!D.sched.p) {
        STATUS_TRY(ensure(D.sched, 8 * sizeof(unsigned int)));
        CUDA_TRY(cudaMemsetAsync(D.sched.p, 0, D.sched.bytes, D.stream));
    }
    return {};
}

// mean (+ the operand scale for scale factor k, 0 = none) of X into sc, and the
// per-call counters cleared -- one launch (prep_stats)
Status prep(Device& D, bool pdl, const double* dX, size_t n, int d, double k, PassScalars* sc,
            bool score) {
    const int nparts = static_cast<int>(std::min<size_t>(256, std::max<size_t>(1, n / 64)));
    STATUS_TRY(ensure(D.colpart, static_cast<size_t>(nparts) * 48 * sizeof(double)));
    PrepArgs a{};
    a.x = dX;
    a.n = n;
    a.d = d;
    a.k = k;
    a.sc = sc;
    a.part = D.colpart.as<double>();
    a.done = D.pdone.as<unsigned int>();
    a.clear_u32[0] = D.flags.as<unsigned int>();
    if (score) {
        a.clear_max = D.err.as<unsigned long long>();
        a.clear_stats = D.skipstats.as<unsigned long long>();
    }
    CUDA_TRY(launch_chain(pdl, prep_stats, dim3(nparts), dim3(256), 0, D.stream, a));
    ++D.launches;
    CUDA_TRY(cudaGetLastError());
    return {};
}

// operand packing arguments (pack_two packs the row and column operands of a pass
// in one launch)
Status pack_args(Device& D, const double* x, size_t rows, int d, int format, bool center, double k,
                 const PassScalars* sc, DevBuf& out, size_t* rows_padded, PackArgs* pa,
                 size_t align = kTileRows, float a_offset = 0.f) {
    const size_t rp = round_up(std::max<size_t>(rows, 1), align);
    STATUS_TRY(ensure(out, rp * kRowBytes));
    if (format == 0) STATUS_TRY(ensure(D.risk, rp));
    PackArgs& a = *pa;
    a = PackArgs{};
    a.x = x;
    a.rows = rows;
    a.rows_padded = rp;
    a.d = d;
    a.format = format;
    a.center = center ? 1 : 0;
    a.k = k;
    a.sc = sc;
    a.out = out.as<uint4>();
    a.a_offset = a_offset;
    a.risk = format == 0 ? D.risk.as<uint8_t>() : nullptr;   // row side: spread flags
    a.risk_half_norm = risk_half_norm();
    *rows_padded = rp;
    return {};
}

Status pack2(Device& D, bool pdl, const PackArgs& a, const PackArgs& b) {
    const unsigned ba = grid1(a.rows_padded, 128), bb = grid1(b.rows_padded, 128);
    CUDA_TRY(launch_chain(pdl, pack_two, dim3(ba + bb), dim3(128), 0, D.stream, a, b, ba));
    ++D.launches;
    CUDA_TRY(cudaGetLastError());
    return {};
}

// one pairwise pass over (row operand x column operand) with density partials
Status density_pass(Device& D, const Options& o, int mode, size_t rows_pad, size_t n_cols,
                    const PassScalars* sc, int* nparts_out, const uint32_t* skip_mask = nullptr,
                    int mask_words = 0) {
    const size_t rt = rows_pad / kTileRows;
    const size_t ct = round_up(n_cols, kTileRows) / kTileRows;
    const int splits =
        choose_splits(o, rt, ct, o.max_ctas > 0 ? std::min(o.max_ctas, D.num_sms) : D.num_sms);
    // partial sums per (split, row): one per epilogue tile phase
    const size_t per = TcConfig<kModeGauss>::kNP;
    const size_t nparts = static_cast<size_t>(splits) * per;
    STATUS_TRY(ensure(D.part0, nparts * rows_pad * sizeof(float)));
    if (mode == kModeLaplace) STATUS_TRY(ensure(D.part1, nparts * rows_pad * sizeof(float)));
    PairArgs a{};
    a.opA = D.opA.as<uint8_t>();
    a.opB = D.opB.as<uint8_t>();
    a.n_row_tiles = static_cast<int>(rt);
    a.n_col_tiles = static_cast<int>(ct);
    a.splits = splits;
    a.sc = sc;
    a.part0 = D.part0.as<float>();
    a.part1 = mode == kModeLaplace ? D.part1.as<float>() : nullptr;
    a.flush_log2 = 0;
    a.rows_pad = rows_pad;
    a.diag_row0 = -1;
    a.skip_mask = const_cast<uint32_t*>(skip_mask);
    a.mask_words = mask_words;
#ifdef FKDE_CTA_TIMES
    a.trace = o.trace;
#endif
    if (mode == kModeGauss)
        STATUS_TRY(launch_pairwise<kModeGauss>(D, o, a, n_cols));
    else
        STATUS_TRY(launch_pairwise<kModeLaplace>(D, o, a, n_cols));
    *nparts_out = static_cast<int>(nparts);
    return {};
}

// flag list for direct_rows_kernel: D.flags = [0] count, [1..] local row indices
// (sized by ensure_call_scratch, the count cleared by prep_stats / scale_two)

// Recompute the flagged rows by direct differences (direct_rows.cuh).  The
// flagged count lives on the device; the launch exits at once when it is 0.
Status launch_direct(Device& D, bool pdl, DirectArgs& e, size_t rows) {
    // partials: at most (row blocks x splits) < 2 * kDirTargetItems items of 128 rows
    STATUS_TRY(ensure(D.dpart, static_cast<size_t>(2 * kDirTargetItems) * kDirRows * kDirPart *
                                   sizeof(double)));
    // completion counters: one per row block, or per row when few rows are flagged
    const size_t blocks = std::max<size_t>((rows + kDirRows - 1) / kDirRows + 1, kDirFewRows);
    if (D.ddone.bytes < blocks * sizeof(unsigned int)) {   // counters start at zero, then self-reset
        STATUS_TRY(ensure(D.ddone, blocks * sizeof(unsigned int)));
        CUDA_TRY(cudaMemsetAsync(D.ddone.p, 0, D.ddone.bytes, D.stream));
    }
    e.part = D.dpart.as<double>();
    e.done = D.ddone.as<unsigned int>();
    CUDA_TRY(launch_chain(pdl, direct_rows_kernel, dim3(kDirTargetItems), dim3(kDirRows), 0, D.stream, e));
    ++D.launches;
    CUDA_TRY(cudaGetLastError());
    return {};
}

Status allgather(Device& D, void* buf, size_t count_per_rank, ncclDataType_t t) {
    if (D.world <= 1) return {};
    const size_t elt = t == ncclFloat64 ? 8 : 4;
    char* base = static_cast<char*>(buf);
    NCCL_TRY(nccl().AllGather(base + D.rank * count_per_rank * elt, buf, count_per_rank, t, D.comm,
                              D.stream));
    return {};
}

// ---- per-device programs ---------------------------------------------------------------
struct Job {
    enum Kind { kScore, kScoreAcc, kKde, kSdkde, kDist } kind;
    // host (h*) or device (d*) inputs
    const double* hX = nullptr;
    const double* hY = nullptr;
    const double* dX = nullptr;
    const double* dY = nullptr;
    size_t n = 0, m = 0;
    int d = 0;
    double h = 1.0, h_score = 1.0;
    int kernel = FKDE_KERNEL_GAUSSIAN;
    int fused = 1;
    // host outputs (only device 0 / every rank writes them)
    double* out = nullptr;       // densities [m] | scores [n*d] | phi_sum [n]
    double* out2 = nullptr;      // debiased [n*d] | weighted [n*d]
    double* d_out = nullptr;     // device output (device-resident API)
    bool sync = true;
};

// smallest n for which the score pass runs on the spatial order by default: below
// it the few extra launches outweigh the skipped tiles (BASELINE configs 2-5 use it)
constexpr size_t kSpatialMinN = 32768;
// centroid half-distance^2 (log2 units) above which a tile pair is checked for
// skipping: skipping needs max log2 phi' < -26, i.e. r^2/2 > 41 for every pair
constexpr float kSkipPredict = 40.0f;
// score pass on the spatial order: O is drained at every change of the B2 tile group
// (kB2GroupLog2 column tiles, pairwise_tc.cuh) or after kCentredFlush visited tiles
constexpr int kCentredFlush = 1 << kB2GroupLog2;   // a whole B2 group

bool use_spatial(const Options& o, size_t n) {
    return o.spatial == 1 || o.spatial == 3 || (o.spatial == 0 && n >= kSpatialMinN);
}

// Spatial order of the training points (spatial_order.cuh): D.Xs = X[perm],
// D.perm = perm.  Identical on every rank (deterministic from the same input).
Status spatial_order(Device& D, const double* dX, size_t n, int d, const PassScalars* sc) {
    const size_t ns = cov_sample_count(n);
    const int nparts = static_cast<int>(std::min<size_t>(296, std::max<size_t>(1, ns / 256)));
    STATUS_TRY(ensure(D.colpart, static_cast<size_t>(nparts) * 256 * sizeof(double)));
    STATUS_TRY(ensure(D.ordsc, sizeof(OrderScalars)));
    cov_stage1<<<nparts, 256, 0, D.stream>>>(dX, n, ns, d, sc, D.colpart.as<double>());
    order_axes<<<1, 256, 0, D.stream>>>(D.colpart.as<double>(), nparts, d, D.ordsc.as<OrderScalars>());
    STATUS_TRY(ensure(D.keys, 2 * n * sizeof(uint32_t)));        // keys in | keys out
    STATUS_TRY(ensure(D.perm, 2 * n * sizeof(uint32_t)));        // idx in | perm
    uint32_t* kin = D.keys.as<uint32_t>();
    uint32_t* kout = kin + n;
    uint32_t* iin = D.perm.as<uint32_t>() + n;
    uint32_t* perm = D.perm.as<uint32_t>();
    morton_keys<<<grid1(n, 256), 256, 0, D.stream>>>(dX, n, d, std::sqrt(static_cast<double>(ns)), sc,
                                                      D.ordsc.as<OrderScalars>(), kin, iin);
    size_t tmp = 0;
    CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kin, kout, iin, perm, static_cast<int>(n),
                                             0, kSortBits, D.stream));
    STATUS_TRY(ensure(D.cubtmp, tmp));
    CUDA_TRY(cub::DeviceRadixSort::SortPairs(D.cubtmp.p, tmp, kin, kout, iin, perm, static_cast<int>(n),
                                             0, kSortBits, D.stream));
    STATUS_TRY(ensure(D.Xs, n * d * sizeof(double)));
    gather_rows<<<grid1(n * d, 256), 256, 0, D.stream>>>(dX, perm, n, d, D.Xs.as<double>());
    D.launches += 4;   // (+ CUB's own sort kernels)
    CUDA_TRY(cudaGetLastError());
    return {};
}

// Density pass on the spatial order: a tile pair is skipped when the box bound
// proves every pair's log2 phi < -(kDensitySkipHalfR2 - 0.5) (0.5: margin for the
// float boxes).  tile_predict sums, per query tile, the bound on what one row loses
// to its skipped tiles (128 columns x the largest phi the box bound allows, times
// 1 + d/2 + ln2 |log2 phi| for the Laplace-fused terms phi (1 + d/2 - u)), and a row
// whose term mass (|ca| s0 + |cb| |s1|: the scale of the fp32 sums' own rounding of
// that row) is not at least 2^24 times that bound is recomputed by direct
// differences (reduce_density flags it).  The skip therefore changes no row by more
// than 2^-24 of its term mass.  The threshold trades skipped tiles against rows sent
// to the recompute: 45 / 43 / 41.5 give config 5's density pass 12.2 / 11.9 / 11.6 ms
// but config 4 (Laplace-fused) 2.10 / 2.06 / 2.22 ms per call (1 / ~3 / 7 recomputed
// rows there); 43 is the best of both (tools/density_skip_probe.sh).
constexpr float kDensitySkipHalfR2 = 43.0f;
float density_skip_half_r2() {   // (FKDE_DENSITY_SKIP: debug override for A/B runs)
    static const float v = [] {
        const char* e = std::getenv("FKDE_DENSITY_SKIP");
        return e && *e ? static_cast<float>(std::atof(e)) : kDensitySkipHalfR2;
    }();
    return v;
}

// Queries sorted on the training order's axes (D.ordsc; sc: the training mean,
// n_cov: the count the covariance was summed over): D.Qs = Q[qperm]
Status order_queries(Device& D, const double* dQ, size_t m, int d, size_t n_cov,
                     const PassScalars* sc) {
    STATUS_TRY(ensure(D.qkeys, 2 * m * sizeof(uint32_t)));
    STATUS_TRY(ensure(D.qperm, 2 * m * sizeof(uint32_t)));
    uint32_t* kin = D.qkeys.as<uint32_t>();
    uint32_t* kout = kin + m;
    uint32_t* iin = D.qperm.as<uint32_t>() + m;
    uint32_t* perm = D.qperm.as<uint32_t>();
    morton_keys<<<grid1(m, 256), 256, 0, D.stream>>>(dQ, m, d,
                                                      std::sqrt(static_cast<double>(cov_sample_count(n_cov))), sc,
                                                      D.ordsc.as<OrderScalars>(), kin, iin);
    size_t tmp = 0;
    CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kin, kout, iin, perm, static_cast<int>(m), 0,
                                             kSortBits, D.stream));
    STATUS_TRY(ensure(D.qcubtmp, tmp));
    CUDA_TRY(cub::DeviceRadixSort::SortPairs(D.qcubtmp.p, tmp, kin, kout, iin, perm, static_cast<int>(m),
                                             0, kSortBits, D.stream));
    STATUS_TRY(ensure(D.Qs, m * d * sizeof(double)));
    gather_rows<<<grid1(m * d, 256), 256, 0, D.stream>>>(dQ, perm, m, d, D.Qs.as<double>());
    D.launches += 2;
    CUDA_TRY(cudaGetLastError());
    return {};
}

// Score pass on this rank's row shard; leaves the requested per-row outputs in
// D.aux0 / D.aux1 / D.xsd in global row layout (gathered when world > 1).  With
// the spatial order (D.ordered) that layout is the sorted one: unpermute_score()
// restores the caller's order for the host / device outputs.
Status score_program(Device& D, const Options& o, const Job& J, const double* dX,
                     PassScalars* sc, bool want_xsd) {
    const int d = J.d;
    const size_t n = J.n;
    const double ks = std::sqrt(kLog2e) / J.h_score;
    // mean + operand scale (bounding-box bound) + per-call counters: one launch
    STATUS_TRY(prep(D, o.pdl, dX, n, d, ks, sc, true));
    D.ordered = use_spatial(o, n);
    if (D.ordered) {
        STATUS_TRY(spatial_order(D, dX, n, d, sc));
        dX = D.Xs.as<double>();
    }
    // row shards start on a tile boundary so the diagonal is tile aligned
    const Shard sh = shard_of(n, D.world, D.rank, kTileRows);
    size_t rows_pad = 0, cols_pad = 0;
    PackArgs pa, pb;
    // A rows carry the P' = phi * 2^15 offset (layout.cuh): S = log2 P' off the tensor core
    STATUS_TRY(pack_args(D, dX + sh.begin * d, sh.rows, d, 0, true, ks, sc, D.opA, &rows_pad, &pa,
                         kTileRows, kPScaleF));
    // score-pass column tiles are TcConfig<kModeScore>::kNCol points wide: pad the
    // column operand to a whole number of those and of 128-point pack tiles
    constexpr size_t kScoreNCol = TcConfig<kModeScore>::kNCol;
    const size_t col_align = std::lcm<size_t>(kScoreNCol, kTileRows);
    STATUS_TRY(pack_args(D, dX, n, d, 1, true, ks, sc, D.opB, &cols_pad, &pb, col_align));
    STATUS_TRY(pack2(D, o.pdl, pa, pb));
    record(D, o, FKDE_T_SCORE);

    const size_t rt = rows_pad / kTileRows;
    const size_t ct = cols_pad / kScoreNCol;
    const int ctas = o.max_ctas > 0 ? std::min(o.max_ctas, D.num_sms) : D.num_sms;
    const int splits = choose_splits(o, rt, ct, ctas);
    // fp64 partials per split
    STATUS_TRY(ensure(D.part0, static_cast<size_t>(splits) * rows_pad * sizeof(double)));
    STATUS_TRY(ensure(D.part1, static_cast<size_t>(splits) * rows_pad * kMaxDim * sizeof(double)));
    PairArgs a{};
    a.opA = D.opA.as<uint8_t>();
    a.opB = D.opB.as<uint8_t>();
    a.n_row_tiles = static_cast<int>(rt);
    a.n_col_tiles = static_cast<int>(ct);
    a.splits = splits;
    a.sc = sc;
    a.dpart0 = D.part0.as<double>();
    a.dpart1 = D.part1.as<double>();
    // drain interval: the option, or by default every 2 tiles (~192 columns: the
    // accumulation length that keeps the tensor core's truncation error near 2e-4,
    // DESIGN §4); the spatial order drains every tile (below)
    const int flush = o.flush_tiles > 0 ? o.flush_tiles
                                        : std::max<int>(1, 256 / static_cast<int>(kScoreNCol));
    a.flush_log2 = 0;
    while ((2 << a.flush_log2) <= flush) ++a.flush_log2;
    a.rows_pad = rows_pad;
    a.diag_row0 = static_cast<long long>(sh.begin);
    a.trace = o.trace;
    a.stats = D.skipstats.as<unsigned long long>();   // (cleared by prep_stats)
    D.mask_bytes = 0;
    D.tiles_total = static_cast<uint64_t>(rt) * ct;
    if (D.ordered) {
        // spatial order: tile centroids, and GEMM2 on the column operand centred per
        // column tile (B2, layout.cuh) with a drain after every visited tile
        STATUS_TRY(ensure(D.cenA, rt * kMaxDim * sizeof(float)));
        STATUS_TRY(ensure(D.cenB, ct * kMaxDim * sizeof(float)));
        STATUS_TRY(ensure(D.boxA, rt * kBoxFloats * sizeof(float)));
        STATUS_TRY(ensure(D.boxB, ct * kBoxFloats * sizeof(float)));
        tile_summary<<<static_cast<unsigned>(rt), 128, 0, D.stream>>>(
            dX + sh.begin * d, sh.rows, d, sc, D.ordsc.as<OrderScalars>(), ks, kTileRows, 0,
            D.cenA.as<float>(), D.boxA.as<float>());
        tile_summary<<<static_cast<unsigned>(ct), 128, 0, D.stream>>>(
            dX, n, d, sc, D.ordsc.as<OrderScalars>(), ks, static_cast<int>(kScoreNCol), 0,
            D.cenB.as<float>(), D.boxB.as<float>());
        size_t b2_pad = 0;
        PackArgs p2;
        STATUS_TRY(pack_args(D, dX, n, d, 2, true, ks, sc, D.opB2, &b2_pad, &p2, col_align));
        p2.cen = D.cenB.as<float>();
        p2.cen_tile = static_cast<int>(kScoreNCol);
        p2.ones_mask = (1 << kB2GroupLog2) - 1;
        pack_operands<<<grid1(b2_pad, 128), 128, 0, D.stream>>>(p2);
        D.launches += 3;
        CUDA_TRY(cudaGetLastError());
        static const bool no_b2 = std::getenv("FKDE_NO_B2") != nullptr;   // debug A/B
        if (!no_b2) {
            a.opB2 = D.opB2.as<uint8_t>();
            a.cenB = D.cenB.as<float>();
            const int fl = o.flush_tiles > 0 ? o.flush_tiles : kCentredFlush;
            a.flush_log2 = 0;
            while ((2 << a.flush_log2) <= fl) ++a.flush_log2;
        }
    }
    if (D.ordered && o.spatial != 3) {
        // tile skipping: centroids -> predicted pairs -> exact check -> skip mask
        const int words = static_cast<int>((ct + 31) / 32);
        const size_t mbytes = rt * words * sizeof(uint32_t);
        STATUS_TRY(ensure(D.pmask, mbytes));
        STATUS_TRY(ensure(D.smask, mbytes));
        static const float pred = [] {   // debug override for A/B runs (tools/spatial_probe.py)
            const char* e = std::getenv("FKDE_SKIP_PRED");
            return e && *e ? static_cast<float>(std::atof(e)) : kSkipPredict;
        }();
        // proven-zero threshold on the lower bound of r^2/2 (log2 units): every pair
        // then has log2 phi' = 15 - r^2/2 < kSkipLog2 - 0.5 (float boxes' margin)
        const float proven = 15.0f - kSkipLog2 + 0.5f;
        const PredShape ps = pred_shape(rt, words, D.num_sms);
        tile_predict<<<dim3(ps.gx, ps.gy), ps.rows, 0, D.stream>>>(
            D.cenA.as<float>(), D.boxA.as<float>(), static_cast<int>(rt), D.cenB.as<float>(),
            D.boxB.as<float>(), static_cast<int>(ct), words, pred, proven, D.pmask.as<uint32_t>(),
            D.smask.as<uint32_t>(), nullptr, nullptr, -1, 128.f, static_cast<int>(ps.wpb));
        D.launches += 1;
        CUDA_TRY(cudaGetLastError());
        PairArgs c = a;
        c.opB2 = nullptr;
        c.cenB = nullptr;
#ifdef FKDE_CTA_TIMES
        if (true) {
            c.trace = a.trace;   // (regions per MODE)
        } else
#endif
        if (std::getenv("FKDE_TRACE_CHECK")) {   // debug: trace the check pass, not the score pass
            c.trace = a.trace;
            a.trace = nullptr;
        } else {
            c.trace = nullptr;
        }
        c.pred_mask = D.pmask.as<uint32_t>();
        c.skip_mask = D.smask.as<uint32_t>();
        c.mask_words = words;
        c.splits = choose_splits(o, rt, ct, ctas);
        STATUS_TRY(launch_pairwise<kModeCheck>(D, o, c, n));
        a.skip_mask = D.smask.as<uint32_t>();
        a.mask_words = words;
        D.mask_bytes = mbytes;
    }
    STATUS_TRY(launch_pairwise<kModeScore>(D, o, a, n));
    record(D, o, FKDE_T_FINALIZE);

    const size_t nrows_g = sh.chunk * D.world;  // gather layout
    FinalizeArgs f{};
    f.part_s = D.part0.as<double>();
    f.part_t = D.part1.as<double>();
    f.splits = splits;
    f.rows_pad = rows_pad;
    f.rows = sh.rows;
    f.row0 = sh.begin;
    f.d = d;
    f.x = dX;
    f.sc = sc;
    f.k = ks;
    f.h_score = J.h_score;
    f.shift = 0.5 * J.h * J.h;
    f.underflow_row = D.err.as<unsigned long long>();   // (set to ~0 by prep_stats)
    if (J.kind == Job::kScore) {
        STATUS_TRY(ensure(D.aux0, nrows_g * d * sizeof(double)));
        f.score = D.aux0.as<double>();
    } else if (J.kind == Job::kScoreAcc) {
        STATUS_TRY(ensure(D.aux0, nrows_g * sizeof(double)));
        STATUS_TRY(ensure(D.aux1, nrows_g * d * sizeof(double)));
        f.phi_sum = D.aux0.as<double>();
        f.weighted = D.aux1.as<double>();
    }
    if (want_xsd) {
        STATUS_TRY(ensure(D.xsd, nrows_g * d * sizeof(double)));
        f.xsd_c = D.xsd.as<double>();
    }
    f.flag_count = D.flags.as<unsigned int>();
    f.flag_rows = f.flag_count + 1;
    f.risk = D.risk.as<uint8_t>();
    CUDA_TRY(launch_chain(o.pdl, finalize_score, dim3(grid1(std::max<size_t>(sh.rows, 1) * d, 256)),
                          dim3(256), 0, D.stream, f));
    ++D.launches;
    CUDA_TRY(cudaGetLastError());
    {
        DirectArgs e{};
        e.mode = kExactScore;
        e.count = f.flag_count;
        e.rows = f.flag_rows;
        e.rowpts = dX + sh.begin * d;
        e.row0 = sh.begin;
        e.center_rows = 1;
        e.cols = dX;
        e.center_cols = 1;
        e.n = n;
        e.d = d;
        e.sc = sc;
        e.h = J.h_score;
        e.shift = f.shift;
        e.score = f.score;
        e.xsd_c = f.xsd_c;
        e.phi_sum = f.phi_sum;
        e.weighted = f.weighted;
        STATUS_TRY(launch_direct(D, o.pdl, e, sh.rows));
        // (statistics: the score pass's directly recomputed row count, skipstats[1])
        CUDA_TRY(cudaMemcpyAsync(D.skipstats.as<unsigned long long>() + 1, f.flag_count, sizeof(unsigned int),
                                 cudaMemcpyDeviceToDevice, D.stream));
    }
    record(D, o, FKDE_T_GATHER);
    if (J.kind == Job::kScore) STATUS_TRY(allgather(D, D.aux0.p, sh.chunk * d, ncclFloat64));
    if (J.kind == Job::kScoreAcc) {
        STATUS_TRY(allgather(D, D.aux0.p, sh.chunk, ncclFloat64));
        STATUS_TRY(allgather(D, D.aux1.p, sh.chunk * d, ncclFloat64));
    }
    if (want_xsd) STATUS_TRY(allgather(D, D.xsd.p, sh.chunk * d, ncclFloat64));
    if (D.ordered) {   // per-row outputs back to the caller's order
        const uint32_t* perm = D.perm.as<uint32_t>();
        if (J.kind == Job::kScore) {
            STATUS_TRY(ensure(D.unperm0, n * d * sizeof(double)));
            scatter_rows<<<grid1(n * d, 256), 256, 0, D.stream>>>(D.aux0.as<double>(), perm, n, d,
                                                                  nullptr, D.unperm0.as<double>());
            ++D.launches;
        } else if (J.kind == Job::kScoreAcc) {
            STATUS_TRY(ensure(D.unperm0, n * sizeof(double)));
            STATUS_TRY(ensure(D.unperm1, n * d * sizeof(double)));
            scatter_rows<<<grid1(n, 256), 256, 0, D.stream>>>(D.aux0.as<double>(), perm, n, 1,
                                                              nullptr, D.unperm0.as<double>());
            scatter_rows<<<grid1(n * d, 256), 256, 0, D.stream>>>(D.aux1.as<double>(), perm, n, d,
                                                                  nullptr, D.unperm1.as<double>());
            D.launches += 2;
        }
        CUDA_TRY(cudaGetLastError());
    }
    return {};
}

// Density of the rank's query shard against `dCols` (n x d; centred iff
// !center_cols), gathered into D.out (m doubles, gather layout).
Status query_program(Device& D, const Options& o, const Job& J, const double* dCols,
                     bool cols_centred, const double* dQ, const PassScalars* mu_src,
                     PassScalars* sc_q, int kernel, int fused) {
    const int d = J.d;
    const size_t n = J.n, m = J.m;
    const double kh = std::sqrt(kLog2e) / J.h;
    // scale exponent over both point sets (identical on every rank), the mean copied
    // from mu_src, the density flag counter cleared: one launch (scale_two)
    {
        const unsigned g = grid1(n + m, 256);
        STATUS_TRY(ensure(D.qmax, g * sizeof(unsigned int)));
        ScaleArgs s2{};
        s2.cols = dCols;
        s2.n = n;
        s2.cols_centred = cols_centred ? 1 : 0;
        s2.rows = dQ;
        s2.m = m;
        s2.d = d;
        s2.k = kh;
        s2.mu_src = mu_src;
        s2.sc = sc_q;
        s2.block_max = D.qmax.as<unsigned int>();
        s2.done = D.pdone.as<unsigned int>() + 1;
        s2.clear_u32 = D.flags.as<unsigned int>();
        CUDA_TRY(launch_chain(o.pdl, scale_two, dim3(g), dim3(256), 0, D.stream, s2));
        ++D.launches;
        CUDA_TRY(cudaGetLastError());
    }
    // spatial order (the columns were sorted by the score pass / spatial_order): the
    // queries sorted on the same axes, and -- Gaussian and Laplace-fused passes --
    // tile pairs skipped on the box bound (kDensitySkipHalfR2)
    D.qordered = D.ordered;
    D.dtiles_rows = 0;
    if (D.qordered) {
        STATUS_TRY(order_queries(D, dQ, m, d, n, sc_q));
        dQ = D.Qs.as<double>();
    }
    const bool skipping = D.qordered && o.spatial != 3 && (kernel == FKDE_KERNEL_GAUSSIAN || fused);
    const Shard sh = shard_of(m, D.world, D.rank);
    size_t rows_pad = 0, cols_pad = 0;
    PackArgs pa, pb;
    STATUS_TRY(pack_args(D, dQ + sh.begin * d, sh.rows, d, 0, true, kh, sc_q, D.opA, &rows_pad, &pa));
    STATUS_TRY(pack_args(D, dCols, n, d, 1, !cols_centred, kh, sc_q, D.opB, &cols_pad, &pb));
    STATUS_TRY(pack2(D, o.pdl, pa, pb));
    record(D, o, FKDE_T_QUERY);
    const uint32_t* dmask = nullptr;
    int dwords = 0, mass_parts = 0;
    const size_t q_rt = rows_pad / kTileRows, q_ct = cols_pad / kTileRows;
    D.dtiles_total = static_cast<uint64_t>(q_rt) * q_ct;
    if (skipping) {
        dwords = static_cast<int>((q_ct + 31) / 32);
        STATUS_TRY(ensure(D.cenA, q_rt * kMaxDim * sizeof(float)));
        STATUS_TRY(ensure(D.cenB, q_ct * kMaxDim * sizeof(float)));
        STATUS_TRY(ensure(D.boxA, q_rt * kBoxFloats * sizeof(float)));
        STATUS_TRY(ensure(D.boxB, q_ct * kBoxFloats * sizeof(float)));
        STATUS_TRY(ensure(D.dpmask, q_rt * dwords * sizeof(uint32_t)));
        STATUS_TRY(ensure(D.dsmask, q_rt * dwords * sizeof(uint32_t)));
        STATUS_TRY(ensure(D.qskip, q_rt * sizeof(unsigned int)));
        const PredShape ps = pred_shape(q_rt, dwords, D.num_sms);
        mass_parts = static_cast<int>(ps.gy);   // tile_predict's gridDim.y
        STATUS_TRY(ensure(D.qmass, q_rt * mass_parts * sizeof(float)));
        CUDA_TRY(cudaMemsetAsync(D.qskip.p, 0, q_rt * sizeof(unsigned int), D.stream));
        if (sh.rows)
            tile_summary<<<static_cast<unsigned>(q_rt), 128, 0, D.stream>>>(
                dQ + sh.begin * d, sh.rows, d, sc_q, D.ordsc.as<OrderScalars>(), kh, kTileRows, 0,
                D.cenA.as<float>(), D.boxA.as<float>());
        tile_summary<<<static_cast<unsigned>(q_ct), 128, 0, D.stream>>>(
            dCols, n, d, sc_q, D.ordsc.as<OrderScalars>(), kh, kTileRows, cols_centred ? 1 : 0,
            D.cenB.as<float>(), D.boxB.as<float>());
        // (no predicted pairs: thresh = inf; only the proven bound skips)
        tile_predict<<<dim3(ps.gx, ps.gy), ps.rows, 0, D.stream>>>(
            D.cenA.as<float>(), D.boxA.as<float>(), static_cast<int>(q_rt), D.cenB.as<float>(),
            D.boxB.as<float>(), static_cast<int>(q_ct), dwords, INFINITY, density_skip_half_r2(),
            D.dpmask.as<uint32_t>(), D.dsmask.as<uint32_t>(), D.qskip.as<unsigned int>(), D.qmass.as<float>(),
            kernel == FKDE_KERNEL_GAUSSIAN ? -1 : d, static_cast<float>(kTileRows), static_cast<int>(ps.wpb));
        D.launches += 3;
        CUDA_TRY(cudaGetLastError());
        dmask = D.dsmask.as<uint32_t>();
        D.dtiles_rows = q_rt;
    }

    const double norm = std::pow(2.0 * M_PI, -0.5 * d) * std::pow(J.h, -static_cast<double>(d)) /
                        static_cast<double>(n);  // gaussian_norm_const(h,d)/n, kernels.cpp:26-29
    STATUS_TRY(ensure(D.out, sh.chunk * D.world * sizeof(double)));
    double* outp = D.out.as<double>() + sh.begin;
    ReduceArgs r{};
    r.rows_pad = rows_pad;
    r.rows = sh.rows;
    r.scale = norm;
    r.out = outp;
    unsigned int* flag_count = D.flags.as<unsigned int>();
    int nparts = 0;
    if (kernel == FKDE_KERNEL_GAUSSIAN) {
        STATUS_TRY(density_pass(D, o, kModeGauss, rows_pad, n, sc_q, &nparts, dmask, dwords));
        record(D, o, FKDE_T_REDUCE);
        r.part0 = D.part0.as<float>();
        r.nparts = nparts;
        r.ca = 1.0;
        r.cb = 0.0;
        r.accumulate = 0;
        r.flag_count = flag_count;
        r.flag_rows = flag_count + 1;
        r.risk = D.risk.as<uint8_t>();
        r.skip_mass = dmask ? D.qmass.as<float>() : nullptr;
        r.mass_parts = mass_parts;
        r.mass_stride = q_rt;
        if (sh.rows) CUDA_TRY(launch_chain(o.pdl, reduce_density, dim3(grid1(sh.rows, 256)), dim3(256), 0, D.stream, r));
        ++D.launches;
    } else if (fused) {
        // LaplaceFused: phi (1 + d/2 - u) = (1 + d/2) phi + ln2 * phi * log2(phi)
        STATUS_TRY(density_pass(D, o, kModeLaplace, rows_pad, n, sc_q, &nparts, dmask, dwords));
        record(D, o, FKDE_T_REDUCE);
        r.part0 = D.part0.as<float>();
        r.part1 = D.part1.as<float>();
        r.nparts = nparts;
        r.ca = 1.0 + 0.5 * d;
        r.cb = kLn2;
        r.accumulate = 0;
        r.flag_count = flag_count;
        r.flag_rows = flag_count + 1;
        r.risk = D.risk.as<uint8_t>();
        r.skip_mass = dmask ? D.qmass.as<float>() : nullptr;
        r.mass_parts = mass_parts;
        r.mass_stride = q_rt;
        if (sh.rows) CUDA_TRY(launch_chain(o.pdl, reduce_density, dim3(grid1(sh.rows, 256)), dim3(256), 0, D.stream, r));
        ++D.launches;
    } else {
        // engine.cpp:372-379: Gaussian pass, then the correction pass
        // phi (d/2 - u), accumulated into the same values.
        STATUS_TRY(density_pass(D, o, kModeGauss, rows_pad, n, sc_q, &nparts));
        r.part0 = D.part0.as<float>();
        r.nparts = nparts;
        r.ca = 1.0;
        r.cb = 0.0;
        r.accumulate = 0;
        if (sh.rows) CUDA_TRY(launch_chain(o.pdl, reduce_density, dim3(grid1(sh.rows, 256)), dim3(256), 0, D.stream, r));
        ++D.launches;
        STATUS_TRY(density_pass(D, o, kModeLaplace, rows_pad, n, sc_q, &nparts));
        record(D, o, FKDE_T_REDUCE);
        r.part0 = D.part0.as<float>();
        r.part1 = D.part1.as<float>();
        r.nparts = nparts;
        r.ca = 0.5 * d;
        r.cb = kLn2;
        r.accumulate = 1;
        r.flag_count = flag_count;
        r.flag_rows = flag_count + 1;
        r.risk = D.risk.as<uint8_t>();
        if (sh.rows) CUDA_TRY(launch_chain(o.pdl, reduce_density, dim3(grid1(sh.rows, 256)), dim3(256), 0, D.stream, r));
        ++D.launches;
    }
    CUDA_TRY(cudaGetLastError());
    {
        DirectArgs e{};
        e.mode = kernel == FKDE_KERNEL_GAUSSIAN ? kExactGauss : kExactLaplace;
        e.count = flag_count;
        e.rows = flag_count + 1;
        e.rowpts = dQ + sh.begin * d;
        e.row0 = sh.begin;
        e.center_rows = 1;
        e.cols = dCols;
        e.center_cols = cols_centred ? 0 : 1;
        e.n = n;
        e.d = d;
        e.sc = sc_q;
        e.h = J.h;
        e.norm = norm;
        e.out = outp;
        STATUS_TRY(launch_direct(D, o.pdl, e, sh.rows));
    }
    STATUS_TRY(allgather(D, D.out.p, sh.chunk, ncclFloat64));
    if (D.qordered) {   // densities back to the caller's query order
        STATUS_TRY(ensure(D.qout, m * sizeof(double)));
        scatter_rows<<<grid1(m, 256), 256, 0, D.stream>>>(D.out.as<double>(), D.qperm.as<uint32_t>(), m, 1,
                                                          nullptr, D.qout.as<double>());
        ++D.launches;
        CUDA_TRY(cudaGetLastError());
    }
    return {};
}

Status run_job(Device& D, const Options& o, const Job& J) {
    CUDA_TRY(cudaSetDevice(D.dev));
    D.launches = 0;
    for (bool& k : D.kran) k = false;
    if (o.timing && !D.ev[0])
        for (auto& e : D.ev) CUDA_TRY(cudaEventCreate(&e));
    record(D, o, FKDE_T_PREP);
    const int d = J.d;
    const double* dX = J.dX;
    const double* dY = J.dY;
    if (J.kind == Job::kDist) {
        STATUS_TRY(ensure(D.X, J.n * d * sizeof(double)));
        STATUS_TRY(ensure(D.Y, J.m * d * sizeof(double)));
        STATUS_TRY(ensure(D.aux0, (J.n + J.m) * sizeof(double)));
        STATUS_TRY(ensure(D.out, J.n * J.m * sizeof(double)));
        CUDA_TRY(cudaMemcpyAsync(D.X.p, J.hX, J.n * d * 8, cudaMemcpyHostToDevice, D.stream));
        CUDA_TRY(cudaMemcpyAsync(D.Y.p, J.hY, J.m * d * 8, cudaMemcpyHostToDevice, D.stream));
        double* an = D.aux0.as<double>();
        sq_norms_fp64<<<grid1(J.n, 256), 256, 0, D.stream>>>(D.X.as<double>(), J.n, d, an);
        sq_norms_fp64<<<grid1(J.m, 256), 256, 0, D.stream>>>(D.Y.as<double>(), J.m, d, an + J.n);
        dim3 g(grid1(J.m, 128), static_cast<unsigned>(std::min<size_t>(J.n, 65535)));
        block_sq_dists_fp64<<<g, 128, 0, D.stream>>>(D.X.as<double>(), an, J.n, D.Y.as<double>(),
                                                     an + J.n, J.m, d, D.out.as<double>());
        D.launches += 3;
        CUDA_TRY(cudaGetLastError());
        CUDA_TRY(cudaMemcpyAsync(J.out, D.out.p, J.n * J.m * 8, cudaMemcpyDeviceToHost, D.stream));
        CUDA_TRY(cudaStreamSynchronize(D.stream));
        return {};
    }
    if (!dX) {
        STATUS_TRY(ensure(D.X, J.n * d * sizeof(double)));
        CUDA_TRY(cudaMemcpyAsync(D.X.p, J.hX, J.n * d * sizeof(double), cudaMemcpyHostToDevice,
                                 D.stream));
        dX = D.X.as<double>();
    }
    bool y_async = false;
    if (J.m && !dY) {
        STATUS_TRY(ensure(D.Y, J.m * d * sizeof(double)));
        if (J.kind == Job::kSdkde) {
            // the queries are first read by the density pass: their upload runs on the
            // side stream once X's has finished, overlapping the score pass
            CUDA_TRY(cudaEventRecord(D.ev_y_in, D.stream));
            CUDA_TRY(cudaStreamWaitEvent(D.side, D.ev_y_in, 0));
            CUDA_TRY(cudaMemcpyAsync(D.Y.p, J.hY, J.m * d * sizeof(double), cudaMemcpyHostToDevice,
                                     D.side));
            CUDA_TRY(cudaEventRecord(D.ev_y, D.side));
            y_async = true;
        } else {
            CUDA_TRY(cudaMemcpyAsync(D.Y.p, J.hY, J.m * d * sizeof(double), cudaMemcpyHostToDevice,
                                     D.stream));
        }
        dY = D.Y.as<double>();
    }
    STATUS_TRY(ensure(D.scal, 2 * sizeof(PassScalars)));
    // both slots start clean on every call: the non-finite flags read back below
    // must describe this call's inputs only, whichever slots the job writes
    CUDA_TRY(cudaMemsetAsync(D.scal.p, 0, 2 * sizeof(PassScalars), D.stream));
    PassScalars* sc_s = D.scal.as<PassScalars>();
    PassScalars* sc_q = sc_s + 1;
    STATUS_TRY(ensure_call_scratch(
        D, std::max(shard_of(J.n, D.world, D.rank, kTileRows).rows, shard_of(J.m, D.world, D.rank).rows)));

    switch (J.kind) {
        case Job::kScore:
        case Job::kScoreAcc:
            STATUS_TRY(score_program(D, o, J, dX, sc_s, false));
            record(D, o, FKDE_T_QUERY);
            record(D, o, FKDE_T_REDUCE);
            break;
        case Job::kSdkde: {
            STATUS_TRY(score_program(D, o, J, dX, sc_s, true));
            if (J.out2) {
                // debiased samples to the host on the side stream, overlapping the
                // density pass (it only reads D.xsd)
                STATUS_TRY(ensure(D.aux1, J.n * d * sizeof(double)));
                if (D.ordered)   // x_sd = x_sd_c + mu, back in the caller's order
                    scatter_rows<<<grid1(J.n * d, 256), 256, 0, D.stream>>>(
                        D.xsd.as<double>(), D.perm.as<uint32_t>(), J.n, d, sc_s, D.aux1.as<double>());
                else
                    add_mean<<<grid1(J.n * d, 256), 256, 0, D.stream>>>(D.xsd.as<double>(), J.n, d,
                                                                        sc_s, D.aux1.as<double>());
                ++D.launches;
                CUDA_TRY(cudaGetLastError());
                CUDA_TRY(cudaEventRecord(D.ev_side_in, D.stream));
                CUDA_TRY(cudaStreamWaitEvent(D.side, D.ev_side_in, 0));
                CUDA_TRY(cudaMemcpyAsync(J.out2, D.aux1.p, J.n * d * sizeof(double),
                                         cudaMemcpyDeviceToHost, D.side));
                CUDA_TRY(cudaEventRecord(D.ev_side_out, D.side));
            }
            // sc_q: same centring mean (copied from sc_s by scale_two), fresh scale
            // (x_sd is already centred)
            if (y_async) CUDA_TRY(cudaStreamWaitEvent(D.stream, D.ev_y, 0));
            STATUS_TRY(query_program(D, o, J, D.xsd.as<double>(), true, dY, sc_s, sc_q,
                                     FKDE_KERNEL_GAUSSIAN, 1));
            break;
        }
        case Job::kKde: {
            STATUS_TRY(prep(D, o.pdl, dX, J.n, d, 0.0, sc_q, false));   // the mean only
            // large point sets: training points and queries on the spatial order, so
            // the density pass skips tile pairs too (query_program)
            D.ordered = use_spatial(o, J.n);
            if (D.ordered) {
                STATUS_TRY(spatial_order(D, dX, J.n, d, sc_q));
                dX = D.Xs.as<double>();
            }
            record(D, o, FKDE_T_SCORE);
            record(D, o, FKDE_T_FINALIZE);
            record(D, o, FKDE_T_GATHER);
            STATUS_TRY(query_program(D, o, J, dX, false, dY, sc_q, sc_q, J.kernel, J.fused));
            break;
        }
        default:
            break;
    }

    // outputs
    const size_t nd = J.n * d;
    if (J.kind == Job::kSdkde || J.kind == Job::kKde) {
        const void* dens = D.qordered ? D.qout.p : D.out.p;
        if (J.d_out) {
            CUDA_TRY(cudaMemcpyAsync(J.d_out, dens, J.m * sizeof(double), cudaMemcpyDeviceToDevice,
                                     D.stream));
        }
        if (J.out) {
            CUDA_TRY(cudaMemcpyAsync(J.out, dens, J.m * sizeof(double), cudaMemcpyDeviceToHost,
                                     D.stream));
        }
        if (J.kind == Job::kSdkde && J.out2)   // the side-stream copy joins the main stream
            CUDA_TRY(cudaStreamWaitEvent(D.stream, D.ev_side_out, 0));
    } else if (J.kind == Job::kScore) {   // (host outputs only on the first device)
        const void* src = D.ordered ? D.unperm0.p : D.aux0.p;
        if (J.d_out)
            CUDA_TRY(cudaMemcpyAsync(J.d_out, src, nd * sizeof(double), cudaMemcpyDeviceToDevice,
                                     D.stream));
        if (J.out)
            CUDA_TRY(cudaMemcpyAsync(J.out, src, nd * sizeof(double), cudaMemcpyDeviceToHost,
                                     D.stream));
    } else if (J.kind == Job::kScoreAcc) {
        if (J.out)
            CUDA_TRY(cudaMemcpyAsync(J.out, D.ordered ? D.unperm0.p : D.aux0.p, J.n * sizeof(double),
                                     cudaMemcpyDeviceToHost, D.stream));
        if (J.out2)
            CUDA_TRY(cudaMemcpyAsync(J.out2, D.ordered ? D.unperm1.p : D.aux1.p, nd * sizeof(double),
                                     cudaMemcpyDeviceToHost, D.stream));
    }
    record(D, o, FKDE_T_TOTAL);
    if (!J.sync) return {};

    CUDA_TRY(cudaStreamSynchronize(D.stream));
    // input validity (SampleSet::validate) and score underflow (engine.cpp:326-330)
    PassScalars hs[2];
    CUDA_TRY(cudaMemcpy(hs, D.scal.p, sizeof(hs), cudaMemcpyDeviceToHost));
    if (hs[0].nonfinite || hs[1].nonfinite)
        return make_status(FKDE_NON_FINITE, "SampleSet: non-finite entry");
    if (J.kind == Job::kScore || J.kind == Job::kScoreAcc || J.kind == Job::kSdkde) {
        unsigned long long row = ~0ull;
        CUDA_TRY(cudaMemcpy(&row, D.err.p, sizeof(row), cudaMemcpyDeviceToHost));
        if (row != ~0ull && D.ordered) {   // sorted position -> the caller's row index
            uint32_t orig = 0;
            CUDA_TRY(cudaMemcpy(&orig, D.perm.as<uint32_t>() + row, sizeof(orig), cudaMemcpyDeviceToHost));
            row = orig;
        }
        if (row != ~0ull && J.kind != Job::kScoreAcc) {
            Status s = make_status(FKDE_SCORE_UNDERFLOW,
                                   "score denominator underflowed to zero at train point %llu",
                                   row);
            s.index = static_cast<size_t>(row);
            return s;
        }
    }
    return {};
}

// Runs the job on every device of the context (one host thread per device in
// the single-process multi-device case).  Host outputs are written by device 0.
Status run_all(fkde_gpu_ctx* ctx, const Job& J) {
    std::lock_guard<std::mutex> lock(ctx->mu);
    if (ctx->devs.size() == 1) return run_job(ctx->devs[0], ctx->opt, J);
    std::vector<Status> st(ctx->devs.size());
    std::vector<std::thread> th;
    for (size_t i = 0; i < ctx->devs.size(); ++i) {
        Job Ji = J;
        if (i > 0) {
            Ji.out = nullptr;
            Ji.out2 = nullptr;
        }
        th.emplace_back([&, i, Ji] { st[i] = run_job(ctx->devs[i], ctx->opt, Ji); });
    }
    for (auto& t : th) t.join();
    for (auto& s : st)
        if (!s.ok()) return s;
    return {};
}

bool finite_h(double h) { return h > 0.0 && std::isfinite(h); }

Status validate_set(const void* p, size_t n, size_t d, const char* what) {
    if (!p) return make_status(FKDE_INVALID_ARGUMENT, "%s: null pointer", what);
    if (n == 0 || d == 0) return make_status(FKDE_INVALID_ARGUMENT, "SampleSet: n and d must be >= 1");
    if (d > static_cast<size_t>(kMaxDim))
        return make_status(FKDE_UNSUPPORTED_D, "d=%zu exceeds the tensor-core path's limit of %d",
                           d, kMaxDim);
    return {};
}

int finish(fkde_gpu_ctx* ctx, const Status& s, size_t* err_index = nullptr) {
    if (ctx) {
        std::lock_guard<std::mutex> lock(ctx->err_mu);
        ctx->err = s.msg;
        thread_error_slot(ctx) = s.msg;
    }
    if (err_index && s.code == FKDE_SCORE_UNDERFLOW) *err_index = s.index;
    return s.code;
}

Status init_device(Device& D, int dev, int rank, int world) {
    D.dev = dev;
    D.rank = rank;
    D.world = world;
    CUDA_TRY(cudaSetDevice(dev));
    cudaDeviceProp prop;
    CUDA_TRY(cudaGetDeviceProperties(&prop, dev));
    if (prop.major != 10)
        return make_status(FKDE_NO_DEVICE, "device %d is sm_%d%d; this build targets sm_100a", dev,
                           prop.major, prop.minor);
    D.num_sms = prop.multiProcessorCount;
    CUDA_TRY(cudaStreamCreateWithFlags(&D.stream, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&D.side, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&D.ev_side_in, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&D.ev_side_out, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&D.ev_y_in, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&D.ev_y, cudaEventDisableTiming));
    return {};
}

}  // namespace

// =============================================================================
// C ABI
// =============================================================================
extern "C" {

int fkde_gpu_shard_range(size_t n, int world, int rank, size_t align, size_t* begin,
                         size_t* rows, size_t* chunk) {
    if (world < 1 || rank < 0 || rank >= world || align == 0) return FKDE_INVALID_ARGUMENT;
    const Shard s = shard_of(n, world, rank, align);
    if (begin) *begin = s.begin;
    if (rows) *rows = s.rows;
    if (chunk) *chunk = s.chunk;
    return FKDE_OK;
}

int fkde_gpu_device_count(int* count) {
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    if (count) *count = e == cudaSuccess ? c : 0;
    return e == cudaSuccess ? FKDE_OK : FKDE_NO_DEVICE;
}

int fkde_gpu_create(const int* devices, int n_devices, fkde_gpu_ctx** out) {
    if (!out || n_devices < 1) return FKDE_INVALID_ARGUMENT;
    *out = nullptr;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) return FKDE_NO_DEVICE;
    std::vector<int> ids(n_devices);
    for (int i = 0; i < n_devices; ++i) {
        ids[i] = devices ? devices[i] : i;
        if (ids[i] < 0 || ids[i] >= count) return FKDE_INVALID_ARGUMENT;
        // (a repeated id is allowed: ranks sharing a GPU, e.g. over the tests'
        // in-process NCCL emulator; real NCCL rejects it at ncclCommInitAll)
    }
    auto* ctx = new fkde_gpu_ctx();
    ctx->devs.resize(n_devices);
    ctx->world = n_devices;
    for (int i = 0; i < n_devices; ++i) {
        Status s = init_device(ctx->devs[i], ids[i], i, n_devices);
        if (!s.ok()) {
            fkde_gpu_destroy(ctx);
            return s.code;
        }
    }
    if (n_devices > 1) {
        if (!nccl().loaded) {
            fkde_gpu_destroy(ctx);
            return FKDE_NCCL_ERROR;
        }
        std::vector<ncclComm_t> comms(n_devices);
        if (nccl().CommInitAll(comms.data(), n_devices, ids.data()) != ncclSuccess) {
            fkde_gpu_destroy(ctx);
            return FKDE_NCCL_ERROR;
        }
        for (int i = 0; i < n_devices; ++i) ctx->devs[i].comm = comms[i];
    }
    *out = ctx;
    return FKDE_OK;
}

int fkde_gpu_nccl_unique_id(unsigned char id[128]) {
    if (!nccl().loaded) return FKDE_NCCL_ERROR;
    ncclUniqueId uid;
    if (nccl().GetUniqueId(&uid) != ncclSuccess) return FKDE_NCCL_ERROR;
    std::memcpy(id, uid.internal, sizeof(uid.internal));
    return FKDE_OK;
}

int fkde_gpu_create_rank(int device, int rank, int world, const unsigned char id[128],
                         fkde_gpu_ctx** out) {
    if (!out || world < 1 || rank < 0 || rank >= world) return FKDE_INVALID_ARGUMENT;
    *out = nullptr;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) return FKDE_NO_DEVICE;
    if (device < 0 || device >= count) return FKDE_INVALID_ARGUMENT;
    auto* ctx = new fkde_gpu_ctx();
    ctx->devs.resize(1);
    ctx->world = world;
    ctx->per_rank = true;
    Status s = init_device(ctx->devs[0], device, rank, world);
    if (!s.ok()) {
        fkde_gpu_destroy(ctx);
        return s.code;
    }
    if (world > 1) {
        if (!nccl().loaded || !id) {
            fkde_gpu_destroy(ctx);
            return FKDE_NCCL_ERROR;
        }
        ncclUniqueId uid;
        std::memcpy(uid.internal, id, sizeof(uid.internal));
        if (nccl().CommInitRank(&ctx->devs[0].comm, world, uid, rank) != ncclSuccess) {
            fkde_gpu_destroy(ctx);
            return FKDE_NCCL_ERROR;
        }
    }
    *out = ctx;
    return FKDE_OK;
}

void fkde_gpu_destroy(fkde_gpu_ctx* ctx) {
    if (!ctx) return;
    for (size_t i = 0; i < t_errors.size(); ++i)
        if (t_errors[i].ctx == ctx) {
            t_errors.erase(t_errors.begin() + i);
            break;
        }
    for (auto& D : ctx->devs) {
        cudaSetDevice(D.dev);
        if (D.stream) cudaStreamSynchronize(D.stream);
        if (D.comm && nccl().loaded) nccl().CommDestroy(D.comm);
        for (DevBuf* b : D.buffers())
            if (b->p) cudaFree(b->p);
        for (auto& e : D.ev)
            if (e) cudaEventDestroy(e);
        if (D.graph) cudaGraphExecDestroy(D.graph);
        if (D.stream) cudaStreamDestroy(D.stream);
        if (D.side) cudaStreamDestroy(D.side);
        if (D.ev_side_in) cudaEventDestroy(D.ev_side_in);
        if (D.ev_side_out) cudaEventDestroy(D.ev_side_out);
        if (D.ev_y_in) cudaEventDestroy(D.ev_y_in);
        for (cudaEvent_t e : D.kev)
            if (e) cudaEventDestroy(e);
        if (D.ev_y) cudaEventDestroy(D.ev_y);
    }
    delete ctx;
}

const char* fkde_gpu_last_error(const fkde_gpu_ctx* ctx) {
    if (!ctx) return "";
    for (auto& e : t_errors)
        if (e.ctx == ctx) return e.msg.c_str();
    // this thread made no call on ctx: a private copy of the context's last message
    auto* c = const_cast<fkde_gpu_ctx*>(ctx);
    std::lock_guard<std::mutex> lock(c->err_mu);
    std::string& slot = thread_error_slot(ctx);
    slot = c->err;
    return slot.c_str();
}

int fkde_gpu_set_option(fkde_gpu_ctx* ctx, int key, int64_t value) {
    if (!ctx) return FKDE_INVALID_ARGUMENT;
    switch (key) {
        case FKDE_OPT_ENGINE:
            if (value != FKDE_ENGINE_TC) return FKDE_INVALID_ARGUMENT;   // the only engine
            ctx->opt.engine = static_cast<int>(value);
            return FKDE_OK;
        case FKDE_OPT_SPLITS:
            if (value < 0) return FKDE_INVALID_ARGUMENT;
            ctx->opt.splits = static_cast<int>(value);
            return FKDE_OK;
        case FKDE_OPT_TIMING:
            ctx->opt.timing = value ? 1 : 0;
            return FKDE_OK;
        case FKDE_OPT_MAX_CTAS:
            if (value < 0) return FKDE_INVALID_ARGUMENT;
            ctx->opt.max_ctas = static_cast<int>(value);
            return FKDE_OK;
        case FKDE_OPT_TRACE_PTR:
            ctx->opt.trace = reinterpret_cast<long long*>(value);
            return FKDE_OK;
        case FKDE_OPT_PDL:
            ctx->opt.pdl = value != 0;
            return FKDE_OK;
        case FKDE_OPT_SPATIAL:
            if (value < 0 || value > 3) return FKDE_INVALID_ARGUMENT;
            ctx->opt.spatial = static_cast<int>(value);
            return FKDE_OK;
        case FKDE_OPT_FLUSH_TILES:
            if (value < 0 || value > 1 << 20 || (value & (value - 1))) return FKDE_INVALID_ARGUMENT;
            ctx->opt.flush_tiles = static_cast<int>(value);
            return FKDE_OK;
        default:
            return FKDE_INVALID_ARGUMENT;
    }
}

int fkde_gpu_world(const fkde_gpu_ctx* ctx, int* rank, int* world) {
    if (!ctx) return FKDE_INVALID_ARGUMENT;
    if (rank) *rank = ctx->devs[0].rank;
    if (world) *world = ctx->world;
    return FKDE_OK;
}

void* fkde_gpu_stream(fkde_gpu_ctx* ctx) {
    return ctx ? static_cast<void*>(ctx->devs[0].stream) : nullptr;
}

int fkde_gpu_last_timing(const fkde_gpu_ctx* ctx, float* ms, int n) {
    if (!ctx || !ms) return FKDE_INVALID_ARGUMENT;
    const Device& D = ctx->devs[0];
    if (!ctx->opt.timing || !D.ev[0]) {
        for (int i = 0; i < n && i < FKDE_T_COUNT; ++i) ms[i] = 0.f;
        return FKDE_OK;
    }
    cudaSetDevice(D.dev);
    if (cudaEventSynchronize(D.ev[FKDE_T_TOTAL]) != cudaSuccess) return FKDE_CUDA_ERROR;
    for (int i = 0; i < n && i < FKDE_T_COUNT; ++i) {
        float v = 0.f;
        if (i < FKDE_T_TOTAL)
            cudaEventElapsedTime(&v, D.ev[i], D.ev[i + 1]);
        else
            cudaEventElapsedTime(&v, D.ev[FKDE_T_PREP], D.ev[FKDE_T_TOTAL]);
        ms[i] = v;
    }
    return FKDE_OK;
}

int fkde_gpu_workspace_bytes(const fkde_gpu_ctx* ctx, size_t* bytes) {
    if (!ctx || !bytes) return FKDE_INVALID_ARGUMENT;
    size_t total = 0;
    for (const Device& D : ctx->devs) {
        for (const DevBuf* b : const_cast<Device&>(D).buffers()) total += b->bytes;
    }
    *bytes = total;
    return FKDE_OK;
}

int fkde_gpu_last_skip_stats(fkde_gpu_ctx* ctx, uint64_t* out, size_t n) {
    if (!ctx || (!out && n)) return FKDE_INVALID_ARGUMENT;
    const Device& D = ctx->devs[0];
    uint64_t v[FKDE_SKIP_STATS_COUNT] = {};
    if (D.skipstats.p) {
        cudaSetDevice(D.dev);
        if (cudaStreamSynchronize(D.stream) != cudaSuccess) return FKDE_CUDA_ERROR;
        unsigned long long h[2] = {0, 0};
        if (cudaMemcpy(h, D.skipstats.p, sizeof(h), cudaMemcpyDeviceToHost) != cudaSuccess)
            return FKDE_CUDA_ERROR;
        uint64_t skipped = 0;
        if (D.mask_bytes) {   // popcount of the score pass's skip mask
            std::vector<uint32_t> m(D.mask_bytes / sizeof(uint32_t));
            if (cudaMemcpy(m.data(), D.smask.p, D.mask_bytes, cudaMemcpyDeviceToHost) != cudaSuccess)
                return FKDE_CUDA_ERROR;
            for (uint32_t w : m) skipped += static_cast<uint64_t>(__builtin_popcount(w));
        }
        uint64_t dskipped = 0;
        if (D.dtiles_rows) {   // the density pass's per-query-tile skip counts
            std::vector<unsigned int> c(D.dtiles_rows);
            if (cudaMemcpy(c.data(), D.qskip.p, c.size() * sizeof(unsigned int), cudaMemcpyDeviceToHost) !=
                cudaSuccess)
                return FKDE_CUDA_ERROR;
            for (unsigned int x : c) dskipped += x;
        }
        unsigned int dflag = 0;
        if (D.flags.p && cudaMemcpy(&dflag, D.flags.p, sizeof(dflag), cudaMemcpyDeviceToHost) != cudaSuccess)
            return FKDE_CUDA_ERROR;
        v[0] = h[0];
        v[1] = skipped;
        v[2] = D.tiles_total;
        v[3] = D.ordered ? 1 : 0;
        v[4] = dskipped;
        v[5] = D.dtiles_total;
        v[6] = D.qordered ? 1 : 0;
        v[7] = dflag;
        v[8] = h[1] & 0xFFFFFFFFull;
    }
    for (size_t i = 0; i < n && i < FKDE_SKIP_STATS_COUNT; ++i) out[i] = v[i];
    return FKDE_OK;
}

int fkde_gpu_last_kernel_timing(const fkde_gpu_ctx* ctx, float* ms, int n) {
    if (!ctx || (!ms && n > 0)) return FKDE_INVALID_ARGUMENT;
    const Device& D = ctx->devs[0];
    for (int i = 0; i < n && i < FKDE_KT_COUNT; ++i) ms[i] = 0.f;
    if (!ctx->opt.timing || !D.kev[0]) return FKDE_OK;
    cudaSetDevice(D.dev);
    for (int i = 0; i < n && i < FKDE_KT_COUNT; ++i) {
        if (!D.kran[i]) continue;
        if (cudaEventSynchronize(D.kev[2 * i + 1]) != cudaSuccess) return FKDE_CUDA_ERROR;
        float v = 0.f;
        if (cudaEventElapsedTime(&v, D.kev[2 * i], D.kev[2 * i + 1]) != cudaSuccess) return FKDE_CUDA_ERROR;
        ms[i] = v;
    }
    return FKDE_OK;
}

int64_t fkde_gpu_last_launch_count(const fkde_gpu_ctx* ctx) {
    return ctx ? ctx->devs[0].launches : 0;
}

int fkde_gpu_score(fkde_gpu_ctx* ctx, const double* X, size_t n, size_t d, double h_score,
                   double* scores, size_t* err_index) {
    if (!ctx) return FKDE_INVALID_ARGUMENT;
    Status s = validate_set(X, n, d, "train");
    if (s.ok() && !finite_h(h_score))
        s = make_status(FKDE_INVALID_ARGUMENT, "Bandwidth: h_score must be positive and finite");
    if (s.ok() && !scores) s = make_status(FKDE_INVALID_ARGUMENT, "scores: null pointer");
    if (!s.ok()) return finish(ctx, s);
    Job J;
    J.kind = Job::kScore;
    J.hX = X;
    J.n = n;
    J.d = static_cast<int>(d);
    J.h = h_score;
    J.h_score = h_score;
    J.out = scores;
    return finish(ctx, run_all(ctx, J), err_index);
}

int fkde_gpu_score_accumulate(fkde_gpu_ctx* ctx, const double* X, size_t n, size_t d,
                              double h_score, double* phi_sum, double* weighted) {
    if (!ctx) return FKDE_INVALID_ARGUMENT;
    Status s = validate_set(X, n, d, "train");
    if (s.ok() && !finite_h(h_score))
        s = make_status(FKDE_INVALID_ARGUMENT, "Bandwidth: h_score must be positive and finite");
    if (s.ok() && (!phi_sum || !weighted))
        s = make_status(FKDE_INVALID_ARGUMENT, "outputs: null pointer");
    if (!s.ok()) return finish(ctx, s);
    Job J;
    J.kind = Job::kScoreAcc;
    J.hX = X;
    J.n = n;
    J.d = static_cast<int>(d);
    J.h = h_score;
    J.h_score = h_score;
    J.out = phi_sum;
    J.out2 = weighted;
    return finish(ctx, run_all(ctx, J));
}

static Status validate_pair(const void* X, size_t n, const void* Y, size_t m, size_t d, double h) {
    Status s = validate_set(X, n, d, "train");
    if (s.ok()) s = validate_set(Y, m, d, "queries");
    if (s.ok() && !finite_h(h))
        s = make_status(FKDE_INVALID_ARGUMENT, "Bandwidth: h must be positive and finite");
    return s;
}

int fkde_gpu_kde(fkde_gpu_ctx* ctx, const double* X, size_t n, const double* Y, size_t m,
                 size_t d, double h, int kernel, int fused, double* out) {
    if (!ctx) return FKDE_INVALID_ARGUMENT;
    Status s = validate_pair(X, n, Y, m, d, h);
    if (s.ok() && kernel != FKDE_KERNEL_GAUSSIAN && kernel != FKDE_KERNEL_LAPLACE_CORRECTED)
        s = make_status(FKDE_INVALID_ARGUMENT, "unknown kernel kind %d", kernel);
    if (s.ok() && !out) s = make_status(FKDE_INVALID_ARGUMENT, "out: null pointer");
    if (!s.ok()) return finish(ctx, s);
    Job J;
    J.kind = Job::kKde;
    J.hX = X;
    J.hY = Y;
    J.n = n;
    J.m = m;
    J.d = static_cast<int>(d);
    J.h = h;
    J.kernel = kernel;
    J.fused = fused;
    J.out = out;
    return finish(ctx, run_all(ctx, J));
}

int fkde_gpu_sdkde(fkde_gpu_ctx* ctx, const double* X, size_t n, const double* Y, size_t m,
                   size_t d, double h, double h_score, double* out, double* debiased,
                   size_t* err_index) {
    if (!ctx) return FKDE_INVALID_ARGUMENT;
    Status s = validate_pair(X, n, Y, m, d, h);
    if (s.ok() && !finite_h(h_score))
        s = make_status(FKDE_INVALID_ARGUMENT, "Bandwidth: h_score must be positive and finite");
    if (s.ok() && !out) s = make_status(FKDE_INVALID_ARGUMENT, "out: null pointer");
    if (!s.ok()) return finish(ctx, s);
    Job J;
    J.kind = Job::kSdkde;
    J.hX = X;
    J.hY = Y;
    J.n = n;
    J.m = m;
    J.d = static_cast<int>(d);
    J.h = h;
    J.h_score = h_score;
    J.out = out;
    J.out2 = debiased;
    return finish(ctx, run_all(ctx, J), err_index);
}

int fkde_gpu_estimate(fkde_gpu_ctx* ctx, const double* X, size_t n, const double* Y, size_t m,
                      size_t d, int method, double h, double h_score, size_t tile_m,
                      size_t tile_n, int fused, double* out, double* debiased,
                      double* negative_mass, size_t* err_index) {
    if (!ctx) return FKDE_INVALID_ARGUMENT;
    // EstimatorConfig::validate (types.cpp:74-79)
    if (!finite_h(h))
        return finish(ctx, make_status(FKDE_INVALID_ARGUMENT, "Bandwidth: h must be positive and finite"));
    if (!finite_h(h_score))
        return finish(ctx, make_status(FKDE_INVALID_ARGUMENT,
                                       "Bandwidth: h_score must be positive and finite"));
    if (tile_m == 0 || tile_n == 0)
        return finish(ctx, make_status(FKDE_INVALID_ARGUMENT,
                                       "EstimatorConfig: tile_m and tile_n must be >= 1"));
    int rc;
    switch (method) {
        case FKDE_METHOD_KDE:
            rc = fkde_gpu_kde(ctx, X, n, Y, m, d, h, FKDE_KERNEL_GAUSSIAN, 1, out);
            break;
        case FKDE_METHOD_SDKDE:
            rc = fkde_gpu_sdkde(ctx, X, n, Y, m, d, h, h_score, out, debiased, err_index);
            break;
        case FKDE_METHOD_LAPLACE:
            rc = fkde_gpu_kde(ctx, X, n, Y, m, d, h, FKDE_KERNEL_LAPLACE_CORRECTED, fused, out);
            if (rc == FKDE_OK && negative_mass) {  // estimator.cpp:14-20
                double acc = 0.0;
                for (size_t j = 0; j < m; ++j) acc += std::max(0.0, -out[j]);
                *negative_mass = acc / static_cast<double>(m);
            }
            break;
        default:
            return finish(ctx, make_status(FKDE_INVALID_ARGUMENT, "estimate: unknown method"));
    }
    return rc;
}

int fkde_gpu_pairwise_sq_dists(fkde_gpu_ctx* ctx, const double* A, size_t na, const double* B,
                               size_t nb, size_t d, double* out) {
    if (!ctx) return FKDE_INVALID_ARGUMENT;
    Status s = validate_set(A, na, std::min<size_t>(d, 1), "a");
    if (s.ok()) s = validate_set(B, nb, std::min<size_t>(d, 1), "b");
    if (s.ok() && d == 0) s = make_status(FKDE_INVALID_ARGUMENT, "SampleSet: n and d must be >= 1");
    if (s.ok() && !out) s = make_status(FKDE_INVALID_ARGUMENT, "out: null pointer");
    if (!s.ok()) return finish(ctx, s);
    for (size_t i = 0; i < na * d; ++i)
        if (!std::isfinite(A[i])) return finish(ctx, make_status(FKDE_NON_FINITE, "SampleSet: non-finite entry"));
    for (size_t i = 0; i < nb * d; ++i)
        if (!std::isfinite(B[i])) return finish(ctx, make_status(FKDE_NON_FINITE, "SampleSet: non-finite entry"));
    Job J;
    J.kind = Job::kDist;
    J.hX = A;
    J.hY = B;
    J.n = na;
    J.m = nb;
    J.d = static_cast<int>(d);
    J.out = out;
    std::lock_guard<std::mutex> lock(ctx->mu);
    return finish(ctx, run_job(ctx->devs[0], ctx->opt, J));
}

namespace {
// Device-resident jobs (J.sync == false, single rank): the first call with a
// given argument/option set runs eagerly (and makes every allocation), the
// second is captured into a CUDA graph, later ones replay it.
Status run_device_job(fkde_gpu_ctx* ctx, const Job& J) {
    Device& D = ctx->devs[0];
    const Options& o = ctx->opt;
    // (per-phase event timing and the debug trace run eagerly)
    if (D.world != 1 || o.trace || o.timing) return run_job(D, o, J);
    char buf[512];
    std::snprintf(buf, sizeof(buf), "%d|%p|%p|%p|%zu|%zu|%d|%a|%a|%d|%d|%d|%d|%d|%d|%d|%d", J.kind,
                  (const void*)J.dX, (const void*)J.dY, (void*)J.d_out, J.n, J.m, J.d, J.h,
                  J.h_score, J.kernel, J.fused, o.engine, o.splits, o.timing, o.max_ctas,
                  o.flush_tiles, o.spatial * 2 + (o.pdl ? 1 : 0));
    const std::string key(buf);
    CUDA_TRY(cudaSetDevice(D.dev));
    if (D.graph && key == D.graph_key && D.graph_epoch == g_alloc_epoch.load()) {
        CUDA_TRY(cudaGraphLaunch(D.graph, D.stream));
        D.launches = D.graph_launches;
        return {};
    }
    if (key != D.graph_seen) {   // first sighting: eager
        D.graph_seen = key;
        return run_job(D, o, J);
    }
    if (D.graph) {
        cudaGraphExecDestroy(D.graph);
        D.graph = nullptr;
        D.graph_key.clear();
    }
    cudaGraph_t g = nullptr;
    CUDA_TRY(cudaStreamBeginCapture(D.stream, cudaStreamCaptureModeThreadLocal));
    Status s = run_job(D, o, J);
    const cudaError_t ce = cudaStreamEndCapture(D.stream, &g);
    if (!s.ok()) {
        if (g) cudaGraphDestroy(g);
        return s;
    }
    if (ce != cudaSuccess) return make_status(FKDE_CUDA_ERROR, "stream capture: %s", cudaGetErrorString(ce));
    const cudaError_t ie = cudaGraphInstantiate(&D.graph, g, 0);
    cudaGraphDestroy(g);
    if (ie != cudaSuccess) {
        D.graph = nullptr;
        return make_status(FKDE_CUDA_ERROR, "graph instantiate: %s", cudaGetErrorString(ie));
    }
    D.graph_key = key;
    D.graph_launches = D.launches;
    D.graph_epoch = g_alloc_epoch.load();
    CUDA_TRY(cudaGraphLaunch(D.graph, D.stream));
    return {};
}
}  // namespace

int fkde_gpu_sdkde_device(fkde_gpu_ctx* ctx, const double* dX, size_t n, const double* dY,
                          size_t m, size_t d, double h, double h_score, double* d_out) {
    if (!ctx) return FKDE_INVALID_ARGUMENT;
    if (ctx->devs.size() != 1)
        return finish(ctx, make_status(FKDE_INVALID_ARGUMENT, "device API needs a 1-device context"));
    Status s = validate_pair(dX, n, dY, m, d, h);
    if (s.ok() && !finite_h(h_score))
        s = make_status(FKDE_INVALID_ARGUMENT, "Bandwidth: h_score must be positive and finite");
    if (s.ok() && !d_out) s = make_status(FKDE_INVALID_ARGUMENT, "out: null pointer");
    if (!s.ok()) return finish(ctx, s);
    Job J;
    J.kind = Job::kSdkde;
    J.dX = dX;
    J.dY = dY;
    J.n = n;
    J.m = m;
    J.d = static_cast<int>(d);
    J.h = h;
    J.h_score = h_score;
    J.d_out = d_out;
    J.sync = false;
    std::lock_guard<std::mutex> lock(ctx->mu);
    return finish(ctx, run_device_job(ctx, J));
}

int fkde_gpu_score_device(fkde_gpu_ctx* ctx, const double* dX, size_t n, size_t d, double h_score,
                          double* d_scores) {
    if (!ctx) return FKDE_INVALID_ARGUMENT;
    if (ctx->devs.size() != 1)
        return finish(ctx, make_status(FKDE_INVALID_ARGUMENT, "device API needs a 1-device context"));
    Status s = validate_set(dX, n, d, "score train");
    if (s.ok() && !finite_h(h_score))
        s = make_status(FKDE_INVALID_ARGUMENT, "score_flash: h_score must be positive and finite");
    if (s.ok() && !d_scores) s = make_status(FKDE_INVALID_ARGUMENT, "score_flash: null output");
    if (!s.ok()) return finish(ctx, s);
    Job J;
    J.kind = Job::kScore;
    J.dX = dX;
    J.n = n;
    J.d = static_cast<int>(d);
    J.h = h_score;
    J.h_score = h_score;
    J.d_out = d_scores;
    J.sync = false;
    std::lock_guard<std::mutex> lock(ctx->mu);
    return finish(ctx, run_device_job(ctx, J));
}

int fkde_gpu_kde_device(fkde_gpu_ctx* ctx, const double* dX, size_t n, const double* dY,
                        size_t m, size_t d, double h, int kernel, int fused, double* d_out) {
    if (!ctx) return FKDE_INVALID_ARGUMENT;
    if (ctx->devs.size() != 1)
        return finish(ctx, make_status(FKDE_INVALID_ARGUMENT, "device API needs a 1-device context"));
    Status s = validate_pair(dX, n, dY, m, d, h);
    if (s.ok() && kernel != FKDE_KERNEL_GAUSSIAN && kernel != FKDE_KERNEL_LAPLACE_CORRECTED)
        s = make_status(FKDE_INVALID_ARGUMENT, "unknown kernel kind %d", kernel);
    if (s.ok() && !d_out) s = make_status(FKDE_INVALID_ARGUMENT, "out: null pointer");
    if (!s.ok()) return finish(ctx, s);
    Job J;
    J.kind = Job::kKde;
    J.dX = dX;
    J.dY = dY;
    J.n = n;
    J.m = m;
    J.d = static_cast<int>(d);
    J.h = h;
    J.kernel = kernel;
    J.fused = fused;
    J.d_out = d_out;
    J.sync = false;
    std::lock_guard<std::mutex> lock(ctx->mu);
    return finish(ctx, run_device_job(ctx, J));
}

}  // extern "C"
