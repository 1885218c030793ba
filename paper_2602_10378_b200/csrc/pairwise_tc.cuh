// pairwise_tc.cuh -- the two O(n^2) passes of Flash-SD-KDE as one persistent,
// warp-specialised sm_100a kernel (tcgen05 + TMEM + bulk-async copies).
//
// Reference: fkde::engine::stream_score_totals (engine.cpp:172-244) and
// stream_kde_pass (engine.cpp:103-168).  The reference tiles the conceptual
// (rows x cols) pair matrix into tile_m x tile_n blocks, forms each block's
// squared distances with a Gram GEMM + norm expansion (engine.cpp:41-51),
// applies exp (engine.cpp:83-97/197) and reduces row sums (engine.cpp:128,198)
// and, for the score, the second product Phi_tile * X_j (engine.cpp:199).
//
// Here one work unit = (128-row tile, contiguous range of column tiles: 96
// points in the score pass, 128 in the density passes).  Per column tile:
//   GEMM1  S[128xN] = A_rows(128x64 fp16) . B_cols(Nx64 fp16)^T  -> TMEM
//          (S is log2(phi) directly; see layout.cuh)
//   epilogue warps: tcgen05.ld S -> phi = ex2(S*dscale) in registers;
//          KDE: row sums (Gaussian) or (sum phi, sum phi*log2 phi) (Laplace);
//          SCORE: phi -> fp16 hi/lo -> tcgen05.st back into S's own TMEM
//          columns (P aliases S, flash-attention-4 style: no SMEM round trip)
//   GEMM2 (SCORE only, A from TMEM)  O[128x48] += P_hi . B[:, 0:48] + P_lo . B[:, 0:32]
//          (B = the same column tile, MN-major) -> sum_j phi y_hi_j,
//          sum_j phi y_lo_j, sum_j phi  (TMEM, fp32; drained by the drain warps)
// The n x n kernel matrix never leaves the SM; per column tile the SMEM
// traffic is the 12 KiB B tile read by both GEMMs and the 16 KiB A tile.
//
// Tile skipping (score pass on the spatial order, spatial_order.cuh): the score
// pass carries phi' = phi 2^15 as fp16 hi + lo, so a pair with log2 phi' < -25
// contributes exactly zero.  A CHECK pass (MODE kModeCheck: GEMM1 + an exact
// max over the tile, no exps) visits the tile pairs a centroid predictor marked
// (pred mask) and leaves in the skip mask those whose every pair is below
// kSkipLog2; the SCORE pass then visits only the column tiles whose skip bit is
// clear.  A skipped tile would have added exact zeros: the result is the same as
// visiting it.
//
// Warp roles: warp 0 = bulk-copy producer, warp 1 = TMEM owner + GEMM1 issuer;
// score pass: warp 2 = GEMM2 issuer, warps 4..7 = O drain warps (one per TMEM
// lane quadrant), warps 8.. = epilogue; KDE / check: warps 2.. = epilogue.
// Epilogue warp w reads TMEM lane quadrant w%4 of every kNP-th tile.  Pipelines
// (mbarriers): A tiles x2, B tiles x kStages, S/P accumulators x kSBuf (TMEM),
// O x2 (TMEM, score).
#pragma once
#include <cuda_fp16.h>
#include <climits>
#include <cstdint>

#include "layout.cuh"
#include "ptx.cuh"

namespace fkde_b200 {

enum PairMode : int {
    kModeScore = 0,     // stream_score_totals
    kModeGauss = 1,     // stream_kde_pass, PairTerm::Gaussian
    kModeLaplace = 2,   // two sums (phi, phi*log2 phi): LaplaceFused / LaplaceCorrection
    kModeCheck = 3,     // score tile skipping: exact per-tile max of log2 phi' (no exps)
};

struct PairArgs {
    const uint8_t* opA;   // row tiles (A format), n_row_tiles * 16 KiB
    const uint8_t* opB;   // column tiles (B format), n_col_tiles * kColBytes
    int n_row_tiles;
    int n_col_tiles;
    int splits;           // column ranges per row tile
    const PassScalars* sc;
    float* part0;         // KDE: [splits*kNP][rows_pad]
    float* part1;         // Laplace: [splits*kNP][rows_pad]
    double* dpart0;       // SCORE: S' [splits][rows_pad]   (fp64)
    double* dpart1;       // SCORE: T' [splits][rows_pad][16] (fp64)
    int flush_log2;       // SCORE: O is drained every 2^flush_log2 visited column tiles
    size_t rows_pad;
    // SCORE: column tile holding row tile 0's diagonal (rows and columns are
    // the same point set, row shard starting at global point diag_row0); the self pair
    // phi_ii = 1 is excluded from the tensor-core sums and added back exactly
    // in finalize_score, so that T - x S never cancels against the self term.
    long long diag_row0;  // -1: no diagonal
    // tile masks, one bit per (row tile, column tile), rows of mask_words words:
    //   SCORE / KDE: skip_mask (nullptr = visit every tile): visit tiles whose bit is 0
    //   CHECK: pred_mask selects the tiles to check (bit 1); skip_mask starts as a
    //          copy of it and loses the bit of every tile that is not skippable
    const uint32_t* pred_mask;
    uint32_t* skip_mask;
    int mask_words;
    unsigned long long* stats;   // CHECK (optional): [0] += tiles checked
    // dynamic unit scheduler: [0] next unit (atomic fetch-and-add by each CTA's
    // producer), [1] CTAs finished; both zero at launch, reset by the last CTA
    unsigned int* sched;
    // SCORE on the spatial order (nullptr otherwise): GEMM2's column operand centred
    // per column tile (layout.cuh "B2") and the column-tile centroids the drain adds
    // back (log2 units, unscaled).  Tiles are grouped by 2^kB2GroupLog2 consecutive
    // column tiles; tile J's ones column is 16 + (J mod 2^kB2GroupLog2), so an O
    // sub-unit may hold several tiles of one group and still give each tile's own
    // S_J for its centroid term c_J S_J.  A sub-unit never spans two groups: it ends
    // at a group change or after 2^flush_log2 visited tiles.
    const uint8_t* opB2;
    const float* cenB;
    // debug (builds with -DFKDE_ENABLE_TRACE only): per-event clock64 trace of
    // block 0 (nullptr = off).  Layout [warp][event slot][tile] -> long long
    long long* trace;
};
// log2 phi' (S * dscale, with the 2^15 offset) below which both fp16 halves of
// phi' are exactly zero (phi' < 2^-25 rounds to zero; one unit of margin for ex2.approx)
constexpr float kSkipLog2 = -26.0f;
// score epilogue: unroll factor of the per-tile loop over 32-column chunks (1: fully
// unrolled, 3, made the score phase ~2 % slower in an interleaved A/B)
#ifndef FKDE_SCORE_CH_UNROLL
#define FKDE_SCORE_CH_UNROLL 1
#endif
constexpr int kScoreChUnroll = FKDE_SCORE_CH_UNROLL;
// score pass on the spatial order: column tiles per B2 group (ones columns 16 .. 16 + 2^glog - 1)
#ifndef FKDE_B2_GROUP_LOG2
#define FKDE_B2_GROUP_LOG2 3
#endif
constexpr int kB2GroupLog2 = FKDE_B2_GROUP_LOG2;
static_assert(kB2GroupLog2 >= 2 && kB2GroupLog2 <= 4, "ones columns 16 .. 16 + 2^glog - 1 within the block");

#ifdef FKDE_ENABLE_TRACE
#define FKDE_TRACE(slot, tile)                                                               \
    do {                                                                                     \
        if (args.trace && blockIdx.x == 0 && lane == 0 && (tile) < 256)                      \
            args.trace[(warp * 8 + (slot)) * 256 + (tile)] = clock64();                      \
    } while (0)
#else
#define FKDE_TRACE(slot, tile) \
    do {                       \
    } while (0)
#endif

// Column tiles of one unit that a pass visits: [.., end) filtered by a mask row
// (bit == want).  Every warp of the CTA walks the same sequence, warp-uniformly
// (first / next / count are called by whole converged warps), keeping the current
// word's remaining bits in a register.  kWindow (the check pass, whose predicted
// set is ~2 % dense): a window of the next 32 mask words is held one per lane,
// loaded together, and the next non-empty word is found by a ballot -- one L2
// round trip per 32 words instead of one per word, which was one per visited tile
// on such a sparse mask.  The score / density masks are ~30 % dense (a load per ~9
// visited tiles), where the window's registers cost more (spills in the control
// warps) than the loads it saves.
template <bool kWindow>
struct TileWalkT {
    const uint32_t* row;   // nullptr: every tile
    int end;
    uint32_t want;         // 0u: visit clear bits, ~0u: visit set bits
    int w = 0;             // current word
    uint32_t bits = 0;     // visited tiles of word w not yet returned
    int base = 0;          // kWindow: lane l holds word base + l (0 past the range)
    uint32_t cache = 0;    // !kWindow: word w + 1 (prefetched)
    __device__ __forceinline__ uint32_t word(int i) const { return ~(row[i] ^ want); }
    __device__ __forceinline__ void load(int b) {
        base = b;
        const int i = b + static_cast<int>(threadIdx.x & 31u);
        cache = (i << 5) < end ? word(i) : 0u;
    }
    __device__ __forceinline__ int first(int from) {   // first visited tile >= from, or end
        if (!row) {
            w = from;
            return from < end ? from : end;
        }
        if (from >= end) return end;
        w = from >> 5;
        if constexpr (kWindow) {
            load(w);
            bits = __shfl_sync(0xffffffffu, cache, 0) & (0xFFFFFFFFu << (from & 31));
        } else {
            bits = word(w) & (0xFFFFFFFFu << (from & 31));
            cache = ((w + 1) << 5) < end ? word(w + 1) : 0u;   // the next word, in flight
        }
        return next();
    }
    __device__ __forceinline__ int next() {   // the following visited tile, or end
        if (!row) {
            ++w;
            return w < end ? w : end;
        }
        while (!bits) {
            if constexpr (kWindow) {
                const int lane = static_cast<int>(threadIdx.x & 31u);
                const unsigned ahead = __ballot_sync(0xffffffffu, cache != 0u && base + lane > w);
                if (ahead) {
                    const int l = __ffs(ahead) - 1;
                    w = base + l;
                    bits = __shfl_sync(0xffffffffu, cache, l);
                } else {
                    if (((base + 32) << 5) >= end) return end;
                    load(base + 32);
                    w = base - 1;
                }
            } else {
                // the next word was loaded one word ahead, so its L2 round trip
                // overlaps the visited tiles of this one (the GEMM2 issuer's walk
                // sits on the S/P ring's critical path)
                if (((w + 1) << 5) >= end) return end;
                bits = cache;
                ++w;
                cache = ((w + 1) << 5) < end ? word(w + 1) : 0u;
            }
        }
        const int c = (w << 5) + __ffs(bits) - 1;
        bits &= bits - 1u;
        return c < end ? c : end;
    }
    // visited tiles in [from, end).  Called by whole converged warps (every role
    // walks its units warp-uniformly): the lanes load the range's mask words in
    // parallel and the popcounts are reduced across the warp.  (One lane walking the
    // ~50 words of a unit's column range serially put ~50 dependent L2 round trips
    // at the start of every unit in every warp: 24 % of the check kernel's stall
    // samples, ncu source view.)
    __device__ __forceinline__ int count(int from) const {
        if (!row) return end > from ? end - from : 0;
        if (from >= end) return 0;
        const int lane = static_cast<int>(threadIdx.x & 31u);
        const int w0 = from >> 5, w1 = (end - 1) >> 5;
        int n = 0;
        for (int i = w0 + lane; i <= w1; i += 32) {
            uint32_t b = word(i);
            if (i == w0) b &= 0xFFFFFFFFu << (from & 31);
            const int top = end - (i << 5);
            if (top < 32) b &= (1u << top) - 1u;
            n += __popc(b);
        }
        return static_cast<int>(__reduce_add_sync(0xffffffffu, static_cast<unsigned>(n)));
    }
};

template <int MODE>
struct TcConfig {
    static constexpr bool kScore = MODE == kModeScore;
    static constexpr bool kCheck = MODE == kModeCheck;
    static constexpr bool kScoreTiling = kScore || kCheck;   // 96-column tiles
    // KDE / CHECK: warps 0 producer, 1 GEMM1 issuer (+ TMEM owner), 2 .. 2+4*kNP-1
    // epilogue (kNP warps per TMEM lane quadrant, one per SM sub-partition each).
    // SCORE: warpgroup 0 = control (0 producer, 1 GEMM1 issuer + TMEM owner,
    // 2 GEMM2 issuer, 3 idle), warpgroups 1..kNP = epilogue.  tcgen05.mma issue
    // blocks while the tensor core is busy, so GEMM1 and GEMM2 get their own
    // issuing warps and the tensor core never idles behind a GEMM2 that waits for
    // P.  The control warpgroup gives its registers to the epilogue warpgroups
    // (setmaxnreg), which is what makes four epilogue warps per sub-partition fit.
#ifndef FKDE_EPI_NP
#define FKDE_EPI_NP 4
#endif
#ifndef FKDE_SCORE_NP
#define FKDE_SCORE_NP 3
#endif
#ifndef FKDE_CHECK_NP
#define FKDE_CHECK_NP 2
#endif
#ifndef FKDE_CTRL_REGS
#define FKDE_CTRL_REGS 56
#endif
    static constexpr int kNP = kScore ? FKDE_SCORE_NP : (kCheck ? FKDE_CHECK_NP : FKDE_EPI_NP);
    // score: warpgroup 1 (warps 4..7) = the O drain warps, one per lane quadrant
    // GEMM1 issuing warps: the check pass does little per tile, so its GEMM1 loop
    // (two barrier waits + four blocking MMA issues, ~900 cycles a tile on one
    // warp: trace_check.py) is the bottleneck; three issuers take turns by tile
    // and overlap one another's waits with the MMAs in flight
#ifndef FKDE_CHECK_ISSUERS
#define FKDE_CHECK_ISSUERS 3
#endif
    static constexpr int kIssuers = kCheck ? FKDE_CHECK_ISSUERS : 1;
    static constexpr int kCtrlEnd = kScore ? 4 : 1 + kIssuers;
    static constexpr int kEpi0 = kScore ? 8 : (kCheck ? 4 : 2);
    static_assert(kEpi0 >= kCtrlEnd, "control warps before the epilogue warps");
    static constexpr int kEpiEnd = kEpi0 + 4 * kNP;
    static constexpr int kG2Warp = kScore ? 2 : -1;
    static constexpr int kThreads = kEpiEnd * 32;
    // score register split: launch at kLaunchRegs (x kThreads <= 64K, multiple of 8),
    // control warpgroup down to kCtrlRegs, drain warpgroup up to kDrainRegs (its
    // float-float sums + one tile's O + the tile centroid), epilogue warpgroups up to
    // kEpiRegs (the pool is what the launch allocated)
    static constexpr int kLaunchRegs = kScore ? (65536 / kThreads) / 8 * 8 : 128;
    static constexpr int kCtrlRegs = FKDE_CTRL_REGS;
    static constexpr int kDrainRegs = kScore ? 112 : 0;
    static constexpr int kEpiRegs =
        kScore ? (kLaunchRegs * kThreads - 128 * kCtrlRegs - 128 * kDrainRegs) / (128 * kNP) / 8 * 8
               : 0;
    static_assert(!kScore || (kEpiRegs >= kLaunchRegs && kEpiRegs <= 256 && kDrainRegs >= kLaunchRegs),
                  "setmaxnreg split");
    // B-stage ring: 96-column tiles are 12 KiB; the check pass finishes a tile in a
    // fraction of the score pass's time, so its ring covers many tiles of L2 latency
#ifndef FKDE_SCORE_STAGES
#define FKDE_SCORE_STAGES 14
#endif
    // score stages hold the B tile and (spatial order) its centred B2 twin: 7 x 24 KiB
    static constexpr int kStages = kScore ? 7 : (kCheck ? FKDE_SCORE_STAGES : 8);
    static constexpr uint32_t kOffA = 0;
    // column tile width: score 96 points (4 S/P buffers of 96 TMEM columns fit
    // beside the two O buffers; 3 of 128 made the S ring the bottleneck), KDE 128
#ifndef FKDE_SCORE_NCOL
#define FKDE_SCORE_NCOL 96
#endif
    static constexpr int kNCol = kScoreTiling ? FKDE_SCORE_NCOL : 128;
    static constexpr uint32_t kColBytes = kNCol * kRowBytes;   // one B column tile
    static_assert(kNCol % 32 == 0 && kColBytes % 1024 == 0, "column tiles of whole SW128 atoms");
    static constexpr uint32_t kBStride = kScore ? 2 * kColBytes : kColBytes;   // B (+ B2) per stage
    static constexpr uint32_t kOffB = 2 * kTileBytes;
    static constexpr uint32_t kOffCen = kOffB + kStages * kBStride;   // score: drain centroid ring
    static constexpr uint32_t kCenBytes = kScore ? 4 * (1u << kB2GroupLog2) * kMaxDim * 4 : 0;
    static constexpr uint32_t kOffBar = kOffCen + kCenBytes;
    // S accumulators in TMEM.  Score: 4 S/P buffers of 96 columns (a tile's S is
    // overwritten by its P; the buffer is free again once GEMM2 has read P) +
    // O[2] at column 384.  KDE: 4 of 128, check: 5 of 96 (freed once S is loaded).
    static constexpr int kSBuf = kScore ? 384 / kNCol : (kCheck ? 512 / kNCol : 4);
    // unit queue: the producer fetches units (dynamic scheduling) and hands them to
    // the other warps through kQ shared slots
    static constexpr int kQ = 4;
    static constexpr int kConsumers = (kEpiEnd - 1) - (kScore ? 1 : 0);   // warps taking units
    static constexpr uint32_t kNumBars = 4 + 2 * kStages + 4 * kSBuf + 4 + 2 * kQ;
    // + tmem slot + stage column table, 1 KiB alignment slack
    static constexpr uint32_t kSmemBytes = kOffBar + kNumBars * 8 + 16 + 4 * kStages + 4 * kQ + 1024;
    static constexpr uint32_t kTmemCols = 512;
    static constexpr uint32_t kTmemO = 384;   // score: O[2] (2 x 64 cols: T_hi, S, T_lo)
    static_assert(!kScore || kSBuf * kNCol <= kTmemO, "S/P buffers overlap O");
    static_assert(kSBuf * kNCol <= kTmemCols, "S buffers fit TMEM");
    static constexpr uint32_t kN2 = 48;       // GEMM2 N
};

// score epilogue: how phi' is split into fp16 hi + lo.  0: hi = phi' with the
// low 13 mantissa bits masked (2 LOP3 per pair, ALU pipe); 1: Veltkamp split
// (t = phi' (2^13 + 1), hi = t - (t - phi'), FMA pipe only; more accurate --
// config-1 score error 1.6e-4 vs 2.2e-4 -- but 7 % slower: the epilogue is
// sensitive to every added instruction, tools/ubench_pipe.cu)
#ifndef FKDE_SPLIT
#define FKDE_SPLIT 0
#endif
// score drain: per-row sums of the O sub-units in fp64 (1: F2F + DADD per value) or
// float-float (0: 2Sum in packed f32x2)
#ifndef FKDE_DRAIN_F64
#define FKDE_DRAIN_F64 0
#endif
// GEMM2 N for the P_lo half: 32 (y_hi + the ones block; P_lo . y_lo dropped) or 48
#ifndef FKDE_G2_LO_N
#define FKDE_G2_LO_N 32
#endif

template <int MODE>
__global__ void __launch_bounds__(TcConfig<MODE>::kThreads, 1)
pairwise_tc_kernel(PairArgs args) {
    using Cfg = TcConfig<MODE>;
    constexpr bool kScore = Cfg::kScore;
    constexpr bool kCheck = Cfg::kCheck;
    constexpr int kStages = Cfg::kStages;

    extern __shared__ uint8_t smem_raw[];
    const uint32_t smem_s = ptx::smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((smem_s + 1023u) & ~1023u) - smem_s);
    uint8_t* smA = smem + Cfg::kOffA;
    uint8_t* smB = smem + Cfg::kOffB;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::kOffBar);
    uint64_t* a_full = bars;              // [2]
    uint64_t* a_empty = bars + 2;         // [2]
    uint64_t* b_full = bars + 4;          // [kStages]
    uint64_t* b_empty = b_full + kStages; // [kStages]
    constexpr int kSB = Cfg::kSBuf;
    uint64_t* s_full = b_empty + kStages; // [kSB]
    uint64_t* s_empty = s_full + kSB;     // [kSB]
    uint64_t* p_full = s_empty + kSB;     // [kSB]
    uint64_t* s_free = p_full + kSB;      // [kSB] score: GEMM2 done reading P (S buffer reusable)
    uint64_t* o_full = s_free + kSB;      // [2]
    uint64_t* o_empty = o_full + 2;       // [2]
    uint64_t* uq_full = o_empty + 2;      // [kQ] unit queue
    uint64_t* uq_empty = uq_full + Cfg::kQ;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(uq_empty + Cfg::kQ);
    // the column tile each B stage holds (written by the producer before the stage's
    // b_full arrive): the other warps look it up instead of walking the tile mask
    int* stage_ct = reinterpret_cast<int*>(tmem_slot + 1);   // [kStages]
    int* uq_slot = stage_ct + kStages;                        // [kQ]

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&a_full[i], 1);
            ptx::mbar_init(&a_empty[i], Cfg::kIssuers);   // one commit per GEMM1 issuer
        }
        for (int i = 0; i < kSB; ++i) {
            ptx::mbar_init(&s_full[i], 1);
            ptx::mbar_init(&s_empty[i], 4);
            ptx::mbar_init(&p_full[i], 4);
            ptx::mbar_init(&s_free[i], 1);
        }
        for (int i = 0; i < kStages; ++i) {
            ptx::mbar_init(&b_full[i], 1);
            // check pass: the four quadrant warps release a stage once they have read
            // its column index (stage_ct) and the tile's S; elsewhere an MMA commit
            ptx::mbar_init(&b_empty[i], kCheck ? 4 : 1);
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&o_full[i], 1);
            ptx::mbar_init(&o_empty[i], 4);
        }
        for (int i = 0; i < Cfg::kQ; ++i) {
            ptx::mbar_init(&uq_full[i], 1);
            ptx::mbar_init(&uq_empty[i], Cfg::kConsumers);
        }
        ptx::fence_barrier_init();
    }
    pdl_launch_dependents();
    if (warp == 1) ptx::tmem_alloc<Cfg::kTmemCols>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // (barriers and TMEM are set up while the previous kernel of the chain drains)
    pdl_wait();
#ifdef FKDE_CTA_TIMES
    // debug build (tools/cta_balance.py): per-CTA start / end globaltimer and the
    // number of tiles the CTA visited, region MODE * 4096 of args.trace
    if (args.trace && threadIdx.x == 0) args.trace[MODE * 4096 + 2 * blockIdx.x] = ptx::globaltimer();
#endif

    const int n_units = args.n_row_tiles * args.splits;
    // Dynamic scheduling: the producer warp fetches the next unit from a global
    // counter when it is ready to stream it (units stay in chunk-major order, so the
    // CTAs running at any time still share one column chunk in L2) and publishes it
    // in the unit queue; every other role takes the units from the queue in the
    // same order (-1 ends the kernel).  A CTA that drew short units simply draws
    // more: the per-CTA work no longer depends on which rows sit where.
    auto publish_unit = [&](uint32_t qi) -> int {
        const uint32_t sl = qi % Cfg::kQ;
        int u = 0;
        if (lane == 0) u = static_cast<int>(atomicAdd(args.sched, 1u));
        u = __shfl_sync(0xffffffffu, u, 0);
        if (u >= n_units) u = -1;
        ptx::mbar_wait(&uq_empty[sl], ((qi / Cfg::kQ) & 1) ^ 1);
        if (lane == 0) {
            uq_slot[sl] = u;
            ptx::mbar_arrive(&uq_full[sl]);   // (release: the slot write)
        }
        __syncwarp();
        return u;
    };
    auto take_unit = [&](uint32_t qi) -> int {
        const uint32_t sl = qi % Cfg::kQ;
        ptx::mbar_wait(&uq_full[sl], (qi / Cfg::kQ) & 1);
        const int u = *reinterpret_cast<volatile int*>(&uq_slot[sl]);
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&uq_empty[sl]);
        return u;
    };
    // the column tiles a unit visits (score: clear skip bits; check: set pred bits)
    auto walk_of = [&](int rt, int ct1) {
        TileWalkT<kCheck> w;
        const uint32_t* m = kCheck ? args.pred_mask : args.skip_mask;
        w.row = m ? m + (size_t)rt * args.mask_words : nullptr;
        w.end = ct1;
        w.want = kCheck ? ~0u : 0u;
        return w;
    };

    // Control warps (producer, MMA issuers) and epilogue warps live in separate
    // warpgroups in the score pass; each side resizes its register file at the
    // top of its own branch so that ptxas can allocate the epilogue's code for
    // kEpiRegs registers (the resize dominates every epilogue instruction).
    if (warp < Cfg::kCtrlEnd) {
    if constexpr (kScore) ptx::setmaxnreg_dec<Cfg::kCtrlRegs>();
    if (warp == 0) {
        // ===================== producer: bulk async copies =====================
        // The whole warp runs the loop (all values warp-uniform, no waterfall
        // loops around the uniform-register operands); one elected lane issues.
        const uint64_t pol_b = ptx::policy_evict_last();
        uint32_t it_a = 0, it_b = 0;
        for (uint32_t qi = 0;; ++qi) {
            const int u = publish_unit(qi);
            if (u < 0) break;
            // chunk-major unit order: CTAs running concurrently share one column
            // chunk, which therefore stays L2-resident while they stream it
            const int sp = u / args.n_row_tiles, rt = u % args.n_row_tiles;
            const int ct0 = static_cast<int>((long long)sp * args.n_col_tiles / args.splits);
            const int ct1 = static_cast<int>((long long)(sp + 1) * args.n_col_tiles / args.splits);
            auto wk = walk_of(rt, ct1);
            int ct = wk.first(ct0);
            if (ct >= ct1) continue;   // nothing to visit: no A tile either
            const int ab = it_a & 1;
            ptx::mbar_wait(&a_empty[ab], ((it_a >> 1) & 1) ^ 1);
            if (ptx::elect_one()) {
                ptx::mbar_arrive_expect_tx(&a_full[ab], kTileBytes);
                ptx::bulk_g2s(smA + ab * kTileBytes, args.opA + (size_t)rt * kTileBytes,
                              kTileBytes, &a_full[ab]);
            }
            __syncwarp();
            ++it_a;
            for (; ct < ct1; ct = wk.next()) {
                const int st = it_b % kStages;
                ptx::mbar_wait(&b_empty[st], ((it_b / kStages) & 1) ^ 1);
                if (ptx::elect_one()) {
                    stage_ct[st] = ct;   // (ordered before the arrive below: release)
                    const bool b2 = kScore && args.opB2;
                    ptx::mbar_arrive_expect_tx(&b_full[st], Cfg::kColBytes * (b2 ? 2u : 1u));
                    ptx::bulk_g2s_hint(smB + st * Cfg::kBStride, args.opB + (size_t)ct * Cfg::kColBytes,
                                       Cfg::kColBytes, &b_full[st], pol_b);
                    if (b2)
                        ptx::bulk_g2s_hint(smB + st * Cfg::kBStride + Cfg::kColBytes,
                                           args.opB2 + (size_t)ct * Cfg::kColBytes, Cfg::kColBytes,
                                           &b_full[st], pol_b);
                }
                __syncwarp();
                ++it_b;
            }
        }
    } else if ((warp >= 1 && warp <= Cfg::kIssuers) || (kScore && warp == Cfg::kG2Warp)) {
        static_assert(Cfg::kNP <= Cfg::kSBuf, "each epilogue warp holds one S buffer");
        // ===================== MMA issuers =====================
        // Whole warp in the loop, one elected lane issues every tcgen05 op
        // (commits must come from the issuing thread; elect.sync on a
        // converged warp always picks the same lane).  Descriptors are built
        // once and advanced by adding (byte offset >> 4) to the start-address
        // field, so each MMA costs a uniform add + the instruction.
        constexpr uint32_t idesc1 = ptx::idesc_f16_f32(128, Cfg::kNCol, false, false);
        constexpr uint32_t idesc2 = ptx::idesc_f16_f32(128, Cfg::kN2, false, true);
        // P_lo rows only need the y_hi and ones columns: P_lo . y_lo is 2^-22 of the
        // sum and is dropped, which takes 1/6 of GEMM2's MACs (and power) away
        constexpr uint32_t idesc2_lo = ptx::idesc_f16_f32(128, FKDE_G2_LO_N, false, true);
        const uint64_t descA = ptx::smem_desc_sw128(ptx::smem_u32(smA), 16, 1024);
        const uint64_t descB = ptx::smem_desc_sw128(ptx::smem_u32(smB), 16, 1024);
        // GEMM2's operand: the stage's B tile, or its centred B2 twin (spatial order)
        const uint64_t descBmn = ptx::smem_desc_sw128(
            ptx::smem_u32(smB) + ((kScore && args.opB2) ? Cfg::kColBytes : 0u), kTileBytes, 1024);
        uint32_t it_a = 0, it_b = 0, it_s = 0, it_u = 0;
        const bool g1 = warp >= 1 && warp <= Cfg::kIssuers;
        const uint32_t my_turn = static_cast<uint32_t>(warp - 1);   // GEMM1: tiles it_s % kIssuers
        // GEMM2 (warp 2): O += P_hi.B + P_lo.B, P read from TMEM.  The
        // epilogue stored, for each 32-column chunk c of S buffer sb, P_hi
        // (packed fp16 pairs) for K = 32c..32c+31 in the chunk's first 16
        // columns and P_lo in the next 16.  O is accumulated in TMEM over
        // 2^flush_log2 visited column tiles (a "sub-unit"), then drained by the
        // drain warps; two O buffers alternate so the drain overlaps the next
        // sub-unit.  This bounds the tensor core's fp32 accumulation length (its
        // truncation error grows with the accumulator magnitude x the number of steps).
        // sub-unit boundaries (identical in the drain warps): a new sub-unit starts at
        // the unit's first visited tile, when the column-tile group changes (centred
        // B2) and after 2^flush_log2 tiles.  The GEMM2 warp walks the tile mask itself
        // (it knows the next tile's group without waiting for its stage), so the
        // sub-unit's o_full commit follows its last MMAs at once: the drain, and
        // with it the O buffer's release, is not held back by the next tile's p_full.
        const int fcap = 1 << args.flush_log2;
        const bool grouped = kScore && args.opB2 != nullptr;
        constexpr int glog = kB2GroupLog2;
        for (uint32_t qi = 0;; ++qi) {
            const int u = take_unit(qi);
            if (u < 0) break;
            const int sp = u / args.n_row_tiles, rt = u % args.n_row_tiles;
            const int ct0 = static_cast<int>((long long)sp * args.n_col_tiles / args.splits);
            const int ct1 = static_cast<int>((long long)(sp + 1) * args.n_col_tiles / args.splits);
            // (GEMM1 only needs how many tiles the unit visits, not which)
            auto wk2 = walk_of(rt, ct1);
            const int len = wk2.count(ct0);
            if (len == 0) continue;
            int sub_cnt = 0;
            int cur_ct = (kScore && !g1) ? wk2.first(ct0) : 0;
            const int ab = it_a & 1;
            if (g1) {
                ptx::mbar_wait(&a_full[ab], (it_a >> 1) & 1);
                ptx::tc_fence_after();
            }
            for (int rel = 0; rel < len; ++rel) {
                const uint32_t st = it_b % kStages;
                const uint32_t sb = it_s % Cfg::kSBuf;
                const uint32_t ph = (it_s / Cfg::kSBuf) & 1;
                if (g1) {
                    if (Cfg::kIssuers > 1 && it_s % Cfg::kIssuers != my_turn) {   // another issuer's tile
                        ++it_b;
                        ++it_s;
                        continue;
                    }
                    FKDE_TRACE(0, it_s);
                    ptx::mbar_wait(&b_full[st], (it_b / kStages) & 1);
                    FKDE_TRACE(1, it_s);
                    // KDE / check: the epilogue frees S after loading it.  SCORE: GEMM2
                    // of the tile that last used this buffer has finished reading P.
                    if constexpr (!kScore) ptx::mbar_wait(&s_empty[sb], ph ^ 1);
                    else ptx::mbar_wait(&s_free[sb], ph ^ 1);
                    FKDE_TRACE(5, it_s);
                    ptx::tc_fence_after();
                    if (ptx::elect_one()) {
                        const uint64_t da0 = descA + ((ab * kTileBytes) >> 4);
                        const uint64_t db0 = descB + ((st * Cfg::kBStride) >> 4);
                        // K-step order: the half-norm chunk first, then y_hi.y_hi, so the
                        // large terms cancel inside one fused MMA step before the small
                        // hi/lo cross terms are added.
                        // (the check pass needs only the norms and y_hi . y_hi: the hi/lo
                        // cross terms are bounded by 2^-9 max|y|^2/2 and covered by the
                        // margin of its threshold -- half the MMAs)
#pragma unroll
                        for (int kk = 0; kk < (kCheck ? 2 : 4); ++kk) {
                            const int k = kk == 0 ? 1 : (kk == 1 ? 0 : kk);  // 1 (norms), 0, 2, 3
                            ptx::umma_f16(tmem_base + sb * Cfg::kNCol, da0 + ((k * 32) >> 4),
                                          db0 + ((k * 32) >> 4), idesc1, kk > 0 ? 1u : 0u);
                        }
                        ptx::umma_commit(&s_full[sb]);
                        if constexpr (!kScore && !kCheck) ptx::umma_commit(&b_empty[st]);
                    }
                    __syncwarp();
                    FKDE_TRACE(4, it_s);
                } else if constexpr (kScore) {
                    const int next_ct = wk2.next();
                    const bool first = sub_cnt == 0;
                    ++sub_cnt;
                    const bool last = rel == len - 1 || sub_cnt == fcap ||
                                      (grouped && (next_ct >> glog) != (cur_ct >> glog));
                    cur_ct = next_ct;
                    FKDE_TRACE(2, it_s);
                    ptx::mbar_wait(&p_full[sb], ph);
                    FKDE_TRACE(3, it_s);
                    const uint32_t ob = it_u & 1;
                    if (first) ptx::mbar_wait(&o_empty[ob], ((it_u >> 1) & 1) ^ 1);
                    ptx::tc_fence_after();
                    if (ptx::elect_one()) {
                        const uint64_t db0 = descBmn + ((st * Cfg::kBStride) >> 4);
                        const uint32_t ta0 = tmem_base + sb * Cfg::kNCol;
                        const uint32_t to = tmem_base + Cfg::kTmemO + ob * 64;
#ifndef FKDE_DBG_NO_G2MMA
#pragma unroll
                        for (int k = 0; k < Cfg::kNCol / 16; ++k) {
#pragma unroll
                            for (int part = 0; part < 2; ++part) {
                                // one N=48 MMA per K step: columns 0-15 T_hi, 16 S, 32-47 T_lo
                                ptx::umma_f16_ts(to, ta0 + (k >> 1) * 32 + part * 16 + (k & 1) * 8,
                                                 db0 + ((k * 2048) >> 4), part ? idesc2_lo : idesc2,
                                                 (first && part == 0 && k == 0) ? 0u : 1u);
                            }
                        }
#endif
                        ptx::umma_commit(&b_empty[st]);
                        ptx::umma_commit(&s_free[sb]);
                        if (last) ptx::umma_commit(&o_full[ob]);
                    }
                    __syncwarp();
                    FKDE_TRACE(5, it_s);
                    if (last) {
                        ++it_u;
                        sub_cnt = 0;
                    }
                }
                ++it_b;
                ++it_s;
            }
            if (g1) {
                if (ptx::elect_one()) ptx::umma_commit(&a_empty[ab]);
                __syncwarp();
            }

            ++it_a;
        }
    }
    } else if (warp < Cfg::kEpi0) {
        if constexpr (kScore) {
            ptx::setmaxnreg_inc<Cfg::kDrainRegs>();
            // ===================== O drain warps (score) =====================
            // Warp 4+q drains lane quadrant q of every O sub-unit (2^flush_log2
            // visited column tiles) in order: wait for GEMM2's commit, read T_hi,
            // S, T_lo, release the buffer, fold into float-float sums (2Sum,
            // ~48-bit significand) and write one fp64 partial per (split, row) at
            // the unit's end (zero for a unit that visits no tile).  Keeping this
            // off the epilogue warps leaves them a uniform ld -> ex2 -> st stream.
            const int q = warp & 3;
            const int r = q * 32 + lane;
            const uint32_t lane_addr = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
            const int fcap = 1 << args.flush_log2;
            constexpr int glog = kB2GroupLog2;
            constexpr int gmask = (1 << glog) - 1;
            const float escale = exp2f(static_cast<float>(-args.sc->e));   // 2^-e (exact)
            // centred GEMM2 (B2): each tile J of a sub-unit adds c_J S_J (c_J scaled
            // like the operands, 2^-e, exact; S_J from J's own ones column).  The
            // centroids are copied into this warp's shared-memory ring (cp.async,
            // slot J mod 2^glog) when the tile joins the sub-unit, a tile or more
            // before the drain reads them (broadcast) -- no L2 round trip on the path
            // that releases O to GEMM2, and no registers held for them.
            const bool centred = args.opB2 != nullptr;
            const uint32_t cring = ptx::smem_u32(smem + Cfg::kOffCen) + q * ((1u << glog) * kMaxDim * 4);
            const float* cring_p = reinterpret_cast<const float*>(smem + Cfg::kOffCen) + q * (1 << glog) * kMaxDim;
            uint32_t it_u = 0;
            for (uint32_t qi = 0;; ++qi) {
            const int u = take_unit(qi);
            if (u < 0) break;
                const int sp = u / args.n_row_tiles, rt = u % args.n_row_tiles;
                const int ct0 = static_cast<int>((long long)sp * args.n_col_tiles / args.splits);
                const int ct1 = static_cast<int>((long long)(sp + 1) * args.n_col_tiles / args.splits);
                auto wk = walk_of(rt, ct1);
                const int len = wk.count(ct0);
#if FKDE_DRAIN_F64
                double acc[kMaxDim + 1];
#pragma unroll
                for (int c = 0; c <= kMaxDim; ++c) acc[c] = 0.0;
#else
                float ahi[kMaxDim + 1], alo[kMaxDim + 1];
#pragma unroll
                for (int c = 0; c <= kMaxDim; ++c) ahi[c] = alo[c] = 0.f;
#endif
                int pend = 0, cur_grp = -1;
                uint32_t pmask = 0;   // ring slots (tiles) of the pending sub-unit
                int ct = len > 0 ? wk.first(ct0) : ct1;
                // the sub-unit schedule of the GEMM2 issuer, replayed from the tile walk;
                // k == len drains the last sub-unit
#pragma unroll 1
                for (int k = 0; k <= len; ++k) {
                    const int grp = (k < len && centred) ? (ct >> glog) : 0;
                    if (pend > 0 && (k == len || grp != cur_grp || pend == fcap)) {
                    const uint32_t g = it_u++;
                    pend = 0;
                    const uint32_t to = lane_addr + Cfg::kTmemO + (g & 1) * 64;
                    constexpr int kSlots = 1 << kB2GroupLog2;
                    uint32_t od[16], ol[16], os4[kSlots];
                    FKDE_TRACE(4, g);
                    ptx::mbar_wait(&o_full[g & 1], (g >> 1) & 1);
                    FKDE_TRACE(5, g);
                    ptx::tc_fence_after();
                    ptx::tmem_ld16(to, od);
                    ptx::tmem_ldn(to + 16, os4);   // S_J per ring slot (non-centred: 16 = S)
                    ptx::tmem_ld16(to + 32, ol);
                    ptx::tmem_ld_wait();
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(&o_empty[g & 1]);
                    // x = T_hi + T_lo (+ sum_J c_J S_J when centred), then 2Sum into the
                    // float-float sums -- all in packed f32x2 pairs
                    float sv = __uint_as_float(os4[0]);
                    float2 xs[kMaxDim / 2];
#pragma unroll
                    for (int c = 0; c < kMaxDim; c += 2)
                        xs[c >> 1] = ptx::fadd2(make_float2(__uint_as_float(od[c]), __uint_as_float(od[c + 1])),
                                                make_float2(__uint_as_float(ol[c]), __uint_as_float(ol[c + 1])));
                    if (centred) {
                        ptx::cp_async_wait_all();
                        __syncwarp();
                        sv = 0.f;
#pragma unroll
                        for (int sl = 0; sl <= gmask; ++sl) {
                            if (!(pmask & (1u << sl))) continue;   // (warp-uniform)
                            const float sj = __uint_as_float(os4[sl]);
                            sv += sj;
                            const float sjs = sj * escale;   // S_J 2^-e: c_J (log2 units) -> operand scale
                            const float4* cp = reinterpret_cast<const float4*>(cring_p + sl * kMaxDim);
#pragma unroll
                            for (int w = 0; w < 4; ++w) {
                                const float4 cq = cp[w];
                                xs[2 * w] = ptx::ffma2(make_float2(cq.x, cq.y), make_float2(sjs, sjs), xs[2 * w]);
                                xs[2 * w + 1] = ptx::ffma2(make_float2(cq.z, cq.w), make_float2(sjs, sjs), xs[2 * w + 1]);
                            }
                        }
                    }
                    pmask = 0;
#ifdef FKDE_DBG_NO_DRAIN_MATH
                    if (xs[0].x == 12345.f) ahi[0] += sv;   // (keeps the loads alive)
#elif FKDE_DRAIN_F64
#pragma unroll
                    for (int c = 0; c < kMaxDim; c += 2) {
                        acc[c] += static_cast<double>(xs[c >> 1].x);
                        acc[c + 1] += static_cast<double>(xs[c >> 1].y);
                    }
                    acc[kMaxDim] += static_cast<double>(sv);
#else
#pragma unroll
                    for (int c = 0; c < kMaxDim; c += 2) {
                        const float2 x = xs[c >> 1];
                        // 2Sum(ahi, x); a - b as fma(b, -1, a) (exact negation, one rounding)
                        const float2 m1 = make_float2(-1.f, -1.f);
                        const float2 a2 = make_float2(ahi[c], ahi[c + 1]);
                        const float2 s2 = ptx::fadd2(a2, x);
                        const float2 bb = ptx::ffma2(a2, m1, s2);                 // s - a
                        const float2 e = ptx::fadd2(ptx::ffma2(ptx::ffma2(bb, m1, s2), m1, a2),   // a - (s - bb)
                                                    ptx::ffma2(bb, m1, x));                        // + (x - bb)
                        ahi[c] = s2.x;
                        ahi[c + 1] = s2.y;
                        const float2 l2 = ptx::fadd2(make_float2(alo[c], alo[c + 1]), e);
                        alo[c] = l2.x;
                        alo[c + 1] = l2.y;
                    }
                    {   // S
                        const float s2 = ahi[kMaxDim] + sv;
                        const float bb = s2 - ahi[kMaxDim];
                        alo[kMaxDim] += (ahi[kMaxDim] - (s2 - bb)) + (sv - bb);
                        ahi[kMaxDim] = s2;
                    }
#endif
                    }
                    if (k == len) break;
                    if (pend == 0) cur_grp = grp;   // a new sub-unit
                    if (centred) {   // tile ct joins it: its centroid into ring slot ct mod 2^glog
                        const int sl = ct & gmask;
                        if (lane < 4)
                            ptx::cp_async16(cring + (sl * kMaxDim + lane * 4) * 4,
                                            args.cenB + (size_t)ct * kMaxDim + lane * 4);
                        ptx::cp_async_commit();
                        pmask |= 1u << sl;
                    }
                    ++pend;
                    ct = wk.next();
                }
                const size_t idx = static_cast<size_t>(sp) * args.rows_pad + static_cast<size_t>(rt) * kTileRows + r;
                double2* t = reinterpret_cast<double2*>(args.dpart1 + idx * kMaxDim);
#if FKDE_DRAIN_F64
                args.dpart0[idx] = acc[kMaxDim];
#pragma unroll
                for (int w = 0; w < kMaxDim / 2; ++w) t[w] = make_double2(acc[2 * w], acc[2 * w + 1]);
#else
                args.dpart0[idx] = static_cast<double>(ahi[kMaxDim]) + static_cast<double>(alo[kMaxDim]);
#pragma unroll
                for (int w = 0; w < kMaxDim / 2; ++w)
                    t[w] = make_double2(static_cast<double>(ahi[2 * w]) + static_cast<double>(alo[2 * w]),
                                        static_cast<double>(ahi[2 * w + 1]) + static_cast<double>(alo[2 * w + 1]));
#endif
            }
        }
    } else if (warp < Cfg::kEpiEnd) {
        if constexpr (kScore) ptx::setmaxnreg_inc<Cfg::kEpiRegs>();
        // ===================== epilogue warps =====================
        // Warp w reads TMEM lane quadrant w%4 and handles every kNP-th visited
        // column tile (phase par = (w-kEpi0)/4), all its columns, in 32-column
        // chunks.  The kNP warps sharing an SM sub-partition (and a lane
        // quadrant) therefore work on different tiles, out of phase: while one
        // waits for its next S tile (GEMM1 of tile t + kNP can only start once
        // GEMM2 of tile t has released the buffer) the others keep the MUFU pipe
        // busy.  The own-tile loop carries only a few integer ops of bookkeeping.
        constexpr int NP = Cfg::kNP;
        const int q = warp & 3;                      // TMEM lane quadrant
        const int par = (warp - Cfg::kEpi0) >> 2;    // tile phase handled by this warp
        const int r = q * 32 + lane;                 // row within the 128-row tile
        const float dsc = args.sc->dscale;
        // check pass: S lacks the hi/lo cross terms y_hi.y_lo + y_lo.y_hi, each bounded
        // by 2^-11 |y_i| |y_j| <= 2^-11 max|y|^2, so their sum by 2^-9 max|y|^2/2 (the
        // bound prep_stats stored, log2 units): a tile is skippable when even the
        // bound-raised maximum is below kSkipLog2
        const float skip_below =
            kSkipLog2 - (ldexpf(__uint_as_float(args.sc->max_half_norm_bits), -9) + 0.0625f);
        const uint32_t lane_addr = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
        uint32_t it_s = 0;                           // global visited-tile counter (all phases)
        unsigned long long n_checked = 0;            // check statistics (quadrant 0 counts)
        for (uint32_t qi = 0;; ++qi) {
            const int u = take_unit(qi);
            if (u < 0) break;
            const int sp = u / args.n_row_tiles, rt = u % args.n_row_tiles;
            const int ct0 = static_cast<int>((long long)sp * args.n_col_tiles / args.splits);
            const int ct1 = static_cast<int>((long long)(sp + 1) * args.n_col_tiles / args.splits);
            auto wk = walk_of(rt, ct1);
            float2 acc2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
            float2 accl2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
            // score: global index of this lane's row minus the unit's first
            // column; the row's self pair sits at column jd0 - (ct - ct0) * kNCol
            // of column tile ct (masked where that lies in [0, kNCol))
            const long long jd0 = args.diag_row0 >= 0
                                      ? args.diag_row0 + (long long)rt * kTileRows + r - (long long)ct0 * Cfg::kNCol
                                      : -(1ll << 40);
            // column tiles (relative to ct0) the row tile's diagonal crosses:
            // [drel_lo, drel_hi] (floor division; empty when the pass has no diagonal)
            const long long drow0 = jd0 - r;
            auto fdiv = [](long long a) {
                return a >= 0 ? a / Cfg::kNCol : -((-a + Cfg::kNCol - 1) / Cfg::kNCol);
            };
            const bool has_diag = args.diag_row0 >= 0;
            const int drel_lo = has_diag ? static_cast<int>(fdiv(drow0)) : INT_MAX;
            const int drel_hi = has_diag ? static_cast<int>(fdiv(drow0 + kTileRows - 1)) : -1;
            // visited tiles of this unit so far (k) and the current one (ct).  Without
            // a mask every tile is visited and the walk jumps straight from one own
            // tile to the next (the KDE pass keeps its original bookkeeping cost);
            // with a mask it steps through the visited tiles, skipping other phases'.
            const bool dense = wk.row == nullptr;
            const int len = wk.count(ct0);
            // score with a mask: the visited-tile indices (within the unit) of the
            // column tiles the diagonal crosses, so that a tile's column index is never
            // needed (no b_full wait / stage_ct load per tile on the epilogue's path)
            int kd_lo = -1, kd_hi = -1;
            if (kScore && !dense && has_diag) {
                auto vidx = [&](int rel) {
                    const int c = ct0 + rel;
                    if (rel < 0 || c >= ct1 || !((wk.word(c >> 5) >> (c & 31)) & 1u)) return -1;
                    auto w2 = wk;
                    w2.end = c;
                    return w2.count(ct0);
                };
                kd_lo = vidx(drel_lo);
                kd_hi = drel_hi != drel_lo ? vidx(drel_hi) : -1;
            }
            int first_own = par - static_cast<int>(it_s % NP);
            if (first_own < 0) first_own += NP;
            for (int k = first_own; k < len; k += NP) {
                const uint32_t sidx = it_s + k;
                const uint32_t sb = sidx % Cfg::kSBuf, ph = (sidx / Cfg::kSBuf) & 1;
                int ct = ct0 + k;
                if (kCheck && !dense) {   // the visited tile's column index, from its B stage
                    const uint32_t st = sidx % kStages;
                    ptx::mbar_wait(&b_full[st], (sidx / kStages) & 1);   // (complete: GEMM1 used it)
                    ct = *reinterpret_cast<volatile int*>(&stage_ct[st]);
                }
                if (kScore && !dense)   // only the diagonal's tiles need their column index
                    ct = k == kd_lo ? ct0 + drel_lo : (k == kd_hi ? ct0 + drel_hi : INT_MIN / 2);
                const int rel = ct - ct0;
                FKDE_TRACE(0, sidx);
                ptx::mbar_wait(&s_full[sb], ph);
                FKDE_TRACE(1, sidx);
                ptx::tc_fence_after();
                const uint32_t ts = lane_addr + sb * Cfg::kNCol;
                const float2 dsc2 = make_float2(dsc, dsc);
                if constexpr (kScore) {
                    // the row tile's diagonal crosses this column tile (warp-uniform: a
                    // plain branch per chunk, no vote); jdiag = this row's diagonal
                    // column, masked below where it lies in the chunk
                    const bool diag_tile = rel >= drel_lo && rel <= drel_hi;
                    const int jdiag = diag_tile ? static_cast<int>(jd0 - (long long)rel * Cfg::kNCol) : -1;
                    const float2 neg1 = make_float2(-1.f, -1.f);
                    const float2 vk2 = make_float2(8193.f, 8193.f);   // 2^13 + 1
                    (void)vk2;
#pragma unroll kScoreChUnroll
                    for (int ch = 0; ch < Cfg::kNCol / 32; ++ch) {
                        uint32_t v[32];
                        ptx::tmem_ld32(ts + ch * 32, v);
                        ptx::tmem_ld_wait();
                        if (ch == 0) FKDE_TRACE(6, sidx);
                        if (diag_tile) {
#pragma unroll
                            for (int c = 0; c < 32; ++c)    // -inf -> phi = 0
                                v[c] = ptx::sel_eq(v[c], c + ch * 32, jdiag, 0xFF800000u);
                        }
                        // phi' = phi * 2^15 split exactly into fp16 hi + lo: hi keeps
                        // the top 11 significant bits (mask), lo = phi' - hi (exact),
                        // both convert to fp16 exactly / to nearest.  (S may exceed 0
                        // by rounding for coincident points: phi' <= 2^15 (1 + 1e-5),
                        // well inside fp16, so no clamp.)  The chunk's 32 S columns
                        // are overwritten by its own P: hi words in the first 16
                        // columns, lo words in the next 16.
                        uint32_t hi_w[16], lo_w[16];
#pragma unroll
                        for (int w = 0; w < 16; ++w) {
                            // S already includes the 2^15 offset (A rows' column c)
                            const float2 s2 =
                                make_float2(__uint_as_float(v[2 * w]), __uint_as_float(v[2 * w + 1]));
                            // (an FMUL2 even when dscale == 1: measured faster than feeding S to ex2
                            // directly, the schedule spaces the MUFU issues better)
                            const float2 t = ptx::fmul2(s2, dsc2);
                            const float2 p = make_float2(ptx::ex2(t.x), ptx::ex2(t.y));
#if FKDE_SPLIT == 1
                            const float2 vt = ptx::fmul2(p, vk2);
                            const float2 h = ptx::fadd2(vt, ptx::ffma2(vt, neg1, p));   // t + (p - t)
#else
                            const float2 h = make_float2(
                                __uint_as_float(__float_as_uint(p.x) & 0xFFFFE000u),
                                __uint_as_float(__float_as_uint(p.y) & 0xFFFFE000u));
#endif
                            const float2 l = ptx::ffma2(h, neg1, p);
                            hi_w[w] = ptx::cvt_f16x2(h.x, h.y);
                            lo_w[w] = ptx::cvt_f16x2(l.x, l.y);
                        }
                        ptx::tmem_st16(ts + ch * 32, hi_w);
                        ptx::tmem_st16(ts + ch * 32 + 16, lo_w);
                    }
                    FKDE_TRACE(7, sidx);
                    ptx::tmem_st_wait();
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(&p_full[sb]);
                    FKDE_TRACE(2, sidx);
                } else if constexpr (kCheck) {
                    // exact max of log2 phi' over this quadrant's 32 rows x 96 columns:
                    // the three loads are in flight together, the buffer is released
                    // as soon as they have landed
                    uint32_t v0[32], v1[32], v2[32];
                    ptx::tmem_ld32(ts, v0);
                    ptx::tmem_ld32(ts + 32, v1);
                    ptx::tmem_ld32(ts + 64, v2);
                    ptx::tmem_ld_wait();
                    FKDE_TRACE(6, sidx);
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) {
                        ptx::mbar_arrive(&s_empty[sb]);
                        ptx::mbar_arrive(&b_empty[sidx % kStages]);   // (stage_ct read above)
                    }
                    float m0 = -INFINITY, m1 = -INFINITY, m2 = -INFINITY, m3 = -INFINITY;
#pragma unroll
                    for (int c = 0; c < 32; c += 2) {
                        m0 = fmaxf(m0, __uint_as_float(v0[c]));
                        m1 = fmaxf(m1, __uint_as_float(v0[c + 1]));
                        m2 = fmaxf(m2, __uint_as_float(v1[c]));
                        m3 = fmaxf(m3, __uint_as_float(v1[c + 1]));
                        m0 = fmaxf(m0, __uint_as_float(v2[c]));
                        m1 = fmaxf(m1, __uint_as_float(v2[c + 1]));
                    }
                    const float mx = fmaxf(fmaxf(m0, m1), fmaxf(m2, m3));
                    const bool keep = __any_sync(0xffffffffu, !(mx * dsc < skip_below));
                    if (lane == 0) {
                        if (keep)   // some pair of this quadrant contributes: not skippable
                            atomicAnd(args.skip_mask + (size_t)rt * args.mask_words + (ct >> 5),
                                      ~(1u << (ct & 31)));
                        if (q == 0) ++n_checked;
                    }
                    FKDE_TRACE(7, sidx);
                } else {
                    // (phi <= 1 up to the expansion's rounding: no clamp needed)
#pragma unroll 1
                    for (int ch = 0; ch < 4; ++ch) {
                        uint32_t v[32];
                        ptx::tmem_ld32(ts + ch * 32, v);
                        ptx::tmem_ld_wait();
                        if (ch == 3) {
                            ptx::tc_fence_before();
                            __syncwarp();
                            if (lane == 0) ptx::mbar_arrive(&s_empty[sb]);
                        }
#pragma unroll
                        for (int c = 0; c < 32; c += 2) {
                            const float2 s2 = make_float2(__uint_as_float(v[c]), __uint_as_float(v[c + 1]));
                            const float2 dd = ptx::fmul2(s2, dsc2);
                            const float2 p = make_float2(ptx::ex2(dd.x), ptx::ex2(dd.y));
                            const int a = (c >> 1) & 1;
                            acc2[a] = ptx::fadd2(acc2[a], p);
                            if constexpr (MODE == kModeLaplace) accl2[a] = ptx::ffma2(p, dd, accl2[a]);
                        }
                    }
                }
            }
            if constexpr (!kScore && !kCheck) {
                // the kNP phases hold disjoint column subsets of this unit.  The slot
                // is the phase RELATIVE to the unit (visited tiles k = first_own mod
                // NP), not the warp's phase: which warp takes a unit's first tile
                // depends on the tiles the CTA visited before it, i.e. on the dynamic
                // schedule, and the fixed-order fp64 sum over slots in reduce_density
                // is then bitwise reproducible from run to run
                const size_t row = static_cast<size_t>(rt) * kTileRows + r;
                const size_t idx = static_cast<size_t>(sp * NP + first_own) * args.rows_pad + row;
                args.part0[idx] = (acc2[0].x + acc2[0].y) + (acc2[1].x + acc2[1].y);
                if constexpr (MODE == kModeLaplace)
                    args.part1[idx] = (accl2[0].x + accl2[0].y) + (accl2[1].x + accl2[1].y);
            }
            it_s += static_cast<uint32_t>(len);
        }
#ifdef FKDE_CTA_TIMES
        if (args.trace && warp == Cfg::kEpi0 && lane == 0) args.trace[MODE * 4096 + 2048 + blockIdx.x] = it_s;
#endif
        if (kCheck && args.stats && lane == 0 && q == 0 && n_checked)
            atomicAdd(&args.stats[0], n_checked);
    }

    ptx::tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) {   // the last CTA to finish resets the scheduler for the next launch
        __threadfence();
        if (atomicAdd(args.sched + 1, 1u) == gridDim.x - 1) {
            args.sched[0] = 0;
            args.sched[1] = 0;
            __threadfence();
        }
    }
#ifdef FKDE_CTA_TIMES
    if (args.trace && threadIdx.x == 0) args.trace[MODE * 4096 + 2 * blockIdx.x + 1] = ptx::globaltimer();
#endif
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<Cfg::kTmemCols>(tmem_base);
    }
}

}  // namespace fkde_b200
