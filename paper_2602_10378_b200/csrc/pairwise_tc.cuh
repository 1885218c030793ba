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
// Here one work unit = (128-row tile, contiguous range of 128-column tiles).
// Per column tile:
//   GEMM1  S[128x128] = A_rows(128x64 fp16) . B_cols(128x64 fp16)^T  -> TMEM
//          (S is log2(phi) directly; see layout.cuh)
//   epilogue warps: tcgen05.ld S -> phi = ex2(min(S*dscale, 0)) in registers;
//          KDE: row sums (Gaussian) or (sum phi, sum phi*log2 phi) (Laplace);
//          SCORE: phi -> fp16 hi/lo -> tcgen05.st back into S's own TMEM
//          columns (P aliases S, flash-attention-4 style: no SMEM round trip)
//   GEMM2 (SCORE only, A from TMEM)  O[128x48] += [P_hi | P_lo](128x256) . [B;B]
//          (B = the same column tile, MN-major) -> sum_j phi y_hi_j,
//          sum_j phi y_lo_j, sum_j phi  (TMEM, fp32)
// The n x n kernel matrix never leaves the SM; per column tile the SMEM
// traffic is the 16 KiB B tile read by both GEMMs and the 16 KiB A tile.
//
// Warp roles (320 threads): warp 0 = bulk-copy producer, warp 1 = TMEM owner +
// single-thread MMA issuer, warps 2..9 = epilogue (warp w reads TMEM lane
// quadrant w%4, column half (w-2)/4).  Pipelines (mbarriers): A tiles x2,
// B tiles x kStages, S/P accumulators x2 (TMEM), O x1 (TMEM).  The MMA
// thread's tcgen05 ops execute in issue order, so GEMM1(t+2) overwriting the
// S/P buffer of tile t is ordered after GEMM2(t) reading P(t) from it.
#pragma once
#include <cuda_fp16.h>
#include <cstdint>

#include "layout.cuh"
#include "ptx.cuh"

namespace fkde_b200 {

enum PairMode : int {
    kModeScore = 0,     // stream_score_totals
    kModeGauss = 1,     // stream_kde_pass, PairTerm::Gaussian
    kModeLaplace = 2,   // two sums (phi, phi*log2 phi): LaplaceFused / LaplaceCorrection
};

struct PairArgs {
    const uint8_t* opA;   // row tiles (A format), n_row_tiles * 16 KiB
    const uint8_t* opB;   // column tiles (B format), n_col_tiles * 16 KiB
    int n_row_tiles;
    int n_col_tiles;
    int splits;           // column ranges per row tile
    const PassScalars* sc;
    float* part0;         // SCORE: S [splits][rows_pad]; KDE: [splits*2][rows_pad]
    float* part1;         // SCORE: T [splits][rows_pad][16]; Laplace: [splits*2][rows_pad]
    size_t rows_pad;
    // SCORE: column tile holding row tile 0's diagonal (rows and columns are
    // the same point set, row shard start = diag_tile0 * 128); the self pair
    // phi_ii = 1 is excluded from the tensor-core sums and added back exactly
    // in finalize_score, so that T - x S never cancels against the self term.
    int diag_tile0;       // -1: no diagonal
};

template <int MODE>
struct TcConfig {
    static constexpr bool kScore = MODE == kModeScore;
    static constexpr int kStages = 8;
    static constexpr int kThreads = 320;
    static constexpr uint32_t kOffA = 0;
    static constexpr uint32_t kOffB = 2 * kTileBytes;
    static constexpr uint32_t kOffBar = kOffB + kStages * kTileBytes;
    static constexpr uint32_t kNumBars = 4 + 2 * kStages + 4 + 4 + 2;
    static constexpr uint32_t kSmemBytes = kOffBar + kNumBars * 8 + 16 + 1024;  // + align slack
    static constexpr uint32_t kTmemCols = 512;
    static constexpr uint32_t kTmemO = 256;   // O accumulator column (score)
    static constexpr uint32_t kN2 = 48;       // GEMM2 N
};

template <int MODE>
__global__ void __launch_bounds__(320, 1) pairwise_tc_kernel(PairArgs args) {
    using Cfg = TcConfig<MODE>;
    constexpr bool kScore = Cfg::kScore;
    constexpr int kStages = Cfg::kStages;

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~static_cast<uintptr_t>(1023));
    uint8_t* smA = smem + Cfg::kOffA;
    uint8_t* smB = smem + Cfg::kOffB;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::kOffBar);
    uint64_t* a_full = bars;              // [2]
    uint64_t* a_empty = bars + 2;         // [2]
    uint64_t* b_full = bars + 4;          // [kStages]
    uint64_t* b_empty = b_full + kStages; // [kStages]
    uint64_t* s_full = b_empty + kStages; // [2]
    uint64_t* s_empty = s_full + 2;       // [2]
    uint64_t* p_full = s_empty + 2;       // [2]
    uint64_t* p_empty = p_full + 2;       // [2]
    uint64_t* o_full = p_empty + 2;       // [1]
    uint64_t* o_empty = o_full + 1;       // [1]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_empty + 1);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&a_full[i], 1);
            ptx::mbar_init(&a_empty[i], 1);
            ptx::mbar_init(&s_full[i], 1);
            ptx::mbar_init(&s_empty[i], 8);
            ptx::mbar_init(&p_full[i], 8);
            ptx::mbar_init(&p_empty[i], 1);  // unused (P lives in TMEM)
        }
        for (int i = 0; i < kStages; ++i) {
            ptx::mbar_init(&b_full[i], 1);
            ptx::mbar_init(&b_empty[i], 1);
        }
        ptx::mbar_init(o_full, 1);
        ptx::mbar_init(o_empty, 4);
        ptx::fence_barrier_init();
    }
    if (warp == 1) ptx::tmem_alloc<Cfg::kTmemCols>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int n_units = args.n_row_tiles * args.splits;

    if (warp == 0) {
        // ===================== producer: bulk async copies =====================
        // The whole warp runs the loop (all values warp-uniform, no waterfall
        // loops around the uniform-register operands); one elected lane issues.
        const uint64_t pol_b = ptx::policy_evict_last();
        uint32_t it_a = 0, it_b = 0;
        for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
            const int rt = u / args.splits, sp = u % args.splits;
            const int ct0 = static_cast<int>((long long)sp * args.n_col_tiles / args.splits);
            const int ct1 = static_cast<int>((long long)(sp + 1) * args.n_col_tiles / args.splits);
            const int ab = it_a & 1;
            ptx::mbar_wait(&a_empty[ab], ((it_a >> 1) & 1) ^ 1);
            if (ptx::elect_one()) {
                ptx::mbar_arrive_expect_tx(&a_full[ab], kTileBytes);
                ptx::bulk_g2s(smA + ab * kTileBytes, args.opA + (size_t)rt * kTileBytes,
                              kTileBytes, &a_full[ab]);
            }
            __syncwarp();
            ++it_a;
            for (int ct = ct0; ct < ct1; ++ct) {
                const int st = it_b % kStages;
                ptx::mbar_wait(&b_empty[st], ((it_b / kStages) & 1) ^ 1);
                if (ptx::elect_one()) {
                    ptx::mbar_arrive_expect_tx(&b_full[st], kTileBytes);
                    ptx::bulk_g2s_hint(smB + st * kTileBytes, args.opB + (size_t)ct * kTileBytes,
                                       kTileBytes, &b_full[st], pol_b);
                }
                __syncwarp();
                ++it_b;
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer =====================
        // Whole warp in the loop, one elected lane issues every tcgen05 op
        // (commits must come from the issuing thread; elect.sync on a
        // converged warp always picks the same lane).  Descriptors are built
        // once and advanced by adding (byte offset >> 4) to the start-address
        // field, so each MMA costs a uniform add + the instruction.
        constexpr uint32_t idesc1 = ptx::idesc_f16_f32(128, 128, false, false);
        constexpr uint32_t idesc2 = ptx::idesc_f16_f32(128, Cfg::kN2, false, true);
        const uint64_t descA = ptx::smem_desc_sw128(ptx::smem_u32(smA), 16, 1024);
        const uint64_t descB = ptx::smem_desc_sw128(ptx::smem_u32(smB), 16, 1024);
        const uint64_t descBmn = ptx::smem_desc_sw128(ptx::smem_u32(smB), kTileBytes, 1024);
        uint32_t it_a = 0, it_b = 0, it_s = 0, it_u = 0;
        // GEMM2 of a finished tile: O += P_hi.B + P_lo.B, P read from TMEM.
        // Warp-group hf of the epilogue stored, in S buffer sb's columns
        // [hf*64, hf*64+64): P_hi (packed fp16 pairs) for K = hf*64..+63 in
        // the first 32 columns, P_lo in the next 32.
        auto gemm2 = [&](uint32_t st, uint32_t sb, uint32_t its, bool first, bool last) {
            ptx::mbar_wait(&p_full[sb], (its >> 1) & 1);
            if (first) ptx::mbar_wait(o_empty, (it_u & 1) ^ 1);
            ptx::tc_fence_after();
            if (ptx::elect_one()) {
                const uint64_t db0 = descBmn + ((st * kTileBytes) >> 4);
                const uint32_t ta0 = tmem_base + sb * 128;
#pragma unroll
                for (int part = 0; part < 2; ++part) {
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        ptx::umma_f16_ts(tmem_base + Cfg::kTmemO,
                                         ta0 + (k >> 2) * 64 + part * 32 + (k & 3) * 8,
                                         db0 + ((k * 2048) >> 4), idesc2,
                                         (first && part == 0 && k == 0) ? 0u : 1u);
                    }
                }
                ptx::umma_commit(&b_empty[st]);
                if (last) ptx::umma_commit(o_full);
            }
            __syncwarp();
            if (last) ++it_u;
        };
        for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
            const int sp = u % args.splits;
            const int ct0 = static_cast<int>((long long)sp * args.n_col_tiles / args.splits);
            const int ct1 = static_cast<int>((long long)(sp + 1) * args.n_col_tiles / args.splits);
            const int ab = it_a & 1;
            ptx::mbar_wait(&a_full[ab], (it_a >> 1) & 1);
            ptx::tc_fence_after();
            uint32_t prev_st = 0, prev_sb = 0, prev_its = 0;
            for (int ct = ct0; ct < ct1; ++ct) {
                const uint32_t st = it_b % kStages;
                const uint32_t sb = it_s & 1;
                ptx::mbar_wait(&b_full[st], (it_b / kStages) & 1);
                // KDE: the epilogue frees S after loading it.  SCORE: S/P of
                // tile it_s-2 was consumed by GEMM2, issued (in order) above.
                if constexpr (!kScore) ptx::mbar_wait(&s_empty[sb], ((it_s >> 1) & 1) ^ 1);
                ptx::tc_fence_after();
                if (ptx::elect_one()) {
                    const uint64_t da0 = descA + ((ab * kTileBytes) >> 4);
                    const uint64_t db0 = descB + ((st * kTileBytes) >> 4);
                    // K-step order: the half-norm chunk first, then y_hi.y_hi, so the
                    // large terms cancel inside one fused MMA step before the small
                    // hi/lo cross terms are added.
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const int k = kk == 0 ? 2 : (kk == 3 ? 3 : kk - 1);  // 2, 0, 1, 3
                        ptx::umma_f16(tmem_base + sb * 128, da0 + ((k * 32) >> 4),
                                      db0 + ((k * 32) >> 4), idesc1, kk > 0 ? 1u : 0u);
                    }
                    ptx::umma_commit(&s_full[sb]);
                    if constexpr (!kScore) ptx::umma_commit(&b_empty[st]);
                }
                __syncwarp();
                if constexpr (kScore) {
                    if (ct > ct0) gemm2(prev_st, prev_sb, prev_its, ct - 1 == ct0, false);
                    prev_st = st;
                    prev_sb = sb;
                    prev_its = it_s;
                }
                ++it_b;
                ++it_s;
            }
            if (ptx::elect_one()) ptx::umma_commit(&a_empty[ab]);
            __syncwarp();
            ++it_a;
            if constexpr (kScore) {
                if (ct1 > ct0) gemm2(prev_st, prev_sb, prev_its, ct1 - 1 == ct0, true);
            }
        }
    } else {
        // ===================== epilogue warps =====================
        const int q = warp & 3;             // TMEM lane quadrant
        const int hf = (warp - 2) >> 2;     // column half of each tile
        const int r = q * 32 + lane;        // row within the 128-row tile
        const float dsc = args.sc->dscale;
        const uint32_t lane_addr = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
        uint32_t it_s = 0, it_u = 0;
        for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
            const int rt = u / args.splits, sp = u % args.splits;
            const int ct0 = static_cast<int>((long long)sp * args.n_col_tiles / args.splits);
            const int ct1 = static_cast<int>((long long)(sp + 1) * args.n_col_tiles / args.splits);
            float acc0[4] = {0.f, 0.f, 0.f, 0.f};
            float acc1[4] = {0.f, 0.f, 0.f, 0.f};
            for (int ct = ct0; ct < ct1; ++ct) {
                const uint32_t sb = it_s & 1;
                ptx::mbar_wait(&s_full[sb], (it_s >> 1) & 1);
                ptx::tc_fence_after();
                uint32_t v0[32], v1[32];
                uint32_t hi_w[32], lo_w[32];
                const uint32_t ta = lane_addr + sb * 128 + hf * 64;
                ptx::tmem_ld32(ta, v0);
                ptx::tmem_ld32(ta + 32, v1);
                ptx::tmem_ld_wait();
                if constexpr (!kScore) {
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(&s_empty[sb]);
                }
                if constexpr (kScore) {
                    if (args.diag_tile0 >= 0 && ct == args.diag_tile0 + rt) {
                        const int jj = r - hf * 64;  // this row's diagonal column in v0|v1
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            if (j == jj) v0[j] = 0xFF800000u;        // -inf -> phi = 0
                            if (j + 32 == jj) v1[j] = 0xFF800000u;
                        }
                    }
                    // phi' = phi * 2^15 split into fp16 hi + lo; v0/v1 are reused as
                    // the packed P_hi / P_lo words (32 each: 64 columns, 2 per word)
#pragma unroll
                    for (int w = 0; w < 32; ++w) {
                        const uint32_t ra = w < 16 ? v0[2 * w] : v1[2 * w - 32];
                        const uint32_t rb = w < 16 ? v0[2 * w + 1] : v1[2 * w + 1 - 32];
                        const float p0 = ptx::ex2(fminf(fmaf(__uint_as_float(ra), dsc, kPScaleF), kPScaleF));
                        const float p1 = ptx::ex2(fminf(fmaf(__uint_as_float(rb), dsc, kPScaleF), kPScaleF));
                        const __half2 h = __floats2half2_rn(p0, p1);
                        const float2 hf2 = __half22float2(h);
                        const __half2 l = __floats2half2_rn(p0 - hf2.x, p1 - hf2.y);
                        hi_w[w] = *reinterpret_cast<const uint32_t*>(&h);
                        lo_w[w] = *reinterpret_cast<const uint32_t*>(&l);
                    }
                    const uint32_t tp = lane_addr + sb * 128 + hf * 64;
                    ptx::tmem_st32(tp, hi_w);
                    ptx::tmem_st32(tp + 32, lo_w);
                    ptx::tmem_st_wait();
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(&p_full[sb]);
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const float d0 = fminf(__uint_as_float(v0[j]) * dsc, 0.f);
                        const float p0 = ptx::ex2(d0);
                        acc0[j & 3] += p0;
                        if constexpr (MODE == kModeLaplace) acc1[j & 3] = fmaf(p0, d0, acc1[j & 3]);
                    }
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const float d1 = fminf(__uint_as_float(v1[j]) * dsc, 0.f);
                        const float p1 = ptx::ex2(d1);
                        acc0[j & 3] += p1;
                        if constexpr (MODE == kModeLaplace) acc1[j & 3] = fmaf(p1, d1, acc1[j & 3]);
                    }
                }
                ++it_s;
            }
            const size_t row = static_cast<size_t>(rt) * kTileRows + r;
            if constexpr (kScore) {
                if (hf == 0) {
                    ptx::mbar_wait(o_full, it_u & 1);
                    ptx::tc_fence_after();
                    uint32_t o0[32], o1[16];
                    ptx::tmem_ld32(lane_addr + Cfg::kTmemO, o0);
                    ptx::tmem_ld16(lane_addr + Cfg::kTmemO + 32, o1);
                    ptx::tmem_ld_wait();
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(o_empty);
                    const size_t idx = static_cast<size_t>(sp) * args.rows_pad + row;
                    args.part0[idx] = __uint_as_float(o1[0]);
                    float4* t = reinterpret_cast<float4*>(args.part1 + idx * kMaxDim);
#pragma unroll
                    for (int w = 0; w < 4; ++w) {
                        float4 f;
                        f.x = __uint_as_float(o0[4 * w + 0]) + __uint_as_float(o0[16 + 4 * w + 0]);
                        f.y = __uint_as_float(o0[4 * w + 1]) + __uint_as_float(o0[16 + 4 * w + 1]);
                        f.z = __uint_as_float(o0[4 * w + 2]) + __uint_as_float(o0[16 + 4 * w + 2]);
                        f.w = __uint_as_float(o0[4 * w + 3]) + __uint_as_float(o0[16 + 4 * w + 3]);
                        t[w] = f;
                    }
                }
                ++it_u;
            } else {
                const size_t idx = static_cast<size_t>(sp * 2 + hf) * args.rows_pad + row;
                args.part0[idx] = (acc0[0] + acc0[1]) + (acc0[2] + acc0[3]);
                if constexpr (MODE == kModeLaplace)
                    args.part1[idx] = (acc1[0] + acc1[1]) + (acc1[2] + acc1[3]);
            }
        }
    }

    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<Cfg::kTmemCols>(tmem_base);
    }
}

}  // namespace fkde_b200
