// direct_rows.cuh -- direct-difference recompute of the rows the tensor-core
// expansion cannot resolve to the stated tolerance.
//
// The tcgen05 passes form log2 phi as a Gram expansion
//   -|y_i - y_j|^2 / 2 = -|y_i|^2/2 - |y_j|^2/2 + y_i . y_j
// in fp32 (tensor-core accumulate) and carry phi in fp16 (score) / fp32
// (density).  Two kinds of row fall outside that range:
//   * mass: every neighbour so far away that phi underflows the fp16 / fp32
//     ranges (score: S' < 2^-16; density: sum < 2^-90);
//   * spread: |y_i|^2/2 so large (data spread >> h) that the fp32 rounding of
//     the expanded norms costs more than the tolerance (kRiskHalfNorm).
// Such rows are flagged (finalize_score / reduce_density / the pack kernel's
// risk bytes) and recomputed here the way the reference oracle does it
// (oracle.cpp:25-32, 53-85: direct coordinate differences), with a per-row
// running maximum of the exponent (online rescaling, flash style) so that
// sums far below the fp32 range keep their digits, and the self pair of the
// score handled exactly like the tensor-core path (excluded from the sums,
// added back as phi_ii = 1 in fp64).
//
// Schedule: one thread per flagged row, 128 rows per block, column range
// split so that (row blocks x splits) fills the GPU whatever the (device-side)
// flagged count is; column tiles are staged centred in fp32 in shared memory
// and broadcast to the 128 rows.  Few flagged rows (<= kDirFewRows, the usual
// case: a handful of outliers) would leave most threads of such a block idle
// and each active thread walking a long column range alone, so there the block
// works on ONE row instead, its 128 threads striding over the columns, with a
// block reduction (online maximum, then rescaled sums).  Either way the
// per-(row, split) partials are merged by the last block to finish (threadfence
// + counter), so the whole recompute is one launch that exits at once when
// nothing is flagged.
#pragma once
#include <cstdint>

#include "layout.cuh"

namespace fkde_b200 {

enum { kExactScore = 0, kExactGauss = 1, kExactLaplace = 2 };

// |y|^2/2 (y = (x - mu) sqrt(log2 e) / h, i.e. log2 units) above which a row's
// expanded-norm rounding (~|y|^2/2 * 2^-23 in log2 phi) is no longer well
// inside the 1e-3 score tolerance: such rows are recomputed here.
constexpr double kRiskHalfNorm = 128.0;

constexpr int kDirRows = 128;        // rows per block (one per thread)
constexpr int kDirTileCols = 128;    // columns per shared-memory tile
constexpr int kDirTargetItems = 4 * 148;
constexpr int kDirMaxSplits = 256;
constexpr int kDirPart = 20;         // doubles per (row, split) partial: m, S, L, T[16], pad
constexpr int kDirFewRows = 64;      // up to this many flagged rows: one row per block
// The running maximum m of the exponents (log2 units) is raised only when a new
// exponent exceeds it by more than kDirLazy: terms are then 2^(t - m) <= 2^8, far
// inside the fp32 / fp64 ranges, and the sums keep their relative precision, but
// the rescale (an fp64 exp2 and 18 multiplies, divergent across the warp's rows)
// runs a few times per row instead of at every new record (~20 % of the kernel's
// stall samples on isolated points, ncu source view).
constexpr float kDirLazy = 8.0f;

struct DirectArgs {
    int mode;                    // kExactScore / kExactGauss / kExactLaplace
    const unsigned int* count;   // flagged rows
    const unsigned int* rows;    // local row indices
    const double* rowpts;        // local row 0's point (original coordinates)
    size_t row0;                 // global index of local row 0 (score: the self column)
    int center_rows;             // subtract sc->mu from the row points
    const double* cols;          // column points, n x d
    int center_cols;             // subtract sc->mu from the column points
    size_t n;
    int d;
    const PassScalars* sc;
    double h;                    // kernel bandwidth of this pass
    double shift;                // score: h^2/2 of the SD shift
    double norm;                 // density: gaussian_norm_const(h, d) / n
    double* part;                // workspace: kDirTargetItems * kDirRows * kDirPart doubles
    unsigned int* done;          // per row block completion counters (zeroed, self-resetting)
    // score outputs (global row layout) / density output (local layout)
    double* score;
    double* xsd_c;
    double* phi_sum;
    double* weighted;
    double* out;
};

// splits per row block for a given flagged count: enough (row block, split)
// items to fill the GPU, at least one column tile per split; the same function
// runs in every block, so the merge knows the partial layout
__device__ __forceinline__ int direct_splits(unsigned int count, size_t n) {
    const int blocks = static_cast<int>((count + kDirRows - 1) / kDirRows);
    int s = (kDirTargetItems + blocks - 1) / blocks;
    const size_t max_by_cols = (n + kDirTileCols - 1) / kDirTileCols;
    if (static_cast<size_t>(s) > max_by_cols) s = static_cast<int>(max_by_cols);
    if (s > kDirMaxSplits) s = kDirMaxSplits;
    return s < 1 ? 1 : s;
}

__device__ __forceinline__ float dir_ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// finalize one row from merged (M, S, L, T) in the scaled form sum_j 2^(t_ij - M)
__device__ __forceinline__ void direct_finish_row(const DirectArgs& a, size_t i, float M, double S, double L,
                                  const double* T, int tstride = 1) {
    const double em = M == -INFINITY ? 0.0 : exp2(static_cast<double>(M));
    if (a.mode == kExactScore) {
        const size_t g = a.row0 + i;
        const double Sp = em * S;               // sum_{j != i} phi_ij
        const double Stot = 1.0 + Sp;           // + the self pair (engine.cpp:43-50)
        if (a.phi_sum) a.phi_sum[g] = Stot;
        const double inv = 1.0 / (a.h * a.h * Stot);
        for (int c = 0; c < a.d; ++c) {
            const double num = em * T[c * tstride];   // sum_j phi_ij (x_j - x_i)
            const double s = num * inv;
            const double xi = a.rowpts[i * a.d + c];
            if (a.score) a.score[g * a.d + c] = s;
            if (a.xsd_c) a.xsd_c[g * a.d + c] = (xi - a.sc->mu[c]) + a.shift * s;
            if (a.weighted) a.weighted[g * a.d + c] = num + xi * Stot;
        }
    } else if (a.mode == kExactGauss) {
        a.out[i] = a.norm * (em * S);
    } else {
        // phi (1 + d/2 - u): u = r^2/(2h^2) = -t ln 2
        a.out[i] = a.norm * (em * ((1.0 + 0.5 * a.d) * S - L));
    }
}

// Block-wide merge of per-thread (m, v[kMaxDim + 2]) = scaled sums sum 2^(t - m):
// returns (in every thread) the block maximum M and v rescaled to it and summed.
__device__ __forceinline__ float direct_block_merge(float m, double (&v)[kMaxDim + 2]) {
    __shared__ double red[kDirRows / 32][kMaxDim + 2];
    __shared__ float redm[kDirRows / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    float M = m;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    if (lane == 0) redm[w] = M;
    __syncthreads();
    M = redm[0];
#pragma unroll
    for (int q = 1; q < kDirRows / 32; ++q) M = fmaxf(M, redm[q]);
    const double f = m == -INFINITY ? 0.0 : exp2(static_cast<double>(m) - static_cast<double>(M));
#pragma unroll
    for (int k = 0; k < kMaxDim + 2; ++k) {
        v[k] *= f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
    }
    if (lane == 0)
#pragma unroll
        for (int k = 0; k < kMaxDim + 2; ++k) red[w][k] = v[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kMaxDim + 2; ++k) {
        v[k] = red[0][k];
        for (int q = 1; q < kDirRows / 32; ++q) v[k] += red[q][k];
    }
    __syncthreads();   // (red / redm reused by the next call)
    return M;
}

// Few flagged rows: block = (row, column split), threads stride over the columns.
__device__ __forceinline__ void direct_few_rows(const DirectArgs& a, unsigned int count) {
    __shared__ int s_last;
    const int d = a.d;
    int S = (kDirTargetItems + static_cast<int>(count) - 1) / static_cast<int>(count);
    const size_t max_by_cols = (a.n + kDirTileCols - 1) / kDirTileCols;
    if (static_cast<size_t>(S) > max_by_cols) S = static_cast<int>(max_by_cols);
    if (S < 1) S = 1;
    const int items = static_cast<int>(count) * S;
    const float k2 = static_cast<float>(1.4426950408889634 / (2.0 * a.h * a.h));
    const double ln2 = 0.69314718055994530942;
    for (int it = blockIdx.x; it < items; it += gridDim.x) {
        const int ridx = it / S, sp = it % S;
        const size_t i = a.rows[ridx];
        float u[kMaxDim];
#pragma unroll
        for (int c = 0; c < kMaxDim; ++c)
            u[c] = c < d ? static_cast<float>(a.rowpts[i * d + c] - (a.center_rows ? a.sc->mu[c] : 0.0)) : 0.f;
        const size_t self = a.mode == kExactScore ? a.row0 + i : ~static_cast<size_t>(0);
        const size_t j0 = a.n * sp / S, j1 = a.n * (sp + 1) / S;
        float m = -INFINITY;
        double S64 = 0.0, L64 = 0.0, T64[kMaxDim];
#pragma unroll
        for (int c = 0; c < kMaxDim; ++c) T64[c] = 0.0;
        // one column's contribution (coordinates already loaded into vv)
        auto pair = [&](size_t j, const float (&vv)[kMaxDim]) {
            float df[kMaxDim];
            float r2 = 0.f;
#pragma unroll
            for (int c = 0; c < kMaxDim; ++c) {
                df[c] = vv[c] - u[c];
                r2 = fmaf(df[c], df[c], r2);
            }
            if (j == self) return;   // phi_ii = 1 is added back in fp64
            const float t = -r2 * k2;
            if (t > m + kDirLazy) {   // lazy running maximum (see kDirLazy)
                const double f64 = exp2(static_cast<double>(m) - static_cast<double>(t));
                S64 *= f64;
                L64 *= f64;
#pragma unroll
                for (int c = 0; c < kMaxDim; ++c) T64[c] *= f64;
                m = t;
            }
            const float p = dir_ex2(t - m);
            S64 += p;
            if (a.mode == kExactLaplace) L64 += static_cast<double>(p) * static_cast<double>(-t);
            if (a.mode == kExactScore) {
#pragma unroll
                for (int c = 0; c < kMaxDim; ++c) T64[c] += static_cast<double>(p * df[c]);
            }
        };
        auto load = [&](size_t j, float (&vv)[kMaxDim]) {
#pragma unroll
            for (int c = 0; c < kMaxDim; ++c)
                vv[c] = c < d ? static_cast<float>(a.cols[j * d + c] - (a.center_cols ? a.sc->mu[c] : 0.0)) : 0.f;
        };
        // two columns per step, both loaded before either is used: the loop is bound by
        // the L2 round trip of its column loads (ncu: 83 % of the stall samples at config
        // 4, issue slots 12 % busy), so two round trips overlap
        for (size_t j = j0 + threadIdx.x; j < j1; j += 2 * kDirRows) {
            const size_t j2 = j + kDirRows;
            float va[kMaxDim], vb[kMaxDim];
            load(j, va);
            if (j2 < j1) load(j2, vb);
            pair(j, va);
            if (j2 < j1) pair(j2, vb);
        }
        // block reduction: maximum, then the sums rescaled to it
        double v[kMaxDim + 2];
        v[0] = S64;
        v[1] = L64;
#pragma unroll
        for (int c = 0; c < kMaxDim; ++c) v[2 + c] = T64[c];
        const float M = direct_block_merge(m, v);
        if (threadIdx.x == 0) {
            if (S == 1) {
                direct_finish_row(a, i, M, v[0], v[1] * ln2, v + 2);
            } else {
                double* p = a.part + (static_cast<size_t>(ridx) * S + sp) * kDirPart;
                p[0] = static_cast<double>(M);
                p[1] = v[0];
                p[2] = v[1] * ln2;
#pragma unroll
                for (int c = 0; c < kMaxDim; ++c) p[3 + c] = v[2 + c];
                __threadfence();
                s_last = atomicAdd(&a.done[ridx], 1u) == static_cast<unsigned int>(S - 1);
            }
        }
        __syncthreads();
        if (S > 1 && s_last) {
            // last split of this row to finish: merge the S partials across the block
            // (thread t takes splits t, t + 128, ...; a fixed order, so deterministic)
            __threadfence();
            const double* p = a.part + static_cast<size_t>(ridx) * S * kDirPart;
            float mt = -INFINITY;
            for (int s = threadIdx.x; s < S; s += kDirRows) mt = fmaxf(mt, static_cast<float>(__ldcg(p + s * kDirPart)));
            double w[kMaxDim + 2];
#pragma unroll
            for (int k = 0; k < kMaxDim + 2; ++k) w[k] = 0.0;
            for (int s = threadIdx.x; s < S; s += kDirRows) {
                const double* q = p + s * kDirPart;
                const float ms = static_cast<float>(__ldcg(q));
                if (ms == -INFINITY) continue;
                const double fs = exp2(static_cast<double>(ms) - static_cast<double>(mt));
#pragma unroll
                for (int k = 0; k < kMaxDim + 2; ++k) w[k] += fs * __ldcg(q + 1 + k);
            }
            const float Mm = direct_block_merge(mt, w);
            if (threadIdx.x == 0) {
                direct_finish_row(a, i, Mm, w[0], w[1], w + 2);
                a.done[ridx] = 0u;   // ready for the next call
            }
        }
        __syncthreads();   // (s_last reused by the next item)
    }
}

// (<= 128 registers: four blocks per SM, the grid is one wave; the few-row loop's
// two-column unroll would otherwise take the kernel to ~170)
__global__ void __launch_bounds__(kDirRows, 4) direct_rows_kernel(DirectArgs a) {
    pdl_launch_dependents();
    pdl_wait();
    __shared__ float4 tile[kDirTileCols][kMaxDim / 4];
    __shared__ int s_last;
    const unsigned int count = *a.count;
    if (count == 0) return;
    if (count <= static_cast<unsigned int>(kDirFewRows)) {
        direct_few_rows(a, count);
        return;
    }
    const int nblk = static_cast<int>((count + kDirRows - 1) / kDirRows);
    const int S = direct_splits(count, a.n);
    const int items = nblk * S;
    const int d = a.d;
    // exponent in log2 units: t = -r^2 * k2, k2 = log2(e) / (2 h^2)
    const float k2 = static_cast<float>(1.4426950408889634 / (2.0 * a.h * a.h));
    const double ln2 = 0.69314718055994530942;

    for (int it = blockIdx.x; it < items; it += gridDim.x) {
        const int rb = it / S, sp = it % S;
        const unsigned int ridx = static_cast<unsigned int>(rb * kDirRows + threadIdx.x);
        const bool active = ridx < count;
        const size_t i = active ? a.rows[ridx] : 0;
        float u[kMaxDim];
#pragma unroll
        for (int c = 0; c < kMaxDim; ++c) {
            double v = 0.0;
            if (active && c < d)
                v = a.rowpts[i * d + c] - (a.center_rows ? a.sc->mu[c] : 0.0);
            u[c] = static_cast<float>(v);
        }
        const size_t self = (a.mode == kExactScore && active) ? a.row0 + i : ~static_cast<size_t>(0);
        const size_t j0 = a.n * sp / S, j1 = a.n * (sp + 1) / S;
        float m = -INFINITY;
        double S64 = 0.0, L64 = 0.0, T64[kMaxDim];
#pragma unroll
        for (int c = 0; c < kMaxDim; ++c) T64[c] = 0.0;
        for (size_t jt = j0; jt < j1; jt += kDirTileCols) {
            const int nt = static_cast<int>(j1 - jt < static_cast<size_t>(kDirTileCols) ? j1 - jt : kDirTileCols);
            __syncthreads();
            // stage nt columns, centred, fp32 (zero-padded beyond d)
            for (int e = threadIdx.x; e < nt * kMaxDim; e += blockDim.x) {
                const int jj = e / kMaxDim, c = e % kMaxDim;
                float v = 0.f;
                if (c < d)
                    v = static_cast<float>(a.cols[(jt + jj) * d + c] -
                                           (a.center_cols ? a.sc->mu[c] : 0.0));
                reinterpret_cast<float*>(&tile[jj][0])[c] = v;
            }
            __syncthreads();
            float s32 = 0.f, l32 = 0.f, t32[kMaxDim];
#pragma unroll
            for (int c = 0; c < kMaxDim; ++c) t32[c] = 0.f;
            // the self pair (score): its exponent is pushed to -1e30 (phi = 0 exactly;
            // phi_ii = 1 is added back in fp64) -- an int compare against one index
            // per tile instead of a 64-bit compare and a divergent branch per pair
            const int jself = (self >= jt && self < jt + static_cast<size_t>(nt)) ? static_cast<int>(self - jt) : -1;
            if (active) {
#pragma unroll 2
                for (int jj = 0; jj < nt; ++jj) {
                    float df[kMaxDim];
                    float r2 = 0.f;
#pragma unroll
                    for (int q = 0; q < kMaxDim / 4; ++q) {
                        const float4 cv = tile[jj][q];
                        df[4 * q + 0] = cv.x - u[4 * q + 0];
                        df[4 * q + 1] = cv.y - u[4 * q + 1];
                        df[4 * q + 2] = cv.z - u[4 * q + 2];
                        df[4 * q + 3] = cv.w - u[4 * q + 3];
                    }
                    // four partial sums: a 16-deep dependent FFMA chain per pair was the
                    // latency that bound this loop at 4 warps per sub-partition
                    float r2p[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                    for (int c = 0; c < kMaxDim; ++c) r2p[c & 3] = fmaf(df[c], df[c], r2p[c & 3]);
                    r2 = (r2p[0] + r2p[1]) + (r2p[2] + r2p[3]);
                    const float t = jj == jself ? -1e30f : -r2 * k2;
                    if (t > m + kDirLazy) {   // new running maximum (lazy): rescale the sums
                        // (one fp32 ex2 for both: a software fp64 exp2 here, executed by the
                        // whole warp whenever any of its rows rescaled, was 11 % of the
                        // kernel's instructions; the factor's 2^-22 relative error is far
                        // inside the tolerance, and it underflows to 0 exactly when the old
                        // terms are below 2^-126 of the new maximum)
                        const float f = dir_ex2(m - t);
                        const double f64 = static_cast<double>(f);
                        s32 *= f;
                        l32 *= f;
#pragma unroll
                        for (int c = 0; c < kMaxDim; ++c) t32[c] *= f;
                        S64 *= f64;
                        L64 *= f64;
#pragma unroll
                        for (int c = 0; c < kMaxDim; ++c) T64[c] *= f64;
                        m = t;
                    }
                    const float p = dir_ex2(t - m);
                    s32 += p;
                    if (a.mode == kExactLaplace) l32 = fmaf(p, -t, l32);   // phi * (-t) = phi u / ln 2
                    if (a.mode == kExactScore) {
#pragma unroll
                        for (int c = 0; c < kMaxDim; ++c) t32[c] = fmaf(p, df[c], t32[c]);
                    }
                }
            }
            S64 += s32;
            L64 += l32;
#pragma unroll
            for (int c = 0; c < kMaxDim; ++c) T64[c] += t32[c];
        }
        if (S == 1) {
            if (active) {
                L64 *= ln2;
                direct_finish_row(a, i, m, S64, L64, T64);
            }
            continue;
        }
        // partial of (row, split)
        if (active) {
            double* p = a.part + (static_cast<size_t>(ridx) * S + sp) * kDirPart;
            p[0] = static_cast<double>(m);
            p[1] = S64;
            p[2] = L64 * ln2;
#pragma unroll
            for (int c = 0; c < kMaxDim; ++c) p[3 + c] = T64[c];
        }
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned int prev = atomicAdd(&a.done[rb], 1u);
            s_last = prev == static_cast<unsigned int>(S - 1);
        }
        __syncthreads();
        if (s_last) {
            // last split of this row block to finish: merge in split order
            __threadfence();
            if (active) {
                // (L2 reads: other blocks wrote these, this SM's L1 may hold stale lines)
                const double* p = a.part + static_cast<size_t>(ridx) * S * kDirPart;
                float M = -INFINITY;
                for (int s = 0; s < S; ++s) M = fmaxf(M, static_cast<float>(__ldcg(p + s * kDirPart)));
                double Sm = 0.0, Lm = 0.0, Tm[kMaxDim];
#pragma unroll
                for (int c = 0; c < kMaxDim; ++c) Tm[c] = 0.0;
                for (int s = 0; s < S; ++s) {
                    const double* q = p + s * kDirPart;
                    const float ms = static_cast<float>(__ldcg(q));
                    if (ms == -INFINITY) continue;
                    const double f = exp2(static_cast<double>(ms) - static_cast<double>(M));
                    Sm += f * __ldcg(q + 1);
                    Lm += f * __ldcg(q + 2);
#pragma unroll
                    for (int c = 0; c < kMaxDim; ++c) Tm[c] += f * __ldcg(q + 3 + c);
                }
                direct_finish_row(a, i, M, Sm, Lm, Tm);
            }
            if (threadIdx.x == 0) a.done[rb] = 0u;   // ready for the next call
        }
    }
}

}  // namespace fkde_b200
