// spatial_order.cuh -- spatially coherent ordering of the training points for
// the score pass, and the per-tile summaries its tile skipping reads.
//
// The score pass carries phi' = phi * 2^15 as fp16 hi + lo (pairwise_tc.cuh), so
// every pair with log2 phi' < -25 contributes exactly zero (both halves round
// to fp16 zero).  For clustered data most (row tile, column tile) pairs consist
// only of such pairs -- if the tiles are spatially coherent.  The reference
// processes points in input order (engine.cpp:172-244); here the points are
// first ordered along a Morton (Z-order) curve over their top three principal
// axes, so that a 128-point tile is a compact neighbourhood, and the score
// kernel skips the exp work of tile pairs that contribute exactly zero.  The
// outputs are permuted back to the caller's order.  Only the summation order
// changes; the arithmetic of every contributing pair is the same.
//
//   cov_stage1      per-block partial covariance of the centred points (fp64)
//   order_axes      reduce partials -> covariance -> top-3 principal axes
//                   (subspace iteration, one block, deterministic signs)
//   morton_keys     project, quantise to 10 bits per axis, interleave -> 30-bit key
//   (cub::DeviceRadixSort::SortPairs: keys + original indices -> permutation)
//   gather_rows / scatter_rows   X -> X[perm], and outputs back to input order
//   tile_summary    per-tile centroid + coordinate / principal-axis boxes (log2 units)
//   tile_predict    proven-zero tile pairs (box bound) and the pairs to check exactly
#pragma once
#include <cstdint>

#include "layout.cuh"

namespace fkde_b200 {

constexpr int kOrderAxes = 3;
constexpr int kMortonBits = 10;     // per axis -> 30-bit keys
// bits of the key the sort orders by: the top FKDE_MORTON_SORT_BITS of the 30-bit
// Morton key (the top 8 bits of each axis at 24: a cell is 1/256 of +-4 sigma per
// axis, far finer than a 128-point tile) -- CUB's onesweep sort then runs 3
// passes of 8 bits instead of 4
#ifndef FKDE_MORTON_SORT_BITS
#define FKDE_MORTON_SORT_BITS 24
#endif
constexpr int kSortBits = FKDE_MORTON_SORT_BITS;
static_assert(kSortBits <= kOrderAxes * kMortonBits, "sort bits within the key");

struct OrderScalars {
    double axis[kOrderAxes][kMaxDim];   // unit principal axes
    double inv_scale[kOrderAxes];       // 1 / (4 sqrt(lambda_k)): projections -> ~[-1, 1]
};

// ---- covariance partials: block b sums (x - mu)(x - mu)^T over its sample range ---------
// The axes only choose the ordering (any basis orders correctly; the results'
// arithmetic never depends on it), so the covariance is taken over a fixed strided
// sample of ns <= kCovSample points -- point (k n) / ns for k < ns, deterministic --
// rather than all n (at n = 2^20 the full sum was ~0.2 ms per call).
constexpr size_t kCovSample = 65536;
inline size_t cov_sample_count(size_t n) { return n < kCovSample ? n : kCovSample; }
__global__ void __launch_bounds__(256) cov_stage1(const double* __restrict__ x, size_t n, size_t ns,
                                                  int d, const PassScalars* __restrict__ sc,
                                                  double* __restrict__ part /* [grid][256] */) {
    __shared__ double rows[64][kMaxDim];
    const int a = threadIdx.x >> 4, b = threadIdx.x & 15;
    const size_t r0 = ns * blockIdx.x / gridDim.x, r1 = ns * (blockIdx.x + 1) / gridDim.x;
    double acc = 0.0;
    for (size_t base = r0; base < r1; base += 64) {
        const int nr = static_cast<int>(r1 - base < 64 ? r1 - base : 64);
        __syncthreads();
        for (int e = threadIdx.x; e < 64 * kMaxDim; e += 256) {
            const int r = e / kMaxDim, c = e % kMaxDim;
            const size_t row = (base + r) * n / ns;   // (== base + r when ns == n)
            rows[r][c] = (r < nr && c < d) ? x[row * d + c] - sc->mu[c] : 0.0;
        }
        __syncthreads();
        for (int r = 0; r < nr; ++r) acc = fma(rows[r][a], rows[r][b], acc);
    }
    part[blockIdx.x * 256 + threadIdx.x] = acc;
}

// ---- covariance -> top principal axes (one block of 256 threads) -----------------------
// Subspace iteration Q <- orth(C Q) on the 16 x 16 covariance, one warp: lane r < 16
// owns row r of C and of Q, dot products are warp reductions (a single thread
// running Gram-Schmidt took ~120 us).  The top-3 eigengap of clustered data is
// large; for unclustered data any basis of the top subspace orders equally well.
__device__ __forceinline__ double warp_sum16(double v) {
    for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__global__ void __launch_bounds__(256) order_axes(const double* __restrict__ part, int nparts,
                                                  int d, OrderScalars* __restrict__ os) {
    __shared__ double C[kMaxDim][kMaxDim];
    const int t = threadIdx.x;
    {
        // (unrolled: 8 independent L2 loads in flight instead of one round trip per
        // partial; the association order is fixed, so C is deterministic)
        double s = 0.0;
        int p = 0;
        for (; p + 8 <= nparts; p += 8) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = part[(p + u) * 256 + t];
#pragma unroll
            for (int u = 0; u < 8; ++u) s += v[u];
        }
        for (; p < nparts; ++p) s += part[p * 256 + t];
        C[t >> 4][t & 15] = s;
    }
    __syncthreads();
    if (t >= 32) return;
    const int r = t & 15;   // lanes 16..31 mirror 0..15 (the reductions stay within halves)
    double q[kOrderAxes];
#pragma unroll
    for (int k = 0; k < kOrderAxes; ++k) q[k] = (r == k) ? 1.0 : 0.0;
    double crow[kMaxDim];
#pragma unroll
    for (int c = 0; c < kMaxDim; ++c) crow[c] = C[r][c];
    for (int it = 0; it < 24; ++it) {
        double z[kOrderAxes];
#pragma unroll
        for (int k = 0; k < kOrderAxes; ++k) {   // z = C q (row r)
            double acc0 = 0.0, acc1 = 0.0;   // two chains: half the dependent-FMA latency
#pragma unroll
            for (int c = 0; c < kMaxDim; c += 2) {
                acc0 = fma(crow[c], __shfl_sync(0xffffffffu, q[k], c), acc0);
                acc1 = fma(crow[c + 1], __shfl_sync(0xffffffffu, q[k], c + 1), acc1);
            }
            z[k] = acc0 + acc1;
        }
#pragma unroll
        for (int k = 0; k < kOrderAxes; ++k) {   // modified Gram-Schmidt
#pragma unroll
            for (int j = 0; j < k; ++j) {
                const double dp = warp_sum16(z[k] * z[j]);
                z[k] -= dp * z[j];
            }
            double nn = warp_sum16(z[k] * z[k]);
            if (!(nn > 1e-300)) {   // degenerate (d < 3, zero-variance subspace): a coordinate axis
                z[k] = (r == k) ? 1.0 : 0.0;
#pragma unroll
                for (int j = 0; j < k; ++j) {
                    const double dp = warp_sum16(z[k] * z[j]);
                    z[k] -= dp * z[j];
                }
                nn = warp_sum16(z[k] * z[k]);
            }
            z[k] *= nn > 1e-300 ? 1.0 / sqrt(nn) : 0.0;
        }
#pragma unroll
        for (int k = 0; k < kOrderAxes; ++k) q[k] = z[k];
    }
#pragma unroll
    for (int k = 0; k < kOrderAxes; ++k) {
        // deterministic sign: largest-magnitude component positive (ties: lowest index)
        double best = fabs(q[k]);
        int am = r;
        for (int o = 8; o > 0; o >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int oa = __shfl_xor_sync(0xffffffffu, am, o);
            if (ob > best || (ob == best && oa < am)) {
                best = ob;
                am = oa;
            }
        }
        const double sg = __shfl_sync(0xffffffffu, q[k], am) < 0.0 ? -1.0 : 1.0;
        double cq = 0.0;
#pragma unroll
        for (int c = 0; c < kMaxDim; ++c) cq = fma(crow[c], __shfl_sync(0xffffffffu, q[k], c), cq);
        const double lam = warp_sum16(q[k] * cq);
        if (t < 16) os->axis[k][r] = (r < d) ? sg * q[k] : 0.0;
        // covariance is a sum over n points: lam / n is the variance (the caller's
        // projection multiplies by sqrt(n))
        if (t == 0) os->inv_scale[k] = lam > 0.0 ? 1.0 / (4.0 * sqrt(lam)) : 0.0;
    }
}

__device__ __forceinline__ uint32_t spread3(uint32_t v) {   // 10 bits -> every third bit
    v &= 0x3FFu;
    v = (v | (v << 16)) & 0x030000FFu;
    v = (v | (v << 8)) & 0x0300F00Fu;
    v = (v | (v << 4)) & 0x030C30C3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}

// n_total: the point count the covariance was summed over (variance = lam / n_total)
__global__ void morton_keys(const double* __restrict__ x, size_t n, int d, double sqrt_n,
                            const PassScalars* __restrict__ sc, const OrderScalars* __restrict__ os,
                            uint32_t* __restrict__ keys, uint32_t* __restrict__ idx) {
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double p[kOrderAxes] = {0.0, 0.0, 0.0};
    for (int c = 0; c < d; ++c) {
        const double v = x[i * d + c] - sc->mu[c];
#pragma unroll
        for (int k = 0; k < kOrderAxes; ++k) p[k] = fma(v, os->axis[k][c], p[k]);
    }
    uint32_t key = 0;
#pragma unroll
    for (int k = 0; k < kOrderAxes; ++k) {
        // p / (4 sigma_k), sigma_k = sqrt(lam_k / n): [-1, 1] -> [0, 1023]
        double u = p[k] * os->inv_scale[k] * sqrt_n;
        u = (u + 1.0) * 0.5 * static_cast<double>((1 << kMortonBits) - 1);
        u = u < 0.0 ? 0.0 : (u > 1023.0 ? 1023.0 : u);
        if (!(u == u)) u = 0.0;
        key |= spread3(static_cast<uint32_t>(u)) << (kOrderAxes - 1 - k);
    }
    keys[i] = key >> (kOrderAxes * kMortonBits - kSortBits);
    idx[i] = static_cast<uint32_t>(i);
}

// out[g] = x[perm[g]]  (rows of d doubles)
__global__ void gather_rows(const double* __restrict__ x, const uint32_t* __restrict__ perm, size_t n,
                            int d, double* __restrict__ out) {
    const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (t >= n * d) return;
    const size_t g = t / d;
    const int c = static_cast<int>(t % d);
    out[t] = x[static_cast<size_t>(perm[g]) * d + c];
}

// out[perm[g]] = in[g] (+ mu)   for g < n; rows of `width` doubles
__global__ void scatter_rows(const double* __restrict__ in, const uint32_t* __restrict__ perm,
                             size_t n, int width, const PassScalars* __restrict__ add_mu,
                             double* __restrict__ out) {
    const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (t >= n * width) return;
    const size_t g = t / width;
    const int c = static_cast<int>(t % width);
    out[static_cast<size_t>(perm[g]) * width + c] = in[t] + (add_mu ? add_mu->mu[c] : 0.0);
}

// Per-tile summaries (log2 units: y = (x - mu) sqrt(log2 e) / h), one block of
// 128 threads (one point each) per tile of tile_w <= 128 points (rows beyond n
// are padding and ignored):
//   cen[tile][16]   centroid (the skip predictor's input)
//   box[tile][38]   [0..15] / [16..31] per-coordinate min / max, [32..37] min / max
//                   of the projections on the three principal axes -- two boxes
//                   whose separation bounds every point distance from below
constexpr int kBoxFloats = 38;
__global__ void __launch_bounds__(128) tile_summary(const double* __restrict__ x, size_t n, int d,
                                                    const PassScalars* __restrict__ sc,
                                                    const OrderScalars* __restrict__ os, double k,
                                                    int tile_w, int centred, float* __restrict__ cen,
                                                    float* __restrict__ box) {
    constexpr int V = kMaxDim + kOrderAxes;
    // the 128 points' 19 values go through shared memory and are reduced by 76
    // threads (value v, interleaved quarter p of the rows), not by 19 x 3 five-level
    // shuffle trees per warp (~1100 SHFL per tile)
    constexpr int kStride = V + 1;
    __shared__ float vals[128 * kStride];
    __shared__ unsigned char ok[128];
    const size_t r0 = static_cast<size_t>(blockIdx.x) * tile_w;
    const size_t r1 = r0 + tile_w < n ? r0 + tile_w : n;
    const size_t r = r0 + threadIdx.x;
    const bool valid = threadIdx.x < tile_w && r < r1;
    {
        double y[kMaxDim];
#pragma unroll
        for (int c = 0; c < kMaxDim; ++c)
            y[c] = (valid && c < d) ? (x[r * d + c] - (centred ? 0.0 : sc->mu[c])) * k : 0.0;
        float* row = vals + threadIdx.x * kStride;
#pragma unroll
        for (int c = 0; c < kMaxDim; ++c) row[c] = static_cast<float>(y[c]);
#pragma unroll
        for (int a = 0; a < kOrderAxes; ++a) {
            double p = 0.0;
#pragma unroll
            for (int c = 0; c < kMaxDim; ++c) p = fma(y[c], os->axis[a][c], p);
            row[kMaxDim + a] = static_cast<float>(p);
        }
        ok[threadIdx.x] = valid ? 1 : 0;
    }
    __syncthreads();
    const int t = threadIdx.x;
    if (t >= 96) return;   // warps 0-2 (whole warps: the shuffles below): t = 4v + p, v < V work
    const int v = t >> 2, p = t & 3;
    float s = 0.f, l = INFINITY, h = -INFINITY;
    if (v < V)
        for (int i = p; i < 128; i += 4) {   // fixed order per quarter: deterministic
            if (!ok[i]) continue;
            const float x = vals[i * kStride + v];
            s += x;
            l = fminf(l, x);
            h = fmaxf(h, x);
        }
    for (int o = 1; o < 4; o <<= 1) {   // the four quarters (lanes 4v .. 4v+3)
        s += __shfl_xor_sync(0xffffffffu, s, o);
        l = fminf(l, __shfl_xor_sync(0xffffffffu, l, o));
        h = fmaxf(h, __shfl_xor_sync(0xffffffffu, h, o));
    }
    if (p == 0 && v < V) {
        const float cnt = r1 > r0 ? static_cast<float>(r1 - r0) : 1.f;
        if (v < kMaxDim) {
            cen[static_cast<size_t>(blockIdx.x) * kMaxDim + v] = r1 > r0 ? s / cnt : 1e18f;
            box[static_cast<size_t>(blockIdx.x) * kBoxFloats + v] = l;
            box[static_cast<size_t>(blockIdx.x) * kBoxFloats + kMaxDim + v] = h;
        } else {
            const int a = v - kMaxDim;
            box[static_cast<size_t>(blockIdx.x) * kBoxFloats + 2 * kMaxDim + 2 * a] = l;
            box[static_cast<size_t>(blockIdx.x) * kBoxFloats + 2 * kMaxDim + 2 * a + 1] = h;
        }
    }
}


// Skip predictor.  Per tile pair:
//   * proven: the box separation (coordinates, or the principal-axis projections;
//     projections never lengthen a distance) bounds every pair's r^2 from below;
//     if even that pair has log2 phi' = 15 - r^2/2 below kSkipLog2 (with a margin
//     for the float boxes), the tile is skipped without a check (pred 0, skip 1);
//   * predicted: centroid half-distance^2 > thresh -> checked exactly by the
//     check pass (pred 1, skip 1 until the check clears it);
//   * otherwise computed (pred 0, skip 0).
// skip_count (optional, zeroed by the caller): += skipped tiles per row tile.
// skip_mass (optional, zeroed by the caller; density passes): += per row tile the
// bound on what one row loses to the skipped tiles, sum over them of tile_w *
// phi_max * (1 (Gaussian) | 1 + d/2 + ln2 |log2 phi_max| (Laplace-fused, lap_d = d)),
// phi_max = 2^-(r^2/2 lower bound - 0.5): reduce_density recomputes the rows whose
// mass does not dominate it.
// Block = 128 row tiles (one per thread) x kPredWords mask words (32 column tiles
// each): the column tiles' summaries are staged once in shared memory, so each
// summary is read from global memory once per 128 row tiles (a thread per (row
// tile, word) re-reading its 32 column summaries moved ~14 GB at n = 2^20).
constexpr int kPredWords = 4;   // mask words per block at most (wpb <= kPredWords)

// tile_predict's launch shape: blocks of `rows` row tiles (one per thread) x `wpb`
// mask words.  Large problems use 128 x kPredWords (each column summary read from
// global memory once per 128 row tiles); small ones (a few hundred tiles a side)
// halve both until the grid covers the GPU twice, instead of leaving a handful of
// blocks to walk 128 column tiles per thread.
struct PredShape {
    unsigned rows, wpb, gx, gy;
};
inline PredShape pred_shape(size_t row_tiles, int words, int sms) {
    PredShape p{128u, static_cast<unsigned>(kPredWords), 0u, 0u};
    for (;;) {
        p.gx = static_cast<unsigned>((row_tiles + p.rows - 1) / p.rows);
        p.gy = static_cast<unsigned>((words + p.wpb - 1) / p.wpb);
        if (static_cast<size_t>(p.gx) * p.gy >= 2u * static_cast<unsigned>(sms)) break;
        if (p.wpb > 1) p.wpb >>= 1;
        else if (p.rows > 32) p.rows >>= 1;
        else break;
    }
    return p;
}
constexpr int kSumFloats = kMaxDim + kBoxFloats;   // centroid + boxes
__global__ void __launch_bounds__(128) tile_predict(const float* __restrict__ cenA,
                                                    const float* __restrict__ boxA, int row_tiles,
                                                    const float* __restrict__ cenB,
                                                    const float* __restrict__ boxB, int col_tiles,
                                                    int words, float thresh, float proven_half_r2,
                                                    uint32_t* __restrict__ pred,
                                                    uint32_t* __restrict__ skip,
                                                    unsigned int* __restrict__ skip_count,
                                                    float* __restrict__ skip_mass = nullptr,   // [gridDim.y][row_tiles]
                                                    int lap_d = -1, float tile_w = 128.f,
                                                    int wpb = kPredWords) {
    pdl_launch_dependents();
    pdl_wait();
    __shared__ float colsum[kPredWords * 32][kSumFloats];
    const int w0 = blockIdx.y * wpb;
    const int ct0 = w0 * 32;
    const int nct = min(wpb * 32, col_tiles - ct0);
    for (int e = threadIdx.x; e < nct * kSumFloats; e += blockDim.x) {
        const int j = e / kSumFloats, v = e % kSumFloats;
        colsum[j][v] = v < kMaxDim ? cenB[(size_t)(ct0 + j) * kMaxDim + v]
                                   : boxB[(size_t)(ct0 + j) * kBoxFloats + (v - kMaxDim)];
    }
    __syncthreads();
    const int rt = blockIdx.x * blockDim.x + threadIdx.x;
    if (rt >= row_tiles) return;
    float a[kMaxDim], ab[kBoxFloats];
#pragma unroll
    for (int c = 0; c < kMaxDim; ++c) a[c] = cenA[(size_t)rt * kMaxDim + c];
#pragma unroll
    for (int c = 0; c < kBoxFloats; ++c) ab[c] = boxA[(size_t)rt * kBoxFloats + c];
    unsigned int nskip = 0;
    float mass = 0.f;
    for (int wi = 0; wi < wpb && w0 + wi < words; ++wi) {
        uint32_t pbits = 0, sbits = 0;
        for (int b = 0; b < 32; ++b) {
            const int j = wi * 32 + b;
            if (j >= nct) break;
            const float* cs = colsum[j];   // (all threads read the same address: broadcast)
            float lower = 0.f;
#pragma unroll
            for (int c = 0; c < kMaxDim; ++c) {   // coordinate boxes
                const float g = fmaxf(0.f, fmaxf(cs[kMaxDim + c] - ab[kMaxDim + c],
                                                 ab[c] - cs[2 * kMaxDim + c]));
                lower = fmaf(g, g, lower);
            }
            float lbp = 0.f;
#pragma unroll
            for (int q = 0; q < kOrderAxes; ++q) {   // principal-axis boxes
                const float alo = ab[2 * kMaxDim + 2 * q], ahi = ab[2 * kMaxDim + 2 * q + 1];
                const float blo = cs[3 * kMaxDim + 2 * q], bhi = cs[3 * kMaxDim + 2 * q + 1];
                const float g = fmaxf(0.f, fmaxf(blo - ahi, alo - bhi));
                lbp = fmaf(g, g, lbp);
            }
            if (0.5f * fmaxf(lower, lbp) > proven_half_r2) {
                sbits |= 1u << b;
                if (skip_mass) {
                    const float x = 0.5f * fmaxf(lower, lbp) - 0.5f;   // -log2 phi_max
                    mass += exp2f(-x) * (lap_d >= 0 ? 1.f + 0.5f * lap_d + 0.6931472f * x : 1.f);
                }
                continue;
            }
            float dd = 0.f;
#pragma unroll
            for (int c = 0; c < kMaxDim; ++c) {
                const float df = a[c] - cs[c];
                dd = fmaf(df, df, dd);
            }
            if (0.5f * dd > thresh) {
                pbits |= 1u << b;
                sbits |= 1u << b;
            }
        }
        const size_t t = (size_t)rt * words + w0 + wi;
        pred[t] = pbits;
        skip[t] = sbits;
        nskip += __popc(sbits);
    }
    if (skip_count && nskip) atomicAdd(skip_count + rt, nskip);
    // one partial per (column-word block, row tile), summed in a fixed order by the
    // consumer (reduce_density): a float atomicAdd here made the bound -- and with
    // it which rows are recomputed -- depend on the blocks' arrival order
    if (skip_mass) skip_mass[(size_t)blockIdx.y * row_tiles + rt] = mass * tile_w * 1.001f;
}

}  // namespace fkde_b200
