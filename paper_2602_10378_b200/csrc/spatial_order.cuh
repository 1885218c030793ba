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
//   tile_centroids  per-tile centroid in log2 units (the skip predictor's input)
#pragma once
#include <cstdint>

#include "layout.cuh"

namespace fkde_b200 {

constexpr int kOrderAxes = 3;
constexpr int kMortonBits = 10;     // per axis -> 30-bit keys

struct OrderScalars {
    double axis[kOrderAxes][kMaxDim];   // unit principal axes
    double inv_scale[kOrderAxes];       // 1 / (4 sqrt(lambda_k)): projections -> ~[-1, 1]
};

// ---- covariance partials: block b sums (x - mu)(x - mu)^T over its row range ------------
__global__ void __launch_bounds__(256) cov_stage1(const double* __restrict__ x, size_t n, int d,
                                                  const PassScalars* __restrict__ sc,
                                                  double* __restrict__ part /* [grid][256] */) {
    __shared__ double rows[64][kMaxDim];
    const int a = threadIdx.x >> 4, b = threadIdx.x & 15;
    const size_t r0 = n * blockIdx.x / gridDim.x, r1 = n * (blockIdx.x + 1) / gridDim.x;
    double acc = 0.0;
    for (size_t base = r0; base < r1; base += 64) {
        const int nr = static_cast<int>(r1 - base < 64 ? r1 - base : 64);
        __syncthreads();
        for (int e = threadIdx.x; e < 64 * kMaxDim; e += 256) {
            const int r = e / kMaxDim, c = e % kMaxDim;
            rows[r][c] = (r < nr && c < d) ? x[(base + r) * d + c] - sc->mu[c] : 0.0;
        }
        __syncthreads();
        for (int r = 0; r < nr; ++r) acc = fma(rows[r][a], rows[r][b], acc);
    }
    part[blockIdx.x * 256 + threadIdx.x] = acc;
}

// ---- covariance -> top principal axes (one block of 256 threads) -----------------------
__global__ void __launch_bounds__(256) order_axes(const double* __restrict__ part, int nparts,
                                                  int d, OrderScalars* __restrict__ os) {
    __shared__ double C[kMaxDim][kMaxDim];
    __shared__ double Q[kMaxDim][kOrderAxes], Z[kMaxDim][kOrderAxes];
    const int t = threadIdx.x;
    {
        double s = 0.0;
        for (int p = 0; p < nparts; ++p) s += part[p * 256 + t];
        C[t >> 4][t & 15] = s;
    }
    if (t < kMaxDim * kOrderAxes) {   // start from the coordinate axes of largest variance order
        const int r = t / kOrderAxes, k = t % kOrderAxes;
        Q[r][k] = (r == k) ? 1.0 : 0.0;
    }
    __syncthreads();
    // subspace (orthogonal) iteration: Q <- orth(C Q); the top-3 eigengap of
    // clustered data is large, and for unclustered data any basis of the top
    // subspace orders equally well
    for (int it = 0; it < 48; ++it) {
        if (t < kMaxDim * kOrderAxes) {
            const int r = t / kOrderAxes, k = t % kOrderAxes;
            double s = 0.0;
            for (int c = 0; c < kMaxDim; ++c) s = fma(C[r][c], Q[c][k], s);
            Z[r][k] = s;
        }
        __syncthreads();
        if (t == 0) {   // modified Gram-Schmidt (3 vectors of 16)
            for (int k = 0; k < kOrderAxes; ++k) {
                for (int j = 0; j < k; ++j) {
                    double dp = 0.0;
                    for (int r = 0; r < kMaxDim; ++r) dp += Z[r][k] * Z[r][j];
                    for (int r = 0; r < kMaxDim; ++r) Z[r][k] -= dp * Z[r][j];
                }
                double nn = 0.0;
                for (int r = 0; r < kMaxDim; ++r) nn += Z[r][k] * Z[r][k];
                if (nn > 1e-300) {
                    const double inv = 1.0 / sqrt(nn);
                    for (int r = 0; r < kMaxDim; ++r) Z[r][k] *= inv;
                } else {   // degenerate (d < 3 or a zero-variance subspace): a spare coordinate axis
                    for (int r = 0; r < kMaxDim; ++r) Z[r][k] = (r == k) ? 1.0 : 0.0;
                    for (int j = 0; j < k; ++j) {
                        double dp = 0.0;
                        for (int r = 0; r < kMaxDim; ++r) dp += Z[r][k] * Z[r][j];
                        for (int r = 0; r < kMaxDim; ++r) Z[r][k] -= dp * Z[r][j];
                    }
                    nn = 0.0;
                    for (int r = 0; r < kMaxDim; ++r) nn += Z[r][k] * Z[r][k];
                    const double inv = nn > 1e-300 ? 1.0 / sqrt(nn) : 0.0;
                    for (int r = 0; r < kMaxDim; ++r) Z[r][k] *= inv;
                }
            }
        }
        __syncthreads();
        if (t < kMaxDim * kOrderAxes) Q[t / kOrderAxes][t % kOrderAxes] = Z[t / kOrderAxes][t % kOrderAxes];
        __syncthreads();
    }
    if (t < kOrderAxes) {
        const int k = t;
        // deterministic sign: largest-magnitude component positive
        int am = 0;
        for (int r = 1; r < kMaxDim; ++r)
            if (fabs(Q[r][k]) > fabs(Q[am][k])) am = r;
        const double sg = Q[am][k] < 0.0 ? -1.0 : 1.0;
        double lam = 0.0;
        for (int r = 0; r < kMaxDim; ++r) {
            double cq = 0.0;
            for (int c = 0; c < kMaxDim; ++c) cq += C[r][c] * Q[c][k];
            lam += Q[r][k] * cq;
        }
        for (int r = 0; r < kMaxDim; ++r) os->axis[k][r] = (r < d) ? sg * Q[r][k] : 0.0;
        // covariance is a sum over n points, so lam / n is the variance (n folded
        // into the scale by the caller's mean-free projection: use the ratio only)
        os->inv_scale[k] = lam > 0.0 ? 1.0 / (4.0 * sqrt(lam)) : 0.0;
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
    keys[i] = key;
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

// centroid (log2 units: (x - mu) * sqrt(log2 e) / h) of each tile of `tile_w` rows of
// x (rows beyond n are padding and ignored); one block of 128 threads per tile
__global__ void __launch_bounds__(128) tile_centroids(const double* __restrict__ x, size_t n, int d,
                                                      const PassScalars* __restrict__ sc, double k,
                                                      int tile_w, float* __restrict__ out) {
    __shared__ double part[8][kMaxDim];
    const size_t r0 = static_cast<size_t>(blockIdx.x) * tile_w;
    const size_t r1 = r0 + tile_w < n ? r0 + tile_w : n;
    const int c = threadIdx.x & 15, g = threadIdx.x >> 4;
    double s = 0.0;
    if (c < d)
        for (size_t r = r0 + g; r < r1; r += 8) s += x[r * d + c] - sc->mu[c];
    part[g][c] = s;
    __syncthreads();
    if (threadIdx.x < kMaxDim) {
        double t = 0.0;
        for (int q = 0; q < 8; ++q) t += part[q][threadIdx.x];
        const double cnt = r1 > r0 ? static_cast<double>(r1 - r0) : 1.0;
        out[static_cast<size_t>(blockIdx.x) * kMaxDim + threadIdx.x] =
            r1 > r0 ? static_cast<float>(t / cnt * k) : 1e18f;
    }
}

// Skip predictor: one thread per (row tile, 32 column tiles): bit ct of the
// row's mask words = centroid half-distance^2 > thresh (log2 units).  The bit
// only selects the tile pair for the exact check (kModeCheck); pred and skip
// masks start equal, the check clears skip bits of tiles that contribute.
__global__ void tile_predict(const float* __restrict__ cenA, int row_tiles,
                             const float* __restrict__ cenB, int col_tiles, int words, float thresh,
                             uint32_t* __restrict__ pred, uint32_t* __restrict__ skip) {
    pdl_launch_dependents();
    pdl_wait();
    const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (t >= static_cast<size_t>(row_tiles) * words) return;
    const int rt = static_cast<int>(t / words), w = static_cast<int>(t % words);
    float a[kMaxDim];
#pragma unroll
    for (int c = 0; c < kMaxDim; ++c) a[c] = cenA[(size_t)rt * kMaxDim + c];
    uint32_t bits = 0;
    for (int b = 0; b < 32; ++b) {
        const int ct = w * 32 + b;
        if (ct >= col_tiles) break;
        float dd = 0.f;
#pragma unroll
        for (int c = 0; c < kMaxDim; ++c) {
            const float df = a[c] - cenB[(size_t)ct * kMaxDim + c];
            dd = fmaf(df, df, dd);
        }
        if (0.5f * dd > thresh) bits |= 1u << b;
    }
    pred[t] = bits;
    skip[t] = bits;
}

}  // namespace fkde_b200
