// prep_kernels.cuh -- O(n*d) kernels around the two O(n^2) passes:
//   column mean (centring), operand scale exponent, operand packing into the
//   swizzled tile image, score finalize (+ SD shift), density reduction, plus
//   the fp64 block-distance kernel behind pairwise_sq_dists_block.
#pragma once
#include <cuda_fp16.h>
#include <cstdint>

#include "layout.cuh"

namespace fkde_b200 {

constexpr double kLog2e = 1.4426950408889634073599246810019;
constexpr double kLn2 = 0.69314718055994530941723212145818;

// ---- fused pass prologue -------------------------------------------------------------------
// One launch instead of colsum_stage1 + colsum_stage2 + max_half_norm + set_scale_exponent
// (+ memsets): per-block column sums (same partition and summation order as
// colsum_stage1, so the mean is deterministic) and per-column min / max; the last
// block to finish (threadfence + counter) reduces the partials in block order into
// mu, bounds max_i |(x_i - mu) k|^2 / 2 by the bounding box (>= the exact maximum,
// so the fp16 operand range stays safe; the scale is a power of two, so a larger
// one costs no precision), sets e / dscale, and clears the per-call counters.
struct PrepArgs {
    const double* x;
    size_t n;
    int d;
    double k;                       // sqrt(log2 e) / h of the pass that packs x (0: no scale)
    PassScalars* sc;                // out: mu, e, dscale, nonfinite (zeroed here first)
    double* part;                   // [grid][3][16] sums, min, max
    unsigned int* done;             // self-resetting completion counter
    unsigned int* clear_u32[4];     // per-call counters to zero (nullptr: unused)
    unsigned long long* clear_max;  // set to ~0 (underflow row), nullptr: unused
    unsigned long long* clear_stats;   // 4 x 0, nullptr: unused
};

__global__ void __launch_bounds__(256) prep_stats(PrepArgs a) {
    pdl_launch_dependents();
    pdl_wait();
    __shared__ double sm[16][17], mn[16][17], mx[16][17];
    __shared__ int s_last;
    const int c = threadIdx.x & 15, g = threadIdx.x >> 4;
    const size_t b0 = a.n * blockIdx.x / gridDim.x, b1 = a.n * (blockIdx.x + 1) / gridDim.x;
    double acc = 0.0, lo = INFINITY, hi = -INFINITY;
    bool bad = false;
    if (c < a.d)
        for (size_t r = b0 + g; r < b1; r += 16) {
            const double v = a.x[r * a.d + c];
            bad |= !isfinite(v);
            acc += v;
            lo = fmin(lo, v);
            hi = fmax(hi, v);
        }
    sm[g][c] = acc;
    mn[g][c] = lo;
    mx[g][c] = hi;
    __syncthreads();
    double* p = a.part + static_cast<size_t>(blockIdx.x) * 48;
    if (threadIdx.x < 16) {
        double s = 0.0, l = INFINITY, h = -INFINITY;
        for (int k = 0; k < 16; ++k) {
            s += sm[k][threadIdx.x];
            l = fmin(l, mn[k][threadIdx.x]);
            h = fmax(h, mx[k][threadIdx.x]);
        }
        p[threadIdx.x] = s;
        p[16 + threadIdx.x] = l;
        p[32 + threadIdx.x] = h;
    }
    const int any_bad = __syncthreads_or(bad ? 1 : 0);
    if (threadIdx.x == 0) {
        if (any_bad) atomicOr(&a.sc->nonfinite, 1u);
        __threadfence();
        s_last = atomicAdd(a.done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    __shared__ double bound[16];
    // the partials reduced by all 256 threads: thread (g, c) folds blocks g, g + 16, ...
    // in order, then thread c folds the 16 group sums in order -- a fixed association,
    // so the mean stays deterministic; a single thread per column walking every block's
    // partial serially was a chain of L2 round trips (~40 us at 256 blocks)
    {
        double s = 0.0, l = INFINITY, h = -INFINITY;
        for (unsigned b = g; b < gridDim.x; b += 16) {
            const double* q = a.part + static_cast<size_t>(b) * 48;
            s += __ldcg(q + c);
            l = fmin(l, __ldcg(q + 16 + c));
            h = fmax(h, __ldcg(q + 32 + c));
        }
        sm[g][c] = s;
        mn[g][c] = l;
        mx[g][c] = h;
    }
    __syncthreads();
    if (threadIdx.x < 16) {
        const int cc = threadIdx.x;
        double s = 0.0, l = INFINITY, h = -INFINITY;
        for (int k = 0; k < 16; ++k) {
            s += sm[k][cc];
            l = fmin(l, mn[k][cc]);
            h = fmax(h, mx[k][cc]);
        }
        const double mu = (cc < a.d) ? s / static_cast<double>(a.n) : 0.0;
        a.sc->mu[cc] = mu;
        const double ext = cc < a.d ? fmax(h - mu, mu - l) : 0.0;
        bound[cc] = ext * ext;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double b = 0.0;
        for (int cc = 0; cc < 16; ++cc) b += bound[cc];
        const double hn = 0.5 * b * a.k * a.k * 1.0000001;
        float hf = !(hn == hn) || hn > 3.0e38 ? 3.0e38f : static_cast<float>(hn);
        a.sc->max_half_norm_bits = __float_as_uint(hf);
        int e = 0;
        while (e < 60 && ldexpf(hf, -2 * e) > 8192.0f) ++e;
        a.sc->e = e;
        a.sc->dscale = ldexpf(1.0f, 2 * e);
        for (int i = 0; i < 4; ++i)
            if (a.clear_u32[i]) *a.clear_u32[i] = 0u;
        if (a.clear_max) *a.clear_max = ~0ull;
        if (a.clear_stats)
            for (int i = 0; i < 4; ++i) a.clear_stats[i] = 0ull;
        *a.done = 0u;   // ready for the next call
    }
}

// Density-pass scale over both point sets (columns: centred or not; queries:
// centred by mu) in one launch, last-block reduction of the exact maxima
// (replaces max_half_norm x 2 + set_scale_exponent + the PassScalars copy).
struct ScaleArgs {
    const double* cols;
    size_t n;
    int cols_centred;
    const double* rows;
    size_t m;
    int d;
    double k;
    const PassScalars* mu_src;   // mean (both sets are centred by it)
    PassScalars* sc;             // out: mu (copied), e, dscale, max_half_norm_bits, nonfinite
    unsigned int* block_max;     // [grid] float bits
    unsigned int* done;
    unsigned int* clear_u32;     // flag counter of the density pass (nullptr: unused)
};

__global__ void __launch_bounds__(256) scale_two(ScaleArgs a) {
    pdl_launch_dependents();
    pdl_wait();
    __shared__ float wmax[8];
    __shared__ int s_last;
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    float hn = 0.f;
    bool bad = false;
    if (i < a.n + a.m) {
        const bool is_col = i < a.n;
        const double* x = is_col ? a.cols + i * a.d : a.rows + (i - a.n) * a.d;
        const bool center = !is_col || !a.cols_centred;
        double s = 0.0;
        for (int c = 0; c < a.d; ++c) {
            const double raw = x[c];
            bad |= !isfinite(raw);
            const double v = (raw - (center ? a.mu_src->mu[c] : 0.0)) * a.k;
            s += v * v;
        }
        hn = static_cast<float>(0.5 * s);
        if (!(hn == hn) || hn > 3.0e38f) hn = 3.0e38f;
    }
    for (int o = 16; o > 0; o >>= 1) hn = fmaxf(hn, __shfl_xor_sync(0xffffffffu, hn, o));
    if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = hn;
    const int any_bad = __syncthreads_or(bad ? 1 : 0);
    if (threadIdx.x == 0) {
        float m = 0.f;
        for (int w = 0; w < 8; ++w) m = fmaxf(m, wmax[w]);
        a.block_max[blockIdx.x] = __float_as_uint(m);
        if (any_bad) atomicOr(&a.sc->nonfinite, 1u);
        __threadfence();
        s_last = atomicAdd(a.done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // every thread of the last block folds a strided slice of the block maxima (a
    // max: any order gives the same bits), then a warp + block max
    float m = 0.f;
    for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x)
        m = fmaxf(m, __uint_as_float(__ldcg(a.block_max + b)));
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    __syncthreads();
    if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x != 0) return;
    m = 0.f;
    for (int w = 0; w < 8; ++w) m = fmaxf(m, wmax[w]);
    for (int c = 0; c < kMaxDim; ++c) a.sc->mu[c] = a.mu_src->mu[c];
    a.sc->max_half_norm_bits = __float_as_uint(m);
    int e = 0;
    while (e < 60 && ldexpf(m, -2 * e) > 8192.0f) ++e;
    a.sc->e = e;
    a.sc->dscale = ldexpf(1.0f, 2 * e);
    if (a.clear_u32) *a.clear_u32 = 0u;
    *a.done = 0u;
}

// ---- operand packing ------------------------------------------------------------
// One thread per operand row (rows_padded threads).  Writes row `out_row0+i`
// of the tile image.  format 0 = A (row side), 1 = B (column side).
struct PackArgs {
    const double* x;         // source points, row-major, d doubles per row
    size_t rows;             // valid rows
    size_t rows_padded;      // multiple of kTileRows
    int d;
    int format;
    int center;              // subtract sc->mu
    double k;                // sqrt(log2 e) / h
    const PassScalars* sc;   // mu (if center) and e
    uint4* out;              // rows_padded * 8 uint4
    float a_offset;          // A rows: constant added to every Gram entry (before the
                             // 2^(2e) scale): chunk-2 element 6 = a_offset * 2^-2e,
                             // paired with a 1 in the B rows (score pass: kPScaleF)
    uint8_t* risk;           // A rows (optional): 1 where |y|^2/2 > risk_half_norm (the
                             // expanded norms' fp32 rounding is too coarse: direct_rows)
    double risk_half_norm;
    const float* cen;        // format 2: per column-tile centroids (log2 units, unscaled)
    int cen_tile;            // format 2: points per column tile
    int ones_mask;           // format 2: tile J's ones column is 16 + (J & ones_mask)
};

__device__ __forceinline__ uint32_t pack_h2(__half a, __half b) {
    return static_cast<uint32_t>(__half_as_ushort(a)) |
           (static_cast<uint32_t>(__half_as_ushort(b)) << 16);
}

__device__ __forceinline__ void pack_row(const PackArgs& a, size_t i);

__global__ void pack_operands(PackArgs a) {
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i < a.rows_padded) pack_row(a, i);
}

// both operands of a pass in one launch: blocks [0, blocks_a) pack a, the rest b
__global__ void pack_two(PackArgs a, PackArgs b, unsigned int blocks_a) {
    pdl_launch_dependents();
    pdl_wait();
    if (blockIdx.x < blocks_a) {
        const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
        if (i < a.rows_padded) pack_row(a, i);
    } else {
        const size_t i = (blockIdx.x - blocks_a) * (size_t)blockDim.x + threadIdx.x;
        if (i < b.rows_padded) pack_row(b, i);
    }
}

// format 2 (B2, score pass on the spatial order): the column operand of GEMM2 only,
// y - c_J with c_J the row's column-tile centroid, so the tensor core accumulates
// sum_j phi_ij (y_j - c_J) -- values of the tile's size, not of |y| -- and the
// drain adds c_J * sum_j phi_ij in float-float (layout.cuh)
__device__ __forceinline__ void pack_row_centred(const PackArgs& a, size_t i) {
    uint32_t ch[8][4];
#pragma unroll
    for (int c = 0; c < 8; ++c)
#pragma unroll
        for (int w = 0; w < 4; ++w) ch[c][w] = 0u;
    if (i < a.rows) {
        const int e = a.sc->e;
        const double ys = ldexp(a.k, -e);
        const float* cj = a.cen + (i / a.cen_tile) * kMaxDim;
        __half vh[kMaxDim], vl[kMaxDim];
#pragma unroll
        for (int c = 0; c < kMaxDim; ++c) {
            double v = 0.0;
            if (c < a.d)
                v = (a.x[i * a.d + c] - a.sc->mu[c]) * ys - ldexp(static_cast<double>(cj[c]), -e);
            vh[c] = __double2half(v);
            vl[c] = __double2half(v - static_cast<double>(__half2float(vh[c])));
        }
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int w = 0; w < 4; ++w) {
                const int k0 = c * 8 + 2 * w;
                ch[c][w] = pack_h2(vh[k0], vh[k0 + 1]);
                ch[4 + c][w] = pack_h2(vl[k0], vl[k0 + 1]);
            }
        // the ones (S_J) in column 16 + (J mod group): chunk 2 + slot/8, word (slot/2) mod 4,
        // half slot%2 (groups of up to 16 tiles: columns 16..31)
        const int slot = static_cast<int>(i / a.cen_tile) & a.ones_mask;
        ch[2 + (slot >> 3)][(slot >> 1) & 3] = (slot & 1) ? pack_h2(__float2half(0.f), __float2half(1.f))
                                      : pack_h2(__float2half(1.f), __float2half(0.f));
    }
    const size_t tile = i / kTileRows;
    const int r = static_cast<int>(i % kTileRows);
    uint4* base = a.out + tile * (kTileBytes / 16) + r * 8;
#pragma unroll
    for (int c = 0; c < 8; ++c) base[c ^ (r & 7)] = make_uint4(ch[c][0], ch[c][1], ch[c][2], ch[c][3]);
}

__device__ __forceinline__ void pack_row(const PackArgs& a, size_t i) {
    if (a.format == 2) {
        pack_row_centred(a, i);
        return;
    }
    __half yh[kMaxDim], yl[kMaxDim];
    __half n1 = __float2half(0.f), n2 = n1, n3 = n1;
    const __half one = __float2half(1.f), zero = __float2half(0.f);
    bool valid = i < a.rows;
    if (valid) {
        const double ys = ldexp(a.k, -a.sc->e);
        double nrm = 0.0;
#pragma unroll
        for (int c = 0; c < kMaxDim; ++c) {
            double y = 0.0;
            if (c < a.d) y = (a.x[i * a.d + c] - (a.center ? a.sc->mu[c] : 0.0)) * ys;
            yh[c] = __double2half(y);
            const double h = static_cast<double>(__half2float(yh[c]));
            yl[c] = __double2half(y - h);
            const double l = static_cast<double>(__half2float(yl[c]));
            nrm += h * h + 2.0 * h * l;  // exactly what the 3-term MMA forms on the diagonal
        }
        const double m = -0.5 * nrm;
        if (a.risk) a.risk[i] = (-m * ldexp(1.0, 2 * a.sc->e) > a.risk_half_norm) ? 1 : 0;
        n1 = __double2half(m);
        const double r1 = m - static_cast<double>(__half2float(n1));
        n2 = __double2half(r1);
        n3 = __double2half(r1 - static_cast<double>(__half2float(n2)));
    } else {
#pragma unroll
        for (int c = 0; c < kMaxDim; ++c) yh[c] = yl[c] = zero;
        if (a.risk && i < a.rows_padded) a.risk[i] = 0;
    }
    // chunk layout (see layout.cuh):      A                 B
    //   0-1  y_hi                          y_hi              y_hi
    //   2    norms                         a1 a2 a3 1 1 1 c  1 1 1 b1 b2 b3 1
    //   3    zero
    //   4-5                                y_hi              y_lo
    //   6-7                                y_lo              y_hi
    uint32_t ch[8][4];
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            const int k0 = c * 8 + 2 * w;
            ch[c][w] = pack_h2(yh[k0], yh[k0 + 1]);
            ch[4 + c][w] = a.format == 0 ? pack_h2(yh[k0], yh[k0 + 1])
                                         : pack_h2(yl[k0], yl[k0 + 1]);
            ch[6 + c][w] = a.format == 0 ? pack_h2(yl[k0], yl[k0 + 1])
                                         : pack_h2(yh[k0], yh[k0 + 1]);
        }
    if (valid) {
        if (a.format == 0) {  // a1 a2 a3 1 1 1 c 0   (c = a_offset * 2^-2e, exact)
            ch[2][0] = pack_h2(n1, n2);
            ch[2][1] = pack_h2(n3, one);
            ch[2][2] = pack_h2(one, one);
            ch[2][3] = pack_h2(__float2half(ldexpf(a.a_offset, -2 * a.sc->e)), zero);
        } else {              // 1 1 1 b1 b2 b3 1 0
            ch[2][0] = pack_h2(one, one);
            ch[2][1] = pack_h2(one, n1);
            ch[2][2] = pack_h2(n2, n3);
            ch[2][3] = pack_h2(one, zero);
        }
    } else {
        if (a.format == 0) {
            ch[2][0] = ch[2][1] = ch[2][2] = ch[2][3] = 0u;
        } else {  // far-away column: b1 + b2 = -60000 -> phi = 0 exactly
            const __half big = __float2half(-30000.f);
            ch[2][0] = 0u;
            ch[2][1] = pack_h2(zero, big);
            ch[2][2] = pack_h2(big, zero);
            ch[2][3] = 0u;
        }
    }
#pragma unroll
    for (int w = 0; w < 4; ++w) ch[3][w] = 0u;
    const size_t tile = i / kTileRows;
    const int r = static_cast<int>(i % kTileRows);
    uint4* base = a.out + tile * (kTileBytes / 16) + r * 8;
#pragma unroll
    for (int c = 0; c < 8; ++c) base[c ^ (r & 7)] = make_uint4(ch[c][0], ch[c][1], ch[c][2], ch[c][3]);
}

// ---- score finalize ----------------------------------------------------------------
// engine.cpp:322-337 (s = (T - x S) / (h^2 S), ScoreUnderflowError when S == 0)
// and the SD shift engine.cpp:396-399 (x + h^2/2 s).  Local shard row i is
// global row g = row0 + i; every output is indexed by g (in-place allgather
// layout).  part_s: [splits][rows_pad]; part_t: [splits][rows_pad][16] with
// T' = sum_j phi_ij y'_j in scaled, centred coordinates.
struct FinalizeArgs {
    const double* part_s;
    const double* part_t;
    int splits;
    size_t rows_pad;
    size_t rows;          // rows in this shard
    size_t row0;          // global index of shard row 0
    int d;
    const double* x;      // full training set (fp64, original coordinates)
    const PassScalars* sc;
    double k;             // sqrt(log2 e)/h_score
    double h_score;
    double shift;         // h^2/2
    double* score;        // [n][d] or nullptr
    double* xsd_c;        // [n][d] centred debiased samples or nullptr
    double* phi_sum;      // [n] raw S or nullptr
    double* weighted;     // [n][d] raw sum_j phi_ij x_j or nullptr
    unsigned long long* underflow_row;  // atomicMin of failing global row
    unsigned int* flag_count;           // rows handed to direct_rows_kernel
    unsigned int* flag_rows;            // (local indices)
    const uint8_t* risk;                // pack's spread flags (local rows) or nullptr
};

// One thread per (row, coordinate): consecutive threads read consecutive
// doubles of the [split][row][16] partials and write consecutive score /
// x^SD entries (a thread per row strided every access by 128 B).
__global__ void finalize_score(FinalizeArgs a) {
    pdl_launch_dependents();
    pdl_wait();
    const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    const size_t i = t / static_cast<size_t>(a.d);
    const int c = static_cast<int>(t % static_cast<size_t>(a.d));
    if (i >= a.rows) return;
    // S' and T' exclude the self pair (phi_ii = exp(0) = 1, engine.cpp:43-50
    // snaps r_ii^2 to 0): S = 1 + S', and T - x_i S = T' - x_i S'.
    double Sp = 0.0;
#pragma unroll 4
    for (int s = 0; s < a.splits; ++s) Sp += a.part_s[s * a.rows_pad + i];
    Sp = ldexp(Sp, -kPScaleExp);  // the tc/simt score sums carry phi * 2^15
    // too little neighbour mass for fp16 P, or too much spread for the expansion
    if (a.flag_rows && (Sp < kScoreFlagMass || (a.risk && a.risk[i]))) {
        if (c == 0) a.flag_rows[atomicAdd(a.flag_count, 1u)] = static_cast<unsigned int>(i);
        return;
    }
    const double S = 1.0 + Sp;
    const double ys = ldexp(a.k, -a.sc->e);
    const size_t g = a.row0 + i;
    if (a.phi_sum && c == 0) a.phi_sum[g] = S;
    if (!(S > 0.0) || !isfinite(S)) {
        if (c == 0) atomicMin(a.underflow_row, static_cast<unsigned long long>(g));
        return;
    }
    const double inv = 1.0 / (a.h_score * a.h_score * S);
    double Tp = 0.0;
#pragma unroll 4
    for (int s = 0; s < a.splits; ++s) Tp += a.part_t[(s * a.rows_pad + i) * kMaxDim + c];
    const double tc = ldexp(Tp, -kPScaleExp) / ys;  // sum_{j != i} phi_ij xc_j
    const double x = a.x[g * a.d + c];
    const double xc = x - a.sc->mu[c];
    const double sc = (tc - xc * Sp) * inv;         // (T - x S) / (h^2 S)
    if (a.score) a.score[g * a.d + c] = sc;
    if (a.xsd_c) a.xsd_c[g * a.d + c] = xc + a.shift * sc;
    if (a.weighted) a.weighted[g * a.d + c] = (tc + xc) + S * a.sc->mu[c];
}

// debiased samples in original coordinates: x_sd = x_sd_c + mu
__global__ void add_mean(const double* __restrict__ xc, size_t n, int d,
                         const PassScalars* __restrict__ sc, double* __restrict__ out) {
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i >= n * d) return;
    out[i] = xc[i] + sc->mu[i % d];
}

// ---- density reduction ----------------------------------------------------------------
// out[j] (+)= scale * (ca * sum_p part0[p][j] + cb * sum_p part1[p][j])
struct ReduceArgs {
    const float* part0;
    const float* part1;   // may be nullptr
    int nparts;
    size_t rows_pad;
    size_t rows;
    double ca, cb, scale;
    int accumulate;
    double* out;
    unsigned int* flag_count;   // rows whose Gaussian mass underflows fp32 ranges
    unsigned int* flag_rows;
    const uint8_t* risk;        // pack's spread flags (local rows) or nullptr
    // density tile skipping (nullptr: none): per 128-row tile, the bound on the
    // term mass one row loses to the skipped tiles (tile_predict); a row whose term
    // mass |ca| s0 + |cb| |s1| (the scale of the fp32 sums' own rounding of the row)
    // is below 2^24 times that bound is flagged
    const float* skip_mass;
    int mass_parts;          // skip_mass holds [mass_parts][mass_stride] partials
    size_t mass_stride;
};

__global__ void reduce_density(ReduceArgs a) {
    pdl_launch_dependents();
    pdl_wait();
    const size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (j >= a.rows) return;
    double s0 = 0.0, s1 = 0.0;
    for (int p = 0; p < a.nparts; ++p) s0 += static_cast<double>(a.part0[p * a.rows_pad + j]);
    if (a.part1)
        for (int p = 0; p < a.nparts; ++p) s1 += static_cast<double>(a.part1[p * a.rows_pad + j]);
    bool skipped_mass = false;
    if (a.skip_mass) {   // (all lanes of a warp read the same row tile's partials: broadcast)
        float mass = 0.f;
        for (int p = 0; p < a.mass_parts; ++p) mass += a.skip_mass[p * a.mass_stride + j / kTileRows];
        skipped_mass = fabs(a.ca) * s0 + fabs(a.cb * s1) < 0x1p24 * static_cast<double>(mass);
    }
    if (a.flag_rows && (s0 < kDensityFlagMass || (a.risk && a.risk[j]) || skipped_mass)) {
        a.flag_rows[atomicAdd(a.flag_count, 1u)] = static_cast<unsigned int>(j);
        return;
    }
    const double v = a.scale * (a.ca * s0 + a.cb * s1);
    a.out[j] = a.accumulate ? a.out[j] + v : v;
}

// ---- public block distances (engine.cpp:41-51 / 261-277 semantics, fp64) ---------------
__global__ void sq_norms_fp64(const double* __restrict__ x, size_t rows, int d,
                              double* __restrict__ out) {
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i >= rows) return;
    double s = 0.0;
    for (int c = 0; c < d; ++c) s += x[i * d + c] * x[i * d + c];
    out[i] = s;
}

__global__ void block_sq_dists_fp64(const double* __restrict__ a, const double* __restrict__ an,
                                    size_t na, const double* __restrict__ b,
                                    const double* __restrict__ bn, size_t nb, int d,
                                    double* __restrict__ out) {
    const size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (j >= nb) return;
    for (size_t i = blockIdx.y; i < na; i += gridDim.y) {
        double g = 0.0;
        for (int c = 0; c < d; ++c) g = fma(a[i * d + c], b[j * d + c], g);
        const double base = bn[j] + an[i];
        const double v = base - 2.0 * g;
        out[i * nb + j] = (v < 16.0 * 2.220446049250313e-16 * base) ? 0.0 : v;
    }
}

}  // namespace fkde_b200
