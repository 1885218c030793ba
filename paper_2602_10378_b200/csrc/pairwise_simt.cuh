// pairwise_simt.cuh -- CUDA-core validation engine for the same passes.
//
// Independent of the tensor-core path's Gram expansion: reconstructs the
// scaled coordinates y = y_hi + y_lo from the operand rows and forms
// r'^2 = sum_k (y_i,k - y_j,k)^2 by direct subtraction in fp32 (the
// oracle's formulation, oracle.cpp:25-32).  Selected with
// FKDE_OPT_ENGINE = FKDE_ENGINE_SIMT; used by the GPU tests as a second,
// structurally different device implementation next to the fp64 oracle.
// Writes the same partial layout as pairwise_tc_kernel with splits = 1.
#pragma once
#include <cuda_fp16.h>
#include <cstdint>

#include "layout.cuh"
#include "pairwise_tc.cuh"

namespace fkde_b200 {

__device__ __forceinline__ void unpack_y(const uint8_t* tiles, size_t row, bool a_format,
                                         float* y) {
    const size_t tile = row / kTileRows;
    const int r = static_cast<int>(row % kTileRows);
    const uint4* base = reinterpret_cast<const uint4*>(tiles + tile * kTileBytes + r * kRowBytes);
    __align__(16) __half hi[16];
    __align__(16) __half lo[16];
    const int lo_chunk = a_format ? 6 : 4;
    for (int c = 0; c < 2; ++c) {
        reinterpret_cast<uint4*>(hi)[c] = base[c ^ (r & 7)];
        reinterpret_cast<uint4*>(lo)[c] = base[(lo_chunk + c) ^ (r & 7)];
    }
    for (int k = 0; k < 16; ++k) y[k] = __half2float(hi[k]) + __half2float(lo[k]);
}

template <int MODE>
__global__ void __launch_bounds__(128) pairwise_simt_kernel(PairArgs args, size_t n_cols) {
    // score pass: global column index of this row (self pair excluded, see PairArgs)
    const long long diag_col = (MODE == kModeScore && args.diag_row0 >= 0)
                                   ? args.diag_row0 + blockIdx.x * 128ll + threadIdx.x
                                   : -1;
    __shared__ float cols[128][17];
    const size_t row = blockIdx.x * 128ull + threadIdx.x;
    float yi[16];
    unpack_y(args.opA, row, true, yi);
    const float dsc = args.sc->dscale;
    float s0 = 0.f, s1 = 0.f, t[16];
    for (int k = 0; k < 16; ++k) t[k] = 0.f;
    for (int ct = 0; ct < args.n_col_tiles; ++ct) {
        __syncthreads();
        float yj[16];
        unpack_y(args.opB, ct * 128ull + threadIdx.x, false, yj);
        for (int k = 0; k < 16; ++k) cols[threadIdx.x][k] = yj[k];
        __syncthreads();
        const int nvalid = static_cast<int>(n_cols - ct * 128ull < 128ull ? n_cols - ct * 128ull : 128ull);
        for (int j = 0; j < nvalid; ++j) {
            float r2 = 0.f;
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const float df = yi[k] - cols[j][k];
                r2 = fmaf(df, df, r2);
            }
            const float dd = fminf(-0.5f * r2 * dsc, 0.f);
            // score sums carry the same 2^kPScaleExp factor as the tc path
            const float p = (ct * 128ll + j == diag_col)
                                ? 0.f
                                : ptx::ex2(MODE == kModeScore ? dd + kPScaleF : dd);
            s0 += p;
            if constexpr (MODE == kModeLaplace) s1 = fmaf(p, dd, s1);
            if constexpr (MODE == kModeScore) {
#pragma unroll
                for (int k = 0; k < 16; ++k) t[k] = fmaf(p, cols[j][k], t[k]);
            }
        }
    }
    if constexpr (MODE == kModeScore) {
        args.dpart0[row] = s0;
        for (int k = 0; k < 16; ++k) args.dpart1[row * kMaxDim + k] = t[k];
    } else {
        args.part0[row] = s0;
        args.part0[args.rows_pad + row] = 0.f;  // second column half (tc layout) is empty
        if constexpr (MODE == kModeLaplace) {
            args.part1[row] = s1;
            args.part1[args.rows_pad + row] = 0.f;
        }
    }
}

}  // namespace fkde_b200
