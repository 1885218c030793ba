// Epilogue instruction-mix microbenchmark (B200): elements per clock per SM of
// the score / KDE epilogue arithmetic on register data (no TMEM, no barriers),
// to separate the instruction mix's own throughput from pipeline stalls.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/ubench_pipe tools/ubench_pipe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2602_10378_b200/csrc/ptx.cuh"

using namespace fkde_b200;

// outputs are folded into 4 independent XOR accumulators: one 3-input LOP3
// per pair of output words (the real kernel hands them to tcgen05.st instead)
#define KEEP2(a, b) (acc[w & 3] ^= (a) ^ (b))

template <int MODE>
__global__ void mix(int iters, float seed, uint32_t* sink, unsigned long long* cyc) {
    float v[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) v[c] = -0.001f * (threadIdx.x + c) + seed;
    float2 facc[4] = {};
    uint32_t acc[4] = {0, 0, 0, 0};
    const float2 off2 = make_float2(15.f, 15.f), neg1 = make_float2(-1.f, -1.f);
    float sc = 1.0f;
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        sc += 1e-7f;                       // new inputs every iteration (no hoisting)
        const float2 dsc2 = make_float2(sc, sc);
#pragma unroll
        for (int w = 0; w < 16; ++w) {
            const float2 t = ptx::ffma2(make_float2(v[2 * w], v[2 * w + 1]), dsc2, off2);
            if constexpr (MODE == 0) {          // MUFU only
                KEEP2(__float_as_uint(ptx::ex2(t.x)), __float_as_uint(ptx::ex2(t.y)));
            } else if constexpr (MODE == 1) {   // score epilogue mix
                const float2 p = make_float2(ptx::ex2(t.x), ptx::ex2(t.y));
                const float2 h = make_float2(__uint_as_float(__float_as_uint(p.x) & 0xFFFFE000u),
                                             __uint_as_float(__float_as_uint(p.y) & 0xFFFFE000u));
                const float2 l = ptx::ffma2(h, neg1, p);
                KEEP2(ptx::cvt_f16x2(h.x, h.y), ptx::cvt_f16x2(l.x, l.y));
            } else if constexpr (MODE == 2) {   // score mix without the f16 converts
                const float2 p = make_float2(ptx::ex2(t.x), ptx::ex2(t.y));
                const float2 h = make_float2(__uint_as_float(__float_as_uint(p.x) & 0xFFFFE000u),
                                             __uint_as_float(__float_as_uint(p.y) & 0xFFFFE000u));
                const float2 l = ptx::ffma2(h, neg1, p);
                KEEP2(__float_as_uint(h.x), __float_as_uint(h.y));
                KEEP2(__float_as_uint(l.x), __float_as_uint(l.y));
            } else if constexpr (MODE == 3) {   // ex2 + two converts
                const float2 p = make_float2(ptx::ex2(t.x), ptx::ex2(t.y));
                KEEP2(ptx::cvt_f16x2(p.x, p.y), ptx::cvt_f16x2(p.y, p.x));
            } else if constexpr (MODE == 4) {   // KDE mix
                const float2 p = make_float2(ptx::ex2(t.x), ptx::ex2(t.y));
                facc[w & 3] = ptx::fadd2(facc[w & 3], p);
            } else if constexpr (MODE == 5) {   // converts only (no MUFU)
                KEEP2(ptx::cvt_f16x2(t.x, t.y), ptx::cvt_f16x2(t.y, t.x));
            } else if constexpr (MODE == 6) {   // LOP3 mask only
                KEEP2(__float_as_uint(t.x) & 0xFFFFE000u, __float_as_uint(t.y) & 0xFFFFE000u);
            } else if constexpr (MODE == 7) {   // score mix, one F2FP per pair via bf16x2 hi + f16x2 lo
                const float2 p = make_float2(ptx::ex2(t.x), ptx::ex2(t.y));
                const float2 h = make_float2(__uint_as_float(__float_as_uint(p.x) & 0xFFFFE000u),
                                             __uint_as_float(__float_as_uint(p.y) & 0xFFFFE000u));
                const float2 l = ptx::ffma2(h, neg1, p);
                KEEP2(__byte_perm(__float_as_uint(h.x), __float_as_uint(h.y), 0x7632), ptx::cvt_f16x2(l.x, l.y));
            }
        }
    }
    const unsigned long long t1 = clock64();
    if (facc[0].x + facc[1].x + facc[2].x + facc[3].y == 1.2345f || (acc[0] ^ acc[1] ^ acc[2] ^ acc[3]) == 0x9e3779b9u) sink[threadIdx.x] = 1;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, int warps) {
    const int iters = 2000;
    uint32_t* sink;
    unsigned long long* cyc;
    cudaMalloc(&sink, 4096 * 4);
    cudaMalloc(&cyc, 148 * 8);
    mix<MODE><<<148, warps * 32>>>(10, -1.f, sink, cyc);
    mix<MODE><<<148, warps * 32>>>(iters, -1.f, sink, cyc);
    cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    const double elems = (double)iters * 32 * 32 * warps;
    printf("%-22s warps/SM %2d: %6.2f elem/clk/SM (%.1f%% of 16/clk)\n", name, warps, elems / mx,
           elems / mx / 16 * 100);
    cudaFree(sink);
    cudaFree(cyc);
}


// the score epilogue with its TMEM traffic: per 96-column tile 3 chunks of
// (tcgen05.ld 32 cols -> wait -> math -> 2 x tcgen05.st 16 cols), st wait per tile;
// warp w uses lane quadrant w % 4 and its own 96 columns (w / 4)
template <int PIPE>
__global__ void tmem_mix(int iters, uint32_t* sink, unsigned long long* cyc) {
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x / 32;
    if (warp == 0) ptx::tmem_alloc<512>(&tslot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tb = tslot + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 96;
    const float2 off2 = make_float2(15.f, 15.f), neg1 = make_float2(-1.f, -1.f);
    const float2 dsc2 = make_float2(1.0001f, 1.0001f);
    {   // initialise S with small negative numbers
        uint32_t z[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) z[i] = __float_as_uint(-0.01f * (i + 1));
        for (int c = 0; c < 96; c += 16) ptx::tmem_st16(tb + c, z);
        ptx::tmem_st_wait();
    }
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll 1
        for (int ch = 0; ch < 3; ++ch) {
            uint32_t v[32];
            ptx::tmem_ld32(tb + ch * 32, v);
            ptx::tmem_ld_wait();
            uint32_t hi_w[16], lo_w[16];
#pragma unroll
            for (int w = 0; w < 16; ++w) {
                const float2 t = ptx::ffma2(make_float2(__uint_as_float(v[2 * w]), __uint_as_float(v[2 * w + 1])), dsc2, off2);
                const float2 p = make_float2(ptx::ex2(t.x), ptx::ex2(t.y));
                const float2 h = make_float2(__uint_as_float(__float_as_uint(p.x) & 0xFFFFE000u),
                                             __uint_as_float(__float_as_uint(p.y) & 0xFFFFE000u));
                const float2 l = ptx::ffma2(h, neg1, p);
                hi_w[w] = ptx::cvt_f16x2(h.x, h.y) & 0xBFFFBFFFu;   // keep S negative
                lo_w[w] = ptx::cvt_f16x2(l.x, l.y);
            }
            if constexpr (PIPE == 0) {
                ptx::tmem_st16(tb + ch * 32, hi_w);
                ptx::tmem_st16(tb + ch * 32 + 16, lo_w);
            } else {
                uint32_t a = 0;
#pragma unroll
                for (int w = 0; w < 16; ++w) a ^= hi_w[w] ^ lo_w[w];
                if (a == 0x9e3779b9u) sink[threadIdx.x] = a;
            }
        }
        ptx::tmem_st_wait();
    }
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<512>(tslot);
    }
}

template <int PIPE>
void run_tmem(const char* name, int warps) {
    const int iters = 600;
    uint32_t* sink;
    unsigned long long* cyc;
    cudaMalloc(&sink, 4096 * 4);
    cudaMalloc(&cyc, 148 * 8);
    tmem_mix<PIPE><<<148, warps * 32>>>(5, sink, cyc);
    tmem_mix<PIPE><<<148, warps * 32>>>(iters, sink, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); exit(1); }
    unsigned long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    const double elems = (double)iters * 96 * 32 * warps;
    printf("%-22s warps/SM %2d: %6.2f elem/clk/SM (%.1f%% of 16/clk)\n", name, warps, elems / mx,
           elems / mx / 16 * 100);
    cudaFree(sink);
    cudaFree(cyc);
}

// software-pipelined variant: 16-column sub-chunks, the load of sub-chunk k+1
// is in flight while sub-chunk k is computed (P: 8 hi + 8 lo columns per 16)
__global__ void tmem_mix_pipe(int iters, uint32_t* sink, unsigned long long* cyc) {
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x / 32;
    if (warp == 0) ptx::tmem_alloc<512>(&tslot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tb = tslot + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 96;
    const float2 off2 = make_float2(15.f, 15.f), neg1 = make_float2(-1.f, -1.f);
    const float2 dsc2 = make_float2(1.0001f, 1.0001f);
    {
        uint32_t z[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) z[i] = __float_as_uint(-0.01f * (i + 1));
        for (int c = 0; c < 96; c += 16) ptx::tmem_st16(tb + c, z);
        ptx::tmem_st_wait();
    }
    __syncthreads();
    auto comp = [&](uint32_t (&v)[16], uint32_t col) {
        uint32_t hi_w[8], lo_w[8];
#pragma unroll
        for (int w = 0; w < 8; ++w) {
            const float2 t = ptx::ffma2(make_float2(__uint_as_float(v[2 * w]), __uint_as_float(v[2 * w + 1])), dsc2, off2);
            const float2 p = make_float2(ptx::ex2(t.x), ptx::ex2(t.y));
            const float2 h = make_float2(__uint_as_float(__float_as_uint(p.x) & 0xFFFFE000u),
                                         __uint_as_float(__float_as_uint(p.y) & 0xFFFFE000u));
            const float2 l = ptx::ffma2(h, neg1, p);
            hi_w[w] = ptx::cvt_f16x2(h.x, h.y) & 0xBFFFBFFFu;
            lo_w[w] = ptx::cvt_f16x2(l.x, l.y);
        }
        ptx::tmem_st8(col, hi_w);
        ptx::tmem_st8(col + 8, lo_w);
    };
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        uint32_t va[16], vb[16];
        ptx::tmem_ld16(tb, va);
        ptx::tmem_ld_wait_tie(va);
#pragma unroll
        for (int k = 0; k < 6; k += 2) {
            ptx::tmem_ld16(tb + (k + 1) * 16, vb);
            comp(va, tb + k * 16);
            ptx::tmem_ld_wait_tie(vb);
            if (k + 2 < 6) ptx::tmem_ld16(tb + (k + 2) * 16, va);
            comp(vb, tb + (k + 1) * 16);
            if (k + 2 < 6) ptx::tmem_ld_wait_tie(va);
        }
        ptx::tmem_st_wait();
    }
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<512>(tslot);
    }
}

void run_tmem_pipe(const char* name, int warps) {
    const int iters = 600;
    uint32_t* sink;
    unsigned long long* cyc;
    cudaMalloc(&sink, 4096 * 4);
    cudaMalloc(&cyc, 148 * 8);
    tmem_mix_pipe<<<148, warps * 32>>>(5, sink, cyc);
    tmem_mix_pipe<<<148, warps * 32>>>(iters, sink, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); exit(1); }
    unsigned long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    const double elems = (double)iters * 96 * 32 * warps;
    printf("%-22s warps/SM %2d: %6.2f elem/clk/SM (%.1f%% of 16/clk)\n", name, warps, elems / mx,
           elems / mx / 16 * 100);
    cudaFree(sink);
    cudaFree(cyc);
}

// tmem_mix with a concurrent tensor-core stream: warp 0 issues, per "tile",
// 4 SS MMAs M=128 N=96 (GEMM1-like, into TMEM cols 288..383) then 12 TS MMAs
// N=48 reading A from those columns (GEMM2-like, into cols 384..431), commits,
// waits, idles `gap` cycles; warps 4..15 run the score epilogue's TMEM
// ld -> math -> st pattern on cols 0..287.  Does tensor traffic slow the epilogue?
__global__ void __launch_bounds__(512, 1) tmem_mix_mma(int iters, int mma_on, int gap, uint32_t* sink,
                                                      unsigned long long* cyc) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    __shared__ int done;     // epilogue warps finished
    const int warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) {
        ptx::mbar_init(&bar, 1);
        ptx::fence_barrier_init();
        done = 0;
    }
    if (warp == 0) ptx::tmem_alloc<512>(&tslot);
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tb0 = tslot;
    if (warp == 0) {
        if (mma_on) {
            const uint32_t sA = ptx::smem_u32(smem), sB = sA + 32768;
            constexpr uint32_t id1 = ptx::idesc_f16_f32(128, 96, false, false);
            constexpr uint32_t id2 = ptx::idesc_f16_f32(128, 48, false, true);
            uint32_t ph = 0;
            while (*(volatile int*)&done < 12) {
                if (ptx::elect_one()) {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        ptx::umma_f16(tb0 + 288, ptx::smem_desc_sw128(sA + k * 32, 16, 1024),
                                      ptx::smem_desc_sw128(sB + k * 32, 16, 1024), id1, k ? 1u : 0u);
#pragma unroll
                    for (int k = 0; k < 12; ++k)
                        ptx::umma_f16_ts(tb0 + 384, tb0 + 288 + k * 8, ptx::smem_desc_sw128(sB + (k & 3) * 2048, 16384, 1024),
                                         id2, 1u);
                    ptx::umma_commit(&bar);
                }
                __syncwarp();
                ptx::mbar_wait(&bar, ph);
                ph ^= 1;
                const long long t = clock64();
                while (clock64() - t < gap) {
                }
            }
        }
    } else if (warp >= 4) {
        const uint32_t tb = tb0 + ((uint32_t)((warp & 3) * 32) << 16) + ((warp - 4) >> 2) * 96;
        const float2 off2 = make_float2(15.f, 15.f), neg1 = make_float2(-1.f, -1.f);
        const float2 dsc2 = make_float2(1.0001f, 1.0001f);
        {
            uint32_t z[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) z[i] = __float_as_uint(-0.01f * (i + 1));
            for (int c = 0; c < 96; c += 16) ptx::tmem_st16(tb + c, z);
            ptx::tmem_st_wait();
        }
        const unsigned long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll 1
            for (int ch = 0; ch < 3; ++ch) {
                uint32_t v[32];
                ptx::tmem_ld32(tb + ch * 32, v);
                ptx::tmem_ld_wait();
                uint32_t hi_w[16], lo_w[16];
#pragma unroll
                for (int w = 0; w < 16; ++w) {
                    const float2 t = ptx::ffma2(make_float2(__uint_as_float(v[2 * w]), __uint_as_float(v[2 * w + 1])), dsc2, off2);
                    const float2 p = make_float2(ptx::ex2(t.x), ptx::ex2(t.y));
                    const float2 h = make_float2(__uint_as_float(__float_as_uint(p.x) & 0xFFFFE000u),
                                                 __uint_as_float(__float_as_uint(p.y) & 0xFFFFE000u));
                    const float2 l = ptx::ffma2(h, neg1, p);
                    hi_w[w] = ptx::cvt_f16x2(h.x, h.y) & 0xBFFFBFFFu;
                    lo_w[w] = ptx::cvt_f16x2(l.x, l.y);
                }
                ptx::tmem_st16(tb + ch * 32, hi_w);
                ptx::tmem_st16(tb + ch * 32 + 16, lo_w);
            }
            ptx::tmem_st_wait();
        }
        const unsigned long long t1 = clock64();
        if ((threadIdx.x & 31) == 0) {
            cyc[blockIdx.x * 16 + warp] = t1 - t0;
            atomicAdd(&done, 1);
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<512>(tb0);
    }
    if (threadIdx.x == 1000) sink[0] = 0;
}

void run_tmem_mma(int mma_on, int gap) {
    const int iters = 600;
    uint32_t* sink;
    unsigned long long* cyc;
    cudaMalloc(&sink, 4096 * 4);
    cudaMalloc(&cyc, 148 * 16 * 8);
    cudaFuncSetAttribute(tmem_mix_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    tmem_mix_mma<<<148, 512, 65536>>>(5, mma_on, gap, sink, cyc);
    tmem_mix_mma<<<148, 512, 65536>>>(iters, mma_on, gap, sink, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("tmem_mma: %s\n", cudaGetErrorString(e)); exit(1); }
    unsigned long long h[148 * 16];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int b = 0; b < 148; ++b)
        for (int w = 4; w < 16; ++w) mx = h[b * 16 + w] > mx ? h[b * 16 + w] : mx;
    const double elems = (double)iters * 96 * 32 * 12;
    printf("tmem ld+math+st, 12 warps, MMA stream %s (gap %4d): %6.2f elem/clk/SM (%.1f%% of 16/clk)\n",
           mma_on ? "on " : "off", gap, elems / mx, elems / mx / 16 * 100);
    fflush(stdout);
    cudaFree(sink);
    cudaFree(cyc);
}

int main() {
    run_tmem_mma(0, 0);
    run_tmem_mma(1, 0);
    run_tmem_mma(1, 300);
    run_tmem_mma(1, 800);
    return 0;
    for (int w : {8, 12, 16}) {
        run_tmem<0>("tmem ld+math+st", w);
        run_tmem<1>("tmem ld+math", w);
        run_tmem_pipe("tmem pipelined 16", w);
    }
    return 0;
    for (int w : {4, 8, 12, 16}) {
        run<0>("ex2 only", w);
        run<1>("score mix", w);
        run<2>("score mix, no cvt", w);
        run<3>("ex2 + 2 cvt", w);
        run<4>("kde mix", w);
        run<5>("2 cvt only", w);
        run<6>("2 lop3 only", w);
        run<7>("score mix, prmt hi", w);
    }
    return 0;
}
