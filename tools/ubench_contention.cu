// Does tcgen05.ld/st traffic from epilogue warps slow down concurrent
// tcgen05.mma (TS: A from TMEM, and SS)?  Warp 0 issues MMAs; warps 2..9
// optionally stream tcgen05.ld / tcgen05.st over other TMEM columns.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o ubench_contention ubench_contention.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2602_10378_b200/csrc/ptx.cuh"

using namespace fkde_b200;

template <int TS, int N, int BG>
__global__ void __launch_bounds__(320, 1) bench(int iters, unsigned long long* out, float* sink) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    __shared__ volatile int stop;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) {
        ptx::mbar_init(&bar, 1);
        ptx::fence_barrier_init();
        stop = 0;
    }
    if (warp == 0) ptx::tmem_alloc<512>(&tslot);
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tb = tslot;
    float acc = 0.f;
    if (warp == 0) {
        const uint32_t sA = ptx::smem_u32(smem), sB = sA + 32768;
        constexpr uint32_t idesc = ptx::idesc_f16_f32(128, N, false, TS ? true : false);
        uint64_t da[4], db[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            da[k] = ptx::smem_desc_sw128(sA + k * 32, 16, 1024);
            db[k] = TS ? ptx::smem_desc_sw128(sB + k * 2048, 16384, 1024)
                       : ptx::smem_desc_sw128(sB + k * 32, 16, 1024);
        }
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            if (ptx::elect_one()) {
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    if (TS)
                        ptx::umma_f16_ts(tb + 384, tb + (k & 3) * 8, db[k & 3], idesc, 1u);
                    else
                        ptx::umma_f16(tb + 384, da[k & 3], db[k & 3], idesc, 1u);
                }
            }
            __syncwarp();
        }
        if (ptx::elect_one()) ptx::umma_commit(&bar);
        __syncwarp();
        ptx::mbar_wait(&bar, 0);
        long long t1 = clock64();
        if (lane == 0) {
            out[blockIdx.x] = t1 - t0;
            stop = 1;
        }
    } else if (warp >= 2 && BG) {
        const int q = warp & 3, hf = (warp - 2) >> 2;
        const uint32_t base = tb + ((uint32_t)(q * 32) << 16) + 128 + hf * 64;  // cols 128..255
        uint32_t r[32], s2[32];
        for (int i = 0; i < 32; ++i) r[i] = i;
        while (!stop) {
            ptx::tmem_ld32(base, r);
            ptx::tmem_ld32(base + 32, s2);
            ptx::tmem_ld_wait();
            uint32_t x = 0;
#pragma unroll
            for (int i = 0; i < 32; ++i) x ^= r[i] ^ s2[i];
            acc += __uint_as_float(x);
            if (BG == 2) {
                ptx::tmem_st32(base + 128, r);       // cols 256..383
                ptx::tmem_st32(base + 160, s2);
                ptx::tmem_st_wait();
            }
        }
    }
    sink[blockIdx.x * 320 + threadIdx.x] = acc;
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<512>(tb);
    }
}

template <int TS, int N, int BG>
void run(unsigned long long* d, float* sink) {
    const int iters = 64;
    cudaFuncSetAttribute(bench<TS, N, BG>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    bench<TS, N, BG><<<148, 320, 65536>>>(iters, d, sink);
    bench<TS, N, BG><<<148, 320, 65536>>>(iters, d, sink);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148;
    const char* bg[] = {"idle", "LDTM", "LDTM+STTM"};
    printf("%s N=%3d with background %-10s: %6.1f cycles/MMA (%s)\n", TS ? "TS" : "SS", N, bg[BG],
           avg / (iters * 8.0), cudaGetErrorString(e));
}

int main() {
    unsigned long long* d;
    float* sink;
    cudaMalloc(&d, 8 * 148);
    cudaMalloc(&sink, 148 * 320 * 4);
    run<1, 48, 0>(d, sink);
    run<1, 48, 1>(d, sink);
    run<1, 48, 2>(d, sink);
    run<0, 128, 0>(d, sink);
    run<0, 128, 1>(d, sink);
    run<0, 128, 2>(d, sink);
    run<0, 48, 0>(d, sink);
    run<0, 48, 2>(d, sink);
    return 0;
}
