// Microbenchmarks for the score-pass design decisions (run on the B200 box):
//   - tcgen05.mma throughput for the shapes the pairwise kernels issue
//     (SS vs TS operand sources, N = 48 / 128 / 256, one vs several
//     independent accumulators)
//   - tcgen05.ld / tcgen05.st throughput (TMEM <-> registers)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o ubench ubench_tc.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2602_10378_b200/csrc/ptx.cuh"

using namespace fkde_b200;

__global__ void __launch_bounds__(256, 1) mma_bench(int mode, int n_mma, int N, int chains,
                                                    unsigned long long* out, int warp_issue) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x / 32;
    // zero operands (values irrelevant for timing)
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
    if (threadIdx.x == 0) {
        ptx::mbar_init(&bar, 1);
        ptx::fence_barrier_init();
    }
    if (warp == 0) ptx::tmem_alloc<512>(&tslot);
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tb = tslot;
    if (warp_issue ? warp == 0 : threadIdx.x == 0) {
        const bool leader = warp_issue ? ptx::elect_one() : true;
        const uint32_t sA = ptx::smem_u32(smem), sB = sA + 32768;
        const uint32_t idesc = ptx::idesc_f16_f32(128, N, false, mode >= 2);
        long long t0 = clock64();
        for (int i = 0; i < n_mma; ++i) {
            const int c = i % chains;
            const uint32_t d = tb + 256 + c * (N > 64 ? 0 : 48);   // chains: separate D regions (N<=48)
            const uint32_t dd = N > 64 ? ((mode == 1 || chains == 1) ? tb + 256 : tb + (c & 1) * 256) : d;
            if (mode == 0 || mode == 2) {   // SS; mode 2 = B MN-major
                const uint64_t da = ptx::smem_desc_sw128(sA + (i & 3) * 32, 16, 1024);
                const uint64_t db = mode == 0 ? ptx::smem_desc_sw128(sB + (i & 3) * 32, 16, 1024)
                                              : ptx::smem_desc_sw128(sB + (i & 7) * 2048, 16384, 1024);
                if (leader) ptx::umma_f16(dd, da, db, idesc, i >= chains ? 1u : 0u);
                if (warp_issue) __syncwarp();
            } else {                          // TS: A from TMEM cols [0,128); B MN-major
                const uint64_t db = ptx::smem_desc_sw128(sB + (i & 7) * 2048, 16384, 1024);
                if (leader) ptx::umma_f16_ts(dd, tb + (i & 15) * 8, db, idesc, i >= chains ? 1u : 0u);
                if (warp_issue) __syncwarp();
            }
        }
        if (leader) ptx::umma_commit(&bar);
        ptx::mbar_wait(&bar, 0);
        long long t1 = clock64();
        if (leader) out[blockIdx.x] = t1 - t0;
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<512>(tb);
    }
}

__global__ void __launch_bounds__(256, 1) tmem_bench(int mode, int iters, unsigned long long* out,
                                                     float* sink) {
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x / 32;
    if (warp == 0) ptx::tmem_alloc<512>(&tslot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tb = tslot + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 64;
    uint32_t r[32];
    for (int i = 0; i < 32; ++i) r[i] = i;
    float acc = 0.f;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (mode == 0) {
            ptx::tmem_ld32(tb + (it & 1) * 128, r);
            ptx::tmem_ld_wait();
            acc += __uint_as_float(r[it & 31]);
        } else {
            ptx::tmem_st32(tb + (it & 1) * 128, r);
            ptx::tmem_st_wait();
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    sink[threadIdx.x] = acc;
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<512>(tslot);
    }
}

int main() {
    unsigned long long* d;
    float* sink;
    cudaMalloc(&d, 8 * 148);
    cudaMalloc(&sink, 4096);
    cudaFuncSetAttribute(mma_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    const char* mname[] = {"SS K-major B", "TS (A tmem)", "SS MN-major B"};
    int modes[] = {0, 1, 2};
    for (int mi = 0; mi < 3; ++mi) {
        int mode = modes[mi] == 1 ? 1 : (modes[mi] == 2 ? 2 : 0);
        for (int N : {48, 128, 256})
        for (int wi : {0, 1}) {
            for (int chains : {1, 2}) {
                if (mode == 1 && N > 128) continue;
                const int n = 512;
                mma_bench<<<148, 128, 65536>>>(mode, n, N, chains, d, wi);
                mma_bench<<<148, 128, 65536>>>(mode, n, N, chains, d, wi);
                cudaError_t e = cudaDeviceSynchronize();
                unsigned long long h[148];
                cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
                double avg = 0;
                for (int i = 0; i < 148; ++i) avg += h[i];
                avg /= 148;
                printf("mma %-14s %s M=128 N=%3d K=16 chains=%d: %7.1f cycles/MMA  (math floor %5.1f)  %s\n",
                       mname[mi], wi ? "warp+elect" : "lane0     ", N, chains, avg / n, 128.0 * N / 256.0, cudaGetErrorString(e));
            }
        }
    }
    for (int mode = 0; mode < 2; ++mode) {
        for (int warps : {4, 8}) {
            const int iters = 4096;
            tmem_bench<<<148, warps * 32>>>(mode, iters, d, sink);
            tmem_bench<<<148, warps * 32>>>(mode, iters, d, sink);
            cudaError_t e = cudaDeviceSynchronize();
            unsigned long long h[148];
            cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
            double avg = 0;
            for (int i = 0; i < 148; ++i) avg += h[i];
            avg /= 148;
            const double bytes = (double)iters * warps * 32 * 32 * 4;
            printf("tmem %s 32x32b.x32, %d warps: %.1f B/clk/SM (%s)\n", mode ? "st" : "ld", warps,
                   bytes / avg, cudaGetErrorString(e));
        }
    }
    return 0;
}
