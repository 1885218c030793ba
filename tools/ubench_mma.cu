// tcgen05.mma throughput microbenchmark: cycles per instruction for the
// shapes the pairwise kernels issue.  Descriptors are loop-invariant and the
// issue loop is unrolled so the number measures the tensor core, not issue.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o ubench_mma ubench_mma.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2602_10378_b200/csrc/ptx.cuh"

using namespace fkde_b200;

template <int M, int N, int TS, int CHAINS>
__global__ void __launch_bounds__(128, 1) bench(int iters, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
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
    if (warp == 0) {
        const uint32_t sA = ptx::smem_u32(smem), sB = sA + 32768;
        constexpr uint32_t idesc = ptx::idesc_f16_f32(M, N, false, TS ? true : false);
        uint64_t da[4], db[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            da[k] = ptx::smem_desc_sw128(sA + k * 32, 16, 1024);
            db[k] = TS ? ptx::smem_desc_sw128(sB + k * 2048, 16384, 1024)
                       : ptx::smem_desc_sw128(sB + k * 32, 16, 1024);
        }
        const uint32_t dcol = TS ? 256u : 0u;
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            if (ptx::elect_one()) {
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const uint32_t d = tb + dcol + (k % CHAINS) * (N <= 64 ? 64u : 0u);
                    if (TS)
                        ptx::umma_f16_ts(d, tb + (k & 3) * 8, db[k & 3], idesc, 1u);
                    else
                        ptx::umma_f16(d, da[k & 3], db[k & 3], idesc, 1u);
                }
            }
            __syncwarp();
        }
        if (ptx::elect_one()) ptx::umma_commit(&bar);
        __syncwarp();
        ptx::mbar_wait(&bar, 0);
        long long t1 = clock64();
        if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<512>(tb);
    }
}

template <int M, int N, int TS, int CHAINS>
void run(unsigned long long* d, int iters) {
    cudaFuncSetAttribute(bench<M, N, TS, CHAINS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    bench<M, N, TS, CHAINS><<<148, 128, 65536>>>(iters, d);
    bench<M, N, TS, CHAINS><<<148, 128, 65536>>>(iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148;
    const double per = avg / (iters * 8.0);
    printf("%s M=%3d N=%3d K=16 chains=%d iters=%4d: %7.1f cyc/MMA  -> %6.0f MAC/clk/SM  %s\n",
           TS ? "TS" : "SS", M, N, CHAINS, iters, per, M * N * 16.0 / per, cudaGetErrorString(e));
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 8 * 148);
    for (int iters : {8, 64}) {
        run<128, 256, 0, 1>(d, iters);
        run<128, 128, 0, 1>(d, iters);
        run<128, 64, 0, 1>(d, iters);
        run<128, 48, 0, 1>(d, iters);
        run<128, 48, 0, 4>(d, iters);
        run<128, 16, 0, 1>(d, iters);
        run<64, 128, 0, 1>(d, iters);
        run<128, 128, 1, 1>(d, iters);
        run<128, 48, 1, 1>(d, iters);
        run<128, 48, 1, 4>(d, iters);
    }
    return 0;
}
