// ubench_mbar.cu -- latency of mbarrier probes on an already completed phase
// (try_wait / test_wait, one warp), and of a dependent chain of two probes vs
// two independent ones.   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_mbar tools/ubench_mbar.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void k(long long* out) {
    __shared__ uint64_t bar[2];
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[1])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&bar[0])) : "memory");
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&bar[1])) : "memory");
    }
    __syncthreads();
    const int N = 1000;
    uint32_t acc = 0;
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) {
        uint32_t ok;
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(su(&bar[(i + acc) & 1])) : "memory");
        acc += ok;
    }
    long long t1 = clock64();
    for (int i = 0; i < N; ++i) {
        uint32_t ok;
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(su(&bar[(i + acc) & 1])) : "memory");
        acc += ok;
    }
    long long t2 = clock64();
    for (int i = 0; i < N; ++i) {   // ld.shared round trip for comparison
        uint32_t v;
        asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v) : "r"(su(&bar[(i + acc) & 1])) : "memory");
        acc += v & 1;
    }
    long long t3 = clock64();
    if (threadIdx.x == 0) {
        out[0] = (t1 - t0) / N;
        out[1] = (t2 - t1) / N;
        out[2] = (t3 - t2) / N;
        out[3] = acc;
    }
}

int main() {
    long long* d;
    cudaMalloc(&d, 4 * sizeof(long long));
    k<<<1, 32>>>(d);
    long long h[4];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("completed-phase probe latency (cycles, dependent chain): try_wait %lld  test_wait %lld  ld.shared %lld\n",
           h[0], h[1], h[2]);
    return 0;
}
