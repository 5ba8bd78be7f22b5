// Microbenchmark: tcgen05.mma kind::tf32 issue throughput vs N and vs the
// number of independent TMEM accumulators (one CTA per SM, operands resident
// in shared memory, no loads).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_probe scripts/mma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(const void* p) {
    uint64_t d = (su32(p) >> 4) & 0x3FFF;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}
template <int KIND>  // 0 tf32, 1 f16 (bf16), 2 i8 (s8 x s8 -> s32)
__host__ __device__ constexpr uint32_t idesc(int M, int N) {
    return KIND == 0   ? ((1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24))
           : KIND == 1 ? ((1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24))
                       : ((2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24));
}

template <int N, int NACC, int KIND>
__global__ void __launch_bounds__(128, 1) probe(int iters, unsigned long long* out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char* s = (unsigned char*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar;
    for (int i = threadIdx.x; i < (128 + 256) * 128 / 4; i += blockDim.x) ((float*)s)[i] = 0.001f * (i % 7);
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = slot;
    unsigned long long t0 = 0, t1 = 0;
    if (threadIdx.x == 0) {
        const uint64_t a = desc(s), b = desc(s + 128 * 128);
        constexpr uint32_t id = idesc<KIND>(128, N);
        t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int j = 0; j < 12; ++j) {
                const uint32_t d = tmem + (uint32_t)((j % NACC) * N);
                const uint64_t adv = (uint64_t)((j & 3) * 32) >> 4;
                if (KIND == 0)
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d), "l"(a + adv), "l"(b + adv), "r"(id));
                else if (KIND == 2)
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(d), "l"(a + adv), "l"(b + adv), "r"(id));
                else
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d), "l"(a + adv), "l"(b + adv), "r"(id));
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
        uint32_t done = 0;
        while (!done)
            asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0;\n\tselp.u32 %0, 1, 0, P;\n}" : "=r"(done) : "r"(su32(&bar)) : "memory");
        t1 = clock64();
        if (blockIdx.x == 0) out[0] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

static int g_iters = 2000;

template <int N, int NACC, int KIND>
void run(const char* name) {
    unsigned long long* d;
    cudaMalloc(&d, 8);
    int smem = (128 + 256) * 128 + 1024;
    cudaFuncSetAttribute(probe<N, NACC, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = g_iters;
    probe<N, NACC, KIND><<<148, 128, smem>>>(iters, d);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    probe<N, NACC, KIND><<<148, 128, smem>>>(iters, d);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long cyc;
    cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
    const double mmas = 12.0 * iters;
    const double k = KIND == 0 ? 8 : KIND == 1 ? 16 : 32;
    const double flops = mmas * 2.0 * 128 * N * k * 148;
    printf("%-6s N=%3d acc=%d iters=%6d: %7.1f cyc/mma  %8.1f TFLOP/s  %6.0f MHz  %.2f ms  (%s)\n",
           KIND == 0 ? "tf32" : KIND == 1 ? "bf16" : "i8", N, NACC, iters, cyc / mmas, flops / (ms * 1e-3) / 1e12,
           cyc / (ms * 1e3), ms, cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

int main(int argc, char** argv) {
    if (argc > 1) g_iters = atoi(argv[1]);
    run<64, 1, 0>("");
    run<64, 3, 0>("");
    run<128, 1, 0>("");
    run<128, 3, 0>("");
    run<256, 1, 0>("");
    run<256, 2, 0>("");
    run<128, 1, 1>("");
    run<256, 1, 1>("");
    run<128, 1, 2>("");
    run<256, 1, 2>("");
    run<256, 2, 2>("");
    // sustained (seconds-long, under the power cap): tf32 N=256, the 3xTF32 GEMM's shape
    g_iters *= 200;
    run<256, 2, 0>("");
    run<256, 2, 1>("");
    run<256, 2, 2>("");
    return 0;
}
