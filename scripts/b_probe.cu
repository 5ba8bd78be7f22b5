// Ceiling probe for config B's access pattern (not product code): how fast a
// plain hand-written kernel moves read 2 x 256 MiB + write 256 MiB (+ row sums)
// on this B200, to calibrate the fused VM kernel's roofline fraction.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/b_probe scripts/b_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) chain(const float4* __restrict__ a, const float4* __restrict__ b,
                                             const float4* __restrict__ c, float4* __restrict__ t3,
                                             float* __restrict__ rs, int rows, int cols4) {
    // one warp per row, 8 float4 per lane per iteration (cols = 1024 -> 256 float4 -> one pass)
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    for (int r = warp; r < rows; r += nwarps) {
        const float4* ar = a + (size_t)r * cols4;
        const float4* br = b + (size_t)r * cols4;
        float4* tr = t3 + (size_t)r * cols4;
        float s = 0.f;
        float4 av[8], bv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            av[u] = __ldcs(ar + lane + 32 * u);
            bv[u] = __ldcs(br + lane + 32 * u);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const float4 cv = __ldg(c + lane + 32 * u);
            float4 t;
            t.x = fmaxf(av[u].x + cv.x, 0.f) * bv[u].x;
            t.y = fmaxf(av[u].y + cv.y, 0.f) * bv[u].y;
            t.z = fmaxf(av[u].z + cv.z, 0.f) * bv[u].z;
            t.w = fmaxf(av[u].w + cv.w, 0.f) * bv[u].w;
            __stcs(tr + lane + 32 * u, t);
            s += (t.x + t.y) + (t.z + t.w);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) rs[r] = s;
    }
}

int main() {
    const int rows = 65536, cols = 1024, cols4 = cols / 4;
    float4 *a, *b, *c, *t;
    float* rs;
    cudaMalloc(&a, (size_t)rows * cols * 4);
    cudaMalloc(&b, (size_t)rows * cols * 4);
    cudaMalloc(&c, cols * 4);
    cudaMalloc(&t, (size_t)rows * cols * 4);
    cudaMalloc(&rs, rows * 4);
    cudaMemset(a, 0, (size_t)rows * cols * 4);
    cudaMemset(b, 0, (size_t)rows * cols * 4);
    const double bytes = 3.0 * rows * cols * 4 + cols * 4 + rows * 4;
    for (int blocks : {148 * 4, 148 * 8, 148 * 16, 148 * 32}) {
        for (int i = 0; i < 3; ++i) chain<<<blocks, 256>>>(a, b, c, t, rs, rows, cols4);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        const int reps = 50;
        for (int i = 0; i < reps; ++i) chain<<<blocks, 256>>>(a, b, c, t, rs, rows, cols4);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("blocks %5d: %.1f us  %.0f GB/s (%s)\n", blocks, 1e3 * ms / reps, bytes / (ms / reps * 1e-3) / 1e9,
               cudaGetErrorString(cudaGetLastError()));
    }
    // plain copy for reference
    for (int i = 0; i < 3; ++i) cudaMemcpyAsync(t, a, (size_t)rows * cols * 4, cudaMemcpyDeviceToDevice);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int i = 0; i < 20; ++i) cudaMemcpyAsync(t, a, (size_t)rows * cols * 4, cudaMemcpyDeviceToDevice);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("cudaMemcpy D2D 256 MiB: %.0f GB/s (read+write)\n", 2.0 * rows * cols * 4 / (ms / 20 * 1e-3) / 1e9);
    return 0;
}
