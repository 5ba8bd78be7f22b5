// Grid-size sweep of config B's generated ROW kernel (not product code): the
// kernel `jit.py` emits for config B (v0), the same with its row loop unrolled
// (v1) and with __launch_bounds__(256, 6) (v2), each timed back to back at
// several grid sizes.  Build and run: scripts/b_sweep.sh.
#include "ew_ops.cuh"
#include <cstdio>
#include <vector>
using namespace gfb;
__device__ __forceinline__ uint32_t mod_of(uint32_t q, uint32_t mul, uint32_t sh, uint32_t m) { return q - fast_div(q, mul, sh) * m; }
#define GFB_LD(p) __ldg(p)
#define GFB_LOADV(p, x) loadV<T, V>((p), (x))
#include "v0.inc"
#include "v1.inc"
#include "v2.inc"
typedef void (*KF)(const gfb_ew_args);
int main() {
  const size_t rows = 65536, cols = 1024, n = rows * cols;
  float *a, *b, *c, *t, *rs; void** tab;
  cudaMalloc(&a, n * 4); cudaMalloc(&b, n * 4); cudaMalloc(&c, cols * 4); cudaMalloc(&t, n * 4); cudaMalloc(&rs, rows * 4);
  // non-zero data
  std::vector<float> h(n); for (size_t i = 0; i < n; ++i) h[i] = (float)((i * 2654435761u) % 2001) / 1000.f - 1.f;
  cudaMemcpy(a, h.data(), n * 4, cudaMemcpyHostToDevice); cudaMemcpy(b, h.data() + 7, (n - 7) * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(c, h.data(), cols * 4, cudaMemcpyHostToDevice);
  void* ht[8] = {0, 0, a, b, c, t, rs, 0};
  cudaMalloc(&tab, sizeof(ht)); cudaMemcpy(tab, ht, sizeof(ht), cudaMemcpyHostToDevice);
  gfb_ew_args pa; memset(&pa, 0, sizeof(pa)); pa.tab = (const void* const*)tab;
  const double bytes = 3.0 * n * 4 + cols * 4 + rows * 4;
  KF ks[3] = {k_v0, k_v1, k_v2}; const char* nm[3] = {"gen", "unroll", "lb6"};
  for (int kv = 0; kv < 3; ++kv)
  for (int blocks : {592, 740, 888, 1184, 1480, 2368, 4736, 8192}) {
    for (int i = 0; i < 5; ++i) ks[kv]<<<blocks, 256>>>(pa);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int reps = 200; cudaEventRecord(e0);
    for (int i = 0; i < reps; ++i) ks[kv]<<<blocks, 256>>>(pa);
    cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-7s blocks %5d: %.1f us %.0f GB/s (%s)\n", nm[kv], blocks, 1e3 * ms / reps, bytes / (ms / reps * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
