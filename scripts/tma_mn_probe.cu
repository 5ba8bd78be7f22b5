// Probe (not product code): can TMA write the MN-major tf32 operand layout
// tcgen05 needs (SWIZZLE_128B_BASE32B: 4-row K atoms of 128 B, 32-byte chunks
// XOR the row, MN atoms 4096 B apart, K groups 512 B apart)?  A is stored in
// global memory MN-contiguous (A_g[k][m], the transpose-free view of a
// row-major activation for a weight-gradient GEMM); a 3-D tensor map
// (32 MN, 32 K, MN/32) with a given swizzle mode loads a 128 x 32 tile in one
// TMA; one MMA chain D = A^T B against a host product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o scripts/tma_mn_probe scripts/tma_mn_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                                  const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_mn(uint32_t addr) {
    uint64_t d = 0;
    d |= (addr >> 4) & 0x3FFFull;
    d |= (uint64_t)(4096 >> 4) << 16;
    d |= (uint64_t)(512 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)1 << 61;  // SWIZZLE_128B_BASE32B
    return d;
}
__host__ __device__ constexpr uint32_t idesc(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__global__ void probe(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, float* D) {
    extern __shared__ __align__(1024) unsigned char raw[];
    unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    unsigned char* sa = sm;           // 128 MN x 32 K = 16 KB
    unsigned char* sb = sm + 16384;   // 64 MN x 32 K = 8 KB
    __shared__ uint64_t bar, mbar;
    __shared__ uint32_t slot;
    const int t = threadIdx.x;
    if (t < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(su32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = slot;
    if (t == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&mbar)), "r"(16384 + 8192) : "memory");
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                     ::"r"(su32(sa)), "l"(&ta), "r"(0), "r"(0), "r"(0), "r"(su32(&mbar)) : "memory");
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                     ::"r"(su32(sb)), "l"(&tb), "r"(0), "r"(0), "r"(0), "r"(su32(&mbar)) : "memory");
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0;\n\tselp.u32 %0, 1, 0, P;\n}"
                         : "=r"(ok) : "r"(su32(&mbar)) : "memory");
        asm volatile("tcgen05.fence::after_thread_sync;");
        for (int j = 0; j < 4; ++j) {  // K step j: 8 K rows = 2 atoms of 4 rows, 1024 B further
            const uint64_t ad = desc_mn(su32(sa) + j * 1024), bd = desc_mn(su32(sb) + j * 1024);
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
                         "l"(ad), "l"(bd), "r"(idesc(128, 64)), "r"(j > 0 ? 1u : 0u));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    }
    uint32_t done = 0;
    while (!done)
        asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0;\n\tselp.u32 %0, 1, 0, P;\n}"
                     : "=r"(done) : "r"(su32(&bar)) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int w = t / 32, lane = t % 32;
    if (w < 4)
        for (int c = 0; c < 64; ++c) {
            uint32_t r;
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(tmem + ((uint32_t)(w * 32) << 16) + c));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            D[(w * 32 + lane) * 64 + c] = __uint_as_float(r);
        }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
}

int main() {
    const int M = 128, N = 64, Kk = 32, ldA = M + 32, ldB = N + 32;  // padded rows: the tile is a window of a wider matrix
    std::vector<float> A(Kk * ldA), B(Kk * ldB), D(M * N), R(M * N, 0.f);
    srand(3);
    for (auto& x : A) x = (float)(rand() % 7 - 3);
    for (auto& x : B) x = (float)(rand() % 5 - 2);
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
            double s = 0;
            for (int k = 0; k < Kk; ++k) s += (double)A[k * ldA + m] * B[k * ldB + n];
            R[m * N + n] = (float)s;
        }
    float *dA, *dB, *dD;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB, B.size() * 4);
    cudaMalloc(&dD, D.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    EncodeTiledFn enc = (EncodeTiledFn)f;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    const CUtensorMapSwizzle modes[3] = {CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_SWIZZLE_128B,
                                         CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B_FLIP_8B};
    const char* names[3] = {"128B_ATOM_32B", "128B", "128B_ATOM_32B_FLIP_8B"};
    for (int mi = 0; mi < 3; ++mi) {
        alignas(64) CUtensorMap ta, tb;
        cuuint64_t da[3] = {32, (cuuint64_t)Kk, (cuuint64_t)(M / 32)}, sa_[2] = {(cuuint64_t)ldA * 4, 128};
        cuuint64_t db[3] = {32, (cuuint64_t)Kk, (cuuint64_t)(N / 32)}, sb_[2] = {(cuuint64_t)ldB * 4, 128};
        cuuint32_t ba[3] = {32, 32, (cuuint32_t)(M / 32)}, bb[3] = {32, 32, (cuuint32_t)(N / 32)}, es[3] = {1, 1, 1};
        CUresult r1 = enc(&ta, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, dA, da, sa_, ba, es, CU_TENSOR_MAP_INTERLEAVE_NONE, modes[mi],
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        CUresult r2 = enc(&tb, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, dB, db, sb_, bb, es, CU_TENSOR_MAP_INTERLEAVE_NONE, modes[mi],
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r1 || r2) {
            printf("%-22s encode failed (%d, %d)\n", names[mi], (int)r1, (int)r2);
            continue;
        }
        cudaMemset(dD, 0, D.size() * 4);
        probe<<<1, 128, 64 * 1024>>>(ta, tb, dD);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int i = 0; i < M * N; ++i) bad += D[i] != R[i];
        printf("%-22s %s: %d / %d mismatches (%s)\n", names[mi], bad ? "NO " : "YES", bad, M * N, cudaGetErrorString(e));
    }
    return 0;
}
