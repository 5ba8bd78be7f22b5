// Probe (not product code): tcgen05.mma kind::tf32 with MN-major A and B in
// SWIZZLE_128B shared memory.  A is 128 x 32 (M x K), B is 64 x 32 (N x K);
// atoms of 32 MN elements (128 B) x 8 K rows, swizzled 16-byte chunks
// (chunk ^ row), MN atoms LBO = 4096 B apart, K groups SBO = 1024 B apart.
// D = A B^T accumulated over four K = 8 steps, read back from TMEM and
// compared with a host product.  Values are small integers (exact in TF32).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o scripts/mn_probe scripts/mn_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cmath>
#include <cstring>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc_mn(const void* p, uint32_t lbo, uint32_t sbo, uint32_t layout = 2) {
    uint64_t d = 0;
    d |= (su32(p) >> 4) & 0x3FFFull;
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)layout << 61;  // 2: SWIZZLE_128B, 1: SWIZZLE_128B_BASE32B
    return d;
}

__host__ __device__ constexpr uint32_t idesc(int M, int N, int amaj, int bmaj) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)amaj << 15) | ((uint32_t)bmaj << 16) |
           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// byte offset of element (mn, k) of an MN-major SWIZZLE_128B_BASE32B tile
// (the only MN-major smem layout for tf32): atoms of 4 K rows x 128 B (32 MN
// elements), 32-byte chunks XOR-swizzled with the row; variant 0: K groups
// at ks = 512, MN atoms at ms = 4096; variant 1: MN atoms at 512, K groups
// at 2048; variant 2: the K-major SW128 control
__host__ __device__ inline uint32_t mn_off(int mn, int k, int var) {
    if (var == 2) return (mn / 8) * 1024 + (mn % 8) * 128 + ((((k / 4) ^ (mn % 8))) << 4) + (k % 4) * 4;
    const uint32_t ms = var == 0 ? 4096 : 512, ks = var == 0 ? 512 : 2048;
    const int mb = mn / 32, m_in = mn % 32, kg = k / 4, kin = k % 4;
    return mb * ms + kg * ks + kin * 128 + (((m_in / 8) ^ kin) << 5) + (m_in % 8) * 4;
}

__global__ void probe(const float* A, const float* B, float* D, int var) {
    extern __shared__ __align__(1024) unsigned char raw[];
    unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    unsigned char* sa = sm;          // 4 MN atoms x 4 K groups = 16 KB
    unsigned char* sb = sm + 32768;  // B (at most 16 KB span)
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int t = threadIdx.x;
    for (int i = t; i < 128 * 32; i += blockDim.x) {
        const int m = i / 32, k = i % 32;
        *reinterpret_cast<float*>(sa + mn_off(m, k, var)) = A[m * 32 + k];
    }
    for (int i = t; i < 64 * 32; i += blockDim.x) {
        const int n = i / 32, k = i % 32;
        *reinterpret_cast<float*>(sb + mn_off(n, k, var)) = B[n * 32 + k];
    }
    if (t < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(su32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (t == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = slot;
    if (t == 0) {
        for (int j = 0; j < 4; ++j) {
            uint64_t ad, bd;
            uint32_t id;
            if (var == 2) {  // K-major control: SBO 1024, advance 32 B per K step
                ad = desc_mn(sa, 16, 1024) + (uint64_t)((j * 32) >> 4);
                bd = desc_mn(sb, 16, 1024) + (uint64_t)((j * 32) >> 4);
                id = idesc(128, 64, 0, 0);
            } else {
                const uint32_t ms = var == 0 ? 4096 : 512, ks = var == 0 ? 512 : 2048;
                ad = desc_mn(sa + j * 2 * ks, ms, ks, 1);
                bd = desc_mn(sb + j * 2 * ks, ms, ks, 1);
                id = idesc(128, 64, 1, 1);
            }
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
                "l"(ad), "l"(bd), "r"(id), "r"(j > 0 ? 1u : 0u));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    }
    uint32_t done = 0;
    while (!done)
        asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0;\n\tselp.u32 %0, 1, 0, P;\n}"
                     : "=r"(done) : "r"(su32(&bar)) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int w = t / 32, lane = t % 32;
    if (w < 4) {
        for (int c = 0; c < 64; ++c) {
            uint32_t r;
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(tmem + ((uint32_t)(w * 32) << 16) + c));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            D[(w * 32 + lane) * 64 + c] = __uint_as_float(r);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
}

// MMA throughput: `iters` x 4 K steps of M=128 N=n on one CTA, clock64 timed
template <int N>
__global__ void mma_rate(int var, int iters, long long* cycles) {
    extern __shared__ __align__(1024) unsigned char raw[];
    unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int t = threadIdx.x;
    for (int i = t; i < 65536 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
    if (t < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (t == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = slot;
    if (t == 0) {
        const long long c0 = clock64();
        for (int it = 0; it < iters; ++it)
            for (int j = 0; j < 4; ++j) {
                uint64_t ad, bd;
                uint32_t id;
                if (var == 2) {
                    ad = desc_mn(sm, 16, 1024) + (uint64_t)((j * 32) >> 4);
                    bd = desc_mn(sm + 32768, 16, 1024) + (uint64_t)((j * 32) >> 4);
                    id = idesc(128, N, 0, 0);
                } else {
                    ad = desc_mn(sm + j * 1024, 4096, 512, 1);
                    bd = desc_mn(sm + 32768 + j * 1024, 4096, 512, 1);
                    id = idesc(128, N, var == 0 ? 1 : 0, 1);  // var 0: both MN-major, var 1: only B MN-major
                }
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
                    "l"(ad), "l"(bd), "r"(id), "r"(1u));
            }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
        uint32_t done = 0;
        while (!done)
            asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0;\n\tselp.u32 %0, 1, 0, P;\n}"
                         : "=r"(done) : "r"(su32(&bar)) : "memory");
        *cycles = clock64() - c0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

static float trunc_tf32_h(float x) {
    uint32_t u;
    memcpy(&u, &x, 4);
    u &= 0xffffe000u;
    memcpy(&x, &u, 4);
    return x;
}

int main(int argc, char** argv) {
    const bool raw = argc > 1;  // operands with full fp32 mantissas: does the MMA truncate them to TF32?
    std::vector<float> A(128 * 32), B(64 * 32), D(128 * 64), R(128 * 64, 0.f);
    srand(1);
    for (auto& x : A) x = raw ? (float)(rand() % 7 - 3) * (1.0f + (float)(rand() % 8191) / 8192.0f / 1024.0f) : (float)(rand() % 7 - 3);
    for (auto& x : B) x = raw ? (float)(rand() % 5 - 2) * (1.0f + (float)(rand() % 8191) / 8192.0f / 1024.0f) : (float)(rand() % 5 - 2);
    double maxdiff_trunc = 0, maxdiff_full = 0;
    for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 64; ++n) {
            double rt = 0, rf = 0;
            for (int k = 0; k < 32; ++k) {
                rt += (double)trunc_tf32_h(A[m * 32 + k]) * (double)trunc_tf32_h(B[n * 32 + k]);
                rf += (double)A[m * 32 + k] * (double)B[n * 32 + k];
            }
            R[m * 64 + n] = raw ? (float)rt : (float)rf;
        }
    float *dA, *dB, *dD;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB, B.size() * 4);
    cudaMalloc(&dD, D.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
    int fails = 0;
    for (int var = 0; var < 3; ++var) {
        cudaMemset(dD, 0, D.size() * 4);
        probe<<<1, 128, 80 * 1024>>>(dA, dB, dD, var);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        int bad = 0, zeros = 0;
        for (int i = 0; i < 128 * 64; ++i) {
            zeros += D[i] == 0.f;
            if (D[i] != R[i]) {
                if (bad < 3) printf("  var %d mismatch m=%d n=%d got %g want %g\n", var, i / 64, i % 64, D[i], R[i]);
                ++bad;
            }
        }
        if (raw) {  // compare against the truncated-operand and the full-precision products
            double dt = 0, df = 0;
            for (int m = 0; m < 128; ++m)
                for (int n = 0; n < 64; ++n) {
                    double rt = 0, rf = 0;
                    for (int k = 0; k < 32; ++k) {
                        rt += (double)trunc_tf32_h(A[m * 32 + k]) * (double)trunc_tf32_h(B[n * 32 + k]);
                        rf += (double)A[m * 32 + k] * (double)B[n * 32 + k];
                    }
                    dt = fmax(dt, fabs(D[m * 64 + n] - rt));
                    df = fmax(df, fabs(D[m * 64 + n] - rf));
                }
            printf("variant %d raw operands: max |D - trunc product| = %.3g, max |D - full product| = %.3g\n", var, dt, df);
        }
        printf("variant %d: %s, %d mismatches, %d zeros (%s)\n", var, bad ? "FAIL" : "OK", bad, zeros, cudaGetErrorString(e));
        fails += bad != 0;
    }
    long long* dc;
    cudaMalloc(&dc, 8);
    cudaFuncSetAttribute(mma_rate<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
    cudaFuncSetAttribute(mma_rate<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
    const char* names[3] = {"A,B MN-major", "A K-major? (B MN)", "K-major"};
    for (int n = 64; n <= 128; n += 64)
        for (int var = 0; var < 3; ++var) {
            if (var == 1) continue;
            long long c = 0;
            if (n == 64) mma_rate<64><<<1, 128, 80 * 1024>>>(var, 1000, dc);
            else mma_rate<128><<<1, 128, 80 * 1024>>>(var, 1000, dc);
            cudaDeviceSynchronize();
            cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
            printf("N=%d %s: %.1f cycles per MMA\n", n, names[var], c / 4000.0);
        }
    return fails;
}
