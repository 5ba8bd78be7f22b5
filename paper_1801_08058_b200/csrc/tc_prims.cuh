// Tensor-core primitives shared by the sm_100a kernels: mbarriers, TMA,
// UMMA descriptors, tcgen05.mma / commit (single CTA and CTA pair).
#pragma once

#include <cuda_fp16.h>

#include <cstdint>

#include "gfb_common.cuh"

namespace gfb {
namespace tc {

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
// Bounded wait: a protocol bug traps instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    uint32_t done = 0;
    for (uint32_t spin = 0; spin < (1u << 28); ++spin) {
        asm volatile(
            "{\n\t.reg .pred P;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, P;\n}"
            : "=r"(done)
            : "r"(su32(b)), "r"(parity)
            : "memory");
        if (done) return;
    }
    __trap();
}
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            su32(dst)),
        "l"(tmap), "r"(c0), "r"(c1), "r"(su32(bar))
        : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const void* tmap) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(tmap) : "memory");
}

__device__ __forceinline__ float4 lds128(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts128(uint32_t a, float4 v) {
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}

// UMMA shared-memory descriptor: K-major, 128B swizzle, 8-row atoms of 1 KB.
__device__ __forceinline__ uint64_t smem_desc(const void* p) {
    const uint64_t addr = su32(p);
    uint64_t d = 0;
    d |= (addr >> 4) & 0x3FFFull;          // start address
    d |= (uint64_t)0 << 16;                // LBO (unused for swizzled K-major)
    d |= (uint64_t)(1024 >> 4) << 32;      // SBO: 8 rows x 128 B
    d |= (uint64_t)1 << 46;                // version (sm100)
    d |= (uint64_t)2 << 61;                // SWIZZLE_128B
    return d;
}

// Instruction descriptor: kind::tf32, fp32 accumulate, K-major A and B.
constexpr uint32_t idesc_tf32(int M, int N) {
    return (1u << 4)               // c_format F32
           | (2u << 7)             // a_format TF32
           | (2u << 10)            // b_format TF32
           | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
        "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
                 : "memory");
}

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same object in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t peer_addr(const void* p, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(su32(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const void* tmap, int c0, int c1, uint32_t bar_cluster) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            su32(dst)),
        "l"(tmap), "r"(c0), "r"(c1), "r"(bar_cluster)
        : "memory");
}
// The same loads with an L2 cache policy (createpolicy: evict_first for a
// streamed operand, evict_last for one every tile re-reads).
__device__ __forceinline__ uint64_t l2_policy(bool keep) {
    uint64_t p;
    if (keep)
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    else
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void tma_load_2d_pair_hint(void* dst, const void* tmap, int c0, int c1, uint32_t bar_cluster,
                                                      uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(
            su32(dst)),
        "l"(tmap), "r"(c0), "r"(c1), "r"(bar_cluster), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d_pair_hint(void* dst, const void* tmap, int c0, int c1, int c2, uint32_t bar_cluster,
                                                      uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(
            su32(dst)),
        "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(bar_cluster), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d_pair(void* dst, const void* tmap, int c0, int c1, int c2, uint32_t bar_cluster) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            su32(dst)),
        "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(bar_cluster)
        : "memory");
}
// MN-major SWIZZLE_128B_BASE32B operand (see the tcgw kernel below): MN atoms
// 4096 B apart (LBO), 4-row K groups 512 B apart (SBO)
__device__ __forceinline__ uint64_t smem_desc_mn_at(uint32_t addr) {
    uint64_t d = 0;
    d |= (addr >> 4) & 0x3FFFull;
    d |= (uint64_t)(4096 >> 4) << 16;
    d |= (uint64_t)(512 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)1 << 61;
    return d;
}
// The Relu gradient's mask Maximum(Divide(Relu(x), x), 0) (autodiff.py:143-148)
// as a function of x alone, value for value: Relu(x) / x is exactly 1 for
// 0 < x < inf, -0 for x < 0 (0 / negative, including -inf), and NaN for
// x = +-0, +inf, NaN, which Maximum(NaN, 0) turns into +0.
__device__ __forceinline__ float relu_grad_mask(float x) {
    return (x > 0.f && x < INFINITY) ? 1.f : (x < 0.f ? -0.f : 0.f);
}
__device__ __forceinline__ void mma_tf32_pair(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
        "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                     su32(bar)),
                 "h"((uint16_t)3)
                 : "memory");
}

__device__ __forceinline__ void tma_load_4d(void* dst, const void* tmap, int c0, int c1, int c2, int c3, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(
            su32(dst)),
        "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(su32(bar))
        : "memory");
}

// Output rows of a pixel-box tile.
struct BoxRows {
    int n0, y0, x0, BX, BY, No, Yo, Xo;
    int64_t o_n, o_y, o_x;
    __device__ __forceinline__ int64_t operator()(int r) const {
        const int xx = r % BX, t = r / BX, yy = t % BY, ni = t / BY;
        const int n = n0 + ni, y = y0 + yy, x = x0 + xx;
        if (n >= No || y >= Yo || x >= Xo) return -1;
        return n * o_n + y * o_y + x * o_x;
    }
};

// ---- kind::f16 (the 2xFP16 block-scaled GEMM, gemm_f16.cu) ----
// Instruction descriptor: F16 A and B, F32 accumulate; bits 15 / 16 select
// MN-major A / B.
constexpr uint32_t idesc_f16(int M, int N) {
    return (1u << 4)               // c_format F32
           | (0u << 7)             // a_format F16
           | (0u << 10)            // b_format F16
           | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// MN-major 16-bit operand in the canonical SWIZZLE_128B layout: 64-element
// (128 B) MN rows per K index, 8-K-row atoms of 1 KB (SBO), MN chunks of 64
// elements `lbo` bytes apart.
__device__ __forceinline__ uint64_t smem_desc_mn16(uint32_t addr, uint32_t lbo) {
    uint64_t d = 0;
    d |= (addr >> 4) & 0x3FFFull;
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;  // SWIZZLE_128B
    return d;
}
__device__ __forceinline__ void mma_f16_pair(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
        "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}
// Power-of-two scale of a tile whose largest magnitude is mx: brings mx into
// [2^14, 2^15), so x * s rounds to a normal fp16 hi part and the remainder
// keeps 11 more bits (subnormal only below 2^-39 of the tile maximum); 1 for
// an all-zero tile or a non-finite maximum.
__device__ __forceinline__ float f16_tile_scale(float mx) {
    if (!(mx > 0.f) || !(mx < INFINITY)) return 1.f;
    int e;
    frexpf(mx, &e);           // mx = f * 2^e, f in [0.5, 1): floor(log2 mx) = e - 1
    int k = 15 - e;           // 14 - floor(log2 mx)
    k = k > 126 ? 126 : k;
    return ldexpf(1.f, k);
}
// fp16 hi / lo pieces
__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
    const __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&h);
}
// hi / lo fp16 pieces of four values already multiplied by their scale
__device__ __forceinline__ void split4_f16(float4 v, uint2& hi, uint2& lo) {
    const __half2 h01 = __floats2half2_rn(v.x, v.y), h23 = __floats2half2_rn(v.z, v.w);
    const float2 f01 = __half22float2(h01), f23 = __half22float2(h23);
    hi = make_uint2(*reinterpret_cast<const uint32_t*>(&h01), *reinterpret_cast<const uint32_t*>(&h23));
    lo = make_uint2(pack_h2(__fsub_rn(v.x, f01.x), __fsub_rn(v.y, f01.y)), pack_h2(__fsub_rn(v.z, f23.x), __fsub_rn(v.w, f23.y)));
}
__device__ __forceinline__ float4 scale4(float4 v, float s) {
    return make_float4(__fmul_rn(v.x, s), __fmul_rn(v.y, s), __fmul_rn(v.z, s), __fmul_rn(v.w, s));
}
// |x| for the scale maxima: infinities (and NaN, which fmaxf drops) do not
// count, so a tile holding an inf keeps the scale of its finite values (inf
// * s stays inf; with scale 1 its finite neighbours could overflow fp16)
__device__ __forceinline__ float fin_abs(float x) { return fabsf(x) < INFINITY ? fabsf(x) : 0.f; }
__device__ __forceinline__ float amax4(float m, float4 v) {
    return fmaxf(fmaxf(m, fmaxf(fin_abs(v.x), fin_abs(v.y))), fmaxf(fin_abs(v.z), fin_abs(v.w)));
}
// 16 TMEM columns of this warp's 32 lanes (one per thread), fp32
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]),
          "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
        "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
        "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
        "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15]))
        : "memory");
}
}  // namespace tc
}  // namespace gfb
