// 2xFP16 block-scaled GEMM for F32 Dots on tcgen05 kind::f16 (sm_100a).
//
// The reference Dot (kernels.py:123-133) is an f32 multiply-add chain; the
// 3xTF32 kernel (gemm_tc.cu) reproduces it within the 1e-5 normwise Dot
// tolerance with three kind::tf32 MMAs per K-step.  fp16
// has the same 11-bit significand as TF32 and runs at twice the rate, but a
// 5-bit exponent.  So each operand is stored as two fp16 planes of the
// operand scaled by a power of two per 128 x 128 tile of its storage:
//   s = 2^(14 - floor(log2 max|x|)),  hi = fp16_rn(x s),  lo = fp16_rn(x s - hi)
// (x s - hi is exact in fp32; max |x s| lies in [2^14, 2^15), so hi is
// normal, and lo keeps 11 more bits down to 2^-39 of the tile maximum).  The
// representation error is <= 2^-22 |x| (3xTF32 truncates: <= 2^-20), and
//   C = sum over 128-K chunks of (Ahi Bhi + Ahi Blo + Alo Bhi) / (s_a s_b)
// drops only Alo Blo (<= 2^-22 relative): three kind::f16 MMAs per 16-wide
// K-step, promoted every 128 K (one scale block) into round-to-nearest fp32
// registers multiplied by the exact power of two 1 / (s_a s_b).
//
// The kernel is the persistent CTA-pair design of gfb_gemm_tc2_kernel (256 x
// 256 tiles, cta_group::2, 3-stage ring of [A hi | A lo | B hi | B lo] 64 KB
// stages, two 256-column TMEM accumulators, 8 epilogue warps); a stage now
// holds 64 K instead of 32, so the same bytes feed twice the flops.  Planes
// come from gfb_split16_kernel or from the epilogue of the GEMM that
// produces the tensor (epi_flags bit 2).

#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "gfb_common.cuh"
#include "tc_prims.cuh"

namespace gfb {
namespace tc {
struct HCfg {
    static constexpr int BM = 128, BN = 128, BK = 64;  // per CTA: rows of A, rows of B; K per stage (fp16)
    static constexpr int STAGES = 3;
    static constexpr int A_BYTES = BM * BK * 2, B_BYTES = BN * BK * 2;
    static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
    static constexpr int CHUNK_KB = 2, NBUF = 2, NT = 256;  // 128 K per promotion: one scale block
    static constexpr uint32_t TMEM_COLS = 512;
    static constexpr int EPI_WARPS = 8;
    static constexpr int THREADS = 64 + 32 * EPI_WARPS;
    static constexpr int XPOSE_BYTES = EPI_WARPS * 32 * 32 * 4;
    static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256 + XPOSE_BYTES;
};

struct HTile {
    int m0, n0, z, nk;
    int64_t k_begin;
};
__device__ __forceinline__ HTile f16_tile(const gfb_tc_args& p, int t, int ntm, int ntn) {
    const int GROUP_M = p.group_m > 1 ? (int)p.group_m : 1;
    const int per_z = ntm * ntn;
    const int z = t / per_z, r = t % per_z;
    const int g = r / (GROUP_M * ntn), gr = r % (GROUP_M * ntn);
    const int gm = min(GROUP_M, ntm - g * GROUP_M);
    HTile o;
    o.m0 = (g * GROUP_M + gr % gm) * 256;
    o.n0 = (gr / gm) * 256;
    o.z = z;
    o.k_begin = p.k_splits > 1 ? (int64_t)z * p.k_per_split : 0;  // k_per_split % 128 == 0
    const int64_t k_end = p.k_splits > 1 ? min(p.K, o.k_begin + p.k_per_split) : p.K;
    o.nk = k_end > o.k_begin ? (int)((k_end - o.k_begin + HCfg::BK - 1) / HCfg::BK) : 0;
    return o;
}

// Relu-gradient mask bytes (gfb_tc_args.e_mask): the value of
// Maximum(Divide(Relu(x), x), 0) -- 1 for 0 < x < inf, -0 for x < 0, +0
// otherwise -- as 1, 2, 0 (relu_grad_mask in tc_prims.cuh).
__device__ __forceinline__ uint32_t mask_code(float x) { return (x > 0.f && x < INFINITY) ? 1u : (x < 0.f ? 2u : 0u); }
__device__ __forceinline__ float mask_value(uint32_t code) {
    code &= 0xffu;
    return code == 1u ? 1.f : (code == 2u ? -0.f : 0.f);
}
}  // namespace tc

// ---------------------------------------------------------------------------
// Planes of a dense F32 matrix (gfb_split16_args): one 128 x 128 tile per
// iteration, held in registers (16 float4 per thread, all loads in flight),
// block maximum, then the scaled fp16 hi / lo stores.  HBM-bound: 4 B read,
// 4 B written per element.
__global__ void __launch_bounds__(256) gfb_split16_kernel(const __grid_constant__ gfb_split16_args p) {
    using namespace tc;
    __shared__ float red[8];
    const float* src = resolve<const float>(p.tab, p.src);
    __half* hi = resolve<__half>(p.tab, p.hi);
    __half* lo = resolve<__half>(p.tab, p.lo);
    float* sc = resolve<float>(p.tab, p.sc);
    const int64_t tr = (p.rows + 127) / 128, tcn = (p.cols + 127) / 128;
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    for (int64_t tile = blockIdx.x; tile < tr * tcn; tile += gridDim.x) {
        const int64_t r0 = (tile / tcn) * 128, col = (tile % tcn) * 128 + 4 * lane;
        const bool cok = col < p.cols;
        float4 v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int64_t row = r0 + w + 8 * i;
            v[i] = (cok && row < p.rows) ? __ldg(reinterpret_cast<const float4*>(src + row * p.ld + col))
                                         : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        float m = 0.f;
#pragma unroll
        for (int i = 0; i < 16; ++i) m = amax4(m, v[i]);
#pragma unroll
        for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (lane == 0) red[w] = m;
        __syncthreads();
        m = red[0];
#pragma unroll
        for (int i = 1; i < 8; ++i) m = fmaxf(m, red[i]);
        const float s = f16_tile_scale(m);
        if (t == 0) sc[tile] = s;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int64_t row = r0 + w + 8 * i;
            if (!cok || row >= p.rows) continue;
            uint2 h, l;
            split4_f16(scale4(v[i], s), h, l);
            *reinterpret_cast<uint2*>(hi + row * p.cols + col) = h;
            *reinterpret_cast<uint2*>(lo + row * p.cols + col) = l;
        }
        __syncthreads();  // red[] is rewritten by the next tile
    }
}

// ---------------------------------------------------------------------------
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(tc::HCfg::THREADS, 1)
    gfb_gemm_f16p_kernel(const __grid_constant__ gfb_tc_args p) {
    using namespace tc;
    using C_ = HCfg;
    constexpr int BK = C_::BK, STAGES = C_::STAGES, NBUF = C_::NBUF, NT = C_::NT;
    constexpr int A_BYTES = C_::A_BYTES, B_BYTES = C_::B_BYTES, STAGE_BYTES = C_::STAGE_BYTES;
    constexpr int CHUNK_KB = C_::CHUNK_KB, EPI_WARPS = C_::EPI_WARPS;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + NBUF;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + NBUF);
    float* red = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES + 128);  // [8] block maxima (epilogue)

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    const int ntn = (int)((p.N + 255) / 256), ntm = (int)((p.M + 255) / 256);
    const int ntiles = ntn * ntm * (p.k_splits > 1 ? (int)p.k_splits : 1);
    const int pair_id = (int)(blockIdx.x >> 1), npairs = (int)(gridDim.x >> 1);

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < NBUF; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 2 * EPI_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int i = 0; i < 4; ++i) prefetch_tmap(p.tmap[i]);
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                     "r"(C_::TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    cluster_sync_all();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            const uint32_t full0 = peer_addr(full, 0);
            int g = 0;
            for (int t = pair_id; t < ntiles; t += npairs) {
                const HTile T = f16_tile(p, t, ntm, ntn);
                const int am = T.m0 + 128 * rank, bn = T.n0 + 128 * rank;
                for (int kb = 0; kb < T.nk; ++kb, ++g) {
                    const int s = g % STAGES;
                    mbar_wait(&empty[s], ((g / STAGES) & 1) ^ 1);
                    unsigned char* st = smem + s * STAGE_BYTES;
                    if (leader) mbar_expect_tx(&full[s], 2 * STAGE_BYTES);
                    const uint32_t bar = full0 + s * 8;
                    const int kc = (int)T.k_begin + kb * BK;
                    if (p.pad[0] & 3) {  // L2 policies per operand (gfb_tc_args.pad[0]: bit 0 keep A, bit 1 keep B)
                        const uint64_t pa = l2_policy(p.pad[0] & 1), pb = l2_policy(p.pad[0] & 2);
                        if (p.a_ld_mn > 0) {
                            tma_load_3d_pair_hint(st, p.tmap[0], 0, kc, am >> 6, bar, pa);
                            tma_load_3d_pair_hint(st + A_BYTES, p.tmap[1], 0, kc, am >> 6, bar, pa);
                        } else {
                            tma_load_2d_pair_hint(st, p.tmap[0], kc, am, bar, pa);
                            tma_load_2d_pair_hint(st + A_BYTES, p.tmap[1], kc, am, bar, pa);
                        }
                        if (p.b_ld_mn > 0) {
                            tma_load_3d_pair_hint(st + 2 * A_BYTES, p.tmap[2], 0, kc, bn >> 6, bar, pb);
                            tma_load_3d_pair_hint(st + 2 * A_BYTES + B_BYTES, p.tmap[3], 0, kc, bn >> 6, bar, pb);
                        } else {
                            tma_load_2d_pair_hint(st + 2 * A_BYTES, p.tmap[2], kc, bn, bar, pb);
                            tma_load_2d_pair_hint(st + 2 * A_BYTES + B_BYTES, p.tmap[3], kc, bn, bar, pb);
                        }
                    } else if (p.a_ld_mn > 0) {  // MN-major: (64 MN, 64 K, 2 MN chunks) boxes
                        tma_load_3d_pair(st, p.tmap[0], 0, kc, am >> 6, bar);
                        tma_load_3d_pair(st + A_BYTES, p.tmap[1], 0, kc, am >> 6, bar);
                    } else {
                        tma_load_2d_pair(st, p.tmap[0], kc, am, bar);
                        tma_load_2d_pair(st + A_BYTES, p.tmap[1], kc, am, bar);
                    }
                    if (!(p.pad[0] & 3)) {
                        if (p.b_ld_mn > 0) {
                            tma_load_3d_pair(st + 2 * A_BYTES, p.tmap[2], 0, kc, bn >> 6, bar);
                            tma_load_3d_pair(st + 2 * A_BYTES + B_BYTES, p.tmap[3], 0, kc, bn >> 6, bar);
                        } else {
                            tma_load_2d_pair(st + 2 * A_BYTES, p.tmap[2], kc, bn, bar);
                            tma_load_2d_pair(st + 2 * A_BYTES + B_BYTES, p.tmap[3], kc, bn, bar);
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && leader) {
            const bool a_mn = p.a_ld_mn > 0, b_mn = p.b_ld_mn > 0;
            const uint32_t idesc = idesc_f16(256, 256) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16);
            int g = 0, gchunk = 0;
            for (int t = pair_id; t < ntiles; t += npairs) {
                const HTile T = f16_tile(p, t, ntm, ntn);
                for (int kb = 0; kb < T.nk; ++kb, ++g) {
                    const int s = g % STAGES;
                    const int chunk = gchunk + kb / CHUNK_KB, b = chunk % NBUF;
                    const bool chunk_start = kb % CHUNK_KB == 0;
                    if (chunk_start) {
                        mbar_wait(&tempty[b], ((chunk / NBUF) & 1) ^ 1);
                        asm volatile("tcgen05.fence::after_thread_sync;");
                    }
                    mbar_wait(&full[s], (g / STAGES) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    unsigned char* st = smem + s * STAGE_BYTES;
                    const uint32_t sa = su32(st), sb = sa + 2 * A_BYTES;
                    const uint32_t d = tmem + (uint32_t)(b * NT);
#pragma unroll
                    for (int j = 0; j < BK / 16; ++j) {
                        // K-major SW128: 16 fp16 = 32 B along K inside the atom; MN-major:
                        // 16 K rows = two 1 KB atoms further, MN chunks 8 KB apart
                        const uint64_t ah = a_mn ? smem_desc_mn16(sa + j * 2048, 8192) : smem_desc(st) + ((uint64_t)(j * 32) >> 4);
                        const uint64_t al = a_mn ? smem_desc_mn16(sa + A_BYTES + j * 2048, 8192)
                                                 : smem_desc(st + A_BYTES) + ((uint64_t)(j * 32) >> 4);
                        const uint64_t bh = b_mn ? smem_desc_mn16(sb + j * 2048, 8192)
                                                 : smem_desc(st + 2 * A_BYTES) + ((uint64_t)(j * 32) >> 4);
                        const uint64_t bl = b_mn ? smem_desc_mn16(sb + B_BYTES + j * 2048, 8192)
                                                 : smem_desc(st + 2 * A_BYTES + B_BYTES) + ((uint64_t)(j * 32) >> 4);
                        const uint32_t acc = !(chunk_start && j == 0);
                        mma_f16_pair(d, ah, bh, idesc, acc);
                        mma_f16_pair(d, ah, bl, idesc, 1);
                        mma_f16_pair(d, al, bh, idesc, 1);
                    }
                    mma_commit_pair(&empty[s]);
                    if (kb % CHUNK_KB == CHUNK_KB - 1 || kb == T.nk - 1) mma_commit_pair(&tfull[b]);
                }
                gchunk += (T.nk + CHUNK_KB - 1) / CHUNK_KB;
            }
        }
    } else {
        // epilogue: warp w owns TMEM lanes [32 (w % 4), +32) = this CTA's rows and
        // the 128 columns of group cg = one 128-column scale block of B
        constexpr int EC = 128;
        const int q = warp & 3, cg = (warp - 2) >> 2;
        const uint32_t tempty0 = peer_addr(tempty, 0);
        const int mblocks = (int)((p.M + 127) / 128), nblocks = (int)((p.N + 127) / 128);
        int gchunk = 0;
        for (int t = pair_id; t < ntiles; t += npairs) {
            const HTile T = f16_tile(p, t, ntm, ntn);
            const int nchunk = (T.nk + CHUNK_KB - 1) / CHUNK_KB;
            const int mb = (T.m0 >> 7) + (int)rank, nb = (T.n0 >> 7) + cg;
            // this tile's scale columns: chunk c0 reads sa[c0 * a_sc_k], sb[c0 * b_sc_k]
            const int kb0 = (int)(T.k_begin >> 7);
            const float* sa_p = mb < mblocks ? resolve<const float>(p.tab, p.a_sc) + (int64_t)mb * p.a_sc_r + (int64_t)kb0 * p.a_sc_k : nullptr;
            const float* sb_p = nb < nblocks ? resolve<const float>(p.tab, p.b_sc) + (int64_t)nb * p.b_sc_r + (int64_t)kb0 * p.b_sc_k : nullptr;
            const int pf_at = p.epi_kind == 2 ? max(0, nchunk - 3) : -1;
            float acc[EC];
#pragma unroll
            for (int j = 0; j < EC; ++j) acc[j] = 0.0f;
            int b_last = 0;
            for (int c0 = 0; c0 < nchunk; ++c0) {
                const int chunk = gchunk + c0, b = chunk % NBUF;
                const float sa = sa_p ? __ldg(sa_p + (int64_t)c0 * p.a_sc_k) : 1.f;
                const float sb = sb_p ? __ldg(sb_p + (int64_t)c0 * p.b_sc_k) : 1.f;
                const float ia = __frcp_rn(sa), ib = __frcp_rn(sb), inv = ia * ib;  // exact powers of two
                const bool one_step = inv >= 1.17549435e-38f && inv < INFINITY;
                mbar_wait(&tfull[b], (chunk / NBUF) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * NT + cg * EC);
#pragma unroll
                for (int c = 0; c < EC / 16; ++c) {
                    // 16 columns per load: the accumulators plus one load stay inside the
                    // register budget (spills would go through the small L1 to L2)
                    uint32_t r[16];
                    asm volatile(
                        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                        : "r"(tbase + c * 16));
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    if (one_step) {
#pragma unroll
                        for (int j = 0; j < 16; ++j) acc[c * 16 + j] = fmaf(__uint_as_float(r[j]), inv, acc[c * 16 + j]);
                    } else {
#pragma unroll
                        for (int j = 0; j < 16; ++j) acc[c * 16 + j] = fmaf(__fmul_rn(__uint_as_float(r[j]), ia), ib, acc[c * 16 + j]);
                    }
                }
                if (c0 == nchunk - 1) {
                    // the tile's sums go back into the buffer just drained (released
                    // after the store phase), so the stores below run from TMEM
                    // with a few live registers instead of the 128 accumulators
#pragma unroll
                    for (int c = 0; c < EC / 16; ++c) tmem_st16(tbase + c * 16, &acc[c * 16]);
                    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                    b_last = b;
                    break;
                }
                asm volatile("tcgen05.fence::before_thread_sync;");
                __syncwarp();
                if (lane == 0)
                    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(tempty0 + b * 8) : "memory");
                if (c0 == pf_at) {
                    // the store phase reads this row's 128 mask bytes (or 512 B of x): pull
                    // them into L2 while the last chunks are still being multiplied
                    const int64_t row = T.m0 + 128 * (int64_t)rank + q * 32 + lane, col = T.n0 + cg * EC;
                    if (row < p.M && col < p.N) {
                        if (p.epi_flags & 16) {
                            asm volatile("prefetch.global.L2 [%0];" ::"l"(resolve<const uint8_t>(p.tab, p.e_mask) + row * p.N + col));
                        } else {
                            const float* xr = resolve<const float>(p.tab, p.e_aux2) + row * p.c_sm + col;
#pragma unroll
                            for (int l = 0; l < 4; ++l) asm volatile("prefetch.global.L2 [%0];" ::"l"(xr + 32 * l));
                        }
                    }
                }
            }
            gchunk += nchunk;
            if (nchunk == 0) continue;
            const uint32_t tsum = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b_last * NT + cg * EC);
            float* C = resolve<float>(p.tab, p.c) + (p.k_splits > 1 ? (int64_t)T.z * p.split_stride : 0);
            const int64_t rowA = T.m0 + 128 * (int64_t)rank + q * 32;  // this warp's 32 rows
            const int64_t prow = rowA + lane, colb = T.n0 + cg * EC;
            const bool rok = prow < p.M;
            const bool coalesced = p.c_sn == 1 && (p.c_sm & 3) == 0 && (p.N & 3) == 0;
            bool released = false;
            if (!coalesced) {
                if (p.epi_kind != 0 || (p.epi_flags & 4)) __trap();  // the lowering fuses epilogues into dense outputs only
#pragma unroll 1
                for (int c = 0; c < EC / 16; ++c) {
                    float v[16];
                    tmem_ld16(tsum + c * 16, v);
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const int64_t col = colb + c * 16 + j;
                        if (rok && col < p.N) C[prow * p.c_sm + col * p.c_sn] = v[j];
                    }
                }
            } else {
                // Pass 1, row layout (lane = row prow, 16 columns per TMEM load): the
                // absorbed elementwise maps, their row-layout side stores (the mask
                // bytes, C / out2 of kind 1), y written back to TMEM and the block
                // maximum.  Pass 2, through the swizzled transpose tile: C of kinds
                // 0 / 2 (= y) and the fp16 planes with row-contiguous stores.
                const bool store_c = (p.epi_flags & 32) == 0;
                const bool planes = (p.epi_flags & 4) != 0;
                float ymax = 0.f;
                if (p.epi_kind != 0 || planes) {
                    const float* bias = p.epi_kind == 1 ? resolve<const float>(p.tab, p.e_bias) : nullptr;
                    const bool mask_in = p.epi_kind == 2 && (p.epi_flags & 16);
                    uint8_t* mkout = p.epi_kind == 1 && (p.epi_flags & 8) ? resolve<uint8_t>(p.tab, p.e_mask) + prow * p.N : nullptr;
                    const uint8_t* mkrow = mask_in ? resolve<const uint8_t>(p.tab, p.e_mask) + prow * p.N : nullptr;
                    const float* xrow = p.epi_kind == 2 && !mask_in ? resolve<const float>(p.tab, p.e_aux2) + prow * p.c_sm : nullptr;
                    float* crow = p.epi_kind == 1 && store_c ? C + prow * p.c_sm : nullptr;
                    float* orow = (p.epi_flags & 1) ? resolve<float>(p.tab, p.e_out2) + prow * p.c_sm : nullptr;
#pragma unroll 2
                    for (int c = 0; c < EC / 16; ++c) {
                        const int64_t col0 = colb + 16 * c;
                        const bool full16 = rok && col0 + 16 <= p.N;
                        float v[16];
                        tmem_ld16(tsum + c * 16, v);
                        if (p.epi_kind == 1) {
                            uint32_t code[4];
#pragma unroll
                            for (int d = 0; d < 4; ++d) {
                                const int64_t col = col0 + 4 * d;
                                const bool ok = rok && col < p.N;
                                const float4 b4 = col < p.N ? __ldg(reinterpret_cast<const float4*>(bias + col)) : make_float4(0.f, 0.f, 0.f, 0.f);
                                const float4 z = make_float4(__fadd_rn(v[4 * d], b4.x), __fadd_rn(v[4 * d + 1], b4.y),
                                                             __fadd_rn(v[4 * d + 2], b4.z), __fadd_rn(v[4 * d + 3], b4.w));
                                const float4 y = make_float4(z.x > 0.f ? z.x : 0.f, z.y > 0.f ? z.y : 0.f, z.z > 0.f ? z.z : 0.f,
                                                             z.w > 0.f ? z.w : 0.f);
                                code[d] = mask_code(z.x) | (mask_code(z.y) << 8) | (mask_code(z.z) << 16) | (mask_code(z.w) << 24);
                                if (ok) {
                                    ymax = amax4(ymax, y);
                                    if (crow) *reinterpret_cast<float4*>(crow + col) = z;
                                    if (orow) *reinterpret_cast<float4*>(orow + col) = y;
                                }
                                v[4 * d] = y.x, v[4 * d + 1] = y.y, v[4 * d + 2] = y.z, v[4 * d + 3] = y.w;
                            }
                            if (mkout && full16) {
                                *reinterpret_cast<uint4*>(mkout + col0) = make_uint4(code[0], code[1], code[2], code[3]);
                            } else if (mkout && rok) {
#pragma unroll
                                for (int d = 0; d < 4; ++d)
                                    if (col0 + 4 * d < p.N) *reinterpret_cast<uint32_t*>(mkout + col0 + 4 * d) = code[d];
                            }
                        } else if (p.epi_kind == 2) {
                            uint32_t code[4] = {0u, 0u, 0u, 0u};
                            float4 x4[4];
                            if (mask_in) {
                                if (full16) {
                                    const uint4 m = __ldg(reinterpret_cast<const uint4*>(mkrow + col0));
                                    code[0] = m.x, code[1] = m.y, code[2] = m.z, code[3] = m.w;
                                } else if (rok) {
#pragma unroll
                                    for (int d = 0; d < 4; ++d)
                                        if (col0 + 4 * d < p.N) code[d] = __ldg(reinterpret_cast<const uint32_t*>(mkrow + col0 + 4 * d));
                                }
                            } else {
#pragma unroll
                                for (int d = 0; d < 4; ++d)
                                    x4[d] = rok && col0 + 4 * d < p.N ? __ldg(reinterpret_cast<const float4*>(xrow + col0 + 4 * d))
                                                                    : make_float4(0.f, 0.f, 0.f, 0.f);
                            }
#pragma unroll
                            for (int d = 0; d < 4; ++d) {
                                float4 y;
                                if (mask_in)
                                    y = make_float4(__fmul_rn(v[4 * d], mask_value(code[d])), __fmul_rn(v[4 * d + 1], mask_value(code[d] >> 8)),
                                                    __fmul_rn(v[4 * d + 2], mask_value(code[d] >> 16)),
                                                    __fmul_rn(v[4 * d + 3], mask_value(code[d] >> 24)));
                                else
                                    y = make_float4(__fmul_rn(v[4 * d], relu_grad_mask(x4[d].x)), __fmul_rn(v[4 * d + 1], relu_grad_mask(x4[d].y)),
                                                    __fmul_rn(v[4 * d + 2], relu_grad_mask(x4[d].z)),
                                                    __fmul_rn(v[4 * d + 3], relu_grad_mask(x4[d].w)));
                                if (rok && col0 + 4 * d < p.N) ymax = amax4(ymax, y);
                                v[4 * d] = y.x, v[4 * d + 1] = y.y, v[4 * d + 2] = y.z, v[4 * d + 3] = y.w;
                            }
                        } else {
#pragma unroll
                            for (int j = 0; j < 16; j += 4)
                                if (rok && col0 + j < p.N) ymax = amax4(ymax, make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]));
                        }
                        if (p.epi_kind != 0) tmem_st16(tsum + c * 16, v);
                    }
                    if (p.epi_kind != 0) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                }
                float s = 1.f;
                __half* ehi = nullptr;
                __half* elo = nullptr;
                if (planes) {
                    // block maximum over the 4 warps of this column group (one 128 x 128 block)
#pragma unroll
                    for (int o = 16; o; o >>= 1) ymax = fmaxf(ymax, __shfl_xor_sync(0xffffffffu, ymax, o));
                    if (lane == 0) red[warp - 2] = ymax;
                    asm volatile("bar.sync 1, 256;" ::: "memory");
                    float m = red[cg * 4];
#pragma unroll
                    for (int i = 1; i < 4; ++i) m = fmaxf(m, red[cg * 4 + i]);
                    asm volatile("bar.sync 1, 256;" ::: "memory");  // red[] is rewritten by the next tile
                    s = f16_tile_scale(m);
                    ehi = resolve<__half>(p.tab, p.e_hi);
                    elo = resolve<__half>(p.tab, p.e_lo);
                    if (q == 0 && lane == 0 && mb < mblocks && nb < nblocks) resolve<float>(p.tab, p.e_sc)[(int64_t)mb * nblocks + nb] = s;
                }
                const bool c_pass2 = store_c && p.epi_kind != 1;  // C == y
                float* csum = (p.epi_flags & 64) ? resolve<float>(p.tab, p.e_csum) + (rowA >> 5) * p.N : nullptr;
                if (c_pass2 || planes || csum) {
                    // y back into registers, then the TMEM buffer goes back to the MMA
                    // warp before the stores: the next tile's MMAs overlap them
                    float yv[EC];
#pragma unroll
                    for (int c = 0; c < EC / 16; ++c) tmem_ld16(tsum + c * 16, &yv[c * 16]);
                    asm volatile("tcgen05.fence::before_thread_sync;");
                    __syncwarp();
                    if (lane == 0)
                        asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(tempty0 + b_last * 8) : "memory");
                    released = true;
                    float* xt = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES + 256) + (warp - 2) * 1024;
                    const int qd = lane & 7;
#pragma unroll
                    for (int c = 0; c < EC / 32; ++c) {
                        // lane r writes its row's 32 values as 8 swizzled 16-byte pieces
#pragma unroll
                        for (int d = 0; d < 8; ++d)
                            *reinterpret_cast<float4*>(xt + lane * 32 + ((d ^ (lane & 7)) << 2)) =
                                make_float4(yv[c * 32 + 4 * d], yv[c * 32 + 4 * d + 1], yv[c * 32 + 4 * d + 2], yv[c * 32 + 4 * d + 3]);
                        __syncwarp();
                        const int64_t col = colb + c * 32 + 4 * qd;
                        float4 cs = make_float4(0.f, 0.f, 0.f, 0.f);  // this lane's rows, in order
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const int rr = 4 * i + (lane >> 3);  // lanes 8k..8k+7 cover one 128-byte row piece
                            const int64_t row = rowA + rr;
                            const float4 y = *reinterpret_cast<const float4*>(xt + rr * 32 + ((qd ^ (rr & 7)) << 2));
                            if (col >= p.N || row >= p.M) continue;
                            if (csum) cs = make_float4(__fadd_rn(cs.x, y.x), __fadd_rn(cs.y, y.y), __fadd_rn(cs.z, y.z), __fadd_rn(cs.w, y.w));
                            if (c_pass2) *reinterpret_cast<float4*>(C + row * p.c_sm + col) = y;
                            if (planes) {
                                uint2 hh, ll;
                                split4_f16(scale4(y, s), hh, ll);
                                *reinterpret_cast<uint2*>(ehi + row * p.N + col) = hh;
                                *reinterpret_cast<uint2*>(elo + row * p.N + col) = ll;
                            }
                        }
                        if (csum) {
                            // the four row groups (lane >> 3) of one column quad: (p0 + p1) + (p2 + p3)
#pragma unroll
                            for (int o = 8; o <= 16; o <<= 1)
                                cs = make_float4(__fadd_rn(cs.x, __shfl_xor_sync(0xffffffffu, cs.x, o)),
                                                 __fadd_rn(cs.y, __shfl_xor_sync(0xffffffffu, cs.y, o)),
                                                 __fadd_rn(cs.z, __shfl_xor_sync(0xffffffffu, cs.z, o)),
                                                 __fadd_rn(cs.w, __shfl_xor_sync(0xffffffffu, cs.w, o)));
                            if (lane < 8 && col < p.N) *reinterpret_cast<float4*>(csum + col) = cs;
                        }
                        __syncwarp();
                    }
                }
            }
            if (!released) {  // release the staged buffer to the MMA warp
                asm volatile("tcgen05.fence::before_thread_sync;");
                __syncwarp();
                if (lane == 0)
                    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(tempty0 + b_last * 8) : "memory");
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    cluster_sync_all();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C_::TMEM_COLS));
    }
}

}  // namespace gfb

extern "C" const void* gfb_f16_kernel_ptr(int kind) {
    if (kind == GFB_K_DOT_F16P) return (const void*)gfb::gfb_gemm_f16p_kernel;
    if (kind == GFB_K_SPLIT_F16) return (const void*)gfb::gfb_split16_kernel;
    return nullptr;
}
extern "C" int gfb_f16_pair_smem_bytes(void) { return gfb::tc::HCfg::SMEM_BYTES; }
