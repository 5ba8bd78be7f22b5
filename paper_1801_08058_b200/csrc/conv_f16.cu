// 2xFP16 implicit-GEMM convolution on tcgen05 kind::f16 (sm_100a).
//
// The 3xTF32 TMA-box convolution (gfb_conv_tcx_kernel) splits every landed
// fp32 activation tile into TF32 hi / lo in shared memory; at 64 channels that
// conversion chain and its shared-memory traffic pace the kernel (DESIGN.md
// "Convolutions").  Here the activation arrives already split: fp16 hi / lo
// planes of x s_c, s_c a power of two per channel (gfb_chsplit_kernel), and
// the filter planes carry 1 / s_c (gfb_fsplit_kernel), so the channel scales
// cancel inside each product:
//   C[p, n] = (1 / t_n) sum_k (Ahi Bhi + Ahi Blo + Alo Bhi)[p, k, n]
// with t_n the filter row's own power-of-two scale, applied once at the end.
// Per-element representation error <= 2^-22 |x| down to 2^-39 of the
// channel's maximum (3xTF32: 2^-20).  The kernel has no converter warps: TMA
// lands the hi and lo boxes (64 channels x the pixel box, 128 B rows,
// SWIZZLE_128B K-major) straight into the MMA stage.
//   warp 0  TMA producer (A hi / lo boxes with the convolution's strides and
//           zero-filled padding, B hi / lo planes)
//   warp 1  TMEM allocator + MMA issuer (three kind::f16 MMAs per 16-wide K)
//   2..5    epilogue: 128-K chunks promoted into fp32 registers, 1 / t_n,
//           pixel-box stores
// Persistent: CTA b walks (column tile, pixel tile) items b, b + gridDim.x, ...

#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "gfb_common.cuh"
#include "tc_prims.cuh"

namespace gfb {
namespace tc {
template <int BN_>
struct HXCfg {
    static constexpr int BM = 128, BN = BN_, BK = 64;  // K per stage: 64 fp16 channels = one 128 B row
    static constexpr int A_BYTES = BM * BK * 2, B_BYTES = BN * BK * 2;
    static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
    static constexpr int STAGES = BN_ == 128 ? 3 : 4;
    static constexpr int CHUNK_KB = 2, NBUF = 512 / BN;
    static constexpr uint32_t TMEM_COLS = 512;
    static constexpr int EPI_WARPS = 4;
    static constexpr int THREADS = 64 + 32 * EPI_WARPS;
    static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 256 + 1024;
};

__device__ __forceinline__ void mma_f16_cta(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
        "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}
}  // namespace tc

// ---------------------------------------------------------------------------
// Channel maxima (gfb_chsplit_args): block b folds |x| over its share of the
// P pixel rows, eight rows per thread in flight (thread t owns the 4 channels
// 4 (t % C4), C4 = C / 4 divides 256), then one atomicMax per channel.
__global__ void __launch_bounds__(256) gfb_chmax_kernel(const __grid_constant__ gfb_chsplit_args p) {
    using namespace tc;
    __shared__ float4 red[256];
    const float* src = resolve<const float>(p.tab, p.src);
    float* part = resolve<float>(p.tab, p.partial);
    const int C4 = (int)(p.C / 4), t = threadIdx.x, g = t % C4, rpi = 256 / C4;
    const int64_t per = (p.P + gridDim.x - 1) / gridDim.x, r0 = (int64_t)blockIdx.x * per, r1 = min(p.P, r0 + per);
    float4 m = make_float4(0.f, 0.f, 0.f, 0.f);
    auto fold = [&](float4 v) {
        m = make_float4(fmaxf(m.x, fin_abs(v.x)), fmaxf(m.y, fin_abs(v.y)), fmaxf(m.z, fin_abs(v.z)), fmaxf(m.w, fin_abs(v.w)));
    };
    int64_t row = r0 + t / C4;
    for (; row + 7 * rpi < r1; row += 8 * rpi) {
        float4 v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = __ldg(reinterpret_cast<const float4*>(src + (row + i * rpi) * p.C) + g);
#pragma unroll
        for (int i = 0; i < 8; ++i) fold(v[i]);
    }
    for (; row < r1; row += rpi) fold(__ldg(reinterpret_cast<const float4*>(src + row * p.C) + g));
    red[t] = m;
    __syncthreads();
    if (t < C4) {
        for (int i = t + C4; i < 256; i += C4) {
            const float4 v = red[i];
            m = make_float4(fmaxf(m.x, v.x), fmaxf(m.y, v.y), fmaxf(m.z, v.z), fmaxf(m.w, v.w));
        }
        // non-negative floats order like their bit patterns
        unsigned int* pm = reinterpret_cast<unsigned int*>(part) + 4 * t;
        atomicMax(pm, __float_as_uint(m.x));
        atomicMax(pm + 1, __float_as_uint(m.y));
        atomicMax(pm + 2, __float_as_uint(m.z));
        atomicMax(pm + 3, __float_as_uint(m.w));
    }
}

// Channel-scaled planes: the scales from the channel maxima (block 0
// publishes them for the filter split), pixel rows streamed eight per thread.
__global__ void __launch_bounds__(256) gfb_chsplit_kernel(const __grid_constant__ gfb_chsplit_args p) {
    using namespace tc;
    const int t = threadIdx.x;
    const float* src = resolve<const float>(p.tab, p.src);
    __half* hi = resolve<__half>(p.tab, p.hi);
    __half* lo = resolve<__half>(p.tab, p.lo);
    const int C4 = (int)(p.C / 4), g = t % C4, rpi = 256 / C4;
    const float4 m4 = __ldg(reinterpret_cast<const float4*>(resolve<const float>(p.tab, p.partial)) + g);
    const float4 s4 = make_float4(f16_tile_scale(m4.x), f16_tile_scale(m4.y), f16_tile_scale(m4.z), f16_tile_scale(m4.w));
    if (blockIdx.x == 0 && t < C4) reinterpret_cast<float4*>(resolve<float>(p.tab, p.sc))[g] = s4;
    auto put = [&](int64_t row, float4 v) {
        uint2 h, l;
        split4_f16(make_float4(__fmul_rn(v.x, s4.x), __fmul_rn(v.y, s4.y), __fmul_rn(v.z, s4.z), __fmul_rn(v.w, s4.w)), h, l);
        const int64_t off = row * p.C + 4 * g;
        *reinterpret_cast<uint2*>(hi + off) = h;
        *reinterpret_cast<uint2*>(lo + off) = l;
    };
    const int64_t stride = (int64_t)gridDim.x * rpi;
    int64_t row = (int64_t)blockIdx.x * rpi + t / C4;
    for (; row + 7 * stride < p.P; row += 8 * stride) {
        float4 v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = __ldg(reinterpret_cast<const float4*>(src + (row + i * stride) * p.C) + g);
#pragma unroll
        for (int i = 0; i < 8; ++i) put(row + i * stride, v[i]);
    }
    for (; row < p.P; row += stride) put(row, __ldg(reinterpret_cast<const float4*>(src + row * p.C) + g));
}

// Filter planes (gfb_fsplit_args): one block per row, 32-bit index math
// (a filter has < 2^31 elements).
__global__ void __launch_bounds__(256) gfb_fsplit_kernel(const __grid_constant__ gfb_fsplit_args p) {
    using namespace tc;
    __shared__ float red[8];
    __shared__ float isc[1024];  // 1 / s_c (exact: powers of two)
    const float* w = resolve<const float>(p.tab, p.w) + (int64_t)blockIdx.x * p.s_r;
    const float* sc = resolve<const float>(p.tab, p.sc);
    const int K = (int)p.K, e1 = (int)p.e1, e2 = (int)p.e2, t0 = (int)p.t0, t1 = (int)p.t1, t2 = (int)p.t2;
    for (int c = threadIdx.x; c < e2; c += 256) isc[c] = __frcp_rn(__ldg(sc + c));
    __syncthreads();
    auto value = [&](int k) {
        const int d2 = k % e2, d01 = k / e2, d1 = d01 % e1, d0 = d01 / e1;
        return __fmul_rn(__ldg(w + d0 * t0 + d1 * t1 + d2 * t2), isc[d2]);
    };
    float m = 0.f;
    int k = threadIdx.x;
    for (; k + 768 < K; k += 1024) {  // four gathers in flight
        float v[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) v[i] = value(k + 256 * i);
#pragma unroll
        for (int i = 0; i < 4; ++i) m = fmaxf(m, fin_abs(v[i]));
    }
    for (; k < K; k += 256) m = fmaxf(m, fin_abs(value(k)));
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    m = red[0];
#pragma unroll
    for (int i = 1; i < 8; ++i) m = fmaxf(m, red[i]);
    const float t = f16_tile_scale(m);
    if (threadIdx.x == 0) resolve<float>(p.tab, p.inv)[blockIdx.x] = __frcp_rn(t);
    __half* hi = resolve<__half>(p.tab, p.hi) + (int64_t)blockIdx.x * K;
    __half* lo = resolve<__half>(p.tab, p.lo) + (int64_t)blockIdx.x * K;
    auto put = [&](int kk, float x) {
        const float v = __fmul_rn(x, t);
        const __half h = __float2half_rn(v);
        hi[kk] = h;
        lo[kk] = __float2half_rn(__fsub_rn(v, __half2float(h)));
    };
    k = threadIdx.x;
    for (; k + 768 < K; k += 1024) {
        float v[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) v[i] = value(k + 256 * i);
#pragma unroll
        for (int i = 0; i < 4; ++i) put(k + 256 * i, v[i]);
    }
    for (; k < K; k += 256) put(k, value(k));
}

// ---------------------------------------------------------------------------
template <int BN_>
__global__ void __launch_bounds__(tc::HXCfg<BN_>::THREADS, 1) gfb_conv_tcxh_kernel(const __grid_constant__ gfb_tcxh_args p) {
    using namespace tc;
    using C_ = HXCfg<BN_>;
    constexpr int BN = C_::BN, BK = C_::BK, STAGES = C_::STAGES, NBUF = C_::NBUF;
    constexpr int A_BYTES = C_::A_BYTES, B_BYTES = C_::B_BYTES, STAGE_BYTES = C_::STAGE_BYTES;
    constexpr int CHUNK_KB = C_::CHUNK_KB, EPI_WARPS = C_::EPI_WARPS;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + NBUF;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + NBUF);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nk = (int)(p.K / BK);
    const int nchunk = (nk + CHUNK_KB - 1) / CHUNK_KB;
    const int ntn = (int)((p.N + BN - 1) / BN);
    const int npix = p.tiles_x * p.tiles_y * ((p.No + p.BNI - 1) / p.BNI);
    const int nitems = ntn * npix;
    struct Item {
        int x0, y0, n0, col0;
    };
    auto item_at = [&](int it) {
        Item r;
        const int tile = it / ntn;
        const int tx = tile % p.tiles_x, ty = (tile / p.tiles_x) % p.tiles_y, tn = tile / (p.tiles_x * p.tiles_y);
        r.x0 = tx * p.BX;
        r.y0 = ty * p.BY;
        r.n0 = tn * p.BNI;
        r.col0 = (it % ntn) * BN;
        return r;
    };

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < NBUF; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], EPI_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int i = 0; i < 4; ++i) prefetch_tmap(p.tmap[i]);
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                     "r"(C_::TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            uint32_t gk = 0;
            for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
                const Item I = item_at(it);
                int cb = 0, r = 0, s_ = 0;
                for (int kb = 0; kb < nk; ++kb, ++gk) {
                    const int s = gk % STAGES;
                    mbar_wait(&empty[s], ((gk / STAGES) & 1) ^ 1);
                    unsigned char* st = smem + s * STAGE_BYTES;
                    mbar_expect_tx(&full[s], STAGE_BYTES);
                    const int cx = I.x0 * p.sx + p.ox + p.ksign * s_, cy = I.y0 * p.sy + p.oy + p.ksign * r;
                    tma_load_4d(st, p.tmap[0], cb * 64, cx, cy, I.n0, &full[s]);
                    tma_load_4d(st + A_BYTES, p.tmap[1], cb * 64, cx, cy, I.n0, &full[s]);
                    tma_load_2d(st + 2 * A_BYTES, p.tmap[2], kb * BK, I.col0, &full[s]);
                    tma_load_2d(st + 2 * A_BYTES + B_BYTES, p.tmap[3], kb * BK, I.col0, &full[s]);
                    if (++cb == p.CB) {  // k = (r, s, c): channel blocks fastest
                        cb = 0;
                        if (++s_ == p.S) {
                            s_ = 0;
                            ++r;
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_f16(128, BN);
            uint32_t gk = 0, gc = 0;
            for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
                for (int i = 0; i < nk; ++i, ++gk) {
                    const int s = gk % STAGES;
                    const uint32_t chunk = gc + i / CHUNK_KB;
                    const int b = chunk % NBUF;
                    const bool chunk_start = i % CHUNK_KB == 0;
                    if (chunk_start) {
                        mbar_wait(&tempty[b], ((chunk / NBUF) & 1) ^ 1);
                        asm volatile("tcgen05.fence::after_thread_sync;");
                    }
                    mbar_wait(&full[s], (gk / STAGES) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    unsigned char* st = smem + s * STAGE_BYTES;
                    const uint64_t ah = smem_desc(st), al = smem_desc(st + A_BYTES);
                    const uint64_t bh = smem_desc(st + 2 * A_BYTES), bl = smem_desc(st + 2 * A_BYTES + B_BYTES);
                    const uint32_t d = tmem + (uint32_t)(b * BN);
#pragma unroll
                    for (int j = 0; j < BK / 16; ++j) {
                        const uint64_t adv = (uint64_t)(j * 32) >> 4;  // 16 fp16 = 32 B along K
                        const uint32_t acc = !(chunk_start && j == 0);
                        mma_f16_cta(d, ah + adv, bh + adv, idesc, acc);
                        mma_f16_cta(d, ah + adv, bl + adv, idesc, 1);
                        mma_f16_cta(d, al + adv, bh + adv, idesc, 1);
                    }
                    mma_commit(&empty[s]);
                    if (i % CHUNK_KB == CHUNK_KB - 1 || i == nk - 1) mma_commit(&tfull[b]);
                }
                gc += nchunk;
            }
        }
    } else {
        constexpr int EC = BN < 128 ? BN : 128;
        const int q = warp & 3;
        uint32_t gc = 0;
        float* C = resolve<float>(p.tab, p.c);
        const float* inv = resolve<const float>(p.tab, p.b_inv);
        for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
            const Item I = item_at(it);
            float acc[EC];
#pragma unroll
            for (int j = 0; j < EC; ++j) acc[j] = 0.0f;
            for (int c0 = 0; c0 < nchunk; ++c0) {
                const uint32_t chunk = gc + c0;
                const int b = chunk % NBUF;
                mbar_wait(&tfull[b], (chunk / NBUF) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
                for (int c = 0; c < EC / 16; ++c) {
                    float v[16];
                    tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * BN + c * 16), v);
#pragma unroll
                    for (int j = 0; j < 16; ++j) acc[c * 16 + j] = __fadd_rn(acc[c * 16 + j], v[j]);
                }
                asm volatile("tcgen05.fence::before_thread_sync;");
                __syncwarp();
                if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&tempty[b])) : "memory");
            }
            gc += nchunk;
            const BoxRows rows{I.n0, I.y0, I.x0, p.BX, p.BY, p.No, p.Yo, p.Xo, p.o_n, p.o_y, p.o_x};
            const int64_t roff = rows(q * 32 + lane);
            if (roff >= 0) {
                float* dst = C + roff;
#pragma unroll
                for (int c = 0; c < EC / 32; ++c) {
                    const int col0 = I.col0 + c * 32;
                    if (p.c_sn == 1 && col0 + 32 <= p.N && ((reinterpret_cast<uintptr_t>(dst + col0) & 15) == 0)) {
#pragma unroll
                        for (int j = 0; j < 32; j += 4) {
                            const float4 f = __ldg(reinterpret_cast<const float4*>(inv + col0 + j));
                            *reinterpret_cast<float4*>(dst + col0 + j) =
                                make_float4(__fmul_rn(acc[c * 32 + j], f.x), __fmul_rn(acc[c * 32 + j + 1], f.y),
                                            __fmul_rn(acc[c * 32 + j + 2], f.z), __fmul_rn(acc[c * 32 + j + 3], f.w));
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (col0 + j < p.N) dst[(int64_t)(col0 + j) * p.c_sn] = __fmul_rn(acc[c * 32 + j], __ldg(inv + col0 + j));
                    }
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C_::TMEM_COLS));
    }
}

template __global__ void gfb_conv_tcxh_kernel<64>(const __grid_constant__ gfb_tcxh_args);
template __global__ void gfb_conv_tcxh_kernel<128>(const __grid_constant__ gfb_tcxh_args);

// ---------------------------------------------------------------------------
// Weight gradient (gfb_tcgwh_args): rows (r, s, c), columns dy's channels,
// contraction over 64-pixel boxes.  Stage = [A hi | A lo | B hi | B lo], A as
// two 64-channel x boxes (8 KB each: 64 pixels x 128 B, the canonical
// SWIZZLE_128B MN-major layout), B as one or two dy boxes.
namespace tc {
template <int BN_>
struct HWCfg {
    static constexpr int BM = 128, BN = BN_, BKP = 64;  // pixels per stage
    static constexpr int BOX_BYTES = 64 * BKP * 2;       // 64 channels x 64 pixels fp16
    static constexpr int A_BYTES = 2 * BOX_BYTES, B_BYTES = (BN / 64) * BOX_BYTES;
    static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
    static constexpr int STAGES = BN_ == 128 ? 3 : 4;
    static constexpr int CHUNK_KB = 2, NBUF = 512 / BN;
    static constexpr uint32_t TMEM_COLS = 512;
    static constexpr int EPI_WARPS = 4;
    static constexpr int THREADS = 64 + 32 * EPI_WARPS;
    static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 256 + 1024;
};
}  // namespace tc

template <int BN_>
__global__ void __launch_bounds__(tc::HWCfg<BN_>::THREADS, 1) gfb_conv_tcgwh_kernel(const __grid_constant__ gfb_tcgwh_args p) {
    using namespace tc;
    using C_ = HWCfg<BN_>;
    constexpr int BN = C_::BN, STAGES = C_::STAGES, NBUF = C_::NBUF, BOX = C_::BOX_BYTES;
    constexpr int A_BYTES = C_::A_BYTES, B_BYTES = C_::B_BYTES, STAGE_BYTES = C_::STAGE_BYTES;
    constexpr int CHUNK_KB = C_::CHUNK_KB, EPI_WARPS = C_::EPI_WARPS;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + NBUF;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + NBUF);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ntm = (int)((p.M + 127) / 128), ntn = (int)((p.N + BN - 1) / BN);
    const int nbox = p.tiles_x * p.tiles_y * ((p.No + p.BNI - 1) / p.BNI);
    const int splits = p.k_splits > 1 ? (int)p.k_splits : 1;
    const int nitems = ntm * ntn * splits;
    struct Item {
        int mt, nt, z, b0, nk;
    };
    auto item_at = [&](int it) {
        Item r;
        r.mt = it % ntm;
        r.nt = (it / ntm) % ntn;
        r.z = it / (ntm * ntn);
        r.b0 = splits > 1 ? r.z * (int)p.boxes_per_split : 0;
        const int b1 = splits > 1 ? min(nbox, r.b0 + (int)p.boxes_per_split) : nbox;
        r.nk = max(0, b1 - r.b0);
        return r;
    };

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < NBUF; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], EPI_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int i = 0; i < 4; ++i) prefetch_tmap(p.tmap[i]);
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                     "r"(C_::TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            uint32_t gk = 0;
            for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
                const Item I = item_at(it);
                // the two 64-row halves of the A tile: tap and first channel of each
                int acx[2], acy[2], acc_[2];
                bool aok[2];
                for (int j = 0; j < 2; ++j) {
                    const int64_t row = (int64_t)I.mt * 128 + 64 * j;
                    aok[j] = row < p.M;
                    const int tap = (int)(row / p.C);
                    acc_[j] = (int)(row % p.C);
                    acx[j] = (int)(tap % p.S) - (int)p.pl;
                    acy[j] = (int)(tap / p.S) - (int)p.pt;
                }
                uint32_t bytes = 0;
                for (int j = 0; j < 2; ++j) bytes += aok[j] ? 2 * BOX : 0;
                for (int jj = 0; jj < BN / 64; ++jj) bytes += (I.nt * BN + 64 * jj < p.N) ? 2 * BOX : 0;
                for (int kb = 0; kb < I.nk; ++kb, ++gk) {
                    const int s = gk % STAGES;
                    mbar_wait(&empty[s], ((gk / STAGES) & 1) ^ 1);
                    unsigned char* st = smem + s * STAGE_BYTES;
                    mbar_expect_tx(&full[s], bytes);
                    const int box = I.b0 + kb;
                    const int tx = box % p.tiles_x, ty = (box / p.tiles_x) % p.tiles_y, tn = box / (p.tiles_x * p.tiles_y);
                    const int x0 = tx * p.BX, y0 = ty * p.BY, n0 = tn * p.BNI;
                    for (int j = 0; j < 2; ++j) {
                        if (!aok[j]) continue;
                        tma_load_4d(st + j * BOX, p.tmap[0], acc_[j], x0 + acx[j], y0 + acy[j], n0, &full[s]);
                        tma_load_4d(st + A_BYTES + j * BOX, p.tmap[1], acc_[j], x0 + acx[j], y0 + acy[j], n0, &full[s]);
                    }
                    for (int jj = 0; jj < BN / 64; ++jj) {
                        const int kc = I.nt * BN + 64 * jj;
                        if (kc >= p.N) continue;
                        tma_load_4d(st + 2 * A_BYTES + jj * BOX, p.tmap[2], kc, x0, y0, n0, &full[s]);
                        tma_load_4d(st + 2 * A_BYTES + B_BYTES + jj * BOX, p.tmap[3], kc, x0, y0, n0, &full[s]);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_f16(128, BN) | (1u << 15) | (1u << 16);  // MN-major A and B
            uint32_t gk = 0, gc = 0;
            for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
                const Item I = item_at(it);
                for (int i = 0; i < I.nk; ++i, ++gk) {
                    const int s = gk % STAGES;
                    const uint32_t chunk = gc + i / CHUNK_KB;
                    const int b = chunk % NBUF;
                    const bool chunk_start = i % CHUNK_KB == 0;
                    if (chunk_start) {
                        mbar_wait(&tempty[b], ((chunk / NBUF) & 1) ^ 1);
                        asm volatile("tcgen05.fence::after_thread_sync;");
                    }
                    mbar_wait(&full[s], (gk / STAGES) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    const uint32_t sa = su32(smem + s * STAGE_BYTES), sb = sa + 2 * A_BYTES;
                    const uint32_t d = tmem + (uint32_t)(b * BN);
#pragma unroll
                    for (int j = 0; j < C_::BKP / 16; ++j) {
                        // 16 pixels (K rows) = two 1 KB atoms; 64-channel MN chunks one box apart
                        const uint32_t acc = !(chunk_start && j == 0);
                        const uint64_t ah = smem_desc_mn16(sa + j * 2048, BOX), al = smem_desc_mn16(sa + A_BYTES + j * 2048, BOX);
                        const uint64_t bh = smem_desc_mn16(sb + j * 2048, BOX), bl = smem_desc_mn16(sb + B_BYTES + j * 2048, BOX);
                        mma_f16_cta(d, ah, bh, idesc, acc);
                        mma_f16_cta(d, ah, bl, idesc, 1);
                        mma_f16_cta(d, al, bh, idesc, 1);
                    }
                    mma_commit(&empty[s]);
                    if (i % CHUNK_KB == CHUNK_KB - 1 || i == I.nk - 1) mma_commit(&tfull[b]);
                }
                gc += (I.nk + CHUNK_KB - 1) / CHUNK_KB;
            }
        }
    } else {
        constexpr int EC = BN;
        const int q = warp & 3;
        uint32_t gc = 0;
        const float* asc = resolve<const float>(p.tab, p.a_sc);
        const float* bsc = resolve<const float>(p.tab, p.b_sc);
        for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
            const Item I = item_at(it);
            const int nchunk = (I.nk + CHUNK_KB - 1) / CHUNK_KB;
            float acc[EC];
#pragma unroll
            for (int j = 0; j < EC; ++j) acc[j] = 0.0f;
            for (int c0 = 0; c0 < nchunk; ++c0) {
                const uint32_t chunk = gc + c0;
                const int b = chunk % NBUF;
                mbar_wait(&tfull[b], (chunk / NBUF) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
                for (int c = 0; c < EC / 16; ++c) {
                    float v[16];
                    tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * BN + c * 16), v);
#pragma unroll
                    for (int j = 0; j < 16; ++j) acc[c * 16 + j] = __fadd_rn(acc[c * 16 + j], v[j]);
                }
                asm volatile("tcgen05.fence::before_thread_sync;");
                __syncwarp();
                if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&tempty[b])) : "memory");
            }
            gc += nchunk;
            const int64_t row = (int64_t)I.mt * 128 + q * 32 + lane;
            if (row >= p.M) continue;
            const float ia = __frcp_rn(__ldg(asc + row % p.C));
            const int col0 = I.nt * BN;
            if (splits > 1) {
                float* dst = resolve<float>(p.tab, p.c) + (int64_t)I.z * p.split_stride + row * p.N;
#pragma unroll
                for (int j = 0; j < EC; j += 4) {
                    if (col0 + j >= p.N) break;
                    const float4 f = __ldg(reinterpret_cast<const float4*>(bsc + col0 + j));
                    *reinterpret_cast<float4*>(dst + col0 + j) =
                        make_float4(__fmul_rn(__fmul_rn(acc[j], ia), __frcp_rn(f.x)), __fmul_rn(__fmul_rn(acc[j + 1], ia), __frcp_rn(f.y)),
                                    __fmul_rn(__fmul_rn(acc[j + 2], ia), __frcp_rn(f.z)), __fmul_rn(__fmul_rn(acc[j + 3], ia), __frcp_rn(f.w)));
                }
            } else {
                float* dst = resolve<float>(p.tab, p.c) + (row / p.C) * p.c_s_hi + (row % p.C) * p.c_s_lo;
#pragma unroll
                for (int j = 0; j < EC; ++j)
                    if (col0 + j < p.N)
                        dst[(int64_t)(col0 + j) * p.c_sn] = __fmul_rn(__fmul_rn(acc[j], ia), __frcp_rn(__ldg(bsc + col0 + j)));
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C_::TMEM_COLS));
    }
}

template __global__ void gfb_conv_tcgwh_kernel<64>(const __grid_constant__ gfb_tcgwh_args);
template __global__ void gfb_conv_tcgwh_kernel<128>(const __grid_constant__ gfb_tcgwh_args);

}  // namespace gfb

extern "C" const void* gfb_conv_f16_kernel_ptr(int kind) {
    if (kind == GFB_K_CHMAX) return (const void*)gfb::gfb_chmax_kernel;
    if (kind == GFB_K_CHSPLIT) return (const void*)gfb::gfb_chsplit_kernel;
    if (kind == GFB_K_FSPLIT) return (const void*)gfb::gfb_fsplit_kernel;
    if (kind == GFB_K_CONV_TCXH64) return (const void*)gfb::gfb_conv_tcxh_kernel<64>;
    if (kind == GFB_K_CONV_TCXH128) return (const void*)gfb::gfb_conv_tcxh_kernel<128>;
    if (kind == GFB_K_CONV_TCGWH64) return (const void*)gfb::gfb_conv_tcgwh_kernel<64>;
    if (kind == GFB_K_CONV_TCGWH128) return (const void*)gfb::gfb_conv_tcgwh_kernel<128>;
    return nullptr;
}
extern "C" int gfb_tcgwh_smem_bytes(int bn) { return bn == 64 ? gfb::tc::HWCfg<64>::SMEM_BYTES : gfb::tc::HWCfg<128>::SMEM_BYTES; }
extern "C" int gfb_tcxh_smem_bytes(int bn) { return bn == 64 ? gfb::tc::HXCfg<64>::SMEM_BYTES : gfb::tc::HXCfg<128>::SMEM_BYTES; }
