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
    unsigned char* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);  // stays a shared-space pointer
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
    unsigned char* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);  // stays a shared-space pointer
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

// ---------------------------------------------------------------------------
// Few-channel forward convolution (the 3-channel ResNet stem) in 2xFP16
// (gfb_stemh_args): the tile walk and shared-memory input patch of
// gemm_tc.cu's gfb_conv_stem_kernel, on kind::f16.  The K = R S C <= 192
// columns (r, s, c) are one to three 64-wide K-blocks; a K-block issues only
// the 16-wide K-steps below K.  Scales, all exact powers of two:
//   * activation: one per 128-pixel tile, u = 2^(14 - floor(log2 m)), m the
//     largest finite |x| of the tile's input patch (computed while the patch
//     is staged, no extra pass); the patch is parked as fp16 hi / lo words
//     of x u, from which the builders assemble A;
//   * filter: one per output channel, t_n from the row's largest finite |w|;
//     every CTA splits the (tiny) filter into resident SW128 hi / lo planes
//     in its prologue.
//   y[p, n] = ((sum_k AhBh + AhBl + AlBh) / u) / t_n
// Warp roles: 1 TMEM + MMA issuer, 2..5 epilogue, 6..13 patch + A builders.
namespace tc {
struct HSCfg {
    static constexpr int BM = 128, BN = 64, BK = 64, TH = 4, TW = 32;
    static constexpr int MAXKB = 3;  // K <= 192 (the filter stays resident)
    static constexpr int STAGES = 4;
    static constexpr int A_BYTES = BM * BK * 2, B_BYTES = BN * BK * 2;
    static constexpr int STAGE_BYTES = 2 * A_BYTES;
    static constexpr int BRES_BYTES = MAXKB * 2 * B_BYTES;
    static constexpr int PATCH_FLOATS = 1536;  // (4 + R - 1)(32 + S - 1) C + zero pad <= 1536
    static constexpr int OUT_BYTES = 4 * 32 * BN * 4;  // per epilogue warp: one 32-pixel row of the tile
    static constexpr int NBUF = 8, RING = 2 * NBUF;
    static constexpr uint32_t TMEM_COLS = 512;
    static constexpr int EPI_WARPS = 4, LOAD_WARPS = 8;
    static constexpr int THREADS = 64 + 32 * (EPI_WARPS + LOAD_WARPS);
    static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + BRES_BYTES + OUT_BYTES + 2 * PATCH_FLOATS * 4 + MAXKB * BK * 4 +
                                      (RING + BN + 2 * LOAD_WARPS) * 4 + 256 + 1024;
};
}  // namespace tc

// patch word offset of K index k = (r, s, c) (c fastest) in the [c][py][px]
// patch; k >= K: the zero pad
__host__ __device__ constexpr int stemh_off(int C, int R, int S, int PH, int PW, int k) {
    return k < C * R * S ? ((k % C) * PH + (k / C) / S) * PW + (k / C) % S : PH * PW * C;
}

// One tile's A blocks for a compile-time (C, R, S): every gather offset is an
// immediate (LDS [row + imm]), no offset table.  Thread half HF of row m.
template <int CC, int RR, int SS, int HF>
__device__ __forceinline__ void stemh_build(unsigned char* smem, const uint32_t* prow, uint32_t& gk, uint64_t* empty,
                                            uint64_t* full, int m, int rsw, int lane) {
    using C_ = tc::HSCfg;
    constexpr int K_ = CC * RR * SS, NK = (K_ + C_::BK - 1) / C_::BK;
    constexpr int PH_ = C_::TH + RR - 1, PW_ = C_::TW + SS - 1;
    static_assert(NK <= C_::MAXKB, "K <= 192");
#pragma unroll
    for (int kb = 0; kb < NK; ++kb, ++gk) {
        const int s = gk % C_::STAGES;
        tc::mbar_wait(&empty[s], ((gk / C_::STAGES) & 1) ^ 1);
        unsigned char* st = smem + s * C_::STAGE_BYTES + m * 128;
        const int ks = (K_ - kb * C_::BK + 15) / 16 < 4 ? (K_ - kb * C_::BK + 15) / 16 : 4;
        uint32_t e[32];
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
            if (jj < ks) {
#pragma unroll
                for (int q = 0; q < 8; ++q) e[8 * jj + q] = prow[stemh_off(CC, RR, SS, PH_, PW_, kb * C_::BK + 8 * (HF * ks + jj) + q)];
            }
        }
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
            if (jj < ks) {
                const uint32_t* q = e + 8 * jj;
                const int o = (((HF * ks + jj) ^ rsw) << 4);
                *reinterpret_cast<uint4*>(st + o) = make_uint4(__byte_perm(q[0], q[1], 0x5410), __byte_perm(q[2], q[3], 0x5410),
                                                               __byte_perm(q[4], q[5], 0x5410), __byte_perm(q[6], q[7], 0x5410));
                *reinterpret_cast<uint4*>(st + C_::A_BYTES + o) = make_uint4(
                    __byte_perm(q[0], q[1], 0x7632), __byte_perm(q[2], q[3], 0x7632), __byte_perm(q[4], q[5], 0x7632),
                    __byte_perm(q[6], q[7], 0x7632));
            }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::su32(&full[s])) : "memory");
    }
}

// CC > 0: specialised for that (C, R, S) (the 3-channel 7x7 stem); 0: any
template <int CC, int RR, int SS>
__global__ void __launch_bounds__(tc::HSCfg::THREADS, 1) gfb_conv_stemh_kernel(const __grid_constant__ gfb_stemh_args p) {
    using namespace tc;
    using C_ = HSCfg;
    constexpr int BN = C_::BN, BK = C_::BK, TH = C_::TH, TW = C_::TW, STAGES = C_::STAGES, NBUF = C_::NBUF;
    constexpr int RING = C_::RING, A_BYTES = C_::A_BYTES, B_BYTES = C_::B_BYTES, STAGE_BYTES = C_::STAGE_BYTES;
    constexpr int EPI_WARPS = C_::EPI_WARPS, LW = C_::LOAD_WARPS;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // (offset from the __shared__ array itself, so every derived pointer stays a
    // shared-space pointer: LDS / STS, not generic loads)
    unsigned char* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
    unsigned char* bres = smem + STAGES * STAGE_BYTES;  // K-block kb: hi at kb * 2 * B_BYTES, lo after it
    unsigned char* ostage = bres + C_::BRES_BYTES;                     // epilogue staging
    float* patch = reinterpret_cast<float*>(ostage + C_::OUT_BYTES);  // two buffers of PATCH_FLOATS
    int* ktab = reinterpret_cast<int*>(patch + 2 * C_::PATCH_FLOATS);  // patch offset of every k
    float* iu = reinterpret_cast<float*>(ktab + C_::MAXKB * BK);       // 1 / u of tile gt at gt % RING
    float* invt = iu + RING;                                           // 1 / t_n
    float* wmax = invt + BN;                                           // per loader warp patch maxima
    uint64_t* full = reinterpret_cast<uint64_t*>(wmax + 2 * LW);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + NBUF;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + NBUF);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int K = (int)p.K, nk = (K + BK - 1) / BK;
    const int Cc = p.C, S = p.S, R = K / (Cc * S);
    const int PH = TH + R - 1, PW = TW + S - 1, PSZ = PH * PW * Cc;
    const int tiles_x = (p.X + TW - 1) / TW, tiles_y = (p.Y + TH - 1) / TH;
    const int nitems = (int)(p.M / ((int64_t)p.Y * p.X)) * tiles_y * tiles_x;  // M = N * Y * X

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], LW);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < NBUF; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], EPI_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                     "r"(C_::TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    // K -> patch offset table: k = (r, s, c), c fastest; patch layout [c][py][px]
    for (int k = threadIdx.x; k < C_::MAXKB * BK; k += blockDim.x) {
        int off = PSZ;  // k >= K: the zero pad (PSZ + (TH - 1) PW + TW <= PATCH_FLOATS)
        if (k < K) {
            const int tap = k / Cc, c = k - tap * Cc, r = tap / S, s = tap - r * S;
            off = (c * PH + r) * PW + s;
        }
        ktab[k] = off;
    }
    // the filter: row n's scale t_n, then its fp16 hi / lo pieces in the SW128
    // K-major layout (row n at n * 128 B, 16-byte chunk j at (j ^ (n & 7)) * 16)
    {
        const float* w = resolve<const float>(p.tab, p.w);
        auto wv = [&](int n, int k) {
            if (n >= p.N || k >= K) return 0.0f;
            const int tap = k / Cc, c = k - tap * Cc, r = tap / S, s = tap - r * S;
            return __ldg(w + n * p.ws0 + c * p.ws1 + r * p.ws2 + s * p.ws3);
        };
        for (int n = warp; n < BN; n += C_::THREADS / 32) {
            float m = 0.0f;
            for (int k = lane; k < K; k += 32) m = fmaxf(m, fin_abs(wv(n, k)));
#pragma unroll
            for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
            const float t = f16_tile_scale(m);
            if (lane == 0) invt[n] = __frcp_rn(t);
            for (int k = lane; k < nk * BK; k += 32) {
                const float v = __fmul_rn(wv(n, k), t);
                const __half h = __float2half_rn(v), l = __float2half_rn(__fsub_rn(v, __half2float(h)));
                const int kb = k / BK, kk = k - kb * BK;
                const int off = kb * 2 * B_BYTES + n * 128 + ((((kk >> 3) ^ (n & 7))) << 4) + (kk & 7) * 2;
                *reinterpret_cast<__half*>(bres + off) = h;
                *reinterpret_cast<__half*>(bres + off + B_BYTES) = l;
            }
        }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;

    // item -> (image, tile row, tile column) with float-reciprocal divisions
    // (item indices < 2^24 are exact in float; one correction step each)
    const float inv_tx = 1.0f / (float)tiles_x, inv_ty = 1.0f / (float)tiles_y;
    auto divmod = [](int a, int d, float inv, int& q) {
        q = (int)((float)a * inv);
        if (q * d > a) --q;
        else if ((q + 1) * d <= a) ++q;
        return a - q * d;
    };
    auto item_at = [&](int it, int& n, int& y0, int& x0) {
        int t;
        const int tx = divmod(it, tiles_x, inv_tx, t);
        const int ty = divmod(t, tiles_y, inv_ty, n);
        y0 = ty * TH;
        x0 = tx * TW;
    };

    if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_f16(128, BN);
            uint32_t gk = 0, gt = 0;
            for (int it = blockIdx.x; it < nitems; it += gridDim.x, ++gt) {
                const int b = gt % NBUF;
                mbar_wait(&tempty[b], ((gt / NBUF) & 1) ^ 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t d = tmem + (uint32_t)(b * BN);
                for (int kb = 0; kb < nk; ++kb, ++gk) {
                    const int s = gk % STAGES;
                    mbar_wait(&full[s], (gk / STAGES) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    unsigned char* st = smem + s * STAGE_BYTES;
                    const uint64_t ah = smem_desc(st), al = smem_desc(st + A_BYTES);
                    const uint64_t bh = smem_desc(bres + kb * 2 * B_BYTES), bl = smem_desc(bres + kb * 2 * B_BYTES + B_BYTES);
                    const int ks = min(4, (K - kb * BK + 15) / 16);
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        if (j < ks) {
                            const uint64_t adv = (uint64_t)(j * 32) >> 4;  // 16 fp16 = 32 B along K
                            const uint32_t acc = !(kb == 0 && j == 0);
                            mma_f16_cta(d, ah + adv, bh + adv, idesc, acc);
                            mma_f16_cta(d, ah + adv, bl + adv, idesc, 1);
                            mma_f16_cta(d, al + adv, bh + adv, idesc, 1);
                        }
                    }
                    mma_commit(&empty[s]);
                }
                mma_commit(&tfull[b]);
            }
        }
    } else if (warp >= 2 && warp < 2 + EPI_WARPS) {
        // warp q owns TMEM lanes 32q.. = tile row q (TW = 32 pixels).  Dense
        // channel-last output: the row's 32 x 64 values go through a swizzled
        // per-warp staging buffer and leave as 512-byte contiguous stores
        // (two whole pixels per instruction) instead of 16-byte pieces of 32
        // different pixels.
        static_assert(TW == 32, "one tile row per epilogue warp");
        const int q = warp & 3;
        float* C = resolve<float>(p.tab, p.c);
        float* C2 = (p.flags & 1) ? resolve<float>(p.tab, p.c2) : nullptr;  // Relu side output
        unsigned char* ost = ostage + q * (32 * BN * 4);
        const bool dense = p.c_sn == 1 && p.N == BN && p.c_s_lo == BN && p.c_sm % 4 == 0 && p.c_s_hi % 4 == 0 &&
                           (reinterpret_cast<uintptr_t>(C) & 15) == 0;
        uint32_t gt = 0;
        for (int it = blockIdx.x; it < nitems; it += gridDim.x, ++gt) {
            int n, y0, x0;
            item_at(it, n, y0, x0);
            const int b = gt % NBUF;
            mbar_wait(&tfull[b], (gt / NBUF) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            float acc[BN];
#pragma unroll
            for (int c = 0; c < BN / 16; ++c) tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * BN + c * 16), acc + c * 16);
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&tempty[b])) : "memory");
            const float f = iu[gt % RING];
            const int y = y0 + q;
            if (dense) {
#pragma unroll
                for (int j = 0; j < BN / 4; ++j)
                    *reinterpret_cast<float4*>(ost + lane * (BN * 4) + ((j ^ (lane & 7)) << 4)) =
                        make_float4(__fmul_rn(__fmul_rn(acc[4 * j], f), invt[4 * j]),
                                    __fmul_rn(__fmul_rn(acc[4 * j + 1], f), invt[4 * j + 1]),
                                    __fmul_rn(__fmul_rn(acc[4 * j + 2], f), invt[4 * j + 2]),
                                    __fmul_rn(__fmul_rn(acc[4 * j + 3], f), invt[4 * j + 3]));
                __syncwarp();
                if (y < p.Y) {
                    const int64_t ro = (int64_t)n * p.c_s_hi + (int64_t)y * p.c_sm;
                    const int quad = lane & 15;
#pragma unroll 4
                    for (int i2 = 0; i2 < 16; ++i2) {
                        const int pp = 2 * i2 + (lane >> 4), x = x0 + pp;
                        const float4 v = *reinterpret_cast<const float4*>(ost + pp * (BN * 4) + ((quad ^ (pp & 7)) << 4));
                        if (x < p.X) {
                            *reinterpret_cast<float4*>(C + ro + (int64_t)x * BN + quad * 4) = v;
                            if (C2)
                                *reinterpret_cast<float4*>(C2 + ro + (int64_t)x * BN + quad * 4) =
                                    make_float4(v.x > 0.f ? v.x : 0.f, v.y > 0.f ? v.y : 0.f, v.z > 0.f ? v.z : 0.f, v.w > 0.f ? v.w : 0.f);
                        }
                    }
                }
                __syncwarp();
            } else {
                const int x = x0 + lane;
                if (y < p.Y && x < p.X) {
                    const int64_t ro = (int64_t)n * p.c_s_hi + (int64_t)y * p.c_sm + (int64_t)x * p.c_s_lo;
#pragma unroll
                    for (int j = 0; j < BN; ++j) {
                        if (j < p.N) {
                            const float v = __fmul_rn(__fmul_rn(acc[j], f), invt[j]);
                            C[ro + (int64_t)j * p.c_sn] = v;
                            if (C2) C2[ro + (int64_t)j * p.c_sn] = v > 0.f ? v : 0.f;
                        }
                    }
                }
            }
        }
    } else if (warp >= 2 + EPI_WARPS) {
        // builders.  The next tile's input patch is loaded into registers
        // while this tile's A blocks are built; its largest finite |x| gives
        // the tile scale u, and the patch is parked already scaled and split:
        // one 32-bit word per element, fp16 hi in the low half, lo in the
        // high half.  A K-block chunk (8 consecutive k of one row) is then 8
        // word gathers and 8 byte permutes; k >= K points into a zero pad
        // after the patch.  Thread t builds row m = t & 127; of each K-block's
        // used 16-byte chunks (2 per 16-wide K-step) it takes half.
        const int t = threadIdx.x - (2 + EPI_WARPS) * 32;  // 0 .. 32 * LW - 1
        const int m = t & 127, hf = t >> 7, lw = t >> 5;
        const int py = m / TW, px = m % TW;
        const uint32_t rsw = (uint32_t)(m & 7);
        const float* X = resolve<const float>(p.tab, p.a);
        uint32_t* pw = reinterpret_cast<uint32_t*>(patch);
        constexpr int PPT = (C_::PATCH_FLOATS + 32 * LW - 1) / (32 * LW);  // patch elements per thread
        float pre[PPT];
        int pyy[PPT], pxx[PPT];
        int64_t poff[PPT];
#pragma unroll
        for (int u = 0; u < PPT; ++u) {
            const int i = t + u * 32 * LW;
            const int c = i / (PH * PW), rem = i - c * (PH * PW), yy = rem / PW, xx = rem - yy * PW;
            pyy[u] = i < PSZ ? yy + p.oy : -(1 << 28);
            pxx[u] = xx + p.ox;
            poff[u] = (int64_t)c * p.xs1 + (int64_t)(yy + p.oy) * p.xs2 + (int64_t)(xx + p.ox) * p.xs3;
        }
        // zero pads of both patch buffers (never overwritten)
        for (int i = PSZ + t; i < C_::PATCH_FLOATS; i += 32 * LW) pw[i] = pw[C_::PATCH_FLOATS + i] = 0u;
        auto fetch = [&](int it2) {
            int n2, ya, xa;
            item_at(it2, n2, ya, xa);
            const float* base = X + (int64_t)n2 * p.xs0 + (int64_t)ya * p.xs2 + (int64_t)xa * p.xs3;
#pragma unroll
            for (int u = 0; u < PPT; ++u) {
                const int h = ya + pyy[u], w = xa + pxx[u];
                pre[u] = ((uint32_t)h < (uint32_t)p.H && (uint32_t)w < (uint32_t)p.W) ? __ldg(base + poff[u]) : 0.0f;
            }
        };
        // the fetched patch's scale (two loader barriers) and its parked words;
        // thread 0 publishes 1 / u for tile gt2 before any arrive of that tile
        auto park = [&](uint32_t* pt, uint32_t gt2) {
            float mm = 0.0f;
#pragma unroll
            for (int u = 0; u < PPT; ++u) mm = fmaxf(mm, fin_abs(pre[u]));
#pragma unroll
            for (int o = 16; o; o >>= 1) mm = fmaxf(mm, __shfl_xor_sync(0xffffffffu, mm, o));
            if (lane == 0) wmax[lw] = mm;
            asm volatile("bar.sync 1, %0;" ::"n"(32 * LW) : "memory");
            float mx = wmax[0];
#pragma unroll
            for (int i = 1; i < LW; ++i) mx = fmaxf(mx, wmax[i]);
            const float u = f16_tile_scale(mx);
            if (t == 0) iu[gt2 % RING] = __frcp_rn(u);
#pragma unroll
            for (int q = 0; q < PPT; ++q) {
                if (t + q * 32 * LW < PSZ) {
                    const float v = __fmul_rn(pre[q], u);
                    const __half h = __float2half_rn(v), l = __float2half_rn(__fsub_rn(v, __half2float(h)));
                    pt[t + q * 32 * LW] = (uint32_t)__half_as_ushort(h) | ((uint32_t)__half_as_ushort(l) << 16);
                }
            }
        };
        if ((int)blockIdx.x < nitems) {
            fetch(blockIdx.x);
            park(pw, 0);
        }
        asm volatile("bar.sync 1, %0;" ::"n"(32 * LW) : "memory");
        uint32_t gk = 0, gt = 0;
        for (int it = blockIdx.x; it < nitems; it += gridDim.x, ++gt) {
            const bool more = it + (int)gridDim.x < nitems;
            if (more) fetch(it + gridDim.x);
            const uint32_t* prow = pw + (gt & 1) * C_::PATCH_FLOATS + py * PW + px;
            if constexpr (CC > 0) {
                if (hf == 0) stemh_build<CC, RR, SS, 0>(smem, prow, gk, empty, full, m, (int)rsw, lane);
                else stemh_build<CC, RR, SS, 1>(smem, prow, gk, empty, full, m, (int)rsw, lane);
            } else
            for (int kb = 0; kb < nk; ++kb, ++gk) {
                const int s = gk % STAGES;
                mbar_wait(&empty[s], ((gk / STAGES) & 1) ^ 1);
                unsigned char* st = smem + s * STAGE_BYTES + m * 128;
                const int ks = min(4, (K - kb * BK + 15) / 16);  // chunks 2 ks; this thread: [hf ks, hf ks + ks)
                // all offsets, then all gathers, then the permutes and stores (no
                // per-chunk load -> load -> store chain)
                int4 ko[8];
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    if (jj < ks) {
                        const int j = hf * ks + jj;
                        ko[2 * jj] = *reinterpret_cast<const int4*>(ktab + kb * BK + 8 * j);
                        ko[2 * jj + 1] = *reinterpret_cast<const int4*>(ktab + kb * BK + 8 * j + 4);
                    }
                }
                uint32_t e[32];
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    if (jj < ks) {
                        e[8 * jj + 0] = prow[ko[2 * jj].x];
                        e[8 * jj + 1] = prow[ko[2 * jj].y];
                        e[8 * jj + 2] = prow[ko[2 * jj].z];
                        e[8 * jj + 3] = prow[ko[2 * jj].w];
                        e[8 * jj + 4] = prow[ko[2 * jj + 1].x];
                        e[8 * jj + 5] = prow[ko[2 * jj + 1].y];
                        e[8 * jj + 6] = prow[ko[2 * jj + 1].z];
                        e[8 * jj + 7] = prow[ko[2 * jj + 1].w];
                    }
                }
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    if (jj < ks) {
                        const uint32_t* q = e + 8 * jj;
                        const int o = (((hf * ks + jj) ^ (int)rsw) << 4);
                        *reinterpret_cast<uint4*>(st + o) = make_uint4(__byte_perm(q[0], q[1], 0x5410), __byte_perm(q[2], q[3], 0x5410),
                                                                       __byte_perm(q[4], q[5], 0x5410), __byte_perm(q[6], q[7], 0x5410));
                        *reinterpret_cast<uint4*>(st + A_BYTES + o) =
                            make_uint4(__byte_perm(q[0], q[1], 0x7632), __byte_perm(q[2], q[3], 0x7632), __byte_perm(q[4], q[5], 0x7632),
                                       __byte_perm(q[6], q[7], 0x7632));
                    }
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&full[s])) : "memory");
            }
            // the other buffer's last readers (tile it - gridDim.x) passed the previous barrier
            if (more) park(pw + ((gt + 1) & 1) * C_::PATCH_FLOATS, gt + 1);
            asm volatile("bar.sync 1, %0;" ::"n"(32 * LW) : "memory");
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C_::TMEM_COLS));
    }
}


// ---------------------------------------------------------------------------
// Few-channel weight gradient in 2xFP16 (the 3-channel 7x7 stem's dW), the
// transpose of gfb_conv_stemh_kernel's product: rows k = (r, s, c) (M, two
// 128-row MMA tiles over K = C R S <= 192), columns the 64 output channels,
// contraction over the output pixels in 2 x 32 tiles (one 64-pixel stage
// each).  Per tile the builders stage the x patch (pre-split words, scale u)
// and dy's 64 x 64 block (scale v, split straight into the stage), then
// assemble the im2col block exactly as the forward does: the same bytes read
// as MN-major operands (pixel = K row of 128 B, k = M within it).  The
// tile's products carry u v, so each tile's accumulator is promoted into
// fp32 registers with one FFMA by 1 / (u v) (exact power of two).  CTA z
// walks a contiguous range of tiles and writes its partial dW[k, n] at
// c + z K N (the compiler adds the split reduction).  Arguments:
// gfb_stemh_args with w = dy, strides ws0..ws3 along (n, k_out, y, x) (k_out
// contiguous, ws1 = 1), (Y, X) = dy's (Ho, Wo), N = 64.
namespace tc {
struct HSWCfg {
    static constexpr int BN = 64, TH = 2, TW = 32, PIX = TH * TW;  // 64 pixels per stage
    static constexpr int MAXKB = 3;
    static constexpr int BLK = PIX * 128;                  // one 64-k block of one plane: 8 KB
    static constexpr int A_BYTES = MAXKB * BLK;            // per plane
    static constexpr int B_BYTES = PIX * 128;              // dy: 64 pixels x 64 channels fp16, per plane
    static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;  // 64 KB
    static constexpr int STAGES = 2;
    static constexpr int RAW = 4, RAW_BYTES = PIX * BN * 4;  // dy blocks in flight (cp.async), fp32: 3 tiles ahead
    static constexpr int PATCH_WORDS = 1024;               // (2 + R - 1)(32 + S - 1) C + zero pad
    static constexpr int NBUF = 4, RING = 16;              // TMEM: 4 x (2 M-tiles x 64 columns)
    static constexpr uint32_t TMEM_COLS = 512;
    static constexpr int EPI_WARPS = 8, LOAD_WARPS = 8;
    static constexpr int THREADS = 64 + 32 * (EPI_WARPS + LOAD_WARPS);
    static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + RAW * RAW_BYTES + RAW * PATCH_WORDS * 4 + 2 * PATCH_WORDS * 4 +
                                      (RING + 2 * LOAD_WARPS) * 4 + 256 + 1024;
};
}  // namespace tc

// Quarter HQ of one pixel row's im2col chunks (chunk c = k 8c .. 8c + 7, at
// K-block c / 8, slot c % 8), immediate gather offsets.
template <int CC, int RR, int SS, int HQ, int NQ>
__device__ __forceinline__ void stemwh_build(unsigned char* st, const uint32_t* prow, int rsw) {
    using C_ = tc::HSWCfg;
    constexpr int K_ = CC * RR * SS, NCH = 2 * ((K_ + 15) / 16), PER = (NCH + NQ - 1) / NQ;
    constexpr int PH = C_::TH + RR - 1, PW = C_::TW + SS - 1;
    uint32_t e[8 * PER];
#pragma unroll
    for (int cc = 0; cc < PER; ++cc) {
        const int c = HQ * PER + cc;
        if (c < NCH)
#pragma unroll
            for (int q = 0; q < 8; ++q) e[8 * cc + q] = prow[stemh_off(CC, RR, SS, PH, PW, 8 * c + q)];
    }
#pragma unroll
    for (int cc = 0; cc < PER; ++cc) {
        const int c = HQ * PER + cc;
        if (c < NCH) {
            const uint32_t* q = e + 8 * cc;
            const int o = (c / 8) * C_::BLK + (((c % 8) ^ rsw) << 4);
            *reinterpret_cast<uint4*>(st + o) = make_uint4(__byte_perm(q[0], q[1], 0x5410), __byte_perm(q[2], q[3], 0x5410),
                                                           __byte_perm(q[4], q[5], 0x5410), __byte_perm(q[6], q[7], 0x5410));
            *reinterpret_cast<uint4*>(st + C_::A_BYTES + o) = make_uint4(__byte_perm(q[0], q[1], 0x7632), __byte_perm(q[2], q[3], 0x7632),
                                                                         __byte_perm(q[4], q[5], 0x7632), __byte_perm(q[6], q[7], 0x7632));
        }
    }
}

template <int CC, int RR, int SS>
__global__ void __launch_bounds__(tc::HSWCfg::THREADS, 1) gfb_conv_stemwh_kernel(const __grid_constant__ gfb_stemh_args p) {
    using namespace tc;
    using C_ = HSWCfg;
    constexpr int BN = C_::BN, TH = C_::TH, TW = C_::TW, PIX = C_::PIX, STAGES = C_::STAGES, NBUF = C_::NBUF, RING = C_::RING;
    constexpr int BLK = C_::BLK, A_BYTES = C_::A_BYTES, B_BYTES = C_::B_BYTES, STAGE_BYTES = C_::STAGE_BYTES;
    constexpr int LW = C_::LOAD_WARPS, EPI_WARPS = C_::EPI_WARPS;
    constexpr int K_ = CC * RR * SS, NK = (K_ + 63) / 64;
    constexpr int PH = TH + RR - 1, PW = TW + SS - 1, PSZ = PH * PW * CC;
    static_assert(PSZ + (TH - 1) * PW + TW <= C_::PATCH_WORDS && NK <= C_::MAXKB, "stem shape");
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
    unsigned char* raw = smem + STAGES * STAGE_BYTES;                          // dy blocks, fp32 [64 px][64]
    float* rawp = reinterpret_cast<float*>(raw + C_::RAW * C_::RAW_BYTES);     // x patches in flight (cp.async)
    uint32_t* pw = reinterpret_cast<uint32_t*>(rawp + C_::RAW * C_::PATCH_WORDS);  // two parked patch buffers
    float* ifac = reinterpret_cast<float*>(pw + 2 * C_::PATCH_WORDS);         // 1 / (u v) of tile gt at gt % RING
    float* wmax = ifac + RING;                                                // [2][LW]: x and dy maxima
    uint64_t* full = reinterpret_cast<uint64_t*>(wmax + 2 * LW);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + NBUF;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + NBUF);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tiles_x = (p.X + TW - 1) / TW, tiles_y = (p.Y + TH - 1) / TH;
    const int ntiles = (int)(p.M / ((int64_t)p.Y * p.X)) * tiles_y * tiles_x;  // M = N * Y * X pixels
    const int per = (ntiles + (int)gridDim.x - 1) / (int)gridDim.x;
    const int t0 = min(ntiles, (int)blockIdx.x * per), t1 = min(ntiles, t0 + per);

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], LW);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < NBUF; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], EPI_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
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

    auto item_at = [&](int it, int& n, int& y0, int& x0) {
        const int tx = it % tiles_x, r = it / tiles_x, ty = r % tiles_y;
        n = r / tiles_y;
        y0 = ty * TH;
        x0 = tx * TW;
    };

    if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_f16(128, BN) | (1u << 15) | (1u << 16);  // MN-major A and B
            uint32_t g = 0;
            for (int it = t0; it < t1; ++it, ++g) {
                const int s = g % STAGES, b = g % NBUF;
                mbar_wait(&tempty[b], ((g / NBUF) & 1) ^ 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
                mbar_wait(&full[s], (g / STAGES) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t sa = su32(smem + s * STAGE_BYTES), sb = sa + 2 * A_BYTES;
#pragma unroll
                for (int mt = 0; mt < 2; ++mt) {
                    if (mt * 128 >= K_) continue;
                    const uint32_t d = tmem + (uint32_t)(b * 2 * BN + mt * BN);
#pragma unroll
                    for (int j = 0; j < PIX / 16; ++j) {
                        // 16 pixels (K rows) = two 1 KB atoms; the two 64-k M chunks one block apart
                        const uint64_t ah = smem_desc_mn16(sa + mt * 2 * BLK + j * 2048, BLK);
                        const uint64_t al = smem_desc_mn16(sa + A_BYTES + mt * 2 * BLK + j * 2048, BLK);
                        const uint64_t bh = smem_desc_mn16(sb + j * 2048, BLK), bl = smem_desc_mn16(sb + B_BYTES + j * 2048, BLK);
                        mma_f16_cta(d, ah, bh, idesc, j > 0);
                        mma_f16_cta(d, ah, bl, idesc, 1);
                        mma_f16_cta(d, al, bh, idesc, 1);
                    }
                }
                mma_commit(&empty[s]);
                mma_commit(&tfull[b]);
            }
        }
    } else if (warp >= 2 && warp < 2 + EPI_WARPS) {
        // warp w: TMEM lanes 32 (w & 3) .., M-tile (w - 2) / 4; 64 fp32 partials per thread
        const int q = warp & 3, mt = (warp - 2) >> 2;
        float acc[BN];
#pragma unroll
        for (int j = 0; j < BN; ++j) acc[j] = 0.0f;
        uint32_t g = 0;
        for (int it = t0; it < t1; ++it, ++g) {
            const int b = g % NBUF;
            mbar_wait(&tfull[b], (g / NBUF) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            const float f = ifac[g % RING];
            if (mt * 128 < K_) {
#pragma unroll
                for (int c = 0; c < BN / 16; ++c) {
                    float v[16];
                    tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * 2 * BN + mt * BN + c * 16), v);
#pragma unroll
                    for (int j = 0; j < 16; ++j) acc[c * 16 + j] = __fmaf_rn(v[j], f, acc[c * 16 + j]);
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&tempty[b])) : "memory");
        }
        const int row = mt * 128 + q * 32 + lane;
        if (row < K_) {
            float* dst = resolve<float>(p.tab, p.c) + ((int64_t)blockIdx.x * K_ + row) * BN;
#pragma unroll
            for (int j = 0; j < BN; j += 4) *reinterpret_cast<float4*>(dst + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
        }
    } else if (warp >= 2 + EPI_WARPS) {
        // builders: thread t takes pixel row m = t & 63 (a quarter hq of its
        // 16-byte chunks) for A, and 4 float4 of dy's 64 x 64 block for B
        const int t = threadIdx.x - (2 + EPI_WARPS) * 32;  // 0 .. 255
        const int m = t & 63, hq = t >> 6, lw = t >> 5;
        const int py = m / TW, px = m % TW;
        const int rsw = m & 7;
        const float* X = resolve<const float>(p.tab, p.a);
        const float* DY = resolve<const float>(p.tab, p.w);
        constexpr int PPT = (PSZ + 32 * LW - 1) / (32 * LW), DPT = PIX * 16 / (32 * LW);  // patch words, dy float4
        int pyy[PPT], pxx[PPT];
        int64_t poff[PPT];
#pragma unroll
        for (int u = 0; u < PPT; ++u) {
            const int i = t + u * 32 * LW;
            const int c = i / (PH * PW), rem = i - c * (PH * PW), yy = rem / PW, xx = rem - yy * PW;
            pyy[u] = i < PSZ ? yy + p.oy : -(1 << 28);
            pxx[u] = xx + p.ox;
            poff[u] = (int64_t)c * p.xs1 + (int64_t)(yy + p.oy) * p.xs2 + (int64_t)(xx + p.ox) * p.xs3;
        }
        for (int i = PSZ + t; i < C_::PATCH_WORDS; i += 32 * LW) pw[i] = pw[C_::PATCH_WORDS + i] = 0u;
        // dy block of tile g2 into raw buffer g2 % RAW with 16-byte cp.async
        // (zero-filled outside the image), one commit group per tile (empty
        // past the range, so the group count stays uniform): float4 i = t +
        // 128 u is pixel i / 16 of the tile, channels 4 (i % 16) ..
        auto issue = [&](uint32_t g2) {
            const int it2 = t0 + (int)g2;
            if (it2 < t1) {
                int n2, ya, xa;
                item_at(it2, n2, ya, xa);
                const uint32_t dst0 = su32(raw + (g2 % C_::RAW) * C_::RAW_BYTES);
                const float* base = X + (int64_t)n2 * p.xs0 + (int64_t)ya * p.xs2 + (int64_t)xa * p.xs3;
                const uint32_t dstp = su32(rawp + (g2 % C_::RAW) * C_::PATCH_WORDS);
#pragma unroll
                for (int u = 0; u < PPT; ++u) {
                    const int h = ya + pyy[u], w = xa + pxx[u];
                    const bool in = (uint32_t)h < (uint32_t)p.H && (uint32_t)w < (uint32_t)p.W;
                    if (t + u * 32 * LW < PSZ)
                        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dstp + (t + u * 32 * LW) * 4),
                                     "l"(in ? base + poff[u] : X), "r"(in ? 4 : 0)
                                     : "memory");
                }
#pragma unroll
                for (int u = 0; u < DPT; ++u) {
                    const int i = t + 32 * LW * u, pp = i >> 4, y = ya + pp / TW, x = xa + pp % TW;
                    const bool in = y < p.Y && x < p.X;
                    const float* src = in ? DY + (int64_t)n2 * p.ws0 + (int64_t)y * p.ws2 + (int64_t)x * p.ws3 + 4 * (i & 15) : DY;
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst0 + i * 16), "l"(src), "r"(in ? 16 : 0)
                                 : "memory");
                }
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
        // tile g2's scales (two loader barriers), its parked patch words, and
        // its dy block split into stage g2 % STAGES (acquired here)
        auto park = [&](uint32_t g2) {
            asm volatile("cp.async.wait_group %0;" ::"n"(C_::RAW - 2) : "memory");  // this thread's copies of tile g2 landed
            const float4* dr = reinterpret_cast<const float4*>(raw + (g2 % C_::RAW) * C_::RAW_BYTES);
            const float* xr = rawp + (g2 % C_::RAW) * C_::PATCH_WORDS;
            float pre[PPT];
#pragma unroll
            for (int u = 0; u < PPT; ++u) pre[u] = t + u * 32 * LW < PSZ ? xr[t + u * 32 * LW] : 0.0f;
            float mx = 0.0f, md = 0.0f;
#pragma unroll
            for (int u = 0; u < PPT; ++u) mx = fmaxf(mx, fin_abs(pre[u]));
#pragma unroll
            for (int u = 0; u < DPT; ++u) md = amax4(md, dr[t + 32 * LW * u]);
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                md = fmaxf(md, __shfl_xor_sync(0xffffffffu, md, o));
            }
            if (lane == 0) {
                wmax[lw] = mx;
                wmax[LW + lw] = md;
            }
            asm volatile("bar.sync 1, %0;" ::"n"(32 * LW) : "memory");
            mx = wmax[0];
            md = wmax[LW];
#pragma unroll
            for (int i = 1; i < LW; ++i) {
                mx = fmaxf(mx, wmax[i]);
                md = fmaxf(md, wmax[LW + i]);
            }
            const float u = f16_tile_scale(mx), v = f16_tile_scale(md);
            if (t == 0) ifac[g2 % RING] = __fmul_rn(__frcp_rn(u), __frcp_rn(v));
            uint32_t* pt = pw + (g2 & 1) * C_::PATCH_WORDS;
#pragma unroll
            for (int q2 = 0; q2 < PPT; ++q2) {
                if (t + q2 * 32 * LW < PSZ) {
                    const float x = __fmul_rn(pre[q2], u);
                    const __half h = __float2half_rn(x), l = __float2half_rn(__fsub_rn(x, __half2float(h)));
                    pt[t + q2 * 32 * LW] = (uint32_t)__half_as_ushort(h) | ((uint32_t)__half_as_ushort(l) << 16);
                }
            }
            const int s = g2 % STAGES;
            mbar_wait(&empty[s], ((g2 / STAGES) & 1) ^ 1);
            unsigned char* sb = smem + s * STAGE_BYTES + 2 * A_BYTES;
#pragma unroll
            for (int u2 = 0; u2 < DPT; ++u2) {
                const int i = t + 32 * LW * u2, pp = i >> 4, qd = i & 15;
                uint2 h, l;
                split4_f16(scale4(dr[i], v), h, l);
                const int o = pp * 128 + (((qd >> 1) ^ (pp & 7)) << 4) + (qd & 1) * 8;
                *reinterpret_cast<uint2*>(sb + o) = h;
                *reinterpret_cast<uint2*>(sb + B_BYTES + o) = l;
            }
        };
#pragma unroll
        for (int g2 = 0; g2 < C_::RAW - 1; ++g2) issue(g2);
        if (t0 < t1) park(0);
        asm volatile("bar.sync 1, %0;" ::"n"(32 * LW) : "memory");
        uint32_t g = 0;
        for (int it = t0; it < t1; ++it, ++g) {
            const bool more = it + 1 < t1;
            issue(g + C_::RAW - 1);  // raw buffers (g + RAW - 1) % RAW were last read by park(g - 1)
            const uint32_t* prow = pw + (g & 1) * C_::PATCH_WORDS + py * PW + px;
            const int s = g % STAGES;
            unsigned char* st = smem + s * STAGE_BYTES + m * 128;
            if (hq == 0) stemwh_build<CC, RR, SS, 0, 4>(st, prow, rsw);
            else if (hq == 1) stemwh_build<CC, RR, SS, 1, 4>(st, prow, rsw);
            else if (hq == 2) stemwh_build<CC, RR, SS, 2, 4>(st, prow, rsw);
            else stemwh_build<CC, RR, SS, 3, 4>(st, prow, rsw);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&full[s])) : "memory");
            if (more) park(g + 1);
            asm volatile("bar.sync 1, %0;" ::"n"(32 * LW) : "memory");
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C_::TMEM_COLS));
    }
}

template __global__ void gfb_conv_stemh_kernel<0, 0, 0>(const __grid_constant__ gfb_stemh_args);
template __global__ void gfb_conv_stemwh_kernel<3, 7, 7>(const __grid_constant__ gfb_stemh_args);
template __global__ void gfb_conv_stemh_kernel<3, 7, 7>(const __grid_constant__ gfb_stemh_args);

}  // namespace gfb

extern "C" const void* gfb_conv_f16_kernel_ptr(int kind) {
    if (kind == GFB_K_CHMAX) return (const void*)gfb::gfb_chmax_kernel;
    if (kind == GFB_K_CHSPLIT) return (const void*)gfb::gfb_chsplit_kernel;
    if (kind == GFB_K_FSPLIT) return (const void*)gfb::gfb_fsplit_kernel;
    if (kind == GFB_K_CONV_TCXH64) return (const void*)gfb::gfb_conv_tcxh_kernel<64>;
    if (kind == GFB_K_CONV_TCXH128) return (const void*)gfb::gfb_conv_tcxh_kernel<128>;
    if (kind == GFB_K_CONV_TCGWH64) return (const void*)gfb::gfb_conv_tcgwh_kernel<64>;
    if (kind == GFB_K_CONV_TCGWH128) return (const void*)gfb::gfb_conv_tcgwh_kernel<128>;
    if (kind == GFB_K_CONV_STEMH) return (const void*)gfb::gfb_conv_stemh_kernel<0, 0, 0>;
    if (kind == GFB_K_CONV_STEMH_C3R7) return (const void*)gfb::gfb_conv_stemh_kernel<3, 7, 7>;
    if (kind == GFB_K_CONV_STEMWH_C3R7) return (const void*)gfb::gfb_conv_stemwh_kernel<3, 7, 7>;
    return nullptr;
}
extern "C" int gfb_tcgwh_smem_bytes(int bn) { return bn == 64 ? gfb::tc::HWCfg<64>::SMEM_BYTES : gfb::tc::HWCfg<128>::SMEM_BYTES; }
extern "C" int gfb_stemh_smem_bytes(void) { return gfb::tc::HSCfg::SMEM_BYTES; }
extern "C" int gfb_stemwh_smem_bytes(void) { return gfb::tc::HSWCfg::SMEM_BYTES; }
extern "C" int gfb_tcxh_smem_bytes(int bn) { return bn == 64 ? gfb::tc::HXCfg<64>::SMEM_BYTES : gfb::tc::HXCfg<128>::SMEM_BYTES; }
