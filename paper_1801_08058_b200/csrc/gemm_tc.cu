// tcgen05 tensor-core Dot for F32 graphs (3xTF32), sm_100a.
//
// The reference Dot (kernels.py:123-133) is an f32 multiply-add chain.  A
// single TF32 product keeps 11 significant bits, which gives a normwise
// error of ~3e-4 on config A's shapes (SURVEY.md §7 hard part 1).  So every
// operand x is split as hi = rna_tf32(x), lo = rna_tf32(x - hi), and
//   C = Ahi*Bhi + Ahi*Blo + Alo*Bhi
// is accumulated by three tcgen05.mma kind::tf32 instructions per K-step
// into fp32 TMEM accumulators that are promoted into round-to-nearest fp32
// registers every 128 K (the tensor core's own accumulation truncates),
// which keeps the result well inside the 1e-5 normwise Dot tolerance of
// SURVEY.md §8(c).
//
// gfb_split_kernel writes the hi/lo planes in K-major layout into the
// arena.  Any operand strides are accepted, so autodiff's
// Reshape(x, (1, 0)) transposes fold into this pass.  The GEMM itself is
// one 128x128 output tile per CTA, 192 threads:
//   warp 0        TMA producer: 4 tensor-map loads per K-block (SW128) into a
//                 3-stage ring, completion on full[s] mbarriers
//   warp 1        TMEM allocator + single-thread MMA issuer; tcgen05.commit
//                 frees a stage (empty[s]) and marks an accumulator chunk done
//   warps 2..5    epilogue: tcgen05.ld 32x32b of each finished chunk, fp32
//                 register accumulation, then 128-bit stores to global
// Shared memory: 3 x (16 KB Ahi + 16 KB Alo + 16 KB Bhi + 16 KB Blo).

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "gfb_common.cuh"

namespace gfb {
namespace tc {

// Tile configurations.  BN = 128: 3-stage ring of 64 KB stages, 4 epilogue
// warps.  BN = 256: 2-stage ring of 96 KB stages, 8 epilogue warps; it moves
// 25 % fewer operand bytes per MMA clock, which the latency-bound 3xTF32
// pipeline needs (ncu: the 128-wide tile keeps the tensor pipe 65 % busy
// with L2 at 47 %).
template <int BN_>
struct Cfg {
    static constexpr int BM = 128, BN = BN_, BK = 32;
    static constexpr int STAGES = BN_ == 256 ? 2 : 3;
    static constexpr int A_BYTES = BM * BK * 4, B_BYTES = BN * BK * 4;
    static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
    static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;
    // The tensor core's fp32 accumulation truncates, so a 4096-deep K chain
    // drifts by ~3e-5.  Partial sums are promoted to CUDA-core fp32
    // registers (round-to-nearest adds) every CHUNK_KB K-blocks (128 K): the
    // MMA warp cycles through NBUF TMEM accumulators while the epilogue warps
    // drain finished ones, so the promotion overlaps the MMAs.
    static constexpr int CHUNK_KB = 4;
    static constexpr int NBUF = 512 / BN;
    static constexpr uint32_t TMEM_COLS = 512;
    static constexpr int EPI_WARPS = 4 * (BN / 128);  // each owns 32 rows x 128 columns
    static constexpr int THREADS = 64 + 32 * EPI_WARPS;
};

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

}  // namespace tc

template <int BN_>
__global__ void __launch_bounds__(tc::Cfg<BN_>::THREADS, 1) gfb_gemm_tc_kernel(const __grid_constant__ gfb_tc_args p) {
    using namespace tc;
    using C_ = Cfg<BN_>;
    constexpr int BM = C_::BM, BN = C_::BN, BK = C_::BK, STAGES = C_::STAGES, NBUF = C_::NBUF;
    constexpr int A_BYTES = C_::A_BYTES, B_BYTES = C_::B_BYTES, STAGE_BYTES = C_::STAGE_BYTES;
    constexpr int CHUNK_KB = C_::CHUNK_KB, EPI_WARPS = C_::EPI_WARPS;
    constexpr uint32_t TMEM_COLS = C_::TMEM_COLS;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;   // [NBUF] accumulator chunk ready
    uint64_t* tempty = tfull + NBUF;    // [NBUF] accumulator drained (4 epilogue warps)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + NBUF);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;  // N-fastest raster: CTAs sharing A tiles run together
    // split-K: CTA z owns K range [k_begin, k_end) (k_per_split is a multiple of BK)
    const int64_t k_begin = p.k_splits > 1 ? (int64_t)blockIdx.z * p.k_per_split : 0;
    const int64_t k_end = p.k_splits > 1 ? min(p.K, k_begin + p.k_per_split) : p.K;
    const int nk = k_end > k_begin ? (int)((k_end - k_begin + BK - 1) / BK) : 0;
    const int nchunk = nk > 0 ? (nk + CHUNK_KB - 1) / CHUNK_KB : 0;

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
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % STAGES;
                const uint32_t ph = (kb / STAGES) & 1;
                mbar_wait(&empty[s], ph ^ 1);
                unsigned char* st = smem + s * STAGE_BYTES;
                mbar_expect_tx(&full[s], STAGE_BYTES);
                const int kc = (int)k_begin + kb * BK;
                tma_load_2d(st, p.tmap[0], kc, m0, &full[s]);
                tma_load_2d(st + A_BYTES, p.tmap[1], kc, m0, &full[s]);
                tma_load_2d(st + 2 * A_BYTES, p.tmap[2], kc, n0, &full[s]);
                tma_load_2d(st + 2 * A_BYTES + B_BYTES, p.tmap[3], kc, n0, &full[s]);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_tf32(BM, BN);
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % STAGES;
                const uint32_t ph = (kb / STAGES) & 1;
                const int chunk = kb / CHUNK_KB, b = chunk % NBUF;
                const bool chunk_start = kb % CHUNK_KB == 0;
                if (chunk_start) {
                    mbar_wait(&tempty[b], ((chunk / NBUF) & 1) ^ 1);  // epilogue drained this buffer
                    asm volatile("tcgen05.fence::after_thread_sync;");
                }
                mbar_wait(&full[s], ph);
                asm volatile("tcgen05.fence::after_thread_sync;");
                unsigned char* st = smem + s * STAGE_BYTES;
                const uint64_t ah = smem_desc(st), al = smem_desc(st + A_BYTES);
                const uint64_t bh = smem_desc(st + 2 * A_BYTES), bl = smem_desc(st + 2 * A_BYTES + B_BYTES);
                const uint32_t d = tmem + (uint32_t)(b * BN);
#pragma unroll
                for (int j = 0; j < BK / 8; ++j) {
                    const uint64_t adv = (uint64_t)(j * 32) >> 4;  // 8 tf32 = 32 B along K inside the atom
                    const uint32_t acc = !(chunk_start && j == 0);
                    mma_tf32(d, ah + adv, bh + adv, idesc, acc);
                    mma_tf32(d, ah + adv, bl + adv, idesc, 1);
                    mma_tf32(d, al + adv, bh + adv, idesc, 1);
                }
                mma_commit(&empty[s]);
                if (kb % CHUNK_KB == CHUNK_KB - 1 || kb == nk - 1) mma_commit(&tfull[b]);
            }
        }
    } else {
        // Epilogue: warp w owns TMEM lanes [32*(w%4), +32) = tile rows and
        // 128 columns (group cg); it promotes every finished chunk into fp32
        // registers, then stores.
        constexpr int EC = 128;  // columns per epilogue warp
        const int q = warp & 3, cg = (warp - 2) >> 2;
        float acc[EC];
#pragma unroll
        for (int j = 0; j < EC; ++j) acc[j] = 0.0f;
        for (int chunk = 0; chunk < nchunk; ++chunk) {
            const int b = chunk % NBUF;
            mbar_wait(&tfull[b], (chunk / NBUF) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
            for (int c = 0; c < EC / 32; ++c) {
                uint32_t r[32];
                const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * BN + cg * EC + c * 32);
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                    "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                    : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                      "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                      "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                      "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                      "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                    : "r"(taddr));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int j = 0; j < 32; ++j) acc[c * 32 + j] = __fadd_rn(acc[c * 32 + j], __uint_as_float(r[j]));
            }
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&tempty[b])) : "memory");
        }
        float* C = resolve<float>(p.tab, p.c) + (p.k_splits > 1 ? (int64_t)blockIdx.z * p.split_stride : 0);
        const int row = m0 + q * 32 + lane;
        if (row < p.M) {
            const int64_t roff = p.c_rdiv > 0 ? (row / p.c_rdiv) * p.c_s_hi + (row % p.c_rdiv) * p.c_s_lo
                                               : (int64_t)row * p.c_sm;
            float* dst = C + roff;
#pragma unroll
            for (int c = 0; c < EC / 32; ++c) {
                const int col0 = n0 + cg * EC + c * 32;
                if (p.c_sn == 1 && col0 + 32 <= p.N && ((reinterpret_cast<uintptr_t>(dst + col0) & 15) == 0)) {
#pragma unroll
                    for (int j = 0; j < 32; j += 4)
                        *reinterpret_cast<float4*>(dst + col0 + j) =
                            make_float4(acc[c * 32 + j], acc[c * 32 + j + 1], acc[c * 32 + j + 2], acc[c * 32 + j + 3]);
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        if (col0 + j < p.N) dst[(int64_t)(col0 + j) * p.c_sn] = acc[c * 32 + j];
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
    }
}

// Source offset of plane element (row, k) for the gather modes, or -1 for a
// zero tap (padding / out of range).  See gfb_split_args in gfb200.h.
__device__ __forceinline__ int64_t gather_offset(const gfb_split_args& p, int64_t row, int64_t k) {
    const int64_t* g = p.geo;
    switch (p.mode) {
        case 1: {  // conv im2col: row=(n,p,q), k=(c,r,s)
            const int64_t HoWo = g[6] * g[7], RS = g[4] * g[5];
            const int64_t n = row / HoWo, pq = row % HoWo, pp = pq / g[7], q = pq % g[7];
            const int64_t c = k / RS, rs = k % RS, r = rs / g[5], s = rs % g[5];
            const int64_t h = pp * g[8] - g[10] + r, w = q * g[9] - g[11] + s;
            if (h < 0 || h >= g[2] || w < 0 || w >= g[3]) return -1;
            return n * p.st[0] + c * p.st[1] + h * p.st[2] + w * p.st[3];
        }
        case 2: {  // dgrad: row=(n,h,w), k=(kk,r,s) -> delta[n, kk, h+pt-r, w+pl-s]
            const int64_t HW = g[2] * g[3], RS = g[4] * g[5];
            const int64_t n = row / HW, hw = row % HW, h = hw / g[3], w = hw % g[3];
            const int64_t kk = k / RS, rs = k % RS, r = rs / g[5], s = rs % g[5];
            const int64_t pp = h + g[10] - r, q = w + g[11] - s;
            if (pp < 0 || pp >= g[6] || q < 0 || q >= g[7]) return -1;
            return n * p.st[0] + kk * p.st[1] + pp * p.st[2] + q * p.st[3];
        }
        case 3: {  // digits: k = (d0, d1, d2) over extents e0, e1, e2
            const int64_t d2 = k % g[14], d01 = k / g[14], d1 = d01 % g[13], d0 = d01 / g[13];
            return row * p.s_r + d0 * p.st[0] + d1 * p.st[1] + d2 * p.st[2];
        }
        case 4: {  // wgrad: row=(c,r,s), k=(n,p,q) -> x[n, c, p+r-pt, q+s-pl]
            const int64_t RS = g[4] * g[5], HoWo = g[6] * g[7];
            const int64_t c = row / RS, rs = row % RS, r = rs / g[5], s = rs % g[5];
            const int64_t n = k / HoWo, pq = k % HoWo, pp = pq / g[7], q = pq % g[7];
            const int64_t h = pp + r - g[10], w = q + s - g[11];
            if (h < 0 || h >= g[2] || w < 0 || w >= g[3]) return -1;
            return n * p.st[0] + c * p.st[1] + h * p.st[2] + w * p.st[3];
        }
        default:
            return row * p.s_r + k * p.s_k;
    }
}

// hi/lo TF32 planes, K-major [rows, kp], zero-padded past k.  32x32 tiles
// through shared memory so both the strided read and the plane writes are
// coalesced whichever axis of the source is contiguous.
__device__ __forceinline__ void split_tf32(float x, float& h, float& l) {
    uint32_t hb, lb;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(x));
    const float rest = __fsub_rn(x, __uint_as_float(hb));
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(lb) : "f"(rest));
    h = __uint_as_float(hb);
    l = __uint_as_float(lb);
}

__global__ void __launch_bounds__(256) gfb_split_kernel(const __grid_constant__ gfb_split_args p) {
    __shared__ float tile[32][33];
    const float* src = resolve<const float>(p.tab, p.src);
    float* hi = resolve<float>(p.tab, p.hi);
    float* lo = resolve<float>(p.tab, p.lo);
    if (p.mode == 5) {
        // Row-contiguous source (s_k == 1, k == kp, 16-byte aligned rows): a
        // streaming pass with 128-bit loads and stores.
        const int64_t n4 = p.rows * p.kp / 4;
        const int64_t k4 = p.kp / 4;
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
            const int64_t r = i / k4, c = (i % k4) * 4;
            const float4 x = __ldg(reinterpret_cast<const float4*>(src + r * p.s_r + c));
            float4 h, l;
            split_tf32(x.x, h.x, l.x);
            split_tf32(x.y, h.y, l.y);
            split_tf32(x.z, h.z, l.z);
            split_tf32(x.w, h.w, l.w);
            reinterpret_cast<float4*>(hi)[i] = h;
            reinterpret_cast<float4*>(lo)[i] = l;
        }
        return;
    }
    // 1-D grid over (row tile, k tile): either extent can exceed 65535 (the
    // N*H*W rows of a 224x224 batch, or the K of a weight gradient)
    const int64_t row_tiles = (p.rows + 31) / 32;
    const int64_t tid2 = blockIdx.x;
    const int64_t r0 = (tid2 % row_tiles) * 32, k0 = (tid2 / row_tiles) * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const bool k_fast = p.mode != 0 || p.s_k <= p.s_r;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        int rr, kk;
        if (k_fast) { rr = ty + 8 * i; kk = tx; } else { rr = tx; kk = ty + 8 * i; }
        const int64_t r = r0 + rr, k = k0 + kk;
        float v = 0.0f;
        if (r < p.rows && k < p.k) {
            const int64_t off = gather_offset(p, r, k);
            if (off >= 0) v = src[off];
        }
        tile[rr][kk] = v;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int rr = ty + 8 * i, kk = tx;
        const int64_t r = r0 + rr, k = k0 + kk;
        if (r < p.rows && k < p.kp) {
            const float x = tile[rr][kk];
            uint32_t h, l;
            asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
            const float rest = __fsub_rn(x, __uint_as_float(h));
            asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(l) : "f"(rest));
            hi[r * p.kp + k] = __uint_as_float(h);
            lo[r * p.kp + k] = __uint_as_float(l);
        }
    }
}

}  // namespace gfb

template __global__ void gfb::gfb_gemm_tc_kernel<128>(const __grid_constant__ gfb_tc_args);
template __global__ void gfb::gfb_gemm_tc_kernel<256>(const __grid_constant__ gfb_tc_args);

extern "C" const void* gfb_tc_kernel_ptr(int kind) {
    if (kind == GFB_K_DOT_TC32) return (const void*)gfb::gfb_gemm_tc_kernel<128>;
    if (kind == GFB_K_DOT_TC32W) return (const void*)gfb::gfb_gemm_tc_kernel<256>;
    if (kind == GFB_K_SPLIT_TF32) return (const void*)gfb::gfb_split_kernel;
    return nullptr;
}

extern "C" int gfb_tc_smem_bytes(int wide) { return wide ? gfb::tc::Cfg<256>::SMEM_BYTES : gfb::tc::Cfg<128>::SMEM_BYTES; }
