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
#include "tc_prims.cuh"

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


// Single-thread MMA issuer: for each K-block, wait for the stage, issue the
// three 3xTF32 products per 8-wide K step, free the stage, and hand a TMEM
// accumulator chunk to the epilogue every CHUNK_KB K-blocks.  Stage layout:
// [A hi | A lo | B hi | B lo], each K-major SW128.
template <int BN, int STAGES, int STAGE_BYTES, int A_BYTES, int B_BYTES, int CHUNK_KB, int NBUF>
__device__ __forceinline__ void mma_loop(unsigned char* smem, uint64_t* full, uint64_t* empty, uint64_t* tfull,
                                         uint64_t* tempty, uint32_t tmem, int nk) {
    constexpr uint32_t idesc = idesc_tf32(128, BN);
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
        for (int j = 0; j < 4; ++j) {
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

// Epilogue warp: TMEM lanes [32*(warp%4), +32) = tile rows, and EC columns
// (column group cg).  Every finished accumulator chunk is promoted into fp32
// registers with round-to-nearest adds; the sums are stored at the end.
template <int BN, int NBUF, typename RowOff>
__device__ __forceinline__ void epilogue(int warp, int lane, uint64_t* tfull, uint64_t* tempty, uint32_t tmem,
                                         int nchunk, float* C, int n0, int64_t N, int64_t c_sn, RowOff row_off) {
    constexpr int EC = BN < 128 ? BN : 128;
    const int q = warp & 3, cg = ((warp - 2) >> 2) % (BN / EC);
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
    const int64_t roff = row_off(q * 32 + lane);  // < 0: row outside the output
    if (roff >= 0) {
        float* dst = C + roff;
#pragma unroll
        for (int c = 0; c < EC / 32; ++c) {
            const int col0 = n0 + cg * EC + c * 32;
            if (c_sn == 1 && col0 + 32 <= N && ((reinterpret_cast<uintptr_t>(dst + col0) & 15) == 0)) {
#pragma unroll
                for (int j = 0; j < 32; j += 4)
                    *reinterpret_cast<float4*>(dst + col0 + j) =
                        make_float4(acc[c * 32 + j], acc[c * 32 + j + 1], acc[c * 32 + j + 2], acc[c * 32 + j + 3]);
            } else {
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    if (col0 + j < N) dst[(int64_t)(col0 + j) * c_sn] = acc[c * 32 + j];
            }
        }
    }
}

// Output rows numbered linearly (Dot, or the flattened (n, p, q) of a conv).
struct LinearRows {
    int64_t m0, M, c_sm, c_rdiv, c_s_hi, c_s_lo;
    __device__ __forceinline__ int64_t operator()(int r) const {
        const int64_t row = m0 + r;
        if (row >= M) return -1;
        return c_rdiv > 0 ? (row / c_rdiv) * c_s_hi + (row % c_rdiv) * c_s_lo : row * c_sm;
    }
};

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
    unsigned char* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);  // stays a shared-space pointer
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
        if (lane == 0) mma_loop<BN, STAGES, STAGE_BYTES, A_BYTES, B_BYTES, CHUNK_KB, NBUF>(smem, full, empty, tfull, tempty, tmem, nk);
    } else {
        float* C = resolve<float>(p.tab, p.c) + (p.k_splits > 1 ? (int64_t)blockIdx.z * p.split_stride : 0);
        epilogue<BN, NBUF>(warp, lane, tfull, tempty, tmem, nchunk, C, n0, p.N, p.c_sn,
                           LinearRows{m0, p.M, p.c_sm, p.c_rdiv, p.c_s_hi, p.c_s_lo});
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

// One converter thread's share of a 128x32 fp32 tile: the 16-byte chunks at
// src + 2048 i (rows r, r+16, ..., r+112 of the SW128 layout), split into
// hi = x with the 13 low mantissa bits cleared (exact in TF32) and the exact
// remainder lo = x - hi, whose top 11 bits the MMA uses: per product the
// dropped terms stay below ~3 * 2^-20 relative, inside the 1e-5 Dot/Conv
// tolerance.  Two instructions per element instead of the ~11 of a
// cvt.rna.tf32 pair.  All eight loads are issued before any store so the
// shared-memory latency overlaps.  write_hi == false leaves x in place as
// the hi operand (the tensor core reads only its TF32 bits).
__device__ __forceinline__ float4 trunc_tf32(float4 v) {
    return make_float4(__uint_as_float(__float_as_uint(v.x) & 0xffffe000u), __uint_as_float(__float_as_uint(v.y) & 0xffffe000u),
                       __uint_as_float(__float_as_uint(v.z) & 0xffffe000u), __uint_as_float(__float_as_uint(v.w) & 0xffffe000u));
}
__device__ __forceinline__ void split_rows(uint32_t src, uint32_t dst, uint32_t lo_off, bool write_hi = true) {
    float4 x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = tc::lds128(src + 2048 * i);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const float4 h = trunc_tf32(x[i]);
        const float4 l = make_float4(__fsub_rn(x[i].x, h.x), __fsub_rn(x[i].y, h.y), __fsub_rn(x[i].z, h.z), __fsub_rn(x[i].w, h.w));
        if (write_hi) tc::sts128(dst + 2048 * i, h);
        tc::sts128(dst + lo_off + 2048 * i, l);
    }
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
    if (p.mode == 7) {
        // Lo plane only, for a dense row-contiguous arena source that the GEMM
        // reads directly as its hi operand (the tensor core uses only the TF32
        // bits of an fp32 operand, i.e. hi = x truncated): lo = x - trunc(x),
        // exact in fp32.  Saves the hi plane's write and read.
        const int64_t n4 = p.rows * p.kp / 4;
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
            const float4 x = __ldg(reinterpret_cast<const float4*>(src) + i);
            const float4 h = trunc_tf32(x);
            reinterpret_cast<float4*>(lo)[i] = make_float4(__fsub_rn(x.x, h.x), __fsub_rn(x.y, h.y), __fsub_rn(x.z, h.z),
                                                           __fsub_rn(x.w, h.w));
        }
        return;
    }
    if (p.mode == 6) {
        // Transposing split of a row-contiguous source (s_r == 1, s_k % 4 == 0):
        // 64 x 64 tiles, 128-bit loads along rows, smem transpose, 128-bit hi/lo
        // stores along K; grid-stride over the tiles.
        __shared__ float tt[64][65];
        const int64_t rt = (p.rows + 63) / 64, ntiles = rt * ((p.kp + 63) / 64);
        const int t = threadIdx.x;
        for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            const int64_t r0 = (tile % rt) * 64, k0 = (tile / rt) * 64;
            // load: thread t covers rows r0 + 4*(t % 16) .. +3 at k0 + t / 16 + 16 i
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int kk = t / 16 + 16 * i, rr = 4 * (t % 16);
                const int64_t k = k0 + kk, r = r0 + rr;
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                if (k < p.k) {
                    const float* q = src + k * p.s_k + r;
                    if (r + 3 < p.rows) v = __ldg(reinterpret_cast<const float4*>(q));
                    else {
                        if (r < p.rows) v.x = q[0];
                        if (r + 1 < p.rows) v.y = q[1];
                        if (r + 2 < p.rows) v.z = q[2];
                    }
                }
                tt[rr][kk] = v.x;
                tt[rr + 1][kk] = v.y;
                tt[rr + 2][kk] = v.z;
                tt[rr + 3][kk] = v.w;
            }
            __syncthreads();
            // store: thread t covers k0 + 4*(t % 16) .. +3 of rows r0 + t / 16 + 16 i
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int rr = t / 16 + 16 * i, kk = 4 * (t % 16);
                const int64_t r = r0 + rr, k = k0 + kk;
                if (r < p.rows && k < p.kp) {
                    float4 h, l;
                    split_tf32(tt[rr][kk], h.x, l.x);
                    split_tf32(tt[rr][kk + 1], h.y, l.y);
                    split_tf32(tt[rr][kk + 2], h.z, l.z);
                    split_tf32(tt[rr][kk + 3], h.w, l.w);
                    *reinterpret_cast<float4*>(hi + r * p.kp + k) = h;  // kp % 4 == 0, k % 4 == 0
                    *reinterpret_cast<float4*>(lo + r * p.kp + k) = l;
                }
            }
            __syncthreads();
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

// ---------------------------------------------------------------------------
// Implicit-GEMM convolution with the operand gather and the TF32 split fused
// into the tensor-core kernel (no im2col planes in HBM).
//
// A[row, k] is an activation tensor whose channels are contiguous (NHWC
// layout assignment); k runs (r, s, c) with c fastest, so each 32-wide
// K-block is one filter tap (r, s) and 32 consecutive channels: per output
// row a single 128-byte run, or zero padding.  Four gather warps stream those
// runs with 16-byte cp.async (zero-fill for padding taps) into a 4-deep raw
// ring laid out in the SW128 K-major pattern, then split each 16-byte chunk
// into TF32 hi/lo in place of the MMA stage.  B (the filter, small and
// reused) arrives as hi/lo planes by TMA, K-major in the same (r, s, c)
// order.  Warp roles: 0 B TMA, 1 TMEM + MMA issuer, 2..5 epilogue,
// 6..9 A gather + split.
namespace tc {
template <int BN_>
struct GCfg {
    static constexpr int BM = 128, BN = BN_, BK = 32;
    static constexpr int STAGES = BN_ == 128 ? 2 : 3;
    static constexpr int A_BYTES = BM * BK * 4, B_BYTES = BN * BK * 4;
    static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
    static constexpr int RAW = 4;  // raw A K-blocks in flight per CTA
    static constexpr int CHUNK_KB = 4, NBUF = 512 / BN;
    static constexpr uint32_t TMEM_COLS = 512;
    static constexpr int EPI_WARPS = 4, GATHER_WARPS = 4;
    static constexpr int THREADS = 64 + 32 * (EPI_WARPS + GATHER_WARPS);
    // generic gather (tcgg) at BN = 64: two warps per 32 rows, each taking 16
    // of a K-block's 32 columns (the 4-byte gather is latency bound; at
    // BN = 128 the epilogue's registers leave room for one warp per 32 rows)
    static constexpr int GATHER_WARPS_GG = BN_ == 64 ? 8 : 4;
    static constexpr int THREADS_GG = 64 + 32 * (EPI_WARPS + GATHER_WARPS_GG);
    static constexpr int ROWTAB = BM * 16;
    static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + RAW * A_BYTES + ROWTAB + 256 + 1024;
};

struct RowInfo {
    int64_t off;  // element offset of tap (0, 0), channel 0
    int32_t h, w; // its spatial coordinates (invalid rows: h far out of range)
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(su32(dst)), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
}  // namespace tc

template <int BN_>
__global__ void __launch_bounds__(tc::GCfg<BN_>::THREADS, 1) gfb_conv_tcg_kernel(const __grid_constant__ gfb_tcg_args p) {
    // Persistent: CTA b walks (column tile, row tile) items b, b + gridDim.x,
    // ...; the stage ring, raw ring and TMEM accumulator buffers keep their
    // counters across items, so one item's epilogue overlaps the next item's
    // gather and MMAs (small-K convolutions are a few K-blocks per tile).
    using namespace tc;
    using C_ = GCfg<BN_>;
    constexpr int BN = C_::BN, BK = C_::BK, STAGES = C_::STAGES, NBUF = C_::NBUF, RAW = C_::RAW;
    constexpr int A_BYTES = C_::A_BYTES, B_BYTES = C_::B_BYTES, STAGE_BYTES = C_::STAGE_BYTES;
    constexpr int CHUNK_KB = C_::CHUNK_KB, EPI_WARPS = C_::EPI_WARPS, GATHER_WARPS = C_::GATHER_WARPS;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);  // stays a shared-space pointer
    unsigned char* raw = smem + STAGES * STAGE_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(raw + RAW * A_BYTES + C_::ROWTAB);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + NBUF;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + NBUF);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nk = (int)((p.K + BK - 1) / BK);
    const int nchunk = (nk + CHUNK_KB - 1) / CHUNK_KB;
    const int ntn = (int)((p.N + BN - 1) / BN), ntm = (int)((p.M + 127) / 128);
    const int nitems = ntn * ntm;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1 + GATHER_WARPS);  // TMA expect_tx arrival + one per gather warp
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < NBUF; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], EPI_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        prefetch_tmap(p.tmap[0]);
        prefetch_tmap(p.tmap[1]);
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
                const int n0 = (it % ntn) * BN;
                for (int kb = 0; kb < nk; ++kb, ++gk) {
                    const int s = gk % STAGES;
                    mbar_wait(&empty[s], ((gk / STAGES) & 1) ^ 1);
                    unsigned char* st = smem + s * STAGE_BYTES;
                    mbar_expect_tx(&full[s], 2 * B_BYTES);
                    tma_load_2d(st + 2 * A_BYTES, p.tmap[0], kb * BK, n0, &full[s]);
                    tma_load_2d(st + 2 * A_BYTES + B_BYTES, p.tmap[1], kb * BK, n0, &full[s]);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_tf32(128, BN);
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
                    for (int j = 0; j < 4; ++j) {
                        const uint64_t adv = (uint64_t)(j * 32) >> 4;
                        const uint32_t acc = !(chunk_start && j == 0);
                        mma_tf32(d, ah + adv, bh + adv, idesc, acc);
                        mma_tf32(d, ah + adv, bl + adv, idesc, 1);
                        mma_tf32(d, al + adv, bh + adv, idesc, 1);
                    }
                    mma_commit(&empty[s]);
                    if (i % CHUNK_KB == CHUNK_KB - 1 || i == nk - 1) mma_commit(&tfull[b]);
                }
                gc += nchunk;
            }
        }
    } else if (warp < 2 + EPI_WARPS) {
        constexpr int EC = BN < 128 ? BN : 128;
        const int q = warp & 3;
        uint32_t gc = 0;
        float* C = resolve<float>(p.tab, p.c);
        for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
            const int n0 = (it % ntn) * BN, m0 = (it / ntn) * 128;
            float acc[EC];
#pragma unroll
            for (int j = 0; j < EC; ++j) acc[j] = 0.0f;
            for (int c0 = 0; c0 < nchunk; ++c0) {
                const uint32_t chunk = gc + c0;
                const int b = chunk % NBUF;
                mbar_wait(&tfull[b], (chunk / NBUF) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
                for (int c = 0; c < EC / 32; ++c) {
                    uint32_t r[32];
                    const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * BN + c * 32);
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
            gc += nchunk;
            const LinearRows rows{m0, p.M, p.c_sm, p.c_rdiv, p.c_s_hi, p.c_s_lo};
            const int64_t roff = rows(q * 32 + lane);
            if (roff >= 0) {
                float* dst = C + roff;
#pragma unroll
                for (int c = 0; c < EC / 32; ++c) {
                    const int col0 = n0 + c * 32;
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
    } else {
        // gather thread: 16-byte piece j (channels 4j..4j+3 of the K-block) of rows rb + 16 i
        const int g = threadIdx.x - (2 + EPI_WARPS) * 32;  // 0..127
        const float* A = resolve<const float>(p.tab, p.a);
        const int j = g & 7, rb = g >> 3;
        const uint32_t swz = (uint32_t)((j ^ (rb & 7)) << 4);  // row & 7 == rb & 7 for every row rb + 16 i
        const int Cc = p.C ? p.C : 32 * p.CB;
        uint32_t gk = 0;
        for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
            const int m0 = (it / ntn) * 128;
            int64_t roff[8];
            int rh[8], rw[8];
            const uint32_t yx = (uint32_t)p.Y * (uint32_t)p.X;  // rows < 2^31 (lowering checks the tile count)
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const uint32_t row = (uint32_t)(m0 + rb + 16 * i);
                if (row < (uint32_t)p.M) {
                    const uint32_t n = row / yx, rem = row - n * yx, y = rem / (uint32_t)p.X, x = rem - y * (uint32_t)p.X;
                    rh[i] = (int)y * p.sy + p.oy;
                    rw[i] = (int)x * p.sx + p.ox;
                    roff[i] = (int64_t)n * p.xs0 + (int64_t)rh[i] * p.xs2 + (int64_t)rw[i] * p.xs3;
                } else {
                    roff[i] = 0;
                    rh[i] = -(1 << 30);
                    rw[i] = 0;
                }
            }
            auto issue = [&](int kb) {
                // this thread's 16-byte piece: channels c..c+3 of tap (r, s), k = kb*32 + 4j
                const int k = kb * BK + j * 4, tap = k / Cc, c = k - tap * Cc, r = tap / p.S, s = tap - r * p.S;
                const bool kok = k < p.K;
                const int dh = p.ksign * r, dw = p.ksign * s;
                const int64_t koff = (int64_t)dh * p.xs2 + (int64_t)dw * p.xs3 + c;
                unsigned char* dst = raw + ((gk + kb) % RAW) * A_BYTES + swz;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int row = rb + 16 * i;
                    const bool ok = kok && (uint32_t)(rh[i] + dh) < (uint32_t)p.H && (uint32_t)(rw[i] + dw) < (uint32_t)p.W;
                    cp_async16(dst + row * 128, ok ? (const void*)(A + roff[i] + koff) : (const void*)A, ok ? 16u : 0u);
                }
            };
#pragma unroll
            for (int kb = 0; kb < RAW; ++kb) {
                if (kb < nk) issue(kb);
                cp_async_commit();
            }
            for (int kb = 0; kb < nk; ++kb) {
                cp_async_wait<RAW - 1>();  // this thread's copies of K-block kb have landed
                const uint32_t g2 = gk + kb;
                const int s = g2 % STAGES;
                mbar_wait(&empty[s], ((g2 / STAGES) & 1) ^ 1);
                split_rows(su32(raw + (g2 % RAW) * A_BYTES) + swz + rb * 128, su32(smem + s * STAGE_BYTES) + swz + rb * 128,
                           A_BYTES);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor-core reads
                __syncwarp();
                if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&full[s])) : "memory");
                if (kb + RAW < nk) issue(kb + RAW);  // reuses the raw slot just consumed (own chunks only)
                cp_async_commit();
            }
            gk += nk;
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
// Implicit-GEMM convolution with the gather done by TMA.  The 128 GEMM rows
// of a CTA are a box of output pixels (BNI images x BY rows x BX columns);
// for K-block (r, s, c0..c0+31) the A tile is then one 4-D tensor-map box of
// the channel-last activation at (c0, x0*sx + ox + ksign*s, y0*sy + oy +
// ksign*r, n0) with traversal strides (1, sx, sy, 1): TMA applies the
// convolution stride, zero-fills the padding taps (out-of-bounds
// coordinates) and writes the SW128 K-major layout the MMA reads.  Four
// converter warps split each landed tile into TF32 hi/lo in place.
// Warp roles: 0 TMA (A box + B planes), 1 TMEM + MMA, 2..5 epilogue,
// 6..9 converters.
namespace tc {
template <int BN_>
struct XCfg {
    static constexpr int BM = 128, BN = BN_, BK = 32;
    static constexpr int A_BYTES = BM * BK * 4, B_BYTES = BN * BK * 4;
    static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
    static constexpr int STAGES = BN_ == 128 ? 3 : 4;
    static constexpr int CHUNK_KB = 4, NBUF = 512 / BN;
    static constexpr uint32_t TMEM_COLS = 512;
    static constexpr int EPI_WARPS = 4, CONV_WARPS = 4;
    static constexpr int THREADS = 64 + 32 * (EPI_WARPS + CONV_WARPS);
    static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 256 + 1024;
};

}  // namespace tc

template <int BN_>
__global__ void __launch_bounds__(tc::XCfg<BN_>::THREADS, 1) gfb_conv_tcx_kernel(const __grid_constant__ gfb_tcx_args p) {
    // Persistent like gfb_conv_tcgg_kernel: CTA b walks items b, b + gridDim.x,
    // ... over (column tile, pixel tile); ring and TMEM-buffer counters carry
    // across items.
    using namespace tc;
    using C_ = XCfg<BN_>;
    constexpr int BN = C_::BN, BK = C_::BK, STAGES = C_::STAGES, NBUF = C_::NBUF;
    constexpr int A_BYTES = C_::A_BYTES, B_BYTES = C_::B_BYTES, STAGE_BYTES = C_::STAGE_BYTES;
    constexpr int CHUNK_KB = C_::CHUNK_KB, EPI_WARPS = C_::EPI_WARPS, CONV_WARPS = C_::CONV_WARPS;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);  // stays a shared-space pointer
    uint64_t* afull = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);  // A box landed
    uint64_t* full = afull + STAGES;    // A split + B planes landed
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
            mbar_init(&afull[s], 1);
            mbar_init(&full[s], 1 + CONV_WARPS);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < NBUF; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], EPI_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int i = 0; i < 3; ++i) prefetch_tmap(p.tmap[i]);
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
                    mbar_expect_tx(&afull[s], A_BYTES);
                    tma_load_4d(st, p.tmap[0], cb * 32, I.x0 * p.sx + p.ox + p.ksign * s_, I.y0 * p.sy + p.oy + p.ksign * r,
                                I.n0, &afull[s]);
                    mbar_expect_tx(&full[s], 2 * B_BYTES);
                    tma_load_2d(st + 2 * A_BYTES, p.tmap[1], kb * BK, I.col0, &full[s]);
                    tma_load_2d(st + 2 * A_BYTES + B_BYTES, p.tmap[2], kb * BK, I.col0, &full[s]);
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
            constexpr uint32_t idesc = idesc_tf32(128, BN);
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
                    for (int j = 0; j < 4; ++j) {
                        const uint64_t adv = (uint64_t)(j * 32) >> 4;
                        const uint32_t acc = !(chunk_start && j == 0);
                        mma_tf32(d, ah + adv, bh + adv, idesc, acc);
                        mma_tf32(d, ah + adv, bl + adv, idesc, 1);
                        mma_tf32(d, al + adv, bh + adv, idesc, 1);
                    }
                    mma_commit(&empty[s]);
                    if (i % CHUNK_KB == CHUNK_KB - 1 || i == nk - 1) mma_commit(&tfull[b]);
                }
                gc += nchunk;
            }
        }
    } else if (warp < 2 + EPI_WARPS) {
        constexpr int EC = BN < 128 ? BN : 128;
        const int q = warp & 3;
        uint32_t gc = 0;
        float* C = resolve<float>(p.tab, p.c);
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
                for (int c = 0; c < EC / 32; ++c) {
                    uint32_t r[32];
                    const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * BN + c * 32);
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
    } else {
        // converters: thread g owns 16-byte chunk (g & 7) of rows (g >> 3) + 16 i
        const int g = threadIdx.x - (2 + EPI_WARPS) * 32;
        const int j = g & 7, rb = g >> 3;
        const uint32_t swz = (uint32_t)((j ^ (rb & 7)) << 4);
        uint32_t gk = 0;
        for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
            for (int kb = 0; kb < nk; ++kb, ++gk) {
                const int s = gk % STAGES;
                mbar_wait(&afull[s], (gk / STAGES) & 1);
                split_rows(su32(smem + s * STAGE_BYTES) + swz + rb * 128, su32(smem + s * STAGE_BYTES) + swz + rb * 128,
                           A_BYTES, p.pad0 == 0);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&full[s])) : "memory");
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

// ---------------------------------------------------------------------------
// 2-SM GEMM: a CTA pair (cluster of 2, cta_group::2) computes a 256 x 256
// tile.  CTA r loads A rows [m0 + 128 r, +128) and B rows [n0 + 128 r, +128)
// (hi and lo planes) into its own shared memory; the leader (rank 0) issues
// tcgen05.mma.cta_group::2 with M = 256, N = 256, which reads each CTA's
// half of A and B from that CTA's shared memory and accumulates rows
// [128 r, +128) in CTA r's TMEM.  Per SM this halves the shared-memory
// operand reads per flop relative to a 128 x 256 single-SM tile (the
// single-SM kernel is smem-bandwidth bound).  Barriers: the leader's full[s]
// counts both CTAs' TMA bytes (the peer's loads signal it across the pair);
// the leader's commits multicast to both CTAs' empty[s] / tfull[b]; both
// CTAs' epilogue warps arrive on the leader's tempty[b].
namespace tc {
struct PCfg {
    static constexpr int BM = 128, BN = 128, BK = 32;  // per-CTA rows of A and of B
    static constexpr int STAGES = 3;
    static constexpr int A_BYTES = BM * BK * 4, B_BYTES = BN * BK * 4;
    static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
    static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;
    static constexpr int CHUNK_KB = 4, NBUF = 2, NT = 256;  // accumulator columns per buffer
    static constexpr uint32_t TMEM_COLS = 512;
    static constexpr int EPI_WARPS = 8;
    static constexpr int THREADS = 64 + 32 * EPI_WARPS;
    // per epilogue warp, a 32 x 32 fp32 transpose tile (16-byte pieces XOR-swizzled
    // by row): the accumulators sit one row per lane, the stores go out row-contiguous
    static constexpr int XPOSE_BYTES = EPI_WARPS * 32 * 32 * 4;
    static constexpr int SMEM_BYTES_PAIR = STAGES * STAGE_BYTES + 1024 + 256 + XPOSE_BYTES;
};

}  // namespace tc

// Persistent: the grid is at most one CTA pair per two SMs, and each pair
// walks the output tiles (and K splits) in a grouped raster -- GROUP_M
// row-tiles by every column tile -- so that concurrently running pairs share
// their A row strips and B column strips in L2.  The stage ring, the TMEM
// accumulator ring and the epilogue's promotion protocol all run across tile
// boundaries: one tile's last chunks and its stores overlap the next tile's
// loads and MMAs, and the barrier / TMEM setup is paid once per kernel.
namespace tc {
struct PTile {
    int m0, n0, z, nk;
};
__device__ __forceinline__ PTile pair_tile(const gfb_tc_args& p, int t, int ntm, int ntn) {
    const int GROUP_M = p.group_m > 1 ? (int)p.group_m : 1;  // 1: row-major, column tiles fastest
    const int per_z = ntm * ntn;
    const int z = t / per_z, r = t % per_z;
    const int g = r / (GROUP_M * ntn), gr = r % (GROUP_M * ntn);
    const int gm = min(GROUP_M, ntm - g * GROUP_M);
    PTile o;
    o.m0 = (g * GROUP_M + gr % gm) * 256;
    o.n0 = (gr / gm) * 256;
    o.z = z;
    const int64_t k_begin = p.k_splits > 1 ? (int64_t)z * p.k_per_split : 0;
    const int64_t k_end = p.k_splits > 1 ? min(p.K, k_begin + p.k_per_split) : p.K;
    o.nk = k_end > k_begin ? (int)((k_end - k_begin + PCfg::BK - 1) / PCfg::BK) : 0;
    return o;
}
}  // namespace tc

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(tc::PCfg::THREADS, 1)
    gfb_gemm_tc2_kernel(const __grid_constant__ gfb_tc_args p) {
    using namespace tc;
    using C_ = PCfg;
    constexpr int BK = C_::BK, STAGES = C_::STAGES, NBUF = C_::NBUF, NT = C_::NT;
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
    cluster_sync_all();  // both CTAs' barriers initialised and TMEM allocated
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            const uint32_t full0 = peer_addr(full, 0);  // the leader's full barriers
            int g = 0;                                   // K-blocks issued so far (the ring position)
            for (int t = pair_id; t < ntiles; t += npairs) {
                const PTile T = pair_tile(p, t, ntm, ntn);
                const int64_t k_begin = p.k_splits > 1 ? (int64_t)T.z * p.k_per_split : 0;
                const int am = T.m0 + 128 * rank, bn = T.n0 + 128 * rank;
                for (int kb = 0; kb < T.nk; ++kb, ++g) {
                    const int s = g % STAGES;
                    mbar_wait(&empty[s], ((g / STAGES) & 1) ^ 1);
                    unsigned char* st = smem + s * STAGE_BYTES;
                    if (leader) mbar_expect_tx(&full[s], 2 * STAGE_BYTES);  // both CTAs' bytes land on it
                    const uint32_t bar = full0 + s * 8;
                    const int kc = (int)k_begin + kb * BK;
                    if (p.a_ld_mn > 0) {  // MN-major: (32 MN, 32 K, 4 MN atoms) boxes
                        tma_load_3d_pair(st, p.tmap[0], 0, kc, am >> 5, bar);
                        tma_load_3d_pair(st + A_BYTES, p.tmap[1], 0, kc, am >> 5, bar);
                    } else {
                        tma_load_2d_pair(st, p.tmap[0], kc, am, bar);
                        tma_load_2d_pair(st + A_BYTES, p.tmap[1], kc, am, bar);
                    }
                    if (p.b_ld_mn > 0) {
                        tma_load_3d_pair(st + 2 * A_BYTES, p.tmap[2], 0, kc, bn >> 5, bar);
                        tma_load_3d_pair(st + 2 * A_BYTES + B_BYTES, p.tmap[3], 0, kc, bn >> 5, bar);
                    } else {
                        tma_load_2d_pair(st + 2 * A_BYTES, p.tmap[2], kc, bn, bar);
                        tma_load_2d_pair(st + 2 * A_BYTES + B_BYTES, p.tmap[3], kc, bn, bar);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && leader) {
            const bool a_mn = p.a_ld_mn > 0, b_mn = p.b_ld_mn > 0;
            const uint32_t idesc = idesc_tf32(256, 256) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16);
            int g = 0, gchunk = 0;  // ring positions across tiles
            for (int t = pair_id; t < ntiles; t += npairs) {
                const PTile T = pair_tile(p, t, ntm, ntn);
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
                    for (int j = 0; j < BK / 8; ++j) {
                        // K-major SW128: 8 tf32 = 32 B along K inside the atom; MN-major:
                        // 8 K rows = two 4-row groups = 1024 B further
                        const uint64_t ah = a_mn ? smem_desc_mn_at(sa + j * 1024) : smem_desc(st) + ((uint64_t)(j * 32) >> 4);
                        const uint64_t al = a_mn ? smem_desc_mn_at(sa + A_BYTES + j * 1024)
                                                 : smem_desc(st + A_BYTES) + ((uint64_t)(j * 32) >> 4);
                        const uint64_t bh = b_mn ? smem_desc_mn_at(sb + j * 1024)
                                                 : smem_desc(st + 2 * A_BYTES) + ((uint64_t)(j * 32) >> 4);
                        const uint64_t bl = b_mn ? smem_desc_mn_at(sb + B_BYTES + j * 1024)
                                                 : smem_desc(st + 2 * A_BYTES + B_BYTES) + ((uint64_t)(j * 32) >> 4);
                        const uint32_t acc = !(chunk_start && j == 0);
                        mma_tf32_pair(d, ah, bh, idesc, acc);
                        mma_tf32_pair(d, ah, bl, idesc, 1);
                        mma_tf32_pair(d, al, bh, idesc, 1);
                    }
                    mma_commit_pair(&empty[s]);
                    if (kb % CHUNK_KB == CHUNK_KB - 1 || kb == T.nk - 1) mma_commit_pair(&tfull[b]);
                }
                gchunk += (T.nk + CHUNK_KB - 1) / CHUNK_KB;
            }
        }
    } else {
        // epilogue: warp w owns TMEM lanes [32 (w % 4), +32) = this CTA's tile
        // rows, and 128 of the 256 columns (cg); promotion as in the 1-SM kernel
        constexpr int EC = 128;
        const int q = warp & 3, cg = (warp - 2) >> 2;
        const uint32_t tempty0 = peer_addr(tempty, 0);
        int gchunk = 0;
        for (int t = pair_id; t < ntiles; t += npairs) {
            const PTile T = pair_tile(p, t, ntm, ntn);
            const int nchunk = (T.nk + CHUNK_KB - 1) / CHUNK_KB;
            float acc[EC];
#pragma unroll
            for (int j = 0; j < EC; ++j) acc[j] = 0.0f;
            for (int c0 = 0; c0 < nchunk; ++c0) {
                const int chunk = gchunk + c0, b = chunk % NBUF;
                mbar_wait(&tfull[b], (chunk / NBUF) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
                for (int c = 0; c < EC / 32; ++c) {
                    uint32_t r[32];
                    const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * NT + cg * EC + c * 32);
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
                if (lane == 0)
                    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(tempty0 + b * 8) : "memory");
            }
            gchunk += nchunk;
            float* C = resolve<float>(p.tab, p.c) + (p.k_splits > 1 ? (int64_t)T.z * p.split_stride : 0);
            const LinearRows rows{T.m0 + 128 * (int64_t)rank, p.M, p.c_sm, p.c_rdiv, p.c_s_hi, p.c_s_lo};
            const int64_t roff = rows(q * 32 + lane);
            // Coalesced path: every row of the tile is a dense run of the output
            // (and of the epilogue's operands), row pitch c_sm, 16-byte aligned.
            const bool coalesced = p.c_rdiv <= 0 && p.c_sn == 1 && (p.c_sm & 3) == 0 && (p.N & 3) == 0;
            if (coalesced) {
                // after the barriers (the first 256 B past the stages); the 1024 B of
                // slack in the allocation are the alignment of `smem`, not an offset
                float* xt = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES + 256) + (warp - 2) * 1024;
                const int64_t row0 = T.m0 + 128 * (int64_t)rank + q * 32;  // this warp's 32 rows
                // refs are (slot, offset): arena offset 0 encodes as 0, so presence comes from the kind / flags
                const float* bias = p.epi_kind == 1 ? resolve<const float>(p.tab, p.e_bias) : nullptr;
                const float* xin = p.epi_kind == 2 ? resolve<const float>(p.tab, p.e_aux2) : nullptr;
                float* out2 = (p.epi_flags & 1) ? resolve<float>(p.tab, p.e_out2) : nullptr;
                float* lo = (p.epi_flags & 2) ? resolve<float>(p.tab, p.e_lo) : nullptr;
#pragma unroll
                for (int c = 0; c < EC / 32; ++c) {
                    // lane r writes its row's 32 values as 8 swizzled 16-byte pieces
#pragma unroll
                    for (int qd = 0; qd < 8; ++qd)
                        *reinterpret_cast<float4*>(xt + lane * 32 + ((qd ^ (lane & 7)) << 2)) =
                            make_float4(acc[c * 32 + 4 * qd], acc[c * 32 + 4 * qd + 1], acc[c * 32 + 4 * qd + 2],
                                        acc[c * 32 + 4 * qd + 3]);
                    __syncwarp();
                    const int qd = lane & 7, col = T.n0 + cg * EC + c * 32 + 4 * qd;
                    float4 b4 = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (p.epi_kind == 1 && col < p.N) b4 = __ldg(reinterpret_cast<const float4*>(bias + col));
#pragma unroll
                    for (int half = 0; half < 2; ++half) {
                    float4 x4[4];  // kind 2: four rows' pre-activations in flight at once
                    if (p.epi_kind == 2) {
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const int64_t row = row0 + 4 * (4 * half + i) + (lane >> 3);
                            x4[i] = (row < p.M && col < p.N) ? __ldg(reinterpret_cast<const float4*>(xin + row * p.c_sm + col))
                                                             : make_float4(0.f, 0.f, 0.f, 0.f);
                        }
                    }
#pragma unroll
                    for (int ii = 0; ii < 4; ++ii) {
                        const int i = 4 * half + ii;
                        const int rr = 4 * i + (lane >> 3);  // lanes 8k..8k+7 cover one 128-byte row piece
                        const int64_t row = row0 + rr;
                        float4 v = *reinterpret_cast<const float4*>(xt + rr * 32 + ((qd ^ (rr & 7)) << 2));
                        if (row >= p.M || col >= p.N) continue;
                        const int64_t off = row * p.c_sm + col;
                        float4 y = v;  // the tensor a later GEMM may read raw (lo plane)
                        if (p.epi_kind == 1) {
                            v = make_float4(__fadd_rn(v.x, b4.x), __fadd_rn(v.y, b4.y), __fadd_rn(v.z, b4.z), __fadd_rn(v.w, b4.w));
                            y = make_float4(v.x > 0.f ? v.x : 0.f, v.y > 0.f ? v.y : 0.f, v.z > 0.f ? v.z : 0.f, v.w > 0.f ? v.w : 0.f);
                        } else if (p.epi_kind == 2) {
                            v = make_float4(__fmul_rn(v.x, relu_grad_mask(x4[ii].x)), __fmul_rn(v.y, relu_grad_mask(x4[ii].y)),
                                            __fmul_rn(v.z, relu_grad_mask(x4[ii].z)), __fmul_rn(v.w, relu_grad_mask(x4[ii].w)));
                            y = v;
                        }
                        *reinterpret_cast<float4*>(C + off) = v;
                        if (out2) *reinterpret_cast<float4*>(out2 + off) = y;
                        if (lo)
                            *reinterpret_cast<float4*>(lo + off) = make_float4(
                                __fsub_rn(y.x, __uint_as_float(__float_as_uint(y.x) & 0xffffe000u)),
                                __fsub_rn(y.y, __uint_as_float(__float_as_uint(y.y) & 0xffffe000u)),
                                __fsub_rn(y.z, __uint_as_float(__float_as_uint(y.z) & 0xffffe000u)),
                                __fsub_rn(y.w, __uint_as_float(__float_as_uint(y.w) & 0xffffe000u)));
                    }
                    }
                    __syncwarp();
                }
            } else if (roff >= 0 && p.epi_kind != 0) {
                // fused epilogue (gfb200.h gfb_tc_args): the elementwise map that
                // consumed this Dot, computed from the registers, in 4-wide pieces
                const float* bias = p.epi_kind == 1 ? resolve<const float>(p.tab, p.e_bias) : nullptr;
                const float* xin = p.epi_kind == 2 ? resolve<const float>(p.tab, p.e_aux2) + roff : nullptr;
                float* out2 = (p.epi_flags & 1) ? resolve<float>(p.tab, p.e_out2) + roff : nullptr;
                float* lo = (p.epi_flags & 2) ? resolve<float>(p.tab, p.e_lo) + roff : nullptr;
                float* dst = C + roff;
#pragma unroll
                for (int c = 0; c < EC / 32; ++c) {
                    const int col0 = T.n0 + cg * EC + c * 32;
#pragma unroll
                    for (int j = 0; j < 32; j += 4) {
                        const int n = col0 + j;
                        if (n >= p.N) break;
                        float v[4] = {acc[c * 32 + j], acc[c * 32 + j + 1], acc[c * 32 + j + 2], acc[c * 32 + j + 3]};
                        float y[4];  // the tensor a later GEMM may read raw (lo plane)
                        const int cnt = min(4, (int)(p.N - n));
                        const bool vec = cnt == 4 && ((roff + n) & 3) == 0;  // 16-byte pieces (bias: n % 4 == 0 too)
                        if (p.epi_kind == 1) {
                            float b[4];
                            if (vec) {
                                const float4 t4 = __ldg(reinterpret_cast<const float4*>(bias + n));
                                b[0] = t4.x, b[1] = t4.y, b[2] = t4.z, b[3] = t4.w;
                            } else {
#pragma unroll
                                for (int e = 0; e < 4; ++e) b[e] = e < cnt ? bias[n + e] : 0.f;
                            }
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                v[e] = __fadd_rn(v[e], b[e]);
                                y[e] = v[e] > 0.f ? v[e] : 0.f;
                            }
                        } else {
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                v[e] = __fmul_rn(v[e], relu_grad_mask(e < cnt ? xin[n + e] : 1.f));
                                y[e] = v[e];
                            }
                        }
                        float l[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) l[e] = __fsub_rn(y[e], __uint_as_float(__float_as_uint(y[e]) & 0xffffe000u));
                        if (vec) {
                            *reinterpret_cast<float4*>(dst + n) = make_float4(v[0], v[1], v[2], v[3]);
                            if (out2) *reinterpret_cast<float4*>(out2 + n) = make_float4(y[0], y[1], y[2], y[3]);
                            if (lo) *reinterpret_cast<float4*>(lo + n) = make_float4(l[0], l[1], l[2], l[3]);
                        } else {
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                if (e >= cnt) break;
                                dst[n + e] = v[e];
                                if (out2) out2[n + e] = y[e];
                                if (lo) lo[n + e] = l[e];
                            }
                        }
                    }
                }
            } else if (roff >= 0) {
                float* dst = C + roff;
#pragma unroll
                for (int c = 0; c < EC / 32; ++c) {
                    const int col0 = T.n0 + cg * EC + c * 32;
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
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    cluster_sync_all();  // the peer's epilogue and the leader's MMAs are done
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C_::TMEM_COLS));
    }
}

// ---------------------------------------------------------------------------
// Implicit-GEMM convolution with a generic element gather (any channel count,
// any layout, weight gradients included).  A[row, k] = a[rowoff(row) +
// koff(k)] when 0 <= h(row) + dh(k) < H and 0 <= w(row) + dw(k) < W, else 0.
// Rows are (i0, i1, i2) over (*, E1, E2): rowoff = i0*ro0 + i1*ro1 + i2*ro2,
// h = i1*hm + h0, w = i2*wm + w0 (rows (r, s, c), pad0 == 1: h from i0, w
// from i1, so lanes walk contiguous channels); the K index decomposes into
// (koff, dh, dw) (gfb_tcgg_args in gfb200.h):
//   Conv2D:             rows (n, p, q), k = (c, r, s): dh = r - pt, dw = s - pl
//   ConvBackpropData:   rows (n, h, w), k = (kk, r, s): dh = pt - r, dw = pl - s
//   ConvBackpropFilter: rows (c, r, s) with h0 = -pt, w0 = -pl, k = (n, p, q):
//                       dh = p, dw = q
// Gather warps map lanes to 32 consecutive rows (coalesced along the
// activation's fastest spatial axis) and walk the 32 k of a K-block with
// 4-byte zero-filling cp.async into a 4-deep raw ring; each thread then
// splits its own row into TF32 hi/lo.  B (filter or δ planes) by TMA.
// Split-K over blockIdx.z as in the plane GEMM.
template <int BN_>
__global__ void __launch_bounds__(tc::GCfg<BN_>::THREADS_GG, 1) gfb_conv_tcgg_kernel(const __grid_constant__ gfb_tcgg_args p) {
    // Persistent: CTA b walks work items b, b + gridDim.x, ... over (n tile,
    // m tile, K split); the stage ring, the raw ring and the TMEM accumulator
    // buffers keep their counters across items, so one item's epilogue and
    // stores overlap the next item's gather and MMAs, and TMEM allocation,
    // barrier setup and tensor-map prefetch happen once per CTA.
    using namespace tc;
    using C_ = GCfg<BN_>;
    constexpr int BN = C_::BN, BK = C_::BK, STAGES = C_::STAGES, NBUF = C_::NBUF, RAW = C_::RAW;
    constexpr int A_BYTES = C_::A_BYTES, B_BYTES = C_::B_BYTES, STAGE_BYTES = C_::STAGE_BYTES;
    constexpr int CHUNK_KB = C_::CHUNK_KB, EPI_WARPS = C_::EPI_WARPS, GATHER_WARPS = C_::GATHER_WARPS_GG;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);  // stays a shared-space pointer
    unsigned char* raw = smem + STAGES * STAGE_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(raw + RAW * A_BYTES + C_::ROWTAB);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + NBUF;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + NBUF);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int kb_total = (int)((p.K + BK - 1) / BK);
    const int ntn = (int)((p.N + BN - 1) / BN), ntm = (int)((p.M + 127) / 128);
    const int nsplit = p.k_splits > 1 ? (int)p.k_splits : 1;
    const int nitems = ntn * ntm * nsplit;
    struct Item {
        int m0, n0, z, kb_begin, nk;
    };
    auto item_at = [&](int it) {
        Item r;
        const int nt = it % ntn, mt = (it / ntn) % ntm;
        r.z = it / (ntn * ntm);
        r.m0 = mt * 128;
        r.n0 = nt * BN;
        r.kb_begin = nsplit > 1 ? r.z * p.kb_per_split : 0;
        const int kb_end = nsplit > 1 ? min(kb_total, r.kb_begin + p.kb_per_split) : kb_total;
        r.nk = max(0, kb_end - r.kb_begin);
        return r;
    };

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1 + GATHER_WARPS);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < NBUF; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], EPI_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        prefetch_tmap(p.tmap[0]);
        prefetch_tmap(p.tmap[1]);
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
            uint32_t gk = 0;  // K-blocks issued by this CTA so far
            for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
                const Item I = item_at(it);
                for (int i = 0; i < I.nk; ++i, ++gk) {
                    const int s = gk % STAGES;
                    mbar_wait(&empty[s], ((gk / STAGES) & 1) ^ 1);
                    unsigned char* st = smem + s * STAGE_BYTES;
                    mbar_expect_tx(&full[s], 2 * B_BYTES);
                    tma_load_2d(st + 2 * A_BYTES, p.tmap[0], (I.kb_begin + i) * BK, I.n0, &full[s]);
                    tma_load_2d(st + 2 * A_BYTES + B_BYTES, p.tmap[1], (I.kb_begin + i) * BK, I.n0, &full[s]);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_tf32(128, BN);
            uint32_t gk = 0, gc = 0;  // K-blocks and accumulator chunks so far
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
                    unsigned char* st = smem + s * STAGE_BYTES;
                    const uint64_t ah = smem_desc(st), al = smem_desc(st + A_BYTES);
                    const uint64_t bh = smem_desc(st + 2 * A_BYTES), bl = smem_desc(st + 2 * A_BYTES + B_BYTES);
                    const uint32_t d = tmem + (uint32_t)(b * BN);
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint64_t adv = (uint64_t)(j * 32) >> 4;
                        const uint32_t acc = !(chunk_start && j == 0);
                        mma_tf32(d, ah + adv, bh + adv, idesc, acc);
                        mma_tf32(d, ah + adv, bl + adv, idesc, 1);
                        mma_tf32(d, al + adv, bh + adv, idesc, 1);
                    }
                    mma_commit(&empty[s]);
                    if (i % CHUNK_KB == CHUNK_KB - 1 || i == I.nk - 1) mma_commit(&tfull[b]);
                }
                gc += (I.nk + CHUNK_KB - 1) / CHUNK_KB;
            }
        }
    } else if (warp < 2 + EPI_WARPS) {
        // epilogue: drain each item's chunks, then store its rows
        constexpr int EC = BN < 128 ? BN : 128;
        const int q = warp & 3;
        uint32_t gc = 0;
        float* C0 = resolve<float>(p.tab, p.c);
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
                for (int c = 0; c < EC / 32; ++c) {
                    uint32_t r[32];
                    const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * BN + c * 32);
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
            gc += nchunk;
            float* C = C0 + (nsplit > 1 ? (int64_t)I.z * p.split_stride : 0);
            const LinearRows rows{I.m0, p.M, p.c_sm, p.c_rdiv, p.c_s_hi, p.c_s_lo};
            const int64_t roff = rows(q * 32 + lane);
            if (roff >= 0) {
                float* dst = C + roff;
#pragma unroll
                for (int c = 0; c < EC / 32; ++c) {
                    const int col0 = I.n0 + c * 32;
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
    } else {
        // gather thread: one row of the item's tile, lanes over 32 consecutive
        // rows; `half` picks the 16 columns of each K-block it gathers and splits
        constexpr int NH = GATHER_WARPS / 4, CW = 32 / NH, CCH = 8 / NH;  // column groups, columns / chunks each
        const int gt = threadIdx.x - (2 + EPI_WARPS) * 32;
        const int g = gt & 127, half = gt >> 7;  // tile row, column group
        const float* A = resolve<const float>(p.tab, p.a);
        const uint32_t rbase = (uint32_t)g * 128u, rsw = (uint32_t)(g & 7);
        const int ke12 = p.Ke1 * p.Ke2;
        uint32_t gk = 0;
        for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
            const Item I = item_at(it);
            const int64_t row = I.m0 + g;
            int64_t rowoff = 0;
            int hr = -(1 << 28), wr = 0;
            if (row < p.M) {  // M < 2^31
                const uint32_t e12 = (uint32_t)p.E1 * (uint32_t)p.E2, r32 = (uint32_t)row;
                const uint32_t i0 = r32 / e12, rem = r32 - i0 * e12, i1 = rem / (uint32_t)p.E2, i2 = rem - i1 * (uint32_t)p.E2;
                rowoff = (int64_t)i0 * p.ro0 + (int64_t)i1 * p.ro1 + (int64_t)i2 * p.ro2;
                if (p.pad0 == 1) {  // rows (r, s, c): the spatial offsets come from the two outer digits
                    hr = (int)(i0 * p.hm + p.h0);
                    wr = (int)(i1 * p.wm + p.w0);
                } else {
                    hr = (int)(i1 * p.hm + p.h0);
                    wr = (int)(i2 * p.wm + p.w0);
                }
            }
            const float* arow = A + rowoff;
            auto issue = [&](int i) {
                // lane's K index of this block -> (koff, dh, dw), broadcast by shuffles
                const int64_t k = (int64_t)(I.kb_begin + i) * BK + lane;
                int koff = 0, dh = -(1 << 28), dw = 0;
                if (k < p.K) {
                    const int kk = (int)k, k0 = kk / ke12, kr = kk - k0 * ke12, k1 = kr / p.Ke2, k2 = kr - k1 * p.Ke2;
                    koff = (int)(p.kbase + k0 * p.ko0 + k1 * p.ko1 + k2 * p.ko2);
                    dh = k1 * p.kh + p.dh0;
                    dw = k2 * p.kw + p.dw0;
                }
                const uint32_t dst0 = su32(raw + ((gk + i) % RAW) * A_BYTES) + rbase;
#pragma unroll 8
                for (int t = half * CW; t < half * CW + CW; ++t) {
                    const int ko = __shfl_sync(0xffffffffu, koff, t);
                    const int h = hr + __shfl_sync(0xffffffffu, dh, t), w = wr + __shfl_sync(0xffffffffu, dw, t);
                    const bool ok = (uint32_t)h < (uint32_t)p.H && (uint32_t)w < (uint32_t)p.W;
                    const float* src = ok ? arow + ko : A;
                    const uint32_t dst = dst0 + ((((uint32_t)t >> 2) ^ rsw) << 4) + ((uint32_t)t & 3u) * 4u;
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(ok ? 4u : 0u) : "memory");
                }
            };
#pragma unroll
            for (int i = 0; i < RAW; ++i) {
                if (i < I.nk) issue(i);
                cp_async_commit();
            }
            for (int i = 0; i < I.nk; ++i) {
                cp_async_wait<RAW - 1>();  // this thread's row of K-block i has landed
                const uint32_t g2 = gk + i;
                const int s = g2 % STAGES;
                mbar_wait(&empty[s], ((g2 / STAGES) & 1) ^ 1);
                const uint32_t src = su32(raw + (g2 % RAW) * A_BYTES) + rbase;
                const uint32_t dst = su32(smem + s * STAGE_BYTES) + rbase;
                // the split is elementwise and the raw ring has the stage's
                // swizzle, so each half splits the physical 16-byte slots of its
                // logical chunks in place: for fixed j the 32 lanes (rows 128 B
                // apart) hit 8 distinct slots, the 4-wavefront minimum
                float4 x[CCH];
#pragma unroll
                for (int j = 0; j < CCH; ++j) x[j] = lds128(src + (((uint32_t)(half * CCH + j) ^ rsw) << 4));
#pragma unroll
                for (int j = 0; j < CCH; ++j) {
                    const uint32_t o = ((uint32_t)(half * CCH + j) ^ rsw) << 4;
                    const float4 h = trunc_tf32(x[j]);
                    const float4 l = make_float4(__fsub_rn(x[j].x, h.x), __fsub_rn(x[j].y, h.y), __fsub_rn(x[j].z, h.z),
                                                 __fsub_rn(x[j].w, h.w));
                    sts128(dst + o, h);
                    sts128(dst + A_BYTES + o, l);
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&full[s])) : "memory");
                if (i + RAW < I.nk) issue(i + RAW);  // reuses the raw slot just consumed
                cp_async_commit();
            }
            gk += I.nk;
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
// Weight gradient over channel-last data (gfb_tcgw_args): both operands are
// loaded raw with 16-byte cp.async straight into MN-major tiles -- A rows
// (r, s, c) are contiguous channels of x, B columns contiguous channels of
// dy -- and split into TF32 hi/lo in place.  tcgen05 kind::tf32 reads
// MN-major operands only in the SWIZZLE_128B_BASE32B layout: atoms of 4 K
// rows x 128 B (32 MN elements) with 32-byte chunks XOR-swizzled by the row
// (verified by scripts/mn_probe.cu); atoms along K are SBO = 512 B apart,
// along MN LBO = 4096 B (one K-block of 8 atoms).  This replaces tcgg's
// 4-byte element gather (latency bound) and the separate TF32 split pass
// over dy that the plane form needs.
namespace tc {
template <int BN_>
struct WCfg {
    static constexpr int BM = 128, BN = BN_, BK = 32;
    static constexpr int STAGES = BN_ == 128 ? 2 : 3, RAW = BN_ == 128 ? 2 : 3;
    static constexpr int A_BYTES = BM * BK * 4, B_BYTES = BN * BK * 4;
    static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES, RAW_BYTES = A_BYTES + B_BYTES;
    static constexpr int CHUNK_KB = 4, NBUF = 512 / BN;
    static constexpr uint32_t TMEM_COLS = 512;
    static constexpr int EPI_WARPS = 4, GATHER_WARPS = BN_ == 64 ? 8 : 4;
    static constexpr int THREADS = 64 + 32 * (EPI_WARPS + GATHER_WARPS);
    static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + RAW * RAW_BYTES + 256 + 1024;
};

__device__ __forceinline__ uint64_t smem_desc_mn(uint32_t addr) {
    uint64_t d = 0;
    d |= (addr >> 4) & 0x3FFFull;          // start address
    d |= (uint64_t)(4096 >> 4) << 16;      // LBO: MN atoms
    d |= (uint64_t)(512 >> 4) << 32;       // SBO: 4-row K atoms
    d |= (uint64_t)1 << 46;                // version (sm100)
    d |= (uint64_t)1 << 61;                // SWIZZLE_128B_BASE32B
    return d;
}
// byte offset of the 16-byte piece holding MN elements mn..mn+3 (mn % 4 == 0) at K row kl
__device__ __forceinline__ uint32_t mn_piece(int mn, int kl) {
    const int mi = mn & 31;
    return (uint32_t)(mn >> 5) * 4096u + (uint32_t)(kl >> 2) * 512u + (uint32_t)(kl & 3) * 128u +
           ((uint32_t)((mi >> 3) ^ (kl & 3)) << 5) + (uint32_t)((mi >> 2) & 1) * 16u;
}
}  // namespace tc

template <int BN_>
__global__ void __launch_bounds__(tc::WCfg<BN_>::THREADS, 1) gfb_conv_tcgw_kernel(const __grid_constant__ gfb_tcgw_args p) {
    using namespace tc;
    using C_ = WCfg<BN_>;
    constexpr int BN = C_::BN, BK = C_::BK, STAGES = C_::STAGES, NBUF = C_::NBUF, RAW = C_::RAW;
    constexpr int A_BYTES = C_::A_BYTES, B_BYTES = C_::B_BYTES, STAGE_BYTES = C_::STAGE_BYTES, RAW_BYTES = C_::RAW_BYTES;
    constexpr int CHUNK_KB = C_::CHUNK_KB, EPI_WARPS = C_::EPI_WARPS, GW = C_::GATHER_WARPS;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);  // stays a shared-space pointer
    unsigned char* raw = smem + STAGES * STAGE_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(raw + RAW * RAW_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + NBUF;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + NBUF);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int kb_total = (int)((p.K + BK - 1) / BK);
    const int ntn = (int)((p.N + BN - 1) / BN), ntm = (int)((p.M + 127) / 128);
    const int nsplit = p.k_splits > 1 ? (int)p.k_splits : 1;
    const int nitems = ntn * ntm * nsplit;
    struct Item {
        int m0, n0, z, kb_begin, nk;
    };
    auto item_at = [&](int it) {
        Item r;
        const int nt = it % ntn, mt = (it / ntn) % ntm;
        r.z = it / (ntn * ntm);
        r.m0 = mt * 128;
        r.n0 = nt * BN;
        r.kb_begin = nsplit > 1 ? r.z * p.kb_per_split : 0;
        const int kb_end = nsplit > 1 ? min(kb_total, r.kb_begin + p.kb_per_split) : kb_total;
        r.nk = max(0, kb_end - r.kb_begin);
        return r;
    };

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], GW);
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

    if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_tf32(128, BN) | (1u << 15) | (1u << 16);  // MN-major A and B
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
                    const uint32_t st = su32(smem + s * STAGE_BYTES);
                    const uint64_t ah = smem_desc_mn(st), al = smem_desc_mn(st + A_BYTES);
                    const uint64_t bh = smem_desc_mn(st + 2 * A_BYTES), bl = smem_desc_mn(st + 2 * A_BYTES + B_BYTES);
                    const uint32_t d = tmem + (uint32_t)(b * BN);
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint64_t adv = (uint64_t)(j * 1024) >> 4;  // two 4-row K atoms per K = 8 step
                        const uint32_t acc = !(chunk_start && j == 0);
                        mma_tf32(d, ah + adv, bh + adv, idesc, acc);
                        mma_tf32(d, ah + adv, bl + adv, idesc, 1);
                        mma_tf32(d, al + adv, bh + adv, idesc, 1);
                    }
                    mma_commit(&empty[s]);
                    if (i % CHUNK_KB == CHUNK_KB - 1 || i == I.nk - 1) mma_commit(&tfull[b]);
                }
                gc += (I.nk + CHUNK_KB - 1) / CHUNK_KB;
            }
        }
    } else if (warp >= 2 && warp < 2 + EPI_WARPS) {
        constexpr int EC = BN < 128 ? BN : 128;
        const int q = warp & 3;
        uint32_t gc = 0;
        float* C0 = resolve<float>(p.tab, p.c);
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
                for (int c = 0; c < EC / 32; ++c) {
                    uint32_t r[32];
                    const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * BN + c * 32);
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
            gc += nchunk;
            float* C = C0 + (nsplit > 1 ? (int64_t)I.z * p.split_stride : 0);
            const LinearRows rows{I.m0, p.M, p.c_sm, p.c_rdiv, p.c_s_hi, p.c_s_lo};
            const int64_t roff = rows(q * 32 + lane);
            if (roff >= 0) {
                float* dst = C + roff;
#pragma unroll
                for (int c = 0; c < EC / 32; ++c) {
                    const int col0 = I.n0 + c * 32;
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
    } else if (warp >= 2 + EPI_WARPS) {
        // loaders: lane = 4-row group of the tile (rows 4*rg..4*rg+3 are four
        // contiguous channels of one tap), each warp KPW of a K-block's 32
        // pixels for A; B pieces (four contiguous dy channels of one pixel)
        // striped over all loader threads
        constexpr int KPW = 32 / GW, NQ = BN / 4, BPT = (32 * NQ) / (32 * GW);
        const int gt = threadIdx.x - (2 + EPI_WARPS) * 32;
        const int rg = gt & 31, gw = gt >> 5;
        const float* X = resolve<const float>(p.tab, p.a);
        const float* Y = resolve<const float>(p.tab, p.b);
        const int ke2 = p.Ke2, ke12 = p.Ke1 * p.Ke2, e12 = p.E1 * p.E2;
        uint32_t gk = 0;
        for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
            const Item I = item_at(it);
            const int row = I.m0 + 4 * rg;
            int64_t rowoff = 0;
            int hr = -(1 << 28), wr = 0;
            if (row < p.M) {
                const int i0 = row / e12, rem = row - i0 * e12, i1 = rem / p.E2, i2 = rem - i1 * p.E2;
                rowoff = i0 * p.ro0 + i1 * p.ro1 + i2 * p.ro2 + p.kbase;
                hr = i0 + p.h0;
                wr = i1 + p.w0;
            }
            const float* arow = X + rowoff;
            // lane l tracks pixel kb*32 + l as (c0, c1, c2) over (*, Ke1, Ke2):
            // one division at the item's first K-block, then carries (K-blocks
            // are issued in order, 32 pixels apart)
            int c0 = 0, c1 = 0, c2 = 0, ckb = -1;
            auto issue = [&](int i) {
                const int kb = I.kb_begin + i;
                const uint32_t slot = su32(raw + ((gk + i) % RAW) * RAW_BYTES);
                const int k = kb * BK + lane;
                if (ckb < 0) {
                    c0 = k / ke12;
                    const int kr = k - c0 * ke12;
                    c1 = kr / ke2;
                    c2 = kr - c1 * ke2;
                } else {
                    for (c2 += (kb - ckb) * BK; c2 >= ke2;) {
                        c2 -= ke2;
                        if (++c1 == p.Ke1) c1 = 0, ++c0;
                    }
                }
                ckb = kb;
                int koff = 0, yoff = -1, k1 = -(1 << 28), k2 = 0;
                if (k < p.K) {
                    k1 = c1;
                    k2 = c2;
                    koff = (int)(c0 * p.ko0 + c1 * p.ko1 + c2 * p.ko2);
                    yoff = (int)(c0 * p.yo0 + c1 * p.yo1 + c2 * p.yo2);
                }
#pragma unroll
                for (int t = 0; t < KPW; ++t) {
                    const int kl = gw * KPW + t;
                    const int ko = __shfl_sync(0xffffffffu, koff, kl);
                    const int h = hr + __shfl_sync(0xffffffffu, k1, kl), w = wr + __shfl_sync(0xffffffffu, k2, kl);
                    const bool ok = (uint32_t)h < (uint32_t)p.H && (uint32_t)w < (uint32_t)p.W;
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(slot + mn_piece(4 * rg, kl)),
                                 "l"(ok ? arow + ko : X), "r"(ok ? 16u : 0u) : "memory");
                }
#pragma unroll
                for (int u = 0; u < BPT; ++u) {
                    const int pc = gt + u * 32 * GW, kl = pc / NQ, nq = pc - kl * NQ;
                    const int yo = __shfl_sync(0xffffffffu, yoff, kl);
                    const int n = I.n0 + 4 * nq;
                    const bool ok = yo >= 0 && n < p.N;
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(slot + A_BYTES + mn_piece(4 * nq, kl)),
                                 "l"(ok ? Y + yo + n : Y), "r"(ok ? 16u : 0u) : "memory");
                }
            };
#pragma unroll
            for (int i = 0; i < RAW; ++i) {
                if (i < I.nk) issue(i);
                cp_async_commit();
            }
            for (int i = 0; i < I.nk; ++i) {
                cp_async_wait<RAW - 1>();  // this thread's pieces of K-block i have landed
                const uint32_t g2 = gk + i;
                const int s = g2 % STAGES;
                mbar_wait(&empty[s], ((g2 / STAGES) & 1) ^ 1);
                const uint32_t src = su32(raw + (g2 % RAW) * RAW_BYTES);
                const uint32_t dst = su32(smem + s * STAGE_BYTES);
                // the split is elementwise: each thread converts exactly the pieces it
                // loaded; all shared loads first (the stores' memory clobbers would
                // otherwise serialise load -> convert -> store per piece)
                float4 xa[KPW], xb[BPT];
                uint32_t oa[KPW], ob[BPT];
#pragma unroll
                for (int t = 0; t < KPW; ++t) {
                    oa[t] = mn_piece(4 * rg, gw * KPW + t);
                    xa[t] = lds128(src + oa[t]);
                }
#pragma unroll
                for (int u = 0; u < BPT; ++u) {
                    const int pc = gt + u * 32 * GW, kl = pc / NQ, nq = pc - kl * NQ;
                    ob[u] = 2 * A_BYTES + mn_piece(4 * nq, kl);
                    xb[u] = lds128(src + ob[u] - A_BYTES);
                }
#pragma unroll
                for (int t = 0; t < KPW; ++t) {
                    const float4 x = xa[t], h = trunc_tf32(x);
                    sts128(dst + oa[t], h);
                    sts128(dst + A_BYTES + oa[t], make_float4(__fsub_rn(x.x, h.x), __fsub_rn(x.y, h.y), __fsub_rn(x.z, h.z),
                                                              __fsub_rn(x.w, h.w)));
                }
#pragma unroll
                for (int u = 0; u < BPT; ++u) {
                    const float4 x = xb[u], h = trunc_tf32(x);
                    sts128(dst + ob[u], h);
                    sts128(dst + B_BYTES + ob[u], make_float4(__fsub_rn(x.x, h.x), __fsub_rn(x.y, h.y), __fsub_rn(x.z, h.z),
                                                              __fsub_rn(x.w, h.w)));
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&full[s])) : "memory");
                if (i + RAW < I.nk) issue(i + RAW);  // reuses the raw slot just consumed
                cp_async_commit();
            }
            gk += I.nk;
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
// Few-channel forward convolution (the 3-channel ResNet stem): a persistent
// implicit GEMM whose 128 rows are an 8 x 16 block of output pixels.  The
// block's input patch ((8 + R - 1) x (16 + S - 1) x C, zero outside the
// image) is staged once per tile in shared memory with plain loads; loader
// warps then build each K-block's A tile (K order (r, s, c), the filter
// planes' order) from the patch through a per-K offset table, splitting
// into TF32 hi/lo as they write.  The filter planes (K <= 160) stay
// resident in shared memory for the whole kernel (one TMA load per CTA).
// Arguments: gfb_tcg_args with C the channel count, pad[0] the channel
// stride of x, unit strides; the output row (n, y, x) is written at
// n * c_s_hi + y * c_sm + x * c_s_lo, column j at j * c_sn.
namespace tc {
struct SCfg {
    static constexpr int BM = 128, BN = 64, BK = 32, TH = 8, TW = 16;
    static constexpr int MAXKB = 5;  // K <= 160 (the filter stays resident)
    static constexpr int STAGES = 4;
    static constexpr int A_BYTES = BM * BK * 4, B_BYTES = BN * BK * 4;
    static constexpr int STAGE_BYTES = 2 * A_BYTES;
    static constexpr int BRES_BYTES = MAXKB * 2 * B_BYTES;  // resident filter hi/lo planes
    static constexpr int PATCH_FLOATS = 1536;              // (8 + R - 1)(16 + S - 1) C <= 1536
    static constexpr int NBUF = 8;
    static constexpr uint32_t TMEM_COLS = 512;
    static constexpr int EPI_WARPS = 4, LOAD_WARPS = 8;
    static constexpr int THREADS = 64 + 32 * (EPI_WARPS + LOAD_WARPS);
    static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + BRES_BYTES + 2 * PATCH_FLOATS * 4 + MAXKB * 32 * 4 + 256 + 1024;
};
}  // namespace tc

__global__ void __launch_bounds__(tc::SCfg::THREADS, 1) gfb_conv_stem_kernel(const __grid_constant__ gfb_tcg_args p) {
    using namespace tc;
    using C_ = SCfg;
    constexpr int BN = C_::BN, BK = C_::BK, TH = C_::TH, TW = C_::TW, STAGES = C_::STAGES, NBUF = C_::NBUF;
    constexpr int A_BYTES = C_::A_BYTES, B_BYTES = C_::B_BYTES, STAGE_BYTES = C_::STAGE_BYTES;
    constexpr int EPI_WARPS = C_::EPI_WARPS, LW = C_::LOAD_WARPS;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);  // stays a shared-space pointer
    unsigned char* bres = smem + STAGES * STAGE_BYTES;  // K-block kb: hi at kb * 2 * B_BYTES, lo after it
    float* patch = reinterpret_cast<float*>(bres + C_::BRES_BYTES);  // two buffers of PATCH_FLOATS
    int* ktab = reinterpret_cast<int*>(patch + 2 * C_::PATCH_FLOATS);  // patch offset of every k (-1: k >= K)
    uint64_t* full = reinterpret_cast<uint64_t*>(ktab + C_::MAXKB * 32);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + NBUF;
    uint64_t* bbar = tempty + NBUF;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bbar + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nk = (int)((p.K + BK - 1) / BK);
    const int Cc = p.C, S = p.S, R = (int)(p.K / ((int64_t)Cc * S));
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
        mbar_init(bbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                     "r"(C_::TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    // K -> patch offset table: k = (r, s, c), c fastest; patch layout [c][py][px]
    for (int k = threadIdx.x; k < C_::MAXKB * 32; k += blockDim.x) {
        int off = -1;
        if (k < p.K) {
            const int tap = k / Cc, c = k - tap * Cc, r = tap / S, s = tap - r * S;
            off = (c * PH + r) * PW + s;
        }
        ktab[k] = off;
    }
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

    if (warp == 0) {
        if (lane == 0) {  // the filter planes, once
            prefetch_tmap(p.tmap[0]);
            prefetch_tmap(p.tmap[1]);
            mbar_expect_tx(bbar, (uint32_t)(nk * 2 * B_BYTES));
            for (int kb = 0; kb < nk; ++kb) {
                tma_load_2d(bres + kb * 2 * B_BYTES, p.tmap[0], kb * BK, 0, bbar);
                tma_load_2d(bres + kb * 2 * B_BYTES + B_BYTES, p.tmap[1], kb * BK, 0, bbar);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            mbar_wait(bbar, 0);
            constexpr uint32_t idesc = idesc_tf32(128, BN);
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
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint64_t adv = (uint64_t)(j * 32) >> 4;
                        const uint32_t acc = !(kb == 0 && j == 0);
                        mma_tf32(d, ah + adv, bh + adv, idesc, acc);
                        mma_tf32(d, ah + adv, bl + adv, idesc, 1);
                        mma_tf32(d, al + adv, bh + adv, idesc, 1);
                    }
                    mma_commit(&empty[s]);
                }
                mma_commit(&tfull[b]);
            }
        }
    } else if (warp < 2 + EPI_WARPS) {
        const int q = warp & 3;
        float* C = resolve<float>(p.tab, p.c);
        uint32_t gt = 0;
        for (int it = blockIdx.x; it < nitems; it += gridDim.x, ++gt) {
            int n, y0, x0;
            item_at(it, n, y0, x0);
            const int b = gt % NBUF;
            mbar_wait(&tfull[b], (gt / NBUF) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            float acc[BN];
#pragma unroll
            for (int c = 0; c < BN / 32; ++c) {
                uint32_t r[32];
                const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * BN + c * 32);
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
                for (int j = 0; j < 32; ++j) acc[c * 32 + j] = __uint_as_float(r[j]);
            }
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&tempty[b])) : "memory");
            const int m = q * 32 + lane, y = y0 + m / TW, x = x0 + m % TW;
            if (y < p.Y && x < p.X) {
                float* dst = C + (int64_t)n * p.c_s_hi + (int64_t)y * p.c_sm + (int64_t)x * p.c_s_lo;
                if (p.c_sn == 1 && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0) && p.N == BN) {
#pragma unroll
                    for (int j = 0; j < BN; j += 4)
                        *reinterpret_cast<float4*>(dst + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
                } else {
#pragma unroll
                    for (int j = 0; j < BN; ++j)
                        if (j < p.N) dst[(int64_t)j * p.c_sn] = acc[j];
                }
            }
        }
    } else {
        // loaders: stage the tile's input patch, then build its A tiles.
        // Thread t builds row m = t & 127 of each K-block, 16-byte chunks
        // 4 (t >> 7) .. 4 (t >> 7) + 3 (half of the row's 32 columns).
        const int t = threadIdx.x - (2 + EPI_WARPS) * 32;  // 0 .. 32 * LW - 1
        const int m = t & 127, hf = t >> 7;
        const int py = m / TW, px = m % TW;
        const uint32_t rsw = (uint32_t)(m & 7);
        const float* X = resolve<const float>(p.tab, p.a);
        const int64_t xs1 = p.pad[0];
        // the next tile's patch is loaded into registers while this tile's A
        // tiles are built, so the global-load latency stays off the critical path
        constexpr int PPT = (C_::PATCH_FLOATS + 32 * LW - 1) / (32 * LW);  // patch elements per thread
        float pre[PPT];
        // this thread's patch elements (c, yy, xx) are the same for every tile
        int pyy[PPT], pxx[PPT];
        int64_t poff[PPT];
#pragma unroll
        for (int u = 0; u < PPT; ++u) {
            const int i = t + u * 32 * LW;
            const int c = i / (PH * PW), rem = i - c * (PH * PW), yy = rem / PW, xx = rem - yy * PW;
            pyy[u] = i < PSZ ? yy + p.oy : -(1 << 28);
            pxx[u] = xx + p.ox;
            poff[u] = (int64_t)c * xs1 + (int64_t)(yy + p.oy) * p.xs2 + (int64_t)(xx + p.ox) * p.xs3;
        }
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
        auto park = [&](float* pt) {
#pragma unroll
            for (int u = 0; u < PPT; ++u)
                if (t + u * 32 * LW < PSZ) pt[t + u * 32 * LW] = pre[u];
        };
        if ((int)blockIdx.x < nitems) {
            fetch(blockIdx.x);
            park(patch);
        }
        asm volatile("bar.sync 1, %0;" ::"n"(32 * LW) : "memory");
        uint32_t gk = 0, gt = 0;
        for (int it = blockIdx.x; it < nitems; it += gridDim.x, ++gt) {
            const bool more = it + (int)gridDim.x < nitems;
            if (more) fetch(it + gridDim.x);
            const float* pt = patch + (gt & 1) * C_::PATCH_FLOATS;
            const float* prow = pt + py * PW + px;
            for (int kb = 0; kb < nk; ++kb, ++gk) {
                const int s = gk % STAGES;
                mbar_wait(&empty[s], ((gk / STAGES) & 1) ^ 1);
                const uint32_t st = su32(smem + s * STAGE_BYTES) + (uint32_t)m * 128u;
                // all 16 offsets, then all 16 patch reads, then the split (no
                // load -> dependent load -> store chain per element)
                int4 ko[4];
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) ko[jj] = *reinterpret_cast<const int4*>(ktab + kb * BK + 4 * (hf * 4 + jj));
                float4 xv[4];
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    xv[jj].x = ko[jj].x >= 0 ? prow[ko[jj].x] : 0.0f;
                    xv[jj].y = ko[jj].y >= 0 ? prow[ko[jj].y] : 0.0f;
                    xv[jj].z = ko[jj].z >= 0 ? prow[ko[jj].z] : 0.0f;
                    xv[jj].w = ko[jj].w >= 0 ? prow[ko[jj].w] : 0.0f;
                }
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    const int j = hf * 4 + jj;
                    const float4 x = xv[jj], h = trunc_tf32(x);
                    const uint32_t o = ((uint32_t)j ^ rsw) << 4;
                    sts128(st + o, h);
                    sts128(st + A_BYTES + o, make_float4(__fsub_rn(x.x, h.x), __fsub_rn(x.y, h.y), __fsub_rn(x.z, h.z),
                                                         __fsub_rn(x.w, h.w)));
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&full[s])) : "memory");
            }
            // the other buffer's last readers (tile it - gridDim.x) passed the previous barrier
            if (more) park(patch + ((gt + 1) & 1) * C_::PATCH_FLOATS);
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

}  // namespace gfb


template __global__ void gfb::gfb_conv_tcgw_kernel<64>(const __grid_constant__ gfb_tcgw_args);
template __global__ void gfb::gfb_conv_tcgw_kernel<128>(const __grid_constant__ gfb_tcgw_args);
template __global__ void gfb::gfb_gemm_tc_kernel<128>(const __grid_constant__ gfb_tc_args);
template __global__ void gfb::gfb_gemm_tc_kernel<256>(const __grid_constant__ gfb_tc_args);
template __global__ void gfb::gfb_conv_tcg_kernel<64>(const __grid_constant__ gfb_tcg_args);
template __global__ void gfb::gfb_conv_tcg_kernel<128>(const __grid_constant__ gfb_tcg_args);
template __global__ void gfb::gfb_conv_tcx_kernel<64>(const __grid_constant__ gfb_tcx_args);
template __global__ void gfb::gfb_conv_tcgg_kernel<64>(const __grid_constant__ gfb_tcgg_args);
template __global__ void gfb::gfb_conv_tcgg_kernel<128>(const __grid_constant__ gfb_tcgg_args);
template __global__ void gfb::gfb_conv_tcx_kernel<128>(const __grid_constant__ gfb_tcx_args);

extern "C" const void* gfb_tc_kernel_ptr(int kind) {
    if (kind == GFB_K_DOT_TC32) return (const void*)gfb::gfb_gemm_tc_kernel<128>;
    if (kind == GFB_K_DOT_TC32W) return (const void*)gfb::gfb_gemm_tc_kernel<256>;
    if (kind == GFB_K_DOT_TC32P) return (const void*)gfb::gfb_gemm_tc2_kernel;
    if (kind == GFB_K_SPLIT_TF32) return (const void*)gfb::gfb_split_kernel;
    if (kind == GFB_K_CONV_TCG64) return (const void*)gfb::gfb_conv_tcg_kernel<64>;
    if (kind == GFB_K_CONV_TCG128) return (const void*)gfb::gfb_conv_tcg_kernel<128>;
    if (kind == GFB_K_CONV_TCX64) return (const void*)gfb::gfb_conv_tcx_kernel<64>;
    if (kind == GFB_K_CONV_TCGG64) return (const void*)gfb::gfb_conv_tcgg_kernel<64>;
    if (kind == GFB_K_CONV_TCGG128) return (const void*)gfb::gfb_conv_tcgg_kernel<128>;
    if (kind == GFB_K_CONV_TCX128) return (const void*)gfb::gfb_conv_tcx_kernel<128>;
    if (kind == GFB_K_CONV_TCGW64) return (const void*)gfb::gfb_conv_tcgw_kernel<64>;
    if (kind == GFB_K_CONV_STEM64) return (const void*)gfb::gfb_conv_stem_kernel;
    if (kind == GFB_K_CONV_TCGW128) return (const void*)gfb::gfb_conv_tcgw_kernel<128>;
    return nullptr;
}

extern "C" int gfb_tc_smem_bytes(int wide) { return wide ? gfb::tc::Cfg<256>::SMEM_BYTES : gfb::tc::Cfg<128>::SMEM_BYTES; }
extern "C" int gfb_tc_pair_smem_bytes(void) { return gfb::tc::PCfg::SMEM_BYTES_PAIR; }
extern "C" int gfb_tcgw_smem_bytes(int bn) { return bn == 64 ? gfb::tc::WCfg<64>::SMEM_BYTES : gfb::tc::WCfg<128>::SMEM_BYTES; }
extern "C" int gfb_stem_smem_bytes(void) { return gfb::tc::SCfg::SMEM_BYTES; }
extern "C" int gfb_tcg_smem_bytes(int bn) { return bn == 64 ? gfb::tc::GCfg<64>::SMEM_BYTES : gfb::tc::GCfg<128>::SMEM_BYTES; }
