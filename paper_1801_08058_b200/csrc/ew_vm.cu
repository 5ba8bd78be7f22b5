// Fused elementwise / Broadcast / Reshape / ConvertLayout / Sum kernels.
//
// The compile pass (paper_1801_08058_b200/compiler.py) turns each fusion
// group of memory-bound IR nodes into one *program* for this kernel: a short
// accumulator-stack bytecode over "leaves" (loads / stores through
// mixed-radix index maps, gfb200.h gfb_digit).  One launch evaluates the
// whole group in a single pass over HBM over a 2-level index space (o, r):
//   ROW  one warp (or `wpr` warps) per o, lanes take V-vectors along r
//   COL  one thread per V-vector of o, r looped (split `split` ways)
// with an optional fold over r (Sum / max-reduce).  Side outputs (STORE)
// write intermediates the graph also needs, so config B's
// `t3 = Relu(a + Broadcast(c)) * b` and `Sum(t3)` are one read of a and b and
// one write of t3.
//
// Arithmetic follows the reference contract (numeric.py / kernels.py):
// F32 + - x / are IEEE round-to-nearest with no contraction (__f*_rn), so
// they are bit-exact with the reference's double-then-round; Exp / Log / Tanh
// / Sigmoid are evaluated in double and rounded once to F32 like
// `round_f32(math.exp(x))`; Maximum is the literal `x >= y ? x : y` and Relu
// `x > 0 ? x : 0`; I64 wraps.  No --use_fast_math, no FTZ (sigmoid(-100)
// in F32 is a subnormal).
//
// Interpreter cost is kept off the memory path: leaf base offsets for the
// thread's o are computed once (shared memory), the per-vector r offset is
// r * rlin, the first `npre` leaves of every vector are loaded before the
// program runs (all in flight together, 128-bit accesses), and the operand
// stack lives in shared memory so the register file holds only data.

#include <cuda_runtime.h>

#include "ew_ops.cuh"

namespace gfb {

// Per-block shared state.
struct Shared {
    const char* base[GFB_MAX_LEAVES];  // slot pointer + byte offset of every leaf
};

__device__ __forceinline__ uint32_t part_offset(const gfb_leaf& L, uint32_t idx, int src) {
    uint32_t off = 0;
    const int n = L.ndig;
#pragma unroll 1
    for (int i = 0; i < n; ++i) {
        const gfb_digit& d = L.dig[i];
        if (d.src != src) continue;
        uint32_t q = fast_div(idx, (uint32_t)d.div_mul, d.div_sh);
        if (d.mod) q -= fast_div(q, (uint32_t)d.mod_mul, d.mod_sh) * d.mod;
        off += q * (uint32_t)d.stride;
    }
    return off;
}

__device__ __forceinline__ uint32_t r_offset(const gfb_leaf& L, uint32_t r) {
    const int rl = L.rlin;
    return rl >= 0 ? r * (uint32_t)rl : part_offset(L, r, 1);
}

// Thread context: the vector at (o, r) with nvalid live lanes.
template <typename T, int V>
struct Ctx {
    const gfb_ew_args& p;
    const char* const* base;  // Shared::base
    const uint32_t* ob;       // per-thread o-part offsets, stride `obs`
    int obs;
    T* stack;                 // per-thread stack, element stride `obs`
    uint32_t o, r;
    int nvalid, vaxis;
    const uint32_t* rb = nullptr;  // ROW with cache_r: r-part offsets of the current vector, stride `obs`

    __device__ __forceinline__ uint32_t roff(const gfb_leaf& L, int k) const { return rb ? rb[k * obs] : r_offset(L, r); }

    __device__ __forceinline__ void load(int k, T (&out)[V]) const {
        const gfb_leaf& L = p.leaves[k];
        if (L.mode == 1) {
            const T s = from_bits<T>(L.splat);
#pragma unroll
            for (int v = 0; v < V; ++v) out[v] = s;
            return;
        }
        const T* bp = reinterpret_cast<const T*>(base[k]);
        if (nvalid == V && L.vec != 0) {
            const uint32_t off = ob[k * obs] + roff(L, k);
            if (L.vec == 1) {
                loadV<T, V>(bp + off, out);
            } else if (L.vec == 3) {  // patterned vector: element v at off + dv[v]
#pragma unroll
                for (int v = 0; v < V; ++v) out[v] = __ldg(bp + (int32_t)off + L.dv[v]);
            } else {
                const T s = __ldg(bp + off);
#pragma unroll
                for (int v = 0; v < V; ++v) out[v] = s;
            }
            return;
        }
#pragma unroll
        for (int v = 0; v < V; ++v)
            out[v] = v < nvalid ? __ldg(bp + leaf_offset(L, o + (vaxis ? 0 : v), r + (vaxis ? v : 0))) : T(0);
    }

    __device__ __forceinline__ void store(int k, const T (&val)[V]) const {
        const gfb_leaf& L = p.leaves[k];
        T* bp = reinterpret_cast<T*>(const_cast<char*>(base[k]));
        if (nvalid == V && L.vec == 1) {
            storeV<T, V>(bp + ob[k * obs] + roff(L, k), val);
            return;
        }
        if (nvalid == V && L.vec == 3) {
            const int32_t off = (int32_t)(ob[k * obs] + roff(L, k));
#pragma unroll
            for (int v = 0; v < V; ++v) bp[off + L.dv[v]] = val[v];
            return;
        }
#pragma unroll
        for (int v = 0; v < V; ++v)
            if (v < nvalid) bp[leaf_offset(L, o + (vaxis ? 0 : v), r + (vaxis ? v : 0))] = val[v];
    }
};

// Register-cached addressing of a preloaded leaf for the thread's current o.
template <typename T>
struct Pre {
    const T* ptr;  // leaf base + o-part offset
    int rl;        // r-part = r * rl (-1: general digits)
    int vec;       // 1 contiguous, 2 uniform, 0 gather
};

template <typename T, int V>
__device__ __forceinline__ void setup_pre(const Ctx<T, V>& c, Pre<T> (&pr)[4]) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (k < c.p.npre) {
            const gfb_leaf& L = c.p.leaves[k];
            pr[k].ptr = reinterpret_cast<const T*>(c.base[k]) + c.ob[k * c.obs];
            pr[k].rl = L.rlin;
            pr[k].vec = (L.mode == 1 || L.vec == 3) ? 0 : L.vec;  // splats / strided vectors: generic path
        }
    }
}

template <typename T, int V>
__device__ __forceinline__ void load_pre(const Ctx<T, V>& c, const Pre<T>& q, int k, T (&out)[V]) {
    if (c.nvalid == V && q.vec != 0 && q.rl >= 0) {
        const T* a = q.ptr + c.r * (uint32_t)q.rl;
        if (q.vec == 1) {
            loadV<T, V>(a, out);
        } else {
            const T x = __ldg(a);
#pragma unroll
            for (int v = 0; v < V; ++v) out[v] = x;
        }
    } else {
        c.load(k, out);
    }
}

// Run the program on the context's vector; leaves the last value in acc.
template <typename T, int V>
__device__ __forceinline__ void vm_run(const Ctx<T, V>& c, const Pre<T> (&pr)[4], T (&acc)[V]) {
    const gfb_ew_args& p = c.p;
    const int npre = p.npre;
    T p0[V], p1[V], p2[V], p3[V];
    if (npre > 0) load_pre<T, V>(c, pr[0], 0, p0);
    if (npre > 1) load_pre<T, V>(c, pr[1], 1, p1);
    if (npre > 2) load_pre<T, V>(c, pr[2], 2, p2);
    if (npre > 3) load_pre<T, V>(c, pr[3], 3, p3);
    int sp = 0;
    const uint32_t n = p.ninstr;
#define GFB_APPLY(OPC, S, B) \
    _Pragma("unroll") for (int v = 0; v < V; ++v) acc[v] = (S) ? bin1<T>(OPC, B[v], acc[v]) : bin1<T>(OPC, acc[v], B[v]);
#define GFB_CASE(SRC, OPC, S, PREP, B)                 \
    case F_BIN + ((SRC) * 5 + (OPC)) * 2 + (S): {      \
        PREP                                          \
        GFB_APPLY(OPC, S, B)                          \
        break;                                        \
    }
#define GFB_OPS(SRC, PREP, B)                                                     \
    GFB_CASE(SRC, OP_ADD, 0, PREP, B) GFB_CASE(SRC, OP_ADD, 1, PREP, B)           \
    GFB_CASE(SRC, OP_SUB, 0, PREP, B) GFB_CASE(SRC, OP_SUB, 1, PREP, B)           \
    GFB_CASE(SRC, OP_MUL, 0, PREP, B) GFB_CASE(SRC, OP_MUL, 1, PREP, B)           \
    GFB_CASE(SRC, OP_DIV, 0, PREP, B) GFB_CASE(SRC, OP_DIV, 1, PREP, B)           \
    GFB_CASE(SRC, OP_MAX, 0, PREP, B) GFB_CASE(SRC, OP_MAX, 1, PREP, B)
#define GFB_PREP_NONE
#define GFB_PREP_MEM T b[V]; c.load(k, b);
#define GFB_PREP_POP                                                        \
    T b[V];                                                                 \
    --sp;                                                                   \
    _Pragma("unroll") for (int v = 0; v < V; ++v) b[v] = c.stack[(sp * V + v) * c.obs];
#define GFB_UN(OPC) \
    case F_UN + (OPC) - OP_NEG: apply_unary<T, V>(OPC, acc); break;
#pragma unroll 1
    for (uint32_t pc = 0; pc < n; ++pc) {
        const uint32_t ins = p.prog[pc];
        const int k = (int)((ins >> 8) & 0xffu);
        switch (ins & 0xffu) {
            case F_LOADP + 0: copyV<T, V>(acc, p0); break;
            case F_LOADP + 1: copyV<T, V>(acc, p1); break;
            case F_LOADP + 2: copyV<T, V>(acc, p2); break;
            case F_LOADP + 3: copyV<T, V>(acc, p3); break;
            case F_LOADM: c.load(k, acc); break;
            case F_PUSH:
#pragma unroll
                for (int v = 0; v < V; ++v) c.stack[(sp * V + v) * c.obs] = acc[v];
                ++sp;
                break;
            case F_STORE: c.store(k, acc); break;
            case F_DOT: {  // acc = acc + leaf[k] * leaf[k2]: one tiny-Dot term (two roundings)
                const int k2 = (int)((ins >> 16) & 0xffu);
                T a[V], b[V];  // the compiler keeps multiply-add operands out of the preload set
                c.load(k, a);
                c.load(k2, b);
#pragma unroll
                for (int v = 0; v < V; ++v) acc[v] = bin1<T>(OP_ADD, acc[v], bin1<T>(OP_MUL, a[v], b[v]));
                break;
            }
            GFB_UN(OP_NEG) GFB_UN(OP_EXP) GFB_UN(OP_LOG) GFB_UN(OP_TANH) GFB_UN(OP_SIGMOID) GFB_UN(OP_RELU)
            GFB_OPS(0, GFB_PREP_NONE, p0)
            GFB_OPS(1, GFB_PREP_NONE, p1)
            GFB_OPS(2, GFB_PREP_NONE, p2)
            GFB_OPS(3, GFB_PREP_NONE, p3)
            GFB_OPS(4, GFB_PREP_MEM, b)
            GFB_OPS(5, GFB_PREP_POP, b)
            GFB_OPS(6, GFB_PREP_NONE, acc)
            default: __trap();
        }
    }
#undef GFB_APPLY
#undef GFB_CASE
#undef GFB_OPS
#undef GFB_PREP_NONE
#undef GFB_PREP_MEM
#undef GFB_PREP_POP
#undef GFB_UN
}

// Dynamic shared memory: [ob: nleaves x blockDim u32][stack: depth*V x blockDim T][fold: V x blockDim T]
// __launch_bounds__(256, 4): occupancy over registers.  The V-wide variants
// spill a little at 64 registers and still measured faster on configs A, C
// and D than at 80 / 110 registers (the general VM is latency bound).
template <typename T, int V>
__global__ void __launch_bounds__(256, 4) gfb_ew_kernel(const __grid_constant__ gfb_ew_args p) {
    __shared__ Shared sh;
    extern __shared__ __align__(128) unsigned char dyn[];
    const int nthr = blockDim.x, tid = threadIdx.x;
    const int nleaves = p.nleaves;
    uint32_t* ob = reinterpret_cast<uint32_t*>(dyn) + tid;
    const int nofs = p.pad ? 2 * nleaves : nleaves;  // o-part (+ cached r-part) offsets
    T* stack = reinterpret_cast<T*>(dyn + sizeof(uint32_t) * nofs * nthr) + tid;
    T* scratch = reinterpret_cast<T*>(dyn + sizeof(uint32_t) * nofs * nthr + sizeof(T) * p.depth * V * nthr);
    if (tid < nleaves) {
        const gfb_leaf& L = p.leaves[tid];
        sh.base[tid] = L.mode == 1 ? nullptr : reinterpret_cast<const char*>(p.tab[L.ref >> 56]) + (L.ref & kOffsetMask);
    }
    __syncthreads();
    const int kind = p.red_kind;

    if (p.mode == 1) {
        // ROW: `wpr` warps per o, lanes along r.  Loop bounds are block-uniform
        // so the cross-warp combine may use __syncthreads.
        const int lane = tid & 31, warp = tid >> 5;
        const int wpr = p.wpr, rpb = (nthr >> 5) / wpr;
        const int sub = warp % wpr, slot = warp / wpr;
        const uint32_t rstep = 32u * V * wpr, nr = p.n_r;
        T* red = kind ? resolve<T>(p.tab, p.red_out.ref) : nullptr;
        for (uint32_t o0 = blockIdx.x * rpb; o0 < p.n_o; o0 += gridDim.x * rpb) {
            const uint32_t o = o0 + slot;
            const bool active = o < p.n_o;
            T part = fold_init<T>(kind);
            if (active) {
                for (int k = 0; k < nleaves; ++k) {
                    const int sm = p.leaves[k].same;
                    ob[k * nthr] = sm >= 0 ? ob[sm * nthr] : part_offset(p.leaves[k], o, 0);
                }
                Ctx<T, V> c{p, sh.base, ob, nthr, stack, o, 0, V, 1};
                Pre<T> pr[4];
                setup_pre<T, V>(c, pr);
                for (uint32_t rl = (sub * 32u + lane) * V; rl < nr; rl += rstep) {
                    uint32_t r = rl;
                    if (p.ty_ext) {  // transposing order along r (see gfb_ew_args)
                        const uint32_t w = rl / V, xblocks = (uint32_t)p.ty_div / V;
                        const uint32_t y = w % (uint32_t)p.ty_ext, t = w / (uint32_t)p.ty_ext;
                        r = ((t / xblocks) * (uint32_t)p.ty_ext + y) * (uint32_t)p.ty_div + (t % xblocks) * V;
                    }
                    c.r = r;
                    c.nvalid = (int)min((uint32_t)V, nr - r);
                    if (p.pad) {  // cache_r: general r-part offsets once per vector, shared by equal maps
                        uint32_t* rbw = ob + nleaves * nthr;
                        for (int k = 0; k < nleaves; ++k) {
                            const gfb_leaf& L = p.leaves[k];
                            const int sm = L.same;
                            rbw[k * nthr] = sm >= 0 ? rbw[sm * nthr] : r_offset(L, r);
                        }
                        c.rb = rbw;
                    }
                    T acc[V];
                    vm_run<T, V>(c, pr, acc);
                    if (kind) {
#pragma unroll
                        for (int v = 0; v < V; ++v)
                            if (v < c.nvalid) part = fold<T>(kind, part, acc[v]);
                    }
                }
            }
            if (!kind) continue;
            if constexpr (sizeof(T) > 1) {
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) part = fold<T>(kind, part, __shfl_xor_sync(0xffffffffu, part, off));
                if (wpr > 1) {
                    if (lane == 0) scratch[warp] = part;
                    __syncthreads();
                    if (active && sub == 0 && lane == 0) {
                        for (int s = 1; s < wpr; ++s) part = fold<T>(kind, part, scratch[warp + s]);
                        red[leaf_offset(p.red_out, o, 0)] = part;
                    }
                    __syncthreads();
                } else if (active && lane == 0) {
                    red[leaf_offset(p.red_out, o, 0)] = part;
                }
            }
        }
        return;
    }

    // COL: one thread per V-vector of o, r looped, split `split` ways.
    const uint32_t split = p.split;
    const uint32_t per_row = nthr / split;
    const uint32_t lane_o = tid % per_row, rs = tid / per_row;
    const uint32_t o_stride = gridDim.x * per_row * V;
    const uint32_t ty_ext = (uint32_t)p.ty_ext, ty_div = (uint32_t)p.ty_div;
    for (uint32_t o0 = (blockIdx.x * per_row) * V; o0 < p.n_o; o0 += o_stride) {
        const uint32_t olin = o0 + lane_o * V;
        const bool active = olin < p.n_o;
        uint32_t o = olin;
        if (ty_ext && active) {  // transposing order: vector w -> (rest, x block, y) with y fastest
            const uint32_t w = olin / V, xblocks = ty_div / V;
            const uint32_t y = w % ty_ext, t = w / ty_ext, xb = t % xblocks, rest = t / xblocks;
            o = (rest * ty_ext + y) * ty_div + xb * V;
        }
        const int nvalid = active ? (int)min((uint32_t)V, p.n_o - o) : 0;
        T part[V];
#pragma unroll
        for (int v = 0; v < V; ++v) part[v] = fold_init<T>(kind);
        if (active) {
            for (int k = 0; k < nleaves; ++k) {
                const int sm = p.leaves[k].same;  // operands sharing an index map share its offset
                ob[k * nthr] = sm >= 0 ? ob[sm * nthr] : part_offset(p.leaves[k], o, 0);
            }
            Ctx<T, V> c{p, sh.base, ob, nthr, stack, o, 0, nvalid, 0};
            Pre<T> pr[4];
            setup_pre<T, V>(c, pr);
            for (uint32_t r = rs; r < p.n_r; r += split) {
                c.r = r;
                T acc[V];
                vm_run<T, V>(c, pr, acc);
                if (kind) {
#pragma unroll
                    for (int v = 0; v < V; ++v) part[v] = fold<T>(kind, part[v], acc[v]);
                }
            }
        }
        if (!kind) continue;
        if (split > 1) {
            __syncthreads();
#pragma unroll
            for (int v = 0; v < V; ++v) scratch[v * nthr + tid] = part[v];
            __syncthreads();
            if (rs == 0) {
                for (uint32_t s = 1; s < split; ++s)
#pragma unroll
                    for (int v = 0; v < V; ++v) part[v] = fold<T>(kind, part[v], scratch[v * nthr + s * per_row + lane_o]);
            }
        }
        if (active && rs == 0) {
            const gfb_leaf& L = p.red_out;
            T* bp = resolve<T>(p.tab, L.ref);
            if (nvalid == V && L.vec == 1) {
                storeV<T, V>(bp + part_offset(L, o, 0), part);
            } else {
#pragma unroll
                for (int v = 0; v < V; ++v)
                    if (v < nvalid) bp[leaf_offset(L, o + v, 0)] = part[v];
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Staged ROW kernel (mode 3): the Blackwell path for row-contiguous programs.
//
// Each warp walks (row, chunk) pairs; lane 0 streams the next chunk of every
// preloaded leaf into a per-warp, double-buffered shared-memory stage with
// cp.async.bulk (TMA bulk copies completing on an mbarrier) while the warp
// computes on the current one.  A VM instruction is dispatched once per
// U x V elements per thread, operands come from shared memory, leaves that
// do not depend on r (e.g. a column Broadcast) are per-row scalars, and the
// accumulator stays in registers.  Requirements (checked by the compiler):
// no operand stack, every memory leaf preloaded (<= 4), staged leaves with
// r-stride 1 and 16-byte aligned rows.

__device__ __forceinline__ void fence_proxy() {
    // generic-proxy reads of a stage must complete before the async proxy rewrites it
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra WAIT_%=;\n}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

constexpr uint32_t kResidentBytes = 8192;  // block-resident leaf budget (per leaf)

template <typename T, int U_>
struct StagedCfg {
    static constexpr int HV = 16 / sizeof(T);  // elements per 16-byte half
    static constexpr int V = 2 * HV;           // elements per thread per sub-vector
    static constexpr int U = U_;               // sub-vectors per dispatch
    static constexpr int CH = 32 * V * U;      // elements per warp chunk
};

// element index (within a chunk) of (u, half h, j) for `lane`
template <typename T>
__device__ __forceinline__ int sidx(int u, int h, int lane, int j) {
    constexpr int HV = 16 / sizeof(T), V = 2 * HV;
    return u * 32 * V + h * 32 * HV + lane * HV + j;
}

// U = sub-vectors per thread per dispatch (a 512-float chunk per warp item;
// smaller chunks measured 1.7x slower: per-item issue/wait overhead), NS =
// depth of each warp's stage ring (2 measured best: deeper rings cost warps).
// __launch_bounds__(256, 3): the shared-memory budget fits three blocks per
// SM; the hint (62 registers) measured 150.7 -> 137.5 us on config B.
template <typename T, int U_, int NS_>
__global__ void __launch_bounds__(256, 3) gfb_ew_staged_kernel(const __grid_constant__ gfb_ew_args p) {
    using Cfg = StagedCfg<T, U_>;
    constexpr int HV = Cfg::HV, V = Cfg::V, U = Cfg::U, CH = Cfg::CH;
    extern __shared__ __align__(128) unsigned char dyn[];
    constexpr int MAXST = 4;
    __shared__ uint64_t bars[8][MAXST];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int npre = p.npre, kind = p.red_kind;
    constexpr int NS = NS_;  // ring depth (stages per warp)
    const uint32_t n_o = p.n_o, n_r = p.n_r;
    // leaf classes (uniform): 1 = staged per item (r-contiguous), 2 = row
    // scalar, 3 = splat, 4 = block-resident (r-contiguous, independent of
    // o, e.g. a row Broadcast of a bias: copied into shared memory once per
    // block instead of once per item).  Staged / resident leaves get
    // consecutive slots in their regions.
    const uint32_t n_r_pad = (n_r + CH - 1) / CH * CH;
    int cls[4], slot[4], nst = 0, nres = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        cls[k] = 0;
        slot[k] = 0;
        if (k < npre) {
            const gfb_leaf& L = p.leaves[k];
            cls[k] = L.mode == 1 ? 3 : (L.rlin == 1 ? 1 : 2);
            if (cls[k] == 1) {
                bool o_free = true;
                for (int i = 0; i < L.ndig; ++i) o_free &= L.dig[i].src == 1;
                if (o_free && n_r_pad * sizeof(T) <= kResidentBytes) cls[k] = 4;
            }
            if (cls[k] == 1) slot[k] = nst++;
            if (cls[k] == 4) slot[k] = nres++;
        }
    }
    // dynamic smem: [resident: nres x n_r_pad][per-warp stages: NS x nst x CH]
    T* res0 = reinterpret_cast<T*>(dyn);
    T* stage0 = res0 + (size_t)nres * n_r_pad + (size_t)warp * NS * nst * CH;
    __shared__ uint64_t rbar;
    if (lane == 0) {
        for (int st = 0; st < NS; ++st) mbar_init(&bars[warp][st], 1);
        if (warp == 0) mbar_init(&rbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0 && nres) {
        mbar_expect_tx(&rbar, (uint32_t)(nres * n_r * sizeof(T)));
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (k < npre && cls[k] == 4) {
                const gfb_leaf& L = p.leaves[k];
                bulk_g2s(res0 + (size_t)slot[k] * n_r_pad,
                         reinterpret_cast<const char*>(p.tab[L.ref >> 56]) + (L.ref & kOffsetMask),
                         (uint32_t)(n_r * sizeof(T)), &rbar);
            }
    }
    const uint32_t gw = blockIdx.x * (blockDim.x >> 5) + warp, tw = gridDim.x * (blockDim.x >> 5);
    const uint32_t nch = (n_r + CH - 1) / CH;
    // Work items are (o, chunk).  Row-wise (split == 0): a warp owns whole
    // rows (o = gw, gw + tw, ...) and folds them itself.  Chunk-wise
    // (split == 1, few long rows): items gw, gw + tw, ... of the flattened
    // (o, chunk) space, and a fold writes one partial per chunk to
    // red_out[o * nch + chunk] for a second, deterministic pass.
    const bool chunkwise = p.split == 1;
    uint32_t total;
    if (chunkwise) {
        const uint32_t items = n_o * nch;
        total = gw < items ? (items - gw + tw - 1) / tw : 0;
    } else {
        total = gw < n_o ? ((n_o - gw + tw - 1) / tw) * nch : 0;
    }
    if (total == 0) return;
    auto item_of = [&](uint32_t it, uint32_t& o, uint32_t& chunk) {
        if (chunkwise) {
            const uint32_t g = gw + it * tw;
            o = g / nch;
            chunk = g % nch;
        } else {
            o = gw + (it / nch) * tw;
            chunk = it % nch;
        }
    };
    const char* lbase[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
        lbase[k] = (k < npre && cls[k] != 3) ? reinterpret_cast<const char*>(p.tab[p.leaves[k].ref >> 56]) + (p.leaves[k].ref & kOffsetMask) : nullptr;

    auto issue = [&](uint32_t it) {
        uint32_t o, chunk;
        item_of(it, o, chunk);
        const uint32_t r0 = chunk * CH, len = min((uint32_t)CH, n_r - r0);
        const int st = it % NS;
        if (lane == 0) {
            fence_proxy();
            mbar_expect_tx(&bars[warp][st], len * sizeof(T) * nst);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (k < npre && cls[k] == 1) {
                    const T* src = reinterpret_cast<const T*>(lbase[k]) + part_offset(p.leaves[k], o, 0) + r0;
                    bulk_g2s(stage0 + ((size_t)st * nst + slot[k]) * CH, src, len * sizeof(T), &bars[warp][st]);
                }
            }
        }
    };

    for (int k = 0; k < NS && (uint32_t)k < total; ++k) issue(k);
    if (nres) mbar_wait(&rbar, 0);
    uint32_t phase_bits = 0;  // bit st = parity of stage st
    T part = fold_init<T>(kind);
    T rs[4];  // row scalars
    uint32_t cur_o = 0xffffffffu;
    for (uint32_t it = 0; it < total; ++it) {
        const int st = it % NS;
        uint32_t o, chunk;
        item_of(it, o, chunk);
        const uint32_t r0 = chunk * CH, len = min((uint32_t)CH, n_r - r0);
        if (o != cur_o) {
            cur_o = o;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (k < npre && cls[k] == 2)
                    rs[k] = __ldg(reinterpret_cast<const T*>(lbase[k]) + part_offset(p.leaves[k], o, 0));
                else if (k < npre && cls[k] == 3)
                    rs[k] = from_bits<T>(p.leaves[k].splat);
            }
        }
        mbar_wait(&bars[warp][st], (phase_bits >> st) & 1u);
        phase_bits ^= 1u << st;
        const T* sb = stage0 + (size_t)st * nst * CH;
        const bool full = len == (uint32_t)CH;

        T acc[U][V];
        auto operand = [&](int k, int u, T(&b)[V]) {
            if (cls[k] == 1 || cls[k] == 4) {
                const T* src = cls[k] == 1 ? sb + slot[k] * CH : res0 + (size_t)slot[k] * n_r_pad + r0;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int4 q = *reinterpret_cast<const int4*>(src + sidx<T>(u, h, lane, 0));
                    const T* qq = reinterpret_cast<const T*>(&q);
#pragma unroll
                    for (int j = 0; j < HV; ++j) b[h * HV + j] = qq[j];
                }
            } else {
#pragma unroll
                for (int v = 0; v < V; ++v) b[v] = rs[k];
            }
        };
        const uint32_t n = p.ninstr;
#define GFB_S_APPLY(OPC, S, B) \
    _Pragma("unroll") for (int v = 0; v < V; ++v) acc[u][v] = (S) ? bin1<T>(OPC, B[v], acc[u][v]) : bin1<T>(OPC, acc[u][v], B[v]);
#define GFB_S_CASE(SRC, OPC, S)                                    \
    case F_BIN + ((SRC) * 5 + (OPC)) * 2 + (S):                    \
        _Pragma("unroll") for (int u = 0; u < U; ++u) {            \
            T b[V];                                                \
            operand(SRC, u, b);                                    \
            GFB_S_APPLY(OPC, S, b)                                 \
        }                                                          \
        break;
#define GFB_S_OPS(SRC)                                                           \
    GFB_S_CASE(SRC, OP_ADD, 0) GFB_S_CASE(SRC, OP_ADD, 1)                        \
    GFB_S_CASE(SRC, OP_SUB, 0) GFB_S_CASE(SRC, OP_SUB, 1)                        \
    GFB_S_CASE(SRC, OP_MUL, 0) GFB_S_CASE(SRC, OP_MUL, 1)                        \
    GFB_S_CASE(SRC, OP_DIV, 0) GFB_S_CASE(SRC, OP_DIV, 1)                        \
    GFB_S_CASE(SRC, OP_MAX, 0) GFB_S_CASE(SRC, OP_MAX, 1)
#define GFB_S_SELF(OPC) \
    case F_BIN + ((SRC_SELF_) * 5 + (OPC)) * 2: \
        _Pragma("unroll") for (int u = 0; u < U; ++u) { GFB_S_APPLY(OPC, 0, acc[u]) } break;
#define GFB_S_UN(OPC) \
    case F_UN + (OPC) - OP_NEG: _Pragma("unroll") for (int u = 0; u < U; ++u) apply_unary<T, V>(OPC, acc[u]); break;
        constexpr int SRC_SELF_ = 6;
#pragma unroll 1
        for (uint32_t pc = 0; pc < n; ++pc) {
            const uint32_t ins = p.prog[pc];
            const int k = (int)((ins >> 8) & 0xffu);
            switch (ins & 0xffu) {
                case F_LOADP + 0:
#pragma unroll
                    for (int u = 0; u < U; ++u) operand(0, u, acc[u]);
                    break;
                case F_LOADP + 1:
#pragma unroll
                    for (int u = 0; u < U; ++u) operand(1, u, acc[u]);
                    break;
                case F_LOADP + 2:
#pragma unroll
                    for (int u = 0; u < U; ++u) operand(2, u, acc[u]);
                    break;
                case F_LOADP + 3:
#pragma unroll
                    for (int u = 0; u < U; ++u) operand(3, u, acc[u]);
                    break;
                case F_STORE: {
                    const gfb_leaf& L = p.leaves[k];
                    T* dst = resolve<T>(p.tab, L.ref);
                    if (full && L.rlin == 1) {
                        T* row = dst + part_offset(L, o, 0) + r0;
#pragma unroll
                        for (int u = 0; u < U; ++u)
#pragma unroll
                            for (int h = 0; h < 2; ++h) {
                                int4 q;
                                T* qq = reinterpret_cast<T*>(&q);
#pragma unroll
                                for (int j = 0; j < HV; ++j) qq[j] = acc[u][h * HV + j];
                                *reinterpret_cast<int4*>(row + sidx<T>(u, h, lane, 0)) = q;
                            }
                    } else {
#pragma unroll
                        for (int u = 0; u < U; ++u)
#pragma unroll
                            for (int h = 0; h < 2; ++h)
#pragma unroll
                                for (int j = 0; j < HV; ++j) {
                                    const uint32_t e = sidx<T>(u, h, lane, j);
                                    if (e < len) dst[leaf_offset(L, o, r0 + e)] = acc[u][h * HV + j];
                                }
                    }
                    break;
                }
                GFB_S_UN(OP_NEG) GFB_S_UN(OP_EXP) GFB_S_UN(OP_LOG) GFB_S_UN(OP_TANH) GFB_S_UN(OP_SIGMOID) GFB_S_UN(OP_RELU)
                GFB_S_OPS(0) GFB_S_OPS(1) GFB_S_OPS(2) GFB_S_OPS(3)
                GFB_S_SELF(OP_ADD) GFB_S_SELF(OP_SUB) GFB_S_SELF(OP_MUL) GFB_S_SELF(OP_DIV) GFB_S_SELF(OP_MAX)
                default: __trap();  // the compiler never emits other opcodes here
            }
        }
#undef GFB_S_APPLY
#undef GFB_S_CASE
#undef GFB_S_OPS
#undef GFB_S_SELF
#undef GFB_S_UN
        if (kind) {
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int j = 0; j < HV; ++j)
                        if (full || sidx<T>(u, h, lane, j) < (int)len) part = fold<T>(kind, part, acc[u][h * HV + j]);
            if (chunkwise || chunk == nch - 1) {
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) part = fold<T>(kind, part, __shfl_xor_sync(0xffffffffu, part, off));
                if (lane == 0) {
                    T* red = resolve<T>(p.tab, p.red_out.ref);
                    if (chunkwise) red[(size_t)o * nch + chunk] = part;  // scratch partials
                    else red[leaf_offset(p.red_out, o, 0)] = part;
                }
                part = fold_init<T>(kind);
            }
        }
        __syncwarp();
        if (it + NS < total) issue(it + NS);
    }
}

template __global__ void gfb_ew_staged_kernel<float, 2, 2>(const __grid_constant__ gfb_ew_args);

// A row-fused launch (GFB_K_ROWJIT) only ever runs its runtime-generated
// kernel (rowfuse.py via jit.py); reaching this entry means the kernel was
// never installed, which must fail loudly rather than compute nothing.
__global__ void gfb_row_unspecialised(const __grid_constant__ gfb_row_args) { __trap(); }
template __global__ void gfb_ew_staged_kernel<double, 2, 2>(const __grid_constant__ gfb_ew_args);

template __global__ void gfb_ew_kernel<float, 8>(const __grid_constant__ gfb_ew_args);
template __global__ void gfb_ew_kernel<double, 4>(const __grid_constant__ gfb_ew_args);
template __global__ void gfb_ew_kernel<long long, 4>(const __grid_constant__ gfb_ew_args);
template __global__ void gfb_ew_kernel<unsigned char, 8>(const __grid_constant__ gfb_ew_args);
template __global__ void gfb_ew_kernel<float, 1>(const __grid_constant__ gfb_ew_args);
template __global__ void gfb_ew_kernel<double, 1>(const __grid_constant__ gfb_ew_args);

}  // namespace gfb

extern "C" const void* gfb_ew_kernel_ptr(int kind) {
    switch (kind) {
        case GFB_K_EW_F32: return (const void*)gfb::gfb_ew_kernel<float, 8>;
        case GFB_K_EW_F64: return (const void*)gfb::gfb_ew_kernel<double, 4>;
        case GFB_K_EW_I64: return (const void*)gfb::gfb_ew_kernel<long long, 4>;
        case GFB_K_EW_U8: return (const void*)gfb::gfb_ew_kernel<unsigned char, 8>;
        case GFB_K_ROWJIT: return (const void*)gfb::gfb_row_unspecialised;
        case GFB_K_EWS_F32: return (const void*)gfb::gfb_ew_staged_kernel<float, 2, 2>;
        case GFB_K_EWS_F64: return (const void*)gfb::gfb_ew_staged_kernel<double, 2, 2>;
        case GFB_K_EW1_F32: return (const void*)gfb::gfb_ew_kernel<float, 1>;
        case GFB_K_EW1_F64: return (const void*)gfb::gfb_ew_kernel<double, 1>;
    }
    return nullptr;
}
