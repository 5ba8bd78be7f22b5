// Fused elementwise / Broadcast / Reshape / ConvertLayout / Sum kernels.
//
// The compile pass (paper_1801_08058_b200/compiler.py) turns each fusion
// group of memory-bound IR nodes into one *program* for this kernel: a short
// accumulator-stack bytecode over "leaves" (loads / stores through
// mixed-radix index maps, gfb200.h gfb_digit).  One launch evaluates the
// whole group in a single pass over HBM:
//   mode 0  map            out[o]            = prog(o)
//   mode 1  row reduce     red[o] = fold_r   prog(o, r)   one warp per o, lanes along r
//   mode 2  column reduce  red[o] = fold_r   prog(o, r)   lanes along o, r split `split` ways
// Side outputs (STORE) write intermediate values the graph also needs, so
// e.g. config B's `t3 = Relu(a + Broadcast(c)) * b` and `Sum(t3)` are one read
// of a and b and one write of t3.
//
// Arithmetic follows the reference contract (numeric.py / kernels.py):
// F32 + - x / are IEEE round-to-nearest with no contraction (__f*_rn), so
// they are bit-exact with the reference's double-then-round; Exp / Log / Tanh
// / Sigmoid are evaluated in double and rounded once to F32 like
// `round_f32(math.exp(x))`; Maximum is the literal `x >= y ? x : y` and Relu
// `x > 0 ? x : 0`; I64 wraps.  No --use_fast_math, no FTZ (sigmoid(-100)
// in F32 is a subnormal).
//
// Each thread evaluates a vector of 4 consecutive indices along the
// launch's vector axis; leaves classified contiguous/uniform at compile
// time use 128-bit loads/stores, and the first `npre` leaves are all loaded
// before the program runs so their HBM requests are in flight together.

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "gfb_common.cuh"

namespace gfb {

enum : uint32_t {
    I_LOAD = 1,
    I_UN = 2,
    I_BIN_LEAF = 3,
    I_BIN_POP = 4,
    I_BIN_SELF = 5,
    I_PUSH = 6,
    I_STORE = 7,
    I_PUSH_LOAD = 8,
};
enum : uint32_t {
    OP_ADD = 0, OP_SUB, OP_MUL, OP_DIV, OP_MAX, OP_NEG, OP_EXP, OP_LOG, OP_TANH, OP_SIGMOID, OP_RELU,
};

template <typename T>
__device__ __forceinline__ T from_bits(uint64_t b) {
    if constexpr (sizeof(T) == 4) return __int_as_float((int)(uint32_t)b);
    else if constexpr (sizeof(T) == 8 && std::is_same<T, double>::value) return __longlong_as_double((long long)b);
    else if constexpr (sizeof(T) == 8) return (T)(long long)b;
    else return (T)(b & 0xff);
}

// ---- vector memory access (4 consecutive elements, 16B-aligned for 4/8-byte T)
template <typename T>
__device__ __forceinline__ void load4(const T* p, T (&v)[4]) {
    if constexpr (sizeof(T) == 4) {
        float4 x = __ldg(reinterpret_cast<const float4*>(p));
        v[0] = *reinterpret_cast<T*>(&x.x);
        v[1] = *reinterpret_cast<T*>(&x.y);
        v[2] = *reinterpret_cast<T*>(&x.z);
        v[3] = *reinterpret_cast<T*>(&x.w);
    } else if constexpr (sizeof(T) == 8) {
        const longlong2* q = reinterpret_cast<const longlong2*>(p);
        longlong2 a = __ldg(q), b = __ldg(q + 1);
        v[0] = *reinterpret_cast<T*>(&a.x);
        v[1] = *reinterpret_cast<T*>(&a.y);
        v[2] = *reinterpret_cast<T*>(&b.x);
        v[3] = *reinterpret_cast<T*>(&b.y);
    } else {
        uchar4 x = __ldg(reinterpret_cast<const uchar4*>(p));
        v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
    }
}

template <typename T>
__device__ __forceinline__ void store4(T* p, const T (&v)[4]) {
    if constexpr (sizeof(T) == 4) {
        float4 x;
        x.x = *reinterpret_cast<const float*>(&v[0]);
        x.y = *reinterpret_cast<const float*>(&v[1]);
        x.z = *reinterpret_cast<const float*>(&v[2]);
        x.w = *reinterpret_cast<const float*>(&v[3]);
        *reinterpret_cast<float4*>(p) = x;
    } else if constexpr (sizeof(T) == 8) {
        longlong2 a, b;
        a.x = *reinterpret_cast<const long long*>(&v[0]);
        a.y = *reinterpret_cast<const long long*>(&v[1]);
        b.x = *reinterpret_cast<const long long*>(&v[2]);
        b.y = *reinterpret_cast<const long long*>(&v[3]);
        reinterpret_cast<longlong2*>(p)[0] = a;
        reinterpret_cast<longlong2*>(p)[1] = b;
    } else {
        *reinterpret_cast<uchar4*>(p) = make_uchar4(v[0], v[1], v[2], v[3]);
    }
}

template <typename T>
__device__ __forceinline__ void load_leaf(const gfb_leaf& L, const void* const* tab, uint32_t o, uint32_t r,
                                          int vaxis, int nvalid, T (&out)[4]) {
    if (L.mode == 1) {
        const T s = from_bits<T>(L.splat);
#pragma unroll
        for (int v = 0; v < 4; ++v) out[v] = s;
        return;
    }
    const T* base = resolve<const T>(tab, L.ref);
    if (nvalid == 4 && L.vec == 1) {
        load4(base + leaf_offset(L, o, r), out);
    } else if (nvalid == 4 && L.vec == 2) {
        const T s = __ldg(base + leaf_offset(L, o, r));
#pragma unroll
        for (int v = 0; v < 4; ++v) out[v] = s;
    } else {
#pragma unroll
        for (int v = 0; v < 4; ++v)
            out[v] = v < nvalid ? __ldg(base + leaf_offset(L, o + (vaxis ? 0 : v), r + (vaxis ? v : 0))) : T(0);
    }
}

template <typename T>
__device__ __forceinline__ void store_leaf(const gfb_leaf& L, const void* const* tab, uint32_t o, uint32_t r,
                                           int vaxis, int nvalid, const T (&val)[4]) {
    T* base = resolve<T>(tab, L.ref);
    if (nvalid == 4 && L.vec == 1) {
        store4(base + leaf_offset(L, o, r), val);
    } else {
#pragma unroll
        for (int v = 0; v < 4; ++v)
            if (v < nvalid) base[leaf_offset(L, o + (vaxis ? 0 : v), r + (vaxis ? v : 0))] = val[v];
    }
}

// ---- scalar semantics (reference numeric.py / kernels.py) ----------------
__device__ __forceinline__ double safe_log(double x) {
    if (x != x) return x;
    if (x < 0.0) return __longlong_as_double(0x7ff8000000000000ll);
    if (x == 0.0) return -__longlong_as_double(0x7ff0000000000000ll);
    return log(x);
}
__device__ __forceinline__ double sigmoid_d(double x) {
    if (x != x) return x;
    if (x >= 0.0) return __ddiv_rn(1.0, __dadd_rn(1.0, exp(-x)));
    double e = exp(x);
    return __ddiv_rn(e, __dadd_rn(1.0, e));
}

template <typename T>
__device__ __forceinline__ void apply_unary(uint32_t op, T (&a)[4]) {
    if constexpr (std::is_same<T, float>::value) {
        switch (op) {
            case OP_NEG:
#pragma unroll
                for (int v = 0; v < 4; ++v) a[v] = -a[v];
                break;
            case OP_EXP:
#pragma unroll
                for (int v = 0; v < 4; ++v) a[v] = __double2float_rn(exp((double)a[v]));
                break;
            case OP_LOG:
#pragma unroll
                for (int v = 0; v < 4; ++v) a[v] = __double2float_rn(safe_log((double)a[v]));
                break;
            case OP_TANH:
#pragma unroll
                for (int v = 0; v < 4; ++v) a[v] = __double2float_rn(tanh((double)a[v]));
                break;
            case OP_SIGMOID:
#pragma unroll
                for (int v = 0; v < 4; ++v) a[v] = __double2float_rn(sigmoid_d((double)a[v]));
                break;
            case OP_RELU:
#pragma unroll
                for (int v = 0; v < 4; ++v) a[v] = a[v] > 0.0f ? a[v] : 0.0f;
                break;
        }
    } else if constexpr (std::is_same<T, double>::value) {
        switch (op) {
            case OP_NEG:
#pragma unroll
                for (int v = 0; v < 4; ++v) a[v] = -a[v];
                break;
            case OP_EXP:
#pragma unroll
                for (int v = 0; v < 4; ++v) a[v] = exp(a[v]);
                break;
            case OP_LOG:
#pragma unroll
                for (int v = 0; v < 4; ++v) a[v] = safe_log(a[v]);
                break;
            case OP_TANH:
#pragma unroll
                for (int v = 0; v < 4; ++v) a[v] = tanh(a[v]);
                break;
            case OP_SIGMOID:
#pragma unroll
                for (int v = 0; v < 4; ++v) a[v] = sigmoid_d(a[v]);
                break;
            case OP_RELU:
#pragma unroll
                for (int v = 0; v < 4; ++v) a[v] = a[v] > 0.0 ? a[v] : 0.0;
                break;
        }
    } else if constexpr (std::is_same<T, long long>::value) {
        if (op == OP_NEG) {
#pragma unroll
            for (int v = 0; v < 4; ++v) a[v] = (long long)(0ull - (unsigned long long)a[v]);
        }
    }
}

// out = op(x, y) elementwise
template <typename T>
__device__ __forceinline__ void apply_binary(uint32_t op, const T (&x)[4], const T (&y)[4], T (&out)[4]) {
    if constexpr (std::is_same<T, float>::value) {
        switch (op) {
            case OP_ADD:
#pragma unroll
                for (int v = 0; v < 4; ++v) out[v] = __fadd_rn(x[v], y[v]);
                break;
            case OP_SUB:
#pragma unroll
                for (int v = 0; v < 4; ++v) out[v] = __fsub_rn(x[v], y[v]);
                break;
            case OP_MUL:
#pragma unroll
                for (int v = 0; v < 4; ++v) out[v] = __fmul_rn(x[v], y[v]);
                break;
            case OP_DIV:
#pragma unroll
                for (int v = 0; v < 4; ++v) out[v] = __fdiv_rn(x[v], y[v]);
                break;
            case OP_MAX:
#pragma unroll
                for (int v = 0; v < 4; ++v) out[v] = x[v] >= y[v] ? x[v] : y[v];
                break;
        }
    } else if constexpr (std::is_same<T, double>::value) {
        switch (op) {
            case OP_ADD:
#pragma unroll
                for (int v = 0; v < 4; ++v) out[v] = __dadd_rn(x[v], y[v]);
                break;
            case OP_SUB:
#pragma unroll
                for (int v = 0; v < 4; ++v) out[v] = __dsub_rn(x[v], y[v]);
                break;
            case OP_MUL:
#pragma unroll
                for (int v = 0; v < 4; ++v) out[v] = __dmul_rn(x[v], y[v]);
                break;
            case OP_DIV:
#pragma unroll
                for (int v = 0; v < 4; ++v) out[v] = __ddiv_rn(x[v], y[v]);
                break;
            case OP_MAX:
#pragma unroll
                for (int v = 0; v < 4; ++v) out[v] = x[v] >= y[v] ? x[v] : y[v];
                break;
        }
    } else if constexpr (std::is_same<T, long long>::value) {
        typedef unsigned long long U;
        switch (op) {
            case OP_ADD:
#pragma unroll
                for (int v = 0; v < 4; ++v) out[v] = (long long)((U)x[v] + (U)y[v]);
                break;
            case OP_SUB:
#pragma unroll
                for (int v = 0; v < 4; ++v) out[v] = (long long)((U)x[v] - (U)y[v]);
                break;
            case OP_MUL:
#pragma unroll
                for (int v = 0; v < 4; ++v) out[v] = (long long)((U)x[v] * (U)y[v]);
                break;
        }
    }
}

template <typename T>
__device__ __forceinline__ void copy4(T (&d)[4], const T (&s)[4]) {
#pragma unroll
    for (int v = 0; v < 4; ++v) d[v] = s[v];
}

// Run the program at the vector group starting at (o, r).  The value left
// in `acc` is what a reduce launch folds.
template <typename T>
__device__ __forceinline__ void vm_run(const gfb_ew_args& p, uint32_t o, uint32_t r, int nvalid, T (&acc)[4]) {
    const void* const* tab = p.tab;
    const int vaxis = p.vec_axis;
    const int npre = p.npre;
    T pre0[4], pre1[4], pre2[4], pre3[4];
    if (npre > 0) load_leaf(p.leaves[0], tab, o, r, vaxis, nvalid, pre0);
    if (npre > 1) load_leaf(p.leaves[1], tab, o, r, vaxis, nvalid, pre1);
    if (npre > 2) load_leaf(p.leaves[2], tab, o, r, vaxis, nvalid, pre2);
    if (npre > 3) load_leaf(p.leaves[3], tab, o, r, vaxis, nvalid, pre3);

    auto fetch = [&](uint32_t k, T(&b)[4]) {
        if ((int)k < npre) {
            switch (k) {
                case 0: copy4(b, pre0); break;
                case 1: copy4(b, pre1); break;
                case 2: copy4(b, pre2); break;
                default: copy4(b, pre3); break;
            }
        } else {
            load_leaf(p.leaves[k], tab, o, r, vaxis, nvalid, b);
        }
    };

    T s0[4], s1[4], s2[4];
    const uint32_t n = p.ninstr;
#pragma unroll 1
    for (uint32_t pc = 0; pc < n; ++pc) {
        const uint32_t ins = p.prog[pc];
        const uint32_t cls = ins & 0xffu, op = (ins >> 8) & 0xffu, k = (ins >> 16) & 0xffu, swap = ins >> 24;
        switch (cls) {
            case I_PUSH_LOAD:
                copy4(s2, s1); copy4(s1, s0); copy4(s0, acc);
                fetch(k, acc);
                break;
            case I_LOAD:
                fetch(k, acc);
                break;
            case I_PUSH:
                copy4(s2, s1); copy4(s1, s0); copy4(s0, acc);
                break;
            case I_UN:
                apply_unary<T>(op, acc);
                break;
            case I_BIN_LEAF: {
                T b[4];
                fetch(k, b);
                if (swap) apply_binary<T>(op, b, acc, acc);
                else apply_binary<T>(op, acc, b, acc);
                break;
            }
            case I_BIN_POP: {
                T b[4];
                copy4(b, s0); copy4(s0, s1); copy4(s1, s2);
                if (swap) apply_binary<T>(op, acc, b, acc);
                else apply_binary<T>(op, b, acc, acc);
                break;
            }
            case I_BIN_SELF:
                apply_binary<T>(op, acc, acc, acc);
                break;
            case I_STORE:
                store_leaf(p.leaves[k], tab, o, r, vaxis, nvalid, acc);
                break;
        }
    }
}

template <typename T>
__device__ __forceinline__ T fold(int kind, T acc, T v) {
    if constexpr (std::is_same<T, float>::value) return kind == 2 ? (acc >= v ? acc : v) : __fadd_rn(acc, v);
    else if constexpr (std::is_same<T, double>::value) return kind == 2 ? (acc >= v ? acc : v) : __dadd_rn(acc, v);
    else return (T)((unsigned long long)acc + (unsigned long long)v);
}

template <typename T>
__device__ __forceinline__ T fold_init(int kind) {
    if constexpr (std::is_same<T, float>::value) return kind == 2 ? -INFINITY : 0.0f;
    else if constexpr (std::is_same<T, double>::value) return kind == 2 ? -(double)INFINITY : 0.0;
    else return T(0);
}

template <typename T>
__global__ void __launch_bounds__(256) gfb_ew_kernel(const __grid_constant__ gfb_ew_args p) {
    const int mode = p.mode;
    if (mode == 0) {
        const uint32_t n = p.n_o;
        const uint32_t groups = (n + 3) >> 2;
        for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < groups; g += gridDim.x * blockDim.x) {
            const uint32_t o = g << 2;
            const int nvalid = min(4u, n - o);
            T acc[4];
            vm_run<T>(p, o, 0, nvalid, acc);
        }
        return;
    }
    if constexpr (sizeof(T) == 1) {
        return;  // BOOL has no reductions (reference ir.py:178-180)
    } else {
        const int kind = p.red_kind;
        const void* const* tab = p.tab;
        if (mode == 1) {
            // One warp per output row, lanes stride along r in vectors of 4.
            const int lane = threadIdx.x & 31;
            const uint32_t warps = blockDim.x >> 5;
            const uint32_t nr = p.n_r;
            for (uint32_t o = blockIdx.x * warps + (threadIdx.x >> 5); o < p.n_o; o += gridDim.x * warps) {
                T part = fold_init<T>(kind);
                for (uint32_t r = lane * 4; r < nr; r += 128) {
                    const int nvalid = min(4u, nr - r);
                    T acc[4];
                    vm_run<T>(p, o, r, nvalid, acc);
#pragma unroll
                    for (int v = 0; v < 4; ++v)
                        if (v < nvalid) part = fold<T>(kind, part, acc[v]);
                }
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) part = fold<T>(kind, part, __shfl_xor_sync(0xffffffffu, part, off));
                if (lane == 0) resolve<T>(tab, p.red_out.ref)[leaf_offset(p.red_out, o, 0)] = part;
            }
            return;
        }
        // mode 2: lanes along o (vectors of 4 outputs), r split `split` ways.
        extern __shared__ unsigned char smem_raw[];
        T* smem = reinterpret_cast<T*>(smem_raw);
        const uint32_t split = p.split;
        const uint32_t per_row = blockDim.x / split;
        const uint32_t lane_o = threadIdx.x % per_row, rs = threadIdx.x / per_row;
        const uint32_t o = (blockIdx.x * per_row + lane_o) * 4;
        const bool active = o < p.n_o;
        const int nvalid = active ? (int)min(4u, p.n_o - o) : 0;
        T part[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) part[v] = fold_init<T>(kind);
        if (active) {
            for (uint32_t r = rs; r < p.n_r; r += split) {
                T acc[4];
                vm_run<T>(p, o, r, nvalid, acc);
#pragma unroll
                for (int v = 0; v < 4; ++v) part[v] = fold<T>(kind, part[v], acc[v]);
            }
        }
        if (split > 1) {
#pragma unroll
            for (int v = 0; v < 4; ++v) smem[(rs * per_row + lane_o) * 4 + v] = part[v];
            __syncthreads();
            if (rs != 0) return;
            for (uint32_t s = 1; s < split; ++s)
#pragma unroll
                for (int v = 0; v < 4; ++v) part[v] = fold<T>(kind, part[v], smem[(s * per_row + lane_o) * 4 + v]);
        }
        if (active) store_leaf(p.red_out, tab, o, 0, 0, nvalid, part);
    }
}

template __global__ void gfb_ew_kernel<float>(const __grid_constant__ gfb_ew_args);
template __global__ void gfb_ew_kernel<double>(const __grid_constant__ gfb_ew_args);
template __global__ void gfb_ew_kernel<long long>(const __grid_constant__ gfb_ew_args);
template __global__ void gfb_ew_kernel<unsigned char>(const __grid_constant__ gfb_ew_args);

}  // namespace gfb

extern "C" const void* gfb_ew_kernel_ptr(int kind) {
    switch (kind) {
        case GFB_K_EW_F32: return (const void*)gfb::gfb_ew_kernel<float>;
        case GFB_K_EW_F64: return (const void*)gfb::gfb_ew_kernel<double>;
        case GFB_K_EW_I64: return (const void*)gfb::gfb_ew_kernel<long long>;
        case GFB_K_EW_U8: return (const void*)gfb::gfb_ew_kernel<unsigned char>;
    }
    return nullptr;
}
