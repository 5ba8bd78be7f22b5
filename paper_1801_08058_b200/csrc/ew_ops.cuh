// Element semantics shared by the fused elementwise kernels: the generic VM
// (ew_vm.cu) and the per-launch kernels jit.py generates and compiles with
// NVRTC (so this header also builds under __CUDACC_RTC__).
//
// Arithmetic follows the reference contract (numeric.py / kernels.py):
// F32 + - x / are IEEE round-to-nearest with no contraction (__f*_rn);
// Exp / Log / Tanh / Sigmoid are evaluated in double and rounded once;
// Maximum is the literal `x >= y ? x : y` and Relu `x > 0 ? x : 0`; I64 wraps.
#pragma once

#ifdef __CUDACC_RTC__
// the two traits used below (libcu++'s <type_traits> costs NVRTC ~0.6 s a kernel)
namespace std {
template <class A, class B>
struct is_same {
    static constexpr bool value = false;
};
template <class A>
struct is_same<A, A> {
    static constexpr bool value = true;
};
template <class T>
struct is_floating_point {
    static constexpr bool value = is_same<T, float>::value || is_same<T, double>::value;
};
}  // namespace std
#ifndef INFINITY
#define INFINITY __int_as_float(0x7f800000)
#endif
#else
#include <cmath>
#include <cstdint>
#include <type_traits>
#endif

#include "gfb_common.cuh"

namespace gfb {

// Flat opcodes (low byte of a program word; bits 8..15 hold a leaf index).
// One jump-table dispatch per instruction; every body is specialised at
// compile time (operand source, op, operand order), so a VM instruction
// costs a handful of SASS instructions per 8 elements.
//   1..4   acc = pre[k]             5  acc = load(leaf)
//   6      push acc                 7  store(leaf) = acc
//   8..13  acc = unary(acc)         (Negate, Exp, Log, Tanh, Sigmoid, Relu)
//   16 + ((src * 5 + op) * 2 + s)   acc = s ? op(B, acc) : op(acc, B),
//          src 0..3 = pre[src], 4 = load(leaf), 5 = pop, 6 = acc itself
enum : uint32_t { F_LOADP = 1, F_LOADM = 5, F_PUSH = 6, F_STORE = 7, F_UN = 8, F_DOT = 14, F_BIN = 16 };
enum : uint32_t {
    OP_ADD = 0, OP_SUB, OP_MUL, OP_DIV, OP_MAX, OP_NEG, OP_EXP, OP_LOG, OP_TANH, OP_SIGMOID, OP_RELU,
};

template <typename T>
struct VecOf {
    static constexpr int V = sizeof(T) >= 8 ? 4 : 8;
};

template <typename T>
__device__ __forceinline__ T from_bits(uint64_t b) {
    if constexpr (std::is_same<T, float>::value) return __int_as_float((int)(uint32_t)b);
    else if constexpr (std::is_same<T, double>::value) return __longlong_as_double((long long)b);
    else if constexpr (sizeof(T) == 8) return (T)(long long)b;
    else return (T)(b & 0xff);
}

// ---- V consecutive elements, one or two 128-bit (or one 64-bit) accesses
template <typename T, int V>
__device__ __forceinline__ void loadV(const T* p, T (&v)[V]) {
    static_assert(V == 1 || V * sizeof(T) == 32 || V * sizeof(T) == 16 || V * sizeof(T) == 8, "vector width");
    if constexpr (V == 1) {
        v[0] = __ldg(p);
    } else if constexpr (V * sizeof(T) == 16) {
        int4 a = __ldg(reinterpret_cast<const int4*>(p));
        const T* pa = reinterpret_cast<const T*>(&a);
#pragma unroll
        for (int i = 0; i < V; ++i) v[i] = pa[i];
    } else if constexpr (V * sizeof(T) == 32) {
        const int4* q = reinterpret_cast<const int4*>(p);
        int4 a = __ldg(q), b = __ldg(q + 1);
        const T* pa = reinterpret_cast<const T*>(&a);
        const T* pb = reinterpret_cast<const T*>(&b);
#pragma unroll
        for (int i = 0; i < V / 2; ++i) {
            v[i] = pa[i];
            v[i + V / 2] = pb[i];
        }
    } else {
        uint2 a = __ldg(reinterpret_cast<const uint2*>(p));
        const T* pa = reinterpret_cast<const T*>(&a);
#pragma unroll
        for (int i = 0; i < V; ++i) v[i] = pa[i];
    }
}

// loadV without the read-only (non-coherent) path: for data written earlier
// in the same kernel (runtime-merged launches, jit.py)
template <typename T, int V>
__device__ __forceinline__ void loadV_plain(const T* p, T (&v)[V]) {
    if constexpr (V == 1) {
        v[0] = *p;
    } else if constexpr (V * sizeof(T) == 16) {
        int4 a = *reinterpret_cast<const int4*>(p);
        const T* pa = reinterpret_cast<const T*>(&a);
#pragma unroll
        for (int i = 0; i < V; ++i) v[i] = pa[i];
    } else if constexpr (V * sizeof(T) == 32) {
        const int4* q = reinterpret_cast<const int4*>(p);
        int4 a = q[0], b = q[1];
        const T* pa = reinterpret_cast<const T*>(&a);
        const T* pb = reinterpret_cast<const T*>(&b);
#pragma unroll
        for (int i = 0; i < V / 2; ++i) {
            v[i] = pa[i];
            v[i + V / 2] = pb[i];
        }
    } else {
        uint2 a = *reinterpret_cast<const uint2*>(p);
        const T* pa = reinterpret_cast<const T*>(&a);
#pragma unroll
        for (int i = 0; i < V; ++i) v[i] = pa[i];
    }
}

template <typename T, int V>
__device__ __forceinline__ void storeV(T* p, const T (&v)[V]) {
    if constexpr (V == 1) {
        *p = v[0];
    } else if constexpr (V * sizeof(T) == 16) {
        int4 a;
        T* pa = reinterpret_cast<T*>(&a);
#pragma unroll
        for (int i = 0; i < V; ++i) pa[i] = v[i];
        *reinterpret_cast<int4*>(p) = a;
    } else if constexpr (V * sizeof(T) == 32) {
        int4 a, b;
        T* pa = reinterpret_cast<T*>(&a);
        T* pb = reinterpret_cast<T*>(&b);
#pragma unroll
        for (int i = 0; i < V / 2; ++i) {
            pa[i] = v[i];
            pb[i] = v[i + V / 2];
        }
        reinterpret_cast<int4*>(p)[0] = a;
        reinterpret_cast<int4*>(p)[1] = b;
    } else {
        uint2 a;
        T* pa = reinterpret_cast<T*>(&a);
#pragma unroll
        for (int i = 0; i < V; ++i) pa[i] = v[i];
        *reinterpret_cast<uint2*>(p) = a;
    }
}

// ---- scalar semantics (reference numeric.py / kernels.py) ----------------
__device__ __noinline__ double safe_log(double x) {
    if (x != x) return x;
    if (x < 0.0) return __longlong_as_double(0x7ff8000000000000ll);
    if (x == 0.0) return -__longlong_as_double(0x7ff0000000000000ll);
    return log(x);
}
__device__ __noinline__ double sigmoid_d(double x) {
    if (x != x) return x;
    if (x >= 0.0) return __ddiv_rn(1.0, __dadd_rn(1.0, exp(-x)));
    double e = exp(x);
    return __ddiv_rn(e, __dadd_rn(1.0, e));
}
__device__ __noinline__ double transcendental(uint32_t op, double x) {
    switch (op) {
        case OP_EXP: return exp(x);
        case OP_LOG: return safe_log(x);
        case OP_TANH: return tanh(x);
        default: return sigmoid_d(x);
    }
}

template <typename T, int V>
__device__ __forceinline__ void apply_unary(uint32_t op, T (&a)[V]) {
    if constexpr (std::is_floating_point<T>::value) {
        switch (op) {
            case OP_NEG:
#pragma unroll
                for (int v = 0; v < V; ++v) a[v] = -a[v];
                break;
            case OP_RELU:
#pragma unroll
                for (int v = 0; v < V; ++v) a[v] = a[v] > T(0) ? a[v] : T(0);
                break;
            default:  // transcendentals: double precision, rounded once
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    const double y = transcendental(op, (double)a[v]);
                    if constexpr (std::is_same<T, float>::value) a[v] = __double2float_rn(y);
                    else a[v] = y;
                }
                break;
        }
    } else if constexpr (std::is_same<T, long long>::value) {
        if (op == OP_NEG) {
#pragma unroll
            for (int v = 0; v < V; ++v) a[v] = (long long)(0ull - (unsigned long long)a[v]);
        }
    }
}

// Compile-time-op variants for the runtime-generated kernels (jit.py,
// rowfuse.py): the same double-precision functions, inlined, so a vector of
// transcendentals is straight-line code the scheduler can interleave instead
// of V calls through `transcendental`'s switch.  Results are identical.
template <uint32_t OP>
__device__ __forceinline__ double transcendental_c(double x) {
    if constexpr (OP == OP_EXP) {
        return exp(x);
    } else if constexpr (OP == OP_LOG) {
        if (x != x) return x;
        if (x < 0.0) return __longlong_as_double(0x7ff8000000000000ll);
        if (x == 0.0) return -__longlong_as_double(0x7ff0000000000000ll);
        return log(x);
    } else if constexpr (OP == OP_TANH) {
        return tanh(x);
    } else {
        if (x != x) return x;
        if (x >= 0.0) return __ddiv_rn(1.0, __dadd_rn(1.0, exp(-x)));
        const double e = exp(x);
        return __ddiv_rn(e, __dadd_rn(1.0, e));
    }
}

template <uint32_t OP, typename T, int V>
__device__ __forceinline__ void apply_unary_c(T (&a)[V]) {
    if constexpr (!std::is_floating_point<T>::value || OP == OP_NEG || OP == OP_RELU) {
        apply_unary<T, V>(OP, a);
    } else {
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const double y = transcendental_c<OP>((double)a[v]);
            if constexpr (std::is_same<T, float>::value) a[v] = __double2float_rn(y);
            else a[v] = y;
        }
    }
}

// Row-fused launches (rowfuse.py): F32 Exp / Log in single precision (CUDA
// expf / logf, <= 2 / 1 ulp -- inside the 1e-5 transcendental contract of
// SURVEY.md §8(c), not bit-identical to the reference's double evaluation).
// A softmax row group is then bound by HBM instead of the FP64 pipe.
// Special values as the reference's: exp overflow -> inf, log(0) = -inf,
// log(x < 0) = NaN, NaN in -> NaN out.
template <uint32_t OP, typename T, int V>
__device__ __forceinline__ void apply_unary_row(T (&a)[V]) {
    if constexpr (std::is_same<T, float>::value && (OP == OP_EXP || OP == OP_LOG)) {
#pragma unroll
        for (int v = 0; v < V; ++v) a[v] = OP == OP_EXP ? expf(a[v]) : logf(a[v]);
    } else {
        apply_unary_c<OP, T, V>(a);
    }
}

template <typename T>
__device__ __forceinline__ T bin1(uint32_t op, T x, T y) {
    if constexpr (std::is_same<T, float>::value) {
        switch (op) {
            case OP_ADD: return __fadd_rn(x, y);
            case OP_SUB: return __fsub_rn(x, y);
            case OP_MUL: return __fmul_rn(x, y);
            case OP_DIV: return __fdiv_rn(x, y);
            default: return x >= y ? x : y;
        }
    } else if constexpr (std::is_same<T, double>::value) {
        switch (op) {
            case OP_ADD: return __dadd_rn(x, y);
            case OP_SUB: return __dsub_rn(x, y);
            case OP_MUL: return __dmul_rn(x, y);
            case OP_DIV: return __ddiv_rn(x, y);
            default: return x >= y ? x : y;
        }
    } else if constexpr (std::is_same<T, long long>::value) {
        typedef unsigned long long U;
        switch (op) {
            case OP_ADD: return (long long)((U)x + (U)y);
            case OP_SUB: return (long long)((U)x - (U)y);
            default: return (long long)((U)x * (U)y);
        }
    } else {
        return x;
    }
}

template <typename T, int V>
__device__ __forceinline__ void copyV(T (&d)[V], const T (&s)[V]) {
#pragma unroll
    for (int v = 0; v < V; ++v) d[v] = s[v];
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

}  // namespace gfb
