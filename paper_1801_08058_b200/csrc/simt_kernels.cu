// Exact-order SIMT kernels for Dot and the convolution family.
//
// These keep the reference's accumulation order per output element —
// Dot: k ascending (kernels.py:123-133); Conv2D: c, r, s (kernels.py:180-206);
// ConvBackpropData: k, r, s (kernels.py:209-235); ConvBackpropFilter: n, p, q
// (kernels.py:238-264) — with one IEEE round-to-nearest per multiply and per
// add (no FMA), so F32/F64 results are bit-identical to the reference.  They
// serve F64 graphs, small F32 contractions (launch-latency bound anyway) and
// any shape the tcgen05 path does not take; large F32 Dots run on the tensor
// cores (gemm_tc.cu) under the normwise tolerance of SURVEY.md §8(c).
//
// All operands are addressed through per-axis element strides, so the
// transposing Reshapes autodiff emits for Dot (autodiff.py:163-177) and the
// NCHW/NHWC layouts chosen by layout assignment are consumed in place.

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "gfb_common.cuh"

namespace gfb {

__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }

// 64x64 output tile per 256-thread block, 4x4 per thread, K staged 16 at a time.
template <typename T>
__global__ void __launch_bounds__(256) gfb_dot_kernel(const __grid_constant__ gfb_dot_args p) {
    constexpr int BM = 64, BN = 64, BK = 16;
    __shared__ T As[BK][BM + 1];
    __shared__ T Bs[BK][BN + 1];
    const T* A = resolve<const T>(p.tab, p.a);
    const T* B = resolve<const T>(p.tab, p.b);
    T* C = resolve<T>(p.tab, p.c);
    const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    // Coalesce the tile loads along whichever axis is contiguous in memory.
    const bool a_k_fast = p.a_sk <= p.a_sm;
    const bool b_n_fast = p.b_sn <= p.b_sk;
    T acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = T(0);

    for (int64_t k0 = 0; k0 < p.k; k0 += BK) {
        const int kn = (int)min((int64_t)BK, p.k - k0);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int idx = tid + 256 * e;
            int mm, kk;
            if (a_k_fast) { mm = idx / BK; kk = idx % BK; } else { mm = idx % BM; kk = idx / BM; }
            const int64_t gm = m0 + mm, gk = k0 + kk;
            As[kk][mm] = (gm < p.m && kk < kn) ? A[gm * p.a_sm + gk * p.a_sk] : T(0);
            int nn, kb;
            if (b_n_fast) { nn = idx % BN; kb = idx / BN; } else { nn = idx / BK; kb = idx % BK; }
            const int64_t gn = n0 + nn, gkb = k0 + kb;
            Bs[kb][nn] = (gn < p.n && kb < kn) ? B[gkb * p.b_sk + gn * p.b_sn] : T(0);
        }
        __syncthreads();
        for (int kk = 0; kk < kn; ++kk) {
            T a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = add_rn(acc[i][j], mul_rn(a[i], b[j]));
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t gm = m0 + ty + 16 * i;
        if (gm >= p.m) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t gn = n0 + tx + 16 * j;
            if (gn < p.n) C[gm * p.c_sm + gn * p.c_sn] = acc[i][j];
        }
    }
}

// Dot with few rows (m <= 8): one thread per output column computes all m
// outputs, k ascending — the reference order, bit-exact.  This is the shape
// of the maxpool composite's one-hot selections ([1,4] x [4, N*C*H*W]) and
// their gradients ([4,1] x [1, M]), where a 64x64 tile would idle 63 of 64
// threads.  B is read once, coalesced along n.
template <typename T>
__global__ void __launch_bounds__(256) gfb_dot_small_m_kernel(const __grid_constant__ gfb_dot_args p) {
    const T* A = resolve<const T>(p.tab, p.a);
    const T* B = resolve<const T>(p.tab, p.b);
    T* C = resolve<T>(p.tab, p.c);
    const int m = (int)p.m;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < p.n; j += (int64_t)gridDim.x * blockDim.x) {
        T acc[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = T(0);
        for (int64_t t = 0; t < p.k; ++t) {
            const T b = B[t * p.b_sk + j * p.b_sn];
#pragma unroll
            for (int i = 0; i < 8; ++i)
                if (i < m) acc[i] = add_rn(acc[i], mul_rn(__ldg(A + i * p.a_sm + t * p.a_sk), b));
        }
#pragma unroll
        for (int i = 0; i < 8; ++i)
            if (i < m) C[i * p.c_sm + j * p.c_sn] = acc[i];
    }
}

// Dot with few outputs (a narrow classifier layer, its gradients): one
// thread per output element, k ascending — the reference order, bit-exact.
// Consecutive threads take consecutive columns, so B loads coalesce and A
// loads broadcast; the add chain runs in registers (no tile barriers).
template <typename T>
__global__ void __launch_bounds__(256) gfb_dot_thread_kernel(const __grid_constant__ gfb_dot_args p) {
    const T* A = resolve<const T>(p.tab, p.a);
    const T* B = resolve<const T>(p.tab, p.b);
    T* C = resolve<T>(p.tab, p.c);
    const int64_t total = p.m * p.n;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = idx / p.n, j = idx - i * p.n;
        const T* a = A + i * p.a_sm;
        const T* b = B + j * p.b_sn;
        T acc = T(0);
        // 16 products' operands in flight per step: the add chain is the
        // only serial part (software-pipelined against the loads)
        constexpr int D = 16;
        T av[D], bv[D];
        int64_t t = 0;
        const int64_t kfull = p.k - p.k % D;
        if (kfull > 0) {
#pragma unroll
            for (int u = 0; u < D; ++u) {
                av[u] = __ldg(a + (int64_t)u * p.a_sk);
                bv[u] = __ldg(b + (int64_t)u * p.b_sk);
            }
        }
        for (; t < kfull; t += D) {
            T an[D], bn[D];
            const bool more = t + D < kfull;
#pragma unroll
            for (int u = 0; u < D; ++u) {
                an[u] = more ? __ldg(a + (t + D + u) * p.a_sk) : T(0);
                bn[u] = more ? __ldg(b + (t + D + u) * p.b_sk) : T(0);
            }
#pragma unroll
            for (int u = 0; u < D; ++u) acc = add_rn(acc, mul_rn(av[u], bv[u]));
#pragma unroll
            for (int u = 0; u < D; ++u) {
                av[u] = an[u];
                bv[u] = bn[u];
            }
        }
        for (; t < p.k; ++t) acc = add_rn(acc, mul_rn(__ldg(a + t * p.a_sk), __ldg(b + t * p.b_sk)));
        C[i * p.c_sm + j * p.c_sn] = acc;
    }
}

// One thread per output element, the reference loop nest verbatim.
template <typename T>
__global__ void __launch_bounds__(256) gfb_conv_kernel(const __grid_constant__ gfb_conv_args p) {
    const T* X = resolve<const T>(p.tab, p.x);
    const T* Y = resolve<const T>(p.tab, p.y);
    T* O = resolve<T>(p.tab, p.out);
    int64_t total;
    if (p.op == 0) total = p.N * p.K * p.Ho * p.Wo;
    else if (p.op == 1 || p.op == 4) total = p.N * p.C * p.H * p.W;
    else if (p.op == 3) total = p.N * p.C * p.Ho * p.Wo;
    else total = p.K * p.C * p.R * p.S;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        T acc = T(0);
        if (p.op == 0) {
            // out[n,k,p,q] = sum_{c,r,s} x[n,c,p*sh-pt+r,q*sw-pl+s] * f[k,c,r,s]
            const int64_t q = idx % p.Wo, pp = (idx / p.Wo) % p.Ho, k = (idx / (p.Wo * p.Ho)) % p.K,
                          n = idx / (p.Wo * p.Ho * p.K);
            for (int64_t c = 0; c < p.C; ++c)
                for (int64_t r = 0; r < p.R; ++r) {
                    const int64_t h = pp * p.sh - p.pt + r;
                    if (h < 0 || h >= p.H) continue;
                    for (int64_t s = 0; s < p.S; ++s) {
                        const int64_t w = q * p.sw - p.pl + s;
                        if (w < 0 || w >= p.W) continue;
                        acc = add_rn(acc, mul_rn(X[n * p.xs[0] + c * p.xs[1] + h * p.xs[2] + w * p.xs[3]],
                                                 Y[k * p.ys[0] + c * p.ys[1] + r * p.ys[2] + s * p.ys[3]]));
                    }
                }
            O[n * p.os[0] + k * p.os[1] + pp * p.os[2] + q * p.os[3]] = acc;
        } else if (p.op == 1) {
            // out[n,c,h,w] = sum_{k,r,s} delta[n,k,(h+pt-r)/sh,(w+pl-s)/sw] * f[k,c,r,s]
            // over the taps divisible by the stride (1 for the reference's ops)
            const int64_t w = idx % p.W, h = (idx / p.W) % p.H, c = (idx / (p.W * p.H)) % p.C,
                          n = idx / (p.W * p.H * p.C);
            for (int64_t k = 0; k < p.K; ++k)
                for (int64_t r = 0; r < p.R; ++r) {
                    const int64_t pn = h + p.pt - r;
                    if (pn < 0 || pn % p.sh) continue;
                    const int64_t pp = pn / p.sh;
                    if (pp >= p.Ho) continue;
                    for (int64_t s = 0; s < p.S; ++s) {
                        const int64_t qn = w + p.pl - s;
                        if (qn < 0 || qn % p.sw) continue;
                        const int64_t q = qn / p.sw;
                        if (q >= p.Wo) continue;
                        acc = add_rn(acc, mul_rn(X[n * p.xs[0] + k * p.xs[1] + pp * p.xs[2] + q * p.xs[3]],
                                                 Y[k * p.ys[0] + c * p.ys[1] + r * p.ys[2] + s * p.ys[3]]));
                    }
                }
            O[n * p.os[0] + c * p.os[1] + h * p.os[2] + w * p.os[3]] = acc;
        } else if (p.op == 3) {
            // MaxPool (IR extension): fold acc >= v ? acc : v from -inf over
            // the (R, S) window in row-major order, padding taps skipped
            const int64_t q = idx % p.Wo, pp = (idx / p.Wo) % p.Ho, c = (idx / (p.Wo * p.Ho)) % p.C,
                          n = idx / (p.Wo * p.Ho * p.C);
            acc = -(T)INFINITY;
            for (int64_t i = 0; i < p.R; ++i) {
                const int64_t h = pp * p.sh + i - p.pt;
                if (h < 0 || h >= p.H) continue;
                for (int64_t j = 0; j < p.S; ++j) {
                    const int64_t w = q * p.sw + j - p.pl;
                    if (w < 0 || w >= p.W) continue;
                    const T v = X[n * p.xs[0] + c * p.xs[1] + h * p.xs[2] + w * p.xs[3]];
                    acc = acc >= v ? acc : v;
                }
            }
            O[n * p.os[0] + c * p.os[1] + pp * p.os[2] + q * p.os[3]] = acc;
        } else if (p.op == 4) {
            // MaxPoolBackprop: sum over the windows (p, q) ascending that hold
            // (h, w) and select it (the element where the forward fold last
            // changed) of delta[n, c, p, q]
            const int64_t w = idx % p.W, h = (idx / p.W) % p.H, c = (idx / (p.W * p.H)) % p.C,
                          n = idx / (p.W * p.H * p.C);
            const T* xc = X + n * p.xs[0] + c * p.xs[1];
            for (int64_t pp = 0; pp < p.Ho; ++pp) {
                const int64_t i = h + p.pt - pp * p.sh;
                if (i < 0 || i >= p.R) continue;
                for (int64_t q = 0; q < p.Wo; ++q) {
                    const int64_t j = w + p.pl - q * p.sw;
                    if (j < 0 || j >= p.S) continue;
                    T best = -(T)INFINITY;
                    int64_t arg = -1;
                    for (int64_t a = 0; a < p.R; ++a) {
                        const int64_t hh = pp * p.sh + a - p.pt;
                        if (hh < 0 || hh >= p.H) continue;
                        for (int64_t b = 0; b < p.S; ++b) {
                            const int64_t ww = q * p.sw + b - p.pl;
                            if (ww < 0 || ww >= p.W) continue;
                            const T v = xc[hh * p.xs[2] + ww * p.xs[3]];
                            if (!(best >= v)) {
                                best = v;
                                arg = hh * p.W + ww;
                            }
                        }
                    }
                    if (arg == h * p.W + w) acc = add_rn(acc, Y[n * p.ys[0] + c * p.ys[1] + pp * p.ys[2] + q * p.ys[3]]);
                }
            }
            O[n * p.os[0] + c * p.os[1] + h * p.os[2] + w * p.os[3]] = acc;
        } else {
            // out[k,c,r,s] = sum_{n,p,q} delta[n,k,p,q] * x[n,c,p*sh+r-pt,q*sw+s-pl]
            const int64_t s = idx % p.S, r = (idx / p.S) % p.R, c = (idx / (p.S * p.R)) % p.C,
                          k = idx / (p.S * p.R * p.C);
            for (int64_t n = 0; n < p.N; ++n)
                for (int64_t pp = 0; pp < p.Ho; ++pp) {
                    const int64_t h = pp * p.sh + r - p.pt;
                    if (h < 0 || h >= p.H) continue;
                    for (int64_t q = 0; q < p.Wo; ++q) {
                        const int64_t w = q * p.sw + s - p.pl;
                        if (w < 0 || w >= p.W) continue;
                        acc = add_rn(acc, mul_rn(Y[n * p.ys[0] + k * p.ys[1] + pp * p.ys[2] + q * p.ys[3]],
                                                 X[n * p.xs[0] + c * p.xs[1] + h * p.xs[2] + w * p.xs[3]]));
                    }
                }
            O[k * p.os[0] + c * p.os[1] + r * p.os[2] + s * p.os[3]] = acc;
        }
    }
}

template __global__ void gfb_dot_kernel<float>(const __grid_constant__ gfb_dot_args);
template __global__ void gfb_dot_kernel<double>(const __grid_constant__ gfb_dot_args);
template __global__ void gfb_dot_small_m_kernel<float>(const __grid_constant__ gfb_dot_args);
template __global__ void gfb_dot_small_m_kernel<double>(const __grid_constant__ gfb_dot_args);
template __global__ void gfb_dot_thread_kernel<float>(const __grid_constant__ gfb_dot_args);
template __global__ void gfb_dot_thread_kernel<double>(const __grid_constant__ gfb_dot_args);
template __global__ void gfb_conv_kernel<float>(const __grid_constant__ gfb_conv_args);
template __global__ void gfb_conv_kernel<double>(const __grid_constant__ gfb_conv_args);

}  // namespace gfb

extern "C" const void* gfb_simt_kernel_ptr(int kind) {
    switch (kind) {
        case GFB_K_DOT_F32: return (const void*)gfb::gfb_dot_kernel<float>;
        case GFB_K_DOT_F64: return (const void*)gfb::gfb_dot_kernel<double>;
        case GFB_K_DOT_SM_F32: return (const void*)gfb::gfb_dot_small_m_kernel<float>;
        case GFB_K_DOT_SM_F64: return (const void*)gfb::gfb_dot_small_m_kernel<double>;
        case GFB_K_DOT_TH_F32: return (const void*)gfb::gfb_dot_thread_kernel<float>;
        case GFB_K_DOT_TH_F64: return (const void*)gfb::gfb_dot_thread_kernel<double>;
        case GFB_K_CONV_F32: return (const void*)gfb::gfb_conv_kernel<float>;
        case GFB_K_CONV_F64: return (const void*)gfb::gfb_conv_kernel<double>;
    }
    return nullptr;
}
