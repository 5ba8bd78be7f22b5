/*
 * gf_oracle.cpp -- CPU restatement of the reference interpreter kernels.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker for the B200 path
 * and the timed CPU baseline of bench.py's reference arm; nothing in the
 * product package links or calls it.
 *
 * Each kernel restates /root/reference/pkg/src/graphforge/kernels.py with
 * the arithmetic contract of numeric.py:
 *   - F32: every primitive computed in double, rounded once to binary32
 *     (numeric.py:23-31, kernels.py:32-37).  Compiled with
 *     -ffp-contract=off so no FMA ever fuses a multiply into an add.
 *   - I64: two's-complement wrap (numeric.py:34-36) via unsigned arithmetic.
 *   - Fixed accumulation orders: Sum over reduced axes ascending row-major
 *     (kernels.py:156-177), Dot over k ascending (kernels.py:123-133),
 *     Conv2D over c,r,s (kernels.py:180-206), dgrad over k,r,s
 *     (kernels.py:209-235), wgrad over n,p,q (kernels.py:238-264).
 * Parallelism (std::thread) is only across independent output elements, so
 * results are identical for any thread count.
 *
 * All buffers are logical row-major; layouts are value-transparent in the
 * reference (layout.py:1-12) and are not modelled here.
 */
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

using std::int64_t;
using std::uint64_t;

namespace {

enum { ET_F32 = 0, ET_F64 = 1, ET_I64 = 2, ET_BOOL = 3 };
enum { OP_ADD = 0, OP_SUB, OP_MUL, OP_DIV, OP_MAX, OP_NEG, OP_EXP, OP_LOG, OP_TANH, OP_SIGMOID, OP_RELU };

int g_threads = 1;

/* Static block split of [0, n) over g_threads std::threads. */
template <typename F>
void parfor(int64_t n, F body) {
    int t = g_threads;
    if (t <= 1 || n < 256) {
        for (int64_t i = 0; i < n; i++) body(i);
        return;
    }
    std::vector<std::thread> pool;
    int64_t chunk = (n + t - 1) / t;
    for (int w = 0; w < t; w++) {
        int64_t lo = w * chunk, hi = lo + chunk < n ? lo + chunk : n;
        if (lo >= hi) break;
        pool.emplace_back([=] {
            for (int64_t i = lo; i < hi; i++) body(i);
        });
    }
    for (auto& th : pool) th.join();
}

const double kInf = HUGE_VAL;

/* numeric.py:39-46 */
double safe_div(double x, double y) {
    if (y != 0.0) return x / y;
    if (x != x || x == 0.0) return std::nan("");
    return std::copysign(kInf, std::copysign(1.0, x) * std::copysign(1.0, y));
}
/* numeric.py:56-63 */
double safe_log(double x) {
    if (x != x) return x;
    if (x < 0.0) return std::nan("");
    if (x == 0.0) return -kInf;
    return std::log(x);
}
/* numeric.py:66-73 */
double sigmoid(double x) {
    if (x != x) return x;
    if (x >= 0.0) return 1.0 / (1.0 + std::exp(-x));
    double e = std::exp(x);
    return e / (1.0 + e);
}
/* numeric.py:76-78: first operand wins ties, NaN first -> second */
double bmax(double x, double y) { return x >= y ? x : y; }

double apply_f(int op, double x, double y) {
    switch (op) {
        case OP_ADD: return x + y;
        case OP_SUB: return x - y;
        case OP_MUL: return x * y;
        case OP_DIV: return safe_div(x, y);
        case OP_MAX: return bmax(x, y);
        case OP_NEG: return -x;
        case OP_EXP: return std::exp(x); /* overflow -> inf, numeric.py:49-53 */
        case OP_LOG: return safe_log(x);
        case OP_TANH: return std::tanh(x);
        case OP_SIGMOID: return sigmoid(x);
        case OP_RELU: return x > 0.0 ? x : 0.0; /* kernels.py:62 */
    }
    return std::nan("");
}

int64_t apply_i(int op, int64_t x, int64_t y) {
    uint64_t ux = (uint64_t)x, uy = (uint64_t)y;
    switch (op) {
        case OP_ADD: return (int64_t)(ux + uy);
        case OP_SUB: return (int64_t)(ux - uy);
        case OP_MUL: return (int64_t)(ux * uy);
        case OP_NEG: return (int64_t)(0u - ux);
    }
    return 0;
}

inline float f32(double v) { return (float)v; }  // round-to-nearest-even, overflow -> inf

/* acc = round(acc + round(a * b)) -- the F32 MAC of kernels.py:130-132 */
inline float mac32(float acc, float a, float b) { return f32((double)acc + (double)f32((double)a * (double)b)); }

int64_t unravel_off(int64_t flat, int nd, const int64_t* dim, const int64_t* stride) {
    int64_t off = 0;
    for (int d = nd - 1; d >= 0; d--) {
        int64_t q = flat / dim[d];
        off += (flat - q * dim[d]) * stride[d];
        flat = q;
    }
    return off;
}

}  // namespace

extern "C" {

struct orc_red_desc {
    int32_t nk, nr;
    int64_t kdim[8], kstride[8], rdim[8], rstride[8];
};

void orc_set_threads(int n) { g_threads = n > 0 ? n : 1; }
int orc_max_threads(void) { return (int)std::thread::hardware_concurrency(); }

/* kernels.py:101-120: one output element per logical index */
void orc_elementwise(int op, int et, const void* a, const void* b, void* out, int64_t n) {
    if (et == ET_F32) {
        const float *x = (const float*)a, *y = (const float*)b;
        float* o = (float*)out;
        parfor(n, [&](int64_t i) { o[i] = f32(apply_f(op, (double)x[i], y ? (double)y[i] : 0.0)); });
    } else if (et == ET_F64) {
        const double *x = (const double*)a, *y = (const double*)b;
        double* o = (double*)out;
        parfor(n, [&](int64_t i) { o[i] = apply_f(op, x[i], y ? y[i] : 0.0); });
    } else if (et == ET_I64) {
        const int64_t *x = (const int64_t*)a, *y = (const int64_t*)b;
        int64_t* o = (int64_t*)out;
        parfor(n, [&](int64_t i) { o[i] = apply_i(op, x[i], y ? y[i] : 0); });
    }
}

/* kernels.py:143-153 for the 2-D transpose Reshape(x, (1, 0)) (autodiff's
 * dW / dX operands): out[c, r] = in[r, c], a pure copy (bit-exact), in
 * 64 x 64 tiles over all threads */
void orc_transpose2d(int esize, const void* in, void* out, int64_t rows, int64_t cols) {
    const int64_t TB = 64, nbr = (rows + TB - 1) / TB, nbc = (cols + TB - 1) / TB;
    parfor(nbr * nbc, [&](int64_t blk) {
        const int64_t r0 = (blk / nbc) * TB, c0 = (blk % nbc) * TB;
        const int64_t r1 = std::min(rows, r0 + TB), c1 = std::min(cols, c0 + TB);
        if (esize == 4) {
            const uint32_t* x = (const uint32_t*)in;
            uint32_t* y = (uint32_t*)out;
            for (int64_t c = c0; c < c1; c++)
                for (int64_t r = r0; r < r1; r++) y[c * rows + r] = x[r * cols + c];
        } else if (esize == 8) {
            const uint64_t* x = (const uint64_t*)in;
            uint64_t* y = (uint64_t*)out;
            for (int64_t c = c0; c < c1; c++)
                for (int64_t r = r0; r < r1; r++) y[c * rows + r] = x[r * cols + c];
        } else {
            const uint8_t* x = (const uint8_t*)in;
            uint8_t* y = (uint8_t*)out;
            for (int64_t c = c0; c < c1; c++)
                for (int64_t r = r0; r < r1; r++) y[c * rows + r] = x[r * cols + c];
        }
    });
}

/* kernels.py:123-133: acc = add(acc, mul(a[i,k], b[k,j])), k ascending */
void orc_dot(int et, const void* a, const void* b, void* out, int64_t m, int64_t k, int64_t n) {
    if (et == ET_F32) {
        const float *A = (const float*)a, *B = (const float*)b;
        float* C = (float*)out;
        // Work item = 8 rows x 256 columns of C: the accumulators stay in
        // registers / L1 while k ascends and B streams row by row (no
        // transpose).  Every output is still its own k-ascending chain.
        constexpr int64_t RI = 8, CJ = 256;
        const int64_t ni = (m + RI - 1) / RI, nj = (n + CJ - 1) / CJ;
        parfor(ni * nj, [&](int64_t item) {
            const int64_t i0 = (item / nj) * RI, j0 = (item % nj) * CJ;
            const int64_t ri = std::min(RI, m - i0), cj = std::min(CJ, n - j0);
            float acc[RI][CJ];
            for (int64_t ii = 0; ii < ri; ii++)
                for (int64_t jj = 0; jj < cj; jj++) acc[ii][jj] = 0.0f;
            for (int64_t t = 0; t < k; t++) {
                const float* br = B + t * n + j0;
                for (int64_t ii = 0; ii < ri; ii++) {
                    const float av = A[(i0 + ii) * k + t];
                    for (int64_t jj = 0; jj < cj; jj++) acc[ii][jj] = mac32(acc[ii][jj], av, br[jj]);
                }
            }
            for (int64_t ii = 0; ii < ri; ii++)
                for (int64_t jj = 0; jj < cj; jj++) C[(i0 + ii) * n + j0 + jj] = acc[ii][jj];
        });
    } else {
        const double *A = (const double*)a, *B = (const double*)b;
        double* C = (double*)out;
        parfor(m * n, [&](int64_t ij) {
            int64_t i = ij / n, j = ij % n;
            double acc = 0.0;
            for (int64_t t = 0; t < k; t++) acc = acc + A[i * k + t] * B[t * n + j];
            C[ij] = acc;
        });
    }
}

/*
 * kernels.py:156-177.  The input is addressed as [kept..., reduced...]
 * through per-axis strides: out[o] = fold over r ascending of
 * in[koff(o) + roff(r)], starting from 0 (sum) or -inf (max).
 */
void orc_reduce(int is_max, int et, const void* in, void* out, const orc_red_desc* d, int64_t n_out, int64_t n_red) {
    if (et == ET_F32 || et == ET_F64) {
        parfor(n_out, [&](int64_t i) {
            int64_t base = unravel_off(i, d->nk, d->kdim, d->kstride);
            double acc = is_max ? -kInf : 0.0;
            for (int64_t r = 0; r < n_red; r++) {
                int64_t off = base + unravel_off(r, d->nr, d->rdim, d->rstride);
                double v = et == ET_F32 ? (double)((const float*)in)[off] : ((const double*)in)[off];
                if (is_max) acc = bmax(acc, v);
                else acc = et == ET_F32 ? (double)f32(acc + v) : acc + v;
            }
            if (et == ET_F32) ((float*)out)[i] = (float)acc;
            else ((double*)out)[i] = acc;
        });
    } else if (et == ET_I64) {
        const int64_t* x = (const int64_t*)in;
        parfor(n_out, [&](int64_t i) {
            int64_t base = unravel_off(i, d->nk, d->kdim, d->kstride);
            uint64_t acc = 0;
            for (int64_t r = 0; r < n_red; r++) acc += (uint64_t)x[base + unravel_off(r, d->nr, d->rdim, d->rstride)];
            ((int64_t*)out)[i] = (int64_t)acc;
        });
    }
}

/* kernels.py:180-206: NCHW x KCRS, zero padding, order c, r, s */
void orc_conv2d(int et, const void* data, const void* flt, void* out, int64_t N, int64_t C, int64_t H, int64_t W,
                int64_t K, int64_t R, int64_t S, int64_t sh, int64_t sw, int64_t pt, int64_t pl, int64_t Ho,
                int64_t Wo) {
    parfor(N * K * Ho * Wo, [&](int64_t idx) {
        int64_t q = idx % Wo, p = (idx / Wo) % Ho, k = (idx / (Wo * Ho)) % K, n = idx / (Wo * Ho * K);
        float a32 = 0.0f;
        double a64 = 0.0;
        for (int64_t c = 0; c < C; c++)
            for (int64_t r = 0; r < R; r++) {
                int64_t h = p * sh - pt + r;
                if (h < 0 || h >= H) continue;
                for (int64_t s = 0; s < S; s++) {
                    int64_t w = q * sw - pl + s;
                    if (w < 0 || w >= W) continue;
                    int64_t xi = ((n * C + c) * H + h) * W + w, fi = ((k * C + c) * R + r) * S + s;
                    if (et == ET_F32) a32 = mac32(a32, ((const float*)data)[xi], ((const float*)flt)[fi]);
                    else a64 = a64 + ((const double*)data)[xi] * ((const double*)flt)[fi];
                }
            }
        if (et == ET_F32) ((float*)out)[idx] = a32;
        else ((double*)out)[idx] = a64;
    });
}

/* kernels.py:209-235: adjoint w.r.t. data, order k, r, s.  The reference is
 * stride-1 only; for the IR extension (strided Conv2D gradients) the same
 * loop keeps the taps with (h + pt - r) and (w + pl - s) divisible by the
 * stride: p = (h + pt - r) / sh, q = (w + pl - s) / sw. */
void orc_conv_bwd_data(int et, const void* delta, const void* flt, void* out, int64_t N, int64_t C, int64_t H,
                       int64_t W, int64_t K, int64_t R, int64_t S, int64_t Ho, int64_t Wo, int64_t pt, int64_t pl,
                       int64_t sh, int64_t sw) {
    parfor(N * C * H * W, [&](int64_t idx) {
        int64_t w = idx % W, h = (idx / W) % H, c = (idx / (W * H)) % C, n = idx / (W * H * C);
        float a32 = 0.0f;
        double a64 = 0.0;
        for (int64_t k = 0; k < K; k++)
            for (int64_t r = 0; r < R; r++) {
                int64_t pn = h + pt - r;
                if (pn < 0 || pn % sh) continue;
                int64_t p = pn / sh;
                if (p >= Ho) continue;
                for (int64_t s = 0; s < S; s++) {
                    int64_t qn = w + pl - s;
                    if (qn < 0 || qn % sw) continue;
                    int64_t q = qn / sw;
                    if (q >= Wo) continue;
                    int64_t di = ((n * K + k) * Ho + p) * Wo + q, fi = ((k * C + c) * R + r) * S + s;
                    if (et == ET_F32) a32 = mac32(a32, ((const float*)delta)[di], ((const float*)flt)[fi]);
                    else a64 = a64 + ((const double*)delta)[di] * ((const double*)flt)[fi];
                }
            }
        if (et == ET_F32) ((float*)out)[idx] = a32;
        else ((double*)out)[idx] = a64;
    });
}

/* kernels.py:238-264: adjoint w.r.t. filter, order n, p, q (strided taps
 * h = p * sh + r - pt for the IR extension; the reference has sh = sw = 1) */
void orc_conv_bwd_filter(int et, const void* data, const void* delta, void* out, int64_t N, int64_t C, int64_t H,
                         int64_t W, int64_t K, int64_t R, int64_t S, int64_t Ho, int64_t Wo, int64_t pt, int64_t pl,
                         int64_t sh, int64_t sw) {
    parfor(K * C * R * S, [&](int64_t idx) {
        int64_t s = idx % S, r = (idx / S) % R, c = (idx / (S * R)) % C, k = idx / (S * R * C);
        float a32 = 0.0f;
        double a64 = 0.0;
        for (int64_t n = 0; n < N; n++)
            for (int64_t p = 0; p < Ho; p++) {
                int64_t h = p * sh + r - pt;
                if (h < 0 || h >= H) continue;
                for (int64_t q = 0; q < Wo; q++) {
                    int64_t w = q * sw + s - pl;
                    if (w < 0 || w >= W) continue;
                    int64_t di = ((n * K + k) * Ho + p) * Wo + q, xi = ((n * C + c) * H + h) * W + w;
                    if (et == ET_F32) a32 = mac32(a32, ((const float*)delta)[di], ((const float*)data)[xi]);
                    else a64 = a64 + ((const double*)delta)[di] * ((const double*)data)[xi];
                }
            }
        if (et == ET_F32) ((float*)out)[idx] = a32;
        else ((double*)out)[idx] = a64;
    });
}

/* IR extension (no reference counterpart): MaxPool over (kh, kw) windows
 * with strides and padding.  out = fold over the window in row-major order
 * of acc >= v ? acc : v from -inf (the reference's max-reduce fold,
 * kernels.py:156-177), padding taps skipped. */
void orc_maxpool(int et, const void* data, void* out, int64_t N, int64_t C, int64_t H, int64_t W, int64_t kh,
                 int64_t kw, int64_t sh, int64_t sw, int64_t pt, int64_t pl, int64_t Ho, int64_t Wo) {
    parfor(N * C * Ho * Wo, [&](int64_t idx) {
        int64_t q = idx % Wo, p = (idx / Wo) % Ho, nc = idx / (Wo * Ho);
        double acc = -kInf;
        for (int64_t i = 0; i < kh; i++) {
            int64_t h = p * sh + i - pt;
            if (h < 0 || h >= H) continue;
            for (int64_t j = 0; j < kw; j++) {
                int64_t w = q * sw + j - pl;
                if (w < 0 || w >= W) continue;
                int64_t xi = (nc * H + h) * W + w;
                double v = et == ET_F32 ? (double)((const float*)data)[xi] : ((const double*)data)[xi];
                acc = bmax(acc, v);
            }
        }
        if (et == ET_F32) ((float*)out)[idx] = (float)acc;
        else ((double*)out)[idx] = acc;
    });
}

/* MaxPoolBackprop: dx[n,c,h,w] = sum, over the windows (p, q) ascending that
 * contain (h, w) and whose selected element (the position where the forward
 * fold last took a new value) is (h, w), of delta[n,c,p,q]; from +0.0 with
 * one rounding per add. */
void orc_maxpool_bwd(int et, const void* data, const void* delta, void* out, int64_t N, int64_t C, int64_t H,
                     int64_t W, int64_t kh, int64_t kw, int64_t sh, int64_t sw, int64_t pt, int64_t pl, int64_t Ho,
                     int64_t Wo) {
    auto X = [&](int64_t i) { return et == ET_F32 ? (double)((const float*)data)[i] : ((const double*)data)[i]; };
    auto D = [&](int64_t i) { return et == ET_F32 ? (double)((const float*)delta)[i] : ((const double*)delta)[i]; };
    parfor(N * C * H * W, [&](int64_t idx) {
        int64_t w = idx % W, h = (idx / W) % H, nc = idx / (W * H);
        double acc = 0.0;
        for (int64_t p = 0; p < Ho; p++) {
            int64_t i = h + pt - p * sh;
            if (i < 0 || i >= kh) continue;
            for (int64_t q = 0; q < Wo; q++) {
                int64_t j = w + pl - q * sw;
                if (j < 0 || j >= kw) continue;
                double best = -kInf;
                int64_t arg = -1;
                for (int64_t a = 0; a < kh; a++) {
                    int64_t hh = p * sh + a - pt;
                    if (hh < 0 || hh >= H) continue;
                    for (int64_t b = 0; b < kw; b++) {
                        int64_t ww = q * sw + b - pl;
                        if (ww < 0 || ww >= W) continue;
                        double v = X((nc * H + hh) * W + ww);
                        if (!(best >= v)) {
                            best = v;
                            arg = hh * W + ww;
                        }
                    }
                }
                if (arg == h * W + w) {
                    double d = D((nc * Ho + p) * Wo + q);
                    acc = et == ET_F32 ? (double)f32(acc + d) : acc + d;
                }
            }
        }
        if (et == ET_F32) ((float*)out)[idx] = (float)acc;
        else ((double*)out)[idx] = acc;
    });
}

}  // extern "C"
