/*
 * gfb200.h -- C ABI of the B200 backend transformer (libgfb200.so).
 *
 * This is the drop-in boundary for the reference interpreter backend.  The
 * reference has no FFI: its backend API is the Python functions
 * `compile_function` / `call` / `create_tensor`
 * (/root/reference/pkg/src/graphforge/interpreter.py:92-245, tensor.py:78-102,
 * re-exported from __init__.py:10-45).  The Python package
 * `paper_1801_08058_b200` keeps those signatures and lowers a compiled
 * Function to a *plan* (arena size, constant pool, launch records); this
 * library owns everything on the device:
 *
 *   gfb_exe_create   <- the device half of compile_function  (interpreter.py:92-170)
 *   gfb_exe_run      <- call                                  (interpreter.py:191-245)
 *   gfb_exe_destroy  <- Executable going out of scope
 *   gfb_comm_*       <- collectives the paper lists as future work
 *
 * Conventions: every entry point returns an int status (GFB_OK == 0) and
 * leaves a thread-local message for gfb_last_error().  No torch or CUDA
 * types cross the boundary: device buffers are plain pointers, streams are
 * `void*` (a cudaStream_t, NULL = the per-thread default stream).  The
 * caller owns input/output buffers ("results and parameters are
 * caller-allocated"); the library owns the arena, the constant pool, the
 * device pointer table and the captured CUDA graph.  Concurrent runs of one
 * executable are safe (the reference allows concurrent calls on one
 * Executable): submission is serialised by an internal mutex,
 * and on the device each run waits for the previous run's completion event
 * before it rewrites the pointer table or touches the arena, whatever
 * streams the two runs were issued on.  gfb_exe_destroy waits for the last
 * run.
 */
#ifndef GFB200_H
#define GFB200_H

#ifdef __CUDACC_RTC__ /* runtime-compiled kernels (jit.py): fixed-width types from libcu++ */
#include <cuda/std/cstdint>
typedef cuda::std::int32_t int32_t;
typedef cuda::std::int64_t int64_t;
typedef cuda::std::uint8_t uint8_t;
typedef cuda::std::uint32_t uint32_t;
typedef cuda::std::uint64_t uint64_t;
#else
#include <stdint.h>
#endif

#ifdef __cplusplus
extern "C" {
#endif

enum {
    GFB_OK = 0,
    GFB_ERR_CUDA = 1,
    GFB_ERR_INVALID = 2,
    GFB_ERR_NCCL = 3,
    GFB_ERR_UNSUPPORTED = 4,
};

/* ---- kernel families a launch record can name ------------------------- */
enum {
    GFB_K_EW_F32 = 1, /* fused elementwise / broadcast / reduce VM (gfb_ew_args) */
    GFB_K_EW_F64 = 2,
    GFB_K_EW_I64 = 3,
    GFB_K_EW_U8 = 4,
    GFB_K_EWS_F32 = 5, /* staged ROW variant: cp.async.bulk double-buffered stages (gfb_ew_args, mode 3) */
    GFB_K_EWS_F64 = 6,
    GFB_K_EW1_F32 = 7, /* VM kernel with one element per thread (small, latency-bound launches) */
    GFB_K_EW1_F64 = 8,
    GFB_K_DOT_F32 = 10, /* SIMT Dot, sequential k, bit-exact (gfb_dot_args) */
    GFB_K_DOT_F64 = 11,
    GFB_K_DOT_TC32 = 12, /* tcgen05 3xTF32 Dot on split planes (gfb_tc_args) */
    GFB_K_SPLIT_TF32 = 13, /* F32 -> TF32 hi/lo K-major planes (gfb_split_args) */
    GFB_K_DOT_TC32W = 14,  /* as GFB_K_DOT_TC32 with 128x256 tiles (gfb_tc_args) */
    GFB_K_DOT_TC32P = 19,  /* as GFB_K_DOT_TC32 on a 2-SM CTA pair (cta_group::2), 256x256 tiles; grid.x = 2 * column tiles */
    GFB_K_DOT_SM_F32 = 15, /* SIMT Dot for m <= 8, thread per column, bit-exact (gfb_dot_args) */
    GFB_K_DOT_SM_F64 = 16,
    GFB_K_CONV_TCG64 = 17,  /* implicit-GEMM conv, in-kernel gather + TF32 split, 128x64 tiles (gfb_tcg_args) */
    GFB_K_CONV_TCG128 = 18, /* as GFB_K_CONV_TCG64 with 128x128 tiles */
    GFB_K_CONV_TCX64 = 22,  /* implicit-GEMM conv, TMA box gather + in-smem TF32 split, 128x64 (gfb_tcx_args) */
    GFB_K_CONV_TCX128 = 23, /* as GFB_K_CONV_TCX64 with 128x128 tiles */
    GFB_K_CONV_TCGG64 = 24, /* implicit-GEMM conv, generic k-table gather (any layout, wgrad too), 128x64 (gfb_tcgg_args) */
    GFB_K_CONV_TCGG128 = 25,
    GFB_K_CONV_TCGW64 = 28,  /* weight gradient over channel-last data, MN-major 16-byte gathers, in-kernel TF32 split of both operands, 128x64 (gfb_tcgw_args) */
    GFB_K_CONV_TCGW128 = 29,
    GFB_K_CONV_STEM64 = 32, /* few-channel forward conv: 8x16 pixel tiles built from a shared-memory input patch, resident filter planes (gfb_tcg_args) */
    GFB_K_DOT_TH_F32 = 26, /* SIMT Dot, one thread per output, bit-exact (gfb_dot_args) */
    GFB_K_DOT_TH_F64 = 27,
    GFB_K_CONV_F32 = 20, /* direct Conv2D / ConvBackpropData / ConvBackpropFilter (gfb_conv_args) */
    GFB_K_CONV_F64 = 21,
    GFB_K_ALLREDUCE = 30, /* NCCL sum all-reduce over a byte range (gfb_allreduce_args) */
    GFB_K_DOT_F16P = 34,  /* 2xFP16 block-scaled Dot on a 2-SM CTA pair (kind::f16, 256x256 tiles; gfb_tc_args
                             with the fp16 plane fields): the fp32 accuracy of the 3xTF32 kernel at the f16 rate */
    GFB_K_SPLIT_F16 = 35, /* F32 -> fp16 hi / lo planes + per-128x128-tile power-of-two scales (gfb_split16_args) */
    GFB_K_CHMAX = 36,     /* per-block channel maxima of a channel-last activation (gfb_chsplit_args) */
    GFB_K_CHSPLIT = 37,   /* channel-scaled fp16 hi / lo planes of a channel-last activation (gfb_chsplit_args) */
    GFB_K_FSPLIT = 38,    /* filter -> fp16 hi / lo K-major planes divided by the activation's channel scales,
                             row-scaled (gfb_fsplit_args) */
    GFB_K_CONV_TCXH64 = 39,  /* 2xFP16 implicit-GEMM conv on TMA boxes of fp16 activation planes, 128x64 (gfb_tcxh_args) */
    GFB_K_CONV_TCXH128 = 40, /* as GFB_K_CONV_TCXH64 with 128x128 tiles */
    GFB_K_CONV_TCGWH64 = 41,  /* 2xFP16 weight gradient on TMA boxes of the fp16 planes of x and dy, 128x64 (gfb_tcgwh_args) */
    GFB_K_CONV_TCGWH128 = 42, /* as GFB_K_CONV_TCGWH64 with 128x128 tiles */
    GFB_K_MEMSET = 43,        /* zero a byte range of the arena (gfb_memset_args; a memset node of the graph) */
    GFB_K_CONV_STEMH = 44,    /* few-channel forward conv in 2xFP16: 4x32 pixel tiles built from a shared-memory
                                 input patch, filter split in the prologue (gfb_stemh_args) */
    GFB_K_CONV_STEMH_C3R7 = 45, /* GFB_K_CONV_STEMH compiled for C = 3, R = S = 7 (immediate gather offsets) */
    GFB_K_CONV_STEMWH_C3R7 = 46, /* its weight gradient in 2xFP16 (gfb_stemh_args, w = dy; per-CTA partials) */
    GFB_K_ROWJIT = 33,    /* row-fused launch (softmax-shaped subgraph, one team per row; gfb_row_args):
                             always a runtime-generated kernel (jit.py / rowfuse.py), the built-in
                             entry only traps */
};

/* ---- tensor references inside kernel arguments ------------------------- */
/* A tensor is (slot, byte offset): slot 0 = arena, 1 = constant pool,
 * 2 + i = input i, 2 + n_inputs + j = output j.  Kernels resolve slots
 * through the executable's device pointer table, so the captured CUDA graph
 * stays valid while callers pass new buffers every run. */
#define GFB_REF(slot, offset) ((((uint64_t)(slot)) << 56) | (uint64_t)(offset))
#define GFB_SLOT_ARENA 0
#define GFB_SLOT_CONST 1
#define GFB_SLOT_IO 2

#define GFB_MAX_LEAVES 16
#define GFB_MAX_DIGITS 6
#define GFB_MAX_INSTR 128

/* One mixed-radix digit of an index map: coord = (idx / div) % mod,
 * offset += coord * stride, idx being the output (src 0) or reduced (src 1)
 * flat index of the launch.  Division is by multiply-shift:
 * idx / d == (idx * mul) >> sh for idx < 2^31 (mul == 0 means d == 1);
 * mod == 0 means "no modulo". */
typedef struct {
    uint64_t div_mul;
    uint64_t mod_mul;
    uint32_t div_sh;
    uint32_t mod_sh;
    uint32_t mod;
    int32_t stride;
    int32_t src;
    int32_t pad;
} gfb_digit;

/* A load or store site of the fused program. */
typedef struct {
    uint64_t ref;   /* GFB_REF(slot, byte offset) */
    uint64_t splat; /* raw value bits when mode == 1 */
    int32_t mode;   /* 0 = memory, 1 = splat constant (no memory access) */
    int32_t ndig;
    int32_t vec;    /* along the launch's vector axis: 0 gather, 1 contiguous, 2 uniform,
                       3 patterned: element v of an aligned vector at offset(v0) + dv[v] */
    int32_t rlin;   /* r-part of the offset is r * rlin (0: no r digits); -1: general digits */
    gfb_digit dig[GFB_MAX_DIGITS];
    int32_t dv[8];  /* vec == 3: per-element offsets inside a vector (elements) */
    int32_t same;   /* index of an earlier leaf with the same digits (its offsets are reused), or -1 */
    int32_t pad;
} gfb_leaf;

/* Fused elementwise / broadcast / reduce launch (one VM program).
 * The launch iterates a 2-level index space (o, r), o < n_o, r < n_r.  Each
 * thread evaluates the program on a vector of V consecutive indices (V = 8
 * for 1/4-byte types, 4 for 8-byte types) along r (ROW mode: one warp, or
 * `wpr` warps, per o) or along o (COL mode: r looped per thread, split
 * `split` ways).  red_kind 0 = map (values leave only through STOREs),
 * 1 = sum over r, 2 = max over r into red_out. */
typedef struct {
    const void* const* tab; /* patched by gfb_exe_create */
    uint32_t n_o;
    uint32_t n_r;
    uint32_t ninstr;
    uint32_t nleaves;
    int32_t mode;     /* 1 ROW (vectors along r), 2 COL (vectors along o) */
    int32_t red_kind; /* 0 map, 1 sum, 2 max */
    int32_t vec_axis; /* 1 for ROW, 0 for COL */
    int32_t split;    /* COL: threads splitting r per output vector */
    int32_t npre;     /* leaves 0..npre-1 (<= 4) are loaded up front, all in flight at once */
    int32_t depth;    /* max stack depth of the program (stack lives in shared memory) */
    int32_t wpr;      /* ROW: warps cooperating on one o */
    /* Maps in transposing order: when ty_ext > 0, consecutive lanes take
     * vectors at consecutive values of the digit (i / ty_div) % ty_ext of the
     * vector index i (o in COL, r in ROW; an operand's unit-stride axis)
     * instead of consecutive vectors, so that operand's loads coalesce while
     * every vector store stays whole.  The index extent is a multiple of
     * ty_div * ty_ext and ty_div of the vector width. */
    int32_t ty_ext;
    int32_t ty_div;
    int32_t pad;      /* ROW: nonzero = cache every leaf's r-part offset once per vector
                         (shared between leaves with equal maps); the dynamic shared
                         memory then holds 2 x nleaves offset arrays */
    uint32_t prog[GFB_MAX_INSTR];
    gfb_leaf leaves[GFB_MAX_LEAVES];
    gfb_leaf red_out;
} gfb_ew_args;

/* Dot: C[m, n] = sum_k A[m, k] * B[k, n] with arbitrary element strides
 * (a transposing Reshape feeding a Dot becomes a stride swap). */
typedef struct {
    const void* const* tab;
    uint64_t a, b, c; /* GFB_REF */
    int64_t m, n, k;
    int64_t a_sm, a_sk, b_sk, b_sn, c_sm, c_sn;
} gfb_dot_args;

/* Conv family, operands addressed through per-axis strides (NCHW logical
 * axes, any storage order, so NHWC layout assignment needs no copies). */
typedef struct {
    const void* const* tab;
    uint64_t x, y, out;   /* op-specific roles, see kernels_conv.cu */
    int32_t op;           /* 0 Conv2D, 1 ConvBackpropData, 2 ConvBackpropFilter (sh, sw: the strides of all three),
                             3 MaxPool, 4 MaxPoolBackprop (R, S = window; y = delta for 4) */
    int32_t pad0;
    int64_t N, C, H, W, K, R, S, Ho, Wo;
    int64_t sh, sw, pt, pl;
    int64_t xs[4], ys[4], os[4]; /* element strides of the three operands */
} gfb_conv_args;

/* Split an F32 operand into TF32 hi / lo planes, K-major, rows x kp:
 * hi = rna_tf32(x), lo = rna_tf32(x - hi).  `mode` picks how (row, k)
 * addresses the source (implicit-GEMM forms of the convolution family):
 *   0 plain      src[row * s_r + k * s_k]
 *   1 conv im2col  row=(n,p,q), k=(c,r,s): x[n, c, p*sh-pt+r, q*sw-pl+s]
 *   2 dgrad gather row=(n,h,w), k=(k,r,s): delta[n, k, h+pt-r, w+pl-s]
 *   3 digits     src[row * s_r + d0*t0 + d1*t1 + d2*t2], k=(d0,d1,d2) over e0,e1,e2
 *   4 wgrad gather row=(c,r,s), k=(n,p,q): x[n, c, p+r-pt, q+s-pl]
 *   5 streaming  as 0 with s_k == 1, k == kp (128-bit grid-stride pass)
 * Out-of-range taps read as zero (the reference's zero padding). */
typedef struct {
    const void* const* tab;
    uint64_t src, hi, lo; /* GFB_REF */
    int64_t rows, k, kp;
    int64_t s_r, s_k;
    int32_t mode;
    int32_t pad;
    /* conv geometry: N, C, H, W, R, S, Ho, Wo, sh, sw, pt, pl, e0, e1, e2, unused */
    int64_t geo[16];
    int64_t st[4]; /* element strides of the gathered 4-D tensor, or t0, t1, t2 for mode 3 */
} gfb_split_args;

#if defined(__GNUC__) || defined(__CUDACC__)
#define GFB_ALIGN64 __attribute__((aligned(64)))
#else
#define GFB_ALIGN64
#endif

/* tcgen05 Dot on split planes: C[m, n] = sum_k (Ahi*Bhi + Ahi*Blo + Alo*Bhi).
 * A planes are [M, kp_a] and B planes [N, kp_b] (both K-major); the four
 * CUtensorMap blocks are encoded by gfb_exe_create from the plane refs.
 * Output element (m, n) lives at (m / c_rdiv) * c_s_hi + (m % c_rdiv) * c_s_lo
 * + n * c_sn when c_rdiv > 0 (rows that flatten (n, p, q) of a convolution),
 * else at m * c_sm + n * c_sn.  With k_splits > 1, CTA z reduces the K range
 * [z * k_per_split, +k_per_split) into C + z * split_stride (a partial to be
 * summed by a second pass). */
typedef struct GFB_ALIGN64 {
    const void* const* tab;
    uint64_t c;
    int64_t M, N, K;
    int64_t c_sm, c_sn;
    uint64_t a_hi, a_lo, b_hi, b_lo;
    int64_t kp_a, kp_b;
    int64_t c_rdiv, c_s_hi, c_s_lo;
    int64_t k_splits, k_per_split, split_stride;
    /* MN-major operands (GFB_K_DOT_TC32P only): when a_ld_mn > 0, the A hi /
     * lo operands are stored MN-contiguous, element (m, k) at k * a_ld_mn + m
     * (e.g. a row-major activation read as its own transpose by a weight
     * gradient), loaded as SWIZZLE_128B_ATOM_32B boxes (the tf32 MN-major
     * layout); likewise b_ld_mn for B.  0 = K-major planes [rows, kp]. */
    int64_t a_ld_mn, b_ld_mn;
    int64_t group_m; /* persistent pair kernel: tile raster grouped by this many tile rows (<= 1: row-major) */
    /* Fused epilogue (pair kernel, no split-K; every [M, N] operand dense
     * row-major with row pitch N, bias unit stride), element (m, n), z = the
     * promoted fp32 accumulator:
     *   epi_kind 1 (Dot -> Add(Broadcast(bias)) -> Relu): C = x = z + bias[n];
     *              e_out2[m, n] = x > 0 ? x : 0
     *   epi_kind 2 (Dot -> Multiply(Maximum(Divide(h, x), 0))): C = z * r,
     *              r = h / x >= 0 ? h / x : 0 with h = e_aux1, x = e_aux2
     * and when e_lo != 0, e_lo[m, n] = y - trunc_tf32(y) for the tensor a
     * later GEMM reads as its TF32 hi operand (y = e_out2 for kind 1, C for
     * kind 2).  Each op is the unfused plan's IEEE op: bit-identical. */
    int64_t epi_kind;
    uint64_t e_bias, e_aux1, e_aux2, e_out2, e_lo; /* GFB_REF (an arena ref may be 0: presence is in epi_flags) */
    int64_t epi_flags; /* bit 0: e_out2 is written, bit 1: e_lo is written, bit 2: the fp16 planes
                          e_hi / e_lo / e_sc of y are written (GFB_K_DOT_F16P) */
    /* GFB_K_DOT_F16P: a_hi / a_lo / b_hi / b_lo are fp16 planes (K-major: element (r, k)
     * at r * kp + k; MN-major: at k * ld_mn + r) holding x * s rounded to fp16 (hi) and
     * the rounded remainder (lo), s a power of two per 128 x 128 tile of the plane's
     * storage: s(r, k) = sc[(r / 128) * sc_r + (k / 128) * sc_k].  Every 128-K chunk of
     * the three products is promoted into fp32 registers times 1 / (s_a s_b). */
    uint64_t a_sc, b_sc;
    int64_t a_sc_r, a_sc_k, b_sc_r, b_sc_k;
    /* epi_flags bit 2: fp16 planes of y (e_hi, e_lo: [M, N], pitch N) and their scale
     * grid e_sc ([ceil(M / 128), ceil(N / 128)], row-major) */
    uint64_t e_hi, e_sc;
    /* Relu-gradient mask bytes, [M, N] pitch N: 1 = 1.0, 2 = -0.0, 0 = +0.0, the value of
     * Maximum(Divide(Relu(x), x), 0) (GFB_K_DOT_F16P).  epi_flags bit 3 (kind 1): write
     * the mask of x = C; bit 4 (kind 2): read it instead of e_aux2; bit 5: C is not
     * stored (no reader: the mask and the planes carry everything later launches need). */
    uint64_t e_mask;
    /* epi_flags bit 6: column sums of C over each 32-row block, e_csum[(m / 32) * N + n]
     * (rows in order within a lane, then a fixed shuffle tree): the bias gradient's Sum
     * over the batch finishes as a reduction over ceil(M / 32) rows */
    uint64_t e_csum;
    int64_t pad[1];
    uint64_t tmap[4][16];
} gfb_tc_args;

/* Channel-scaled fp16 planes of a dense channel-last activation [P pixels, C]
 * (C a power of two, 8 <= C <= 1024): GFB_K_CHMAX folds max |x[p, c]| into
 * partial[c] (float bits, atomicMax; zeroed by a GFB_K_MEMSET launch before
 * it); GFB_K_CHSPLIT takes sc[c] = 2^(14 - floor(log2 partial[c])) (block 0
 * stores them in sc) and writes hi = fp16_rn(x sc[c]), lo = fp16_rn(x sc[c] -
 * hi), planes [P, C]. */
typedef struct {
    const void* const* tab;
    uint64_t src, partial, sc, hi, lo; /* GFB_REF */
    int64_t P, C;
    int32_t nblocks, mode;
} gfb_chsplit_args;

/* Filter planes for a channel-scaled activation: B[row, k] with k = (d0, d1,
 * d2) over extents (e0, e1, e2) reads w[row * s_r + d0 t0 + d1 t1 + d2 t2]
 * (d2 = the activation channel); b = w / sc[d2] (exact), t_row = the power of
 * two bringing max_k |b| into [2^14, 2^15); hi / lo = fp16 planes of b t_row,
 * K-major [rows, K]; inv[row] = 1 / t_row.  One block per row. */
typedef struct {
    const void* const* tab;
    uint64_t w, sc, hi, lo, inv; /* GFB_REF */
    int64_t rows, K, s_r;
    int64_t e0, e1, e2, t0, t1, t2;
} gfb_fsplit_args;

/* 2xFP16 implicit-GEMM convolution on TMA boxes of the activation's
 * channel-scaled fp16 planes (gfb_chsplit_args): the layout and tile walk of
 * gfb_tcx_args with K-blocks of 64 channels (C = 64 CB) and two activation
 * maps (hi, lo); the channel scales cancel against the filter planes
 * (gfb_fsplit_args), so C[p, n] = inv[n] * sum_k (Ahi Bhi + Ahi Blo + Alo Bhi),
 * promoted every 128 K into round-to-nearest fp32 registers. */
typedef struct GFB_ALIGN64 {
    const void* const* tab;
    uint64_t c, a_hi, a_lo, b_hi, b_lo, b_inv;
    int64_t N, K;
    int64_t o_n, o_y, o_x, c_sn;
    int64_t a_dims[4];    /* C, W, H, N of the planes (innermost first) */
    int64_t a_strides[4]; /* their element strides */
    int32_t No, Yo, Xo, BX, BY, BNI, tiles_x, tiles_y;
    int32_t sx, sy, ox, oy, S, CB, ksign, pad0;
    int64_t pad[3];
    uint64_t tmap[4][16];
} gfb_tcxh_args;

/* 2xFP16 ConvBackpropFilter (stride 1) on the channel-scaled fp16 planes of
 * x [N, H, W, C] and dy [N, Ho, Wo, K] (gfb_chsplit_args): GEMM rows (r, s, c)
 * (tap-major, C % 64 == 0), columns the K output channels, contraction over
 * the output pixels in boxes of 64 (BX x BY x BNI, tile walk as gfb_tcxh_args).
 * The A tile of a box is two 64-channel TMA boxes of x shifted by their tap
 * (zero-filled padding), B one or two 64-channel boxes of dy, both MN-major;
 * dW[row, col] = sum / (a_sc[c] b_sc[col]) at (row / C) * c_s_hi + (row % C) *
 * c_s_lo + col * c_sn, or, with k_splits > 1, split z's partial at
 * c + z * split_stride + row * N + col (reduced by a second pass). */
typedef struct GFB_ALIGN64 {
    const void* const* tab;
    uint64_t c, a_hi, a_lo, b_hi, b_lo, a_sc, b_sc;
    int64_t M, N, C, S, pt, pl;
    int64_t c_s_hi, c_s_lo, c_sn;
    int64_t k_splits, boxes_per_split, split_stride;
    int64_t a_dims[4], a_strides[4]; /* x planes: C, W, H, N innermost first */
    int64_t b_dims[4], b_strides[4]; /* dy planes: K, Wo, Ho, N */
    int32_t No, Yo, Xo, BX, BY, BNI, tiles_x, tiles_y;
    int64_t pad[8];
    uint64_t tmap[4][16];
} gfb_tcgwh_args;

/* Few-channel forward convolution in 2xFP16 (the 3-channel ResNet stem,
 * stride 1): GEMM row (n, y, x) over (*, Y, X), K index k = (r, s, c) over
 * (R, S, C), K = R S C <= 192, reads x[n, c, y + oy + r, x + ox + s] through
 * the element strides xs0..xs3 (along n, c, h, w; zero outside [0, H) x
 * [0, W)) and the filter w[col, c, r, s] through ws0..ws3 (along the output
 * channel, c, r, s); N <= 64 output channels.  Each 4 x 32 pixel tile takes
 * its own power-of-two activation scale, each filter row its own; both are
 * undone in the epilogue.  Output row (n, y, x), column j at n * c_s_hi +
 * y * c_sm + x * c_s_lo + j * c_sn (and, with flags bit 0, Relu of it at c2:
 * the Relu map of the stem folded into the epilogue). */
typedef struct {
    const void* const* tab;
    uint64_t c, a, w; /* GFB_REF */
    int64_t M, N, K;
    int64_t c_s_hi, c_sm, c_s_lo, c_sn;
    int64_t xs0, xs1, xs2, xs3;
    int64_t ws0, ws1, ws2, ws3;
    int32_t Y, X, oy, ox, H, W, S, C;
    uint64_t c2;   /* GFB_REF: flags bit 0 -- also write Relu(y) (x > 0 ? x : 0) here, same addressing */
    int64_t flags;
} gfb_stemh_args;

/* fp16 split of a dense F32 matrix [rows, cols] (row pitch ld elements, cols % 8 == 0):
 * per 128 x 128 tile, s = 2^(14 - floor(log2(max |x|))) (1 for an all-zero tile),
 * hi = fp16_rn(x s), lo = fp16_rn(x s - hi); sc[tile] = s over the row-major tile grid
 * [ceil(rows / 128), ceil(cols / 128)].  The planes are [rows, cols] dense. */
typedef struct {
    const void* const* tab;
    uint64_t src, hi, lo, sc; /* GFB_REF */
    int64_t rows, cols, ld;
} gfb_split16_args;

/* Implicit-GEMM convolution with the A gather fused into the tensor-core
 * kernel.  A is a 4-D activation with unit channel stride (NHWC storage):
 * GEMM row `row` = (n, y, x) over extents (*, Y, X) has spatial origin
 * h = y*sy + oy, w = x*sx + ox; K index k = (r, s, c) over (R, S, C), C a
 * multiple of 4 (16-byte pieces of 4 channels; K-blocks may span taps)
 * reads a[n, h + ksign*r, w + ksign*s, c] (element strides xs0, xs2, xs3
 * along n, h, w), zero outside [0, H) x [0, W).  Conv2D: (Y, X) = (Ho, Wo),
 * (sy, sx) = strides, (oy, ox) = -(pt, pl), ksign = +1.  ConvBackpropData:
 * (Y, X) = (H, W), unit strides, (oy, ox) = (pt, pl), ksign = -1, and H, W
 * here are the delta's Ho, Wo.  B is the filter as TF32 hi/lo planes
 * [N, K] (K-major, same k order), tensor maps encoded by gfb_exe_create.
 * The output is addressed as in gfb_tc_args. */
typedef struct GFB_ALIGN64 {
    const void* const* tab;
    uint64_t c;
    int64_t M, N, K;
    int64_t c_sm, c_sn, c_rdiv, c_s_hi, c_s_lo;
    uint64_t a, b_hi, b_lo;
    int64_t xs0, xs2, xs3;
    int32_t Y, X, sy, sx, oy, ox, H, W, S, CB, ksign, C; /* C: channel count (multiple of 4; 0 = 32*CB) */
    int64_t pad[2];
    uint64_t tmap[2][16];
} gfb_tcg_args;

/* Implicit-GEMM convolution whose A tiles are TMA boxes.  A CTA's 128 GEMM
 * rows are a box of BNI images x BY output rows x BX output columns (tile
 * `blockIdx.y` = (tn, ty, tx) over tiles_y x tiles_x per image group); the
 * K index is k = (r, s, c) over (R, S, C = 32*CB).  A is a channel-last 4-D
 * activation in the arena (dims a_dims = C, W, H, N innermost first,
 * element strides a_strides); its tensor map (box 32 x BX*sx x BY*sy x BNI,
 * traversal strides 1, sx, sy, 1, zero fill outside) is encoded by
 * gfb_exe_create together with the B plane maps.  The box for K-block
 * (r, s, cb) starts at (32 cb, x0*sx + ox + ksign*s, y0*sy + oy + ksign*r, n0).
 * Output (n, y, x, col) lives at n*o_n + y*o_y + x*o_x + col*c_sn for
 * n < No, y < Yo, x < Xo. */
typedef struct GFB_ALIGN64 {
    const void* const* tab;
    uint64_t c, a, b_hi, b_lo;
    int64_t N, K;
    int64_t o_n, o_y, o_x, c_sn;
    int64_t a_dims[4];
    int64_t a_strides[4];
    int32_t No, Yo, Xo, BX, BY, BNI, tiles_x, tiles_y;
    int32_t sx, sy, ox, oy, S, CB, ksign, pad0;
    int64_t pad[5];
    uint64_t tmap[3][16];
} gfb_tcx_args;

/* Implicit-GEMM convolution with a generic gather.  Row `row` = (i0, i1, i2)
 * over (*, E1, E2) starts at rowoff = i0*ro0 + i1*ro1 + i2*ro2 with spatial
 * origin (h, w) = (i1*hm + h0, i2*wm + w0), or (i0*hm + h0, i1*wm + w0) when
 * pad0 == 1 (weight-gradient rows (r, s, c) over channel-last data, lanes
 * along the contiguous channels).  K index k < K = (k0, k1, k2)
 * over (*, Ke1, Ke2) adds koff = kbase + k0*ko0 + k1*ko1 + k2*ko2 and
 * (dh, dw) = (k1*kh + dh0, k2*kw + dw0).  A[row, k] = a[rowoff + koff] when
 * 0 <= h + dh < H and 0 <= w + dw < W (and k < K), else 0.  Kp = K rounded
 * up to 32.  B is a TF32 hi/lo plane pair [N, >= K] (tensor maps encoded by
 * gfb_exe_create; columns past the plane read as zero); output as
 * gfb_tc_args; split-K over blockIdx.z (kb_per_split K-blocks each) into
 * c + z * split_stride. */
typedef struct GFB_ALIGN64 {
    const void* const* tab;
    uint64_t c, a, b_hi, b_lo;
    int64_t M, N, K, Kp, kp_b;
    int64_t c_sm, c_sn, c_rdiv, c_s_hi, c_s_lo;
    int64_t ro0, ro1, ro2;
    int64_t ko0, ko1, ko2, kbase;
    int64_t k_splits, split_stride;
    int32_t E1, E2, hm, wm, h0, w0, H, W;
    int32_t Ke1, Ke2, kh, kw, dh0, dw0, kb_per_split, pad0;
    uint64_t tmap[2][16]; /* offset 256 */
} gfb_tcgg_args;

/* Weight gradient dW[(r, s, c), k] = sum over pixels (n, p, q) of
 * x[n, p + r - pt, q + s - pl, c] * dy[(n, p, q), k] for channel-last x and
 * dy (c and k contiguous, C and K multiples of 4).  Rows (r, s, c) over
 * (*, E1 = S, E2 = C): rowoff = i0*ro0 + i1*ro1 + i2*ro2, spatial origin
 * (i0 + h0, i1 + w0).  Pixel k = (k0, k1, k2) over (*, Ke1, Ke2): x offset
 * kbase + k0*ko0 + k1*ko1 + k2*ko2 at (dh, dw) = (k1, k2); dy offset
 * k0*yo0 + k1*yo1 + k2*yo2 (+ column).  Both operands are loaded raw with
 * 16-byte cp.async into MN-major tiles and split into TF32 hi/lo in shared
 * memory.  Output and split-K as gfb_tcgg_args. */
typedef struct {
    const void* const* tab;
    uint64_t c, a, b;
    int64_t M, N, K;
    int64_t c_sm, c_sn, c_rdiv, c_s_hi, c_s_lo;
    int64_t ro0, ro1, ro2;
    int64_t ko0, ko1, ko2, kbase;
    int64_t yo0, yo1, yo2;
    int64_t k_splits, split_stride;
    int32_t E1, E2, h0, w0, H, W, Ke1, Ke2, kb_per_split, pad;
} gfb_tcgw_args;

typedef struct {
    const void* const* tab;
    uint64_t buf;   /* GFB_REF of the contiguous gradient bucket */
    uint64_t count; /* elements */
    int32_t dtype;  /* 0 f32, 1 f64 */
    int32_t op;     /* 0 sum (partial gradients), 1 max (a max-reduction over the sharded batch axis) */
} gfb_allreduce_args;

typedef struct {
    const void* const* tab;
    uint64_t buf;   /* GFB_REF into the arena */
    uint64_t bytes;
} gfb_memset_args;

/* Row-fused launch: the generated kernel's tensors, by position (inputs,
 * outputs, per-team partials of cross-row reductions; rowfuse.py). */
#define GFB_ROW_MAX_REFS 30
typedef struct {
    const void* const* tab;
    uint32_t n_refs;
    uint32_t pad;
    uint64_t refs[GFB_ROW_MAX_REFS]; /* GFB_REF */
} gfb_row_args;

/* One kernel launch of the plan; its argument block is args[arg_offset, +arg_size). */
typedef struct {
    uint32_t kind;
    uint32_t grid[3];
    uint32_t block[3];
    uint32_t smem;
    uint32_t arg_offset;
    uint32_t arg_size;
} gfb_launch;

typedef struct {
    uint64_t arena_bytes;
    uint64_t const_bytes;
    const void* const_data; /* uploaded once at create */
    uint32_t n_inputs;
    uint32_t n_outputs;
    uint32_t n_launches;
    uint32_t flags; /* GFB_PLAN_* */
    const gfb_launch* launches;
    uint64_t args_bytes;
    const void* args;
    void* comm; /* gfb_comm* for plans containing GFB_K_ALLREDUCE, else NULL */
} gfb_plan;

enum { GFB_PLAN_CUDA_GRAPH = 1 };

typedef struct gfb_exe gfb_exe;
typedef struct gfb_comm gfb_comm;

int gfb_init(int device);
const char* gfb_last_error(void);
int gfb_device_info(int* sm_major, int* sm_minor, int* num_sms);

int gfb_exe_create(const gfb_plan* plan, gfb_exe** out);
/* inputs[i] / outputs[j]: device pointers for this run (caller-owned), each
 * 16-byte aligned (vector, cp.async and TMA operands; GFB_ERR_INVALID otherwise). */
int gfb_exe_run(gfb_exe* exe, void* const* inputs, void* const* outputs, void* stream);
int gfb_exe_destroy(gfb_exe* exe);
/* Host-buffer runs.  gfb_exe_set_io gives the byte size of every input and
 * result, the inputs each launch reads (CSR over the launch list:
 * reads[read_offsets[i] .. read_offsets[i + 1])) and the last launch writing
 * each result, and allocates device staging buffers for them.
 * gfb_exe_run_host then runs one step on page-locked host buffers: the H2D
 * copies (in first-use order, one stream), the launches (each waiting only
 * for the copies of the inputs it reads) and the D2H copies (each right
 * after the last writer of its result) are one CUDA graph, so the copies
 * overlap the step.  Results are in host_outputs once `stream` reaches the
 * run's end.  Replaces interpreter.py:191-245 `call` on host TensorValues. */
int gfb_exe_set_io(gfb_exe* exe, const uint64_t* in_bytes, const uint64_t* out_bytes, const uint32_t* read_offsets,
                   const uint32_t* reads, const uint32_t* out_writer);
int gfb_exe_run_host(gfb_exe* exe, const void* const* host_inputs, void* const* host_outputs, void* stream);
/* Optional, after gfb_exe_set_io: copy the inputs in pieces (piece p = bytes
 * [piece_offset[p], + piece_bytes[p]) of input piece_input[p]) and let each
 * launch wait only for the pieces it reads (CSR over the launch list, piece
 * indices), e.g. the row chunks of a large input whose first GEMM runs chunk
 * by chunk, so the step starts once the first piece has crossed PCIe. */
int gfb_exe_set_io_pieces(gfb_exe* exe, uint32_t n_pieces, const uint32_t* piece_input, const uint64_t* piece_offset,
                          const uint64_t* piece_bytes, const uint32_t* read_offsets, const uint32_t* reads);
/* Number of kernels one run launches (for bench accounting). */
int gfb_exe_num_launches(const gfb_exe* exe);
/* Launch only record `index` of the plan (profiling / per-kernel timing). */
int gfb_exe_run_one(gfb_exe* exe, uint32_t index, void* const* inputs, void* const* outputs, void* stream);

/* Runtime-compiled kernels (paper_1801_08058_b200/jit.py).  gfb_kernel_load
 * loads an sm_100a cubin and returns the handle of its kernel `name`;
 * gfb_exe_set_kernel makes launch `index` (a GFB_K_EW* record, same grid,
 * block and argument block) use that kernel with `smem` bytes of dynamic
 * shared memory; a NULL kernel skips the launch (its work was merged into
 * an earlier specialised kernel).  The executable's CUDA graph is
 * re-captured on its next run. */
int gfb_kernel_load(const void* cubin, const char* name, const void** kernel);
int gfb_exe_set_kernel(gfb_exe* exe, uint32_t index, const void* kernel, uint32_t smem);
/* Multi-stream capture schedule: launch i is captured on stream stream_of[i]
 * (< n_streams <= 16) after waiting for the earlier launches
 * deps[dep_offsets[i] .. dep_offsets[i + 1]) it conflicts with, so
 * independent launches become concurrent nodes of the executable's CUDA
 * graph (re-captured on the next run).  n_streams == 1 restores the single
 * in-order stream. */
int gfb_exe_set_schedule(gfb_exe* exe, uint32_t n_streams, const uint32_t* stream_of, const uint32_t* dep_offsets,
                         const uint32_t* deps);

/* NCCL communicator, one per process / GPU.  `unique_id` is the 128-byte
 * ncclUniqueId created by rank 0 with gfb_comm_unique_id and shared by the
 * caller's own rendezvous (torch.distributed in the Python layer). */
int gfb_comm_unique_id(void* unique_id_128);
int gfb_comm_create(int nranks, int rank, const void* unique_id_128, gfb_comm** out);
int gfb_comm_destroy(gfb_comm* comm);

#ifdef __cplusplus
}
#endif

#endif /* GFB200_H */
