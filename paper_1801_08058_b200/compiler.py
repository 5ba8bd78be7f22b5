"""Lowering of a compiled Function to B200 launches (the transformer proper).

The reference turns every IR node into one interpreter instruction over a
per-node arena plan (`/root/reference/pkg/src/graphforge/interpreter.py:92-170`,
`memory.py:77-120`).  This pass instead:

1. **Fusion.**  Memory-bound nodes (elementwise, Broadcast, Reshape,
   ConvertLayout, Sum) are grouped; only tensors somebody must see are
   *materialised* — results, Sum outputs, operands of Dot/Conv that cannot
   be read through strides, and values with several consumers.  Each group
   becomes one launch of the fused VM kernel (`csrc/ew_vm.cu`): the node
   expressions compile to a short accumulator-stack program, every read of
   a materialised tensor becomes a *leaf* addressed through a mixed-radix
   digit map (Broadcast = dropped digit, axis permutation / ConvertLayout =
   permuted strides, row-major Reshape = re-split digits), so index ops cost
   no memory traffic at all.  A Sum whose input is also a result stores that
   input as a side output of the same pass (config B: one read of a and b,
   one write of t3, one write of the row sums).
2. **Strided heavy operands.**  Dot / Conv kernels take per-axis strides,
   so the `Reshape(x, (1, 0))` transposes autodiff emits
   (`autodiff.py:163-177`) and NHWC layouts are read in place.
3. **Liveness over launches.**  Arena placement (`memory.plan_buffers`) is
   first-fit over materialised buffers with live ranges in launch indices;
   fused intermediates never touch memory.

The result is a list of launch records + argument blocks (`abi.py`) that
`libgfb200.so` captures into one CUDA graph.
"""

from __future__ import annotations

import ctypes as C
import os
import struct
from dataclasses import dataclass, field

import numpy as np

from . import abi
from .errors import UnsupportedOp
from .ir import (
    conv_strides,
    ELEMENTWISE_BINARY,
    ELEMENTWISE_UNARY,
    ConstantData,
    ElementType,
    Function,
    OpKind,
    element_count,
    reachable_from_results,
    topological_order,
)
from .memory import DEVICE_ALIGNMENT, align_up, plan_buffers
from .layout import NHWC_ORDER, Layout

NUM_SMS = 148
# Grid cap of the ROW / COL elementwise launches, in blocks per SM.  Measured
# on config B (scripts/b_sweep.cu): 16 blocks/SM (a grid-stride loop of ~3.5
# row groups per block) 123.3 us, 32 -> 119.7, 55 (one row group per block)
# 119.2; the blocks of the last wave are then short, so the tail is short too.
EW_BLOCKS_PER_SM = int(os.environ.get("GFB_EW_BLOCKS_PER_SM", 64))
# ROW launches add warps per row (up to 8) while the grid has fewer than this
# many 8-warp blocks per SM.
ROW_BLOCKS_PER_SM = int(os.environ.get("GFB_EW_ROW_BLOCKS_PER_SM", 32))
HEAVY = frozenset({OpKind.DOT, OpKind.CONV2D, OpKind.CONV_BACKPROP_DATA, OpKind.CONV_BACKPROP_FILTER,
                   OpKind.MAX_POOL, OpKind.MAX_POOL_BACKPROP})
INDEX_OPS = frozenset({OpKind.BROADCAST, OpKind.RESHAPE, OpKind.CONVERT_LAYOUT})
MAX_STACK = 3
TINY_DOT_K = 4  # Dots contracting over at most this many terms fuse as light ops
MAX_PRELOAD = 4

# Program construction opcodes (internal), encoded to the kernel's flat
# jump-table opcodes by `encode_flat` (csrc/ew_vm.cu, "Flat opcodes").
I_LOAD, I_UN, I_BIN_LEAF, I_BIN_POP, I_BIN_SELF, I_PUSH, I_STORE, I_PUSH_LOAD = 1, 2, 3, 4, 5, 6, 7, 8
I_DOT = 9  # acc = acc + leaf[k] * leaf[k2] (two roundings): one tiny-Dot term, no operand stack
F_LOADP, F_LOADM, F_PUSH, F_STORE, F_UN, F_BIN = 1, 5, 6, 7, 8, 16
F_DOT = 14
SRC_MEM, SRC_POP, SRC_SELF = 4, 5, 6


def encode_flat(code, npre: int) -> list:
    """(cls, op, leaf, swap) tuples -> kernel words (low byte opcode, leaf << 8)."""
    out = []
    for cls, op, k, swap in code:
        if cls == I_PUSH_LOAD:
            out.append(F_PUSH)
            cls = I_LOAD
        if cls == I_DOT:
            out.append(F_DOT | (k << 8) | (swap << 16))  # swap holds the second leaf
            continue
        if cls == I_LOAD:
            out.append(F_LOADP + k if k < npre else F_LOADM | (k << 8))
        elif cls == I_PUSH:
            out.append(F_PUSH)
        elif cls == I_STORE:
            out.append(F_STORE | (k << 8))
        elif cls == I_UN:
            out.append(F_UN + op - 5)
        elif cls == I_BIN_LEAF:
            src = k if k < npre else SRC_MEM
            out.append(F_BIN + (src * 5 + op) * 2 + swap | ((k << 8) if src == SRC_MEM else 0))
        elif cls == I_BIN_POP:
            out.append(F_BIN + (SRC_POP * 5 + op) * 2 + (1 - swap))
        elif cls == I_BIN_SELF:
            out.append(F_BIN + (SRC_SELF * 5 + op) * 2)
        else:
            raise ValueError(cls)
    return out


def _staged_policy() -> str:
    """GFB_STAGED: "1" staged kernel wherever it applies, "0" never, "auto"
    (default with runtime specialisation) only for few long rows."""
    from . import jit

    return os.environ.get("GFB_STAGED", "auto" if jit.enabled() else "1")


def decode_flat(word: int):
    """Kernel word -> (kind, arg...) for the host emulator."""
    code, k = word & 0xFF, (word >> 8) & 0xFF
    if F_LOADP <= code < F_LOADP + 4:
        return ("loadp", code - F_LOADP)
    if code == F_LOADM:
        return ("loadm", k)
    if code == F_PUSH:
        return ("push",)
    if code == F_STORE:
        return ("store", k)
    if code == F_DOT:
        return ("dot", k, (word >> 16) & 0xFF)
    if F_UN <= code < F_UN + 6:
        return ("un", code - F_UN + 5)
    rel = code - F_BIN
    s, rest = rel % 2, rel // 2
    src, op = rest // 5, rest % 5
    return ("bin", src, op, s, k)
VM_OP = {
    OpKind.ADD: 0, OpKind.SUBTRACT: 1, OpKind.MULTIPLY: 2, OpKind.DIVIDE: 3, OpKind.MAXIMUM: 4,
    OpKind.NEGATE: 5, OpKind.EXP: 6, OpKind.LOG: 7, OpKind.TANH: 8, OpKind.SIGMOID: 9, OpKind.RELU: 10,
}
EW_KIND = {ElementType.F32: abi.K_EW_F32, ElementType.F64: abi.K_EW_F64, ElementType.I64: abi.K_EW_I64, ElementType.BOOL: abi.K_EW_U8}
EW1_KIND = {ElementType.F32: abi.K_EW1_F32, ElementType.F64: abi.K_EW1_F64}
SCALAR_VM_MAX = 1 << 17  # launches of at most this many (o, r) elements use one element per thread
INDEX_LIMIT = 1 << 31

# tcgen05 Dot (csrc/gemm_tc.cu): 128x128 tiles (3 stages of 64 KB) or, for
# N >= 256, 128x256 tiles (2 stages of 96 KB, 320 threads).
TC_TILE = 128
TC_SMEM = 3 * 4 * 128 * 32 * 4 + 1024 + 256
TC_SMEM_W = 2 * (2 * 128 + 2 * 256) * 32 * 4 + 1024 + 256
TC_SMEM_PAIR = TC_SMEM + 8 * 32 * 32 * 4  # + the epilogue warps' transpose tiles (gemm_tc.cu PCfg::SMEM_BYTES_PAIR)
F16_SMEM_PAIR = TC_SMEM_PAIR  # gemm_f16.cu HCfg::SMEM_BYTES: same 64 KB stages (64 fp16 K instead of 32 fp32 K)
# gfb_conv_tcg_kernel: MMA stages + 4 raw A K-blocks + row table + barriers (gemm_tc.cu GCfg)
# gfb_conv_tcx_kernel: MMA stages (3 at BN=128, 4 at BN=64) + barriers (gemm_tc.cu XCfg)
TCX_SMEM = {bn: (3 if bn == 128 else 4) * (2 * 128 + 2 * bn) * 32 * 4 + 256 + 1024 for bn in (64, 128)}
TCXH_SMEM = {bn: (3 if bn == 128 else 4) * (2 * 128 + 2 * bn) * 64 * 2 + 256 + 1024 for bn in (64, 128)}  # conv_f16.cu HXCfg
TCGWH_SMEM = {bn: (3 if bn == 128 else 4) * (2 * 128 + 2 * bn) * 64 * 2 + 256 + 1024 for bn in (64, 128)}  # conv_f16.cu HWCfg
CHMAX_BLOCKS = 2 * 148  # channel-max blocks: more only adds atomicMax contention
STEM_THREADS = 64 + 32 * (4 + 8)  # csrc/gemm_tc.cu SCfg
STEM_SMEM = 4 * 32768 + 5 * 2 * 8192 + 2 * 1536 * 4 + 5 * 32 * 4 + 256 + 1024
STEMH_SMEM = 4 * 32768 + 3 * 2 * 8192 + 32768 + 2 * 1536 * 4 + 3 * 64 * 4 + (16 + 64 + 16) * 4 + 256 + 1024  # conv_f16.cu HSCfg
STEMWH_THREADS = 64 + 32 * (8 + 8)  # conv_f16.cu HSWCfg
STEMWH_SMEM = 2 * 65536 + 4 * 16384 + 4 * 1024 * 4 + 2 * 1024 * 4 + (16 + 2 * 8) * 4 + 256 + 1024
TCGW_THREADS = {64: 64 + 32 * (4 + 8), 128: 64 + 32 * (4 + 4)}  # csrc/gemm_tc.cu WCfg::THREADS
TCGW_SMEM = {64: 3 * (2 * 16384 + 2 * 8192) + 3 * (16384 + 8192) + 1280,
             128: 2 * (2 * 16384 + 2 * 16384) + 2 * (16384 + 16384) + 1280}  # WCfg::SMEM_BYTES
TCGG_THREADS = {64: 64 + 32 * (4 + 8), 128: 64 + 32 * (4 + 4)}  # csrc/gemm_tc.cu GCfg::THREADS_GG
TCG_SMEM = {bn: (2 if bn == 128 else 3) * (2 * 128 + 2 * bn) * 32 * 4 + 4 * 128 * 32 * 4 + 128 * 16 + 256 + 1024
            for bn in (64, 128)}


def _conv_tc_ok(m: int, n: int, k: int) -> bool:
    """Convolutions as implicit GEMMs go to the tensor cores when big enough
    (skinny outputs with a deep K run split-K)."""
    return m * n * k >= (1 << 22) and (max(m, n) >= 128 or k >= 4096) and k >= 16


def _conv_out_digits(addr: dict, m: int, ncols: int) -> list:
    """Digits of the implicit-GEMM output map (o = row * ncols + col)."""
    if "c_rdiv" in addr:
        rdiv = addr["c_rdiv"]
        digs = [(0, ncols * rdiv, None, addr["c_s_hi"]), (0, ncols, rdiv, addr["c_s_lo"]), (0, 1, ncols, addr["c_sn"])]
    else:
        digs = [(0, ncols, None, addr["c_sm"]), (0, 1, ncols, addr["c_sn"])]
    return [d for d in digs if d[3] != 0]


def use_f16() -> bool:
    """Large dense F32 Dots on the 2xFP16 block-scaled pair GEMM (kind::f16,
    csrc/gemm_f16.cu) instead of 3xTF32; GFB_F16=0 selects 3xTF32."""
    import os

    return os.environ.get("GFB_F16", "1") == "1"


def use_tensor_cores(m: int, n: int, k: int) -> bool:
    """F32 Dots big enough to fill tensor-core tiles go to tcgen05 3xTF32
    (normwise 1e-5 contract); small / skinny ones keep the exact-order SIMT
    kernel (bit-exact).  GFB_DOT=simt|tc overrides for tests."""
    import os

    mode = os.environ.get("GFB_DOT", "auto")
    if mode == "simt":
        return False
    if mode == "tc":
        return m >= 1 and n >= 1 and k >= 1
    if m * n * k < (1 << 22):
        return False
    return (m >= 64 and n >= 64 and k >= 64) or k >= 4096  # deep, skinny: split-K


def magic_u31(d: int) -> tuple[int, int]:
    """(mul, sh) with n // d == (n * mul >> 32) >> sh for all 0 <= n < 2**31."""
    if d <= 0:
        raise ValueError(d)
    if d == 1:
        return 0, 0
    l = (d - 1).bit_length()  # ceil(log2 d)
    mul = (1 << (31 + l)) // d + 1
    assert mul < (1 << 32)
    return mul, l - 1


def _prod(xs) -> int:
    p = 1
    for x in xs:
        p *= x
    return p


# ---------------------------------------------------------------------------
# Buffers and index maps


@dataclass
class Buffer:
    key: int
    et: ElementType
    shape: tuple
    strides: tuple  # element stride per logical axis
    slot: int = abi.SLOT_ARENA
    offset: int = 0
    splat: object = None  # python scalar for splat constants (no memory)
    base: object = None   # a strided view of this Buffer (shares its storage and final offset)
    elem_off: int = 0     # view origin, in elements from the base's origin
    subaxes: dict = None  # axis -> [(extent, stride), ...] outer to inner: a flattened axis stored permuted
    bucket: object = None  # (gradient region, is_max) for a data-parallel partial root
    exact: bool = False   # a contiguous view [elem_off, + its element count) of its base (row chunks)

    @property
    def nbytes(self) -> int:
        return element_count(self.shape) * self.et.byte_size


# An axis expression: coordinate = (idx[src] // div) % mod, or None (always 0).
AxisExpr = tuple  # (src, div, mod)


def iteration_axes(shape, src=0) -> list:
    out = []
    for a, d in enumerate(shape):
        out.append(None if d == 1 else (src, _prod(shape[a + 1:]), d))
    return out


class Unexpressible(Exception):
    pass


class _TooManyDigits(Exception):
    """An operand's index map needs more than GFB_MAX_DIGITS digits."""


class Lin:
    """A composite axis coordinate: const + sum of mul * ((idx[src] // div) % mod).

    Plain digits stay (src, div, mod) tuples; Lin appears where a Reshape
    merges several iteration digits into one input axis (a pool window's
    h = 2*h2 + dy) or where a coordinate is a compile-time constant (a tiny
    Dot's contraction index)."""

    __slots__ = ("terms", "const")

    def __init__(self, terms=(), const=0):
        self.terms = tuple(terms)
        self.const = int(const)

    def __repr__(self):
        return f"Lin({self.terms}, {self.const})"


def axis_terms(e):
    """(terms, const) of an axis expression; terms are (src, div, mod, mul)."""
    if e is None:
        return (), 0
    if isinstance(e, Lin):
        return e.terms, e.const
    return ((e[0], e[1], e[2], 1),), 0


def _mk_axis(terms, const):
    terms = tuple(t for t in terms)
    if not terms and const == 0:
        return None
    if len(terms) == 1 and const == 0 and terms[0][3] == 1:
        return terms[0][:3]
    return Lin(terms, const)


def _split_expr(e, dims):
    """Coordinates over `dims` (row-major) of an out axis holding e.

    A plain digit splits into sub-digits; a composite coordinate splits when
    each of its terms lands inside one dim without carrying into the next
    (term mul = P_i * m with m * mod <= dims[i], P_i the inner product), and
    its constant decomposes likewise."""
    if e is None:
        return [None] * len(dims)
    if not isinstance(e, Lin):
        src, div, mod = e
        return [None if d == 1 else (src, div * _prod(dims[i + 1:]), d) for i, d in enumerate(dims)]
    if len(e.terms) == 1 and e.const == 0 and e.terms[0][3] == 1 and e.terms[0][2] is not None \
            and e.terms[0][2] == _prod(dims):
        return _split_expr(e.terms[0][:3], dims)
    inner = [_prod(dims[i + 1:]) for i in range(len(dims))]
    per_terms = [[] for _ in dims]
    per_max = [0] * len(dims)
    c = e.const
    consts = [(c // inner[i]) % d for i, d in enumerate(dims)]
    if sum(consts[i] * inner[i] for i in range(len(dims))) != c:
        raise Unexpressible()
    for src, div, mod, mul in e.terms:
        if mod is None:
            raise Unexpressible()
        for i in range(len(dims)):
            if mul % inner[i] == 0 and (mul // inner[i]) * (mod - 1) < dims[i]:
                m = mul // inner[i]
                per_terms[i].append((src, div, mod, m))
                per_max[i] += m * (mod - 1)
                break
        else:
            raise Unexpressible()
    for i, d in enumerate(dims):
        if consts[i] + per_max[i] >= d:
            raise Unexpressible()  # would carry into the next dim
    return [_mk_axis(per_terms[i], consts[i]) for i in range(len(dims))]


def _reshape_groups(out_shape, perm_dims):
    """Minimal aligned groups (out axes, perm axes) with equal extents."""
    groups, i, j = [], 0, 0
    no, npm = len(out_shape), len(perm_dims)
    while i < no or j < npm:
        go, gp, po, pp = [], [], 1, 1
        while True:
            if po == pp and (go or gp):
                # absorb trailing unit axes into this group
                while i < no and out_shape[i] == 1:
                    go.append(i)
                    i += 1
                while j < npm and perm_dims[j] == 1:
                    gp.append(j)
                    j += 1
                break
            if (po <= pp and i < no) or j >= npm:
                po *= out_shape[i]
                go.append(i)
                i += 1
            else:
                pp *= perm_dims[j]
                gp.append(j)
                j += 1
            if i >= no and j >= npm:
                break
        groups.append((go, gp))
    return groups


def through_reshape(node, out_axes) -> list:
    """Axis expressions of a Reshape's input given those of its output."""
    in_shape = node.inputs_shape
    order = node.attrs["input_order"]
    out_shape = tuple(node.output.shape)
    perm_dims = tuple(in_shape[a] for a in order)
    in_axes = [None] * len(in_shape)
    if perm_dims == out_shape:
        for i, a in enumerate(order):
            in_axes[a] = out_axes[i]
        return in_axes
    simple = all(e is None or not isinstance(e, Lin) for e in out_axes)
    if simple:
        # The output's axes as one contiguous digit block re-split as a whole.
        live = [(a, e) for a, e in enumerate(out_axes) if e is not None and out_shape[a] > 1]
        if not live:
            return in_axes  # single element
        srcs = {e[0] for _, e in live}
        ok = len(srcs) == 1
        if ok:
            src = srcs.pop()
            last_axis, last = live[-1]
            base = last[1] // _prod(out_shape[last_axis + 1:])
            ok = all(e[2] == out_shape[a] and e[1] == base * _prod(out_shape[a + 1:]) for a, e in live)
        if ok:
            for i, a in enumerate(order):
                d = perm_dims[i]
                in_axes[a] = None if d == 1 else (src, base * _prod(perm_dims[i + 1:]), d)
            return in_axes
    # Aligned groups: merges become linear combinations, splits sub-digits.
    perm_axes = [None] * len(perm_dims)
    for go, gp in _reshape_groups(out_shape, perm_dims):
        outs = [a for a in go if out_shape[a] > 1]
        perms = [i for i in gp if perm_dims[i] > 1]
        if not perms:
            continue
        if len(perms) == 1:
            terms, const = [], 0
            for a in outs:
                w = _prod(out_shape[b] for b in outs if b > a)
                t, c = axis_terms(out_axes[a])
                terms += [(src, div, mod, mul * w) for src, div, mod, mul in t]
                const += c * w
            perm_axes[perms[0]] = _mk_axis(terms, const)
        elif len(outs) == 1:
            for i, e in zip(perms, _split_expr(out_axes[outs[0]], [perm_dims[i] for i in perms])):
                perm_axes[i] = e
        elif not outs:
            continue
        else:
            raise Unexpressible()
    for i, a in enumerate(order):
        in_axes[a] = perm_axes[i]
    return in_axes


def through_index_op(node, out_axes) -> list:
    if node.op is OpKind.CONVERT_LAYOUT:
        return list(out_axes)
    if node.op is OpKind.BROADCAST:
        drop = set(node.attrs["broadcast_axes"])
        return [e for a, e in enumerate(out_axes) if a not in drop]
    return through_reshape(node, out_axes)


def _axis_parts(buf: Buffer, a: int, e):
    """(terms (src, div, mod, stride), constant element offset) of axis a at e."""
    sub = buf.subaxes.get(a) if buf.subaxes else None
    if sub is None:
        terms, const = axis_terms(e)
        return [(src, div, mod, buf.strides[a] * mul) for src, div, mod, mul in terms], const * buf.strides[a]
    parts = _split_expr(e, [x for x, _ in sub])
    terms, off = [], 0
    for (x, stride), pe in zip(sub, parts):
        t, c = axis_terms(pe)
        terms += [(src, div, mod, stride * mul) for src, div, mod, mul in t]
        off += c * stride
    return terms, off


def axes_offset(buf: Buffer, axes) -> int:
    """Element offset contributed by the constant parts of `axes`."""
    off = 0
    for a, e in enumerate(axes):
        if e is not None and buf.shape[a] > 1 and (isinstance(e, Lin) or (buf.subaxes and a in buf.subaxes)):
            off += _axis_parts(buf, a, e)[1]
    return off


def make_digits(buf: Buffer, axes, extents) -> list:
    """Mixed-radix digits (src, div, mod, stride) addressing `buf` at `axes`
    (constant parts excluded: see axes_offset)."""
    digs = []
    for a, e in enumerate(axes):
        if e is None or buf.shape[a] <= 1 or (buf.strides[a] == 0 and not (buf.subaxes and a in buf.subaxes)):
            continue
        for src, div, mod, stride in _axis_parts(buf, a, e)[0]:
            digs.append([src, div, mod, stride])
    digs.sort(key=lambda d: (d[0], d[1], d[2] or 0))
    same = []
    for d in digs:  # the same digit on two axes: one digit with the summed stride
        if same and same[-1][:3] == d[:3]:
            same[-1][3] += d[3]
        else:
            same.append(d)
    digs = [d for d in same if d[3] != 0]
    merged = []
    for d in digs:
        if merged:
            lo = merged[-1]
            if lo[0] == d[0] and lo[2] is not None and d[1] == lo[1] * lo[2] and d[3] == lo[3] * lo[2]:
                lo[2] = None if d[2] is None else lo[2] * d[2]
                continue
        merged.append(d)
    out = []
    for src, div, mod, stride in merged:
        if mod is not None and div * mod >= extents[src]:
            mod = None
        out.append((src, div, mod, stride))
    return out


def vec_width(et: ElementType) -> int:
    """Elements per thread-vector in the VM kernel (32 bytes, or 8 for BOOL)."""
    return 4 if et.byte_size == 8 else 8


def vec_class(digits, vec_src: int, is_store: bool, V: int, esize: int) -> int:
    """0 gather, 1 contiguous (vector access), 2 uniform (one value per vector).

    Vectors are V consecutive indices of `vec_src` starting at a multiple of
    V; contiguous access also needs the base element offset aligned to the
    16-byte (8-byte for BOOL) memory transaction.
    """
    align = max(1, (8 if esize == 1 else 16) // esize)
    own = [d for d in digits if d[0] == vec_src]
    unit = [d for d in own if d[1] == 1]
    if not any(d[1] % V for d in own if d[1] != 1):
        if not unit:
            return 0 if is_store else 2
        if len(unit) == 1:
            _, _, mod, stride = unit[0]
            if stride == 1 and (mod is None or mod % V == 0) and not any(d[3] % align for d in digits if d is not unit[0]):
                return 1
    return 3 if vec_pattern(digits, vec_src, V) is not None else 0


def vec_pattern(digits, vec_src: int, V: int):
    """Per-element offsets inside a V-aligned vector when they do not depend
    on the vector's position: digits with div % V == 0 are constant across
    it, digits with V % div == 0 and (div*mod) % V == 0 advance by
    (v // div) * stride without wrapping.  None when neither holds."""
    dv = [0] * V
    for src, div, mod, stride in digits:
        if src != vec_src:
            continue
        if div % V == 0:
            continue
        if V % div or (mod is not None and (div * mod) % V):
            return None
        for v in range(V):
            dv[v] += (v // div) * stride
    if max(abs(x) for x in dv) >= 2 ** 30:
        return None
    return dv


def r_linear(digits) -> int:
    """Stride of the r-part when it is one linear digit, 0 without r, -1 otherwise."""
    rd = [d for d in digits if d[0] == 1]
    if not rd:
        return 0
    if len(rd) == 1 and rd[0][1] == 1 and rd[0][2] is None:
        return rd[0][3]
    return -1


def split_axes(shape, inner_from: int) -> list:
    """Axis expressions with axes < inner_from on o (src 0), the rest on r (src 1)."""
    out = []
    for a, d in enumerate(shape):
        if d == 1:
            out.append(None)
        elif a < inner_from:
            out.append((0, _prod(shape[a + 1:inner_from]), d))
        else:
            out.append((1, _prod(shape[a + 1:]), d))
    return out


# ---------------------------------------------------------------------------
# Lowered plan


@dataclass
class LaunchRec:
    kind: int
    grid: tuple
    block: tuple
    smem: int
    args: C.Structure
    reads: list  # buffer keys read
    writes: list  # buffer keys written
    label: str = ""
    algo_bytes: int = 0  # algorithmic HBM bytes (roofline accounting)
    flops: int = 0


@dataclass
class Lowered:
    launches: list
    arena_bytes: int
    const_blob: bytes
    n_inputs: int
    n_outputs: int
    buffers: dict
    groups: list = field(default_factory=list)
    arena_offsets: dict = field(default_factory=dict)
    channels_last: bool = False

    def pack(self):
        """(launch array, argument blob) ready for gfb_exe_create."""
        recs = (abi.Launch * max(1, len(self.launches)))()
        blob = bytearray()
        for i, L in enumerate(self.launches):
            raw = bytes(L.args)
            off = align_up(len(blob), 64)  # tensor maps inside TcArgs need 64 B
            blob.extend(b"\0" * (off - len(blob)))
            blob.extend(raw)
            r = recs[i]
            r.kind = L.kind
            r.grid[:] = list(L.grid)
            r.block[:] = list(L.block)
            r.smem = L.smem
            r.arg_offset = off
            r.arg_size = len(raw)
        return recs, bytes(blob)


class _DropRowGroup(Exception):
    """A row group turned out not to be expressible: lower without it."""

    def __init__(self, group):
        self.group = group


class _Retry(Exception):
    def __init__(self, nid):
        self.nid = nid


class _Node:
    """IR node plus the shape of its first input (for Reshape inversion)."""

    __slots__ = ("id", "op", "attrs", "inputs", "output", "inputs_shape")

    def __init__(self, node, g):
        self.id, self.op, self.attrs, self.inputs, self.output = node.id, node.op, node.attrs, node.inputs, node.output
        self.inputs_shape = g.nodes[node.inputs[0][0]].output.shape if node.inputs else ()


# ---------------------------------------------------------------------------


class Lowering:
    def __init__(self, g: Function, layouts: dict, private: bool = False, allreduce=frozenset(),
                 channels_last: bool = False, allreduce_max=frozenset()):
        self.g = g
        self.layouts = layouts
        self.private = private
        self.allreduce = set(allreduce)  # data-parallel partial roots (dp.analyse)
        self.allreduce_max = set(allreduce_max)  # the roots reduced with max (a max over the batch shard)
        self.order = [n for n in topological_order(g) if n in reachable_from_results(g)]
        self.topo = {n: i for i, n in enumerate(self.order)}
        self.nodes = {n: _Node(g.nodes[n], g) for n in self.order}
        self.consumers: dict = {n: [] for n in self.order}
        for n in self.order:
            for r, _ in g.nodes[n].inputs:
                if n not in self.consumers[r]:
                    self.consumers[r].append(n)
        self.param_pos = {pid: i for i, pid in enumerate(g.parameters)}
        # Dots with a tiny contraction (the pool composite's one-hot selections
        # [1,4]x[4,M] and their [4,1]x[1,M] gradients) are elementwise work:
        # they fuse into VM programs as exact-order multiply-add chains.
        self.tiny = {n for n in self.order if g.nodes[n].op is OpKind.DOT and g.nodes[n].output.element_type.is_float
                     and g.nodes[g.nodes[n].inputs[0][0]].output.shape[1] <= TINY_DOT_K}
        # NHWC layout policy in force: 4-D intermediates are stored channel-last
        self.channels_last = channels_last
        self.buf: dict = {}
        self.n_in = len(g.parameters)
        self.n_out = len(g.results)
        self._key = 0

    # -- helpers
    def new_key(self) -> int:
        self._key += 1
        return self._key

    def is_light(self, n) -> bool:
        op = self.nodes[n].op
        return (op in ELEMENTWISE_BINARY or op in ELEMENTWISE_UNARY or op in INDEX_OPS or op is OpKind.SUM
                or n in self.tiny)

    def is_heavy(self, n) -> bool:
        return self.nodes[n].op in HEAVY and n not in self.tiny

    def strides_of(self, n) -> tuple:
        return self.layouts[(n, 0)].strides(self.nodes[n].output.shape)

    # -- materialisation policy
    def initial_materialised(self) -> set:
        M = self.M = set()
        results = {r for r, _ in self.g.results}
        for n in self.order:
            node = self.nodes[n]
            if not self.is_light(n):
                continue
            if node.op is OpKind.SUM or n in results or n in self.allreduce:
                M.add(n)
                continue
            if (self.channels_last and node.op is OpKind.RESHAPE and len(node.output.shape) == 4
                    and len(node.inputs_shape) != 4 and os.environ.get("GFB_RELAYOUT", "1") == "1"):
                # a rank-changing Reshape back to 4-D (the pool composite's window
                # merge) is where NCHW-ordered flat data meets channel-last
                # storage: one transposing map writes it channel-last, instead
                # of every consumer gathering across the layouts
                M.add(n)
                continue
            cons = self.consumers[n]
            heavy = [c for c in cons if self.is_heavy(c)]
            light = [c for c in cons if c not in heavy]
            if heavy and not self.viewable(n):
                M.add(n)
                continue
            if len(light) >= 2 and not self.free_view(n):
                M.add(n)
        return M

    def is_source(self, n) -> bool:
        """Materialised already: parameter, constant, heavy output or member of M."""
        op = self.nodes[n].op
        return op in (OpKind.PARAMETER, OpKind.CONSTANT) or self.is_heavy(n) or n in self.M

    def free_view(self, n) -> bool:
        """Index ops over materialised sources cost nothing to recompute."""
        node = self.nodes[n]
        while node.op in INDEX_OPS and node.id not in self.M:
            node = self.nodes[node.inputs[0][0]]
        return self.is_source(node.id)

    def viewable(self, n) -> bool:
        try:
            return self.heavy_operand(n, probe=True) is not None
        except Unexpressible:
            return False

    # -- heavy operands: (buffer, strides per logical axis)
    def heavy_operand(self, n, probe=False):
        node = self.nodes[n]
        if n in self.buf:
            b = self.buf[n]
            return b, b.strides
        if probe and self.is_source(n):
            return True, None
        if node.op is OpKind.CONVERT_LAYOUT:
            return self.heavy_operand(node.inputs[0][0], probe)
        if node.op is OpKind.RESHAPE:
            src = node.inputs[0][0]
            inner = self.heavy_operand(src, probe)
            if inner is None:
                return None
            order = node.attrs["input_order"]
            in_shape = node.inputs_shape
            perm = tuple(in_shape[a] for a in order)
            if perm == tuple(node.output.shape):
                if probe:
                    return True, None
                b, st = inner
                return b, tuple(st[a] for a in order)
            if order == tuple(range(len(order))):
                # row-major re-read of a contiguous identity-order operand
                if probe:
                    return (True, None) if self.is_source(src) else None
                b, st = inner
                if _dense_rowmajor(in_shape, st):
                    return b, _rowmajor(node.output.shape)
            return None
        return None

    # -- main entry
    def run(self) -> Lowered:
        self._topo_order = list(self.order)
        self.M = set()
        self.initial_materialised()
        self.row_groups = []
        from . import rowfuse

        if rowfuse.enabled():
            self.row_groups = rowfuse.find_groups(self)
        self._apply_row_groups()
        for _ in range(1000):
            try:
                return self._lower()
            except _Retry as r:
                g = self._row_of.get(r.nid)
                if g is not None:  # a member someone must read from memory: store it too
                    if r.nid in g.outputs:
                        raise UnsupportedOp(f"cannot lower node {r.nid} ({self.nodes[r.nid].op.wire_name})")
                    g.outputs.append(r.nid)
                    self.M.add(r.nid)
                    continue
                if r.nid in self.M:
                    raise UnsupportedOp(f"cannot lower node {r.nid} ({self.nodes[r.nid].op.wire_name})")
                self.M.add(r.nid)
            except _DropRowGroup as d:
                self.row_groups.remove(d.group)
                self.M = set()
                self.initial_materialised()
                self._apply_row_groups()
        raise UnsupportedOp("lowering did not converge")

    def _apply_row_groups(self):
        """Materialisation and order for the row-fused groups (rowfuse.py):
        internal members live in registers, outputs and forced inputs in
        memory, and each group's members become contiguous in the order."""
        from . import rowfuse

        self._row_of, self._row_nodes = {}, set()
        for g in self.row_groups:
            for m in g.members:
                self._row_of[m] = g
                if m not in g.outputs:
                    self.M.discard(m)
            self.M.update(g.outputs)
            self.M.update(g.force)
            self._row_nodes |= set(g.members)
        self.order = rowfuse.reorder(self._topo_order, self.consumers, lambda n: [r for r, _ in self.nodes[n].inputs],
                                     self.row_groups) if self.row_groups else list(self._topo_order)
        self.topo = {n: i for i, n in enumerate(self.order)}

    def _lower(self) -> Lowered:
        g = self.g
        self.buf: dict = {}
        self.launches: list = []
        self.const_values: dict = {}  # small constants' row-major values, by buffer key
        self._splats: dict = {}
        self._pads: dict = {}  # channel-padded channel-last copies of conv inputs
        self._window_factors = None
        const_blob = bytearray()
        results = list(g.results)
        result_slot = {}  # node -> output index written directly by its producer
        for j, (r, _) in enumerate(results):
            node = self.nodes[r]
            # all-reduced roots need a fixed (arena) address inside the CUDA graph
            if node.op not in (OpKind.PARAMETER, OpKind.CONSTANT) and r not in result_slot and r not in self.allreduce:
                result_slot[r] = j

        self._csum_done = set()
        self._f16_chunks = {}   # caller input key -> its row chunks' plane views (_f16_planes)
        self._row_chunked = {}  # tensor key -> row chunks its fp16 planes were written in (chunked epilogues)
        self._epi_planes = set()  # tensors whose fp16 planes a GEMM epilogue writes
        self._epi = self._plan_epilogues()
        self._epi_nodes = {m for sp in self._epi.values() for m in sp["absorbed"]}
        self._conv_relu = self._plan_conv_relu()  # stem conv -> the Relu its epilogue writes
        self._conv_relu_done = set()
        self._epi_nodes |= set(self._conv_relu.values())
        for n in self.order:
            node = self.nodes[n]
            d = node.output
            if n in self._epi:
                continue  # a Dot whose consumer map runs in its epilogue: never materialised
            if element_count(d.shape) >= INDEX_LIMIT:
                raise UnsupportedOp(f"tensor of {element_count(d.shape)} elements exceeds the 2^31 index limit")
            if node.op is OpKind.PARAMETER:
                self.buf[n] = Buffer(self.new_key(), d.element_type, d.shape, self.strides_of(n), abi.SLOT_IO + self.param_pos[n])
            elif node.op is OpKind.CONSTANT:
                data: ConstantData = node.attrs["data"]
                b = Buffer(self.new_key(), d.element_type, d.shape, _rowmajor(d.shape), abi.SLOT_CONST)
                if data.is_splat and self._splat_ok(n):
                    b.splat = data.splat_value()
                else:
                    if element_count(d.shape) <= 4096:
                        self.const_values[b.key] = np.ascontiguousarray(data.to_numpy()).reshape(-1)
                    off = align_up(len(const_blob), DEVICE_ALIGNMENT)
                    const_blob.extend(b"\0" * (off - len(const_blob)))
                    const_blob.extend(np.ascontiguousarray(data.to_numpy()).tobytes())
                    b.offset = off
                self.buf[n] = b
            elif n in self.M or self.is_heavy(n):
                slot = abi.SLOT_ARENA
                strides = self.strides_of(n)
                if n in result_slot:
                    slot = abi.SLOT_IO + self.n_in + result_slot[n]
                elif self.channels_last and len(d.shape) == 4 and node.op is not OpKind.CONV_BACKPROP_FILTER:
                    # intermediates are stored channel-last under the NHWC policy: every
                    # kernel reads through strides, and the convolutions' gathers then
                    # find 32-channel runs contiguous (gfb_conv_tcg_kernel)
                    strides = Layout(NHWC_ORDER).strides(d.shape)
                subaxes = self._flat_channel_last(n) if slot == abi.SLOT_ARENA else None
                if subaxes is not None:
                    strides = (d.shape[1], 1)
                self.buf[n] = Buffer(self.new_key(), d.element_type, d.shape, strides, slot, subaxes=subaxes)

        self._grad_regions = self._gradient_regions() if self.allreduce else []

        # merge rule: a materialised node consumed only by one Sum is that Sum's side output
        side_of = {}
        for n in self.order:
            if (n in self.M and self.nodes[n].op is not OpKind.SUM and self.is_light(n) and n not in self._row_nodes
                    and n not in self._epi_nodes):
                cons = self.consumers[n]
                if len(cons) == 1 and self.nodes[cons[0]].op is OpKind.SUM and cons[0] not in self._row_nodes:
                    side_of[cons[0]] = n
        merged = set(side_of.values())

        groups = self._sibling_groups(merged)
        grouped = {m for g in groups.values() for m in g[1:]}
        self._map_side = self._chains(merged | grouped | set(groups))
        chained = set(self._map_side.values())
        for n in self.order:
            node = self.nodes[n]
            rg = self._row_of.get(n)
            if rg is not None:
                if n == rg.anchor:
                    self.emit_row_group(rg)
                continue
            if n in self._epi_nodes or n in self._csum_done:
                continue  # written by the epilogue of the Dot it consumes (or reduced from its partials)
            if self.is_heavy(n):
                self.emit_heavy(n)
            elif n in self.M and n not in merged and n not in grouped and n not in chained:
                if node.op is OpKind.SUM:
                    self.emit_reduce(n, side_of.get(n))
                else:
                    self.emit_map(n, groups.get(n, [n]))

        if self.allreduce:
            self._bucket_allreduces()
        self._interleave_row_chunks()
        self._hoist_result_writers()

        # results that are parameters / constants / repeated: copy launches
        for j, (r, _) in enumerate(results):
            if result_slot.get(r) == j:
                continue
            src = self.buf[r]
            d = self.nodes[r].output
            dst = Buffer(self.new_key(), d.element_type, d.shape, _rowmajor(d.shape), abi.SLOT_IO + self.n_in + j)
            self.emit_copy(src, dst)

        for chunks in self._f16_chunks.values():
            for ch in chunks:
                if ch[5] is not None:
                    raise UnsupportedOp("a row-chunked fp16 split was never consumed")
        dropped = self._drop_unread_epilogue_outputs()

        # arena plan over launch-index live ranges
        live: dict = {}
        view_base = {b.key: b.base.key for b in self.buf.values() if b.exact and b.base is not None}
        for i, L in enumerate(self.launches):
            for k0 in L.writes + L.reads:
                for k in (k0, view_base.get(k0)):  # a row view keeps its base alive
                    if k is None:
                        continue
                    lo, hi = live.get(k, (i, i))
                    live[k] = (min(lo, i), max(hi, i))
        arena_bufs = {b.key: b for b in self.buf.values() if b.slot == abi.SLOT_ARENA and b.base is None
                      and b.key not in dropped}
        items = {k: (b.nbytes, live.get(k, (0, 0))[0], live.get(k, (0, 0))[1]) for k, b in arena_bufs.items()}
        for region, members in self._grad_regions:
            # the gradient region lives from its first member's producer to its last reader
            spans = [live[m.key] for m in members if m.key in live] or [(0, 0)]
            arena_bufs[region.key] = region
            items[region.key] = (region.nbytes, min(a for a, _ in spans), max(b for _, b in spans))
        plan = plan_buffers(items, private=self.private)
        for k, b in arena_bufs.items():
            b.offset = plan.offsets[k]
        for L in self.launches:
            L.finalize()
        buffers = {b.key: b for b in self.buf.values()}
        for region, _ in self._grad_regions:
            buffers[region.key] = region
        return Lowered(self.launches, plan.arena_size, bytes(const_blob), self.n_in, self.n_out,
                       buffers, arena_offsets=plan.offsets)

    def _interleave_row_chunks(self):
        """Chunk-major order for the row-chunked launches (a large input's
        split chunks and the GEMMs of every layer that follows them): chunk
        c's path through all the layers runs as soon as its input piece has
        arrived, while the later pieces cross PCIe.  A list schedule over the
        span from the first to the last chunk launch: each step places the
        ready launch of the smallest chunk index (a launch without one takes
        the smallest chunk index of the chunk launches that depend on it)."""
        idx = [i for i, L in enumerate(self.launches) if getattr(L, "row_chunk", None) is not None]
        if not idx or os.environ.get("GFB_CHUNK_MAJOR", "1") != "1":
            return
        lo, hi = idx[0], idx[-1] + 1
        span = self.launches[lo:hi]
        by_key = {b.key: b for b in self.buf.values()}

        def extents(keys, write):
            out = []
            for k in keys:
                b = by_key.get(k)
                if b is None:
                    out.append((("?", k), 0, 1 << 62, write))
                elif b.exact and b.base is not None:
                    a0 = b.elem_off * b.et.byte_size
                    out.append((b.base.key, a0, a0 + b.nbytes, write))
                else:
                    root = b.base if b.base is not None else b
                    out.append((root.key, 0, 1 << 62, write))
            return out

        acc = [extents(L.reads, False) + extents(L.writes, True) for L in span]

        def conflict(a, b):
            return any((wa or wb) and ka == kb and la < hb and lb < ha for ka, la, ha, wa in a for kb, lb, hb, wb in b)

        n = len(span)
        deps = [[j for j in range(i) if conflict(acc[i], acc[j])] for i in range(n)]
        key = [getattr(L, "row_chunk", None) for L in span]
        users = [[] for _ in range(n)]
        for i in range(n):
            for j in deps[i]:
                users[j].append(i)
        for i in range(n - 1, -1, -1):  # a launch takes the earliest chunk that needs it
            if key[i] is None:
                ks = [key[u] for u in users[i] if key[u] is not None]
                key[i] = min(ks) if ks else 1 << 30
        placed, order = [False] * n, []
        for _ in range(n):
            ready = [i for i in range(n) if not placed[i] and all(placed[j] for j in deps[i])]
            i = min(ready, key=lambda t: (key[t], t))
            placed[i] = True
            order.append(i)
        self.launches[lo:hi] = [span[i] for i in order]

    def _hoist_result_writers(self):
        """Move each launch that writes a caller result (the optimizer
        updates of a training step, which the graph orders last) to just
        after the last launch it depends on.  Host-buffer runs copy a result
        back right after its writer, so config E's new weights then cross
        PCIe under the rest of the backward pass instead of after it."""
        if os.environ.get("GFB_HOIST_RESULTS", "1") != "1":
            return
        root_of = {b.key: (b.base.key if b.exact and b.base is not None else b.key) for b in self.buf.values()}
        res_lo = abi.SLOT_IO + self.n_in
        out_keys = {b.key for b in self.buf.values() if b.base is None and b.slot >= res_lo}

        def acc(L):
            r = {root_of.get(k, k) for k in L.reads}
            w = {root_of.get(k, k) for k in L.writes}
            return r, w

        out, accs = [], []
        for L in self.launches:
            r, w = acc(L)
            pos = len(out)
            if (L.kind != abi.K_ALLREDUCE and getattr(L, "chain", None) is None and w & out_keys
                    and not any(k is None for k in w)):
                pos = 0
                for idx in range(len(out) - 1, -1, -1):
                    r2, w2 = accs[idx]
                    if (r & w2) or (w & (r2 | w2)) or out[idx].kind == abi.K_ALLREDUCE:
                        pos = idx + 1
                        break
            out.insert(pos, L)
            accs.insert(pos, (r, w))
        self.launches = out

    def _drop_unread_epilogue_outputs(self) -> set:
        """fp16 GEMM epilogues store the fp32 tensors of the maps they absorb
        (the pre-activation C, the Relu output); when no launch reads one --
        its consumers take the fp16 planes and the mask bytes instead -- the
        store is dropped and the tensor gets no arena space.  Returns the
        dropped buffer keys."""
        base_of = {b.key: (b.base if b.exact and b.base is not None else b) for b in self.buf.values()}
        read = set()
        for L in self.launches:
            for k in L.reads:
                read.add(k)
                if k in base_of:
                    read.add(base_of[k].key)  # a row view read reads its base
        dropped = set()

        def unread(b):  # an arena tensor (or a row view of one) nobody reads
            if b is None:
                return None
            root = b.base if b.exact and b.base is not None else b
            if root.slot != abi.SLOT_ARENA or root.base is not None or root.key in read or b.key in read:
                return None
            return root

        for L in self.launches:
            if L.kind != abi.K_DOT_F16P or not L.args.epi_kind:
                continue
            a, bufs = L.args, L.epi_bufs
            r2 = unread(bufs.get("out2")) if a.epi_flags & 1 else None
            if r2 is not None:
                a.epi_flags &= ~1
                L.writes.remove(bufs["out2"].key)
                dropped.add(r2.key)
            rc = unread(bufs["c"]) if a.epi_flags & (4 | 8) else None
            if rc is not None and rc.key not in self._region_keys():
                a.epi_flags |= 32
                L.writes.remove(bufs["c"].key)
                dropped.add(rc.key)
        return dropped

    def _region_keys(self) -> set:
        return {m.key for _, members in self._grad_regions for m in members}

    def _flat_channel_last(self, n):
        """Sub-axis storage for a flattened pool-window matrix [k, M] under the
        NHWC policy: M enumerates (n, c, h2, w2) (the composite's window
        Reshape); stored as (n, h2, w2, c) it lines up with the channel-last
        activations it is computed from and scattered back to, so neither
        side transposes.  Only for matrices read exclusively by fused maps
        (every access goes through index maps, never raw strides)."""
        if not self.channels_last or os.environ.get("GFB_SUBAXES", "1") != "1":
            return None
        node = self.nodes[n]
        shape = node.output.shape
        if len(shape) != 2 or self.is_heavy(n) or n in self.allreduce:
            return None
        if getattr(self, "_window_factors", None) is None:
            wf = {}
            for x in self.order:
                nd = self.nodes[x]
                if nd.op is not OpKind.RESHAPE:
                    continue
                for shp in (tuple(nd.output.shape), tuple(nd.inputs_shape)):
                    if len(shp) == 6 and shp[3] == 2 and shp[5] == 2:  # (n, c, h2, 2, w2, 2)
                        wf[shp[0] * shp[1] * shp[2] * shp[4]] = (shp[0], shp[1], shp[2], shp[4])
                    if len(shp) == 6 and shp[0] == 2 and shp[1] == 2:  # (2, 2, n, c, h2, w2)
                        wf[shp[2] * shp[3] * shp[4] * shp[5]] = shp[2:]
            self._window_factors = wf
        f = self._window_factors.get(shape[1])
        if f is None or f[1] == 1:
            return None
        stack, seen = [n], {n}
        while stack:  # every reader is a fused map (possibly through index ops)
            x = stack.pop()
            for c in self.consumers[x]:
                if not self.is_light(c) or c in seen:
                    if not self.is_light(c):
                        return None
                    continue
                if self.nodes[c].op in INDEX_OPS:
                    seen.add(c)
                    stack.append(c)
        N_, C_, H2, W2 = f
        return {1: [(N_, H2 * W2 * C_), (C_, 1), (H2, W2 * C_), (W2, C_)]}

    def splat_buffer(self, et: ElementType, value) -> Buffer:
        """A memory-less scalar operand (one per distinct bit pattern)."""
        v = value.item() if hasattr(value, "item") else value
        key = (et, struct.pack("<d", float(v)) if et.is_float else int(v))
        if key not in self._splats:
            self._splats[key] = Buffer(self.new_key(), et, (), (), abi.SLOT_CONST, 0, v)
        return self._splats[key]

    def _splat_ok(self, n) -> bool:
        """Splat constants stay scalars unless a heavy op or a result reads memory."""
        results = {r for r, _ in self.g.results}
        if n in results:
            return False
        for c in self.consumers[n]:
            if self.is_heavy(c):
                return False
            # an index view feeding a heavy op also needs memory
            if self.nodes[c].op in INDEX_OPS and any(self.is_heavy(cc) for cc in self.consumers[c]):
                return False
        return True

    # -- fused VM groups
    def _row_launch(self, prog, n_o, n_r, red_kind, label, et):
        """ROW: warps per o, vectors along r; more warps per o when o is short.

        Programs whose memory operands are all row-contiguous (or constant
        along the row) take the staged kernel: cp.async.bulk double-buffered
        shared-memory stages, one dispatch per 16 elements per thread."""
        V = vec_width(et)
        staged = self._staged_ok(prog, n_o, n_r, et)
        wpr = 1
        while not staged and wpr < 8 and n_o * wpr < ROW_BLOCKS_PER_SM * NUM_SMS * 8 and n_r >= 32 * V * wpr * 2:
            wpr *= 2
        rpb = 8 // wpr
        if staged:
            chunk = 32 * 2 * (16 // et.byte_size) * 2  # csrc/ew_vm.cu StagedCfg<T, 2>
            nch = (n_r + chunk - 1) // chunk
            stages, wpb = 2, 8  # ring depth, warps per block (swept: scripts/sweep_staged.sh)
            n_r_pad = nch * chunk
            lin = [l for l in prog.leaf_specs if not l.is_store and l.buf.splat is None and r_linear(l.digits) == 1]
            resident = [l for l in lin if all(d[0] == 1 for d in l.digits) and n_r_pad * et.byte_size <= 8192]
            nstaged = max(1, len(lin) - len(resident))
            smem = len(resident) * n_r_pad * et.byte_size + wpb * stages * nstaged * chunk * et.byte_size
            per_sm = max(1, min(8, (220 * 1024) // max(smem, 1)))
            slots = NUM_SMS * per_sm * wpb  # resident warps
            chunkwise = n_o < slots and nch > 1
            partial = None
            if chunkwise and red_kind:
                # few long rows: per-chunk partials, then a short second pass
                partial = Buffer(self.new_key(), et, (n_o, nch), (nch, 1))
                self.buf[("partial", partial.key)] = partial
                final = prog.red_out
                prog.red_out = LeafSpec(partial, [(0, 1, None, 1)], True, 0)
            args = prog.args(mode=3, n_o=n_o, n_r=n_r, red_kind=red_kind, split=1 if chunkwise else 0, wpr=stages)
            items = n_o * nch if chunkwise else n_o
            grid = max(1, min((items + wpb - 1) // wpb, NUM_SMS * per_sm))
            kind = abi.K_EWS_F32 if et is ElementType.F32 else abi.K_EWS_F64
            self.add_launch(kind, (grid, 1, 1), (32 * wpb, 1, 1), smem, args, prog,
                            label + (":staged2" if chunkwise else ":staged"))
            if partial is not None:
                # second pass over the partials: rows again when they are long
                row2 = nch >= 4096
                p2 = Program(self, extents=(n_o, nch), vec_src=1 if row2 else 0, et=et)
                k = p2.leaf(partial, [(0, 1, n_o), (1, 1, nch)] if n_o > 1 else [None, (1, 1, nch)])
                p2.emit(I_LOAD, k=k)
                p2.red_out = LeafSpec(final.buf, final.digits, True, vec_class(final.digits, 0, True, vec_width(et), et.byte_size))
                if row2:
                    self._row_launch(p2, n_o, nch, red_kind, label + ":pass2", et)
                else:
                    self._col_launch(p2, n_o, nch, red_kind, label + ":pass2", et)
            return
        scalar = self._scalar_ok(prog, n_o, n_r, et)
        if scalar:
            prog.set_vector_width(1)
        grid = max(1, min((n_o + rpb - 1) // rpb, NUM_SMS * EW_BLOCKS_PER_SM))
        args = prog.args(mode=1, n_o=n_o, n_r=n_r, red_kind=red_kind, wpr=wpr)
        general_r = [l.digits for l in prog.leaf_specs if l.buf.splat is None and r_linear(l.digits) < 0]
        if len(general_r) >= 2 and len(set(map(tuple, general_r))) < len(general_r):
            args.pad = 1  # cache_r: leaves sharing an r map compute it once per vector
            ty = _transpose_order(prog, n_r, vec_width(et), src=1)
            if ty is not None:
                args.ty_ext, args.ty_div = ty
                label += ":T"
        kind = EW1_KIND[et] if scalar else EW_KIND[et]
        self.add_launch(kind, (grid, 1, 1), (256, 1, 1), prog.smem_bytes(args), args, prog, label + (":s" if scalar else ""))

    def _staged_ok(self, prog, n_o, n_r, et) -> bool:
        # With runtime specialisation (jit.py) a generated ROW kernel beats the
        # staged interpreter on every measured workload (B, A, C, D); the
        # staged kernel keeps the few-long-rows case, where its chunk-wise
        # split fills the GPU and warps-per-row cannot.
        policy = _staged_policy()
        if et not in (ElementType.F32, ElementType.F64) or n_r < 256 or policy == "0":
            return False
        if policy == "auto" and not (n_o < 2 * NUM_SMS and n_r >= 4096):
            return False
        es = et.byte_size
        if (n_r * es) % 16:
            return False
        if any(c[0] in (I_PUSH, I_PUSH_LOAD, I_BIN_POP, I_DOT) for c in prog.code):
            return False
        if sum(1 for l in prog.leaf_specs if not l.is_store) > MAX_PRELOAD:
            return False  # every operand must be a preloaded leaf
        loads = [l for l in prog.leaf_specs if not l.is_store and l.buf.splat is None]
        def o_aligned(l):
            return all((d[3] * es) % 16 == 0 for d in l.digits if d[0] == 0)
        for l in loads:
            rl = r_linear(l.digits)
            if rl == 1:
                if not o_aligned(l):
                    return False
            elif rl != 0 or any(d[0] == 1 for d in l.digits):
                return False
        for l in prog.leaf_specs:
            if l.is_store and r_linear(l.digits) == 1 and not o_aligned(l):
                return False
        return True

    @staticmethod
    def _scalar_ok(prog, n_o, n_r, et) -> bool:
        """Small launches are latency-bound: one element per thread (8x the
        threads of the vector kernel for the same work)."""
        return (et in (ElementType.F32, ElementType.F64) and n_o * n_r <= SCALAR_VM_MAX
                and os.environ.get("GFB_SCALAR_VM", "1") == "1")

    def _col_launch(self, prog, n_o, n_r, red_kind, label, et):
        """COL: one thread per V-vector of o, r looped (split when o is short)."""
        scalar = self._scalar_ok(prog, n_o, n_r, et)
        if scalar:
            prog.set_vector_width(1)
        V = prog.V
        vectors = (n_o + V - 1) // V
        split = 1
        if red_kind and n_r > 16:
            while split < 256 and ((vectors * split + 255) // 256) < 3 * NUM_SMS and n_r // (split * 2) >= 8:
                split *= 2
        per_row = 256 // split
        grid = max(1, min((vectors + per_row - 1) // per_row, NUM_SMS * EW_BLOCKS_PER_SM))
        args = prog.args(mode=2, n_o=n_o, n_r=n_r, red_kind=red_kind, split=split)
        if red_kind == 0 and split == 1 and n_r == 1 and not scalar:
            ty = _transpose_order(prog, n_o, V)
            if ty is not None:
                args.ty_ext, args.ty_div = ty
                label += ":T"
        kind = EW1_KIND[et] if scalar else EW_KIND[et]
        self.add_launch(kind, (grid, 1, 1), (256, 1, 1), prog.smem_bytes(args), args, prog, label + (":s" if scalar else ""))

    def _chains(self, taken) -> dict:
        """consumer -> producer: a materialised map whose first consumer is an
        elementwise map over the same storage is written as a side output of
        that consumer's launch (e.g. E's bias Add and the ReLU after it: the
        pre-activation is still stored for the backward pass, but read once
        less and one launch fewer)."""
        if os.environ.get("GFB_CHAINS", "1") != "1":
            return {}
        pos = {n: i for i, n in enumerate(self.order)}
        out, used = {}, set()
        for n in self.order:
            if (n not in self.M or n in taken or n in used or n in self.allreduce or not self.is_light(n)
                    or self.nodes[n].op is OpKind.SUM or n not in self.buf or n in self._row_nodes or n in self._epi_nodes):
                continue
            cons = sorted(set(self.consumers[n]), key=lambda c: pos.get(c, 1 << 30))
            if not cons:
                continue
            c = cons[0]
            if (c in taken or c in out or c in used or c not in self.M or not self.is_light(c) or c in self.allreduce
                    or c in self._row_nodes or c in self._epi_nodes
                    or self.nodes[c].op is OpKind.SUM or self.nodes[c].op in INDEX_OPS or c not in self.buf
                    or pos.get(c) is None):
                continue
            bn, bc = self.buf[n], self.buf[c]
            if (bn.shape != bc.shape or bn.et != bc.et or bn.strides != bc.strides or bn.subaxes != bc.subaxes
                    or bn.splat is not None or bc.splat is not None):
                continue
            out[c] = n
            used |= {n, c}
        return out

    def _sibling_groups(self, merged) -> dict:
        """Materialised maps over the same iteration space whose inputs are
        ready when the first of them is emitted run as one launch with several
        stores (e.g. the pool composite's four one-hot selections of one
        window tensor: the window is read once instead of four times)."""
        if os.environ.get("GFB_SIBLINGS", "1") != "1":
            return {}
        pos = {n: i for i, n in enumerate(self.order)}

        def sources(n):  # nearest materialised inputs of n's fused expression
            out, stack, seen = set(), [r for r, _ in self.g.nodes[n].inputs], set()
            while stack:
                x = stack.pop()
                if x in seen:
                    continue
                seen.add(x)
                if self.is_source(x):
                    out.add(x)
                else:
                    stack += [r for r, _ in self.g.nodes[x].inputs]
            return out

        cands = [n for n in self.order if n in self.M and n not in merged and self.is_light(n) and n not in self._row_nodes
                 and n not in self._epi_nodes
                 and self.nodes[n].op is not OpKind.SUM and n in self.buf and self.buf[n].slot == abi.SLOT_ARENA]
        groups, taken = {}, set()
        for i, n in enumerate(cands):
            if n in taken:
                continue
            b0 = self.buf[n]
            src0 = sources(n)
            g = [n]
            for m in cands[i + 1:]:
                if m in taken or len(g) >= 4:
                    continue
                bm = self.buf[m]
                if (bm.shape != b0.shape or bm.et != b0.et or bm.strides != b0.strides or bm.subaxes != b0.subaxes):
                    continue
                sm = sources(m)
                # ready at n's position, and sharing an input (the point of fusing)
                if any(pos[x] > pos[n] for x in sm if x in pos and x not in (n,)) or not (sm & src0):
                    continue
                if any(x in sm for x in g):
                    continue
                g.append(m)
            if len(g) > 1:
                groups[n] = g
                taken.update(g)
        return groups

    def emit_map(self, root: int, stores: list):
        if len(stores) > 1:
            mark = len(self.launches)
            try:
                self._emit_group(stores)
                return
            except (_Retry, UnsupportedOp, Unexpressible):
                del self.launches[mark:]
            for m in stores:  # too big together: one launch each
                self.emit_map(m, [m])
            return
        node = self.nodes[root]
        shape = tuple(node.output.shape)
        et = node.output.element_type
        total = element_count(shape)
        if total == 0:
            return
        # Iterate in the output's storage order so stores coalesce (channel-last
        # intermediates); fall back to logical order when an index op on the
        # way down cannot follow the permuted digits.
        buf = self.buf[root]
        if buf.subaxes:
            # flattened axes stored permuted: iterate their sub-digits in storage order
            cand = []
            for a, d in enumerate(shape):
                if a in buf.subaxes:
                    sub = buf.subaxes[a]
                    for i, (x, st) in enumerate(sub):
                        cand.append((st, a, _prod(x2 for x2, _ in sub[i + 1:]), x))
                else:
                    cand.append((buf.strides[a], a, 1, d))
            dims = [(a, mul, x) for _, a, mul, x in sorted(cand, key=lambda t: -t[0])]
        else:
            dims = [(a, 1, shape[a]) for a in _storage_perm(buf)]
        if [d[0] for d in dims] != list(range(len(shape))) or any(d[1] != 1 for d in dims):
            mark = len(self.launches)
            try:
                self._emit_map_in(root, shape, dims, et, total, node)
                return
            except (_Retry, Unexpressible):
                del self.launches[mark:]
        self._emit_map_in(root, shape, [(a, 1, shape[a]) for a in range(len(shape))], et, total, node)

    def _emit_group(self, roots):
        """One flat (COL) launch storing several same-shaped maps."""
        node = self.nodes[roots[0]]
        shape = tuple(node.output.shape)
        et = node.output.element_type
        total = element_count(shape)
        buf = self.buf[roots[0]]
        if buf.subaxes:
            cand = []
            for a, d in enumerate(shape):
                if a in buf.subaxes:
                    sub = buf.subaxes[a]
                    for i, (x, st) in enumerate(sub):
                        cand.append((st, a, _prod(x2 for x2, _ in sub[i + 1:]), x))
                else:
                    cand.append((buf.strides[a], a, 1, d))
            dims = [(a, mul, x) for _, a, mul, x in sorted(cand, key=lambda t: -t[0])]
        else:
            dims = [(a, 1, shape[a]) for a in _storage_perm(buf)]
        pshape = tuple(x for _, _, x in dims)
        terms_of = lambda axes_p: [_mk_axis([(t[0], t[1], t[2], t[3] * mul) for (a2, mul, _), e in zip(dims, axes_p)
                                             if a2 == a and e is not None for t in axis_terms(e)[0]], 0)
                                   for a in range(len(shape))]
        prog = Program(self, extents=(total, 1), vec_src=0, et=et)
        axes = terms_of(iteration_axes(pshape))
        for r in roots:
            prog.eval_store(r, axes, self.buf[r])
        self._col_launch(prog, total, 1, 0, "map:" + "+".join(f"{self.nodes[r].op.wire_name}#{r}" for r in roots), et)

    def _emit_map_in(self, root, shape, dims, et, total, node):
        """One map launch iterating `dims` = [(logical axis, multiplier,
        extent)] outer to inner (a permutation of the axes, or of the
        sub-digits of flattened axes).  A chained producer (`_chains`) is
        stored by the same launch; if the pair does not fit one program the
        producer gets its own launch first."""
        side = getattr(self, "_map_side", {}).get(root)
        if side is None:
            return self._emit_map_in1(root, shape, dims, et, total, node)
        mark = len(self.launches)
        try:
            return self._emit_map_in1(root, shape, dims, et, total, node)
        except (UnsupportedOp, _TooManyDigits):
            del self.launches[mark:]
            del self._map_side[root]
            self.emit_map(side, [side])
            return self._emit_map_in1(root, shape, dims, et, total, node)

    def _emit_map_in1(self, root, shape, dims, et, total, node):
        pshape = tuple(x for _, _, x in dims)

        def logical(axes_p):
            terms = [[] for _ in shape]
            for (a, mul, _), e in zip(dims, axes_p):
                if e is not None:
                    terms[a] += [(t[0], t[1], t[2], t[3] * mul) for t in axis_terms(e)[0]]
            return [_mk_axis(t, 0) for t in terms]

        # Split the iteration space into rows (o) x contiguous columns (r)
        # when the trailing extent is long enough for warp-wide vectors.
        inner_from = len(pshape)
        while inner_from > 0 and _prod(pshape[inner_from:]) < 256:
            inner_from -= 1
        n_r = _prod(pshape[inner_from:])
        # rows x columns only when there are enough rows to fill the GPU;
        # a map has no reason to run few, very long rows (flat mode instead)
        few_rows = total // max(n_r, 1) < NUM_SMS * 8 and n_r > 8192
        side = getattr(self, "_map_side", {}).get(root)
        label = f"map:{node.op.wire_name}#{root}"
        if side is not None:
            label += f"+side:{self.nodes[side].op.wire_name}#{side}"

        def stores(prog, axes):
            if side is not None:  # the producer first, then the consumer recomputing it inline
                prog.eval_store(side, axes, self.buf[side])
                prog.eval_store(root, axes, self.buf[root], also_inline=(side,))
            else:
                prog.eval_store(root, axes, self.buf[root])

        if n_r >= 128 and inner_from < len(pshape) and not few_rows:
            n_o = total // n_r
            prog = Program(self, extents=(max(n_o, 1), n_r), vec_src=1, et=et)
            try:
                stores(prog, logical(split_axes(pshape, inner_from)))
            except _Retry:
                prog = None  # a Reshape straddles the row split: use the flat form
            if prog is not None:
                self._row_launch(prog, n_o, n_r, 0, label, et)
                return
        prog = Program(self, extents=(total, 1), vec_src=0, et=et)
        stores(prog, logical(iteration_axes(pshape)))
        self._col_launch(prog, total, 1, 0, label, et)

    def emit_reduce(self, s: int, side: int | None):
        node = self.nodes[s]
        src = node.inputs[0][0]
        in_shape = node.inputs_shape
        axes_red = node.attrs["reduction_axes"]
        kept = [a for a in range(len(in_shape)) if a not in axes_red]
        n_o = element_count([in_shape[a] for a in kept])
        n_r = element_count([in_shape[a] for a in axes_red])
        if n_o == 0:
            return
        in_axes = [None] * len(in_shape)
        for i, a in enumerate(kept):
            d = in_shape[a]
            in_axes[a] = None if d == 1 else (0, _prod(in_shape[k] for k in kept[i + 1:]), d)
        for i, a in enumerate(axes_red):
            d = in_shape[a]
            in_axes[a] = None if d == 1 else (1, _prod(in_shape[k] for k in axes_red[i + 1:]), d)
        et = node.output.element_type
        row = self._prefer_rows(src, in_axes, n_o, n_r, et)
        prog = Program(self, extents=(max(n_o, 1), max(n_r, 1)), vec_src=1 if row else 0, et=et)
        if side is not None:
            prog.eval_store(side, in_axes, self.buf[side])
        elif n_r > 0:
            prog.eval_value(src, in_axes)
        prog.set_red_out(self.buf[s], iteration_axes(node.output.shape))
        kind = 2 if node.attrs["reduction_kind"] == "max" else 1
        if row:
            self._row_launch(prog, n_o, n_r, kind, f"rowsum#{s}", et)
        else:
            self._col_launch(prog, n_o, n_r, kind, f"colsum#{s}", et)

    def _prefer_rows(self, src, in_axes, n_o, n_r, et) -> bool:
        if n_r < 32:
            return False
        probe = Program(self, extents=(max(n_o, 1), max(n_r, 1)), vec_src=1, et=et, dry=True)
        try:
            probe.eval_value(src, in_axes)
        except _Retry:
            return n_r >= 128
        mem = [l for l in probe.leaf_specs if l.buf.splat is None]
        if not mem:
            return True
        best = max(mem, key=lambda l: l.buf.nbytes)
        return any(d[0] == 1 and d[1] == 1 and d[3] == 1 for d in best.digits)

    def emit_copy(self, src: Buffer, dst: Buffer):
        n_o = element_count(dst.shape)
        if n_o == 0:
            return
        prog = Program(self, extents=(n_o, 1), vec_src=0, et=dst.et)
        axes = iteration_axes(dst.shape)
        k = prog.leaf(src, axes)
        prog.emit(I_LOAD, k=k)
        prog.emit(I_STORE, k=prog.store_leaf(dst, axes))
        self._col_launch(prog, n_o, 1, 0, "copy", dst.et)
        self.buf[("copy", dst.key)] = dst

    def _pad_channels(self, xb, xs, shape, cp):
        """Channel-last copy of activation (xb, strides xs) with its channel
        count padded to `cp` (zeros), for the 16-byte conv kernels; one copy
        per source, shared by the convolutions that read it."""
        key = (xb.key, xb.elem_off, tuple(xs), cp)
        if key in self._pads:
            return self._pads[key]
        N, Cc, H, W = shape
        P = Buffer(self.new_key(), ElementType.F32, (N, cp, H, W), (H * W * cp, 1, W * cp, cp))
        self.buf[("padc", P.key)] = P
        root = xb.base if xb.base is not None else xb
        src = Buffer(xb.key, xb.et, shape, tuple(xs), xb.slot, xb.offset, xb.splat, base=root, elem_off=xb.elem_off)
        parts = [(src, Buffer(P.key, P.et, shape, P.strides, P.slot, P.offset, None, base=P, elem_off=0))]
        zshape = (N, cp - Cc, H, W)
        parts.append((self.splat_buffer(ElementType.F32, 0.0),
                      Buffer(P.key, P.et, zshape, P.strides, P.slot, P.offset, None, base=P, elem_off=Cc)))
        for s_, d_ in parts:
            n_o = element_count(d_.shape)
            prog = Program(self, extents=(n_o, 1), vec_src=0, et=ElementType.F32)
            axes = iteration_axes(d_.shape)
            prog.emit(I_LOAD, k=prog.leaf(s_, axes))
            prog.emit(I_STORE, k=prog.store_leaf(d_, axes))
            self._col_launch(prog, n_o, 1, 0, f"padc#{P.key}", ElementType.F32)
        self._pads[key] = (P, P.strides)
        return self._pads[key]

    def add_launch(self, kind, grid, block, smem, args, prog, label):
        rec = LaunchRec(kind, grid, block, smem, args, prog.reads(), prog.writes(), label)
        rec.algo_bytes = prog.algo_bytes()
        rec.finalize = prog.finalize_fn(args)
        self.launches.append(rec)

    def emit_row_group(self, g):
        """One row-fused launch for a group (rowfuse.py) plus a short second
        pass per cross-row reduction over the per-team partials."""
        from . import rowfuse as RF

        et, esize = g.et, g.et.byte_size
        refs, reads, writes = [], [], []
        vals, index, ext_val = [], {}, {}
        full_access = []  # (s0, s1, buffer) of every FULL load / store: decides the vector width

        def ref_of(b):
            for i, x in enumerate(refs):
                if x is b:
                    return i
            refs.append(b)
            return len(refs) - 1

        def access(x):
            b = self.buf.get(x)
            if b is not None:
                return b, b.strides
            hv = self.heavy_operand(x)
            if hv is None or hv[1] is None:
                raise _DropRowGroup(g)
            return hv

        def ext(x, cls):
            key = (x, cls)
            if key in ext_val:
                return ext_val[key]
            if cls == RF.UNI:
                b = self.buf.get(x)
                if b is not None and b.splat is not None:
                    vals.append((RF.UNI, ("imm", RF.splat_bits(et, b.splat))))
                else:
                    b, _ = access(x)
                    vals.append((RF.UNI, ("loadu", ref_of(b))))
                    reads.append(b.key)
            else:
                b, st = access(x)
                if b.subaxes or b.splat is not None:
                    raise _DropRowGroup(g)
                reads.append(b.key)
                if cls == RF.FULL:
                    vals.append((RF.FULL, ("load", ref_of(b), int(st[0]), int(st[1]))))
                    full_access.append((int(st[0]), int(st[1]), b))
                elif cls == RF.ROWV:
                    vals.append((RF.ROWV, ("loadr", ref_of(b), int(st[0]))))
                else:  # COLV: only as the operand of a Broadcast along rows
                    vals.append((RF.FULL, ("colv", ref_of(b), int(st[0]))))
            ext_val[key] = len(vals) - 1
            return ext_val[key]

        def operand(r, cls):
            return index[r] if r in index else ext(r, g.externals[r])

        for n in g.members:
            node = self.nodes[n]
            c = g.cls[n]
            ins = [r for r, _ in node.inputs]
            if node.op in ELEMENTWISE_UNARY:
                e = ("un", RF.UNARY_CODE[node.op], operand(ins[0], c))
            elif node.op in ELEMENTWISE_BINARY:
                e = ("bin", RF.BINARY_CODE[node.op], operand(ins[0], c), operand(ins[1], c))
            elif node.op is OpKind.BROADCAST:
                r = ins[0]
                if r not in index and g.externals[r] == RF.COLV:
                    index[n] = ext(r, RF.COLV)
                    continue
                e = ("bcast", operand(r, None))
            else:  # Sum: a row reduction or a cross-row one
                kind = 2 if node.attrs["reduction_kind"] == "max" else 1
                a = operand(ins[0], None)
                e = ("rred", kind, a) if c == RF.ROWV else ("xred", kind, a, vals[a][0])
            vals.append((c, e))
            index[n] = len(vals) - 1
        stores, xrow, pass2 = [], [], []
        for o in g.outputs:
            b = self.buf[o]
            if b.subaxes:
                raise _DropRowGroup(g)
            writes.append(b.key)
            if g.cls[o] == RF.XROW:
                continue
            st = b.strides
            if g.cls[o] == RF.FULL:
                stores.append((index[o], ref_of(b), int(st[0]), int(st[1])))
                full_access.append((int(st[0]), int(st[1]), b))
            else:
                stores.append((index[o], ref_of(b), int(st[0]), 0))
        vec_ok = all(s1 == 1 and s0 % (16 // esize) == 0 and (b.elem_off * esize) % 16 == 0 for s0, s1, b in full_access)
        team, block, vec = RF.geometry(g.C, esize, vec_ok)
        per_block = block // team
        blocks = max(1, min((g.R + per_block - 1) // per_block, NUM_SMS * max(1, 2048 // block)))
        n_teams = blocks * per_block
        for o in g.outputs:
            if g.cls[o] != RF.XROW:
                continue
            kind = vals[index[o]][1][1]
            partial = Buffer(self.new_key(), et, (n_teams,), (1,))
            self.buf[("rowpart", partial.key)] = partial
            writes.append(partial.key)
            xrow.append((index[o], kind, ref_of(partial)))
            pass2.append((o, kind, partial))
        if len(refs) > abi.ROW_MAX_REFS:
            raise _DropRowGroup(g)
        live = sum(1 for c, _ in vals if c == RF.FULL)
        if live > 4 * RF.MAX_FULL_LIVE:
            raise _DropRowGroup(g)
        spec = RF.RowSpec(g.R, g.C, "float" if et is ElementType.F32 else "double", team, block, vec, vals, stores, xrow,
                          n_teams)
        args = abi.RowArgs(n_refs=len(refs))
        label = f"row:{self.nodes[g.members[0]].op.wire_name}#{g.members[0]}..{self.nodes[g.anchor].op.wire_name}#{g.anchor}"
        rec = LaunchRec(abi.K_ROWJIT, (blocks, 1, 1), (block, 1, 1), 0, args, sorted(set(reads)), sorted(set(writes)), label)
        ext_bytes = {RF.FULL: g.R * g.C, RF.ROWV: g.R, RF.COLV: g.C, RF.UNI: 1}
        rec.algo_bytes = esize * (sum(ext_bytes[c] for c in g.externals.values())
                                  + sum(ext_bytes.get(g.cls[o], 1) for o in g.outputs))
        bufs = list(refs)

        def fin():
            for i, b in enumerate(bufs):
                args.refs[i] = _buf_ref(b)
        rec.finalize = fin
        rec.row_spec = spec
        self.launches.append(rec)
        for o, kind, partial in pass2:
            rowwise = n_teams >= 256
            p2 = Program(self, extents=(1, n_teams), vec_src=1 if rowwise else 0, et=et)
            k = p2.leaf(partial, [(1, 1, n_teams)])
            p2.emit(I_LOAD, k=k)
            p2.set_red_out(self.buf[o], iteration_axes(self.nodes[o].output.shape))
            if rowwise:
                self._row_launch(p2, 1, n_teams, kind, f"rowsum#{o}:teams", et)
            else:
                self._col_launch(p2, 1, n_teams, kind, f"rowsum#{o}:teams", et)

    def _gradient_regions(self):
        """Place the data-parallel partial roots contiguously, in production
        order (for a training step: the loss, then the gradients in reverse
        layer order), one arena region per (element type, reduction op).
        Each root becomes a dense view into its region, so a run of
        consecutive roots is one all-reduce bucket."""
        groups: dict = {}
        for n in self.order:
            if n not in self.allreduce:
                continue
            b = self.buf.get(n)
            if b is None or b.slot != abi.SLOT_ARENA or b.base is not None:
                raise UnsupportedOp(f"data parallel: partial root {n} is not materialised in the arena")
            if b.et not in (ElementType.F32, ElementType.F64):
                raise UnsupportedOp("data parallel all-reduce needs a float tensor")
            groups.setdefault((b.et, n in self.allreduce_max), []).append(n)
        regions = []
        for (et, is_max), ns in groups.items():
            region = Buffer(self.new_key(), et, (0,), (1,), abi.SLOT_ARENA)
            off, members = 0, []
            for n in ns:
                b = self.buf[n]
                b.base, b.elem_off = region, off // et.byte_size
                b.bucket = (region, is_max)
                members.append(b)
                off = align_up(off + b.nbytes, DEVICE_ALIGNMENT)
            region.shape = (max(1, off // et.byte_size),)
            regions.append((region, members))
        return regions

    def _bucket_allreduces(self):
        """Insert the all-reduce launches over the gradient regions.

        A bucket is a run of consecutive roots of one region; it is reduced
        right after the launch that finishes its last member once it holds
        GFB_BUCKET_MB (default 32) MiB, or earlier if a later launch reads
        one of its members before that (the SGD update of that parameter).
        Buckets are issued in the order their members were produced, so a
        layer's gradients are summed while the earlier layers' backward
        GEMMs still run (the schedule keeps collectives in program order on
        stream 0; everything else may overlap them)."""
        cap = int(float(os.environ.get("GFB_BUCKET_MB", "32")) * (1 << 20))
        member_of = {}
        for region, members in self._grad_regions:
            for b in members:
                member_of[b.key] = b
        last_write = {}
        for i, L in enumerate(self.launches):
            for k in L.writes:
                if k in member_of:
                    last_write[k] = i
        out = []
        pending: list = []  # members fully produced, not yet reduced

        def flush():
            runs = []
            for b in sorted(pending, key=lambda b: (id(b.bucket[0]), b.elem_off)):
                if runs and runs[-1][-1].bucket[0] is b.bucket[0] and \
                        align_up(runs[-1][-1].elem_off * b.et.byte_size + runs[-1][-1].nbytes, DEVICE_ALIGNMENT) \
                        == b.elem_off * b.et.byte_size:
                    runs[-1].append(b)
                else:
                    runs.append([b])
            for run in runs:
                out.append(self._allreduce_rec(run))
            pending.clear()

        for i, L in enumerate(self.launches):
            if L.kind != abi.K_ALLREDUCE and any(k in member_of and last_write.get(k, -1) < i and
                                                 member_of[k] in pending for k in L.reads):
                flush()
            out.append(L)
            done = [member_of[k] for k, j in last_write.items() if j == i]
            pending.extend(b for b in done if b not in pending)
            if pending and sum(b.nbytes for b in pending) >= cap:
                flush()
        if pending:
            flush()
        self.launches = out

    def _allreduce_rec(self, run):
        """One in-place NCCL all-reduce over consecutive members of a region."""
        region, is_max = run[0].bucket
        et = run[0].et
        first, last = run[0], run[-1]
        count = last.elem_off + element_count(last.shape) - first.elem_off
        args = abi.AllReduceArgs(count=count, dtype=0 if et is ElementType.F32 else 1, op=1 if is_max else 0)
        keys = [b.key for b in run]
        label = "allreduce#" + ",".join(str(n) for n in self._nodes_of(keys))
        rec = LaunchRec(abi.K_ALLREDUCE, (1, 1, 1), (1, 1, 1), 0, args, keys, keys, label)
        rec.algo_bytes = count * et.byte_size
        rec.finalize = _finalize_refs(args, {"buf": first})
        return rec

    def _nodes_of(self, keys):
        ks = set(keys)
        return [n for n, b in self.buf.items() if b.key in ks]

    # -- heavy ops
    def operand(self, ref_node):
        op = self.heavy_operand(ref_node)
        if op is None:
            raise _Retry(ref_node)
        return op

    def emit_dot_tc(self, n, a_op, b_op, out, m, nn, k):
        """Split both operands into K-major TF32 hi/lo planes, then one
        tcgen05 3xTF32 GEMM (csrc/gemm_tc.cu), split-K when the output is
        too small to fill the GPU."""
        (ab, ast), (bb, bst) = a_op, b_op
        pair = m >= 256 and nn >= 256 and os.environ.get("GFB_TC_PAIR", "1") == "1" and os.environ.get("GFB_TC_WIDE", "1") == "1"
        if pair and use_f16():
            # B first: its planes (a weight, typically) are then split -- and under
            # host-buffer runs copied -- before the row chunks of a large A input
            b16 = self._f16_operand(bb, bst[1], bst[0], nn, k)
            a16 = self._f16_operand(ab, ast[0], ast[1], m, k) if b16 is not None else None
            if b16 is not None and a16 is None:
                self._flush_chunks(bb)  # (planes made for nothing; keep them consistent)
            if a16 is not None:
                addr = {"c_sm": out.strides[0], "c_sn": out.strides[1]}
                root = ab.base if ab.base is not None else ab
                chunks = self._f16_chunks.get(root.key) if a16[4] == 0 else None
                if a16[4] == 0 and chunks is None and root.key in self._row_chunked:
                    # A's planes were written row chunk by row chunk by the previous
                    # layer's GEMM: this layer follows the same chunks (the forward
                    # pipelines with the input's row pieces)
                    hi, lo, sc = a16[:3]
                    tcn = (k + 127) // 128
                    chunks = [[r0, r1, self._row_view(hi, r0, r1, k // 2), self._row_view(lo, r0, r1, k // 2),
                               self._row_view(sc, r0 // 128, r1 // 128, tcn), None] for r0, r1 in self._row_chunked[root.key]]
                epi = self._epi.get(n, {})
                self._flush_chunks(bb)
                if (chunks and self._tc_splits(chunks[0][1] - chunks[0][0], nn, k) == 1 and k % 2 == 0
                        and (chunks[0][5] is not None or root.key in self._row_chunked)
                        and "colsum" not in epi and out.strides == (nn, 1) and not out.elem_off and out.base is None):
                    for c, ch in enumerate(chunks):  # split chunk c (an input), then the GEMM over its rows
                        r0, r1, hv, lv, sv, split = ch
                        if split is not None:
                            split.chain, split.row_chunk = ("rows",), c
                        self._emit_chunk(ch)
                        rec = self._f16_gemm(n, (hv, lv, sv) + a16[3:], b16, out, r1 - r0, nn, k, addr,
                                             f"dot_f16#{n}:rows{r0}", rows=(r0, m))
                        rec.algo_bytes = ((r1 - r0) * k + k * nn + (r1 - r0) * nn) * 4
                        rec.chain, rec.row_chunk = ("rows",), c  # one chain: persistent GEMMs never overlap
                        if rec.args.epi_flags & 4 and epi:
                            y = self.buf[epi["lo_of"]]
                            yroot = y.base if y.base is not None else y
                            self._row_chunked[yroot.key] = [(ch_[0], ch_[1]) for ch_ in chunks]
                    return
                self._flush_chunks(ab)
                rec = self._f16_gemm(n, a16, b16, out, m, nn, k, addr, f"dot_f16#{n}")
                rec.algo_bytes = (m * k + k * nn + m * nn) * 4
                return
        a = self._raw_mn(ab, ast[0], ast[1], m, k) if pair else None
        b = self._raw_mn(bb, bst[1], bst[0], nn, k) if pair else None
        if a is None:
            a = self._split(n, "a", ab, m, k, 0, s_r=ast[0], s_k=ast[1])
        if b is None:
            b = self._split(n, "b", bb, nn, k, 0, s_r=bst[1], s_k=bst[0])
        rec = self._tc_gemm(n, a, b, out, m, nn, k, {"c_sm": out.strides[0], "c_sn": out.strides[1]}, f"dot_tc#{n}")
        rec.algo_bytes = (m * k + k * nn + m * nn) * 4

    def _plan_epilogues(self) -> dict:
        """Dots whose only consumer is an elementwise map the pair GEMM can
        apply in its epilogue (gfb_tc_args.epi_kind): config E's forward
        Dot -> Add(Broadcast(bias)) -> Relu, and its backward
        Dot -> Multiply(Maximum(Divide(relu, x), 0)) (the Relu gradient,
        autodiff.py:143-148).  The maps' nodes are then written by the GEMM
        (every op the same IEEE op, so bit-identical) and the Dot's own
        [M, N] output never touches memory."""
        if os.environ.get("GFB_TC_EPILOGUE", "1") != "1" or os.environ.get("GFB_TC_PAIR", "1") != "1":
            return {}
        out = {}
        results = {r for r, _ in self.g.results}
        nodes = self.nodes

        def dense2(n, M, N):
            return (tuple(nodes[n].output.shape) == (M, N) and self.layouts[(n, 0)].order == (0, 1)
                    and nodes[n].output.element_type is ElementType.F32)

        def plain(n):  # a node the epilogue may write: materialised, not claimed by other fusions
            return (n in self.M and n not in self._row_nodes and n not in self.allreduce
                    and n not in results and n not in self.tiny)

        def splat_zero(n):
            nd = nodes[n]
            if nd.op is not OpKind.CONSTANT or not nd.attrs["data"].is_splat:
                return False
            v = nd.attrs["data"].splat_value()
            return float(v) == 0.0 and not np.signbit(v)

        for d in self.order:
            nd = nodes[d]
            if nd.op is not OpKind.DOT or not self.is_heavy(d) or nd.output.element_type is not ElementType.F32:
                continue
            M, N = nd.output.shape
            Kd = nodes[nd.inputs[0][0]].output.shape[1]
            if (M < 256 or N < 256 or not use_tensor_cores(M, N, Kd) or len(self.consumers[d]) != 1 or d in results
                    or self._tc_splits(M, N, Kd) > 1):
                continue  # (a split-K GEMM writes partials: no place for an epilogue)
            c = self.consumers[d][0]
            cn = nodes[c]
            kinds = os.environ.get("GFB_TC_EPILOGUE_KINDS", "1,2").split(",")
            if cn.op is OpKind.ADD and "1" in kinds and plain(c) and dense2(c, M, N):
                other = [r for r, _ in cn.inputs if r != d]
                if len(other) != 1:
                    continue
                bc = nodes[other[0]]
                if not (bc.op is OpKind.BROADCAST and tuple(bc.attrs["broadcast_axes"]) == (0,)
                        and tuple(bc.inputs_shape) == (N,) and bc.id not in self.M):
                    continue
                bias = bc.inputs[0][0]
                if not (self.is_source(bias) and nodes[bias].output.element_type is ElementType.F32):
                    continue
                relus = [r for r in self.consumers[c] if nodes[r].op is OpKind.RELU and plain(r) and dense2(r, M, N)]
                if not relus:
                    continue
                out[d] = {"kind": 1, "out": c, "out2": relus[0], "bias": bias, "absorbed": {c, relus[0]},
                          "lo_of": relus[0]}
            elif cn.op is OpKind.MULTIPLY and "2" in kinds and plain(c) and dense2(c, M, N):
                other = [r for r, _ in cn.inputs if r != d]
                if len(other) != 1:
                    continue
                mk = nodes[other[0]]
                if mk.op is not OpKind.MAXIMUM or mk.id in self.M or not splat_zero(mk.inputs[1][0]):
                    continue
                dv = nodes[mk.inputs[0][0]]
                if dv.op is not OpKind.DIVIDE or dv.id in self.M:
                    continue
                h, x = dv.inputs[0][0], dv.inputs[1][0]
                if not (self.is_source(h) and self.is_source(x) and dense2(h, M, N) and dense2(x, M, N)):
                    continue
                out[d] = {"kind": 2, "out": c, "aux1": h, "aux2": x, "absorbed": {c}, "lo_of": c}
                # the bias gradient Sum(c, axes (0,)) reads c once more: the epilogue
                # writes 32-row column partials and the Sum reduces those instead
                for r in self.consumers[c]:
                    rn = nodes[r]
                    if (rn.op is OpKind.SUM and tuple(rn.attrs["reduction_axes"]) == (0,)
                            and rn.attrs["reduction_kind"] == "sum" and r in self.M and r not in self._row_nodes
                            and os.environ.get("GFB_TC_COLSUM", "1") == "1"):
                        out[d]["colsum"] = r
                        break
        # A Relu-gradient epilogue whose x is the pre-activation a bias + Relu
        # epilogue writes reads that GEMM's mask bytes (1 B per element) instead
        # of x (4 B); x and the Relu output then often have no reader left and
        # are not stored at all (_drop_unread_epilogue_outputs).
        if os.environ.get("GFB_TC_MASK", "1") == "1":
            writer = {sp["out"]: d for d, sp in out.items() if sp["kind"] == 1}
            for d, sp in out.items():
                if sp["kind"] == 2 and sp["aux2"] in writer:
                    sp["mask"] = sp["aux2"]
                    out[writer[sp["aux2"]]]["mask_of"] = sp["aux2"]
        return out

    def _plan_conv_relu(self) -> dict:
        """The 3-channel 7x7 stem conv whose output feeds a Relu: the 2xFP16
        stem kernel writes Relu(y) beside y (gfb_stemh_args.c2), so the Relu
        map (a 1.6 GB read + write at config D's 224x224) is not launched.
        If the conv takes another kernel after all, emit_heavy emits the map."""
        if os.environ.get("GFB_STEM_RELU", "1") != "1" or os.environ.get("GFB_CONV_F16", "1") != "1":
            return {}
        out = {}
        results = {r for r, _ in self.g.results}
        for d in self.order:
            nd = self.nodes[d]
            if nd.op is not OpKind.CONV2D or nd.output.element_type is not ElementType.F32 or not self.is_heavy(d):
                continue
            xs_, ws_ = self.nodes[nd.inputs[0][0]].output.shape, self.nodes[nd.inputs[1][0]].output.shape
            if tuple(nd.attrs["strides"]) != (1, 1) or tuple(ws_[1:]) != (3, 7, 7) or ws_[0] != 64 or xs_[1] != 3:
                continue
            # the Relu reads y directly or through a ConvertLayout (an index view: same
            # values at the same logical index); _conv_stemh checks the two buffers'
            # strides agree before it takes the Relu
            cands = [r for r in self.consumers[d]]
            for c in self.consumers[d]:
                if self.nodes[c].op is OpKind.CONVERT_LAYOUT and c not in self.M:
                    cands += self.consumers[c]
            for r in cands:
                rn = self.nodes[r]
                if (rn.op is OpKind.RELU and r in self.M and r not in results and r not in self._row_nodes
                        and r not in self.allreduce and r not in self._epi_nodes
                        and tuple(rn.output.shape) == tuple(nd.output.shape)):
                    out[d] = r
                    break
        return out

    def _feeds_tc(self, n) -> bool:
        """Some Dot reads `n` (directly or through index views) on the tensor cores."""
        stack, seen = [n], set()
        while stack:
            x = stack.pop()
            for c in self.consumers[x]:
                if c in seen:
                    continue
                seen.add(c)
                cn = self.nodes[c]
                if cn.op in INDEX_OPS:
                    stack.append(c)
                elif cn.op is OpKind.DOT and self.is_heavy(c) and cn.output.element_type is ElementType.F32:
                    m, k = self.nodes[cn.inputs[0][0]].output.shape
                    if use_tensor_cores(m, cn.output.shape[1], k):
                        return True
        return False

    def _dense_root(self, src):
        """The whole dense arena buffer `src` views at offset 0, or None."""
        root = src.base if src.base is not None else src
        if (src.splat is not None or root.slot != abi.SLOT_ARENA or src.elem_off != 0 or root.subaxes
                or root.et is not ElementType.F32 or not _dense_rowmajor(root.shape, root.strides)
                or element_count(root.shape) % 4):
            return None
        return root

    def _lo_plane(self, root):
        """lo = x - trunc_tf32(x) of a dense arena tensor, in the tensor's own
        layout, written once (split mode 7) and shared by every GEMM that
        reads the tensor as a raw-hi operand, K-major or MN-major."""
        key = ("lo", root.key)
        lo = self.buf.get(key)
        if lo is None:
            total = element_count(root.shape)
            lo = Buffer(self.new_key(), ElementType.F32, root.shape, root.strides)
            self.buf[key] = lo
            sa = abi.SplitArgs(rows=1, k=total, kp=total, s_r=total, s_k=1, mode=7)
            grid = (max(1, min((total // 4 + 255) // 256, NUM_SMS * 16)), 1, 1)
            rec = LaunchRec(abi.K_SPLIT_TF32, grid, (256, 1, 1), 0, sa, [root.key], [lo.key], f"lo#{root.key}")
            rec.algo_bytes = 2 * total * 4
            rec.finalize = _finalize_refs(sa, {"src": root, "hi": root, "lo": lo})
            self.launches.append(rec)
        return lo

    # -- 2xFP16 block-scaled GEMM (csrc/gemm_f16.cu)
    def _f16_operand(self, src, s_r, s_k, rows, kdim):
        """Operand [rows, k] of the fp16 pair GEMM: a dense row-major F32
        tensor read K-major (s_k == 1) or MN-major (s_r == 1), with its fp16
        planes and tile scales (shared by every GEMM that reads the tensor,
        either way).  Returns (hi, lo, sc, kp, ld_mn, sc_r, sc_k) or None."""
        root = src.base if src.base is not None else src
        if (src.splat is not None or src.elem_off or root.subaxes or root.et is not ElementType.F32
                or not _dense_rowmajor(root.shape, root.strides) or element_count(root.shape) != rows * kdim):
            return None
        if s_k == 1 and s_r == kdim and kdim % 8 == 0:
            hi, lo, sc = self._f16_planes(root, rows, kdim)
            return hi, lo, sc, kdim, 0, (kdim + 127) // 128, 1
        if s_r == 1 and s_k == rows and rows % 64 == 0:
            hi, lo, sc = self._f16_planes(root, kdim, rows)
            return hi, lo, sc, align_up(kdim, 8), rows, 1, (rows + 127) // 128
        return None

    def _f16_planes(self, root, R, Cc):
        """fp16 hi / lo planes of the dense tensor `root` viewed as [R, Cc]
        and its 128 x 128 tile scales: written by the epilogue of the GEMM
        producing `root` when there is one (epi_flags bit 2), else by one
        split pass (gfb_split16_kernel, 8 B of traffic per element)."""
        got = self._f16_get(root)
        if got is not None:
            return got
        planes = self._f16_buffers(root, R, Cc)
        hi, lo, sc = planes
        nch = self._input_chunks(root, R, Cc)
        if nch > 1:
            # a large caller input crosses PCIe in row chunks under host-buffer
            # runs: split (and multiply, _f16_gemm) chunk by chunk, so the
            # first GEMM starts when the first rows have arrived
            rows = R // nch
            tcn = (Cc + 127) // 128
            chunks = []
            for c in range(nch):
                r0, r1 = c * rows, (c + 1) * rows
                src = self._row_view(root, r0, r1, Cc)
                hv, lv = self._row_view(hi, r0, r1, Cc // 2), self._row_view(lo, r0, r1, Cc // 2)
                sv = self._row_view(sc, r0 // 128, r1 // 128, tcn)
                sa = abi.Split16Args(rows=rows, cols=Cc, ld=Cc)
                tiles = (rows // 128) * tcn
                rec = LaunchRec(abi.K_SPLIT_F16, (max(1, min(tiles, NUM_SMS * 4)), 1, 1), (256, 1, 1), 0, sa, [src.key],
                                [hv.key, lv.key, sv.key], f"split16#{root.key}:rows{r0}")
                rec.algo_bytes = rows * Cc * 8
                rec.finalize = _finalize_refs(sa, {"src": src, "hi": hv, "lo": lv, "sc": sv})
                chunks.append([r0, r1, hv, lv, sv, rec])  # emitted by _emit_chunk (before its GEMM chunk)
            self._f16_chunks[root.key] = chunks
            return planes
        sa = abi.Split16Args(rows=R, cols=Cc, ld=Cc)
        tiles = ((R + 127) // 128) * ((Cc + 127) // 128)
        rec = LaunchRec(abi.K_SPLIT_F16, (max(1, min(tiles, NUM_SMS * 4)), 1, 1), (256, 1, 1), 0, sa, [root.key],
                        [hi.key, lo.key, sc.key], f"split16#{root.key}")
        rec.algo_bytes = R * Cc * 8
        rec.finalize = _finalize_refs(sa, {"src": root, "hi": hi, "lo": lo, "sc": sc})
        self.launches.append(rec)
        return planes

    def _input_chunks(self, root, R, Cc) -> int:
        """Row chunks of a caller input's fp16 split (GFB_INPUT_CHUNKS, 4):
        inputs of at least 256 MB whose rows split into whole 256-row tiles."""
        nch = int(os.environ.get("GFB_INPUT_CHUNKS", "4"))
        min_mb = float(os.environ.get("GFB_INPUT_CHUNK_MIN_MB", "256"))
        if (nch <= 1 or not (abi.SLOT_IO <= root.slot < abi.SLOT_IO + self.n_in) or R * Cc * 4 < min_mb * (1 << 20)
                or R % (nch * 256) or Cc % 8):
            return 1
        return nch

    def _emit_chunk(self, ch):
        if ch[5] is not None:
            self.launches.append(ch[5])
            ch[5] = None

    def _flush_chunks(self, *bufs):
        """Every pending split chunk of these operands' inputs (a consumer
        that reads the whole planes)."""
        for b in bufs:
            root = b.base if b.base is not None else b
            for ch in self._f16_chunks.get(root.key, ()):
                self._emit_chunk(ch)

    def _row_view(self, base, r0, r1, row_elems):
        """Rows [r0, r1) of the dense row-major `base` (row_elems elements of
        base.et per row) as an exact contiguous view with its own key."""
        v = Buffer(self.new_key(), base.et, ((r1 - r0) * row_elems,), (1,), base.slot, base.offset, None, base=base,
                   elem_off=r0 * row_elems, exact=True)
        self.buf[("view", v.key)] = v
        return v

    def _f16_get(self, root):
        parts = [self.buf.get(("f16", root.key, p)) for p in ("hi", "lo", "sc")]
        return None if parts[0] is None else tuple(parts)

    def _f16_buffers(self, root, R, Cc):
        """Register the planes of `root` (fp16 planes are sized as F32
        buffers of half the element count)."""
        hi = Buffer(self.new_key(), ElementType.F32, ((R * Cc + 1) // 2,), (1,))
        lo = Buffer(self.new_key(), ElementType.F32, ((R * Cc + 1) // 2,), (1,))
        sc = Buffer(self.new_key(), ElementType.F32, (((R + 127) // 128) * ((Cc + 127) // 128),), (1,))
        for p, b in (("hi", hi), ("lo", lo), ("sc", sc)):
            self.buf[("f16", root.key, p)] = b
        return hi, lo, sc

    def _f16_gemm(self, n, a, b, out, m, ncols, kdim, addr, label, rows=None):
        """The fp16 pair GEMM over planes (split-K on 128-K boundaries, the
        scale blocks, + the deterministic reduce pass).  rows = (r0, M): this
        launch covers rows [r0, r0 + m) of an M-row product (a row chunk of a
        split input): the output and every epilogue tensor are row views."""
        (ahi, alo, asc, kpa, a_mn, a_r, a_k), (bhi, blo, bsc, kpb, b_mn, b_r, b_k) = a, b
        r0, m_full = rows if rows is not None else (0, m)

        def chunk(buf, row_elems):  # rows [r0, r0 + m) of a full [m_full, ...] buffer
            return buf if rows is None else self._row_view(buf, r0, r0 + m, row_elems)
        splits = self._tc_splits(m, ncols, kdim)
        ta = abi.TcArgs(M=m, N=ncols, K=kdim, kp_a=kpa, kp_b=kpb, a_ld_mn=a_mn, b_ld_mn=b_mn,
                        a_sc_r=a_r, a_sc_k=a_k, b_sc_r=b_r, b_sc_k=b_k,
                        group_m=int(os.environ.get("GFB_TC_GROUP_M", "1")))
        ta.pad[0] = int(os.environ.get("GFB_F16_L2", "0"))  # L2 policy bits (gemm_f16.cu producer): 1 keep A, 2 keep B
        target = chunk(out, ncols)
        if splits > 1:
            kchunks = (kdim + 127) // 128
            per = ((kchunks + splits - 1) // splits) * 128
            splits = (kdim + per - 1) // per
        if splits > 1:
            scratch = Buffer(self.new_key(), ElementType.F32, (splits, m, ncols), (m * ncols, ncols, 1))
            self.buf[("splitk", n)] = scratch
            ta.k_splits, ta.k_per_split, ta.split_stride = splits, per, m * ncols
            ta.c_sm, ta.c_sn = ncols, 1
            target = scratch
        else:
            for k_, v_ in addr.items():
                setattr(ta, k_, v_)
        ntiles = ((ncols + 255) // 256) * ((m + 255) // 256) * max(1, splits)
        pairs = NUM_SMS // 2 if os.environ.get("GFB_TC_PERSIST", "1") == "1" else ntiles
        grid = (2 * min(ntiles, pairs), 1, 1)
        reads, writes = [ahi.key, alo.key, asc.key, bhi.key, blo.key, bsc.key], [target.key]
        refs = {"c": target, "a_hi": ahi, "a_lo": alo, "a_sc": asc, "b_hi": bhi, "b_lo": blo, "b_sc": bsc}
        epi = self._epi.get(n) if hasattr(self, "_epi") else None
        if epi is not None:
            if splits > 1 or ncols % 4 or (rows is None and (target.strides != (ncols, 1) or target.elem_off)):
                raise UnsupportedOp(f"fused epilogue of Dot {n} needs an unsplit GEMM and a dense output")
            ta.epi_kind = epi["kind"]
            ta.epi_flags = 1 if "out2" in epi else 0
            mask = self.buf.get(("mask", epi["mask"])) if "mask" in epi else None
            if mask is not None:
                refs["e_mask"] = mask
                reads.append(mask.key)
                ta.epi_flags |= 16
            # (the kernel derives the Relu-gradient mask from x alone: e_aux1 is never read)
            if mask is not None and rows is not None:
                mask = chunk(mask, ncols)
                refs["e_mask"] = mask
                reads[-1] = mask.key
            for field, key in (("e_bias", "bias"), ("e_aux2", "aux2"), ("e_out2", "out2")):
                if key in epi and not (field == "e_aux2" and mask is not None):
                    bb = self.buf[epi[key]]
                    if field != "e_bias":
                        bb = chunk(bb, ncols)
                    refs[field] = bb
                    (writes if field == "e_out2" else reads).append(bb.key)
            if "mask_of" in epi:
                mb = self.buf.get(("mask", epi["mask_of"]))
                if mb is None:
                    mb = Buffer(self.new_key(), ElementType.BOOL, (m_full * ncols,), (1,))
                    self.buf[("mask", epi["mask_of"])] = mb
                mb = chunk(mb, ncols)
                refs["e_mask"] = mb
                writes.append(mb.key)
                ta.epi_flags |= 8
            y = self.buf[epi["lo_of"]]
            root = y.base if y.base is not None else y
            fresh = self._f16_get(root) is None
            if (y.splat is None and not y.elem_off and not root.subaxes and _dense_rowmajor(root.shape, root.strides)
                    and element_count(root.shape) == m_full * ncols and ncols % 8 == 0 and self._feeds_tc(epi["lo_of"])
                    and (fresh or root.key in self._epi_planes)):
                if fresh:  # _f16_planes finds them: no split pass
                    self._f16_buffers(root, m_full, ncols)
                    self._epi_planes.add(root.key)
                hi, lo, sc = self._f16_get(root)
                planes = (chunk(hi, ncols // 2), chunk(lo, ncols // 2),
                          sc if rows is None else self._row_view(sc, r0 // 128, (r0 + m) // 128, (ncols + 127) // 128))
                refs["e_hi"], refs["e_lo"], refs["e_sc"] = planes
                writes.extend(pl.key for pl in planes)
                ta.epi_flags |= 4
            label += ":epi" + ("bias_relu" if epi["kind"] == 1 else "relu_grad")
        colsum = None
        if epi is not None and "colsum" in epi and ncols % 4 == 0:
            rp = (m + 31) // 32
            part = Buffer(self.new_key(), ElementType.F32, (rp, ncols), (ncols, 1))
            self.buf[("csum", n)] = part
            refs["e_csum"] = part
            writes.append(part.key)
            ta.epi_flags |= 64
            colsum = (epi["colsum"], part, rp)
        rec = LaunchRec(abi.K_DOT_F16P, grid, (320, 1, 1), F16_SMEM_PAIR, ta, reads, writes, label)
        rec.flops = 2 * m * ncols * kdim
        rec.epi_bufs = {"c": target, "out2": refs.get("e_out2")}  # (row views when chunked)
        rec.finalize = _finalize_refs(ta, refs)
        self.launches.append(rec)
        if colsum is not None:
            s, part, rp = colsum
            p2 = Program(self, extents=(ncols, rp), vec_src=0, et=ElementType.F32)
            k = p2.leaf(part, [(1, 1, rp), (0, 1, ncols)])
            p2.emit(I_LOAD, k=k)
            p2.set_red_out(self.buf[s], iteration_axes(self.nodes[s].output.shape))
            self._col_launch(p2, ncols, rp, 1, f"colsum#{s}:part", ElementType.F32)
            self._csum_done.add(s)
        if splits > 1:
            p2 = Program(self, extents=(m * ncols, splits), vec_src=0, et=ElementType.F32)
            k = p2.leaf(target, [(1, 1, splits), (0, ncols, m), (0, 1, ncols)])
            p2.emit(I_LOAD, k=k)
            p2.red_out = LeafSpec(out, _conv_out_digits(addr, m, ncols), True)
            p2.red_out.vec = vec_class(p2.red_out.digits, 0, True, vec_width(ElementType.F32), 4)
            self._col_launch(p2, m * ncols, splits, 1, label + ":splitk", ElementType.F32)
        return rec

    def _raw_mn(self, src, s_r, s_k, rows, kdim):
        """Operand [rows, k] read in place from its arena tensor: as an
        MN-major operand when rows are contiguous (s_r == 1; e.g. the
        activation of a weight gradient Dot(Reshape(h, (1, 0)), dz)), with the
        shared lo plane.  Returns (hi, lo, kp, ld_mn) or None (split instead)."""
        if s_r != 1 or rows % 32 or s_k % 4 or s_k < rows or os.environ.get("GFB_MN_MAJOR", "1") != "1":
            return None
        root = self._dense_root(src)
        if root is None or element_count(root.shape) < s_k * kdim:
            return None
        return root, self._lo_plane(root), align_up(kdim, 4), s_k

    def _split(self, n, name, src, rows, kdim, mode, s_r=0, s_k=0, geo=(), st=()):
        """hi/lo TF32 planes [rows, kp] of an implicit-GEMM operand.

        A dense, row-contiguous operand that lives in the arena (a fixed
        address the tensor maps can name) is its own hi plane: the tensor
        core reads only the TF32 bits of an fp32 value, i.e. hi = trunc(x);
        only lo = x - trunc(x) is written (split mode 7), which saves the hi
        plane's write and read (1 GiB each for a config-E activation)."""
        kp = align_up(kdim, 4)
        root = self._dense_root(src) if mode == 0 else None
        if (root is not None and s_k == 1 and kdim == kp and s_r == kp and element_count(root.shape) == rows * kp
                and os.environ.get("GFB_RAW_HI", "1") == "1"):
            return root, self._lo_plane(root), kp
        hi = Buffer(self.new_key(), ElementType.F32, (rows, kp), (kp, 1))
        lo = Buffer(self.new_key(), ElementType.F32, (rows, kp), (kp, 1))
        self.buf[("tc", n, name, "hi")] = hi
        self.buf[("tc", n, name, "lo")] = lo
        if mode == 3 and len(geo) >= 15 and len(st) >= 3:
            e0, e1, e2 = geo[12:15]
            t0, t1, t2 = st[:3]
            if (e1 <= 1 or t1 == e2 * t2) and (e0 <= 1 or t0 == e1 * e2 * t2):
                mode, s_k = 0, t2  # the K digits collapse to one linear stride (e.g. NHWC pixels)
        if mode == 0 and s_k == 1 and kdim == kp and s_r % 4 == 0 and src.splat is None:
            mode = 5  # streaming, 128-bit
        elif (mode == 0 and s_r == 1 and s_k % 4 == 0 and src.splat is None and (src.offset + src.elem_off * 4) % 16 == 0
              and os.environ.get("GFB_SPLIT_T", "1") == "1"):
            mode = 6  # transposing, 64x64 tiles with 128-bit loads and stores
        sa = abi.SplitArgs(rows=rows, k=kdim, kp=kp, s_r=s_r, s_k=s_k, mode=mode)
        sa.geo[:len(geo)] = list(geo)
        sa.st[:len(st)] = list(st)
        if mode == 5:
            grid = (max(1, min((rows * kp // 4 + 255) // 256, NUM_SMS * 16)), 1, 1)
        elif mode == 6:
            grid = (max(1, min(((rows + 63) // 64) * ((kp + 63) // 64), NUM_SMS * 8)), 1, 1)
        else:
            grid = (((rows + 31) // 32) * ((kp + 31) // 32), 1, 1)
        rec = LaunchRec(abi.K_SPLIT_TF32, grid, (256, 1, 1), 0, sa, [src.key], [hi.key, lo.key], f"split_{name}#{n}")
        rec.algo_bytes = rows * kdim * 4 + 2 * rows * kp * 4
        rec.finalize = _finalize_refs(sa, {"src": src, "hi": hi, "lo": lo})
        self.launches.append(rec)
        return hi, lo, kp

    def _tc_gemm(self, n, a, b, out, m, ncols, kdim, addr, label):
        """tcgen05 GEMM over split planes; split-K (+ a reduce pass) when the
        output has too few tiles to fill the GPU for a long K."""
        (ahi, alo, kpa), (bhi, blo, kpb) = a[:3], b[:3]
        a_mn = a[3] if len(a) > 3 else 0
        b_mn = b[3] if len(b) > 3 else 0
        splits = self._tc_splits(m, ncols, kdim)
        tiles = ((ncols + TC_TILE - 1) // TC_TILE) * ((m + TC_TILE - 1) // TC_TILE)
        kblocks = (kdim + 31) // 32
        ta = abi.TcArgs(M=m, N=ncols, K=kdim, kp_a=kpa, kp_b=kpb, a_ld_mn=a_mn, b_ld_mn=b_mn,
                        group_m=int(os.environ.get("GFB_TC_GROUP_M", "1")))
        target = out
        if splits > 1:
            per = ((kblocks + splits - 1) // splits) * 32
            splits = (kdim + per - 1) // per
            scratch = Buffer(self.new_key(), ElementType.F32, (splits, m, ncols), (m * ncols, ncols, 1))
            self.buf[("splitk", n)] = scratch
            ta.k_splits, ta.k_per_split, ta.split_stride = splits, per, m * ncols
            ta.c_sm, ta.c_sn = ncols, 1
            target = scratch
        else:
            for k_, v_ in addr.items():
                setattr(ta, k_, v_)
        return self._tc_gemm_emit(n, ahi, alo, bhi, blo, ta, target, out, m, ncols, kdim, splits, addr, label)

    @staticmethod
    def _tc_splits(m, ncols, kdim) -> int:
        """K splits of a tensor-core GEMM (see _tc_gemm)."""
        tiles = ((ncols + TC_TILE - 1) // TC_TILE) * ((m + TC_TILE - 1) // TC_TILE)
        kblocks = (kdim + 31) // 32
        splits = 1
        pair_tiles = ((ncols + 255) // 256) * ((m + 255) // 256)
        pairs = NUM_SMS // 2
        if (ncols >= 256 and m >= 256 and pair_tiles >= pairs and kblocks >= 64
                and os.environ.get("GFB_TC_PAIR", "1") == "1" and os.environ.get("GFB_TC_QSPLIT", "1") == "1"):
            # the persistent pair kernel runs pair_tiles / 74 waves; a weight
            # gradient (16 x 16 tiles of 256, K = the batch) is 3.46 waves, i.e.
            # 13 % idle in the last one: split K where that fills the waves
            # (the partials cost one extra pass over the output, ~1 % here)
            def fill(sp):
                w = pair_tiles * sp / pairs
                return w / -(-w // 1)
            splits = max((sp for sp in range(1, 5) if kblocks // sp >= 32), key=lambda sp: fill(sp) - 0.02 * (sp - 1))
        elif tiles < NUM_SMS and kblocks >= 64:
            splits = max(1, min((2 * NUM_SMS) // tiles, kblocks // 16))
        elif tiles <= 8 and kblocks >= 16:
            # a handful of tiles over a medium K (an MLP's first layer): spread K
            splits = max(1, min(NUM_SMS // tiles, kblocks // 4))
        return splits

    def _tc_gemm_emit(self, n, ahi, alo, bhi, blo, ta, target, out, m, ncols, kdim, splits, addr, label):
        a_mn, b_mn = ta.a_ld_mn, ta.b_ld_mn
        wide = ncols >= 256 and os.environ.get("GFB_TC_WIDE", "1") == "1"
        pair = wide and m >= 256 and os.environ.get("GFB_TC_PAIR", "1") == "1"
        if (a_mn or b_mn) and not pair:
            raise UnsupportedOp("MN-major tensor-core operands need the CTA-pair kernel")
        if pair:  # 2-SM CTA pairs, 256x256 tiles, persistent (gfb_gemm_tc2_kernel)
            kind, block, smem = abi.K_DOT_TC32P, 320, TC_SMEM_PAIR
            ntiles = ((ncols + 255) // 256) * ((m + 255) // 256) * splits
            pairs = NUM_SMS // 2 if os.environ.get("GFB_TC_PERSIST", "1") == "1" else ntiles
            grid = (2 * min(ntiles, pairs), 1, 1)
        elif wide:
            kind, block, smem = abi.K_DOT_TC32W, 320, TC_SMEM_W
            grid = ((ncols + 255) // 256, (m + TC_TILE - 1) // TC_TILE, splits)
        else:
            kind, block, smem = abi.K_DOT_TC32, 192, TC_SMEM
            grid = ((ncols + TC_TILE - 1) // TC_TILE, (m + TC_TILE - 1) // TC_TILE, splits)
        if grid[1] > 65535:
            raise UnsupportedOp(f"tensor-core GEMM with {m} rows exceeds the 65535-tile grid")
        reads, writes = [ahi.key, alo.key, bhi.key, blo.key], [target.key]
        refs = {"c": target, "a_hi": ahi, "a_lo": alo, "b_hi": bhi, "b_lo": blo}
        epi = self._epi.get(n) if hasattr(self, "_epi") else None
        if epi is not None:
            if not pair or splits > 1 or target.strides != (ncols, 1) or target.elem_off:
                raise UnsupportedOp(f"fused epilogue of Dot {n} needs the unsplit pair kernel and a dense output")
            ta.epi_kind = epi["kind"]
            for field, key in (("e_bias", "bias"), ("e_aux1", "aux1"), ("e_aux2", "aux2"), ("e_out2", "out2")):
                if key in epi:
                    b = self.buf[epi[key]]
                    refs[field] = b
                    (writes if field == "e_out2" else reads).append(b.key)
            ta.epi_flags = 1 if "out2" in epi else 0
            y = self.buf[epi["lo_of"]]
            root = self._dense_root(y)
            if root is not None and self._feeds_tc(epi["lo_of"]) and ("lo", root.key) not in self.buf:
                lo = Buffer(self.new_key(), ElementType.F32, root.shape, root.strides)
                self.buf[("lo", root.key)] = lo  # _lo_plane finds it: no separate pass
                refs["e_lo"] = lo
                writes.append(lo.key)
                ta.epi_flags |= 2
            label += ":epi" + ("bias_relu" if epi["kind"] == 1 else "relu_grad")
        rec = LaunchRec(kind, grid, (block, 1, 1), smem, ta, reads, writes, label)
        rec.flops = 2 * m * ncols * kdim
        rec.finalize = _finalize_refs(ta, refs)
        self.launches.append(rec)
        if splits > 1:
            # deterministic second pass: out[o] = sum over splits of scratch[z, o]
            p2 = Program(self, extents=(m * ncols, splits), vec_src=0, et=ElementType.F32)
            k = p2.leaf(target, [(1, 1, splits), (0, ncols, m), (0, 1, ncols)])  # the split-K scratch
            p2.emit(I_LOAD, k=k)
            p2.red_out = LeafSpec(out, _conv_out_digits(addr, m, ncols), True)
            p2.red_out.vec = vec_class(p2.red_out.digits, 0, True, vec_width(ElementType.F32), 4)
            self._col_launch(p2, m * ncols, splits, 1, label + ":splitk", ElementType.F32)
        return rec

    @staticmethod
    def _gather_ok(xb, xs, channels, m) -> bool:
        """The fused-gather conv kernel needs unit channel stride (NHWC
        storage) and 16-byte aligned runs of 4 channels."""
        return (os.environ.get("GFB_CONV_GATHER", "1") == "1" and xb.splat is None and xs[1] == 1
                and channels % 4 == 0 and all(v % 4 == 0 for v in (xs[0], xs[2], xs[3]))
                and xb.offset % 16 == 0 and (m + TC_TILE - 1) // TC_TILE <= 65535
                and max(abs(v) for v in xs) * 4 < 2 ** 62)

    @staticmethod
    def _generic_gather_ok(xb, xs) -> bool:
        """Element-gather conv kernel: 32-bit element offsets and a real buffer."""
        return (os.environ.get("GFB_CONV_GATHER", "1") == "1" and xb.splat is None
                and max(abs(v) for v in xs) * max(xb.shape) < 2 ** 30 and element_count(xb.shape) < 2 ** 31)

    @staticmethod
    def _wgrad_mn_ok(xb, xs, yb, ys, Cc, K) -> bool:
        """MN-major weight-gradient kernel: channel-last x and dy with channel
        counts and every stride multiples of 4 (16-byte pieces)."""
        return (os.environ.get("GFB_TCGW", "1") == "1" and xb.splat is None and yb.splat is None
                and xs[1] == 1 and ys[1] == 1 and Cc % 4 == 0 and K % 4 == 0
                and all(v % 4 == 0 for v in (xs[0], xs[2], xs[3], ys[0], ys[2], ys[3]))
                and max(abs(v) for v in xs) * max(xb.shape) < 2 ** 30 and element_count(xb.shape) < 2 ** 31
                and max(abs(v) for v in ys) * max(yb.shape) < 2 ** 30 and element_count(yb.shape) < 2 ** 31)

    def _conv_tcgw(self, n, xb, yb, out, m, ncols, kdim, geo, addr, label, real_c=None):
        """Weight gradient on gemm_tc.cu gfb_conv_tcgw_kernel (split-K over
        the pixels when the (r, s, c) x k tiles do not fill the GPU).  With
        `real_c`, the kernel's rows have zero-padded channels (geo E2) and the
        reduction pass writes only the first real_c of each tap."""
        bn = 64 if ncols <= 64 else 128
        kblocks = (kdim + 31) // 32
        tiles = ((ncols + bn - 1) // bn) * ((m + TC_TILE - 1) // TC_TILE)
        splits = 1
        if tiles < NUM_SMS and kblocks >= 64:
            splits = max(1, min((2 * NUM_SMS) // tiles, kblocks // 16))
        per = (kblocks + splits - 1) // splits
        splits = (kblocks + per - 1) // per
        ta = abi.TcgwArgs(M=m, N=ncols, K=kdim, **geo)
        target = out
        if splits > 1 or real_c is not None:
            scratch = Buffer(self.new_key(), ElementType.F32, (splits, m, ncols), (m * ncols, ncols, 1))
            self.buf[("splitk", n)] = scratch
            ta.k_splits, ta.kb_per_split, ta.split_stride = splits, per, m * ncols
            ta.c_sm, ta.c_sn = ncols, 1
            target = scratch
        else:
            ta.k_splits, ta.kb_per_split = 1, kblocks
            for k_, v_ in addr.items():
                setattr(ta, k_, v_)
        kind = abi.K_CONV_TCGW64 if bn == 64 else abi.K_CONV_TCGW128
        items = ((ncols + bn - 1) // bn) * ((m + TC_TILE - 1) // TC_TILE) * splits
        grid = (max(1, min(items, NUM_SMS)), 1, 1)
        rec = LaunchRec(kind, grid, (TCGW_THREADS[bn], 1, 1), TCGW_SMEM[bn], ta, [xb.key, yb.key], [target.key], label)
        rec.flops = 2 * m * ncols * kdim
        rec.algo_bytes = xb.nbytes + yb.nbytes + out.nbytes
        rec.finalize = _finalize_refs(ta, {"c": target, "a": xb, "b": yb})
        self.launches.append(rec)
        if real_c is not None:
            cp = geo["E2"]
            taps = m // cp
            mo = taps * real_c
            view = Buffer(scratch.key, ElementType.F32, (splits, taps, cp, ncols), (m * ncols, cp * ncols, ncols, 1),
                          scratch.slot, scratch.offset, None, base=scratch, elem_off=0)
            p2 = Program(self, extents=(mo * ncols, splits), vec_src=0, et=ElementType.F32)
            k = p2.leaf(view, [(1, 1, splits), (0, real_c * ncols, taps), (0, ncols, real_c), (0, 1, ncols)])
            p2.emit(I_LOAD, k=k)
            p2.red_out = LeafSpec(out, _conv_out_digits(addr, mo, ncols), True)
            p2.red_out.vec = vec_class(p2.red_out.digits, 0, True, vec_width(ElementType.F32), 4)
            self._col_launch(p2, mo * ncols, splits, 1, label + ":splitk", ElementType.F32)
        elif splits > 1:
            p2 = Program(self, extents=(m * ncols, splits), vec_src=0, et=ElementType.F32)
            k = p2.leaf(target, [(1, 1, splits), (0, ncols, m), (0, 1, ncols)])  # the split-K scratch
            p2.emit(I_LOAD, k=k)
            p2.red_out = LeafSpec(out, _conv_out_digits(addr, m, ncols), True)
            p2.red_out.vec = vec_class(p2.red_out.digits, 0, True, vec_width(ElementType.F32), 4)
            self._col_launch(p2, m * ncols, splits, 1, label + ":splitk", ElementType.F32)
        return rec

    @staticmethod
    def _tma_box_ok(xb, shape, sx, sy) -> bool:
        """TMA box gather: the activation needs a fixed (arena) address for
        its tensor map, and the strided box must fit the 256-element limit."""
        return (os.environ.get("GFB_CONV_TMA", "1") == "1" and xb.slot == abi.SLOT_ARENA
                and sx <= 2 and sy <= 2 and max(shape) < 2 ** 31)

    @staticmethod
    def _tcxh_ok(xb, xs, shape, sx, sy) -> bool:
        """2xFP16 TMA-box convolution (conv_f16.cu): a dense channel-last
        activation with a power-of-two channel count, 64 <= C <= 1024."""
        N_, C_, H_, W_ = shape
        return (use_f16() and os.environ.get("GFB_CONV_F16", "1") == "1" and xb.splat is None and xb.elem_off == 0
                and C_ >= 64 and C_ <= 1024 and C_ & (C_ - 1) == 0 and tuple(xs) == (H_ * W_ * C_, 1, W_ * C_, C_)
                and sx <= 2 and sy <= 2 and N_ * H_ * W_ * C_ < 2 ** 31)

    def _ch_planes(self, xb, P, C):
        """Channel-scaled fp16 planes of a dense channel-last activation
        [P, C] (gfb_chmax_kernel + gfb_chsplit_kernel), shared by every
        convolution that reads it."""
        root = xb.base if xb.base is not None else xb
        key = ("ch16", root.key)
        got = self.buf.get(key + ("hi",))
        if got is not None:
            return got, self.buf[key + ("lo",)], self.buf[key + ("sc",)]
        part = Buffer(self.new_key(), ElementType.F32, (C,), (1,))
        sc = Buffer(self.new_key(), ElementType.F32, (C,), (1,))
        hi = Buffer(self.new_key(), ElementType.F32, ((P * C + 1) // 2,), (1,))
        lo = Buffer(self.new_key(), ElementType.F32, ((P * C + 1) // 2,), (1,))
        for p_, b_ in (("part", part), ("sc", sc), ("hi", hi), ("lo", lo)):
            self.buf[key + (p_,)] = b_
        a0 = abi.MemsetArgs(bytes=C * 4)
        r0 = LaunchRec(abi.K_MEMSET, (1, 1, 1), (1, 1, 1), 0, a0, [], [part.key], f"memset#{root.key}")
        r0.finalize = _finalize_refs(a0, {"buf": part})
        self.launches.append(r0)
        nb = max(1, min(CHMAX_BLOCKS, (P * (C // 4)) // (256 * 16)))  # >= 16 rows of float4 per thread
        a1 = abi.ChsplitArgs(P=P, C=C, nblocks=nb)
        r1 = LaunchRec(abi.K_CHMAX, (nb, 1, 1), (256, 1, 1), 0, a1, [xb.key, part.key], [part.key],
                       f"chmax#{root.key}")
        r1.algo_bytes = P * C * 4
        r1.finalize = _finalize_refs(a1, {"src": xb, "partial": part})
        self.launches.append(r1)
        a3 = abi.ChsplitArgs(P=P, C=C, nblocks=CHMAX_BLOCKS)
        grid = max(1, min(NUM_SMS * 8, (P * (C // 4) + 255) // 256))
        r3 = LaunchRec(abi.K_CHSPLIT, (grid, 1, 1), (256, 1, 1), 0, a3, [xb.key, part.key], [sc.key, hi.key, lo.key],
                       f"chsplit#{root.key}")
        r3.algo_bytes = P * C * 8
        r3.finalize = _finalize_refs(a3, {"src": xb, "partial": part, "sc": sc, "hi": hi, "lo": lo})
        self.launches.append(r3)
        return hi, lo, sc

    def _conv_tcxh(self, n, xb, xshape, wb, wgeo, out, oshape, ncols, kdim, geo, label):
        """Conv2D / ConvBackpropData on conv_f16.cu gfb_conv_tcxh_kernel: the
        activation's channel-scaled fp16 planes by TMA pixel boxes, filter
        planes divided by the same channel scales (rows scaled on their own,
        undone in the epilogue).  wgeo = (row stride, e0, e1, e2, t0, t1, t2)
        of the filter gather, e2 / t2 along the activation's channels."""
        N_, C_, H_, W_ = xshape
        ahi, alo, sc = self._ch_planes(xb, N_ * H_ * W_, C_)
        s_r, e0, e1, e2, t0, t1, t2 = wgeo
        bhi = Buffer(self.new_key(), ElementType.F32, ((ncols * kdim + 1) // 2,), (1,))
        blo = Buffer(self.new_key(), ElementType.F32, ((ncols * kdim + 1) // 2,), (1,))
        binv = Buffer(self.new_key(), ElementType.F32, (ncols,), (1,))
        for p_, b_ in (("hi", bhi), ("lo", blo), ("inv", binv)):
            self.buf[("fsplit", n, p_)] = b_
        fa = abi.FsplitArgs(rows=ncols, K=kdim, s_r=s_r, e0=e0, e1=e1, e2=e2, t0=t0, t1=t1, t2=t2)
        fr = LaunchRec(abi.K_FSPLIT, (ncols, 1, 1), (256, 1, 1), 0, fa, [wb.key, sc.key], [bhi.key, blo.key, binv.key],
                       f"fsplit#{n}")
        fr.algo_bytes = ncols * kdim * 8
        fr.finalize = _finalize_refs(fa, {"w": wb, "sc": sc, "hi": bhi, "lo": blo, "inv": binv})
        self.launches.append(fr)
        No, Yo, Xo = oshape
        BX = min(128, 1 << max(0, (Xo - 1).bit_length()))
        BY = min(128 // BX, 1 << max(0, (Yo - 1).bit_length()))
        BNI = 128 // (BX * BY)
        tiles_x, tiles_y = (Xo + BX - 1) // BX, (Yo + BY - 1) // BY
        tiles = tiles_x * tiles_y * ((No + BNI - 1) // BNI)
        os_ = out.strides
        ta = abi.TcxhArgs(N=ncols, K=kdim, o_n=os_[0], o_y=os_[2], o_x=os_[3], c_sn=os_[1], No=No, Yo=Yo, Xo=Xo,
                          BX=BX, BY=BY, BNI=BNI, tiles_x=tiles_x, tiles_y=tiles_y, **geo)
        ta.a_dims[:] = [C_, W_, H_, N_]
        ta.a_strides[:] = [1, C_, W_ * C_, H_ * W_ * C_]
        bn = 64 if ncols <= 64 else 128
        kind = abi.K_CONV_TCXH64 if bn == 64 else abi.K_CONV_TCXH128
        grid = (max(1, min(tiles * ((ncols + bn - 1) // bn), NUM_SMS)), 1, 1)
        rec = LaunchRec(kind, grid, (192, 1, 1), TCXH_SMEM[bn], ta, [ahi.key, alo.key, bhi.key, blo.key, binv.key],
                        [out.key], label)
        rec.flops = 2 * No * Yo * Xo * ncols * kdim
        rec.algo_bytes = xb.nbytes + wb.nbytes + out.nbytes
        rec.finalize = _finalize_refs(ta, {"c": out, "a_hi": ahi, "a_lo": alo, "b_hi": bhi, "b_lo": blo, "b_inv": binv})
        self.launches.append(rec)

    def _conv_tcgwh(self, n, xb, xshape, yb, yshape, out, R, S, pt, pl, label):
        """ConvBackpropFilter on conv_f16.cu gfb_conv_tcgwh_kernel: the fp16
        planes of x and dy (shared with the forward / data-gradient
        convolutions that read them) by TMA boxes of 64 output pixels, rows
        (r, s, c), split-K over the pixel boxes (+ the reduce pass)."""
        N_, C_, H_, W_ = xshape
        _, K_, Ho, Wo = yshape
        ahi, alo, asc = self._ch_planes(xb, N_ * H_ * W_, C_)
        bhi, blo, bsc = self._ch_planes(yb, N_ * Ho * Wo, K_)
        m, ncols = R * S * C_, K_
        BX = min(64, 1 << max(0, (Wo - 1).bit_length()))
        BY = min(64 // BX, 1 << max(0, (Ho - 1).bit_length()))
        BNI = 64 // (BX * BY)
        tiles_x, tiles_y = (Wo + BX - 1) // BX, (Ho + BY - 1) // BY
        nbox = tiles_x * tiles_y * ((N_ + BNI - 1) // BNI)
        bn = 64 if ncols <= 64 else 128
        tiles = ((m + 127) // 128) * ((ncols + bn - 1) // bn)
        splits = max(1, min(max(1, nbox // 16), -(-2 * NUM_SMS // tiles)))
        per = -(-nbox // splits)
        splits = -(-nbox // per)
        os_ = out.strides
        addr = {"c_rdiv": C_, "c_s_hi": os_[3], "c_s_lo": os_[1], "c_sn": os_[0]}
        ta = abi.TcgwhArgs(M=m, N=ncols, C=C_, S=S, pt=pt, pl=pl, c_s_hi=os_[3], c_s_lo=os_[1], c_sn=os_[0],
                           k_splits=splits, boxes_per_split=per, No=N_, Yo=Ho, Xo=Wo, BX=BX, BY=BY, BNI=BNI,
                           tiles_x=tiles_x, tiles_y=tiles_y)
        ta.a_dims[:] = [C_, W_, H_, N_]
        ta.a_strides[:] = [1, C_, W_ * C_, H_ * W_ * C_]
        ta.b_dims[:] = [K_, Wo, Ho, N_]
        ta.b_strides[:] = [1, K_, Wo * K_, Ho * Wo * K_]
        target = out
        if splits > 1:
            scratch = Buffer(self.new_key(), ElementType.F32, (splits, m, ncols), (m * ncols, ncols, 1))
            self.buf[("splitk", n)] = scratch
            ta.split_stride = m * ncols
            target = scratch
        kind = abi.K_CONV_TCGWH64 if bn == 64 else abi.K_CONV_TCGWH128
        grid = (max(1, min(tiles * splits, NUM_SMS)), 1, 1)
        rec = LaunchRec(kind, grid, (192, 1, 1), TCGWH_SMEM[bn], ta, [ahi.key, alo.key, asc.key, bhi.key, blo.key, bsc.key],
                        [target.key], label)
        rec.flops = 2 * m * ncols * N_ * Ho * Wo
        rec.algo_bytes = xb.nbytes + yb.nbytes + out.nbytes
        rec.finalize = _finalize_refs(ta, {"c": target, "a_hi": ahi, "a_lo": alo, "b_hi": bhi, "b_lo": blo, "a_sc": asc,
                                           "b_sc": bsc})
        self.launches.append(rec)
        if splits > 1:
            p2 = Program(self, extents=(m * ncols, splits), vec_src=0, et=ElementType.F32)
            k = p2.leaf(target, [(1, 1, splits), (0, ncols, m), (0, 1, ncols)])
            p2.emit(I_LOAD, k=k)
            p2.red_out = LeafSpec(out, _conv_out_digits(addr, m, ncols), True)
            p2.red_out.vec = vec_class(p2.red_out.digits, 0, True, vec_width(ElementType.F32), 4)
            self._col_launch(p2, m * ncols, splits, 1, label + ":splitk", ElementType.F32)
        return rec

    def _conv_tcx(self, n, xb, xs, xshape, b, out, oshape, ncols, kdim, geo, yb, label):
        """Conv2D / ConvBackpropData whose A tiles are TMA boxes of output
        pixels (gemm_tc.cu, gfb_conv_tcx_kernel)."""
        bhi, blo, _ = b
        No, Yo, Xo = oshape
        BX = min(128, 1 << max(0, (Xo - 1).bit_length()))
        BY = min(128 // BX, 1 << max(0, (Yo - 1).bit_length()))
        BNI = 128 // (BX * BY)
        tiles_x, tiles_y = (Xo + BX - 1) // BX, (Yo + BY - 1) // BY
        tiles = tiles_x * tiles_y * ((No + BNI - 1) // BNI)
        os_ = out.strides
        N_, C_, H_, W_ = xshape
        ta = abi.TcxArgs(N=ncols, K=kdim, o_n=os_[0], o_y=os_[2], o_x=os_[3], c_sn=os_[1], No=No, Yo=Yo, Xo=Xo,
                         BX=BX, BY=BY, BNI=BNI, tiles_x=tiles_x, tiles_y=tiles_y, **geo)
        ta.pad0 = 1 if os.environ.get("GFB_TCX_RAWHI") == "1" else 0  # experiment: MMA reads raw fp32 as hi
        ta.a_dims[:] = [C_, W_, H_, N_]
        ta.a_strides[:] = [xs[1], xs[3], xs[2], xs[0]]
        bn = 64 if ncols <= 64 else 128
        kind = abi.K_CONV_TCX64 if bn == 64 else abi.K_CONV_TCX128
        # persistent: one CTA per SM walks the (column tile, pixel tile) items
        grid = (max(1, min(tiles * ((ncols + bn - 1) // bn), NUM_SMS)), 1, 1)
        rec = LaunchRec(kind, grid, (320, 1, 1), TCX_SMEM[bn], ta, [xb.key, bhi.key, blo.key], [out.key], label)
        rec.flops = 2 * No * Yo * Xo * ncols * kdim
        rec.algo_bytes = xb.nbytes + yb.nbytes + out.nbytes
        rec.finalize = _finalize_refs(ta, {"c": out, "a": xb, "b_hi": bhi, "b_lo": blo})
        self.launches.append(rec)

    def _conv_stem(self, n, xb, xs, b, out, m, ncols, kdim, geo, yb, label):
        """Few-channel forward convolution on gemm_tc.cu gfb_conv_stem_kernel
        (persistent over 8x16 output-pixel tiles)."""
        bhi, blo, kp = b
        ta = abi.TcgArgs(M=m, N=ncols, K=kdim, xs0=xs[0], xs2=xs[2], xs3=xs[3], **geo)
        ta.pad[0], ta.pad[1] = xs[1], kp  # channel stride of x, filter-plane pitch
        tiles = (m // (geo["Y"] * geo["X"])) * ((geo["Y"] + 7) // 8) * ((geo["X"] + 15) // 16)
        grid = (max(1, min(tiles, NUM_SMS)), 1, 1)
        rec = LaunchRec(abi.K_CONV_STEM64, grid, (STEM_THREADS, 1, 1), STEM_SMEM, ta, [xb.key, bhi.key, blo.key],
                        [out.key], label)
        rec.flops = 2 * m * ncols * kdim
        rec.algo_bytes = xb.nbytes + yb.nbytes + out.nbytes
        rec.finalize = _finalize_refs(ta, {"c": out, "a": xb, "b_hi": bhi, "b_lo": blo})
        self.launches.append(rec)

    def _conv_stemh(self, n, xb, xs, yb, ys, out, m, ncols, kdim, geo, label):
        """Few-channel forward convolution in 2xFP16 on conv_f16.cu
        gfb_conv_stemh_kernel (persistent over 4x32 output-pixel tiles; reads
        x and the fp32 filter directly, no split launches)."""
        ta = abi.StemhArgs(M=m, N=ncols, K=kdim, xs0=xs[0], xs1=xs[1], xs2=xs[2], xs3=xs[3],
                           ws0=ys[0], ws1=ys[1], ws2=ys[2], ws3=ys[3], **geo)
        refs, writes = {"c": out, "a": xb, "w": yb}, [out.key]
        r = self._conv_relu.get(n)
        if r is not None and self.buf[r].strides == out.strides and self.buf[r].et is out.et:
            refs["c2"], ta.flags = self.buf[r], 1  # Relu(y) from the epilogue
            writes.append(self.buf[r].key)
            self._conv_relu_done.add(n)
        tiles = (m // (geo["Y"] * geo["X"])) * ((geo["Y"] + 3) // 4) * ((geo["X"] + 31) // 32)
        grid = (max(1, min(tiles, NUM_SMS)), 1, 1)
        # the 3-channel 7x7 stem: a build with immediate gather offsets
        kind = abi.K_CONV_STEMH_C3R7 if (geo["C"], kdim // geo["C"] // geo["S"], geo["S"]) == (3, 7, 7) else abi.K_CONV_STEMH
        rec = LaunchRec(kind, grid, (STEM_THREADS, 1, 1), STEMH_SMEM, ta, [xb.key, yb.key], writes, label)
        rec.flops = 2 * m * ncols * kdim
        rec.algo_bytes = xb.nbytes + yb.nbytes + out.nbytes * len(writes)
        rec.finalize = _finalize_refs(ta, refs)
        self.launches.append(rec)

    def _conv_stemwh(self, n, xb, xs, yb, ys, out, xshape, oshape, pt, pl, addr, label):
        """The 3-channel 7x7 weight gradient on conv_f16.cu
        gfb_conv_stemwh_kernel: every CTA reduces a contiguous range of
        2 x 32 output-pixel tiles into its own [K, 64] partial; a second pass
        sums the partials in CTA order into dW."""
        N_, Cc, H, W = xshape
        Ho, Wo = oshape
        kdim, ncols = Cc * 49, 64
        tiles = N_ * ((Ho + 1) // 2) * ((Wo + 31) // 32)
        grid = max(1, min(tiles, NUM_SMS))
        scratch = Buffer(self.new_key(), ElementType.F32, (grid, kdim, ncols), (kdim * ncols, ncols, 1))
        self.buf[("splitk", n)] = scratch
        ta = abi.StemhArgs(M=N_ * Ho * Wo, N=ncols, K=kdim, xs0=xs[0], xs1=xs[1], xs2=xs[2], xs3=xs[3],
                           ws0=ys[0], ws1=ys[1], ws2=ys[2], ws3=ys[3], Y=Ho, X=Wo, oy=-pt, ox=-pl, H=H, W=W, S=7, C=Cc)
        rec = LaunchRec(abi.K_CONV_STEMWH_C3R7, (grid, 1, 1), (STEMWH_THREADS, 1, 1), STEMWH_SMEM, ta, [xb.key, yb.key],
                        [scratch.key], label)
        rec.flops = 2 * N_ * Ho * Wo * ncols * kdim
        rec.algo_bytes = xb.nbytes + yb.nbytes + out.nbytes
        rec.finalize = _finalize_refs(ta, {"c": scratch, "a": xb, "w": yb})
        self.launches.append(rec)
        p2 = Program(self, extents=(kdim * ncols, grid), vec_src=0, et=ElementType.F32)
        k = p2.leaf(scratch, [(1, 1, grid), (0, ncols, kdim), (0, 1, ncols)])
        p2.emit(I_LOAD, k=k)
        p2.red_out = LeafSpec(out, _conv_out_digits(addr, kdim, ncols), True)
        p2.red_out.vec = vec_class(p2.red_out.digits, 0, True, vec_width(ElementType.F32), 4)
        self._col_launch(p2, kdim * ncols, grid, 1, label + ":splitk", ElementType.F32)

    def _conv_tcg(self, n, xb, xs, b, out, m, ncols, kdim, geo, addr, yb, label):
        """Conv2D / ConvBackpropData with the activation gather and TF32
        split inside the tensor-core kernel (gemm_tc.cu, gfb_conv_tcg_kernel)."""
        bhi, blo, _ = b
        bn = 64 if ncols <= 64 else 128
        ta = abi.TcgArgs(M=m, N=ncols, K=kdim, xs0=xs[0], xs2=xs[2], xs3=xs[3], c_sm=0, **addr, **geo)
        kind = abi.K_CONV_TCG64 if bn == 64 else abi.K_CONV_TCG128
        # persistent: one CTA per SM walks the (column tile, row tile) items
        grid = (max(1, min(((ncols + bn - 1) // bn) * ((m + TC_TILE - 1) // TC_TILE), NUM_SMS)), 1, 1)
        rec = LaunchRec(kind, grid, (320, 1, 1), TCG_SMEM[bn], ta, [xb.key, bhi.key, blo.key], [out.key], label)
        rec.flops = 2 * m * ncols * kdim
        rec.algo_bytes = xb.nbytes + yb.nbytes + out.nbytes
        rec.finalize = _finalize_refs(ta, {"c": out, "a": xb, "b_hi": bhi, "b_lo": blo})
        self.launches.append(rec)

    def _conv_tcgg(self, n, xb, b, out, m, ncols, kdim, geo, addr, yb, label):
        """Implicit-GEMM convolution whose A operand is gathered element-wise
        inside the tensor-core kernel (gemm_tc.cu, gfb_conv_tcgg_kernel):
        any channel count, any layout, and weight gradients (split-K)."""
        bhi, blo, kpb = b
        bn = 64 if ncols <= 64 else 128
        kblocks = (kdim + 31) // 32
        tiles = ((ncols + bn - 1) // bn) * ((m + TC_TILE - 1) // TC_TILE)
        splits = 1
        if tiles < NUM_SMS and kblocks >= 64:
            splits = max(1, min((2 * NUM_SMS) // tiles, kblocks // 16))
        per = (kblocks + splits - 1) // splits
        splits = (kblocks + per - 1) // per
        ta = abi.TcggArgs(M=m, N=ncols, K=kdim, Kp=kblocks * 32, kp_b=kpb, **geo)
        target = out
        if splits > 1:
            scratch = Buffer(self.new_key(), ElementType.F32, (splits, m, ncols), (m * ncols, ncols, 1))
            self.buf[("splitk", n)] = scratch
            ta.k_splits, ta.kb_per_split, ta.split_stride = splits, per, m * ncols
            ta.c_sm, ta.c_sn = ncols, 1
            target = scratch
        else:
            ta.k_splits, ta.kb_per_split = 1, kblocks
            for k_, v_ in addr.items():
                setattr(ta, k_, v_)
        kind = abi.K_CONV_TCGG64 if bn == 64 else abi.K_CONV_TCGG128
        # persistent: one CTA per SM walks the (n tile, m tile, split) items
        items = ((ncols + bn - 1) // bn) * ((m + TC_TILE - 1) // TC_TILE) * splits
        grid = (max(1, min(items, NUM_SMS)), 1, 1)
        rec = LaunchRec(kind, grid, (TCGG_THREADS[bn], 1, 1), TCG_SMEM[bn], ta, [xb.key, bhi.key, blo.key], [target.key], label)
        rec.flops = 2 * m * ncols * kdim
        rec.algo_bytes = xb.nbytes + yb.nbytes + out.nbytes
        rec.finalize = _finalize_refs(ta, {"c": target, "a": xb, "b_hi": bhi, "b_lo": blo})
        self.launches.append(rec)
        if splits > 1:
            p2 = Program(self, extents=(m * ncols, splits), vec_src=0, et=ElementType.F32)
            k = p2.leaf(target, [(1, 1, splits), (0, ncols, m), (0, 1, ncols)])  # the split-K scratch
            p2.emit(I_LOAD, k=k)
            p2.red_out = LeafSpec(out, _conv_out_digits(addr, m, ncols), True)
            p2.red_out.vec = vec_class(p2.red_out.digits, 0, True, vec_width(ElementType.F32), 4)
            self._col_launch(p2, m * ncols, splits, 1, label + ":splitk", ElementType.F32)
        return rec

    def emit_conv_tc(self, n) -> bool:
        """Conv2D / ConvBackpropData / ConvBackpropFilter as implicit GEMMs on
        the tensor cores; returns False when the shape or layout does not fit
        (the exact-order SIMT kernel then runs)."""
        node = self.nodes[n]
        if node.output.element_type is not ElementType.F32 or os.environ.get("GFB_CONV", "auto") == "simt":
            return False
        if node.op in (OpKind.MAX_POOL, OpKind.MAX_POOL_BACKPROP):
            return False
        if node.op is not OpKind.CONV2D and conv_strides(node) != (1, 1):
            return False  # strided gradients (IR extension): the exact-order kernel
        x, y = node.inputs[0][0], node.inputs[1][0]
        try:
            (xb, xs), (yb, ys) = self.operand(x), self.operand(y)
        except _Retry:
            raise
        out = self.buf[n]
        os_ = out.strides
        pt, _, pl, _ = node.attrs["padding"]
        xshape, yshape, oshape = self.nodes[x].output.shape, self.nodes[y].output.shape, node.output.shape
        force = os.environ.get("GFB_CONV", "auto") == "tc"
        if node.op is OpKind.CONV2D:
            N, Cc, H, W = xshape
            K, _, R, S = yshape
            Ho, Wo = oshape[2], oshape[3]
            sh, sw = node.attrs["strides"]
            m, ncols, kdim = N * Ho * Wo, K, Cc * R * S
            if os_[2] != Wo * os_[3] or not (force or _conv_tc_ok(m, ncols, kdim)):
                return False
            if (Cc < 16 and ncols <= 64 and kdim <= 192 and (sh, sw) == (1, 1) and xb.splat is None and yb.splat is None
                    and (4 + R - 1) * (32 + S - 1) * Cc + 3 * (32 + S - 1) + 32 <= 1536  # 4x32 tile patch + zero pad
                    and os.environ.get("GFB_CONV_STEM", "1") == "1"
                    and os.environ.get("GFB_CONV_F16", "1") == "1"
                    and ((Cc, R, S) == (3, 7, 7) or kdim > 160 or os.environ.get("GFB_STEMH_ALL", "0") == "1")
                    and max(abs(v) for v in xs) * max(xb.shape) < 2 ** 62):
                # the same tiles in 2xFP16 (conv_f16.cu gfb_conv_stemh_kernel): per-tile
                # activation scales, the filter split inside the kernel.  For the
                # 3-channel 7x7 stem (and K > 160); smaller few-channel layers (config
                # C's 3x3 x 16 columns: 4x the MMA work at N = 64, a short walk per CTA)
                # stay on the TF32 stem kernel, 0.039 vs 0.058 ms
                self._conv_stemh(n, xb, xs, yb, ys, out, m, ncols, kdim,
                                 dict(Y=Ho, X=Wo, oy=-pt, ox=-pl, H=H, W=W, S=S, C=Cc,
                                      c_s_hi=os_[0], c_sm=os_[2], c_s_lo=os_[3], c_sn=os_[1]),
                                 f"{node.op.wire_name}_stemh#{n}")
                return True
            if (Cc < 16 and ncols <= 64 and kdim <= 160 and (sh, sw) == (1, 1) and xb.splat is None
                    and (8 + R - 1) * (16 + S - 1) * Cc <= 1536 and os.environ.get("GFB_CONV_STEM", "1") == "1"
                    and max(abs(v) for v in xs) * max(xb.shape) < 2 ** 62):
                # few input channels (the ResNet stem): 8x16 pixel tiles built from a
                # shared-memory input patch, the filter resident (gemm_tc.cu gfb_conv_stem_kernel)
                b = self._split(n, "b", yb, ncols, kdim, 3, s_r=ys[0], geo=(0,) * 12 + (R, S, Cc), st=(ys[2], ys[3], ys[1]))
                self._conv_stem(n, xb, xs, b, out, m, ncols, kdim,
                                dict(Y=Ho, X=Wo, sy=1, sx=1, oy=-pt, ox=-pl, H=H, W=W, S=S, C=Cc, ksign=1,
                                     c_s_hi=os_[0], c_sm=os_[2], c_s_lo=os_[3], c_sn=os_[1]),
                                yb, f"{node.op.wire_name}_stem#{n}")
                return True
            if (Cc % 4 and Cc < 32 and xb.splat is None and yb.splat is None and ncols >= 32
                    and os.environ.get("GFB_PAD_CHANNELS_FWD", "0") == "1"):
                # (measured no faster than the element gather for the 3-channel stem: off by default)
                # few channels (the 3-channel stem): zero-padded channel-last copies of the
                # input (shared with its weight gradient) and of the filter feed the 16-byte gather
                cp = align_up(Cc, 4)
                xb, xs = self._pad_channels(xb, xs, (N, Cc, H, W), cp)
                yb, ys = self._pad_channels(yb, ys, (K, Cc, R, S), cp)
                Cc, kdim = cp, cp * R * S
            if self._gather_ok(xb, xs, Cc, m):
                if self._tcxh_ok(xb, xs, (N, Cc, H, W), sw, sh):
                    self._conv_tcxh(n, xb, (N, Cc, H, W), yb, (ys[0], R, S, Cc, ys[2], ys[3], ys[1]), out, (N, Ho, Wo),
                                    ncols, kdim, dict(sx=sw, sy=sh, ox=-pl, oy=-pt, S=S, CB=Cc // 64, ksign=1),
                                    f"{node.op.wire_name}_tcxh#{n}")
                    return True
                b = self._split(n, "b", yb, ncols, kdim, 3, s_r=ys[0], geo=(0,) * 12 + (R, S, Cc), st=(ys[2], ys[3], ys[1]))
                if Cc % 32 == 0 and self._tma_box_ok(xb, (N, Cc, H, W), sw, sh):
                    self._conv_tcx(n, xb, xs, (N, Cc, H, W), b, out, (N, Ho, Wo), ncols, kdim,
                                   dict(sx=sw, sy=sh, ox=-pl, oy=-pt, S=S, CB=Cc // 32, ksign=1), yb,
                                   f"{node.op.wire_name}_tcx#{n}")
                    return True
                self._conv_tcg(n, xb, xs, b, out, m, ncols, kdim, dict(Y=Ho, X=Wo, sy=sh, sx=sw, oy=-pt, ox=-pl, H=H, W=W, S=S,
                               CB=Cc // 32, C=Cc, ksign=1), {"c_rdiv": Ho * Wo, "c_s_hi": os_[0], "c_s_lo": os_[3], "c_sn": os_[1]},
                               yb, f"{node.op.wire_name}_tcg#{n}")
                return True
            addr = {"c_rdiv": Ho * Wo, "c_s_hi": os_[0], "c_s_lo": os_[3], "c_sn": os_[1]}
            if self._generic_gather_ok(xb, xs):
                b = self._split(n, "b", yb, ncols, kdim, 3, s_r=ys[0], geo=(0,) * 12 + (Cc, R, S), st=ys[1:])
                geo = dict(E1=Ho, E2=Wo, ro0=xs[0], ro1=sh * xs[2], ro2=sw * xs[3], hm=sh, wm=sw, h0=0, w0=0, H=H, W=W,
                           Ke1=R, Ke2=S, ko0=xs[1], ko1=xs[2], ko2=xs[3], kbase=-pt * xs[2] - pl * xs[3],
                           kh=1, kw=1, dh0=-pt, dw0=-pl)
                self._conv_tcgg(n, xb, b, out, m, ncols, kdim, geo, addr, yb, f"{node.op.wire_name}_tcgg#{n}")
                return True
            geo = (N, Cc, H, W, R, S, Ho, Wo, sh, sw, pt, pl)
            a = self._split(n, "a", xb, m, kdim, 1, geo=geo, st=xs)
            b = self._split(n, "b", yb, ncols, kdim, 3, s_r=ys[0], geo=(0,) * 12 + (Cc, R, S), st=ys[1:])
        elif node.op is OpKind.CONV_BACKPROP_DATA:
            N, K, Ho, Wo = xshape
            _, Cc, R, S = yshape
            H, W = oshape[2], oshape[3]
            m, ncols, kdim = N * H * W, Cc, K * R * S
            if os_[2] != W * os_[3] or not (force or _conv_tc_ok(m, ncols, kdim)):
                return False
            if self._gather_ok(xb, xs, K, m):
                if self._tcxh_ok(xb, xs, (N, K, Ho, Wo), 1, 1):
                    self._conv_tcxh(n, xb, (N, K, Ho, Wo), yb, (ys[1], R, S, K, ys[2], ys[3], ys[0]), out, (N, H, W),
                                    ncols, kdim, dict(sx=1, sy=1, ox=pl, oy=pt, S=S, CB=K // 64, ksign=-1),
                                    f"{node.op.wire_name}_tcxh#{n}")
                    return True
                b = self._split(n, "b", yb, ncols, kdim, 3, s_r=ys[1], geo=(0,) * 12 + (R, S, K), st=(ys[2], ys[3], ys[0]))
                if K % 32 == 0 and self._tma_box_ok(xb, (N, K, Ho, Wo), 1, 1):
                    self._conv_tcx(n, xb, xs, (N, K, Ho, Wo), b, out, (N, H, W), ncols, kdim,
                                   dict(sx=1, sy=1, ox=pl, oy=pt, S=S, CB=K // 32, ksign=-1), yb,
                                   f"{node.op.wire_name}_tcx#{n}")
                    return True
                self._conv_tcg(n, xb, xs, b, out, m, ncols, kdim, dict(Y=H, X=W, sy=1, sx=1, oy=pt, ox=pl, H=Ho, W=Wo, S=S,
                               CB=K // 32, C=K, ksign=-1), {"c_rdiv": H * W, "c_s_hi": os_[0], "c_s_lo": os_[3], "c_sn": os_[1]},
                               yb, f"{node.op.wire_name}_tcg#{n}")
                return True
            addr = {"c_rdiv": H * W, "c_s_hi": os_[0], "c_s_lo": os_[3], "c_sn": os_[1]}
            if self._generic_gather_ok(xb, xs):
                b = self._split(n, "b", yb, ncols, kdim, 3, s_r=ys[1], geo=(0,) * 12 + (K, R, S), st=(ys[0], ys[2], ys[3]))
                geo = dict(E1=H, E2=W, ro0=xs[0], ro1=xs[2], ro2=xs[3], hm=1, wm=1, h0=0, w0=0, H=Ho, W=Wo,
                           Ke1=R, Ke2=S, ko0=xs[1], ko1=-xs[2], ko2=-xs[3], kbase=pt * xs[2] + pl * xs[3],
                           kh=-1, kw=-1, dh0=pt, dw0=pl)
                self._conv_tcgg(n, xb, b, out, m, ncols, kdim, geo, addr, yb, f"{node.op.wire_name}_tcgg#{n}")
                return True
            geo = (N, K, H, W, R, S, Ho, Wo, 1, 1, pt, pl)
            a = self._split(n, "a", xb, m, kdim, 2, geo=geo, st=xs)
            b = self._split(n, "b", yb, ncols, kdim, 3, s_r=ys[1], geo=(0,) * 12 + (K, R, S), st=(ys[0], ys[2], ys[3]))
        else:
            N, Cc, H, W = xshape
            _, K, Ho, Wo = yshape
            R, S = oshape[2], oshape[3]
            m, ncols, kdim = K, Cc * R * S, N * Ho * Wo
            if os_[1] != R * S * os_[3] or os_[2] != S * os_[3] or not (force or _conv_tc_ok(m, ncols, kdim)):
                return False
            if ((Cc, R, S, K) == (3, 7, 7, 64) and xb.splat is None and yb.splat is None and ys[1] == 1
                    and all(v % 4 == 0 for v in (ys[0], ys[2], ys[3])) and yb.elem_off % 4 == 0
                    and os.environ.get("GFB_CONV_F16", "1") == "1" and os.environ.get("GFB_CONV_STEM", "1") == "1"
                    and max(abs(v) for v in xs) * max(xb.shape) < 2 ** 62 and max(abs(v) for v in ys) * max(yb.shape) < 2 ** 62):
                # the 3-channel 7x7 stem's dW: 2xFP16 on the forward's patch tiles
                # (conv_f16.cu gfb_conv_stemwh_kernel), per-CTA partials + a reduction
                self._conv_stemwh(n, xb, xs, yb, ys, out, (N, Cc, H, W), (Ho, Wo), pt, pl,
                                  {"c_rdiv": Cc, "c_s_hi": os_[3], "c_s_lo": os_[1], "c_sn": os_[0]},
                                  f"{node.op.wire_name}_stemwh#{n}")
                return True
            real_c = None
            if (Cc % 4 and Cc < 32 and xb.splat is None and os.environ.get("GFB_PAD_CHANNELS", "1") == "1"
                    and self._wgrad_mn_ok(xb, (4 * H * W, 1, 4 * W, 4), yb, ys, 4, K)):
                # few channels (the 3-channel stem): a zero-padded channel-last copy of x
                # lets the MN-major kernel run; the padded rows of dW are dropped
                real_c = Cc
                xb, xs = self._pad_channels(xb, xs, (N, Cc, H, W), align_up(Cc, 4))
                Cc = align_up(Cc, 4)
            if self._generic_gather_ok(xb, xs):
                # rows (c, r, s) of the gathered data, columns = output channels
                b = None if self._wgrad_mn_ok(xb, xs, yb, ys, Cc, K) else self._split(
                    n, "b", yb, K, kdim, 3, s_r=ys[1], geo=(0,) * 12 + (N, Ho, Wo), st=(ys[0], ys[2], ys[3]))
                kgeo = dict(Ke1=Ho, Ke2=Wo, ko0=xs[0], ko1=xs[2], ko2=xs[3], kbase=-pt * xs[2] - pl * xs[3],
                            kh=1, kw=1, dh0=0, dw0=0)
                if (real_c is None and self._tcxh_ok(xb, xs, (N, Cc, H, W), 1, 1)
                        and self._tcxh_ok(yb, ys, (N, K, Ho, Wo), 1, 1)):
                    self._conv_tcgwh(n, xb, (N, Cc, H, W), yb, (N, K, Ho, Wo), out, R, S, pt, pl,
                                     f"{node.op.wire_name}_tcgwh#{n}")
                    return True
                if self._wgrad_mn_ok(xb, xs, yb, ys, Cc, K):
                    # channel-last x and dy: 16-byte MN-major loads of both raw
                    # operands, split to TF32 in the kernel (no dy planes)
                    geo = dict(E1=S, E2=Cc, ro0=xs[2], ro1=xs[3], ro2=xs[1], h0=-pt, w0=-pl, H=H, W=W,
                               Ke1=Ho, Ke2=Wo, ko0=xs[0], ko1=xs[2], ko2=xs[3], kbase=-pt * xs[2] - pl * xs[3],
                               yo0=ys[0], yo1=ys[2], yo2=ys[3])
                    addr = {"c_rdiv": real_c or Cc, "c_s_hi": os_[3], "c_s_lo": os_[1], "c_sn": os_[0]}
                    self._conv_tcgw(n, xb, yb, out, Cc * R * S, K, kdim, geo, addr, f"{node.op.wire_name}_tcgw#{n}",
                                    real_c=real_c)
                    return True
                if xs[1] == 1 and Cc > 1:
                    # channel-last data: rows (r, s, c) so lanes read contiguous channels
                    geo = dict(E1=S, E2=Cc, ro0=xs[2], ro1=xs[3], ro2=xs[1], hm=1, wm=1, h0=-pt, w0=-pl, H=H, W=W,
                               pad0=1, **kgeo)
                    addr = {"c_rdiv": Cc, "c_s_hi": os_[3], "c_s_lo": os_[1], "c_sn": os_[0]}
                else:
                    geo = dict(E1=R, E2=S, ro0=xs[1], ro1=xs[2], ro2=xs[3], hm=1, wm=1, h0=-pt, w0=-pl, H=H, W=W, **kgeo)
                    addr = {"c_sm": os_[3], "c_sn": os_[0]}
                self._conv_tcgg(n, xb, b, out, Cc * R * S, K, kdim, geo, addr, yb, f"{node.op.wire_name}_tcgg#{n}")
                return True
            a = self._split(n, "a", yb, m, kdim, 3, s_r=ys[1], geo=(0,) * 12 + (N, Ho, Wo), st=(ys[0], ys[2], ys[3]))
            geo = (N, Cc, H, W, R, S, Ho, Wo, 1, 1, pt, pl)
            b = self._split(n, "b", xb, ncols, kdim, 4, geo=geo, st=xs)
            addr = {"c_sm": os_[0], "c_sn": os_[3]}
        rec = self._tc_gemm(n, a, b, out, m, ncols, kdim, addr, f"{node.op.wire_name}_tc#{n}")
        rec.algo_bytes = xb.nbytes + yb.nbytes + out.nbytes
        return True

    def emit_pool(self, n: int):
        _pool_emit(self, n)

    def emit_heavy(self, n: int):
        node = self.nodes[n]
        if n in self._epi:
            (ab, ast), (bb, bst) = self.operand(node.inputs[0][0]), self.operand(node.inputs[1][0])
            m, k = self.nodes[node.inputs[0][0]].output.shape
            self.emit_dot_tc(n, (ab, ast), (bb, bst), self.buf[self._epi[n]["out"]], m, node.output.shape[1], k)
            return
        out = self.buf[n]
        et = node.output.element_type
        if node.op is not OpKind.DOT and self.emit_conv_tc(n):
            r = self._conv_relu.get(n)
            if r is not None and n not in self._conv_relu_done:
                self.emit_map(r, [r])  # the conv took a kernel without the Relu side output
            return
        if n in self._conv_relu:
            raise AssertionError("a stem conv planned with a Relu side output did not lower to a tensor-core kernel")
        if node.op is OpKind.DOT:
            (ab, ast), (bb, bst) = self.operand(node.inputs[0][0]), self.operand(node.inputs[1][0])
            m, k = self.nodes[node.inputs[0][0]].output.shape
            nn = node.output.shape[1]
            if m == 0 or nn == 0:
                return
            if et is ElementType.F32 and use_tensor_cores(m, nn, k):
                self.emit_dot_tc(n, (ab, ast), (bb, bst), out, m, nn, k)
                return
            args = abi.DotArgs(m=m, n=nn, k=k, a_sm=ast[0], a_sk=ast[1], b_sk=bst[0], b_sn=bst[1],
                               c_sm=out.strides[0], c_sn=out.strides[1])
            if m <= 8 and nn >= 256:
                kind = abi.K_DOT_SM_F32 if et is ElementType.F32 else abi.K_DOT_SM_F64
                grid = (max(1, min((nn + 255) // 256, NUM_SMS * 16)), 1, 1)
            elif m * nn <= 1 << 16 and (m < 64 or nn < 64):
                # few outputs: a 64x64 tile would idle most threads
                kind = abi.K_DOT_TH_F32 if et is ElementType.F32 else abi.K_DOT_TH_F64
                grid = (max(1, (m * nn + 255) // 256), 1, 1)
            else:
                kind = abi.K_DOT_F32 if et is ElementType.F32 else abi.K_DOT_F64
                grid = ((nn + 63) // 64, (m + 63) // 64, 1)
            rec = LaunchRec(kind, grid, (256, 1, 1), 0, args, [ab.key, bb.key], [out.key], f"dot#{n}")
            rec.flops = 2 * m * nn * k
            rec.algo_bytes = (m * k + k * nn + m * nn) * et.byte_size
            rec.finalize = _finalize_refs(args, {"a": ab, "b": bb, "c": out})
            self.launches.append(rec)
            return
        if node.op in (OpKind.MAX_POOL, OpKind.MAX_POOL_BACKPROP):
            self.emit_pool(n)
            return
        x, y = node.inputs[0][0], node.inputs[1][0]
        (xb, xs), (yb, ys) = self.operand(x), self.operand(y)
        xshape, yshape = self.nodes[x].output.shape, self.nodes[y].output.shape
        oshape = node.output.shape
        a = node.attrs
        if node.op is OpKind.CONV2D:
            N, Cc, H, W = xshape
            K, _, R, S = yshape
            Ho, Wo = oshape[2], oshape[3]
            sh, sw = a["strides"]
            opc, total = 0, N * K * Ho * Wo
            macs = total * Cc * R * S
        elif node.op is OpKind.CONV_BACKPROP_DATA:
            N, K, Ho, Wo = xshape
            _, Cc, R, S = yshape
            H, W = oshape[2], oshape[3]
            sh, sw = conv_strides(node)
            opc, total = 1, N * Cc * H * W
            macs = N * K * Ho * Wo * Cc * R * S
        else:
            N, Cc, H, W = xshape
            _, K, Ho, Wo = yshape
            R, S = oshape[2], oshape[3]
            sh, sw = conv_strides(node)
            opc, total = 2, K * Cc * R * S
            macs = N * K * Ho * Wo * Cc * R * S
        if total == 0:
            return
        pt, _, pl, _ = a["padding"]
        args = abi.ConvArgs(op=opc, N=N, C=Cc, H=H, W=W, K=K, R=R, S=S, Ho=Ho, Wo=Wo, sh=sh, sw=sw, pt=pt, pl=pl)
        args.xs[:] = list(xs)
        args.ys[:] = list(ys)
        args.os[:] = list(out.strides)
        kind = abi.K_CONV_F32 if et is ElementType.F32 else abi.K_CONV_F64
        grid = max(1, min((total + 255) // 256, NUM_SMS * 64))
        rec = LaunchRec(kind, (grid, 1, 1), (256, 1, 1), 0, args, [xb.key, yb.key], [out.key], f"{node.op.wire_name}#{n}")
        rec.flops = 2 * macs
        rec.algo_bytes = xb.nbytes + yb.nbytes + out.nbytes
        rec.finalize = _finalize_refs(args, {"x": xb, "y": yb, "out": out})
        self.launches.append(rec)


def _pool_emit(low, n):
    """MaxPool (op 3) / MaxPoolBackprop (op 4) on the SIMT convolution-family
    kernel (csrc/simt_kernels.cu): one thread per output element, operands
    through per-axis strides (any layout), the window scanned in row-major
    order exactly as the oracle folds it."""
    node = low.nodes[n]
    out = low.buf[n]
    et = node.output.element_type
    a = node.attrs
    x = node.inputs[0][0]
    xb, xs = low.operand(x)
    N, Cc, H, W = low.nodes[x].output.shape
    kh, kw = a["window"]
    sh, sw = a["strides"]
    pt, _, pl, _ = a["padding"]
    if node.op is OpKind.MAX_POOL:
        Ho, Wo = node.output.shape[2], node.output.shape[3]
        yb, ys, opc, total = xb, xs, 3, N * Cc * Ho * Wo
    else:
        yb, ys = low.operand(node.inputs[1][0])
        Ho, Wo = low.nodes[node.inputs[1][0]].output.shape[2:]
        opc, total = 4, N * Cc * H * W
    if total == 0:
        return
    args = abi.ConvArgs(op=opc, N=N, C=Cc, H=H, W=W, K=Cc, R=kh, S=kw, Ho=Ho, Wo=Wo, sh=sh, sw=sw, pt=pt, pl=pl)
    args.xs[:] = list(xs)
    args.ys[:] = list(ys)
    args.os[:] = list(out.strides)
    kind = abi.K_CONV_F32 if et is ElementType.F32 else abi.K_CONV_F64
    grid = max(1, min((total + 255) // 256, NUM_SMS * 64))
    rec = LaunchRec(kind, (grid, 1, 1), (256, 1, 1), 0, args, sorted({xb.key, yb.key}), [out.key],
                    f"{node.op.wire_name}#{n}")
    rec.algo_bytes = xb.nbytes + out.nbytes + (yb.nbytes if opc == 4 else 0)
    rec.finalize = _finalize_refs(args, {"x": xb, "y": yb, "out": out})
    low.launches.append(rec)


def _storage_perm(buf) -> list:
    """Logical axes from outermost to innermost in memory (unit axes stay put)."""
    live = sorted((a for a in range(len(buf.shape)) if buf.shape[a] > 1), key=lambda a: (-buf.strides[a], a))
    it = iter(live)
    return [a if buf.shape[a] <= 1 else next(it) for a in range(len(buf.shape))]


def _dense_rowmajor(shape, strides) -> bool:
    """Row-major contiguous, ignoring the (meaningless) strides of unit axes."""
    want = _rowmajor(shape)
    return all(d == 1 or s == w for d, s, w in zip(shape, strides, want))


def _rowmajor(shape) -> tuple:
    out = [0] * len(shape)
    s = 1
    for a in range(len(shape) - 1, -1, -1):
        out[a] = s
        s *= shape[a]
    return tuple(out)


def _buf_ref(b: Buffer) -> int:
    if b.base is not None:
        return abi.ref(b.base.slot, b.base.offset + b.elem_off * b.et.byte_size)
    return abi.ref(b.slot, b.offset)


def _finalize_refs(args, fields: dict):
    def fin():
        for name, b in fields.items():
            setattr(args, name, _buf_ref(b))
    return fin


# ---------------------------------------------------------------------------
# VM program construction


@dataclass
class LeafSpec:
    buf: Buffer
    digits: list
    is_store: bool
    vec: int = 0
    vec_src: int = 0  # the index source vectors run along (0 = o, 1 = r)
    dv: list = None   # vec == 3: per-element offsets inside a vector


def _splat_bits(b: Buffer) -> int:
    v = b.splat
    if b.et is ElementType.F32:
        return struct.unpack("<I", struct.pack("<f", v))[0]
    if b.et is ElementType.F64:
        return struct.unpack("<Q", struct.pack("<d", v))[0]
    if b.et is ElementType.I64:
        return int(v) & ((1 << 64) - 1)
    return int(bool(v))


def _transpose_order(prog, n_o: int, V: int, src: int = 0):
    """(ty_ext, ty_div) for a map whose stores are vector-contiguous but
    whose biggest operand is contiguous along another digit of the vector
    index (`src`: o for COL, r for ROW) — a layout transposition: lanes then
    walk that digit, so the operand's loads coalesce across lanes while each
    thread still stores whole vectors."""
    if os.environ.get("GFB_TRANSPOSE_ORDER", "1") != "1" or n_o % V:
        return None
    stores = [l for l in prog.leaf_specs if l.is_store]
    if not stores or any(l.vec != 1 for l in stores):
        return None
    loads = [l for l in prog.leaf_specs if not l.is_store and l.buf.splat is None and l.vec in (0, 3)]
    if not loads:
        return None
    # the strided operand with the most bytes decides (vector-contiguous ones
    # keep whole-sector accesses either way)
    big = max(loads, key=lambda l: (any(d[0] == src and abs(d[3]) == 1 and d[1] >= V for d in l.digits), l.buf.nbytes))
    for dsrc, div, mod, stride in big.digits:
        if dsrc != src or abs(stride) != 1 or div < V or div % V:
            continue
        ext = mod if mod is not None else n_o // div
        if ext >= 8 and n_o % (div * ext) == 0 and ext * div <= n_o:
            return ext, div
    return None


def _dot_term_axes(node, axes, low):
    """Operand axes of each term t of a tiny Dot at output axes (i, j)."""
    k = low.g.nodes[node.inputs[0][0]].output.shape[1]
    ei, ej = axes
    return [([ei, _mk_axis((), t)], [_mk_axis((), t), ej]) for t in range(k)]


class Program:
    def __init__(self, low: Lowering, extents, vec_src: int, et: ElementType, dry: bool = False):
        self.low = low
        self.extents = extents
        self.vec_src = vec_src
        self.et = et
        self.V = vec_width(et)
        self.dry = dry
        self.leaf_specs: list = []
        self.leaf_index: dict = {}
        self.code: list = []  # (cls, op, k, swap) with k = leaf spec index
        self.red_out = None
        self.spans: dict = {}  # inlined node -> instructions it emitted
        self._inline: set = set()

    # -- leaves
    def leaf(self, buf: Buffer, axes) -> int:
        if buf.splat is None and buf.slot == abi.SLOT_CONST and self.low.const_values.get(buf.key) is not None \
                and all(e is None or (isinstance(e, Lin) and not e.terms) for e in axes):
            # one element of a constant at a compile-time coordinate: an immediate
            buf = self.low.splat_buffer(buf.et, self.low.const_values[buf.key][buf.elem_off + axes_offset(buf, axes)])
        digits = make_digits(buf, axes, self.extents) if buf.splat is None else []
        off = axes_offset(buf, axes) if buf.splat is None else 0
        if off:
            root = buf.base if buf.base is not None else buf
            buf = Buffer(buf.key, buf.et, buf.shape, buf.strides, buf.slot, buf.offset, None, base=root,
                         elem_off=buf.elem_off + off)
        key = (buf.key, buf.elem_off, tuple(digits), False)
        if key not in self.leaf_index:
            if len(digits) > abi.MAX_DIGITS:
                raise _TooManyDigits()
            spec = LeafSpec(buf, digits, False, vec_src=self.vec_src)
            spec.vec = 2 if buf.splat is not None else vec_class(digits, self.vec_src, False, self.V, buf.et.byte_size)
            if spec.vec == 1 and (buf.elem_off * buf.et.byte_size) % 16:
                spec.vec = 0  # a constant offset breaks the vector alignment
            if spec.vec == 3:
                spec.dv = vec_pattern(digits, self.vec_src, self.V)
            self.leaf_index[key] = len(self.leaf_specs)
            self.leaf_specs.append(spec)
        return self.leaf_index[key]

    def store_leaf(self, buf: Buffer, axes) -> int:
        digits = make_digits(buf, axes, self.extents)
        if len(digits) > abi.MAX_DIGITS:
            raise UnsupportedOp(f"index map needs {len(digits)} digits (> {abi.MAX_DIGITS})")
        spec = LeafSpec(buf, digits, True, vec_class(digits, self.vec_src, True, self.V, buf.et.byte_size), self.vec_src)
        if spec.vec == 3:
            spec.dv = vec_pattern(digits, self.vec_src, self.V)
        self.leaf_specs.append(spec)
        return len(self.leaf_specs) - 1

    def set_red_out(self, buf: Buffer, axes):
        digits = make_digits(buf, axes, self.extents)
        self.red_out = LeafSpec(buf, digits, True, vec_class(digits, 0, True, self.V, buf.et.byte_size))

    def set_vector_width(self, V: int):
        """Re-derive every leaf's access class for a kernel variant with V
        elements per thread-vector (the scalar VM uses V = 1)."""
        self.V = V
        for spec in self.leaf_specs + ([self.red_out] if self.red_out is not None else []):
            if spec.buf.splat is not None:
                spec.vec = 2
                continue
            spec.vec = vec_class(spec.digits, spec.vec_src, spec.is_store, V, spec.buf.et.byte_size)
            if spec.vec == 1 and (spec.buf.elem_off * spec.buf.et.byte_size) % 16:
                spec.vec = 0
            spec.dv = vec_pattern(spec.digits, spec.vec_src, V) if spec.vec == 3 else None

    def emit(self, cls, op=0, k=0, swap=0):
        self.code.append((cls, op, k, swap))

    # -- expression evaluation
    def view_of(self, n):
        """A strided view Buffer for index node `n` over a materialised buffer
        (a re-split Reshape of a row-major buffer is free even when the
        iteration digits cannot follow it), or None."""
        low = self.low
        if os.environ.get("GFB_NO_VIEW"):
            return None
        try:
            hv = low.heavy_operand(n)
        except Unexpressible:
            return None
        if hv is None or hv[1] is None:
            return None
        b, st = hv
        node = low.nodes[n]
        root = b.base if b.base is not None else b
        return Buffer(b.key, b.et, tuple(node.output.shape), tuple(st), b.slot, b.offset, b.splat, base=root,
                      elem_off=b.elem_off)

    def need(self, n, axes) -> int:
        low = self.low
        if n in low.buf:
            return 0
        node = low.nodes[n]
        if node.op in INDEX_OPS:
            try:
                return self.need(node.inputs[0][0], through_index_op(node, axes))
            except Unexpressible:
                if self.view_of(n) is not None:
                    return 0
                raise _Retry(n)
        if node.op in ELEMENTWISE_UNARY:
            return self.need(node.inputs[0][0], axes)
        if n in low.tiny:
            a, b = node.inputs[0][0], node.inputs[1][0]
            terms = _dot_term_axes(node, axes, low)
            if terms and all(self.is_plain(a, aa) and self.is_plain(b, ba) for aa, ba in terms):
                return 0
            worst = 0
            for t, (aa, ba) in enumerate(_dot_term_axes(node, axes, low)):
                na, nb = self.need(a, aa), self.need(b, ba)
                term = max(na, nb) if (self.is_plain(a, aa) or self.is_plain(b, ba)) else min(max(na, 1 + nb), max(nb, 1 + na))
                worst = max(worst, term + (1 if t else 0))
            return worst
        if node.op is OpKind.ADD:
            fold = self._add_dot1(n, axes)
            if fold is not None:
                return self.need(fold[0], axes)
        if node.op in ELEMENTWISE_BINARY:
            a, b = node.inputs[0][0], node.inputs[1][0]
            if a == b:
                return self.need(a, axes)
            na, nb = self.need(a, axes), self.need(b, axes)
            la, lb = self.is_plain(a, axes), self.is_plain(b, axes)
            if la or lb:
                return max(na, nb)
            return min(max(na, 1 + nb), max(nb, 1 + na))
        raise _Retry(n)  # Sum / heavy not inlinable

    def is_plain(self, n, axes) -> bool:
        low = self.low
        while n not in low.buf and low.nodes[n].op in INDEX_OPS:
            node = low.nodes[n]
            try:
                axes = through_index_op(node, axes)
            except Unexpressible:
                return self.view_of(n) is not None
            n = node.inputs[0][0]
        return n in low.buf

    def value(self, n, axes):
        """Emit code leaving node `n` at `axes` in acc; returns ('leaf', k) or ('acc',)."""
        start = len(self.code)
        r = self._value(n, axes)
        if r[0] == "acc" and n not in self._inline:
            self.spans[n] = max(self.spans.get(n, 0), len(self.code) - start)
        return r

    def _too_big(self, what):
        """A fused program over the VM limits: materialise its largest inlined
        sub-expression and lower again."""
        cands = [(size, n) for n, size in self.spans.items() if n not in self.low.M]
        if cands:
            raise _Retry(max(cands)[1])
        raise UnsupportedOp(what)

    def _value(self, n, axes):
        low = self.low
        node = low.nodes[n]
        if n in low.buf and n not in self._inline:
            return ("leaf", self.leaf(low.buf[n], axes))
        if node.op in INDEX_OPS:
            try:
                inner = through_index_op(node, axes)
            except Unexpressible:
                inner = None
            try:
                if inner is not None:
                    return self.value(node.inputs[0][0], inner)
                view = self.view_of(n)
                if view is None:
                    raise _Retry(n)
                return ("leaf", self.leaf(view, axes))
            except (_TooManyDigits, Unexpressible):
                raise _Retry(n)  # materialise the index op: its consumers then read it plainly
        if node.op in ELEMENTWISE_UNARY:
            self.to_acc(self.value(node.inputs[0][0], axes))
            self.emit(I_UN, VM_OP[node.op])
            return ("acc",)
        if n in low.tiny:
            # kernels.py:123-133: acc = 0; acc = rn(acc + rn(a*b)) for k ascending
            a, b = node.inputs[0][0], node.inputs[1][0]
            mul, add = VM_OP[OpKind.MULTIPLY], VM_OP[OpKind.ADD]
            terms = _dot_term_axes(node, axes, low)
            if terms and all(self.is_plain(a, aa) and self.is_plain(b, ba) for aa, ba in terms):
                # every operand a plain leaf: one two-operand multiply-add per term
                self.emit(I_LOAD, k=self.leaf(low.splat_buffer(node.output.element_type, 0.0), []))
                for aa, ba in terms:
                    self.emit(I_DOT, 0, self.value(a, aa)[1], self.value(b, ba)[1])
                return ("acc",)
            if not terms:  # empty contraction: the reference's 0.0
                self.emit(I_LOAD, k=self.leaf(low.splat_buffer(node.output.element_type, 0.0), []))
            for t, (aa, ba) in enumerate(terms):
                if t:
                    self.emit(I_PUSH)  # running sum
                if self.is_plain(b, ba):
                    self.to_acc(self.value(a, aa))
                    self.emit(I_BIN_LEAF, mul, self.value(b, ba)[1], 0)
                elif self.is_plain(a, aa):
                    self.to_acc(self.value(b, ba))
                    self.emit(I_BIN_LEAF, mul, self.value(a, aa)[1], 1)
                else:
                    self.to_acc(self.value(a, aa))
                    self.emit(I_PUSH)
                    self.to_acc(self.value(b, ba))
                    self.emit(I_BIN_POP, mul, 0, 0)
                if t:
                    self.emit(I_BIN_POP, add, 0, 0)  # acc = sum + term
                else:
                    zero = self.leaf(low.splat_buffer(node.output.element_type, 0.0), [])
                    self.emit(I_BIN_LEAF, add, zero, 1)  # acc = 0 + term
            return ("acc",)
        if node.op is OpKind.ADD:
            fold = self._add_dot1(n, axes)
            if fold is not None:
                # x + (0 + p) == x + p when x can never be -0: append the term
                other, t = fold
                self.to_acc(self.value(other, axes))
                (aa, ba) = t
                d = low.nodes[t[2]]
                self.emit(I_DOT, 0, self.value(d.inputs[0][0], aa)[1], self.value(d.inputs[1][0], ba)[1])
                return ("acc",)
        if node.op in ELEMENTWISE_BINARY:
            a, b = node.inputs[0][0], node.inputs[1][0]
            op = VM_OP[node.op]
            if a == b:
                r = self.value(a, axes)
                if r[0] == "leaf":
                    self.emit(I_LOAD, k=r[1])
                    self.emit(I_BIN_LEAF, op, r[1])
                else:
                    self.emit(I_BIN_SELF, op)
                return ("acc",)
            la, lb = self.is_plain(a, axes), self.is_plain(b, axes)
            if lb:
                self.to_acc(self.value(a, axes))
                rb = self.value(b, axes)
                self.emit(I_BIN_LEAF, op, rb[1], 0)
                return ("acc",)
            if la:
                self.to_acc(self.value(b, axes))
                ra = self.value(a, axes)
                self.emit(I_BIN_LEAF, op, ra[1], 1)
                return ("acc",)
            na, nb = self.need(a, axes), self.need(b, axes)
            if max(na, 1 + nb) <= max(nb, 1 + na):
                self.to_acc(self.value(a, axes))
                self.emit(I_PUSH)
                self.to_acc(self.value(b, axes))
                self.emit(I_BIN_POP, op, 0, 0)  # acc = op(pop=a, acc=b)
            else:
                self.to_acc(self.value(b, axes))
                self.emit(I_PUSH)
                self.to_acc(self.value(a, axes))
                self.emit(I_BIN_POP, op, 0, 1)  # acc = op(acc=a, pop=b)
            return ("acc",)
        raise _Retry(n)

    def _never_neg_zero(self, n, depth=0) -> bool:
        """Values of n are never -0: a tiny Dot starts its sum at +0, and a sum
        is -0 only when both addends are."""
        low = self.low
        node = low.nodes[n]
        if n in low.tiny:
            return True
        if node.op is OpKind.ADD and depth < 8:
            return any(self._never_neg_zero(r, depth + 1) for r, _ in node.inputs)
        return False

    def _add_dot1(self, n, axes):
        """(other operand, (a axes, b axes, dot node)) when Add n has a k = 1
        tiny-Dot operand computed inline from plain leaves and the other
        operand can never be -0, else None."""
        low = self.low
        if n in low.buf and n not in self._inline:
            return None
        x, y = (r for r, _ in low.nodes[n].inputs)
        for d, other in ((y, x), (x, y)):
            if d == other or d not in low.tiny or d in low.buf:
                continue
            dn = low.nodes[d]
            if low.g.nodes[dn.inputs[0][0]].output.shape[1] != 1:
                continue
            (aa, ba), = _dot_term_axes(dn, axes, low)
            if self.is_plain(dn.inputs[0][0], aa) and self.is_plain(dn.inputs[1][0], ba) \
                    and self._never_neg_zero(other):
                return other, (aa, ba, d)
        return None

    def to_acc(self, r):
        if r[0] == "leaf":
            self.emit(I_LOAD, k=r[1])

    def eval_value(self, n, axes):
        self._inline = set()
        if self.need(n, axes) > MAX_STACK:
            raise _Retry(self._deepest_child(n, axes))
        self.to_acc(self.value(n, axes))

    def eval_store(self, n, axes, out_buf: Buffer, also_inline=()):
        """Compute node `n` itself (even though it is materialised) and store it
        (`also_inline`: materialised inputs recomputed rather than loaded)."""
        self._inline = {n}
        node = self.low.nodes[n]
        if node.op in INDEX_OPS:
            try:
                inner = through_index_op(node, axes)
            except Unexpressible:
                inner = None
            self._inline = set()
            if inner is not None:
                r = self.value(node.inputs[0][0], inner)
            else:
                saved = self.low.buf.pop(n)
                try:
                    view = self.view_of(n)
                finally:
                    self.low.buf[n] = saved
                if view is None:
                    raise _Retry(n)
                r = ("leaf", self.leaf(view, axes))
        else:
            # also_inline: those inputs' buffers are hidden while n is evaluated, so
            # every query (need, is_plain, value) recomputes them
            hidden = {x: self.low.buf.pop(x) for x in also_inline if x in self.low.buf}
            try:
                if self.need_root(n, axes) > MAX_STACK:
                    raise _Retry(self._deepest_child(n, axes))
                r = self.value(n, axes)
            finally:
                self.low.buf.update(hidden)
        self.to_acc(r)
        self.emit(I_STORE, k=self.store_leaf(out_buf, axes))

    def need_root(self, n, axes) -> int:
        saved = self.low.buf.pop(n)
        try:
            return self.need(n, axes)
        finally:
            self.low.buf[n] = saved

    def _deepest_child(self, n, axes):
        node = self.low.nodes[n]
        kids = [r for r, _ in node.inputs if r not in self.low.buf]
        return max(kids, key=lambda k: self.need(k, axes)) if kids else n

    # -- encoding
    def finalize_order(self):
        """Reorder leaves: preloaded loads first, then other loads, then stores."""
        loads = [i for i, s in enumerate(self.leaf_specs) if not s.is_store]
        stores = [i for i, s in enumerate(self.leaf_specs) if s.is_store]
        uses = {i: 0 for i in loads}
        for cls, _, k, k2 in self.code:
            if cls in (I_LOAD, I_BIN_LEAF, I_PUSH_LOAD) and k in uses:
                uses[k] += 1
            if cls == I_DOT:
                for x in (k, k2):
                    if x in uses:
                        uses[x] += 1
        dot_only = set()
        other = set()
        for cls, _, k, k2 in self.code:
            if cls == I_DOT:
                dot_only.update((k, k2))
            elif cls in (I_LOAD, I_BIN_LEAF, I_PUSH_LOAD):
                other.add(k)
        dot_only -= other  # read only by multiply-adds: loaded there, never preloaded
        mem = [i for i in loads if self.leaf_specs[i].buf.splat is None and i not in dot_only]
        mem.sort(key=lambda i: -self.leaf_specs[i].buf.nbytes)
        pre = mem[:MAX_PRELOAD]
        pre += [i for i in loads if i not in pre and i not in dot_only][: MAX_PRELOAD - len(pre)]  # splats ride along
        rest = [i for i in loads if i not in pre]
        new_order = pre + rest + stores
        if len(new_order) > abi.MAX_LEAVES:
            self._too_big(f"fused group needs {len(new_order)} leaves (> {abi.MAX_LEAVES})")
        remap = {old: new for new, old in enumerate(new_order)}
        self.leaf_specs = [self.leaf_specs[i] for i in new_order]
        code = []
        for cls, op, k, swap in self.code:
            if cls in (I_LOAD, I_BIN_LEAF, I_STORE, I_PUSH_LOAD):
                k = remap[k]
            elif cls == I_DOT:
                k, swap = remap[k], remap[swap]
            code.append((cls, op, k, swap))
        self.code = code
        if len(self.code) > abi.MAX_INSTR:
            self._too_big(f"fused program of {len(self.code)} instructions (> {abi.MAX_INSTR})")
        return len(pre)

    def depth(self) -> int:
        d = best = 0
        for cls, _, _, _ in self.code:
            if cls in (I_PUSH, I_PUSH_LOAD):
                d += 1
                best = max(best, d)
            elif cls == I_BIN_POP:
                d -= 1
        return best

    def args(self, mode, n_o, n_r, red_kind=0, split=1, wpr=1) -> abi.EwArgs:
        npre = self.finalize_order()
        a = abi.EwArgs()
        a.n_o, a.n_r = n_o, n_r
        a.ninstr = len(self.code)
        a.nleaves = len(self.leaf_specs)
        a.mode, a.red_kind, a.vec_axis, a.split = mode, red_kind, self.vec_src, split
        a.npre, a.depth, a.wpr = npre, self.depth(), wpr
        words = encode_flat(self.code, npre)
        if len(words) > abi.MAX_INSTR:
            self._too_big(f"fused program of {len(words)} instructions (> {abi.MAX_INSTR})")
        a.ninstr = len(words)
        for i, w in enumerate(words):
            a.prog[i] = w
        return a

    def smem_bytes(self, a: abi.EwArgs, threads: int = 256) -> int:
        es = self.et.byte_size
        nofs = a.nleaves * (2 if a.pad else 1)
        return 4 * nofs * threads + es * a.depth * self.V * threads + es * max(self.V * threads, 8)

    def finalize_fn(self, a: abi.EwArgs):
        specs = list(self.leaf_specs)
        red = self.red_out

        def fin():
            first = {}
            for i, s in enumerate(specs):
                _encode_leaf(a.leaves[i], s)
                key = tuple(s.digits) if s.buf.splat is None else None
                a.leaves[i].same = first.get(key, -1) if key is not None else -1
                if key is not None:
                    first.setdefault(key, i)
            if red is not None:
                _encode_leaf(a.red_out, red)
                a.red_out.same = -1
        return fin

    def reads(self):
        return [s.buf.key for s in self.leaf_specs if not s.is_store and s.buf.splat is None]

    def writes(self):
        w = [s.buf.key for s in self.leaf_specs if s.is_store]
        if self.red_out is not None:
            w.append(self.red_out.buf.key)
        return w

    def algo_bytes(self) -> int:
        seen = set()
        total = 0
        for s in self.leaf_specs + ([self.red_out] if self.red_out else []):
            if s.buf.splat is not None or (s.buf.key, s.is_store) in seen:
                continue
            seen.add((s.buf.key, s.is_store))
            total += s.buf.nbytes
        return total

    _inline: set = set()


def _encode_leaf(L: abi.Leaf, s: LeafSpec):
    b = s.buf
    if b.splat is not None:
        L.mode = 1
        L.splat = _splat_bits(b)
        L.ndig = 0
        L.vec = 2
        L.rlin = 0
        return
    L.mode = 0
    L.ref = _buf_ref(b)
    L.ndig = len(s.digits)
    L.vec = s.vec
    L.rlin = r_linear(s.digits)
    digits = list(s.digits)
    for v in range(len(L.dv)):
        L.dv[v] = s.dv[v] if s.vec == 3 and s.dv is not None and v < len(s.dv) else 0
    if s.vec == 3 and s.dv is None:
        L.vec = 0
    for i, (src, div, mod, stride) in enumerate(digits):
        d = L.dig[i]
        d.src = src
        d.div_mul, d.div_sh = magic_u31(div)
        if mod is None:
            d.mod, d.mod_mul, d.mod_sh = 0, 0, 0
        else:
            d.mod = mod
            d.mod_mul, d.mod_sh = magic_u31(mod)
        d.stride = stride


def lower(g: Function, layouts: dict, private: bool = False, allreduce=frozenset(), channels_last: bool = False,
          allreduce_max=frozenset()) -> Lowered:
    low = Lowering(g, layouts, private, allreduce, channels_last, allreduce_max).run()
    low.channels_last = channels_last
    return low
