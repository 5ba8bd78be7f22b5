"""CPU oracle: executes a graph with the reference interpreter's semantics.

TEST INFRASTRUCTURE ONLY — imported by `tests/`, `__graft_entry__.smoke()`
and `bench.py`'s cpu_baseline / `--impl reference` leg, never by the
`paper_1801_08058_b200` package.  It restates `graphforge.call` on an
unoptimised compile (`/root/reference/pkg/src/graphforge/interpreter.py:191-245`)
over logical row-major numpy arrays: the arithmetic kernels are the C
restatement in `gf_oracle.cpp` (`kernels.py:101-264`); the pure index ops
(Broadcast `kernels.py:136-140`, Reshape `kernels.py:143-153`,
ConvertLayout `kernels.py:267-269`) are exact numpy gathers.

Pinned against the reference itself by `tests/test_oracle.py`, which
replays the golden documents in `tests/golden/` (produced by
`tests/golden/make_golden.py` running graphforge) and requires bit-equal
results.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from paper_1801_08058_b200.ir import ConstantData, ElementType, OpKind, reachable_from_results, topological_order

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

_ET = {ElementType.F32: 0, ElementType.F64: 1, ElementType.I64: 2, ElementType.BOOL: 3}
_OP = {
    OpKind.ADD: 0, OpKind.SUBTRACT: 1, OpKind.MULTIPLY: 2, OpKind.DIVIDE: 3, OpKind.MAXIMUM: 4,
    OpKind.NEGATE: 5, OpKind.EXP: 6, OpKind.LOG: 7, OpKind.TANH: 8, OpKind.SIGMOID: 9, OpKind.RELU: 10,
}


class _RedDesc(ctypes.Structure):
    _fields_ = [
        ("nk", ctypes.c_int32), ("nr", ctypes.c_int32),
        ("kdim", ctypes.c_int64 * 8), ("kstride", ctypes.c_int64 * 8),
        ("rdim", ctypes.c_int64 * 8), ("rstride", ctypes.c_int64 * 8),
    ]


_lib = None


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = ctypes.CDLL(LIB_PATH)
        i64, vp = ctypes.c_int64, ctypes.c_void_p
        _lib.orc_elementwise.argtypes = [ctypes.c_int, ctypes.c_int, vp, vp, vp, i64]
        _lib.orc_dot.argtypes = [ctypes.c_int, vp, vp, vp, i64, i64, i64]
        _lib.orc_reduce.argtypes = [ctypes.c_int, ctypes.c_int, vp, vp, ctypes.POINTER(_RedDesc), i64, i64]
        _lib.orc_conv2d.argtypes = [ctypes.c_int, vp, vp, vp] + [i64] * 13
        _lib.orc_conv_bwd_data.argtypes = [ctypes.c_int, vp, vp, vp] + [i64] * 13
        _lib.orc_conv_bwd_filter.argtypes = [ctypes.c_int, vp, vp, vp] + [i64] * 13
        _lib.orc_maxpool.argtypes = [ctypes.c_int, vp, vp] + [i64] * 12
        _lib.orc_maxpool_bwd.argtypes = [ctypes.c_int, vp, vp, vp] + [i64] * 12
        _lib.orc_set_threads.argtypes = [ctypes.c_int]
        _lib.orc_transpose2d.argtypes = [ctypes.c_int, vp, vp, i64, i64]
    return _lib


def set_threads(n: int) -> None:
    lib().orc_set_threads(int(n))


def max_threads() -> int:
    return int(lib().orc_max_threads())


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _c(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a)


def eval_node(node, args: list) -> np.ndarray:
    """Logical output array of one node given logical input arrays."""
    desc = node.output
    et = desc.element_type
    kind = node.op
    out = np.empty(desc.shape, dtype=et.numpy_dtype)
    L = lib()
    if kind in _OP:
        a = _c(args[0])
        b = _c(args[1]) if len(args) > 1 else None
        if out.size:
            L.orc_elementwise(_OP[kind], _ET[et], _ptr(a), _ptr(b), _ptr(out), out.size)
        return out
    if kind is OpKind.DOT:
        a, b = _c(args[0]), _c(args[1])
        m, k = a.shape
        n = b.shape[1]
        if out.size:
            L.orc_dot(_ET[et], _ptr(a), _ptr(b), _ptr(out), m, k, n)
        return out
    if kind is OpKind.BROADCAST:
        axes = node.attrs["broadcast_axes"]
        return np.broadcast_to(np.expand_dims(args[0], axes), desc.shape).copy()
    if kind is OpKind.RESHAPE:
        x = args[0]
        if tuple(node.attrs["input_order"]) == (1, 0) and x.ndim == 2 and x.size >= 65536:
            x = _c(x)
            out = np.empty((x.shape[1], x.shape[0]), dtype=x.dtype)
            L.orc_transpose2d(x.itemsize, _ptr(x), _ptr(out), x.shape[0], x.shape[1])
            return out.reshape(desc.shape)
        return _c(x.transpose(node.attrs["input_order"])).reshape(desc.shape).copy()
    if kind is OpKind.CONVERT_LAYOUT:
        return args[0].copy()
    if kind is OpKind.SUM:
        a = _c(args[0])
        axes = node.attrs["reduction_axes"]
        kept = [i for i in range(a.ndim) if i not in axes]
        strides = [s // a.itemsize for s in a.strides] if a.size else [0] * a.ndim
        d = _RedDesc()
        d.nk, d.nr = len(kept), len(axes)
        for j, ax in enumerate(kept):
            d.kdim[j], d.kstride[j] = a.shape[ax], strides[ax]
        for j, ax in enumerate(axes):
            d.rdim[j], d.rstride[j] = a.shape[ax], strides[ax]
        n_red = int(np.prod([a.shape[ax] for ax in axes], dtype=np.int64)) if axes else 1
        if out.size:
            L.orc_reduce(int(node.attrs["reduction_kind"] == "max"), _ET[et], _ptr(a), _ptr(out), ctypes.byref(d), out.size, n_red)
        return out
    if kind is OpKind.CONV2D:
        x, f = _c(args[0]), _c(args[1])
        N, C, H, Wd = x.shape
        K, _, R, S = f.shape
        sh, sw = node.attrs["strides"]
        pt, _, pl, _ = node.attrs["padding"]
        if out.size:
            L.orc_conv2d(_ET[et], _ptr(x), _ptr(f), _ptr(out), N, C, H, Wd, K, R, S, sh, sw, pt, pl, desc.shape[2], desc.shape[3])
        return out
    if kind is OpKind.CONV_BACKPROP_DATA:
        dlt, f = _c(args[0]), _c(args[1])
        N, C, H, Wd = desc.shape
        K, _, R, S = f.shape
        pt, _, pl, _ = node.attrs["padding"]
        sh, sw = node.attrs.get("strides", (1, 1))
        if out.size:
            L.orc_conv_bwd_data(_ET[et], _ptr(dlt), _ptr(f), _ptr(out), N, C, H, Wd, K, R, S, dlt.shape[2], dlt.shape[3], pt, pl,
                                sh, sw)
        return out
    if kind is OpKind.CONV_BACKPROP_FILTER:
        x, dlt = _c(args[0]), _c(args[1])
        N, C, H, Wd = x.shape
        K, _, R, S = desc.shape
        pt, _, pl, _ = node.attrs["padding"]
        sh, sw = node.attrs.get("strides", (1, 1))
        if out.size:
            L.orc_conv_bwd_filter(_ET[et], _ptr(x), _ptr(dlt), _ptr(out), N, C, H, Wd, K, R, S, dlt.shape[2], dlt.shape[3], pt, pl,
                                  sh, sw)
        return out
    if kind in (OpKind.MAX_POOL, OpKind.MAX_POOL_BACKPROP):  # IR extension: parity pinned by FD gradients only
        x = _c(args[0])
        N, C, H, Wd = x.shape
        kh, kw = node.attrs["window"]
        sh, sw = node.attrs["strides"]
        pt, _, pl, _ = node.attrs["padding"]
        if kind is OpKind.MAX_POOL:
            Ho, Wo = desc.shape[2], desc.shape[3]
            if out.size:
                L.orc_maxpool(_ET[et], _ptr(x), _ptr(out), N, C, H, Wd, kh, kw, sh, sw, pt, pl, Ho, Wo)
        else:
            dlt = _c(args[1])
            if out.size:
                L.orc_maxpool_bwd(_ET[et], _ptr(x), _ptr(dlt), _ptr(out), N, C, H, Wd, kh, kw, sh, sw, pt, pl,
                                  dlt.shape[2], dlt.shape[3])
        return out
    raise NotImplementedError(kind)


def run_function(fn, inputs: list) -> list:
    """Reference semantics of `call(compile_function(fn, optimize=False), inputs)`.

    `inputs` are logical arrays (or anything `np.asarray` accepts) in
    parameter order; returns one fresh logical array per result.
    """
    env = {}
    position = {pid: i for i, pid in enumerate(fn.parameters)}
    live = reachable_from_results(fn)
    for nid in topological_order(fn):
        if nid not in live:
            continue
        node = fn.nodes[nid]
        desc = node.output
        if node.op is OpKind.PARAMETER:
            env[nid] = np.asarray(inputs[position[nid]], dtype=desc.element_type.numpy_dtype).reshape(desc.shape)
        elif node.op is OpKind.CONSTANT:
            env[nid] = node.attrs["data"].to_numpy().reshape(desc.shape)
        else:
            env[nid] = eval_node(node, [env[r] for r, _ in node.inputs])
    return [np.array(env[r], copy=True) for r, _ in fn.results]


def fold_evaluator(node, inputs: list, input_descs: list) -> ConstantData:
    """`rewrite.constant_fold` evaluator backed by the oracle (tests only)."""
    args = [d.to_numpy().reshape(desc.shape) for d, desc in zip(inputs, input_descs)]
    out = eval_node(node, args)
    return ConstantData.from_array(node.output.element_type, out.reshape(-1))
