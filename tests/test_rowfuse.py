"""Row-fused launches (paper_1801_08058_b200/rowfuse.py).

CPU: which subgraphs form row groups, that the plans stay correct on the
emulator (sequential reference folds: bit-identical to the oracle), and
that the generated kernels compile for sm_100a.  GPU: the fused kernel
against the oracle (Sum-order tolerance; everything else exact), and
against the unfused plan of the same graph.
"""

import numpy as np
import pytest

import golden_io as G
from hostcompile import emulate, host_compile
from oracle import interp

import paper_1801_08058_b200 as gf
from paper_1801_08058_b200 import abi, jit, rowfuse
from paper_1801_08058_b200 import workloads as W

F32, F64, K = gf.ElementType.F32, gf.ElementType.F64, gf.OpKind


def _softmax_fn(R, C, et=F32):
    fn = gf.Function("softmax")
    x = fn.add_parameter(et, (R, C))
    fn.set_results([gf.build_softmax(fn, x, 1)])
    return fn


def _head_fn(R, C, et=F32):
    """Config E's head: logits + bias -> softmax cross-entropy, and its gradient."""
    step = W.mlp_step(gf, batch=R, in_dim=8, hidden=(), out_dim=C, f32=(et is F32), loss_batch=65536)
    return step


def _rows(h):
    return [L for L in h.lowered.launches if L.kind == abi.K_ROWJIT]


def test_softmax_is_one_launch():
    h = host_compile(_softmax_fn(512, 1000))
    assert len(h.lowered.launches) == 1 and h.lowered.launches[0].kind == abi.K_ROWJIT
    spec = h.lowered.launches[0].row_spec
    assert [v[1][0] for v in spec.values].count("rred") == 2  # max and sum
    assert h.lowered.arena_bytes == 0  # nothing but the input and p touches memory


def test_loss_head_forward_and_backward_fuse():
    """The E head (bias add, softmax, log, t * log p, and the whole softmax /
    cross-entropy gradient) is one row launch: reads logits, b, t once,
    writes dz once; the loss is a per-team partial + a second pass."""
    step = W.wide_mlp_step(gf, batch=512, width=256, layers=2, loss_batch=65536)
    h = host_compile(step.fn)
    rows = _rows(h)
    assert len(rows) == 1
    spec = rows[0].row_spec
    kinds = [e[0] for _, e in spec.values]
    assert kinds.count("load") == 2 and kinds.count("colv") == 1  # logits, t; the bias along rows
    assert len(spec.stores) == 1 and len(spec.xrow) == 1  # dz; the loss partials
    assert 4 * (3 * 512 * 256 + 256) <= rows[0].algo_bytes <= 4 * (3 * 512 * 256 + 256) + 64
    off = host_compile(step.fn, optimize=True)  # same plan twice: deterministic grouping
    assert [L.label for L in off.lowered.launches] == [L.label for L in h.lowered.launches]


def test_fused_plans_emulate_exactly(monkeypatch):
    for et in (F32, F64):
        step = W.mlp_step(gf, batch=32, in_dim=16, hidden=(24,), out_dim=40, f32=(et is F32))
        arrays = W.step_inputs(step, W.parameter_shapes(step), seed=5, f32=(et is F32))
        h = host_compile(step.fn)
        assert _rows(h)
        outs = emulate(h, [gf.tensor_from_flat(et, a.shape, a) for a in arrays])
        for o, w in zip(outs, interp.run_function(step.fn, arrays)):
            assert G.same_bits(np.asarray(o, dtype=w.dtype).reshape(w.shape), w)


def test_small_and_few_long_rows(monkeypatch):
    # few long rows stay on the chunk-wise reductions; small ones fuse
    assert not _rows(host_compile(_softmax_fn(4, 65536)))
    assert _rows(host_compile(_softmax_fn(4, 100)))
    assert not _rows(host_compile(_softmax_fn(512, 20000)))  # beyond MAX_C
    monkeypatch.setenv("GFB_ROWFUSE", "0")
    assert not _rows(host_compile(_softmax_fn(512, 1000)))


@pytest.mark.parametrize("R,C,et", [(512, 1000, F32), (300, 10, F32), (64, 4096, F64), (1000, 257, F32)])
def test_generated_kernel_compiles(R, C, et, tmp_path, monkeypatch):
    try:
        jit._lib_nvrtc()
    except RuntimeError as exc:
        pytest.skip(str(exc))
    monkeypatch.setenv("GFB_JIT_CACHE", str(tmp_path))
    step = _head_fn(R, C, et)
    for L in _rows(host_compile(step.fn)):
        src = rowfuse.generate_source(L.row_spec)
        assert "gfb_jit_ew" in src
        assert jit.compile_cubin(src)[:4] == b"\x7fELF"


# ---------------------------------------------------------------- GPU


def _call(fn, arrays, et=F32):
    exe = gf.compile_function(fn)
    return exe, [t.to_numpy() for t in gf.call(exe, [gf.tensor_from_flat(et, a.shape, a) for a in arrays])]


@pytest.mark.gpu
@pytest.mark.parametrize("R,C", [(512, 1000), (300, 10), (4096, 4096), (1000, 257), (2048, 8192)])
def test_softmax_gpu_vs_oracle(R, C):
    fn = _softmax_fn(R, C)
    x = np.random.default_rng(R + C).uniform(-8, 8, (R, C)).astype(np.float32)
    exe, out = _call(fn, [x])
    assert any(L.kind == abi.K_ROWJIT for L in exe.lowered.launches)
    interp.set_threads(interp.max_threads())
    want = interp.run_function(fn, [x])[0]
    # the reference's sequential fp32 row sums carry ~sqrt(C) * 2^-24 of error
    # themselves: compare both against the exact softmax (float64)
    x64 = x.astype(np.float64)
    e = np.exp(x64 - x64.max(axis=1, keepdims=True))
    exact = e / e.sum(axis=1, keepdims=True)
    assert G.normwise(out[0], exact) <= 1e-5
    assert G.normwise(out[0], exact) <= G.normwise(want, exact) + 1e-6
    assert np.max(np.abs(out[0] - exact) / exact) <= 1e-5  # elementwise, not only normwise


@pytest.mark.gpu
@pytest.mark.parametrize("R,C,f32", [(4096, 4096, True), (128, 10, True), (256, 10, False), (2000, 300, True)])
def test_loss_head_gpu_fused_vs_unfused_and_oracle(R, C, f32, monkeypatch):
    et = F32 if f32 else F64
    step = _head_fn(R, C, et)
    arrays = W.step_inputs(step, W.parameter_shapes(step), seed=9, f32=f32, x_range=(-1, 1))
    exe, fused = _call(step.fn, arrays, et)
    assert any(L.kind == abi.K_ROWJIT for L in exe.lowered.launches)
    monkeypatch.setenv("GFB_ROWFUSE", "0")
    exe0, plain = _call(step.fn, arrays, et)
    assert not any(L.kind == abi.K_ROWJIT for L in exe0.lowered.launches)
    interp.set_threads(interp.max_threads())
    want = interp.run_function(step.fn, arrays)
    tol = 1e-5 if f32 else 1e-12
    for a, b, w in zip(fused, plain, want):
        assert G.normwise(a, w) <= tol and G.normwise(a, b) <= tol


@pytest.mark.gpu
def test_row_launch_is_the_generated_kernel():
    """No silent fallback: the built-in entry of a row launch traps."""
    exe, _ = _call(_softmax_fn(512, 1000), [np.zeros((512, 1000), np.float32)])
    prog = exe.program()
    rows = [i for i, L in enumerate(exe.lowered.launches) if L.kind == abi.K_ROWJIT]
    assert rows and set(rows) <= set(prog.jit_launches)
