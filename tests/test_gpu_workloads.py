"""Full-size BASELINE.json configs on the B200 against the C oracle.

Config A (MLP 784-512-10, batch 128) runs at full size on the oracle in
well under a second; config B at full size (64 Mi elements) too.  The
oracle is itself pinned against the reference (tests/test_oracle.py).
"""

import numpy as np
import pytest

import golden_io as G
from oracle import interp

pytestmark = pytest.mark.gpu

gf = pytest.importorskip("paper_1801_08058_b200")
from paper_1801_08058_b200 import workloads as W  # noqa: E402


def _run_step(step, seed=0):
    shapes = W.parameter_shapes(step)
    arrays = W.step_inputs(step, shapes, seed=seed)
    want = interp.run_function(step.fn, arrays)
    exe = gf.compile_function(step.fn)
    outs = [t.to_numpy() for t in gf.call(exe, [gf.tensor_from_flat(gf.ElementType.F32, a.shape, a) for a in arrays])]
    return outs, want


def test_config_A_full_size():
    interp.set_threads(interp.max_threads())
    outs, want = _run_step(W.mlp_step(gf, batch=128))
    for o, w in zip(outs, want):
        assert G.normwise(o, w) <= 1e-4, G.normwise(o, w)
    assert abs(float(outs[-1]) - float(want[-1])) <= 1e-4 * max(1.0, abs(float(want[-1])))


def test_config_C_reduced():
    interp.set_threads(interp.max_threads())
    outs, want = _run_step(W.cnn_step(gf, batch=4, image=16, channels=(3, 8, 16)))
    for o, w in zip(outs, want):
        assert G.normwise(o, w) <= 1e-4


@pytest.mark.parametrize("rows", [257, 4096, 65536])
def test_config_B(rows):
    interp.set_threads(interp.max_threads())
    fn = W.fused_chain(gf, rows=rows, cols=1024)
    arrays = W.chain_inputs(rows, 1024)
    want = interp.run_function(fn, arrays)
    exe = gf.compile_function(fn)
    assert exe.num_launches <= 2 and (rows != 65536 or exe.num_launches == 1)  # one pass (+ partials pass for few rows)
    outs = [t.to_numpy() for t in gf.call(exe, [gf.tensor_from_flat(gf.ElementType.F32, a.shape, a) for a in arrays])]
    assert G.same_bits(outs[0], want[0])  # elementwise chain: bit-exact
    assert G.normwise(outs[1], want[1]) <= 1e-5  # tree-ordered row sums


@pytest.mark.parametrize("shape,axes", [((3, 5000), (1,)), ((2, 300, 40), (1, 2)), ((1 << 22,), (0,)), ((16, 65536), (0, 1))])
def test_long_row_reductions(shape, axes):
    K, F32 = gf.OpKind, gf.ElementType.F32
    fn = gf.Function("red")
    x = fn.add_parameter(F32, shape)
    e = fn.add_node(K.EXP, [x])
    fn.set_results([fn.add_node(K.SUM, [e], {"reduction_axes": axes}), fn.add_node(K.NEGATE, [e])])
    rng = np.random.default_rng(0)
    v = rng.uniform(-1, 1, size=shape).astype(np.float32)
    outs = [t.to_numpy() for t in gf.call(gf.compile_function(fn), [gf.tensor_from_flat(F32, shape, v)])]
    interp.set_threads(interp.max_threads())
    want = interp.run_function(fn, [v])
    # A sequential fp32 sum (the reference order) of millions of terms drifts
    # by ~1e-3; the tree-ordered device sum must be within 1e-5 of the exact
    # sum and never less accurate than the reference order.
    exact = np.exp(v.astype(np.float64)).sum(axis=axes)
    assert G.normwise(outs[0], exact) <= 1e-5
    assert G.normwise(outs[0], exact) <= G.normwise(want[0], exact) + 1e-7
    assert G.same_bits(outs[1], want[1])


def test_data_parallel_plan_single_rank_nccl():
    """The DP plan with real NCCL all-reduces captured in the CUDA graph
    (one rank) equals the plain plan; multi-rank sums are covered on CPU."""
    step = W.mlp_step(gf, batch=64, in_dim=96, hidden=(64,), out_dim=10)
    arrays = W.step_inputs(step, W.parameter_shapes(step), seed=2)
    names = step.param_names
    dp = gf.DataParallel([step.fn.parameters[names.index("x")], step.fn.parameters[names.index("t")]])
    exe = gf.compile_function(step.fn, data_parallel=dp)
    ar = [L for L in exe.lowered.launches if L.label.startswith("allreduce")]
    assert 1 <= len(ar) <= 5 and sum(len(L.reads) for L in ar) == 5  # 5 roots in gradient buckets
    tens = [gf.tensor_from_flat(gf.ElementType.F32, a.shape, a) for a in arrays]
    got = [t.to_numpy() for t in gf.call(exe, tens)]
    plain = [t.to_numpy() for t in gf.call(gf.compile_function(step.fn), tens)]
    for a, b in zip(got, plain):
        assert G.same_bits(a, b)


def test_call_streamed_equals_call():
    from paper_1801_08058_b200.runtime import pinned_tensor
    from paper_1801_08058_b200.streaming import call_streamed

    fn = W.fused_chain(gf, rows=4096, cols=1024)
    arrays = W.chain_inputs(4096, 1024)
    exe = gf.compile_function(fn)
    host = []
    for a in arrays:
        t = pinned_tensor(gf.ElementType.F32, a.shape)
        t.buffer[:] = a.reshape(-1)
        host.append(t)
    out = [pinned_tensor(d.element_type, d.shape) for d, _ in exe.result_signature]
    call_streamed(exe, host, out, chunks=8)
    ref = [t.to_numpy() for t in gf.call(exe, host)]
    assert G.same_bits(out[0].to_numpy(), ref[0])
    assert G.normwise(out[1].to_numpy(), ref[1]) <= 1e-6


@pytest.mark.parametrize("layout", ["identity", "nhwc"])
def test_config_D_reduced(layout):
    """ResNet-18-style step (config D topology) at 32x32 / batch 4 with the
    tensor-core conv path, both layouts, against the oracle."""
    interp.set_threads(interp.max_threads())
    step = W.resnet_step(gf, batch=4, image=32, widths=(16, 32), blocks=1)
    arrays = W.step_inputs(step, W.parameter_shapes(step), seed=4)
    want = interp.run_function(step.fn, arrays)
    exe = gf.compile_function(step.fn, conv_layout=layout)
    outs = [t.to_numpy() for t in gf.call(exe, [gf.tensor_from_flat(gf.ElementType.F32, a.shape, a) for a in arrays])]
    for o, w in zip(outs, want):
        assert G.normwise(o, w) <= 1e-4
