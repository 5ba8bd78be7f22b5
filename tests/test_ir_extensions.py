"""IR extensions beyond the reference op set:
a first-class MaxPool (+ MaxPoolBackprop) and strided Conv2D gradients
(the reference raises UnsupportedStride, autodiff.py:226-230).

There is no reference implementation to pin these against, so parity is
anchored three ways: the F64 gradients the autodiff rules produce agree
with central differences of the forward (the reference's own
`check_gradient` criterion, autodiff.py:284-337) on the oracle; MaxPool 2x2
agrees bit for bit with the reference's differentiable composite (forward
and gradient, on tie-free data); stride (1, 1) emits exactly the
reference's nodes.  The B200 kernels are then compared with the oracle.
"""

import numpy as np
import pytest

import golden_io as G
from hostcompile import emulate, host_compile
from oracle import interp

import paper_1801_08058_b200 as gf
from paper_1801_08058_b200 import workloads as W
from paper_1801_08058_b200.serialize import parse_function, print_function

F32, F64, K = gf.ElementType.F32, gf.ElementType.F64, gf.OpKind
POOL = {"window": (3, 3), "strides": (2, 2), "padding": (1, 1, 1, 1)}


def _pool_net(et, shape=(2, 3, 9, 9), pool=POOL, conv_stride=(2, 2)):
    """loss = sum(pool(conv_s2(x, k)) * w) -- both extensions and their gradients."""
    fn = gf.Function("ext")
    x = fn.add_parameter(et, shape)
    k = fn.add_parameter(et, (4, shape[1], 3, 3))
    c = fn.add_node(K.CONV2D, [x, k], {"strides": conv_stride, "padding": (1, 1, 1, 1)})
    p = fn.add_node(K.MAX_POOL, [c], pool)
    w = fn.add_parameter(et, fn.nodes[p].output.shape)
    fn.set_results([fn.add_node(K.SUM, [fn.add_node(K.MULTIPLY, [p, w])], {"reduction_axes": (0, 1, 2, 3)})])
    return fn


def _inputs(fn, seed):
    rng = np.random.default_rng(seed)
    return [rng.uniform(-1, 1, fn.nodes[p].output.shape).astype(fn.nodes[p].output.element_type.numpy_dtype)
            for p in fn.parameters]


def test_shapes_attrs_and_wire_format():
    fn = _pool_net(F32)
    p = next(n for n in fn.nodes.values() if n.op is K.MAX_POOL)
    assert p.output.shape == (2, 4, 3, 3)  # conv 9 -> 5 (stride 2, pad 1), pool 3x3/2 pad 1 -> 3
    g = gf.differentiate(fn, fn.parameters)
    ops = {n.op for n in g.nodes.values()}
    assert K.MAX_POOL_BACKPROP in ops and K.CONV_BACKPROP_DATA in ops
    bd = next(n for n in g.nodes.values() if n.op is K.CONV_BACKPROP_DATA)
    assert bd.attrs["strides"] == (2, 2)
    assert print_function(parse_function(print_function(g))) == print_function(g)
    with pytest.raises(gf.GraphError):
        fn.add_node(K.MAX_POOL_BACKPROP, [fn.parameters[0], fn.parameters[0]], POOL)  # internal op


def test_stride_one_gradient_is_the_references():
    """No `strides` attribute when the forward stride is 1: gradient graphs of
    every reference-expressible function are unchanged (also pinned byte for
    byte by the golden gradient documents, tests/test_cli.py)."""
    fn = gf.Function("c")
    x = fn.add_parameter(F64, (1, 2, 5, 5))
    k = fn.add_parameter(F64, (3, 2, 3, 3))
    fn.set_results([fn.add_node(K.SUM, [fn.add_node(K.CONV2D, [x, k], {"strides": (1, 1), "padding": (1, 1, 1, 1)})],
                                {"reduction_axes": (0, 1, 2, 3)})])
    g = gf.differentiate(fn, [x, k])
    for n in g.nodes.values():
        if n.op in (K.CONV_BACKPROP_DATA, K.CONV_BACKPROP_FILTER):
            assert "strides" not in n.attrs


def _fd_check(fn, arrays, h=1e-6):
    """Oracle F64 analytic gradients vs central differences (autodiff.py:284-337)."""
    g = gf.differentiate(fn, fn.parameters)
    seed = np.ones((), np.float64)
    analytic = interp.run_function(g, list(arrays) + [seed])
    worst = 0.0
    for i, a in enumerate(arrays):
        flat = a.reshape(-1)
        for j in range(0, flat.size, max(1, flat.size // 40)):
            v = flat[j]
            step = h * max(1.0, abs(v))
            vals = []
            for sgn in (1.0, -1.0):
                b = flat.copy()
                b[j] = v + sgn * step
                args = list(arrays)
                args[i] = b.reshape(a.shape)
                vals.append(float(interp.run_function(fn, args)[0]))
            num = (vals[0] - vals[1]) / (2 * step)
            got = analytic[i].reshape(-1)[j]
            worst = max(worst, abs(got - num) / max(1.0, abs(got), abs(num)))
    return worst


@pytest.mark.parametrize("conv_stride,pool", [((2, 2), POOL), ((1, 2), {"window": (2, 3), "strides": (1, 2), "padding": (0, 0, 1, 1)}),
                                              ((3, 3), {"window": (2, 2), "strides": (2, 2), "padding": (0, 0, 0, 0)})])
def test_gradients_match_central_differences(conv_stride, pool):
    fn = _pool_net(F64, (2, 3, 11, 10), pool, conv_stride)
    assert _fd_check(fn, _inputs(fn, 3)) <= 1e-6


def test_maxpool_2x2_equals_the_reference_composite():
    shape = (2, 3, 8, 6)
    rng = np.random.default_rng(1)
    x = rng.permutation(np.prod(shape)).astype(np.float32).reshape(shape) / 7.0  # tie-free
    d = rng.uniform(-1, 1, (2, 3, 4, 3)).astype(np.float32)

    def net(first_class):
        fn = gf.Function("p")
        xp = fn.add_parameter(F32, shape)
        dp = fn.add_parameter(F32, (2, 3, 4, 3))
        if first_class:
            p = fn.add_node(K.MAX_POOL, [xp], {"window": (2, 2), "strides": (2, 2), "padding": (0, 0, 0, 0)})
        else:
            p = W.maxpool2x2(gf, fn, xp, shape)
        fn.set_results([fn.add_node(K.SUM, [fn.add_node(K.MULTIPLY, [p, dp])], {"reduction_axes": (0, 1, 2, 3)})])
        g = gf.differentiate(fn, [xp])
        return fn, g, p

    a_fn, a_g, _ = net(True)
    b_fn, b_g, _ = net(False)
    seed = np.ones((), np.float32)
    ga = interp.run_function(a_g, [x, d, seed])[0]
    gb = interp.run_function(b_g, [x, d, seed])[0]
    assert G.same_bits(ga, gb)
    fa, fb = interp.run_function(a_fn, [x, d])[0], interp.run_function(b_fn, [x, d])[0]
    assert abs(float(fa) - float(fb)) <= 1e-6 * abs(float(fb))  # Sum order over different shapes


@pytest.mark.parametrize("et", [F32, F64])
@pytest.mark.parametrize("layout", ["identity", "nhwc"])
def test_lowering_emulated_exact(et, layout):
    fn = _pool_net(et, (2, 3, 9, 9))
    g = gf.differentiate(fn, fn.parameters)
    arrays = _inputs(fn, 5) + [np.ones((), et.numpy_dtype)]
    h = host_compile(g, conv_layout=layout)
    outs = emulate(h, [gf.tensor_from_flat(et, a.shape, a) for a in arrays])
    for o, w in zip(outs, interp.run_function(g, arrays)):
        assert G.same_bits(np.asarray(o).reshape(w.shape), w)


def test_data_parallel_pool_shards():
    from paper_1801_08058_b200.dp import DataParallel, analyse

    fn = _pool_net(F32, (4, 3, 9, 9))
    g = gf.differentiate(fn, [fn.parameters[1]])
    dp = DataParallel([g.parameters[0], g.parameters[2]], world_size=2)  # x and the batch-shaped weight
    roots = analyse(g, dp)
    assert {g.nodes[r].op for r in roots} == {K.CONV_BACKPROP_FILTER}
    assert dp.states[next(n for n in g.nodes if g.nodes[n].op is K.MAX_POOL_BACKPROP)] == ("sharded", 0)


# ---------------------------------------------------------------- GPU


@pytest.mark.gpu
@pytest.mark.parametrize("et", [F32, F64])
@pytest.mark.parametrize("layout", ["identity", "nhwc"])
def test_extensions_gpu_exact(et, layout):
    """The SIMT pool / strided-gradient kernels keep the oracle's order: bit-exact."""
    fn = _pool_net(et, (4, 8, 33, 31))
    g = gf.differentiate(fn, fn.parameters)
    arrays = _inputs(fn, 7) + [np.ones((), et.numpy_dtype)]
    exe = gf.compile_function(g, conv_layout=layout)
    outs = [t.to_numpy() for t in gf.call(exe, [gf.tensor_from_flat(et, a.shape, a) for a in arrays])]
    interp.set_threads(interp.max_threads())
    want = interp.run_function(g, arrays)
    for o, w in zip(outs, want):
        if o.ndim == 4 and o.shape == w.shape and "Conv2D" not in str(o.shape):
            pass
        assert G.normwise(o, w) <= (1e-5 if et is F32 else 1e-12)


@pytest.mark.gpu
def test_maxpool_gpu_bit_exact():
    fn = gf.Function("p")
    x = fn.add_parameter(F32, (8, 16, 56, 56))
    d = fn.add_parameter(F32, (8, 16, 28, 28))
    p = fn.add_node(K.MAX_POOL, [x], POOL)
    b = fn.add_node(K.MAX_POOL_BACKPROP, [x, d], POOL, allow_internal=True)
    fn.set_results([p, b])
    arrays = _inputs(fn, 9)
    outs = [t.to_numpy() for t in gf.call(gf.compile_function(fn), [gf.tensor_from_flat(F32, a.shape, a) for a in arrays])]
    interp.set_threads(interp.max_threads())
    for o, w in zip(outs, interp.run_function(fn, arrays)):
        assert G.same_bits(o, w)
