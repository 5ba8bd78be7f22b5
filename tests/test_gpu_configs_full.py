"""Parity of the BASELINE.json training-step configs at their real
dimensions (VERDICT r1 "parity stops short of the configs").

Each step graph runs through `compile_function` / `call` on the B200 and
through the C oracle (`oracle/`, pinned bit-for-bit to the reference
interpreter by tests/test_oracle.py) on the same seeded inputs:

* C -- small CNN at full size: batch 256, 32x32x3, conv 3->16->32, pool, fc;
* D -- ResNet-18-style, the full topology (7x7 stem, widths 64/128/256/512,
  2 BasicBlocks per stage) at 224x224, batch 2, identity and NHWC layouts,
  in F32 and (NHWC) in F64;
* E -- wide MLP, 8 layers of 4096, batch 256 (loss divided by 65536, as in
  the batch-sharded config).

The graphs also expose every gradient as a result, so the 1e-4 end-to-end
tolerance of `north_star` is checked on the gradients themselves.

Relu kinks.  A Relu gradient is a step function of its pre-activation z.
Two correct fp32 evaluations of z = h.W + b round differently (the
reference sums k sequentially, the tensor cores in 3xTF32 blocks), by about
sqrt(K) * 2^-24 of the terms' scale; every unit whose z lies inside that
band may get the opposite mask, and its whole gradient contribution flips.
At width 4096 x batch 256 x 8 layers the float64 forward has pre-activations
at 1.6e-7 of the term scale (tests' own measurement),
so a gradient comparison against the reference is only meaningful where no
mask sits in between:
* the forward (activations, logits, loss) is continuous: checked against the
  oracle at 1e-4;
* E's gradients are checked against the exact (float64) backward of the
  masks the device's own forward produced (the gradient given the forward,
  a continuous function), at 1e-4;
* D's F32 conv gradients are reported against the oracle but only bounded
  loosely; D's lowering at full topology is checked exactly in F64, where the
  rounding band (1e-16) contains no pre-activation, against the oracle at
  1e-10.
"""

import functools

import numpy as np
import pytest

import golden_io as G
from oracle import interp

pytestmark = pytest.mark.gpu

gf = pytest.importorskip("paper_1801_08058_b200")
from paper_1801_08058_b200 import workloads as W  # noqa: E402

TOL = 1e-4  # north_star: end-to-end losses and gradients


def _expose(step, forward_relus=False):
    """Results := gradients (+ forward Relu outputs) + new parameters + loss.
    The SGD update is Subtract(p, Multiply(Broadcast(lr), grad))
    (workloads._append_sgd)."""
    g = step.fn
    new = list(g.results[:step.loss_index])
    grads = [g.nodes[g.nodes[r].inputs[1][0]].inputs[1] for r, _ in new]
    relus = []
    if forward_relus:
        relus = [(n, 0) for n in gf.topological_order(g) if g.nodes[n].op is gf.OpKind.RELU]
    g.set_results(grads + relus + list(g.results))
    return len(grads), len(relus)


@functools.lru_cache(maxsize=None)
def _case(name, f32=True):
    if name == "C":
        step = W.cnn_step(gf, batch=256)
    elif name == "D":
        step = W.resnet_step(gf, batch=2, image=224, f32=f32)
    else:
        step = W.wide_mlp_step(gf, batch=256, loss_batch=65536)
    n_grads, n_relus = _expose(step, forward_relus=(name == "E"))
    arrays = W.step_inputs(step, W.parameter_shapes(step), seed=11, f32=f32, x_range=W.x_range_of(name),
                           conv_gain=W.conv_gain_of(name))
    interp.set_threads(interp.max_threads())
    want = interp.run_function(step.fn, arrays)
    assert all(np.all(np.isfinite(w)) for w in want), "reference step not finite"
    return step, n_grads, n_relus, arrays, want


def _run(name, layout="identity", f32=True):
    step, n_grads, n_relus, arrays, want = _case(name, f32)
    et = gf.ElementType.F32 if f32 else gf.ElementType.F64
    exe = gf.compile_function(step.fn, conv_layout=layout)
    outs = [t.to_numpy() for t in gf.call(exe, [gf.tensor_from_flat(et, a.shape, a) for a in arrays])]
    assert all(np.all(np.isfinite(o)) for o in outs)
    return exe, step, n_grads, n_relus, arrays, want, outs


def _check_loss(outs, want, tol=TOL):
    loss, wloss = float(outs[-1]), float(want[-1])
    assert abs(loss - wloss) <= tol * max(1.0, abs(wloss)), (loss, wloss)


def test_config_C_full_size():
    exe, step, n_grads, _, _, want, outs = _run("C")
    bad = [(i, G.normwise(o, w)) for i, (o, w) in enumerate(zip(outs, want)) if G.normwise(o, w) > TOL]
    assert not bad, bad
    _check_loss(outs, want)


@pytest.mark.parametrize("layout", ["identity", "nhwc"])
def test_config_D_full_topology_224_f32(layout):
    exe, step, n_grads, _, _, want, outs = _run("D", layout)
    convs = sum(1 for n in exe.function.nodes.values() if n.op.wire_name.startswith("Conv"))
    assert convs >= 59  # 20 convolutions forward, 20 filter and 19 data gradients
    _check_loss(outs, want)
    names = step.weight_names
    errs = {nm: (G.normwise(o, w), float(np.linalg.norm(o - w) / np.linalg.norm(w)))
            for nm, o, w in zip(names, outs[:n_grads], want[:n_grads])}
    # the classifier gradient has no Relu mask below it: strict
    assert errs["Wf"][0] <= TOL, errs["Wf"]
    # conv filter gradients: mask flips at kink pre-activations (module doc);
    # the F64 test below checks the same lowering exactly
    assert all(fro <= 5e-2 for _, fro in errs.values()), errs
    print("D f32", layout, {k: (f"{a:.1e}", f"{b:.1e}") for k, (a, b) in errs.items()})


def test_config_D_full_topology_224_f64():
    exe, step, n_grads, _, _, want, outs = _run("D", "nhwc", f32=False)
    bad = [(i, G.normwise(o, w)) for i, (o, w) in enumerate(zip(outs, want)) if G.normwise(o, w) > 1e-10]
    assert not bad, bad


def _exact_backward(step, arrays, hs, batch_div=65536.0):
    """float64 gradients of config E's step given the device's forward Relu
    outputs hs = [h1..h7] (masks h > 0), in the order W1, b1, ..., W8, b8."""
    d = dict(zip(step.param_names, [a.astype(np.float64) for a in arrays]))
    h = [d["x"]] + [np.asarray(v, dtype=np.float64) for v in hs]
    logits = h[7] @ d["W8"] + d["b8"]
    e = np.exp(logits - logits.max(axis=1, keepdims=True))
    p = e / e.sum(axis=1, keepdims=True)
    dz = (p - d["t"]) / batch_div
    grads = {}
    for l in range(8, 0, -1):
        grads[f"W{l}"] = h[l - 1].T @ dz
        grads[f"b{l}"] = dz.sum(axis=0)
        if l > 1:
            dz = (dz @ d[f"W{l}"].T) * (h[l - 1] > 0)
    return [grads[n] for n in step.weight_names]


def test_config_E_width_4096_x8():
    exe, step, n_grads, n_relus, arrays, want, outs = _run("E")
    assert sum(1 for L in exe.lowered.launches if L.flops) >= 23  # the step's 23 GEMMs on tcgen05
    # forward: activations and loss against the reference interpreter
    for o, w in zip(outs[n_grads:n_grads + n_relus], want[n_grads:n_grads + n_relus]):
        assert G.normwise(o, w) <= TOL
    _check_loss(outs, want)
    # backward: against the exact backward of the device's own forward masks
    exact = _exact_backward(step, arrays, outs[n_grads:n_grads + n_relus])
    bad = [(nm, G.normwise(o, x)) for nm, o, x in zip(step.weight_names, outs[:n_grads], exact) if G.normwise(o, x) > TOL]
    assert not bad, bad
    # and the new parameters against the reference
    for o, w in zip(outs[n_grads + n_relus:-1], want[n_grads + n_relus:-1]):
        assert G.normwise(o, w) <= TOL
