"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container only (needs /root/reference; never imported by
the test suite):

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests:. \
        python tests/golden/make_golden.py

Everything written here is produced by `graphforge` itself — graphs through
its construction API / `random_function` corpus generator
(`pkg/tests/_graphgen.py:209-284`), outputs through its interpreter
`compile_function` + `call` (`pkg/src/graphforge/interpreter.py:92-245`),
backward graphs through its `differentiate` (`autodiff.py:34-261`) — and
stored in the reference's own wire format (`serialize.py:94-280`).  The
B200 tests load these documents and compare against them.
"""

from __future__ import annotations

import gzip
import json
import os
import random
import sys
import time

import graphforge as gf
from graphforge import serialize as gser
from graphforge.ir import OpKind

from _gradcases import build_mlp, op_gradient_cases, sample_mlp_point
from _graphgen import random_function, random_inputs

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
from paper_1801_08058_b200 import workloads as W  # noqa: E402  (builders take `api`)

HERE = os.path.dirname(os.path.abspath(__file__))


def tdoc(t):
    return gser.tensor_to_document(t)


def fdoc(fn):
    return gser.function_to_document(fn)


def dump(name, obj):
    path = os.path.join(HERE, name)
    with gzip.open(path, "wt") as fh:
        json.dump(obj, fh, separators=(",", ":"))
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


def corpus(n=200):
    cases = []
    for seed in range(n):
        fn = random_function(seed, max_nodes=25)
        inputs = random_inputs(fn, seed + 100_000)
        exe_opt = gf.compile_function(fn)
        exe_raw = gf.compile_function(fn, optimize=False)
        cases.append(
            {
                "seed": seed,
                "fn": fdoc(fn),
                "inputs": [tdoc(t) for t in inputs],
                "outputs_opt": [tdoc(t) for t in gf.call(exe_opt, inputs)],
                "outputs_noopt": [tdoc(t) for t in gf.call(exe_raw, inputs)],
                "listing_opt": exe_opt.listing(),
                "listing_noopt": exe_raw.listing(),
            }
        )
    return cases


def layout_cases():
    """Permuted parameter layouts (test_acceptance.py:271-285) and the nhwc
    conv network (test_acceptance.py:212-230)."""
    out = []
    rng = random.Random(99)
    for trial in range(10):
        fn = random_function(trial + 400)
        base = random_inputs(fn, trial)
        layouts, tensors = [], []
        for t in base:
            order = list(range(len(t.shape)))
            rng.shuffle(order)
            layouts.append(order)
            tensors.append(gf.tensor_from_flat(t.element_type, t.shape, t.to_flat(), gf.Layout(tuple(order))))
        exe = gf.compile_function(fn, optimize=False, parameter_layouts=[gf.Layout(tuple(o)) for o in layouts])
        out.append(
            {
                "name": f"permuted{trial}",
                "fn": fdoc(fn),
                "conv_layout": "identity",
                "parameter_layouts": layouts,
                "inputs": [tdoc(t) for t in tensors],
                "outputs": [tdoc(t) for t in gf.call(exe, tensors)],
                "listing": exe.listing(),
            }
        )
    fn = gf.Function("convnet")
    F64 = gf.ElementType.F64
    x = fn.add_parameter(F64, (1, 2, 6, 6))
    w1 = fn.add_parameter(F64, (3, 2, 3, 3))
    w2 = fn.add_parameter(F64, (2, 3, 2, 2))
    c1 = fn.add_node(OpKind.CONV2D, [x, w1], {"strides": (1, 1), "padding": (1, 1, 1, 1)})
    r1 = fn.add_node(OpKind.RELU, [c1])
    c2 = fn.add_node(OpKind.CONV2D, [r1, w2], {"strides": (2, 2), "padding": (0, 0, 0, 0)})
    fn.set_results([fn.add_node(OpKind.TANH, [c2])])
    inputs = random_inputs(fn, 777)
    for mode in ("identity", "nhwc"):
        exe = gf.compile_function(fn, conv_layout=mode)
        out.append(
            {
                "name": f"convnet_{mode}",
                "fn": fdoc(fn),
                "conv_layout": mode,
                "parameter_layouts": None,
                "inputs": [tdoc(t) for t in inputs],
                "outputs": [tdoc(t) for t in gf.call(exe, inputs)],
                "listing": exe.listing(),
            }
        )
    return out


def gradient_cases(points=3):
    out = []
    cases = op_gradient_cases() + [("mlp", build_mlp(), sample_mlp_point)]
    for name, fn, sampler in cases:
        wrt = [p for p in fn.parameters if fn.nodes[p].output.element_type.is_float]
        g = gf.differentiate(fn, wrt)
        exe = gf.compile_function(g, optimize=False)
        rng = random.Random(1234 + len(out))
        pts = []
        for _ in range(points):
            point = sampler(rng)
            seed = gf.tensor_from_flat(gf.ElementType.F64, (), [1.0])
            grads = gf.call(exe, list(point) + [seed])
            pts.append({"inputs": [tdoc(t) for t in point], "grads": [tdoc(t) for t in grads]})
        out.append({"name": name, "fn": fdoc(fn), "wrt": wrt, "grad_fn": fdoc(g), "points": pts})
    return out


def _step_fixture(name, step, seed, f32=True):
    shapes = W.parameter_shapes(step)
    arrays = W.step_inputs(step, shapes, seed=seed, f32=f32)
    et = gf.ElementType.F32 if f32 else gf.ElementType.F64
    tensors = [gf.tensor_from_flat(et, a.shape, a.reshape(-1).tolist()) for a in arrays]
    t0 = time.time()
    exe = gf.compile_function(step.fn)
    outs = gf.call(exe, tensors)
    print(f"  {name}: reference call {time.time() - t0:.1f}s, {len(exe.instructions)} instructions")
    return {
        "name": name,
        "fn": fdoc(step.fn),
        "param_names": step.param_names,
        "weights": step.weight_names,
        "loss_index": step.loss_index,
        "seed": seed,
        "inputs": [tdoc(t) for t in tensors],
        "outputs": [tdoc(t) for t in outs],
        "listing": exe.listing(),
    }


def workload_cases():
    out = []
    out.append(_step_fixture("mlp_A_small", W.mlp_step(gf, batch=4, hidden=(32,)), seed=0))
    out.append(_step_fixture("mlp_E_small", W.mlp_step(gf, batch=16, in_dim=24, hidden=(24, 24), out_dim=24), seed=5))
    out.append(_step_fixture("cnn_C_small", W.cnn_step(gf, batch=2, image=8, channels=(3, 4, 4)), seed=3))
    out.append(_step_fixture("mlp_A_f64", W.mlp_step(gf, batch=3, in_dim=12, hidden=(8,), out_dim=5, f32=False), seed=7, f32=False))
    out.append(_step_fixture("resnet_D_small", W.resnet_step(gf, batch=2, image=16, widths=(4, 8), blocks=1), seed=11))
    fn = W.fused_chain(gf, rows=16, cols=64)
    arrays = W.chain_inputs(16, 64, seed=1)
    et = gf.ElementType.F32
    tensors = [gf.tensor_from_flat(et, a.shape, a.reshape(-1).tolist()) for a in arrays]
    exe = gf.compile_function(fn)
    out.append(
        {
            "name": "chain_B_small",
            "fn": fdoc(fn),
            "inputs": [tdoc(t) for t in tensors],
            "outputs": [tdoc(t) for t in gf.call(exe, tensors)],
            "listing": exe.listing(),
        }
    )
    return out


if __name__ == "__main__":
    t0 = time.time()
    which = set(sys.argv[1:]) or {"corpus", "layouts", "gradients", "workloads"}
    if "corpus" in which:
        dump("corpus.json.gz", corpus())
    if "layouts" in which:
        dump("layouts.json.gz", layout_cases())
    if "gradients" in which:
        dump("gradients.json.gz", gradient_cases())
    if "workloads" in which:
        dump("workloads.json.gz", workload_cases())
    print(f"done in {time.time() - t0:.1f}s")
