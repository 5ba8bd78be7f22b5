"""Pin the CPU oracle against outputs of the reference itself.

The golden documents were produced by graphforge's own interpreter
(tests/golden/make_golden.py).  The oracle must reproduce every one of them
bit for bit (NaNs compared as a class) — that is what makes it usable as
the parity checker for the B200 kernels.
"""

import numpy as np
import pytest

import golden_io as G
from oracle import interp


def _run(case, key):
    fn = G.fn_of(case["fn"])
    inputs = [G.logical(d) for d in case["inputs"]]
    outs = interp.run_function(fn, inputs)
    want = [G.logical(d) for d in case[key]]
    assert len(outs) == len(want)
    for o, w in zip(outs, want):
        assert G.same_bits(o, w), (case.get("seed", case.get("name")), o, w)


@pytest.mark.parametrize("seed", range(200))
def test_corpus_bit_exact(seed):
    _run(G.load("corpus.json.gz")[seed], "outputs_noopt")


@pytest.mark.parametrize("idx", range(12))
def test_layout_cases_bit_exact(idx):
    case = G.load("layouts.json.gz")[idx]
    _run(case, "outputs")


def test_gradient_graphs_bit_exact():
    for case in G.load("gradients.json.gz"):
        g = G.fn_of(case["grad_fn"])
        for pt in case["points"]:
            inputs = [G.logical(d) for d in pt["inputs"]] + [np.array(1.0)]
            outs = interp.run_function(g, inputs)
            for o, w in zip(outs, pt["grads"]):
                assert G.same_bits(o, G.logical(w)), case["name"]


@pytest.mark.parametrize("name", ["mlp_A_small", "mlp_E_small", "cnn_C_small", "mlp_A_f64", "chain_B_small", "resnet_D_small"])
def test_workload_steps_bit_exact(name):
    case = next(c for c in G.load("workloads.json.gz") if c["name"] == name)
    _run(case, "outputs")


def test_thread_count_does_not_change_bits():
    case = next(c for c in G.load("workloads.json.gz") if c["name"] == "mlp_A_small")
    fn = G.fn_of(case["fn"])
    inputs = [G.logical(d) for d in case["inputs"]]
    interp.set_threads(1)
    one = interp.run_function(fn, inputs)
    interp.set_threads(4)
    four = interp.run_function(fn, inputs)
    interp.set_threads(1)
    for a, b in zip(one, four):
        assert G.same_bits(a, b)
