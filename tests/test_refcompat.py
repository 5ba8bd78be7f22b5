"""refcompat: reference-built objects mirror structurally (CPU)."""

import os
import sys

import numpy as np
import pytest

from paper_1801_08058_b200.ir import topological_order
from paper_1801_08058_b200.refcompat import as_function, as_layout, as_tensor
from paper_1801_08058_b200.serialize import print_function

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for src in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(os.path.join(src, "graphforge")):
        if src not in sys.path:
            sys.path.append(src)
        break
graphforge = pytest.importorskip("graphforge")


def _mlp_ref():
    gf = graphforge
    fn = gf.Function("mlp")
    x = fn.add_parameter(gf.ElementType.F32, (4, 3))
    w = fn.add_parameter(gf.ElementType.F32, (3, 2))
    c = fn.add_constant(gf.ElementType.F32, (2,), [0.5, -0.25])
    h = fn.add_node(gf.OpKind.DOT, [x, w])
    h = fn.add_node(gf.OpKind.ADD, [h, fn.add_node(gf.OpKind.BROADCAST, [c], {"output_shape": (4, 2), "broadcast_axes": (0,)})])
    p = gf.build_softmax(fn, fn.add_node(gf.OpKind.RELU, [h]), 1)
    fn.set_results([fn.add_node(gf.OpKind.SUM, [p], {"reduction_axes": (0, 1)})])
    return fn, [x, w]


def test_function_mirrors_node_for_node():
    fn, wrt = _mlp_ref()
    g = graphforge.differentiate(fn, wrt)  # a reference-built gradient graph, ids with gaps allowed
    ours = as_function(g)
    assert sorted(ours.nodes) == sorted(g.nodes) and ours.parameters == g.parameters
    assert ours.results == [tuple(r) for r in g.results]
    assert topological_order(ours) == graphforge.topological_order(g)
    # byte-identical wire documents: the reference printer on its graph, ours on the mirror
    assert print_function(ours) == graphforge.print_function(g)
    assert as_function(ours) is ours


def test_tensor_and_layout_mirror():
    t = graphforge.tensor_from_flat(graphforge.ElementType.F32, (2, 3), [0.1 * i for i in range(6)], graphforge.Layout((1, 0)))
    o = as_tensor(t)
    assert o.layout.order == (1, 0) and o.to_flat() == t.to_flat()
    assert np.asarray(o.to_flat()).dtype == np.float64
    assert as_layout(graphforge.Layout((0, 2, 1))).order == (0, 2, 1)


def test_errors_keep_the_callers_taxonomy():
    from paper_1801_08058_b200.errors import SignatureMismatch
    from paper_1801_08058_b200.refcompat import caller_errors, foreign_errors

    fn, _ = _mlp_ref()
    mod = foreign_errors(fn)
    assert mod is graphforge.errors
    with pytest.raises(graphforge.errors.SignatureMismatch):
        with caller_errors(mod):
            raise SignatureMismatch("x")
    with pytest.raises(SignatureMismatch):  # our own objects: our own classes
        with caller_errors(foreign_errors(as_function(fn))):
            raise SignatureMismatch("x")
