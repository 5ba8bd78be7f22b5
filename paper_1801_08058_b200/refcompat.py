"""Structural adapters from the reference package's objects to this one's.

A caller holding objects built with the reference `graphforge` package
(`/root/reference/pkg/src/graphforge`) -- a `Function` from its builder,
`differentiate` or `parse_function`, `TensorValue`s from its
`create_tensor` / `tensor_from_flat`, `Layout`s -- can hand them straight to
`compile_function` / `call` here: they are mirrored node for node (same
ids, attributes, parameters and results; `ir.py:527-603`) and value for
value (same descriptor, layout order and logical contents; `tensor.py:27-102`),
without a print/parse round trip.  Detection is duck-typed on the objects'
structure and their defining module, never on an import of the reference
(which this package must not depend on).

Errors keep the caller's taxonomy: when the objects came from the
reference package, a `GraphError` raised here is re-raised as the
reference's class of the same name (`errors.py:6-84`), so `except
graphforge.errors.SignatureMismatch` keeps working after the swap.
"""

from __future__ import annotations

import contextlib
import sys

from .errors import GraphError
from .ir import ElementType, Function, Node, OpKind, infer_output, normalize_attrs
from .layout import Layout
from .tensor import TensorValue, tensor_from_flat


def _foreign(obj, cls) -> bool:
    return not isinstance(obj, cls) and type(obj).__module__.split(".")[0] != __name__.split(".")[0]


def _enum(value, enum_cls):
    """Map a foreign enum member (or its wire string) onto ours by value."""
    if isinstance(value, enum_cls):
        return value
    return enum_cls(getattr(value, "value", value))


def _attr(v):
    if hasattr(v, "value") and type(v).__name__ == "ElementType":
        return _enum(v, ElementType)
    return v


def as_function(fn):
    """Our `Function` for `fn`: itself, or a node-for-node mirror of a
    reference-built one (node ids preserved, so listings, placements and
    pool keys match the reference's)."""
    if not _foreign(fn, Function):
        return fn
    if not (hasattr(fn, "nodes") and hasattr(fn, "parameters") and hasattr(fn, "results")):
        raise TypeError(f"not a graph Function: {type(fn).__name__}")
    g = Function(fn.name)
    for nid in sorted(fn.nodes):
        rn = fn.nodes[nid]
        kind = _enum(rn.op, OpKind)
        attrs = normalize_attrs(kind, {k: _attr(v) for k, v in dict(rn.attrs).items()})
        refs = tuple((int(r), int(p)) for r, p in rn.inputs)
        out = infer_output(kind, attrs, [g.nodes[r].outputs[p] for r, p in refs])
        g.nodes[nid] = Node(nid, kind, attrs, refs, (out,))
    g.parameters = [int(p) for p in fn.parameters]
    g.results = [(int(r), int(p)) for r, p in fn.results]
    return g


def as_layout(layout):
    if layout is None or isinstance(layout, Layout):
        return layout
    return Layout(tuple(layout.order))


def as_tensor(t):
    """Our `TensorValue` for `t` (same descriptor, layout order, contents)."""
    if not _foreign(t, TensorValue):
        return t
    d = t.descriptor
    return tensor_from_flat(_enum(d.element_type, ElementType), tuple(d.shape), t.to_flat(), as_layout(t.layout))


def foreign_errors(*objs):
    """The reference package's `errors` module if any of `objs` (or, for a
    list, its first element) was built by it, else None."""
    ours = __name__.split(".")[0]
    for obj in objs:
        if isinstance(obj, (list, tuple)):
            obj = obj[0] if obj else None
        if obj is None:
            continue
        top = type(obj).__module__.split(".")[0]
        if top not in (ours, "builtins"):
            return sys.modules.get(top + ".errors")
    return None


@contextlib.contextmanager
def caller_errors(errors_mod):
    """Re-raise our GraphError subclasses as `errors_mod`'s same-named class."""
    try:
        yield
    except GraphError as exc:
        cls = getattr(errors_mod, type(exc).__name__, None) if errors_mod is not None else None
        if not (isinstance(cls, type) and issubclass(cls, Exception)):
            raise
        try:
            new = cls(*exc.args)
        except TypeError:
            raise exc
        raise new from exc
