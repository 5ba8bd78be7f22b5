"""Function / tensor documents (the reference wire format).

Reads and writes the JSON documents of the reference
(`/root/reference/pkg/src/graphforge/serialize.py:94-280`, format in
`SPEC.md:406-413`): nodes sorted by id with fields (id, op, attrs, inputs),
attribute keys sorted, NaN / +-Inf as the strings "NaN" / "Inf" / "-Inf".
The golden fixtures under `tests/golden/` are documents printed by the
reference itself, so this module is how parity inputs reach the B200 path.
"""

from __future__ import annotations

import json
import math

import numpy as np

from .errors import DocumentSyntaxError, UnknownOp, ValidationFailure
from .ir import (
    OP_BY_WIRE_NAME,
    ConstantData,
    Diagnostic,
    ElementType,
    Function,
    Node,
    OpKind,
    infer_output,
    normalize_attrs,
    validate_function,
)
from .layout import Layout
from .tensor import TensorValue, coerce_array, create_tensor

_SPECIAL = {"NaN": math.nan, "Inf": math.inf, "-Inf": -math.inf}


def _enc(v):
    if isinstance(v, float):
        if math.isnan(v):
            return "NaN"
        if math.isinf(v):
            return "Inf" if v > 0 else "-Inf"
    return v


def _encode_data(values, et: ElementType) -> list:
    values = list(values)
    return [_enc(float(v)) for v in values] if et.is_float else [(bool(v) if et is ElementType.BOOL else int(v)) for v in values]


def _decode(v, et: ElementType):
    if isinstance(v, str):
        if not et.is_float or v not in _SPECIAL:
            raise DocumentSyntaxError(f"bad numeric entry {v!r}")
        return _SPECIAL[v]
    return v


def _require(cond, message):
    if not cond:
        raise DocumentSyntaxError(message)


def function_to_document(fn: Function) -> dict:
    nodes = []
    for nid in sorted(fn.nodes):
        node = fn.nodes[nid]
        attrs = {}
        et = node.attrs.get("element_type")
        for key in sorted(node.attrs):
            v = node.attrs[key]
            if isinstance(v, ElementType):
                v = v.value
            elif key == "data":
                v = _encode_data(v, et)
            elif isinstance(v, tuple):
                v = list(v)
            attrs[key] = v
        nodes.append({"id": nid, "op": node.op.wire_name, "attrs": attrs, "inputs": [[r, p] for r, p in node.inputs]})
    return {
        "name": fn.name,
        "nodes": nodes,
        "parameters": list(fn.parameters),
        "results": [[r, p] for r, p in fn.results],
    }


def print_function(fn: Function) -> str:
    return json.dumps(function_to_document(fn), indent=2) + "\n"


def _is_ref(x) -> bool:
    return isinstance(x, list) and len(x) == 2 and all(isinstance(v, int) for v in x)


def _attrs_from_json(kind: OpKind, raw: dict) -> dict:
    attrs = dict(raw)
    if kind is OpKind.CONSTANT and isinstance(attrs.get("data"), list):
        et_name = attrs.get("element_type")
        if et_name in ("F32", "F64"):
            et = ElementType(et_name)
            attrs["data"] = [_decode(v, et) for v in attrs["data"]]
    return normalize_attrs(kind, attrs)


def document_to_function(doc) -> Function:
    _require(isinstance(doc, dict), "document must be a JSON object")
    extra = set(doc) - {"name", "nodes", "parameters", "results"}
    _require(not extra, f"unknown document fields {sorted(extra)}")
    _require(isinstance(doc.get("name"), str), "'name' must be a string")
    for key in ("nodes", "parameters", "results"):
        _require(isinstance(doc.get(key), list), f"'{key}' must be a list")

    specs = {}
    for entry in doc["nodes"]:
        _require(isinstance(entry, dict), "node entries must be objects")
        extra = set(entry) - {"id", "op", "attrs", "inputs"}
        _require(not extra, f"unknown node fields {sorted(extra)}")
        nid = entry.get("id")
        _require(isinstance(nid, int) and not isinstance(nid, bool), "node id must be an integer")
        _require(nid not in specs, f"duplicate node id {nid}")
        if entry.get("op") not in OP_BY_WIRE_NAME:
            raise UnknownOp(f"unknown op {entry.get('op')!r}")
        attrs = entry.get("attrs", {})
        _require(isinstance(attrs, dict), f"node {nid}: attrs must be an object")
        inputs = entry.get("inputs", [])
        _require(isinstance(inputs, list), f"node {nid}: inputs must be a list")
        for ref in inputs:
            _require(_is_ref(ref), f"node {nid}: inputs must be [id, port] pairs")
        specs[nid] = (OP_BY_WIRE_NAME[entry["op"]], attrs, tuple((r[0], r[1]) for r in inputs))

    diags = []
    fn = Function(doc["name"])
    pending = dict(specs)
    progress = True
    while pending and progress:
        ready = sorted(n for n, (_, _, refs) in pending.items() if all(r in fn.nodes for r, _ in refs))
        progress = bool(ready)
        for nid in ready:
            kind, raw, refs = pending.pop(nid)
            try:
                attrs = _attrs_from_json(kind, raw)
                bad = [(r, p) for r, p in refs if p >= len(fn.nodes[r].outputs)]
                if bad:
                    diags.append(Diagnostic("unknown-input", nid, f"bad port {bad[0][0]}:{bad[0][1]}"))
                    continue
                out = infer_output(kind, attrs, [fn.nodes[r].outputs[p] for r, p in refs])
            except DocumentSyntaxError:
                raise
            except Exception as exc:
                diags.append(Diagnostic("bad-attrs", nid, str(exc)))
                continue
            fn.nodes[nid] = Node(nid, kind, attrs, refs, (out,))
    for nid, (_, _, refs) in sorted(pending.items()):
        missing = [r for r, _ in refs if r not in specs]
        if missing:
            diags.append(Diagnostic("unknown-input", nid, f"missing inputs {missing}"))
        else:
            diags.append(Diagnostic("cycle", nid, "node participates in a cycle"))
    for pid in doc["parameters"]:
        _require(isinstance(pid, int), "'parameters' entries must be node ids")
        fn.parameters.append(pid)
    for ref in doc["results"]:
        _require(_is_ref(ref), "'results' entries must be [id, port] pairs")
        fn.results.append((ref[0], ref[1]))
    diags = diags or validate_function(fn)
    if diags:
        raise ValidationFailure(diags)
    return fn


def parse_function(text: str) -> Function:
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as exc:
        raise DocumentSyntaxError(exc.msg, position=exc.pos)
    return document_to_function(doc)


def tensor_to_document(t: TensorValue) -> dict:
    storage = t.to_host().buffer
    return {
        "element_type": t.element_type.value,
        "shape": list(t.shape),
        "order": list(t.layout.order),
        "data": _encode_data(storage.tolist(), t.element_type),
    }


def print_tensor(t: TensorValue) -> str:
    return json.dumps(tensor_to_document(t), indent=2) + "\n"


def document_to_tensor(doc) -> TensorValue:
    _require(isinstance(doc, dict), "tensor document must be a JSON object")
    extra = set(doc) - {"element_type", "shape", "order", "data"}
    _require(not extra, f"unknown tensor fields {sorted(extra)}")
    try:
        et = ElementType(doc.get("element_type"))
    except ValueError:
        raise DocumentSyntaxError(f"unknown element type {doc.get('element_type')!r}")
    shape = doc.get("shape")
    _require(isinstance(shape, list) and all(isinstance(d, int) and d >= 0 for d in shape),
             "'shape' must be a list of non-negative integers")
    order = doc.get("order", list(range(len(shape))))
    _require(isinstance(order, list), "'order' must be a list")
    data = doc.get("data")
    _require(isinstance(data, list), "'data' must be a list")
    t = create_tensor(et, tuple(shape), Layout(tuple(order)))
    _require(len(data) == t.descriptor.element_count,
             f"data length {len(data)} != element count {t.descriptor.element_count}")
    decoded = [_decode(v, et) for v in data]
    t.buffer[:] = coerce_array(et, np.array(decoded, dtype=object) if et is ElementType.I64 else decoded)
    return t


def parse_tensor(text: str) -> TensorValue:
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as exc:
        raise DocumentSyntaxError(exc.msg, position=exc.pos)
    return document_to_tensor(doc)


def export_dot(fn: Function) -> str:
    lines = [f'digraph "{fn.name}" {{']
    for nid in sorted(fn.nodes):
        node = fn.nodes[nid]
        lines.append(f'  n{nid} [label="{nid}: {node.op.wire_name} {list(node.output.shape)}"];')
    for nid in sorted(fn.nodes):
        for ref, _ in fn.nodes[nid].inputs:
            lines.append(f"  n{ref} -> n{nid};")
    lines.append("}")
    return "\n".join(lines) + "\n"
