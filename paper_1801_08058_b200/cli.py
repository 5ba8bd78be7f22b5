"""Command-line driver over the B200 backend.

The same verbs, arguments, document formats, output naming and exit codes as
the reference CLI (`/root/reference/pkg/src/graphforge/cli.py:47-292`), so
scripts and the TypeScript bridge that shell out to `graphforge` can point
at `python -m paper_1801_08058_b200` instead:

    validate FILE                         parse + validate a function document
    run FILE --input [p<k>=]T --out DIR   compile and execute on the B200
    grad FILE [--wrt p0,p1] [--out F]     emit the gradient function
    optimize FILE [--passes ...] --out F  run rewrite passes (fold on the device)
    plan FILE                             liveness intervals + arena offsets
    dot FILE                              Graphviz digraph
    launches FILE                         the fused B200 launch list (new)

Exit codes: 0 ok, 2 validation / parse failure, 3 runtime failure, 4 usage.
GRAPHFORGE_CONV_LAYOUT=identity|nhwc picks the Conv2D layout for `run`.
`partition` is not offered: the north star excludes CPU fallback, so there
is nothing to partition between.
"""

from __future__ import annotations

import argparse
import os
import sys
from pathlib import Path

from . import errors as E
from .autodiff import differentiate
from .memory import liveness, plan_memory
from .rewrite import run_pipeline
from .serialize import export_dot, parse_function, parse_tensor, print_function, print_tensor

EXIT_OK, EXIT_VALIDATION, EXIT_RUNTIME, EXIT_USAGE = 0, 2, 3, 4


class UsageError(Exception):
    pass


def _text(path: str) -> str:
    try:
        return Path(path).read_text(encoding="utf-8")
    except OSError as exc:
        raise UsageError(f"cannot read {path}: {exc}")


def _function(path: str):
    return parse_function(_text(path))


def _conv_layout() -> str:
    value = os.environ.get("GRAPHFORGE_CONV_LAYOUT", "identity")
    if value not in ("identity", "nhwc"):
        raise UsageError(f"GRAPHFORGE_CONV_LAYOUT must be 'identity' or 'nhwc', got {value!r}")
    return value


def _bind(fn, specs: list) -> list:
    """--input entries by position, or by name p<k>=PATH."""
    named, positional = {}, []
    for spec in specs:
        name, sep, path = spec.partition("=")
        if sep and name.startswith("p") and name[1:].isdigit():
            k = int(name[1:])
            if k in named:
                raise UsageError(f"duplicate input for p{k}")
            named[k] = path
        else:
            positional.append(spec)
    paths = []
    for k in range(len(fn.parameters)):
        if k in named:
            paths.append(named.pop(k))
        elif positional:
            paths.append(positional.pop(0))
        else:
            raise UsageError(f"missing input for parameter p{k}")
    if named or positional:
        raise UsageError("more inputs than parameters")
    return [parse_tensor(_text(p)) for p in paths]


def _wrt(fn, text):
    if text is None:
        return list(fn.parameters)
    out = []
    for item in (t.strip() for t in text.split(",")):
        if not (item.startswith("p") and item[1:].isdigit()):
            raise UsageError(f"--wrt entries look like p0,p1,...; got {item!r}")
        k = int(item[1:])
        if k >= len(fn.parameters):
            raise UsageError(f"no parameter p{k}")
        out.append(fn.parameters[k])
    return out


def cmd_validate(a):
    _function(a.file)
    print("OK")
    return EXIT_OK


def cmd_run(a):
    from .runtime import call, compile_function

    fn = _function(a.file)
    tensors = _bind(fn, a.input or [])
    exe = compile_function(fn, optimize=not a.no_optimize, conv_layout=_conv_layout(),
                           parameter_layouts=[t.layout for t in tensors])
    results = call(exe, tensors)
    out = Path(a.out)
    out.mkdir(parents=True, exist_ok=True)
    for j, t in enumerate(results):
        path = out / f"result{j}.tensor.json"
        path.write_text(print_tensor(t), encoding="utf-8")
        print(f"result{j} {t.descriptor} {path}")
    return EXIT_OK


def cmd_grad(a):
    fn = _function(a.file)
    text = print_function(differentiate(fn, _wrt(fn, a.wrt)))
    if a.out:
        Path(a.out).write_text(text, encoding="utf-8")
        print(f"wrote {a.out}")
    else:
        sys.stdout.write(text)
    return EXIT_OK


def cmd_optimize(a):
    fn = _function(a.file)
    names = [n for n in (a.passes if a.passes is not None else "simplify,cse,fold").split(",") if n]
    g = run_pipeline(fn, names)
    Path(a.out).write_text(print_function(g), encoding="utf-8")
    print(f"nodes before {len(fn.nodes)} after {len(g.nodes)}")
    return EXIT_OK


def cmd_plan(a):
    fn = _function(a.file)
    plan = plan_memory(fn)
    for iv in liveness(fn):
        size = fn.nodes[iv.tensor[0]].outputs[iv.tensor[1]].byte_size
        off = plan.placements.get(iv.tensor)
        end = "inf" if iv.end == float("inf") else str(iv.end)
        print("\t".join((str(iv.tensor[0]), str(iv.start), end, "-" if off is None else str(off), str(size))))
    print(f"arena {plan.arena_size} bytes")
    return EXIT_OK


def cmd_dot(a):
    sys.stdout.write(export_dot(_function(a.file)))
    return EXIT_OK


def cmd_launches(a):
    from .runtime import prepare_function

    h = prepare_function(_function(a.file), optimize=not a.no_optimize, conv_layout=_conv_layout())
    low = h.lowered
    print(f"device arena {low.arena_bytes} bytes, {len(low.launches)} launches")
    for i, L in enumerate(low.launches):
        print(f"{i}\t{L.label}\tgrid={L.grid}\tbytes={L.algo_bytes}\tflops={L.flops}")
    return EXIT_OK


def parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="graphforge-b200", description="B200 backend for graphforge function documents")
    sub = ap.add_subparsers(dest="command", required=True)
    p = sub.add_parser("validate")
    p.add_argument("file")
    p.set_defaults(handler=cmd_validate)
    p = sub.add_parser("run")
    p.add_argument("file")
    p.add_argument("--input", action="append", metavar="[p<k>=]TENSORFILE")
    p.add_argument("--out", required=True)
    p.add_argument("--no-optimize", action="store_true")
    p.set_defaults(handler=cmd_run)
    p = sub.add_parser("grad")
    p.add_argument("file")
    p.add_argument("--wrt")
    p.add_argument("--out")
    p.set_defaults(handler=cmd_grad)
    p = sub.add_parser("optimize")
    p.add_argument("file")
    p.add_argument("--passes")
    p.add_argument("--out", required=True)
    p.set_defaults(handler=cmd_optimize)
    p = sub.add_parser("plan")
    p.add_argument("file")
    p.set_defaults(handler=cmd_plan)
    p = sub.add_parser("dot")
    p.add_argument("file")
    p.set_defaults(handler=cmd_dot)
    p = sub.add_parser("launches")
    p.add_argument("file")
    p.add_argument("--no-optimize", action="store_true")
    p.set_defaults(handler=cmd_launches)
    return ap


_VALIDATION_ERRORS = (
    E.DocumentError, E.SignatureMismatch, E.InvalidAttribute, E.NonDifferentiableOp, E.UnsupportedStride,
    E.MultipleResults, E.ShapeMismatch, E.ElementTypeMismatch, E.ArityMismatch, E.UnknownInput, E.CycleDetected,
)


def main(argv=None) -> int:
    try:
        args = parser().parse_args(argv)
    except SystemExit as exc:
        return EXIT_OK if exc.code == 0 else EXIT_USAGE
    try:
        return args.handler(args)
    except (UsageError, E.UnknownPass) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_USAGE
    except E.ValidationFailure as exc:
        for d in exc.diagnostics:
            print(str(d), file=sys.stderr)
        return EXIT_VALIDATION
    except _VALIDATION_ERRORS as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_VALIDATION
    except E.GraphError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_RUNTIME
