"""The reference's own interpreter tests, run against this backend.

`graphforge.compile_function` / `graphforge.call` of the UNMODIFIED
reference package are replaced by this package's (which accept the
reference's own `Function` / `TensorValue` / `Layout` objects through
`refcompat`), then the reference test module
`pkg/tests/test_interpreter.py` is imported and its known-answer, compile
and call/arena test classes are collected here (the
binding a maintainer would add is the same two-line swap).

Where the reference comes from: `baseline/_ref` (installed offline by
scripts/install_reference.sh; git-ignored, shipped to the GPU box), else
`/root/reference/pkg` in the build container.  Without either the module
is skipped.  TestFallback (partitioned CPU fallback) and TestCreateTensor
(reference-only tensor construction) are out of scope.
"""

import importlib.util
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_CANDIDATES = [(os.path.join(ROOT, "baseline", "_ref"), os.path.join(ROOT, "baseline", "_ref", "tests")),
               ("/root/reference/pkg/src", "/root/reference/pkg/tests")]
_src, _tests = next(((s, t) for s, t in _CANDIDATES
                     if os.path.isdir(os.path.join(s, "graphforge")) and os.path.isfile(os.path.join(t, "test_interpreter.py"))),
                    (None, None))
if _src is None:
    pytest.skip("reference package not installed (scripts/install_reference.sh)", allow_module_level=True)

pytestmark = pytest.mark.gpu

for p in (_tests, _src):
    if p not in sys.path:
        sys.path.append(p)
graphforge = importlib.import_module("graphforge")

import paper_1801_08058_b200 as gfb  # noqa: E402


def _compile(fn, **kw):
    return gfb.compile_function(fn, **kw)


def _call(exe, inputs, **kw):
    return gfb.call(exe, inputs, **kw)


graphforge.compile_function = _compile
graphforge.call = _call
_spec = importlib.util.spec_from_file_location("graphforge_ref_test_interpreter", os.path.join(_tests, "test_interpreter.py"))
_mod = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(_mod)

TestKernels = _mod.TestKernels
TestCompile = _mod.TestCompile
TestCall = _mod.TestCall


def test_backend_is_swapped():
    assert _mod.compile_function is _compile and _mod.call is _call
