import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)
# a runtime-specialised kernel that fails to compile is an error here, not a
# silent fallback to the generic kernel (paper_1801_08058_b200/jit.py)
os.environ.setdefault("GFB_JIT_STRICT", "1")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run on the GPU box via gpurun)")
