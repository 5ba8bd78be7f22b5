"""The C ABI: ctypes mirror matches include/gfb200.h; the library exports it."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_1801_08058_b200 import abi, compiler
from paper_1801_08058_b200.runtime import library_path

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gfb200.h")


def _probe(tmp_path):
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "gfb200.h"', "int main(void) {"]
    for cname, cls in abi.STRUCTS.items():
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for fname, _ in cls._fields_:
            lines.append(f'printf("{cname}.{fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("return 0; }")
    src = tmp_path / "probe.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-I", os.path.dirname(HEADER), str(src), "-o", str(exe)], check=True)
    return subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout


def test_struct_layout_matches_header(tmp_path):
    out = _probe(tmp_path)
    got = dict(line.rsplit(" ", 1) for line in out.strip().splitlines())
    for cname, cls in abi.STRUCTS.items():
        assert int(got[f"{cname} size"]) == ctypes.sizeof(cls), cname
        for fname, _ in cls._fields_:
            assert int(got[f"{cname}.{fname}"]) == getattr(cls, fname).offset, (cname, fname)


def test_library_exports_every_declared_entry_point():
    from paper_1801_08058_b200 import _build

    _build.build()
    declared = set(re.findall(r"^(?:int|const char\*)\s+(gfb_\w+)\(", open(HEADER).read(), re.M))
    assert {"gfb_exe_create", "gfb_exe_run", "gfb_exe_destroy", "gfb_comm_create"} <= declared
    lib = ctypes.CDLL(library_path())  # loads without a GPU
    for name in sorted(declared):
        assert hasattr(lib, name), name


def test_kernels_are_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", library_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("d", [1, 2, 3, 4, 5, 7, 10, 12, 64, 100, 255, 256, 257, 784, 1000, 4096, 65536, 2**20 + 1, 2**30, 2**31 - 1])
def test_magic_division(d):
    import numpy as np

    mul, sh = compiler.magic_u31(d)
    rng = np.random.default_rng(d)
    n = np.concatenate([np.arange(0, 5000), rng.integers(0, 2**31, 20000), np.array([2**31 - 1, d - 1, d, d + 1]) % (2**31)])
    n = n.astype(np.uint64)
    q = n if mul == 0 else (n * np.uint64(mul)) >> np.uint64(32 + sh)
    assert np.array_equal(q, n // np.uint64(d))


def test_launch_shared_memory_matches_kernels():
    """The lowering's dynamic shared-memory sizes equal the kernels' own
    configurations (host-only entry points of libgfb200.so; no GPU)."""
    from paper_1801_08058_b200 import compiler as Cm

    lib = ctypes.CDLL(library_path())
    assert lib.gfb_tc_smem_bytes(0) == Cm.TC_SMEM
    assert lib.gfb_tc_smem_bytes(1) == Cm.TC_SMEM_W
    assert lib.gfb_stem_smem_bytes() == Cm.STEM_SMEM
    assert lib.gfb_stemh_smem_bytes() == Cm.STEMH_SMEM
    assert lib.gfb_stemwh_smem_bytes() == Cm.STEMWH_SMEM
    assert lib.gfb_f16_pair_smem_bytes() == Cm.F16_SMEM_PAIR
    assert lib.gfb_tc_pair_smem_bytes() == Cm.TC_SMEM_PAIR
    for bn in (64, 128):
        assert lib.gfb_tcg_smem_bytes(bn) == Cm.TCG_SMEM[bn]
        assert lib.gfb_tcgw_smem_bytes(bn) == Cm.TCGW_SMEM[bn]
