"""Runtime-specialised elementwise kernels (paper_1801_08058_b200/jit.py).

CPU: every fused elementwise launch of the golden corpus and workloads has a
generated kernel, and a sample of them compiles with NVRTC for sm_100a (NVRTC
needs no GPU).  GPU: specialised kernels are bit-identical to the generic VM
on the corpus and the workload steps, with every eligible launch specialised.
"""

import numpy as np
import pytest

import golden_io as G
from hostcompile import host_compile

from paper_1801_08058_b200 import abi, jit


def _ew_args(h):
    recs, blob = h.lowered.pack()
    for i, L in enumerate(h.lowered.launches):
        if L.kind in jit.KINDS:
            r = recs[i]
            yield L, r, abi.EwArgs.from_buffer_copy(blob[r.arg_offset:r.arg_offset + r.arg_size])


def _plans():
    for case in G.load("corpus.json.gz")[::5]:
        fn = G.fn_of(case["fn"])
        yield host_compile(fn), host_compile(fn, optimize=False)
    for case in G.load("workloads.json.gz"):
        fn = G.fn_of(case["fn"])
        yield (host_compile(fn, conv_layout="nhwc" if case["name"].startswith("resnet") else "identity"),)


def test_every_ew_launch_generates(monkeypatch):
    monkeypatch.setenv("GFB_ROWFUSE", "0")  # the unfused plans: every VM mode appears
    n = modes = 0
    seen = set()
    for plans in _plans():
        for h in plans:
            for L, r, a in _ew_args(h):
                src, smem = jit.generate(L.kind, a, r.block[0])
                assert "None" not in src and "gfb_jit_ew" in src
                assert smem >= 0
                n += 1
                seen.add((a.mode, a.red_kind, bool(a.ty_ext)))
    assert n > 100
    assert {(1, 0, False), (2, 0, False), (2, 1, False), (1, 1, False)} <= seen


def test_nvrtc_compiles_sample(tmp_path, monkeypatch):
    pytest.importorskip("ctypes")
    try:
        jit._lib_nvrtc()
    except RuntimeError as exc:
        pytest.skip(str(exc))
    monkeypatch.setenv("GFB_JIT_CACHE", str(tmp_path))
    monkeypatch.setenv("GFB_ROWFUSE", "0")
    picked = {}
    for plans in _plans():
        for h in plans:
            for L, r, a in _ew_args(h):
                key = (L.kind, a.mode, a.red_kind, a.split > 1, a.wpr > 1, bool(a.ty_ext))
                picked.setdefault(key, (L, r, a))
    assert len(picked) >= 4
    for L, r, a in list(picked.values())[:8]:
        cubin = jit.compile_cubin(jit.generate(L.kind, a, r.block[0])[0])
        assert cubin[:4] == b"\x7fELF"


def test_single_block_launches_merge(tmp_path, monkeypatch):
    """Consecutive single-block launches (config A's softmax / loss chain)
    form one group, generate one kernel with block barriers between the
    members and plain (coherent) loads, and compile."""
    case = next(c for c in G.load("workloads.json.gz") if c["name"] == "mlp_A_small")
    h = host_compile(G.fn_of(case["fn"]))
    recs, blob = h.lowered.pack()
    todo = [i for i, L in enumerate(h.lowered.launches) if L.kind in jit.KINDS]
    groups = jit._groups(h.lowered.launches, recs, todo)
    big = max(groups, key=len)
    assert len(big) >= 3 and all(tuple(recs[i].grid) == (1, 1, 1) for i in big)
    assert sorted(i for g in groups for i in g) == todo
    members = [(h.lowered.launches[i].kind, abi.EwArgs.from_buffer_copy(blob[recs[i].arg_offset:recs[i].arg_offset + recs[i].arg_size]))
               for i in big]
    src, smem = jit.generate_merged(members, recs[big[0]].block[0])
    assert src.count("__syncthreads();\nm") == len(big) - 1 and "__ldg" not in src.split("#define GFB_LOADV")[1]
    try:
        jit._lib_nvrtc()
    except RuntimeError as exc:
        pytest.skip(str(exc))
    monkeypatch.setenv("GFB_JIT_CACHE", str(tmp_path))
    assert jit.compile_cubin(src)[:4] == b"\x7fELF"


# ---------------------------------------------------------------- GPU
gf = pytest.importorskip("paper_1801_08058_b200")


def _run(fn, tensors, conv_layout="identity", optimize=True):
    exe = gf.compile_function(fn, optimize=optimize, conv_layout=conv_layout)
    return exe, [t.to_numpy() for t in gf.call(exe, tensors)]


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["mlp_A_small", "mlp_E_small", "cnn_C_small", "mlp_A_f64", "resnet_D_small", "chain_B_small"])
def test_workload_jit_bit_identical(name, monkeypatch):
    case = next(c for c in G.load("workloads.json.gz") if c["name"] == name)
    fn = G.fn_of(case["fn"])
    tensors = [G.tensor_of(d) for d in case["inputs"]]
    layout = "nhwc" if name.startswith("resnet") else "identity"
    monkeypatch.setenv("GFB_JIT", "1")
    monkeypatch.setenv("GFB_ROWFUSE", "0")  # row fusion changes the plan; it is tested in test_rowfuse.py
    monkeypatch.setenv("GFB_STAGED", "auto")  # the same plan with and without specialisation
    monkeypatch.setattr(jit, "MIN_BYTES", 0)
    exe, spec = _run(fn, tensors, layout)
    assert exe.program().jit_launches, "no launch was specialised"
    if name.startswith("mlp_A") and jit.MERGE:
        assert exe.program().skipped, "no single-block launches were merged"
    monkeypatch.setenv("GFB_JIT", "0")
    exe0, gen = _run(fn, tensors, layout)
    assert not exe0.program().jit_launches
    for a, b in zip(spec, gen):
        assert G.same_bits(a, b), name


@pytest.mark.gpu
def test_corpus_jit_bit_identical(monkeypatch):
    monkeypatch.setenv("GFB_JIT", "1")
    monkeypatch.setenv("GFB_ROWFUSE", "0")
    monkeypatch.setenv("GFB_STAGED", "auto")
    monkeypatch.setattr(jit, "MIN_BYTES", 0)
    cases = G.load("corpus.json.gz")[::4]
    spec = [_run(G.fn_of(c["fn"]), [G.tensor_of(d) for d in c["inputs"]])[1] for c in cases]
    monkeypatch.setenv("GFB_JIT", "0")
    for c, outs in zip(cases, spec):
        gen = _run(G.fn_of(c["fn"]), [G.tensor_of(d) for d in c["inputs"]])[1]
        for a, b in zip(outs, gen):
            assert G.same_bits(a, b), c["seed"]
            if a.dtype.kind == "f":
                assert np.array_equal(np.isnan(a), np.isnan(b))


def _long_rows_fn(rows=4, cols=65536):
    fn = gf.Function("long_rows")
    a = fn.add_parameter(gf.ElementType.F32, (rows, cols))
    b = fn.add_parameter(gf.ElementType.F32, (rows, cols))
    fn.set_results([fn.add_node(gf.OpKind.SUM, [fn.add_node(gf.OpKind.MULTIPLY, [a, b])], {"reduction_axes": (1,)})])
    return fn


def test_chunkwise_mode_generates_and_compiles(tmp_path, monkeypatch):
    """A few-long-rows Sum lowers to the chunk-wise staged mode (3, split 1),
    whose generated kernel walks 16-byte pieces like the VM's sidx()."""
    monkeypatch.setenv("GFB_STAGED", "auto")
    h = host_compile(_long_rows_fn())
    modes = [(a.mode, a.split) for _, _, a in _ew_args(h)]
    assert (3, 1) in modes
    L, r, a = next(x for x in _ew_args(h) if x[2].mode == 3)
    src, _ = jit.generate(L.kind, a, r.block[0])
    assert "constexpr int V = 4;" in src and "piece * 32u * V + lane * V" in src
    try:
        jit._lib_nvrtc()
    except RuntimeError as exc:
        pytest.skip(str(exc))
    monkeypatch.setenv("GFB_JIT_CACHE", str(tmp_path))
    assert jit.compile_cubin(src)[:4] == b"\x7fELF"


@pytest.mark.gpu
def test_chunkwise_jit_bit_identical(monkeypatch):
    """the generated chunk-wise kernel folds the same elements in
    the same order as gfb_ew_staged_kernel -> identical row-sum bits."""
    fn = _long_rows_fn()
    rng = np.random.default_rng(7)
    tensors = [gf.tensor_from_flat(gf.ElementType.F32, (4, 65536), rng.uniform(-1, 1, 4 * 65536).astype(np.float32))
               for _ in range(2)]
    monkeypatch.setenv("GFB_STAGED", "auto")
    monkeypatch.setattr(jit, "MIN_BYTES", 0)
    monkeypatch.setenv("GFB_JIT", "1")
    exe, spec = _run(fn, tensors)
    assert any(exe.lowered.launches[i].kind == abi.K_EWS_F32 for i in exe.program().jit_launches)
    monkeypatch.setenv("GFB_JIT", "0")
    _, gen = _run(fn, tensors)
    assert G.same_bits(spec[0], gen[0])
