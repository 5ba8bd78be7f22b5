"""Host-buffer runs (gfb_exe_run_host): `call` on page-locked host tensors
with `out=` puts the H2D / D2H copies inside the step's CUDA graph.  The
results must carry the same bits as the device-resident run of the same
executable, for multi-stream and single-stream schedules, and again after the
copy nodes are retargeted at new host buffers."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

gf = pytest.importorskip("paper_1801_08058_b200")
from paper_1801_08058_b200 import runtime  # noqa: E402
from paper_1801_08058_b200 import workloads as W  # noqa: E402


def _pinned(arrays):
    out = []
    for a in arrays:
        t = gf.pinned_tensor(gf.ElementType.F32, a.shape)
        t.buffer[...] = a.reshape(-1)
        out.append(t)
    return out


def _device_results(exe, arrays):
    ts = [gf.tensor_from_flat(gf.ElementType.F32, a.shape, a) for a in arrays]
    os.environ["GFB_HOST_GRAPH"] = "0"
    try:
        return [t.to_numpy() for t in gf.call(exe, ts)]
    finally:
        os.environ.pop("GFB_HOST_GRAPH", None)


@pytest.mark.parametrize("streams", ["4", "1"])
def test_host_run_matches_device_run(streams, monkeypatch):
    monkeypatch.setenv("GFB_STREAMS", streams)
    step = W.mlp_step(gf, batch=256, in_dim=512, hidden=(384, 256), out_dim=64)
    arrays = W.step_inputs(step, W.parameter_shapes(step), seed=3)
    exe = gf.compile_function(step.fn)
    want = _device_results(exe, arrays)
    calls = []
    orig = runtime.DeviceProgram.run_host

    def spy(self, *a, **k):
        calls.append(1)
        return orig(self, *a, **k)

    monkeypatch.setattr(runtime.DeviceProgram, "run_host", spy)
    for rep in range(3):  # rep 1 / 2: new host buffers, copy nodes retargeted
        ins = _pinned(arrays)
        outs = [gf.pinned_tensor(d.element_type, d.shape) for d, _ in exe.result_signature]
        res = gf.call(exe, ins, out=outs)
        assert res[0] is outs[0]
        for r, w in zip(res, want):
            assert np.array_equal(r.to_numpy().view(np.uint32), w.view(np.uint32))
    assert len(calls) == 3


def test_host_run_same_buffers_new_values():
    step = W.mlp_step(gf, batch=128, in_dim=256, hidden=(128,), out_dim=10)
    shapes = W.parameter_shapes(step)
    exe = gf.compile_function(step.fn)
    ins = _pinned(W.step_inputs(step, shapes, seed=0))
    outs = [gf.pinned_tensor(d.element_type, d.shape) for d, _ in exe.result_signature]
    gf.call(exe, ins, out=outs)
    arrays = W.step_inputs(step, shapes, seed=1)
    for t, a in zip(ins, arrays):
        t.buffer[...] = a.reshape(-1)
    res = [r.to_numpy().copy() for r in gf.call(exe, ins, out=outs)]
    for r, w in zip(res, _device_results(exe, arrays)):
        assert np.array_equal(r, w)


def test_pageable_buffers_take_the_plain_path(monkeypatch):
    step = W.mlp_step(gf, batch=64, in_dim=128, hidden=(64,), out_dim=10)
    arrays = W.step_inputs(step, W.parameter_shapes(step), seed=2)
    exe = gf.compile_function(step.fn)
    monkeypatch.setattr(runtime.DeviceProgram, "run_host", lambda *a, **k: pytest.fail("pageable buffers on the host-run path"))
    ins = [gf.tensor_from_flat(gf.ElementType.F32, a.shape, a) for a in arrays]
    outs = [gf.tensor_from_flat(d.element_type, d.shape, np.zeros(d.shape, np.float32)) for d, _ in exe.result_signature]
    res = gf.call(exe, ins, out=outs)
    for r, w in zip(res, _device_results(exe, arrays)):
        assert np.array_equal(r.to_numpy(), w)


@pytest.mark.parametrize("streams", ["4", "1"])
def test_host_run_input_pieces(streams, monkeypatch):
    """A large input copied in row pieces (each split / GEMM chunk waits only
    for its own piece): same bits as the device-resident run, also after the
    piece copy nodes are retargeted at new host buffers."""
    monkeypatch.setenv("GFB_STREAMS", streams)
    monkeypatch.setenv("GFB_INPUT_CHUNK_MIN_MB", "1")
    monkeypatch.setenv("GFB_INPUT_CHUNKS", "4")
    step = W.mlp_step(gf, batch=4096, in_dim=512, hidden=(256,), out_dim=256)
    arrays = W.step_inputs(step, W.parameter_shapes(step), seed=4)
    exe = gf.compile_function(step.fn)
    assert sum(":rows" in L.label for L in exe.lowered.launches) == 12  # 4 split chunks, 2 layers x 4 GEMM chunks
    want = _device_results(exe, arrays)
    for rep in range(2):
        ins = _pinned(arrays)
        outs = [gf.pinned_tensor(d.element_type, d.shape) for d, _ in exe.result_signature]
        res = gf.call(exe, ins, out=outs)
        for r, w in zip(res, want):
            assert np.array_equal(r.to_numpy().view(np.uint32), w.view(np.uint32))


def test_misaligned_device_pointer_fails_loudly():
    """gfb_exe_run rejects a caller buffer that is not 16-byte aligned (the
    kernels read caller buffers with 16-byte vector loads, cp.async and TMA)
    with GFB_ERR_INVALID instead of faulting on the device."""
    import torch

    fn = gf.Function("axpy")
    x = fn.add_parameter(gf.ElementType.F32, (1024,))
    y = fn.add_parameter(gf.ElementType.F32, (1024,))
    fn.set_results([fn.add_node(gf.OpKind.ADD, [x, y])])
    exe = gf.compile_function(fn)
    a = torch.ones(1025, device="cuda")
    b = torch.ones(1024, device="cuda")
    out = exe.allocate_outputs()
    exe.run_device([a[:1024], b], out)  # aligned: fine
    torch.cuda.synchronize()
    assert float(out[0][0]) == 2.0
    from paper_1801_08058_b200.errors import DeviceError

    with pytest.raises(DeviceError, match="16-byte aligned"):
        exe.run_device([a[1:], b], out)
