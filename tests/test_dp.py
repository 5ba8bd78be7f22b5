"""Data parallelism: partial-root analysis and a lock-step
multi-rank execution of the exact plans, checked against the single-GPU
(global batch) oracle; plus a real 2-process gloo run of the same plans."""

import os
import socket

import numpy as np
import pytest

import golden_io as G
import plan_emulator
from hostcompile import host_compile
from oracle import interp

import paper_1801_08058_b200 as gf
from paper_1801_08058_b200 import workloads as W
from paper_1801_08058_b200.dp import DataParallel


def _split_inputs(step, arrays, world):
    names = step.param_names
    per = []
    for r in range(world):
        ins = []
        for name, a in zip(names, arrays):
            if name in ("x", "t"):
                n = a.shape[0] // world
                ins.append(np.ascontiguousarray(a[r * n:(r + 1) * n]))
            else:
                ins.append(a)
        per.append(ins)
    return per


def _dp_case(kind, world):
    if kind == "mlp":
        glob = W.mlp_step(gf, batch=16, in_dim=12, hidden=(16,), out_dim=5)
        loc = W.mlp_step(gf, batch=16 // world, in_dim=12, hidden=(16,), out_dim=5, loss_batch=16)
    else:
        glob = W.cnn_step(gf, batch=4, image=8, channels=(3, 4, 4))
        loc = W.cnn_step(gf, batch=4 // world, image=8, channels=(3, 4, 4), loss_batch=4)
    arrays = W.step_inputs(glob, W.parameter_shapes(glob), seed=3)
    want = interp.run_function(glob.fn, arrays)
    names = loc.param_names
    dp = DataParallel([loc.fn.parameters[names.index("x")], loc.fn.parameters[names.index("t")]], world_size=world)
    h = host_compile(loc.fn, data_parallel=dp)
    return loc, h, arrays, want


@pytest.mark.parametrize("kind", ["mlp", "cnn"])
def test_partial_roots(kind):
    loc, h, _, _ = _dp_case(kind, 2)
    ops = sorted(h.graph.nodes[r].op.wire_name for r in h.allreduce)
    if kind == "mlp":
        assert ops == ["Dot", "Dot", "Sum", "Sum", "Sum"]  # dW1, dW2, db1, db2, loss
    else:
        assert ops == ["ConvBackpropFilter", "ConvBackpropFilter", "Dot", "Sum"]
    assert sum(1 for L in h.lowered.launches if L.label.startswith("allreduce")) == len(h.allreduce)


@pytest.mark.parametrize("kind,world", [("mlp", 2), ("mlp", 4), ("cnn", 2)])
def test_lockstep_ranks_match_global_batch(kind, world):
    loc, h, arrays, want = _dp_case(kind, world)
    specs = [(d.element_type.numpy_dtype, d.element_count) for d, _ in h.result_signature]
    outs = plan_emulator.execute_ranks(h.lowered, _split_inputs(loc, arrays, world), specs)
    for r in range(world):
        for o, w in zip(outs[r], want):
            assert G.normwise(o, w.reshape(-1)) <= 1e-5
    for r in range(1, world):  # replicas stay bit-identical
        for a, b in zip(outs[0], outs[r]):
            assert G.same_bits(a, b)


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        loc, h, arrays, want = _dp_case("mlp", world)
        specs = [(d.element_type.numpy_dtype, d.element_count) for d, _ in h.result_signature]

        def allreduce(views):
            t = torch.from_numpy(views[0])
            dist.all_reduce(t)  # the real collective, over processes

        mine = _split_inputs(loc, arrays, world)[rank]
        outs = plan_emulator.execute_ranks(h.lowered, [mine], specs, allreduce=allreduce)[0]
        ok = all(G.normwise(o, w.reshape(-1)) <= 1e-5 for o, w in zip(outs, want))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_two_process_gloo_allreduce():
    import multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    results = sorted(q.get(timeout=5) for _ in procs)
    assert results == [(0, True), (1, True)]


def test_rebatch_chunk_graph_equals_row_slices():
    """streaming.rebatch: the chunk graph computes exactly the rows of the full graph."""
    from hostcompile import emulate

    from paper_1801_08058_b200.streaming import rebatch

    fn = W.fused_chain(gf, rows=64, cols=256)
    sub = rebatch(fn, fn.parameters[:2], 4)
    assert [sub.nodes[p].output.shape for p in sub.parameters] == [(16, 256), (16, 256), (256,)]
    arrays = W.chain_inputs(64, 256)
    h = host_compile(sub)
    full = interp.run_function(fn, arrays)
    for i in range(4):
        part = [arrays[0][16 * i:16 * (i + 1)], arrays[1][16 * i:16 * (i + 1)], arrays[2]]
        outs = emulate(h, [gf.tensor_from_flat(gf.ElementType.F32, a.shape, a) for a in part])
        assert G.same_bits(outs[0], full[0][16 * i:16 * (i + 1)])
        assert G.normwise(outs[1], full[1][16 * i:16 * (i + 1)]) <= 1e-6


def test_rebatch_rejects_batch_reductions():
    from paper_1801_08058_b200.errors import UnsupportedOp
    from paper_1801_08058_b200.streaming import rebatch

    step = W.mlp_step(gf, batch=8, in_dim=4, hidden=(4,), out_dim=3)
    with pytest.raises(UnsupportedOp):
        rebatch(step.fn, [step.fn.parameters[0]], 2)
