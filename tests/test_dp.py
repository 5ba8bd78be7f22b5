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
from paper_1801_08058_b200 import abi
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
    if kind == "wide":  # pair-sized layers: the fp16 GEMM, its fused epilogues and bias-gradient partials
        glob = W.mlp_step(gf, batch=1024, in_dim=256, hidden=(256, 256), out_dim=256)
        loc = W.mlp_step(gf, batch=1024 // world, in_dim=256, hidden=(256, 256), out_dim=256, loss_batch=1024)
    elif kind == "mlp":
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
    # the roots share one contiguous gradient region; buckets cover each root exactly once
    ar = [L for L in h.lowered.launches if L.kind == abi.K_ALLREDUCE]
    covered = [k for L in ar for k in L.reads]
    assert len(covered) == len(set(covered)) == len(h.allreduce)
    assert 1 <= len(ar) <= len(h.allreduce)


def test_small_roots_share_one_bucket():
    """A, C-sized steps: the loss sum is reduced where the forward divides it;
    the four gradients fit one 32 MiB bucket -> one all-reduce, issued after
    the last gradient and before the first SGD update reads one."""
    loc, h, _, _ = _dp_case("mlp", 2)
    launches = h.lowered.launches
    ar = [i for i, L in enumerate(launches) if L.kind == abi.K_ALLREDUCE]
    assert len(ar) == 2 and len(launches[ar[0]].reads) == 1 and len(launches[ar[1]].reads) == 4
    a = launches[ar[1]].args
    assert a.op == 0 and a.count >= sum(h.graph.nodes[r].output.element_count for r in h.allreduce) - 1
    first_sgd = min(i for i, L in enumerate(launches) if "Subtract" in L.label)
    assert ar[1] < first_sgd


def test_bucket_cap_splits_and_orders(monkeypatch):
    monkeypatch.setenv("GFB_BUCKET_MB", "0")  # every root its own bucket, reduced right after it lands
    loc, h, arrays, want = _dp_case("mlp", 2)
    ar = [L for L in h.lowered.launches if L.kind == abi.K_ALLREDUCE]
    assert len(ar) == len(h.allreduce)
    outs = plan_emulator.execute_ranks(h.lowered, _split_inputs(loc, arrays, 2),
                                       [(d.element_type.numpy_dtype, d.element_count) for d, _ in h.result_signature])
    for o, w in zip(outs[0], want):
        assert G.normwise(o, w.reshape(-1)) <= 1e-5


def test_max_over_batch_is_a_max_allreduce():
    """A max-reduction over the sharded axis is reduced with ncclMax, not summed."""
    def build(batch):
        fn = gf.Function("maxbatch")
        x = fn.add_parameter(gf.ElementType.F32, (batch, 5))
        w = fn.add_parameter(gf.ElementType.F32, (5,))
        m = fn.add_node(gf.OpKind.SUM, [x], {"reduction_axes": (0,), "reduction_kind": "max"})
        fn.set_results([fn.add_node(gf.OpKind.MULTIPLY, [m, w])])
        return fn, x

    fn, _ = build(8)
    loc, x = build(4)
    dp = DataParallel([x], world_size=2)
    h = host_compile(loc, data_parallel=dp)
    ar = [L for L in h.lowered.launches if L.kind == abi.K_ALLREDUCE]
    assert len(ar) == 1 and ar[0].args.op == 1
    rng = np.random.default_rng(0)
    xs, ws = rng.uniform(-1, 1, (8, 5)).astype(np.float32), rng.uniform(-1, 1, 5).astype(np.float32)
    want = interp.run_function(fn, [xs, ws])[0]
    outs = plan_emulator.execute_ranks(h.lowered, [[xs[:4], ws], [xs[4:], ws]], [(np.float32, 5)])
    for r in range(2):
        assert G.same_bits(outs[r][0], want.reshape(-1))


@pytest.mark.parametrize("kind,world", [("mlp", 2), ("mlp", 4), ("cnn", 2), ("wide", 2), ("wide-chunked", 2)])
def test_lockstep_ranks_match_global_batch(kind, world, monkeypatch):
    if kind == "wide-chunked":  # each rank's x split and multiplied in row chunks, chunk-major forward
        monkeypatch.setenv("GFB_INPUT_CHUNK_MIN_MB", "0.1")
        monkeypatch.setenv("GFB_INPUT_CHUNKS", "2")
        kind = "wide"
    loc, h, arrays, want = _dp_case(kind, world)
    if kind == "wide":
        f16 = [L for L in h.lowered.launches if L.kind == abi.K_DOT_F16P]
        assert f16 and any(L.args.epi_flags & 64 for L in f16)  # bias partials feed all-reduced Sums
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

        def allreduce(views, op=0):
            t = torch.from_numpy(views[0])
            dist.all_reduce(t, op=dist.ReduceOp.MAX if op == 1 else dist.ReduceOp.SUM)  # the real collective

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
