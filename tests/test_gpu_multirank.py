"""Data-parallel training steps across real GPUs with NCCL.

Runs only when at least two GPUs are visible (the round's GPU boxes have
one; the same path is covered there by the single-rank NCCL test and on the
CPU by the lock-step emulator and a two-process gloo run, tests/test_dp.py).
Each rank runs the step specialised to its batch shard with the partial
gradients summed by the NCCL all-reduce buckets captured in the CUDA graph;
replicas must stay bit-identical and match the global-batch oracle."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    import golden_io as G
    import paper_1801_08058_b200 as gf
    from oracle import interp
    from paper_1801_08058_b200 import workloads as W

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        glob = W.mlp_step(gf, batch=512, in_dim=256, hidden=(512,), out_dim=64)
        loc = W.mlp_step(gf, batch=512 // world, in_dim=256, hidden=(512,), out_dim=64, loss_batch=512)
        arrays = W.step_inputs(glob, W.parameter_shapes(glob), seed=4)
        names = loc.param_names
        dp = gf.DataParallel([loc.fn.parameters[names.index("x")], loc.fn.parameters[names.index("t")]], world_size=world)
        exe = gf.compile_function(loc.fn, data_parallel=dp)
        mine = []
        for name, a in zip(names, arrays):
            if name in ("x", "t"):
                n = a.shape[0] // world
                a = np.ascontiguousarray(a[rank * n:(rank + 1) * n])
            mine.append(gf.tensor_from_flat(gf.ElementType.F32, a.shape, a))
        outs = [t.to_numpy() for t in gf.call(exe, mine)]
        gathered = [None] * world
        dist.all_gather_object(gathered, outs)
        ok = all(G.same_bits(a, b) for a, b in zip(gathered[0], outs))
        if rank == 0:
            want = interp.run_function(glob.fn, arrays)
            ok = ok and all(G.normwise(o, w) <= 1e-5 for o, w in zip(outs, want))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_two_gpu_nccl_step_matches_global_batch():
    import multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert sorted(q.get(timeout=10) for _ in procs) == [(0, True), (1, True)]
