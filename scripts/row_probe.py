"""Time the row-fused loss head of config E alone (and the unfused head)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1801_08058_b200 as gf
from paper_1801_08058_b200 import abi, workloads as W

R = int(os.environ.get("ROWS", 65536)); C = int(os.environ.get("COLS", 4096))
step = W.mlp_step(gf, batch=R, in_dim=8, hidden=(), out_dim=C, loss_batch=65536)
arrays = W.step_inputs(step, W.parameter_shapes(step), seed=1, x_range=(-1, 1))
exe = gf.compile_function(step.fn)
dev = [torch.from_numpy(np.ascontiguousarray(a).reshape(-1)).cuda() for a in arrays]
outs = exe.allocate_outputs()
s = torch.cuda.current_stream()
prog = exe.program()
pin, pout = [t.data_ptr() for t in dev], [t.data_ptr() for t in outs]
for i, L in enumerate(exe.lowered.launches):
    for _ in range(3):
        prog.run_one(i, pin, pout, s.cuda_stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(10):
        prog.run_one(i, pin, pout, s.cuda_stream)
    e1.record(s)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 10
    print(f"{t:8.3f} ms  {L.label:40s} grid={L.grid} block={L.block} {L.algo_bytes / t / 1e6:8.1f} GB/s", flush=True)
