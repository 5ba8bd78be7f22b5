"""One config-A training step (and a config-E-shaped row group) through
compile_function / call, for `compute-sanitizer --tool racecheck` (shared
memory races) and `--tool memcheck` runs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1801_08058_b200 as gf
from paper_1801_08058_b200 import workloads as W

step = W.mlp_step(gf, batch=128)
arrays = W.step_inputs(step, W.parameter_shapes(step), seed=0)
exe = gf.compile_function(step.fn)
outs = gf.call(exe, [gf.tensor_from_flat(gf.ElementType.F32, a.shape, a) for a in arrays])
print("config A step ok, loss", float(outs[-1].to_numpy()), "launches", exe.num_launches)

# the fp16 pair GEMM with its fused epilogues (bias + Relu, Relu gradient,
# mask bytes, planes, column partials) on a small wide-MLP step
step = W.mlp_step(gf, batch=512, in_dim=256, hidden=(256, 256), out_dim=256)
arrays = W.step_inputs(step, W.parameter_shapes(step), seed=1)
exe = gf.compile_function(step.fn)
outs = gf.call(exe, [gf.tensor_from_flat(gf.ElementType.F32, a.shape, a) for a in arrays])
kinds = sorted({L.kind for L in exe.lowered.launches})
print("wide step ok, loss", float(outs[-1].to_numpy()), "kernel kinds", kinds)
