"""A/B timing of tensor-core GEMM variants on config-E shapes, interleaved in
one process (the power cap moves clocks between runs and boxes, so only
same-process alternation compares kernels fairly).

    python scripts/gemm_ab.py VAR=a,b [VAR=c,d ...]   e.g. GFB_TC_PERSIST=1,0
Each variant's executables are compiled with its environment; then the
variants' runs alternate for several rounds; prints ms and TF/s per shape."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1801_08058_b200 as gf

K, F32 = gf.OpKind, gf.ElementType.F32
B, W = int(os.environ.get("AB_BATCH", 65536)), 4096


def graphs():
    fwd = gf.Function("fwd")  # z = relu(h) . W: A K-major in the arena, B = W (split)
    h = fwd.add_parameter(F32, (B, W))
    w = fwd.add_parameter(F32, (W, W))
    rh = fwd.add_node(K.RELU, [h])
    fwd.set_results([fwd.add_node(K.DOT, [rh, w]), fwd.add_node(K.SUM, [rh], {"reduction_axes": (0,)})])
    dw = gf.Function("dw")  # dW = relu(h)^T . (-dz): both MN-major
    h2 = dw.add_parameter(F32, (B, W))
    dz = dw.add_parameter(F32, (B, W))
    rh2, nd = dw.add_node(K.RELU, [h2]), dw.add_node(K.NEGATE, [dz])
    ht = dw.add_node(K.RESHAPE, [rh2], {"input_order": (1, 0), "output_shape": (W, B)})
    dw.set_results([dw.add_node(K.DOT, [ht, nd]), dw.add_node(K.SUM, [rh2], {"reduction_axes": (0,)}),
                    dw.add_node(K.SUM, [nd], {"reduction_axes": (0,)})])
    return {"fwd": fwd, "dW": dw}


def main():
    variants = []
    for arg in sys.argv[1:]:
        k, vals = arg.split("=")
        variants = [dict(v, **{k: x}) for v in (variants or [{}]) for x in vals.split(",")]
    variants = variants or [{}]
    rng = np.random.default_rng(0)
    data = torch.from_numpy(rng.uniform(-1, 1, size=(2, B * W)).astype(np.float32)).cuda()
    wt = torch.from_numpy(rng.uniform(-1 / 64, 1 / 64, size=W * W).astype(np.float32)).cuda()
    s = torch.cuda.current_stream()
    exes = []
    for v in variants:
        old = {k: os.environ.get(k) for k in v}
        os.environ.update(v)
        per = {}
        for name, fn in graphs().items():
            exe = gf.compile_function(fn)
            ins = [data[0], wt] if name == "fwd" else [data[0], data[1]]
            gi = [i for i, L in enumerate(exe.lowered.launches) if L.label.startswith(("dot_tc", "dot_f16"))]  # GEMM (+ split-K pass)
            per[name] = (exe, ins, exe.allocate_outputs(), gi)
        exes.append(per)
        for k, x in old.items():
            if x is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = x
    res = {(i, n): [] for i in range(len(variants)) for n in ("fwd", "dW")}
    for rnd in range(6):
        for i, per in enumerate(exes):
            for name, (exe, ins, outs, gi) in per.items():
                prog = exe.program()
                pin, pout = [t.data_ptr() for t in ins], [t.data_ptr() for t in outs]
                exe.run_device(ins, outs, stream=s.cuda_stream)  # planes / lo for this graph
                for _ in range(2):
                    for g in gi:
                        prog.run_one(g, pin, pout, s.cuda_stream)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                for _ in range(5):
                    for g in gi:
                        prog.run_one(g, pin, pout, s.cuda_stream)
                e1.record(s)
                torch.cuda.synchronize()
                if rnd:
                    res[(i, name)].append(e0.elapsed_time(e1) / 5)
    flops = 2 * B * W * W
    for (i, name), ts in res.items():
        t = float(np.median(ts))
        print(f"{str(variants[i]):40s} {name:4s} {t:7.3f} ms  {flops / t / 1e9:7.1f} TF/s  (min {min(ts):.3f}, max {max(ts):.3f})")


if __name__ == "__main__":
    main()
