"""Benchmark driver (one JSON line on rank 0).

Default workload = BASELINE.json configs[1] (config B): the fused
elementwise / Broadcast / Sum chain over 64 Mi-element fp32 tensors,
`t3 = Relu(a + Broadcast(c)) * b`, results t3 and its row sums, executed
through `compile_function` / the C ABI as ONE fused launch per step.
Metric: fused-op HBM GB/s = algorithmic bytes per step (SURVEY.md §8(d):
805,572,608 B) / step time.  Inputs (805 MB) exceed the 126 MB L2, so no
flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload B|A]

N > 1 (torchrun): config B shards by rows with no collective, each rank
processing its own 64 Mi-element chain (weak scaling); value = all ranks'
bytes / max-over-ranks time.  `--impl reference` times the reference
semantics on the host CPU (the C oracle port, all host threads) on the same
config; under torchrun only rank 0 runs it.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM = 6650.0
ROWS, COLS = 65536, 1024


def peaks():
    try:
        with open(PEAKS_FILE) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), float(p.get("bf16_tflops", 1590.0)), "measured"
    except Exception:
        return FALLBACK_HBM, 1590.0, "fallback"


def chain_bytes(rows, cols, esize=4):
    # read a, b (rows*cols each) + c (cols); write t3 (rows*cols) + sums (rows)
    return esize * (3 * rows * cols + cols + rows)


class ClockSampler:
    """SM clocks and throttle reasons sampled during the timed region.

    NVML (nvidia_ml_py) is polled from a thread every 2 ms, so even a 30 ms
    timed region yields samples; nvidia-smi at 100 ms is the fallback."""

    REASONS = {  # nvmlClocksEventReason bits
        "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40, "sw_power_cap": 0x4,
    }

    def __init__(self, index: int):
        self.index = index
        self.sm, self.mx, self.reasons = [], None, set()
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.mx = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))

            def poll():
                while not self._stop.is_set():
                    try:
                        self.sm.append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
                        bits = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        for name, bit in self.REASONS.items():
                            if bits & bit:
                                self.reasons.add(name)
                    except Exception:
                        pass
                    time.sleep(0.002)

            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            self.mode = "nvml"
        except Exception:
            self.mode = "nvidia-smi"
            self._start_smi()
        return self

    def _start_smi(self):
        fields = "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_power_cap"
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={fields}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)

            def drain():
                for line in self.proc.stdout:
                    parts = [x.strip() for x in line.split(",")]
                    try:
                        self.sm.append(float(parts[0]))
                        self.mx = float(parts[1])
                    except (ValueError, IndexError):
                        continue
                    for name, v in zip(["hw_slowdown", "sw_thermal_slowdown", "hw_thermal_slowdown", "sw_power_cap"], parts[2:6]):
                        if v.lower() == "active":
                            self.reasons.add(name)

            self.thread = threading.Thread(target=drain, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def __exit__(self, *exc):
        self._stop.set()
        if self.mode == "nvidia-smi" and getattr(self, "proc", None):
            self.proc.terminate()
            self.proc.wait(timeout=5)
        elif getattr(self, "thread", None):
            self.thread.join(timeout=1)

    def summary(self):
        sm = list(self.sm)
        loaded = [x for x in sm if self.mx and x > 0.5 * self.mx] or sm
        return {"sm_mhz": float(np.median(loaded)) if loaded else None, "sm_max_mhz": self.mx,
                "reasons": sorted(self.reasons), "samples": len(sm), "source": self.mode}


def dist_setup():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_reference(rows, cols, steps, warmup, budget_s=120.0):
    """Reference semantics on the host: the oracle (C restatement of the
    reference kernels) over the fused chain, all host threads."""
    import paper_1801_08058_b200 as gf
    from oracle import interp
    from paper_1801_08058_b200 import workloads as W

    threads = interp.max_threads()
    interp.set_threads(threads)
    sample_rows = rows

    def one(r):
        fn = W.fused_chain(gf, rows=r, cols=cols)
        arrays = W.chain_inputs(r, cols)
        t0 = time.perf_counter()
        interp.run_function(fn, arrays)
        return time.perf_counter() - t0

    probe = one(min(rows, 4096)) * (rows / min(rows, 4096))
    per_step_budget = budget_s / max(1, steps + warmup)
    if probe > per_step_budget:
        sample_rows = max(256, int(rows * per_step_budget / probe) // 256 * 256)
    for _ in range(warmup):
        one(sample_rows)
    times = [one(sample_rows) for _ in range(steps)]
    t = float(np.mean(times))
    return chain_bytes(sample_rows, cols) / t / 1e9, threads, f"config B sample [{sample_rows},{cols}] per step, {steps} steps"


def bench_chain(args, ws, rank, local):
    import torch

    import paper_1801_08058_b200 as gf
    from paper_1801_08058_b200 import workloads as W
    from paper_1801_08058_b200.runtime import pinned_tensor

    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    fn = W.fused_chain(gf, rows=ROWS, cols=COLS)
    exe = gf.compile_function(fn)
    arrays = W.chain_inputs(ROWS, COLS, seed=1 + rank)
    dev_in = [torch.from_numpy(a.reshape(-1)).cuda() for a in arrays]
    outs = exe.allocate_outputs()
    stream = torch.cuda.current_stream()
    sh = stream.cuda_stream
    nbytes = chain_bytes(ROWS, COLS)
    launches_per_step = exe.num_launches

    def barrier():
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    with ClockSampler(local) as clk:
        for _ in range(args.warmup):
            exe.run_device(dev_in, outs, stream=sh)
        barrier()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(args.steps):
            exe.run_device(dev_in, outs, stream=sh)
        t1.record(stream)
        barrier()
        ms = t0.elapsed_time(t1) / args.steps
        # dominant kernel alone, same stream, for the roofline
        dom = max(range(launches_per_step), key=lambda i: exe.lowered.launches[i].algo_bytes)
        prog = exe.program()
        ptr_in = [t.data_ptr() for t in dev_in]
        ptr_out = [t.data_ptr() for t in outs]
        for _ in range(3):
            prog.run_one(dom, ptr_in, ptr_out, sh)
        k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k0.record(stream)
        kreps = max(10, args.steps)
        for _ in range(kreps):
            prog.run_one(dom, ptr_in, ptr_out, sh)
        k1.record(stream)
        torch.cuda.synchronize()
        kernel_ms = k0.elapsed_time(k1) / kreps
    ms_t = torch.tensor([ms], device="cuda")
    if ws > 1:
        torch.distributed.all_reduce(ms_t, op=torch.distributed.ReduceOp.MAX)
    ms = float(ms_t.item())

    # end to end through the public API: pinned host inputs -> call() -> pinned host results
    host_in = []
    for a in arrays:
        t = pinned_tensor(gf.ElementType.F32, a.shape)
        t.buffer[:] = a.reshape(-1)
        host_in.append(t)
    host_out = [pinned_tensor(d.element_type, d.shape) for d, _ in exe.result_signature]
    e2e_steps = max(3, min(20, args.steps))

    def timed(fn_call):
        for _ in range(2):
            fn_call()
        barrier()
        e0 = time.perf_counter()
        for _ in range(e2e_steps):
            fn_call()
        t = torch.tensor([(time.perf_counter() - e0) / e2e_steps], device="cuda")
        if ws > 1:
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    # plain call(): H2D, run, D2H back to back
    call_s = timed(lambda: gf.call(exe, host_in, out=host_out))
    # call_streamed(): row chunks with H2D / compute / D2H overlapped on 3 streams
    chunks = int(os.environ.get("GFB_BENCH_CHUNKS", 16))
    e2e_s = timed(lambda: gf.call_streamed(exe, host_in, host_out, chunks=chunks))
    h2d = sum(a.nbytes for a in arrays)
    d2h = sum(t.buffer.nbytes for t in host_out)

    hbm, _, peak_src = peaks()
    achieved = nbytes / (kernel_ms * 1e-3) / 1e9
    line = {
        "metric": "fused-op HBM GB/s (config B: Relu(a+Broadcast(c))*b + row Sum, 64Mi fp32)",
        "value": ws * nbytes / (ms * 1e-3) / 1e9,
        "unit": "GB/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (numpy PCG64 seeded U(-1,1))",
        "config": {"workload": "B: fused_chain rows=65536 cols=1024 per GPU", "bytes_per_step_per_gpu": nbytes,
                   "l2": "inputs 805 MB > 126 MB L2, no flush needed", "parallelism": f"replicas x{ws} (row shards, no collective)"},
        "e2e": {"value": ws * nbytes / e2e_s / 1e9, "unit": "GB/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e_s * 1e3,
                "api": f"paper_1801_08058_b200.call_streamed(exe, pinned host inputs, pinned host results, chunks={chunks})",
                "call_value": ws * nbytes / call_s / 1e9, "call_ms_per_step": call_s * 1e3,
                "call_api": "paper_1801_08058_b200.call(exe, pinned host tensors, out=pinned host tensors)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                     "traffic": _traffic("B"), "kernel": exe.lowered.launches[dom].label + (":jit" if dom in prog.jit_launches else ""),
                     "kernel_ms": kernel_ms,
                     "peak_source": f"{peak_src} (MEASURED_PEAKS.json hbm_gbs)"},
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clk.summary(),
    }
    return line


def _traffic(workload):
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            return json.load(fh).get(workload)
    except Exception:
        return None


def launch_times(exe, dev_in, outs, stream, reps=3):
    """Each launch alone (CUDA events on the launch stream), worst first, to stderr."""
    import torch

    prog = exe.program()
    pin = [t.data_ptr() for t in dev_in]
    pout = [t.data_ptr() for t in outs]
    rows = []
    for i, L in enumerate(exe.lowered.launches):
        prog.run_one(i, pin, pout, stream.cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            prog.run_one(i, pin, pout, stream.cuda_stream)
        e1.record(stream)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / reps
        rows.append((t, i, L))
    total = sum(r[0] for r in rows)
    sys.stderr.write(f"# per-launch times (ms), total {total:.3f}\n")
    jitted = set(getattr(prog, "jit_launches", ()))
    merged = set(getattr(prog, "skipped", ()))
    for t, i, L in sorted(rows, key=lambda r: -r[0]):
        gbs = L.algo_bytes / (t * 1e-3) / 1e9 if t else 0
        tfs = L.flops / (t * 1e-3) / 1e12 if t else 0
        label = L.label + (":jit" if i in jitted else "") + (":merged-above" if i in merged else "")
        sys.stderr.write(f"{t:9.3f} {100 * t / total:5.1f}% #{i:3d} {label:28s} grid={L.grid} {gbs:8.1f} GB/s {tfs:7.1f} TF/s\n")


def bench_gemm(args, local):
    """One config-E layer as a graph: Dot([8192, 4096], [4096, 4096]) on tcgen05."""
    import torch

    import paper_1801_08058_b200 as gf

    torch.cuda.set_device(local)
    m = args.batch or 8192
    fn = gf.Function("layer")
    a = fn.add_parameter(gf.ElementType.F32, (m, 4096))
    w = fn.add_parameter(gf.ElementType.F32, (4096, 4096))
    fn.set_results([fn.add_node(gf.OpKind.DOT, [a, w])])
    exe = gf.compile_function(fn)
    rng = np.random.default_rng(0)
    dev = [torch.from_numpy(rng.uniform(-1, 1, size=s).astype(np.float32).reshape(-1)).cuda() for s in ((m, 4096), (4096, 4096))]
    outs = exe.allocate_outputs()
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        exe.run_device(dev, outs, stream=stream.cuda_stream)
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        exe.run_device(dev, outs, stream=stream.cuda_stream)
    t1.record(stream)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / args.steps
    if args.launch_times:
        launch_times(exe, dev, outs, stream)
    flops = 2 * m * 4096 * 4096
    return {"metric": "F32 Dot TFLOP/s (config E layer, 3xTF32 tcgen05)", "value": flops / (ms * 1e-3) / 1e12,
            "unit": "TFLOP/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "config": {"workload": f"G: Dot [{m},4096]x[4096,4096]", "launches": exe.num_launches}}


def bench_conv(args, local):
    """One config-D layer-1 convolution as a graph (3x3, 64->64, 56x56,
    batch 128, NHWC): forward (Conv2D) and data gradient (ConvBackpropData),
    both on gfb_conv_tcx_kernel.  `value` counts the two convolutions' flops
    over the whole step (the two Relu producers included)."""
    import torch

    import paper_1801_08058_b200 as gf

    torch.cuda.set_device(local)
    n = args.batch or 128
    C = int(os.environ.get("GFB_BENCH_C", 64))   # shape overrides for kernel studies
    K = int(os.environ.get("GFB_BENCH_K", 64))
    H = W = int(os.environ.get("GFB_BENCH_HW", 56))
    F32 = gf.ElementType.F32
    fn = gf.Function("conv_layer")
    x = fn.add_parameter(F32, (n, C, H, W))
    f = fn.add_parameter(F32, (K, C, 3, 3))
    d = fn.add_parameter(F32, (n, K, H, W))
    pad = {"padding": (1, 1, 1, 1)}
    # the activations come from a producer in the arena, as inside a network
    # (tensor maps need fixed addresses): Relu in front of each convolution
    rx, rd = fn.add_node(gf.OpKind.RELU, [x]), fn.add_node(gf.OpKind.RELU, [d])
    y = fn.add_node(gf.OpKind.CONV2D, [rx, f], {"strides": (1, 1), **pad})
    dx = fn.add_node(gf.OpKind.CONV_BACKPROP_DATA, [rd, f], {"data_shape": (n, C, H, W), **pad}, allow_internal=True)
    fn.set_results([y, dx])
    nhwc = gf.Layout((0, 2, 3, 1))
    exe = gf.compile_function(fn, conv_layout="nhwc", parameter_layouts=[nhwc, None, nhwc])
    rng = np.random.default_rng(0)
    dev = [torch.from_numpy(rng.uniform(-1, 1, size=s).astype(np.float32).reshape(-1)).cuda()
           for s in ((n, C, H, W), (K, C, 3, 3), (n, K, H, W))]
    outs = exe.allocate_outputs()
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        exe.run_device(dev, outs, stream=stream.cuda_stream)
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        exe.run_device(dev, outs, stream=stream.cuda_stream)
    t1.record(stream)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / args.steps
    if args.launch_times:
        launch_times(exe, dev, outs, stream)
    flops = 2 * (2 * n * H * W * K * C * 9)  # both convolutions
    return {"metric": "F32 conv TFLOP/s (config D layer-1 3x3 conv fwd + dgrad, 3xTF32 tcgen05, fused gather)",
            "value": flops / (ms * 1e-3) / 1e12, "unit": "TFLOP/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "config": {"workload": f"H: Conv2D + ConvBackpropData [{n},{C},{H},{W}] -> {K} channels, 3x3 NHWC",
                       "launches": exe.num_launches}}


def _step_for(workload, batch=None, ws=1):
    """(step graph, per-GPU batch, description); `batch` is the GLOBAL batch."""
    import paper_1801_08058_b200 as gf
    from paper_1801_08058_b200 import workloads as W

    if workload == "A":
        g = batch or 128
        return W.mlp_step(gf, batch=g // ws, loss_batch=g), g // ws, "A: MLP 784-512-10"
    if workload == "C":
        g = batch or 256
        return (W.cnn_step(gf, batch=g // ws, loss_batch=g), g // ws,
                "C: CNN 32x32x3, conv 3->16->32, maxpool, fc 8192->10")
    if workload == "D":
        g = batch or 128 * ws  # config D is weak-scaled: 128 images per GPU
        return (W.resnet_step(gf, batch=g // ws, loss_batch=g), g // ws,
                "D: ResNet-18-style 224x224, NHWC layout assignment")
    if workload == "E":
        g = batch or 65536
        return (W.mlp_step(gf, batch=g // ws, in_dim=4096, hidden=(4096,) * 7, out_dim=4096, loss_batch=g), g // ws,
                "E: wide MLP 4096 x 8 layers")
    raise ValueError(workload)


def bench_step(args, ws, rank, local):
    """Training step (fwd + autodiff bwd + SGD as one Function), samples/s.

    Under torchrun the global batch is sharded over the ranks (strong
    scaling): each rank runs the graph specialised to batch/ws with the loss
    still divided by the global batch, and the partial gradients are summed
    by NCCL all-reduces captured inside the step's CUDA graph."""
    import torch

    import paper_1801_08058_b200 as gf
    from paper_1801_08058_b200 import workloads as W

    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    step, batch, desc = _step_for(args.workload, args.batch, ws)
    t_compile = time.perf_counter()
    dp = None
    if ws > 1 or args.dp:
        names = step.param_names
        dp = gf.DataParallel([step.fn.parameters[names.index("x")], step.fn.parameters[names.index("t")]], world_size=ws)
    exe = gf.compile_function(step.fn, data_parallel=dp, conv_layout="nhwc" if args.workload == "D" else "identity")
    t_compile = time.perf_counter() - t_compile
    shapes = W.parameter_shapes(step)
    arrays = W.step_inputs(step, shapes, seed=rank)
    dev_in = [torch.from_numpy(np.ascontiguousarray(a).reshape(-1)).cuda() for a in arrays]
    del arrays
    outs = exe.allocate_outputs()
    stream = torch.cuda.current_stream()
    def barrier():
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    with ClockSampler(local) as clk:
        for _ in range(args.warmup):
            exe.run_device(dev_in, outs, stream=stream.cuda_stream)
        barrier()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(args.steps):
            exe.run_device(dev_in, outs, stream=stream.cuda_stream)
        t1.record(stream)
        barrier()
    ms = t0.elapsed_time(t1) / args.steps
    if ws > 1:
        ms_t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(ms_t, op=torch.distributed.ReduceOp.MAX)
        ms = float(ms_t.item())
    if args.launch_times:
        launch_times(exe, dev_in, outs, stream)
    flops = sum(L.flops for L in exe.lowered.launches)
    _, tf_peak, _ = peaks()
    gbatch = batch * ws
    return {
        "metric": f"training-step samples/sec (config {desc}, global batch {gbatch}, fwd+autodiff bwd+SGD)",
        "value": gbatch / (ms * 1e-3), "unit": "samples/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak" if args.workload == "D" else "strong",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": {"workload": desc, "global_batch": gbatch, "batch_per_gpu": batch,
                                        "parallelism": f"dp{ws}", "launches": exe.num_launches,
                                        "allreduces": len(getattr(exe, "allreduce", ()) or ()),
                                        "flops_per_step_per_gpu": flops, "arena_bytes": exe.lowered.arena_bytes,
                                        "compile_s": t_compile},
        "achieved_tflops": ws * flops / (ms * 1e-3) / 1e12,
        "gpu_launches": exe.num_launches * args.steps, "clocks": clk.summary(),
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="B", choices=["B", "A", "C", "D", "E", "G", "H"])
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--launch-times", action="store_true", help="per-launch timing table to stderr")
    ap.add_argument("--dp", action="store_true", help="data-parallel plan even at one GPU (NCCL all-reduces)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    ws, rank, local = dist_setup()

    if args.impl == "reference":
        if rank != 0:
            return
        value, threads, sample = cpu_reference(ROWS, COLS, args.steps, args.warmup)
        line = {
            "impl": "reference", "metric": "fused-op HBM GB/s (config B: Relu(a+Broadcast(c))*b + row Sum, 64Mi fp32)",
            "value": value, "unit": "GB/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "B: fused_chain rows=65536 cols=1024 per GPU"},
            "cpu_baseline": {"value": value, "unit": "GB/s", "cores": threads, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line))
        return

    if args.workload == "G":
        line = bench_gemm(args, local)
    elif args.workload == "H":
        line = bench_conv(args, local)
    else:
        line = bench_chain(args, ws, rank, local) if args.workload == "B" else bench_step(args, ws, rank, local)
    if rank == 0 and ws == 1 and not args.no_cpu_baseline and args.workload == "B":
        value, threads, sample = cpu_reference(ROWS, COLS, 2, 1, budget_s=30.0)
        line["cpu_baseline"] = {"value": value, "unit": "GB/s", "cores": threads, "kind": "port", "sample": sample}
    if rank == 0:
        print(json.dumps(line))
    if ws > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
