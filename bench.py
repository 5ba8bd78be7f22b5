"""Benchmark driver (one JSON line on rank 0).

Headline (BASELINE.json metric "training-step samples/sec per graph ...
at 1/2/4/8 B200"): config E, the wide-MLP (4096 x 8 layers) training step
-- forward, autodiff backward and SGD as ONE Function -- at global batch
65536, batch-sharded over the N GPUs (strong scaling) with the partial
gradients summed by NCCL all-reduces captured inside the step's CUDA graph.
Metric: samples/s = 65536 / step time (max over ranks).  Inputs (x alone is
1 GiB at N=1) exceed the 126 MB L2, so no flush is needed between steps.

The same line carries config B (BASELINE.json's "fused-op HBM GB/s": the
fused Relu(a + Broadcast(c)) * b + row Sum chain over 64 Mi fp32) as the
`secondary` block, with its own roofline.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload E|B|A|C|D|G|H]

`--gpus N` without torchrun re-launches itself under torch.distributed.run
with N ranks (one per GPU, rendezvous on 127.0.0.1).  `--impl reference`
times the reference semantics on the host CPU (the C oracle port, all host
threads) on the same workload and metric, at a bounded sample batch; under
torchrun only rank 0 runs it.
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


def maybe_relaunch(args):
    """`--gpus N` outside torchrun: re-exec this script under
    torch.distributed.run with N local ranks (rendezvous on 127.0.0.1)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def tf32_peak():
    """Measured tcgen05 kind::tf32 dense TFLOP/s (scripts/mma_probe.cu on a
    B200 of this pool, profiles/tf32_peak.json), else the nominal 1,100."""
    try:
        with open(os.path.join(ROOT, "profiles", "tf32_peak.json")) as fh:
            p = json.load(fh)
        return float(p["tf32_dense_tflops"]), float(p.get("tf32_dense_tflops_sustained", p["tf32_dense_tflops"])), \
            "measured (profiles/tf32_peak.json, scripts/mma_probe.cu)"
    except Exception:
        return 1100.0, 1100.0, "nominal (no profiles/tf32_peak.json)"


def f16_peak():
    """Measured tcgen05 kind::f16 dense TFLOP/s, sustained (same probe)."""
    try:
        with open(os.path.join(ROOT, "profiles", "tf32_peak.json")) as fh:
            return float(json.load(fh)["f16_dense_tflops_sustained"])
    except Exception:
        return 2 * tf32_peak()[1]


def _traffic(workload):
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            return json.load(fh).get(workload)
    except Exception:
        return None


E_DESC = ("E: wide MLP 4096 x 8 layers (+bias, Relu), softmax cross-entropy loss, fwd + autodiff bwd + SGD "
          "as one Function, global batch 65536")


def step_config(workload, ws, batch=None):
    """The `config` dict of a training-step line (identical in both arms)."""
    g = {"A": 128, "C": 256, "D": 128 * ws, "E": 65536}[workload] if batch is None else batch
    desc = {"A": "A: MLP 784-512-10", "C": "C: CNN 32x32x3, conv 3->16->32, maxpool, fc 8192->10",
            "D": "D: ResNet-18-style 224x224, NHWC layout assignment", "E": E_DESC}[workload]
    return {"workload": desc, "global_batch": g, "batch_per_gpu": g // ws, "parallelism": f"dp{ws}",
            "scaling": "weak" if workload == "D" else "strong",
            "l2": "per-step inputs exceed the 126 MB L2 (E: x alone is 1 GiB per GPU at N=1); no flush needed"
            if workload in ("D", "E") else "small step: inputs L2-resident between steps (latency-bound config)"}


def _step_for(workload, batch=None, ws=1):
    """(step graph, per-GPU batch); `batch` is the GLOBAL batch."""
    import paper_1801_08058_b200 as gf
    from paper_1801_08058_b200 import workloads as W

    g = step_config(workload, ws, batch)["global_batch"]
    if workload == "A":
        return W.mlp_step(gf, batch=g // ws, loss_batch=g), g // ws
    if workload == "C":
        return W.cnn_step(gf, batch=g // ws, loss_batch=g), g // ws
    if workload == "D":
        return W.resnet_step(gf, batch=g // ws, loss_batch=g), g // ws
    if workload == "E":
        return W.wide_mlp_step(gf, batch=g // ws, loss_batch=g), g // ws
    raise ValueError(workload)


# ---------------------------------------------------------------------------
# reference arm / CPU baseline: the oracle port of the reference interpreter


def _oracle_step_seconds(workload, batch, threads, global_batch):
    import paper_1801_08058_b200 as gf
    from oracle import interp
    from paper_1801_08058_b200 import workloads as W

    interp.set_threads(threads)
    if workload == "E":
        step = W.wide_mlp_step(gf, batch=batch, loss_batch=global_batch)
    else:
        step, _ = _step_for(workload, batch, 1)
    arrays = W.step_inputs(step, W.parameter_shapes(step), seed=0, x_range=W.x_range_of(workload),
                           conv_gain=W.conv_gain_of(workload))
    t0 = time.perf_counter()
    interp.run_function(step.fn, arrays)
    return time.perf_counter() - t0


def cpu_step_sample(workload, per_step_budget, threads, global_batch):
    """Largest power-of-two sample batch whose oracle step fits the budget:
    two probes give the fixed cost (SGD over every parameter, which does not
    shrink with the batch) and the per-sample cost."""
    t16 = _oracle_step_seconds(workload, 16, threads, global_batch)
    t64 = _oracle_step_seconds(workload, 64, threads, global_batch)
    per = max(1e-6, (t64 - t16) / 48.0)
    fixed = max(0.0, t16 - 16 * per)
    b = 16
    while b * 2 <= min(global_batch, 512) and fixed + 2 * b * per <= per_step_budget:
        b *= 2
    return b


def reference_arm(args, ws):
    """The reference interpreter's semantics timed on the host cores (the C
    oracle port, all threads), on our arm's workload, metric and config."""
    from oracle import interp

    threads = interp.max_threads()
    wl = args.workload
    if wl == "B":
        value, _, sample = cpu_reference_chain(ROWS, COLS, args.steps, min(args.warmup, 1), threads)
        line = {"impl": "reference", "metric": CHAIN_METRIC, "value": value, "unit": "GB/s", "n_gpus": ws,
                "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": chain_config(ws)}
        unit = "GB/s"
    else:
        cfg = step_config(wl, ws, args.batch)
        g = cfg["global_batch"]
        budget = float(os.environ.get("GFB_REF_BUDGET_S", 120.0)) / max(1, args.steps + 1)
        b = cpu_step_sample(wl, budget, threads, g) if wl == "E" else min(g, 2)
        _oracle_step_seconds(wl, b, threads, g)  # warm-up
        times = [_oracle_step_seconds(wl, b, threads, g) for _ in range(args.steps)]
        t = float(np.mean(times))
        value = b / t
        sample = f"oracle step at batch {b} (of {g}), loss divided by {g}, {args.steps} steps, mean {t:.2f} s/step"
        line = {"impl": "reference", "metric": step_metric(wl), "value": value, "unit": "samples/s", "n_gpus": ws,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
                "scaling": cfg["scaling"], "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": cfg}
        unit = "samples/s"
    line["cpu_baseline"] = {"value": value, "unit": unit, "cores": threads, "kind": "port", "sample": sample,
                            "cpu": _cpu_model()}
    line["e2e"] = {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    return line


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


CHAIN_METRIC = "fused-op HBM GB/s (config B: Relu(a+Broadcast(c))*b + row Sum, 64Mi fp32)"


def chain_config(ws):
    return {"workload": "B: fused_chain rows=65536 cols=1024 per GPU",
            "l2": "inputs 805 MB > 126 MB L2, no flush needed", "parallelism": f"replicas x{ws} (row shards, no collective)"}


def step_metric(workload):
    return f"training-step samples/sec per graph (config {step_config(workload, 1)['workload'].split(':')[0]})"


def cpu_reference_chain(rows, cols, steps, warmup, threads, budget_s=120.0):
    """Config B on the oracle (C restatement of the reference kernels)."""
    import paper_1801_08058_b200 as gf
    from oracle import interp
    from paper_1801_08058_b200 import workloads as W

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


# ---------------------------------------------------------------------------
# GPU arm


def _barrier(ws):
    import torch

    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()


def _max_over_ranks(x, ws):
    import torch

    t = torch.tensor([x], device="cuda", dtype=torch.float64)
    if ws > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


def _own_launches(exe) -> int:
    """Kernels of ours one run launches (NCCL's all-reduce kernels and memset nodes excluded)."""
    from paper_1801_08058_b200 import abi

    return exe.num_launches - sum(1 for L in exe.lowered.launches if L.kind in (abi.K_ALLREDUCE, abi.K_MEMSET))


def _time_launch(exe, idx, dev_in, outs, stream, reps):
    """Average duration of launch `idx` alone, CUDA events on its stream."""
    import torch

    prog = exe.program()
    pin = [t.data_ptr() for t in dev_in]
    pout = [t.data_ptr() for t in outs]
    for _ in range(2):
        prog.run_one(idx, pin, pout, stream.cuda_stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        prog.run_one(idx, pin, pout, stream.cuda_stream)
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


_KIND_NAMES = {34: "gfb_gemm_f16p_kernel", 39: "gfb_conv_tcxh_kernel<64>", 40: "gfb_conv_tcxh_kernel<128>",
               41: "gfb_conv_tcgwh_kernel<64>", 42: "gfb_conv_tcgwh_kernel<128>", 44: "gfb_conv_stemh_kernel<0,0,0>", 45: "gfb_conv_stemh_kernel<3,7,7>", 46: "gfb_conv_stemwh_kernel<3,7,7>", 19: "gfb_gemm_tc2_kernel", 12: "gfb_gemm_tc_kernel<128>", 14: "gfb_gemm_tc_kernel<256>",
               22: "gfb_conv_tcx_kernel<64>", 23: "gfb_conv_tcx_kernel<128>", 17: "gfb_conv_tcg_kernel<64>",
               18: "gfb_conv_tcg_kernel<128>", 24: "gfb_conv_tcgg_kernel<64>", 25: "gfb_conv_tcgg_kernel<128>",
               28: "gfb_conv_tcgw_kernel<64>", 29: "gfb_conv_tcgw_kernel<128>", 32: "gfb_conv_stem_kernel",
               10: "gfb_dot_kernel<float>", 26: "gfb_dot_thread_kernel<float>", 15: "gfb_dot_small_m_kernel<float>"}


def launch_times(exe, dev_in, outs, stream, reps=3, to_stderr=True):
    """Each launch alone (CUDA events on the launch stream); worst first."""
    prog = exe.program()
    rows = []
    for i, L in enumerate(exe.lowered.launches):
        rows.append((_time_launch(exe, i, dev_in, outs, stream, reps), i, L))
    total = sum(r[0] for r in rows)
    if to_stderr:
        sys.stderr.write(f"# per-launch times (ms), total {total:.3f}\n")
        jitted = set(getattr(prog, "jit_launches", ()))
        merged = set(getattr(prog, "skipped", ()))
        for t, i, L in sorted(rows, key=lambda r: -r[0]):
            gbs = L.algo_bytes / (t * 1e-3) / 1e9 if t else 0
            tfs = L.flops / (t * 1e-3) / 1e12 if t else 0
            label = L.label + (":jit" if i in jitted else "") + (":merged-above" if i in merged else "")
            sys.stderr.write(f"{t:9.3f} {100 * t / total:5.1f}% #{i:3d} {label:28s} grid={L.grid} {gbs:8.1f} GB/s {tfs:7.1f} TF/s\n")
    return rows, total


def bench_chain(args, ws, rank, local, e2e=True):
    import torch

    import paper_1801_08058_b200 as gf
    from paper_1801_08058_b200 import workloads as W
    from paper_1801_08058_b200.runtime import pinned_tensor

    fn = W.fused_chain(gf, rows=ROWS, cols=COLS)
    exe = gf.compile_function(fn)
    arrays = W.chain_inputs(ROWS, COLS, seed=1 + rank)
    dev_in = [torch.from_numpy(a.reshape(-1)).cuda() for a in arrays]
    outs = exe.allocate_outputs()
    stream = torch.cuda.current_stream()
    sh = stream.cuda_stream
    nbytes = chain_bytes(ROWS, COLS)
    steps = args.steps if args.workload == "B" else max(20, min(args.steps, 200))

    with ClockSampler(local) as clk:
        for _ in range(args.warmup):
            exe.run_device(dev_in, outs, stream=sh)
        _barrier(ws)
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(steps):
            exe.run_device(dev_in, outs, stream=sh)
        t1.record(stream)
        _barrier(ws)
    ms = _max_over_ranks(t0.elapsed_time(t1) / steps, ws)
    dom = max(range(len(exe.lowered.launches)), key=lambda i: exe.lowered.launches[i].algo_bytes)
    kernel_ms = _time_launch(exe, dom, dev_in, outs, stream, max(10, steps))
    hbm, _, peak_src = peaks()
    achieved = nbytes / (kernel_ms * 1e-3) / 1e9
    prog = exe.program()
    line = {
        "metric": CHAIN_METRIC, "value": ws * nbytes / (ms * 1e-3) / 1e9, "unit": "GB/s", "n_gpus": ws,
        "steps": steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (numpy PCG64 seeded U(-1,1))",
        "config": dict(chain_config(ws), bytes_per_step_per_gpu=nbytes),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                     "traffic": _traffic("B"), "kernel": exe.lowered.launches[dom].label + (":jit" if dom in prog.jit_launches else ""),
                     "kernel_ms": kernel_ms, "algorithmic_bytes": nbytes,
                     "peak_source": f"{peak_src} (MEASURED_PEAKS.json hbm_gbs)"},
        "gpu_launches": _own_launches(exe) * steps, "clocks": clk.summary(),
    }
    if e2e:
        host_in = []
        for a in arrays:
            t = pinned_tensor(gf.ElementType.F32, a.shape)
            t.buffer[:] = a.reshape(-1)
            host_in.append(t)
        host_out = [pinned_tensor(d.element_type, d.shape) for d, _ in exe.result_signature]
        n = max(3, min(20, steps))

        def timed(call):
            for _ in range(2):
                call()
            _barrier(ws)
            e0 = time.perf_counter()
            for _ in range(n):
                call()
            return _max_over_ranks((time.perf_counter() - e0) / n, ws)

        call_s = timed(lambda: gf.call(exe, host_in, out=host_out))
        chunks = int(os.environ.get("GFB_BENCH_CHUNKS", 16))
        e2e_s = timed(lambda: gf.call_streamed(exe, host_in, host_out, chunks=chunks))
        line["e2e"] = {"value": ws * nbytes / e2e_s / 1e9, "unit": "GB/s",
                       "h2d_bytes_per_step": sum(a.nbytes for a in arrays),
                       "d2h_bytes_per_step": sum(t.buffer.nbytes for t in host_out), "ms_per_step": e2e_s * 1e3,
                       "api": f"paper_1801_08058_b200.call_streamed(exe, pinned host inputs, pinned host results, chunks={chunks})",
                       "call_value": ws * nbytes / call_s / 1e9, "call_ms_per_step": call_s * 1e3,
                       "call_api": "paper_1801_08058_b200.call(exe, pinned host tensors, out=pinned host tensors)"}
    return line


def bench_step(args, ws, rank, local):
    """Training step (fwd + autodiff bwd + SGD as one Function), samples/s.

    At N > 1 the global batch is sharded over the ranks: each rank runs the
    graph specialised to batch/N with the loss still divided by the global
    batch, and the partial gradients are summed by NCCL all-reduces captured
    inside the step's CUDA graph (dp.py; gradient buckets in compiler.py)."""
    import torch

    import paper_1801_08058_b200 as gf
    from paper_1801_08058_b200 import workloads as W
    from paper_1801_08058_b200.runtime import pinned_tensor

    wl = args.workload
    cfg = step_config(wl, ws, args.batch)
    step, batch = _step_for(wl, args.batch, ws)
    t_compile = time.perf_counter()
    dp = None
    if ws > 1 or args.dp:
        names = step.param_names
        dp = gf.DataParallel([step.fn.parameters[names.index("x")], step.fn.parameters[names.index("t")]], world_size=ws)
    exe = gf.compile_function(step.fn, data_parallel=dp, conv_layout="nhwc" if wl == "D" else "identity")
    t_compile = time.perf_counter() - t_compile
    shapes = W.parameter_shapes(step)
    arrays = W.step_inputs(step, shapes, seed=rank, x_range=W.x_range_of(wl), conv_gain=W.conv_gain_of(wl))
    dev_in = [torch.from_numpy(np.ascontiguousarray(a).reshape(-1)).cuda() for a in arrays]
    outs = exe.allocate_outputs()
    stream = torch.cuda.current_stream()

    with ClockSampler(local) as clk:
        for _ in range(args.warmup):
            exe.run_device(dev_in, outs, stream=stream.cuda_stream)
        _barrier(ws)
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(args.steps):
            exe.run_device(dev_in, outs, stream=stream.cuda_stream)
        t1.record(stream)
        _barrier(ws)
    ms = _max_over_ranks(t0.elapsed_time(t1) / args.steps, ws)
    gbatch = cfg["global_batch"]
    flops = sum(L.flops for L in exe.lowered.launches)

    # dominant kernel (the largest-flop launch: a tcgen05 GEMM / conv) alone,
    # same stream; and every launch alone for its share of the step
    rows, total = launch_times(exe, dev_in, outs, stream, reps=2, to_stderr=args.launch_times)
    # the dominant kernel: the kernel kind with the largest share of the step's
    # device time (config E: the pair GEMM, 23 launches); achieved = its
    # launches' useful flops over their summed durations (each launch timed
    # alone with CUDA events on the launch stream)
    by_kind: dict = {}
    for t, i, L in rows:
        if L.flops:
            by_kind.setdefault(L.kind, []).append((t, i, L))
    dom_kind = max(by_kind, key=lambda k: sum(t for t, _, _ in by_kind[k]))
    dom_rows = by_kind[dom_kind]
    dom_ms = sum(t for t, _, _ in dom_rows)
    dom_flops = sum(L.flops for _, _, L in dom_rows)
    kernel_ms = dom_ms / len(dom_rows)
    tf32, tf32_sus, tf_src = tf32_peak()
    if dom_kind in (34, 39, 40, 41, 42, 44, 45, 46):  # 2xFP16: three kind::f16 MMAs per useful product
        mma_sus, mma_name = f16_peak(), "2xFP16 useful ceiling = kind::f16"
    else:  # 3xTF32: three kind::tf32 MMAs per useful product
        mma_sus, mma_name = tf32_sus, "3xTF32 useful ceiling = kind::tf32"
    useful_peak = mma_sus / 3.0
    achieved = dom_flops / (dom_ms * 1e-3) / 1e12
    gemm_ms = sum(t for t, i, L in rows if L.flops)
    best = max(dom_rows, key=lambda r: r[2].flops / r[0])
    Ld = dom_rows[0][2]
    line = {
        "metric": step_metric(wl), "value": gbatch / (ms * 1e-3), "unit": "samples/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": cfg["scaling"], "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (numpy PCG64 seeded; random-init weights of the config's architecture)",
        "config": cfg,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": useful_peak, "unit": "TFLOP/s",
                     "frac": achieved / useful_peak, "traffic": _traffic(wl),
                     "kernel": f"{_KIND_NAMES.get(dom_kind, dom_kind)} ({len(dom_rows)} launches per step, e.g. {Ld.label})",
                     "kernel_ms": kernel_ms, "algorithmic_flops": dom_flops // len(dom_rows),
                     "step_share": dom_ms / total if total else None,
                     "best_launch": {"label": best[2].label, "ms": best[0], "tflops": best[2].flops / (best[0] * 1e-3) / 1e12},
                     "peak_source": f"{mma_name} dense {mma_sus:.0f} TFLOP/s / 3, {tf_src}",
                     "tensor_pipe_frac": 3 * achieved / mma_sus,
                     "frac_of_measured_bf16": achieved / peaks()[1]},
        "step_detail": {"launches": exe.num_launches, "allreduces": sum(1 for L in exe.lowered.launches if L.label.startswith("allreduce")),
                        "flops_per_step_per_gpu": flops, "achieved_tflops_step": ws * flops / (ms * 1e-3) / 1e12,
                        "gemm_launch_ms_sum": gemm_ms, "launch_ms_sum": total,
                        "arena_bytes": exe.lowered.arena_bytes, "compile_s": t_compile},
        "gpu_launches": _own_launches(exe) * args.steps, "clocks": clk.summary(),
    }

    # end to end through the public API: pinned host inputs -> call() -> pinned host results
    host_in = []
    for a in arrays:
        t = pinned_tensor(gf.ElementType.F32, a.shape)
        t.buffer[:] = np.ascontiguousarray(a).reshape(-1)
        host_in.append(t)
    host_out = [pinned_tensor(d.element_type, d.shape) for d, _ in exe.result_signature]
    n = max(3, min(10, args.steps))
    for _ in range(2):
        gf.call(exe, host_in, out=host_out)
    _barrier(ws)
    e0 = time.perf_counter()
    for _ in range(n):
        gf.call(exe, host_in, out=host_out)
    e2e_s = _max_over_ranks((time.perf_counter() - e0) / n, ws)
    line["e2e"] = {"value": gbatch / e2e_s, "unit": "samples/s", "ms_per_step": e2e_s * 1e3,
                   "h2d_bytes_per_step": ws * sum(a.nbytes for a in arrays),
                   "d2h_bytes_per_step": ws * sum(t.buffer.nbytes for t in host_out),
                   "api": "paper_1801_08058_b200.call(exe, pinned host TensorValues, out=pinned host TensorValues) "
                          "on every rank (its batch shard; replicated parameters), wall clock, max over ranks; the "
                          "copies run inside the step's CUDA graph (gfb_exe_run_host): inputs in first-use order "
                          "under the launches that do not need them yet, each result right after its last writer"}
    return line


# sample batches of the CPU baseline per config: (all threads, one thread)
CPU_SAMPLE = {"E": (64, 4), "A": (128, 128), "C": (16, 2), "D": (1, 1)}


def cpu_baseline_step(wl):
    """Oracle port on the host cores, bounded samples (a few to ~20 s): all
    threads at a sample batch, and one thread at a smaller one (labelled)."""
    from oracle import interp

    threads = interp.max_threads()
    g = step_config(wl, 1)["global_batch"]
    b_all, b_one = CPU_SAMPLE[wl]
    t_all = _oracle_step_seconds(wl, b_all, threads, g)
    t_one = _oracle_step_seconds(wl, b_one, 1, g) if wl != "D" else None
    return {"value": b_all / t_all, "unit": "samples/s", "cores": threads, "kind": "port",
            "sample": f"one oracle step at batch {b_all} of {g} (loss / {g}) on {threads} threads: {t_all:.2f} s",
            "single_core": None if t_one is None else {"value": b_one / t_one, "cores": 1,
                                                       "sample": f"one oracle step at batch {b_one} on 1 thread: {t_one:.2f} s"},
            "cpu": _cpu_model(),
            "note": "the step has a batch-independent part (SGD over every parameter), so samples/s grows with the sample batch"}


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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="E", choices=["E", "B", "A", "C", "D", "G", "H"])
    ap.add_argument("--batch", type=int, default=None, help="global batch (training steps)")
    ap.add_argument("--launch-times", action="store_true", help="per-launch timing table to stderr")
    ap.add_argument("--dp", action="store_true", help="data-parallel plan even at one GPU (NCCL all-reduces)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the config-B block of the E line")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    maybe_relaunch(args)
    ws, rank, local = dist_setup()

    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(reference_arm(args, ws)), flush=True)
        return

    import torch

    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if args.workload == "G":
        line = bench_gemm(args, local)
    elif args.workload == "H":
        line = bench_conv(args, local)
    elif args.workload == "B":
        line = bench_chain(args, ws, rank, local)
        if rank == 0 and ws == 1 and not args.no_cpu_baseline:
            from oracle import interp

            value, threads, sample = cpu_reference_chain(ROWS, COLS, 2, 1, interp.max_threads(), budget_s=30.0)
            line["cpu_baseline"] = {"value": value, "unit": "GB/s", "cores": threads, "kind": "port", "sample": sample,
                                    "cpu": _cpu_model()}
    else:
        keys = ("metric", "value", "unit", "ms_per_step", "steps", "warmup", "scaling", "config", "roofline", "e2e",
                "gpu_launches", "clocks", "step_detail", "cpu_baseline")
        b = None
        if args.workload == "E" and not args.no_secondary:
            b = bench_chain(args, ws, rank, local)  # config B first, on a GPU not yet heated by E's GEMMs
            torch.cuda.empty_cache()
        line = bench_step(args, ws, rank, local)
        if rank == 0 and ws == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline_step(args.workload)
        if b is not None:
            # the other BASELINE.json configs, each measured the same way (own
            # roofline, e2e through call(), CPU baseline at N = 1)
            line["secondary"] = {k: b[k] for k in keys if k in b}
            line["configs"] = {}
            for wl, steps in (("A", 200), ("C", 50), ("D", 10)):
                torch.cuda.empty_cache()
                sub = argparse.Namespace(**dict(vars(args), workload=wl, steps=steps, batch=None, launch_times=False))
                r = bench_step(sub, ws, rank, local)
                if rank == 0 and ws == 1 and not args.no_cpu_baseline:
                    r["cpu_baseline"] = cpu_baseline_step(wl)
                line["configs"][wl] = {k: r[k] for k in keys if k in r}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
