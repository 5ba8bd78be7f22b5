"""`compile_function` / `call` on the B200 (drop-in for the reference backend).

Mirrors `/root/reference/pkg/src/graphforge/interpreter.py:92-245`:

* `compile_function(fn, *, optimize=True, conv_layout="identity",
  parameter_layouts=None)` validates (`ValidationFailure`), runs
  simplify / cse / fold (folding through the device kernels), assigns
  layouts, and records the reference's per-node instruction listing and
  memory plan for compatibility.  It then lowers the graph to fused
  launches (`compiler.py`) and creates the device executable through the
  C ABI (`include/gfb200.h`, `libgfb200.so`).
* `call(exe, inputs, *, private_buffers=False)` checks the signature
  exactly like the reference (`SignatureMismatch` on descriptor or layout
  order), uploads host inputs, runs the captured CUDA graph and returns
  fresh result tensors that never alias inputs.  Device-resident
  `TensorValue`s (CUDA `torch.Tensor` buffers) are consumed in place, and
  `call(..., device=True)` leaves results on the GPU.

There is no CPU execution path: if the library or a B200 is missing every
entry point raises `BackendUnavailable`.
"""

from __future__ import annotations

import contextlib
import ctypes as C
import os
import threading
import weakref
from collections.abc import Mapping
from dataclasses import dataclass

import numpy as np

from . import abi, jit
from .compiler import Lowered, lower
from .errors import BackendUnavailable, DeviceError, SignatureMismatch, ValidationFailure
from .ir import (ConstantData, Function, OpKind, TensorDescriptor, element_count, reachable_from_results, topological_order,
                 validate_function)
from .layout import NHWC_ORDER, Layout, assign_layouts, layout_policy, tensor_layouts
from .memory import MemoryPlan, plan_memory
from .rewrite import run_pipeline
from .tensor import TensorValue, storage_to_logical, tensor_from_flat, torch_dtype

_LIB = None
_LOCK = threading.Lock()
_DEVICE_READY: set = set()


def library_path() -> str:
    return os.path.join(os.path.dirname(os.path.abspath(__file__)), "libgfb200.so")


def lib():
    """Load libgfb200.so (building it in-tree first if it is stale)."""
    global _LIB
    with _LOCK:
        if _LIB is not None:
            return _LIB
        from . import _build

        if not _build.up_to_date():
            try:
                _build.build()
            except Exception as exc:  # no silent fallback: the backend is unusable
                raise BackendUnavailable(f"cannot build libgfb200.so: {exc}") from exc
        try:
            L = C.CDLL(library_path())
        except OSError as exc:
            raise BackendUnavailable(f"cannot load {library_path()}: {exc}") from exc
        vp, i32, u32 = C.c_void_p, C.c_int, C.c_uint32
        L.gfb_init.argtypes = [i32]
        L.gfb_last_error.restype = C.c_char_p
        L.gfb_device_info.argtypes = [C.POINTER(i32)] * 3
        L.gfb_exe_create.argtypes = [C.POINTER(abi.Plan), C.POINTER(vp)]
        L.gfb_exe_run.argtypes = [vp, C.POINTER(vp), C.POINTER(vp), vp]
        L.gfb_exe_run_one.argtypes = [vp, u32, C.POINTER(vp), C.POINTER(vp), vp]
        L.gfb_exe_destroy.argtypes = [vp]
        L.gfb_exe_num_launches.argtypes = [vp]
        L.gfb_comm_unique_id.argtypes = [vp]
        L.gfb_comm_create.argtypes = [i32, i32, vp, C.POINTER(vp)]
        L.gfb_comm_destroy.argtypes = [vp]
        L.gfb_kernel_load.argtypes = [vp, C.c_char_p, C.POINTER(vp)]
        L.gfb_exe_set_kernel.argtypes = [vp, u32, vp, u32]
        L.gfb_exe_set_schedule.argtypes = [vp, u32, C.POINTER(u32), C.POINTER(u32), C.POINTER(u32)]
        u64 = C.c_uint64
        L.gfb_exe_set_io.argtypes = [vp, C.POINTER(u64), C.POINTER(u64), C.POINTER(u32), C.POINTER(u32), C.POINTER(u32)]
        L.gfb_exe_run_host.argtypes = [vp, C.POINTER(vp), C.POINTER(vp), vp]
        L.gfb_exe_set_io_pieces.argtypes = [vp, C.c_uint32, C.POINTER(u32), C.POINTER(u64), C.POINTER(u64), C.POINTER(u32),
                                            C.POINTER(u32)]
        _LIB = L
        return L


def check(rc: int, what: str):
    if rc != abi.GFB_OK:
        msg = lib().gfb_last_error().decode(errors="replace")
        raise DeviceError(f"{what}: {msg} (status {rc})")


def ensure_device():
    import torch

    if not torch.cuda.is_available():
        raise BackendUnavailable("no CUDA device visible; the B200 backend has no CPU fallback")
    dev = torch.cuda.current_device()
    if dev not in _DEVICE_READY:
        check(lib().gfb_init(dev), "gfb_init")
        _DEVICE_READY.add(dev)
    return dev


# ---------------------------------------------------------------------------
# Executable


@dataclass(frozen=True)
class Instruction:
    node_id: int
    kernel: str
    input_slots: tuple
    output_slot: str


class _ConstPool(Mapping):
    """Constant pool as TensorValues, materialised lazily (splats stay scalars)."""

    def __init__(self, g: Function, refs: list):
        self._g = g
        self._refs = list(refs)
        self._cache: dict = {}

    def __getitem__(self, ref):
        if ref not in self._refs:
            raise KeyError(ref)
        if ref not in self._cache:
            a = self._g.nodes[ref[0]].attrs
            self._cache[ref] = tensor_from_flat(a["element_type"], a["shape"], a["data"].to_numpy())
        return self._cache[ref]

    def __iter__(self):
        return iter(self._refs)

    def __len__(self):
        return len(self._refs)


class DeviceProgram:
    """Owner of one gfb_exe handle."""

    def __init__(self, lowered: Lowered, cuda_graph: bool = True, comm=None):
        self.lowered = lowered
        recs, blob = lowered.pack()
        self._recs, self._blob = recs, C.create_string_buffer(blob, max(1, len(blob)))
        self._consts = C.create_string_buffer(lowered.const_blob, max(1, len(lowered.const_blob)))
        plan = abi.Plan()
        plan.arena_bytes = lowered.arena_bytes
        plan.const_bytes = len(lowered.const_blob)
        plan.const_data = C.cast(self._consts, C.c_void_p)
        plan.n_inputs, plan.n_outputs = lowered.n_inputs, lowered.n_outputs
        plan.n_launches = len(lowered.launches)
        plan.flags = abi.PLAN_CUDA_GRAPH if cuda_graph else 0
        plan.launches = C.cast(recs, C.POINTER(abi.Launch))
        plan.args_bytes = len(blob)
        plan.args = C.cast(self._blob, C.c_void_p)
        plan.comm = comm
        handle = C.c_void_p()
        ensure_device()
        check(lib().gfb_exe_create(C.byref(plan), C.byref(handle)), "gfb_exe_create")
        self.handle = handle
        self._io = None  # host-buffer runs: None = not set up yet
        # launches running a runtime-specialised kernel (jit.py) instead of the generic VM,
        # and launches folded into a preceding merged kernel (not launched at all)
        self.jit_launches, self.skipped = (jit.specialise(lib(), handle, lowered.launches, blob, recs)
                                           if jit.enabled() else ([], []))
        # independent launches as concurrent graph nodes (schedule.py)
        self.n_streams = int(os.environ.get("GFB_STREAMS", "4"))
        if cuda_graph and self.n_streams > 1 and len(lowered.launches) > 1:
            from . import schedule

            st, off, deps = schedule.build(lowered, self.skipped, self.n_streams)
            arr = lambda v: (C.c_uint32 * max(1, len(v)))(*v)
            check(lib().gfb_exe_set_schedule(handle, self.n_streams, arr(st), arr(off), arr(deps)), "gfb_exe_set_schedule")

    def run(self, in_ptrs: list, out_ptrs: list, stream=None):
        ins = (C.c_void_p * max(1, len(in_ptrs)))(*in_ptrs)
        outs = (C.c_void_p * max(1, len(out_ptrs)))(*out_ptrs)
        check(lib().gfb_exe_run(self.handle, ins, outs, stream), "gfb_exe_run")

    def host_io(self, in_bytes: list, out_bytes: list) -> bool:
        """Set up host-buffer runs once (device staging buffers, copy
        schedule); False when the plan does not support them."""
        if self._io is None:
            from . import schedule

            acc = schedule.io_access(self.lowered, self.skipped)
            if acc is None:
                self._io = False
                return False
            off, reads, writer = acc
            u32 = lambda v: (C.c_uint32 * max(1, len(v)))(*v)
            u64 = lambda v: (C.c_uint64 * max(1, len(v)))(*v)
            check(lib().gfb_exe_set_io(self.handle, u64(in_bytes), u64(out_bytes), u32(off), u32(reads), u32(writer)),
                  "gfb_exe_set_io")
            pieces = schedule.io_pieces(self.lowered, in_bytes, self.skipped) if os.environ.get("GFB_IO_PIECES", "1") == "1" else None
            if pieces is not None:
                p_in, p_off, p_len, poff, preads = pieces
                check(lib().gfb_exe_set_io_pieces(self.handle, len(p_in), u32(p_in), u64(p_off), u64(p_len), u32(poff),
                                                  u32(preads)), "gfb_exe_set_io_pieces")
            self._io = True
        return self._io

    def run_host(self, in_ptrs: list, out_ptrs: list, stream=None):
        ins = (C.c_void_p * max(1, len(in_ptrs)))(*in_ptrs)
        outs = (C.c_void_p * max(1, len(out_ptrs)))(*out_ptrs)
        check(lib().gfb_exe_run_host(self.handle, ins, outs, stream), "gfb_exe_run_host")

    def run_one(self, index: int, in_ptrs: list, out_ptrs: list, stream=None):
        ins = (C.c_void_p * max(1, len(in_ptrs)))(*in_ptrs)
        outs = (C.c_void_p * max(1, len(out_ptrs)))(*out_ptrs)
        check(lib().gfb_exe_run_one(self.handle, index, ins, outs, stream), "gfb_exe_run_one")

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and _LIB is not None:
            _LIB.gfb_exe_destroy(h)
            self.handle = None


class Executable:
    """Compiled graph: the reference's attributes plus the device program."""

    def __init__(self, function, instructions, plan, pool, layouts, param_index, result_index,
                 parameter_signature, result_signature, lowered, cuda_graph=True, comm=None):
        self.function = function
        self.instructions = instructions
        self.plan = plan
        self.pool = pool
        self.layouts = layouts
        self.param_index = param_index
        self.result_index = result_index
        self.parameter_signature = parameter_signature
        self.result_signature = result_signature
        self.lowered = lowered
        self._cuda_graph = cuda_graph
        self._comm = comm
        self._program = DeviceProgram(lowered, cuda_graph, comm)
        self._private = None

    def listing(self) -> str:
        """Per-IR-node listing in the reference format (interpreter.py:82-89)."""
        lines = [f"arena {self.plan.arena_size} bytes"]
        for i, ins in enumerate(self.instructions):
            lines.append(f"{i}\t{ins.node_id}\t{ins.kernel}\t{','.join(ins.input_slots) or '-'}\t{ins.output_slot}")
        return "\n".join(lines) + "\n"

    def launch_listing(self) -> str:
        """What actually runs: one line per fused B200 launch."""
        lines = [f"device arena {self.lowered.arena_bytes} bytes, {len(self.lowered.launches)} launches"]
        for i, L in enumerate(self.lowered.launches):
            lines.append(f"{i}\t{L.label}\tkind={L.kind}\tgrid={L.grid}\tbytes={L.algo_bytes}\tflops={L.flops}")
        return "\n".join(lines) + "\n"

    @property
    def num_launches(self) -> int:
        """Kernels one run launches (merged single-block launches count once)."""
        return len(self.lowered.launches) - len(self._program.skipped)

    def program(self, private: bool = False) -> DeviceProgram:
        if not private:
            return self._program
        if self._private is None:
            g = self.function
            low = lower(g, self.layouts, private=True, channels_last=self.lowered.channels_last)
            self._private = DeviceProgram(low, self._cuda_graph, self._comm)
        return self._private

    # -- device-level entry (inputs already resident; bench / DP path)
    def run_device(self, inputs: list, outputs: list, stream=None, private: bool = False):
        self.program(private).run([_ptr(t) for t in inputs], [_ptr(t) for t in outputs], stream)

    def allocate_outputs(self):
        import torch

        return [torch.empty(int(np.prod(d.shape, dtype=np.int64)), dtype=torch_dtype(d.element_type), device="cuda")
                for d, _ in self.result_signature]


def _ptr(t) -> int:
    return t.data_ptr() if t.numel() else 0


def _build_listing(g: Function, plan: MemoryPlan):
    """Reference instruction list + pool refs (interpreter.py:120-159)."""
    reachable = reachable_from_results(g)
    result_index: dict = {}
    for j, ref in enumerate(g.results):
        result_index.setdefault(ref, j)
    param_index = {(pid, 0): i for i, pid in enumerate(g.parameters)}
    pool_refs = []
    instructions = []

    def slot(ref):
        if ref in param_index:
            return f"param{param_index[ref]}"
        if ref in pool_set:
            return f"const{ref[0]}"
        if ref in result_index:
            return f"result{result_index[ref]}"
        return f"arena+{plan.placements[ref]}"

    pool_set = set()
    for nid in topological_order(g):
        if nid not in reachable:
            continue
        node = g.nodes[nid]
        if node.op is OpKind.PARAMETER:
            continue
        if node.op is OpKind.CONSTANT:
            pool_refs.append((nid, 0))
            pool_set.add((nid, 0))
            continue
        instructions.append(Instruction(nid, node.op.wire_name, tuple(slot(r) for r in node.inputs), slot((nid, 0))))
    return instructions, pool_refs, param_index, result_index


@dataclass
class HostCompiled:
    """Everything compile_function decides on the host, before the device."""

    graph: Function
    layouts: dict
    plan: MemoryPlan
    instructions: list
    pool_refs: list
    param_index: dict
    result_index: dict
    parameter_signature: list
    result_signature: list
    lowered: Lowered
    allreduce: frozenset = frozenset()

    def listing(self) -> str:
        return Executable.listing(self)


def prepare_function(fn: Function, *, optimize: bool = True, conv_layout: str = "identity",
                     parameter_layouts=None, evaluate=None, private: bool = False,
                     data_parallel=None) -> HostCompiled:
    """Validate, optimise, assign layouts, plan and lower (reference
    interpreter.py:92-170 plus the B200 lowering).  `evaluate` overrides the
    constant-folding evaluator (the device by default)."""
    diags = validate_function(fn)
    if diags:
        raise ValidationFailure(diags)
    policy = layout_policy(conv_layout)
    g = fn
    if optimize:
        g = run_pipeline(g, ["simplify", "cse", "fold"], evaluate=evaluate)
    g = assign_layouts(g, policy, parameter_layouts)
    layouts = tensor_layouts(g, policy, parameter_layouts)
    plan = plan_memory(g)
    instructions, pool_refs, param_index, result_index = _build_listing(g, plan)
    param_sig = [(g.nodes[pid].output, layouts[(pid, 0)]) for pid in g.parameters]
    result_sig = [(g.nodes[r].outputs[p], layouts[(r, p)]) for r, p in g.results]
    roots = frozenset()
    if data_parallel is not None:
        from .dp import analyse

        position = {pid: i for i, pid in enumerate(fn.parameters)}
        data_parallel.batch_params = [g.parameters[position[p]] if p in position else p for p in data_parallel.batch_params]
        roots = frozenset(analyse(g, data_parallel))
    # Intermediate 4-D activations are stored channel-last whatever the
    # caller's layout policy (parameters and results keep theirs): the conv
    # kernels then gather 16-byte runs of channels.  GFB_CHANNELS_LAST=0
    # stores intermediates in the policy's order instead.
    channels_last = os.environ.get("GFB_CHANNELS_LAST", "1") == "1" or policy.conv_order == NHWC_ORDER
    rmax = frozenset(getattr(data_parallel, "allreduce_max", ()) or ())
    lowered = lower(g, layouts, private=private, allreduce=roots, channels_last=channels_last, allreduce_max=rmax)
    cap = int(os.environ.get("GFB_PRIVATE_ARENA_MAX", 64 << 20))
    if not private and int(os.environ.get("GFB_STREAMS", "4")) > 1 and lowered.arena_bytes <= cap:
        # small arenas: one range per tensor, so reuse adds no false ordering
        # between launches that could run concurrently (schedule.py) -- kept
        # only if the no-reuse plan itself stays within the cap
        private_plan = lower(g, layouts, private=True, allreduce=roots, channels_last=channels_last, allreduce_max=rmax)
        if private_plan.arena_bytes <= cap:
            lowered = private_plan
    return HostCompiled(g, layouts, plan, instructions, pool_refs, param_index, result_index,
                        param_sig, result_sig, lowered, roots)


@contextlib.contextmanager
def _nvtx(name: str):
    """NVTX range (visible to nsys / ncu --nvtx); a no-op without torch's NVTX bindings."""
    try:
        import torch

        torch.cuda.nvtx.range_push(name)
        pushed = True
    except Exception:
        pushed = False
    try:
        yield
    finally:
        if pushed:
            torch.cuda.nvtx.range_pop()


def compile_function(fn: Function, *, optimize: bool = True, conv_layout: str = "identity",
                     parameter_layouts=None, cuda_graph: bool = True, data_parallel=None,
                     comm=None) -> Executable:
    """Reference `compile_function` plus B200 options: `cuda_graph` (capture
    the launch list once), `data_parallel` (a `dp.DataParallel`: batch-shard
    the listed parameters and all-reduce the partial gradients) with the
    NCCL communicator `comm` from `init_distributed()`."""
    from .refcompat import as_function, as_layout, caller_errors, foreign_errors

    errors_mod = foreign_errors(fn)
    with caller_errors(errors_mod), _nvtx("compile_function"):
        fn = as_function(fn)  # a reference-built graphforge.Function is mirrored node for node
        if parameter_layouts is not None:
            parameter_layouts = [as_layout(lay) for lay in parameter_layouts]
        h = prepare_function(fn, optimize=optimize, conv_layout=conv_layout, parameter_layouts=parameter_layouts,
                             data_parallel=data_parallel)
    if h.allreduce and comm is None:
        comm = init_distributed()
    handle = comm.handle if comm is not None else None
    exe = Executable(h.graph, h.instructions, h.plan, _ConstPool(h.graph, h.pool_refs), h.layouts,
                     h.param_index, h.result_index, h.parameter_signature, h.result_signature,
                     h.lowered, cuda_graph, handle)
    exe.comm = comm
    exe.allreduce = h.allreduce
    exe.caller_errors = errors_mod
    return exe


class Comm:
    """NCCL communicator owned by libgfb200.so (one per process / GPU)."""

    def __init__(self, handle, rank: int, world: int):
        self.handle, self.rank, self.world = handle, rank, world

    def __del__(self):
        if getattr(self, "handle", None) and _LIB is not None:
            _LIB.gfb_comm_destroy(self.handle)
            self.handle = None


_COMM = None


def init_distributed(rank: int | None = None, world: int | None = None) -> Comm:
    """NCCL communicator over the current torch.distributed group (or a
    single-rank one).  Rank 0 creates the ncclUniqueId; it travels through
    torch.distributed (any backend) — torch is only the rendezvous."""
    global _COMM
    import torch.distributed as dist

    ensure_device()
    if rank is None:
        rank = dist.get_rank() if dist.is_available() and dist.is_initialized() else 0
        world = dist.get_world_size() if dist.is_available() and dist.is_initialized() else 1
    if _COMM is not None and (_COMM.rank, _COMM.world) == (rank, world):
        return _COMM
    # Collective pinning for the gradient buckets: single-node
    # NVSwitch all-reduces of 1-64 MiB buckets -- NVLS (in-switch reduction)
    # or Ring, Simple / LL128 protocols; Tree and LL do not pay at these sizes.
    # Callers' own settings win; GFB_NCCL_PIN=0 leaves NCCL to choose.
    if os.environ.get("GFB_NCCL_PIN", "1") == "1":
        os.environ.setdefault("NCCL_ALGO", "NVLS,Ring")
        os.environ.setdefault("NCCL_PROTO", "Simple,LL128")
    uid = C.create_string_buffer(128)
    if rank == 0:
        check(lib().gfb_comm_unique_id(uid), "gfb_comm_unique_id")
    if world > 1:
        box = [bytes(uid.raw)]
        dist.broadcast_object_list(box, src=0)
        uid = C.create_string_buffer(box[0], 128)
    handle = C.c_void_p()
    check(lib().gfb_comm_create(world, rank, uid, C.byref(handle)), "gfb_comm_create")
    _COMM = Comm(handle, rank, world)
    return _COMM


def _check_signature(exe: Executable, inputs: list):
    expected = exe.parameter_signature
    if len(inputs) != len(expected):
        raise SignatureMismatch(f"expected {len(expected)} inputs, got {len(inputs)}")
    for i, (t, (desc, layout)) in enumerate(zip(inputs, expected)):
        if t.descriptor != desc:
            raise SignatureMismatch(f"input {i}: expected {desc}, got {t.descriptor}")
        if t.layout.order != layout.order:
            raise SignatureMismatch(
                f"input {i}: expected layout order {list(layout.order)}, got {list(t.layout.order)}"
            )


def to_device(t: TensorValue):
    """Storage-order CUDA tensor for `t` (no copy when already resident)."""
    import torch

    if t.is_device:
        return t.buffer
    host = torch.from_numpy(np.ascontiguousarray(t.buffer))
    return host.to("cuda", non_blocking=host.is_pinned())


def _forget_pinned(addr):
    _PINNED.pop(addr, None)


def pinned_tensor(et, shape) -> TensorValue:
    """Zero host TensorValue in page-locked memory (fast H2D / D2H DMA)."""
    import torch

    from .ir import TensorDescriptor, element_count
    from .layout import identity_layout

    buf = torch.zeros(element_count(shape), dtype=torch_dtype(et), pin_memory=True).numpy()
    if buf.size:
        _PINNED[buf.ctypes.data] = buf.nbytes  # page-locked for as long as the array lives
        weakref.finalize(buf, _forget_pinned, buf.ctypes.data)
    return TensorValue(TensorDescriptor(et, tuple(shape)), identity_layout(len(shape)), buf)


# host buffers allocated by pinned_tensor (address -> bytes), dropped when freed
_PINNED: dict = {}


def _pinned_host(t: TensorValue, desc) -> bool:
    import torch

    b = t.buffer
    if not (not t.is_device and isinstance(b, np.ndarray) and b.flags.c_contiguous and b.size > 0
            and t.descriptor == desc and b.nbytes == element_count(desc.shape) * desc.element_type.byte_size):
        return False
    if _PINNED.get(b.ctypes.data, -1) >= b.nbytes:  # one of ours (no driver query per call)
        return True
    return torch.from_numpy(b).is_pinned()


def _host_run(exe: Executable, inputs: list, out: list, stream) -> bool:
    """One step on page-locked host buffers with the copies inside the
    step's CUDA graph (gfb_exe_run_host): inputs cross PCIe in first-use
    order under the launches that do not need them yet, and each result
    leaves as soon as its last writer finishes.  False (nothing done) when a
    buffer is not page-locked or the plan has no host-run schedule."""
    if os.environ.get("GFB_HOST_GRAPH", "1") == "0" or len(out) != len(exe.result_signature):
        return False
    if not all(_pinned_host(t, d) for t, (d, _) in zip(inputs, exe.parameter_signature)):
        return False
    if not all(_pinned_host(t, d) and t.layout.order == lay.order for t, (d, lay) in zip(out, exe.result_signature)):
        return False
    prog = exe.program(False)
    if not prog.host_io([t.buffer.nbytes for t in inputs], [t.buffer.nbytes for t in out]):
        return False
    prog.run_host([t.buffer.ctypes.data for t in inputs], [t.buffer.ctypes.data for t in out], stream.cuda_stream)
    stream.synchronize()
    return True


def call(exe: Executable, inputs: list, *, private_buffers: bool = False, device: bool = False, out=None) -> list:
    """Execute on the B200; one fresh result tensor per result.

    `out`, if given, is a list of host TensorValues (e.g. `pinned_tensor`)
    the results are copied into instead of newly allocated ones.
    """
    import torch

    from .refcompat import as_tensor, caller_errors, foreign_errors

    with caller_errors(getattr(exe, "caller_errors", None) or foreign_errors(inputs)):
        inputs = [as_tensor(t) for t in inputs]  # reference-built TensorValues are accepted as they are
        _check_signature(exe, inputs)
    ensure_device()
    cur = torch.cuda.current_stream()
    if out is not None and not private_buffers and not device and _host_run(exe, inputs, out, cur):
        return list(out)
    dev_in = [to_device(t) for t in inputs]
    outs = exe.allocate_outputs()
    exe.run_device(dev_in, outs, stream=cur.cuda_stream, private=private_buffers)
    if device:
        return [TensorValue(desc, layout, buf) for (desc, layout), buf in zip(exe.result_signature, outs)]
    results = []
    if out is not None:
        if len(out) != len(outs):
            raise SignatureMismatch(f"expected {len(outs)} output tensors, got {len(out)}")
        for (desc, layout), buf, host in zip(exe.result_signature, outs, out):
            if host.descriptor != desc:
                raise SignatureMismatch(f"output buffer {host.descriptor} != result {desc}")
            dst = torch.from_numpy(host.buffer)
            dst.copy_(buf, non_blocking=dst.is_pinned())
            results.append(host)
        cur.synchronize()
        return results
    cur.synchronize()
    for (desc, layout), buf in zip(exe.result_signature, outs):
        results.append(TensorValue(desc, layout, buf.cpu().numpy()))
    return results


# ---------------------------------------------------------------------------
# Constant folding through the device kernels (rewrite.constant_fold)


_FOLD_CACHE: dict = {}


def device_fold_evaluator(node, inputs: list, input_descs: list) -> ConstantData:
    from .ir import attrs_key

    key = (node.op, attrs_key(node), tuple(input_descs), node.output)
    exe = _FOLD_CACHE.get(key)
    if exe is None:
        f = Function("fold")
        params = [f.add_parameter(d.element_type, d.shape) for d in input_descs]
        f.set_results([f.add_node(node.op, params, node.attrs, allow_internal=True)])
        exe = compile_function(f, optimize=False)
        if len(_FOLD_CACHE) < 256:
            _FOLD_CACHE[key] = exe
    tensors = [tensor_from_flat(d.element_type, d.shape, data.to_numpy()) for data, d in zip(inputs, input_descs)]
    out = call(exe, tensors)[0]
    return ConstantData.from_array(node.output.element_type, out.to_numpy().reshape(-1))
