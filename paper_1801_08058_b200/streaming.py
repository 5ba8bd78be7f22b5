"""Streamed execution of batch-independent graphs from host memory.

`call()` moves inputs host->device, runs, and moves results back, one after
the other.  For a forward graph whose results are all batch-sharded (no
batch reduction), each slab of rows is an independent problem.  Config B is
such a graph: a, b, t3 and the row sums are row-sharded, and c is
replicated.  `call_streamed` exploits that:

* it re-specialises the graph to a chunk of the batch (`rebatch`, using the
  sharding states of `dp.py`);
* it runs the chunks on three CUDA streams, so the PCIe H2D copy of chunk
  i+1, the kernels of chunk i and the D2H copy of chunk i-1 overlap.

Against `call()` the step takes max(H2D, D2H) instead of their sum.  torch
provides only the streams, events and pinned-buffer copies; the compute is
the same captured CUDA graph.
"""

from __future__ import annotations

import numpy as np

from .dp import DataParallel, _propagate
from .errors import UnsupportedOp
from .ir import ELEMENTWISE_BINARY, ELEMENTWISE_UNARY, Function, OpKind, topological_order


def rebatch(fn: Function, batch_params: list, chunks: int, axis: int = 0) -> Function:
    """Copy of `fn` whose batch-sharded axes are `chunks` times shorter."""
    dp = DataParallel(list(batch_params), axis)
    states, demand = _propagate(fn, dp)
    if demand:
        raise UnsupportedOp("streamed execution needs a graph with no reduction over the batch")
    for r, _ in fn.results:
        if not isinstance(states[r], tuple):
            raise UnsupportedOp("every result of a streamed graph must be batch-sharded")
    # Replicated values combined elementwise with sharded ones (e.g. a bias
    # Broadcast along the batch) carry the batch extent too: find the axis.
    order = topological_order(fn)
    batch_axis: dict = {n: s[1] for n, s in states.items() if isinstance(s, tuple)}
    for nid in reversed(order):
        node = fn.nodes[nid]
        a = batch_axis.get(nid)
        if a is None:
            continue
        if node.op in ELEMENTWISE_BINARY or node.op in ELEMENTWISE_UNARY or node.op is OpKind.CONVERT_LAYOUT:
            for r, _ in node.inputs:
                batch_axis.setdefault(r, a)
        elif node.op is OpKind.BROADCAST and a not in node.attrs["broadcast_axes"] and not isinstance(states[nid], tuple):
            kept = [i for i in range(len(node.output.shape)) if i not in node.attrs["broadcast_axes"]]
            batch_axis.setdefault(node.inputs[0][0], kept.index(a))
    g = Function(f"{fn.name}_chunk")
    new_id = {}

    def scaled(shape, nid):
        shape = list(shape)
        a = batch_axis.get(nid)
        if a is not None:
            if shape[a] % chunks:
                raise UnsupportedOp(f"batch extent {shape[a]} is not divisible by {chunks} chunks")
            shape[a] //= chunks
        return tuple(shape)

    for nid in order:
        node = fn.nodes[nid]
        if node.op is OpKind.PARAMETER:
            if nid in batch_axis and not isinstance(states[nid], tuple):
                raise UnsupportedOp(f"parameter {nid} has the batch extent but is not listed as batch-sharded")
            new_id[nid] = g.add_parameter(node.output.element_type, scaled(node.output.shape, nid))
            continue
        if node.op is OpKind.CONSTANT:
            data = node.attrs["data"]
            shape = node.attrs["shape"]
            if nid in batch_axis:
                if not data.is_splat:
                    raise UnsupportedOp(f"constant {nid} spans the batch with distinct values")
                shape = scaled(shape, nid)
                data = type(data).splat(data.element_type, int(np.prod(shape, dtype=np.int64)), data.splat_value())
            new_id[nid] = g.add_constant(node.attrs["element_type"], shape, data)
            continue
        attrs = dict(node.attrs)
        if node.op in (OpKind.BROADCAST, OpKind.RESHAPE):
            attrs["output_shape"] = scaled(attrs["output_shape"], nid)
        new_id[nid] = g.add_node(node.op, [(new_id[r], p) for r, p in node.inputs], attrs, allow_internal=True)
    g.parameters = [new_id[p] for p in fn.parameters]
    g.set_results([(new_id[r], p) for r, p in fn.results])
    g._chunk_states = {new_id[n]: s for n, s in states.items() if n in new_id}
    return g


class StreamedCall:
    """Chunk executable + double-buffered device slabs + three streams."""

    def __init__(self, fn: Function, batch_params: list, chunks: int, **compile_kw):
        import torch

        from .runtime import compile_function

        self.chunks = chunks
        self.sub = rebatch(fn, batch_params, chunks)
        self.exe = compile_function(self.sub, **compile_kw)
        st = self.sub._chunk_states
        self.in_sharded = [isinstance(st[p], tuple) and st[p][1] == 0 for p in self.sub.parameters]
        self.out_sharded = [isinstance(st[r], tuple) and st[r][1] == 0 for r, _ in self.sub.results]
        if not all(self.out_sharded) or any(isinstance(st[p], tuple) and st[p][1] != 0 for p in self.sub.parameters):
            raise UnsupportedOp("streaming needs batch-major (axis 0) inputs and results")
        self.s_in, self.s_run, self.s_out = (torch.cuda.Stream() for _ in range(3))
        self.dev_in = [[None] * len(self.sub.parameters) for _ in range(2)]
        self.dev_out = [self.exe.allocate_outputs() for _ in range(2)]

    def __call__(self, inputs: list, out: list) -> list:
        """`inputs`/`out`: host TensorValues in the full-batch signature
        (pinned for asynchronous copies)."""
        import torch

        k = self.chunks
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_run = [torch.cuda.Event() for _ in range(2)]
        ev_out = [torch.cuda.Event() for _ in range(2)]
        host_in = [torch.from_numpy(t.buffer) for t in inputs]
        host_out = [torch.from_numpy(t.buffer) for t in out]
        # replicated inputs: one copy, shared by both slab sets
        with torch.cuda.stream(self.s_in):
            for j, (h, sh) in enumerate(zip(host_in, self.in_sharded)):
                if not sh:
                    d = h.to("cuda", non_blocking=True)
                    self.dev_in[0][j] = self.dev_in[1][j] = d
        for i in range(k):
            b = i % 2
            with torch.cuda.stream(self.s_in):
                if i >= 2:
                    self.s_in.wait_event(ev_run[b])  # slab b's previous chunk has been consumed
                for j, (h, sh) in enumerate(zip(host_in, self.in_sharded)):
                    if sh:
                        n = h.numel() // k
                        src = h[i * n:(i + 1) * n]
                        if self.dev_in[b][j] is None:
                            self.dev_in[b][j] = torch.empty(n, dtype=src.dtype, device="cuda")
                        self.dev_in[b][j].copy_(src, non_blocking=True)
                ev_in[b].record(self.s_in)
            self.s_run.wait_event(ev_in[b])
            if i >= 2:
                self.s_run.wait_event(ev_out[b])  # slab b's previous results are on the host
            self.exe.run_device(self.dev_in[b], self.dev_out[b], stream=self.s_run.cuda_stream)
            ev_run[b].record(self.s_run)
            with torch.cuda.stream(self.s_out):
                self.s_out.wait_event(ev_run[b])
                for h, d in zip(host_out, self.dev_out[b]):
                    n = h.numel() // k
                    h[i * n:(i + 1) * n].copy_(d, non_blocking=True)
                ev_out[b].record(self.s_out)
        self.s_out.synchronize()
        return out


def call_streamed(exe_or_fn, inputs: list, out: list, batch_params=None, chunks: int = 8):
    """Host-to-host execution with copy/compute overlap (see module doc).

    `exe_or_fn` is a Function or an Executable (its graph is reused);
    `batch_params` defaults to every parameter with a leading axis equal to
    the first parameter's."""
    fn = getattr(exe_or_fn, "function", exe_or_fn)
    cache = getattr(exe_or_fn, "_streamed", None)
    if cache is None or cache.chunks != chunks:
        if batch_params is None:
            lead = fn.nodes[fn.parameters[0]].output.shape[0]
            batch_params = [p for p in fn.parameters
                            if fn.nodes[p].output.shape and fn.nodes[p].output.shape[0] == lead]
        cache = StreamedCall(fn, batch_params, chunks)
        try:
            exe_or_fn._streamed = cache
        except AttributeError:
            pass
    return cache(inputs, out)
