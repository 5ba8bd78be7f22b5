"""Batch-sharded data parallelism: where a training graph needs an all-reduce.

SURVEY.md §8(e): examples are independent, so `x` and `t` are split on
axis 0 and the weights are replicated; every tensor that sums over the batch
axis becomes a per-rank *partial*.  These include the dW Dots fed by
autodiff's `Reshape(x, (1, 0))` (`autodiff.py:163-177`), batch `Sum`s (bias
gradients, the loss) and `ConvBackpropFilter`.  A partial may flow through
ops that are linear in it (Add/Sub of partials, scaling by a replicated
value, index ops, Sum, Dot with a replicated operand).  Before the first
consumer that needs the full value — the SGD `Subtract(W, ·)`, any
nonlinearity, a result — the *root* that created the partial is summed
across ranks.  The paper lists AllReduce among the collectives transformers
should emit (`PAPER.md:49`).

`analyse` returns the roots to all-reduce.  The lowering emits an in-place
NCCL sum all-reduce right after each root's producing launch, inside the
same CUDA graph.  The per-rank graph is the reference graph specialised to
the local batch.  The loss divisor stays the global batch (the
`loss_batch` argument of `workloads.mlp_step`), so the summed partials are
exactly the single-GPU values.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from .errors import UnsupportedOp
from .ir import ELEMENTWISE_BINARY, ELEMENTWISE_UNARY, Function, OpKind, reachable_from_results, topological_order

REPL, PART = "replicated", "partial"
# per-rank max over the batch shard (a max-reduction along the sharded axis):
# nothing is linear in it, so its first consumer needs the max across ranks
PMAX = "partial_max"


def sharded(axis: int):
    return ("sharded", axis)


@dataclass
class DataParallel:
    """Batch-sharded execution spec for `compile_function(data_parallel=...)`."""

    batch_params: list  # parameter node ids split along `axis`
    axis: int = 0
    world_size: int = 1
    allreduce: set = field(default_factory=set)  # filled by analyse()
    allreduce_max: set = field(default_factory=set)  # the roots among them reduced with max, not sum


def _reshape_axis(node, in_shape, axis: int):
    """Output axis that holds a sharded input axis through a Reshape, or None.

    After the axis permutation the sharded axis is permuted position i, with
    flat weight w = prod(P[i+1:]) and extent P[i].  It survives the row-major
    re-read when some output axis j has the same top boundary
    (u_j * out[j] == w * P[i], u_j = prod(out[j+1:])) and reaches down to it
    (u_j divides w), or is carved from its top (w divides u_j, a split such as
    the maxpool backward [4, N*C*H*W] -> [.., N, C, H, W]).  The batch factor
    is then the most significant part of axis j, so each rank still owns a
    contiguous block of it.
    """
    order = node.attrs["input_order"]
    out_shape = node.output.shape
    perm = [in_shape[a] for a in order]
    i = list(order).index(axis)
    w = 1
    for d in perm[i + 1:]:
        w *= d
    top = w * perm[i]
    u = 1
    for j in range(len(out_shape) - 1, -1, -1):
        if u * out_shape[j] == top and (w % u == 0 or u % w == 0):
            return j  # top-aligned: merges the shard with lower digits, or splits it batch-first
        u *= out_shape[j]
    return None


def _propagate(g: Function, dp: DataParallel):
    """State of every tensor; returns (states, demand) where demand lists
    (consumer, partial input) pairs that need the full value."""
    order = [n for n in topological_order(g) if n in reachable_from_results(g)]
    st: dict = {}
    demand = []
    bp = set(dp.batch_params)
    for n in order:
        node = g.nodes[n]
        op = node.op
        ins = [st[r] for r, _ in node.inputs]
        if op is OpKind.PARAMETER:
            st[n] = sharded(dp.axis) if n in bp else REPL
            continue
        if op is OpKind.CONSTANT:
            st[n] = REPL
            continue
        if n in dp.allreduce:
            st[n] = REPL  # summed across ranks right after it is produced
            continue
        pmax = [r for (r, _), s in zip(node.inputs, ins) if s == PMAX]
        if pmax:
            for r in pmax:
                demand.append((n, r))
            ins = [REPL if s == PMAX else s for s in ins]
        parts = [r for (r, _), s in zip(node.inputs, ins) if s == PART]
        shards = [s for s in ins if isinstance(s, tuple)]

        def need_all():
            for r in parts:
                demand.append((n, r))

        if op in ELEMENTWISE_UNARY:
            if ins[0] == PART:
                if op is OpKind.NEGATE:
                    st[n] = PART
                else:
                    need_all()
                    st[n] = REPL
            else:
                st[n] = ins[0]
        elif op in ELEMENTWISE_BINARY:
            if parts:
                a, b = ins
                linear = (op in (OpKind.ADD, OpKind.SUBTRACT) and a == PART and b == PART) or \
                         (op is OpKind.MULTIPLY and {a, b} == {PART, REPL}) or \
                         (op is OpKind.DIVIDE and a == PART and b == REPL)
                if linear:
                    st[n] = PART
                else:
                    need_all()
                    st[n] = shards[0] if shards else REPL
            else:
                axes = {s for s in shards}
                if len(axes) > 1:
                    raise UnsupportedOp(f"data parallel: node {n} mixes batch axes {axes}")
                st[n] = shards[0] if shards else REPL
        elif op is OpKind.CONVERT_LAYOUT:
            st[n] = ins[0]
        elif op is OpKind.BROADCAST:
            s = ins[0]
            if isinstance(s, tuple):
                kept = [i for i in range(len(node.output.shape)) if i not in node.attrs["broadcast_axes"]]
                st[n] = sharded(kept[s[1]])
            else:
                st[n] = s
        elif op is OpKind.RESHAPE:
            s = ins[0]
            if isinstance(s, tuple):
                in_shape = g.nodes[node.inputs[0][0]].output.shape
                j = _reshape_axis(node, in_shape, s[1])
                if j is None:
                    raise UnsupportedOp(f"data parallel: Reshape node {n} scatters the batch axis")
                st[n] = sharded(j)
            else:
                st[n] = s
        elif op is OpKind.SUM:
            s = ins[0]
            axes = node.attrs["reduction_axes"]
            if isinstance(s, tuple):
                if s[1] in axes:
                    st[n] = PMAX if node.attrs["reduction_kind"] == "max" else PART
                else:
                    st[n] = sharded(s[1] - sum(1 for a in axes if a < s[1]))
            elif s == PART and node.attrs["reduction_kind"] == "max":
                need_all()
                st[n] = REPL
            else:
                st[n] = s
        elif op is OpKind.DOT:
            a, b = ins
            if a == sharded(1) and b == sharded(0):
                st[n] = PART
            elif a == sharded(0) and b == REPL:
                st[n] = sharded(0)
            elif a == REPL and b == sharded(1):
                st[n] = sharded(1)
            elif (a == PART and b == REPL) or (a == REPL and b == PART):
                st[n] = PART
            elif a == REPL and b == REPL:
                st[n] = REPL
            else:
                need_all()
                st[n] = REPL
        elif op in (OpKind.CONV2D, OpKind.CONV_BACKPROP_DATA):
            a, b = ins
            if a == sharded(0) and b == REPL:
                st[n] = sharded(0)
            elif a == REPL and b == REPL:
                st[n] = REPL
            else:
                need_all()
                st[n] = sharded(0) if a == sharded(0) else REPL
        elif op in (OpKind.MAX_POOL, OpKind.MAX_POOL_BACKPROP):
            # pooling is per image: the batch shard carries through
            if all(s == sharded(0) for s in ins):
                st[n] = sharded(0)
            elif all(s == REPL for s in ins):
                st[n] = REPL
            else:
                need_all()
                st[n] = REPL
        elif op is OpKind.CONV_BACKPROP_FILTER:
            a, b = ins
            if a == sharded(0) and b == sharded(0):
                st[n] = PART
            elif a == REPL and b == REPL:
                st[n] = REPL
            else:
                need_all()
                st[n] = REPL
        else:
            raise UnsupportedOp(f"data parallel: no rule for {op.wire_name}")
    for r, _ in g.results:
        if st[r] in (PART, PMAX):
            demand.append((None, r))
    return st, demand


def _root_of(g: Function, st: dict, n: int):
    """Walk back through linear ops to the materialised node that created the partial."""
    node = g.nodes[n]
    op = node.op
    if st[n] == PMAX:
        return [n]
    if op in (OpKind.DOT, OpKind.CONV_BACKPROP_FILTER):
        ins = [st[r] for r, _ in node.inputs]
        if PART not in ins:
            return [n]  # batch contraction creates the partial here
    if op is OpKind.SUM and st[node.inputs[0][0]] != PART:
        return [n]
    roots = []
    for r, _ in node.inputs:
        if st[r] == PART:
            roots.extend(_root_of(g, st, r))
    return roots


def analyse(g: Function, dp: DataParallel) -> set:
    """Fill `dp.allreduce` with the partial roots that must be summed."""
    dp.allreduce = set()
    dp.allreduce_max = set()
    for _ in range(len(g.nodes) + 1):
        st, demand = _propagate(g, dp)
        if not demand:
            dp.states = st
            return dp.allreduce
        for _, r in demand:
            for root in _root_of(g, st, r):
                dp.allreduce.add(root)
                if st[root] == PMAX:
                    dp.allreduce_max.add(root)
    raise UnsupportedOp("data parallel analysis did not converge")
