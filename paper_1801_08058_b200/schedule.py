"""Multi-stream capture schedule for an executable's launch list.

`call` replays one CUDA graph per step.  Captured from a single stream, the
graph is a chain: every launch waits for the previous one.  Many launches of
a training step are independent (a layer's weight gradient and its data
gradient, bias sums, the optimizer updates), so the schedule computed here
captures each launch on one of a few streams and makes it wait, by event,
only for the earlier launches it conflicts with.  The graph then has those
launches as concurrent nodes.

Conflicts are decided on physical memory, not on tensor identity: the arena
planner reuses an arena range once its tensor is dead *in launch order*, so
two launches touching overlapping arena bytes with at least one write must
stay ordered (read-after-write, write-after-read and write-after-write).
Caller buffers and the constant pool are compared per slot.
"""

from __future__ import annotations

from . import abi


def _ranges(lowered, keys, write):
    """(space, lo, hi, write) per tensor key; unknown keys conflict with everything."""
    out = []
    for k in keys:
        b = lowered.buffers.get(k)
        if b is None:
            out.append(("*", 0, 1 << 62, write))
            continue
        root = b.base if b.base is not None else b
        if root.splat is not None:
            continue  # a scalar in the argument block: no memory
        if getattr(b, "bucket", None) is not None or (getattr(b, "exact", False) and b.base is not None):
            # a partial root inside the gradient region, or a row-chunk view:
            # exactly its own bytes
            base = lowered.arena_offsets.get(root.key, root.offset) if root.slot == abi.SLOT_ARENA else 0
            lo = base + b.elem_off * b.et.byte_size
            out.append((0 if root.slot == abi.SLOT_ARENA else root.slot, lo, lo + max(1, b.nbytes), write))
            continue
        if root.slot == abi.SLOT_ARENA:
            lo = lowered.arena_offsets.get(root.key, root.offset)
            out.append((0, lo, lo + max(1, root.nbytes), write))
        else:
            out.append((root.slot, 0, 1 << 62, write))
    return out


def _conflict(a, b) -> bool:
    for sa, la, ha, wa in a:
        for sb, lb, hb, wb in b:
            if (wa or wb) and (sa == sb or sa == "*" or sb == "*") and la < hb and lb < ha:
                return True
    return False


def build(lowered, skipped=(), n_streams: int = 4):
    """(stream_of, dep_offsets, deps) for gfb_exe_set_schedule.  `skipped`:
    launches folded into the preceding merged kernel (their accesses belong
    to it)."""
    n = len(lowered.launches)
    skipped = set(skipped)
    acc = []
    head = list(range(n))
    for i, L in enumerate(lowered.launches):
        acc.append(_ranges(lowered, L.reads, False) + _ranges(lowered, L.writes, True))
        if i in skipped and i > 0:
            head[i] = head[i - 1]
    for i in range(n):  # a merged kernel does its members' work
        if head[i] != i:
            acc[head[i]] += acc[i]
    deps = [[] for _ in range(n)]
    live = [i for i in range(n) if head[i] == i]
    chain_last = {}
    for x, i in enumerate(live):
        for j in live[:x]:
            if _conflict(acc[i], acc[j]):
                deps[i].append(j)
        # launches of one chain (the split / GEMM row chunks of a large input)
        # stay in order: run concurrently, a chunk's split kernel takes SMs
        # from the persistent GEMM of the previous chunk (measured: +18 ms on
        # config E's host-buffer step)
        ch = getattr(lowered.launches[i], "chain", None)
        if ch is not None:
            if ch in chain_last and chain_last[ch] not in deps[i]:
                deps[i].append(chain_last[ch])
            chain_last[ch] = i
    stream_of = [0] * n
    tail = [-1] * n_streams
    last_collective = None
    for i in range(n):
        if head[i] != i:
            stream_of[i] = stream_of[head[i]]
            deps[i] = [head[i]]
            continue
        if lowered.launches[i].kind == abi.K_ALLREDUCE:
            # collectives stay on stream 0 in program order: every rank's graph
            # then issues them in the same sequence
            if last_collective is not None and last_collective not in deps[i]:
                deps[i].append(last_collective)
            last_collective = i
            stream_of[i] = 0
            tail[0] = i
            continue
        ends = [d for d in deps[i] if tail[stream_of[d]] == d]
        if ends:
            st = stream_of[max(ends)]  # continue the chain of the latest dependency
        else:
            st = min(range(n_streams), key=lambda k: tail[k])  # the least recently used stream
        stream_of[i] = st
        tail[st] = i
    offsets, flat = [0], []
    for d in deps:
        flat += d
        offsets.append(len(flat))
    return stream_of, offsets, flat


def io_pieces(lowered, in_bytes, skipped=()):
    """Input pieces for gfb_exe_set_io_pieces, or None when every launch
    reads whole inputs: (piece_input, piece_offset, piece_bytes,
    read_offsets, reads) where launches reading a row-chunk view of a caller
    input read only the pieces it covers, so those bytes cross PCIe (and
    their readers start) ahead of the rest of the input."""
    n = len(lowered.launches)
    skipped = set(skipped)
    head = list(range(n))
    for i in range(1, n):
        if i in skipped:
            head[i] = head[i - 1]
    n_in = lowered.n_inputs
    sizes = [int(b) for b in in_bytes]
    if len(sizes) != n_in:
        return None
    acc = [[] for _ in range(n)]  # (input, lo, hi) per launch
    cuts = [{0, sizes[k]} for k in range(n_in)]
    ranged = False
    for i, L in enumerate(lowered.launches):
        for k in L.reads:
            b = lowered.buffers.get(k)
            if b is None:
                acc[head[i]] += [(j, 0, sizes[j]) for j in range(n_in)]
                continue
            root = b.base if b.base is not None else b
            if root.splat is not None or not (abi.SLOT_IO <= root.slot < abi.SLOT_IO + n_in):
                continue
            j = root.slot - abi.SLOT_IO
            if getattr(b, "exact", False) and b.base is not None:
                lo = b.elem_off * b.et.byte_size
                hi = min(sizes[j], lo + b.nbytes)
                cuts[j] |= {lo, hi}
                acc[head[i]].append((j, lo, hi))
                ranged = True
            else:
                acc[head[i]].append((j, 0, sizes[j]))
    if not ranged:
        return None
    p_in, p_off, p_len, first = [], [], [], []
    for j in range(n_in):
        c = sorted(cuts[j])
        first.append(len(p_in))
        for a, b_ in zip(c, c[1:]):
            p_in.append(j)
            p_off.append(a)
            p_len.append(b_ - a)
        if len(c) == 1:  # an empty input: one empty piece
            p_in.append(j)
            p_off.append(0)
            p_len.append(0)
    offsets, flat = [0], []
    for i in range(n):
        ps = set()
        for j, lo, hi in acc[i]:
            for p in range(first[j], len(p_in)):
                if p_in[p] != j:
                    break
                if p_off[p] < hi and lo < p_off[p] + p_len[p] or (lo == hi == p_off[p] == 0 and p_len[p] == 0):
                    ps.add(p)
        flat += sorted(ps)
        offsets.append(len(flat))
    return p_in, p_off, p_len, offsets, flat


def io_access(lowered, skipped=()):
    """(read_offsets, reads, out_writer) for gfb_exe_set_io: the caller inputs
    each launch reads and the last launch writing each result (None if some
    result is written by no launch).  A launch
    folded into a preceding merged kernel counts as that kernel's access."""
    n = len(lowered.launches)
    skipped = set(skipped)
    head = list(range(n))
    for i in range(1, n):
        if i in skipped:
            head[i] = head[i - 1]
    n_in = lowered.n_inputs
    reads = [set() for _ in range(n)]
    writer = [None] * lowered.n_outputs

    def slots(keys):
        for k in keys:
            b = lowered.buffers.get(k)
            if b is None:
                yield None
                continue
            root = b.base if b.base is not None else b
            if root.splat is None:
                yield root.slot

    for i, L in enumerate(lowered.launches):
        h = head[i]
        for s in slots(L.reads):
            if s is None:  # unknown access: wait for every input
                reads[h].update(range(n_in))
            elif abi.SLOT_IO <= s < abi.SLOT_IO + n_in:
                reads[h].add(s - abi.SLOT_IO)
        for s in slots(L.writes):
            if s is not None and s >= abi.SLOT_IO + n_in:
                writer[s - abi.SLOT_IO - n_in] = h
    if any(w is None for w in writer):
        return None  # a result no launch writes: host-buffer runs are not offered
    offsets, flat = [0], []
    for r in reads:
        flat += sorted(r)
        offsets.append(len(flat))
    return offsets, flat, writer
