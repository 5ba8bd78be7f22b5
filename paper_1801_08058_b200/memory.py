"""Liveness analysis and first-fit arena planning.

Two planners live here:

* `liveness` / `plan_memory` restate the reference planner
  (`/root/reference/pkg/src/graphforge/memory.py:45-120`) over IR nodes: the
  per-node plan that `Executable.plan` and `listing()` expose, kept so the
  compiled listing is comparable with the reference's.
* `plan_buffers` is what the device actually uses: the same first-fit rule
  over *materialised buffers of fused launches* (liveness measured in launch
  indices), 256-byte aligned so every buffer starts on a TMA / 128-bit
  vector boundary.  Intermediates that fusion keeps in registers never get a
  slot at all.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

from .ir import Function, OpKind, reachable_from_results, topological_order

ALIGNMENT = 64
DEVICE_ALIGNMENT = 256
END_OF_PROGRAM = math.inf


@dataclass(frozen=True)
class LiveInterval:
    tensor: tuple[int, int]
    start: int
    end: int | float


@dataclass
class MemoryPlan:
    arena_size: int
    placements: dict
    intervals: list
    alignment: int = ALIGNMENT
    sizes: dict = field(default_factory=dict)


def align_up(n: int, alignment: int = ALIGNMENT) -> int:
    return (n + alignment - 1) // alignment * alignment


def intervals_overlap(a: LiveInterval, b: LiveInterval) -> bool:
    # Inclusive on both ends: a tensor is still live while its last
    # consumer writes, so producer and consumer never share bytes.
    return a.start <= b.end and b.start <= a.end


def liveness(fn: Function) -> list[LiveInterval]:
    order = topological_order(fn)
    index = {nid: i for i, nid in enumerate(order)}
    reachable = reachable_from_results(fn)
    results = set(fn.results)
    last_use: dict = {}
    for nid in reachable:
        for ref in fn.nodes[nid].inputs:
            last_use[ref] = max(last_use.get(ref, -1), index[nid])
    out = []
    for nid in sorted(reachable, key=lambda i: (index[i], i)):
        node = fn.nodes[nid]
        start = 0 if node.op in (OpKind.PARAMETER, OpKind.CONSTANT) else index[nid]
        for port in range(len(node.outputs)):
            ref = (nid, port)
            end = END_OF_PROGRAM if ref in results else last_use.get(ref, index[nid])
            out.append(LiveInterval(ref, start, end))
    return out


def first_fit(items, sizes, alignment):
    """Place (key, start, end) items first-fit; returns (placements, size).

    Items are visited in (start asc, size desc, key asc) order and each gets
    the lowest aligned offset disjoint from every placed, live-overlapping
    item.
    """
    ordered = sorted(items, key=lambda it: (it[1], -sizes[it[0]], it[0]))
    placed: list = []
    placements = {}
    for key, start, end in ordered:
        size = sizes[key]
        busy = sorted(
            (off, off + sizes[k2])
            for k2, s2, e2, off in placed
            if start <= e2 and s2 <= end
        )
        offset = 0
        for lo, hi in busy:
            if offset + size <= lo:
                break
            offset = max(offset, align_up(hi, alignment))
        placements[key] = offset
        placed.append((key, start, end, offset))
    top = max((placements[k] + sizes[k] for k in placements), default=0)
    return placements, align_up(top, alignment)


def plan_memory(fn: Function) -> MemoryPlan:
    intervals = liveness(fn)
    results = set(fn.results)
    sizes = {}
    items = []
    for iv in intervals:
        node = fn.nodes[iv.tensor[0]]
        sizes[iv.tensor] = node.outputs[iv.tensor[1]].byte_size
        if node.op in (OpKind.PARAMETER, OpKind.CONSTANT) or iv.tensor in results:
            continue
        items.append((iv.tensor, iv.start, iv.end))
    placements, arena = first_fit(items, sizes, ALIGNMENT)
    return MemoryPlan(arena, placements, intervals, ALIGNMENT, sizes)


def liveness_reference(fn: Function) -> list[LiveInterval]:
    """Quadratic re-scan used by tests to pin `liveness`."""
    order = topological_order(fn)
    index = {nid: i for i, nid in enumerate(order)}
    reachable = reachable_from_results(fn)
    results = set(fn.results)
    out = []
    for nid in sorted(reachable, key=lambda i: (index[i], i)):
        node = fn.nodes[nid]
        start = 0 if node.op in (OpKind.PARAMETER, OpKind.CONSTANT) else index[nid]
        for port in range(len(node.outputs)):
            ref = (nid, port)
            if ref in results:
                end = END_OF_PROGRAM
            else:
                end = start
                for later in order:
                    if later in reachable and ref in fn.nodes[later].inputs:
                        end = max(end, index[later])
            out.append(LiveInterval(ref, start, end))
    return out


@dataclass
class BufferPlan:
    """Device arena plan over materialised launch buffers."""

    arena_size: int
    offsets: dict  # buffer key -> byte offset
    sizes: dict
    intervals: dict  # buffer key -> (first launch, last launch)


def plan_buffers(buffers: dict, private: bool = False) -> BufferPlan:
    """`buffers`: key -> (byte_size, first_launch, last_launch).

    With `private` every buffer gets disjoint bytes (the device analogue of
    the reference `call(..., private_buffers=True)` plan-corruption check).
    """
    sizes = {k: max(v[0], 1) for k, v in buffers.items()}
    if private:
        items = [(k, 0, END_OF_PROGRAM) for k in buffers]
    else:
        items = [(k, v[1], v[2]) for k, v in buffers.items()]
    offsets, arena = first_fit(items, sizes, DEVICE_ALIGNMENT)
    return BufferPlan(arena, offsets, sizes, {k: (v[1], v[2]) for k, v in buffers.items()})
