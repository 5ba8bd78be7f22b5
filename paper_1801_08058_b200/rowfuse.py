"""Row-fused launches: a softmax-shaped subgraph in one kernel.

The reference builds softmax as a 7-node composite (`build_softmax`,
`/root/reference/pkg/src/graphforge/ir.py:735-763`: max-reduce, Broadcast,
Subtract, Exp, Sum, Broadcast, Divide); `differentiate` expands its
gradient into about ten more nodes (`autodiff.py:116-252`), and a
cross-entropy loss adds Log / Multiply / Sum.  Lowered node by node, every
row reduction is a separate launch and every [rows, classes] intermediate
an HBM round trip: config E's loss head ([65536, 4096]) made a dozen passes
over 1 GiB tensors.

A *row group* is a convex subgraph over an R x C iteration space whose
members are

* FULL [R, C]: elementwise ops, and Broadcasts of a ROWV member / [R] input
  along axis 1, of a [C] input along axis 0, or of a scalar;
* ROWV [R]: Sum or max over axis 1 of a FULL member, elementwise ops on ROWV
  values, Broadcasts of scalars;
* UNI []: elementwise ops on scalars (every thread computes them once);
* XROW []: a Sum (or max) over both axes of a FULL member, or over axis 0 of
  a ROWV member -- a cross-row reduction, consumed only outside the group.

The whole group runs as one generated kernel (NVRTC, like jit.py's): a team
of threads owns one row at a time, holds every FULL value of the row in
registers (16 elements per thread at C = 4096) across the row reductions,
reads each external input once and writes only the members consumed outside
the group.  XROW values are folded per team and summed by a short second
launch.  Element operations are the generic kernels' own (csrc/ew_ops.cuh
`bin1`, `apply_unary`, `fold`), so every elementwise result is bit-identical
to the unfused plan; row reductions use a per-thread fold plus a fixed tree
(the tolerance the reference's sequential folds are compared at, like every
other device reduction).  E's head becomes: read the last GEMM's output and
t once, write dz once.
"""

from __future__ import annotations

import os
import struct
from dataclasses import dataclass, field

from . import abi
from .ir import ELEMENTWISE_BINARY, ELEMENTWISE_UNARY, ElementType, OpKind

FULL, ROWV, UNI, XROW, COLV = "full", "rowv", "uni", "xrow", "colv"
MAX_C = 8192
MIN_ROWS = 296  # two teams per SM, else only small (latency-bound) groups are fused
SMALL = 1 << 17
MAX_FULL_LIVE = 12  # FULL values a thread may hold at once (registers)

UNARY_CODE = {OpKind.NEGATE: 5, OpKind.EXP: 6, OpKind.LOG: 7, OpKind.TANH: 8, OpKind.SIGMOID: 9, OpKind.RELU: 10}
BINARY_CODE = {OpKind.ADD: 0, OpKind.SUBTRACT: 1, OpKind.MULTIPLY: 2, OpKind.DIVIDE: 3, OpKind.MAXIMUM: 4}


def enabled() -> bool:
    from . import jit

    return jit.enabled() and os.environ.get("GFB_ROWFUSE", "1") == "1"


@dataclass
class RowGroup:
    R: int
    C: int
    et: ElementType
    members: list  # node ids, evaluation (topological) order
    cls: dict  # member -> FULL / ROWV / UNI / XROW
    externals: dict  # external input -> FULL / ROWV / COLV / UNI
    outputs: list = field(default_factory=list)  # members stored to memory
    anchor: int = -1  # the member after which the group launch is emitted


def _class_of(low, n, R, C):
    node = low.nodes[n]
    d = node.output
    if not d.element_type.is_float or n in low.tiny or low.is_heavy(n):
        return None
    shape = tuple(d.shape)
    op = node.op
    if op in ELEMENTWISE_UNARY or op in ELEMENTWISE_BINARY:
        return {(R, C): FULL, (R,): ROWV, (): UNI}.get(shape)
    if op is OpKind.BROADCAST:
        ins, axes = tuple(node.inputs_shape), tuple(sorted(node.attrs["broadcast_axes"]))
        if shape == (R, C):
            if ins == (R,) and axes == (1,):
                return FULL
            if ins == (C,) and axes == (0,):
                return FULL
            if ins == ():
                return FULL
        if shape == (R,) and ins == ():
            return ROWV
        return None
    if op is OpKind.SUM:
        ins, axes = tuple(node.inputs_shape), tuple(sorted(node.attrs["reduction_axes"]))
        if ins == (R, C) and axes == (1,):
            return ROWV
        if (ins == (R, C) and axes == (0, 1)) or (ins == (R,) and axes == (0,)):
            return XROW
    return None


def _grow(low, seed, R, C, taken):
    cls = {seed: ROWV}
    stack = [seed]
    while stack:
        n = stack.pop()
        for r, _ in low.nodes[n].inputs:  # upward: any light input (materialised or not)
            if r in cls or r in taken or low.nodes[r].op in (OpKind.PARAMETER, OpKind.CONSTANT) or low.is_heavy(r):
                continue
            c = _class_of(low, r, R, C)
            if c is None or c == XROW:
                continue
            cls[r] = c
            stack.append(r)
        if cls[n] in (XROW, UNI):  # nothing in the group may read a cross-row value; scalars are replicated
            continue
        for c_ in low.consumers[n]:  # downward
            if c_ in cls or c_ in taken:
                continue
            c = _class_of(low, c_, R, C)
            if c is not None:
                cls[c_] = c
                stack.append(c_)
    return cls


def _convex(low, members) -> bool:
    """No path leaves the group and re-enters it."""
    down, stack = set(), [c for m in members for c in low.consumers[m] if c not in members]
    while stack:
        x = stack.pop()
        if x in down:
            continue
        down.add(x)
        stack += [c for c in low.consumers[x] if c not in members]
    up, stack = set(), [r for m in members for r, _ in low.nodes[m].inputs if r not in members]
    while stack:
        x = stack.pop()
        if x in up or x not in low.nodes:
            continue
        up.add(x)
        stack += [r for r, _ in low.nodes[x].inputs if r not in members]
    return not (down & up)


def _validate(low, cls, R, C):
    """(externals, outputs, force) or None.  `force`: external inputs that
    must be materialised for the group to read them."""
    members = set(cls)
    results = {r for r, _ in low.g.results}
    externals, force = {}, set()
    for n in members:
        node = low.nodes[n]
        c = cls[n]
        ins = [r for r, _ in node.inputs]
        if c == XROW and any(x in members for x in low.consumers[n]):
            return None
        if c == UNI and any(low.nodes[r].output.shape != () for r in ins):
            return None
        for r in ins:
            if r in members:
                rc = cls[r]
                if node.op is OpKind.BROADCAST:
                    axes = tuple(sorted(node.attrs["broadcast_axes"]))
                    ok = (rc == ROWV and axes == (1,) and c == FULL) or rc == UNI
                elif node.op is OpKind.SUM:
                    ok = (rc == FULL) or (rc == ROWV and c == XROW)
                else:
                    ok = rc == c or (rc == UNI and c == UNI)
                if not ok:
                    return None
                continue
            shape = tuple(low.nodes[r].output.shape)
            if node.op is OpKind.BROADCAST:
                axes = tuple(sorted(node.attrs["broadcast_axes"]))
                ec = UNI if shape == () else (COLV if axes == (0,) else ROWV)
            elif node.op is OpKind.SUM:
                ec = FULL if shape == (R, C) else ROWV
            else:
                ec = c
            if {FULL: (R, C), ROWV: (R,), COLV: (C,), UNI: (), XROW: ()}[ec] != shape:
                return None
            if externals.get(r, ec) != ec:
                return None
            externals[r] = ec
            if low.nodes[r].output.element_type != low.nodes[n].output.element_type:
                return None
            if not low.is_source(r) and not (low.viewable(r) if ec != UNI else False):
                force.add(r)
    outputs = [n for n in members if cls[n] != UNI and (n in results or n in low.allreduce
                                                         or any(x not in members for x in low.consumers[n]))]
    if not any(cls[n] == ROWV and low.nodes[n].op is OpKind.SUM for n in members):
        return None
    if sum(1 for n in members if cls[n] == FULL) < 2:
        return None
    return externals, outputs, force


def find_groups(low) -> list:
    """Row groups of a lowering (before buffers exist; uses its
    materialisation set M).  Largest first; members never overlap."""
    groups, taken = [], set()
    seeds = [n for n in low.order if low.nodes[n].op is OpKind.SUM and len(low.nodes[n].inputs_shape) == 2
             and tuple(sorted(low.nodes[n].attrs["reduction_axes"])) == (1,)]
    for s in seeds:
        if s in taken:
            continue
        R, C = low.nodes[s].inputs_shape
        et = low.nodes[s].output.element_type
        if not (2 <= C <= MAX_C) or R < 1 or et not in (ElementType.F32, ElementType.F64):
            continue
        if R < MIN_ROWS and R * C > SMALL:
            continue  # few long rows: the chunk-wise reductions spread them over the GPU instead
        cls = _grow(low, s, R, C, taken)
        if any(low.nodes[n].output.element_type != et for n in cls):
            continue
        v = _validate(low, cls, R, C)
        if v is None or not _convex(low, set(cls)):
            continue
        externals, outputs, force = v
        order = [n for n in low.order if n in cls]
        g = RowGroup(R, C, et, order, cls, externals, outputs)
        g.force = force
        g.anchor = order[-1]
        groups.append(g)
        taken |= set(cls)
    return groups


def reorder(order: list, consumers: dict, inputs_of, groups: list) -> list:
    """A topological order in which each group's members are contiguous
    (groups are convex, so contracting each to one unit keeps a DAG); ties
    go to the smallest node id, like ir.topological_order."""
    import heapq

    unit_of = {}
    for gi, g in enumerate(groups):
        for m in g.members:
            unit_of[m] = ("g", gi)
    units = {}
    for n in order:
        u = unit_of.get(n, ("n", n))
        units.setdefault(u, []).append(n)
    indeg = {u: 0 for u in units}
    succ = {u: set() for u in units}
    for u, ns in units.items():
        for n in ns:
            for r in inputs_of(n):
                ur = unit_of.get(r, ("n", r))
                if ur in units and ur != u and u not in succ[ur]:
                    succ[ur].add(u)
                    indeg[u] += 1
    heap = [(min(ns), u) for u, ns in units.items() if indeg[u] == 0]
    heapq.heapify(heap)
    out = []
    while heap:
        _, u = heapq.heappop(heap)
        out += units[u]
        for v in succ[u]:
            indeg[v] -= 1
            if indeg[v] == 0:
                heapq.heappush(heap, (min(units[v]), v))
    assert len(out) == len(order), "row groups broke the topological order"
    return out


# ---------------------------------------------------------------------------
# The launch: a small value program shared by the code generator and the
# host emulator (tests/plan_emulator.py)


@dataclass
class RowSpec:
    R: int
    C: int
    dtype: str  # "float" / "double"
    team: int
    block: int
    vec: int
    values: list  # (class, expr) in evaluation order; exprs reference earlier values by index
    stores: list  # (value index, ref index, s0, s1)
    xrow: list  # (value index, kind, ref index of the per-team partials)
    n_teams: int = 0


def geometry(C: int, esize: int, vec_ok: bool):
    """(team threads, block threads, vector width) for C columns."""
    vec = (16 // esize) if vec_ok and C % (16 // esize) == 0 else 1
    if C <= 256:
        team = 32
        block = 256
    else:
        team = 64
        while team < 512 and C > team * vec * 4:
            team *= 2
        block = team
    return team, block, vec


def splat_bits(et: ElementType, value) -> int:
    if et is ElementType.F32:
        return struct.unpack("<I", struct.pack("<f", float(value)))[0]
    return struct.unpack("<Q", struct.pack("<d", float(value)))[0]


def generate_source(spec: RowSpec) -> str:
    """CUDA C of a row group's kernel (entry `gfb_jit_ew`, like jit.py's)."""
    T, TEAM, BLOCK, VEC, C, R = spec.dtype, spec.team, spec.block, spec.vec, spec.C, spec.R
    ufn = "row" if os.environ.get("GFB_ROW_F32_TRANSCENDENTALS", "0") == "1" else "c"  # (off: the reference's bits)
    NSLOT = (C + TEAM * VEC - 1) // (TEAM * VEC)
    EPT = NSLOT * VEC
    full_rows = C % (TEAM * VEC) == 0
    L = ['#include "ew_ops.cuh"', "using namespace gfb;", f"typedef {T} T;",
         f"constexpr int TEAM = {TEAM}, VEC = {VEC}, EPT = {EPT}, NSLOT = {NSLOT};",
         f"constexpr uint32_t C_ = {C}u, R_ = {R}u;",
         "__device__ __forceinline__ uint32_t col_of(int i, int lane) { return ((uint32_t)(i / VEC) * TEAM + lane) * VEC + (i % VEC); }"]
    if TEAM > 32:
        L += ["template <int KIND> __device__ __forceinline__ T team_reduce(T v, T* sm, int lane) {",
              "  _Pragma(\"unroll\") for (int off = 16; off > 0; off >>= 1) v = fold<T>(KIND, v, __shfl_xor_sync(0xffffffffu, v, off));",
              "  if ((lane & 31) == 0) sm[lane >> 5] = v;",
              "  __syncthreads();",
              "  v = sm[0];",
              "  _Pragma(\"unroll\") for (int w = 1; w < TEAM / 32; ++w) v = fold<T>(KIND, v, sm[w]);",
              "  __syncthreads();",
              "  return v;", "}"]
    else:
        L += ["template <int KIND> __device__ __forceinline__ T team_reduce(T v, T*, int) {",
              "  _Pragma(\"unroll\") for (int off = 16; off > 0; off >>= 1) v = fold<T>(KIND, v, __shfl_xor_sync(0xffffffffu, v, off));",
              "  return v;", "}"]
    L += [f'extern "C" __global__ void __launch_bounds__({BLOCK}) gfb_jit_ew(const __grid_constant__ gfb_row_args pa) {{',
          f"__shared__ T red_sm[{max(1, TEAM // 32)}];",
          "const int lane = threadIdx.x % TEAM;",
          "const uint32_t team = blockIdx.x * (blockDim.x / TEAM) + threadIdx.x / TEAM;",
          "const uint32_t nteams = gridDim.x * (blockDim.x / TEAM);"]
    refs_used = sorted({e[1] for _, e in spec.values if e[0] in ("load", "loadr", "loadu", "colv")}
                       | {s[1] for s in spec.stores} | {x[2] for x in spec.xrow})
    for i in refs_used:
        L.append(f"T* const P{i} = resolve<T>(pa.tab, pa.refs[{i}]);")

    def valid(i):
        return "true" if full_rows else f"(col_of({i}, lane) < C_)"

    # scalars (UNI) before the row loop
    for k, (c, e) in enumerate(spec.values):
        if c != UNI:
            continue
        if e[0] == "imm":
            L.append(f"const T v{k} = from_bits<T>({e[1]}ull);")
        elif e[0] == "loadu":
            L.append(f"const T v{k} = P{e[1]}[0];")
        elif e[0] == "un":
            L.append(f"T v{k}_[1] = {{v{e[2]}}}; apply_unary_{ufn}<{e[1]}u, T, 1>(v{k}_); const T v{k} = v{k}_[0];")
        elif e[0] == "bin":
            L.append(f"const T v{k} = bin1<T>({e[1]}u, v{e[2]}, v{e[3]});")
        else:
            raise ValueError(e)
    for x, kind, _ in spec.xrow:
        L.append(f"T xacc{x} = fold_init<T>({kind});")
    L.append("for (uint32_t row = team; row < R_; row += nteams) {")
    for k, (c, e) in enumerate(spec.values):
        if c == UNI:
            continue
        op = e[0]
        if c == FULL:
            if op == "load":
                _, ref, s0, s1 = e
                L.append(f"T v{k}[EPT];")
                if VEC > 1 and s1 == 1:
                    L.append(f"_Pragma(\"unroll\") for (int j = 0; j < NSLOT; ++j) {{ const uint32_t c0 = col_of(j * VEC, lane);"
                             f" if ({'true' if full_rows else 'c0 < C_'}) {{ T tmp[VEC]; loadV_plain<T, VEC>(P{ref} + (size_t)row * {s0}u + c0, tmp);"
                             f" _Pragma(\"unroll\") for (int v = 0; v < VEC; ++v) v{k}[j * VEC + v] = tmp[v]; }}"
                             f" else {{ _Pragma(\"unroll\") for (int v = 0; v < VEC; ++v) v{k}[j * VEC + v] = T(0); }} }}")
                else:
                    L.append(f"_Pragma(\"unroll\") for (int i = 0; i < EPT; ++i) v{k}[i] = {valid('i')} ? "
                             f"P{ref}[(size_t)row * {s0}u + (size_t)col_of(i, lane) * {s1}u] : T(0);")
            elif op == "colv":
                _, ref, s = e
                L.append(f"T v{k}[EPT]; _Pragma(\"unroll\") for (int i = 0; i < EPT; ++i) v{k}[i] = {valid('i')} ? "
                         f"P{ref}[(size_t)col_of(i, lane) * {s}u] : T(0);")
            elif op == "bcast":  # a ROWV / UNI value across the columns
                L.append(f"T v{k}[EPT]; _Pragma(\"unroll\") for (int i = 0; i < EPT; ++i) v{k}[i] = v{e[1]};")
            elif op == "un":
                L.append(f"T v{k}[EPT]; copyV<T, EPT>(v{k}, v{e[2]}); apply_unary_{ufn}<{e[1]}u, T, EPT>(v{k});")
            elif op == "bin":
                L.append(f"T v{k}[EPT]; _Pragma(\"unroll\") for (int i = 0; i < EPT; ++i) v{k}[i] = bin1<T>({e[1]}u, v{e[2]}[i], v{e[3]}[i]);")
            else:
                raise ValueError(e)
        elif c == ROWV:
            if op == "loadr":
                L.append(f"const T v{k} = P{e[1]}[(size_t)row * {e[2]}u];")
            elif op == "bcast":
                L.append(f"const T v{k} = v{e[1]};")
            elif op == "un":
                L.append(f"T v{k}_[1] = {{v{e[2]}}}; apply_unary_{ufn}<{e[1]}u, T, 1>(v{k}_); const T v{k} = v{k}_[0];")
            elif op == "bin":
                L.append(f"const T v{k} = bin1<T>({e[1]}u, v{e[2]}, v{e[3]});")
            elif op == "rred":
                _, kind, a = e
                L.append(f"T v{k} = fold_init<T>({kind}); _Pragma(\"unroll\") for (int i = 0; i < EPT; ++i)"
                         f" if ({valid('i')}) v{k} = fold<T>({kind}, v{k}, v{a}[i]);")
                L.append(f"v{k} = team_reduce<{kind}>(v{k}, red_sm, lane);")
            else:
                raise ValueError(e)
        elif c == XROW:
            _, kind, a, src_cls = e
            if src_cls == FULL:
                L.append(f"{{ T p = fold_init<T>({kind}); _Pragma(\"unroll\") for (int i = 0; i < EPT; ++i)"
                         f" if ({valid('i')}) p = fold<T>({kind}, p, v{a}[i]);")
                L.append(f"  p = team_reduce<{kind}>(p, red_sm, lane); xacc{k} = fold<T>({kind}, xacc{k}, p); }}")
            else:
                L.append(f"xacc{k} = fold<T>({kind}, xacc{k}, v{a});")
    for k, ref, s0, s1 in spec.stores:
        c = spec.values[k][0]
        if c == FULL:
            if VEC > 1 and s1 == 1:
                L.append(f"_Pragma(\"unroll\") for (int j = 0; j < NSLOT; ++j) {{ const uint32_t c0 = col_of(j * VEC, lane);"
                         f" if ({'true' if full_rows else 'c0 < C_'}) {{ T tmp[VEC]; _Pragma(\"unroll\") for (int v = 0; v < VEC; ++v)"
                         f" tmp[v] = v{k}[j * VEC + v]; storeV<T, VEC>(P{ref} + (size_t)row * {s0}u + c0, tmp); }} }}")
            else:
                L.append(f"_Pragma(\"unroll\") for (int i = 0; i < EPT; ++i) if ({valid('i')}) "
                         f"P{ref}[(size_t)row * {s0}u + (size_t)col_of(i, lane) * {s1}u] = v{k}[i];")
        else:  # ROWV
            L.append(f"if (lane == 0) P{ref}[(size_t)row * {s0}u] = v{k};")
    L.append("}")  # row loop
    for x, kind, ref in spec.xrow:
        L.append(f"if (lane == 0) P{ref}[team] = xacc{x};")
    L.append("}")
    return "\n".join(L) + "\n"
