"""Multi-stream capture schedule (paper_1801_08058_b200/schedule.py): every
pair of launches that touch overlapping memory with a write stays ordered,
merged launches follow their head, collectives keep program order."""

import pytest

import golden_io as G
from hostcompile import host_compile

from paper_1801_08058_b200 import abi, schedule


def _closure(deps_of, n):
    reach = [set() for _ in range(n)]
    for i in range(n):
        for d in deps_of[i]:
            reach[i] |= {d} | reach[d]
    return reach


def _check(lowered, skipped=()):
    st, off, flat = schedule.build(lowered, skipped, 4)
    n = len(lowered.launches)
    head = list(range(n))
    for i in range(1, n):
        if i in skipped:
            head[i] = head[i - 1]
    deps_of = [flat[off[i]:off[i + 1]] for i in range(n)]
    assert all(d < i for i in range(n) for d in deps_of[i])
    assert all(0 <= s < 4 for s in st)
    reach = _closure(deps_of, n)
    acc = [schedule._ranges(lowered, L.reads, False) + schedule._ranges(lowered, L.writes, True) for L in lowered.launches]
    for i in range(n):
        for j in range(i):
            if head[i] != head[j] and schedule._conflict(acc[i], acc[j]):  # one merged kernel runs in order
                # ordered through a chain of waits (a merged launch runs as its head)
                assert head[j] in reach[head[i]], (i, j)
    return st, deps_of


@pytest.mark.parametrize("name", ["mlp_A_small", "cnn_C_small", "resnet_D_small", "mlp_E_small"])
def test_schedule_orders_every_conflict(name):
    case = next(c for c in G.load("workloads.json.gz") if c["name"] == name)
    h = host_compile(G.fn_of(case["fn"]), conv_layout="nhwc" if name.startswith("resnet") else "identity")
    st, _ = _check(h.lowered)
    assert len(set(st)) > 1  # some launches do run on other streams


def test_schedule_merged_members_follow_their_head():
    case = next(c for c in G.load("workloads.json.gz") if c["name"] == "mlp_A_small")
    h = host_compile(G.fn_of(case["fn"]))
    n = len(h.lowered.launches)
    skipped = [i for i in range(1, n) if tuple(h.lowered.launches[i].grid) == (1, 1, 1)
               and tuple(h.lowered.launches[i - 1].grid) == (1, 1, 1)][:3]
    st, deps_of = _check(h.lowered, skipped)
    for i in skipped:
        h0 = i - 1
        while h0 in skipped:
            h0 -= 1
        assert deps_of[i] == [h0] and st[i] == st[h0]


def test_schedule_keeps_collectives_in_order():
    from paper_1801_08058_b200 import workloads as W
    import paper_1801_08058_b200 as gf
    from paper_1801_08058_b200.dp import DataParallel

    step = W.mlp_step(gf, batch=8, in_dim=16, hidden=(8,), out_dim=4)
    names = step.param_names
    dp = DataParallel([step.fn.parameters[names.index("x")], step.fn.parameters[names.index("t")]], world_size=2)
    h = host_compile(step.fn, data_parallel=dp)
    coll = [i for i, L in enumerate(h.lowered.launches) if L.kind == abi.K_ALLREDUCE]
    assert len(coll) >= 1
    st, deps_of = _check(h.lowered)
    assert all(st[i] == 0 for i in coll)
    for a, b in zip(coll, coll[1:]):
        assert a in deps_of[b]


@pytest.mark.parametrize("name", ["mlp_A_small", "cnn_C_small", "resnet_D_small", "mlp_E_small"])
def test_io_access_covers_every_input_and_result(name):
    """Host-buffer runs wait for an input's copy only at the launches that
    read it: every launch touching an input slot must be listed, and every
    result's D2H follows its last writer."""
    case = next(c for c in G.load("workloads.json.gz") if c["name"] == name)
    h = host_compile(G.fn_of(case["fn"]), conv_layout="nhwc" if name.startswith("resnet") else "identity")
    low = h.lowered
    off, reads, writer = schedule.io_access(low)
    n, n_in = len(low.launches), low.n_inputs
    assert len(off) == n + 1 and off[-1] == len(reads) and len(writer) == low.n_outputs
    for i, L in enumerate(low.launches):
        mine = set(reads[off[i]:off[i + 1]])
        for k in L.reads:
            b = low.buffers[k]
            root = b.base if b.base is not None else b
            if root.splat is None and abi.SLOT_IO <= root.slot < abi.SLOT_IO + n_in:
                assert root.slot - abi.SLOT_IO in mine
        for k in L.writes:
            b = low.buffers[k]
            root = b.base if b.base is not None else b
            if root.slot >= abi.SLOT_IO + n_in:
                assert writer[root.slot - abi.SLOT_IO - n_in] >= i
    assert set(reads) == set(range(n_in)) - {i for i in range(n_in) if not any(
        (low.buffers[k].base or low.buffers[k]).slot == abi.SLOT_IO + i for L in low.launches for k in L.reads)}
