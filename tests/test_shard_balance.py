"""Multi-GPU shard cut (include/triadcensus.h
tc_shard_bounds): the census kernels' own per-dyad work -- t merge trips,
or the skewed-pair search units on hub graphs (tests/shard_work.py, a numpy
restatement from the arc list) -- plus kappa = 8 per dyad is cut into equal
contiguous ranges by the library's host cut rule, the rule the device
applies (the -m gpu tests check that the device cut equals this one).
Balance is measured in the kernels' work, the quantity that sets each
rank's census time.  No GPU needed."""
import numpy as np
import pytest

import paper_1603_02655_b200 as tcb
import synth
from shard_work import dyad_work, neighbour_crs, rank_work

KAPPA = 8


def _imbalance(bounds, work):
    r = rank_work(bounds, work)
    return max(r) / (sum(r) / len(r))


@pytest.mark.parametrize("name", ["C2", "C3"])
def test_work_balanced_cut(name):
    a = synth.make_config(name)
    t, cost = dyad_work(a.n, a.src, a.dst)
    work = cost + KAPPA
    off, col, key = neighbour_crs(a.n, a.src, a.dst)
    row = key // a.n
    canon = row < col
    deg = np.diff(off)
    uniform = deg[row[canon]] + deg[col[canon]]          # |N(u)| + |N(v)|
    for world in (2, 4, 8):
        b = tcb.tc_shard_bounds_host(cost, world, kappa=KAPPA)
        assert b[0] == 0 and b[-1] == t.size and b == sorted(b)
        assert _imbalance(b, work) <= 1.05, (name, world)
        # the paper's uniform estimate (round-1 cut) balances the wrong thing
        bu = tcb.tc_shard_bounds_host(uniform, world, kappa=KAPPA)
        if name == "C3":
            assert _imbalance(bu, work) > 1.15, (name, world)


def test_cut_rule_small_exact():
    # bounds[r] = first k whose exclusive prefix of cost + kappa >= floor(T r / world)
    cost = np.array([5, 0, 0, 9, 1, 1, 30, 2], np.uint64)
    for world in (1, 2, 3, 5):
        b = tcb.tc_shard_bounds_host(cost, world, kappa=2)
        pre = np.concatenate([[0], np.cumsum(cost + 2)])
        T = int(pre[-1])
        for r in range(1, world):
            want = int(np.searchsorted(pre, T * r // world, side="left"))
            assert b[r] == min(want, cost.size), (world, r)


def test_world_limits():
    with pytest.raises(tcb.TCError, match="TC_E_INVALID"):
        tcb.tc_shard_bounds_host(np.ones(4, np.uint64), 1025)
    with pytest.raises(tcb.TCError, match="TC_E_INVALID"):
        tcb.tc_shard_bounds_host(np.ones(4, np.uint64), 0)
