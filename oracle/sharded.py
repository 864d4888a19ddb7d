"""oracle/sharded.py -- TEST INFRASTRUCTURE ONLY (tests/, bench.py's
cpu_baseline and --impl reference legs).

The oracle's census over canonical-dyad ranges in forked host processes:
[0, D) is cut into contiguous ranges of about equal sum(|N[u]| + |N[v]| +
kappa) (the paper's uniform work unit) and each range is one
single-threaded ``og_census_range`` call (Fig. P:269-309 restricted to the
range).  Partials over a partition of the dyads sum to the full census
(S:433); class 003 is C(n,3) - sum.  No arithmetic of the
method lives here -- only the split and the sum.
"""
from __future__ import annotations

import multiprocessing as mp
import time

import numpy as np

from . import Graph, choose3

KAPPA = 8
_G = None          # the graph, built in the parent, shared with the workers by fork


def equal_cost_ranges(cost: np.ndarray, chunks: int, kappa: int = KAPPA):
    """`chunks` contiguous ranges of [0, D) with about equal sum(cost + kappa)."""
    D = int(cost.size)
    if D == 0:
        return []
    pre = np.cumsum(cost.astype(np.uint64) + np.uint64(kappa))
    tot = int(pre[-1])
    cuts = [0] + [int(np.searchsorted(pre, tot * r // chunks, side="right"))
                  for r in range(1, chunks)] + [D]
    cuts = sorted(set(cuts))
    return [(cuts[i], cuts[i + 1]) for i in range(len(cuts) - 1) if cuts[i + 1] > cuts[i]]


def _work(rng):
    b, e = rng
    t0 = time.perf_counter()
    part = _G.census_range(b, e)
    return b, e, part, time.perf_counter() - t0


def census_ranges(g: Graph, ranges, procs: int, on_result=None):
    """Runs og_census_range on every range in `procs` forked processes (or in
    this process if procs == 1).  Returns ({(b, e): partial}, wall seconds,
    sum of per-range seconds)."""
    global _G
    _G = g
    out, cpu = {}, 0.0
    t0 = time.perf_counter()
    if procs <= 1:
        it = map(_work, ranges)
        pool = None
    else:
        pool = mp.get_context("fork").Pool(procs)
        it = pool.imap_unordered(_work, ranges)
    try:
        for b, e, part, sec in it:
            out[(b, e)] = part
            cpu += sec
            if on_result:
                on_result(b, e, part, sec)
    finally:
        if pool is not None:
            pool.close()
            pool.join()
    return out, time.perf_counter() - t0, cpu


def close(n: int, partials) -> list[int]:
    """Sum range partials (classes 2..16) and close 003 = C(n,3) - sum."""
    tot = [0] * 16
    for p in partials:
        assert p[0] == 0
        tot = [x + int(y) for x, y in zip(tot, p)]
    tot[0] = choose3(n) - sum(tot[1:])
    return tot
