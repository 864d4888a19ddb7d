"""the multithreaded version's task queues.

CPU: the oracle's literal queue generation (oracle/bm_oracle.c
og_task_queues) pinned by closed forms and by an independent restatement of
the weights from Python sets:
  * aggregate NsetSize: uniform  sum(|N[u]|+|N[v]|-2) = sum d^2 - 2D (the
    two columns of Table P:1842-1855 differ by exactly 2D); non-uniform
    sum |S| = sum d^2 - 2D - 3T (every triangle puts one element into the
    intersection of each of its three dyads);
  * out-star closed form: every dyad weighs k - 1 under both strategies, so
    queues hold floor(M / (k-1)) + 1 dyads;
  * each closed queue is cut at the FIRST dyad whose running NsetSize
    exceeds MaxNsetSize (lines 10-13), the weights recomputed from sets;
  * the "nearly proportional" queue count: (W - wmax)/(M + wmax)
    <= closed queues <= W / M.
GPU: tc_task_queues equals the oracle bit for bit (starts and totals) for
both strategies, and censuses over the queues sum to the full census.
"""
from math import comb

import numpy as np
import pytest

import oracle
import synth
from test_oracle_identities import graph_quantities


def _sets(a):
    N = [set() for _ in range(a.n)]
    for s, d in zip(a.src.tolist(), a.dst.tolist()):
        if s != d:
            N[s].add(d)
            N[d].add(s)
    return N


def _weights(a, strategy):
    """per canonical dyad, canonical order, from Python sets (independent)"""
    N = _sets(a)
    w = []
    for u in range(a.n):
        for v in sorted(N[u]):
            if u < v:
                if strategy == "uniform":
                    w.append(len(N[u]) + len(N[v]) - 2)
                else:
                    w.append(len((N[u] | N[v]) - {u, v}))
    return np.array(w, np.int64)


GRAPHS = [lambda: synth.make_config("C1"),
          lambda: synth.random_digraph(60, 0.15, seed=3, loops=True, dups=5),
          lambda: synth.random_digraph(200, 0.05, seed=4),
          lambda: synth.complete_mutual(12),
          lambda: synth.rmat(9, 8, seed=5)]


@pytest.mark.parametrize("gi", range(len(GRAPHS)))
def test_oracle_queue_totals_closed_form(gi):
    a = GRAPHS[gi]()
    q = graph_quantities(a.n, a.src, a.dst)
    g = oracle.Graph(a.n, a.src, a.dst)
    _, tu = g.task_queues("uniform", 10**18)
    _, tn = g.task_queues("nonuniform", 10**18)
    assert tu == q["sumd2"] - 2 * q["D"]
    assert tn == q["sumd2"] - 2 * q["D"] - 3 * q["tri"]


@pytest.mark.parametrize("strategy", ["uniform", "nonuniform"])
@pytest.mark.parametrize("k,M", [(10, 0), (10, 8), (10, 9), (10, 100), (50, 1000), (7, 10**9)])
def test_oracle_queues_out_star(strategy, k, M):
    a = synth.out_star(k, k + 5)
    starts, tot = oracle.Graph(a.n, a.src, a.dst).task_queues(strategy, M)
    assert tot == k * (k - 1)
    L = M // (k - 1) + 1                     # dyads per closed queue
    assert starts.tolist() == list(range(0, k, L))


@pytest.mark.parametrize("strategy", ["uniform", "nonuniform"])
@pytest.mark.parametrize("gi", [0, 1, 2, 4])
def test_oracle_queues_cut_at_first_crossing(strategy, gi):
    a = GRAPHS[gi]()
    w = _weights(a, strategy)
    g = oracle.Graph(a.n, a.src, a.dst)
    for M in (0, int(w.max()), int(w.sum() // 37), int(w.sum() // 3), int(w.sum())):
        starts, tot = g.task_queues(strategy, M)
        assert tot == int(w.sum())
        b = starts.tolist() + [w.size]
        assert b[0] == 0 and all(x < y for x, y in zip(b, b[1:]))
        for q in range(len(b) - 1):
            part = np.cumsum(w[b[q]:b[q + 1]])
            assert (part[:-1] <= M).all()            # no earlier dyad crossed
            if q < len(b) - 2:
                assert part[-1] > M                  # closed by its last dyad


@pytest.mark.parametrize("strategy", ["uniform", "nonuniform"])
def test_oracle_queue_count_nearly_proportional(strategy):
    """changing MaxNsetSize from M1 to M2 changes the number of
    queues by ~M1/M2 -- bounded here by the cut rule itself."""
    a = synth.rmat(12, 8, seed=6)
    g = oracle.Graph(a.n, a.src, a.dst)
    w = _weights(a, strategy)
    W, wmax = int(w.sum()), int(w.max())
    counts = {}
    for M in (W // 400, W // 200, W // 100, W // 50):
        starts, _ = g.task_queues(strategy, M)
        closed = len(starts) - 1 + (1 if np.cumsum(w[int(starts[-1]):])[-1] > M else 0)
        assert (W - wmax * 1.0) / (M + wmax) - 1 <= closed <= W / M
        counts[M] = len(starts)
    Ms = sorted(counts)
    for m1, m2 in zip(Ms, Ms[1:]):
        ratio = counts[m1] / counts[m2]
        assert 1.6 < ratio < 2.4, (m1, m2, counts)


def test_oracle_queues_empty_graph():
    starts, tot = oracle.Graph(10, np.zeros(0, np.uint32), np.zeros(0, np.uint32)).task_queues(
        "uniform", 5)
    assert starts.size == 0 and tot == 0


# ---------------------------------------------------------------------------
# GPU: tc_task_queues vs the oracle
# ---------------------------------------------------------------------------
@pytest.fixture(scope="module")
def tcb():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1603_02655_b200 as m
    return m


GPU_GRAPHS = GRAPHS + [lambda: synth.make_config("C2"), lambda: synth.out_star(300, 400),
                       lambda: synth.livejournal_like(n=20000, m_target=150000, scale=15, seed=2)]


@pytest.mark.gpu
@pytest.mark.parametrize("gi", range(len(GPU_GRAPHS)))
@pytest.mark.parametrize("strategy", ["uniform", "nonuniform"])
def test_gpu_task_queues_match_oracle(tcb, gi, strategy):
    a = GPU_GRAPHS[gi]()
    og = oracle.Graph(a.n, a.src, a.dst)
    g = tcb.tc_graph_create(a.n, a.src, a.dst)
    try:
        _, W = og.task_queues(strategy, 10**18)
        for M in (0, 1, W // 1000 + 1, W // 64, W // 7, W, 10**18):
            exp_s, exp_t = og.task_queues(strategy, M)
            got_s, got_t = tcb.tc_task_queues(g, strategy, M)
            assert got_t == exp_t
            assert np.array_equal(got_s, exp_s), (M, got_s[:8], exp_s[:8])
    finally:
        g.close()


@pytest.mark.gpu
def test_gpu_census_over_task_queues(tcb):
    a = synth.make_config("C2")
    g = tcb.tc_graph_create(a.n, a.src, a.dst)
    try:
        full = g.census()
        D = g.stats()["dyads"]
        starts, W = tcb.tc_task_queues(g, "nonuniform", 0)
        starts, _ = tcb.tc_task_queues(g, "nonuniform", W // 97)
        b = starts.tolist() + [D]
        acc = [0] * 16
        for q in range(len(b) - 1):
            p = tcb.tc_census_range(g, b[q], b[q + 1])
            acc = [x + y for x, y in zip(acc, p)]
        assert acc[1:] == full[1:]
        assert sum(full) == comb(a.n, 3)
    finally:
        g.close()


@pytest.mark.gpu
def test_gpu_task_queues_empty_and_errors(tcb):
    g = tcb.tc_graph_create(10, np.zeros(0, np.uint32), np.zeros(0, np.uint32))
    try:
        s, t = tcb.tc_task_queues(g, "uniform", 3)
        assert s.size == 0 and t == 0
        with pytest.raises(KeyError):
            tcb.tc_task_queues(g, "chin", 3)
    finally:
        g.close()
