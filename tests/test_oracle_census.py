"""Pins of the oracle census (Fig. P:269-309) against brute force,
networkx, worked examples, closed forms and 128-bit closing."""
import json
import os

import numpy as np
import pytest

import oracle
import synth
from oracle import pyref

NAMES = oracle.CLASS_NAMES


def vec(d):
    return [int(d.get(k, 0)) for k in NAMES]


def test_single_triad_graphs_are_unit_vectors():
    for i, name in enumerate(NAMES):
        a = synth.single_triad(name)
        c = oracle.census(3, a.src, a.dst)
        assert c == [1 if j == i else 0 for j in range(16)], name
        assert oracle.bruteforce(3, a.src, a.dst) == c


def test_spec_census_examples(golden_dir):
    ex = json.load(open(os.path.join(golden_dir, "spec_examples.json")))
    for e in ex["census"]:
        arcs = np.array(e["arcs"], dtype=np.uint32).reshape(-1, 2)
        g = oracle.Graph(e["n"], arcs[:, 0], arcs[:, 1])
        got = g.census()
        exp = vec(e["expect"])
        for k, v in e["expect"].items():
            assert got[NAMES.index(k)] == v, e["cite"]
        assert sum(got) == oracle.choose3(e["n"])
        if "stats" in e:
            st = g.stats()
            for k, v in e["stats"].items():
                assert st[k] == v, e["cite"]
        del exp
    for e in ex["null_count"]:
        assert oracle.choose3(e["n"]) - e["sum"] == e["result"], e["cite"]
    for e in ex["canonical_dyads"]:
        arcs = np.array(e["arcs"], dtype=np.uint32).reshape(-1, 2)
        assert oracle.Graph(e["n"], arcs[:, 0], arcs[:, 1]).stats()["dyads"] == e["dyads"]


@pytest.mark.parametrize("n", [0, 1, 2, 3])
def test_tiny_orders(n):
    a = synth.random_digraph(n, 0.9, seed=n + 100)
    c = oracle.census(n, a.src, a.dst)
    assert sum(c) == oracle.choose3(n)
    assert c == oracle.bruteforce(n, a.src, a.dst)


def test_bm_equals_bruteforce_random_small():
    # oracle equivalence on many random digraphs, n <= 12,
    # p in {.05,.2,.5,.9}; here 400 graphs n <= 40 plus noise arcs
    for s in range(400):
        n = 3 + s % 38
        p = (0.05, 0.2, 0.5, 0.9)[s % 4]
        a = synth.random_digraph(n, p, seed=s, loops=(s % 3 == 0), dups=s % 5)
        g = oracle.Graph(n, a.src, a.dst)
        assert g.census() == g.bruteforce(), (n, p, s)


@pytest.mark.parametrize("n,p", [(200, 0.05), (200, 0.2), (200, 0.5), (200, 0.9), (120, 0.02)])
def test_bm_equals_bruteforce_n200(n, p):
    a = synth.random_digraph(n, p, seed=n + int(p * 1000))
    g = oracle.Graph(n, a.src, a.dst)
    c = g.census()
    assert c == g.bruteforce()
    assert sum(c) == oracle.choose3(n)


def test_config_C1_against_bruteforce():
    a = synth.make_config("C1")
    g = oracle.Graph(a.n, a.src, a.dst)
    assert g.census() == g.bruteforce()


def test_pure_python_restatement_agrees():
    T = oracle.triad_table()
    for s in range(60):
        n = 3 + s % 14
        a = synth.random_digraph(n, (0.1, 0.3, 0.6)[s % 3], seed=1000 + s, loops=True, dups=2)
        c = oracle.census(n, a.src, a.dst)
        assert pyref.census_bm(n, a.src, a.dst, T) == c
        assert pyref.census_brute(n, a.src, a.dst, T) == c


def test_networkx_triadic_census():
    nx = pytest.importorskip("networkx")
    for s in range(30):
        n = 20 + 4 * s
        a = synth.random_digraph(n, (0.01, 0.05, 0.1, 0.3)[s % 4], seed=2000 + s)
        G = nx.DiGraph()
        G.add_nodes_from(range(n))
        G.add_edges_from(zip(a.src.tolist(), a.dst.tolist()))
        ref = nx.triadic_census(G)
        assert oracle.census(n, a.src, a.dst) == [ref[k] for k in NAMES]


def test_relabelling_invariance():
    a = synth.make_config("C1")
    c = oracle.census(a.n, a.src, a.dst)
    for seed in (1, 2, 3):
        b = synth.relabel(a, seed)
        assert oracle.census(b.n, b.src, b.dst) == c


def C3(n):
    return n * (n - 1) * (n - 2) // 6 if n >= 3 else 0


def C2(n):
    return n * (n - 1) // 2


@pytest.mark.parametrize("k,n", [(5, 6), (40, 100), (700, 2000)])
def test_closed_form_stars(k, n):
    for gen, cls_pair, cls_star in ((synth.out_star, "012", "021D"),
                                    (synth.in_star, "012", "021U"),
                                    (synth.mutual_star, "102", "201")):
        a = gen(k, n)
        exp = {cls_pair: k * (n - k - 1), cls_star: C2(k)}
        exp["003"] = C3(n) - sum(exp.values())
        assert oracle.census(a.n, a.src, a.dst) == vec(exp), gen.__name__


@pytest.mark.parametrize("n", [4, 5, 50, 1000])
def test_closed_form_cycle(n):
    a = synth.directed_cycle(n)
    exp = {"012": n * (n - 4), "021C": n}
    exp["003"] = C3(n) - sum(exp.values())
    assert oracle.census(n, a.src, a.dst) == vec(exp)


@pytest.mark.parametrize("n", [3, 10, 150])
def test_closed_form_tournament_and_clique(n):
    a = synth.transitive_tournament(n)
    assert oracle.census(n, a.src, a.dst) == vec({"030T": C3(n)})
    b = synth.complete_mutual(n)
    assert oracle.census(n, b.src, b.dst) == vec({"300": C3(n)})


@pytest.mark.parametrize("a_,b_", [(4, 300), (30, 30), (1, 50)])
def test_closed_form_bipartite(a_, b_):
    a = synth.complete_bipartite(a_, b_)
    exp = {"021U": b_ * C2(a_), "021D": a_ * C2(b_), "003": C3(a_) + C3(b_)}
    assert oracle.census(a.n, a.src, a.dst) == vec(exp)


def test_choose3_128bit():
    # C(n,3) >= 2^64 for n > 4,801,280 (SURVEY.md reading 8)
    for n in (0, 1, 2, 3, 4, 4_801_279, 4_801_280, 4_801_281, 4_847_571, 67_108_864,
              2**32):
        assert oracle.choose3(n) == C3(n)
    assert C3(4_801_280) < 2**64 <= C3(4_801_281)


def test_null_class_needs_high_word():
    # a big out-star padded with isolated vertices: 003 > 2^64
    n, k = 5_000_000, 3
    a = synth.out_star(k, n)
    c = oracle.census(n, a.src, a.dst)
    assert c[0] >= 2**64
    assert c == vec({"012": k * (n - k - 1), "021D": C2(k), "003": C3(n) - k * (n - k - 1) - C2(k)})


def test_sanitising_and_range_errors():
    g = oracle.Graph(3, [0, 0, 2, 1], [1, 1, 2, 0])
    st = g.stats()
    assert (st["m"], st["dups_dropped"], st["loops_dropped"], st["mutual_dyads"]) == (2, 1, 1, 1)
    with pytest.raises(oracle.OracleError):
        oracle.Graph(3, [0, 3], [1, 0])


def test_dyad_range_partials_sum_to_full():
    for s, (n, p) in enumerate([(60, 0.1), (200, 0.05), (30, 0.7)]):
        a = synth.random_digraph(n, p, seed=3000 + s)
        g = oracle.Graph(n, a.src, a.dst)
        full = g.census()
        D = g.stats()["dyads"]
        rng = np.random.default_rng(s)
        cuts = sorted(set([0, D] + rng.integers(0, D + 1, size=5).tolist()))
        tot = [0] * 16
        for b, e in zip(cuts[:-1], cuts[1:]):
            part = g.census_range(b, e)
            assert part[0] == 0
            tot = [x + y for x, y in zip(tot, part)]
        assert tot[1:] == full[1:]
        assert oracle.choose3(n) - sum(tot) == full[0]


def test_dyad_range_partials_vs_brute_force_attribution():
    # og_census_range range by range (all 16 entries) against triples
    # enumerated by brute force and attributed to their counting dyad
    # (pyref.census_range_brute: the lexicographically smallest adjacent pair)
    T = oracle.triad_table()
    for s in range(24):
        n = 6 + s % 11
        a = synth.random_digraph(n, (0.15, 0.35, 0.7)[s % 3], seed=5000 + s, loops=True, dups=2)
        g = oracle.Graph(n, a.src, a.dst)
        D = g.stats()["dyads"]
        assert len(pyref.canonical_dyads(n, a.src, a.dst)) == D
        rng = np.random.default_rng(s)
        cuts = sorted(set([0, D] + rng.integers(0, D + 1, size=4).tolist()))
        for b, e in zip(cuts[:-1], cuts[1:]):
            assert g.census_range(b, e) == pyref.census_range_brute(n, a.src, a.dst, T, b, e), \
                (s, b, e)
        for k in range(D):              # every single dyad
            assert g.census_range(k, k + 1) == pyref.census_range_brute(n, a.src, a.dst, T, k,
                                                                        k + 1), (s, k)


def test_golden_files_are_complete(golden_dir):
    for name in ("C1", "C2", "C3"):
        p = os.path.join(golden_dir, "census_%s.json" % name)
        if not os.path.exists(p):
            pytest.skip("golden %s not generated" % name)
        rec = json.load(open(p))
        c = [int(x) for x in rec["census"]]
        assert sum(c) == C3(rec["n"])
