"""f1: the oracle's 64-type census (P:258, P:327,
P:343) in the B-M labelling, pinned by an independent O(n^3) brute force that
assigns each triple its B-M code from the canonicity rule, and by the
64 -> 16 fold through the published TriadTable."""
import json
import os

import pytest

import oracle
import synth


def fold(c64, T):
    out = [0] * 16
    for code, v in enumerate(c64):
        out[T[code] - 1] += v
    return out


def test_census64_equals_bm_order_bruteforce():
    for s in range(150):
        n = 3 + s % 35
        a = synth.random_digraph(n, (0.05, 0.2, 0.5, 0.9)[s % 4], seed=500 + s, loops=True,
                                 dups=s % 3)
        g = oracle.Graph(n, a.src, a.dst)
        assert g.census64() == g.bruteforce64(), s


def test_census64_folds_to_census(golden_dir):
    T = json.load(open(os.path.join(golden_dir, "tricodes.json")))["tricodes"]
    for s in range(40):
        a = synth.random_digraph(60, (0.02, 0.1, 0.4)[s % 3], seed=900 + s)
        g = oracle.Graph(a.n, a.src, a.dst)
        assert fold(g.census64(), T) == g.census()
    a = synth.make_config("C1")
    g = oracle.Graph(a.n, a.src, a.dst)
    assert fold(g.census64(), T) == g.census()


def test_census64_structure():
    # a counting dyad is connected, so codes with pre = 0 other than 0 are
    # empty; the single-triad graphs land on exactly one code each
    a = synth.random_digraph(80, 0.2, seed=3)
    c = oracle.Graph(a.n, a.src, a.dst).census64()
    assert all(c[code] == 0 for code in range(1, 64) if code & 3 == 0)
    assert sum(c) == oracle.choose3(a.n)
    for name in oracle.CLASS_NAMES:
        t = synth.single_triad(name)
        c = oracle.Graph(3, t.src, t.dst).census64()
        assert sum(c) == 1
