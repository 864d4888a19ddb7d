"""Linear census identities ("What pins each part"):
O(n+m) (and triangle) quantities computed straight from the arc list with
numpy/scipy, independent of both census implementations, that any correct
16-class census must satisfy.  Used to pin the full-size oracle results
stored under tests/golden/ (written by tests/golden/make_golden.py)."""
import json
import os
from math import comb

import numpy as np
import pytest

import oracle
import synth

NAMES = oracle.CLASS_NAMES


def _class_constants():
    """Per-class structural counts from the Holland-Leinhardt representatives."""
    rows = {}
    for name in NAMES:
        E = set(synth.REPRESENTATIVES[name])
        pairs = [(0, 1), (0, 2), (1, 2)]
        M = sum(1 for a, b in pairs if (a, b) in E and (b, a) in E)
        A = sum(1 for a, b in pairs if ((a, b) in E) != ((b, a) in E))
        P = sum(1 for i in range(3) for b in range(3) for j in range(3)
                if len({i, b, j}) == 3 and (i, b) in E and (b, j) in E)
        out = [sum(1 for x in range(3) if (b, x) in E) for b in range(3)]
        inn = [sum(1 for x in range(3) if (x, b) in E) for b in range(3)]
        OS = sum(comb(o, 2) for o in out)
        IS = sum(comb(i, 2) for i in inn)
        rows[name] = dict(M=M, A=A, P=P, OS=OS, IS=IS, conn=M + A)
    return rows


def _uniq(x):
    x = np.sort(x)
    return x[np.concatenate([[True], x[1:] != x[:-1]])] if x.size else x


def graph_quantities(n, src, dst, triangles=True):
    src = np.asarray(src, np.int64)
    dst = np.asarray(dst, np.int64)
    keep = src != dst
    key = _uniq(src[keep] * n + dst[keep])
    s, d = key // n, key % n
    rk = d * n + s
    pos = np.minimum(np.searchsorted(key, rk), max(key.size - 1, 0))
    rev = (key[pos] == rk) if key.size else np.zeros(0, bool)
    mut_arcs = int(rev.sum())           # arcs whose reverse exists
    M = mut_arcs // 2
    A = int(key.size) - mut_arcs
    out = np.bincount(s, minlength=n).astype(np.int64)
    inn = np.bincount(d, minlength=n).astype(np.int64)
    mutb = np.bincount(s[rev], minlength=n).astype(np.int64)
    und = _uniq(np.minimum(s, d) * n + np.maximum(s, d))
    us, ud = und // n, und % n
    deg = (np.bincount(us, minlength=n) + np.bincount(ud, minlength=n)).astype(np.int64)
    q = dict(n=n, M=M, A=A, D=int(und.size),
             paths=int((out * inn - mutb).sum()),
             os=int((out * (out - 1) // 2).sum()),
             is_=int((inn * (inn - 1) // 2).sum()),
             sumd2=int((deg * deg).sum()),
             sumdc2=int((deg * (deg - 1) // 2).sum()))
    if triangles:
        import scipy.sparse as sp
        Au = sp.coo_matrix((np.ones(und.size, np.int64), (us, ud)), shape=(n, n)).tocsr()
        Af = (Au + Au.T).tocsr()
        # T = sum_{u<v adjacent} |N(u) ∩ N(v)| / 3
        q["tri"] = int((Au.multiply(Af @ Af)).sum()) // 3
    return q


def check_identities(c, q):
    K = _class_constants()
    n = q["n"]
    cs = dict(zip(NAMES, c))
    assert sum(c) == comb(n, 3)
    assert sum(cs[k] * K[k]["M"] for k in NAMES) == q["M"] * (n - 2)
    assert sum(cs[k] * K[k]["A"] for k in NAMES) == q["A"] * (n - 2)
    assert sum(cs[k] * K[k]["P"] for k in NAMES) == q["paths"]
    assert sum(cs[k] * K[k]["OS"] for k in NAMES) == q["os"]
    assert sum(cs[k] * K[k]["IS"] for k in NAMES) == q["is_"]
    if "tri" in q:
        T = q["tri"]
        assert sum(cs[k] for k in NAMES if K[k]["conn"] == 3) == T
        assert sum(cs[k] for k in NAMES if K[k]["conn"] == 2) == q["sumdc2"] - 3 * T
        assert cs["012"] + cs["102"] == q["D"] * n - q["sumd2"] + 3 * T


def test_identity_rows_have_rank_8():
    K = _class_constants()
    rows = [[1] * 16] + [[K[k][f] for k in NAMES] for f in ("M", "A", "P", "OS", "IS")]
    rows += [[1 if K[k]["conn"] == 3 else 0 for k in NAMES],
             [1 if K[k]["conn"] == 2 else 0 for k in NAMES],
             [1 if k in ("012", "102") else 0 for k in NAMES]]
    assert np.linalg.matrix_rank(np.array(rows[:6], float)) == 6
    assert np.linalg.matrix_rank(np.array(rows, float)) == 8


def test_identities_random_graphs():
    for s in range(30):
        n = 10 + 13 * s
        a = synth.random_digraph(n, (0.02, 0.1, 0.4)[s % 3], seed=4000 + s, loops=True, dups=3)
        check_identities(oracle.census(n, a.src, a.dst), graph_quantities(n, a.src, a.dst))


def test_identity_catches_a_dropped_term():
    # sanity of the pin itself: moving one count between classes breaks it
    a = synth.make_config("C1")
    c = oracle.census(a.n, a.src, a.dst)
    q = graph_quantities(a.n, a.src, a.dst)
    check_identities(c, q)
    for i, j in ((3, 4), (8, 9), (1, 2), (5, 6)):
        bad = list(c)
        bad[i] -= 1
        bad[j] += 1
        with pytest.raises(AssertionError):
            check_identities(bad, q)


@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_identities_on_golden_configs(name, golden_dir):
    p = os.path.join(golden_dir, "census_%s.json" % name)
    if not os.path.exists(p):
        pytest.skip("golden file missing; run tests/golden/make_golden.py")
    rec = json.load(open(p))
    a = synth.make_config(name)
    assert a.n == rec["n"] and a.m == rec["m_drawn"]
    c = [int(x) for x in rec["census"]]
    q = graph_quantities(a.n, a.src, a.dst, triangles=(name != "C3"))
    if name == "C3":                      # scipy's A @ A is too big here
        from native import triangles
        q["tri"] = triangles(a.n, a.src, a.dst)
    check_identities(c, q)
    assert q["sumd2"] == rec["stats"]["sum_deg_sq"]
    assert q["D"] == rec["stats"]["dyads"]
