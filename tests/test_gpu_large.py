"""-m gpu, large configs, bit-exact against the oracle.

C4 (LiveJournal-shaped, n = 4,847,571 > 4,801,280 so class 003 needs the
high word): the full GPU census equals tests/golden/census_C4.json (the
oracle over equal-cost canonical-dyad ranges in forked host processes,
tests/golden/make_golden_sharded.py), and every one of the golden's range
partials equals tc_census_range on the same range; the golden itself is
pinned by the linear census identities with the triangle rows on
(triangles from tests/native/tri_count.c, independent of both censuses).

C5 (R-MAT scale 26, 1.07e9 drawn arcs, drawn on the GPU by synth/device.py):
the full census satisfies the six O(n+m) identities computed with plain
torch ops from the arcs, and the oracle is run on spot ranges -- the
costliest hub dyads and random ranges -- over the sub-digraph of all arcs
incident to an endpoint of a dyad in the range.  That sub-digraph holds
N(u), N(v) and every arc the B-M loop body probes for those dyads
(IsEdge/IsNeighbour of u-w and v-w pairs), so the oracle's
partial over the same dyads (located by their canonical keys) is the
paper's value for the range (Fig. P:269-309 restricted to the range).
"""
import json
import os

import numpy as np
import pytest

import oracle
import synth
from test_oracle_identities import check_identities, graph_quantities

pytestmark = pytest.mark.gpu


def _tcb():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1603_02655_b200 as tcb
    return tcb


@pytest.fixture(scope="module")
def c4():
    tcb = _tcb()
    a = synth.make_config("C4")
    g = tcb.tc_graph_create(a.n, a.src, a.dst)
    yield tcb, a, g
    g.close()


@pytest.fixture(scope="module")
def c4_golden(golden_dir):
    return json.load(open(os.path.join(golden_dir, "census_C4.json")))


def test_c4_full_census_vs_golden(c4, c4_golden):
    tcb, a, g = c4
    assert a.n == c4_golden["n"] and a.m == c4_golden["m_drawn"]
    c = g.census()
    assert c == [int(x) for x in c4_golden["census"]]
    assert c[0] >= 2**64                      # 003 high word exercised
    assert g.stats() == c4_golden["stats"]


def test_c4_golden_identities_with_triangles(c4, c4_golden):
    from native import triangles
    _, a, _ = c4
    q = graph_quantities(a.n, a.src, a.dst, triangles=False)
    q["tri"] = triangles(a.n, a.src, a.dst)
    check_identities([int(x) for x in c4_golden["census"]], q)


def test_c4_every_golden_range(c4, c4_golden):
    # all 16 entries of every oracle range partial, range by range
    tcb, _, g = c4
    parts = c4_golden["range_partials"]
    assert parts[0]["begin"] == 0 and parts[-1]["end"] == g.stats()["dyads"]
    for p in parts:
        got = tcb.tc_census_range(g, p["begin"], p["end"])
        assert got == [int(x) for x in p["partial"]], (p["begin"], p["end"])


def test_c4_costliest_dyads_vs_oracle(c4):
    tcb, a, g = c4
    og = oracle.Graph(a.n, a.src, a.dst)
    D = og.stats()["dyads"]
    cost = og.dyad_costs()
    hub = int(np.argmax(cost))               # the costliest dyad (warp items, skewed pairs)
    for b, e in [(max(0, hub - 3), hub + 3), (hub, hub + 1)]:
        assert tcb.tc_census_range(g, b, e) == og.census_range(b, e), (b, e)


# ---------------------------------------------------------------------------
# C5: device-drawn arcs, identities from torch ops, oracle spot ranges
# ---------------------------------------------------------------------------
def torch_quantities(n, s, d):
    """O(n+m) identity inputs (test_oracle_identities.graph_quantities) with
    plain torch ops; also the canonical dyad keys min*n+max in canonical
    order and the undirected degrees."""
    import torch
    s = s.long()
    d = d.long()
    keep = s != d
    key = torch.unique(s[keep] * n + d[keep])
    s, d = key // n, key % n
    rk = d * n + s
    pos = torch.searchsorted(key, rk).clamp(max=key.numel() - 1)
    rev = key[pos] == rk
    mut_arcs = int(rev.sum())
    out = torch.bincount(s, minlength=n)
    inn = torch.bincount(d, minlength=n)
    mutb = torch.bincount(s[rev], minlength=n)
    del rk, pos
    und = torch.unique(torch.minimum(s, d) * n + torch.maximum(s, d))
    del s, d, key
    deg = torch.bincount(und // n, minlength=n) + torch.bincount(und % n, minlength=n)
    q = dict(n=n, M=mut_arcs // 2, A=int(out.sum()) - mut_arcs, D=int(und.numel()),
             paths=int((out * inn - mutb).sum()), os=int((out * (out - 1) // 2).sum()),
             is_=int((inn * (inn - 1) // 2).sum()), sumd2=int((deg * deg).sum()),
             sumdc2=int((deg * (deg - 1) // 2).sum()))
    return q, und, deg


def spot_range_oracle(n, s, d, und, b, e):
    """Oracle partial of canonical dyads [b, e) (keys und[b:e]) over the arcs
    incident to their endpoints (see the module docstring)."""
    import torch
    keys = und[b:e]
    ends = torch.unique(torch.cat([keys // n, keys % n]))
    mark = torch.zeros(n, dtype=torch.bool, device=s.device)
    mark[ends] = True
    sel = mark[s.long()] | mark[d.long()]
    ss = s[sel].cpu().numpy().view(np.uint32)
    dd = d[sel].cpu().numpy().view(np.uint32)
    og = oracle.Graph(n, ss, dd)
    lo, hi = np.minimum(ss, dd).astype(np.int64), np.maximum(ss, dd).astype(np.int64)
    sub = np.unique((lo * n + hi)[ss != dd])        # the sub-digraph's canonical dyads
    kk = keys.cpu().numpy()
    b2 = int(np.searchsorted(sub, kk[0]))
    assert np.array_equal(sub[b2:b2 + (e - b)], kk)  # the same dyads, contiguous
    return og.census_range(b2, b2 + (e - b))


def test_c5_identities_and_oracle_spot_ranges():
    tcb = _tcb()
    import torch
    from synth.device import make_device_config
    n, s, d, meta = make_device_config("C5", torch.device("cuda", 0))
    g = tcb.tc_graph_create(n, s, d)
    try:
        st = g.stats()
        c = g.census()
        q, und, deg = torch_quantities(n, s, d)
        assert st["dyads"] == q["D"] and st["sum_deg_sq"] == q["sumd2"]
        assert st["max_degree"] == int(deg.max())
        check_identities(c, q)
        D = q["D"]
        cost = deg[und // n] + deg[und % n]
        hub = int(torch.argmax(cost))
        hub_u = int(und[hub] // n)
        first_of_hub = int(torch.searchsorted(und, torch.tensor([hub_u * n], device=und.device)))
        del cost
        rng = np.random.default_rng(26)
        ranges = [(max(0, hub - 8), min(D, hub + 8)), (first_of_hub, min(D, first_of_hub + 16))]
        ranges += [(int(x), int(x) + 2000) for x in rng.integers(0, D - 2000, size=4)]
        ranges += [(D - 500, D)]
        for b, e in ranges:
            got = tcb.tc_census_range(g, b, e)
            assert got == spot_range_oracle(n, s, d, und, b, e), (b, e)
    finally:
        g.close()
