"""-m gpu: the CUDA path (through the C ABI) against the CPU oracle, element
by element, bit-exact (integer counts, zero tolerance -- BASELINE.json
north_star)."""
import json
import os

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

NAMES = oracle.CLASS_NAMES


@pytest.fixture(scope="module")
def tcb():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1603_02655_b200 as m
    return m


def gpu_census(tcb, a):
    g = tcb.tc_graph_create(a.n, a.src, a.dst)
    try:
        return g.census(), g.stats()
    finally:
        g.close()


def vec(d):
    return [int(d.get(k, 0)) for k in NAMES]


def C3(n):
    return n * (n - 1) * (n - 2) // 6 if n >= 3 else 0


def test_single_triads(tcb):
    for i, name in enumerate(NAMES):
        a = synth.single_triad(name)
        c, _ = gpu_census(tcb, a)
        assert c == [1 if j == i else 0 for j in range(16)], name


def test_spec_examples(tcb, golden_dir):
    ex = json.load(open(os.path.join(golden_dir, "spec_examples.json")))
    for e in ex["census"]:
        arcs = np.array(e["arcs"], dtype=np.uint32).reshape(-1, 2)
        a = synth.Arcs(e["n"], arcs[:, 0].copy(), arcs[:, 1].copy())
        c, st = gpu_census(tcb, a)
        for k, v in e["expect"].items():
            assert c[NAMES.index(k)] == v, e["cite"]
        for k, v in e.get("stats", {}).items():
            assert st[k] == v, e["cite"]


@pytest.mark.parametrize("n", [0, 1, 2, 3])
def test_tiny_orders(tcb, n):
    a = synth.random_digraph(n, 0.9, seed=n, loops=True)
    c, _ = gpu_census(tcb, a)
    assert c == oracle.census(n, a.src, a.dst)


def test_empty_and_loop_only(tcb):
    a = synth.Arcs(10, np.zeros(0, np.uint32), np.zeros(0, np.uint32))
    assert gpu_census(tcb, a)[0] == vec({"003": 120})
    b = synth.Arcs(10, np.arange(10, dtype=np.uint32), np.arange(10, dtype=np.uint32))
    c, st = gpu_census(tcb, b)
    assert c == vec({"003": 120}) and st["loops_dropped"] == 10 and st["m"] == 0


def test_random_graphs_vs_oracle(tcb):
    rng = np.random.default_rng(0)
    for s in range(120):
        n = int(rng.integers(3, 400))
        p = float(rng.choice([0.005, 0.02, 0.1, 0.4, 0.9]))
        a = synth.random_digraph(n, p, seed=10_000 + s, loops=bool(s % 2), dups=s % 7)
        c, st = gpu_census(tcb, a)
        g = oracle.Graph(n, a.src, a.dst)
        assert c == g.census(), (n, p, s)
        assert st == g.stats(), (n, p, s)


def test_C1_vs_bruteforce(tcb):
    a = synth.make_config("C1")
    c, _ = gpu_census(tcb, a)
    assert c == oracle.bruteforce(a.n, a.src, a.dst)


@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_full_config_vs_golden(tcb, golden_dir, name):
    rec = json.load(open(os.path.join(golden_dir, "census_%s.json" % name)))
    a = synth.make_config(name)
    c, st = gpu_census(tcb, a)
    assert c == [int(x) for x in rec["census"]]
    assert st == rec["stats"]


def test_dyad_range_small(tcb):
    # T6: every class of a dyad range, exact, on small random digraphs,
    # including every single-dyad range of the first graphs
    for seed in range(6):
        a = synth.random_digraph(60 + 20 * seed, 0.08 + 0.02 * seed, seed=100 + seed)
        og = oracle.Graph(a.n, a.src, a.dst)
        D = og.stats()["dyads"]
        g = tcb.tc_graph_create(a.n, a.src, a.dst)
        rng = np.random.default_rng(seed)
        bounds = sorted({0, D, *[int(x) for x in rng.integers(0, D, size=5)]})
        tot = [0] * 16
        for b, e in zip(bounds[:-1], bounds[1:]):
            part = tcb.tc_census_range(g, b, e)
            assert part == og.census_range(b, e), (seed, b, e)
            tot = [x + y for x, y in zip(tot, part)]
        assert tcb.tc_close_census(a.n, tot) == og.census()
        if seed < 2:
            for k in range(D):
                assert tcb.tc_census_range(g, k, k + 1) == og.census_range(k, k + 1), (seed, k)
        g.close()


@pytest.mark.parametrize("name", ["C2", "C3"])
def test_dyad_range_parity(tcb, name):
    # T6: random canonical-dyad ranges, all 16 entries equal the oracle's
    # partial (Fig. P:269-309 restricted to the range)
    a = synth.make_config(name)
    og = oracle.Graph(a.n, a.src, a.dst)
    D = og.stats()["dyads"]
    g = tcb.tc_graph_create(a.n, a.src, a.dst)
    rng = np.random.default_rng(1)
    cuts = [0]
    for _ in range(4):
        b = int(rng.integers(cuts[-1], D))
        e = min(D, b + int(rng.integers(1, 20_000)))
        assert tcb.tc_census_range(g, b, e) == og.census_range(b, e), (b, e)
        cuts += [b, e]
    for k in rng.integers(0, D, size=20).tolist():   # single dyads
        assert tcb.tc_census_range(g, k, k + 1) == og.census_range(k, k + 1), k
    assert tcb.tc_census_range(g, D - 3, D + 100) == og.census_range(D - 3, D)
    assert tcb.tc_census_range(g, 5, 5) == [0] * 16
    cuts = sorted(set(cuts + [D]))
    tot = [0] * 16
    for b, e in zip(cuts[:-1], cuts[1:]):
        tot = [x + y for x, y in zip(tot, tcb.tc_census_range(g, b, e))]
    assert tcb.tc_close_census(a.n, tot) == og.census()
    g.close()


@pytest.mark.parametrize("name", ["C2", "hub"])
def test_partials_sum_and_shard_bounds(tcb, name):
    # the device shard cut (cached per world) equals the host cut rule over
    # the kernels' work restated in numpy (tests/shard_work.py); the rank
    # partials sum to the full census
    from shard_work import dyad_work
    if name == "hub":
        n, s, d = _hub_graph(3)
        a = synth.Arcs(n, s, d)
    else:
        a = synth.make_config(name)
    g = tcb.tc_graph_create(a.n, a.src, a.dst)
    full = g.census()
    _, cost = dyad_work(a.n, a.src, a.dst)
    for world in (1, 2, 3, 8):
        b = tcb.tc_shard_bounds(g, world)
        assert b == tcb.tc_shard_bounds_host(cost, world, kappa=8)
        assert tcb.tc_shard_bounds(g, world) == b          # cached
        tot = [0] * 16
        for r in range(world):
            part = tcb.tc_census_range(g, b[r], b[r + 1])
            tot = [x + y for x, y in zip(tot, part)]
        assert tcb.tc_close_census(a.n, tot) == full
    with pytest.raises(tcb.TCError, match="TC_E_INVALID"):
        tcb.tc_shard_bounds(g, 1025)
    g.close()


def test_relabelling_invariance(tcb):
    a = synth.make_config("C2")
    c, _ = gpu_census(tcb, a)
    for seed in (5, 6):
        assert gpu_census(tcb, synth.relabel(a, seed))[0] == c


def test_device_arcs_equal_host_arcs(tcb):
    import torch
    a = synth.make_config("C2")
    s = torch.from_numpy(a.src.astype(np.int32)).cuda()
    d = torch.from_numpy(a.dst.astype(np.int32)).cuda()
    g = tcb.tc_graph_create(a.n, s, d)
    assert g.census() == gpu_census(tcb, a)[0]
    g.close()


def test_device_arcs_any_alignment(tcb):
    """The first sort pass reads the arc arrays with 16-byte loads when both
    are 16-byte aligned and per arc otherwise (radix_sort.cu rs_upsweep):
    arrays starting 0..3 elements into an allocation give the same census
    and stats as the host path."""
    import torch
    a = synth.make_config("C2")
    m = a.src.size
    exp = gpu_census(tcb, a)

    def at(x, off):   # x on the device, starting `off` int32 into a fresh allocation
        buf = torch.zeros(m + 4, dtype=torch.int32, device="cuda")
        buf[off:off + m] = torch.from_numpy(x.astype(np.int32)).cuda()
        return buf[off:off + m]
    for off_s, off_d in ((0, 0), (1, 0), (0, 2), (3, 3)):
        g = tcb.tc_graph_create(a.n, at(a.src, off_s), at(a.dst, off_d))
        try:
            assert (g.census(), g.stats()) == exp, (off_s, off_d)
        finally:
            g.close()


def test_out_of_range_arc_index_full_tiles(tcb):
    """The smallest index of an out-of-range arc is reported from full
    4096-arc tiles as well as from the partial last tile."""
    rng = np.random.default_rng(5)
    n, m = 1000, 20000
    src = rng.integers(0, n, m).astype(np.uint32)
    dst = rng.integers(0, n, m).astype(np.uint32)
    src[7001] = n + 5
    dst[5003] = n
    with pytest.raises(tcb.TCError, match="arc 5003 "):
        tcb.tc_graph_create(n, src, dst)
    src[5] = 2**31   # one more, in the first tile
    with pytest.raises(tcb.TCError, match="arc 5 "):
        tcb.tc_graph_create(n, src, dst)


def test_closed_form_hub_star_warp_bin_and_high_word(tcb):
    # cost 2e5+1 per dyad -> warp-bin items (skewed pairs); n = 1e7 -> 003
    # needs the high word
    n, k = 10_000_000, 200_000
    for gen, cp, cs in ((synth.out_star, "012", "021D"), (synth.mutual_star, "102", "201")):
        a = gen(k, n)
        exp = {cp: k * (n - k - 1), cs: k * (k - 1) // 2}
        exp["003"] = C3(n) - sum(exp.values())
        c, _ = gpu_census(tcb, a)
        assert c == vec(exp)
        assert c[0] >= 2**64


def test_closed_form_tournament_clique_bipartite_cycle(tcb):
    a = synth.transitive_tournament(3000)
    assert gpu_census(tcb, a)[0] == vec({"030T": C3(3000)})
    b = synth.complete_mutual(200)
    assert gpu_census(tcb, b)[0] == vec({"300": C3(200)})
    x, y = 4, 200_000
    c = synth.complete_bipartite(x, y)
    assert gpu_census(tcb, c)[0] == vec({"021U": y * 6, "021D": x * (y * (y - 1) // 2),
                                         "003": C3(x) + C3(y)})
    n = 1_000_000
    d = synth.directed_cycle(n)
    exp = {"012": n * (n - 4), "021C": n}
    exp["003"] = C3(n) - sum(exp.values())
    assert gpu_census(tcb, d)[0] == vec(exp)


def test_mixed_bins_skewed_rmat(tcb):
    # R-MAT scale 12 edge factor 16: dyads in both the thread and warp bins
    a = synth.rmat(scale=12, edge_factor=16, seed=99)
    g = tcb.tc_graph_create(a.n, a.src, a.dst)
    g.profile(True)
    c = g.census()
    prof = g.profile_get()
    assert c == oracle.census(a.n, a.src, a.dst)
    assert all(x > 0 for x in prof["bin_items"][:2])
    g.close()


def test_errors(tcb):
    with pytest.raises(tcb.TCError, match="arc 1 "):
        tcb.tc_graph_create(5, np.array([0, 7, 1], np.uint32), np.array([1, 0, 2], np.uint32))
    with pytest.raises(tcb.TCError, match="TC_E_INVALID"):
        tcb.tc_graph_create(2**30, np.zeros(0, np.uint32), np.zeros(0, np.uint32))


def test_census_multi_world1_nccl(tcb):
    # tc_census_multi through a 1-rank NCCL communicator equals tc_census
    a = synth.make_config("C2")
    g = tcb.tc_graph_create(a.n, a.src, a.dst)
    comm = tcb.tc_comm_create(tcb.tc_comm_unique_id(), 1, 0, 0)
    try:
        assert tcb.tc_census_multi(g, comm) == g.census()
    finally:
        comm.close()
        g.close()


def test_census_multi_world1_borrowed_torch_comm(tcb):
    # tc_comm_wrap: torch's own NCCL communicator (1-rank group), borrowed
    import socket
    import torch.distributed as dist
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    dist.init_process_group("nccl", init_method="tcp://127.0.0.1:%d" % port, rank=0,
                            world_size=1)
    a = synth.make_config("C2")
    g = tcb.tc_graph_create(a.n, a.src, a.dst)
    try:
        comm = tcb.comm_wrap_process_group(0)
        try:
            assert tcb.tc_census_multi(g, comm) == g.census()
        finally:
            comm.close()          # frees the wrapper only; torch keeps its comm
    finally:
        g.close()
        dist.destroy_process_group()


def test_census64_vs_oracle(tcb):
    # f1: 64-type census, GPU vs oracle element by element
    cases = [synth.random_digraph(n, p, seed=7000 + n, loops=True, dups=3)
             for n, p in ((5, 0.5), (60, 0.1), (300, 0.05), (200, 0.6))]
    cases += [synth.make_config("C1"), synth.make_config("C2"), synth.rmat(12, 16, seed=3)]
    for a in cases:
        g = tcb.tc_graph_create(a.n, a.src, a.dst)
        assert tcb.tc_census64(g) == oracle.Graph(a.n, a.src, a.dst).census64(), a.meta
        g.close()


def _hub_graph(seed):
    """Two hubs (degree > kSparseMinDegree = 4096) inside a sparse random
    digraph with mutual arcs and triangles: big dyads with one short and one
    long list, so the warp bin takes the skewed-pair path (both modes)."""
    rng = np.random.default_rng(seed)
    n = 12000
    leaves = rng.choice(np.arange(100, n), 7000, replace=False)
    src = [np.full(7000, 5), leaves[:2000], rng.choice(np.arange(100, n), 6000), ]
    dst = [leaves, np.full(2000, 5), np.full(6000, 17)]
    src.append(rng.integers(0, n, 60000))          # background arcs
    dst.append(rng.integers(0, n, 60000))
    src.append(np.full(300, 17))                   # hub-hub and hub-leaf mutuals
    dst.append(leaves[:300])
    src.append(np.array([5, 17]))
    dst.append(np.array([17, 5]))
    s = np.concatenate(src).astype(np.uint32)
    d = np.concatenate(dst).astype(np.uint32)
    return n, s, d


@pytest.mark.parametrize("seed", [1, 2])
def test_skewed_pair_path_vs_oracle(tcb, seed):
    n, s, d = _hub_graph(seed)
    g = tcb.tc_graph_create(n, s, d)
    try:
        assert g.stats()["max_degree"] >= 4096
        g.profile(True)
        got = g.census()
        prof = g.profile_get()
        assert prof["bin_items"][3] > 0              # skewed-pair dyads were planned
        og = oracle.Graph(n, s, d)
        assert got == og.census()
        D = g.stats()["dyads"]
        for b, e in [(0, D // 3), (D // 3, D)]:
            assert tcb.tc_census_range(g, b, e) == og.census_range(b, e)
    finally:
        g.close()


def test_concurrent_census_on_shared_graph(tcb):
    # include/triadcensus.h: a graph may be shared by concurrent census calls
    # on different streams (host threads); each call publishes its own launch
    # count / profile under the graph's mutex
    import threading
    import torch
    a = synth.make_config("C2")
    g = tcb.tc_graph_create(a.n, a.src, a.dst)
    g.profile(True)
    want = g.census()
    og = oracle.Graph(a.n, a.src, a.dst)
    D = og.stats()["dyads"]
    out, errs = {}, []

    def work(t):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            for rep in range(5):
                if t % 2:
                    out[(t, rep)] = g.census(stream=s)
                else:
                    b, e = (t * 997) % D, min(D, (t * 997) % D + 5000)
                    out[(t, rep)] = (b, e, tcb.tc_census_range(g, b, e, stream=s))
        except Exception as ex:   # pragma: no cover - reported below
            errs.append(ex)

    th = [threading.Thread(target=work, args=(t,)) for t in range(6)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errs, errs
    for (t, rep), v in out.items():
        if t % 2:
            assert v == want
        else:
            b, e, part = v
            assert part == og.census_range(b, e)
    assert g.launches() > 0 and g.profile_get()["census_ms"] > 0
    g.close()


def _row_lengths_graph(lengths, n, seed):
    """Vertices 0..len(lengths)-1 get upper rows of exactly the given lengths
    (random targets above them, random directions, some arcs duplicated or
    reciprocated -- duplicates and mutual pairs sit in the row as extra keys
    of one (row, max) run), over a sparse random background."""
    rng = np.random.default_rng(seed)
    src, dst = [], []
    for u, L in enumerate(lengths):           # row u: exactly L canonical keys
        k = L // 5
        w = rng.choice(np.arange(u + 1, n), size=L - k, replace=False)
        fwd = rng.random(L - k) < 0.5
        src += list(np.where(fwd, u, w)); dst += list(np.where(fwd, w, u))
        extra = rng.choice(w, size=k, replace=False)       # duplicates / reciprocations
        rev = rng.random(k) < 0.5
        src += list(np.where(rev, extra, u)); dst += list(np.where(rev, u, extra))
    bg = synth.random_digraph(n, 4.0 / n, seed=seed + 1)
    keep = np.minimum(bg.src, bg.dst) >= len(lengths)     # background leaves those rows alone
    src = np.concatenate([np.array(src, np.uint32), bg.src[keep]])
    dst = np.concatenate([np.array(dst, np.uint32), bg.dst[keep]])
    perm = rng.permutation(src.size)
    return synth.Arcs(n, src[perm], dst[perm])


@pytest.mark.parametrize("lengths", [
    [31, 32, 33, 1, 2, 63, 64, 65, 30, 34],          # short/long boundary, chunk crossings
    [5] * 40 + [29, 3, 31, 7, 32, 32, 33],           # many short rows across 32-key chunks
    [700, 1000, 1024, 12, 300],                       # long rows up to the shared-memory bound
    [1025, 40, 3],                                    # one row above it: the full-LSD path
])
def test_row_sort_lengths_vs_oracle(tcb, lengths):
    """a1 row sort (csr_build.cu k_row_sort / k_row_sort_long): rows of
    exactly 32 / 33 / 1024 / 1025 canonical keys, rows crossing the 32-key
    chunks, duplicates and mutual pairs inside a row; census and stats equal
    the oracle's."""
    for seed in range(3):
        a = _row_lengths_graph(lengths, 3000, seed)
        c, st = gpu_census(tcb, a)
        g = oracle.Graph(a.n, a.src, a.dst)
        assert c == g.census(), (lengths, seed)
        assert st == g.stats(), (lengths, seed)


def test_build_sort_report(tcb):
    """tc_profile.build_sort names the a1 path the build took: a graph with
    short rows takes ceil(b / 8) LSD passes on the row bits plus the per-row
    networks (every canonical key of a row of <= 1024 keys); a graph with one
    1025-key row adds the composite LSD over that row; a hub graph (more than
    a fifth of the keys in rows of > 64 keys) takes the full LSD and no
    networks.  The transposed sort is ceil(b / 8) passes either way."""
    n = 3000
    b = int(np.ceil(np.log2(n)))
    passes = (b + 7) // 8
    cases = [(_row_lengths_graph([31, 33, 64, 65], n, 0), "rows"),
             (_row_lengths_graph([1025, 40], n, 1), "huge"),
             (synth.out_star(n - 1), "hub")]
    for a, kind in cases:
        g = tcb.tc_graph_create(a.n, a.src, a.dst)
        try:
            bs = g.profile_get()["build_sort"]
            st = g.stats()
        finally:
            g.close()
        assert bs[1] == passes, (kind, bs)
        keys = st["m_in"] - st["loops_dropped"]
        if kind == "hub":
            assert bs[0] == 3 * passes, (kind, bs)     # the row-bit passes, then max + min bits
            assert bs[2] == 0 and bs[3] == 0, (kind, bs)
        else:
            assert bs[0] == passes, (kind, bs)
            huge = 1025 if kind == "huge" else 0
            assert bs[2] == keys - huge, (kind, bs, keys)
            assert (bs[3] > 0) == (kind == "huge"), (kind, bs)


def test_default_allocator_cache_and_trim(tcb):
    """The default allocator (exact-size block cache, abi.cu) reuses a freed
    graph's blocks for the next graph of the same size on the same stream;
    tc_trim_memory returns them to the driver; the census is unchanged
    through both (and with the torch allocator)."""
    a = synth.random_digraph(2000, 0.004, seed=77, dups=3)
    exp = oracle.census(a.n, a.src, a.dst)
    for torch_alloc in (False, True):
        for _ in range(3):
            g = tcb.tc_graph_create(a.n, a.src, a.dst, use_torch_allocator=torch_alloc)
            try:
                assert g.census() == exp
            finally:
                g.close()
        tcb.tc_trim_memory()
    g = tcb.tc_graph_create(a.n, a.src, a.dst, use_torch_allocator=False)
    try:
        assert g.census() == exp and g.stats()["dyads"] > 0
    finally:
        g.close()
