"""f2: the native graph-file reader (host code of
libtriadcensus, no GPU needed).  Cases from SPEC.md "ingest"."""
import numpy as np
import pytest

import oracle
import synth


@pytest.fixture(scope="module")
def tcb():
    import paper_1603_02655_b200 as m
    return m


def write(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


def arcs(src, dst):
    return sorted(zip(src.tolist(), dst.tolist()))


def test_pajek_minimal(tcb, tmp_path):
    n, s, d = tcb.tc_read_arcs(write(tmp_path, "a.net", "*Vertices 3\n*Arcs\n1 2\n"))
    assert n == 3 and arcs(s, d) == [(0, 1)]


def test_pajek_edges_expand(tcb, tmp_path):
    n, s, d = tcb.tc_read_arcs(write(tmp_path, "b.net", "*Vertices 2\n*Edges\n1 2\n"))
    assert n == 2 and arcs(s, d) == [(0, 1), (1, 0)]


def test_pajek_labels_comments_case(tcb, tmp_path):
    txt = ('% comment\n*vertices 4\n1 "a"\n2 "b"\n3 "c"\n4 "d"\n*ARCS\n1 2 0.5\n\n3 4 1\n'
           '*edges\n2 3\n')
    n, s, d = tcb.tc_read_arcs(write(tmp_path, "c.net", txt))
    assert n == 4 and arcs(s, d) == [(0, 1), (1, 2), (2, 1), (2, 3)]


def test_pajek_errors(tcb, tmp_path):
    with pytest.raises(tcb.TCError, match="line 3"):
        tcb.tc_read_arcs(write(tmp_path, "d.net", "*Vertices 2\n*Arcs\n1 x\n"))
    with pytest.raises(tcb.TCError, match="TC_E_RANGE"):
        tcb.tc_read_arcs(write(tmp_path, "e.net", "*Vertices 2\n*Arcs\n1 3\n"))


def test_edgelist_bases(tcb, tmp_path):
    n, s, d = tcb.tc_read_arcs(write(tmp_path, "f.txt", "# comment\n0 1\n1 2\n"))
    assert n == 3 and arcs(s, d) == [(0, 1), (1, 2)]
    n, s, d = tcb.tc_read_arcs(write(tmp_path, "g.txt", "1 2\n2 3\n"))
    assert n == 3 and arcs(s, d) == [(0, 1), (1, 2)]
    with pytest.raises(tcb.TCError, match="line 1"):   # three tokens
        tcb.tc_read_arcs(write(tmp_path, "h.txt", "1 2 3\n"))


def test_pajek_round_trip_census(tcb, tmp_path):
    a = synth.random_digraph(40, 0.1, seed=9)
    lines = ["*Vertices %d" % a.n, "*Arcs"] + ["%d %d" % (x + 1, y + 1) for x, y in zip(a.src, a.dst)]
    n, s, d = tcb.tc_read_arcs(write(tmp_path, "r.net", "\n".join(lines) + "\n"))
    assert n == a.n and arcs(s, d) == arcs(a.src, a.dst)
    assert oracle.census(n, s, d) == oracle.census(a.n, a.src, a.dst)


def _write_snap(path, a, base):
    with open(path, "w") as f:
        f.write("# Directed graph (each unordered pair a line)\n# FromNodeId\tToNodeId\n")
        np.savetxt(f, np.stack([a.src.astype(np.int64) + base, a.dst.astype(np.int64) + base], 1),
                   fmt="%d", delimiter="\t")


@pytest.mark.gpu
@pytest.mark.parametrize("fmt", ["pajek", "snap0", "snap1"])
def test_census_file_gpu_vs_oracle(tmp_path, fmt):
    # f2 end to end on the GPU: file -> native reader -> CUDA census, against
    # the oracle on the generator's own arcs; the paper's phase breakdown
    # (read graph / neighbour sets / task queues / census) is
    # reported
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1603_02655_b200 as tcb
    a = synth.make_config("C2")
    if fmt == "pajek":
        p = str(tmp_path / "c2.net")
        half = a.src.size // 2           # second half as *Edges (each -> two arcs)
        with open(p, "w") as f:
            f.write("*Vertices %d\n*Arcs\n" % a.n)
            np.savetxt(f, np.stack([a.src[:half] + 1, a.dst[:half] + 1], 1).astype(np.int64),
                       fmt="%d")
            f.write("*Edges\n")
            np.savetxt(f, np.stack([a.src[half:] + 1, a.dst[half:] + 1], 1).astype(np.int64),
                       fmt="%d")
        src = np.concatenate([a.src, a.dst[half:]])
        dst = np.concatenate([a.dst, a.src[half:]])
        n = a.n
    else:
        base = int(fmt[-1])
        p = str(tmp_path / "c2.txt")
        _write_snap(p, a, base)
        src, dst = a.src, a.dst
        n = int(max(a.src.max(), a.dst.max())) + 1      # SNAP: n = max id - base + 1
    counts, timing = tcb.census_file(p, index_base=None if fmt == "pajek" else int(fmt[-1]))
    assert counts == oracle.census(n, src, dst)
    for k in ("read_graph", "build_csr", "plan", "census_kernels", "total"):
        assert timing[k] >= 0.0
