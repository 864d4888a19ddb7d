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
