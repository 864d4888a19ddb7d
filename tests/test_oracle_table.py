"""Pins of the oracle's orbit-derived TriadTable (contents not
printed in the paper) against things fixed outside the oracle."""
import itertools
import json
import os

import oracle
from oracle import pyref

NAMES = oracle.CLASS_NAMES


def test_table_equals_published_tricodes(golden_dir):
    ref = json.load(open(os.path.join(golden_dir, "tricodes.json")))["tricodes"]
    assert oracle.triad_table() == ref


def test_class_sizes(golden_dir):
    sizes = json.load(open(os.path.join(golden_dir, "spec_examples.json")))["class_sizes"]["sizes"]
    T = oracle.triad_table()
    assert [T.count(k) for k in range(1, 17)] == sizes
    assert sum(sizes) == 64


def _permute(code, p):
    # bit for x_a -> x_b in the (u,v,w) layout of Fig. TriadCode
    bit = {(0, 1): 1, (1, 0): 2, (0, 2): 4, (2, 0): 8, (1, 2): 16, (2, 1): 32}
    out = 0
    for (a, b), m in bit.items():
        if code & m:
            out |= bit[(p[a], p[b])]
    return out


def test_table_invariant_under_relabelling():
    T = oracle.triad_table()
    for code in range(64):
        for p in itertools.permutations(range(3)):
            assert T[_permute(code, p)] == T[code]
    # 16 distinct classes
    assert sorted(set(T)) == list(range(1, 17))


def test_man_digits_match_class_names():
    # every code's (mutual, asymmetric, null) digits equal the first three
    # characters of its class name (MAN naming convention)
    T = oracle.triad_table()
    for code in range(64):
        m, a, n = pyref.man_digits(code)
        assert NAMES[T[code] - 1][:3] == "%d%d%d" % (m, a, n), code


def test_spec_triad_code_examples(golden_dir):
    ex = json.load(open(os.path.join(golden_dir, "spec_examples.json")))["triad_code"]
    T = oracle.triad_table()
    for e in ex:
        assert NAMES[T[e["code"]] - 1] == e["class"], e["cite"]
