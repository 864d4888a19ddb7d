"""CPU-side checks of the boundary: the library loads without a GPU, exports
every symbol include/triadcensus.h declares, and its host-only functions
(128-bit closing a5, shard cut rule) behave.  No device compute here."""
import json
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    txt = open(os.path.join(ROOT, "include", "triadcensus.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(tc_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    import paper_1603_02655_b200 as tcb
    names = header_functions()
    assert len(names) >= 15
    for nm in names:
        assert hasattr(tcb.lib, nm), nm
    out = subprocess.check_output(["nm", "-D", "--defined-only", tcb._lib.LIB_PATH], text=True)
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [nm for nm in names if nm not in exported]
    assert not missing, missing
    assert set(tcb._lib.EXPORTED) >= set(names)


def test_abi_version():
    import paper_1603_02655_b200 as tcb
    assert tcb.lib.tc_abi_version() == 1


def test_no_oracle_in_product_path():
    # the product package must never import or link the oracle
    pkg = os.path.join(ROOT, "paper_1603_02655_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f), errors="replace").read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "bm_oracle" not in src and "liboracle" not in src, f
    out = subprocess.check_output(["ldd", os.path.join(pkg, "libtriadcensus.so")], text=True)
    assert "oracle" not in out


def test_device_table_literal_is_published_tricodes():
    # the CUDA path hard-codes TriadTable; it must be the B-M 2001 table
    src = open(os.path.join(ROOT, "paper_1603_02655_b200", "csrc", "census.cu")).read()
    body = re.search(r"c_triad_table\[64\]\s*=\s*\{([^}]*)\}", src).group(1)
    vals = [int(x) for x in re.findall(r"\d+", body)]
    ref = json.load(open(os.path.join(ROOT, "tests", "golden", "tricodes.json")))["tricodes"]
    assert vals == [x - 1 for x in ref]


def C3(n):
    return n * (n - 1) * (n - 2) // 6 if n >= 3 else 0


@pytest.mark.parametrize("n", [0, 1, 2, 3, 1000, 4_801_280, 4_801_281, 67_108_864, 2**30 - 1])
def test_close_census_128bit(n):
    import paper_1603_02655_b200 as tcb
    rng = np.random.default_rng(n)
    rest = [0] + [int(x) for x in rng.integers(0, 1000, size=15)] if n > 100 else [0] * 16
    out = tcb.tc_close_census(n, rest)
    assert out[1:] == rest[1:]
    assert out[0] == C3(n) - sum(rest)


def test_close_census_rejects_inconsistent_sum():
    import paper_1603_02655_b200 as tcb
    with pytest.raises(tcb.TCError):
        tcb.tc_close_census(3, [0, 2] + [0] * 14)


def test_close_census_overflow_needs_high_word():
    import ctypes
    import paper_1603_02655_b200 as tcb
    c = (ctypes.c_uint64 * 16)()
    assert tcb.lib.tc_close_census(5_000_000, c, None) == tcb._lib.TC_E_OVERFLOW
    assert tcb.lib.tc_close_census(4_801_280, c, None) == tcb._lib.TC_OK


def test_shard_bounds_host_rule():
    import paper_1603_02655_b200 as tcb
    rng = np.random.default_rng(5)
    cost = rng.integers(2, 5000, size=10_000).astype(np.uint64)
    for world in (1, 2, 3, 4, 8):
        b = tcb.tc_shard_bounds_host(cost, world, kappa=8)
        assert b[0] == 0 and b[-1] == cost.size and b == sorted(b)
        pre = np.concatenate([[0], np.cumsum(cost + 8)])
        T = int(pre[-1])
        for r in range(1, world):
            t = T * r // world
            # first k with exclusive prefix >= t
            assert b[r] == int(np.searchsorted(pre[:-1], t, side="left"))
        # balance: every shard within one max dyad cost of T/world
        for r in range(world):
            s = int(pre[b[r + 1]] - pre[b[r]])
            assert abs(s - T / world) <= int(cost.max()) + 8 + 1
