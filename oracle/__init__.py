"""oracle -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU triad census written from PAPER.md
(arXiv 1603.02655), used to prove the CUDA path right.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import this package.  The product package
``paper_1603_02655_b200`` never imports it, and the two share no code: the
only common input is the arc list from ``synth/``.

* ``bm_oracle.c``  literal Batagelj-Mrvar census (Fig. P:269-309 + v0.4
  P:1396-1432), O(n^3) brute force, orbit-derived TriadTable
  (P:327/P:343), 128-bit null closing, dyad-range mode.
* ``pyref.py``     a tiny pure-Python restatement for n <= ~30.

Pins (tests/test_oracle_*.py, ``-m "not gpu"``): the published B-M 2001
TRICODES tuple, class sizes, the 16 single-triad graphs, SPEC worked
examples (tests/golden/), brute force, networkx.triadic_census, closed-form
graphs, linear census identities, and C(n,3) with Python integers.
Nothing here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bm_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

CLASS_NAMES = ("003", "012", "102", "021D", "021U", "021C", "111D", "111U",
               "030T", "030C", "201", "120D", "120U", "120C", "210", "300")


def build(force: bool = False) -> str:
    """Compile bm_oracle.c into liboracle.so with gcc (plain -O2)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-Wextra", "-shared",
                               "-fPIC", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


class _Stats(ctypes.Structure):
    _fields_ = [(k, ctypes.c_uint64) for k in (
        "n", "m_in", "m", "loops_dropped", "dups_dropped", "dyads", "mutual_dyads",
        "max_degree", "sum_deg_sq")]


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            u64, u32p, u64p, vp = (ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint32),
                                   ctypes.POINTER(ctypes.c_uint64), ctypes.c_void_p)
            lib.og_graph_build.restype = vp
            lib.og_graph_build.argtypes = [u64, u32p, u32p, u64, u64p]
            lib.og_graph_free.argtypes = [vp]
            lib.og_graph_stats.argtypes = [vp, ctypes.POINTER(_Stats)]
            lib.og_triad_table.argtypes = [ctypes.POINTER(ctypes.c_uint8)]
            lib.og_census.argtypes = [vp, u64p, u64p]
            lib.og_census_range.argtypes = [vp, u64, u64, u64p]
            lib.og_bruteforce.argtypes = [vp, u64p, u64p]
            lib.og_census64.argtypes = [vp, u64p, u64p]
            lib.og_bruteforce64.argtypes = [vp, u64p, u64p]
            lib.og_dyad_costs.argtypes = [vp, u64p]
            lib.og_task_queues.argtypes = [vp, ctypes.c_int, u64, u64p, u64, u64p, u64p]
            lib.og_choose3_u128.argtypes = [u64, u64p, u64p]
            lib.og_graph_n.restype = u64
            lib.og_graph_m.restype = u64
            lib.og_graph_nnz.restype = u64
            for f in (lib.og_graph_n, lib.og_graph_m, lib.og_graph_nnz):
                f.argtypes = [vp]
            lib.og_graph_copy_n.argtypes = [vp, u64p, u32p]
            _lib = lib
    return _lib


def _u32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint32))


def _p(a, t):
    return a.ctypes.data_as(ctypes.POINTER(t))


class OracleError(RuntimeError):
    pass


class Graph:
    """Sanitised digraph (loops dropped, duplicates merged) in the oracle's
    own two-CRS layout (E out-arcs, N undirected)."""

    def __init__(self, n: int, src, dst):
        lib = _load()
        s, d = _u32(src), _u32(dst)
        if s.shape != d.shape:
            raise OracleError("src/dst length mismatch")
        bad = ctypes.c_uint64(0)
        h = lib.og_graph_build(int(n), _p(s, ctypes.c_uint32), _p(d, ctypes.c_uint32),
                               int(s.size), ctypes.byref(bad))
        if not h:
            if bad.value != 2**64 - 1:
                raise OracleError("arc %d has an endpoint >= n" % bad.value)
            raise MemoryError("oracle graph build")
        self._h = h
        self._lib = lib
        self.n = int(n)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._lib.og_graph_free(h)
            self._h = None

    def stats(self) -> dict:
        st = _Stats()
        self._lib.og_graph_stats(self._h, ctypes.byref(st))
        return {k: int(getattr(st, k)) for k, _ in _Stats._fields_}

    def census(self) -> list[int]:
        """Full 16-class census as Python ints (class 003 exact, 128-bit)."""
        c = np.zeros(16, np.uint64)
        hi = ctypes.c_uint64(0)
        rc = self._lib.og_census(self._h, _p(c, ctypes.c_uint64), ctypes.byref(hi))
        if rc != 0:
            raise OracleError("og_census failed: %d" % rc)
        out = [int(x) for x in c]
        out[0] += int(hi.value) << 64
        return out

    def census_range(self, begin: int, end: int) -> list[int]:
        """Classes 2..16 of canonical dyads [begin, end) (counts[0] = 0)."""
        c = np.zeros(16, np.uint64)
        rc = self._lib.og_census_range(self._h, int(begin), int(end), _p(c, ctypes.c_uint64))
        if rc != 0:
            raise OracleError("og_census_range failed: %d" % rc)
        return [int(x) for x in c]

    def bruteforce(self) -> list[int]:
        c = np.zeros(16, np.uint64)
        hi = ctypes.c_uint64(0)
        rc = self._lib.og_bruteforce(self._h, _p(c, ctypes.c_uint64), ctypes.byref(hi))
        if rc != 0:
            raise OracleError("og_bruteforce failed: %d" % rc)
        out = [int(x) for x in c]
        out[0] += int(hi.value) << 64
        return out

    def census64(self) -> list[int]:
        """64-type (non-isomorphic) census in the B-M labelling."""
        return self._c64(self._lib.og_census64, "og_census64")

    def bruteforce64(self) -> list[int]:
        return self._c64(self._lib.og_bruteforce64, "og_bruteforce64")

    def _c64(self, fn, name):
        c = np.zeros(64, np.uint64)
        hi = ctypes.c_uint64(0)
        rc = fn(self._h, _p(c, ctypes.c_uint64), ctypes.byref(hi))
        if rc != 0:
            raise OracleError("%s failed: %d" % (name, rc))
        out = [int(x) for x in c]
        out[0] += int(hi.value) << 64
        return out

    def dyad_costs(self) -> np.ndarray:
        st = self.stats()
        out = np.zeros(st["dyads"], np.uint64)
        self._lib.og_dyad_costs(self._h, _p(out, ctypes.c_uint64))
        return out

    def task_queues(self, strategy: str, max_nset: int):
        """The paper's task queues: (starts of the non-empty
        queues in canonical dyad order, aggregate NsetSize)."""
        strat = {"uniform": 0, "nonuniform": 1}[strategy]
        cap = max(self.stats()["dyads"], 1)
        starts = np.zeros(cap, np.uint64)
        nq, tot = ctypes.c_uint64(0), ctypes.c_uint64(0)
        rc = self._lib.og_task_queues(self._h, strat, int(max_nset), _p(starts, ctypes.c_uint64),
                                      cap, ctypes.byref(nq), ctypes.byref(tot))
        if rc != 0:
            raise OracleError("og_task_queues failed (%d)" % rc)
        return starts[:nq.value].copy(), int(tot.value)

    def neighbours_crs(self):
        nnz = int(self._lib.og_graph_nnz(self._h))
        off = np.zeros(self.n + 1, np.uint64)
        col = np.zeros(max(nnz, 1), np.uint32)
        self._lib.og_graph_copy_n(self._h, _p(off, ctypes.c_uint64), _p(col, ctypes.c_uint32))
        return off, col[:nnz]


def triad_table() -> list[int]:
    """The 64-entry code -> class table (1-based classes), orbit-derived."""
    t = (ctypes.c_uint8 * 64)()
    if _load().og_triad_table(t) != 0:
        raise OracleError("orbit derivation failed")
    return list(t)


def choose3(n: int) -> int:
    lo, hi = ctypes.c_uint64(0), ctypes.c_uint64(0)
    _load().og_choose3_u128(int(n), ctypes.byref(lo), ctypes.byref(hi))
    return int(lo.value) + (int(hi.value) << 64)


def census(n: int, src, dst) -> list[int]:
    return Graph(n, src, dst).census()


def census_range(n: int, src, dst, begin: int, end: int) -> list[int]:
    return Graph(n, src, dst).census_range(begin, end)


def bruteforce(n: int, src, dst) -> list[int]:
    return Graph(n, src, dst).bruteforce()
