"""ctypes binding of libtriadcensus.so (include/triadcensus.h).

Argument marshalling only: every step of the census runs in the library's
CUDA kernels.  If the shared library is missing this module raises at
import time -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtriadcensus.so")
# dev only (tools/ab.sh): same-box A/B timing of a variant build of the library
if os.environ.get("TC_LIB_VARIANT"):
    LIB_PATH = os.path.abspath(os.environ["TC_LIB_VARIANT"])

if not os.path.exists(LIB_PATH):
    raise ImportError(
        "libtriadcensus.so not built (%s); run `python -c 'import __graft_entry__ as g; "
        "g.build()'` -- there is no CPU fallback" % LIB_PATH)

lib = ctypes.CDLL(LIB_PATH)

u64 = ctypes.c_uint64
u32p = ctypes.POINTER(ctypes.c_uint32)
u64p = ctypes.POINTER(ctypes.c_uint64)
vp = ctypes.c_void_p
cint = ctypes.c_int

ALLOC_FN = ctypes.CFUNCTYPE(vp, ctypes.c_size_t, vp, vp)
FREE_FN = ctypes.CFUNCTYPE(None, vp, ctypes.c_size_t, vp, vp)


class tc_allocator(ctypes.Structure):
    _fields_ = [("alloc", ALLOC_FN), ("free", FREE_FN), ("ctx", vp)]


class tc_graph_stats(ctypes.Structure):
    _fields_ = [(k, u64) for k in ("n", "m_in", "m", "loops_dropped", "dups_dropped", "dyads",
                                   "mutual_dyads", "max_degree", "sum_deg_sq")]


class tc_profile(ctypes.Structure):
    _fields_ = [("build_ms", ctypes.c_float), ("plan_ms", ctypes.c_float),
                ("census_ms", ctypes.c_float), ("kernel_ms", ctypes.c_float * 4),
                ("bin_items", u64 * 4), ("bin_work", u64 * 4), ("sparse_sum_c", u64),
                ("sparse_units", u64), ("build_sort", u64 * 4)]


TC_OK, TC_E_INVALID, TC_E_RANGE, TC_E_OOM, TC_E_CUDA, TC_E_NCCL, TC_E_OVERFLOW = range(7)
STATUS_NAMES = {0: "TC_OK", 1: "TC_E_INVALID", 2: "TC_E_RANGE", 3: "TC_E_OOM", 4: "TC_E_CUDA",
                5: "TC_E_NCCL", 6: "TC_E_OVERFLOW"}

_SIGS = {
    "tc_graph_create": (cint, [cint, u64, vp, vp, u64, cint, vp, ctypes.POINTER(tc_allocator),
                               ctypes.POINTER(vp)]),
    "tc_graph_stats_get": (cint, [vp, ctypes.POINTER(tc_graph_stats)]),
    "tc_graph_destroy": (None, [vp]),
    "tc_census": (cint, [vp, vp, u64p, u64p]),
    "tc_census_range": (cint, [vp, u64, u64, vp, u64p]),
    "tc_census64": (cint, [vp, vp, u64p, u64p]),
    "tc_census_enqueue": (cint, [vp, u64, u64, vp, vp]),
    "tc_close_census": (cint, [u64, u64p, u64p]),
    "tc_shard_bounds_host": (cint, [u64p, u64, cint, u64, u64p]),
    "tc_shard_bounds": (cint, [vp, cint, vp, u64p]),
    "tc_task_queues": (cint, [vp, cint, u64, vp, u64p, u64, u64p, u64p]),
    "tc_comm_unique_id": (cint, [ctypes.POINTER(ctypes.c_uint8)]),
    "tc_comm_create": (cint, [ctypes.POINTER(ctypes.c_uint8), cint, cint, cint, ctypes.POINTER(vp)]),
    "tc_comm_destroy": (None, [vp]),
    "tc_comm_wrap": (cint, [vp, ctypes.POINTER(vp)]),
    "tc_census_multi": (cint, [vp, vp, vp, u64p, u64p]),
    "tc_profile_enable": (cint, [vp, cint]),
    "tc_profile_get": (cint, [vp, ctypes.POINTER(tc_profile)]),
    "tc_launch_count": (u64, [vp]),
    "tc_trim_memory": (cint, []),
    "tc_read_arcs": (cint, [ctypes.c_char_p, cint, cint, u64p, ctypes.POINTER(u32p),
                            ctypes.POINTER(u32p), u64p]),
    "tc_free_arcs": (None, [u32p]),
    "tc_last_error": (ctypes.c_char_p, []),
    "tc_abi_version": (cint, []),
}

for _name, (_res, _args) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_SIGS)


class TCError(RuntimeError):
    def __init__(self, status, where):
        msg = lib.tc_last_error().decode(errors="replace")
        super().__init__("%s failed: %s: %s" % (where, STATUS_NAMES.get(status, status), msg))
        self.status = status


def check(status, where):
    if status != TC_OK:
        raise TCError(status, where)
