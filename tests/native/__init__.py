"""Test-only native helpers (plain C, built with gcc on first use)."""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))


def _lib(name):
    src = os.path.join(_HERE, name + ".c")
    so = os.path.join(_HERE, "lib%s.so" % name)
    if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
        tmp = so + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", tmp, src])
        os.replace(tmp, so)
    return ctypes.CDLL(so)


def triangles(n, src, dst):
    """Undirected triangle count (forward algorithm, tri_count.c)."""
    lib = _lib("tri_count")
    lib.tri_count.restype = ctypes.c_uint64
    lib.tri_count.argtypes = [ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64]
    s = np.ascontiguousarray(np.asarray(src, np.uint32))
    d = np.ascontiguousarray(np.asarray(dst, np.uint32))
    t = lib.tri_count(int(n), s.ctypes.data, d.ctypes.data, int(s.size))
    if t == 2**64 - 1:
        raise MemoryError("tri_count")
    return int(t)
