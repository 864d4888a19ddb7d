"""paper_1603_02655_b200 -- B200-native directed triad census (arXiv 1603.02655).

The Batagelj-Mrvar subquadratic census (Fig. "Subquadratic Triad Census
Algorithm") as hand-written sm_100a CUDA behind the C ABI
of ``include/triadcensus.h`` (``libtriadcensus.so``).  This module is the
thin Python binding: the same function names as the ABI, marshalling only.
PyTorch is used for device memory (its caching allocator through the ABI's
allocator hook), streams and torch.distributed process groups.

    import paper_1603_02655_b200 as tcb
    g = tcb.tc_graph_create(n, src, dst)          # numpy (host) or torch CUDA tensors
    counts = tcb.tc_census(g)                      # 16 Python ints, 003 exact
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._lib import TCError, check, lib

CLASS_NAMES = ("003", "012", "102", "021D", "021U", "021C", "111D", "111U",
               "030T", "030C", "201", "120D", "120U", "120C", "210", "300")

__all__ = ["tc_read_arcs", "census_file", "CLASS_NAMES", "Graph", "TCError", "tc_graph_create", "tc_census", "tc_census_range",
           "tc_census_enqueue", "tc_census_multi", "tc_census64", "tc_close_census", "tc_shard_bounds",
           "tc_shard_bounds_host", "tc_comm_create", "tc_comm_unique_id", "tc_comm_wrap",
           "comm_from_process_group", "comm_wrap_process_group", "tc_task_queues", "Comm",
           "census", "lib"]


def _torch():
    import torch
    return torch


class _TorchAllocator:
    """Routes the library's device allocations through torch's caching
    allocator (ABI allocator hook)."""

    def __init__(self, device):
        torch = _torch()
        self._torch = torch
        self.device = device

        def _alloc(nbytes, stream, ctx):
            try:
                return torch.cuda.caching_allocator_alloc(int(nbytes), self.device,
                                                          int(stream or 0))
            except Exception:   # OOM -> NULL -> TC_E_OOM
                return None

        def _free(ptr, nbytes, stream, ctx):
            torch.cuda.caching_allocator_delete(ptr)

        self._alloc = _lib.ALLOC_FN(_alloc)
        self._free = _lib.FREE_FN(_free)
        self.struct = _lib.tc_allocator(self._alloc, self._free, None)


def _stream_ptr(stream):
    if stream is None:
        return _torch().cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


class Graph:
    """Owns a ``tc_graph*`` (device CSR built by ``tc_graph_create``)."""

    def __init__(self, handle, device, allocator, keepalive=None):
        self._h = handle
        self.device = device
        self._alloc = allocator
        self._keep = keepalive

    @property
    def handle(self):
        return self._h

    def stats(self) -> dict:
        st = _lib.tc_graph_stats()
        check(lib.tc_graph_stats_get(self._h, ctypes.byref(st)), "tc_graph_stats_get")
        return {k: int(getattr(st, k)) for k, _ in _lib.tc_graph_stats._fields_}

    def profile(self, on: bool = True):
        check(lib.tc_profile_enable(self._h, int(on)), "tc_profile_enable")

    def profile_get(self) -> dict:
        p = _lib.tc_profile()
        check(lib.tc_profile_get(self._h, ctypes.byref(p)), "tc_profile_get")
        return {"build_ms": p.build_ms, "plan_ms": p.plan_ms, "census_ms": p.census_ms,
                "kernel_ms": list(p.kernel_ms), "bin_items": [int(x) for x in p.bin_items],
                "bin_work": [int(x) for x in p.bin_work], "sparse_sum_c": int(p.sparse_sum_c),
                "sparse_units": int(p.sparse_units),
                "build_sort": [int(x) for x in p.build_sort]}

    def launches(self) -> int:
        return int(lib.tc_launch_count(self._h))

    def close(self):
        if self._h:
            lib.tc_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def census(self, stream=None) -> list[int]:
        return tc_census(self, stream)


def tc_graph_create(n: int, src, dst, device: int = 0, stream=None,
                    use_torch_allocator: bool = True) -> Graph:
    """Build the device graph from arcs src[i] -> dst[i].  src/dst are numpy
    uint32 arrays (host; copied H2D inside the call) or CUDA uint32/int32
    torch tensors (device)."""
    torch = _torch()
    keep = []
    on_device = 0
    if hasattr(src, "is_cuda") and src.is_cuda:
        if src.dtype not in (torch.int32, torch.uint32) or dst.dtype != src.dtype:
            raise TypeError("device arcs must be int32/uint32 CUDA tensors")
        s, d = src.contiguous(), dst.contiguous()
        keep += [s, d]
        ps, pd, m, on_device = s.data_ptr(), d.data_ptr(), s.numel(), 1
        device = s.device.index
    else:
        s = np.ascontiguousarray(np.asarray(src, dtype=np.uint32))
        d = np.ascontiguousarray(np.asarray(dst, dtype=np.uint32))
        if s.shape != d.shape:
            raise ValueError("src/dst length mismatch")
        keep += [s, d]
        ps, pd, m = s.ctypes.data, d.ctypes.data, s.size
    torch.cuda.set_device(device)
    alloc = _TorchAllocator(device) if use_torch_allocator else None
    h = ctypes.c_void_p()
    st = lib.tc_graph_create(int(device), int(n), ps, pd, int(m), on_device, _stream_ptr(stream),
                             ctypes.byref(alloc.struct) if alloc else None, ctypes.byref(h))
    check(st, "tc_graph_create")
    return Graph(h.value, device, alloc)


def _join003(c, hi):
    out = [int(x) for x in c]
    out[0] += int(hi) << 64
    return out


def tc_census(g: Graph, stream=None) -> list[int]:
    """Full 16-class census; counts[0] (003) is exact (128-bit)."""
    c = (ctypes.c_uint64 * 16)()
    hi = ctypes.c_uint64(0)
    check(lib.tc_census(g.handle, _stream_ptr(stream), c, ctypes.byref(hi)), "tc_census")
    return _join003(c, hi.value)


def tc_census64(g: Graph, stream=None) -> list[int]:
    """64-type (non-isomorphic) census in the B-M labelling; [0] exact."""
    c = (ctypes.c_uint64 * 64)()
    hi = ctypes.c_uint64(0)
    check(lib.tc_census64(g.handle, _stream_ptr(stream), c, ctypes.byref(hi)), "tc_census64")
    out = [int(x) for x in c]
    out[0] += int(hi.value) << 64
    return out


def tc_census_range(g: Graph, begin: int, end: int, stream=None) -> list[int]:
    """Classes 2..16 over canonical dyads [begin, end); element 0 is 0."""
    c = (ctypes.c_uint64 * 16)()
    check(lib.tc_census_range(g.handle, int(begin), int(end), _stream_ptr(stream), c),
          "tc_census_range")
    return [int(x) for x in c]


def tc_census_enqueue(g: Graph, d_counts, begin: int = 0, end: int | None = None, stream=None):
    """Enqueue a partial census adding into d_counts (torch uint64/int64 CUDA
    tensor of 16); no host sync beyond the plan's size read-back."""
    end = g.stats()["dyads"] if end is None else end
    check(lib.tc_census_enqueue(g.handle, int(begin), int(end), _stream_ptr(stream),
                                d_counts.data_ptr()), "tc_census_enqueue")


def tc_close_census(n: int, counts) -> list[int]:
    c = (ctypes.c_uint64 * 16)(*[int(x) & (2**64 - 1) for x in counts])
    hi = ctypes.c_uint64(0)
    check(lib.tc_close_census(int(n), c, ctypes.byref(hi)), "tc_close_census")
    return _join003(c, hi.value)


def tc_shard_bounds_host(cost, world: int, kappa: int = 8) -> list[int]:
    a = np.ascontiguousarray(np.asarray(cost, dtype=np.uint64))
    b = (ctypes.c_uint64 * (world + 1))()
    check(lib.tc_shard_bounds_host(a.ctypes.data_as(_lib.u64p), a.size, int(world), int(kappa),
                                   b), "tc_shard_bounds_host")
    return [int(x) for x in b]


def tc_shard_bounds(g: Graph, world: int, stream=None) -> list[int]:
    b = (ctypes.c_uint64 * (world + 1))()
    check(lib.tc_shard_bounds(g.handle, int(world), _stream_ptr(stream), b), "tc_shard_bounds")
    return [int(x) for x in b]


def tc_task_queues(g: Graph, strategy: str, max_nset_size: int, stream=None):
    """The paper's task queues on the GPU: (starts of the
    non-empty queues as a uint64 array in canonical dyad order, aggregate
    NsetSize).  strategy: "uniform" or "nonuniform"."""
    strat = {"uniform": 0, "nonuniform": 1}[strategy]
    nq, tot = ctypes.c_uint64(0), ctypes.c_uint64(0)
    cap = max(min(int(g.stats()["dyads"]), 1 << 16), 1)   # never more queues than dyads
    while True:
        out = np.zeros(cap, np.uint64)
        st = lib.tc_task_queues(g.handle, strat, int(max_nset_size), _stream_ptr(stream),
                                out.ctypes.data_as(_lib.u64p), cap, ctypes.byref(nq),
                                ctypes.byref(tot))
        if st == _lib.TC_E_RANGE and nq.value > cap:
            cap = int(nq.value)                 # rerun with the exact count
            continue
        check(st, "tc_task_queues")
        return out[:nq.value].copy(), int(tot.value)


def tc_comm_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    check(lib.tc_comm_unique_id(buf), "tc_comm_unique_id")
    return bytes(buf)


class Comm:
    def __init__(self, handle):
        self._h = handle

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h:
            lib.tc_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def tc_comm_create(uid: bytes, world: int, rank: int, device: int) -> Comm:
    buf = (ctypes.c_uint8 * 128)(*uid)
    h = ctypes.c_void_p()
    check(lib.tc_comm_create(buf, int(world), int(rank), int(device), ctypes.byref(h)),
          "tc_comm_create")
    return Comm(h.value)


def comm_from_process_group(device: int, group=None) -> Comm:
    """Bootstrap a tc_comm over an initialised torch.distributed group: rank 0
    makes the NCCL unique id, the group broadcasts it."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    obj = [tc_comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return tc_comm_create(obj[0], world, rank, device)


def tc_comm_wrap(nccl_comm_ptr: int) -> Comm:
    """Wrap a borrowed ncclComm_t (not owned; see include/triadcensus.h)."""
    h = ctypes.c_void_p()
    check(lib.tc_comm_wrap(ctypes.c_void_p(int(nccl_comm_ptr)), ctypes.byref(h)), "tc_comm_wrap")
    return Comm(h.value)


def comm_wrap_process_group(device: int, group=None) -> Comm:
    """Borrow torch's own NCCL communicator of an initialised NCCL process
    group (private API ProcessGroupNCCL._comm_ptr(); version-coupled, so
    comm_from_process_group stays the default)."""
    import torch
    import torch.distributed as dist
    pg = group if group is not None else dist.distributed_c10d._get_default_group()
    dev = torch.device("cuda", device)
    backend = pg._get_backend(dev)
    # make sure torch has created the communicator for this device
    t = torch.zeros(1, device=dev)
    dist.all_reduce(t, group=group)
    return tc_comm_wrap(backend._comm_ptr())


def tc_census_multi(g: Graph, comm: Comm, stream=None) -> list[int]:
    c = (ctypes.c_uint64 * 16)()
    hi = ctypes.c_uint64(0)
    check(lib.tc_census_multi(g.handle, comm.handle, _stream_ptr(stream), c, ctypes.byref(hi)),
          "tc_census_multi")
    return _join003(c, hi.value)


def tc_trim_memory() -> None:
    """Give the default allocator's cached device blocks back to the driver
    (include/triadcensus.h tc_trim_memory)."""
    check(lib.tc_trim_memory(), "tc_trim_memory")


def census(n: int, src, dst, device: int = 0) -> list[int]:
    """One-shot: build the graph, run the census, free the graph."""
    g = tc_graph_create(n, src, dst, device=device)
    try:
        return tc_census(g)
    finally:
        g.close()


def tc_read_arcs(path: str, fmt: str = "auto", index_base=None):
    """Read a Pajek (.net) or SNAP edge-list file with the library's native
    reader.  Returns (n, src, dst) with 0-based uint32 numpy arrays."""
    f = {"auto": 0, "pajek": 1, "edgelist": 2}[fmt]
    b = -1 if index_base is None else int(index_base)
    n = ctypes.c_uint64(0)
    m = ctypes.c_uint64(0)
    ps, pd = _lib.u32p(), _lib.u32p()
    check(lib.tc_read_arcs(str(path).encode(), f, b, ctypes.byref(n), ctypes.byref(ps),
                           ctypes.byref(pd), ctypes.byref(m)), "tc_read_arcs")
    try:
        k = int(m.value)
        src = np.ctypeslib.as_array(ps, shape=(k,)).copy() if k else np.zeros(0, np.uint32)
        dst = np.ctypeslib.as_array(pd, shape=(k,)).copy() if k else np.zeros(0, np.uint32)
    finally:
        lib.tc_free_arcs(ps)
        lib.tc_free_arcs(pd)
    return int(n.value), src, dst


def census_file(path: str, fmt: str = "auto", index_base=None, device: int = 0):
    """Read a graph file, build, census; returns (counts, timing breakdown in
    seconds) with the phases of the paper's tables:
    read graph, CSR build (neighbour sets), plan (task queues), census."""
    import time
    torch = _torch()
    t0 = time.perf_counter()
    n, src, dst = tc_read_arcs(path, fmt, index_base)
    t1 = time.perf_counter()
    g = tc_graph_create(n, src, dst, device=device)
    torch.cuda.synchronize(device)
    t2 = time.perf_counter()
    g.profile(True)
    counts = tc_census(g)
    t3 = time.perf_counter()
    prof = g.profile_get()
    g.close()
    timing = {"read_graph": t1 - t0, "build_csr": t2 - t1, "build_csr_device": prof["build_ms"] / 1e3,
              "plan": prof["plan_ms"] / 1e3, "census_kernels": prof["census_ms"] / 1e3,
              "census_call": t3 - t2, "total": t3 - t0}
    # the paper's phase names (Table: read, neighbour sets, task
    # queues, census) for the same numbers
    timing["paper_phases"] = {"read_graph": timing["read_graph"],
                              "neighbour_sets": timing["build_csr"],
                              "task_queues": timing["plan"],
                              "census": timing["census_call"] - timing["plan"]}
    return counts, timing
