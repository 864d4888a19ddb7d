"""N > 1 path on CPU (gloo, world_size 2 and 3): every rank computes the
library's degree-balanced shard cut (tc_shard_bounds_host, the rule the
device applies in tc_census_multi), censuses its canonical-dyad range with
the oracle, the partial counts meet in one all_reduce, and the closed census
equals the single-process census.  No GPU needed."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import paper_1603_02655_b200 as tcb
        import synth
        a = synth.rmat(**cfg)
        g = oracle.Graph(a.n, a.src, a.dst)
        bounds = tcb.tc_shard_bounds_host(g.dyad_costs(), world, kappa=8)
        part = g.census_range(bounds[rank], bounds[rank + 1])
        # uint64 partials as two 32-bit halves so int64 sums cannot overflow
        t = torch.tensor([x & 0xffffffff for x in part] + [x >> 32 for x in part],
                         dtype=torch.int64)
        dist.all_reduce(t)
        tot = [int(t[i]) + (int(t[16 + i]) << 32) for i in range(16)]
        full = tcb.tc_close_census(a.n, tot)
        q.put((rank, bounds, full, g.census() if rank == 0 else None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_census_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    cfg = dict(scale=11, edge_factor=8, seed=5)
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    bounds = res[0][1]
    assert all(r[1] == bounds for r in res)          # same cut on every rank
    assert bounds[0] == 0 and bounds == sorted(bounds)
    single = res[0][3]
    for r in res:
        assert r[2] == single                        # identical full census everywhere
