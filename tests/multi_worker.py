"""Rank worker of tests/test_multi_gloo.py, started by the same one-node
launcher as `bench.py --gpus N` (paper_1603_02655_b200/launch.py), on the
gloo backend: every rank computes the library's shard cut (the host rule
tc_shard_bounds_host applies on the device) over the numpy-restated kernel
work (tests/shard_work.py), censuses its canonical-dyad range with the
oracle, the partial counts meet in one all_reduce, and rank 0 prints one
JSON line (bounds, reduced census, single-process census)."""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    scale, ef, seed = (int(x) for x in sys.argv[1:4])
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    try:
        import oracle
        import paper_1603_02655_b200 as tcb
        import synth
        from shard_work import dyad_work
        a = synth.rmat(scale=scale, edge_factor=ef, seed=seed)
        g = oracle.Graph(a.n, a.src, a.dst)
        _, cost = dyad_work(a.n, a.src, a.dst)
        bounds = tcb.tc_shard_bounds_host(cost, world, kappa=8)
        part = g.census_range(bounds[rank], bounds[rank + 1])
        # uint64 partials as two 32-bit halves so int64 sums cannot overflow
        t = torch.tensor([x & 0xffffffff for x in part] + [x >> 32 for x in part],
                         dtype=torch.int64)
        dist.all_reduce(t)
        tot = [int(t[i]) + (int(t[16 + i]) << 32) for i in range(16)]
        full = tcb.tc_close_census(a.n, tot)
        allb = [None] * world
        dist.all_gather_object(allb, bounds)
        if rank == 0:
            print(json.dumps({"world": world, "env_world": int(os.environ["WORLD_SIZE"]),
                              "bounds": allb, "census": [str(x) for x in full],
                              "single": [str(x) for x in g.census()]}), flush=True)
    finally:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
