"""N > 1 path on CPU (gloo, world_size 2 and 3), launched exactly as
`bench.py --gpus N` launches its ranks (paper_1603_02655_b200/launch.py:
torch.distributed.run, rendezvous on 127.0.0.1): every rank computes the
library's work-balanced shard cut, censuses its canonical-dyad range with
the oracle, the partial counts meet in one all_reduce, and the closed census
equals the single-process census (tests/multi_worker.py).  No GPU needed."""
import json
import os

import pytest

from paper_1603_02655_b200 import launch

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_census_gloo(world):
    rc, out = launch.spawn_local(world, os.path.join(HERE, "multi_worker.py"), ["11", "8", "5"],
                                 capture=True, timeout=600)
    assert rc == 0
    lines = [json.loads(x) for x in out.splitlines() if x.startswith("{")]
    assert len(lines) == 1                              # rank 0 alone prints
    r = lines[0]
    assert r["world"] == r["env_world"] == world
    bounds = r["bounds"][0]
    assert all(b == bounds for b in r["bounds"])       # same cut on every rank
    assert bounds[0] == 0 and bounds == sorted(bounds) and len(bounds) == world + 1
    assert r["census"] == r["single"]                   # identical full census


def test_bench_refuses_missing_gpus():
    # `bench.py --gpus N` with fewer than N GPUs exits non-zero instead of
    # running on one GPU (round 1 silently ran one)
    import subprocess
    import sys
    import torch
    n = max(2, torch.cuda.device_count() + 1)
    p = subprocess.run([sys.executable, os.path.join(os.path.dirname(HERE), "bench.py"),
                        "--gpus", str(n), "--steps", "1", "--warmup", "1"],
                       capture_output=True, text=True, timeout=300,
                       env={k: v for k, v in os.environ.items() if k != "WORLD_SIZE"})
    assert p.returncode != 0
    assert "CUDA device" in p.stderr
