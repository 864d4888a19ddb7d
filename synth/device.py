"""Device-side (torch, CUDA) seeded R-MAT generator for the configurations too
large to draw with numpy on the host (no census arithmetic here).

* C5  R-MAT scale 26, edge factor 16 (1,073,741,824 drawn arcs), Graph500
      probabilities (a,b,c,d) = (.57,.19,.19,.05), seed 26.
* C5p the same recipe at scale 24 (268,435,456 drawn arcs), seed 24: the
      C5 proxy the GPU tests run (census in seconds).

Same recipe as synth.rmat (one uniform draw per level picks the quadrant),
then a seeded vertex permutation and a shuffle of the arc order; loops and
duplicates stay in the list (step a1 drops them).  Randomness: torch's
counter-based Philox CUDA generator seeded with `seed`, so the arcs are a
deterministic function of (seed, scale, edge factor) on this image -- but
they differ from what numpy's Philox would draw, so these graphs exist only
on the device.  Parity at this size comes from the O(n+m) census identities
(tests/test_gpu_large.py), not from the oracle.
"""
from __future__ import annotations

DEVICE_CONFIGS = {
    "C5": dict(scale=26, edge_factor=16, seed=26,
               label="R-MAT scale 26 edge factor 16 (Graph500 a,b,c,d=.57,.19,.19,.05), "
                     "device-generated"),
    "C5p": dict(scale=24, edge_factor=16, seed=24,
                label="R-MAT scale 24 edge factor 16 (C5 proxy), device-generated"),
}


def rmat_device(scale: int, edge_factor: int, seed: int, device, a=0.57, b=0.19, c=0.19):
    """Returns (n, src, dst): int32 CUDA tensors of the drawn arcs (uint32 ids
    in int32 storage; scale <= 30)."""
    import torch
    assert scale <= 30
    n = 1 << scale
    count = edge_factor * n
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    src = torch.zeros(count, dtype=torch.int32, device=device)
    dst = torch.zeros(count, dtype=torch.int32, device=device)
    ab, abc = a + b, a + b + c
    for level in range(scale):
        r = torch.rand(count, generator=g, device=device, dtype=torch.float32)
        bit = 1 << (scale - 1 - level)
        src |= (r >= ab).to(torch.int32) * bit
        dst |= (((r >= a) & (r < ab)) | (r >= abc)).to(torch.int32) * bit
        del r
    perm = torch.randperm(n, generator=g, device=device, dtype=torch.int32)
    src = perm[src.long()]
    dst = perm[dst.long()]
    del perm
    order = torch.randperm(count, generator=g, device=device)
    src = src[order]
    dst = dst[order]
    del order
    return n, src, dst


def make_device_config(name: str, device):
    cfg = DEVICE_CONFIGS[name]
    n, s, d = rmat_device(cfg["scale"], cfg["edge_factor"], cfg["seed"], device)
    meta = {"config": name, "label": cfg["label"], "generator": "rmat_device",
            "seed": cfg["seed"], "scale": cfg["scale"], "edge_factor": cfg["edge_factor"]}
    return n, s, d, meta
