"""Quick per-phase timing of the CUDA path on one config (dev tool)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
import paper_1603_02655_b200 as tcb

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
# arcs cached in /tmp for the duration of one gpurun call (A/B runs of many
# library variants regenerate nothing)
cache = "/tmp/tc_arcs_%s.npz" % name
from synth.device import DEVICE_CONFIGS, make_device_config
if name in DEVICE_CONFIGS:
    n_, s_, d_, _ = make_device_config(name, torch.device("cuda", 0))
    a = synth.Arcs(n_, None, None, {"config": name})
elif os.path.exists(cache):
    z = np.load(cache)
    a = synth.Arcs(int(z["n"]), z["src"], z["dst"], {"config": name})
else:
    a = synth.make_config(name)
    np.savez(cache, n=a.n, src=a.src, dst=a.dst)
if a.src is None:
    s, d = s_, d_
else:
    s = torch.from_numpy(a.src.view('int32')).cuda()
    d = torch.from_numpy(a.dst.view('int32')).cuda()
for rep in range(2 if name in DEVICE_CONFIGS else 4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    g = tcb.tc_graph_create(a.n, s, d, use_torch_allocator=os.environ.get("TC_TORCH_ALLOC", "1") == "1")
    torch.cuda.synchronize(); t1 = time.perf_counter()
    g.profile(True)
    c = g.census()
    t2 = time.perf_counter()
    p = g.profile_get()
    print(name, "build %.3f ms (ev %.3f)  census %.3f ms  plan %.3f  kernels %s  items %s work %s" % (
        (t1 - t0) * 1e3, p["build_ms"], (t2 - t1) * 1e3, p["plan_ms"],
        ["%.3f" % x for x in p["kernel_ms"][:3]], p["bin_items"][:3], p["bin_work"][:3]))
    g.close()
print(c)
