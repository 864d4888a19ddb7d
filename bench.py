#!/usr/bin/env python
"""bench.py -- directed triad census throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl reference]

One step = one pass of the whole hot path (SURVEY.md section 8(a) rows
a1..a5) over the synthetic workload: GPU CSR build from the device-resident
arc list (a1), degree-binned plan (a2), merge/classify kernels with the
block histogram (a3+a4), closing (a5).  `value` = arcs processed by all ranks
per second, timed with CUDA events on the launch stream, max over ranks.
`e2e` = the same through the C ABI with HOST (pinned) arc buffers, the H2D
copy and the result D2H inside the timed region.

N > 1: `bench.py --gpus N` starts N ranks itself (torch.distributed.run on
127.0.0.1) unless it already runs under a launcher (WORLD_SIZE set).  Every
rank holds the replicated CSR, computes its work-balanced canonical-dyad
shard, and the 16 partial counts meet in one NCCL allreduce
(tc_census_multi) -- strong scaling of one census.

--impl reference: the CPU oracle (oracle/, plain single-threaded C) on one
pinned host core; its K steps are K equal-cost canonical-dyad ranges that
cover the census once, so the line is one measured full census; rank 0 only.
cpu_baseline (our arm, rank 0, N = 1): the same oracle over the whole census
in forked single-threaded processes on the host's cores (bounded wall time).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from synth.device import DEVICE_CONFIGS, make_device_config  # noqa: E402

METRIC = "triad-census arcs/sec at 1/2/4/8 B200 (Patents-shaped); % HBM roofline"
UNIT = "arcs/s"
FALLBACK_HBM_GBS = 6650.0   # /opt/skills/guides/B200_PROFILING.md fallback


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default="C3")
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--mode", default="16", choices=["16", "64"],
                   help="16-class isomorphic census (default) or the 64-type census (f1)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--alloc", default="pool", choices=["pool", "torch"],
                   help="device allocator of the library: its own stream-ordered pool "
                        "(default) or torch's caching allocator through the Python hook")
    p.add_argument("--cpu-seconds", type=float, default=25.0,
                   help="wall-time budget of the cpu_baseline oracle run (full census if it fits)")
    return p.parse_args()


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        # one long-lived nvidia-smi sampling every 50 ms (our own child process)
        try:
            self._p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" +
                                        self.FIELDS, "--format=csv,noheader,nounits",
                                        "-lms", "50"], stdout=subprocess.PIPE,
                                       stderr=subprocess.DEVNULL, text=True)
        except Exception:
            return
        for line in self._p.stdout:
            f = [x.strip() for x in line.strip().split(",")]
            if len(f) >= 7:
                self.samples.append(f)
            if self._stop.is_set():
                break

    def __enter__(self):
        self._p = None
        self._t.start()
        time.sleep(0.3)       # let the sampler start before the timed region
        return self

    def __exit__(self, *a):
        time.sleep(0.1)
        self._stop.set()
        if self._p is not None:
            self._p.terminate()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"],
                    "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if s[2 + i].lower().startswith("active")})
        util = [float(s[6]) for s in self.samples if s[6].replace(".", "").isdigit()]
        loaded = [c for c, u in zip(sm, util) if u > 0] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# CPU oracle baseline (rank 0, N = 1; and --impl reference)
# ---------------------------------------------------------------------------
def host_cpu():
    """lscpu model, logical CPUs, the affinity set."""
    model = None
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True,
                                   timeout=10).stdout.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
    except Exception:
        pass
    aff = sorted(os.sched_getaffinity(0))
    return {"model": model, "logical_cpus": os.cpu_count(), "affinity": len(aff),
            "affinity_first": aff[0] if aff else None}


def oracle_full_census(a, procs, budget_s=None):
    """The oracle (as it stands) over the whole census: its graph build
    (a1) once, then og_census_range over equal-cost canonical-dyad ranges in
    `procs` forked single-threaded processes (oracle/sharded.py), summed and
    closed.  If a calibration says one full pass would exceed `budget_s`
    of wall time, only a systematic sample of the ranges (every j-th) runs
    and the rate is extrapolated in the paper's uniform work units."""
    import oracle
    from oracle import sharded
    t0 = time.perf_counter()
    g = oracle.Graph(a.n, a.src, a.dst)
    t_build = time.perf_counter() - t0
    cost = g.dyad_costs()
    chunks = max(8 * procs, 64)
    ranges = sharded.equal_cost_ranges(cost, chunks)
    pre = np.concatenate([[0], np.cumsum(cost.astype(np.float64) + sharded.KAPPA)])
    units = [pre[e] - pre[b] for b, e in ranges]
    sample = list(range(len(ranges)))
    if budget_s is not None:
        # calibrate on one middle range, single process
        mid = len(ranges) // 2
        _, _, c1 = sharded.census_ranges(g, [ranges[mid]], 1)
        est_wall = c1 * len(ranges) / max(procs, 1)
        if est_wall > budget_s:
            keep = max(procs, int(len(ranges) * budget_s / est_wall))
            step = max(1, len(ranges) // keep)
            sample = list(range(step // 2, len(ranges), step))
    parts, wall, cpu = sharded.census_ranges(g, [ranges[i] for i in sample], procs)
    full = len(sample) == len(ranges)
    frac = sum(units[i] for i in sample) / pre[-1]
    census = sharded.close(a.n, [parts[r] for r in ranges]) if full else None
    t_census = wall / frac
    return {"value": a.m / (t_build + t_census), "t_build_s": t_build, "t_census_s": t_census,
            "wall_s": wall, "cpu_s": cpu, "procs": procs, "ranges": len(ranges),
            "ranges_run": len(sample), "work_frac": frac, "full": full, "census": census}


def golden_census(name):
    p = os.path.join(ROOT, "tests", "golden", "census_%s.json" % name)
    if os.path.exists(p):
        return [int(x) for x in json.load(open(p))["census"]]
    return None


def run_reference(args):
    """The reference arm: the CPU oracle (oracle/, plain single-threaded C)
    on one pinned host core.  The K timed steps are K contiguous equal-cost
    canonical-dyad ranges that together cover [0, D), each one
    og_census_range call: their sum is one MEASURED full census (after the
    oracle's own graph build, timed once and charged to the steps), summed
    and closed, and checked against tests/golden/ when present.  The W
    warm-up steps re-run the first W ranges (untimed)."""
    rank, _, world = env_rank()
    if rank != 0:
        return 0
    if args.config in DEVICE_CONFIGS:
        print(json.dumps({"impl": "reference", "unavailable": "config %s is drawn on the GPU "
                          "(synth/device.py); the CPU oracle runs on host-drawn configs only"
                          % args.config}), flush=True)
        return 0
    import oracle
    from oracle import sharded
    cpu = host_cpu()
    if cpu["affinity_first"] is not None:
        os.sched_setaffinity(0, {cpu["affinity_first"]})     # one pinned core
    a = synth.make_config(args.config)
    steps = max(args.steps, 1)
    t0 = time.perf_counter()
    g = oracle.Graph(a.n, a.src, a.dst)
    t_build = time.perf_counter() - t0
    st = g.stats()
    ranges = sharded.equal_cost_ranges(g.dyad_costs(), steps)
    for b, e in ranges[:args.warmup]:
        g.census_range(b, e)
    times, parts = [], []
    for b, e in ranges:
        t0 = time.perf_counter()
        parts.append(g.census_range(b, e))
        times.append(time.perf_counter() - t0)
    census = sharded.close(a.n, parts)
    gold = golden_census(args.config)
    total = t_build + sum(times)
    value = a.m / total
    k = len(ranges)
    sample = ("one full census measured: the oracle's graph build (%.2f s) + %d contiguous "
              "equal-cost canonical-dyad ranges covering [0, D) (one og_census_range call per "
              "step, %.2f s in total), single-threaded on one pinned core (%s)" %
              (t_build, k, sum(times), cpu["model"]))
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": world, "steps": k, "warmup": args.warmup,
            "ms_per_step": total * 1e3 / k, "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": bench_config(a, st, world),
            "step_s": [round(x, 4) for x in times], "oracle_build_s": t_build,
            "census_matches_golden": (census == gold) if gold else None,
            "census": [str(x) for x in census],
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": sample, "host": cpu},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def bench_config(a, stats, world, m_drawn=None):
    """The workload description both arms print unchanged (config)."""
    m = a.m if m_drawn is None else m_drawn
    c = {"workload": "%s: %s" % (a.meta.get("config"), a.meta.get("label")),
         "generator": a.meta.get("generator"), "seed": a.meta.get("seed"), "n": a.n,
         "m_drawn": m,
         "l2": "%s (arcs %.0f MB, sort keys + scratch %.0f MB); the GPU arm writes a 512 MB "
               "buffer (L2 flush) before every timed step"
               % ("inputs > L2" if 8 * m > 126e6 else "inputs fit in L2", 8 * m / 1e6,
                  16 * m / 1e6),
         "parallelism": ("dp%d: replicated CSR, work-balanced canonical-dyad shards, one NCCL "
                         "allreduce of 16 counts" % world) if world > 1 else "single GPU"}
    if stats:
        c.update({"m": stats["m"], "dyads": stats["dyads"], "sum_deg_sq": stats["sum_deg_sq"],
                  "max_degree": stats["max_degree"]})
    return c


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args):
    import torch
    rank, local, world = env_rank()
    if world != args.gpus:
        raise SystemExit("bench.py: --gpus %d but WORLD_SIZE %d" % (args.gpus, world))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1603_02655_b200 as tcb

    dev = torch.device("cuda", local)
    if args.config in DEVICE_CONFIGS:
        # too large for the host generator: drawn on the device (synth/device.py)
        n_, s_dev, d_dev, meta_ = make_device_config(args.config, dev)
        a = synth.Arcs(n_, None, None, meta_)
        a_m = int(s_dev.numel())
        # the draw's temporaries stay in torch's cache otherwise; the library
        # allocates from its own pool (C5 needs ~130 GB of it)
        torch.cuda.synchronize(dev)
        torch.cuda.empty_cache()
    else:
        a = synth.make_config(args.config)
        a_m = a.m
        s_dev = torch.from_numpy(a.src.view(np.int32)).to(dev)
        d_dev = torch.from_numpy(a.dst.view(np.int32)).to(dev)
    stream = torch.cuda.current_stream(dev)
    comm = tcb.comm_from_process_group(local) if world > 1 else None
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)  # > 126 MB L2

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def one_step(src, dst, profile=False, done=None):
        # done(): called as soon as the census is on the host (the end of a
        # step: a1..a5); the profile read-out and the graph's release follow
        # the library's own stream-ordered pool (the ABI's default allocator)
        # rather than torch's caching allocator through the Python hook: no
        # Python callback per device allocation on the build's critical path
        g = tcb.tc_graph_create(a.n, src, dst, device=local, stream=stream,
                                use_torch_allocator=args.alloc == "torch")
        launches = g.launches()
        if profile:
            g.profile(True)
        if args.mode == "64":
            counts = tcb.tc_census64(g, stream)
        else:
            counts = tcb.tc_census_multi(g, comm, stream) if comm else tcb.tc_census(g, stream)
        if done is not None:
            done()
        launches += g.launches()
        prof = g.profile_get() if profile else None
        stats = g.stats()
        g.close()
        return counts, launches, prof, stats

    # warm-up
    ref_counts = None
    for _ in range(args.warmup):
        ref_counts, _, _, stats = one_step(s_dev, d_dev)
    barrier()

    # timed region: device-resident arcs
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    launches_total = 0
    profs = []
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.fill_(i)                       # L2 flush between steps (outside timing)
            barrier()
            ev[i][0].record(stream)
            counts, nl, prof, stats = one_step(s_dev, d_dev, profile=True,
                                               done=lambda e=ev[i][1]: e.record(stream))
            launches_total += nl
            profs.append(prof)
            if ref_counts is not None:
                assert counts == ref_counts, "census changed between steps"
            ref_counts = counts
        barrier()
    step_ms = [e0.elapsed_time(e1) for e0, e1 in ev]
    total_ms = sum(step_ms)
    if dist is not None:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps

    # e2e: host (pinned) arcs through the C ABI, H2D + D2H inside the region
    if a.src is None:
        s_host = torch.empty(a_m, dtype=torch.int32, pin_memory=True)
        d_host = torch.empty(a_m, dtype=torch.int32, pin_memory=True)
        s_host.copy_(s_dev)
        d_host.copy_(d_dev)
    else:
        s_host = torch.from_numpy(a.src.view(np.int32)).pin_memory()
        d_host = torch.from_numpy(a.dst.view(np.int32)).pin_memory()
    s_np = s_host.numpy().view(np.uint32)
    d_np = d_host.numpy().view(np.uint32)
    one_step(s_np, d_np)          # warm
    e2e_ms = []
    for i in range(args.steps):
        flush.fill_(i)
        barrier()
        t0 = time.perf_counter()
        t1 = []

        def stop():
            torch.cuda.synchronize()
            t1.append(time.perf_counter())
        counts, _, _, _ = one_step(s_np, d_np, done=stop)
        e2e_ms.append((t1[0] - t0) * 1e3)
        assert counts == ref_counts
    e2e_total = sum(e2e_ms)
    if dist is not None:
        t = torch.tensor([e2e_total], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_total = float(t.item())

    if rank != 0:
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    # roofline of the dominant kernel: the bin with more work (the bins run
    # side by side; the warp bin's time runs from the bins' start to its end)
    hbm, peak_src = peaks()
    kms = np.array([p["kernel_ms"][:2] for p in profs])
    avg_k = kms.mean(axis=0)
    dom = int(np.argmax([profs[-1]["bin_work"][0], profs[-1]["bin_work"][1]]))
    # dyads and work per bin: thread bin = items[0]/work[0], warp bin = items[2]/work[1]
    bin_dyads = [profs[-1]["bin_items"][0], profs[-1]["bin_items"][2]]
    bin_work = [profs[-1]["bin_work"][0], profs[-1]["bin_work"][1]]
    items = bin_dyads[dom]
    work = bin_work[dom]
    # 4(du+dv)+24 B per merged dyad; the warp bin's skewed-pair
    # dyads (searched, not merged) count the entries they read instead
    sp_dyads = int(profs[-1]["bin_items"][3]) if dom == 1 else 0
    sp_c = int(profs[-1].get("sparse_sum_c", 0)) if dom == 1 else 0
    sp_units = int(profs[-1].get("sparse_units", 0)) if dom == 1 else 0
    bytes_merge_equiv = 4.0 * work + 24.0 * items
    bytes_alg = 4.0 * (work - sp_c) + 24.0 * (items - sp_dyads) + 4.0 * sp_units + 24.0 * sp_dyads
    achieved = bytes_alg / (avg_k[dom] * 1e-3) / 1e9
    names = ["k_census_thread", "k_census_warp"]
    if args.mode == "64":
        names = ["k_census_thread64", "k_census_warp64"]
    traffic, traffic_src = None, None
    tp = os.path.join(ROOT, "profiles", "traffic_%s.json" % args.config)
    if os.path.exists(tp):
        tr = json.load(open(tp))
        traffic = tr.get(names[dom])
        traffic_src = ("profiles/traffic_%s.json: dram__bytes_read.sum + dram__bytes_write.sum "
                       "per launch from a committed ncu --set full capture (%s), not measured in "
                       "this run" % (args.config, tr.get("_source", "see profiles/")))
    # bytes the dominant kernel's merges touch (merge trips over the entries
    # w > u, reading 21) + the per-dyad 24 B -- below B_alg
    trips = int(profs[-1]["bin_work"][2 + dom])
    touched = 4.0 * (trips + (sp_units if dom == 1 else 0)) + 24.0 * items
    # a1 build: compulsory bytes (read the arcs once, write the CSR, the five
    # dyad arrays, off and ups) and the sort traffic of the passes the build
    # reports it ran (tc_profile.build_sort)
    passes_m, passes_d, row_keys, huge_kp = profs[-1]["build_sort"]
    m_, d_ = stats["m_in"], stats["dyads"]
    compulsory = 8.0 * m_ + 4.0 * (2 * d_ + a.n) + 20.0 * d_ + 8.0 * a.n
    sort_bytes = 24.0 * (passes_m * m_ + passes_d * d_ + huge_kp) + 16.0 * row_keys
    census_ms = float(np.mean([p["census_ms"] for p in profs]))
    plan_ms = float(np.mean([p["plan_ms"] for p in profs]))
    build_ms = float(np.mean([p["build_ms"] for p in profs]))
    sp_all = (int(profs[-1].get("sparse_sum_c", 0)), int(profs[-1].get("sparse_units", 0)))
    sum_all_bins_bytes = 4.0 * (sum(bin_work) - sp_all[0] + sp_all[1]) + 24.0 * sum(bin_dyads)
    m_arcs = a_m
    line = {"metric": METRIC, "value": m_arcs * args.steps / (total_ms * 1e-3), "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": bench_config(a, stats, world, a_m),
            "step": "a1 build from device arcs + a2 plan + a3/a4 kernels + a5 closing",
            "census_mode": "64-type (f1)" if args.mode == "64" else "16-class",
            "phases_ms": {"build": build_ms, "plan": plan_ms, "census_kernels": census_ms,
                          "bin_kernels": [float(x) for x in avg_k],
                          "census_arcs_per_s": m_arcs / ((plan_ms + census_ms) * 1e-3)},
            "work": {"bin_dyads": [int(x) for x in bin_dyads],
                     "bin_sum_c": [int(x) for x in bin_work],
                     "bin_merge_trips": [int(profs[-1]["bin_work"][2]),
                                         int(profs[-1]["bin_work"][3])]},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": traffic, "traffic_source": traffic_src,
                         "kernel": names[dom],
                         "bytes_alg_per_launch": bytes_alg,
                         "bytes_alg_model": "SURVEY 8(d) B-M model: 4 (d_u + d_v) + 24 B per "
                                            "merged dyad (skewed pairs: 4 (s ceil(log2(l+1)) "
                                            "+ 4) + 24), not the bytes the kernel reads",
                         "touched_bytes_per_launch": touched,
                         "touched_frac": (touched / (avg_k[dom] * 1e-3) / 1e9) / hbm,
                         "dram_frac": ((traffic / (avg_k[dom] * 1e-3) / 1e9) / hbm)
                         if traffic else None,
                         "skewed_pair_dyads": sp_dyads,
                         "merge_equivalent_frac": (bytes_merge_equiv / (avg_k[dom] * 1e-3) / 1e9) / hbm,
                         "peak_source": peak_src,
                         "all_bins_frac": (sum_all_bins_bytes / (census_ms * 1e-3) / 1e9) / hbm},
            "build_roofline": {
                "bound": "hbm", "build_ms": build_ms, "peak": hbm, "unit": "GB/s",
                "compulsory_bytes": compulsory,
                "compulsory_frac": (compulsory / (build_ms * 1e-3) / 1e9) / hbm,
                "sort_passes": {"over_m_keys": passes_m, "over_D_keys": passes_d,
                                "row_network_keys": row_keys,
                                "long_row_lsd_key_passes": huge_kp},
                "sort_bytes": sort_bytes,
                "sort_gbps_if_all_time": sort_bytes / (build_ms * 1e-3) / 1e9,
                "model": "compulsory = 8m (arcs) + 4(2D+n) (adj) + 20D (dyad arrays) + 8n "
                         "(off, ups); sort = 24 B per key per LSD pass (upsweep read + "
                         "downsweep read + write) + 16 B per key left to the per-row "
                         "networks (read + write)"},
            "e2e": {"value": m_arcs * args.steps / (e2e_total * 1e-3), "unit": UNIT,
                    "h2d_bytes_per_step": 8 * a_m, "d2h_bytes_per_step": 320},
            "gpu_launches": launches_total,
            "clocks": clk.summary(),
            "census": [str(x) for x in ref_counts]}
    if world == 1 and not args.no_cpu_baseline and a.src is None:
        line["cpu_baseline"] = None
        line["cpu_baseline_note"] = ("device-generated config: the oracle would need the "
                                     "1e9-arc graph on the host; see the C3 line")
    elif world == 1 and not args.no_cpu_baseline:
        cpu = host_cpu()
        procs = max(1, min(cpu["affinity"], 64))
        r = oracle_full_census(a, procs, budget_s=args.cpu_seconds)
        gold = golden_census(args.config)
        if r["full"]:
            sample = ("one full census measured: oracle graph build (%.2f s, 1 core) + the "
                      "census as %d equal-cost canonical-dyad ranges in %d forked "
                      "single-threaded oracle processes (%.2f s wall, %.1f CPU-s)" %
                      (r["t_build_s"], r["ranges"], procs, r["wall_s"], r["cpu_s"]))
        else:
            sample = ("oracle graph build (%.2f s) + %d of %d equal-cost canonical-dyad ranges "
                      "(a systematic sample, %.1f%% of sum(|N(u)|+|N(v)|)) in %d forked "
                      "processes, extrapolated linearly in that work unit" %
                      (r["t_build_s"], r["ranges_run"], r["ranges"], 100 * r["work_frac"], procs))
        line["cpu_baseline"] = {
            "value": r["value"], "unit": UNIT, "cores": procs, "kind": "oracle",
            "sample": sample, "measured_full_census": r["full"],
            "census_matches_gpu": (r["census"] == ref_counts) if r["full"] else None,
            "census_matches_golden": (r["census"] == gold) if (r["full"] and gold) else None,
            "single_thread_equivalent_s": r["t_build_s"] + r["cpu_s"] / r["work_frac"],
            "host": cpu}
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def spawn_ranks(n):
    """`bench.py --gpus N` without a launcher: start N ranks on this node
    (paper_1603_02655_b200/launch.py: torch.distributed.run, rendezvous on
    127.0.0.1), never fall back to one GPU.  The ranks inherit stdout: rank 0
    prints the JSON line."""
    if not args_impl_is_reference():
        import torch
        if torch.cuda.device_count() < n:
            print("bench.py --gpus %d: only %d CUDA device(s) visible"
                  % (n, torch.cuda.device_count()), file=sys.stderr)
            return 2
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "tc_launch", os.path.join(ROOT, "paper_1603_02655_b200", "launch.py"))
    launch = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(launch)
    return launch.spawn_local(n, os.path.abspath(__file__), sys.argv[1:])


def args_impl_is_reference():
    return "--impl" in sys.argv and sys.argv[sys.argv.index("--impl") + 1:][:1] == ["reference"]


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
