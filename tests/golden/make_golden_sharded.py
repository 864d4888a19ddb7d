"""Writes tests/golden/census_<CFG>.json for configs too big for one oracle
run (C4: ~69M arcs, hours single-threaded), computed ONLY by the CPU oracle.

    python tests/golden/make_golden_sharded.py C4 [--procs K] [--chunks R]

The canonical dyads, in the algorithm's own (u asc, v asc) order,
are cut into R contiguous ranges of about equal oracle cost (the paper's
uniform work unit |N[u]| + |N[v]| per dyad, plus a constant), and
K forked host processes run ``og_census_range`` (Fig. P:269-309 restricted to
a dyad range) on them, each oracle single-threaded.  Partials over any
partition of the dyads sum to the full census; class 003 is then
C(n,3) - sum with Python integers.  Finished ranges are cached in
``census_<CFG>.partials.jsonl`` beside the output, so an interrupted run
resumes.  The per-range partials are stored in the golden file too: the GPU
tests compare ``tc_census_range`` with them range by range.

Nothing here touches the CUDA path: inputs come from ``synth/`` and every
number from ``oracle/``.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import oracle  # noqa: E402
import synth  # noqa: E402
from oracle import sharded  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--procs", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--chunks", type=int, default=256)
    ap.add_argument("--reverse", action="store_true",
                    help="run the uncached ranges last-first (a second host sharing the work)")
    ap.add_argument("--cache", default=None,
                    help="append finished ranges here (default: beside the output); "
                         "ranges cached in either file are skipped")
    ap.add_argument("--note", default=None, help="free-text provenance note stored in the file")
    ap.add_argument("--no-write", action="store_true",
                    help="only fill the cache (another host writes the golden)")
    args = ap.parse_args()
    for name in args.configs:
        t_start = time.time()
        a = synth.make_config(name)
        g = oracle.Graph(a.n, a.src, a.dst)
        st = g.stats()
        ranges = sharded.equal_cost_ranges(g.dyad_costs(), args.chunks)
        default_cache = os.path.join(HERE, "census_%s.partials.jsonl" % name)
        cache = args.cache or default_cache
        done = {}
        for c in {default_cache, cache}:
            if os.path.exists(c):
                with open(c) as f:
                    for line in f:
                        r = json.loads(line)
                        done[(r["begin"], r["end"])] = r
        todo = [r for r in ranges if r not in done]
        if args.reverse:
            todo = todo[::-1]
        print("%s: n=%d m=%d D=%d, %d ranges (%d cached), %d procs"
              % (name, a.n, st["m"], st["dyads"], len(ranges), len(ranges) - len(todo), args.procs),
              flush=True)
        cpu_s = sum(r["seconds"] for r in done.values())
        with open(cache, "a") as f:
            def record(b, e, part, sec):
                rec = {"begin": b, "end": e, "partial": [str(x) for x in part],
                       "seconds": round(sec, 2)}
                f.write(json.dumps(rec) + "\n")
                f.flush()
                done[(b, e)] = rec
                print("  [%d/%d] %d..%d %.1fs" % (len(done), len(ranges), b, e, sec), flush=True)
            _, _, cpu = sharded.census_ranges(g, todo, args.procs, record)
        cpu_s += cpu
        if args.no_write:
            continue
        parts = [[int(x) for x in done[r]["partial"]] for r in ranges]
        total = sharded.close(a.n, parts)
        rec = {"config": name, "label": a.meta["label"], "generator": a.meta["generator"],
               "seed": a.meta["seed"], "n": a.n, "m_drawn": a.m, "stats": st,
               "census": [str(x) for x in total], "classes": list(oracle.CLASS_NAMES),
               "oracle_seconds": round(time.time() - t_start, 2),
               "oracle_cpu_seconds": round(cpu_s, 2),
               "sharding": {"ranges": len(ranges), "procs": args.procs, "kappa": sharded.KAPPA,
                            "cost": "d_u + d_v + kappa per canonical dyad (P:1693)"},
               "note": args.note,
               "range_partials": [{"begin": b, "end": e, "partial": [str(x) for x in p]}
                                  for (b, e), p in zip(ranges, parts)],
               "written_by": "tests/golden/make_golden_sharded.py (oracle/ only)"}
        with open(os.path.join(HERE, "census_%s.json" % name), "w") as f:
            json.dump(rec, f, indent=1)
        print(name, rec["oracle_seconds"], "s wall,", rec["oracle_cpu_seconds"], "s cpu", total)


if __name__ == "__main__":
    main()
