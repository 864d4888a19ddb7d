"""Writes tests/golden/census_<CFG>.json: the full 16-class census of each
synthetic config, computed ONLY by the CPU oracle (oracle/bm_oracle.c).

    python tests/golden/make_golden.py C1 C2 C3

The GPU parity tests compare the CUDA path against these files element by
element; the oracle's own -m "not gpu" pins (brute force, networkx, closed
forms, the linear census identities in tests/test_oracle_identities.py)
check the same files independently.  Nothing here touches the CUDA path.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import oracle  # noqa: E402
import synth  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main(names):
    for name in names:
        a = synth.make_config(name)
        t0 = time.time()
        g = oracle.Graph(a.n, a.src, a.dst)
        c = g.census()
        st = g.stats()
        rec = {"config": name, "label": a.meta["label"], "generator": a.meta["generator"],
               "seed": a.meta["seed"], "n": a.n, "m_drawn": a.m, "stats": st,
               "census": [str(x) for x in c], "classes": list(oracle.CLASS_NAMES),
               "oracle_seconds": round(time.time() - t0, 2),
               "written_by": "tests/golden/make_golden.py (oracle/ only)"}
        with open(os.path.join(HERE, "census_%s.json" % name), "w") as f:
            json.dump(rec, f, indent=1)
        print(name, rec["oracle_seconds"], "s", c)


if __name__ == "__main__":
    main(sys.argv[1:] or ["C1", "C2", "C3"])
