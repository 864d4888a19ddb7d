"""dev: small censuses + task queues for compute-sanitizer (memcheck/racecheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import synth
import paper_1603_02655_b200 as tcb

cases = [synth.make_config("C1"), synth.random_digraph(300, 0.05, seed=7, loops=True, dups=9),
         synth.out_star(3000, 3500), synth.complete_mutual(40), synth.rmat(12, 8, seed=3),
         synth.livejournal_like(n=20000, m_target=150000, scale=15, seed=2)]
for a in cases:
    g = tcb.tc_graph_create(a.n, a.src, a.dst)
    c = g.census()
    D = g.stats()["dyads"]
    p = tcb.tc_census_range(g, D // 3, 2 * D // 3)
    c64 = tcb.tc_census64(g)
    for st in ("uniform", "nonuniform"):
        tcb.tc_task_queues(g, st, 1000)
    g.close()
    print(a.meta.get("name", "?"), sum(c))
print("sanitize run done")
