"""synth -- seeded synthetic digraphs shaped like the paper's workloads.

The one module both sides (the CUDA path and the CPU oracle) may use.  It
holds none of the census arithmetic: it only draws arcs.  Every generator
returns ``Arcs(n, src, dst, meta)`` with uint32 endpoint arrays in shuffled
order, possibly containing self-loops and duplicate arcs (sanitising them is
step a1 of the method, done by the consumer).  Randomness comes from numpy's
counter-based Philox generator keyed by the seed, so the arcs are identical
on every machine with this image.  See DESIGN.md "Input recipe".
"""
from .generators import (Arcs, CONFIGS, make_config, erdos_renyi, rmat, patents_like,
                         livejournal_like, random_digraph, out_star, in_star, mutual_star,
                         directed_cycle, transitive_tournament, complete_mutual,
                         complete_bipartite, single_triad, REPRESENTATIVES, relabel)

__all__ = ["Arcs", "CONFIGS", "make_config", "erdos_renyi", "rmat", "patents_like",
           "livejournal_like", "random_digraph", "out_star", "in_star", "mutual_star",
           "directed_cycle", "transitive_tournament", "complete_mutual",
           "complete_bipartite", "single_triad", "REPRESENTATIVES", "relabel"]
