"""Seeded synthetic digraph generators (no census arithmetic here).

Recipes:

* C1  directed Erdos-Renyi G(n=1000, m=8000): 8,000 distinct ordered pairs
      u != v drawn uniformly; seed 1.
* C2  R-MAT scale 16, edge factor 8 (524,288 drawn arcs), Graph500
      probabilities (a,b,c,d) = (.57,.19,.19,.05); loops and duplicates kept
      in the arc list (the CSR builder drops them); seed 16.
* C3  Patents-shaped: lognormal Chung-Lu DAG, n = 3,774,768 and exactly
      m = 16,518,948 distinct arcs (Table).  Vertex weights
      w_i ~ LogNormal(0, 0.92); endpoints drawn proportional to w; arcs
      oriented from the larger to the smaller (pre-permutation) id, as a
      citation points from newer to older; loops dropped and pairs
      deduplicated until exactly m distinct arcs; seed 7.  Calibrated so
      sum_u d_u^2 ~ 7.07e8 against the paper's 704,600,440.
* C4  LiveJournal-shaped social R-MAT: n = 4,847,571, R-MAT scale 23 with
      (.57,.19,.19,.05), ids >= n rejected; every kept base arc is
      reciprocated with probability q = 0.538 (reciprocated-arc fraction
      2q/(1+q) ~ 0.70); drawn until ~69.0M distinct arcs; seed 11.

After drawing, every generator applies a seeded random vertex permutation
(Graph500 practice; the census is invariant under relabelling) and shuffles
the arc order, so the consumer's sort does real work.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class Arcs:
    n: int
    src: np.ndarray  # uint32
    dst: np.ndarray  # uint32
    meta: dict = field(default_factory=dict)

    @property
    def m(self) -> int:
        return int(self.src.size)


def _unique(keys: np.ndarray) -> np.ndarray:
    """Sorted distinct values (sort + adjacent compare; numpy's hash-based
    np.unique is several times slower on large uint64 arrays)."""
    keys = np.sort(keys)
    if keys.size:
        keys = keys[np.concatenate([[True], keys[1:] != keys[:-1]])]
    return keys


def _rng(seed: int, stream: int = 0) -> np.random.Generator:
    # Philox-4x32-10, counter based; the key is (seed, stream)
    return np.random.Generator(np.random.Philox(key=[int(seed), int(stream)]))


def _finish(n, src, dst, seed, name, permute=True, shuffle=True, **meta) -> Arcs:
    src = np.asarray(src, dtype=np.uint64)
    dst = np.asarray(dst, dtype=np.uint64)
    if permute and n > 0:
        perm = _rng(seed, 101).permutation(n).astype(np.uint64)
        src, dst = perm[src], perm[dst]
    if shuffle and src.size:
        order = _rng(seed, 102).permutation(src.size)
        src, dst = src[order], dst[order]
    meta = dict(meta, generator=name, seed=int(seed), m_drawn=int(src.size))
    return Arcs(int(n), src.astype(np.uint32), dst.astype(np.uint32), meta)


def relabel(a: Arcs, seed: int) -> Arcs:
    """Same graph under a random vertex permutation (census-invariant)."""
    perm = _rng(seed, 103).permutation(a.n).astype(np.uint32) if a.n else np.zeros(0, np.uint32)
    return Arcs(a.n, perm[a.src], perm[a.dst], dict(a.meta, relabel_seed=seed))


# ----------------------------------------------------------------------------
# paper-shaped workloads
# ----------------------------------------------------------------------------

def erdos_renyi(n: int = 1000, m: int = 8000, seed: int = 1) -> Arcs:
    """m distinct ordered pairs (u, v), u != v, uniform (C1)."""
    rng = _rng(seed)
    if m > n * (n - 1):
        raise ValueError("too many arcs")
    keys = np.zeros(0, np.uint64)
    while keys.size < m:
        k = rng.integers(0, n * n, size=2 * (m - keys.size) + 16, dtype=np.uint64)
        k = k[(k // n) != (k % n)]
        keys = np.concatenate([keys, k])
        _, first = np.unique(keys, return_index=True)
        keys = keys[np.sort(first)]
    keys = keys[:m]
    return _finish(n, keys // n, keys % n, seed, "erdos_renyi", permute=False)


def _rmat_ids(rng, scale, count, a, b, c):
    src = np.zeros(count, np.uint64)
    dst = np.zeros(count, np.uint64)
    ab, abc = a + b, a + b + c
    for level in range(scale):
        r = rng.random(count, dtype=np.float32)
        sbit = (r >= ab)
        dbit = ((r >= a) & (r < ab)) | (r >= abc)
        bit = np.uint64(1) << np.uint64(scale - 1 - level)
        src |= sbit.astype(np.uint64) * bit
        dst |= dbit.astype(np.uint64) * bit
    return src, dst


def rmat(scale: int = 16, edge_factor: int = 8, a=0.57, b=0.19, c=0.19, seed: int = 16) -> Arcs:
    """R-MAT with Graph500 probabilities; loops/duplicates kept (C2)."""
    n = 1 << scale
    count = edge_factor * n
    src, dst = _rmat_ids(_rng(seed), scale, count, a, b, c)
    return _finish(n, src, dst, seed, "rmat", scale=scale, edge_factor=edge_factor)


PATENTS_N = 3_774_768
PATENTS_M = 16_518_948


def patents_like(n: int = PATENTS_N, m: int = PATENTS_M, sigma: float = 0.92,
                 seed: int = 7) -> Arcs:
    """Lognormal Chung-Lu DAG with exactly m distinct arcs (C3)."""
    rng = _rng(seed)
    w = rng.lognormal(0.0, sigma, size=n)
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    keys = np.zeros(0, np.uint64)
    while keys.size < m:
        need = int((m - keys.size) * 1.1) + 1024
        # inverse-CDF sampling; sorted queries make searchsorted cache
        # friendly, and permuting j afterwards keeps the pairs independent
        i = np.searchsorted(cdf, np.sort(rng.random(need)), side="right").astype(np.uint64)
        j = np.searchsorted(cdf, np.sort(rng.random(need)), side="right").astype(np.uint64)
        j = j[rng.permutation(need)]
        np.minimum(i, n - 1, out=i)
        np.minimum(j, n - 1, out=j)
        keep = i != j
        hi = np.maximum(i, j)[keep]      # newer (larger id) cites older
        lo = np.minimum(i, j)[keep]
        keys = _unique(np.concatenate([keys, hi * np.uint64(n) + lo]))
    pick = _rng(seed, 1).choice(keys.size, size=m, replace=False)
    keys = keys[np.sort(pick)]
    return _finish(n, keys // np.uint64(n), keys % np.uint64(n), seed, "patents_like",
                   sigma=sigma)


LJ_N = 4_847_571
LJ_M_TARGET = 69_000_000


def livejournal_like(n: int = LJ_N, m_target: int = LJ_M_TARGET, q: float = 0.538,
                     scale: int = 23, seed: int = 11) -> Arcs:
    """Social R-MAT with ~70% reciprocated arcs (C4)."""
    rng = _rng(seed)
    keys = np.zeros(0, np.uint64)
    nn = np.uint64(n)
    while keys.size < m_target:
        base = int((m_target - keys.size) / (1 + q) * 1.15) + 1024
        s, d = _rmat_ids(rng, scale, base, 0.57, 0.19, 0.19)
        ok = (s < nn) & (d < nn) & (s != d)
        s, d = s[ok], d[ok]
        rec = rng.random(s.size) < q
        new = np.concatenate([s * nn + d, d[rec] * nn + s[rec]])
        keys = _unique(np.concatenate([keys, new]))
    return _finish(n, keys // nn, keys % nn, seed, "livejournal_like", q=q, scale=scale)


CONFIGS = {
    "C1": dict(fn="erdos_renyi", kwargs=dict(n=1000, m=8000, seed=1),
               label="directed Erdos-Renyi n=1,000 m=8,000"),
    "C2": dict(fn="rmat", kwargs=dict(scale=16, edge_factor=8, seed=16),
               label="directed R-MAT scale 16 edge factor 8"),
    "C3": dict(fn="patents_like", kwargs=dict(seed=7),
               label="Patents-shaped lognormal Chung-Lu DAG n=3,774,768 m=16,518,948"),
    "C4": dict(fn="livejournal_like", kwargs=dict(seed=11),
               label="LiveJournal-shaped social R-MAT n=4,847,571 m~69M reciprocity~0.70"),
}


def make_config(name: str) -> Arcs:
    cfg = CONFIGS[name]
    a = globals()[cfg["fn"]](**cfg["kwargs"])
    a.meta["config"] = name
    a.meta["label"] = cfg["label"]
    return a


# ----------------------------------------------------------------------------
# small random and closed-form graphs (tests)
# ----------------------------------------------------------------------------

def random_digraph(n: int, p: float, seed: int, loops: bool = False, dups: int = 0) -> Arcs:
    """Each ordered pair u != v an arc with probability p; optional noise."""
    rng = _rng(seed)
    if n == 0:
        return Arcs(0, np.zeros(0, np.uint32), np.zeros(0, np.uint32), {})
    mask = rng.random((n, n)) < p
    np.fill_diagonal(mask, False)
    s, d = np.nonzero(mask)
    s, d = s.astype(np.uint64), d.astype(np.uint64)
    if loops:
        k = max(1, n // 4)
        v = rng.integers(0, n, size=k).astype(np.uint64)
        s, d = np.concatenate([s, v]), np.concatenate([d, v])
    if dups and s.size:
        idx = rng.integers(0, s.size, size=dups)
        s, d = np.concatenate([s, s[idx]]), np.concatenate([d, d[idx]])
    return _finish(n, s, d, seed, "random_digraph", permute=False, p=p)


def _plain(n, pairs, name):
    pairs = np.asarray(pairs, dtype=np.uint64).reshape(-1, 2)
    return Arcs(int(n), pairs[:, 0].astype(np.uint32), pairs[:, 1].astype(np.uint32),
                {"generator": name})


def out_star(k: int, n: int | None = None) -> Arcs:
    """Centre 0 -> leaves 1..k, padded with isolated vertices up to n."""
    n = k + 1 if n is None else n
    leaves = np.arange(1, k + 1, dtype=np.uint64)
    return Arcs(n, np.zeros(k, np.uint32), leaves.astype(np.uint32), {"generator": "out_star"})


def in_star(k: int, n: int | None = None) -> Arcs:
    a = out_star(k, n)
    return Arcs(a.n, a.dst, a.src, {"generator": "in_star"})


def mutual_star(k: int, n: int | None = None) -> Arcs:
    a = out_star(k, n)
    return Arcs(a.n, np.concatenate([a.src, a.dst]), np.concatenate([a.dst, a.src]),
                {"generator": "mutual_star"})


def directed_cycle(n: int) -> Arcs:
    i = np.arange(n, dtype=np.uint64)
    return _plain(n, np.stack([i, (i + 1) % n], 1), "directed_cycle")


def transitive_tournament(n: int) -> Arcs:
    """i -> j for all i < j."""
    iu = np.triu_indices(n, 1)
    return Arcs(n, iu[0].astype(np.uint32), iu[1].astype(np.uint32),
                {"generator": "transitive_tournament"})


def complete_mutual(n: int) -> Arcs:
    s, d = np.nonzero(~np.eye(n, dtype=bool))
    return Arcs(n, s.astype(np.uint32), d.astype(np.uint32), {"generator": "complete_mutual"})


def complete_bipartite(a: int, b: int) -> Arcs:
    """All arcs from part A = {0..a-1} to part B = {a..a+b-1}."""
    s = np.repeat(np.arange(a, dtype=np.uint32), b)
    d = np.tile(np.arange(a, a + b, dtype=np.uint32), a)
    return Arcs(a + b, s, d, {"generator": "complete_bipartite"})


# Holland-Leinhardt representative digraphs on (A,B,C) = (0,1,2)
REPRESENTATIVES = {
    "003": [],
    "012": [(0, 1)],
    "102": [(0, 1), (1, 0)],
    "021D": [(1, 0), (1, 2)],
    "021U": [(0, 1), (2, 1)],
    "021C": [(0, 1), (1, 2)],
    "111D": [(0, 1), (1, 0), (2, 0)],
    "111U": [(0, 1), (1, 0), (0, 2)],
    "030T": [(0, 1), (0, 2), (1, 2)],
    "030C": [(0, 1), (1, 2), (2, 0)],
    "201": [(0, 1), (1, 0), (0, 2), (2, 0)],
    "120D": [(0, 1), (1, 0), (2, 0), (2, 1)],
    "120U": [(0, 1), (1, 0), (0, 2), (1, 2)],
    "120C": [(0, 1), (1, 0), (0, 2), (2, 1)],
    "210": [(0, 1), (1, 0), (0, 2), (2, 0), (1, 2)],
    "300": [(0, 1), (1, 0), (0, 2), (2, 0), (1, 2), (2, 1)],
}


def single_triad(name: str) -> Arcs:
    return _plain(3, REPRESENTATIVES[name] or np.zeros((0, 2)), "single_triad:" + name)
