"""Per-canonical-dyad census work, restated with numpy from the arc list
(test helper; no census arithmetic): the quantity the multi-GPU shard cut
balances (include/triadcensus.h tc_shard_bounds).

For canonical dyad (u, v), u < v (order: u asc, v asc):
  a = |{w in N(u): w > u}|, b = |{w in N(v): w > u}|, t = a + b
  (the merge trips of the census kernels, reading 21);
on hub graphs (max degree >= 4096) a dyad with t > 254 whose short list
s = min(a, b) and long list l = max(a, b) satisfy s (L + 4) < a + b,
L = bit_length(l) = ceil(log2(l + 1)), is searched instead of merged
(reading 23) and costs s L + 4 search units.
"""
import numpy as np

THREAD_BIN_MAX = 254
SPARSE_MIN_DEGREE = 4096


def neighbour_crs(n, src, dst):
    src = np.asarray(src, np.int64)
    dst = np.asarray(dst, np.int64)
    keep = src != dst
    s, d = src[keep], dst[keep]
    und = np.sort(np.concatenate([s * n + d, d * n + s]))     # both orientations
    if und.size:
        und = und[np.concatenate([[True], und[1:] != und[:-1]])]
    row, col = und // n, und % n
    off = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(row, minlength=n), out=off[1:])
    return off, col, und


def dyad_work(n, src, dst):
    """(t, cost) per canonical dyad in canonical order; cost = t, or the
    skewed-pair search units where the census searches instead of merging."""
    off, col, key = neighbour_crs(n, src, dst)
    row = key // n
    canon = row < col
    u, v = row[canon], col[canon]
    # entries > u of row u and of row v: one past the position of (x, u)
    a = off[u + 1] - np.searchsorted(key, u * n + u, side="right")
    b = off[v + 1] - np.searchsorted(key, v * n + u, side="right")
    t = a + b
    cost = t.copy()
    deg = np.diff(off)
    if deg.size and deg.max() >= SPARSE_MIN_DEGREE:
        sh, lg = np.minimum(a, b), np.maximum(a, b)
        L = np.frexp((lg | 1).astype(np.float64))[1].astype(np.int64)   # bit_length(l | 1)
        sp = (t > THREAD_BIN_MAX) & (sh * (L + 4) < a + b)
        cost[sp] = sh[sp] * L[sp] + 4
    return t, cost


def rank_work(bounds, work):
    pre = np.concatenate([[0], np.cumsum(work, dtype=np.int64)])
    return [int(pre[bounds[r + 1]] - pre[bounds[r]]) for r in range(len(bounds) - 1)]
