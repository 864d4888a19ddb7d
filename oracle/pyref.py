"""oracle/pyref.py -- TEST INFRASTRUCTURE ONLY.

A tiny pure-Python restatement of the census, for n <= ~30, written
independently of bm_oracle.c so the two can pin each other.

* ``census_bm``    Fig. "Subquadratic Triad Census Algorithm",
                   6-probe TriadCode, Python sets for N and S.
* ``census_brute`` the naive O(n^3) census.
* ``census_range_brute``  the per-dyad-range census by brute force over
                   triples: a triple with exactly one connected pair is a
                   dyadic triad of that pair (lines 9-14); a
                   connected triple a < b < c belongs to its
                   lexicographically smallest adjacent pair -- (a,b) if
                   a~b, else (a,c) -- which is the one canonical dyad whose
                   predicate (line 16: v < w, or u < w < v with w not
                   adjacent to u) admits the third vertex.
* ``man_digits``   the M, A, N digit counts of a code.
The code->class map is taken as an argument (the table under test).
"""
from __future__ import annotations

from itertools import combinations


def _arcs(n, src, dst):
    return {(int(a), int(b)) for a, b in zip(src, dst) if int(a) != int(b)}


def _code(E, u, v, w):
    # Fig. TriadCode
    return ((u, v) in E) + 2 * ((v, u) in E) + 4 * ((u, w) in E) + 8 * ((w, u) in E) \
        + 16 * ((v, w) in E) + 32 * ((w, v) in E)


def census_bm(n, src, dst, table):
    E = _arcs(n, src, dst)
    N = {x: set() for x in range(n)}
    for a, b in E:
        N[a].add(b)
        N[b].add(a)
    C = [0] * 17
    for u in range(n):
        for v in sorted(N[u]):
            if u < v:
                S = (N[u] | N[v]) - {u, v}
                t = 3 if ((u, v) in E and (v, u) in E) else 2
                C[t] += n - len(S) - 2
                for w in S:
                    if v < w or (w < v and u < w and w not in N[u]):
                        C[table[_code(E, u, v, w)]] += 1
    total = n * (n - 1) * (n - 2) // 6 if n >= 3 else 0
    C[1] = total - sum(C[2:])
    return C[1:]


def census_brute(n, src, dst, table):
    E = _arcs(n, src, dst)
    C = [0] * 17
    for a, b, c in combinations(range(n), 3):
        C[table[_code(E, a, b, c)]] += 1
    return C[1:]


def canonical_dyads(n, src, dst):
    """Connected pairs (u, v), u < v, in the algorithm's order (u asc, v asc,
    P:277-281)."""
    return sorted({(min(int(a), int(b)), max(int(a), int(b)))
                   for a, b in zip(src, dst) if int(a) != int(b)})


def census_range_brute(n, src, dst, table, b, e):
    """Classes 2..16 (element 0 = 0) of canonical dyads with index in [b, e)."""
    E = _arcs(n, src, dst)
    index = {d: k for k, d in enumerate(canonical_dyads(n, src, dst))}
    adj = lambda x, y: (x, y) in E or (y, x) in E
    C = [0] * 17
    for a, bb, c in combinations(range(n), 3):
        pairs = [p for p in ((a, bb), (a, c), (bb, c)) if adj(*p)]
        if not pairs:
            continue
        k = index[pairs[0]]            # lexicographically smallest adjacent pair
        if b <= k < e:
            C[table[_code(E, a, bb, c)]] += 1
    C[1] = 0
    return C[1:]


def man_digits(code):
    """(mutual, asymmetric, null) dyad counts of a 6-bit code."""
    pairs = [(code & 1, code & 2), (code & 4, code & 8), (code & 16, code & 32)]
    m = sum(1 for a, b in pairs if a and b)
    a = sum(1 for x, y in pairs if bool(x) != bool(y))
    return m, a, 3 - m - a
