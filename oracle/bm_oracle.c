/*
 * oracle/bm_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded CPU implementation of the Batagelj-Mrvar
 * (B-M) subquadratic directed triad census exactly as PAPER.md states it.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this library.  The product path
 * (paper_1603_02655_b200/) never links, imports or calls it, and this file
 * shares no code, header, table or constant with the CUDA path: the only
 * thing both sides see is the arc list produced by synth/.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n, "S:n" = SPEC.md line n.
 *
 *   og_triad_table   P:327, P:343 (TriadTable, contents not printed) -- derived
 *                    here by orbit enumeration of the 64 codes of Fig. TriadCode
 *                     under the 6 relabellings of (u,v,w); class
 *                    order 1..16 = 003,012,102,021D,021U,021C,111D,111U,030T,
 *                    030C,201,120D,120U,120C,210,300; D/U/C/T labels
 *                    placed by the Holland-Leinhardt representatives.
 *   og_census        Fig. "Subquadratic Triad Census Algorithm"
 *                    with the v0.4 pre-computed dyad code.
 *                    IsEdge / IsNeighbour by binary search over sorted rows
 *                    (v0.5).  Null triads closed with
 *                    n(n-1)(n-2)/6 - sum in 128-bit arithmetic.
 *   og_census_range  the same loop restricted to canonical dyads with index in
 *                    [b, e) in the algorithm's own (u asc, v asc) order
 *                    (P:277-281); classes 2..16 only.  Partials over any
 *                    partition sum to the full census.
 *   og_bruteforce    the naive O(n^3) census of P:261: every unordered triple
 *                    classified by the 6-probe TriadCode of Fig. P:329-347.
 *   og_census64      the non-isomorphic (64-type) census of the same loop
 *                    (TriadCode "returns this value + 1
 *                    if main algorithm calculates non-isomorphic triad
 *                    census"); dyadic triads go to code pre (DESIGN.md
 *                    reading 12); code 0 closes as C(n,3) - sum.
 *   og_bruteforce64  O(n^3) 64-type census in the labelling B-M uses: a
 *                    connected triple a<b<c is coded at (u,v,w) = (a,b,c) if
 *                    a,b are adjacent, else (a,c,b) (the canonical dyad that
 *                    counts it); a dyadic triple at its one connected
 *                    pair (x<y) with code pre(x,y); an empty triple at 0.
 *   og_task_queues   the multithreaded version's task-queue generation
 *                    (SURVEY.md 8(f) f3): Fig. "Distributed Task Queue
 *                    generation ... Canonical Dyad(non-uniform distr.)"
 *                    (NsetSize += |S|, S = N[u] U N[v] \ {u,v})
 *                    and "... Canonical Dyad(uniform distr.)" (P:1676-1698:
 *                    NsetSize += |N[u]| + |N[v]| - 2), line by line; a queue
 *                    is closed (thid + 1, NsetSize <- 0) right after the dyad
 *                    that makes NsetSize > MaxNsetSize.
 *
 * Graph sanitising (reading 9): self-loops are dropped,
 * duplicate arcs are merged.  Vertex ids are 0-based, n is explicit.
 *
 * Two separate CRS structures are kept on purpose:
 * E (out-arcs, sorted) and N (undirected open neighbourhood, sorted).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 og_u128;

/* ------------------------------------------------------------------ */
/* Graph: E and N as CRS (row offsets n+1, sorted columns)             */
/* ------------------------------------------------------------------ */
typedef struct {
    uint64_t n;
    uint64_t m;              /* arcs after loop drop + dedup */
    uint64_t m_in;           /* arcs given */
    uint64_t loops;          /* self-loops dropped */
    uint64_t dups;           /* duplicate arcs dropped */
    uint64_t *e_off;         /* n+1 */
    uint32_t *e_col;         /* m */
    uint64_t *n_off;         /* n+1 */
    uint32_t *n_col;         /* 2 * (number of connected dyads) */
} og_graph;

typedef struct {
    uint64_t n, m_in, m, loops_dropped, dups_dropped, dyads, mutual_dyads,
             max_degree, sum_deg_sq;
} og_stats;

static int og_cmp_u64(const void *a, const void *b)
{
    uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
    return (x > y) - (x < y);
}

void og_graph_free(og_graph *g)
{
    if (!g) return;
    free(g->e_off); free(g->e_col); free(g->n_off); free(g->n_col);
    free(g);
}

/* Returns NULL on allocation failure or range error; *bad_arc gets the index
 * of the first arc with an endpoint >= n (or UINT64_MAX if none). */
og_graph *og_graph_build(uint64_t n, const uint32_t *src, const uint32_t *dst,
                         uint64_t m_in, uint64_t *bad_arc)
{
    *bad_arc = UINT64_MAX;
    for (uint64_t i = 0; i < m_in; i++) {
        if ((uint64_t)src[i] >= n || (uint64_t)dst[i] >= n) { *bad_arc = i; return NULL; }
    }
    og_graph *g = (og_graph *)calloc(1, sizeof(og_graph));
    if (!g) return NULL;
    g->n = n; g->m_in = m_in;

    /* 1. arcs as (src<<32 | dst), loops dropped, sorted, deduplicated */
    uint64_t *key = (uint64_t *)malloc((m_in ? m_in : 1) * sizeof(uint64_t));
    if (!key) { og_graph_free(g); return NULL; }
    uint64_t k = 0;
    for (uint64_t i = 0; i < m_in; i++) {
        if (src[i] == dst[i]) { g->loops++; continue; }
        key[k++] = ((uint64_t)src[i] << 32) | (uint64_t)dst[i];
    }
    qsort(key, k, sizeof(uint64_t), og_cmp_u64);
    uint64_t m = 0;
    for (uint64_t i = 0; i < k; i++)
        if (i == 0 || key[i] != key[i - 1]) key[m++] = key[i];
    g->dups = k - m;
    g->m = m;

    /* 2. E: out-arc CRS */
    g->e_off = (uint64_t *)calloc(n + 1, sizeof(uint64_t));
    g->e_col = (uint32_t *)malloc((m ? m : 1) * sizeof(uint32_t));
    if (!g->e_off || !g->e_col) { free(key); og_graph_free(g); return NULL; }
    for (uint64_t i = 0; i < m; i++) {
        g->e_off[(key[i] >> 32) + 1]++;
        g->e_col[i] = (uint32_t)(key[i] & 0xffffffffu);
    }
    for (uint64_t v = 0; v < n; v++) g->e_off[v + 1] += g->e_off[v];

    /* 3. N: undirected neighbour CRS = sorted, deduplicated {u,v} of every arc */
    uint64_t *und = (uint64_t *)malloc((m ? 2 * m : 1) * sizeof(uint64_t));
    if (!und) { free(key); og_graph_free(g); return NULL; }
    for (uint64_t i = 0; i < m; i++) {
        uint64_t s = key[i] >> 32, d = key[i] & 0xffffffffu;
        und[2 * i] = (s << 32) | d;
        und[2 * i + 1] = (d << 32) | s;
    }
    free(key);
    qsort(und, 2 * m, sizeof(uint64_t), og_cmp_u64);
    uint64_t nn = 0;
    for (uint64_t i = 0; i < 2 * m; i++)
        if (i == 0 || und[i] != und[i - 1]) und[nn++] = und[i];
    g->n_off = (uint64_t *)calloc(n + 1, sizeof(uint64_t));
    g->n_col = (uint32_t *)malloc((nn ? nn : 1) * sizeof(uint32_t));
    if (!g->n_off || !g->n_col) { free(und); og_graph_free(g); return NULL; }
    for (uint64_t i = 0; i < nn; i++) {
        g->n_off[(und[i] >> 32) + 1]++;
        g->n_col[i] = (uint32_t)(und[i] & 0xffffffffu);
    }
    for (uint64_t v = 0; v < n; v++) g->n_off[v + 1] += g->n_off[v];
    free(und);
    return g;
}

/* binary search in a sorted row (v0.5) */
static int og_row_has(const uint64_t *off, const uint32_t *col, uint64_t u, uint64_t x)
{
    uint64_t lo = off[u], hi = off[u + 1];
    while (lo < hi) {
        uint64_t mid = lo + (hi - lo) / 2;
        if ((uint64_t)col[mid] < x) lo = mid + 1; else hi = mid;
    }
    return lo < off[u + 1] && (uint64_t)col[lo] == x;
}

/* IsEdge(u,v): arc u->v exists */
static int og_is_edge(const og_graph *g, uint64_t u, uint64_t v)
{
    return og_row_has(g->e_off, g->e_col, u, v);
}

/* IsNeighbour(u,v): u,v adjacent in the undirected sense */
static int og_is_neighbour(const og_graph *g, uint64_t u, uint64_t v)
{
    return og_row_has(g->n_off, g->n_col, u, v);
}

void og_graph_stats(const og_graph *g, og_stats *s)
{
    memset(s, 0, sizeof(*s));
    s->n = g->n; s->m_in = g->m_in; s->m = g->m;
    s->loops_dropped = g->loops; s->dups_dropped = g->dups;
    s->dyads = (g->n_off[g->n]) / 2;
    for (uint64_t u = 0; u < g->n; u++) {
        uint64_t d = g->n_off[u + 1] - g->n_off[u];
        if (d > s->max_degree) s->max_degree = d;
        s->sum_deg_sq += d * d;
        for (uint64_t i = g->e_off[u]; i < g->e_off[u + 1]; i++) {
            uint64_t v = g->e_col[i];
            if (u < v && og_is_edge(g, v, u)) s->mutual_dyads++;
        }
    }
}

/* ------------------------------------------------------------------ */
/* TriadTable by orbit enumeration */
/* ------------------------------------------------------------------ */

/* Code bits of Fig. TriadCode over the ordered triple
 * (x0,x1,x2) = (u,v,w):  1:u->v 2:v->u 4:u->w 8:w->u 16:v->w 32:w->v.
 * arc(a,b) for a != b in {0,1,2} is the bit for x_a -> x_b. */
static int og_arc_bit(int a, int b)
{
    if (a == 0 && b == 1) return 1;
    if (a == 1 && b == 0) return 2;
    if (a == 0 && b == 2) return 4;
    if (a == 2 && b == 0) return 8;
    if (a == 1 && b == 2) return 16;
    return 32; /* a == 2 && b == 1 */
}

/* code of the same triad after renaming vertex i to p[i] */
static int og_permute_code(int code, const int p[3])
{
    int out = 0;
    for (int a = 0; a < 3; a++)
        for (int b = 0; b < 3; b++)
            if (a != b && (code & og_arc_bit(a, b))) out |= og_arc_bit(p[a], p[b]);
    return out;
}

/* representative code for an arc list on (A,B,C) = (0,1,2) */
static int og_code_of(const int (*arcs)[2], int k)
{
    int c = 0;
    for (int i = 0; i < k; i++) c |= og_arc_bit(arcs[i][0], arcs[i][1]);
    return c;
}

/* Fills T[64] with 1-based class indices (1..16).  Returns 0 on success,
 * -1 if the orbit structure is not the expected one (16 orbits). */
int og_triad_table(uint8_t T[64])
{
    static const int perms[6][3] = {{0,1,2},{0,2,1},{1,0,2},{1,2,0},{2,0,1},{2,1,0}};
    /* orbit id = smallest code in the orbit */
    int orbit[64];
    for (int c = 0; c < 64; c++) {
        int mn = c;
        for (int p = 0; p < 6; p++) {
            int q = og_permute_code(c, perms[p]);
            if (q < mn) mn = q;
        }
        orbit[c] = mn;
    }
    int norb = 0;
    for (int c = 0; c < 64; c++) if (orbit[c] == c) norb++;
    if (norb != 16) return -1;

    /* MAN digits of a code: mutual, asymmetric, null dyads */
    /* Class order of P:253-256 with the representatives of S:278 for the
     * classes whose MAN digits are shared. */
    static const int r021D[][2] = {{1,0},{1,2}};
    static const int r021U[][2] = {{0,1},{2,1}};
    static const int r021C[][2] = {{0,1},{1,2}};
    static const int r111D[][2] = {{0,1},{1,0},{2,0}};
    static const int r111U[][2] = {{0,1},{1,0},{0,2}};
    static const int r030T[][2] = {{0,1},{0,2},{1,2}};
    static const int r030C[][2] = {{0,1},{1,2},{2,0}};
    static const int r120D[][2] = {{0,1},{1,0},{2,0},{2,1}};
    static const int r120U[][2] = {{0,1},{1,0},{0,2},{1,2}};
    static const int r120C[][2] = {{0,1},{1,0},{0,2},{2,1}};
    static const int r210[][2]  = {{0,1},{1,0},{0,2},{2,0},{1,2}};
    static const int r012[][2]  = {{0,1}};
    static const int r102[][2]  = {{0,1},{1,0}};
    static const int r201[][2]  = {{0,1},{1,0},{0,2},{2,0}};
    static const int r300[][2]  = {{0,1},{1,0},{0,2},{2,0},{1,2},{2,1}};
    int rep[17];
    rep[1]  = 0;                       /* 003 */
    rep[2]  = og_code_of(r012, 1);
    rep[3]  = og_code_of(r102, 2);
    rep[4]  = og_code_of(r021D, 2);
    rep[5]  = og_code_of(r021U, 2);
    rep[6]  = og_code_of(r021C, 2);
    rep[7]  = og_code_of(r111D, 3);
    rep[8]  = og_code_of(r111U, 3);
    rep[9]  = og_code_of(r030T, 3);
    rep[10] = og_code_of(r030C, 3);
    rep[11] = og_code_of(r201, 4);
    rep[12] = og_code_of(r120D, 4);
    rep[13] = og_code_of(r120U, 4);
    rep[14] = og_code_of(r120C, 4);
    rep[15] = og_code_of(r210, 5);
    rep[16] = og_code_of(r300, 6);
    for (int c = 0; c < 64; c++) T[c] = 0;
    for (int k = 1; k <= 16; k++) {
        int o = orbit[rep[k]];
        for (int c = 0; c < 64; c++)
            if (orbit[c] == o) {
                if (T[c] != 0) return -1;  /* two classes share an orbit */
                T[c] = (uint8_t)k;
            }
    }
    for (int c = 0; c < 64; c++) if (T[c] == 0) return -1;
    return 0;
}

/* ------------------------------------------------------------------ */
/* C(n,3) and the null-triad closing, 128-bit               */
/* ------------------------------------------------------------------ */
static og_u128 og_choose3(uint64_t n)
{
    if (n < 3) return 0;                          /* DESIGN.md reading 18 */
    og_u128 a = n, b = n - 1, c = n - 2;
    /* callers enforce n <= 2^32, so a*b*c < 2^96 fits in 128 bits */
    return a * b * c / 6;
}

/* ------------------------------------------------------------------ */
/* Census (Fig. P:269-309 with v0.4 P:1396-1432)                       */
/* ------------------------------------------------------------------ */

/* Accumulates classes 2..16 of the canonical dyads with index in [db, de)
 * into C[1..16] (1-based).  S is materialised exactly as line 8:
 * S <- N(u) U N(v) \ {u,v}.  Returns -1 on allocation failure. */
static int og_census_core(const og_graph *g, const uint8_t T[64],
                          uint64_t db, uint64_t de, uint64_t *C, int mode64)
{
    uint64_t n = g->n;
    uint64_t maxd = 0;
    for (uint64_t u = 0; u < n; u++) {
        uint64_t d = g->n_off[u + 1] - g->n_off[u];
        if (d > maxd) maxd = d;
    }
    uint32_t *S = (uint32_t *)malloc((2 * maxd + 1) * sizeof(uint32_t));
    if (!S) return -1;
    uint64_t k = 0;                                   /* canonical dyad index */
    for (uint64_t u = 0; u < n; u++) {                /* line 5 */
        for (uint64_t a = g->n_off[u]; a < g->n_off[u + 1]; a++) {   /* line 6 */
            uint64_t v = g->n_col[a];
            if (!(u < v)) continue;                   /* line 7 */
            uint64_t kk = k++;
            if (kk < db || kk >= de) continue;
            /* line 8: S <- N(u) U N(v) \ {u,v} (sorted two-way union) */
            uint64_t i = g->n_off[u], ie = g->n_off[u + 1];
            uint64_t j = g->n_off[v], je = g->n_off[v + 1];
            uint64_t s = 0;
            while (i < ie || j < je) {
                uint64_t x;
                if (j >= je || (i < ie && g->n_col[i] < g->n_col[j])) x = g->n_col[i++];
                else if (i >= ie || g->n_col[j] < g->n_col[i]) x = g->n_col[j++];
                else { x = g->n_col[i]; i++; j++; }
                if (x != u && x != v) S[s++] = (uint32_t)x;
            }
            /* v0.4: IsEdge[0], IsEdge[1], precomputed_triad_type */
            int e0 = og_is_edge(g, u, v);
            int e1 = og_is_edge(g, v, u);
            int pre = e0 + 2 * e1;
            /* lines 9-14 (64-type mode: the dyadic triads' code is pre) */
            int type = mode64 ? pre + 1 : ((e0 && e1) ? 3 : 2);
            C[type] += n - s - 2;
            /* lines 15-20 */
            for (uint64_t t = 0; t < s; t++) {
                uint64_t w = S[t];
                if (v < w || (w < v && u < w && !og_is_neighbour(g, u, w))) {   /* line 16 */
                    /* Modified TriadCode (Fig. P:1420-1431) */
                    int code = pre;
                    code += 4 * og_is_edge(g, u, w);
                    code += 8 * og_is_edge(g, w, u);
                    code += 16 * og_is_edge(g, v, w);
                    code += 32 * og_is_edge(g, w, v);
                    C[mode64 ? code + 1 : T[code]] += 1;                    /* line 18 */
                }
            }
        }
    }
    free(S);
    return 0;
}

/* Full census.  counts[k-1] = class k (k = 1..16); the 003 count is a
 * 128-bit value returned as counts[0] (low word) and *c003_hi.
 * Returns 0, -1 (OOM), -2 (n >= 2^32), -3 (table), -4 (consistency). */
int og_census(const og_graph *g, uint64_t counts[16], uint64_t *c003_hi)
{
    uint8_t T[64];
    if (og_triad_table(T) != 0) return -3;
    if (g->n > 0xffffffffull) return -2;
    uint64_t C[17];
    memset(C, 0, sizeof(C));
    if (og_census_core(g, T, 0, UINT64_MAX, C, 0) != 0) return -1;
    /* lines 24-28: Census[1] <- n(n-1)(n-2)/6 - sum */
    og_u128 sum = 0;
    for (int i = 2; i <= 16; i++) sum += C[i];
    og_u128 total = og_choose3(g->n);
    if (sum > total) return -4;
    og_u128 c1 = total - sum;
    counts[0] = (uint64_t)c1;
    *c003_hi = (uint64_t)(c1 >> 64);
    for (int i = 2; i <= 16; i++) counts[i - 1] = C[i];
    return 0;
}

/* Partial census over canonical dyads [db, de): classes 2..16, counts[0]=0. */
int og_census_range(const og_graph *g, uint64_t db, uint64_t de, uint64_t counts[16])
{
    uint8_t T[64];
    if (og_triad_table(T) != 0) return -3;
    uint64_t C[17];
    memset(C, 0, sizeof(C));
    if (og_census_core(g, T, db, de, C, 0) != 0) return -1;
    counts[0] = 0;
    for (int i = 2; i <= 16; i++) counts[i - 1] = C[i];
    return 0;
}

/* 64-type census: counts[c] = triads with TriadCode c (c = 0..63) in the
 * B-M labelling; counts[0] low word, *c0_hi high word. */
int og_census64(const og_graph *g, uint64_t counts[64], uint64_t *c0_hi)
{
    uint8_t T[64];
    if (og_triad_table(T) != 0) return -3;
    if (g->n > 0xffffffffull) return -2;
    uint64_t C[65];
    memset(C, 0, sizeof(C));
    if (og_census_core(g, T, 0, UINT64_MAX, C, 1) != 0) return -1;
    og_u128 sum = 0;
    for (int i = 2; i <= 64; i++) sum += C[i];
    og_u128 total = og_choose3(g->n);
    if (sum > total) return -4;
    og_u128 c0 = total - sum;
    counts[0] = (uint64_t)c0;
    *c0_hi = (uint64_t)(c0 >> 64);
    for (int i = 2; i <= 64; i++) counts[i - 1] = C[i];
    return 0;
}

/* Per-canonical-dyad uniform cost |N(u)| + |N(v)| (P:1693 without the -2),
 * in canonical order; out must hold `dyads` entries.  Used only by tests of
 * the sharding rule. */
void og_dyad_costs(const og_graph *g, uint64_t *out)
{
    uint64_t k = 0;
    for (uint64_t u = 0; u < g->n; u++)
        for (uint64_t a = g->n_off[u]; a < g->n_off[u + 1]; a++) {
            uint64_t v = g->n_col[a];
            if (u < v)
                out[k++] = (g->n_off[u + 1] - g->n_off[u]) + (g->n_off[v + 1] - g->n_off[v]);
        }
}

/* ------------------------------------------------------------------ */
/* Task queues of the multithreaded version              */
/* ------------------------------------------------------------------ */

/* strategy 0 = Canonical Dyad(uniform distr.) (Fig. P:1676-1698),
 * strategy 1 = Canonical Dyad(non-uniform distr.) (Fig. P:1650-1672).
 * Queues are contiguous runs of canonical dyads (TQ[thid] <- TQ[thid] U
 * <u,v> in the loop order of lines 4-6).  starts[q] = index of the first
 * dyad of the q-th non-empty queue (q = 0 .. *nq - 1); a cut after the
 * very last dyad opens no queue.  *total = aggregate NsetSize over all
 * dyads (Table).  Returns 0, -1 (OOM), -2 (more than cap
 * queues; *nq is still set). */
int og_task_queues(const og_graph *g, int strategy, uint64_t max_nset, uint64_t *starts,
                   uint64_t cap, uint64_t *nq, uint64_t *total)
{
    uint64_t n = g->n, maxd = 0;
    for (uint64_t u = 0; u < n; u++) {
        uint64_t d = g->n_off[u + 1] - g->n_off[u];
        if (d > maxd) maxd = d;
    }
    uint32_t *S = (uint32_t *)malloc((2 * maxd + 1) * sizeof(uint32_t));
    if (!S) return -1;
    uint64_t thid = 0, nset = 0, k = 0, q = 0, tot = 0;
    int open = 0;                                      /* TQ[thid] non-empty */
    for (uint64_t u = 0; u < n; u++) {                 /* line 4 */
        for (uint64_t a = g->n_off[u]; a < g->n_off[u + 1]; a++) {   /* line 5 */
            uint64_t v = g->n_col[a];
            if (!(u < v)) continue;                    /* line 6 */
            if (!open) {                               /* line 7: TQ[thid] gets <u,v> */
                if (q < cap) starts[q] = k;
                q++;
                open = 1;
            }
            uint64_t w;
            if (strategy == 1) {                       /* lines 8-9: |S| */
                uint64_t i = g->n_off[u], ie = g->n_off[u + 1];
                uint64_t j = g->n_off[v], je = g->n_off[v + 1];
                uint64_t s = 0;
                while (i < ie || j < je) {
                    uint64_t x;
                    if (j >= je || (i < ie && g->n_col[i] < g->n_col[j])) x = g->n_col[i++];
                    else if (i >= ie || g->n_col[j] < g->n_col[i]) x = g->n_col[j++];
                    else { x = g->n_col[i]; i++; j++; }
                    if (x != u && x != v) S[s++] = (uint32_t)x;
                }
                w = s;
            } else {                                   /* line 8: |N[u]| + |N[v]| - 2 */
                w = (g->n_off[u + 1] - g->n_off[u]) + (g->n_off[v + 1] - g->n_off[v]) - 2;
            }
            nset += w;
            tot += w;
            if (nset > max_nset) {                     /* lines 10-13 */
                thid++;
                nset = 0;
                open = 0;
            }
            k++;
        }
    }
    (void)thid;
    free(S);
    *nq = q;
    *total = tot;
    return q > cap ? -2 : 0;
}

/* ------------------------------------------------------------------ */
/* Naive O(n^3) census over a bit-packed adjacency matrix       */
/* ------------------------------------------------------------------ */
int og_bruteforce(const og_graph *g, uint64_t counts[16], uint64_t *c003_hi)
{
    uint8_t T[64];
    if (og_triad_table(T) != 0) return -3;
    uint64_t n = g->n;
    if (n > 20000) return -2;
    uint64_t words = (n + 63) / 64;
    uint64_t *adj = (uint64_t *)calloc((n && words) ? n * words : 1, sizeof(uint64_t));
    if (!adj) return -1;
    for (uint64_t u = 0; u < n; u++)
        for (uint64_t i = g->e_off[u]; i < g->e_off[u + 1]; i++) {
            uint64_t v = g->e_col[i];
            adj[u * words + v / 64] |= 1ull << (v % 64);
        }
#define OG_ARC(a, b) ((adj[(a) * words + (b) / 64] >> ((b) % 64)) & 1ull)
    og_u128 C[17];
    for (int i = 0; i < 17; i++) C[i] = 0;
    for (uint64_t a = 0; a < n; a++)
        for (uint64_t b = a + 1; b < n; b++) {
            int ab = (int)(OG_ARC(a, b) + 2 * OG_ARC(b, a));
            for (uint64_t c = b + 1; c < n; c++) {
                /* TriadCode (Fig. P:329-347) with (u,v,w) = (a,b,c) */
                int code = ab;
                code += 4 * (int)OG_ARC(a, c);
                code += 8 * (int)OG_ARC(c, a);
                code += 16 * (int)OG_ARC(b, c);
                code += 32 * (int)OG_ARC(c, b);
                C[T[code]] += 1;
            }
        }
#undef OG_ARC
    free(adj);
    counts[0] = (uint64_t)C[1];
    *c003_hi = (uint64_t)(C[1] >> 64);
    for (int i = 2; i <= 16; i++) counts[i - 1] = (uint64_t)C[i];
    return 0;
}

/* O(n^3) 64-type census in the B-M labelling (see header). */
int og_bruteforce64(const og_graph *g, uint64_t counts[64], uint64_t *c0_hi)
{
    uint64_t n = g->n;
    if (n > 20000) return -2;
    uint64_t words = (n + 63) / 64;
    uint64_t *adj = (uint64_t *)calloc((n && words) ? n * words : 1, sizeof(uint64_t));
    if (!adj) return -1;
    for (uint64_t u = 0; u < n; u++)
        for (uint64_t i = g->e_off[u]; i < g->e_off[u + 1]; i++) {
            uint64_t v = g->e_col[i];
            adj[u * words + v / 64] |= 1ull << (v % 64);
        }
#define OG_ARC(a, b) ((int)((adj[(a) * words + (b) / 64] >> ((b) % 64)) & 1ull))
#define OG_CODE(u, v, w) (OG_ARC(u, v) + 2 * OG_ARC(v, u) + 4 * OG_ARC(u, w) + 8 * OG_ARC(w, u) + \
                          16 * OG_ARC(v, w) + 32 * OG_ARC(w, v))
    og_u128 C[64];
    for (int i = 0; i < 64; i++) C[i] = 0;
    for (uint64_t a = 0; a < n; a++)
        for (uint64_t b = a + 1; b < n; b++)
            for (uint64_t c = b + 1; c < n; c++) {
                int ab = OG_ARC(a, b) | OG_ARC(b, a);
                int ac = OG_ARC(a, c) | OG_ARC(c, a);
                int bc = OG_ARC(b, c) | OG_ARC(c, b);
                int code;
                if (ab + ac + bc >= 2) code = ab ? OG_CODE(a, b, c) : OG_CODE(a, c, b);
                else if (ab) code = OG_CODE(a, b, c) & 3;
                else if (ac) code = OG_CODE(a, c, b) & 3;
                else if (bc) code = OG_CODE(b, c, a) & 3;
                else code = 0;
                C[code] += 1;
            }
#undef OG_CODE
#undef OG_ARC
    free(adj);
    counts[0] = (uint64_t)C[0];
    *c0_hi = (uint64_t)(C[0] >> 64);
    for (int i = 1; i < 64; i++) counts[i] = (uint64_t)C[i];
    return 0;
}

/* C(n,3) as (lo, hi) -- exposed so tests can check the 128-bit closing. */
void og_choose3_u128(uint64_t n, uint64_t *lo, uint64_t *hi)
{
    og_u128 t = og_choose3(n);
    *lo = (uint64_t)t;
    *hi = (uint64_t)(t >> 64);
}

/* CRS accessors for tests */
uint64_t og_graph_n(const og_graph *g) { return g->n; }
uint64_t og_graph_m(const og_graph *g) { return g->m; }
uint64_t og_graph_nnz(const og_graph *g) { return g->n_off[g->n]; }
void og_graph_copy_n(const og_graph *g, uint64_t *off, uint32_t *col)
{
    memcpy(off, g->n_off, (g->n + 1) * sizeof(uint64_t));
    memcpy(col, g->n_col, g->n_off[g->n] * sizeof(uint32_t));
}
