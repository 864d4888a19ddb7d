/*
 * triadcensus.h -- C ABI of libtriadcensus.so, the B200 (sm_100a) directed
 * triad census of arXiv 1603.02655 (Batagelj-Mrvar subquadratic algorithm).
 *
 * Citations: "P:n" = PAPER.md line n (the thesis LaTeX), "S:n" = SPEC.md.
 *
 * What is computed.  For a strict digraph G = [V, E], V = {0..n-1},
 * counts[k-1] is the number of unordered vertex triples whose induced
 * sub-digraph is isomorphic to class k, in the paper's order:
 *   k:  1    2    3    4    5    6    7    8    9    10   11  12   13   14   15  16
 *      003  012  102  021D 021U 021C 111D 111U 030T 030C 201 120D 120U 120C 210 300
 * The device computes classes 2..16 by the B-M loop of Fig. "Subquadratic
 * Triad Census Algorithm": for every canonical connected dyad
 * u < v it adds n - |S| - 2 dyadic triads, S = N(u) U N(v) \ {u,v}, to class
 * 3 (mutual dyad) or 2 (asymmetric), and classifies each canonical w in S
 * (predicate P:292: v < w or (u < w < v and w not adjacent to u)) through
 * the 64-code TriadCode (v0.4 form P:1396-1432) and the 64->16
 * TriadTable.  Class 1 is closed on the host as
 * n(n-1)(n-2)/6 - sum in 128-bit arithmetic.
 *
 * Conventions.
 *  - Vertex ids are 0-based uint32; n must satisfy 0 <= n < 2^30 (ids are
 *    packed as (w<<2)|tag in the device CSR) else TC_E_INVALID.
 *  - Self-loops are dropped and duplicate arcs merged (strict digraph,
 *    P:239/P:264); both are counted in tc_graph_stats.
 *  - m (arcs given) must be < 2^31 and the number of distinct connected
 *    dyads D < 2^31, else TC_E_INVALID.
 *  - "Canonical dyad index" k numbers the connected unordered pairs {u,v},
 *    u < v, in the algorithm's own order: u ascending, then v ascending
 *    (S:312-320).  tc_census_range and sharding use it.
 *  - Class 003 can exceed 2^64 (n > 4,801,280): its high word is returned
 *    separately.  Every other class fits in uint64.
 *  - All functions return tc_status; nothing throws across the ABI.  On
 *    error, tc_last_error() gives a message (thread-local, valid until the
 *    next call on that thread).
 *  - Device work is issued on the caller's CUDA stream (cudaStream_t passed
 *    as void*; NULL = legacy default stream).  tc_census, tc_census_range
 *    and tc_census_multi return after the stream has drained (results on the
 *    host); tc_census_enqueue does not synchronise.  tc_graph_create returns
 *    once the build is enqueued (arc range errors are reported by it, after
 *    a mid-build host read); the graph's statistics reach the host at the
 *    first call that needs them (stats, profile, any census, shard or queue
 *    call), which waits for the build to finish.  Host arc arrays may be
 *    reused as soon as tc_graph_create returns (they are copied first).
 *  - A tc_graph may be shared read-only by concurrent census calls on
 *    different streams (and host threads): a call keeps its launch count
 *    and profile in its own locals and publishes them to the graph's
 *    "most recent call" slot under a mutex at its end (tc_launch_count,
 *    tc_profile_get report whichever call finished last).
 */
#ifndef TRIADCENSUS_H
#define TRIADCENSUS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TC_ABI_VERSION 1

typedef struct tc_graph tc_graph;
typedef struct tc_comm tc_comm;

typedef enum {
    TC_OK = 0,
    TC_E_INVALID = 1,   /* bad argument (NULL pointer, n >= 2^30, size limits) */
    TC_E_RANGE = 2,     /* an arc endpoint >= n; tc_last_error names the arc index */
    TC_E_OOM = 3,       /* device allocation failed */
    TC_E_CUDA = 4,      /* CUDA runtime error; message holds cudaGetErrorString */
    TC_E_NCCL = 5,      /* NCCL error or NCCL library not loadable */
    TC_E_OVERFLOW = 6   /* c003_hi == NULL but the 003 count needs a high word */
} tc_status;

/* Device memory hook.  alloc(bytes, stream, ctx) returns a device pointer
 * usable on `stream` (or NULL on failure); free(ptr, bytes, stream, ctx)
 * releases it.  Pass NULL for the default: cudaMallocAsync on the call's
 * stream behind an exact-size block cache (a freed block is kept under its
 * device, stream and size and handed to the next request of that size on
 * that stream; up to 120 GB per process; tc_trim_memory returns it to the
 * driver).  The Python binding passes torch's caching allocator unless asked
 * for the default. */
typedef struct {
    void *(*alloc)(size_t bytes, void *stream, void *ctx);
    void (*free)(void *ptr, size_t bytes, void *stream, void *ctx);
    void *ctx;
} tc_allocator;

/* Graph statistics after sanitising (a1 of SURVEY.md section 8(a)). */
typedef struct {
    uint64_t n;             /* vertices, including isolated ones */
    uint64_t m_in;          /* arcs given */
    uint64_t m;             /* distinct arcs after loop drop + dedup */
    uint64_t loops_dropped;
    uint64_t dups_dropped;
    uint64_t dyads;         /* D: connected unordered pairs (canonical dyads) */
    uint64_t mutual_dyads;  /* pairs with both arcs */
    uint64_t max_degree;    /* Delta = max |N(u)| (undirected degree) */
    uint64_t sum_deg_sq;    /* sum_u |N(u)|^2 = sum over canonical dyads of |N(u)|+|N(v)| */
} tc_graph_stats;

/* Per-phase device times (ms, CUDA events on the call's stream) of the most
 * recent tc_graph_create / census call on this graph, when profiling is on. */
typedef struct {
    float build_ms;         /* a1: sort + dedup + symmetrise + offsets + stats */
    float plan_ms;          /* a2: per-dyad cost and degree bins */
    float census_ms;        /* a3+a4: all bin kernels incl. histogram flush */
    float kernel_ms[4];     /* a3+a4 per bin: [0] thread bin, [1] warp bin (it runs on a
                               side stream beside the thread bin: from the bins' start
                               to its end), [2..3] 0 */
    uint64_t bin_items[4];  /* [0] thread-bin dyads, [1] warp items, [2] warp-bin dyads,
                               [3] of those, skewed-pair dyads (searched, not merged) */
    uint64_t bin_work[4];   /* [0] / [1] thread / warp bin: sum of |N(u)|+|N(v)| (the
                               paper's uniform work unit, SURVEY 8(d) B_alg);
                               [2] / [3]: merge trips actually walked (entries
                               w > u of both rows, census.cu) */
    uint64_t sparse_sum_c;  /* skewed-pair dyads: sum of |N(u)|+|N(v)| (part of bin_work[1]) */
    uint64_t sparse_units;  /* skewed-pair dyads: entries they read = sum over dyads of
                               s * ceil(log2(l + 1)) + 4 (s, l: short and long list) */
    uint64_t build_sort[4]; /* a1, the graph's build (filled whether or not profiling is
                               on): [0] LSD passes over the m arc keys, [1] LSD passes
                               over the D transposed keys, [2] keys in rows of at most
                               1024 keys left to the per-row networks (0 when the build
                               took the full LSD: hub graphs), [3] key-passes of the
                               composite LSD over the rows longer than that */
} tc_profile;

/* Build the device graph from an arc list (a1).
 *   device          CUDA device ordinal.
 *   n               number of vertices (explicit: isolated vertices count).
 *   src, dst        m arc endpoints (arc i is src[i] -> dst[i]); host
 *                   pointers if arcs_on_device == 0 (copied H2D inside the
 *                   call), else device pointers (only read).  Borrowed.
 *   cuda_stream     cudaStream_t or NULL.
 *   alloc           allocator hook or NULL.
 *   out             receives the graph; owned by the caller, release with
 *                   tc_graph_destroy.
 * Layout built: uint32 off[n+1]; uint32
 * adj[2D] with entry (w<<2)|tag, rows sorted by w, tag bit0 = u->w,
 * bit1 = w->u (P:458-469 adjacency array, symmetric and tagged); uint32
 * dyad lists of the canonical entries.
 * Errors: TC_E_INVALID, TC_E_RANGE (first offending arc index in the
 * message), TC_E_OOM, TC_E_CUDA. */
tc_status tc_graph_create(int device, uint64_t n, const uint32_t *src, const uint32_t *dst,
                          uint64_t m, int arcs_on_device, void *cuda_stream,
                          const tc_allocator *alloc, tc_graph **out);

tc_status tc_graph_stats_get(const tc_graph *g, tc_graph_stats *out);

/* Frees every device buffer of the graph (stream-ordered on the creating
 * stream).  NULL is a no-op. */
void tc_graph_destroy(tc_graph *g);

/* Full census (a2..a5), synchronous.
 *   counts   host uint64[16]; counts[k-1] = class k, counts[0] = low word of 003.
 *   c003_hi  host uint64 receiving the high word of the 003 count; may be
 *            NULL only if that word is 0, else TC_E_OVERFLOW (counts still
 *            filled). */
tc_status tc_census(const tc_graph *g, void *cuda_stream, uint64_t counts[16],
                    uint64_t *c003_hi);

/* 64-type (non-isomorphic) census, SURVEY.md section 8(f) f1 (P:258,
 * P:327): counts[c] = triads whose TriadCode (bit weights of Fig.
 * P:329-347) is c, in the labelling the B-M loop assigns -- a connected
 * triad is coded at (u, v, w) with (u, v) its counting canonical dyad and w
 * the canonical third vertex; a dyadic triad gets code pre =
 * IsEdge(u,v) + 2 IsEdge(v,u) (reading 12); code 0 = C(n,3) -
 * sum, low word in counts[0], high word in *c0_hi (same rules as c003_hi).
 * Folding counts through the TriadTable gives tc_census.  Synchronous. */
tc_status tc_census64(const tc_graph *g, void *cuda_stream, uint64_t counts[64],
                      uint64_t *c0_hi);

/* Partial census over canonical dyads [dyad_begin, dyad_end) (clamped to
 * [0, D)): classes 2..16 only, partial[0] = 0 -- exactly the loop of Fig.
 * P:269-309 (lines 5-21) restricted to the dyads of the range in the
 * algorithm's own order: each dyad (u,v) of the range adds its
 * n - |S| - 2 dyadic triads to class 102 (mutual) or 012, and
 * its canonical connected triads to their classes.  Every entry is
 * a non-negative count; partials over any partition of [0, D) sum to the
 * full census minus 003.  This is the test / shard hook: the full
 * and multi-GPU census do not call it (they split 012 / 102 differently,
 * see tc_census_enqueue).  Synchronous. */
tc_status tc_census_range(const tc_graph *g, uint64_t dyad_begin, uint64_t dyad_end,
                          void *cuda_stream, uint64_t partial[16]);

/* Asynchronous partial census: enqueues a2..a4 for dyads [dyad_begin,
 * dyad_end) on the stream and ADDS classes 2..16 into the device array
 * d_counts[16] (uint64, caller-owned, caller zeroes it).  No host sync and
 * no closing (unless profiling is on): bin sizes stay on the device.
 * Classes 4..16 (021D..300) are exactly the range's (as tc_census_range).
 * Classes 2..3 use the kernels' owed-credit attribution (DESIGN.md reading
 * 21): dyad (u,v) adds n - |N(u)| - |N(v)| + |{x > u : x in N(u) & N(v)}|
 * to its class, plus one to the class of dyad (v,x) for every x > v in
 * N(u) & N(v).  Summed over a partition of [0, D) this is the paper's total
 * exactly; a single range's 012 / 102 may differ from tc_census_range and
 * its uint64 slots are exact only modulo 2^64 (they can be "negative"). */
tc_status tc_census_enqueue(const tc_graph *g, uint64_t dyad_begin, uint64_t dyad_end,
                            void *cuda_stream, uint64_t *d_counts);

/* Host closing (a5): counts[0], *c003_hi = C(n,3) - sum(counts[1..15]) in
 * 128-bit.  Returns TC_E_INVALID if the sum exceeds C(n,3). */
tc_status tc_close_census(uint64_t n, uint64_t counts[16], uint64_t *c003_hi);

/* Shard cuts: splits canonical dyads [0, D) into
 * `world` contiguous ranges of near-equal sum(cost[k] + kappa): the paper's
 * task-queue cut applied across GPUs.  bounds[r],
 * bounds[r+1] delimit rank r; bounds must hold world+1 entries (1 <= world
 * <= 1024).  bounds[r] = first k whose exclusive prefix of cost + kappa is
 * >= floor(T r / world), T = the total.  Host-only pure function over host
 * `cost` (length D). */
tc_status tc_shard_bounds_host(const uint64_t *cost, uint64_t D, int world, uint64_t kappa,
                               uint64_t *bounds);

/* The cut the multi-GPU census uses, on the device graph (host array of
 * world+1 entries): the same rule with kappa = 8 and cost[k] = the census
 * kernels' own work for dyad k = (u,v) -- t = |{w in N(u): w > u}| +
 * |{w in N(v): w > u}| merge trips, or, for a skewed-pair dyad (hub graphs,
 * census.cu: short list s, long list l, s (ceil(log2(l + 1)) + 4) < s + l),
 * s * ceil(log2(l + 1)) + 4 search units.  Computed once per world size and
 * cached in the graph.  Errors: TC_E_INVALID (world outside [1, 1024]). */
tc_status tc_shard_bounds(const tc_graph *g, int world, void *cuda_stream, uint64_t *bounds);

/* The multithreaded version's task queues, as a GPU scheduler (SURVEY.md
 * section 8(f) f3).  Fig. "Distributed Task Queue generation algorithm ...
 * Canonical Dyad(uniform distr.)": NsetSize += |N[u]| + |N[v]|
 * - 2; Fig. "... Canonical Dyad(non-uniform distr.)": NsetSize
 * += |S|, S = N[u] U N[v] \ {u,v}.  Walking the canonical dyads in the
 * algorithm's order, a queue is closed (thid + 1, NsetSize <- 0)
 * right after the dyad that makes NsetSize > max_nset_size; queues are
 * therefore contiguous dyad ranges, usable with tc_census_range.
 *   starts      host array: starts[q] = first canonical dyad of the q-th
 *               non-empty queue (a cut after the last dyad opens no queue);
 *               queue q = [starts[q], starts[q+1]) with starts[nqueues] = D
 *               implied.  Capacity `cap` entries (may be 0 with starts NULL
 *               to query the count).
 *   *nqueues    number of non-empty queues (always set on TC_OK/TC_E_RANGE)
 *   *total_nset aggregate NsetSize over all dyads (Table)
 * Errors: TC_E_INVALID (bad strategy / NULL outputs), TC_E_RANGE (more than
 * cap queues; nothing written to starts).  Synchronous on the stream. */
enum { TC_QUEUES_UNIFORM = 0, TC_QUEUES_NONUNIFORM = 1 };
tc_status tc_task_queues(const tc_graph *g, int strategy, uint64_t max_nset_size,
                         void *cuda_stream, uint64_t *starts, uint64_t cap, uint64_t *nqueues,
                         uint64_t *total_nset);

/* NCCL communicator.  Rank 0 calls tc_comm_unique_id, the 128 bytes are
 * broadcast by the caller (e.g. torch.distributed), then every rank calls
 * tc_comm_create.  NCCL is loaded lazily (libnccl.so.2, the copy torch
 * loaded if present); TC_E_NCCL if unavailable. */
tc_status tc_comm_unique_id(uint8_t id[128]);
tc_status tc_comm_create(const uint8_t id[128], int world, int rank, int device, tc_comm **out);

/* Optional alternative bootstrap: borrow an
 * existing ncclComm_t, e.g. torch's own through the private
 * ProcessGroupNCCL._comm_ptr().  Valid only because the library dlopens the
 * libnccl.so.2 already loaded into the process (torch's copy): the handle
 * must come from that same library.  World size, rank and device are read
 * from the communicator (ncclCommCount / UserRank / CuDevice).  The caller
 * keeps ownership: tc_comm_destroy frees only the wrapper.  Errors:
 * TC_E_INVALID (NULL), TC_E_NCCL (library or query failure). */
tc_status tc_comm_wrap(void *borrowed_nccl_comm, tc_comm **out);
void tc_comm_destroy(tc_comm *c);

/* Multi-GPU census: each rank holds the full graph (replicated CSR),
 * computes its work-balanced shard of canonical dyads (tc_shard_bounds: the
 * cut is computed once per world size and cached), and the 16 partial
 * counts are summed by one ncclAllReduce (uint64, sum) on the stream.  Every
 * rank receives the identical full census (closing done after the
 * reduction).  Synchronous. */
tc_status tc_census_multi(const tc_graph *g, tc_comm *comm, void *cuda_stream,
                          uint64_t counts[16], uint64_t *c003_hi);

/* Profiling: when on, every build / census records CUDA events around its
 * phases on the call's stream (adds one host sync per call). */
tc_status tc_profile_enable(tc_graph *g, int on);
tc_status tc_profile_get(const tc_graph *g, tc_profile *out);

/* Number of device kernels the last census/build call launched (for the
 * bench's gpu_launches claim). */
uint64_t tc_launch_count(const tc_graph *g);

/* Graph file reader (host, the step before the
 * path).  format: 0 auto (Pajek if the first non-comment line starts with
 * '*'), 1 Pajek (`*Vertices N` 1-based, `*Arcs` directed, `*Edges` -> two
 * arcs, `%` comments, trailing label/weight tokens ignored),
 * 2 edge list ("u v" per line, `#` comments, exactly two integer tokens;
 * S:152).  index_base: -1 auto (edge lists: 0 if any id is 0, else 1),
 * 0 or 1 forced (edge lists only).  On success *n, *m and two malloc'ed
 * 0-based arrays *src, *dst (release with tc_free_arcs).  Errors:
 * TC_E_INVALID (unreadable file, malformed record -- the message names the
 * line), TC_E_RANGE (id outside [1, N] in Pajek, 0 in a one-based list),
 * TC_E_OOM. */
tc_status tc_read_arcs(const char *path, int format, int index_base, uint64_t *n, uint32_t **src,
                       uint32_t **dst, uint64_t *m);
void tc_free_arcs(uint32_t *p);

/* Return the default allocator's cached device blocks (all devices) and the
 * pools' unused reservations to the driver; waits for every device to go
 * idle.  Call it before destroying a stream whose graphs or census calls
 * used the default allocator, or to give memory back to other libraries. */
tc_status tc_trim_memory(void);

const char *tc_last_error(void);
int tc_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* TRIADCENSUS_H */
