// census.cu -- a3 (merge/classify) and a4 (histogram reduction) kernels.
//
// For a canonical dyad (u, v), u < v, with pre = tag of v in N(u)
// (= IsEdge(u,v) + 2*IsEdge(v,u), the v0.4 pre-computed code),
// the B-M loop body (Fig. P:269-309) is evaluated as ONE sorted merge of the
// tagged rows A = N(u) and B = N(v) (entries (w<<2)|tag, sorted by w):
//   * every merged id w is an element of N(u) U N(v); tu / tv are its tags in
//     A / B (0 if absent): exactly IsEdge(u,w)+2*IsEdge(w,u) and
//     IsEdge(v,w)+2*IsEdge(w,v) of Fig. TriadCode;
//   * line 16's predicate  v < w or (u < w < v and not IsNeighbour(u,w))
//     never holds for w <= u, so the merge starts at the first entry w > u
//     of both rows (ups[u] in row u, dyad_pb in row v; csr_build.cu).  Then
//     the predicate is, for w from A (tu != 0): w > v, and for w only in B
//     (tu == 0): always (w > u by construction);
//   * code = pre | tu<<2 | tv<<4 (bit weights 1,2,4,8,16,32 of P:329-347) and
//     class = TriadTable[code], looked up in shared memory;
//   * the dyadic term n - |S| - 2 of line 14, with |S| = |N(u)|+|N(v)|-I-2
//     (I = |N(u) & N(v)|), is  n - du - dv  (added by the plan, schedule.cu)
//     plus one per element of I.  Elements w > u of I are met by this merge.
//     An element x < u of I is the smallest vertex of a triangle x < u < v;
//     it is met, instead, by the merge of dyad (x, u) as its canonical
//     intersection element v > u -- so every canonical intersection element
//     w > v of dyad (u, v) also adds the dyadic triad (v, w, u-excluded)
//     owed to dyad (v, w): one to class 102 if tv == 3 (v <-> w mutual),
//     else to class 012 (reading 21).  Each triangle's three
//     intersections are thus counted exactly once, and the census is the
//     paper's; only the split of 012/102 between dyad ranges moves.
//
// Merge-path form: trip t consumes exactly one list element (A first on
// equal ids), so a dyad of merge length t (entries > u of both rows) is
// exactly t trips; an intersection element is classified when its A copy is
// consumed (both tags are visible then) and its B twin is skipped.  A thread
// or a lane processes any diagonal range [d0, d1) after a merge-path split
// of d0.  Rows end in a sentinel (csr_build.cu), so the loop has no bounds
// checks, the next element of each list is loaded one consumption ahead, and
// the thread bin prefetches both rows into L2 when a dyad starts.
// Thread-bin warps hold dyads of identical merge length, so every lane runs
// the same trip count (no divergence); warp items split one dyad over 32
// lanes.
//
// a4: per thread, one uint64 of 16 4-bit class counters; a canonical trip
// adds the 64-bit increment table[code] (one nibble for its class, plus one
// for the dyadic correction above), spilled every <= 15 trips into two
// uint64 of 8-bit counters (even / odd classes), which a warp flushes (REDUX
// sum per class) into per-warp shared totals before they can overflow;
// blocks end with one global atomicAdd per class.
#include <atomic>

#include "census.cuh"

namespace tc {

// TriadTable, 0-based classes in the paper's order 003..300.
// The literal B-M 2001 TRICODES table minus one (reading 1); the
// oracle derives its own table by orbit enumeration and the tests compare.
__constant__ uint8_t c_triad_table[64] = {
    0, 1, 1, 2, 1, 3, 5, 7, 1, 5, 4, 6, 2, 7, 6, 10, 1, 5, 3, 7, 4, 8, 8, 12, 5, 9, 8, 13, 6, 13, 11, 14,
    1, 4, 5, 6, 5, 8, 9, 13, 3, 8, 8, 11, 7, 12, 13, 14, 2, 6, 7, 10, 6, 11, 13, 14, 7, 13, 12, 14, 10, 14, 14, 15};

namespace {

constexpr int kWarps = kCensusThreads / 32;
constexpr uint64_t kNib = 0x0F0F0F0F0F0F0F0Full;

struct Acc {
    uint64_t n4;            // 16 x 4-bit counters, nibble k = class k (0-based)
    uint64_t ev8, od8;      // 8-bit counters: byte j = class 2j / class 2j+1
    uint32_t pending;       // trips since the last warp flush (<= 255)
    uint64_t dy012, dy102;  // dyadic triads of classes 012 / 102
};

__device__ __forceinline__ void acc_init(Acc &c) {
    c.n4 = c.ev8 = c.od8 = 0;
    c.pending = 0;
    c.dy012 = c.dy102 = 0;
}

__device__ __forceinline__ void add_dyadic(Acc &c, uint32_t pre, uint64_t x) {
    if (pre == 3u) c.dy102 += x;
    else c.dy012 += x;
}

// nibbles -> bytes (nibble 0 is moved to the dyadic counters by the caller)
__device__ __forceinline__ void spill(Acc &c) {
    c.ev8 += c.n4 & (kNib & ~0xFull);
    c.od8 += (c.n4 >> 4) & kNib;
    c.n4 = 0;
}

__device__ __forceinline__ uint64_t lds_u64(uint32_t addr) {
    uint64_t v;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(addr));
    return v;
}

// v = canonical ? shared u64 at addr : dflt (the load is predicated off, so
// non-canonical lanes cost no shared-memory wavefront)
__device__ __forceinline__ uint64_t lds_u64_if(uint32_t addr, bool p, uint64_t dflt) {
    uint64_t v = dflt;
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.shared.u64 %0, [%1];\n\t}"
        : "+l"(v)
        : "r"(addr), "r"((uint32_t)p));
    return v;
}

// Warp-level flush (all 32 lanes active): each class 1..15 is summed over
// the warp with one REDUX and lane 0 adds it to the warp's own shared slots
// (plain adds; 64-bit shared atomics are CAS loops on sm_100).
__device__ __forceinline__ void warp_flush(Acc &c, unsigned long long *wsh) {
    const uint32_t lane = threadIdx.x & 31;
#pragma unroll
    for (int k = 1; k < 16; k++) {
        uint32_t x = (uint32_t)(((k & 1) ? c.od8 : c.ev8) >> (8 * (k >> 1))) & 255u;
        uint32_t s = __reduce_add_sync(0xffffffffu, x);
        if (lane == 0) wsh[k] += s;
    }
    c.ev8 = c.od8 = 0;
    c.pending = 0;
}

// flush before `len` more trips if any lane could overflow a byte counter
__device__ __forceinline__ void warp_reserve(Acc &c, unsigned long long *wsh, uint32_t len) {
    if (__any_sync(0xffffffffu, c.pending + len > 255u)) warp_flush(c, wsh);
    c.pending += len;
}

// merge-path split of diagonal d: number of A elements among the first d
// merged elements (A before B on equal ids)
__device__ __forceinline__ uint32_t merge_path(const uint32_t *__restrict__ A, uint32_t a,
                                               const uint32_t *__restrict__ B, uint32_t b,
                                               uint32_t d) {
    uint32_t lo = d > b ? d - b : 0u, hi = d < a ? d : a;
    while (lo < hi) {
        uint32_t mid = (lo + hi) >> 1;
        if ((__ldg(A + mid) | 3u) <= (__ldg(B + (d - mid - 1)) | 3u)) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Classify merge diagonals [d0, d1) of dyad (u, v).  A = adj[oa, oa+a) (the
// entries w > u of N(u)), B = adj[ob, ob+b) (the entries w > u of N(v)),
// both followed by more of their row and a sentinel; kv = v<<2|3; tab =
// shared address of the 128-entry uint64 increment table.  The caller has
// reserved d1 - d0 byte-counter increments (warp_reserve).
// LA2: two elements of look-ahead per list instead of one (the load issued
// at a trip is consumed two consumptions of that list later; two more
// registers and selects per trip)
template <bool PRED, bool LA2 = false>
__device__ __forceinline__ void merge_diag(const uint32_t *__restrict__ adj, uint32_t oa,
                                           uint32_t a, uint32_t ob, uint32_t b, uint32_t kv,
                                           uint32_t pre, uint32_t d0, uint32_t d1, uint32_t tab,
                                           Acc &c) {
    uint32_t i = 0;
    if (d0 > 0) i = merge_path(adj + oa, a, adj + ob, b, d0);
    uint32_t pa = oa + i, pb = ob + (d0 - i);
    uint32_t lastA = i > 0 ? (__ldg(adj + pa - 1) | 3u) : 0u;
    // current heads and the next elements (sentinel-terminated rows; the
    // look-ahead may read past a sentinel into the next row or the slack)
    uint32_t x = __ldg(adj + pa), xn = __ldg(adj + pa + 1);
    uint32_t y = __ldg(adj + pb), yn = __ldg(adj + pb + 1);
    uint32_t xnn = LA2 ? __ldg(adj + pa + 2) : 0u, ynn = LA2 ? __ldg(adj + pb + 2) : 0u;
    // canonical increments of this pre: 16 entries (tu | tv << 2), 8 bytes each,
    // one 128-byte bank row
    const uint32_t tabp = PRED ? tab + 128u * pre : tab + 8u * pre;
    uint32_t t = d0;
    while (t < d1) {
        const uint32_t lim = min(d1, t + 15u);   // nibble counters hold 15
#pragma unroll 2   // measured: 2 beats the default 4 (C3 thread bin 0.889 vs 0.899 ms) and 8
        for (; t < lim; t++) {
            const uint32_t kx = x | 3u, ky = y | 3u;
            const bool ta = kx <= ky;            // consume A (ties: A first)
            const bool tb = ky <= kx;            // B's id is the merged id
            // tu = tag in A, tv = tag in B; PRED: 8 * (tu | tv << 2), else
            // 8 * (code - pre) = tu << 5 | tv << 7
            const uint32_t ca = ta ? ((x << (PRED ? 3 : 5)) & (PRED ? 0x18u : 0x60u)) : 0u;
            const uint32_t cb = tb ? ((y << (PRED ? 5 : 7)) & (PRED ? 0x60u : 0x180u)) : 0u;
            // A element: w > v.  B-only element: canonical unless it is the
            // B twin of the A element just consumed (classified already).
            const bool canon = ta ? (kx > kv) : (ky != lastA);
            // non-canonical: an intersection element u < w < v adds nibble 0
            // (own I); only canonical trips read the table (predicated LDS)
            if (PRED)
                c.n4 += lds_u64_if(tabp + (ca | cb), canon, (ta && tb) ? 1ull : 0ull);
            else   // thread bin: unpredicated, non-canonical half of the table
                c.n4 += lds_u64(tabp + (ca | cb | (canon ? 512u : 0u)));
            lastA = ta ? kx : lastA;
            pa += ta;
            pb += !ta;
            if (LA2) {
                const uint32_t nv = __ldg(adj + (ta ? pa : pb) + 2u);
                x = ta ? xn : x;
                xn = ta ? xnn : xn;
                xnn = ta ? nv : xnn;
                y = ta ? y : yn;
                yn = ta ? yn : ynn;
                ynn = ta ? ynn : nv;
            } else {
                const uint32_t nv = __ldg(adj + (ta ? pa : pb) + 1u);
                x = ta ? xn : x;
                xn = ta ? nv : xn;
                y = ta ? y : yn;
                yn = ta ? yn : nv;
            }
        }
        // nibble 0 counts this dyad's intersection elements w > u (own-I)
        add_dyadic(c, pre, c.n4 & 15u);
        spill(c);
    }
}

// measured slower (C3 thread bin 1.49 ms at 54 registers, 1.03 ms capped at
// 48; the shared table: 0.87 ms): the trip loop is issue-bound, and the
// 64-bit variable shift + selects cost more issue slots than one LDS.64
#ifndef TC_WARP_LA2
#define TC_WARP_LA2 false
#endif
#ifndef TC_THREAD_LA2
#define TC_THREAD_LA2 false
#endif

#ifndef TC_THREAD_REGTAB
#define TC_THREAD_REGTAB 0
#endif

// Thread bin, TriadTable out of the trip loop (SURVEY.md 8(a) "Table in
// registers"): a canonical trip counts its tag pair, not its class -- nibble
// idx = tu | tv << 2 of a per-thread uint64 (no shared-memory load, no bank
// conflicts); nibble 0 (tu = tv = 0 never occurs in a canonical trip) counts
// the non-canonical intersection elements u < w < v (own I).  Every <= 15
// trips the nibbles move to 8-bit counters of the dyad's pre (three pairs of
// uint64: even / odd idx); the warp flush (every <= 255 trips per lane) maps
// (pre, idx) to the class TriadTable[pre | tu << 2 | tv << 4] and,
// for idx with tu, tv != 0 (canonical intersection elements w > v), adds the
// dyad's own I and the owed dyadic triad (class 102 if tv == 3, else 012).
#if TC_THREAD_REGTAB
struct AccT {
    uint64_t n4;                     // nibble idx: canonical trips with tags idx
    uint64_t e1, o1, e2, o2, e3, o3; // bytes: pre p, even idx / odd idx (byte idx >> 1)
    uint32_t pending;
    uint64_t dy012, dy102;
};

__device__ __forceinline__ void acct_init(AccT &c) {
    c.n4 = c.e1 = c.o1 = c.e2 = c.o2 = c.e3 = c.o3 = 0;
    c.pending = 0;
    c.dy012 = c.dy102 = 0;
}

__device__ __forceinline__ void acct_spill(AccT &c, uint32_t pre) {
    const uint64_t own = c.n4 & 15u;            // non-canonical intersections
    if (pre == 3u) c.dy102 += own;
    else c.dy012 += own;
    const uint64_t E = c.n4 & (kNib & ~0xFull), O = (c.n4 >> 4) & kNib;
    c.e1 += pre == 1u ? E : 0ull;
    c.o1 += pre == 1u ? O : 0ull;
    c.e2 += pre == 2u ? E : 0ull;
    c.o2 += pre == 2u ? O : 0ull;
    c.e3 += pre == 3u ? E : 0ull;
    c.o3 += pre == 3u ? O : 0ull;
    c.n4 = 0;
}

template <uint32_t P>
__device__ __forceinline__ void acct_flush_pre(uint64_t &e, uint64_t &o, uint32_t lane,
                                               unsigned long long *wsh) {
    if (!__any_sync(0xffffffffu, (e | o) != 0ull)) return;
#pragma unroll
    for (uint32_t idx = 1; idx < 16; idx++) {
        const uint32_t x = (uint32_t)(((idx & 1u) ? o : e) >> (8u * (idx >> 1))) & 255u;
        const uint32_t sum = __reduce_add_sync(0xffffffffu, x);
        if (lane == 0 && sum) {
            const uint32_t tu = idx & 3u, tv = idx >> 2;
            wsh[c_triad_table[P | idx << 2]] += sum;
            if (tu && tv) {
                wsh[P == 3u ? 2 : 1] += sum;     // own I of dyad (u, v)
                wsh[tv == 3u ? 2 : 1] += sum;    // owed to dyad (v, w)
            }
        }
    }
    e = o = 0;
}

__device__ __forceinline__ void acct_flush(AccT &c, unsigned long long *wsh) {
    const uint32_t lane = threadIdx.x & 31;
    acct_flush_pre<1u>(c.e1, c.o1, lane, wsh);
    acct_flush_pre<2u>(c.e2, c.o2, lane, wsh);
    acct_flush_pre<3u>(c.e3, c.o3, lane, wsh);
    c.pending = 0;
}

__device__ __forceinline__ void acct_reserve(AccT &c, unsigned long long *wsh, uint32_t len) {
    if (__any_sync(0xffffffffu, c.pending + len > 255u)) acct_flush(c, wsh);
    c.pending += len;
}

// thread-bin merge of a whole dyad: A = adj[pa..), B = adj[pb..), t trips
__device__ __forceinline__ void merge_thread_reg(const uint32_t *__restrict__ adj, uint32_t pa,
                                                 uint32_t pb, uint32_t kv, uint32_t pre,
                                                 uint32_t t1, AccT &c) {
    uint32_t lastA = 0u;
    uint32_t x = __ldg(adj + pa), xn = __ldg(adj + pa + 1);
    uint32_t y = __ldg(adj + pb), yn = __ldg(adj + pb + 1);
    uint32_t t = 0;
    while (t < t1) {
        const uint32_t lim = min(t1, t + 15u);   // nibble counters hold 15
#pragma unroll 2
        for (; t < lim; t++) {
            const uint32_t kx = x | 3u, ky = y | 3u;
            const bool ta = kx <= ky;            // consume A (ties: A first)
            const bool tb = ky <= kx;            // B's id is the merged id
            const uint32_t ca = ta ? ((x & 3u) << 2) : 0u;    // 4 tu
            const uint32_t cb = tb ? ((y & 3u) << 4) : 0u;    // 16 tv
            const bool canon = ta ? (kx > kv) : (ky != lastA);
            const uint32_t sh = canon ? (ca | cb) : 0u;       // 4 idx, or nibble 0
            c.n4 += (canon || (ta && tb)) ? (1ull << sh) : 0ull;
            lastA = ta ? kx : lastA;
            pa += ta;
            pb += !ta;
            const uint32_t nv = __ldg(adj + (ta ? pa : pb) + 1u);
            x = ta ? xn : x;
            xn = ta ? nv : xn;
            y = ta ? y : yn;
            yn = ta ? yn : nv;
        }
        acct_spill(c, pre);
    }
}

__device__ __forceinline__ void block_finish_t(AccT &c, unsigned long long (*wsh)[16],
                                               unsigned long long *d_counts) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    acct_flush(c, wsh[warp]);
    unsigned long long d0 = c.dy012, d1 = c.dy102;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        d0 += __shfl_xor_sync(0xffffffffu, d0, o);
        d1 += __shfl_xor_sync(0xffffffffu, d1, o);
    }
    if (lane == 0) {
        wsh[warp][1] += d0;
        wsh[warp][2] += d1;
    }
    __syncthreads();
    if (threadIdx.x >= 1 && threadIdx.x < 16) {
        unsigned long long s = 0;
#pragma unroll
        for (int w = 0; w < kWarps; w++) s += wsh[w][threadIdx.x];
        if (s) atomicAdd(&d_counts[threadIdx.x], s);
    }
}

#endif  // TC_THREAD_REGTAB

// shared increment tables: thread bin: 128 entries (canonical << 6 | code);
// warp bin: 64 entries (pre << 4 | tu | tv << 2), canonical trips only; code = pre | tu << 2 | tv << 4: one nibble at 4 * class, and,
// both tags set (an intersection element w > v), nibble 0 (own I) plus one
// nibble at class 102 if tv == 3 else 012 (the dyadic triad owed to dyad
// (v, w)).  A non-canonical trip adds nibble 0 iff both tags are set (an
// intersection element u < w < v; the dyad's own intersection count I,
// moved to 012 / 102 by pre at every spill).  Every nibble gets at most 1
// per trip.  The warp bin (one pre per warp) reads only the canonical half,
// with a predicated load (a 128-byte bank row per pre: no bank conflicts);
// the thread bin (mixed pre) measured faster with one unpredicated load.  wsh: per-warp totals.
template <bool WARPBIN>
__device__ __forceinline__ void block_setup(unsigned long long *tab,
                                            unsigned long long (*wsh)[16]) {
    if (threadIdx.x < (WARPBIN ? 64 : 128)) {
        const uint32_t code = threadIdx.x & 63u, canon = threadIdx.x >> 6;
        const uint32_t tu = (code >> 2) & 3u, tv = code >> 4;
        unsigned long long inc = (tu && tv) ? 1ull : 0ull;
        if (canon || WARPBIN) {
            inc += 1ull << (4u * c_triad_table[code]);
            if (tu && tv) inc += 1ull << (tv == 3u ? 8u : 4u);
        }
        if (WARPBIN) tab[(code & 3u) << 4 | tu | tv << 2] = inc;   // pre << 4 | tu | tv << 2
        else tab[threadIdx.x] = inc;                               // canonical << 6 | code
    }
    for (int i = threadIdx.x; i < kWarps * 16; i += blockDim.x) (&wsh[0][0])[i] = 0;
    __syncthreads();
}

__device__ __forceinline__ void block_finish(Acc &c, unsigned long long (*wsh)[16],
                                             unsigned long long *d_counts) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    warp_flush(c, wsh[warp]);
    unsigned long long d0 = c.dy012, d1 = c.dy102;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        d0 += __shfl_xor_sync(0xffffffffu, d0, o);
        d1 += __shfl_xor_sync(0xffffffffu, d1, o);
    }
    if (lane == 0) {
        wsh[warp][1] += d0;
        wsh[warp][2] += d1;
    }
    __syncthreads();
    if (threadIdx.x >= 1 && threadIdx.x < 16) {
        unsigned long long s = 0;
#pragma unroll
        for (int w = 0; w < kWarps; w++) s += wsh[w][threadIdx.x];
        if (s) atomicAdd(&d_counts[threadIdx.x], s);
    }
}

// prefetch the 128-byte lines of adj[o, o+len] into L2 (fire and forget;
// prefetch.global.L1 measured no different)
__device__ __forceinline__ void prefetch_row_l2(const uint32_t *adj, uint32_t o, uint32_t len) {
    const char *p = reinterpret_cast<const char *>(adj + o);
    const char *e = reinterpret_cast<const char *>(adj + o + len);
    for (const char *q = reinterpret_cast<const char *>(reinterpret_cast<uintptr_t>(p) & ~(uintptr_t)127);
         q <= e; q += 128)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(q));
}

// merge of a warp-bin dyad k: starts and lengths of A and B
struct WarpDyad {
    uint32_t oa, a, ob, b, e;
};
__device__ __forceinline__ WarpDyad warp_dyad(const BinLists &L, const uint32_t *__restrict__ off,
                                              const uint32_t *__restrict__ ups, uint32_t k) {
    WarpDyad w;
    const uint32_t u = __ldg(L.du + k);
    w.e = __ldg(L.de + k);
    w.oa = __ldg(ups + u);
    w.a = __ldg(off + u + 1) - 1u - w.oa;
    w.ob = __ldg(L.dpb + k);
    w.b = __ldg(off + (w.e >> 2) + 1) - 1u - w.ob;
    return w;
}

// Thread-bin work is handed out dynamically: a block takes the next unit
// (a half or a quarter of a plan tile's item slots, in canonical tile order)
// from a global cursor, so the kernel's tail is at most one unit per
// resident block instead of a static round-robin's extra tiles.
// Units per tile (host-chosen, launch_bins): halves when there are >= 4 tiles
// per resident block (C3: 0.891 vs 0.899 ms), quarters otherwise (C2: 117
// tiles for 740 blocks; halves cost 0.155 vs 0.13 ms there).
static_assert(kPlanTile % (4 * kCensusThreads) == 0, "unit = whole block rounds");

__device__ __forceinline__ uint64_t next_unit(unsigned long long *cursor, uint32_t *unit_s) {
    __syncthreads();   // every warp is done with the previous unit's unit_s
    if (threadIdx.x == 0) *unit_s = (uint32_t)atomicAdd(cursor, 1ull);
    __syncthreads();
    return *unit_s;
}

// thread bin: one thread per dyad.  Block-persistent over tiles of
// kPlanTile consecutive canonical dyads; inside a tile the plan ordered the
// thread-bin dyads by merge length, so each warp's lanes run equal trip
// counts while the tile keeps the N(u) rows of nearby u hot in L1/L2.
// (an explicit minimum of 1 block per SM lets ptxas take 56 registers, 4
// blocks/SM: 0.87 ms; the plain bound keeps 48 registers, 5 blocks/SM)
#ifdef TC_THREAD_MINB
__global__ void __launch_bounds__(kCensusThreads, TC_THREAD_MINB)
#else
__global__ void __launch_bounds__(kCensusThreads)
#endif
k_census_thread(const BinItemT *__restrict__ items, const uint32_t *__restrict__ tile_count,
                uint64_t ntiles, const uint32_t *__restrict__ adj, unsigned long long *d_counts,
                unsigned long long *cursor, uint32_t upt) {
    __shared__ unsigned long long wsh[kWarps][16];
#if TC_THREAD_REGTAB
    for (int i = threadIdx.x; i < kWarps * 16; i += blockDim.x) (&wsh[0][0])[i] = 0;
    __syncthreads();
    AccT c;
    acct_init(c);
#else
    __shared__ unsigned long long tab_s[128];
    block_setup<false>(tab_s, wsh);
    const uint32_t tab = (uint32_t)__cvta_generic_to_shared(tab_s);
    Acc c;
    acc_init(c);
#endif
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ uint32_t unit_s;
    const uint32_t unit_dyads = kPlanTile / upt;
    for (uint64_t unit = next_unit(cursor, &unit_s); unit < ntiles * upt;
         unit = next_unit(cursor, &unit_s)) {
        const uint64_t tile = unit / upt;
        const uint32_t part = (uint32_t)(unit % upt) * unit_dyads;
        const uint32_t cnt = min(__ldg(tile_count + tile), part + unit_dyads);
        const BinItemT *it = items + tile * kPlanTile;
        for (uint32_t base = part + warp * 32; base < cnt; base += kCensusThreads) {
            const bool valid = base + lane < cnt;
            BinItemT e{0, 0, 0, 0};
            if (valid) {
                e = it[base + lane];
                // item word 3 = t | |A| << 16: prefetch exactly the B part
                // (N(v) above u) into L2.  A (N(u) above u) is shared by the
                // tile's dyads of the same u and stays cached: prefetching it
                // too measured 0.856 ms, t entries of both rows 0.884, B only
                // 0.830
                const uint32_t alen = e.t >> 16;
                e.t &= 0xffffu;
                prefetch_row_l2(adj, e.pb, e.t - alen);
            }
#if TC_THREAD_REGTAB
            acct_reserve(c, wsh[warp], e.t);
            if (valid) merge_thread_reg(adj, e.pa, e.pb, e.e | 3u, e.e & 3u, e.t, c);
        }
    }
    block_finish_t(c, wsh, d_counts);
#else
            warp_reserve(c, wsh[warp], e.t);
            if (valid)
                merge_diag<false, TC_THREAD_LA2>(adj, e.pa, 0, e.pb, 0, e.e | 3u, e.e & 3u, 0,
                                                 e.t, tab, c);
        }
    }
    block_finish(c, wsh, d_counts);
#endif
}

// warp bin: a warp takes the next item from a global cursor (dynamic, so
// the tail is one item per resident warp)
__device__ __forceinline__ uint64_t next_item(unsigned long long *cursor) {
    unsigned long long it = 0;
    if ((threadIdx.x & 31) == 0) it = atomicAdd(cursor, 1ull);
    return __shfl_sync(0xffffffffu, it, 0);
}

// ---------------------------------------------------------------------------
// Skewed-pair items (schedule.cu sparse_mode): instead of merging a short
// list with a long one, every entry of the short list is looked up in the
// long list by binary search, and the long list's own contribution is read
// from the tag prefix counts.  The same canonical triads are counted as by
// the merge (census.cu header):
//   mode 1, iterate A (entries w > u of N(u)), search B (entries > u of
//   N(v)): w > v -> class T[pre | tu<<2 | tv<<4]; an intersection element
//   (tv != 0) adds own I and, for w > v, the owed dyadic triad; B-only
//   elements are all canonical with T[pre | tv<<4]: item chunk 0 adds every B
//   entry by tag, each intersection element found takes its one back.
//   mode 2, iterate B, search A: tu == 0 -> T[pre | tv<<4]; an intersection
//   element adds own I and, for w > v, T[pre | tu<<2 | tv<<4] + the owed
//   dyadic triad; A-only elements w > v are canonical with T[pre | tu<<2]:
//   chunk 0 adds every A entry after v by tag, each intersection w > v
//   takes its one back.
// Class counts go to block shared u64 counters (wrapping adds: a take-back
// may run ahead of its chunk-0 add; the totals are exact).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t lower_id(const uint32_t *__restrict__ L, uint32_t len,
                                             uint32_t x) {
    uint32_t lo = 0, hi = len;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if ((__ldg(L + mid) >> 2) < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// K independent lower_id searches in lockstep (fixed-step branch-free binary
// search: the same number of probes for every key of the same list), so K
// dependent-load chains are in flight per lane instead of one (the skewed
// path is bound by the probes' L2 latency)
template <int K>
__device__ __forceinline__ void tag_in_k(const uint32_t *__restrict__ L, uint32_t len,
                                         const uint32_t (&x)[K], uint32_t (&tag)[K]) {
    uint32_t lo[K];
#pragma unroll
    for (int q = 0; q < K; q++) lo[q] = 0;
    uint32_t step = len ? 1u << (31 - __clz(len)) : 0u;
    for (; step; step >>= 1) {
#pragma unroll
        for (int q = 0; q < K; q++) {
            const uint32_t p = lo[q] + step;
            if (p <= len && (__ldg(L + p - 1) >> 2) < x[q]) lo[q] = p;
        }
    }
#pragma unroll
    for (int q = 0; q < K; q++) {
        tag[q] = 0u;
        if (lo[q] < len) {
            const uint32_t e = __ldg(L + lo[q]);
            if ((e >> 2) == x[q]) tag[q] = e & 3u;
        }
    }
}

#ifndef TC_SP_K
#define TC_SP_K 2
#endif

// skewed-pair class counts: per-warp uint32 shared counters (native 32-bit
// shared atomics; 64-bit shared atomics are CAS loops on sm_100), added
// modulo 2^32 (a take-back may precede its add) and moved, sign-extended,
// into the warp's uint64 totals after every item (an item's net count per
// class is below 2^31 in magnitude: <= 3 * 256 entries + one row's tags)
#ifndef TC_SP_U32
#define TC_SP_U32 1
#endif
#if TC_SP_U32
typedef uint32_t sp_t;
#else
typedef unsigned long long sp_t;
#endif
__device__ __forceinline__ void sp_add(sp_t *sp, uint32_t cls, uint32_t x) {
#if TC_SP_U32
    atomicAdd(&sp[cls], x);
#else
    atomicAdd(&sp[cls], (unsigned long long)(long long)(int32_t)x);
#endif
}

__device__ __forceinline__ void sp_drain(sp_t *sp, unsigned long long *wsh) {
    __syncwarp();
    const uint32_t lane = threadIdx.x & 31;
    if (lane < 16) {
#if TC_SP_U32
        wsh[lane] += (unsigned long long)(long long)(int32_t)sp[lane];
#else
        wsh[lane] += sp[lane];
#endif
        sp[lane] = 0;
    }
    __syncwarp();
}

__device__ void sparse_item(const uint32_t *__restrict__ adj, const uint64_t *__restrict__ P,
                            const WarpDyad &w, uint32_t mode, uint32_t d0, uint32_t d1,
                            sp_t *sp) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t v = w.e >> 2, pre = w.e & 3u;
    const uint32_t minus1 = ~0u;
    uint32_t own = 0, o012 = 0, o102 = 0;
    constexpr int K = TC_SP_K;
    if (mode == 1u) {
        for (uint32_t j0 = d0 + lane; j0 < d1; j0 += 32 * K) {
            uint32_t xs[K], ids[K], tvs[K];
#pragma unroll
            for (int q = 0; q < K; q++) {
                const uint32_t j = j0 + 32 * q;
                xs[q] = j < d1 ? __ldg(adj + w.oa + j) : 0xffffffffu;
                ids[q] = xs[q] >> 2;
            }
            tag_in_k<K>(adj + w.ob, w.b, ids, tvs);
#pragma unroll
            for (int q = 0; q < K; q++) {
                const uint32_t id = ids[q], tu = xs[q] & 3u, tv = tvs[q];
                if (j0 + 32 * q >= d1 || id == v) continue;
                if (id > v) sp_add(sp, c_triad_table[pre | tu << 2 | tv << 4], 1u);
                if (tv) {
                    own++;
                    if (id > v) {
                        o102 += tv == 3u;
                        o012 += tv != 3u;
                    }
                    sp_add(sp, c_triad_table[pre | tv << 4], minus1);
                }
            }
        }
        if (d0 == 0 && lane == 0) {
            const uint64_t dd = __ldg(P + w.ob + w.b) - __ldg(P + w.ob);
            const uint32_t c1 = (uint32_t)(dd >> 32), c2 = (uint32_t)dd;
            const uint32_t cnt[4] = {0u, c1, c2, w.b - c1 - c2};
            for (uint32_t t = 1; t <= 3; t++)
                if (cnt[t]) sp_add(sp, c_triad_table[pre | t << 4], cnt[t]);
        }
    } else {
        for (uint32_t j0 = d0 + lane; j0 < d1; j0 += 32 * K) {
            uint32_t ys[K], ids[K], tus[K];
#pragma unroll
            for (int q = 0; q < K; q++) {
                const uint32_t j = j0 + 32 * q;
                ys[q] = j < d1 ? __ldg(adj + w.ob + j) : 0xffffffffu;
                ids[q] = ys[q] >> 2;
            }
            tag_in_k<K>(adj + w.oa, w.a, ids, tus);
#pragma unroll
            for (int q = 0; q < K; q++) {
                const uint32_t id = ids[q], tv = ys[q] & 3u, tu = tus[q];
                if (j0 + 32 * q >= d1) continue;
                if (!tu) {
                    sp_add(sp, c_triad_table[pre | tv << 4], 1u);
                } else {
                    own++;
                    if (id > v) {
                        sp_add(sp, c_triad_table[pre | tu << 2 | tv << 4], 1u);
                        o102 += tv == 3u;
                        o012 += tv != 3u;
                        sp_add(sp, c_triad_table[pre | tu << 2], minus1);
                    }
                }
            }
        }
        if (d0 == 0 && lane == 0) {
            const uint32_t pv = lower_id(adj + w.oa, w.a, v) + 1u;   // entries after v
            const uint64_t dd = __ldg(P + w.oa + w.a) - __ldg(P + w.oa + pv);
            const uint32_t c1 = (uint32_t)(dd >> 32), c2 = (uint32_t)dd;
            const uint32_t cnt[4] = {0u, c1, c2, (w.a - pv) - c1 - c2};
            for (uint32_t t = 1; t <= 3; t++)
                if (cnt[t]) sp_add(sp, c_triad_table[pre | t << 2], cnt[t]);
        }
    }
    // own I -> the dyad's dyadic class; owed dyadic triads by tv
    own = __reduce_add_sync(0xffffffffu, own);
    o012 = __reduce_add_sync(0xffffffffu, o012);
    o102 = __reduce_add_sync(0xffffffffu, o102);
    if (lane == 0) {
        if (own) sp_add(sp, pre == 3u ? 2u : 1u, own);
        if (o012) sp_add(sp, 1u, o012);
        if (o102) sp_add(sp, 2u, o102);
    }
}

// warp bin: one warp per item = one dyad's diagonals [d0, d1), 32 lane
// segments of <= kLaneSpan diagonals each; or a skewed-pair item (pad =
// mode) = short-list entries [d0, d1)
__global__ void __launch_bounds__(kCensusThreads)
k_census_warp(const BinLists L, const uint32_t *__restrict__ off, const uint32_t *__restrict__ ups,
              const uint32_t *__restrict__ adj, unsigned long long *d_counts) {
    __shared__ unsigned long long tab_s[64];
    __shared__ unsigned long long wsh[kWarps][16];
    block_setup<true>(tab_s, wsh);
    const uint32_t tab = (uint32_t)__cvta_generic_to_shared(tab_s);
    Acc c;
    acc_init(c);
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ sp_t spw[kWarps][16];   // skewed-pair class counts, per warp (wrapping)
    if (lane < 16) spw[warp][lane] = 0;
    __syncwarp();
    const uint64_t count = *L.w_count;
    for (uint64_t it = next_item(L.wcursor); it < count; it = next_item(L.wcursor)) {
        const BinItemW e = L.w[it];
        const WarpDyad w = warp_dyad(L, off, ups, e.k);
        if (e.pad) {   // warp-uniform
            sparse_item(adj, L.tagpre, w, e.pad, e.d0, e.d1, spw[warp]);
            sp_drain(spw[warp], wsh[warp]);
            continue;
        }
        const uint32_t span = e.d1 - e.d0, per = (span + 31) >> 5;
        const uint32_t d0 = e.d0 + min(span, lane * per), d1 = e.d0 + min(span, (lane + 1) * per);
        warp_reserve(c, wsh[warp], d1 - d0);
        if (d0 < d1)
            merge_diag<true, TC_WARP_LA2>(adj, w.oa, w.a, w.ob, w.b, w.e | 3u, w.e & 3u, d0, d1,
                                          tab, c);
    }
    block_finish(c, wsh, d_counts);
}

// ---------------------------------------------------------------------------
// 64-type (non-isomorphic) census: the same
// merge, but every canonical trip counts its TriadCode itself (P:327, P:343:
// "returns this value + 1 if main algorithm calculates non-isomorphic triad
// census"), in a per-warp shared uint32 histogram of 64 codes (flushed to
// per-warp uint64 totals before it can overflow); dyadic triads go to code
// pre (reading 12), the owed triad of a canonical intersection to
// code tv.  Code 0 is closed on the host.
// ---------------------------------------------------------------------------
struct Acc64 {
    uint64_t dy[3];          // dyadic triads of codes 1, 2, 3 (= pre)
    uint32_t pending;        // trips since the last flush
};

__device__ __forceinline__ void merge_diag64(const uint32_t *__restrict__ adj, uint32_t oa,
                                             uint32_t a, uint32_t ob, uint32_t b, uint32_t kv,
                                             uint32_t pre, uint32_t d0, uint32_t d1,
                                             uint32_t *hist, Acc64 &c) {
    uint32_t i = 0;
    if (d0 > 0) i = merge_path(adj + oa, a, adj + ob, b, d0);
    uint32_t pa = oa + i, pb = ob + (d0 - i);
    uint32_t lastA = i > 0 ? (__ldg(adj + pa - 1) | 3u) : 0u;
    uint32_t x = __ldg(adj + pa), y = __ldg(adj + pb);
    uint32_t I = 0;
    for (uint32_t t = d0; t < d1; t++) {
        const uint32_t kx = x | 3u, ky = y | 3u;
        const bool ta = kx <= ky;
        const bool tb = ky <= kx;
        const uint32_t ca = ta ? ((x << 2) & 12u) : 0u;
        const uint32_t cb = tb ? ((y << 4) & 48u) : 0u;
        const bool canon = ta ? (kx > kv) : (ky != lastA);
        I += (uint32_t)(ta & tb);
        if (canon) {
            atomicAdd(&hist[pre | ca | cb], 1u);
            if (ta & tb) atomicAdd(&hist[y & 3u], 1u);   // owed to dyad (v, w)
        }
        lastA = ta ? kx : lastA;
        pa += ta;
        pb += !ta;
        const uint32_t nv = __ldg(adj + (ta ? pa : pb));
        x = ta ? nv : x;
        y = ta ? y : nv;
    }
    c.dy[pre - 1] += I;
}

// flush the warp's uint32 histogram into its uint64 totals (all lanes active)
__device__ __forceinline__ void warp_flush64(uint32_t *hist, unsigned long long *tot, Acc64 &c) {
    __syncwarp();
    const uint32_t lane = threadIdx.x & 31;
    for (int k = lane; k < 64; k += 32) {
        tot[k] += hist[k];
        hist[k] = 0;
    }
    __syncwarp();
    c.pending = 0;
}

// a trip adds at most 1 to any code (its own code is >= 4, the owed dyadic
// code is 1..3)
__device__ __forceinline__ void warp_reserve64(uint32_t *hist, unsigned long long *tot, Acc64 &c,
                                               uint32_t len) {
    if (__any_sync(0xffffffffu, c.pending + len > (1u << 26))) warp_flush64(hist, tot, c);
    c.pending += len;
}

struct Smem64 {
    uint32_t hist[kWarps][64];
    unsigned long long tot[kWarps][64];
};

__device__ __forceinline__ void block_setup64(Smem64 &S) {
    for (int i = threadIdx.x; i < kWarps * 64; i += blockDim.x) {
        (&S.hist[0][0])[i] = 0;
        (&S.tot[0][0])[i] = 0;
    }
    __syncthreads();
}

__device__ __forceinline__ void block_finish64(Smem64 &S, Acc64 &c, unsigned long long *d_counts) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    warp_flush64(S.hist[warp], S.tot[warp], c);
#pragma unroll
    for (int q = 0; q < 3; q++) {
        unsigned long long v = c.dy[q];
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) S.tot[warp][q + 1] += v;
    }
    __syncthreads();
    for (int k = threadIdx.x; k < 64; k += blockDim.x) {
        if (k == 0) continue;
        unsigned long long v = 0;
        for (int w = 0; w < kWarps; w++) v += S.tot[w][k];
        if (v) atomicAdd(&d_counts[k], v);
    }
}

__global__ void __launch_bounds__(kCensusThreads)
k_census_thread64(const BinItemT *__restrict__ items, const uint32_t *__restrict__ tile_count,
                  uint64_t ntiles, const uint32_t *__restrict__ adj, unsigned long long *d_counts,
                  unsigned long long *cursor, uint32_t upt) {
    __shared__ Smem64 S;
    block_setup64(S);
    Acc64 c{{0, 0, 0}, 0};
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ uint32_t unit_s;
    const uint32_t unit_dyads = kPlanTile / upt;
    for (uint64_t unit = next_unit(cursor, &unit_s); unit < ntiles * upt;
         unit = next_unit(cursor, &unit_s)) {
        const uint64_t tile = unit / upt;
        const uint32_t part = (uint32_t)(unit % upt) * unit_dyads;
        const uint32_t cnt = min(__ldg(tile_count + tile), part + unit_dyads);
        const BinItemT *it = items + tile * kPlanTile;
        for (uint32_t base = part + warp * 32; base < cnt; base += kCensusThreads) {
            const bool valid = base + lane < cnt;
            BinItemT e{0, 0, 0, 0};
            if (valid) {
                e = it[base + lane];
                e.t &= 0xffffu;
            }
            warp_reserve64(S.hist[warp], S.tot[warp], c, e.t);
            if (valid)
                merge_diag64(adj, e.pa, 0, e.pb, 0, e.e | 3u, e.e & 3u, 0, e.t, S.hist[warp], c);
        }
    }
    block_finish64(S, c, d_counts);
}

__global__ void __launch_bounds__(kCensusThreads)
k_census_warp64(const BinLists L, const uint32_t *__restrict__ off,
                const uint32_t *__restrict__ ups, const uint32_t *__restrict__ adj,
                unsigned long long *d_counts) {
    __shared__ Smem64 S;
    block_setup64(S);
    Acc64 c{{0, 0, 0}, 0};
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t count = *L.w_count;
    for (uint64_t it = next_item(L.wcursor); it < count; it = next_item(L.wcursor)) {
        const BinItemW e = L.w[it];
        const WarpDyad w = warp_dyad(L, off, ups, e.k);
        const uint32_t span = e.d1 - e.d0, per = (span + 31) >> 5;
        const uint32_t d0 = e.d0 + min(span, lane * per), d1 = e.d0 + min(span, (lane + 1) * per);
        warp_reserve64(S.hist[warp], S.tot[warp], c, d1 - d0);
        if (d0 < d1)
            merge_diag64(adj, w.oa, w.a, w.ob, w.b, w.e | 3u, w.e & 3u, d0, d1, S.hist[warp], c);
    }
    block_finish64(S, c, d_counts);
}

}  // namespace

tc_status launch_bins(const tc_graph *g, const BinLists &bl, cudaStream_t s, uint64_t *d_counts,
                      cudaEvent_t *ev, uint64_t *launches, int mode64) {
    unsigned long long *out = reinterpret_cast<unsigned long long *>(d_counts);
    // SM count and resident blocks per SM of the four bin kernels, queried
    // once per device (host time between the plan and the bins is exposed)
    struct Occ {
        int sms, thread, warp, thread64, warp64;
        cudaStream_t side;   // the warp bin runs here, beside the thread bin
    };
    static Occ occ[64];
    static std::atomic<uint64_t> occ_done{0};
    const int dv = g->device & 63;
    if (!(occ_done.load() & (1ull << dv))) {
        Occ o{148, 0, 0, 0, 0, nullptr};
        TC_CUDA(cudaStreamCreateWithFlags(&o.side, cudaStreamNonBlocking));
        cudaDeviceGetAttribute(&o.sms, cudaDevAttrMultiProcessorCount, g->device);
        TC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o.warp64, k_census_warp64,
                                                              kCensusThreads, 0));
        TC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o.warp, k_census_warp,
                                                              kCensusThreads, 0));
        TC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o.thread64, k_census_thread64,
                                                              kCensusThreads, 0));
        TC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o.thread, k_census_thread,
                                                              kCensusThreads, 0));
        occ[dv] = o;
        occ_done.fetch_or(1ull << dv);
    }
    const int sms = occ[dv].sms;
    const int perw = mode64 ? occ[dv].warp64 : occ[dv].warp;
    const int per = mode64 ? occ[dv].thread64 : occ[dv].thread;
    // warp bin: one resident wave, items handed out by bl.wcursor
    const unsigned grid = (unsigned)sms * (unsigned)(perw > 0 ? perw : 1);
    // thread bin: one resident wave, units handed out by bl.cursor
    uint64_t tgrid = (uint64_t)sms * (per > 0 ? per : 1);
    const uint32_t upt = bl.ntiles >= 4 * tgrid ? 2u : 4u;   // units per plan tile
    const uint64_t units = bl.ntiles * upt;
    if (tgrid > units) tgrid = units ? units : 1;
    // the two bins are independent (own item lists and cursors, atomic adds
    // into the census): the warp bin runs on a side stream, so it fills the
    // SMs the thread bin's tail leaves idle (and the reverse at C2/C4/C5).
    // ev (profiling): [0] start, [1] thread bin done, [2] both done (on s),
    // [3] warp bin done (on the side stream)
    const cudaStream_t side = occ[dv].side;
    cudaEvent_t fork = nullptr, join = nullptr;
    TC_CUDA(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
    if (ev) {
        fork = ev[0];
    } else {
        TC_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    }
    TC_CUDA(cudaEventRecord(fork, s));
    TC_CUDA(cudaStreamWaitEvent(side, fork, 0));
    if (mode64)
        k_census_thread64<<<(unsigned)tgrid, kCensusThreads, 0, s>>>(bl.t, bl.t_count, bl.ntiles,
                                                                    g->adj, out, bl.cursor, upt);
    else
        k_census_thread<<<(unsigned)tgrid, kCensusThreads, 0, s>>>(bl.t, bl.t_count, bl.ntiles,
                                                                  g->adj, out, bl.cursor, upt);
    TC_CUDA(cudaGetLastError());
    if (ev) TC_CUDA(cudaEventRecord(ev[1], s));
    if (mode64)
        k_census_warp64<<<grid, kCensusThreads, 0, side>>>(bl, g->off, g->ups, g->adj, out);
    else
        k_census_warp<<<grid, kCensusThreads, 0, side>>>(bl, g->off, g->ups, g->adj, out);
    TC_CUDA(cudaGetLastError());
    if (ev) TC_CUDA(cudaEventRecord(ev[3], side));
    TC_CUDA(cudaEventRecord(join, side));
    TC_CUDA(cudaStreamWaitEvent(s, join, 0));
    if (ev) TC_CUDA(cudaEventRecord(ev[2], s));
    cudaEventDestroy(join);
    if (!ev) cudaEventDestroy(fork);
    *launches += 2;
    return TC_OK;
}

}  // namespace tc
