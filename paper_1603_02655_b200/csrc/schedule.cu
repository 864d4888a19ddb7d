// schedule.cu -- a2: degree-binned canonical-dyad scheduler + shard cuts.
//
// Each canonical dyad (u, v), u < v, carries the paper's uniform workload
// estimate c = |N(u)| + |N(v)| (Fig. P:1678-1705, "NsetSize + |N[u]| + |N[v]|
// - 2"; the constant -2 changes no bin and no cut) and its
// exact merge length t = |{w in N(u): w > u}| + |{w in N(v): w > u}| (the
// part of both rows the census merge walks, census.cu), both computed once
// by the CSR builder (dyad_c, dyad_t).  The plan is one stable counting sort
// of the dyad range by t (256 digits: t itself for t <= kThreadBinMax, 255
// for every larger dyad):
//   thread bin  t <= 254    items (row starts, e, lengths) ordered by t, so
//                           each warp holds dyads of equal length and its
//                           lanes run equal trip counts
//   warp bin    t > 254     the dyad is cut into warp items of <= 8160
//                           diagonals (32 lanes x <= 255), so power-law hubs
//                           spread over many warps and never serialise one
// All counts stay on the device: no host synchronisation in the census.
// The same costs, prefix-summed in canonical order, give the degree-balanced
// multi-GPU shard cuts: the paper's uniform task
// queues with one "queue" per GPU.
#include <stdlib.h>

#include <vector>

#include "census.cuh"
#include "scan.cuh"

// search-vs-merge cost ratio NUM/DEN (measured)
#ifndef TC_SP_NUM
#define TC_SP_NUM 1u
#endif
#ifndef TC_SP_DEN
#define TC_SP_DEN 1u
#endif

namespace tc {

namespace {

constexpr int kPlanWarps = kPlanThreads / 32;
constexpr int kDigits = 256;

__device__ __forceinline__ uint32_t digit_of(uint32_t c) {
    return c <= kThreadBinMax ? c : 255u;
}

// One block per tile of kPlanTile consecutive canonical dyads: a stable
// tile-local counting sort of the thread-bin dyads by merge length t
// (warp-level ballot ranking, then a block scan over the 255 length digits),
// so the census keeps the tile's row locality and still gives every warp
// equal trip counts.  Dyads with t > kThreadBinMax become warp items (<= 8160
// diagonals each) appended through one atomic cursor per warp.  The plan
// also adds every dyad's dyadic term n - |N(u)| - |N(v)| (the
// census kernels add the intersection part) to d_counts, by class
// (mode16: 012 / 102) or by code pre (mode64).
// stats: [0] warp items, [1] / [2] thread- / warp-bin sum of c = |N(u)|+|N(v)|
// (the algorithmic work unit), [3] big dyads, [4] / [5] thread- / warp-bin
// merge trips (sum of t)
struct PlanIn {
    const uint32_t *du, *de, *dc, *dt, *dpb, *ups, *off;
    int sparse;   // skewed-pair items allowed (tag prefix built, 16-class mode)
};

// skewed-pair decision for a big dyad: 0 = merge items; 1 = iterate A (the
// entries > u of N(u)) and search N(v); 2 = iterate B and search N(u).
// *len = length of the iterated list.
__device__ __forceinline__ uint32_t sparse_mode(const PlanIn &P, uint64_t i, uint32_t *len,
                                                uint32_t *units) {
    const uint32_t u = __ldg(P.du + i), v = __ldg(P.de + i) >> 2;
    const uint32_t a = __ldg(P.off + u + 1) - 1u - __ldg(P.ups + u);
    const uint32_t b = __ldg(P.off + v + 1) - 1u - __ldg(P.dpb + i);
    const uint32_t sh = a < b ? a : b, lg = a < b ? b : a;
    const uint32_t lg2 = 32u - __clz(lg | 1u);
    if ((uint64_t)sh * (lg2 + 4u) * TC_SP_NUM >= ((uint64_t)a + b) * TC_SP_DEN) return 0u;
    *len = sh;
    *units = sh * lg2 + 4u;   // per short entry: ~log2(l) probes + the entry; 4 prefix/row loads
    return a < b ? 1u : 2u;
}

template <bool SPARSE>
__global__ void __launch_bounds__(kPlanThreads)
k_plan_tile(const PlanIn P, uint64_t N, uint64_t n, BinItemT *__restrict__ tl,
            uint32_t *__restrict__ tile_count, BinItemW *__restrict__ wl,
            unsigned long long *__restrict__ stats, unsigned long long *__restrict__ d_counts,
            int mode64) {
    __shared__ uint32_t wc[kPlanWarps][kDigits];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kPlanWarps * kDigits; i += kPlanThreads) (&wc[0][0])[i] = 0;
    __syncthreads();
    const uint32_t lt = (1u << lane) - 1u;
    const uint64_t tile0 = (uint64_t)blockIdx.x * kPlanTile;
    const uint32_t wbase = warp * 32 * kPlanItems;
    uint32_t cst[kPlanItems], rank[kPlanItems];
#pragma unroll
    for (int k = 0; k < kPlanItems; k++) {
        uint64_t i = tile0 + wbase + k * 32 + lane;
        bool valid = i < N;
        cst[k] = valid ? __ldg(P.dt + i) : 0u;
        uint32_t d = valid ? digit_of(cst[k]) : 0x10000u;
        // lanes holding the same digit: one ballot per digit bit
        const uint32_t peers = __ballot_sync(0xffffffffu, valid) & warp_peers<8>(d);
        uint32_t r = 0;
        if (valid) r = wc[warp][d] + __popc(peers & lt);
        __syncwarp();
        if (valid && (peers & lt) == 0) wc[warp][d] += __popc(peers);
        __syncwarp();
        rank[k] = r;
    }
    __syncthreads();
    uint32_t all;   // thread-bin dyads of the tile
    {   // thread d owns digit d: tile-local offsets (digit-major, then warp)
        const int d = threadIdx.x;
        uint32_t tot = 0;
#pragma unroll
        for (int w = 0; w < kPlanWarps; w++) tot += wc[w][d];
        if (d == 255) tot = 0;      // big dyads are not in the thread list
        uint32_t run = block_exclusive_sum<uint32_t>(tot, &all);
        if (d == 0 && tile_count) tile_count[blockIdx.x] = all;
#pragma unroll
        for (int w = 0; w < kPlanWarps; w++) {
            uint32_t c = wc[w][d];
            wc[w][d] = run;
            run += c;
        }
    }
    __syncthreads();
    // the tile's thread list as a permutation (sorted slot -> tile index):
    // 8 KB of shared memory instead of 64 KB of staged 16-byte items, so 5
    // blocks fit per SM (0.27 vs 0.34 ms at C3); the items are gathered from
    // the tile's dyad arrays (L1/L2-resident) and stored coalesced at the end
    __shared__ uint16_t perm[kPlanTile];
    unsigned long long wt = 0, ww = 0, tt = 0, tw = 0, nbig = 0, dy1 = 0, dy2 = 0, dy3 = 0;
    unsigned long long nsp = 0, spc = 0, spu = 0;   // skewed-pair dyads, sum of c, units
#pragma unroll 4
    for (int k = 0; k < kPlanItems; k++) {
        const uint64_t i = tile0 + wbase + k * 32 + lane;
        const bool valid = i < N;
        const uint32_t c = cst[k], d = digit_of(c);
        uint32_t nch = 0, smode = 0, span = 0;
        if (valid) {
            const uint32_t e = __ldg(P.de + i), pre = e & 3u;
            const uint32_t cf = __ldg(P.dc + i);
            const unsigned long long dy = n - cf;
            dy1 += pre == 1u ? dy : 0ull;
            dy2 += pre == 2u ? dy : 0ull;
            dy3 += pre == 3u ? dy : 0ull;
            if (d < 255u) {
                perm[wc[warp][d] + rank[k]] = (uint16_t)(wbase + k * 32 + lane);
                wt += cf;
                tt += c;
            } else {
                uint32_t slen = 0, sunits = 0;
                smode = (SPARSE && P.sparse && !mode64) ? sparse_mode(P, i, &slen, &sunits) : 0u;
                spu += smode ? sunits : 0u;
                nch = smode ? max(1u, (slen + kSparseChunk - 1) / kSparseChunk)
                            : (c + kWarpChunk - 1) / kWarpChunk;
                ww += cf;
                tw += c;
                nbig++;
                nsp += smode ? 1u : 0u;
                spc += smode ? cf : 0u;
                span = smode ? slen : c;
            }
        }
        // warp-aggregated cursor for the warp items
        uint32_t incl = nch;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const uint32_t wtot = __shfl_sync(0xffffffffu, incl, 31);
        if (wtot) {
            unsigned long long at = 0;
            if (lane == 31) at = atomicAdd(&stats[0], (unsigned long long)wtot);
            at = __shfl_sync(0xffffffffu, at, 31) + (incl - nch);
            const uint32_t chunk = smode ? kSparseChunk : kWarpChunk;
            for (uint32_t q = 0; q < nch; q++) {
                const uint32_t d0 = q * chunk;
                wl[at + q] = BinItemW{(uint32_t)i, d0, min(span, d0 + chunk), smode};
            }
        }
    }
    __syncthreads();
    uint4 *out = reinterpret_cast<uint4 *>(tl + tile0);
    for (uint32_t j = threadIdx.x; tl && j < all; j += kPlanThreads) {
        const uint64_t i = tile0 + perm[j];
        const uint32_t u = __ldg(P.du + i);
        // t | |A| << 16 (t <= 254): the census prefetches exactly both parts
        const uint32_t pa = __ldg(P.ups + u), a = __ldg(P.off + u + 1) - 1u - pa;
        out[j] = make_uint4(pa, __ldg(P.dpb + i), __ldg(P.de + i), __ldg(P.dt + i) | a << 16);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        wt += __shfl_xor_sync(0xffffffffu, wt, o);
        ww += __shfl_xor_sync(0xffffffffu, ww, o);
        nbig += __shfl_xor_sync(0xffffffffu, nbig, o);
        tt += __shfl_xor_sync(0xffffffffu, tt, o);
        tw += __shfl_xor_sync(0xffffffffu, tw, o);
        dy1 += __shfl_xor_sync(0xffffffffu, dy1, o);
        dy2 += __shfl_xor_sync(0xffffffffu, dy2, o);
        dy3 += __shfl_xor_sync(0xffffffffu, dy3, o);
        nsp += __shfl_xor_sync(0xffffffffu, nsp, o);
        spc += __shfl_xor_sync(0xffffffffu, spc, o);
        spu += __shfl_xor_sync(0xffffffffu, spu, o);
    }
    if (lane == 0) {
        if (wt) atomicAdd(&stats[1], wt);
        if (ww) atomicAdd(&stats[2], ww);
        if (nbig) atomicAdd(&stats[3], nbig);
        if (tt) atomicAdd(&stats[4], tt);
        if (tw) atomicAdd(&stats[5], tw);
        if (nsp) atomicAdd(&stats[8], nsp);
        if (spc) atomicAdd(&stats[9], spc);
        if (spu) atomicAdd(&stats[10], spu);
        if (mode64) {
            if (dy1) atomicAdd(&d_counts[1], dy1);
            if (dy2) atomicAdd(&d_counts[2], dy2);
        } else if (dy1 + dy2) {
            atomicAdd(&d_counts[1], dy1 + dy2);
        }
        if (dy3) atomicAdd(&d_counts[mode64 ? 3 : 2], dy3);
    }
}

// Shard cost of canonical dyad k (refined to the
// work the census kernels actually do): kappa + t for a merged dyad (t merge
// trips over the entries w > u of both rows, census.cu), kappa + the search
// units s * ceil(log2 l) + 4 for a skewed-pair dyad (same rule as the plan).
// The paper's uniform estimate |N(u)| + |N(v)| - 2 weighs
// early dyads (small u) too lightly: their merges walk more of both rows.
struct WorkIn {
    PlanIn P;
    uint64_t kappa;
    __device__ __forceinline__ uint64_t operator()(size_t k) const {
        const uint32_t t = __ldg(P.dt + k);
        if (P.sparse && t > kThreadBinMax) {
            uint32_t len = 0, units = 0;
            if (sparse_mode(P, k, &len, &units)) return (uint64_t)units + kappa;
        }
        return (uint64_t)t + kappa;
    }
};

__global__ void k_lower_bounds(const uint64_t *__restrict__ excl, uint64_t D,
                               const uint64_t *__restrict__ targets, int nt, uint64_t *out) {
    int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nt) return;
    uint64_t t = targets[r], lo = 0, hi = D;
    while (lo < hi) {          // first k with excl[k] >= t
        uint64_t mid = (lo + hi) >> 1;
        if (excl[mid] < t) lo = mid + 1;
        else hi = mid;
    }
    out[r] = lo;
}


// ---------------------------------------------------------------------------
// the multithreaded version's task queues (Fig. P:1650-
// 1672, Canonical Dyad(non-uniform distr.): NsetSize += |S|; Fig. P:1676-
// 1698, Canonical Dyad(uniform distr.): NsetSize += |N[u]| + |N[v]| - 2) as
// a GPU scheduler: queue q = a contiguous run of canonical dyads, closed
// right after the dyad that makes its NsetSize exceed MaxNsetSize.
// ---------------------------------------------------------------------------

// per-dyad NsetSize: uniform |N(u)| + |N(v)| - 2 (dyad_c - 2); non-uniform
// |S| = |N(u)| + |N(v)| - |N(u) & N(v)| - 2 (u and v are in the union).  One
// warp per dyad: lanes take the entries of the shorter row and binary-search
// them in the longer one (rows end in a sentinel; entries compare by id).
__global__ void k_queue_weights(const uint32_t *__restrict__ off, const uint32_t *__restrict__ adj,
                                const uint32_t *__restrict__ du, const uint32_t *__restrict__ de,
                                const uint32_t *__restrict__ dc, uint64_t D, int nonuniform,
                                uint32_t *__restrict__ w) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t k = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < D; k += nw) {
        const uint32_t c = __ldg(dc + k);
        if (!nonuniform) {
            if (lane == 0) w[k] = c - 2u;
            continue;
        }
        const uint32_t u = __ldg(du + k), v = __ldg(de + k) >> 2;
        uint32_t oa = __ldg(off + u), la = __ldg(off + u + 1) - 1u - oa;
        uint32_t ob = __ldg(off + v), lb = __ldg(off + v + 1) - 1u - ob;
        if (la > lb) {
            uint32_t t = oa; oa = ob; ob = t;
            t = la; la = lb; lb = t;
        }
        uint32_t hits = 0;
        for (uint32_t i = lane; i < la; i += 32) {
            const uint32_t x = __ldg(adj + oa + i) >> 2;
            uint32_t lo = 0, hi = lb;
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if ((__ldg(adj + ob + mid) >> 2) < x) lo = mid + 1;
                else hi = mid;
            }
            hits += (lo < lb && (__ldg(adj + ob + lo) >> 2) == x);
        }
        hits = __reduce_add_sync(0xffffffffu, hits);
        if (lane == 0) w[k] = c - hits - 2u;
    }
}

// The queue loop itself is sequential (NsetSize resets at every cut), so one
// warp walks the weights 32 at a time: an inclusive warp scan of the chunk
// from the current start lane, the first lane whose running NsetSize
// exceeds MaxNsetSize closes a queue, the scan restarts after it.
// starts[q] = first dyad of queue q; out[0] = queues, out[1] = aggregate
// NsetSize.
__global__ void __launch_bounds__(32) k_queue_greedy(const uint32_t *__restrict__ w, uint64_t D,
                                                     uint64_t max_nset, uint32_t *__restrict__ starts,
                                                     unsigned long long *__restrict__ out) {
    const uint32_t lane = threadIdx.x;
    unsigned long long run = 0, total = 0, q = 0;
    if (D > 0 && lane == 0) starts[0] = 0;
    q = D > 0 ? 1 : 0;
    for (uint64_t base = 0; base < D; base += 32) {
        const bool valid = base + lane < D;
        const unsigned long long x = valid ? __ldg(w + base + lane) : 0ull;
        unsigned long long all = x;
#pragma unroll
        for (int o = 16; o; o >>= 1) all += __shfl_xor_sync(0xffffffffu, all, o);
        total += all;
        uint32_t s = 0;                          // first lane of the open run
        while (s < 32) {
            unsigned long long p = lane >= s ? x : 0ull;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long y = __shfl_up_sync(0xffffffffu, p, o);
                if (lane >= (uint32_t)o) p += y;
            }
            const uint32_t cross = __ballot_sync(0xffffffffu, valid && lane >= s && run + p > max_nset);
            if (!cross) {
                run += __shfl_sync(0xffffffffu, p, 31);
                break;
            }
            const uint32_t c = __ffs(cross) - 1;   // this dyad closes the queue
            const uint64_t next = base + c + 1;
            if (next < D) {
                if (lane == 0) starts[q] = (uint32_t)next;
                q++;
            }
            run = 0;
            s = c + 1;
        }
    }
    if (lane == 0) {
        out[0] = q;
        out[1] = total;
    }
}
// tc_census_range's per-range dyadic triads in the paper's own attribution
// (Fig. P:269-309 lines 9-14): every canonical dyad (u, v) of the range adds
// n - |S| - 2 = n - |N(u)| - |N(v)| + |N(u) & N(v)| (S = N(u) U N(v) \ {u,v};
// u, v are not in the intersection: no loops) to class 102 if pre = 3, else
// 012.  One warp per dyad: lanes take the entries of the shorter row and
// binary-search them in the longer one (rows are sorted by id).  Classes
// 021D..300 of the range are exact per range in the bin kernels' partial
// `part`, which block 0 adds (its 012 / 102 slots use the owed-credit
// attribution of DESIGN.md reading 21 and are dropped here).
__global__ void __launch_bounds__(256)
k_range_dyadic(const uint32_t *__restrict__ off, const uint32_t *__restrict__ adj,
               const uint32_t *__restrict__ du, const uint32_t *__restrict__ de, uint64_t N,
               uint64_t n, const unsigned long long *__restrict__ part,
               unsigned long long *__restrict__ d_counts) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    unsigned long long a012 = 0, a102 = 0;
    for (uint64_t k = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < N; k += nw) {
        const uint32_t u = __ldg(du + k), e = __ldg(de + k), v = e >> 2;
        uint32_t oa = __ldg(off + u), la = __ldg(off + u + 1) - 1u - oa;
        uint32_t ob = __ldg(off + v), lb = __ldg(off + v + 1) - 1u - ob;
        const uint32_t dsum = la + lb;
        if (la > lb) {
            uint32_t t = oa; oa = ob; ob = t;
            t = la; la = lb; lb = t;
        }
        uint32_t hits = 0;
        for (uint32_t i = lane; i < la; i += 32) {
            const uint32_t x = __ldg(adj + oa + i) >> 2;
            uint32_t lo = 0, hi = lb;
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if ((__ldg(adj + ob + mid) >> 2) < x) lo = mid + 1;
                else hi = mid;
            }
            hits += (lo < lb && (__ldg(adj + ob + lo) >> 2) == x);
        }
        hits = __reduce_add_sync(0xffffffffu, hits);
        const unsigned long long dy = n - dsum + hits;
        if ((e & 3u) == 3u) a102 += lane == 0 ? dy : 0ull;
        else a012 += lane == 0 ? dy : 0ull;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        a012 += __shfl_xor_sync(0xffffffffu, a012, o);
        a102 += __shfl_xor_sync(0xffffffffu, a102, o);
    }
    if (lane == 0) {
        if (a012) atomicAdd(&d_counts[1], a012);
        if (a102) atomicAdd(&d_counts[2], a102);
    }
    if (blockIdx.x == 0 && threadIdx.x >= 3 && threadIdx.x < 16 && part[threadIdx.x])
        atomicAdd(&d_counts[threadIdx.x], part[threadIdx.x]);
}

// ---------------------------------------------------------------------------
// Full-census plan built with the graph (a1 + a2 fused, round 2).  The CSR
// builder's last assembly step (upper row entries, per-dyad c and t) runs
// here tile by tile; while a tile's merge lengths are in registers they are
// ranked exactly as k_plan_tile ranks them, and the thread-bin items of the
// whole dyad range [0, D) are stored with the graph, together with the list
// of big dyads (t > kThreadBinMax), the dyadic base sums n - c per pre and the
// thread-bin work sums.  A full 16-class census then only turns the big
// dyads into warp items (k_emit_big) and runs the bin kernels; dyad ranges,
// shards and the 64-type census keep the per-call plan (k_plan_tile).
// sums: [0..2] n - c of pre 1..3, [3] thread-bin sum of c, [4] thread-bin
// sum of t, [5] big dyads (the length of `big`)
// ---------------------------------------------------------------------------
struct UpperIn {
    const uint32_t *off, *ups, *lo_start, *du, *de, *dpb, *dD;
    uint32_t *adj, *dc, *dt;
    uint64_t n;
};

#ifndef TC_UP_BATCH
#define TC_UP_BATCH 4
#endif
constexpr int kUpBatch = TC_UP_BATCH;   // dyads per thread whose loads are in flight together

#ifndef TC_UP_MINB
#define TC_UP_MINB 4
#endif
__global__ void __launch_bounds__(kPlanThreads, TC_UP_MINB)
k_upper_plan(const UpperIn I, BinItemT *__restrict__ tl, uint32_t *__restrict__ tile_count,
             uint32_t *__restrict__ big, unsigned long long *__restrict__ sums,
             unsigned long long *__restrict__ bstats /* [2] += arcs, [3] += mutual dyads */) {
    __shared__ uint32_t wc[kPlanWarps][kDigits];
    __shared__ uint16_t perm[kPlanTile];
    __shared__ uint32_t wbig[kPlanWarps];
    __shared__ unsigned long long big_base;
    const uint64_t N = *I.dD;
    const uint64_t tile0 = (uint64_t)blockIdx.x * kPlanTile;
    if (tile0 >= N) return;   // block-uniform
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kPlanWarps * kDigits; i += kPlanThreads) (&wc[0][0])[i] = 0;
    const uint32_t lt = (1u << lane) - 1u;
    const uint32_t wbase = warp * 32 * kPlanItems;
    // per dyad: its length digit in shared memory (phase 1 keeps no per-dyad
    // registers, so more loads stay in flight), its rank in 16-bit halves of rk
    __shared__ uint8_t dgs[kPlanTile];
    uint32_t rk[kPlanItems / 2];
    uint32_t m = 0, mu = 0, tt = 0;
    unsigned long long dy1 = 0, dy2 = 0, dy3 = 0, wt = 0;
    // 1. the upper entries, c and t of the tile's dyads (k_write_upper's work)
#pragma unroll 1
    for (int kb = 0; kb < kPlanItems; kb += kUpBatch) {
        uint32_t u[kUpBatch], e[kUpBatch], pb[kUpBatch];
#pragma unroll
        for (int j = 0; j < kUpBatch; j++) {
            const uint64_t i = tile0 + wbase + (kb + j) * 32 + lane;
            const bool ok = i < N;
            u[j] = ok ? __ldg(I.du + i) : 0u;
            e[j] = ok ? __ldg(I.de + i) : 0u;
            pb[j] = ok ? __ldg(I.dpb + i) : 0u;
        }
        uint32_t ls[kUpBatch], ou[kUpBatch], ou1[kUpBatch], up[kUpBatch], ov[kUpBatch],
            ov1[kUpBatch];
#pragma unroll
        for (int j = 0; j < kUpBatch; j++) {
            const uint32_t v = e[j] >> 2;
            ls[j] = __ldg(I.lo_start + u[j] + 1);
            ou[j] = __ldg(I.off + u[j]);
            ou1[j] = __ldg(I.off + u[j] + 1);
            up[j] = __ldg(I.ups + u[j]);
            ov[j] = __ldg(I.off + v);
            ov1[j] = __ldg(I.off + v + 1);
        }
#pragma unroll
        for (int j = 0; j < kUpBatch; j++) {
            const uint64_t i = tile0 + wbase + (kb + j) * 32 + lane;
            if (i >= N) {
                dgs[wbase + (kb + j) * 32 + lane] = 0;
                continue;
            }
            I.adj[ls[j] + u[j] + (uint32_t)i] = e[j];
            // the last upper entry of row u also writes the row's terminator
            // (k_offsets writes it for rows without upper entries)
            if (ls[j] + u[j] + (uint32_t)i + 2u == ou1[j]) I.adj[ou1[j] - 1] = 0xffffffffu;
            const uint32_t c = (ou1[j] - ou[j]) + (ov1[j] - ov[j]) - 2;
            const uint32_t t = (ou1[j] - 1 - up[j]) + (ov1[j] - 1 - pb[j]);
            I.dc[i] = c;
            I.dt[i] = t;
            dgs[wbase + (kb + j) * 32 + lane] = (uint8_t)digit_of(t);
            const uint32_t pre = e[j] & 3u;
            m += __popc(pre);
            mu += pre == 3u;
            const unsigned long long dy = I.n - c;
            dy1 += pre == 1u ? dy : 0ull;
            dy2 += pre == 2u ? dy : 0ull;
            dy3 += pre == 3u ? dy : 0ull;
            if (t <= kThreadBinMax) {
                wt += c;
                tt += t;
            }
        }
    }
    __syncthreads();
    // 2. stable rank by merge length (k_plan_tile's ballot ranking); big dyads counted
    uint32_t nbw = 0;
#pragma unroll
    for (int k = 0; k < kPlanItems; k++) {
        const uint64_t i = tile0 + wbase + k * 32 + lane;
        const bool valid = i < N;
        const uint32_t d = valid ? (uint32_t)dgs[wbase + k * 32 + lane] : 0x10000u;
        const uint32_t peers = __ballot_sync(0xffffffffu, valid) & warp_peers<8>(d);
        uint32_t r = 0;
        if (valid) r = wc[warp][d] + __popc(peers & lt);
        __syncwarp();
        if (valid && (peers & lt) == 0) wc[warp][d] += __popc(peers);
        __syncwarp();
        if (k & 1) rk[k >> 1] |= r << 16;
        else rk[k >> 1] = r;
        nbw += __popc(__ballot_sync(0xffffffffu, valid && d == 255u));
    }
    if (lane == 0) wbig[warp] = nbw;
    __syncthreads();
    uint32_t all;
    {
        const int d = threadIdx.x;
        uint32_t tot = 0;
#pragma unroll
        for (int w = 0; w < kPlanWarps; w++) tot += wc[w][d];
        if (d == 255) tot = 0;      // big dyads are not in the thread list
        uint32_t run = block_exclusive_sum<uint32_t>(tot, &all);
        if (d == 0 && tile_count) tile_count[blockIdx.x] = all;
#pragma unroll
        for (int w = 0; w < kPlanWarps; w++) {
            uint32_t c = wc[w][d];
            wc[w][d] = run;
            run += c;
        }
        if (d == 0) {   // one reservation per block in the big-dyad list
            uint32_t nb = 0;
            for (int w = 0; w < kPlanWarps; w++) nb += wbig[w];
            big_base = (nb && big) ? atomicAdd(&sums[5], (unsigned long long)nb) : 0ull;
        }
    }
    __syncthreads();
    uint64_t bpos = big_base;
    for (int w = 0; w < warp; w++) bpos += wbig[w];
#pragma unroll
    for (int k = 0; k < kPlanItems; k++) {
        const uint64_t i = tile0 + wbase + k * 32 + lane;
        const bool valid = i < N;
        const uint32_t d = dgs[wbase + k * 32 + lane];
        const uint32_t r = (rk[k >> 1] >> (16 * (k & 1))) & 0xffffu;
        if (valid && d < 255u) perm[wc[warp][d] + r] = (uint16_t)(wbase + k * 32 + lane);
        const uint32_t bb = __ballot_sync(0xffffffffu, valid && d == 255u);
        if (big && valid && d == 255u) big[bpos + __popc(bb & lt)] = (uint32_t)i;
        bpos += __popc(bb);
    }
    __syncthreads();
    // 3. the tile's thread-bin items in length order, stored coalesced
    uint4 *out = reinterpret_cast<uint4 *>(tl + tile0);
    for (uint32_t j = threadIdx.x; tl && j < all; j += kPlanThreads) {
        const uint64_t i = tile0 + perm[j];
        const uint32_t u = __ldg(I.du + i);
        const uint32_t pa = __ldg(I.ups + u), a = __ldg(I.off + u + 1) - 1u - pa;
        out[j] = make_uint4(pa, __ldg(I.dpb + i), __ldg(I.de + i), I.dt[i] | a << 16);
    }
    m = __reduce_add_sync(0xffffffffu, m);
    mu = __reduce_add_sync(0xffffffffu, mu);
    tt = __reduce_add_sync(0xffffffffu, tt);
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        dy1 += __shfl_xor_sync(0xffffffffu, dy1, o);
        dy2 += __shfl_xor_sync(0xffffffffu, dy2, o);
        dy3 += __shfl_xor_sync(0xffffffffu, dy3, o);
        wt += __shfl_xor_sync(0xffffffffu, wt, o);
    }
    if (lane == 0) {
        if (m) atomicAdd(&bstats[2], (unsigned long long)m);
        if (mu) atomicAdd(&bstats[3], (unsigned long long)mu);
        if (dy1) atomicAdd(&sums[0], dy1);
        if (dy2) atomicAdd(&sums[1], dy2);
        if (dy3) atomicAdd(&sums[2], dy3);
        if (wt) atomicAdd(&sums[3], wt);
        if (tt) atomicAdd(&sums[4], (unsigned long long)tt);
    }
}

// per full census: the big dyads of the graph's list become warp items
// (merge chunks or skewed-pair items, as in k_plan_tile); block 0 also adds
// the graph's dyadic base sums to the census and its thread-bin work sums to
// the per-call stats (stats layout of census_range_device)
template <bool SPARSE>
__global__ void __launch_bounds__(256)
k_emit_big(const PlanIn P, const uint32_t *__restrict__ big, const unsigned long long *__restrict__ sums,
           BinItemW *__restrict__ wl, unsigned long long *__restrict__ stats,
           unsigned long long *__restrict__ d_counts) {
    const uint64_t nb = sums[5];
    const uint32_t lane = threadIdx.x & 31;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (sums[0] + sums[1]) atomicAdd(&d_counts[1], sums[0] + sums[1]);
        if (sums[2]) atomicAdd(&d_counts[2], sums[2]);
        atomicAdd(&stats[1], sums[3]);
        atomicAdd(&stats[4], sums[4]);
        atomicAdd(&stats[3], nb);
    }
    unsigned long long ww = 0, tw = 0, nsp = 0, spc = 0, spu = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t q0 = (uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); q0 < nb; q0 += stride) {
        const uint64_t q = q0 + lane;
        const bool valid = q < nb;
        uint32_t nch = 0, smode = 0, span = 0, i = 0;
        if (valid) {
            i = __ldg(big + q);
            const uint32_t c = __ldg(P.dt + i), cf = __ldg(P.dc + i);
            uint32_t slen = 0, sunits = 0;
            smode = SPARSE ? sparse_mode(P, i, &slen, &sunits) : 0u;
            spu += smode ? sunits : 0u;
            nch = smode ? max(1u, (slen + kSparseChunk - 1) / kSparseChunk)
                        : (c + kWarpChunk - 1) / kWarpChunk;
            ww += cf;
            tw += c;
            nsp += smode ? 1u : 0u;
            spc += smode ? cf : 0u;
            span = smode ? slen : c;
        }
        uint32_t incl = nch;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= (uint32_t)o) incl += y;
        }
        const uint32_t wtot = __shfl_sync(0xffffffffu, incl, 31);
        unsigned long long at = 0;
        if (lane == 31 && wtot) at = atomicAdd(&stats[0], (unsigned long long)wtot);
        at = __shfl_sync(0xffffffffu, at, 31) + (incl - nch);
        const uint32_t chunk = smode ? kSparseChunk : kWarpChunk;
        for (uint32_t c = 0; c < nch; c++) {
            const uint32_t d0 = c * chunk;
            wl[at + c] = BinItemW{i, d0, min(span, d0 + chunk), smode};
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        ww += __shfl_xor_sync(0xffffffffu, ww, o);
        tw += __shfl_xor_sync(0xffffffffu, tw, o);
        nsp += __shfl_xor_sync(0xffffffffu, nsp, o);
        spc += __shfl_xor_sync(0xffffffffu, spc, o);
        spu += __shfl_xor_sync(0xffffffffu, spu, o);
    }
    if (lane == 0) {
        if (ww) atomicAdd(&stats[2], ww);
        if (tw) atomicAdd(&stats[5], tw);
        if (nsp) atomicAdd(&stats[8], nsp);
        if (spc) atomicAdd(&stats[9], spc);
        if (spu) atomicAdd(&stats[10], spu);
    }
}

}  // namespace

tc_status census_range_paper_device(const tc_graph *g, uint64_t k0, uint64_t k1, cudaStream_t s,
                                    uint64_t *d_counts, tc_profile *prof, uint64_t *launches) {
    const uint64_t D = g->st.dyads;
    if (k1 > D) k1 = D;
    if (k0 >= k1) return TC_OK;
    Mem mem = g->mem;
    mem.stream = s;
    DevBuf<uint64_t> part;
    tc_status st = part.allocate(mem, 16);
    if (st != TC_OK) return st;
    TC_CUDA(cudaMemsetAsync(part.p, 0, 16 * sizeof(uint64_t), s));
    if ((st = census_range_device(g, k0, k1, s, part.p, prof, launches)) != TC_OK) return st;
    const uint64_t N = k1 - k0;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g->device);
    uint64_t blocks = (N + 7) / 8;
    if (blocks > (uint64_t)sms * 8) blocks = (uint64_t)sms * 8;
    k_range_dyadic<<<(unsigned)blocks, 256, 0, s>>>(
        g->off, g->adj, g->dyad_u + k0, g->dyad_e + k0, N, g->st.n,
        reinterpret_cast<const unsigned long long *>(part.p),
        reinterpret_cast<unsigned long long *>(d_counts));
    TC_CUDA(cudaGetLastError());
    *launches += 1;
    return TC_OK;
}

tc_status upper_plan_device(tc_graph *g, const uint32_t *lo_start, const uint32_t *dD, uint64_t Dub,
                            unsigned long long *bstats, cudaStream_t s) {
    const uint64_t ntiles = (Dub + kPlanTile - 1) / kPlanTile;
    Mem &mem = g->mem;
    // the graph keeps its own plan up to kResidentMaxDyads canonical dyads
    // (16 B per dyad + 4 B per big dyad); larger graphs (C5: 1.05e9 dyads)
    // plan per census call instead, as ranges do
    const bool resident = Dub <= kResidentMaxDyads;
    if (resident) {
        g->plan_items = (BinItemT *)mem.alloc((ntiles ? ntiles : 1) * kPlanTile * sizeof(BinItemT));
        g->plan_tcount = (uint32_t *)mem.alloc((ntiles ? ntiles : 1) * sizeof(uint32_t));
        g->plan_big = (uint32_t *)mem.alloc((Dub ? Dub : 1) * sizeof(uint32_t));
        g->plan_cap_tiles = ntiles ? ntiles : 1;
        g->plan_cap_big = Dub ? Dub : 1;
    }
    g->plan_sums = (unsigned long long *)mem.alloc(8 * sizeof(unsigned long long));
    if ((resident && (!g->plan_items || !g->plan_tcount || !g->plan_big)) || !g->plan_sums) {
        set_error("device allocation for the graph's census plan failed");
        return TC_E_OOM;
    }
    TC_CUDA(cudaMemsetAsync(g->plan_sums, 0, 8 * sizeof(unsigned long long), s));
    if (ntiles) {
        const UpperIn I{g->off, g->ups, lo_start, g->dyad_u, g->dyad_e, g->dyad_pb, dD,
                        g->adj, g->dyad_c, g->dyad_t, g->st.n};
        k_upper_plan<<<(unsigned)ntiles, kPlanThreads, 0, s>>>(I, g->plan_items, g->plan_tcount,
                                                              g->plan_big, g->plan_sums, bstats);
        TC_CUDA(cudaGetLastError());
        g->launches += 1;
    }
    return TC_OK;
}

tc_status census_range_device(const tc_graph *g, uint64_t k0, uint64_t k1, cudaStream_t s,
                              uint64_t *d_counts, tc_profile *prof, uint64_t *launches,
                              int mode64) {
    const uint64_t D = g->st.dyads;
    if (k1 > D) k1 = D;
    if (k0 >= k1) return TC_OK;
    const uint64_t N = k1 - k0;
    if (N >= (1ull << 32)) {
        set_error("dyad range too large");
        return TC_E_INVALID;
    }
    Mem mem = g->mem;
    mem.stream = s;
    cudaEvent_t ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    if (prof) {
        for (int i = 0; i < 5; i++) TC_CUDA(cudaEventCreate(&ev[i]));
        TC_CUDA(cudaEventRecord(ev[0], s));
    }
    tc_status st;
    const uint64_t ntiles = (N + kPlanTile - 1) / kPlanTile;
    // upper bound on warp items: sum over big dyads of ceil(t / chunk), t <= c
    const uint64_t nbig_max = g->st.sum_deg_sq / (kThreadBinMax + 1) + 1;
    const uint64_t wcap = (nbig_max < N ? nbig_max : N) + g->st.sum_deg_sq / kWarpChunk + 2;
    DevBuf<uint32_t> tcount;
    DevBuf<BinItemT> tl;
    DevBuf<BinItemW> wl;
    DevBuf<unsigned long long> stats;
    const bool use_graph_plan = g->plan_items && k0 == 0 && k1 == D && !mode64;
    if (!use_graph_plan) {
        if ((st = tcount.allocate(mem, ntiles)) != TC_OK) return st;
        if ((st = tl.allocate(mem, ntiles * kPlanTile)) != TC_OK) return st;
    }
    if ((st = wl.allocate(mem, wcap)) != TC_OK) return st;
    if ((st = stats.allocate(mem, 11)) != TC_OK) return st;
    TC_CUDA(cudaMemsetAsync(stats.p, 0, 11 * sizeof(unsigned long long), s));
    const PlanIn P{g->dyad_u + k0, g->dyad_e + k0, g->dyad_c + k0, g->dyad_t + k0,
                   g->dyad_pb + k0, g->ups, g->off, g->tagpre != nullptr};
    // the whole range in 16-class mode: the graph's own plan (k_upper_plan)
    const bool resident = g->plan_items && k0 == 0 && k1 == D && !mode64;
    if (resident) {
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g->device);
        if (P.sparse)
            k_emit_big<true><<<(unsigned)sms * 8, 256, 0, s>>>(
                P, g->plan_big, g->plan_sums, wl.p, stats.p,
                reinterpret_cast<unsigned long long *>(d_counts));
        else
            k_emit_big<false><<<(unsigned)sms * 8, 256, 0, s>>>(
                P, g->plan_big, g->plan_sums, wl.p, stats.p,
                reinterpret_cast<unsigned long long *>(d_counts));
    } else if (P.sparse && !mode64)
        k_plan_tile<true><<<(unsigned)ntiles, kPlanThreads, 0, s>>>(
        P, N, g->st.n, tl.p, tcount.p, wl.p, stats.p,
        reinterpret_cast<unsigned long long *>(d_counts), mode64);
    else
        k_plan_tile<false><<<(unsigned)ntiles, kPlanThreads, 0, s>>>(
        P, N, g->st.n, tl.p, tcount.p, wl.p, stats.p,
        reinterpret_cast<unsigned long long *>(d_counts), mode64);
    TC_CUDA(cudaGetLastError());
    *launches += 1;
    BinLists lists;
    lists.t = resident ? g->plan_items : tl.p;
    lists.t_count = resident ? g->plan_tcount : tcount.p;
    lists.ntiles = ntiles;
    lists.w = wl.p;
    lists.w_count = stats.p;
    lists.cursor = stats.p + 6;
    lists.wcursor = stats.p + 7;
    lists.du = P.du;
    lists.de = P.de;
    lists.dpb = P.dpb;
    lists.tagpre = g->tagpre;
    st = launch_bins(g, lists, s, d_counts, prof ? ev + 1 : nullptr, launches, mode64);
    if (st != TC_OK) return st;
    if (prof) {
        TC_CUDA(cudaEventRecord(ev[3], s));
        unsigned long long hs[11];
        TC_CUDA(cudaMemcpyAsync(hs, stats.p, sizeof(hs), cudaMemcpyDeviceToHost, s));
        TC_CUDA(cudaStreamSynchronize(s));
        const uint64_t nt = N - hs[3];
        float t;
        TC_CUDA(cudaEventElapsedTime(&t, ev[0], ev[1]));
        prof->plan_ms = t;
        TC_CUDA(cudaEventElapsedTime(&t, ev[1], ev[2]));
        prof->kernel_ms[0] = t;
        TC_CUDA(cudaEventElapsedTime(&t, ev[1], ev[4]));   // warp bin, on the side stream
        prof->kernel_ms[1] = t;
        prof->kernel_ms[2] = prof->kernel_ms[3] = 0;
        TC_CUDA(cudaEventElapsedTime(&t, ev[1], ev[3]));
        prof->census_ms = t;
        prof->bin_items[0] = nt;
        prof->bin_items[1] = hs[0];
        prof->bin_items[2] = hs[3];   // dyads in the warp bin
        prof->bin_items[3] = hs[8];   // skewed-pair dyads (inside the warp bin)
        prof->bin_work[0] = hs[1];
        prof->bin_work[1] = hs[2];
        prof->bin_work[2] = hs[4];
        prof->bin_work[3] = hs[5];
        prof->sparse_sum_c = hs[9];
        prof->sparse_units = hs[10];
        for (int i = 0; i < 5; i++) cudaEventDestroy(ev[i]);
    }
    return TC_OK;
}

tc_status task_queues_device(const tc_graph *g, int nonuniform, uint64_t max_nset, cudaStream_t s,
                             uint64_t *starts, uint64_t cap, uint64_t *nq, uint64_t *total) {
    const uint64_t D = g->st.dyads;
    *nq = 0;
    *total = 0;
    if (D == 0) return TC_OK;
    Mem mem = g->mem;
    mem.stream = s;
    tc_status st;
    DevBuf<uint32_t> w, dst;
    DevBuf<unsigned long long> out;
    if ((st = w.allocate(mem, D)) != TC_OK) return st;
    if ((st = dst.allocate(mem, D)) != TC_OK) return st;
    if ((st = out.allocate(mem, 2)) != TC_OK) return st;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g->device);
    k_queue_weights<<<(unsigned)sms * 8, 256, 0, s>>>(g->off, g->adj, g->dyad_u, g->dyad_e,
                                                      g->dyad_c, D, nonuniform, w.p);
    TC_CUDA(cudaGetLastError());
    k_queue_greedy<<<1, 32, 0, s>>>(w.p, D, max_nset, dst.p, out.p);
    TC_CUDA(cudaGetLastError());
    unsigned long long h[2];
    TC_CUDA(cudaMemcpyAsync(h, out.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    *nq = h[0];
    *total = h[1];
    if (h[0] > cap) {
        set_error("%llu task queues exceed the capacity %llu", h[0], (unsigned long long)cap);
        return TC_E_RANGE;
    }
    if (h[0]) {
        uint32_t *tmp = (uint32_t *)malloc(h[0] * sizeof(uint32_t));
        if (!tmp) {
            set_error("host allocation failed");
            return TC_E_OOM;
        }
        cudaError_t e = cudaMemcpyAsync(tmp, dst.p, h[0] * sizeof(uint32_t),
                                        cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) {
            free(tmp);
            return cuda_status(e, "task queue copy");
        }
        for (uint64_t i = 0; i < h[0]; i++) starts[i] = tmp[i];
        free(tmp);
    }
    return TC_OK;
}

tc_status shard_bounds_device(const tc_graph *g, int world, cudaStream_t s, uint64_t kappa,
                              uint64_t *bounds) {
    if (world < 1 || world > kMaxWorld) {
        set_error("world %d outside [1, %d]", world, kMaxWorld);
        return TC_E_INVALID;
    }
    const uint64_t D = g->st.dyads;
    {   // cached per world size (the graph is immutable after the build)
        std::lock_guard<std::mutex> lk(g->mu);
        auto it = g->shard_cache.find(world);
        if (it != g->shard_cache.end() && kappa == kShardKappa) {
            for (int r = 0; r <= world; r++) bounds[r] = it->second[r];
            return TC_OK;
        }
    }
    bounds[0] = 0;
    bounds[world] = D;
    if (world > 1 && D > 0) {
        Mem mem = g->mem;
        mem.stream = s;
        tc_status st;
        DevBuf<uint64_t> excl, tot, tg, out;
        if ((st = excl.allocate(mem, D)) != TC_OK) return st;
        if ((st = tot.allocate(mem, 1)) != TC_OK) return st;
        const PlanIn P{g->dyad_u, g->dyad_e, g->dyad_c, g->dyad_t, g->dyad_pb, g->ups, g->off,
                       g->tagpre != nullptr};
        st = scan_exclusive<uint64_t>(mem, D, WorkIn{P, kappa}, ArrayOutExcl<uint64_t>{excl.p},
                                      tot.p, s, nullptr);
        if (st != TC_OK) return st;
        uint64_t T = 0;
        TC_CUDA(cudaMemcpyAsync(&T, tot.p, sizeof(T), cudaMemcpyDeviceToHost, s));
        TC_CUDA(cudaStreamSynchronize(s));
        std::vector<uint64_t> targets(world - 1);
        for (int r = 1; r < world; r++)
            targets[r - 1] = (uint64_t)(((unsigned __int128)T * (unsigned)r) / (unsigned)world);
        if ((st = tg.allocate(mem, world)) != TC_OK) return st;
        if ((st = out.allocate(mem, world)) != TC_OK) return st;
        TC_CUDA(cudaMemcpyAsync(tg.p, targets.data(), (world - 1) * sizeof(uint64_t),
                                cudaMemcpyHostToDevice, s));
        k_lower_bounds<<<(unsigned)((world + 255) / 256), 256, 0, s>>>(excl.p, D, tg.p, world - 1,
                                                                      out.p);
        TC_CUDA(cudaGetLastError());
        TC_CUDA(cudaMemcpyAsync(bounds + 1, out.p, (world - 1) * sizeof(uint64_t),
                                cudaMemcpyDeviceToHost, s));
        TC_CUDA(cudaStreamSynchronize(s));
    }
    if (kappa == kShardKappa) {
        std::lock_guard<std::mutex> lk(g->mu);
        g->shard_cache[world].assign(bounds, bounds + world + 1);
    }
    return TC_OK;
}

}  // namespace tc
