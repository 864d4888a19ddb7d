// csr_build.cu -- a1: GPU CSR builder.
//
// From an arc list it builds ONE symmetric neighbour CSR over N(u) (the
// paper's "array of neighbour lists" N, stored as the adjacency array
// of P:458-469) where every entry carries the 2-bit direction code, so the
// census never probes IsEdge / IsNeighbour -- the tags answer them.
//
//   1. keys      arc (s,d), s != d -> one canonical key (min<<32 | max<<2 |
//                dir), dir = 1 if min->max else 2; self-loops and arcs with
//                an endpoint >= n -> all-ones sentinel keys that sort last
//                (strict digraph); computed by the first radix
//                pass straight from the arc list, which also counts them.
//   2. sort      LSD radix sort (radix_sort.cu) on the min (row) bits, then
//                a row sort by the max bits (bitonic networks per row, in
//                registers for rows <= 64 keys, in shared memory up to
//                kRowMed): canonical pairs in the algorithm's own dyad order (u
//                ascending, v ascending).  Rows of more than
//                kRowMed keys are sorted together by one LSD (max bits, row
//                bits) of their keys (k_huge_rows).  Hub graphs (more than a
//                fifth of the keys in rows of > 64, known after one host read)
//                take the full LSD (max bits, then min bits) instead.  The row
//                sort also flags duplicate (row, max) keys; without any, the
//                run-head count below skips reading the keys.
//   3. compact   a ballot/popc compaction keeps the first key of each (min,
//                max) run with the OR of the run's direction bits (dedup +
//                mutual merge): the canonical dyad list dyad_u / dyad_e (the
//                upper halves of the rows), the transposed keys (max<<32 |
//                dyad index) and the lower entries (min<<2 | swapped tag).
//   4. sort      stable LSD sort of the D transposed keys on the row bits
//                only (they arrive sorted by min, so each row ends up sorted);
//                D is read on the device (no host round trip).
//   5. assemble  row u = lower part (w < u) then upper part (w > u), both
//                already sorted, then one sentinel 0xffffffff (greater than
//                any real entry) so the census merge runs off a row end
//                without bounds checks:  row u = adj[off[u], off[u+1] - 1),
//                off[u] = lo_start[u] + up_start[u] + u; ups[u] = start of
//                the upper part of row u.
//   6. stats     m, mutual dyads, sum d^2, max degree, per-dyad cost c,
//                where the entries w > u of row v start (dyad_pb: one past
//                the lower entry u of row v) and the merge length t
//                (census.cu); the upper entries, c and t are written by
//                schedule.cu k_upper_plan, which also stores the graph's
//                full-census plan (thread-bin items sorted by t per tile).
// Sorting one key per arc and D transposed keys (instead of both
// orientations of every arc) cuts the sort work by a quarter and halves the
// compaction.
#include <stdio.h>

#include "radix_sort.cuh"
#include "scan.cuh"

namespace tc {

namespace {

constexpr uint64_t kSentinel = ~0ull;
constexpr int kHcThreads = 256;
constexpr int kHcWarps = kHcThreads / 32;
constexpr int kHcItems = 16;
constexpr int kHcTile = kHcThreads * kHcItems;   // keys per block

__global__ void k_emit(const uint32_t *__restrict__ src, const uint32_t *__restrict__ dst,
                       uint64_t m, uint64_t n, uint64_t *__restrict__ keys,
                       unsigned long long *__restrict__ scratch /* [0]=bad, [1]=dropped */) {
    unsigned long long loops = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t s = src[i], d = dst[i];
        uint64_t k;
        if (s >= n || d >= n) {
            atomicMin(&scratch[0], (unsigned long long)i);
            loops++;                 // dropped-arc count: loops + out of range
            k = kSentinel;
        } else if (s == d) {
            loops++;
            k = kSentinel;
        } else {
            const uint32_t lo = s < d ? s : d, hi = s < d ? d : s;
            k = ((uint64_t)lo << 32) | ((uint64_t)hi << 2) | (s < d ? 1ull : 2ull);
        }
        keys[i] = k;
    }
    for (int o = 16; o; o >>= 1) loops += __shfl_xor_sync(0xffffffffu, loops, o);
    if ((threadIdx.x & 31) == 0 && loops) atomicAdd(&scratch[1], loops);
}

__device__ __forceinline__ unsigned long long warp_sum64(unsigned long long x) {
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

__device__ __forceinline__ uint32_t key_row(uint64_t k) { return (uint32_t)(k >> 32); }
__device__ __forceinline__ uint32_t key_col(uint64_t k) { return (uint32_t)((k >> 2) & 0x3fffffffu); }
__device__ __forceinline__ uint32_t swap_tag(uint32_t t) { return ((t & 1u) << 1) | (t >> 1); }

// The warp's 512 keys (iteration r holds keys base + 32 r + lane), all loaded
// before use (16 loads in flight per lane), plus the key before the chunk
// (lane 0) and the key after it (lane 31).
struct HeadChunk {
    uint64_t k[kHcItems];
    uint64_t before, after;
};

__device__ __forceinline__ void load_chunk(const uint64_t *__restrict__ key, size_t L, size_t base,
                                           HeadChunk &c) {
    const uint32_t lane = threadIdx.x & 31;
#pragma unroll
    for (int r = 0; r < kHcItems; r++) {
        const size_t i = base + (size_t)r * 32 + lane;
        c.k[r] = i < L ? __ldg(key + i) : kSentinel;
    }
    c.before = (lane == 0 && base > 0 && base - 1 < L) ? __ldg(key + base - 1) : kSentinel;
    const size_t ia = base + 32 * kHcItems;
    c.after = (lane == 31 && ia < L) ? __ldg(key + ia) : kSentinel;
}

// iteration r: key, predecessor, successor, and whether it starts a (row,
// col) run (all lanes must call it: shuffles)
__device__ __forceinline__ bool chunk_head(const HeadChunk &c, int r, size_t L, size_t i,
                                           uint64_t &k, uint64_t &prev, uint64_t &nxt) {
    const uint32_t lane = threadIdx.x & 31;
    k = c.k[r];
    prev = __shfl_up_sync(0xffffffffu, k, 1);
    const uint64_t pl = __shfl_sync(0xffffffffu, c.k[r > 0 ? r - 1 : 0], 31);
    if (lane == 0) prev = r > 0 ? pl : c.before;
    nxt = __shfl_down_sync(0xffffffffu, k, 1);
    const uint64_t nf = __shfl_sync(0xffffffffu, c.k[r < kHcItems - 1 ? r + 1 : r], 0);
    if (lane == 31) nxt = r < kHcItems - 1 ? nf : c.after;
    return i < L && (i == 0 || (prev >> 2) != (k >> 2));
}

// ---------------------------------------------------------------------------
// Row sort (step 2, round 2): the LSD passes run over the min (row) bits only,
// so the keys leave the sort grouped by row (rows in ascending order) but
// unordered inside a row; each row is then ordered by its low word (max << 2 |
// dir) in place, instead of ceil(b / 8) more LSD passes over all m keys.  Rows
// are independent, so they are sorted by length class:
//   k_row_bounds    start / end of every row (the keys at row changes)
//   k_row_classify  per vertex: length class -> the class's work list
//   k_row_sort_net  rows of <= 8 / 16 / 32 keys: one THREAD per row, the
//                   row's low words in registers through a bitonic network
//   k_row_sort_warp rows of 33..kRowMed keys: one warp per row, a bitonic
//                   network over the low words in shared memory
// Rows of more than kRowMed keys (hub rows) are gathered into one array of
// (row-list index, low word) keys, LSD-sorted and scattered back.
// Keys equal in (row, max) are duplicates or the two arcs of a mutual pair;
// the compaction merges them in any order.
// ---------------------------------------------------------------------------
constexpr int kRowMed = 1024;
constexpr int kRowClasses = 6;   // <= 8, <= 16, <= 32, <= 64, <= kRowMed, larger

// two keys per thread (one 16-byte load); a row start / end writes its
// position into rstart / rend of the row (rows ascend with the position)
__global__ void k_row_bounds(const uint64_t *__restrict__ X, size_t m,
                             const unsigned long long *__restrict__ dropped,
                             uint32_t *__restrict__ rstart, uint32_t *__restrict__ rend) {
    const size_t L = m - *dropped;
    const uint32_t lane = threadIdx.x & 31;
    const size_t p = 2 * ((size_t)blockIdx.x * blockDim.x + threadIdx.x);
    if (p - 2 * lane >= L) return;   // warp-uniform
    uint32_t r0 = ~0u, r1 = ~0u;
    if (p + 1 < L) {
        const ulonglong2 k = __ldg(reinterpret_cast<const ulonglong2 *>(X + p));
        r0 = (uint32_t)(k.x >> 32);
        r1 = (uint32_t)(k.y >> 32);
    } else if (p < L) {
        r0 = (uint32_t)(__ldg(X + p) >> 32);
    }
    uint32_t prv = __shfl_up_sync(0xffffffffu, r1, 1);
    uint32_t nxt = __shfl_down_sync(0xffffffffu, r0, 1);
    if (lane == 0) prv = p ? (uint32_t)(__ldg(X + p - 1) >> 32) : ~r0;
    if (lane == 31) nxt = p + 2 < L ? (uint32_t)(__ldg(X + p + 2) >> 32) : ~r1;
    if (p < L) {
        if (prv != r0) rstart[r0] = (uint32_t)p;
        if (p + 1 < L) {
            if (r1 != r0) {
                rend[r0] = (uint32_t)(p + 1);
                rstart[r1] = (uint32_t)(p + 1);
            }
            if (nxt != r1) rend[r1] = (uint32_t)(p + 2);
        } else {
            rend[r0] = (uint32_t)(p + 1);
        }
    }
}

__device__ __forceinline__ int row_class(uint32_t len) {
    return len <= 1 ? -1 : len <= 8 ? 0 : len <= 16 ? 1 : len <= 32 ? 2 : len <= 64 ? 3
         : len <= (uint32_t)kRowMed ? 4 : 5;
}

// lists: kRowClasses arrays of n entries each; cnt[c] = entries of class c,
// cnt[kRowClasses] / cnt[kRowClasses + 1] = keys in rows of more than 64 /
// more than kRowMed keys.
// Each block takes one contiguous range of vertices: it counts its classes,
// reserves them with one atomic per class (no contention on the counters),
// then writes its entries (vertex order inside the block's share).
constexpr int kRcThreads = 256;
__global__ void __launch_bounds__(kRcThreads)
k_row_classify(const uint32_t *__restrict__ rstart, const uint32_t *__restrict__ rend,
               uint64_t n, uint32_t *__restrict__ lists, unsigned long long *__restrict__ cnt) {
    __shared__ uint32_t wcnt[kRcThreads / 32][kRowClasses];
    __shared__ unsigned long long base[kRowClasses];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t per = (n + gridDim.x - 1) / gridDim.x;
    const uint64_t u0 = (uint64_t)blockIdx.x * per, u1 = min(n, u0 + per);
    if (threadIdx.x < kRcThreads / 32 * kRowClasses) (&wcnt[0][0])[threadIdx.x] = 0;
    __syncthreads();
    // pass 1: per-warp class counts over the block's range
    uint32_t c_loc[kRowClasses] = {0, 0, 0, 0, 0, 0};
    unsigned long long long_keys = 0, huge_keys = 0;   // keys in rows of > 64 / > kRowMed
    for (uint64_t u = u0 + threadIdx.x; u < u1; u += kRcThreads) {
        const uint32_t len = __ldg(rend + u) - __ldg(rstart + u);
        const int c = row_class(len);
        long_keys += len > 64 ? len : 0;
        huge_keys += len > (uint32_t)kRowMed ? len : 0;
#pragma unroll
        for (int k = 0; k < kRowClasses; k++) c_loc[k] += c == k;
    }
#pragma unroll
    for (int k = 0; k < kRowClasses; k++) {
        const uint32_t t = __reduce_add_sync(0xffffffffu, c_loc[k]);
        if (lane == 0) wcnt[warp][k] = t;
    }
    long_keys = warp_sum64(long_keys);
    huge_keys = warp_sum64(huge_keys);
    if (lane == 0 && long_keys) atomicAdd(&cnt[kRowClasses], long_keys);
    if (lane == 0 && huge_keys) atomicAdd(&cnt[kRowClasses + 1], huge_keys);
    __syncthreads();
    if (threadIdx.x < kRowClasses) {
        uint32_t t = 0;
        for (int w = 0; w < kRcThreads / 32; w++) t += wcnt[w][threadIdx.x];
        base[threadIdx.x] = t ? atomicAdd(&cnt[threadIdx.x], (unsigned long long)t) : 0ull;
    }
    __syncthreads();
    // pass 2: block-ordered write positions (running per-class offsets)
    for (uint64_t u00 = u0; u00 < u1; u00 += kRcThreads) {
        const uint64_t u = u00 + threadIdx.x;
        const int c = u < u1 ? row_class(__ldg(rend + u) - __ldg(rstart + u)) : -1;
        uint32_t mine = 0;
#pragma unroll
        for (int k = 0; k < kRowClasses; k++) {
            const uint32_t bal = __ballot_sync(0xffffffffu, c == k);
            if (lane == 0) wcnt[warp][k] = __popc(bal);
            if (c == k) mine = __popc(bal & ((1u << lane) - 1u));
        }
        __syncthreads();
        if (c >= 0) {
            uint32_t off = 0;
            for (int w = 0; w < (int)warp; w++) off += wcnt[w][c];
            lists[(size_t)c * n + base[c] + off + mine] = (uint32_t)u;
        }
        __syncthreads();
        if (threadIdx.x < kRowClasses) {
            uint32_t t = 0;
            for (int w = 0; w < kRcThreads / 32; w++) t += wcnt[w][threadIdx.x];
            base[threadIdx.x] += t;
        }
        __syncthreads();
    }
}

// one thread per row of <= P keys: bitonic network over the row's low words
// in registers (the row key is the same for all)
template <int P>
__device__ __forceinline__ void sort_row_regs(uint64_t *__restrict__ X, uint32_t u, uint32_t s0,
                                              uint32_t len, unsigned long long *dupf) {
    uint32_t v[P];
#pragma unroll
    for (int j = 0; j < P; j++) v[j] = j < (int)len ? (uint32_t)__ldg(X + s0 + j) : ~0u;
#pragma unroll
    for (int k = 2; k <= P; k <<= 1) {
#pragma unroll
        for (int h = k >> 1; h > 0; h >>= 1) {
#pragma unroll
            for (int j = 0; j < P; j++) {
                const int x = j ^ h;
                if (x > j) {
                    const uint32_t a = v[j], b = v[x];
                    const bool up = (j & k) == 0;
                    v[j] = up ? min(a, b) : max(a, b);
                    v[x] = up ? max(a, b) : min(a, b);
                }
            }
        }
    }
    const uint64_t hi = (uint64_t)u << 32;
    bool dup = false;   // two keys of one (row, max): a duplicate arc or a mutual pair
#pragma unroll
    for (int j = 0; j < P; j++) {
        if (j < (int)len) X[s0 + j] = hi | v[j];
        if (j + 1 < P) dup |= j + 1 < (int)len && (v[j] >> 2) == (v[j + 1] >> 2);
    }
    if (dup) atomicOr(dupf, 1ull);
}

// classes 0..2 (rows of 2..32 keys) in one launch: block b belongs to the
// class whose block range holds it (class c has ceil(cnt[c] / 128) blocks)
constexpr int kRssThreads = 128;
#ifndef TC_RSS_MINB
#define TC_RSS_MINB 8
#endif
__global__ void __launch_bounds__(kRssThreads, TC_RSS_MINB)
k_row_sort_small(uint64_t *__restrict__ X, const uint32_t *__restrict__ rstart,
                 const uint32_t *__restrict__ rend, const uint32_t *__restrict__ lists, uint64_t n,
                 const unsigned long long *__restrict__ cnt, unsigned long long *dupf) {
    uint64_t b = blockIdx.x;
    int c = 0;
    for (; c < 3; c++) {
        const uint64_t nb = (cnt[c] + kRssThreads - 1) / kRssThreads;
        if (b < nb) break;
        b -= nb;
    }
    if (c == 3) return;   // block-uniform
    const uint64_t i = b * kRssThreads + threadIdx.x;
    if (i >= cnt[c]) return;
    const uint32_t u = __ldg(lists + (size_t)c * n + i);
    const uint32_t s0 = __ldg(rstart + u), len = __ldg(rend + u) - s0;
    if (c == 0) sort_row_regs<8>(X, u, s0, len, dupf);
    else if (c == 1) sort_row_regs<16>(X, u, s0, len, dupf);
    else sort_row_regs<32>(X, u, s0, len, dupf);
}

// class 3 (33..64 keys): one warp per row, two elements per lane, bitonic
// network across lanes by shuffles
__global__ void __launch_bounds__(256)
k_row_sort_w64(uint64_t *__restrict__ X, const uint32_t *__restrict__ rstart,
               const uint32_t *__restrict__ rend, const uint32_t *__restrict__ list,
               const unsigned long long *__restrict__ cnt, unsigned long long *dupf) {
    const uint64_t nr = *cnt;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t i = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < nr; i += nw) {
        const uint32_t u = __ldg(list + i);
        const uint32_t s0 = __ldg(rstart + u), len = __ldg(rend + u) - s0;
        uint32_t e0 = lane < len ? (uint32_t)__ldg(X + s0 + lane) : ~0u;
        uint32_t e1 = lane + 32 < len ? (uint32_t)__ldg(X + s0 + 32 + lane) : ~0u;
    #pragma unroll
        for (uint32_t k = 2; k <= 64; k <<= 1) {
    #pragma unroll
            for (uint32_t h = k >> 1; h > 0; h >>= 1) {
                if (h == 32) {   // pairs (lane, lane + 32), k = 64: ascending
                    const uint32_t lo = min(e0, e1), hv = max(e0, e1);
                    e0 = lo;
                    e1 = hv;
                } else {
                    const uint32_t o0 = __shfl_xor_sync(0xffffffffu, e0, h);
                    const uint32_t o1 = __shfl_xor_sync(0xffffffffu, e1, h);
                    // element index lane (+ 32): keep the min iff ascending == lower
                    const bool lower = (lane & h) == 0;
                    const bool up0 = (lane & k) == 0, up1 = ((lane + 32) & k) == 0;
                    e0 = (up0 == lower) ? min(e0, o0) : max(e0, o0);
                    e1 = (up1 == lower) ? min(e1, o1) : max(e1, o1);
                }
            }
        }
        const uint64_t hi = (uint64_t)u << 32;
        if (lane < len) X[s0 + lane] = hi | e0;
        if (lane + 32 < len) X[s0 + 32 + lane] = hi | e1;
        // duplicates: element i against element i + 1 (i = lane, lane + 32)
        const uint32_t n0 = __shfl_down_sync(0xffffffffu, e0, 1), f1 = __shfl_sync(0xffffffffu, e1, 0);
        const uint32_t n1 = __shfl_down_sync(0xffffffffu, e1, 1);
        const uint32_t next0 = lane < 31 ? n0 : f1;
        const bool dup = (lane + 1 < len && (e0 >> 2) == (next0 >> 2)) ||
                         (lane < 31 && lane + 33 < len && (e1 >> 2) == (n1 >> 2));
        if (__any_sync(0xffffffffu, dup) && lane == 0) atomicOr(dupf, 1ull);
    }
}

// class 4 (65..kRowMed keys): one warp per row, bitonic network in shared memory
constexpr int kRswThreads = 256;
__global__ void __launch_bounds__(kRswThreads)
k_row_sort_warp(uint64_t *__restrict__ X, const uint32_t *__restrict__ rstart,
                const uint32_t *__restrict__ rend, const uint32_t *__restrict__ list,
                const unsigned long long *__restrict__ cnt, unsigned long long *dupf) {
    __shared__ uint32_t buf[kRswThreads / 32][kRowMed];
    const uint64_t nr = *cnt;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t *b = buf[warp];
    const size_t nw = ((size_t)gridDim.x * kRswThreads) >> 5;
    for (size_t i = ((size_t)blockIdx.x * kRswThreads + threadIdx.x) >> 5; i < nr; i += nw) {
        const uint32_t u = __ldg(list + i);
        const uint32_t s0 = __ldg(rstart + u), len = __ldg(rend + u) - s0;
        uint32_t P = 128;
        while (P < len) P <<= 1;
        for (uint32_t j = lane; j < P; j += 32) b[j] = j < len ? (uint32_t)__ldg(X + s0 + j) : ~0u;
        __syncwarp();
        for (uint32_t k = 2; k <= P; k <<= 1) {
            for (uint32_t h = k >> 1; h > 0; h >>= 1) {
                // P / 2 compare-exchanges per step, one pair (j, j ^ h), j with bit h clear
                for (uint32_t q = lane; q < P / 2; q += 32) {
                    const uint32_t j = ((q & ~(h - 1)) << 1) | (q & (h - 1)), x = j | h;
                    const uint32_t va = b[j], vb = b[x];
                    const bool up = (j & k) == 0;
                    b[j] = up ? min(va, vb) : max(va, vb);
                    b[x] = up ? max(va, vb) : min(va, vb);
                }
                __syncwarp();
            }
        }
        const uint64_t hi = (uint64_t)u << 32;
        bool dup = false;
        for (uint32_t j = lane; j < len; j += 32) {
            X[s0 + j] = hi | b[j];
            dup |= j + 1 < len && (b[j] >> 2) == (b[j + 1] >> 2);
        }
        if (__any_sync(0xffffffffu, dup) && lane == 0) atomicOr(dupf, 1ull);
        __syncwarp();
    }
}

// rows of more than kRowMed keys (hub rows): gathered into one array of
// composite keys (index of the row in the class list << 32 | low word), LSD
// sorted on the max bits and then the row-index bits (radix_sort.cu), and
// scattered back; hoff = exclusive prefix of the rows' lengths (list order)
struct HugeLen {
    const uint32_t *list, *rstart, *rend;
    __device__ __forceinline__ uint32_t operator()(size_t i) const {
        const uint32_t u = list[i];
        return rend[u] - rstart[u];
    }
};

template <bool GATHER>
__global__ void k_huge_rows(uint64_t *__restrict__ X, uint64_t *__restrict__ S,
                            const uint32_t *__restrict__ rstart, const uint32_t *__restrict__ list,
                            const uint32_t *__restrict__ hoff, uint64_t nh, uint64_t ns) {
    // one thread per element of S: its row i = last hoff[i] <= e (binary search)
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < ns;
         e += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t lo = 0, hi = nh;
        while (hi - lo > 1) {
            const uint64_t mid = (lo + hi) >> 1;
            if (__ldg(hoff + mid) <= e) lo = mid;
            else hi = mid;
        }
        const uint32_t u = __ldg(list + lo);
        const uint64_t x = __ldg(rstart + u) + (e - __ldg(hoff + lo));
        if (GATHER) S[e] = lo << 32 | (uint32_t)X[x];
        else X[x] = (uint64_t)u << 32 | (uint32_t)S[e];
    }
}

// pass 1: per warp (512 keys), number of run heads
__global__ void __launch_bounds__(kHcThreads)
k_head_count(const uint64_t *__restrict__ key, size_t m, const unsigned long long *dropped,
             uint32_t *__restrict__ warp_tot, const unsigned long long *dupf) {
    const size_t L = m - *dropped;   // canonical keys (dropped arcs sort last)
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const size_t base = (size_t)blockIdx.x * kHcTile + (size_t)warp * 32 * kHcItems;
    if (!*dupf) {   // the row sort saw no two keys of one (row, max): every key heads its run
        if (lane == 0)
            warp_tot[(size_t)blockIdx.x * kHcWarps + warp] =
                (uint32_t)(base >= L ? 0 : min((size_t)(32 * kHcItems), L - base));
        return;
    }
    HeadChunk c;
    load_chunk(key, L, base, c);
    uint32_t nh = 0;
#pragma unroll
    for (int r = 0; r < kHcItems; r++) {
        uint64_t k, prev, nxt;
        const bool head = chunk_head(c, r, L, base + (size_t)r * 32 + lane, k, prev, nxt);
        nh += __popc(__ballot_sync(0xffffffffu, head));
    }
    if (lane == 0) warp_tot[(size_t)blockIdx.x * kHcWarps + warp] = nh;
}

// TC_HW_MINB: minimum blocks per SM for k_head_write (unset: plain
// __launch_bounds__, 64 registers; an explicit 1 lets ptxas take 96)
// pass 2: canonical dyad list, transposed keys (row v, dyad index k), the
// lower entry of each dyad (ul[k] = u<<2 | swapped tag) and up_start at row
// changes (warp_off = exclusive scan of pass 1's per-warp counts)
#ifdef TC_HW_MINB
__global__ void __launch_bounds__(kHcThreads, TC_HW_MINB)
#else
__global__ void __launch_bounds__(kHcThreads)
#endif
k_head_write(const uint64_t *__restrict__ key, size_t m, const unsigned long long *dropped,
             const uint32_t *__restrict__ warp_off,
             uint32_t *__restrict__ du, uint32_t *__restrict__ de, uint64_t *__restrict__ tk,
             uint32_t *__restrict__ ul, uint32_t *__restrict__ up_start) {
    const size_t L = m - *dropped;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    const size_t base = (size_t)blockIdx.x * kHcTile + (size_t)warp * 32 * kHcItems;
    uint32_t k0 = warp_off[(size_t)blockIdx.x * kHcWarps + warp];
    HeadChunk c;
    load_chunk(key, L, base, c);
#pragma unroll
    for (int r = 0; r < kHcItems; r++) {
        const size_t i = base + (size_t)r * 32 + lane;
        uint64_t k, prev, nxt;
        const bool head = chunk_head(c, r, L, i, k, prev, nxt);
        const uint32_t bh = __ballot_sync(0xffffffffu, head);
        if (head) {
            const uint32_t kk = k0 + __popc(bh & lt);
            const uint32_t row = key_row(k), col = key_col(k);
            uint32_t tag = (uint32_t)(k & 3u);
            if ((nxt >> 2) == (k >> 2)) {            // mutual pair and/or duplicates
                tag |= (uint32_t)(nxt & 3u);
#pragma unroll 1
                for (size_t j = i + 2; j < L && tag != 3u; j++) {   // longer runs: duplicates
                    const uint64_t kj = __ldg(key + j);
                    if ((kj >> 2) != (k >> 2)) break;
                    tag |= (uint32_t)(kj & 3u);
                }
            }
            du[kk] = row;
            de[kk] = (col << 2) | tag;
            tk[kk] = ((uint64_t)col << 32) | kk;
            ul[kk] = (row << 2) | swap_tag(tag);
            if (i == 0 || key_row(prev) != row) {     // rows (prev_row, row] start here
                const uint32_t first = i == 0 ? 0u : key_row(prev) + 1;
#pragma unroll 1
                for (uint32_t x = first; x <= row; x++) up_start[x] = kk;
            }
        }
        k0 += __popc(bh);
    }
}


// lower entries: row r's i-th key of the row-sorted transposed list is dyad
// k = (u, r); its entry ul[k] goes to off[r] + (i - lo_start[r]) =
// up_start[r] + r + i, and ul[k] is overwritten with that position + 1 (the
// first entry w > u of row r: dyad_pb).  One random read-modify-write per
// dyad into a D-word array (L2-resident at the Patents size) instead of a
// search of row r.
// The same pass records lo_start[x] = first index of row x among the
// row-sorted transposed keys (rows with no lower entries get the next row's
// start; the rows after the last one are filled by k_fill_tail_last).
// Each thread takes kWlBatch keys (grid-strided) and issues all their loads --
// the keys, up_start of their rows, the random ul[k] -- before any store, so
// the random L2 round trips overlap instead of serialising behind the
// (possibly aliasing) ul[k] stores of the previous key.
constexpr int kWlBatch = 4;
// TC_WL_PARTS: the dyads are handled in that many launches by dyad-index
// range [klo, khi) (the random ul[k] working set of one launch is D / parts
// words, so it stays in L2 while the sorted keys stream past); the row starts
// are written by the first launch
#ifndef TC_WL_PARTS
#define TC_WL_PARTS 1
#endif
// TC_WL_HINT: L2 cache hints.  1 = the sorted keys and the adj stores
// stream (evict-first); 2 = also the random ul[k] read-modify-write carries
// an evict_last policy, so the D-word array stays in L2 while the 8-byte
// keys stream past it and its partially written sectors are not written
// back and re-fetched
#ifndef TC_WL_HINT
#define TC_WL_HINT 0
#endif
#if TC_WL_HINT >= 2
__device__ __forceinline__ uint32_t wl_ld_keep(const uint32_t *p, uint64_t pol) {
    uint32_t v;
    asm volatile("ld.global.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void wl_st_keep(uint32_t *p, uint32_t v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.u32 [%0], %1, %2;" :: "l"(p), "r"(v), "l"(pol) : "memory");
}
#endif
__global__ void k_write_lower(const uint64_t *__restrict__ tk, const uint32_t *__restrict__ dD,
                              const uint32_t *__restrict__ up_start, uint32_t *__restrict__ adj,
                              uint32_t *__restrict__ ul, uint32_t *__restrict__ lo_start,
                              uint32_t klo, uint32_t khi, int starts) {
    const size_t D = *dD;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
#if TC_WL_HINT >= 2
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
#endif
    for (size_t i0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < D;
         i0 += kWlBatch * stride) {
        uint64_t key[kWlBatch], prv[kWlBatch];
        uint32_t us[kWlBatch], val[kWlBatch];
#pragma unroll
        for (int j = 0; j < kWlBatch; j++) {
            const size_t i = i0 + j * stride;
#if TC_WL_HINT >= 1
            key[j] = i < D ? __ldcs(tk + i) : 0ull;
            prv[j] = (i < D && i) ? __ldcs(tk + i - 1) : ~0ull;
#else
            key[j] = i < D ? __ldg(tk + i) : 0ull;
            prv[j] = (i < D && i) ? __ldg(tk + i - 1) : ~0ull;
#endif
        }
#pragma unroll
        for (int j = 0; j < kWlBatch; j++) {
            const size_t i = i0 + j * stride;
            const uint32_t k = (uint32_t)key[j];
            const bool mine = i < D && k >= klo && k < khi;
            us[j] = mine ? __ldg(up_start + key_row(key[j])) : 0u;
#if TC_WL_HINT >= 2
            val[j] = mine ? wl_ld_keep(ul + k, pol) : 0u;
#else
            val[j] = mine ? ul[k] : 0u;
#endif
        }
#pragma unroll
        for (int j = 0; j < kWlBatch; j++) {
            const size_t i = i0 + j * stride;
            if (i >= D) continue;
            const uint32_t r = key_row(key[j]), k = (uint32_t)key[j];
            if (k >= klo && k < khi) {
                const uint32_t pos = us[j] + r + (uint32_t)i;
#if TC_WL_HINT >= 1
                __stcs(adj + pos, val[j]);
#else
                adj[pos] = val[j];
#endif
#if TC_WL_HINT >= 2
                wl_st_keep(ul + k, pos + 1u, pol);
#else
                ul[k] = pos + 1u;
#endif
            }
            const uint32_t prev = i ? key_row(prv[j]) : 0xffffffffu;
            if (starts && (i == 0 || prev != r)) {
                const uint32_t first = i == 0 ? 0u : prev + 1;
                for (uint32_t x = first; x <= r; x++) lo_start[x] = (uint32_t)i;
            }
        }
    }
}

// up_start[x] = D for the rows after the last canonical row (L and D read
// on the device)
__global__ void k_fill_tail_up(uint32_t *start, const uint64_t *__restrict__ key, uint64_t m,
                               const unsigned long long *dropped, uint64_t n,
                               const uint32_t *__restrict__ total) {
    const uint64_t L = m - *dropped;
    const uint32_t D = *total;
    const uint64_t from = (L && D) ? (uint64_t)key_row(key[L - 1]) + 1 : 0;
    for (uint64_t x = from + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x <= n;
         x += (uint64_t)gridDim.x * blockDim.x)
        start[x] = D;
}

// start[x] = val for x in (row of the last key, n]: the rows after the last
// one of a row-sorted key array (read on the device: no host round trip)
__global__ void k_fill_tail_last(uint32_t *start, const uint64_t *__restrict__ key,
                                 const uint32_t *__restrict__ dL, uint64_t n) {
    const uint32_t val = *dL;
    const uint64_t L = val;
    const uint64_t from = L ? (uint64_t)key_row(key[L - 1]) + 1 : 0;
    for (uint64_t x = from + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x <= n;
         x += (uint64_t)gridDim.x * blockDim.x)
        start[x] = val;
}

// off[u] = lo_start[u] + up_start[u] + u; sentinel at off[u+1] - 1; slack
// after; ups[u] = off[u] + |lower part of u| = first entry w > u of row u
// also the vertex stats: out[0] += sum d^2, out[1] = max d, d_u = |N(u)| =
// (lo_start[u+1] - lo_start[u]) + (up_start[u+1] - up_start[u])
__global__ void k_offsets(const uint32_t *__restrict__ lo_start,
                          const uint32_t *__restrict__ up_start, uint64_t n,
                          uint32_t *__restrict__ off, uint32_t *__restrict__ ups,
                          uint32_t *__restrict__ adj, unsigned long long *out) {
    unsigned long long s2 = 0, mx = 0;
    for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u <= n + 8;
         u += (uint64_t)gridDim.x * blockDim.x) {
        if (u <= n) {
            const uint32_t o = lo_start[u] + up_start[u] + (uint32_t)u;
            off[u] = o;
            // terminator of row u - 1, if it has no upper entries (the rows
            // with upper entries get theirs from k_upper_plan, next to their
            // last entry)
            if (u > 0 && up_start[u] == up_start[u - 1]) adj[o - 1] = 0xffffffffu;
            if (u < n) {
                const uint32_t l1 = lo_start[u + 1], u1 = up_start[u + 1];
                ups[u] = l1 + up_start[u] + (uint32_t)u;
                const unsigned long long d = (l1 - lo_start[u]) + (u1 - up_start[u]);
                s2 += d * d;
                mx = d > mx ? d : mx;
            }
        } else {
            adj[lo_start[n] + up_start[n] + (uint32_t)u - 1] = 0xffffffffu;   // slack
        }
    }
    s2 = warp_sum64(s2);
    for (int o = 16; o; o >>= 1) {
        const unsigned long long y = __shfl_xor_sync(0xffffffffu, mx, o);
        mx = y > mx ? y : mx;
    }
    if ((threadIdx.x & 31) == 0) {
        if (s2) atomicAdd(&out[0], s2);
        atomicMax(&out[1], mx);
    }
}


// upper entries + per-dyad data (c, t, arc / mutual stats): schedule.cu
// k_upper_plan, fused with the tile-local length sort of the census plan
// (entry of v in row u at lo_start[u+1] + u + k; c = |N(u)| + |N(v)|, P:1693;
// t = entries > u of both rows, census.cu)

// (tag == 1) << 32 | (tag == 2) of adj entry i (sentinels count as tag 3)
struct TagIn {
    const uint32_t *adj;
    __device__ __forceinline__ uint64_t operator()(size_t i) const {
        const uint32_t t = __ldg(adj + i) & 3u;
        return (t == 1u ? (1ull << 32) : 0ull) | (t == 2u ? 1ull : 0ull);
    }
};

inline unsigned grid_for(uint64_t work, int threads, int cap = 148 * 16) {
    uint64_t b = (work + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > (uint64_t)cap) b = cap;
    return (unsigned)b;
}

}  // namespace

tc_status build_csr(tc_graph *g, const uint32_t *d_src, const uint32_t *d_dst, uint64_t m,
                    cudaStream_t s) {
    const uint64_t n = g->st.n;
    tc_status st;
    Mem &mem = g->mem;

    DevBuf<unsigned long long> scratch;
    if ((st = scratch.allocate(mem, 8)) != TC_OK) return st;
    unsigned long long init[8] = {~0ull, 0, 0, 0, 0, 0, 0, 0};
    TC_CUDA(cudaMemcpyAsync(scratch.p, init, sizeof(init), cudaMemcpyHostToDevice, s));

    if (2ull * m + n + 8 >= (1ull << 33)) {   // 2D + n < 2^32 is checked exactly below
        set_error("%llu arcs: 2D + n can exceed the 32-bit CSR offset range",
                  (unsigned long long)m);
        return TC_E_INVALID;
    }
    DevBuf<uint64_t> keys, tmp;
    if ((st = keys.allocate(mem, m)) != TC_OK) return st;
    if ((st = tmp.allocate(mem, m)) != TC_OK) return st;

    // 1 + 2. canonical keys by (min, max), sorted: max bits first, then min
    // bits; the first radix pass computes the keys from the arcs itself and
    // counts the dropped ones (no separate emit pass, no host round trip)
    int b = 1;
    while (b < 32 && (1ull << b) < n) b++;
    RadixPass passes[16];
    uint64_t *sorted = keys.p;
    uint64_t dropped_h = 0;   // loops + out-of-range arcs (host copy, m >= 2)
    if (m >= 2) {
        const ArcSource as{d_src, d_dst, n, scratch.p};
        // LSD over the row (min) bits only, then the row sort (above)
        int np = radix_passes_for(32, b, passes);
        if ((st = radix_sort_u64(mem, keys.p, tmp.p, m, passes, np, s, &g->launches, &sorted,
                                 &as)) != TC_OK)
            return st;
        g->build_sort[0] = (uint64_t)np;
        // row sort, in place in `sorted`
        DevBuf<uint32_t> rb, lists;
        DevBuf<unsigned long long> rc;
        if ((st = rb.allocate(mem, 2 * (n + 1))) != TC_OK) return st;
        if ((st = lists.allocate(mem, (size_t)kRowClasses * n)) != TC_OK) return st;
        if ((st = rc.allocate(mem, kRowClasses + 2)) != TC_OK) return st;
        uint32_t *rstart = rb.p, *rend = rb.p + n + 1;
        TC_CUDA(cudaMemsetAsync(rb.p, 0, 2 * (n + 1) * sizeof(uint32_t), s));
        TC_CUDA(cudaMemsetAsync(rc.p, 0, (kRowClasses + 2) * sizeof(unsigned long long), s));
        k_row_bounds<<<(unsigned)((m + 511) / 512), 256, 0, s>>>(sorted, m, scratch.p + 1, rstart,
                                                                 rend);
        k_row_classify<<<grid_for(n, kRcThreads, 148 * 8), kRcThreads, 0, s>>>(rstart, rend, n,
                                                                         lists.p, rc.p);
        TC_CUDA(cudaGetLastError());
        g->launches += 2;
        // host read: range check, the row classes (hub graph or not)
        unsigned long long h0[2], rch[kRowClasses + 2];
        TC_CUDA(cudaMemcpyAsync(h0, scratch.p, sizeof(h0), cudaMemcpyDeviceToHost, s));
        TC_CUDA(cudaMemcpyAsync(rch, rc.p, sizeof(rch), cudaMemcpyDeviceToHost, s));
        TC_CUDA(cudaStreamSynchronize(s));
        if (h0[0] != ~0ull) {
            set_error("arc %llu has an endpoint >= n (n = %llu)", h0[0], (unsigned long long)n);
            return TC_E_RANGE;
        }
        dropped_h = h0[1];
        if (5 * rch[kRowClasses] > m - dropped_h) {
            // hub graph (more than a fifth of the keys in rows of > 64): the
            // full LSD (max bits, then min bits) from the arcs again is cheaper
            // than sorting the long rows (DESIGN 5.2)
            // scratch[2] = 1: duplicates unknown (the head count reads the keys)
            unsigned long long init2[3] = {~0ull, 0, 1};
            TC_CUDA(cudaMemcpyAsync(scratch.p, init2, sizeof(init2), cudaMemcpyHostToDevice, s));
            np = radix_passes_for(2, b, passes);
            np += radix_passes_for(32, b, passes + np);
            if ((st = radix_sort_u64(mem, keys.p, tmp.p, m, passes, np, s, &g->launches, &sorted,
                                     &as)) != TC_OK)
                return st;
            g->build_sort[0] += (uint64_t)np;
        } else {
            g->build_sort[2] = m - dropped_h - rch[kRowClasses + 1];
            k_row_sort_small<<<(unsigned)(n / kRssThreads + 3), kRssThreads, 0, s>>>(
                sorted, rstart, rend, lists.p, n, rc.p, scratch.p + 2);
            const uint64_t n33 = n < m / 33 ? n : m / 33;   // rows of >= 33 keys
            k_row_sort_w64<<<grid_for(n33 * 32, 256, 148 * 16), 256, 0, s>>>(
                sorted, rstart, rend, lists.p + 3 * n, rc.p + 3, scratch.p + 2);
            k_row_sort_warp<<<148 * 7, kRswThreads, 0, s>>>(sorted, rstart, rend,
                                                            lists.p + 4 * n, rc.p + 4,
                                                            scratch.p + 2);
            TC_CUDA(cudaGetLastError());
            g->launches += 3;
        }
        if (5 * rch[kRowClasses] <= m - dropped_h && rch[kRowClasses - 1]) {
            const uint64_t nh = rch[kRowClasses - 1];   // rows of > kRowMed keys
            const unsigned long long one = 1;   // duplicates in these rows: not checked
            TC_CUDA(cudaMemcpyAsync(scratch.p + 2, &one, sizeof(one), cudaMemcpyHostToDevice, s));
            const uint32_t *hl = lists.p + (size_t)(kRowClasses - 1) * n;
            const uint64_t ns = rch[kRowClasses + 1];
            DevBuf<uint32_t> hoff;
            if ((st = hoff.allocate(mem, nh)) != TC_OK) return st;
            if ((st = scan_exclusive<uint32_t>(mem, nh, HugeLen{hl, rstart, rend},
                                               ArrayOutExcl<uint32_t>{hoff.p}, (uint32_t *)nullptr,
                                               s, &g->launches)) != TC_OK)
                return st;
            DevBuf<uint64_t> S, S2;
            if ((st = S.allocate(mem, ns)) != TC_OK) return st;
            if ((st = S2.allocate(mem, ns)) != TC_OK) return st;
            const unsigned gh = grid_for(ns, 256, 148 * 16);
            k_huge_rows<true><<<gh, 256, 0, s>>>(sorted, S.p, rstart, hl, hoff.p, nh, ns);
            int hb = 1;
            while (hb < 32 && (1ull << hb) < nh) hb++;
            np = radix_passes_for(2, b, passes);
            np += radix_passes_for(32, hb, passes + np);
            uint64_t *ss = S.p;
            if ((st = radix_sort_u64(mem, S.p, S2.p, ns, passes, np, s, &g->launches, &ss)) !=
                TC_OK)
                return st;
            g->build_sort[3] = ns * (uint64_t)np;
            k_huge_rows<false><<<gh, 256, 0, s>>>(sorted, ss, rstart, hl, hoff.p, nh, ns);
            TC_CUDA(cudaGetLastError());
            g->launches += 2;
        }
    } else if (m == 1) {
        k_emit<<<1, 32, 0, s>>>(d_src, d_dst, m, n, keys.p, scratch.p);
        g->launches++;
        TC_CUDA(cudaGetLastError());
    }
    uint64_t *spare = sorted == keys.p ? tmp.p : keys.p;

    // 3. compaction -> canonical dyads (upper halves) + transposed keys; the
    // canonical key count L = m - dropped is read on the device
    const size_t cap = m ? m : 1;
    uint32_t *du = (uint32_t *)mem.alloc(cap * sizeof(uint32_t));
    uint32_t *de = (uint32_t *)mem.alloc(cap * sizeof(uint32_t));
    uint32_t *dc = (uint32_t *)mem.alloc(cap * sizeof(uint32_t));
    uint32_t *dpb = (uint32_t *)mem.alloc(cap * sizeof(uint32_t));
    uint32_t *dt = (uint32_t *)mem.alloc(cap * sizeof(uint32_t));
    uint32_t *off = (uint32_t *)mem.alloc((n + 1) * sizeof(uint32_t));
    uint32_t *ups = (uint32_t *)mem.alloc((n ? n : 1) * sizeof(uint32_t));
    g->dyad_u = du; g->dyad_n = cap;
    g->dyad_e = de;
    g->dyad_c = dc;
    g->dyad_pb = dpb;
    g->dyad_t = dt;
    g->off = off; g->off_n = n + 1;
    g->ups = ups; g->ups_n = n ? n : 1;
    DevBuf<uint32_t> up_start, lo_start;
    if (!du || !de || !dc || !dpb || !dt || !off || !ups) {
        set_error("device allocation for the CSR failed");
        return TC_E_OOM;
    }
    if ((st = up_start.allocate(mem, n + 1)) != TC_OK) return st;
    if ((st = lo_start.allocate(mem, n + 1)) != TC_OK) return st;
    uint32_t D = 0;
    DevBuf<uint32_t> total;
    if ((st = total.allocate(mem, 1)) != TC_OK) return st;
    TC_CUDA(cudaMemsetAsync(total.p, 0, sizeof(uint32_t), s));
    if (m) {
        const size_t ntiles = (m + kHcTile - 1) / kHcTile;
        DevBuf<uint32_t> wt;
        if ((st = wt.allocate(mem, ntiles * kHcWarps)) != TC_OK) return st;
        k_head_count<<<(unsigned)ntiles, kHcThreads, 0, s>>>(sorted, m, scratch.p + 1, wt.p,
                                                             scratch.p + 2);
        TC_CUDA(cudaGetLastError());
        st = scan_exclusive<uint32_t>(mem, ntiles * kHcWarps, ArrayIn<uint32_t>{wt.p},
                                      ArrayOutExcl<uint32_t>{wt.p}, total.p, s, &g->launches);
        if (st != TC_OK) return st;
        k_head_write<<<(unsigned)ntiles, kHcThreads, 0, s>>>(sorted, m, scratch.p + 1, wt.p, du,
                                                             de, spare, dpb, up_start.p);
        TC_CUDA(cudaGetLastError());
        g->launches += 2;
    }
    // rows after the last canonical row have no upper entries
    k_fill_tail_up<<<grid_for(n + 1, 256), 256, 0, s>>>(up_start.p, sorted, m, scratch.p + 1, n,
                                                        total.p);
    TC_CUDA(cudaGetLastError());
    // D stays on the device (total.p): the transposed sort and the assembly
    // kernels read it there and are sized by the host-side bound Dub (the
    // canonical key count L, known from the row sort's host read), so the
    // build has one host round trip.  Graphs whose bound could overflow the
    // 32-bit offsets (2 Dub + n >= 2^32), and m < 2, read D exactly here.
    unsigned long long h[8];
    uint64_t Dub = m >= 2 ? m - dropped_h : 0;
    if (m < 2 || 2ull * Dub + n + 8 >= (1ull << 32)) {
        TC_CUDA(cudaMemcpyAsync(h, scratch.p, sizeof(h), cudaMemcpyDeviceToHost, s));
        TC_CUDA(cudaMemcpyAsync(&D, total.p, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        TC_CUDA(cudaStreamSynchronize(s));
        if (h[0] != ~0ull) {
            set_error("arc %llu has an endpoint >= n (n = %llu)", h[0], (unsigned long long)n);
            return TC_E_RANGE;
        }
        if (2ull * D + n + 8 >= (1ull << 32)) {
            set_error("2D + n = %llu exceeds the 32-bit CSR offset range",
                      (unsigned long long)(2ull * D + n));
            return TC_E_INVALID;
        }
        Dub = D;
    }

    // 4. lower halves: stable sort of the transposed keys on the row bits
    uint64_t *tsorted = spare;
    RadixPass rpasses[8];
    const int nrp = radix_passes_for(32, b, rpasses);
    uint64_t *tother = spare == keys.p ? tmp.p : keys.p;
    if ((st = radix_sort_u64(mem, spare, tother, Dub, rpasses, nrp, s, &g->launches, &tsorted,
                             nullptr, total.p)) != TC_OK)
        return st;
    g->build_sort[1] = Dub ? (uint64_t)nrp : 0;
    // 5. assemble the symmetric rows: lower entries (+ lo_start, dyad_pb),
    // then offsets, sentinels and vertex stats, then upper entries
    uint32_t *adj = (uint32_t *)mem.alloc((2ull * Dub + n + 8) * sizeof(uint32_t));
    g->adj = adj;
    g->adj_alloc_n = 2ull * Dub + n + 8;
    if (!adj) {
        set_error("device allocation for the CSR failed");
        return TC_E_OOM;
    }
    if (Dub) {
        const uint64_t per = (Dub + TC_WL_PARTS - 1) / TC_WL_PARTS;
        for (int part = 0; part < TC_WL_PARTS; part++) {
            const uint64_t klo = per * part, khi = per * (part + 1);
            k_write_lower<<<grid_for(Dub, 256), 256, 0, s>>>(
                tsorted, total.p, up_start.p, adj, dpb, lo_start.p, (uint32_t)klo,
                (uint32_t)(khi < 0xffffffffull ? khi : 0xffffffffull), part == 0);
        }
        g->launches += TC_WL_PARTS;
    }
    k_fill_tail_last<<<grid_for(n + 1, 256), 256, 0, s>>>(lo_start.p, tsorted, total.p, n);
    k_offsets<<<grid_for(n + 9, 256), 256, 0, s>>>(lo_start.p, up_start.p, n, off, ups, adj,
                                                   scratch.p + 4);
    g->launches += 2;
    // the sort buffers are dead from here on (stream-ordered frees)
    keys.release();
    tmp.release();
    // upper entries, c, t, and the graph's own full-census plan (schedule.cu)
    if ((st = upper_plan_device(g, lo_start.p, total.p, Dub, scratch.p + 4, s)) != TC_OK)
        return st;
    TC_CUDA(cudaGetLastError());
    g->st.m_in = m;
    if (g->pin) {   // lazy end: the stats land in the graph's pinned slot
        TC_CUDA(cudaMemcpyAsync(g->pin, scratch.p, 8 * sizeof(unsigned long long),
                                cudaMemcpyDeviceToHost, s));
        TC_CUDA(cudaMemcpyAsync(g->pin + 8, total.p, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        TC_CUDA(cudaEventRecord(g->ready, s));
        g->final_ = false;
        return TC_OK;
    }
    TC_CUDA(cudaMemcpyAsync(h, scratch.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaMemcpyAsync(&D, total.p, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    return build_finish(g, h, D);
}

tc_status build_finish(tc_graph *g, const unsigned long long *h, uint32_t D) {
    const uint64_t n = g->st.n, m = g->st.m_in;
    const uint64_t loops = h[1];
    const uint64_t nnz = 2ull * D;
    g->adj_n = nnz + n + 8;
    // the stats first: a failed tag prefix below leaves a graph whose big
    // dyads are merged instead of searched (same census)
    g->st.loops_dropped = loops;
    g->st.dyads = D;
    g->st.sum_deg_sq = h[4];
    g->st.max_degree = h[5];
    g->st.m = h[6];
    g->st.mutual_dyads = h[7];
    g->st.dups_dropped = m - loops - h[6];
    // 7. tag prefix counts for the skewed-pair path (hub graphs only)
    if (h[5] >= kSparseMinDegree) {
        Mem &mem = g->mem;
        cudaStream_t s = g->stream;
        const size_t nt = nnz + n + 8;
        uint64_t *tp = (uint64_t *)mem.alloc((nt + 1) * sizeof(uint64_t));
        if (!tp) {
            set_error("device allocation for the tag prefix failed");
            return TC_E_OOM;
        }
        tc_status st;
        if ((st = scan_exclusive<uint64_t>(mem, nt, TagIn{g->adj}, ArrayOutExcl<uint64_t>{tp},
                                           tp + nt, s, &g->launches)) != TC_OK) {
            mem.free(tp, (nt + 1) * sizeof(uint64_t));
            return st;
        }
        TC_CUDA(cudaStreamSynchronize(s));
        g->tagpre = tp;   // published only once complete
        g->tagpre_n = nt + 1;
    }
    return TC_OK;
}

}  // namespace tc
