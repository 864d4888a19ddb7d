// radix_sort.cu -- hand-written LSD radix sort of 64-bit keys on selected bit
// fields (a1's sort; SURVEY.md section 7 decision D1: written here, no CUB).
//
// One pass per digit of <= 8 bits (256 buckets), tiles of 4096 keys:
//   upsweep    per-tile digit histogram (shared-memory atomics)
//   scan       per digit, exclusive scan over tiles + digit totals (one
//              block per digit); the downsweep adds the digits' prefix
//   downsweep  stable tile-local counting sort: per warp, one ballot per
//              digit bit groups the lanes holding the same digit (__match_any
//              is ~35% slower here) (rank = earlier peers
//              + running per-warp digit count, 16-bit shared counters); the
//              tile is reordered by digit in shared memory and written out
//              so consecutive threads store consecutive addresses of each
//              digit run (coalesced), instead of a 32-way scatter per warp.
#include <atomic>

#include "radix_sort.cuh"
#include "scan.cuh"

namespace tc {

namespace {

constexpr int kRsThreads = 256;                  // upsweep
#ifndef TC_RS_ITEMS
#define TC_RS_ITEMS 16
#endif
#ifndef TC_DS_MINB
#define TC_DS_MINB 4
#endif
constexpr int kRsItems = TC_RS_ITEMS;
constexpr int kRsTile = kRsThreads * kRsItems;   // 4096 keys per block
constexpr int kDsThreads = 256;                  // downsweep: 16 keys per thread,
constexpr int kDsWarps = kDsThreads / 32;        // no register spills
constexpr int kDsItems = kRsTile / kDsThreads;
constexpr int kMaxBits = 8;
constexpr int kMaxRadix = 1 << kMaxBits;

// The CSR builder's canonical key of arc (s, d) (csr_build.cu step 1):
// min << 32 | max << 2 | dir, dir = 1 if min -> max else 2; self-loops and
// arcs with an endpoint >= nv become all-ones keys that sort last.
__device__ __forceinline__ uint64_t arc_key(uint32_t s, uint32_t d, uint64_t nv) {
    if (s >= nv || d >= nv || s == d) return ~0ull;
    const uint32_t lo = s < d ? s : d, hi = s < d ? d : s;
    return ((uint64_t)lo << 32) | ((uint64_t)hi << 2) | (s < d ? 1ull : 2ull);
}

// ARCS: the first pass reads the arc list itself (no separate key-emit pass)
// and counts the dropped arcs: a.scratch[1] += loops + out-of-range arcs,
// a.scratch[0] = min index of an out-of-range arc.
template <bool ARCS>
__global__ void __launch_bounds__(kRsThreads)
rs_upsweep(const uint64_t *__restrict__ keys, size_t n, int shift, uint32_t mask, int radix,
           uint32_t *__restrict__ hist, size_t ntiles, ArcSource a, const uint32_t *dn) {
    __shared__ uint32_t h[kMaxRadix];
    if (dn) n = min(n, (size_t)*dn);   // device-side key count (tiles past it count zero)
    for (int i = threadIdx.x; i < radix; i += kRsThreads) h[i] = 0;
    __syncthreads();
    const size_t base = (size_t)blockIdx.x * kRsTile;
    if (ARCS) {
        unsigned long long dropped = 0;
        if (base + kRsTile <= n &&
            ((reinterpret_cast<uintptr_t>(a.src) | reinterpret_cast<uintptr_t>(a.dst)) & 15u) == 0) {
            // full tile of 16-byte-aligned arc arrays: 4 arcs per load, all
            // loads in flight before the first count (as the key path)
            const uint4 *s4 = reinterpret_cast<const uint4 *>(a.src + base);
            const uint4 *d4 = reinterpret_cast<const uint4 *>(a.dst + base);
            uint4 sv[kRsItems / 4], dv[kRsItems / 4];
#pragma unroll
            for (int k = 0; k < kRsItems / 4; k++) {
                sv[k] = __ldcs(s4 + k * kRsThreads + threadIdx.x);
                dv[k] = __ldcs(d4 + k * kRsThreads + threadIdx.x);
            }
#pragma unroll
            for (int k = 0; k < kRsItems / 4; k++) {
                const uint32_t ss[4] = {sv[k].x, sv[k].y, sv[k].z, sv[k].w};
                const uint32_t dd[4] = {dv[k].x, dv[k].y, dv[k].z, dv[k].w};
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const uint64_t key = arc_key(ss[j], dd[j], a.nv);
                    if (key == ~0ull) {
                        dropped++;
                        if (ss[j] >= a.nv || dd[j] >= a.nv)
                            atomicMin(&a.scratch[0], (unsigned long long)(
                                base + 4 * ((size_t)k * kRsThreads + threadIdx.x) + j));
                    }
                    atomicAdd(&h[(uint32_t)(key >> shift) & mask], 1u);
                }
            }
        } else {
#pragma unroll 4
            for (int k = 0; k < kRsItems; k++) {
                const size_t i = base + (size_t)k * kRsThreads + threadIdx.x;
                if (i < n) {
                    const uint32_t sv = __ldg(a.src + i), dv = __ldg(a.dst + i);
                    const uint64_t key = arc_key(sv, dv, a.nv);
                    if (key == ~0ull) {
                        dropped++;
                        if (sv >= a.nv || dv >= a.nv)
                            atomicMin(&a.scratch[0], (unsigned long long)i);
                    }
                    atomicAdd(&h[(uint32_t)(key >> shift) & mask], 1u);
                }
            }
        }
        for (int o = 16; o; o >>= 1) dropped += __shfl_xor_sync(0xffffffffu, dropped, o);
        if ((threadIdx.x & 31) == 0 && dropped) atomicAdd(&a.scratch[1], dropped);
    } else if (base + kRsTile <= n) {
        // full tile: all 16 keys in flight as 8 x 16-byte loads, then count
        const ulonglong2 *k2 = reinterpret_cast<const ulonglong2 *>(keys + base);
        ulonglong2 v[kRsItems / 2];
#pragma unroll
        for (int k = 0; k < kRsItems / 2; k++) v[k] = __ldcs(k2 + k * kRsThreads + threadIdx.x);
#pragma unroll
        for (int k = 0; k < kRsItems / 2; k++) {
            atomicAdd(&h[(uint32_t)(v[k].x >> shift) & mask], 1u);
            atomicAdd(&h[(uint32_t)(v[k].y >> shift) & mask], 1u);
        }
    } else {
#pragma unroll 4
        for (int k = 0; k < kRsItems; k++) {
            size_t i = base + (size_t)k * kRsThreads + threadIdx.x;
            if (i < n) atomicAdd(&h[(uint32_t)(__ldg(keys + i) >> shift) & mask], 1u);
        }
    }
    __syncthreads();
    for (int d = threadIdx.x; d < radix; d += kRsThreads) hist[(size_t)d * ntiles + blockIdx.x] = h[d];
}

// Digit-major histogram -> per-digit exclusive prefix over tiles, in place
// (one block per digit, chunks of 4096 tiles with a running carry), and the
// digit totals; the downsweep adds the exclusive prefix of the totals.  One
// launch per pass instead of a device-wide reduce-then-scan pair.
__global__ void __launch_bounds__(256) rs_scan_digits(uint32_t *__restrict__ hist, size_t ntiles,
                                                      uint32_t *__restrict__ totals) {
    uint32_t *row = hist + (size_t)blockIdx.x * ntiles;
    uint32_t carry = 0;
    for (size_t base = 0; base < ntiles; base += 256 * 16) {
        uint32_t v[16], sum = 0;
#pragma unroll
        for (int k = 0; k < 16; k++) {
            const size_t i = base + (size_t)threadIdx.x * 16 + k;
            v[k] = i < ntiles ? row[i] : 0u;
            sum += v[k];
        }
        uint32_t all;
        uint32_t run = block_exclusive_sum<uint32_t, 256>(sum, &all) + carry;
#pragma unroll
        for (int k = 0; k < 16; k++) {
            const size_t i = base + (size_t)threadIdx.x * 16 + k;
            if (i < ntiles) row[i] = run;
            run += v[k];
        }
        carry += all;
    }
    if (threadIdx.x == 0) totals[blockIdx.x] = carry;
}

struct DownSmem {
    uint32_t klo[kRsTile], khi[kRsTile];     // tile reordered by digit (split halves:
                                             // 4-byte banks, fewer store conflicts)
    uint16_t wc[kDsWarps][kMaxRadix];        // per-warp digit counts, then offsets
    uint32_t gbase[kMaxRadix];               // global offset - local offset per digit
};

// the tile's keys of this warp (warp-striped: iteration k holds keys wbase +
// 32 k + lane) and their stable ranks among the warp's keys of equal digit:
// one ballot per digit bit groups the lanes holding the same digit, the
// earlier peers plus the running per-warp count give the rank
template <int BITS, bool ARCS, bool FULL>
__device__ __forceinline__ void ds_load_rank(const uint64_t *__restrict__ keys, size_t n, int shift,
                                             uint32_t mask, const ArcSource &a, size_t wbase,
                                             uint16_t *wc, uint64_t (&key)[kDsItems],
                                             uint32_t (&rank2)[kDsItems / 2]) {
    const int lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;
    // all 16 loads in flight before the first use (the ranking chain below
    // is serial per warp)
#pragma unroll
    for (int k = 0; k < kDsItems; k++) {
        const size_t i = wbase + (size_t)k * 32 + lane;
        const bool valid = FULL || i < n;
        if (ARCS) key[k] = valid ? arc_key(__ldcs(a.src + i), __ldcs(a.dst + i), a.nv) : 0ull;
        else key[k] = valid ? __ldcs(keys + i) : 0ull;
    }
#pragma unroll
    for (int k = 0; k < kDsItems; k++) {
        const size_t i = wbase + (size_t)k * 32 + lane;
        const bool valid = FULL || i < n;
        const uint32_t d = valid ? ((uint32_t)(key[k] >> shift) & mask) : 0x10000u;
        // lanes holding the same digit: intersect one ballot per digit bit
        // (cheaper than __match_any_sync on sm_100)
        uint32_t peers = FULL ? 0xffffffffu : __ballot_sync(0xffffffffu, valid);
        peers &= warp_peers<BITS>(d);   // only the digit's own bits
        uint32_t r = 0;
        if (valid) r = wc[d] + __popc(peers & lt);
        __syncwarp();
        if (valid && (peers & lt) == 0) wc[d] += __popc(peers);
        __syncwarp();
        if (k & 1) rank2[k >> 1] |= r << 16;
        else rank2[k >> 1] = r;
    }
}

template <int BITS, bool ARCS>
__global__ void __launch_bounds__(kDsThreads, TC_DS_MINB)
rs_downsweep(const uint64_t *__restrict__ keys, uint64_t *__restrict__ out, size_t n, int shift,
             uint32_t mask, int radix, const uint32_t *__restrict__ offs, size_t ntiles,
             const uint32_t *__restrict__ totals, ArcSource a, const uint32_t *dn) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    if (dn) {
        n = min(n, (size_t)*dn);
        if ((size_t)blockIdx.x * kRsTile >= n) return;   // block-uniform
    }
    DownSmem &S = *reinterpret_cast<DownSmem *>(smem_raw);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kDsWarps * radix; i += kDsThreads) S.wc[i / radix][i % radix] = 0;
    __syncthreads();
    const size_t tile0 = (size_t)blockIdx.x * kRsTile;
    const size_t wbase = tile0 + (size_t)warp * 32 * kDsItems;
    uint64_t key[kDsItems];
    uint32_t rank2[kDsItems / 2];      // two 16-bit ranks per register
    // every tile but the last is full: no per-key bounds checks or validity
    // ballot there
    if (tile0 + kRsTile <= n)
        ds_load_rank<BITS, ARCS, true>(keys, n, shift, mask, a, wbase, S.wc[warp], key, rank2);
    else
        ds_load_rank<BITS, ARCS, false>(keys, n, shift, mask, a, wbase, S.wc[warp], key, rank2);
    __syncthreads();
    // tile-local digit offsets: exclusive scan over digits of the digit totals
    // (each thread owns radix/256 consecutive digits), then per-warp offsets
    {
        const int per = (radix + kDsThreads - 1) / kDsThreads;
        const int d0 = threadIdx.x * per;
        uint32_t tot = 0;
        for (int d = d0; d < d0 + per && d < radix; d++)
            for (int w = 0; w < kDsWarps; w++) tot += S.wc[w][d];
        uint32_t gt = 0;   // keys of the digits before mine, all tiles
        for (int d = d0; d < d0 + per && d < radix; d++) gt += __ldg(totals + d);
        uint32_t all;
        uint32_t run = block_exclusive_sum<uint32_t, kDsThreads>(tot, &all);
        uint32_t grun = block_exclusive_sum<uint32_t, kDsThreads>(gt, &all);
        for (int d = d0; d < d0 + per && d < radix; d++) {
            S.gbase[d] = grun + offs[(size_t)d * ntiles + blockIdx.x] - run;
            grun += __ldg(totals + d);
            for (int w = 0; w < kDsWarps; w++) {
                uint32_t c = S.wc[w][d];
                S.wc[w][d] = (uint16_t)run;
                run += c;
            }
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kDsItems; k++) {
        size_t i = wbase + (size_t)k * 32 + lane;
        if (i < n) {
            uint32_t d = (uint32_t)(key[k] >> shift) & mask;
            const uint32_t pos = S.wc[warp][d] + ((rank2[k >> 1] >> (16 * (k & 1))) & 0xffffu);
            S.klo[pos] = (uint32_t)key[k];
            S.khi[pos] = (uint32_t)(key[k] >> 32);
        }
    }
    __syncthreads();
    const uint32_t cnt = (uint32_t)min((size_t)kRsTile, n - tile0);
    for (uint32_t i = threadIdx.x; i < cnt; i += kDsThreads) {
        uint64_t k = ((uint64_t)S.khi[i] << 32) | S.klo[i];
        uint32_t d = (uint32_t)(k >> shift) & mask;
        out[S.gbase[d] + i] = k;
    }
}

typedef void (*DownFn)(const uint64_t *, uint64_t *, size_t, int, uint32_t, int, const uint32_t *,
                       size_t, const uint32_t *, ArcSource, const uint32_t *);
#define TC_DS(A) {nullptr, rs_downsweep<1, A>, rs_downsweep<2, A>, rs_downsweep<3, A>,       \
                  rs_downsweep<4, A>, rs_downsweep<5, A>, rs_downsweep<6, A>,            \
                  rs_downsweep<7, A>, rs_downsweep<8, A>}

}  // namespace

tc_status radix_sort_u64(Mem &mem, uint64_t *keys, uint64_t *tmp, size_t n,
                         const RadixPass *passes, int npasses, cudaStream_t s,
                         uint64_t *launches, uint64_t **sorted, const ArcSource *arcs,
                         const uint32_t *dn) {
    *sorted = keys;
    if (n <= 1 || npasses == 0) return TC_OK;
    if (n >= (1ull << 32)) {
        set_error("radix sort: %zu keys exceed the 32-bit offset range", n);
        return TC_E_INVALID;
    }
    if (arcs && npasses == 0) {
        set_error("radix sort: an arc source needs at least one pass");
        return TC_E_INVALID;
    }
    static const DownFn kDown[2][kMaxBits + 1] = {TC_DS(false), TC_DS(true)};
    // the shared-memory opt-in of the 16 downsweep instances, once per device
    // (driver calls on every sort cost host time on the build's critical path)
    static std::atomic<uint64_t> attr_done{0};
    int dev = 0;
    TC_CUDA(cudaGetDevice(&dev));
    const uint64_t bit = 1ull << (dev & 63);
    if (!(attr_done.load() & bit)) {
        for (int a = 0; a < 2; a++)
            for (int b = 1; b <= kMaxBits; b++)
                TC_CUDA(cudaFuncSetAttribute(kDown[a][b],
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)sizeof(DownSmem)));
        attr_done.fetch_or(bit);
    }
    const ArcSource none{nullptr, nullptr, 0, nullptr};
    size_t ntiles = (n + kRsTile - 1) / kRsTile;
    int maxbits = 1;
    for (int p = 0; p < npasses; p++) maxbits = passes[p].bits > maxbits ? passes[p].bits : maxbits;
    DevBuf<uint32_t> hist, totals;
    tc_status st = hist.allocate(mem, ntiles << maxbits);
    if (st != TC_OK) return st;
    if ((st = totals.allocate(mem, (size_t)1 << maxbits)) != TC_OK) return st;
    uint64_t *src = keys, *dst = tmp;
    for (int p = 0; p < npasses; p++) {
        int bits = passes[p].bits;
        if (bits < 1 || bits > kMaxBits) {
            set_error("radix sort: digit width %d out of [1,%d]", bits, kMaxBits);
            return TC_E_INVALID;
        }
        int radix = 1 << bits;
        uint32_t mask = (uint32_t)radix - 1u;
        const bool from_arcs = arcs && p == 0;
        if (from_arcs)
            rs_upsweep<true><<<(unsigned)ntiles, kRsThreads, 0, s>>>(
                src, n, passes[p].shift, mask, radix, hist.p, ntiles, *arcs, dn);
        else
            rs_upsweep<false><<<(unsigned)ntiles, kRsThreads, 0, s>>>(
                src, n, passes[p].shift, mask, radix, hist.p, ntiles, none, dn);
        TC_CUDA(cudaGetLastError());
        rs_scan_digits<<<(unsigned)radix, 256, 0, s>>>(hist.p, ntiles, totals.p);
        TC_CUDA(cudaGetLastError());
        kDown[from_arcs][bits]<<<(unsigned)ntiles, kDsThreads, sizeof(DownSmem), s>>>(
            src, dst, n, passes[p].shift, mask, radix, hist.p, ntiles, totals.p,
            from_arcs ? *arcs : none, dn);
        TC_CUDA(cudaGetLastError());
        if (launches) *launches += 3;
        uint64_t *t = src;
        src = dst;
        dst = t;
    }
    *sorted = src;
    return TC_OK;
}

// passes covering bits [lo, lo + width) with digits of at most 11 bits
int radix_passes_for(int lo, int width, RadixPass *out) {
    if (width <= 0) return 0;
    int np = (width + kMaxBits - 1) / kMaxBits;
    int per = (width + np - 1) / np;
    int done = 0, k = 0;
    while (done < width) {
        int b = per < width - done ? per : width - done;
        out[k].shift = lo + done;
        out[k].bits = b;
        done += b;
        k++;
    }
    return k;
}

}  // namespace tc
