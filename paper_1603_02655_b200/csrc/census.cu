// census.cu -- a3 (merge/classify) and a4 (histogram reduction) kernels.
//
// For a canonical dyad (u, v), u < v, with pre = tag of v in N(u)
// (= IsEdge(u,v) + 2*IsEdge(v,u), the v0.4 pre-computed code),
// the B-M loop body (Fig. P:269-309) is evaluated as one sorted merge of the
// tagged rows A = N(u) and B = N(v):
//   * every merged id w is an element of N(u) U N(v); tu / tv are its tags in
//     A / B (0 if absent), which are exactly IsEdge(u,w)+2*IsEdge(w,u) and
//     IsEdge(v,w)+2*IsEdge(w,v) of Fig. TriadCode;
//   * line 16's predicate  v < w or (u < w < v and not IsNeighbour(u,w))
//     becomes  (w > v) | (tu == 0 & w > u), which also rejects w = u (tu = 0,
//     w = u) and w = v (w = v not > v, tu != 0);
//   * code = pre | tu<<2 | tv<<4 (bit weights 1,2,4,8,16,32 of P:329-347) and
//     class = TriadTable[code], the 64-entry table held in shared
//     memory (16 banks, no conflicts: all 64 entries share 16 words);
//   * the dyadic term n - |S| - 2 of line 14, with |S| = |N(u)|+|N(v)|-I-2
//     (I = |N(u) & N(v)|), is accumulated as (n - du - dv) once per dyad plus
//     one per intersection element, into class 3 (pre == 3, mutual) or 2.
// The merge is split along merge-path diagonals so any number of threads can
// share one dyad: a segment [d0, d1) starts at the merge-path split of d0
// (ties go to A first; an equal pair is consumed together, so a segment that
// starts right after a pair's A element skips the B element).
//
// a4: per-thread 8-bit packed class counters (two uint64 registers, flushed
// before they can overflow) -> per-block shared uint64[16] -> one global
// atomicAdd per class per block.
#include "census.cuh"

namespace tc {

// TriadTable, 0-based classes in the paper's order 003..300.
// Literal B-M 2001 TRICODES table minus one (reading 1); the
// oracle derives its own table by orbit enumeration and the tests compare.
__constant__ uint8_t c_triad_table[64] = {
    0, 1, 1, 2, 1, 3, 5, 7, 1, 5, 4, 6, 2, 7, 6, 10, 1, 5, 3, 7, 4, 8, 8, 12, 5, 9, 8, 13, 6, 13, 11, 14,
    1, 4, 5, 6, 5, 8, 9, 13, 3, 8, 8, 11, 7, 12, 13, 14, 2, 6, 7, 10, 6, 11, 13, 14, 7, 13, 12, 14, 10, 14, 14, 15};

namespace {

struct Acc {
    uint64_t lo, hi;      // 8-bit counters: classes 0..7 | 8..15 (0-based)
    uint32_t pending;     // upper bound on increments since the last flush
    uint64_t dy012, dy102;  // dyadic triads of classes 012 / 102
};

__device__ __forceinline__ void add_dyadic(Acc &c, uint32_t pre, uint64_t x) {
    if (pre == 3u) c.dy102 += x;
    else c.dy012 += x;
}

__device__ __forceinline__ void acc_init(Acc &c) {
    c.lo = c.hi = 0;
    c.pending = 0;
    c.dy012 = c.dy102 = 0;
}

__device__ __forceinline__ void acc_flush(Acc &c, unsigned long long *sh) {
#pragma unroll
    for (int b = 0; b < 8; b++) {
        uint32_t x = (uint32_t)(c.lo >> (8 * b)) & 255u;
        if (x) atomicAdd(&sh[b], (unsigned long long)x);
    }
#pragma unroll
    for (int b = 0; b < 8; b++) {
        uint32_t x = (uint32_t)(c.hi >> (8 * b)) & 255u;
        if (x) atomicAdd(&sh[8 + b], (unsigned long long)x);
    }
    c.lo = c.hi = 0;
    c.pending = 0;
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

// classify the merged elements on diagonals [d0, d1) of dyad (u, v)
__device__ __forceinline__ void merge_segment(const uint32_t *__restrict__ A, uint32_t a,
                                              const uint32_t *__restrict__ B, uint32_t b,
                                              uint32_t u, uint32_t v, uint32_t pre, uint32_t d0,
                                              uint32_t d1, const uint8_t *__restrict__ tab,
                                              Acc &c, unsigned long long *sh) {
    uint32_t i = 0, j = 0;
    if (d0 > 0) {
        i = merge_path(A, a, B, b, d0);
        j = d0 - i;
        // the pair (A[i-1], B[j]) was consumed by the previous segment
        if (i > 0 && j < b && (__ldg(A + i - 1) | 3u) == (__ldg(B + j) | 3u)) j++;
    }
    if (c.pending + (d1 - d0) > 255u) acc_flush(c, sh);
    c.pending += d1 - d0;
    uint32_t I = 0;
    while (i + j < d1) {
        uint32_t x = i < a ? __ldg(A + i) : 0xffffffffu;
        uint32_t y = j < b ? __ldg(B + j) : 0xffffffffu;
        uint32_t kx = x | 3u, ky = y | 3u;
        uint32_t ta = kx <= ky, tb = ky <= kx;
        uint32_t w = (ta ? x : y) >> 2;
        uint32_t tu = ta ? (x & 3u) : 0u;
        uint32_t tv = tb ? (y & 3u) : 0u;
        i += ta;
        j += tb;
        I += ta & tb;
        uint32_t canon = (w > v) | ((tu == 0u) & (w > u));
        uint32_t cls = tab[pre | (tu << 2) | (tv << 4)];
        uint64_t inc = (uint64_t)canon << ((cls & 7u) * 8u);
        if (cls & 8u) c.hi += inc;
        else c.lo += inc;
    }
    add_dyadic(c, pre, I);
}

__device__ __forceinline__ void block_setup(uint8_t *tab, unsigned long long *sh) {
    if (threadIdx.x < 64) tab[threadIdx.x] = c_triad_table[threadIdx.x];
    if (threadIdx.x < 16) sh[threadIdx.x] = 0;
    __syncthreads();
}

__device__ __forceinline__ void block_finish(Acc &c, unsigned long long *sh,
                                             unsigned long long *d_counts) {
    acc_flush(c, sh);
    // dyadic terms: warp reduce then shared atomics
    unsigned long long d0 = c.dy012, d1 = c.dy102;
    for (int o = 16; o; o >>= 1) {
        d0 += __shfl_xor_sync(0xffffffffu, d0, o);
        d1 += __shfl_xor_sync(0xffffffffu, d1, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&sh[1], d0);
        atomicAdd(&sh[2], d1);
    }
    __syncthreads();
    if (threadIdx.x >= 1 && threadIdx.x < 16 && sh[threadIdx.x])
        atomicAdd(&d_counts[threadIdx.x], sh[threadIdx.x]);
}

__global__ void __launch_bounds__(256)
k_census_thread(const BinItem2 *__restrict__ items, uint64_t count,
                const uint32_t *__restrict__ off, const uint32_t *__restrict__ adj, uint64_t n,
                unsigned long long *d_counts) {
    __shared__ uint8_t tab[64];
    __shared__ unsigned long long sh[16];
    block_setup(tab, sh);
    Acc c;
    acc_init(c);
    for (uint64_t it = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; it < count;
         it += (uint64_t)gridDim.x * blockDim.x) {
        BinItem2 e = items[it];
        uint32_t ev = __ldg(adj + e.p);
        uint32_t v = ev >> 2, pre = ev & 3u;
        uint32_t ou = __ldg(off + e.u), a = __ldg(off + e.u + 1) - ou;
        uint32_t ov = __ldg(off + v), b = __ldg(off + v + 1) - ov;
        add_dyadic(c, pre, n - a - b);
        merge_segment(adj + ou, a, adj + ov, b, e.u, v, pre, 0, a + b, tab, c, sh);
    }
    block_finish(c, sh, d_counts);
}

__global__ void __launch_bounds__(256)
k_census_warp(const BinItem2 *__restrict__ items, uint64_t count,
              const uint32_t *__restrict__ off, const uint32_t *__restrict__ adj, uint64_t n,
              unsigned long long *d_counts) {
    __shared__ uint8_t tab[64];
    __shared__ unsigned long long sh[16];
    block_setup(tab, sh);
    Acc c;
    acc_init(c);
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t wid = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t it = wid; it < count; it += nw) {
        BinItem2 e = items[it];
        uint32_t ev = __ldg(adj + e.p);
        uint32_t v = ev >> 2, pre = ev & 3u;
        uint32_t ou = __ldg(off + e.u), a = __ldg(off + e.u + 1) - ou;
        uint32_t ov = __ldg(off + v), b = __ldg(off + v + 1) - ov;
        uint32_t cst = a + b, per = (cst + 31) >> 5;
        uint32_t d0 = lane * per, d1 = min(cst, d0 + per);
        if (lane == 0) add_dyadic(c, pre, n - a - b);
        if (d0 < d1) merge_segment(adj + ou, a, adj + ov, b, e.u, v, pre, d0, d1, tab, c, sh);
    }
    block_finish(c, sh, d_counts);
}

__global__ void __launch_bounds__(kBlockThreads)
k_census_block(const BinItem4 *__restrict__ items, uint64_t count,
               const uint32_t *__restrict__ off, const uint32_t *__restrict__ adj, uint64_t n,
               unsigned long long *d_counts) {
    __shared__ uint8_t tab[64];
    __shared__ unsigned long long sh[16];
    block_setup(tab, sh);
    Acc c;
    acc_init(c);
    for (uint64_t it = blockIdx.x; it < count; it += gridDim.x) {
        BinItem4 e = items[it];
        uint32_t ev = __ldg(adj + e.p);
        uint32_t v = ev >> 2, pre = ev & 3u;
        uint32_t ou = __ldg(off + e.u), a = __ldg(off + e.u + 1) - ou;
        uint32_t ov = __ldg(off + v), b = __ldg(off + v + 1) - ov;
        uint32_t span = e.d1 - e.d0, per = (span + kBlockThreads - 1) / kBlockThreads;
        uint32_t d0 = e.d0 + threadIdx.x * per, d1 = min(e.d1, d0 + per);
        if (e.d0 == 0 && threadIdx.x == 0) add_dyadic(c, pre, n - a - b);
        if (d0 < d1) merge_segment(adj + ou, a, adj + ov, b, e.u, v, pre, d0, d1, tab, c, sh);
    }
    block_finish(c, sh, d_counts);
}

inline unsigned grid_cap(uint64_t blocks, unsigned cap) {
    if (blocks < 1) blocks = 1;
    return (unsigned)(blocks < cap ? blocks : cap);
}

}  // namespace

tc_status launch_bins(const tc_graph *g, const BinLists &bl, cudaStream_t s, uint64_t *d_counts,
                      tc_profile *prof, uint64_t *launches) {
    const uint64_t n = g->st.n;
    unsigned long long *out = reinterpret_cast<unsigned long long *>(d_counts);
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    if (prof) {
        for (int i = 0; i < 4; i++) TC_CUDA(cudaEventCreate(&ev[i]));
        TC_CUDA(cudaEventRecord(ev[0], s));
    }
    const unsigned sms = 148;
    if (bl.count[0]) {
        k_census_thread<<<grid_cap((bl.count[0] + 255) / 256, sms * 8), 256, 0, s>>>(
            bl.t, bl.count[0], g->off, g->adj, n, out);
        TC_CUDA(cudaGetLastError());
        *launches += 1;
    }
    if (prof) TC_CUDA(cudaEventRecord(ev[1], s));
    if (bl.count[1]) {
        k_census_warp<<<grid_cap((bl.count[1] + 7) / 8, sms * 8), 256, 0, s>>>(
            bl.w, bl.count[1], g->off, g->adj, n, out);
        TC_CUDA(cudaGetLastError());
        *launches += 1;
    }
    if (prof) TC_CUDA(cudaEventRecord(ev[2], s));
    if (bl.count[2]) {
        k_census_block<<<grid_cap(bl.count[2], sms * 8), kBlockThreads, 0, s>>>(
            bl.b, bl.count[2], g->off, g->adj, n, out);
        TC_CUDA(cudaGetLastError());
        *launches += 1;
    }
    if (prof) {
        TC_CUDA(cudaEventRecord(ev[3], s));
        TC_CUDA(cudaEventSynchronize(ev[3]));
        float t;
        for (int i = 0; i < 3; i++) {
            TC_CUDA(cudaEventElapsedTime(&t, ev[i], ev[i + 1]));
            prof->kernel_ms[i] = t;
        }
        TC_CUDA(cudaEventElapsedTime(&t, ev[0], ev[3]));
        prof->census_ms = t;
        for (int i = 0; i < 4; i++) cudaEventDestroy(ev[i]);
    }
    return TC_OK;
}

}  // namespace tc
