// csr_build.cu -- a1: GPU CSR builder.
//
// From an arc list it builds ONE symmetric neighbour CSR over N(u) (the
// paper's "array of neighbour lists" N, stored as the adjacency array
// of P:458-469) where every entry carries the 2-bit direction code, so the
// census never probes IsEdge / IsNeighbour -- the tags answer them.
//
//   1. emit      arc (s,d), s != d  ->  keys (s<<32 | d<<2 | 1) and
//                (d<<32 | s<<2 | 2); self-loops -> all-ones sentinel keys
//                that sort last (strict digraph); range check.
//   2. sort      LSD radix sort on the column bits then the row bits.
//   3. scan      head = first key of a (row, col) run; one fused exclusive
//                scan counts heads (entry index r) and canonical heads
//                row < col (dyad index k, canonical order P:277-281) and its
//                output pass ORs the run's tags (dedup, mutual merge),
//                writes adj[r] = col<<2 | tag, the dyad list, and the row
//                offsets at row boundaries.
//   4. stats     m, mutual dyads, sum d^2, max degree.
#include <stdio.h>

#include "radix_sort.cuh"
#include "scan.cuh"

namespace tc {

namespace {

constexpr uint64_t kSentinel = ~0ull;

__global__ void k_emit(const uint32_t *__restrict__ src, const uint32_t *__restrict__ dst,
                       uint64_t m, uint64_t n, uint64_t *__restrict__ keys,
                       unsigned long long *__restrict__ scratch /* [0]=bad, [1]=loops */) {
    unsigned long long loops = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t s = src[i], d = dst[i];
        if (s >= n || d >= n) {
            atomicMin(&scratch[0], (unsigned long long)i);
            keys[2 * i] = kSentinel;
            keys[2 * i + 1] = kSentinel;
            continue;
        }
        if (s == d) {
            loops++;
            keys[2 * i] = kSentinel;
            keys[2 * i + 1] = kSentinel;
        } else {
            keys[2 * i] = ((uint64_t)s << 32) | ((uint64_t)d << 2) | 1ull;
            keys[2 * i + 1] = ((uint64_t)d << 32) | ((uint64_t)s << 2) | 2ull;
        }
    }
    // warp-aggregated loop count
    for (int o = 16; o; o >>= 1) loops += __shfl_xor_sync(0xffffffffu, loops, o);
    if ((threadIdx.x & 31) == 0 && loops) atomicAdd(&scratch[1], loops);
}

struct HeadIn {
    const uint64_t *key;
    __device__ __forceinline__ uint64_t operator()(size_t i) const {
        uint64_t k = key[i];
        bool head = (i == 0) || ((key[i - 1] >> 2) != (k >> 2));
        bool canon = head && ((uint32_t)(k >> 32) < (uint32_t)((k >> 2) & 0x3fffffffu));
        return (uint64_t)head | ((uint64_t)canon << 32);
    }
};

struct HeadOut {
    const uint64_t *key;
    size_t L;
    uint32_t *adj, *du, *dp, *off;
    __device__ __forceinline__ void operator()(size_t i, uint64_t excl, uint64_t v) const {
        if (!(v & 1ull)) return;
        uint32_t r = (uint32_t)excl, k = (uint32_t)(excl >> 32);
        uint64_t kk = key[i];
        uint32_t row = (uint32_t)(kk >> 32);
        uint32_t col = (uint32_t)((kk >> 2) & 0x3fffffffu);
        uint32_t tag = (uint32_t)(kk & 3u);
        for (size_t j = i + 1; j < L && (key[j] >> 2) == (kk >> 2); j++) tag |= (uint32_t)(key[j] & 3u);
        adj[r] = (col << 2) | tag;
        if (v >> 32) {
            du[k] = row;
            dp[k] = r;
        }
        // first entry of row `row`: rows (prev_row, row] start at r
        uint32_t first = 0;
        bool boundary = (i == 0);
        if (!boundary) {
            uint32_t prev = (uint32_t)(key[i - 1] >> 32);
            if (prev != row) {
                boundary = true;
                first = prev + 1;
            }
        }
        if (boundary)
            for (uint32_t x = first; x <= row; x++) off[x] = r;
    }
};

__global__ void k_fill_tail(uint32_t *off, uint64_t from, uint64_t n, uint32_t val) {
    for (uint64_t x = from + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x <= n;
         x += (uint64_t)gridDim.x * blockDim.x)
        off[x] = val;
}

__device__ __forceinline__ unsigned long long warp_sum64(unsigned long long x) {
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

// [0] = sum d^2, [1] = max d
__global__ void k_vertex_stats(const uint32_t *__restrict__ off, uint64_t n,
                               unsigned long long *out) {
    unsigned long long s2 = 0, mx = 0;
    for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n;
         u += (uint64_t)gridDim.x * blockDim.x) {
        unsigned long long d = off[u + 1] - off[u];
        s2 += d * d;
        mx = d > mx ? d : mx;
    }
    s2 = warp_sum64(s2);
    for (int o = 16; o; o >>= 1) {
        unsigned long long y = __shfl_xor_sync(0xffffffffu, mx, o);
        mx = y > mx ? y : mx;
    }
    if ((threadIdx.x & 31) == 0) {
        if (s2) atomicAdd(&out[0], s2);
        atomicMax(&out[1], mx);
    }
}

// [2] = distinct arcs m, [3] = mutual dyads
__global__ void k_dyad_stats(const uint32_t *__restrict__ adj, const uint32_t *__restrict__ dp,
                             uint64_t D, unsigned long long *out) {
    unsigned long long m = 0, mu = 0;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < D;
         k += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t t = adj[dp[k]] & 3u;
        m += __popc(t);
        mu += (t == 3u);
    }
    m = warp_sum64(m);
    mu = warp_sum64(mu);
    if ((threadIdx.x & 31) == 0) {
        if (m) atomicAdd(&out[2], m);
        if (mu) atomicAdd(&out[3], mu);
    }
}

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

    size_t L0 = 2 * (size_t)m;
    DevBuf<uint64_t> keys, tmp;
    if ((st = keys.allocate(mem, L0)) != TC_OK) return st;
    if ((st = tmp.allocate(mem, L0)) != TC_OK) return st;

    if (m) {
        k_emit<<<grid_for(m, 256), 256, 0, s>>>(d_src, d_dst, m, n, keys.p, scratch.p);
        g->launches++;
        TC_CUDA(cudaGetLastError());
    }
    unsigned long long h[8];
    TC_CUDA(cudaMemcpyAsync(h, scratch.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    if (h[0] != ~0ull) {
        set_error("arc %llu has an endpoint >= n (n = %llu)", h[0], (unsigned long long)n);
        return TC_E_RANGE;
    }
    const uint64_t loops = h[1];
    const size_t L = L0 - 2 * loops;

    // 2. sort by (row, col): column bits first, then row bits
    int b = 1;
    while (b < 32 && (1ull << b) < n) b++;
    RadixPass passes[16];
    int np = radix_passes_for(2, b, passes);
    np += radix_passes_for(32, b, passes + np);
    uint64_t *sorted = keys.p;
    if ((st = radix_sort_u64(mem, keys.p, tmp.p, L0, passes, np, s, &g->launches, &sorted)) !=
        TC_OK)
        return st;

    // 3. fused head scan -> adj, dyad list, offsets
    size_t cap = L ? L : 1;
    uint32_t *adj = (uint32_t *)mem.alloc(cap * sizeof(uint32_t));
    uint32_t *du = (uint32_t *)mem.alloc((cap / 2 + 1) * sizeof(uint32_t));
    uint32_t *dp = (uint32_t *)mem.alloc((cap / 2 + 1) * sizeof(uint32_t));
    uint32_t *off = (uint32_t *)mem.alloc((n + 1) * sizeof(uint32_t));
    g->adj = adj; g->adj_n = cap;
    g->dyad_u = du; g->dyad_n = cap / 2 + 1;
    g->dyad_p = dp;
    g->off = off; g->off_n = n + 1;
    if (!adj || !du || !dp || !off) {
        set_error("device allocation for the CSR failed");
        return TC_E_OOM;
    }
    DevBuf<uint64_t> total;
    if ((st = total.allocate(mem, 1)) != TC_OK) return st;
    st = scan_exclusive<uint64_t>(mem, L, HeadIn{sorted}, HeadOut{sorted, L, adj, du, dp, off},
                                  total.p, s, &g->launches);
    if (st != TC_OK) return st;
    uint64_t tot = 0, lastkey = 0;
    TC_CUDA(cudaMemcpyAsync(&tot, total.p, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    if (L) TC_CUDA(cudaMemcpyAsync(&lastkey, sorted + (L - 1), sizeof(uint64_t),
                                   cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    const uint64_t nnz = tot & 0xffffffffull, D = tot >> 32;
    uint64_t from = L ? ((lastkey >> 32) + 1) : 0;
    k_fill_tail<<<grid_for(n + 1 - from, 256), 256, 0, s>>>(off, from, n, (uint32_t)nnz);
    g->launches++;
    TC_CUDA(cudaGetLastError());

    // 4. stats
    k_vertex_stats<<<grid_for(n, 256), 256, 0, s>>>(off, n, scratch.p + 4);
    if (D) k_dyad_stats<<<grid_for(D, 256), 256, 0, s>>>(adj, dp, D, scratch.p + 4);
    g->launches += D ? 2 : 1;
    TC_CUDA(cudaGetLastError());
    TC_CUDA(cudaMemcpyAsync(h, scratch.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    g->st.m_in = m;
    g->st.loops_dropped = loops;
    g->st.dyads = D;
    g->st.sum_deg_sq = h[4];
    g->st.max_degree = h[5];
    g->st.m = h[6];
    g->st.mutual_dyads = h[7];
    g->st.dups_dropped = m - loops - h[6];
    if (nnz != 2 * D) {
        set_error("internal: CSR has %llu entries for %llu dyads", (unsigned long long)nnz,
                  (unsigned long long)D);
        return TC_E_CUDA;
    }
    return TC_OK;
}

}  // namespace tc
