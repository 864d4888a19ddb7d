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
//   3. compact   head = first key of a (row, col) run.  A ballot/popc
//                compaction (count pass, scan of tile counts, write pass)
//                numbers the heads (entry index r) and the canonical heads
//                row < col (dyad index k, canonical order P:277-281); each
//                head ORs its run's tags (dedup, mutual merge) and writes
//                adj[r + row] = col<<2 | tag, the dyad list and, at row
//                boundaries, the row offsets.  Every row ends with one
//                sentinel entry 0xffffffff (greater than any real entry), so
//                the census merge runs off a row end without bounds checks:
//                row u = adj[off[u], off[u+1] - 1), |N(u)| = off[u+1]-off[u]-1.
//   4. stats     m, mutual dyads, sum d^2, max degree, per-dyad cost.
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
                       unsigned long long *__restrict__ scratch /* [0]=bad, [1]=loops */) {
    unsigned long long loops = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t s = src[i], d = dst[i];
        ulonglong2 kv;
        if (s >= n || d >= n) {
            atomicMin(&scratch[0], (unsigned long long)i);
            kv = make_ulonglong2(kSentinel, kSentinel);
        } else if (s == d) {
            loops++;
            kv = make_ulonglong2(kSentinel, kSentinel);
        } else {
            kv = make_ulonglong2(((uint64_t)s << 32) | ((uint64_t)d << 2) | 1ull,
                                 ((uint64_t)d << 32) | ((uint64_t)s << 2) | 2ull);
        }
        reinterpret_cast<ulonglong2 *>(keys)[i] = kv;
    }
    for (int o = 16; o; o >>= 1) loops += __shfl_xor_sync(0xffffffffu, loops, o);
    if ((threadIdx.x & 31) == 0 && loops) atomicAdd(&scratch[1], loops);
}

// (row, col) of a sorted key; heads: first key of each (row, col) run
__device__ __forceinline__ uint32_t key_row(uint64_t k) { return (uint32_t)(k >> 32); }
__device__ __forceinline__ uint32_t key_col(uint64_t k) { return (uint32_t)((k >> 2) & 0x3fffffffu); }

// flags of key i (warp-striped: lanes hold consecutive keys)
__device__ __forceinline__ void head_flags(const uint64_t *__restrict__ key, size_t L, size_t i,
                                           uint64_t &k, uint64_t &prev, bool &head, bool &canon) {
    const uint32_t lane = threadIdx.x & 31;
    k = i < L ? __ldg(key + i) : kSentinel;
    prev = __shfl_up_sync(0xffffffffu, k, 1);
    if (lane == 0) prev = (i > 0 && i - 1 < L) ? __ldg(key + i - 1) : kSentinel;
    head = i < L && (i == 0 || (prev >> 2) != (k >> 2));
    canon = head && key_row(k) < key_col(k);
}

// pass 1: per warp (512 keys), number of heads | canonical heads << 32
__global__ void __launch_bounds__(kHcThreads)
k_head_count(const uint64_t *__restrict__ key, size_t L, uint64_t *__restrict__ warp_tot) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const size_t base = (size_t)blockIdx.x * kHcTile + (size_t)warp * 32 * kHcItems;
    uint32_t nh = 0, nc = 0;
#pragma unroll 4
    for (int r = 0; r < kHcItems; r++) {
        uint64_t k, prev;
        bool head, canon;
        head_flags(key, L, base + (size_t)r * 32 + lane, k, prev, head, canon);
        nh += __popc(__ballot_sync(0xffffffffu, head));
        nc += __popc(__ballot_sync(0xffffffffu, canon));
    }
    if (lane == 0) warp_tot[(size_t)blockIdx.x * kHcWarps + warp] = (uint64_t)nh | ((uint64_t)nc << 32);
}

// pass 2: write adj / dyad lists / row offsets at the compacted positions
// (warp_off = exclusive scan of pass 1's per-warp totals)
__global__ void __launch_bounds__(kHcThreads)
k_head_write(const uint64_t *__restrict__ key, size_t L, const uint64_t *__restrict__ warp_off,
             uint32_t *__restrict__ adj, uint32_t *__restrict__ du, uint32_t *__restrict__ de,
             uint32_t *__restrict__ off) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    const size_t base = (size_t)blockIdx.x * kHcTile + (size_t)warp * 32 * kHcItems;
    const uint64_t woff = warp_off[(size_t)blockIdx.x * kHcWarps + warp];
    uint32_t r0 = (uint32_t)woff, k0 = (uint32_t)(woff >> 32);
    for (int r = 0; r < kHcItems; r++) {
        const size_t i = base + (size_t)r * 32 + lane;
        uint64_t k, prev;
        bool head, canon;
        head_flags(key, L, i, k, prev, head, canon);
        const uint32_t bh = __ballot_sync(0xffffffffu, head);
        const uint32_t bc = __ballot_sync(0xffffffffu, canon);
        // next key (lane + 1, or a load for lane 31) for the run's tag OR
        uint64_t nxt = __shfl_down_sync(0xffffffffu, k, 1);
        if (lane == 31) nxt = i + 1 < L ? __ldg(key + i + 1) : kSentinel;
        if (head) {
            const uint32_t rr = r0 + __popc(bh & lt);
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
            const uint32_t e = (col << 2) | tag;
            adj[rr + row] = e;
            if (canon) {
                const uint32_t kk = k0 + __popc(bc & lt);
                du[kk] = row;
                de[kk] = e;
            }
            // first entry of row `row`: rows (prev_row, row] start here
            if (i == 0 || key_row(prev) != row) {
                off[row] = rr + row;
                const uint32_t first = i == 0 ? 0u : key_row(prev) + 1;
#pragma unroll 1
                for (uint32_t x = first; x < row; x++) off[x] = rr + x;   // empty rows
            }
        }
        r0 += __popc(bh);
        k0 += __popc(bc);
    }
}

__global__ void k_fill_tail(uint32_t *off, uint64_t from, uint64_t n, uint32_t nnz) {
    for (uint64_t x = from + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x <= n;
         x += (uint64_t)gridDim.x * blockDim.x)
        off[x] = nnz + (uint32_t)x;
}

// row terminators (and slack entries past the last row for look-ahead loads)
__global__ void k_sentinels(const uint32_t *__restrict__ off, uint64_t n, uint32_t *adj) {
    for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n + 8;
         x += (uint64_t)gridDim.x * blockDim.x)
        adj[x < n ? off[x + 1] - 1 : off[n] + (x - n)] = 0xffffffffu;
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
        unsigned long long d = off[u + 1] - off[u] - 1;
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

// per canonical dyad: cost c = |N(u)| + |N(v)| (uniform workload);
// stats [2] = distinct arcs m, [3] = mutual dyads
__global__ void k_dyad_cost_stats(const uint32_t *__restrict__ off,
                                  const uint32_t *__restrict__ du,
                                  const uint32_t *__restrict__ de, uint64_t D,
                                  uint32_t *__restrict__ dc, unsigned long long *out) {
    unsigned long long m = 0, mu = 0;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < D;
         k += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t u = du[k], e = de[k], v = e >> 2, t = e & 3u;
        dc[k] = (__ldg(off + u + 1) - __ldg(off + u)) + (__ldg(off + v + 1) - __ldg(off + v)) - 2;
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
    if ((st = scratch.allocate(mem, 16)) != TC_OK) return st;
    unsigned long long init[16] = {~0ull, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
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
    if ((uint64_t)L + n + 8 >= (1ull << 32)) {
        set_error("2D + n = %llu exceeds the 32-bit CSR offset range",
                  (unsigned long long)(L + n));
        return TC_E_INVALID;
    }

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

    // 3. compaction -> adj, dyad list, offsets
    size_t cap = L ? L : 1;
    uint32_t *adj = (uint32_t *)mem.alloc((L + n + 8) * sizeof(uint32_t));
    uint32_t *du = (uint32_t *)mem.alloc((cap / 2 + 1) * sizeof(uint32_t));
    uint32_t *de = (uint32_t *)mem.alloc((cap / 2 + 1) * sizeof(uint32_t));
    uint32_t *dc = (uint32_t *)mem.alloc((cap / 2 + 1) * sizeof(uint32_t));
    uint32_t *off = (uint32_t *)mem.alloc((n + 1) * sizeof(uint32_t));
    g->adj = adj; g->adj_n = L + n + 8;
    g->dyad_u = du; g->dyad_n = cap / 2 + 1;
    g->dyad_e = de;
    g->dyad_c = dc;
    g->off = off; g->off_n = n + 1;
    if (!adj || !du || !de || !dc || !off) {
        set_error("device allocation for the CSR failed");
        return TC_E_OOM;
    }
    uint64_t tot = 0, lastkey = 0;
    if (L) {
        const size_t ntiles = (L + kHcTile - 1) / kHcTile;
        DevBuf<uint64_t> tt, total;
        if ((st = tt.allocate(mem, ntiles * kHcWarps)) != TC_OK) return st;
        if ((st = total.allocate(mem, 1)) != TC_OK) return st;
        k_head_count<<<(unsigned)ntiles, kHcThreads, 0, s>>>(sorted, L, tt.p);
        TC_CUDA(cudaGetLastError());
        st = scan_exclusive<uint64_t>(mem, ntiles * kHcWarps, ArrayIn<uint64_t>{tt.p},
                                      ArrayOutExcl<uint64_t>{tt.p}, total.p, s, &g->launches);
        if (st != TC_OK) return st;
        k_head_write<<<(unsigned)ntiles, kHcThreads, 0, s>>>(sorted, L, tt.p, adj, du, de, off);
        TC_CUDA(cudaGetLastError());
        g->launches += 2;
        TC_CUDA(cudaMemcpyAsync(&tot, total.p, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
        TC_CUDA(cudaMemcpyAsync(&lastkey, sorted + (L - 1), sizeof(uint64_t),
                                cudaMemcpyDeviceToHost, s));
        TC_CUDA(cudaStreamSynchronize(s));
    }
    const uint64_t nnz = tot & 0xffffffffull, D = tot >> 32;
    uint64_t from = L ? ((lastkey >> 32) + 1) : 0;
    k_fill_tail<<<grid_for(n + 1 - from, 256), 256, 0, s>>>(off, from, n, (uint32_t)nnz);
    k_sentinels<<<grid_for(n + 8, 256), 256, 0, s>>>(off, n, adj);
    g->launches += 2;
    TC_CUDA(cudaGetLastError());

    // 4. stats
    k_vertex_stats<<<grid_for(n, 256), 256, 0, s>>>(off, n, scratch.p + 4);
    if (D) k_dyad_cost_stats<<<grid_for(D, 256), 256, 0, s>>>(off, du, de, D, dc, scratch.p + 4);
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
