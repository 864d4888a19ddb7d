// schedule.cu -- a2: degree-binned canonical-dyad scheduler + shard cuts.
//
// Each canonical dyad (u, v), u < v, gets the paper's uniform workload
// estimate c = |N(u)| + |N(v)| (Fig. P:1678-1705, "NsetSize + |N[u]| + |N[v]|
// - 2"; the constant -2 does not change any bin or cut) and is
// placed in one of three bins so power-law hubs do not serialise a warp:
//   thread bin  c <= kThreadBinMax      one thread merges the whole dyad
//   warp bin    c <= kWarpBinMax        32 lanes split it by merge-path
//   block bin   c >  kWarpBinMax        chunks of kBlockSpan diagonals, one
//                                       256-thread block per chunk
// The same costs, prefix-summed in canonical order, give the degree-balanced
// multi-GPU shard cuts: the paper's uniform task
// queues with one "queue" per GPU.
#include "census.cuh"
#include "scan.cuh"

namespace tc {

namespace {

__device__ __forceinline__ uint32_t dyad_cost(const uint32_t *__restrict__ off,
                                              const uint32_t *__restrict__ adj, uint32_t u,
                                              uint32_t p, uint32_t *v_out) {
    uint32_t v = __ldg(adj + p) >> 2;
    *v_out = v;
    return (__ldg(off + u + 1) - __ldg(off + u)) + (__ldg(off + v + 1) - __ldg(off + v));
}

__device__ __forceinline__ int bin_of(uint32_t c) {
    return c <= kThreadBinMax ? 0 : (c <= kWarpBinMax ? 1 : 2);
}

// cnt[0..2] items per bin (bin 2 counts chunks), cnt[3..5] work per bin
__global__ void k_plan_count(const uint32_t *__restrict__ du, const uint32_t *__restrict__ dp,
                             const uint32_t *__restrict__ off, const uint32_t *__restrict__ adj,
                             uint64_t k0, uint64_t k1, unsigned long long *cnt) {
    unsigned long long c0 = 0, c1 = 0, c2 = 0, w0 = 0, w1 = 0, w2 = 0;
    for (uint64_t k = k0 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < k1;
         k += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t v;
        uint32_t c = dyad_cost(off, adj, __ldg(du + k), __ldg(dp + k), &v);
        int b = bin_of(c);
        if (b == 0) { c0++; w0 += c; }
        else if (b == 1) { c1++; w1 += c; }
        else { c2 += (c + kBlockSpan - 1) / kBlockSpan; w2 += c; }
    }
    for (int o = 16; o; o >>= 1) {
        c0 += __shfl_xor_sync(0xffffffffu, c0, o);
        c1 += __shfl_xor_sync(0xffffffffu, c1, o);
        c2 += __shfl_xor_sync(0xffffffffu, c2, o);
        w0 += __shfl_xor_sync(0xffffffffu, w0, o);
        w1 += __shfl_xor_sync(0xffffffffu, w1, o);
        w2 += __shfl_xor_sync(0xffffffffu, w2, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (c0) atomicAdd(&cnt[0], c0);
        if (c1) atomicAdd(&cnt[1], c1);
        if (c2) atomicAdd(&cnt[2], c2);
        if (w0) atomicAdd(&cnt[3], w0);
        if (w1) atomicAdd(&cnt[4], w1);
        if (w2) atomicAdd(&cnt[5], w2);
    }
}

__global__ void k_plan_fill(const uint32_t *__restrict__ du, const uint32_t *__restrict__ dp,
                            const uint32_t *__restrict__ off, const uint32_t *__restrict__ adj,
                            uint64_t k0, uint64_t k1, BinItem2 *tl, BinItem2 *wl, BinItem4 *bl,
                            unsigned long long *cur) {
    const uint32_t lane = threadIdx.x & 31, lt = (1u << lane) - 1u;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t base = k0 + ((uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u));
         base < k1; base += stride) {
        uint64_t k = base + lane;
        bool valid = k < k1;
        uint32_t u = 0, p = 0, v = 0, c = 0;
        int b = -1;
        if (valid) {
            u = __ldg(du + k);
            p = __ldg(dp + k);
            c = dyad_cost(off, adj, u, p, &v);
            b = bin_of(c);
        }
#pragma unroll
        for (int q = 0; q < 2; q++) {
            uint32_t m = __ballot_sync(0xffffffffu, b == q);
            if (m) {
                int leader = __ffs(m) - 1;
                unsigned long long at = 0;
                if ((int)lane == leader) at = atomicAdd(&cur[q], (unsigned long long)__popc(m));
                at = __shfl_sync(0xffffffffu, at, leader);
                if (b == q) {
                    BinItem2 it{u, p};
                    (q == 0 ? tl : wl)[at + __popc(m & lt)] = it;
                }
            }
        }
        if (b == 2) {
            uint32_t nch = (c + kBlockSpan - 1) / kBlockSpan;
            unsigned long long at = atomicAdd(&cur[2], (unsigned long long)nch);
            for (uint32_t q = 0; q < nch; q++) {
                uint32_t d0 = q * kBlockSpan, d1 = min(c, d0 + kBlockSpan);
                bl[at + q] = BinItem4{u, p, d0, d1};
            }
        }
    }
}

struct CostIn {
    const uint32_t *du, *dp, *off, *adj;
    uint64_t kappa;
    __device__ __forceinline__ uint64_t operator()(size_t k) const {
        uint32_t v;
        return (uint64_t)dyad_cost(off, adj, __ldg(du + k), __ldg(dp + k), &v) + kappa;
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

inline unsigned grid_for(uint64_t work, int threads, unsigned cap = 148 * 16) {
    uint64_t b = (work + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > cap) b = cap;
    return (unsigned)b;
}

}  // namespace

tc_status census_range_device(const tc_graph *g, uint64_t k0, uint64_t k1, cudaStream_t s,
                              uint64_t *d_counts, tc_profile *prof, uint64_t *launches) {
    const uint64_t D = g->st.dyads;
    if (k1 > D) k1 = D;
    if (k0 >= k1) return TC_OK;
    Mem mem = g->mem;
    mem.stream = s;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (prof) {
        TC_CUDA(cudaEventCreate(&e0));
        TC_CUDA(cudaEventCreate(&e1));
        TC_CUDA(cudaEventRecord(e0, s));
    }
    tc_status st;
    DevBuf<unsigned long long> cnt;
    if ((st = cnt.allocate(mem, 12)) != TC_OK) return st;
    TC_CUDA(cudaMemsetAsync(cnt.p, 0, 12 * sizeof(unsigned long long), s));
    k_plan_count<<<grid_for(k1 - k0, 256), 256, 0, s>>>(g->dyad_u, g->dyad_p, g->off, g->adj, k0,
                                                        k1, cnt.p);
    TC_CUDA(cudaGetLastError());
    unsigned long long h[6];
    TC_CUDA(cudaMemcpyAsync(h, cnt.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    DevBuf<BinItem2> tl, wl;
    DevBuf<BinItem4> bl;
    if ((st = tl.allocate(mem, h[0])) != TC_OK) return st;
    if ((st = wl.allocate(mem, h[1])) != TC_OK) return st;
    if ((st = bl.allocate(mem, h[2])) != TC_OK) return st;
    k_plan_fill<<<grid_for(k1 - k0, 256), 256, 0, s>>>(g->dyad_u, g->dyad_p, g->off, g->adj, k0,
                                                       k1, tl.p, wl.p, bl.p, cnt.p + 6);
    TC_CUDA(cudaGetLastError());
    *launches += 2;
    if (prof) {
        TC_CUDA(cudaEventRecord(e1, s));
        TC_CUDA(cudaEventSynchronize(e1));
        float t;
        TC_CUDA(cudaEventElapsedTime(&t, e0, e1));
        prof->plan_ms = t;
        for (int i = 0; i < 3; i++) {
            prof->bin_items[i] = h[i];
            prof->bin_work[i] = h[3 + i];
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    }
    BinLists lists;
    lists.t = tl.p;
    lists.w = wl.p;
    lists.b = bl.p;
    for (int i = 0; i < 3; i++) lists.count[i] = h[i];
    return launch_bins(g, lists, s, d_counts, prof, launches);
}

tc_status shard_bounds_device(const tc_graph *g, int world, cudaStream_t s, uint64_t kappa,
                              uint64_t *bounds) {
    const uint64_t D = g->st.dyads;
    bounds[0] = 0;
    bounds[world] = D;
    if (world == 1) return TC_OK;
    Mem mem = g->mem;
    mem.stream = s;
    tc_status st;
    DevBuf<uint64_t> excl, tot, tg, out;
    if ((st = excl.allocate(mem, D)) != TC_OK) return st;
    if ((st = tot.allocate(mem, 1)) != TC_OK) return st;
    st = scan_exclusive<uint64_t>(mem, D, CostIn{g->dyad_u, g->dyad_p, g->off, g->adj, kappa},
                                  ArrayOutExcl<uint64_t>{excl.p}, tot.p, s, nullptr);
    if (st != TC_OK) return st;
    uint64_t T = 0;
    TC_CUDA(cudaMemcpyAsync(&T, tot.p, sizeof(T), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    uint64_t targets[1024];
    if (world > 1024) {
        set_error("world %d > 1024", world);
        return TC_E_INVALID;
    }
    for (int r = 1; r < world; r++)
        targets[r - 1] = (uint64_t)(((unsigned __int128)T * (unsigned)r) / (unsigned)world);
    if ((st = tg.allocate(mem, world)) != TC_OK) return st;
    if ((st = out.allocate(mem, world)) != TC_OK) return st;
    TC_CUDA(cudaMemcpyAsync(tg.p, targets, (world - 1) * sizeof(uint64_t), cudaMemcpyHostToDevice,
                            s));
    k_lower_bounds<<<1, 1024, 0, s>>>(excl.p, D, tg.p, world - 1, out.p);
    TC_CUDA(cudaGetLastError());
    TC_CUDA(cudaMemcpyAsync(bounds + 1, out.p, (world - 1) * sizeof(uint64_t),
                            cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    return TC_OK;
}

}  // namespace tc
