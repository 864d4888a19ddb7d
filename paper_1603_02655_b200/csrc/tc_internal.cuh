// tc_internal.cuh -- internal declarations of libtriadcensus (not installed).
//
// Device data layout:
//   off[n+1]   uint32 row offsets of the symmetric neighbour CSR
//   adj[2D]    uint32 entries (w << 2) | tag, each row sorted by w;
//              tag bit0 = u->w, bit1 = w->u (the 2-bit direction code)
//   ups[n]     uint32 index in adj of the first entry w > u of row u
//   dyad_u[D], dyad_e[D], dyad_c[D], dyad_pb[D], dyad_t[D]   canonical
//              dyads (u < v) in canonical order (u ascending, v ascending,
//              P:277-281): row u, the entry of v in row u, e = (v << 2) | pre
//              with pre = IsEdge(u,v) + 2 IsEdge(v,u) (v0.4), the
//              uniform cost c = |N(u)| + |N(v)|, the index in adj of
//              the first entry w > u of row v, and the merge length
//              t = |{w in N(u): w > u}| + |{w in N(v): w > u}| (census.cu)
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "triadcensus.h"

namespace tc {

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
void set_error(const char *fmt, ...);
tc_status cuda_status(cudaError_t e, const char *what);

#define TC_CUDA(call)                                                          \
    do {                                                                       \
        cudaError_t _e = (call);                                               \
        if (_e != cudaSuccess) return ::tc::cuda_status(_e, #call);            \
    } while (0)

// ---------------------------------------------------------------------------
// stream-ordered device memory through the caller's allocator hook
// ---------------------------------------------------------------------------
struct Mem {
    tc_allocator hook;
    bool custom = false;
    cudaStream_t stream = nullptr;
    void *alloc(size_t bytes);
    void free(void *p, size_t bytes);
};

template <typename T>
struct DevBuf {
    T *p = nullptr;
    size_t n = 0;
    Mem *mem = nullptr;
    tc_status allocate(Mem &m, size_t count) {
        mem = &m;
        n = count;
        size_t bytes = (count ? count : 1) * sizeof(T);
        p = static_cast<T *>(m.alloc(bytes));
        if (!p) {
            set_error("device allocation of %zu bytes failed", bytes);
            return TC_E_OOM;
        }
        return TC_OK;
    }
    void release() {
        if (p && mem) mem->free(p, (n ? n : 1) * sizeof(T));
        p = nullptr;
        n = 0;
    }
    ~DevBuf() { release(); }
};

// ---------------------------------------------------------------------------
// bin thresholds of the degree-binned scheduler (a2).  Cost c = |N(u)|+|N(v)|.
// ---------------------------------------------------------------------------
constexpr uint32_t kThreadBinMax = 254;    // c <= 254: one thread per dyad, sorted by c
constexpr uint32_t kLaneSpan = 255;        // max diagonals per lane (8-bit packed counters)
constexpr uint32_t kWarpChunk = 32 * kLaneSpan;   // c > 254: warp items of <= 8160 diagonals
constexpr int kNumBins = 2;
// skewed-pair path (census.cu, schedule.cu): enabled on graphs with a row of
// >= kSparseMinDegree entries; a big dyad whose short list s and long list l
// satisfy s * (log2(l) + 4) * 2 < s + l is classified by binary searches of
// the short list's entries in the long one (kSparseChunk short-list entries
// per warp item) plus tag-count ranges of the long list
constexpr uint64_t kSparseMinDegree = 4096;
constexpr uint32_t kSparseChunk = 256;
// per-dyad overhead of the shard cost model, in list-entry equivalents
// (8 B item + 16 B offsets ~ 6 entries; SURVEY.md section 8(e) kappa ~ 8)
constexpr uint64_t kShardKappa = 8;
constexpr int kMaxWorld = 1024;   // ranks a shard cut supports

constexpr uint64_t kPlanTileItems = 4096;   // = kPlanTile (census.cuh)
constexpr uint64_t kResidentMaxDyads = 1ull << 27;   // graph-resident census plan up to this D
struct BinItemT {   // thread bin: merge starts in adj, e = v<<2|pre, t = merge length
    uint32_t pa, pb, e, t;   // | (length of the A part) << 16 (both <= 254)
};
struct BinItemW {   // warp bin: dyad index (in the planned range), diagonals [d0, d1)
    uint32_t k, d0, d1, pad;
};

#ifdef __CUDACC__
// Lanes of the (full) warp whose value d agrees with mine on bits [0, BITS):
// one ballot per bit, each bit tested once -- the predicate feeds both the
// ballot and the lane's own mask (peers &= bit ? b : ~b as one XNOR).  The
// plain C form tests the bit twice (7 instructions per bit, 4 here; the LSD
// downsweep 96 -> 82 us per pass at C3).  Callers AND the result with the
// lanes that hold a valid d.
template <int BITS>
__device__ __forceinline__ uint32_t warp_peers(uint32_t d) {
    uint32_t peers = 0xffffffffu;
#pragma unroll
    for (int bit = 0; bit < BITS; bit++) {
        uint32_t b, msk;
        asm("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\t"
            "and.b32 t, %2, %3;\n\tsetp.ne.u32 p, t, 0;\n\t"
            "vote.sync.ballot.b32 %0, p, 0xffffffff;\n\t"
            "selp.b32 %1, -1, 0, p;\n\t}"
            : "=r"(b), "=r"(msk)
            : "r"(d), "r"(1u << bit));
        peers &= ~(b ^ msk);
    }
    return peers;
}
#endif

}  // namespace tc

// the opaque graph
struct tc_graph {
    int device = 0;
    cudaStream_t stream = nullptr;      // creating stream (used for frees)
    tc::Mem mem;
    tc_graph_stats st{};
    uint32_t *off = nullptr;   size_t off_n = 0;
    uint32_t *adj = nullptr;   size_t adj_n = 0;
    uint32_t *dyad_u = nullptr; size_t dyad_n = 0;
    uint32_t *dyad_e = nullptr;
    uint32_t *dyad_c = nullptr;
    uint32_t *dyad_pb = nullptr;
    uint32_t *dyad_t = nullptr;
    uint32_t *ups = nullptr;   size_t ups_n = 0;
    // exclusive prefix over adj of (tag == 1) << 32 | (tag == 2), adj_n + 1
    // entries; built only when some row is long (max degree >=
    // kSparseMinDegree): the skewed-pair path of the warp bin counts the tags
    // of a row range with two loads instead of a merge (census.cu)
    uint64_t *tagpre = nullptr; size_t tagpre_n = 0;
    size_t adj_alloc_n = 0;             // entries allocated for adj (>= adj_n)
    uint64_t build_sort[4] = {0, 0, 0, 0};   // tc_profile.build_sort (csr_build.cu)
    // lazy end of the build: the stats and D are copied into a pinned slot
    // and `ready` is recorded; the first call that needs the host-side stats
    // waits there (graph_finalize), so the caller's own host work between
    // tc_graph_create and the census overlaps the build's last kernels
    unsigned long long *pin = nullptr;
    int pin_slot = -1;
    cudaEvent_t ready = nullptr, ev_b0 = nullptr, ev_b1 = nullptr;
    std::atomic<bool> final_{true};
    // the full-census plan built with the graph (schedule.cu k_upper_plan):
    // thread-bin items per tile of kPlanTile dyads sorted by merge length, the
    // tiles' item counts, the big dyads (t > kThreadBinMax) and the sums
    // [n - c of pre 1..3, thread-bin sum c, thread-bin sum t, big dyads]
    tc::BinItemT *plan_items = nullptr;
    uint32_t *plan_tcount = nullptr;
    uint32_t *plan_big = nullptr;
    unsigned long long *plan_sums = nullptr;
    uint64_t plan_cap_tiles = 0, plan_cap_big = 0;
    int profile = 0;
    // results of the most recent build / census call: written once at the
    // end of a call from that call's own locals, under `mu` (a graph may be
    // shared read-only by concurrent census calls on different streams)
    mutable std::mutex mu;
    mutable tc_profile prof{};
    mutable uint64_t launches = 0;
    // shard cuts per world size (tc_shard_bounds / tc_census_multi), computed
    // once on first use, under `mu`
    mutable std::map<int, std::vector<uint64_t>> shard_cache;
};

namespace tc {

// phase entry points (each file owns one step of SURVEY.md section 8(a))
tc_status build_csr(tc_graph *g, const uint32_t *d_src, const uint32_t *d_dst, uint64_t m,
                    cudaStream_t s);                                  // a1, csr_build.cu
tc_status census_range_device(const tc_graph *g, uint64_t k0, uint64_t k1, cudaStream_t s,
                              uint64_t *d_counts, tc_profile *prof, uint64_t *launches,
                              int mode64 = 0);  // a2-a4
// tc_census_range: the same range census, but classes 012 / 102 in the
// paper's per-dyad attribution n - |S| - 2 (schedule.cu k_range_dyadic)
tc_status census_range_paper_device(const tc_graph *g, uint64_t k0, uint64_t k1, cudaStream_t s,
                                    uint64_t *d_counts, tc_profile *prof, uint64_t *launches);
// the host side of the build's end (stats, adjacency size, the tag prefix
// of hub graphs) from the values the device wrote: h[8] stats, D (csr_build.cu)
tc_status build_finish(tc_graph *g, const unsigned long long *h, uint32_t D);
// waits for a lazily ended build and runs build_finish once (abi.cu); every
// entry point that reads the graph's host-side stats calls it first
tc_status graph_finalize(const tc_graph *g);
// a1 + a2 fused: upper row entries, c, t and the graph's full-census plan
tc_status upper_plan_device(tc_graph *g, const uint32_t *lo_start, const uint32_t *dD, uint64_t Dub,
                            unsigned long long *bstats, cudaStream_t s);   // schedule.cu
tc_status shard_bounds_device(const tc_graph *g, int world, cudaStream_t s, uint64_t kappa,
                              uint64_t *bounds);                      // schedule.cu
tc_status task_queues_device(const tc_graph *g, int nonuniform, uint64_t max_nset, cudaStream_t s,
                             uint64_t *starts, uint64_t cap, uint64_t *nq,
                             uint64_t *total);                        // schedule.cu (f3)

// generic device-wide exclusive scan with a per-element input functor and an
// output functor; scan.cuh
}  // namespace tc
