// abi.cu -- the C ABI of libtriadcensus.so (include/triadcensus.h): argument
// checks, device/stream/allocator plumbing, the host closing (a5) and the
// NCCL multi-GPU census.  No census arithmetic lives here beyond the 128-bit
// null-triad closing n(n-1)(n-2)/6 - sum.
#include <dlfcn.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "census.cuh"

namespace tc {

static thread_local std::string g_err;

void set_error(const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
}

tc_status cuda_status(cudaError_t e, const char *what) {
    set_error("CUDA error %s (%s) in %s", cudaGetErrorName(e), cudaGetErrorString(e), what);
    return e == cudaErrorMemoryAllocation ? TC_E_OOM : TC_E_CUDA;
}

// default allocator: the device's CUDA memory pool, stream ordered, with
// freed blocks kept for reuse (release threshold = unlimited), so repeated
// builds and censuses do not return memory to the driver
static void keep_default_pool() {
    static thread_local int done_dev = -1;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev == done_dev) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done_dev = dev;
}

// Exact-size block cache in front of the pool: a freed block is kept under
// (device, stream, bytes) and handed to the next request of the same size on
// the same stream (stream order makes the reuse safe without a sync), so the
// repeated builds and censuses of one graph size allocate nothing from the
// driver after the first.  Measured: with cudaMallocAsync alone, C4's build
// and plan swung between 15 and 600 ms per step (pool growth on the large
// requests); with the cache they are as steady as torch's caching allocator.
// Blocks beyond kCacheCap bytes in total, or above kCacheMaxBlock each, go
// back to the pool.
namespace {
struct BlockKey {
    int dev;
    cudaStream_t stream;
    size_t bytes;
    bool operator<(const BlockKey &o) const {
        if (dev != o.dev) return dev < o.dev;
        if (stream != o.stream) return stream < o.stream;
        return bytes < o.bytes;
    }
};
std::mutex g_cache_mu;
std::map<BlockKey, std::vector<void *>> g_cache;
size_t g_cached = 0;
constexpr size_t kCacheCap = 120ull << 30;
constexpr size_t kCacheMaxBlock = 80ull << 30;
}  // namespace

void *Mem::alloc(size_t bytes) {
    if (bytes == 0) bytes = 1;
    if (custom) return hook.alloc(bytes, (void *)stream, hook.ctx);
    int dev = 0;
    cudaGetDevice(&dev);
    {
        std::lock_guard<std::mutex> lk(g_cache_mu);
        auto it = g_cache.find(BlockKey{dev, stream, bytes});
        if (it != g_cache.end() && !it->second.empty()) {
            void *p = it->second.back();
            it->second.pop_back();
            g_cached -= bytes;
            return p;
        }
    }
    keep_default_pool();
    void *p = nullptr;
    if (cudaMallocAsync(&p, bytes, stream) != cudaSuccess) {
        cudaGetLastError();
        // give the cached blocks back to the pool, the pool's unused
        // reservations back to the driver, and retry once (a request larger
        // than any free chunk needs fresh physical memory)
        std::lock_guard<std::mutex> lk(g_cache_mu);
        for (auto it2 = g_cache.begin(); it2 != g_cache.end();) {
            if (it2->first.dev != dev) {   // other devices' blocks stay cached
                ++it2;
                continue;
            }
            for (void *q : it2->second) {
                cudaFreeAsync(q, it2->first.stream);
                g_cached -= it2->first.bytes;
            }
            it2 = g_cache.erase(it2);
        }
        cudaDeviceSynchronize();
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
        if (cudaMallocAsync(&p, bytes, stream) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
    }
    return p;
}

void Mem::free(void *p, size_t bytes) {
    if (!p) return;
    if (bytes == 0) bytes = 1;
    if (custom) {
        hook.free(p, bytes, (void *)stream, hook.ctx);
        return;
    }
    int dev = 0;
    cudaGetDevice(&dev);
    {
        std::lock_guard<std::mutex> lk(g_cache_mu);
        if (bytes <= kCacheMaxBlock && g_cached + bytes <= kCacheCap) {
            g_cache[BlockKey{dev, stream, bytes}].push_back(p);
            g_cached += bytes;
            return;
        }
    }
    cudaFreeAsync(p, stream);
}

// ---- 128-bit closing (a5) ------------------------------------------------
static unsigned __int128 choose3(uint64_t n) {
    if (n < 3) return 0;   // DESIGN.md reading 18
    return (unsigned __int128)n * (n - 1) * (n - 2) / 6;
}

// pinned host slots for the lazy end of the build (16 words each), allocated
// once per process on first use
namespace {
std::mutex g_pin_mu;
unsigned long long *g_pin_base = nullptr;
std::vector<int> g_pin_free;
constexpr int kPinSlots = 1024, kPinWords = 16;

int pin_acquire(unsigned long long **p) {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    if (!g_pin_base) {
        void *q = nullptr;
        if (cudaMallocHost(&q, (size_t)kPinSlots * kPinWords * 8) != cudaSuccess) {
            cudaGetLastError();
            return -1;
        }
        g_pin_base = (unsigned long long *)q;
        for (int i = kPinSlots - 1; i >= 0; i--) g_pin_free.push_back(i);
    }
    if (g_pin_free.empty()) return -1;
    const int slot = g_pin_free.back();
    g_pin_free.pop_back();
    *p = g_pin_base + (size_t)slot * kPinWords;
    return slot;
}

void pin_release(int slot) {
    if (slot < 0) return;
    std::lock_guard<std::mutex> lk(g_pin_mu);
    g_pin_free.push_back(slot);
}
}  // namespace

tc_status graph_finalize(const tc_graph *gc) {
    tc_graph *g = const_cast<tc_graph *>(gc);
    if (g->final_.load()) return TC_OK;
    std::lock_guard<std::mutex> lk(g->mu);
    if (g->final_.load()) return TC_OK;
    TC_CUDA(cudaSetDevice(g->device));
    TC_CUDA(cudaEventSynchronize(g->ready));
    if (g->ev_b0) {
        cudaEventElapsedTime(&g->prof.build_ms, g->ev_b0, g->ev_b1);
        cudaEventDestroy(g->ev_b0);
        cudaEventDestroy(g->ev_b1);
        g->ev_b0 = g->ev_b1 = nullptr;
    }
    const tc_status st = build_finish(g, g->pin, (uint32_t)g->pin[8]);
    cudaEventDestroy(g->ready);
    g->ready = nullptr;
    pin_release(g->pin_slot);
    g->pin_slot = -1;
    g->pin = nullptr;
    g->final_ = true;
    return st;
}

}  // namespace tc

using namespace tc;

extern "C" {

const char *tc_last_error(void) { return g_err.c_str(); }

tc_status tc_trim_memory(void) {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    int cur = 0;
    cudaGetDevice(&cur);
    for (auto &kv : g_cache) {
        cudaSetDevice(kv.first.dev);
        for (void *q : kv.second) cudaFreeAsync(q, kv.first.stream);
    }
    g_cache.clear();
    g_cached = 0;
    int ndev = 0;
    cudaGetDeviceCount(&ndev);
    for (int d = 0; d < ndev; d++) {
        cudaSetDevice(d);
        cudaDeviceSynchronize();
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, d) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
    }
    cudaSetDevice(cur);
    return TC_OK;
}
int tc_abi_version(void) { return TC_ABI_VERSION; }

tc_status tc_close_census(uint64_t n, uint64_t counts[16], uint64_t *c003_hi) {
    if (!counts) {
        set_error("counts is NULL");
        return TC_E_INVALID;
    }
    unsigned __int128 sum = 0;
    for (int k = 1; k < 16; k++) sum += counts[k];
    unsigned __int128 total = choose3(n);
    if (sum > total) {
        set_error("census sum exceeds C(n,3): internal inconsistency");
        return TC_E_INVALID;
    }
    unsigned __int128 c1 = total - sum;
    counts[0] = (uint64_t)c1;
    uint64_t hi = (uint64_t)(c1 >> 64);
    if (c003_hi) *c003_hi = hi;
    else if (hi) {
        set_error("the 003 count needs a high word (n > 4,801,280) but c003_hi is NULL");
        return TC_E_OVERFLOW;
    }
    return TC_OK;
}

tc_status tc_graph_create(int device, uint64_t n, const uint32_t *src, const uint32_t *dst,
                          uint64_t m, int arcs_on_device, void *cuda_stream,
                          const tc_allocator *alloc, tc_graph **out) {
    if (!out) {
        set_error("out is NULL");
        return TC_E_INVALID;
    }
    *out = nullptr;
    if (n >= (1ull << 30)) {
        set_error("n = %llu must be < 2^30", (unsigned long long)n);
        return TC_E_INVALID;
    }
    if (m >= (1ull << 31)) {
        set_error("m = %llu must be < 2^31", (unsigned long long)m);
        return TC_E_INVALID;
    }
    if (m && (!src || !dst)) {
        set_error("src/dst is NULL");
        return TC_E_INVALID;
    }
    if (alloc && (!alloc->alloc || !alloc->free)) {
        set_error("allocator hook has NULL functions");
        return TC_E_INVALID;
    }
    TC_CUDA(cudaSetDevice(device));
    cudaStream_t s = (cudaStream_t)cuda_stream;
    tc_graph *g = new tc_graph();
    g->device = device;
    g->stream = s;
    g->mem.stream = s;
    if (alloc) {
        g->mem.custom = true;
        g->mem.hook = *alloc;
    }
    g->st.n = n;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    tc_status st = TC_OK;
    const uint32_t *ds = src, *dd = dst;
    DevBuf<uint32_t> hs, hd;
    if (!arcs_on_device && m) {
        if ((st = hs.allocate(g->mem, m)) != TC_OK || (st = hd.allocate(g->mem, m)) != TC_OK) {
            delete g;
            return st;
        }
        cudaError_t e = cudaMemcpyAsync(hs.p, src, m * 4, cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess) e = cudaMemcpyAsync(hd.p, dst, m * 4, cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) {
            hs.release();
            hd.release();
            delete g;
            return cuda_status(e, "H2D arc copy");
        }
        ds = hs.p;
        dd = hd.p;
    }
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    // lazy end of the build (graph_finalize) when a pinned slot is free
    g->pin_slot = pin_acquire(&g->pin);
    if (g->pin_slot >= 0 && cudaEventCreateWithFlags(&g->ready, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        pin_release(g->pin_slot);
        g->pin_slot = -1;
        g->pin = nullptr;
    }
    cudaEventRecord(e0, s);
    st = build_csr(g, ds, dd, m, s);
    cudaEventRecord(e1, s);
    if (st == TC_OK && !g->final_.load()) {   // finalized by the first query
        g->ev_b0 = e0;
        g->ev_b1 = e1;
    } else {
        if (cudaEventSynchronize(e1) == cudaSuccess)
            cudaEventElapsedTime(&g->prof.build_ms, e0, e1);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        if (g->ready) cudaEventDestroy(g->ready);
        g->ready = nullptr;
        pin_release(g->pin_slot);
        g->pin_slot = -1;
        g->pin = nullptr;
        g->final_ = true;
    }
    hs.release();
    hd.release();
    if (st != TC_OK) {
        std::string keep = g_err;
        tc_graph_destroy(g);
        g_err = keep;
        return st;
    }
    *out = g;
    return TC_OK;
}

tc_status tc_graph_stats_get(const tc_graph *g, tc_graph_stats *out) {
    if (!g || !out) {
        set_error("NULL argument");
        return TC_E_INVALID;
    }
    if (tc_status fs = graph_finalize(g)) return fs;
    *out = g->st;
    return TC_OK;
}

void tc_graph_destroy(tc_graph *g) {
    if (!g) return;
    cudaSetDevice(g->device);
    if (!g->final_.load()) {   // a graph destroyed before any query
        cudaEventSynchronize(g->ready);
        if (g->ev_b0) cudaEventDestroy(g->ev_b0);
        if (g->ev_b1) cudaEventDestroy(g->ev_b1);
        cudaEventDestroy(g->ready);
        pin_release(g->pin_slot);
        g->final_ = true;
    }
    g->mem.free(g->off, g->off_n * 4);
    g->mem.free(g->adj, (g->adj_alloc_n ? g->adj_alloc_n : g->adj_n) * 4);
    g->mem.free(g->dyad_u, g->dyad_n * 4);
    g->mem.free(g->dyad_e, g->dyad_n * 4);
    g->mem.free(g->dyad_c, g->dyad_n * 4);
    g->mem.free(g->dyad_pb, g->dyad_n * 4);
    g->mem.free(g->dyad_t, g->dyad_n * 4);
    g->mem.free(g->ups, g->ups_n * 4);
    if (g->tagpre) g->mem.free(g->tagpre, g->tagpre_n * 8);
    g->mem.free(g->plan_items, g->plan_cap_tiles * tc::kPlanTileItems * sizeof(tc::BinItemT));
    g->mem.free(g->plan_tcount, g->plan_cap_tiles * 4);
    g->mem.free(g->plan_big, g->plan_cap_big * 4);
    g->mem.free(g->plan_sums, 8 * 8);
    cudaStreamSynchronize(g->stream);
    delete g;
}

tc_status tc_profile_enable(tc_graph *g, int on) {
    if (!g) {
        set_error("NULL graph");
        return TC_E_INVALID;
    }
    g->profile = on;
    return TC_OK;
}

tc_status tc_profile_get(const tc_graph *g, tc_profile *out) {
    if (!g || !out) {
        set_error("NULL argument");
        return TC_E_INVALID;
    }
    if (tc_status fs = graph_finalize(g)) return fs;
    std::lock_guard<std::mutex> lk(g->mu);
    *out = g->prof;
    for (int i = 0; i < 4; i++) out->build_sort[i] = g->build_sort[i];
    return TC_OK;
}

uint64_t tc_launch_count(const tc_graph *g) {
    if (!g) return 0;
    std::lock_guard<std::mutex> lk(g->mu);
    return g->launches;
}

// A census call counts its launches and records its profile in locals and
// publishes them to the graph's "most recent call" slot once, under the
// graph's mutex: concurrent census calls on a shared graph do not race.
struct CallRec {
    uint64_t launches = 0;
    tc_profile prof{};
    tc_profile *profp(const tc_graph *g) { return g->profile ? &prof : nullptr; }
};

static void publish(const tc_graph *g, const CallRec &r) {
    std::lock_guard<std::mutex> lk(g->mu);
    g->launches = r.launches;
    if (g->profile) {
        const float build = g->prof.build_ms;
        g->prof = r.prof;
        g->prof.build_ms = build;
    }
}

tc_status tc_census_enqueue(const tc_graph *g, uint64_t dyad_begin, uint64_t dyad_end,
                            void *cuda_stream, uint64_t *d_counts) {
    if (!g || !d_counts) {
        set_error("NULL argument");
        return TC_E_INVALID;
    }
    if (tc_status fs = graph_finalize(g)) return fs;
    TC_CUDA(cudaSetDevice(g->device));
    CallRec r;
    const tc_status st = census_range_device(g, dyad_begin, dyad_end, (cudaStream_t)cuda_stream,
                                             d_counts, r.profp(g), &r.launches);
    publish(g, r);
    return st;
}

// paper = 1: classes 012 / 102 in the paper's per-dyad attribution (the
// tc_census_range contract); 0: the owed-credit attribution of the full and
// multi-GPU paths (reading 21; partials sum to the same census)
static tc_status census_partial_sync(const tc_graph *g, uint64_t k0, uint64_t k1,
                                     cudaStream_t s, uint64_t out[16], int paper) {
    TC_CUDA(cudaSetDevice(g->device));
    Mem mem = g->mem;
    mem.stream = s;
    DevBuf<uint64_t> d;
    tc_status st = d.allocate(mem, 16);
    if (st != TC_OK) return st;
    TC_CUDA(cudaMemsetAsync(d.p, 0, 16 * sizeof(uint64_t), s));
    CallRec r;
    st = paper ? census_range_paper_device(g, k0, k1, s, d.p, r.profp(g), &r.launches)
               : census_range_device(g, k0, k1, s, d.p, r.profp(g), &r.launches);
    publish(g, r);
    if (st != TC_OK) return st;
    TC_CUDA(cudaMemcpyAsync(out, d.p, 16 * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    out[0] = 0;
    return TC_OK;
}

tc_status tc_census(const tc_graph *g, void *cuda_stream, uint64_t counts[16], uint64_t *c003_hi) {
    if (!g || !counts) {
        set_error("NULL argument");
        return TC_E_INVALID;
    }
    if (tc_status fs = graph_finalize(g)) return fs;
    tc_status st = census_partial_sync(g, 0, g->st.dyads, (cudaStream_t)cuda_stream, counts, 0);
    if (st != TC_OK) return st;
    return tc_close_census(g->st.n, counts, c003_hi);
}

tc_status tc_census_range(const tc_graph *g, uint64_t dyad_begin, uint64_t dyad_end,
                          void *cuda_stream, uint64_t partial[16]) {
    if (!g || !partial) {
        set_error("NULL argument");
        return TC_E_INVALID;
    }
    if (tc_status fs = graph_finalize(g)) return fs;
    return census_partial_sync(g, dyad_begin, dyad_end, (cudaStream_t)cuda_stream, partial, 1);
}

tc_status tc_census64(const tc_graph *g, void *cuda_stream, uint64_t counts[64],
                      uint64_t *c0_hi) {
    if (!g || !counts) {
        set_error("NULL argument");
        return TC_E_INVALID;
    }
    if (tc_status fs = graph_finalize(g)) return fs;
    TC_CUDA(cudaSetDevice(g->device));
    cudaStream_t s = (cudaStream_t)cuda_stream;
    Mem mem = g->mem;
    mem.stream = s;
    DevBuf<uint64_t> d;
    tc_status st = d.allocate(mem, 64);
    if (st != TC_OK) return st;
    TC_CUDA(cudaMemsetAsync(d.p, 0, 64 * sizeof(uint64_t), s));
    CallRec r;
    st = census_range_device(g, 0, g->st.dyads, s, d.p, r.profp(g), &r.launches, 1);
    publish(g, r);
    if (st != TC_OK) return st;
    TC_CUDA(cudaMemcpyAsync(counts, d.p, 64 * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    unsigned __int128 sum = 0;
    for (int k = 1; k < 64; k++) sum += counts[k];
    unsigned __int128 total = choose3(g->st.n);
    if (sum > total) {
        set_error("64-type census sum exceeds C(n,3): internal inconsistency");
        return TC_E_INVALID;
    }
    unsigned __int128 c0 = total - sum;
    counts[0] = (uint64_t)c0;
    const uint64_t hi = (uint64_t)(c0 >> 64);
    if (c0_hi) *c0_hi = hi;
    else if (hi) {
        set_error("code 0 count needs a high word but c0_hi is NULL");
        return TC_E_OVERFLOW;
    }
    return TC_OK;
}

tc_status tc_shard_bounds_host(const uint64_t *cost, uint64_t D, int world, uint64_t kappa,
                               uint64_t *bounds) {
    if (!bounds || world < 1 || world > kMaxWorld || (D && !cost)) {
        set_error("invalid shard arguments");
        return TC_E_INVALID;
    }
    unsigned __int128 T = 0;
    for (uint64_t k = 0; k < D; k++) T += cost[k] + kappa;
    bounds[0] = 0;
    bounds[world] = D;
    // bounds[r] = first k whose exclusive cost prefix >= floor(T * r / world)
    unsigned __int128 pre = 0;
    uint64_t k = 0;
    for (int r = 1; r < world; r++) {
        unsigned __int128 t = T * (unsigned)r / (unsigned)world;
        while (k < D && pre < t) {
            pre += cost[k] + kappa;
            k++;
        }
        bounds[r] = k;
    }
    return TC_OK;
}

tc_status tc_task_queues(const tc_graph *g, int strategy, uint64_t max_nset_size,
                         void *cuda_stream, uint64_t *starts, uint64_t cap, uint64_t *nqueues,
                         uint64_t *total_nset) {
    if (!g || !nqueues || !total_nset || (strategy != TC_QUEUES_UNIFORM &&
                                           strategy != TC_QUEUES_NONUNIFORM) ||
        (cap && !starts)) {
        set_error("invalid task-queue arguments");
        return TC_E_INVALID;
    }
    if (tc_status fs = graph_finalize(g)) return fs;
    TC_CUDA(cudaSetDevice(g->device));
    return task_queues_device(g, strategy == TC_QUEUES_NONUNIFORM, max_nset_size,
                              (cudaStream_t)cuda_stream, starts, cap, nqueues, total_nset);
}

tc_status tc_shard_bounds(const tc_graph *g, int world, void *cuda_stream, uint64_t *bounds) {
    if (!g || !bounds || world < 1 || world > kMaxWorld) {
        set_error("invalid shard arguments");
        return TC_E_INVALID;
    }
    if (tc_status fs = graph_finalize(g)) return fs;
    TC_CUDA(cudaSetDevice(g->device));
    return shard_bounds_device(g, world, (cudaStream_t)cuda_stream, kShardKappa, bounds);
}

}  // extern "C"

// ---------------------------------------------------------------------------
// NCCL, loaded lazily so the library loads (and the CPU tests run) without it
// ---------------------------------------------------------------------------
namespace {

typedef struct { char internal[128]; } nccl_uid;
typedef void *nccl_comm_t;
typedef int (*fn_get_uid)(nccl_uid *);
typedef int (*fn_init_rank)(nccl_comm_t *, int, nccl_uid, int);
typedef int (*fn_allreduce)(const void *, void *, size_t, int, int, nccl_comm_t, cudaStream_t);
typedef int (*fn_destroy)(nccl_comm_t);
typedef const char *(*fn_errstr)(int);
typedef int (*fn_comm_int)(nccl_comm_t, int *);

struct Nccl {
    void *h = nullptr;
    fn_get_uid get_uid = nullptr;
    fn_init_rank init_rank = nullptr;
    fn_allreduce allreduce = nullptr;
    fn_destroy destroy = nullptr;
    fn_errstr errstr = nullptr;
    fn_comm_int count = nullptr, user_rank = nullptr, cu_device = nullptr;
};

Nccl *nccl() {
    static Nccl n;
    static bool tried = false;
    if (tried) return n.h ? &n : nullptr;
    tried = true;
    const char *names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char *nm : names) {
        n.h = dlopen(nm, RTLD_NOW | RTLD_NOLOAD);   // the copy torch already loaded
        if (!n.h) n.h = dlopen(nm, RTLD_NOW);
        if (n.h) break;
    }
    if (!n.h) return nullptr;
    n.get_uid = (fn_get_uid)dlsym(n.h, "ncclGetUniqueId");
    n.init_rank = (fn_init_rank)dlsym(n.h, "ncclCommInitRank");
    n.allreduce = (fn_allreduce)dlsym(n.h, "ncclAllReduce");
    n.destroy = (fn_destroy)dlsym(n.h, "ncclCommDestroy");
    n.errstr = (fn_errstr)dlsym(n.h, "ncclGetErrorString");
    n.count = (fn_comm_int)dlsym(n.h, "ncclCommCount");
    n.user_rank = (fn_comm_int)dlsym(n.h, "ncclCommUserRank");
    n.cu_device = (fn_comm_int)dlsym(n.h, "ncclCommCuDevice");
    if (!n.get_uid || !n.init_rank || !n.allreduce || !n.destroy) {
        n.h = nullptr;
        return nullptr;
    }
    return &n;
}

const int kNcclUint64 = 5;   // ncclUint64 in nccl.h
const int kNcclSum = 0;      // ncclSum

tc_status nccl_fail(Nccl *n, int rc, const char *what) {
    set_error("NCCL error %d (%s) in %s", rc, n && n->errstr ? n->errstr(rc) : "?", what);
    return TC_E_NCCL;
}

}  // namespace

struct tc_comm {
    nccl_comm_t comm = nullptr;
    int world = 1, rank = 0, device = 0;
    bool borrowed = false;   // tc_comm_wrap: the caller owns the ncclComm_t
};

extern "C" {

tc_status tc_comm_unique_id(uint8_t id[128]) {
    Nccl *n = nccl();
    if (!n) {
        set_error("libnccl.so.2 could not be loaded");
        return TC_E_NCCL;
    }
    nccl_uid u;
    int rc = n->get_uid(&u);
    if (rc) return nccl_fail(n, rc, "ncclGetUniqueId");
    memcpy(id, u.internal, 128);
    return TC_OK;
}

tc_status tc_comm_create(const uint8_t id[128], int world, int rank, int device, tc_comm **out) {
    if (!id || !out || world < 1 || world > kMaxWorld || rank < 0 || rank >= world) {
        set_error("invalid communicator arguments");
        return TC_E_INVALID;
    }
    Nccl *n = nccl();
    if (!n) {
        set_error("libnccl.so.2 could not be loaded");
        return TC_E_NCCL;
    }
    TC_CUDA(cudaSetDevice(device));
    nccl_uid u;
    memcpy(u.internal, id, 128);
    tc_comm *c = new tc_comm();
    int rc = n->init_rank(&c->comm, world, u, rank);
    if (rc) {
        delete c;
        return nccl_fail(n, rc, "ncclCommInitRank");
    }
    c->world = world;
    c->rank = rank;
    c->device = device;
    *out = c;
    return TC_OK;
}

tc_status tc_comm_wrap(void *borrowed_nccl_comm, tc_comm **out) {
    if (!borrowed_nccl_comm || !out) {
        set_error("invalid communicator arguments");
        return TC_E_INVALID;
    }
    Nccl *n = nccl();
    if (!n || !n->count || !n->user_rank || !n->cu_device) {
        set_error("libnccl.so.2 (with ncclCommCount/UserRank/CuDevice) could not be loaded");
        return TC_E_NCCL;
    }
    nccl_comm_t cm = (nccl_comm_t)borrowed_nccl_comm;
    int world = 0, rank = 0, dev = 0, rc;
    if ((rc = n->count(cm, &world))) return nccl_fail(n, rc, "ncclCommCount");
    if ((rc = n->user_rank(cm, &rank))) return nccl_fail(n, rc, "ncclCommUserRank");
    if ((rc = n->cu_device(cm, &dev))) return nccl_fail(n, rc, "ncclCommCuDevice");
    if (world < 1 || world > kMaxWorld) {
        set_error("communicator of %d ranks: at most %d supported", world, kMaxWorld);
        return TC_E_INVALID;
    }
    tc_comm *c = new tc_comm();
    c->comm = cm;
    c->world = world;
    c->rank = rank;
    c->device = dev;
    c->borrowed = true;
    *out = c;
    return TC_OK;
}

void tc_comm_destroy(tc_comm *c) {
    if (!c) return;
    Nccl *n = nccl();
    if (n && c->comm && !c->borrowed) n->destroy(c->comm);
    delete c;
}

tc_status tc_census_multi(const tc_graph *g, tc_comm *comm, void *cuda_stream,
                          uint64_t counts[16], uint64_t *c003_hi) {
    if (!g || !comm || !counts) {
        set_error("NULL argument");
        return TC_E_INVALID;
    }
    if (tc_status fs = graph_finalize(g)) return fs;
    Nccl *n = nccl();
    if (!n) {
        set_error("libnccl.so.2 could not be loaded");
        return TC_E_NCCL;
    }
    TC_CUDA(cudaSetDevice(g->device));
    cudaStream_t s = (cudaStream_t)cuda_stream;
    std::vector<uint64_t> bounds((size_t)comm->world + 1);
    tc_status st = shard_bounds_device(g, comm->world, s, kShardKappa, bounds.data());
    if (st != TC_OK) return st;
    Mem mem = g->mem;
    mem.stream = s;
    DevBuf<uint64_t> d;
    if ((st = d.allocate(mem, 16)) != TC_OK) return st;
    TC_CUDA(cudaMemsetAsync(d.p, 0, 16 * sizeof(uint64_t), s));
    if ((st = tc_census_enqueue(g, bounds[comm->rank], bounds[comm->rank + 1], s, d.p)) != TC_OK)
        return st;
    int rc = n->allreduce(d.p, d.p, 16, kNcclUint64, kNcclSum, comm->comm, s);
    if (rc) return nccl_fail(n, rc, "ncclAllReduce");
    TC_CUDA(cudaMemcpyAsync(counts, d.p, 16 * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    counts[0] = 0;
    return tc_close_census(g->st.n, counts, c003_hi);
}

}  // extern "C"
