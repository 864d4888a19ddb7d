// radix_sort.cu -- hand-written LSD radix sort of 64-bit keys on selected bit
// fields (a1's sort; SURVEY.md section 7 decision D1: written here, no CUB).
//
// One pass per digit of <= 8 bits:
//   upsweep    per-tile digit histogram (per-warp shared counters)
//   scan       exclusive scan of the digit-major histogram (scan.cuh)
//   downsweep  stable scatter: per warp, __match_any_sync groups the lanes
//              holding the same digit, rank = earlier peers + running per-warp
//              digit count; warp offsets within the tile come from a scan over
//              warps in shared memory.
#include "radix_sort.cuh"
#include "scan.cuh"

namespace tc {

namespace {

constexpr int kRsThreads = 256;
constexpr int kRsWarps = kRsThreads / 32;
constexpr int kRsItems = 16;
constexpr int kRsTile = kRsThreads * kRsItems;   // 4096 keys per block
constexpr int kMaxRadix = 256;

__global__ void __launch_bounds__(kRsThreads)
rs_upsweep(const uint64_t *__restrict__ keys, size_t n, int shift, uint32_t mask, int radix,
           uint32_t *__restrict__ hist, size_t ntiles) {
    __shared__ uint32_t wh[kRsWarps][kMaxRadix];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kRsWarps * kMaxRadix; i += kRsThreads) (&wh[0][0])[i] = 0;
    __syncthreads();
    size_t base = (size_t)blockIdx.x * kRsTile + (size_t)warp * 32 * kRsItems;
#pragma unroll 4
    for (int k = 0; k < kRsItems; k++) {
        size_t i = base + (size_t)k * 32 + lane;
        if (i < n) {
            uint32_t d = (uint32_t)(keys[i] >> shift) & mask;
            atomicAdd(&wh[warp][d], 1u);
        }
    }
    __syncthreads();
    for (int d = threadIdx.x; d < radix; d += kRsThreads) {
        uint32_t s = 0;
#pragma unroll
        for (int w = 0; w < kRsWarps; w++) s += wh[w][d];
        hist[(size_t)d * ntiles + blockIdx.x] = s;
    }
}

__global__ void __launch_bounds__(kRsThreads)
rs_downsweep(const uint64_t *__restrict__ keys, uint64_t *__restrict__ out, size_t n, int shift,
             uint32_t mask, int radix, const uint32_t *__restrict__ offs, size_t ntiles) {
    __shared__ uint32_t wc[kRsWarps][kMaxRadix];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kRsWarps * kMaxRadix; i += kRsThreads) (&wc[0][0])[i] = 0;
    __syncthreads();
    const uint32_t lt = (1u << lane) - 1u;
    size_t base = (size_t)blockIdx.x * kRsTile + (size_t)warp * 32 * kRsItems;
    uint64_t key[kRsItems];
    uint32_t rank[kRsItems];
#pragma unroll
    for (int k = 0; k < kRsItems; k++) {
        size_t i = base + (size_t)k * 32 + lane;
        bool valid = i < n;
        key[k] = valid ? keys[i] : 0ull;
        uint32_t d = valid ? ((uint32_t)(key[k] >> shift) & mask) : 0x10000u;
        uint32_t peers = __match_any_sync(0xffffffffu, d);
        uint32_t r = 0;
        if (valid) r = wc[warp][d] + __popc(peers & lt);
        __syncwarp();
        if (valid && (peers & lt) == 0) wc[warp][d] += __popc(peers);
        __syncwarp();
        rank[k] = r;
    }
    __syncthreads();
    // per digit: exclusive scan over warps + global offset of (digit, tile)
    for (int d = threadIdx.x; d < radix; d += kRsThreads) {
        uint32_t run = offs[(size_t)d * ntiles + blockIdx.x];
#pragma unroll
        for (int w = 0; w < kRsWarps; w++) {
            uint32_t c = wc[w][d];
            wc[w][d] = run;
            run += c;
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kRsItems; k++) {
        size_t i = base + (size_t)k * 32 + lane;
        if (i < n) {
            uint32_t d = (uint32_t)(key[k] >> shift) & mask;
            out[wc[warp][d] + rank[k]] = key[k];
        }
    }
}

}  // namespace

tc_status radix_sort_u64(Mem &mem, uint64_t *keys, uint64_t *tmp, size_t n,
                         const RadixPass *passes, int npasses, cudaStream_t s,
                         uint64_t *launches, uint64_t **sorted) {
    *sorted = keys;
    if (n <= 1 || npasses == 0) return TC_OK;
    if (n >= (1ull << 32)) {
        set_error("radix sort: %zu keys exceed the 32-bit offset range", n);
        return TC_E_INVALID;
    }
    size_t ntiles = (n + kRsTile - 1) / kRsTile;
    DevBuf<uint32_t> hist;
    tc_status st = hist.allocate(mem, ntiles * kMaxRadix);
    if (st != TC_OK) return st;
    uint64_t *src = keys, *dst = tmp;
    for (int p = 0; p < npasses; p++) {
        int bits = passes[p].bits;
        if (bits < 1 || bits > 8) {
            set_error("radix sort: digit width %d out of [1,8]", bits);
            return TC_E_INVALID;
        }
        int radix = 1 << bits;
        uint32_t mask = (uint32_t)radix - 1u;
        rs_upsweep<<<(unsigned)ntiles, kRsThreads, 0, s>>>(src, n, passes[p].shift, mask, radix,
                                                           hist.p, ntiles);
        TC_CUDA(cudaGetLastError());
        st = scan_exclusive<uint32_t>(mem, (size_t)radix * ntiles, ArrayIn<uint32_t>{hist.p},
                                      ArrayOutExcl<uint32_t>{hist.p}, (uint32_t *)nullptr, s,
                                      launches);
        if (st != TC_OK) return st;
        rs_downsweep<<<(unsigned)ntiles, kRsThreads, 0, s>>>(src, dst, n, passes[p].shift, mask,
                                                             radix, hist.p, ntiles);
        TC_CUDA(cudaGetLastError());
        if (launches) *launches += 2;
        uint64_t *t = src;
        src = dst;
        dst = t;
    }
    *sorted = src;
    return TC_OK;
}

}  // namespace tc

namespace tc {
int radix_passes_for(int lo, int width, RadixPass *out) {
    if (width <= 0) return 0;
    int np = (width + 7) / 8;
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
