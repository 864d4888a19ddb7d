// scan.cuh -- device-wide exclusive prefix scan (reduce-then-scan, 3 phases)
// with an input functor (element i -> T) and an output functor (i, exclusive
// prefix, value) so callers fuse the flag computation and the scatter into
// the scan passes instead of materialising flag arrays.
#pragma once

#include "tc_internal.cuh"

namespace tc {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;  // 4096 elements per block

template <typename T>
__device__ __forceinline__ T warp_inclusive_sum(T x) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    return x;
}

// Exclusive scan of one value per thread across the block (blockDim.x ==
// kScanThreads).  Returns the thread's exclusive prefix; *total = block sum.
template <typename T, int NT = kScanThreads>
__device__ __forceinline__ T block_exclusive_sum(T x, T *total) {
    constexpr int NW = NT / 32;
    __shared__ T warp_sums[NW];
    __shared__ T block_total;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T inc = warp_inclusive_sum(x);
    if (lane == 31) warp_sums[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        T w = lane < NW ? warp_sums[lane] : T(0);
        T wi = warp_inclusive_sum(w);
        if (lane < NW) warp_sums[lane] = wi - w;
        if (lane == NW - 1) block_total = wi;
    }
    __syncthreads();
    T excl = warp_sums[warp] + inc - x;
    *total = block_total;
    __syncthreads();  // shared scratch may be reused by the next call
    return excl;
}

template <typename T, typename In>
__global__ void __launch_bounds__(kScanThreads) scan_reduce_kernel(size_t n, In in, T *partials) {
    size_t base = (size_t)blockIdx.x * kScanTile;
    T s = 0;
#pragma unroll 4
    for (int k = 0; k < kScanItems; k++) {
        size_t i = base + (size_t)k * kScanThreads + threadIdx.x;   // striped: coalesced
        if (i < n) s += in(i);
    }
    T tot;
    block_exclusive_sum<T>(s, &tot);
    if (threadIdx.x == 0) partials[blockIdx.x] = tot;
}

template <typename T, typename In, typename Out>
__global__ void __launch_bounds__(kScanThreads) scan_down_kernel(size_t n, In in, Out out,
                                                                 const T *offsets, T *d_total,
                                                                 int write_total) {
    size_t base = (size_t)blockIdx.x * kScanTile + (size_t)threadIdx.x * kScanItems;  // blocked
    T v[kScanItems];
    T s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; k++) {
        size_t i = base + k;
        v[k] = (i < n) ? in(i) : T(0);
        s += v[k];
    }
    T tot;
    T run = block_exclusive_sum<T>(s, &tot) + (offsets ? offsets[blockIdx.x] : T(0));
    if (write_total && blockIdx.x == gridDim.x - 1 && threadIdx.x == 0)
        *d_total = (offsets ? offsets[blockIdx.x] : T(0)) + tot;
#pragma unroll
    for (int k = 0; k < kScanItems; k++) {
        size_t i = base + k;
        if (i < n) out(i, run, v[k]);
        run += v[k];
    }
}

template <typename T>
struct ArrayIn {
    const T *a;
    __device__ __forceinline__ T operator()(size_t i) const { return a[i]; }
};
template <typename T>
struct ArrayOutExcl {
    T *a;
    __device__ __forceinline__ void operator()(size_t i, T excl, T) const { a[i] = excl; }
};

// Exclusive scan of in(0..n-1).  out(i, excl, v) is called once per element.
// If d_total != nullptr it receives the sum (device memory).
template <typename T, typename In, typename Out>
tc_status scan_exclusive(Mem &mem, size_t n, In in, Out out, T *d_total, cudaStream_t s,
                         uint64_t *launches) {
    if (n == 0) {
        if (d_total) TC_CUDA(cudaMemsetAsync(d_total, 0, sizeof(T), s));
        return TC_OK;
    }
    size_t nb = (n + kScanTile - 1) / kScanTile;
    if (nb == 1) {
        scan_down_kernel<T, In, Out><<<1, kScanThreads, 0, s>>>(n, in, out, nullptr, d_total,
                                                                 d_total != nullptr);
        if (launches) *launches += 1;
        TC_CUDA(cudaGetLastError());
        return TC_OK;
    }
    DevBuf<T> part;
    tc_status st = part.allocate(mem, nb);
    if (st != TC_OK) return st;
    scan_reduce_kernel<T, In><<<(unsigned)nb, kScanThreads, 0, s>>>(n, in, part.p);
    if (launches) *launches += 1;
    TC_CUDA(cudaGetLastError());
    // scan the per-block partials in place (recursive)
    st = scan_exclusive<T>(mem, nb, ArrayIn<T>{part.p}, ArrayOutExcl<T>{part.p}, (T *)nullptr,
                           s, launches);
    if (st != TC_OK) return st;
    scan_down_kernel<T, In, Out><<<(unsigned)nb, kScanThreads, 0, s>>>(n, in, out, part.p,
                                                                        d_total,
                                                                        d_total != nullptr);
    if (launches) *launches += 1;
    TC_CUDA(cudaGetLastError());
    return TC_OK;
}

}  // namespace tc
