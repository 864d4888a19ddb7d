// microbenchmark: random global atomics (counting-sort cost model for a1)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k_hist(const uint32_t* keys, size_t m, uint32_t* cnt) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < m; i += (size_t)gridDim.x * blockDim.x)
    atomicAdd(&cnt[keys[i]], 1u);
}
__global__ void k_scatter(const uint32_t* keys, size_t m, uint32_t* cur, uint32_t* out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < m; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t p = atomicAdd(&cur[keys[i]], 1u);
    out[p % m] = (uint32_t)i;
  }
}
__global__ void k_gen(uint32_t* keys, size_t m, uint32_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < m; i += (size_t)gridDim.x * blockDim.x) {
    uint64_t x = i * 0x9E3779B97F4A7C15ull; x ^= x >> 29; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 32;
    keys[i] = (uint32_t)(x % n);
  }
}
int main() {
  size_t m = 33037896; uint32_t n = 3774768;
  uint32_t *keys, *cnt, *out; cudaMalloc(&keys, m*4); cudaMalloc(&cnt, n*4); cudaMalloc(&out, m*4);
  k_gen<<<2048,256>>>(keys, m, n);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); float t;
  for (int r = 0; r < 3; r++) {
    cudaMemset(cnt, 0, n*4);
    cudaEventRecord(a); k_hist<<<148*16,256>>>(keys, m, cnt); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&t, a, b); printf("hist (RED) %.1f us\n", t*1e3);
    cudaMemset(cnt, 0, n*4);
    cudaEventRecord(a); k_scatter<<<148*16,256>>>(keys, m, cnt, out); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&t, a, b); printf("scatter (ATOM+store) %.1f us\n", t*1e3);
  }
  return 0;
}
