// L2 residency microbenchmark: write G bytes (gray-like, plain stores), stream R bytes with
// evict_first (RGB-like, TMA-free ld.global with cache hint), then read G back; report
// read-back time vs a cold read of G.  Answers: does plain-stored data survive an
// evict_first stream of R bytes in the 126 MB L2?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void write_k(uint4* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_uint4(i, i + 1, i + 2, i + 3);
}
__global__ void stream_k(const uint4* p, size_t n, unsigned* sink, int mode) {
  uint64_t pol;
  if (mode == 1) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  unsigned acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v;
    asm volatile("ld.global.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p + i), "l"(pol));
    acc ^= v.x ^ v.w;
  }
  if (acc == 0x12345678) *sink = acc;
}
__global__ void read_k(const uint4* p, size_t n, unsigned* sink) {
  unsigned acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = __ldcs(p + i);
    acc ^= v.x ^ v.w;
  }
  if (acc == 0x12345678) *sink = acc;
}
int main() {
  const size_t G = 33u << 20, R = 72u << 20, F = 512u << 20;
  uint4 *g, *r, *f; unsigned* sink;
  cudaMalloc(&g, G); cudaMalloc(&r, R); cudaMalloc(&f, F); cudaMalloc(&sink, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int grid = 148 * 8, blk = 256;
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      read_k<<<grid, blk>>>(f, F / 16, sink);               // flush L2
      write_k<<<grid, blk>>>(g, G / 16);
      if (mode > 0) stream_k<<<grid, blk>>>(r, R / 16, sink, mode);   // 1: evict_first, 2: evict_normal
      cudaEventRecord(a);
      read_k<<<grid, blk>>>(g, G / 16, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (rep == 2) printf("mode %d (%s): read-back of 33 MB %.1f us = %.0f GB/s\n", mode,
                           mode == 0 ? "no stream" : mode == 1 ? "72MB evict_first stream" : "72MB normal stream",
                           ms * 1e3, G / (ms * 1e-3) / 1e9);
    }
  }
  // cold read
  read_k<<<grid, blk>>>(f, F / 16, sink);
  cudaEventRecord(a); read_k<<<grid, blk>>>(g, G / 16, sink); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("cold read of 33 MB %.1f us = %.0f GB/s\n", ms * 1e3, G / (ms * 1e-3) / 1e9);
  return 0;
}
