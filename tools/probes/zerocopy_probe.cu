// zerocopy_probe.cu -- can SMs pull expert weights from pinned host memory (zero-copy over
// PCIe) as fast as the copy engine?  A device-driven a6 (serving non-resident experts without
// a host round trip) depends on it.  Measures on one B200: cudaMemcpyAsync H2D of 256 MB vs a
// kernel that copies the same bytes from mapped pinned memory into HBM with 16-byte loads
// (grid x threads x unroll variants), best of 5, CUDA events.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__global__ void zc_copy(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n16) {
  constexpr int U = 8;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n16; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(src + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) __stcs(dst + i + u * stride, v[u]);
  }
  for (; i < n16; i += stride) dst[i] = __ldcs(src + i);
}

int main() {
  const size_t bytes = 256ull << 20;
  void* h;
  void* d;
  cudaHostAlloc(&h, bytes, cudaHostAllocMapped);
  cudaMalloc(&d, bytes);
  memset(h, 1, bytes);
  void* hd;
  cudaHostGetDevicePointer(&hd, h, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9, ms;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  printf("{\"memcpy_h2d_GBps\": %.2f", bytes / (best * 1e-3) / 1e9);
  const int grids[] = {74, 148, 296, 592};
  const int blocks[] = {128, 256, 512};
  for (int g : grids)
    for (int t : blocks) {
      best = 1e9;
      for (int r = 0; r < 5; ++r) {
        cudaEventRecord(a);
        zc_copy<<<g, t>>>((const uint4*)hd, (uint4*)d, bytes / 16);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      printf(", \"zc_%dx%d_GBps\": %.2f", g, t, bytes / (best * 1e-3) / 1e9);
    }
  printf(", \"error\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
