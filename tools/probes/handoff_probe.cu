// handoff_probe.cu -- what a kernel boundary costs on the layer-step's critical path, versus
// an in-kernel grid barrier (the only thing a persistent single-launch step, would
// replace it with).  Measures, with %globaltimer, on one B200:
//   (a) PDL:  kernel A (148 CTAs x 192 threads, each stores 4 KB and exits) -> kernel B
//             launched with programmatic stream serialization; B's CTAs are resident early and
//             time the return of griddepcontrol.wait.  latency = B's earliest return - A's
//             last CTA exit stamp.
//   (b) grid barrier: one kernel of 148 CTAs; after the same stores, every CTA does a
//             release arrival on a counter (after __syncthreads) and spins (acquire) until it
//             reaches the grid size.  latency = earliest release - last arrival stamp.
// Each is repeated 200 times; medians are printed.  Build: nvcc -O3 -gencode
// arch=compute_100a,code=sm_100a handoff_probe.cu -o handoff_probe
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdio>
#include <vector>

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(192) kernel_a(float* buf, unsigned long long* stamp) {
  buf[(size_t)blockIdx.x * 1024 + threadIdx.x] = (float)threadIdx.x;  // some global stores
  buf[(size_t)blockIdx.x * 1024 + 512 + threadIdx.x] = 1.f;
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(stamp, gtime());  // last exit
}

__global__ void __launch_bounds__(192) kernel_b(const float* buf, unsigned long long* stamp) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const unsigned long long t = gtime();
  if (threadIdx.x == 0) atomicMin(stamp + 1, t);
  if (threadIdx.x == 0) atomicMax(stamp + 2, t);
  if (buf[(size_t)blockIdx.x * 1024] < -1.f) stamp[3] = 1;  // keep the load
}

__global__ void __launch_bounds__(192) kernel_bar(float* buf, int* ctr, unsigned long long* stamp,
                                                 int target) {
  buf[(size_t)blockIdx.x * 1024 + threadIdx.x] = (float)threadIdx.x;
  buf[(size_t)blockIdx.x * 1024 + 512 + threadIdx.x] = 1.f;
  __syncthreads();
  __shared__ int s_go;
  if (threadIdx.x == 0) {
    atomicMax(stamp, gtime());
    asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(ctr) : "memory");
    int v;
    do {
      asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    } while (v < target);
    const unsigned long long t = gtime();
    atomicMin(stamp + 1, t);
    atomicMax(stamp + 2, t);
    s_go = 1;
  }
  __syncthreads();
  if (s_go && buf[(size_t)((blockIdx.x + 1) % gridDim.x) * 1024] < -1.f) stamp[3] = 1;
}

static double median(std::vector<double> v) {
  std::sort(v.begin(), v.end());
  return v[v.size() / 2];
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* buf;
  int* ctr;
  unsigned long long* st;
  cudaMalloc(&buf, sizeof(float) * 1024 * sms);
  cudaMalloc(&ctr, sizeof(int));
  cudaMalloc(&st, sizeof(unsigned long long) * 4);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  std::vector<double> pdl_first, pdl_last, bar_first, bar_last;
  const unsigned long long init[4] = {0ull, ~0ull, 0ull, 0ull};
  for (int rep = 0; rep < 220; ++rep) {
    cudaMemcpyAsync(st, init, sizeof(init), cudaMemcpyHostToDevice, s);
    kernel_a<<<sms, 192, 0, s>>>(buf, st);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(sms);
    cfg.blockDim = dim3(192);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kernel_b, (const float*)buf, st);
    unsigned long long h[4];
    cudaMemcpyAsync(h, st, sizeof(h), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    if (rep >= 20) {
      pdl_first.push_back((double)(h[1] - h[0]) / 1e3);
      pdl_last.push_back((double)(h[2] - h[0]) / 1e3);
    }
    cudaMemcpyAsync(st, init, sizeof(init), cudaMemcpyHostToDevice, s);
    cudaMemsetAsync(ctr, 0, sizeof(int), s);
    kernel_bar<<<sms, 192, 0, s>>>(buf, ctr, st, sms);
    cudaMemcpyAsync(h, st, sizeof(h), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    if (rep >= 20) {
      bar_first.push_back((double)(h[1] - h[0]) / 1e3);
      bar_last.push_back((double)(h[2] - h[0]) / 1e3);
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("{\"sms\": %d, \"reps\": %zu, \"error\": \"%s\",\n", sms, pdl_first.size(), cudaGetErrorString(e));
  printf(" \"pdl_wait_return_after_last_exit_us\": {\"first_cta\": %.3f, \"last_cta\": %.3f},\n",
         median(pdl_first), median(pdl_last));
  printf(" \"grid_barrier_release_after_last_arrival_us\": {\"first_cta\": %.3f, \"last_cta\": %.3f}}\n",
         median(bar_first), median(bar_last));
  return 0;
}
