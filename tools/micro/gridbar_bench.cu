// Standalone: cost of one grid-wide barrier among 148 persistent CTAs (1 / SM)
// under variants of the fences the decode loop needs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gridbar_bench gridbar_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_rlx(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int VAR>
__global__ void bar_kernel(unsigned* gbar, float* junk, int iters) {
  const int G = gridDim.x;
  for (int it = 0; it < iters; ++it) {
    if (VAR >= 3) junk[(blockIdx.x * blockDim.x + threadIdx.x) + (it & 7) * G * blockDim.x] = it;  // global stores
    if (VAR == 2 || VAR == 3) asm volatile("fence.proxy.async;" ::: "memory");
    if (VAR == 5) asm volatile("fence.proxy.async.global;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      if (VAR != 0 && VAR != 6) __threadfence();
      if (VAR == 6) asm volatile("fence.acq_rel.gpu;" ::: "memory");
      asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(gbar) : "memory");
      const unsigned target = (unsigned)(it + 1) * G;
      if (VAR == 7) {
        while (ld_rlx(gbar) < target) {}
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      } else {
        while (ld_acq(gbar) < target) {}
      }
    }
    __syncthreads();
  }
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* gbar; float* junk;
  cudaMalloc(&gbar, 256); cudaMalloc(&junk, (size_t)sms * 256 * 8 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 2000;
  const char* names[] = {"bare", "threadfence", "+proxy.async(all thr)", "+stores+proxy.async", "+stores",
                         "+stores+proxy.async.global", "fence.acq_rel only", "relaxed poll + fence"};
  for (int v = 0; v < 8; ++v) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(gbar, 0, 4);
      void* args[] = {&gbar, &junk, (void*)&iters};
      void (*k)(unsigned*, float*, int) = nullptr;
      switch (v) { case 0: k = bar_kernel<0>; break; case 1: k = bar_kernel<1>; break; case 2: k = bar_kernel<2>; break;
        case 3: k = bar_kernel<3>; break; case 4: k = bar_kernel<4>; break; case 5: k = bar_kernel<5>; break;
        case 6: k = bar_kernel<6>; break; default: k = bar_kernel<7>; }
      cudaEventRecord(e0);
      cudaLaunchCooperativeKernel((void*)k, sms, 256, args, 0, 0);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (rep) printf("%-28s %6.3f us / barrier  (%s)\n", names[v], ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
