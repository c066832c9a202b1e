// Standalone: streaming rate of the decode loop's smem pool mechanism.
// 148 CTAs (1/SM), one producer thread issuing cp.async.bulk of CH-byte chunks
// into a ring of NS slots; consumer warps wait on full[slot], touch the data,
// bar.sync, one thread arrives on empty[slot].  Bytes per CTA = NCH * CH.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pool_bench pool_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t par) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(su(b)), "r"(par) : "memory");
}

__global__ void pool_kernel(const uint8_t* __restrict__ src, int ns, int ch, int nch, int stride_chunks, uint4* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t full[32], empty[32];
  if (threadIdx.x == 0) {
    for (int i = 0; i < ns; ++i) {
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su(&full[i])));
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su(&empty[i])));
    }
  }
  __syncthreads();
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    if (threadIdx.x == 0) {
      for (int it = 0; it < nch; ++it) {
        const int st = it % ns;
        if (it >= ns) wait(&empty[st], ((it / ns) - 1) & 1);
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su(&full[st])), "r"(ch));
        const uint8_t* g = src + ((size_t)it * stride_chunks * gridDim.x + blockIdx.x) * ch;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         su(sm + st * ch)), "l"(g), "r"(ch), "r"(su(&full[st])) : "memory");
      }
    }
  } else {
    uint32_t acc = 0;
    for (int it = 0; it < nch; ++it) {
      const int st = it % ns;
      wait(&full[st], (it / ns) & 1);
      acc ^= reinterpret_cast<const uint32_t*>(sm + st * ch)[threadIdx.x];
      asm volatile("bar.sync 1, %0;" ::"r"(blockDim.x - 32));
      if (threadIdx.x == 32) asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(su(&empty[st])) : "memory");
    }
    if (acc == 0x12345u) out[0] = make_uint4(acc, 0, 0, 0);
  }
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t total = (size_t)2 << 30;
  uint8_t* src; uint4* out;
  cudaMalloc(&src, total); cudaMalloc(&out, 64); cudaMemset(src, 1, total);
  cudaFuncSetAttribute(pool_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  struct { int ns, ch, nch; } cfgs[] = {{4, 16384, 24}, {8, 16384, 24}, {11, 16384, 24}, {11, 16384, 96},
                                        {6, 32768, 48}, {22, 8192, 96}, {11, 16384, 384}};
  for (auto c : cfgs) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      pool_kernel<<<sms, 288, c.ns * c.ch>>>(src, c.ns, c.ch, c.nch, 1, out);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double bytes = (double)sms * c.nch * c.ch;
      if (rep == 2) printf("ns %2d chunk %5d chunks/CTA %4d: %8.2f us  %7.0f GB/s (%s)\n", c.ns, c.ch, c.nch, ms * 1e3,
                           bytes / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
