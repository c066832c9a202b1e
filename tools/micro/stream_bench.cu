// Standalone: how fast can 384 CTAs each read 2 x ctx x 128 B (the c2 decode KV
// footprint) on this GPU?  Variants: plain 16 B loads, bulk async copies into a
// ring.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_bench stream_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void plain(const uint4* __restrict__ k, const uint4* __restrict__ v, int Smax, int ctx, uint4* out) {
  const uint4* K = k + (size_t)blockIdx.x * Smax * 8;
  const uint4* V = v + (size_t)blockIdx.x * Smax * 8;
  uint32_t acc = 0;
  const int n = ctx * 8;
#pragma unroll 4
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    uint4 a = K[i], b = V[i];
    acc ^= a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w;
  }
  if (acc == 0x12345678u) out[0] = make_uint4(acc, 0, 0, 0);
}

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int NS>
__global__ void bulk(const uint16_t* __restrict__ k, const uint16_t* __restrict__ v, int Smax, int ctx, uint4* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t bar[2 * NS];
  const uint16_t* src[2] = {k + (size_t)blockIdx.x * Smax * 64, v + (size_t)blockIdx.x * Smax * 64};
  const int nblk = (ctx + 63) / 64;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2 * NS; ++i) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  auto issue = [&](int which, int blk) {
    if (blk >= nblk) return;
    const int rows = min(64, ctx - blk * 64), slot = which * NS + blk % NS;
    uint32_t b = su(&bar[slot]);
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(b), "r"(rows * 128));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su(sm + slot * 8192)), "l"(src[which] + (size_t)blk * 64 * 64), "r"(rows * 128), "r"(b) : "memory");
  };
  if (threadIdx.x == 0)
    for (int i = 0; i < NS; ++i) { issue(0, i); issue(1, i); }
  uint32_t acc = 0;
  for (int which = 0; which < 2; ++which)
    for (int blk = 0; blk < nblk; ++blk) {
      const int slot = which * NS + blk % NS;
      uint32_t b = su(&bar[slot]), par = (blk / NS) & 1, done = 0;
      while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(b), "r"(par) : "memory");
      acc ^= reinterpret_cast<const uint32_t*>(sm + slot * 8192)[threadIdx.x];
      __syncthreads();
      if (threadIdx.x == 0) issue(which, blk + NS);
    }
  if (acc == 0x12345678u) out[0] = make_uint4(acc, 0, 0, 0);
}

int main() {
  const int BH = 384, Smax = 512, L = 12;
  uint16_t *k, *v; uint4* out;
  cudaMalloc(&k, (size_t)L * BH * Smax * 128); cudaMalloc(&v, (size_t)L * BH * Smax * 128); cudaMalloc(&out, 64);
  cudaMemset(k, 1, (size_t)L * BH * Smax * 128); cudaMemset(v, 2, (size_t)L * BH * Smax * 128);
  cudaFuncSetAttribute(bulk<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaFuncSetAttribute(bulk<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int ctx : {257, 384, 512}) {
    for (int var = 0; var < 5; ++var) {
      auto run = [&](int l) {
        const uint16_t* kk = k + (size_t)l * BH * Smax * 64; const uint16_t* vv = v + (size_t)l * BH * Smax * 64;
        if (var == 0) plain<<<BH, 256>>>((const uint4*)kk, (const uint4*)vv, Smax, ctx, out);
        if (var == 1) plain<<<BH, 512>>>((const uint4*)kk, (const uint4*)vv, Smax, ctx, out);
        if (var == 2) bulk<4><<<BH, 256, 65536>>>(kk, vv, Smax, ctx, out);
        if (var == 3) bulk<8><<<BH, 256, 131072>>>(kk, vv, Smax, ctx, out);
        if (var == 4) bulk<4><<<BH, 128, 65536>>>(kk, vv, Smax, ctx, out);
      };
      for (int l = 0; l < L; ++l) run(l);
      cudaEventRecord(e0);
      for (int it = 0; it < 4; ++it) for (int l = 0; l < L; ++l) run(l);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double us = ms * 1e3 / (4 * L), bytes = 2.0 * BH * ctx * 128;
      const char* names[] = {"plain256", "plain512", "bulk4", "bulk8", "bulk4_128t"};
      printf("ctx %d %-10s %7.2f us  %6.0f GB/s  err=%s\n", ctx, names[var], us, bytes / us / 1e3,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
