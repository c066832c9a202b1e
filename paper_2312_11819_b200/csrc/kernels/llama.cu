// llama.cu — the element kernels of the LLaMA family (rlhf_arch.family == 1) that the
// OPT path does not have: rotary position embedding of q / k (forward, fused with the
// KV-cache store for generation, and its transpose for backward) and the SwiGLU gate
// (forward and backward).  RMSNorm shares rowwise.cu's LayerNorm kernels (RMS template
// flag).  All HBM-bound; 16-byte accesses, one thread per 8 (or 4+4) elements.
// Rounding (oracle/ppo_oracle.cpp): inputs bf16, math fp32, outputs bf16.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "launch_util.cuh"
#include "rlhf_kernels.h"

namespace rlhf {
namespace {

__device__ __forceinline__ float lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float hi(uint32_t u) { return __uint_as_float(u & 0xFFFF0000u); }
__device__ __forceinline__ uint32_t pack(float a, float b) {
  return static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(a))) |
         (static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(b))) << 16);
}
inline cudaStream_t S(rlhf_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

// Rotate 4 pairs (x[i], x[i + hd/2]) held as two uint2 (4 bf16 each) by the table's
// (cos, sin); inverse = transpose (backward).
__device__ __forceinline__ void rot4(uint2& a, uint2& b, const float2* cs, bool inverse) {
  const float sg = inverse ? -1.f : 1.f;
  float x0[4] = {lo(a.x), hi(a.x), lo(a.y), hi(a.y)};
  float x1[4] = {lo(b.x), hi(b.x), lo(b.y), hi(b.y)};
  float y0[4], y1[4];
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const float c = cs[t].x, s = sg * cs[t].y;
    y0[t] = x0[t] * c - x1[t] * s;
    y1[t] = x1[t] * c + x0[t] * s;
  }
  a = make_uint2(pack(y0[0], y0[1]), pack(y0[2], y0[3]));
  b = make_uint2(pack(y1[0], y1[1]), pack(y1[2], y1[3]));
}

// One thread per (row, head, group of 4 rotary pairs): q and k of the packed qkv row are
// rotated in place; with a cache, the rotated k and the v of the same 8 elements are
// stored at position p of (b, h) — the generation path's KV-cache write.
__global__ void rope_qkv_kernel(uint16_t* __restrict__ qkv, int T, int p0, const int* __restrict__ p0_dev, int H, int hd,
                                const float2* __restrict__ table, int inverse, uint16_t* __restrict__ kc,
                                uint16_t* __restrict__ vc, int Smax, int rows) {
  pdl_entry();
  const int half = hd / 2, groups = half / 4, d = H * hd;
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<int64_t>(rows) * H * groups) return;
  const int g = static_cast<int>(idx % groups);
  const int h = static_cast<int>((idx / groups) % H);
  const int r = static_cast<int>(idx / (static_cast<int64_t>(groups) * H));
  const int b = r / T, i = r % T;
  const int p = (p0_dev ? *p0_dev : p0) + i;
  float2 cs[4];
#pragma unroll
  for (int t = 0; t < 4; ++t) cs[t] = table[static_cast<int64_t>(p) * half + g * 4 + t];
  uint16_t* row = qkv + static_cast<int64_t>(r) * 3 * d + h * hd + g * 4;
  uint2 q0 = *reinterpret_cast<const uint2*>(row), q1 = *reinterpret_cast<const uint2*>(row + half);
  uint2 k0 = *reinterpret_cast<const uint2*>(row + d), k1 = *reinterpret_cast<const uint2*>(row + d + half);
  rot4(q0, q1, cs, inverse);
  rot4(k0, k1, cs, inverse);
  *reinterpret_cast<uint2*>(row) = q0;
  *reinterpret_cast<uint2*>(row + half) = q1;
  *reinterpret_cast<uint2*>(row + d) = k0;
  *reinterpret_cast<uint2*>(row + d + half) = k1;
  if (kc) {
    const int64_t dst = ((static_cast<int64_t>(b) * H + h) * Smax + p) * hd + g * 4;
    *reinterpret_cast<uint2*>(kc + dst) = k0;
    *reinterpret_cast<uint2*>(kc + dst + half) = k1;
    *reinterpret_cast<uint2*>(vc + dst) = *reinterpret_cast<const uint2*>(row + 2 * d);
    *reinterpret_cast<uint2*>(vc + dst + half) = *reinterpret_cast<const uint2*>(row + 2 * d + half);
  }
}

__device__ __forceinline__ float sigm(float g) { return 1.0f / (1.0f + expf(-g)); }

// act[r, j] = bf16(silu(gate) * up) with gu[r] = [gate (ff) | up (ff)]; 8 columns per thread.
__global__ void swiglu_kernel(const uint16_t* __restrict__ gu, uint16_t* __restrict__ act, int ff, int rows) {
  pdl_entry();
  const int per = ff / 8;
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<int64_t>(rows) * per) return;
  const int64_t r = idx / per;
  const int c = static_cast<int>(idx % per) * 8;
  const uint4 G = *reinterpret_cast<const uint4*>(gu + r * 2 * ff + c);
  const uint4 U = *reinterpret_cast<const uint4*>(gu + r * 2 * ff + ff + c);
  const uint32_t gw[4] = {G.x, G.y, G.z, G.w}, uw[4] = {U.x, U.y, U.z, U.w};
  uint32_t o[4];
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const float g0 = lo(gw[t]), g1 = hi(gw[t]);
    o[t] = pack(g0 * sigm(g0) * lo(uw[t]), g1 * sigm(g1) * hi(uw[t]));
  }
  *reinterpret_cast<uint4*>(act + r * ff + c) = make_uint4(o[0], o[1], o[2], o[3]);
}

// dgu[r] = [d gate | d up]: dgate = dact * up * s * (1 + g (1 - s)), dup = dact * g * s.
__global__ void swiglu_bwd_kernel(const uint16_t* __restrict__ gu, const uint16_t* __restrict__ dact,
                                  uint16_t* __restrict__ dgu, int ff, int rows) {
  const int per = ff / 8;
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<int64_t>(rows) * per) return;
  const int64_t r = idx / per;
  const int c = static_cast<int>(idx % per) * 8;
  const uint4 G = *reinterpret_cast<const uint4*>(gu + r * 2 * ff + c);
  const uint4 U = *reinterpret_cast<const uint4*>(gu + r * 2 * ff + ff + c);
  const uint4 D = *reinterpret_cast<const uint4*>(dact + r * ff + c);
  const uint32_t gw[4] = {G.x, G.y, G.z, G.w}, uw[4] = {U.x, U.y, U.z, U.w}, dw[4] = {D.x, D.y, D.z, D.w};
  uint32_t og[4], ou[4];
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    float dg[2], du[2];
    const float gg[2] = {lo(gw[t]), hi(gw[t])}, uu[2] = {lo(uw[t]), hi(uw[t])}, dd[2] = {lo(dw[t]), hi(dw[t])};
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const float s = sigm(gg[e]);
      dg[e] = dd[e] * uu[e] * s * (1.0f + gg[e] * (1.0f - s));
      du[e] = dd[e] * gg[e] * s;
    }
    og[t] = pack(dg[0], dg[1]);
    ou[t] = pack(du[0], du[1]);
  }
  *reinterpret_cast<uint4*>(dgu + r * 2 * ff + c) = make_uint4(og[0], og[1], og[2], og[3]);
  *reinterpret_cast<uint4*>(dgu + r * 2 * ff + ff + c) = make_uint4(ou[0], ou[1], ou[2], ou[3]);
}

}  // namespace
}  // namespace rlhf

using namespace rlhf;

extern "C" int rlhf_rope_qkv(void* qkv, int B, int T, int p0, const int* p0_dev, int H, int hd, const float* table,
                             int inverse, void* kcache, void* vcache, int Smax, rlhf_stream_t s) {
  if (hd % 8 || !table || (kcache && !vcache)) return 2;
  const int rows = B * T;
  const int64_t n = static_cast<int64_t>(rows) * H * (hd / 8);
  if (n == 0) return 0;
  return launch_k(rope_qkv_kernel, dim3(static_cast<unsigned>((n + 255) / 256)), dim3(256), 0, S(s),
                  static_cast<uint16_t*>(qkv), T, p0, p0_dev, H, hd, reinterpret_cast<const float2*>(table), inverse,
                  static_cast<uint16_t*>(kcache), static_cast<uint16_t*>(vcache), Smax, rows);
}

extern "C" int rlhf_swiglu(const void* gu, void* act, int rows, int ff, rlhf_stream_t s) {
  if (ff % 8) return 2;
  const int64_t n = static_cast<int64_t>(rows) * (ff / 8);
  if (n == 0) return 0;
  return launch_k(swiglu_kernel, dim3(static_cast<unsigned>((n + 255) / 256)), dim3(256), 0, S(s),
                  static_cast<const uint16_t*>(gu), static_cast<uint16_t*>(act), ff, rows);
}

extern "C" int rlhf_swiglu_bwd(const void* gu, const void* dact, void* dgu, int rows, int ff, rlhf_stream_t s) {
  if (ff % 8) return 2;
  const int64_t n = static_cast<int64_t>(rows) * (ff / 8);
  if (n == 0) return 0;
  swiglu_bwd_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, S(s)>>>(
      static_cast<const uint16_t*>(gu), static_cast<const uint16_t*>(dact), static_cast<uint16_t*>(dgu), ff, rows);
  return cudaGetLastError() == cudaSuccess ? 0 : 5;
}
