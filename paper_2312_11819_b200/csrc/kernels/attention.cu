// attention.cu — causal softmax (fwd/bwd) over tcgen05-GEMM scores, KV-cache
// store and the HBM-bound decode attention of the Generation stage.
// Probabilities are normalised then rounded to bf16 before P.V (DESIGN.md §3,
// oracle/ppo_oracle.cpp forward_chunk).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cfloat>

#include "launch_util.cuh"
#include "rlhf_kernels.h"

namespace rlhf {

__device__ __forceinline__ float bf2f_a(uint16_t h) { return __uint_as_float(static_cast<uint32_t>(h) << 16); }
__device__ __forceinline__ uint16_t f2bf_a(float f) { return __bfloat16_as_ushort(__float2bfloat16_rn(f)); }

__device__ __forceinline__ float wmax(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float wsum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// One warp per score row i: the causal prefix j <= i is read once into registers
// (float4), max / sum / normalise from registers, bf16 probabilities written for
// the whole row (zeros above the diagonal).  CH = float4 chunks per lane.
template <int CH>
__global__ void attn_softmax_kernel(const float* __restrict__ sc, uint16_t* __restrict__ P, int Z, int S) {
  const int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (row >= static_cast<int64_t>(Z) * S) return;
  const int i = static_cast<int>(row % S);
  const float4* s4 = reinterpret_cast<const float4*>(sc + row * S);
  float4 v[CH];
  float mx = -FLT_MAX;
#pragma unroll
  for (int k = 0; k < CH; ++k) {
    const int j0 = (lane + 32 * k) * 4;
    v[k] = j0 <= i ? s4[lane + 32 * k] : make_float4(-FLT_MAX, -FLT_MAX, -FLT_MAX, -FLT_MAX);
    if (j0 + 1 > i) v[k].y = -FLT_MAX;
    if (j0 + 2 > i) v[k].z = -FLT_MAX;
    if (j0 + 3 > i) v[k].w = -FLT_MAX;
    mx = fmaxf(mx, fmaxf(fmaxf(v[k].x, v[k].y), fmaxf(v[k].z, v[k].w)));
  }
  mx = wmax(mx);
  float sum = 0.f;
#pragma unroll
  for (int k = 0; k < CH; ++k) {
    const int j0 = (lane + 32 * k) * 4;
    v[k].x = j0 <= i ? expf(v[k].x - mx) : 0.f;
    v[k].y = j0 + 1 <= i ? expf(v[k].y - mx) : 0.f;
    v[k].z = j0 + 2 <= i ? expf(v[k].z - mx) : 0.f;
    v[k].w = j0 + 3 <= i ? expf(v[k].w - mx) : 0.f;
    sum += (v[k].x + v[k].y) + (v[k].z + v[k].w);
  }
  sum = wsum(sum);
  const float inv = 1.0f / sum;
  uint2* p2 = reinterpret_cast<uint2*>(P + row * S);
#pragma unroll
  for (int k = 0; k < CH; ++k) {
    const int c = lane + 32 * k;
    if (c * 4 >= S) break;
    p2[c] = make_uint2(f2bf_a(v[k].x * inv) | (static_cast<uint32_t>(f2bf_a(v[k].y * inv)) << 16),
                       f2bf_a(v[k].z * inv) | (static_cast<uint32_t>(f2bf_a(v[k].w * inv)) << 16));
  }
}

// dS_ij = bf16(P_ij (dP_ij - D_i) scale), D_i = sum_j P_ij dP_ij (j <= i); zero above the diagonal.
template <int CH>
__global__ void attn_softmax_bwd_kernel(const uint16_t* __restrict__ P, const float* __restrict__ dP,
                                        uint16_t* __restrict__ dS, int Z, int S, float scale) {
  const int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (row >= static_cast<int64_t>(Z) * S) return;
  const int i = static_cast<int>(row % S);
  const uint2* p2 = reinterpret_cast<const uint2*>(P + row * S);
  const float4* g4 = reinterpret_cast<const float4*>(dP + row * S);
  float pv[CH][4], gv[CH][4];
  float D = 0.f;
#pragma unroll
  for (int k = 0; k < CH; ++k) {
    const int c = lane + 32 * k;
    const int j0 = c * 4;
    if (j0 <= i) {
      const uint2 u = p2[c];
      const float4 g = g4[c];
      pv[k][0] = bf2f_a(static_cast<uint16_t>(u.x & 0xFFFFu)); pv[k][1] = bf2f_a(static_cast<uint16_t>(u.x >> 16));
      pv[k][2] = bf2f_a(static_cast<uint16_t>(u.y & 0xFFFFu)); pv[k][3] = bf2f_a(static_cast<uint16_t>(u.y >> 16));
      gv[k][0] = g.x; gv[k][1] = g.y; gv[k][2] = g.z; gv[k][3] = g.w;
    } else {
#pragma unroll
      for (int t = 0; t < 4; ++t) pv[k][t] = gv[k][t] = 0.f;
    }
#pragma unroll
    for (int t = 0; t < 4; ++t)
      if (j0 + t <= i) D += pv[k][t] * gv[k][t];
  }
  D = wsum(D);
  uint2* o2 = reinterpret_cast<uint2*>(dS + row * S);
#pragma unroll
  for (int k = 0; k < CH; ++k) {
    const int c = lane + 32 * k;
    if (c * 4 >= S) break;
    uint16_t h[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) h[t] = c * 4 + t <= i ? f2bf_a(pv[k][t] * (gv[k][t] - D) * scale) : static_cast<uint16_t>(0);
    o2[c] = make_uint2(h[0] | (static_cast<uint32_t>(h[1]) << 16), h[2] | (static_cast<uint32_t>(h[3]) << 16));
  }
}

// cache[b][h][p][e] <- qkv[(b*T + i)][d + h*hd + e] (k) / [2d + ...] (v)
__global__ void kv_store_kernel(const uint16_t* __restrict__ qkv, int T, int p0, const int* __restrict__ p0_dev, int H,
                                int hd, int Smax, uint16_t* __restrict__ kc, uint16_t* __restrict__ vc, int rows) {
  pdl_entry();
  const int d = H * hd;
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;  // unit: 8 elements
  const int per_row = d / 8;
  if (idx >= static_cast<int64_t>(rows) * per_row) return;
  const int r = static_cast<int>(idx / per_row), c = static_cast<int>(idx % per_row) * 8;
  const int b = r / T, i = r % T;
  const int p = (p0_dev ? *p0_dev : p0) + i;
  const int h = c / hd, e = c % hd;
  const int64_t dst = ((static_cast<int64_t>(b) * H + h) * Smax + p) * hd + e;
  const uint16_t* src = qkv + static_cast<int64_t>(r) * 3 * d;
  *reinterpret_cast<uint4*>(kc + dst) = *reinterpret_cast<const uint4*>(src + d + c);
  *reinterpret_cast<uint4*>(vc + dst) = *reinterpret_cast<const uint4*>(src + 2 * d + c);
}

constexpr int kDecThreads = 256;
constexpr int kDecMaxCtx = 4096;

// One CTA per (sample, head): scores (thread per key, 16B loads), block softmax,
// bf16-rounded probabilities, then P.V with (dim, key-group) thread split.
template <int HD>
__global__ void __launch_bounds__(kDecThreads) attn_decode_kernel(const uint16_t* __restrict__ qkv, int H, int Smax,
                                                                  const uint16_t* __restrict__ kc,
                                                                  const uint16_t* __restrict__ vc,
                                                                  const int* __restrict__ pos_dev,
                                                                  uint16_t* __restrict__ out) {
  __shared__ float q[HD];
  __shared__ float sc[kDecMaxCtx];
  __shared__ float red[kDecThreads / 32];
  pdl_entry();
  const int bh = blockIdx.x, b = bh / H, h = bh % H;
  const int d = H * HD;
  const int ctx = *pos_dev + 1;
  const float scale = rsqrtf(static_cast<float>(HD));
  const uint16_t* qsrc = qkv + static_cast<int64_t>(b) * 3 * d + h * HD;
  for (int e = threadIdx.x; e < HD; e += kDecThreads) q[e] = bf2f_a(qsrc[e]);
  __syncthreads();
  const uint16_t* K = kc + static_cast<int64_t>(bh) * Smax * HD;
  const uint16_t* V = vc + static_cast<int64_t>(bh) * Smax * HD;
  float mx = -FLT_MAX;
  for (int j = threadIdx.x; j < ctx; j += kDecThreads) {
    const uint4* kr = reinterpret_cast<const uint4*>(K + static_cast<int64_t>(j) * HD);
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < HD / 8; ++c) {
      const uint4 u = kr[c];
      const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        s += q[c * 8 + 2 * t] * bf2f_a(static_cast<uint16_t>(w[t] & 0xFFFFu));
        s += q[c * 8 + 2 * t + 1] * bf2f_a(static_cast<uint16_t>(w[t] >> 16));
      }
    }
    s *= scale;
    sc[j] = s;
    mx = fmaxf(mx, s);
  }
  mx = wmax(mx);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x / 32] = mx;
  __syncthreads();
  mx = red[0];
#pragma unroll
  for (int w = 1; w < kDecThreads / 32; ++w) mx = fmaxf(mx, red[w]);
  __syncthreads();
  float sum = 0.f;
  for (int j = threadIdx.x; j < ctx; j += kDecThreads) {
    const float e = expf(sc[j] - mx);
    sc[j] = e;
    sum += e;
  }
  sum = wsum(sum);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x / 32] = sum;
  __syncthreads();
  sum = 0.f;
#pragma unroll
  for (int w = 0; w < kDecThreads / 32; ++w) sum += red[w];
  const float inv = 1.0f / sum;
  // O[e] = sum_j bf16(p_j) V[j][e]: thread = (16-byte dim chunk c, key group g);
  // a warp reads whole contiguous V rows (coalesced 16B vectors).
  constexpr int CH = HD / 8;              // 16-byte chunks per row
  constexpr int G = kDecThreads / CH;     // key groups
  const int c = threadIdx.x % CH, grp = threadIdx.x / CH;
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
  for (int j = grp; j < ctx; j += G) {
    const float pj = bf2f_a(f2bf_a(sc[j] * inv));
    const uint4 u = *reinterpret_cast<const uint4*>(V + static_cast<int64_t>(j) * HD + c * 8);
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      acc[2 * t] += pj * bf2f_a(static_cast<uint16_t>(w[t] & 0xFFFFu));
      acc[2 * t + 1] += pj * bf2f_a(static_cast<uint16_t>(w[t] >> 16));
    }
  }
  float* part = sc;  // scores no longer needed: reuse as [G][HD] partials
  __syncthreads();
#pragma unroll
  for (int t = 0; t < 8; ++t) part[grp * HD + c * 8 + t] = acc[t];
  __syncthreads();
  for (int e = threadIdx.x; e < HD; e += kDecThreads) {
    float o = 0.f;
    for (int g2 = 0; g2 < G; ++g2) o += part[g2 * HD + e];
    out[static_cast<int64_t>(b) * d + h * HD + e] = f2bf_a(o);
  }
}

}  // namespace rlhf

using namespace rlhf;

static inline cudaStream_t AS(rlhf_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }
static inline int AST() { return cudaGetLastError() == cudaSuccess ? 0 : 5; }

extern "C" int rlhf_attn_softmax(const float* scores, void* probs, int Z, int S, rlhf_stream_t s) {
  const int64_t rows = static_cast<int64_t>(Z) * S;
  if (S % 4) return 2;
  const unsigned g = static_cast<unsigned>((rows + 7) / 8);
  auto* p = static_cast<uint16_t*>(probs);
  if (S <= 128) attn_softmax_kernel<1><<<g, 256, 0, AS(s)>>>(scores, p, Z, S);
  else if (S <= 512) attn_softmax_kernel<4><<<g, 256, 0, AS(s)>>>(scores, p, Z, S);
  else if (S <= 1536) attn_softmax_kernel<12><<<g, 256, 0, AS(s)>>>(scores, p, Z, S);
  else return 2;
  return AST();
}

extern "C" int rlhf_attn_softmax_bwd(const void* probs, const float* dP, void* dS, int Z, int S, float scale,
                                     rlhf_stream_t s) {
  const int64_t rows = static_cast<int64_t>(Z) * S;
  if (S % 4) return 2;
  const unsigned g = static_cast<unsigned>((rows + 7) / 8);
  const auto* p = static_cast<const uint16_t*>(probs);
  auto* o = static_cast<uint16_t*>(dS);
  if (S <= 128) attn_softmax_bwd_kernel<1><<<g, 256, 0, AS(s)>>>(p, dP, o, Z, S, scale);
  else if (S <= 512) attn_softmax_bwd_kernel<4><<<g, 256, 0, AS(s)>>>(p, dP, o, Z, S, scale);
  else if (S <= 1536) attn_softmax_bwd_kernel<12><<<g, 256, 0, AS(s)>>>(p, dP, o, Z, S, scale);
  else return 2;
  return AST();
}

extern "C" int rlhf_kv_store(const void* qkv, int B, int T, int p0, const int* p0_dev, int H, int hd, int Smax,
                             void* kcache, void* vcache, rlhf_stream_t s) {
  if (hd % 8) return 2;
  const int rows = B * T;
  const int64_t n = static_cast<int64_t>(rows) * (H * hd / 8);
  return launch_k(kv_store_kernel, dim3(static_cast<unsigned>((n + 255) / 256)), dim3(256), 0, AS(s),
                  static_cast<const uint16_t*>(qkv), T, p0, p0_dev, H, hd, Smax, static_cast<uint16_t*>(kcache),
                  static_cast<uint16_t*>(vcache), rows);
}

extern "C" int rlhf_attn_decode(const void* qkv, int B, int H, int hd, int Smax, const void* kcache, const void* vcache,
                                const int* pos_dev, void* out, rlhf_stream_t s) {
  if (Smax > kDecMaxCtx) return 2;
  const auto* q = static_cast<const uint16_t*>(qkv);
  const auto* k = static_cast<const uint16_t*>(kcache);
  const auto* v = static_cast<const uint16_t*>(vcache);
  auto* o = static_cast<uint16_t*>(out);
  switch (hd) {
    case 64: return launch_k(attn_decode_kernel<64>, dim3(B * H), dim3(kDecThreads), 0, AS(s), q, H, Smax, k, v, pos_dev, o);
    case 128: return launch_k(attn_decode_kernel<128>, dim3(B * H), dim3(kDecThreads), 0, AS(s), q, H, Smax, k, v, pos_dev, o);
    default: return 2;
  }
}
