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

// One warp per score row i of matrix z: valid keys j <= i.
__global__ void attn_softmax_kernel(const float* __restrict__ sc, uint16_t* __restrict__ P, int Z, int S) {
  const int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (row >= static_cast<int64_t>(Z) * S) return;
  const int i = static_cast<int>(row % S);
  const float* s = sc + row * S;
  uint16_t* p = P + row * S;
  float mx = -FLT_MAX;
  for (int j = lane; j <= i; j += 32) mx = fmaxf(mx, s[j]);
  mx = wmax(mx);
  float sum = 0.f;
  for (int j = lane; j <= i; j += 32) sum += expf(s[j] - mx);
  sum = wsum(sum);
  const float inv = 1.0f / sum;
  for (int j = lane; j < S; j += 32) p[j] = j <= i ? f2bf_a(expf(s[j] - mx) * inv) : static_cast<uint16_t>(0);
}

// dS_ij = bf16(P_ij (dP_ij - D_i) scale), D_i = sum_j P_ij dP_ij (j <= i); zero above the diagonal.
__global__ void attn_softmax_bwd_kernel(const uint16_t* __restrict__ P, const float* __restrict__ dP,
                                        uint16_t* __restrict__ dS, int Z, int S, float scale) {
  const int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (row >= static_cast<int64_t>(Z) * S) return;
  const int i = static_cast<int>(row % S);
  const uint16_t* p = P + row * S;
  const float* g = dP + row * S;
  uint16_t* o = dS + row * S;
  float D = 0.f;
  for (int j = lane; j <= i; j += 32) D += bf2f_a(p[j]) * g[j];
  D = wsum(D);
  for (int j = lane; j < S; j += 32) o[j] = j <= i ? f2bf_a(bf2f_a(p[j]) * (g[j] - D) * scale) : static_cast<uint16_t>(0);
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
  attn_softmax_kernel<<<static_cast<unsigned>((rows + 7) / 8), 256, 0, AS(s)>>>(scores, static_cast<uint16_t*>(probs), Z, S);
  return AST();
}

extern "C" int rlhf_attn_softmax_bwd(const void* probs, const float* dP, void* dS, int Z, int S, float scale,
                                     rlhf_stream_t s) {
  const int64_t rows = static_cast<int64_t>(Z) * S;
  attn_softmax_bwd_kernel<<<static_cast<unsigned>((rows + 7) / 8), 256, 0, AS(s)>>>(
      static_cast<const uint16_t*>(probs), dP, static_cast<uint16_t*>(dS), Z, S, scale);
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
