// rowwise.cu — HBM-bound row / element kernels of the PPO step: embedding
// (fwd + scatter-add bwd), LayerNorm (fwd + bwd), bf16 rounding, bias-gradient
// column sums, response-row gather/scatter, fused AdamW.
// All follow the rounding contract in DESIGN.md §3 (mirrored by oracle/ppo_oracle.cpp).
#include <cfloat>
#include <cstdlib>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "launch_util.cuh"
#include "rlhf_kernels.h"

namespace rlhf {

__device__ __forceinline__ float bf2f(uint16_t h) { return __uint_as_float(static_cast<uint32_t>(h) << 16); }
__device__ __forceinline__ uint16_t f2bf(float f) { return __bfloat16_as_ushort(__float2bfloat16_rn(f)); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

static inline int cuda_status() { return cudaGetLastError() == cudaSuccess ? 0 : 5; }
static inline cudaStream_t S(rlhf_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

// x[r] = E[tok] + Pm[p]; one thread per (row, 4 columns).
__global__ void embed_kernel(const int32_t* __restrict__ tokens, int64_t tok_stride, int T, int p0,
                             const int* __restrict__ p0_dev, const uint16_t* __restrict__ E,
                             const uint16_t* __restrict__ Pm, int d, float* __restrict__ x, int rows) {
  pdl_entry();
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int qd = d / 4;
  if (idx >= static_cast<int64_t>(rows) * qd) return;
  const int r = static_cast<int>(idx / qd), c = static_cast<int>(idx % qd) * 4;
  const int b = r / T, i = r % T;
  const int p = (p0_dev ? *p0_dev : p0) + i;
  const int id = tokens[b * tok_stride + p];
  const uint2 e = *reinterpret_cast<const uint2*>(E + static_cast<int64_t>(id) * d + c);
  const uint2 q = Pm ? *reinterpret_cast<const uint2*>(Pm + static_cast<int64_t>(p) * d + c) : make_uint2(0u, 0u);
  float4 o;
  o.x = bf2f(e.x & 0xFFFFu) + bf2f(q.x & 0xFFFFu);
  o.y = bf2f(e.x >> 16) + bf2f(q.x >> 16);
  o.z = bf2f(e.y & 0xFFFFu) + bf2f(q.y & 0xFFFFu);
  o.w = bf2f(e.y >> 16) + bf2f(q.y >> 16);
  *reinterpret_cast<float4*>(x + static_cast<int64_t>(r) * d + c) = o;
}

__global__ void embed_bwd_kernel(const int32_t* __restrict__ tokens, int64_t tok_stride, int T,
                                 const float* __restrict__ dx, int d, float* __restrict__ dE, float* __restrict__ dP,
                                 int rows) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<int64_t>(rows) * d) return;
  const int r = static_cast<int>(idx / d), c = static_cast<int>(idx % d);
  const int b = r / T, i = r % T;
  const int id = tokens[b * tok_stride + i];
  const float g = dx[idx];
  atomicAdd(dE + static_cast<int64_t>(id) * d + c, g);
  if (dP) atomicAdd(dP + static_cast<int64_t>(i) * d + c, g);
}

// Decode step entry: x[b] = tok_emb[tokens[b*stride + *pos]] + pos_emb[*pos] (fp32, the
// residual stream) and y[b] = bf16(LN1_layer0(x[b])), one warp per sample.  Waits on its
// predecessor before triggering dependents (the step chain relies on it, see attention.cu).
//
// Fused greedy sampler (t2 != null): the previous step's LM-head per-tile top-2 partials
// t2 [tiles][B] are merged first (the argmax_tiles_kernel reduction: max, ties -> lowest
// id, second max -- order-independent, so the same token and margin), written to
// dst[b*stride + *pos + 1] / margin, *pos advanced by one, and the step then embeds position
// *pos + 1: the merged token itself (dst == tokens, free-running) or tokens[...] (teacher
// forcing, dst = predictions).  The position is advanced BEFORE dependents are triggered
// (per-CTA ticket right after the wait; the last CTA writes it): later kernels of the step
// read *pos before their own griddepcontrol.wait.
__device__ __forceinline__ void top2_fold(float& v1, int& i1, float& v2, float bv1, int bi1, float bv2) {
  if (bv1 > v1 || (bv1 == v1 && bi1 < i1)) {
    v2 = fmaxf(v1, bv2);
    v1 = bv1;
    i1 = bi1;
  } else {
    v2 = fmaxf(v2, bv1);
  }
}

template <int VPL, bool RMS>
__global__ void embed_ln_kernel(const int32_t* __restrict__ tokens, int64_t tok_stride, const int* __restrict__ pos_dev,
                                const uint16_t* __restrict__ E, const uint16_t* __restrict__ Pm, int d,
                                float* __restrict__ x, const uint16_t* __restrict__ g, const uint16_t* __restrict__ bta,
                                uint16_t* __restrict__ y, int B, const float4* __restrict__ t2, int tiles,
                                int32_t* __restrict__ dst, float* __restrict__ margin) {
  const int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  int p = *pos_dev;
  if (t2) {
    __syncthreads();  // every thread of this CTA has read *pos
    if (threadIdx.x == 0) {
      __threadfence();
      unsigned* ticket = reinterpret_cast<unsigned*>(const_cast<int*>(pos_dev) + 1);
      if (atomicAdd(ticket, 1u) == gridDim.x - 1) {
        *ticket = 0u;
        *const_cast<int*>(pos_dev) = p + 1;
        __threadfence();
      }
    }
    __syncthreads();
  }
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (row >= B) return;
  int id;
  if (t2) {
    float v1 = -FLT_MAX, v2 = -FLT_MAX;
    int i1 = 0x7fffffff;
    // 8 partial loads in flight per lane, folded in ascending tile order (the same order as
    // one load per iteration; out-of-range slots are neutral (-FLT_MAX, INT_MAX, -FLT_MAX))
    for (int i0 = lane; i0 < tiles; i0 += 32 * 8) {
      float4 o[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int i = i0 + 32 * j;
        o[j] = i < tiles ? t2[static_cast<int64_t>(i) * B + row] : make_float4(-FLT_MAX, __int_as_float(0x7fffffff), -FLT_MAX, 0.f);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) top2_fold(v1, i1, v2, o[j].x, __float_as_int(o[j].y), o[j].z);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const float bv1 = __shfl_xor_sync(0xffffffffu, v1, o), bv2 = __shfl_xor_sync(0xffffffffu, v2, o);
      const int bi1 = __shfl_xor_sync(0xffffffffu, i1, o);
      top2_fold(v1, i1, v2, bv1, bi1, bv2);
    }
    const int64_t at = static_cast<int64_t>(row) * tok_stride + p + 1;
    if (lane == 0) {
      dst[at] = i1;
      if (margin) margin[at] = v1 - v2;
    }
    p += 1;
    id = dst == tokens ? i1 : tokens[at];
  } else {
    id = tokens[static_cast<int64_t>(row) * tok_stride + p];
  }
  const uint2* e2 = reinterpret_cast<const uint2*>(E + static_cast<int64_t>(id) * d);
  const uint2* p2 = reinterpret_cast<const uint2*>(Pm + static_cast<int64_t>(p) * d);
  const uint2* g2 = reinterpret_cast<const uint2*>(g);
  const uint2* b2 = reinterpret_cast<const uint2*>(bta);
  float4* xr = reinterpret_cast<float4*>(x + static_cast<int64_t>(row) * d);
  const int q = d / 4;
  float4 v[VPL];
  uint2 gg[VPL], bb[VPL];
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    const int c = lane + 32 * k;
    if (c < q) {
      const uint2 ev = e2[c], pv = RMS ? make_uint2(0u, 0u) : p2[c];
      v[k] = make_float4(bf2f(ev.x & 0xFFFFu) + bf2f(pv.x & 0xFFFFu), bf2f(ev.x >> 16) + bf2f(pv.x >> 16),
                         bf2f(ev.y & 0xFFFFu) + bf2f(pv.y & 0xFFFFu), bf2f(ev.y >> 16) + bf2f(pv.y >> 16));
      xr[c] = v[k];
      gg[k] = g2[c];
      bb[k] = RMS ? make_uint2(0u, 0u) : b2[c];
    }
  }
  float s = 0.f;
  if (!RMS) {
#pragma unroll
    for (int k = 0; k < VPL; ++k)
      if (lane + 32 * k < q) s += (v[k].x + v[k].y) + (v[k].z + v[k].w);
  }
  const float mu = RMS ? 0.f : warp_sum(s) / d;  // RMSNorm: no centring
  float vs = 0.f;
#pragma unroll
  for (int k = 0; k < VPL; ++k)
    if (lane + 32 * k < q)
      vs += (v[k].x - mu) * (v[k].x - mu) + (v[k].y - mu) * (v[k].y - mu) + (v[k].z - mu) * (v[k].z - mu) +
            (v[k].w - mu) * (v[k].w - mu);
  const float rs = 1.0f / sqrtf(warp_sum(vs) / d + (RMS ? 1e-6f : 1e-5f));
  uint2* yr = reinterpret_cast<uint2*>(y + static_cast<int64_t>(row) * d);
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    const int c = lane + 32 * k;
    if (c >= q) continue;
    const float o0 = (v[k].x - mu) * rs * bf2f(gg[k].x & 0xFFFFu) + bf2f(bb[k].x & 0xFFFFu);
    const float o1 = (v[k].y - mu) * rs * bf2f(gg[k].x >> 16) + bf2f(bb[k].x >> 16);
    const float o2 = (v[k].z - mu) * rs * bf2f(gg[k].y & 0xFFFFu) + bf2f(bb[k].y & 0xFFFFu);
    const float o3 = (v[k].w - mu) * rs * bf2f(gg[k].y >> 16) + bf2f(bb[k].y >> 16);
    yr[c] = make_uint2(f2bf(o0) | (static_cast<uint32_t>(f2bf(o1)) << 16), f2bf(o2) | (static_cast<uint32_t>(f2bf(o3)) << 16));
  }
}

// One warp per row, row held in registers (d <= 4096): a single round trip to
// memory for x, gamma and beta, then two register passes (mean, variance).
template <int VPL, bool RMS>  // float4 vectors per lane; RMS: RMSNorm (no centring, no beta)
__global__ void layernorm_kernel(const float* __restrict__ x, const uint16_t* __restrict__ g,
                                 const uint16_t* __restrict__ bta, uint16_t* __restrict__ y, float* __restrict__ mean,
                                 float* __restrict__ rstd, int M, int d) {
  // gamma / beta are weights: requested before griddepcontrol.wait, only x waits for the
  // predecessor (the dependents are triggered first, as in pdl_entry_early)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  const uint2* g2 = reinterpret_cast<const uint2*>(g);
  const uint2* b2 = reinterpret_cast<const uint2*>(bta);
  const int q = d / 4;
  float4 v[VPL];
  uint2 gg[VPL], bb[VPL];
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    const int c = lane + 32 * k;
    if (c < q) {
      gg[k] = g2[c];
      bb[k] = RMS ? make_uint2(0u, 0u) : b2[c];
    }
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (row >= M) return;
  const float4* xr = reinterpret_cast<const float4*>(x + static_cast<int64_t>(row) * d);
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    const int c = lane + 32 * k;
    if (c < q) v[k] = xr[c];
  }
  float s = 0.f;
  if (!RMS) {
#pragma unroll
    for (int k = 0; k < VPL; ++k)
      if (lane + 32 * k < q) s += (v[k].x + v[k].y) + (v[k].z + v[k].w);
  }
  const float mu = RMS ? 0.f : warp_sum(s) / d;  // RMSNorm: no centring
  float vs = 0.f;
#pragma unroll
  for (int k = 0; k < VPL; ++k)
    if (lane + 32 * k < q)
      vs += (v[k].x - mu) * (v[k].x - mu) + (v[k].y - mu) * (v[k].y - mu) + (v[k].z - mu) * (v[k].z - mu) +
            (v[k].w - mu) * (v[k].w - mu);
  const float rs = 1.0f / sqrtf(warp_sum(vs) / d + (RMS ? 1e-6f : 1e-5f));
  uint2* yr = reinterpret_cast<uint2*>(y + static_cast<int64_t>(row) * d);
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    const int c = lane + 32 * k;
    if (c >= q) continue;
    const float o0 = (v[k].x - mu) * rs * bf2f(gg[k].x & 0xFFFFu) + bf2f(bb[k].x & 0xFFFFu);
    const float o1 = (v[k].y - mu) * rs * bf2f(gg[k].x >> 16) + bf2f(bb[k].x >> 16);
    const float o2 = (v[k].z - mu) * rs * bf2f(gg[k].y & 0xFFFFu) + bf2f(bb[k].y & 0xFFFFu);
    const float o3 = (v[k].w - mu) * rs * bf2f(gg[k].y >> 16) + bf2f(bb[k].y >> 16);
    yr[c] = make_uint2(f2bf(o0) | (static_cast<uint32_t>(f2bf(o1)) << 16), f2bf(o2) | (static_cast<uint32_t>(f2bf(o3)) << 16));
  }
  if (lane == 0) {
    if (mean) mean[row] = mu;
    if (rstd) rstd[row] = rs;
  }
}

constexpr int kLnBwdRows = 64;  // rows per block (8 warps x 8 rows)

// dx += rstd*(dy*g - mean(dy*g) - xhat*mean(dy*g*xhat)).  Each warp keeps its
// rows' dgamma/dbeta column partials in registers (lane owns columns lane+32k),
// the block reduces its 8 warps in smem in fixed order -> ws[blk][2][d].
template <int VPL, bool RMS>  // float4 vectors per lane (d <= 128*VPL); RMS: RMSNorm, dgamma only
__global__ void layernorm_bwd_kernel(const float* __restrict__ dy, const float* __restrict__ x,
                                     const float* __restrict__ mean, const float* __restrict__ rstd,
                                     const uint16_t* __restrict__ g, float* __restrict__ dx, float* __restrict__ ws,
                                     int M, int d) {
  extern __shared__ float red[];  // [8 warps][NP][d]
  constexpr int NP = RMS ? 1 : 2;  // column partials per warp: dgamma (, dbeta)
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int r0 = blockIdx.x * kLnBwdRows;
  const int q = d / 4;
  float4 gg[VPL], pg[VPL], pb[VPL];
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    const int c = lane + 32 * k;
    if (c < q) {
      const uint2 u = reinterpret_cast<const uint2*>(g)[c];
      gg[k] = make_float4(bf2f(u.x & 0xFFFFu), bf2f(u.x >> 16), bf2f(u.y & 0xFFFFu), bf2f(u.y >> 16));
    } else {
      gg[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    pg[k] = pb[k] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  for (int rr = warp; rr < kLnBwdRows; rr += 8) {
    const int row = r0 + rr;
    if (row >= M) break;
    const float4* dr = reinterpret_cast<const float4*>(dy + static_cast<int64_t>(row) * d);
    const float4* xr = reinterpret_cast<const float4*>(x + static_cast<int64_t>(row) * d);
    float4* o = reinterpret_cast<float4*>(dx + static_cast<int64_t>(row) * d);
    const float mu = RMS ? 0.f : mean[row], rs = rstd[row];
    float4 dyv[VPL], xh[VPL], dxo[VPL];
#pragma unroll
    for (int k = 0; k < VPL; ++k) {  // every load of the row in flight at once
      const int c = lane + 32 * k;
      const bool ok = c < q;
      dyv[k] = ok ? dr[c] : make_float4(0.f, 0.f, 0.f, 0.f);
      xh[k] = ok ? xr[c] : make_float4(0.f, 0.f, 0.f, 0.f);
      dxo[k] = ok ? o[c] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    float a = 0.f, cs = 0.f;
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      if (lane + 32 * k >= q) continue;
      xh[k] = make_float4((xh[k].x - mu) * rs, (xh[k].y - mu) * rs, (xh[k].z - mu) * rs, (xh[k].w - mu) * rs);
      const float t0 = dyv[k].x * gg[k].x, t1 = dyv[k].y * gg[k].y, t2 = dyv[k].z * gg[k].z, t3 = dyv[k].w * gg[k].w;
      a += (t0 + t1) + (t2 + t3);
      cs += (t0 * xh[k].x + t1 * xh[k].y) + (t2 * xh[k].z + t3 * xh[k].w);
      pg[k].x += dyv[k].x * xh[k].x; pg[k].y += dyv[k].y * xh[k].y;
      pg[k].z += dyv[k].z * xh[k].z; pg[k].w += dyv[k].w * xh[k].w;
      pb[k].x += dyv[k].x; pb[k].y += dyv[k].y; pb[k].z += dyv[k].z; pb[k].w += dyv[k].w;
    }
    a = RMS ? 0.f : warp_sum(a) / d;
    cs = warp_sum(cs) / d;
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const int c = lane + 32 * k;
      if (c >= q) continue;
      float4 r = dxo[k];
      r.x += rs * (dyv[k].x * gg[k].x - a - xh[k].x * cs);
      r.y += rs * (dyv[k].y * gg[k].y - a - xh[k].y * cs);
      r.z += rs * (dyv[k].z * gg[k].z - a - xh[k].z * cs);
      r.w += rs * (dyv[k].w * gg[k].w - a - xh[k].w * cs);
      o[c] = r;
    }
  }
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    const int c = lane + 32 * k;
    if (c < q) {
      reinterpret_cast<float4*>(red + (warp * NP) * d)[c] = pg[k];
      if (!RMS) reinterpret_cast<float4*>(red + (warp * NP + 1) * d)[c] = pb[k];
    }
  }
  __syncthreads();
  float* wg = ws + static_cast<int64_t>(blockIdx.x) * NP * d;
  for (int j = threadIdx.x; j < NP * d; j += blockDim.x) {
    const int which = j / d, col = j % d;
    float acc = 0.f;
    for (int w = 0; w < 8; ++w) acc += red[(w * NP + which) * d + col];  // fixed warp order
    wg[j] = acc;
  }
}

// Norm backward for wide rows (LayerNorm d = 2048 (OPT-1.3B), RMSNorm d = 2048 / 4096 (LLaMA)):
// a row is split between the two warps of a pair (half the columns each, VPLH float4 per lane),
// so the row arrays stay in registers (the one-warp-per-row kernel spills: 0.7 TB/s at
// d = 4096, 2.1-2.5 TB/s at d = 2048).  The pair exchanges its partial row sums (sum dy*g and,
// for LayerNorm, sum dy*g*xhat) through shared memory (double-buffered slot, named barrier per
// pair, fixed summation order: half 0 then half 1); gamma is staged in shared memory; the
// dgamma (, dbeta) column partials stay in registers per warp half.
template <int VPLH, bool RMS>
__global__ void __launch_bounds__(256) norm_bwd_pair_kernel(const float* __restrict__ dy, const float* __restrict__ x,
                                                            const float* __restrict__ mean, const float* __restrict__ rstd,
                                                            const uint16_t* __restrict__ g, float* __restrict__ dx,
                                                            float* __restrict__ ws, int M, int d, int rpb) {
  constexpr int NP = RMS ? 1 : 2;
  extern __shared__ float red[];  // [8 warps][NP][d] (each warp fills its half), gamma [d], exchange [2][8][2]
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int pair = warp >> 1, half = warp & 1;
  const int q = d / 4, qh = q / 2;
  float4* gs = reinterpret_cast<float4*>(red + 8 * NP * d);
  float* xch = red + (8 * NP + 1) * d;
  for (int c = threadIdx.x; c < q; c += blockDim.x) {
    const uint2 u = reinterpret_cast<const uint2*>(g)[c];
    gs[c] = make_float4(bf2f(u.x & 0xFFFFu), bf2f(u.x >> 16), bf2f(u.y & 0xFFFFu), bf2f(u.y >> 16));
  }
  __syncthreads();
  const int cb = half * qh;
  float4 pg[VPLH], pb[VPLH];
#pragma unroll
  for (int k = 0; k < VPLH; ++k) pg[k] = pb[k] = make_float4(0.f, 0.f, 0.f, 0.f);
  const int r0 = blockIdx.x * rpb;
  int par = 0;
  for (int rr = pair; rr < rpb; rr += 4, par ^= 1) {
    const int row = r0 + rr;
    if (row >= M) break;
    const float4* dr = reinterpret_cast<const float4*>(dy + static_cast<int64_t>(row) * d);
    const float4* xr = reinterpret_cast<const float4*>(x + static_cast<int64_t>(row) * d);
    float4* o = reinterpret_cast<float4*>(dx + static_cast<int64_t>(row) * d);
    const float mu = RMS ? 0.f : mean[row], rs = rstd[row];
    float4 dyv[VPLH], xh[VPLH];
#pragma unroll
    for (int k = 0; k < VPLH; ++k) {
      const int c = cb + lane + 32 * k;
      const bool ok = lane + 32 * k < qh;
      dyv[k] = ok ? dr[c] : make_float4(0.f, 0.f, 0.f, 0.f);
      xh[k] = ok ? xr[c] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    float a = 0.f, cs = 0.f;
#pragma unroll
    for (int k = 0; k < VPLH; ++k) {
      if (lane + 32 * k >= qh) continue;
      const float4 gv = gs[cb + lane + 32 * k];
      xh[k] = make_float4((xh[k].x - mu) * rs, (xh[k].y - mu) * rs, (xh[k].z - mu) * rs, (xh[k].w - mu) * rs);
      const float t0 = dyv[k].x * gv.x, t1 = dyv[k].y * gv.y, t2 = dyv[k].z * gv.z, t3 = dyv[k].w * gv.w;
      if (!RMS) a += (t0 + t1) + (t2 + t3);
      cs += (t0 * xh[k].x + t1 * xh[k].y) + (t2 * xh[k].z + t3 * xh[k].w);
      pg[k].x += dyv[k].x * xh[k].x; pg[k].y += dyv[k].y * xh[k].y;
      pg[k].z += dyv[k].z * xh[k].z; pg[k].w += dyv[k].w * xh[k].w;
      if (!RMS) { pb[k].x += dyv[k].x; pb[k].y += dyv[k].y; pb[k].z += dyv[k].z; pb[k].w += dyv[k].w; }
    }
    cs = warp_sum(cs);
    if (!RMS) a = warp_sum(a);
    if (lane == 0) {
      xch[(par * 8 + warp) * 2] = cs;
      xch[(par * 8 + warp) * 2 + 1] = a;
    }
    asm volatile("bar.sync %0, 64;" ::"r"(1 + pair) : "memory");
    const float* xp = xch + (par * 8 + 2 * pair) * 2;
    cs = (xp[0] + xp[2]) / d;  // fixed order: half 0, half 1
    a = RMS ? 0.f : (xp[1] + xp[3]) / d;
#pragma unroll
    for (int k = 0; k < VPLH; ++k) {
      const int c = cb + lane + 32 * k;
      if (lane + 32 * k >= qh) continue;
      const float4 gv = gs[c];
      float4 r = o[c];
      r.x += rs * (dyv[k].x * gv.x - a - xh[k].x * cs);
      r.y += rs * (dyv[k].y * gv.y - a - xh[k].y * cs);
      r.z += rs * (dyv[k].z * gv.z - a - xh[k].z * cs);
      r.w += rs * (dyv[k].w * gv.w - a - xh[k].w * cs);
      o[c] = r;
    }
  }
#pragma unroll
  for (int k = 0; k < VPLH; ++k)
    if (lane + 32 * k < qh) {
      reinterpret_cast<float4*>(red + (warp * NP) * d)[cb + lane + 32 * k] = pg[k];
      if (!RMS) reinterpret_cast<float4*>(red + (warp * NP + 1) * d)[cb + lane + 32 * k] = pb[k];
    }
  __syncthreads();
  float* wg = ws + static_cast<int64_t>(blockIdx.x) * NP * d;
  for (int j = threadIdx.x; j < NP * d; j += blockDim.x) {
    const int which = j / d, col = j % d;
    const int h = (col / 4) >= qh ? 1 : 0;
    float acc = 0.f;
    for (int p = 0; p < 4; ++p) acc += red[((2 * p + h) * NP + which) * d + col];  // fixed pair order
    wg[j] = acc;
  }
}

// rows per block for the pair kernel: shorter blocks for micro-batch-sized M fill the SMs, longer
// ones keep the dgamma partial reduction small (measured, tools/norm_bwd_bench.py with
// RLHF_NORM_RPB: M >= 8192 -> 64 (32 when the partial row is only np*d <= 2048 floats: RMS
// 8192x2048 70 -> 62 us), 4096 -> 32 (RMS 4096x4096 82 -> 68 us), <= 2048 -> 16)
static int pair_rows_per_block(int M, int d, int np, size_t ws_floats) {
  static const int force = [] { const char* e = getenv("RLHF_NORM_RPB"); return e ? atoi(e) : 0; }();  // timing only
  int rpb = force == 16 || force == 32 || force == 64 ? force : (M >= 8192 && np * d > 2048 ? kLnBwdRows : M >= 4096 ? 32 : 16);
  if (ws_floats < static_cast<size_t>((M + rpb - 1) / rpb) * np * d) rpb = kLnBwdRows;  // small workspace
  return rpb;
}

template <int VPLH, bool RMS>
static void launch_norm_bwd_pair(const float* dy, const float* x, const float* mean, const float* rstd, const uint16_t* g,
                                 float* dx, float* ws, int M, int d, int rpb, cudaStream_t s) {
  constexpr int NP = RMS ? 1 : 2;
  const size_t sm = static_cast<size_t>(8 * NP + 1) * d * 4 + 32 * 4;
  cudaFuncSetAttribute(norm_bwd_pair_kernel<VPLH, RMS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (8 * NP + 1) * (VPLH * 256) * 4 + 32 * 4);
  norm_bwd_pair_kernel<VPLH, RMS><<<(M + rpb - 1) / rpb, 256, sm, s>>>(dy, x, mean, rstd, g, dx, ws, M, d, rpb);
}

// out[j] += sum_k ws[k][j], fixed order: a block holds 32 columns x 8 row slices; slice t
// sums rows t, t+8, ... (loads of 8 slices in flight instead of one serial chain per
// column), then slice 0 adds the 8 slice sums in slice order.
__global__ void reduce_partials_kernel(const float* __restrict__ ws, int nblk, int ncol, int64_t blk_stride,
                                       float* __restrict__ out0, float* __restrict__ out1, int split) {
  __shared__ float red[8][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int j = blockIdx.x * 32 + tx;
  float s = 0.f;
  if (j < ncol) {
#pragma unroll 4
    for (int k = ty; k < nblk; k += 8) s += ws[k * blk_stride + j];
  }
  red[ty][tx] = s;
  __syncthreads();
  if (ty == 0 && j < ncol) {
    float t = red[0][tx];
#pragma unroll
    for (int q = 1; q < 8; ++q) t += red[q][tx];
    if (j < split) out0[j] += t;
    else out1[j - split] += t;
  }
}
static void reduce_partials(const float* ws, int nblk, int ncol, int64_t blk_stride, float* out0, float* out1, int split,
                            cudaStream_t s) {
  reduce_partials_kernel<<<(ncol + 31) / 32, 256, 0, s>>>(ws, nblk, ncol, blk_stride, out0, out1, split);
}

__global__ void round_bf16_kernel(const float* __restrict__ x, uint16_t* __restrict__ y, int64_t n) {
  const int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
  if (i + 3 < n) {
    const float4 v = *reinterpret_cast<const float4*>(x + i);
    *reinterpret_cast<uint2*>(y + i) =
        make_uint2(f2bf(v.x) | (static_cast<uint32_t>(f2bf(v.y)) << 16), f2bf(v.z) | (static_cast<uint32_t>(f2bf(v.w)) << 16));
  } else {
    for (int64_t k = i; k < n; ++k) y[k] = f2bf(x[k]);
  }
}

constexpr int kColsumChunks = 64;

// Partial column sums of a bf16 [M, N] matrix: block = 32 column groups of 8
// (16 B loads, a warp reads 512 contiguous bytes of a row) x 8 row lanes; rows of
// chunk blockIdx.y; fixed-order smem reduction of the 8 row lanes -> ws[chunk][N].
__global__ void colsum_bf16_kernel(const uint16_t* __restrict__ G, int M, int N, float* __restrict__ ws) {
  __shared__ float red[8][256];
  const int cg = threadIdx.x & 31, rl = threadIdx.x >> 5;
  const int col0 = blockIdx.x * 256 + cg * 8;
  const int per = (M + kColsumChunks - 1) / kColsumChunks;
  const int r0 = blockIdx.y * per, r1 = min(M, r0 + per);
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (col0 + 8 <= N) {
    for (int r = r0 + rl; r < r1; r += 8) {
      const uint4 u = *reinterpret_cast<const uint4*>(G + static_cast<int64_t>(r) * N + col0);
      const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        acc[2 * t] += bf2f(static_cast<uint16_t>(w[t] & 0xFFFFu));
        acc[2 * t + 1] += bf2f(static_cast<uint16_t>(w[t] >> 16));
      }
    }
  } else {
    for (int r = r0 + rl; r < r1; r += 8)
      for (int t = 0; t < 8; ++t)
        if (col0 + t < N) acc[t] += bf2f(G[static_cast<int64_t>(r) * N + col0 + t]);
  }
#pragma unroll
  for (int t = 0; t < 8; ++t) red[rl][cg * 8 + t] = acc[t];
  __syncthreads();
  const int c = blockIdx.x * 256 + threadIdx.x;
  if (c < N) {
    float sum = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) sum += red[k][threadIdx.x];
    ws[static_cast<int64_t>(blockIdx.y) * N + c] = sum;
  }
}

__global__ void gather_rows_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, int S, int R, int off,
                                   int row_bytes) {
  const int r = blockIdx.x;  // response row b*R + j
  const int b = r / R, j = r % R;
  const uint4* s4 = reinterpret_cast<const uint4*>(src + (static_cast<int64_t>(b) * S + off + j) * row_bytes);
  uint4* d4 = reinterpret_cast<uint4*>(dst + static_cast<int64_t>(r) * row_bytes);
  for (int c = threadIdx.x; c < row_bytes / 16; c += blockDim.x) d4[c] = s4[c];
}

__global__ void scatter_rows_kernel(const float* __restrict__ src, float* __restrict__ dst, int S, int R, int off, int d) {
  const int r = blockIdx.x;
  const int b = r / R, j = r % R;
  const float4* s4 = reinterpret_cast<const float4*>(src + static_cast<int64_t>(r) * d);
  float4* d4 = reinterpret_cast<float4*>(dst + (static_cast<int64_t>(b) * S + off + j) * d);
  for (int c = threadIdx.x; c < d / 4; c += blockDim.x) d4[c] = s4[c];
}

__global__ void adamw_kernel(float* __restrict__ w, float* __restrict__ m, float* __restrict__ v,
                             const float* __restrict__ g, uint16_t* __restrict__ wb, int64_t n, float lr, float b1,
                             float b2, float eps, float wd, float bc1, float bc2) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i * 4 >= n) return;
  float4 W = reinterpret_cast<float4*>(w)[i], Mm = reinterpret_cast<float4*>(m)[i], Vv = reinterpret_cast<float4*>(v)[i];
  const float4 G = reinterpret_cast<const float4*>(g)[i];
  float* Wp = &W.x;
  float* Mp = &Mm.x;
  float* Vp = &Vv.x;
  const float* Gp = &G.x;
  uint16_t o[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    Mp[k] = b1 * Mp[k] + (1.0f - b1) * Gp[k];
    Vp[k] = b2 * Vp[k] + (1.0f - b2) * Gp[k] * Gp[k];
    const float upd = (Mp[k] / bc1) / (sqrtf(Vp[k] / bc2) + eps);
    Wp[k] = Wp[k] - lr * (upd + wd * Wp[k]);
    o[k] = f2bf(Wp[k]);
  }
  reinterpret_cast<float4*>(w)[i] = W;
  reinterpret_cast<float4*>(m)[i] = Mm;
  reinterpret_cast<float4*>(v)[i] = Vv;
  reinterpret_cast<uint2*>(wb)[i] = make_uint2(o[0] | (static_cast<uint32_t>(o[1]) << 16), o[2] | (static_cast<uint32_t>(o[3]) << 16));
}

__global__ void add_int_kernel(int* p, int v) {
  pdl_entry();
  *p += v;
}

}  // namespace rlhf

using namespace rlhf;

extern "C" void rlhf_set_pdl(int on) { g_pdl = on; }

extern "C" int rlhf_add_int(int* p, int v, rlhf_stream_t s) {
  return launch_k(add_int_kernel, dim3(1), dim3(1), 0, S(s), p, v);
}

extern "C" int rlhf_embed(const int32_t* tokens, int64_t tok_stride, int B, int T, int p0, const int* p0_dev,
                          const void* tok_emb, const void* pos_emb, int d, float* x, rlhf_stream_t s) {
  if (d % 4) return 2;
  const int rows = B * T;
  const int64_t n = static_cast<int64_t>(rows) * (d / 4);
  return launch_k(embed_kernel, dim3(static_cast<unsigned>((n + 255) / 256)), dim3(256), 0, S(s), tokens, tok_stride, T, p0,
                  p0_dev, static_cast<const uint16_t*>(tok_emb), static_cast<const uint16_t*>(pos_emb), d, x, rows);
}

extern "C" int rlhf_embed_bwd(const int32_t* tokens, int64_t tok_stride, int B, int T, const float* dx, int d,
                              float* dtok, float* dpos, rlhf_stream_t s) {
  const int rows = B * T;
  const int64_t n = static_cast<int64_t>(rows) * d;
  embed_bwd_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, S(s)>>>(tokens, tok_stride, T, dx, d, dtok, dpos, rows);
  return cuda_status();
}

extern "C" int rlhf_layernorm(const float* x, const void* g, const void* b, void* y, float* mean, float* rstd, int M,
                              int d, rlhf_stream_t s) {
  if (d % 4) return 2;
  const dim3 grid((M + 7) / 8), blk(256);
  const auto* gp = static_cast<const uint16_t*>(g);
  const auto* bp = static_cast<const uint16_t*>(b);
  auto* yp = static_cast<uint16_t*>(y);
  if (d <= 1024) return launch_k(layernorm_kernel<8, false>, grid, blk, 0, S(s), x, gp, bp, yp, mean, rstd, M, d);
  if (d <= 2048) return launch_k(layernorm_kernel<16, false>, grid, blk, 0, S(s), x, gp, bp, yp, mean, rstd, M, d);
  if (d <= 4096) return launch_k(layernorm_kernel<32, false>, grid, blk, 0, S(s), x, gp, bp, yp, mean, rstd, M, d);
  return 2;
}

extern "C" int rlhf_rmsnorm(const float* x, const void* g, void* y, float* rstd, int M, int d, rlhf_stream_t s) {
  if (d % 4) return 2;
  const dim3 grid((M + 7) / 8), blk(256);
  const auto* gp = static_cast<const uint16_t*>(g);
  auto* yp = static_cast<uint16_t*>(y);
  const uint16_t* nb = nullptr;
  float* nm = nullptr;
  if (d <= 1024) return launch_k(layernorm_kernel<8, true>, grid, blk, 0, S(s), x, gp, nb, yp, nm, rstd, M, d);
  if (d <= 2048) return launch_k(layernorm_kernel<16, true>, grid, blk, 0, S(s), x, gp, nb, yp, nm, rstd, M, d);
  if (d <= 4096) return launch_k(layernorm_kernel<32, true>, grid, blk, 0, S(s), x, gp, nb, yp, nm, rstd, M, d);
  return 2;
}

extern "C" int rlhf_rmsnorm_bwd(const float* dy, const float* x, const float* rstd, const void* g, float* dx, float* dg,
                                int M, int d, float* ws, size_t ws_floats, rlhf_stream_t s) {
  const int nblk = (M + kLnBwdRows - 1) / kLnBwdRows;
  if (d % 4 || ws_floats < static_cast<size_t>(nblk) * d) return 2;
  const size_t sm = static_cast<size_t>(8) * d * 4;
  const auto* gp = static_cast<const uint16_t*>(g);
  const float* nm = nullptr;
  if (d <= 1024) {
    cudaFuncSetAttribute(layernorm_bwd_kernel<8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 1024 * 4);
    layernorm_bwd_kernel<8, true><<<nblk, 256, sm, S(s)>>>(dy, x, nm, rstd, gp, dx, ws, M, d);
  } else if (d <= 4096 && d % 8 == 0) {
    const int rpb = pair_rows_per_block(M, d, 1, ws_floats);
    if (d <= 2048) launch_norm_bwd_pair<8, true>(dy, x, nm, rstd, gp, dx, ws, M, d, rpb, S(s));
    else launch_norm_bwd_pair<16, true>(dy, x, nm, rstd, gp, dx, ws, M, d, rpb, S(s));
    reduce_partials(ws, (M + rpb - 1) / rpb, d, d, dg, dg, d, S(s));
    return cuda_status();
  } else if (d <= 2048) {
    cudaFuncSetAttribute(layernorm_bwd_kernel<16, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 2048 * 4);
    layernorm_bwd_kernel<16, true><<<nblk, 256, sm, S(s)>>>(dy, x, nm, rstd, gp, dx, ws, M, d);
  } else {
    return 2;
  }
  reduce_partials(ws, nblk, d, d, dg, dg, d, S(s));
  return cuda_status();
}

extern "C" int rlhf_layernorm_bwd(const float* dy, const float* x, const float* mean, const float* rstd, const void* g,
                                  float* dx, float* dg, float* db, int M, int d, float* ws, size_t ws_floats,
                                  rlhf_stream_t s) {
  const int nblk = (M + kLnBwdRows - 1) / kLnBwdRows;
  if (d % 4 || ws_floats < static_cast<size_t>(nblk) * 2 * d) return 2;
  const size_t sm = static_cast<size_t>(16) * d * 4;
  const auto* gp = static_cast<const uint16_t*>(g);
  if (d <= 1024) {
    cudaFuncSetAttribute(layernorm_bwd_kernel<8, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 1024 * 4);
    layernorm_bwd_kernel<8, false><<<nblk, 256, sm, S(s)>>>(dy, x, mean, rstd, gp, dx, ws, M, d);
  } else if (d <= 2048 && d % 8 == 0) {
    const int rpb = pair_rows_per_block(M, d, 2, ws_floats);
    launch_norm_bwd_pair<8, false>(dy, x, mean, rstd, gp, dx, ws, M, d, rpb, S(s));
    reduce_partials(ws, (M + rpb - 1) / rpb, 2 * d, 2 * d, dg, db, d, S(s));
    return cuda_status();
  } else if (d <= 2048) {
    cudaFuncSetAttribute(layernorm_bwd_kernel<16, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 2048 * 4);
    layernorm_bwd_kernel<16, false><<<nblk, 256, sm, S(s)>>>(dy, x, mean, rstd, gp, dx, ws, M, d);
  } else {
    return 2;
  }
  reduce_partials(ws, nblk, 2 * d, 2 * d, dg, db, d, S(s));
  return cuda_status();
}

__global__ void add_f32_kernel(float* __restrict__ y, const float* __restrict__ x, int64_t n) {
  const int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
  if (i + 3 < n) {
    float4 a = *reinterpret_cast<float4*>(y + i);
    const float4 b = *reinterpret_cast<const float4*>(x + i);
    a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
    *reinterpret_cast<float4*>(y + i) = a;
  } else {
    for (int64_t k = i; k < n; ++k) y[k] += x[k];
  }
}

extern "C" int rlhf_add_f32(float* y, const float* x, int64_t n, rlhf_stream_t s) {
  if (n <= 0) return 0;
  if ((reinterpret_cast<uintptr_t>(y) | reinterpret_cast<uintptr_t>(x)) & 15) return 2;
  const int64_t q = (n + 3) / 4;
  add_f32_kernel<<<static_cast<unsigned>((q + 255) / 256), 256, 0, S(s)>>>(y, x, n);
  return cuda_status();
}

extern "C" int rlhf_round_bf16(const float* x, void* out, int64_t n, rlhf_stream_t s) {
  const int64_t q = (n + 3) / 4;
  round_bf16_kernel<<<static_cast<unsigned>((q + 255) / 256), 256, 0, S(s)>>>(x, static_cast<uint16_t*>(out), n);
  return cuda_status();
}

extern "C" int rlhf_colsum_bf16(const void* G, int M, int N, float* db, float* ws, rlhf_stream_t s) {
  if (N % 8) return 2;
  dim3 grid((N + 255) / 256, kColsumChunks);
  colsum_bf16_kernel<<<grid, 256, 0, S(s)>>>(static_cast<const uint16_t*>(G), M, N, ws);
  reduce_partials(ws, kColsumChunks, N, N, db, db, N, S(s));
  return cuda_status();
}

extern "C" int rlhf_gather_rows(const void* src, void* dst, int B, int S_, int R, int off, int d, int elem_bytes,
                                rlhf_stream_t s) {
  const int row_bytes = d * elem_bytes;
  if (row_bytes % 16) return 2;
  gather_rows_kernel<<<B * R, 128, 0, S(s)>>>(static_cast<const uint8_t*>(src), static_cast<uint8_t*>(dst), S_, R, off,
                                               row_bytes);
  return cuda_status();
}

extern "C" int rlhf_scatter_rows_f32(const float* src, float* dst, int B, int S_, int R, int off, int d, rlhf_stream_t s) {
  if (d % 4) return 2;
  scatter_rows_kernel<<<B * R, 128, 0, S(s)>>>(src, dst, S_, R, off, d);
  return cuda_status();
}

extern "C" int rlhf_adamw(float* master, float* m, float* v, const float* grad, void* w_bf16, int64_t n, float lr,
                          float beta1, float beta2, float eps, float weight_decay, int step, rlhf_stream_t s) {
  if (n % 4) return 2;
  const float bc1 = 1.0f - powf(beta1, static_cast<float>(step));
  const float bc2 = 1.0f - powf(beta2, static_cast<float>(step));
  const int64_t q = n / 4;
  adamw_kernel<<<static_cast<unsigned>((q + 255) / 256), 256, 0, S(s)>>>(master, m, v, grad, static_cast<uint16_t*>(w_bf16), n,
                                                                          lr, beta1, beta2, eps, weight_decay, bc1, bc2);
  return cuda_status();
}

static int embed_ln_launch(const int32_t* tokens, int64_t tok_stride, int B, const int* pos_dev, const void* tok_emb,
                           const void* pos_emb, int d, float* x, const void* ln_g, const void* ln_b, void* y,
                           rlhf_stream_t s, const float4* t2, int tiles, int32_t* dst, float* margin) {
  if (d % 4 || d > 4096 || !pos_dev) return 2;
  const dim3 grid((B + 7) / 8), blk(256);
  const auto* E = static_cast<const uint16_t*>(tok_emb);
  const auto* Pm = static_cast<const uint16_t*>(pos_emb);
  const auto* g = static_cast<const uint16_t*>(ln_g);
  const auto* b = static_cast<const uint16_t*>(ln_b);
  auto* yp = static_cast<uint16_t*>(y);
  if (d <= 1024) return launch_k(embed_ln_kernel<8, false>, grid, blk, 0, S(s), tokens, tok_stride, pos_dev, E, Pm, d, x, g, b, yp, B, t2, tiles, dst, margin);
  if (d <= 2048) return launch_k(embed_ln_kernel<16, false>, grid, blk, 0, S(s), tokens, tok_stride, pos_dev, E, Pm, d, x, g, b, yp, B, t2, tiles, dst, margin);
  return launch_k(embed_ln_kernel<32, false>, grid, blk, 0, S(s), tokens, tok_stride, pos_dev, E, Pm, d, x, g, b, yp, B, t2, tiles, dst, margin);
}

static int embed_rmsnorm_launch(const int32_t* tokens, int64_t tok_stride, int B, const int* pos_dev,
                                const void* tok_emb, int d, float* x, const void* g, void* y, rlhf_stream_t s,
                                const float4* t2, int tiles, int32_t* dst, float* margin) {
  if (d % 4 || d > 4096 || !pos_dev) return 2;
  const dim3 grid((B + 7) / 8), blk(256);
  const auto* E = static_cast<const uint16_t*>(tok_emb);
  const auto* gp = static_cast<const uint16_t*>(g);
  const uint16_t* nil = nullptr;
  auto* yp = static_cast<uint16_t*>(y);
  if (d <= 1024) return launch_k(embed_ln_kernel<8, true>, grid, blk, 0, S(s), tokens, tok_stride, pos_dev, E, nil, d, x, gp, nil, yp, B, t2, tiles, dst, margin);
  if (d <= 2048) return launch_k(embed_ln_kernel<16, true>, grid, blk, 0, S(s), tokens, tok_stride, pos_dev, E, nil, d, x, gp, nil, yp, B, t2, tiles, dst, margin);
  return launch_k(embed_ln_kernel<32, true>, grid, blk, 0, S(s), tokens, tok_stride, pos_dev, E, nil, d, x, gp, nil, yp, B, t2, tiles, dst, margin);
}

extern "C" int rlhf_embed_ln(const int32_t* tokens, int64_t tok_stride, int B, const int* pos_dev, const void* tok_emb,
                             const void* pos_emb, int d, float* x, const void* ln_g, const void* ln_b, void* y,
                             rlhf_stream_t s) {
  return embed_ln_launch(tokens, tok_stride, B, pos_dev, tok_emb, pos_emb, d, x, ln_g, ln_b, y, s, nullptr, 0, nullptr,
                         nullptr);
}

extern "C" int rlhf_embed_rmsnorm(const int32_t* tokens, int64_t tok_stride, int B, const int* pos_dev,
                                  const void* tok_emb, int d, float* x, const void* g, void* y, rlhf_stream_t s) {
  return embed_rmsnorm_launch(tokens, tok_stride, B, pos_dev, tok_emb, d, x, g, y, s, nullptr, 0, nullptr, nullptr);
}

extern "C" int rlhf_argmax_embed_ln(const float* top2, int tiles, int32_t* dst, float* margin, const int32_t* tokens,
                                    int64_t tok_stride, int B, int* pos_dev, const void* tok_emb, const void* pos_emb,
                                    int d, float* x, const void* ln_g, const void* ln_b, void* y, rlhf_stream_t s) {
  if (!top2 || tiles < 1 || !dst) return 2;
  return embed_ln_launch(tokens, tok_stride, B, pos_dev, tok_emb, pos_emb, d, x, ln_g, ln_b, y, s,
                         reinterpret_cast<const float4*>(top2), tiles, dst, margin);
}

extern "C" int rlhf_argmax_embed_rmsnorm(const float* top2, int tiles, int32_t* dst, float* margin,
                                         const int32_t* tokens, int64_t tok_stride, int B, int* pos_dev,
                                         const void* tok_emb, int d, float* x, const void* g, void* y,
                                         rlhf_stream_t s) {
  if (!top2 || tiles < 1 || !dst) return 2;
  return embed_rmsnorm_launch(tokens, tok_stride, B, pos_dev, tok_emb, d, x, g, y, s,
                              reinterpret_cast<const float4*>(top2), tiles, dst, margin);
}
