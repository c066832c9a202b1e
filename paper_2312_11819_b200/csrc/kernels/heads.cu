// heads.cu — output heads and the experience-buffer / PPO math of one step:
// LM log-softmax gather (fwd + bwd), greedy argmax sampler, scalar value/reward
// head (fwd + bwd), reward shaping + GAE, clipped actor / value losses.
// Numerics: DeepSpeed-Chat step 3 conventions; reference
// structure: experience-buffer barrier /root/reference/proj/src/workload.cpp:153-163.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cfloat>

#include "launch_util.cuh"
#include "rlhf_kernels.h"

namespace rlhf {

__device__ __forceinline__ float hb2f(uint16_t h) { return __uint_as_float(static_cast<uint32_t>(h) << 16); }
__device__ __forceinline__ uint16_t hf2b(float f) { return __bfloat16_as_ushort(__float2bfloat16_rn(f)); }

template <typename T, typename Op>
__device__ __forceinline__ T block_reduce(T v, Op op, T* sh) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x / 32, nw = blockDim.x / 32;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[w] = v;
  __syncthreads();
  T r = sh[0];
  for (int k = 1; k < nw; ++k) r = op(r, sh[k]);
  return r;
}

struct MaxOp { __device__ float operator()(float a, float b) const { return fmaxf(a, b); } };
struct SumOp { __device__ float operator()(float a, float b) const { return a + b; } };

// One CTA per logits row r = b*R + j; target y = tokens[b*S + P + j].  Single
// pass: online (max, sum-exp) per thread over float4 loads, then block merge.
__global__ void logprob_kernel(const float* __restrict__ z, int V, const int32_t* __restrict__ tok, int S, int P, int R,
                               float* __restrict__ logp, float* __restrict__ lse_out) {
  __shared__ float shm[32], shs[32];
  const int r = blockIdx.x;
  const float* zr = z + static_cast<int64_t>(r) * V;
  float m = -FLT_MAX, s = 0.f;
  auto add = [&](float x) {
    if (x > m) {
      s = s * expf(m - x) + 1.0f;
      m = x;
    } else {
      s += expf(x - m);
    }
  };
  const int V4 = V / 4;
  const float4* z4 = reinterpret_cast<const float4*>(zr);
  for (int v = threadIdx.x; v < V4; v += blockDim.x) {
    const float4 q = z4[v];
    add(q.x); add(q.y); add(q.z); add(q.w);
  }
  for (int v = V4 * 4 + threadIdx.x; v < V; v += blockDim.x) add(zr[v]);
  // warp merge
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, s, o);
    const float mm = fmaxf(m, m2);
    s = s * expf(m - mm) + s2 * expf(m2 - mm);
    m = mm;
  }
  const int w = threadIdx.x / 32, nw = blockDim.x / 32;
  if ((threadIdx.x & 31) == 0) { shm[w] = m; shs[w] = s; }
  __syncthreads();
  if (threadIdx.x == 0) {
    float M = shm[0], Ssum = shs[0];
    for (int k = 1; k < nw; ++k) {
      const float mm = fmaxf(M, shm[k]);
      Ssum = Ssum * expf(M - mm) + shs[k] * expf(shm[k] - mm);
      M = mm;
    }
    const float lse = M + logf(Ssum);
    const int b = r / R, j = r % R;
    const int y = tok[static_cast<int64_t>(b) * S + P + j];
    logp[r] = zr[y] - lse;
    if (lse_out) lse_out[r] = lse;
  }
}

// one warp per row: merge the LM-head GEMM's (max, sumexp) partials, logp = z_y - lse
__global__ void lse_merge_kernel(const float2* __restrict__ part, const float* __restrict__ tgt, int rows, int parts,
                                 float* __restrict__ logp) {
  const int r = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x & 31;
  if (r >= rows) return;
  float m = -FLT_MAX, s = 0.f;
  for (int k = lane; k < parts; k += 32) {
    const float2 p = part[static_cast<int64_t>(r) * parts + k];
    if (p.x == -FLT_MAX) continue;
    const float mm = fmaxf(m, p.x);
    s = (m == -FLT_MAX ? 0.f : s * expf(m - mm)) + p.y * expf(p.x - mm);
    m = mm;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, s, o);
    const float mm = fmaxf(m, m2);
    s = (m == -FLT_MAX ? 0.f : s * expf(m - mm)) + (m2 == -FLT_MAX ? 0.f : s2 * expf(m2 - mm));
    m = mm;
  }
  if (lane == 0) logp[r] = tgt[r] - (m + logf(s));
}

__global__ void logprob_bwd_kernel(const float* __restrict__ z, const float* __restrict__ lse, const float* __restrict__ g,
                                   int V, const int32_t* __restrict__ tok, int S, int P, int R, uint16_t* __restrict__ dz) {
  const int r = blockIdx.x;
  const int b = r / R, j = r % R;
  const int y = tok[static_cast<int64_t>(b) * S + P + j];
  const float* zr = z + static_cast<int64_t>(r) * V;
  uint16_t* o = dz + static_cast<int64_t>(r) * V;
  const float L = lse[r], gr = g[r];
  const int V4 = V / 4;
  const float4* z4 = reinterpret_cast<const float4*>(zr);
  uint2* o4 = reinterpret_cast<uint2*>(o);
  for (int v = threadIdx.x; v < V4; v += blockDim.x) {
    const float4 q = z4[v];
    const int b0 = 4 * v;
    const uint16_t h0 = hf2b(gr * ((b0 == y ? 1.0f : 0.0f) - expf(q.x - L)));
    const uint16_t h1 = hf2b(gr * ((b0 + 1 == y ? 1.0f : 0.0f) - expf(q.y - L)));
    const uint16_t h2 = hf2b(gr * ((b0 + 2 == y ? 1.0f : 0.0f) - expf(q.z - L)));
    const uint16_t h3 = hf2b(gr * ((b0 + 3 == y ? 1.0f : 0.0f) - expf(q.w - L)));
    o4[v] = make_uint2(h0 | (static_cast<uint32_t>(h1) << 16), h2 | (static_cast<uint32_t>(h3) << 16));
  }
  for (int v = V4 * 4 + threadIdx.x; v < V; v += blockDim.x) o[v] = hf2b(gr * ((v == y ? 1.0f : 0.0f) - expf(zr[v] - L)));
}

// Greedy argmax per sample (ties -> lowest id) + top-2 margin.  Two phases:
// 64 CTAs per row scan slices into ws, then one warp per row merges.
constexpr int kArgSlices = 64;

struct Top2 { float v1; int i1; float v2; };

__device__ __forceinline__ Top2 top2_merge(Top2 a, Top2 b) {
  Top2 r;
  if (b.v1 > a.v1 || (b.v1 == a.v1 && b.i1 < a.i1)) {
    r.v1 = b.v1; r.i1 = b.i1; r.v2 = fmaxf(a.v1, b.v2);
  } else {
    r.v1 = a.v1; r.i1 = a.i1; r.v2 = fmaxf(a.v2, b.v1);
  }
  return r;
}

__global__ void argmax_slice_kernel(const float* __restrict__ z, int V, float* __restrict__ ws) {
  pdl_entry();
  const int b = blockIdx.y, sl = blockIdx.x;
  const int per = (V + kArgSlices - 1) / kArgSlices;
  const int v0 = sl * per, v1 = min(V, v0 + per);
  Top2 t{-FLT_MAX, 0x7fffffff, -FLT_MAX};
  for (int v = v0 + threadIdx.x; v < v1; v += blockDim.x) t = top2_merge(t, Top2{z[static_cast<int64_t>(b) * V + v], v, -FLT_MAX});
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    Top2 u{__shfl_xor_sync(0xffffffffu, t.v1, o), __shfl_xor_sync(0xffffffffu, t.i1, o), __shfl_xor_sync(0xffffffffu, t.v2, o)};
    t = top2_merge(t, u);
  }
  __shared__ Top2 sh[8];
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x / 32] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < blockDim.x / 32; ++w) t = top2_merge(t, sh[w]);
    float* o = ws + (static_cast<int64_t>(b) * kArgSlices + sl) * 4;
    o[0] = t.v1; o[1] = __int_as_float(t.i1); o[2] = t.v2;
  }
}

__global__ void argmax_merge_kernel(const float* __restrict__ ws, int B, int32_t* __restrict__ tok, int S,
                                    const int* __restrict__ pos_dev, float* __restrict__ margin) {
  pdl_entry();
  const int b = blockIdx.x;
  const int lane = threadIdx.x;
  Top2 t{-FLT_MAX, 0x7fffffff, -FLT_MAX};
  for (int s = lane; s < kArgSlices; s += 32) {
    const float* o = ws + (static_cast<int64_t>(b) * kArgSlices + s) * 4;
    t = top2_merge(t, Top2{o[0], __float_as_int(o[1]), o[2]});
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    Top2 u{__shfl_xor_sync(0xffffffffu, t.v1, o), __shfl_xor_sync(0xffffffffu, t.i1, o), __shfl_xor_sync(0xffffffffu, t.v2, o)};
    t = top2_merge(t, u);
  }
  if (lane == 0) {
    tok[static_cast<int64_t>(b) * S + *pos_dev + 1] = t.i1;
    if (margin) margin[static_cast<int64_t>(b) * S + *pos_dev + 1] = t.v1 - t.v2;
  }
}

// one warp per sample: merge the LM-head GEMM's per-tile top-2 partials
// One CTA: warp w merges samples w, w+32, ...; afterwards the position counter
// advances (the decode step's last kernel, so no separate increment launch).
// One CTA per sample: the CTA's threads split the vocabulary tiles (their loads spread over
// B SMs instead of one SM's load queue), merge inside each warp, then across warps in warp
// order (top-2 merging is order-independent: the same token and margin as a serial merge).
// advance: the last CTA to finish (ticket in pos_dev[1], self-resetting) writes *pos + 1,
// after every CTA has read *pos.
constexpr int kArgmaxThreads = 128;
__global__ void __launch_bounds__(kArgmaxThreads) argmax_tiles_kernel(const float4* __restrict__ t2, int tiles, int B,
                                                                      int32_t* __restrict__ tok, int64_t S,
                                                                      int* __restrict__ pos_dev, float* __restrict__ margin,
                                                                      int advance) {
  pdl_entry();
  __shared__ Top2 red[kArgmaxThreads / 32];
  const int b = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int pos = *pos_dev;
  Top2 t{-FLT_MAX, 0x7fffffff, -FLT_MAX};
  for (int i = threadIdx.x; i < tiles; i += kArgmaxThreads) {
    const float4 o = t2[static_cast<int64_t>(i) * B + b];
    t = top2_merge(t, Top2{o.x, __float_as_int(o.y), o.z});
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    Top2 u{__shfl_xor_sync(0xffffffffu, t.v1, o), __shfl_xor_sync(0xffffffffu, t.i1, o),
           __shfl_xor_sync(0xffffffffu, t.v2, o)};
    t = top2_merge(t, u);
  }
  if (lane == 0) red[warp] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    t = red[0];
#pragma unroll
    for (int w = 1; w < kArgmaxThreads / 32; ++w) t = top2_merge(t, red[w]);
    const int64_t at = static_cast<int64_t>(b) * S + pos + 1;
    tok[at] = t.i1;
    if (margin) margin[at] = t.v1 - t.v2;
    if (advance) {
      __threadfence();  // this CTA's read of *pos precedes its ticket
      unsigned* ticket = reinterpret_cast<unsigned*>(pos_dev + 1);
      if (atomicAdd(ticket, 1u) == gridDim.x - 1) {
        *ticket = 0u;
        *pos_dev = pos + 1;
      }
    }
  }
}

// out[b*R + j] = hf[b*S + off + j] . w   (warp per row)
__global__ void scalar_head_kernel(const uint16_t* __restrict__ hf, const uint16_t* __restrict__ w, int S, int R, int off,
                                   int d, float* __restrict__ out, int rows) {
  const int r = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const int b = r / R, j = r % R;
  const uint16_t* h = hf + (static_cast<int64_t>(b) * S + off + j) * d;
  float s = 0.f;
  for (int e = lane; e < d; e += 32) s += hb2f(h[e]) * hb2f(w[e]);
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[r] = s;
}

// dhf[row] += g * w ; per-chunk partials of dw (fixed order)
constexpr int kHeadChunks = 64;
__global__ void scalar_head_bwd_kernel(const uint16_t* __restrict__ hf, const uint16_t* __restrict__ w,
                                       const float* __restrict__ g, int S, int R, int off, int d, float* __restrict__ dhf,
                                       float* __restrict__ ws, int rows) {
  const int chunk = blockIdx.y;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= d) return;
  const int per = (rows + kHeadChunks - 1) / kHeadChunks;
  const int r0 = chunk * per, r1 = min(rows, r0 + per);
  const float we = hb2f(w[e]);
  float acc = 0.f;
  for (int r = r0; r < r1; ++r) {
    const int b = r / R, j = r % R;
    const int64_t row = static_cast<int64_t>(b) * S + off + j;
    dhf[row * d + e] += g[r] * we;
    acc += g[r] * hb2f(hf[row * d + e]);
  }
  ws[static_cast<int64_t>(chunk) * d + e] = acc;
}

__global__ void sum_chunks_kernel(const float* __restrict__ ws, int chunks, int n, float* __restrict__ out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  float s = 0.f;
  for (int c = 0; c < chunks; ++c) s += ws[static_cast<int64_t>(c) * n + e];
  out[e] += s;
}

// Experience buffer, one warp per sample.  A_t = delta_t + c A_{t+1} (c = gamma lam) is a
// first-order linear recurrence: lane i owns the contiguous chunk [i*n, i*n+n) of the
// response, reduces it to the affine map A_lo = u + c^n A_hi (one reverse pass over its
// chunk, fully parallel across lanes), the 32 maps are composed by a reverse warp scan
// (Kogge-Stone over __shfl_down), and each lane replays its chunk from its exact incoming
// A_hi.  All loads are lane-contiguous (each lane streams its own chunk), every value is
// produced in a fixed order, so the result is deterministic.
__global__ void gae_kernel(const float* __restrict__ logp, const float* __restrict__ logp_ref, const float* __restrict__ val,
                           const float* __restrict__ score, int B, int R, float kl, float clip_r, float gamma, float lam,
                           float* __restrict__ rew, float* __restrict__ adv, float* __restrict__ ret) {
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (b >= B) return;
  const int64_t o = static_cast<int64_t>(b) * R;
  const float c = gamma * lam;
  const int n = (R + 31) / 32;
  const int j0 = min(R, lane * n), j1 = min(R, j0 + n);
  const float sc = fminf(fmaxf(score[b], -clip_r), clip_r);
  auto delta = [&](int j) {
    float r = -kl * (logp[o + j] - logp_ref[o + j]);
    if (j == R - 1) r += sc;
    const float nextv = j < R - 1 ? val[o + j + 1] : 0.0f;
    return r + gamma * nextv - val[o + j];
  };
  // this lane's chunk as an affine map of the advantage just after it: A_{j0} = u + m A_{j1}
  float u = 0.f, m = 1.f;
  for (int j = j1 - 1; j >= j0; --j) {
    u = delta(j) + c * u;
    m *= c;
  }
  // reverse inclusive scan: lane i composes its map with every map to its right
  for (int k = 1; k < 32; k <<= 1) {
    const float u2 = __shfl_down_sync(0xffffffffu, u, k), m2 = __shfl_down_sync(0xffffffffu, m, k);
    if (lane + k < 32) {
      u = u + m * u2;
      m = m * m2;
    }
  }
  // incoming advantage of this chunk = the composed map of the lanes to its right applied to 0
  float last = __shfl_down_sync(0xffffffffu, u, 1);
  if (lane == 31) last = 0.f;
  for (int j = j1 - 1; j >= j0; --j) {
    float r = -kl * (logp[o + j] - logp_ref[o + j]);
    if (j == R - 1) r += sc;
    const float nextv = j < R - 1 ? val[o + j + 1] : 0.0f;
    last = (r + gamma * nextv - val[o + j]) + c * last;
    rew[o + j] = r;
    adv[o + j] = last;
    ret[o + j] = last + val[o + j];
  }
}

// PPO losses: one block, a fixed per-thread stride and a fixed block-reduction tree, so
// the loss sum is bit-reproducible (no atomics); `loss` accumulates across the TrainFB
// micro-batches in stream order.
__global__ void actor_loss_kernel(const float* __restrict__ lp, const float* __restrict__ lpo, const float* __restrict__ A,
                                  int n, float clip, float denom, float* __restrict__ g, float* __restrict__ loss) {
  __shared__ float sh[32];
  float l = 0.f;
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const float ratio = expf(lp[k] - lpo[k]);
    const float a = A[k];
    const float cl = fminf(fmaxf(ratio, 1.0f - clip), 1.0f + clip);
    const float pg1 = -a * ratio, pg2 = -a * cl;
    l += fmaxf(pg1, pg2);
    const bool inside = ratio >= 1.0f - clip && ratio <= 1.0f + clip;
    const float d1 = -a * ratio / denom, d2 = inside ? -a * ratio / denom : 0.0f;
    g[k] = pg1 > pg2 ? d1 : (pg1 < pg2 ? d2 : 0.5f * (d1 + d2));
  }
  l = block_reduce(l, SumOp(), sh);
  if (threadIdx.x == 0) *loss += l;
}

__global__ void critic_loss_kernel(const float* __restrict__ v, const float* __restrict__ vo, const float* __restrict__ ret,
                                   int n, float clip, float denom, float* __restrict__ g, float* __restrict__ loss) {
  __shared__ float sh[32];
  float l = 0.f;
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const float x = v[k], o = vo[k], R = ret[k];
    const float vc = fminf(fmaxf(x, o - clip), o + clip);
    const float l1 = (x - R) * (x - R), l2 = (vc - R) * (vc - R);
    l += fmaxf(l1, l2);
    const bool inside = x >= o - clip && x <= o + clip;
    const float d1 = (x - R) / denom, d2 = inside ? (vc - R) / denom : 0.0f;
    g[k] = l1 > l2 ? d1 : (l1 < l2 ? d2 : 0.5f * (d1 + d2));
  }
  l = block_reduce(l, SumOp(), sh);
  if (threadIdx.x == 0) *loss += l;
}

// out[0] = sum(score[b]), out[1] = sum(logp - logp_ref) over the experience rows (fixed order).
__global__ void experience_stats_kernel(const float* __restrict__ lp, const float* __restrict__ lpr,
                                        const float* __restrict__ score, int B, int R, float* __restrict__ out) {
  __shared__ float sh[32];
  float kl = 0.f, sc = 0.f;
  const int n = B * R;
  for (int k = threadIdx.x; k < n; k += blockDim.x) kl += lp[k] - lpr[k];
  for (int k = threadIdx.x; k < B; k += blockDim.x) sc += score[k];
  kl = block_reduce(kl, SumOp(), sh);
  __syncthreads();
  sc = block_reduce(sc, SumOp(), sh);
  if (threadIdx.x == 0) {
    out[0] = sc;
    out[1] = kl;
  }
}

}  // namespace rlhf

using namespace rlhf;

static inline cudaStream_t HS(rlhf_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }
static inline int HST() { return cudaGetLastError() == cudaSuccess ? 0 : 5; }

extern "C" int rlhf_logprob(const float* logits, int rows, int V, const int32_t* tokens, int S, int P, int R, float* logp,
                            float* lse, rlhf_stream_t s) {
  logprob_kernel<<<rows, 512, 0, HS(s)>>>(logits, V, tokens, S, P, R, logp, lse);
  return HST();
}

extern "C" int rlhf_logprob_bwd(const float* logits, const float* lse, const float* g, int rows, int V,
                                const int32_t* tokens, int S, int P, int R, void* dz, rlhf_stream_t s) {
  logprob_bwd_kernel<<<rows, 512, 0, HS(s)>>>(logits, lse, g, V, tokens, S, P, R, static_cast<uint16_t*>(dz));
  return HST();
}

extern "C" int rlhf_argmax_tokens(const float* logits, int B, int V, int32_t* tokens, int S, const int* pos_dev,
                                  float* margin, float* ws, rlhf_stream_t s) {
  const int st = launch_k(argmax_slice_kernel, dim3(kArgSlices, B), dim3(256), 0, HS(s), logits, V, ws);
  if (st) return st;
  return launch_k(argmax_merge_kernel, dim3(B), dim3(32), 0, HS(s), ws, B, tokens, S, pos_dev, margin);
}

extern "C" int rlhf_scalar_head(const void* hf, const void* w, int B, int S, int R, int off, int d, float* out,
                                rlhf_stream_t s) {
  const int rows = B * R;
  scalar_head_kernel<<<(rows + 7) / 8, 256, 0, HS(s)>>>(static_cast<const uint16_t*>(hf), static_cast<const uint16_t*>(w), S,
                                                        R, off, d, out, rows);
  return HST();
}

extern "C" int rlhf_scalar_head_bwd(const void* hf, const void* w, const float* g, int B, int S, int R, int off, int d,
                                    float* dhf, float* dw, float* ws, rlhf_stream_t s) {
  const int rows = B * R;
  scalar_head_bwd_kernel<<<dim3((d + 255) / 256, kHeadChunks), 256, 0, HS(s)>>>(
      static_cast<const uint16_t*>(hf), static_cast<const uint16_t*>(w), g, S, R, off, d, dhf, ws, rows);
  sum_chunks_kernel<<<(d + 255) / 256, 256, 0, HS(s)>>>(ws, kHeadChunks, d, dw);
  return HST();
}

extern "C" int rlhf_gae(const float* logp, const float* logp_ref, const float* values, const float* score, int B, int R,
                        float kl_ctl, float clip_reward, float gamma, float lam, float* rewards, float* adv, float* ret,
                        rlhf_stream_t s) {
  if (B < 1 || R < 1) return 2;
  gae_kernel<<<(B + 3) / 4, 128, 0, HS(s)>>>(logp, logp_ref, values, score, B, R, kl_ctl, clip_reward, gamma, lam,
                                             rewards, adv, ret);
  return HST();
}

extern "C" int rlhf_ppo_actor_loss(const float* logp, const float* logp_old, const float* adv, int n, float clip,
                                   float denom, float* g, float* loss_sum, rlhf_stream_t s) {
  actor_loss_kernel<<<1, 1024, 0, HS(s)>>>(logp, logp_old, adv, n, clip, denom, g, loss_sum);
  return HST();
}

extern "C" int rlhf_ppo_critic_loss(const float* v, const float* v_old, const float* ret, int n, float clip, float denom,
                                    float* g, float* loss_sum, rlhf_stream_t s) {
  critic_loss_kernel<<<1, 1024, 0, HS(s)>>>(v, v_old, ret, n, clip, denom, g, loss_sum);
  return HST();
}

extern "C" int rlhf_experience_stats(const float* logp, const float* logp_ref, const float* score, int B, int R,
                                     float* out, rlhf_stream_t s) {
  if (B < 1 || R < 1) return 2;
  experience_stats_kernel<<<1, 1024, 0, HS(s)>>>(logp, logp_ref, score, B, R, out);
  return HST();
}

extern "C" int rlhf_argmax_tiles(const float* top2, int tiles, int B, int32_t* tok, int64_t tok_stride, int* pos,
                                 float* margin, int advance_pos, rlhf_stream_t s) {
  if (tiles < 1 || B < 1 || !pos) return 2;
  return launch_k(argmax_tiles_kernel, dim3(B), dim3(kArgmaxThreads), 0, reinterpret_cast<cudaStream_t>(s),
                  reinterpret_cast<const float4*>(top2), tiles, B, tok, tok_stride, pos, margin, advance_pos);
}

extern "C" int rlhf_lse_merge(const float* lse_part, const float* lse_tgt, int rows, int parts, float* logp,
                              rlhf_stream_t s) {
  if (rows < 1 || parts < 1) return 2;
  lse_merge_kernel<<<(rows + 7) / 8, 256, 0, HS(s)>>>(reinterpret_cast<const float2*>(lse_part), lse_tgt, rows, parts, logp);
  return HST();
}
