// attention.cu — causal softmax (fwd/bwd) over tcgen05-GEMM scores, KV-cache
// store and the HBM-bound decode attention of the Generation stage.
// Probabilities are normalised then rounded to bf16 before P.V (DESIGN.md §3,
// oracle/ppo_oracle.cpp forward_chunk).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdlib>

#include "launch_util.cuh"
#include "sm100_common.cuh"
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

// One CTA per (sample, head).  The key and value rows [0, ctx) of the head are
// streamed into shared memory with bulk async copies (cp.async.bulk, one
// mbarrier per 64-row block) through two rings of NS blocks each: the first NS
// key blocks and NS value blocks are in flight from the first instruction, and
// every consumed block's slot is refilled NS blocks ahead, so the CTA never
// waits for more than the HBM stream.  Scores: LPR lanes per key row (16 B
// each, conflict-free rows), block softmax, bf16-rounded probabilities, then
// P.V with a (dim chunk, key group) thread split over the staged value rows.
template <int HD, int NS_ = (HD == 64 ? 4 : 2)>
struct DecCfg {
  static constexpr int RB = 64;                     // rows per block (one bulk copy, one mbarrier)
  static constexpr int NS = NS_;                    // ring slots per K / V (default: K + V = 64 KB)
  static constexpr int LPR = HD / 8;                // lanes per key row
  static constexpr int RPW = 32 / LPR;              // key rows per warp pass
  static constexpr size_t smem(int Smax) {
    return static_cast<size_t>(2) * NS * RB * HD * 2 + static_cast<size_t>((Smax + 3) / 4 * 4) * 4 + HD * 4;
  }
};

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// block blk (rows [64 blk, +64) clipped to ctx) of src -> ring slot blk % NS
template <int HD, int NS>
__device__ __forceinline__ void dec_issue(uint16_t* ring, const uint16_t* src, int blk, int ctx, uint64_t* bars) {
  using Cf = DecCfg<HD, NS>;
  const int rows = min(Cf::RB, ctx - blk * Cf::RB);
  if (rows <= 0) return;
  const int slot = blk % Cf::NS;
  mbar_arrive_expect_tx(&bars[slot], static_cast<uint32_t>(rows * HD * 2));
  bulk_g2s(ring + slot * Cf::RB * HD, src + static_cast<int64_t>(blk) * Cf::RB * HD, static_cast<uint32_t>(rows * HD * 2),
           &bars[slot]);
}

__device__ __forceinline__ void prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

template <int HD, int NS_>
__global__ void __launch_bounds__(kDecThreads) attn_decode_kernel(const uint16_t* __restrict__ qkv, int H, int Smax,
                                                                  const uint16_t* __restrict__ kc,
                                                                  const uint16_t* __restrict__ vc,
                                                                  const int* __restrict__ pos_dev,
                                                                  uint16_t* __restrict__ out,
                                                                  const uint16_t* __restrict__ kc_next,
                                                                  const uint16_t* __restrict__ vc_next) {
  using Cf = DecCfg<HD, NS_>;
  constexpr int RB = Cf::RB, NS = Cf::NS, LPR = Cf::LPR, RPW = Cf::RPW, NW = kDecThreads / 32;
  extern __shared__ __align__(128) uint8_t dsm[];
  uint16_t* Ks = reinterpret_cast<uint16_t*>(dsm);
  uint16_t* Vs = Ks + NS * RB * HD;
  float* sc = reinterpret_cast<float*>(Vs + NS * RB * HD);
  float* q = sc + (Smax + 3) / 4 * 4;
  __shared__ float red[NW];
  __shared__ uint64_t kbar[NS], vbar[NS];
  // Programmatic dependent launch: only the new row `pos` (K/V written by the QKV GEMM's
  // epilogue) and q depend on the predecessor.  The position counter and the cached rows
  // [0, pos) were final before the predecessor started (every earlier kernel of the step
  // chain waited on its own predecessor), so their bulk loads are issued before
  // griddepcontrol.wait and stream while the QKV GEMM is still running.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int bh = blockIdx.x, b = bh / H, h = bh % H;
  const int d = H * HD;
  const int pos = *pos_dev;
  const int ctx = pos + 1;
  const int nblk = (ctx + RB - 1) / RB;
  const uint16_t* K = kc + static_cast<int64_t>(bh) * Smax * HD;
  const uint16_t* V = vc + static_cast<int64_t>(bh) * Smax * HD;
  const int npre = min(NS, pos / RB);  // leading blocks made only of cached rows
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NS; ++i) {
      mbar_init(&kbar[i], 1);
      mbar_init(&vbar[i], 1);
    }
    mbar_fence_init();
    for (int i = 0; i < npre; ++i) {
      dec_issue<HD, NS>(Ks, K, i, ctx, kbar);
      dec_issue<HD, NS>(Vs, V, i, ctx, vbar);
    }
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) {
    for (int i = npre; i < NS; ++i) {
      dec_issue<HD, NS>(Ks, K, i, ctx, kbar);
      dec_issue<HD, NS>(Vs, V, i, ctx, vbar);
    }
  }
  const float scale = rsqrtf(static_cast<float>(HD));
  const uint16_t* qsrc = qkv + static_cast<int64_t>(b) * 3 * d + h * HD;
  for (int e = threadIdx.x; e < HD; e += kDecThreads) q[e] = bf2f_a(qsrc[e]);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = lane % LPR, rsub = lane / LPR;
  float qr[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) qr[t] = q[sub * 8 + t];
  float mx = -FLT_MAX;
  for (int blk = 0; blk < nblk; ++blk) {
    const int slot = blk % NS;
    mbar_wait(&kbar[slot], (blk / NS) & 1);
    const int rows = min(RB, ctx - blk * RB);
    const uint16_t* Kb = Ks + slot * RB * HD;
    for (int r0 = warp * RPW; r0 < rows; r0 += NW * RPW) {  // warp-uniform trip count
      const int r = r0 + rsub;
      float s = 0.f;
      if (r < rows) {
        const uint4 u = *reinterpret_cast<const uint4*>(Kb + r * HD + sub * 8);
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          s += qr[2 * t] * bf2f_a(static_cast<uint16_t>(w[t] & 0xFFFFu));
          s += qr[2 * t + 1] * bf2f_a(static_cast<uint16_t>(w[t] >> 16));
        }
      }
#pragma unroll
      for (int o = LPR / 2; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (sub == 0 && r < rows) {
        s *= scale;
        sc[blk * RB + r] = s;
        mx = fmaxf(mx, s);
      }
    }
    if (blk + NS < nblk) {
      __syncthreads();  // every warp is done with this slot
      if (threadIdx.x == 0) {
        fence_proxy_async_smem();
        dec_issue<HD, NS>(Ks, K, blk + NS, ctx, kbar);
      }
    }
  }
  mx = wmax(mx);
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  mx = red[0];
#pragma unroll
  for (int w = 1; w < NW; ++w) mx = fmaxf(mx, red[w]);
  __syncthreads();
  float sum = 0.f;
  for (int j = threadIdx.x; j < ctx; j += kDecThreads) {
    const float e = expf(sc[j] - mx);
    sc[j] = e;
    sum += e;
  }
  sum = wsum(sum);
  if (lane == 0) red[warp] = sum;
  __syncthreads();
  sum = 0.f;
#pragma unroll
  for (int w = 0; w < NW; ++w) sum += red[w];
  const float inv = 1.0f / sum;
  // O[e] = sum_j bf16(p_j) V[j][e]: thread = (16-byte dim chunk cc, key group grp)
  constexpr int CH = HD / 8;
  constexpr int G = kDecThreads / CH;
  const int cc = threadIdx.x % CH, grp = threadIdx.x / CH;
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  for (int blk = 0; blk < nblk; ++blk) {
    const int slot = blk % NS;
    mbar_wait(&vbar[slot], (blk / NS) & 1);
    const int rows = min(RB, ctx - blk * RB);
    const uint16_t* Vb = Vs + slot * RB * HD;
#pragma unroll
    for (int r = grp; r < RB; r += G) {
      if (r >= rows) break;
      const float pj = bf2f_a(f2bf_a(sc[blk * RB + r] * inv));
      const uint4 u = *reinterpret_cast<const uint4*>(Vb + r * HD + cc * 8);
      const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        acc[2 * t] += pj * bf2f_a(static_cast<uint16_t>(w[t] & 0xFFFFu));
        acc[2 * t + 1] += pj * bf2f_a(static_cast<uint16_t>(w[t] >> 16));
      }
    }
    if (blk + NS < nblk) {
      __syncthreads();
      if (threadIdx.x == 0) {
        fence_proxy_async_smem();
        dec_issue<HD, NS>(Vs, V, blk + NS, ctx, vbar);
      }
    }
  }
  float* part = reinterpret_cast<float*>(Ks);  // [G][HD] partials (key ring no longer needed)
  __syncthreads();
#pragma unroll
  for (int t = 0; t < 8; ++t) part[grp * HD + cc * 8 + t] = acc[t];
  __syncthreads();
  for (int e = threadIdx.x; e < HD; e += kDecThreads) {
    float o = 0.f;
    for (int g2 = 0; g2 < G; ++g2) o += part[g2 * HD + e];
    out[static_cast<int64_t>(b) * d + h * HD + e] = f2bf_a(o);
  }
  // The next attention of the step chain (layer l+1, or layer 0 of the next step) reads this
  // (sample, head)'s cached rows [0, ctx) of its own layer: nothing computed in between
  // changes them, so they are pulled into L2 now, while the latency-bound O-proj / FFN /
  // QKV kernels leave HBM mostly idle, and that attention streams them from L2.
  if (kc_next && threadIdx.x < 2) {
    const uint16_t* src = (threadIdx.x == 0 ? kc_next : vc_next) + static_cast<int64_t>(bh) * Smax * HD;
    for (int blk = 0; blk < nblk; ++blk) {
      const int rows = min(RB, ctx - blk * RB);
      prefetch_l2(src + static_cast<int64_t>(blk) * RB * HD, static_cast<uint32_t>(rows * HD * 2));
    }
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

template <int HD, int NS>
static int launch_dec_ns(int grid, cudaStream_t st, const uint16_t* q, int H, int Smax, const uint16_t* k,
                         const uint16_t* v, const int* pos_dev, uint16_t* o, const uint16_t* kn, const uint16_t* vn) {
  const size_t smem = DecCfg<HD, NS>::smem(Smax);
  static size_t configured = 0;  // per-instantiation opt-in to > 48 KB dynamic shared memory
  if (smem > configured) {
    if (cudaFuncSetAttribute(attn_decode_kernel<HD, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem)) != cudaSuccess)
      return 5;
    configured = smem;
  }
  return launch_k(attn_decode_kernel<HD, NS>, dim3(grid), dim3(kDecThreads), smem, st, q, H, Smax, k, v, pos_dev, o, kn,
                  vn);
}

template <int HD>
static int launch_dec(int grid, cudaStream_t st, const uint16_t* q, int H, int Smax, const uint16_t* k, const uint16_t* v,
                      const int* pos_dev, uint16_t* o, const uint16_t* kn, const uint16_t* vn) {
  // RLHF_ATTN_NS: ring depth override (timing experiments only)
  static const int ns = [] { const char* e = getenv("RLHF_ATTN_NS"); return e ? atoi(e) : 0; }();
  switch (ns) {
    case 1: return launch_dec_ns<HD, 1>(grid, st, q, H, Smax, k, v, pos_dev, o, kn, vn);
    case 2: return launch_dec_ns<HD, 2>(grid, st, q, H, Smax, k, v, pos_dev, o, kn, vn);
    case 4: return launch_dec_ns<HD, 4>(grid, st, q, H, Smax, k, v, pos_dev, o, kn, vn);
    case 8: return launch_dec_ns<HD, 8>(grid, st, q, H, Smax, k, v, pos_dev, o, kn, vn);
    default: break;
  }
  // one wave: 4 ring slots (3 CTAs / SM) while the (sample, head) grid fits, else 3 slots
  // (4 CTAs / SM), else 2
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  if (HD == 128 || grid <= 3 * sms) return launch_dec_ns<HD, DecCfg<HD>::NS>(grid, st, q, H, Smax, k, v, pos_dev, o, kn, vn);
  if (grid <= 4 * sms) return launch_dec_ns<HD, 3>(grid, st, q, H, Smax, k, v, pos_dev, o, kn, vn);
  return launch_dec_ns<HD, 2>(grid, st, q, H, Smax, k, v, pos_dev, o, kn, vn);
}

extern "C" int rlhf_attn_decode_prefetch(const void* qkv, int B, int H, int hd, int Smax, const void* kcache,
                                         const void* vcache, const int* pos_dev, void* out, const void* kcache_next,
                                         const void* vcache_next, rlhf_stream_t s) {
  if (Smax > kDecMaxCtx) return 2;
  if (!kcache_next != !vcache_next) return 2;
  const auto* q = static_cast<const uint16_t*>(qkv);
  const auto* k = static_cast<const uint16_t*>(kcache);
  const auto* v = static_cast<const uint16_t*>(vcache);
  const auto* kn = static_cast<const uint16_t*>(kcache_next);
  const auto* vn = static_cast<const uint16_t*>(vcache_next);
  auto* o = static_cast<uint16_t*>(out);
  switch (hd) {
    case 64: return launch_dec<64>(B * H, AS(s), q, H, Smax, k, v, pos_dev, o, kn, vn);
    case 128: return launch_dec<128>(B * H, AS(s), q, H, Smax, k, v, pos_dev, o, kn, vn);
    default: return 2;
  }
}

extern "C" int rlhf_attn_decode(const void* qkv, int B, int H, int hd, int Smax, const void* kcache, const void* vcache,
                                const int* pos_dev, void* out, rlhf_stream_t s) {
  return rlhf_attn_decode_prefetch(qkv, B, H, hd, Smax, kcache, vcache, pos_dev, out, nullptr, nullptr, s);
}
