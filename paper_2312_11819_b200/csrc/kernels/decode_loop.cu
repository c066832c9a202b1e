// decode_loop.cu — the Generation stage's greedy decode loop as ONE persistent
// kernel (all R-1 decode steps of all layers in a single launch).
//
// Why: at B = 32 / GPU the decode step is latency-bound.  As separate kernels
// (even PDL-chained inside a CUDA graph) every launch pays ~5 us of fixed cost
// (grid ramp, first HBM round trip, drain), and a step of an L-layer decoder is
// ~7L launches.  Here one CTA per SM runs the whole loop; phases are separated
// by a grid-wide barrier (~1 us) and, crucially, the weight stream never stops:
// a producer warp walks this CTA's whole schedule of weight tiles ahead of the
// math, so weight HBM traffic overlaps barriers, attention and LayerNorms.
//
// Warp roles (384 threads, 1 CTA / SM, cooperative launch):
//   warp 0      weight producer: TMA of 128x64 weight tiles into a ring (prefetch
//               runs ahead across phases / layers / steps, gated only by the ring)
//   warp 1      TMEM owner + single-thread tcgen05.mma issuer (swap-AB: weight
//               rows = M 128, batch = N (32 | 64), fp32 accumulators, 2 buffers)
//   warp 2      activation producer: TMA of the (N x 64) activation tile, issued
//               once the grid barrier that publishes the activations has passed
//   warps 4-11  compute: GEMM epilogues (TMEM -> split-K partials / LM top-2),
//               attention, residual + LayerNorm, FFN activation, argmax + embed
//
// Phases of one step (L layers), each followed by a grid barrier:
//   per layer: QKV-GEMM | ATT | WO-GEMM | RES+LN2 | W1-GEMM | RELU | W2-GEMM | RES+LN1'
//   then:      LM-GEMM (per-tile top-2 epilogue, logits never stored) | ARGMAX+EMBED+LN1
// Split-K partials go to an fp32 workspace [split][b][m] and are reduced by the
// consuming phase in fixed split order (deterministic, no atomics).
//
// Numerics follow the per-kernel decode path: bf16 GEMM operands,
// fp32 accumulation, qkv / h / o / f rounded to bf16, fp32 residual stream,
// probabilities normalised then rounded to bf16, greedy ties -> lowest token id.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cfloat>
#include <cstdio>
#include <mutex>

#include "rlhf_init.h"
#include "rlhf_kernels.h"
#include "sm100_common.cuh"

namespace rlhf {
namespace dl {

constexpr int BM = 128, BK = 64;
constexpr int kWarps = 12, kThreads = kWarps * 32;
constexpr int kCT = 256;                 // compute threads (warps 4..11)
constexpr int kWT = BM * BK * 2;         // weight tile bytes (== kSlot)
constexpr int kSlot = 16384;             // pool slot: one 128x64 weight tile or one K / V block
constexpr uint32_t kBarC = 1, kBarE = 2;  // named barriers: compute warps, epilogue warps
constexpr int kQN = 4;                   // attention units whose q/k/v are reduced together

enum { M_QKV = 0, M_WO, M_W1, M_W2, M_LM, M_XH, M_XO, M_XF, M_KC, M_VC, NMAP };
struct Maps {
  CUtensorMap m[NMAP];
};

struct Args {
  int d, H, ff, V, L, B, S;
  int64_t per_layer;
  const uint16_t *tok_emb, *pos_emb, *ln1_g, *ln1_b, *bqkv, *bo, *ln2_g, *ln2_b, *b1, *b2, *lnf_g, *lnf_b;
  int32_t* tokens;
  int32_t* pred;
  float* margin;
  int* pos;
  int steps;
  uint16_t *kc, *vc;
  int kvB, Smax;
  unsigned* gbar;
  float* x;
  uint16_t *hbuf, *obuf, *fbuf;
  float* part;
  int G, np, xs, tmem_cols;
  int S_[5], kbper_[5];
  unsigned long long* probe;
  int probe_q;
};

struct Shape {
  int M, KB, kbper, S, T, U;
};

__device__ __forceinline__ Shape shape_of(const Args& a, int j) {
  Shape s;
  s.M = j == M_QKV ? 3 * a.d : (j == M_W1 ? a.ff : (j == M_LM ? a.V : a.d));
  s.KB = (j == M_W2 ? a.ff : a.d) / BK;
  s.kbper = a.kbper_[j];
  s.S = a.S_[j];
  s.T = (s.M + BM - 1) / BM;
  s.U = s.T * s.S;
  return s;
}

// phase q of a step (P = 8L + 2 phases): GEMM map id or -1, and the layer
__device__ __forceinline__ int gemm_of(int q, int L, int& layer) {
  layer = 0;
  if (q == 8 * L) return M_LM;
  if (q > 8 * L) return -1;
  layer = q / 8;
  switch (q % 8) {
    case 0: return M_QKV;
    case 2: return M_WO;
    case 4: return M_W1;
    case 6: return M_W2;
    default: return -1;
  }
}
__device__ __forceinline__ bool is_att(int q, int L) { return q < 8 * L && q % 8 == 1; }
__device__ __forceinline__ int units_of(int cta, int G, int n) { return cta < n ? (n - 1 - cta) / G + 1 : 0; }
__device__ __forceinline__ int xmap_of(int j) { return j == M_WO ? M_XO : (j == M_W2 ? M_XF : M_XH); }

__device__ __forceinline__ float b2f(uint16_t h) { return __uint_as_float(static_cast<uint32_t>(h) << 16); }
__device__ __forceinline__ uint16_t f2b(float f) { return __bfloat16_as_ushort(__float2bfloat16_rn(f)); }
__device__ __forceinline__ float rbf(float f) { return b2f(f2b(f)); }

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Spin until *p >= target.  Relaxed polls (an acquire load per iteration would
// invalidate this SM's L1 on every trip and slow every other warp on the SM),
// then one acquire fence.
__device__ __forceinline__ void wait_geq(const unsigned* p, unsigned target, int sleep_ns) {
  while (ld_relaxed(p) < target) {
    if (sleep_ns) __nanosleep(sleep_ns);
  }
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async;" ::: "memory"); }
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// streaming loads (weights, cached K / V): evict-first in L2 so the small hot
// data (workspace, parameter pack) stays resident
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d_hint(void* smem, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2,
                                                 int c3, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], %7;" ::"r"(smem_u32(smem)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "l"(pol)
      : "memory");
}

// warp-level bf16 MMA m16n8k16 (fp32 accumulate) and transposed 8x8 matrix loads:
// the decode attention of head dim 64 runs its q.K^T and P.V on these
__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                               uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldsm_x2_trans(uint32_t addr, uint32_t& r0, uint32_t& r1) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0, %1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(addr));
}
__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  return static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(lo))) |
         (static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(hi))) << 16);
}

struct Top2 {
  float v1;
  int i1;
  float v2;
};
__device__ __forceinline__ Top2 top2_merge(Top2 a, Top2 b) {
  Top2 r;
  if (b.v1 > a.v1 || (b.v1 == a.v1 && b.i1 < a.i1)) {
    r.v1 = b.v1; r.i1 = b.i1; r.v2 = fmaxf(a.v1, b.v2);
  } else {
    r.v1 = a.v1; r.i1 = a.i1; r.v2 = fmaxf(a.v2, b.v1);
  }
  return r;
}
__device__ __forceinline__ Top2 top2_warp(Top2 t) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    Top2 u{__shfl_xor_sync(0xffffffffu, t.v1, o), __shfl_xor_sync(0xffffffffu, t.i1, o),
           __shfl_xor_sync(0xffffffffu, t.v2, o)};
    t = top2_merge(t, u);
  }
  return t;
}

constexpr int kMaxSplit = 8;  // split-K partials per output (plan() caps S)

// sum_{s < S} p[s * stride] in fixed order; every load is issued before the adds
__device__ __forceinline__ float sum_splits(const float* p, int64_t stride, int S) {
  float v[kMaxSplit];
#pragma unroll
  for (int sp = 0; sp < kMaxSplit; ++sp) v[sp] = sp < S ? __ldcg(p + sp * stride) : 0.f;
  float r = 0.f;
#pragma unroll
  for (int sp = 0; sp < kMaxSplit; ++sp)
    if (sp < S) r += v[sp];
  return r;
}

// block-wide (compute warps) sum; red = 8 floats of smem
__device__ __forceinline__ float csum(float v, float* red, int cw, int lane) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) red[cw] = v;
  named_bar_sync(kBarC, kCT);
  float s = 0.f;
#pragma unroll
  for (int w = 0; w < kCT / 32; ++w) s += red[w];
  named_bar_sync(kBarC, kCT);
  return s;
}
__device__ __forceinline__ float cmax(float v, float* red, int cw, int lane) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (lane == 0) red[cw] = v;
  named_bar_sync(kBarC, kCT);
  float s = red[0];
#pragma unroll
  for (int w = 1; w < kCT / 32; ++w) s = fmaxf(s, red[w]);
  named_bar_sync(kBarC, kCT);
  return s;
}

// residual row b of width d: x += bias + sum_s part[s][b][:]; y = bf16(LN(x) * g + beta)
template <int MAXV>
__device__ __forceinline__ void res_ln_row(const Args& a, int b, int S, const uint16_t* bias, const uint16_t* g,
                                           const uint16_t* beta, float* red, int ctid, int cw, int lane, bool add,
                                           unsigned long long* sp = nullptr) {
  const int d = a.d;
  float xv[MAXV], gv[MAXV], bv[MAXV];
  float sum = 0.f;
#pragma unroll
  for (int k = 0; k < MAXV; ++k) {
    const int c = ctid + k * kCT;
    gv[k] = c < d ? b2f(g[c]) : 0.f;
    bv[k] = c < d ? b2f(beta[c]) : 0.f;
  }
#pragma unroll
  for (int k = 0; k < MAXV; ++k) {
    const int c = ctid + k * kCT;
    xv[k] = 0.f;
    if (c < d) {
      float xn = __ldcg(a.x + static_cast<int64_t>(b) * d + c);
      if (add) {
        const float s = sum_splits(a.part + static_cast<int64_t>(b) * d + c, static_cast<int64_t>(a.B) * d, S);
        xn = (s + b2f(bias[c])) + xn;
        a.x[static_cast<int64_t>(b) * d + c] = xn;
      }
      xv[k] = xn;
      sum += xn;
    }
  }
  if (sp) *sp = gtime();
  const float mu = csum(sum, red, cw, lane) / d;
  float vs = 0.f;
#pragma unroll
  for (int k = 0; k < MAXV; ++k)
    if (ctid + k * kCT < d) vs += (xv[k] - mu) * (xv[k] - mu);
  const float rs = 1.0f / sqrtf(csum(vs, red, cw, lane) / d + 1e-5f);
  if (sp) sp[1] = gtime();
#pragma unroll
  for (int k = 0; k < MAXV; ++k) {
    const int c = ctid + k * kCT;
    if (c < d) a.hbuf[static_cast<int64_t>(b) * d + c] = f2b((xv[k] - mu) * rs * gv[k] + bv[k]);
  }
}

template <int BN, int HD>
__global__ void __launch_bounds__(kThreads, 1)
    decode_loop_kernel(const __grid_constant__ Maps maps, const __grid_constant__ Args a) {
  constexpr int XT = BN * BK * 2;  // activation tile bytes
  constexpr int NEPI = BN / 32 * 4;  // epilogue warps
  constexpr int KVR = kSlot / (HD * 2);  // cached K / V rows per pool slot
  constexpr int LPR = HD / 8, RPW = 32 / LPR;
  constexpr int WAVE = (kCT / 32) * RPW, NWV = KVR / WAVE;  // score pass: rows per CTA pass, passes per block
  constexpr int NRV = KVR / (kCT / (HD / 8));               // P.V: rows per thread per block
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // pool: ONE ring of 16 KB slots shared, in schedule order, by the weight tiles
  // of GEMM phases and the cached K / V blocks of attention phases
  uint8_t* pool = smem;
  uint8_t* xring = pool + a.np * kSlot;
  float* sc = reinterpret_cast<float*>(xring + a.xs * XT);
  float* qn = sc + ((a.Smax + 3) & ~3);  // [kQN units][3][HD]
  float* pacc = qn + kQN * 3 * HD;       // [kCT / (HD / 8)][HD] P.V partials (8 KB)
  float* red = pacc + 2048;              // 8
  Top2* t2s = reinterpret_cast<Top2*>(red + 8);  // [8][32]
  int* itok = reinterpret_cast<int*>(t2s + 8 * 32);
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uintptr_t>(itok + 4 + 7) & ~uintptr_t(7));
  uint64_t* p_full = bars;
  uint64_t* p_empty = p_full + a.np;
  uint64_t* x_full = p_empty + a.np;
  uint64_t* x_empty = x_full + a.xs;
  uint64_t* acc_full = x_empty + a.xs;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = static_cast<int>(warp_id()), lane = static_cast<int>(lane_id());
  const int cta = blockIdx.x, G = a.G, L = a.L;
  const int P = 8 * L + 2;
  const int nphase = 1 + a.steps * P;
  const int pos0 = *a.pos;
  const int natt = units_of(cta, G, a.B * a.H);  // attention units of this CTA
  auto kv_blocks = [&](int gq) { return (pos0 + (gq - 1) / P + KVR - 1) / KVR; };  // per K (or V) stream

  if (threadIdx.x == 0) {
    for (int i = 0; i < a.np; ++i) {
      mbar_init(&p_full[i], 1);
      mbar_init(&p_empty[i], 1);
    }
    for (int i = 0; i < a.xs; ++i) {
      mbar_init(&x_full[i], 1);
      mbar_init(&x_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], NEPI);
    }
    mbar_fence_init();
    for (int i = 0; i < NMAP; ++i) tma_prefetch(&maps.m[i]);
  }
  if (warp == 1) tmem_alloc(tmem_slot, a.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- pool producer: weight tiles + cached K / V blocks ----------------
    if (lane == 0) {
      uint32_t it = 0;
      const uint64_t pol = policy_evict_first();
      auto slot_acquire = [&](uint32_t bytes) {
        const int st = static_cast<int>(it % a.np);
        if (it >= static_cast<uint32_t>(a.np)) mbar_wait(&p_empty[st], ((it / a.np) - 1) & 1);
        mbar_arrive_expect_tx(&p_full[st], bytes);
        ++it;
        return st;
      };
      for (int gq = 1; gq < nphase; ++gq) {
        const int q = (gq - 1) % P;
        int layer;
        const int j = gemm_of(q, L, layer);
        if (j == M_LM) {  // k-block major over this CTA's vocabulary tiles (one X tile per k-block)
          const Shape sh = shape_of(a, j);
          const int nu = units_of(cta, G, sh.U);
          for (int kb = 0; kb < sh.KB; ++kb)
            for (int k = 0; k < nu; ++k) {
              const int st = slot_acquire(kWT);
              tma_load_4d_hint(pool + st * kSlot, &maps.m[j], &p_full[st], kb * BK, 0, (cta + k * G) * BM, 0, pol);
            }
        } else if (j >= 0) {
          const Shape sh = shape_of(a, j);
          for (int u = cta; u < sh.U; u += G) {
            const int tile = u / sh.S, split = u % sh.S;
            const int kb0 = split * sh.kbper, kb1 = min(sh.KB, kb0 + sh.kbper);
            for (int kb = kb0; kb < kb1; ++kb) {
              const int st = slot_acquire(kWT);
              tma_load_4d_hint(pool + st * kSlot, &maps.m[j], &p_full[st], kb * BK, 0, tile * BM, layer, pol);
            }
          }
        } else if (is_att(q, L) && natt > 0) {
          const int pos = pos0 + (gq - 1) / P, nblk = kv_blocks(gq);
          // row pos-1 of this layer was appended by this CTA one step ago
          if (gq > P) {
            wait_geq(a.gbar, static_cast<unsigned>(gq - P + 1) * G, 256);
            fence_proxy_async();
          }
          for (int k = 0; k < natt; ++k) {
            const int u = cta + k * G, b = u / a.H, h = u % a.H;
            const int64_t head = ((static_cast<int64_t>(layer) * a.kvB + b) * a.H + h) * a.Smax * HD;
            for (int isv = 0; isv < 2; ++isv)
              for (int i = 0; i < nblk; ++i) {
                if constexpr (HD == 64) {
                  // SWIZZLE_128B tile of KVR rows (rows >= pos are masked by the consumer)
                  const int st = slot_acquire(kSlot);
                  tma_load_4d_hint(pool + st * kSlot, &maps.m[isv ? M_VC : M_KC], &p_full[st], 0, 0, i * KVR,
                                   (layer * a.kvB + b) * a.H + h, pol);
                } else {
                  const uint32_t bytes = static_cast<uint32_t>(min(KVR, pos - i * KVR) * HD * 2);
                  const int st = slot_acquire(bytes);
                  bulk_g2s_hint(pool + st * kSlot, (isv ? a.vc : a.kc) + head + static_cast<int64_t>(i) * KVR * HD,
                                bytes, &p_full[st], pol);
                }
              }
          }
        }
      }
    }
  } else if (warp == 2) {
    // ---------------- activation producer ----------------
    if (lane == 0) {
      uint32_t it = 0;
      for (int gq = 1; gq < nphase; ++gq) {
        int layer;
        const int j = gemm_of((gq - 1) % P, L, layer);
        if (j < 0) continue;
        const Shape sh = shape_of(a, j);
        if (cta >= sh.U) continue;
        // activations of phase gq are published by grid barrier gq-1
        wait_geq(a.gbar, static_cast<unsigned>(gq) * G, 64);
        fence_proxy_async();
        const CUtensorMap* xm = &maps.m[xmap_of(j)];
        if (j == M_LM) {
          for (int kb = 0; kb < sh.KB; ++kb, ++it) {
            const int st = static_cast<int>(it % a.xs);
            if (it >= static_cast<uint32_t>(a.xs)) mbar_wait(&x_empty[st], ((it / a.xs) - 1) & 1);
            mbar_arrive_expect_tx(&x_full[st], XT);
            tma_load_4d(xring + st * XT, xm, &x_full[st], kb * BK, 0, 0, 0);
          }
          continue;
        }
        for (int u = cta; u < sh.U; u += G) {
          const int split = u % sh.S;
          const int kb0 = split * sh.kbper, kb1 = min(sh.KB, kb0 + sh.kbper);
          for (int kb = kb0; kb < kb1; ++kb, ++it) {
            const int st = static_cast<int>(it % a.xs);
            if (it >= static_cast<uint32_t>(a.xs)) mbar_wait(&x_empty[st], ((it / a.xs) - 1) & 1);
            mbar_arrive_expect_tx(&x_full[st], XT);
            tma_load_4d(xring + st * XT, xm, &x_full[st], kb * BK, 0, 0, 0);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      const uint32_t idesc = umma_idesc_bf16(BM, BN, 0, 0);
      uint32_t wit = 0, xit = 0, ucount = 0;
      for (int gq = 1; gq < nphase; ++gq) {
        int layer;
        const int j = gemm_of((gq - 1) % P, L, layer);
        if (is_att((gq - 1) % P, L)) wit += natt * 2 * kv_blocks(gq);  // pool entries the attention consumes
        if (j < 0) continue;
        const Shape sh = shape_of(a, j);
        if (j == M_LM) {
          // all of this CTA's vocabulary tiles at once: accumulator k at TMEM column k*BN
          const int nu = units_of(cta, G, sh.U);
          if (nu == 0) continue;
          const uint32_t ab = ucount & 1;
          if (ucount >= 1) mbar_wait(&acc_empty[ab ^ 1], ((ucount - 1) >> 1) & 1);
          if (ucount >= 2) mbar_wait(&acc_empty[ab], ((ucount >> 1) - 1) & 1);
          tc_fence_after();
          for (int kb = 0; kb < sh.KB; ++kb, ++xit) {
            const int xs = static_cast<int>(xit % a.xs);
            mbar_wait(&x_full[xs], (xit / a.xs) & 1);
            const uint32_t sb = smem_u32(xring + xs * XT);
            for (int k = 0; k < nu; ++k, ++wit) {
              const int ws = static_cast<int>(wit % a.np);
              mbar_wait(&p_full[ws], (wit / a.np) & 1);
              tc_fence_after();
              const uint32_t sa = smem_u32(pool + ws * kSlot);
#pragma unroll
              for (int kk = 0; kk < BK / 16; ++kk)
                umma_bf16(tmem + k * BN, umma_desc_sw128(sa + kk * 32, 16, 1024),
                          umma_desc_sw128(sb + kk * 32, 16, 1024), idesc, (kb > 0 || kk > 0) ? 1u : 0u);
              umma_commit(&p_empty[ws]);
            }
            umma_commit(&x_empty[xs]);
          }
          umma_commit(&acc_full[ab]);
          mbar_wait(&acc_empty[ab], (ucount >> 1) & 1);  // TMEM columns >= 2*BN free again
          ++ucount;
          continue;
        }
        for (int u = cta; u < sh.U; u += G, ++ucount) {
          const int split = u % sh.S;
          const int kb0 = split * sh.kbper, kb1 = min(sh.KB, kb0 + sh.kbper);
          const uint32_t ab = ucount & 1;
          if (ucount >= 2) mbar_wait(&acc_empty[ab], ((ucount >> 1) - 1) & 1);
          tc_fence_after();
          for (int kb = kb0; kb < kb1; ++kb, ++wit, ++xit) {
            const int ws = static_cast<int>(wit % a.np), xs = static_cast<int>(xit % a.xs);
            mbar_wait(&p_full[ws], (wit / a.np) & 1);
            mbar_wait(&x_full[xs], (xit / a.xs) & 1);
            tc_fence_after();
            const uint32_t sa = smem_u32(pool + ws * kSlot), sb = smem_u32(xring + xs * XT);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              umma_bf16(tmem + ab * BN, umma_desc_sw128(sa + k * 32, 16, 1024), umma_desc_sw128(sb + k * 32, 16, 1024),
                        idesc, (kb > kb0 || k > 0) ? 1u : 0u);
            umma_commit(&p_empty[ws]);
            umma_commit(&x_empty[xs]);
          }
          umma_commit(&acc_full[ab]);
        }
      }
    }
  } else if (warp >= 4) {
    // ---------------- compute warps ----------------
    const int ctid = static_cast<int>(threadIdx.x) - 128, cw = warp - 4;
    const int d = a.d, H = a.H, B = a.B;
    const float scale = rsqrtf(static_cast<float>(HD));
    int pos = *a.pos;
    uint32_t ucount = 0, pit = 0;  // accumulator count, pool position
    int layer = 0;
    for (int gq = 0; gq < nphase; ++gq) {
      const int q = gq == 0 ? P - 1 : (gq - 1) % P;
      const int step = gq == 0 ? -1 : (gq - 1) / P;
      const int j = gq == 0 ? -1 : gemm_of(q, L, layer);
      const bool tma_data = j < 0 && (gq == 0 || q == P - 1 || q % 8 == 3 || q % 8 == 7)
                                ? cta < B
                                : (j < 0 && q % 8 == 1 ? natt > 0 : (j < 0 && q % 8 == 5));
      // debug sub-probes (16 timestamps per CTA) inside phase probe_q of step 1
      const bool sp_on = a.probe && step == 1 && q == a.probe_q && ctid == 0;
      unsigned long long* spb = a.probe + static_cast<int64_t>(2 * P) * G + static_cast<int64_t>(cta) * 16;
#define ATT_PROBE(slot) do { if (sp_on && (slot) < 16) spb[(slot)] = gtime(); } while (0)
      if (j >= 0) {
        // ======== GEMM epilogue ========
        const Shape sh = shape_of(a, j);
        if (j == M_LM) {
          // per vocabulary tile and sample: top-2 (value, lowest id) over its 128 rows
          const int nu = units_of(cta, G, sh.U);
          pit += nu * sh.KB;
          if (nu > 0 && cw < NEPI) {
            const uint32_t ab = ucount & 1;
            mbar_wait(&acc_full[ab], (ucount >> 1) & 1);
            tc_fence_after();
            const int quarter = warp & 3, colbase = (cw / 4) * 32;
            for (int k = 0; k < nu; ++k) {
              const int tile = cta + k * G;
              float v[32];
              tmem_ld32(tmem + k * BN + colbase + (static_cast<uint32_t>(quarter * 32) << 16), v);
              const int m = tile * BM + quarter * 32 + lane;
              Top2 keep{-FLT_MAX, 0x7fffffff, -FLT_MAX};
#pragma unroll
              for (int c = 0; c < 32; ++c) {
                Top2 t{m < sh.M ? v[c] : -FLT_MAX, m < sh.M ? m : 0x7fffffff, -FLT_MAX};
                t = top2_warp(t);
                if (lane == c) keep = t;
              }
              t2s[cw * 32 + lane] = keep;
              named_bar_sync(kBarE, NEPI * 32);
              if (ctid < BN && ctid < B) {
                const int grp = ctid / 32, cl = ctid % 32;
                Top2 t = t2s[(grp * 4) * 32 + cl];
#pragma unroll
                for (int qq = 1; qq < 4; ++qq) t = top2_merge(t, t2s[(grp * 4 + qq) * 32 + cl]);
                float* o = a.part + (static_cast<int64_t>(tile) * B + ctid) * 4;
                __stcg(o, t.v1);
                __stcg(o + 1, __int_as_float(t.i1));
                __stcg(o + 2, t.v2);
              }
              named_bar_sync(kBarE, NEPI * 32);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[ab]);
          }
          if (nu > 0) ++ucount;
        } else
        for (int u = cta; u < sh.U; u += G, ++ucount) {
          const int tile = u / sh.S, split = u % sh.S;
          pit += min(sh.KB, (split + 1) * sh.kbper) - split * sh.kbper;
          const uint32_t ab = ucount & 1;
          if (cw < NEPI) {  // only the epilogue warps track the accumulator barriers
            mbar_wait(&acc_full[ab], (ucount >> 1) & 1);
            tc_fence_after();
            const int quarter = warp & 3, colbase = (cw / 4) * 32;
            float v[32];
            tmem_ld32(tmem + ab * BN + colbase + (static_cast<uint32_t>(quarter * 32) << 16), v);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[ab]);
            const int m = tile * BM + quarter * 32 + lane;
            if (m < sh.M) {
              float* dst = a.part + static_cast<int64_t>(split) * B * sh.M + m;
#pragma unroll
              for (int c = 0; c < 32; ++c)
                if (colbase + c < B) __stcg(dst + static_cast<int64_t>(colbase + c) * sh.M, v[c]);
            }
          }
        }
      } else if (gq > 0 && q < 8 * L && q % 8 == 1) {
        // ======== attention: one (b, h) per unit ========
        // This CTA's cached K / V rows [0, pos) arrive through the pool (the
        // producer streams them right behind the QKV weight tiles, so they fly
        // during the QKV phase and its barrier); q/k/v of kQN units are reduced
        // from the split-K partials together (one L2 round trip).
        const uint16_t* bq = a.bqkv + layer * a.per_layer;
        const int S = a.S_[M_QKV];
        const int nold = pos, nblk = (nold + KVR - 1) / KVR, per = 2 * nblk;
        const int nunits = natt;
        ATT_PROBE(0);
        for (int k0 = 0; k0 < nunits; k0 += kQN) {
          const int kn = min(kQN, nunits - k0);
          for (int i = ctid; i < kn * 3 * HD; i += kCT) {
            const int kk = k0 + i / (3 * HD), ii = i % (3 * HD);
            const int u = cta + kk * G, b = u / H, h = u % H;
            const int sec = ii / HD, e = ii % HD;
            const int col = sec * d + h * HD + e;
            const float s = sum_splits(a.part + static_cast<int64_t>(b) * 3 * d + col, static_cast<int64_t>(B) * 3 * d, S);
            const uint16_t hb = f2b(s + b2f(bq[col]));
            qn[i] = b2f(hb);
            if (sec > 0) {
              const int64_t head = ((static_cast<int64_t>(layer) * a.kvB + b) * H + h) * a.Smax * HD;
              (sec == 1 ? a.kc : a.vc)[head + static_cast<int64_t>(pos) * HD + e] = hb;
            }
          }
          named_bar_sync(kBarC, kCT);
          ATT_PROBE(1);
          for (int k = k0; k < k0 + kn; ++k) {
            const int u = cta + k * G, b = u / H, h = u % H;
            const float* qk = qn + (k - k0) * 3 * HD;
            if constexpr (HD == 64) {
              // ---- tensor cores: K / V blocks are SWIZZLE_128B tiles of KVR (128) rows:
              //      byte(r, dim) = r*128 + ((dim/8) ^ (r%8))*16 + (dim%8)*2  (conflict-free
              //      fragment loads).  q.K^T: warp cw owns key groups 2cw, 2cw+1 of each block,
              //      q is row 0 of the m16 A operand.  P.V: warp cw owns output dims 8cw..8cw+7.
              uint32_t qa0[4], qa2[4];
#pragma unroll
              for (int kc = 0; kc < 4; ++kc) {
                qa0[kc] = lane < 4 ? pack_bf16(qk[kc * 16 + lane * 2], qk[kc * 16 + lane * 2 + 1]) : 0u;
                qa2[kc] = lane < 4 ? pack_bf16(qk[kc * 16 + 8 + lane * 2], qk[kc * 16 + 8 + lane * 2 + 1]) : 0u;
              }
              float mx = -FLT_MAX;
              for (int i = 0; i < nblk; ++i) {
                const uint32_t gi = pit + k * per + i, slot = gi % a.np;
                mbar_wait(&p_full[slot], (gi / a.np) & 1);
                if (k == 0 && i < 3) ATT_PROBE(2 + 2 * i);
                const int rows = min(KVR, nold - i * KVR);
                const uint32_t kb_s = smem_u32(pool + slot * kSlot);
#pragma unroll
                for (int gg = 0; gg < 2; ++gg) {
                  const int g = 2 * cw + gg;
                  if (g * 8 >= rows) continue;
                  const int row = g * 8 + lane / 4;
                  const uint32_t base = kb_s + row * 128 + (lane % 4) * 4;
                  float dacc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                  for (int kc = 0; kc < 4; ++kc) {
                    const uint32_t b0 = lds32(base + (((2 * kc) ^ (row & 7)) << 4));
                    const uint32_t b1 = lds32(base + (((2 * kc + 1) ^ (row & 7)) << 4));
                    mma_bf16_16816(dacc, qa0[kc], 0u, qa2[kc], 0u, b0, b1);
                  }
                  if (lane < 4) {
                    const int key = g * 8 + lane * 2;
                    if (key < rows) {
                      const float sx = dacc[0] * scale;
                      sc[i * KVR + key] = sx;
                      mx = fmaxf(mx, sx);
                    }
                    if (key + 1 < rows) {
                      const float sx = dacc[1] * scale;
                      sc[i * KVR + key + 1] = sx;
                      mx = fmaxf(mx, sx);
                    }
                  }
                }
                named_bar_sync(kBarC, kCT);  // every warp is done with this slot
                if (k == 0 && i < 3) ATT_PROBE(3 + 2 * i);
                if (ctid == 0) mbar_arrive(&p_empty[slot]);
              }
              if (cw == 0) {  // the new key (position pos)
                float s = 0.f;
                for (int e = lane; e < HD; e += 32) s += qk[e] * qk[HD + e];
#pragma unroll
                for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                s *= scale;
                if (lane == 0) sc[nold] = s;
                mx = fmaxf(mx, s);
              }
              mx = cmax(mx, red, cw, lane);
              float sum = 0.f;
              for (int jj = ctid; jj <= nold; jj += kCT) {
                const float e = expf(sc[jj] - mx);
                sc[jj] = e;
                sum += e;
              }
              sum = csum(sum, red, cw, lane);
              const float inv = 1.0f / sum;
              if (k == 0) ATT_PROBE(8);
              float oacc[4] = {0.f, 0.f, 0.f, 0.f};
              for (int i = 0; i < nblk; ++i) {
                const uint32_t gi = pit + k * per + nblk + i, slot = gi % a.np;
                mbar_wait(&p_full[slot], (gi / a.np) & 1);
                if (k == 0 && i < 2) ATT_PROBE(9 + i);
                const int rows = min(KVR, nold - i * KVR);
                const uint32_t vb_s = smem_u32(pool + slot * kSlot);
                const float* sp = sc + i * KVR;
                const int nkc = (rows + 15) / 16;
                for (int kc = 0; kc < nkc; ++kc) {
                  uint32_t pa0 = 0u, pa2 = 0u;
                  if (lane < 4) {
                    const int j0 = kc * 16 + lane * 2, j2 = j0 + 8;
                    pa0 = pack_bf16(j0 < rows ? sp[j0] * inv : 0.f, j0 + 1 < rows ? sp[j0 + 1] * inv : 0.f);
                    pa2 = pack_bf16(j2 < rows ? sp[j2] * inv : 0.f, j2 + 1 < rows ? sp[j2 + 1] * inv : 0.f);
                  }
                  const int vrow = kc * 16 + (lane & 15);
                  uint32_t b0, b1;
                  ldsm_x2_trans(vb_s + vrow * 128 + ((cw ^ (vrow & 7)) << 4), b0, b1);
                  mma_bf16_16816(oacc, pa0, 0u, pa2, 0u, b0, b1);
                }
                named_bar_sync(kBarC, kCT);
                if (ctid == 0) mbar_arrive(&p_empty[slot]);
              }
              if (lane < 4) {  // + the new value row; lanes 0..3 hold dims 8cw + 2*lane, +1
                const float pj = rbf(sc[nold] * inv);
                const int e0 = cw * 8 + lane * 2;
                const float o0 = oacc[0] + pj * qk[2 * HD + e0];
                const float o1 = oacc[1] + pj * qk[2 * HD + e0 + 1];
                *reinterpret_cast<uint32_t*>(a.obuf + static_cast<int64_t>(b) * d + h * HD + e0) = pack_bf16(o0, o1);
              }
            } else {
            // scores of the cached keys (ring) and of the new key
            const int sub = lane % LPR, rsub = lane / LPR;
            float qr[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) qr[t] = qk[sub * 8 + t];
            float mx = -FLT_MAX;
            for (int i = 0; i < nblk; ++i) {
              const uint32_t gi = pit + k * per + i, slot = gi % a.np;
              mbar_wait(&p_full[slot], (gi / a.np) & 1);
              if (k == 0 && i < 2) ATT_PROBE(2 + 2 * i);
              const int rows = min(KVR, nold - i * KVR);
              const uint16_t* Kb = reinterpret_cast<const uint16_t*>(pool + slot * kSlot);
              // NWV independent row groups per warp (ILP): rows w*WAVE + cw*RPW + rsub
              float sv[NWV];
#pragma unroll
              for (int w = 0; w < NWV; ++w) {
                const int r = w * WAVE + cw * RPW + rsub;
                float s0 = 0.f, s1 = 0.f;
                if (r < rows) {
                  const uint4 w4 = *reinterpret_cast<const uint4*>(Kb + r * HD + sub * 8);
                  const uint32_t wd[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
                  for (int t = 0; t < 4; ++t) {
                    s0 += qr[2 * t] * b2f(static_cast<uint16_t>(wd[t] & 0xFFFFu));
                    s1 += qr[2 * t + 1] * b2f(static_cast<uint16_t>(wd[t] >> 16));
                  }
                }
                sv[w] = s0 + s1;
              }
#pragma unroll
              for (int o = LPR / 2; o; o >>= 1)
#pragma unroll
                for (int w = 0; w < NWV; ++w) sv[w] += __shfl_xor_sync(0xffffffffu, sv[w], o);
#pragma unroll
              for (int w = 0; w < NWV; ++w) {
                const int r = w * WAVE + cw * RPW + rsub;
                if (sub == 0 && r < rows) {
                  const float sx = sv[w] * scale;
                  sc[i * KVR + r] = sx;
                  mx = fmaxf(mx, sx);
                }
              }
              named_bar_sync(kBarC, kCT);  // every warp is done with this slot
              if (k == 0 && i < 2) ATT_PROBE(3 + 2 * i);
              if (ctid == 0) mbar_arrive(&p_empty[slot]);
            }
            if (cw == 0) {  // the new key (position pos)
              float s = 0.f;
              for (int e = lane; e < HD; e += 32) s += qk[e] * qk[HD + e];
#pragma unroll
              for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
              s *= scale;
              if (lane == 0) sc[nold] = s;
              mx = fmaxf(mx, s);
            }
            if (k == 0) ATT_PROBE(6);
            mx = cmax(mx, red, cw, lane);
            float sum = 0.f;
            for (int jj = ctid; jj <= nold; jj += kCT) {
              const float e = expf(sc[jj] - mx);
              sc[jj] = e;
              sum += e;
            }
            sum = csum(sum, red, cw, lane);
            const float inv = 1.0f / sum;
            if (k == 0) ATT_PROBE(7);
            constexpr int CH = HD / 8, GR = kCT / CH;
            const int cc = ctid % CH, grp = ctid / CH;
            float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            for (int i = 0; i < nblk; ++i) {
              const uint32_t gi = pit + k * per + nblk + i, slot = gi % a.np;
              mbar_wait(&p_full[slot], (gi / a.np) & 1);
              if (k == 0 && i < 2) ATT_PROBE(8 + 2 * i);
              const int rows = min(KVR, nold - i * KVR);
              const uint16_t* Vb = reinterpret_cast<const uint16_t*>(pool + slot * kSlot);
              uint4 w4[NRV];
              float pj[NRV];
#pragma unroll
              for (int m = 0; m < NRV; ++m) {
                const int r = grp + m * GR;
                if (r < rows) {
                  w4[m] = *reinterpret_cast<const uint4*>(Vb + r * HD + cc * 8);
                  pj[m] = rbf(sc[i * KVR + r] * inv);
                } else {
                  w4[m] = make_uint4(0u, 0u, 0u, 0u);
                  pj[m] = 0.f;
                }
              }
#pragma unroll
              for (int m = 0; m < NRV; ++m) {
                const uint32_t wd[4] = {w4[m].x, w4[m].y, w4[m].z, w4[m].w};
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                  acc[2 * t] += pj[m] * b2f(static_cast<uint16_t>(wd[t] & 0xFFFFu));
                  acc[2 * t + 1] += pj[m] * b2f(static_cast<uint16_t>(wd[t] >> 16));
                }
              }
              named_bar_sync(kBarC, kCT);
              if (k == 0 && i < 2) ATT_PROBE(9 + 2 * i);
              if (ctid == 0) mbar_arrive(&p_empty[slot]);
            }
            if (grp == 0) {  // the new value row
              const float pj = rbf(sc[nold] * inv);
#pragma unroll
              for (int t = 0; t < 8; ++t) acc[t] += pj * qk[2 * HD + cc * 8 + t];
            }
#pragma unroll
            for (int t = 0; t < 8; ++t) pacc[grp * HD + cc * 8 + t] = acc[t];
            named_bar_sync(kBarC, kCT);
            for (int e = ctid; e < HD; e += kCT) {
              float o = 0.f;
              for (int g2 = 0; g2 < GR; ++g2) o += pacc[g2 * HD + e];
              a.obuf[static_cast<int64_t>(b) * d + h * HD + e] = f2b(o);
            }
            }
            if (k < 2) ATT_PROBE(11 + k);
            named_bar_sync(kBarC, kCT);
          }
        }
        pit += nunits * per;
      } else if (gq > 0 && q < 8 * L && (q % 8 == 3 || q % 8 == 7)) {
        // ======== residual + LayerNorm (one CTA per sample row) ========
        const bool after_wo = q % 8 == 3;
        const int64_t lo = layer * a.per_layer;
        const uint16_t* bias = after_wo ? a.bo + lo : a.b2 + lo;
        const uint16_t *g, *beta;
        if (after_wo) {
          g = a.ln2_g + lo;
          beta = a.ln2_b + lo;
        } else if (layer + 1 < L) {
          g = a.ln1_g + lo + a.per_layer;
          beta = a.ln1_b + lo + a.per_layer;
        } else {
          g = a.lnf_g;
          beta = a.lnf_b;
        }
        const int S = a.S_[after_wo ? M_WO : M_W2];
        ATT_PROBE(0);
        for (int b = cta; b < B; b += G) {
          unsigned long long* spp = sp_on ? spb + 1 : nullptr;
          if (d <= 1024) res_ln_row<4>(a, b, S, bias, g, beta, red, ctid, cw, lane, true, spp);
          else res_ln_row<16>(a, b, S, bias, g, beta, red, ctid, cw, lane, true, spp);
          ATT_PROBE(3);
        }
      } else if (gq > 0 && q < 8 * L && q % 8 == 5) {
        // ======== FFN activation: f = bf16(relu(sum_s part + b1)) ========
        const uint16_t* b1 = a.b1 + layer * a.per_layer;
        const int S = a.S_[M_W1], ff = a.ff;
        const int64_t n = static_cast<int64_t>(B) * ff;
        for (int64_t i = static_cast<int64_t>(cta) * kCT + ctid; i < n; i += static_cast<int64_t>(G) * kCT) {
          const int b = static_cast<int>(i / ff), m = static_cast<int>(i % ff);
          const float s = sum_splits(a.part + static_cast<int64_t>(b) * ff + m, static_cast<int64_t>(B) * ff, S);
          a.fbuf[static_cast<int64_t>(b) * ff + m] = f2b(fmaxf(s + b2f(b1[m]), 0.0f));
        }
      } else {
        // ======== greedy argmax of the previous step + embedding + LN1 of layer 0 ========
        const bool has_prev = gq > 0, has_next = step + 1 < a.steps;
        for (int b = cta; b < B; b += G) {
          if (has_prev) {
            Top2 t{-FLT_MAX, 0x7fffffff, -FLT_MAX};
            const int T = (a.V + BM - 1) / BM;
#pragma unroll 4
            for (int tl = ctid; tl < T; tl += kCT) {
              const float* o = a.part + (static_cast<int64_t>(tl) * B + b) * 4;
              t = top2_merge(t, Top2{__ldcg(o), __float_as_int(__ldcg(o + 1)), __ldcg(o + 2)});
            }
            t = top2_warp(t);
            if (lane == 0) t2s[cw] = t;
            named_bar_sync(kBarC, kCT);
            if (ctid == 0) {
              for (int w = 1; w < kCT / 32; ++w) t = top2_merge(t, t2s[w]);
              const int64_t at = static_cast<int64_t>(b) * a.S + pos + 1;
              (a.pred ? a.pred : a.tokens)[at] = t.i1;
              if (a.margin) a.margin[at] = t.v1 - t.v2;
              itok[0] = a.pred ? a.tokens[at] : t.i1;
            }
            named_bar_sync(kBarC, kCT);
          } else if (ctid == 0) {
            itok[0] = a.tokens[static_cast<int64_t>(b) * a.S + pos];
          }
          if (!has_next) continue;
          named_bar_sync(kBarC, kCT);
          const int tok = itok[0];
          const int p = has_prev ? pos + 1 : pos;
          for (int c = ctid; c < d; c += kCT)
            a.x[static_cast<int64_t>(b) * d + c] =
                b2f(a.tok_emb[static_cast<int64_t>(tok) * d + c]) + b2f(a.pos_emb[static_cast<int64_t>(p) * d + c]);
          named_bar_sync(kBarC, kCT);
          if (d <= 1024) res_ln_row<4>(a, b, 0, nullptr, a.ln1_g, a.ln1_b, red, ctid, cw, lane, false);
          else res_ln_row<16>(a, b, 0, nullptr, a.ln1_g, a.ln1_b, red, ctid, cw, lane, false);
          named_bar_sync(kBarC, kCT);
        }
        if (has_prev) ++pos;
      }
      // ======== grid barrier: publish this phase ========
      if (a.probe && ctid == 0 && step == 1) a.probe[(static_cast<int64_t>(q) * 2) * G + cta] = gtime();
      ATT_PROBE(13);
      // data a later TMA / bulk copy reads (h, o, f, K/V rows): generic -> async proxy
      if (tma_data) asm volatile("fence.proxy.async.global;" ::: "memory");
      named_bar_sync(kBarC, kCT);
      ATT_PROBE(14);
      if (ctid == 0) {
        // release is cumulative over the CTA's writes ordered before it by bar.sync
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.gbar) : "memory");
        const unsigned target = static_cast<unsigned>(gq + 1) * G;
        ATT_PROBE(15);
        while (ld_acquire(a.gbar) < target) {
        }
      }
      named_bar_sync(kBarC, kCT);
      if (a.probe && ctid == 0 && step == 1) a.probe[(static_cast<int64_t>(q) * 2 + 1) * G + cta] = gtime();
    }
    if (cta == 0 && ctid == 0) *a.pos = pos;
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, a.tmem_cols);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 4-D view (K, 1, rows, layers) of a K-contiguous bf16 matrix stack; box (64, 1, box_rows, 1)
int map4(CUtensorMap* m, const void* ptr, int64_t K, int64_t rows, int64_t layers, int64_t layer_stride, int box_rows) {
  auto fn = encode_fn();
  if (!fn || (reinterpret_cast<uintptr_t>(ptr) & 15) || (K * 2) % 16 || (layer_stride * 2) % 16) return 2;
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(K), 1, static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(layers)};
  if (layers <= 1) layer_stride = K * rows;
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(K * 2), static_cast<cuuint64_t>(K * 2),
                           static_cast<cuuint64_t>(layer_stride * 2)};
  cuuint32_t box[4] = {64u, 1u, static_cast<cuuint32_t>(box_rows), 1u};
  cuuint32_t es[4] = {1u, 1u, 1u, 1u};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(ptr), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS
             ? 0
             : 5;
}

struct Plan {
  int BN, G, S_[5], kbper_[5], np, xs, tmem_cols;
  size_t smem, off_x, off_h, off_o, off_f, off_pk, off_part, total;
};

static size_t al(size_t v) { return (v + 255) & ~static_cast<size_t>(255); }

int plan(const rlhf_decode_loop_params* p, Plan* out) {
  const rlhf_arch& A = *p->arch;
  const int d = A.d_model, ff = A.d_ff, V = A.vocab, H = A.n_heads;
  if (!p->arch || p->B < 1 || p->B > 64 || d % 64 || ff % 64 || H < 1 || d % H) return 2;
  const int hd = d / H;
  if (hd != 32 && hd != 64 && hd != 128) return 2;
  if (d > 4096 || p->Smax < 1) return 2;
  Plan pl{};
  pl.BN = p->B <= 32 ? 32 : 64;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  pl.G = p->sms > 0 ? std::min(p->sms, sms) : sms;
  const int Ms[5] = {3 * d, d, ff, d, V};
  const int KBs[5] = {d / 64, d / 64, d / 64, ff / 64, d / 64};
  size_t part = 0;
  for (int j = 0; j < 5; ++j) {
    const int T = (Ms[j] + 127) / 128;
    int kbper = std::max((T * KBs[j] + pl.G - 1) / pl.G, (KBs[j] + kMaxSplit - 1) / kMaxSplit);
    if (j == 4 || kbper > KBs[j]) kbper = KBs[j];
    pl.kbper_[j] = kbper;
    pl.S_[j] = (KBs[j] + kbper - 1) / kbper;
    part = std::max(part, static_cast<size_t>(j == 4 ? 4 : pl.S_[j]) * p->B * (j == 4 ? T : Ms[j]) * 4);
  }
  {
    const int nu = ((V + 127) / 128 + pl.G - 1) / pl.G;  // vocabulary tiles per CTA (LM accumulators)
    int cols = 32;
    while (cols < std::max(2 * pl.BN, nu * pl.BN)) cols *= 2;
    if (cols > 512) return 2;
    pl.tmem_cols = cols;
  }
  const int XT = pl.BN * 64 * 2;
  const size_t fixed = ((p->Smax + 3) & ~3) * 4 + kQN * 3 * hd * 4 + 8192 + 32 + 8 * 32 * 12 + 32 + 8 * 64 + 1024 + 256;
  pl.xs = pl.BN == 32 ? 6 : 4;
  const size_t budget = 232448 - fixed - static_cast<size_t>(pl.xs) * XT;
  pl.np = static_cast<int>(std::min<size_t>(24, budget / kSlot));
  if (pl.np < 4) return 2;
  pl.smem = fixed + static_cast<size_t>(pl.xs) * XT + static_cast<size_t>(pl.np) * kSlot;
  size_t o = 256;  // grid barrier counter
  pl.off_x = o;
  o = al(o + static_cast<size_t>(p->B) * d * 4);
  pl.off_h = o;
  o = al(o + static_cast<size_t>(pl.BN) * d * 2);
  pl.off_o = o;
  o = al(o + static_cast<size_t>(pl.BN) * d * 2);
  pl.off_f = o;
  o = al(o + static_cast<size_t>(pl.BN) * ff * 2);
  pl.off_pk = o;  // small per-layer parameters, packed: [L][9d + ff] + lnf (2d), bf16
  o = al(o + (static_cast<size_t>(A.n_layers) * (9 * d + ff) + 2 * d) * 2);
  pl.off_part = o;
  o = al(o + part);
  pl.total = o;
  *out = pl;
  return 0;
}

template <int BN, int HD>
int launch(const Maps& maps, const Args& a, size_t smem, cudaStream_t s) {
  static int configured = 0;
  if (static_cast<int>(smem) > configured) {
    if (cudaFuncSetAttribute(decode_loop_kernel<BN, HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem)) != cudaSuccess)
      return 5;
    configured = static_cast<int>(smem);
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(a.G);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident (grid barriers)
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, decode_loop_kernel<BN, HD>, maps, a) == cudaSuccess ? 0 : 5;
}

}  // namespace dl
}  // namespace rlhf

using namespace rlhf;

extern "C" size_t rlhf_decode_loop_workspace_bytes(const rlhf_decode_loop_params* p) {
  dl::Plan pl;
  return dl::plan(p, &pl) ? 0 : pl.total;
}

extern "C" int rlhf_decode_loop(const rlhf_decode_loop_params* p, rlhf_stream_t stream) {
  dl::Plan pl;
  if (!p || !p->arch || p->arch->family != 0 || dl::plan(p, &pl)) return 2;  // OPT family only
  if (p->steps < 1) return 0;
  if (!p->workspace || p->workspace_bytes < pl.total) return 2;
  const rlhf_arch& A = *p->arch;
  const int d = A.d_model, ff = A.d_ff, hd = d / A.n_heads, L = A.n_layers;
  const auto* w = static_cast<const uint16_t*>(p->weights);
  const int64_t per_layer = rlhf_tensor_offset(&A, RLHF_T_LN1_G, 1) - rlhf_tensor_offset(&A, RLHF_T_LN1_G, 0);
  auto T = [&](int t) { return w + rlhf_tensor_offset(&A, t, 0); };
  uint8_t* ws = static_cast<uint8_t*>(p->workspace);
  dl::Args a{};
  a.d = d;
  a.H = A.n_heads;
  a.ff = ff;
  a.V = A.vocab;
  a.L = L;
  a.B = p->B;
  a.S = p->tok_stride;
  // pack the small per-layer tensors (LN gains / biases, linear biases) into the
  // workspace: one L2-persisting window instead of scattered lines between the
  // weight matrices that the weight stream would evict
  const int64_t PL = 9 * d + ff;  // ln1 g,b | bqkv | bo | ln2 g,b | b1 | b2
  uint16_t* pk = reinterpret_cast<uint16_t*>(ws + pl.off_pk);
  a.per_layer = PL;
  a.tok_emb = T(RLHF_T_TOK_EMB);
  a.pos_emb = T(RLHF_T_POS_EMB);
  const struct { int t; int64_t off, n; } packs[8] = {
      {RLHF_T_LN1_G, 0, d}, {RLHF_T_LN1_B, d, d}, {RLHF_T_BQKV, 2 * d, 3 * d}, {RLHF_T_BO, 5 * d, d},
      {RLHF_T_LN2_G, 6 * d, d}, {RLHF_T_LN2_B, 7 * d, d}, {RLHF_T_B1, 8 * d, ff}, {RLHF_T_B2, 8 * d + ff, d}};
  cudaStream_t s0 = reinterpret_cast<cudaStream_t>(stream);
  for (const auto& t : packs)
    if (cudaMemcpy2DAsync(pk + t.off, PL * 2, T(t.t), (L > 1 ? per_layer : t.n) * 2, t.n * 2, L,
                          cudaMemcpyDeviceToDevice, s0) != cudaSuccess)
      return 5;
  if (cudaMemcpyAsync(pk + L * PL, T(RLHF_T_LNF_G), d * 2, cudaMemcpyDeviceToDevice, s0) != cudaSuccess ||
      cudaMemcpyAsync(pk + L * PL + d, T(RLHF_T_LNF_B), d * 2, cudaMemcpyDeviceToDevice, s0) != cudaSuccess)
    return 5;
  a.ln1_g = pk;
  a.ln1_b = pk + d;
  a.bqkv = pk + 2 * d;
  a.bo = pk + 5 * d;
  a.ln2_g = pk + 6 * d;
  a.ln2_b = pk + 7 * d;
  a.b1 = pk + 8 * d;
  a.b2 = pk + 8 * d + ff;
  a.lnf_g = pk + L * PL;
  a.lnf_b = pk + L * PL + d;
  a.tokens = p->tokens;
  a.pred = p->pred;
  a.margin = p->margin;
  a.pos = p->pos;
  a.steps = p->steps;
  a.kc = static_cast<uint16_t*>(p->kcache);
  a.vc = static_cast<uint16_t*>(p->vcache);
  a.kvB = p->kv_B;
  a.Smax = p->Smax;
  a.gbar = reinterpret_cast<unsigned*>(ws);
  a.x = reinterpret_cast<float*>(ws + pl.off_x);
  a.hbuf = reinterpret_cast<uint16_t*>(ws + pl.off_h);
  a.obuf = reinterpret_cast<uint16_t*>(ws + pl.off_o);
  a.fbuf = reinterpret_cast<uint16_t*>(ws + pl.off_f);
  a.part = reinterpret_cast<float*>(ws + pl.off_part);
  a.G = pl.G;
  a.np = pl.np;
  a.tmem_cols = pl.tmem_cols;
  a.xs = pl.xs;
  for (int j = 0; j < 5; ++j) {
    a.S_[j] = pl.S_[j];
    a.kbper_[j] = pl.kbper_[j];
  }
  a.probe = p->probe;
  a.probe_q = p->probe_q;
  const int64_t Lst = L > 1 ? per_layer : 0;
  dl::Maps maps;
  int rc = 0;
  rc |= dl::map4(&maps.m[dl::M_QKV], T(RLHF_T_WQKV), d, 3 * d, L, Lst, dl::BM);
  rc |= dl::map4(&maps.m[dl::M_WO], T(RLHF_T_WO), d, d, L, Lst, dl::BM);
  rc |= dl::map4(&maps.m[dl::M_W1], T(RLHF_T_W1), d, ff, L, Lst, dl::BM);
  rc |= dl::map4(&maps.m[dl::M_W2], T(RLHF_T_W2), ff, d, L, Lst, dl::BM);
  rc |= dl::map4(&maps.m[dl::M_LM], T(RLHF_T_TOK_EMB), d, A.vocab, 1, 0, dl::BM);
  rc |= dl::map4(&maps.m[dl::M_XH], a.hbuf, d, pl.BN, 1, 0, pl.BN);
  rc |= dl::map4(&maps.m[dl::M_XO], a.obuf, d, pl.BN, 1, 0, pl.BN);
  rc |= dl::map4(&maps.m[dl::M_XF], a.fbuf, ff, pl.BN, 1, 0, pl.BN);
  if (hd == 64) {  // K / V cache as (hd, 1, Smax, L*kv_B*H), 128-row SWIZZLE_128B tiles
    const int64_t heads = static_cast<int64_t>(L) * p->kv_B * A.n_heads;
    rc |= dl::map4(&maps.m[dl::M_KC], p->kcache, hd, p->Smax, heads, static_cast<int64_t>(p->Smax) * hd, 128);
    rc |= dl::map4(&maps.m[dl::M_VC], p->vcache, hd, p->Smax, heads, static_cast<int64_t>(p->Smax) * hd, 128);
  } else {
    maps.m[dl::M_KC] = maps.m[dl::M_XH];
    maps.m[dl::M_VC] = maps.m[dl::M_XH];
  }
  if (rc) return 2;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  // barrier counter + zero activation rows >= B (MMA N padding)
  if (cudaMemsetAsync(ws, 0, pl.off_pk, s) != cudaSuccess) return 5;
  // keep the workspace (activations, partials, parameter pack) resident in L2
  // while weights and K/V stream through with evict-first hints
  {
    int dev = 0, maxp = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev);
    const size_t win = std::min<size_t>(pl.total, static_cast<size_t>(maxp));
    if (win > 0) {
      size_t cur = 0;
      cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
      if (cur < win) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, win);
      cudaStreamAttrValue v{};
      v.accessPolicyWindow.base_ptr = ws;
      v.accessPolicyWindow.num_bytes = win;
      v.accessPolicyWindow.hitRatio = 1.0f;
      v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v);
    }
  }
  int rc2;
  if (pl.BN == 32)
    rc2 = hd == 32 ? dl::launch<32, 32>(maps, a, pl.smem, s)
                   : (hd == 64 ? dl::launch<32, 64>(maps, a, pl.smem, s) : dl::launch<32, 128>(maps, a, pl.smem, s));
  else
    rc2 = hd == 32 ? dl::launch<64, 32>(maps, a, pl.smem, s)
                   : (hd == 64 ? dl::launch<64, 64>(maps, a, pl.smem, s) : dl::launch<64, 128>(maps, a, pl.smem, s));
  cudaStreamAttrValue off{};  // later kernels on this stream get no window
  cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &off);
  return rc2;
}
