// gemm_sm100.cu — persistent, warp-specialised tcgen05 + TMA GEMM for sm_100a.
//
// Serves every matmul of the PPO step (reference TaskKind work items,
// costmodel.hpp:63-64 / SPEC.md:209):
//   forward  Y = X W^T        (A K-major, B K-major)
//   decode   Y^T = W X^T      (swap-AB: weights fill the 128-row MMA M, batch is N)
//   backward dX = dY W        (B MN-major)      dW = dY^T X   (A, B MN-major)
//   attention S = Q K^T, O = P V, dP, dQ, dK, dV (batched over (b, h), causal tile skipping)
//
// CTA = 192 threads, persistent over a static round-robin list of work units
// (tile x split-K slice):
//   warp 0      TMA producer (4-D tensor maps, SWIZZLE_128B) into a STAGES-deep ring
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=BN, K=16)
//   warps 2..5  epilogue: TMEM -> registers -> smem transpose -> fused epilogue ->
//               contiguous row-segment stores
// The fp32 accumulator is double-buffered in TMEM (2 x BN columns): the epilogue of
// unit i overlaps the mainloop of unit i+1.
// Deterministic split-K: each slice writes its fp32 partial; the last slice of a tile
// (atomic ticket) sums all partials in slice order and runs the epilogue.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cfloat>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "launch_util.cuh"
#include "rlhf_kernels.h"
#include "sm100_common.cuh"

namespace rlhf {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kThreads = 64 + 32 * 4 * 1;  // warp 0 TMA, warp 1 MMA, 4 epilogue warps
constexpr int kEpiWarps = 4;
constexpr int kStagePitch = 33;  // fp32 epilogue staging pitch (conflict-free transpose)

template <int BN, int DEEP = 0>
struct TileCfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int EPI_BYTES = kEpiWarps * 32 * kStagePitch * 4;  // per-epilogue-warp transpose tiles
  // narrow tiles serve decode (few k-blocks per unit): 3 stages -> 2 CTAs/SM.  DEEP (the
  // decode LM head): one CTA per SM with the full ring, so the 393 c2 vocabulary tiles split
  // 3/2 per SM instead of up to 4 on an SM whose two CTAs both drew a second tile
  static constexpr int RAW_STAGES = BN <= 32 && !DEEP ? 3 : (218 * 1024 - EPI_BYTES) / STAGE_BYTES;
  static constexpr int STAGES = RAW_STAGES > (DEEP ? 10 : 8) ? (DEEP ? 10 : 8) : RAW_STAGES;
  static constexpr int TOP2_BYTES = 4 * 32 * 16;  // per-quarter top-2 of a 32-column chunk
  static constexpr int SMEM = STAGES * STAGE_BYTES + EPI_BYTES + TOP2_BYTES + 1024 + 256;
  static constexpr int TMEM_COLS = 2 * BN;
};

struct GemmArgs {
  int M, N, batch_h, splits, num_kb, tiles_m, tiles_n, units;
  int a_mn, b_mn;
  void* C;
  int c_f32;
  int64_t c_rs, c_cs, c_sh, c_sb;
  float alpha;
  int accumulate;
  const void* bias;
  int bias_f32, bias_along_m;
  int relu;
  const uint16_t* aux;
  int64_t aux_rs, aux_cs;
  const float* residual;
  int causal;
  float* ws;
  int* counters;
  unsigned long long* probe;
  int debug;
  float* top2;  // column-major top-2 epilogue (decode LM head): [tile][N] x float4
  float2* lse_part;  // row-major log-sum-exp epilogue (pair path): [row][tiles_n][2 halves]
  float* lse_tgt;
  const int32_t* lse_tok;
  int lse_S, lse_P, lse_R;
};

__device__ __forceinline__ unsigned long long clk() {
  unsigned long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
  return c;
}
#define PROBE(k)                                                                        \
  do {                                                                                  \
    if (e.probe && first) e.probe[static_cast<size_t>(blockIdx.x) * 16 + (k)] = clk();   \
  } while (0)

struct Unit {
  int z, h, b, m_tile, n_tile, split, m0, n0, kb_begin, kb_end;
  bool skip;
};

// Work unit u -> (batch z, m tile, n tile, split); split fastest, then n, then m.
template <int BN>
__device__ __forceinline__ Unit get_unit(const GemmArgs& e, int u) {
  Unit w;
  w.split = u % e.splits;
  int t = u / e.splits;
  w.n_tile = t % e.tiles_n;
  t /= e.tiles_n;
  w.m_tile = t % e.tiles_m;
  w.z = t / e.tiles_m;
  w.h = w.z % e.batch_h;
  w.b = w.z / e.batch_h;
  w.m0 = w.m_tile * BM;
  w.n0 = w.n_tile * BN;
  w.kb_begin = 0;
  w.kb_end = e.num_kb;
  w.skip = e.causal == 1 && w.n0 > w.m0 + BM - 1;  // tile strictly above the diagonal
  if (e.causal == 2) w.kb_end = min(w.kb_end, (w.m0 + BM + BK - 1) / BK);
  if (e.causal == 3) w.kb_begin = w.m0 / BK;
  if (e.splits > 1) {
    const int per = (e.num_kb + e.splits - 1) / e.splits;
    w.kb_begin = w.split * per;
    w.kb_end = min(e.num_kb, w.kb_begin + per);
  }
  return w;
}

__device__ __forceinline__ float bf16_bits_to_f32(uint16_t h) { return __uint_as_float(static_cast<uint32_t>(h) << 16); }
__device__ __forceinline__ uint16_t f32_to_bf16_bits(float f) { return __bfloat16_as_ushort(__float2bfloat16_rn(f)); }
// two floats -> packed bf16x2 (one cvt.rn.bf16x2.f32)
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  const __nv_bfloat162 p = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&p);
}

__device__ __forceinline__ void unpack8(const uint4 u, float (&f)[8]) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    f[2 * t] = bf16_bits_to_f32(static_cast<uint16_t>(w[t] & 0xFFFFu));
    f[2 * t + 1] = bf16_bits_to_f32(static_cast<uint16_t>(w[t] >> 16));
  }
}

// Scalar epilogue for one element (tails, unaligned and column-major outputs).
__device__ __noinline__ void epi_scalar(const GemmArgs& e, int b, int h, int m, int n, float x) {
  if (m >= e.M || n >= e.N) return;
  const int64_t off = b * e.c_sb + h * e.c_sh + static_cast<int64_t>(m) * e.c_rs + static_cast<int64_t>(n) * e.c_cs;
  x *= e.alpha;
  if (e.bias) {
    const int bi = e.bias_along_m ? m : n;
    x += e.bias_f32 ? static_cast<const float*>(e.bias)[bi] : bf16_bits_to_f32(static_cast<const uint16_t*>(e.bias)[bi]);
  }
  if (e.relu) x = fmaxf(x, 0.0f);
  if (e.aux) {
    const uint16_t a = e.aux[b * e.c_sb + h * e.c_sh + static_cast<int64_t>(m) * e.aux_rs + static_cast<int64_t>(n) * e.aux_cs];
    if ((a & 0x8000u) || a == 0) x = 0.0f;
  }
  if (e.residual) x += e.residual[off];
  if (e.c_f32) {
    float* d = static_cast<float*>(e.C) + off;
    *d = e.accumulate ? *d + x : x;
  } else {
    uint16_t* d = static_cast<uint16_t*>(e.C) + off;
    *d = f32_to_bf16_bits(e.accumulate ? bf16_bits_to_f32(*d) + x : x);
  }
}

// Column-major C (swap-AB decode outputs, c_rs == 1): lane = row m, 32 columns of
// one chunk (vals[j] in smem).  All global inputs are loaded before use so their
// latencies overlap; stores are coalesced across the warp (consecutive m).
__device__ __forceinline__ void epi_column32(const GemmArgs& e, int b, int h, int m, int n0, const float* vals) {
  if (m >= e.M) return;
  if (n0 + 32 > e.N) {
#pragma unroll 1
    for (int j = 0; j < 32; ++j) epi_scalar(e, b, h, m, n0 + j, vals[j]);
    return;
  }
  const int64_t base = b * e.c_sb + h * e.c_sh + static_cast<int64_t>(m) * e.c_rs + static_cast<int64_t>(n0) * e.c_cs;
  float x[32], r[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) x[j] = vals[j] * e.alpha;
  if (e.residual) {
#pragma unroll
    for (int j = 0; j < 32; ++j) r[j] = e.residual[base + j * e.c_cs];
  }
  if (e.accumulate) {
    if (e.c_f32) {
#pragma unroll
      for (int j = 0; j < 32; ++j) r[j] = (e.residual ? r[j] : 0.0f) + static_cast<const float*>(e.C)[base + j * e.c_cs];
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        r[j] = (e.residual ? r[j] : 0.0f) + bf16_bits_to_f32(static_cast<const uint16_t*>(e.C)[base + j * e.c_cs]);
    }
  }
  if (e.bias) {
    if (e.bias_along_m) {
      const float bm = e.bias_f32 ? static_cast<const float*>(e.bias)[m] : bf16_bits_to_f32(static_cast<const uint16_t*>(e.bias)[m]);
#pragma unroll
      for (int j = 0; j < 32; ++j) x[j] += bm;
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        x[j] += e.bias_f32 ? static_cast<const float*>(e.bias)[n0 + j] : bf16_bits_to_f32(static_cast<const uint16_t*>(e.bias)[n0 + j]);
    }
  }
  if (e.relu) {
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = fmaxf(x[j], 0.0f);
  }
  if (e.aux) {
    const int64_t ab = b * e.c_sb + h * e.c_sh + static_cast<int64_t>(m) * e.aux_rs + static_cast<int64_t>(n0) * e.aux_cs;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const uint16_t av = e.aux[ab + j * e.aux_cs];
      if ((av & 0x8000u) || av == 0) x[j] = 0.0f;
    }
  }
  if (e.residual || e.accumulate) {
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] += r[j];
  }
  if (e.c_f32) {
#pragma unroll
    for (int j = 0; j < 32; ++j) static_cast<float*>(e.C)[base + j * e.c_cs] = x[j];
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) static_cast<uint16_t*>(e.C)[base + j * e.c_cs] = f32_to_bf16_bits(x[j]);
  }
}

// Row-major C: 4 rows (m, m+8, m+16, m+24) x 8 consecutive columns [n, n+8).
// Vectorised; every global input of the 4 rows is loaded before any is used.
__device__ __noinline__ void epi_rows4_slow(const GemmArgs& e, int b, int h, int m, int n, const float* st, int pitch) {
#pragma unroll 1
  for (int i = 0; i < 4; ++i)
#pragma unroll 1
    for (int t = 0; t < 8; ++t) epi_scalar(e, b, h, m + 8 * i, n + t, st[8 * i * pitch + t]);
}

// st: this lane's first value in the smem staging tile (row stride `pitch`), for the slow path.
__device__ __forceinline__ void epi_rows4(const GemmArgs& e, int b, int h, int m, int n, float (&v)[4][8], const float* st,
                                          int pitch) {
  const int64_t bh = b * e.c_sb + h * e.c_sh;
  const int esz = e.c_f32 ? 4 : 2;
  const int64_t c0 = bh + static_cast<int64_t>(m) * e.c_rs + n;
  const int64_t a0 = bh + static_cast<int64_t>(m) * e.aux_rs + n;
  uintptr_t align = reinterpret_cast<uintptr_t>(static_cast<const char*>(e.C) + c0 * esz) | static_cast<uintptr_t>(e.c_rs * esz);
  if (e.residual) align |= reinterpret_cast<uintptr_t>(e.residual + c0) | static_cast<uintptr_t>(e.c_rs * 4);
  if (e.aux) align |= reinterpret_cast<uintptr_t>(e.aux + a0) | static_cast<uintptr_t>(e.aux_rs * 2) | (e.aux_cs != 1 ? 1 : 0);
  if (e.bias && !e.bias_along_m) align |= e.bias_f32 ? 1 : reinterpret_cast<uintptr_t>(static_cast<const uint16_t*>(e.bias) + n);
  if (n + 8 > e.N || m + 24 >= e.M || (align & 15)) {
    epi_rows4_slow(e, b, h, m, n, st, pitch);
    return;
  }
  // ---- issue loads
  uint4 braw = make_uint4(0, 0, 0, 0);
  float bm[4] = {0.f, 0.f, 0.f, 0.f};
  if (e.bias) {
    if (!e.bias_along_m) {
      braw = *reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(e.bias) + n);
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        bm[i] = e.bias_f32 ? static_cast<const float*>(e.bias)[m + 8 * i]
                           : bf16_bits_to_f32(static_cast<const uint16_t*>(e.bias)[m + 8 * i]);
    }
  }
  float4 res[4][2];
  if (e.residual) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float4* r = reinterpret_cast<const float4*>(e.residual + c0 + 8 * i * e.c_rs);
      res[i][0] = r[0];
      res[i][1] = r[1];
    }
  }
  uint4 ax[4];
  if (e.aux) {
#pragma unroll
    for (int i = 0; i < 4; ++i) ax[i] = *reinterpret_cast<const uint4*>(e.aux + a0 + 8 * i * e.aux_rs);
  }
  float4 old[4][2];
  if (e.accumulate) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (e.c_f32) {
        const float4* d = reinterpret_cast<const float4*>(static_cast<const float*>(e.C) + c0 + 8 * i * e.c_rs);
        old[i][0] = d[0];
        old[i][1] = d[1];
      } else {
        const uint4 u = *reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(e.C) + c0 + 8 * i * e.c_rs);
        old[i][0] = make_float4(__uint_as_float(u.x), __uint_as_float(u.y), __uint_as_float(u.z), __uint_as_float(u.w));
      }
    }
  }
  // ---- compute + store
  float bb[8];
  unpack8(braw, bb);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float x[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) x[t] = v[i][t] * e.alpha + (e.bias_along_m ? bm[i] : bb[t]);
    if (e.relu) {
#pragma unroll
      for (int t = 0; t < 8; ++t) x[t] = fmaxf(x[t], 0.0f);
    }
    if (e.aux) {
      const uint32_t aw[4] = {ax[i].x, ax[i].y, ax[i].z, ax[i].w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const uint16_t lo = static_cast<uint16_t>(aw[t] & 0xFFFFu), hi = static_cast<uint16_t>(aw[t] >> 16);
        if ((lo & 0x8000u) || lo == 0) x[2 * t] = 0.0f;
        if ((hi & 0x8000u) || hi == 0) x[2 * t + 1] = 0.0f;
      }
    }
    if (e.residual) {
      x[0] += res[i][0].x; x[1] += res[i][0].y; x[2] += res[i][0].z; x[3] += res[i][0].w;
      x[4] += res[i][1].x; x[5] += res[i][1].y; x[6] += res[i][1].z; x[7] += res[i][1].w;
    }
    const int64_t ci = c0 + 8 * i * e.c_rs;
    if (e.c_f32) {
      if (e.accumulate) {
        x[0] += old[i][0].x; x[1] += old[i][0].y; x[2] += old[i][0].z; x[3] += old[i][0].w;
        x[4] += old[i][1].x; x[5] += old[i][1].y; x[6] += old[i][1].z; x[7] += old[i][1].w;
      }
      float4* d4 = reinterpret_cast<float4*>(static_cast<float*>(e.C) + ci);
      d4[0] = make_float4(x[0], x[1], x[2], x[3]);
      d4[1] = make_float4(x[4], x[5], x[6], x[7]);
    } else {
      if (e.accumulate) {
        float o8[8];
        unpack8(make_uint4(__float_as_uint(old[i][0].x), __float_as_uint(old[i][0].y), __float_as_uint(old[i][0].z),
                           __float_as_uint(old[i][0].w)),
                o8);
#pragma unroll
        for (int t = 0; t < 8; ++t) x[t] += o8[t];
      }
      *reinterpret_cast<uint4*>(static_cast<uint16_t*>(e.C) + ci) =
          make_uint4(pack_bf16x2(x[0], x[1]), pack_bf16x2(x[2], x[3]), pack_bf16x2(x[4], x[5]), pack_bf16x2(x[6], x[7]));
    }
  }
}

// Split-K fixup: s[i][t] = sum over slices (in slice order) of the partial at
// row (row0 + 8i), column col+t of this tile; two slices' loads in flight at a time.
__device__ __forceinline__ void reduce_partials(const GemmArgs& e, size_t tile_id, int row0, int col, int bn, float (&s)[4][8]) {
#pragma unroll 1
  for (int s0 = 0; s0 < e.splits; s0 += 2) {
    float4 p[2][4][2];
#pragma unroll
    for (int k = 0; k < 2; ++k)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (s0 + k < e.splits) {
          const float4* src = reinterpret_cast<const float4*>(e.ws + ((tile_id * e.splits + s0 + k) * BM + row0 + 8 * i) * bn + col);
          p[k][i][0] = __ldcg(src);
          p[k][i][1] = __ldcg(src + 1);
        } else {
          p[k][i][0] = p[k][i][1] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
#pragma unroll
    for (int k = 0; k < 2; ++k)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        s[i][0] += p[k][i][0].x; s[i][1] += p[k][i][0].y; s[i][2] += p[k][i][0].z; s[i][3] += p[k][i][0].w;
        s[i][4] += p[k][i][1].x; s[i][5] += p[k][i][1].y; s[i][6] += p[k][i][1].z; s[i][7] += p[k][i][1].w;
      }
  }
}

template <int BN, int COLMAJOR, int DEEP = 0>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_sm100_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const __grid_constant__ GemmArgs e) {
  using Cfg = TileCfg<BN, DEEP>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* epi_stage = reinterpret_cast<float*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  float4* t2s = reinterpret_cast<float4*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES + Cfg::EPI_BYTES);  // [4][32]
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES + Cfg::EPI_BYTES + Cfg::TOP2_BYTES);
  uint64_t* empty_bar = full_bar + Cfg::STAGES;
  uint64_t* tfull = empty_bar + Cfg::STAGES;  // [2] accumulator ready
  uint64_t* tempty = tfull + 2;               // [2] accumulator drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const uint32_t warp = warp_id(), lane = lane_id();
  bool first = threadIdx.x == 0;
  PROBE(0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kEpiWarps);  // one arrive per epilogue warp
    }
    mbar_fence_init();
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
  }
  if (warp == 1) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  PROBE(1);
  // programmatic dependent launch (decode LM head inside the step graph): setup above
  // overlapped the predecessor; operands and outputs are touched only after the wait
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      first = true;
      for (int u = blockIdx.x; u < e.units; u += gridDim.x) {
        const Unit w = get_unit<BN>(e, u);
        if (w.skip) continue;
        for (int kb = w.kb_begin; kb < w.kb_end; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1u);
          PROBE(2);
          first = false;
          uint8_t* sa = smem + stage * Cfg::STAGE_BYTES;
          uint8_t* sb = sa + Cfg::A_BYTES;
          mbar_arrive_expect_tx(&full_bar[stage], Cfg::STAGE_BYTES);
          const int k0 = kb * BK;
          if (!e.a_mn) {
            tma_load_4d(sa, &tmA, &full_bar[stage], k0, w.h, w.m0, w.b);
          } else {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j) tma_load_4d(sa + j * 8192, &tmA, &full_bar[stage], w.m0 + 64 * j, w.h, k0, w.b);
          }
          if (!e.b_mn) {
            tma_load_4d(sb, &tmB, &full_bar[stage], k0, w.h, w.n0, w.b);
          } else {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j) tma_load_4d(sb + j * 8192, &tmB, &full_bar[stage], w.n0 + 64 * j, w.h, k0, w.b);
          }
          if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1u; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- UMMA issuer (one thread)
      const uint32_t idesc = umma_idesc_bf16(BM, BN, e.a_mn, e.b_mn);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int u = blockIdx.x; u < e.units; u += gridDim.x) {
        const Unit w = get_unit<BN>(e, u);
        if (w.skip) continue;
        const int acc = it & 1;
        const uint32_t aph = (it >> 1) & 1;
        ++it;
        mbar_wait(&tempty[acc], aph ^ 1u);  // epilogue has drained this accumulator
        tc_fence_after();
        const uint32_t d = tmem + static_cast<uint32_t>(acc * BN);
        first = it == 1;
        for (int kb = w.kb_begin; kb < w.kb_end; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          if (kb == w.kb_begin) PROBE(3);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * Cfg::STAGE_BYTES);
          const uint32_t sb = sa + Cfg::A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = e.a_mn ? umma_desc_sw128(sa + k * 2048, 8192, 1024) : umma_desc_sw128(sa + k * 32, 16, 1024);
            const uint64_t bd = e.b_mn ? umma_desc_sw128(sb + k * 2048, 8192, 1024) : umma_desc_sw128(sb + k * 32, 16, 1024);
            umma_bf16(d, ad, bd, idesc, (kb > w.kb_begin || k > 0) ? 1u : 0u);
          }
          umma_commit(&empty_bar[stage]);  // frees the smem slot when these MMAs retire
          if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1u; }
        }
        PROBE(4);
        if (w.kb_end > w.kb_begin) umma_commit(&tfull[acc]);
        else mbar_arrive(&tfull[acc]);
      }
    }
    __syncwarp();
  } else {  // ---- epilogue warps 2..9: TMEM lane quarter q = warp % 4, chunk parity = half
    const int q = static_cast<int>(warp & 3u);
    const int half = static_cast<int>(warp - 2) >> 2;  // 0 with 4 epilogue warps
    constexpr int NCH = BN / 32;
    const int my_last = kEpiWarps == 4 ? NCH - 1 : (((NCH - 1 - half) >= 0) ? NCH - 1 - ((NCH - 1 - half) & 1) : -1);
    float* st = epi_stage + (warp - 2) * 32 * kStagePitch;
    const uint32_t tq = static_cast<uint32_t>(q * 32) << 16;
    constexpr bool row_major = COLMAJOR == 0;
    const int rr0 = static_cast<int>(lane >> 2), cc = static_cast<int>(lane & 3) * 8;
    int it = 0;
    for (int u = blockIdx.x; u < e.units; u += gridDim.x) {
      const Unit w = get_unit<BN>(e, u);
      if (w.skip) continue;
      const int acc = it & 1;
      const uint32_t aph = (it >> 1) & 1;
      ++it;
      const bool has_k = w.kb_end > w.kb_begin;
      mbar_wait(&tfull[acc], aph);
      first = threadIdx.x == 64 && it == 1;
      PROBE(5);
      tc_fence_after();
      const uint32_t tbase = tmem + tq + static_cast<uint32_t>(acc * BN);
      const size_t tile_id = (static_cast<size_t>(w.z) * e.tiles_m + w.m_tile) * e.tiles_n + w.n_tile;
      float* part = e.splits > 1 ? e.ws + ((tile_id * e.splits + w.split) * BM + q * 32) * BN : nullptr;
      const int mq = w.m0 + q * 32;
      if (my_last < 0) {  // no chunk for this warp (BN == 32): release immediately
        tc_fence_before();
        if (lane == 0) mbar_arrive(&tempty[acc]);
      }
#pragma unroll 1
      for (int c = half; c < NCH; c += kEpiWarps / 4) {
        float v[32];
        if (has_k) tmem_ld32(tbase + c * 32, v);
        else {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = 0.0f;
        }
        if (c == half) PROBE(8);
        if (c == my_last) {  // this warp is done with the accumulator
          tc_fence_before();
          if (lane == 0) mbar_arrive(&tempty[acc]);
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) st[lane * kStagePitch + j] = v[j];
        __syncwarp();
        if (c == half) PROBE(9);
        if constexpr (!row_major) {
          if (e.top2) {  // per column: top-2 over this tile's rows (lane j scans staged column j)
            float4 keep = make_float4(-FLT_MAX, __int_as_float(0x7fffffff), -FLT_MAX, 0.f);
#pragma unroll 8
            for (int r = 0; r < 32; ++r) {
              const int m = mq + r;
              if (m >= e.M) break;
              const float x = st[r * kStagePitch + lane] * e.alpha;
              if (x > keep.x) {  // rows ascend: ties keep the lower id
                keep.z = keep.x;
                keep.x = x;
                keep.y = __int_as_float(m);
              } else {
                keep.z = fmaxf(keep.z, x);
              }
            }
            t2s[q * 32 + lane] = keep;
            named_bar_sync(2, 32 * kEpiWarps);
            if (q == 0) {
              float4 r = t2s[lane];
#pragma unroll
              for (int qq = 1; qq < 4; ++qq) {
                const float4 o = t2s[qq * 32 + lane];
                if (o.x > r.x || (o.x == r.x && __float_as_int(o.y) < __float_as_int(r.y))) {
                  r = make_float4(o.x, o.y, fmaxf(r.x, o.z), 0.f);
                } else {
                  r.z = fmaxf(r.z, o.x);
                }
              }
              const int n = w.n0 + c * 32 + static_cast<int>(lane);
              if (n < e.N) reinterpret_cast<float4*>(e.top2)[static_cast<size_t>(w.m_tile) * e.N + n] = r;
            }
            named_bar_sync(2, 32 * kEpiWarps);
          } else if (!part) {
            epi_column32(e, w.b, w.h, mq + static_cast<int>(lane), w.n0 + c * 32, st + lane * kStagePitch);
          }
        }
        if (row_major || part) {
          // lane l owns rows l/4 + 8i (i < 4), columns 8*(l%4)..+8 -> 64 B contiguous per row
          float s[4][8];
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int t = 0; t < 8; ++t) s[i][t] = st[(rr0 + 8 * i) * kStagePitch + cc + t];
          if (part) {  // split-K slice: fp32 partial tile -> workspace
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              float4* dst = reinterpret_cast<float4*>(part + (rr0 + 8 * i) * BN + c * 32 + cc);
              dst[0] = make_float4(s[i][0], s[i][1], s[i][2], s[i][3]);
              dst[1] = make_float4(s[i][4], s[i][5], s[i][6], s[i][7]);
            }
          } else {
            epi_rows4(e, w.b, w.h, mq + rr0, w.n0 + c * 32 + cc, s, st + rr0 * kStagePitch + cc, kStagePitch);
          }
        }
        __syncwarp();
        if (c == half) PROBE(10);
        if (c == half + 3) PROBE(11);
      }
      PROBE(6);
      if (!part) continue;
      // split-K: ticket; the last slice of the tile reduces all partials in order
      __threadfence();
      named_bar_sync(1, 32 * kEpiWarps);
      if (threadIdx.x == 64) *last_flag = (atomicAdd(&e.counters[tile_id], 1) == e.splits - 1);
      named_bar_sync(1, 32 * kEpiWarps);
      const bool last = *last_flag != 0;
      named_bar_sync(1, 32 * kEpiWarps);  // flag consumed before the next unit may rewrite it
      if (!last) continue;
      __threadfence();
#pragma unroll 1
      for (int c = half; c < NCH; c += kEpiWarps / 4) {
        float s[4][8];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int t = 0; t < 8; ++t) s[i][t] = 0.0f;
        reduce_partials(e, tile_id, q * 32 + rr0, c * 32 + cc, BN, s);
        if constexpr (row_major) {  // row-segment epilogue straight from the reduced values
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int t = 0; t < 8; ++t) st[(rr0 + 8 * i) * kStagePitch + cc + t] = s[i][t];
          __syncwarp();
          epi_rows4(e, w.b, w.h, mq + rr0, w.n0 + c * 32 + cc, s, st + rr0 * kStagePitch + cc, kStagePitch);
          __syncwarp();
        } else {  // column-major output: back to lane = row for coalesced stores
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int t = 0; t < 8; ++t) st[(rr0 + 8 * i) * kStagePitch + cc + t] = s[i][t];
          __syncwarp();
          epi_column32(e, w.b, w.h, mq + static_cast<int>(lane), w.n0 + c * 32, st + lane * kStagePitch);
          __syncwarp();
        }
      }
      if (threadIdx.x == 64) e.counters[tile_id] = 0;  // re-arm for the next launch
      PROBE(7);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, Cfg::TMEM_COLS);
  }
}


// ---- CTA-pair (cta_group::2) variant ------------------------------------------
// Two CTAs of a cluster (one TPC) compute a 256 x 256 tile: each holds its 128 rows
// of A and 128 of B's 256 rows per k-block (32 KB / stage instead of 48 KB, so 6
// stages and 1.5x less L2->SM operand traffic per FLOP); the leader issues
// tcgen05.mma.cta_group::2 (M = 256, N = 256) which reads both CTAs' shared memory
// and writes each CTA's 128 accumulator lanes into its own TMEM.  Both producers'
// TMA loads complete on the leader's full barrier; the MMA commit is multicast to
// both CTAs' empty / accumulator-ready barriers; both CTAs' epilogue warps arrive on
// the leader's accumulator-drained barrier.  Same K order as the 1-CTA kernel, so
// results are bit-identical to it.  Row-major C, no split-K.
namespace pair {
constexpr int PBM = 2 * BM, PBN = 256;
constexpr int A_BYTES = BM * BK * 2;
constexpr int BH_BYTES = (PBN / 2) * BK * 2;
constexpr int STAGE_BYTES = A_BYTES + BH_BYTES;
constexpr int EPI_WARPS = 8;  // two warps per TMEM lane quarter, alternating 32-column chunks
constexpr int THREADS = 64 + 32 * EPI_WARPS;
constexpr int EPI_BYTES = EPI_WARPS * 32 * kStagePitch * 4;
constexpr int RAW_STAGES = (218 * 1024 - EPI_BYTES) / STAGE_BYTES;
constexpr int STAGES = RAW_STAGES > 8 ? 8 : RAW_STAGES;
constexpr int SMEM = STAGES * STAGE_BYTES + EPI_BYTES + 1024 + 256;
constexpr int TMEM_COLS = 2 * PBN;

__device__ __forceinline__ uint32_t ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load_4d_pair(void* smem, const CUtensorMap* m, uint32_t bar_cluster, int c0, int c1,
                                                 int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.cta_group::2"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(smem)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(bar_cluster), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void umma_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit_pair(uint64_t* bar) {
  const uint16_t mask = 3;
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
__device__ __forceinline__ void arrive_remote(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}

// pair unit u -> (batch z, 256-row m tile, 256-col n tile)
__device__ __forceinline__ Unit get_unit(const GemmArgs& e, int u) {
  Unit w;
  w.split = 0;
  int t = u;
  w.n_tile = t % e.tiles_n;
  t /= e.tiles_n;
  w.m_tile = t % e.tiles_m;
  w.z = t / e.tiles_m;
  w.h = w.z % e.batch_h;
  w.b = w.z / e.batch_h;
  w.m0 = w.m_tile * PBM;
  w.n0 = w.n_tile * PBN;
  w.kb_begin = 0;
  w.kb_end = e.num_kb;
  w.skip = e.causal == 1 && w.n0 > w.m0 + PBM - 1;
  if (e.causal == 2) w.kb_end = min(w.kb_end, (w.m0 + PBM + BK - 1) / BK);
  if (e.causal == 3) w.kb_begin = w.m0 / BK;
  return w;
}
}  // namespace pair

__global__ void __launch_bounds__(pair::THREADS, 1)
    gemm_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ GemmArgs e) {
  using namespace pair;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* epi_stage = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES);
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES + EPI_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull = empty_bar + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = warp_id(), lane = lane_id();
  const uint32_t rank = ctarank();
  const bool leader = rank == 0;
  const int cid = blockIdx.x / 2, ncl = gridDim.x / 2;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * EPI_WARPS);  // both CTAs' epilogue warps (leader's copy is used)
    }
    mbar_fence_init();
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // the peer's barriers exist before any TMA / commit targets them
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer (both CTAs): this CTA's 128 rows of A and of B
      int stage = 0;
      uint32_t phase = 0;
      for (int u = cid; u < e.units; u += ncl) {
        const Unit w = pair::get_unit(e, u);
        if (w.skip) continue;
        const int ma = w.m0 + static_cast<int>(rank) * BM, nb = w.n0 + static_cast<int>(rank) * (PBN / 2);
        for (int kb = w.kb_begin; kb < w.kb_end; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1u);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          uint8_t* sb = sa + A_BYTES;
          const uint32_t fb = mapa(smem_u32(&full_bar[stage]), 0);
          if (leader) mbar_arrive_expect_tx(&full_bar[stage], 2 * STAGE_BYTES);
          const int k0 = kb * BK;
          if (!e.a_mn) {
            tma_load_4d_pair(sa, &tmA, fb, k0, w.h, ma, w.b);
          } else {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j) tma_load_4d_pair(sa + j * 8192, &tmA, fb, ma + 64 * j, w.h, k0, w.b);
          }
          if (!e.b_mn) {
            tma_load_4d_pair(sb, &tmB, fb, k0, w.h, nb, w.b);
          } else {
#pragma unroll
            for (int j = 0; j < (PBN / 2) / 64; ++j) tma_load_4d_pair(sb + j * 8192, &tmB, fb, nb + 64 * j, w.h, k0, w.b);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1u; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {  // ---- pair MMA issuer (leader CTA only)
      const uint32_t idesc = umma_idesc_bf16(PBM, PBN, e.a_mn, e.b_mn);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int u = cid; u < e.units; u += ncl) {
        const Unit w = pair::get_unit(e, u);
        if (w.skip) continue;
        const int acc = it & 1;
        const uint32_t aph = (it >> 1) & 1;
        ++it;
        mbar_wait(&tempty[acc], aph ^ 1u);  // both CTAs drained this accumulator
        tc_fence_after();
        const uint32_t d = tmem + static_cast<uint32_t>(acc * PBN);
        for (int kb = w.kb_begin; kb < w.kb_end; ++kb) {
          mbar_wait(&full_bar[stage], phase);  // both CTAs' halves landed
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * STAGE_BYTES);
          const uint32_t sb = sa + A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = e.a_mn ? umma_desc_sw128(sa + k * 2048, 8192, 1024) : umma_desc_sw128(sa + k * 32, 16, 1024);
            const uint64_t bd = e.b_mn ? umma_desc_sw128(sb + k * 2048, 8192, 1024) : umma_desc_sw128(sb + k * 32, 16, 1024);
            umma_pair(d, ad, bd, idesc, (kb > w.kb_begin || k > 0) ? 1u : 0u);
          }
          commit_pair(&empty_bar[stage]);  // frees the slot in BOTH CTAs
          if (++stage == STAGES) { stage = 0; phase ^= 1u; }
        }
        if (w.kb_end > w.kb_begin) {
          commit_pair(&tfull[acc]);
        } else {  // empty K range: release both CTAs' epilogues directly
          mbar_arrive(&tfull[acc]);
          arrive_remote(mapa(smem_u32(&tfull[acc]), 1));
        }
      }
    }
    __syncwarp();
  } else {  // ---- epilogue warps (both CTAs): this CTA's 128 rows of the 256 x 256 tile
    const int q = static_cast<int>(warp & 3u);
    const int half = static_cast<int>(warp - 2) >> 2;
    constexpr int NCH = PBN / 32;
    float* st = epi_stage + (warp - 2) * 32 * kStagePitch;
    const uint32_t tq = static_cast<uint32_t>(q * 32) << 16;
    const int rr0 = static_cast<int>(lane >> 2), cc = static_cast<int>(lane & 3) * 8;
    int it = 0;
    for (int u = cid; u < e.units; u += ncl) {
      const Unit w = pair::get_unit(e, u);
      if (w.skip) continue;
      const int acc = it & 1;
      const uint32_t aph = (it >> 1) & 1;
      ++it;
      const bool has_k = w.kb_end > w.kb_begin;
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      const uint32_t tbase = tmem + tq + static_cast<uint32_t>(acc * PBN);
      const int mq = w.m0 + static_cast<int>(rank) * BM + q * 32;
      // log-sum-exp mode: lane = row, running (max, sum) over this warp's columns
      const int mrow = mq + static_cast<int>(lane);
      int tgt = -1;
      if (e.lse_part && mrow < e.M) {
        const int bb = mrow / e.lse_R, jj = mrow % e.lse_R;
        tgt = e.lse_tok[static_cast<int64_t>(bb) * e.lse_S + e.lse_P + jj];
      }
      float lm = -FLT_MAX, ls = 0.f;
#pragma unroll 1
      for (int c = half; c < NCH; c += 2) {
        float v[32];
        if (has_k) tmem_ld32(tbase + c * 32, v);
        else {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = 0.0f;
        }
        if (c + 2 >= NCH) {  // this warp is done with the accumulator: tell the leader
          tc_fence_before();
          if (lane == 0) arrive_remote(mapa(smem_u32(&tempty[acc]), 0));
        }
        if (e.lse_part) {  // (max, sum) in natural units; exponentials as 2^(v*a2 - m*log2e)
          const int nc0 = w.n0 + c * 32;
          const float a2 = e.alpha * 1.4426950408889634f;
          float cm = -FLT_MAX, cs = 0.f;
          if (nc0 + 32 <= e.N) {  // every column valid (alpha > 0: max commutes with the scale)
#pragma unroll
            for (int j = 0; j < 32; ++j) cm = fmaxf(cm, v[j]);
            const float nm = fmaxf(lm, cm * e.alpha), nm2 = nm * 1.4426950408889634f;
#pragma unroll
            for (int j = 0; j < 32; ++j) cs += ex2_ftz(fmaf(v[j], a2, -nm2));
            ls = ls * ex2_ftz((lm - nm) * 1.4426950408889634f) + cs;
            lm = nm;
          } else if (nc0 < e.N) {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (nc0 + j < e.N) cm = fmaxf(cm, v[j]);
            const float nm = fmaxf(lm, cm * e.alpha), nm2 = nm * 1.4426950408889634f;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (nc0 + j < e.N) cs += ex2_ftz(fmaf(v[j], a2, -nm2));
            ls = ls * ex2_ftz((lm - nm) * 1.4426950408889634f) + cs;
            lm = nm;
          }
          if (tgt >= nc0 && tgt < nc0 + 32) {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (tgt == nc0 + j) e.lse_tgt[mrow] = v[j] * e.alpha;
          }
          continue;
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) st[lane * kStagePitch + j] = v[j];
        __syncwarp();
        float sv[4][8];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int t = 0; t < 8; ++t) sv[i][t] = st[(rr0 + 8 * i) * kStagePitch + cc + t];
        epi_rows4(e, w.b, w.h, mq + rr0, w.n0 + c * 32 + cc, sv, st + rr0 * kStagePitch + cc, kStagePitch);
        __syncwarp();
      }
      if (e.lse_part && mrow < e.M)
        e.lse_part[(static_cast<int64_t>(mrow) * e.tiles_n + w.n_tile) * 2 + half] = make_float2(lm, ls);
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // the leader's MMAs wrote this CTA's TMEM: both done before dealloc
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

// ---- host side -----------------------------------------------------------------

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

// 4-D view (inner, h, rows, b) of one operand; box (64, 1, box_rows, 1), SWIZZLE_128B.
static int make_map(CUtensorMap* map, const void* ptr, int64_t inner, int64_t rows, int64_t ld, int64_t sh,
                    int64_t sb, int bh, int bb, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return 5;
  if (reinterpret_cast<uintptr_t>(ptr) & 15) return 2;
  const int64_t e = 2;
  if ((ld * e) % 16) return 2;
  if (bh == 1) sh = ld * rows;  // unused dims get a harmless 16B-multiple stride
  if (bb == 1) sb = (bh == 1 ? ld * rows : sh * bh);
  if ((sh * e) % 16 || (sb * e) % 16) return 2;
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(bh), static_cast<cuuint64_t>(rows),
                        static_cast<cuuint64_t>(bb)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(sh * e), static_cast<cuuint64_t>(ld * e),
                           static_cast<cuuint64_t>(sb * e)};
  cuuint32_t box[4] = {64u, 1u, static_cast<cuuint32_t>(box_rows), 1u};
  cuuint32_t estr[4] = {1u, 1u, 1u, 1u};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(ptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    fprintf(stderr, "cuTensorMapEncodeTiled failed (%d): inner=%lld rows=%lld ld=%lld sh=%lld sb=%lld bh=%d bb=%d box=%d\n",
            static_cast<int>(r), (long long)inner, (long long)rows, (long long)ld, (long long)sh, (long long)sb, bh, bb,
            box_rows);
    return 5;
  }
  return 0;
}

static int pick_bn(const rlhf_gemm_params* p) {
  if (p->block_n) return p->block_n;
  const int N = p->N;
  int bn = N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : 256;
  if (p->b_mn_major && bn < 64) bn = 64;
  if (bn == 256) {
    const long tiles256 = static_cast<long>((p->M + BM - 1) / BM) * ((N + 255) / 256) * p->batch * (p->split_k > 1 ? p->split_k : 1);
    if (tiles256 < 148) bn = 128;  // prefer a fuller first wave
  }
  return bn;
}

static int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <int BN, int COLMAJOR, int DEEP = 0>
static int launch_mode(const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& a, cudaStream_t s) {
  using Cfg = TileCfg<BN, DEEP>;
  static int per_sm = 0;
  if (!per_sm) {
    if (cudaFuncSetAttribute(gemm_sm100_kernel<BN, COLMAJOR, DEEP>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM) != cudaSuccess)
      return 5;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gemm_sm100_kernel<BN, COLMAJOR, DEEP>, kThreads, Cfg::SMEM) != cudaSuccess)
      per_sm = 1;
    per_sm = std::max(1, std::min(per_sm, 512 / Cfg::TMEM_COLS));
  }
  int grid = std::min(a.units, per_sm * sm_count());
  if (DEEP) {
    // as few CTAs as keep the same tiles-per-CTA maximum (393 c2 tiles: 131 CTAs x 3, not
    // 97 x 3 + 51 x 2): same makespan, fewer CTAs contending for HBM at the tail
    static int g = -1;
    if (g < 0) g = getenv("RLHF_LMHEAD_GRID") ? atoi(getenv("RLHF_LMHEAD_GRID")) : 0;
    const int per = (a.units + grid - 1) / grid;
    grid = g > 0 ? std::min(a.units, g) : (a.units + per - 1) / per;
  }
  return launch_k(gemm_sm100_kernel<BN, COLMAJOR, DEEP>, dim3(grid), dim3(kThreads), Cfg::SMEM, s, ta, tb, a);
}

static int launch_pair(const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& a, cudaStream_t s) {
  static bool init = false;
  if (!init) {
    if (cudaFuncSetAttribute(gemm_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, pair::SMEM) != cudaSuccess)
      return 5;
    init = true;
  }
  cudaLaunchConfig_t cfg{};
  const int pairs = std::min(a.units, sm_count() / 2);
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(pair::THREADS);
  cfg.dynamicSmemBytes = pair::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, gemm_pair_kernel, ta, tb, a) == cudaSuccess ? 0 : 5;
}

// CTA-pair path: full 256-wide N tiles, row-major C, no split-K, enough 256 x 256 tiles
// to fill the pairs (RLHF_GEMM_PAIR=0 disables it)
static bool use_pair(const rlhf_gemm_params* p, int bn, int splits) {
  static int env = -1;
  if (env < 0) env = getenv("RLHF_GEMM_PAIR") ? atoi(getenv("RLHF_GEMM_PAIR")) : 1;
  if (!env || bn != 256 || splits != 1 || p->c_cs != 1) return false;
  const long tiles = static_cast<long>((p->M + 255) / 256) * ((p->N + 255) / 256) * p->batch;
  return tiles >= sm_count() / 2;
}

template <int BN>
static int launch(const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& a, cudaStream_t s) {
  if constexpr (BN == 32) {
    static int deep = -1;
    if (deep < 0) deep = getenv("RLHF_LMHEAD_DEEP") ? atoi(getenv("RLHF_LMHEAD_DEEP")) : 1;
    if (a.c_cs != 1 && a.top2 && deep) return launch_mode<32, 1, 1>(ta, tb, a, s);
  }
  return a.c_cs == 1 ? launch_mode<BN, 0>(ta, tb, a, s) : launch_mode<BN, 1>(ta, tb, a, s);
}

}  // namespace rlhf

using namespace rlhf;

extern "C" int rlhf_gemm_block_n(const rlhf_gemm_params* p) { return pick_bn(p); }

extern "C" const char* rlhf_gemm_kernel_name(const rlhf_gemm_params* p) {
  const int bn = pick_bn(p);
  const int splits = p->split_k > 1 ? std::min(p->split_k, (p->K + BK - 1) / BK) : 1;
  if (use_pair(p, bn, splits)) return "gemm_pair_kernel";
  switch (bn) {
    case 32: return "gemm_sm100_kernel<32>";
    case 64: return "gemm_sm100_kernel<64>";
    case 128: return "gemm_sm100_kernel<128>";
    default: return "gemm_sm100_kernel<256>";
  }
}

extern "C" size_t rlhf_gemm_workspace_bytes(const rlhf_gemm_params* p) {
  if (p->split_k <= 1 || p->causal) return 0;
  const int bn = pick_bn(p);
  const int splits = std::min(p->split_k, (p->K + BK - 1) / BK);
  const size_t tiles = static_cast<size_t>((p->M + BM - 1) / BM) * ((p->N + bn - 1) / bn) * p->batch;
  return tiles * splits * BM * bn * sizeof(float);
}

extern "C" int rlhf_gemm(const rlhf_gemm_params* p, rlhf_stream_t stream) {
  if (p->M <= 0 || p->N <= 0 || p->K <= 0 || p->batch <= 0 || p->batch_h <= 0 || p->batch % p->batch_h) return 2;
  const int bn = pick_bn(p);
  if (bn != 32 && bn != 64 && bn != 128 && bn != 256) return 2;
  if (p->b_mn_major && bn < 64) return 2;
  const int num_kb = (p->K + BK - 1) / BK;
  // split-K: deterministic (fp32 partials, the last slice of a tile reduces them in order)
  const int splits = p->split_k > 1 ? std::min(p->split_k, num_kb) : 1;
  if (splits > 1 && p->causal) return 2;
  const int bb = p->batch / p->batch_h;
  const bool pair_mode = use_pair(p, bn, splits);
  CUtensorMap ta, tb;
  int st;
  // A: K-major -> (K, h, M, b) box (64, 1, 128, 1); MN-major -> (M, h, K, b) box (64, 1, 64, 1)
  if (!p->a_mn_major) st = make_map(&ta, p->A, p->K, p->M, p->lda, p->a_stride_h, p->a_stride_b, p->batch_h, bb, BM);
  else st = make_map(&ta, p->A, p->M, p->K, p->lda, p->a_stride_h, p->a_stride_b, p->batch_h, bb, BK);
  if (st) return st;
  if (!p->b_mn_major)
    st = make_map(&tb, p->B, p->K, p->N, p->ldb, p->b_stride_h, p->b_stride_b, p->batch_h, bb, pair_mode ? bn / 2 : bn);
  else st = make_map(&tb, p->B, p->N, p->K, p->ldb, p->b_stride_h, p->b_stride_b, p->batch_h, bb, BK);
  if (st) return st;

  GemmArgs a{};
  a.M = p->M;
  a.N = p->N;
  a.batch_h = p->batch_h;
  a.splits = splits;
  a.num_kb = num_kb;
  a.tiles_m = (p->M + BM - 1) / BM;
  a.tiles_n = (p->N + bn - 1) / bn;
  a.units = a.tiles_m * a.tiles_n * p->batch * splits;
  a.a_mn = p->a_mn_major;
  a.b_mn = p->b_mn_major;
  a.C = p->C;
  a.c_f32 = p->c_f32;
  a.c_rs = p->c_rs;
  a.c_cs = p->c_cs;
  a.c_sh = p->c_stride_h;
  a.c_sb = p->c_stride_b;
  a.alpha = p->alpha;
  a.accumulate = p->accumulate;
  a.bias = p->bias;
  a.bias_f32 = p->bias_f32;
  a.bias_along_m = p->bias_along_m;
  a.relu = p->relu;
  a.aux = static_cast<const uint16_t*>(p->aux);
  a.aux_rs = p->aux_rs;
  a.aux_cs = p->aux_cs;
  a.residual = p->residual;
  a.causal = p->causal;
  a.probe = p->probe;
  a.top2 = p->top2;
  a.lse_part = reinterpret_cast<float2*>(p->lse_part);
  a.lse_tgt = p->lse_tgt;
  a.lse_tok = p->lse_tokens;
  a.lse_S = p->lse_S;
  a.lse_P = p->lse_P;
  a.lse_R = p->lse_R;
  if (a.lse_part && (!p->lse_tgt || !p->lse_tokens || p->lse_R < 1 || p->batch != 1 || !(p->alpha > 0.f))) return 2;
  if (a.top2 && (p->c_cs == 1 || p->split_k > 1 || p->batch != 1 || bn != 32 && bn != 64 && bn != 128 && bn != 256))
    return 2;
  {
    static int dbg = -1;
    if (dbg < 0) dbg = getenv("RLHF_GEMM_DEBUG") ? atoi(getenv("RLHF_GEMM_DEBUG")) : 0;
    a.debug = dbg;
  }
  if (splits > 1) {
    if (!p->workspace || p->workspace_bytes < rlhf_gemm_workspace_bytes(p)) return 2;
    if (!p->counters || p->counters_len < a.tiles_m * a.tiles_n * p->batch) return 2;
    a.ws = static_cast<float*>(p->workspace);
    a.counters = p->counters;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (a.lse_part && !pair_mode) return 2;  // the log-sum-exp epilogue lives on the pair path
  if (pair_mode) {
    a.tiles_m = (p->M + pair::PBM - 1) / pair::PBM;
    a.tiles_n = (p->N + pair::PBN - 1) / pair::PBN;
    a.units = a.tiles_m * a.tiles_n * p->batch;
    return launch_pair(ta, tb, a, s);
  }
  switch (bn) {
    case 32: return launch<32>(ta, tb, a, s);
    case 64: return launch<64>(ta, tb, a, s);
    case 128: return launch<128>(ta, tb, a, s);
    default: return launch<256>(ta, tb, a, s);
  }
}
