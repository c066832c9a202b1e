// attn_fused.cu — causal attention forward in one tcgen05 kernel (prefill, Forward x4,
// TrainFB forward) for sequences S <= 512 and head dim 64: scores, softmax and P.V.
//
// The unfused path writes the fp32 score matrix S = alpha Q K^T (B*H*S*S*4 bytes,
// 400 MB per layer for c2) and reads it back in a separate softmax kernel.  Here one
// CTA owns (sample, head, 128 query rows): Q (128 x 64) and the causal key range K
// (up to 512 x 64) arrive by TMA (SWIZZLE_128B), tcgen05.mma writes the 128 x (m0+128)
// fp32 score tile into TMEM (<= 512 columns), and four epilogue warps (one TMEM lane
// quarter each, thread = query row) run an online max / sum pass and a second pass that
// writes P = bf16(exp(s - max) / sum) (zeros above the diagonal) as 64-byte row segments
// (training only), and into one of two shared-memory P tiles (SW128, K-major; the softmax
// warps fill tile t+1 while tcgen05.mma accumulates O += P_t V_t in TMEM, columns [0, 64),
// reused once key tile 0 has been consumed).  V has its own shared-memory tiles, loaded
// together with K.  Inference forwards never write P to HBM.  Eight epilogue
// warps (two per lane quarter) split the column chunks; exponentials use ex2.approx
// (__expf, ~2 ulp).
//
// Numerics: fp32 scores (same MMA accumulation as the GEMM path), fp32
// softmax, probabilities normalised then rounded to bf16; the running sum is rescaled
// when the row max grows (online softmax), so sums differ from the two-pass kernel at
// fp32 rounding level only; __expf adds ~2 ulp per exponential.
#include <cudaTypedefs.h>

#include <cfloat>
#include <cstdio>
#include <mutex>

#include "rlhf_kernels.h"
#include "sm100_common.cuh"

namespace rlhf {
namespace af {

constexpr int BMq = 128, HD = 64, kEpi = 8, kThreads = 64 + 32 * kEpi, kMaxS = 512;
constexpr int Q_BYTES = BMq * HD * 2;   // 16 KB
constexpr int KT_BYTES = BMq * HD * 2;  // one 128-key tile, 16 KB
constexpr int PB_BYTES = BMq * BMq * 2;  // one 128 x 128 bf16 P tile (two SW128 64-key blocks)
// dynamic shared memory by mode: when O is produced, V tiles of their own (loaded with K,
// not after the QK^T MMAs) and a double-buffered P tile (the softmax warps write tile t+1
// while the tensor core multiplies tile t)
__host__ __device__ constexpr int smem_bytes(bool want_p, bool want_o) {
  return Q_BYTES + (kMaxS / BMq) * KT_BYTES * (want_o ? 2 : 1) + (want_o ? 2 * PB_BYTES : 0) + 4 * BMq * 4 + 1024 +
         256 + 0 * want_p;
}
constexpr int SMEM = smem_bytes(true, true);

__device__ __forceinline__ uint16_t f2b(float f) { return __bfloat16_as_ushort(__float2bfloat16_rn(f)); }
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {  // one cvt.rn.bf16x2
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}
__device__ __forceinline__ float ex2f(float x) { return ex2_ftz(x); }

__global__ void __launch_bounds__(kThreads, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, int H, int S, float alpha, uint16_t* __restrict__ P,
                    uint16_t* __restrict__ O, int64_t ldo) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sq = smem;
  uint8_t* skv = smem + Q_BYTES;                      // K tiles
  const bool want_o = O != nullptr, want_p = P != nullptr;
  uint8_t* svv = skv + (kMaxS / BMq) * KT_BYTES;      // V tiles (want_o)
  uint8_t* spb = svv + (want_o ? (kMaxS / BMq) * KT_BYTES : 0);  // 2 P tiles (A operand of P.V)
  float* rowst = reinterpret_cast<float*>(spb + (want_o ? 2 * PB_BYTES : 0));  // [2][2][128]
  uint64_t* full = reinterpret_cast<uint64_t*>(rowst + 4 * BMq);  // [4] Q + key tile 0, key tiles 1..3 landed
  uint64_t* done = full + 4;   // [4] QK^T MMAs of key tile t complete
  uint64_t* vfull = done + 4;  // V tiles landed
  uint64_t* pfull = vfull + 1;  // [2] P tile written by the epilogue warps
  uint64_t* pfree = pfull + 2;  // [2] P.V MMAs done with the P tile
  uint64_t* ofull = pfree + 2;  // O accumulated
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ofull + 1);

  const int mb = blockIdx.x, z = blockIdx.y, b = z / H, h = z % H;
  const int m0 = mb * BMq;
  const int nkt = mb + 1;  // causal key tiles
  const uint32_t warp = warp_id(), lane = lane_id();
  if (threadIdx.x == 0) {
    for (int t = 0; t < kMaxS / BMq; ++t) {
      mbar_init(&full[t], 1);
      mbar_init(&done[t], 1);
    }
    mbar_init(vfull, 1);
    for (int k = 0; k < 2; ++k) {
      mbar_init(&pfull[k], kEpi);
      mbar_init(&pfree[k], 1);
    }
    mbar_init(ofull, 1);
    mbar_fence_init();
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
  }
  int tcols = 128;  // score tile (nkt * 128 columns) rounded up to a power of two; O reuses
  while (tcols < nkt * BMq) tcols *= 2;  // columns [0, 64) once key tile 0 is consumed
  if (warp == 1) tmem_alloc(tmem_slot, tcols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // per-key-tile barriers: the MMA of tile t and the softmax of its columns start as soon
      // as that tile has landed, not after the whole key range
      mbar_arrive_expect_tx(&full[0], Q_BYTES + KT_BYTES);
      tma_load_4d(sq, &tmQ, &full[0], 0, h, m0, b);
      for (int t = 0; t < nkt; ++t) {
        if (t > 0) mbar_arrive_expect_tx(&full[t], KT_BYTES);
        tma_load_4d(skv + t * KT_BYTES, &tmK, &full[t], 0, h, t * BMq, b);
      }
      if (want_o) {  // V tiles into their own buffers, streaming while QK^T and the softmax run
        mbar_arrive_expect_tx(vfull, nkt * KT_BYTES);
        for (int t = 0; t < nkt; ++t) tma_load_4d(svv + t * KT_BYTES, &tmV, vfull, 0, h, t * BMq, b);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = umma_idesc_bf16(BMq, BMq, 0, 0);
      const uint32_t a = smem_u32(sq);
      for (int t = 0; t < nkt; ++t) {
        mbar_wait(&full[t], 0);
        tc_fence_after();
        const uint32_t bk = smem_u32(skv + t * KT_BYTES);
#pragma unroll
        for (int k = 0; k < HD / 16; ++k)
          umma_bf16(tmem + t * BMq, umma_desc_sw128(a + k * 32, 16, 1024), umma_desc_sw128(bk + k * 32, 16, 1024), idesc,
                    k > 0 ? 1u : 0u);
        umma_commit(&done[t]);
      }
      if (want_o) {
        // O[128 x 64] += P_t[128 x 128 keys] . V_t[128 keys x 64], key tiles in order
        const uint32_t idv = umma_idesc_bf16(BMq, HD, 0, 1);
        mbar_wait(vfull, 0);
        for (int t = 0; t < nkt; ++t) {
          mbar_wait(&pfull[t & 1], (t >> 1) & 1);
          tc_fence_after();
          const uint32_t pa = smem_u32(spb + (t & 1) * PB_BYTES), vb = smem_u32(svv + t * KT_BYTES);
#pragma unroll
          for (int kb2 = 0; kb2 < 2; ++kb2)
#pragma unroll
            for (int k = 0; k < 4; ++k)
              umma_bf16(tmem, umma_desc_sw128(pa + kb2 * (PB_BYTES / 2) + k * 32, 16, 1024),
                        umma_desc_sw128(vb + (kb2 * 4 + k) * 2048, 8192, 1024), idv,
                        (t > 0 || kb2 > 0 || k > 0) ? 1u : 0u);
          umma_commit(&pfree[t & 1]);
        }
        umma_commit(ofull);
      }
    }
    __syncwarp();
  } else {
    // ---- softmax epilogue: 8 warps, two per TMEM lane quarter (thread = query row i),
    //      the pair splits the 32-column chunks (even / odd) and merges its (max, sum)
    const int q = static_cast<int>(warp & 3u), half = static_cast<int>(warp - 2) >> 2;
    const int il = q * 32 + static_cast<int>(lane);
    const int i = m0 + il;
    const uint32_t tq = tmem + (static_cast<uint32_t>(q * 32) << 16);
    const int nch = (m0 + q * 32 + 32) / 32;  // chunks holding any j <= (this warp's last row)
    int tdone = -1;  // key tiles whose scores this warp has seen complete
    // Scores in log2 units (a2 = alpha * log2 e): every exponential is one FFMA + one
    // ex2.approx.ftz.  Only the chunk holding this quarter's diagonal (c == nch - 1) is
    // masked; chunks left of it are entirely causal-visible for all 32 rows of the warp.
    const float a2 = alpha * 1.4426950408889634f;
    float mx = -FLT_MAX, sum = 0.f;
    auto absorb = [&](const uint32_t (&r)[32], int c) {
      float cm = -FLT_MAX, cs = 0.f;
      if (c != nch - 1) {
#pragma unroll
        for (int t = 0; t < 32; ++t) cm = fmaxf(cm, __uint_as_float(r[t]));
        const float nm = fmaxf(mx, cm * a2);
#pragma unroll
        for (int t = 0; t < 32; ++t) cs += ex2f(fmaf(__uint_as_float(r[t]), a2, -nm));
        sum = sum * ex2f(mx - nm) + cs;
        mx = nm;
      } else {
#pragma unroll
        for (int t = 0; t < 32; ++t)
          if (c * 32 + t <= i) cm = fmaxf(cm, __uint_as_float(r[t]));
        const float nm = fmaxf(mx, cm * a2);
#pragma unroll
        for (int t = 0; t < 32; ++t)
          if (c * 32 + t <= i) cs += ex2f(fmaf(__uint_as_float(r[t]), a2, -nm));
        sum = sum * ex2f(mx - nm) + cs;
        mx = nm;
      }
    };
    // two TMEM loads in flight per wait (chunks c and c + 2 of this warp's parity)
    for (int c = half; c < nch; c += 4) {
      if (c / 4 > tdone) {  // chunks c and c + 2 lie in key tile c / 4
        tdone = c / 4;
        mbar_wait(&done[tdone], 0);
        tc_fence_after();
      }
      uint32_t ra[32], rb[32];
      tmem_ld32_nowait(tq + c * 32, ra);
      const bool two = c + 2 < nch;
      if (two) tmem_ld32_nowait(tq + (c + 2) * 32, rb);
      tmem_ld_wait32x2(ra, rb);
      absorb(ra, c);
      if (two) absorb(rb, c + 2);
    }
    rowst[(half * 2) * BMq + il] = mx;
    rowst[(half * 2 + 1) * BMq + il] = sum;
    named_bar_sync(1, 32 * kEpi);
    {  // an empty half has (-FLT_MAX, 0): its weight ex2(-huge) * 0 is 0
      const float ma = rowst[il], sa = rowst[BMq + il], mb2 = rowst[2 * BMq + il], sb = rowst[3 * BMq + il];
      mx = fmaxf(ma, mb2);
      sum = sa * ex2f(ma - mx) + sb * ex2f(mb2 - mx);
    }
    const float inv = 1.0f / sum;
    uint16_t* prow = want_p ? P + (static_cast<int64_t>(z) * S + i) * S : nullptr;
    for (int t = 0; t < nkt; ++t) {
      if (want_o && t >= 2) mbar_wait(&pfree[t & 1], ((t >> 1) - 1) & 1);  // the MMA has read tile t-2
      uint8_t* pbuf = spb + (t & 1) * PB_BYTES;
      uint32_t ra[32], rb[32];
      {
        const int c0 = t * 4 + half;
        if (c0 < nch) tmem_ld32_nowait(tq + c0 * 32, ra);
        if (c0 + 2 < nch) tmem_ld32_nowait(tq + (c0 + 2) * 32, rb);
        if (c0 < nch) tmem_ld_wait32x2(ra, rb);
      }
#pragma unroll
      for (int k2 = 0; k2 < 2; ++k2) {
        const int cc = half + 2 * k2;
        const int c = t * 4 + cc;
        uint32_t pk[16];
        if (c < nch - 1) {
          const uint32_t(&r)[32] = k2 == 0 ? ra : rb;
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            const float p0 = ex2f(fmaf(__uint_as_float(r[2 * u]), a2, -mx)) * inv;
            const float p1 = ex2f(fmaf(__uint_as_float(r[2 * u + 1]), a2, -mx)) * inv;
            pk[u] = pack_bf16(p0, p1);
          }
        } else if (c == nch - 1) {
          const uint32_t(&r)[32] = k2 == 0 ? ra : rb;
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            const int j = c * 32 + 2 * u;
            const float p0 = j <= i ? ex2f(fmaf(__uint_as_float(r[2 * u]), a2, -mx)) * inv : 0.f;
            const float p1 = j + 1 <= i ? ex2f(fmaf(__uint_as_float(r[2 * u + 1]), a2, -mx)) * inv : 0.f;
            pk[u] = pack_bf16(p0, p1);
          }
        } else {
#pragma unroll
          for (int u = 0; u < 16; ++u) pk[u] = 0u;
        }
        if (want_o) {  // SW128 K-major P tile: byte(r, key) = blk*16K + r*128 + ((key%64/8) ^ (r%8))*16 + (key%8)*2
          uint8_t* rowp = pbuf + (cc >> 1) * (PB_BYTES / 2) + il * 128;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int ch = (cc & 1) * 4 + u;
            *reinterpret_cast<uint4*>(rowp + ((ch ^ (il & 7)) << 4)) =
                make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
          }
        }
        if (want_p) {  // probabilities for backward: this row's 32 values of chunk c (64 B)
          uint4* dst = reinterpret_cast<uint4*>(prow + c * 32);
#pragma unroll
          for (int u = 0; u < 4; ++u) dst[u] = make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
        }
      }
      if (want_o) {  // P tile t visible to the tensor core; this warp's score reads are done
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&pfull[t & 1]);
      }
    }
    if (want_o && half == 0) {  // O rows of this quarter: TMEM columns [0, 64) -> bf16
      mbar_wait(ofull, 0);
      tc_fence_after();
      uint16_t* orow = O + (static_cast<int64_t>(b) * S + i) * ldo + h * HD;
#pragma unroll
      for (int cch = 0; cch < 2; ++cch) {
        float v[32];
        tmem_ld32(tq + cch * 32, v);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          uint32_t w[4];
#pragma unroll
          for (int e = 0; e < 4; ++e)
            w[e] = static_cast<uint32_t>(f2b(v[8 * u + 2 * e])) | (static_cast<uint32_t>(f2b(v[8 * u + 2 * e + 1])) << 16);
          *reinterpret_cast<uint4*>(orow + cch * 32 + u * 8) = make_uint4(w[0], w[1], w[2], w[3]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, tcols);
  }
}

// Attention backward, score-gradient part, in one tcgen05 kernel (S <= 512, hd 64):
//   dP = dO V^T (fp32, TMEM, causal key tiles), D_i = sum_j P_ij dP_ij,
//   dS_ij = bf16(P_ij (dP_ij - D_i) scale)  (0 above the diagonal)
// replacing the dO V^T GEMM (which wrote fp32 dP, 4 B per score) and the separate softmax
// backward (which read it back): per score only P is read (2 B, twice, the second time
// mostly from L2) and dS written (2 B).  CTA = (sample, head, 128 query rows); dO (128 x 64)
// and V (up to 512 x 64) arrive by TMA; the eight epilogue warps (thread = query row, two
// warps per TMEM lane quarter splitting the 32-column chunks) run D in pass 1 and dS in pass
// 2.  dS is written for key columns < m0 + 128 (every column the dQ / dK GEMMs read).
__global__ void __launch_bounds__(kThreads, 1)
    attn_bwd_ds_kernel(const __grid_constant__ CUtensorMap tmO, const __grid_constant__ CUtensorMap tmV, int H, int S,
                       float scale, const uint16_t* __restrict__ P, uint16_t* __restrict__ dS) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* so = smem;
  uint8_t* sv = smem + Q_BYTES;
  float* rowst = reinterpret_cast<float*>(sv + (kMaxS / BMq) * KT_BYTES);  // [2 halves][128]
  uint64_t* full = reinterpret_cast<uint64_t*>(rowst + 2 * BMq);  // [4] dO + V tile 0, V tiles 1..3 landed
  uint64_t* done = full + 4;                                      // [4] dO V_t^T complete
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 4);
  const int mb = blockIdx.x, z = blockIdx.y, b = z / H, h = z % H;
  const int m0 = mb * BMq, nkt = mb + 1;
  const uint32_t warp = warp_id(), lane = lane_id();
  if (threadIdx.x == 0) {
    for (int t = 0; t < kMaxS / BMq; ++t) {
      mbar_init(&full[t], 1);
      mbar_init(&done[t], 1);
    }
    mbar_fence_init();
    tma_prefetch(&tmO);
    tma_prefetch(&tmV);
  }
  int tcols = 128;
  while (tcols < nkt * BMq) tcols *= 2;
  if (warp == 1) tmem_alloc(tmem_slot, tcols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(&full[0], Q_BYTES + KT_BYTES);
      tma_load_4d(so, &tmO, &full[0], 0, h, m0, b);
      for (int t = 0; t < nkt; ++t) {
        if (t > 0) mbar_arrive_expect_tx(&full[t], KT_BYTES);
        tma_load_4d(sv + t * KT_BYTES, &tmV, &full[t], 0, h, t * BMq, b);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = umma_idesc_bf16(BMq, BMq, 0, 0);
      const uint32_t a = smem_u32(so);
      for (int t = 0; t < nkt; ++t) {
        mbar_wait(&full[t], 0);
        tc_fence_after();
        const uint32_t bv = smem_u32(sv + t * KT_BYTES);
#pragma unroll
        for (int k = 0; k < HD / 16; ++k)
          umma_bf16(tmem + t * BMq, umma_desc_sw128(a + k * 32, 16, 1024), umma_desc_sw128(bv + k * 32, 16, 1024), idesc,
                    k > 0 ? 1u : 0u);
        umma_commit(&done[t]);
      }
    }
    __syncwarp();
  } else {
    const int q = static_cast<int>(warp & 3u), half = static_cast<int>(warp - 2) >> 2;
    const int il = q * 32 + static_cast<int>(lane);
    const int i = m0 + il;
    const uint32_t tq = tmem + (static_cast<uint32_t>(q * 32) << 16);
    const int nch = (m0 + q * 32 + 32) / 32;  // chunks holding any j <= (this warp's last row)
    const uint16_t* prow = P + (static_cast<int64_t>(z) * S + i) * S;
    uint16_t* drow = dS + (static_cast<int64_t>(z) * S + i) * S;
    auto pload = [&](int c, uint32_t (&pw)[16]) {
      const uint4* src = reinterpret_cast<const uint4*>(prow + c * 32);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint4 x = src[u];
        pw[4 * u] = x.x; pw[4 * u + 1] = x.y; pw[4 * u + 2] = x.z; pw[4 * u + 3] = x.w;
      }
    };
    auto plo = [](uint32_t w) { return __uint_as_float(w << 16); };
    auto phi = [](uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); };
    int tdone = -1;  // key tiles whose dP this warp has seen complete
    // pass 1: D over this warp's chunks (P is 0 above the diagonal; the diagonal chunk is
    // masked anyway so stale dP never enters)
    float D = 0.f;
    auto absorb = [&](const uint32_t (&r)[32], const uint32_t (&pw)[16], int c) {
      if (c != nch - 1) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          D = fmaf(plo(pw[u]), __uint_as_float(r[2 * u]), D);
          D = fmaf(phi(pw[u]), __uint_as_float(r[2 * u + 1]), D);
        }
      } else {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const int j = c * 32 + 2 * u;
          if (j <= i) D = fmaf(plo(pw[u]), __uint_as_float(r[2 * u]), D);
          if (j + 1 <= i) D = fmaf(phi(pw[u]), __uint_as_float(r[2 * u + 1]), D);
        }
      }
    };
    for (int c = half; c < nch; c += 4) {
      if (c / 4 > tdone) {  // chunks c and c + 2 lie in key tile c / 4
        tdone = c / 4;
        mbar_wait(&done[tdone], 0);
        tc_fence_after();
      }
      uint32_t ra[32], rb[32], pa[16], pb[16];
      tmem_ld32_nowait(tq + c * 32, ra);
      const bool two = c + 2 < nch;
      if (two) tmem_ld32_nowait(tq + (c + 2) * 32, rb);
      pload(c, pa);
      if (two) pload(c + 2, pb);
      tmem_ld_wait32x2(ra, rb);
      absorb(ra, pa, c);
      if (two) absorb(rb, pb, c + 2);
    }
    rowst[half * BMq + il] = D;
    named_bar_sync(1, 32 * kEpi);
    D = rowst[il] + rowst[BMq + il];
    // pass 2: dS for every chunk left of the diagonal tile's end (zeros past the diagonal)
    for (int t = 0; t < nkt; ++t) {
      uint32_t ra[32], rb[32], pa[16], pb[16];
      const int c0 = t * 4 + half;
      if (c0 < nch) {
        tmem_ld32_nowait(tq + c0 * 32, ra);
        if (c0 + 2 < nch) tmem_ld32_nowait(tq + (c0 + 2) * 32, rb);
        pload(c0, pa);
        if (c0 + 2 < nch) pload(c0 + 2, pb);
        tmem_ld_wait32x2(ra, rb);
      }
#pragma unroll
      for (int k2 = 0; k2 < 2; ++k2) {
        const int c = c0 + 2 * k2;
        uint32_t o[16];
        if (c < nch) {
          const uint32_t(&r)[32] = k2 == 0 ? ra : rb;
          const uint32_t(&pw)[16] = k2 == 0 ? pa : pb;
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            const int j = c * 32 + 2 * u;
            const float g0 = plo(pw[u]) * (__uint_as_float(r[2 * u]) - D) * scale;
            const float g1 = phi(pw[u]) * (__uint_as_float(r[2 * u + 1]) - D) * scale;
            o[u] = pack_bf16(j <= i ? g0 : 0.f, j + 1 <= i ? g1 : 0.f);
          }
        } else {
#pragma unroll
          for (int u = 0; u < 16; ++u) o[u] = 0u;
        }
        uint4* dst = reinterpret_cast<uint4*>(drow + c * 32);
#pragma unroll
        for (int u = 0; u < 4; ++u) dst[u] = make_uint4(o[4 * u], o[4 * u + 1], o[4 * u + 2], o[4 * u + 3]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, tcols);
  }
}
constexpr int BWD_SMEM = Q_BYTES + (kMaxS / BMq) * KT_BYTES + 2 * BMq * 4 + 128 + 1024;

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult qr;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// (hd, head, row, sample) view of packed qkv rows (row stride 3d), box (64, 1, 128, 1)
int qkv_map(CUtensorMap* m, const void* base, int H, int S, int B, int64_t ld) {
  auto fn = encode_fn();
  if (!fn || (reinterpret_cast<uintptr_t>(base) & 15) || (ld * 2) % 16) return 2;
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(HD), static_cast<cuuint64_t>(H), static_cast<cuuint64_t>(S),
                        static_cast<cuuint64_t>(B)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(HD * 2), static_cast<cuuint64_t>(ld * 2),
                           static_cast<cuuint64_t>(ld * S * 2)};
  cuuint32_t box[4] = {64u, 1u, static_cast<cuuint32_t>(BMq), 1u};
  cuuint32_t es[4] = {1u, 1u, 1u, 1u};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS
             ? 0
             : 5;
}

}  // namespace af
}  // namespace rlhf

using namespace rlhf;

extern "C" int rlhf_attn_fwd_fused(const void* qkv, int B, int H, int hd, int S, float alpha, void* P, void* O,
                                   rlhf_stream_t stream) {
  if (hd != af::HD || S % af::BMq || S > af::kMaxS || B < 1 || H < 1 || (!P && !O)) return 2;
  const int d = H * hd;
  const auto* base = static_cast<const uint16_t*>(qkv);
  CUtensorMap tq, tk, tv;
  if (af::qkv_map(&tq, base, H, S, B, 3 * d) || af::qkv_map(&tk, base + d, H, S, B, 3 * d) ||
      af::qkv_map(&tv, base + 2 * d, H, S, B, 3 * d))
    return 2;
  static bool init = false;
  if (!init) {
    if (cudaFuncSetAttribute(af::attn_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, af::SMEM) != cudaSuccess)
      return 5;
    init = true;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  af::attn_fwd_kernel<<<dim3(S / af::BMq, B * H), af::kThreads, af::smem_bytes(P != nullptr, O != nullptr), s>>>(
      tq, tk, tv, H, S, alpha, static_cast<uint16_t*>(P), static_cast<uint16_t*>(O), static_cast<int64_t>(d));
  return cudaGetLastError() == cudaSuccess ? 0 : 5;
}

extern "C" int rlhf_attn_bwd_ds_fused(const void* dO, const void* qkv, const void* P, void* dS, int B, int H, int hd,
                                      int S, float scale, rlhf_stream_t stream) {
  if (hd != af::HD || S % af::BMq || S > af::kMaxS || B < 1 || H < 1 || !P || !dS) return 2;
  const int d = H * hd;
  CUtensorMap to, tv;
  if (af::qkv_map(&to, dO, H, S, B, d) || af::qkv_map(&tv, static_cast<const uint16_t*>(qkv) + 2 * d, H, S, B, 3 * d))
    return 2;
  static bool init = false;
  if (!init) {
    if (cudaFuncSetAttribute(af::attn_bwd_ds_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, af::BWD_SMEM) !=
        cudaSuccess)
      return 5;
    init = true;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  af::attn_bwd_ds_kernel<<<dim3(S / af::BMq, B * H), af::kThreads, af::BWD_SMEM, s>>>(
      to, tv, H, S, scale, static_cast<const uint16_t*>(P), static_cast<uint16_t*>(dS));
  return cudaGetLastError() == cudaSuccess ? 0 : 5;
}
