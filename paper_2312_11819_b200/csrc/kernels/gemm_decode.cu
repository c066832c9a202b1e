// gemm_decode.cu — HBM-bound decode GEMM: Y^T[Bg, N] = W[N, K] . X[Bg, K]^T (swap-AB).
//
// Generation-stage workhorse (reference: stage_compute_time(Generation) decode term,
// SPEC.md:209 "gen_len x max(compute, bytes_infer_per_param*P/tp / hbm)").
//  * weights fill the 128-row tcgen05 M dimension, the (<= 64) batch is N;
//  * one 128-row weight tile = one thread-block CLUSTER of `splits` CTAs (1,2,4,8),
//    each CTA streams a K-slice through TMA into smem and accumulates in TMEM;
//  * partials are reduced across the cluster through distributed shared memory
//    (mapa + ld.shared::cluster) in fixed slice order: deterministic, no global
//    workspace, no atomics;
//  * programmatic dependent launch: the weight TMA loads are issued before
//    griddepcontrol.wait (they do not depend on the previous kernel), so their
//    latency overlaps the previous kernel's tail.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <mutex>

#include "rlhf_kernels.h"
#include "sm100_common.cuh"

namespace rlhf {

namespace dec {
constexpr int BM = 128, BK = 64, kThreads = 128;

template <int BN>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int MAX_KB = BN <= 32 ? 8 : 6;
  // receive buffer: [slice][row of this CTA][PITCH] fp32.  The 16-byte row padding puts the
  // rows read by one quarter-warp (consecutive rows, same 4 columns) on distinct banks: with
  // an unpadded 128-byte row every reduction load was an 8-way bank conflict (0.5 us per
  // epilogue unit, clock64 probes)
  static constexpr int PITCH = BN + 4;
  static constexpr int PART_BYTES = BM * PITCH * 4;
  static constexpr int TAIL = 1024;               // barriers (<= 256 B) + per-row (mean, rstd) (512 B)
  static constexpr int SMEM = MAX_KB * STAGE_BYTES + PART_BYTES + TAIL + 1024;
  static int smem_for(int stages) { return stages * STAGE_BYTES + PART_BYTES + TAIL + 1024; }
};

struct Args {
  int M, N, K, splits, kb_per, stages;
  void* Y;
  int y_f32;
  int64_t ldy;  // Y element (n, m) at Y + n*ldy + m
  const uint16_t* bias;  // [M] bf16 or null
  int relu;
  const float* residual;  // same layout as Y (may alias), or null
  unsigned long long* probe;
  // fused LayerNorm prologue: X = bf16(LN(ln_x) * ln_g + ln_b), ln_x fp32 [N, K]
  const float* ln_x;
  const uint16_t* ln_g;
  const uint16_t* ln_b;
  // fused KV-cache store of the k / v column blocks of a packed qkv output
  uint16_t* kc;
  uint16_t* vc;
  const int* pos;
  int kv_d, kv_hd, kv_H, kv_Smax;
  // LayerNorm statistics between decode GEMMs: partial (sum, sum sq) out / in
  float* st_out;
  const float* st_in;
  int st_parts;
  // split-K partials staged in the (consumed) operand ring and sent to their owners with one
  // bulk DSMEM copy per owner instead of per-thread st.async stores
  int bulk;
};
__device__ __forceinline__ unsigned long long dclk() {
  unsigned long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
  return c;
}
#define DPROBE(k) do { if (e.probe && threadIdx.x == 0) e.probe[blockIdx.x * 16 + (k)] = dclk(); } while (0)

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t map_rank(uint32_t local_saddr, uint32_t rank) {
  uint32_t remote;
  asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local_saddr), "r"(rank));
  return remote;
}
// non-volatile: independent DSMEM loads may be issued back to back (ordering is
// provided by the cluster barriers around the reduction)
__device__ __forceinline__ float ld_cluster_f32(uint32_t remote) {
  float v;
  asm("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(remote));
  return v;
}
__device__ __forceinline__ float4 ld_cluster_v4(uint32_t remote) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(remote));
  return v;
}
// async 16 B store into a peer CTA's shared memory, completing bytes on the peer's mbarrier
__device__ __forceinline__ void st_async_v4(uint32_t remote_addr, float a, float b, float c, float d, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(remote_addr),
               "r"(__float_as_uint(a)), "r"(__float_as_uint(b)), "r"(__float_as_uint(c)), "r"(__float_as_uint(d)),
               "r"(remote_bar)
               : "memory");
}
__device__ __forceinline__ void cluster_arrive_relaxed() { asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.aligned;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ float b2f(uint16_t h) { return __uint_as_float(static_cast<uint32_t>(h) << 16); }

// LayerNorm prologue of the fused decode GEMM: each warp normalises RPW batch rows at a
// time (their loads in flight together), gamma/beta of this CTA's K-slice are fetched
// before griddepcontrol.wait (weights do not depend on the predecessor).  Same per-lane
// element assignment and reduction order as layernorm_kernel (rowwise.cu), so the bf16
// operand is bit-identical to the unfused LN output.
template <int VPL, int RPW>
__device__ __forceinline__ void ln_prologue(const Args& e, uint8_t* btile0, int stage_bytes, int kb0, int kb1,
                                            uint32_t warp, uint32_t lane) {
  const int K4 = e.K / 4;
  uint2 gg[VPL], bb[VPL];
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const int c = static_cast<int>(lane) + 32 * i, k = 4 * c;
    const bool in = c < K4 && k >= kb0 * BK && k < kb1 * BK;
    gg[i] = in ? *reinterpret_cast<const uint2*>(e.ln_g + k) : make_uint2(0u, 0u);
    bb[i] = in ? *reinterpret_cast<const uint2*>(e.ln_b + k) : make_uint2(0u, 0u);
  }
  pdl_wait();
  for (int n0 = static_cast<int>(warp); n0 < e.N; n0 += RPW * (kThreads / 32)) {
    float4 v[RPW][VPL];
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      const int n = n0 + r * (kThreads / 32);
      const float4* xr = reinterpret_cast<const float4*>(e.ln_x + static_cast<int64_t>(n < e.N ? n : 0) * e.K);
#pragma unroll
      for (int i = 0; i < VPL; ++i) {
        const int c = static_cast<int>(lane) + 32 * i;
        v[r][i] = (c < K4 && n < e.N) ? xr[c] : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      const int n = n0 + r * (kThreads / 32);
      if (n >= e.N) break;
      float sum = 0.f;
#pragma unroll
      for (int i = 0; i < VPL; ++i)
        if (static_cast<int>(lane) + 32 * i < K4) sum += (v[r][i].x + v[r][i].y) + (v[r][i].z + v[r][i].w);
#pragma unroll
      for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      const float mu = sum / e.K;
      float vs = 0.f;
#pragma unroll
      for (int i = 0; i < VPL; ++i) {
        if (static_cast<int>(lane) + 32 * i < K4)
          vs += (v[r][i].x - mu) * (v[r][i].x - mu) + (v[r][i].y - mu) * (v[r][i].y - mu) +
                (v[r][i].z - mu) * (v[r][i].z - mu) + (v[r][i].w - mu) * (v[r][i].w - mu);
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) vs += __shfl_xor_sync(0xffffffffu, vs, o);
      const float rs = 1.0f / sqrtf(vs / e.K + 1e-5f);
#pragma unroll
      for (int i = 0; i < VPL; ++i) {
        const int c = static_cast<int>(lane) + 32 * i;
        const int k = 4 * c;
        if (c >= K4 || k < kb0 * BK || k >= kb1 * BK) continue;
        const float y0 = (v[r][i].x - mu) * rs * b2f(static_cast<uint16_t>(gg[i].x & 0xFFFFu)) + b2f(static_cast<uint16_t>(bb[i].x & 0xFFFFu));
        const float y1 = (v[r][i].y - mu) * rs * b2f(static_cast<uint16_t>(gg[i].x >> 16)) + b2f(static_cast<uint16_t>(bb[i].x >> 16));
        const float y2 = (v[r][i].z - mu) * rs * b2f(static_cast<uint16_t>(gg[i].y & 0xFFFFu)) + b2f(static_cast<uint16_t>(bb[i].y & 0xFFFFu));
        const float y3 = (v[r][i].w - mu) * rs * b2f(static_cast<uint16_t>(gg[i].y >> 16)) + b2f(static_cast<uint16_t>(bb[i].y >> 16));
        const int j = k / BK - kb0, kk = k % BK;
        uint8_t* dst = btile0 + j * stage_bytes + n * 128 + (((kk >> 3) ^ (n & 7)) << 4) + (kk & 7) * 2;
        const uint32_t w0 = static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(y0))) |
                            (static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(y1))) << 16);
        const uint32_t w1 = static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(y2))) |
                            (static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(y3))) << 16);
        *reinterpret_cast<uint2*>(dst) = make_uint2(w0, w1);
      }
    }
  }
}

// LayerNorm prologue from the producer's partial statistics (no row re-reduction): per batch
// row, mean and rstd from the st_parts (sum, sum sq) partials (one warp per row, lanes over the
// partials, fixed order), then this CTA's K-slice normalised into the swizzled B tiles.
__device__ __forceinline__ void ln_stats_prologue(const Args& e, uint8_t* btile0, int stage_bytes, int kb0, int kb1,
                                                  uint32_t warp, uint32_t lane, float* stat) {
  const int k0 = kb0 * BK, k1 = min(kb1 * BK, e.K);
  pdl_wait();  // the partials and ln_x come from the previous kernels
  for (int n = static_cast<int>(warp); n < e.N; n += kThreads / 32) {
    float s1 = 0.f, s2 = 0.f;
    for (int q = static_cast<int>(lane); q < e.st_parts; q += 32) {
      const float2 v = *reinterpret_cast<const float2*>(e.st_in + (static_cast<int64_t>(q) * e.N + n) * 2);
      s1 += v.x;
      s2 += v.y;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
      s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    }
    if (lane == 0) {
      const float mu = s1 / e.K;
      const float var = fmaxf(s2 / e.K - mu * mu, 0.f);
      stat[2 * n] = mu;
      stat[2 * n + 1] = 1.0f / sqrtf(var + 1e-5f);
    }
  }
  __syncthreads();
  // (n, 4 consecutive k of the slice): float4 of x, 4 gamma / beta
  const int kq = (k1 - k0) / 4;
  for (int u = threadIdx.x; u < e.N * kq; u += kThreads) {
    const int n = u / kq, k = k0 + 4 * (u % kq);
    const float4 v = *reinterpret_cast<const float4*>(e.ln_x + static_cast<int64_t>(n) * e.K + k);
    const uint2 gg = *reinterpret_cast<const uint2*>(e.ln_g + k), bb = *reinterpret_cast<const uint2*>(e.ln_b + k);
    const float mu = stat[2 * n], rs = stat[2 * n + 1];
    const float y0 = (v.x - mu) * rs * b2f(static_cast<uint16_t>(gg.x & 0xFFFFu)) + b2f(static_cast<uint16_t>(bb.x & 0xFFFFu));
    const float y1 = (v.y - mu) * rs * b2f(static_cast<uint16_t>(gg.x >> 16)) + b2f(static_cast<uint16_t>(bb.x >> 16));
    const float y2 = (v.z - mu) * rs * b2f(static_cast<uint16_t>(gg.y & 0xFFFFu)) + b2f(static_cast<uint16_t>(bb.y & 0xFFFFu));
    const float y3 = (v.w - mu) * rs * b2f(static_cast<uint16_t>(gg.y >> 16)) + b2f(static_cast<uint16_t>(bb.y >> 16));
    const int j = k / BK - kb0, kk = k % BK;
    uint8_t* dst = btile0 + j * stage_bytes + n * 128 + (((kk >> 3) ^ (n & 7)) << 4) + (kk & 7) * 2;
    const uint32_t w0 = static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(y0))) |
                        (static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(y1))) << 16);
    const uint32_t w1 = static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(y2))) |
                        (static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(y3))) << 16);
    *reinterpret_cast<uint2*>(dst) = make_uint2(w0, w1);
  }
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_decode_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                       const __grid_constant__ Args e) {
  using C = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* part = reinterpret_cast<float*>(smem + e.stages * C::STAGE_BYTES);
  uint8_t* tail = smem + e.stages * C::STAGE_BYTES + C::PART_BYTES;
  float* stat = reinterpret_cast<float*>(tail + 256);
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(tail);
  uint64_t* empty_bar = full_bar + e.stages;
  uint64_t* acc_bar = empty_bar + e.stages;
  uint64_t* recv_bar = acc_bar + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(recv_bar + 1);
  const int rows_per = BM / e.splits;  // a power of two: index arithmetic by shift / mask
  const int rp_shift = __ffs(rows_per) - 1, rp_mask = rows_per - 1;

  const int split = static_cast<int>(cluster_rank());
  const int tile = blockIdx.x / e.splits;
  const int m0 = tile * BM;
  const int num_kb = (e.K + BK - 1) / BK;
  const int kb0 = split * e.kb_per;
  const int kb1 = min(num_kb, kb0 + e.kb_per);
  const int nkb = kb1 > kb0 ? kb1 - kb0 : 0;
  const uint32_t warp = warp_id(), lane = lane_id();
  DPROBE(0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < e.stages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(acc_bar, 1);
    mbar_init(recv_bar, 1);
    // every slice pushes its rows_per x BN fp32 rows of this CTA's share here (bulk mode:
    // rows_per padded rows, PITCH floats each)
    mbar_arrive_expect_tx(recv_bar, static_cast<uint32_t>(e.splits * rows_per * (e.bulk ? C::PITCH : BN) * 4));
    mbar_fence_init();
    tma_prefetch(&tmW);
    tma_prefetch(&tmX);
  }
  if (warp == 1) tmem_alloc(tmem_slot, BN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  DPROBE(1);
  pdl_trigger();  // the next kernel may start its (independent) prologue
  // the bias does not depend on the predecessor: fetch it now (every unit of this thread
  // has the same row, since rows_per divides the thread count)
  const int m_own = m0 + split * rows_per + (static_cast<int>(threadIdx.x) & rp_mask);
  const float bias_own = (e.bias && m_own < e.M) ? b2f(e.bias[m_own]) : 0.0f;
  // announce "receive barrier initialised" to the cluster now (non-blocking); the
  // matching wait sits right before the partial pushes, so a producer thread that
  // blocks on ring slots (K slices longer than the ring) cannot deadlock the MMA
  cluster_arrive_relaxed();

  const bool ln = e.ln_x != nullptr;
  if (threadIdx.x == 0) {
    // weights do not depend on the previous kernel: fill the ring with them first
    const int first = min(nkb, e.stages);
    for (int j = 0; j < first; ++j) {
      uint8_t* sa = smem + j * C::STAGE_BYTES;
      mbar_arrive_expect_tx(&full_bar[j], ln ? C::A_BYTES : C::STAGE_BYTES);
      tma_load_4d(sa, &tmW, &full_bar[j], (kb0 + j) * BK, 0, m0, 0);
    }
    DPROBE(2);
    if (!ln) {
      pdl_wait();  // activations X are produced by the previous kernel
      DPROBE(3);
      for (int j = 0; j < first; ++j) {
        uint8_t* sb = smem + j * C::STAGE_BYTES + C::A_BYTES;
        tma_load_4d(sb, &tmX, &full_bar[j], (kb0 + j) * BK, 0, 0, 0);
      }
      for (int j = first; j < nkb; ++j) {  // ring reuse once the MMA released a slot
        const int st = j % e.stages;
        mbar_wait(&empty_bar[st], ((j / e.stages) - 1) & 1);
        uint8_t* sa = smem + st * C::STAGE_BYTES;
        mbar_arrive_expect_tx(&full_bar[st], C::STAGE_BYTES);
        tma_load_4d(sa, &tmW, &full_bar[st], (kb0 + j) * BK, 0, m0, 0);
        tma_load_4d(sa + C::A_BYTES, &tmX, &full_bar[st], (kb0 + j) * BK, 0, 0, 0);
      }
    }
  }
  if (ln) {
    // LayerNorm of every batch row (full K for the statistics), written for this
    // CTA's K-slice straight into the SWIZZLE_128B K-major B tiles:
    //   byte(n, kk) = n*128 + ((kk/8) ^ (n%8))*16 + (kk%8)*2   within a 64-wide k block
    __syncwarp();  // warp 0 arrives diverged (lane 0 issued the weight TMAs alone)
    if (e.st_in) ln_stats_prologue(e, smem + C::A_BYTES, C::STAGE_BYTES, kb0, kb1, warp, lane, stat);
    else if (e.K <= 768) ln_prologue<6, 4>(e, smem + C::A_BYTES, C::STAGE_BYTES, kb0, kb1, warp, lane);
    else if (e.K <= 1024) ln_prologue<8, 2>(e, smem + C::A_BYTES, C::STAGE_BYTES, kb0, kb1, warp, lane);
    else ln_prologue<16, 1>(e, smem + C::A_BYTES, C::STAGE_BYTES, kb0, kb1, warp, lane);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> visible to tcgen05.mma
    __syncthreads();
    DPROBE(3);
  }
  if (warp == 1 && lane == 0) {
    const uint32_t idesc = umma_idesc_bf16(BM, BN, 0, 0);
    for (int j = 0; j < nkb; ++j) {
      const int st = j % e.stages;
      mbar_wait(&full_bar[st], (j / e.stages) & 1);
      tc_fence_after();
      const uint32_t sa = smem_u32(smem + st * C::STAGE_BYTES);
      const uint32_t sb = sa + C::A_BYTES;
#pragma unroll
      for (int k = 0; k < BK / 16; ++k)
        umma_bf16(tmem, umma_desc_sw128(sa + k * 32, 16, 1024), umma_desc_sw128(sb + k * 32, 16, 1024), idesc,
                  (j > 0 || k > 0) ? 1u : 0u);
      umma_commit(&empty_bar[st]);
    }
    if (nkb > 0) umma_commit(acc_bar);
    else mbar_arrive(acc_bar);
  }
  pdl_wait();  // residual (and Y when aliased) come from earlier kernels

  // ---- partial accumulator rows -> the owning CTA's receive buffer (st.async, DSMEM)
  cluster_wait();  // every peer's receive barrier is initialised
  mbar_wait(acc_bar, 0);
  DPROBE(4);
  tc_fence_after();
  if (e.bulk) {
    // thread = accumulator row -> staging row (padded pitch: conflict-free 16-byte stores),
    // then one cp.async.bulk per owner CTA: rows [o * rows_per, +rows_per) land in slot `split`
    // of its receive buffer and complete on its receive barrier
    const int row = static_cast<int>(warp) * 32 + static_cast<int>(lane);
    const uint32_t tb = tmem + (static_cast<uint32_t>(warp * 32) << 16);
    const uint32_t stg = smem_u32(smem) + static_cast<uint32_t>(row * C::PITCH * 4);
#pragma unroll
    for (int c = 0; c < BN / 32; ++c) {
      float v[32];
      if (nkb > 0) tmem_ld32(tb + c * 32, v);
      else {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = 0.0f;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q)
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(stg + static_cast<uint32_t>((c * 32 + 4 * q) * 4)),
                     "f"(v[4 * q]), "f"(v[4 * q + 1]), "f"(v[4 * q + 2]), "f"(v[4 * q + 3])
                     : "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < static_cast<unsigned>(e.splits)) {
      const uint32_t o = threadIdx.x;
      const uint32_t bytes = static_cast<uint32_t>(rows_per * C::PITCH * 4);
      const uint32_t src = smem_u32(smem) + o * bytes;
      const uint32_t dst = map_rank(smem_u32(part) + static_cast<uint32_t>(split) * bytes, o);
      const uint32_t rbar = map_rank(smem_u32(recv_bar), o);
      asm volatile(
          "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
          "r"(src), "r"(bytes), "r"(rbar)
          : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  } else {
    const int row = static_cast<int>(warp) * 32 + static_cast<int>(lane);
    const uint32_t tb = tmem + (static_cast<uint32_t>(warp * 32) << 16);
    const int owner = row / rows_per, rl = row % rows_per;
    const uint32_t dst = map_rank(smem_u32(part) + static_cast<uint32_t>(((split * rows_per + rl) * C::PITCH) * 4),
                                  static_cast<uint32_t>(owner));
    const uint32_t rbar = map_rank(smem_u32(recv_bar), static_cast<uint32_t>(owner));
#pragma unroll
    for (int c = 0; c < BN / 32; ++c) {
      float v[32];
      if (nkb > 0) tmem_ld32(tb + c * 32, v);
      else {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = 0.0f;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q)
        st_async_v4(dst + static_cast<uint32_t>((c * 32 + 4 * q) * 4), v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3],
                    rbar);
    }
  }
  tc_fence_before();
  DPROBE(5);
  // ---- reduce rows [split*rows_per, +rows_per) over the slices in slice order.
  // Work unit = (row r, 4 consecutive columns); consecutive threads -> consecutive m.
  const int units = rows_per * (BN / 4);
  // the first unit's residual (the common case: one unit per thread) is loaded while the
  // peers' partial rows are still in flight
  float res0[4] = {0.f, 0.f, 0.f, 0.f};
  if (e.residual && static_cast<int>(threadIdx.x) < units) {
    const int u = threadIdx.x, m = m0 + split * rows_per + (u & rp_mask), c4 = (u >> rp_shift) * 4;
    if (m < e.M) {
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (c4 + t < e.N) res0[t] = e.residual[static_cast<int64_t>(c4 + t) * e.ldy + m];
    }
  }
  // KV-cache destination of this thread's output row (loop-invariant: every unit of the
  // thread has m == m_own): cache element (n, h, *pos, ee) = kv_row + n * H * Smax * hd
  uint16_t* kv_row = nullptr;
  if (e.kc && m_own < e.M && m_own >= e.kv_d) {
    const int mm = m_own - e.kv_d, which = mm / e.kv_d, within = mm % e.kv_d;
    const int h = within / e.kv_hd, ee = within % e.kv_hd;
    kv_row = (which == 0 ? e.kc : e.vc) + (static_cast<int64_t>(h) * e.kv_Smax + *e.pos) * e.kv_hd + ee;
  }
  const int64_t kv_nstride = static_cast<int64_t>(e.kv_H) * e.kv_Smax * e.kv_hd;
  mbar_wait(recv_bar, 0);  // all slices' rows of this CTA's share have landed
  DPROBE(6);

#pragma unroll 1
  for (int u = threadIdx.x; u < units; u += kThreads) {
    const int rl = u & rp_mask;
    const int r = split * rows_per + rl;
    const int c4 = (u >> rp_shift) * 4;
    const int m = m0 + r;
    const bool mok = m < e.M;
    float res[4] = {res0[0], res0[1], res0[2], res0[3]};
    if (e.residual && mok && u >= kThreads) {
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (c4 + t < e.N) res[t] = e.residual[static_cast<int64_t>(c4 + t) * e.ldy + m];
    }
    const float bm = bias_own;  // m == m_own
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 8
    for (int s2 = 0; s2 < e.splits; ++s2) {  // fixed slice order
      const float4 v = *reinterpret_cast<const float4*>(part + (s2 * rows_per + rl) * C::PITCH + c4);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    const float a4[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int n = c4 + t;
      if (!mok || n >= e.N) continue;
      float x = a4[t] + bm;
      if (e.relu) x = fmaxf(x, 0.0f);
      x += res[t];
      const int64_t o = static_cast<int64_t>(n) * e.ldy + m;
      if (e.y_f32) {
        static_cast<float*>(e.Y)[o] = x;
      } else {
        const uint16_t hb = __bfloat16_as_ushort(__float2bfloat16_rn(x));
        static_cast<uint16_t*>(e.Y)[o] = hb;
        if (kv_row) kv_row[n * kv_nstride] = hb;  // k / v columns of qkv -> KV cache [n][h][pos][e]
      }
    }
  }
  if (e.st_out) {
    // this CTA's partial LayerNorm statistics of the output rows it just stored, per batch
    // column: one warp per column, lanes over the rows (read back from Y, visible to the CTA
    // after the barrier; rows past M count 0)
    __syncthreads();
    const float* yf = static_cast<const float*>(e.Y);
    for (int n = static_cast<int>(warp); n < e.N; n += kThreads / 32) {
      float s1 = 0.f, s2 = 0.f;
      for (int r = static_cast<int>(lane); r < rows_per; r += 32) {
        const int m = m0 + split * rows_per + r;
        const float v = m < e.M ? yf[static_cast<int64_t>(n) * e.ldy + m] : 0.f;
        s1 += v;
        s2 += v * v;
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
      }
      if (lane == 0)
        *reinterpret_cast<float2*>(e.st_out + (static_cast<int64_t>(blockIdx.x) * e.N + n) * 2) = make_float2(s1, s2);
    }
  }
  DPROBE(7);
  DPROBE(8);
  if (e.bulk && threadIdx.x < static_cast<unsigned>(e.splits))
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // staging rows read out before exit
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, BN);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode() {
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

int map2d(CUtensorMap* m, const void* ptr, int64_t K, int64_t rows, int64_t ld, int box_rows) {
  auto fn = encode();
  if (!fn || (reinterpret_cast<uintptr_t>(ptr) & 15) || (ld * 2) % 16) return 2;
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(K), 1, static_cast<cuuint64_t>(rows), 1};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(ld * rows * 2), static_cast<cuuint64_t>(ld * 2),
                           static_cast<cuuint64_t>(ld * rows * 2)};
  cuuint32_t box[4] = {64u, 1u, static_cast<cuuint32_t>(box_rows), 1u};
  cuuint32_t es[4] = {1u, 1u, 1u, 1u};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(ptr), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS
             ? 0
             : 5;
}

template <int BN>
int launch(const CUtensorMap& tw, const CUtensorMap& tx, const Args& a, int tiles, int pdl, cudaStream_t s) {
  using C = Cfg<BN>;
  static bool init = false;
  if (!init) {
    if (cudaFuncSetAttribute(gemm_decode_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM) != cudaSuccess)
      return 5;
    // 16 K-slices per tile = a 16-CTA cluster (non-portable size, allowed on B200)
    cudaFuncSetAttribute(gemm_decode_kernel<BN>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    init = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(tiles * a.splits);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = C::smem_for(a.stages);
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = a.splits;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, gemm_decode_kernel<BN>, tw, tx, a) == cudaSuccess ? 0 : 5;
}

}  // namespace dec
}  // namespace rlhf

using namespace rlhf;

extern "C" int rlhf_gemm_decode(const rlhf_gemm_decode_params* p, rlhf_stream_t stream) {
  const int bn = p->N <= 32 ? 32 : 64;
  if (p->N < 1 || p->N > 64 || p->M < 1 || p->K < 1 || p->K % 8) return 2;
  const int num_kb = (p->K + dec::BK - 1) / dec::BK;
  const int max_kb = bn == 32 ? dec::Cfg<32>::MAX_KB : dec::Cfg<64>::MAX_KB;
  const int splits = p->splits;
  if (splits != 1 && splits != 2 && splits != 4 && splits != 8 && splits != 16) return 2;
  const int kb_per = (num_kb + splits - 1) / splits;
  // smem ring (weights stream through it); a grid larger than the SM count gets a
  // 4-stage ring so two CTAs fit per SM and every CTA is resident at once
  int sms = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int tiles_all = (p->M + dec::BM - 1) / dec::BM;
  const bool big_grid = tiles_all * splits > sms && !p->ln_x;  // (the LN prologue needs every B tile resident)
  const int stages = std::min(kb_per, big_grid ? std::min(max_kb, 4) : max_kb);
  if (p->ln_x && kb_per > stages) return 2;    // fused LN writes every B tile up front
  CUtensorMap tw, tx;
  if (dec::map2d(&tw, p->W, p->K, p->M, p->ldw, dec::BM)) return 2;
  if (dec::map2d(&tx, p->X ? p->X : p->W, p->K, p->X ? p->N : p->M, p->X ? p->ldx : p->ldw, bn)) return 2;
  dec::Args a{};
  a.M = p->M;
  a.N = p->N;
  a.K = p->K;
  a.splits = splits;
  a.kb_per = kb_per;
  a.stages = stages;
  static const int bulk_env = [] { const char* v = getenv("RLHF_DEC_BULK_PUSH"); return v ? atoi(v) : 1; }();
  const int pitch = bn == 32 ? dec::Cfg<32>::PITCH : dec::Cfg<64>::PITCH;
  const int stage_bytes = bn == 32 ? dec::Cfg<32>::STAGE_BYTES : dec::Cfg<64>::STAGE_BYTES;
  a.bulk = bulk_env && splits > 1 && stages * stage_bytes >= dec::BM * pitch * 4;
  a.Y = p->Y;
  a.y_f32 = p->y_f32;
  a.ldy = p->ldy;
  a.bias = static_cast<const uint16_t*>(p->bias);
  a.relu = p->relu;
  a.residual = p->residual;
  a.probe = p->probe;
  a.ln_x = p->ln_x;
  a.ln_g = static_cast<const uint16_t*>(p->ln_g);
  a.ln_b = static_cast<const uint16_t*>(p->ln_b);
  a.kc = static_cast<uint16_t*>(p->kcache);
  a.vc = static_cast<uint16_t*>(p->vcache);
  a.pos = p->pos;
  a.kv_d = p->kv_d;
  a.kv_hd = p->kv_hd;
  a.kv_H = p->kv_H;
  a.kv_Smax = p->kv_Smax;
  a.st_out = p->ln_stats_out;
  a.st_in = p->ln_stats_in;
  a.st_parts = p->ln_stats_parts;
  if (a.st_in && (!a.ln_x || a.st_parts < 1)) return 2;
  if (a.st_out && !p->y_f32) return 2;  // statistics of the fp32 residual stream
  if (a.ln_x && (p->K > 2048 || p->K % 4 || p->N > 64)) return 2;
  if (a.kc && (p->y_f32 || !p->pos || p->M != 3 * p->kv_d)) return 2;
  const int tiles = (p->M + dec::BM - 1) / dec::BM;
  if (p->ln_stats_parts_out) *p->ln_stats_parts_out = tiles * splits;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  return bn == 32 ? dec::launch<32>(tw, tx, a, tiles, p->pdl, s) : dec::launch<64>(tw, tx, a, tiles, p->pdl, s);
}
