// gemm_sm100.cu — warp-specialised tcgen05 + TMA GEMM for sm_100a.
//
// Serves every matmul of the PPO step (reference TaskKind work items,
// costmodel.hpp:63-64 / SPEC.md:209):
//   forward  Y = X W^T        (A K-major, B K-major)
//   decode   Y^T = W X^T      (swap-AB: weights fill the 128-row MMA M, batch is N)
//   backward dX = dY W        (B MN-major)      dW = dY^T X   (A, B MN-major)
//   attention S = Q K^T, O = P V, dP, dQ, dK, dV (batched over (b, h), causal tile skipping)
//
// CTA = 192 threads: warp 0 TMA producer, warp 1 TMEM allocator + single-thread
// UMMA issuer, warps 2-5 epilogue (TMEM -> registers -> fused epilogue -> HBM).
// Tile 128 x BN x 64 (BN in {32, 64, 128, 256}), 4-8 stage mbarrier ring,
// SWIZZLE_128B smem operands, fp32 accumulator in TMEM (BN columns).
// Deterministic split-K: every split writes its fp32 partial, the last CTA of a
// tile (atomic ticket) reduces all partials in split order and runs the epilogue.
#include <cudaTypedefs.h>

#include <cstdio>
#include <mutex>

#include "rlhf_kernels.h"
#include "sm100_common.cuh"

namespace rlhf {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kThreads = 192;

template <int BN>
struct TileCfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  // narrow tiles serve decode (few k-blocks per CTA): 4 stages -> 2-3 CTAs/SM
  static constexpr int RAW_STAGES = BN <= 64 ? 4 : (196 * 1024) / STAGE_BYTES;
  static constexpr int STAGES = RAW_STAGES > 8 ? 8 : RAW_STAGES;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
};

struct GemmArgs {
  int M, N, batch_h, splits, num_kb, tiles_m, tiles_n;
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
};

__device__ __forceinline__ float bf16_bits_to_f32(uint16_t h) { return __uint_as_float(static_cast<uint32_t>(h) << 16); }

__device__ __forceinline__ uint16_t f32_to_bf16_bits(float f) {
  return __bfloat16_as_ushort(__float2bfloat16_rn(f));
}

// Apply the fused epilogue to 32 consecutive columns of one row and store.
__device__ __forceinline__ void epilogue_store(const GemmArgs& e, int b, int h, int m, int n_base, float (&v)[32]) {
  if (m >= e.M) return;
  const int64_t cbase = b * e.c_sb + h * e.c_sh + static_cast<int64_t>(m) * e.c_rs;
  float bm = 0.0f;
  if (e.bias && e.bias_along_m)
    bm = e.bias_f32 ? static_cast<const float*>(e.bias)[m] : bf16_bits_to_f32(static_cast<const uint16_t*>(e.bias)[m]);
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const int n = n_base + j;
    float x = v[j] * e.alpha;
    if (e.bias) {
      if (e.bias_along_m) x += bm;
      else if (n < e.N)
        x += e.bias_f32 ? static_cast<const float*>(e.bias)[n] : bf16_bits_to_f32(static_cast<const uint16_t*>(e.bias)[n]);
    }
    if (e.relu) x = fmaxf(x, 0.0f);
    if (e.aux && n < e.N) {
      const uint16_t a = e.aux[b * e.c_sb + h * e.c_sh + static_cast<int64_t>(m) * e.aux_rs + static_cast<int64_t>(n) * e.aux_cs];
      if ((a & 0x8000u) || a == 0) x = 0.0f;
    }
    if (e.residual && n < e.N) x += e.residual[cbase + static_cast<int64_t>(n) * e.c_cs];
    v[j] = x;
  }
  const bool full = n_base + 32 <= e.N;
  if (e.c_cs == 1 && full) {
    if (e.c_f32) {
      float* dst = static_cast<float*>(e.C) + cbase + n_base;
      if ((reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
        float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          float4 o = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
          if (e.accumulate) {
            const float4 old = d4[q];
            o.x += old.x; o.y += old.y; o.z += old.z; o.w += old.w;
          }
          d4[q] = o;
        }
        return;
      }
    } else {
      uint16_t* dst = static_cast<uint16_t*>(e.C) + cbase + n_base;
      if ((reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
        uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float f[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) f[t] = v[8 * q + t];
          if (e.accumulate) {
            const uint4 old = d4[q];
            const uint32_t ow[4] = {old.x, old.y, old.z, old.w};
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              f[2 * t] += bf16_bits_to_f32(static_cast<uint16_t>(ow[t] & 0xFFFFu));
              f[2 * t + 1] += bf16_bits_to_f32(static_cast<uint16_t>(ow[t] >> 16));
            }
          }
          uint32_t w[4];
#pragma unroll
          for (int t = 0; t < 4; ++t)
            w[t] = static_cast<uint32_t>(f32_to_bf16_bits(f[2 * t])) | (static_cast<uint32_t>(f32_to_bf16_bits(f[2 * t + 1])) << 16);
          d4[q] = make_uint4(w[0], w[1], w[2], w[3]);
        }
        return;
      }
    }
  }
#pragma unroll 4
  for (int j = 0; j < 32; ++j) {
    const int n = n_base + j;
    if (n >= e.N) break;
    const int64_t off = cbase + static_cast<int64_t>(n) * e.c_cs;
    if (e.c_f32) {
      float* d = static_cast<float*>(e.C) + off;
      *d = e.accumulate ? *d + v[j] : v[j];
    } else {
      uint16_t* d = static_cast<uint16_t*>(e.C) + off;
      const float x = e.accumulate ? bf16_bits_to_f32(*d) + v[j] : v[j];
      *d = f32_to_bf16_bits(x);
    }
  }
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 2)
    gemm_sm100_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const GemmArgs e) {
  using Cfg = TileCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty_bar = full_bar + Cfg::STAGES;
  uint64_t* acc_bar = empty_bar + Cfg::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_bar + 1);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int n_tile = blockIdx.x, m_tile = blockIdx.y;
  const int z = blockIdx.z / e.splits, split = blockIdx.z % e.splits;
  const int h = z % e.batch_h, b = z / e.batch_h;
  const int m0 = m_tile * BM, n0 = n_tile * BN;
  if (e.causal == 1 && n0 > m0 + BM - 1) return;  // tile strictly above the diagonal

  int kb_begin = 0, kb_end = e.num_kb;
  if (e.causal == 2) kb_end = min(kb_end, (m0 + BM + BK - 1) / BK);
  if (e.causal == 3) kb_begin = m0 / BK;
  if (e.splits > 1) {
    const int per = (e.num_kb + e.splits - 1) / e.splits;
    kb_begin = split * per;
    kb_end = min(e.num_kb, kb_begin + per);
  }
  const int nkb = kb_end > kb_begin ? kb_end - kb_begin : 0;

  const uint32_t warp = warp_id(), lane = lane_id();
  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(acc_bar, 1);
    mbar_fence_init();
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
  }
  if (warp == 1) tmem_alloc(tmem_slot, BN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = kb_begin; kb < kb_end; ++kb) {
        mbar_wait(&empty_bar[stage], phase ^ 1u);
        uint8_t* sa = smem + stage * Cfg::STAGE_BYTES;
        uint8_t* sb = sa + Cfg::A_BYTES;
        mbar_arrive_expect_tx(&full_bar[stage], Cfg::STAGE_BYTES);
        const int k0 = kb * BK;
        if (!e.a_mn) {
          tma_load_4d(sa, &tmA, &full_bar[stage], k0, h, m0, b);
        } else {
#pragma unroll
          for (int j = 0; j < BM / 64; ++j) tma_load_4d(sa + j * 8192, &tmA, &full_bar[stage], m0 + 64 * j, h, k0, b);
        }
        if (!e.b_mn) {
          tma_load_4d(sb, &tmB, &full_bar[stage], k0, h, n0, b);
        } else {
#pragma unroll
          for (int j = 0; j < BN / 64; ++j) tma_load_4d(sb + j * 8192, &tmB, &full_bar[stage], n0 + 64 * j, h, k0, b);
        }
        if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1u; }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- UMMA issuer (one thread)
      const uint32_t idesc = umma_idesc_bf16(BM, BN, e.a_mn, e.b_mn);
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = kb_begin; kb < kb_end; ++kb) {
        mbar_wait(&full_bar[stage], phase);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + stage * Cfg::STAGE_BYTES);
        const uint32_t sb = sa + Cfg::A_BYTES;
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) {
          const uint64_t ad = e.a_mn ? umma_desc_sw128(sa + k * 2048, 8192, 1024) : umma_desc_sw128(sa + k * 32, 16, 1024);
          const uint64_t bd = e.b_mn ? umma_desc_sw128(sb + k * 2048, 8192, 1024) : umma_desc_sw128(sb + k * 32, 16, 1024);
          umma_bf16(tmem, ad, bd, idesc, (kb > kb_begin || k > 0) ? 1u : 0u);
        }
        umma_commit(&empty_bar[stage]);  // frees the smem slot when these MMAs retire
        if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1u; }
      }
      if (nkb > 0) umma_commit(acc_bar);
      else mbar_arrive(acc_bar);
    }
    __syncwarp();
  } else {  // ---- epilogue warps 2..5: TMEM lane quarter = warp % 4
    mbar_wait(acc_bar, 0);
    tc_fence_after();
    const int q = static_cast<int>(warp & 3u);
    const int row = q * 32 + static_cast<int>(lane);
    const int m = m0 + row;
    const uint32_t tbase = tmem + (static_cast<uint32_t>(q * 32) << 16);
    bool final_pass = true;
    size_t tile_id = 0;
    if (e.splits > 1) {
      tile_id = (static_cast<size_t>(z) * e.tiles_m + m_tile) * e.tiles_n + n_tile;
      float* mine = e.ws + ((tile_id * e.splits + split) * BM + row) * BN;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        float v[32];
        if (nkb > 0) tmem_ld32(tbase + c * 32, v);
        else {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = 0.0f;
        }
        float4* d4 = reinterpret_cast<float4*>(mine + c * 32);
#pragma unroll
        for (int t = 0; t < 8; ++t) d4[t] = make_float4(v[4 * t], v[4 * t + 1], v[4 * t + 2], v[4 * t + 3]);
      }
      __threadfence();
      named_bar_sync(1, 128);
      if (threadIdx.x == 64) *last_flag = (atomicAdd(&e.counters[tile_id], 1) == e.splits - 1);
      named_bar_sync(1, 128);
      final_pass = *last_flag != 0;
      __threadfence();
    }
    if (final_pass) {
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        float v[32];
        if (e.splits > 1) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = 0.0f;
          for (int s = 0; s < e.splits; ++s) {  // fixed order -> deterministic
            const float4* src = reinterpret_cast<const float4*>(e.ws + ((tile_id * e.splits + s) * BM + row) * BN + c * 32);
#pragma unroll
            for (int t = 0; t < 8; ++t) {
              const float4 p = __ldcg(src + t);
              v[4 * t] += p.x; v[4 * t + 1] += p.y; v[4 * t + 2] += p.z; v[4 * t + 3] += p.w;
            }
          }
        } else if (nkb > 0) {
          tmem_ld32(tbase + c * 32, v);
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = 0.0f;
        }
        epilogue_store(e, b, h, m, n0 + c * 32, v);
      }
      if (e.splits > 1 && threadIdx.x == 64) e.counters[tile_id] = 0;  // re-arm for the next launch
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, BN);
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

template <int BN>
static int launch(const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& a, dim3 grid, cudaStream_t s) {
  using Cfg = TileCfg<BN>;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(gemm_sm100_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM) != cudaSuccess)
      return 5;
    configured = true;
  }
  gemm_sm100_kernel<BN><<<grid, kThreads, Cfg::SMEM, s>>>(ta, tb, a);
  return cudaGetLastError() == cudaSuccess ? 0 : 5;
}

}  // namespace rlhf

using namespace rlhf;

extern "C" int rlhf_gemm_block_n(const rlhf_gemm_params* p) { return pick_bn(p); }

extern "C" size_t rlhf_gemm_workspace_bytes(const rlhf_gemm_params* p) {
  if (p->split_k <= 1) return 0;
  const int bn = pick_bn(p);
  const size_t tiles = static_cast<size_t>((p->M + BM - 1) / BM) * ((p->N + bn - 1) / bn) * p->batch;
  return tiles * p->split_k * BM * bn * sizeof(float);
}

extern "C" int rlhf_gemm(const rlhf_gemm_params* p, rlhf_stream_t stream) {
  if (p->M <= 0 || p->N <= 0 || p->K <= 0 || p->batch <= 0 || p->batch_h <= 0 || p->batch % p->batch_h) return 2;
  const int bn = pick_bn(p);
  if (bn != 32 && bn != 64 && bn != 128 && bn != 256) return 2;
  if (p->b_mn_major && bn < 64) return 2;
  const int splits = p->split_k > 1 ? p->split_k : 1;
  if (splits > 1 && p->causal) return 2;
  const int bb = p->batch / p->batch_h;
  CUtensorMap ta, tb;
  int st;
  // A: K-major -> (K, h, M, b) box (64, 1, 128, 1); MN-major -> (M, h, K, b) box (64, 1, 64, 1)
  if (!p->a_mn_major) st = make_map(&ta, p->A, p->K, p->M, p->lda, p->a_stride_h, p->a_stride_b, p->batch_h, bb, BM);
  else st = make_map(&ta, p->A, p->M, p->K, p->lda, p->a_stride_h, p->a_stride_b, p->batch_h, bb, BK);
  if (st) return st;
  if (!p->b_mn_major) st = make_map(&tb, p->B, p->K, p->N, p->ldb, p->b_stride_h, p->b_stride_b, p->batch_h, bb, bn);
  else st = make_map(&tb, p->B, p->N, p->K, p->ldb, p->b_stride_h, p->b_stride_b, p->batch_h, bb, BK);
  if (st) return st;

  GemmArgs a{};
  a.M = p->M;
  a.N = p->N;
  a.batch_h = p->batch_h;
  a.splits = splits;
  a.num_kb = (p->K + BK - 1) / BK;
  a.tiles_m = (p->M + BM - 1) / BM;
  a.tiles_n = (p->N + bn - 1) / bn;
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
  if (splits > 1) {
    if (!p->workspace || p->workspace_bytes < rlhf_gemm_workspace_bytes(p)) return 2;
    if (!p->counters || p->counters_len < a.tiles_m * a.tiles_n * p->batch) return 2;
    a.ws = static_cast<float*>(p->workspace);
    a.counters = p->counters;
  }
  dim3 grid(a.tiles_n, a.tiles_m, p->batch * splits);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  switch (bn) {
    case 32: return launch<32>(ta, tb, a, grid, s);
    case 64: return launch<64>(ta, tb, a, grid, s);
    case 128: return launch<128>(ta, tb, a, grid, s);
    default: return launch<256>(ta, tb, a, grid, s);
  }
}
