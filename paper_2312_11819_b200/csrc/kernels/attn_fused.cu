// attn_fused.cu — causal attention scores + softmax in one tcgen05 kernel (prefill,
// Forward x4, TrainFB forward), for sequences S <= 512 and head dim 64.
//
// The unfused path writes the fp32 score matrix S = alpha Q K^T (B*H*S*S*4 bytes,
// 400 MB per layer for c2) and reads it back in a separate softmax kernel.  Here one
// CTA owns (sample, head, 128 query rows): Q (128 x 64) and the causal key range K
// (up to 512 x 64) arrive by TMA (SWIZZLE_128B), tcgen05.mma writes the 128 x (m0+128)
// fp32 score tile into TMEM (<= 512 columns), and four epilogue warps (one TMEM lane
// quarter each, thread = query row) run an online max / sum pass and a second pass that
// writes P = bf16(exp(s - max) / sum) (zeros above the diagonal) through a shared-memory
// transpose as coalesced row segments.  Only P (bf16) reaches HBM.  Eight epilogue
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
constexpr int STG_PITCH = 40;           // bf16 staging row pitch (80 B: conflict-light)
constexpr int SMEM = Q_BYTES + (kMaxS / BMq) * KT_BYTES + kEpi * 32 * STG_PITCH * 2 + 4 * BMq * 4 + 1024 + 128;

__device__ __forceinline__ uint16_t f2b(float f) { return __bfloat16_as_ushort(__float2bfloat16_rn(f)); }

__global__ void __launch_bounds__(kThreads, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK, int H, int S,
                    float alpha, uint16_t* __restrict__ P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sq = smem;
  uint8_t* sk = smem + Q_BYTES;
  uint16_t* stg = reinterpret_cast<uint16_t*>(sk + (kMaxS / BMq) * KT_BYTES);
  float* rowst = reinterpret_cast<float*>(stg + kEpi * 32 * STG_PITCH);  // [2 halves][max, sum][128 rows]
  uint64_t* full = reinterpret_cast<uint64_t*>(rowst + 4 * BMq);
  uint64_t* done = full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

  const int mb = blockIdx.x, z = blockIdx.y, b = z / H, h = z % H;
  const int m0 = mb * BMq;
  const int nkt = mb + 1;  // causal key tiles
  const uint32_t warp = warp_id(), lane = lane_id();
  if (threadIdx.x == 0) {
    mbar_init(full, 1);
    mbar_init(done, 1);
    mbar_fence_init();
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
  }
  int tcols = 128;  // causal extent (nkt * 128 columns), rounded up to a power of two
  while (tcols < nkt * BMq) tcols *= 2;
  if (warp == 1) tmem_alloc(tmem_slot, tcols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(full, Q_BYTES + nkt * KT_BYTES);
      tma_load_4d(sq, &tmQ, full, 0, h, m0, b);
      for (int t = 0; t < nkt; ++t) tma_load_4d(sk + t * KT_BYTES, &tmK, full, 0, h, t * BMq, b);
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = umma_idesc_bf16(BMq, BMq, 0, 0);
      mbar_wait(full, 0);
      tc_fence_after();
      const uint32_t a = smem_u32(sq);
      for (int t = 0; t < nkt; ++t) {
        const uint32_t bk = smem_u32(sk + t * KT_BYTES);
#pragma unroll
        for (int k = 0; k < HD / 16; ++k)
          umma_bf16(tmem + t * BMq, umma_desc_sw128(a + k * 32, 16, 1024), umma_desc_sw128(bk + k * 32, 16, 1024), idesc,
                    k > 0 ? 1u : 0u);
      }
      umma_commit(done);
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
    const int nout = (m0 + BMq) / 32;         // chunks written (the block's causal extent)
    mbar_wait(done, 0);
    tc_fence_after();
    float mx = -FLT_MAX, sum = 0.f;
    for (int c = half; c < nch; c += 2) {
      float v[32];
      tmem_ld32(tq + c * 32, v);
      float cm = -FLT_MAX;
#pragma unroll
      for (int t = 0; t < 32; ++t) {
        v[t] *= alpha;
        if (c * 32 + t <= i) cm = fmaxf(cm, v[t]);
      }
      const float nm = fmaxf(mx, cm);
      if (nm == -FLT_MAX) continue;  // whole chunk above this row's diagonal
      float cs = 0.f;
#pragma unroll
      for (int t = 0; t < 32; ++t)
        if (c * 32 + t <= i) cs += __expf(v[t] - nm);
      sum = (mx == -FLT_MAX ? 0.f : sum * __expf(mx - nm)) + cs;
      mx = nm;
    }
    rowst[(half * 2) * BMq + il] = mx;
    rowst[(half * 2 + 1) * BMq + il] = sum;
    named_bar_sync(1, 32 * kEpi);
    {
      const float ma = rowst[il], sa = rowst[BMq + il], mb2 = rowst[2 * BMq + il], sb = rowst[3 * BMq + il];
      mx = fmaxf(ma, mb2);
      sum = (ma == -FLT_MAX ? 0.f : sa * __expf(ma - mx)) + (mb2 == -FLT_MAX ? 0.f : sb * __expf(mb2 - mx));
    }
    const float inv = 1.0f / sum;
    uint16_t* st = stg + (warp - 2) * 32 * STG_PITCH;
    uint16_t* prow0 = P + (static_cast<int64_t>(z) * S + m0 + q * 32) * S;
    for (int c = half; c < nout; c += 2) {
      uint32_t pk[16];
      if (c < nch) {
        float v[32];
        tmem_ld32(tq + c * 32, v);
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          const int j = c * 32 + 2 * t;
          const float p0 = j <= i ? __expf(v[2 * t] * alpha - mx) * inv : 0.f;
          const float p1 = j + 1 <= i ? __expf(v[2 * t + 1] * alpha - mx) * inv : 0.f;
          pk[t] = static_cast<uint32_t>(f2b(p0)) | (static_cast<uint32_t>(f2b(p1)) << 16);
        }
      } else {
#pragma unroll
        for (int t = 0; t < 16; ++t) pk[t] = 0u;
      }
      // transpose through smem: row `lane` of this warp's 32 x 32 bf16 block
      uint32_t* srow = reinterpret_cast<uint32_t*>(st + lane * STG_PITCH);
#pragma unroll
      for (int t = 0; t < 16; ++t) srow[t] = pk[t];
      __syncwarp();
      // 32 rows x 64 B: lane -> (row lane/4 + 8 r, 16 B segment lane%4)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int row = static_cast<int>(lane >> 2) + 8 * r, seg = static_cast<int>(lane & 3);
        const uint4 val = *reinterpret_cast<const uint4*>(st + row * STG_PITCH + seg * 8);
        *reinterpret_cast<uint4*>(prow0 + static_cast<int64_t>(row) * S + c * 32 + seg * 8) = val;
      }
      __syncwarp();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, tcols);
  }
}

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

extern "C" int rlhf_attn_fwd_fused(const void* qkv, int B, int H, int hd, int S, float alpha, void* P,
                                   rlhf_stream_t stream) {
  if (hd != af::HD || S % af::BMq || S > af::kMaxS || B < 1 || H < 1) return 2;
  const int d = H * hd;
  CUtensorMap tq, tk;
  if (af::qkv_map(&tq, qkv, H, S, B, 3 * d) || af::qkv_map(&tk, static_cast<const uint16_t*>(qkv) + d, H, S, B, 3 * d))
    return 2;
  static bool init = false;
  if (!init) {
    if (cudaFuncSetAttribute(af::attn_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, af::SMEM) != cudaSuccess)
      return 5;
    init = true;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  af::attn_fwd_kernel<<<dim3(S / af::BMq, B * H), af::kThreads, af::SMEM, s>>>(tq, tk, H, S, alpha,
                                                                                 static_cast<uint16_t*>(P));
  return cudaGetLastError() == cudaSuccess ? 0 : 5;
}
