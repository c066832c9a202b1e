// engine_model.cpp — per-model execution on one device: weight init, the
// teacher-forced forward (Forward / TrainFB tasks), the backward pass, the
// LM-head logprobs and greedy generation (Generation task: prefill + CUDA-graph
// decode loop).  Every launch goes through the C-ABI of include/rlhf_kernels.h.
// Rounding points follow DESIGN.md §3 and are mirrored by oracle/ppo_oracle.cpp.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <vector>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <thread>

#include "engine.hpp"
#include "flexrlhf/errors.hpp"
#include "nccl_dyn.hpp"

namespace flexrlhf {

std::atomic<int64_t> g_device_bytes{0};

DevBuf::~DevBuf() {
  if (p) {
    cudaFree(p);
    g_device_bytes -= static_cast<int64_t>(bytes);
  }
}

void DevBuf::alloc(size_t n) {
  if (p) {
    cudaFree(p);
    g_device_bytes -= static_cast<int64_t>(bytes);
  }
  p = nullptr;
  bytes = 0;
  if (n == 0) return;
  if (cudaMalloc(&p, n) != cudaSuccess) {
    cudaGetLastError();
    p = nullptr;
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    // an allocation the placement cannot hold is an infeasible plan (exit code 3,
    // reference errors.hpp), not a device fault
    throw InfeasibleError("device allocation of " + std::to_string(n) + " bytes does not fit (" +
                          std::to_string(free_b) + " of " + std::to_string(total_b) + " bytes free)");
  }
  bytes = n;
  g_device_bytes += static_cast<int64_t>(n);
  cudaMemset(p, 0, n);
}

Arena::~Arena() {
  for (DevBuf* b : owned) delete b;
}

void Engine::kcheck(int status, const char* what) {
  if (status != 0) {
    cudaError_t e = cudaGetLastError();
    throw DeviceError(std::string(what) + " failed (status " + std::to_string(status) + ", " + cudaGetErrorString(e) + ")");
  }
}

#define NK(x)                                                                                     \
  do {                                                                                            \
    ncclResult_t r_ = (x);                                                                        \
    if (r_ != ncclSuccess) throw DeviceError(std::string(#x) + ": " + nccl().GetErrorString(r_)); \
  } while (0)
#define CK(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess) throw DeviceError(std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)
#define K(call, n)                \
  do {                            \
    kcheck((call), #call);        \
    launches_ += (n);             \
  } while (0)

void Engine::gemm(rlhf_gemm_params& p) {
  if (p.split_k > 1) {
    p.workspace = arp_->gemm_ws;
    p.workspace_bytes = arp_->gemm_ws_bytes;
    p.counters = arp_->counters;
    p.counters_len = arp_->counters_len;
    if (rlhf_gemm_workspace_bytes(&p) > arp_->gemm_ws_bytes) p.split_k = 1;
  }
  K(rlhf_gemm(&p, stream_), 1);
}

// Y[M,N] = X[M,K] W[N,K]^T (+bias) (relu) (+residual), token-major output.
void Engine::linear(const uint16_t* X, int M, int Kd, const uint16_t* W, int N, const uint16_t* bias, void* Y,
                    bool y_f32, bool relu, const float* residual) {
  rlhf_gemm_params p{};
  p.M = M; p.N = N; p.K = Kd; p.batch = 1; p.batch_h = 1;
  p.A = X; p.lda = Kd;
  p.B = W; p.ldb = Kd;
  p.C = Y; p.c_f32 = y_f32; p.c_rs = N; p.c_cs = 1;
  p.alpha = 1.0f;
  p.bias = bias;
  p.relu = relu;
  p.residual = residual;
  gemm(p);
}

// Decode: Y[Bg, N_out] via the swap-AB decode GEMM (weights fill the MMA M
// dimension); K split over a thread-block cluster so ~2 CTAs per SM stream weights.
void Engine::linear_decode(const uint16_t* W, int N_out, int Kd, const uint16_t* X, int Bg, const uint16_t* bias,
                           void* Y, bool y_f32, bool relu, const float* residual, const float* ln_x,
                           const uint16_t* ln_g, const uint16_t* ln_b, int kv_layer, int kv_b0, const float* st_in,
                           int st_parts, float* st_out, int* parts_out) {
  // the decode kernel takes at most 64 batch columns: larger batches whose epilogue stores
  // K/V (or whose operand is LayerNorm-fused) run as 64-column chunks (the cache is indexed
  // by the chunk-local sample, so its base moves with the chunk)
  if (Bg > 64 && (ln_x || kv_layer >= 0)) {
    for (int b0 = 0; b0 < Bg; b0 += 64) {
      const int nb = std::min(64, Bg - b0);
      const size_t ey = static_cast<size_t>(b0) * N_out * (y_f32 ? 4 : 2);
      linear_decode(W, N_out, Kd, X ? X + static_cast<size_t>(b0) * Kd : nullptr, nb, bias,
                    static_cast<char*>(Y) + ey, y_f32, relu, residual ? residual + static_cast<size_t>(b0) * N_out : nullptr,
                    ln_x ? ln_x + static_cast<size_t>(b0) * Kd : nullptr, ln_g, ln_b, kv_layer, b0);
    }
    return;
  }
  rlhf_gemm_decode_params p{};
  p.ln_x = ln_x;
  p.ln_g = ln_g;
  p.ln_b = ln_b;
  if (kv_layer >= 0) {
    const size_t kv_off = static_cast<size_t>(kv_b0) * kv_.H * kv_.Smax * kv_.hd;
    p.kcache = kv_.Kc(kv_layer) + kv_off;
    p.vcache = kv_.Vc(kv_layer) + kv_off;
    p.pos = pos_.as<int>();
    p.kv_d = N_out / 3;
    p.kv_hd = kv_.hd;
    p.kv_H = kv_.H;
    p.kv_Smax = kv_.Smax;
  }
  p.M = N_out; p.N = Bg; p.K = Kd;
  p.W = W; p.ldw = Kd;
  p.X = X; p.ldx = Kd;
  p.Y = Y; p.y_f32 = y_f32; p.ldy = N_out;
  p.bias = bias;
  p.relu = relu;
  p.residual = residual;
  const int tiles = (N_out + 127) / 128;
  const int kb = (Kd + 63) / 64;
  // batches above the decode kernel's N <= 64: the persistent GEMM, column-major out.  (Large
  // projections stay on the decode kernel: LLaMA-7B gate|up, 172 tiles, streams at 4.65 TB/s
  // there vs 2.86 TB/s through the persistent GEMM, tools/decode_gemm_bw_7b.py.)
  if (Bg > 64 && !ln_x && kv_layer < 0) {
    rlhf_gemm_params q{};
    q.M = N_out; q.N = Bg; q.K = Kd; q.batch = 1; q.batch_h = 1;
    q.A = W; q.lda = Kd;
    q.B = X; q.ldb = Kd;
    q.C = Y; q.c_f32 = y_f32; q.c_rs = 1; q.c_cs = N_out;
    q.alpha = 1.0f;
    q.bias = bias; q.bias_along_m = 1;
    q.relu = relu;
    q.residual = residual;
    gemm(q);
    return;
  }
  // K slices of one 128-row tile form a cluster, up to two CTAs per SM (the kernel then
  // uses a 4-stage ring)
  int split = 1;
  // >= 1 k-block per slice: short-K projections of small models (c2: K = 768) run more,
  // shorter slices (measured: c2 decode 128.4 -> 123.5 ms per PPO step against >= 2);
  // RLHF_DEC_MINKB overrides the minimum for timing experiments
  static const int minkb = [] { const char* e = getenv("RLHF_DEC_MINKB"); return e ? atoi(e) : 1; }();
  while (split < 8 && tiles * split * 2 <= 2 * 148 && kb / (split * 2) >= minkb) split *= 2;
  // very long K (OPT-1.3B FFN-down, K = 8192) on few tiles: a 16-CTA cluster per tile
  if (split == 8 && tiles * 16 <= 2 * 148 && kb / 16 >= 8) split = 16;
  // long K (>= 4096): two CTAs per SM pay off (LLaMA-7B O-proj 13.9 -> 12.5 us, FFN-down
  // 22.4 -> 20.4 us with 8 slices instead of 4)
  if (kb >= 64)
    while (split < 16 && tiles * split * 2 <= 2 * 148 && kb / (split * 2) >= 8) split *= 2;
  // few tiles (c2's O-proj / FFN-down: 6): one more doubling while every CTA still has an SM
  // of its own, even if some slices get no k-block (c2 decode step 432 -> 415 us, same-box A/B;
  // the idle slices push zero partials)
  if (split < 16 && tiles * split * 2 <= 148 && kb >= split) split *= 2;
  {  // RLHF_DEC_FORCE="N_out:K:splits,...": per-projection split override (timing experiments)
    static const char* force = getenv("RLHF_DEC_FORCE");
    for (const char* f = force; f && *f;) {
      int n = 0, k = 0, sp = 0;
      if (sscanf(f, "%d:%d:%d", &n, &k, &sp) == 3 && n == N_out && k == Kd) split = sp;
      f = strchr(f, ',');
      if (f) ++f;
    }
  }
  p.splits = split;
  p.pdl = pdl_;
  p.ln_stats_out = st_out;
  p.ln_stats_parts_out = parts_out;
  if (st_in) {
    // LayerNorm from the producer's statistics in the prologue, when every B tile of the
    // K-slice fits the ring; otherwise the LayerNorm kernel writes the operand X first
    const int max_kb = Bg <= 32 ? 8 : 6;
    if ((kb + split - 1) / split <= max_kb) {
      p.X = nullptr;
      p.ln_stats_in = st_in;
      p.ln_stats_parts = st_parts;
    } else {
      K(rlhf_layernorm(ln_x, ln_g, ln_b, const_cast<uint16_t*>(X), nullptr, nullptr, Bg, Kd, stream_), 1);
      p.ln_x = nullptr;
      p.ln_g = p.ln_b = nullptr;
    }
  }
  K(rlhf_gemm_decode(&p, stream_), 1);
}

void Engine::init_decoder(Decoder& m, const rlhf_arch& a, uint64_t seed, bool trainable, ncclComm_t dp_comm) {
  m.a = a;
  m.seed = seed;
  m.trainable = trainable;
  m.n = rlhf_param_total(&a);
  m.npad = m.shard = m.n;
  m.shard_off = 0;
  m.sharded = trainable && opt_.zero_stage == 1 && dp_comm;
  m.zero2 = trainable && opt_.zero_stage >= 2;
  m.zero3 = trainable && opt_.zero_stage == 3;
  if (m.zero2) {
    // buckets: embeddings | layer 0 .. L-1 | final norm + heads; each rank owns a
    // 64-aligned slice of every bucket (costmodel.hpp:48-50 ZeRO-2: 2 + 14/dp B/param)
    if (dp_comm) {
      NK(nccl().CommCount(dp_comm, &m.dp));
      NK(nccl().CommUserRank(dp_comm, &m.dp_rank));
    }
    m.layers_start = rlhf_tensor_offset(&a, RLHF_LAYER_FIRST, 0);
    m.layer_len = a.n_layers > 1 ? rlhf_tensor_offset(&a, RLHF_LAYER_FIRST, 1) - m.layers_start
                                 : rlhf_tensor_offset(&a, RLHF_T_LNF_G, 0) - m.layers_start;
    m.post_start = rlhf_tensor_offset(&a, RLHF_T_LNF_G, 0);
    auto add = [&](int64_t start, int64_t len) {
      GradBucket g;
      g.start = start;
      g.len = len;
      g.slice = ((len + m.dp - 1) / m.dp + 63) / 64 * 64;
      g.soff = m.buckets.empty() ? 0 : m.buckets.back().soff + m.buckets.back().slice;
      m.buckets.push_back(g);
    };
    add(0, m.layers_start);
    for (int l = 0; l < a.n_layers; ++l) add(m.layers_start + static_cast<int64_t>(l) * m.layer_len, m.layer_len);
    add(m.post_start, m.n - m.post_start);
    m.shard = m.buckets.back().soff + m.buckets.back().slice;
    m.work_len = m.buckets[1].slice * m.dp;  // a layer bucket padded to dp slices
  }
  if (m.sharded) {
    int dp = 1, r = 0;
    NK(nccl().CommCount(dp_comm, &dp));
    NK(nccl().CommUserRank(dp_comm, &r));
    m.shard = (m.n + dp - 1) / dp;
    m.shard = (m.shard + 63) / 64 * 64;  // 16-byte vectors in AdamW, aligned NCCL chunks
    m.npad = m.shard * dp;
    m.shard_off = m.shard * r;
  }
  std::vector<uint16_t> host(static_cast<size_t>(m.n), 0);
  struct Piece { int t, l; int64_t i0, i1; };
  std::vector<Piece> pieces;
  const int64_t chunk = 1 << 18;
  for (int t = 0; t < RLHF_T_COUNT; ++t) {
    const bool per_layer = t >= RLHF_LAYER_FIRST && t <= RLHF_LAYER_LAST;
    for (int l = 0; l < (per_layer ? a.n_layers : 1); ++l) {
      const int64_t ne = rlhf_tensor_numel(&a, t);
      for (int64_t i = 0; i < ne; i += chunk) pieces.push_back({t, l, i, std::min(ne, i + chunk)});
    }
  }
  const unsigned nth = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  std::vector<std::thread> th;
  for (unsigned w = 0; w < nth; ++w)
    th.emplace_back([&, w] {
      for (size_t i = w; i < pieces.size(); i += nth) {
        const Piece& pc = pieces[i];
        rlhf_init_tensor_range(&a, seed, pc.t, pc.l, pc.i0, pc.i1,
                               host.data() + rlhf_tensor_offset(&a, pc.t, pc.l) + pc.i0);
      }
    });
  for (auto& t : th) t.join();
  if (m.zero3) {  // only the embedding / head buckets whole; the layers as this rank's slices
    const GradBucket &pre = m.buckets.front(), &post = m.buckets.back();
    m.wpre.alloc(static_cast<size_t>(pre.len) * 2);
    m.wpost.alloc(static_cast<size_t>(post.len) * 2);
    for (DevBuf& b : m.wwork) b.alloc(static_cast<size_t>(m.work_len) * 2);
    std::vector<uint16_t> sl(static_cast<size_t>(m.shard), 0);
    for (const GradBucket& g : m.buckets)
      for (int64_t i = 0; i < g.slice; ++i) {
        const int64_t e = static_cast<int64_t>(m.dp_rank) * g.slice + i;
        if (e < g.len) sl[g.soff + i] = host[g.start + e];
      }
    m.wshard.alloc(sl.size() * 2);
    bool ok = cudaMemcpy(m.wpre.p, host.data(), pre.len * 2, cudaMemcpyHostToDevice) == cudaSuccess;
    ok &= cudaMemcpy(m.wpost.p, host.data() + post.start, post.len * 2, cudaMemcpyHostToDevice) == cudaSuccess;
    ok &= cudaMemcpy(m.wshard.p, sl.data(), sl.size() * 2, cudaMemcpyHostToDevice) == cudaSuccess;
    if (!ok) throw DeviceError("weight upload failed");
    for (auto& e : m.wgather_done)
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) throw DeviceError("event create failed");
  } else {
    m.w.alloc(static_cast<size_t>(m.npad) * 2);
    if (cudaMemcpy(m.w.p, host.data(), host.size() * 2, cudaMemcpyHostToDevice) != cudaSuccess)
      throw DeviceError("weight upload failed");
  }
  if (trainable) {
    std::vector<float> f(static_cast<size_t>(m.shard), 0.0f);  // this rank's slice of the fp32 master
    if (m.zero2) {
      for (const GradBucket& g : m.buckets)
        for (int64_t i = 0; i < g.slice; ++i) {
          const int64_t e = static_cast<int64_t>(m.dp_rank) * g.slice + i;
          if (e < g.len) f[g.soff + i] = rlhf_bf16_to_f32(host[g.start + e]);
        }
    } else {
      for (int64_t i = 0; i < m.shard && m.shard_off + i < m.n; ++i) f[i] = rlhf_bf16_to_f32(host[m.shard_off + i]);
    }
    m.master.alloc(f.size() * 4);
    cudaMemcpy(m.master.p, f.data(), f.size() * 4, cudaMemcpyHostToDevice);
    m.m.alloc(f.size() * 4);
    m.v.alloc(f.size() * 4);
    if (m.zero2) {
      const GradBucket &pre = m.buckets.front(), &post = m.buckets.back();
      m.gpre.alloc(static_cast<size_t>(pre.slice * m.dp) * 4);
      m.gpost.alloc(static_cast<size_t>(post.slice * m.dp) * 4);
      for (DevBuf& b : m.gwork) b.alloc(static_cast<size_t>(m.work_len) * 4);
      m.gshard.alloc(static_cast<size_t>(m.shard) * 4);
      int64_t smax = 0;
      for (const GradBucket& g : m.buckets) smax = std::max(smax, g.slice);
      m.rs_tmp.alloc(static_cast<size_t>(smax) * 4);
      if (!m.zero3) m.wshard.alloc(static_cast<size_t>(m.shard) * 2);
      m.ag_stage.alloc(static_cast<size_t>(smax * m.dp) * 2);
      for (auto& e : m.rs_done) {
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) throw DeviceError("event create failed");
        cudaEventRecord(e, stream_);  // both working buckets start free
      }
    } else {
      m.grad.alloc(static_cast<size_t>(m.npad) * 4);
    }
  }
  if (m.llama()) {
    const int hd = a.d_model / a.n_heads, half = hd / 2;
    std::vector<float> tab(static_cast<size_t>(a.max_pos) * half * 2);
    for (int p = 0; p < a.max_pos; ++p)
      for (int i = 0; i < half; ++i)
        rlhf_rope_cos_sin(p, i, hd, &tab[(static_cast<size_t>(p) * half + i) * 2], &tab[(static_cast<size_t>(p) * half + i) * 2 + 1]);
    m.rope.alloc(tab.size() * 4);
    if (cudaMemcpy(m.rope.p, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess)
      throw DeviceError("rotary table upload failed");
  }
}

// Pre-norm of the residual stream: LayerNorm (OPT) or RMSNorm (LLaMA; tensor `g`'s
// beta is absent).  mean is only written for LayerNorm.
void Engine::norm(const Decoder& m, const float* x, int g, int l, uint16_t* y, float* mean, float* rstd, int rows) {
  const int d = m.a.d_model;
  if (m.llama()) K(rlhf_rmsnorm(x, m.T(g, l), y, rstd, rows, d, stream_), 1);
  else K(rlhf_layernorm(x, m.T(g, l), m.T(g + 1, l), y, mean, rstd, rows, d, stream_), 1);
}

void Engine::norm_bwd(Decoder& m, const float* dy, const float* x, const float* mean, const float* rstd, int g, int l,
                      int rows) {
  const int d = m.a.d_model;
  if (m.llama())
    K(rlhf_rmsnorm_bwd(dy, x, rstd, m.T(g, l), arp_->dres, m.G(g, l), rows, d, arp_->ws, arp_->ws_floats, stream_), 2);
  else
    K(rlhf_layernorm_bwd(dy, x, mean, rstd, m.T(g, l), arp_->dres, m.G(g, l), m.G(g + 1, l), rows, d, arp_->ws,
                         arp_->ws_floats, stream_), 2);
}

// Teacher-forced forward over positions [0, T) of B sequences (row r = b*T + i).
// save: keep every layer's activations for backward (TrainFB); kv: store K/V
// (Generation prefill).  Result: final-LN hidden states in arp_->hf (bf16).
void Engine::forward(const Decoder& m, const int32_t* tokens, int B, int tok_stride, int T, bool save, KVCache* kv) {
  const rlhf_arch& a = m.a;
  const int d = a.d_model, H = a.n_heads, hd = d / H, ff = a.d_ff, L = a.n_layers;
  const int rows = B * T;
  const int64_t Td = static_cast<int64_t>(rows) * d;
  // saved layers are strided by the training micro-batch's rows (Arena::Ts, Zs)
  if (save && rows > arp_->Ts) throw ConfigError("saved forward exceeds the training micro-batch capacity");
  auto X = [&](int k) { return arp_->xres + (save ? static_cast<int64_t>(k) * arp_->Ts * arp_->d : 0); };
  auto MEAN = [&](int k) { return save ? arp_->mean + static_cast<int64_t>(k) * arp_->Ts : nullptr; };
  auto RSTD = [&](int k) { return save ? arp_->rstd + static_cast<int64_t>(k) * arp_->Ts : nullptr; };
  auto slot = [&](uint16_t* base, int64_t per, int l) { return base + (save ? static_cast<int64_t>(l) * per : 0); };
  (void)Td;
  K(rlhf_embed(tokens, tok_stride, B, T, 0, nullptr, m.T(RLHF_T_TOK_EMB), m.T(RLHF_T_POS_EMB), d, X(0), stream_), 1);
  for (int l = 0; l < L; ++l) {
    if (m.zero3) zero3_fetch(m, l, l + 1 < L ? l + 1 : -1);
    uint16_t* h1 = slot(arp_->h1, arp_->Ts * arp_->d, l);
    uint16_t* qkv = slot(arp_->qkv, arp_->Ts * 3 * arp_->d, l);
    uint16_t* P = slot(arp_->P, arp_->Zs * arp_->S * arp_->S, l);
    uint16_t* o = slot(arp_->o, arp_->Ts * arp_->d, l);
    uint16_t* h2 = slot(arp_->h2, arp_->Ts * arp_->d, l);
    uint16_t* f = slot(arp_->f, arp_->Ts * arp_->ff, l);
    float* xin = X(2 * l);
    float* xmid = X(2 * l + 1);
    float* xout = X(2 * l + 2);
    norm(m, xin, RLHF_T_LN1_G, l, h1, MEAN(2 * l), RSTD(2 * l), rows);
    linear(h1, rows, d, m.T(RLHF_T_WQKV, l), 3 * d, m.T(RLHF_T_BQKV, l), qkv, false, false, nullptr);
    if (m.llama())  // rotary q, k in place (+ the K/V-cache store of the rotated k)
      K(rlhf_rope_qkv(qkv, B, T, 0, nullptr, H, hd, m.rope.as<float>(), 0, kv ? kv->Kc(l) : nullptr,
                      kv ? kv->Vc(l) : nullptr, kv ? kv->Smax : 0, stream_), 1);
    else if (kv)
      K(rlhf_kv_store(qkv, B, T, 0, nullptr, H, hd, kv->Smax, kv->Kc(l), kv->Vc(l), stream_), 1);
    attention_fwd(qkv, P, o, B, T, H, hd, save);
    linear(o, rows, d, m.T(RLHF_T_WO, l), d, m.T(RLHF_T_BO, l), xmid, true, false, xin);
    norm(m, xmid, RLHF_T_LN2_G, l, h2, MEAN(2 * l + 1), RSTD(2 * l + 1), rows);
    if (m.llama()) {  // f = [gate | up] (kept for backward), act = silu(gate) * up
      linear(h2, rows, d, m.T(RLHF_T_W1, l), 2 * ff, nullptr, f, false, false, nullptr);
      K(rlhf_swiglu(f, arp_->act, rows, ff, stream_), 1);
      linear(arp_->act, rows, ff, m.T(RLHF_T_W2, l), d, nullptr, xout, true, false, xmid);
    } else {
      linear(h2, rows, d, m.T(RLHF_T_W1, l), ff, m.T(RLHF_T_B1, l), f, false, true, nullptr);
      linear(f, rows, ff, m.T(RLHF_T_W2, l), d, m.T(RLHF_T_B2, l), xout, true, false, xmid);
    }
  }
  norm(m, X(2 * L), RLHF_T_LNF_G, 0, arp_->hf, MEAN(2 * L), RSTD(2 * L), rows);
}

// S = softmax(Q K^T / sqrt(hd)) (causal), O = P V — batched over (b, h) straight
// out of the packed qkv rows; P kept (bf16) for backward.
void Engine::attention_fwd(const uint16_t* qkv, uint16_t* P, uint16_t* o, int B, int T, int H, int hd, bool keep_p) {
  const int d = H * hd;
  const int64_t TT = static_cast<int64_t>(T) * T;
  static const bool unfused = getenv("RLHF_ATTN_UNFUSED") != nullptr;  // A/B switch for timing
  if (!unfused && hd == 64 && T % 128 == 0 && T <= 512) {
    // one kernel: scores in TMEM, softmax, P.V in TMEM; P kept only for backward
    K(rlhf_attn_fwd_fused(qkv, B, H, hd, T, 1.0f / std::sqrt(static_cast<float>(hd)), keep_p ? P : nullptr, o, stream_),
      1);
    return;
  }
  rlhf_gemm_params s{};
  s.M = T; s.N = T; s.K = hd; s.batch = B * H; s.batch_h = H;
  s.A = qkv; s.lda = 3 * d; s.a_stride_h = hd; s.a_stride_b = static_cast<int64_t>(T) * 3 * d;
  s.B = qkv + d; s.ldb = 3 * d; s.b_stride_h = hd; s.b_stride_b = static_cast<int64_t>(T) * 3 * d;
  s.C = arp_->scores; s.c_f32 = 1; s.c_rs = T; s.c_cs = 1; s.c_stride_h = TT; s.c_stride_b = H * TT;
  s.alpha = 1.0f / std::sqrt(static_cast<float>(hd));
  s.causal = 1;
  gemm(s);
  K(rlhf_attn_softmax(arp_->scores, P, B * H, T, stream_), 1);
  rlhf_gemm_params pv{};
  pv.M = T; pv.N = hd; pv.K = T; pv.batch = B * H; pv.batch_h = H;
  pv.A = P; pv.lda = T; pv.a_stride_h = TT; pv.a_stride_b = H * TT;
  pv.B = qkv + 2 * d; pv.b_mn_major = 1; pv.ldb = 3 * d; pv.b_stride_h = hd; pv.b_stride_b = static_cast<int64_t>(T) * 3 * d;
  pv.C = o; pv.c_f32 = 0; pv.c_rs = d; pv.c_cs = 1; pv.c_stride_h = hd; pv.c_stride_b = static_cast<int64_t>(T) * d;
  pv.alpha = 1.0f;
  pv.causal = 2;
  gemm(pv);
}

void Engine::attention_bwd(const uint16_t* qkv, const uint16_t* P, const uint16_t* dov, uint16_t* dqkv, int B, int T, int H,
                           int hd) {
  const int d = H * hd;
  const int64_t TT = static_cast<int64_t>(T) * T;
  const int64_t qb = static_cast<int64_t>(T) * 3 * d, ob = static_cast<int64_t>(T) * d;
  static const bool unfused = getenv("RLHF_ATTN_BWD_UNFUSED") != nullptr;  // A/B switch for timing
  if (!unfused && !getenv("RLHF_ATTN_UNFUSED") && hd == 64 && T % 128 == 0 && T <= 512) {
    // dP = dO V^T, D and dS in one kernel: fp32 dP never leaves TMEM
    K(rlhf_attn_bwd_ds_fused(dov, qkv, P, arp_->dS, B, H, hd, T, 1.0f / std::sqrt(static_cast<float>(hd)), stream_), 1);
  } else {
    // dP = dO V^T (fp32, causal tiles)
    rlhf_gemm_params dp{};
    dp.M = T; dp.N = T; dp.K = hd; dp.batch = B * H; dp.batch_h = H;
    dp.A = dov; dp.lda = d; dp.a_stride_h = hd; dp.a_stride_b = ob;
    dp.B = qkv + 2 * d; dp.ldb = 3 * d; dp.b_stride_h = hd; dp.b_stride_b = qb;
    dp.C = arp_->scores; dp.c_f32 = 1; dp.c_rs = T; dp.c_cs = 1; dp.c_stride_h = TT; dp.c_stride_b = H * TT;
    dp.alpha = 1.0f; dp.causal = 1;
    gemm(dp);
    K(rlhf_attn_softmax_bwd(P, arp_->scores, arp_->dS, B * H, T, 1.0f / std::sqrt(static_cast<float>(hd)), stream_), 1);
  }
  // dQ = dS K
  rlhf_gemm_params dq{};
  dq.M = T; dq.N = hd; dq.K = T; dq.batch = B * H; dq.batch_h = H;
  dq.A = arp_->dS; dq.lda = T; dq.a_stride_h = TT; dq.a_stride_b = H * TT;
  dq.B = qkv + d; dq.b_mn_major = 1; dq.ldb = 3 * d; dq.b_stride_h = hd; dq.b_stride_b = qb;
  dq.C = dqkv; dq.c_rs = 3 * d; dq.c_cs = 1; dq.c_stride_h = hd; dq.c_stride_b = qb;
  dq.alpha = 1.0f; dq.causal = 2;
  gemm(dq);
  // dK = dS^T Q
  rlhf_gemm_params dk{};
  dk.M = T; dk.N = hd; dk.K = T; dk.batch = B * H; dk.batch_h = H;
  dk.A = arp_->dS; dk.a_mn_major = 1; dk.lda = T; dk.a_stride_h = TT; dk.a_stride_b = H * TT;
  dk.B = qkv; dk.b_mn_major = 1; dk.ldb = 3 * d; dk.b_stride_h = hd; dk.b_stride_b = qb;
  dk.C = dqkv + d; dk.c_rs = 3 * d; dk.c_cs = 1; dk.c_stride_h = hd; dk.c_stride_b = qb;
  dk.alpha = 1.0f; dk.causal = 3;
  gemm(dk);
  // dV = P^T dO
  rlhf_gemm_params dv{};
  dv.M = T; dv.N = hd; dv.K = T; dv.batch = B * H; dv.batch_h = H;
  dv.A = P; dv.a_mn_major = 1; dv.lda = T; dv.a_stride_h = TT; dv.a_stride_b = H * TT;
  dv.B = dov; dv.b_mn_major = 1; dv.ldb = d; dv.b_stride_h = hd; dv.b_stride_b = ob;
  dv.C = dqkv + 2 * d; dv.c_rs = 3 * d; dv.c_cs = 1; dv.c_stride_h = hd; dv.c_stride_b = qb;
  dv.alpha = 1.0f; dv.causal = 3;
  gemm(dv);
}

// dL/dhf is in arp_->dhf (fp32 [B*S, d]); accumulates every parameter gradient of m.
void Engine::backward(Decoder& m, const int32_t* tokens, int B, int S) {
  const rlhf_arch& a = m.a;
  const int d = a.d_model, H = a.n_heads, hd = d / H, ff = a.d_ff, L = a.n_layers;
  const int rows = B * S;
  auto X = [&](int k) { return arp_->xres + static_cast<int64_t>(k) * arp_->Ts * arp_->d; };
  auto MEAN = [&](int k) { return arp_->mean + static_cast<int64_t>(k) * arp_->Ts; };
  auto RSTD = [&](int k) { return arp_->rstd + static_cast<int64_t>(k) * arp_->Ts; };
  cudaMemsetAsync(arp_->dres, 0, static_cast<size_t>(rows) * d * 4, stream_);
  norm_bwd(m, arp_->dhf, X(2 * L), MEAN(2 * L), RSTD(2 * L), RLHF_T_LNF_G, 0, rows);
  auto colsum = [&](const uint16_t* Gm, int N, float* db) {  // bias gradient (absent in LLaMA)
    if (db) K(rlhf_colsum_bf16(Gm, rows, N, db, arp_->ws, stream_), 2);
  };
  // dW[N_out, K_in] += dY[T, N_out]^T X[T, K_in]
  auto wgrad = [&](const uint16_t* dY, int N_out, const uint16_t* Xin, int K_in, float* dW) {
    rlhf_gemm_params p{};
    p.M = N_out; p.N = K_in; p.K = rows; p.batch = 1; p.batch_h = 1;
    p.A = dY; p.a_mn_major = 1; p.lda = N_out;
    p.B = Xin; p.b_mn_major = 1; p.ldb = K_in;
    p.C = dW; p.c_f32 = 1; p.c_rs = K_in; p.c_cs = 1;
    p.alpha = 1.0f; p.accumulate = 1;
    // very few output tiles (O-projection: 18), long K (tokens): deterministic split-K
    // fills the SMs.  Larger weight gradients stay unsplit: they are L2-operand-bandwidth
    // bound and the partial round trip costs more than the idle SMs (tools/gemm_bench.py).
    const int bn = rlhf_gemm_block_n(&p);
    const int tiles = ((N_out + 127) / 128) * ((K_in + bn - 1) / bn);
    int split = 1;
    if (tiles * 4 <= 148)
      while (split < 8 && tiles * split * 2 <= 148 && rows / 64 / (split * 2) >= 8) split *= 2;
    // default: 128 x 256 tiles (87 FLOP per operand byte against 64 for 128 x 128) with
    // deterministic split-K filling the SMs (c2 TrainFB 27.3 -> 26.0 ms); RLHF_WGRAD=0: the
    // previous 128 x 128 unsplit tiles
    static const int wmode = [] { const char* e = getenv("RLHF_WGRAD"); return e ? atoi(e) : 1; }();
    if (wmode == 1) {
      p.block_n = 256;
      const int t2 = ((N_out + 127) / 128) * ((K_in + 255) / 256);
      split = 1;
      while (split < 8 && t2 * split * 2 <= 148 && rows / 64 / (split * 2) >= 8) split *= 2;
    }
    p.split_k = split;
    gemm(p);
  };
  // dX[T, K_in] = dY[T, N_out] W[N_out, K_in]
  auto dgrad = [&](const uint16_t* dY, int N_out, const uint16_t* W, int K_in, void* dX, bool f32, const uint16_t* mask) {
    rlhf_gemm_params p{};
    p.M = rows; p.N = K_in; p.K = N_out; p.batch = 1; p.batch_h = 1;
    p.A = dY; p.lda = N_out;
    p.B = W; p.b_mn_major = 1; p.ldb = K_in;
    p.C = dX; p.c_f32 = f32; p.c_rs = K_in; p.c_cs = 1;
    p.alpha = 1.0f;
    p.aux = mask; p.aux_rs = K_in; p.aux_cs = 1;
    gemm(p);
  };
  for (int l = L - 1; l >= 0; --l) {
    if (m.zero3) zero3_fetch(m, l, l > 0 ? l - 1 : -1);
    if (m.zero2) zero2_layer_begin(m, l);
    const int64_t Tn = arp_->Ts;
    const uint16_t* h1 = arp_->h1 + l * Tn * arp_->d;
    const uint16_t* qkv = arp_->qkv + l * Tn * 3 * arp_->d;
    const uint16_t* P = arp_->P + l * arp_->Zs * arp_->S * arp_->S;
    const uint16_t* o = arp_->o + l * Tn * arp_->d;
    const uint16_t* h2 = arp_->h2 + l * Tn * arp_->d;
    const uint16_t* f = arp_->f + l * Tn * arp_->ff;
    // FFN: x_out = x_mid + relu(h2 W1^T + b1) W2^T + b2
    K(rlhf_round_bf16(arp_->dres, arp_->g, static_cast<int64_t>(rows) * d, stream_), 1);
    colsum(arp_->g, d, m.G(RLHF_T_B2, l));
    if (m.llama()) {
      // SwiGLU: act recomputed from the saved [gate | up] (not kept per layer), then
      // dact (bf16, into the same buffer) -> [dgate | dup]
      K(rlhf_swiglu(f, arp_->act, rows, ff, stream_), 1);
      wgrad(arp_->g, d, arp_->act, ff, m.G(RLHF_T_W2, l));
      dgrad(arp_->g, d, m.T(RLHF_T_W2, l), ff, arp_->act, false, nullptr);
      K(rlhf_swiglu_bwd(f, arp_->act, arp_->dpre, rows, ff, stream_), 1);
      wgrad(arp_->dpre, 2 * ff, h2, d, m.G(RLHF_T_W1, l));
      dgrad(arp_->dpre, 2 * ff, m.T(RLHF_T_W1, l), d, arp_->dh, true, nullptr);
    } else {
      wgrad(arp_->g, d, f, ff, m.G(RLHF_T_W2, l));
      dgrad(arp_->g, d, m.T(RLHF_T_W2, l), ff, arp_->dpre, false, f);
      colsum(arp_->dpre, ff, m.G(RLHF_T_B1, l));
      wgrad(arp_->dpre, ff, h2, d, m.G(RLHF_T_W1, l));
      dgrad(arp_->dpre, ff, m.T(RLHF_T_W1, l), d, arp_->dh, true, nullptr);
    }
    norm_bwd(m, arp_->dh, X(2 * l + 1), MEAN(2 * l + 1), RSTD(2 * l + 1), RLHF_T_LN2_G, l, rows);
    // attention block: x_mid = x_in + attn(h1) Wo^T + bo
    K(rlhf_round_bf16(arp_->dres, arp_->g, static_cast<int64_t>(rows) * d, stream_), 1);
    colsum(arp_->g, d, m.G(RLHF_T_BO, l));
    wgrad(arp_->g, d, o, d, m.G(RLHF_T_WO, l));
    dgrad(arp_->g, d, m.T(RLHF_T_WO, l), d, arp_->dov, false, nullptr);
    attention_bwd(qkv, P, arp_->dov, arp_->dqkv, B, S, H, hd);
    if (m.llama())  // dq, dk through the rotation's transpose (the saved q, k are rotated)
      K(rlhf_rope_qkv(arp_->dqkv, B, S, 0, nullptr, H, hd, m.rope.as<float>(), 1, nullptr, nullptr, 0, stream_), 1);
    colsum(arp_->dqkv, 3 * d, m.G(RLHF_T_BQKV, l));
    wgrad(arp_->dqkv, 3 * d, h1, d, m.G(RLHF_T_WQKV, l));
    dgrad(arp_->dqkv, 3 * d, m.T(RLHF_T_WQKV, l), d, arp_->dh, true, nullptr);
    norm_bwd(m, arp_->dh, X(2 * l), MEAN(2 * l), RSTD(2 * l), RLHF_T_LN1_G, l, rows);
    if (m.zero2) zero2_layer_end(m, l);
  }
  K(rlhf_embed_bwd(tokens, S, B, S, arp_->dres, d, m.G(RLHF_T_TOK_EMB), m.G(RLHF_T_POS_EMB), stream_), 1);
}

// Per-token logprobs of the response tokens under m (tied LM head); logits and
// lse stay in the arena for the backward when keep_logits.
void Engine::lm_logprobs(const Decoder& m, const int32_t* tokens, int B, float* logp, bool keep_logits) {
  const int d = m.a.d_model, V = m.a.vocab;
  K(rlhf_gather_rows(arp_->hf, arp_->hf_resp, B, S_, R_, P_ - 1, d, 2, stream_), 1);
  if (!keep_logits) {
    // no backward: the LM-head GEMM epilogue reduces each row's logits to per-tile
    // (max, sum exp) partials + the target logit; the logits never reach HBM
    rlhf_gemm_params p{};
    p.M = B * R_; p.N = V; p.K = d; p.batch = 1; p.batch_h = 1;
    p.A = arp_->hf_resp; p.lda = d;
    p.B = m.T(m.head_id()); p.ldb = d;
    p.C = arp_->logits; p.c_f32 = 1; p.c_rs = V; p.c_cs = 1;
    p.alpha = 1.0f;
    p.lse_part = arp_->logits;  // (max, sum) partials: rows x tiles x 2 float2, far below the logits' size
    p.lse_tgt = arp_->lse;
    p.lse_tokens = tokens; p.lse_S = S_; p.lse_P = P_; p.lse_R = R_;
    const int st = rlhf_gemm(&p, stream_);
    if (st == 0) {
      ++launches_;
      K(rlhf_lse_merge(arp_->logits, arp_->lse, B * R_, 2 * ((V + 255) / 256), logp, stream_), 1);
      return;
    }
    if (st != 2) kcheck(st, "rlhf_gemm (LM head, log-sum-exp epilogue)");
  }
  linear(arp_->hf_resp, B * R_, d, m.T(m.head_id()), V, nullptr, arp_->logits, true, false, nullptr);
  K(rlhf_logprob(arp_->logits, B * R_, V, tokens, S_, P_, R_, logp, arp_->lse, stream_), 1);
}

// One decode step at position *pos: embed -> L x (LN, qkv, KV store, attention,
// o-proj, LN, FFN) -> final LN -> LM head -> greedy argmax -> pos += 1.
void Engine::decode_step(const Decoder& m, int B) {
  const rlhf_arch& a = m.a;
  const int d = a.d_model, H = a.n_heads, hd = d / H, ff = a.d_ff, V = a.vocab;
  int* pos = pos_.as<int>();
  float* x = dec_x_.as<float>();
  uint16_t* h = dec_h_.as<uint16_t>();
  uint16_t* qkv = dec_qkv_.as<uint16_t>();
  uint16_t* o = dec_o_.as<uint16_t>();
  uint16_t* f = dec_f_.as<uint16_t>();
  const int32_t* tok = gen_tok_.as<int32_t>();
  // RLHF_DECODE_SKIP (debug timing only, results become wrong): bit 0 LN, 1 attention,
  // 2 qkv GEMM, 3 o-proj, 4 FFN GEMMs, 5 LM head + argmax
  static const int skip = [] { const char* e = getenv("RLHF_DECODE_SKIP"); return e ? atoi(e) : 0; }();
  // next-attention K/V pulled into L2 by each decode attention: measured SLOWER (c2 decode step 492 -> 512 us,
  // c3 1547 -> 1664 us), so off unless RLHF_DEC_KV_PREFETCH=1
  static const bool pf_kv = [] { const char* e = getenv("RLHF_DEC_KV_PREFETCH"); return e && atoi(e) != 0; }();
  if (m.llama()) {
    // LLaMA: RMSNorm, [QKV GEMM], rotary q/k + KV-cache store, attention, [O-proj + residual],
    // RMSNorm, [gate|up GEMM], SwiGLU, [down + residual]; final RMSNorm, untied head
    uint16_t* act = dec_act_.as<uint16_t>();
    if (fuse_merge_)
      K(rlhf_argmax_embed_rmsnorm(dec_top2_.as<float>(), (V + 127) / 128, graph_for_pred_ ? pred_.as<int32_t>() : gen_tok_.as<int32_t>(),
                                  margin_.as<float>(), tok, S_, B, pos, m.T(RLHF_T_TOK_EMB), d, x, m.T(RLHF_T_LN1_G, 0), h,
                                  stream_),
        1);
    else
      K(rlhf_embed_rmsnorm(tok, S_, B, pos, m.T(RLHF_T_TOK_EMB), d, x, m.T(RLHF_T_LN1_G, 0), h, stream_), 1);
    for (int l = 0; l < a.n_layers; ++l) {
      if (l > 0) K(rlhf_rmsnorm(x, m.T(RLHF_T_LN1_G, l), h, nullptr, B, d, stream_), 1);
      linear_decode(m.T(RLHF_T_WQKV, l), 3 * d, d, h, B, nullptr, qkv, false, false, nullptr);
      K(rlhf_rope_qkv(qkv, B, 1, 0, pos, H, hd, m.rope.as<float>(), 0, kv_.Kc(l), kv_.Vc(l), kv_.Smax, stream_), 1);
      K(rlhf_attn_decode_prefetch(qkv, B, H, hd, kv_.Smax, kv_.Kc(l), kv_.Vc(l), pos, o,
                                  pf_kv ? kv_.Kc((l + 1) % a.n_layers) : nullptr,
                                  pf_kv ? kv_.Vc((l + 1) % a.n_layers) : nullptr, stream_), 1);
      linear_decode(m.T(RLHF_T_WO, l), d, d, o, B, nullptr, x, true, false, x);
      K(rlhf_rmsnorm(x, m.T(RLHF_T_LN2_G, l), h, nullptr, B, d, stream_), 1);
      linear_decode(m.T(RLHF_T_W1, l), 2 * ff, d, h, B, nullptr, f, false, false, nullptr);
      K(rlhf_swiglu(f, act, B, ff, stream_), 1);
      linear_decode(m.T(RLHF_T_W2, l), d, ff, act, B, nullptr, x, true, false, x);
    }
    K(rlhf_rmsnorm(x, m.T(RLHF_T_LNF_G), dec_hf_.as<uint16_t>(), nullptr, B, d, stream_), 1);
    lm_head_argmax(m, dec_hf_.as<uint16_t>(), B, graph_for_pred_ ? pred_.as<int32_t>() : gen_tok_.as<int32_t>(),
                   !fuse_merge_);
    return;
  }
  // fuse_merge_: the previous LM head's greedy merge (token, margin, *pos += 1) runs inside
  // this entry kernel -- one launch, one PDL link fewer per step
  if (fuse_merge_)
    K(rlhf_argmax_embed_ln(dec_top2_.as<float>(), (V + 127) / 128, graph_for_pred_ ? pred_.as<int32_t>() : gen_tok_.as<int32_t>(),
                           margin_.as<float>(), tok, S_, B, pos, m.T(RLHF_T_TOK_EMB), m.T(RLHF_T_POS_EMB), d, x,
                           m.T(RLHF_T_LN1_G, 0), m.T(RLHF_T_LN1_B, 0), h, stream_),
      1);
  else
    K(rlhf_embed_ln(tok, S_, B, pos, m.T(RLHF_T_TOK_EMB), m.T(RLHF_T_POS_EMB), d, x, m.T(RLHF_T_LN1_G, 0),
                    m.T(RLHF_T_LN1_B, 0), h, stream_),
      1);
  // per layer 7 launches: LN1 (layer 0: fused with the embedding), [QKV GEMM + KV-cache
  // store], attention, [O-proj + residual], LN2, [FFN-up + ReLU], [FFN-down + residual];
  // then final LN, [LM head + per-tile top-2], [merge -> token, *pos += 1]
  // RLHF_DEC_LN_STATS=1: LayerNorm statistics carried between the decode GEMMs instead of
  // LayerNorm kernels -- the O-proj / FFN-down epilogues write per-CTA (sum, sum sq) partials
  // of the residual rows they produce, the next GEMM (FFN-up / QKV of the next layer)
  // normalises its K-slice in its prologue: 23 fewer launches per c2 step, parity-green, but
  // measured SLOWER (c2 decode step 498 -> 716 us, c3 1558 -> 2567 us), so off
  static const bool ln_stats_env = [] { const char* e = getenv("RLHF_DEC_LN_STATS"); return e && atoi(e) != 0; }();
  const bool fs = ln_stats_env && B <= 64 && d % 64 == 0 && d <= 2048;
  float* st_a = dec_st_[0].as<float>();
  float* st_b = dec_st_[1].as<float>();
  int parts_a = 0, parts_b = 0;
  for (int l = 0; l < a.n_layers; ++l) {
    const bool fs1 = fs && l > 0;  // layer 0's LN1 ran in rlhf_embed_ln
    if (l > 0 && !(skip & 1) && !fs1)
      K(rlhf_layernorm(x, m.T(RLHF_T_LN1_G, l), m.T(RLHF_T_LN1_B, l), h, nullptr, nullptr, B, d, stream_), 1);
    if (!(skip & 4))
      linear_decode(m.T(RLHF_T_WQKV, l), 3 * d, d, h, B, m.T(RLHF_T_BQKV, l), qkv, false, false, nullptr,
                    fs1 ? x : nullptr, fs1 ? m.T(RLHF_T_LN1_G, l) : nullptr, fs1 ? m.T(RLHF_T_LN1_B, l) : nullptr, l, 0,
                    fs1 ? st_b : nullptr, parts_b);
    if (!(skip & 2))
      K(rlhf_attn_decode_prefetch(qkv, B, H, hd, kv_.Smax, kv_.Kc(l), kv_.Vc(l), pos, o,
                                  pf_kv ? kv_.Kc((l + 1) % a.n_layers) : nullptr,
                                  pf_kv ? kv_.Vc((l + 1) % a.n_layers) : nullptr, stream_), 1);
    if (!(skip & 8))
      linear_decode(m.T(RLHF_T_WO, l), d, d, o, B, m.T(RLHF_T_BO, l), x, true, false, x, nullptr, nullptr, nullptr, -1, 0,
                    nullptr, 0, fs ? st_a : nullptr, &parts_a);
    if (!(skip & 1) && !fs) K(rlhf_layernorm(x, m.T(RLHF_T_LN2_G, l), m.T(RLHF_T_LN2_B, l), h, nullptr, nullptr, B, d, stream_), 1);
    if (!(skip & 16)) {
      linear_decode(m.T(RLHF_T_W1, l), ff, d, h, B, m.T(RLHF_T_B1, l), f, false, true, nullptr, fs ? x : nullptr,
                    fs ? m.T(RLHF_T_LN2_G, l) : nullptr, fs ? m.T(RLHF_T_LN2_B, l) : nullptr, -1, 0,
                    fs ? st_a : nullptr, parts_a);
      const bool prod = fs && l + 1 < a.n_layers;
      linear_decode(m.T(RLHF_T_W2, l), d, ff, f, B, m.T(RLHF_T_B2, l), x, true, false, x, nullptr, nullptr, nullptr, -1, 0,
                    nullptr, 0, prod ? st_b : nullptr, &parts_b);
    }
  }
  if (skip & 32) {
    K(rlhf_add_int(pos, 1, stream_), 1);
    return;
  }
  K(rlhf_layernorm(x, m.T(RLHF_T_LNF_G), m.T(RLHF_T_LNF_B), dec_hf_.as<uint16_t>(), nullptr, nullptr, B, d, stream_), 1);
  int32_t* dst = graph_for_pred_ ? pred_.as<int32_t>() : gen_tok_.as<int32_t>();
  lm_head_argmax(m, dec_hf_.as<uint16_t>(), B, dst, !fuse_merge_);  // the merge also advances *pos
}

// Tied LM head of the final hidden rows hf [B, d] fused with the greedy sampler: the
// swap-AB GEMM keeps only each 128-token tile's top-2 per sample (logits never stored),
// then one warp per sample merges the tiles -> dst[b*S + *pos + 1] and the margin.
void Engine::lm_head_argmax(const Decoder& m, const uint16_t* hf, int B, int32_t* dst, bool merge) {
  const int d = m.a.d_model, V = m.a.vocab;
  rlhf_gemm_params q{};
  q.M = V; q.N = B; q.K = d; q.batch = 1; q.batch_h = 1;
  q.A = m.T(m.head_id()); q.lda = d;
  q.B = hf; q.ldb = d;
  q.C = dec_logits_.p; q.c_f32 = 1; q.c_rs = 1; q.c_cs = V;
  q.alpha = 1.0f;
  q.top2 = dec_top2_.as<float>();
  gemm(q);
  if (merge)
    K(rlhf_argmax_tiles(dec_top2_.as<float>(), (V + 127) / 128, B, dst, S_, pos_.as<int>(), margin_.as<float>(), 1,
                        stream_),
      1);
}

// Greedy generation of R tokens for the B prompts already in gen_tok_[:, :P] (the fixed
// staging rows the decode graph was captured on).  teacher_forced: gen_tok_ already holds
// full sequences; predictions go to pred_.
void Engine::generate(const Decoder& m, int B, bool teacher_forced) {
  const int d = m.a.d_model, V = m.a.vocab;
  // prefill: forward over the prompt, K/V stored for every prompt position
  forward(m, gen_tok_.as<int32_t>(), B, S_, P_, false, &kv_);
  K(rlhf_gather_rows(arp_->hf, dec_hf_.p, B, P_, 1, P_ - 1, d, 2, stream_), 1);
  const int start = P_ - 1;
  cudaMemcpyAsync(pos_.p, &start, sizeof(int), cudaMemcpyHostToDevice, stream_);
  int32_t* dst = teacher_forced ? pred_.as<int32_t>() : gen_tok_.as<int32_t>();
  // RLHF_DEC_FUSE_MERGE=0: the greedy merge as its own launch after every LM head (timing A/B)
  static const bool fuse_env = [] { const char* e = getenv("RLHF_DEC_FUSE_MERGE"); return !e || atoi(e) != 0; }();
  static const bool skip_env = getenv("RLHF_DECODE_SKIP") != nullptr;
  fuse_merge_ = fuse_env && !skip_env && R_ > 1 && !(opt_.use_cuda_graph == 3 && !m.llama());
  // with the fused merge, each decode step's entry kernel merges the previous LM head; the
  // last step's LM head is merged after the loop
  lm_head_argmax(m, dec_hf_.as<uint16_t>(), B, dst, !fuse_merge_);  // the merge also advances *pos
  if (ev_prefill_) cudaEventRecord(ev_prefill_, stream_);  // prefill done (per Generation task)
  if (R_ <= 1) return;
  if (opt_.use_cuda_graph == 3 && !m.llama()) {  // the persistent loop implements the OPT family
    // persistent decode loop: all R-1 steps in one cooperative kernel (opt-in;
    // on one B200 at B = 32 it is not yet faster than the PDL graph)
    rlhf_decode_loop_params lp{};
    lp.arch = &m.a;
    lp.weights = m.w.p;
    lp.B = B;
    lp.tokens = gen_tok_.as<int32_t>();
    lp.tok_stride = S_;
    lp.pred = teacher_forced ? pred_.as<int32_t>() : nullptr;
    lp.margin = margin_.as<float>();
    lp.pos = pos_.as<int>();
    lp.steps = R_ - 1;
    lp.kcache = kv_.k.p;
    lp.vcache = kv_.v.p;
    lp.kv_B = kv_.B;
    lp.Smax = kv_.Smax;
    const size_t need = rlhf_decode_loop_workspace_bytes(&lp);
    if (need > 0) {
      if (loop_ws_.bytes < need) loop_ws_.alloc(need);
      lp.workspace = loop_ws_.p;
      lp.workspace_bytes = loop_ws_.bytes;
      // RLHF_LOOP_PROBE=1 (debug): per-phase timestamps of decode step 1 -> stderr summary
      static const char* probe_env = getenv("RLHF_LOOP_PROBE");
      const bool probe = probe_env != nullptr;
      lp.probe_q = probe ? std::max(1, atoi(probe_env)) : 1;
      int sms = 0;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, opt_.device);
      const int P = 8 * m.a.n_layers + 2;
      DevBuf pb;
      if (probe && R_ > 2) {
        pb.alloc(static_cast<size_t>(P) * 2 * sms * 8 + static_cast<size_t>(sms) * 16 * 8);
        lp.probe = pb.as<unsigned long long>();
      }
      K(rlhf_decode_loop(&lp, stream_), 1);
      if (lp.probe) {
        std::vector<unsigned long long> h(static_cast<size_t>(P) * 2 * sms);
        cudaStreamSynchronize(stream_);
        cudaMemcpy(h.data(), pb.p, h.size() * 8, cudaMemcpyDeviceToHost);
        auto med = [&](int row) {
          std::vector<unsigned long long> v(h.begin() + static_cast<size_t>(row) * sms,
                                            h.begin() + static_cast<size_t>(row + 1) * sms);
          std::sort(v.begin(), v.end());
          return std::make_pair(v[v.size() / 2], v.back());
        };
        const char* names[8] = {"qkv", "att", "wo", "resln2", "w1", "relu", "w2", "resln1"};
        unsigned long long prev = med(2 * (P - 1) + 1).first;  // previous phase exit (approx: last of step)
        prev = 0;
        double tot = 0;
        for (int q = 0; q < P; ++q) {
          const auto work = med(2 * q), exitb = med(2 * q + 1);
          if (q > 0) {
            const double ph = (work.second - prev) * 1e-3, bar = (exitb.first - work.second) * 1e-3;
            tot += (exitb.first - prev) * 1e-3;
            if (q < 8 || q >= P - 2)
              fprintf(stderr, "[loop probe] phase %2d %-7s work(max) %7.2f us  barrier %6.2f us\n", q,
                      q >= P - 2 ? (q == P - 2 ? "lm" : "argmax") : names[q % 8], ph, bar);
          }
          prev = exitb.first;
        }
        fprintf(stderr, "[loop probe] step total (phases 1..%d) %.2f us\n", P - 1, tot);
        std::vector<unsigned long long> sub(static_cast<size_t>(sms) * 16);
        cudaMemcpy(sub.data(), pb.as<unsigned long long>() + static_cast<size_t>(P) * 2 * sms, sub.size() * 8,
                   cudaMemcpyDeviceToHost);
        const unsigned long long att0 = med(2 * (lp.probe_q - 1) + 1).first;  // exit of the barrier opening probe_q
        for (int k = 0; k < 16; ++k) {
          std::vector<double> v;
          for (int c = 0; c < sms; ++c)
            if (sub[static_cast<size_t>(c) * 16 + k]) v.push_back((sub[static_cast<size_t>(c) * 16 + k] - att0) * 1e-3);
          if (v.empty()) continue;
          std::sort(v.begin(), v.end());
          fprintf(stderr, "[loop probe] sub %2d: n=%3zu median %7.2f max %7.2f us\n", k, v.size(), v[v.size() / 2],
                  v.back());
        }
      }
      return;
    }
  }
  const bool use_graph = opt_.use_cuda_graph != 0;
  if (use_graph) {
    // k decode steps per CUDA graph (RLHF_DEC_GRAPH_STEPS, default 8): the PDL chain then also
    // runs across step boundaries inside a graph; the R-1 steps are floor((R-1)/k) launches of
    // the k-step graph plus the rest as launches of a one-step graph
    static const int ksteps = [] { const char* e = getenv("RLHF_DEC_GRAPH_STEPS"); return e ? std::max(1, atoi(e)) : 8; }();
    const int k = std::max(1, std::min(ksteps, R_ - 1));
    auto capture = [&](int nsteps, cudaGraphExec_t* out, int* nlaunch) {
      cudaGraph_t g;
      const int before = launches_;
      if (cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
        throw DeviceError("decode graph capture begin failed");
      pdl_ = opt_.use_cuda_graph == 2 ? 0 : 1;  // programmatic dependent launches inside the graph
      rlhf_set_pdl(pdl_);  // (thread-local: engines on other host threads are unaffected)
      try {
        for (int st = 0; st < nsteps; ++st) decode_step(m, B);
      } catch (...) {  // leave the stream usable: end the capture, drop the partial graph
        rlhf_set_pdl(0);
        pdl_ = 0;
        cudaGraph_t partial = nullptr;
        cudaStreamEndCapture(stream_, &partial);
        if (partial) cudaGraphDestroy(partial);
        cudaGetLastError();
        throw;
      }
      rlhf_set_pdl(0);
      pdl_ = 0;
      if (cudaStreamEndCapture(stream_, &g) != cudaSuccess) throw DeviceError("decode graph capture failed");
      if (cudaGraphInstantiate(out, g, 0) != cudaSuccess) throw DeviceError("decode graph instantiate failed");
      cudaGraphDestroy(g);
      *nlaunch = launches_ - before;
      launches_ = before;
    };
    if (!decode_graph_ || graph_for_pred_ != teacher_forced || graph_steps_ != k) {
      for (cudaGraphExec_t* gp : {&decode_graph_, &decode_graph1_})
        if (*gp) cudaGraphExecDestroy(*gp), *gp = nullptr;
      graph_for_pred_ = teacher_forced;
      graph_steps_ = k;
      capture(k, &decode_graph_, &graph_launches_);
      if (k > 1) capture(1, &decode_graph1_, &graph1_launches_);
    }
    const int reps = (R_ - 1) / k, rest = (R_ - 1) % k;
    for (int r = 0; r < reps; ++r) {
      if (cudaGraphLaunch(decode_graph_, stream_) != cudaSuccess) throw DeviceError("decode graph launch failed");
      launches_ += graph_launches_;
    }
    for (int r = 0; r < rest; ++r) {
      if (cudaGraphLaunch(decode_graph1_, stream_) != cudaSuccess) throw DeviceError("decode graph launch failed");
      launches_ += graph1_launches_;
    }
  } else {
    graph_for_pred_ = teacher_forced;
    for (int s = 1; s < R_; ++s) decode_step(m, B);
  }
  if (fuse_merge_) {
    K(rlhf_argmax_tiles(dec_top2_.as<float>(), (V + 127) / 128, B, dst, S_, pos_.as<int>(), margin_.as<float>(), 1,
                        stream_),
      1);
    fuse_merge_ = false;
  }
}

// ---- ZeRO-2: per-layer reduce-scatter of the working gradient bucket (comm lane) ----------

void Engine::zero2_layer_begin(Decoder& m, int l) {
  // the bucket's previous reduce-scatter (layer l + 2, or the previous chunk) has read it
  CK(cudaStreamWaitEvent(stream_, m.rs_done[l & 1], 0));
  CK(cudaMemsetAsync(m.gwork[l & 1].p, 0, static_cast<size_t>(m.work_len) * 4, stream_));
}

void Engine::zero2_layer_end(Decoder& m, int l) {
  const GradBucket& g = m.buckets[static_cast<size_t>(l) + 1];
  cudaEvent_t ready = take_event();
  CK(cudaEventRecord(ready, stream_));
  cudaStream_t cs = lane_[2];
  CK(cudaStreamWaitEvent(cs, ready, 0));
  float* src = m.gwork[l & 1].as<float>();
  ncclComm_t comm = dp_comm(m);
  if (comm) {
    NK(nccl().ReduceScatter(src, m.rs_tmp.p, static_cast<size_t>(g.slice), ncclFloat32, ncclSum, comm, cs));
    comm_bytes_ += 4.0 * static_cast<double>(g.slice) * (m.dp - 1);
    kcheck(rlhf_add_f32(m.gshard.as<float>() + g.soff, m.rs_tmp.as<float>(), g.slice, cs), "rlhf_add_f32");
  } else {  // one rank: the slice is the whole bucket
    kcheck(rlhf_add_f32(m.gshard.as<float>() + g.soff, src, g.slice, cs), "rlhf_add_f32");
  }
  ++launches_;
  CK(cudaEventRecord(m.rs_done[l & 1], cs));
}

// ZeRO-3: layer l's bf16 weights all-gathered (comm stream) into working buffer l % 2 unless
// already there; `next` is gathered into the other buffer ahead of its use.
void Engine::zero3_fetch(const Decoder& m, int l, int next) {
  auto gather = [&](int layer) {
    const int b = layer & 1;
    if (m.wwork_layer[b] == layer) return;
    cudaEvent_t free_ev = take_event();  // the compute stream's earlier kernels used buffer b
    CK(cudaEventRecord(free_ev, stream_));
    cudaStream_t cs = lane_[2];
    CK(cudaStreamWaitEvent(cs, free_ev, 0));
    const GradBucket& g = m.buckets[static_cast<size_t>(layer) + 1];
    const uint16_t* mine = m.wshard.as<uint16_t>() + g.soff;
    if (ncclComm_t comm = dp_comm(m)) {
      NK(nccl().AllGather(mine, m.wwork[b].p, static_cast<size_t>(g.slice), ncclBfloat16, comm, cs));
      comm_bytes_ += 2.0 * static_cast<double>(g.slice) * (m.dp - 1);
    } else {
      CK(cudaMemcpyAsync(m.wwork[b].p, mine, static_cast<size_t>(g.len) * 2, cudaMemcpyDeviceToDevice, cs));
    }
    CK(cudaEventRecord(m.wgather_done[b], cs));
    m.wwork_layer[b] = layer;
  };
  gather(l);
  CK(cudaStreamWaitEvent(stream_, m.wgather_done[l & 1], 0));
  if (next >= 0) gather(next);
}

// Optimizer step under ZeRO-2: the embedding / head buckets (accumulated over the whole epoch
// in full) are reduce-scattered into their slices, AdamW updates the rank's slices of every
// bucket, and each bucket's bf16 slices are all-gathered back into the flat weights.
void Engine::zero2_optimizer(Decoder& m, ncclComm_t comm, float lr, int i) {
  const ExecStep& s = xp_.steps[static_cast<size_t>(i)];
  const int st = static_cast<int>(Stage::Training);
  const int ml = lane_of(s.model);
  begin_event(i, s, static_cast<int>(TaskKind::Collective), 2, st);
  for (int k : {0, static_cast<int>(m.buckets.size()) - 1}) {
    const GradBucket& g = m.buckets[static_cast<size_t>(k)];
    float* full = (k == 0 ? m.gpre : m.gpost).as<float>();
    if (comm) {
      NK(nccl().ReduceScatter(full, m.rs_tmp.p, static_cast<size_t>(g.slice), ncclFloat32, ncclSum, comm, stream_));
      comm_bytes_ += 4.0 * static_cast<double>(g.slice) * (m.dp - 1);
      K(rlhf_add_f32(m.gshard.as<float>() + g.soff, m.rs_tmp.as<float>(), g.slice, stream_), 1);
    } else {
      K(rlhf_add_f32(m.gshard.as<float>() + g.soff, full, g.slice, stream_), 1);
    }
  }
  end_event();
  cudaEvent_t prev = evs_.back().b;
  begin_event(i, s, 7, ml, st);
  CK(cudaStreamWaitEvent(stream_, prev, 0));
  m.adam_step += 1;
  K(rlhf_adamw(m.master.as<float>(), m.m.as<float>(), m.v.as<float>(), m.gshard.as<float>(), m.wshard.p, m.shard, lr,
               cfg_.beta1, cfg_.beta2, cfg_.adam_eps, cfg_.weight_decay, m.adam_step, stream_), 1);
  end_event();
  prev = evs_.back().b;
  begin_event(i, s, static_cast<int>(TaskKind::Collective), 2, st);
  CK(cudaStreamWaitEvent(stream_, prev, 0));
  // ZeRO-2: every bucket back into the flat weights; ZeRO-3: only the embedding / head
  // buckets (the layers are gathered when they run; the gathered copies are stale now)
  for (size_t k = 0; k < m.buckets.size(); ++k) {
    if (m.zero3 && k != 0 && k + 1 != m.buckets.size()) continue;
    const GradBucket& g = m.buckets[k];
    const uint16_t* mine = m.wshard.as<uint16_t>() + g.soff;
    uint16_t* dst = !m.zero3 ? m.w.as<uint16_t>() + g.start : (k == 0 ? m.wpre : m.wpost).as<uint16_t>();
    if (comm) {
      NK(nccl().AllGather(mine, m.ag_stage.p, static_cast<size_t>(g.slice), ncclBfloat16, comm, stream_));
      comm_bytes_ += 2.0 * static_cast<double>(g.slice) * (m.dp - 1);
      CK(cudaMemcpyAsync(dst, m.ag_stage.p, static_cast<size_t>(g.len) * 2, cudaMemcpyDeviceToDevice, stream_));
    } else {
      CK(cudaMemcpyAsync(dst, mine, static_cast<size_t>(g.len) * 2, cudaMemcpyDeviceToDevice, stream_));
    }
  }
  m.wwork_layer[0] = m.wwork_layer[1] = -1;
  end_event();
}

// Fused AdamW on this rank's master slice (ZeRO-1: the reduce-scattered gradient shard at
// grad[shard_off, +shard); unsharded: the whole vector), writing the bf16 compute copy.
void Engine::adam(Decoder& m, float lr) {
  m.adam_step += 1;
  K(rlhf_adamw(m.master.as<float>(), m.m.as<float>(), m.v.as<float>(), m.grad.as<float>() + m.shard_off,
               m.w.as<uint16_t>() + m.shard_off, m.shard, lr, cfg_.beta1, cfg_.beta2, cfg_.adam_eps,
               cfg_.weight_decay, m.adam_step, stream_), 1);
}

}  // namespace flexrlhf
