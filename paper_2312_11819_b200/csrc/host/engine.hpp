// engine.hpp — the executor that replaces the reference simulator's analytic
// clock (simulate(), /root/reference/proj/include/rlhfsim/simulator.hpp:46-47)
// with real execution of the PPO iteration on one GPU per process.
//
// Per rank: the models this rank hosts under its placement, their bf16 weights
// (+ fp32 master / Adam state for trainable ones), activation arenas, the
// generator's KV cache, one row-set buffer per device group it belongs to
// (execplan.hpp), and NCCL communicators (world, one per trained model's
// data-parallel group, one per ParamSync pair).  The step walks the ExecPlan --
// the task DAG plus the exchanges the comm schedule induces -- on three CUDA
// streams ("lanes": main compute, side compute, comm) joined by per-step events.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <atomic>
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "execplan.hpp"
#include "flexrlhf/simulator.hpp"
#include "flexrlhf/placement.hpp"
#include "rlhf_engine.h"
#include "rlhf_kernels.h"

namespace flexrlhf {

extern std::atomic<int64_t> g_device_bytes;  // bytes held by DevBufs of this process

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  explicit DevBuf(size_t n) { alloc(n); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf();
  void alloc(size_t n);
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
};

// ZeRO-2 gradient bucket: a contiguous range of the flat parameter vector (the embeddings,
// one decoder layer, or the final norm + heads), reduce-scattered as a unit.  Rank r owns
// elements [start + r * slice, start + (r + 1) * slice) of it (padded: slice * dp >= len),
// stored at [soff, soff + slice) of the rank's concatenated shard arrays.
struct GradBucket {
  int64_t start = 0, len = 0, slice = 0, soff = 0;
};

// One decoder (OPT or LLaMA family) resident on this device.
struct Decoder {
  rlhf_arch a{};
  uint64_t seed = 0;
  bool trainable = false;
  int64_t n = 0;  // flat parameter count (rlhf_param_total)
  // ZeRO-1: the fp32 master/m/v hold elements [shard_off, shard_off + shard) of the flat
  // vector (padded to npad = dp * shard); unsharded: shard = npad = n, shard_off = 0.
  // ZeRO-2: master/m/v/gshard hold the rank's slice of every GradBucket (shard = their sum).
  int64_t npad = 0, shard = 0, shard_off = 0;
  bool sharded = false;
  DevBuf w;       // bf16 flat
  DevBuf master, m, v, grad;  // fp32 flat (trainable only; grad unused under ZeRO-2)
  int adam_step = 0;
  DevBuf rope;    // LLaMA: float2 (cos, sin) [max_pos][hd/2] (rlhf_rope_cos_sin)
  // ---- ZeRO-2 (bucket-sharded gradients): no full-size gradient is ever resident.  Layer
  // l's gradients accumulate in working bucket l % 2 (reduce-scattered into gshard after
  // the layer's backward), the embedding / head groups in full-size buffers that are
  // reduce-scattered once per optimizer step (the tied LM head adds into the embedding).
  bool zero2 = false;
  int dp = 1, dp_rank = 0;
  std::vector<GradBucket> buckets;  // [pre, layer 0 .. L-1, post]
  int64_t layers_start = 0, layer_len = 0, post_start = 0, work_len = 0;
  DevBuf gpre, gpost, gwork[2], gshard, rs_tmp, wshard, ag_stage;
  cudaEvent_t rs_done[2] = {nullptr, nullptr};  // working bucket free again (comm lane)
  // ---- ZeRO-3 (also the bf16 weights sharded): wshard holds the rank's slices of every
  // bucket; the embedding / head buckets stay whole in wpre / wpost, a decoder layer's
  // weights are all-gathered on the comm stream into working buffer l % 2 just before the
  // layer runs (the next layer's gather overlaps this one's compute).
  bool zero3 = false;
  DevBuf wpre, wpost, wwork[2];
  mutable int wwork_layer[2] = {-1, -1};
  cudaEvent_t wgather_done[2] = {nullptr, nullptr};
  bool llama() const { return a.family == 1; }
  // tensors absent from the family's layout (size 0) are NULL
  const uint16_t* T(int t, int l = 0) const {
    if (!rlhf_tensor_numel(&a, t)) return nullptr;
    const int64_t off = rlhf_tensor_offset(&a, t, l);
    if (!zero3) return w.as<uint16_t>() + off;
    if (off < layers_start) return wpre.as<uint16_t>() + off;
    if (off >= post_start) return wpost.as<uint16_t>() + (off - post_start);
    return wwork[l & 1].as<uint16_t>() + (off - layers_start - static_cast<int64_t>(l) * layer_len);
  }
  float* G(int t, int l = 0) const {
    if (!rlhf_tensor_numel(&a, t)) return nullptr;
    const int64_t off = rlhf_tensor_offset(&a, t, l);
    if (!zero2) return grad.as<float>() + off;
    if (off < layers_start) return gpre.as<float>() + off;
    if (off >= post_start) return gpost.as<float>() + (off - post_start);
    return gwork[l & 1].as<float>() + (off - layers_start - static_cast<int64_t>(l) * layer_len);
  }
  int head_id() const { return llama() ? RLHF_T_LM_HEAD : RLHF_T_TOK_EMB; }  // LM head (tied for OPT)
};

// Activation arena shared by every model on the rank (they run one at a time).
struct Arena {
  int B = 0, S = 0, R = 0, d = 0, ff = 0, H = 0, V = 0, L = 0;  // capacities (ff: FFN-up width, 2 d_ff for SwiGLU)
  int ffa = 0;                                                     // SwiGLU output width (0: OPT only)
  uint16_t* act = nullptr;                                         // SwiGLU output / its gradient [T, ffa]
  int64_t T = 0, Z = 0;    // rows / (sample, head) pairs of a whole Forward stage
  int64_t Ts = 0, Zs = 0;  // the same for one TrainFB micro-batch: stride of the saved layers
  std::vector<DevBuf*> owned;
  float *xres = nullptr, *mean = nullptr, *rstd = nullptr;  // [(2L+1)][T*d], [(2L+1)][T]
  uint16_t *h1 = nullptr, *qkv = nullptr, *P = nullptr, *o = nullptr, *h2 = nullptr, *f = nullptr, *hf = nullptr;
  float* scores = nullptr;
  uint16_t* dS = nullptr;
  uint16_t* hf_resp = nullptr;
  float *logits = nullptr, *lse = nullptr, *dhf_resp = nullptr;
  uint16_t* dz = nullptr;
  float *dres = nullptr, *dhf = nullptr, *dh = nullptr;
  uint16_t *g = nullptr, *dpre = nullptr, *dov = nullptr, *dqkv = nullptr;
  float* ws = nullptr;
  size_t ws_floats = 0;
  float* gemm_ws = nullptr;
  size_t gemm_ws_bytes = 0;
  int* counters = nullptr;
  int counters_len = 0;
  ~Arena();
};

struct KVCache {
  DevBuf k, v;  // [L][B][H][Smax][hd] bf16
  int L = 0, B = 0, H = 0, Smax = 0, hd = 0;
  uint16_t* Kc(int l) const { return k.as<uint16_t>() + static_cast<int64_t>(l) * B * H * Smax * hd; }
  uint16_t* Vc(int l) const { return v.as<uint16_t>() + static_cast<int64_t>(l) * B * H * Smax * hd; }
};

// Per row set this rank belongs to (ExecPlan::sets): the experience rows of its samples.
struct RowBufs {
  int rows = 0;
  bool trainer = false;                            // holds a trained model: GAE + training buffers
  DevBuf tokens;                                   // int32 [rows][S]
  DevBuf logp_old, logp_ref, values, score;        // f32 [rows][R] ([rows] for score)
  DevBuf rewards, adv, ret, logp_new, values_new;  // f32 [rows][R] (trainers)
  DevBuf gbuf, gbuf2;                              // loss gradients wrt logp / values
  void* field(Field f) const;
};

// One executed interval of the step (rlhf_event in include/rlhf_engine.h).
struct ExecEvent {
  int step = -1, task = -1, kind = 0, model = 0, mb = 0, rollout = 0, epoch = 0, lane = 0, comm_op = -1, stage = 0;
  cudaEvent_t a = nullptr, b = nullptr;
  double start = 0, end = 0;
};

class Engine {
 public:
  Engine(const rlhf_ppo_config& cfg, const rlhf_engine_options& opt);
  ~Engine();
  void step(const int32_t* prompts_host, rlhf_step_report* rep);
  size_t tensor_bytes(const std::string& name) const;
  void read(const std::string& name, void* host, size_t bytes);
  void greedy_check(const int32_t* tokens_host, int32_t* pred_host, float* margin_host);
  cudaStream_t stream() const { return lane_[0]; }
  const std::vector<ExecEvent>& events() const { return evs_; }
  const ExecPlan& exec_plan() const { return xp_; }
  int rank() const { return rank_; }

 private:
  // ---- building blocks (engine_model.cpp) ----
  void init_decoder(Decoder& m, const rlhf_arch& a, uint64_t seed, bool trainable, ncclComm_t dp_comm = nullptr);
  void forward(const Decoder& m, const int32_t* tokens, int B, int tok_stride, int T, bool save, KVCache* kv);
  void attention_fwd(const uint16_t* qkv, uint16_t* P, uint16_t* o, int B, int T, int H, int hd, bool keep_p);
  void attention_bwd(const uint16_t* qkv, const uint16_t* P, const uint16_t* dov, uint16_t* dqkv, int B, int T, int H, int hd);
  void backward(Decoder& m, const int32_t* tokens, int B, int S);
  void zero2_layer_begin(Decoder& m, int l);   // working bucket l % 2 free -> zeroed
  void zero2_layer_end(Decoder& m, int l);     // reduce-scatter + accumulate its shard (comm lane)
  void zero2_optimizer(Decoder& m, ncclComm_t comm, float lr, int step_index);
  void zero3_fetch(const Decoder& m, int l, int next);  // layer l's weights resident (+ prefetch next)
  ncclComm_t dp_comm(const Decoder& m) const { return &m == &actor_ ? actor_comm_ : critic_comm_; }
  void norm(const Decoder& m, const float* x, int g, int l, uint16_t* y, float* mean, float* rstd, int rows);
  void norm_bwd(Decoder& m, const float* dy, const float* x, const float* mean, const float* rstd, int g, int l, int rows);
  void lm_logprobs(const Decoder& m, const int32_t* tokens, int B, float* logp, bool keep_logits);
  void generate(const Decoder& m, int B, bool teacher_forced);
  void decode_step(const Decoder& m, int B);
  void lm_head_argmax(const Decoder& m, const uint16_t* hf, int B, int32_t* dst, bool merge = true);
  bool fuse_merge_ = false;  // decode: greedy merge folded into the next step's embed (generate())
  void adam(Decoder& m, float lr);
  void score_logp(const Decoder& m, const int32_t* tok, int B, float* logp);
  void score_values(const Decoder& m, const int32_t* tok, int B, float* values);
  void score_reward(const Decoder& m, const int32_t* tok, int B, float* score);
  void build_arena(Arena& A, bool trains, bool critic_only = false);

  // ---- the executor (engine.cpp) ----
  Decoder* model(ModelName m);
  int lane_of(ModelName m) const;
  void use_lane(int l);
  void run_exchange(const ExecStep& s);
  void run_task(const ExecStep& s);
  void run_experience(const ExecStep& s);
  void run_optimizer(const ExecStep& s, int step_index);
  void train_rows(Decoder& m, bool actor, RowBufs& rb, int row0, int B, float denom, bool reuse = false);
  void begin_event(int step_index, const ExecStep& s, int kind, int lane, int stage);
  void end_event();
  void wait_deps(int step_index, int lane);
  void finish_report(rlhf_step_report* rep, double loss_denom);

  // GEMM helpers (all go through rlhf_gemm)
  void linear(const uint16_t* X, int M, int K, const uint16_t* W, int N, const uint16_t* bias, void* Y, bool y_f32,
              bool relu, const float* residual);
  void linear_decode(const uint16_t* W, int N_out, int K, const uint16_t* X, int Bg, const uint16_t* bias, void* Y,
                     bool y_f32, bool relu, const float* residual, const float* ln_x = nullptr,
                     const uint16_t* ln_g = nullptr, const uint16_t* ln_b = nullptr, int kv_layer = -1,
                     int kv_b0 = 0, const float* st_in = nullptr, int st_parts = 0, float* st_out = nullptr,
                     int* parts_out = nullptr);
  void gemm(rlhf_gemm_params& p);
  void kcheck(int status, const char* what);

  rlhf_ppo_config cfg_;
  rlhf_engine_options opt_;
  std::string strategy_;
  int P_, R_, S_;
  int rank_ = 0, world_n_ = 1;
  int Bg_ = 0;        // prompts of this rank's home shard per rollout
  int Bcap_ = 0;      // rows of the largest Forward / Generation block this rank runs
  int gen_B_ = 0;     // sequences per Generation task (the generator row set's per)
  int train_mb_ = 0;  // samples per TrainFB chunk (gradients accumulate over them)
  ExecPlan xp_;
  StrategyTag tag_ = StrategyTag::Colocated;
  // lanes: 0 main compute, 1 side compute (critic-shaped models, Co-located-style ranks), 2 comm
  cudaStream_t lane_[3] = {nullptr, nullptr, nullptr};
  bool side_ = false;
  bool reuse_fwd_[2] = {false, false};  // Actor / Critic: epoch-0 TrainFB reuses the experience Forward
  cudaStream_t stream_ = nullptr;  // the lane currently enqueued on
  int cur_lane_ = 0;
  ncclComm_t world_ = nullptr, actor_comm_ = nullptr, critic_comm_ = nullptr;
  ncclComm_t sync_comm_[2] = {nullptr, nullptr};  // ParamSync: Actor -> ShadowActor, Critic -> ShadowCritic
  int sync_root_[2] = {0, 0};
  double comm_bytes_ = 0;
  int launches_ = 0;
  int pdl_ = 0;  // launch decode kernels as programmatic dependents
  bool hosts_[6] = {false, false, false, false, false, false};

  Decoder actor_, critic_, ref_, reward_, shadow_actor_, shadow_critic_;
  Decoder* generator_ = nullptr;
  Arena ar_main_, ar_side_;  // activation arenas (main lane / side lane)
  Arena* arp_ = &ar_main_;   // the arena of the lane currently in use
  KVCache kv_;
  std::unique_ptr<RowBufs[]> rs_;  // indexed like xp_.sets (empty for sets this rank is not in)
  DevBuf home_;               // int32 [rollouts * Bg][S]: this rank's prompts (first P columns)
  DevBuf gen_tok_, pred_, margin_, pos_;  // generation staging [gen_B][S] (the decode graph's fixed rows)
  DevBuf loss_;                           // f32 [actor_loss, critic_loss, sum score, sum kl]
  DevBuf loop_ws_;   // persistent decode loop workspace
  DevBuf dec_top2_;  // LM-head per-tile top-2 partials [V/128][B] x float4
  DevBuf dec_x_, dec_h_, dec_qkv_, dec_o_, dec_f_, dec_act_, dec_hf_, dec_logits_, argmax_ws_;
  DevBuf dec_st_[2];  // LayerNorm (sum, sum sq) partials of the O-proj / FFN-down outputs [CTAs][B][2]
  cudaGraphExec_t decode_graph_ = nullptr, decode_graph1_ = nullptr;  // k decode steps / one step
  int graph_launches_ = 0, graph1_launches_ = 0, graph_steps_ = 0;
  bool graph_for_pred_ = false;
  // per-step timing: events of every executed interval, the step's start/end
  std::vector<ExecEvent> evs_;
  std::vector<cudaEvent_t> ev_pool_;
  size_t ev_next_ = 0;
  std::vector<std::vector<int>> deps_;   // per ExecPlan step: the steps it waits for
  std::vector<int> step_lane_;           // per ExecPlan step: lane of its last event on this rank (-1: not run)
  std::vector<cudaEvent_t> step_done_;   // per ExecPlan step: its completion event on this rank
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prefill_;  // (gen start, prefill end), (prefill end, gen end)
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> decode_;
  cudaEvent_t ev_begin_ = nullptr, ev_end_ = nullptr, ev_prefill_ = nullptr;
  cudaEvent_t take_event();
};

// The measured counterpart of simulate() (simulator.hpp:46-47) in the same vocabulary: one
// PPO iteration on this rank's device, returned as a SimReport whose events are this rank's
// measured intervals (devices = {rank}, comm_lane for lane 2), per-stage seconds / fractions
// with the same compute-lane attribution, busy seconds, bubble fraction and memory.
SimReport execute(Engine& engine, const int32_t* prompts_host = nullptr);

}  // namespace flexrlhf
