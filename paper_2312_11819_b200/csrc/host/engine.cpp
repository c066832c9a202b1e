// engine.cpp — the PPO iteration driver and its C-ABI (include/rlhf_engine.h).
//
// Walks the reference's one-iteration stage DAG (task_graph,
// /root/reference/proj/src/workload.cpp:109-175): Generation -> Forward for
// every scorer model -> experience-buffer barrier (GAE) -> TrainFB(Actor),
// TrainFB(Critic) -> (shadows) ParamSync.  Each stage is timed with CUDA events
// and reported in the reference's SimReport vocabulary (simulator.hpp:30-44).
//
// One process per GPU.  The rank's role comes from the placement plan
// (build_strategy over ClusterTopology::b200_box(world)): which models it hosts,
// its data-parallel groups, and the partner rank (i <-> i + N/2) it exchanges
// experience with -- the executed form of derive_comm_schedule
// (placement.hpp:101-102):
//   colocated     every model everywhere; gradient all-reduce over the world
//   interleaving1 Actor/Critic everywhere, Ref on the first half, Reward on the
//                 second: AllGather of (query,response) within the pair, each
//                 side scores 2*Bg samples, AlltoAll of the outputs back
//   interleaving2 {Actor, Ref} on the first half, {Critic, Reward} on the second:
//                 the Actor side generates the pair's 2*Bg samples, tokens go
//                 over, outputs are swapped, Actor and Critic train concurrently
//   disaggregated {Actor, Critic} trainers on the first half, {ShadowActor,
//                 ShadowCritic, Ref, Reward} on the second: inference side
//                 generates + scores, sends experience to the trainers, trainers
//                 send updated weights back (ParamSync) after training.
#include "engine.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>

#include "capi_util.hpp"
#include "flexrlhf/errors.hpp"
#include "nccl_dyn.hpp"

namespace flexrlhf {

#define CK(x)                                                                                    \
  do {                                                                                           \
    cudaError_t e_ = (x);                                                                        \
    if (e_ != cudaSuccess) throw DeviceError(std::string(#x) + ": " + cudaGetErrorString(e_));   \
  } while (0)
#define NK(x)                                                                                     \
  do {                                                                                            \
    ncclResult_t r_ = (x);                                                                        \
    if (r_ != ncclSuccess) throw DeviceError(std::string(#x) + ": " + nccl().GetErrorString(r_)); \
  } while (0)
#define K(call, n)         \
  do {                     \
    kcheck((call), #call); \
    launches_ += (n);      \
  } while (0)

namespace {

rlhf_arch fixed(rlhf_arch a, int scalar_head) {
  a.scalar_head = scalar_head;
  return a;
}

void validate(const rlhf_ppo_config& c) {
  if (c.batch < 1 || c.prompt_len < 1 || c.gen_len < 1) throw ConfigError("batch, prompt_len, gen_len must be >= 1");
  const int S = c.prompt_len + c.gen_len;
  for (const rlhf_arch* a : {&c.actor, &c.critic}) {
    if (a->family != 0 && a->family != 1) throw ConfigError("family must be 0 (OPT) or 1 (LLaMA)");
    if (a->d_model > 4096) throw ConfigError("d_model above 4096 is not supported");
    if (S > a->max_pos) throw ConfigError("prompt_len + gen_len exceeds max_pos");
    if (a->d_model % a->n_heads) throw ConfigError("d_model must divide by n_heads");
    const int hd = a->d_model / a->n_heads;
    if (hd != 64 && hd != 128) throw ConfigError("head_dim must be 64 or 128");
    if (a->d_model % 64 || a->d_ff % 64 || a->vocab % 8) throw ConfigError("d_model/d_ff must be multiples of 64, vocab of 8");
  }
  if (c.prompt_len % 8 || S % 8) throw ConfigError("prompt_len and prompt_len+gen_len must be multiples of 8");
}

bool in(const std::vector<int>& v, int x) { return std::find(v.begin(), v.end(), x) != v.end(); }

}  // namespace

Engine::Engine(const rlhf_ppo_config& cfg, const rlhf_engine_options& opt) : cfg_(cfg), opt_(opt) {
  validate(cfg_);
  if (opt_.zero_stage < 0 || opt_.zero_stage > 1)
    throw ConfigError("zero_stage must be 0 or 1 (ZeRO-2/3 are planned, DESIGN.md §8)");
  cfg_.actor.scalar_head = 0;
  cfg_.critic.scalar_head = 1;
  strategy_ = opt.strategy ? opt.strategy : "colocated";
  opt_.strategy = nullptr;
  rank_ = opt_.rank;
  world_n_ = std::max(1, opt_.world_size);
  Bg_ = cfg_.batch;
  P_ = cfg_.prompt_len;
  R_ = cfg_.gen_len;
  S_ = P_ + R_;

  // ---- role of this rank from the placement plan -------------------------------
  {
    ModelSizes sz;
    sz.actor = ArchSpec{}.param_count(false);  // sizes only matter for memory planning
    sz.critic = sz.ref = sz.reward = sz.actor;
    LoopParams lp;
    lp.batch_size = Bg_ * world_n_;
    lp.prompt_len = P_;
    lp.gen_len = R_;
    StrategyConfig sc;
    sc.name = strategy_;
    sc.tp_gen = 1;
    sc.inference_ratio = 0.5;
    const BuiltStrategy bs = build_strategy(sc, ClusterTopology::b200_box(world_n_),
                                            build_pipeline(PipelineStructure::ACNonShare, sz, lp));
    plan_ = bs.plan;
    for (int m = 0; m < 6; ++m) {
      const ModelName mn = static_cast<ModelName>(m);
      hosts_[m] = plan_.has(mn) && in(plan_.cfg(mn).devices, rank_);
    }
    tag_ = plan_.strategy_tag;
    if (tag_ != StrategyTag::Colocated && world_n_ % 2) throw ConfigError(strategy_ + " needs an even number of GPUs");
    partner_ = tag_ == StrategyTag::Colocated ? -1 : (rank_ < world_n_ / 2 ? rank_ + world_n_ / 2 : rank_ - world_n_ / 2);
  }
  const bool pair_batch = tag_ == StrategyTag::Interleaving2 || tag_ == StrategyTag::Disaggregated;
  Bcap_ = (tag_ == StrategyTag::Colocated) ? Bg_ : 2 * Bg_;
  train_mb_ = opt_.train_micro_batch > 0 ? std::min(opt_.train_micro_batch, Bcap_) : Bcap_;
  gen_B_ = pair_batch ? 2 * Bg_ : Bg_;

  CK(cudaSetDevice(opt_.device));
  CK(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
  for (auto& e : ev_) CK(cudaEventCreate(&e));

  // ---- communicators: world + one data-parallel group per trainable model -----
  if (world_n_ > 1) {
    if (!opt_.nccl_id) throw ConfigError("world_size > 1 needs an NCCL unique id");
    ncclUniqueId id;
    std::memcpy(&id, opt_.nccl_id, sizeof(id));
    NK(nccl().CommInitRank(&world_, world_n_, id, rank_));
    auto split = [&](ModelName m, ncclComm_t* out) {
      const std::vector<int>& g = plan_.cfg(m).devices;
      const int color = in(g, rank_) ? 1 : NCCL_SPLIT_NOCOLOR;
      NK(nccl().CommSplit(world_, color, rank_, out, nullptr));
      if (!in(g, rank_) || g.size() < 2) {  // nothing to all-reduce with
        if (*out) nccl().CommDestroy(*out);
        *out = nullptr;
      }
    };
    split(ModelName::Actor, &actor_comm_);
    split(ModelName::Critic, &critic_comm_);
  }
  opt_.nccl_id = nullptr;

  if (hosts_[0]) init_decoder(actor_, fixed(cfg_.actor, 0), rlhf_model_seed(cfg_.seed, 0), true, actor_comm_);
  if (hosts_[1]) init_decoder(critic_, fixed(cfg_.critic, 1), rlhf_model_seed(cfg_.seed, 1), true, critic_comm_);
  if (hosts_[2]) init_decoder(ref_, fixed(cfg_.actor, 0), rlhf_model_seed(cfg_.seed, 2), false);
  if (hosts_[3]) init_decoder(reward_, fixed(cfg_.critic, 1), rlhf_model_seed(cfg_.seed, 3), false);
  // shadows start from the trainers' initial weights (same seeds), then ParamSync
  if (hosts_[4]) init_decoder(shadow_actor_, fixed(cfg_.actor, 0), rlhf_model_seed(cfg_.seed, 0), false);
  if (hosts_[5]) init_decoder(shadow_critic_, fixed(cfg_.critic, 1), rlhf_model_seed(cfg_.seed, 1), false);

  // ---- activation arenas: the main one, plus a forward-only one for the second
  // stream of the Co-located Forward stage (Critic + Reward beside Actor + Ref)
  build_arena(ar_main_, hosts_[0] || hosts_[1]);
  if (tag_ == StrategyTag::Colocated) {
    // Critic-shaped arena for the second stream (Critic/Reward forwards, Critic training);
    // when it does not fit (long sequences, large models) the step stays single-stream
    try {
      build_arena(ar_side_, true, true);
      // keep room for the generation state allocated next (KV cache + decode buffers)
      const size_t kv = 2ull * cfg_.actor.n_layers * gen_B_ * S_ * cfg_.actor.d_model * 2;
      size_t free_b = 0, total_b = 0;
      CK(cudaMemGetInfo(&free_b, &total_b));
      if (free_b < kv + (4ull << 30)) throw DeviceError("second-stream arena leaves too little memory");
      CK(cudaStreamCreateWithFlags(&stream_side_, cudaStreamNonBlocking));
    } catch (const DeviceError&) {
      for (DevBuf* b : ar_side_.owned) delete b;
      ar_side_.owned.clear();
      cudaGetLastError();
      stream_side_ = nullptr;
    }
  }

  // ---- generation state (the generator: Actor or ShadowActor) -----------------
  if (hosts_[0] && tag_ != StrategyTag::Disaggregated) generator_ = &actor_;
  if (hosts_[4]) generator_ = &shadow_actor_;
  if (tag_ == StrategyTag::Interleaving2 && !hosts_[0]) generator_ = nullptr;
  if (generator_) {
    kv_.L = cfg_.actor.n_layers;
    kv_.B = gen_B_;
    kv_.H = cfg_.actor.n_heads;
    kv_.Smax = S_;
    kv_.hd = cfg_.actor.d_model / cfg_.actor.n_heads;
    const size_t kvb = static_cast<size_t>(kv_.L) * gen_B_ * kv_.H * kv_.Smax * kv_.hd * 2;
    kv_.k.alloc(kvb);
    kv_.v.alloc(kvb);
    const int ad = cfg_.actor.d_model;
    dec_x_.alloc(static_cast<size_t>(gen_B_) * ad * 4);
    dec_h_.alloc(static_cast<size_t>(gen_B_) * ad * 2);
    dec_qkv_.alloc(static_cast<size_t>(gen_B_) * 3 * ad * 2);
    dec_o_.alloc(static_cast<size_t>(gen_B_) * ad * 2);
    const bool glu = cfg_.actor.family == 1;  // SwiGLU: gate|up rows, then the gated product
    dec_f_.alloc(static_cast<size_t>(gen_B_) * cfg_.actor.d_ff * (glu ? 2 : 1) * 2);
    dec_act_.alloc(glu ? static_cast<size_t>(gen_B_) * cfg_.actor.d_ff * 2 : 16);
    dec_hf_.alloc(static_cast<size_t>(gen_B_) * ad * 2);
    dec_logits_.alloc(static_cast<size_t>(gen_B_) * cfg_.actor.vocab * 4);
    dec_top2_.alloc(static_cast<size_t>((cfg_.actor.vocab + 127) / 128) * gen_B_ * 16);
    argmax_ws_.alloc(static_cast<size_t>(gen_B_) * 64 * 4 * 4);
  }
  pos_.alloc(16);

  const size_t bs = static_cast<size_t>(Bcap_) * S_, br = static_cast<size_t>(Bcap_) * R_;
  tokens_.alloc(bs * 4);
  tok2_.alloc(bs * 4);
  pred_.alloc(bs * 4);
  margin_.alloc(bs * 4);
  prompt_stage_.alloc(static_cast<size_t>(Bg_) * P_ * 4);
  for (DevBuf* b : {&logp_old_, &logp_ref_, &values_, &rewards_, &adv_, &ret_, &logp_new_, &values_new_, &gbuf_, &gbuf2_,
                    &out2_})
    b->alloc(br * 4);
  score_.alloc(static_cast<size_t>(Bcap_) * 4);
  score2_.alloc(static_cast<size_t>(Bcap_) * 4);
  loss_.alloc(16);

  // global sample id of every row this rank holds (experience rows)
  sample_ids_.assign(static_cast<size_t>(Bcap_), -1);
  const int lo = std::min(rank_, partner_ < 0 ? rank_ : partner_), hi = std::max(rank_, partner_ < 0 ? rank_ : partner_);
  if (tag_ == StrategyTag::Colocated || tag_ == StrategyTag::Interleaving1) {
    for (int b = 0; b < Bg_; ++b) sample_ids_[b] = rank_ * Bg_ + b;
  } else {
    for (int b = 0; b < Bg_; ++b) {
      sample_ids_[b] = lo * Bg_ + b;
      sample_ids_[Bg_ + b] = hi * Bg_ + b;
    }
  }
  CK(cudaDeviceSynchronize());
}

Engine::~Engine() {
  if (decode_graph_) cudaGraphExecDestroy(decode_graph_);
  for (ncclComm_t c : {actor_comm_, critic_comm_, world_})
    if (c) nccl().CommDestroy(c);
  for (auto& e : ev_) cudaEventDestroy(e);
  if (stream_) cudaStreamDestroy(stream_);
  if (stream_side_) cudaStreamDestroy(stream_side_);
}

void Engine::allreduce_grads(Decoder& m, ncclComm_t comm) {
  if (!comm) return;
  if (m.sharded) {  // ZeRO-1: each rank only needs the summed gradient of its own shard
    NK(nccl().ReduceScatter(m.grad.p, m.grad.as<float>() + m.shard_off, static_cast<size_t>(m.shard), ncclFloat32,
                            ncclSum, comm, stream_));
    comm_bytes_ += 4.0 * static_cast<double>(m.npad - m.shard);
    return;
  }
  NK(nccl().AllReduce(m.grad.p, m.grad.p, static_cast<size_t>(m.n), ncclFloat32, ncclSum, comm, stream_));
  comm_bytes_ += 2.0 * 4.0 * m.n;
}

// Paired P2P exchange with the partner rank inside one NCCL group (sends and
// receives between a pair match in issue order per direction).
void Engine::p2p(const std::vector<std::pair<const void*, size_t>>& sends, const std::vector<std::pair<void*, size_t>>& recvs) {
  NK(nccl().GroupStart());
  for (const auto& [p, n] : sends) {
    NK(nccl().Send(p, n, ncclInt8, partner_, world_, stream_));
    comm_bytes_ += static_cast<double>(n);
  }
  for (const auto& [p, n] : recvs) NK(nccl().Recv(p, n, ncclInt8, partner_, world_, stream_));
  NK(nccl().GroupEnd());
}

// TrainFB over micro-batches of train_mb_ samples: each runs forward (activations saved),
// loss, backward, accumulating into the flat gradient; then one all-reduce and AdamW.
void Engine::train_actor(Decoder& m, int B, ncclComm_t comm) {
  const float denom = cfg_.loss_denominator > 0 ? cfg_.loss_denominator : static_cast<float>(B * R_);
  cudaMemsetAsync(m.grad.p, 0, static_cast<size_t>(m.n) * 4, stream_);
  for (int b0 = 0; b0 < B; b0 += train_mb_) train_actor_mb(m, b0, std::min(train_mb_, B - b0), denom);
  allreduce_grads(m, comm);
  adam(m, cfg_.lr_actor, comm);
}

void Engine::train_actor_mb(Decoder& m, int b0, int B, float denom) {
  const int d = m.a.d_model, V = m.a.vocab, BR = B * R_;
  const int32_t* tok = tokens_.as<int32_t>() + static_cast<size_t>(b0) * S_;
  const size_t r0 = static_cast<size_t>(b0) * R_;
  float* logp = logp_new_.as<float>() + r0;
  float* g = gbuf_.as<float>() + r0;
  forward(m, tok, B, S_, S_, true, nullptr);
  lm_logprobs(m, tok, B, logp, true);
  K(rlhf_ppo_actor_loss(logp, logp_old_.as<float>() + r0, adv_.as<float>() + r0, BR, cfg_.cliprange, denom, g,
                        loss_.as<float>(), stream_), 1);
  K(rlhf_logprob_bwd(arp_->logits, arp_->lse, g, BR, V, tok, S_, P_, R_, arp_->dz, stream_), 1);
  // dhf_resp = dz E ; dE += dz^T hf_resp
  rlhf_gemm_params p{};
  p.M = BR; p.N = d; p.K = V; p.batch = 1; p.batch_h = 1;
  p.A = arp_->dz; p.lda = V;
  p.B = m.T(m.head_id()); p.b_mn_major = 1; p.ldb = d;
  p.C = arp_->dhf_resp; p.c_f32 = 1; p.c_rs = d; p.c_cs = 1; p.alpha = 1.0f;
  gemm(p);
  rlhf_gemm_params q{};
  q.M = V; q.N = d; q.K = BR; q.batch = 1; q.batch_h = 1;
  q.A = arp_->dz; q.a_mn_major = 1; q.lda = V;
  q.B = arp_->hf_resp; q.b_mn_major = 1; q.ldb = d;
  q.C = m.G(m.head_id()); q.c_f32 = 1; q.c_rs = d; q.c_cs = 1; q.alpha = 1.0f; q.accumulate = 1;
  gemm(q);
  cudaMemsetAsync(arp_->dhf, 0, static_cast<size_t>(B) * S_ * d * 4, stream_);
  K(rlhf_scatter_rows_f32(arp_->dhf_resp, arp_->dhf, B, S_, R_, P_ - 1, d, stream_), 1);
  backward(m, tok, B, S_);
}

void Engine::train_critic(Decoder& m, int B, ncclComm_t comm) {
  const float denom = cfg_.loss_denominator > 0 ? cfg_.loss_denominator : static_cast<float>(B * R_);
  cudaMemsetAsync(m.grad.p, 0, static_cast<size_t>(m.n) * 4, stream_);
  for (int b0 = 0; b0 < B; b0 += train_mb_) train_critic_mb(m, b0, std::min(train_mb_, B - b0), denom);
  allreduce_grads(m, comm);
  adam(m, cfg_.lr_critic, comm);
}

void Engine::train_critic_mb(Decoder& m, int b0, int B, float denom) {
  const int d = m.a.d_model, BR = B * R_;
  const int32_t* tok = tokens_.as<int32_t>() + static_cast<size_t>(b0) * S_;
  const size_t r0 = static_cast<size_t>(b0) * R_;
  float* v = values_new_.as<float>() + r0;
  float* g = gbuf2_.as<float>() + r0;
  forward(m, tok, B, S_, S_, true, nullptr);
  K(rlhf_scalar_head(arp_->hf, m.T(RLHF_T_VHEAD), B, S_, R_, P_ - 1, d, v, stream_), 1);
  K(rlhf_ppo_critic_loss(v, values_.as<float>() + r0, ret_.as<float>() + r0, BR, cfg_.cliprange_value, denom, g,
                         loss_.as<float>() + 1, stream_), 1);
  cudaMemsetAsync(arp_->dhf, 0, static_cast<size_t>(B) * S_ * d * 4, stream_);
  K(rlhf_scalar_head_bwd(arp_->hf, m.T(RLHF_T_VHEAD), g, B, S_, R_, P_ - 1, d, arp_->dhf, m.G(RLHF_T_VHEAD), arp_->ws,
                         stream_), 2);
  backward(m, tok, B, S_);
}

// Scoring helpers on tokens `tok` [B, S] -> per-row outputs.
void Engine::score_logp(const Decoder& m, const int32_t* tok, int B, float* logp) {
  forward(m, tok, B, S_, S_, false, nullptr);
  lm_logprobs(m, tok, B, logp, false);
}
void Engine::score_values(const Decoder& m, const int32_t* tok, int B, float* values) {
  forward(m, tok, B, S_, S_, false, nullptr);
  K(rlhf_scalar_head(arp_->hf, m.T(RLHF_T_VHEAD), B, S_, R_, P_ - 1, m.a.d_model, values, stream_), 1);
}
void Engine::score_reward(const Decoder& m, const int32_t* tok, int B, float* score) {
  forward(m, tok, B, S_, S_, false, nullptr);
  K(rlhf_scalar_head(arp_->hf, m.T(RLHF_T_VHEAD), B, S_, 1, S_ - 1, m.a.d_model, score, stream_), 1);
}

// Activation arena: capacities = max over hosted models.  `trains` keeps every layer's
// saved activations and the backward buffers; a forward-only arena keeps one layer.
void Engine::build_arena(Arena& A, bool trains, bool critic_only) {
  A.B = Bcap_;
  A.S = S_;
  A.R = R_;
  for (const rlhf_arch* a : {&cfg_.actor, &cfg_.critic}) {
    if (critic_only && a == &cfg_.actor) continue;
    A.d = std::max(A.d, a->d_model);
    A.ff = std::max(A.ff, a->d_ff * (a->family == 1 ? 2 : 1));
    A.ffa = std::max(A.ffa, a->family == 1 ? a->d_ff : 0);
    A.H = std::max(A.H, a->n_heads);
    A.V = std::max(A.V, critic_only ? 1 : a->vocab);  // scalar heads only: no logits
    A.L = std::max(A.L, a->n_layers);
  }
  A.T = static_cast<int64_t>(Bcap_) * S_;
  A.Z = static_cast<int64_t>(Bcap_) * A.H;
  A.Ts = trains ? static_cast<int64_t>(train_mb_) * S_ : A.T;
  A.Zs = trains ? static_cast<int64_t>(train_mb_) * A.H : A.Z;
  auto mk = [&](size_t bytes) {
    DevBuf* b = new DevBuf(bytes);
    A.owned.push_back(b);
    return b->p;
  };
  const int64_t T = A.T, d = A.d, SS = static_cast<int64_t>(A.S) * A.S, BR = static_cast<int64_t>(Bcap_) * R_;
  const int64_t Ls = trains ? A.L : 1;  // layers of saved activations (inference-only ranks keep one)
  // per-layer saved activations: Ls slots of one training micro-batch (Ts rows), and at
  // least one slot of a whole Forward stage (T rows, layer buffers reused across layers)
  const int64_t Ts = A.Ts, Zs = A.Zs;
  auto cap = [&](int64_t slots, int64_t per_row, int64_t rows_s, int64_t rows_all) {
    return std::max(slots * rows_s, rows_all) * per_row;
  };
  A.xres = static_cast<float*>(mk(cap(2 * Ls + 1, d * 4, Ts, T)));
  A.mean = static_cast<float*>(mk(cap(2 * Ls + 1, 4, Ts, T)));
  A.rstd = static_cast<float*>(mk(cap(2 * Ls + 1, 4, Ts, T)));
  A.h1 = static_cast<uint16_t*>(mk(cap(Ls, d * 2, Ts, T)));
  A.qkv = static_cast<uint16_t*>(mk(cap(Ls, 3 * d * 2, Ts, T)));
  A.P = static_cast<uint16_t*>(mk(cap(Ls, SS * 2, Zs, A.Z)));
  A.o = static_cast<uint16_t*>(mk(cap(Ls, d * 2, Ts, T)));
  A.h2 = static_cast<uint16_t*>(mk(cap(Ls, d * 2, Ts, T)));
  A.f = static_cast<uint16_t*>(mk(cap(Ls, A.ff * 2, Ts, T)));
  A.hf = static_cast<uint16_t*>(mk(T * d * 2));
  A.act = static_cast<uint16_t*>(mk(A.ffa ? T * A.ffa * 2 : 16));
  A.scores = static_cast<float*>(mk(A.Z * SS * 4));
  A.dS = static_cast<uint16_t*>(mk(trains ? A.Z * SS * 2 : 16));
  A.hf_resp = static_cast<uint16_t*>(mk(BR * d * 2));
  A.logits = static_cast<float*>(mk(BR * A.V * 4));
  A.lse = static_cast<float*>(mk(BR * 4));
  A.dz = static_cast<uint16_t*>(mk(trains ? BR * A.V * 2 : 16));
  A.dhf_resp = static_cast<float*>(mk(trains ? BR * d * 4 : 16));
  A.dres = static_cast<float*>(mk(trains ? T * d * 4 : 16));
  A.dhf = static_cast<float*>(mk(trains ? T * d * 4 : 16));
  A.dh = static_cast<float*>(mk(trains ? T * d * 4 : 16));
  A.g = static_cast<uint16_t*>(mk(trains ? T * d * 2 : 16));
  A.dpre = static_cast<uint16_t*>(mk(trains ? T * A.ff * 2 : 16));
  A.dov = static_cast<uint16_t*>(mk(trains ? T * d * 2 : 16));
  A.dqkv = static_cast<uint16_t*>(mk(trains ? T * 3 * d * 2 : 16));
  A.ws_floats = std::max<size_t>(static_cast<size_t>((T + 31) / 32) * 2 * d, 64 * static_cast<size_t>(std::max<int64_t>(3 * d, A.ff)));
  A.ws = static_cast<float*>(mk(A.ws_floats * 4));
  A.gemm_ws_bytes = 64ull << 20;
  A.gemm_ws = static_cast<float*>(mk(A.gemm_ws_bytes));
  A.counters_len = 1 << 16;
  A.counters = static_cast<int*>(mk(A.counters_len * 4));

}

void Engine::gae(int B) {
  K(rlhf_gae(logp_old_.as<float>(), logp_ref_.as<float>(), values_.as<float>(), score_.as<float>(), B, R_, cfg_.kl_ctl,
             cfg_.clip_reward, cfg_.gamma, cfg_.lam, rewards_.as<float>(), adv_.as<float>(), ret_.as<float>(), stream_), 1);
}

// Put this rank's prompts [Bg, P] into rows [row0, row0+Bg) of tokens_.
void Engine::place_prompts(const int32_t* dev_prompts, int row0) {
  CK(cudaMemcpy2DAsync(tokens_.as<int32_t>() + static_cast<size_t>(row0) * S_, static_cast<size_t>(S_) * 4, dev_prompts,
                       static_cast<size_t>(P_) * 4, static_cast<size_t>(P_) * 4, Bg_, cudaMemcpyDeviceToDevice, stream_));
}

void Engine::step(const int32_t* prompts_host, rlhf_step_report* rep) {
  CK(cudaSetDevice(opt_.device));
  launches_ = 0;
  comm_bytes_ = 0;
  // this rank's prompt shard (global samples [rank*Bg, rank*Bg + Bg)) -> device
  std::vector<int32_t> pr(static_cast<size_t>(Bg_) * P_);
  for (int b = 0; b < Bg_; ++b)
    for (int t = 0; t < P_; ++t)
      pr[static_cast<size_t>(b) * P_ + t] =
          prompts_host ? prompts_host[static_cast<size_t>(b) * P_ + t]
                       : rlhf_prompt_token(cfg_.prompt_seed, b + cfg_.sample_offset, t, cfg_.actor.vocab);
  CK(cudaMemcpyAsync(prompt_stage_.p, pr.data(), pr.size() * 4, cudaMemcpyHostToDevice, stream_));
  cudaMemsetAsync(loss_.p, 0, 16, stream_);
  cudaEventRecord(ev_[0], stream_);  // device-resident inputs from here on
  cudaEventRecord(ev_[1], stream_);  // (prefill end; re-recorded by generate)

  const int Bg = Bg_;
  int32_t* tok = tokens_.as<int32_t>();
  const bool lower = partner_ < 0 || rank_ < partner_;
  switch (tag_) {
    case StrategyTag::Colocated: {
      place_prompts(prompt_stage_.as<int32_t>(), 0);
      generate(actor_, Bg, false);
      cudaEventRecord(ev_[2], stream_);
      // Forward x4 (workload.cpp:119 lists Actor, Critic, Ref, Reward; they are
      // independent): Critic + Reward on a second stream with their own arena, Actor +
      // Ref on the main stream, joined before the experience-buffer barrier
      if (stream_side_) {
        cudaEventRecord(ev_[6], stream_);
        CK(cudaStreamWaitEvent(stream_side_, ev_[6], 0));
        std::swap(stream_, stream_side_);
        arp_ = &ar_side_;
      }
      score_values(critic_, tok, Bg, values_.as<float>());
      score_reward(reward_, tok, Bg, score_.as<float>());
      if (stream_side_) {
        cudaEventRecord(ev_[7], stream_);
        std::swap(stream_, stream_side_);
        arp_ = &ar_main_;
      }
      score_logp(actor_, tok, Bg, logp_old_.as<float>());
      score_logp(ref_, tok, Bg, logp_ref_.as<float>());
      if (stream_side_) CK(cudaStreamWaitEvent(stream_, ev_[7], 0));
      cudaEventRecord(ev_[3], stream_);
      gae(Bg);
      // TrainFB(Actor) and TrainFB(Critic) are independent given the experience buffer:
      // the Critic trains on the second stream / arena
      if (stream_side_) {
        cudaEventRecord(ev_[6], stream_);
        CK(cudaStreamWaitEvent(stream_side_, ev_[6], 0));
        std::swap(stream_, stream_side_);
        arp_ = &ar_side_;
      }
      train_critic(critic_, Bg, critic_comm_);
      if (stream_side_) {
        cudaEventRecord(ev_[7], stream_);
        std::swap(stream_, stream_side_);
        arp_ = &ar_main_;
      }
      train_actor(actor_, Bg, actor_comm_);
      if (stream_side_) CK(cudaStreamWaitEvent(stream_, ev_[7], 0));
      cudaEventRecord(ev_[4], stream_);
      break;
    }
    case StrategyTag::Interleaving1: {
      place_prompts(prompt_stage_.as<int32_t>(), 0);
      generate(actor_, Bg, false);
      cudaEventRecord(ev_[2], stream_);
      score_logp(actor_, tok, Bg, logp_old_.as<float>());
      score_values(critic_, tok, Bg, values_.as<float>());
      // AllGather of (query, response) within the Ref|Reward pair (Alg. 1 line 8)
      int32_t* t2 = tok2_.as<int32_t>();
      const size_t sb = static_cast<size_t>(Bg) * S_ * 4;
      int32_t* mine = t2 + (lower ? 0 : static_cast<size_t>(Bg) * S_);
      int32_t* theirs = t2 + (lower ? static_cast<size_t>(Bg) * S_ : 0);
      CK(cudaMemcpyAsync(mine, tok, sb, cudaMemcpyDeviceToDevice, stream_));
      p2p({{tok, sb}}, {{theirs, sb}});
      const int own0 = lower ? 0 : Bg, oth0 = lower ? Bg : 0;
      if (hosts_[2]) {  // Ref side: logprobs of both shards; swap with the Reward side's scores
        score_logp(ref_, t2, 2 * Bg, out2_.as<float>());
        const size_t rb = static_cast<size_t>(Bg) * R_ * 4;
        CK(cudaMemcpyAsync(logp_ref_.p, out2_.as<float>() + static_cast<size_t>(own0) * R_, rb, cudaMemcpyDeviceToDevice,
                           stream_));
        p2p({{out2_.as<float>() + static_cast<size_t>(oth0) * R_, rb}}, {{score_.p, static_cast<size_t>(Bg) * 4}});
      } else {  // Reward side
        score_reward(reward_, t2, 2 * Bg, score2_.as<float>());
        CK(cudaMemcpyAsync(score_.p, score2_.as<float>() + own0, static_cast<size_t>(Bg) * 4, cudaMemcpyDeviceToDevice,
                           stream_));
        p2p({{score2_.as<float>() + oth0, static_cast<size_t>(Bg) * 4}}, {{logp_ref_.p, static_cast<size_t>(Bg) * R_ * 4}});
      }
      cudaEventRecord(ev_[3], stream_);
      gae(Bg);
      train_actor(actor_, Bg, actor_comm_);
      train_critic(critic_, Bg, critic_comm_);
      cudaEventRecord(ev_[4], stream_);
      break;
    }
    case StrategyTag::Interleaving2:
    case StrategyTag::Disaggregated: {
      const bool disagg = tag_ == StrategyTag::Disaggregated;
      // generator side: Actor ranks (I2) / inference ranks (disaggregated)
      const bool gen_side = disagg ? hosts_[4] : hosts_[0];
      const int B2 = 2 * Bg;
      const size_t rbytes = static_cast<size_t>(B2) * R_ * 4, tbytes = static_cast<size_t>(B2) * S_ * 4;
      if (gen_side) {
        place_prompts(prompt_stage_.as<int32_t>(), lower ? 0 : Bg);
        p2p({}, {{tok2_.p, static_cast<size_t>(Bg) * P_ * 4}});  // the partner's prompt shard
        place_prompts(tok2_.as<int32_t>(), lower ? Bg : 0);
        generate(*generator_, B2, false);
        cudaEventRecord(ev_[2], stream_);
        if (disagg) {
          score_logp(shadow_actor_, tok, B2, logp_old_.as<float>());
          score_values(shadow_critic_, tok, B2, values_.as<float>());
          score_logp(ref_, tok, B2, logp_ref_.as<float>());
          score_reward(reward_, tok, B2, score_.as<float>());
          // Send the experience to the training side (Alg. 2)
          p2p({{tok, tbytes}, {logp_old_.p, rbytes}, {logp_ref_.p, rbytes}, {values_.p, rbytes},
               {score_.p, static_cast<size_t>(B2) * 4}},
              {});
          cudaEventRecord(ev_[3], stream_);
          cudaEventRecord(ev_[4], stream_);
          // ParamSync: trained weights -> shadows, before the next Generation
          p2p({}, {{shadow_actor_.w.p, static_cast<size_t>(shadow_actor_.n) * 2},
                   {shadow_critic_.w.p, static_cast<size_t>(shadow_critic_.n) * 2}});
        } else {
          p2p({{tok, tbytes}}, {});
          score_logp(actor_, tok, B2, logp_old_.as<float>());
          score_logp(ref_, tok, B2, logp_ref_.as<float>());
          p2p({{logp_old_.p, rbytes}, {logp_ref_.p, rbytes}}, {{values_.p, rbytes}, {score_.p, static_cast<size_t>(B2) * 4}});
          cudaEventRecord(ev_[3], stream_);
          gae(B2);
          train_actor(actor_, B2, actor_comm_);
          cudaEventRecord(ev_[4], stream_);
        }
      } else {
        p2p({{prompt_stage_.p, static_cast<size_t>(Bg) * P_ * 4}}, {});
        cudaEventRecord(ev_[1], stream_);
        cudaEventRecord(ev_[2], stream_);
        if (disagg) {
          p2p({}, {{tok, tbytes}, {logp_old_.p, rbytes}, {logp_ref_.p, rbytes}, {values_.p, rbytes},
                   {score_.p, static_cast<size_t>(B2) * 4}});
          cudaEventRecord(ev_[3], stream_);
          gae(B2);
          train_actor(actor_, B2, actor_comm_);
          train_critic(critic_, B2, critic_comm_);
          cudaEventRecord(ev_[4], stream_);
          p2p({{actor_.w.p, static_cast<size_t>(actor_.n) * 2}, {critic_.w.p, static_cast<size_t>(critic_.n) * 2}}, {});
        } else {
          p2p({}, {{tok, tbytes}});
          score_values(critic_, tok, B2, values_.as<float>());
          score_reward(reward_, tok, B2, score_.as<float>());
          p2p({{values_.p, rbytes}, {score_.p, static_cast<size_t>(B2) * 4}}, {{logp_old_.p, rbytes}, {logp_ref_.p, rbytes}});
          cudaEventRecord(ev_[3], stream_);
          gae(B2);
          train_critic(critic_, B2, critic_comm_);
          cudaEventRecord(ev_[4], stream_);
        }
      }
      break;
    }
    default:
      throw ConfigError("strategy not executable: " + strategy_);
  }
  cudaEventRecord(ev_[5], stream_);
  float loss[2];
  CK(cudaMemcpyAsync(loss, loss_.p, 8, cudaMemcpyDeviceToHost, stream_));
  CK(cudaStreamSynchronize(stream_));

  auto sec = [&](int a, int b) {
    float t = 0;
    cudaEventElapsedTime(&t, ev_[a], ev_[b]);
    return static_cast<double>(t) * 1e-3;
  };
  std::memset(rep, 0, sizeof(*rep));
  rep->step_seconds = sec(0, 5);
  const double global_batch = cfg_.loss_denominator > 0 ? cfg_.loss_denominator / R_ : Bg_;
  rep->throughput_samples_per_sec = global_batch / rep->step_seconds;
  rep->stage_seconds[0] = sec(0, 2);
  rep->stage_seconds[1] = sec(2, 3);
  rep->stage_seconds[2] = sec(3, 4);
  rep->stage_seconds[3] = sec(4, 5);
  rep->prefill_seconds = sec(0, 1);
  rep->decode_seconds = sec(1, 2);
  const float denom = cfg_.loss_denominator > 0 ? cfg_.loss_denominator : static_cast<float>(Bg_ * R_);
  rep->actor_loss = loss[0] / denom;
  rep->critic_loss = 0.5 * loss[1] / denom;
  rep->comm_bytes_total = comm_bytes_;
  rep->gpu_launches = launches_;
}

size_t Engine::tensor_bytes(const std::string& name) const {
  const size_t br = static_cast<size_t>(Bcap_) * R_ * 4;
  static const std::map<std::string, int> kBR = {{"logp_old", 0}, {"logp_ref", 0}, {"values", 0}, {"rewards", 0},
                                                 {"advantages", 0}, {"returns", 0}, {"logp_new", 0}, {"values_new", 0}};
  if (kBR.count(name)) return br;
  if (name == "tokens" || name == "pred" || name == "margin") return static_cast<size_t>(Bcap_) * S_ * 4;
  if (name == "score") return static_cast<size_t>(Bcap_) * 4;
  if (name == "sample_ids") return static_cast<size_t>(Bcap_) * 4;
  auto flat = [](const Decoder& m, size_t e) { return static_cast<size_t>(m.n) * e; };
  if (name == "actor_grad") return flat(actor_, 4);
  if (name == "critic_grad") return flat(critic_, 4);
  if (name == "actor_master") return static_cast<size_t>(actor_.shard) * 4;  // this rank's slice under ZeRO-1
  if (name == "critic_master") return static_cast<size_t>(critic_.shard) * 4;
  if (name == "actor_params") return flat(actor_, 2);
  if (name == "critic_params") return flat(critic_, 2);
  if (name == "ref_params") return flat(ref_, 2);
  if (name == "reward_params") return flat(reward_, 2);
  if (name == "shadow_actor_params") return flat(shadow_actor_, 2);
  if (name == "shadow_critic_params") return flat(shadow_critic_, 2);
  return 0;
}

void Engine::read(const std::string& name, void* host, size_t bytes) {
  CK(cudaSetDevice(opt_.device));
  if (bytes != tensor_bytes(name) || bytes == 0) throw ConfigError("size mismatch (or tensor absent on this rank): " + name);
  if (name == "sample_ids") {
    std::memcpy(host, sample_ids_.data(), bytes);
    return;
  }
  const std::map<std::string, const DevBuf*> m = {
      {"tokens", &tokens_}, {"pred", &pred_}, {"margin", &margin_}, {"logp_old", &logp_old_}, {"logp_ref", &logp_ref_},
      {"values", &values_}, {"score", &score_}, {"rewards", &rewards_}, {"advantages", &adv_}, {"returns", &ret_},
      {"logp_new", &logp_new_}, {"values_new", &values_new_}, {"actor_grad", &actor_.grad},
      {"critic_grad", &critic_.grad}, {"actor_master", &actor_.master}, {"critic_master", &critic_.master},
      {"actor_params", &actor_.w}, {"critic_params", &critic_.w}, {"ref_params", &ref_.w}, {"reward_params", &reward_.w},
      {"shadow_actor_params", &shadow_actor_.w}, {"shadow_critic_params", &shadow_critic_.w}};
  auto it = m.find(name);
  if (it == m.end()) throw ConfigError("unknown tensor " + name);
  CK(cudaStreamSynchronize(stream_));
  CK(cudaMemcpy(host, it->second->p, bytes, cudaMemcpyDeviceToHost));
}

void Engine::greedy_check(const int32_t* tokens_host, int32_t* pred_host, float* margin_host) {
  CK(cudaSetDevice(opt_.device));
  if (!generator_) throw ConfigError("this rank does not generate");
  const int B = gen_B_;
  CK(cudaMemcpyAsync(tokens_.p, tokens_host, static_cast<size_t>(B) * S_ * 4, cudaMemcpyHostToDevice, stream_));
  cudaMemsetAsync(pred_.p, 0, static_cast<size_t>(B) * S_ * 4, stream_);
  generate(*generator_, B, true);
  std::vector<int32_t> pred(static_cast<size_t>(B) * S_);
  std::vector<float> mar(pred.size());
  CK(cudaStreamSynchronize(stream_));
  CK(cudaMemcpy(pred.data(), pred_.p, pred.size() * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(mar.data(), margin_.p, mar.size() * 4, cudaMemcpyDeviceToHost));
  for (int b = 0; b < B; ++b)
    for (int j = 0; j < R_; ++j) {
      pred_host[b * R_ + j] = pred[static_cast<size_t>(b) * S_ + P_ + j];
      margin_host[b * R_ + j] = mar[static_cast<size_t>(b) * S_ + P_ + j];
    }
}

}  // namespace flexrlhf

// ---- C-ABI ---------------------------------------------------------------------

using flexrlhf::Engine;

struct rlhf_engine {
  Engine* impl;
};

extern "C" int rlhf_nccl_unique_id(uint8_t out[128]) {
  try {
    ncclUniqueId id;
    if (flexrlhf::nccl().GetUniqueId(&id) != ncclSuccess) throw flexrlhf::DeviceError("ncclGetUniqueId failed");
    std::memcpy(out, &id, sizeof(id));
    return 0;
  } catch (const std::exception& ex) {
    return flexrlhf::capi_status(ex);
  }
}

extern "C" int rlhf_engine_create(const rlhf_ppo_config* cfg, const rlhf_engine_options* opt, rlhf_engine** out) {
  try {
    *out = nullptr;
    auto* e = new rlhf_engine{nullptr};
    try {
      e->impl = new Engine(*cfg, *opt);
    } catch (...) {
      delete e;
      throw;
    }
    *out = e;
    return 0;
  } catch (const std::exception& ex) {
    return flexrlhf::capi_status(ex);
  }
}

extern "C" void rlhf_engine_destroy(rlhf_engine* e) {
  if (!e) return;
  delete e->impl;
  delete e;
}

extern "C" int rlhf_engine_step(rlhf_engine* e, const int32_t* prompts_host, rlhf_step_report* rep) {
  try {
    e->impl->step(prompts_host, rep);
    return 0;
  } catch (const std::exception& ex) {
    return flexrlhf::capi_status(ex);
  }
}

extern "C" void* rlhf_engine_stream(rlhf_engine* e) { return e->impl->stream(); }

extern "C" size_t rlhf_engine_tensor_bytes(rlhf_engine* e, const char* name) { return e->impl->tensor_bytes(name); }

extern "C" int rlhf_engine_read(rlhf_engine* e, const char* name, void* host, size_t bytes) {
  try {
    e->impl->read(name, host, bytes);
    return 0;
  } catch (const std::exception& ex) {
    return flexrlhf::capi_status(ex);
  }
}

extern "C" int rlhf_engine_greedy_check(rlhf_engine* e, const int32_t* tokens_host, int32_t* pred_host,
                                        float* margin_host) {
  try {
    e->impl->greedy_check(tokens_host, pred_host, margin_host);
    return 0;
  } catch (const std::exception& ex) {
    return flexrlhf::capi_status(ex);
  }
}
