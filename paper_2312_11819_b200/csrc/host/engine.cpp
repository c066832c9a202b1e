// engine.cpp — the PPO iteration driver and its C-ABI (include/rlhf_engine.h).
//
// Walks the reference's one-iteration stage DAG (task_graph,
// /root/reference/proj/src/workload.cpp:109-175): Generation -> Forward for
// every scorer model -> experience-buffer barrier (GAE) -> TrainFB(Actor),
// TrainFB(Critic) -> (shadows) ParamSync.  Each stage is timed with CUDA events
// and reported in the reference's SimReport vocabulary (simulator.hpp:30-44).
// Data-parallel placements all-reduce gradients over NCCL (costmodel.hpp:59-74).
#include "engine.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>

#include "capi_util.hpp"
#include "nccl_dyn.hpp"
#include "flexrlhf/errors.hpp"

namespace flexrlhf {

#define CK(x)                                                                                    \
  do {                                                                                           \
    cudaError_t e_ = (x);                                                                        \
    if (e_ != cudaSuccess) throw DeviceError(std::string(#x) + ": " + cudaGetErrorString(e_));   \
  } while (0)
#define NK(x)                                                                                    \
  do {                                                                                           \
    ncclResult_t r_ = (x);                                                                       \
    if (r_ != ncclSuccess) throw DeviceError(std::string(#x) + ": " + nccl().GetErrorString(r_)); \
  } while (0)
#define K(call, n)                \
  do {                            \
    kcheck((call), #call);        \
    launches_ += (n);             \
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
    if (a->family != 0) throw ConfigError("only the OPT family is executable in this build");
    if (S > a->max_pos) throw ConfigError("prompt_len + gen_len exceeds max_pos");
    if (a->d_model % a->n_heads) throw ConfigError("d_model must divide by n_heads");
    const int hd = a->d_model / a->n_heads;
    if (hd != 64 && hd != 128) throw ConfigError("head_dim must be 64 or 128");
    if (a->d_model % 64 || a->d_ff % 64 || a->vocab % 8) throw ConfigError("d_model/d_ff must be multiples of 64, vocab of 8");
  }
  if (c.prompt_len % 8 || S % 8) throw ConfigError("prompt_len and prompt_len+gen_len must be multiples of 8");
}

}  // namespace

Engine::Engine(const rlhf_ppo_config& cfg, const rlhf_engine_options& opt) : cfg_(cfg), opt_(opt) {
  validate(cfg_);
  cfg_.actor.scalar_head = 0;
  cfg_.critic.scalar_head = 1;
  strategy_ = opt.strategy ? opt.strategy : "colocated";
  if (strategy_ != "colocated") throw ConfigError("strategy '" + strategy_ + "' is not executable in this build yet");
  opt_.strategy = nullptr;
  B_ = cfg_.batch;
  P_ = cfg_.prompt_len;
  R_ = cfg_.gen_len;
  S_ = P_ + R_;
  CK(cudaSetDevice(opt_.device));
  CK(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
  for (auto& e : ev_) CK(cudaEventCreate(&e));

  // Co-located placement (colocated_plan): every model on every
  // rank, data-parallel over the batch; a world communicator for the gradients.
  for (bool& h : hosts_) h = false;
  hosts_[static_cast<int>(ModelName::Actor)] = hosts_[static_cast<int>(ModelName::Critic)] = true;
  hosts_[static_cast<int>(ModelName::Ref)] = hosts_[static_cast<int>(ModelName::Reward)] = true;
  if (opt_.world_size > 1) {
    if (!opt_.nccl_id) throw ConfigError("world_size > 1 needs an NCCL unique id");
    ncclUniqueId id;
    std::memcpy(&id, opt_.nccl_id, sizeof(id));
    NK(nccl().CommInitRank(&world_, opt_.world_size, id, opt_.rank));
  }
  opt_.nccl_id = nullptr;

  init_decoder(actor_, fixed(cfg_.actor, 0), rlhf_model_seed(cfg_.seed, 0), true);
  init_decoder(critic_, fixed(cfg_.critic, 1), rlhf_model_seed(cfg_.seed, 1), true);
  init_decoder(ref_, fixed(cfg_.actor, 0), rlhf_model_seed(cfg_.seed, 2), false);
  init_decoder(reward_, fixed(cfg_.critic, 1), rlhf_model_seed(cfg_.seed, 3), false);

  // ---- activation arena: capacities = max over hosted models ----------------
  Arena& A = ar_;
  A.B = B_;
  A.S = S_;
  A.R = R_;
  for (const rlhf_arch* a : {&cfg_.actor, &cfg_.critic}) {
    A.d = std::max(A.d, a->d_model);
    A.ff = std::max(A.ff, a->d_ff);
    A.H = std::max(A.H, a->n_heads);
    A.V = std::max(A.V, a->vocab);
    A.L = std::max(A.L, a->n_layers);
  }
  A.T = static_cast<int64_t>(B_) * S_;
  A.Z = static_cast<int64_t>(B_) * A.H;
  auto mk = [&](size_t bytes) {
    DevBuf* b = new DevBuf(bytes);
    A.owned.push_back(b);
    return b->p;
  };
  const int64_t T = A.T, d = A.d, L = A.L, SS = static_cast<int64_t>(A.S) * A.S, BR = static_cast<int64_t>(B_) * R_;
  A.xres = static_cast<float*>(mk((2 * L + 1) * T * d * 4));
  A.mean = static_cast<float*>(mk((2 * L + 1) * T * 4));
  A.rstd = static_cast<float*>(mk((2 * L + 1) * T * 4));
  A.h1 = static_cast<uint16_t*>(mk(L * T * d * 2));
  A.qkv = static_cast<uint16_t*>(mk(L * T * 3 * d * 2));
  A.P = static_cast<uint16_t*>(mk(L * A.Z * SS * 2));
  A.o = static_cast<uint16_t*>(mk(L * T * d * 2));
  A.h2 = static_cast<uint16_t*>(mk(L * T * d * 2));
  A.f = static_cast<uint16_t*>(mk(L * T * A.ff * 2));
  A.hf = static_cast<uint16_t*>(mk(T * d * 2));
  A.scores = static_cast<float*>(mk(A.Z * SS * 4));
  A.dS = static_cast<uint16_t*>(mk(A.Z * SS * 2));
  A.hf_resp = static_cast<uint16_t*>(mk(BR * d * 2));
  A.logits = static_cast<float*>(mk(BR * A.V * 4));
  A.lse = static_cast<float*>(mk(BR * 4));
  A.dz = static_cast<uint16_t*>(mk(BR * A.V * 2));
  A.dhf_resp = static_cast<float*>(mk(BR * d * 4));
  A.dres = static_cast<float*>(mk(T * d * 4));
  A.dhf = static_cast<float*>(mk(T * d * 4));
  A.dh = static_cast<float*>(mk(T * d * 4));
  A.g = static_cast<uint16_t*>(mk(T * d * 2));
  A.dpre = static_cast<uint16_t*>(mk(T * A.ff * 2));
  A.dov = static_cast<uint16_t*>(mk(T * d * 2));
  A.dqkv = static_cast<uint16_t*>(mk(T * 3 * d * 2));
  A.ws_floats = std::max<size_t>(static_cast<size_t>((T + 31) / 32) * 2 * d, 64 * static_cast<size_t>(std::max<int64_t>(3 * d, A.ff)));
  A.ws = static_cast<float*>(mk(A.ws_floats * 4));
  A.gemm_ws_bytes = 64ull << 20;
  A.gemm_ws = static_cast<float*>(mk(A.gemm_ws_bytes));
  A.counters_len = 1 << 16;
  A.counters = static_cast<int*>(mk(A.counters_len * 4));

  // ---- generation state: Actor KV cache + decode-step buffers --------------
  kv_.L = cfg_.actor.n_layers;
  kv_.B = B_;
  kv_.H = cfg_.actor.n_heads;
  kv_.Smax = S_;
  kv_.hd = cfg_.actor.d_model / cfg_.actor.n_heads;
  const size_t kvb = static_cast<size_t>(kv_.L) * B_ * kv_.H * kv_.Smax * kv_.hd * 2;
  kv_.k.alloc(kvb);
  kv_.v.alloc(kvb);
  const int ad = cfg_.actor.d_model;
  dec_x_.alloc(static_cast<size_t>(B_) * ad * 4);
  dec_h_.alloc(static_cast<size_t>(B_) * ad * 2);
  dec_qkv_.alloc(static_cast<size_t>(B_) * 3 * ad * 2);
  dec_o_.alloc(static_cast<size_t>(B_) * ad * 2);
  dec_f_.alloc(static_cast<size_t>(B_) * cfg_.actor.d_ff * 2);
  dec_hf_.alloc(static_cast<size_t>(B_) * ad * 2);
  dec_logits_.alloc(static_cast<size_t>(B_) * cfg_.actor.vocab * 4);
  argmax_ws_.alloc(static_cast<size_t>(B_) * 64 * 4 * 4);
  pos_.alloc(16);

  const size_t bs = static_cast<size_t>(B_) * S_, br = static_cast<size_t>(B_) * R_;
  tokens_.alloc(bs * 4);
  pred_.alloc(bs * 4);
  margin_.alloc(bs * 4);
  for (DevBuf* b : {&logp_old_, &logp_ref_, &values_, &rewards_, &adv_, &ret_, &logp_new_, &values_new_, &gbuf_})
    b->alloc(br * 4);
  score_.alloc(static_cast<size_t>(B_) * 4);
  loss_.alloc(16);
  CK(cudaDeviceSynchronize());
}

Engine::~Engine() {
  if (decode_graph_) cudaGraphExecDestroy(decode_graph_);
  if (world_) nccl().CommDestroy(world_);
  for (auto& e : ev_) cudaEventDestroy(e);
  if (stream_) cudaStreamDestroy(stream_);
}

void Engine::allreduce_grads(Decoder& m, ncclComm_t comm) {
  if (!comm) return;
  NK(nccl().AllReduce(m.grad.p, m.grad.p, static_cast<size_t>(m.n), ncclFloat32, ncclSum, comm, stream_));
}

void Engine::train_actor() {
  Decoder& m = actor_;
  const int d = m.a.d_model, V = m.a.vocab, BR = B_ * R_;
  const float denom = cfg_.loss_denominator > 0 ? cfg_.loss_denominator : static_cast<float>(BR);
  cudaMemsetAsync(m.grad.p, 0, static_cast<size_t>(m.n) * 4, stream_);
  forward(m, tokens_.as<int32_t>(), B_, S_, S_, true, nullptr);
  lm_logprobs(m, tokens_.as<int32_t>(), B_, logp_new_.as<float>(), true);
  K(rlhf_ppo_actor_loss(logp_new_.as<float>(), logp_old_.as<float>(), adv_.as<float>(), BR, cfg_.cliprange, denom,
                        gbuf_.as<float>(), loss_.as<float>(), stream_), 1);
  K(rlhf_logprob_bwd(ar_.logits, ar_.lse, gbuf_.as<float>(), BR, V, tokens_.as<int32_t>(), S_, P_, R_, ar_.dz, stream_), 1);
  // dhf_resp = dz E ; dE += dz^T hf_resp
  rlhf_gemm_params p{};
  p.M = BR; p.N = d; p.K = V; p.batch = 1; p.batch_h = 1;
  p.A = ar_.dz; p.lda = V;
  p.B = m.T(RLHF_T_TOK_EMB); p.b_mn_major = 1; p.ldb = d;
  p.C = ar_.dhf_resp; p.c_f32 = 1; p.c_rs = d; p.c_cs = 1; p.alpha = 1.0f;
  gemm(p);
  rlhf_gemm_params q{};
  q.M = V; q.N = d; q.K = BR; q.batch = 1; q.batch_h = 1;
  q.A = ar_.dz; q.a_mn_major = 1; q.lda = V;
  q.B = ar_.hf_resp; q.b_mn_major = 1; q.ldb = d;
  q.C = m.G(RLHF_T_TOK_EMB); q.c_f32 = 1; q.c_rs = d; q.c_cs = 1; q.alpha = 1.0f; q.accumulate = 1;
  gemm(q);
  cudaMemsetAsync(ar_.dhf, 0, static_cast<size_t>(B_) * S_ * d * 4, stream_);
  K(rlhf_scatter_rows_f32(ar_.dhf_resp, ar_.dhf, B_, S_, R_, P_ - 1, d, stream_), 1);
  backward(m, tokens_.as<int32_t>(), B_, S_);
  allreduce_grads(m, world_);
  adam(m, cfg_.lr_actor);
}

void Engine::train_critic() {
  Decoder& m = critic_;
  const int d = m.a.d_model, BR = B_ * R_;
  const float denom = cfg_.loss_denominator > 0 ? cfg_.loss_denominator : static_cast<float>(BR);
  cudaMemsetAsync(m.grad.p, 0, static_cast<size_t>(m.n) * 4, stream_);
  forward(m, tokens_.as<int32_t>(), B_, S_, S_, true, nullptr);
  K(rlhf_scalar_head(ar_.hf, m.T(RLHF_T_VHEAD), B_, S_, R_, P_ - 1, d, values_new_.as<float>(), stream_), 1);
  K(rlhf_ppo_critic_loss(values_new_.as<float>(), values_.as<float>(), ret_.as<float>(), BR, cfg_.cliprange_value, denom,
                         gbuf_.as<float>(), loss_.as<float>() + 1, stream_), 1);
  cudaMemsetAsync(ar_.dhf, 0, static_cast<size_t>(B_) * S_ * d * 4, stream_);
  K(rlhf_scalar_head_bwd(ar_.hf, m.T(RLHF_T_VHEAD), gbuf_.as<float>(), B_, S_, R_, P_ - 1, d, ar_.dhf, m.G(RLHF_T_VHEAD),
                         ar_.ws, stream_), 2);
  backward(m, tokens_.as<int32_t>(), B_, S_);
  allreduce_grads(m, world_);
  adam(m, cfg_.lr_critic);
}

void Engine::step(const int32_t* prompts_host, rlhf_step_report* rep) {
  CK(cudaSetDevice(opt_.device));
  launches_ = 0;
  // prompts -> tokens[:, :P]
  std::vector<int32_t> tok(static_cast<size_t>(B_) * S_, 0);
  for (int b = 0; b < B_; ++b)
    for (int t = 0; t < P_; ++t)
      tok[static_cast<size_t>(b) * S_ + t] =
          prompts_host ? prompts_host[static_cast<size_t>(b) * P_ + t]
                       : rlhf_prompt_token(cfg_.prompt_seed, b + cfg_.sample_offset, t, cfg_.actor.vocab);
  CK(cudaMemcpyAsync(tokens_.p, tok.data(), tok.size() * 4, cudaMemcpyHostToDevice, stream_));
  cudaMemsetAsync(loss_.p, 0, 16, stream_);
  cudaEventRecord(ev_[0], stream_);  // device-resident inputs from here on

  // ---- Generation: Actor.generate(Query) (workload.cpp:148) ----------------
  generate(actor_, B_, false);
  cudaEventRecord(ev_[2], stream_);
  // ---- Forward x4 in the reference's order (workload.cpp:119) -------------
  forward(actor_, tokens_.as<int32_t>(), B_, S_, S_, false, nullptr);
  lm_logprobs(actor_, tokens_.as<int32_t>(), B_, logp_old_.as<float>(), false);
  forward(critic_, tokens_.as<int32_t>(), B_, S_, S_, false, nullptr);
  K(rlhf_scalar_head(ar_.hf, critic_.T(RLHF_T_VHEAD), B_, S_, R_, P_ - 1, critic_.a.d_model, values_.as<float>(), stream_), 1);
  forward(ref_, tokens_.as<int32_t>(), B_, S_, S_, false, nullptr);
  lm_logprobs(ref_, tokens_.as<int32_t>(), B_, logp_ref_.as<float>(), false);
  forward(reward_, tokens_.as<int32_t>(), B_, S_, S_, false, nullptr);
  K(rlhf_scalar_head(ar_.hf, reward_.T(RLHF_T_VHEAD), B_, S_, 1, S_ - 1, reward_.a.d_model, score_.as<float>(), stream_), 1);
  cudaEventRecord(ev_[3], stream_);
  // ---- Experience buffer barrier: rewards + GAE (workload.cpp:153-163) ----
  K(rlhf_gae(logp_old_.as<float>(), logp_ref_.as<float>(), values_.as<float>(), score_.as<float>(), B_, R_, cfg_.kl_ctl,
             cfg_.clip_reward, cfg_.gamma, cfg_.lam, rewards_.as<float>(), adv_.as<float>(), ret_.as<float>(), stream_), 1);
  // ---- TrainFB(Actor), TrainFB(Critic) -------------------------------------
  train_actor();
  train_critic();
  cudaEventRecord(ev_[4], stream_);
  cudaEventRecord(ev_[5], stream_);  // no ParamSync under Co-located
  float loss[2];
  CK(cudaMemcpyAsync(loss, loss_.p, 8, cudaMemcpyDeviceToHost, stream_));
  CK(cudaStreamSynchronize(stream_));

  auto ms = [&](int a, int b) {
    float t = 0;
    cudaEventElapsedTime(&t, ev_[a], ev_[b]);
    return static_cast<double>(t) * 1e-3;
  };
  std::memset(rep, 0, sizeof(*rep));
  rep->step_seconds = ms(0, 5);
  const double global_batch = cfg_.loss_denominator > 0 ? cfg_.loss_denominator / R_ : B_;
  rep->throughput_samples_per_sec = global_batch / rep->step_seconds;
  rep->stage_seconds[0] = ms(0, 2);
  rep->stage_seconds[1] = ms(2, 3);
  rep->stage_seconds[2] = ms(3, 4);
  rep->stage_seconds[3] = ms(4, 5);
  rep->prefill_seconds = ms(0, 1);
  rep->decode_seconds = ms(1, 2);
  const float denom = cfg_.loss_denominator > 0 ? cfg_.loss_denominator : static_cast<float>(B_ * R_);
  rep->actor_loss = loss[0] / denom;
  rep->critic_loss = 0.5 * loss[1] / denom;
  rep->comm_bytes_total = world_ ? 4.0 * (actor_.n + critic_.n) : 0.0;
  rep->gpu_launches = launches_;
  last_losses_[0] = rep->actor_loss;
  last_losses_[1] = rep->critic_loss;
}

size_t Engine::tensor_bytes(const std::string& name) const {
  const size_t br = static_cast<size_t>(B_) * R_ * 4;
  static const std::map<std::string, int> kBR = {{"logp_old", 0}, {"logp_ref", 0}, {"values", 0}, {"rewards", 0},
                                                 {"advantages", 0}, {"returns", 0}, {"logp_new", 0}, {"values_new", 0}};
  if (kBR.count(name)) return br;
  if (name == "tokens" || name == "pred" || name == "margin") return static_cast<size_t>(B_) * S_ * 4;
  if (name == "score") return static_cast<size_t>(B_) * 4;
  if (name == "actor_grad" || name == "actor_master") return static_cast<size_t>(actor_.n) * 4;
  if (name == "critic_grad" || name == "critic_master") return static_cast<size_t>(critic_.n) * 4;
  if (name == "actor_params") return static_cast<size_t>(actor_.n) * 2;
  if (name == "critic_params") return static_cast<size_t>(critic_.n) * 2;
  if (name == "ref_params") return static_cast<size_t>(ref_.n) * 2;
  if (name == "reward_params") return static_cast<size_t>(reward_.n) * 2;
  return 0;
}

void Engine::read(const std::string& name, void* host, size_t bytes) {
  CK(cudaSetDevice(opt_.device));
  const std::map<std::string, const DevBuf*> m = {
      {"tokens", &tokens_}, {"pred", &pred_}, {"margin", &margin_}, {"logp_old", &logp_old_}, {"logp_ref", &logp_ref_},
      {"values", &values_}, {"score", &score_}, {"rewards", &rewards_}, {"advantages", &adv_}, {"returns", &ret_},
      {"logp_new", &logp_new_}, {"values_new", &values_new_}, {"actor_grad", &actor_.grad},
      {"critic_grad", &critic_.grad}, {"actor_master", &actor_.master}, {"critic_master", &critic_.master},
      {"actor_params", &actor_.w}, {"critic_params", &critic_.w}, {"ref_params", &ref_.w}, {"reward_params", &reward_.w}};
  auto it = m.find(name);
  if (it == m.end()) throw ConfigError("unknown tensor " + name);
  if (bytes != tensor_bytes(name)) throw ConfigError("size mismatch reading " + name);
  CK(cudaStreamSynchronize(stream_));
  CK(cudaMemcpy(host, it->second->p, bytes, cudaMemcpyDeviceToHost));
}

void Engine::greedy_check(const int32_t* tokens_host, int32_t* pred_host, float* margin_host) {
  CK(cudaSetDevice(opt_.device));
  CK(cudaMemcpyAsync(tokens_.p, tokens_host, static_cast<size_t>(B_) * S_ * 4, cudaMemcpyHostToDevice, stream_));
  cudaMemsetAsync(pred_.p, 0, static_cast<size_t>(B_) * S_ * 4, stream_);
  generate(actor_, B_, true);
  std::vector<int32_t> pred(static_cast<size_t>(B_) * S_);
  std::vector<float> mar(pred.size());
  CK(cudaStreamSynchronize(stream_));
  CK(cudaMemcpy(pred.data(), pred_.p, pred.size() * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(mar.data(), margin_.p, mar.size() * 4, cudaMemcpyDeviceToHost));
  for (int b = 0; b < B_; ++b)
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
