// engine.cpp — the PPO iteration executor and its C-ABI (include/rlhf_engine.h).
//
// The executor walks an ExecPlan (execplan.hpp): the reference's one-iteration stage DAG
// (task_graph, /root/reference/proj/src/workload.cpp:109-175 -- rollout_nums x
// micro_batches of Generation -> Forward per scorer, the experience-buffer barrier,
// ppo_epochs x micro_batches of TrainFB, ParamSync + Barrier under shadows) interleaved
// with the exchanges the placement's comm schedule induces (derive_comm_schedule,
// placement.hpp:101-102).  Each step runs only on the ranks that take
// part in it; every rank walks the same list, so NCCL calls pair up.
//
// Streams ("lanes"): 0 main compute, 1 side compute (the Critic-shaped models on ranks
// that also host the Actor-shaped ones, with their own activation arena), 2 comm (every
// NCCL call and every row exchange, so no two collectives ever run concurrently).  A step
// waits only for the events of the DAG steps it depends on that ran on another lane of
// this rank; cross-rank ordering is carried by the exchanges themselves.  Every executed
// interval is bracketed by CUDA events and reported in SimReport's vocabulary
// (simulator.hpp:18-44): per-stage seconds with compute-lane attribution, busy time,
// bubble fraction, the event list.
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

constexpr int kEvExperience = 6, kEvAdam = 7;

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

bool actor_shaped(ModelName m) { return m == ModelName::Actor || m == ModelName::Ref || m == ModelName::ShadowActor; }

size_t field_row_bytes(Field f, int S, int R) {
  switch (f) {
    case Field::Prompt:
    case Field::Tokens: return static_cast<size_t>(S) * 4;
    case Field::Score: return 4;
    default: return static_cast<size_t>(R) * 4;
  }
}

}  // namespace

void* RowBufs::field(Field f) const {
  switch (f) {
    case Field::Prompt:
    case Field::Tokens: return tokens.p;
    case Field::LogpOld: return logp_old.p;
    case Field::LogpRef: return logp_ref.p;
    case Field::Values: return values.p;
    case Field::Score: return score.p;
  }
  return nullptr;
}

Decoder* Engine::model(ModelName m) {
  switch (m) {
    case ModelName::Actor: return &actor_;
    case ModelName::Critic: return &critic_;
    case ModelName::Ref: return &ref_;
    case ModelName::Reward: return &reward_;
    case ModelName::ShadowActor: return &shadow_actor_;
    case ModelName::ShadowCritic: return &shadow_critic_;
  }
  return nullptr;
}

int Engine::lane_of(ModelName m) const { return side_ && !actor_shaped(m) ? 1 : 0; }

void Engine::use_lane(int l) {
  cur_lane_ = l;
  stream_ = lane_[l];
  arp_ = l == 1 ? &ar_side_ : &ar_main_;
}

cudaEvent_t Engine::take_event() {
  if (ev_next_ == ev_pool_.size()) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    ev_pool_.push_back(e);
  }
  return ev_pool_[ev_next_++];
}

Engine::Engine(const rlhf_ppo_config& cfg, const rlhf_engine_options& opt) : cfg_(cfg), opt_(opt) {
  validate(cfg_);
  if (opt_.zero_stage < 0 || opt_.zero_stage > 3) throw ConfigError("zero_stage must be 0..3");
  cfg_.actor.scalar_head = 0;
  cfg_.critic.scalar_head = 1;
  strategy_ = opt.strategy ? opt.strategy : "colocated";
  opt_.strategy = nullptr;
  rank_ = opt_.rank;
  world_n_ = std::max(1, opt_.world_size);
  if (rank_ < 0 || rank_ >= world_n_) throw ConfigError("rank outside [0, world_size)");
  Bg_ = cfg_.batch;
  P_ = cfg_.prompt_len;
  R_ = cfg_.gen_len;
  S_ = P_ + R_;

  // ---- the executed plan: placement, task DAG, comm schedule, sample ownership ----
  {
    StrategyConfig sc;
    sc.name = strategy_;
    sc.zero_level = opt_.zero_stage;
    sc.inference_ratio = opt_.inference_ratio > 0 ? opt_.inference_ratio : 0.5;
    sc.tp_gen = opt_.tp_gen > 0 ? opt_.tp_gen : 1;
    const ModelName order[4] = {ModelName::Actor, ModelName::Critic, ModelName::Ref, ModelName::Reward};
    for (int i = 0; i < 4; ++i)
      if (opt_.ratios[i] > 0) sc.ratios.push_back({order[i], opt_.ratios[i]});
    ModelSizes sz;
    sz.actor = sz.ref = static_cast<double>(rlhf_param_total(&cfg_.actor));
    sz.critic = sz.reward = static_cast<double>(rlhf_param_total(&cfg_.critic));
    xp_ = build_exec_plan(sc, world_n_, Bg_, P_, R_, std::max(1, opt_.micro_batches), std::max(1, opt_.rollout_nums),
                          std::max(1, opt_.ppo_epochs), sz);
    tag_ = xp_.tag;
    for (int m = 0; m < 6; ++m) hosts_[m] = xp_.hosts(rank_, static_cast<ModelName>(m));
  }
  if (opt_.zero_stage == 3 && hosts_[0] && xp_.generator == ModelName::Actor)
    throw ConfigError("ZeRO-3 shards the trainers' weights per layer: the generating Actor needs them whole every "
                      "decode step (use the Disaggregated placement, whose shadow generates, or zero_stage <= 2)");
  int train_per = 0;
  for (int m = 0; m < 6; ++m) {
    if (!hosts_[m]) continue;
    const int per = xp_.sets[xp_.set_of[m]].per;
    Bcap_ = std::max(Bcap_, per);
    if (m <= 1) train_per = std::max(train_per, per);
  }
  Bcap_ = std::max(Bcap_, 1);
  gen_B_ = xp_.hosts(rank_, xp_.generator) ? xp_.sets[xp_.set_of[static_cast<int>(xp_.generator)]].per : 0;
  train_mb_ = std::max(1, opt_.train_micro_batch > 0 ? std::min(opt_.train_micro_batch, std::max(1, train_per))
                                                      : train_per);

  CK(cudaSetDevice(opt_.device));
  for (auto& l : lane_) CK(cudaStreamCreateWithFlags(&l, cudaStreamNonBlocking));
  use_lane(0);
  CK(cudaEventCreate(&ev_begin_));
  CK(cudaEventCreate(&ev_end_));

  // ---- communicators: world, the data-parallel group of each trained model, ParamSync pairs
  if (world_n_ > 1) {
    if (!opt_.nccl_id) throw ConfigError("world_size > 1 needs an NCCL unique id");
    ncclUniqueId id;
    std::memcpy(&id, opt_.nccl_id, sizeof(id));
    NK(nccl().CommInitRank(&world_, world_n_, id, rank_));
    auto split = [&](ModelName m, ncclComm_t* out) {
      *out = nullptr;
      if (!xp_.plan.has(m)) {  // every rank takes part in every split (collective)
        ncclComm_t c = nullptr;
        NK(nccl().CommSplit(world_, NCCL_SPLIT_NOCOLOR, rank_, &c, nullptr));
        return;
      }
      const std::vector<int>& g = xp_.plan.cfg(m).devices;
      const bool member = std::find(g.begin(), g.end(), rank_) != g.end();
      NK(nccl().CommSplit(world_, member ? 1 : NCCL_SPLIT_NOCOLOR, rank_, out, nullptr));
      if (!member || g.size() < 2) {  // nothing to reduce with
        if (*out) nccl().CommDestroy(*out);
        *out = nullptr;
      }
    };
    split(ModelName::Actor, &actor_comm_);
    split(ModelName::Critic, &critic_comm_);
    // ParamSync (workload.cpp:164-172): shadow member j receives from trainer member
    // j % |trainers| by broadcast over the {trainer, its shadows} communicator
    const std::pair<ModelName, ModelName> pairs[2] = {{ModelName::Actor, ModelName::ShadowActor},
                                                      {ModelName::Critic, ModelName::ShadowCritic}};
    for (int k = 0; k < 2; ++k) {
      const auto [src, dst] = pairs[k];
      int color = NCCL_SPLIT_NOCOLOR, key = rank_;
      if (xp_.plan.has(dst) && xp_.plan.has(src)) {
        const std::vector<int>& tg = xp_.plan.cfg(src).devices;
        const std::vector<int>& sg = xp_.plan.cfg(dst).devices;
        for (size_t i = 0; i < tg.size(); ++i)
          if (tg[i] == rank_) color = static_cast<int>(i), key = 0;
        for (size_t j = 0; j < sg.size(); ++j)
          if (sg[j] == rank_) color = static_cast<int>(j % tg.size()), key = 1 + static_cast<int>(j);
      }
      NK(nccl().CommSplit(world_, color, key, &sync_comm_[k], nullptr));
      sync_root_[k] = 0;  // the trainer has the lowest key
    }
  }
  opt_.nccl_id = nullptr;

  if (hosts_[0]) init_decoder(actor_, fixed(cfg_.actor, 0), rlhf_model_seed(cfg_.seed, 0), true, actor_comm_);
  if (hosts_[1]) init_decoder(critic_, fixed(cfg_.critic, 1), rlhf_model_seed(cfg_.seed, 1), true, critic_comm_);
  if (hosts_[2]) init_decoder(ref_, fixed(cfg_.actor, 0), rlhf_model_seed(cfg_.seed, 2), false);
  if (hosts_[3]) init_decoder(reward_, fixed(cfg_.critic, 1), rlhf_model_seed(cfg_.seed, 3), false);
  // shadows start from the trainers' initial weights (same seeds), then ParamSync
  if (hosts_[4]) init_decoder(shadow_actor_, fixed(cfg_.actor, 0), rlhf_model_seed(cfg_.seed, 0), false);
  if (hosts_[5]) init_decoder(shadow_critic_, fixed(cfg_.critic, 1), rlhf_model_seed(cfg_.seed, 1), false);

  // ---- activation arenas: main lane, plus a Critic-shaped one for the side lane when this
  // rank hosts both an Actor-shaped and a Critic-shaped model and it fits
  const bool trains = hosts_[0] || hosts_[1];
  build_arena(ar_main_, trains);
  const bool a_shaped = hosts_[0] || hosts_[2] || hosts_[4], c_shaped = hosts_[1] || hosts_[3] || hosts_[5];
  if (a_shaped && c_shaped) {
    try {
      build_arena(ar_side_, hosts_[1], true);
      // keep room for the generation state allocated next (KV cache + decode buffers)
      const size_t kv = 2ull * cfg_.actor.n_layers * std::max(gen_B_, 1) * S_ * cfg_.actor.d_model * 2;
      size_t free_b = 0, total_b = 0;
      CK(cudaMemGetInfo(&free_b, &total_b));
      // the side lane is a speed-up, not a necessity: keep a quarter of the device free for
      // memory-bound placements (e.g. Disaggregated 7B trainers), which then run one lane
      if (free_b < kv + (4ull << 30) || free_b < total_b / 4)
        throw InfeasibleError("side-lane arena leaves too little memory");
      side_ = true;
    } catch (const InfeasibleError&) {  // the step stays on one compute lane
      for (DevBuf* b : ar_side_.owned) delete b;
      ar_side_.owned.clear();
      cudaGetLastError();
      side_ = false;
    }
  }

  // ---- epoch-0 forward reuse: the experience Forward of a trained model runs with the training
  // forward (activations saved, LM-head logits kept) and its TrainFB of PPO epoch 0 -- same
  // weights, same tokens, so the same activations -- backpropagates through them instead of
  // recomputing the forward.  Needs the Forward block to be the whole TrainFB chunk (one
  // rollout, one micro-batch, train chunk >= block) and an arena of its own per trained model
  // (RLHF_REUSE_FWD=0 disables).
  {
    static const bool env = [] { const char* e = getenv("RLHF_REUSE_FWD"); return !e || atoi(e) != 0; }();
    const bool shape_ok = env && xp_.rollouts == 1 && xp_.M == 1;
    for (int mi : {0, 1}) {
      const ModelName mn = static_cast<ModelName>(mi);
      if (!shape_ok || !hosts_[mi]) continue;
      bool scores = false;  // does this rank run the model's experience Forward?
      for (const StageTask& t : xp_.tasks) scores |= t.kind == TaskKind::Forward && t.model == mn;
      const int per = xp_.sets[xp_.set_of[mi]].per;
      const bool own_arena = side_ || !(hosts_[0] && hosts_[1]);
      reuse_fwd_[mi] = scores && own_arena && train_mb_ >= per;
    }
  }

  // ---- generation state (the generator: Actor or ShadowActor) ----
  if (gen_B_ > 0) generator_ = model(xp_.generator);
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
    for (DevBuf& b : dec_st_) b.alloc(static_cast<size_t>(512) * std::min(gen_B_, 64) * 2 * 4);
    gen_tok_.alloc(static_cast<size_t>(gen_B_) * S_ * 4);
    pred_.alloc(static_cast<size_t>(gen_B_) * S_ * 4);
    margin_.alloc(static_cast<size_t>(gen_B_) * S_ * 4);
  }
  pos_.alloc(16);  // [0] decode position, [1] the tile-merge kernel's ticket (must start at 0)
  CK(cudaMemset(pos_.p, 0, 16));
  loss_.alloc(16);

  // ---- row sets this rank belongs to; home prompt rows ----
  rs_.reset(new RowBufs[xp_.sets.size()]);
  for (size_t s = 0; s < xp_.sets.size(); ++s) {
    if (xp_.member_index(static_cast<int>(s), rank_) < 0) continue;
    RowBufs& b = rs_[s];
    b.rows = xp_.sets[s].rows;
    const size_t rr = static_cast<size_t>(b.rows) * R_ * 4;
    b.tokens.alloc(static_cast<size_t>(b.rows) * S_ * 4);
    b.logp_old.alloc(rr);
    b.logp_ref.alloc(rr);
    b.values.alloc(rr);
    b.score.alloc(static_cast<size_t>(b.rows) * 4);
    b.trainer = (hosts_[0] && xp_.set_of[0] == static_cast<int>(s)) || (hosts_[1] && xp_.set_of[1] == static_cast<int>(s));
    if (b.trainer)
      for (DevBuf* d : {&b.rewards, &b.adv, &b.ret, &b.logp_new, &b.values_new, &b.gbuf, &b.gbuf2}) d->alloc(rr);
  }
  home_.alloc(static_cast<size_t>(xp_.rollouts) * Bg_ * S_ * 4);

  // ---- per-step dependencies (indices into xp_.steps; rank-independent) ----
  const int ns = static_cast<int>(xp_.steps.size());
  deps_.assign(ns, {});
  step_lane_.assign(ns, -1);
  step_done_.resize(ns);
  for (auto& e : step_done_) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  std::map<std::pair<int, int>, int> gen_of, before_of;
  std::map<std::pair<int, int>, std::vector<int>> fwds_of;
  std::map<std::pair<int, int>, int> prompt_of;
  std::vector<int> all_fwd, all_after, all_exp;
  std::map<std::pair<int, int>, std::vector<int>> train_of;  // (model, epoch)
  std::map<std::pair<int, int>, int> opt_of;
  for (int i = 0; i < ns; ++i) {
    const ExecStep& s = xp_.steps[i];
    const auto key = std::make_pair(s.rollout, s.mb);
    std::vector<int>& d = deps_[i];
    if (s.kind == StepKind::Exchange) {
      const bool prompt = !s.moves.empty() && s.moves[0].field == Field::Prompt;
      if (prompt) {
        prompt_of[key] = i;
      } else if (s.attach == AttachKind::Before) {
        d.push_back(gen_of[key]);
        before_of[key] = i;
      } else {
        d.push_back(gen_of[key]);
        d.insert(d.end(), fwds_of[key].begin(), fwds_of[key].end());
        all_after.push_back(i);
      }
      continue;
    }
    if (s.kind == StepKind::Experience) {
      d = all_fwd;
      d.insert(d.end(), all_after.begin(), all_after.end());
      for (auto& [k, g] : gen_of) d.push_back(g);
      all_exp.push_back(i);
      continue;
    }
    if (s.kind == StepKind::OptimizerStep) {
      d = train_of[{static_cast<int>(s.model), s.epoch}];
      opt_of[{static_cast<int>(s.model), s.epoch}] = i;
      continue;
    }
    const StageTask& t = xp_.tasks[s.task];
    switch (t.kind) {
      case TaskKind::Generation:
        if (prompt_of.count(key)) d.push_back(prompt_of[key]);
        gen_of[key] = i;
        break;
      case TaskKind::Forward:
        d.push_back(gen_of[key]);
        if (before_of.count(key)) d.push_back(before_of[key]);
        fwds_of[key].push_back(i);
        all_fwd.push_back(i);
        break;
      case TaskKind::TrainFB:
        d = all_exp;
        if (t.epoch_index > 0 && opt_of.count({static_cast<int>(t.model), t.epoch_index - 1}))
          d.push_back(opt_of[{static_cast<int>(t.model), t.epoch_index - 1}]);
        train_of[{static_cast<int>(t.model), t.epoch_index}].push_back(i);
        break;
      case TaskKind::ParamSync: {
        const int src = t.model == ModelName::ShadowActor ? 0 : 1;
        const auto it = opt_of.find({src, xp_.epochs - 1});
        if (it != opt_of.end()) d.push_back(it->second);
        break;
      }
      default:
        break;
    }
  }
  CK(cudaDeviceSynchronize());
}

Engine::~Engine() {
  if (decode_graph_) cudaGraphExecDestroy(decode_graph_);
  if (decode_graph1_) cudaGraphExecDestroy(decode_graph1_);
  for (Decoder* d : {&actor_, &critic_}) {
    for (cudaEvent_t e : d->rs_done)
      if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : d->wgather_done)
      if (e) cudaEventDestroy(e);
  }
  for (ncclComm_t c : {actor_comm_, critic_comm_, sync_comm_[0], sync_comm_[1], world_})
    if (c) nccl().CommDestroy(c);
  for (cudaEvent_t e : ev_pool_) cudaEventDestroy(e);
  for (cudaEvent_t e : step_done_) cudaEventDestroy(e);
  for (cudaEvent_t e : {ev_begin_, ev_end_})
    if (e) cudaEventDestroy(e);
  for (auto& l : lane_)
    if (l) cudaStreamDestroy(l);
}

// ---- events --------------------------------------------------------------------------

void Engine::wait_deps(int i, int lane) {
  for (int d : deps_[i])
    if (step_lane_[d] >= 0 && step_lane_[d] != lane) CK(cudaStreamWaitEvent(lane_[lane], step_done_[d], 0));
}

void Engine::begin_event(int i, const ExecStep& s, int kind, int lane, int stage) {
  use_lane(lane);
  wait_deps(i, lane);
  ExecEvent e;
  e.step = i;
  e.task = s.task;
  e.kind = kind;
  e.model = static_cast<int>(s.kind == StepKind::Task ? xp_.tasks[s.task].model : s.model);
  e.mb = s.mb;
  e.rollout = s.rollout;
  e.epoch = s.epoch;
  e.lane = lane;
  e.comm_op = s.comm_op;
  e.stage = stage;
  e.a = take_event();
  e.b = take_event();
  CK(cudaEventRecord(e.a, lane_[lane]));
  evs_.push_back(e);
}

void Engine::end_event() {
  ExecEvent& e = evs_.back();
  CK(cudaEventRecord(e.b, lane_[e.lane]));
  step_lane_[e.step] = e.lane;
  CK(cudaEventRecord(step_done_[e.step], lane_[e.lane]));
}

// ---- exchanges: row transfers over NCCL send/recv on the comm lane --------------------

void Engine::run_exchange(const ExecStep& s) {
  const int i = static_cast<int>(&s - xp_.steps.data());
  bool mine = false;
  for (const Move& m : s.moves)
    for (const Transfer& t : m.transfers) mine |= t.src_rank == rank_ || t.dst_rank == rank_;
  if (!mine) return;
  const bool prompt = s.moves[0].field == Field::Prompt;
  begin_event(i, s, static_cast<int>(TaskKind::Collective), 2,
              static_cast<int>(prompt ? Stage::Generation : Stage::Forward));
  auto src_ptr = [&](const Move& m) -> char* {
    return static_cast<char*>(m.src_set < 0 ? home_.p : rs_[m.src_set].field(m.field));
  };
  // local rows first (plain copies), then one NCCL group for the remote ones
  bool remote = false;
  for (const Move& m : s.moves) {
    const size_t rb = field_row_bytes(m.field, S_, R_);
    for (const Transfer& t : m.transfers) {
      if (t.src_rank == rank_ && t.dst_rank == rank_)
        CK(cudaMemcpyAsync(static_cast<char*>(rs_[m.dst_set].field(m.field)) + t.dst_row * rb, src_ptr(m) + t.src_row * rb,
                           t.count * rb, cudaMemcpyDeviceToDevice, stream_));
      else if (t.src_rank == rank_ || t.dst_rank == rank_)
        remote = true;
    }
  }
  if (remote) {
    NK(nccl().GroupStart());
    for (const Move& m : s.moves) {
      const size_t rb = field_row_bytes(m.field, S_, R_);
      for (const Transfer& t : m.transfers) {
        if (t.src_rank == t.dst_rank) continue;
        if (t.src_rank == rank_) {
          NK(nccl().Send(src_ptr(m) + t.src_row * rb, t.count * rb, ncclInt8, t.dst_rank, world_, stream_));
          comm_bytes_ += static_cast<double>(t.count * rb);
        } else if (t.dst_rank == rank_) {
          NK(nccl().Recv(static_cast<char*>(rs_[m.dst_set].field(m.field)) + t.dst_row * rb, t.count * rb, ncclInt8,
                         t.src_rank, world_, stream_));
        }
      }
    }
    NK(nccl().GroupEnd());
  }
  end_event();
}

// ---- tasks ----------------------------------------------------------------------------

// Forward + loss + backward of `B` experience rows starting at row0 of row set rb,
// accumulating into m's flat gradient.
void Engine::train_rows(Decoder& m, bool actor, RowBufs& rb, int row0, int B, float denom, bool reuse) {
  const int d = m.a.d_model, V = m.a.vocab, BR = B * R_;
  const int32_t* tok = rb.tokens.as<int32_t>() + static_cast<size_t>(row0) * S_;
  const size_t r0 = static_cast<size_t>(row0) * R_;
  // reuse: the experience Forward left this block's training activations (and, for the Actor,
  // its logits / lse / response rows) in the arena; the epoch-0 forward would recompute them
  if (!reuse) forward(m, tok, B, S_, S_, true, nullptr);
  if (actor) {
    float* logp = rb.logp_new.as<float>() + r0;
    float* g = rb.gbuf.as<float>() + r0;
    if (reuse)
      CK(cudaMemcpyAsync(logp, rb.logp_old.as<float>() + r0, static_cast<size_t>(BR) * 4, cudaMemcpyDeviceToDevice,
                         stream_));
    else
      lm_logprobs(m, tok, B, logp, true);
    K(rlhf_ppo_actor_loss(logp, rb.logp_old.as<float>() + r0, rb.adv.as<float>() + r0, BR, cfg_.cliprange, denom, g,
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
    CK(cudaMemsetAsync(arp_->dhf, 0, static_cast<size_t>(B) * S_ * d * 4, stream_));
    K(rlhf_scatter_rows_f32(arp_->dhf_resp, arp_->dhf, B, S_, R_, P_ - 1, d, stream_), 1);
  } else {
    float* v = rb.values_new.as<float>() + r0;
    float* g = rb.gbuf2.as<float>() + r0;
    if (reuse)
      CK(cudaMemcpyAsync(v, rb.values.as<float>() + r0, static_cast<size_t>(BR) * 4, cudaMemcpyDeviceToDevice, stream_));
    else
      K(rlhf_scalar_head(arp_->hf, m.T(RLHF_T_VHEAD), B, S_, R_, P_ - 1, d, v, stream_), 1);
    K(rlhf_ppo_critic_loss(v, rb.values.as<float>() + r0, rb.ret.as<float>() + r0, BR, cfg_.cliprange_value, denom, g,
                           loss_.as<float>() + 1, stream_), 1);
    CK(cudaMemsetAsync(arp_->dhf, 0, static_cast<size_t>(B) * S_ * d * 4, stream_));
    K(rlhf_scalar_head_bwd(arp_->hf, m.T(RLHF_T_VHEAD), g, B, S_, R_, P_ - 1, d, arp_->dhf, m.G(RLHF_T_VHEAD), arp_->ws,
                           stream_), 2);
  }
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

void Engine::run_task(const ExecStep& s) {
  const int i = static_cast<int>(&s - xp_.steps.data());
  const StageTask& t = xp_.tasks[s.task];
  const int mi = static_cast<int>(t.model);
  switch (t.kind) {
    case TaskKind::Generation: {
      if (!hosts_[mi]) return;
      RowBufs& rb = rs_[xp_.set_of[mi]];
      const size_t row0 = static_cast<size_t>(s.rollout * xp_.M + s.mb) * gen_B_;
      begin_event(i, s, static_cast<int>(TaskKind::Generation), 0, static_cast<int>(Stage::Generation));
      const size_t bytes = static_cast<size_t>(gen_B_) * S_ * 4;
      CK(cudaMemcpyAsync(gen_tok_.p, rb.tokens.as<int32_t>() + row0 * S_, bytes, cudaMemcpyDeviceToDevice, stream_));
      ev_prefill_ = take_event();
      generate(*generator_, gen_B_, false);
      CK(cudaMemcpyAsync(rb.tokens.as<int32_t>() + row0 * S_, gen_tok_.p, bytes, cudaMemcpyDeviceToDevice, stream_));
      end_event();
      prefill_.push_back({evs_.back().a, ev_prefill_});
      decode_.push_back({ev_prefill_, evs_.back().b});
      ev_prefill_ = nullptr;
      return;
    }
    case TaskKind::Forward: {
      if (!hosts_[mi]) return;
      RowBufs& rb = rs_[xp_.set_of[mi]];
      const int per = xp_.sets[xp_.set_of[mi]].per;
      const size_t row0 = static_cast<size_t>(s.rollout * xp_.M + s.mb) * per;
      const int32_t* tok = rb.tokens.as<int32_t>() + row0 * S_;
      begin_event(i, s, static_cast<int>(TaskKind::Forward), lane_of(t.model), static_cast<int>(Stage::Forward));
      const Decoder& m = *model(t.model);
      if (mi <= 1 && reuse_fwd_[mi]) {  // the training forward, kept for TrainFB epoch 0
        forward(m, tok, per, S_, S_, true, nullptr);
        if (mi == 0) lm_logprobs(m, tok, per, rb.logp_old.as<float>() + row0 * R_, true);
        else K(rlhf_scalar_head(arp_->hf, m.T(RLHF_T_VHEAD), per, S_, R_, P_ - 1, m.a.d_model,
                                rb.values.as<float>() + row0 * R_, stream_), 1);
        end_event();
        return;
      }
      switch (output_field(t.model)) {
        case Field::LogpOld: score_logp(m, tok, per, rb.logp_old.as<float>() + row0 * R_); break;
        case Field::LogpRef: score_logp(m, tok, per, rb.logp_ref.as<float>() + row0 * R_); break;
        case Field::Values: score_values(m, tok, per, rb.values.as<float>() + row0 * R_); break;
        case Field::Score: score_reward(m, tok, per, rb.score.as<float>() + row0); break;
        default: break;
      }
      end_event();
      return;
    }
    case TaskKind::TrainFB: {
      if (!hosts_[mi]) return;
      const bool actor = t.model == ModelName::Actor;
      Decoder& m = *model(t.model);
      RowBufs& rb = rs_[xp_.set_of[mi]];
      const int per = xp_.sets[xp_.set_of[mi]].per;
      begin_event(i, s, static_cast<int>(TaskKind::TrainFB), lane_of(t.model), static_cast<int>(Stage::Training));
      if (t.micro_batch_index == 0) {  // a new epoch's gradient and loss sum
        if (m.zero2) {
          CK(cudaMemsetAsync(m.gpre.p, 0, m.gpre.bytes, stream_));
          CK(cudaMemsetAsync(m.gpost.p, 0, m.gpost.bytes, stream_));
          // the shard accumulator is also written by the comm lane: order after its last use
          for (cudaEvent_t e : m.rs_done) CK(cudaStreamWaitEvent(stream_, e, 0));
          CK(cudaMemsetAsync(m.gshard.p, 0, m.gshard.bytes, stream_));
        } else {
          CK(cudaMemsetAsync(m.grad.p, 0, static_cast<size_t>(m.npad) * 4, stream_));
        }
        CK(cudaMemsetAsync(loss_.as<float>() + (actor ? 0 : 1), 0, 4, stream_));
      }
      // the micro-batch's rows of every rollout (one block per rollout), in chunks of train_mb_
      const float denom = cfg_.loss_denominator > 0 ? cfg_.loss_denominator * xp_.rollouts
                                                    : static_cast<float>(xp_.G) * xp_.rollouts * R_;
      const bool reuse = reuse_fwd_[mi] && t.epoch_index == 0;
      for (int r = 0; r < xp_.rollouts; ++r) {
        const int row0 = (r * xp_.M + t.micro_batch_index) * per;
        for (int c = 0; c < per; c += train_mb_)
          train_rows(m, actor, rb, row0 + c, std::min(train_mb_, per - c), denom, reuse);
      }
      end_event();
      return;
    }
    case TaskKind::ParamSync: {
      const int k = t.model == ModelName::ShadowActor ? 0 : 1;
      if (!sync_comm_[k]) return;  // world 1, or this rank is neither trainer nor shadow
      Decoder& src = k == 0 ? actor_ : critic_;
      Decoder& dst = k == 0 ? shadow_actor_ : shadow_critic_;
      const bool is_src = hosts_[k == 0 ? 0 : 1];
      begin_event(i, s, static_cast<int>(TaskKind::ParamSync), 2, static_cast<int>(Stage::Sync));
      if (opt_.zero_stage == 3) {
        // the trainers hold bucket slices: per bucket, all-gather among the trainers, then
        // broadcast the whole bucket to the shadows (same bucket order on every rank)
        const rlhf_arch& a = is_src ? src.a : dst.a;
        const int64_t ls = rlhf_tensor_offset(&a, RLHF_LAYER_FIRST, 0), ps = rlhf_tensor_offset(&a, RLHF_T_LNF_G, 0);
        const int64_t ll = (ps - ls) / a.n_layers, n = rlhf_param_total(&a);
        std::vector<std::pair<int64_t, int64_t>> rng{{0, ls}};
        for (int l = 0; l < a.n_layers; ++l) rng.push_back({ls + l * ll, ll});
        rng.push_back({ps, n - ps});
        ncclComm_t tcomm = dp_comm(src);
        for (size_t bk = 0; bk < rng.size(); ++bk) {
          const auto [start, len] = rng[bk];
          void* buf = dst.w.p ? static_cast<void*>(dst.w.as<uint16_t>() + start) : nullptr;
          if (is_src) {
            const GradBucket& g = src.buckets[bk];
            const uint16_t* mine = src.wshard.as<uint16_t>() + g.soff;
            if (tcomm) NK(nccl().AllGather(mine, src.ag_stage.p, static_cast<size_t>(g.slice), ncclBfloat16, tcomm, stream_));
            else CK(cudaMemcpyAsync(src.ag_stage.p, mine, static_cast<size_t>(g.len) * 2, cudaMemcpyDeviceToDevice, stream_));
            buf = src.ag_stage.p;
            comm_bytes_ += 2.0 * static_cast<double>(len);
          }
          NK(nccl().Broadcast(buf, buf, static_cast<size_t>(len), ncclBfloat16, sync_root_[k], sync_comm_[k], stream_));
        }
      } else {
        const size_t n = static_cast<size_t>(is_src ? src.n : dst.n);
        NK(nccl().Broadcast(is_src ? src.w.p : dst.w.p, is_src ? src.w.p : dst.w.p, n, ncclBfloat16, sync_root_[k],
                            sync_comm_[k], stream_));
        if (is_src) comm_bytes_ += 2.0 * static_cast<double>(n);
      }
      end_event();
      return;
    }
    default:
      return;
  }
}

// Experience-buffer barrier (workload.cpp:153-163) on one trainer row set: KL-shaped rewards,
// GAE, returns over every row; the reported score / KL means come from the experience set.
void Engine::run_experience(const ExecStep& s) {
  const int i = static_cast<int>(&s - xp_.steps.data());
  if (xp_.member_index(s.set, rank_) < 0 || !rs_[s.set].trainer) return;
  RowBufs& rb = rs_[s.set];
  begin_event(i, s, kEvExperience, 0, static_cast<int>(Stage::Training));
  K(rlhf_gae(rb.logp_old.as<float>(), rb.logp_ref.as<float>(), rb.values.as<float>(), rb.score.as<float>(), rb.rows, R_,
             cfg_.kl_ctl, cfg_.clip_reward, cfg_.gamma, cfg_.lam, rb.rewards.as<float>(), rb.adv.as<float>(),
             rb.ret.as<float>(), stream_), 1);
  if (s.set == xp_.experience_set(rank_))
    K(rlhf_experience_stats(rb.logp_old.as<float>(), rb.logp_ref.as<float>(), rb.score.as<float>(), rb.rows, R_,
                            loss_.as<float>() + 2, stream_), 1);
  end_event();
}

// Gradient sync + AdamW closing a TrainFB epoch of one model (costmodel.hpp:59-74): ZeRO-0
// all-reduce, or ZeRO-1 reduce-scatter -> AdamW on the rank's shard -> all-gather of the
// bf16 weights.  The collectives run on the comm lane, AdamW on the model's compute lane.
void Engine::run_optimizer(const ExecStep& s, int i) {
  const int mi = static_cast<int>(s.model);
  if (!hosts_[mi]) return;
  Decoder& m = *model(s.model);
  ncclComm_t comm = s.model == ModelName::Actor ? actor_comm_ : critic_comm_;
  const float lr = s.model == ModelName::Actor ? cfg_.lr_actor : cfg_.lr_critic;
  const int ml = lane_of(s.model);
  const int st = static_cast<int>(Stage::Training);
  if (m.zero2) {
    // the comm lane must also have finished the per-layer reduce-scatters of the last chunk
    zero2_optimizer(m, comm, lr, i);
    return;
  }
  cudaEvent_t prev = nullptr;
  if (comm) {
    begin_event(i, s, static_cast<int>(TaskKind::Collective), 2, st);
    if (m.sharded) {  // each rank only needs the summed gradient of its own shard
      NK(nccl().ReduceScatter(m.grad.p, m.grad.as<float>() + m.shard_off, static_cast<size_t>(m.shard), ncclFloat32,
                              ncclSum, comm, stream_));
      comm_bytes_ += 4.0 * static_cast<double>(m.npad - m.shard);
    } else {
      NK(nccl().AllReduce(m.grad.p, m.grad.p, static_cast<size_t>(m.n), ncclFloat32, ncclSum, comm, stream_));
      comm_bytes_ += 2.0 * 4.0 * static_cast<double>(m.n);
    }
    end_event();
    prev = evs_.back().b;
  }
  begin_event(i, s, kEvAdam, ml, st);
  if (prev) CK(cudaStreamWaitEvent(stream_, prev, 0));
  adam(m, lr);
  end_event();
  if (m.sharded && comm) {
    prev = evs_.back().b;
    begin_event(i, s, static_cast<int>(TaskKind::Collective), 2, st);
    CK(cudaStreamWaitEvent(stream_, prev, 0));
    NK(nccl().AllGather(m.w.as<uint16_t>() + m.shard_off, m.w.p, static_cast<size_t>(m.shard), ncclBfloat16, comm,
                        stream_));
    comm_bytes_ += 2.0 * static_cast<double>(m.npad - m.shard);
    end_event();
  }
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
    DevBuf* b = new DevBuf();
    A.owned.push_back(b);
    b->alloc(bytes);
    return b->p;
  };
  const int64_t T = A.T, d = A.d, SS = static_cast<int64_t>(A.S) * A.S, BR = static_cast<int64_t>(Bcap_) * R_;
  const int64_t Ls = trains ? A.L : 1;  // layers of saved activations (inference-only ranks keep one)
  // per-layer saved activations: Ls slots of one training chunk (Ts rows), and at least
  // one slot of a whole Forward block (T rows, layer buffers reused across layers)
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

// ---- the step -------------------------------------------------------------------------

void Engine::step(const int32_t* prompts_host, rlhf_step_report* rep) {
  CK(cudaSetDevice(opt_.device));
  launches_ = 0;
  comm_bytes_ = 0;
  evs_.clear();
  ev_next_ = 0;
  prefill_.clear();
  decode_.clear();
  std::fill(step_lane_.begin(), step_lane_.end(), -1);
  // this rank's home prompts: global samples r*G + rank*Bg + [0, Bg) of every rollout,
  // rows of S int32 (first P columns) so an exchange moves whole token rows
  const int rows = xp_.rollouts * Bg_;
  std::vector<int32_t> pr(static_cast<size_t>(rows) * S_, 0);
  const int64_t id_shift = static_cast<int64_t>(cfg_.sample_offset) - static_cast<int64_t>(rank_) * Bg_;
  for (int r = 0; r < xp_.rollouts; ++r)
    for (int b = 0; b < Bg_; ++b) {
      const size_t row = static_cast<size_t>(r) * Bg_ + b;
      const int64_t id = static_cast<int64_t>(r) * xp_.G + static_cast<int64_t>(rank_) * Bg_ + b + id_shift;
      for (int t = 0; t < P_; ++t)
        pr[row * S_ + t] = prompts_host ? prompts_host[row * P_ + t]
                                        : rlhf_prompt_token(cfg_.prompt_seed, static_cast<int>(id), t, cfg_.actor.vocab);
    }
  CK(cudaEventRecord(ev_begin_, lane_[0]));
  for (int l = 1; l < 3; ++l) CK(cudaStreamWaitEvent(lane_[l], ev_begin_, 0));
  // host -> device on the comm lane: the prompt exchanges that follow consume it there
  CK(cudaMemcpyAsync(home_.p, pr.data(), pr.size() * 4, cudaMemcpyHostToDevice, lane_[2]));

  auto is_fwd = [&](size_t i) {
    const ExecStep& s = xp_.steps[i];
    return s.kind == StepKind::Task && xp_.tasks[s.task].kind == TaskKind::Forward;
  };
  for (size_t i = 0; i < xp_.steps.size(); ++i) {
    const ExecStep& s = xp_.steps[i];
    if (is_fwd(i) && (reuse_fwd_[0] || reuse_fwd_[1])) {
      // a run of independent Forward tasks (one generation's scorers): the ones whose
      // activations TrainFB reuses go last on their lane, after the forwards that would
      // overwrite the arena
      size_t j = i;
      while (j < xp_.steps.size() && is_fwd(j)) ++j;
      for (int pass = 0; pass < 2; ++pass)
        for (size_t k = i; k < j; ++k) {
          const int mk = static_cast<int>(xp_.tasks[xp_.steps[k].task].model);
          if ((mk <= 1 && reuse_fwd_[mk]) == (pass == 1)) run_task(xp_.steps[k]);
        }
      i = j - 1;
      continue;
    }
    switch (s.kind) {
      case StepKind::Exchange: run_exchange(s); break;
      case StepKind::Task: run_task(s); break;
      case StepKind::Experience: run_experience(s); break;
      case StepKind::OptimizerStep: run_optimizer(s, static_cast<int>(i)); break;
    }
  }
  // join every lane into the main one
  for (int l = 1; l < 3; ++l) {
    cudaEvent_t j = take_event();
    CK(cudaEventRecord(j, lane_[l]));
    CK(cudaStreamWaitEvent(lane_[0], j, 0));
  }
  use_lane(0);
  CK(cudaEventRecord(ev_end_, lane_[0]));
  float loss[4];
  CK(cudaMemcpyAsync(loss, loss_.p, 16, cudaMemcpyDeviceToHost, lane_[0]));
  CK(cudaStreamSynchronize(lane_[0]));

  std::memset(rep, 0, sizeof(*rep));
  auto since = [&](cudaEvent_t a, cudaEvent_t b) {
    float t = 0;
    cudaEventElapsedTime(&t, a, b);
    return static_cast<double>(t) * 1e-3;
  };
  rep->step_seconds = since(ev_begin_, ev_end_);
  rep->throughput_samples_per_sec = static_cast<double>(xp_.G) * xp_.rollouts / rep->step_seconds;
  for (ExecEvent& e : evs_) {
    e.start = since(ev_begin_, e.a);
    e.end = since(ev_begin_, e.b);
  }
  for (const auto& [a, b] : prefill_) rep->prefill_seconds += since(a, b);
  for (const auto& [a, b] : decode_) rep->decode_seconds += since(a, b);

  // SimReport accounting: every instant of the step is attributed to one
  // stage -- the lowest Stage among the compute-lane intervals active then, else among the
  // comm-lane ones, else (idle) the stage of the next interval to start
  std::vector<double> cut{0.0, rep->step_seconds};
  for (const ExecEvent& e : evs_) {
    cut.push_back(e.start);
    cut.push_back(e.end);
  }
  std::sort(cut.begin(), cut.end());
  cut.erase(std::unique(cut.begin(), cut.end()), cut.end());
  double pending = 0;
  int last_stage = 0;
  for (size_t k = 0; k + 1 < cut.size(); ++k) {
    const double t0 = cut[k], t1 = cut[k + 1], mid = 0.5 * (t0 + t1);
    if (t1 <= t0 || t0 >= rep->step_seconds) continue;
    int comp = 99, comm = 99;
    for (const ExecEvent& e : evs_)
      if (e.start <= mid && mid < e.end) (e.lane == 2 ? comm : comp) = std::min(e.lane == 2 ? comm : comp, e.stage);
    if (comp < 99) rep->busy_seconds += t1 - t0;
    if (comm < 99) rep->comm_seconds += t1 - t0;
    const int stg = comp < 99 ? comp : comm;
    if (stg == 99) {
      pending += t1 - t0;
      continue;
    }
    rep->stage_seconds[stg] += t1 - t0 + pending;
    pending = 0;
    last_stage = stg;
  }
  rep->stage_seconds[last_stage] += pending;
  rep->bubble_fraction = rep->step_seconds > 0 ? 1.0 - rep->busy_seconds / rep->step_seconds : 0.0;
  rep->busiest_stage = static_cast<int>(std::max_element(rep->stage_seconds, rep->stage_seconds + 4) - rep->stage_seconds);
  rep->mem_peak_bytes = static_cast<double>(g_device_bytes.load());
  rep->n_events = static_cast<int>(evs_.size());
  {
    const FeasibilityReport fr = validate_plan(xp_.plan, xp_.pipeline, CostModel{}, ClusterTopology::b200_box(world_n_));
    rep->feasible = fr.feasible ? 1 : 0;
  }
  const float denom = cfg_.loss_denominator > 0 ? cfg_.loss_denominator * xp_.rollouts
                                                : static_cast<float>(xp_.G) * xp_.rollouts * R_;
  rep->actor_loss = hosts_[0] ? loss[0] / denom : 0.0;
  rep->critic_loss = hosts_[1] ? 0.5 * loss[1] / denom : 0.0;
  const int es = xp_.experience_set(rank_);
  if (es >= 0 && rs_[es].trainer) {
    rep->mean_score = loss[2] / rs_[es].rows;
    rep->mean_kl = loss[3] / (static_cast<double>(rs_[es].rows) * R_);
  }
  rep->comm_bytes_total = comm_bytes_;
  rep->gpu_launches = launches_;
}

// ---- tensors for tests ------------------------------------------------------------------

size_t Engine::tensor_bytes(const std::string& name) const {
  const int es = xp_.experience_set(rank_);
  const size_t rows = es >= 0 ? static_cast<size_t>(rs_[es].rows) : 0;
  static const std::map<std::string, int> kBR = {{"logp_old", 0}, {"logp_ref", 0}, {"values", 0}};
  static const std::map<std::string, int> kTrain = {{"rewards", 0},  {"advantages", 0}, {"returns", 0},
                                                    {"logp_new", 0}, {"values_new", 0}};
  if (kBR.count(name)) return rows * R_ * 4;
  if (kTrain.count(name)) return es >= 0 && rs_[es].trainer ? rows * R_ * 4 : 0;
  if (name == "tokens") return rows * S_ * 4;
  if (name == "pred" || name == "margin") return static_cast<size_t>(gen_B_) * S_ * 4;
  if (name == "score" || name == "sample_ids") return rows * 4;
  auto flat = [](const Decoder& m, size_t e) { return static_cast<size_t>(m.n) * e; };
  if (name == "actor_grad") return actor_.zero2 ? 0 : flat(actor_, 4);
  if (name == "critic_grad") return critic_.zero2 ? 0 : flat(critic_, 4);
  if (name == "actor_master") return static_cast<size_t>(actor_.shard) * 4;  // this rank's slice under ZeRO-1
  if (name == "critic_master") return static_cast<size_t>(critic_.shard) * 4;
  // ZeRO-3: this rank's bf16 slices of every bucket (the full weights are never resident)
  if (name == "actor_params") return actor_.zero3 ? static_cast<size_t>(actor_.shard) * 2 : flat(actor_, 2);
  if (name == "critic_params") return critic_.zero3 ? static_cast<size_t>(critic_.shard) * 2 : flat(critic_, 2);
  if (name == "ref_params") return flat(ref_, 2);
  if (name == "reward_params") return flat(reward_, 2);
  if (name == "shadow_actor_params") return flat(shadow_actor_, 2);
  if (name == "shadow_critic_params") return flat(shadow_critic_, 2);
  return 0;
}

void Engine::read(const std::string& name, void* host, size_t bytes) {
  CK(cudaSetDevice(opt_.device));
  if (bytes != tensor_bytes(name) || bytes == 0) throw ConfigError("size mismatch (or tensor absent on this rank): " + name);
  for (auto& l : lane_) CK(cudaStreamSynchronize(l));
  const int es = xp_.experience_set(rank_);
  if (name == "sample_ids") {
    std::vector<int32_t> ids(bytes / 4);
    for (size_t r = 0; r < ids.size(); ++r) ids[r] = static_cast<int32_t>(xp_.sample_id(es, rank_, static_cast<int>(r)));
    std::memcpy(host, ids.data(), bytes);
    return;
  }
  const DevBuf* src = nullptr;
  if (es >= 0) {
    const RowBufs& b = rs_[es];
    const std::map<std::string, const DevBuf*> rowf = {
        {"tokens", &b.tokens}, {"logp_old", &b.logp_old}, {"logp_ref", &b.logp_ref}, {"values", &b.values},
        {"score", &b.score}, {"rewards", &b.rewards}, {"advantages", &b.adv}, {"returns", &b.ret},
        {"logp_new", &b.logp_new}, {"values_new", &b.values_new}};
    auto it = rowf.find(name);
    if (it != rowf.end()) src = it->second;
  }
  const std::map<std::string, const DevBuf*> m = {
      {"pred", &pred_}, {"margin", &margin_}, {"actor_grad", &actor_.grad}, {"critic_grad", &critic_.grad},
      {"actor_master", &actor_.master}, {"critic_master", &critic_.master},
      {"actor_params", actor_.zero3 ? &actor_.wshard : &actor_.w},
      {"critic_params", critic_.zero3 ? &critic_.wshard : &critic_.w}, {"ref_params", &ref_.w}, {"reward_params", &reward_.w},
      {"shadow_actor_params", &shadow_actor_.w}, {"shadow_critic_params", &shadow_critic_.w}};
  if (!src) {
    auto it = m.find(name);
    if (it == m.end()) throw ConfigError("unknown tensor " + name);
    src = it->second;
  }
  CK(cudaMemcpy(host, src->p, bytes, cudaMemcpyDeviceToHost));
}

void Engine::greedy_check(const int32_t* tokens_host, int32_t* pred_host, float* margin_host) {
  CK(cudaSetDevice(opt_.device));
  if (!generator_) throw ConfigError("this rank does not generate");
  use_lane(0);
  const int B = gen_B_;
  CK(cudaMemcpyAsync(gen_tok_.p, tokens_host, static_cast<size_t>(B) * S_ * 4, cudaMemcpyHostToDevice, stream_));
  CK(cudaMemsetAsync(pred_.p, 0, static_cast<size_t>(B) * S_ * 4, stream_));
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

SimReport execute(Engine& engine, const int32_t* prompts_host) {
  rlhf_step_report rep;
  engine.step(prompts_host, &rep);
  SimReport r;
  r.step_seconds = rep.step_seconds;
  r.throughput_samples_per_sec = rep.throughput_samples_per_sec;
  for (const ExecEvent& x : engine.events()) {
    SimEvent e;
    e.task_id = x.task;
    // the experience barrier (GAE) and AdamW intervals are TrainFB-stage work in SimEvent terms
    e.kind = x.kind <= static_cast<int>(TaskKind::Barrier) ? static_cast<TaskKind>(x.kind) : TaskKind::TrainFB;
    e.model = static_cast<ModelName>(x.model);
    e.micro_batch = x.mb;
    e.stage = static_cast<Stage>(x.stage);
    e.comm_lane = x.lane == 2;
    e.start = x.start;
    e.end = x.end;
    e.devices = {engine.rank()};
    r.events.push_back(e);
  }
  for (int k = 0; k < 4; ++k) {
    r.per_stage_seconds[static_cast<Stage>(k)] = rep.stage_seconds[k];
    r.per_stage_fraction[static_cast<Stage>(k)] = rep.step_seconds > 0 ? rep.stage_seconds[k] / rep.step_seconds : 0;
  }
  r.per_device_busy_seconds[engine.rank()] = rep.busy_seconds;
  r.per_device_mem_peak[engine.rank()] = rep.mem_peak_bytes;
  r.comm_bytes_total = rep.comm_bytes_total;
  r.bubble_fraction = rep.bubble_fraction;
  r.busiest_stage = static_cast<Stage>(rep.busiest_stage);
  r.feasible = rep.feasible != 0;
  return r;
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

// Largest per-rank batch whose engine fits the device (max_batch_search, simulator.hpp:53-54,
// against the real allocator instead of the analytic memory model): doubling then bisection
// over engine constructions; an allocation that does not fit surfaces as InfeasibleError.
extern "C" int rlhf_engine_max_batch(const rlhf_ppo_config* cfg, const rlhf_engine_options* opt, int cap, int run_step,
                                     int* best) {
  try {
    if (!best || cap < 1) throw flexrlhf::ConfigError("rlhf_engine_max_batch: cap >= 1 and an output are required");
    if (opt->world_size > 1) throw flexrlhf::ConfigError("rlhf_engine_max_batch: single-GPU engines only");
    const int mb = std::max(1, opt->micro_batches);
    auto fits = [&](int k) {
      rlhf_ppo_config c = *cfg;
      c.batch = k * mb;
      try {
        Engine e(c, *opt);
        if (run_step) {
          rlhf_step_report r;
          e.step(nullptr, &r);
        }
        return true;
      } catch (const flexrlhf::InfeasibleError&) {
        cudaGetLastError();
        return false;
      }
    };
    *best = 0;
    const int kmax = cap / mb;
    if (kmax < 1 || !fits(1)) return 0;
    int lo = 1, hi = 1;
    while (hi < kmax) {  // doubling: lo fits, hi + 1 .. unknown
      const int nxt = std::min(kmax, hi * 2);
      if (!fits(nxt)) {
        hi = nxt - 1;
        break;
      }
      lo = hi = nxt;
    }
    while (lo < hi) {
      const int m = lo + (hi - lo + 1) / 2;
      if (fits(m)) lo = m;
      else hi = m - 1;
    }
    *best = lo * mb;
    return 0;
  } catch (const std::exception& ex) {
    return flexrlhf::capi_status(ex);
  }
}

extern "C" int rlhf_engine_events(rlhf_engine* e, rlhf_event* out, int max) {
  const std::vector<flexrlhf::ExecEvent>& ev = e->impl->events();
  const int n = std::min<int>(max, static_cast<int>(ev.size()));
  for (int i = 0; i < n; ++i) {
    const flexrlhf::ExecEvent& x = ev[i];
    out[i] = rlhf_event{x.task, x.kind, x.model, x.mb, x.rollout, x.epoch, x.lane, x.comm_op, x.stage, x.start, x.end};
  }
  return static_cast<int>(ev.size());
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
