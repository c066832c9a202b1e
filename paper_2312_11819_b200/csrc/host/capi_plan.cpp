// C-ABI over the host placement / workload API (include/rlhf_engine.h).
// Pure host logic: no device calls.
#include <algorithm>
#include <cstring>
#include <exception>
#include <string>

#include "capi_util.hpp"
#include "execplan.hpp"
#include "flexrlhf/simulator.hpp"
#include "flexrlhf/placement.hpp"
#include "rlhf_engine.h"

using namespace flexrlhf;

namespace flexrlhf {
thread_local std::string g_last_error;

int capi_status(const std::exception& e) {
  g_last_error = e.what();
  if (dynamic_cast<const ConfigError*>(&e)) return RLHF_ERR_CONFIG;
  if (dynamic_cast<const InfeasibleError*>(&e)) return RLHF_ERR_INFEASIBLE;
  if (dynamic_cast<const SearchCapError*>(&e)) return 4;
  return RLHF_ERR_DEVICE;
}
}  // namespace flexrlhf

namespace {

PipelineSpec pipeline_for(int structure, int batch, int micro_batches, int rollouts, int epochs, int P, int R) {
  ModelSizes sz;
  sz.actor = sz.critic = sz.ref = sz.reward = 1.0e8;
  LoopParams lp;
  lp.batch_size = batch;
  lp.micro_batches = micro_batches;
  lp.rollout_nums = rollouts;
  lp.ppo_epochs = epochs;
  lp.prompt_len = P;
  lp.gen_len = R;
  return build_pipeline(structure ? PipelineStructure::ACNonShare : PipelineStructure::ACShare, sz, lp);
}

}  // namespace

extern "C" const char* rlhf_last_error(void) { return g_last_error.c_str(); }

extern "C" void rlhf_ppo_config_default(rlhf_ppo_config* c, const rlhf_arch* actor, const rlhf_arch* critic, int batch,
                                        int prompt_len, int gen_len) {
  std::memset(c, 0, sizeof(*c));
  c->actor = *actor;
  c->actor.scalar_head = 0;
  c->critic = *critic;
  c->critic.scalar_head = 1;
  c->batch = batch;
  c->prompt_len = prompt_len;
  c->gen_len = gen_len;
  c->seed = 7;
  c->prompt_seed = 1000;
  c->kl_ctl = 0.1f;
  c->clip_reward = 5.0f;
  c->gamma = 1.0f;
  c->lam = 0.95f;
  c->cliprange = 0.2f;
  c->cliprange_value = 0.2f;
  c->lr_actor = 1e-5f;
  c->lr_critic = 5e-6f;
  c->beta1 = 0.9f;
  c->beta2 = 0.95f;
  c->adam_eps = 1e-8f;
  c->weight_decay = 0.0f;
  c->loss_denominator = 0.0f;
}

extern "C" int rlhf_arch_by_name(const char* name, int max_pos, int scalar_head, rlhf_arch* out) {
  try {
    const ArchSpec a = arch_by_name(name);
    out->family = a.family == ArchFamily::OPT ? 0 : 1;
    out->vocab = a.vocab;
    out->d_model = a.d_model;
    out->n_layers = a.n_layers;
    out->n_heads = a.n_heads;
    out->d_ff = a.d_ff;
    out->max_pos = max_pos;
    out->scalar_head = scalar_head;
    return 0;
  } catch (const std::exception& e) {
    return capi_status(e);
  }
}

extern "C" int rlhf_task_graph(int structure, int batch, int micro_batches, int rollout_nums, int ppo_epochs,
                               int shadows, int max_tasks, int max_deps, int* n_tasks, int* n_deps, int* kind,
                               int* model, int* mb, int* rollout, int* epoch, int* dep_off, int* deps) {
  try {
    PipelineSpec p = pipeline_for(structure, batch, micro_batches, rollout_nums, ppo_epochs, 256, 256);
    if (shadows > 1) p = with_shadows(p);  // 2: add shadow entries; 1: request shadows as given
    const std::vector<StageTask> g = task_graph(p, shadows != 0);
    int nd = 0;
    for (const StageTask& t : g) nd += static_cast<int>(t.depends_on.size());
    *n_tasks = static_cast<int>(g.size());
    *n_deps = nd;
    if (max_tasks == 0) return 0;
    if (max_tasks < *n_tasks || max_deps < nd) throw ConfigError("rlhf_task_graph: output arrays too small");
    int o = 0;
    for (size_t i = 0; i < g.size(); ++i) {
      kind[i] = static_cast<int>(g[i].kind);
      model[i] = static_cast<int>(g[i].model);
      mb[i] = g[i].micro_batch_index;
      rollout[i] = g[i].rollout_index;
      epoch[i] = g[i].epoch_index;
      dep_off[i] = o;
      for (int d : g[i].depends_on) deps[o++] = d;
    }
    dep_off[g.size()] = o;
    return 0;
  } catch (const std::exception& e) {
    return capi_status(e);
  }
}

extern "C" int rlhf_plan(const char* strategy, int n_devices, int zero_level, double inference_ratio, int tp_gen,
                         uint32_t out_mask[6], int* out_role, char* enc, int enc_len) {
  try {
    const ClusterTopology t = ClusterTopology::b200_box(n_devices);
    StrategyConfig sc;
    sc.name = strategy;
    sc.zero_level = zero_level;
    sc.inference_ratio = inference_ratio;
    sc.tp_gen = tp_gen;
    const BuiltStrategy b = build_strategy(sc, t, pipeline_for(1, 64, 1, 1, 1, 256, 256));
    for (int m = 0; m < 6; ++m) {
      out_mask[m] = 0;
      auto it = b.plan.assignments.find(static_cast<ModelName>(m));
      if (it != b.plan.assignments.end())
        for (int d : it->second.devices) out_mask[m] |= 1u << d;
    }
    for (int d = 0; d < n_devices; ++d) out_role[d] = static_cast<int>(b.plan.device_role.at(d));
    const std::string s = b.plan.encoding();
    if (enc && enc_len > 0) {
      std::strncpy(enc, s.c_str(), static_cast<size_t>(enc_len) - 1);
      enc[enc_len - 1] = 0;
    }
    return 0;
  } catch (const std::exception& e) {
    return capi_status(e);
  }
}

extern "C" int rlhf_comm_schedule(const char* strategy, int n_devices, int batch, int prompt_len, int gen_len,
                                  int micro_batches, int max_ops, int* n_ops, int* kind, int* attach, int* anchor,
                                  double* payload, uint32_t* group_mask) {
  try {
    const ClusterTopology t = ClusterTopology::b200_box(n_devices);
    StrategyConfig sc;
    sc.name = strategy;
    sc.tp_gen = 1;
    const BuiltStrategy b = build_strategy(sc, t, pipeline_for(1, batch, micro_batches, 1, 1, prompt_len, gen_len));
    const CommSchedule s = derive_comm_schedule(b.plan, b.pipeline, CostModel{});
    *n_ops = static_cast<int>(s.ops.size());
    if (max_ops == 0) return 0;
    if (max_ops < *n_ops) throw ConfigError("rlhf_comm_schedule: output arrays too small");
    for (size_t i = 0; i < s.ops.size(); ++i) {
      kind[i] = static_cast<int>(s.ops[i].kind);
      attach[i] = s.ops[i].attach == AttachKind::Before ? 0 : 1;
      anchor[i] = s.ops[i].anchor_task;
      payload[i] = s.ops[i].payload_bytes;
      group_mask[i] = 0;
      for (int d : s.ops[i].group) group_mask[i] |= 1u << d;
    }
    return 0;
  } catch (const std::exception& e) {
    return capi_status(e);
  }
}

extern "C" int rlhf_validate_plan(const char* strategy, int n_devices, int zero_level, double inference_ratio, int tp_gen,
                                  double actor_params, double critic_params, int batch, int prompt_len, int gen_len,
                                  double* state_bytes, double* total_bytes, int* feasible) {
  try {
    const ClusterTopology t = ClusterTopology::b200_box(n_devices);
    ModelSizes sz;
    sz.actor = sz.ref = actor_params;
    sz.critic = sz.reward = critic_params;
    LoopParams lp;
    lp.batch_size = batch;
    lp.micro_batches = 1;
    lp.rollout_nums = 1;
    lp.ppo_epochs = 1;
    lp.prompt_len = prompt_len;
    lp.gen_len = gen_len;
    StrategyConfig sc;
    sc.name = strategy;
    sc.zero_level = zero_level;
    sc.inference_ratio = inference_ratio;
    sc.tp_gen = tp_gen;
    const BuiltStrategy b = build_strategy(sc, t, build_pipeline(PipelineStructure::ACNonShare, sz, lp));
    const CostModel c{};
    for (int d = 0; d < n_devices; ++d) state_bytes[d] = total_bytes[d] = 0.0;
    for (const auto& [m, cfg] : b.plan.assignments) {
      if (!b.pipeline.has_model(m)) continue;
      const double st = model_state_bytes(b.pipeline.model(m), cfg, c.mem);
      for (int d : cfg.devices) state_bytes[d] += st;
    }
    const FeasibilityReport rep = validate_plan(b.plan, b.pipeline, c, t);
    for (const auto& [d, bytes] : rep.per_device_bytes) total_bytes[d] = bytes;
    *feasible = rep.feasible ? 1 : 0;
    return 0;
  } catch (const std::exception& e) {
    return capi_status(e);
  }
}

extern "C" int rlhf_exec_plan_json(const char* strategy, int world, int batch_per_rank, int prompt_len, int gen_len,
                                   int micro_batches, int rollout_nums, int ppo_epochs, double inference_ratio,
                                   const double* ratios4, char* out, int out_len, int* needed) {
  try {
    StrategyConfig sc;
    sc.name = strategy ? strategy : "colocated";
    sc.inference_ratio = inference_ratio > 0 ? inference_ratio : 0.5;
    sc.tp_gen = 1;
    const ModelName order[4] = {ModelName::Actor, ModelName::Critic, ModelName::Ref, ModelName::Reward};
    if (ratios4)
      for (int i = 0; i < 4; ++i)
        if (ratios4[i] > 0) sc.ratios.push_back({order[i], ratios4[i]});
    const ExecPlan e = build_exec_plan(sc, world, batch_per_rank, prompt_len, gen_len, std::max(1, micro_batches),
                                       std::max(1, rollout_nums), std::max(1, ppo_epochs));
    const std::string js = to_json(e);
    if (needed) *needed = static_cast<int>(js.size()) + 1;
    if (out && out_len > 0) {
      const size_t n = std::min(js.size(), static_cast<size_t>(out_len - 1));
      std::memcpy(out, js.data(), n);
      out[n] = 0;
    }
    return 0;
  } catch (const std::exception& ex) {
    return capi_status(ex);
  }
}

extern "C" int rlhf_sim_run(const char* command, const char* json, char* out, int out_len, int* needed) {
  try {
    const std::string r = run_command(command ? command : "", json ? json : "");
    if (needed) *needed = static_cast<int>(r.size()) + 1;
    if (out && out_len > 0) {
      const size_t n = std::min(r.size(), static_cast<size_t>(out_len - 1));
      std::memcpy(out, r.data(), n);
      out[n] = 0;
    }
    return 0;
  } catch (const std::exception& ex) {
    return capi_status(ex);
  }
}
