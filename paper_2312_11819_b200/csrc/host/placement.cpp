// Placement strategies + communication schedule.
// Reference declarations: /root/reference/proj/include/rlhfsim/placement.hpp:45-117;
// behaviour: /root/reference/SPEC.md:273-331 (ops) and :350-353 (design decisions).
#include "flexrlhf/placement.hpp"

#include <algorithm>
#include <cmath>
#include <set>
#include <sstream>

#include "flexrlhf/errors.hpp"

namespace flexrlhf {

const char* to_string(StrategyTag s) {
  switch (s) {
    case StrategyTag::Colocated: return "colocated";
    case StrategyTag::Interleaving1: return "interleaving1";
    case StrategyTag::Interleaving2: return "interleaving2";
    case StrategyTag::Disaggregated: return "disaggregated";
    case StrategyTag::HeteroDisaggregated: return "hetero_disaggregated";
    case StrategyTag::TrlxStandalone: return "trlx_standalone";
    case StrategyTag::TrlxCoexisted: return "trlx_coexisted";
    case StrategyTag::RatioVector: return "ratio_vector";
  }
  return "?";
}

StrategyTag strategy_from_string(const std::string& s) {
  for (StrategyTag t : {StrategyTag::Colocated, StrategyTag::Interleaving1, StrategyTag::Interleaving2,
                        StrategyTag::Disaggregated, StrategyTag::HeteroDisaggregated,
                        StrategyTag::TrlxStandalone, StrategyTag::TrlxCoexisted,
                        StrategyTag::RatioVector})
    if (s == to_string(t)) return t;
  throw ConfigError("unknown strategy: " + s);
}

const char* to_string(DeviceRole r) {
  switch (r) {
    case DeviceRole::Training: return "training";
    case DeviceRole::Inference: return "inference";
    case DeviceRole::Mixed: return "mixed";
  }
  return "?";
}

const ParallelCfg& PlacementPlan::cfg(ModelName m) const {
  auto it = assignments.find(m);
  if (it == assignments.end()) throw ConfigError(std::string("plan does not place ") + to_string(m));
  return it->second;
}

std::string PlacementPlan::encoding() const {
  std::ostringstream os;
  os << to_string(strategy_tag) << (hybrid_engine ? "+he" : "");
  for (const auto& [m, c] : assignments) {
    os << '|' << to_string(m) << ":dp" << c.dp_degree << "tp" << c.tp_degree << "z"
       << c.zero_level << (c.inference_runtime ? "i" : "") << '[';
    for (size_t i = 0; i < c.devices.size(); ++i) os << (i ? "," : "") << c.devices[i];
    os << ']';
  }
  return os.str();
}

std::vector<ModelName> PlacementPlan::models_on(int device) const {
  std::vector<ModelName> out;
  for (const auto& [m, c] : assignments)
    if (std::find(c.devices.begin(), c.devices.end(), device) != c.devices.end()) out.push_back(m);
  return out;
}

namespace {

ParallelCfg make_cfg(std::vector<int> devices, int tp, int zero, bool inference_runtime) {
  ParallelCfg c;
  c.tp_degree = tp;
  c.dp_degree = static_cast<int>(devices.size()) / tp;
  c.zero_level = zero;
  c.devices = std::move(devices);
  c.inference_runtime = inference_runtime;
  return c;
}

std::vector<int> all_devices(const ClusterTopology& t) {
  std::vector<int> v(static_cast<size_t>(t.device_count()));
  for (int i = 0; i < t.device_count(); ++i) v[static_cast<size_t>(i)] = i;
  return v;
}

bool is_trainable(const PipelineSpec& p, ModelName m) {
  return p.has_model(m) && p.model(m).trainable;
}

}  // namespace

PlacementPlan apply_ratio(const PlacementRatioVector& rv, const ClusterTopology& t,
                          const PipelineSpec& p, int zero_level) {
  // ceil(ratio*n) devices per model, node-major.  Sub-unit ratios take the next
  // devices from a shared wrapping cursor, so equal sub-unit ratios listed in
  // declaration order land on disjoint sets:
  // [1,1,.5,.5] on 8 -> Ref 0-3, Reward 4-7.
  const int n = t.device_count();
  PlacementPlan plan;
  plan.strategy_tag = StrategyTag::RatioVector;
  int cursor = 0;
  for (const auto& [m, r] : rv.ratios) {
    if (!(r > 0.0) || r > 1.0) throw ConfigError("apply_ratio: ratio must be in (0,1]");
    if (!p.has_model(m)) throw ConfigError(std::string("apply_ratio: pipeline lacks ") + to_string(m));
    const int k = static_cast<int>(std::ceil(r * n - 1e-9));
    if (k < 1 || r * n < 1.0 - 1e-9)
      throw ConfigError(std::string("apply_ratio: ratio gives 0 devices for ") + to_string(m));
    std::vector<int> devs;
    if (k >= n) {
      devs = all_devices(t);
    } else {
      for (int i = 0; i < k; ++i) devs.push_back((cursor + i) % n);
      std::sort(devs.begin(), devs.end());
      cursor = (cursor + k) % n;
    }
    const bool train = is_trainable(p, m);
    plan.assignments[m] = make_cfg(devs, 1, train ? zero_level : 0, false);
  }
  for (int d = 0; d < n; ++d) plan.device_role[d] = DeviceRole::Mixed;
  return plan;
}

PlacementPlan colocated_plan(const ClusterTopology& t, const PipelineSpec& p, bool hybrid_engine,
                             int zero_level, int tp_degree) {
  // Every model on every device, all roles mixed.
  const int n = t.device_count();
  if (tp_degree < 1 || n % tp_degree) throw ConfigError("colocated_plan: tp must divide device count");
  PlacementPlan plan;
  plan.strategy_tag = StrategyTag::Colocated;
  plan.hybrid_engine = hybrid_engine;
  for (const ModelSpec& m : p.models) {
    ParallelCfg c = make_cfg(all_devices(t), tp_degree, m.trainable ? zero_level : 0, false);
    validate_parallel_cfg(c, t, m.trainable);
    plan.assignments[m.name] = c;
  }
  for (int d = 0; d < n; ++d) plan.device_role[d] = DeviceRole::Mixed;
  return plan;
}

PlacementPlan interleaving_plan(const ClusterTopology& t, const PipelineSpec& p, int variant,
                                int zero_level) {
  // v1: {Actor 1, Critic 1, Ref .5, Reward .5}; v2: Actor/Critic also halved
  // on disjoint halves.
  if (t.device_count() < 2) throw ConfigError("interleaving_plan: needs >= 2 devices");
  if (variant != 1 && variant != 2) throw ConfigError("interleaving_plan: variant must be 1 or 2");
  if (variant == 2 && !p.has_model(ModelName::Critic))
    throw ConfigError("interleaving_plan: variant 2 requires a separate Critic (AC-NonShare)");
  PlacementRatioVector rv;
  const double ac = variant == 1 ? 1.0 : 0.5;
  rv.ratios.push_back({ModelName::Actor, ac});
  if (p.has_model(ModelName::Critic)) rv.ratios.push_back({ModelName::Critic, ac});
  rv.ratios.push_back({ModelName::Ref, 0.5});
  rv.ratios.push_back({ModelName::Reward, 0.5});
  PlacementPlan plan = apply_ratio(rv, t, p, zero_level);
  plan.strategy_tag = variant == 1 ? StrategyTag::Interleaving1 : StrategyTag::Interleaving2;
  return plan;
}

PlacementPlan disaggregated_plan(const ClusterTopology& t, const PipelineSpec& p,
                                 const DisaggregatedOptions& o) {
  // Training devices first, inference devices last (Fig. 4: trainers W1-W2,
  // inference W3-W4); roles partition the devices.
  if (!p.has_model(ModelName::ShadowActor))
    throw ConfigError("disaggregated_plan: pipeline must carry shadow models (with_shadows)");
  if (!(o.inference_ratio > 0.0 && o.inference_ratio < 1.0))
    throw ConfigError("disaggregated_plan: inference_ratio must be in (0,1)");
  const int n = t.device_count();
  int n_inf = static_cast<int>(std::lround(o.inference_ratio * n));
  n_inf = std::max(1, std::min(n - 1, n_inf));
  if (n < 2) throw ConfigError("disaggregated_plan: needs >= 2 devices");
  const int n_train = n - n_inf;
  int max_width = 0;
  for (int nd = 0; nd < t.node_count(); ++nd) max_width = std::max(max_width, t.node_width(nd));
  if (o.tp_gen < 1 || o.tp_gen > max_width)
    throw ConfigError("disaggregated_plan: tp_gen exceeds node width");
  if (n_inf % o.tp_gen) throw ConfigError("disaggregated_plan: tp_gen must divide inference devices");

  std::vector<int> train, infer;
  for (int d = 0; d < n; ++d) (d < n_train ? train : infer).push_back(d);
  PlacementPlan plan;
  plan.strategy_tag = StrategyTag::Disaggregated;
  for (ModelName m : {ModelName::Actor, ModelName::Critic})
    if (p.has_model(m)) {
      ParallelCfg c = make_cfg(train, 1, o.zero_train, false);
      validate_parallel_cfg(c, t, true);
      plan.assignments[m] = c;
    }
  {
    ParallelCfg c = make_cfg(infer, o.tp_gen, 0, true);
    validate_parallel_cfg(c, t, false);
    plan.assignments[ModelName::ShadowActor] = c;
  }
  for (ModelName m : {ModelName::ShadowCritic, ModelName::Ref, ModelName::Reward})
    if (p.has_model(m)) plan.assignments[m] = make_cfg(infer, 1, 0, true);
  for (int d : train) plan.device_role[d] = DeviceRole::Training;
  for (int d : infer) plan.device_role[d] = DeviceRole::Inference;
  return plan;
}

CommSchedule derive_comm_schedule(const PlacementPlan& plan, const PipelineSpec& p,
                                  const CostModel& c) {
  const bool shadows = plan.has(ModelName::ShadowActor);
  const std::vector<StageTask> tasks = task_graph(p, shadows);
  const double B = p.batch_size, S = p.seq_len(), R = p.gen_len;
  const double mbB = B / p.micro_batches;
  CommSchedule s;
  auto union_of = [&](std::initializer_list<ModelName> ms) {
    std::set<int> u;
    for (ModelName m : ms)
      if (plan.has(m))
        for (int d : plan.cfg(m).devices) u.insert(d);
    return std::vector<int>(u.begin(), u.end());
  };
  auto train_ids = [&](int epoch) {
    std::vector<int> v;
    for (const StageTask& t : tasks)
      if (t.kind == TaskKind::TrainFB && t.epoch_index == epoch) v.push_back(t.id);
    return v;
  };

  const StrategyTag tag = plan.strategy_tag;
  if (tag == StrategyTag::Colocated) {
    if (plan.hybrid_engine) {
      // One AllGather of 2*P_actor over the Actor group per Generation.
      for (const StageTask& t : tasks)
        if (t.kind == TaskKind::Generation) {
          CommOp op;
          op.kind = CollectiveKind::AllGather;
          op.model = t.model;
          op.group = plan.cfg(ModelName::Actor).devices;
          op.payload_bytes = 2.0 * p.model(ModelName::Actor).param_count;
          op.attach = AttachKind::Before;
          op.anchor_task = t.id;
          op.stage = Stage::Generation;
          op.gates = {t.id};
          s.ops.push_back(op);
        }
    }
    return s;
  }

  if (tag == StrategyTag::Interleaving1 || tag == StrategyTag::Interleaving2 ||
      tag == StrategyTag::RatioVector) {
    // Alg. 1: AllGather (Query,Response) before the Ref/Reward forwards, AlltoAll
    // of their outputs after -- exactly one pair per rollout.
    const std::vector<int> grp = union_of({ModelName::Ref, ModelName::Reward});
    if (grp.size() < 2) return s;
    for (int r = 0; r < p.rollout_nums; ++r) {
      std::vector<int> gens, scorer_fwds;
      for (const StageTask& t : tasks) {
        if (t.rollout_index != r) continue;
        if (t.kind == TaskKind::Generation) gens.push_back(t.id);
        if (t.kind == TaskKind::Forward && (t.model == ModelName::Ref || t.model == ModelName::Reward))
          scorer_fwds.push_back(t.id);
      }
      if (scorer_fwds.empty()) continue;
      CommOp ag;
      ag.kind = CollectiveKind::AllGather;
      ag.model = ModelName::Ref;
      ag.group = grp;
      ag.payload_bytes = B * S * c.comm.token_record_bytes;
      ag.attach = AttachKind::Before;
      ag.anchor_task = scorer_fwds.front();
      ag.stage = Stage::Forward;
      ag.deps = gens;
      ag.gates = scorer_fwds;
      s.ops.push_back(ag);
      CommOp a2a;
      a2a.kind = CollectiveKind::AlltoAll;
      a2a.model = ModelName::Reward;
      a2a.group = grp;
      // Ref per-token logprobs + Reward scalar score.
      a2a.payload_bytes = B * (R + 1.0) * c.comm.output_record_bytes;
      a2a.attach = AttachKind::After;
      a2a.anchor_task = scorer_fwds.back();
      a2a.stage = Stage::Forward;
      a2a.deps = scorer_fwds;
      a2a.gates = train_ids(0);
      s.ops.push_back(a2a);
    }
    return s;
  }

  if (tag == StrategyTag::Disaggregated) {
    // Alg. 2: per micro-batch P2P distribution before and after the inference
    // forwards plus a Send of the outputs to the trainers; one ParamSync per
    // synced model.
    const std::vector<int> inf = union_of({ModelName::ShadowActor, ModelName::ShadowCritic,
                                           ModelName::Ref, ModelName::Reward});
    const std::vector<int> trn = union_of({ModelName::Actor, ModelName::Critic});
    std::vector<int> both = inf;
    both.insert(both.end(), trn.begin(), trn.end());
    std::sort(both.begin(), both.end());
    for (const StageTask& g : tasks) {
      if (g.kind != TaskKind::Generation) continue;
      std::vector<int> fwds;
      for (const StageTask& t : tasks)
        if (t.kind == TaskKind::Forward && t.depends_on.size() == 1 && t.depends_on[0] == g.id)
          fwds.push_back(t.id);
      if (fwds.empty()) continue;
      CommOp in;
      in.kind = CollectiveKind::P2P;
      in.model = ModelName::ShadowActor;
      in.group = inf;
      in.payload_bytes = mbB * S * c.comm.token_record_bytes;
      in.attach = AttachKind::Before;
      in.anchor_task = fwds.front();
      in.stage = Stage::Forward;
      in.deps = {g.id};
      in.gates = fwds;
      s.ops.push_back(in);
      CommOp out = in;
      out.attach = AttachKind::After;
      out.anchor_task = fwds.back();
      out.payload_bytes = mbB * (3.0 * R + 1.0) * c.comm.output_record_bytes;
      out.deps = fwds;
      out.gates = {};
      s.ops.push_back(out);
      CommOp send = out;
      send.group = both;
      send.model = ModelName::Actor;
      // tokens + the four per-sample outputs, to the training devices
      send.payload_bytes = mbB * (S * c.comm.token_record_bytes + (3.0 * R + 1.0) * c.comm.output_record_bytes);
      send.gates = train_ids(0);
      s.ops.push_back(send);
    }
    for (const StageTask& t : tasks) {
      if (t.kind != TaskKind::ParamSync) continue;
      const ModelName src = t.model == ModelName::ShadowActor ? ModelName::Actor : ModelName::Critic;
      CommOp ps;
      ps.kind = CollectiveKind::Broadcast;
      ps.model = t.model;
      std::set<int> u(plan.cfg(src).devices.begin(), plan.cfg(src).devices.end());
      for (int d : plan.cfg(t.model).devices) u.insert(d);
      ps.group.assign(u.begin(), u.end());
      ps.payload_bytes = 2.0 * p.model(src).param_count;
      ps.attach = AttachKind::Before;
      ps.anchor_task = t.id;
      ps.stage = Stage::Sync;
      ps.deps = t.depends_on;
      ps.gates = {t.id};
      s.ops.push_back(ps);
    }
    return s;
  }
  throw ConfigError(std::string("derive_comm_schedule: unsupported strategy ") + to_string(tag));
}

FeasibilityReport validate_plan(const PlacementPlan& plan, const PipelineSpec& p,
                                const CostModel& c, const ClusterTopology& t) {
  FeasibilityReport rep;
  for (const auto& [m, cfg] : plan.assignments) {
    if (!p.has_model(m)) continue;
    const ModelSpec& ms = p.model(m);
    const double bytes = model_state_bytes(ms, cfg, c.mem) + activation_bytes(p, ms, cfg, c.mem);
    for (int d : cfg.devices) rep.per_device_bytes[d] += bytes;
  }
  for (const auto& [d, req] : rep.per_device_bytes) {
    const double budget = c.mem.oom_threshold * t.device(d).memory_bytes;
    if (req > budget) {
      rep.feasible = false;
      rep.offenders.push_back({d, req, budget, req - budget});
    }
  }
  return rep;
}

BuiltStrategy build_strategy(const StrategyConfig& sc, const ClusterTopology& t,
                             const PipelineSpec& base) {
  BuiltStrategy b;
  b.pipeline = base;
  const StrategyTag tag = strategy_from_string(sc.name);
  switch (tag) {
    case StrategyTag::Colocated:
      b.plan = colocated_plan(t, base, sc.hybrid_engine, sc.zero_level, sc.tp_degree);
      break;
    case StrategyTag::Interleaving1:
    case StrategyTag::Interleaving2:
      b.plan = interleaving_plan(t, base, tag == StrategyTag::Interleaving1 ? 1 : 2, sc.zero_level);
      break;
    case StrategyTag::Disaggregated: {
      b.pipeline = with_shadows(base);
      DisaggregatedOptions o;
      o.inference_ratio = sc.inference_ratio;
      o.tp_gen = sc.tp_gen;
      o.zero_train = sc.zero_level;
      o.gen_nodes = sc.gen_nodes;
      b.plan = disaggregated_plan(t, b.pipeline, o);
      break;
    }
    case StrategyTag::RatioVector: {
      PlacementRatioVector rv;
      rv.ratios = sc.ratios;
      b.plan = apply_ratio(rv, t, base, sc.zero_level);
      break;
    }
    default:
      throw ConfigError("build_strategy: strategy not supported on a homogeneous B200 box: " + sc.name);
  }
  return b;
}

}  // namespace flexrlhf
