// Memory arithmetic, parallel-config checks, analytic time formulas and calibration
// (reference costmodel.hpp:11-90, behaviour per /root/reference/SPEC.md:151-252).
#include "flexrlhf/costmodel.hpp"

#include "flexrlhf/simulator.hpp"

#include <algorithm>
#include <cmath>
#include <set>

#include "flexrlhf/errors.hpp"

namespace flexrlhf {

const char* to_string(CollectiveKind k) {
  switch (k) {
    case CollectiveKind::AllGather: return "AllGather";
    case CollectiveKind::ReduceScatter: return "ReduceScatter";
    case CollectiveKind::AllReduce: return "AllReduce";
    case CollectiveKind::AlltoAll: return "AlltoAll";
    case CollectiveKind::Broadcast: return "Broadcast";
    case CollectiveKind::P2P: return "P2P";
  }
  return "?";
}

void validate_parallel_cfg(const ParallelCfg& cfg, const ClusterTopology& t, bool trainable) {
  if (cfg.dp_degree < 1 || cfg.tp_degree < 1) throw ConfigError("parallel cfg: dp/tp must be >= 1");
  if (cfg.zero_level < 0 || cfg.zero_level > 3) throw ConfigError("parallel cfg: zero_level in 0..3");
  if (cfg.zero_level > 0 && !trainable)
    throw ConfigError("parallel cfg: zero_level > 0 on an inference model");
  if (static_cast<int>(cfg.devices.size()) != cfg.dp_degree * cfg.tp_degree)
    throw ConfigError("parallel cfg: |devices| != dp*tp");
  std::set<int> seen;
  for (int d : cfg.devices) {
    t.device(d);  // throws on unknown ids
    if (!seen.insert(d).second) throw ConfigError("parallel cfg: duplicate device");
  }
  // TP groups (consecutive tp_degree devices) must stay inside one node.
  for (int r = 0; r < cfg.dp_degree; ++r) {
    const int node = t.device(cfg.devices[static_cast<size_t>(r * cfg.tp_degree)]).node_id;
    for (int k = 1; k < cfg.tp_degree; ++k)
      if (t.device(cfg.devices[static_cast<size_t>(r * cfg.tp_degree + k)]).node_id != node)
        throw ConfigError("parallel cfg: tensor-parallel group spans nodes");
  }
}

double model_state_bytes(const ModelSpec& m, const ParallelCfg& cfg, const MemoryConstants& c) {
  const double P = m.param_count;
  const double tp = cfg.tp_degree, dp = cfg.dp_degree;
  if (!m.trainable) {
    if (cfg.zero_level != 0) throw ConfigError("model_state_bytes: ZeRO on an inference model");
    return c.bytes_infer_per_param / tp * P;
  }
  // bytes_train_per_param = 2 (param) + 2 (grad) + optimizer (12 by default).
  const double pb = 2.0, gb = 2.0, ob = c.bytes_train_per_param - 4.0;
  const double lf = m.lora_dim > 0 ? c.lora_fraction : 1.0;  // LoRA scales grad+opt only
  double per;
  switch (cfg.zero_level) {
    case 0: per = pb + (gb + ob) * lf; break;
    case 1: per = pb + gb * lf + ob * lf / dp; break;
    case 2: per = pb + (gb + ob) * lf / dp; break;
    case 3: per = (pb + (gb + ob) * lf) / dp; break;
    default: throw ConfigError("model_state_bytes: bad zero level");
  }
  return per / tp * P;
}

double activation_bytes(const PipelineSpec& p, const ModelSpec& m, const ParallelCfg& cfg,
                        const MemoryConstants& c) {
  // coeff * (batch/dp) * seq * sqrt(P) / tp; inference models keep
  // only the KV-cache-class share; checkpointing scales trainable activations.
  double v = c.activation_coeff * (static_cast<double>(p.batch_size) / cfg.dp_degree) * p.seq_len() *
             std::sqrt(m.param_count) / cfg.tp_degree;
  if (!m.trainable) v *= c.activation_infer_factor;
  else if (p.grad_checkpoint) v *= c.grad_ckpt_factor;
  return v;
}

double zero_step_comm_bytes(const ModelSpec& m, const ParallelCfg& cfg, const MemoryConstants&) {
  if (!m.trainable) throw ConfigError("zero_step_comm_bytes: inference model");
  if (cfg.dp_degree <= 1) return 0.0;
  const double grad = 2.0 * 2.0 * m.param_count / cfg.dp_degree / cfg.tp_degree;
  // Z3 adds the forward parameter all-gather and the backward re-gather.
  return cfg.zero_level == 3 ? 3.0 * grad : grad;
}

std::vector<int> dp_subgroup(const ParallelCfg& cfg) {
  std::vector<int> out;
  for (int r = 0; r < cfg.dp_degree; ++r)
    out.push_back(cfg.devices[static_cast<size_t>(r * cfg.tp_degree)]);
  return out;
}

double collective_time(CollectiveKind kind, double size, const std::vector<int>& group, const ClusterTopology& t,
                       const CommConstants& c) {
  if (size < 0) throw ConfigError("collective_time: negative size");
  const double n = static_cast<double>(group.size());
  if (kind == CollectiveKind::P2P) {
    const double B = group.size() >= 2 ? t.group_min_bandwidth(group) : t.intra_node_bw();
    return c.alpha + size / B;
  }
  if (group.size() < 2) throw ConfigError(std::string("collective_time: singleton group for ") + to_string(kind));
  const double B = t.group_min_bandwidth(group);
  const double ring = c.alpha * (n - 1) + ((n - 1) / n) * size / B;
  switch (kind) {
    case CollectiveKind::AllGather:
    case CollectiveKind::ReduceScatter:
    case CollectiveKind::AlltoAll: return ring;
    case CollectiveKind::AllReduce: return 2.0 * ring;
    case CollectiveKind::Broadcast: return c.alpha + size / B;
    default: return ring;
  }
}

double stage_compute_time(TaskKind kind, const ModelSpec& m, const ParallelCfg& cfg, const PipelineSpec& p,
                          const ClusterTopology& t, const CostModel& c) {
  if (cfg.devices.empty()) throw ConfigError("stage_compute_time: model not placed");
  const DeviceSpec& dev = t.device(cfg.devices.front());
  const double F = dev.peak_flops * cfg.tp_degree;
  if (F <= 0) throw ConfigError("stage_compute_time: zero flops");
  const double P = m.param_count;
  const double B_local = static_cast<double>(p.batch_size) / p.micro_batches / cfg.dp_degree;
  const double prompt = p.prompt_len, gen = p.gen_len;
  switch (kind) {
    case TaskKind::Generation: {
      const double mfu_gen = cfg.inference_runtime ? c.comm.mfu_gen_infer : c.comm.mfu_gen;
      const double prefill = 2.0 * P * B_local * prompt / (F * c.comm.mfu_fwd);
      const double per_tok = std::max(2.0 * P * B_local / (F * mfu_gen),
                                      c.mem.bytes_infer_per_param * P / cfg.tp_degree / dev.hbm_bandwidth);
      return prefill + gen * per_tok;
    }
    case TaskKind::Forward: return 2.0 * P * B_local * (prompt + gen) / (F * c.comm.mfu_fwd);
    case TaskKind::TrainFB: return 6.0 * P * B_local * (prompt + gen) / (F * c.comm.mfu_train);
    default: return 0.0;
  }
}

double task_zero_comm_time(TaskKind kind, const ModelSpec& m, const ParallelCfg& cfg, const PipelineSpec& p,
                           const ClusterTopology& t, const CostModel& c, bool last_micro_batch) {
  if (cfg.dp_degree <= 1) return 0.0;
  const std::vector<int> grp = dp_subgroup(cfg);
  const double shard_bytes = 2.0 * m.param_count / cfg.tp_degree;  // bf16 parameters of one TP shard
  double s = 0.0;
  if (m.trainable && cfg.zero_level == 3) {
    const double gather = collective_time(CollectiveKind::AllGather, shard_bytes, grp, t, c.comm);
    if (kind == TaskKind::Generation) s += (p.gen_len + 1.0) * gather;
    if (kind == TaskKind::Forward) s += gather;
    if (kind == TaskKind::TrainFB) s += 2.0 * gather;
  }
  if (m.trainable && kind == TaskKind::TrainFB && last_micro_batch)  // one gradient sync per epoch
    s += collective_time(CollectiveKind::AllReduce, shard_bytes, grp, t, c.comm);
  return s;
}

namespace {

// Simulated (generation, non-generation) seconds and totals of one observation.
struct Pred {
  double gen = 0, other = 0, total = 0;
};

Pred predict(const CalibrationObservation& o, const CostModel& cm) {
  SimOptions so;
  so.allow_infeasible = true;
  const SimReport r = simulate(*o.plan, *o.pipeline, cm, *o.topology, so);
  Pred p;
  p.total = r.step_seconds;
  auto it = r.per_stage_seconds.find(Stage::Generation);
  p.gen = it == r.per_stage_seconds.end() ? 0.0 : it->second;
  p.other = p.total - p.gen;
  return p;
}

// Log-space bisection of a decreasing function err(x) (simulated time falls as an MFU grows)
// for err(x) = 0, x in [lo, hi]; 200 halvings, deterministic.
template <typename F>
double bisect(F err, double lo, double hi) {
  double a = std::log(lo), b = std::log(hi);
  for (int i = 0; i < 200; ++i) {
    const double m = 0.5 * (a + b);
    (err(std::exp(m)) > 0 ? a : b) = m;
  }
  return std::exp(0.5 * (a + b));
}

}  // namespace

CommConstants calibrate(const CommConstants& c0, const std::vector<CalibrationObservation>& obs) {
  if (obs.empty()) throw ConfigError("calibrate: no observations");
  bool any = false;
  for (const auto& o : obs) {
    if (!o.plan || !o.pipeline || !o.topology) throw ConfigError("calibrate: incomplete observation");
    any |= o.measured_step_seconds > 0;
  }
  if (!any) throw ConfigError("calibrate: degenerate observations (all measured times zero)");
  CostModel cm;
  cm.comm = c0;
  const double lo = 1e-7, hi = 1.0;
  bool have_fraction = false;
  for (const auto& o : obs) have_fraction |= o.generation_fraction >= 0;
  if (have_fraction) {
    // (1) scale mfu_fwd and mfu_train together to the non-generation seconds
    const double f0 = cm.comm.mfu_fwd, t0 = cm.comm.mfu_train;
    const double smax = 1.0 / std::max(f0, t0);
    const double s = bisect(
        [&](double x) {
          CostModel k = cm;
          k.comm.mfu_fwd = f0 * x;
          k.comm.mfu_train = t0 * x;
          double e = 0;
          int n = 0;
          for (const auto& o : obs) {
            if (o.generation_fraction < 0 || o.measured_step_seconds <= 0) continue;
            const double target = o.measured_step_seconds * (1.0 - o.generation_fraction);
            e += (predict(o, k).other - target) / target;
            ++n;
          }
          return n ? e / n : 0.0;
        },
        lo / std::min(f0, t0), smax);
    cm.comm.mfu_fwd = f0 * s;
    cm.comm.mfu_train = t0 * s;
  }
  // (2) mfu_gen (mfu_gen_infer in proportion) to the generation seconds, or to the total
  const double g0 = cm.comm.mfu_gen, gi0 = cm.comm.mfu_gen_infer;
  const double ratio = g0 > 0 ? gi0 / g0 : 1.0;
  const double g = bisect(
      [&](double x) {
        CostModel k = cm;
        k.comm.mfu_gen = x;
        k.comm.mfu_gen_infer = std::min(1.0, x * ratio);
        double e = 0;
        int n = 0;
        for (const auto& o : obs) {
          if (o.measured_step_seconds <= 0) continue;
          const Pred p = predict(o, k);
          if (have_fraction && o.generation_fraction >= 0) {
            const double target = o.measured_step_seconds * o.generation_fraction;
            if (target > 0) e += (p.gen - target) / target, ++n;
          } else {
            e += (p.total - o.measured_step_seconds) / o.measured_step_seconds;
            ++n;
          }
        }
        return n ? e / n : 0.0;
      },
      lo, hi);
  cm.comm.mfu_gen = g;
  cm.comm.mfu_gen_infer = std::min(1.0, g * ratio);
  return cm.comm;
}

}  // namespace flexrlhf
