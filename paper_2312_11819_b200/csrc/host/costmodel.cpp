// Memory arithmetic + parallel-config checks (reference costmodel.hpp:36-74,
// behaviour per /root/reference/SPEC.md:164-205).
#include "flexrlhf/costmodel.hpp"

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

}  // namespace flexrlhf
