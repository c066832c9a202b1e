// ref_shim.cpp — C entry points over the COMPILED REFERENCE (test infrastructure).
//
// Built by oracle/Makefile together with the reference's own sources
// /root/reference/proj/src/{topology,workload}.cpp (never copied into this
// repo) into oracle/_ref/librlhfsim_ref.so.  The tests call these functions to
// pin the engine's host logic (task DAG, topology queries) against the
// reference implementation itself.  Only topology + workload are compiled:
// every other reference module is declaration-only.
#include <cstring>
#include <exception>
#include <string>

#include "rlhfsim/errors.hpp"
#include "rlhfsim/topology.hpp"
#include "rlhfsim/workload.hpp"

namespace {
thread_local std::string g_err;
int code_of(const std::exception& e) {
  if (dynamic_cast<const rlhfsim::ConfigError*>(&e)) return rlhfsim::ConfigError::exit_code;
  return 1;
}
}  // namespace

extern "C" const char* ref_last_error() { return g_err.c_str(); }

// Same flattening as rlhf_task_graph in include/rlhf_engine.h.
extern "C" int ref_task_graph(int structure, int batch, int micro_batches, int rollout_nums, int ppo_epochs,
                              int shadows, double actor, double critic, double ref, double reward,
                              int max_tasks, int max_deps, int* n_tasks, int* n_deps, int* kind, int* model,
                              int* mb, int* rollout, int* epoch, int* dep_off, int* deps) {
  try {
    rlhfsim::ModelSizes sz;
    sz.actor = actor;
    sz.critic = critic;
    sz.ref = ref;
    sz.reward = reward;
    rlhfsim::LoopParams lp;
    lp.batch_size = batch;
    lp.micro_batches = micro_batches;
    lp.rollout_nums = rollout_nums;
    lp.ppo_epochs = ppo_epochs;
    auto p = rlhfsim::build_pipeline(structure ? rlhfsim::PipelineStructure::ACNonShare
                                               : rlhfsim::PipelineStructure::ACShare,
                                     sz, lp);
    if (shadows > 1) p = rlhfsim::with_shadows(p);  // 2: add shadows, 1: request without adding
    auto g = rlhfsim::task_graph(p, shadows != 0);
    int nd = 0;
    for (auto& t : g) nd += static_cast<int>(t.depends_on.size());
    *n_tasks = static_cast<int>(g.size());
    *n_deps = nd;
    if (max_tasks == 0) return 0;
    if (max_tasks < *n_tasks || max_deps < nd) return 2;
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
    g_err = e.what();
    return code_of(e);
  }
}

// group_min_bandwidth / bandwidth_between over a 1- or 2-group topology.
extern "C" int ref_topology_query(int groups, const int* nodes, const int* dpn, const char* const* kinds,
                                  double intra, double inter, double intertype, int n_group,
                                  const int* group, double* out_min_bw, int* out_devices, int* out_nodes) {
  try {
    rlhfsim::TopologySpec s;
    for (int i = 0; i < groups; ++i) {
      rlhfsim::NodeGroupSpec g;
      g.nodes = nodes[i];
      g.devices_per_node = dpn[i];
      g.kind = kinds[i];
      s.groups.push_back(g);
    }
    s.intra_node_bw = intra;
    s.inter_node_bw = inter;
    s.inter_type_bw = intertype;
    auto t = rlhfsim::ClusterTopology::build(s);
    *out_devices = t.device_count();
    *out_nodes = t.node_count();
    if (n_group > 0) *out_min_bw = t.group_min_bandwidth(std::vector<int>(group, group + n_group));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return code_of(e);
  }
}
