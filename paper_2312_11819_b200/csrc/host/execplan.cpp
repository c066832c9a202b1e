// execplan.cpp — see execplan.hpp.  Pure host logic.
#include "execplan.hpp"

#include <algorithm>
#include <sstream>

#include "flexrlhf/errors.hpp"

namespace flexrlhf {

const char* to_string(Field f) {
  switch (f) {
    case Field::Prompt: return "prompt";
    case Field::Tokens: return "tokens";
    case Field::LogpOld: return "logp_old";
    case Field::LogpRef: return "logp_ref";
    case Field::Values: return "values";
    case Field::Score: return "score";
  }
  return "?";
}

const char* to_string(StepKind k) {
  switch (k) {
    case StepKind::Exchange: return "exchange";
    case StepKind::Task: return "task";
    case StepKind::Experience: return "experience";
    case StepKind::OptimizerStep: return "optimizer_step";
  }
  return "?";
}

Field output_field(ModelName m) {
  switch (m) {
    case ModelName::Actor:
    case ModelName::ShadowActor: return Field::LogpOld;
    case ModelName::Ref: return Field::LogpRef;
    case ModelName::Critic:
    case ModelName::ShadowCritic: return Field::Values;
    case ModelName::Reward: return Field::Score;
  }
  return Field::Tokens;
}

std::vector<Transfer> plan_transfers(const std::vector<Segment>& src, const std::vector<Segment>& dst) {
  std::vector<Transfer> out;
  for (const Segment& s : src)
    for (const Segment& d : dst) {
      const int64_t lo = std::max(s.first_id, d.first_id);
      const int64_t hi = std::min(s.first_id + s.count, d.first_id + d.count);
      if (lo >= hi) continue;
      Transfer t;
      t.src_rank = s.rank;
      t.dst_rank = d.rank;
      t.src_row = s.row0 + (lo - s.first_id);
      t.dst_row = d.row0 + (lo - d.first_id);
      t.count = static_cast<int>(hi - lo);
      out.push_back(t);
    }
  return out;
}

bool ExecPlan::hosts(int rank, ModelName m) const {
  const int s = set_of[static_cast<int>(m)];
  return s >= 0 && member_index(s, rank) >= 0;
}

int ExecPlan::member_index(int set, int rank) const {
  const std::vector<int>& g = sets[set].group;
  for (size_t i = 0; i < g.size(); ++i)
    if (g[i] == rank) return static_cast<int>(i);
  return -1;
}

std::vector<Segment> ExecPlan::segments(int set, int r, int mb) const {
  std::vector<Segment> v;
  if (set < 0) {
    for (int k = 0; k < world; ++k)
      v.push_back(Segment{k, static_cast<int64_t>(r) * G + static_cast<int64_t>(k) * batch_per_rank, batch_per_rank,
                          static_cast<int64_t>(r) * batch_per_rank});
    return v;
  }
  const RowSet& s = sets[set];
  for (size_t i = 0; i < s.group.size(); ++i)
    v.push_back(Segment{s.group[i],
                        static_cast<int64_t>(r) * G + static_cast<int64_t>(mb) * Gm + static_cast<int64_t>(i) * s.per,
                        s.per, static_cast<int64_t>(r * M + mb) * s.per});
  return v;
}

int64_t ExecPlan::sample_id(int set, int rank, int row) const {
  const int i = member_index(set, rank);
  if (i < 0) return -1;
  const int per = sets[set].per;
  const int slot = row / per, within = row % per;
  const int r = slot / M, mb = slot % M;
  return static_cast<int64_t>(r) * G + static_cast<int64_t>(mb) * Gm + static_cast<int64_t>(i) * per + within;
}

int ExecPlan::experience_set(int rank) const {
  if (hosts(rank, ModelName::Actor)) return set_of[static_cast<int>(ModelName::Actor)];
  if (hosts(rank, ModelName::Critic)) return set_of[static_cast<int>(ModelName::Critic)];
  if (hosts(rank, generator)) return set_of[static_cast<int>(generator)];
  return -1;
}

ExecPlan build_exec_plan(const StrategyConfig& sc_in, int world, int batch_per_rank, int prompt_len, int gen_len,
                         int micro_batches, int rollouts, int epochs, const ModelSizes& sizes) {
  if (world < 1 || batch_per_rank < 1) throw ConfigError("world and batch must be >= 1");
  if (micro_batches < 1 || rollouts < 1 || epochs < 1)
    throw ConfigError("micro_batches, rollout_nums and ppo_epochs must be >= 1");
  StrategyConfig sc = sc_in;
  const StrategyTag tag = strategy_from_string(sc.name);
  if (tag == StrategyTag::Disaggregated && sc.tp_gen > 1)
    throw ConfigError("tp_gen > 1 (tensor-parallel shadow generation) is not executed; use tp_gen = 1");
  if (tag == StrategyTag::Disaggregated) sc.tp_gen = 1;
  if (sc.tp_degree > 1) throw ConfigError("tp_degree > 1 is not executed; models run data-parallel");

  ExecPlan e;
  e.world = world;
  e.batch_per_rank = batch_per_rank;
  e.prompt_len = prompt_len;
  e.gen_len = gen_len;
  e.G = world * batch_per_rank;
  e.M = micro_batches;
  e.rollouts = rollouts;
  e.epochs = epochs;
  if (e.G % e.M) throw ConfigError("world * batch must be divisible by micro_batches");
  e.Gm = e.G / e.M;
  e.tag = tag;

  ModelSizes sz = sizes;  // parameter counts only matter to the memory/cost formulas, not to execution
  if (sz.actor <= 0) sz.actor = 1.0e8;
  if (sz.critic <= 0) sz.critic = sz.actor;
  if (sz.ref <= 0) sz.ref = sz.actor;
  if (sz.reward <= 0) sz.reward = sz.critic;
  LoopParams lp;
  lp.batch_size = e.G;
  lp.prompt_len = prompt_len;
  lp.gen_len = gen_len;
  lp.micro_batches = micro_batches;
  lp.rollout_nums = rollouts;
  lp.ppo_epochs = epochs;
  const BuiltStrategy bs =
      build_strategy(sc, ClusterTopology::b200_box(world), build_pipeline(PipelineStructure::ACNonShare, sz, lp));
  e.plan = bs.plan;
  e.pipeline = bs.pipeline;
  const bool shadows = e.plan.has(ModelName::ShadowActor);
  e.generator = shadows ? ModelName::ShadowActor : ModelName::Actor;
  e.tasks = task_graph(e.pipeline, shadows);
  e.schedule = derive_comm_schedule(e.plan, e.pipeline, CostModel{});

  for (int mi = 0; mi < 6; ++mi) {
    const ModelName m = static_cast<ModelName>(mi);
    if (!e.plan.has(m)) continue;
    const std::vector<int>& g = e.plan.cfg(m).devices;
    int s = -1;
    for (size_t k = 0; k < e.sets.size(); ++k)
      if (e.sets[k].group == g) s = static_cast<int>(k);
    if (s < 0) {
      if (g.empty() || e.Gm % static_cast<int>(g.size()))
        throw ConfigError(std::string("micro-batch of ") + std::to_string(e.Gm) + " samples does not split over the " +
                          std::to_string(g.size()) + " devices of " + to_string(m));
      RowSet rs;
      rs.group = g;
      rs.per = e.Gm / static_cast<int>(g.size());
      rs.rows = rollouts * e.M * rs.per;
      e.sets.push_back(rs);
      s = static_cast<int>(e.sets.size()) - 1;
    }
    e.set_of[mi] = s;
  }
  const int gen_set = e.set_of[static_cast<int>(e.generator)];
  std::vector<int> trainer_sets;
  for (ModelName m : {ModelName::Actor, ModelName::Critic}) {
    const int s = e.set_of[static_cast<int>(m)];
    if (s >= 0 && std::find(trainer_sets.begin(), trainer_sets.end(), s) == trainer_sets.end()) trainer_sets.push_back(s);
  }

  // the CommOp an exchange realises: attached (Before / After) to one of the Forwards of the
  // same Generation (the schedule anchors at the first / last scorer it gates)
  auto find_op = [&](int fwd_task, AttachKind at) {
    const std::vector<int>& gen = e.tasks[fwd_task].depends_on;
    for (size_t i = 0; i < e.schedule.ops.size(); ++i) {
      const CommOp& c = e.schedule.ops[i];
      if (c.attach != at || c.anchor_task < 0) continue;
      const StageTask& a = e.tasks[c.anchor_task];
      if (a.kind == TaskKind::Forward && a.depends_on == gen) return static_cast<int>(i);
    }
    return -1;
  };
  auto move = [&](Field f, int src, int dst, int r, int mb) {
    Move mv;
    mv.field = f;
    mv.src_set = src;
    mv.dst_set = dst;
    mv.transfers = plan_transfers(e.segments(src, r, mb), e.segments(dst, r, mb));
    return mv;
  };

  bool experience_done = false;
  const int n = static_cast<int>(e.tasks.size());
  for (int i = 0; i < n; ++i) {
    const StageTask& t = e.tasks[i];
    const int r = t.rollout_index, mb = t.micro_batch_index;
    if (t.kind == TaskKind::Generation) {
      ExecStep x;
      x.kind = StepKind::Exchange;
      x.task = t.id;
      x.rollout = r;
      x.mb = mb;
      x.moves.push_back(move(Field::Prompt, -1, gen_set, r, mb));
      e.steps.push_back(x);
    }
    const bool fwd = t.kind == TaskKind::Forward;
    if (fwd && (i == 0 || e.tasks[i - 1].kind == TaskKind::Generation)) {
      // (query, response) to every scorer row set of this generation (Alg. 1 line 8 / Alg. 2 P2P)
      ExecStep x;
      x.kind = StepKind::Exchange;
      x.task = t.id;
      x.comm_op = find_op(t.id, AttachKind::Before);
      x.rollout = r;
      x.mb = mb;
      std::vector<int> done{gen_set};
      for (int j = i; j < n && e.tasks[j].kind == TaskKind::Forward && e.tasks[j].depends_on == t.depends_on; ++j) {
        const int s = e.set_of[static_cast<int>(e.tasks[j].model)];
        if (std::find(done.begin(), done.end(), s) != done.end()) continue;
        done.push_back(s);
        x.moves.push_back(move(Field::Tokens, gen_set, s, r, mb));
      }
      e.steps.push_back(x);
    }
    if (t.kind == TaskKind::TrainFB && !experience_done) {
      for (int s : trainer_sets) {  // experience-buffer barrier: rewards + GAE on each trainer row set
        ExecStep x;
        x.kind = StepKind::Experience;
        x.task = t.id;
        x.set = s;
        e.steps.push_back(x);
      }
      experience_done = true;
    }
    ExecStep ts;
    ts.kind = StepKind::Task;
    ts.task = t.id;
    ts.model = t.model;
    ts.rollout = r;
    ts.mb = mb;
    ts.epoch = t.epoch_index;
    e.steps.push_back(ts);
    if (fwd && (i + 1 == n || e.tasks[i + 1].kind != TaskKind::Forward || e.tasks[i + 1].depends_on != t.depends_on)) {
      // outputs (and the sequences) to the trainers' row sets (Alg. 1 line 12 AlltoAll / Alg. 2 Send)
      ExecStep x;
      x.kind = StepKind::Exchange;
      x.task = t.id;
      x.comm_op = find_op(t.id, AttachKind::After);
      x.attach = AttachKind::After;
      x.rollout = r;
      x.mb = mb;
      int first = i;
      while (first > 0 && e.tasks[first - 1].kind == TaskKind::Forward && e.tasks[first - 1].depends_on == t.depends_on)
        --first;
      for (int ts_set : trainer_sets) {
        bool has_tokens = ts_set == gen_set;  // the Before exchange already filled the scorer sets
        for (int j = first; j <= i; ++j) has_tokens |= e.set_of[static_cast<int>(e.tasks[j].model)] == ts_set;
        if (!has_tokens) x.moves.push_back(move(Field::Tokens, gen_set, ts_set, r, mb));
        for (int j = first; j <= i; ++j) {
          const ModelName m = e.tasks[j].model;
          const int s = e.set_of[static_cast<int>(m)];
          if (s != ts_set) x.moves.push_back(move(output_field(m), s, ts_set, r, mb));
        }
      }
      e.steps.push_back(x);
    }
    if (t.kind == TaskKind::TrainFB && mb == e.M - 1) {
      ExecStep o;
      o.kind = StepKind::OptimizerStep;
      o.task = t.id;
      o.model = t.model;
      o.epoch = t.epoch_index;
      e.steps.push_back(o);
    }
  }
  return e;
}

std::string to_json(const ExecPlan& e) {
  std::ostringstream o;
  o << "{\"strategy\":\"" << to_string(e.tag) << "\",\"world\":" << e.world << ",\"batch_per_rank\":" << e.batch_per_rank
    << ",\"G\":" << e.G << ",\"micro_batches\":" << e.M << ",\"rollouts\":" << e.rollouts << ",\"epochs\":" << e.epochs
    << ",\"generator\":\"" << to_string(e.generator) << "\",\"sets\":[";
  for (size_t i = 0; i < e.sets.size(); ++i) {
    o << (i ? "," : "") << "{\"group\":[";
    for (size_t k = 0; k < e.sets[i].group.size(); ++k) o << (k ? "," : "") << e.sets[i].group[k];
    o << "],\"per\":" << e.sets[i].per << ",\"rows\":" << e.sets[i].rows << "}";
  }
  o << "],\"set_of\":{";
  bool first = true;
  for (int m = 0; m < 6; ++m) {
    if (e.set_of[m] < 0) continue;
    o << (first ? "" : ",") << "\"" << to_string(static_cast<ModelName>(m)) << "\":" << e.set_of[m];
    first = false;
  }
  o << "},\"tasks\":[";
  for (size_t i = 0; i < e.tasks.size(); ++i) {
    const StageTask& t = e.tasks[i];
    o << (i ? "," : "") << "{\"id\":" << t.id << ",\"kind\":\"" << to_string(t.kind) << "\",\"model\":\""
      << to_string(t.model) << "\",\"mb\":" << t.micro_batch_index << ",\"rollout\":" << t.rollout_index
      << ",\"epoch\":" << t.epoch_index << "}";
  }
  o << "],\"comm_ops\":[";
  for (size_t i = 0; i < e.schedule.ops.size(); ++i) {
    const CommOp& c = e.schedule.ops[i];
    o << (i ? "," : "") << "{\"kind\":\"" << to_string(c.kind) << "\",\"anchor\":" << c.anchor_task
      << ",\"attach\":\"" << (c.attach == AttachKind::Before ? "before" : "after") << "\",\"payload\":"
      << c.payload_bytes << "}";
  }
  o << "],\"steps\":[";
  for (size_t i = 0; i < e.steps.size(); ++i) {
    const ExecStep& s = e.steps[i];
    o << (i ? "," : "") << "{\"kind\":\"" << to_string(s.kind) << "\",\"task\":" << s.task << ",\"comm_op\":" << s.comm_op
      << ",\"attach\":\"" << (s.attach == AttachKind::Before ? "before" : "after") << "\",\"set\":" << s.set
      << ",\"model\":\"" << to_string(s.model) << "\",\"rollout\":" << s.rollout << ",\"mb\":" << s.mb
      << ",\"epoch\":" << s.epoch << ",\"moves\":[";
    for (size_t k = 0; k < s.moves.size(); ++k) {
      const Move& m = s.moves[k];
      o << (k ? "," : "") << "{\"field\":\"" << to_string(m.field) << "\",\"src_set\":" << m.src_set
        << ",\"dst_set\":" << m.dst_set << ",\"transfers\":[";
      for (size_t q = 0; q < m.transfers.size(); ++q) {
        const Transfer& t = m.transfers[q];
        o << (q ? "," : "") << "[" << t.src_rank << "," << t.dst_rank << "," << t.src_row << "," << t.dst_row << ","
          << t.count << "]";
      }
      o << "]}";
    }
    o << "]}";
  }
  o << "]}";
  return o.str();
}

}  // namespace flexrlhf
