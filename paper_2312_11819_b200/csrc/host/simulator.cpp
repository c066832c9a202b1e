// simulator.cpp — analytic simulation, trace, report, max-batch search, strategy comparison,
// scenario config and planner (flexrlhf/simulator.hpp).  Pure host logic.
//
// Behaviour follows /root/reference/SPEC.md:369-547 (the reference declares these in
// simulator.hpp:12-64, report.hpp:11-15, scenario.hpp:28-52, planner.hpp:10-37 and defines
// none of them).
#include "flexrlhf/simulator.hpp"

#include <algorithm>
#include <cmath>
#include <cctype>
#include <cstdio>
#include <cstring>
#include <exception>
#include <limits>
#include <set>
#include <sstream>

#include "flexrlhf/errors.hpp"

namespace flexrlhf {

namespace {

std::string fmt(double v, int prec = 9) {
  char b[64];
  std::snprintf(b, sizeof b, "%.*g", prec, v);
  return b;
}

const char* stage_name(Stage s) { return to_string(s); }

}  // namespace

double SimReport::device_idle_fraction(int device) const {
  auto it = per_device_busy_seconds.find(device);
  const double busy = it == per_device_busy_seconds.end() ? 0.0 : it->second;
  return step_seconds > 0 ? std::max(0.0, 1.0 - busy / step_seconds) : 0.0;
}

std::map<Stage, double> attribute_stages(const std::vector<SimEvent>& ev, double span) {
  std::map<Stage, double> out;
  for (Stage s : {Stage::Generation, Stage::Forward, Stage::Training, Stage::Sync}) out[s] = 0.0;
  std::vector<double> cut{0.0, span};
  for (const SimEvent& e : ev) {
    cut.push_back(e.start);
    cut.push_back(e.end);
  }
  std::sort(cut.begin(), cut.end());
  cut.erase(std::unique(cut.begin(), cut.end()), cut.end());
  double pending = 0;
  Stage last = Stage::Generation;
  for (size_t k = 0; k + 1 < cut.size(); ++k) {
    const double t0 = cut[k], t1 = std::min(cut[k + 1], span), mid = 0.5 * (t0 + t1);
    if (t1 <= t0 || t0 >= span) continue;
    int comp = 99, comm = 99;
    for (const SimEvent& e : ev)
      if (e.start <= mid && mid < e.end) {
        int& tgt = e.comm_lane ? comm : comp;
        tgt = std::min(tgt, static_cast<int>(e.stage));
      }
    const int st = comp < 99 ? comp : comm;
    if (st == 99) {
      pending += t1 - t0;
      continue;
    }
    out[static_cast<Stage>(st)] += t1 - t0 + pending;
    pending = 0;
    last = static_cast<Stage>(st);
  }
  out[last] += pending;
  return out;
}

SimReport simulate(const PlacementPlan& plan, const PipelineSpec& p, const CostModel& c, const ClusterTopology& t,
                   const SimOptions& opts) {
  if (opts.iterations < 1) throw ConfigError("simulate: iterations must be >= 1");
  const FeasibilityReport fr = validate_plan(plan, p, c, t);
  if (!fr.feasible && !opts.allow_infeasible) {
    const auto& o = fr.offenders.front();
    throw InfeasibleError("simulate: plan exceeds memory on device " + std::to_string(o.device) + " (" +
                          fmt(o.required_bytes / 1e9, 5) + " GB needed, " + fmt(o.budget_bytes / 1e9, 5) + " GB budget)");
  }
  const bool shadows = plan.has(ModelName::ShadowActor);
  const std::vector<StageTask> tasks = task_graph(p, shadows);
  const CommSchedule sched = derive_comm_schedule(plan, p, c);
  for (const StageTask& tk : tasks)
    if (tk.kind != TaskKind::Barrier && !plan.has(tk.model))
      throw ConfigError(std::string("simulate: task references unplaced model ") + to_string(tk.model));

  std::map<int, double> comp_free, comm_free, busy;
  auto free_at = [&](const std::vector<int>& devs, bool comm) {
    double f = 0;
    for (int d : devs) {
      const double a = comp_free[d], b = comm_free[d];
      f = std::max(f, opts.overlap ? (comm ? b : a) : std::max(a, b));
    }
    return f;
  };
  auto occupy = [&](const std::vector<int>& devs, bool comm, double end) {
    for (int d : devs) {
      if (!opts.overlap || !comm) comp_free[d] = std::max(comp_free[d], end);
      if (!opts.overlap || comm) comm_free[d] = std::max(comm_free[d], end);
    }
  };

  SimReport r;
  r.feasible = fr.feasible;
  r.per_device_mem_peak = fr.per_device_bytes;
  double t0 = 0, makespan = 0;
  for (int it = 0; it < opts.iterations; ++it) {
    std::vector<double> tend(tasks.size(), t0), gate(tasks.size(), t0);
    auto run_op = [&](const CommOp& op) {
      double ready = t0;
      for (int d : op.deps) ready = std::max(ready, tend[static_cast<size_t>(d)]);
      const double dur = op.group.size() >= 2 || op.kind == CollectiveKind::P2P
                             ? collective_time(op.kind, op.payload_bytes, op.group, t, c.comm)
                             : 0.0;
      const double start = std::max(ready, free_at(op.group, true));
      const double end = start + dur;
      occupy(op.group, true, end);
      for (int g : op.gates) gate[static_cast<size_t>(g)] = std::max(gate[static_cast<size_t>(g)], end);
      SimEvent e;
      e.task_id = op.anchor_task;
      e.kind = TaskKind::Collective;
      e.model = op.model;
      e.stage = op.stage;
      e.comm_lane = true;
      e.start = start;
      e.end = end;
      e.devices = op.group;
      r.events.push_back(e);
      makespan = std::max(makespan, end);
    };
    for (size_t i = 0; i < tasks.size(); ++i) {
      const StageTask& tk = tasks[i];
      for (const CommOp& op : sched.ops)
        if (op.anchor_task == tk.id && op.attach == AttachKind::Before) run_op(op);
      double ready = gate[i];
      for (int d : tk.depends_on) ready = std::max(ready, tend[static_cast<size_t>(d)]);
      std::vector<int> devs;
      double dur = 0;
      if (tk.kind != TaskKind::Barrier) {
        const ParallelCfg& cfg = plan.cfg(tk.model);
        devs = cfg.devices;
        if (tk.kind != TaskKind::ParamSync) {
          const ModelSpec& ms = p.model(tk.model);
          dur = stage_compute_time(tk.kind, ms, cfg, p, t, c) +
                task_zero_comm_time(tk.kind, ms, cfg, p, t, c, tk.micro_batch_index == p.micro_batches - 1);
        }
      }
      const double start = std::max(ready, devs.empty() ? 0.0 : free_at(devs, false));
      const double end = start + dur;
      if (dur > 0) occupy(devs, false, end);
      tend[i] = end;
      for (int d : devs) busy[d] += dur;
      SimEvent e;
      e.task_id = tk.id;
      e.kind = tk.kind;
      e.model = tk.model;
      e.micro_batch = tk.micro_batch_index;
      e.stage = stage_of(tk.kind);
      e.start = start;
      e.end = end;
      e.devices = devs;
      r.events.push_back(e);
      makespan = std::max(makespan, end);
      for (const CommOp& op : sched.ops)
        if (op.anchor_task == tk.id && op.attach == AttachKind::After) run_op(op);
    }
    t0 = makespan;  // synchronous PPO: the next iteration starts after ParamSync / the last TrainFB
  }
  r.step_seconds = makespan / opts.iterations;
  r.throughput_samples_per_sec = r.step_seconds > 0 ? p.batch_size * p.rollout_nums / r.step_seconds : 0.0;
  std::map<Stage, double> st = attribute_stages(r.events, makespan);
  for (auto& [s, v] : st) {
    r.per_stage_seconds[s] = v / opts.iterations;
    r.per_stage_fraction[s] = makespan > 0 ? v / makespan : 0.0;
  }
  for (const auto& [d, b] : busy) r.per_device_busy_seconds[d] = b / opts.iterations;
  for (int d = 0; d < t.device_count(); ++d) r.per_device_busy_seconds.emplace(d, 0.0);
  for (const CommOp& op : sched.ops) r.comm_bytes_total += op.payload_bytes * opts.iterations;
  for (ModelName m : {ModelName::Actor, ModelName::Critic})
    if (plan.has(m) && p.has_model(m) && p.model(m).trainable)
      r.comm_bytes_total += zero_step_comm_bytes(p.model(m), plan.cfg(m), c.mem) * plan.cfg(m).dp_degree *
                            p.ppo_epochs * opts.iterations;
  r.busiest_stage = std::max_element(r.per_stage_seconds.begin(), r.per_stage_seconds.end(),
                                     [](const auto& a, const auto& b) { return a.second < b.second; })
                        ->first;
  std::set<int> bdev;
  for (const SimEvent& e : r.events)
    if (!e.comm_lane && e.stage == r.busiest_stage && e.end > e.start) bdev.insert(e.devices.begin(), e.devices.end());
  double idle = 0;
  for (int d : bdev) idle += r.device_idle_fraction(d);
  r.bubble_fraction = bdev.empty() ? 0.0 : idle / bdev.size();
  return r;
}

std::string emit_trace(const SimReport& r, const ClusterTopology& t) {
  if (r.events.empty()) throw ConfigError("emit_trace: report has no events");
  std::ostringstream o;
  o << "{\"displayTimeUnit\":\"ms\",\"traceEvents\":[";
  bool first = true;
  auto sep = [&] {
    if (!first) o << ",";
    first = false;
  };
  for (int d = 0; d < t.device_count(); ++d) {
    sep();
    o << "{\"ph\":\"M\",\"name\":\"process_name\",\"pid\":" << d << ",\"args\":{\"name\":\"device " << d << " ("
      << t.device(d).kind << ")\"}}";
    for (int lane = 0; lane < 2; ++lane) {
      sep();
      o << "{\"ph\":\"M\",\"name\":\"thread_name\",\"pid\":" << d << ",\"tid\":" << lane << ",\"args\":{\"name\":\""
        << (lane ? "comm" : "compute") << "\"}}";
    }
  }
  for (const SimEvent& e : r.events) {
    if (e.end <= e.start) continue;
    for (int d : e.devices) {
      sep();
      char b[96];
      std::snprintf(b, sizeof b, "\"ts\":%.3f,\"dur\":%.3f", e.start * 1e6, (e.end - e.start) * 1e6);
      o << "{\"ph\":\"X\",\"pid\":" << d << ",\"tid\":" << (e.comm_lane ? 1 : 0) << ",\"name\":\"" << stage_name(e.stage)
        << ":" << to_string(e.model) << ":mb" << e.micro_batch << "\",\"cat\":\"" << to_string(e.kind) << "\"," << b
        << ",\"args\":{\"task\":" << e.task_id << "}}";
    }
  }
  o << "]}";
  return o.str();
}

int max_batch_search(const PlacementPlan& plan, const PipelineSpec& p0, const CostModel& c, const ClusterTopology& t,
                     int cap) {
  const int mb = std::max(1, p0.micro_batches);
  auto feasible = [&](int k) {
    PipelineSpec p = p0;
    p.batch_size = k * mb;
    return validate_plan(plan, p, c, t).feasible;
  };
  int lo = 0, hi = cap / mb;  // invariant: lo feasible (0 = none), hi + 1 infeasible or beyond cap
  if (hi < 1 || !feasible(1)) return 0;
  lo = 1;
  while (lo < hi) {
    const int m = lo + (hi - lo + 1) / 2;
    if (feasible(m)) lo = m;
    else hi = m - 1;
  }
  return lo * mb;
}

// ---- report -------------------------------------------------------------------------

std::string report_json(const SimReport& r, const CostModel& c, const PlacementPlan& plan, const PipelineSpec& p) {
  std::ostringstream o;
  auto stage_map = [&](const std::map<Stage, double>& m) {
    std::ostringstream s;
    s << "{";
    bool f = true;
    for (const auto& [k, v] : m) {
      s << (f ? "" : ",") << "\"" << to_string(k) << "\":" << fmt(v);
      f = false;
    }
    s << "}";
    return s.str();
  };
  auto dev_map = [&](const std::map<int, double>& m) {
    std::ostringstream s;
    s << "{";
    bool f = true;
    for (const auto& [k, v] : m) {
      s << (f ? "" : ",") << "\"" << k << "\":" << fmt(v);
      f = false;
    }
    s << "}";
    return s.str();
  };
  o << "{\"plan\":\"" << plan.encoding() << "\",\"pipeline\":{\"batch\":" << p.batch_size << ",\"prompt_len\":"
    << p.prompt_len << ",\"gen_len\":" << p.gen_len << ",\"micro_batches\":" << p.micro_batches
    << ",\"ppo_epochs\":" << p.ppo_epochs << ",\"rollout_nums\":" << p.rollout_nums << ",\"models\":{";
  for (size_t i = 0; i < p.models.size(); ++i)
    o << (i ? "," : "") << "\"" << to_string(p.models[i].name) << "\":" << fmt(p.models[i].param_count);
  o << "}},\"step_seconds\":" << fmt(r.step_seconds) << ",\"throughput_samples_per_sec\":"
    << fmt(r.throughput_samples_per_sec) << ",\"per_stage_seconds\":" << stage_map(r.per_stage_seconds)
    << ",\"per_stage_fraction\":" << stage_map(r.per_stage_fraction)
    << ",\"per_device_mem_peak\":" << dev_map(r.per_device_mem_peak)
    << ",\"per_device_busy_seconds\":" << dev_map(r.per_device_busy_seconds)
    << ",\"comm_bytes_total\":" << fmt(r.comm_bytes_total) << ",\"bubble_fraction\":" << fmt(r.bubble_fraction)
    << ",\"busiest_stage\":\"" << to_string(r.busiest_stage) << "\",\"feasible\":" << (r.feasible ? "true" : "false")
    << ",\"events\":" << r.events.size() << ",\"constants\":{\"alpha\":" << fmt(c.comm.alpha)
    << ",\"mfu_gen\":" << fmt(c.comm.mfu_gen) << ",\"mfu_fwd\":" << fmt(c.comm.mfu_fwd)
    << ",\"mfu_train\":" << fmt(c.comm.mfu_train) << ",\"mfu_gen_infer\":" << fmt(c.comm.mfu_gen_infer)
    << ",\"token_record_bytes\":" << fmt(c.comm.token_record_bytes)
    << ",\"output_record_bytes\":" << fmt(c.comm.output_record_bytes)
    << ",\"bytes_train_per_param\":" << fmt(c.mem.bytes_train_per_param)
    << ",\"bytes_infer_per_param\":" << fmt(c.mem.bytes_infer_per_param)
    << ",\"lora_fraction\":" << fmt(c.mem.lora_fraction) << ",\"activation_coeff\":" << fmt(c.mem.activation_coeff)
    << ",\"activation_infer_factor\":" << fmt(c.mem.activation_infer_factor)
    << ",\"grad_ckpt_factor\":" << fmt(c.mem.grad_ckpt_factor) << ",\"oom_threshold\":" << fmt(c.mem.oom_threshold)
    << "}}";
  return o.str();
}

std::string compare_csv(const std::vector<StrategyResult>& rows) {
  std::ostringstream o;
  o << "strategy,feasible,max_batch,throughput_samples_per_sec,step_seconds,generation,forward,training,sync,"
       "comm_bytes_total\n";
  for (const auto& r : rows) {
    auto fr = [&](Stage s) {
      auto it = r.per_stage_fraction.find(s);
      return fmt(it == r.per_stage_fraction.end() ? 0.0 : it->second, 6);
    };
    o << r.name << "," << (r.feasible ? 1 : 0) << "," << r.max_batch << "," << fmt(r.throughput, 6) << ","
      << fmt(r.step_seconds, 6) << "," << fr(Stage::Generation) << "," << fr(Stage::Forward) << ","
      << fr(Stage::Training) << "," << fr(Stage::Sync) << "," << fmt(r.comm_bytes_total, 6) << "\n";
  }
  return o.str();
}

std::string compare_table(const std::vector<StrategyResult>& rows) {
  std::ostringstream o;
  char b[256];
  std::snprintf(b, sizeof b, "%-16s %8s %9s %14s %12s %6s %6s %6s %6s\n", "strategy", "feasible", "max_batch",
                "samples/s", "step_s", "gen%", "fwd%", "train%", "sync%");
  o << b;
  for (const auto& r : rows) {
    auto fr = [&](Stage s) {
      auto it = r.per_stage_fraction.find(s);
      return 100.0 * (it == r.per_stage_fraction.end() ? 0.0 : it->second);
    };
    if (!r.feasible) {
      std::snprintf(b, sizeof b, "%-16s %8s %9d %14s %12s\n", r.name.c_str(), "OOM", r.max_batch, "-", "-");
    } else {
      std::snprintf(b, sizeof b, "%-16s %8s %9d %14.4f %12.6f %6.1f %6.1f %6.1f %6.1f\n", r.name.c_str(), "yes",
                    r.max_batch, r.throughput, r.step_seconds, fr(Stage::Generation), fr(Stage::Forward),
                    fr(Stage::Training), fr(Stage::Sync));
    }
    o << b;
  }
  return o.str();
}

// ---- scenario: a strict JSON reader ------------------------------------------------

namespace {

struct JVal {
  enum Type { Null, Bool, Num, Str, Arr, Obj } type = Null;
  bool b = false;
  double n = 0;
  std::string s;
  std::vector<JVal> a;
  std::vector<std::pair<std::string, JVal>> o;
};

class JParser {
 public:
  explicit JParser(const std::string& t) : t_(t) {}
  JVal parse() {
    JVal v = value();
    ws();
    if (i_ != t_.size()) fail("trailing characters");
    return v;
  }

 private:
  const std::string& t_;
  size_t i_ = 0;
  [[noreturn]] void fail(const std::string& what) {
    int line = 1, col = 1;
    for (size_t k = 0; k < i_ && k < t_.size(); ++k) {
      if (t_[k] == '\n') line++, col = 1;
      else col++;
    }
    throw ConfigError("scenario JSON: " + what + " at line " + std::to_string(line) + ", column " + std::to_string(col));
  }
  void ws() {
    while (i_ < t_.size() && std::isspace(static_cast<unsigned char>(t_[i_]))) ++i_;
  }
  bool lit(const char* w) {
    const size_t n = std::strlen(w);
    if (t_.compare(i_, n, w) == 0) {
      i_ += n;
      return true;
    }
    return false;
  }
  JVal value() {
    ws();
    if (i_ >= t_.size()) fail("unexpected end");
    JVal v;
    const char ch = t_[i_];
    if (ch == '{') {
      v.type = JVal::Obj;
      ++i_;
      ws();
      if (i_ < t_.size() && t_[i_] == '}') return ++i_, v;
      for (;;) {
        ws();
        if (i_ >= t_.size() || t_[i_] != '"') fail("expected a key");
        std::string k = str();
        for (const auto& kv : v.o)
          if (kv.first == k) fail("duplicate key \"" + k + "\"");
        ws();
        if (i_ >= t_.size() || t_[i_] != ':') fail("expected ':'");
        ++i_;
        v.o.emplace_back(k, value());
        ws();
        if (i_ < t_.size() && t_[i_] == ',') { ++i_; continue; }
        if (i_ < t_.size() && t_[i_] == '}') { ++i_; return v; }
        fail("expected ',' or '}'");
      }
    }
    if (ch == '[') {
      v.type = JVal::Arr;
      ++i_;
      ws();
      if (i_ < t_.size() && t_[i_] == ']') return ++i_, v;
      for (;;) {
        v.a.push_back(value());
        ws();
        if (i_ < t_.size() && t_[i_] == ',') { ++i_; continue; }
        if (i_ < t_.size() && t_[i_] == ']') { ++i_; return v; }
        fail("expected ',' or ']'");
      }
    }
    if (ch == '"') {
      v.type = JVal::Str;
      v.s = str();
      return v;
    }
    if (lit("true")) { v.type = JVal::Bool; v.b = true; return v; }
    if (lit("false")) { v.type = JVal::Bool; v.b = false; return v; }
    if (lit("null")) return v;
    const char* b = t_.c_str() + i_;
    char* e = nullptr;
    v.n = std::strtod(b, &e);
    if (e == b) fail("unexpected character");
    v.type = JVal::Num;
    i_ += static_cast<size_t>(e - b);
    return v;
  }
  std::string str() {
    ++i_;  // opening quote
    std::string out;
    while (i_ < t_.size() && t_[i_] != '"') {
      if (t_[i_] == '\\') {
        ++i_;
        if (i_ >= t_.size()) break;
        const char e = t_[i_];
        out += e == 'n' ? '\n' : e == 't' ? '\t' : e;
      } else {
        out += t_[i_];
      }
      ++i_;
    }
    if (i_ >= t_.size()) fail("unterminated string");
    ++i_;
    return out;
  }
};

// Strict object access: every key must be consumed (unknown keys are errors).
class Obj {
 public:
  Obj(const JVal& v, std::string where) : v_(v), where_(std::move(where)) {
    if (v.type != JVal::Obj) throw ConfigError("scenario: " + where_ + " must be an object");
  }
  ~Obj() noexcept(false) {
    if (std::uncaught_exceptions()) return;
    for (const auto& kv : v_.o)
      if (!used_.count(kv.first)) throw ConfigError("scenario: unknown key \"" + kv.first + "\" in " + where_);
  }
  const JVal* get(const std::string& k) {
    used_.insert(k);
    for (const auto& kv : v_.o)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
  double num(const std::string& k, double def) {
    const JVal* v = get(k);
    if (!v) return def;
    if (v->type != JVal::Num) throw ConfigError("scenario: " + where_ + "." + k + " must be a number");
    return v->n;
  }
  int integer(const std::string& k, int def) {
    const double d = num(k, def);
    if (d != std::floor(d)) throw ConfigError("scenario: " + where_ + "." + k + " must be an integer");
    return static_cast<int>(d);
  }
  bool boolean(const std::string& k, bool def) {
    const JVal* v = get(k);
    if (!v) return def;
    if (v->type != JVal::Bool) throw ConfigError("scenario: " + where_ + "." + k + " must be true/false");
    return v->b;
  }
  std::string text(const std::string& k, const std::string& def) {
    const JVal* v = get(k);
    if (!v) return def;
    if (v->type != JVal::Str) throw ConfigError("scenario: " + where_ + "." + k + " must be a string");
    return v->s;
  }

 private:
  const JVal& v_;
  std::string where_;
  std::set<std::string> used_;
};

}  // namespace

namespace {

ScenarioStrategy parse_strategy(const JVal& v, const std::string& where) {
  Obj so(v, where);
  ScenarioStrategy x;
  x.cfg.name = so.text("name", "colocated");
  strategy_from_string(x.cfg.name);  // validates the name
  x.cfg.hybrid_engine = so.boolean("hybrid_engine", false);
  x.cfg.zero_level = so.integer("zero_level", 0);
  x.cfg.tp_degree = so.integer("tp_degree", 1);
  x.cfg.inference_ratio = so.num("inference_ratio", 0.5);
  x.cfg.tp_gen = so.integer("tp_gen", 8);
  x.cfg.gen_nodes = so.integer("gen_nodes", 0);
  x.batch_override = so.integer("batch", 0);
  x.use_max_batch = so.boolean("use_max_batch", x.batch_override == 0);
  if (const JVal* rv = so.get("ratios")) {
    if (rv->type != JVal::Obj) throw ConfigError("scenario: ratios must be an object");
    for (const auto& [k, val] : rv->o) {
      if (val.type != JVal::Num) throw ConfigError("scenario: ratio of " + k + " must be a number");
      x.cfg.ratios.push_back({model_name_from_string(k), val.n});
    }
  }
  return x;
}

Scenario parse_scenario(const JVal& root);

}  // namespace

Scenario parse_scenario_json(const std::string& text) { return parse_scenario(JParser(text).parse()); }

namespace {

Scenario parse_scenario(const JVal& root) {
  Scenario s;
  Obj r(root, "scenario");
  if (const JVal* tv = r.get("topology")) {
    Obj to(*tv, "topology");
    if (const JVal* box = to.get("b200_box")) {
      if (box->type != JVal::Num || box->n < 1) throw ConfigError("scenario: topology.b200_box must be a device count");
      const ClusterTopology bt = ClusterTopology::b200_box(static_cast<int>(box->n));
      NodeGroupSpec g;
      g.devices_per_node = static_cast<int>(box->n);
      g.kind = "B200";
      g.memory_bytes = bt.device(0).memory_bytes;
      g.peak_flops = bt.device(0).peak_flops;
      g.hbm_bandwidth = bt.device(0).hbm_bandwidth;
      s.topology.groups = {g};
      s.topology.intra_node_bw = s.topology.inter_node_bw = s.topology.inter_type_bw = bt.intra_node_bw();
    }
    if (const JVal* gs = to.get("groups")) {
      if (gs->type != JVal::Arr) throw ConfigError("scenario: topology.groups must be an array");
      s.topology.groups.clear();
      for (size_t i = 0; i < gs->a.size(); ++i) {
        Obj go(gs->a[i], "topology.groups[" + std::to_string(i) + "]");
        NodeGroupSpec g;
        g.nodes = go.integer("nodes", 1);
        g.devices_per_node = go.integer("devices_per_node", 8);
        g.kind = go.text("kind", "B200");
        g.memory_bytes = go.num("memory_GB", 180) * 1e9;
        g.peak_flops = go.num("peak_TFLOPs", 1670.1) * 1e12;
        g.hbm_bandwidth = go.num("hbm_GBps", 6555.8) * 1e9;
        s.topology.groups.push_back(g);
      }
    }
    s.topology.intra_node_bw = to.num("intra_node_GBps", s.topology.intra_node_bw / 1e9) * 1e9;
    s.topology.inter_node_bw = to.num("inter_node_GBps", s.topology.inter_node_bw / 1e9) * 1e9;
    s.topology.inter_type_bw = to.num("inter_type_GBps", s.topology.inter_type_bw / 1e9) * 1e9;
  }
  if (s.topology.groups.empty()) throw ConfigError("scenario: topology needs groups or b200_box");
  if (const JVal* wv = r.get("workload")) {
    Obj w(*wv, "workload");
    const std::string st = w.text("structure", "ac_nonshare");
    if (st == "ac_nonshare") s.structure = PipelineStructure::ACNonShare;
    else if (st == "ac_share") s.structure = PipelineStructure::ACShare;
    else throw ConfigError("scenario: workload.structure must be ac_share or ac_nonshare");
    if (const JVal* zv = w.get("sizes_B")) {
      Obj z(*zv, "workload.sizes_B");
      s.sizes.actor = z.num("actor", 0) * 1e9;
      s.sizes.critic = z.num("critic", 0) * 1e9;
      s.sizes.ref = z.num("ref", 0) * 1e9;
      s.sizes.reward = z.num("reward", 0) * 1e9;
      s.sizes.lora_dim = z.integer("lora_dim", 0);
    }
    s.loop.batch_size = w.integer("batch", 1);
    s.loop.prompt_len = w.integer("prompt_len", 256);
    s.loop.gen_len = w.integer("gen_len", 256);
    s.loop.micro_batches = w.integer("micro_batches", 1);
    s.loop.ppo_epochs = w.integer("ppo_epochs", 1);
    s.loop.rollout_nums = w.integer("rollout_nums", 1);
    s.loop.grad_checkpoint = w.boolean("grad_checkpoint", false);
  } else {
    throw ConfigError("scenario: missing workload");
  }
  if (const JVal* sv = r.get("strategies")) {
    if (sv->type != JVal::Arr) throw ConfigError("scenario: strategies must be an array");
    for (size_t i = 0; i < sv->a.size(); ++i)
      s.strategies.push_back(parse_strategy(sv->a[i], "strategies[" + std::to_string(i) + "]"));
  }
  if (s.strategies.empty()) s.strategies.push_back(ScenarioStrategy{});  // (plan / search ignore it)
  if (const JVal* cv = r.get("cost_model")) {
    Obj c(*cv, "cost_model");
    CommConstants& k = s.cost.comm;
    MemoryConstants& m = s.cost.mem;
    k.alpha = c.num("alpha_us", k.alpha * 1e6) * 1e-6;
    k.mfu_gen = c.num("mfu_gen", k.mfu_gen);
    k.mfu_fwd = c.num("mfu_fwd", k.mfu_fwd);
    k.mfu_train = c.num("mfu_train", k.mfu_train);
    k.mfu_gen_infer = c.num("mfu_gen_infer", k.mfu_gen_infer);
    k.token_record_bytes = c.num("token_record_bytes", k.token_record_bytes);
    k.output_record_bytes = c.num("output_record_bytes", k.output_record_bytes);
    m.bytes_train_per_param = c.num("bytes_train_per_param", m.bytes_train_per_param);
    m.bytes_infer_per_param = c.num("bytes_infer_per_param", m.bytes_infer_per_param);
    m.lora_fraction = c.num("lora_fraction", m.lora_fraction);
    m.activation_coeff = c.num("activation_coeff", m.activation_coeff);
    m.activation_infer_factor = c.num("activation_infer_factor", m.activation_infer_factor);
    m.grad_ckpt_factor = c.num("grad_ckpt_factor", m.grad_ckpt_factor);
    m.oom_threshold = c.num("oom_threshold", m.oom_threshold);
    for (double v : {k.mfu_gen, k.mfu_fwd, k.mfu_train, k.mfu_gen_infer})
      if (!(v > 0 && v <= 1)) throw ConfigError("scenario: MFU constants must be in (0, 1]");
    if (!(m.oom_threshold > 0 && m.oom_threshold <= 1)) throw ConfigError("scenario: oom_threshold must be in (0, 1]");
  }
  if (const JVal* mv = r.get("sim")) {
    Obj o(*mv, "sim");
    s.sim.overlap = o.boolean("overlap", true);
    s.sim.iterations = o.integer("iterations", 1);
    s.sim.allow_infeasible = o.boolean("allow_infeasible", false);
  }
  return s;
}

}  // namespace

std::string scenario_to_json(const Scenario& s) {
  std::ostringstream o;
  o << "{\"topology\":{\"groups\":[";
  for (size_t i = 0; i < s.topology.groups.size(); ++i) {
    const NodeGroupSpec& g = s.topology.groups[i];
    o << (i ? "," : "") << "{\"nodes\":" << g.nodes << ",\"devices_per_node\":" << g.devices_per_node
      << ",\"kind\":\"" << g.kind << "\",\"memory_GB\":" << fmt(g.memory_bytes / 1e9)
      << ",\"peak_TFLOPs\":" << fmt(g.peak_flops / 1e12) << ",\"hbm_GBps\":" << fmt(g.hbm_bandwidth / 1e9) << "}";
  }
  o << "],\"intra_node_GBps\":" << fmt(s.topology.intra_node_bw / 1e9)
    << ",\"inter_node_GBps\":" << fmt(s.topology.inter_node_bw / 1e9)
    << ",\"inter_type_GBps\":" << fmt(s.topology.inter_type_bw / 1e9) << "},\"workload\":{\"structure\":\""
    << (s.structure == PipelineStructure::ACShare ? "ac_share" : "ac_nonshare") << "\",\"sizes_B\":{\"actor\":"
    << fmt(s.sizes.actor / 1e9) << ",\"critic\":" << fmt(s.sizes.critic / 1e9) << ",\"ref\":" << fmt(s.sizes.ref / 1e9)
    << ",\"reward\":" << fmt(s.sizes.reward / 1e9) << "},\"batch\":" << s.loop.batch_size
    << ",\"prompt_len\":" << s.loop.prompt_len << ",\"gen_len\":" << s.loop.gen_len
    << ",\"micro_batches\":" << s.loop.micro_batches << ",\"ppo_epochs\":" << s.loop.ppo_epochs
    << ",\"rollout_nums\":" << s.loop.rollout_nums << "},\"strategies\":[";
  for (size_t i = 0; i < s.strategies.size(); ++i) {
    const ScenarioStrategy& x = s.strategies[i];
    o << (i ? "," : "") << "{\"name\":\"" << x.cfg.name << "\",\"zero_level\":" << x.cfg.zero_level
      << ",\"tp_degree\":" << x.cfg.tp_degree << ",\"inference_ratio\":" << fmt(x.cfg.inference_ratio)
      << ",\"tp_gen\":" << x.cfg.tp_gen << ",\"batch\":" << x.batch_override
      << ",\"use_max_batch\":" << (x.use_max_batch ? "true" : "false") << "}";
  }
  const CostModel& c = s.cost;
  o << "],\"cost_model\":{\"alpha_us\":" << fmt(c.comm.alpha * 1e6) << ",\"mfu_gen\":" << fmt(c.comm.mfu_gen)
    << ",\"mfu_fwd\":" << fmt(c.comm.mfu_fwd) << ",\"mfu_train\":" << fmt(c.comm.mfu_train)
    << ",\"mfu_gen_infer\":" << fmt(c.comm.mfu_gen_infer) << ",\"oom_threshold\":" << fmt(c.mem.oom_threshold)
    << "},\"sim\":{\"overlap\":" << (s.sim.overlap ? "true" : "false") << ",\"iterations\":" << s.sim.iterations
    << ",\"allow_infeasible\":" << (s.sim.allow_infeasible ? "true" : "false") << "}}";
  return o.str();
}

std::vector<StrategyResult> compare_strategies(const Scenario& s, const ClusterTopology& t) {
  std::vector<StrategyResult> rows;
  for (const ScenarioStrategy& x : s.strategies) {
    StrategyResult row;
    row.name = x.cfg.name;
    try {
      const BuiltStrategy bs = build_strategy(x.cfg, t, build_pipeline(s.structure, s.sizes, s.loop));
      PipelineSpec p = bs.pipeline;
      int batch = p.batch_size;
      if (x.batch_override > 0) batch = x.batch_override;
      else if (x.use_max_batch) batch = max_batch_search(bs.plan, p, s.cost, t);
      row.max_batch = batch;
      if (batch > 0) {
        p.batch_size = batch;
        SimOptions so = s.sim;
        const SimReport r = simulate(bs.plan, p, s.cost, t, so);
        row.feasible = r.feasible;
        row.throughput = r.throughput_samples_per_sec;
        row.step_seconds = r.step_seconds;
        row.per_stage_fraction = r.per_stage_fraction;
        row.comm_bytes_total = r.comm_bytes_total;
      }
    } catch (const InfeasibleError&) {
      row.feasible = false;
    }
    rows.push_back(row);
  }
  std::stable_sort(rows.begin(), rows.end(), [](const StrategyResult& a, const StrategyResult& b) {
    if (a.feasible != b.feasible) return a.feasible;
    return a.throughput > b.throughput;
  });
  return rows;
}

// ---- planner ------------------------------------------------------------------------

namespace {

double max_stage(const SimReport& r) {
  double m = 0;
  for (const auto& [s, v] : r.per_stage_seconds) m = std::max(m, v);
  return m;
}

double mem_peak(const SimReport& r) {
  double m = 0;
  for (const auto& [d, v] : r.per_device_mem_peak) m = std::max(m, v);
  return m;
}

struct Candidate {
  StrategyConfig sc;
  int micro_batches = 1;
};

// Simulate one candidate at its (max) batch; false when infeasible or not constructible.
bool evaluate(const Candidate& cand, const ClusterTopology& t, const PipelineSpec& base, const CostModel& c,
              bool search_batch, PlacementPlan* plan, PipelineSpec* pipe, SimReport* rep) {
  try {
    PipelineSpec p0 = base;
    p0.micro_batches = cand.micro_batches;
    if (p0.batch_size % p0.micro_batches) return false;
    const BuiltStrategy bs = build_strategy(cand.sc, t, p0);
    PipelineSpec p = bs.pipeline;
    if (search_batch) {
      const int b = max_batch_search(bs.plan, p, c, t);
      if (b < 1) return false;
      p.batch_size = b;
    }
    const SimReport r = simulate(bs.plan, p, c, t);
    if (!r.feasible) return false;
    *plan = bs.plan;
    *pipe = p;
    *rep = r;
    return true;
  } catch (const ConfigError&) {
    return false;
  } catch (const InfeasibleError&) {
    return false;
  }
}

}  // namespace

Recommendation recommend(const ClusterTopology& t, const PipelineSpec& p, const CostModel& c) {
  Recommendation rec;
  const int nodes = t.node_count();
  const int width = t.node_width(0);
  const double node_mem = c.mem.oom_threshold * t.device(0).memory_bytes * width;
  auto infer_fits_node = [&](ModelName m) {
    return p.has_model(m) && c.mem.bytes_infer_per_param * p.model(m).param_count <= node_mem;
  };
  std::vector<Candidate> cands;
  if (nodes <= 2) {
    // rule 1: few nodes -> Interleaving when Ref or Reward fits a node, else Co-located
    if (t.device_count() >= 2 && (infer_fits_node(ModelName::Ref) || infer_fits_node(ModelName::Reward))) {
      rec.rationale.push_back("R1: <= 2 nodes and Ref/Reward fits one node -> Interleaving");
      for (int v : {1, 2}) {
        Candidate x;
        x.sc.name = v == 1 ? "interleaving1" : "interleaving2";
        for (int z : {0, 1, 2, 3}) {
          x.sc.zero_level = z;
          cands.push_back(x);
        }
      }
    } else {
      rec.rationale.push_back("R1: <= 2 nodes and neither Ref nor Reward fits one node -> Co-located");
    }
    for (int z : {0, 1, 2, 3}) {
      Candidate x;
      x.sc.name = "colocated";
      x.sc.zero_level = z;
      cands.push_back(x);
    }
  } else {
    // rules 2-3: > 2 nodes -> Disaggregated, inference share 30-50 %, one ShadowActor replica per node
    rec.rationale.push_back("R2: > 2 nodes -> Disaggregated with inference_ratio in {0.3 .. 0.5}");
    rec.rationale.push_back("R3: ShadowActor tensor-parallel inside a node (tp_gen = node width), DP across nodes");
    for (double ir : {0.3, 0.35, 0.4, 0.45, 0.5})
      for (int z : {2, 3}) {
        Candidate x;
        x.sc.name = "disaggregated";
        x.sc.inference_ratio = ir;
        x.sc.tp_gen = width;
        x.sc.zero_level = z;
        cands.push_back(x);
      }
    for (int z : {1, 2, 3}) {  // fallback when the shadows do not fit
      Candidate x;
      x.sc.name = "interleaving2";
      x.sc.zero_level = z;
      cands.push_back(x);
      x.sc.name = "colocated";
      cands.push_back(x);
    }
  }
  rec.rationale.push_back("R4: micro_batches in {1, 2, 4, 8} minimising the largest stage time");
  rec.rationale.push_back("R5: batch raised by max_batch_search to the 95 % memory cap");
  bool found = false;
  double best_thr = -1, best_bal = std::numeric_limits<double>::max();
  for (const Candidate& base : cands)
    for (int mb : {1, 2, 4, 8}) {
      Candidate x = base;
      x.micro_batches = mb;
      PlacementPlan plan;
      PipelineSpec pipe;
      SimReport r;
      if (!evaluate(x, t, p, c, true, &plan, &pipe, &r)) continue;
      // highest throughput; equal throughput -> better stage balance
      const double thr = r.throughput_samples_per_sec, bal = max_stage(r);
      if (!found || thr > best_thr * (1 + 1e-9) || (std::abs(thr - best_thr) <= best_thr * 1e-9 && bal < best_bal)) {
        found = true;
        best_thr = thr;
        best_bal = bal;
        rec.plan = plan;
        rec.pipeline = pipe;
        rec.strategy = x.sc;
        rec.predicted = r;
      }
    }
  if (!found) throw InfeasibleError("recommend: no feasible placement for this pipeline on this cluster");
  rec.rationale.push_back("chosen: " + rec.plan.encoding() + " micro_batches " + std::to_string(rec.pipeline.micro_batches) +
                          " batch " + std::to_string(rec.pipeline.batch_size));
  return rec;
}

SearchResult exhaustive_search(const ClusterTopology& t, const PipelineSpec& p, const CostModel& c,
                               const SearchBounds& bounds) {
  std::vector<StrategyTag> tags = bounds.strategies;
  if (tags.empty())
    tags = {StrategyTag::Colocated, StrategyTag::Interleaving1, StrategyTag::Interleaving2, StrategyTag::Disaggregated};
  std::vector<Candidate> cands;
  const int n = t.device_count(), width = t.node_width(0);
  std::vector<int> tps;
  for (int k = 1; k <= width; ++k)
    if (width % k == 0) tps.push_back(k);
  for (StrategyTag tag : tags)
    for (int z : {0, 1, 2, 3})
      for (int mb : {1, 2, 4, 8}) {
        Candidate x;
        x.sc.name = to_string(tag);
        x.sc.zero_level = z;
        x.micro_batches = mb;
        if (tag == StrategyTag::Disaggregated) {
          for (int k = 1; k < std::max(2, t.node_count()); ++k)  // ratio grid: steps of 1/nodes (or 1/2 in a node)
            for (int tp : tps) {
              x.sc.inference_ratio = t.node_count() > 1 ? static_cast<double>(k) / t.node_count() : 0.5;
              x.sc.tp_gen = tp;
              cands.push_back(x);
            }
        } else {
          cands.push_back(x);
        }
      }
  SearchResult res;
  res.candidates_total = static_cast<int>(cands.size());
  if (res.candidates_total > bounds.max_candidates)
    throw SearchCapError("exhaustive_search: " + std::to_string(res.candidates_total) + " candidates exceed the cap of " +
                         std::to_string(bounds.max_candidates));
  (void)n;
  bool found = false;
  std::string best_enc;
  for (const Candidate& x : cands) {
    PlacementPlan plan;
    PipelineSpec pipe;
    SimReport r;
    if (!evaluate(x, t, p, c, true, &plan, &pipe, &r)) continue;
    res.candidates_feasible++;
    const double thr = r.throughput_samples_per_sec;
    const std::string enc = plan.encoding() + "|mb" + std::to_string(pipe.micro_batches);
    bool better = !found || thr > res.report.throughput_samples_per_sec * (1 + 1e-12);
    if (found && !better && std::abs(thr - res.report.throughput_samples_per_sec) <=
                                1e-12 * res.report.throughput_samples_per_sec) {
      const double m0 = mem_peak(res.report), m1 = mem_peak(r);
      better = m1 < m0 || (m1 == m0 && enc < best_enc);
    }
    if (better) {
      found = true;
      res.plan = plan;
      res.pipeline = pipe;
      res.strategy = x.sc;
      res.report = r;
      best_enc = enc;
    }
  }
  if (!found) throw InfeasibleError("exhaustive_search: no feasible candidate");
  return res;
}

// ---- the command front end (SPEC.md:505-547 subcommands) -------------------------------

namespace {

std::string stage_fracs_json(const std::map<Stage, double>& m) {
  std::ostringstream o;
  o << "{";
  bool f = true;
  for (const auto& [k, v] : m) {
    o << (f ? "" : ",") << "\"" << to_string(k) << "\":" << fmt(v);
    f = false;
  }
  o << "}";
  return o.str();
}

std::string rows_json(const std::vector<StrategyResult>& rows) {
  std::ostringstream o;
  o << "[";
  for (size_t i = 0; i < rows.size(); ++i) {
    const StrategyResult& r = rows[i];
    o << (i ? "," : "") << "{\"name\":\"" << r.name << "\",\"feasible\":" << (r.feasible ? "true" : "false")
      << ",\"max_batch\":" << r.max_batch << ",\"throughput\":" << fmt(r.throughput)
      << ",\"step_seconds\":" << fmt(r.step_seconds) << ",\"per_stage_fraction\":"
      << stage_fracs_json(r.per_stage_fraction) << ",\"comm_bytes_total\":" << fmt(r.comm_bytes_total) << "}";
  }
  o << "]";
  return o.str();
}

std::string json_escape(const std::string& s) {
  std::string o;
  for (char ch : s) {
    if (ch == '"' || ch == '\\') o += '\\';
    if (ch == '\n') {
      o += "\\n";
      continue;
    }
    o += ch;
  }
  return o;
}

// strategies[0] of a scenario built on its topology, at its pinned / searched / loop batch
struct Built {
  ClusterTopology topo;
  BuiltStrategy bs;
};

Built build_first(const Scenario& s) {
  Built b{ClusterTopology::build(s.topology), {}};
  const ScenarioStrategy& x = s.strategies.front();
  b.bs = build_strategy(x.cfg, b.topo, build_pipeline(s.structure, s.sizes, s.loop));
  if (x.batch_override > 0) b.bs.pipeline.batch_size = x.batch_override;
  else if (x.use_max_batch) {
    const int mb = max_batch_search(b.bs.plan, b.bs.pipeline, s.cost, b.topo);
    if (mb < 1) throw InfeasibleError("no feasible batch for " + x.cfg.name);
    b.bs.pipeline.batch_size = mb;
  }
  return b;
}

}  // namespace

std::string run_command(const std::string& cmd, const std::string& json) {
  if (cmd == "calibrate") {
    // {"scenario": {...}, "observations": [{"strategy": {...}, "devices": n, "batch": B,
    //   "measured_step_seconds": t, "generation_fraction": f}]}
    const JVal root = JParser(json).parse();
    Obj r(root, "calibrate input");
    const JVal* sv = r.get("scenario");
    const JVal* ov = r.get("observations");
    if (!sv || !ov || ov->type != JVal::Arr) throw ConfigError("calibrate: needs scenario and observations[]");
    const Scenario sc = parse_scenario(*sv);
    struct Ob {
      ClusterTopology topo;
      BuiltStrategy bs;
      double measured = 0, frac = -1;
      std::string name;
      int devices = 1;
    };
    std::vector<Ob> obs;
    for (size_t i = 0; i < ov->a.size(); ++i) {
      Obj o(ov->a[i], "observations[" + std::to_string(i) + "]");
      Ob x;
      const JVal* stv = o.get("strategy");
      if (!stv) throw ConfigError("calibrate: observation without strategy");
      const ScenarioStrategy ss = parse_strategy(*stv, "observations[].strategy");
      x.name = ss.cfg.name;
      // the scenario's device kind at the observation's device count (one node)
      TopologySpec ts = sc.topology;
      x.devices = o.integer("devices", ClusterTopology::build(ts).device_count());
      ts.groups.resize(1);
      ts.groups[0].nodes = 1;
      ts.groups[0].devices_per_node = x.devices;
      x.topo = ClusterTopology::build(ts);
      LoopParams lp = sc.loop;
      lp.batch_size = o.integer("batch", lp.batch_size);
      lp.micro_batches = o.integer("micro_batches", lp.micro_batches);
      lp.prompt_len = o.integer("prompt_len", lp.prompt_len);
      lp.gen_len = o.integer("gen_len", lp.gen_len);
      x.bs = build_strategy(ss.cfg, x.topo, build_pipeline(sc.structure, sc.sizes, lp));
      x.measured = o.num("measured_step_seconds", 0);
      x.frac = o.num("generation_fraction", -1);
      obs.push_back(std::move(x));
    }
    std::vector<CalibrationObservation> co;
    for (const Ob& x : obs) {
      CalibrationObservation c;
      c.topology = &x.topo;
      c.pipeline = &x.bs.pipeline;
      c.plan = &x.bs.plan;
      c.measured_step_seconds = x.measured;
      c.generation_fraction = x.frac;
      co.push_back(c);
    }
    CostModel fitted = sc.cost;
    fitted.comm = calibrate(sc.cost.comm, co);
    std::ostringstream o;
    o << "{\"constants\":{\"mfu_gen\":" << fmt(fitted.comm.mfu_gen) << ",\"mfu_gen_infer\":" << fmt(fitted.comm.mfu_gen_infer)
      << ",\"mfu_fwd\":" << fmt(fitted.comm.mfu_fwd) << ",\"mfu_train\":" << fmt(fitted.comm.mfu_train)
      << ",\"alpha\":" << fmt(fitted.comm.alpha) << "},\"observations\":[";
    for (size_t i = 0; i < obs.size(); ++i) {
      SimOptions so;
      so.allow_infeasible = true;
      const SimReport rp = simulate(obs[i].bs.plan, obs[i].bs.pipeline, fitted, obs[i].topo, so);
      o << (i ? "," : "") << "{\"strategy\":\"" << obs[i].name << "\",\"devices\":" << obs[i].devices
        << ",\"batch\":" << obs[i].bs.pipeline.batch_size << ",\"measured_step_seconds\":" << fmt(obs[i].measured)
        << ",\"predicted_step_seconds\":" << fmt(rp.step_seconds) << ",\"measured_generation_fraction\":"
        << fmt(obs[i].frac) << ",\"predicted_per_stage_fraction\":" << stage_fracs_json(rp.per_stage_fraction)
        << ",\"predicted_throughput\":" << fmt(rp.throughput_samples_per_sec) << "}";
    }
    Scenario pred = sc;
    pred.cost = fitted;
    o << "],\"predictions\":" << rows_json(compare_strategies(pred, ClusterTopology::build(sc.topology))) << "}";
    return o.str();
  }
  const Scenario s = parse_scenario_json(json);
  if (cmd == "simulate" || cmd == "trace") {
    const Built b = build_first(s);
    const SimReport r = simulate(b.bs.plan, b.bs.pipeline, s.cost, b.topo, s.sim);
    return cmd == "simulate" ? report_json(r, s.cost, b.bs.plan, b.bs.pipeline) : emit_trace(r, b.topo);
  }
  if (cmd == "compare") {
    const std::vector<StrategyResult> rows = compare_strategies(s, ClusterTopology::build(s.topology));
    return "{\"rows\":" + rows_json(rows) + ",\"csv\":\"" + json_escape(compare_csv(rows)) + "\",\"table\":\"" +
           json_escape(compare_table(rows)) + "\"}";
  }
  if (cmd == "maxbatch") {
    const ClusterTopology t = ClusterTopology::build(s.topology);
    std::ostringstream o;
    o << "[";
    for (size_t i = 0; i < s.strategies.size(); ++i) {
      const BuiltStrategy bs = build_strategy(s.strategies[i].cfg, t, build_pipeline(s.structure, s.sizes, s.loop));
      o << (i ? "," : "") << "{\"name\":\"" << s.strategies[i].cfg.name
        << "\",\"max_batch\":" << max_batch_search(bs.plan, bs.pipeline, s.cost, t) << "}";
    }
    o << "]";
    return o.str();
  }
  if (cmd == "plan" || cmd == "search") {
    const ClusterTopology t = ClusterTopology::build(s.topology);
    const PipelineSpec p = build_pipeline(s.structure, s.sizes, s.loop);
    std::ostringstream o;
    if (cmd == "plan") {
      const Recommendation rec = recommend(t, p, s.cost);
      o << "{\"strategy\":\"" << rec.strategy.name << "\",\"plan\":\"" << rec.plan.encoding()
        << "\",\"batch\":" << rec.pipeline.batch_size << ",\"micro_batches\":" << rec.pipeline.micro_batches
        << ",\"rationale\":[";
      for (size_t i = 0; i < rec.rationale.size(); ++i) o << (i ? "," : "") << "\"" << json_escape(rec.rationale[i]) << "\"";
      o << "],\"predicted\":" << report_json(rec.predicted, s.cost, rec.plan, rec.pipeline) << "}";
    } else {
      const SearchResult res = exhaustive_search(t, p, s.cost);
      o << "{\"strategy\":\"" << res.strategy.name << "\",\"plan\":\"" << res.plan.encoding()
        << "\",\"batch\":" << res.pipeline.batch_size << ",\"micro_batches\":" << res.pipeline.micro_batches
        << ",\"candidates_total\":" << res.candidates_total << ",\"candidates_feasible\":" << res.candidates_feasible
        << ",\"predicted\":" << report_json(res.report, s.cost, res.plan, res.pipeline) << "}";
    }
    return o.str();
  }
  throw ConfigError("unknown command: " + cmd + " (simulate | trace | compare | maxbatch | plan | search | calibrate)");
}

}  // namespace flexrlhf
