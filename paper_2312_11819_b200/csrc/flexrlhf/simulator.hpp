// Analytic discrete-event simulator of one RLHF iteration under a plan, its trace and
// report, the max-batch search, strategy comparison, the scenario config and the planner.
//
// Reference declarations (no definitions exist there):
//   simulator.hpp:12-64 (SimOptions, SimEvent, SimReport, simulate, emit_trace,
//   max_batch_search, StrategyResult), report.hpp:11-15, scenario.hpp:28-52,
//   planner.hpp:10-37; behaviour from /root/reference/SPEC.md:369-547.
// B200 role: the engine (engine.hpp) EXECUTES the same DAG and measures it; simulate()
// predicts it from the cost model whose constants calibrate() fits to those
// measurements, which is how placements are compared at GPU counts gpurun cannot reach.
#pragma once

#include <map>
#include <string>
#include <vector>

#include "flexrlhf/placement.hpp"

namespace flexrlhf {

struct SimOptions {
  bool overlap = true;  // comm and compute lanes run concurrently on a device
  int iterations = 1;
  bool allow_infeasible = false;
};

struct SimEvent {
  int task_id = 0;
  TaskKind kind = TaskKind::Generation;
  ModelName model = ModelName::Actor;
  int micro_batch = 0;
  Stage stage = Stage::Generation;
  bool comm_lane = false;
  double start = 0;
  double end = 0;
  std::vector<int> devices;
};

struct SimReport {
  double step_seconds = 0;
  double throughput_samples_per_sec = 0;
  std::map<Stage, double> per_stage_seconds;
  std::map<Stage, double> per_stage_fraction;
  std::map<int, double> per_device_mem_peak;
  std::map<int, double> per_device_busy_seconds;
  double comm_bytes_total = 0;
  double bubble_fraction = 0;
  Stage busiest_stage = Stage::Generation;
  bool feasible = true;
  std::vector<SimEvent> events;

  double device_idle_fraction(int device) const;
};

// List scheduling of task_graph + derive_comm_schedule in task-id order.
// InfeasibleError when validate_plan fails and !opts.allow_infeasible.
SimReport simulate(const PlacementPlan& plan, const PipelineSpec& p, const CostModel& c, const ClusterTopology& t,
                   const SimOptions& opts = {});

// Per-stage seconds with compute-lane attribution: every instant goes to the
// lowest Stage among the compute intervals active then, else among the comm intervals, else
// (idle) to the stage of the next interval to start; the result sums to `span`.
std::map<Stage, double> attribute_stages(const std::vector<SimEvent>& events, double span);

// Chrome trace-event JSON: one process per device, thread 0 compute / 1 comm, events
// "<stage>:<model>:mb<i>"; byte-stable.  ConfigError for a report without events.
std::string emit_trace(const SimReport& r, const ClusterTopology& t);

// Largest batch (a multiple of micro_batches, <= cap) with validate_plan feasible; 0 if
// none.  Feasibility is monotone in the batch (linear activation model).
int max_batch_search(const PlacementPlan& plan, const PipelineSpec& p, const CostModel& c, const ClusterTopology& t,
                     int cap = 4096);

struct StrategyResult {
  std::string name;
  bool feasible = false;
  int max_batch = 0;
  double throughput = 0;
  double step_seconds = 0;
  std::map<Stage, double> per_stage_fraction;
  double comm_bytes_total = 0;
};

// ---- report (report.hpp:11-15) ----
std::string report_json(const SimReport& r, const CostModel& c, const PlacementPlan& plan, const PipelineSpec& p);
std::string compare_csv(const std::vector<StrategyResult>& rows);
std::string compare_table(const std::vector<StrategyResult>& rows);

// ---- scenario (scenario.hpp:28-52) ----
struct ScenarioStrategy {
  StrategyConfig cfg;
  int batch_override = 0;  // > 0: pin the batch
  bool use_max_batch = true;
};

struct Scenario {
  TopologySpec topology;
  PipelineStructure structure = PipelineStructure::ACNonShare;
  ModelSizes sizes;
  LoopParams loop;
  CostModel cost;
  std::vector<ScenarioStrategy> strategies;
  SimOptions sim;
};

// Strict JSON: unknown keys are a ConfigError; human units (GB, TFLOPs, GB/s) converted here.
Scenario parse_scenario_json(const std::string& text);
std::string scenario_to_json(const Scenario& s);

// Per strategy: feasibility, (max) batch, simulated throughput, stage fractions, comm bytes;
// sorted by throughput descending, infeasible rows last.
std::vector<StrategyResult> compare_strategies(const Scenario& s, const ClusterTopology& t);

// ---- planner (planner.hpp:10-37) ----
struct Recommendation {
  PlacementPlan plan;
  PipelineSpec pipeline;  // batch raised to the searched maximum
  StrategyConfig strategy;
  std::vector<std::string> rationale;
  SimReport predicted;
};

// SPEC.md:460-466 guideline cascade.  InfeasibleError when nothing is feasible.
Recommendation recommend(const ClusterTopology& t, const PipelineSpec& p, const CostModel& c);

struct SearchBounds {
  int max_candidates = 10000;
  std::vector<StrategyTag> strategies;  // empty: all executable ones
};

struct SearchResult {
  PlacementPlan plan;
  PipelineSpec pipeline;
  StrategyConfig strategy;
  SimReport report;
  int candidates_total = 0;
  int candidates_feasible = 0;
};

// Bounded grid (strategy x inference ratio x tp_gen x micro_batches); argmax throughput,
// ties by lower memory peak then plan encoding.  SearchCapError / InfeasibleError.
SearchResult exhaustive_search(const ClusterTopology& t, const PipelineSpec& p, const CostModel& c,
                               const SearchBounds& bounds = {});

// Command front end over the functions above (the reference CLI's subcommands):
// "simulate" (report JSON), "trace" (Chrome trace), "compare" (rows + CSV + table),
// "maxbatch", "plan" (recommend), "search" (exhaustive_search) take a scenario JSON;
// "calibrate" takes {"scenario", "observations": [measured steps]} and returns the fitted
// constants, predicted-vs-measured per observation and the scenario's strategies predicted
// with them.  Errors are the usual exceptions (exit codes 2 / 3 / 4).
std::string run_command(const std::string& cmd, const std::string& json);

}  // namespace flexrlhf
