// execplan.hpp — the executed form of a placement plan: which rank runs which task of the
// stage DAG on which samples, and which rows move between ranks at which attach point.
//
// Inputs are the reference's own planning objects:
//   * the placement (build_strategy -> PlacementPlan, placement.hpp:34-63),
//   * the stage DAG task_graph(pipeline, shadows) (workload.cpp:109-175): per rollout x
//     micro-batch one Generation then one Forward per scorer, the experience barrier,
//     TrainFB per micro-batch x trainee x epoch, ParamSync + Barrier under shadows,
//   * the comm schedule derive_comm_schedule(plan, pipeline) (placement.hpp:101-102,
//     SPEC.md:323-331): every exchange below is tagged with the CommOp it realises.
// Pure host logic (no CUDA): the GPU executor (engine.cpp) walks `steps` in order, and
// tests/test_dp_gloo.py executes the same plan on CPU ranks over gloo.
//
// Sample ownership.  G = world * batch_per_rank samples per rollout (global ids
// r*G + [0, G)); micro-batch mb of rollout r is ids r*G + mb*Gm + [0, Gm), Gm = G / M.
// A model hosted on device group D processes micro-batch (r, mb) split evenly over D:
// member i owns ids r*G + mb*Gm + i*per + [0, per), per = Gm / |D|, at local rows
// (r*M + mb)*per + [0, per) of its "row set" (one row set per distinct device group).
// Prompts start "home": rank k holds ids r*G + k*batch_per_rank + [0, batch_per_rank).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "flexrlhf/placement.hpp"

namespace flexrlhf {

// Row fields that cross devices (8 B per token of (query, response), 4 B per
// scalar output field).
enum class Field { Prompt, Tokens, LogpOld, LogpRef, Values, Score };
const char* to_string(Field f);

// Global sample ids [first_id, first_id + count) held by `rank` at local rows [row0, ...).
struct Segment {
  int rank = 0;
  int64_t first_id = 0;
  int count = 0;
  int64_t row0 = 0;
};

// `count` rows from src_rank's src_row.. to dst_rank's dst_row.. (src == dst: local copy).
struct Transfer {
  int src_rank = 0, dst_rank = 0;
  int64_t src_row = 0, dst_row = 0;
  int count = 0;
};

// Intersections of the source and destination ownership maps, ordered by (src segment,
// dst segment) -- identical on every rank, so NCCL send/recv pairs match.
std::vector<Transfer> plan_transfers(const std::vector<Segment>& src, const std::vector<Segment>& dst);

struct RowSet {
  std::vector<int> group;  // ordered devices (the hosting models' ParallelCfg::devices)
  int per = 0;             // samples per member per micro-batch
  int rows = 0;            // rows per member: rollouts * M * per
};

struct Move {
  Field field = Field::Tokens;
  int src_set = -1;  // -1: the home prompt shards
  int dst_set = 0;
  std::vector<Transfer> transfers;
};

enum class StepKind { Exchange, Task, Experience, OptimizerStep };
const char* to_string(StepKind k);

struct ExecStep {
  StepKind kind = StepKind::Task;
  int task = -1;     // task id (Task / OptimizerStep: the TrainFB closing the epoch); Exchange: anchor task
  int comm_op = -1;  // index into `schedule.ops` this exchange realises (-1: data placement only)
  AttachKind attach = AttachKind::Before;
  int set = -1;      // Experience: the trainer row set whose GAE runs
  ModelName model = ModelName::Actor;  // OptimizerStep: the trained model
  int rollout = 0, mb = 0, epoch = 0;
  std::vector<Move> moves;
};

struct ExecPlan {
  int world = 1, batch_per_rank = 1, prompt_len = 0, gen_len = 0;
  int G = 0, M = 1, rollouts = 1, epochs = 1, Gm = 0;
  StrategyTag tag = StrategyTag::Colocated;
  PlacementPlan plan;
  PipelineSpec pipeline;
  std::vector<StageTask> tasks;
  CommSchedule schedule;
  std::vector<RowSet> sets;
  int set_of[6] = {-1, -1, -1, -1, -1, -1};  // row set of each ModelName (-1: not placed)
  ModelName generator = ModelName::Actor;
  std::vector<ExecStep> steps;

  bool hosts(int rank, ModelName m) const;
  int member_index(int set, int rank) const;  // -1 if rank is not in the set's group
  // Ownership of micro-batch (r, mb) in row set `set` (set -1: home prompt shards of rollout r).
  std::vector<Segment> segments(int set, int rollout, int mb) const;
  // Global sample id held at local row `row` of `set` by `rank`.
  int64_t sample_id(int set, int rank, int row) const;
  // The trainer row set whose rows a rank reports as its experience (Actor's, else Critic's,
  // else the generator's), or -1 when the rank holds none.
  int experience_set(int rank) const;
};

// Field produced by a scorer's Forward (Actor/ShadowActor -> LogpOld, Ref -> LogpRef,
// Critic/ShadowCritic -> Values, Reward -> Score).
Field output_field(ModelName m);

// `sc.tp_gen` > 1 (tensor-parallel shadow generation) is not executed: ConfigError.
// `sizes` (parameter counts) only feed the memory / cost formulas (validate_plan, simulate);
// zero sizes mean 1e8 placeholders.
ExecPlan build_exec_plan(const StrategyConfig& sc, int world, int batch_per_rank, int prompt_len, int gen_len,
                         int micro_batches, int rollouts, int epochs, const ModelSizes& sizes = ModelSizes{});

// The plan as JSON (sets, model -> set, steps with moves and transfers, tasks).
std::string to_json(const ExecPlan& e);

}  // namespace flexrlhf
