/* rlhf_engine.h — C-ABI of the B200 RLHF PPO step engine.
 *
 * Drop-in boundary.  The reference (arXiv 2312.11819 artifact, /root/reference)
 * is a C++ simulator whose executor slot is
 *     SimReport simulate(const PlacementPlan&, const PipelineSpec&, const CostModel&,
 *                        const ClusterTopology&, const SimOptions&)
 *     (/root/reference/proj/include/rlhfsim/simulator.hpp:46-47)
 * with per-task cost  stage_compute_time(...)  (costmodel.hpp:63-64) and per-
 * collective cost  collective_time(...)  (costmodel.hpp:55-56).  This ABI
 * replaces that slot with real execution: rlhf_engine_step() runs one PPO
 * iteration of the task DAG (workload.cpp:109-175) on the local GPU and fills
 * an rlhf_step_report whose fields are SimReport's (simulator.hpp:30-44),
 * measured with CUDA events instead of the analytic clock.
 *
 * Conventions: plain C types, caller-owned host buffers, int status
 * (0 ok; 2 config, 3 infeasible, 5 device error — the reference's exit codes,
 * errors.hpp:8-22, plus 5).  No exceptions cross the ABI.  rlhf_last_error()
 * returns the message of the calling thread's last failure.
 */
#ifndef RLHF_ENGINE_H
#define RLHF_ENGINE_H

#include <stddef.h>
#include <stdint.h>

#include "rlhf_init.h"

#ifdef __cplusplus
extern "C" {
#endif

#define RLHF_OK 0
#define RLHF_ERR_CONFIG 2
#define RLHF_ERR_INFEASIBLE 3
#define RLHF_ERR_DEVICE 5

/* PPO hyper-parameters + shapes of one RLHF step (DeepSpeed-Chat step-3
 * conventions).  Ref shares the Actor's arch, Reward the
 * Critic's arch. */
typedef struct rlhf_ppo_config {
  rlhf_arch actor;        /* scalar_head forced to 0 */
  rlhf_arch critic;       /* scalar_head forced to 1 */
  int batch;              /* samples of this rank's shard */
  int prompt_len;
  int gen_len;
  uint64_t seed;          /* model seeds = rlhf_model_seed(seed, role) */
  uint64_t prompt_seed;   /* prompts: rlhf_prompt_token(prompt_seed, b + sample_offset, t, V) */
  int sample_offset;      /* global index of this rank's first sample */
  float kl_ctl;           /* 0.1 */
  float clip_reward;      /* 5.0 */
  float gamma;            /* 1.0 */
  float lam;              /* 0.95 */
  float cliprange;        /* 0.2 */
  float cliprange_value;  /* 0.2 */
  float lr_actor;         /* 1e-5 */
  float lr_critic;        /* 5e-6 */
  float beta1, beta2, adam_eps, weight_decay; /* 0.9, 0.95, 1e-8, 0 */
  float loss_denominator; /* global B*R (DP mean); 0 -> local batch*gen_len */
} rlhf_ppo_config;

/* Fill cfg with the defaults above for the given arch pair and shapes. */
void rlhf_ppo_config_default(rlhf_ppo_config* cfg, const rlhf_arch* actor, const rlhf_arch* critic,
                             int batch, int prompt_len, int gen_len);

/* Resolve a named shape ("tiny", "opt-125m", "opt-350m", "opt-1.3b") into an
 * arch with max_pos = max_pos.  Returns 0 or RLHF_ERR_CONFIG. */
int rlhf_arch_by_name(const char* name, int max_pos, int scalar_head, rlhf_arch* out);

/* ---- placement / stage DAG queries (pure host logic, no GPU) -------------- */

/* Stage DAG of one iteration, flattened: for task i, kind/model/mb/rollout/
 * epoch and deps[dep_off[i] .. dep_off[i+1]).  Mirrors task_graph()
 * (workload.cpp:109-175).  Arrays sized by the caller: call once with
 * max_tasks = 0 to get the counts in *n_tasks / *n_deps. */
int rlhf_task_graph(int structure /*0 ACShare, 1 ACNonShare*/, int batch, int micro_batches,
                    int rollout_nums, int ppo_epochs, int shadows, int max_tasks, int max_deps,
                    int* n_tasks, int* n_deps, int* kind, int* model, int* mb, int* rollout,
                    int* epoch, int* dep_off, int* deps);

/* Placement of the four (or six) models on an n-device B200 box.
 * strategy: "colocated" | "interleaving1" | "interleaving2" | "disaggregated".
 * out_mask[m] = bitmask of devices hosting ModelName m (Actor, Critic, Ref,
 * Reward, ShadowActor, ShadowCritic); out_role[d] = DeviceRole of device d.
 * Returns the plan encoding (PlacementPlan::encoding) in enc (NUL-terminated). */
int rlhf_plan(const char* strategy, int n_devices, int zero_level, double inference_ratio,
              int tp_gen, uint32_t out_mask[6], int* out_role, char* enc, int enc_len);

/* Memory model of a placement (model_state_bytes / activation_bytes / validate_plan,
 * reference costmodel.hpp:48-50, placement.hpp:104-117): per device, the model-state
 * bytes (16 B/param train split by ZeRO level, 2 B/param inference, / tp) and the total
 * with activations; feasible = every device within 95 % of its HBM (180 GB per B200). */
int rlhf_validate_plan(const char* strategy, int n_devices, int zero_level, double inference_ratio, int tp_gen,
                       double actor_params, double critic_params, int batch, int prompt_len, int gen_len,
                       double* state_bytes, double* total_bytes, int* feasible);

/* Communication schedule the plan induces (derive_comm_schedule): per op
 * kind (CollectiveKind), attach (0 Before, 1 After), anchor task, payload. */
int rlhf_comm_schedule(const char* strategy, int n_devices, int batch, int prompt_len, int gen_len,
                       int micro_batches, int max_ops, int* n_ops, int* kind, int* attach,
                       int* anchor, double* payload, uint32_t* group_mask);

/* The planner/simulator front end (the reference's simulate / emit_trace /
 * compare_strategies / max_batch_search / recommend / exhaustive_search /
 * calibrate, simulator.hpp:46-54, scenario.hpp:52, planner.hpp:18-37,
 * costmodel.hpp:89; CLI subcommands SPEC.md:547).  command: "simulate" |
 * "trace" | "compare" | "maxbatch" | "plan" | "search" take a scenario JSON;
 * "calibrate" takes {"scenario": ..., "observations": [...]} (measured engine
 * steps).  Result JSON in out (NUL-terminated, up to out_len bytes); *needed =
 * its full length + 1.  Status 2 config, 3 infeasible, 4 search cap. */
int rlhf_sim_run(const char* command, const char* json, char* out, int out_len, int* needed);

/* ---- engine --------------------------------------------------------------- */

typedef struct rlhf_engine rlhf_engine;

/* Roles this rank executes in a placement (bit i = ModelName i), and the
 * collective wiring.  world_size == 1 needs no NCCL id. */
typedef struct rlhf_engine_options {
  int device;                 /* CUDA ordinal */
  int rank, world_size;
  const char* strategy;       /* colocated | interleaving1 | interleaving2 | disaggregated */
  const uint8_t* nccl_id;     /* 128 bytes from rlhf_nccl_unique_id (rank 0), NULL at world 1 */
  int use_cuda_graph;         /* decode loop: 0 eager kernels, 1 CUDA graph of one step with programmatic
                                 dependent launches (default), 2 graph without PDL, 3 persistent
                                 cooperative decode kernel (rlhf_decode_loop) */
  int zero_stage;             /* trainable models' AdamW state over their data-parallel group
                                 (StrategyConfig::zero_level, scenario.hpp:12-26; memory model
                                 costmodel.hpp:48-50): 0 replicated (gradient all-reduce); 1 fp32
                                 master/m/v sharded 1/dp per rank (gradient reduce-scatter, AdamW on
                                 the shard, bf16 weight all-gather) -- bit-identical updates; 2 also
                                 the gradients: per-layer buckets reduce-scattered on the comm stream
                                 as the backward finishes each layer, no full fp32 gradient resident */
  int train_micro_batch;      /* samples per TrainFB chunk: forward + backward run per chunk and
                                 the gradients accumulate; only one chunk's activations are kept,
                                 which is what bounds the batch that fits.  0 = a whole TrainFB
                                 micro-batch */
  /* ---- LoopParams (workload.hpp:25-40) and StrategyConfig (scenario.hpp:12-26) fields;
   * zero-initialised options mean the reference defaults ---- */
  int micro_batches;          /* LoopParams::micro_batches: the task DAG's Generation / Forward /
                                 TrainFB micro-batches (workload.cpp:145-163); 0 -> 1 */
  int rollout_nums;           /* LoopParams::rollout_nums: Generation+Forward rounds per step, each
                                 on new prompts (ids r*G + ...); 0 -> 1 */
  int ppo_epochs;             /* LoopParams::ppo_epochs: TrainFB passes over the experience, one
                                 AdamW step each; 0 -> 1 */
  double inference_ratio;     /* DisaggregatedOptions::inference_ratio (placement.hpp:54-58); 0 -> 0.5 */
  int tp_gen;                 /* DisaggregatedOptions::tp_gen; must be <= 1 (tensor-parallel shadow
                                 generation is not executed) */
  double ratios[4];           /* strategy "ratio_vector": PlacementRatioVector fractions of
                                 {Actor, Critic, Ref, Reward} (placement.hpp:29-46); 0 = omitted */
} rlhf_engine_options;

int rlhf_nccl_unique_id(uint8_t out[128]);

int rlhf_engine_create(const rlhf_ppo_config* cfg, const rlhf_engine_options* opt, rlhf_engine** out);
void rlhf_engine_destroy(rlhf_engine* e);

/* Per-stage measured time (CUDA events), SimReport vocabulary. */
typedef struct rlhf_step_report {
  double step_seconds;
  double throughput_samples_per_sec;   /* global batch * rollouts / step_seconds */
  double stage_seconds[4];             /* Stage: generation, forward, training, sync */
  double decode_seconds;               /* generation minus prefill */
  double prefill_seconds;
  double comm_bytes_total;
  double actor_loss, critic_loss;
  double mean_score, mean_kl;
  int gpu_launches;                    /* kernels this rank launched in the step */
  /* ---- the remaining SimReport fields, measured on this rank (simulator.hpp:30-44) ---- */
  double busy_seconds;                 /* union of this rank's compute-lane intervals */
  double bubble_fraction;              /* 1 - busy_seconds / step_seconds (idle compute lanes) */
  double comm_seconds;                 /* union of this rank's comm-lane intervals */
  double mem_peak_bytes;               /* device bytes the engine holds on this rank */
  int busiest_stage;                   /* argmax stage_seconds */
  int n_events;                        /* intervals recorded (rlhf_engine_events) */
  int feasible;                        /* validate_plan of the executed placement with the real
                                          parameter counts (analytic memory model, 95 % cap) */
} rlhf_step_report;

/* One measured interval of the last step (SimEvent, simulator.hpp:18-28).
 * kind: 0 Generation, 1 Forward, 2 TrainFB, 3 Collective (exchanges, gradient
 * sync), 4 ParamSync, 6 experience buffer (rewards + GAE), 7 AdamW.
 * lane: 0 main compute stream, 1 side compute stream, 2 comm stream.
 * stage: Stage (0 generation, 1 forward, 2 training, 3 sync). */
typedef struct rlhf_event {
  int task, kind, model, micro_batch, rollout, epoch, lane, comm_op, stage;
  double start, end;      /* seconds from the step's start */
} rlhf_event;

/* max_batch_search (simulator.hpp:53-54) against the real allocator: the largest per-rank
 * batch (a multiple of opt->micro_batches, <= cap) whose single-GPU engine allocates (and,
 * with run_step, runs one PPO step); 0 when batch 1 does not fit. */
int rlhf_engine_max_batch(const rlhf_ppo_config* cfg, const rlhf_engine_options* opt, int cap, int run_step,
                          int* best);

/* Copy up to max events of the last step; returns the count (or -status). */
int rlhf_engine_events(rlhf_engine* e, rlhf_event* out, int max);

/* The executed plan (execplan.hpp) as JSON: row sets, model -> set, the task DAG,
 * the derived comm schedule and every exchange step with its row transfers.
 * Writes up to out_len bytes (NUL-terminated); *needed = full length + 1. */
int rlhf_exec_plan_json(const char* strategy, int world, int batch_per_rank, int prompt_len, int gen_len,
                        int micro_batches, int rollout_nums, int ppo_epochs, double inference_ratio,
                        const double* ratios4, char* out, int out_len, int* needed);

/* One PPO iteration: the task DAG of task_graph (workload.cpp:109-175) --
 * rollout_nums x micro_batches of Generation -> Forward per scorer, the
 * experience barrier (rewards + GAE), ppo_epochs x micro_batches of TrainFB
 * with one AdamW step per epoch, ParamSync to the shadows -- plus the exchanges
 * the placement's comm schedule induces.  prompts_host: [rollout_nums * batch,
 * prompt_len] int32 for this rank's home shard (rollout-major), or NULL to use
 * the seeded synthetic prompts.  Launches on the engine's streams; returns
 * after the step completed (rlhf_engine_stream() is the stream that brackets it). */
int rlhf_engine_step(rlhf_engine* e, const int32_t* prompts_host, rlhf_step_report* rep);

/* Copy a named engine tensor to host (parity tests).  Names: "tokens" int32
 * [B,S]; "logp_old", "logp_ref", "values", "rewards", "advantages", "returns"
 * fp32 [B,R]; "score" [B]; "actor_grad", "critic_grad", "actor_master",
 * "critic_master" fp32 flat; "actor_params", "critic_params", "ref_params",
 * "reward_params" bf16 flat.  bytes must equal the tensor size. */
int rlhf_engine_read(rlhf_engine* e, const char* name, void* host, size_t bytes);
/* Size in bytes of a named tensor (0 if unknown). */
size_t rlhf_engine_tensor_bytes(rlhf_engine* e, const char* name);

/* Teacher-forced generation check: feed `tokens_host` [B,S] through the decode
 * path and return the greedy prediction + top-2 margin at every generated
 * position ([B,R] each). */
int rlhf_engine_greedy_check(rlhf_engine* e, const int32_t* tokens_host, int32_t* pred_host,
                             float* margin_host);

/* The engine's CUDA stream (cudaStream_t) — callers time steps with events on it. */
void* rlhf_engine_stream(rlhf_engine* e);

const char* rlhf_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* RLHF_ENGINE_H */
