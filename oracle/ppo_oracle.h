/* ppo_oracle.h — CPU oracle for the RLHF PPO step (TEST INFRASTRUCTURE ONLY).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load this.  The product path (paper_2312_11819_b200) never
 * links or calls it.
 *
 * PARITY PROVENANCE.  The reference (/root/reference) contains no numeric PPO
 * path: SPEC.md:15 puts NN training/inference out of scope and SPEC.md:145
 * lists reward/KL semantics as non-goals.  The oracle therefore restates
 *   - the STRUCTURE of the reference: stage order Generation -> Forward x4 ->
 *     experience barrier -> TrainFB (workload.cpp:145-163), forward order
 *     Actor, Critic, Ref, Reward (workload.cpp:119), one PPO epoch, fixed
 *     generation length;
 *   - the NUMERICS of DeepSpeed-Chat step 3 (the paper's AC-NonShare baseline,
 *     PAPER.md:291,:293), frozen in SURVEY.md §8(c): KL-shaped rewards with a
 *     clipped score, GAE(gamma=1, lambda=0.95), clipped PPO actor loss, clipped
 *     value loss, AdamW.
 * Numeric parity is "unpinned by the reference" (it has no numbers); the oracle
 * is pinned instead against (a) torch autograd on the same model
 * (tests/golden/, tests/golden/make_golden.py) and (b) the compiled reference's
 * own task_graph / topology (oracle/_ref, oracle/ref_shim.cpp).
 */
#ifndef PPO_ORACLE_H
#define PPO_ORACLE_H

#include <stdint.h>

#include "rlhf_engine.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct oracle_ppo_outputs {
  int32_t* tokens;        /* [B,S] generated sequences (prompt + response) */
  float* greedy_margin;   /* [B,R] top1-top2 logit margin of each greedy pick */
  float* logp_old;        /* [B,R] */
  float* logp_ref;        /* [B,R] */
  float* values;          /* [B,R] */
  float* score;           /* [B]   */
  float* rewards;         /* [B,R] */
  float* advantages;      /* [B,R] */
  float* returns;         /* [B,R] */
  float* logp_new;        /* [B,R] training forward of the Actor */
  float* values_new;      /* [B,R] training forward of the Critic */
  double actor_loss, critic_loss;
  float* actor_grad;      /* flat fp32 [rlhf_param_total(actor)] */
  float* critic_grad;     /* flat fp32 [rlhf_param_total(critic)] */
  float* actor_master;    /* flat fp32 after AdamW */
  float* critic_master;
} oracle_ppo_outputs;

/* One PPO step.  tokens_in: NULL -> greedy generation from the seeded prompts;
 * else teacher-forced sequences [B,S] (generation skipped, greedy_margin and
 * the greedy predictions are still computed along tokens_in).
 * greedy_pred (optional [B,R]) receives the argmax at every generated position.
 * stop_after: 0 full step, 1 after experience (no training). */
int oracle_ppo_step(const rlhf_ppo_config* cfg, const int32_t* tokens_in, int32_t* greedy_pred,
                    int stop_after, int n_threads, oracle_ppo_outputs* out);

/* The same with ppo_epochs TrainFB passes over the experience (one AdamW step per pass,
 * each pass on the bf16 copy of the previous pass's master): logp_new / values_new /
 * losses / grads are those of the last pass, masters after it.  A batch of B samples
 * with prompt ids sample_offset + [0, B) equals rollout_nums rollouts of B / rollout_nums
 * (the engine's rollout r uses ids r * G + ...). */
int oracle_ppo_step_epochs(const rlhf_ppo_config* cfg, int ppo_epochs, const int32_t* tokens_in, int32_t* greedy_pred,
                           int stop_after, int n_threads, oracle_ppo_outputs* out);

/* Teacher-forced forward of one model over tokens [B,S]: final-LN hidden
 * states hf [B,S,d] (bf16-rounded values as fp32) — building block checks. */
int oracle_forward_hidden(const rlhf_arch* arch, uint64_t model_seed, const int32_t* tokens, int B,
                          int S, int n_threads, float* hf);

#ifdef __cplusplus
}
#endif
#endif
