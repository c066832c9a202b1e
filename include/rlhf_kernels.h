/* rlhf_kernels.h — per-op C-ABI of the sm_100a kernels (lower boundary).
 *
 * The reference prices every stage task with
 *     double stage_compute_time(TaskKind, const ModelSpec&, const ParallelCfg&,
 *                               const PipelineSpec&, const ClusterTopology&, const CostModel&)
 *     (/root/reference/proj/include/rlhfsim/costmodel.hpp:63-64; formula SPEC.md:209:
 *      Generation = prefill + gen_len x decode, Forward = 2*P*B*(prompt+gen),
 *      TrainFB = 6*P*B*(prompt+gen))
 * The engine executes those tasks instead; each entry point below is one piece
 * of that execution, tagged with the TaskKind it serves.
 *
 * Conventions: POD params, raw device pointers, caller-owned
 * memory (workspaces included), asynchronous on the given stream, int status
 * (0 ok, 2 bad argument, 5 CUDA error).  No CPU fallback.
 * Element types: bf16 = uint16 bit pattern (__nv_bfloat16), f32 = float.
 */
#ifndef RLHF_KERNELS_H
#define RLHF_KERNELS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* rlhf_stream_t; /* == cudaStream_t */

/* ---- GEMM (Generation prefill/decode, Forward, TrainFB fwd+bwd) -----------
 * Per batch z = b*batch_h + h:  C[m,n] = epilogue( alpha * sum_k A[m,k] B[n,k] )
 *   A logical [M,K]: a_mn_major=0 -> element (m,k) at A + m*lda + k (K contiguous)
 *                    a_mn_major=1 -> element (m,k) at A + k*lda + m (M contiguous)
 *   B logical [N,K]: same with ldb / b_mn_major.   (+ h*stride_h + b*stride_b)
 *   C element (m,n) at C + b*c_stride_b + h*c_stride_h + m*c_rs + n*c_cs.
 * Epilogue: v = alpha*acc (+ bias[n] or bias[m]); relu; v *= (aux[m,n] > 0);
 *           v += residual[m,n] (f32, C's strides; may alias C); accumulate -> v += C_old;
 *           store bf16/f32.
 * causal: 0 none; 1 "QK" skip tiles strictly above the diagonal; 2 "PV"
 *         reduce k < m0+128 only; 3 "TN" reduce k >= floor(m0/64)*64 only.
 * split_k > 1: deterministic split-K (fixed-order reduction) needing
 *   workspace >= rlhf_gemm_workspace_bytes() and zeroed int counters. */
typedef struct rlhf_gemm_params {
  int M, N, K;
  int batch, batch_h;
  const void* A; int a_mn_major; int64_t lda, a_stride_h, a_stride_b;
  const void* B; int b_mn_major; int64_t ldb, b_stride_h, b_stride_b;
  void* C; int c_f32; int64_t c_rs, c_cs, c_stride_h, c_stride_b;
  float alpha;
  int accumulate;
  const void* bias; int bias_f32; int bias_along_m;
  int relu;
  const void* aux; int64_t aux_rs, aux_cs; /* bf16 mask source, same batch strides as C */
  const float* residual;                    /* f32, same strides as C */
  int causal;
  int split_k;
  int block_n;        /* 0 = auto; else 32/64/128/256 */
  void* workspace; size_t workspace_bytes;
  int* counters; int counters_len;
  unsigned long long* probe; /* optional: per-CTA phase timestamps (clock64), 8 per CTA */
  /* optional, column-major swap-AB outputs only (LM head of a decode step): instead of
   * storing C, write per (128-row tile, column n) the top-2 of the tile's rows as
   * float4 {max, bits(argmax, lowest id on ties), second, 0} at top2[(tile*N + n)*4] */
  float* top2;
  /* optional, row-major C = logits [rows, V] (LM head of a forward that needs no backward):
   * instead of storing C, write per (row, 128-column half of a 256-wide N tile) the
   * (max, sum exp(z - max)) of the row's logits to lse_part[(row*tiles_n + n_tile)*2 + half]
   * (float2) and the target logit z[row, y] to lse_tgt[row], y = lse_tokens[b*lse_S + lse_P + j]
   * for row = b*lse_R + j.  Only on the CTA-pair path (status 2 otherwise). */
  float* lse_part; float* lse_tgt; const int32_t* lse_tokens; int lse_S, lse_P, lse_R;
} rlhf_gemm_params;

int rlhf_gemm(const rlhf_gemm_params* p, rlhf_stream_t s);
/* Merge per-tile top-2 partials (rlhf_gemm_params.top2) of `tiles` tiles: greedy token
 * (ties -> lowest id) -> tok[b*tok_stride + *pos + 1], margin (top1 - top2) likewise;
 * advance_pos != 0: then *pos += 1 (the decode step's last kernel); pos then points to two
 * ints, pos[1] a zero-initialised ticket the kernel uses (and resets) to advance once. */
int rlhf_argmax_tiles(const float* top2, int tiles, int B, int32_t* tok, int64_t tok_stride, int* pos,
                      float* margin, int advance_pos, rlhf_stream_t s);

/* ---- decode GEMM (Generation): Y^T[N, M] = W[M, K] . X[N, K]^T, N <= 64 -----
 * swap-AB tcgen05; each 128-row weight tile is a thread-block cluster of `splits`
 * (1/2/4/8) CTAs over K, reduced through distributed shared memory in fixed order.
 * Y element (n, m) at Y + n*ldy + m; epilogue bias[m] (bf16), relu, + residual
 * (f32, same layout as Y, may alias Y).  pdl: launch as a programmatic dependent
 * (weights are prefetched before waiting on the previous kernel). */
typedef struct rlhf_gemm_decode_params {
  int M, N, K;
  const void* W; int64_t ldw;
  const void* X; int64_t ldx;
  void* Y; int y_f32; int64_t ldy;
  const void* bias;
  int relu;
  const float* residual;
  int splits;
  int pdl;
  unsigned long long* probe; /* optional: per-CTA phase timestamps (clock64), 16 per CTA */
  /* fused LayerNorm prologue (X may be NULL): X = bf16(LN(ln_x) * ln_g + ln_b), ln_x f32 [N, K], K <= 2048 */
  const float* ln_x; const void* ln_g; const void* ln_b;
  /* fused KV-cache store (Y = packed qkv [N, 3*kv_d] bf16): k/v -> cache[n][h][*pos][e] */
  void* kcache; void* vcache; const int* pos; int kv_d, kv_hd, kv_H, kv_Smax;
  /* LayerNorm statistics carried between decode GEMMs (no LayerNorm launch):
   * ln_stats_out (producer, fp32 output): this GEMM's CTAs write per-CTA partial
   *   (sum, sum of squares) of their output rows for every batch column n:
   *   [gridDim][N][2] (gridDim = ceil(M/128) * splits, written to the HOST int *ln_stats_parts_out);
   * ln_stats_in (consumer, with ln_x / ln_g / ln_b): X = bf16((ln_x - mean) * rstd * g + b)
   *   with mean / var combined from ln_stats_parts such partials (var = E[x^2] - mean^2). */
  float* ln_stats_out; int* ln_stats_parts_out;
  const float* ln_stats_in; int ln_stats_parts;
} rlhf_gemm_decode_params;
int rlhf_gemm_decode(const rlhf_gemm_decode_params* p, rlhf_stream_t s);
size_t rlhf_gemm_workspace_bytes(const rlhf_gemm_params* p);

/* ---- persistent greedy decode loop (Generation stage) ----------------------
 * Runs `steps` greedy decode steps of one decoder in ONE cooperative kernel
 * (one CTA per SM, grid barriers between phases, weight tiles prefetched by a
 * producer warp across phases).  Step semantics equal `steps` calls of the
 * per-kernel decode step: embed tokens[b*tok_stride + *pos] at position *pos,
 * L layers (K/V of *pos appended to the cache), final LN, tied LM head, greedy
 * argmax (ties -> lowest id) written to tokens (or pred when non-NULL, inputs
 * then keep coming from tokens: teacher forcing) at *pos + 1 with the top-2
 * margin, *pos += 1.  Requires B <= 64, d % 64 == 0, d_ff % 64 == 0,
 * head dim in {32, 64, 128}.  KV cache [L][kv_B][H][Smax][hd] bf16.
 * Replaces the decode loop of the reference's Generation stage cost term
 * (/root/reference/proj/include/rlhfsim/costmodel.hpp:63-64). */
typedef struct rlhf_decode_loop_params {
  const struct rlhf_arch* arch;
  const void* weights;  /* bf16 flat parameters, rlhf_tensor_offset layout */
  int B;
  int32_t* tokens; int64_t tok_stride;
  int32_t* pred;   /* NULL: free-running generation */
  float* margin;   /* optional, same indexing as tokens */
  int* pos;        /* device position counter */
  int steps;
  void* kcache; void* vcache; int kv_B; int Smax;
  void* workspace; size_t workspace_bytes;
  int sms;         /* CTAs (0: every SM) */
  unsigned long long* probe; /* optional: globaltimer per (phase of step 1, CTA): [P][2][G] + [G][16] */
  int probe_q;               /* phase of step 1 whose inside gets the [G][16] sub-probes */
} rlhf_decode_loop_params;
size_t rlhf_decode_loop_workspace_bytes(const rlhf_decode_loop_params* p);
int rlhf_decode_loop(const rlhf_decode_loop_params* p, rlhf_stream_t s);
int rlhf_gemm_block_n(const rlhf_gemm_params* p); /* tile width the dispatcher picks */
/* Name of the kernel rlhf_gemm(p) dispatches to ("gemm_pair_kernel" or
 * "gemm_sm100_kernel<BN>"), for labelling timings and ncu captures. */
const char* rlhf_gemm_kernel_name(const rlhf_gemm_params* p);

/* ---- embedding / norms (all stages) --------------------------------------
 * x[r] = tok_emb[tokens[b*tok_stride + p]] + pos_emb[p],  r = b*T + i,
 * p = p0 + i, with p0 = *p0_dev when p0_dev != NULL (decode steps in a graph). */
int rlhf_embed(const int32_t* tokens, int64_t tok_stride, int B, int T, int p0, const int* p0_dev,
               const void* tok_emb, const void* pos_emb, int d, float* x, rlhf_stream_t s);
/* Decode step entry: x[b] = tok_emb[tokens[b*tok_stride + *pos]] + pos_emb[*pos] (f32) and
 * y[b] = bf16(LN(x[b]) * ln_g + ln_b) (layer 0's LN1), one launch. */
int rlhf_embed_ln(const int32_t* tokens, int64_t tok_stride, int B, const int* pos_dev, const void* tok_emb,
                  const void* pos_emb, int d, float* x, const void* ln_g, const void* ln_b, void* y, rlhf_stream_t s);
/* Decode step entry fused with the previous step's greedy sampler: merges the LM-head
 * per-tile top-2 partials (as rlhf_argmax_tiles: ties -> lowest id) into dst[b*tok_stride +
 * *pos + 1] and margin, advances *pos by one (pos points to two ints, pos[1] a zero ticket),
 * then embeds position *pos + 1 as rlhf_embed_ln: the merged token when dst == tokens
 * (free-running), else tokens[b*tok_stride + *pos + 1] (teacher forcing).  One launch replaces
 * the merge + embed pair of the decode step chain (reference: the Generation term of
 * stage_compute_time, /root/reference/proj/include/rlhfsim/costmodel.hpp:63-64). */
int rlhf_argmax_embed_ln(const float* top2, int tiles, int32_t* dst, float* margin, const int32_t* tokens,
                         int64_t tok_stride, int B, int* pos, const void* tok_emb, const void* pos_emb, int d,
                         float* x, const void* ln_g, const void* ln_b, void* y, rlhf_stream_t s);
/* tok_emb grad (+ pos grad) scatter-add of dx [B*T, d] (TrainFB). */
int rlhf_embed_bwd(const int32_t* tokens, int64_t tok_stride, int B, int T, const float* dx, int d,
                   float* dtok_emb, float* dpos_emb, rlhf_stream_t s);
/* y = bf16(LN(x) * g + b), eps 1e-5; mean/rstd optional (saved for backward). */
int rlhf_layernorm(const float* x, const void* g, const void* b, void* y, float* mean, float* rstd, int M,
                   int d, rlhf_stream_t s);
/* dx += LN backward of dy; dg/db partials -> ws [nblk, 2, d] -> reduced into dg, db (+=). */
int rlhf_layernorm_bwd(const float* dy, const float* x, const float* mean, const float* rstd, const void* g,
                       float* dx, float* dg, float* db, int M, int d, float* ws, size_t ws_floats,
                       rlhf_stream_t s);
/* ---- LLaMA family (rlhf_arch.family == 1) --------------------------------
 * The reference models the 7B Actor/Critic only through its cost formulas
 * (workload.hpp:25-60 ModelSizes); these are the element ops
 * a LLaMA-shaped decoder adds to the OPT path.  pos_emb may be NULL in rlhf_embed /
 * rlhf_embed_bwd (no learned positions).
 * RMSNorm: y = bf16(x * rstd * g), rstd = 1/sqrt(mean(x^2) + 1e-6); rstd optional. */
int rlhf_rmsnorm(const float* x, const void* g, void* y, float* rstd, int M, int d, rlhf_stream_t s);
/* dx += RMSNorm backward of dy (saved rstd); dg partials -> ws [nblk, d] -> dg (+=). */
int rlhf_rmsnorm_bwd(const float* dy, const float* x, const float* rstd, const void* g, float* dx, float* dg, int M,
                     int d, float* ws, size_t ws_floats, rlhf_stream_t s);
/* Decode step entry of the LLaMA family: x[b] = tok_emb[tokens[b*stride + *pos]], y = RMSNorm(x). */
int rlhf_embed_rmsnorm(const int32_t* tokens, int64_t tok_stride, int B, const int* pos_dev, const void* tok_emb,
                       int d, float* x, const void* g, void* y, rlhf_stream_t s);
/* rlhf_argmax_embed_ln for the LLaMA family (no learned positions, RMSNorm). */
int rlhf_argmax_embed_rmsnorm(const float* top2, int tiles, int32_t* dst, float* margin, const int32_t* tokens,
                              int64_t tok_stride, int B, int* pos, const void* tok_emb, int d, float* x, const void* g,
                              void* y, rlhf_stream_t s);
/* Rotary embedding in place on the q and k parts of packed qkv rows [B*T, 3*H*hd] (bf16),
 * row b*T + i at position p0 + i (p0 = *p0_dev when given); table: float2 (cos, sin)
 * [positions][hd/2] from rlhf_rope_cos_sin.  inverse: the transpose (backward of dq, dk).
 * kcache/vcache (optional, [B][H][Smax][hd]): also store the rotated k and v at p. */
int rlhf_rope_qkv(void* qkv, int B, int T, int p0, const int* p0_dev, int H, int hd, const float* table, int inverse,
                  void* kcache, void* vcache, int Smax, rlhf_stream_t s);
/* act[r, j] = bf16(silu(gu[r, j]) * gu[r, ff + j]) over rows x ff. */
int rlhf_swiglu(const void* gu, void* act, int rows, int ff, rlhf_stream_t s);
/* dgu[r] = [dact * up * s(g) * (1 + g (1 - s(g))) | dact * silu(g)] (bf16). */
int rlhf_swiglu_bwd(const void* gu, const void* dact, void* dgu, int rows, int ff, rlhf_stream_t s);

/* out_bf16 = bf16(x) elementwise (n elements). */
int rlhf_round_bf16(const float* x, void* out, int64_t n, rlhf_stream_t s);
/* y[i] += x[i] (fp32, 16-byte aligned): ZeRO-2 accumulation of reduce-scattered gradient shards. */
int rlhf_add_f32(float* y, const float* x, int64_t n, rlhf_stream_t s);
/* db[n] += sum_m G[m, n] (bf16 G, fp32 sums, fixed order).  ws >= 64*N floats. */
int rlhf_colsum_bf16(const void* G, int M, int N, float* db, float* ws, rlhf_stream_t s);
/* Row gather/scatter between [B*S, d] and response rows [B*R, d]: row (b, j) <-> b*S + off + j. */
int rlhf_gather_rows(const void* src, void* dst, int B, int S, int R, int off, int d, int elem_bytes,
                     rlhf_stream_t s);
int rlhf_scatter_rows_f32(const float* src, float* dst, int B, int S, int R, int off, int d, rlhf_stream_t s);

/* Fused causal attention forward (S % 128 == 0, S <= 512, hd == 64): per (b, h, 128 query
 * rows) the scores alpha*QK^T live in TMEM, an online softmax produces p = bf16(softmax), and
 * (O != NULL) O[b*S + i][h*hd + e] = bf16(sum_j p_ij v_j) accumulates in TMEM from the P tiles
 * in shared memory; (P != NULL) P[z][i][j] is stored for backward (zeros above the diagonal
 * up to the end of each 128-row block).  q / k / v come from packed qkv rows [B*S, 3*H*hd].
 * Replaces QK^T GEMM + rlhf_attn_softmax (+ the P.V GEMM when O != NULL). */
int rlhf_attn_fwd_fused(const void* qkv, int B, int H, int hd, int S, float alpha, void* P, void* O, rlhf_stream_t s);
/* Attention backward, score-gradient part (S % 128 == 0, S <= 512, hd 64), one tcgen05 kernel:
 * dP = dO V^T in TMEM, D_i = sum_j P_ij dP_ij, dS = bf16(P (dP - D) * scale) with zeros above the
 * diagonal, written for key columns < (query block + 1) * 128 (what the dQ / dK GEMMs read).
 * dO [B, S, H*hd] bf16, qkv packed [B, S, 3*H*hd] (V at offset 2*H*hd), P / dS [B*H, S, S] bf16.
 * Replaces the dO V^T GEMM (fp32 dP) + rlhf_attn_softmax_bwd pair. */
int rlhf_attn_bwd_ds_fused(const void* dO, const void* qkv, const void* P, void* dS, int B, int H, int hd, int S,
                           float scale, rlhf_stream_t s);

/* ---- attention (Generation prefill, Forward, TrainFB) ---------------------
 * Row-wise causal softmax of scores [Z, S, S] (f32) -> probs bf16 (zeros above
 * the diagonal); scores already scaled. */
int rlhf_attn_softmax(const float* scores, void* probs, int Z, int S, rlhf_stream_t s);
/* dS = bf16(P * (dP - rowsum(P*dP)) * scale) for the causal lower triangle. */
int rlhf_attn_softmax_bwd(const void* probs, const float* dP, void* dS, int Z, int S, float scale,
                          rlhf_stream_t s);
/* KV cache [B, H, Smax, hd] <- k,v columns of qkv rows [B*T, 3d] at positions p0+i. */
int rlhf_kv_store(const void* qkv, int B, int T, int p0, const int* p0_dev, int H, int hd, int Smax,
                  void* kcache, void* vcache, rlhf_stream_t s);
/* Decode attention: one query per sample at position p (= *pos_dev), keys 0..p. */
int rlhf_attn_decode(const void* qkv, int B, int H, int hd, int Smax, const void* kcache, const void* vcache,
                     const int* pos_dev, void* out, rlhf_stream_t s);
/* The same, then pulls the (sample, head) rows [0, pos] of the NEXT attention's K/V cache
 * (kcache_next / vcache_next: layer l+1, or layer 0 of the next decode step) into L2 with
 * cp.async.bulk.prefetch.L2 -- those rows do not change before that attention runs, and
 * the latency-bound GEMMs in between leave HBM idle. */
int rlhf_attn_decode_prefetch(const void* qkv, int B, int H, int hd, int Smax, const void* kcache, const void* vcache,
                              const int* pos_dev, void* out, const void* kcache_next, const void* vcache_next,
                              rlhf_stream_t s);

/* ---- heads, experience, PPO (Generation, Forward, TrainFB) ---------------- */
/* logp[r] = z[r, y_r] - logsumexp(z[r, :]), y_r = tokens[b*S + P + j] for r = b*R + j; lse saved. */
/* logp[r] = lse_tgt[r] - logsumexp over the lse_part partials of row r (2*tiles_n per row). */
int rlhf_lse_merge(const float* lse_part, const float* lse_tgt, int rows, int parts, float* logp, rlhf_stream_t s);
int rlhf_logprob(const float* logits, int rows, int V, const int32_t* tokens, int S, int P, int R,
                 float* logp, float* lse, rlhf_stream_t s);
/* dz[r, v] = bf16(g[r] * (1[v == y_r] - exp(z[r,v] - lse[r]))) */
int rlhf_logprob_bwd(const float* logits, const float* lse, const float* g, int rows, int V,
                     const int32_t* tokens, int S, int P, int R, void* dz, rlhf_stream_t s);
/* Greedy pick over logits rows [B, V]: tokens[b*S + *pos_dev + 1] = argmax (ties -> lowest id);
 * margin (optional, [B,S] like tokens) = top1 - top2.  ws >= B * 64 * 4 floats. */
int rlhf_argmax_tokens(const float* logits, int B, int V, int32_t* tokens, int S, const int* pos_dev,
                       float* margin, float* ws, rlhf_stream_t s);
/* out[b*R + j] = hf[(b*S + off + j)] . w  (bf16 hf rows, bf16 w, fp32 out) */
int rlhf_scalar_head(const void* hf, const void* w, int B, int S, int R, int off, int d, float* out,
                     rlhf_stream_t s);
/* dhf rows += g * w ; dw += sum g * hf  (fp32, fixed order).  ws >= 64*d floats. */
int rlhf_scalar_head_bwd(const void* hf, const void* w, const float* g, int B, int S, int R, int off, int d,
                         float* dhf, float* dw, float* ws, rlhf_stream_t s);
/* Experience buffer: rewards = -kl*(logp-logp_ref) (+clip(score) at the last
 * token); GAE(gamma, lam) -> advantages, returns.  One warp per sample: the
 * reverse recurrence A_t = delta_t + gamma*lam*A_{t+1} as a warp scan of affine
 * maps over 32 contiguous chunks of the response (deterministic). */
int rlhf_gae(const float* logp, const float* logp_ref, const float* values, const float* score, int B, int R,
             float kl_ctl, float clip_reward, float gamma, float lam, float* rewards, float* adv, float* ret,
             rlhf_stream_t s);
/* PPO clipped policy loss: g = dL/dlogp; loss_sum[0] += sum(max(pg1, pg2))
 * (one block, fixed-order reduction: bit-reproducible). */
int rlhf_ppo_actor_loss(const float* logp, const float* logp_old, const float* adv, int n, float clip, float denom,
                        float* g, float* loss_sum, rlhf_stream_t s);
/* Clipped value loss: g = dL/dv; loss_sum[0] += sum(max(l1, l2)) (x0.5/denom on host). */
int rlhf_ppo_critic_loss(const float* v, const float* v_old, const float* ret, int n, float clip, float denom,
                         float* g, float* loss_sum, rlhf_stream_t s);
/* out[0] = sum of score[B], out[1] = sum of (logp - logp_ref)[B,R] (fixed order):
 * the report's mean_score / mean_kl. */
int rlhf_experience_stats(const float* logp, const float* logp_ref, const float* score, int B, int R, float* out,
                          rlhf_stream_t s);
/* Programmatic dependent launch for the decode-step kernels issued by this host
 * thread (embed, layernorm, kv_store, attn_decode, argmax, add_int; decode GEMM
 * takes its own flag).  Used while recording the decode CUDA graph. */
void rlhf_set_pdl(int on);
/* *p += v on the device (decode position counter inside the CUDA graph). */
int rlhf_add_int(int* p, int v, rlhf_stream_t s);
/* Fused AdamW over a flat fp32 master: m, v updated; bf16 copy written. */
int rlhf_adamw(float* master, float* m, float* v, const float* grad, void* w_bf16, int64_t n, float lr,
               float beta1, float beta2, float eps, float weight_decay, int step, rlhf_stream_t s);

#ifdef __cplusplus
}
#endif
#endif /* RLHF_KERNELS_H */
