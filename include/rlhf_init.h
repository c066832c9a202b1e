/* rlhf_init.h — input format shared by the CUDA engine and the CPU oracle.
 *
 * This header defines INPUTS only (never the algorithm under test):
 *   1. the flat parameter layout of one decoder model (tensor order, shapes,
 *      128-byte-aligned offsets), and
 *   2. the seeded, counter-based initialisation of weights and prompts
 *      (SplitMix64 -> Box-Muller, SURVEY.md §8(d) "Synthetic inputs").
 * Both sides generate bit-identical bf16 weights and int32 prompts from the same
 * seed, so parity compares algorithms on identical inputs.
 *
 * Plain C99 + static inline so it compiles into nvcc, g++ and gcc units alike.
 */
#ifndef RLHF_INIT_H
#define RLHF_INIT_H

#include <math.h>
#include <stdint.h>
#include <string.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- model shape --------------------------------------------------------- */

typedef struct rlhf_arch {
  int family;        /* 0 = OPT (pre-LN LayerNorm, ReLU, learned positions, tied LM head);
                        1 = LLaMA (pre-norm RMSNorm eps 1e-6, SwiGLU FFN, rotary positions theta 1e4,
                            no biases, untied LM head) */
  int vocab;
  int d_model;
  int n_layers;
  int n_heads;
  int d_ff;
  int max_pos;       /* rows of the learned position table (>= prompt+gen) */
  int scalar_head;   /* 1: value/reward head v[d] (Critic, Reward); 0: LM head = tok_emb */
} rlhf_arch;

/* Tensor ids in layout order.  Per-layer tensors repeat n_layers times. */
enum {
  RLHF_T_TOK_EMB = 0, /* [V, d]   */
  RLHF_T_POS_EMB,     /* [max_pos, d] */
  RLHF_T_LN1_G,       /* [d] per layer from here ... */
  RLHF_T_LN1_B,
  RLHF_T_WQKV,        /* [3d, d] rows: q(d) | k(d) | v(d); head h uses cols h*hd.. */
  RLHF_T_BQKV,        /* [3d] */
  RLHF_T_WO,          /* [d, d] */
  RLHF_T_BO,
  RLHF_T_LN2_G,
  RLHF_T_LN2_B,
  RLHF_T_W1,          /* [ff, d] */
  RLHF_T_B1,          /* [ff] */
  RLHF_T_W2,          /* [d, ff] */
  RLHF_T_B2,          /* [d] ... to here */
  RLHF_T_LNF_G,       /* [d] */
  RLHF_T_LNF_B,
  RLHF_T_VHEAD,       /* [d] (scalar_head only, else size 0) */
  RLHF_T_LM_HEAD,     /* [V, d] untied LM head (LLaMA, !scalar_head; else size 0) */
  RLHF_T_COUNT
};
#define RLHF_LAYER_FIRST RLHF_T_LN1_G
#define RLHF_LAYER_LAST RLHF_T_B2
#define RLHF_LAYER_TENSORS (RLHF_LAYER_LAST - RLHF_LAYER_FIRST + 1)

static inline int64_t rlhf_align64(int64_t n) { return (n + 63) & ~(int64_t)63; }

/* Element count of tensor `t` (layer-independent). */
static inline int64_t rlhf_tensor_numel(const rlhf_arch* a, int t) {
  const int64_t V = a->vocab, d = a->d_model, f = a->d_ff;
  if (a->family == 1) { /* LLaMA: W1 = [gate (ff rows) | up (ff rows)]; no biases, no LN betas, no positions */
    switch (t) {
      case RLHF_T_POS_EMB: case RLHF_T_LN1_B: case RLHF_T_LN2_B: case RLHF_T_LNF_B:
      case RLHF_T_BQKV: case RLHF_T_BO: case RLHF_T_B1: case RLHF_T_B2: return 0;
      case RLHF_T_W1: return 2 * f * d;
      case RLHF_T_LM_HEAD: return a->scalar_head ? 0 : V * d;
      default: break;
    }
  }
  switch (t) {
    case RLHF_T_LM_HEAD: return 0;
    case RLHF_T_TOK_EMB: return V * d;
    case RLHF_T_POS_EMB: return (int64_t)a->max_pos * d;
    case RLHF_T_WQKV: return 3 * d * d;
    case RLHF_T_BQKV: return 3 * d;
    case RLHF_T_WO: return d * d;
    case RLHF_T_W1: return f * d;
    case RLHF_T_B1: return f;
    case RLHF_T_W2: return d * f;
    case RLHF_T_VHEAD: return a->scalar_head ? d : 0;
    default: return d; /* LN gains/biases, bo, b2 */
  }
}

/* Offset (elements) of tensor t of layer l (l ignored for global tensors). */
static inline int64_t rlhf_tensor_offset(const rlhf_arch* a, int t, int l) {
  int64_t off = 0;
  off += rlhf_align64(rlhf_tensor_numel(a, RLHF_T_TOK_EMB));
  if (t == RLHF_T_TOK_EMB) return 0;
  if (t == RLHF_T_POS_EMB) return off;
  off += rlhf_align64(rlhf_tensor_numel(a, RLHF_T_POS_EMB));
  int64_t per_layer = 0;
  for (int k = RLHF_LAYER_FIRST; k <= RLHF_LAYER_LAST; ++k) per_layer += rlhf_align64(rlhf_tensor_numel(a, k));
  if (t >= RLHF_LAYER_FIRST && t <= RLHF_LAYER_LAST) {
    off += per_layer * l;
    for (int k = RLHF_LAYER_FIRST; k < t; ++k) off += rlhf_align64(rlhf_tensor_numel(a, k));
    return off;
  }
  off += per_layer * a->n_layers;
  for (int k = RLHF_T_LNF_G; k < t; ++k) off += rlhf_align64(rlhf_tensor_numel(a, k));
  return off;
}

/* Total flat parameter count (including alignment padding, which stays 0). */
static inline int64_t rlhf_param_total(const rlhf_arch* a) {
  return rlhf_tensor_offset(a, RLHF_T_LM_HEAD, 0) + rlhf_align64(rlhf_tensor_numel(a, RLHF_T_LM_HEAD));
}

/* Rotary table entry (LLaMA): angle = pos * theta^(-2i/hd) for pair i in [0, hd/2),
 * evaluated in double and rounded to fp32 so the engine's table and the oracle's agree
 * bit for bit.  Pair i rotates elements (i, i + hd/2) of each q / k head (HF LLaMA). */
static inline void rlhf_rope_cos_sin(int pos, int i, int hd, float* c, float* s) {
  const double ang = (double)pos * pow(10000.0, -2.0 * (double)i / (double)hd);
  *c = (float)cos(ang);
  *s = (float)sin(ang);
}

/* ---- deterministic generators -------------------------------------------- */

static inline uint64_t rlhf_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

/* Uniform in (0,1) from a (stream, counter) pair. */
static inline double rlhf_uniform(uint64_t stream, uint64_t counter) {
  uint64_t z = rlhf_splitmix64(stream ^ rlhf_splitmix64(counter + 0x632BE59BD9B4E019ull));
  return ((double)(z >> 11) + 0.5) * (1.0 / 9007199254740992.0);
}

/* Standard normal, element `i` of stream `stream` (Box-Muller on counters 2i, 2i+1). */
static inline double rlhf_normal(uint64_t stream, uint64_t i) {
  const double u1 = rlhf_uniform(stream, 2 * i), u2 = rlhf_uniform(stream, 2 * i + 1);
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

/* fp32 -> bf16 bits, round-to-nearest-even (NaN kept quiet). */
static inline uint16_t rlhf_f32_to_bf16(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40);
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}
static inline float rlhf_bf16_to_f32(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

/* Init distribution of one tensor (mean, std).  Chosen so that the LM logits
 * have std ~2 (tok_emb std 2/sqrt(d), LN output ~unit variance), which keeps
 * greedy top-2 margins well above the parity tolerance. */
static inline void rlhf_tensor_init_dist(const rlhf_arch* a, int t, double* mean, double* std) {
  *mean = 0.0;
  *std = 0.02;
  switch (t) {
    case RLHF_T_TOK_EMB: *std = 2.0 / sqrt((double)a->d_model); break;
    /* large learned positions keep the residual stream from being dominated by
     * the (tied) input embedding, so greedy decoding of a random-init model does
     * not collapse onto repeating its last token */
    case RLHF_T_POS_EMB: *std = 1.0; break;
    case RLHF_T_LN1_G: case RLHF_T_LN2_G: case RLHF_T_LNF_G: *mean = 1.0; *std = 0.05; break;
    case RLHF_T_VHEAD: *std = 1.0 / sqrt((double)a->d_model); break;
    case RLHF_T_LM_HEAD: *std = 2.0 / sqrt((double)a->d_model); break;
    /* fan-in scaled matrices (unit-variance pre-activations) */
    case RLHF_T_WQKV: case RLHF_T_WO: case RLHF_T_W1: *std = 1.0 / sqrt((double)a->d_model); break;
    case RLHF_T_W2: *std = 1.0 / sqrt((double)a->d_ff); break;
    default: break;
  }
}

/* Stream id of (model seed, tensor, layer). */
static inline uint64_t rlhf_tensor_stream(uint64_t seed, int t, int l) {
  return rlhf_splitmix64(seed * 0x100000001B3ull + (uint64_t)t * 4099u + (uint64_t)l * 131u + 17u);
}

/* Fill elements [i0, i1) of tensor (t, l) as bf16 bits into dst[0 .. i1-i0). */
static inline void rlhf_init_tensor_range(const rlhf_arch* a, uint64_t seed, int t, int l, int64_t i0,
                                          int64_t i1, uint16_t* dst) {
  double mean, std;
  rlhf_tensor_init_dist(a, t, &mean, &std);
  const uint64_t s = rlhf_tensor_stream(seed, t, l);
  for (int64_t i = i0; i < i1; ++i)
    dst[i - i0] = rlhf_f32_to_bf16((float)(mean + std * rlhf_normal(s, (uint64_t)i)));
}

/* Prompt token (b, t) of a batch, uniform iid in [0, V). */
static inline int32_t rlhf_prompt_token(uint64_t seed, int b, int t, int vocab) {
  const uint64_t z = rlhf_splitmix64(rlhf_splitmix64(seed ^ 0xA5A5A5A5ull) + (uint64_t)b * 1000003ull + (uint64_t)t);
  return (int32_t)(z % (uint64_t)vocab);
}

/* Model seeds: base*16 + role (Actor 0, Critic 1, Ref 2, Reward 3). */
static inline uint64_t rlhf_model_seed(uint64_t base, int role) { return base * 16u + (uint64_t)role; }

#ifdef __cplusplus
}
#endif
#endif /* RLHF_INIT_H */
