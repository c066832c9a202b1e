// ppo_oracle.cpp — CPU restatement of one RLHF PPO step.  TEST INFRASTRUCTURE.
//
// See ppo_oracle.h for provenance.  Structure follows the reference task DAG
// (/root/reference/proj/src/workload.cpp:145-163: Generation, then one Forward
// per scorer model, experience barrier, TrainFB for Actor and Critic).  Numerics
// follow DeepSpeed-Chat step 3 as frozen in SURVEY.md §8(c).  Rounding contract
// (identical on the GPU path):
//   * residual stream fp32; every GEMM operand bf16; GEMM accumulation fp32;
//   * LN / qkv / attention probs / attention out / relu out / final LN -> bf16;
//   * backward: the gradient feeding each GEMM is rounded to bf16, LN and
//     residual gradients stay fp32, weight gradients accumulate in fp32.
#include "ppo_oracle.h"

#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

namespace {

using Vec = std::vector<float>;

inline float bfr(float x) { return rlhf_bf16_to_f32(rlhf_f32_to_bf16(x)); }

inline float dotf(const float* a, const float* b, int n) {
  float s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int i = 0;
  for (; i + 8 <= n; i += 8)
    for (int j = 0; j < 8; ++j) s[j] += a[i + j] * b[i + j];
  float r = ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
  for (; i < n; ++i) r += a[i] * b[i];
  return r;
}

struct Net {
  rlhf_arch a;
  Vec w;  // bf16 parameter values held as fp32, flat layout of rlhf_init.h
  // tensors absent from the family's layout (size 0) are NULL
  const float* t(int id, int l = 0) const {
    return rlhf_tensor_numel(&a, id) ? w.data() + rlhf_tensor_offset(&a, id, l) : nullptr;
  }
  bool llama() const { return a.family == 1; }
  int head_id() const { return llama() ? RLHF_T_LM_HEAD : RLHF_T_TOK_EMB; }
  Vec rope;  // LLaMA: (cos, sin) [max_pos][hd/2] from rlhf_rope_cos_sin
};

Net make_net(const rlhf_arch& a, uint64_t seed) {
  Net n;
  n.a = a;
  n.w.assign(static_cast<size_t>(rlhf_param_total(&a)), 0.0f);
  struct Piece { int t, l; int64_t i0, i1; };
  std::vector<Piece> pieces;
  const int64_t chunk = 1 << 16;
  for (int t = 0; t < RLHF_T_COUNT; ++t) {
    const bool per_layer = t >= RLHF_LAYER_FIRST && t <= RLHF_LAYER_LAST;
    for (int l = 0; l < (per_layer ? a.n_layers : 1); ++l) {
      const int64_t ne = rlhf_tensor_numel(&a, t);
      for (int64_t i = 0; i < ne; i += chunk) pieces.push_back({t, l, i, std::min(ne, i + chunk)});
    }
  }
#pragma omp parallel for schedule(dynamic)
  for (size_t p = 0; p < pieces.size(); ++p) {
    const Piece& pc = pieces[p];
    std::vector<uint16_t> tmp(static_cast<size_t>(pc.i1 - pc.i0));
    rlhf_init_tensor_range(&a, seed, pc.t, pc.l, pc.i0, pc.i1, tmp.data());
    float* dst = n.w.data() + rlhf_tensor_offset(&a, pc.t, pc.l) + pc.i0;
    for (size_t i = 0; i < tmp.size(); ++i) dst[i] = rlhf_bf16_to_f32(tmp[i]);
  }
  if (n.llama()) {
    const int hd = a.d_model / a.n_heads, half = hd / 2;
    n.rope.assign(static_cast<size_t>(a.max_pos) * half * 2, 0.0f);
    for (int p = 0; p < a.max_pos; ++p)
      for (int i = 0; i < half; ++i)
        rlhf_rope_cos_sin(p, i, hd, &n.rope[(static_cast<size_t>(p) * half + i) * 2],
                          &n.rope[(static_cast<size_t>(p) * half + i) * 2 + 1]);
  }
  return n;
}

// ---- LLaMA family (rlhf_arch.family == 1): RMSNorm, rotary q/k, SwiGLU ----------------

// y = bf16(x * rstd * g), rstd = 1/sqrt(mean(x^2) + 1e-6)
void rmsnorm(const float* x, int M, int d, const float* g, float* y, float* rstd) {
#pragma omp parallel for schedule(static)
  for (int m = 0; m < M; ++m) {
    const float* xr = x + static_cast<size_t>(m) * d;
    float v = 0;
    for (int j = 0; j < d; ++j) v += xr[j] * xr[j];
    const float rs = 1.0f / std::sqrt(v / d + 1e-6f);
    for (int j = 0; j < d; ++j) y[static_cast<size_t>(m) * d + j] = bfr(xr[j] * rs * g[j]);
    if (rstd) rstd[m] = rs;
  }
}

// dx += rstd * (dy*g - xhat * mean(dy*g*xhat)); dg += dy * xhat
void rmsnorm_bwd(const float* dy, const float* x, const float* rstd, const float* g, int M, int d, float* dx, float* dg) {
  for (int m = 0; m < M; ++m) {
    const float* xr = x + static_cast<size_t>(m) * d;
    const float* dr = dy + static_cast<size_t>(m) * d;
    float c = 0;
    for (int j = 0; j < d; ++j) {
      const float xh = xr[j] * rstd[m];
      c += dr[j] * g[j] * xh;
      dg[j] += dr[j] * xh;
    }
    c /= d;
    for (int j = 0; j < d; ++j) dx[static_cast<size_t>(m) * d + j] += rstd[m] * (dr[j] * g[j] - xr[j] * rstd[m] * c);
  }
}

// Rotate q and k of every head of one packed qkv row at position p (HF LLaMA pairing:
// element i with i + hd/2); inverse = transpose.  Values are bf16-rounded.
void rope_row(const Net& n, float* row, int p, bool inverse) {
  const int d = n.a.d_model, hd = d / n.a.n_heads, half = hd / 2;
  const float sg = inverse ? -1.0f : 1.0f;
  for (int part = 0; part < 2; ++part)
    for (int h = 0; h < n.a.n_heads; ++h) {
      float* v = row + part * d + h * hd;
      for (int i = 0; i < half; ++i) {
        const float c = n.rope[(static_cast<size_t>(p) * half + i) * 2], s = sg * n.rope[(static_cast<size_t>(p) * half + i) * 2 + 1];
        const float x0 = v[i], x1 = v[i + half];
        v[i] = bfr(x0 * c - x1 * s);
        v[i + half] = bfr(x1 * c + x0 * s);
      }
    }
}

inline float sigmoid(float g) { return 1.0f / (1.0f + std::exp(-g)); }

// Y[M,N] = X[M,K] . W[N,K]^T (+ bias[N]); fp32 accumulation.
void linear(const float* X, int M, int K, const float* W, int N, const float* bias, float* Y) {
#pragma omp parallel for schedule(static)
  for (int n = 0; n < N; ++n) {
    const float* wr = W + static_cast<size_t>(n) * K;
    const float b = bias ? bias[n] : 0.0f;
    for (int m = 0; m < M; ++m) Y[static_cast<size_t>(m) * N + n] = dotf(X + static_cast<size_t>(m) * K, wr, K) + b;
  }
}

Vec transpose(const float* A, int R, int C) {
  Vec t(static_cast<size_t>(R) * C);
#pragma omp parallel for schedule(static)
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < C; ++c) t[static_cast<size_t>(c) * R + r] = A[static_cast<size_t>(r) * C + c];
  return t;
}

// dW[N,K] += dY[M,N]^T . X[M,K]
void matmul_tn_acc(const float* dY, int M, int N, const float* X, int K, float* dW) {
  Vec dYt = transpose(dY, M, N), Xt = transpose(X, M, K);
#pragma omp parallel for schedule(static)
  for (int n = 0; n < N; ++n)
    for (int k = 0; k < K; ++k)
      dW[static_cast<size_t>(n) * K + k] += dotf(dYt.data() + static_cast<size_t>(n) * M, Xt.data() + static_cast<size_t>(k) * M, M);
}

// dX[M,K] = dY[M,N] . W[N,K]
void matmul_nn(const float* dY, int M, int N, const float* W, int K, float* dX) {
  Vec Wt = transpose(W, N, K);
  linear(dY, M, N, Wt.data(), K, nullptr, dX);
}

void colsum_acc(const float* G, int M, int N, float* db) {
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) db[n] += G[static_cast<size_t>(m) * N + n];
}

void layernorm(const float* x, int M, int d, const float* g, const float* b, float* y, float* mean,
               float* rstd) {
#pragma omp parallel for schedule(static)
  for (int m = 0; m < M; ++m) {
    const float* xr = x + static_cast<size_t>(m) * d;
    float s = 0;
    for (int j = 0; j < d; ++j) s += xr[j];
    const float mu = s / d;
    float v = 0;
    for (int j = 0; j < d; ++j) v += (xr[j] - mu) * (xr[j] - mu);
    const float rs = 1.0f / std::sqrt(v / d + 1e-5f);
    for (int j = 0; j < d; ++j) y[static_cast<size_t>(m) * d + j] = bfr((xr[j] - mu) * rs * g[j] + b[j]);
    if (mean) mean[m] = mu;
    if (rstd) rstd[m] = rs;
  }
}

// dx += LN backward of dy through LN(x) with saved mean/rstd; dg, db accumulate.
void layernorm_bwd(const float* dy, const float* x, const float* mean, const float* rstd, const float* g,
                   int M, int d, float* dx, float* dg, float* db) {
  for (int m = 0; m < M; ++m) {
    const float* xr = x + static_cast<size_t>(m) * d;
    const float* dr = dy + static_cast<size_t>(m) * d;
    float a = 0, c = 0;
    for (int j = 0; j < d; ++j) {
      const float xh = (xr[j] - mean[m]) * rstd[m];
      const float dxh = dr[j] * g[j];
      a += dxh;
      c += dxh * xh;
      dg[j] += dr[j] * xh;
      db[j] += dr[j];
    }
    a /= d;
    c /= d;
    for (int j = 0; j < d; ++j) {
      const float xh = (xr[j] - mean[m]) * rstd[m];
      dx[static_cast<size_t>(m) * d + j] += rstd[m] * (dr[j] * g[j] - a - xh * c);
    }
  }
}

struct Cache {  // K/V per layer per sample: [L][B][S][d]
  int B = 0, S = 0, d = 0;
  Vec k, v;
  void init(int L, int B_, int S_, int d_) {
    B = B_; S = S_; d = d_;
    k.assign(static_cast<size_t>(L) * B * S * d, 0.0f);
    v.assign(k.size(), 0.0f);
  }
  float* K(int l, int b) { return k.data() + (static_cast<size_t>(l) * B + b) * S * d; }
  float* V(int l, int b) { return v.data() + (static_cast<size_t>(l) * B + b) * S * d; }
};

struct Saved {  // activations of a whole-sequence forward, for backward
  std::vector<Vec> x_in, mean1, rstd1, h1, qkv, P, o, x_mid, mean2, rstd2, h2, f;
  Vec x_fin, meanf, rstdf, hf;
};

// Forward of positions [i0, i1) of every sample; K/V of earlier positions come
// from `c`.  Returns final-LN hidden rows hf[B*(i1-i0), d] (bf16 values).
Vec forward_chunk(const Net& n, const int32_t* tok, int B, int S, int i0, int i1, Cache& c, Saved* sv) {
  const rlhf_arch& a = n.a;
  const int d = a.d_model, H = a.n_heads, hd = d / H, ff = a.d_ff, T = i1 - i0, M = B * T;
  const float scale = 1.0f / std::sqrt(static_cast<float>(hd));
  Vec x(static_cast<size_t>(M) * d);
  const float* E = n.t(RLHF_T_TOK_EMB);
  const float* Pm = n.t(RLHF_T_POS_EMB);
  for (int b = 0; b < B; ++b)
    for (int i = i0; i < i1; ++i) {
      const int r = b * T + (i - i0);
      const int id = tok[static_cast<size_t>(b) * S + i];
      for (int j = 0; j < d; ++j)
        x[static_cast<size_t>(r) * d + j] = E[static_cast<size_t>(id) * d + j] + (Pm ? Pm[static_cast<size_t>(i) * d + j] : 0.0f);
    }
  if (sv) {
    const size_t L = static_cast<size_t>(a.n_layers);
    for (auto* v : {&sv->x_in, &sv->mean1, &sv->rstd1, &sv->h1, &sv->qkv, &sv->P, &sv->o, &sv->x_mid,
                    &sv->mean2, &sv->rstd2, &sv->h2, &sv->f})
      v->assign(L, Vec());
  }
  Vec h(static_cast<size_t>(M) * d), qkv(static_cast<size_t>(M) * 3 * d), o(static_cast<size_t>(M) * d),
      tmp(static_cast<size_t>(M) * d), pre(static_cast<size_t>(M) * ff * (n.llama() ? 2 : 1)), mean(M), rstd(M),
      act(n.llama() ? static_cast<size_t>(M) * ff : 0);
  auto norm = [&](int g, int l, float* y) {  // LayerNorm (OPT) / RMSNorm (LLaMA)
    if (n.llama()) rmsnorm(x.data(), M, d, n.t(g, l), y, rstd.data());
    else layernorm(x.data(), M, d, n.t(g, l), n.t(g + 1, l), y, mean.data(), rstd.data());
  };
  for (int l = 0; l < a.n_layers; ++l) {
    if (sv) sv->x_in[l] = x;
    norm(RLHF_T_LN1_G, l, h.data());
    if (sv) { sv->mean1[l] = mean; sv->rstd1[l] = rstd; sv->h1[l] = h; }
    linear(h.data(), M, d, n.t(RLHF_T_WQKV, l), 3 * d, n.t(RLHF_T_BQKV, l), qkv.data());
    for (float& q : qkv) q = bfr(q);
    if (n.llama())
      for (int r = 0; r < M; ++r) rope_row(n, qkv.data() + static_cast<size_t>(r) * 3 * d, i0 + r % T, false);
    if (sv) sv->qkv[l] = qkv;
    for (int b = 0; b < B; ++b)
      for (int i = i0; i < i1; ++i) {
        const float* row = qkv.data() + static_cast<size_t>(b * T + (i - i0)) * 3 * d;
        std::memcpy(c.K(l, b) + static_cast<size_t>(i) * d, row + d, sizeof(float) * d);
        std::memcpy(c.V(l, b) + static_cast<size_t>(i) * d, row + 2 * d, sizeof(float) * d);
      }
    if (sv) sv->P[l].assign(static_cast<size_t>(B) * H * S * S, 0.0f);
#pragma omp parallel for collapse(2) schedule(static)
    for (int b = 0; b < B; ++b)
      for (int hh = 0; hh < H; ++hh) {
        const float* Kc = c.K(l, b);
        const float* Vc = c.V(l, b);
        Vec s(static_cast<size_t>(i1));
        for (int i = i0; i < i1; ++i) {
          const int r = b * T + (i - i0);
          const float* q = qkv.data() + static_cast<size_t>(r) * 3 * d + hh * hd;
          float mx = -INFINITY;
          for (int j = 0; j <= i; ++j) {
            s[j] = dotf(q, Kc + static_cast<size_t>(j) * d + hh * hd, hd) * scale;
            mx = std::max(mx, s[j]);
          }
          float sum = 0;
          for (int j = 0; j <= i; ++j) { s[j] = std::exp(s[j] - mx); sum += s[j]; }
          const float inv = 1.0f / sum;
          float acc[256];
          for (int e = 0; e < hd; ++e) acc[e] = 0;
          for (int j = 0; j <= i; ++j) {
            const float p = bfr(s[j] * inv);
            if (sv) sv->P[l][((static_cast<size_t>(b) * H + hh) * S + i) * S + j] = p;
            const float* vr = Vc + static_cast<size_t>(j) * d + hh * hd;
            for (int e = 0; e < hd; ++e) acc[e] += p * vr[e];
          }
          for (int e = 0; e < hd; ++e) o[static_cast<size_t>(r) * d + hh * hd + e] = bfr(acc[e]);
        }
      }
    if (sv) sv->o[l] = o;
    linear(o.data(), M, d, n.t(RLHF_T_WO, l), d, n.t(RLHF_T_BO, l), tmp.data());
    for (size_t k = 0; k < x.size(); ++k) x[k] += tmp[k];
    if (sv) sv->x_mid[l] = x;
    norm(RLHF_T_LN2_G, l, h.data());
    if (sv) { sv->mean2[l] = mean; sv->rstd2[l] = rstd; sv->h2[l] = h; }
    if (n.llama()) {  // pre = [gate | up] (bf16), act = bf16(silu(gate) * up)
      linear(h.data(), M, d, n.t(RLHF_T_W1, l), 2 * ff, nullptr, pre.data());
      for (float& p : pre) p = bfr(p);
      for (int m = 0; m < M; ++m)
        for (int j = 0; j < ff; ++j) {
          const float g = pre[static_cast<size_t>(m) * 2 * ff + j], u = pre[static_cast<size_t>(m) * 2 * ff + ff + j];
          act[static_cast<size_t>(m) * ff + j] = bfr(g * sigmoid(g) * u);
        }
      if (sv) sv->f[l] = pre;
      linear(act.data(), M, ff, n.t(RLHF_T_W2, l), d, nullptr, tmp.data());
    } else {
      linear(h.data(), M, d, n.t(RLHF_T_W1, l), ff, n.t(RLHF_T_B1, l), pre.data());
      for (float& p : pre) p = bfr(p > 0.0f ? p : 0.0f);
      if (sv) sv->f[l] = pre;
      linear(pre.data(), M, ff, n.t(RLHF_T_W2, l), d, n.t(RLHF_T_B2, l), tmp.data());
    }
    for (size_t k = 0; k < x.size(); ++k) x[k] += tmp[k];
  }
  Vec hf(static_cast<size_t>(M) * d);
  norm(RLHF_T_LNF_G, 0, hf.data());
  if (sv) { sv->x_fin = x; sv->meanf = mean; sv->rstdf = rstd; sv->hf = hf; }
  return hf;
}

// LM logits of one hidden row against the tied embedding.
void logits_row(const Net& n, const float* hrow, float* z) {
  const int V = n.a.vocab, d = n.a.d_model;
  const float* E = n.t(n.head_id());
  for (int v = 0; v < V; ++v) z[v] = dotf(hrow, E + static_cast<size_t>(v) * d, d);
}

float logsumexp(const float* z, int V) {
  float mx = -INFINITY;
  for (int v = 0; v < V; ++v) mx = std::max(mx, z[v]);
  float s = 0;
  for (int v = 0; v < V; ++v) s += std::exp(z[v] - mx);
  return mx + std::log(s);
}

void greedy(const float* z, int V, int32_t* tok, float* margin) {
  int best = 0;
  for (int v = 1; v < V; ++v)
    if (z[v] > z[best]) best = v;  // ties -> lowest index
  float second = -INFINITY;
  for (int v = 0; v < V; ++v)
    if (v != best) second = std::max(second, z[v]);
  *tok = best;
  if (margin) *margin = z[best] - second;
}

// Per-token log-probs logp[b, j] of tokens[t+1] at positions t = P-1+j.
void logprobs(const Net& n, const Vec& hf, const int32_t* tok, int B, int S, int P, float* logp) {
  const int R = S - P, d = n.a.d_model, V = n.a.vocab;
#pragma omp parallel
  {
    Vec z(static_cast<size_t>(V));
#pragma omp for collapse(2) schedule(static)
    for (int b = 0; b < B; ++b)
      for (int j = 0; j < R; ++j) {
        const int t = P - 1 + j;
        logits_row(n, hf.data() + (static_cast<size_t>(b) * S + t) * d, z.data());
        logp[b * R + j] = z[tok[static_cast<size_t>(b) * S + t + 1]] - logsumexp(z.data(), V);
      }
  }
}

// Backward through the decoder given dL/dhf [B*S, d] (fp32).  Accumulates into grad (flat fp32).
void backward(const Net& n, const int32_t* tok, int B, int S, const Saved& sv, const Vec& dhf, Vec& grad) {
  const rlhf_arch& a = n.a;
  const int d = a.d_model, H = a.n_heads, hd = d / H, ff = a.d_ff, M = B * S;
  const float scale = 1.0f / std::sqrt(static_cast<float>(hd));
  auto G = [&](int id, int l = 0) -> float* {
    return rlhf_tensor_numel(&a, id) ? grad.data() + rlhf_tensor_offset(&a, id, l) : nullptr;
  };
  Vec dres(static_cast<size_t>(M) * d, 0.0f);
  auto norm_bwd = [&](const float* dy, const Vec& x, const Vec& mean, const Vec& rstd, int gid, int l) {
    if (n.llama()) rmsnorm_bwd(dy, x.data(), rstd.data(), n.t(gid, l), M, d, dres.data(), G(gid, l));
    else layernorm_bwd(dy, x.data(), mean.data(), rstd.data(), n.t(gid, l), M, d, dres.data(), G(gid, l), G(gid + 1, l));
  };
  auto colsum = [&](const Vec& Gm, int N, float* db) { if (db) colsum_acc(Gm.data(), M, N, db); };
  norm_bwd(dhf.data(), sv.x_fin, sv.meanf, sv.rstdf, RLHF_T_LNF_G, 0);
  Vec g(static_cast<size_t>(M) * d), df(static_cast<size_t>(M) * ff * (n.llama() ? 2 : 1)), dh(static_cast<size_t>(M) * d),
      dqkv(static_cast<size_t>(M) * 3 * d), dov(static_cast<size_t>(M) * d);
  for (int l = a.n_layers - 1; l >= 0; --l) {
    // FFN: x_out = x_mid + relu(h2 W1^T + b1) W2^T + b2
    for (size_t k = 0; k < g.size(); ++k) g[k] = bfr(dres[k]);
    colsum(g, d, G(RLHF_T_B2, l));
    if (n.llama()) {  // SwiGLU backward from the saved [gate | up]
      const Vec& gu = sv.f[l];
      Vec act(static_cast<size_t>(M) * ff), dact(static_cast<size_t>(M) * ff);
      for (int m = 0; m < M; ++m)
        for (int j = 0; j < ff; ++j) {
          const float gg = gu[static_cast<size_t>(m) * 2 * ff + j], u = gu[static_cast<size_t>(m) * 2 * ff + ff + j];
          act[static_cast<size_t>(m) * ff + j] = bfr(gg * sigmoid(gg) * u);
        }
      matmul_tn_acc(g.data(), M, d, act.data(), ff, G(RLHF_T_W2, l));
      matmul_nn(g.data(), M, d, n.t(RLHF_T_W2, l), ff, dact.data());
      for (int m = 0; m < M; ++m)
        for (int j = 0; j < ff; ++j) {
          const float gg = gu[static_cast<size_t>(m) * 2 * ff + j], u = gu[static_cast<size_t>(m) * 2 * ff + ff + j];
          const float da = bfr(dact[static_cast<size_t>(m) * ff + j]), s = sigmoid(gg);
          df[static_cast<size_t>(m) * 2 * ff + j] = bfr(da * u * s * (1.0f + gg * (1.0f - s)));
          df[static_cast<size_t>(m) * 2 * ff + ff + j] = bfr(da * gg * s);
        }
      matmul_tn_acc(df.data(), M, 2 * ff, sv.h2[l].data(), d, G(RLHF_T_W1, l));
      matmul_nn(df.data(), M, 2 * ff, n.t(RLHF_T_W1, l), d, dh.data());
    } else {
      matmul_tn_acc(g.data(), M, d, sv.f[l].data(), ff, G(RLHF_T_W2, l));
      matmul_nn(g.data(), M, d, n.t(RLHF_T_W2, l), ff, df.data());
      for (size_t k = 0; k < df.size(); ++k) df[k] = sv.f[l][k] > 0.0f ? bfr(df[k]) : 0.0f;
      colsum(df, ff, G(RLHF_T_B1, l));
      matmul_tn_acc(df.data(), M, ff, sv.h2[l].data(), d, G(RLHF_T_W1, l));
      matmul_nn(df.data(), M, ff, n.t(RLHF_T_W1, l), d, dh.data());
    }
    norm_bwd(dh.data(), sv.x_mid[l], sv.mean2[l], sv.rstd2[l], RLHF_T_LN2_G, l);
    // Attention block: x_mid = x_in + attn(h1) Wo^T + bo
    for (size_t k = 0; k < g.size(); ++k) g[k] = bfr(dres[k]);
    colsum(g, d, G(RLHF_T_BO, l));
    matmul_tn_acc(g.data(), M, d, sv.o[l].data(), d, G(RLHF_T_WO, l));
    matmul_nn(g.data(), M, d, n.t(RLHF_T_WO, l), d, dov.data());
    for (float& v : dov) v = bfr(v);
    std::fill(dqkv.begin(), dqkv.end(), 0.0f);
    const Vec& qkv = sv.qkv[l];
    const Vec& P = sv.P[l];
#pragma omp parallel for collapse(2) schedule(static)
    for (int b = 0; b < B; ++b)
      for (int hh = 0; hh < H; ++hh) {
        const float* Pb = P.data() + (static_cast<size_t>(b) * H + hh) * S * S;
        Vec dS(static_cast<size_t>(S) * S, 0.0f);
        auto q = [&](int i) { return qkv.data() + (static_cast<size_t>(b) * S + i) * 3 * d + hh * hd; };
        auto k = [&](int i) { return q(i) + d; };
        auto v = [&](int i) { return q(i) + 2 * d; };
        auto dO = [&](int i) { return dov.data() + (static_cast<size_t>(b) * S + i) * d + hh * hd; };
        for (int i = 0; i < S; ++i) {
          float D = 0;
          Vec dP(static_cast<size_t>(i) + 1);
          for (int j = 0; j <= i; ++j) {
            dP[j] = dotf(dO(i), v(j), hd);
            D += Pb[static_cast<size_t>(i) * S + j] * dP[j];
          }
          for (int j = 0; j <= i; ++j) {
            const float p = Pb[static_cast<size_t>(i) * S + j];
            dS[static_cast<size_t>(i) * S + j] = bfr(p * (dP[j] - D) * scale);
          }
        }
        for (int i = 0; i < S; ++i) {
          float* dq = dqkv.data() + (static_cast<size_t>(b) * S + i) * 3 * d + hh * hd;
          float* dk = dq + d;
          float* dv = dq + 2 * d;
          float accq[256], acck[256], accv[256];
          for (int e = 0; e < hd; ++e) accq[e] = acck[e] = accv[e] = 0;
          for (int j = 0; j <= i; ++j) {  // dq_i = sum_j dS_ij k_j
            const float s = dS[static_cast<size_t>(i) * S + j];
            for (int e = 0; e < hd; ++e) accq[e] += s * k(j)[e];
          }
          for (int r = i; r < S; ++r) {  // dk_i = sum_r dS_ri q_r ; dv_i = sum_r P_ri dO_r
            const float s = dS[static_cast<size_t>(r) * S + i];
            const float p = Pb[static_cast<size_t>(r) * S + i];
            for (int e = 0; e < hd; ++e) { acck[e] += s * q(r)[e]; accv[e] += p * dO(r)[e]; }
          }
          for (int e = 0; e < hd; ++e) { dq[e] = bfr(accq[e]); dk[e] = bfr(acck[e]); dv[e] = bfr(accv[e]); }
        }
      }
    if (n.llama())  // dq, dk through the rotation's transpose
      for (int r = 0; r < M; ++r) rope_row(n, dqkv.data() + static_cast<size_t>(r) * 3 * d, r % S, true);
    colsum(dqkv, 3 * d, G(RLHF_T_BQKV, l));
    matmul_tn_acc(dqkv.data(), M, 3 * d, sv.h1[l].data(), d, G(RLHF_T_WQKV, l));
    matmul_nn(dqkv.data(), M, 3 * d, n.t(RLHF_T_WQKV, l), d, dh.data());
    norm_bwd(dh.data(), sv.x_in[l], sv.mean1[l], sv.rstd1[l], RLHF_T_LN1_G, l);
  }
  float* dE = G(RLHF_T_TOK_EMB);
  float* dPm = G(RLHF_T_POS_EMB);
  for (int b = 0; b < B; ++b)
    for (int i = 0; i < S; ++i) {
      const float* gr = dres.data() + (static_cast<size_t>(b) * S + i) * d;
      const int id = tok[static_cast<size_t>(b) * S + i];
      for (int j = 0; j < d; ++j) {
        dE[static_cast<size_t>(id) * d + j] += gr[j];
        if (dPm) dPm[static_cast<size_t>(i) * d + j] += gr[j];
      }
    }
}

void adamw(Vec& master, Vec& m, Vec& v, const Vec& g, float lr, const rlhf_ppo_config& c, int step) {
  const float bc1 = 1.0f - std::pow(c.beta1, static_cast<float>(step));
  const float bc2 = 1.0f - std::pow(c.beta2, static_cast<float>(step));
  for (size_t i = 0; i < master.size(); ++i) {
    m[i] = c.beta1 * m[i] + (1.0f - c.beta1) * g[i];
    v[i] = c.beta2 * v[i] + (1.0f - c.beta2) * g[i] * g[i];
    const float upd = (m[i] / bc1) / (std::sqrt(v[i] / bc2) + c.adam_eps);
    master[i] = master[i] - lr * (upd + c.weight_decay * master[i]);
  }
}

}  // namespace

extern "C" int oracle_forward_hidden(const rlhf_arch* arch, uint64_t model_seed, const int32_t* tokens, int B,
                                     int S, int n_threads, float* hf) {
  if (n_threads > 0) omp_set_num_threads(n_threads);
  Net n = make_net(*arch, model_seed);
  Cache c;
  c.init(arch->n_layers, B, S, arch->d_model);
  Vec h = forward_chunk(n, tokens, B, S, 0, S, c, nullptr);
  std::memcpy(hf, h.data(), h.size() * sizeof(float));
  return 0;
}

extern "C" int oracle_ppo_step_epochs(const rlhf_ppo_config* cfg_in, int ppo_epochs, const int32_t* tokens_in,
                                      int32_t* greedy_pred, int stop_after, int n_threads, oracle_ppo_outputs* out) {
  if (n_threads > 0) omp_set_num_threads(n_threads);
  rlhf_ppo_config cfg = *cfg_in;
  cfg.actor.scalar_head = 0;
  cfg.critic.scalar_head = 1;
  const int B = cfg.batch, P = cfg.prompt_len, R = cfg.gen_len, S = P + R;
  if (B < 1 || P < 1 || R < 1 || S > cfg.actor.max_pos || S > cfg.critic.max_pos) return RLHF_ERR_CONFIG;

  // Models: Actor, Critic, Ref (Actor arch), Reward (Critic arch), seeds by role.
  Net actor = make_net(cfg.actor, rlhf_model_seed(cfg.seed, 0));
  Net critic = make_net(cfg.critic, rlhf_model_seed(cfg.seed, 1));
  Net ref = make_net(cfg.actor, rlhf_model_seed(cfg.seed, 2));
  Net reward = make_net(cfg.critic, rlhf_model_seed(cfg.seed, 3));

  // ---- Generation (greedy, KV cache): Actor.generate(Query) ----------------
  std::vector<int32_t> tok(static_cast<size_t>(B) * S);
  for (int b = 0; b < B; ++b)
    for (int t = 0; t < S; ++t)
      tok[static_cast<size_t>(b) * S + t] =
          tokens_in ? tokens_in[static_cast<size_t>(b) * S + t]
                    : (t < P ? rlhf_prompt_token(cfg.prompt_seed, b + cfg.sample_offset, t, cfg.actor.vocab) : 0);
  {
    Cache c;
    c.init(cfg.actor.n_layers, B, S, cfg.actor.d_model);
    Vec z(static_cast<size_t>(cfg.actor.vocab));
    int i0 = 0, i1 = P;
    for (int step = 0; step < R; ++step) {
      Vec hf = forward_chunk(actor, tok.data(), B, S, i0, i1, c, nullptr);
      const int T = i1 - i0;
      for (int b = 0; b < B; ++b) {
        logits_row(actor, hf.data() + (static_cast<size_t>(b) * T + (T - 1)) * cfg.actor.d_model, z.data());
        int32_t pick;
        float margin;
        greedy(z.data(), cfg.actor.vocab, &pick, &margin);
        if (greedy_pred) greedy_pred[b * R + step] = pick;
        if (out->greedy_margin) out->greedy_margin[b * R + step] = margin;
        if (!tokens_in) tok[static_cast<size_t>(b) * S + P + step] = pick;
      }
      i0 = i1;
      i1 = i1 + 1;
    }
  }
  if (out->tokens) std::memcpy(out->tokens, tok.data(), tok.size() * sizeof(int32_t));

  // ---- Forward stage: Actor, Critic, Ref, Reward (teacher-forced) ---------
  Vec logp_old(static_cast<size_t>(B) * R), logp_ref(logp_old.size()), values(logp_old.size()), score(B);
  auto fwd = [&](const Net& n) {
    Cache c;
    c.init(n.a.n_layers, B, S, n.a.d_model);
    return forward_chunk(n, tok.data(), B, S, 0, S, c, nullptr);
  };
  logprobs(actor, fwd(actor), tok.data(), B, S, P, logp_old.data());
  {
    Vec hf = fwd(critic);
    const float* vh = critic.t(RLHF_T_VHEAD);
    for (int b = 0; b < B; ++b)
      for (int j = 0; j < R; ++j)
        values[b * R + j] = dotf(hf.data() + (static_cast<size_t>(b) * S + P - 1 + j) * cfg.critic.d_model, vh, cfg.critic.d_model);
  }
  logprobs(ref, fwd(ref), tok.data(), B, S, P, logp_ref.data());
  {
    Vec hf = fwd(reward);
    const float* vh = reward.t(RLHF_T_VHEAD);
    for (int b = 0; b < B; ++b)
      score[b] = dotf(hf.data() + (static_cast<size_t>(b) * S + S - 1) * cfg.critic.d_model, vh, cfg.critic.d_model);
  }

  // ---- Experience buffer: KL-shaped rewards + GAE (DS-Chat step 3) --------
  Vec rewards(logp_old.size()), adv(logp_old.size()), ret(logp_old.size());
  for (int b = 0; b < B; ++b) {
    for (int j = 0; j < R; ++j) rewards[b * R + j] = -cfg.kl_ctl * (logp_old[b * R + j] - logp_ref[b * R + j]);
    const float clipped = std::min(std::max(score[b], -cfg.clip_reward), cfg.clip_reward);
    rewards[b * R + R - 1] += clipped;
    float last = 0.0f;
    for (int j = R - 1; j >= 0; --j) {
      const float nextv = j < R - 1 ? values[b * R + j + 1] : 0.0f;
      const float delta = rewards[b * R + j] + cfg.gamma * nextv - values[b * R + j];
      last = delta + cfg.gamma * cfg.lam * last;
      adv[b * R + j] = last;
    }
    for (int j = 0; j < R; ++j) ret[b * R + j] = adv[b * R + j] + values[b * R + j];
  }
  auto put = [](float* dst, const Vec& v) { if (dst) std::memcpy(dst, v.data(), v.size() * sizeof(float)); };
  put(out->logp_old, logp_old);
  put(out->logp_ref, logp_ref);
  put(out->values, values);
  put(out->score, score);
  put(out->rewards, rewards);
  put(out->advantages, adv);
  put(out->returns, ret);
  if (stop_after == 1) return 0;

  const float N = cfg.loss_denominator > 0 ? cfg.loss_denominator : static_cast<float>(B * R);

  // ---- TrainFB(Actor): clipped PPO policy loss, ppo_epochs passes over the experience
  // (one AdamW step each; the next pass runs on the bf16 copy of the updated master) ----
  Vec a_master = actor.w, a_m(a_master.size(), 0.0f), a_v(a_master.size(), 0.0f);
  for (int epoch = 0; epoch < ppo_epochs; ++epoch) {
    if (epoch > 0)
      for (size_t i = 0; i < actor.w.size(); ++i) actor.w[i] = bfr(a_master[i]);
    Saved sv;
    Cache c;
    c.init(actor.a.n_layers, B, S, actor.a.d_model);
    Vec hf = forward_chunk(actor, tok.data(), B, S, 0, S, c, &sv);
    Vec logp(logp_old.size());
    logprobs(actor, hf, tok.data(), B, S, P, logp.data());
    put(out->logp_new, logp);
    double loss = 0;
    Vec gl(logp.size());
    for (size_t k = 0; k < logp.size(); ++k) {
      const float ratio = std::exp(logp[k] - logp_old[k]);
      const float A = adv[k];
      const float cl = std::min(std::max(ratio, 1.0f - cfg.cliprange), 1.0f + cfg.cliprange);
      const float pg1 = -A * ratio, pg2 = -A * cl;
      loss += std::max(pg1, pg2);
      const bool inside = ratio >= 1.0f - cfg.cliprange && ratio <= 1.0f + cfg.cliprange;
      const float d1 = -A * ratio / N, d2 = inside ? -A * ratio / N : 0.0f;
      gl[k] = pg1 > pg2 ? d1 : (pg1 < pg2 ? d2 : 0.5f * (d1 + d2));
    }
    out->actor_loss = loss / N;
    // dlogits = g (onehot - softmax) -> bf16; dhf = dz E; dE += dz^T hf
    const int d = actor.a.d_model, V = actor.a.vocab;
    Vec dhf(static_cast<size_t>(B) * S * d, 0.0f);
    Vec grad(actor.w.size(), 0.0f);
    const int Mr = B * R;
    Vec dz(static_cast<size_t>(Mr) * V), hr(static_cast<size_t>(Mr) * d);
#pragma omp parallel
    {
      Vec z(static_cast<size_t>(V));
#pragma omp for schedule(static)
      for (int r = 0; r < Mr; ++r) {
        const int b = r / R, t = P - 1 + r % R;
        const float* hrow = hf.data() + (static_cast<size_t>(b) * S + t) * d;
        std::memcpy(hr.data() + static_cast<size_t>(r) * d, hrow, sizeof(float) * d);
        logits_row(actor, hrow, z.data());
        const float lse = logsumexp(z.data(), V);
        const int y = tok[static_cast<size_t>(b) * S + t + 1];
        for (int v = 0; v < V; ++v)
          dz[static_cast<size_t>(r) * V + v] = bfr(gl[r] * ((v == y ? 1.0f : 0.0f) - std::exp(z[v] - lse)));
      }
    }
    Vec dhr(static_cast<size_t>(Mr) * d);
    matmul_nn(dz.data(), Mr, V, actor.t(actor.head_id()), d, dhr.data());
    matmul_tn_acc(dz.data(), Mr, V, hr.data(), d, grad.data() + rlhf_tensor_offset(&actor.a, actor.head_id(), 0));
    for (int r = 0; r < Mr; ++r) {
      const int b = r / R, t = P - 1 + r % R;
      std::memcpy(dhf.data() + (static_cast<size_t>(b) * S + t) * d, dhr.data() + static_cast<size_t>(r) * d,
                  sizeof(float) * d);
    }
    backward(actor, tok.data(), B, S, sv, dhf, grad);
    put(out->actor_grad, grad);
    adamw(a_master, a_m, a_v, grad, cfg.lr_actor, cfg, epoch + 1);
    put(out->actor_master, a_master);
  }

  // ---- TrainFB(Critic): clipped value loss, ppo_epochs passes ------------------
  Vec c_master = critic.w, c_m(c_master.size(), 0.0f), c_v(c_master.size(), 0.0f);
  for (int epoch = 0; epoch < ppo_epochs; ++epoch) {
    if (epoch > 0)
      for (size_t i = 0; i < critic.w.size(); ++i) critic.w[i] = bfr(c_master[i]);
    Saved sv;
    Cache c;
    c.init(critic.a.n_layers, B, S, critic.a.d_model);
    Vec hf = forward_chunk(critic, tok.data(), B, S, 0, S, c, &sv);
    const int d = critic.a.d_model;
    const float* vh = critic.t(RLHF_T_VHEAD);
    Vec vals(values.size());
    for (int b = 0; b < B; ++b)
      for (int j = 0; j < R; ++j)
        vals[b * R + j] = dotf(hf.data() + (static_cast<size_t>(b) * S + P - 1 + j) * d, vh, d);
    put(out->values_new, vals);
    double loss = 0;
    Vec gv(vals.size());
    for (size_t k = 0; k < vals.size(); ++k) {
      const float v = vals[k], vo = values[k], Rt = ret[k];
      const float vc = std::min(std::max(v, vo - cfg.cliprange_value), vo + cfg.cliprange_value);
      const float l1 = (v - Rt) * (v - Rt), l2 = (vc - Rt) * (vc - Rt);
      loss += std::max(l1, l2);
      const bool inside = v >= vo - cfg.cliprange_value && v <= vo + cfg.cliprange_value;
      const float d1 = (v - Rt) / N, d2 = inside ? (vc - Rt) / N : 0.0f;
      gv[k] = l1 > l2 ? d1 : (l1 < l2 ? d2 : 0.5f * (d1 + d2));
    }
    out->critic_loss = 0.5 * loss / N;
    Vec dhf(static_cast<size_t>(B) * S * d, 0.0f);
    Vec grad(critic.w.size(), 0.0f);
    float* dvh = grad.data() + rlhf_tensor_offset(&critic.a, RLHF_T_VHEAD, 0);
    for (int b = 0; b < B; ++b)
      for (int j = 0; j < R; ++j) {
        const size_t row = static_cast<size_t>(b) * S + P - 1 + j;
        const float gk = gv[b * R + j];
        for (int e = 0; e < d; ++e) {
          dhf[row * d + e] = gk * vh[e];
          dvh[e] += gk * hf[row * d + e];
        }
      }
    backward(critic, tok.data(), B, S, sv, dhf, grad);
    put(out->critic_grad, grad);
    adamw(c_master, c_m, c_v, grad, cfg.lr_critic, cfg, epoch + 1);
    put(out->critic_master, c_master);
  }
  return 0;
}

extern "C" int oracle_ppo_step(const rlhf_ppo_config* cfg, const int32_t* tokens_in, int32_t* greedy_pred,
                               int stop_after, int n_threads, oracle_ppo_outputs* out) {
  return oracle_ppo_step_epochs(cfg, 1, tokens_in, greedy_pred, stop_after, n_threads, out);
}
