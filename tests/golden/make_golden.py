"""Generate golden vectors for the oracle (tests/golden/c1_golden.npz).

Independent restatement of the PPO step in torch (float64 autograd), used to pin
the C++ oracle (oracle/ppo_oracle.cpp), whose backward pass is hand-derived.
Nothing here is shared with the oracle except the INPUT format: the seeded
weight/prompt generator of include/rlhf_init.h, re-implemented below in numpy.

Forward rounding points (bf16) match the oracle's contract; they are
straight-through in autograd, so gradients here are exact float64 gradients of
the rounded forward -- the oracle (which also rounds gradients to bf16 at GEMM
inputs) must agree within the tolerances in tests/test_oracle_golden.py.

Numerics: DeepSpeed-Chat step 3.  Two fixtures:
  c1_golden.npz        OPT-style tiny decoder (family 0)
  c1_llama_golden.npz  LLaMA-style tiny decoder (family 1: RMSNorm, rotary, SwiGLU,
                       untied head).  Its torch restatement is itself pinned against
                       Hugging Face transformers' LlamaForCausalLM (float64, rounding
                       off) before the fixture is written, and the HF logprobs of the
                       golden tokens are stored (hf_logp) for a direct oracle-vs-HF test.
Run:
    python tests/golden/make_golden.py
"""
from __future__ import annotations

import os

import numpy as np
import torch

torch.set_default_dtype(torch.float64)
HERE = os.path.dirname(os.path.abspath(__file__))

# ---- rlhf_init.h re-implemented in numpy -----------------------------------
M64 = (1 << 64) - 1
T_TOK, T_POS, T_LN1G, T_LN1B, T_WQKV, T_BQKV, T_WO, T_BO, T_LN2G, T_LN2B, T_W1, T_B1, T_W2, T_B2, \
    T_LNFG, T_LNFB, T_VHEAD, T_LMHEAD = range(18)
LAYER_T = list(range(T_LN1G, T_B2 + 1))


def splitmix(x):
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def uniform(stream, counter):
    with np.errstate(over="ignore"):
        z = splitmix(np.uint64(stream) ^ splitmix(np.asarray(counter, np.uint64) + np.uint64(0x632BE59BD9B4E019)))
    return ((z >> np.uint64(11)).astype(np.float64) + 0.5) * (1.0 / 9007199254740992.0)


def normal(stream, n):
    i = np.arange(n, dtype=np.uint64)
    u1, u2 = uniform(stream, 2 * i), uniform(stream, 2 * i + np.uint64(1))
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(6.283185307179586 * u2)


def to_bf16(x):
    """float -> bf16 value (float64 holding it), round-to-nearest-even via float32."""
    f = np.asarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    return (u.astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


def stream_of(seed, t, l):
    with np.errstate(over="ignore"):
        v = np.uint64(seed) * np.uint64(0x100000001B3) + np.uint64(t * 4099) + np.uint64(l * 131) + np.uint64(17)
    return int(splitmix(v))


def init_dist(arch, t):
    if t == T_LMHEAD:
        return 0.0, 2.0 / np.sqrt(arch["d"])
    if t == T_TOK:
        return 0.0, 2.0 / np.sqrt(arch["d"])
    if t == T_POS:
        return 0.0, 1.0
    if t in (T_LN1G, T_LN2G, T_LNFG):
        return 1.0, 0.05
    if t == T_VHEAD:
        return 0.0, 1.0 / np.sqrt(arch["d"])
    if t in (T_WQKV, T_WO, T_W1):
        return 0.0, 1.0 / np.sqrt(arch["d"])
    if t == T_W2:
        return 0.0, 1.0 / np.sqrt(arch["ff"])
    return 0.0, 0.02


def shape_of(arch, t):
    V, d, f, mp = arch["V"], arch["d"], arch["ff"], arch["max_pos"]
    if arch.get("family", 0) == 1 and t == T_W1:
        return (2 * f, d)  # [gate | up]
    return {T_LMHEAD: (V, d), T_TOK: (V, d), T_POS: (mp, d), T_WQKV: (3 * d, d), T_BQKV: (3 * d,), T_WO: (d, d),
            T_W1: (f, d), T_B1: (f,), T_W2: (d, f), T_VHEAD: (d,)}.get(t, (d,))


def make_weights(arch, seed, scalar_head):
    if arch.get("family", 0) == 1:
        return make_weights_llama(arch, seed, scalar_head)

    def gen(t, l):
        shp = shape_of(arch, t)
        mean, std = init_dist(arch, t)
        return torch.tensor(to_bf16(mean + std * normal(stream_of(seed, t, l), int(np.prod(shp)))).reshape(shp))
    w = {"tok": gen(T_TOK, 0), "pos": gen(T_POS, 0), "lnf_g": gen(T_LNFG, 0), "lnf_b": gen(T_LNFB, 0), "layers": []}
    names = ["ln1_g", "ln1_b", "wqkv", "bqkv", "wo", "bo", "ln2_g", "ln2_b", "w1", "b1", "w2", "b2"]
    for l in range(arch["L"]):
        w["layers"].append({n: gen(t, l) for n, t in zip(names, LAYER_T)})
    if scalar_head:
        w["vhead"] = gen(T_VHEAD, 0)
    return w


def make_weights_llama(arch, seed, scalar_head):
    def gen(t, l):
        shp = shape_of(arch, t)
        mean, std = init_dist(arch, t)
        return torch.tensor(to_bf16(mean + std * normal(stream_of(seed, t, l), int(np.prod(shp)))).reshape(shp))
    w = {"tok": gen(T_TOK, 0), "lnf_g": gen(T_LNFG, 0), "layers": []}
    names = {"ln1_g": T_LN1G, "wqkv": T_WQKV, "wo": T_WO, "ln2_g": T_LN2G, "w1": T_W1, "w2": T_W2}
    for l in range(arch["L"]):
        w["layers"].append({n: gen(t, l) for n, t in names.items()})
    if scalar_head:
        w["vhead"] = gen(T_VHEAD, 0)
    else:
        w["lm_head"] = gen(T_LMHEAD, 0)
    return w


def prompt_token(seed, b, t, V):
    with np.errstate(over="ignore"):
        z = splitmix(splitmix(np.uint64(seed) ^ np.uint64(0xA5A5A5A5)) + np.uint64(b * 1000003) + np.uint64(t))
    return int(z % np.uint64(V))


# ---- model in torch ----------------------------------------------------------
class RoundBF16(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x):
        return torch.tensor(to_bf16(x.detach().numpy()))

    @staticmethod
    def backward(ctx, g):
        return g


rb = RoundBF16.apply


def layernorm(x, g, b):
    mu = x.mean(-1, keepdim=True)
    var = ((x - mu) ** 2).mean(-1, keepdim=True)
    return (x - mu) / torch.sqrt(var + 1e-5) * g + b


def rmsnorm(x, g):
    return x / torch.sqrt((x * x).mean(-1, keepdim=True) + 1e-6) * g


def rope_tables(S, hd):
    """rlhf_rope_cos_sin: angle in float64, cos/sin rounded to float32."""
    i = np.arange(hd // 2, dtype=np.float64)
    ang = np.arange(S, dtype=np.float64)[:, None] * np.power(10000.0, -2.0 * i / hd)[None]
    return (torch.tensor(np.cos(ang).astype(np.float32).astype(np.float64)),
            torch.tensor(np.sin(ang).astype(np.float32).astype(np.float64)))


def rope(x, c, s):
    """x [B,H,S,hd]: pair (i, i + hd/2) rotated by position angle (HF LLaMA rotate_half)."""
    half = x.shape[-1] // 2
    x0, x1 = x[..., :half], x[..., half:]
    return torch.cat([x0 * c - x1 * s, x1 * c + x0 * s], -1)


def decoder_llama(w, tok, arch, r=None):
    """LLaMA family: tok [B,S] -> final RMSNorm hidden [B,S,d]; r = rounding (rb, or identity)."""
    r = r or rb
    B, S = tok.shape
    d, H, ff = arch["d"], arch["H"], arch["ff"]
    hd = d // H
    c, s = rope_tables(S, hd)
    x = w["tok"][tok]
    mask = torch.ones(S, S, dtype=torch.bool).tril()
    for lw in w["layers"]:
        h = r(rmsnorm(x, lw["ln1_g"]))
        qkv = r(h @ lw["wqkv"].T)
        q, k, v = qkv.split(d, -1)
        q = r(rope(q.view(B, S, H, hd).transpose(1, 2), c, s))
        k = r(rope(k.view(B, S, H, hd).transpose(1, 2), c, s))
        v = v.view(B, S, H, hd).transpose(1, 2)
        sc = (q @ k.transpose(-1, -2)) * (1.0 / np.sqrt(hd))
        sc = sc.masked_fill(~mask, float("-inf"))
        p = r(torch.softmax(sc, -1))
        o = r((p @ v).transpose(1, 2).reshape(B, S, d))
        x = x + o @ lw["wo"].T
        h2 = r(rmsnorm(x, lw["ln2_g"]))
        gu = r(h2 @ lw["w1"].T)
        g, u = gu.split(ff, -1)
        a = r(g * torch.sigmoid(g) * u)
        x = x + a @ lw["w2"].T
    return r(rmsnorm(x, w["lnf_g"]))


def hf_llama(w, arch):
    """The same weights in transformers' LlamaForCausalLM (float64)."""
    from transformers import LlamaConfig, LlamaForCausalLM
    d, ff = arch["d"], arch["ff"]
    cfg = LlamaConfig(vocab_size=arch["V"], hidden_size=d, intermediate_size=ff, num_hidden_layers=arch["L"],
                      num_attention_heads=arch["H"], num_key_value_heads=arch["H"], rms_norm_eps=1e-6,
                      rope_theta=10000.0, max_position_embeddings=arch["max_pos"], tie_word_embeddings=False,
                      attention_bias=False, mlp_bias=False)
    m = LlamaForCausalLM(cfg).double().eval()
    with torch.no_grad():
        m.model.embed_tokens.weight.copy_(w["tok"])
        for lw, L in zip(w["layers"], m.model.layers):
            L.self_attn.q_proj.weight.copy_(lw["wqkv"][:d])
            L.self_attn.k_proj.weight.copy_(lw["wqkv"][d:2 * d])
            L.self_attn.v_proj.weight.copy_(lw["wqkv"][2 * d:])
            L.self_attn.o_proj.weight.copy_(lw["wo"])
            L.mlp.gate_proj.weight.copy_(lw["w1"][:ff])
            L.mlp.up_proj.weight.copy_(lw["w1"][ff:])
            L.mlp.down_proj.weight.copy_(lw["w2"])
            L.input_layernorm.weight.copy_(lw["ln1_g"])
            L.post_attention_layernorm.weight.copy_(lw["ln2_g"])
        m.model.norm.weight.copy_(w["lnf_g"])
        m.lm_head.weight.copy_(w["lm_head"])
    return m


def hf_opt(w, arch):
    """The same weights in transformers' OPTForCausalLM (float64).  OPT's learned position
    table is offset by 2 (OPTLearnedPositionalEmbedding), so row p of ours is its row p + 2;
    the LM head is tied to the token embedding as in our layout."""
    from transformers import OPTConfig, OPTForCausalLM
    d, ff = arch["d"], arch["ff"]
    cfg = OPTConfig(vocab_size=arch["V"], hidden_size=d, num_hidden_layers=arch["L"], ffn_dim=ff,
                    num_attention_heads=arch["H"], max_position_embeddings=arch["max_pos"], do_layer_norm_before=True,
                    word_embed_proj_dim=d, activation_function="relu", dropout=0.0, attention_dropout=0.0,
                    layerdrop=0.0, enable_bias=True, layer_norm_elementwise_affine=True, tie_word_embeddings=True,
                    pad_token_id=1, bos_token_id=2, eos_token_id=2)
    m = OPTForCausalLM(cfg).double().eval()
    dec = m.model.decoder
    with torch.no_grad():
        dec.embed_tokens.weight.copy_(w["tok"])
        dec.embed_positions.weight.zero_()
        dec.embed_positions.weight[2:2 + w["pos"].shape[0]].copy_(w["pos"])
        for lw, L in zip(w["layers"], dec.layers):
            a = L.self_attn
            for proj, sl in ((a.q_proj, slice(0, d)), (a.k_proj, slice(d, 2 * d)), (a.v_proj, slice(2 * d, 3 * d))):
                proj.weight.copy_(lw["wqkv"][sl])
                proj.bias.copy_(lw["bqkv"][sl])
            a.out_proj.weight.copy_(lw["wo"])
            a.out_proj.bias.copy_(lw["bo"])
            L.self_attn_layer_norm.weight.copy_(lw["ln1_g"])
            L.self_attn_layer_norm.bias.copy_(lw["ln1_b"])
            L.final_layer_norm.weight.copy_(lw["ln2_g"])
            L.final_layer_norm.bias.copy_(lw["ln2_b"])
            L.fc1.weight.copy_(lw["w1"])
            L.fc1.bias.copy_(lw["b1"])
            L.fc2.weight.copy_(lw["w2"])
            L.fc2.bias.copy_(lw["b2"])
        dec.final_layer_norm.weight.copy_(w["lnf_g"])
        dec.final_layer_norm.bias.copy_(w["lnf_b"])
        m.lm_head.weight.copy_(w["tok"])
    return m


def decoder(w, tok, arch, r=None):
    """tok [B,S] long -> final-LN hidden [B,S,d] (bf16-rounded; r=identity turns rounding off)."""
    if arch.get("family", 0) == 1:
        return decoder_llama(w, tok, arch, r)
    rb_ = r or rb
    B, S = tok.shape
    d, H = arch["d"], arch["H"]
    hd = d // H
    x = w["tok"][tok] + w["pos"][:S][None]
    mask = torch.ones(S, S, dtype=torch.bool).tril()
    for lw in w["layers"]:
        h = rb_(layernorm(x, lw["ln1_g"], lw["ln1_b"]))
        qkv = rb_(h @ lw["wqkv"].T + lw["bqkv"])
        q, k, v = qkv.split(d, -1)
        q = q.view(B, S, H, hd).transpose(1, 2)
        k = k.view(B, S, H, hd).transpose(1, 2)
        v = v.view(B, S, H, hd).transpose(1, 2)
        s = (q @ k.transpose(-1, -2)) * (1.0 / np.sqrt(hd))
        s = s.masked_fill(~mask, float("-inf"))
        p = rb_(torch.softmax(s, -1))
        o = rb_((p @ v).transpose(1, 2).reshape(B, S, d))
        x = x + (o @ lw["wo"].T + lw["bo"])
        h2 = rb_(layernorm(x, lw["ln2_g"], lw["ln2_b"]))
        f = rb_(torch.relu(h2 @ lw["w1"].T + lw["b1"]))
        x = x + (f @ lw["w2"].T + lw["b2"])
    return rb_(layernorm(x, w["lnf_g"], w["lnf_b"]))


def params_of(w):
    """Parameters in the flat layout order of rlhf_init.h (absent tensors skipped)."""
    ps = [w["tok"]] + ([w["pos"]] if "pos" in w else [])
    for lw in w["layers"]:
        ps += list(lw.values())
    ps += [w["lnf_g"]] + ([w["lnf_b"]] if "lnf_b" in w else [])
    if "vhead" in w:
        ps.append(w["vhead"])
    if "lm_head" in w:
        ps.append(w["lm_head"])
    return ps


def param_names(w, arch):
    names = ["tok"] + (["pos"] if "pos" in w else [])
    names += [f"l{l}.{k}" for l in range(arch["L"]) for k in w["layers"][l]]
    names += ["lnf_g"] + (["lnf_b"] if "lnf_b" in w else [])
    names += (["vhead"] if "vhead" in w else []) + (["lm_head"] if "lm_head" in w else [])
    return names


def head_of(w):
    return w["lm_head"] if "lm_head" in w else w["tok"]


def main():
    run(dict(V=512, d=128, L=2, H=2, ff=512, max_pos=64), "c1_golden.npz")
    run(dict(family=1, V=512, d=128, L=2, H=2, ff=384, max_pos=64), "c1_llama_golden.npz")
    hf_pins()


# OPT shapes pinned against transformers' OPTForCausalLM (teacher-forced logprobs of a fixed
# sequence under the Actor's seeded weights): the c1 tiny decoder and the OPT-125m shape of
# BASELINE.json configs[1] at a short sequence (P + R = 32 + 32, max_pos 64).
HF_PINS = {"tiny": (dict(V=512, d=128, L=2, H=2, ff=512, max_pos=64), 2, 16, 16),
           "opt-125m": (dict(V=50272, d=768, L=12, H=12, ff=3072, max_pos=64), 1, 32, 32)}


def hf_pins(fname="hf_opt_pins.npz"):
    seed, prompt_seed = 7, 1000
    fx = {}
    for name, (arch, B, P, R) in HF_PINS.items():
        S = P + R
        actor = make_weights(arch, seed * 16 + 0, False)
        tok = torch.zeros(B, S, dtype=torch.long)
        for b in range(B):
            for t in range(S):  # prompt ids for t < P; the "response" continues the same seeded stream
                tok[b, t] = prompt_token(prompt_seed, b, t, arch["V"])
        m = hf_opt(actor, arch)
        with torch.no_grad():
            z_hf = m(tok).logits
            z_me = decoder(actor, tok, arch, r=lambda t: t) @ actor["tok"].T
            err = (z_hf - z_me).abs().max().item()
            assert err < 1e-4, f"{name}: OPT restatement differs from transformers by {err}"
            hf_logp = torch.log_softmax(z_hf[:, P - 1:S - 1], -1).gather(-1, tok[:, P:, None])[..., 0]
        fx[f"{name}/config"] = np.array([B, P, R, seed, prompt_seed, arch["max_pos"]])
        fx[f"{name}/tokens"] = tok.numpy().astype(np.int32)
        fx[f"{name}/hf_logp"] = hf_logp.numpy().astype(np.float32)
        fx[f"{name}/hf_max_abs_logit_diff"] = np.array(err)
        print(name, "restatement vs transformers max |dlogit|", err)
    np.savez_compressed(os.path.join(HERE, fname), **fx)


def run(arch, fname):
    B, P, R = 4, 16, 16
    S = P + R
    seed, prompt_seed = 7, 1000
    kl_ctl, clip_reward, gamma, lam, clip, clipv = 0.1, 5.0, 1.0, 0.95, 0.2, 0.2

    actor = make_weights(arch, seed * 16 + 0, False)
    critic = make_weights(arch, seed * 16 + 1, True)
    ref = make_weights(arch, seed * 16 + 2, False)
    reward = make_weights(arch, seed * 16 + 3, True)

    tok = torch.zeros(B, S, dtype=torch.long)
    for b in range(B):
        for t in range(P):
            tok[b, t] = prompt_token(prompt_seed, b, t, arch["V"])
    margins = np.zeros((B, R))
    with torch.no_grad():  # greedy generation by full recomputation (no KV cache)
        for step in range(R):
            t = P - 1 + step
            hf = decoder(actor, tok[:, : t + 1], arch)
            z = hf[:, t] @ head_of(actor).T
            top = torch.topk(z, 2, -1)
            tok[:, t + 1] = top.indices[:, 0]
            margins[:, step] = (top.values[:, 0] - top.values[:, 1]).numpy()

    def logprobs(w, hf):
        z = hf[:, P - 1:S - 1] @ head_of(w).T
        return torch.log_softmax(z, -1).gather(-1, tok[:, P:, None])[..., 0]

    with torch.no_grad():
        logp_old = logprobs(actor, decoder(actor, tok, arch))
        values = decoder(critic, tok, arch)[:, P - 1:S - 1] @ critic["vhead"]
        logp_ref = logprobs(ref, decoder(ref, tok, arch))
        score = decoder(reward, tok, arch)[:, S - 1] @ reward["vhead"]
        rewards = -kl_ctl * (logp_old - logp_ref)
        rewards[:, -1] += score.clamp(-clip_reward, clip_reward)
        adv = torch.zeros(B, R)
        last = torch.zeros(B)
        for j in reversed(range(R)):
            nextv = values[:, j + 1] if j < R - 1 else torch.zeros(B)
            delta = rewards[:, j] + gamma * nextv - values[:, j]
            last = delta + gamma * lam * last
            adv[:, j] = last
        returns = adv + values

    N = B * R
    for p in params_of(actor):
        p.requires_grad_(True)
    logp = logprobs(actor, decoder(actor, tok, arch))
    ratio = torch.exp(logp - logp_old)
    actor_loss = torch.sum(torch.max(-adv * ratio, -adv * ratio.clamp(1 - clip, 1 + clip))) / N
    actor_loss.backward()

    for p in params_of(critic):
        p.requires_grad_(True)
    v = decoder(critic, tok, arch)[:, P - 1:S - 1] @ critic["vhead"]
    vc = torch.max(torch.min(v, values + clipv), values - clipv)
    critic_loss = 0.5 * torch.sum(torch.max((v - returns) ** 2, (vc - returns) ** 2)) / N
    critic_loss.backward()

    def grad_summary(w):
        out = {}
        for name, p in zip(param_names(w, arch), params_of(w)):
            g = p.grad.detach().numpy().ravel()
            out[name] = (g[:256].astype(np.float32), float(np.linalg.norm(g)), float(g.sum()))
        return out

    fx = dict(
        config=np.array([B, P, R, seed, prompt_seed]), arch=np.array([arch[k] for k in ("V", "d", "L", "H", "ff", "max_pos")]),
        family=np.array(arch.get("family", 0)),
        tokens=tok.numpy().astype(np.int32), margins=margins.astype(np.float32),
        logp_old=logp_old.numpy().astype(np.float32), logp_ref=logp_ref.numpy().astype(np.float32),
        values=values.numpy().astype(np.float32), score=score.numpy().astype(np.float32),
        rewards=rewards.numpy().astype(np.float32), advantages=adv.numpy().astype(np.float32),
        returns=returns.numpy().astype(np.float32), losses=np.array([actor_loss.item(), critic_loss.item()]),
    )
    for tag, w in (("actor", actor), ("critic", critic)):
        for name, (head, norm, tot) in grad_summary(w).items():
            fx[f"{tag}_grad/{name}/head"] = head
            fx[f"{tag}_grad/{name}/stats"] = np.array([norm, tot])
    if arch.get("family", 0) == 1:
        # pin the restatement's semantics against transformers' LLaMA (rounding off), then
        # store HF's own logprobs of the golden tokens for the oracle-vs-HF test
        actor_d = {k: (v.detach() if torch.is_tensor(v) else [{n: t.detach() for n, t in lw.items()} for lw in v])
                   for k, v in actor.items()}
        m = hf_llama(actor_d, arch)
        with torch.no_grad():
            z_hf = m(tok).logits
            z_me = decoder_llama(actor_d, tok, arch, r=lambda t: t) @ actor_d["lm_head"].T
            err = (z_hf - z_me).abs().max().item()
            assert err < 1e-4, f"LLaMA restatement differs from transformers by {err}"
            hf_logp = torch.log_softmax(z_hf[:, P - 1:S - 1], -1).gather(-1, tok[:, P:, None])[..., 0]
        fx["hf_logp"] = hf_logp.numpy().astype(np.float32)
        fx["hf_max_abs_logit_diff"] = np.array(err)
    np.savez_compressed(os.path.join(HERE, fname), **fx)
    print("wrote", os.path.join(HERE, fname), "losses", fx["losses"], "min margin", margins.min())


if __name__ == "__main__":
    import sys
    hf_pins() if sys.argv[1:] == ["hf"] else main()
