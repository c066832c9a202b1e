"""ctypes mirror of the C-ABI in include/rlhf_engine.h and include/rlhf_kernels.h.

The product library is ``paper_2312_11819_b200/lib/librlhf_b200.so`` (built by
``paper_2312_11819_b200.build``).  Loading fails loudly when it is missing:
there is no CPU fallback for any engine entry point.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "librlhf_b200.so")


class Arch(C.Structure):
    _fields_ = [("family", C.c_int), ("vocab", C.c_int), ("d_model", C.c_int), ("n_layers", C.c_int),
                ("n_heads", C.c_int), ("d_ff", C.c_int), ("max_pos", C.c_int), ("scalar_head", C.c_int)]


class PPOConfig(C.Structure):
    _fields_ = [("actor", Arch), ("critic", Arch), ("batch", C.c_int), ("prompt_len", C.c_int),
                ("gen_len", C.c_int), ("seed", C.c_uint64), ("prompt_seed", C.c_uint64),
                ("sample_offset", C.c_int), ("kl_ctl", C.c_float), ("clip_reward", C.c_float),
                ("gamma", C.c_float), ("lam", C.c_float), ("cliprange", C.c_float),
                ("cliprange_value", C.c_float), ("lr_actor", C.c_float), ("lr_critic", C.c_float),
                ("beta1", C.c_float), ("beta2", C.c_float), ("adam_eps", C.c_float),
                ("weight_decay", C.c_float), ("loss_denominator", C.c_float)]


class EngineOptions(C.Structure):
    _fields_ = [("device", C.c_int), ("rank", C.c_int), ("world_size", C.c_int), ("strategy", C.c_char_p),
                ("nccl_id", C.POINTER(C.c_uint8)), ("use_cuda_graph", C.c_int), ("zero_stage", C.c_int),
                ("train_micro_batch", C.c_int), ("micro_batches", C.c_int), ("rollout_nums", C.c_int),
                ("ppo_epochs", C.c_int), ("inference_ratio", C.c_double), ("tp_gen", C.c_int),
                ("ratios", C.c_double * 4)]


class StepReport(C.Structure):
    _fields_ = [("step_seconds", C.c_double), ("throughput_samples_per_sec", C.c_double),
                ("stage_seconds", C.c_double * 4), ("decode_seconds", C.c_double),
                ("prefill_seconds", C.c_double), ("comm_bytes_total", C.c_double),
                ("actor_loss", C.c_double), ("critic_loss", C.c_double), ("mean_score", C.c_double),
                ("mean_kl", C.c_double), ("gpu_launches", C.c_int), ("busy_seconds", C.c_double),
                ("bubble_fraction", C.c_double), ("comm_seconds", C.c_double), ("mem_peak_bytes", C.c_double),
                ("busiest_stage", C.c_int), ("n_events", C.c_int), ("feasible", C.c_int)]


class Event(C.Structure):
    """rlhf_event: one measured interval of the last step (SimEvent, simulator.hpp:18-28)."""
    _fields_ = [("task", C.c_int), ("kind", C.c_int), ("model", C.c_int), ("micro_batch", C.c_int),
                ("rollout", C.c_int), ("epoch", C.c_int), ("lane", C.c_int), ("comm_op", C.c_int),
                ("stage", C.c_int), ("start", C.c_double), ("end", C.c_double)]


# Named shapes (SURVEY.md §8 model table); max_pos is set per pipeline.
ARCHS = {
    "tiny": dict(vocab=512, d_model=128, n_layers=2, n_heads=2, d_ff=512),
    "opt-125m": dict(vocab=50272, d_model=768, n_layers=12, n_heads=12, d_ff=3072),
    "opt-350m": dict(vocab=50272, d_model=1024, n_layers=24, n_heads=16, d_ff=4096),
    "opt-1.3b": dict(vocab=50272, d_model=2048, n_layers=24, n_heads=32, d_ff=8192),
    # LLaMA family (family 1: RMSNorm, SwiGLU, rotary, no biases, untied head)
    "llama-tiny": dict(family=1, vocab=512, d_model=128, n_layers=2, n_heads=2, d_ff=384),
    "llama-tiny-hd128": dict(family=1, vocab=512, d_model=256, n_layers=2, n_heads=2, d_ff=704),
    # LLaMA mid shape for end-to-end parity at S = 512 (head_dim 128, the 7B's)
    "llama-mid": dict(family=1, vocab=32000, d_model=1024, n_layers=4, n_heads=8, d_ff=2816),
    "llama-1b": dict(family=1, vocab=32000, d_model=2048, n_layers=16, n_heads=16, d_ff=5504),
    "llama-7b": dict(family=1, vocab=32000, d_model=4096, n_layers=32, n_heads=32, d_ff=11008),
}


def make_arch(name: str, max_pos: int, scalar_head: int) -> Arch:
    a = ARCHS[name]
    return Arch(a.get("family", 0), a["vocab"], a["d_model"], a["n_layers"], a["n_heads"], a["d_ff"], max_pos,
                scalar_head)


def make_config(actor: str, critic: str, batch: int, prompt_len: int, gen_len: int, seed: int = 7,
                prompt_seed: int = 1000, sample_offset: int = 0, loss_denominator: float = 0.0) -> PPOConfig:
    """Defaults = rlhf_ppo_config_default (DeepSpeed-Chat step-3 values)."""
    S = prompt_len + gen_len
    mp = max(64, (S + 63) // 64 * 64)
    return PPOConfig(make_arch(actor, mp, 0), make_arch(critic, mp, 1), batch, prompt_len, gen_len, seed,
                     prompt_seed, sample_offset, 0.1, 5.0, 1.0, 0.95, 0.2, 0.2, 1e-5, 5e-6, 0.9, 0.95,
                     1e-8, 0.0, loss_denominator)


def param_total(a: Arch) -> int:
    """rlhf_param_total() of include/rlhf_init.h (flat layout incl. 64-element alignment)."""
    al = lambda n: (n + 63) // 64 * 64
    return tensor_offset(a, 17) + al(tensor_numel(a, 17))


_lib = None


def lib() -> C.CDLL:
    """Load the engine library (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run paper_2312_11819_b200.build.build() first "
                               "(there is no CPU fallback)")
        # torch first: its libnccl.so.2 is the one the engine dlopens (nccl_dyn.hpp)
        import torch  # noqa: F401
        _lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
        _declare(_lib)
    return _lib


def _declare(L: C.CDLL) -> None:
    i, p, vp = C.c_int, C.POINTER, C.c_void_p
    L.rlhf_last_error.restype = C.c_char_p
    if not hasattr(L, "rlhf_engine_create"):
        return
    L.rlhf_task_graph.argtypes = [i] * 8 + [p(i)] * 9
    L.rlhf_plan.argtypes = [C.c_char_p, i, i, C.c_double, i, p(C.c_uint32), p(i), C.c_char_p, i]
    L.rlhf_comm_schedule.argtypes = [C.c_char_p, i, i, i, i, i, i, p(i), p(i), p(i), p(i), p(C.c_double),
                                     p(C.c_uint32)]
    L.rlhf_nccl_unique_id.argtypes = [p(C.c_uint8)]
    L.rlhf_engine_create.argtypes = [p(PPOConfig), p(EngineOptions), p(vp)]
    L.rlhf_engine_destroy.argtypes = [vp]
    L.rlhf_engine_destroy.restype = None
    L.rlhf_engine_step.argtypes = [vp, p(C.c_int32), p(StepReport)]
    L.rlhf_engine_read.argtypes = [vp, C.c_char_p, vp, C.c_size_t]
    L.rlhf_engine_tensor_bytes.argtypes = [vp, C.c_char_p]
    L.rlhf_engine_tensor_bytes.restype = C.c_size_t
    L.rlhf_engine_stream.argtypes = [vp]
    L.rlhf_engine_stream.restype = vp
    L.rlhf_engine_greedy_check.argtypes = [vp, p(C.c_int32), p(C.c_int32), p(C.c_float)]


def check(status: int) -> None:
    if status != 0:
        msg = lib().rlhf_last_error().decode(errors="replace")
        raise RuntimeError(f"rlhf C-ABI error {status}: {msg}")


# ---- flat parameter layout (include/rlhf_init.h) ------------------------------
TENSOR_NAMES = ["tok", "pos", "ln1_g", "ln1_b", "wqkv", "bqkv", "wo", "bo", "ln2_g", "ln2_b", "w1", "b1", "w2",
                "b2", "lnf_g", "lnf_b", "vhead", "lm_head"]
LAYER_FIRST, LAYER_LAST = 2, 13


def tensor_numel(a: Arch, t: int) -> int:
    V, d, f = a.vocab, a.d_model, a.d_ff
    if a.family == 1:
        if t in (1, 3, 9, 15, 5, 7, 11, 13):  # pos, LN betas, biases
            return 0
        if t == 10:
            return 2 * f * d
        if t == 17:
            return 0 if a.scalar_head else V * d
    if t == 17:
        return 0
    return {0: V * d, 1: a.max_pos * d, 4: 3 * d * d, 5: 3 * d, 6: d * d, 10: f * d, 11: f, 12: d * f,
            16: d if a.scalar_head else 0}.get(t, d)


def tensor_offset(a: Arch, t: int, l: int = 0) -> int:
    al = lambda n: (n + 63) // 64 * 64
    off = al(tensor_numel(a, 0))
    if t == 0:
        return 0
    if t == 1:
        return off
    off += al(tensor_numel(a, 1))
    per_layer = sum(al(tensor_numel(a, k)) for k in range(LAYER_FIRST, LAYER_LAST + 1))
    if LAYER_FIRST <= t <= LAYER_LAST:
        return off + per_layer * l + sum(al(tensor_numel(a, k)) for k in range(LAYER_FIRST, t))
    off += per_layer * a.n_layers
    return off + sum(al(tensor_numel(a, k)) for k in range(14, t))


def named_slices(a: Arch):
    """[(name, offset, numel)] in layout order; per-layer names are 'l{l}.{name}'."""
    out = [("tok", 0, tensor_numel(a, 0)), ("pos", tensor_offset(a, 1), tensor_numel(a, 1))]
    for l in range(a.n_layers):
        for t in range(LAYER_FIRST, LAYER_LAST + 1):
            out.append((f"l{l}.{TENSOR_NAMES[t]}", tensor_offset(a, t, l), tensor_numel(a, t)))
    out += [("lnf_g", tensor_offset(a, 14), a.d_model), ("lnf_b", tensor_offset(a, 15), tensor_numel(a, 15))]
    if a.scalar_head:
        out.append(("vhead", tensor_offset(a, 16), a.d_model))
    if tensor_numel(a, 17):
        out.append(("lm_head", tensor_offset(a, 17), tensor_numel(a, 17)))
    return [s for s in out if s[2] > 0]


def prompt_tokens(seed: int, batch: int, prompt_len: int, vocab: int, sample_offset: int = 0):
    """rlhf_prompt_token() of include/rlhf_init.h, vectorised: uniform iid ids in [0, vocab)."""
    import numpy as np

    def splitmix(x):
        with np.errstate(over="ignore"):
            x = x + np.uint64(0x9E3779B97F4A7C15)
            x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            return x ^ (x >> np.uint64(31))

    b = np.arange(sample_offset, sample_offset + batch, dtype=np.uint64)[:, None]
    t = np.arange(prompt_len, dtype=np.uint64)[None, :]
    with np.errstate(over="ignore"):
        z = splitmix(splitmix(np.uint64(seed) ^ np.uint64(0xA5A5A5A5)) + b * np.uint64(1000003) + t)
    return (z % np.uint64(vocab)).astype(np.int32)


def exec_plan(strategy: str, world: int, batch_per_rank: int, prompt_len: int, gen_len: int, micro_batches: int = 1,
              rollout_nums: int = 1, ppo_epochs: int = 1, inference_ratio: float = 0.5, ratios=None) -> dict:
    """The executed plan (csrc/host/execplan.hpp) the engine walks: row sets, model -> set, the
    task DAG, the derived comm schedule and every exchange step's row transfers (JSON)."""
    import json
    L = lib()
    L.rlhf_exec_plan_json.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                      C.c_double, C.POINTER(C.c_double), C.c_char_p, C.c_int, C.POINTER(C.c_int)]
    r4 = (C.c_double * 4)(*ratios) if ratios is not None else None
    need = C.c_int(0)
    args = (strategy.encode(), world, batch_per_rank, prompt_len, gen_len, micro_batches, rollout_nums, ppo_epochs,
            inference_ratio, r4)
    check(L.rlhf_exec_plan_json(*args, None, 0, C.byref(need)))
    buf = C.create_string_buffer(need.value)
    check(L.rlhf_exec_plan_json(*args, buf, need.value, C.byref(need)))
    return json.loads(buf.value.decode())


def sim_run(command: str, payload) -> object:
    """The planner/simulator front end (rlhf_sim_run): command in simulate | trace | compare |
    maxbatch | plan | search | calibrate; payload a scenario dict (calibrate: {"scenario",
    "observations"}) or its JSON text.  Returns the parsed JSON result."""
    import json
    L = lib()
    L.rlhf_sim_run.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_int, C.POINTER(C.c_int)]
    text = payload if isinstance(payload, str) else json.dumps(payload)
    need = C.c_int(0)
    check(L.rlhf_sim_run(command.encode(), text.encode(), None, 0, C.byref(need)))
    buf = C.create_string_buffer(need.value)
    check(L.rlhf_sim_run(command.encode(), text.encode(), buf, need.value, C.byref(need)))
    return json.loads(buf.value.decode())
