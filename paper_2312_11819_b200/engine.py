"""Python handle on the C++ PPO-step engine (rlhf_engine_* in include/rlhf_engine.h).

    eng = Engine(make_config("tiny", "tiny", 4, 16, 16))
    rep = eng.step()                # one PPO iteration on cuda:<device>
    logp = eng.read("logp_old")     # any named engine tensor, as numpy

The reference's executor slot is ``simulate(plan, pipeline, cost, topo, opts)``
(/root/reference/proj/include/rlhfsim/simulator.hpp:46-47); ``Engine.step`` is
its executed counterpart and returns the same report fields (SimReport,
simulator.hpp:30-44) measured with CUDA events.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from .capi import EngineOptions, Event, PPOConfig, StepReport, check, lib

STAGES = ("generation", "forward", "training", "sync")
MODELS = ("Actor", "Critic", "Ref", "Reward", "ShadowActor", "ShadowCritic")
EVENT_KINDS = {0: "Generation", 1: "Forward", 2: "TrainFB", 3: "Collective", 4: "ParamSync", 6: "Experience",
               7: "AdamW"}

_DTYPES = {"tokens": np.int32, "pred": np.int32, "sample_ids": np.int32, "actor_params": np.uint16,
           "critic_params": np.uint16, "ref_params": np.uint16, "reward_params": np.uint16,
           "shadow_actor_params": np.uint16, "shadow_critic_params": np.uint16}


class Engine:
    def __init__(self, cfg: PPOConfig, device: int = 0, rank: int = 0, world_size: int = 1,
                 strategy: str = "colocated", nccl_id: bytes | None = None, cuda_graph: int = 1,
                 zero_stage: int = 0, train_micro_batch: int = 0, micro_batches: int = 1, rollout_nums: int = 1,
                 ppo_epochs: int = 1, inference_ratio: float = 0.5, ratios=None):
        L = lib()
        self._cfg = cfg
        self._keep = []
        idp = None
        if nccl_id is not None:
            buf = (C.c_uint8 * 128).from_buffer_copy(nccl_id)
            self._keep.append(buf)
            idp = C.cast(buf, C.POINTER(C.c_uint8))
        opt = EngineOptions(device, rank, world_size, strategy.encode(), idp, int(cuda_graph), int(zero_stage),
                            int(train_micro_batch), int(micro_batches), int(rollout_nums), int(ppo_epochs),
                            float(inference_ratio), 1, (C.c_double * 4)(*(ratios or (0, 0, 0, 0))))
        self.rollouts = int(rollout_nums)
        h = C.c_void_p()
        check(L.rlhf_engine_create(C.byref(cfg), C.byref(opt), C.byref(h)))
        self._h = h

    @staticmethod
    def max_batch(cfg: PPOConfig, cap: int, run_step: bool = False, device: int = 0, **kw) -> int:
        """max_batch_search against the real allocator (rlhf_engine_max_batch, one GPU)."""
        L = lib()
        L.rlhf_engine_max_batch.argtypes = [C.POINTER(PPOConfig), C.POINTER(EngineOptions), C.c_int, C.c_int,
                                            C.POINTER(C.c_int)]
        opt = EngineOptions(device, 0, 1, kw.get("strategy", "colocated").encode(), None, 1,
                            int(kw.get("zero_stage", 0)), int(kw.get("train_micro_batch", 0)),
                            int(kw.get("micro_batches", 1)), 1, 1, 0.5, 1, (C.c_double * 4)(0, 0, 0, 0))
        best = C.c_int(0)
        check(L.rlhf_engine_max_batch(C.byref(cfg), C.byref(opt), int(cap), int(run_step), C.byref(best)))
        return best.value

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        check(lib().rlhf_nccl_unique_id(buf))
        return bytes(buf)

    def step(self, prompts: np.ndarray | None = None) -> dict:
        rep = StepReport()
        p = None
        if prompts is not None:
            prompts = np.ascontiguousarray(prompts, dtype=np.int32)
            p = prompts.ctypes.data_as(C.POINTER(C.c_int32))
        check(lib().rlhf_engine_step(self._h, p, C.byref(rep)))
        return {"step_seconds": rep.step_seconds, "throughput_samples_per_sec": rep.throughput_samples_per_sec,
                "per_stage_seconds": dict(zip(STAGES, list(rep.stage_seconds))),
                "decode_seconds": rep.decode_seconds, "prefill_seconds": rep.prefill_seconds,
                "comm_bytes_total": rep.comm_bytes_total, "actor_loss": rep.actor_loss,
                "critic_loss": rep.critic_loss, "gpu_launches": rep.gpu_launches, "mean_score": rep.mean_score,
                "mean_kl": rep.mean_kl, "busy_seconds": rep.busy_seconds, "bubble_fraction": rep.bubble_fraction,
                "comm_seconds": rep.comm_seconds, "mem_peak_bytes": rep.mem_peak_bytes,
                "busiest_stage": STAGES[rep.busiest_stage], "n_events": rep.n_events, "feasible": bool(rep.feasible)}

    def events(self) -> list[dict]:
        """Measured intervals of the last step (SimEvent fields; seconds from the step start)."""
        L = lib()
        L.rlhf_engine_events.argtypes = [C.c_void_p, C.POINTER(Event), C.c_int]
        n = L.rlhf_engine_events(self._h, None, 0)
        buf = (Event * max(1, n))()
        n = L.rlhf_engine_events(self._h, buf, n)
        return [{"task": e.task, "kind": EVENT_KINDS.get(e.kind, str(e.kind)), "model": MODELS[e.model],
                 "micro_batch": e.micro_batch, "rollout": e.rollout, "epoch": e.epoch, "lane": e.lane,
                 "comm_op": e.comm_op, "stage": STAGES[e.stage], "start": e.start, "end": e.end} for e in buf[:n]]

    @property
    def generation_rows(self) -> int:
        """Sequences each Generation task of this rank decodes (0: the rank does not generate)."""
        S = self._cfg.prompt_len + self._cfg.gen_len
        return lib().rlhf_engine_tensor_bytes(self._h, b"pred") // (4 * S)

    @property
    def stream_handle(self) -> int:
        """cudaStream_t the engine launches on (for CUDA-event timing)."""
        return lib().rlhf_engine_stream(self._h)

    def read(self, name: str) -> np.ndarray:
        L = lib()
        nbytes = L.rlhf_engine_tensor_bytes(self._h, name.encode())
        if nbytes == 0:
            raise KeyError(name)
        dt = _DTYPES.get(name, np.float32)
        out = np.empty(nbytes // np.dtype(dt).itemsize, dtype=dt)
        check(L.rlhf_engine_read(self._h, name.encode(), out.ctypes.data_as(C.c_void_p), nbytes))
        R, S = self._cfg.gen_len, self._cfg.prompt_len + self._cfg.gen_len
        rows = L.rlhf_engine_tensor_bytes(self._h, b"sample_ids") // 4  # experience rows held by this rank
        if name in ("sample_ids", "score"):
            return out
        if out.size == rows * R and "params" not in name and "grad" not in name and "master" not in name:
            return out.reshape(rows, R)
        if name in ("pred", "margin"):
            return out.reshape(-1, S)
        if out.size == rows * S and name == "tokens":
            return out.reshape(rows, S)
        return out

    def greedy_check(self, tokens: np.ndarray):
        """Teacher-forced decode of `tokens` [B, S] (B = sequences per Generation task)."""
        R, S = self._cfg.gen_len, self._cfg.prompt_len + self._cfg.gen_len
        B = lib().rlhf_engine_tensor_bytes(self._h, b"pred") // (4 * S)
        tokens = np.ascontiguousarray(tokens, dtype=np.int32)
        pred = np.zeros((B, R), np.int32)
        margin = np.zeros((B, R), np.float32)
        check(lib().rlhf_engine_greedy_check(self._h, tokens.ctypes.data_as(C.POINTER(C.c_int32)),
                                             pred.ctypes.data_as(C.POINTER(C.c_int32)),
                                             margin.ctypes.data_as(C.POINTER(C.c_float))))
        return pred, margin

    def close(self):
        if getattr(self, "_h", None):
            lib().rlhf_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
