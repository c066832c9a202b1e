"""ctypes wrapper of the CPU oracle (oracle/_build/libppo_oracle.so).  TEST ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2312_11819_b200.capi import PPOConfig, param_total

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
ORACLE_SO = os.path.join(ORACLE_DIR, "_build", "libppo_oracle.so")
REF_SO = os.path.join(ORACLE_DIR, "_ref", "librlhfsim_ref.so")


class Outputs(C.Structure):
    _fields_ = [("tokens", C.c_void_p), ("greedy_margin", C.c_void_p), ("logp_old", C.c_void_p),
                ("logp_ref", C.c_void_p), ("values", C.c_void_p), ("score", C.c_void_p),
                ("rewards", C.c_void_p), ("advantages", C.c_void_p), ("returns", C.c_void_p),
                ("logp_new", C.c_void_p), ("values_new", C.c_void_p), ("actor_loss", C.c_double),
                ("critic_loss", C.c_double), ("actor_grad", C.c_void_p), ("critic_grad", C.c_void_p),
                ("actor_master", C.c_void_p), ("critic_master", C.c_void_p)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            subprocess.check_call(["make", "-s", "-C", ORACLE_DIR])
        _lib = C.CDLL(ORACLE_SO)
        _lib.oracle_ppo_step.argtypes = [C.POINTER(PPOConfig), C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                                         C.POINTER(Outputs)]
        _lib.oracle_ppo_step_epochs.argtypes = [C.POINTER(PPOConfig), C.c_int, C.c_void_p, C.c_void_p, C.c_int,
                                                C.c_int, C.POINTER(Outputs)]
        _lib.oracle_forward_hidden.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_int, C.c_int, C.c_int,
                                               C.c_void_p]
    return _lib


def ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def ppo_step(cfg: PPOConfig, tokens_in=None, stop_after=0, threads=0, want_grads=True, ppo_epochs=1):
    B, P, R = cfg.batch, cfg.prompt_len, cfg.gen_len
    S = P + R
    f = lambda *s: np.zeros(s, np.float32)
    o = dict(tokens=np.zeros((B, S), np.int32), greedy_margin=f(B, R), logp_old=f(B, R), logp_ref=f(B, R),
             values=f(B, R), score=f(B), rewards=f(B, R), advantages=f(B, R), returns=f(B, R),
             logp_new=f(B, R), values_new=f(B, R))
    if want_grads and stop_after == 0:
        na, nc = param_total(cfg.actor), param_total(cfg.critic)
        o.update(actor_grad=f(na), critic_grad=f(nc), actor_master=f(na), critic_master=f(nc))
    pred = np.zeros((B, R), np.int32)
    out = Outputs(**{k: ptr(v) for k, v in o.items()})
    tin = None if tokens_in is None else np.ascontiguousarray(tokens_in, np.int32)
    st = lib().oracle_ppo_step_epochs(C.byref(cfg), ppo_epochs, ptr(tin), ptr(pred), stop_after, threads, C.byref(out))
    if st != 0:
        raise RuntimeError(f"oracle_ppo_step failed: {st}")
    o["greedy_pred"] = pred
    o["actor_loss"], o["critic_loss"] = out.actor_loss, out.critic_loss
    return o
