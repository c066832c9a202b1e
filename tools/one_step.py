"""Profiling driver: build the c2 (or c1) engine and run one PPO step.

    python tools/one_step.py [--workload c2] [--steps 1] [--no-graph]
Used under `ncu` to collect per-kernel launch lists (profiles/).
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2312_11819_b200.capi import make_config  # noqa: E402
from paper_2312_11819_b200.engine import Engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c2")
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--no-graph", action="store_true")
ap.add_argument("--graph-mode", type=int, default=1, help="1: graph + PDL, 2: graph without PDL")
a = ap.parse_args()
cfg = {"c2": lambda: make_config("opt-125m", "opt-125m", 32, 256, 256),
       "c3": lambda: make_config("opt-1.3b", "opt-350m", 16, 256, 256),
       "c1": lambda: make_config("tiny", "tiny", 4, 16, 16),
       "c4-llama1b": lambda: make_config("llama-1b", "llama-1b", 16, 256, 256)}[a.workload]()
eng = Engine(cfg, cuda_graph=0 if a.no_graph else a.graph_mode)
for _ in range(a.steps):
    rep = eng.step()
    print({k: (round(v * 1e3, 2) if isinstance(v, float) else v) for k, v in rep.items() if k != "per_stage_seconds"})
