#!/usr/bin/env python
"""Fit the planner's cost model to MEASURED B200 PPO steps and predict the placements at
8 GPUs (BASELINE.json configs[2]/[3]), which gpurun cannot reach (<= 4 GPUs per call).

The reference's calibrate() (costmodel.hpp:78-90) fits mfu_fwd/mfu_train to the
non-generation share and mfu_gen to the generation share of observed steps; here the
observations are bench.py lines measured by the engine (profiles/*.json): step seconds and
the generation share of the gen/fwd/train split.  Output: fitted constants, predicted vs
measured per observation, and each strategy predicted at 8 x B200.

    python tools/calibrate_b200.py > profiles/r2_calibration_b200.json
"""
from __future__ import annotations

import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2312_11819_b200.capi import ARCHS, make_arch, param_total, sim_run  # noqa: E402


def line(path):
    with open(path) as f:
        rows = [json.loads(x) for x in f if x.startswith("{")]
    return rows[-1] if rows else None


def params(name, scalar_head):
    return param_total(make_arch(name, 512, scalar_head)) / 1e9


# workload family -> (actor arch, critic arch, bench-line glob, per-GPU batch at 8 GPUs, zero level, train micro-batch)
FAMILIES = {
    "c2 (OPT-125m x4, 256+256)": ("opt-125m", "opt-125m", "r2b_bench_c2_n*.json|r2b_n4_c2_*.json", 32, 0),
    "c3 / c5 (OPT-1.3B / OPT-350m, prompt 256, response 128..1024)":
        ("opt-1.3b", "opt-350m", "r2b_bench_c3_n*.json|r2b_n4_c3_*.json|r2_sweeps/r2_sweep_c*.json", 8, 0),
    "c4 (LLaMA-7B x4, 256+256)": ("llama-7b", "llama-7b", "r1_bench_c4_llama7b_n4_colocated_*.json|r2_bench_c4_*.json", 32, 1),
}


def main():
    out = {}
    for fam, (actor, critic, pat, per_gpu, zero) in FAMILIES.items():
        sizes = {"actor": params(actor, 0), "critic": params(critic, 1), "ref": params(actor, 0),
                 "reward": params(critic, 1)}
        obs = []
        for path in sorted(sum((glob.glob(os.path.join(ROOT, "profiles", p)) for p in pat.split("|")), [])):
            d = line(path)
            if not d or "split_seconds_per_step" not in d:
                continue
            cfg = d["config"]
            step = d["ms_per_step"] / 1e3
            gen = d["split_seconds_per_step"]["generation"]
            # split placements report rank 0's split in older lines: keep the fraction only for
            # Co-located, where every rank runs every stage
            frac = gen / step if cfg.get("placement", "colocated") == "colocated" else -1
            obs.append({"strategy": {"name": cfg.get("placement", "colocated"), "zero_level": cfg.get("zero_stage", 0),
                                     "tp_gen": 1},
                        "devices": d["n_gpus"], "batch": cfg["global_batch"], "measured_step_seconds": step,
                        "prompt_len": cfg.get("prompt_len", 256), "gen_len": cfg.get("gen_len", 256),
                        "generation_fraction": frac, "source": os.path.basename(path)})
        if not obs:
            continue
        sources = [o.pop("source") for o in obs]
        scen = {"topology": {"b200_box": 8},
                "workload": {"sizes_B": sizes, "batch": per_gpu * 8, "prompt_len": 256, "gen_len": 256},
                "strategies": [{"name": s, "zero_level": zero, "tp_gen": 1, "batch": per_gpu * 8}
                               for s in ("colocated", "interleaving1", "interleaving2", "disaggregated")],
                "sim": {"allow_infeasible": True}}
        res = sim_run("calibrate", {"scenario": scen, "observations": obs})
        for o, src in zip(res["observations"], sources):
            o["source"] = src
            o["error"] = o["predicted_step_seconds"] / o["measured_step_seconds"] - 1
        out[fam] = res
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
