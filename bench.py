#!/usr/bin/env python
"""bench.py — PPO samples/sec per RLHF step (gen/fwd/train split) on B200.

Metric (BASELINE.json): "PPO samples/sec per RLHF step (gen/fwd/train split) at
1/2/4/8 B200"; samples/sec = batch x rollout_nums / step_seconds
(/root/reference/SPEC.md:379).

Workload (N=1 default): BASELINE.json configs[1] — OPT-125m-shaped Actor/Ref +
Critic/Reward, prompt 256 + response 256, batch 32 per GPU, one full PPO
iteration per step (greedy generation, 4 teacher-forced forwards, GAE, Actor
and Critic forward+backward+AdamW), Co-located placement.  Weak scaling: at N
GPUs the global batch is 32*N (one Co-located data-parallel replica per GPU,
NCCL gradient all-reduce).  Random-init weights (seeded), synthetic prompts.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload c2|c1]

One JSON line on rank 0.  `value` = device-timed throughput with inputs already
in HBM (CUDA events on the engine stream, max over ranks); `e2e` = the same
metric through the C-ABI with host prompts copied in and losses copied out
inside the timed region.  `--impl reference` times the CPU oracle (the
reference has no numeric PPO path) on host cores, one sample per step.
"""
from __future__ import annotations

import argparse
import json

import numpy as np
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    "c2": dict(actor="opt-125m", critic="opt-125m", batch=32, prompt=256, gen=256,
               name="c2: OPT-125m-shaped Actor/Ref + Critic/Reward, batch 32/GPU, prompt 256 + response 256"),
    "c1": dict(actor="tiny", critic="tiny", batch=4, prompt=16, gen=16,
               name="c1: tiny decoder x4, batch 4/GPU, prompt 16 + response 16"),
    # c3 / c5 shapes (B=64 over 8 GPUs in the paper's setting; per-GPU 16 here)
    "c3": dict(actor="opt-1.3b", critic="opt-350m", batch=16, prompt=256, gen=256,
               name="c3: OPT-1.3B Actor/Ref + OPT-350m-shaped Critic/Reward, batch 16/GPU, prompt 256 + response 256"),
    # c4 (LLaMA-7B Actor/Critic, Disaggregated on 8 GPUs) needs ZeRO-3 sharding;
    # this is the LLaMA-family step at the largest shape that runs unsharded on one B200
    "c4-llama1b": dict(actor="llama-1b", critic="llama-1b", batch=16, prompt=256, gen=256,
                       name="c4 family study: LLaMA-shaped 1B (d 2048, 16 layers, head_dim 128, SwiGLU 5504, "
                            "V 32000) x4, batch 16/GPU, prompt 256 + response 256"),
    # c4 proper: LLaMA-7B-shaped Actor/Ref + Critic/Reward; needs >= 4 GPUs and ZeRO-1 (--zero 1);
    # the per-GPU batch is what fits next to the placement's resident models (--batch)
    "c4": dict(actor="llama-7b", critic="llama-7b", batch=8, prompt=256, gen=256,
               name="c4: LLaMA-7B-shaped Actor/Ref + Critic/Reward, prompt 256 + response 256"),
    "c5-r1024": dict(actor="opt-1.3b", critic="opt-350m", batch=16, prompt=256, gen=1024,
                     name="c5: OPT-1.3B/350m, batch 16/GPU, prompt 256 + response 1024"),
    # the rest of BASELINE.json configs[4]'s generation-heavy sweep (global batch 64 = --batch 64/N)
    **{f"c5-r{r}": dict(actor="opt-1.3b", critic="opt-350m", batch=16, prompt=256, gen=r,
                        name=f"c5: OPT-1.3B/350m, prompt 256 + response {r}") for r in (128, 256, 512)},
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], p.get("bf16_tflops_sustained", p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


class Clocks:
    """nvidia-smi clock/throttle sampling during the timed region (B200_PROFILING.md)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.path = tempfile.mktemp(suffix=".csv")
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def decode_bytes_per_step(a, B, P, R):
    """Algorithmic HBM bytes of one decode step (weights once + KV read), averaged over the R-1 steps.
    SURVEY.md §8(d): sum_t [2 P_w + Bg (P+t) 4 L d]."""
    d, L, V, ff = a.d_model, a.n_layers, a.vocab, a.d_ff
    nff = 3 if a.family == 1 else 2  # SwiGLU: gate, up, down
    p_w = L * (4 * d * d + nff * d * ff) + V * d  # matmul weights incl. the LM head
    kv = sum(4 * L * d * B * (P + s) for s in range(1, R))
    return (2.0 * p_w * (R - 1) + kv) / max(1, R - 1)


def cpu_oracle_sample(wl, threads=0):
    """Time the CPU oracle on one sample of the workload (all host threads)."""
    from paper_2312_11819_b200.capi import make_config
    from tests import oracle_lib
    cfg = make_config(wl["actor"], wl["critic"], 1, wl["prompt"], wl["gen"])
    t0 = time.perf_counter()
    oracle_lib.ppo_step(cfg, threads=threads, want_grads=False)
    return time.perf_counter() - t0


METRIC = "PPO samples/sec per RLHF step (gen/fwd/train split)"  # identical in both arms


def arm_config(args, wl, world):
    """The `config` object both arms print (the driver compares the arms on it)."""
    B, P, R = wl["batch"], wl["prompt"], wl["gen"]
    return {"workload": wl["name"], "placement": args.strategy, "global_batch": B * world * args.rollouts,
            "prompt_len": P, "gen_len": R, "parallelism": f"dp{world}", "zero_stage": args.zero,
            "train_micro_batch": args.train_mb, "micro_batches": args.micro_batches, "rollout_nums": args.rollouts,
            "ppo_epochs": args.epochs,
            "l2": "working set (4 models' weights + activations) >> 126 MB L2 every step"}


def reference_arm(args, wl, rank, world=1):
    """The reference's CPU path of the PPO step (the oracle port: the reference itself has no
    numeric path) on the host cores.  Each timed step is a bounded sample of the
    workload -- ONE of its samples through the full PPO step (generation, 4 forwards, GAE,
    Actor + Critic training) -- so K + W steps end in minutes; samples/s = samples / seconds,
    the same metric the GPU arm reports for the whole batch."""
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_oracle_sample(wl, cores)
    ts = [cpu_oracle_sample(wl, cores) for _ in range(args.steps)]
    total = sum(ts)
    v = args.steps / total
    sample = (f"1 of the {wl['batch']} samples per GPU of {wl['name']} per timed step: full PPO step "
              f"(oracle/ppo_oracle.cpp, fp32, {cores} threads)")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "samples/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32 (bf16-rounded operands)",
            "data": "synthetic (seeded random-init weights, uniform prompt ids)",
            "config": arm_config(args, wl, world), "sample": sample,
            "cpu_baseline": {"value": v, "unit": "samples/s", "cores": cores, "kind": "port", "sample": sample},
            "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def write_trace(path, per_rank_events):
    """Chrome trace of the measured step: one process per rank, threads = lanes (0 main
    compute, 1 side compute, 2 comm); names "<stage>:<model>:mb<i>" as emit_trace."""
    ev = []
    for rank, events in enumerate(per_rank_events):
        ev.append({"ph": "M", "name": "process_name", "pid": rank, "args": {"name": f"rank {rank} (B200)"}})
        for lane, name in enumerate(("compute", "compute (side)", "comm")):
            ev.append({"ph": "M", "name": "thread_name", "pid": rank, "tid": lane, "args": {"name": name}})
        for e in events:
            ev.append({"ph": "X", "pid": rank, "tid": e["lane"], "cat": e["kind"],
                       "name": f"{e['stage']}:{e['model']}:mb{e['micro_batch']}",
                       "ts": round(e["start"] * 1e6, 3), "dur": round((e["end"] - e["start"]) * 1e6, 3),
                       "args": {"task": e["task"], "rollout": e["rollout"], "epoch": e["epoch"]}})
    with open(path, "w") as f:
        json.dump({"displayTimeUnit": "ms", "traceEvents": ev}, f)


def profile_json(name):
    """Committed ncu-derived numbers (profiles/*.json) for the roofline `traffic` fields."""
    try:
        with open(os.path.join(ROOT, "profiles", name)) as f:
            return json.load(f)
    except Exception:
        return None


def gemm_roofline(a, B, S, tflops_peak):
    """Live CUDA-event timing of the dominant forward/backward GEMM shape of the workload
    (FFN up-projection, M = B*S tokens), through the C-ABI."""
    import torch
    from paper_2312_11819_b200 import ops
    M, N, K = B * S, a.d_ff * (2 if a.family == 1 else 1), a.d_model
    kname = ops.gemm_kernel_name(M, N, K)
    x = torch.randn(M, K, device="cuda").bfloat16()
    w = torch.randn(N, K, device="cuda").bfloat16()
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        ops.gemm(x, w, out=y, out_f32=False)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters = 20
    e0.record()
    for _ in range(iters):
        ops.gemm(x, w, out=y, out_f32=False)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3 / iters
    fl = 2.0 * M * N * K
    tr = profile_json("r2_gemm_traffic.json")
    ok = tr and tr.get("shape") == [M, N, K] and tr.get("kernel") == kname
    traffic = tr["dram_bytes_per_launch"] if ok else None
    return {"bound": "tensor", "kernel": f"{kname} (FFN up-proj, forward)", "shape": [M, N, K],
            "achieved": fl / t / 1e12, "peak": tflops_peak, "unit": "TFLOP/s", "frac": fl / t / 1e12 / tflops_peak,
            "traffic": traffic, "traffic_unit": "bytes/launch (ncu dram read+write of this kernel at this shape, profiles/r2_gemm_traffic.json)",
            "ms": t * 1e3}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--strategy", default="colocated")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--batch", type=int, default=0, help="per-GPU batch override (memory studies)")
    ap.add_argument("--train-mb", type=int, default=0, help="samples per TrainFB micro-batch (0: all)")
    ap.add_argument("--zero", type=int, default=0, choices=[0, 1, 2, 3], help="ZeRO stage of the trainable models")
    ap.add_argument("--micro-batches", type=int, default=1, help="LoopParams::micro_batches (task-DAG micro-batches)")
    ap.add_argument("--rollouts", type=int, default=1, help="LoopParams::rollout_nums")
    ap.add_argument("--epochs", type=int, default=1, help="LoopParams::ppo_epochs")
    ap.add_argument("--trace", default="", help="write a Chrome trace of the last step's measured events (all ranks)")
    args = ap.parse_args()
    wl = dict(WORKLOADS[args.workload])
    if args.batch:
        wl["batch"] = args.batch
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        return reference_arm(args, wl, rank, world)

    import torch
    import torch.distributed as dist
    from paper_2312_11819_b200.capi import make_config, prompt_tokens
    from paper_2312_11819_b200.engine import Engine

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    B, P, R = wl["batch"], wl["prompt"], wl["gen"]
    cfg = make_config(wl["actor"], wl["critic"], B, P, R, sample_offset=rank * B,
                      loss_denominator=float(B * world * R))
    nid = None
    if world > 1:
        obj = [Engine.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    eng = Engine(cfg, device=local, rank=rank, world_size=world, strategy=args.strategy, nccl_id=nid,
                 zero_stage=args.zero, train_micro_batch=args.train_mb, micro_batches=args.micro_batches,
                 rollout_nums=args.rollouts, ppo_epochs=args.epochs)
    # this rank's home prompts, rollout-major ([rollouts * B, P]; rollout r = global ids r*G + ...)
    prompts = np.concatenate([prompt_tokens(cfg.prompt_seed, B, P, cfg.actor.vocab, sample_offset=r * B * world + rank * B)
                              for r in range(args.rollouts)])

    for _ in range(args.warmup):
        eng.step(prompts)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = Clocks(local)
    if rank == 0:
        clocks.start()
    stream = torch.cuda.ExternalStream(eng.stream_handle)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    reps = [eng.step(prompts) for _ in range(args.steps)]
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop() if rank == 0 else None
    e2e_s = e0.elapsed_time(e1) / 1e3
    dev_s = sum(r["step_seconds"] for r in reps)
    free_b, total_b = torch.cuda.mem_get_info()
    # this rank's measured SimReport fields (per step): its own compute-lane stage attribution,
    # busy / bubble, and the sequences its Generation tasks decode
    gen_rows = eng.generation_rows
    mine = {"rank": rank, "stage": {k: sum(r["per_stage_seconds"][k] for r in reps) / args.steps
                                    for k in reps[0]["per_stage_seconds"]},
            "busy_s": sum(r["busy_seconds"] for r in reps) / args.steps,
            "bubble_fraction": sum(r["bubble_fraction"] for r in reps) / args.steps,
            "comm_s": sum(r["comm_seconds"] for r in reps) / args.steps,
            "decode_s": sum(r["decode_seconds"] for r in reps), "gen_rows": gen_rows,
            "launches": sum(r["gpu_launches"] for r in reps), "mem_gb": (total_b - free_b) / 1e9,
            "engine_mem_gb": reps[-1]["mem_peak_bytes"] / 1e9}
    events = eng.events() if args.trace else None
    ranks = [mine]
    if world > 1:
        t = torch.tensor([e2e_s, dev_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s, dev_s = t.tolist()
        ranks = [None] * world
        dist.all_gather_object(ranks, mine)
        if args.trace:
            evs = [None] * world
            dist.all_gather_object(evs, events)
            events = evs
    elif args.trace:
        events = [events]
    if rank != 0:
        dist.destroy_process_group()
        return 0
    if args.trace:
        write_trace(args.trace, events)
    launches = sum(r["launches"] for r in ranks)
    mem_gb = max(r["mem_gb"] for r in ranks)
    # stage split: each stage's seconds on the rank where it is longest (a rank's idle time
    # goes to the stage it waits for); the per-rank splits are reported beside it
    stage = {k: max(r["stage"][k] for r in ranks) for k in ranks[0]["stage"]}
    gen_rank = max(ranks, key=lambda r: (r["gen_rows"], r["decode_s"]))  # the generating rank(s)

    hbm, tf_burst, tf_sus, src = peaks()
    dbytes = decode_bytes_per_step(cfg.actor, gen_rank["gen_rows"], P, R)
    dec_s = gen_rank["decode_s"] / (args.rollouts * args.micro_batches)  # per Generation task
    dec_per_launch = dec_s / (args.steps * max(1, R - 1))
    tr = profile_json("r1_decode_traffic.json") if args.workload == "c2" else None
    roof_decode = {"bound": "hbm", "kernel": "decode step (CUDA graph: swap-AB tcgen05 GEMMs + decode attention)",
                   "achieved": dbytes / dec_per_launch / 1e9, "peak": hbm, "unit": "GB/s",
                   "frac": dbytes / dec_per_launch / 1e9 / hbm,
                   # ncu DRAM bytes of one decode step (profiles/r1_decode_traffic.json, measured at ctx
                   # ~265) scaled by its traffic/algorithmic ratio to this average-context step
                   "traffic": tr["traffic_over_algorithmic"] * dbytes if tr else None,
                   "traffic_ratio_measured": tr["traffic_over_algorithmic"] if tr else None,
                   "algorithmic_bytes_per_launch": dbytes, "us_per_launch": dec_per_launch * 1e6,
                   "peak_source": src}
    roof_gemm = gemm_roofline(cfg.actor, B, P + R, tf_burst)
    roof_gemm["peak_source"] = src + " (burst)"
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        t = cpu_oracle_sample(wl, cores)
        cpu = {"value": 1.0 / t, "unit": "samples/s", "cores": cores, "kind": "port",
               "sample": f"1 sample of {wl['name']}: full PPO step in oracle/ppo_oracle.cpp ({t:.1f} s)"}
    S = P + R
    samples = B * world * args.rollouts * args.steps
    line = {
        "metric": METRIC,
        "value": samples / dev_s, "unit": "samples/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * dev_s / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic (seeded random-init weights, uniform prompt ids)",
        "config": arm_config(args, wl, world),
        "split_seconds_per_step": stage,
        "split_fraction": {k: v / (dev_s / args.steps) for k, v in stage.items()},
        "split_by_rank": [{"rank": r["rank"], **{k: round(v, 6) for k, v in r["stage"].items()},
                           "busy_s": round(r["busy_s"], 6), "bubble_fraction": round(r["bubble_fraction"], 4),
                           "comm_s": round(r["comm_s"], 6), "generation_rows": r["gen_rows"],
                           "engine_mem_gb": round(r["engine_mem_gb"], 2)} for r in ranks],
        "e2e": {"value": samples / e2e_s, "unit": "samples/s",
                "h2d_bytes_per_step": B * args.rollouts * (P + R) * 4, "d2h_bytes_per_step": 16},
        "gpu_launches": launches,
        "roofline": roof_decode,
        "roofline_gemm": roof_gemm,
        "cpu_baseline": cpu,
        "clocks": clk,
        "losses": [reps[-1]["actor_loss"], reps[-1]["critic_loss"]],
        "hbm_used_gb_max_rank": mem_gb,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
