"""Probe: do two half-batch PPO steps on two host threads (two engines, two streams) overlap on
one B200?  Compares wall time of K steps of one B=32 engine against two B=16 engines stepped
concurrently (ctypes releases the GIL inside rlhf_engine_step).  Also times one B=16 engine
alone.  Answers whether splitting the latency-bound decode chain across concurrent streams pays.

    python tools/concurrency_probe.py [--steps 5]
"""
import argparse
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2312_11819_b200.capi import make_config  # noqa: E402
from paper_2312_11819_b200.engine import Engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=5)
a = ap.parse_args()


def run(engines, steps):
    reps = [[] for _ in engines]

    def work(i):
        for _ in range(steps):
            reps[i].append(engines[i].step())

    ths = [threading.Thread(target=work, args=(i,)) for i in range(len(engines))]
    t0 = time.perf_counter()
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    return time.perf_counter() - t0, reps


def fmt(r):
    s = r["per_stage_seconds"]
    return {k: round(v * 1e3, 1) for k, v in s.items() if v}, round(r["decode_seconds"] * 1e3, 1)


one = Engine(make_config("opt-125m", "opt-125m", 32, 256, 256))
run([one], 2)
t, reps = run([one], a.steps)
print("B=32 x1 engine: %.1f samples/s  step %.1f ms  %s" % (32 * a.steps / t, t / a.steps * 1e3, fmt(reps[0][-1])))
one.close()

h = [Engine(make_config("opt-125m", "opt-125m", 16, 256, 256)) for _ in range(2)]
run(h[:1], 2)
t, reps = run(h[:1], a.steps)
print("B=16 x1 engine: %.1f samples/s  step %.1f ms  %s" % (16 * a.steps / t, t / a.steps * 1e3, fmt(reps[0][-1])))
run(h, 2)
t, reps = run(h, a.steps)
print("B=16 x2 engines concurrent: %.1f samples/s  wall/step %.1f ms  %s | %s" %
      (32 * a.steps / t, t / a.steps * 1e3, fmt(reps[0][-1]), fmt(reps[1][-1])))
