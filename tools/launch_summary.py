"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of one PPO step.

    python tools/launch_summary.py gpurun_out/launches_c2_r1.csv [--md out.md]

Phases are located by the decode position-counter kernel (add_int_kernel):
prefill = before the first one, decode = up to the last one, rest = forward + train.
ncu times are cold-cache and serialised: compare shares, not absolutes.
"""
import argparse
import collections
import csv
import io
import re


def load(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    out = []
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        short = re.sub(r"\(.*", "", name)
        m = re.search(r"gemm_sm100_kernel<(\d+)>", name)
        if m:
            short = f"gemm_sm100_kernel<BN={m.group(1)}>"
        out.append((int(r["ID"]), short, r["Grid Size"], float(r["Metric Value"]) * 1e-3))  # us
    return out


def summarise(rows):
    adds = [i for i, (_, n, _, _) in enumerate(rows) if n.startswith("add_int")]
    first, last = (adds[0], adds[-1]) if adds else (0, 0)
    phases = {"prefill": rows[:first], "decode": rows[first:last + 1], "forward+train": rows[last + 1:]}
    total = sum(r[3] for r in rows)
    rep = [f"total kernel time {total / 1e3:.1f} ms over {len(rows)} launches"]
    for ph, rs in phases.items():
        t = sum(r[3] for r in rs)
        rep.append(f"\n## {ph}: {t / 1e3:.1f} ms ({100 * t / total:.1f}%), {len(rs)} launches")
        agg = collections.defaultdict(lambda: [0.0, 0])
        for _, n, g, us in rs:
            agg[n][0] += us
            agg[n][1] += 1
        rep.append("| kernel | launches | total ms | share of phase | avg us |")
        rep.append("|---|---|---|---|---|")
        for n, (us, c) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:14]:
            rep.append(f"| {n} | {c} | {us / 1e3:.2f} | {100 * us / max(t, 1e-9):.1f}% | {us / c:.1f} |")
    return "\n".join(rep)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--md")
    a = ap.parse_args()
    s = summarise(load(a.csv))
    print(s)
    if a.md:
        open(a.md, "w").write(s + "\n")
