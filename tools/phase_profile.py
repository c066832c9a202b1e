"""Aggregate an ncu launch list (gpu__time_duration + dram bytes) per kernel.

    python tools/phase_profile.py gpurun_out/launches_decode_step_r1.csv [--md out.md --title T]

ncu times are cold-cache and serialised: use the SHARES and the DRAM bytes.
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
    by = collections.defaultdict(dict)
    for r in rows:
        d = by[int(r["ID"])]
        d["name"] = re.sub(r"\(.*", "", r["Kernel Name"]).replace("void ", "")
        d["grid"] = r["Grid Size"]
        v = float(r["Metric Value"].replace(",", "")) if r["Metric Value"] else 0.0
        unit = r["Metric Unit"]
        if r["Metric Name"].startswith("dram__bytes"):
            v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        if r["Metric Name"] == "gpu__time_duration.sum":
            v *= {"ns": 1e-3, "us": 1, "usecond": 1, "ms": 1e3}.get(unit, 1e-3)
        d[r["Metric Name"]] = v
    return [by[i] for i in sorted(by)]


def summarise(rows, title):
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for d in rows:
        k = d["name"]
        agg[k][0] += 1
        agg[k][1] += d.get("gpu__time_duration.sum", 0.0)
        agg[k][2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    tot_t = sum(v[1] for v in agg.values())
    tot_b = sum(v[2] for v in agg.values())
    out = [f"## {title}", "", f"{len(rows)} launches, {tot_t / 1e3:.3f} ms kernel time (ncu, serialised, cold), "
           f"{tot_b / 1e6:.1f} MB DRAM traffic", "",
           "| kernel | launches | time ms | share | avg us | DRAM MB | GB/s while running |", "|---|---|---|---|---|---|---|"]
    for k, (c, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| {k} | {c} | {t / 1e3:.3f} | {100 * t / max(tot_t, 1e-9):.1f}% | {t / c:.1f} | {b / 1e6:.1f} | "
                   f"{b / max(t, 1e-9) / 1e3:.0f} |")
    return "\n".join(out), tot_t, tot_b


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--md")
    ap.add_argument("--title", default="launch list")
    a = ap.parse_args()
    s, _, _ = summarise(load(a.csv), a.title)
    print(s)
    if a.md:
        with open(a.md, "a") as f:
            f.write(s + "\n\n")
