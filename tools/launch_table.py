"""Per-kernel table of an ncu launch list (--metrics gpu__time_duration.sum[,dram__bytes_*] --csv).

    python tools/launch_table.py gpurun_out/r2p_launches_c2.csv [--split-decode]
ncu times are cold-cache and serialised: compare shares, not absolutes.
"""
import argparse
import collections
import csv
import io
import re

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--title", default="")
a = ap.parse_args()
lines = open(a.csv).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
k = collections.OrderedDict()
for r in rows:
    i = int(r["ID"])
    d = k.setdefault(i, {"name": r["Kernel Name"], "grid": r["Grid Size"]})
    d[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
DECODE = ("gemm_decode_kernel", "attn_decode_kernel", "argmax_tiles", "embed_ln", "add_int")


def short(n):
    n = re.sub(r"\(CUtensorMap.*|\(const .*|\(float.*|\(int.*|\(unsigned.*|\(uint.*", "", n)
    return n.replace("void ", "").replace("rlhf::", "")


groups = {"decode step kernels": collections.defaultdict(lambda: [0, 0.0, 0.0]),
          "prefill / forward / training kernels": collections.defaultdict(lambda: [0, 0.0, 0.0])}
for d in k.values():
    s = short(d["name"])
    dec = any(x in s for x in DECODE) or (s.startswith("layernorm_kernel") and int(d["grid"].strip("()").split(",")[0]) <= 8) \
        or ("gemm_sm100_kernel<32, 1>" in s)
    g = groups["decode step kernels" if dec else "prefill / forward / training kernels"][s]
    g[0] += 1
    g[1] += d.get("gpu__time_duration.sum", 0) * 1e-3
    g[2] += (d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)) / 1e6
print(f"## {a.title}\n")
for gname, g in groups.items():
    tot = sum(v[1] for v in g.values())
    print(f"### {gname}: {sum(v[0] for v in g.values())} launches, {tot / 1e3:.3f} ms kernel time\n")
    print("| kernel | launches | time ms | share | avg us | DRAM MB | GB/s while running |")
    print("|---|---|---|---|---|---|---|")
    for s, (n, t, mb) in sorted(g.items(), key=lambda x: -x[1][1])[:18]:
        print(f"| {s[:70]} | {n} | {t / 1e3:.3f} | {100 * t / tot:.1f}% | {t / n:.1f} | {mb:.1f} | {mb / t * 1e3 if t else 0:.0f} |")
    print()
