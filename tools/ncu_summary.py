"""Summarise an `ncu --set full` report (.ncu-rep) into a markdown table for profiles/.

    python tools/ncu_summary.py gpurun_out/x.ncu-rep --title "..." >> profiles/r1_ncu_full.md
"""
import argparse
import csv
import io
import subprocess

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "L2 Hit Rate",
        "L1/TEX Hit Rate", "Issued Ipc Active", "No Eligible", "Warp Cycles Per Issued Instruction",
        "Registers Per Thread", "Grid Size", "Block Size", "Cluster Size", "Dynamic Shared Memory Per Block",
        "Achieved Occupancy"]
RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum"]


def ncu(rep, page):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--title", default="")
    a = ap.parse_args()
    rows = ncu(a.rep, "details")
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    print(f"## {a.title}\n\nkernel: `{rows[1][ix['Kernel Name']][:120]}`\n")
    print("| section | metric | unit | value |\n|---|---|---|---|")
    seen = set()
    for r in rows[1:]:
        n = r[ix["Metric Name"]]
        if n in WANT and n not in seen:
            seen.add(n)
            print(f"| {r[ix['Section Name']]} | {n} | {r[ix['Metric Unit']]} | {r[ix['Metric Value']]} |")
    raw = ncu(a.rep, "raw")
    h, u, v = raw[0], raw[1], raw[2]
    for name in RAW:
        if name in h:
            k = h.index(name)
            print(f"| raw | {name} | {u[k]} | {v[k]} |")
    print()


if __name__ == "__main__":
    main()
