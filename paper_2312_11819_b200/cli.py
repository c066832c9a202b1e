"""Command line over the planner / simulator (the reference CLI's subcommands).

    python -m paper_2312_11819_b200.cli simulate --config scenarios/c3_8xb200.json [--out report.json]
    python -m paper_2312_11819_b200.cli trace    --config ... --out trace.json   (chrome://tracing)
    python -m paper_2312_11819_b200.cli compare  --config ... [--format json|csv|table]
    python -m paper_2312_11819_b200.cli maxbatch|plan|search --config ...
    python -m paper_2312_11819_b200.cli calibrate --config calib.json   ({"scenario", "observations"})

Exit codes follow the reference (errors.hpp:8-22): 0 ok, 2 config error, 3 infeasible,
4 search cap.  Every command is one rlhf_sim_run() call into the C++ library.
"""
from __future__ import annotations

import argparse
import json
import re
import sys

from .capi import sim_run

COMMANDS = ("simulate", "trace", "compare", "maxbatch", "plan", "search", "calibrate")


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="flexrlhf-b200")
    ap.add_argument("command", choices=COMMANDS)
    ap.add_argument("--config", required=True)
    ap.add_argument("--out")
    ap.add_argument("--format", choices=("json", "csv", "table"), default="json")
    a = ap.parse_args(argv)
    with open(a.config) as f:
        text = f.read()
    try:
        res = sim_run(a.command, text)
    except RuntimeError as e:
        m = re.search(r"error (\d+)", str(e))
        print(str(e), file=sys.stderr)
        return int(m.group(1)) if m else 1
    if a.command == "compare" and a.format != "json":
        doc = res["csv" if a.format == "csv" else "table"]
    else:
        doc = json.dumps(res, indent=None if a.command == "trace" else 1)
    if a.out:
        with open(a.out, "w") as f:
            f.write(doc)
    else:
        print(doc)
    return 0


if __name__ == "__main__":
    sys.exit(main())
