#!/bin/bash
# A/B two builds of the engine library on the same box (noise between boxes is larger than
# most single-kernel changes): lib/ab/base.so vs lib/ab/new.so, alternating, N rounds.
#   tools/ab_bench.sh [rounds] [bench args...]
cd "$(dirname "$0")/.."
R=${1:-2}; shift
L=paper_2312_11819_b200/lib
for r in $(seq 1 "$R"); do
  for v in base new; do
    cp $L/ab/$v.so $L/librlhf_b200.so
    timeout 300 python bench.py --steps 10 --warmup 3 "$@" 2>/dev/null | tail -1 | python -c "
import json, sys
d = json.loads(sys.stdin.read())
print('$v', round(d['value'], 2), round(d['roofline']['us_per_launch'], 1), {k: round(v * 1e3, 2) for k, v in d['split_seconds_per_step'].items()})"
  done
done
cp $L/ab/new.so $L/librlhf_b200.so
