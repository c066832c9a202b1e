#!/bin/bash
# Same-box A/B of environment settings on one library build, alternating, N rounds:
#   tools/ab_env.sh rounds "A=1" "A=2 B=3" ... [-- bench args]
cd "$(dirname "$0")/.."
R=$1; shift
envs=()
while [ $# -gt 0 ] && [ "$1" != "--" ]; do envs+=("$1"); shift; done
[ "$1" == "--" ] && shift
for r in $(seq 1 "$R"); do
  for e in "${envs[@]}"; do
    env $e timeout 300 python bench.py --steps 10 --warmup 3 "$@" 2>/dev/null | tail -1 | python -c "
import json, sys
d = json.loads(sys.stdin.read())
print('$e', round(d['value'], 2), round(d['roofline']['us_per_launch'], 1), {k: round(v * 1e3, 2) for k, v in d['split_seconds_per_step'].items()})"
  done
done
