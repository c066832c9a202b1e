#!/bin/bash
# Same-box A/B of two library builds (ab_libs/old.so vs ab_libs/new.so), alternating, N rounds:
#   tools/ab_lib.sh rounds [-- bench args]
cd "$(dirname "$0")/.."
R=$1; shift
[ "$1" == "--" ] && shift
LIB=paper_2312_11819_b200/lib/librlhf_b200.so
cp $LIB /tmp/ab_keep.so
for r in $(seq 1 "$R"); do
  for v in old new; do
    cp ab_libs/$v.so $LIB
    timeout 300 python bench.py --steps 10 --warmup 3 "$@" 2>/dev/null | tail -1 | python -c "
import json, sys
d = json.loads(sys.stdin.read())
print('$v', round(d['value'], 2), round(d['roofline']['us_per_launch'], 1), {k: round(v * 1e3, 2) for k, v in d['split_seconds_per_step'].items()})"
  done
done
cp /tmp/ab_keep.so $LIB
