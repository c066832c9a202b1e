#!/bin/bash
# Round-2 (second session) evidence on one B200, run under gpurun: final c2 / c3 bench lines,
# the decode LM-head launches of one c2 step (one CTA per SM, balanced grid) and one
# `--set full` capture of it.  Outputs under gpurun_out/r2b_*.
cd "$(dirname "$0")/.."
O=gpurun_out
python bench.py --steps 20 --warmup 3 > $O/r2b_bench_c2_n1.json 2> $O/r2b_bench_c2_n1.err || exit 1
python bench.py --steps 5 --warmup 3 --workload c3 > $O/r2b_bench_c3_n1.json 2> $O/r2b_bench_c3_n1.err || exit 1
# every LM-head / merge launch of steps 1-2 (prefill + 255 decode steps each)
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"gemm_sm100_kernel|argmax_tiles" -c 600 --csv --log-file $O/r2b_lmhead_launches.csv \
    python tools/one_step.py --workload c2 --steps 2 > $O/r2b_ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_sm100_kernel \
    -s 100 -c 1 -o $O/r2b_lmhead_full python tools/one_step.py --workload c2 --steps 2 > $O/r2b_ncu_full.log 2>&1
ls -la $O/r2b_* > $O/r2b_done.txt
