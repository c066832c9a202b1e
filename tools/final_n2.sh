#!/bin/bash
# 2-GPU evidence (run under `gpurun --gpus 2`): the multi-GPU pytest suite and the c2 placements
# (BASELINE.json configs[1] at N = 2), one bench line each under gpurun_out/r2b_*.
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -x -q > gpurun_out/r2b_pytest_gpu2_multi.log 2>&1
tail -2 gpurun_out/r2b_pytest_gpu2_multi.log
p=29710
for S in colocated interleaving1 interleaving2 disaggregated; do
  p=$((p + 1))
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $p \
    bench.py --gpus 2 --strategy $S --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2b_bench_c2_n2_$S.json 2>gpurun_out/r2b_bench_c2_n2_$S.err
  tail -1 gpurun_out/r2b_bench_c2_n2_$S.json | cut -c1-120
done
