#!/bin/bash
# 4-GPU evidence (run under `gpurun --gpus 4`): c2 Co-located (weak scaling, BASELINE configs[1])
# and the c3 pair (configs[2]: OPT-1.3B Actor/Ref + OPT-350m Critic/Reward, global batch 64)
# for every placement, one bench line each under gpurun_out/r2b_n4_*.
cd "$(dirname "$0")/.."
p=29810
run() {  # name, args...
  local name=$1; shift
  p=$((p + 1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $p \
    bench.py --gpus 4 --steps 5 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/r2b_n4_$name.json 2> gpurun_out/r2b_n4_$name.err
  tail -1 gpurun_out/r2b_n4_$name.json | cut -c1-100
}
run c2_colocated --strategy colocated
for S in colocated interleaving1 interleaving2 disaggregated; do
  run c3_$S --workload c3 --strategy $S --train-mb 8
done
