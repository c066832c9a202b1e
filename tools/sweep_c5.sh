#!/bin/bash
# BASELINE.json configs[4]: response length 128..1024 at global batch 64, every placement, on
# the N GPUs of this gpurun call (2 or 4).  One bench line per (R, placement) under
# gpurun_out/r2_sweep_c5_n<N>_<placement>_r<R>.log.
cd "$(dirname "$0")/.."
N=${1:-2}
for R in 128 256 512 1024; do
  for S in colocated interleaving1 interleaving2 disaggregated; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $((29600 + R % 97)) bench.py --gpus $N --workload c5-r$R --strategy $S --batch $((64 / N)) \
      --train-mb 8 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_sweep_c5_n${N}_${S}_r$R.log 2>&1
  done
done
# BASELINE.json configs[2] at this box size: OPT-1.3B Actor/Ref + OPT-350m Critic/Reward, global
# batch 64, P = R = 256, every placement (the 8-GPU 4+4 split is predicted by the calibrated
# simulator, tools/calibrate_b200.py)
for S in colocated interleaving1 interleaving2 disaggregated; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 29650 bench.py --gpus $N --workload c3 --strategy $S --batch $((64 / N)) --train-mb 8 \
    --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_sweep_c3_n${N}_${S}.log 2>&1
done
