#!/bin/bash
# Round-2 ncu evidence on one B200 (run under gpurun): launch list of one c2 PPO step and
# `--set full` captures of the kernels the c2 step lives on.  Outputs under gpurun_out/r2p_*.
cd "$(dirname "$0")/.."
O=gpurun_out
python tools/one_step.py --workload c2 --steps 2 > $O/r2p_plain.log 2>&1 || exit 1
python tools/ffn_gemm_once.py > $O/r2p_ffn_plain.log 2>&1 || exit 1
# every launch of step 2 (step 1 warms up: ~23.5k launches per c2 step)
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -s 23600 -c 25000 --csv --log-file $O/r2p_launches_c2.csv python tools/one_step.py --workload c2 --steps 2 \
    > $O/r2p_ncu_launches.log 2>&1
# the FFN up-projection GEMM at the bench's roofline shape (launch 4 of 5)
ncu --set full --clock-control none --import-source on -k regex:gemm_pair -s 4 -c 1 -o $O/r2p_ffn_pair \
    python tools/ffn_gemm_once.py > $O/r2p_ncu_ffn.log 2>&1
for spec in "attn_fwd_kernel:40:1" "adamw_kernel:0:2" "gemm_decode_kernel:900:4" "attn_decode_kernel:300:1" \
            "lse_merge_kernel:0:1" "gemm_pair_kernel:40:2" "layernorm_bwd:0:1" "norm_bwd:0:1"; do
  IFS=: read k s c <<< "$spec"
  ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c $c -o $O/r2p_$k \
      python tools/one_step.py --workload c2 --steps 1 > $O/r2p_ncu_$k.log 2>&1
done
ls -la $O/r2p_* > $O/r2p_done.txt
