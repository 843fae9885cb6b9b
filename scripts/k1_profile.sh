#!/bin/bash
# K1 evidence on the B200 box: DRAM bytes per launch of config 2's own launches (single-pass metrics)
# and one `ncu --set full` capture of K1 on the shortened config 2 (2^18 x 5 d, the same per-event
# mix; the second K1 launch = the hot-set variant the bench times).  usage: bash scripts/k1_profile.sh TAG
tag=${1:-k1}
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:"ssa_k1|ssa_tree_leaf" --csv \
  --log-file gpurun_out/traffic_config2_${tag}.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/traffic_config2_${tag}.log 2>&1; echo "traffic c2 rc=$?"
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:ssa_k1 --launch-skip 1 -c 1 -o gpurun_out/k1_${tag} \
  python bench.py --steps 1 --warmup 1 --n-per-gpu 262144 --t-end 5 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_k1_${tag}.log 2>&1; echo "ncu k1 rc=$?"
