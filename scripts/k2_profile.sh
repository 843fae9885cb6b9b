#!/bin/bash
# K2 evidence on the B200 box (after the tests passed): DRAM bytes per launch of config 3's own launches
# (single-pass metrics) and one `ncu --set full` capture of the half-warp K2 on the shortened config 3.
#   usage: bash scripts/k2_profile.sh TAG
tag=${1:-k2}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:"ssa_k2|ssa_tree_leaf" --csv \
  --log-file gpurun_out/traffic_config3_${tag}.csv \
  python bench.py --config 3 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/traffic_config3_${tag}.log 2>&1; echo "traffic c3 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:ssa_k2 -c 1 -o gpurun_out/k2h_${tag} \
  python bench.py --config 3 --steps 1 --warmup 0 --n-per-gpu 262144 --t-end 2 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_${tag}.log 2>&1; echo "ncu rc=$?"
