#!/bin/bash
# Profiling pass (run on the B200 box through gpurun from the repo root, after gpu_check.sh passed):
#   1. pipe_peaks: measured per-SM issue rates of DADD/DMUL/DFMA/FFMA/IADD3/IMAD (the FP64 pipe rate
#      SURVEY.md §8(d) asks to measure before quoting pipe fractions);
#   2. DRAM traffic per launch of the bench's own launches at full size (config 2: K1 + K3;
#      config 3: K2 + K3) -- a single-pass metric collection, for the roofline's `traffic`;
#   3. `ncu --set full` of K1 on the shortened workload (same per-event mix, N/1 x 5 d).
# Outputs land in gpurun_out/.
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/pipe_peaks scripts/pipe_peaks.cu && \
  /tmp/pipe_peaks > gpurun_out/pipe_peaks.txt 2>&1; cat gpurun_out/pipe_peaks.txt
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:"ssa_k1|ssa_tree_leaf" --csv \
  --log-file gpurun_out/traffic_config2.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/traffic_config2.log 2>&1; echo "traffic c2 rc=$?"
timeout 900 ncu --metrics $M --clock-control none -k regex:"ssa_k2|ssa_tree_leaf" --csv \
  --log-file gpurun_out/traffic_config3.csv \
  python bench.py --config 3 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/traffic_config3.log 2>&1; echo "traffic c3 rc=$?"
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:ssa_k1 -c 1 -o gpurun_out/k1_hiv_full \
  python bench.py --steps 1 --warmup 0 --n-per-gpu 262144 --t-end 5 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_k1.log 2>&1; echo "ncu k1 rc=$?"
