#!/bin/bash
# Round-end GPU check (run on the B200 box through gpurun from the repo root):
#   build, every GPU parity test, smoke(), the default bench line (the driver's 20 steps / 5 warm-up),
#   the other workloads, the reference arm, and the ncu launch list of the default bench.
# Outputs land in gpurun_out/ (scratch); copy what is kept into profiles/.
#   usage: bash scripts/gpu_check.sh [quick]
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
cat gpurun_out/bench_default.json
[ "$1" = "quick" ] && exit 0
timeout 900 python bench.py --config 3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 900 python bench.py --workload sweep > gpurun_out/bench_sweep.json 2> gpurun_out/bench_sweep.err
timeout 900 python bench.py --workload union --steps 2 --warmup 1 > gpurun_out/bench_union.json 2> gpurun_out/bench_union.err
timeout 900 python bench.py --workload trajectories --steps 2 --warmup 1 > gpurun_out/bench_traj.json 2> gpurun_out/bench_traj.err
timeout 900 python bench.py --workload dump > gpurun_out/bench_dump.json 2> gpurun_out/bench_dump.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
tail -n1 gpurun_out/bench_c3.json gpurun_out/bench_sweep.json gpurun_out/bench_union.json gpurun_out/bench_traj.json gpurun_out/bench_dump.json gpurun_out/bench_ref.json
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --no-cpu-baseline --no-e2e > gpurun_out/ncu_launches.log 2>&1; echo "ncu rc=$?"
