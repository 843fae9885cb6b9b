#!/bin/bash
# One K2 (half-warp) iteration on the B200 box: build, the GPU tests that run the half-warp
# path, a config-3 bench line, and one `ncu --set full` capture of K2 on the shortened
# config-3 workload (2^18 trajectories x 2 time units).  usage: bash scripts/k2_iter.sh TAG [noncu]
tag=${1:-k2}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -x -q -m gpu -k "halfwarp or config3 or gated or trimolecular or mini_hiv or overflow or numeric or edge or ragged" \
  > gpurun_out/pytest_${tag}.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_${tag}.log
timeout 600 python bench.py --config 3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e \
  > gpurun_out/bench_c3_${tag}.json 2> gpurun_out/bench_c3_${tag}.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/bench_c3_${tag}.json
[ "$2" = "noncu" ] && exit 0
timeout 900 ncu --set full --import-source on --clock-control none -k regex:ssa_k2 -c 1 -o gpurun_out/k2h_${tag} \
  python bench.py --config 3 --steps 1 --warmup 0 --n-per-gpu 262144 --t-end 2 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_${tag}.log 2>&1; echo "ncu rc=$?"
