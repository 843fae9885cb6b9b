python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build20.log 2>&1
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/pytest20.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest20.log
timeout 900 python bench.py > gpurun_out/bench20.json 2> gpurun_out/bench20.err; echo "bench rc=$?"; cat gpurun_out/bench20.json
timeout 900 python bench.py --workload trajectories --steps 2 --warmup 1 > gpurun_out/bench20_traj.json 2>gpurun_out/bench20_traj.err; echo "traj rc=$?"; cat gpurun_out/bench20_traj.json
timeout 900 python bench.py --workload union --steps 2 --warmup 1 > gpurun_out/bench20_union.json 2>gpurun_out/bench20_union.err; echo "union rc=$?"; cat gpurun_out/bench20_union.json
timeout 900 python bench.py --config 3 --no-cpu-baseline > gpurun_out/bench20_c3.json 2>gpurun_out/bench20_c3.err; echo "c3 rc=$?"; cat gpurun_out/bench20_c3.json
timeout 600 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench20_ref.json 2>gpurun_out/bench20_ref.err; echo "ref rc=$?"; cat gpurun_out/bench20_ref.json
