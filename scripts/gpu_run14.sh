python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build14.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest14.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest14.log
timeout 900 python bench.py > gpurun_out/bench14.json 2> gpurun_out/bench14.err; echo "bench rc=$?"; cat gpurun_out/bench14.json
timeout 900 python bench.py --workload sweep --n-per-gpu 65536 > gpurun_out/bench14_sweep.json 2> gpurun_out/bench14_sweep.err; echo "sweep rc=$?"; cat gpurun_out/bench14_sweep.json
