python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build3.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu3.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu3.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo "bench rc=$?"; cat gpurun_out/bench3.json
timeout 900 ncu --set full --import-source on --clock-control none -k regex:ssa_tree_leaf -c 1 -o gpurun_out/k3_full python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_k3.log 2>&1; echo "ncu rc=$?"
