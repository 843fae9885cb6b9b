python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build4.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu4.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu4.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench4.json 2> gpurun_out/bench4.err; echo "bench rc=$?"; cat gpurun_out/bench4.json
timeout 900 ncu --set full --import-source on --clock-control none -k regex:ssa_k1 -c 1 -o gpurun_out/k1_r1b python bench.py --steps 1 --warmup 0 --n-per-gpu 262144 --t-end 5 --no-cpu-baseline --no-e2e > gpurun_out/ncu_k1.log 2>&1; echo "ncu k1 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:ssa_tree_leaf_full -c 1 -o gpurun_out/k3_r1b python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_k3b.log 2>&1; echo "ncu k3 rc=$?"
