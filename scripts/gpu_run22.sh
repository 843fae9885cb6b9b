python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build22.log 2>&1
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/pytest22.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest22.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke22.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke22.log
timeout 900 python bench.py --config 3 --no-cpu-baseline > gpurun_out/bench22_c3.json 2>gpurun_out/bench22_c3.err; echo "c3 rc=$?"; cat gpurun_out/bench22_c3.json
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:ssa_k2 -c 1 -o gpurun_out/k2h_r1f python bench.py --config 3 --steps 1 --warmup 0 --n-per-gpu 65536 --t-end 2 --no-cpu-baseline --no-e2e > gpurun_out/ncu_k2h.log 2>&1; echo "ncu rc=$?"
