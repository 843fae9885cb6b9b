python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build6.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu6.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu6.log
timeout 900 python bench.py > gpurun_out/bench6.json 2> gpurun_out/bench6.err; echo "bench rc=$?"; cat gpurun_out/bench6.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches6.csv python bench.py --no-cpu-baseline > gpurun_out/ncu_launch6.log 2>&1; echo "ncu launches rc=$?"
timeout 900 python bench.py --config 3 --no-cpu-baseline > gpurun_out/bench6_c3.json 2> gpurun_out/bench6_c3.err; echo "bench c3 rc=$?"; cat gpurun_out/bench6_c3.json
