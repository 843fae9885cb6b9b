python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build16.log 2>&1
timeout 900 python bench.py --workload union --steps 2 --warmup 1 > gpurun_out/bench16_union.json 2> gpurun_out/bench16_union.err; echo "union rc=$?"; cat gpurun_out/bench16_union.json; tail -3 gpurun_out/bench16_union.err
timeout 900 python bench.py --workload sweep > gpurun_out/bench16_sweep.json 2> gpurun_out/bench16_sweep.err; echo "sweep rc=$?"; cat gpurun_out/bench16_sweep.json
timeout 900 python bench.py --variant B --no-cpu-baseline --no-e2e --steps 2 > gpurun_out/bench16_varB.json 2> gpurun_out/bench16_varB.err; echo "varB rc=$?"; cat gpurun_out/bench16_varB.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches16_union.csv python bench.py --workload union --steps 1 --warmup 1 > gpurun_out/ncu16.log 2>&1; echo "ncu rc=$?"
