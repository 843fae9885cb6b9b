python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu -k "reduction or chunk or ragged or shard or config2_bench or config1 or config0" > gpurun_out/pytest_k3.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_k3.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_k3.json 2>gpurun_out/bench_k3.err; echo "bench rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/bench_k3.json').read().strip().splitlines()[-1]); print(d['value'], d['roofline_reduce'])"
timeout 600 python bench.py --config 3 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_k3c3.json 2>gpurun_out/bench_k3c3.err; echo "bench c3 rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/bench_k3c3.json').read().strip().splitlines()[-1]); print(d['value'], d['roofline'].get('lsu_pipe'), d['roofline_reduce'])"
