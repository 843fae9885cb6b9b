#!/bin/bash
# union-time reduction: GPU parity, bench line and launch list (run on the B200 box from the repo root)
tag=${1:-x}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_union.py -q -x > gpurun_out/pytest_union_$tag.log 2>&1
echo pytest rc=$?; tail -3 gpurun_out/pytest_union_$tag.log
timeout 600 python bench.py --workload union --steps 2 --warmup 1 > gpurun_out/bench_union_$tag.json 2> gpurun_out/bench_union_$tag.err
tail -c 700 gpurun_out/bench_union_$tag.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/union_launches_$tag.csv \
  python bench.py --workload union --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_union_$tag.log 2>&1
echo ncu rc=$?
