python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build21.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/pytest21.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest21.log
for b in 2 3 4; do timeout 600 python bench.py --config 3 --path 3 --steps 1 --warmup 1 --n-per-gpu 262144 --no-cpu-baseline --no-e2e --blocks-per-sm $b 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('HALF bps=$b', '%.4g ev/s' % d['value'], 'ms=%.1f' % d['roofline']['kernel_ms'])"; done
