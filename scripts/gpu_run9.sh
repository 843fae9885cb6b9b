python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build9.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "config3 or edge_cases or numeric or config0 or config1_parity_ragged or hiv_short or invariance" > gpurun_out/pytest9.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest9.log
for b in 3 4 5; do timeout 600 python bench.py --config 3 --steps 1 --warmup 1 --n-per-gpu 262144 --no-cpu-baseline --no-e2e --blocks-per-sm $b 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('K2 bps=$b', '%.4g ev/s' % d['value'], 'k2_ms=%.1f' % d['roofline']['kernel_ms'])"; done
