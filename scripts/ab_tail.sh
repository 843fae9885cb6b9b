python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build24.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "hiv or config3_thread or config1 or config0 or edge or gated or trimolecular or invariance" > gpurun_out/pytest24.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest24.log
for g in tail=on tail=off; do SSA_K1_GEN=$g timeout 600 python bench.py --steps 2 --warmup 2 --n-per-gpu 262144 --t-end 10 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('K1 $g', '%.4g ev/s' % d['value'], 'ms=%.1f' % d['roofline']['kernel_ms'])"; done
for g in tail=on tail=off; do SSA_K1_GEN=$g timeout 600 python bench.py --config 1 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('K1 config1 $g', '%.4g ev/s' % d['value'], 'ms=%.1f' % d['roofline']['kernel_ms'])"; done
