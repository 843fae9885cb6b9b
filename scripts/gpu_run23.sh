python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build23.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "config3 or edge or trimolecular or gated or config0" > gpurun_out/pytest23.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest23.log
for cfg in "256 3" "256 2" "384 2" "512 2" "512 1" "128 6"; do set -- $cfg; timeout 600 python bench.py --config 3 --path 3 --steps 1 --warmup 1 --n-per-gpu 262144 --no-cpu-baseline --no-e2e --block $1 --blocks-per-sm $2 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('HALF block=$1 bps=$2', '%.4g ev/s' % d['value'], 'ms=%.1f' % d['roofline']['kernel_ms'])"; done
for cfg in "256 4" "256 3" "512 2"; do set -- $cfg; timeout 600 python bench.py --config 3 --path 2 --steps 1 --warmup 1 --n-per-gpu 262144 --no-cpu-baseline --no-e2e --block $1 --blocks-per-sm $2 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('WARP block=$1 bps=$2', '%.4g ev/s' % d['value'], 'ms=%.1f' % d['roofline']['kernel_ms'])"; done
for b in 4 5; do timeout 600 python bench.py --steps 1 --warmup 2 --n-per-gpu 262144 --t-end 10 --no-cpu-baseline --no-e2e --blocks-per-sm $b 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('K1 bps=$b', '%.4g ev/s' % d['value'], 'ms=%.1f' % d['roofline']['kernel_ms'])"; done
