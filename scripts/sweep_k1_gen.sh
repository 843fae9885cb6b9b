#!/bin/bash
# K1 code-generation variant sweep (SSA_K1_GEN x blocks-per-sm): quick parity
# subset per variant, then a shortened config-2 bench (same per-event mix).
# usage: bash scripts/sweep_k1_gen.sh "sel=f64,x=reg sel=i64,x=smem ..." "4 5 6"
VARIANTS=${1:-"sel=f64,x=reg"}
BPS=${2:-"4"}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/sweep_build.log 2>&1
for v in $VARIANTS; do
  SSA_K1_GEN=$v timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu \
    -k "config0_full_parity or config1_parity_ragged or hiv_short_horizon or hiv_full_horizon_sample or edge_cases or numeric_error or overflow" \
    > gpurun_out/sweep_pytest_${v//[=,]/_}.log 2>&1
  echo "PARITY $v rc=$? $(tail -1 gpurun_out/sweep_pytest_${v//[=,]/_}.log)"
  for b in $BPS; do
    SSA_K1_GEN=$v timeout 300 python bench.py --steps 2 --warmup 2 --n-per-gpu 262144 --t-end 5 \
      --no-cpu-baseline --no-e2e --blocks-per-sm $b 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('BENCH', '$v', 'bps=$b', '%.4g ev/s' % d['value'], 'k1_ms=%.1f' % d['roofline']['kernel_ms'], 'frac=%.3f' % d['roofline']['frac'], 'mhz=%s' % d['clocks']['sm_mhz'])"
  done
done
