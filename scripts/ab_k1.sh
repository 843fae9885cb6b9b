#!/bin/bash
# A/B of K1 code-generation knobs on config 2 (run on the B200 box from the repo root):
#   bash scripts/ab_k1.sh TAG "knobs1" "knobs2" ...   (SSA_K1_GEN values; "" = default)
tag=$1; shift
for k in "$@"; do
  SSA_K1_GEN="$k" timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e \
    > gpurun_out/ab_${tag}_${k//[^a-z0-9]/_}.json 2> gpurun_out/ab_${tag}_${k//[^a-z0-9]/_}.err
  python - "$k" gpurun_out/ab_${tag}_${k//[^a-z0-9]/_}.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(f"K1GEN={sys.argv[1]!r}: {d['value']:.4e} events/s frac {d['roofline']['frac']:.4f} k1_ms {d['roofline']['kernel_ms']:.1f} sm {d['clocks']['sm_mhz']}")
except Exception as e:
    print(f"K1GEN={sys.argv[1]!r}: failed {e}")
PY
done
