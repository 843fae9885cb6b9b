#!/bin/bash
# A/B of half-warp K2 code-generation knobs on config 3 (run on the B200 box): bash scripts/ab_k2.sh TAG "knobs"...
tag=$1; shift
for k in "$@"; do
  SSA_K2_GEN="$k" timeout 600 python bench.py --config 3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e \
    > gpurun_out/abk2_${tag}_${k//[^a-z0-9]/_}.json 2> gpurun_out/abk2_${tag}_${k//[^a-z0-9]/_}.err
  python - "$k" gpurun_out/abk2_${tag}_${k//[^a-z0-9]/_}.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(f"K2GEN={sys.argv[1]!r}: {d['value']:.4e} events/s K2 {d['roofline']['kernel_ms']:.1f} ms")
except Exception as e:
    print(f"K2GEN={sys.argv[1]!r}: failed {e}")
PY
done
