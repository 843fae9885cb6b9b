#!/bin/bash
# A/B of the K1 tail-compaction threshold on config 2 (run on the B200 box): bash scripts/ab_tail.sh TAG N...
tag=$1; shift
for k in "$@"; do
  timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --tail-lanes $k \
    > gpurun_out/abt_${tag}_${k}.json 2> gpurun_out/abt_${tag}_${k}.err
  python - "$k" gpurun_out/abt_${tag}_${k}.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(f"tail_lanes={sys.argv[1]}: {d['value']:.4e} events/s frac {d['roofline']['frac']:.4f} k1_ms {d['roofline']['kernel_ms']:.1f} launches {d['gpu_launches']}")
except Exception as e:
    print(f"tail_lanes={sys.argv[1]}: failed {e}")
PY
done
