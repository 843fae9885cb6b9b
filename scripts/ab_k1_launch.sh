#!/bin/bash
# A/B of the K1 launch shape on config 2 (run on the B200 box from the repo root):
#   bash scripts/ab_k1_launch.sh TAG "block:bps" ...   (0:0 = the default 128 x 4)
tag=$1; shift
for k in "$@"; do
  b=${k%%:*}; m=${k##*:}
  timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --block $b --blocks-per-sm $m \
    > gpurun_out/abk1_${tag}_${b}_${m}.json 2> gpurun_out/abk1_${tag}_${b}_${m}.err
  python - "$k" gpurun_out/abk1_${tag}_${b}_${m}.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(f"k1 block:bps={sys.argv[1]}: {d['value']:.4e} events/s frac {d['roofline']['frac']:.4f} k1_ms {d['roofline']['kernel_ms']:.1f} sm {d['clocks']['sm_mhz']}")
except Exception as e:
    print(f"k1 block:bps={sys.argv[1]}: failed {e}")
PY
done
