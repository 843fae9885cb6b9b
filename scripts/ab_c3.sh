#!/bin/bash
# A/B of the half-warp K2 launch shape on config 3 (run on the B200 box from the repo root):
#   bash scripts/ab_c3.sh TAG "block:bps" ...   ("0:0" = library default)
tag=$1; shift
for k in "$@"; do
  b=${k%%:*}; p=${k##*:}
  timeout 600 python bench.py --config 3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --block $b --blocks-per-sm $p \
    > gpurun_out/abc3_${tag}_${b}_${p}.json 2> gpurun_out/abc3_${tag}_${b}_${p}.err
  python - "$k" gpurun_out/abc3_${tag}_${b}_${p}.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(f"c3 block:bps={sys.argv[1]}: {d['value']:.4e} events/s frac {d['roofline']['frac']:.4f} k2_ms {d['roofline']['kernel_ms']:.1f}")
except Exception as e:
    print(f"c3 {sys.argv[1]}: failed {e}")
PY
done
