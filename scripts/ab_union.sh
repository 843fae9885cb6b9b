#!/bin/bash
# A/B of the union pass geometry (SSA_UNION_GT = groups per warp, SSA_UNION_CH = events per batch):
#   bash scripts/ab_union.sh "GW:BT" ...
for k in "$@"; do
  gw=${k%%:*}; bt=${k##*:}
  SSA_UNION_GT=$gw SSA_UNION_CH=$bt timeout 600 python bench.py --workload union --steps 3 --warmup 1 --no-cpu-baseline \
    --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('GW:BT=$k', round(d['union_reduction']['ms'], 3), 'ms')"
done
