#!/bin/bash
# A/B of K1 time-sliced trajectories (SSA_K1_SEG phases per trajectory) on config 2, after a bitwise
# check against the unsliced run.  usage: bash scripts/ab_seg.sh TAG N ...
tag=$1; shift
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python - <<'PY'
import os, numpy as np, inputs
from paper_1007_1768_b200 import ssa as S
cfg = inputs.config(2)
m = S.Model(cfg.network)
n = 1 << 15
ids = np.arange(0, n, 97, dtype=np.uint64)
res = {}
for sv in ("1", "4", "3"):
    os.environ["SSA_K1_SEG"] = sv
    r = S.run(m, n, 30.0, cfg.dt, cfg.seed, path=S.SSA_PATH_THREAD, dump_ids=ids, device=0)
    res[sv] = r
a = res["1"]
for sv in ("4", "3"):
    b = res[sv]
    ok = (np.array_equal(a.mean, b.mean) and np.array_equal(a.var, b.var) and a.events == b.events and
          np.array_equal(a.dump.states, b.dump.states) and np.array_equal(a.dump.summary["hash"], b.dump.summary["hash"]))
    print(f"seg={sv} bitwise equal to seg=1: {ok}  events {b.events}")
PY
for k in "$@"; do
  SSA_K1_SEG=$k timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e \
    > gpurun_out/abseg_${tag}_${k}.json 2> gpurun_out/abseg_${tag}_${k}.err
  python - "$k" gpurun_out/abseg_${tag}_${k}.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(f"seg={sys.argv[1]}: {d['value']:.4e} events/s frac {d['roofline']['frac']:.4f} k1_ms {d['roofline']['kernel_ms']:.1f}")
except Exception as e:
    print(f"seg={sys.argv[1]}: failed {e}")
PY
done
