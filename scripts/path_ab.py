"""Path A/B benchmark: events/s of the thread path (K1), the half-warp K2 and
the one-trajectory-per-warp K2 on synthetic networks of growing size, to set the AUTO dispatch
thresholds.  Run on the GPU box from the repo root:  PYTHONPATH=. python scripts/path_ab.py"""
import json
import sys

import inputs
from paper_1007_1768_b200 import build as B

B.build()
from paper_1007_1768_b200 import ssa as S  # noqa: E402

N, T_END, DT = 1 << 16, 1.0, 0.05
rows = []
for R in (8, 16, 32, 48, 64, 96, 128, 192, 256, 384, 512):
    Sp = max(4, R // 4)
    net = inputs.synthetic(Sp, R, seed=4)
    m = S.Model(net)
    row = {"R": R, "S": Sp}
    for name, path in (("thread", S.SSA_PATH_THREAD), ("halfwarp", S.SSA_PATH_HALFWARP), ("warp", S.SSA_PATH_WARP)):
        if path == S.SSA_PATH_THREAD and R > 256:
            continue
        try:
            S.run(m, N, T_END, DT, 4, path=path)          # JIT + warm-up
            r = S.run(m, N, T_END, DT, 4, path=path)
            row[name] = r.events / (r.ssa_ms / 1e3)
        except Exception as e:  # noqa: BLE001
            row[name] = f"error: {e}"
    rows.append(row)
    print(json.dumps(row), flush=True)
json.dump(rows, sys.stdout)
print()
