"""Small invocations of every kernel family for compute-sanitizer (scripts/sanitize.sh):
K1 (plain, dump, hot-set after profiling, tail compaction, sweep, record/union, stride points),
K2 (one trajectory per warp and half-warp, dump), K3/K4 (full and ragged tiles, multi-chunk merge)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
from paper_1007_1768_b200 import ssa as S  # noqa: E402

c1 = inputs.config(1)
m1 = S.Model(c1.network)
ids = np.arange(0, 5000, 97, dtype=np.uint64)
S.run(m1, 5000, 0.5, 0.1, 2, path=1)                                  # K1 profiling variant, K3 ragged tiles
S.run(m1, 5000, 0.5, 0.1, 2, path=1, dump_ids=ids, chunk=2048)        # K1 dump (hot set), chunks, K4 merges
S.run(m1, 5000, 0.5, 0.1, 2, path=1, tail_lanes=31)                   # tail compaction (suspend / resume)
hiv = S.Model(inputs.config(2).network)
S.run(hiv, 64, 0.2, 0.1, 3, path=1)
S.run(hiv, 64, 0.2, 0.1, 3, path=1, dump_ids=np.arange(0, 64, 7))
c3 = inputs.config(3)
m3 = S.Model(c3.network)
for path in (2, 3):                                                   # K2 warp and half-warp
    S.run(m3, 100, 0.1, 0.05, 4, path=path)
    S.run(m3, 100, 0.1, 0.05, 4, path=path, dump_ids=np.arange(0, 100, 5))
net, rates = inputs.hiv_delta_t_sweep()
S.run_sweep(S.Model(net), rates, 64, 0.2, 0.1, 3)                     # sweep variant
S.run_union(S.Model(inputs.immigration_death()), 8, 20.0, 1, 4)      # record variant + union reduction
S.run_trajectories(hiv, 4, 0.1, 3, 10)                                # stride variant + point gather
print("sanitize_run: done")
