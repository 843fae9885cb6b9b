"""Diagnostics probe of the half-warp K2 against the oracle (order warp16s) on a tiny config-3 run."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import inputs
from paper_1007_1768_b200 import ssa as S
from oracle import oracle as O
t_end = float(sys.argv[1]) if len(sys.argv) > 1 else 0.2
n = int(sys.argv[2]) if len(sys.argv) > 2 else 64
cfg = inputs.config(3)
m = S.Model(cfg.network)
t0 = time.time()
r = S.run(m, n, t_end, t_end / 4, 4, path=3, dump_ids=np.arange(n))
ref = O.run(O.OracleModel(cfg.network), np.arange(n, dtype=np.uint64), 4, t_end, t_end / 4, 3)
ge, oe = r.dump.summary["events"], ref.summaries["events"]
print("events", r.events, "oracle", int(oe.sum()), "states equal", np.array_equal(r.dump.states, ref.grid_x),
      f"{time.time()-t0:.1f}s")
bad = np.nonzero(ge != oe)[0]
print("trajectories with different event counts:", len(bad), "first:", bad[:5], ge[bad[:5]], oe[bad[:5]])
