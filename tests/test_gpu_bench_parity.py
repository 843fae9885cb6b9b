"""Parity of the kernels bench.py actually times, at BASELINE.json's full sizes
(SURVEY.md §8(c) tiered checking; north_star parity rules; "exactly
according to the given probability distributions" under the bitwise contract).

- Config 2 (HIV, 2^18 x 100 d, thread path): the bench's K1 -- no dump, the
  measured hot set with cold-prefix reuse, the seed's Philox keys as
  immediates, the default 128 x 4 launch -- driven exactly as bench.py drives
  it (ShardedEnsemble.step on torch's current stream).  Its grids must be
  bitwise those of the profiling run and of the dump variant, within 1e-9 of
  the exact moments of all 2^18 dumped trajectories (T2), and >= 256 randomly
  chosen trajectories are replayed bit-exactly by the oracle (T1).
- Config 3 (synthetic 64 x 256, 2^20 x 10, half-warp K2 -- the bench's path):
  the bench-path run's grids within 1e-9 of the exact moments of ALL 2^20
  trajectories, accumulated from 64 aligned blocks of 2^14 dumped ids (T2 over
  the whole ensemble), the merge of the 64 block roots bitwise equal to the
  single run (chunk/shard invariance at full size), and 4096 randomly chosen
  trajectories replayed bit-exactly by the oracle in the warp16s order (oracle mode 3, T1).
"""
import numpy as np
import pytest

import inputs

from .helpers import assert_dump_equal, assert_moments_close, exact_moments, oracle_replay

pytestmark = pytest.mark.gpu

THREAD, HALF = 1, 3


@pytest.fixture(scope="module")
def S():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_1007_1768_b200 import build
    build.build()
    from paper_1007_1768_b200 import ssa
    return ssa


def _exact_from_sums(n, s1, s2):
    """Exact mean and population variance from integer sums (Python ints)."""
    from fractions import Fraction
    mean = np.array([float(Fraction(int(a), n)) for a in s1.reshape(-1)])
    var = np.array([float(Fraction(n * int(b) - int(a) * int(a), n * n)) for a, b in zip(s1.reshape(-1),
                                                                                         s2.reshape(-1))])
    return mean.reshape(s1.shape), var.reshape(s1.shape)


def test_config2_bench_kernel_full_size(S):
    import torch
    from paper_1007_1768_b200 import dist as D
    cfg = inputs.config(2)
    n, G = cfg.n_trajectories, S.grid_size(cfg.t_end, cfg.dt)
    m = S.Model(cfg.network)
    prof = S.run(m, n, cfg.t_end, cfg.dt, cfg.seed, path=THREAD)          # first run: the profiling K1
    hot = m.hot_set()
    assert hot and 26 in hot, hot                                          # V4 -> 0 carries most events
    # the bench's step: ShardedEnsemble on torch's current stream, outputs on the device
    dev = torch.device("cuda", 0)
    ens = D.ShardedEnsemble.for_model(m, n, cfg.t_end, cfg.dt, cfg.seed, dev, path=THREAD,
                                      stream=torch.cuda.current_stream(dev).cuda_stream)
    res = ens.step()
    torch.cuda.synchronize()
    out = ens.out.cpu().numpy().reshape(4, G, -1)
    assert res.status == 0 and res.events == prof.events and res.near_ties == prof.near_ties
    assert np.array_equal(out[0], prof.mean) and np.array_equal(out[1], prof.var)
    assert np.array_equal(out[2], prof.m2) and np.all(out[3] == n)
    # the dump variant over every id: same grids, and T2 from its dumped states
    all_ids = np.arange(n, dtype=np.uint64)
    dump = S.run(m, n, cfg.t_end, cfg.dt, cfg.seed, path=THREAD, dump_ids=all_ids)
    assert np.array_equal(dump.mean, out[0]) and np.array_equal(dump.m2, out[2]) and dump.events == res.events
    ref_mean, ref_var = exact_moments(dump.dump.states)
    assert_moments_close(out[0], out[1], ref_mean, ref_var)
    assert res.events == int(dump.dump.summary["events"].sum())
    assert res.near_ties == int(dump.dump.summary["near_ties"].sum())
    # T1: 256 random trajectories replayed by the oracle, bit-exact
    sample = inputs.dump_ids(n, 256, cfg.seed + 101)
    gx, ge, gt, sm = oracle_replay(cfg.network, sample, cfg.seed, cfg.t_end, cfg.dt, 0)
    idx = sample.astype(np.int64)
    sub = S.Dump(sample, dump.dump.states[idx], dump.dump.events_at[idx], dump.dump.time_at[idx],
                 dump.dump.summary[idx])
    assert_dump_equal(sub, gx, ge, gt, sm)


def test_config3_bench_kernel_full_size(S):
    import torch
    cfg = inputs.config(3)
    n, G, Sn = cfg.n_trajectories, S.grid_size(cfg.t_end, cfg.dt), cfg.network.S
    assert cfg.path == HALF
    m = S.Model(cfg.network)
    full = S.run(m, n, cfg.t_end, cfg.dt, cfg.seed, path=HALF)              # the bench's kernel and launch
    assert full.status == 0 and full.path_used == HALF and np.all(full.count == n)
    blk = 1 << 14
    cells = G * Sn
    roots = torch.zeros((n // blk, 3, cells), dtype=torch.float64, device="cuda")
    s1 = np.zeros(cells, dtype=object)
    s2 = np.zeros(cells, dtype=object)
    events = 0
    t1 = inputs.dump_ids(n, 4096, cfg.seed + 101)
    t1_states, t1_e, t1_t, t1_sum = [], [], [], []
    for b in range(n // blk):
        lo = b * blk
        ids = np.arange(lo, lo + blk, dtype=np.uint64)
        r = S.run_shard(m, lo, lo + blk, cfg.t_end, cfg.dt, cfg.seed, roots[b], path=HALF, dump_ids=ids)
        events += r.events
        x = r.dump.states.reshape(blk, cells).astype(np.int64)
        assert x.max() < (1 << 24)                                          # so the int64 sum of squares is exact
        s1 += x.sum(axis=0).astype(object)
        s2 += (x * x).sum(axis=0).astype(object)                          # < 2^62 per block
        sel = t1[(t1 >= lo) & (t1 < lo + blk)].astype(np.int64) - lo
        t1_states.append(r.dump.states[sel]); t1_e.append(r.dump.events_at[sel])
        t1_t.append(r.dump.time_at[sel]); t1_sum.append(r.dump.summary[sel])
    assert events == full.events
    # T2 over the whole ensemble: exact moments of all 2^20 trajectories
    ref_mean, ref_var = _exact_from_sums(n, s1, s2)
    assert_moments_close(full.mean.reshape(-1), full.var.reshape(-1), ref_mean, ref_var)
    # the 64 block roots merged in order are the single run, bitwise (aligned subtrees, R26)
    mean, var, m2, count = S.merge_roots(roots, n // blk, cells)
    assert np.array_equal(mean.reshape(G, -1), full.mean) and np.array_equal(var.reshape(G, -1), full.var)
    assert np.array_equal(m2.reshape(G, -1), full.m2)
    # T1: 4096 random trajectories replayed by the oracle in the warp16s order (mode 3), bit-exact
    gx, ge, gt, sm = oracle_replay(cfg.network, t1, cfg.seed, cfg.t_end, cfg.dt, 3)
    sub = S.Dump(t1, np.concatenate(t1_states), np.concatenate(t1_e), np.concatenate(t1_t),
                 np.concatenate(t1_sum))
    assert_dump_equal(sub, gx, ge, gt, sm)
