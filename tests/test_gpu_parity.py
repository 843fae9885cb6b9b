"""GPU parity: the CUDA path through the C ABI vs the CPU oracle, element by
element on the same seeded inputs (north_star rules): integer grid states,
event counts and firing hashes bit-exact; event times bit-exact (both sides
use the pinned plog); mean/variance within 1e-9 relative of the oracle's
exact-integer moments."""
import numpy as np
import pytest

import inputs
from inputs.networks import Network, _rx

from .helpers import assert_dump_equal, assert_moments_close, exact_moments, oracle_replay

pytestmark = pytest.mark.gpu

THREAD, WARP, HALF = 1, 2, 3
MODE = {THREAD: 0, WARP: 1, HALF: 3}     # summation orders: sequential, warp32, warp16s (oracle mode 3)


@pytest.fixture(scope="module")
def S():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_1007_1768_b200 import build
    build.build()
    from paper_1007_1768_b200 import ssa
    return ssa


def _parity(S, net, n, t_end, dt, seed, path, dump_ids=None, **opts):
    m = S.Model(net)
    ids = np.arange(n, dtype=np.uint64) if dump_ids is None else np.asarray(dump_ids, np.uint64)
    r = S.run(m, n, t_end, dt, seed, path=path, dump_ids=ids, **opts)
    assert r.path_used == path and r.status == 0
    gx, ge, gt, sm = oracle_replay(net, ids, seed, t_end, dt, MODE[path])
    assert_dump_equal(r.dump, gx, ge, gt, sm)
    assert r.events >= int(sm["events"].sum()) if dump_ids is not None else r.events == int(sm["events"].sum())
    if dump_ids is None:
        ref_mean, ref_var = exact_moments(gx)
        assert_moments_close(r.mean, r.var, ref_mean, ref_var)
        assert np.all(r.count == n)
    return r, (gx, ge, gt, sm)


# ------------------------------------------------------------ configs 0 and 1
@pytest.mark.parametrize("path", [THREAD, WARP, HALF])
def test_config0_full_parity(S, path):
    cfg = inputs.config(0)
    _parity(S, cfg.network, cfg.n_trajectories, cfg.t_end, cfg.dt, cfg.seed, path)


@pytest.mark.parametrize("path", [THREAD, WARP, HALF])
def test_config1_parity_ragged(S, path):
    """Several reduction tiles and a ragged tail (5000 = 2*2048 + 904)."""
    cfg = inputs.config(1)
    _parity(S, cfg.network, 5000, cfg.t_end, cfg.dt, cfg.seed, path)


def test_config1_full_size(S):
    """BASELINE configs[1] at full size (65,536 trajectories, ~1e8 events):
    every trajectory replayed by the oracle."""
    cfg = inputs.config(1)
    _parity(S, cfg.network, cfg.n_trajectories, cfg.t_end, cfg.dt, cfg.seed, THREAD)


# ------------------------------------------------------------ HIV (configs 2, 4)
@pytest.mark.parametrize("path", [THREAD, WARP, HALF])
def test_hiv_short_horizon_parity(S, path):
    cfg = inputs.config(2)
    _parity(S, cfg.network, 300, 5.0, cfg.dt, cfg.seed, path)


def test_hiv_full_horizon_sample(S):
    """Full 100-day horizon, a handful of whole trajectories, bit-exact."""
    cfg = inputs.config(2)
    _parity(S, cfg.network, 16, cfg.t_end, cfg.dt, cfg.seed, THREAD)


# (BASELINE configs[2] at full size -- T1 over 256 random ids and T2 over all 2^18 -- is
# tests/test_gpu_bench_parity.py, on the exact kernel and launch bench.py times.)


def test_config4_shards_sampled(S):
    """BASELINE configs[4] (HIV, 400 d, 2^24 ids over W = 8 shards, 65,536 dumped
    ids): an aligned block of 2^16 ids inside shard 0 and one of 4096 ids inside
    shard 7 run at the full horizon through ssa_run_shard with global ids (so the
    Philox streams are the ones the 8-GPU run uses).  Every config-4 dumped id in
    the blocks (>= 256) is replayed by the oracle bit-exactly,
    and the 2^16 block's shard root is checked against the exact moments of all its
    trajectories (T2)."""
    import torch
    cfg = inputs.config(4)
    n_total, W = cfg.n_trajectories, 8
    m = S.Model(cfg.network)
    G = S.grid_size(cfg.t_end, cfg.dt)
    cells = G * cfg.network.S
    dumped = inputs.dump_ids(n_total, cfg.n_dump, cfg.seed)
    replayed = 0
    for rank, blk in ((0, 1 << 16), (W - 1, 4096)):
        b, e = S.shard_bounds(n_total, W, rank)
        lo = b + (e - b) // 2                        # aligned block in the middle of the shard
        hi = lo + blk
        assert lo % blk == 0
        sel = dumped[(dumped >= lo) & (dumped < hi)]
        assert len(sel) >= 4
        ids = np.arange(lo, hi, dtype=np.uint64) if rank == 0 else sel
        root = torch.zeros((1, 3, cells), dtype=torch.float64, device="cuda")
        r = S.run_shard(m, lo, hi, cfg.t_end, cfg.dt, cfg.seed, root[0], path=THREAD, dump_ids=ids)
        assert r.n_errors == 0
        pos = np.searchsorted(ids, sel)
        gx, ge, gt, sm = oracle_replay(cfg.network, sel, cfg.seed, cfg.t_end, cfg.dt, 0)
        sub = S.Dump(sel, r.dump.states[pos], r.dump.events_at[pos], r.dump.time_at[pos], r.dump.summary[pos])
        assert_dump_equal(sub, gx, ge, gt, sm)
        replayed += len(sel)
        if rank == 0:
            mean, var, _, count = S.merge_roots(root, 1, cells)
            ref_mean, ref_var = exact_moments(r.dump.states)
            assert_moments_close(mean.reshape(G, -1), var.reshape(G, -1), ref_mean, ref_var)
            assert np.all(count == blk)
            assert r.events == int(r.dump.summary["events"].sum())
    assert replayed >= 256


# ------------------------------------------------------------ config 3 (warp path)
def test_config3_warp_parity(S):
    cfg = inputs.config(3)
    _parity(S, cfg.network, 96, cfg.t_end, cfg.dt, cfg.seed, WARP)


def test_config3_halfwarp_parity(S):
    """Config 3 on the half-warp path (two trajectories per warp, order
    warp16s), with an odd count so the last warp has one idle half."""
    cfg = inputs.config(3)
    _parity(S, cfg.network, 97, cfg.t_end, cfg.dt, cfg.seed, HALF)


def test_config3_thread_parity(S):
    cfg = inputs.config(3)
    _parity(S, cfg.network, 64, 2.0, cfg.dt, cfg.seed, THREAD)


def test_config3_full_size_sampled(S):
    """BASELINE configs[3] at full size (2^20 trajectories) on the one-trajectory-per-warp
    K2 (order warp32): 64 sampled trajectories replayed bit-exactly, and the full run's
    grids bitwise equal to the merge of four shard runs.  (The bench's half-warp K2 at
    this size, with T1 over 4096 ids and T2 over the whole ensemble, is
    tests/test_gpu_bench_parity.py.)"""
    cfg = inputs.config(3)
    n = cfg.n_trajectories
    m = S.Model(cfg.network)
    ids = inputs.dump_ids(n, 64, cfg.seed)
    r = S.run(m, n, cfg.t_end, cfg.dt, cfg.seed, path=WARP, dump_ids=ids)
    assert r.status == 0
    gx, ge, gt, sm = oracle_replay(cfg.network, ids, cfg.seed, cfg.t_end, cfg.dt, 1)
    assert_dump_equal(r.dump, gx, ge, gt, sm)
    assert np.all(r.count == n)
    # the reduction of the full ensemble equals the merge of shard roots (invariance)
    import torch
    G = S.grid_size(cfg.t_end, cfg.dt)
    cells = G * cfg.network.S
    roots = torch.zeros((4, 3, cells), dtype=torch.float64, device="cuda")
    for w in range(4):
        b, e = S.shard_bounds(n, 4, w)
        S.run_shard(m, b, e, cfg.t_end, cfg.dt, cfg.seed, roots[w], path=WARP)
    mean, var, _, _ = S.merge_roots(roots, 4, cells)
    assert np.array_equal(mean.reshape(G, -1), r.mean) and np.array_equal(var.reshape(G, -1), r.var)


# ------------------------------------------------------------ invariance
def test_chunk_block_and_schedule_invariance(S):
    """Bitwise identical moments and dumps for any chunk size, block size and
    residency (R26: chunks are aligned subtrees)."""
    cfg = inputs.config(1)
    m = S.Model(cfg.network)
    n = 3000
    ids = np.arange(0, n, 7, dtype=np.uint64)
    base = S.run(m, n, cfg.t_end, cfg.dt, cfg.seed, path=THREAD, dump_ids=ids)
    for opts in (dict(chunk=1024), dict(chunk=256, block=64), dict(block=256, blocks_per_sm=1),
                 dict(staging_budget_bytes=1 << 20)):
        r = S.run(m, n, cfg.t_end, cfg.dt, cfg.seed, path=THREAD, dump_ids=ids, **opts)
        assert np.array_equal(r.mean, base.mean) and np.array_equal(r.var, base.var), opts
        assert np.array_equal(r.m2, base.m2)
        assert np.array_equal(r.dump.states, base.dump.states)
    for path in (WARP, HALF):
        a = S.run(m, n, cfg.t_end, cfg.dt, cfg.seed, path=path)
        for opts in (dict(chunk=512), dict(block=128), dict(block=512, blocks_per_sm=1)):
            b = S.run(m, n, cfg.t_end, cfg.dt, cfg.seed, path=path, **opts)
            assert np.array_equal(a.mean, b.mean) and np.array_equal(a.var, b.var), (path, opts)


@pytest.mark.parametrize("path", [THREAD, HALF])
def test_ragged_chunks_reduce_only_written_tiles(S, path):
    """A ragged chunk holds fewer reduction tiles than the chunk span: 5000 ids
    in chunks of 4096 (the last chunk has 904 ids, one tile of its two), and
    5000 ids in one 8192 chunk (3 tiles of 4), each run right after a larger
    run that leaves other data in the pooled buffers.  Counts, moments and M2
    must be those of the exact sums over the 5000 trajectories."""
    cfg = inputs.config(1)
    m = S.Model(cfg.network)
    n = 5000
    ids = np.arange(n, dtype=np.uint64)
    ref = None
    for big, opts in ((8192, dict(chunk=4096)), (8192, dict()), (16384, dict(chunk=8192))):
        S.run(m, big, cfg.t_end, cfg.dt, cfg.seed + 1, path=path, **opts)    # dirty the pool
        r = S.run(m, n, cfg.t_end, cfg.dt, cfg.seed, path=path, dump_ids=ids, **opts)
        assert np.all(r.count == n), opts
        if ref is None:
            ref = exact_moments(r.dump.states)
            first = r
        assert_moments_close(r.mean, r.var, *ref)
        assert np.array_equal(r.mean, first.mean) and np.array_equal(r.m2, first.m2), opts


def test_tail_compaction_is_bitwise_neutral(S, monkeypatch, capfd):
    """K1 tail compaction (ssa_run_options.tail_lanes): once the ids are exhausted, the
    trajectories of sparse warps are suspended at a grid crossing and taken over by lanes of
    dense warps or, 32 at a time, by warps left idle.  Off (-1), 16 and aggressive (31: any
    warp that lost a lane) give bitwise identical grids, counters and dumps, suspensions do
    happen, and the dumped trajectories match the oracle."""
    cfg = inputs.config(1)
    m = S.Model(cfg.network)
    n = 20000
    ids = np.arange(0, n, 37, dtype=np.uint64)
    monkeypatch.setenv("SSA_DEBUG_TAIL", "1")
    runs = {tl: S.run(m, n, cfg.t_end, cfg.dt, cfg.seed, path=THREAD, dump_ids=ids, tail_lanes=tl)
            for tl in (-1, 16, 31)}
    err = capfd.readouterr().err
    import re
    counts = [int(v) for v in re.findall(r"\[ssa tail\] chunk 0: (\d+) suspended", err)]
    assert len(counts) == 2 and counts[-1] > 0, err
    off = runs[-1]
    for tl in (16, 31):
        r = runs[tl]
        assert np.array_equal(r.mean, off.mean) and np.array_equal(r.var, off.var) and np.array_equal(r.m2, off.m2)
        assert r.events == off.events and r.near_ties == off.near_ties
        for f in ("states", "events_at", "time_at"):
            assert np.array_equal(getattr(r.dump, f), getattr(off.dump, f)), (tl, f)
        assert r.dump.summary.tobytes() == off.dump.summary.tobytes()
    gx, ge, gt, sm = oracle_replay(cfg.network, ids[:64], cfg.seed, cfg.t_end, cfg.dt, 0)
    r = runs[31]
    sub = S.Dump(ids[:64], r.dump.states[:64], r.dump.events_at[:64], r.dump.time_at[:64], r.dump.summary[:64])
    assert_dump_equal(sub, gx, ge, gt, sm)
    # HIV (hot-set variant after the profiling run), no dump: the same bits with and without
    hm = S.Model(inputs.config(2).network)
    a = S.run(hm, 40000, 6.0, 1.0, 3, path=THREAD, tail_lanes=-1)
    b = S.run(hm, 40000, 6.0, 1.0, 3, path=THREAD, tail_lanes=31)
    c = S.run(hm, 40000, 6.0, 1.0, 3, path=THREAD, tail_lanes=16)
    for r in (b, c):
        assert np.array_equal(r.mean, a.mean) and np.array_equal(r.m2, a.m2) and r.events == a.events


def test_time_slices_are_bitwise_neutral(S, monkeypatch):
    """K1 time-sliced trajectories (SSA_K1_SEG = phases per trajectory): the jobs
    are (phase, trajectory) pairs handed out phase by phase, a trajectory's state crosses phases
    through memory at a grid crossing, and the resumed lane recomputes the pending candidate.
    1, 2, 3 and 7 phases give bitwise identical grids, counters and dumps (ragged chunk, early
    die-outs and absorbing trajectories included), and the dumped trajectories match the oracle."""
    cfg = inputs.config(1)
    m = S.Model(cfg.network)
    n = 20000
    ids = np.arange(0, n, 37, dtype=np.uint64)
    runs = {}
    for sv in ("1", "2", "3", "7"):
        monkeypatch.setenv("SSA_K1_SEG", sv)
        runs[sv] = S.run(m, n, cfg.t_end, cfg.dt, cfg.seed, path=THREAD, dump_ids=ids, chunk=8192)
    off = runs["1"]
    for sv in ("2", "3", "7"):
        r = runs[sv]
        assert np.array_equal(r.mean, off.mean) and np.array_equal(r.var, off.var) and np.array_equal(r.m2, off.m2)
        assert r.events == off.events and r.near_ties == off.near_ties
        for f in ("states", "events_at", "time_at"):
            assert np.array_equal(getattr(r.dump, f), getattr(off.dump, f)), (sv, f)
        assert r.dump.summary.tobytes() == off.dump.summary.tobytes()
    gx, ge, gt, sm = oracle_replay(cfg.network, ids[:64], cfg.seed, cfg.t_end, cfg.dt, 0)
    r = runs["7"]
    sub = S.Dump(ids[:64], r.dump.states[:64], r.dump.events_at[:64], r.dump.time_at[:64], r.dump.summary[:64])
    assert_dump_equal(sub, gx, ge, gt, sm)
    # HIV (profiling run, then the hot-set variant; ~11% of the trajectories die out early)
    hm = S.Model(inputs.config(2).network)
    hids = np.arange(0, 40000, 211, dtype=np.uint64)
    monkeypatch.setenv("SSA_K1_SEG", "1")
    a = S.run(hm, 40000, 6.0, 1.0, 3, path=THREAD, dump_ids=hids)
    a2 = S.run(hm, 40000, 6.0, 1.0, 3, path=THREAD)
    monkeypatch.setenv("SSA_K1_SEG", "4")
    b = S.run(hm, 40000, 6.0, 1.0, 3, path=THREAD, dump_ids=hids)
    c = S.run(hm, 40000, 6.0, 1.0, 3, path=THREAD)
    for r in (a2, b, c):
        assert np.array_equal(r.mean, a.mean) and np.array_equal(r.m2, a.m2) and r.events == a.events
    assert np.array_equal(b.dump.states, a.dump.states) and b.dump.summary.tobytes() == a.dump.summary.tobytes()


def test_reduction_paths_bitwise_equal(S):
    """K3's full-tile kernel takes an integer fast path for 8-leaf groups below
    2^20 and the fp64 Chan merges otherwise; both must give the canonical
    tree's bits.  Counts straddling 2^20 (immigration from 2^20 - 40) mix the
    two paths in one tile; a chunk of 1024 ids (partial tiles only, general
    kernel) must agree bitwise, and the moments must match the exact ones."""
    net = Network(("A",), (2**20 - 40,), (_rx([], [(0, 1)], 20.0),))
    m = S.Model(net)
    n = 4096
    full = S.run(m, n, 4.0, 0.5, 13, path=THREAD, dump_ids=np.arange(n))
    part = S.run(m, n, 4.0, 0.5, 13, path=THREAD, chunk=1024)
    assert np.array_equal(full.mean, part.mean) and np.array_equal(full.m2, part.m2)
    assert np.any(full.dump.states >= 2**20) and np.any(full.dump.states < 2**20)
    ref_mean, ref_var = exact_moments(full.dump.states)
    assert_moments_close(full.mean, full.var, ref_mean, ref_var)


@pytest.mark.parametrize("W", [2, 4, 8])
def test_shard_merge_equals_single_run(S, W):
    """The multi-GPU form (ssa_run_shard per rank + ssa_merge_roots), run here
    shard by shard on one GPU: bitwise equal to ssa_run for any W."""
    import torch
    cfg = inputs.config(0)
    m = S.Model(cfg.network)
    n = 1000
    base = S.run(m, n, cfg.t_end, cfg.dt, cfg.seed, path=THREAD)
    G = S.grid_size(cfg.t_end, cfg.dt)
    cells = G * cfg.network.S
    roots = torch.zeros((W, 3, cells), dtype=torch.float64, device="cuda")
    events = 0
    for w in range(W):
        b, e = S.shard_bounds(n, W, w)
        if e > b:
            events += S.run_shard(m, b, e, cfg.t_end, cfg.dt, cfg.seed, roots[w], path=THREAD).events
    mean, var, m2, count = S.merge_roots(roots, W, cells)
    assert np.array_equal(mean.reshape(G, -1), base.mean)
    assert np.array_equal(var.reshape(G, -1), base.var)
    assert np.array_equal(m2.reshape(G, -1), base.m2)
    assert events == base.events


# ------------------------------------------------------------ edge cases
def test_edge_cases(S):
    m = S.Model(inputs.immigration_death())
    # N = 1, G = 1 (t_end < dt)
    r = S.run(m, 1, 0.5, 1.0, 9, dump_ids=[0])
    assert r.mean.shape == (1, 1) and r.mean[0, 0] == 0 and r.var[0, 0] == 0
    gx, ge, gt, sm = oracle_replay(inputs.immigration_death(), [0], 9, 0.5, 1.0, 0)
    assert_dump_equal(r.dump, gx, ge, gt, sm)
    # empty network: held state, absorbed
    e = S.Model(inputs.empty_network((7, 0, 3)))
    r = S.run(e, 33, 10.0, 1.0, 1, dump_ids=np.arange(33))
    assert np.all(r.mean == np.array([7, 0, 3])) and np.all(r.var == 0)
    assert np.all(r.dump.summary["absorbed"] == 1) and r.events == 0
    # pure death to extinction (absorbing mid-run), both paths
    for path in (THREAD, WARP, HALF):
        _parity(S, inputs.pure_death(1.0, 5), 257, 10.0, 0.5, 3, path)


@pytest.mark.parametrize("path", [THREAD, WARP, HALF])
def test_trimolecular_and_modifier_network(S, path):
    """Reactant coefficient 3 (C(x,3)), a bimolecular 2A term, a catalyst and a
    negative rate modifier on a small network, both paths (the warp path then
    takes its general propensity evaluator)."""
    net = Network(("A", "B", "C"), (60, 5, 3), (
        _rx([(0, 3)], [(1, 1)], 2e-4),                 # 3A -> B       C(A,3)
        _rx([(1, 1)], [(0, 3)], 0.3),                  # B -> 3A
        _rx([(0, 2)], [(2, 1)], 1e-3),                 # 2A -> C       C(A,2)
        _rx([(2, 1)], [(0, 2)], 0.2),                  # C -> 2A
        _rx([(1, 1), (2, 1)], [(1, 1)], 0.05, mod=(0, -1e-3)),   # B + C -> B, k^ = max(0, k - 1e-3 A)
    ))
    _parity(S, net, 700, 6.0, 0.25, 17, path)


@pytest.mark.parametrize("path", [THREAD, WARP, HALF])
def test_mini_hiv_parity(S, path):
    """The HIV reaction list on its finite CME-pinned version (tests/test_oracle_distribution.py:
    infections with signed infectivity modifiers at F = 2, I+Z clearances, mutation): every
    reaction fires; bit-exact against the oracle on every path."""
    from .test_oracle_distribution import _mini_hiv
    _parity(S, _mini_hiv(), 1500, 3.0, 0.25, 21, path)


def test_numeric_error_reported(S):
    """A propensity that overflows to inf (SPEC.md:85 'NaN/inf -> hard error
    naming the reaction'): SSA_ERR_NUMERIC with the id and reaction."""
    net = Network(("A", "B"), (1, 0), (
        _rx([], [(1, 1)], 1.0),
        _rx([(0, 1)], [(0, 2)], 1e308),           # A doubles; a = 1e308 * A overflows at A = 2
    ))
    m = S.Model(net)
    for path in (THREAD, WARP, HALF):
        r = S.run(m, 8, 10.0, 1.0, 1, path=path, dump_ids=np.arange(8), raise_on_error=False)
        assert r.status == 3 and r.n_errors == 8
        assert r.first_error_id == 0 and r.first_error_reaction == 1
        _, _, _, sm = oracle_replay(net, np.arange(8), 1, 10.0, 1.0, MODE[path])
        assert np.all(sm["status"] == 3) and np.all(sm["err_reaction"] == 1)
        assert np.array_equal(r.dump.summary["status"], sm["status"])
        assert np.array_equal(r.dump.summary["err_reaction"], sm["err_reaction"])
        assert np.array_equal(r.dump.summary["events"], sm["events"])


def test_time_slices_errors_and_absorption(S, monkeypatch):
    """Time-sliced K1 at more trajectories than resident lanes (so the slicing is active): a
    numeric error that strikes only some trajectories, late in their horizon, is reported with the
    same status, error count, first erroring id and reaction as without slicing, and absorbed
    trajectories (pure death reaching 0, then a0 = 0 for the rest of the grid) give the same grids."""
    n = 160000                                   # > 148 SMs x 512 resident lanes
    # A grows by immigration; B doubles at rate 1e-3 per B and its propensity overflows at B = 2:
    # only trajectories whose B fires within the horizon err
    net = Network(("A", "B"), (0, 1), (
        _rx([], [(0, 1)], 5.0),
        _rx([(1, 1)], [(1, 2)], 2e-6),
        _rx([(1, 2)], [(1, 3)], 1e308),           # 2B -> 3B: C(3, 2) * 1e308 = inf once B = 3
    ))
    m = S.Model(net)
    res = {}
    for sv in ("1", "8"):
        monkeypatch.setenv("SSA_K1_SEG", sv)
        res[sv] = S.run(m, n, 40.0, 1.0, 11, path=THREAD, raise_on_error=False)
    a, b = res["1"], res["8"]
    assert a.status == 3 and 0 < a.n_errors < n, (a.status, a.n_errors)
    assert (b.status, b.n_errors, b.first_error_id, b.first_error_reaction, b.events) == \
        (a.status, a.n_errors, a.first_error_id, a.first_error_reaction, a.events)
    # absorption: pure death from 3 molecules at rate 0.2 over 30 time units
    pd = S.Model(inputs.pure_death(k=0.2, x0=3))
    monkeypatch.setenv("SSA_K1_SEG", "1")
    c = S.run(pd, n, 30.0, 0.5, 5, path=THREAD)
    monkeypatch.setenv("SSA_K1_SEG", "8")
    d = S.run(pd, n, 30.0, 0.5, 5, path=THREAD)
    assert c.events == d.events and np.array_equal(c.mean, d.mean) and np.array_equal(c.m2, d.m2)
    assert c.mean[-1, 0] < 0.01                  # nearly every trajectory absorbed by t = 30


@pytest.mark.parametrize("path", [THREAD, WARP, HALF])
def test_overflow_reported(S, path):
    net = Network(("A",), (2**31 - 5,), (_rx([], [(0, 1)], 100.0),))
    m = S.Model(net)
    r = S.run(m, 4, 1.0, 0.5, 1, path=path, raise_on_error=False)
    assert r.status == 4 and r.n_errors == 4


def test_device_outputs_and_determinism(S):
    import torch
    cfg = inputs.config(1)
    m = S.Model(cfg.network)
    G = S.grid_size(cfg.t_end, cfg.dt)
    out = torch.zeros((4, G, 3), dtype=torch.float64, device="cuda")
    S.run_device(m, 2048, cfg.t_end, cfg.dt, cfg.seed, out, path=THREAD)
    h = S.run(m, 2048, cfg.t_end, cfg.dt, cfg.seed, path=THREAD)
    assert np.array_equal(out[0].cpu().numpy(), h.mean) and np.array_equal(out[1].cpu().numpy(), h.var)
    h2 = S.run(m, 2048, cfg.t_end, cfg.dt, cfg.seed, path=THREAD)
    assert np.array_equal(h.mean, h2.mean) and h.events == h2.events


def test_profiled_dispatch_is_bitwise_neutral(S):
    """The first plain thread-path run of a model samples its propensity shares and picks the K1
    hot set (HIV: the two clearances, ~98% of its events); later runs apply those reactions by
    predicated adds ahead of the jump table.  Results, counters and dumps are bitwise those of the
    profiling run, and the dumped trajectories match the oracle."""
    cfg = inputs.config(2)
    m = S.Model(cfg.network)
    assert m.hot_set() is None
    ids = np.arange(0, 4096, 97, dtype=np.uint64)
    a = S.run(m, 4096, 30.0, 1.0, cfg.seed, path=THREAD, dump_ids=ids)
    hot = m.hot_set()
    assert hot is not None and set(hot) <= set(range(27)) and 26 in hot, hot
    b = S.run(m, 4096, 30.0, 1.0, cfg.seed, path=THREAD, dump_ids=ids)
    assert np.array_equal(a.mean, b.mean) and np.array_equal(a.var, b.var) and a.events == b.events
    for f in ("states", "events_at", "time_at"):
        assert np.array_equal(getattr(a.dump, f), getattr(b.dump, f)), f
    assert a.dump.summary.tobytes() == b.dump.summary.tobytes()
    gx, ge, gt, sm = oracle_replay(cfg.network, ids[:8], cfg.seed, 30.0, 1.0, 0)
    sub = S.Dump(ids[:8], b.dump.states[:8], b.dump.events_at[:8], b.dump.time_at[:8], b.dump.summary[:8])
    assert_dump_equal(sub, gx, ge, gt, sm)


def test_dump_accounting_and_pinned(S):
    """a11 dump: dump_bytes is the payload (states, events_at, time_at, summaries), the D2H is timed
    (dump_ms), and page-locked host arrays receive the same bytes as pageable ones."""
    cfg = inputs.config(0)
    m = S.Model(cfg.network)
    G = S.grid_size(cfg.t_end, cfg.dt)
    ids = np.array([0, 3, 17, 999], dtype=np.uint64)
    a = S.run(m, cfg.n_trajectories, cfg.t_end, cfg.dt, cfg.seed, dump_ids=ids)
    b = S.run(m, cfg.n_trajectories, cfg.t_end, cfg.dt, cfg.seed, dump_ids=ids, dump_pinned=True)
    n = len(ids)
    assert a.dump_bytes == n * G * (4 * m.S + 8 + 8) + n * S.SUMMARY_DTYPE.itemsize
    assert a.dump_bytes == b.dump_bytes and a.d2h_bytes >= a.dump_bytes
    assert a.dump_ms > 0.0 and b.dump_ms > 0.0
    for f in ("states", "events_at", "time_at"):
        assert np.array_equal(getattr(a.dump, f), getattr(b.dump, f))
    assert a.dump.summary.tobytes() == b.dump.summary.tobytes()
    c = S.run(m, cfg.n_trajectories, cfg.t_end, cfg.dt, cfg.seed)
    assert c.dump_bytes == 0 and c.dump_ms == 0.0


# ------------------------------------------------------------ gated propensities (NEXT 3)
@pytest.mark.parametrize("path", [THREAD, WARP, HALF])
def test_gated_networks_parity(S, path):
    """SPEC.md:424-style gates and the mass-action switch on both paths,
    bit-exact against the oracle: the one-shot event, constant-rate depletion,
    and the HIV Variant B time-triggered mutation (mu raised so that it fires
    inside the short horizon)."""
    one_shot = Network(("M",), (0,), (_rx([], [(0, 1)], 0.3, gates=[(0, inputs.GATE_ZERO)]),))
    deplete = Network(("A",), (10,), (_rx([(0, 1)], [], 2.0, mass_action=False,
                                           gates=[(0, inputs.GATE_POSITIVE)]),))
    _parity(S, one_shot, 1000, 10.0, 0.5, 21, path)
    _parity(S, deplete, 1000, 8.0, 0.5, 22, path)
    _parity(S, inputs.hiv("B", mu=0.5), 200, 2.0, 0.25, 23, path)
