"""GPU parity of the selective memory at union times (ssa_run_union; SURVEY.md
§8(f) NEXT 2; §3.2.1 Fig. 3): the CUDA
pipeline (K1 event recording, radix sort by time, exact integer scans,
X-groups) against the oracle's offline brute-force definition
(oracle.union_reduce over oracle.stream) on the same seeded trajectories."""
import numpy as np
import pytest

import inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_1007_1768_b200 import build
    build.build()
    from paper_1007_1768_b200 import ssa
    return ssa


def _oracle(net, n, t_end, seed, kx):
    from oracle import oracle as O
    m = O.OracleModel(net)
    return O.union_reduce([O.stream(m, i, seed, t_end) for i in range(n)], kx)


@pytest.mark.parametrize("kx", [1, 3, 16])
def test_union_immigration_death(S, kx):
    net = inputs.immigration_death()
    n, t_end, seed = 16, 8.0, 31
    got = S.run_union(S.Model(net), n, t_end, seed, kx)
    t, mean, var, cnt = _oracle(net, n, t_end, seed, kx)
    assert len(got.times) == len(t)
    assert np.array_equal(got.times, t)                      # union times and group means: bitwise
    assert np.array_equal(got.count, cnt.astype(float))
    assert np.array_equal(got.mean, mean)                    # exact sums, one rounding each
    assert np.array_equal(got.var, var)


@pytest.mark.parametrize("kx", [1, 16])
def test_union_immigration_death_mid_size(S, kx):
    """A non-toy size: 16 immigration-death trajectories (config 0's rates) over
    t = 100, ~1.9e3 events each (~3e4 union times), against the oracle's
    brute-force definition -- times, counts, means and variances bitwise."""
    net = inputs.immigration_death()
    n, t_end, seed = 16, 100.0, 7
    got = S.run_union(S.Model(net), n, t_end, seed, kx)
    t, mean, var, cnt = _oracle(net, n, t_end, seed, kx)
    assert len(t) > 1000 * 16 // kx
    assert np.array_equal(got.times, t) and np.array_equal(got.count, cnt.astype(float))
    assert np.array_equal(got.mean, mean) and np.array_equal(got.var, var)


@pytest.mark.parametrize("gt,ch", [(1, 0), (2, 0), (7, 32), (0, 32)])
def test_union_small_tiles(S, monkeypatch, gt, ch):
    """Tiles of 1, 2 or 7 X-groups and staging chunks of 32 events (the
    SSA_UNION_GT / SSA_UNION_CH test hooks) put group, tile, chunk and run
    boundaries everywhere: same bitwise output as the oracle."""
    net = inputs.immigration_death()
    n, t_end, seed = 16, 30.0, 11
    if gt:
        monkeypatch.setenv("SSA_UNION_GT", str(gt))
    if ch:
        monkeypatch.setenv("SSA_UNION_CH", str(ch))
    for kx in (1, 5, 64):
        got = S.run_union(S.Model(net), n, t_end, seed, kx)
        t, mean, var, cnt = _oracle(net, n, t_end, seed, kx)
        assert np.array_equal(got.times, t) and np.array_equal(got.count, cnt.astype(float))
        assert np.array_equal(got.mean, mean) and np.array_equal(got.var, var)


def test_union_hiv_short(S):
    """The paper's HIV model (Fig. 4's 16 trajectories), over a short horizon."""
    net = inputs.hiv()
    n, t_end, seed, kx = 16, 0.05, 5, 16
    got = S.run_union(S.Model(net), n, t_end, seed, kx)
    t, mean, var, cnt = _oracle(net, n, t_end, seed, kx)
    assert np.array_equal(got.times, t) and np.array_equal(got.count, cnt.astype(float))
    assert np.array_equal(got.mean, mean) and np.array_equal(got.var, var)
    assert np.all(got.mean[:, 0] == 1.0)


def test_union_capacity_and_empty(S):
    """Too small a capacity reports the size needed; an empty network gives
    the two held slices 0 and t_end."""
    net = inputs.immigration_death()
    m = S.Model(net)
    with pytest.raises(S.SSAError) as ei:
        S.run_union(m, 4, 5.0, 1, 1, capacity=3)
    assert ei.value.status == 1
    e = S.run_union(S.Model(inputs.empty_network((4, 2))), 5, 3.0, 1, 1)
    assert np.array_equal(e.times, [0.0, 3.0]) and np.all(e.mean == [4, 2]) and np.all(e.var == 0)
    assert np.all(e.count == 5)


def test_union_record_buffer_rerun(S, monkeypatch):
    """A too-small first record buffer (forced through the SSA_UNION_CAP0 test
    hook) makes the library run once more with the exact size: same output."""
    net = inputs.dimerization(60)
    m = S.Model(net)
    a = S.run_union(m, 8, 1.0, 3, 4)
    monkeypatch.setenv("SSA_UNION_CAP0", "10")
    b = S.run_union(m, 8, 1.0, 3, 4)
    assert np.array_equal(a.times, b.times) and np.array_equal(a.mean, b.mean) and np.array_equal(a.var, b.var)
    assert a.result.events == b.result.events > 10


# ------------------------------------------------------------ stride-sampled output (NEXT 4)
@pytest.mark.parametrize("stride", [1, 10])
def test_trajectory_points_vs_oracle(S, stride):
    """ssa_run_trajectories: per trajectory the points (0, x0), every
    stride-th event and the horizon, bit-exact against oracle.stride_points."""
    from oracle import oracle as O
    net = inputs.dimerization(80)
    n, t_end, seed = 9, 2.0, 41
    got = S.run_trajectories(S.Model(net), n, t_end, seed, stride)
    om = O.OracleModel(net)
    assert np.all(np.diff(got.traj.astype(np.int64)) >= 0)
    for i in range(n):
        sel = got.traj == i
        k, t, x = O.stride_points(om, i, seed, t_end, stride)
        assert np.array_equal(got.event[sel], k)
        assert np.array_equal(got.time[sel], t)
        assert np.array_equal(got.states[sel], x.astype(np.int32))


def test_trajectory_points_hiv_and_rerun(S, monkeypatch):
    """The paper's HIV model with its 1:10 sampling over a short
    horizon, with a forced re-run of the recording (too small a first buffer)."""
    from oracle import oracle as O
    net = inputs.hiv()
    monkeypatch.setenv("SSA_UNION_CAP0", "100")
    got = S.run_trajectories(S.Model(net), 4, 0.2, 3, 10)
    om = O.OracleModel(net)
    for i in range(4):
        sel = got.traj == i
        k, t, x = O.stride_points(om, i, 3, 0.2, 10)
        assert np.array_equal(got.event[sel], k) and np.array_equal(got.time[sel], t)
        assert np.array_equal(got.states[sel], x.astype(np.int32))


def test_union_profiled_dispatch_bitwise(S):
    """The first recording run of a model measures its K1 hot set (HIV: the clearances); the next
    run records through the hot variant -- the event streams, and so every union point, are
    bitwise those of the first run."""
    m = S.Model(inputs.hiv())
    a = S.run_union(m, 16, 5.0, 5, 16)
    assert m.hot_set() is not None
    b = S.run_union(m, 16, 5.0, 5, 16)
    assert a.result.events == b.result.events
    for f in ("times", "mean", "var", "count"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
