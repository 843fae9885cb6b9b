"""GPU parity of the parameter sweep (ssa_run_sweep; SURVEY.md §8(f) NEXT(1),
PAPER.md:131 "a set of parameter-swept simulations", Fig. 4 panels 2-4,
PAPER.md:155/:171).  Definition (R31): point p runs trajectories
0..N-1 with the same seed, so its grids are bitwise those of ssa_run on the
model with point p's constants; checked against ssa_run, against the oracle
(bit-exact replays of dumped trajectories of each point's model, exact
moments), across chunkings, and on the paper's delta_t sweep of the HIV
model."""
import numpy as np
import pytest

import inputs

from .helpers import assert_dump_equal, assert_moments_close, exact_moments, oracle_replay

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


def test_sweep_equals_independent_runs_and_oracle(S):
    net = inputs.immigration_death()
    rates = inputs.rate_matrix(net, [1], [0.1, 0.2, 0.05])      # X -> 0 at k2 = 0.1, 0.2, 0.05
    N, t_end, dt, seed = 700, 40.0, 1.0, 7                     # ragged: 700 = 2048-tile tail only
    m = S.Model(net)
    sw = S.run_sweep(m, rates, N, t_end, dt, seed)
    assert sw.status == 0 and sw.path_used == 1
    total = 0
    for p in range(len(rates)):
        net_p = inputs.with_rates(net, rates[p])
        one = S.run(S.Model(net_p), N, t_end, dt, seed, path=1)
        assert np.array_equal(sw.mean[p], one.mean) and np.array_equal(sw.var[p], one.var)
        assert np.array_equal(sw.m2[p], one.m2) and np.all(sw.count[p] == N)
        gx, ge, gt, sm = oracle_replay(net_p, np.arange(N, dtype=np.uint64), seed, t_end, dt, 0)
        ref_mean, ref_var = exact_moments(gx)
        assert_moments_close(sw.mean[p], sw.var[p], ref_mean, ref_var)
        total += int(sm["events"].sum())
    assert sw.events == total


def test_sweep_hiv_delta_t_fig4(S):
    """The paper's delta_t sensitivity sweep (5.0, 3.0, 0.5) of the HIV model:
    every trajectory of every point dumped; sampled ones replayed by the oracle
    on that point's model (bit-exact), all of them reduced exactly (T2)."""
    net, rates = inputs.hiv_delta_t_sweep()
    N, t_end, dt, seed = 256, 3.0, 0.5, 11
    m = S.Model(net)
    P = len(rates)
    vids = np.arange(P * N, dtype=np.uint64)
    sw = S.run_sweep(m, rates, N, t_end, dt, seed, dump_ids=vids)
    assert sw.status == 0
    G = S.grid_size(t_end, dt)
    for p in range(P):
        states = sw.dump.states[p * N:(p + 1) * N]
        ref_mean, ref_var = exact_moments(states)
        assert_moments_close(sw.mean[p], sw.var[p], ref_mean, ref_var)
        assert np.all(sw.mean[p][:, 0] == 1.0)                   # U0 is a catalyst
        sample = np.array([0, 1, 97, N - 1], dtype=np.uint64)
        gx, ge, gt, sm = oracle_replay(inputs.with_rates(net, rates[p]), sample, seed, t_end, dt, 0)
        rows = (p * N + sample).astype(np.int64)
        assert np.array_equal(sw.dump.states[rows], gx)
        assert np.array_equal(sw.dump.events_at[rows], ge)
        assert np.array_equal(sw.dump.time_at[rows], gt)
        assert np.array_equal(sw.dump.summary["hash"][rows], sm["hash"])
    assert sw.events == int(sw.dump.summary["events"].sum())
    assert sw.mean.shape == (P, G, net.S)
    # the sweep points differ (T clearance 5.0 vs 0.5 changes T by t = 3)
    assert sw.mean[0][-1, 2] < sw.mean[2][-1, 2]


def test_sweep_chunking_and_modifiers(S):
    """Points split over several launches (small staging budget) give the same
    bits as one launch; a sweep over modifier coefficients (sign changes make
    the clamp of P:93 reachable) matches independent runs."""
    net = inputs.hiv()
    N, t_end, dt, seed = 300, 1.0, 0.25, 5
    rates = inputs.rate_matrix(net, [25, 26], [2.0, 1.0, 4.0, 3.0])
    m = S.Model(net)
    G = S.grid_size(t_end, dt)
    one = S.run_sweep(m, rates, N, t_end, dt, seed)
    small = S.run_sweep(m, rates, N, t_end, dt, seed, staging_budget_bytes=N * G * net.S * 4 + 16)
    assert np.array_equal(one.mean, small.mean) and np.array_equal(one.m2, small.m2)
    assert small.kernel_launches > one.kernel_launches
    base = np.array([r.modifier_coef for r in net.reactions])
    mods = np.stack([base, -base, 10 * base])
    sw = S.run_sweep(m, np.tile(rates[0], (3, 1)), N, t_end, dt, seed, mod_coefs=mods)
    for p in range(3):
        rx = tuple(inputs.Reaction(r.reactants, r.products, r.rate, r.modifier_species, float(mods[p, j]), r.name)
                   for j, r in enumerate(net.reactions))
        net_p = inputs.Network(net.species, net.x0, rx, net.name)
        ref = S.run(S.Model(net_p), N, t_end, dt, seed, path=1)
        assert np.array_equal(sw.mean[p], ref.mean) and np.array_equal(sw.var[p], ref.var)


def test_sweep_rejects_warp_path(S):
    net = inputs.immigration_death()
    m = S.Model(net)
    with pytest.raises(S.SSAError) as ei:
        S.run_sweep(m, inputs.rate_matrix(net, [1], [0.1, 0.2]), 10, 5.0, 1.0, 1, path=2)
    assert ei.value.status == 8


def test_sweep_large_network_auto_runs_thread_path(S):
    """A network past the thread path's AUTO threshold (R = 192 > 160): the sweep still runs on the
    thread path under AUTO, and each point equals ssa_run on the thread path bitwise."""
    net = inputs.synthetic(48, 192, seed=9)
    base = np.array([r.rate for r in net.reactions])
    rates = np.stack([base, base * 0.5])
    N, t_end, dt, seed = 96, 0.2, 0.05, 5
    m = S.Model(net)
    sw = S.run_sweep(m, rates, N, t_end, dt, seed)
    assert sw.status == 0 and sw.path_used == 1
    for p in range(2):
        one = S.run(S.Model(inputs.with_rates(net, rates[p])), N, t_end, dt, seed, path=1)
        assert np.array_equal(sw.mean[p], one.mean) and np.array_equal(sw.var[p], one.var)


def test_sweep_rerun_costliest_first_is_bitwise(S):
    """The first run of a sweep records each point's events per trajectory; a re-run hands out the
    costliest point's trajectories first.  Scheduling never changes results: grids, counters and
    dumps are bitwise those of the first run."""
    net = inputs.immigration_death()
    rates = inputs.rate_matrix(net, [0], [2.0, 40.0, 10.0])     # immigration 2 / 40 / 10: unequal costs
    N, t_end, dt, seed = 3000, 20.0, 0.5, 13
    ids = np.array([0, 1, 2999, 3000, 4500, 8999], dtype=np.uint64)
    m = S.Model(net)
    a = S.run_sweep(m, rates, N, t_end, dt, seed, dump_ids=ids)
    b = S.run_sweep(m, rates, N, t_end, dt, seed, dump_ids=ids)
    assert a.events == b.events
    assert np.array_equal(a.mean, b.mean) and np.array_equal(a.var, b.var)
    for f in ("states", "events_at", "time_at"):
        assert np.array_equal(getattr(a.dump, f), getattr(b.dump, f)), f
    assert a.dump.summary.tobytes() == b.dump.summary.tobytes()

