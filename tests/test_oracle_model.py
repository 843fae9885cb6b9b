"""Oracle pins for a3 (propensities), a4/a7 (total + selection), a5 (step),
a6 (grid alignment) and the moment finalize, against printed SPEC values,
hand-derived goldens and exact rational arithmetic."""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import inputs
from inputs.networks import Network, _rx

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ------------------------------------------------------------------ a3
def test_propensity_printed_values(oracle_lib):
    O = oracle_lib
    g = gold("spec_propensity.json")
    m = O.OracleModel(inputs.hiv())
    st, a, _ = O.propensities(m, m.x0)
    assert st == 0
    assert a[7] == g["hiv_x0_a8"]          # reaction 8: beta * T * V5 = 4e-5*1000*100
    assert a[0] == g["hiv_x0_a1"]          # reaction 1: lambda * U0
    # beta_R5 = max(0, beta - K F): isolate k^ with T = V5 = 1
    x = np.zeros(10, np.int64)
    x[2] = 1; x[8] = 1; x[9] = 1000
    assert O.propensities(m, x)[1][7] == g["beta_R5_F1000"]
    x[9] = 250
    k = O.propensities(m, x)[1][7]
    # cancellation: error is a few ulps of beta (the larger operand)
    assert abs(k - g["beta_R5_F250"]) <= 2 * np.spacing(4e-5)
    # beta_X4 = beta + K F increases
    x[7] = 1
    assert O.propensities(m, x)[1][8] > 4e-5


def test_propensity_gated_variant_b(oracle_lib):
    """SPEC.md:424 Variant B: a_18 = mu * step(V5) * (1 - step(V4)) -- exactly mu
    while V5 > 0 and V4 == 0, whatever V5, else exactly 0; every other
    reaction is unchanged from Variant A."""
    O = oracle_lib
    mb, ma = O.OracleModel(inputs.hiv("B")), O.OracleModel(inputs.hiv("A"))
    x = np.array(mb.x0)
    for v5, v4, want in ((100, 0, 2.5e-3), (1, 0, 2.5e-3), (7, 1, 0.0), (0, 0, 0.0), (0, 3, 0.0)):
        x[8], x[7] = v5, v4
        st, a, _ = O.propensities(mb, x)
        assert st == 0 and a[17] == want
        _, aa, _ = O.propensities(ma, x)
        assert aa[17] == 2.5e-3 * v5                        # Variant A: mass action mu * V5
        assert np.array_equal(np.delete(a, 17), np.delete(aa, 17))


def test_propensity_combinatorial_factor(oracle_lib):
    """C(x,2) (unordered pairs, R1): 2 S1 -> S2 at S1=1000 has
    h = 499500; with c2 = 0.002 the product is 999 up to one rounding."""
    O = oracle_lib
    net = inputs.dimerization()
    m = O.OracleModel(net)
    st, a, _ = O.propensities(m, [1000, 0, 0])
    assert a[1] == 0.002 * 499500.0
    assert abs(a[1] - 999.0) <= np.spacing(999.0)
    # exact factors with unit rates: C(x,1), C(x,2), C(x,3), products
    net2 = Network(("A", "B"), (0, 0), (
        _rx([(0, 1)], [], 1.0), _rx([(0, 2)], [], 1.0), _rx([(0, 3)], [], 1.0),
        _rx([(0, 2), (1, 1)], [], 1.0), _rx([], [(0, 1)], 2.5)))
    m2 = O.OracleModel(net2)
    for xa in range(0, 40):
        for xb in (0, 1, 7):
            a = O.propensities(m2, [xa, xb])[1]
            assert a[0] == xa
            assert a[1] == math.comb(xa, 2)
            assert a[2] == math.comb(xa, 3)
            assert a[3] == math.comb(xa, 2) * xb
            assert a[4] == 2.5


def test_propensity_nonfinite_is_error(oracle_lib):
    O = oracle_lib
    net = Network(("A",), (5,), (_rx([(0, 1)], [], 1.0), _rx([(0, 1)], [], float("inf"))))
    st, _, bad = O.propensities(O.OracleModel(net), [5])
    assert st == 3 and bad == 1


# ------------------------------------------------------------------ a4/a5/a7
def test_step_worked_example(oracle_lib):
    O = oracle_lib
    g = gold("spec_step.json")
    net = Network(("X",), (1,), (_rx([(0, 1)], [(0, 1)], g["a"][0]), _rx([(0, 1)], [(0, 1)], g["a"][1])))
    m = O.OracleModel(net)
    u1 = math.exp(-g["u1_is_exp_minus"])
    for mode in (0, 1):
        st, tau, j = O.step(m, [1], u1, g["u2"], mode)
        assert st == 0 and j == g["j0"]
        assert abs(tau - g["tau"]) <= 4 * np.spacing(g["tau"])   # plog is within 2 ulp of ln
    # all-zero -> exhausted
    st, tau, j = O.step(m, [0], 0.5, 0.5)
    assert j == -1 and math.isinf(tau)
    # single reaction -> index 0 for any u2
    single = O.OracleModel(Network(("X",), (1,), (_rx([], [(0, 1)], 5.0),)))
    for u2 in (2.0**-53, 0.3, 1 - 2.0**-53):
        assert O.step(single, [0], 0.5, u2)[2] == 0


def _exact_select(a, u2):
    """Smallest j with exact prefix > u2 * exact total."""
    fa = [Fraction(v) for v in a]
    r = Fraction(u2) * sum(fa)
    c = Fraction(0)
    for j, v in enumerate(fa):
        c += v
        if c > r:
            return j, r, fa
    return -1, r, fa


@pytest.mark.parametrize("R", [1, 2, 5, 27, 32, 33, 64, 100, 256])
def test_selection_matches_exact_arithmetic(oracle_lib, R):
    """Both declared summation orders select the exact-arithmetic reaction,
    except when u2*a0 is within rounding of a prefix boundary; never a zero
    propensity."""
    O = oracle_lib
    rng = np.random.default_rng(R)
    mismatches = 0
    for trial in range(300):
        a = rng.exponential(1.0, R) * np.exp(rng.uniform(-8, 8, R))
        a[rng.random(R) < 0.3] = 0.0
        if trial % 7 == 0:
            a[:] = 0.0
            a[rng.integers(0, R)] = 1.0
        if not np.any(a > 0):
            a[0] = 1.0
        u2 = O.u53(int(rng.integers(0, 2**63)) * 2 + 1)
        jx, r, fa = _exact_select(a, u2)
        for mode in (0, 1, 2, 3):     # sequential, warp32, warp16, warp16 with a scanned lane step
            a0, j = O.select(a, mode, u2)
            assert abs(a0 - float(sum(fa))) <= R * np.spacing(float(sum(fa)))
            assert 0 <= j < R and a[j] > 0
            if j != jx:
                # only allowed when r is within a few ulps of a prefix boundary
                bound = sum(fa[:min(j, jx) + 1])
                assert abs(bound - r) <= Fraction(4 * R) * Fraction(np.spacing(float(sum(fa)))), (R, trial, j, jx)
                mismatches += 1
    assert mismatches <= 5


def test_frozen_state_statistics(oracle_lib):
    """mean tau within 1% of 1/a0, selection frequencies within
    3 sigma over 1e5 draws; uniforms from the Philox stream of one trajectory."""
    O = oracle_lib
    a = np.array([1.0, 3.0, 0.0, 6.0])
    net = Network(("X",), (1,), tuple(_rx([(0, 1)], [(0, 1)], v) for v in a))
    m = O.OracleModel(net)
    n = 100_000
    ctr = np.zeros((n, 4), np.uint32)
    ctr[:, 0] = np.arange(n, dtype=np.uint32)
    ctr[:, 2] = 17
    o = O.philox_n(ctr, (42, 0)).astype(np.uint64)
    u1 = O.u53_n((o[:, 1] << np.uint64(32)) | o[:, 0])
    u2 = O.u53_n((o[:, 3] << np.uint64(32)) | o[:, 2])
    taus = np.zeros(n)
    js = np.zeros(n, np.int64)
    for i in range(n):
        _, taus[i], js[i] = O.step(m, [1], u1[i], u2[i])
    a0 = a.sum()
    assert abs(taus.mean() * a0 - 1) < 0.01
    for j, aj in enumerate(a):
        p = aj / a0
        cnt = np.sum(js == j)
        assert abs(cnt - n * p) <= 3 * math.sqrt(n * p * (1 - p)) + 1e-9, (j, cnt)


# ------------------------------------------------------------------ a6
def test_grid_alignment_spec_example(oracle_lib):
    O = oracle_lib
    g = gold("spec_align_k2.json")
    assert O.grid_size(g["t_end"], g["dt"]) == len(g["grid_times"])
    held = []
    for s in g["streams"]:
        times = [ev[0] for ev in s["events"]]
        states = np.array([ev[1] for ev in s["events"]], np.int64)
        gx, ge, gt, _ = O.align_events(s["x0"], times, states, g["t_end"], g["dt"])
        held.append(gx[:, 0].tolist())
    assert held == g["held"]
    mean, var = O.moments(np.array(held, np.int32).reshape(2, -1))
    assert mean.tolist() == g["mean"]
    assert var.tolist() == g["var_population"]


def test_grid_alignment_edge_cases(oracle_lib):
    O = oracle_lib
    # no events: held x0 everywhere
    gx, ge, gt, nt = O.align_events([7], [], np.zeros((0, 1)), 10.0, 2.5)
    assert gx[:, 0].tolist() == [7] * 5 and ge.tolist() == [0] * 5
    # an event just after, exactly at, and just before a grid point
    dt = 0.1
    s3 = 3 * 0.1
    times = [np.nextafter(s3, 0), s3, np.nextafter(s3, 1)]
    gx, ge, gt, nt = O.align_events([0], times, np.array([[1], [2], [3]]), 0.5, dt)
    assert gx[:, 0].tolist() == [0, 0, 0, 2, 3, 3]
    assert ge.tolist() == [0, 0, 0, 2, 3, 3]
    assert gt[3] == s3
    assert nt >= 1   # near ties within 1e-9 relative are counted
    # K = floor(t_end/dt + 1e-9): 0.3/0.1 = 2.9999999999999996 -> K = 3
    assert O.grid_size(0.3, 0.1) == 4
    assert O.grid_size(100.0, 1.0) == 101
    assert O.grid_size(20.0, 0.1) == 201
    assert O.grid_size(10.0, 0.05) == 201
    assert O.grid_size(400.0, 1.0) == 401


def test_near_tie_counter_constructed_streams(oracle_lib):
    """The near-tie counter (north_star: "any trajectory whose event time lies
    within 1e-9 relative of a sample time flagged and counted"; R22)
    on event streams with known counts.  It counts grid points, not
    trajectories: a crossing of s_k is flagged when the candidate that crosses
    it or the last applied event lies within 1e-9 * s_k of s_k, once per grid
    point.  Each case pins one reading against its plausible misreadings
    (per trajectory instead of per grid point, an absolute 1e-9 tolerance,
    counting only the candidate or only the applied event, counting a point
    twice)."""
    O = oracle_lib

    def ties(times, t_end, dt):
        n = len(times)
        states = np.arange(1, n + 1, dtype=np.int64).reshape(n, 1)
        _, _, _, nt = O.align_events([0], times, states, t_end, dt)
        return int(nt)

    # relative: 5e-10 s_k away is near, 2e-9 s_k away is not (both sides of s_k)
    assert ties([2.0 * (1 + 5e-10), 4.5], 5.0, 1.0) == 1            # candidate just past s_2
    assert ties([2.0 * (1 - 5e-10), 4.5], 5.0, 1.0) == 1            # applied event just before s_2
    assert ties([2.0 * (1 + 2e-9), 4.5], 5.0, 1.0) == 0
    assert ties([2.0 * (1 - 2e-9), 4.5], 5.0, 1.0) == 0
    # an event exactly at s_k is applied (right-continuous hold) and flagged when s_k is crossed
    assert ties([3.0, 4.5], 5.0, 1.0) == 1
    # per grid point: three near ties in one trajectory count 3 (a per-trajectory flag gives 1)
    assert ties([1.0 * (1 + 4e-10), 2.0 * (1 - 4e-10), 2.5, 4.0, 4.7], 5.0, 1.0) == 3
    # applied event and candidate both near the same s_k: one flag for that grid point, not two
    assert ties([5.0 * (1 - 3e-10), 5.0 * (1 + 3e-10)], 5.0, 1.0) == 1
    # relative, not absolute: at s_k = 1000 an offset of 5e-7 (5e-10 relative) is near ...
    assert ties([1000.0 + 5e-7, 2500.0], 3000.0, 1000.0) == 1
    # ... and at s_k = 1e-3 an offset of 5e-10 (5e-7 relative) is not
    assert ties([1e-3 + 5e-10, 2.5e-3], 3e-3, 1e-3) == 0
    # s_0 = 0 is never a near tie (tolerance 0 and no applied event), nor the hold after the last event
    assert ties([1e-300, 0.5], 1.0, 1.0) == 0
    assert ties([], 5.0, 1.0) == 0
    # a candidate that crosses several grid points is compared with each of them
    assert ties([0.5, 3.0 * (1 + 1e-10)], 5.0, 1.0) == 1


# ------------------------------------------------------------------ moments
def test_moments_printed_example(oracle_lib):
    O = oracle_lib
    g = gold("spec_moments.json")
    mean, var = O.moments(np.array(g["samples"], np.int32).reshape(-1, 1))
    assert mean[0] == float(Fraction(g["mean_num"], g["mean_den"]))
    assert var[0] == float(Fraction(g["var_num"], g["var_den"]))


def test_moments_exact_large_values(oracle_lib):
    O = oracle_lib
    rng = np.random.default_rng(3)
    x = rng.integers(0, 2**31 - 1, size=(5000, 3)).astype(np.int32)
    x[:, 2] = 2**31 - 1   # constant column -> variance exactly 0
    mean, var = O.moments(x)
    for c in range(3):
        col = [int(v) for v in x[:, c]]
        n = len(col)
        s1, s2 = sum(col), sum(v * v for v in col)
        assert abs(mean[c] - float(Fraction(s1, n))) <= np.spacing(float(Fraction(s1, n)))
        ev = Fraction(n * s2 - s1 * s1, n * n)
        assert abs(var[c] - float(ev)) <= 2 * np.spacing(max(float(ev), 1e-300))
    assert var[2] == 0.0 and mean[2] == 2**31 - 1


# ------------------------------------------------------------------ union-time selective memory (NEXT 2)
def test_union_reduce_spec_example(oracle_lib):
    """SPEC.md:250-262 worked example of Y-alignment at union times and of
    X-reduction of k_x successive Y-points (golden file, with citation)."""
    O = oracle_lib
    g = gold("spec_union_k2.json")
    streams = [(np.array(s["times"]), np.array(s["states"], np.int64)) for s in g["streams"]]
    for key, kx in (("kx1", 1), ("kx2", 2)):
        t, mean, var, n = O.union_reduce(streams, kx)
        want = g[key]
        assert np.allclose(t, want["times"], rtol=0, atol=1e-15)
        assert np.array_equal(mean[:, 0], want["mean"]) and np.array_equal(var[:, 0], want["var"])
        assert list(n) == want["n"]


def test_union_reduce_identity_and_streams(oracle_lib):
    """k = 1, k_x = 1 is the identity: the output is the
    stream's own points; and a stream built from the event list replays the
    grid states the trajectory oracle reports (zero-order hold at s_k)."""
    O = oracle_lib
    net = inputs.dimerization(50)
    m = O.OracleModel(net)
    t, x = O.stream(m, 3, 2, 4.0)
    assert t[0] == 0.0 and t[-1] == 4.0 and np.all(np.diff(t) > 0)
    ut, mean, var, n = O.union_reduce([(t, x)], 1)
    assert np.array_equal(ut, t) and np.array_equal(mean, x.astype(float)) and np.all(var == 0)
    tr = O.trajectory(m, 3, 2, 4.0, 0.5)
    sk = np.arange(9) * 0.5
    held = x[np.searchsorted(t, sk, side="right") - 1]
    assert np.array_equal(held, tr.grid_x)
    assert tr.summary["events"] in (len(t) - 2, len(t) - 1)   # horizon point appended unless an event is at t_end


# ------------------------------------------------------------------ stride-sampled output (NEXT 4)
def test_stride_points_definition(oracle_lib):
    """SPEC.md:162/:184 Stride(s): first and last points always; every s-th
    event in between; the empty network gives exactly (0, x0), (t_end, x0);
    stride 1 is the full point stream."""
    O = oracle_lib
    k, t, x = O.stride_points(O.OracleModel(inputs.empty_network((7,))), 0, 1, 10.0, 10)
    assert list(k) == [0, 0] and list(t) == [0.0, 10.0] and np.all(x == 7)
    m = O.OracleModel(inputs.immigration_death())
    ts, xs = O.stream(m, 2, 1, 6.0)
    k1, t1, x1 = O.stride_points(m, 2, 1, 6.0, 1)
    assert np.array_equal(t1, ts) and np.array_equal(x1, xs)
    k10, t10, x10 = O.stride_points(m, 2, 1, 6.0, 10)
    E = int(k1[-1])
    assert list(k10[1:-1]) == list(range(10, E + 1, 10))
    assert np.array_equal(t10[1:-1], t1[10:E + 1:10]) and np.array_equal(x10[1:-1], x1[10:E + 1:10])
    assert t10[-1] == 6.0 and np.array_equal(x10[-1], x1[-1])
