"""Distributional pins of the oracle's trajectories (PAPER.md:60 'exactly
according to the given probability distributions'): closed forms, the chemical
master equation by matrix exponential on finite state spaces, and structural
invariants of the HIV network (Table 1)."""
import math

import numpy as np
import pytest
import scipy.linalg

import inputs
from inputs.networks import Network, _rx

Z = 4.0


def _zmean(m, mu, var, n):
    if var < 1e-12:   # a point mass (CME moments carry rounding of order 1e-16)
        return 0.0 if abs(m - mu) < 1e-9 else np.inf
    return abs(m - mu) / math.sqrt(var / n)


def _zvar(v, var, mu4, n):
    # var of the sample (population) variance ~ (mu4 - sigma^4)/n
    d = mu4 - var * var
    if d <= 1e-24:    # a point mass
        return 0.0 if abs(v - var) < 1e-12 else np.inf
    return abs(v - var) / math.sqrt(d / n)


def test_immigration_death_config0_closed_form(oracle_lib):
    """BASELINE.json configs[0]: X(t) ~ Poisson(100 (1 - e^{-0.1 t})) from X0 = 0."""
    O = oracle_lib
    cfg = inputs.config(0)
    m = O.OracleModel(cfg.network)
    res = O.run(m, np.arange(cfg.n_trajectories), cfg.seed, cfg.t_end, cfg.dt, keep=False)
    assert res.status == 0
    G = O.grid_size(cfg.t_end, cfg.dt)
    n = cfg.n_trajectories
    assert res.mean[0, 0] == 0 and res.var[0, 0] == 0
    for k in range(1, G):
        t = k * cfg.dt
        lam = 100.0 * (1 - math.exp(-0.1 * t))
        assert _zmean(res.mean[k, 0], lam, lam, n) < Z, k
        assert _zvar(res.var[k, 0], lam, lam + 3 * lam * lam, n) < Z, k


def test_immigration_death_spec_acceptance4(oracle_lib):
    """SPEC.md:186 / :450: lambda=10, delta=1, 1000 trajectories, t=20:
    mean in [9.7, 10.3], variance in [8.5, 11.5]."""
    O = oracle_lib
    m = O.OracleModel(inputs.immigration_death(10.0, 1.0, 0))
    res = O.run(m, np.arange(1000), 11, 20.0, 20.0, keep=False)
    assert 9.7 <= res.mean[-1, 0] <= 10.3
    assert 8.5 <= res.var[-1, 0] <= 11.5


def test_pure_death_binomial(oracle_lib):
    """X -> 0 at rate k: X(t) ~ Binomial(X0, e^{-k t}); every event removes one."""
    O = oracle_lib
    x0, k, n = 10, 1.0, 20000
    m = O.OracleModel(inputs.pure_death(k, x0))
    res = O.run(m, np.arange(n), 5, 2.0, 0.25)
    gx = res.grid_x[:, :, 0]
    assert np.all(np.diff(gx, axis=1) <= 0)
    assert np.all(res.grid_e[:, :] == (x0 - gx))           # one molecule per event
    assert np.all(res.summaries["absorbed"][gx[:, -1] == 0] == 1)
    for kk in range(res.mean.shape[0]):
        t = kk * 0.25
        p = math.exp(-k * t)
        mu, var = x0 * p, x0 * p * (1 - p)
        mu4 = x0 * p * (1 - p) * (1 + 3 * (x0 - 2) * p * (1 - p))   # binomial 4th central moment
        assert _zmean(res.mean[kk, 0], mu, var, n) < Z
        assert _zvar(res.var[kk, 0], var, mu4, n) < Z


def test_empty_network_holds_state(oracle_lib):
    O = oracle_lib
    m = O.OracleModel(inputs.empty_network((7, 0, 3)))
    tr = O.trajectory(m, 0, 1, 10.0, 1.0)
    assert np.all(tr.grid_x == np.array([7, 0, 3]))
    assert tr.summary["events"] == 0 and tr.summary["absorbed"] == 1


# ---------------------------------------------------------------- CME pins
def _cme_network():
    """A closed (finite) network exercising C(x,2), C(x,3), both modifier
    signs and the clamp at 0 (PAPER.md:93 '0 <= beta_R5 <= beta')."""
    A, B, Cc, P, F, D, E = range(7)
    return Network(("A", "B", "C", "P", "F", "D", "E"), (5, 4, 0, 3, 0, 0, 0), (
        _rx([(A, 1), (B, 1)], [(Cc, 1)], 0.3, "A+B->C (k - 0.1 F)", (F, -0.1)),
        _rx([(Cc, 1)], [(A, 1), (B, 1)], 0.5, "C->A+B"),
        _rx([(P, 1)], [(F, 1)], 1.0, "P->F"),
        _rx([(F, 1)], [(P, 1)], 0.5, "F->P"),
        _rx([(A, 2)], [(D, 1)], 0.05, "2A->D (k + 0.02 F)", (F, +0.02)),
        _rx([(D, 1)], [(A, 2)], 0.4, "D->2A"),
        _rx([(B, 3)], [(E, 1)], 0.01, "3B->E"),
        _rx([(E, 1)], [(B, 3)], 0.3, "E->3B"),
    ))


def _cme_moments(net, times):
    """Enumerate the reachable states by BFS, build the CTMC generator with
    propensities written from their definition (math.comb), and return the
    mean and variance of each species at each time via expm."""
    def props(x):
        out = []
        for rx in net.reactions:
            h = 1
            for sp, mm in rx.reactants:
                h *= math.comb(x[sp], mm)
            k = rx.rate
            if rx.modifier_species >= 0:
                k = max(0.0, k + rx.modifier_coef * x[rx.modifier_species])
            out.append(k * h)
        return out

    def apply(x, rx):
        y = list(x)
        for sp, mm in rx.reactants:
            y[sp] -= mm
        for sp, mm in rx.products:
            y[sp] += mm
        return tuple(y)

    x0 = tuple(net.x0)
    index = {x0: 0}
    states = [x0]
    q = [x0]
    while q:
        x = q.pop()
        for rx, a in zip(net.reactions, props(x)):
            if a > 0:
                y = apply(x, rx)
                if y not in index:
                    index[y] = len(states)
                    states.append(y)
                    q.append(y)
    n = len(states)
    Q = np.zeros((n, n))
    for i, x in enumerate(states):
        for rx, a in zip(net.reactions, props(x)):
            if a > 0:
                Q[i, index[apply(x, rx)]] += a
                Q[i, i] -= a
    X = np.array(states, dtype=np.float64)
    p0 = np.zeros(n)
    p0[0] = 1.0
    out = []
    for t in times:
        p = p0 @ scipy.linalg.expm(Q * t)
        assert abs(p.sum() - 1) < 1e-9
        mu = p @ X
        var = p @ (X - mu) ** 2
        mu4 = p @ (X - mu) ** 4
        out.append((mu, var, mu4))
    return out, n


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_cme_closed_network(oracle_lib, mode):
    O = oracle_lib
    net = _cme_network()
    t_end, dt, n = 3.0, 0.5, 20000
    times = [k * dt for k in range(int(t_end / dt) + 1)]
    ref, nstates = _cme_moments(net, times)
    assert nstates > 50
    res = O.run(O.OracleModel(net), np.arange(n), 99 + mode, t_end, dt, mode, keep=False)
    assert res.status == 0
    for k, (mu, var, mu4) in enumerate(ref):
        for s in range(net.S):
            assert _zmean(res.mean[k, s], mu[s], var[s], n) < Z, (k, s)
            assert _zvar(res.var[k, s], var[s], mu4[s], n) < Z, (k, s)


def test_cme_dimerization_pins_binomial_factor(oracle_lib):
    """Config-1 reaction types with S1(0)=12 (a 140-state chain): the C(x,2)
    convention is pinned -- the ordered x(x-1) reading doubles the
    dimerisation rate and fails these z-tests."""
    O = oracle_lib
    net = inputs.dimerization(12, c=(0.2, 0.1, 0.5, 0.04))
    t_end, dt, n = 4.0, 0.5, 20000
    times = [k * dt for k in range(int(t_end / dt) + 1)]
    ref, nstates = _cme_moments(net, times)
    res = O.run(O.OracleModel(net), np.arange(n), 7, t_end, dt, keep=False)
    for k, (mu, var, mu4) in enumerate(ref):
        for s in range(3):
            assert _zmean(res.mean[k, s], mu[s], var[s], n) < Z, (k, s)
            assert _zvar(res.var[k, s], var[s], mu4[s], n) < Z, (k, s)
    # the alternative (ordered-pairs) reading is rejected by the same data
    alt = inputs.dimerization(12, c=(0.2, 0.2, 0.5, 0.04))
    ref_alt, _ = _cme_moments(alt, times)
    worst = max(_zmean(res.mean[k, 1], ref_alt[k][0][1], ref_alt[k][1][1], n) for k in range(1, len(times)))
    assert worst > 10


# ---------------------------------------------------------------- HIV
def test_hiv_structure_and_event_rate(oracle_lib):
    """Table 1 invariants: U0 is a catalyst (U0 == 1 always); F is never
    consumed (nondecreasing); counts stay >= 0.  Event-rate calibration:
    ~150M simulation points per 4000 days = 3.75e6 per 100 d."""
    O = oracle_lib
    cfg = inputs.config(2)
    m = O.OracleModel(cfg.network)
    res = O.run(m, np.arange(2), cfg.seed, cfg.t_end, cfg.dt)
    assert res.status == 0
    gx = res.grid_x
    assert np.all(gx[:, :, 0] == 1)
    assert np.all(np.diff(gx[:, :, 9], axis=1) >= 0)
    assert np.all(gx >= 0)
    assert np.all(res.var[:, 0] == 0) and np.all(res.mean[:, 0] == 1)
    ev = res.summaries["events"].astype(float)
    assert np.all(np.abs(ev / 3.75e6 - 1) < 0.2), ev
    assert np.all(np.diff(res.grid_e, axis=1) >= 0)
    assert np.all(res.grid_e[:, -1] == res.summaries["events"])


def test_determinism_and_independence(oracle_lib):
    O = oracle_lib
    m = O.OracleModel(inputs.dimerization())
    a = O.trajectory(m, 5, 2, 20.0, 0.1)
    b = O.trajectory(m, 5, 2, 20.0, 0.1)
    c = O.trajectory(m, 6, 2, 20.0, 0.1)
    d = O.trajectory(m, 5, 3, 20.0, 0.1)
    assert a.summary == b.summary and np.array_equal(a.grid_x, b.grid_x)
    assert a.summary["hash"] != c.summary["hash"] and a.summary["hash"] != d.summary["hash"]
    # the grid times of the last applied event are bounded by the grid
    G = a.grid_t.shape[0]
    assert np.all(a.grid_t <= np.arange(G) * 0.1 + 1e-15)


# ---------------------------------------------------------------- gated propensities (NEXT 3)
def test_gate_zero_one_shot_event_closed_form(oracle_lib):
    """0 -> M at rate mu with the gate [M == 0] (SPEC.md:424's 1-step(x)):
    exactly one event, at an Exp(mu) time, so M(t) is Bernoulli with
    p(t) = 1 - exp(-mu t) and never exceeds 1."""
    O = oracle_lib
    mu, n = 0.3, 4000
    net = Network(("M",), (0,), (_rx([], [(0, 1)], mu, gates=[(0, inputs.GATE_ZERO)]),))
    res = O.run(O.OracleModel(net), np.arange(n), 21, 10.0, 0.5)
    assert res.status == 0
    assert set(np.unique(res.grid_x)) <= {0, 1}
    assert np.all(res.summaries["events"] <= 1)
    for k in range(res.mean.shape[0]):
        p = 1.0 - math.exp(-mu * 0.5 * k)
        assert _zmean(res.mean[k, 0], p, p * (1 - p), n) < Z
        assert abs(res.var[k, 0] - res.mean[k, 0] * (1 - res.mean[k, 0])) < 1e-12


def test_gate_positive_constant_rate_closed_form(oracle_lib):
    """A -> 0 with mass_action off (h = 1) and the gate [A > 0] (step(A)):
    A falls by one at constant rate k while positive, so A(t) =
    max(0, A0 - N_t) with N_t ~ Poisson(k t)."""
    O = oracle_lib
    k, A0, n = 2.0, 10, 3000
    net = Network(("A",), (A0,), (_rx([(0, 1)], [], k, mass_action=False, gates=[(0, inputs.GATE_POSITIVE)]),))
    res = O.run(O.OracleModel(net), np.arange(n), 22, 8.0, 0.5)
    assert res.status == 0 and np.all(res.grid_x >= 0)
    for kk in range(res.mean.shape[0]):
        lam = k * 0.5 * kk
        pm = [math.exp(-lam) * lam ** i / math.factorial(i) for i in range(A0)]
        m1 = sum((A0 - i) * p for i, p in enumerate(pm))
        m2 = sum((A0 - i) ** 2 * p for i, p in enumerate(pm))
        assert _zmean(res.mean[kk, 0], m1, m2 - m1 * m1, n) < Z
    # absorbing once A = 0 (the only reaction's gate closes)
    assert np.all(res.summaries["events"] <= A0)


def test_hiv_variant_b_structure(oracle_lib):
    """HIV Variant B (PAPER.md:95 time-triggered mutation): the
    gated reaction 18 can fire only while V5 > 0 and no V4 exists (it re-arms
    if V4 dies out), at rate mu, whatever the V5 count.  With mu = 0 no V4 ever
    appears; with mu raised to 0.5/day mutations happen; Table 1's structural
    invariants hold in both."""
    O = oracle_lib
    for mu, expect_v4 in ((0.0, False), (0.5, True)):
        res = O.run(O.OracleModel(inputs.hiv("B", mu=mu)), np.arange(64), 23, 2.0, 0.25)
        assert res.status == 0
        gx = res.grid_x
        assert np.all(gx[:, :, 0] == 1) and np.all(gx >= 0)
        assert np.all(np.diff(gx[:, :, 9], axis=1) >= 0)
        assert np.all(gx[:, 0, 7] == 0)
        assert bool(np.any(gx[:, :, 7] > 0)) == expect_v4


def test_hiv_linear_subnetwork_closed_form(oracle_lib):
    """HIV network (Table 1) with the infection, mutation and infectivity rates set to
    zero (beta = gamma = mu = K = 0): no cell is infected, so I4 = I5 = V4 = F = 0 and what remains is
    first order -- U0 -> U0 + U (lambda), U -> T (d_ut), U -> Z4 and U -> Z5 (d_uz each), T, Z4, Z5
    and V5 clearance.  For a first-order network the means solve the linear rate equations exactly:
      U(t)  = A + B e^{-a t},  a = d_ut + 2 d_uz, A = lambda / a, B = U(0) - A
      T(t)  = T0 e^{-d_t t} + d_ut [A (1 - e^{-d_t t}) / d_t + B (e^{-a t} - e^{-d_t t}) / (d_t - a)]
      Zi(t) = Z0 e^{-d_z t} + d_uz [A (1 - e^{-d_z t}) / d_z + B (e^{-a t} - e^{-d_z t}) / (d_z - a)]
    and V5 is a pure death: Binomial(100, e^{-d_v t}).  Pins the oracle's reading of Table 1's
    reaction list (which species each reaction consumes and produces, and at which rate)."""
    O = oracle_lib
    p = inputs.networks.HIV_PARAMS
    net = inputs.hiv(beta=0.0, gamma=0.0, mu=0.0, K=0.0)
    n, t_end = 2000, 20.0
    res = O.run(O.OracleModel(net), np.arange(n), 3, t_end, 1.0, keep=False)
    assert res.status == 0
    lam, d_ut, d_uz, d_t, d_z, d_v = p["lam"], p["d_ut"], p["d_uz"], p["d_t"], p["d_z"], p["d_v"]
    x0 = net.x0
    a = d_ut + 2 * d_uz
    A = lam / a
    B = x0[1] - A

    def conv(rate_in, d, y0, t):
        return y0 * math.exp(-d * t) + rate_in * (A * (1 - math.exp(-d * t)) / d
                                                  + B * (math.exp(-a * t) - math.exp(-d * t)) / (d - a))

    for k in range(1, int(t_end) + 1):
        t = float(k)
        mu = {1: A + B * math.exp(-a * t), 2: conv(d_ut, d_t, x0[2], t),
              3: conv(d_uz, d_z, x0[3], t), 4: conv(d_uz, d_z, x0[4], t)}
        for s, m_s in mu.items():
            assert _zmean(res.mean[k, s], m_s, res.var[k, s], n) < 4.5, (k, s, res.mean[k, s], m_s)
        q = math.exp(-d_v * t)
        v5 = 100 * q
        assert _zmean(res.mean[k, 8], v5, 100 * q * (1 - q), n) < 4.5, (k, res.mean[k, 8], v5)
        for s in (5, 6, 7, 9):
            assert res.mean[k, s] == 0 and res.var[k, s] == 0
        assert res.mean[k, 0] == 1 and res.var[k, 0] == 0


def _mini_hiv(swap_modifier_signs: bool = False):
    """Table 1's reaction list on a finite state space: immigration (lambda), the bursts (pi) and the
    productions that need no consumption (s1, s2, s3) off, F held at 2 so the infectivity modifiers
    (d = -K on reactions 8 and 10, +K on 9 and 11) and the F-catalysed clearances
    (reactions 2 and 7) are active; rates raised so every reaction fires within a few time units."""
    p = dict(lam=0.0, d_uf=0.3, d_ut=0.5, d_uz=0.2, d_t=0.1, d_tf=0.2, beta=0.6, K=0.1, gamma=0.4,
             s1=0.0, s2=0.0, d_iz=0.5, mu=0.3, pi=0.0, s3=0.0, d_z=0.1, d_v=0.3)
    net = inputs.hiv(**p)
    rx = list(net.reactions)
    if swap_modifier_signs:
        from inputs.networks import Reaction
        for j in (7, 8, 9, 10):
            r = rx[j]
            rx[j] = Reaction(r.reactants, r.products, r.rate, r.modifier_species, -r.modifier_coef, r.name,
                             r.mass_action, r.gates)
    return Network(net.species, (1, 2, 2, 1, 1, 0, 0, 0, 2, 2), tuple(rx), "mini-hiv")


def test_cme_mini_hiv_reaction_list(oracle_lib):
    """The HIV reaction list (incl. the bimolecular infections, the I+Z clearances, the mutation and
    the signed infectivity modifiers) against the chemical master equation on its 1155 reachable
    states; the opposite modifier signs are rejected by the same data."""
    O = oracle_lib
    net = _mini_hiv()
    t_end, dt, n = 3.0, 0.5, 20000
    times = [k * dt for k in range(int(t_end / dt) + 1)]
    ref, nstates = _cme_moments(net, times)
    assert nstates == 1155
    res = O.run(O.OracleModel(net), np.arange(n), 21, t_end, dt, keep=False)
    assert res.status == 0
    for k, (mu, var, mu4) in enumerate(ref):
        for s in range(net.S):
            assert _zmean(res.mean[k, s], mu[s], var[s], n) < Z, (k, s)
            assert _zvar(res.var[k, s], var[s], mu4[s], n) < Z, (k, s)
    ref_alt, _ = _cme_moments(_mini_hiv(swap_modifier_signs=True), times)
    worst = max(_zmean(res.mean[k, s], ref_alt[k][0][s], ref_alt[k][1][s], n)
                for k in range(1, len(times)) for s in (5, 6))
    assert worst > 10, worst
