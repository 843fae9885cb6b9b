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


@pytest.mark.parametrize("mode", [0, 1, 2, 3])
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


def _linear_moments(net, times):
    """Exact mean and covariance of a network whose propensities are affine in
    the counts (zero- and first-order reactions, coefficient 1), written from
    the reaction list alone: with a_j(x) = c_j + w_j.x and net change nu_j,
      m'     = J m + nu c,                     J = sum_j nu_j w_j^T
      Sigma' = J Sigma + Sigma J^T + sum_j nu_j nu_j^T (c_j + w_j.m)
    (the moment equations of a linear network close exactly).  Solved as one
    linear system z' = M z on z = [m, vec(Sigma), 1] with expm(M t) from
    m = x0, Sigma = 0.  Returns [(mean[S], var[S])] per time."""
    S, R = net.S, net.R
    nu = np.zeros((S, R)); c = np.zeros(R); W = np.zeros((R, S))
    for j, rx in enumerate(net.reactions):
        if rx.rate == 0.0 and rx.modifier_coef == 0.0:
            continue                                    # a switched-off reaction never fires
        assert rx.modifier_species < 0 and rx.mass_action and not rx.gates
        assert len(rx.reactants) <= 1 and all(mm == 1 for _, mm in rx.reactants), "not first order"
        if rx.reactants:
            W[j, rx.reactants[0][0]] = rx.rate
        else:
            c[j] = rx.rate
        for sp, mm in rx.reactants:
            nu[sp, j] -= mm
        for sp, mm in rx.products:
            nu[sp, j] += mm
    J = nu @ W
    n = S + S * S + 1
    M = np.zeros((n, n))
    M[:S, :S] = J
    M[:S, -1] = nu @ c
    I = np.eye(S)
    M[S:S + S * S, S:S + S * S] = np.kron(I, J) + np.kron(J, I)
    for j in range(R):
        v = np.outer(nu[:, j], nu[:, j]).reshape(-1)
        M[S:S + S * S, -1] += v * c[j]
        M[S:S + S * S, :S] += np.outer(v, W[j])
    z0 = np.zeros(n)
    z0[:S] = net.x0
    z0[-1] = 1.0
    out = []
    for t in times:
        z = scipy.linalg.expm(M * t) @ z0
        out.append((z[:S], np.diag(z[S:S + S * S].reshape(S, S)).copy()))
    return out


def _check_linear(O, net, n, t_end, dt, seed, must_move):
    """z < 4 for every species' mean at every grid point, against the closed
    form's own variance (SE = sqrt(Var/n)); constants must be exact.  The
    sample variance is checked against the closed form with the standard error
    of a variance estimate, sqrt((m4 - s^4)/n), m4 from the sample."""
    res = O.run(O.OracleModel(net), np.arange(n), seed, t_end, dt)
    assert res.status == 0
    G = O.grid_size(t_end, dt)
    ref = _linear_moments(net, [k * dt for k in range(G)])
    x = res.grid_x.astype(np.float64)
    for k, (mu, var) in enumerate(ref):
        for s in range(net.S):
            assert _zmean(res.mean[k, s], mu[s], var[s], n) < Z, (k, s, res.mean[k, s], mu[s])
            if var[s] * n > 20:      # enough spread for the normal approximation of the estimator
                m4 = np.mean((x[:, k, s] - x[:, k, s].mean()) ** 4)
                assert _zvar(res.var[k, s], var[s], m4, n) < Z, (k, s, res.var[k, s], var[s])
            elif var[s] < 1e-12:
                assert res.var[k, s] == 0.0, (k, s)
    for s in must_move:   # the pin has power: the species actually changes
        assert abs(ref[-1][0][s] - net.x0[s]) > 10 * math.sqrt(max(ref[-1][1][s], 0.0) / n) + 1e-3, s
    return res, ref


def test_linear_moments_closed_form_self_check():
    """The helper itself against textbook cases: immigration-death is Poisson
    (mean = var = k1/k2 (1 - e^{-k2 t})); pure death is Binomial."""
    ref = _linear_moments(inputs.immigration_death(10.0, 0.1, 0), [0.0, 5.0, 50.0])
    for t, (m, v) in zip([0.0, 5.0, 50.0], ref):
        lam = 100.0 * (1 - math.exp(-0.1 * t))
        assert abs(m[0] - lam) < 1e-9 and abs(v[0] - lam) < 1e-9
    ref = _linear_moments(inputs.pure_death(0.7, 12), [1.3])
    p = math.exp(-0.7 * 1.3)
    assert abs(ref[0][0][0] - 12 * p) < 1e-12 and abs(ref[0][1][0] - 12 * p * (1 - p)) < 1e-12


def test_hiv_linear_subnetwork_closed_form(oracle_lib):
    """HIV network (Table 1) with the infection, mutation and infectivity rates set to
    zero (beta = gamma = mu = K = 0): no cell is infected, so I4 = I5 = V4 = F = 0 and what remains is
    first order -- U0 -> U0 + U (lambda), U -> T (d_ut), U -> Z4 and U -> Z5 (d_uz each), T, Z4, Z5
    and V5 clearance.  Means and variances against the exact linear moment equations
    (_linear_moments), z < 4 with the closed form's variance.  Pins the oracle's reading of Table 1's
    reaction list (which species each reaction consumes and produces, and at which rate)."""
    O = oracle_lib
    net = inputs.hiv(beta=0.0, gamma=0.0, mu=0.0, K=0.0, s1=0.0, d_iz=0.0, d_uf=0.0, d_tf=0.0)
    res, _ = _check_linear(O, net, 2000, 20.0, 1.0, 3, must_move=(1, 2, 3, 4, 8))
    for s in (5, 6, 7, 9):
        assert np.all(res.mean[:, s] == 0) and np.all(res.var[:, s] == 0)
    assert np.all(res.mean[:, 0] == 1) and np.all(res.var[:, 0] == 0)


@pytest.mark.parametrize("raised", [False, True])
def test_hiv_bursts_and_productions_closed_form(oracle_lib, raised):
    """Table 1's bursts "I5 -> V5 x 200" and "I4 -> V4 x 200" (reactions 19-20, PAPER.md:63-64 with
    PAPER.md:91 "I4 x pi") and the productions that consume nothing -- sigma_2 (I -> I + Z, reactions
    12-13), sigma_3 (V4 -> F + V4, reaction 21) -- plus the mutation V5 -> V4 (mu) and the I, V
    clearances, on the first-order sub-network that remains when every bimolecular rate is 0
    (beta = gamma = K = sigma_1 = delta_iz = delta_uf = delta_tf = 0) and I4 = I5 = 5 at t = 0.  The
    means and variances solve the linear moment equations exactly (_linear_moments).  raised=False
    keeps Table 1's own rates (the bursts dominate: ~1000 virions of each strain); raised=True raises
    sigma_2, sigma_3 and lowers pi so every production moves its species by many standard errors --
    a dropped product, a burst multiplicity other than 200, or a burst that keeps its infected cell
    fails the z-tests."""
    O = oracle_lib
    zero = dict(beta=0.0, gamma=0.0, K=0.0, s1=0.0, d_iz=0.0, d_uf=0.0, d_tf=0.0)
    if raised:
        zero.update(s2=0.8, s3=0.05, pi=1.5, mu=0.4, d_v=1.0)
    net = inputs.hiv(**zero)
    x0 = list(net.x0)
    x0[5] = x0[6] = 5                                   # I4 = I5 = 5
    net = Network(net.species, tuple(x0), net.reactions, "hiv-linear-bursts")
    move = (1, 2, 3, 4, 5, 6, 7, 8) + ((9,) if raised else ())
    res, ref = _check_linear(O, net, 3000, 3.0, 0.25, 31, must_move=move)
    # the bursts' multiplicity is visible directly: with Table 1's pi the five I5 burst almost at once
    if not raised:
        assert ref[1][0][8] > 500 and res.mean[1, 8] > 500     # ~60 without the bursts
    # the same data reject the plausible misreadings of reactions 12, 13, 19, 20 and 21 (z > 10)
    from inputs.networks import Reaction
    G = O.grid_size(3.0, 0.25)

    def alt(j, products):
        rx = list(net.reactions)
        r = rx[j]
        rx[j] = Reaction(r.reactants, tuple(products), r.rate, r.modifier_species, r.modifier_coef, r.name,
                         r.mass_action, r.gates)
        return Network(net.species, net.x0, tuple(rx))

    U0, U, T, Z4, Z5, I4, I5, V4, V5, F = range(10)
    wrong = {"burst keeps its cell": alt(18, [(I5, 1), (V5, 200)]),
             "burst of 100": alt(18, [(V5, 100)]),
             "X4 burst into V5": alt(19, [(V5, 200)])}
    if raised:
        wrong.update({"sigma2 consumes I": alt(11, [(Z5, 1)]), "sigma2 into Z4": alt(11, [(I5, 1), (Z4, 1)]),
                      "sigma3 consumes V4": alt(20, [(F, 1)])})
    for name, w in wrong.items():
        ra = _linear_moments(w, [k * 0.25 for k in range(G)])
        worst = max(_zmean(res.mean[k, s], ra[k][0][s], max(ra[k][1][s], 1e-30), 3000)
                    for k in range(1, G) for s in range(10))
        assert worst > 10, (name, worst)


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
