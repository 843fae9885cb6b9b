"""ctypes wrapper for the CPU oracle (oracle/ssa_oracle.c) -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module.  It shares no code with the product
library: the model is packed here from the plain `inputs` descriptions
(dense net-change matrix computed below, independently of
paper_1007_1768_b200/csrc).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "ssa_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")
CFLAGS = ["-O2", "-std=gnu11", "-ffp-contract=off", "-fno-fast-math", "-fexcess-precision=standard",
          "-fPIC", "-shared", "-Wall", "-Wextra", "-Wno-unused-parameter"]

MODE_SEQUENTIAL = 0
MODE_WARP32 = 1


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (no FP contraction, no fast-math)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, SRC, "-o", tmp, "-lm"])
        os.replace(tmp, LIB)
    return LIB


class _Model(C.Structure):
    _fields_ = [("S", C.c_int32), ("R", C.c_int32),
                ("x0", C.POINTER(C.c_int64)), ("n_reac", C.POINTER(C.c_int32)),
                ("reac_sp", C.POINTER(C.c_int32)), ("reac_coef", C.POINTER(C.c_int32)),
                ("nu", C.POINTER(C.c_int64)), ("rate", C.POINTER(C.c_double)),
                ("mod_sp", C.POINTER(C.c_int32)), ("mod_coef", C.POINTER(C.c_double)),
                ("mass_action", C.POINTER(C.c_int32)), ("n_gates", C.POINTER(C.c_int32)),
                ("gate_sp", C.POINTER(C.c_int32)), ("gate_kind", C.POINTER(C.c_int32))]


class Summary(C.Structure):
    _fields_ = [("events", C.c_uint64), ("hash", C.c_uint64), ("t_last", C.c_double),
                ("near_ties", C.c_uint64), ("absorbed", C.c_int32), ("status", C.c_int32),
                ("err_reaction", C.c_int32), ("pad", C.c_int32)]


SUMMARY_DTYPE = np.dtype([("events", "<u8"), ("hash", "<u8"), ("t_last", "<f8"),
                          ("near_ties", "<u8"), ("absorbed", "<i4"), ("status", "<i4"),
                          ("err_reaction", "<i4"), ("pad", "<i4")])

_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        P = C.POINTER
        L.oracle_philox4x32_10.argtypes = [P(C.c_uint32), P(C.c_uint32), P(C.c_uint32)]
        L.oracle_u53.argtypes = [C.c_uint64]
        L.oracle_u53.restype = C.c_double
        L.oracle_plog.argtypes = [C.c_double]
        L.oracle_plog.restype = C.c_double
        L.oracle_plog_n.argtypes = [C.c_int64, P(C.c_double), P(C.c_double)]
        L.oracle_philox_n.argtypes = [C.c_int64, P(C.c_uint32), P(C.c_uint32), P(C.c_uint32)]
        L.oracle_u53_n.argtypes = [C.c_int64, P(C.c_uint64), P(C.c_double)]
        L.oracle_propensities.argtypes = [P(_Model), P(C.c_int64), P(C.c_double), P(C.c_int32)]
        L.oracle_select.argtypes = [P(C.c_double), C.c_int32, C.c_int32, C.c_double,
                                    P(C.c_double), P(C.c_int32)]
        L.oracle_step.argtypes = [P(_Model), P(C.c_int64), C.c_double, C.c_double, C.c_int32,
                                  P(C.c_double), P(C.c_int32)]
        L.oracle_grid_K.argtypes = [C.c_double, C.c_double]
        L.oracle_grid_K.restype = C.c_int64
        L.oracle_align_events.argtypes = [C.c_int32, P(C.c_int64), C.c_int64, P(C.c_double),
                                          P(C.c_int64), C.c_double, C.c_double, P(C.c_int32),
                                          P(C.c_uint64), P(C.c_double), P(C.c_uint64)]
        L.oracle_trajectory.argtypes = [P(_Model), C.c_uint64, C.c_uint64, C.c_double, C.c_double,
                                        C.c_int32, P(C.c_int32), P(C.c_uint64), P(C.c_double),
                                        P(Summary)]
        L.oracle_moments.argtypes = [C.c_int64, C.c_int64, P(C.c_int32), P(C.c_double),
                                     P(C.c_double)]
        L.oracle_run.argtypes = [P(_Model), C.c_int64, P(C.c_uint64), C.c_uint64, C.c_double,
                                 C.c_double, C.c_int32, P(C.c_double), P(C.c_double),
                                 P(C.c_int32), P(C.c_uint64), P(C.c_double), C.c_void_p]
        L.oracle_trajectory_events.argtypes = [P(_Model), C.c_uint64, C.c_uint64, C.c_double, C.c_double,
                                               C.c_int32, P(C.c_int32), P(C.c_uint64), P(C.c_double),
                                               P(Summary), C.c_int64, P(C.c_double), P(C.c_int32),
                                               P(C.c_int64)]
        _lib = L
    return _lib


def _ptr(a: Optional[np.ndarray], ct):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(ct))


class OracleModel:
    """Oracle-side packing of an `inputs.Network` (PAPER.md:157 state vector,
    stoichiometric matrix, propensity vector)."""

    def __init__(self, net):
        S, R = net.S, net.R
        self.S, self.R = S, R
        self.x0 = np.array(net.x0, dtype=np.int64).reshape(max(S, 0))
        self.n_reac = np.zeros(max(R, 1), np.int32)
        self.reac_sp = np.zeros(3 * max(R, 1), np.int32)
        self.reac_coef = np.zeros(3 * max(R, 1), np.int32)
        self.nu = np.zeros(max(R, 1) * max(S, 1), np.int64)
        self.rate = np.zeros(max(R, 1), np.float64)
        self.mod_sp = np.full(max(R, 1), -1, np.int32)
        self.mod_coef = np.zeros(max(R, 1), np.float64)
        self.mass_action = np.ones(max(R, 1), np.int32)
        self.n_gates = np.zeros(max(R, 1), np.int32)
        self.gate_sp = np.zeros(4 * max(R, 1), np.int32)
        self.gate_kind = np.zeros(4 * max(R, 1), np.int32)
        for j, rx in enumerate(net.reactions):
            assert len(rx.reactants) <= 3
            self.n_reac[j] = len(rx.reactants)
            for q, (sp, m) in enumerate(rx.reactants):
                self.reac_sp[3 * j + q] = sp
                self.reac_coef[3 * j + q] = m
                self.nu[j * S + sp] -= m
            for sp, m in rx.products:
                self.nu[j * S + sp] += m
            self.rate[j] = rx.rate
            self.mod_sp[j] = rx.modifier_species
            self.mod_coef[j] = rx.modifier_coef
            self.mass_action[j] = 1 if getattr(rx, "mass_action", True) else 0
            gates = getattr(rx, "gates", ())
            assert len(gates) <= 4
            self.n_gates[j] = len(gates)
            for g, (sp, kind) in enumerate(gates):
                self.gate_sp[4 * j + g] = sp
                self.gate_kind[4 * j + g] = kind
        self._c = _Model(S, R, _ptr(self.x0, C.c_int64), _ptr(self.n_reac, C.c_int32),
                         _ptr(self.reac_sp, C.c_int32), _ptr(self.reac_coef, C.c_int32),
                         _ptr(self.nu, C.c_int64), _ptr(self.rate, C.c_double),
                         _ptr(self.mod_sp, C.c_int32), _ptr(self.mod_coef, C.c_double),
                         _ptr(self.mass_action, C.c_int32), _ptr(self.n_gates, C.c_int32),
                         _ptr(self.gate_sp, C.c_int32), _ptr(self.gate_kind, C.c_int32))

    @property
    def c(self):
        return C.byref(self._c)


# ---------------------------------------------------------------- primitives
def philox(ctr: Sequence[int], key: Sequence[int]) -> np.ndarray:
    c = np.array(ctr, np.uint32)
    k = np.array(key, np.uint32)
    o = np.zeros(4, np.uint32)
    lib().oracle_philox4x32_10(_ptr(c, C.c_uint32), _ptr(k, C.c_uint32), _ptr(o, C.c_uint32))
    return o


def philox_n(ctr: np.ndarray, key: Sequence[int]) -> np.ndarray:
    ctr = np.ascontiguousarray(ctr, np.uint32).reshape(-1, 4)
    k = np.array(key, np.uint32)
    o = np.zeros_like(ctr)
    lib().oracle_philox_n(len(ctr), _ptr(ctr, C.c_uint32), _ptr(k, C.c_uint32), _ptr(o, C.c_uint32))
    return o


def u53(w: int) -> float:
    return lib().oracle_u53(w)


def u53_n(w: np.ndarray) -> np.ndarray:
    w = np.ascontiguousarray(w, np.uint64)
    o = np.zeros(len(w), np.float64)
    lib().oracle_u53_n(len(w), _ptr(w, C.c_uint64), _ptr(o, C.c_double))
    return o


def plog(u: float) -> float:
    return lib().oracle_plog(u)


def plog_n(u: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(u, np.float64)
    o = np.zeros(len(u), np.float64)
    lib().oracle_plog_n(len(u), _ptr(u, C.c_double), _ptr(o, C.c_double))
    return o


def propensities(model: OracleModel, x: Sequence[int]):
    xa = np.array(x, np.int64)
    a = np.zeros(max(model.R, 1), np.float64)
    bad = C.c_int32(-1)
    st = lib().oracle_propensities(model.c, _ptr(xa, C.c_int64), _ptr(a, C.c_double), C.byref(bad))
    return st, a[:model.R], bad.value


def select(a: Sequence[float], mode: int, u2: float):
    aa = np.array(a, np.float64)
    a0 = C.c_double()
    j = C.c_int32()
    lib().oracle_select(_ptr(aa, C.c_double), len(aa), mode, u2, C.byref(a0), C.byref(j))
    return a0.value, j.value


def step(model: OracleModel, x: Sequence[int], u1: float, u2: float, mode: int = 0):
    xa = np.array(x, np.int64)
    tau = C.c_double()
    j = C.c_int32()
    st = lib().oracle_step(model.c, _ptr(xa, C.c_int64), u1, u2, mode, C.byref(tau), C.byref(j))
    return st, tau.value, j.value


def grid_size(t_end: float, dt: float) -> int:
    return int(lib().oracle_grid_K(t_end, dt)) + 1


def align_events(x0: Sequence[int], times: Sequence[float], states: np.ndarray, t_end: float,
                 dt: float):
    S = len(x0)
    G = grid_size(t_end, dt)
    x0a = np.array(x0, np.int64)
    ta = np.array(times, np.float64)
    sa = np.ascontiguousarray(np.array(states, np.int64).reshape(len(ta), S))
    gx = np.zeros((G, S), np.int32)
    ge = np.zeros(G, np.uint64)
    gt = np.zeros(G, np.float64)
    nt = C.c_uint64()
    lib().oracle_align_events(S, _ptr(x0a, C.c_int64), len(ta), _ptr(ta, C.c_double),
                              _ptr(sa, C.c_int64), t_end, dt, _ptr(gx, C.c_int32),
                              _ptr(ge, C.c_uint64), _ptr(gt, C.c_double), C.byref(nt))
    return gx, ge, gt, nt.value


@dataclass
class Trajectory:
    grid_x: np.ndarray   # [G, S] int32
    grid_e: np.ndarray   # [G] uint64
    grid_t: np.ndarray   # [G] float64
    summary: dict


def trajectory(model: OracleModel, tid: int, seed: int, t_end: float, dt: float,
               mode: int = 0) -> Trajectory:
    G = grid_size(t_end, dt)
    gx = np.zeros((G, max(model.S, 1)), np.int32)
    ge = np.zeros(G, np.uint64)
    gt = np.zeros(G, np.float64)
    s = Summary()
    lib().oracle_trajectory(model.c, tid, seed, t_end, dt, mode, _ptr(gx, C.c_int32),
                            _ptr(ge, C.c_uint64), _ptr(gt, C.c_double), C.byref(s))
    summ = {f: getattr(s, f) for f, _ in Summary._fields_ if f != "pad"}
    return Trajectory(gx[:, :model.S], ge, gt, summ)


def moments(samples: np.ndarray):
    """Exact mean and population variance over axis 0 of int32 samples."""
    s = np.ascontiguousarray(samples, np.int32)
    n = s.shape[0]
    cells = int(np.prod(s.shape[1:]))
    mean = np.zeros(cells, np.float64)
    var = np.zeros(cells, np.float64)
    lib().oracle_moments(n, cells, _ptr(s, C.c_int32), _ptr(mean, C.c_double), _ptr(var, C.c_double))
    return mean.reshape(s.shape[1:]), var.reshape(s.shape[1:])


@dataclass
class RunResult:
    mean: np.ndarray       # [G, S]
    var: np.ndarray        # [G, S]
    status: int
    grid_x: Optional[np.ndarray] = None   # [n, G, S]
    grid_e: Optional[np.ndarray] = None   # [n, G]
    grid_t: Optional[np.ndarray] = None   # [n, G]
    summaries: Optional[np.ndarray] = None  # structured [n]


def run(model: OracleModel, ids, seed: int, t_end: float, dt: float, mode: int = 0,
        keep: bool = True) -> RunResult:
    ids = np.ascontiguousarray(np.asarray(ids, dtype=np.uint64))
    n = len(ids)
    G = grid_size(t_end, dt)
    S = model.S
    mean = np.zeros((G, max(S, 1)), np.float64)
    var = np.zeros((G, max(S, 1)), np.float64)
    gx = np.zeros((n, G, max(S, 1)), np.int32) if keep else None
    ge = np.zeros((n, G), np.uint64) if keep else None
    gt = np.zeros((n, G), np.float64) if keep else None
    sums = np.zeros(n, SUMMARY_DTYPE) if keep else None
    st = lib().oracle_run(model.c, n, _ptr(ids, C.c_uint64), seed, t_end, dt, mode,
                          _ptr(mean, C.c_double), _ptr(var, C.c_double), _ptr(gx, C.c_int32),
                          _ptr(ge, C.c_uint64), _ptr(gt, C.c_double),
                          None if sums is None else sums.ctypes.data)
    return RunResult(mean[:, :S], var[:, :S], st,
                     None if gx is None else gx[:, :, :S], ge, gt, sums)


# --------------------------------------------------------------------------
# Union-time selective memory (PAPER.md:143-149
# §3.2.1, Fig. 3), written out as the offline brute-force
# definition of: collect every stream, take the union of their
# point times, hold each stream's value (zero-order hold, right-continuous),
# reduce across streams (Y), then reduce k_x successive Y-points (X).
# --------------------------------------------------------------------------
def events(model: OracleModel, tid: int, seed: int, t_end: float, mode: int = 0):
    """Applied events of trajectory `tid` on [0, t_end]: (times [E], reactions [E])."""
    n = C.c_int64()
    s = Summary()
    lib().oracle_trajectory_events(model.c, tid, seed, t_end, t_end, mode, None, None, None, C.byref(s),
                                   0, None, None, C.byref(n))
    E = n.value
    t = np.zeros(max(E, 1), np.float64)
    j = np.zeros(max(E, 1), np.int32)
    lib().oracle_trajectory_events(model.c, tid, seed, t_end, t_end, mode, None, None, None, C.byref(s),
                                   E, _ptr(t, C.c_double), _ptr(j, C.c_int32), C.byref(n))
    return t[:E], j[:E]


def stream(model: OracleModel, tid: int, seed: int, t_end: float, mode: int = 0):
    """The trajectory as a point stream: (0, x0), one point
    per applied event (time, state after it), and the horizon point (t_end,
    final state) unless an event lies exactly at t_end."""
    t, j = events(model, tid, seed, t_end, mode)
    S = model.S
    nu = model.nu.reshape(-1, max(S, 1))[:, :S] if model.R else np.zeros((0, S), np.int64)
    x = np.array(model.x0, np.int64)
    times = [0.0]
    states = [x.copy()]
    for tt, jj in zip(t, j):
        x = x + nu[jj]
        times.append(float(tt))
        states.append(x.copy())
    if times[-1] < t_end:
        times.append(float(t_end))
        states.append(x.copy())
    return np.array(times), np.array(states, np.int64).reshape(len(times), S)


def union_reduce(streams, kx: int):
    """Y-then-X reduction of k point streams.  Returns (times [P], mean [P,S],
    var [P,S], n [P]): Y-points at every distinct union time u (each stream's
    held value, summed exactly), grouped kx at a time in time order; a group's
    time is the IEEE left-to-right sum of its Y-times divided by its size, its
    moments are exact (n = k * size, mean = S1/n, population variance
    (n S2 - S1^2)/n^2, each rounded once)."""
    from fractions import Fraction
    k = len(streams)
    U = np.unique(np.concatenate([np.asarray(t, np.float64) for t, _ in streams]))
    S = streams[0][1].shape[1]
    S1 = [[0] * S for _ in U]
    S2 = [[0] * S for _ in U]
    for t, x in streams:
        idx = np.searchsorted(t, U, side="right") - 1          # zero-order hold
        assert np.all(idx >= 0)
        held = x[idx]
        for m in range(len(U)):
            for s_ in range(S):
                v = int(held[m, s_])
                S1[m][s_] += v
                S2[m][s_] += v * v
    times, means, vars_, ns = [], [], [], []
    for g0 in range(0, len(U), kx):
        grp = range(g0, min(g0 + kx, len(U)))
        tsum = 0.0
        for m in grp:
            tsum = tsum + float(U[m])
        times.append(tsum / len(grp))
        n = k * len(grp)
        a1 = [sum(S1[m][s_] for m in grp) for s_ in range(S)]
        a2 = [sum(S2[m][s_] for m in grp) for s_ in range(S)]
        means.append([float(Fraction(a1[s_], n)) for s_ in range(S)])
        vars_.append([float(Fraction(n * a2[s_] - a1[s_] * a1[s_], n * n)) for s_ in range(S)])
        ns.append(n)
    return np.array(times), np.array(means).reshape(-1, S), np.array(vars_).reshape(-1, S), np.array(ns)



# --------------------------------------------------------------------------
# Stride-sampled trajectory output (PAPER.md:175
# "a 1:10 sampling (outputting 1 simulation point every 10)"
# SamplingPolicy::Stride(s) "emit every s-th event plus first/last").
# --------------------------------------------------------------------------
def stride_points(model: OracleModel, tid: int, seed: int, t_end: float, stride: int, mode: int = 0):
    """(event_index [P], times [P], states [P, S]) of trajectory `tid`: the
    initial point (0, 0, x0), the point after every stride-th applied event
    (k, t_k, x_k) for k = s, 2s, ..., and the horizon point (E, t_end, x_E)
    unless the last emitted point is already at t_end."""
    t, j = events(model, tid, seed, t_end, mode)
    S = model.S
    nu = model.nu.reshape(-1, max(S, 1))[:, :S] if model.R else np.zeros((0, S), np.int64)
    x = np.array(model.x0, np.int64)
    ks, ts, xs = [0], [0.0], [x.copy()]
    for k, (tt, jj) in enumerate(zip(t, j), start=1):
        x = x + nu[jj]
        if k % stride == 0:
            ks.append(k)
            ts.append(float(tt))
            xs.append(x.copy())
    if ts[-1] < t_end:
        ks.append(len(t))
        ts.append(float(t_end))
        xs.append(x.copy())
    return np.array(ks, np.uint64), np.array(ts), np.array(xs, np.int64).reshape(len(ts), S)
