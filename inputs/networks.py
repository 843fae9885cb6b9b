"""Seeded, synthetic inputs shared by the oracle tests and the CUDA path.

This module holds *only* input descriptions: reaction networks (species,
initial counts, reactions with reactant/product stoichiometry, rate constants,
optional linear rate modifier), the five BASELINE.json configurations, and
seeded choices of which trajectory ids to dump.  It contains none of the
method's arithmetic (no propensities, no net-change vectors, no RNG of the
method): the oracle (`oracle/`) and the product library
(`paper_1007_1768_b200/`) each derive what they need from these descriptions
on their own.

Citations: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

Term = Tuple[int, int]  # (species index, coefficient >= 1)


@dataclass(frozen=True)
class Reaction:
    reactants: Tuple[Term, ...]
    products: Tuple[Term, ...]
    rate: float
    # k^ = max(0, rate + modifier_coef * x[modifier_species])
    modifier_species: int = -1
    modifier_coef: float = 0.0
    name: str = ""
    # Gated propensities ("mu*step(V5)*(1-step(V4))"):
    # mass_action False makes h = 1 (the reactants then only set the stoichiometry);
    # each gate (species, kind) multiplies the propensity by [x > 0] (kind 0,
    # step(x)) or [x == 0] (kind 1, 1 - step(x)).
    mass_action: bool = True
    gates: Tuple[Tuple[int, int], ...] = ()


GATE_POSITIVE, GATE_ZERO = 0, 1


@dataclass(frozen=True)
class Network:
    species: Tuple[str, ...]
    x0: Tuple[int, ...]
    reactions: Tuple[Reaction, ...]
    name: str = ""

    @property
    def S(self) -> int:
        return len(self.species)

    @property
    def R(self) -> int:
        return len(self.reactions)


def _rx(reac: Sequence[Term], prod: Sequence[Term], rate: float, name: str = "",
        mod: Optional[Tuple[int, float]] = None, mass_action: bool = True,
        gates: Sequence[Tuple[int, int]] = ()) -> Reaction:
    ms, mc = (-1, 0.0) if mod is None else mod
    return Reaction(tuple(reac), tuple(prod), float(rate), ms, float(mc), name, bool(mass_action),
                    tuple((int(a), int(b)) for a, b in gates))


# --------------------------------------------------------------------------
# Config 0: immigration-death (BASELINE.json configs[0]).
# --------------------------------------------------------------------------
def immigration_death(k1: float = 10.0, k2: float = 0.1, x0: int = 0) -> Network:
    return Network(("X",), (x0,), (
        _rx([], [(0, 1)], k1, "immigration"),
        _rx([(0, 1)], [], k2, "death"),
    ), "immigration-death")


def pure_death(k: float = 1.0, x0: int = 10) -> Network:
    """X -> 0 at rate k per molecule."""
    return Network(("X",), (x0,), (_rx([(0, 1)], [], k, "death"),), "pure-death")


def empty_network(x0: Sequence[int] = (7,)) -> Network:
    """No reactions: the state is held."""
    return Network(tuple(f"X{i}" for i in range(len(x0))), tuple(int(v) for v in x0), (), "empty")


# --------------------------------------------------------------------------
# Config 1: dimerization-decay (BASELINE.json configs[1]); 2 S1 -> S2 uses
# the combinatorial factor S1(S1-1)/2 (R1).
# --------------------------------------------------------------------------
def dimerization(s1: int = 1000, c=(1.0, 0.002, 0.5, 0.04)) -> Network:
    return Network(("S1", "S2", "S3"), (s1, 0, 0), (
        _rx([(0, 1)], [], c[0], "S1 decay"),
        _rx([(0, 2)], [(1, 1)], c[1], "dimerize"),
        _rx([(1, 1)], [(0, 2)], c[2], "undimerize"),
        _rx([(1, 1)], [(2, 1)], c[3], "convert"),
    ), "dimerization-decay")


# --------------------------------------------------------------------------
# Configs 2 and 4: the paper's HIV model, Table 1 with the rates and
# initial conditions of P:79-93; reaction numbering as SURVEY.md Q27, Variant A
# (literal mass-action mutation, R2), bursts I -> 200 V (R3).
# --------------------------------------------------------------------------
HIV_SPECIES = ("U0", "U", "T", "Z4", "Z5", "I4", "I5", "V4", "V5", "F")
HIV_X0 = (1, 200, 1000, 250, 250, 0, 0, 0, 100, 0)
HIV_PARAMS = dict(lam=200.0, d_uf=1e-5, d_ut=0.129, d_uz=0.005, d_t=0.01, d_tf=1e-5,
                  beta=4e-5, K=1e-7, gamma=2e-5, s1=1e-4, s2=1e-3, d_iz=0.06, mu=2.5e-3,
                  pi=200.0, s3=1e-4, d_i=0.33, d_z=0.01, d_v=2.0)


def hiv(variant: str = "A", **overrides) -> Network:
    """The paper's HIV network (Table 1).  variant "A": the
    mutation V5 -> V4 is Table 1's mass action mu*V5 (R2); "B": the
    time-triggered mutation of PAPER.md:95 ("a stochastic event expected to
    occur at about a given time") as SPEC.md:424's gated propensity
    mu*step(V5)*(1-step(V4)) -- one mutation at rate mu while V5 > 0 and no V4
    exists (NEXT 3, R33)."""
    p = dict(HIV_PARAMS)
    p.update(overrides)
    U0, U, T, Z4, Z5, I4, I5, V4, V5, F = range(10)
    K = p["K"]
    R = [
        _rx([(U0, 1)], [(U0, 1), (U, 1)], p["lam"], "1 U0 -> U0+U"),
        _rx([(U, 1), (F, 1)], [(F, 1)], p["d_uf"], "2 U+F -> F"),
        _rx([(U, 1)], [(T, 1)], p["d_ut"], "3 U -> T"),
        _rx([(U, 1)], [(Z4, 1)], p["d_uz"], "4 U -> Z4"),
        _rx([(U, 1)], [(Z5, 1)], p["d_uz"], "5 U -> Z5"),
        _rx([(T, 1)], [], p["d_t"], "6 T -> 0"),
        _rx([(T, 1), (F, 1)], [(F, 1)], p["d_tf"], "7 T+F -> F"),
        _rx([(T, 1), (V5, 1)], [(I5, 1)], p["beta"], "8 T+V5 -> I5 (beta_R5)", (F, -K)),
        _rx([(T, 1), (V4, 1)], [(I4, 1)], p["beta"], "9 T+V4 -> I4 (beta_X4)", (F, +K)),
        _rx([(Z5, 1), (V5, 1)], [(I5, 1)], p["gamma"], "10 Z5+V5 -> I5 (gamma_R5)", (F, -K)),
        _rx([(Z4, 1), (V4, 1)], [(I4, 1)], p["gamma"], "11 Z4+V4 -> I4 (gamma_X4)", (F, +K)),
        _rx([(I5, 1)], [(I5, 1), (Z5, 1)], p["s2"], "12 I5 -> I5+Z5"),
        _rx([(I4, 1)], [(I4, 1), (Z4, 1)], p["s2"], "13 I4 -> I4+Z4"),
        _rx([(I5, 1), (Z5, 1)], [(U, 1), (I5, 1), (Z5, 1)], p["s1"], "14 I5+Z5 -> U+I5+Z5"),
        _rx([(I4, 1), (Z4, 1)], [(U, 1), (I4, 1), (Z4, 1)], p["s1"], "15 I4+Z4 -> U+I4+Z4"),
        _rx([(I5, 1), (Z5, 1)], [(Z5, 1)], p["d_iz"], "16 I5+Z5 -> Z5"),
        _rx([(I4, 1), (Z4, 1)], [(Z4, 1)], p["d_iz"], "17 I4+Z4 -> Z4"),
        (_rx([(V5, 1)], [(V4, 1)], p["mu"], "18 V5 -> V4") if variant == "A" else
         _rx([(V5, 1)], [(V4, 1)], p["mu"], "18 V5 -> V4 (mu step(V5) (1-step(V4)))", mass_action=False,
             gates=[(V5, GATE_POSITIVE), (V4, GATE_ZERO)])),
        _rx([(I5, 1)], [(V5, 200)], p["pi"], "19 I5 -> 200 V5"),
        _rx([(I4, 1)], [(V4, 200)], p["pi"], "20 I4 -> 200 V4"),
        _rx([(V4, 1)], [(F, 1), (V4, 1)], p["s3"], "21 V4 -> F+V4"),
        _rx([(I5, 1)], [], p["d_i"], "22 I5 -> 0"),
        _rx([(I4, 1)], [], p["d_i"], "23 I4 -> 0"),
        _rx([(Z5, 1)], [], p["d_z"], "24 Z5 -> 0"),
        _rx([(Z4, 1)], [], p["d_z"], "25 Z4 -> 0"),
        _rx([(V5, 1)], [], p["d_v"], "26 V5 -> 0"),
        _rx([(V4, 1)], [], p["d_v"], "27 V4 -> 0"),
    ]
    assert variant in ("A", "B")
    return Network(HIV_SPECIES, HIV_X0, tuple(R), "hiv" if variant == "A" else "hiv-B")


# --------------------------------------------------------------------------
# Config 3: synthetic bounded mass-action network (BASELINE.json configs[3]).
# Drawn with numpy's PCG64 generator seeded by `seed` (R23): type
# uniform over {0->Si, Si->0, Si->Sj, Si+Sj->Sk}; i, j, k uniform; rates
# log-uniform over [1,10], [0.01,0.1], [1e-3,1]; x0 uniform integers [0,1000].
# --------------------------------------------------------------------------
def synthetic(n_species: int = 64, n_reactions: int = 256, seed: int = 4) -> Network:
    rng = np.random.Generator(np.random.PCG64(seed))
    reactions: List[Reaction] = []
    for _ in range(n_reactions):
        typ = int(rng.integers(0, 4))
        i, j, k = (int(v) for v in rng.integers(0, n_species, size=3))
        u = float(rng.random())
        if typ == 0:
            lo, hi = 1.0, 10.0
        elif typ == 1:
            lo, hi = 0.01, 0.1
        else:
            lo, hi = 1e-3, 1.0
        rate = float(np.exp(np.log(lo) + u * (np.log(hi) - np.log(lo))))
        if typ == 0:
            reactions.append(_rx([], [(i, 1)], rate, f"0 -> S{i}"))
        elif typ == 1:
            reactions.append(_rx([(i, 1)], [], rate, f"S{i} -> 0"))
        elif typ == 2:
            reactions.append(_rx([(i, 1)], [(j, 1)], rate, f"S{i} -> S{j}"))
        else:
            reac = [(i, 2)] if i == j else [(i, 1), (j, 1)]
            reactions.append(_rx(reac, [(k, 1)], rate, f"S{i}+S{j} -> S{k}"))
    x0 = tuple(int(v) for v in rng.integers(0, 1001, size=n_species))
    return Network(tuple(f"S{i}" for i in range(n_species)), x0, tuple(reactions),
                   f"synthetic-{n_species}x{n_reactions}-seed{seed}")


# --------------------------------------------------------------------------
# The five BASELINE.json configurations (horizons per DESIGN.md R7).
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class Config:
    index: int
    name: str
    network: Network = field(repr=False)
    n_trajectories: int
    t_end: float
    dt: float
    seed: int
    path: int          # 1 thread path, 2 warp path, 3 half-warp path
    n_dump: int = 0


def configs() -> List[Config]:
    return [
        Config(0, "immigration-death", immigration_death(), 1000, 100.0, 1.0, 1, 1),
        Config(1, "dimerization-decay", dimerization(), 65536, 20.0, 0.1, 2, 1),
        Config(2, "hiv-100d", hiv(), 1 << 18, 100.0, 1.0, 3, 1),
        Config(3, "synthetic-64x256", synthetic(64, 256, 4), 1 << 20, 10.0, 0.05, 4, 3),
        Config(4, "hiv-400d-box", hiv(), 1 << 24, 400.0, 1.0, 5, 1, 65536),
    ]


def config(i: int) -> Config:
    return configs()[i]


# --------------------------------------------------------------------------
# Parameter sweeps ("a set of parameter-swept simulations";
# Fig. 4 panels 2-4: delta_t = 5.0, 3.0, 0.5).
# --------------------------------------------------------------------------
def with_rates(net: Network, rates: Sequence[float]) -> Network:
    """The same network with its rate constants replaced (one sweep point)."""
    assert len(rates) == net.R
    rx = tuple(Reaction(r.reactants, r.products, float(k), r.modifier_species, r.modifier_coef, r.name,
                        r.mass_action, r.gates) for r, k in zip(net.reactions, rates))
    return Network(net.species, net.x0, rx, net.name)


def rate_matrix(net: Network, reaction_index: Sequence[int], values: Sequence[float]) -> np.ndarray:
    """[len(values), R] rate vectors: the network's rates with the listed
    reactions' rate set to each value in turn."""
    base = np.array([r.rate for r in net.reactions], dtype=np.float64)
    out = np.tile(base, (len(values), 1))
    for p, v in enumerate(values):
        out[p, list(reaction_index)] = v
    return out


HIV_DELTA_T_SWEEP = (5.0, 3.0, 0.5)   # Fig. 4 panels 2-4


def hiv_delta_t_sweep(values: Sequence[float] = HIV_DELTA_T_SWEEP, param: str = "d_t"):
    """(network, rates [P, R]) for the Fig. 4 sensitivity sweep.  param 'd_t'
    sweeps the parameter the paper names (T clearance, reaction 6; SPEC.md's
    reading); 'd_v' sweeps the virus clearance (reactions 26, 27), the
    parameter the text describes as "regulating the lifespan of the virus"
    (R32)."""
    net = hiv()
    idx = {"d_t": [5], "d_v": [25, 26]}[param]
    return net, rate_matrix(net, idx, values)


def dump_ids(n_total: int, n_dump: int, seed: int) -> np.ndarray:
    """Sorted, distinct trajectory ids to dump raw (R24)."""
    rng = np.random.Generator(np.random.PCG64(seed + 0x5EED))
    n_dump = min(n_dump, n_total)
    ids = rng.choice(n_total, size=n_dump, replace=False)
    return np.sort(ids.astype(np.uint64))
