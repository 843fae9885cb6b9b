"""bench.py's roofline bookkeeping, on CPU: the algorithmic work counts the
fractions are taken against, and the committed ncu facts the JSON line cites."""
import importlib.util
import os

import pytest

import inputs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_algorithmic_counts(bench):
    hiv = inputs.config(2).network
    # Philox 40 + u53 6 + plog 21 + tau 9 + propensities (27 k*h + 10 bimolecular products) + prefix 26
    # + selection 52 + update 4 + rest 11
    assert bench.alg_instr_per_event(hiv, 1) == 206
    # FP64: u53 2 + plog 12 + tau 9 + propensities 37 + prefix and selection 52 + r and grid 2
    # + the update's count adds (41 net-change entries over 27 reactions)
    assert bench.alg_fp64_per_event(hiv) == pytest.approx(2 + 12 + 9 + 37 + 52 + 2 + 41 / 27)
    c3 = inputs.config(3).network
    # half-warp K2, order warp16s: lane sum 32 + scan 12 + broadcasts 6 + tau 10 + grid 2 + selection 22
    # (lane* ballot, broadcast, load, 4-step scan, add, compare, ballot) + update 5 + recompute 15
    # + RNG 78/16 + loop 3, per two events
    assert bench.alg_warp_instr_per_event(c3, 16) == pytest.approx((32 + 12 + 6 + 10 + 2 + 22 + 5 + 15 + 64 / 16 + 3) / 2)
    assert bench.alg_warp_instr_per_event(c3, 32) == pytest.approx(95.4375 - 14 / 32, abs=0.01)


def test_committed_profile_facts(bench):
    t = bench.measured_traffic("config2-hiv-100d", "ssa_k1", True)
    assert isinstance(t, int) and t > 1_059_061_760          # >= the algorithmic staging bytes
    assert bench.measured_traffic("config2-hiv-100d", "ssa_tree_leaf", True) >= 1_059_061_760
    assert bench.measured_traffic("config2-hiv-100d", "ssa_k1", False) is None
    a = bench.profiled_activity("config2-hiv-100d", "ssa_k1")
    assert 0.5 < a["issue_active"] < 1.0 and os.path.exists(os.path.join(ROOT, a["source"].split(" ")[0]))
