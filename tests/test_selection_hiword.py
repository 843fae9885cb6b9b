"""The high-word selection count (K1Gen sel=hi32x, k1_thread.cuh ssa_count_hi + runtime.cu
ssa_apply_sel) is the a7 selection j* = min{ j : c_j > u2 a0 } = #{ j <= R-2 : c_j <= r } (SURVEY.md §8
row a7, DESIGN.md §2 "Order (a4, a7)"; Gillespie's direct method, PAPER.md:198 ref. [8]) computed as j0 = #{ j : hi(c_j) < hi(r) } plus a
recount when hi(c_j0) == hi(r).  This checks the argument on the host, with numpy doubles:
the kernel's arithmetic is checked against the oracle by the GPU parity suites."""
import numpy as np


def _hi(v):
    return (np.asarray(v, dtype=np.float64).view(np.int64) >> 32).astype(np.int32)


def _select_hiword(c, r):
    R = len(c)
    hc, hr = _hi(c[:-1]), _hi(r)
    j0 = int(np.sum(hc < hr))
    if j0 <= R - 2 and hc[j0] == hr:            # the only entry that can tie
        return int(np.sum(c[:-1] <= r)), True
    return j0, False


def _prefix(rng, R, spread):
    a = rng.random(R) ** spread
    a[rng.random(R) < 0.2] = 0.0                 # zero propensities (repeated prefix values)
    a[-1] = max(a[-1], 1e-3)
    return np.cumsum(a)


def test_hiword_selection_equals_the_fp64_count():
    rng = np.random.default_rng(20261021)
    ties = 0
    for trial in range(4000):
        R = int(rng.integers(2, 40))
        c = _prefix(rng, R, spread=float(rng.choice([1.0, 8.0, 30.0])))
        a0 = c[-1]
        rs = list(rng.random(8) * a0) + [0.0]
        # r next to a prefix value: same high word, the low word on either side (forced ties)
        for q in rng.integers(0, R - 1, 3):
            bits = np.float64(c[q]).view(np.int64)
            for d in (-3, -1, 0, 1, 3, 1 << 20):
                v = np.int64(bits + d).view(np.float64)
                if 0.0 <= v < a0:
                    rs.append(float(v))
        for r in rs:
            j, tied = _select_hiword(c, np.float64(r))
            ties += tied
            assert j == int(np.sum(c[:-1] <= r)), (trial, r)
    assert ties > 1000                           # the recount path was exercised


def test_high_words_order_nonnegative_doubles():
    rng = np.random.default_rng(7)
    v = np.concatenate([rng.random(20000) * 10.0 ** rng.integers(-300, 300, 20000),
                        [0.0, 5e-324, 2.2250738585072014e-308, 1.0, 1.7976931348623157e308]])
    x, y = rng.choice(v, 200000), rng.choice(v, 200000)
    hx, hy = _hi(x), _hi(y)
    assert np.all(x[hx < hy] < y[hx < hy])
    assert np.all(x[hx > hy] > y[hx > hy])
