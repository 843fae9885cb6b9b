"""Pins of the oracle's primitives against things other than itself.

- Philox4x32-10 vs curand_Philox4x32_10 from the cuRAND header
  (/usr/local/cuda/include/curand_philox4x32_x.h), compiled for the host.
- u53 vs its closed form (exact rationals).
- plog vs long-double logl (<= 2 ulp) and special values; its series
  coefficients vs 1/(2k+1); ln2 split vs a 60-digit ln 2.
"""
import os
import re
import subprocess
from decimal import Decimal, getcontext
from fractions import Fraction

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)

CURAND_DRIVER = r"""
#include <stdio.h>
#include <stdint.h>
#include <vector_types.h>
#define QUALIFIERS static inline
#include <curand_philox4x32_x.h>
int main(void) {
  uint32_t in[6];
  while (fread(in, 4, 6, stdin) == 6) {
    uint4 c = {in[0], in[1], in[2], in[3]};
    uint2 k = {in[4], in[5]};
    uint4 o = curand_Philox4x32_10(c, k);
    uint32_t out[4] = {o.x, o.y, o.z, o.w};
    fwrite(out, 4, 4, stdout);
  }
  return 0;
}
"""


@pytest.fixture(scope="module")
def curand_philox(tmp_path_factory):
    d = tmp_path_factory.mktemp("curand")
    src = d / "drv.cpp"
    src.write_text(CURAND_DRIVER)
    exe = d / "drv"
    subprocess.check_call(["g++", "-O1", "-I/usr/local/cuda/include", str(src), "-o", str(exe)])

    def run(ctr_keys: np.ndarray) -> np.ndarray:
        out = subprocess.run([str(exe)], input=np.ascontiguousarray(ctr_keys, np.uint32).tobytes(),
                             stdout=subprocess.PIPE, check=True).stdout
        return np.frombuffer(out, np.uint32).reshape(-1, 4)
    return run


def test_philox_matches_curand_header(oracle_lib, curand_philox):
    O = oracle_lib
    rng = np.random.default_rng(12345)
    n_keys, per_key = 64, 16384  # ~1e6 blocks
    keys = rng.integers(0, 2**32, size=(n_keys, 2), dtype=np.uint64).astype(np.uint32)
    keys[0] = (0, 0)
    keys[1] = (0xFFFFFFFF, 0xFFFFFFFF)
    all_in, all_ours = [], []
    for k in keys:
        ctr = rng.integers(0, 2**32, size=(per_key, 4), dtype=np.uint64).astype(np.uint32)
        ctr[0] = 0
        ctr[1] = 0xFFFFFFFF
        # counters laid out as the SSA uses them: (e lo, e hi, id lo, id hi)
        ctr[2:34, 0] = np.arange(32, dtype=np.uint32)
        ctr[2:34, 1:] = 0
        all_ours.append(O.philox_n(ctr, k))
        all_in.append(np.concatenate([ctr, np.broadcast_to(k, (per_key, 2))], axis=1))
    ref = curand_philox(np.concatenate(all_in))
    ours = np.concatenate(all_ours)
    assert ref.shape == ours.shape == (n_keys * per_key, 4)
    assert np.array_equal(ref, ours)


def test_u53_closed_form(oracle_lib):
    O = oracle_lib
    assert O.u53(0) == 2.0 ** -53
    assert O.u53(2**64 - 1) == 1.0 - 2.0 ** -53
    rng = np.random.default_rng(7)
    w = rng.integers(0, 2**64, size=20000, dtype=np.uint64)
    w[:3] = [0, 4095, 4096]
    u = O.u53_n(w)
    for wi, ui in zip(w[:2000].tolist(), u[:2000].tolist()):
        assert Fraction(ui) == Fraction(2 * (wi >> 12) + 1, 2**53)
    assert np.all((u > 0) & (u < 1))
    # mean of uniforms ~ 1/2 (sanity on the bit choice: top bits used)
    assert abs(u.mean() - 0.5) < 5 * np.sqrt(1 / 12 / len(u))


def _plog_inputs(n, seed=0):
    rng = np.random.default_rng(seed)
    u = np.concatenate([
        rng.random(n) * (1 - 2**-53) + 2**-53,               # uniform (0,1)
        np.exp2(-rng.random(n // 2) * 53),                   # log-uniform over [2^-53, 1]
        1 - rng.random(n // 4) * 2**-20,                     # (1 - 2^-20, 1)
        2**-53 * (1 + rng.random(n // 8) * 2**13),           # [2^-53, 2^-40]
        np.array([0.5, 0.25, 2**-53, 1 - 2**-53, np.sqrt(0.5), np.nextafter(np.sqrt(2) / 2, 1)]),
    ])
    return u[(u >= 2**-53) & (u < 1)]


def test_plog_within_2ulp_of_logl(oracle_lib):
    O = oracle_lib
    u = _plog_inputs(1_000_000)
    assert len(u) > 1_000_000
    p = O.plog_n(u)
    ref = np.log(u.astype(np.longdouble))      # x87 logl, 64-bit significand
    ulp = np.spacing(np.abs(ref.astype(np.float64))).astype(np.longdouble)
    err = np.abs((p.astype(np.longdouble) - ref) / ulp).astype(np.float64)
    assert err.max() <= 2.0, err.max()
    assert np.all(p < 0)


def test_plog_special_values(oracle_lib):
    O = oracle_lib
    getcontext().prec = 50
    ln2 = Decimal(2).ln()
    assert O.plog(0.5) == -float(ln2)
    for k in range(1, 54):
        got = Decimal(O.plog(2.0 ** -k))
        exact = -k * ln2
        assert abs(got - exact) <= Decimal(abs(np.spacing(float(exact)))), k
    # near 1: ln(1 - d) ~ -d
    d = 2.0 ** -53
    assert abs(O.plog(1 - d) + d) <= 2 * np.spacing(d)


def _plog_table(src):
    body = src[src.index("PLOG_TAB[128][3] = {"):]
    body = body[:body.index("};")]
    rows = re.findall(r"\{(-?0x[0-9a-fp.+-]+), (-?0x[0-9a-fp.+-]+), (-?0x[0-9a-fp.+-]+)\}", body)
    return [tuple(float.fromhex(v) for v in r) for r in rows]


def test_plog_constants_are_what_they_claim():
    """The literals of the oracle's plog (R11): Q_k == fl((-1)^(k+1)/k) for
    k = 2..7; the ln 2 split; and every table row -- inv_i = fl(1/c_i) with c_i the
    centre of bucket i (halved for i >= 53), inv = 1 for i = 0 and 127, T_hi = fl(-ln inv_i)
    and T_lo = fl(-ln inv_i - T_hi) -- recomputed in exact / 60-digit arithmetic."""
    src = open(os.path.join(ROOT, "oracle", "ssa_oracle.c")).read()
    lits = re.findall(r"(-?0x1\.[0-9a-f]+p[-+]\d+),\s*/\*\s*(-?)1/(\d+)\s*\*/", src)
    assert [int(d) for _, _, d in lits] == [2, 3, 4, 5, 6, 7]
    for hexlit, sign, den in lits:
        k = int(den)
        assert float.fromhex(hexlit) == float(Fraction((-1) ** (k + 1), k))
        assert (sign == "-") == (k % 2 == 0)
    hi = float.fromhex(re.search(r"LN2_HI = (0x[0-9a-fp.+-]+);", src).group(1))
    lo = float.fromhex(re.search(r"LN2_LO = (0x[0-9a-fp.+-]+);", src).group(1))
    getcontext().prec = 60
    ln2 = Decimal(2).ln()
    # hi has at most 32 significant bits so e*hi is exact for |e| < 2^21
    assert 0.5 <= hi < 1 and (Fraction(hi) * 2**32).denominator == 1
    assert abs(Decimal(hi) + Decimal(lo) - ln2) < Decimal(2) ** -80
    tab = _plog_table(src)
    assert len(tab) == 128
    for i, (inv, th, tl) in enumerate(tab):
        if i in (0, 127):
            assert inv == 1.0 and th == 0.0 and tl == 0.0
            continue
        c = Fraction(256 + 2 * i + 1, 256) / (2 if i >= 53 else 1)
        assert inv == float(1 / c), i
        t = -Decimal(inv).ln()
        assert th == float(t) and tl == float(t - Decimal(th)), i


def test_plog_buckets_and_fold(oracle_lib):
    """The bucket structure of plog: near u = 1 from both sides (buckets 0 and 127, inv = 1)
    ln u ~ u - 1 to the last bit; across every bucket edge and the fold at m = 1.4140625 the
    result stays within 2 ulp of logl (monotonicity across an edge is not part of the definition:
    neighbours may differ by an ulp the other way)."""
    O = oracle_lib
    for d in (2.0 ** -53, 2.0 ** -40, 2.0 ** -20, 2.0 ** -9):
        x = 1 - d
        assert abs(Decimal(O.plog(x)) - Decimal(x).ln()) <= Decimal(np.spacing(abs(float(Decimal(x).ln()))))
    edges = []
    for e in (-1, -7, -30):
        for i in range(128):
            m = 1 + i / 128
            for v in (np.nextafter(m, 0), m, np.nextafter(m, 2)):
                if 1 <= v < 2:
                    edges.append(v * 2.0 ** e)
    u = np.array(sorted(edges))
    p = O.plog_n(u)
    ref = np.log(u.astype(np.longdouble))
    ulp = np.spacing(np.abs(ref.astype(np.float64))).astype(np.longdouble)
    assert np.abs((p.astype(np.longdouble) - ref) / ulp).astype(np.float64).max() <= 2.0
