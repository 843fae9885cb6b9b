"""CPU-side checks of the product library (no GPU needed): libssa.so loads and
exports every symbol include/ssa.h declares, model validation, grid size,
NVRTC specialisation of K1 compiles for sm_100a, and compute calls fail loudly
(no CPU fallback) when no device is present."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import inputs
from inputs.networks import Network, _rx

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ssa():
    from paper_1007_1768_b200 import build
    build.build()
    from paper_1007_1768_b200 import ssa as S
    return S


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "ssa.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\*?\s*(ssa_[a-z0-9_]+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_header_symbols_exported(ssa):
    names = _declared_functions()
    assert {"ssa_model_create", "ssa_run", "ssa_run_shard", "ssa_run_sweep", "ssa_merge_roots", "ssa_grid_size",
            "ssa_status_string", "ssa_last_error"} <= set(names)
    out = subprocess.run(["nm", "-D", "--defined-only", ssa.LIB_PATH], stdout=subprocess.PIPE, text=True,
                         check=True).stdout
    exported = set(line.split()[-1] for line in out.splitlines() if line.strip())
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    lib = ssa.lib()
    for n in names:
        assert hasattr(lib, n)
    assert lib.ssa_abi_version() == 1


def test_header_compiles_as_c(tmp_path):
    src = tmp_path / "t.c"
    src.write_text('#include "ssa.h"\nint main(void){ssa_run_options o; ssa_result r; (void)o; (void)r; return 0;}\n')
    subprocess.check_call(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), "-c",
                           str(src), "-o", str(tmp_path / "t.o")])


def test_no_oracle_in_product_path():
    """The product package never imports, links or executes oracle/."""
    pkg = os.path.join(ROOT, "paper_1007_1768_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, fn)).read()
                assert not re.search(r"(import\s+oracle|from\s+oracle|liboracle|oracle/|ssa_oracle|oracle_)",
                                     text), fn


def test_grid_size_matches_definition(ssa):
    for t_end, dt in [(100.0, 1.0), (20.0, 0.1), (10.0, 0.05), (400.0, 1.0), (0.3, 0.1), (1.5, 0.5), (1.0, 3.0)]:
        K = int(np.floor(t_end / dt + 1e-9))
        assert ssa.grid_size(t_end, dt) == K + 1
    assert ssa.grid_size(0.0, 1.0) == 0 and ssa.grid_size(1.0, 0.0) == 0 and ssa.grid_size(1.0, -1) == 0


def test_model_validation(ssa):
    good = ssa.Model(inputs.hiv())
    assert ssa.lib().ssa_model_n_species(good.handle) == 10
    assert ssa.lib().ssa_model_n_reactions(good.handle) == 27
    bad = [
        Network(("A",), (-1,), ()),                                       # negative count
        Network(("A",), (1,), (_rx([(1, 1)], [], 1.0),)),                  # unknown species
        Network(("A",), (1,), (_rx([(0, 0)], [], 1.0),)),                  # coef < 1
        Network(("A",), (1,), (_rx([(0, 1)], [], -1.0),)),                 # negative rate
        Network(("A",), (1,), (_rx([(0, 1)], [], float("nan")),)),         # non-finite rate
        Network(("A",), (1,), (_rx([(0, 4)], [], 1.0),)),                  # order > 3
        Network(("A",), (1,), (_rx([(0, 1), (0, 1)], [], 1.0),)),          # duplicate reactant
        Network(("A",), (1,), (_rx([(0, 1)], [], 1.0, "", (3, 1.0)),)),    # bad modifier
    ]
    for net in bad:
        with pytest.raises(ssa.SSAError) as ei:
            ssa.Model(net)
        assert ei.value.status == 2
    ssa.Model(inputs.empty_network((3,)))   # R == 0 is valid


@pytest.mark.parametrize("netfn", [inputs.immigration_death, inputs.dimerization, inputs.hiv,
                                   lambda: inputs.synthetic(64, 256, 4), lambda: inputs.empty_network((1, 2))])
def test_k1_nvrtc_compiles_for_sm100a(ssa, netfn):
    m = ssa.Model(netfn())
    src = m.k1_source()
    assert "ssa_k1" in src and "SSA_R" in src
    st, log, nbytes = m.k1_compile()
    assert st == 0, log
    assert nbytes > 1000


def _trimolecular():
    from inputs.networks import Network, _rx
    return Network(("A", "B", "C"), (60, 5, 3), (
        _rx([(0, 3)], [(1, 1)], 2e-4), _rx([(1, 1)], [(0, 3)], 0.3), _rx([(0, 2)], [(2, 1)], 1e-3),
        _rx([(2, 1)], [(0, 2)], 0.2), _rx([(1, 1), (2, 1)], [(1, 1)], 0.05, mod=(0, -1e-3))))


@pytest.mark.parametrize("netfn", [inputs.immigration_death, inputs.hiv, lambda: inputs.hiv("B"),
                                   lambda: inputs.synthetic(64, 256, 4), _trimolecular,
                                   lambda: inputs.empty_network((1, 2))])
@pytest.mark.parametrize("half", [False, True])
@pytest.mark.parametrize("dump", [False, True])
def test_k2_nvrtc_compiles_for_sm100a(ssa, netfn, half, dump):
    """Both warp-path kernels (one trajectory per warp, two per warp) compile for every
    model class: coefficient-3 reactants (the general evaluator), modifiers, gates, R = 0."""
    m = ssa.Model(netfn())
    st, log, nbytes = m.k2_compile(256, dump, half, 3 if half else 4)
    assert st == 0, log
    assert nbytes > 1000


def test_compute_fails_loudly_without_device(ssa):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    m = ssa.Model(inputs.immigration_death())
    with pytest.raises(ssa.SSAError) as ei:
        ssa.run(m, 10, 1.0, 0.1, 1)
    assert ei.value.status == 6


def test_shard_bounds_are_aligned_subtrees(ssa):
    for n in (1, 3, 1000, 1024, 65536, 1 << 18, 12345):
        for w in (1, 2, 4, 8):
            covered = []
            for r in range(w):
                b, e = ssa.shard_bounds(n, w, r)
                if e > b:
                    span = 1
                    while span < e - b:
                        span <<= 1
                    assert b % span == 0
                    covered.extend(range(b, e))
            assert covered == list(range(n))


def test_sweep_validation_without_device(ssa):
    """ssa_run_sweep validates its parameter points before touching a device."""
    net = inputs.immigration_death()
    m = ssa.Model(net)
    bad = inputs.rate_matrix(net, [1], [0.1, -1.0])
    with pytest.raises(ssa.SSAError) as ei:
        ssa.run_sweep(m, bad, 10, 5.0, 1.0, 1)
    assert ei.value.status == 2
    nan = inputs.rate_matrix(net, [0], [float("nan")])
    with pytest.raises(ssa.SSAError) as ei:
        ssa.run_sweep(m, nan, 10, 5.0, 1.0, 1)
    assert ei.value.status == 2


def test_gate_validation(ssa):
    """ssa_model_create_ex rejects bad gates (species, kind, count)."""
    from inputs.networks import Network, _rx
    for gates in ([(3, 0)], [(0, 2)], [(0, 0)] * 5):
        net = Network(("A",), (1,), (_rx([], [(0, 1)], 1.0, gates=gates),))
        with pytest.raises(ssa.SSAError) as ei:
            ssa.Model(net)
        assert ei.value.status == 2
    ok = ssa.Model(Network(("A",), (1,), (_rx([(0, 1)], [], 1.0, mass_action=False, gates=[(0, 0)]),)))
    st, log, _ = ok.k1_compile()
    assert st == 0, log


def test_device_plog_literals_match_the_pinned_definition():
    """The device copy of plog's constants (csrc/ssa_device.cuh: the 128-row table and the
    uniform coefficients) is the same pinned definition as the oracle's copy, which
    tests/test_oracle_primitives.py recomputes in exact arithmetic.  The two files share no
    code; this compares the literals."""
    import re
    from fractions import Fraction
    from decimal import Decimal, getcontext
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    dev = open(os.path.join(root, "paper_1007_1768_b200", "csrc", "ssa_device.cuh")).read()
    body = dev[dev.index("ssa_plog_tab[128][4] = {"):]
    body = body[:body.index("};")]
    rows = re.findall(r"\{(-?0x[0-9a-fp.+-]+), (-?0x[0-9a-fp.+-]+), (-?0x[0-9a-fp.+-]+), 0\.0\}", body)
    assert len(rows) == 128
    getcontext().prec = 60
    for i, r in enumerate(rows):
        inv, th, tl = (float.fromhex(v) for v in r)
        if i in (0, 127):
            assert (inv, th, tl) == (1.0, 0.0, 0.0)
            continue
        c = Fraction(256 + 2 * i + 1, 256) / (2 if i >= 53 else 1)
        assert inv == float(1 / c)
        t = -Decimal(inv).ln()
        assert th == float(t) and tl == float(t - Decimal(th))
    coef = dev[dev.index("#define SSA_PLOG_COEF_INIT"):]
    coef = [float.fromhex(v) for v in re.findall(r"-?0x1\.[0-9a-f]+p[-+]\d+", coef[:coef.index("}")])]
    assert coef[:6] == [float(Fraction((-1) ** (k + 1), k)) for k in (7, 6, 5, 4, 3, 2)]
    assert coef[6:] == [float.fromhex("0x1.62e42fee00000p-1"), float.fromhex("0x1.a39ef35793c76p-33")]


def test_species_names(ssa):
    """ssa_model_set_names / ssa_model_species_name (SURVEY.md §8(b)'s nullable names)."""
    m = ssa.Model(inputs.hiv())
    assert m.species_names() == list(inputs.networks.HIV_SPECIES)
    lib = ssa.lib()
    assert lib.ssa_model_set_names(m.handle, None) == 0
    assert m.species_names() == [None] * m.S
    assert lib.ssa_model_species_name(m.handle, 99) is None
    bad = (C.c_char_p * m.S)(*([b"x"] * (m.S - 1) + [None]))
    assert lib.ssa_model_set_names(m.handle, bad) == 1


def test_halfwarp_fast_evaluator_selection():
    """The half-warp K2's fast evaluator (k2_half.cuh SSA_K2_FE) is compiled in only for plain
    mass-action networks (no modifier, no gate, reactant multisets {}, {i}, {i, j}, {2i}); HIV
    (modifiers) and coefficient-3 networks keep the general evaluator."""
    import inputs
    from paper_1007_1768_b200 import ssa as S
    half = 2
    syn = S.Model(inputs.config(3).network)
    assert "#define SSA_K2_FE 1" in S._k2_source(syn, 256, half)
    assert "#define SSA_K2_FE 0" in S._k2_source(syn, 256, 0)          # one-trajectory-per-warp K2
    hiv = S.Model(inputs.config(2).network)
    assert "#define SSA_K2_FE 0" in S._k2_source(hiv, 256, half)
    dim = S.Model(inputs.config(1).network)                           # 2 S1 -> S2: the {2i} form
    assert "#define SSA_K2_FE 1" in S._k2_source(dim, 256, half)
