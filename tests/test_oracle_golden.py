"""The CPU oracle against golden vectors produced by the reference itself.

Pins oracle/lbm_oracle.c (the checker every GPU parity test uses) bit for
bit: whole sweeps of every case (tests/cases.py) against the reference's
gathered PDFs, larger cases against sha256 digests, unit functions
(collide / equilibrium / macroscopic) against the reference's outputs, and
the known answers of the reference's own tests (pkg/tests/test_lbm.py).
"""
import hashlib
import json
from fractions import Fraction
from pathlib import Path

import numpy as np
import pytest

import cases
import oracle

GOLDEN = Path(__file__).resolve().parent / "golden"
META = json.loads((GOLDEN / "digests.json").read_text())
UNITS = np.load(GOLDEN / "units.npz")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("name", sorted(cases.CASES))
def test_oracle_sweeps_bitwise(name):
    spec = cases.CASES[name]
    res = cases.oracle_run(spec, oracle)
    gold = np.load(GOLDEN / f"{name}.npz")
    for s, arr in res["pdf"].items():
        ref = gold[f"pdf_{s}"]
        assert arr.shape == ref.shape
        assert arr.tobytes() == ref.tobytes(), f"{name} step {s}: max |d| {np.abs(arr - ref).max()}"
        assert sha(arr) == META[name]["digests"][f"pdf_{s}"]


@pytest.mark.parametrize("name", sorted(cases.DIGEST_CASES))
def test_oracle_digest_cases(name):
    spec = cases.DIGEST_CASES[name]
    res = cases.oracle_run(spec, oracle)
    for s, arr in res["pdf"].items():
        assert sha(arr) == META["digest_cases"][name][f"pdf_{s}"]


@pytest.mark.parametrize("name", sorted(cases.CASES))
def test_oracle_link_counts(name):
    spec = cases.CASES[name]
    want = META[name]["links"]
    pdf, flags, bits = cases.oracle_inputs(spec, oracle)
    if flags is None:
        assert not want
        return
    st = oracle.STENCILS[spec["stencil"]]
    dom = oracle.Domain(st, spec["dims"], spec["periodic"], cases.oracle_model(spec, oracle),
                        flags, bits)
    got = oracle.link_sets(dom.flags, st, bits)
    assert {k: len(v) for k, v in got.items()} == want


def test_oracle_macroscopic_fields():
    spec = cases.CASES["c1_trt_guo_porous"]
    res = cases.oracle_run(spec, oracle)
    gold = np.load(GOLDEN / "c1_trt_guo_porous.npz")
    st = oracle.STENCILS["D3Q19"]
    f = res["pdf"][spec["steps"]]
    rho, u = oracle.macroscopic(f, st, force=spec["force"][1])
    fluid = (res["domain"].flags[1:-1, 1:-1, 1:-1] & 1) != 0
    assert np.array_equal(rho[fluid], gold["rho"][fluid])
    assert np.array_equal(u[fluid], gold["vel"][fluid])


def _models(st):
    out = {"srt": oracle.Model("SRT", omega=1.3),
           "trt": oracle.Model("TRT", omega_e=1.3, omega_o=0.9),
           "trtmagic": oracle.Model("TRT", omega_e=oracle.trt_magic(1.7)[0],
                                    omega_o=oracle.trt_magic(1.7)[1])}
    if st.name != "D3Q27":
        M = oracle.moment_basis(st)
        Minv = oracle.basis_inverse(M)
        out["mrtu"] = oracle.Model("MRT", M=M.astype(float), Minv=Minv, S=np.full(st.q, 1.3))
        if st.name == "D3Q19":
            r = np.ones(st.q)
            r[9:16] = 1.4
            out["mrt"] = oracle.Model("MRT", M=M.astype(float), Minv=Minv, S=r)
    return out


@pytest.mark.parametrize("sname", ["D2Q9", "D3Q19", "D3Q27"])
def test_oracle_collide_units(sname):
    st = oracle.STENCILS[sname]
    f = UNITS[f"{sname}_in"]
    for vn, m in _models(st).items():
        for fn, force in (("none", None), ("guo", (3e-4, -2e-4, 1e-4))):
            mm = oracle.Model(m.kind, omega=m.omega, omega_e=m.omega_e, omega_o=m.omega_o,
                              M=m.M, Minv=m.Minv, S=m.S, force=force)
            got = oracle.collide_cells(st, f, mm)
            assert got.tobytes() == UNITS[f"{sname}_{vn}_{fn}"].tobytes(), (vn, fn)
            if mm.G is not None:
                assert mm.G.tobytes() == UNITS[f"{sname}_{vn}_guo_matrix"].tobytes()
    shift = oracle.Model("SRT", omega=1.3, force=(3e-4, -2e-4, 1e-4), force_kind="shift")
    assert oracle.collide_cells(st, f, shift).tobytes() == UNITS[f"{sname}_srt_shift"].tobytes()


@pytest.mark.parametrize("sname", ["D2Q9", "D3Q19", "D3Q27"])
def test_oracle_equilibrium_macroscopic_units(sname):
    st = oracle.STENCILS[sname]
    eq = oracle.equilibrium(UNITS[f"{sname}_eq_rho"], UNITS[f"{sname}_eq_u"], st)
    assert eq.tobytes() == UNITS[f"{sname}_eq"].tobytes()
    r, u = oracle.macroscopic(UNITS[f"{sname}_in"], st)
    assert r.tobytes() == UNITS[f"{sname}_macro_rho"].tobytes()
    assert u.tobytes() == UNITS[f"{sname}_macro_u"].tobytes()
    r, u = oracle.macroscopic(UNITS[f"{sname}_in"], st, force=(3e-4, -2e-4, 1e-4))
    assert u.tobytes() == UNITS[f"{sname}_macroguo_u"].tobytes()


def test_known_answers_of_reference_tests():
    # equilibrium hand value (pkg/tests/test_lbm.py:132-136)
    feq = oracle.equilibrium(1.0, (0.1, 0.0), oracle.STENCILS["D2Q9"])
    assert feq.tobytes() == UNITS["equilibrium_hand"].tobytes()
    assert feq[3] == pytest.approx(0.147778, abs=5e-7)
    # TRT magic rates (collision.py:66-74)
    got = np.array([oracle.trt_magic(w)[1] for w in (0.6, 1.0, 1.4, 1.7, 1.8)])
    assert got.tobytes() == UNITS["magic_omegas"].tobytes()
    # moment bases (stencil.py:174-212)
    for s in ("D2Q9", "D3Q19"):
        M = oracle.moment_basis(oracle.STENCILS[s])
        assert np.array_equal(M, UNITS[f"{s}_M"])
        assert oracle.basis_inverse(M).tobytes() == UNITS[f"{s}_Minv"].tobytes()
    # stencil identities in exact rationals (test_lbm.py:81-96)
    for st in oracle.STENCILS.values():
        assert sum(st.wfrac) == 1
        for a in range(3):
            assert sum(w * c[a] for w, c in zip(st.wfrac, st.c)) == 0
            for b in range(3):
                m = sum(w * c[a] * c[b] for w, c in zip(st.wfrac, st.c))
                assert m == (Fraction(1, 3) if a == b and a < st.d else 0)


def test_walled_box_44_links():
    """test_lbm.py:314-331: a 6x6 NoSlip box with 4x4 fluid has 44 links."""
    st = oracle.STENCILS["D2Q9"]
    bits = {"Fluid": 1, "NoSlip": 2, "UBB": 4, "Pressure": 8, "Solid": 16}
    flags = np.zeros((3, 8, 8), dtype=np.uint32)
    flags[1, 1:-1, 1:-1] = bits["NoSlip"]
    flags[1, 2:-2, 2:-2] = bits["Fluid"]
    got = oracle.link_sets(flags, st, bits)
    assert len(got["NoSlip"]) == 44


def test_d3q27_raw_basis_properties():
    st = oracle.STENCILS["D3Q27"]
    M = oracle.raw_moment_basis_d3q27(st)
    assert np.linalg.matrix_rank(M) == 27
    assert np.linalg.cond(M) < 100
