"""GPU parity: the sm_100a path against the reference's golden vectors and the
pinned CPU oracle, through the public drop-in API (which calls the C-ABI).

fp64 results must be bit-identical (the fp64 kernels round every operation
like the reference's numpy ufuncs); the BASELINE tolerance (max-abs 1e-12)
is therefore never needed but is what a failure message reports against.
fp32 storage is checked at 1e-5 relative against the fp64 oracle.
"""
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

import cases
import oracle

pytestmark = pytest.mark.gpu

GOLDEN = Path(__file__).resolve().parent / "golden"
META = json.loads((GOLDEN / "digests.json").read_text())
UNITS = np.load(GOLDEN / "units.npz")
TOL_F64 = 1e-12      # BASELINE.json: max-abs on PDFs/rho/u in fp64
TOL_F32_REL = 1e-5   # BASELINE.json: relative in fp32


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def api():
    import paper_1909_13772_b200 as P
    P._lib.load()
    return cases.b200_api()


def _ctx():
    import paper_1909_13772_b200 as P
    return P.Context()


@pytest.mark.parametrize("name", sorted(cases.CASES))
def test_cases_bitwise_vs_reference_golden(api, name):
    spec = cases.CASES[name]
    res = cases.run_case(api, _ctx(), spec)
    gold = np.load(GOLDEN / f"{name}.npz")
    for s, arr in res["pdf"].items():
        ref = gold[f"pdf_{s}"]
        d = float(np.abs(arr - ref).max())
        assert arr.tobytes() == ref.tobytes(), f"{name} step {s}: max|d| = {d:.3e} (tol {TOL_F64})"
    if res["macro"] is not None:
        assert res["macro"][0].tobytes() == gold["rho"].tobytes()
        assert res["macro"][1].tobytes() == gold["vel"].tobytes()
    if META[name]["links"]:
        assert res["links"] == META[name]["links"]


@pytest.mark.parametrize("name", sorted(cases.DIGEST_CASES))
def test_digest_cases(api, name):
    spec = cases.DIGEST_CASES[name]
    res = cases.run_case(api, _ctx(), spec)
    for s, arr in res["pdf"].items():
        assert sha(arr) == META["digest_cases"][name][f"pdf_{s}"]


@pytest.mark.parametrize("sname", ["D2Q9", "D3Q19", "D3Q27"])
def test_flat_cell_kernels_bitwise(api, sname):
    st = getattr(api, sname)
    f = UNITS[f"{sname}_in"]
    variants = {"srt": api.SRT(1.3), "trt": api.TRT(1.3, 0.9), "trtmagic": api.TRT.with_magic(1.7)}
    if sname != "D3Q27":
        variants["mrtu"] = api.MRT.uniform(st, 1.3)
        if sname == "D3Q19":
            r = [1.0] * 19
            r[9:16] = [1.4] * 7
            variants["mrt"] = api.MRT(st, r)
    for vn, m in variants.items():
        assert api.collide_pdfs(f, st, m).tobytes() == UNITS[f"{sname}_{vn}_none"].tobytes(), vn
        got = api.collide_pdfs(f, st, m, api.Guo((3e-4, -2e-4, 1e-4)))
        assert got.tobytes() == UNITS[f"{sname}_{vn}_guo"].tobytes(), vn
    got = api.collide_pdfs(f, st, api.SRT(1.3), api.SimpleShift((3e-4, -2e-4, 1e-4)))
    assert got.tobytes() == UNITS[f"{sname}_srt_shift"].tobytes()
    eq = api.equilibrium(UNITS[f"{sname}_eq_rho"], UNITS[f"{sname}_eq_u"], st)
    assert eq.tobytes() == UNITS[f"{sname}_eq"].tobytes()
    r, u = api.macroscopic(f, st)
    assert r.tobytes() == UNITS[f"{sname}_macro_rho"].tobytes()
    assert u.tobytes() == UNITS[f"{sname}_macro_u"].tobytes()
    r, u = api.macroscopic(f, st, force=api.Guo((3e-4, -2e-4, 1e-4)))
    assert u.tobytes() == UNITS[f"{sname}_macroguo_u"].tobytes()


def test_reference_unit_properties(api):
    """SRT omega=1 lands exactly on feq; zero force == unforced bitwise
    (pkg/tests/test_lbm.py:180-184, 239-248); non-positive density raises."""
    st = api.D2Q9
    f = UNITS["D2Q9_in"]
    rho, u = api.macroscopic(f, st)
    assert np.array_equal(api.collide_pdfs(f, st, api.SRT(1.0)), api.equilibrium(rho, u, st))
    for m in (api.SRT(1.3), api.TRT(1.3, 0.9), api.MRT.uniform(st, 1.3)):
        assert np.array_equal(api.collide_pdfs(f, st, m),
                              api.collide_pdfs(f, st, m, api.Guo((0.0, 0.0, 0.0))))
    import paper_1909_13772_b200 as P
    with pytest.raises(P.NumericsError):
        api.macroscopic(np.zeros(9), st)


def _oracle_compare(api, spec, every=None):
    """Run spec on the GPU and the oracle, compare every snapshot bitwise."""
    res = cases.run_case(api, _ctx(), spec)
    ores = cases.oracle_run(spec, oracle)
    for s in spec["snapshots"]:
        a, b = res["pdf"][s], ores["pdf"][s]
        d = float(np.abs(a - b).max())
        assert a.tobytes() == b.tobytes(), f"step {s}: max|d| = {d:.3e} (tol {TOL_F64})"
    return res, ores


def test_config0_full_size_bitwise(api):
    """BASELINE config 0: D3Q19 SRT 1.8, 64^3 periodic, seeded random
    init, 100 steps, compare PDFs every 10 steps."""
    spec = dict(stencil="D3Q19", dims=(64, 64, 64), root_dims=(1, 1, 1),
                periodic=(True, True, True), geometry=None, model=("SRT", 1.8), force=None,
                init=("random", 0), steps=100, snapshots=tuple(range(10, 101, 10)), layout="fzyx")
    _oracle_compare(api, spec)


def test_config1_full_size_bitwise(api):
    """BASELINE config 1 at full size (128^3 porous, 25 % spheres r 4-8, NoSlip
    z walls, TRT magic 1.7, Guo 1e-6); 100 of its 1000 steps (oracle cost),
    plus rho/u."""
    spec = dict(stencil="D3Q19", dims=(128, 128, 128), root_dims=(1, 1, 1),
                periodic=(True, True, False),
                geometry=dict(kind="spheres", seed=1, rmin=4.0, rmax=8.0, frac=0.25, walls_z=True),
                model=("TRT_magic", 1.7), force=("Guo", (1e-6, 0.0, 0.0)), init=("rest",),
                steps=100, snapshots=(50, 100), layout="fzyx")
    _oracle_compare(api, spec)


def test_config2_model_fp64_bitwise(api):
    """BASELINE config 2 physics (D3Q27 raw-moment MRT shear 1.9 / others 1.0,
    NoSlip x5 + UBB lid (0.05, 0, 0)) in fp64 at 48^3 against the oracle."""
    spec = dict(stencil="D3Q27", dims=(48, 48, 48), root_dims=(1, 1, 1),
                periodic=(False, False, False), geometry=dict(kind="cavity"),
                model=("MRT_raw", 1.9, 1.0), force=None, init=("rest",),
                ubb_velocity=(0.05, 0.0, 0.0), steps=60, snapshots=(60,), layout="fzyx")
    _oracle_compare(api, spec)


@pytest.mark.parametrize("spec_name", ["c0", "c1", "c2"])
def test_fp32_storage_within_1e5_relative(api, spec_name):
    """fp32 PDFs (stored as f - w_i, fp32 arithmetic on the centred populations)
    vs the fp64 oracle."""
    specs = {
        "c0": dict(stencil="D3Q19", dims=(48, 48, 48), root_dims=(1, 1, 1),
                   periodic=(True, True, True), geometry=None, model=("TRT_magic", 1.8),
                   force=None, init=("random", 0), steps=200, snapshots=(200,), layout="fzyx"),
        "c1": dict(stencil="D3Q19", dims=(64, 64, 64), root_dims=(1, 1, 1),
                   periodic=(True, True, False),
                   geometry=dict(kind="spheres", seed=100, rmin=4.0, rmax=8.0, frac=0.2,
                                 walls_z=True),
                   model=("TRT_magic", 1.7), force=("Guo", (1e-6, 0.0, 0.0)), init=("random", 2),
                   steps=200, snapshots=(200,), layout="fzyx"),
        "c2": dict(stencil="D3Q27", dims=(40, 40, 40), root_dims=(1, 1, 1),
                   periodic=(False, False, False), geometry=dict(kind="cavity"),
                   model=("MRT_raw", 1.9, 1.0), force=None, init=("rest",),
                   ubb_velocity=(0.05, 0.0, 0.0), steps=300, snapshots=(300,), layout="fzyx"),
    }
    spec = specs[spec_name]
    res = cases.run_case(api, _ctx(), spec, pdf_kwargs={"dtype": "float32"})
    ores = cases.oracle_run(spec, oracle)
    s = spec["steps"]
    a, b = res["pdf"][s], ores["pdf"][s]
    rel = float(np.max(np.abs(a - b) / np.abs(b)))
    assert rel < TOL_F32_REL, rel


@pytest.mark.parametrize("force", [None, ("Guo", (2e-5, -1e-5, 3e-6)), ("Guo", (3e-5, 0.0, 0.0))])
def test_fp32_factorised_d3q27_mrt_with_and_without_guo(api, force):
    """The fp32 D3Q27 raw-moment MRT (moment-space form without force, the
    population-space form with Guo) against the fp64 oracle, 1e-5 relative."""
    spec = dict(stencil="D3Q27", dims=(24, 20, 22), root_dims=(1, 1, 1),
                periodic=(True, True, True), geometry=None, model=("MRT_raw", 1.9, 1.0),
                force=force, init=("random", 13), steps=150, snapshots=(150,), layout="fzyx")
    res = cases.run_case(api, _ctx(), spec, pdf_kwargs={"dtype": "float32"})
    ores = cases.oracle_run(spec, oracle)
    a, b = res["pdf"][150], ores["pdf"][150]
    rel = float(np.max(np.abs(a - b) / np.abs(b)))
    assert rel < TOL_F32_REL, rel


@pytest.mark.parametrize("name", ["c1_trt_guo_porous", "c2_d3q27_trt_cavity", "d2q9_pressure_box",
                                  "d3q19_shift_ghostwalls"])
def test_link_sets_equal_exhaustive_scan(api, name):
    """GPU link masks decoded to the reference's lists == exhaustive scan
    (pkg/tests/test_lbm.py:280-331 scan_links oracle)."""
    import paper_1909_13772_b200 as P
    spec = cases.CASES[name]
    pdf, flags, bits = cases.oracle_inputs(spec, oracle)
    st = oracle.STENCILS[spec["stencil"]]
    dom = oracle.Domain(st, spec["dims"], spec["periodic"], cases.oracle_model(spec, oracle),
                        flags, bits)
    want = oracle.link_sets(dom.flags, st, bits)
    ctx = _ctx()
    nx, ny, nz = spec["dims"]
    d = 2 if spec["stencil"] == "D2Q9" else 3
    forest = P.create_forest(ctx, (0, 0, 0, 1, 1, 1), (1, 1, 1), d=d,
                             periodic=spec["periodic"], cells_per_block=(nx, ny, nz))
    h = P.ensure_flags(forest)
    blk = forest.local_blocks()[0]
    ff = blk.data["flags"]
    assert [int(h.registry[n]) for n in ("Fluid", "NoSlip", "UBB", "Pressure", "Solid")] == \
        [1, 2, 4, 8, 16]
    ff.view[...] = flags
    handling = P.BoundaryHandling(forest, getattr(P, spec["stencil"]))
    handling.freeze()
    lists = handling.links[blk.id]
    for tname in ("NoSlip", "UBB", "Pressure"):
        got = []
        for i, zs, ys, xs in lists[tname]:
            got.append(np.stack([xs - 1, ys - 1, zs - 1, np.full_like(xs, i)], axis=1))
        got = np.concatenate(got) if got else np.zeros((0, 4), np.int64)
        got = got[np.lexsort((got[:, 3], got[:, 0], got[:, 1], got[:, 2]))].astype(np.int32)
        assert np.array_equal(got, want[tname]), tname


def test_validation_errors_mirror_reference(api):
    import paper_1909_13772_b200 as P
    ctx = _ctx()
    forest = P.create_forest(ctx, (0, 0, 0, 1, 1, 1), (1, 1, 1), d=2, periodic=(True, True, False),
                             cells_per_block=(6, 6, 1))
    h = P.ensure_flags(forest)
    ff = forest.local_blocks()[0].data["flags"]
    ff.interior[...] = h.registry["Fluid"]
    ff.interior[0, 2, 2] = h.registry["Solid"]
    handling = P.BoundaryHandling(forest, P.D2Q9)
    with pytest.raises(P.ValidationError):
        handling.freeze()                      # fluid streams from Solid
    ff.interior[0, 2, 2] = 0
    with pytest.raises(P.ValidationError):
        handling.freeze()                      # fluid streams from unflagged
    ff.interior[0, 1:4, 1:4] = h.registry["NoSlip"]
    ff.interior[0, 2, 2] = h.registry["Solid"]
    handling.freeze()                          # wrapped in a boundary layer: fine
    ff.interior[0, 0, 0] |= h.registry["NoSlip"]
    with pytest.raises(P.ValidationError):
        handling.freeze()                      # conflicting flags
    # non-periodic domain without handling
    f2 = P.create_forest(ctx, (0, 0, 0, 1, 1, 1), (1, 1, 1), d=2, periodic=(True, False, False),
                         cells_per_block=(4, 4, 1))
    pdf = P.PdfField(f2, P.D2Q9)
    P.fill_equilibrium(pdf)
    with pytest.raises(P.ValidationError):
        P.stream_collide(pdf, P.SRT(1.2))


def test_model_switch_between_sweeps_matches_oracle(api):
    """Changing the model between calls re-collides the stored state: the
    result equals the reference's per-call semantics (oracle, bitwise)."""
    import paper_1909_13772_b200 as P
    spec = dict(cases.CASES["c0_srt_periodic"])
    ctx = _ctx()
    nx, ny, nz = spec["dims"]
    forest = P.create_forest(ctx, (0, 0, 0, 1, 1, 1), (1, 1, 1), periodic=(True, True, True),
                             cells_per_block=(nx, ny, nz))
    pdf = P.PdfField(forest, P.D3Q19, layout="fzyx")
    P.fill_equilibrium(pdf)
    rho, u = cases.workloads.random_rho_u((nx, ny, nz), 0)
    blk = forest.local_blocks()[0]
    pdf.src(blk).interior[...] = P.equilibrium(rho, u, P.D3Q19)
    for _ in range(3):
        P.stream_collide(pdf, P.SRT(1.8))
    for _ in range(3):
        P.stream_collide(pdf, P.TRT(1.3, 0.9), force=P.Guo((1e-4, 0, 0)))
    got = pdf.src(blk).interior.copy()
    st = oracle.STENCILS["D3Q19"]
    full, _, _ = cases.oracle_inputs(spec, oracle)
    d1 = oracle.Domain(st, (nx, ny, nz), (True, True, True), oracle.Model("SRT", omega=1.8))
    d1.set_full(full)
    d1.run(3)
    d2 = oracle.Domain(st, (nx, ny, nz), (True, True, True),
                       oracle.Model("TRT", omega_e=1.3, omega_o=0.9, force=(1e-4, 0.0, 0.0)))
    d2.set_full(d1.a)
    d2.run(3)
    assert got.tobytes() == d2.rform().tobytes()


def test_host_edit_between_sweeps_is_uploaded(api):
    """A host write into pdf.src(block) after a readout is seen by the next
    sweep (single-cell bump, pkg/tests/test_lbm.py:436-449 pattern)."""
    import paper_1909_13772_b200 as P
    ctx = _ctx()
    forest = P.create_forest(ctx, (0, 0, 0, 2, 1, 1), (2, 1, 1), d=2, periodic=(True, True, False),
                             cells_per_block=(8, 8, 1))
    pdf = P.PdfField(forest, P.D2Q9)
    P.fill_equilibrium(pdf, 1.0, (0.0, 0.0))
    P.stream_collide(pdf, P.SRT(1.0))
    blk = forest.local_blocks()[0]
    m0 = sum(float(pdf.src(b).interior.sum()) for b in forest.local_blocks())
    pdf.src(blk).interior[0, 3, 2] = P.equilibrium(1.3, (0.0, 0.0), P.D2Q9)
    m1 = sum(float(pdf.src(b).interior.sum()) for b in forest.local_blocks())
    assert m1 > m0 + 0.29
    for _ in range(5):
        P.stream_collide(pdf, P.SRT(1.0))
    m2 = sum(float(pdf.src(b).interior.sum()) for b in forest.local_blocks())
    assert abs(m2 - m1) < 1e-13


# ------------------------------------------------------------ multi-rank
def _rank_prog(ctx, spec):
    api = cases.b200_api()
    return cases.run_case(api, ctx, spec)


@pytest.mark.parametrize("n_ranks", [2, 4])
def test_rank_invariance_bitwise_zslabs(api, n_ranks):
    """z-slab partition over P ranks (overlapped boundary/interior kernels +
    halo of crossing directions) == 1 rank, bitwise (test_lbm.py:452-471).
    Ranks share the one GPU of the test box; the halo is staged over gloo."""
    import paper_1909_13772_b200 as P
    spec = dict(stencil="D3Q19", dims=(16, 12, 16), root_dims=(1, 1, 4),
                periodic=(True, True, False),
                geometry=dict(kind="spheres", seed=4, rmin=2.0, rmax=3.5, frac=0.2, walls_z=True),
                model=("TRT_magic", 1.7), force=("Guo", (1e-4, 0.0, 2e-5)), init=("random", 9),
                steps=12, snapshots=(1, 12), macro=True, layout="fzyx")
    base = cases.run_case(api, _ctx(), spec)
    multi = P.run(n_ranks, _rank_prog, spec, backend="gloo", device="cuda")[0]
    for s in spec["snapshots"]:
        assert multi["pdf"][s].tobytes() == base["pdf"][s].tobytes(), s
    assert multi["macro"][0].tobytes() == base["macro"][0].tobytes()
    assert multi["links"] == base["links"]
    ores = cases.oracle_run(spec, oracle)
    assert base["pdf"][12].tobytes() == ores["pdf"][12].tobytes()


def test_rank_invariance_periodic_z_two_ranks(api):
    import paper_1909_13772_b200 as P
    spec = dict(stencil="D3Q27", dims=(10, 8, 12), root_dims=(1, 1, 2),
                periodic=(True, True, True), geometry=None, model=("SRT", 1.6), force=None,
                init=("random", 1), steps=8, snapshots=(8,), layout="zyxf")
    base = cases.run_case(api, _ctx(), spec)
    multi = P.run(2, _rank_prog, spec, backend="gloo", device="cuda")[0]
    assert multi["pdf"][8].tobytes() == base["pdf"][8].tobytes()
    assert base["pdf"][8].tobytes() == cases.oracle_run(spec, oracle)["pdf"][8].tobytes()


def test_rate_field_change_between_sweeps_matches_oracle(api):
    """Per-cell SRT rates (lbm/sweep.py:111-146) are read on every sweep:
    editing the rate field between calls re-collides the stored state with
    the new rates (oracle, bitwise); out-of-range rates raise."""
    import paper_1909_13772_b200 as P
    spec = dict(cases.CASES["d3q19_srt_omegafield"])
    nx, ny, nz = spec["dims"]
    ctx = _ctx()
    forest = P.create_forest(ctx, (0, 0, 0, 1, 1, 1), (1, 1, 1), periodic=(True, True, True),
                             cells_per_block=(nx, ny, nz))
    pdf = P.PdfField(forest, P.D3Q19, layout="fzyx")
    P.fill_equilibrium(pdf)
    rho, u = cases.workloads.random_rho_u((nx, ny, nz), 5)
    blk = forest.local_blocks()[0]
    pdf.src(blk).interior[...] = P.equilibrium(rho, u, P.D3Q19)
    forest.register_data("omega", P.FieldDataHandler(nf=1, ghost_layers=1))
    om1 = cases.rate_field(spec)
    om2 = np.random.default_rng(99).uniform(0.6, 1.95, size=om1.shape)
    force = P.Guo((2e-5, 0.0, -1e-5))
    blk.data["omega"].interior[..., 0] = om1
    for _ in range(4):
        P.stream_collide(pdf, P.SRT(omega_field="omega"), force=force)
    blk.data["omega"].interior[..., 0] = om2
    for _ in range(3):
        P.stream_collide(pdf, P.SRT(omega_field="omega"), force=force)
    got = pdf.src(blk).interior.copy()
    st = oracle.STENCILS["D3Q19"]
    full = np.zeros((st.q, nz + 2, ny + 2, nx + 2))
    full[:, 1:-1, 1:-1, 1:-1] = np.moveaxis(oracle.equilibrium(rho, u, st), 3, 0)
    feq0 = oracle.equilibrium(np.ones((nz + 2, ny + 2, nx + 2)), np.zeros((nz + 2, ny + 2, nx + 2, 3)), st)
    ghost = np.ones((nz + 2, ny + 2, nx + 2), bool)
    ghost[1:-1, 1:-1, 1:-1] = False
    full[:, ghost] = np.moveaxis(feq0, 3, 0)[:, ghost]
    doms = []
    for om in (om1, om2):
        of = np.zeros((nz + 2, ny + 2, nx + 2))
        of[1:-1, 1:-1, 1:-1] = om
        doms.append(oracle.Domain(st, (nx, ny, nz), (True, True, True),
                                  oracle.Model("SRT", omega=0.0, omega_field=of,
                                               force=(2e-5, 0.0, -1e-5))))
    doms[0].set_full(full)
    doms[0].run(4)
    doms[1].set_full(doms[0].a)
    doms[1].run(3)
    assert got.tobytes() == doms[1].rform().tobytes()
    blk.data["omega"].interior[0, 0, 0, 0] = 2.0
    with pytest.raises(P.ValidationError):
        P.stream_collide(pdf, P.SRT(omega_field="omega"))


def test_rate_field_fp32_within_tolerance(api):
    spec = dict(cases.CASES["d3q19_srt_omegafield"])
    spec.update(steps=100, snapshots=(100,))
    res = cases.run_case(api, _ctx(), spec, pdf_kwargs={"dtype": "float32"})
    ores = cases.oracle_run(spec, oracle)
    a, b = res["pdf"][100], ores["pdf"][100]
    rel = float(np.max(np.abs(a - b) / np.abs(b)))
    assert rel < TOL_F32_REL, rel


def test_stream_collide_n_graph_replay_bitwise(api):
    """stream_collide_n (two-step CUDA graph replay + odd remainder) equals
    the per-call loop bit for bit, and the oracle."""
    import paper_1909_13772_b200 as P
    spec = dict(cases.CASES["c1_trt_guo_porous"])
    spec.update(steps=11, snapshots=(11,))
    base = cases.run_case(api, _ctx(), spec)
    orc = cases.oracle_run(spec, oracle)
    assert base["pdf"][11].tobytes() == orc["pdf"][11].tobytes()
    # same case, time loop replaced by stream_collide_n
    api2 = cases.b200_api()
    calls = {"n": 0}

    def collide_n(pdf, model, *, force=None, handling=None):
        calls["n"] += 1
        if calls["n"] == 1:
            P.stream_collide(pdf, model, force=force, handling=handling)
            P.stream_collide_n(pdf, model, 10, force=force, handling=handling)
    api2.stream_collide = collide_n
    spec2 = dict(spec, snapshots=(1,))
    got = cases.run_case(api2, _ctx(), dict(spec2, steps=1))
    assert got["pdf"][1].tobytes() == base["pdf"][11].tobytes()


@pytest.mark.parametrize("name", sorted(cases.CASES))
def test_fp32_every_golden_case_within_1e5_relative(api, name):
    """fp32 storage with fp32 centred arithmetic on every golden case (all
    stencils, models, forces and boundary types) against the reference's fp64
    golden vectors at BASELINE's 1e-5 relative tolerance."""
    spec = cases.CASES[name]
    res = cases.run_case(api, _ctx(), spec, pdf_kwargs={"dtype": "float32"})
    gold = np.load(GOLDEN / f"{name}.npz")
    for s, arr in res["pdf"].items():
        ref = gold[f"pdf_{s}"]
        rel = float(np.max(np.abs(arr - ref) / np.abs(ref)))
        assert rel < TOL_F32_REL, (name, s, rel)


# ------------------------------------------------------------ fused halo
_HALO_SPEC = dict(stencil="D3Q19", dims=(16, 12, 16), root_dims=(1, 1, 4),
                  periodic=(True, True, False),
                  geometry=dict(kind="spheres", seed=4, rmin=2.0, rmax=3.5, frac=0.2, walls_z=True),
                  model=("TRT_magic", 1.7), force=("Guo", (1e-4, 0.0, 2e-5)), init=("random", 9),
                  steps=12, snapshots=(1, 12), macro=True, layout="fzyx")


@pytest.mark.parametrize("n_ranks", [2, 4])
def test_fused_peer_halo_thread_ranks_bitwise(api, n_ranks):
    """z-slab ranks as threads of one process, each with its own streams:
    the boundary kernel stores the crossing directions into the neighbour's
    ghost plane and the phases are ordered by stream flags
    (lbm_stream_signal / lbm_stream_wait) - the device path of a multi-GPU
    run.  Bitwise equal to 1 rank and to the oracle."""
    import paper_1909_13772_b200 as P
    from paper_1909_13772_b200 import halo
    seen = []
    orig = halo.PeerHalo.boundary

    def spy(self, *a, **k):
        seen.append(self.kind)
        return orig(self, *a, **k)
    halo.PeerHalo.boundary = spy
    try:
        multi = P.run(n_ranks, _rank_prog, _HALO_SPEC, backend="threads", device="cuda",
                      timeout=300)[0]
    finally:
        halo.PeerHalo.boundary = orig
    assert seen and set(seen) == {"peer-device"}
    base = cases.run_case(api, _ctx(), _HALO_SPEC)
    for s in _HALO_SPEC["snapshots"]:
        assert multi["pdf"][s].tobytes() == base["pdf"][s].tobytes(), s
    assert multi["macro"][0].tobytes() == base["macro"][0].tobytes()
    assert multi["macro"][1].tobytes() == base["macro"][1].tobytes()
    assert base["pdf"][12].tobytes() == cases.oracle_run(_HALO_SPEC, oracle)["pdf"][12].tobytes()


def test_fused_peer_halo_periodic_z_two_thread_ranks(api):
    """P = 2 periodic: both faces of a rank face the same peer (two flag
    words, two ghost planes)."""
    import paper_1909_13772_b200 as P
    spec = dict(stencil="D3Q27", dims=(10, 8, 12), root_dims=(1, 1, 2),
                periodic=(True, True, True), geometry=None, model=("SRT", 1.6), force=None,
                init=("random", 1), steps=8, snapshots=(8,), layout="zyxf")
    base = cases.run_case(api, _ctx(), spec)
    multi = P.run(2, _rank_prog, spec, backend="threads", device="cuda", timeout=300)[0]
    assert multi["pdf"][8].tobytes() == base["pdf"][8].tobytes()


def test_fused_peer_halo_ipc_processes_host_ordered(api, monkeypatch):
    """Ranks as processes sharing the GPU: peers' buffers opened from CUDA
    IPC handles and written by the boundary kernel; phases host-ordered
    (processes on one GPU must not wait on each other on the device)."""
    import paper_1909_13772_b200 as P
    monkeypatch.setenv("LBM_B200_HALO", "peer")
    multi = P.run(2, _rank_prog, _HALO_SPEC, backend="gloo", device="cuda")[0]
    base = cases.run_case(api, _ctx(), _HALO_SPEC)
    for s in _HALO_SPEC["snapshots"]:
        assert multi["pdf"][s].tobytes() == base["pdf"][s].tobytes(), s


def test_fused_peer_halo_fp32_thread_ranks(api):
    """fp32 storage through the fused halo == fp32 on one rank, bitwise."""
    import paper_1909_13772_b200 as P
    kw = {"dtype": "float32"}
    base = cases.run_case(api, _ctx(), _HALO_SPEC, pdf_kwargs=kw)
    multi = P.run(4, _rank_prog_kw, _HALO_SPEC, kw, backend="threads", device="cuda",
                  timeout=300)[0]
    for s in _HALO_SPEC["snapshots"]:
        assert multi["pdf"][s].tobytes() == base["pdf"][s].tobytes(), s


def _rank_prog_kw(ctx, spec, kw):
    return cases.run_case(cases.b200_api(), ctx, spec, pdf_kwargs=kw)


def test_stream_flag_signal_orders_a_second_stream(api):
    """lbm_stream_signal / lbm_stream_wait: work queued behind a wait on
    stream B runs only after stream A's earlier writes and its signal.
    The signal is enqueued before the wait: streams of one context may share
    a hardware queue, and a wait enqueued ahead of its own signal could then
    block it (the fused halo enqueues every signal of a phase before any
    wait for the same reason)."""
    import ctypes
    import torch
    from paper_1909_13772_b200 import _lib
    dev = torch.device("cuda")
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    data = torch.zeros(1 << 22, dtype=torch.float64, device=dev)
    out = torch.empty_like(data)
    torch.cuda.synchronize()
    sa, sb = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    fp = ctypes.c_void_p(flag.data_ptr())
    with torch.cuda.stream(sa):
        torch.cuda._sleep(2_000_000)         # keep A busy well past B's launch
        data.fill_(3.0)
    _lib.call("lbm_stream_signal", fp, 1, _lib.stream_ptr(sa))
    _lib.call("lbm_stream_wait", fp, 1, _lib.stream_ptr(sb))
    with torch.cuda.stream(sb):
        out.copy_(data)                      # must see the fill
    torch.cuda.synchronize()
    assert float(out.min()) == 3.0 and float(out.max()) == 3.0
    assert int(flag.item()) == 1


def test_fused_peer_halo_typed_links_two_thread_ranks(api):
    """D3Q27 raw-moment MRT cavity with the UBB lid, split over 2 z-slab
    thread ranks: dense-MRT peer instantiation, typed (UBB) links and wall
    links next to the halo planes - bitwise equal to 1 rank."""
    import paper_1909_13772_b200 as P
    spec = dict(cases.CASES["c2_d3q27_rawmrt_cavity"])
    spec.update(dims=(8, 8, 12), root_dims=(1, 1, 2), steps=12, snapshots=(5, 12))
    base = cases.run_case(api, _ctx(), spec)
    multi = P.run(2, _rank_prog, spec, backend="threads", device="cuda", timeout=300)[0]
    for s in spec["snapshots"]:
        assert multi["pdf"][s].tobytes() == base["pdf"][s].tobytes(), s


def _rank_prog_broken_ipc(ctx, spec):
    import warnings
    from paper_1909_13772_b200 import device, halo
    if ctx.rank == 1:
        def broken(self, handle, offset):
            raise RuntimeError("simulated IPC failure")
        halo.PeerHalo._open = broken
    kinds = []
    make = halo.make_halo

    def recording(lat):
        h = make(lat)
        kinds.append(h.kind)
        return h
    halo.make_halo = recording
    with warnings.catch_warnings(record=True) as caught:
        warnings.simplefilter("always")
        res = cases.run_case(cases.b200_api(), ctx, spec)
    fell_back = any("fused peer halo unavailable" in str(w.message) for w in caught)
    return res, kinds, fell_back


def test_fused_peer_halo_setup_failure_falls_back_collectively(api, monkeypatch):
    """One rank failing to map its neighbour makes EVERY rank fall back to
    the send/recv transport (no lone raise, no hang); results stay bitwise."""
    import paper_1909_13772_b200 as P
    monkeypatch.setenv("LBM_B200_HALO", "peer")
    spec = dict(_HALO_SPEC, root_dims=(1, 1, 2), snapshots=(12,))
    per_rank = P.run(2, _rank_prog_broken_ipc, spec, backend="gloo", device="cuda")
    for res, kinds, fell_back in per_rank:
        assert kinds == ["staged"] and fell_back
    base = cases.run_case(api, _ctx(), spec)
    assert per_rank[0][0]["pdf"][12].tobytes() == base["pdf"][12].tobytes()


# ------------------------------------------- parameter identity
def _random_lattice(P, dims, seed, stencil="D3Q19"):
    ctx = _ctx()
    nx, ny, nz = dims
    forest = P.create_forest(ctx, (0, 0, 0, 1, 1, 1), (1, 1, 1), periodic=(True, True, True),
                             cells_per_block=(nx, ny, nz))
    st = getattr(P, stencil)
    pdf = P.PdfField(forest, st, layout="fzyx")
    P.fill_equilibrium(pdf)
    rho, u = cases.workloads.random_rho_u(dims, seed)
    blk = forest.local_blocks()[0]
    pdf.src(blk).interior[...] = P.equilibrium(rho, u, st)
    return forest, pdf, blk


def _oracle_random(dims, seed, model, steps):
    st = oracle.STENCILS["D3Q19"]
    spec = dict(stencil="D3Q19", dims=dims, root_dims=(1, 1, 1), periodic=(True, True, True),
                geometry=None, init=("random", seed))
    full, _, _ = cases.oracle_inputs(spec, oracle)
    d = oracle.Domain(st, dims, (True, True, True), model)
    d.set_full(full)
    d.run(steps)
    return d


def test_mrt_tables_of_two_lattices_across_graph_replays(api):
    """Two MRT lattices with different rates on one device, each advanced
    through stream_collide_n (captured two-step graphs): the constant-memory
    tables a replay reads are re-bound to its own model (lbm_bind_params)."""
    import paper_1909_13772_b200 as P
    dims = (12, 10, 8)
    ra = [1.0] * 19
    ra[9:16] = [1.4] * 7
    rb = [1.2] * 19
    rb[9:16] = [1.8] * 7
    _, pa, ba = _random_lattice(P, dims, 41)
    _, pb, bb = _random_lattice(P, dims, 42)
    ma, mb = P.MRT(P.D3Q19, ra), P.MRT(P.D3Q19, rb)
    force = P.Guo((1e-4, 0.0, -2e-5))
    P.stream_collide_n(pa, ma, 6, force=force)
    P.stream_collide_n(pb, mb, 6, force=force)
    P.stream_collide_n(pa, ma, 6, force=force)
    st = oracle.STENCILS["D3Q19"]
    M = oracle.moment_basis(st)
    for pdf, blk, rates, seed, steps in ((pa, ba, ra, 41, 12), (pb, bb, rb, 42, 6)):
        model = oracle.Model("MRT", M=M.astype(np.float64), Minv=oracle.basis_inverse(M),
                             S=np.array(rates), force=(1e-4, 0.0, -2e-5))
        want = _oracle_random(dims, seed, model, steps).rform()
        assert pdf.src(blk).interior.tobytes() == want.tobytes(), rates


def test_mutated_model_and_wall_velocity_take_effect(api):
    """Parameters are keyed by value, not object identity: a lid velocity
    ramped on the same BoundaryHandling and a rate changed on the same SRT
    object apply to the next sweep, as in the reference (boundary.py:165-171,
    sweep.py:116)."""
    import paper_1909_13772_b200 as P
    spec = dict(stencil="D3Q19", dims=(10, 8, 9), root_dims=(1, 1, 1),
                periodic=(False, False, False), geometry=dict(kind="cavity"),
                model=("SRT", 1.5), force=None, init=("rest",),
                ubb_velocity=(0.05, 0.0, 0.0), layout="fzyx")
    forest, pdf, handling, model, force, st = cases.setup_case(cases.b200_api(), _ctx(), spec)
    phases = (((0.05, 0.0, 0.0), 1.5), ((0.08, 0.01, 0.0), 1.5), ((0.08, 0.01, 0.0), 1.1))
    for uw, om in phases:
        handling.ubb_velocity = uw
        model.omega = om
        for _ in range(3):
            P.stream_collide(pdf, model, handling=handling)
    got = pdf.src(forest.local_blocks()[0]).interior.copy()
    full, flags, bits = cases.oracle_inputs(spec, oracle)
    ost = oracle.STENCILS["D3Q19"]
    for uw, om in phases:
        d = oracle.Domain(ost, spec["dims"], spec["periodic"], oracle.Model("SRT", omega=om),
                          flags, bits, ubb_velocity=uw)
        d.set_full(full)
        d.run(3)
        full = d.a.copy()
    assert got.tobytes() == d.rform().tobytes()
