"""Link-bit map (lbm_build_linkbits / lbm_fused_step_bits, ABI 7).

NoSlip-only lattices sweep with one bit per cell instead of the 4 B/cell
cell mask; the kernel re-derives each cell's link bits from its 3x3 rows of
neighbour bits.  These tests check that

* the map is taken where it applies and results stay bitwise equal to the
  oracle (and to the cell-mask kernel, LBM_B200_LINKBITS=0), on grids whose
  x extent is not a multiple of 32 and with periodic x/y edges;
* the map means what include/lbm_b200.h says: decoded on the host with
  numpy, it reproduces the cell mask on every cell, and the overlapping
  halves of neighbouring words agree;
* typed links (UBB / Pressure), moving walls and flags edited after
  freeze() keep the cell mask (the device check rejects the map).
"""
from pathlib import Path

import numpy as np
import pytest

import cases
import oracle

pytestmark = pytest.mark.gpu

GOLDEN = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def api():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return cases.b200_api()


@pytest.fixture(autouse=True)
def _linkbits_on(monkeypatch):
    """The map is opt-in (device.linkbits_enabled); tests that compare with
    the cell-mask kernel switch it off again with LBM_B200_LINKBITS=0."""
    monkeypatch.setenv("LBM_B200_LINKBITS", "1")


def _ctx():
    import paper_1909_13772_b200 as P
    return P.Context()


RAGGED = dict(stencil="D3Q19", dims=(37, 21, 9), root_dims=(1, 1, 1),
              periodic=(True, True, False),
              geometry=dict(kind="spheres", seed=5, rmin=2.0, rmax=3.5, frac=0.2, walls_z=True),
              model=("TRT_magic", 1.7), force=("Guo", (1e-4, 2e-5, 0.0)), init=("random", 9),
              steps=12, snapshots=(12,), layout="fzyx")
WIDE = dict(RAGGED, dims=(70, 6, 5), geometry=dict(kind="spheres", seed=6, rmin=1.5, rmax=2.5,
                                                     frac=0.25, walls_z=True),
            model=("SRT", 1.4), force=None, steps=9, snapshots=(9,))


def _run(api, spec):
    forest, pdf, handling, model, force, st = cases.setup_case(api, _ctx(), spec)
    snaps = {}
    for s in range(1, spec["steps"] + 1):
        api.stream_collide(pdf, model, force=force, handling=handling)
        if s in spec["snapshots"]:
            snaps[s] = api.gather_slice(forest, "pdf", (0, 0, 0), forest.global_cells(0))
    return snaps, handling, pdf


def _spec(name):
    return dict(cases.CASES.get(name) or cases.DIGEST_CASES.get(name) or
                {"ragged": RAGGED, "wide": WIDE}[name])


@pytest.mark.parametrize("name", ["ragged", "wide", "c1_trt_guo_porous", "c1_trt_guo_porous_24"])
def test_linkbits_taken_and_bitwise(api, name, monkeypatch):
    import torch
    spec = _spec(name)
    got, handling, _ = _run(api, spec)
    masks = handling.masks
    assert isinstance(masks._linkbits, torch.Tensor), "link-bit map not taken"
    ref = cases.oracle_run(spec, oracle)["pdf"]
    for s, a in got.items():
        assert a.tobytes() == ref[s].tobytes(), f"step {s}"
    monkeypatch.setenv("LBM_B200_LINKBITS", "0")
    plain, _, _ = _run(api, spec)
    for s, a in plain.items():
        assert a.tobytes() == got[s].tobytes(), f"cell-mask kernel, step {s}"


@pytest.mark.parametrize("name", ["ragged", "wide", "c1_trt_guo_porous_24"])
def test_linkbits_layout_decodes_to_the_cell_mask(api, name):
    spec = _spec(name)
    _, handling, pdf = _run(api, dict(spec, steps=1, snapshots=()))
    masks = handling.masks
    lat = pdf.lattice
    cm = masks.cellmask.cpu().numpy().view(np.uint32)
    nz, ny, nx = cm.shape
    bw = (nx + 31) // 32
    words = masks._linkbits.cpu().numpy().view(np.uint64).reshape(nz + 2, ny + 2, bw)
    assert int(lat.grid.nx) == nx
    # bit b of word w is ghost-inclusive x = 32 w + b; the upper half of
    # word w and the lower half of word w + 1 describe the same cells
    lo = (words & np.uint64(0xFFFFFFFF)).astype(np.uint64)
    hi = (words >> np.uint64(32)).astype(np.uint64)
    assert np.array_equal(hi[:, :, :-1], lo[:, :, 1:])
    X = nx + 2
    n = np.zeros((nz + 2, ny + 2, X), dtype=np.uint32)
    for xg in range(X):
        w = min(xg // 32, bw - 1)
        n[:, :, xg] = ((words[:, :, w] >> np.uint64(xg - 32 * w)) & np.uint64(1)).astype(np.uint32)
    st = oracle.STENCILS[spec["stencil"]]
    cx, cy, cz = (np.asarray(c) for c in (st.cx, st.cy, st.cz))
    own = n[1:-1, 1:-1, 1:-1]
    code = np.where(own == 0, np.uint32(1), np.uint32(0))
    for i in range(1, len(cx)):
        src = n[1 - cz[i]:nz + 1 - cz[i], 1 - cy[i]:ny + 1 - cy[i], 1 - cx[i]:nx + 1 - cx[i]]
        code |= np.where(own == 0, src << np.uint32(i), np.uint32(0)).astype(np.uint32)
    assert np.array_equal(code, cm)


@pytest.mark.parametrize("name", ["c2_d3q27_trt_cavity", "d2q9_pressure_box", "d3q19_flag_edits"])
def test_typed_and_edited_lattices_keep_the_cell_mask(api, name):
    """Typed links never build a map; flags edited after freeze() give a
    refreshed mask whose map the device check rejects - results stay bitwise
    equal to the reference goldens either way."""
    spec = _spec(name)
    res = cases.run_case(api, _ctx(), spec)
    gold = np.load(GOLDEN / f"{name}.npz")
    for s in spec["snapshots"]:
        assert res["pdf"][s].tobytes() == gold[f"pdf_{s}"].tobytes()
    forest, pdf, handling, model, force, st = cases.setup_case(api, _ctx(), spec)
    api.stream_collide(pdf, model, force=force, handling=handling)
    if name == "d3q19_flag_edits":
        assert handling.masks._linkbits is not False   # frozen NoSlip-only mask: map taken
        cases._edit_flag(api, forest, 2, 2, 2, "NoSlip")
        api.stream_collide(pdf, model, force=force, handling=handling)
        refreshed = handling.sweep_masks()
        assert refreshed is not handling.masks
        assert refreshed._linkbits is False
    else:
        assert handling.masks.linkbits(pdf.lattice) is None


@pytest.mark.parametrize("stencil,model,force", [
    ("D3Q19", ("TRT_magic", 1.7), ("Guo", (1e-5, 0.0, 0.0))),     # k_fused_z2 (fp32)
    ("D3Q27", ("MRT_raw", 1.9, 1.0), None),                       # factorised D3Q27 MRT
])
def test_linkbits_fp32_kernels_bitwise_vs_cell_mask(api, stencil, model, force, monkeypatch):
    """fp32 storage: the link-bit kernels give the same bits as the cell-mask
    kernels (same arithmetic, only the source of the link bits differs), and
    stay within the BASELINE 1e-5 relative of the fp64 oracle."""
    import torch
    spec = dict(stencil=stencil, dims=(45, 19, 14), root_dims=(1, 1, 1),
                periodic=(True, True, False),
                geometry=dict(kind="spheres", seed=8, rmin=2.0, rmax=3.5, frac=0.2, walls_z=True),
                model=model, force=force, init=("random", 4), steps=20, snapshots=(20,),
                layout="fzyx")

    def run():
        forest, pdf, handling, m, f, st = cases.setup_case(
            api, _ctx(), spec, pdf_kwargs={"dtype": "float32"})
        for _ in range(spec["steps"]):
            api.stream_collide(pdf, m, force=f, handling=handling)
        return api.gather_slice(forest, "pdf", (0, 0, 0), forest.global_cells(0)), handling

    got, handling = run()
    assert isinstance(handling.masks._linkbits, torch.Tensor)
    monkeypatch.setenv("LBM_B200_LINKBITS", "0")
    plain, _ = run()
    assert got.tobytes() == plain.tobytes()
    ref = cases.oracle_run(spec, oracle)["pdf"][20]
    assert float(np.max(np.abs(got - ref) / np.abs(ref))) < 1e-5
