"""Formats either side of the sweep: forest images in the
reference's WBCP byte format, restart from an image, legacy VTK output.

Golden data (tests/golden/snapshot_case.npz, digests.json "snapshot_case")
come from the reference itself (make_golden.py make_snapshot): its image and
VTK files after k sweeps of cases.SNAPSHOT_CASE and the PDFs after
SNAPSHOT_MORE further sweeps.
"""
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

import cases

GOLDEN = Path(__file__).resolve().parent / "golden"
SNAP = np.load(GOLDEN / "snapshot_case.npz")
META = json.loads((GOLDEN / "digests.json").read_text())["snapshot_case"]
IMAGE = SNAP["image"].tobytes()


def sha(b) -> str:
    return hashlib.sha256(b).hexdigest()


def _forest(P, ctx, spec):
    nx, ny, nz = spec["dims"]
    R = spec["root_dims"]
    return P.create_forest(ctx, (0, 0, 0) + tuple(R), R, periodic=spec["periodic"],
                           cells_per_block=(nx // R[0], ny // R[1], nz // R[2]))


def _slots(P, image, spec):
    f = _forest(P, P.Context(device="cpu"), spec)
    return {bid: dict(slots) for bid, slots in f.parse_snapshot(image)}


# ------------------------------------------------------------------ host
def test_wire_buffers_roundtrip_and_tags():
    import paper_1909_13772_b200 as P
    b = P.SendBuffer(debug=True)
    b.pack_int(-7)
    b.pack_float(0.1)
    b.pack_str("wbcp")
    b.pack_array(np.arange(12, dtype=np.uint32).reshape(3, 4))
    b.pack_floats([1.5, -0.0])
    r = P.RecvBuffer(b.getvalue(), debug=True)
    assert r.unpack_int() == -7 and r.unpack_float() == 0.1 and r.unpack_str() == "wbcp"
    assert np.array_equal(r.unpack_array(), np.arange(12, dtype=np.uint32).reshape(3, 4))
    assert r.unpack_floats() == [1.5, -0.0] and r.at_end
    with pytest.raises(P.BufferUnderflowError):
        r.unpack_int()
    r = P.RecvBuffer(b.getvalue(), debug=True)
    with pytest.raises(P.TypeTagError):
        r.unpack_float()
    # release mode: no tags (snapshot format)
    c = P.SendBuffer()
    c.pack_int(3)
    assert len(c) == 8


def test_reference_image_parses_and_roundtrips_on_host(tmp_path):
    """The reference's image loads into this forest (host data only) and is
    re-emitted byte for byte; the VTK files written from the loaded rho/vel
    equal the reference's."""
    import paper_1909_13772_b200 as P
    spec = cases.SNAPSHOT_CASE
    ctx = P.Context(device="cpu")
    forest = _forest(P, ctx, spec)
    P.ensure_flags(forest)
    P.PdfField(forest, P.D3Q19, layout=spec["layout"])
    forest.register_data("rho", P.FieldDataHandler(nf=1, ghost_layers=1))
    forest.register_data("vel", P.FieldDataHandler(nf=3, ghost_layers=1))
    forest.load_snapshot_blocks([IMAGE])
    forest.rebuild_neighborhoods()
    assert len(forest.local_blocks()) == 2
    assert forest.snapshot() == IMAGE
    P.write_vtk(forest, str(tmp_path), "out", spec["steps"], [("rho", "rho"), ("u", "vel")])
    got = {p.name: sha(p.read_bytes()) for p in tmp_path.iterdir()}
    assert got == META["vtk"]


def test_snapshot_validation_errors():
    import paper_1909_13772_b200 as P
    spec = cases.SNAPSHOT_CASE
    f = _forest(P, P.Context(device="cpu"), spec)
    with pytest.raises(P.ValidationError):
        f.parse_snapshot(b"JUNK" + IMAGE[4:])
    with pytest.raises(P.ValidationError):
        f.parse_snapshot(IMAGE[:4] + bytes([9]) + IMAGE[5:])
    wrong = P.create_forest(P.Context(device="cpu"), (0, 0, 0, 1, 1, 4), (1, 1, 4),
                            cells_per_block=(8, 6, 2))
    with pytest.raises(P.ValidationError):
        wrong.parse_snapshot(IMAGE)
    f2 = P.create_forest(P.Context(device="cpu"), (0, 0, 0, 1, 1, 1), (1, 1, 1), d=2,
                         cells_per_block=(4, 4, 1))
    with pytest.raises(P.ValidationError):
        f2.parse_snapshot(IMAGE)


# ------------------------------------------------------------------- GPU
def _split_ghosts(raw, layout, g=1):
    """(interior, ghost shell) of a raw PDF slot array."""
    v = raw if layout == "zyxf" else np.moveaxis(raw, 0, 3)
    inner = v[g:-g, g:-g, g:-g].copy()
    mask = np.ones(v.shape[:3], bool)
    mask[g:-g, g:-g, g:-g] = False
    return inner, v[mask]


@pytest.mark.gpu
def test_snapshot_vtk_and_continuation_match_reference(tmp_path):
    """After k sweeps on the GPU: flags, rho, vel and the dst slot (C(R_{k-1})
    with covered ghosts) are byte-identical to the reference's image; the
    src slot matches on the interior and the uncovered (wall-side) ghosts;
    the VTK files are byte-identical; k + m sweeps equal the reference."""
    import paper_1909_13772_b200 as P
    spec = cases.SNAPSHOT_CASE
    res = cases.run_snapshot_case(cases.b200_api(), P.Context(), spec, str(tmp_path))
    assert {n: sha(b) for n, b in res["vtk"].items()} == META["vtk"]
    assert res["pdf_more"].tobytes() == SNAP["pdf_more"].tobytes()
    mine, ref = _slots(P, res["image"], spec), _slots(P, IMAGE, spec)
    assert sorted(mine) == sorted(ref)
    for bid in ref:
        assert sorted(mine[bid]) == sorted(ref[bid]) == ["flags", "pdf", "pdf.dst", "rho", "vel"]
        for key in ("flags", "rho", "vel", "pdf.dst"):
            assert mine[bid][key] == ref[bid][key], (bid, key)
        a = P.RecvBuffer(mine[bid]["pdf"]).unpack_array()
        b = P.RecvBuffer(ref[bid]["pdf"]).unpack_array()
        ia, ga = _split_ghosts(a, spec["layout"])
        ib, gb = _split_ghosts(b, spec["layout"])
        assert ia.tobytes() == ib.tobytes(), bid
        # ghost planes on the non-periodic z faces are uncovered: exact
        za = (a if spec["layout"] == "zyxf" else np.moveaxis(a, 0, 3))
        zb = (b if spec["layout"] == "zyxf" else np.moveaxis(b, 0, 3))
        lo = bid.root == 0
        plane = 0 if lo else -1
        assert za[plane].tobytes() == zb[plane].tobytes(), bid


@pytest.mark.gpu
def test_restart_from_reference_image(tmp_path):
    """Load the reference's image into the GPU framework, continue m sweeps:
    bitwise equal to the reference's own continuation."""
    import paper_1909_13772_b200 as P
    spec = cases.SNAPSHOT_CASE
    res = cases.run_snapshot_case(cases.b200_api(), P.Context(), spec, str(tmp_path), image=IMAGE)
    assert res["pdf_more"].tobytes() == SNAP["pdf_more"].tobytes()
    assert {n: sha(b) for n, b in res["vtk"].items()} == META["vtk"]
