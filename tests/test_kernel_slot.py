"""Kernel slot: `paper_1909_13772_b200.kernel_slot` is the
"b200" backend of blocksim._kernels (pkg/src/blocksim/_kernels/__init__.py:
10-37).  Its collide / stream_pull must reproduce the reference's own
impl.collide / impl.stream_pull (_core_py.py:70-218) bit for bit on the
goldens tests/golden/make_golden.py recorded from the reference (flagged box
with its ghost ring, AoS and strided SoA views, every model and force the
slot accepts, a per-cell omega_window, a multi-bit fluid mask).

The CPU tests pin the oracle against the same goldens; the GPU tests run
the slot itself through the C-ABI (lbm_slot_collide / lbm_slot_stream_pull).
"""
from pathlib import Path

import numpy as np
import pytest

import oracle

GOLD = np.load(Path(__file__).resolve().parent / "golden" / "slot.npz")
CASES = sorted({k.split("__")[0] for k in GOLD.files if not k.startswith("pull_")})
PULLS = ("D2Q9", "D3Q19", "D3Q27")


def _params(name):
    p = {}
    for k in GOLD.files:
        if k.startswith(f"{name}__p_"):
            v = GOLD[k]
            key = k[len(f"{name}__p_"):]
            p[key] = v.item() if v.ndim == 0 else (v.tolist() if key in ("cx", "cy", "cz", "w", "opp", "force") else v)
    p.setdefault("omega_window", None)
    if f"{name}__window" in GOLD.files:
        p["omega_window"] = GOLD[f"{name}__window"]
    if "force" in p:
        p["force"] = tuple(p["force"])
    return p


def _view(name):
    f = GOLD[f"{name}__in"].copy()
    if str(GOLD[f"{name}__layout"]) == "soa":
        raw = np.ascontiguousarray(np.moveaxis(f, 3, 0))
        return raw, np.moveaxis(raw, 0, 3)
    return f, f


def test_slot_goldens_cover_the_contract():
    assert len(CASES) >= 30
    modes = {int(GOLD[f"{n}__mode"]) for n in CASES}
    assert modes == {0, 1, 2}
    assert any(f"{n}__window" in GOLD.files for n in CASES)
    assert any(str(GOLD[f"{n}__layout"]) == "soa" for n in CASES)


@pytest.mark.parametrize("name", [n for n in CASES if f"{n}__window" not in GOLD.files])
def test_oracle_collide_matches_slot_golden(name):
    """The C oracle's collide on the fluid cells == the reference slot."""
    p = _params(name)
    q = len(p["w"])
    st = oracle.STENCILS[{9: "D2Q9", 19: "D3Q19", 27: "D3Q27"}[q]]
    mode = int(GOLD[f"{name}__mode"])
    fm = int(p["force_mode"])
    force = p["force"] if fm else None
    kind = "shift" if fm == 2 else "guo"
    if mode == 0:
        m = oracle.Model("SRT", omega=p["omega"], force=force, force_kind=kind)
    elif mode == 1:
        m = oracle.Model("TRT", omega_e=p["omega_e"], omega_o=p["omega_o"], force=force,
                         force_kind=kind)
    else:
        m = oracle.Model("MRT", M=np.asarray(p["M"], dtype=np.float64), Minv=p["Minv"],
                         S=np.asarray(p["S"], dtype=np.float64), force=force, force_kind=kind)
        if fm:
            m.G = np.ascontiguousarray(p["guo_matrix"], dtype=np.float64)
    f = GOLD[f"{name}__in"]
    fluid = (GOLD[f"{name}__flags"] & GOLD[f"{name}__bits"]) != 0
    want = GOLD[f"{name}__out"]
    got = f.copy()
    got[fluid] = oracle.collide_cells(st, f[fluid], m)
    assert got.tobytes() == want.tobytes(), float(np.abs(got - want).max())


@pytest.mark.parametrize("sname", PULLS)
def test_pull_golden_is_the_pull_rule(sname):
    """R[x, i] = G[x - c_i, i] on the interior, ghosts untouched."""
    st = oracle.STENCILS[sname]
    src, dst = GOLD[f"pull_{sname}__src"], GOLD[f"pull_{sname}__dst"].copy()
    Z, Y, X, q = src.shape
    for i in range(q):
        dst[1:Z - 1, 1:Y - 1, 1:X - 1, i] = src[1 - st.cz[i]:Z - 1 - st.cz[i],
                                                1 - st.cy[i]:Y - 1 - st.cy[i],
                                                1 - st.cx[i]:X - 1 - st.cx[i], i]
    assert dst.tobytes() == GOLD[f"pull_{sname}__out"].tobytes()


def test_slot_module_surface():
    """Same names as the reference's slot (no GPU needed to import)."""
    from paper_1909_13772_b200 import kernel_slot
    assert kernel_slot.BACKEND == "b200"
    mod, label = kernel_slot.get_backend("b200")
    assert mod is kernel_slot and label == "b200"
    with pytest.raises(ValueError):
        kernel_slot.get_backend("cython")
    assert callable(kernel_slot.collide) and callable(kernel_slot.stream_pull)


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_slot_collide_bitwise_vs_reference(name):
    from paper_1909_13772_b200 import kernel_slot
    raw, view = _view(name)
    flags = GOLD[f"{name}__flags"]
    kernel_slot.collide(view, flags, GOLD[f"{name}__bits"], int(GOLD[f"{name}__mode"]),
                        _params(name))
    got = np.ascontiguousarray(view)
    want = GOLD[f"{name}__out"]
    assert got.tobytes() == want.tobytes(), float(np.abs(got - want).max())


@pytest.mark.gpu
@pytest.mark.parametrize("sname", PULLS)
def test_slot_stream_pull_bitwise_vs_reference(sname):
    from paper_1909_13772_b200 import kernel_slot
    st = oracle.STENCILS[sname]
    src = GOLD[f"pull_{sname}__src"]
    dst = GOLD[f"pull_{sname}__dst"].copy()
    # a strided (SoA) destination view, as the reference's fzyx fields give
    raw = np.ascontiguousarray(np.moveaxis(dst, 3, 0))
    kernel_slot.stream_pull(src, np.moveaxis(raw, 0, 3), st.cx, st.cy, st.cz, 1)
    assert np.moveaxis(raw, 0, 3).tobytes() == GOLD[f"pull_{sname}__out"].tobytes()


@pytest.mark.gpu
def test_slot_rejects_foreign_velocity_sets():
    import paper_1909_13772_b200 as P
    from paper_1909_13772_b200 import kernel_slot
    name = CASES[0]
    p = _params(name)
    p["cx"] = list(reversed(p["cx"]))
    raw, view = _view(name)
    with pytest.raises(P.ValidationError):
        kernel_slot.collide(view, GOLD[f"{name}__flags"], 1, int(GOLD[f"{name}__mode"]), p)


# --------------------------------------------- BoundaryHandling.apply
APPLY = np.load(Path(__file__).resolve().parent / "golden" / "apply.npz")
APPLY_DIMS = {"D3Q19": (7, 6, 5), "D3Q27": (6, 5, 6), "D2Q9": (9, 7, 1)}


def _apply_flags(reg, dims, d):
    """tests/golden/make_golden.py:apply_flags, restated."""
    nx, ny, nz = dims
    f = np.full((nz, ny, nx), reg["NoSlip"], dtype=np.uint32)
    inner = (slice(1, -1),) * 3 if d == 3 else (slice(None), slice(1, -1), slice(1, -1))
    f[inner] = reg["Fluid"]
    if d == 3:
        f[-1, 1:-1, 1:-1] = reg["UBB"]
        f[1:-1, 1:-1, -1] = reg["Pressure"]
    else:
        f[:, -1, 1:-1] = reg["UBB"]
        f[:, 1:-1, -1] = reg["Pressure"]
    f[nz // 2, ny // 2, nx // 2] = reg["NoSlip"]
    return f


@pytest.mark.parametrize("name", sorted(APPLY_DIMS))
def test_oracle_apply_matches_reference(name):
    """The C oracle's link rule (orc_apply_links) == the reference's apply."""
    import ctypes
    st = oracle.STENCILS[name]
    dims = APPLY_DIMS[name]
    d = 2 if name == "D2Q9" else 3
    bits = {"Fluid": 1, "NoSlip": 2, "UBB": 4, "Pressure": 8, "Solid": 16}
    nx, ny, nz = dims
    Z, Y, X = nz + 2, ny + 2, nx + 2
    flags = np.zeros((Z, Y, X), dtype=np.uint32)
    flags[1:-1, 1:-1, 1:-1] = _apply_flags(bits, dims, d)
    src = np.ascontiguousarray(np.moveaxis(APPLY[f"{name}__src"], 3, 0))
    dst = np.ascontiguousarray(np.moveaxis(APPLY[f"{name}__dst"], 3, 0))
    L = oracle.lbm_oracle._Links()
    L.fluid, L.noslip, L.ubb, L.pressure = 1, 2, 4, 8
    L.uwx, L.uwy, L.uwz, L.rho0, L.rho_w = 0.03, -0.01, 0.02, 0.99, 1.02
    cst = oracle.lbm_oracle._cstencil(st)
    oracle.lib().orc_apply_links(ctypes.byref(cst), oracle.lbm_oracle._ptr(src),
                                 oracle.lbm_oracle._ptr(dst), oracle.lbm_oracle._ptr(flags),
                                 X, Y, Z, ctypes.byref(L))
    assert np.moveaxis(dst, 0, 3).tobytes() == APPLY[f"{name}__out"].tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(APPLY_DIMS))
def test_boundary_handling_apply_bitwise_vs_reference(name):
    import paper_1909_13772_b200 as P
    st = getattr(P, name)
    dims = APPLY_DIMS[name]
    forest = P.create_forest(P.Context(), (0, 0, 0, 1, 1, 1), (1, 1, 1), d=st.d,
                             periodic=(False, False, False), cells_per_block=dims)
    reg = P.ensure_flags(forest).registry
    blk = forest.local_blocks()[0]
    blk.data["flags"].interior[...] = _apply_flags(reg, dims, st.d)
    h = P.BoundaryHandling(forest, st, ubb_velocity=(0.03, -0.01, 0.02),
                           pressure_density=1.02, reference_density=0.99)
    h.freeze()
    dst = APPLY[f"{name}__dst"].copy()
    h.apply(blk, APPLY[f"{name}__src"], dst)
    assert dst.tobytes() == APPLY[f"{name}__out"].tobytes()
