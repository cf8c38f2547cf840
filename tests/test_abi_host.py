"""CPU tests of the C-ABI library (no compute calls) and the host logic."""
import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

import oracle
import paper_1909_13772_b200 as P
from paper_1909_13772_b200 import _lib, balance, halo
from paper_1909_13772_b200.device import RankBox

HEADER = Path(__file__).resolve().parent.parent / "include" / "lbm_b200.h"


def header_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w]+\*?\s+\*?(lbm_\w+)\(", text, re.M)))


def test_library_loads_and_exports_every_header_symbol():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 15
    assert sorted(syms) == sorted(_lib.EXPORTS)
    for s in syms:
        assert hasattr(lib, s), s
    assert lib.lbm_abi_version() == _lib.ABI_VERSION == 8


def test_library_is_sm100a():
    """The built library carries sm_100a code (cuobjdump listing)."""
    import shutil
    import subprocess
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not Path(exe).exists():
        pytest.skip("cuobjdump unavailable")
    out = subprocess.run([exe, "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_no_kernel_in_two_units():
    """Every kernel is compiled into exactly one unit.  The units differ in
    -fmad (fp64 bitwise units: false, fp32 unit: true) and a kernel in two
    of them shares one host stub, so which copy a launch runs would depend on
    module load order (a fused readout once ran its contracted fp32-unit copy
    and came out 1 ulp off)."""
    import collections
    import shutil
    import subprocess
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not Path(exe).exists():
        pytest.skip("cuobjdump unavailable")
    out = subprocess.run([exe, "-symbols", str(_lib.LIB_PATH)], capture_output=True, text=True)
    names = [ln.split()[-1] for ln in out.stdout.splitlines() if "STO_ENTRY" in ln]
    assert len(names) > 100
    dup = [n for n, c in collections.Counter(names).items() if c > 1]
    assert not dup, f"kernels compiled into more than one unit: {dup[:5]}"


def test_slot_layout_groups_directions_by_cz():
    lib = _lib.load()
    for name in ("D2Q9", "D3Q19", "D3Q27"):
        st = oracle.STENCILS[name]
        slots = [lib.lbm_slot_of(st.q, i) for i in range(st.q)]
        assert sorted(slots) == list(range(st.q))
        order = sorted(range(st.q), key=lambda i: slots[i])
        assert [st.c[i][2] for i in order] == sorted(st.c[i][2] for i in range(st.q))
        for a, b in zip(order, order[1:]):
            if st.c[a][2] == st.c[b][2]:
                assert a < b
    assert lib.lbm_slot_of(19, 19) == -1 and lib.lbm_slot_of(7, 0) == -1


def _grid(q=19, nx=8, ny=6, nz=5, rb=8, lo=1, hi=1):
    g = _lib.Grid()
    g.q, g.real_bytes, g.nx, g.ny, g.nz = q, rb, nx, ny, nz
    g.xoff = 128 // rb
    g.pitch = ((g.xoff + nx + 1 + g.xoff - 1) // g.xoff) * g.xoff
    g.wrap_x = g.wrap_y = 1
    g.zface_lo, g.zface_hi = lo, hi
    return g


@pytest.mark.parametrize("q,ncross", [(19, 5), (27, 9), (9, 0)])
def test_face_spans_cover_crossing_directions(q, ncross):
    g = _grid(q=q)
    spans = halo.face_spans(ctypes.byref(g))
    plane = (g.ny + 2) * g.pitch
    zs = q * plane
    (s0, r0, c0), (s1, r1, c1) = spans[0], spans[1]
    assert c0 == c1 == ncross * plane
    assert s0 == 1 * zs and r1 == (g.nz + 1) * zs          # c_z = -1 run at the front
    assert r0 == (q - ncross) * plane and s1 == g.nz * zs + (q - ncross) * plane
    assert int(_lib.load().lbm_field_elems(ctypes.byref(g))) == (g.nz + 2) * zs


def test_field_elems_rejects_bad_grids():
    g = _grid()
    g.pitch = 4
    assert _lib.load().lbm_field_elems(ctypes.byref(g)) == -1
    g = _grid(q=15)
    assert _lib.load().lbm_field_elems(ctypes.byref(g)) == -1
    assert b"q must be" in _lib.load().lbm_last_error()


def test_plan_ops_pairs_match_for_two_ranks():
    spans = {0: (100, 0, 10), 1: (200, 300, 10)}
    ops = halo.plan_ops(_lib.ZFACE_HALO, _lib.ZFACE_HALO, 1, 1, spans)
    assert [(k, o) for k, _, o, _ in ops] == [("send", 100), ("send", 200), ("recv", 300), ("recv", 0)]
    # the peer's first send (its low face) must land in my high ghost plane
    assert ops[2][2] == spans[1][1]
    assert halo.plan_ops(_lib.ZFACE_GHOST, _lib.ZFACE_WRAP, None, None, spans) == []


class FakeCtx:
    def __init__(self, rank, n):
        self.rank, self.n_ranks = rank, n
        import torch
        self.device = torch.device("cpu")

    def all_gather(self, obj):
        return {r: obj for r in range(self.n_ranks)}


@pytest.mark.parametrize("P_", [1, 2, 4, 8])
def test_zslab_partition_rank_k_owns_slab_k(P_):
    for rank in range(P_):
        f = P.create_forest(FakeCtx(rank, P_), (0, 0, 0, 1, 1, P_), (1, 1, P_),
                            periodic=(True, True, True), cells_per_block=(8, 8, 4))
        blocks = f.local_blocks()
        assert len(blocks) == 1
        lo, hi = f.cell_box(blocks[0].id)
        assert lo[2] == 4 * rank and hi[2] == 4 * rank + 4
        box = RankBox(f)
        if P_ == 1:
            assert box.zface_lo == box.zface_hi == _lib.ZFACE_WRAP
        else:
            assert box.zface_lo == box.zface_hi == _lib.ZFACE_HALO
            assert box.lo_peer == (rank - 1) % P_ and box.hi_peer == (rank + 1) % P_


def test_rankbox_merges_blocks_and_faces():
    f = P.create_forest(FakeCtx(0, 2), (0, 0, 0, 1, 1, 4), (1, 1, 4), periodic=(True, False, False),
                        cells_per_block=(6, 5, 3))
    box = RankBox(f)
    assert (box.nx, box.ny, box.nz) == (6, 5, 6)
    assert box.zface_lo == _lib.ZFACE_GHOST and box.zface_hi == _lib.ZFACE_HALO
    assert box.hi_peer == 1 and box.wrap_x and not box.wrap_y
    # gather/scatter round trip through block views
    views = [np.random.default_rng(i).random((5, 7, 8, 2)) for i in range(2)]
    dense = box.gather(views, 2, np.float64)
    assert dense.shape == (2, 8, 7, 8)
    assert np.array_equal(dense[:, 1:4, 1:-1, 1:-1], np.moveaxis(views[0][1:-1, 1:-1, 1:-1], 3, 0))
    assert np.array_equal(dense[:, 0], np.moveaxis(views[0][0], 2, 0))      # outer ghost shell
    out = [np.zeros_like(v) for v in views]
    box.scatter_interior(dense[:, 1:-1, 1:-1, 1:-1], out)
    assert np.array_equal(out[1][1:-1, 1:-1, 1:-1], views[1][1:-1, 1:-1, 1:-1])


def test_rankbox_rejects_non_slab_partitions():
    f = P.create_forest(FakeCtx(0, 2), (0, 0, 0, 2, 1, 1), (2, 1, 1), cells_per_block=(4, 4, 4))
    with pytest.raises(P.ValidationError):
        RankBox(f)


def test_balance_matches_reference_rule():
    assert balance.owners_along_curve(8, 3) == [0, 0, 0, 1, 1, 2, 2, 2]
    assert balance.owners_along_curve(4, 4) == [0, 1, 2, 3]
    keys = [balance.morton_position((x, y, 0), 2) for y in range(2) for x in range(2)]
    assert keys == [0, 1, 2, 3]


def test_stencils_match_oracle_and_kernel_tables():
    for name in ("D2Q9", "D3Q19", "D3Q27"):
        a, b = P.get_stencil(name), oracle.STENCILS[name]
        assert a.c == b.c and a.opp == b.opp and a.w == b.wfrac
        assert a.weights.tobytes() == b.w.tobytes()


def test_kernel_params_host_constants():
    st = P.D3Q19
    kp = P.kernel_params(st, P.TRT.with_magic(1.7), P.Guo((1e-6, 0, 0)),
                         ubb_velocity=(0.05, 0.01, 0.0), reference_density=1.0)
    s = kp.struct
    we, wo = oracle.trt_magic(1.7)
    assert s.model == 1 and s.force_mode == 3          # Guo along x only
    assert P.kernel_params(st, P.SRT(1.2), P.Guo((0, 0, 0))).struct.force_mode == 0
    assert P.kernel_params(st, P.SRT(1.2), P.Guo((1e-5, 1e-6, 0))).struct.force_mode == 1
    assert s.omega_e == we and s.omega_o == wo
    assert s.he_half == (1.0 - 0.5 * we) * 0.5 and s.ho_half == (1.0 - 0.5 * wo) * 0.5
    assert s.shift_fx == 0.5 * 1e-6
    k = st.index((1, 1, 0))
    assert s.ubb[k] == 6.0 * st.weights[k] * 1.0 * (0.05 + 0.01)
    srt = P.kernel_params(st, P.SRT(1.8)).struct
    assert srt.rem == 1.0 - 1.8 and srt.hw == 1.0 - 0.5 * 1.8
    with pytest.raises(P.ValidationError):
        P.kernel_params(st, P.TRT(1.2, 1.1), P.SimpleShift((1e-5, 0, 0)))
    # per-cell rates: model LBM_SRT_FIELD, the sweep supplies the device rates
    assert P.kernel_params(st, P.SRT(omega_field="om")).struct.model == _lib.SRT_FIELD
    with pytest.raises(P.ValidationError):
        P.kernel_params(st, P.SRT(omega_field="om"), P.SimpleShift((1e-5, 0, 0)))


def test_mrt_tables_match_reference():
    units = np.load(Path(__file__).resolve().parent / "golden" / "units.npz")
    st = P.D3Q19
    rates = [1.0] * 19
    rates[9:16] = [1.4] * 7
    m = P.MRT(st, rates)
    assert np.array_equal(m.M, units["D3Q19_M"]) and m.Minv.tobytes() == units["D3Q19_Minv"].tobytes()
    kp = P.kernel_params(st, m, P.Guo((3e-4, -2e-4, 1e-4)))
    G = kp.tables[2 * 361 + 19:].reshape(19, 19)
    assert G.tobytes() == units["D3Q19_mrt_guo_matrix"].tobytes()
    with pytest.raises(P.ValidationError):
        P.MRT.uniform(P.D3Q27, 1.2)
    raw = P.MRT.raw_moments(P.D3Q27, 1.9)
    assert raw.S[4] == 1.9 and raw.S[0] == 1.0 and raw.M.shape == (27, 27)


def test_model_validation_mirrors_reference():
    for bad in (0.0, 2.0, -0.5, 2.5):
        with pytest.raises(P.ValidationError):
            P.SRT(bad)
        with pytest.raises(P.ValidationError):
            P.TRT(1.0, bad)
    with pytest.raises(P.ValidationError):
        P.SRT()
    with pytest.raises(P.ValidationError):
        P.MRT(P.D2Q9, [1.0] * 8)
    assert P.TRT.with_magic(1.4).magic == pytest.approx(3.0 / 16.0, rel=1e-12)
    assert P.mlups(64 * 64, 100, 2.0) == pytest.approx(0.2048)
    with pytest.raises(P.ValidationError):
        P.mlups(10, 10, 0.0)


def test_fields_and_flags_host_api():
    f = P.Field((4, 3, 2, 5), 1, "fzyx")
    assert f.raw.shape == (5, 4, 5, 6) and f.view.shape == (4, 5, 6, 5)
    f.set(0, 0, 0, 2, 7.0)
    assert f.get(0, 0, 0, 2) == 7.0 and f.interior[0, 0, 0, 2] == 7.0
    g = P.Field((4, 3, 2, 5), 1, "zyxf")
    with pytest.raises(P.ValidationError):
        f.swap_data(g)
    ff = P.FlagField((4, 4, 1), 1)
    m = ff.register("Fluid")
    assert m == 1 and ff.register("NoSlip") == 2
    with pytest.raises(P.ValidationError):
        ff.register("Fluid")
    ff.interior[...] = 1
    assert ff.count("Fluid") == 16


def test_host_exchange_and_gather_single_rank():
    ctx = P.Context(device="cpu")
    forest = P.create_forest(ctx, (0, 0, 0, 2, 1, 1), (2, 1, 1), periodic=(True, True, True),
                             cells_per_block=(4, 3, 2))
    forest.register_data("s", P.FieldDataHandler(nf=1, ghost_layers=1))
    N = forest.global_cells(0)
    for b in forest.local_blocks():
        lo, hi = forest.cell_box(b.id)
        z, y, x = np.meshgrid(np.arange(lo[2], hi[2]), np.arange(lo[1], hi[1]),
                              np.arange(lo[0], hi[0]), indexing="ij")
        b.data["s"].interior[..., 0] = x + 10 * y + 100 * z
    P.exchange_ghosts(forest, ["s"])
    for b in forest.local_blocks():
        lo, hi = forest.cell_box(b.id)
        v = b.data["s"].view[..., 0]
        for (zz, yy, xx) in [(0, 0, 0), (-1, -1, -1), (hi[2] - lo[2], 1, hi[0] - lo[0])]:
            gx, gy, gz = (lo[0] + xx) % N[0], (lo[1] + yy) % N[1], (lo[2] + zz) % N[2]
            assert v[zz + 1, yy + 1, xx + 1] == gx + 10 * gy + 100 * gz
    full = P.gather_slice(forest, "s", (0, 0, 0), N)
    assert full.shape == (2, 3, 8, 1) and full[1, 2, 7, 0] == 7 + 20 + 100


# ------------------------------------------------ run_arrays wavefront plan
@pytest.mark.parametrize("nz,steps,chunk", [
    (512, 20, None), (512, 100, None), (40, 7, 8), (40, 30, 6), (44, 9, 44), (44, 4, 1),
    (41, 6, 3), (10, 30, (4, (1, 2), 3)), (33, 5, (7, (1,), 1)), (5, 3, (2, (), 9)),
    (1, 4, None), (2, 1, None), (64, 1, (32, (4, 4, 8, 16), 4)),
])
def test_job_plan_respects_the_sweep_dependencies(nz, steps, chunk):
    """DeviceLattice.run_job's launch order (device.job_plan), simulated on
    the host: each plane of G_n is written once, only after G_{n-1} holds its
    neighbours (p - 1 .. p + 1; z ghosts are fixed) and before nothing still
    needs the G_{n-2} it overwrites; the moments read finished G_{K-1}
    planes; every plane is filled, swept K times and read out once."""
    from paper_1909_13772_b200.device import job_plan, job_schedule
    plan = job_plan(nz, steps, chunk)
    bounds, _ = job_schedule(nz, steps, chunk)
    assert [a[2:] for a in plan if a[0] == "fill"] == bounds
    # the moments of each round cover exactly the last sweep's planes of that
    # round (run_job fuses them into that launch, lbm_fused_step_moments)
    last = {}
    for act in plan:
        if act[0] == "step" and act[1] == steps:
            last["range"] = act[2:]
        elif act[0] == "moments":
            assert last.pop("range") == act[1:], act
    ver = np.full(nz, -1)                 # ver[p]: newest G_n written on plane p
    reads = {}                            # (n, p): readers of G_n on p still to come
    moments = np.zeros(nz, dtype=bool)
    for act in plan:
        if act[0] == "fill":
            _, _, z0, z1 = act
            assert (ver[z0:z1] == -1).all()
            ver[z0:z1] = 0
            continue
        if act[0] == "step":
            _, n, z0, z1 = act
        else:
            (_, z0, z1), n = act, steps
        for p in range(z0, z1):
            for q in (p - 1, p, p + 1):
                if 0 <= q < nz:
                    # G_{n-1} on q is there and not yet overwritten by G_{n+1}
                    assert ver[q] in (n - 1, n), (act, q, ver[q])
            if act[0] == "step":
                assert ver[p] == n - 1
                # overwriting G_{n-2} on p: step n-1 is past p + 1
                assert p + 1 >= nz or ver[p + 1] >= n - 1
                ver[p] = n
            else:
                assert not moments[p]
                moments[p] = True
    assert (ver == steps).all() and moments.all()
