"""Parity cases: one driver, two implementations.

`run_case(api, ctx, spec)` drives a case through the blocksim sweep API
(create_forest -> PdfField -> flags -> BoundaryHandling -> fill_equilibrium ->
stream_collide -> gather_slice / macroscopic_fields).  The same code runs the
reference (`reference_api()`, only in the container that holds
/root/reference: tests/golden/make_golden.py) and this framework
(`b200_api()`, GPU tests), which is itself a drop-in check.  The oracle runs
the same specs through `oracle_run` (no API, one global block).
"""
from __future__ import annotations

import sys
import types
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

from paper_1909_13772_b200 import workloads  # noqa: E402  (pure numpy generators)

# ------------------------------------------------------------------ specs
CASES = {
    # config 0 shape: D3Q19 SRT 1.8, periodic, random rho/u, 2 blocks in z
    "c0_srt_periodic": dict(stencil="D3Q19", dims=(10, 8, 6), root_dims=(1, 1, 2),
                            periodic=(True, True, True), geometry=None, model=("SRT", 1.8),
                            force=None, init=("random", 0), steps=10, snapshots=(1, 10),
                            layout="fzyx"),
    # config 1 shape: TRT magic 1.7 + Guo, porous spheres + z walls, periodic x,y
    "c1_trt_guo_porous": dict(stencil="D3Q19", dims=(12, 12, 12), root_dims=(1, 1, 2),
                              periodic=(True, True, False),
                              geometry=dict(kind="spheres", seed=1, rmin=2.0, rmax=3.0, frac=0.2,
                                            walls_z=True),
                              model=("TRT_magic", 1.7), force=("Guo", (1e-4, 2e-5, 0.0)),
                              init=("random", 3), steps=30, snapshots=(1, 30), macro=True,
                              layout="fzyx"),
    # config 2 shape, D3Q27 TRT: cavity with UBB lid, non-periodic, rest start
    "c2_d3q27_trt_cavity": dict(stencil="D3Q27", dims=(8, 8, 8), root_dims=(1, 1, 1),
                                periodic=(False, False, False), geometry=dict(kind="cavity"),
                                model=("TRT_magic", 1.6), force=None, init=("rest",),
                                ubb_velocity=(0.05, 0.01, 0.0), steps=20, snapshots=(20,),
                                layout="zyxf"),
    # ghost-plane walls (NoSlip-flagged ghosts), x periodic, coordinate init,
    # SRT + SimpleShift: exercises covered / uncovered ghost corners
    "d3q19_shift_ghostwalls": dict(stencil="D3Q19", dims=(8, 6, 10), root_dims=(1, 1, 2),
                                   periodic=(True, False, False),
                                   geometry=dict(kind="ghost_walls", faces=("y-", "y+", "z-", "z+")),
                                   model=("SRT", 1.3), force=("Shift", (1e-4, 0.0, -2e-5)),
                                   init=("smooth",), steps=20, snapshots=(20,), layout="fzyx"),
    # D3Q19 d'Humieres-type MRT (reference basis) + Guo with an obstacle
    "d3q19_mrt_guo": dict(stencil="D3Q19", dims=(8, 8, 8), root_dims=(1, 1, 1),
                          periodic=(True, True, True),
                          geometry=dict(kind="box_obstacle", lo=(3, 2, 3), hi=(5, 6, 5)),
                          model=("MRT_test", 1.4), force=("Guo", (1e-4, 0.0, -5e-5)),
                          init=("random", 5), steps=15, snapshots=(15,), layout="zyxf"),
    # config 2 model: D3Q27 raw-moment MRT (oracle extension), UBB lid cavity
    "c2_d3q27_rawmrt_cavity": dict(stencil="D3Q27", dims=(8, 8, 8), root_dims=(1, 1, 1),
                                   periodic=(False, False, False), geometry=dict(kind="cavity"),
                                   model=("MRT_raw", 1.9, 1.0), force=None, init=("rest",),
                                   ubb_velocity=(0.05, 0.0, 0.0), steps=15, snapshots=(15,),
                                   layout="fzyx"),
    # D2Q9 channel, TRT + Guo, walls at interior rows, 2 blocks in x
    "d2q9_trt_channel": dict(stencil="D2Q9", dims=(12, 10, 1), root_dims=(2, 1, 1),
                             periodic=(True, False, False), geometry=dict(kind="channel2d"),
                             model=("TRT_magic", 1.2), force=("Guo", (1e-5, 0.0, 0.0)),
                             init=("random", 7), steps=25, snapshots=(25,), layout="zyxf"),
    # per-cell SRT rates (f1 row, lbm/sweep.py:111-146): seeded rate field,
    # spheres + z walls, general Guo force, 2 blocks in z
    "d3q19_srt_omegafield": dict(stencil="D3Q19", dims=(10, 8, 12), root_dims=(1, 1, 2),
                                 periodic=(True, True, False),
                                 geometry=dict(kind="spheres", seed=21, rmin=1.5, rmax=2.5,
                                               frac=0.15, walls_z=True),
                                 model=("SRT_field", 21, 0.7, 1.9),
                                 force=("Guo", (1e-4, -3e-5, 2e-5)), init=("random", 21),
                                 steps=12, snapshots=(1, 12), layout="zyxf"),
    # flags edited between sweeps WITHOUT a new freeze(): the reference keeps
    # its frozen links and collides with the current flags (lbm/sweep.py:
    # 107-108, 124-136) - a Fluid cell turned NoSlip and back, an obstacle
    # core cell turned Fluid (cells away from block / periodic faces)
    "d3q19_flag_edits": dict(stencil="D3Q19", dims=(12, 10, 12), root_dims=(1, 1, 1),
                             periodic=(True, True, True),
                             geometry=dict(kind="box_obstacle", lo=(4, 3, 5), hi=(7, 6, 8)),
                             model=("TRT_magic", 1.6), force=("Guo", (1e-4, 2e-5, 0.0)),
                             init=("random", 31), steps=12, snapshots=(4, 5, 8, 12),
                             edits={4: ((2, 2, 2, "NoSlip"), (5, 4, 6, "Fluid")),
                                    8: ((9, 7, 3, "NoSlip"), (2, 2, 2, "Fluid"))},
                             layout="fzyx"),
    # Pressure anti-bounce-back (f1 row): D2Q9 box, pressure top row
    "d2q9_pressure_box": dict(stencil="D2Q9", dims=(8, 8, 1), root_dims=(1, 1, 1),
                              periodic=(False, False, False), geometry=dict(kind="pressure_box"),
                              model=("SRT", 1.2), force=None, init=("const", 1.05),
                              pressure_density=1.0, steps=30, snapshots=(30,), layout="zyxf"),
}

# larger cases compared through digests only (no array fixtures)
DIGEST_CASES = {
    "c0_srt_periodic_32": dict(stencil="D3Q19", dims=(32, 32, 32), root_dims=(1, 1, 1),
                               periodic=(True, True, True), geometry=None, model=("SRT", 1.8),
                               force=None, init=("random", 0), steps=20, snapshots=(20,),
                               layout="fzyx"),
    "c1_trt_guo_porous_24": dict(stencil="D3Q19", dims=(24, 24, 24), root_dims=(1, 1, 1),
                                 periodic=(True, True, False),
                                 geometry=dict(kind="spheres", seed=11, rmin=3.0, rmax=5.0,
                                               frac=0.25, walls_z=True),
                                 model=("TRT_magic", 1.7), force=("Guo", (1e-6, 0.0, 0.0)),
                                 init=("rest",), steps=50, snapshots=(50,), layout="fzyx"),
}


# ------------------------------------------------------------------ APIs
def reference_api():
    """blocksim from /root/reference (golden generation only)."""
    sys.path.insert(0, "/root/reference/pkg/src")
    import blocksim.lbm as L
    from blocksim.blockforest import create_forest
    from blocksim.field import FieldDataHandler, gather_slice
    from blocksim.lbm.collision import MRT as _MRT
    from blocksim.lbm import D3Q27

    class RawMRT(_MRT):
        """Oracle extension (probe D.10): D3Q27 raw-moment MRT
        through the unmodified stream_collide."""

        def __init__(self, stencil, rates, M):
            self.stencil = stencil
            self.M = np.asarray(M, dtype=np.float64)
            self.Minv = np.linalg.inv(self.M)
            self.S = np.array([float(r) for r in rates])

    def make_raw_mrt(stencil, shear, other):
        import oracle
        M = oracle.raw_moment_basis_d3q27(oracle.STENCILS["D3Q27"])
        rates = [other] * 27
        for k in range(4, 9):
            rates[k] = shear
        return RawMRT(D3Q27, rates, M)

    ns = types.SimpleNamespace(**{k: getattr(L, k) for k in L.__all__})
    ns.create_forest = create_forest
    ns.FieldDataHandler = FieldDataHandler
    ns.gather_slice = gather_slice
    ns.make_raw_mrt = make_raw_mrt
    from blocksim.field import write_vtk
    ns.write_vtk = write_vtk
    import blocksim.coupling as C
    import blocksim.rpd as R
    for name in ("map_bodies", "moving_boundary_sweep", "reduce_hydrodynamic_forces",
                 "reinitialize_uncovered", "covered_cell_counts", "CoupledSystem"):
        setattr(ns, name, getattr(C, name))
    for name in ("register_bodies", "add_sphere", "sync_bodies", "local_bodies"):
        setattr(ns, name, getattr(R, name))
    return ns


def b200_api():
    import paper_1909_13772_b200 as P
    ns = types.SimpleNamespace(**{k: getattr(P.lbm, k) for k in P.lbm.__all__})
    ns.create_forest = P.create_forest
    ns.FieldDataHandler = P.FieldDataHandler
    ns.gather_slice = P.gather_slice
    ns.make_raw_mrt = lambda st, shear, other: P.lbm.MRT.raw_moments(st, shear, other)
    ns.write_vtk = P.write_vtk
    for name in ("map_bodies", "moving_boundary_sweep", "reduce_hydrodynamic_forces",
                 "reinitialize_uncovered", "covered_cell_counts", "CoupledSystem",
                 "register_bodies", "add_sphere", "sync_bodies", "local_bodies"):
        setattr(ns, name, getattr(P, name))
    return ns


# --------------------------------------------------------------- geometry
def flag_codes(spec):
    """Global interior codes (nz, ny, nx): 0 Fluid, 1 NoSlip, 2 UBB,
    3 Pressure; plus ghost faces to flag NoSlip."""
    nx, ny, nz = spec["dims"]
    geo = spec.get("geometry")
    code = np.zeros((nz, ny, nx), dtype=np.int8)
    faces = ()
    if geo is None:
        return None, ()
    kind = geo["kind"]
    if kind == "spheres":
        solid = workloads.sphere_mask((nx, ny, nz), geo["seed"], geo["rmin"], geo["rmax"],
                                      geo["frac"], tuple(spec["periodic"]))
        if geo.get("walls_z"):
            solid[0] = solid[nz - 1] = True
        code[solid] = 1
    elif kind == "cavity":
        code = workloads.cavity_flags((nx, ny, nz))
    elif kind == "ghost_walls":
        faces = tuple(geo["faces"])
    elif kind == "box_obstacle":
        (x0, y0, z0), (x1, y1, z1) = geo["lo"], geo["hi"]
        code[z0:z1, y0:y1, x0:x1] = 1
    elif kind == "channel2d":
        code[:, 0, :] = 1
        code[:, ny - 1, :] = 1
    elif kind == "pressure_box":
        code[...] = 1
        code[:, ny - 1, :] = 3
        code[:, 1:-1, 1:-1] = 0
    else:
        raise ValueError(kind)
    return code, faces


def _names(api):
    return (api.FLUID, api.NO_SLIP, api.UBB, api.PRESSURE)


def model_of(api, spec, st):
    m = spec["model"]
    kind = m[0]
    if kind == "SRT":
        return api.SRT(m[1])
    if kind == "TRT":
        return api.TRT(m[1], m[2])
    if kind == "TRT_magic":
        return api.TRT.with_magic(m[1])
    if kind == "MRT_test":
        rates = [1.0] * st.q
        rates[9:16] = [m[1]] * 7      # pkg/tests/test_lbm.py:207-210
        return api.MRT(st, rates)
    if kind == "MRT_raw":
        return api.make_raw_mrt(st, m[1], m[2])
    if kind == "SRT_field":
        return api.SRT(omega_field="omega")
    raise ValueError(kind)


def rate_field(spec):
    """Global interior per-cell SRT rates (nz, ny, nx) of an SRT_field case."""
    _, seed, lo, hi = spec["model"]
    nx, ny, nz = spec["dims"]
    return np.random.default_rng(seed).uniform(lo, hi, size=(nz, ny, nx))


def force_of(api, spec):
    f = spec.get("force")
    if f is None:
        return None
    return api.Guo(f[1]) if f[0] == "Guo" else api.SimpleShift(f[1])


def smooth_rho(x, y, z):
    return 1.0 + 0.02 * np.cos(0.7 * x) * np.sin(0.45 * y + 0.3) + 0.01 * np.cos(0.31 * z)


def smooth_u(x, y, z):
    return (0.03 * np.sin(0.5 * y + 0.2 * z), 0.02 * np.cos(0.4 * x), 0.015 * np.sin(0.3 * x + 0.6 * y))


# ------------------------------------------------------------ the driver
def run_case(api, ctx, spec, *, pdf_kwargs=None):
    """Returns {"pdf": {step: (nz,ny,nx,q)}, "macro": (rho, u) or None,
    "links": {name: count}} on rank 0 (None elsewhere)."""
    forest, pdf, handling, model, force, st = setup_case(api, ctx, spec, pdf_kwargs=pdf_kwargs)
    nx, ny, nz = spec["dims"]
    d = 2 if spec["stencil"] == "D2Q9" else 3
    out = {"pdf": {}, "macro": None, "links": None}
    snaps = set(spec["snapshots"])
    edits = spec.get("edits", {})
    for s in range(1, spec["steps"] + 1):
        api.stream_collide(pdf, model, force=force, handling=handling)
        if s in snaps:
            g = api.gather_slice(forest, "pdf", (0, 0, 0), forest.global_cells(0))
            if g is not None:
                out["pdf"][s] = g
        for (x, y, z, name) in edits.get(s, ()):
            _edit_flag(api, forest, x, y, z, name)
    if spec.get("macro"):
        forest.register_data("rho", api.FieldDataHandler(nf=1, ghost_layers=0))
        forest.register_data("vel", api.FieldDataHandler(nf=d, ghost_layers=0))
        api.macroscopic_fields(pdf, "rho", "vel", force=force, handling=handling)
        r = api.gather_slice(forest, "rho", (0, 0, 0), forest.global_cells(0))
        v = api.gather_slice(forest, "vel", (0, 0, 0), forest.global_cells(0))
        if r is not None:
            out["macro"] = (r[..., 0], v)
    if handling is not None:
        counts = {}
        for name in ("NoSlip", "UBB", "Pressure"):
            counts[name] = sum(len(zs) for b in forest.local_blocks()
                               for (i, zs, ys, xs) in handling.links[b.id][name])
        tot = ctx.all_gather(counts)
        out["links"] = {n: sum(tot[r][n] for r in tot) for n in counts}
    return out if ctx.rank == 0 else None


def _edit_flag(api, forest, x, y, z, name):
    """Set global interior cell (x, y, z) to flag `name` on the owning
    block, without a new BoundaryHandling.freeze()."""
    for block in forest.local_blocks():
        lo, hi = forest.cell_box(block.id)
        if lo[0] <= x < hi[0] and lo[1] <= y < hi[1] and lo[2] <= z < hi[2]:
            ff = block.data["flags"]
            ff.interior[z - lo[2], y - lo[1], x - lo[0]] = ff.registry[name]


def setup_case(api, ctx, spec, *, pdf_kwargs=None):
    """Forest, PDF field, flags/handling, rate field and initial state of a
    case; returns (forest, pdf, handling, model, force, stencil)."""
    st = getattr(api, spec["stencil"])
    nx, ny, nz = spec["dims"]
    R = spec["root_dims"]
    d = 2 if spec["stencil"] == "D2Q9" else 3
    cells = (nx // R[0], ny // R[1], nz // R[2])
    forest = api.create_forest(ctx, (0, 0, 0, R[0], R[1], R[2]), R, d=d,
                               periodic=tuple(spec["periodic"]), cells_per_block=cells)
    pdf = api.PdfField(forest, st, layout=spec.get("layout", "zyxf"), **(pdf_kwargs or {}))
    code, faces = flag_codes(spec)
    handling = None
    if code is not None or faces:
        handler = api.ensure_flags(forest)
        reg = handler.registry
        bits = [reg[n] for n in _names(api)]
        gl = np.zeros((nz, ny, nx), dtype=np.uint32)
        gl[...] = bits[0]
        if code is not None:
            for k in (1, 2, 3):
                gl[code == k] = bits[k]
        N = (nx, ny, nz)
        for block in forest.local_blocks():
            lo, hi = forest.cell_box(block.id)
            ff = block.data["flags"]
            ff.interior[...] = gl[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]]
            v = ff.view
            for face in faces:
                a = "xyz".index(face[0])
                idx = [slice(None)] * 3
                if face[1] == "-" and lo[a] == 0:
                    idx[2 - a] = 0
                elif face[1] == "+" and hi[a] == N[a]:
                    idx[2 - a] = -1
                else:
                    continue
                v[tuple(idx)] = reg[api.NO_SLIP]
        handling = api.BoundaryHandling(forest, st,
                                        ubb_velocity=spec.get("ubb_velocity", (0.0, 0.0, 0.0)),
                                        pressure_density=spec.get("pressure_density", 1.0))
    init = spec["init"]
    if init[0] == "rest":
        api.fill_equilibrium(pdf)
    elif init[0] == "const":
        api.fill_equilibrium(pdf, init[1], (0.0, 0.0, 0.0))
    elif init[0] == "smooth":
        api.fill_equilibrium(pdf, smooth_rho, smooth_u)
    elif init[0] == "random":
        api.fill_equilibrium(pdf)
        rho, u = workloads.random_rho_u((nx, ny, nz), init[1])
        for block in forest.local_blocks():
            lo, hi = forest.cell_box(block.id)
            sl = (slice(lo[2], hi[2]), slice(lo[1], hi[1]), slice(lo[0], hi[0]))
            pdf.src(block).interior[...] = api.equilibrium(rho[sl], u[sl], st)
    if spec["model"][0] == "SRT_field":
        forest.register_data("omega", api.FieldDataHandler(nf=1, ghost_layers=1))
        om = rate_field(spec)
        for block in forest.local_blocks():
            lo, hi = forest.cell_box(block.id)
            block.data["omega"].interior[..., 0] = om[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]]
    model = model_of(api, spec, st)
    force = force_of(api, spec)
    return forest, pdf, handling, model, force, st


# snapshot / restart / VTK case: k steps, macroscopic
# fields, forest image + VTK files, then m more steps
SNAPSHOT_CASE = dict(stencil="D3Q19", dims=(8, 6, 8), root_dims=(1, 1, 2),
                     periodic=(True, True, False),
                     geometry=dict(kind="spheres", seed=5, rmin=1.5, rmax=2.5, frac=0.15,
                                   walls_z=True),
                     model=("TRT_magic", 1.6), force=("Guo", (1e-4, 0.0, 3e-5)),
                     init=("random", 11), steps=5, snapshots=(), layout="fzyx")
SNAPSHOT_MORE = 4


def run_snapshot_case(api, ctx, spec, vtk_dir, *, image=None, pdf_kwargs=None):
    """k = spec["steps"] sweeps, rho/vel, forest image + VTK, then
    SNAPSHOT_MORE sweeps.  With `image`, the forest is first restored from it
    (restart: the k sweeps are skipped).  Returns {"image", "vtk" {name:
    bytes}, "pdf_more"} on rank 0."""
    import os
    forest, pdf, handling, model, force, st = setup_case(api, ctx, spec, pdf_kwargs=pdf_kwargs)
    forest.register_data("rho", api.FieldDataHandler(nf=1, ghost_layers=1))
    forest.register_data("vel", api.FieldDataHandler(nf=3, ghost_layers=1))
    if image is None:
        for _ in range(spec["steps"]):
            api.stream_collide(pdf, model, force=force, handling=handling)
        api.macroscopic_fields(pdf, "rho", "vel", force=force, handling=handling)
    else:
        forest.load_snapshot_blocks([image])
        forest.rebuild_neighborhoods()
    img = forest.snapshot()
    names = api.write_vtk(forest, vtk_dir, "out", spec["steps"], [("rho", "rho"), ("u", "vel")])
    vtk = {}
    for name in sorted(os.listdir(vtk_dir)):
        with open(os.path.join(vtk_dir, name), "rb") as fh:
            vtk[name] = fh.read()
    del names
    for _ in range(SNAPSHOT_MORE):
        api.stream_collide(pdf, model, force=force, handling=handling)
    g = api.gather_slice(forest, "pdf", (0, 0, 0), forest.global_cells(0))
    return {"image": img, "vtk": vtk, "pdf_more": g} if ctx.rank == 0 else None


# ------------------------------------------------------------- the oracle
def oracle_inputs(spec, oracle):
    """Global ghost-inclusive inputs for oracle.Domain: (pdf (q,Z,Y,X),
    flags (Z,Y,X) or None, bits)."""
    st = oracle.STENCILS[spec["stencil"]]
    nx, ny, nz = spec["dims"]
    X, Y, Z = nx + 2, ny + 2, nz + 2
    code, faces = flag_codes(spec)
    bits = {"Fluid": 1, "NoSlip": 2, "UBB": 4, "Pressure": 8, "Solid": 16}
    flags = None
    if code is not None or faces:
        flags = np.zeros((Z, Y, X), dtype=np.uint32)
        inner = np.full((nz, ny, nx), bits["Fluid"], dtype=np.uint32)
        if code is not None:
            inner[code == 1] = bits["NoSlip"]
            inner[code == 2] = bits["UBB"]
            inner[code == 3] = bits["Pressure"]
        flags[1:-1, 1:-1, 1:-1] = inner
        for face in faces:
            a = "xyz".index(face[0])
            idx = [slice(None)] * 3
            idx[2 - a] = 0 if face[1] == "-" else -1
            flags[tuple(idx)] = bits["NoSlip"]
    # initial R-form including ghosts, as fill_equilibrium + overwrite
    init = spec["init"]
    R = spec["root_dims"]
    xs = _centres(nx, R[0]); ys = _centres(ny, R[1]); zs = _centres(nz, R[2])
    z, y, x = np.meshgrid(zs, ys, xs, indexing="ij")
    if init[0] == "smooth":
        rho = smooth_rho(x, y, z)
        u = np.stack(np.broadcast_arrays(*smooth_u(x, y, z)), axis=-1)
    elif init[0] == "const":
        rho = np.full(x.shape, float(init[1]))
        u = np.zeros(x.shape + (3,))
    else:
        rho = np.ones(x.shape)
        u = np.zeros(x.shape + (3,))
    feq = oracle.equilibrium(rho, u, st)
    if init[0] == "random":
        r, uu = workloads.random_rho_u((nx, ny, nz), init[1])
        feq[1:-1, 1:-1, 1:-1] = oracle.equilibrium(r, uu, st)
    pdf = np.ascontiguousarray(np.moveaxis(feq, 3, 0))
    return pdf, flags, bits


def _centres(n, roots):
    """Global ghost-inclusive cell-centre coordinates of the reference's
    unit-block domain (0..roots), block-local expressions as in
    fill_equilibrium (sweep.py:58-62) + forest.cell_centers."""
    per = n // roots
    sx = (roots - 0.0) / roots
    dx = (roots - 0.0) / (roots * per)
    out = np.empty(n + 2)
    for i in range(-1, n + 1):
        b = min(max(i, 0), n - 1) // per          # block owning the clamped index
        c0 = (0.0 + b * sx) + 0.5 * dx
        out[i + 1] = c0 + dx * np.float64(i - b * per)
    return out


def oracle_model(spec, oracle):
    st = oracle.STENCILS[spec["stencil"]]
    m = spec["model"]
    f = spec.get("force")
    force = None if f is None else f[1]
    fk = "guo" if f is None or f[0] == "Guo" else "shift"
    if m[0] == "SRT":
        return oracle.Model("SRT", omega=m[1], force=force, force_kind=fk)
    if m[0] == "SRT_field":
        nx, ny, nz = spec["dims"]
        of = np.zeros((nz + 2, ny + 2, nx + 2))
        of[1:-1, 1:-1, 1:-1] = rate_field(spec)
        return oracle.Model("SRT", omega=0.0, omega_field=of, force=force, force_kind=fk)
    if m[0] in ("TRT", "TRT_magic"):
        we, wo = (m[1], m[2]) if m[0] == "TRT" else oracle.trt_magic(m[1])
        return oracle.Model("TRT", omega_e=we, omega_o=wo, force=force, force_kind=fk)
    if m[0] == "MRT_test":
        M = oracle.moment_basis(st)
        rates = [1.0] * st.q
        rates[9:16] = [m[1]] * 7
        return oracle.Model("MRT", M=M.astype(np.float64), Minv=oracle.basis_inverse(M),
                            S=np.array(rates), force=force, force_kind=fk)
    if m[0] == "MRT_raw":
        M = oracle.raw_moment_basis_d3q27(st)
        rates = [m[2]] * 27
        for k in range(4, 9):
            rates[k] = m[1]
        return oracle.Model("MRT", M=M, Minv=np.linalg.inv(M), S=np.array(rates), force=force,
                            force_kind=fk)
    raise ValueError(m[0])


def oracle_run(spec, oracle):
    """{"pdf": {step: (nz,ny,nx,q)}} from the C oracle on one global block."""
    st = oracle.STENCILS[spec["stencil"]]
    pdf, flags, bits = oracle_inputs(spec, oracle)
    dom = oracle.Domain(st, spec["dims"], spec["periodic"], oracle_model(spec, oracle), flags,
                        bits, ubb_velocity=spec.get("ubb_velocity", (0.0, 0.0, 0.0)),
                        pressure_density=spec.get("pressure_density", 1.0))
    dom.set_full(pdf)
    out = {}
    done = 0
    edits = spec.get("edits", {})
    for s in sorted(set(spec["snapshots"]) | set(edits)):
        dom.run(s - done)
        done = s
        if s in spec["snapshots"]:
            out[s] = dom.rform()
        for (x, y, z, name) in edits.get(s, ()):
            dom.edit_flag(x, y, z, name)
    return {"pdf": out, "domain": dom}


# -------------------------------------------------- moving bodies (row f2)
COUPLING_CASES = {
    # a translating + rotating sphere and one straddling the periodic corner,
    # TRT + Guo, bodies displaced every step (coverage changes: re-collision
    # of the stored state, uncovered-cell reinitialisation), 2x2x2 blocks
    "moving_spheres": dict(stencil="D3Q19", dims=(16, 16, 16), root_dims=(2, 2, 2),
                           model=("TRT_magic", 1.6), force=("Guo", (2e-5, 0.0, -1e-5)),
                           bodies=[((8.2, 8.1, 7.9), 3.0, 100.0, (0.08, -0.05, 0.03),
                                    (0.0, 0.003, 0.001)),
                                   ((1.3, 14.6, 15.4), 2.5, 50.0, (-0.06, 0.07, 0.09),
                                    (0.002, 0.0, -0.004))],
                           steps=8, move=True, layout="fzyx"),
    # stationary body, SRT: equals a NoSlip obstacle (test_coupling.py:236-265)
    "static_sphere_srt": dict(stencil="D3Q19", dims=(16, 16, 16), root_dims=(1, 1, 1),
                              model=("SRT", 1.6), force=None,
                              bodies=[((8.2, 8.1, 7.9), 3.0, 1.0, (0.0, 0.0, 0.0),
                                       (0.0, 0.0, 0.0))],
                              steps=12, move=False, layout="zyxf"),
    # the AoS layout ("zyxf": the reference sums densities with numpy's
    # pairwise kernel there) with D3Q27 and moving bodies, 2 blocks in z:
    # released cells are re-initialised on the device in that order
    "moving_d3q27_aos": dict(stencil="D3Q27", dims=(14, 12, 16), root_dims=(1, 1, 2),
                             model=("SRT", 1.5), force=None,
                             bodies=[((6.6, 5.9, 7.3), 2.8, 60.0, (0.11, 0.07, -0.09),
                                      (0.004, -0.002, 0.003))],
                             steps=7, move=True, layout="zyxf"),
}


def coupling_velocity(x, y, z):
    return (0.02 * np.sin(2 * np.pi * z / 16.0), 0.01 * np.cos(2 * np.pi * x / 16.0), 0.0 * x)


def run_coupling_case(api, ctx, spec, *, pdf_kwargs=None, all_ranks=False):
    """The coupled step spelled out with the public functions (system.py:
    164-196 with the DEM substeps replaced by a prescribed displacement
    x += v per step): map -> moving_boundary_sweep -> reduce -> move ->
    sync_bodies -> remap -> reinitialize_uncovered.  Returns (rank 0) the
    final PDFs, per-step record forces/torques, final body forces, uncovered
    and link counts (this rank's; all_ranks=True returns them on every rank)."""
    st = getattr(api, spec["stencil"])
    nx, ny, nz = spec["dims"]
    R = spec["root_dims"]
    forest = api.create_forest(ctx, (0, 0, 0, nx, ny, nz), R, periodic=(True, True, True),
                               cells_per_block=(nx // R[0], ny // R[1], nz // R[2]))
    pdf = api.PdfField(forest, st, layout=spec["layout"], **(pdf_kwargs or {}))
    api.register_bodies(forest, contact_threshold=1.0)
    for pos, r, m, v, w in spec["bodies"]:
        api.add_sphere(forest, pos, r, mass=m, velocity=v, angular_velocity=w)
    api.sync_bodies(forest)
    api.fill_equilibrium(pdf, 1.0, coupling_velocity)
    model = model_of(api, spec, st)
    force = force_of(api, spec)
    mapping = api.map_bodies(forest, st)
    out = {"records": [], "uncovered": [], "links": []}
    for _ in range(spec["steps"]):
        out["links"].append(sum(mapping.link_count(b.id) for b in forest.local_blocks()))
        records = api.moving_boundary_sweep(pdf, model, mapping, force=force)
        out["records"].append([(r[3], tuple(float(v) for v in r[5]), tuple(float(v) for v in r[6]))
                               for r in records])
        api.reduce_hydrodynamic_forces(forest, records)
        if spec["move"]:
            for b in api.local_bodies(forest):
                b.position = b.position + b.linear_velocity
        api.sync_bodies(forest)
        new = api.map_bodies(forest, st)
        out["uncovered"].append(api.reinitialize_uncovered(pdf, mapping, new))
        mapping = new
    out["pdf"] = api.gather_slice(forest, "pdf", (0, 0, 0), forest.global_cells(0))
    out["bodies"] = [(b.uid, tuple(b.position), tuple(b.hydrodynamic_force),
                      tuple(b.hydrodynamic_torque)) for b in api.local_bodies(forest)]
    out["covered"] = api.covered_cell_counts(forest, mapping)
    return out if (ctx.rank == 0 or all_ranks) else None
