"""Generate golden vectors by running the REFERENCE implementation.

Run in the container that holds /root/reference (read-only):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports blocksim from /root/reference/pkg/src, drives every case of
tests/cases.py through the reference's own sweep API under SimRuntime
(1 rank, plus 2 ranks where the partition allows, asserting the reference's
bitwise rank invariance), and writes:

  golden/<case>.npz      snapshots of the gathered R-form PDFs (z,y,x,q),
                         macroscopic fields, link counts, sha256 digests
  golden/digests.json    sha256 of larger cases (no arrays committed)
  golden/units.npz       reference unit outputs: collide_pdfs for every model
                         variant, equilibrium/macroscopic, TRT magic rates,
                         moment bases, guo_matrix

Nothing here runs on the GPU box (/root/reference does not exist there);
the committed files are what the tests read.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
from pathlib import Path

import numpy as np

os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
os.environ.setdefault("BLOCKSIM_KERNELS", "python")
HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
sys.path.insert(0, "/root/reference/pkg/src")

import cases  # noqa: E402
from blocksim.runtime import SimRuntime  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def run_ref(spec, n_ranks=1):
    api = cases.reference_api()
    return SimRuntime(n_ranks, seed=0).run(lambda ctx: cases.run_case(api, ctx, spec))[0]


def main(only=None):
    """only: case names to (re)generate; the other entries of digests.json
    and the unit vectors are kept as committed."""
    meta = json.loads((HERE / "digests.json").read_text()) if only else {}
    for name, spec in cases.CASES.items():
        if only and name not in only:
            continue
        res = run_ref(spec)
        if spec["root_dims"][2] >= 2 or spec["root_dims"][0] >= 2:
            res2 = run_ref(spec, 2)
            for s in res["pdf"]:
                assert res["pdf"][s].tobytes() == res2["pdf"][s].tobytes(), f"{name}: rank variance"
        arrays = {}
        digests = {}
        for s, arr in res["pdf"].items():
            arrays[f"pdf_{s}"] = arr
            digests[f"pdf_{s}"] = sha(arr)
        if res["macro"] is not None:
            arrays["rho"], arrays["vel"] = res["macro"]
            digests["rho"], digests["vel"] = sha(res["macro"][0]), sha(res["macro"][1])
        links = res["links"] or {}
        np.savez(HERE / f"{name}.npz", **arrays)
        meta[name] = {"digests": digests, "links": links, "spec": repr(spec)}
        print(name, {k: v[:12] for k, v in digests.items()}, links, flush=True)
    (HERE / "digests.json").write_text(json.dumps(meta, indent=1, sort_keys=True))
    if only:
        return
    dig = {}
    for name, spec in cases.DIGEST_CASES.items():
        res = run_ref(spec)
        dig[name] = {f"pdf_{s}": sha(a) for s, a in res["pdf"].items()}
        dig[name]["links"] = res["links"]
        print(name, dig[name], flush=True)
    meta["digest_cases"] = dig
    (HERE / "digests.json").write_text(json.dumps(meta, indent=1, sort_keys=True))
    make_units()


def make_snapshot():
    """f3 formats: the reference's forest image + VTK files after k sweeps of
    cases.SNAPSHOT_CASE, and the PDFs after SNAPSHOT_MORE more sweeps."""
    import tempfile
    spec = cases.SNAPSHOT_CASE
    with tempfile.TemporaryDirectory() as tmp:
        api = cases.reference_api()
        res = SimRuntime(1, seed=0).run(lambda ctx: cases.run_snapshot_case(api, ctx, spec, tmp))[0]
    np.savez(HERE / "snapshot_case.npz", image=np.frombuffer(res["image"], dtype=np.uint8),
             pdf_more=res["pdf_more"])
    meta = json.loads((HERE / "digests.json").read_text())
    meta["snapshot_case"] = {"vtk": {n: sha(np.frombuffer(b, dtype=np.uint8))
                                     for n, b in res["vtk"].items()},
                             "image": sha(np.frombuffer(res["image"], dtype=np.uint8))}
    (HERE / "digests.json").write_text(json.dumps(meta, indent=1, sort_keys=True))
    print("snapshot:", len(res["image"]), "bytes,", len(res["vtk"]), "vtk files")


def make_coupling():
    """Row f2: the reference's coupled steps (cases.COUPLING_CASES) - final
    PDFs as arrays, forces/counts as JSON."""
    meta = json.loads((HERE / "digests.json").read_text())
    meta["coupling"] = {}
    for name, spec in cases.COUPLING_CASES.items():
        api = cases.reference_api()
        res = SimRuntime(1, seed=0).run(lambda ctx: cases.run_coupling_case(api, ctx, spec))[0]
        np.savez(HERE / f"coupling_{name}.npz", pdf=res["pdf"])
        meta["coupling"][name] = {"records": res["records"], "uncovered": res["uncovered"],
                                  "links": res["links"], "bodies": res["bodies"],
                                  "covered": {str(k): v for k, v in res["covered"].items()},
                                  "pdf": sha(res["pdf"])}
        print("coupling", name, res["links"], res["uncovered"], flush=True)
    (HERE / "digests.json").write_text(json.dumps(meta, indent=1, sort_keys=True))


SLOT_DIMS = (7, 5, 6)   # x, y, z of the slot box, ghost ring included


def slot_cases():
    """(name, stencil name, model kind, force, omega_window?, fluid bits,
    view layout) of the kernel-slot goldens (make_slot)."""
    out = []
    forces = {"none": None, "guo": ("Guo", (3e-4, -2e-4, 1e-4)), "guox": ("Guo", (1e-4, 0.0, 0.0))}
    for sname, models in (("D2Q9", ("srt", "trt", "mrt")),
                          ("D3Q19", ("srt", "trt", "trtmagic", "mrt")),
                          ("D3Q27", ("srt", "trt", "rawmrt"))):
        for m in models:
            for fname in forces:
                lay = "soa" if (len(out) % 2) else "aos"
                out.append((f"{sname}_{m}_{fname}", sname, m, fname, False, 1, lay))
        out.append((f"{sname}_srt_shift", sname, "srt", "shift", False, 1, "aos"))
        out.append((f"{sname}_srt_window_guo", sname, "srt", "guo", True, 1, "soa"))
    out.append(("D3Q19_trt_multibit", "D3Q19", "trt", "none", False, 1 | 8, "soa"))
    return out


def make_slot():
    """Kernel slot: the reference's own impl.collide and
    impl.stream_pull (_kernels/_core_py.py:70-218) on a flagged box with its
    ghost ring, for every model / force / view layout the slot accepts."""
    import blocksim.lbm as L
    from blocksim._kernels import _core_py as impl
    from blocksim.lbm.collision import _kernel_params
    import oracle
    rng = np.random.default_rng(77)
    X, Y, Z = SLOT_DIMS
    out = {}
    stencils = {"D2Q9": L.D2Q9, "D3Q19": L.D3Q19, "D3Q27": L.D3Q27}
    for name, sname, m, fname, window, bits, lay in slot_cases():
        st = stencils[sname]
        q = st.q
        rho = rng.uniform(0.8, 1.2, (Z, Y, X))
        u = rng.uniform(-0.08, 0.08, (Z, Y, X, 3))
        if st.d == 2:
            u[..., 2] = 0.0
        f = L.equilibrium(rho, u, st) * (1.0 + 0.03 * rng.uniform(-1, 1, (Z, Y, X, q)))
        flags = rng.choice(np.array([0, 1, 2, 4, 8, 9, 16], dtype=np.uint32), size=(Z, Y, X))
        if m == "srt":
            model = L.SRT(1.3)
        elif m == "trt":
            model = L.TRT(1.3, 0.9)
        elif m == "trtmagic":
            model = L.TRT.with_magic(1.7)
        elif m == "mrt":
            rates = [1.0] * q
            rates[q // 2:] = [1.4] * (q - q // 2)
            model = L.MRT(st, rates)
        else:   # D3Q27 raw-moment MRT through the generic branch
            model = None
        force = None
        if fname in ("guo", "guox"):
            force = L.Guo({"guo": (3e-4, -2e-4, 1e-4), "guox": (1e-4, 0.0, 0.0)}[fname])
        elif fname == "shift":
            force = L.SimpleShift((3e-4, -2e-4, 1e-4))
        if model is None:
            params = _kernel_params(st, L.SRT(1.0), force)
            del params["omega"]
            M = oracle.raw_moment_basis_d3q27(oracle.STENCILS["D3Q27"])
            S = np.full(q, 1.0)
            S[4:9] = 1.9
            params["M"], params["Minv"], params["S"] = M, np.linalg.inv(M), S
            if force is not None:
                params["guo_matrix"] = params["Minv"] @ (np.eye(q) - 0.5 * np.diag(S)) @ M
            mode = 2
        else:
            params = _kernel_params(st, model, force)
            mode = model.mode
        if window:
            params["omega_window"] = rng.uniform(0.7, 1.9, (Z, Y, X))
        if lay == "soa":
            raw = np.ascontiguousarray(np.moveaxis(f, 3, 0))
            view = np.moveaxis(raw, 0, 3)
        else:
            view = f.copy()
        impl.collide(view, flags, np.uint32(bits), mode, params)
        out[f"{name}__in"] = f
        out[f"{name}__flags"] = flags
        out[f"{name}__out"] = np.ascontiguousarray(view)
        if window:
            out[f"{name}__window"] = params["omega_window"]
        # the params dict itself, as plain arrays (keys with a scalar / array value)
        for k, v in params.items():
            if v is None:
                continue
            out[f"{name}__p_{k}"] = np.asarray(v)
        out[f"{name}__mode"] = np.asarray(mode)
        out[f"{name}__bits"] = np.asarray(bits, dtype=np.uint32)
        out[f"{name}__layout"] = np.asarray(lay)
    for sname, st in stencils.items():
        q = st.q
        src = rng.standard_normal((Z, Y, X, q))
        dst = rng.standard_normal((Z, Y, X, q))
        out[f"pull_{sname}__src"], out[f"pull_{sname}__dst"] = src, dst.copy()
        impl.stream_pull(src, dst, st.cx, st.cy, st.cz, 1)
        out[f"pull_{sname}__out"] = dst
    np.savez(HERE / "slot.npz", **out)
    print("slot:", len(slot_cases()), "collide cases")


OWNERSHIP_FORESTS = [  # (root_dims, d, periodic, n_ranks)
    ((1, 1, 8), 3, (True, True, False), 8), ((1, 1, 8), 3, (True, True, True), 3),
    ((2, 2, 2), 3, (True, False, True), 3), ((3, 2, 5), 3, (False, True, False), 7),
    ((4, 3, 1), 2, (True, False, False), 5), ((5, 1, 1), 2, (True, True, False), 2),
    ((1, 1, 1), 3, (True, True, True), 1), ((2, 3, 4), 3, (True, True, True), 24),
]


def make_ownership():
    """Rank ownership + neighbour records: the reference's own balance.py
    routines and create_forest on a set of root grids and rank counts."""
    from blocksim import balance as B
    from blocksim.blockforest import create_forest
    from blocksim.runtime import SimRuntime
    parts = {}
    for n in range(0, 41):
        for p in range(1, 13):
            parts[f"{n},{p}"] = B.partition_curve([1.0] * n, p)
    forests = []
    for dims, d, per, ranks in OWNERSHIP_FORESTS:
        def prog(ctx):
            f = create_forest(ctx, (0, 0, 0) + tuple(float(v) for v in dims), dims, d=d,
                              periodic=per, cells_per_block=(2, 2, 2 if d == 3 else 1))
            return [[b.id.root, [[list(r.direction), r.block_id.root, r.rank, list(r.shift)]
                                 for r in b.neighbors]] for b in f.local_blocks()]
        res = SimRuntime(ranks, seed=0).run(prog)
        forests.append({"dims": dims, "d": d, "periodic": per, "ranks": ranks,
                        "blocks": {str(r): res[r] for r in range(ranks)}})
    (HERE / "ownership.json").write_text(json.dumps({"partition": parts, "forests": forests}))
    print("ownership:", len(parts), "partitions,", len(forests), "forests")


APPLY_CASES = {  # name: (stencil, dims x, y, z)
    "D3Q19": ("D3Q19", (7, 6, 5)),
    "D3Q27": ("D3Q27", (6, 5, 6)),
    "D2Q9": ("D2Q9", (9, 7, 1)),
}


def apply_flags(reg, dims, d):
    """Interior flag codes of the apply goldens: a closed box - NoSlip walls,
    a UBB lid (top y plane in 2D, top z plane in 3D), a Pressure outlet on
    the high-x face - around Fluid with one NoSlip obstacle cell."""
    nx, ny, nz = dims
    f = np.full((nz, ny, nx), reg["NoSlip"], dtype=np.uint32)
    if d == 3:
        f[1:-1, 1:-1, 1:-1] = reg["Fluid"]
        f[-1, 1:-1, 1:-1] = reg["UBB"]
        f[1:-1, 1:-1, -1] = reg["Pressure"]
    else:
        f[:, 1:-1, 1:-1] = reg["Fluid"]
        f[:, -1, 1:-1] = reg["UBB"]
        f[:, 1:-1, -1] = reg["Pressure"]
    f[nz // 2, ny // 2, nx // 2] = reg["NoSlip"]
    return f


def make_apply():
    """BoundaryHandling.apply of the reference (lbm/boundary.py:154-195) on
    random post-collision src / dst views of one block, every link type."""
    import blocksim.lbm as L
    from blocksim.blockforest import create_forest
    rng = np.random.default_rng(55)
    out = {}
    for name, (sname, dims) in APPLY_CASES.items():
        st = getattr(L, sname)
        d = st.d

        def prog(ctx):
            forest = create_forest(ctx, (0, 0, 0, 1, 1, 1), (1, 1, 1), d=d,
                                   periodic=(False, False, False), cells_per_block=dims)
            handler = L.ensure_flags(forest)
            blk = forest.local_blocks()[0]
            blk.data["flags"].interior[...] = apply_flags(handler.registry, dims, d)
            h = L.BoundaryHandling(forest, st, ubb_velocity=(0.03, -0.01, 0.02)[:3],
                                   pressure_density=1.02, reference_density=0.99)
            h.freeze()
            shape = blk.data["flags"].view.shape + (st.q,)
            src = st.weights * (1.0 + 0.1 * rng.uniform(-1, 1, shape))
            dst = rng.standard_normal(shape)
            res = dst.copy()
            h.apply(blk, src, res)
            return src, dst, res, {k: h.link_count(blk) for k in ("all",)}
        src, dst, res, counts = SimRuntime(1, seed=0).run(prog)[0]
        out[f"{name}__src"], out[f"{name}__dst"], out[f"{name}__out"] = src, dst, res
        print("apply", name, counts)
    np.savez(HERE / "apply.npz", **out)


def make_units():
    """Reference unit functions on seeded random cells."""
    import blocksim.lbm as L
    from blocksim.lbm.collision import _kernel_params
    out = {}
    rng = np.random.default_rng(2024)
    for st in (L.D2Q9, L.D3Q19, L.D3Q27):
        n = 64
        rho = rng.uniform(0.5, 2.0, n)
        u = rng.uniform(-0.1, 0.1, (n, 3))
        if st.d == 2:
            u[:, 2] = 0.0
        f = L.equilibrium(rho, u, st)
        f *= 1.0 + 0.05 * rng.uniform(-1.0, 1.0, f.shape)
        out[f"{st.name}_in"] = f
        out[f"{st.name}_eq_rho"], out[f"{st.name}_eq_u"] = rho, u
        out[f"{st.name}_eq"] = L.equilibrium(rho, u, st)
        r, v = L.macroscopic(f, st)
        out[f"{st.name}_macro_rho"], out[f"{st.name}_macro_u"] = r, v
        r, v = L.macroscopic(f, st, force=L.Guo((3e-4, -2e-4, 1e-4)))
        out[f"{st.name}_macroguo_rho"], out[f"{st.name}_macroguo_u"] = r, v
        variants = {"srt": L.SRT(1.3), "trt": L.TRT(1.3, 0.9), "trtmagic": L.TRT.with_magic(1.7)}
        if st.name != "D3Q27":
            variants["mrtu"] = L.MRT.uniform(st, 1.3)
            if st.name == "D3Q19":
                rates = [1.0] * st.q
                rates[9:16] = [1.4] * 7
                variants["mrt"] = L.MRT(st, rates)
        forces = {"none": None, "guo": L.Guo((3e-4, -2e-4, 1e-4))}
        for vn, model in variants.items():
            for fn, force in forces.items():
                out[f"{st.name}_{vn}_{fn}"] = L.collide_pdfs(f, st, model, force)
            if isinstance(model, L.MRT):
                p = _kernel_params(st, model, L.Guo((3e-4, -2e-4, 1e-4)))
                out[f"{st.name}_{vn}_guo_matrix"] = p["guo_matrix"]
        out[f"{st.name}_srt_shift"] = L.collide_pdfs(f, st, L.SRT(1.3),
                                                     L.SimpleShift((3e-4, -2e-4, 1e-4)))
    for st in (L.D2Q9, L.D3Q19):
        out[f"{st.name}_M"] = L.moment_basis(st)
        out[f"{st.name}_Minv"] = L.basis_inverse(L.moment_basis(st))
    out["magic_omegas"] = np.array([L.TRT.with_magic(w).omega_o for w in (0.6, 1.0, 1.4, 1.7, 1.8)])
    out["equilibrium_hand"] = L.equilibrium(1.0, (0.1, 0.0), L.D2Q9)
    np.savez(HERE / "units.npz", **out)
    print("units:", len(out), "arrays")


if __name__ == "__main__":
    # python tests/golden/make_golden.py [case ... | snapshot]   (no args: everything)
    args = sys.argv[1:]
    if args == ["snapshot"]:
        make_snapshot()
    elif args == ["slot"]:
        make_slot()
    elif args == ["ownership"]:
        make_ownership()
    elif args == ["apply"]:
        make_apply()
    elif args == ["coupling"]:
        make_coupling()
    else:
        main(args or None)
        if not args:
            make_snapshot()
            make_coupling()
            make_slot()
            make_ownership()
            make_apply()
