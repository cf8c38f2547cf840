"""ctypes driver for lbm_oracle.c plus small numpy restatements.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Every function cites the
reference code it restates (paths under /root/reference/pkg/src/blocksim).
"""
from __future__ import annotations

import ctypes
import os
from fractions import Fraction
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "build" / "liblbm_oracle.so"
MAGIC_DEFAULT = Fraction(3, 16)  # lbm/collision.py:19

# ------------------------------------------------------------------ stencils
_WEIGHTS = {  # lbm/stencil.py:16-21
    "D2Q9": {0: Fraction(4, 9), 1: Fraction(1, 9), 2: Fraction(1, 36)},
    "D3Q19": {0: Fraction(1, 3), 1: Fraction(1, 18), 2: Fraction(1, 36)},
    "D3Q27": {0: Fraction(8, 27), 1: Fraction(2, 27), 2: Fraction(1, 54), 3: Fraction(1, 216)},
}


class OStencil:
    """Velocity set built by the reference's rule (lbm/stencil.py:97-111)."""

    def __init__(self, name):
        d = 2 if name.startswith("D2") else 3
        cs = []
        for cz in ((-1, 0, 1) if d == 3 else (0,)):
            for cy in (-1, 0, 1):
                for cx in (-1, 0, 1):
                    n2 = cx * cx + cy * cy + cz * cz
                    if name == "D3Q19" and n2 > 2:
                        continue
                    cs.append((cx, cy, cz))
        cs.sort(key=lambda c: (c[0] ** 2 + c[1] ** 2 + c[2] ** 2, c[2], c[1], c[0]))
        self.name, self.d, self.q = name, d, len(cs)
        self.c = tuple(cs)
        self.wfrac = tuple(_WEIGHTS[name][c[0] ** 2 + c[1] ** 2 + c[2] ** 2] for c in cs)
        self.w = np.array([float(w) for w in self.wfrac])
        index = {c: i for i, c in enumerate(cs)}
        self.opp = tuple(index[(-c[0], -c[1], -c[2])] for c in cs)
        self.cx = np.array([c[0] for c in cs], dtype=np.int64)
        self.cy = np.array([c[1] for c in cs], dtype=np.int64)
        self.cz = np.array([c[2] for c in cs], dtype=np.int64)


STENCILS = {n: OStencil(n) for n in ("D2Q9", "D3Q19", "D3Q27")}


def moment_basis(st: OStencil) -> np.ndarray:
    """Gram-Schmidt integer basis (lbm/stencil.py:131-206)."""
    def c2(c):
        return c[0] ** 2 + c[1] ** 2 + c[2] ** 2
    if st.name == "D2Q9":
        seeds = [lambda c: 1, c2, lambda c: c2(c) ** 2, lambda c: c[0], lambda c: c[0] * c2(c),
                 lambda c: c[1], lambda c: c[1] * c2(c), lambda c: c[0] ** 2 - c[1] ** 2,
                 lambda c: c[0] * c[1]]
    elif st.name == "D3Q19":
        seeds = [lambda c: 1, c2, lambda c: c2(c) ** 2, lambda c: c[0], lambda c: c[0] * c2(c),
                 lambda c: c[1], lambda c: c[1] * c2(c), lambda c: c[2], lambda c: c[2] * c2(c),
                 lambda c: 3 * c[0] ** 2 - c2(c), lambda c: (3 * c[0] ** 2 - c2(c)) * c2(c),
                 lambda c: c[1] ** 2 - c[2] ** 2, lambda c: (c[1] ** 2 - c[2] ** 2) * c2(c),
                 lambda c: c[0] * c[1], lambda c: c[1] * c[2], lambda c: c[0] * c[2],
                 lambda c: (c[1] ** 2 - c[2] ** 2) * c[0], lambda c: (c[2] ** 2 - c[0] ** 2) * c[1],
                 lambda c: (c[0] ** 2 - c[1] ** 2) * c[2]]
    else:
        raise ValueError(f"no moment basis for {st.name}")
    rows = []
    for seed in seeds:
        v = [Fraction(seed(c)) for c in st.c]
        for r in rows:
            dot = sum(a * b for a, b in zip(v, r))
            if dot:
                nrm = sum(a * a for a in r)
                v = [a - dot * b / nrm for a, b in zip(v, r)]
        rows.append(v)
    out = np.zeros((st.q, st.q), dtype=np.int64)
    for k, r in enumerate(rows):
        scale = np.lcm.reduce([f.denominator for f in r])
        ints = [int(f * scale) for f in r]
        g = np.gcd.reduce([abs(i) for i in ints if i])
        out[k] = [i // g for i in ints]
    return out


def basis_inverse(M) -> np.ndarray:
    """M^-1 = M^T diag(1/|m|^2) (lbm/stencil.py:209-212)."""
    norms = np.einsum("ij,ij->i", M, M)
    return (M.T / norms[None, :]).astype(np.float64)


def raw_moment_basis_d3q27(st: OStencil) -> np.ndarray:
    """Oracle extension (the reference has no D3Q27 basis, stencil.py:171):
    shear-separated raw moments {1, x, y, z, xy, xz, yz, x2-y2, x2-z2,
    x2+y2+z2, then the 17 remaining monomials x^a y^b z^c, a,b,c in 0..2, in
    (a+b+c, c, b, a) order}.  Rows 4..8 are the shear moments."""
    def mono(a, b, c):
        return [cx ** a * cy ** b * cz ** c for cx, cy, cz in st.c]
    rows = [mono(0, 0, 0), mono(1, 0, 0), mono(0, 1, 0), mono(0, 0, 1),
            mono(1, 1, 0), mono(1, 0, 1), mono(0, 1, 1)]
    x2, y2, z2 = mono(2, 0, 0), mono(0, 2, 0), mono(0, 0, 2)
    rows.append([a - b for a, b in zip(x2, y2)])
    rows.append([a - b for a, b in zip(x2, z2)])
    rows.append([a + b + c for a, b, c in zip(x2, y2, z2)])
    used = {(0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1), (1, 1, 0), (1, 0, 1), (0, 1, 1),
            (2, 0, 0), (0, 2, 0), (0, 0, 2)}
    rest = sorted(((a, b, c) for a in range(3) for b in range(3) for c in range(3)
                   if (a, b, c) not in used), key=lambda t: (sum(t), t[2], t[1], t[0]))
    for a, b, c in rest:
        rows.append(mono(a, b, c))
    return np.array(rows, dtype=np.float64)


def trt_magic(omega_e, magic=MAGIC_DEFAULT):
    """TRT.with_magic (lbm/collision.py:66-74)."""
    lam_e = 1.0 / float(omega_e) - 0.5
    return float(omega_e), 1.0 / (float(magic) / lam_e + 0.5)


def equilibrium(rho, u, st: OStencil) -> np.ndarray:
    """lbm/collision.py:138-154, same numpy expression."""
    rho = np.asarray(rho, dtype=np.float64)
    u = np.asarray(u, dtype=np.float64)
    if u.shape[-1] == 2:
        u = np.concatenate([u, np.zeros(u.shape[:-1] + (1,))], axis=-1)
    ux, uy, uz = u[..., 0], u[..., 1], u[..., 2]
    usq = ux * ux + uy * uy + uz * uz
    out = np.empty(np.broadcast(rho, ux).shape + (st.q,))
    for i, (cx, cy, cz) in enumerate(st.c):
        cu = cx * ux + cy * uy + cz * uz
        out[..., i] = float(st.wfrac[i]) * rho * (1.0 + 3.0 * cu + 4.5 * cu * cu - 1.5 * usq)
    return out


def macroscopic(f, st: OStencil, force=None):
    """lbm/collision.py:157-184 (force: Guo vector or None)."""
    f = np.asarray(f, dtype=np.float64)
    rho = f[..., 0].copy()
    for i in range(1, st.q):
        rho = rho + f[..., i]
    m = np.zeros(rho.shape + (3,))
    for i, (cx, cy, cz) in enumerate(st.c):
        if cx:
            m[..., 0] += cx * f[..., i]
        if cy:
            m[..., 1] += cy * f[..., i]
        if cz:
            m[..., 2] += cz * f[..., i]
    inv = (1.0 / rho)[..., None]
    u = m * inv
    if force is not None:
        u = u + 0.5 * np.asarray(force, dtype=np.float64) * inv
    return rho, u


def link_sets(flags_g, st: OStencil, bits):
    """Exhaustive scan of boundary links (the reference test oracle scan_links,
    pkg/tests/test_lbm.py:280-296, and build_index_lists, lbm/boundary.py:48-97).
    flags_g: ghost-inclusive (Z, Y, X) with exchanged ghosts.  bits: dict of
    Fluid/NoSlip/UBB/Pressure masks.  Returns {name: sorted int array (n, 4)
    of (x, y, z, i)} in interior coordinates."""
    Z, Y, X = flags_g.shape
    nz, ny, nx = Z - 2, Y - 2, X - 2
    inner = flags_g[1:-1, 1:-1, 1:-1]
    fluid = (inner & bits["Fluid"]) != 0
    out = {}
    for name in ("NoSlip", "UBB", "Pressure"):
        rows = []
        for i in range(1, st.q):
            cx, cy, cz = st.c[i]
            nb = flags_g[1 + cz:1 + cz + nz, 1 + cy:1 + cy + ny, 1 + cx:1 + cx + nx]
            hit = fluid & ((nb & bits[name]) != 0)
            zs, ys, xs = np.nonzero(hit)
            rows.append(np.stack([xs, ys, zs, np.full_like(xs, i)], axis=1))
        arr = np.concatenate(rows, axis=0) if rows else np.zeros((0, 4), np.int64)
        order = np.lexsort((arr[:, 3], arr[:, 0], arr[:, 1], arr[:, 2]))
        out[name] = arr[order].astype(np.int32)
    return out


# ---------------------------------------------------------------- C driver
class _Stencil(ctypes.Structure):
    _fields_ = [("q", ctypes.c_int), ("cx", ctypes.c_int * 27), ("cy", ctypes.c_int * 27),
                ("cz", ctypes.c_int * 27), ("opp", ctypes.c_int * 27), ("w", ctypes.c_double * 27)]


class _Params(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int), ("force_mode", ctypes.c_int), ("omega", ctypes.c_double),
                ("omega_field", ctypes.c_void_p), ("omega_e", ctypes.c_double),
                ("omega_o", ctypes.c_double), ("M", ctypes.c_void_p), ("Minv", ctypes.c_void_p),
                ("S", ctypes.c_void_p), ("G", ctypes.c_void_p), ("fx", ctypes.c_double),
                ("fy", ctypes.c_double), ("fz", ctypes.c_double), ("shift_tau", ctypes.c_double)]


class _Links(ctypes.Structure):
    _fields_ = [("fluid", ctypes.c_uint32), ("noslip", ctypes.c_uint32), ("ubb", ctypes.c_uint32),
                ("pressure", ctypes.c_uint32), ("uwx", ctypes.c_double), ("uwy", ctypes.c_double),
                ("uwz", ctypes.c_double), ("rho0", ctypes.c_double), ("rho_w", ctypes.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            import subprocess
            import sys
            here = LIB_PATH.parent.parent
            subprocess.run([sys.executable, "-c",
                            "import sys; sys.path.insert(0, %r); "
                            "from paper_1909_13772_b200 import _build; _build.build_oracle()"
                            % str(here.parent)], check=True)
        _lib = ctypes.CDLL(str(LIB_PATH))
        P = ctypes.c_void_p
        _lib.orc_run.argtypes = [P, P, P, P, P, ctypes.c_uint32, ctypes.c_int, ctypes.c_int,
                                 ctypes.c_int, P, P, P, ctypes.c_int]
        _lib.orc_run.restype = ctypes.c_int
        _lib.orc_collide.argtypes = [P, P, P, ctypes.c_uint32, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_int, P]
        _lib.orc_exchange.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, P]
        _lib.orc_exchange_u32.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.c_int, P]
        _lib.orc_stream_pull.argtypes = [P, P, P, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        _lib.orc_apply_links.argtypes = [P, P, P, P, ctypes.c_int, ctypes.c_int, ctypes.c_int, P]
    return _lib


def _cstencil(st: OStencil):
    s = _Stencil()
    s.q = st.q
    for i in range(st.q):
        s.cx[i], s.cy[i], s.cz[i] = st.c[i]
        s.opp[i] = st.opp[i]
        s.w[i] = st.w[i]
    return s


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


class Model:
    """Collision + force description mirroring _kernel_params
    (lbm/collision.py:187-230)."""

    def __init__(self, kind, *, omega=None, omega_e=None, omega_o=None, M=None, Minv=None,
                 S=None, force=None, force_kind="guo", omega_field=None):
        self.kind = kind
        self.omega = omega
        self.omega_e, self.omega_o = omega_e, omega_o
        self.M = None if M is None else np.ascontiguousarray(M, dtype=np.float64)
        self.Minv = None if Minv is None else np.ascontiguousarray(Minv, dtype=np.float64)
        self.S = None if S is None else np.ascontiguousarray(S, dtype=np.float64)
        self.force = None if force is None else tuple(float(v) for v in force)
        self.force_kind = force_kind
        self.omega_field = omega_field
        self.G = None
        if kind == "MRT" and self.force is not None and force_kind == "guo":
            q = self.M.shape[0]
            half = np.eye(q) - 0.5 * np.diag(self.S)
            self.G = np.ascontiguousarray(self.Minv @ half @ self.M)

    def cparams(self):
        p = _Params()
        p.mode = {"SRT": 0, "TRT": 1, "MRT": 2}[self.kind]
        p.force_mode = 0 if self.force is None else (1 if self.force_kind == "guo" else 2)
        p.omega = self.omega or 0.0
        p.omega_field = _ptr(self.omega_field)
        p.omega_e = self.omega_e or 0.0
        p.omega_o = self.omega_o or 0.0
        p.M, p.Minv, p.S, p.G = _ptr(self.M), _ptr(self.Minv), _ptr(self.S), _ptr(self.G)
        if self.force is not None:
            p.fx, p.fy, p.fz = self.force
        if self.force_kind == "shift" and self.omega:
            p.shift_tau = 1.0 / self.omega
        return p


class Domain:
    """One global ghost-inclusive block driven with the reference step order.

    pdf: (q, Z, Y, X) float64 ("fzyx" raw).  flags: (Z, Y, X) uint32 or None
    (no handling: every cell collides, lbm/sweep.py:333-334).  periodic:
    (x, y, z) booleans.
    """

    def __init__(self, st: OStencil, dims, periodic, model: Model, flags=None, bits=None,
                 ubb_velocity=(0.0, 0.0, 0.0), reference_density=1.0, pressure_density=1.0):
        nx, ny, nz = dims
        self.st = st
        self.dims = (nx, ny, nz)
        self.X, self.Y, self.Z = nx + 2, ny + 2, nz + 2
        self.periodic = np.array([1 if p else 0 for p in periodic], dtype=np.int32)
        self.model = model
        self.a = np.zeros((st.q, self.Z, self.Y, self.X))
        self.b = np.zeros_like(self.a)
        if flags is None:
            self.flags = np.ones((self.Z, self.Y, self.X), dtype=np.uint32)
            self.fluid_bits = 1
            self.links = None
        else:
            self.flags = np.ascontiguousarray(flags, dtype=np.uint32).copy()
            # BoundaryHandling.freeze: exchange flag ghosts (boundary.py:128-131)
            lib().orc_exchange_u32(_ptr(self.flags), self.X, self.Y, self.Z, _ptr(self.periodic))
            self.fluid_bits = int(bits["Fluid"])
            self.bits = dict(bits)
            L = _Links()
            L.fluid, L.noslip, L.ubb = int(bits["Fluid"]), int(bits["NoSlip"]), int(bits["UBB"])
            L.pressure = int(bits["Pressure"])
            L.uwx, L.uwy, L.uwz = (float(v) for v in (tuple(ubb_velocity) + (0.0,))[:3])
            L.rho0 = float(reference_density)
            L.rho_w = float(pressure_density)
            self.links = L
        self._cst = _cstencil(st)
        if model.omega_field is not None:
            of = np.ascontiguousarray(model.omega_field, dtype=np.float64).copy()
            lib().orc_exchange(_ptr(of), 1, self.X, self.Y, self.Z, _ptr(self.periodic))
            model.omega_field = of
        self._cp = model.cparams()
        self.link_flags = None
        self.steps = 0

    def edit_flag(self, x, y, z, name):
        """Set interior cell (x, y, z) to flag `name` WITHOUT re-freezing:
        the links stay those of the initial flags (boundary.py:128-131), the
        collision reads the edited flags (lbm/sweep.py:124-136); ghost flags
        keep their last exchange, as in the reference."""
        if self.link_flags is None:
            self.link_flags = self.flags.copy()
        self.flags[z + 1, y + 1, x + 1] = self.bits[name]

    def set_full(self, pdf_qzyx):
        self.a[...] = pdf_qzyx
        self.b[...] = pdf_qzyx

    def run(self, steps):
        L = lib()
        odd = L.orc_run(ctypes.byref(self._cst), _ptr(self.a), _ptr(self.b), _ptr(self.flags),
                        _ptr(self.link_flags), self.fluid_bits, self.X, self.Y, self.Z, _ptr(self.periodic),
                        ctypes.byref(self._cp),
                        ctypes.byref(self.links) if self.links is not None else None, int(steps))
        if odd:
            self.a, self.b = self.b, self.a
        self.steps += steps

    def rform(self):
        """Interior R-form as the reference's logical (z, y, x, q) array."""
        return np.ascontiguousarray(np.moveaxis(self.a[:, 1:-1, 1:-1, 1:-1], 0, 3))


def threads_available():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def collide_cells(st: OStencil, f, model: Model):
    """impl.collide on a flat (n, q) population array (returns a copy)."""
    f = np.asarray(f, dtype=np.float64)
    n = f.shape[0]
    pdf = np.ascontiguousarray(f.T.reshape(st.q, 1, 1, n)).copy()
    flags = np.ones((1, 1, n), dtype=np.uint32)
    cst = _cstencil(st)
    cp = model.cparams()
    lib().orc_collide(ctypes.byref(cst), _ptr(pdf), _ptr(flags), 1, n, 1, 1, ctypes.byref(cp))
    return pdf.reshape(st.q, n).T.copy()
