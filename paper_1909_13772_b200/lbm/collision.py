"""Collision operators, body forces and the kernel parameter block.

Model classes keep the reference's constructors, validation and attributes
(pkg/src/blocksim/lbm/collision.py:38-135).  `kernel_params` is the B200
counterpart of `_kernel_params` (:187-230): it fills the C-ABI struct
lbm_params_t with host-computed constants in the reference's arithmetic
(1 - omega, (1 - omega_e/2)/2, 6 w_k rho_0 (c_k . u_w), the BLAS-computed
guo_matrix ...), so the device never recomputes them differently.

`equilibrium`, `macroscopic` and `collide_pdfs` run on the GPU through the
flat-cell entry points of the kernel library (no CPU fallback).
"""
from __future__ import annotations

import ctypes
from fractions import Fraction

import numpy as np

from .. import _lib
from ..errors import NumericsError, ValidationError
from .stencil import Stencil, basis_inverse, moment_basis, raw_moment_basis

MAGIC_DEFAULT = Fraction(3, 16)


def _rate(label, value):
    """A relaxation rate, validated in the open interval (0, 2)."""
    v = float(value)
    if 0.0 < v < 2.0:
        return v
    raise ValidationError(f"{label} must lie in (0, 2), got {value}")


def _vector3(value, what="force"):
    """2 or 3 components -> a 3-tuple of floats (a 2D vector gets z = 0)."""
    v = tuple(map(float, value))
    if len(v) in (2, 3):
        return v + (0.0,) * (3 - len(v))
    raise ValidationError(f"{what} needs 2 or 3 components, got {value!r}")


class _Described:
    """repr() from the attributes listed in `_shown`."""

    _shown = ()

    def __repr__(self):
        body = ", ".join(f"{k}={getattr(self, k)!r}" for k in self._shown
                         if getattr(self, k) is not None)
        return f"{type(self).__name__}({body})"


class SRT(_Described):
    """Single relaxation rate: one global omega, or omega_field = the name
    of a per-cell rate field (read on every sweep)."""

    mode = 0
    _shown = ("omega", "omega_field")

    def __init__(self, omega=None, *, omega_field=None):
        if (omega is None) is (omega_field is None):
            raise ValidationError("SRT takes exactly one of omega and omega_field")
        self.omega = _rate("omega", omega) if omega is not None else None
        self.omega_field = omega_field


class TRT(_Described):
    """Two relaxation rates: even (omega_e) and odd (omega_o) parts."""

    mode = 1
    omega_field = None
    _shown = ("omega_e", "omega_o")

    def __init__(self, omega_e, omega_o):
        self.omega_e, self.omega_o = _rate("omega_e", omega_e), _rate("omega_o", omega_o)

    @classmethod
    def with_magic(cls, omega_e, magic=MAGIC_DEFAULT):
        """omega_o from the magic parameter Lambda = (1/omega_e - 1/2)(1/omega_o - 1/2)."""
        we = _rate("omega_e", omega_e)
        lam_e = 1.0 / we - 0.5
        if not lam_e > 0.0:
            raise ValidationError("omega_e = 2 leaves the magic value undefined")
        return cls(we, 1.0 / (float(magic) / lam_e + 0.5))

    @property
    def magic(self):
        return (1.0 / self.omega_e - 0.5) * (1.0 / self.omega_o - 0.5)


class MRT(_Described):
    """One relaxation rate per moment of a q x q basis: the stencil's
    Gram-Schmidt basis (M^-1 = M^T diag(1/|m|^2)), or an explicit invertible
    `basis=` (B200 extension; M^-1 = inv(basis)), which is how D3Q27 MRT is
    expressed - the reference's moment_basis rejects D3Q27."""

    mode = 2
    omega_field = None

    def __init__(self, stencil, rates, *, basis=None):
        self.stencil = stencil
        if basis is None:
            ints = moment_basis(stencil)
            self.M, self.Minv = ints.astype(np.float64), basis_inverse(ints)
        else:
            self.M = np.asarray(basis, dtype=np.float64)
            if self.M.shape != (stencil.q, stencil.q):
                raise ValidationError(f"basis must be {stencil.q}x{stencil.q}")
            self.Minv = np.linalg.inv(self.M)
        checked = [_rate(f"rate[{k}]", r) for k, r in enumerate(rates)]
        if len(checked) != stencil.q:
            raise ValidationError(f"{stencil.name} takes {stencil.q} rates, got {len(checked)}")
        self.S = np.array(checked)

    @classmethod
    def uniform(cls, stencil, omega):
        return cls(stencil, [omega] * stencil.q)

    @classmethod
    def raw_moments(cls, stencil, shear, other=1.0):
        """D3Q27 raw-moment MRT: the shear rows 4..8 relax at `shear`, all
        others at `other` (BASELINE config 2: 1.9 / 1.0)."""
        rates = [shear if 4 <= k <= 8 else other for k in range(stencil.q)]
        return cls(stencil, rates, basis=raw_moment_basis(stencil))

    def __repr__(self):
        return f"MRT({self.stencil.name}, rates={self.S.tolist()})"


class Guo(_Described):
    """Body force: half-shifted equilibrium velocity + relaxed source term."""

    mode = 1
    _shown = ("force",)

    def __init__(self, force):
        self.force = _vector3(force)


class SimpleShift(_Described):
    """Body force by shifting the equilibrium velocity by tau F / rho."""

    mode = 2
    _shown = ("force",)

    def __init__(self, force):
        self.force = _vector3(force)


class KernelParams:
    """lbm_params_t plus the arrays it points to (kept alive here)."""

    def __init__(self, struct, tables=None):
        self.struct = struct
        self.tables = tables

    @property
    def ref(self):
        return ctypes.byref(self.struct)


def kernel_params(stencil: Stencil, model, force=None, *, ubb_velocity=(0.0, 0.0, 0.0),
                  reference_density=1.0) -> KernelParams:
    """Validated kernel parameters (collision.py:187-230 + boundary.py:165-170)."""
    if isinstance(model, MRT) and model.stencil is not stencil:
        raise ValidationError(f"MRT basis built for {model.stencil.name}, sweep uses {stencil.name}")
    p = _lib.Params()
    tables = None
    if isinstance(model, SRT):
        if model.omega is None:
            # per-cell rates: the sweep points omega_cells at the device copy
            # of the rate field (lbm/sweep.py:111-146)
            p.model = _lib.SRT_FIELD
        else:
            p.model = 0
            p.omega = model.omega
            p.rem = 1.0 - model.omega
            p.hw = 1.0 - 0.5 * model.omega
    elif isinstance(model, TRT):
        p.model = 1
        p.omega_e, p.omega_o = model.omega_e, model.omega_o
        p.he_half = (1.0 - 0.5 * model.omega_e) * 0.5
        p.ho_half = (1.0 - 0.5 * model.omega_o) * 0.5
    elif isinstance(model, MRT):
        p.model = 2
    else:
        raise ValidationError(f"unknown collision model {model!r}")
    if force is not None:
        if isinstance(force, SimpleShift):
            if not isinstance(model, SRT) or model.omega is None:
                raise ValidationError("SimpleShift needs an SRT model with one global rate")
            tau = 1.0 / model.omega
            p.force_mode = 2
            p.fx, p.fy, p.fz = force.force
            p.shift_fx, p.shift_fy, p.shift_fz = (tau * v for v in force.force)
        elif isinstance(force, Guo):
            fx, fy, fz = force.force
            # Guo(0, 0, 0) is bitwise the unforced collision (test_lbm.py:239-248);
            # a force along x alone drops the +-0 y/z source terms (value-identical)
            if fx == 0.0 and fy == 0.0 and fz == 0.0:
                p.force_mode = 0
            elif fy == 0.0 and fz == 0.0:
                p.force_mode = 3
            else:
                p.force_mode = 1
            p.fx, p.fy, p.fz = force.force
            p.shift_fx, p.shift_fy, p.shift_fz = (0.5 * v for v in force.force)
        else:
            raise ValidationError(f"unknown force model {force!r}")
    if isinstance(model, MRT):
        q = stencil.q
        G = np.zeros((q, q))
        if isinstance(force, Guo):
            half = np.eye(q) - 0.5 * np.diag(model.S)
            G = model.Minv @ half @ model.M
        tables = np.ascontiguousarray(np.concatenate(
            [model.M.ravel(), model.Minv.ravel(), model.S.ravel(), G.ravel()]), dtype=np.float64)
        p.mrt = tables.ctypes.data
    uw = tuple(float(v) for v in ubb_velocity)
    if len(uw) == 2:
        uw = (uw[0], uw[1], 0.0)
    rho0 = float(reference_density)
    for k in range(stencil.q):
        cx, cy, cz = stencil.c[k]
        cu = cx * uw[0] + cy * uw[1] + cz * uw[2]
        p.ubb[k] = 6.0 * stencil.weights[k] * rho0 * cu
    return KernelParams(p, tables)


# ----------------------------------------------- flat-cell GPU utilities
def _device():
    import torch
    if not torch.cuda.is_available():
        from ..errors import BackendError
        raise BackendError("no CUDA device: the B200 path has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def equilibrium(rho, velocity, stencil: Stencil):
    """Second-order equilibrium populations, shape (..., q), computed on the
    GPU with equilibrium()'s operation order (collision.py:138-154)."""
    import torch
    rho = np.asarray(rho, dtype=np.float64)
    u = np.asarray(velocity, dtype=np.float64)
    if u.shape[-1] == 2:
        u = np.concatenate([u, np.zeros(u.shape[:-1] + (1,))], axis=-1)
    if u.shape[-1] != 3:
        raise ValidationError(f"velocity needs 2 or 3 components, got shape {u.shape}")
    shape = np.broadcast(rho, u[..., 0]).shape
    r = np.array(np.broadcast_to(rho, shape), dtype=np.float64).reshape(-1)
    uu = np.array(np.broadcast_to(u, shape + (3,)), dtype=np.float64).reshape(-1, 3)
    n = r.size
    dev = _device()
    tr = torch.from_numpy(r).to(dev)
    tu = torch.from_numpy(uu).to(dev)
    tf = torch.empty((n, stencil.q), dtype=torch.float64, device=dev)
    _lib.call("lbm_equilibrium_cells", stencil.q, _lib.ptr(tr), _lib.ptr(tu), _lib.ptr(tf), n,
              _lib.stream_ptr(torch.cuda.current_stream(dev)))
    return tf.cpu().numpy().reshape(shape + (stencil.q,))


def macroscopic(pdfs, stencil: Stencil, force=None):
    """Density and velocity of populations (..., q) on the GPU
    (collision.py:157-184); Guo adds F / (2 rho).  Raises NumericsError on a
    non-positive density."""
    import torch
    f = np.asarray(pdfs, dtype=np.float64)
    if f.shape[-1] != stencil.q:
        raise ValidationError(f"expected {stencil.q} populations, got {f.shape[-1]}")
    shape = f.shape[:-1]
    flat = np.ascontiguousarray(f.reshape(-1, stencil.q))
    n = flat.shape[0]
    kp = kernel_params(stencil, SRT(1.0), force if isinstance(force, Guo) else None)
    dev = _device()
    tf = torch.from_numpy(flat).to(dev)
    tr = torch.empty(n, dtype=torch.float64, device=dev)
    tu = torch.empty((n, 3), dtype=torch.float64, device=dev)
    bad = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.call("lbm_macroscopic_cells", stencil.q, kp.ref, _lib.ptr(tf), _lib.ptr(tr),
              _lib.ptr(tu), _lib.ptr(bad), n, _lib.stream_ptr(torch.cuda.current_stream(dev)))
    if int(bad.item()):
        rho = tr.cpu().numpy()
        raise NumericsError(f"non-positive density {float(np.min(rho))}")
    rho = tr.cpu().numpy().reshape(shape)
    u = tu.cpu().numpy().reshape(shape + (3,))
    return (float(rho) if rho.ndim == 0 else rho), u


def collide_pdfs(pdfs, stencil: Stencil, model, force=None):
    """Collide populations (..., q) on the GPU and return the result
    (collision.py:245-261)."""
    import torch
    if getattr(model, "omega_field", None) is not None:
        raise ValidationError("per-cell rates need a field context; use the block sweep")
    arr = np.array(pdfs, dtype=np.float64)
    if arr.shape[-1] != stencil.q:
        raise ValidationError(f"expected {stencil.q} populations, got {arr.shape[-1]}")
    kp = kernel_params(stencil, model, force)
    flat = np.ascontiguousarray(arr.reshape(-1, stencil.q))
    dev = _device()
    tf = torch.from_numpy(flat).to(dev)
    _lib.call("lbm_collide_cells", stencil.q, kp.ref, _lib.ptr(tf), flat.shape[0],
              _lib.stream_ptr(torch.cuda.current_stream(dev)))
    return tf.cpu().numpy().reshape(arr.shape)
