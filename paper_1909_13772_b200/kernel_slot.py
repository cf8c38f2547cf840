"""The reference's kernel slot served by the sm_100a library.

`blocksim._kernels` picks its per-cell kernels at import
(pkg/src/blocksim/_kernels/__init__.py:10-37): `impl.collide(pdf, flags,
fluid_mask_bits, mode, params)` and `impl.stream_pull(src, dst, cx, cy, cz,
gl)` on numpy host views, with the contract "same expressions in the same
order ... agree bit for bit" (_core_py.py:3-6).  This module is that slot's
"b200" backend: the same two functions, the same arguments (the params dict
of `_kernel_params`, collision.py:187-230), computed on the GPU by
`lbm_slot_collide` / `lbm_slot_stream_pull` and written back into the views.

It is a per-call PARITY shim: each call copies its views to HBM and back,
so it is as slow as PCIe, not as fast as the sweep.  The performance
boundary is the sweep level (`stream_collide` keeps the state in HBM).
INTEGRATION.md shows the three lines that register it in the reference.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .errors import BackendError, ValidationError
from .lbm.stencil import D2Q9, D3Q19, D3Q27

BACKEND = "b200"
_STENCILS = {9: D2Q9, 19: D3Q19, 27: D3Q27}


def _device():
    import torch
    if not torch.cuda.is_available():
        raise BackendError("no CUDA device: the b200 kernel slot has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def _stencil_of(params):
    """The device kernels carry D2Q9/D3Q19/D3Q27 as compile-time tables:
    the caller's velocity set must be one of them, in the same order."""
    w = [float(v) for v in params["w"]]
    st = _STENCILS.get(len(w))
    if st is None:
        raise ValidationError(f"no device stencil with {len(w)} directions")
    same = (list(params["cx"]) == st.cx.tolist() and list(params["cy"]) == st.cy.tolist()
            and list(params["cz"]) == st.cz.tolist() and w == st.weights.tolist()
            and list(params["opp"]) == list(st.opp))
    if not same:
        raise ValidationError(f"velocity set differs from the device's {st.name} tables")
    return st


def _params_struct(q, mode, params):
    """lbm_params_t from the reference's params dict, with the constants
    computed in _core_py.py's own expressions (rem = 1 - omega, hw = 1 -
    0.5 omega, he * 0.5, tau F, 0.5 F)."""
    p = _lib.Params()
    keep = []
    if mode == 0:
        if params.get("omega_window") is None:
            om = float(params["omega"])
            p.model = _lib.SRT
            p.omega, p.rem, p.hw = om, 1.0 - om, 1.0 - 0.5 * om
        else:
            p.model = _lib.SRT_FIELD
    elif mode == 1:
        we, wo = float(params["omega_e"]), float(params["omega_o"])
        p.model = _lib.TRT
        p.omega_e, p.omega_o = we, wo
        p.he_half = (1.0 - 0.5 * we) * 0.5
        p.ho_half = (1.0 - 0.5 * wo) * 0.5
    elif mode == 2:
        p.model = _lib.MRT
    else:
        raise ValidationError(f"unknown collision mode {mode!r}")
    fm = int(params.get("force_mode", 0))
    fx, fy, fz = (float(v) for v in params.get("force", (0.0, 0.0, 0.0)))
    p.fx, p.fy, p.fz = fx, fy, fz
    if fm == 1:
        # Guo(0, 0, 0) is bitwise the unforced collision (test_lbm.py:239-248);
        # a force along x alone drops the +-0 y/z source terms (value-identical)
        p.force_mode = 0 if (fx == 0.0 and fy == 0.0 and fz == 0.0) else (
            3 if (fy == 0.0 and fz == 0.0) else 1)
        p.shift_fx, p.shift_fy, p.shift_fz = 0.5 * fx, 0.5 * fy, 0.5 * fz
    elif fm == 2:
        if mode != 0 or params.get("omega_window") is not None:
            raise ValidationError("SimpleShift needs an SRT model with one global rate")
        tau = float(params["shift_tau"])
        p.force_mode = 2
        p.shift_fx, p.shift_fy, p.shift_fz = tau * fx, tau * fy, tau * fz
    elif fm != 0:
        raise ValidationError(f"unknown force mode {fm!r}")
    if mode == 2:
        G = params.get("guo_matrix") if fm == 1 else None
        G = np.zeros((q, q)) if G is None else np.asarray(G, dtype=np.float64)
        tables = np.ascontiguousarray(np.concatenate(
            [np.asarray(params["M"], dtype=np.float64).ravel(),
             np.asarray(params["Minv"], dtype=np.float64).ravel(),
             np.asarray(params["S"], dtype=np.float64).ravel(), G.ravel()]))
        if tables.size != 3 * q * q + q:
            raise ValidationError("MRT tables do not match the velocity set")
        keep.append(tables)
        p.mrt = tables.ctypes.data
    return p, keep


def collide(pdf, flags, fluid_mask_bits, mode, params) -> None:
    """impl.collide (_core_py.py:70-200): collide, in place, every cell of
    the (z, y, x, q) view `pdf` (ghost ring included) whose flags have a bit
    of `fluid_mask_bits`."""
    import torch
    st = _stencil_of(params)
    q = st.q
    if pdf.ndim != 4 or pdf.shape[3] != q:
        raise ValidationError(f"pdf must be a (z, y, x, {q}) view, got {pdf.shape}")
    if tuple(flags.shape) != tuple(pdf.shape[:3]):
        raise ValidationError(f"flags {flags.shape} do not match pdf {pdf.shape[:3]}")
    p, keep = _params_struct(q, mode, params)
    dev = _device()
    n = int(np.prod(pdf.shape[:3]))
    tf = torch.from_numpy(np.ascontiguousarray(pdf, dtype=np.float64).reshape(n, q)).to(dev)
    tfl = torch.from_numpy(np.ascontiguousarray(flags, dtype=np.uint32).reshape(n)
                           .view(np.int32)).to(dev)
    tw = None
    if p.model == _lib.SRT_FIELD:
        win = np.asarray(params["omega_window"], dtype=np.float64)
        if tuple(win.shape) != tuple(pdf.shape[:3]):
            raise ValidationError(f"omega_window {win.shape} does not match pdf {pdf.shape[:3]}")
        tw = torch.from_numpy(np.ascontiguousarray(win).reshape(n)).to(dev)
        p.omega_cells = tw.data_ptr()
    _lib.call("lbm_slot_collide", q, ctypes.byref(p), _lib.ptr(tf), _lib.ptr(tfl),
              ctypes.c_uint32(int(fluid_mask_bits) & 0xFFFFFFFF), n,
              _lib.stream_ptr(torch.cuda.current_stream(dev)))
    pdf[...] = tf.cpu().numpy().reshape(pdf.shape)
    del keep, tw


def stream_pull(src, dst, cx, cy, cz, gl) -> None:
    """impl.stream_pull (_core_py.py:203-218): dst_i(x) = src_i(x - c_i) on
    the interior of the (z, y, x, q) views; dst's ghost cells are untouched."""
    import torch
    if src.ndim != 4 or tuple(src.shape) != tuple(dst.shape):
        raise ValidationError(f"src {src.shape} and dst {dst.shape} must be equal (z, y, x, q) views")
    nzg, nyg, nxg, q = src.shape
    gl = int(gl)
    c = [np.ascontiguousarray(np.asarray(v, dtype=np.int32)) for v in (cx, cy, cz)]
    if any(a.shape != (q,) for a in c):
        raise ValidationError("cx/cy/cz must have one entry per direction")
    nx, ny, nz = nxg - 2 * gl, nyg - 2 * gl, nzg - 2 * gl
    if min(nx, ny, nz) <= 0:
        return
    dev = _device()
    ts = torch.from_numpy(np.ascontiguousarray(src, dtype=np.float64)).to(dev)
    out = torch.empty((nz, ny, nx, q), dtype=torch.float64, device=dev)
    _lib.call("lbm_slot_stream_pull", q, c[0].ctypes.data, c[1].ctypes.data, c[2].ctypes.data,
              _lib.ptr(ts), _lib.ptr(out), nxg, nyg, nzg, gl,
              _lib.stream_ptr(torch.cuda.current_stream(dev)))
    dst[gl:gl + nz, gl:gl + ny, gl:gl + nx, :] = out.cpu().numpy()


def get_backend(name=None):
    """(module, label) as blocksim._kernels.get_backend returns them."""
    import sys
    if name not in (None, "", BACKEND):
        raise ValueError(f"unknown kernel backend {name!r}")
    return sys.modules[__name__], BACKEND
