"""ctypes binding of the sm_100a kernel library (include/lbm_b200.h).

The library is loaded from the package directory (built in-tree by
`_build.build_kernels`).  Every compute entry point of the package goes
through `call()`, which maps status codes onto the reference's exception
classes.  There is no fallback: a missing library or a failed launch raises.
"""
from __future__ import annotations

import ctypes
from pathlib import Path

from .errors import BackendError, NumericsError, ValidationError

LIB_PATH = Path(__file__).resolve().parent / "_lbm_b200.so"

LBM_OK, LBM_EINVAL, LBM_ECUDA, LBM_ENUMERIC, LBM_EFLAGS = 0, -1, -2, -3, -4
ZFACE_GHOST, ZFACE_HALO, ZFACE_WRAP = 0, 1, 2
ABI_VERSION = 8
SRT, TRT, MRT, SRT_FIELD = 0, 1, 2, 3
MASK_FLUID = 0x1
MASK_UBB = 0x80000000
MASK_MOVING = 0x20000000

# every symbol include/lbm_b200.h declares (tests check the export table)
EXPORTS = (
    "lbm_abi_version", "lbm_struct_size", "lbm_last_error", "lbm_slot_of", "lbm_field_elems", "lbm_face_span",
    "lbm_fused_step", "lbm_collide_only", "lbm_stream_only", "lbm_moments",
    "lbm_pack_rform", "lbm_unpack_rform", "lbm_fill_equilibrium", "lbm_build_cellmask",
    "lbm_collide_cells", "lbm_equilibrium_cells", "lbm_macroscopic_cells",
    "lbm_build_moving_masks", "lbm_fused_step_peer", "lbm_ghost_block_offset",
    "lbm_stream_signal", "lbm_stream_wait", "lbm_copy_async",
    "lbm_ipc_export", "lbm_ipc_open", "lbm_ipc_close",
    "lbm_bind_params", "lbm_slot_collide", "lbm_slot_stream_pull", "lbm_refresh_fluid_mask",
    "lbm_map_spheres", "lbm_copy_shell", "lbm_slot_apply_links",
    "lbm_fill_equilibrium_planes", "lbm_collide_only_planes", "lbm_moments_planes",
    "lbm_fill_collide_planes", "lbm_can_flush_remote_writes", "lbm_fused_step_moments",
    "lbm_fused_step_bits", "lbm_linkbits_words", "lbm_build_linkbits",
)


class Grid(ctypes.Structure):
    """lbm_grid_t"""
    _fields_ = [("q", ctypes.c_int), ("real_bytes", ctypes.c_int), ("nx", ctypes.c_int),
                ("ny", ctypes.c_int), ("nz", ctypes.c_int), ("pitch", ctypes.c_int),
                ("xoff", ctypes.c_int), ("wrap_x", ctypes.c_int), ("wrap_y", ctypes.c_int),
                ("zface_lo", ctypes.c_int), ("zface_hi", ctypes.c_int)]


class Params(ctypes.Structure):
    """lbm_params_t"""
    _fields_ = [("model", ctypes.c_int), ("force_mode", ctypes.c_int),
                ("omega", ctypes.c_double), ("rem", ctypes.c_double), ("hw", ctypes.c_double),
                ("omega_e", ctypes.c_double), ("omega_o", ctypes.c_double),
                ("he_half", ctypes.c_double), ("ho_half", ctypes.c_double),
                ("fx", ctypes.c_double), ("fy", ctypes.c_double), ("fz", ctypes.c_double),
                ("shift_fx", ctypes.c_double), ("shift_fy", ctypes.c_double),
                ("shift_fz", ctypes.c_double), ("ubb", ctypes.c_double * 27),
                ("pressure", ctypes.c_double * 27), ("mrt", ctypes.c_void_p),
                ("omega_cells", ctypes.c_void_p), ("moving", ctypes.c_void_p)]


class Moving(ctypes.Structure):
    """lbm_moving_t"""
    _fields_ = [("owner", ctypes.c_void_p), ("linkmask", ctypes.c_void_p),
                ("bodies", ctypes.c_void_p), ("cell0", ctypes.c_void_p),
                ("forces", ctypes.c_void_p), ("n_slots", ctypes.c_int),
                ("blocks", ctypes.c_int * 3), ("block_cells", ctypes.c_int * 3),
                ("rho0", ctypes.c_double)]


_lib = None


def load(path: Path | None = None):
    """Load (once) and return the kernel library; raises BackendError."""
    global _lib
    if _lib is not None:
        return _lib
    import os
    p = Path(path or os.environ.get("LBM_B200_LIB") or LIB_PATH)
    if not p.exists():
        raise BackendError(
            f"B200 kernel library {p} is missing; build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)")
    lib = ctypes.CDLL(str(p))
    P, I, I64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
    G, PR = ctypes.POINTER(Grid), ctypes.POINTER(Params)
    sig = {
        "lbm_abi_version": ([], I),
        "lbm_struct_size": ([I], ctypes.c_size_t),
        "lbm_last_error": ([], ctypes.c_char_p),
        "lbm_slot_of": ([I, I], I),
        "lbm_field_elems": ([G], I64),
        "lbm_face_span": ([G, I, ctypes.POINTER(I64), ctypes.POINTER(I64), ctypes.POINTER(I64)], I),
        "lbm_fused_step": ([G, PR, P, P, P, P, I, I, P], I),
        "lbm_collide_only": ([G, PR, P, P, P], I),
        "lbm_stream_only": ([G, PR, P, P, P, P, P], I),
        "lbm_moments": ([G, PR, P, P, P, I, P, P, P, P], I),
        "lbm_pack_rform": ([G, P, P, P], I),
        "lbm_unpack_rform": ([G, P, P, P], I),
        "lbm_fill_equilibrium": ([G, P, P, P, P], I),
        "lbm_build_cellmask": ([G, P, P, P, P, P, P], I),
        "lbm_collide_cells": ([I, PR, P, I64, P], I),
        "lbm_equilibrium_cells": ([I, P, P, P, I64, P], I),
        "lbm_macroscopic_cells": ([I, PR, P, P, P, P, I64, P], I),
        "lbm_build_moving_masks": ([G, P, P, P, P, P, P], I),
        "lbm_fused_step_peer": ([G, PR, P, P, P, P, I, I, P, P, P], I),
        "lbm_ghost_block_offset": ([G, I, ctypes.POINTER(I64)], I),
        "lbm_stream_signal": ([P, ctypes.c_uint32, P], I),
        "lbm_stream_wait": ([P, ctypes.c_uint32, P], I),
        "lbm_copy_async": ([P, P, I64, P], I),
        "lbm_ipc_export": ([P, P, ctypes.POINTER(I64)], I),
        "lbm_ipc_open": ([P, ctypes.POINTER(P)], I),
        "lbm_ipc_close": ([P], I),
        "lbm_bind_params": ([G, PR, P], I),
        "lbm_slot_collide": ([I, PR, P, P, ctypes.c_uint32, I64, P], I),
        "lbm_slot_stream_pull": ([I, P, P, P, P, P, I, I, I, I, P], I),
        "lbm_refresh_fluid_mask": ([G, P, P, P, P, P, P], I),
        "lbm_map_spheres": ([I, P, P, P, P, P, P, ctypes.c_uint32, P, P], I),
        "lbm_copy_shell": ([G, P, P, P], I),
        "lbm_slot_apply_links": ([I, PR, P, P, P, I64, P, P, P], I),
        "lbm_fill_equilibrium_planes": ([G, P, P, I, I, P, P, P], I),
        "lbm_collide_only_planes": ([G, PR, P, P, I, I, P], I),
        "lbm_moments_planes": ([G, PR, P, P, P, I, I, I, P, P, P, P], I),
        "lbm_fused_step_moments": ([G, PR, PR, P, P, P, P, I, I, P, P, P, P], I),
        "lbm_fill_collide_planes": ([G, PR, P, P, I, I, P, P, P, P], I),
        "lbm_can_flush_remote_writes": ([], I),
        "lbm_fused_step_bits": ([G, PR, P, P, P, P, P, I, I, P], I),
        "lbm_linkbits_words": ([G], I64),
        "lbm_build_linkbits": ([G, P, P, P, P], I),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if lib.lbm_abi_version() != ABI_VERSION:
        raise BackendError("kernel library ABI mismatch")
    if (lib.lbm_struct_size(0) != ctypes.sizeof(Grid)
            or lib.lbm_struct_size(1) != ctypes.sizeof(Params)
            or lib.lbm_struct_size(2) != ctypes.sizeof(Moving)):
        raise BackendError("lbm_grid_t / lbm_params_t / lbm_moving_t layout differs between "
                           "include/lbm_b200.h "
                           "and the ctypes mirror")
    _lib = lib
    return lib


def call(name, *args):
    """Invoke `name`, turning a non-zero status into the matching exception."""
    lib = load()
    st = getattr(lib, name)(*args)
    if st != LBM_OK:
        msg = (lib.lbm_last_error() or b"").decode(errors="replace")
        if st == LBM_EINVAL or st == LBM_EFLAGS:
            raise ValidationError(f"{name}: {msg}")
        if st == LBM_ENUMERIC:
            raise NumericsError(f"{name}: {msg}")
        raise BackendError(f"{name}: {msg}")
    return st


def ptr(t) -> ctypes.c_void_p:
    """Device pointer of a torch tensor (or None)."""
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def stream_ptr(stream) -> ctypes.c_void_p:
    return ctypes.c_void_p(stream.cuda_stream)
