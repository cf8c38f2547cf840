"""Stream-collide time step on HBM-resident PDF fields.

Drop-in for pkg/src/blocksim/lbm/sweep.py: same functions, arguments,
validation and results.  One `stream_collide` call is one fused sm_100a
pass (pull -> bounce-back -> collide) per rank box plus, across ranks, the
zero-copy halo of the crossing directions; the host arrays of the PDF slot
are a lazily synced mirror (see field.py / device.py).
"""
from __future__ import annotations

import numpy as np

from ..device import DeviceLattice
from ..errors import NumericsError, TopologyError, ValidationError
from ..field import FieldDataHandler
from .boundary import BoundaryHandling
from .collision import kernel_params
from .stencil import Stencil


class _Mirror:
    """Hook object installed on the src slot's host Fields."""

    def __init__(self, pdf):
        self.pdf = pdf

    def host_access(self):
        lat = self.pdf._lattice
        if lat is not None:
            lat.sync_host()
            lat.host_touched()


class _DstMirror:
    """Hook on the dst slot's host Fields: after a sweep the reference's dst
    slot holds the previous post-collision state C(R_{n-1}) with its covered
    ghosts (what the swap left there); it is read back from the device on
    access.  Host writes into the dst slot are not uploaded (the next sweep
    overwrites it in the reference too)."""

    def __init__(self, pdf):
        self.pdf = pdf

    def host_access(self):
        lat = self.pdf._lattice
        if lat is not None:
            lat.sync_host_dst()


class PdfSlotHandler(FieldDataHandler):
    """Data handler of the two PDF slots: lazily allocated host mirrors of
    the HBM state; snapshots serialise the reference's Field.raw content
    (src: R_n, dst: C(R_{n-1})) through the mirror, and restoring the src
    slot makes the host data authoritative again (the device lattice is
    rebuilt and re-uploaded before the next sweep)."""

    def __init__(self, pdf, which, nf, ghost_layers, layout):
        super().__init__(nf=nf, ghost_layers=ghost_layers, layout=layout, lazy=True)
        self.pdf = pdf
        self.which = which

    def create(self, forest, block):
        field = super().create(forest, block)
        field._mirror = self.pdf._mirror if self.which == "src" else self.pdf._dst_mirror
        return field

    def deserialize(self, forest, block, buf):
        if self.which == "src":
            self.pdf._lattice = None      # block objects change: new box, fresh upload
        field = FieldDataHandler.create(self, forest, block)
        raw = buf.unpack_array()
        if raw.shape != field._raw.shape:
            raise ValidationError(f"serialized field shape {raw.shape} != expected "
                                  f"{field._raw.shape}")
        field._raw[...] = raw
        field._mirror = self.pdf._mirror if self.which == "src" else self.pdf._dst_mirror
        return field


class PdfField:
    """Population storage: `key` (src) and `key.dst` host slots plus the
    device lattice (two HBM buffers) behind them.

    dtype="float32" (B200 extension) stores the centred populations f - w_i
    in fp32 and collides them in fp32 registers (checked at 1e-5 relative
    against the fp64 path); the host mirror stays fp64."""

    def __init__(self, forest, stencil: Stencil, key="pdf", *, layout="zyxf", ghost_layers=1,
                 dtype="float64"):
        if stencil.d != forest.d:
            raise ValidationError(f"{stencil.name} does not match a {forest.d}D forest")
        if dtype not in ("float64", "float32"):
            raise ValidationError(f"dtype must be 'float64' or 'float32', got {dtype!r}")
        self.forest = forest
        self.stencil = stencil
        self.key = key
        self.dst_key = key + ".dst"
        self.dtype = dtype
        self._lattice = None
        self._mirror = _Mirror(self)
        self._dst_mirror = _DstMirror(self)
        forest.register_data(key, PdfSlotHandler(self, "src", stencil.q, ghost_layers, layout))
        forest.register_data(self.dst_key, PdfSlotHandler(self, "dst", stencil.q, ghost_layers,
                                                          layout))
        self._kp_cache = {}

    def src(self, block):
        return block.data[self.key]

    def dst(self, block):
        return block.data[self.dst_key]

    def swap_all(self) -> None:
        for block in self.forest.local_blocks():
            self.src(block).swap_data(self.dst(block))

    @property
    def lattice(self) -> DeviceLattice:
        if self._lattice is None:
            self._lattice = DeviceLattice(self, self.dtype)
        return self._lattice

    @property
    def g(self):
        for block in self.forest.local_blocks():
            return block.data[self.key].g
        return 1

    def params(self, model, force, handling):
        """Kernel parameters + the collision identity key, cached by the
        parameter VALUES: the reference rebuilds its parameters on every
        sweep (lbm/sweep.py:116) and reads the handling's wall velocity and
        densities on every apply (boundary.py:165-171), so a model, force or
        handling mutated between sweeps (a ramped lid velocity, a new rate)
        must take effect here too."""
        ck = _value_key(model, force, handling)
        hit = self._kp_cache.get(ck)
        if hit is not None:
            return hit[1], hit[2]
        if len(self._kp_cache) >= 64:
            self._kp_cache.clear()
        uw = handling.ubb_velocity if handling is not None else (0.0, 0.0, 0.0)
        rho0 = handling.reference_density if handling is not None else 1.0
        kp = kernel_params(self.stencil, model, force, ubb_velocity=uw, reference_density=rho0)
        if handling is not None:
            for k in range(self.stencil.q):
                kp.struct.pressure[k] = 2.0 * self.stencil.weights[k] * handling.pressure_density
        s = kp.struct
        # (struct minus its three trailing pointers, MRT tables)
        key = (bytes(memoryview(s))[:-24], b"" if kp.tables is None else kp.tables.tobytes())
        self._kp_cache[ck] = (None, kp, key)
        return kp, key


def _floats(v):
    return None if v is None else tuple(float(x) for x in np.ravel(np.asarray(v, dtype=np.float64)))


def _value_key(model, force, handling):
    """Everything kernel_params / the boundary constants read, by value."""
    mk = (type(model).__name__, getattr(model, "omega", None), getattr(model, "omega_e", None),
          getattr(model, "omega_o", None), getattr(model, "omega_field", None))
    if getattr(model, "S", None) is not None:
        mk = mk + (id(model.stencil), np.asarray(model.S, dtype=np.float64).tobytes(),
                   np.asarray(model.M, dtype=np.float64).tobytes(),
                   np.asarray(model.Minv, dtype=np.float64).tobytes())
    fk = None if force is None else (type(force).__name__, _floats(force.force))
    hk = None if handling is None else (_floats(handling.ubb_velocity),
                                        float(handling.pressure_density),
                                        float(handling.reference_density))
    return mk, fk, hk


def fill_equilibrium(pdf: PdfField, rho=1.0, velocity=(0.0, 0.0, 0.0)) -> None:
    """Set the field to the equilibrium of (rho, velocity), ghosts included
    (sweep.py:51-76).  Callables are evaluated on the host over cell-centre
    coordinates exactly as the reference does; the equilibrium itself is
    computed on the device straight into the HBM layout."""
    forest = pdf.forest
    lat = pdf.lattice
    box = lat.box
    rviews, uviews = [], []
    for block in box.blocks:
        field = pdf.src(block)
        g = field.g
        (cx0, cy0, cz0), (dx, dy, dz) = forest.cell_centers(block.id)
        xs = cx0 + dx * (np.arange(field.nx + 2 * g) - g)
        ys = cy0 + dy * (np.arange(field.ny + 2 * g) - g)
        zs = cz0 + dz * (np.arange(field.nz + 2 * g) - g)
        z, y, x = np.meshgrid(zs, ys, xs, indexing="ij")
        r = rho(x, y, z) if callable(rho) else np.full(x.shape, float(rho))
        r = np.broadcast_to(np.asarray(r, dtype=np.float64), x.shape)
        if callable(velocity):
            u = np.stack(np.broadcast_arrays(*velocity(x, y, z)), axis=-1)
        else:
            u = np.broadcast_to(np.asarray(velocity, dtype=np.float64), x.shape + (len(velocity),))
        u = np.asarray(u, dtype=np.float64)
        if u.shape[-1] == 2:
            u = np.concatenate([u, np.zeros(u.shape[:-1] + (1,))], axis=-1)
        if u.shape[-1] != 3:
            raise ValidationError(f"velocity needs 2 or 3 components, got shape {u.shape}")
        rviews.append(r[..., None])
        uviews.append(u)
    rho_g = box.gather(rviews, 1, np.float64)[0]
    u_g = np.moveaxis(box.gather(uviews, 3, np.float64), 0, 3)
    lat.fill_equilibrium(rho_g, u_g)


def fill_equilibrium_arrays(pdf: PdfField, rho, u) -> None:
    """B200 extension: equilibrium of per-cell arrays of this rank's box,
    rho (nz, ny, nx) and u (nz, ny, nx, 3) (host numpy / pinned or device
    tensors).  Ghost cells take the nearest interior value.  One H2D copy of
    32 bytes per cell, the equilibrium is evaluated on the device."""
    import torch
    lat = pdf.lattice
    b = lat.box
    dev = lat.device
    tr = torch.empty((b.nz + 2, b.ny + 2, b.nx + 2), dtype=torch.float64, device=dev)
    tu = torch.empty((b.nz + 2, b.ny + 2, b.nx + 2, 3), dtype=torch.float64, device=dev)
    r = rho if isinstance(rho, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(rho))
    v = u if isinstance(u, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(u))
    if tuple(r.shape) != (b.nz, b.ny, b.nx) or tuple(v.shape) != (b.nz, b.ny, b.nx, 3):
        raise ValidationError("rho / u must cover this rank's box: "
                              f"({b.nz}, {b.ny}, {b.nx}) and (..., 3)")
    tr[1:-1, 1:-1, 1:-1].copy_(r, non_blocking=True)
    tu[1:-1, 1:-1, 1:-1].copy_(v, non_blocking=True)
    for t in (tr, tu):
        t[0] = t[1]
        t[-1] = t[-2]
        t[:, 0] = t[:, 1]
        t[:, -1] = t[:, -2]
        t[:, :, 0] = t[:, :, 1]
        t[:, :, -1] = t[:, :, -2]
    from .. import _lib
    _lib.call("lbm_fill_equilibrium", lat.gref, _lib.ptr(tr), _lib.ptr(tu),
              _lib.ptr(lat.buf[lat.cur]), lat._sp())
    lat.cur_kind, lat.prev_kind, lat.coll_key = "R", None, None
    lat.host_state, lat.snapshot = "device", None
    lat._dst_synced = None


def macroscopic_arrays(pdf: PdfField, *, force=None, out=None):
    """B200 extension: (rho, u) of this rank's box as device tensors, or
    copied into `out = (rho_host, u_host)` (e.g. pinned) - the D2H half of
    an end-to-end run.  Raises NumericsError on a non-positive density."""
    lat = pdf.lattice
    if lat.host_changed():
        lat.upload_host()
    from .collision import SRT, Guo, kernel_params as _kp
    kp = _kp(pdf.stencil, SRT(1.0), force if isinstance(force, Guo) else None)
    rho_t, u_t, bad = lat.moments(kp, lat.stream_masks or lat.default_masks())
    if out is not None:
        out[0].copy_(rho_t)
        out[1].copy_(u_t)
    if int(bad.item()):
        raise NumericsError(f"non-positive density {float(rho_t.min().item())}")
    return (rho_t, u_t) if out is None else out


def _require_uniform(forest) -> None:
    for block in forest.local_blocks():
        if block.level != 0:
            raise TopologyError("stream-collide needs a uniform refinement level")


def _prepare(pdf: PdfField, model, force, handling):
    forest = pdf.forest
    st = pdf.stencil
    _require_uniform(forest)
    if handling is not None and handling.stencil is not st:
        raise ValidationError("boundary handling built for a different stencil")
    if handling is None:
        for a in range(forest.d):
            if not forest.periodic[a]:
                raise ValidationError("without boundary handling the domain must be fully periodic")
    elif not handling.frozen:
        handling.freeze()
    if pdf.g != 1:
        raise ValidationError("stream-collide needs exactly one pdf ghost layer")
    lat = pdf.lattice
    if handling is not None:
        for block in forest.local_blocks():
            if block.data[handling.flags_key].g != pdf.g:
                raise ValidationError("flag and pdf ghost layers differ")
        masks = handling.sweep_masks()
        if masks.unflagged_cell is not None:
            raise ValidationError(f"unflagged cell {masks.unflagged_cell}")
    else:
        masks = lat.default_masks()
    kp, key = pdf.params(model, force, handling)
    key = key + (id(masks),)
    omega_key = getattr(model, "omega_field", None)
    if omega_key is not None:
        key = key + (("omega", _upload_rates(lat, omega_key)),)
        kp.struct.omega_cells = lat.omega_ptr
    if lat.host_changed():
        lat.upload_host()
    return lat, kp, key, masks


def _upload_rates(lat, omega_key):
    """Per-cell SRT rates of this rank's box interior -> HBM (sweep.py:
    138-146: validated in (0, 2) on every sweep).  Re-uploaded only when the
    host values changed; returns the content version (a change re-collides
    the stored state, as the reference collides with the current rates)."""
    box = lat.box
    dense = np.empty((box.nz, box.ny, box.nx), dtype=np.float64)
    for block, (ox, oy, oz) in zip(box.blocks, box.offsets):
        ow = block.data[omega_key]
        win = ow.field.view[..., 0] if hasattr(ow, "field") else ow.view[..., 0]
        inner = win[1:-1, 1:-1, 1:-1]
        if np.any(inner <= 0.0) or np.any(inner >= 2.0):
            raise ValidationError("per-cell rates must lie in (0, 2)")
        dense[oz:oz + inner.shape[0], oy:oy + inner.shape[1], ox:ox + inner.shape[2]] = inner
    return lat.set_rates(dense)


def stream_collide(pdf: PdfField, model, *, force=None, handling=None) -> None:
    """Advance the lattice by one time step (collective, sweep.py:93-151)."""
    lat, kp, key, masks = _prepare(pdf, model, force, handling)
    lat.step(kp, key, masks, 1)


def stream_collide_n(pdf: PdfField, model, steps, *, force=None, handling=None) -> None:
    """`steps` calls of stream_collide with one validation pass (B200
    extension for long time loops; bitwise identical to the loop)."""
    if steps < 0:
        raise ValidationError("steps must be >= 0")
    if steps == 0:
        return
    lat, kp, key, masks = _prepare(pdf, model, force, handling)
    lat.step(kp, key, masks, int(steps))


def macroscopic_fields(pdf: PdfField, density="rho", velocity="vel", *, force=None,
                       handling=None) -> None:
    """Per-cell density and velocity of fluid cells into registered fields
    (sweep.py:154-176), computed on the device from the current R-form."""
    forest = pdf.forest
    lat = pdf.lattice
    if lat.host_changed():
        lat.upload_host()
    from .collision import SRT, Guo, kernel_params as _kp
    kp = _kp(pdf.stencil, SRT(1.0), force if isinstance(force, Guo) else None)
    masks = lat.stream_masks or lat.default_masks()
    rho_t, u_t, bad = lat.moments(kp, masks)
    if int(bad.item()):
        raise NumericsError(f"non-positive density {float(rho_t.min().item())}")
    rho = rho_t.cpu().numpy()
    u = u_t.cpu().numpy()
    box = lat.box
    for block, (ox, oy, oz) in zip(box.blocks, box.offsets):
        n = forest.cells_per_block
        sl = (slice(oz, oz + n[2]), slice(oy, oy + n[1]), slice(ox, ox + n[0]))
        if handling is not None:
            flags = block.data[handling.flags_key]
            fluid = (flags.field.interior[..., 0] & handling.fluid_mask(block)) != 0
        else:
            fluid = slice(None)
        if density is not None:
            block.data[density].interior[..., 0][fluid] = rho[sl][fluid]
        if velocity is not None:
            out = block.data[velocity].interior
            for a in range(out.shape[-1]):
                out[..., a][fluid] = u[sl][..., a][fluid]


def mlups(interior_cells, steps, seconds) -> float:
    """Million lattice-cell updates per second (sweep.py:179-183)."""
    if seconds <= 0.0:
        raise ValidationError(f"need a positive wall time, got {seconds}")
    return interior_cells * steps / seconds / 1.0e6
