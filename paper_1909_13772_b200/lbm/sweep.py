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
        self.layout = layout
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
    lat = pdf.lattice
    rviews, uviews = [], []
    for block in lat.box.blocks:
        x, y, z = _cell_centres(pdf.forest, block.id, pdf.src(block))
        r = rho(x, y, z) if callable(rho) else float(rho)
        rviews.append(np.broadcast_to(np.asarray(r, dtype=np.float64), x.shape)[..., np.newaxis])
        if callable(velocity):
            comps = np.broadcast_arrays(*velocity(x, y, z))
        else:
            comps = [np.full(x.shape, float(v)) for v in velocity]
        if len(comps) not in (2, 3):
            raise ValidationError(f"velocity needs 2 or 3 components, got {len(comps)}")
        comps = list(comps) + [np.zeros(x.shape)] * (3 - len(comps))
        uviews.append(np.stack([np.asarray(c, dtype=np.float64) for c in comps], axis=-1))
    rho_g = lat.box.gather(rviews, 1, np.float64)[0]
    u_g = np.moveaxis(lat.box.gather(uviews, 3, np.float64), 0, 3)
    lat.fill_equilibrium(rho_g, u_g)


def _cell_centres(forest, block_id, field):
    """(x, y, z) grids of a block's ghost-inclusive cell centres: corner
    centre + spacing * index, index running from -g (the reference's
    expressions, sweep.py:58-62, so callables see identical coordinates)."""
    c0, h = forest.cell_centers(block_id)
    g = field.g
    axes = [c0[a] + h[a] * np.arange(-g, n + g) for a, n in enumerate((field.nx, field.ny,
                                                                        field.nz))]
    z, y, x = np.meshgrid(axes[2], axes[1], axes[0], indexing="ij")
    return x, y, z


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


def _require_uniform(forest):
    if any(block.level != 0 for block in forest.local_blocks()):
        raise TopologyError("stream-collide needs a uniform refinement level")


def sweep_masks(pdf, handling):
    """Device masks of the next sweep after the reference's checks
    (sweep.py:97-136): one level, a handling of this stencil or a fully
    periodic domain, one ghost layer on pdf and flags, no unflagged interior
    cell.  A handling is frozen on first use (sweep.py:107-108)."""
    forest = pdf.forest
    _require_uniform(forest)
    if handling is None:
        if not all(forest.periodic[:forest.d]):
            raise ValidationError("without boundary handling the domain must be fully periodic")
    elif handling.stencil is not pdf.stencil:
        raise ValidationError("boundary handling built for a different stencil")
    if pdf.g != 1:
        raise ValidationError("stream-collide needs exactly one pdf ghost layer")
    if handling is None:
        return pdf.lattice.default_masks()
    if not handling.frozen:
        handling.freeze()
    if any(b.data[handling.flags_key].g != pdf.g for b in forest.local_blocks()):
        raise ValidationError("flag and pdf ghost layers differ")
    masks = handling.sweep_masks()
    if masks.unflagged_cell is not None:
        raise ValidationError(f"unflagged cell {masks.unflagged_cell}")
    return masks


def _prepare(pdf, model, force, handling, upload=True):
    masks = sweep_masks(pdf, handling)
    lat = pdf.lattice
    kp, key = pdf.params(model, force, handling)
    key = key + (id(masks),)
    omega_key = getattr(model, "omega_field", None)
    if omega_key is not None:
        key = key + (("omega", _upload_rates(lat, omega_key)),)
        kp.struct.omega_cells = lat.omega_ptr
    if upload and lat.host_changed():
        lat.upload_host()
    return lat, kp, key, masks


def _upload_rates(lat, omega_key):
    """Per-cell SRT rates of this rank's box interior -> HBM (sweep.py:
    138-146: validated in (0, 2) on every sweep).  Re-uploaded only when the
    host values changed; returns the content version (a change re-collides
    the stored state, as the reference collides with the current rates)."""
    box = lat.box
    views = []
    for block in box.blocks:
        slot = block.data[omega_key]
        views.append(getattr(slot, "field", slot).view[..., :1])
    dense = box.gather(views, 1, np.float64)[0, 1:-1, 1:-1, 1:-1]
    if not np.all((dense > 0.0) & (dense < 2.0)):
        raise ValidationError("per-cell rates must lie in (0, 2)")
    return lat.set_rates(np.ascontiguousarray(dense))


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


def run_arrays(pdf: PdfField, model, steps, rho, u, *, force=None, handling=None, out=None,
               chunk_planes=None):
    """B200 extension: one job from host arrays to host arrays,
        fill_equilibrium_arrays(pdf, rho, u)
        steps x stream_collide(pdf, model, force=force, handling=handling)
        return macroscopic_arrays(pdf, force=force, out=out)
    with bitwise the same results and end state.  On one rank with a
    non-periodic z axis it runs as a wavefront over chunks of z-planes
    (DeviceLattice.run_job): the upload of later planes, the sweeps of
    earlier ones and the download of finished ones overlap, so a job pays
    for PCIe roughly once instead of on top of its sweeps.  `out` = (rho,
    u) host tensors (pinned for overlap); without it host tensors are
    allocated."""
    import torch
    steps = int(steps)
    if steps < 0:
        raise ValidationError("steps must be >= 0")
    lat = pdf.lattice
    b = lat.box
    r = rho if isinstance(rho, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(rho))
    v = u if isinstance(u, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(u))
    if tuple(r.shape) != (b.nz, b.ny, b.nx) or tuple(v.shape) != (b.nz, b.ny, b.nx, 3):
        raise ValidationError("rho / u must cover this rank's box: "
                              f"({b.nz}, {b.ny}, {b.nx}) and (..., 3)")
    if steps == 0 or not lat.can_pipeline() or r.is_cuda or v.is_cuda:
        fill_equilibrium_arrays(pdf, r, v)
        for _ in range(steps):
            stream_collide(pdf, model, force=force, handling=handling)
        return macroscopic_arrays(pdf, force=force, out=out)
    r = r.to(torch.float64).contiguous()
    v = v.to(torch.float64).contiguous()
    if out is None:
        out = (torch.empty(tuple(r.shape), dtype=torch.float64),
               torch.empty(tuple(v.shape), dtype=torch.float64))
    # validation and parameters of the sweeps; the job replaces the whole
    # device state, so host-side PDF data is not uploaded first
    lat, kp, key, masks = _prepare(pdf, model, force, handling, upload=False)
    from .collision import SRT, Guo, kernel_params as _kp
    kp_m = _kp(pdf.stencil, SRT(1.0), force if isinstance(force, Guo) else None)
    bad = lat.run_job(kp, key, masks, kp_m, r, v, steps, out, chunk_planes)
    if int(bad.item()):
        raise NumericsError(f"non-positive density {float(out[0].min())}")
    return out


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
    rho, u = rho_t.cpu().numpy(), u_t.cpu().numpy()
    cpb = forest.cells_per_block
    for block, off in zip(lat.box.blocks, lat.box.offsets):
        window = tuple(slice(off[a], off[a] + cpb[a]) for a in (2, 1, 0))
        keep = np.ones(tuple(cpb[::-1]), dtype=bool)
        if handling is not None:
            bits = block.data[handling.flags_key].field.interior[..., 0]
            keep = (bits & handling.fluid_mask(block)) != 0
        if density is not None:
            dst = block.data[density].interior[..., 0]
            dst[keep] = rho[window][keep]
        if velocity is not None:
            dst = block.data[velocity].interior
            src = u[window][..., :dst.shape[-1]]
            dst[keep] = src[keep]


def mlups(interior_cells, steps, seconds):
    """Million lattice-cell updates per second (sweep.py:179-183): every
    interior cell counts, solid ones included."""
    if not seconds > 0.0:
        raise ValidationError(f"mlups needs a positive wall time, got {seconds}")
    return interior_cells * steps / seconds / 1.0e6
