"""Flag-driven boundary conditions: registry, validation, device link masks.

Same flags, registry order and validation rules as the reference
(pkg/src/blocksim/lbm/boundary.py:26-195).  Instead of per-type link lists
scattered after the stream (BoundaryHandling.apply), `freeze()` builds a
per-cell link mask on the device (lbm_build_cellmask) that the fused
stream-collide kernel consumes, so bounce-back costs 4 bytes per cell inside
the one pass over HBM.  `links` / `build_index_lists` decode that mask back
into the reference's list format for inspection and tests.
"""
from __future__ import annotations

import ctypes

import numpy as np

from .. import _lib
from ..device import Masks, RankBox
from ..errors import ValidationError
from ..field import FlagFieldHandler, GhostPackInfo, exchange_ghosts
from .stencil import Stencil

# the five canonical flag names, in registration order
BOUNDARY_FLAGS = FLUID, NO_SLIP, UBB, PRESSURE, SOLID = ("Fluid", "NoSlip", "UBB", "Pressure",
                                                         "Solid")
_LINK_FLAGS = BOUNDARY_FLAGS[1:4]     # flags a fluid cell bounces back from


def ensure_flags(forest, flags="flags", ghost_layers=1):
    """The flag slot `flags` (registered on first use) with the five
    canonical names registered in their fixed order (boundary.py:35-45):
    on a fresh slot Fluid=1, NoSlip=2, UBB=4, Pressure=8, Solid=16."""
    handler = forest.handlers.get(flags)
    if handler is None:
        handler = FlagFieldHandler(ghost_layers)
        forest.register_data(flags, handler)
    elif not isinstance(handler, FlagFieldHandler):
        raise ValidationError(f"data slot {flags!r} holds no flag field")
    for name in (n for n in BOUNDARY_FLAGS if n not in handler.registry):
        handler.register(name)
    return handler


def _flag_bits(registry):
    return (ctypes.c_uint32 * 5)(*(int(registry[n]) for n in (FLUID, NO_SLIP, UBB, PRESSURE, SOLID)))


def build_masks(forest, stencil: Stencil, flags="flags", device=None) -> Masks:
    """Device link masks of this rank's box from the host flags (ghost
    flags must be current).  Raises the reference's ValidationErrors."""
    import torch
    box = RankBox(forest)
    blocks = box.blocks
    for b in blocks:
        if b.data[flags].g < 1:
            raise ValidationError("boundary links need one flag ghost layer")
    views = [b.data[flags].field.view_nosync for b in blocks]
    dense = box.gather(views, 1, np.uint32)[0]
    if device is None:
        device = forest.ctx.device if forest.ctx.device.type == "cuda" else torch.device("cuda")
    g = _lib.Grid()
    g.q, g.real_bytes = stencil.q, 8
    g.nx, g.ny, g.nz = box.nx, box.ny, box.nz
    g.xoff, g.pitch = 1, box.nx + 2
    g.wrap_x, g.wrap_y = int(box.wrap_x), int(box.wrap_y)
    g.zface_lo, g.zface_hi = box.zface_lo, box.zface_hi
    tf = torch.from_numpy(dense.view(np.int32)).to(device)
    cm = torch.empty((box.nz, box.ny, box.nx), dtype=torch.int32, device=device)
    tm = torch.empty((box.nz, box.ny, box.nx, 2), dtype=torch.int32, device=device)
    big = np.iinfo(np.int32).max
    err = torch.tensor([big, big, big, big, 0, 0, 0, big], dtype=torch.int32, device=device)
    registry = blocks[0].data[flags].registry
    _lib.call("lbm_build_cellmask", ctypes.byref(g), _lib.ptr(tf), _flag_bits(registry),
              _lib.ptr(cm), _lib.ptr(tm), _lib.ptr(err),
              _lib.stream_ptr(torch.cuda.current_stream(device)))
    e = err.cpu().numpy().tolist()

    def where(v):
        c = v - 1
        x = c % box.nx
        y = (c // box.nx) % box.ny
        z = c // (box.nx * box.ny)
        return (box.lo[0] + x, box.lo[1] + y, box.lo[2] + z)

    if e[0] != big:
        raise ValidationError(f"cell {where(e[0])} carries conflicting boundary flags")
    if e[1] != big:
        raise ValidationError(f"fluid cell {where(e[1])} streams from a Solid cell; flag the "
                              "obstacle surface NoSlip/UBB/Pressure")
    if e[2] != big:
        raise ValidationError(f"fluid cell {where(e[2])} streams from an unflagged cell")
    if e[7] != big:
        raise ValidationError(f"fluid cell {where(e[7])} streams from a Fluid-flagged ghost cell "
                              "outside a non-periodic domain face (not supported on the B200 path)")
    counts = {NO_SLIP: e[5], UBB: e[4], PRESSURE: e[6]}
    return Masks(cm, tm, counts, None if e[3] == big else where(e[3]))


def decode_links(forest, stencil: Stencil, masks: Masks, flags="flags"):
    """{block_id: {name: [(i, zs, ys, xs)]}} from device masks, in the
    reference's format (boundary.py:91-96): i is the direction from the
    fluid cell into the boundary cell, indices are ghost-inclusive."""
    box = RankBox(forest)
    cm = masks.cellmask.cpu().numpy().view(np.uint32)
    tm = masks.typemask.cpu().numpy().view(np.uint32)
    fluid = (cm & _lib.MASK_FLUID) != 0
    out = {}
    for block, (ox, oy, oz) in zip(box.blocks, box.offsets):
        g = block.data[flags].g
        n = forest.cells_per_block
        sl = (slice(oz, oz + n[2]), slice(oy, oy + n[1]), slice(ox, ox + n[0]))
        c, t0, t1, fl = cm[sl], tm[sl][..., 0], tm[sl][..., 1], fluid[sl]
        lists = {name: [] for name in _LINK_FLAGS}
        for i in range(1, stencil.q):
            j = stencil.opp[i]                     # pulled direction carrying the link
            hit = fl & (((c >> j) & 1) != 0)
            is_ubb = ((t0 >> j) & 1) != 0
            is_pr = ((t1 >> j) & 1) != 0
            for name, sel in ((NO_SLIP, hit & ~is_ubb & ~is_pr), (UBB, hit & is_ubb),
                              (PRESSURE, hit & is_pr)):
                if sel.any():
                    zs, ys, xs = np.nonzero(sel)
                    lists[name].append((i, zs + g, ys + g, xs + g))
        out[block.id] = lists
    return out


def build_index_lists(forest, stencil: Stencil, flags="flags"):
    """Boundary links per local block (boundary.py:48-97), computed on the
    device.  Ghost flags must be current (exchange first; freeze does)."""
    return decode_links(forest, stencil, build_masks(forest, stencil, flags), flags)


class BoundaryHandling:
    """Boundary configuration plus frozen device link masks (boundary.py:100-152).

    freeze() is collective: it refreshes flag ghosts, then builds the masks.
    Call it again after editing flags."""

    def __init__(self, forest, stencil: Stencil, *, flags="flags", ubb_velocity=(0.0, 0.0, 0.0),
                 pressure_density=1.0, reference_density=1.0):
        if stencil.d != forest.d:
            raise ValidationError(f"{stencil.name} does not match a {forest.d}D forest")
        self.forest = forest
        self.stencil = stencil
        self.flags_key = flags
        uw = tuple(float(v) for v in ubb_velocity)
        if len(uw) not in (2, 3):
            raise ValidationError(f"wall velocity needs 2 or 3 components, got {ubb_velocity!r}")
        self.ubb_velocity = uw + (0.0,) * (3 - len(uw))
        self.pressure_density, self.reference_density = (float(pressure_density),
                                                         float(reference_density))
        self.handler = ensure_flags(forest, flags)
        self._masks = self._links = None
        self.generation = 0

    def freeze(self):
        """Collective: refresh the flag ghosts, then build the device masks."""
        exchange_ghosts(self.forest, [GhostPackInfo(self.flags_key)])
        self._masks = build_masks(self.forest, self.stencil, self.flags_key)
        self._flag_snapshot = self._dense_flags()
        self._sweep_masks = self._masks
        self._sweep_flags = self._flag_snapshot
        self._links = None
        self.generation += 1
        for block in self.forest.local_blocks():
            block.data[self.flags_key].touched = False

    frozen = property(lambda self: self._masks is not None)

    @property
    def masks(self):
        if self._masks is None:
            raise ValidationError("freeze() the boundary handling first")
        return self._masks

    @property
    def links(self):
        """The reference's link lists, decoded from the device masks."""
        if self._links is None:
            self._links = decode_links(self.forest, self.stencil, self.masks, self.flags_key)
        return self._links

    def link_count(self, block):
        return sum(len(entry[1]) for per_type in self.links[block.id].values()
                   for entry in per_type)

    def known_mask(self, block):
        reg = block.data[self.flags_key].registry
        return np.bitwise_or.reduce([reg[n] for n in BOUNDARY_FLAGS], initial=np.uint32(0))

    def fluid_mask(self, block):
        return block.data[self.flags_key].registry[FLUID]

    def _dense_flags(self):
        box = RankBox(self.forest)
        return box.gather([b.data[self.flags_key].field.view_nosync for b in box.blocks], 1,
                          np.uint32)

    def sweep_masks(self) -> Masks:
        """The masks of the next sweep.  As in the reference, the links are
        the ones frozen at freeze() (boundary.py:128-131, sweep.py:107-108),
        while the collision follows the CURRENT flags and an unflagged
        interior cell is rejected (sweep.py:124-136): flags edited after
        freeze() keep the frozen link bits and get the fluid bit of their
        current flags (lbm_refresh_fluid_mask).  Only a host access to the
        flag fields triggers the comparison.

        One reference quirk is not reproduced: the reference collides the
        ghost images of a cell with the ghost flags of the last exchange, so
        an edited cell next to a block face or a periodic face collides with
        its stale flag in its neighbours' ghost layer until freeze(); here
        its images follow its current flag."""
        blocks = self.forest.local_blocks()
        if not any(b.data[self.flags_key].touched for b in blocks):
            return self._sweep_masks
        dense = self._dense_flags()
        for b in blocks:
            b.data[self.flags_key].touched = False
        if np.array_equal(dense, self._sweep_flags):
            return self._sweep_masks
        self._sweep_masks = self._refresh(dense)
        self._sweep_flags = dense
        return self._sweep_masks

    def _refresh(self, dense) -> Masks:
        import torch
        frozen = self.masks
        if np.array_equal(dense, self._flag_snapshot):
            return frozen
        box = RankBox(self.forest)
        g = _lib.Grid()
        g.q, g.real_bytes = self.stencil.q, 8
        g.nx, g.ny, g.nz = box.nx, box.ny, box.nz
        g.xoff, g.pitch = 1, box.nx + 2
        g.wrap_x, g.wrap_y = int(box.wrap_x), int(box.wrap_y)
        g.zface_lo, g.zface_hi = box.zface_lo, box.zface_hi
        dev = frozen.cellmask.device
        tf = torch.from_numpy(dense[0].view(np.int32)).to(dev)
        cm = torch.empty_like(frozen.cellmask)
        big = np.iinfo(np.int32).max
        err = torch.tensor([big], dtype=torch.int32, device=dev)
        registry = box.blocks[0].data[self.flags_key].registry
        _lib.call("lbm_refresh_fluid_mask", ctypes.byref(g), _lib.ptr(tf), _flag_bits(registry),
                  _lib.ptr(frozen.cellmask), _lib.ptr(cm), _lib.ptr(err),
                  _lib.stream_ptr(torch.cuda.current_stream(dev)))
        e = int(err.item())
        unflagged = None
        if e != big:
            c = e - 1
            unflagged = (box.lo[0] + c % box.nx, box.lo[1] + (c // box.nx) % box.ny,
                         box.lo[2] + c // (box.nx * box.ny))
        return Masks(cm, frozen.typemask, frozen.counts, unflagged)

    def apply(self, block, src, dst):
        """Write the block's boundary links into dst from the post-collision
        src (boundary.py:154-195): src / dst are ghost-inclusive (z, y, x, q)
        host views.  The per-call host-view entry point of the kernel-slot
        route (collide -> stream_pull -> apply); stream_collide fuses the
        same rule into its sweep kernel.  Runs on the GPU
        (lbm_slot_apply_links) with the frozen link lists."""
        import torch
        from .collision import SRT, kernel_params
        st = self.stencil
        if src.shape != dst.shape or src.ndim != 4 or src.shape[3] != st.q:
            raise ValidationError(f"src / dst must be matching (z, y, x, {st.q}) views")
        Z, Y, X, q = src.shape
        kinds, dirs, cells = [], [], []
        for kind, name in enumerate(_LINK_FLAGS):      # 0 NoSlip, 1 UBB, 2 Pressure
            for i, zs, ys, xs in self.links[block.id][name]:
                kinds.append(np.full(len(zs), kind, dtype=np.int32))
                dirs.append(np.full(len(zs), i, dtype=np.int32))
                cells.append((np.asarray(zs) * Y + np.asarray(ys)) * X + np.asarray(xs))
        if not kinds:
            return
        kp = kernel_params(st, SRT(1.0), None, ubb_velocity=self.ubb_velocity,
                           reference_density=self.reference_density)
        for k in range(q):
            kp.struct.pressure[k] = 2.0 * st.weights[k] * self.pressure_density
        dev = torch.device("cuda", torch.cuda.current_device())
        put = lambda a, dt: torch.from_numpy(np.ascontiguousarray(np.concatenate(a), dtype=dt)
                                              ).to(dev)
        t_kind, t_dir, t_cell = put(kinds, np.int32), put(dirs, np.int32), put(cells, np.int64)
        t_src = torch.from_numpy(np.ascontiguousarray(src, dtype=np.float64)).to(dev)
        t_dst = torch.from_numpy(np.ascontiguousarray(dst, dtype=np.float64)).to(dev)
        _lib.call("lbm_slot_apply_links", q, kp.ref, _lib.ptr(t_kind), _lib.ptr(t_dir),
                  _lib.ptr(t_cell), int(t_cell.numel()), _lib.ptr(t_src), _lib.ptr(t_dst),
                  _lib.stream_ptr(torch.cuda.current_stream(dev)))
        dst[...] = t_dst.cpu().numpy()
