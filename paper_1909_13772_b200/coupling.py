"""Momentum-exchange coupling of the lattice fluid to moving rigid bodies
(SURVEY 8f row f2): body mapping, the moving-boundary sweep, the per-body
hydrodynamic force fold, uncovered-cell reinitialisation and the coupled
step.  Drop-in for pkg/src/blocksim/coupling (mapping.py, sweep.py,
system.py).

`moving_boundary_sweep` is the second caller of the fused sm_100a sweep: the
mapping's coverage becomes a device cell mask (covered cells skip the
collision, fluid cells next to a covered cell get moving-wall links,
`lbm_build_moving_masks`), the wall rule R[x, opp(i)] = G[x, i] -
((6 w_i) rho0)(c_i . u_w) runs inside `lbm_fused_step` with the body
kinematics in a small device table, and the momentum each link hands to its
body is reduced on the device into per-(block, body) force/torque
accumulators - one pass over HBM, as for the plain sweep.  PDFs are bitwise
equal to the reference; forces agree to round-off (the device sums links in
a different order than numpy's pairwise sums).

The mapping (a voxelisation of a few spheres) and the force fold are host
work on small arrays, as in the reference.  Bodies move by whatever the
caller does between steps: the DEM substeps of CoupledSystem (rpd contact
pipeline) are not on the B200 path, so CoupledSystem requires n_sub == 0.
"""
from __future__ import annotations

import ctypes
import hashlib
import logging
import math

import numpy as np
import torch

from . import _lib
from .bodies import handler_of, local_bodies, sync_bodies
from .device import Masks
from .errors import SyncError, TopologyError, ValidationError

log = logging.getLogger("paper_1909_13772_b200.coupling")

# a body covering a ghost-ring cell sits at most half a cell diagonal
# outside the block (mapping.py:27-29)
_MIN_THRESHOLD = math.sqrt(3.0) / 2.0


class ParticleMapping:
    """Body coverage of one forest state (mapping.py:32-54): owner[block_id]
    (nz+2, ny+2, nx+2) int64 covering uid or -1; links[block_id] = link
    groups (uid, direction, zs, ys, xs) in ghost-inclusive coordinates,
    sorted by (uid, direction)."""

    def __init__(self, stencil):
        self.stencil = stencil
        self.owner = {}
        self.links = {}

    def covered_interior(self, block_id):
        return self.owner[block_id][1:-1, 1:-1, 1:-1]

    def link_count(self, block_id) -> int:
        return sum(len(zs) for _, _, zs, _, _ in self.links[block_id])


def _claimable(block, handling):
    if handling is None:
        return None
    ff = block.data[handling.flags_key]
    if ff.g != 1:
        raise ValidationError("body mapping needs exactly one ghost layer")
    return (ff.field.view_nosync[..., 0] & handling.fluid_mask(block)) != 0


def map_bodies(forest, stencil, *, handling=None, key="bodies"):
    """Coverage + boundary links for the current (synchronised) body
    positions (mapping.py:68-155): a cell is covered when its centre lies
    strictly inside a sphere, lower uid first; only static fluid cells may
    be claimed; links are (interior fluid cell, direction into a covered
    cell)."""
    if forest.d != 3:
        raise ValidationError("resolved particle coupling needs a 3D forest")
    if stencil.d != 3:
        raise ValidationError(f"{stencil.name} does not match a 3D forest")
    if forest.cells_per_block is None:
        raise ValidationError("forest has no cells_per_block")
    dx_max = max((max(forest.dx(b.level)) for b in forest.local_blocks()), default=1.0)
    if handler_of(forest, key).contact_threshold < _MIN_THRESHOLD * dx_max:
        raise ValidationError("coverage in the ghost ring needs body ghosts on every block a "
                              "body's cells can touch: register bodies with contact_threshold "
                              f">= sqrt(3)/2 cells ({_MIN_THRESHOLD * dx_max:.4f})")
    if handling is not None and not handling.frozen:
        handling.freeze()
    mapping = ParticleMapping(stencil)
    ncx, ncy, ncz = forest.cells_per_block
    overlap = 0
    for block in forest.local_blocks():
        storage = block.data[key]
        (cx0, cy0, cz0), (dx, dy, dz) = forest.cell_centers(block.id)
        xs = cx0 + dx * (np.arange(ncx + 2) - 1)
        ys = cy0 + dy * (np.arange(ncy + 2) - 1)
        zs = cz0 + dz * (np.arange(ncz + 2) - 1)
        ow = np.full((ncz + 2, ncy + 2, ncx + 2), -1, dtype=np.int64)
        claimable = _claimable(block, handling)
        for uid in sorted(storage.bodies):
            body = storage.bodies[uid]
            r = body.shape.bounding_radius
            p = body.position
            ix0, ix1 = np.searchsorted(xs, (p[0] - r, p[0] + r))
            iy0, iy1 = np.searchsorted(ys, (p[1] - r, p[1] + r))
            iz0, iz1 = np.searchsorted(zs, (p[2] - r, p[2] + r))
            if ix0 == ix1 or iy0 == iy1 or iz0 == iz1:
                continue
            d2 = ((xs[ix0:ix1][None, None, :] - p[0]) ** 2
                  + (ys[iy0:iy1][None, :, None] - p[1]) ** 2
                  + (zs[iz0:iz1][:, None, None] - p[2]) ** 2)
            inside = d2 < r * r
            win = ow[iz0:iz1, iy0:iy1, ix0:ix1]
            overlap += int(np.count_nonzero(inside & (win >= 0)))
            claim = inside & (win == -1)
            if claimable is not None:
                claim &= claimable[iz0:iz1, iy0:iy1, ix0:ix1]
            win[claim] = uid
        mapping.owner[block.id] = ow
        inner = ow[1:-1, 1:-1, 1:-1] == -1
        fluid = inner if claimable is None else (claimable[1:-1, 1:-1, 1:-1] & inner)
        groups = []
        for i in range(1, stencil.q):
            cz, cy, cx = int(stencil.cz[i]), int(stencil.cy[i]), int(stencil.cx[i])
            nb = ow[1 + cz:1 + cz + ncz, 1 + cy:1 + cy + ncy, 1 + cx:1 + cx + ncx]
            hit = fluid & (nb >= 0)
            if not hit.any():
                continue
            hz, hy, hx = np.nonzero(hit)
            uids = nb[hz, hy, hx]
            for uid in np.unique(uids):
                m = uids == uid
                groups.append((int(uid), i, hz[m] + 1, hy[m] + 1, hx[m] + 1))
        groups.sort(key=lambda t: (t[0], t[1]))
        mapping.links[block.id] = groups
    if overlap:
        log.debug("body overlap: %d cells claimed by the lower uid", overlap)
    return mapping


def covered_cell_counts(forest, mapping) -> dict:
    """Collective: global number of covered interior cells per uid."""
    local = {}
    for block in forest.local_blocks():
        inner = mapping.covered_interior(block.id)
        uids, counts = np.unique(inner[inner >= 0], return_counts=True)
        for uid, n in zip(uids, counts):
            local[int(uid)] = local.get(int(uid), 0) + int(n)
    gathered = forest.ctx.all_gather(local)
    total = {}
    for rank in sorted(gathered):
        for uid, n in gathered[rank].items():
            total[uid] = total.get(uid, 0) + n
    return total


# ------------------------------------------------------------- the sweep
class _MovingState:
    """Device arrays of one moving-boundary sweep (kept alive with the
    kernel parameters: later readouts of R_n re-apply the same walls)."""

    def __init__(self, owner, linkmask, bodies, cell0, forces, struct):
        self.owner, self.linkmask, self.bodies, self.cell0, self.forces = (
            owner, linkmask, bodies, cell0, forces)
        self.struct = struct


def _require_unit_spacing(forest):
    for block in forest.local_blocks():
        if forest.dx(block.level) != (1.0, 1.0, 1.0):
            raise ValidationError("coupling runs in lattice units: build the forest with unit "
                                  f"cell spacing, got {forest.dx(block.level)}")


def _block_grid(box, cpb):
    """(nbx, nby, nbz) and, per local block (box order), its linear index
    in the box's block grid."""
    nb = (box.nx // cpb[0], box.ny // cpb[1], box.nz // cpb[2])
    index = []
    for ox, oy, oz in box.offsets:
        bx, by, bz = ox // cpb[0], oy // cpb[1], oz // cpb[2]
        index.append((bz * nb[1] + by) * nb[0] + bx)
    return nb, index


def _combined_masks(lat, static, owner_box):
    """Device cell mask of the current coverage (cached on its content, so a
    coverage that did not change keeps the stored collision valid)."""
    digest = hashlib.blake2b(owner_box.tobytes(), digest_size=16).digest()
    cache = getattr(lat, "_moving_masks", None)
    if cache is not None and cache[0] == (id(static), digest):
        return cache[1], cache[2], cache[3]
    b = lat.box
    dev = lat.device
    owner_t = torch.from_numpy(owner_box).to(dev)
    cm = torch.empty((b.nz, b.ny, b.nx), dtype=torch.int32, device=dev)
    lm = torch.empty((b.nz, b.ny, b.nx), dtype=torch.int32, device=dev)
    n = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.call("lbm_build_moving_masks", lat.gref, _lib.ptr(static.cellmask), _lib.ptr(owner_t),
              _lib.ptr(cm), _lib.ptr(lm), _lib.ptr(n), lat._sp())
    masks = Masks(cm, static.typemask, dict(static.counts), static.unflagged_cell)
    masks.n_moving = int(n.item())
    masks.static = static
    lat._moving_masks = ((id(static), digest), masks, owner_t, lm)
    return masks, owner_t, lm


def moving_boundary_sweep(pdf, model, mapping, *, handling=None, force=None, bodies_key="bodies",
                          reference_density=1.0):
    """Advance the lattice one step against the mapped bodies (collective,
    coupling/sweep.py:45-155).  Returns the momentum-exchange records
    [(root, level, path_bits, uid, owner_rank, force, torque), ...] of this
    rank, one per (block, body with links on it), blocks ascending, uids
    ascending."""
    from .lbm.sweep import _require_uniform
    forest = pdf.forest
    st = pdf.stencil
    _require_uniform(forest)
    _require_unit_spacing(forest)
    if mapping.stencil is not st:
        raise ValidationError("mapping built for a different stencil")
    if handling is not None and handling.stencil is not st:
        raise ValidationError("boundary handling built for a different stencil")
    if handling is None:
        for a in range(forest.d):
            if not forest.periodic[a]:
                raise ValidationError("without boundary handling the domain must be fully periodic")
    elif not handling.frozen:
        handling.freeze()
    if getattr(model, "omega_field", None) is not None:
        raise ValidationError("per-cell rates are not supported with resolved bodies")
    if pdf.g != 1:
        raise ValidationError("stream-collide needs exactly one pdf ghost layer")
    lat = pdf.lattice
    if handling is not None:
        for block in forest.local_blocks():
            if block.data[handling.flags_key].g != pdf.g:
                raise ValidationError("flag and pdf ghost layers differ")
        static = handling.sweep_masks()
        if static.unflagged_cell is not None:
            raise ValidationError(f"unflagged cell {static.unflagged_cell}")
    else:
        static = lat.default_masks()
    box = lat.box
    cpb = forest.cells_per_block
    nb, bindex = _block_grid(box, cpb)

    # body slots: every uid linked on this rank; the table holds, per block,
    # the copy that block's storage sees (periodic images are pre-shifted)
    slot_of = {}
    for block in box.blocks:
        try:
            groups = mapping.links[block.id]
            mapping.owner[block.id]
        except KeyError:
            raise ValidationError(f"mapping does not cover {block.id}") from None
        storage = block.data[bodies_key]
        for uid, *_ in groups:
            if storage.bodies.get(uid) is None:
                raise SyncError(f"mapped body {uid} is not visible on {block.id}")
            slot_of.setdefault(uid, None)
    owner_uids = set()
    for block in box.blocks:
        ow = mapping.owner[block.id]
        owner_uids.update(int(u) for u in np.unique(ow[ow >= 0]))
    uids = sorted(set(slot_of) | owner_uids)
    slot_of = {u: k for k, u in enumerate(uids)}
    n_slots = len(uids)
    n_blocks = nb[0] * nb[1] * nb[2]
    table = np.full((n_blocks, max(n_slots, 1), 9), np.nan)
    cell0 = np.zeros((n_blocks, 3))
    for block, bi in zip(box.blocks, bindex):
        cell0[bi] = forest.cell_centers(block.id)[0]
        storage = block.data[bodies_key]
        for uid, k in slot_of.items():
            body = storage.bodies.get(uid)
            if body is not None:
                table[bi, k, 0:3] = body.position
                table[bi, k, 3:6] = body.linear_velocity
                table[bi, k, 6:9] = body.angular_velocity
    owner_views = []
    for block in box.blocks:
        ow = mapping.owner[block.id]
        lut = np.full(ow.shape, -1, dtype=np.int32)
        for uid, k in slot_of.items():
            lut[ow == uid] = k
        owner_views.append(lut[..., None])
    owner_box = np.ascontiguousarray(box.gather(owner_views, 1, np.int32)[0])

    masks, owner_t, linkmask = _combined_masks(lat, static, owner_box)
    dev = lat.device
    bodies_t = torch.from_numpy(table.reshape(-1, 9)).to(dev)
    cell0_t = torch.from_numpy(cell0).to(dev)
    forces_t = torch.zeros((n_blocks * max(n_slots, 1), 6), dtype=torch.float64, device=dev)
    mv = _lib.Moving()
    mv.owner, mv.linkmask = owner_t.data_ptr(), linkmask.data_ptr()
    mv.bodies, mv.cell0, mv.forces = bodies_t.data_ptr(), cell0_t.data_ptr(), forces_t.data_ptr()
    mv.n_slots = n_slots
    mv.blocks[:] = nb
    mv.block_cells[:] = cpb
    mv.rho0 = float(reference_density)
    kp, key = pdf.params(model, force, handling)
    kp_mv = type(kp)(type(kp.struct).from_buffer_copy(kp.struct), kp.tables)
    kp_mv.struct.moving = ctypes.cast(ctypes.pointer(mv), ctypes.c_void_p).value
    kp_mv.moving = _MovingState(owner_t, linkmask, bodies_t, cell0_t, forces_t, mv)
    if lat.host_changed():
        lat.upload_host()
    lat.step(kp_mv, key + (id(masks),), masks, 1)
    # readouts of R_n re-apply these walls; they must not add forces again
    mv.forces = None

    acc = forces_t.view(n_blocks, max(n_slots, 1), 6).cpu().numpy()
    records = []
    for block, bi in zip(box.blocks, bindex):
        linked = sorted({uid for uid, *_ in mapping.links[block.id]})
        storage = block.data[bodies_key]
        bits = block.id.path_bits(forest.d)
        for uid in linked:
            k = slot_of[uid]
            records.append((block.id.root, block.id.level, bits, uid,
                            storage.bodies[uid].owner_rank, acc[bi, k, 0:3].copy(),
                            acc[bi, k, 3:6].copy()))
    records.sort(key=lambda r: ((r[0], r[1], r[2]), r[3]))
    return records


def reduce_hydrodynamic_forces(forest, records, *, key="bodies"):
    """Collective (coupling/sweep.py:158-215): every local body's
    hydrodynamic force and torque = the fold of this step's records in
    (root, level, path) order; bodies without records end at zero."""
    ctx = forest.ctx
    me = ctx.rank
    for body in local_bodies(forest, key):
        body.hydrodynamic_force = np.zeros(3)
        body.hydrodynamic_torque = np.zeros(3)
    peers = set(forest.neighbor_ranks())
    entries, outgoing = {}, {}
    for root, level, bits, uid, owner, f, t in records:
        if owner == me:
            entries.setdefault(uid, []).append((root, level, bits, f, t))
        elif owner in peers:
            outgoing.setdefault(owner, []).append((uid, root, level, bits, tuple(f), tuple(t)))
        else:
            raise SyncError(f"hydrodynamic force for body {uid} owned by non-neighbor rank {owner}")
    if ctx.n_ranks > 1:
        got = ctx.all_gather(outgoing)
        for src in sorted(got):
            for uid, root, level, bits, f, t in got[src].get(me, []):
                entries.setdefault(uid, []).append((root, level, bits, np.array(f), np.array(t)))
    if not entries:
        return
    owned = {b.uid: b for b in local_bodies(forest, key)}
    for uid in sorted(entries):
        body = owned.get(uid)
        if body is None:
            raise SyncError(f"hydrodynamic force for body {uid}, which is not local here")
        for e in sorted(entries[uid], key=lambda e: (e[0], e[1], e[2])):
            body.hydrodynamic_force += e[3]
            body.hydrodynamic_torque += e[4]


def reinitialize_uncovered(pdf, old_mapping, new_mapping, *, handling=None, bodies_key="bodies",
                           reference_density=1.0):
    """Cells a body released get the equilibrium of the mean density of
    their surviving fluid neighbours (same block) and the departing body's
    surface velocity at the cell centre (system.py:26-100).  Host edit of the
    src slot; the next sweep re-uploads it.  Returns the local count."""
    from .lbm.collision import equilibrium
    forest = pdf.forest
    st = pdf.stencil
    n_total = 0
    for block in forest.local_blocks():
        ow_new = new_mapping.owner[block.id]
        ow_old = old_mapping.owner.get(block.id)
        if ow_old is None or ow_old.shape != ow_new.shape:
            raise ValidationError(f"mappings disagree on {block.id}")
        old_in = ow_old[1:-1, 1:-1, 1:-1]
        new_in = ow_new[1:-1, 1:-1, 1:-1]
        freed = (old_in >= 0) & (new_in == -1)
        if not freed.any():
            continue
        interior = pdf.src(block).interior
        nz, ny, nx = interior.shape[:3]
        fz, fy, fx = np.nonzero(freed)
        n = len(fz)
        n_total += n
        donor = (old_in == -1) & (new_in == -1)
        if handling is not None:
            flags = block.data[handling.flags_key]
            donor &= (flags.field.view_nosync[1:-1, 1:-1, 1:-1, 0] & handling.fluid_mask(block)) != 0
        rho = interior.sum(axis=-1)
        acc = np.zeros(n)
        cnt = np.zeros(n)
        for i in range(1, st.q):
            tz = fz + int(st.cz[i])
            ty = fy + int(st.cy[i])
            tx = fx + int(st.cx[i])
            ok = (tz >= 0) & (tz < nz) & (ty >= 0) & (ty < ny) & (tx >= 0) & (tx < nx)
            ok[ok] = donor[tz[ok], ty[ok], tx[ok]]
            acc[ok] += rho[tz[ok], ty[ok], tx[ok]]
            cnt[ok] += 1.0
        rho_bar = np.where(cnt > 0.0, acc / np.maximum(cnt, 1.0), float(reference_density))
        (cx0, cy0, cz0), _ = forest.cell_centers(block.id)
        px = cx0 + fx.astype(np.float64)
        py = cy0 + fy.astype(np.float64)
        pz = cz0 + fz.astype(np.float64)
        uids = old_in[fz, fy, fx]
        u = np.empty((n, 3))
        storage = block.data[bodies_key]
        for uid in np.unique(uids):
            body = storage.bodies.get(int(uid))
            if body is None:
                raise SyncError(f"body {uid} released cells on {block.id} but is no longer "
                                "visible there")
            m = uids == uid
            rx = px[m] - body.position[0]
            ry = py[m] - body.position[1]
            rz = pz[m] - body.position[2]
            v = body.linear_velocity
            w = body.angular_velocity
            u[m, 0] = v[0] + w[1] * rz - w[2] * ry
            u[m, 1] = v[1] + w[2] * rx - w[0] * rz
            u[m, 2] = v[2] + w[0] * ry - w[1] * rx
        interior[fz, fy, fx, :] = equilibrium(rho_bar, u, st)
    return n_total


class CoupledSystem:
    """One lattice and one body population (system.py:103-196).  step()
    runs map -> moving_boundary_sweep -> reduce_hydrodynamic_forces ->
    sync_bodies -> remap -> reinitialize_uncovered.  Bodies move by the
    caller between steps; the DEM substeps (n_sub > 0) are not on the B200
    path."""

    def __init__(self, pdf, collision_model, contact_model=None, *, handling=None,
                 bodies_key="bodies", n_sub=0, gravity=(0.0, 0.0, 0.0), density_ratio=1.0,
                 fluid_force=None, reference_density=1.0, scheme="VelocityVerlet",
                 broad_method="HashGrids"):
        n_sub = int(n_sub)
        if n_sub < 0:
            raise ValidationError(f"n_sub must be >= 0, got {n_sub}")
        if n_sub > 0:
            raise ValidationError("DEM particle substeps (the rpd contact pipeline) are not on the "
                                  "B200 path: use n_sub=0 and move bodies between steps")
        if not float(density_ratio) > 0.0:
            raise ValidationError(f"density ratio must be positive, got {density_ratio}")
        self.pdf = pdf
        self.collision_model = collision_model
        self.contact_model = contact_model
        self.handling = handling
        self.bodies_key = bodies_key
        self.n_sub = n_sub
        self.gravity = np.asarray(gravity, dtype=np.float64)
        self.density_ratio = float(density_ratio)
        self.fluid_force = fluid_force
        self.reference_density = float(reference_density)
        self.scheme = scheme
        self.broad_method = broad_method
        self.mapping = None
        self.steps = 0

    @property
    def forest(self):
        return self.pdf.forest

    def effective_gravity(self):
        return self.gravity * (1.0 - 1.0 / self.density_ratio)

    def remap(self):
        self.mapping = map_bodies(self.forest, self.pdf.stencil, handling=self.handling,
                                  key=self.bodies_key)
        return self.mapping

    def step(self):
        forest = self.forest
        m_old = self.mapping if self.mapping is not None else self.remap()
        records = moving_boundary_sweep(self.pdf, self.collision_model, m_old,
                                        handling=self.handling, force=self.fluid_force,
                                        bodies_key=self.bodies_key,
                                        reference_density=self.reference_density)
        reduce_hydrodynamic_forces(forest, records, key=self.bodies_key)
        sync_bodies(forest, key=self.bodies_key)
        m_new = map_bodies(forest, self.pdf.stencil, handling=self.handling, key=self.bodies_key)
        uncovered = reinitialize_uncovered(self.pdf, m_old, m_new, handling=self.handling,
                                           bodies_key=self.bodies_key,
                                           reference_density=self.reference_density)
        self.mapping = m_new
        self.steps += 1
        return {"contacts": 0, "uncovered": uncovered}


def coupled_time_step(system: CoupledSystem):
    return system.step()


__all__ = ["CoupledSystem", "ParticleMapping", "coupled_time_step", "covered_cell_counts",
           "map_bodies", "moving_boundary_sweep", "reduce_hydrodynamic_forces",
           "reinitialize_uncovered"]
del TopologyError
