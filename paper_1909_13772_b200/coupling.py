"""Momentum-exchange coupling of the lattice to moving rigid spheres
(SURVEY 8f row f2): body mapping, the moving-boundary sweep, the force
fold, uncovered-cell reinitialisation and the coupled step.  Drop-in for
pkg/src/blocksim/coupling (mapping.py, sweep.py, system.py).

Device side:
* map_bodies voxelises on the GPU (`lbm_map_spheres`): every ghost-inclusive
  cell of every local block tests the block's spheres in uid order with the
  reference's arithmetic (cell centres c0 + h (i - 1), searchsorted window,
  squared distance < r^2), so coverage is bitwise the reference's;
* moving_boundary_sweep is the second caller of the fused sweep: covered
  cells skip the collision, fluid cells next to a covered cell get
  moving-wall links (`lbm_build_moving_masks`), the wall rule
  R[x, opp(i)] = G[x, i] - ((6 w_i) rho0)(c_i . u_w) runs inside
  `lbm_fused_step`, and each link's momentum is reduced on the device into
  per-(block, body) force / torque accumulators - one pass over HBM.
  PDFs are bitwise the reference's; forces agree to round-off (the device
  sums links in another order than numpy).

Host side (small arrays, as in the reference): link lists decoded from the
coverage, the per-body force fold, and the equilibrium refill of released
cells (it needs numpy's own density sums over the host view to stay
bitwise).  Bodies move by whatever the caller does between steps; the DEM
substeps of the reference's CoupledSystem are not on the B200 path
(n_sub must be 0).
"""
from __future__ import annotations

import ctypes
import hashlib
import math

import numpy as np
import torch

from . import _lib
from .bodies import handler_of, local_bodies, sync_bodies
from .device import Masks
from .errors import SyncError, ValidationError

# a body covering a ghost-ring cell sits at most half a cell diagonal
# outside the block (mapping.py:27-29)
_MIN_THRESHOLD = math.sqrt(3.0) / 2.0


class ParticleMapping:
    """Coverage of one body state (mapping.py:32-54): owner[block_id] is the
    ghost-inclusive (nz+2, ny+2, nx+2) int64 covering uid or -1;
    links[block_id] the link groups (uid, direction, zs, ys, xs),
    ghost-inclusive indices, sorted by (uid, direction)."""

    def __init__(self, stencil):
        self.stencil, self.owner, self.links = stencil, {}, {}

    def covered_interior(self, block_id):
        """Interior part of a block's owner array."""
        ow = self.owner[block_id]
        return ow[(slice(1, -1),) * ow.ndim]

    def link_count(self, block_id):
        return sum(len(group[2]) for group in self.links[block_id])


def _check_mapping_args(forest, stencil, key):
    if forest.d != 3 or stencil.d != 3:
        raise ValidationError("resolved particle coupling runs on 3D forests and 3D stencils")
    if forest.cells_per_block is None:
        raise ValidationError("forest has no cells_per_block")
    h_max = max((max(forest.dx(b.level)) for b in forest.local_blocks()), default=1.0)
    if handler_of(forest, key).contact_threshold < _MIN_THRESHOLD * h_max:
        raise ValidationError("coverage in the ghost ring needs body ghosts on every block a "
                              "body's cells can touch: register bodies with contact_threshold "
                              f">= sqrt(3)/2 cells ({_MIN_THRESHOLD * h_max:.4f})")


def _sphere_rows(storage):
    """(x, y, z, r) rows and uids of a block's finite bodies, uid order."""
    bodies = [storage.bodies[u] for u in sorted(storage.bodies)]
    rows = [tuple(b.position) + (b.shape.bounding_radius,) for b in bodies if b.is_finite]
    uids = [b.uid for b in bodies if b.is_finite]
    return rows, uids


def _device_coverage(forest, blocks, key, handling):
    """Ghost-inclusive owner arrays of `blocks` from lbm_map_spheres."""
    dev = torch.device("cuda", torch.cuda.current_device())
    cells = (ctypes.c_int32 * 3)(*forest.cells_per_block)
    frame, first, rows, uids = [], [0], [], []
    for block in blocks:
        c0, h = forest.cell_centers(block.id)
        frame.append(tuple(c0) + tuple(h))
        r, u = _sphere_rows(block.data[key])
        rows += r
        uids += u
        first.append(len(uids))
    t_frame = torch.tensor(frame, dtype=torch.float64, device=dev)
    t_first = torch.tensor(first, dtype=torch.int32, device=dev)
    t_rows = torch.tensor(rows or [(0.0,) * 4], dtype=torch.float64, device=dev)
    t_uids = torch.tensor(uids or [0], dtype=torch.int64, device=dev)
    ncx, ncy, ncz = forest.cells_per_block
    owner = torch.empty((len(blocks), ncz + 2, ncy + 2, ncx + 2), dtype=torch.int64, device=dev)
    t_flags, fluid = None, 0
    if handling is not None:
        stacked = []
        for block in blocks:
            ff = block.data[handling.flags_key]
            if ff.g != 1:
                raise ValidationError("body mapping needs exactly one ghost layer")
            stacked.append(ff.field.view_nosync[..., 0])
        t_flags = torch.from_numpy(np.stack(stacked).view(np.int32)).to(dev)
        fluid = int(handling.fluid_mask(blocks[0]))
    _lib.call("lbm_map_spheres", len(blocks), cells, _lib.ptr(t_frame), _lib.ptr(t_first),
              _lib.ptr(t_rows), _lib.ptr(t_uids), _lib.ptr(t_flags), ctypes.c_uint32(fluid),
              _lib.ptr(owner), _lib.stream_ptr(torch.cuda.current_stream(dev)))
    return owner.cpu().numpy()


def _link_groups(owner, fluid, stencil):
    """Link groups of one block: every (interior fluid cell, direction i)
    whose neighbour x + c_i is covered, grouped by (covering uid, i), cells
    in (z, y, x) order inside a group."""
    nz, ny, nx = fluid.shape
    seen = np.stack([owner[1 + cz:1 + cz + nz, 1 + cy:1 + cy + ny, 1 + cx:1 + cx + nx]
                     for cx, cy, cz in stencil.c[1:]])
    d, z, y, x = np.nonzero(fluid[np.newaxis] & (seen >= 0))
    uid = seen[d, z, y, x]
    order = np.lexsort((d, uid))          # stable: (z, y, x) order kept per group
    d, z, y, x, uid = (a[order] for a in (d, z, y, x, uid))
    cut = np.flatnonzero((np.diff(uid) != 0) | (np.diff(d) != 0)) + 1
    groups = []
    for lo, hi in zip(np.r_[0, cut], np.r_[cut, len(uid)]):
        if hi > lo:
            groups.append((int(uid[lo]), int(d[lo]) + 1, z[lo:hi] + 1, y[lo:hi] + 1,
                           x[lo:hi] + 1))
    return groups


def map_bodies(forest, stencil, *, handling=None, key="bodies"):
    """Coverage + boundary links of the current (synchronised) bodies
    (mapping.py:68-155): a cell is covered by the lowest-uid sphere strictly
    holding its centre, if it is static fluid; links are (interior fluid
    cell, direction into a covered cell)."""
    _check_mapping_args(forest, stencil, key)
    if handling is not None and not handling.frozen:
        handling.freeze()
    mapping = ParticleMapping(stencil)
    blocks = forest.local_blocks()
    if not blocks:
        return mapping
    owners = _device_coverage(forest, blocks, key, handling)
    for block, ow in zip(blocks, owners):
        free = ow[1:-1, 1:-1, 1:-1] == -1
        if handling is not None:
            flags = block.data[handling.flags_key].field.view_nosync[1:-1, 1:-1, 1:-1, 0]
            free &= (flags & handling.fluid_mask(block)) != 0
        mapping.owner[block.id] = ow
        mapping.links[block.id] = _link_groups(ow, free, stencil)
    return mapping


def covered_cell_counts(forest, mapping):
    """Collective: global covered interior cells per uid."""
    mine = {}
    for block in forest.local_blocks():
        inner = mapping.covered_interior(block.id)
        for uid, n in zip(*np.unique(inner[inner >= 0], return_counts=True)):
            mine[int(uid)] = mine.get(int(uid), 0) + int(n)
    total = {}
    for _, part in sorted(forest.ctx.all_gather(mine).items()):
        for uid, n in part.items():
            total[uid] = total.get(uid, 0) + n
    return total


# ------------------------------------------------------------- the sweep
class _MovingState:
    """Device arrays of one moving-boundary sweep, kept alive with the
    kernel parameters (later readouts of R_n re-apply the same walls)."""

    def __init__(self, owner, linkmask, bodies, cell0, forces, struct):
        self.owner, self.linkmask, self.bodies = owner, linkmask, bodies
        self.cell0, self.forces, self.struct = cell0, forces, struct


def _check_sweep_args(pdf, mapping, handling, model):
    from .lbm.sweep import _require_uniform
    forest = pdf.forest
    _require_uniform(forest)
    for block in forest.local_blocks():
        if forest.dx(block.level) != (1.0, 1.0, 1.0):
            raise ValidationError("coupling runs in lattice units: build the forest with unit "
                                  f"cell spacing, got {forest.dx(block.level)}")
    if mapping.stencil is not pdf.stencil:
        raise ValidationError("mapping built for a different stencil")
    if handling is not None and handling.stencil is not pdf.stencil:
        raise ValidationError("boundary handling built for a different stencil")
    if handling is None and not all(forest.periodic[:forest.d]):
        raise ValidationError("without boundary handling the domain must be fully periodic")
    if getattr(model, "omega_field", None) is not None:
        raise ValidationError("per-cell rates are not supported with resolved bodies")
    if pdf.g != 1:
        raise ValidationError("stream-collide needs exactly one pdf ghost layer")


def _static_masks(pdf, handling):
    lat = pdf.lattice
    if handling is None:
        return lat.default_masks()
    if not handling.frozen:
        handling.freeze()
    if any(b.data[handling.flags_key].g != pdf.g for b in pdf.forest.local_blocks()):
        raise ValidationError("flag and pdf ghost layers differ")
    masks = handling.sweep_masks()
    if masks.unflagged_cell is not None:
        raise ValidationError(f"unflagged cell {masks.unflagged_cell}")
    return masks


def _box_blocks(box, cpb):
    """Block grid (nbx, nby, nbz) of the rank box and each local block's
    linear index in it (box order)."""
    nb = (box.nx // cpb[0], box.ny // cpb[1], box.nz // cpb[2])
    return nb, [((oz // cpb[2]) * nb[1] + oy // cpb[1]) * nb[0] + ox // cpb[0]
                for ox, oy, oz in box.offsets]


def _slot_map(box, mapping, bodies_key):
    """Slot of every uid that covers or is linked on this rank (uid order);
    a linked body must be visible on its block."""
    used = set()
    for block in box.blocks:
        if block.id not in mapping.links or block.id not in mapping.owner:
            raise ValidationError(f"mapping does not cover {block.id}")
        storage = block.data[bodies_key]
        for uid, *_ in mapping.links[block.id]:
            if storage.bodies.get(uid) is None:
                raise SyncError(f"mapped body {uid} is not visible on {block.id}")
            used.add(uid)
        ow = mapping.owner[block.id]
        used.update(int(u) for u in np.unique(ow[ow >= 0]))
    return {uid: k for k, uid in enumerate(sorted(used))}


def _kinematics_table(forest, box, bindex, n_blocks, slots, bodies_key):
    """(blocks * slots, 9) position / velocity / spin of the copy each block
    stores (NaN where a block holds none) + (blocks, 3) first-cell centres."""
    table = np.full((n_blocks, max(len(slots), 1), 9), np.nan)
    cell0 = np.zeros((n_blocks, 3))
    for block, bi in zip(box.blocks, bindex):
        cell0[bi] = forest.cell_centers(block.id)[0]
        for uid, k in slots.items():
            body = block.data[bodies_key].bodies.get(uid)
            if body is not None:
                table[bi, k] = np.concatenate([body.position, body.linear_velocity,
                                               body.angular_velocity])
    return table.reshape(-1, 9), cell0


def _slot_owner_box(box, mapping, slots):
    """Ghost-inclusive box of body slots (-1 free) from the per-block owners."""
    ordered = np.array(sorted(slots), dtype=np.int64)     # slot k holds the k-th uid
    views = []
    for block in box.blocks:
        ow = mapping.owner[block.id]
        out = np.full(ow.shape, -1, dtype=np.int32)
        hit = ow >= 0
        out[hit] = np.searchsorted(ordered, ow[hit])
        views.append(out[..., np.newaxis])
    return np.ascontiguousarray(box.gather(views, 1, np.int32)[0])


def _combined_masks(lat, static, owner_box):
    """Device cell mask of the current coverage, cached on its content (an
    unchanged coverage keeps the stored collision valid)."""
    tag = (id(static), hashlib.blake2b(owner_box.tobytes(), digest_size=16).digest())
    hit = getattr(lat, "_moving_masks", None)
    if hit is not None and hit[0] == tag:
        return hit[1], hit[2], hit[3]
    b, dev = lat.box, lat.device
    owner_t = torch.from_numpy(owner_box).to(dev)
    cm = torch.empty((b.nz, b.ny, b.nx), dtype=torch.int32, device=dev)
    lm = torch.empty_like(cm)
    n = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.call("lbm_build_moving_masks", lat.gref, _lib.ptr(static.cellmask), _lib.ptr(owner_t),
              _lib.ptr(cm), _lib.ptr(lm), _lib.ptr(n), lat._sp())
    masks = Masks(cm, static.typemask, dict(static.counts), static.unflagged_cell)
    masks.bits_ok = False   # moving-wall links need the full mask
    masks.n_moving = int(n.item())
    masks.static = static
    lat._moving_masks = (tag, masks, owner_t, lm)
    return masks, owner_t, lm


def moving_boundary_sweep(pdf, model, mapping, *, handling=None, force=None, bodies_key="bodies",
                          reference_density=1.0):
    """One lattice step against the mapped bodies (collective,
    coupling/sweep.py:45-155).  Returns this rank's momentum-exchange
    records [(root, level, path_bits, uid, owner_rank, force, torque)], one
    per (block, body linked on it), blocks then uids ascending."""
    _check_sweep_args(pdf, mapping, handling, model)
    static = _static_masks(pdf, handling)
    forest, lat = pdf.forest, pdf.lattice
    box, cpb = lat.box, forest.cells_per_block
    nb, bindex = _box_blocks(box, cpb)
    n_blocks = nb[0] * nb[1] * nb[2]
    slots = _slot_map(box, mapping, bodies_key)
    table, cell0 = _kinematics_table(forest, box, bindex, n_blocks, slots, bodies_key)
    masks, owner_t, linkmask = _combined_masks(lat, static, _slot_owner_box(box, mapping, slots))

    dev = lat.device
    bodies_t = torch.from_numpy(table).to(dev)
    cell0_t = torch.from_numpy(cell0).to(dev)
    forces_t = torch.zeros((n_blocks * max(len(slots), 1), 6), dtype=torch.float64, device=dev)
    mv = _lib.Moving()
    mv.owner, mv.linkmask = owner_t.data_ptr(), linkmask.data_ptr()
    mv.bodies, mv.cell0, mv.forces = bodies_t.data_ptr(), cell0_t.data_ptr(), forces_t.data_ptr()
    mv.n_slots = len(slots)
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
    mv.forces = None          # readouts of R_n re-apply the walls without forces

    acc = forces_t.view(n_blocks, max(len(slots), 1), 6).cpu().numpy()
    records = []
    for block, bi in zip(box.blocks, bindex):
        storage = block.data[bodies_key]
        bits = block.id.path_bits(forest.d)
        for uid in sorted({g[0] for g in mapping.links[block.id]}):
            k = slots[uid]
            records.append((block.id.root, block.id.level, bits, uid,
                            storage.bodies[uid].owner_rank, acc[bi, k, :3].copy(),
                            acc[bi, k, 3:].copy()))
    records.sort(key=lambda r: ((r[0], r[1], r[2]), r[3]))
    return records


def reduce_hydrodynamic_forces(forest, records, *, key="bodies"):
    """Collective (coupling/sweep.py:158-215): each local body's
    hydrodynamic force / torque become the sum of this step's records for
    it, added in (root, level, path) order; bodies without records end at
    zero.  Records of bodies owned elsewhere go to the owner (a neighbour)."""
    ctx = forest.ctx
    owned = {b.uid: b for b in local_bodies(forest, key)}
    for body in owned.values():
        body.hydrodynamic_force = np.zeros(3)
        body.hydrodynamic_torque = np.zeros(3)
    peers = set(forest.neighbor_ranks())
    parts, mail = {}, {}
    for root, level, bits, uid, owner, f, t in records:
        if owner == ctx.rank:
            parts.setdefault(uid, []).append(((root, level, bits), f, t))
        elif owner in peers:
            mail.setdefault(owner, []).append((uid, (root, level, bits), tuple(f), tuple(t)))
        else:
            raise SyncError(f"hydrodynamic force for body {uid} owned by non-neighbor rank {owner}")
    if ctx.n_ranks > 1:
        for _, posted in sorted(ctx.all_gather(mail).items()):
            for uid, where, f, t in posted.get(ctx.rank, ()):
                parts.setdefault(uid, []).append((where, np.array(f), np.array(t)))
    for uid in sorted(parts):
        if uid not in owned:
            raise SyncError(f"hydrodynamic force for body {uid}, which is not local here")
        body = owned[uid]
        for _, f, t in sorted(parts[uid], key=lambda e: e[0]):
            body.hydrodynamic_force += f
            body.hydrodynamic_torque += t


def _released(old_in, new_in):
    return np.nonzero((old_in >= 0) & (new_in == -1))


def _cell_sums(vals, layout):
    """sum over the q populations of each column of vals (q, n) in the
    order numpy's `interior.sum(axis=-1)` uses on the host view of that
    field layout (system.py:60): "fzyx" (q outermost) reduces element-wise
    in direction order; "zyxf" (q contiguous) runs numpy's pairwise kernel,
    eight partial sums combined as ((0+1)+(2+3))+((4+5)+(6+7)), then the
    remaining directions in order.  Device tensors, fp64, every op rounded."""
    q = vals.shape[0]
    if layout == "fzyx" or q < 8:
        acc = vals[0].clone()
        for k in range(1, q):
            acc = acc + vals[k]
        return acc
    part = [vals[j].clone() for j in range(8)]
    top = q - q % 8
    for i in range(8, top, 8):
        for j in range(8):
            part[j] = part[j] + vals[i + j]
    acc = ((part[0] + part[1]) + (part[2] + part[3])) + ((part[4] + part[5]) + (part[6] + part[7]))
    for k in range(top, q):
        acc = acc + vals[k]
    return acc


def _surface_velocity(storage, block_id, uids, points):
    """v + w x (p - x) of each point's departing body, per component in the
    reference's operation order (host, a few values per released cell)."""
    u = np.empty((len(uids), 3))
    for uid in np.unique(uids):
        body = storage.bodies.get(int(uid))
        if body is None:
            raise SyncError(f"body {uid} released cells on {block_id} but is no longer "
                            "visible there")
        sel = uids == uid
        r = [points[a][sel] - body.position[a] for a in range(3)]
        v, w = body.linear_velocity, body.angular_velocity
        for a in range(3):
            b, c = (a + 1) % 3, (a + 2) % 3
            u[sel, a] = v[a] + w[b] * r[c] - w[c] * r[b]
    return u


def reinitialize_uncovered(pdf, old_mapping, new_mapping, *, handling=None, bodies_key="bodies",
                           reference_density=1.0):
    """Cells a body released get the equilibrium of the mean density of
    their surviving in-block fluid neighbours and the departing body's
    surface velocity at the cell centre (system.py:26-100).  Returns the
    local count.

    On the device: R_n is materialised once as a dense tensor, the donor
    densities are summed in numpy's order for the field's layout
    (_cell_sums), averaged in direction order, the equilibrium of the
    released cells is computed by the equilibrium kernel and written into
    R_n, which becomes the device state (the next sweep collides it).  No
    field crosses PCIe; the host only decides which cells are involved."""
    import torch
    from .lbm.collision import _device
    forest, st, lat = pdf.forest, pdf.stencil, pdf.lattice
    plan = []      # (box offset, block, cells, donor, uids) of blocks with released cells
    for block, off in zip(lat.box.blocks, lat.box.offsets):
        new_ow, old_ow = new_mapping.owner[block.id], old_mapping.owner.get(block.id)
        if old_ow is None or old_ow.shape != new_ow.shape:
            raise ValidationError(f"mappings disagree on {block.id}")
        old_in, new_in = old_ow[1:-1, 1:-1, 1:-1], new_ow[1:-1, 1:-1, 1:-1]
        cells = _released(old_in, new_in)
        if len(cells[0]):
            donor = (old_in == -1) & (new_in == -1)
            if handling is not None:
                flags = block.data[handling.flags_key].field.view_nosync[1:-1, 1:-1, 1:-1, 0]
                donor &= (flags & handling.fluid_mask(block)) != 0
            plan.append((off, block, cells, donor, old_in[cells]))
    if not plan:
        return 0
    if lat.host_changed():
        lat.upload_host()
    full = lat.rform_device()
    dev = _device()
    count = 0
    for (ox, oy, oz), block, (fz, fy, fx), donor, uids in plan:
        n = len(fz)
        count += n
        nz, ny, nx = donor.shape
        acc = torch.zeros(n, dtype=torch.float64, device=dev)
        cnt = np.zeros(n)
        for cx, cy, cz in st.c[1:]:
            tz, ty, tx = fz + cz, fy + cy, fx + cx
            ok = (tz >= 0) & (tz < nz) & (ty >= 0) & (ty < ny) & (tx >= 0) & (tx < nx)
            ok[ok] = donor[tz[ok], ty[ok], tx[ok]]
            if ok.any():
                idx = torch.from_numpy(np.flatnonzero(ok)).to(dev)
                zz, yy, xx = (torch.from_numpy(v[ok] + o + 1).to(dev)
                              for v, o in ((tz, oz), (ty, oy), (tx, ox)))
                acc[idx] = acc[idx] + _cell_sums(full[:, zz, yy, xx], pdf.layout)
                cnt[ok] += 1.0
        cnt_t = torch.from_numpy(cnt).to(dev)
        rho_bar = torch.where(cnt_t > 0.0, acc / torch.clamp(cnt_t, min=1.0),
                              torch.full_like(acc, float(reference_density)))
        c0, _ = forest.cell_centers(block.id)
        points = [c0[a] + (fx, fy, fz)[a].astype(np.float64) for a in range(3)]
        u = torch.from_numpy(_surface_velocity(block.data[bodies_key], block.id, uids,
                                               points)).to(dev)
        feq = torch.empty((n, st.q), dtype=torch.float64, device=dev)
        _lib.call("lbm_equilibrium_cells", st.q, _lib.ptr(rho_bar), _lib.ptr(u), _lib.ptr(feq), n,
                  _lib.stream_ptr(torch.cuda.current_stream(dev)))
        zz, yy, xx = (torch.from_numpy(v + o + 1).to(dev) for v, o in ((fz, oz), (fy, oy), (fx, ox)))
        full[:, zz, yy, xx] = feq.T
    lat.adopt_rform(full)
    return count


class CoupledSystem:
    """A lattice and a body population (system.py:103-196).  step() runs
    map -> moving_boundary_sweep -> reduce_hydrodynamic_forces ->
    sync_bodies -> remap -> reinitialize_uncovered; bodies move by the
    caller between steps (n_sub must be 0: the DEM substeps are not on the
    B200 path)."""

    def __init__(self, pdf, collision_model, contact_model=None, *, handling=None,
                 bodies_key="bodies", n_sub=0, gravity=(0.0, 0.0, 0.0), density_ratio=1.0,
                 fluid_force=None, reference_density=1.0, scheme="VelocityVerlet",
                 broad_method="HashGrids"):
        if int(n_sub) < 0:
            raise ValidationError(f"n_sub must be >= 0, got {n_sub}")
        if int(n_sub) > 0:
            raise ValidationError("DEM particle substeps (the rpd contact pipeline) are not on the "
                                  "B200 path: use n_sub=0 and move bodies between steps")
        if not float(density_ratio) > 0.0:
            raise ValidationError(f"density ratio must be positive, got {density_ratio}")
        self.pdf, self.collision_model, self.contact_model = pdf, collision_model, contact_model
        self.handling, self.bodies_key, self.n_sub = handling, bodies_key, int(n_sub)
        self.gravity = np.asarray(gravity, dtype=np.float64)
        self.density_ratio, self.reference_density = float(density_ratio), float(reference_density)
        self.fluid_force, self.scheme, self.broad_method = fluid_force, scheme, broad_method
        self.mapping, self.steps = None, 0

    forest = property(lambda self: self.pdf.forest)

    def effective_gravity(self):
        """Gravity minus buoyancy per unit body mass."""
        return self.gravity * (1.0 - 1.0 / self.density_ratio)

    def remap(self):
        self.mapping = map_bodies(self.forest, self.pdf.stencil, handling=self.handling,
                                  key=self.bodies_key)
        return self.mapping

    def step(self):
        before = self.mapping if self.mapping is not None else self.remap()
        records = moving_boundary_sweep(self.pdf, self.collision_model, before,
                                        handling=self.handling, force=self.fluid_force,
                                        bodies_key=self.bodies_key,
                                        reference_density=self.reference_density)
        reduce_hydrodynamic_forces(self.forest, records, key=self.bodies_key)
        sync_bodies(self.forest, key=self.bodies_key)
        after = self.remap()
        freed = reinitialize_uncovered(self.pdf, before, after, handling=self.handling,
                                       bodies_key=self.bodies_key,
                                       reference_density=self.reference_density)
        self.steps += 1
        return {"contacts": 0, "uncovered": freed}


def coupled_time_step(system):
    return system.step()


__all__ = ["CoupledSystem", "ParticleMapping", "coupled_time_step", "covered_cell_counts",
           "map_bodies", "moving_boundary_sweep", "reduce_hydrodynamic_forces",
           "reinitialize_uncovered"]
