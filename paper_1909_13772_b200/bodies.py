"""Rigid bodies on the block forest: the data model the moving-boundary sweep
reads (host side; bodies are a few hundred bytes each).

Same names, semantics and snapshot byte format as the reference's body
storage (pkg/src/blocksim/rpd/body.py:63-202, storage.py:24-313,
step.py:123-243): spheres with kinematic state, one BodyStorage per block
holding Local bodies (centre inside the block) and Ghost copies (pre-shifted
periodic images of bodies reaching into the block), collective
`add_sphere`, and `sync_bodies` (ownership migration, then a full ghost
rebuild).  Cross-rank traffic goes through the rank context's all_gather;
every rank applies the same deterministic order, so ghosts are bitwise
copies of their masters as in the reference.

Not here: the DEM contact pipeline (rpd/contact.py, step.time_step) and
half spaces - the B200 path couples the fluid to bodies moved by the caller.
"""
from __future__ import annotations

import math

import numpy as np

from .errors import SyncError, ValidationError

LOCAL = "Local"
GHOST = "Ghost"


def _vec3(value, name):
    v = np.array(value, dtype=np.float64).reshape(-1)
    if v.shape != (3,):
        raise ValidationError(f"{name} must have 3 components, got {value!r}")
    return v


def _unit_quat(q):
    q = np.asarray(q, dtype=np.float64).reshape(-1)
    if q.shape != (4,):
        raise ValidationError(f"quaternion must have 4 components, got {q.shape}")
    n = math.sqrt(float(np.dot(q, q)))
    if not (n > 1e-8 and math.isfinite(n)):
        raise ValidationError("quaternion norm too small to normalize")
    return q / n


class Sphere:
    __slots__ = ("radius",)
    kind = "sphere"

    def __init__(self, radius):
        radius = float(radius)
        if not (radius > 0 and math.isfinite(radius)):
            raise ValidationError(f"sphere radius must be positive, got {radius}")
        self.radius = radius

    @property
    def bounding_radius(self):
        return self.radius

    def inertia(self, mass):
        i = 0.4 * mass * self.radius * self.radius
        return np.diag([i, i, i]), np.diag([1.0 / i] * 3)

    def __repr__(self):
        return f"Sphere({self.radius})"


class RigidBody:
    """Sphere + kinematic state + accumulators (body.py:145-202)."""

    __slots__ = ("uid", "shape", "position", "orientation", "linear_velocity",
                 "angular_velocity", "force", "torque", "mass", "inv_mass", "inertia_body",
                 "inv_inertia_body", "classification", "owner_rank", "hydrodynamic_force",
                 "hydrodynamic_torque", "_accel", "_ang_accel", "_kicked", "_image")

    def __init__(self, uid, shape, position, *, orientation=(1.0, 0.0, 0.0, 0.0),
                 linear_velocity=(0.0, 0.0, 0.0), angular_velocity=(0.0, 0.0, 0.0), mass=None,
                 classification=LOCAL, owner_rank=0):
        if classification not in (LOCAL, GHOST):
            raise ValidationError(f"unknown classification {classification!r}")
        if mass is None or not (float(mass) > 0 and math.isfinite(float(mass))):
            raise ValidationError(f"finite body needs a positive mass, got {mass}")
        self.uid = int(uid)
        self.shape = shape
        self.position = _vec3(position, "position")
        self.orientation = _unit_quat(orientation)
        self.linear_velocity = _vec3(linear_velocity, "linear_velocity")
        self.angular_velocity = _vec3(angular_velocity, "angular_velocity")
        self.force = np.zeros(3)
        self.torque = np.zeros(3)
        self.mass = float(mass)
        self.inv_mass = 1.0 / self.mass
        self.inertia_body, self.inv_inertia_body = shape.inertia(self.mass)
        self.classification = classification
        self.owner_rank = int(owner_rank)
        self.hydrodynamic_force = np.zeros(3)
        self.hydrodynamic_torque = np.zeros(3)
        self._accel = np.zeros(3)
        self._ang_accel = np.zeros(3)
        self._kicked = False
        self._image = (0, 0, 0)

    @property
    def is_finite(self):
        return True

    @property
    def bounding_radius(self):
        return self.shape.bounding_radius

    def velocity_at(self, point):
        return self.linear_velocity + np.cross(self.angular_velocity, point - self.position)

    def __repr__(self):
        return f"RigidBody(uid={self.uid}, {self.shape!r}, {self.classification}@{self.owner_rank})"


class BodyStorage:
    __slots__ = ("bodies",)

    def __init__(self):
        self.bodies = {}

    def add(self, body):
        if body.uid in self.bodies:
            raise ValidationError(f"uid {body.uid} already stored on this block")
        self.bodies[body.uid] = body

    def remove(self, uid):
        return self.bodies.pop(uid)

    def get(self, uid):
        return self.bodies.get(uid)

    def local(self):
        return [self.bodies[u] for u in sorted(self.bodies)
                if self.bodies[u].classification == LOCAL]

    def ghosts(self):
        return [self.bodies[u] for u in sorted(self.bodies)
                if self.bodies[u].classification == GHOST]

    def clear_ghosts(self):
        for uid in [u for u, b in self.bodies.items() if b.classification == GHOST]:
            del self.bodies[uid]

    def __contains__(self, uid):
        return uid in self.bodies

    def __len__(self):
        return len(self.bodies)


def pack_body(buf, body):
    """Snapshot / message record of one body (storage.py:60-76)."""
    buf.pack_int(body.uid)
    buf.pack_int(0)                       # shape kind: sphere
    buf.pack_float(body.shape.radius)
    buf.pack_float(body.mass)
    for v in (body.position, body.orientation, body.linear_velocity, body.angular_velocity,
              body.hydrodynamic_force, body.hydrodynamic_torque, body._accel, body._ang_accel):
        buf.pack_floats(v)
    buf.pack_bool(body._kicked)


def unpack_body(buf, *, classification=LOCAL, owner_rank=0):
    uid = buf.unpack_int()
    if buf.unpack_int() != 0:
        raise ValidationError("only sphere bodies exist on the B200 path")
    shape = Sphere(buf.unpack_float())
    mass = buf.unpack_float()
    body = RigidBody(uid, shape, buf.unpack_floats(), orientation=buf.unpack_floats(),
                     linear_velocity=buf.unpack_floats(), angular_velocity=buf.unpack_floats(),
                     mass=mass, classification=classification, owner_rank=owner_rank)
    body.hydrodynamic_force = np.array(buf.unpack_floats())
    body.hydrodynamic_torque = np.array(buf.unpack_floats())
    body._accel = np.array(buf.unpack_floats())
    body._ang_accel = np.array(buf.unpack_floats())
    body._kicked = buf.unpack_bool()
    return body


def _contains(aabb, p):
    """Half-open block box (lower faces inclusive)."""
    return (aabb[0] <= p[0] < aabb[3] and aabb[1] <= p[1] < aabb[4]
            and aabb[2] <= p[2] < aabb[5])


class BodyStorageHandler:
    """Forest data handler of the body slot (storage.py:94-152); snapshots
    carry Local bodies only (ghosts are rebuilt by sync_bodies)."""

    def __init__(self, contact_threshold=None):
        if contact_threshold is not None and not contact_threshold >= 0:
            raise ValidationError(f"contact threshold must be >= 0, got {contact_threshold}")
        self.fixed_threshold = contact_threshold
        self.auto_threshold = 0.0

    @property
    def contact_threshold(self):
        return self.fixed_threshold if self.fixed_threshold is not None else self.auto_threshold

    def create(self, forest, block):
        return BodyStorage()

    def serialize(self, forest, block, storage, buf):
        bodies = storage.local()
        buf.pack_int(len(bodies))
        for body in bodies:
            pack_body(buf, body)

    def deserialize(self, forest, block, buf):
        storage = BodyStorage()
        for _ in range(buf.unpack_int()):
            storage.add(unpack_body(buf, owner_rank=forest.ctx.rank))
        return storage


def register_bodies(forest, key="bodies", *, contact_threshold=None):
    """Collective: attach a body storage slot to every block."""
    forest.register_data(key, BodyStorageHandler(contact_threshold))
    return key


def handler_of(forest, key):
    h = forest.handlers.get(key)
    if not isinstance(h, BodyStorageHandler):
        raise ValidationError(f"slot {key!r} is not a body storage")
    return h


def _next_uid(forest, key):
    top = -1
    for block in forest.local_blocks():
        for uid in block.data[key].bodies:
            top = max(top, uid)
    return int(forest.ctx.all_reduce((top,), "max")[0]) + 1


def _refresh_threshold(forest, key):
    smallest = math.inf
    for block in forest.local_blocks():
        for body in block.data[key].local():
            smallest = min(smallest, body.bounding_radius)
    smallest = forest.ctx.all_reduce((smallest,), "min")[0]
    handler_of(forest, key).auto_threshold = 0.1 * smallest if math.isfinite(smallest) else 0.0


def add_sphere(forest, position, radius, *, key="bodies", mass=None, density=None,
               velocity=(0.0, 0.0, 0.0), angular_velocity=(0.0, 0.0, 0.0),
               orientation=(1.0, 0.0, 0.0, 0.0)):
    """Collective: store a sphere on the block containing its centre; returns
    its uid (the same on every rank)."""
    if (mass is None) == (density is None):
        raise ValidationError("give exactly one of mass or density")
    shape = Sphere(radius)
    if density is not None:
        if not float(density) > 0:
            raise ValidationError(f"density must be positive, got {density}")
        mass = float(density) * 4.0 / 3.0 * math.pi * shape.radius ** 3
    uid = _next_uid(forest, key)
    mine = 0
    for block in forest.local_blocks():
        if _contains(forest.block_aabb(block.id), position):
            block.data[key].add(RigidBody(uid, shape, position, orientation=orientation,
                                          linear_velocity=velocity,
                                          angular_velocity=angular_velocity, mass=mass,
                                          owner_rank=forest.ctx.rank))
            mine = 1
            break
    if int(forest.ctx.all_reduce((mine,), "sum")[0]) != 1:
        raise ValidationError(f"sphere center {tuple(position)} is outside the domain")
    _refresh_threshold(forest, key)
    return uid


def local_bodies(forest, key="bodies"):
    out = []
    for block in forest.local_blocks():
        out.extend(block.data[key].local())
    out.sort(key=lambda b: b.uid)
    return out


def ghost_bodies(forest, key="bodies"):
    out = []
    for block in forest.local_blocks():
        out.extend(block.data[key].ghosts())
    return out


def find_body(forest, uid, key="bodies"):
    for block in forest.local_blocks():
        body = block.data[key].get(uid)
        if body is not None and body.classification == LOCAL:
            return body
    return None


# ---------------------------------------------------------------- sync
def _extents(forest):
    x0, y0, z0, x1, y1, z1 = forest.domain
    return np.array([x1 - x0, y1 - y0, z1 - z0])


def _images(block):
    """Unique (neighbour block id, shift, rank), deterministic order."""
    seen = {}
    for rec in block.neighbors:
        seen[(rec.block_id, rec.shift)] = rec.rank
    return [(bid, shift, seen[(bid, shift)]) for bid, shift in sorted(seen)]


def _shifted_aabb(forest, bid, shift, ext):
    b = forest.block_aabb(bid)
    return (b[0] + shift[0] * ext[0], b[1] + shift[1] * ext[1], b[2] + shift[2] * ext[2],
            b[3] + shift[0] * ext[0], b[4] + shift[1] * ext[1], b[5] + shift[2] * ext[2])


def _sphere_overlaps(aabb, c, r):
    d2 = 0.0
    for a in range(3):
        if c[a] < aabb[a]:
            d2 += (aabb[a] - c[a]) ** 2
        elif c[a] > aabb[a + 3]:
            d2 += (c[a] - aabb[a + 3]) ** 2
    return d2 <= r * r


def _copy(body, classification, owner):
    out = RigidBody(body.uid, body.shape, body.position.copy(),
                    orientation=body.orientation.copy(),
                    linear_velocity=body.linear_velocity.copy(),
                    angular_velocity=body.angular_velocity.copy(), mass=body.mass,
                    classification=classification, owner_rank=owner)
    return out


def _add_ghost(forest, key, bid, ghost):
    block = forest.blocks.get(bid)
    if block is None:
        raise SyncError(f"ghost of body {ghost.uid} targets non-local block {bid}")
    storage = block.data[key]
    if ghost.uid in storage:
        raise SyncError(f"two images of body {ghost.uid} meet in one block; the domain is too "
                        "small for its size")
    storage.add(ghost)


def sync_bodies(forest, *, key="bodies"):
    """Collective (step.py:136-232): migrate ownership of bodies whose centre
    left their block (periodic wrap by whole domain extents), then rebuild
    every ghost copy (each Local body on every neighbour image its bounding
    sphere + contact threshold touches)."""
    ctx = forest.ctx
    me = ctx.rank
    threshold = handler_of(forest, key).contact_threshold
    ext = _extents(forest)
    for block in forest.local_blocks():
        block.data[key].clear_ghosts()

    outgoing = {}
    for block in forest.local_blocks():
        box = forest.block_aabb(block.id)
        for body in block.data[key].local():
            if _contains(box, body.position):
                continue
            target = None
            for bid, shift, rank in _images(block):
                if _contains(_shifted_aabb(forest, bid, shift, ext), body.position):
                    target = (bid, shift, rank)
                    break
            if target is None:
                raise SyncError(f"body {body.uid} moved farther than one block in one step "
                                "(or left the domain)")
            bid, shift, rank = target
            block.data[key].remove(body.uid)
            if any(shift):
                body.position = body.position - np.array(shift, dtype=np.float64) * ext
            if rank == me:
                body.owner_rank = me
                forest.blocks[bid].data[key].add(body)
            else:
                outgoing.setdefault(rank, []).append((bid, body))
    if ctx.n_ranks > 1:
        got = ctx.all_gather(outgoing)
        for src in sorted(got):
            for bid, body in got[src].get(me, []):
                body.owner_rank = me
                block = forest.blocks.get(bid)
                if block is None:
                    raise SyncError(f"body {body.uid} migrated to non-local block {bid}")
                block.data[key].add(body)

    outgoing = {}
    for block in forest.local_blocks():
        for body in block.data[key].local():
            reach = body.bounding_radius + threshold
            for bid, shift, rank in _images(block):
                if not _sphere_overlaps(_shifted_aabb(forest, bid, shift, ext), body.position,
                                        reach):
                    continue
                if bid == block.id:
                    raise SyncError(f"body {body.uid} overlaps its own periodic image; the "
                                    "domain is too small for its size")
                ghost = _copy(body, GHOST, me)
                if any(shift):
                    ghost.position = ghost.position - np.array(shift, dtype=np.float64) * ext
                ghost._image = tuple(shift)
                if rank == me:
                    _add_ghost(forest, key, bid, ghost)
                else:
                    outgoing.setdefault(rank, []).append((bid, ghost))
    if ctx.n_ranks > 1:
        got = ctx.all_gather(outgoing)
        for src in sorted(got):
            for bid, ghost in got[src].get(me, []):
                _add_ghost(forest, key, bid, ghost)
