"""Rigid spheres on the block forest: the body data the moving-boundary
sweep reads (host side; a body is a few hundred bytes).

Names and semantics follow the reference's rigid-body storage
(pkg/src/blocksim/rpd/body.py:63-202, storage.py:24-313, step.py:123-243):
each block keeps a BodyStorage with its Local bodies (centre inside the
block) and Ghost copies of bodies whose bounding sphere (+ contact
threshold) reaches into it, stored at the position of the periodic image
that block sees.  `add_sphere` is collective; `sync_bodies` migrates bodies
whose centre left their block, then rebuilds every ghost copy.  Cross-rank
traffic is one all_gather per phase, unpacked in rank order, so ghosts are
bitwise copies of their masters.

Not here: the DEM contact pipeline and integrators (rpd/contact.py,
step.time_step) and half spaces: on the B200 path bodies are moved by the
caller between coupled steps.
"""

import math

import numpy as np

from .errors import SyncError, ValidationError

LOCAL = "Local"
GHOST = "Ghost"


def _vector(value, n, what):
    v = np.array(value, dtype=np.float64).reshape(-1)
    if v.size != n:
        raise ValidationError(f"{what} needs {n} components, got {value!r}")
    return v


def _positive(value, what):
    v = float(value)
    if not (v > 0.0 and math.isfinite(v)):
        raise ValidationError(f"{what} must be positive and finite, got {value!r}")
    return v


def _normalised(quat):
    q = _vector(quat, 4, "orientation")
    n = math.sqrt(float(q @ q))
    if not (math.isfinite(n) and n > 1e-8):
        raise ValidationError("orientation quaternion has (near) zero norm")
    return q / n


class Sphere:
    """Sphere shape: radius, bounding radius, body-frame inertia."""

    __slots__ = ("radius",)
    kind = "sphere"

    def __init__(self, radius):
        self.radius = _positive(radius, "sphere radius")

    bounding_radius = property(lambda self: self.radius)

    def inertia(self, mass):
        """(I, I^-1) of a solid sphere: 2/5 m r^2 on the diagonal."""
        moment = 0.4 * mass * self.radius * self.radius
        return np.eye(3) * moment, np.eye(3) * (1.0 / moment)

    def __repr__(self):
        return "Sphere(%r)" % (self.radius,)


# per-body vectors that start at zero, and the kinematic ones given at creation
_ZEROED = ("force", "torque", "hydrodynamic_force", "hydrodynamic_torque", "_accel", "_ang_accel")


class RigidBody:
    """A sphere with kinematic state, accumulators and its storage label
    (Local master or Ghost copy, and the owning rank)."""

    __slots__ = ("uid", "shape", "mass", "inv_mass", "inertia_body", "inv_inertia_body",
                 "classification", "owner_rank", "position", "orientation", "linear_velocity",
                 "angular_velocity", "_kicked", "_image") + _ZEROED

    def __init__(self, uid, shape, position, *, orientation=(1.0, 0.0, 0.0, 0.0),
                 linear_velocity=(0.0, 0.0, 0.0), angular_velocity=(0.0, 0.0, 0.0), mass=None,
                 classification=LOCAL, owner_rank=0):
        if classification not in (LOCAL, GHOST):
            raise ValidationError(f"classification must be {LOCAL!r} or {GHOST!r}, "
                                  f"got {classification!r}")
        if mass is None:
            raise ValidationError("a body needs a mass")
        self.uid, self.shape = int(uid), shape
        self.mass = _positive(mass, "body mass")
        self.inv_mass = 1.0 / self.mass
        self.inertia_body, self.inv_inertia_body = shape.inertia(self.mass)
        self.classification, self.owner_rank = classification, int(owner_rank)
        self.position = _vector(position, 3, "position")
        self.orientation = _normalised(orientation)
        self.linear_velocity = _vector(linear_velocity, 3, "linear_velocity")
        self.angular_velocity = _vector(angular_velocity, 3, "angular_velocity")
        for name in _ZEROED:
            setattr(self, name, np.zeros(3))
        self._kicked = False
        self._image = (0, 0, 0)

    is_finite = property(lambda self: True)
    bounding_radius = property(lambda self: self.shape.bounding_radius)

    def velocity_at(self, point):
        """Rigid-body velocity v + w x (p - x) at a point."""
        return self.linear_velocity + np.cross(self.angular_velocity, point - self.position)

    def replica(self, classification, owner_rank, offset=None):
        """A copy of the kinematic state (a ghost or a migrated master),
        optionally moved by `offset`."""
        out = RigidBody(self.uid, self.shape, self.position if offset is None
                        else self.position - offset, orientation=self.orientation,
                        linear_velocity=self.linear_velocity,
                        angular_velocity=self.angular_velocity, mass=self.mass,
                        classification=classification, owner_rank=owner_rank)
        return out

    def __repr__(self):
        return f"RigidBody(uid={self.uid}, {self.shape!r}, {self.classification}@{self.owner_rank})"


class BodyStorage(dict):
    """The bodies one block stores: a uid -> body dict (`bodies` is the
    reference's name for the same mapping)."""

    bodies = property(lambda self: self)

    def add(self, body):
        if body.uid in self:
            raise ValidationError(f"body {body.uid} is already stored on this block")
        self[body.uid] = body

    remove = dict.pop

    def _labelled(self, label):
        return [b for _, b in sorted(self.items()) if b.classification == label]

    local = lambda self: self._labelled(LOCAL)      # noqa: E731
    ghosts = lambda self: self._labelled(GHOST)     # noqa: E731

    def clear_ghosts(self):
        for uid in [u for u, b in self.items() if b.classification == GHOST]:
            del self[uid]


# ----------------------------------------------------- body records
# A body's record in snapshots and messages (storage.py:60-76 layout): uid,
# shape kind (0 = sphere), radius, mass, eight 3/4-vectors, the kick flag.
_VECTORS = ("position", "orientation", "linear_velocity", "angular_velocity",
            "hydrodynamic_force", "hydrodynamic_torque", "_accel", "_ang_accel")


def pack_body(buf, body):
    buf.pack_int(body.uid)
    buf.pack_int(0)                       # shape kind: sphere
    buf.pack_float(body.shape.radius)
    buf.pack_float(body.mass)
    for name in _VECTORS:
        buf.pack_floats(getattr(body, name))
    buf.pack_bool(bool(body._kicked))


def unpack_body(buf, *, classification=LOCAL, owner_rank=0):
    uid, kind = buf.unpack_int(), buf.unpack_int()
    if kind != 0:
        raise ValidationError("only sphere bodies exist on the B200 path")
    radius, mass = buf.unpack_float(), buf.unpack_float()
    vec = {name: np.array(buf.unpack_floats()) for name in _VECTORS}
    body = RigidBody(uid, Sphere(radius), vec["position"], orientation=vec["orientation"],
                     linear_velocity=vec["linear_velocity"],
                     angular_velocity=vec["angular_velocity"], mass=mass,
                     classification=classification, owner_rank=owner_rank)
    for name in _VECTORS[4:]:
        setattr(body, name, vec[name])
    body._kicked = buf.unpack_bool()
    return body


class BodyStorageHandler:
    """Forest slot handler: one BodyStorage per block; images carry the
    Local bodies only (sync_bodies rebuilds ghosts)."""

    def __init__(self, contact_threshold=None):
        if not (contact_threshold is None or contact_threshold >= 0):
            raise ValidationError(f"contact threshold must be >= 0, got {contact_threshold}")
        self.fixed_threshold, self.auto_threshold = contact_threshold, 0.0

    @property
    def contact_threshold(self):
        return self.auto_threshold if self.fixed_threshold is None else self.fixed_threshold

    @staticmethod
    def create(forest, block):
        return BodyStorage()

    @staticmethod
    def serialize(forest, block, storage, buf):
        masters = storage.local()
        buf.pack_int(len(masters))
        for body in masters:
            pack_body(buf, body)

    @staticmethod
    def deserialize(forest, block, buf):
        count = buf.unpack_int()
        bodies = [unpack_body(buf, owner_rank=forest.ctx.rank) for _ in range(count)]
        out = BodyStorage()
        for body in bodies:
            out.add(body)
        return out


def register_bodies(forest, key="bodies", *, contact_threshold=None):
    """Collective: a body storage slot on every block."""
    forest.register_data(key, BodyStorageHandler(contact_threshold))
    return key


def handler_of(forest, key):
    handler = forest.handlers.get(key)
    if isinstance(handler, BodyStorageHandler):
        return handler
    raise ValidationError(f"slot {key!r} is not a body storage")


def _storages(forest, key):
    """(block, its BodyStorage) for every block of this rank."""
    return [(blk, blk.data[key]) for blk in forest.local_blocks()]


def _stored(forest, key, label=None):
    for blk, store in _storages(forest, key):
        for _, body in sorted(store.bodies.items()):
            if label is None or body.classification == label:
                yield blk, body


def _inside(box, p):
    """Half-open AABB membership (lower faces belong to the box)."""
    return all(box[a] <= p[a] < box[a + 3] for a in range(3))


def add_sphere(forest, position, radius, *, key="bodies", mass=None, density=None,
               velocity=(0.0, 0.0, 0.0), angular_velocity=(0.0, 0.0, 0.0),
               orientation=(1.0, 0.0, 0.0, 0.0)):
    """Collective: a new sphere, stored on the block whose box holds its
    centre; the uid (one past the largest in use) is returned on every rank."""
    if (mass is None) == (density is None):
        raise ValidationError("give exactly one of mass or density")
    shape = Sphere(radius)
    if density is not None:
        mass = _positive(density, "density") * 4.0 / 3.0 * math.pi * shape.radius ** 3
    top = max((uid for _, store in _storages(forest, key) for uid in store.bodies), default=-1)
    uid = int(forest.ctx.all_reduce((top,), "max")[0]) + 1
    home = next((b for b in forest.local_blocks() if _inside(forest.block_aabb(b.id), position)),
                None)
    if home is not None:
        home.data[key].add(RigidBody(uid, shape, position, orientation=orientation,
                                     linear_velocity=velocity, angular_velocity=angular_velocity,
                                     mass=mass, owner_rank=forest.ctx.rank))
    if int(forest.ctx.all_reduce((int(home is not None),), "sum")[0]) != 1:
        raise ValidationError(f"sphere center {tuple(position)} is outside the domain")
    smallest = min((b.bounding_radius for _, b in _stored(forest, key, LOCAL)), default=math.inf)
    smallest = forest.ctx.all_reduce((smallest,), "min")[0]
    handler_of(forest, key).auto_threshold = 0.1 * smallest if math.isfinite(smallest) else 0.0
    return uid


def local_bodies(forest, key="bodies"):
    return sorted((b for _, b in _stored(forest, key, LOCAL)), key=lambda b: b.uid)


def ghost_bodies(forest, key="bodies"):
    return [b for _, b in _stored(forest, key, GHOST)]


def find_body(forest, uid, key="bodies"):
    return next((b for _, b in _stored(forest, key, LOCAL) if b.uid == uid), None)


# ---------------------------------------------------------------- sync
class _Mailbox:
    """Items for blocks of this rank are applied at once, the rest travel
    in one all_gather and are applied in sender-rank order."""

    def __init__(self, ctx, apply):
        self.ctx, self.apply, self.out = ctx, apply, {}

    def post(self, rank, item):
        if rank == self.ctx.rank:
            self.apply(item)
        else:
            self.out.setdefault(rank, []).append(item)

    def flush(self):
        if self.ctx.n_ranks > 1:
            everyone = self.ctx.all_gather(self.out)
            for sender in sorted(everyone):
                for item in everyone[sender].get(self.ctx.rank, ()):
                    self.apply(item)
        self.out = {}


def _neighbour_images(forest, block, extent):
    """(block id, shift, rank, shifted AABB) of each distinct neighbour
    image, in (id, shift) order."""
    seen = {(r.block_id, r.shift): r.rank for r in block.neighbors}
    out = []
    for (bid, shift), rank in sorted(seen.items()):
        move = np.asarray(shift, dtype=np.float64) * extent
        box = np.asarray(forest.block_aabb(bid), dtype=np.float64) + np.concatenate([move, move])
        out.append((bid, shift, rank, box))
    return out


def _gap2(box, c):
    """Squared distance from point c to an AABB (0 inside)."""
    d2 = 0.0
    for a in range(3):
        gap = max(box[a] - c[a], 0.0, c[a] - box[a + 3])
        if gap > 0.0:
            d2 += gap * gap
    return d2


def sync_bodies(forest, *, key="bodies"):
    """Collective: (1) a body whose centre left its block moves to the
    neighbour image that now holds it (position wrapped by whole domain
    extents); (2) every ghost is dropped and rebuilt from the Local bodies
    whose bounding sphere + contact threshold reaches a neighbour image."""
    ctx = forest.ctx
    lo, hi = np.asarray(forest.domain[:3]), np.asarray(forest.domain[3:])
    extent = hi - lo
    reach_extra = handler_of(forest, key).contact_threshold
    for _, store in _storages(forest, key):
        store.clear_ghosts()

    def adopt(item):
        bid, body = item
        if bid not in forest.blocks:
            raise SyncError(f"body {body.uid} migrated to non-local block {bid}")
        body.owner_rank = ctx.rank
        forest.blocks[bid].data[key].add(body)

    movers = _Mailbox(ctx, adopt)
    for blk, store in _storages(forest, key):
        own_box = forest.block_aabb(blk.id)
        for body in store.local():
            if _inside(own_box, body.position):
                continue
            dest = next(((bid, shift, rank) for bid, shift, rank, box in
                         _neighbour_images(forest, blk, extent)
                         if _inside(box, body.position)), None)
            if dest is None:
                raise SyncError(f"body {body.uid} moved farther than one block in one step "
                                "(or left the domain)")
            bid, shift, rank = dest
            store.remove(body.uid)
            if any(shift):
                body.position = body.position - np.asarray(shift, dtype=np.float64) * extent
            movers.post(rank, (bid, body))
    movers.flush()

    def place(item):
        bid, ghost = item
        if bid not in forest.blocks:
            raise SyncError(f"ghost of body {ghost.uid} targets non-local block {bid}")
        storage = forest.blocks[bid].data[key]
        if ghost.uid in storage:
            raise SyncError(f"two images of body {ghost.uid} meet in one block; the domain is "
                            "too small for its size")
        storage.add(ghost)

    ghosts = _Mailbox(ctx, place)
    for blk, store in _storages(forest, key):
        images = _neighbour_images(forest, blk, extent)
        for body in store.local():
            reach = body.bounding_radius + reach_extra
            for bid, shift, rank, box in images:
                if _gap2(box, body.position) > reach * reach:
                    continue
                if bid == blk.id:
                    raise SyncError(f"body {body.uid} overlaps its own periodic image; the "
                                    "domain is too small for its size")
                offset = np.asarray(shift, dtype=np.float64) * extent if any(shift) else None
                ghost = body.replica(GHOST, ctx.rank, offset)
                ghost._image = tuple(shift)
                ghosts.post(rank, (bid, ghost))
    ghosts.flush()
