"""Host-side block fields: storage, flags, slot handlers, ghost rounds.

The drop-in surface of the reference's field package (Field, FlagField,
FieldDataHandler, FlagFieldHandler, GhostPackInfo, exchange_ghosts,
gather_slice, sweep; pkg/src/blocksim/field/core.py:16-175,
handler.py:36-129, ghost.py:202-264, gather.py:10-79) on uniform root
blocks.  What differs is where data lives: the PDF slots of a PdfField are
HBM-resident, and their host arrays here are a lazily allocated *mirror*
(`_mirror` hook): reading raw / view / interior pulls the current R-form
from the device (a stream-only readout kernel), and host writes are
detected and uploaded before the next sweep.  Flags and scalar fields are
plain host data.
"""
from __future__ import annotations

import numpy as np

from .errors import ValidationError

LAYOUTS = ("zyxf", "fzyx")


def _raw_shape(dims, g, layout):
    nx, ny, nz, nf = dims
    cells = (nz + 2 * g, ny + 2 * g, nx + 2 * g)
    return cells + (nf,) if layout == "zyxf" else (nf,) + cells


def _logical(raw, layout):
    """(z, y, x, f) view of a raw array of either layout."""
    return np.moveaxis(raw, 0, 3) if layout == "fzyx" else raw


class Field:
    """nf values per cell of an (nx, ny, nz) block plus g ghost layers,
    stored AoS ("zyxf") or SoA ("fzyx"); every accessor speaks the logical
    (z, y, x, f) order.  lazy=True defers the host allocation until first
    use (a 512^3 D3Q19 mirror is 21 GB and usually never touched)."""

    __slots__ = ("nx", "ny", "nz", "nf", "g", "layout", "dx", "_raw_", "_mirror", "_lazy")

    def __init__(self, dims, ghost_layers=0, layout="zyxf", init=0.0, dtype=np.float64, dx=1.0,
                 lazy=False):
        dims = tuple(int(v) for v in dims)
        if len(dims) != 4 or min(dims) < 1:
            raise ValidationError(f"field dims must be four positive extents, got {dims}")
        if ghost_layers < 0:
            raise ValidationError(f"ghost layers must be >= 0, got {ghost_layers}")
        if layout not in LAYOUTS:
            raise ValidationError(f"layout must be one of {LAYOUTS}, got {layout!r}")
        self.nx, self.ny, self.nz, self.nf = dims
        self.g = int(ghost_layers)
        self.layout = layout
        self.dx = float(dx)
        spec = (_raw_shape(dims, self.g, layout), init, dtype)
        self._lazy = spec if lazy else None
        self._raw_ = None if lazy else np.full(*spec)
        self._mirror = None

    # storage: `_raw` is the array itself, `raw` syncs a device mirror first
    @property
    def _raw(self):
        if self._raw_ is None:
            self._raw_ = np.full(*self._lazy)
        return self._raw_

    @_raw.setter
    def _raw(self, value):
        self._raw_ = value

    @property
    def allocated(self) -> bool:
        return self._raw_ is not None

    def _sync(self):
        if self._mirror is not None:
            self._mirror.host_access()

    @property
    def raw(self):
        self._sync()
        return self._raw

    @raw.setter
    def raw(self, value):
        self._sync()
        self._raw = value

    @property
    def dims(self):
        return (self.nx, self.ny, self.nz, self.nf)

    @property
    def view(self):
        return _logical(self.raw, self.layout)

    @property
    def view_nosync(self):
        """The logical view without a device sync (the mirror's own access)."""
        return _logical(self._raw, self.layout)

    @property
    def interior(self):
        return self.view[self._inner()]

    def _inner(self):
        g = self.g
        return (slice(g, g + self.nz), slice(g, g + self.ny), slice(g, g + self.nx))

    def _at(self, x, y, z, f):
        g = self.g
        inside = all(-g <= c < n + g for c, n in ((x, self.nx), (y, self.ny), (z, self.nz)))
        if not (inside and 0 <= f < self.nf):
            raise IndexError(f"({x}, {y}, {z}, {f}) outside field of dims {self.dims} "
                             f"with {g} ghost layers")
        return (z + g, y + g, x + g, f)

    def get(self, x, y, z, f=0):
        return self.view[self._at(x, y, z, f)]

    def set(self, x, y, z, f, value):
        self.view[self._at(x, y, z, f)] = value

    def _signature(self):
        return (self.dims, self.g, self.layout, self._raw.dtype)

    def swap_data(self, other: "Field") -> None:
        """O(1) storage exchange between two fields of one shape."""
        if self._signature() != other._signature():
            raise ValidationError(f"cannot swap fields {self.dims}/g={self.g}/{self.layout} and "
                                  f"{other.dims}/g={other.g}/{other.layout}")
        self._raw_, other._raw_ = other._raw, self._raw

    def copy(self) -> "Field":
        twin = Field(self.dims, self.g, self.layout, 0.0, self._raw.dtype, self.dx)
        np.copyto(twin._raw, self.raw)
        return twin

    def __repr__(self):
        return f"Field(dims={self.dims}, g={self.g}, layout={self.layout!r}, dtype={self._raw.dtype})"


def make_field(dims, ghost_layers, layout, init=0.0, dtype=np.float64, dx=1.0) -> Field:
    return Field(dims, ghost_layers, layout, init, dtype, dx)


def swap_data(a: Field, b: Field) -> None:
    a.swap_data(b)


# ---------------------------------------------------------------- flags
# A registry maps flag name -> one-bit uint32 mask; bits are handed out in
# registration order (the first name gets bit 0), at most 32 names.  One
# registry (any dict) is shared by every FlagField of a forest slot, so a
# name means the same bit on every block.
def _new_bit(registry: dict, name: str) -> np.uint32:
    if name in registry:
        raise ValidationError(f"flag {name!r} already registered")
    if len(registry) == 32:
        raise ValidationError("flag registry full (32 bits)")
    bit = np.uint32(1) << np.uint32(len(registry))
    registry[name] = bit
    return bit


def _bit_of(registry: dict, name: str) -> np.uint32:
    if name not in registry:
        raise ValidationError(f"flag {name!r} is not registered")
    return registry[name]


class FlagRegistry(dict):
    """A registry with the three operations as methods."""

    def register(self, name: str) -> np.uint32:
        return _new_bit(self, name)

    def bit(self, name: str) -> np.uint32:
        return _bit_of(self, name)

    def union(self, names) -> np.uint32:
        return np.bitwise_or.reduce([_bit_of(self, n) for n in names], initial=np.uint32(0))


class FlagField:
    """uint32 bitmask per cell (core.py:121-169).  Touching view/interior
    sets `touched`, which is how a sweep notices flags edited after
    BoundaryHandling.freeze()."""

    def __init__(self, dims3, ghost_layers=0, registry=None):
        self.field = Field(tuple(dims3) + (1,), ghost_layers, "zyxf", init=0, dtype=np.uint32)
        self.registry = FlagRegistry() if registry is None else registry
        self.touched = True

    @property
    def g(self):
        return self.field.g

    @property
    def view(self):
        self.touched = True
        return self.field.view[..., 0]

    @property
    def interior(self):
        self.touched = True
        return self.field.interior[..., 0]

    def register(self, name: str):
        return _new_bit(self.registry, name)

    def mask(self, name: str):
        return _bit_of(self.registry, name)

    def combined_mask(self, names):
        return np.bitwise_or.reduce([_bit_of(self.registry, n) for n in names],
                                    initial=np.uint32(0))

    def count(self, name: str) -> int:
        """Interior cells carrying the flag."""
        bit = _bit_of(self.registry, name)
        return int(np.count_nonzero(np.bitwise_and(self.field.interior[..., 0], bit)))


def sweep(forest, kernel) -> None:
    """kernel(block) on every local block, ascending ids."""
    for block in forest.local_blocks():
        kernel(block)


# --------------------------------------------------------- slot handlers
class _ArraySlot:
    """Shared snapshot format of the field slots: the raw array itself
    (handler.py:53-63 / 103-110).  Subclasses say which array that is."""

    def _array(self, value):
        raise NotImplementedError   # abstract hook, never called directly

    def serialize(self, forest, block, value, buf) -> None:
        buf.pack_array(self._array(value))

    def deserialize(self, forest, block, buf):
        value = self.create(forest, block)
        incoming = buf.unpack_array()
        target = self._array(value)
        if incoming.shape != target.shape:
            raise ValidationError(f"serialized array {incoming.shape} does not fit the slot's "
                                  f"{target.shape}")
        target[...] = incoming
        return value


def _block_cells(forest):
    if forest.cells_per_block is None:
        raise ValidationError("forest has no cells_per_block")
    return tuple(forest.cells_per_block)


class FieldDataHandler(_ArraySlot):
    """One Field per block (handler.py:36-67)."""

    def __init__(self, nf=1, ghost_layers=1, layout="zyxf", init=0.0, dtype=np.float64,
                 lazy=False):
        self.nf, self.g = int(nf), int(ghost_layers)
        self.layout, self.init, self.dtype, self.lazy = layout, init, dtype, lazy

    def create(self, forest, block) -> Field:
        cells = _block_cells(forest)
        return Field(cells + (self.nf,), self.g, self.layout, self.init, self.dtype,
                     forest.dx(block.level)[0], lazy=self.lazy)

    def _array(self, field):
        return field.raw


class FlagFieldHandler(_ArraySlot):
    """FlagFields of one slot sharing a FlagRegistry (handler.py:83-110)."""

    def __init__(self, ghost_layers=1):
        self.g = int(ghost_layers)
        self.registry = FlagRegistry()

    def register(self, name: str):
        return self.registry.register(name)

    def create(self, forest, block) -> FlagField:
        return FlagField(_block_cells(forest), self.g, self.registry)

    def _array(self, flags):
        return flags.field.raw


# ------------------------------------------------------------ ghost rounds
class GhostPackInfo:
    __slots__ = ("key", "width")

    def __init__(self, key: str, width=None):
        self.key = key
        self.width = width


def _field_of(value):
    return getattr(value, "field", value)


class _Box:
    """Half-open global cell box [lo, hi)."""

    __slots__ = ("lo", "hi")

    def __init__(self, lo, hi):
        self.lo, self.hi = tuple(lo), tuple(hi)

    def moved(self, delta):
        return _Box([l + d for l, d in zip(self.lo, delta)], [h + d for h, d in zip(self.hi, delta)])

    def grown(self, w):
        return _Box([l - w for l in self.lo], [h + w for h in self.hi])

    def clip(self, other):
        lo = [max(a, b) for a, b in zip(self.lo, other.lo)]
        hi = [min(a, b) for a, b in zip(self.hi, other.hi)]
        return _Box(lo, hi) if all(l < h for l, h in zip(lo, hi)) else None

    def window(self, origin, g):
        """(z, y, x) slices of this box in a field whose interior starts at origin."""
        return tuple(slice(self.lo[a] - origin[a] + g, self.hi[a] - origin[a] + g)
                     for a in (2, 1, 0))


def _widths(forest, infos):
    out = []
    for info in infos:
        info = GhostPackInfo(info) if isinstance(info, str) else info
        w = info.width
        if w is None:
            first = next(iter(forest.local_blocks()), None)
            w = None if first is None else _field_of(first.data[info.key]).g
        if w is not None and w < 1:
            raise ValidationError(f"pack width for {info.key!r} must be >= 1")
        out.append((info.key, w))
    return sorted(out)


def exchange_ghosts(forest, infos, *, tag=110) -> None:
    """One collective ghost round on host data (ghost.py:202-264): for each
    distinct neighbour image (block, periodic shift) of a block, the part of
    the block's interior that lies in the image's box grown by the pack
    width lands in the neighbour's ghost cells.  Same-rank images are copied
    directly, the rest travel in one all-gather.  For a PdfField slot this
    is the reference meaning (all q components, R-form; the host mirror is
    synced from the device first)."""
    ctx = forest.ctx
    period = forest.global_cells(0)
    packs = _widths(forest, infos)
    mail = {}
    for block in forest.local_blocks():
        mine = _Box(*forest.cell_box(block.id))
        images = sorted({(rec.block_id, rec.shift): rec.rank for rec in block.neighbors}.items())
        for (nb_id, shift), rank in images:
            wrap = [s * n for s, n in zip(shift, period)]
            image = _Box(*forest.cell_box(nb_id)).moved(wrap)
            for key, w in packs:
                part = image.grown(w).clip(mine)
                if part is None:
                    continue
                field = _field_of(block.data[key])
                payload = np.ascontiguousarray(field.view[part.window(mine.lo, field.g)])
                item = (nb_id, key, part.moved([-v for v in wrap]), payload)
                if rank == ctx.rank:
                    _deliver(forest, item)
                else:
                    mail.setdefault(rank, []).append(item)
    if ctx.n_ranks > 1:
        posted = ctx.all_gather(mail)
        for sender in sorted(posted):
            for item in posted[sender].get(ctx.rank, ()):
                _deliver(forest, item)


def _deliver(forest, item):
    nb_id, key, box, payload = item
    if nb_id not in forest.blocks:
        raise ValidationError(f"ghost data for non-local block {nb_id}")
    field = _field_of(forest.blocks[nb_id].data[key])
    origin = forest.cell_box(nb_id)[0]
    field.view[box.window(origin, field.g)] = payload


def gather_slice(forest, key, lo, hi, level=0):
    """Dense (z, y, x, f) array of the global cell box [lo, hi) on rank 0,
    None elsewhere (gather.py:10-79)."""
    if level != 0:
        raise ValidationError("only level 0 exists on the B200 path")
    want = _Box([int(v) for v in lo], [int(v) for v in hi])
    ext = forest.global_cells(level)
    if not all(0 <= want.lo[a] < want.hi[a] <= ext[a] for a in range(3)):
        raise ValidationError(f"slice box {want.lo}..{want.hi} outside the level-{level} grid {ext}")
    pieces = []
    for block in forest.local_blocks():
        own = _Box(*forest.cell_box(block.id))
        part = own.clip(want)
        if part is not None:
            inner = _field_of(block.data[key]).interior
            pieces.append((part.lo, np.ascontiguousarray(inner[part.window(own.lo, 0)])))
    everyone = forest.ctx.all_gather(pieces)
    arrays = [arr for r in sorted(everyone) for _, arr in everyone[r]]
    if not arrays:
        raise ValidationError("slice box covers no stored blocks")
    if forest.ctx.rank != 0:
        return None
    shape = tuple(want.hi[a] - want.lo[a] for a in (2, 1, 0)) + (arrays[0].shape[3],)
    out = np.zeros(shape, dtype=arrays[0].dtype)
    for r in sorted(everyone):
        for plo, arr in everyone[r]:
            at = _Box(plo, [plo[a] + arr.shape[2 - a] for a in range(3)])
            out[at.window(want.lo, 0)] = arr
    return out
