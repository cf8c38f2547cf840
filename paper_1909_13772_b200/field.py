"""Ghost-layered block fields (host side) and their collective helpers.

Same API and semantics as the reference's field package
(pkg/src/blocksim/field/core.py:16-175, handler.py:36-129, ghost.py:202-264,
gather.py:10-79).  For the PDF slots of a PdfField these host arrays are a
*mirror* of the HBM-resident state: reading `raw` / `view` / `interior`
pulls the current R-form from the device on demand (a stream-only readout
kernel, no CPU compute), and host writes are detected and re-uploaded before
the next sweep.  Everything else (flags, scalar fields) is host data as in
the reference.
"""
from __future__ import annotations

import numpy as np

from .errors import ValidationError

LAYOUTS = ("zyxf", "fzyx")


class Field:
    """(nx, ny, nz, nf) values plus g ghost layers, layout "zyxf" or "fzyx"."""

    __slots__ = ("nx", "ny", "nz", "nf", "g", "layout", "dx", "_raw_", "_mirror", "_lazy")

    def __init__(self, dims, ghost_layers=0, layout="zyxf", init=0.0, dtype=np.float64, dx=1.0,
                 lazy=False):
        nx, ny, nz, nf = (int(v) for v in dims)
        if min(nx, ny, nz, nf) < 1:
            raise ValidationError(f"field dims must be positive, got {dims}")
        if ghost_layers < 0:
            raise ValidationError(f"ghost layers must be >= 0, got {ghost_layers}")
        if layout not in LAYOUTS:
            raise ValidationError(f"layout must be one of {LAYOUTS}, got {layout!r}")
        self.nx, self.ny, self.nz, self.nf = nx, ny, nz, nf
        self.g = int(ghost_layers)
        self.layout = layout
        self.dx = float(dx)
        g2 = 2 * self.g
        shape = (nz + g2, ny + g2, nx + g2, nf) if layout == "zyxf" else (nf, nz + g2, ny + g2, nx + g2)
        # lazy: the host copy of an HBM-resident field is only allocated
        # when the host actually touches it (a 512^3 D3Q19 field is 21 GB)
        self._lazy = (shape, init, dtype) if lazy else None
        self._raw_ = None if lazy else np.full(shape, init, dtype=dtype)
        self._mirror = None

    @property
    def _raw(self):
        if self._raw_ is None:
            shape, init, dtype = self._lazy
            self._raw_ = np.full(shape, init, dtype=dtype)
        return self._raw_

    @_raw.setter
    def _raw(self, value):
        self._raw_ = value

    @property
    def allocated(self) -> bool:
        return self._raw_ is not None

    # device mirror hook: sync before handing the array out
    @property
    def raw(self):
        if self._mirror is not None:
            self._mirror.host_access()
        return self._raw

    @raw.setter
    def raw(self, value):
        if self._mirror is not None:
            self._mirror.host_access()
        self._raw = value

    @property
    def dims(self):
        return (self.nx, self.ny, self.nz, self.nf)

    @property
    def view(self):
        """Logical (z, y, x, f) array including ghost layers."""
        raw = self.raw
        return raw if self.layout == "zyxf" else np.moveaxis(raw, 0, 3)

    @property
    def interior(self):
        g = self.g
        return self.view[g:g + self.nz, g:g + self.ny, g:g + self.nx]

    @property
    def view_nosync(self):
        """Logical view of the host array without triggering a device sync
        (used by the mirror itself)."""
        raw = self._raw
        return raw if self.layout == "zyxf" else np.moveaxis(raw, 0, 3)

    def get(self, x, y, z, f=0):
        self._check_index(x, y, z, f)
        g = self.g
        return self.view[z + g, y + g, x + g, f]

    def set(self, x, y, z, f, value):
        self._check_index(x, y, z, f)
        g = self.g
        self.view[z + g, y + g, x + g, f] = value

    def _check_index(self, x, y, z, f):
        g = self.g
        if not (-g <= x < self.nx + g and -g <= y < self.ny + g and -g <= z < self.nz + g
                and 0 <= f < self.nf):
            raise IndexError(f"({x}, {y}, {z}, {f}) outside field of dims {self.dims} "
                             f"with {g} ghost layers")

    def swap_data(self, other: "Field") -> None:
        if (self.dims != other.dims or self.g != other.g or self.layout != other.layout
                or self._raw.dtype != other._raw.dtype):
            raise ValidationError(f"cannot swap fields {self.dims}/g={self.g}/{self.layout} and "
                                  f"{other.dims}/g={other.g}/{other.layout}")
        self._raw, other._raw = other._raw, self._raw

    def copy(self) -> "Field":
        out = Field(self.dims, self.g, self.layout, 0.0, self._raw.dtype, self.dx)
        out._raw[...] = self.raw
        return out

    def __repr__(self):
        return f"Field(dims={self.dims}, g={self.g}, layout={self.layout!r}, dtype={self._raw.dtype})"


def make_field(dims, ghost_layers, layout, init=0.0, dtype=np.float64, dx=1.0) -> Field:
    return Field(dims, ghost_layers, layout, init, dtype, dx)


def swap_data(a: Field, b: Field) -> None:
    a.swap_data(b)


class FlagField:
    """uint32 bitmask per cell with a shared name -> bit registry
    (core.py:121-169).  Accessing view/interior marks the field touched so a
    sweep can detect edits made after BoundaryHandling.freeze()."""

    def __init__(self, dims3, ghost_layers=0, registry=None):
        self.field = Field(tuple(dims3) + (1,), ghost_layers, "zyxf", init=0, dtype=np.uint32)
        self.registry = {} if registry is None else registry
        self.touched = True

    @property
    def view(self):
        self.touched = True
        return self.field.view[..., 0]

    @property
    def interior(self):
        self.touched = True
        return self.field.interior[..., 0]

    @property
    def g(self):
        return self.field.g

    def register(self, name: str) -> int:
        if name in self.registry:
            raise ValidationError(f"flag {name!r} already registered")
        if len(self.registry) >= 32:
            raise ValidationError("flag registry full (32 bits)")
        mask = np.uint32(1 << len(self.registry))
        self.registry[name] = mask
        return mask

    def mask(self, name: str) -> int:
        try:
            return self.registry[name]
        except KeyError:
            raise ValidationError(f"flag {name!r} is not registered") from None

    def combined_mask(self, names) -> int:
        out = np.uint32(0)
        for name in names:
            out |= self.mask(name)
        return out

    def count(self, name: str) -> int:
        return int(np.count_nonzero(self.field.interior[..., 0] & self.mask(name)))


def sweep(forest, kernel) -> None:
    """Apply kernel(block) to every local block in ascending id order."""
    for block in forest.local_blocks():
        kernel(block)


class FieldDataHandler:
    """Creates one Field per block (handler.py:36-67)."""

    def __init__(self, nf=1, ghost_layers=1, layout="zyxf", init=0.0, dtype=np.float64,
                 lazy=False):
        self.nf = int(nf)
        self.g = int(ghost_layers)
        self.layout = layout
        self.init = init
        self.dtype = dtype
        self.lazy = lazy

    def create(self, forest, block) -> Field:
        if forest.cells_per_block is None:
            raise ValidationError("forest has no cells_per_block")
        dx = forest.dx(block.level)[0]
        return Field(tuple(forest.cells_per_block) + (self.nf,), self.g, self.layout, self.init,
                     self.dtype, dx, lazy=self.lazy)

    # snapshot slot format: the raw array (handler.py:53-63)
    def serialize(self, forest, block, field, buf) -> None:
        buf.pack_array(field.raw)

    def deserialize(self, forest, block, buf) -> Field:
        field = self.create(forest, block)
        raw = buf.unpack_array()
        if raw.shape != field.raw.shape:
            raise ValidationError(f"serialized field shape {raw.shape} != expected "
                                  f"{field.raw.shape}")
        field.raw[...] = raw
        return field


class FlagFieldHandler:
    """FlagFields sharing one registry (handler.py:83-102)."""

    def __init__(self, ghost_layers=1):
        self.g = int(ghost_layers)
        self.registry = {}

    def register(self, name: str) -> int:
        if name in self.registry:
            raise ValidationError(f"flag {name!r} already registered")
        if len(self.registry) >= 32:
            raise ValidationError("flag registry full (32 bits)")
        mask = np.uint32(1 << len(self.registry))
        self.registry[name] = mask
        return mask

    def create(self, forest, block) -> FlagField:
        if forest.cells_per_block is None:
            raise ValidationError("forest has no cells_per_block")
        return FlagField(forest.cells_per_block, self.g, self.registry)

    def serialize(self, forest, block, flags, buf) -> None:
        buf.pack_array(flags.field.raw)

    def deserialize(self, forest, block, buf) -> FlagField:
        flags = self.create(forest, block)
        raw = buf.unpack_array()
        if raw.shape != flags.field.raw.shape:
            raise ValidationError(f"serialized flag shape {raw.shape} != expected "
                                  f"{flags.field.raw.shape}")
        flags.field.raw[...] = raw
        return flags


# ------------------------------------------------------------ ghost exchange
class GhostPackInfo:
    __slots__ = ("key", "width")

    def __init__(self, key: str, width=None):
        self.key = key
        self.width = width


def _field_of(value):
    return getattr(value, "field", value)


def _isect(a, b):
    lo = tuple(max(a[0][i], b[0][i]) for i in range(3))
    hi = tuple(min(a[1][i], b[1][i]) for i in range(3))
    if any(lo[i] >= hi[i] for i in range(3)):
        return None
    return lo, hi


def _image_box(forest, bid, shift):
    lo, hi = forest.cell_box(bid)
    n = forest.global_cells(0)
    lo = tuple(lo[a] + shift[a] * n[a] for a in range(3))
    hi = tuple(hi[a] + shift[a] * n[a] for a in range(3))
    return lo, hi


def _slice(view, box, origin, g):
    lo, hi = box
    return view[lo[2] - origin[2] + g:hi[2] - origin[2] + g,
                lo[1] - origin[1] + g:hi[1] - origin[1] + g,
                lo[0] - origin[0] + g:hi[0] - origin[0] + g]


def exchange_ghosts(forest, infos, *, tag=110) -> None:
    """One collective ghost round on host data (ghost.py:202-264): for every
    unique neighbour image the receiver's box grown by w, intersected with the
    sender's interior, is copied into the receiver's ghost cells.  Uniform
    level only.  For a PdfField slot this is the reference meaning (all q
    components, R-form): the mirror is synced from the device first."""
    ctx = forest.ctx
    if forest.cells_per_block is None:
        raise ValidationError("forest has no cells_per_block")
    resolved = []
    for info in infos:
        if isinstance(info, str):
            info = GhostPackInfo(info)
        width = info.width
        if width is None:
            for block in forest.local_blocks():
                width = _field_of(block.data[info.key]).g
                break
        if width is not None and width < 1:
            raise ValidationError(f"pack width for {info.key!r} must be >= 1")
        resolved.append((info.key, width))
    resolved.sort()
    outgoing = {}
    for block in forest.local_blocks():
        s_box = forest.cell_box(block.id)
        seen = {}
        for rec in block.neighbors:
            seen[(rec.block_id, rec.shift)] = rec
        for (nb_id, shift) in sorted(seen):
            rec = seen[(nb_id, shift)]
            for key, w in resolved:
                field = _field_of(block.data[key])
                r_lo, r_hi = _image_box(forest, nb_id, shift)
                ghost = (tuple(v - w for v in r_lo), tuple(v + w for v in r_hi))
                o = _isect(ghost, s_box)
                if o is None:
                    continue
                data = np.ascontiguousarray(_slice(field.view, o, s_box[0], field.g))
                back = tuple(-v for v in shift)
                # receiver-local box: the overlap seen from the receiver's frame
                n = forest.global_cells(0)
                r_box = (tuple(o[0][a] - shift[a] * n[a] for a in range(3)),
                         tuple(o[1][a] - shift[a] * n[a] for a in range(3)))
                item = (nb_id, key, r_box, data)
                if rec.rank == ctx.rank:
                    _unpack(forest, item)
                else:
                    outgoing.setdefault(rec.rank, []).append(item)
                del back
    if ctx.n_ranks > 1:
        gathered = ctx.all_gather(outgoing)
        for src in sorted(gathered):
            for item in gathered[src].get(ctx.rank, []):
                _unpack(forest, item)


def _unpack(forest, item):
    nb_id, key, r_box, data = item
    block = forest.blocks.get(nb_id)
    if block is None:
        raise ValidationError(f"ghost data for non-local block {nb_id}")
    field = _field_of(block.data[key])
    lo, _ = forest.cell_box(nb_id)
    _slice(field.view, r_box, lo, field.g)[...] = data


def gather_slice(forest, key, lo, hi, level=0):
    """Dense (z, y, x, f) array of the global cell box [lo, hi) on rank 0
    (gather.py:10-79); None on other ranks."""
    ctx = forest.ctx
    lo = tuple(int(v) for v in lo)
    hi = tuple(int(v) for v in hi)
    if level != 0:
        raise ValidationError("only level 0 exists on the B200 path")
    ext = forest.global_cells(level)
    for a in range(3):
        if not (0 <= lo[a] < hi[a] <= ext[a]):
            raise ValidationError(f"slice box {lo}..{hi} outside the level-{level} grid {ext}")
    contributions = []
    for block in forest.local_blocks():
        blo, bhi = forest.cell_box(block.id)
        olo = tuple(max(blo[a], lo[a]) for a in range(3))
        ohi = tuple(min(bhi[a], hi[a]) for a in range(3))
        if any(olo[a] >= ohi[a] for a in range(3)):
            continue
        view = _field_of(block.data[key]).interior
        sub = view[olo[2] - blo[2]:ohi[2] - blo[2], olo[1] - blo[1]:ohi[1] - blo[1],
                   olo[0] - blo[0]:ohi[0] - blo[0]]
        contributions.append((olo, np.ascontiguousarray(sub)))
    gathered = ctx.all_gather(contributions)
    nf = dtype = None
    for rank in sorted(gathered):
        for _, arr in gathered[rank]:
            nf, dtype = arr.shape[3], arr.dtype
            break
        if nf is not None:
            break
    if nf is None:
        raise ValidationError("slice box covers no stored blocks")
    if ctx.rank != 0:
        return None
    out = np.zeros((hi[2] - lo[2], hi[1] - lo[1], hi[0] - lo[0], nf), dtype=dtype)
    for rank in sorted(gathered):
        for olo, arr in gathered[rank]:
            out[olo[2] - lo[2]:olo[2] - lo[2] + arr.shape[0],
                olo[1] - lo[1]:olo[1] - lo[1] + arr.shape[1],
                olo[0] - lo[0]:olo[0] - lo[0] + arr.shape[2]] = arr
    return out
