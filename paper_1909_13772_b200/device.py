"""HBM-resident lattice state behind a PdfField.

`RankBox` maps this rank's blocks onto one contiguous device box (a z-slab
when several ranks share the domain).  `DeviceLattice`
owns the two PDF buffers in the z-q-y-x layout of include/lbm_b200.h and runs
the per-step schedule:

* state is the post-collision G-form G_n = C(R_n); the reference state R_n
  (what `pdf.src(block)` holds after n sweeps, lbm/sweep.py:93-151) is
  recovered on demand as S(G_{n-1}) from the swapped-out buffer;
* P = 1: one fused launch per step (periodic z wraps in the kernel);
* P > 1: boundary planes first on a high-priority stream, the interior
  planes concurrently on the caller's stream.  The boundary kernel stores
  its crossing directions straight into the z-neighbours' ghost planes
  (halo.PeerHalo: peer HBM over NVLink, ordered by stream flags); where the
  ranks cannot map each other they go out by NCCL send/recv of the
  contiguous runs (no pack kernel).

Host<->device traffic happens only on upload (host R-form written by the
user), readout (host arrays touched) and mask builds; never inside the step.
"""
from __future__ import annotations

import ctypes
import gc
import os

import numpy as np
import torch

from . import _lib
from .errors import BackendError, ValidationError


def _round_up(v, m):
    return (v + m - 1) // m * m


def hbm_empty(n, dtype, device) -> torch.Tensor:
    """A large HBM buffer.  Lattices of dropped PdfFields sit in reference
    cycles (forest -> slot handler -> PdfField -> lattice -> forest, as in
    the reference's object graph) that only the cyclic GC frees, and the GC
    is not driven by device memory: on an allocation failure collect them
    and retry once before reporting out of memory."""
    try:
        return torch.empty(n, dtype=dtype, device=device)
    except torch.OutOfMemoryError:
        gc.collect()
        torch.cuda.empty_cache()
        return torch.empty(n, dtype=dtype, device=device)


class RankBox:
    """This rank's blocks as one box in global cell coordinates."""

    def __init__(self, forest):
        if forest.cells_per_block is None:
            raise ValidationError("forest has no cells_per_block")
        ctx = forest.ctx
        blocks = forest.local_blocks()
        if not blocks:
            raise ValidationError(f"rank {ctx.rank} owns no block; use at least as many "
                                  "blocks as ranks")
        boxes = [forest.cell_box(b.id) for b in blocks]
        lo = tuple(min(b[0][a] for b in boxes) for a in range(3))
        hi = tuple(max(b[1][a] for b in boxes) for a in range(3))
        vol = (hi[0] - lo[0]) * (hi[1] - lo[1]) * (hi[2] - lo[2])
        if vol != sum((b[1][0] - b[0][0]) * (b[1][1] - b[0][1]) * (b[1][2] - b[0][2]) for b in boxes):
            raise ValidationError("the blocks of a rank must form one box on the B200 path "
                                  "(use root_dims = (1, 1, P) z-slabs)")
        N = forest.global_cells(0)
        self.global_cells = N
        if ctx.n_ranks > 1 and (lo[0] != 0 or lo[1] != 0 or hi[0] != N[0] or hi[1] != N[1]):
            raise ValidationError("multi-rank B200 runs partition the domain in z-slabs: every "
                                  "rank's box must span the full x and y extent")
        self.lo, self.hi = lo, hi
        self.nx, self.ny, self.nz = (hi[a] - lo[a] for a in range(3))
        self.blocks = blocks
        self.offsets = [tuple(b[0][a] - lo[a] for a in range(3)) for b in boxes]
        per = forest.periodic
        self.wrap_x = bool(per[0]) and lo[0] == 0 and hi[0] == N[0]
        self.wrap_y = bool(per[1]) and lo[1] == 0 and hi[1] == N[1]
        if (per[0] and not self.wrap_x) or (per[1] and not self.wrap_y):
            raise ValidationError("periodic x/y must be owned by one rank (z-slab partition)")
        self.lo_peer = self.hi_peer = None
        # low z face
        if lo[2] > 0:
            self.zface_lo, self.lo_peer = _lib.ZFACE_HALO, forest.owner_of_cell((0, 0, lo[2] - 1))
        elif per[2]:
            peer = forest.owner_of_cell((0, 0, N[2] - 1))
            if peer == ctx.rank:
                self.zface_lo = _lib.ZFACE_WRAP
            else:
                self.zface_lo, self.lo_peer = _lib.ZFACE_HALO, peer
        else:
            self.zface_lo = _lib.ZFACE_GHOST
        # high z face
        if hi[2] < N[2]:
            self.zface_hi, self.hi_peer = _lib.ZFACE_HALO, forest.owner_of_cell((0, 0, hi[2]))
        elif per[2]:
            peer = forest.owner_of_cell((0, 0, 0))
            if peer == ctx.rank:
                self.zface_hi = _lib.ZFACE_WRAP
            else:
                self.zface_hi, self.hi_peer = _lib.ZFACE_HALO, peer
        else:
            self.zface_hi = _lib.ZFACE_GHOST
        if (self.zface_lo == _lib.ZFACE_WRAP) != (self.zface_hi == _lib.ZFACE_WRAP):
            raise ValidationError("periodic z wrap must be owned entirely by one rank")

    @property
    def cells(self) -> int:
        return self.nx * self.ny * self.nz

    # ------------------------------------------------- host box assembly
    def gather(self, views, nf, dtype):
        """Ghost-inclusive box (nf, Z, Y, X) from per-block logical views
        (z, y, x, f) with one ghost layer: block ghost layers first (they
        provide the box's outer ghost shell), then every interior."""
        out = np.zeros((nf, self.nz + 2, self.ny + 2, self.nx + 2), dtype=dtype)
        for v, (ox, oy, oz) in zip(views, self.offsets):
            sub = out[:, oz:oz + v.shape[0], oy:oy + v.shape[1], ox:ox + v.shape[2]]
            sub[...] = np.moveaxis(v, 3, 0)
        for v, (ox, oy, oz) in zip(views, self.offsets):
            n0, n1, n2 = v.shape[0] - 2, v.shape[1] - 2, v.shape[2] - 2
            out[:, 1 + oz:1 + oz + n0, 1 + oy:1 + oy + n1, 1 + ox:1 + ox + n2] = \
                np.moveaxis(v[1:-1, 1:-1, 1:-1], 3, 0)
        return out

    def scatter_interior(self, dense, views):
        """dense (nf, nz, ny, nx) -> block interiors of logical views."""
        for v, (ox, oy, oz) in zip(views, self.offsets):
            n0, n1, n2 = v.shape[0] - 2, v.shape[1] - 2, v.shape[2] - 2
            v[1:-1, 1:-1, 1:-1] = np.moveaxis(dense[:, oz:oz + n0, oy:oy + n1, ox:ox + n2], 0, 3)

    def scatter_full(self, dense_g, views):
        """dense ghost-inclusive (nf, Z, Y, X) -> block views incl. ghosts."""
        for v, (ox, oy, oz) in zip(views, self.offsets):
            v[...] = np.moveaxis(dense_g[:, oz:oz + v.shape[0], oy:oy + v.shape[1],
                                         ox:ox + v.shape[2]], 0, 3)


def linkbits_enabled() -> bool:
    """The link-bit map is opt-in (LBM_B200_LINKBITS=1): measured on B200 it
    moves 3.75 B/cell less but runs config 4 fp32 3.6 % and fp64 1.9 % slower
    than the prefetched cell mask (profiles/ab_variants_r2.md §4)."""
    return os.environ.get("LBM_B200_LINKBITS", "0") == "1"


def job_schedule(nz, steps, chunk=None):
    """Upload chunks and wavefront frontiers of DeviceLattice.run_job.

    `chunk` = (planes, ramp, tail): chunks of `planes` z-planes, preceded by
    the smaller `ramp` chunks (the first sweeps start after a short upload
    instead of a whole chunk); once every plane is filled the frontier keeps
    advancing `tail` planes at a time past nz, so the last steps, moments
    and downloads also move in small pieces (0: the last chunk's steps run
    to the end in one launch each).  An int is (planes, (), 0); None the
    defaults (32, (4, 4, 8, 16), max(4, ceil(steps / 2))), or
    LBM_B200_JOB_CHUNK / _RAMP / _TAIL.
    Returns ([(z0, z1)], [frontier]); frontiers past nz are tail steps."""
    if chunk is None:
        planes = int(os.environ.get("LBM_B200_JOB_CHUNK", "32"))
        ramp = tuple(int(v) for v in os.environ.get("LBM_B200_JOB_RAMP", "4,4,8,16").split(",")
                     if v.strip())
        # two or three tail frontiers (each issues up to `steps` launches;
        # measured at 512^3 K = 20 and 128^3 K = 100, profiles/r2/e2e_tail.log)
        tail = int(os.environ.get("LBM_B200_JOB_TAIL", str(max(4, -(-steps // 2)))))
    elif isinstance(chunk, int):
        planes, ramp, tail = chunk, (), 0
    else:
        planes, ramp, tail = chunk
    planes = max(1, int(planes))
    bounds, z = [], 0
    for size in tuple(ramp) + (planes,) * nz:
        if z >= nz:
            break
        bounds.append((z, min(z + max(1, int(size)), nz)))
        z = bounds[-1][1]
    fronts = [z1 for _, z1 in bounds]
    if tail > 0:
        f = nz
        while f - steps < nz:
            f += int(tail)
            fronts.append(f)
    return bounds, fronts


def job_plan(nz, steps, chunk=None):
    """The ordered launches of DeviceLattice.run_job: ("fill", chunk index,
    z0, z1), ("step", n, z0, z1) - sweep n (G_{n-1} -> G_n) over planes
    [z0, z1) - and ("moments", z0, z1) - rho / u of R_K = S(G_{K-1}).

    G_n lives in buffer n % 2 (relative), so step n at plane p reads G_{n-1}
    on p - 1 .. p + 1 and overwrites G_{n-2} on p, which step n - 1 still
    needs up to p + 1: step n may finish the planes below done[n-1] - 1 (all
    of them once step n - 1 is complete).  The moments read G_{K-1} like a
    step K would.  Past the last chunk, tail frontiers cap step n at
    front - n.  tests/test_abi_host.py checks these rules for many
    schedules; tests/test_pipeline.py that the job is bitwise the call
    sequence on the GPU."""
    bounds, fronts = job_schedule(nz, steps, chunk)
    capped = fronts[-1] > nz
    done = [0] * (steps + 1)
    mdone, ci, plan = 0, 0, []

    def frontier(prev, n, front):
        lim = nz if prev == nz else prev - 1
        return min(lim, front - n) if capped and front - n < nz else lim

    for front in fronts:
        if ci < len(bounds) and bounds[ci][1] == front:
            plan.append(("fill", ci) + bounds[ci])
            done[0] = bounds[ci][1]
            ci += 1
        for n in range(1, steps + 1):
            lim = frontier(done[n - 1], n, front)
            if lim > done[n]:
                plan.append(("step", n, done[n], lim))
                done[n] = lim
        lim = frontier(done[steps - 1], steps, front)
        if lim > mdone:
            plan.append(("moments", mdone, lim))
            mdone = lim
    return plan


class Masks:
    """Device cell mask + link-type mask for one (box, stencil, flags) state."""

    def __init__(self, cellmask, typemask, counts, unflagged_cell=None, all_fluid=False):
        self.cellmask = cellmask      # int32 (nz, ny, nx)
        self.typemask = typemask      # int32 (nz, ny, nx, 2)
        self.counts = counts          # dict NoSlip/UBB/Pressure -> links on this rank
        self.unflagged_cell = unflagged_cell
        self.all_fluid = all_fluid    # the fused step may skip the mask (NULL)
        self.bits_ok = True           # worth deriving a link-bit map (not moving-wall masks)
        self._linkbits = None         # uint64 map, or False when the derivation fails

    def linkbits(self, lat):
        """Device pointer of the link-bit map that reproduces this cell mask
        (lbm_build_linkbits: 1 bit per cell instead of 4 bytes for the fused
        sweep), or None where it does not apply: no mask, typed (UBB /
        Pressure) links, moving walls, or a mask the bits cannot express
        (flags edited after freeze()).  Built once per mask, checked on the
        device on every cell (one sync, at setup)."""
        if self.all_fluid or self.typed or not self.bits_ok or not linkbits_enabled():
            return None
        if self._linkbits is None:
            n = int(_lib.load().lbm_linkbits_words(lat.gref))
            bits = torch.empty(max(n, 1), dtype=torch.int64, device=self.cellmask.device)
            big = np.iinfo(np.int32).max
            mismatch = torch.full((1,), big, dtype=torch.int32, device=self.cellmask.device)
            _lib.call("lbm_build_linkbits", lat.gref, _lib.ptr(self.cellmask), _lib.ptr(bits),
                      _lib.ptr(mismatch), lat._sp())
            self._linkbits = bits if int(mismatch.item()) == big else False
        return _lib.ptr(self._linkbits) if self._linkbits is not False else None

    @property
    def typed(self) -> bool:
        """Some cell has a UBB or Pressure link (the fused step needs the
        typemask; without any it gets NULL and the corrections compile out)."""
        return bool(self.counts.get("UBB", 0) or self.counts.get("Pressure", 0))


def all_fluid_masks(box: RankBox, device) -> Masks:
    cm = torch.full((box.nz, box.ny, box.nx), _lib.MASK_FLUID, dtype=torch.int32, device=device)
    tm = torch.zeros((box.nz, box.ny, box.nx, 2), dtype=torch.int32, device=device)
    return Masks(cm, tm, {"NoSlip": 0, "UBB": 0, "Pressure": 0}, all_fluid=True)


class DeviceLattice:
    """Two HBM PDF buffers plus the step schedule for one PdfField."""

    def __init__(self, pdf, dtype="float64"):
        forest = pdf.forest
        self.pdf = pdf
        self.forest = forest
        self.ctx = forest.ctx
        self.q = pdf.stencil.q
        if dtype not in ("float64", "float32"):
            raise ValidationError(f"PDF dtype must be float64 or float32, got {dtype!r}")
        self.real_bytes = 8 if dtype == "float64" else 4
        self.tdtype = torch.float64 if dtype == "float64" else torch.float32
        if not torch.cuda.is_available():
            raise BackendError("no CUDA device: the B200 path has no CPU fallback")
        _lib.load()
        self.device = self.ctx.device if self.ctx.device.type == "cuda" else torch.device("cuda")
        self.box = box = RankBox(forest)
        elems_line = 128 // self.real_bytes
        g = _lib.Grid()
        g.q, g.real_bytes = self.q, self.real_bytes
        g.nx, g.ny, g.nz = box.nx, box.ny, box.nz
        g.xoff = elems_line
        g.pitch = _round_up(elems_line + box.nx + 1, elems_line)
        g.wrap_x, g.wrap_y = int(box.wrap_x), int(box.wrap_y)
        g.zface_lo, g.zface_hi = box.zface_lo, box.zface_hi
        self.grid = g
        self.gref = ctypes.byref(g)
        self.elems = int(_lib.load().lbm_field_elems(self.gref))
        if self.elems <= 0:
            _lib.call("lbm_field_elems", self.gref)
        self.buf = [hbm_empty(self.elems, self.tdtype, self.device),
                    hbm_empty(self.elems, self.tdtype, self.device)]
        self.cur = 0
        self.cur_kind = None      # None / "R" / "G"
        self.prev_kind = None     # None / "R" / "G"
        self.coll_key = None      # (params key, masks) that produced the current G
        self.stream_masks = None  # masks used by the pull that produced R_n
        self.host_state = "host"  # "host": host authoritative; "device": host stale; "synced"
        self.snapshot = None
        self.steps = 0
        self.launches = 0         # fused-kernel launches issued (bench's gpu_launches)
        self._halo = None
        self._streams = None
        self._fluid_masks = None
        self._rates = None        # (host copy, device tensor, version) of per-cell SRT rates
        self._graphs = {}         # (collision key, parity) -> (two-step CUDA graph, masks)
        self._dst_synced = None   # (steps, kind) the host dst slot was read back at

    # ---------------------------------------------------------- plumbing
    @property
    def stream(self):
        return torch.cuda.current_stream(self.device)

    def _sp(self, stream=None):
        return _lib.stream_ptr(stream if stream is not None else self.stream)

    def default_masks(self) -> Masks:
        if self._fluid_masks is None:
            self._fluid_masks = all_fluid_masks(self.box, self.device)
        return self._fluid_masks

    def _views(self, key):
        return [b.data[key].view_nosync for b in self.box.blocks]

    # ------------------------------------------------------ host <-> HBM
    def set_rates(self, dense) -> int:
        """Per-cell SRT rates (nz, ny, nx) fp64 -> HBM; returns a version
        number that changes only when the values do."""
        if self._rates is not None and np.array_equal(self._rates[0], dense):
            return self._rates[2]
        version = 0 if self._rates is None else self._rates[2] + 1
        t = torch.from_numpy(dense).to(self.device)
        self._rates = (dense.copy(), t, version)
        return version

    @property
    def omega_ptr(self):
        return self._rates[1].data_ptr()

    def upload_host(self):
        """Host R-form (src slot, ghosts incl.) -> buffer[cur] (kind R)."""
        fields = [b.data[self.pdf.key] for b in self.box.blocks]
        if not any(f.allocated for f in fields):
            # never written on the host: the reference's fields start at 0.0
            b = self.box
            z = torch.zeros((b.nz + 2, b.ny + 2, b.nx + 2), dtype=torch.float64, device=self.device)
            zu = torch.zeros((b.nz + 2, b.ny + 2, b.nx + 2, 3), dtype=torch.float64,
                             device=self.device)
            _lib.call("lbm_fill_equilibrium", self.gref, _lib.ptr(z), _lib.ptr(zu),
                      _lib.ptr(self.buf[self.cur]), self._sp())
            self.cur_kind, self.prev_kind = "R", None
            self.coll_key = None
            self.host_state = "device"
            self.snapshot = None
            self._dst_synced = None
            return
        dense = self.box.gather(self._views(self.pdf.key), self.q, np.float64)
        t = torch.from_numpy(dense).pin_memory().to(self.device, non_blocking=True)
        _lib.call("lbm_pack_rform", self.gref, _lib.ptr(t), _lib.ptr(self.buf[self.cur]), self._sp())
        self.cur_kind, self.prev_kind = "R", None
        self.coll_key = None
        self.host_state = "synced"
        self.snapshot = None
        self.halo_sync_rform()
        self._dst_synced = None
        torch.cuda.current_stream(self.device).synchronize()
        del t

    def fill_equilibrium(self, rho_g, u_g):
        """rho (Z,Y,X), u (Z,Y,X,3) ghost-inclusive box -> buffer[cur] (kind R)."""
        tr = torch.from_numpy(np.ascontiguousarray(rho_g, dtype=np.float64)).to(self.device)
        tu = torch.from_numpy(np.ascontiguousarray(u_g, dtype=np.float64)).to(self.device)
        _lib.call("lbm_fill_equilibrium", self.gref, _lib.ptr(tr), _lib.ptr(tu),
                  _lib.ptr(self.buf[self.cur]), self._sp())
        self.cur_kind, self.prev_kind = "R", None
        self.coll_key = None
        self.host_state = "device"
        self.snapshot = None
        self._dst_synced = None

    def halo_sync_rform(self):
        """R-form halos are not needed: G_0 = C(R_0) is computed on the
        interior and its crossing directions exchanged afterwards."""

    def readout_device(self):
        """R_n on the device: ("full", (q,Z,Y,X)) when a raw R-form is held,
        else ("interior", (q,nz,ny,nx)) = S(G_{n-1}) by the stream-only kernel."""
        self.join_streams()
        b = self.box
        if self.cur_kind == "R" or self.prev_kind == "R":
            src = self.buf[self.cur] if self.cur_kind == "R" else self.buf[1 - self.cur]
            out = hbm_empty((self.q, b.nz + 2, b.ny + 2, b.nx + 2), torch.float64, self.device)
            _lib.call("lbm_unpack_rform", self.gref, _lib.ptr(src), _lib.ptr(out), self._sp())
            return "full", out
        if self.cur_kind is None:
            raise ValidationError("PDF field has no device state")
        m = self.stream_masks
        out = hbm_empty((self.q, b.nz, b.ny, b.nx), torch.float64, self.device)
        _lib.call("lbm_stream_only", self.gref, self._kp_stream.ref,
                  _lib.ptr(self.buf[1 - self.cur]), _lib.ptr(m.cellmask), _lib.ptr(m.typemask),
                  _lib.ptr(out), self._sp())
        return "interior", out

    def readout(self):
        kind, t = self.readout_device()
        return kind, t.cpu().numpy()

    def rform_device(self):
        """R_n as a dense ghost-inclusive (q, Z, Y, X) fp64 device tensor:
        S(G_{n-1}) on the interior, the stored ghost shell around it."""
        kind, inner = self.readout_device()
        if kind == "full":
            return inner
        b = self.box
        full = hbm_empty((self.q, b.nz + 2, b.ny + 2, b.nx + 2), torch.float64, self.device)
        _lib.call("lbm_unpack_rform", self.gref, _lib.ptr(self.buf[self.cur]), _lib.ptr(full),
                  self._sp())
        full[:, 1:-1, 1:-1, 1:-1] = inner
        return full

    def adopt_rform(self, full):
        """Make a (possibly edited) dense R_n the device state (kind R): the
        next sweep collides it again, exactly as after a host upload."""
        _lib.call("lbm_pack_rform", self.gref, _lib.ptr(full), _lib.ptr(self.buf[self.cur]),
                  self._sp())
        self.cur_kind, self.prev_kind, self.coll_key = "R", None, None
        self.host_state, self.snapshot, self._dst_synced = "device", None, None

    def _wrap_ghosts(self, full):
        """Covered ghost cells of a ghost-inclusive (q, Z, Y, X) box = their
        periodic images inside the box (x, then y rows incl. x ghosts, then
        z planes: edges and corners come out as the reference's 26-image
        exchange fills them).  Halo and uncovered faces keep their values."""
        b = self.box
        if b.wrap_x:
            full[..., 0] = full[..., b.nx]
            full[..., b.nx + 1] = full[..., 1]
        if b.wrap_y:
            full[:, :, 0] = full[:, :, b.ny]
            full[:, :, b.ny + 1] = full[:, :, 1]
        if b.zface_lo == _lib.ZFACE_WRAP:
            full[:, 0] = full[:, b.nz]
            full[:, b.nz + 1] = full[:, 1]
        return full

    def full_state(self, which="src"):
        """The reference's Field.raw content of a PDF slot as a ghost-inclusive
        (q, Z, Y, X) fp64 device tensor: src = R_n, dst = C(R_{n-1}) after a
        sweep (the R-form fill before any).  Uncovered ghost cells carry the
        device values (never rewritten after the fill, as in the reference);
        covered ghosts are images of the slot's own interior.  (The
        reference's src ghosts hold stale images of C(R_{n-2}) between sweeps;
        every sweep overwrites them before use, so they carry no state.)"""
        self.join_streams()
        b = self.box
        full = hbm_empty((self.q, b.nz + 2, b.ny + 2, b.nx + 2), torch.float64, self.device)
        if which == "dst":
            src = self.buf[1 - self.cur] if self.prev_kind == "G" else self.buf[self.cur]
            _lib.call("lbm_unpack_rform", self.gref, _lib.ptr(src), _lib.ptr(full), self._sp())
        else:
            kind, t = self.readout_device()
            if kind == "full":
                full.copy_(t)
            else:
                _lib.call("lbm_unpack_rform", self.gref, _lib.ptr(self.buf[self.cur]),
                          _lib.ptr(full), self._sp())
                full[:, 1:-1, 1:-1, 1:-1] = t
        return self._wrap_ghosts(full)

    def sync_host(self):
        """Pull R_n into the host block arrays of the src slot (idempotent)."""
        if self.host_state != "device":
            return
        dense = self.full_state("src").cpu().numpy()
        self.box.scatter_full(dense, self._views(self.pdf.key))
        self.host_state = "synced"
        self.snapshot = None

    def sync_host_dst(self):
        """Pull C(R_{n-1}) into the host arrays of the dst slot (once per state)."""
        if self.cur_kind is None or self._dst_synced == (self.steps, self.cur_kind):
            return
        dense = self.full_state("dst").cpu().numpy()
        self.box.scatter_full(dense, self._views(self.pdf.dst_key))
        self._dst_synced = (self.steps, self.cur_kind)

    def host_touched(self):
        """Called when host arrays are handed out while synced: remember the
        content so the next sweep can tell whether the user wrote into it."""
        if self.host_state == "synced" and self.snapshot is None:
            self.snapshot = [v.copy() for v in self._views(self.pdf.key)]

    def host_changed(self) -> bool:
        if self.host_state == "host":
            return True
        if self.host_state == "device" or self.snapshot is None:
            return False
        return any(not np.array_equal(a, b) for a, b in zip(self.snapshot, self._views(self.pdf.key)))

    # ------------------------------------------------------------ steps
    def _streams_get(self):
        if self._streams is None:
            lo, hi = torch.cuda.Stream.priority_range()
            self._streams = {"boundary": torch.cuda.Stream(self.device, priority=hi),
                             "ev_b": torch.cuda.Event(), "ev_i": torch.cuda.Event(),
                             "pending": False}
        return self._streams

    def join_streams(self):
        """Make the caller's stream wait for any boundary/halo work."""
        if self._streams is not None and self._streams["pending"]:
            self.stream.wait_stream(self._streams["boundary"])
            self._streams["pending"] = False

    @property
    def halo(self):
        """z-face transport (collective on first use): the fused peer-store
        halo where the ranks can map each other, else NCCL / gloo-staged."""
        if self._halo is None:
            from .halo import make_halo
            self._halo = make_halo(self)
        return self._halo

    def ensure_collided(self, kp, key, masks):
        """Make buffer[cur] hold G_n = C_key(R_n)."""
        if self.cur_kind == "G" and self.coll_key == key:
            return
        self.join_streams()
        if self.cur_kind == "G":
            # model / flags changed between sweeps: the stored G_n was collided
            # with the old key.  Rebuild R_n = S(G_{n-1}) (old pull masks) into
            # buffer[cur] - its ghost shell stays valid - and collide again.
            _lib.call("lbm_pack_rform", self.gref, _lib.ptr(self.rform_device()),
                      _lib.ptr(self.buf[self.cur]), self._sp())
            self.cur_kind = "R"
        if self.cur_kind != "R":
            raise ValidationError("PDF field has no device state")
        # the other buffer becomes the first step's destination: it needs the
        # ghost shell of R_n (uncovered ghosts keep their fill values in both
        # buffers); its interior is written by that step, so only the shell
        # is copied (about 1 % of the field at 512^3 instead of all of it)
        _lib.call("lbm_copy_shell", self.gref, _lib.ptr(self.buf[self.cur]),
                  _lib.ptr(self.buf[1 - self.cur]), self._sp())
        self.prev_kind = None
        _lib.call("lbm_collide_only", self.gref, kp.ref, _lib.ptr(self.buf[self.cur]),
                  _lib.ptr(masks.cellmask), self._sp())
        if self.has_halo:
            # on the boundary stream, ordered after the collide (main)
            sb = self._streams_get()["boundary"]
            sb.wait_stream(self.stream)
            self.halo.after_collide(self, sb)
            self.stream.wait_stream(sb)
        self.cur_kind = "G"
        self.coll_key = key

    @property
    def has_halo(self) -> bool:
        return self.box.zface_lo == _lib.ZFACE_HALO or self.box.zface_hi == _lib.ZFACE_HALO

    def step(self, kp, key, masks, nsteps=1):
        """nsteps fused sweeps G_{n+1} = C(S(G_n))."""
        self.ensure_collided(kp, key, masks)
        nz = self.box.nz
        if masks.all_fluid:
            cm = tm = lb = None      # fused step reads no mask bytes
        else:
            cm = _lib.ptr(masks.cellmask)
            tm = _lib.ptr(masks.typemask) if masks.typed else None
            lb = masks.linkbits(self)
        lib = _lib.load()
        main = self.stream
        if self.has_halo:
            S = self._streams_get()
            S["boundary"].wait_stream(main)
        if not self.has_halo and nsteps >= 4:
            # launch-bound loops: replay a captured two-step graph (buffer
            # ping-pong returns to the same parity), odd remainder eagerly
            graph = self._pair_graph(kp, key, masks, cm, tm, lb)
            if graph is not None:
                # a graph captures kernel arguments, not constant memory:
                # make the device hold this model's MRT tables again (another
                # lattice may have uploaded its own since the capture)
                _lib.call("lbm_bind_params", self.gref, kp.ref, self._sp(main))
                for _ in range(nsteps // 2):
                    graph.replay()
                pairs = nsteps // 2
                self.steps += 2 * pairs
                self.launches += 2 * pairs
                self.prev_kind = "G"
                nsteps -= 2 * pairs
        for n in range(nsteps):
            src, dst = self.buf[self.cur], self.buf[1 - self.cur]
            if not self.has_halo:
                st = lib.lbm_fused_step_bits(self.gref, kp.ref, _lib.ptr(src), _lib.ptr(dst), cm,
                                             tm, lb, 0, nz, self._sp(main))
                if st:
                    _lib.call("lbm_fused_step_bits", self.gref, kp.ref, _lib.ptr(src),
                              _lib.ptr(dst), cm, tm, lb, 0, nz, self._sp(main))
            else:
                self._halo_step(kp, src, dst, cm, tm, main, lb)
            self.cur = 1 - self.cur
            self.prev_kind = "G"
            self.steps += 1
            self.launches += 1 if not self.has_halo else len({0, nz - 1}) + (1 if nz > 2 else 0)
        self.stream_masks = masks
        self._kp_stream = kp
        self.host_state = "device"
        self.snapshot = None
        self._dst_synced = None

    def _pair_graph(self, kp, key, masks, cm, tm, lb=None):
        """CUDA graph of two fused steps cur -> 1-cur -> cur (P = 1 path).
        Kernel arguments are captured by value, so the graph is keyed by the
        collision key and the buffer parity.  None if capture is unavailable
        (the caller then launches eagerly)."""
        hit = self._graphs.get((key, self.cur))
        if hit is not None:
            return hit[0]
        if len(self._graphs) >= 8:
            self._graphs.clear()
        nz = self.box.nz
        side = torch.cuda.Stream(self.device)
        side.wait_stream(self.stream)
        # both parities at once, so a loop entered at either parity replays
        for par in (0, 1):
            a, b = self.buf[par], self.buf[1 - par]
            graph = torch.cuda.CUDAGraph()
            try:
                with torch.cuda.graph(graph, stream=side):
                    sp = _lib.stream_ptr(torch.cuda.current_stream(self.device))
                    for src, dst in ((a, b), (b, a)):
                        _lib.call("lbm_fused_step_bits", self.gref, kp.ref, _lib.ptr(src),
                                  _lib.ptr(dst), cm, tm, lb, 0, nz, sp)
            except Exception:
                graph = None
            self._graphs[(key, par)] = (graph, masks)   # keeps the mask tensors alive
        self.stream.wait_stream(side)
        return self._graphs[(key, self.cur)][0]

    def _halo_step(self, kp, src, dst, cm, tm, main, lb=None):
        """One overlapped step: B(n) = boundary planes on the high-priority
        stream, its crossing directions handed to the halo transport (fused
        peer stores or send/recv), I(n) = interior
        planes on the caller's stream.  Hazards: B(n) after I(n-1) (B writes
        planes I(n-1) reads); I(n) after B(n-1) (I writes planes B(n-1)
        reads); B(n+1) after the halo of step n (stream order)."""
        S = self._streams_get()
        sb = S["boundary"]
        nz = self.box.nz
        # also across stream_collide calls (one sweep per call is the common
        # case); waiting on a never-recorded event is a no-op
        main.wait_event(S["ev_b"])           # I(n) after B(n-1)
        sb.wait_event(S["ev_i"])             # B(n) after I(n-1)
        self.halo.boundary(self, kp, src, dst, cm, tm, sb)
        S["ev_b"].record(sb)
        self.halo.after_boundary(self, dst, sb)
        if nz > 2:
            _lib.call("lbm_fused_step_bits", self.gref, kp.ref, _lib.ptr(src), _lib.ptr(dst), cm,
                      tm, lb, 1, nz - 1, self._sp(main))
        S["ev_i"].record(main)
        S["pending"] = True

    # ---------------------------------------------------- pipelined job
    def can_pipeline(self) -> bool:
        """One rank, z not periodic: a job's sweeps can run as a wavefront
        behind the upload (a periodic z couples the first and last planes)."""
        return (not self.has_halo and self.box.zface_lo == _lib.ZFACE_GHOST
                and self.box.zface_hi == _lib.ZFACE_GHOST)

    def run_job(self, kp, key, masks, kp_mom, rho_h, u_h, steps, out, chunk=None):
        """fill_equilibrium_arrays -> `steps` fused sweeps -> moments of R_K,
        as a wavefront over chunks of z-planes so the PCIe copies overlap the
        sweeps.  Same kernels and arithmetic as the call sequence, in another
        order (job_plan: the dependency rules, ramp and tail); bitwise
        identical results and end state.  G_n lives in buf[(c0 + n) % 2].
        Uncovered z ghost planes keep their fill values in both buffers (fill
        writes the other buffer's shell).  `chunk`: see job_schedule."""
        b = self.box
        nz = b.nz
        self.join_streams()
        main = self.stream
        dev = self.device
        shape_r, shape_u = (nz, b.ny, b.nx), (nz, b.ny, b.nx, 3)
        st = getattr(self, "_job_stage", None)
        if st is None or st["shape"] != shape_r:
            st = {"shape": shape_r,
                  "rho": hbm_empty(shape_r, torch.float64, dev),
                  "u": hbm_empty(shape_u, torch.float64, dev),
                  "rho_o": hbm_empty(shape_r, torch.float64, dev),
                  "u_o": hbm_empty(shape_u, torch.float64, dev),
                  "bad": torch.zeros(1, dtype=torch.int32, device=dev),
                  "up": torch.cuda.Stream(dev), "dn": torch.cuda.Stream(dev)}
            self._job_stage = st
        up, dn = st["up"], st["dn"]
        # staging reuse across jobs: uploads after the last job's fills,
        # moments after its downloads
        up.wait_stream(main)
        main.wait_stream(dn)
        st["bad"].zero_()
        bounds, _ = job_schedule(nz, steps, chunk)
        evs = []
        with torch.cuda.stream(up):
            for z0, z1 in bounds:
                st["rho"][z0:z1].copy_(rho_h[z0:z1], non_blocking=True)
                st["u"][z0:z1].copy_(u_h[z0:z1], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(up)
                evs.append(ev)
        c0 = self.cur
        buf = self.buf
        if masks.all_fluid:
            cm = tm = lb = None
        else:
            cm = _lib.ptr(masks.cellmask)
            tm = _lib.ptr(masks.typemask) if masks.typed else None
            lb = masks.linkbits(self)
        sp = self._sp(main)
        launches = 0
        # the last sweep also writes the readout (lbm_fused_step_moments) -
        # not with the link-bit map (its kernels read the cell mask);
        # LBM_B200_JOB_FUSE_MOMENTS=0 keeps the separate moments pass
        fuse_mom = lb is None and os.environ.get("LBM_B200_JOB_FUSE_MOMENTS", "1") != "0"
        for act in job_plan(nz, steps, chunk):
            if act[0] == "fill":
                _, ci, z0, z1 = act
                main.wait_event(evs[ci])
                # equilibrium + G_0 = C(R_0) of the chunk in one pass (the
                # other buffer gets the ghost shell)
                _lib.call("lbm_fill_collide_planes", self.gref, kp.ref, _lib.ptr(st["rho"]),
                          _lib.ptr(st["u"]), z0, z1, _lib.ptr(buf[c0]), _lib.ptr(buf[1 - c0]),
                          _lib.ptr(masks.cellmask), sp)
            elif act[0] == "step" and act[1] == steps and fuse_mom:
                # the last sweep reads G_{K-1}: it hands back the moments of
                # R_K = S(G_{K-1}) on the same planes (job_plan gives the
                # moments exactly this step's ranges)
                _, n, z0, z1 = act
                _lib.call("lbm_fused_step_moments", self.gref, kp.ref, kp_mom.ref,
                          _lib.ptr(buf[(c0 + n - 1) % 2]), _lib.ptr(buf[(c0 + n) % 2]),
                          _lib.ptr(masks.cellmask), _lib.ptr(masks.typemask),
                          z0, z1, _lib.ptr(st["rho_o"]), _lib.ptr(st["u_o"]),
                          _lib.ptr(st["bad"]), sp)
                launches += 1
            elif act[0] == "step":
                _, n, z0, z1 = act
                _lib.call("lbm_fused_step_bits", self.gref, kp.ref,
                          _lib.ptr(buf[(c0 + n - 1) % 2]), _lib.ptr(buf[(c0 + n) % 2]), cm, tm,
                          lb, z0, z1, sp)
                launches += 1
            else:
                _, z0, z1 = act
                if not fuse_mom:
                    _lib.call("lbm_moments_planes", self.gref, kp_mom.ref,
                              _lib.ptr(buf[(c0 + steps - 1) % 2]), _lib.ptr(masks.cellmask),
                              _lib.ptr(masks.typemask), 1, z0, z1, _lib.ptr(st["rho_o"]),
                              _lib.ptr(st["u_o"]), _lib.ptr(st["bad"]), sp)
                evm = torch.cuda.Event()
                evm.record(main)
                dn.wait_event(evm)
                with torch.cuda.stream(dn):
                    out[0][z0:z1].copy_(st["rho_o"][z0:z1], non_blocking=True)
                    out[1][z0:z1].copy_(st["u_o"][z0:z1], non_blocking=True)
        dn.synchronize()
        # end state: exactly what the call sequence leaves
        self.cur = (c0 + steps) % 2
        self.cur_kind, self.prev_kind = "G", "G"
        self.coll_key = key
        self.stream_masks = masks
        self._kp_stream = kp
        self.steps += steps
        self.launches += launches
        self.host_state = "device"
        self.snapshot = None
        self._dst_synced = None
        return st["bad"]

    # ---------------------------------------------------------- readout
    def moments(self, kp, masks):
        """rho (nz,ny,nx), u (nz,ny,nx,3) of R_n on the host, fp64."""
        self.join_streams()
        b = self.box
        rho = torch.empty((b.nz, b.ny, b.nx), dtype=torch.float64, device=self.device)
        u = torch.empty((b.nz, b.ny, b.nx, 3), dtype=torch.float64, device=self.device)
        bad = torch.zeros(1, dtype=torch.int32, device=self.device)
        if self.cur_kind == "R":
            _lib.call("lbm_moments", self.gref, kp.ref, _lib.ptr(self.buf[self.cur]), None, None, 0,
                      _lib.ptr(rho), _lib.ptr(u), _lib.ptr(bad), self._sp())
        elif self.prev_kind == "R":
            _lib.call("lbm_moments", self.gref, kp.ref, _lib.ptr(self.buf[1 - self.cur]), None, None,
                      0, _lib.ptr(rho), _lib.ptr(u), _lib.ptr(bad), self._sp())
        else:
            m = self.stream_masks
            _lib.call("lbm_moments", self.gref, kp.ref, _lib.ptr(self.buf[1 - self.cur]),
                      _lib.ptr(m.cellmask), _lib.ptr(m.typemask), 1, _lib.ptr(rho), _lib.ptr(u),
                      _lib.ptr(bad), self._sp())
        return rho, u, bad
