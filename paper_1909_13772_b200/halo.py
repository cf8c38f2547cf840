"""Per-step z-face halo exchange of the G-form: fused peer stores over
NVLink (PeerHalo, the default between GPUs) or NCCL send/recv in place.

Replaces the per-step `exchange_ghosts(forest, [GhostPackInfo("pdf")])`
of stream_collide (lbm/sweep.py:110-114, field/ghost.py:202-264).  Because
the device keeps the post-collision state, a face only needs the directions
whose c_z points into the receiving box (5 of 19 for D3Q19, 9 of 27 for
D3Q27) and, thanks to the z-q-y-x layout with slots grouped by c_z, those are
ONE contiguous run per plane (`lbm_face_span`).  They go straight from the
sender's boundary plane into the receiver's ghost plane - no pack kernel,
no staging buffer - as a single grouped send/recv per neighbour pair
(ncclGroupStart/End through torch.distributed.batch_isend_irecv).

Op order is canonical so sends and receives between the same pair match
even when both faces face one peer (P = 2 periodic): every rank posts
sends as (low face, high face) and receives as (high face, low face) - a
peer's low-face send lands in my high ghost plane and vice versa.

The transport only slices tensors and calls torch.distributed, so the same
code runs on CPU tensors over gloo in the world_size-2 tests.

`PeerHalo` is the B200-native transport: the boundary-plane kernel itself
stores the crossing directions into the neighbour's ghost plane
(lbm_fused_step_peer) - in the neighbour's HBM, mapped through CUDA IPC over
NVLink / NVSwitch, or directly when the ranks share a process - so the halo
moves while the plane is computed and no collective runs at all.  `make_halo`
picks it whenever every rank can map its neighbours; NCCL send/recv (`Halo`)
stays as the fallback transport.
"""
from __future__ import annotations

import ctypes
import os

import torch
import torch.distributed as dist

from . import _lib


def face_spans(grid_ref):
    """{face: (send_off, recv_off, count)} in elements (0 = low z, 1 = high z)."""
    out = {}
    lib = _lib.load()
    for face in (0, 1):
        s, r, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _lib.call("lbm_face_span", grid_ref, face, ctypes.byref(s), ctypes.byref(r), ctypes.byref(c))
        out[face] = (s.value, r.value, c.value)
    del lib
    return out


def plan_ops(zface_lo, zface_hi, lo_peer, hi_peer, spans):
    """Ordered [(kind, peer, offset, count)] for one exchange round."""
    halo = _lib.ZFACE_HALO
    ops = []
    if zface_lo == halo:
        s, _, c = spans[0]
        ops.append(("send", lo_peer, s, c))
    if zface_hi == halo:
        s, _, c = spans[1]
        ops.append(("send", hi_peer, s, c))
    if zface_hi == halo:
        _, r, c = spans[1]
        ops.append(("recv", hi_peer, r, c))
    if zface_lo == halo:
        _, r, c = spans[0]
        ops.append(("recv", lo_peer, r, c))
    return ops


def run_ops(ops, flat, group=None):
    """Issue the grouped send/recv on views of the flat field tensor and
    return the works (the caller's current stream waits on them).

    With NCCL the views are sent/received in place.  With gloo (CPU test
    transport) CUDA views are staged through host copies; this keeps the
    multi-process tests runnable with several ranks sharing one GPU, where
    NCCL cannot run."""
    if not ops:
        return []
    staged = flat.is_cuda and dist.get_backend(group) != "nccl"
    p2p, back = [], []
    for kind, peer, off, count in ops:
        view = flat[off:off + count]
        if staged:
            if kind == "send":
                view = view.cpu()
            else:
                host = view.new_empty(view.shape, device="cpu")
                back.append((flat[off:off + count], host))
                view = host
        fn = dist.isend if kind == "send" else dist.irecv
        p2p.append(dist.P2POp(fn, view, peer, group))
    works = dist.batch_isend_irecv(p2p)
    if staged:
        for w in works:
            w.wait()
        for dst, host in back:
            dst.copy_(host)
        return []
    return works


class Halo:
    """Exchange plan of one DeviceLattice (NCCL send/recv, or gloo-staged)."""

    kind = "nccl"

    def __init__(self, lattice):
        box = lattice.box
        self.spans = face_spans(lattice.gref)
        self.ops = plan_ops(box.zface_lo, box.zface_hi, box.lo_peer, box.hi_peer, self.spans)
        self.bytes_per_exchange = sum(c for k, _, _, c in self.ops if k == "send") * lattice.real_bytes
        if lattice.device.type == "cuda" and dist.is_initialized() and dist.get_backend() != "nccl":
            self.kind = "staged"

    def after_collide(self, lat, stream):
        """G_0's crossing directions -> the neighbours' ghost planes."""
        self.exchange(lat.buf[lat.cur], stream)

    def boundary(self, lat, kp, src, dst, cm, tm, stream):
        """B(n): the boundary planes, then the halo of their crossing runs."""
        nz = lat.box.nz
        for z in sorted({0, nz - 1}):
            _lib.call("lbm_fused_step", lat.gref, kp.ref, _lib.ptr(src), _lib.ptr(dst), cm, tm,
                      z, z + 1, _lib.stream_ptr(stream))
        return stream

    def after_boundary(self, lat, dst, stream):
        self.exchange(dst, stream)

    def exchange(self, flat, stream):
        """Fill the ghost planes of `flat` from the neighbours' boundary
        planes; ordered after prior work on `stream`, and `stream` waits for
        completion (device-side, the host does not block)."""
        import torch
        with torch.cuda.stream(stream):
            works = run_ops(self.ops, flat)
            for w in works:
                w.wait()


# ------------------------------------------------------------ fused halo
def _ipc_export(t):
    """(64-byte IPC handle, byte offset) of a device tensor's storage."""
    h = ctypes.create_string_buffer(64)
    off = ctypes.c_int64()
    _lib.call("lbm_ipc_export", ctypes.c_void_p(t.data_ptr()), h, ctypes.byref(off))
    return h.raw, off.value


def _face_geometry(lat):
    """(send_off, count) per face and the receiving ghost-block offsets."""
    spans = face_spans(lat.gref)
    blocks = {}
    for face in (0, 1):
        off = ctypes.c_int64()
        _lib.call("lbm_ghost_block_offset", lat.gref, face, ctypes.byref(off))
        blocks[face] = off.value
    return spans, blocks


class PeerHalo:
    """Fused peer-store z-face halo with a device-side phase protocol.

    Every rank publishes its two PDF buffers and a two-word flag array
    (from_lo, from_hi) to its z-neighbours.  Rank r's step n then runs, on its
    boundary stream:

      1. phase entry k: write k into the neighbours' flag words (a stream
         memory op, ordered after all earlier work of the stream - including
         the previous phase's peer stores and, through the wait on the main
         stream, every readout), then wait until both own flag words are
         >= k.  Rank and neighbour have now both finished phase k-1 and all
         reads of the buffers phase k writes into;
      2. the boundary planes with lbm_fused_step_peer: each plane also stores
         its crossing directions into the neighbour's dst ghost plane.

    After collide_only (G_0) a phase copies the whole crossing runs (x/y
    ghost ring included, like the NCCL transport) instead.

    mode "device": flags + memops (one process per GPU over NVLink, or the
    in-process thread ranks).  mode "host": ranks are processes sharing one
    GPU; the phase entry is a device synchronize + a host barrier instead of
    stream waits, because processes time-sliced on one GPU must not wait on
    each other on the device (B200_PROFILING: Xid 109).  Peers in another
    process are mapped from CUDA IPC handles into this GPU's context with
    lazy peer access (lbm_ipc_export / lbm_ipc_open); in-process peers are
    used directly.  self.peer holds raw device addresses."""

    def __init__(self, lat, mode: str):
        self.kind = "peer-" + mode
        self.mode = mode
        self.lat = lat
        box = lat.box
        ctx = lat.ctx
        self.spans, self.blocks = _face_geometry(lat)
        self.flags = torch.zeros(2, dtype=torch.int32, device=lat.device)
        # the zero fill must land before any neighbour can signal into it
        torch.cuda.current_stream(lat.device).synchronize()
        self.phase = 0
        in_process = getattr(ctx, "backend", None) == "threads"
        self.lockstep = in_process
        if in_process:
            key = ("peer-halo", id(lat.forest.ctx.group), lat.pdf.key)
            table = ctx.group.shared.setdefault(key, {})
            table[ctx.rank] = tuple(t.data_ptr() for t in (lat.buf[0], lat.buf[1], self.flags))
            mine = None
        else:
            mine = tuple(_ipc_export(t) for t in (lat.buf[0], lat.buf[1], self.flags))
        self._opened = {}       # handle bytes -> mapped base (closed in close())
        info = {"handles": mine, "spans": self.spans, "blocks": self.blocks,
                "pitch": lat.grid.pitch, "rb": lat.real_bytes, "q": lat.q}
        peers = ctx.all_gather(info)
        self.peer = {}          # face -> addresses (buf0, buf1, flags) of the neighbour across it
        self.peer_info = {}
        err = None
        try:
            for face, peer, facing in ((0, box.lo_peer, 1), (1, box.hi_peer, 0)):
                zmode = box.zface_lo if face == 0 else box.zface_hi
                if zmode != _lib.ZFACE_HALO:
                    continue
                pi = peers[peer]
                if (pi["pitch"], pi["rb"], pi["q"]) != (lat.grid.pitch, lat.real_bytes, lat.q):
                    raise RuntimeError("z-neighbours disagree on the row layout")
                if in_process:
                    addrs = table[peer]
                else:
                    addrs = tuple(self._open(h, off) for h, off in pi["handles"])
                self.peer[face] = addrs
                self.peer_info[face] = (pi["blocks"][facing], pi["spans"][facing])
        except Exception as exc:    # decided collectively below, never a lone raise
            err = f"rank {ctx.rank}: {type(exc).__name__}: {exc}"
        self.bytes_per_exchange = sum(self.spans[f][2] for f in self.peer) * lat.real_bytes
        # every rank holds its peers' mappings before any phase (or all fall back)
        errs = [e for e in ctx.all_gather(err).values() if e]
        if errs:
            self.close()
            raise PeerHaloUnavailable("; ".join(errs))
        if mode == "device":
            self._handshake()

    def _handshake(self, timeout_s: float = 30.0):
        """Setup-time check of the device signalling path, without any
        device-side wait: every rank writes a token into its neighbours'
        flag words with the same stream memory op the phases use, then the
        host polls its own words.  Raises PeerHaloUnavailable (the caller
        falls back to send/recv on every rank) if a token does not arrive -
        e.g. memory ops on peer mappings unsupported - so a broken path
        fails at setup instead of hanging a sweep."""
        import time
        lat, ctx = self.lat, self.lat.ctx
        token = 0x5A5A0001
        sp = _lib.stream_ptr(torch.cuda.current_stream(lat.device))
        ok = True
        try:
            for face, word in ((0, 1), (1, 0)):
                if face in self.peer:
                    flags = self.peer[face][2]
                    _lib.call("lbm_stream_signal", ctypes.c_void_p(flags + 4 * word), token, sp)
            torch.cuda.current_stream(lat.device).synchronize()
            t0 = time.monotonic()
            while True:
                got = self.flags.cpu().tolist()
                if all(got[f] == token for f in self.peer):
                    break
                if time.monotonic() - t0 > timeout_s:
                    ok = False
                    break
                time.sleep(0.001)
        except Exception:
            ok = False
        ok = all(ctx.all_gather(ok).values())
        # nobody writes the words any more: reset them for phase 1
        self.flags.zero_()
        torch.cuda.current_stream(lat.device).synchronize()
        ctx.barrier()
        if not ok:
            raise PeerHaloUnavailable("stream memory ops on peer mappings did not arrive")

    def _open(self, handle: bytes, offset: int) -> int:
        """Map a peer allocation once per handle (P = 2 periodic: both faces
        face the same rank) and return the address of its buffer."""
        base = self._opened.get(handle)
        if base is None:
            out = ctypes.c_void_p()
            _lib.call("lbm_ipc_open", handle, ctypes.byref(out))
            base = self._opened[handle] = out.value
        return base + offset

    def close(self):
        """Unmap the neighbours' buffers.  Only this rank's stores go through
        the mappings, so closing needs no collective - but no further phase
        may run on this halo."""
        opened, self._opened = getattr(self, "_opened", {}), {}
        for base in opened.values():
            _lib.call("lbm_ipc_close", ctypes.c_void_p(base))
        self.peer = {}

    def __del__(self):
        # the lattice (and this halo) goes away: drop the IPC mappings so a
        # neighbour's freed buffer is not kept alive by this process
        try:
            self.close()
        except Exception:
            pass

    # -- protocol
    def _enter_phase(self, stream):
        self.phase += 1
        k = self.phase
        if self.mode == "host":
            torch.cuda.synchronize(self.lat.device)
            self.lat.ctx.barrier()
            return
        sp = _lib.stream_ptr(stream)
        # my low face's neighbour sees me as its upper neighbour (its from_hi)
        for face, word in ((0, 1), (1, 0)):
            if face in self.peer:
                flags = self.peer[face][2]
                _lib.call("lbm_stream_signal", ctypes.c_void_p(flags + 4 * word), k, sp)
        if self.lockstep:
            # thread ranks share one CUDA context, where a device-wide
            # synchronisation inside torch (pinned-host allocation, cudaFree)
            # would also wait for a peer's stream blocked on a signal this
            # thread has not enqueued yet: enqueue every wait only after all
            # ranks have enqueued their signal.  GPU-side ordering is still
            # the flags' alone (the barrier does not wait for the device).
            self.lat.ctx.barrier()
        for face in self.peer:
            _lib.call("lbm_stream_wait", ctypes.c_void_p(self.flags.data_ptr() + 4 * face), k, sp)

    def after_collide(self, lat, stream):
        """Phase: copy G_0's crossing runs into the neighbours' current buffer."""
        self._enter_phase(stream)
        mine = lat.buf[lat.cur]
        rb = lat.real_bytes
        for face, addrs in self.peer.items():
            send_off, _, count = self.spans[face]
            _, (_, recv_off, rcount) = self.peer_info[face]
            if rcount != count:
                raise RuntimeError("halo runs of the two sides differ")
            _lib.call("lbm_copy_async", ctypes.c_void_p(addrs[lat.cur] + recv_off * rb),
                      ctypes.c_void_p(mine.data_ptr() + send_off * rb), count * rb,
                      _lib.stream_ptr(stream))

    def boundary(self, lat, kp, src, dst, cm, tm, stream):
        """Phase: B(n) with the crossing directions stored into the peers."""
        self._enter_phase(stream)
        dpar = 1 - lat.cur
        lo = hi = None
        if 0 in self.peer:
            lo = ctypes.c_void_p(self.peer[0][dpar] + self.peer_info[0][0] * lat.real_bytes)
        if 1 in self.peer:
            hi = ctypes.c_void_p(self.peer[1][dpar] + self.peer_info[1][0] * lat.real_bytes)
        nz = lat.box.nz
        sp = _lib.stream_ptr(stream)
        for z in sorted({0, nz - 1}):
            _lib.call("lbm_fused_step_peer", lat.gref, kp.ref, _lib.ptr(src), _lib.ptr(dst), cm, tm,
                      z, z + 1, lo if z == 0 else None, hi if z == nz - 1 else None, sp)
        return stream

    def after_boundary(self, lat, dst, stream):
        pass


def select_transport(lat) -> str:
    """'peer-device', 'peer-host', 'nccl' or 'staged' - the same on every
    rank (decided from the environment and an all_gather of capabilities).
    LBM_B200_HALO=nccl forces NCCL send/recv, =peer asks for the fused
    transport also where ranks are processes sharing a GPU (host-ordered)."""
    ctx = lat.ctx
    want = os.environ.get("LBM_B200_HALO", "auto")
    if want not in ("auto", "peer", "nccl"):
        raise ValueError(f"LBM_B200_HALO must be auto, peer or nccl, got {want!r}")
    if getattr(ctx, "backend", None) == "threads":
        return "peer-device"
    backend = dist.get_backend() if dist.is_initialized() else None
    if lat.device.type != "cuda" or backend is None:
        return "staged"
    idx = lat.device.index if lat.device.index is not None else torch.cuda.current_device()
    local = {str(torch.cuda.get_device_properties(i).uuid): i
             for i in range(torch.cuda.device_count())}
    uuid = str(torch.cuda.get_device_properties(idx).uuid)
    caps = ctx.all_gather({"uuid": uuid, "node": os.uname().nodename})
    shared = len({c["uuid"] for c in caps.values()}) < len(caps)
    same_node = len({c["node"] for c in caps.values()}) == 1
    # every peer GPU visible here and reachable by peer access (NVLink / NVSwitch)
    can_map = same_node and all(
        c["uuid"] in local and (local[c["uuid"]] == idx
                                or torch.cuda.can_device_access_peer(idx, local[c["uuid"]]))
        for c in caps.values())
    can_map = all(ctx.all_gather(bool(can_map)).values())
    if backend == "nccl":
        if want == "nccl" or shared or not can_map:
            return "nccl"
        # a peer GPU's halo stores and its later flag write may be reordered
        # on arrival unless the stream wait can flush remote writes
        # (CU_STREAM_WAIT_VALUE_FLUSH): without it, send/recv
        with torch.cuda.device(idx):
            flush = bool(_lib.load().lbm_can_flush_remote_writes())
        if not all(ctx.all_gather(flush).values()):
            return "nccl"
        return "peer-device"
    # gloo on CUDA tensors: host-staged unless the fused transport is asked for
    if want == "peer" and same_node:
        return "peer-host" if shared else "peer-device"
    return "staged"


class PeerHaloUnavailable(RuntimeError):
    """The fused halo's setup check failed on some rank (collective)."""


def make_halo(lat):
    kind = select_transport(lat)
    if kind.startswith("peer-"):
        try:
            return PeerHalo(lat, kind[5:])
        except PeerHaloUnavailable as exc:
            import warnings
            warnings.warn(f"fused peer halo unavailable ({exc}); using send/recv", RuntimeWarning)
    return Halo(lat)
