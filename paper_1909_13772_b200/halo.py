"""Per-step z-face halo exchange of the G-form, zero-copy over NCCL.

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
"""
from __future__ import annotations

import ctypes

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
    """Exchange plan of one DeviceLattice."""

    def __init__(self, lattice):
        box = lattice.box
        self.spans = face_spans(lattice.gref)
        self.ops = plan_ops(box.zface_lo, box.zface_hi, box.lo_peer, box.hi_peer, self.spans)
        self.bytes_per_exchange = sum(c for k, _, _, c in self.ops if k == "send") * lattice.real_bytes

    def exchange(self, flat, stream):
        """Fill the ghost planes of `flat` from the neighbours' boundary
        planes; ordered after prior work on `stream`, and `stream` waits for
        completion (device-side, the host does not block)."""
        import torch
        with torch.cuda.stream(stream):
            works = run_ops(self.ops, flat)
            for w in works:
                w.wait()
