"""world_size-2/4 tests of the multi-rank host path on CPU (gloo).

Covers what a z-slab run does outside the kernels: the zero-copy halo plan
and transport (halo.py) on tensors in the device layout, and the host-side
collectives of the drop-in API (exchange_ghosts, gather_slice, all_reduce).
"""
import ctypes

import numpy as np
import pytest
import torch

import paper_1909_13772_b200 as P
from paper_1909_13772_b200 import _lib, halo
from paper_1909_13772_b200.device import RankBox


def _grid_for(box, q=19, rb=8):
    g = _lib.Grid()
    g.q, g.real_bytes = q, rb
    g.nx, g.ny, g.nz = box.nx, box.ny, box.nz
    g.xoff = 128 // rb
    g.pitch = ((g.xoff + box.nx + 1 + g.xoff - 1) // g.xoff) * g.xoff
    g.wrap_x, g.wrap_y = int(box.wrap_x), int(box.wrap_y)
    g.zface_lo, g.zface_hi = box.zface_lo, box.zface_hi
    return g


def _halo_prog(ctx, periodic_z, q):
    forest = P.create_forest(ctx, (0, 0, 0, 1, 1, ctx.n_ranks), (1, 1, ctx.n_ranks),
                             periodic=(True, True, periodic_z), cells_per_block=(5, 4, 3))
    box = RankBox(forest)
    g = _grid_for(box, q)
    spans = halo.face_spans(ctypes.byref(g))
    ops = halo.plan_ops(box.zface_lo, box.zface_hi, box.lo_peer, box.hi_peer, spans)
    n = int(_lib.load().lbm_field_elems(ctypes.byref(g)))
    flat = torch.arange(n, dtype=torch.float64) + 1e6 * (ctx.rank + 1)
    before = flat.clone()
    works = halo.run_ops(ops, flat)
    for w in works:
        w.wait()
    return {"rank": ctx.rank, "spans": spans, "ops": ops, "before": before.numpy(),
            "after": flat.numpy(), "box": (box.zface_lo, box.zface_hi, box.lo_peer, box.hi_peer)}


@pytest.mark.parametrize("n_ranks,periodic_z", [(2, True), (2, False), (4, True), (3, False)])
@pytest.mark.parametrize("q", [19, 27])
def test_halo_transport_fills_crossing_ghost_planes(n_ranks, periodic_z, q):
    res = P.run(n_ranks, _halo_prog, periodic_z, q, backend="gloo")
    for r in res:
        (s0, r0, c0), (s1, r1, c1) = r["spans"][0], r["spans"][1]
        zlo, zhi, lo_peer, hi_peer = r["box"]
        after, before = r["after"], r["before"]
        if zlo == _lib.ZFACE_HALO:
            # my low ghost plane (c_z=+1 run) == low peer's top interior plane run
            peer = res[lo_peer]
            ps1, _, pc1 = peer["spans"][1]
            assert np.array_equal(after[r0:r0 + c0], peer["before"][ps1:ps1 + pc1])
        else:
            assert np.array_equal(after[r0:r0 + c0], before[r0:r0 + c0])
        if zhi == _lib.ZFACE_HALO:
            peer = res[hi_peer]
            ps0, _, pc0 = peer["spans"][0]
            assert np.array_equal(after[r1:r1 + c1], peer["before"][ps0:ps0 + pc0])
        # nothing outside the receive runs changed
        mask = np.ones(after.size, bool)
        if zlo == _lib.ZFACE_HALO:
            mask[r0:r0 + c0] = False
        if zhi == _lib.ZFACE_HALO:
            mask[r1:r1 + c1] = False
        assert np.array_equal(after[mask], before[mask])


def _host_prog(ctx):
    forest = P.create_forest(ctx, (0, 0, 0, 1, 1, 2 * ctx.n_ranks), (1, 1, 2 * ctx.n_ranks),
                             periodic=(True, False, True), cells_per_block=(4, 3, 2))
    forest.register_data("s", P.FieldDataHandler(nf=2, ghost_layers=1, layout="fzyx"))
    N = forest.global_cells(0)
    for b in forest.local_blocks():
        lo, hi = forest.cell_box(b.id)
        z, y, x = np.meshgrid(np.arange(lo[2], hi[2]), np.arange(lo[1], hi[1]),
                              np.arange(lo[0], hi[0]), indexing="ij")
        b.data["s"].interior[..., 0] = x + 10 * y + 100 * z
        b.data["s"].interior[..., 1] = -(x + 10 * y + 100 * z)
    P.exchange_ghosts(forest, ["s"])
    bad = 0
    for b in forest.local_blocks():
        lo, hi = forest.cell_box(b.id)
        v = b.data["s"].view
        for zz in range(-1, hi[2] - lo[2] + 1):
            for yy in range(0, hi[1] - lo[1]):
                for xx in range(-1, hi[0] - lo[0] + 1):
                    gx, gy, gz = (lo[0] + xx) % N[0], lo[1] + yy, (lo[2] + zz) % N[2]
                    want = gx + 10 * gy + 100 * gz
                    bad += v[zz + 1, yy + 1, xx + 1, 0] != want
                    bad += v[zz + 1, yy + 1, xx + 1, 1] != -want
    full = P.gather_slice(forest, "s", (0, 0, 0), N)
    tot = ctx.all_reduce(float(ctx.rank + 1))
    return bad, (None if full is None else full[..., 0].copy()), tot, forest.neighbor_ranks()


def test_host_collectives_two_ranks():
    res = P.run(2, _host_prog, backend="gloo")
    assert all(r[0] == 0 for r in res)
    full = res[0][1]
    z, y, x = np.meshgrid(np.arange(8), np.arange(3), np.arange(4), indexing="ij")
    assert np.array_equal(full, x + 10 * y + 100 * z)
    assert res[1][1] is None
    assert res[0][2] == res[1][2] == 3.0
    assert res[0][3] == [1] and res[1][3] == [0]


# ------------------------------------------------------ in-process rank group
def _thread_prog(ctx, payload):
    got = ctx.all_gather({"rank": ctx.rank, "payload": payload * (ctx.rank + 1)})
    total = ctx.all_reduce((float(ctx.rank), 1.0), "sum")
    ctx.barrier()
    return got, total


def test_thread_rank_group_collectives_in_rank_order():
    """ThreadContext (the in-process rank group the fused device halo is
    tested with) keeps the process transport's collective semantics."""
    res = P.run(3, _thread_prog, 2, backend="threads", device="cpu")
    for r, (got, total) in enumerate(res):
        assert sorted(got) == [0, 1, 2]
        assert [got[k]["payload"] for k in range(3)] == [2, 4, 6]
        assert total == [3.0, 3.0]


def _thread_fail(ctx):
    if ctx.rank == 1:
        raise ValueError("boom")
    ctx.barrier()       # released by the failing rank's abort, not hung


def test_thread_rank_group_reports_failures():
    with pytest.raises(RuntimeError, match="boom"):
        P.run(2, _thread_fail, backend="threads", device="cpu", timeout=60)


def _select_prog(ctx):
    forest = P.create_forest(ctx, (0, 0, 0, 4, 4, 2 * ctx.n_ranks), (1, 1, ctx.n_ranks),
                             periodic=(True, True, True), cells_per_block=(4, 4, 2))

    class _Lat:     # what select_transport reads of a DeviceLattice
        pass
    lat = _Lat()
    lat.ctx, lat.device, lat.forest = ctx, torch.device("cpu"), forest
    return halo.select_transport(lat)


def test_transport_selection_on_cpu_ranks():
    # CPU tensors over gloo: the host-staged transport; threads: the fused one
    assert P.run(2, _select_prog, backend="gloo") == ["staged", "staged"]
    assert P.run(2, _select_prog, backend="threads", device="cpu") == ["peer-device"] * 2


def test_transport_env_is_validated(monkeypatch):
    class _Lat:
        pass
    lat = _Lat()
    lat.ctx, lat.device = P.Context(device="cpu"), torch.device("cpu")
    monkeypatch.setenv("LBM_B200_HALO", "carrier-pigeon")
    with pytest.raises(ValueError, match="LBM_B200_HALO"):
        halo.select_transport(lat)
    monkeypatch.setenv("LBM_B200_HALO", "nccl")
    assert halo.select_transport(lat) == "staged"      # single process: nothing to exchange
