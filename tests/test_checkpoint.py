"""Buddy checkpoints (reference
blockforest/checkpoint.py:23-109) on world_size 2 and 4 over gloo (CPU):
stride groups, image exchange, adoption plan, roll-back and adoption of a
lost rank's blocks, and the unrecoverable case."""
import numpy as np
import pytest

import paper_1909_13772_b200 as P


def _forest(ctx):
    f = P.create_forest(ctx, (0, 0, 0, 1, 1, ctx.n_ranks), (1, 1, ctx.n_ranks),
                        periodic=(True, True, False), cells_per_block=(4, 3, 2))
    f.register_data("rho", P.FieldDataHandler(nf=1, ghost_layers=1))
    for b in f.local_blocks():
        b.data["rho"].interior[..., 0] = 100.0 * b.id.root + np.arange(24).reshape(2, 3, 4)
    return f


def _prog(ctx, group_size, failed):
    f = _forest(ctx)
    cp = P.BuddyCheckpoint(ctx, group_size)
    before = {b.id.root: b.data["rho"].interior.copy() for b in f.local_blocks()}
    cp.save(f, 7)
    held = sorted(cp._images)
    for b in f.local_blocks():                     # state drifts after the save
        b.data["rho"].interior[...] = -1.0
    step, plan = cp.recover(f, failed=failed)
    after = {b.id.root: b.data["rho"].interior.copy() for b in f.local_blocks()}
    return {"held": held, "step": step, "plan": plan, "before": before, "after": after,
            "group": cp.group_of(ctx.rank), "bytes": cp.memory_bytes()}


@pytest.mark.parametrize("n,group_size,failed", [(2, 2, ()), (2, 2, (1,)), (4, 2, (1,)),
                                                 (4, 2, (0, 3)), (4, 4, (1, 2, 3))])
def test_save_recover_and_adopt(n, group_size, failed):
    res = P.run(n, _prog, group_size, failed, backend="gloo")
    n_groups = n // group_size
    blocks = {}
    for rank, r in enumerate(res):
        assert r["group"] == rank % n_groups
        assert r["held"] == list(range(rank % n_groups, n, n_groups))   # saved before the loss
        assert r["step"] == 7
        for root, arr in r["after"].items():
            assert root not in blocks
            blocks[root] = arr
        if rank in failed:
            assert r["after"] == {}
    # every block is back, exactly once, with its saved values
    assert sorted(blocks) == list(range(n))
    saved = {root: arr for r in res for root, arr in r["before"].items()}
    for root, arr in blocks.items():
        assert np.array_equal(arr, saved[root])
    for dead in failed:
        adopter = res[0]["plan"][dead]
        assert adopter not in failed and adopter % n_groups == dead % n_groups


def _lost_group(ctx):
    f = _forest(ctx)
    cp = P.BuddyCheckpoint(ctx, 2)
    cp.save(f, 1)
    try:
        cp.recover(f, failed=(0, 2))             # group 0 = {0, 2} lost entirely
    except P.UnrecoverableError as exc:
        return str(exc)
    return None


def test_lost_group_is_unrecoverable():
    res = P.run(4, _lost_group, backend="gloo")
    assert all(r and "group 0" in r for r in res)


def test_group_size_must_divide_ranks():
    with pytest.raises(P.ValidationError):
        P.BuddyCheckpoint(P.Context(device="cpu"), 3)
    cp = P.BuddyCheckpoint(P.Context(device="cpu"), 1)
    with pytest.raises(P.UnrecoverableError):
        cp.recover(_forest(P.Context(device="cpu")))
