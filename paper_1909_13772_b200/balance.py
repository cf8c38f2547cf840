"""Rank ownership of the root blocks.

`create_forest` hands root blocks to ranks in two steps (reference:
pkg/src/blocksim/blockforest/forest.py:439-447 calling balance.py:101-167):
order the blocks along a Morton curve, then cut the curve into one
consecutive segment per rank with every block weighing one.  This module
computes the same map directly:

* the Morton position of root (x, y, z) is its bits interleaved x-y-z from
  the least significant end (bit b of x -> 3b, of y -> 3b+1, of z -> 3b+2;
  d = 2 drops z), which orders blocks exactly like the reference's
  most-significant-first key of a common bit width;
* with unit weights the reference's greedy cut (close a segment at the
  prefix nearest k * n / P, ties taken) ends segment k at
  round-half-up(n (k + 1) / P) = (2 n (k + 1) + P) // (2 P), in integers.

For root_dims = (1, 1, P) this gives rank k the z-slab k.  Both rules are
checked against the reference's own outputs (tests/golden/ownership.json).
"""
from __future__ import annotations

from .errors import ValidationError


def _interleave(v: int, stride: int, lane: int) -> int:
    out, b = 0, 0
    while v:
        if v & 1:
            out |= 1 << (b * stride + lane)
        v >>= 1
        b += 1
    return out


def morton_position(coords, d: int) -> int:
    """Curve key of root coordinates (x, y[, z])."""
    return sum(_interleave(int(coords[a]), d, a) for a in range(d))


def curve_order(coords_of, d: int, curve: str = "morton"):
    """Items sorted along the space-filling curve; coords_of: {item: coords}."""
    if curve != "morton":
        raise ValidationError(f"curve {curve!r} is not supported on the B200 path (morton only)")
    return sorted(coords_of, key=lambda item: morton_position(coords_of[item], d))


def segment_ends(n_blocks: int, n_ranks: int):
    """End (exclusive) of each rank's segment of n_blocks unit-weight
    blocks along the curve."""
    if n_ranks < 1:
        raise ValidationError(f"n_ranks must be >= 1, got {n_ranks}")
    ends = [(2 * n_blocks * (k + 1) + n_ranks) // (2 * n_ranks) for k in range(n_ranks - 1)]
    return ends + [n_blocks]


def owners_along_curve(n_blocks: int, n_ranks: int):
    """Rank of each curve position."""
    out, start = [], 0
    for rank, end in enumerate(segment_ends(n_blocks, n_ranks)):
        out.extend([rank] * (end - start))
        start = end
    return out
