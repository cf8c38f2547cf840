"""Space-filling-curve ordering and curve partitioning of root blocks.

Restates the two routines `create_forest` uses to assign blocks to ranks
(pkg/src/blocksim/balance.py:31-41 morton_key, :101-129 sort_blocks,
:132-167 partition_curve) so the rank <-> block map is the reference's.  With
root_dims = (1, 1, P) rank k owns z-slab k.
"""
from __future__ import annotations

from .errors import ValidationError


def morton_key(coords, level: int, d: int, bits: int) -> int:
    x, y, z = (int(c) for c in coords)
    key = 0
    for b in range(bits - 1, -1, -1):
        if d == 3:
            key = (key << 3) | (((z >> b) & 1) << 2) | (((y >> b) & 1) << 1) | ((x >> b) & 1)
        else:
            key = (key << 2) | (((y >> b) & 1) << 1) | ((x >> b) & 1)
    return key


def sort_blocks(entries, curve: str, d: int):
    """Payloads of (coords, level, payload) entries in Morton order."""
    entries = list(entries)
    if not entries:
        return []
    if curve != "morton":
        raise ValidationError(f"curve {curve!r} is not supported on the B200 path (morton only)")
    finest = max(level for _, level, _ in entries)
    maxc = 0
    for coords, level, _ in entries:
        lift = finest - level
        maxc = max(maxc, *(int(c) << lift for c in coords[:d]))
    bits = max(1, maxc.bit_length())
    keyed = []
    for coords, level, payload in entries:
        lift = finest - level
        lifted = tuple(int(c) << lift for c in coords)
        keyed.append((morton_key(lifted, finest, d, bits), payload))
    keyed.sort(key=lambda kv: kv[0])
    return [payload for _, payload in keyed]


def partition_curve(weights, n_ranks: int):
    """Consecutive per-rank segments closing at the prefix sum nearest to
    k * total / n_ranks (balance.py:132-167)."""
    weights = [float(w) for w in weights]
    if n_ranks < 1:
        raise ValidationError(f"n_ranks must be >= 1, got {n_ranks}")
    if any(w < 0 for w in weights):
        raise ValidationError("block weights must be non-negative")
    n = len(weights)
    assignment = [0] * n
    total = sum(weights)
    if n == 0 or total == 0.0:
        for i in range(n):
            assignment[i] = i * n_ranks // n
        return assignment
    prefix = 0.0
    i = 0
    for rank in range(n_ranks - 1):
        target = total * (rank + 1) / n_ranks
        while i < n:
            candidate = prefix + weights[i]
            if abs(candidate - target) <= abs(prefix - target):
                assignment[i] = rank
                prefix = candidate
                i += 1
            else:
                break
    for j in range(i, n):
        assignment[j] = n_ranks - 1
    return assignment
