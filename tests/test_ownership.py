"""Root ownership and neighbour records vs the reference (CPU).

tests/golden/ownership.json holds the reference's own partition_curve
results for unit weights (balance.py:132-167) and, for a set of root grids
and rank counts, every rank's blocks and neighbour records from its
create_forest (forest.py:414-449, 226-260).  balance.py / blockforest.py
compute them differently (closed-form segment ends, LSB-first Morton
interleave) and must agree exactly.
"""
import json
from pathlib import Path

import pytest

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "ownership.json").read_text())


def test_unit_weight_partition_matches_reference():
    from paper_1909_13772_b200 import balance
    for key, want in GOLD["partition"].items():
        n, p = (int(v) for v in key.split(","))
        assert balance.owners_along_curve(n, p) == want, key


@pytest.mark.parametrize("k", range(len(GOLD["forests"])))
def test_forest_ownership_and_neighbours_match_reference(k):
    import paper_1909_13772_b200 as P
    spec = GOLD["forests"][k]
    dims, d, per, ranks = tuple(spec["dims"]), spec["d"], tuple(spec["periodic"]), spec["ranks"]

    class Ctx:
        def __init__(self, rank):
            self.rank, self.n_ranks = rank, ranks

    for rank in range(ranks):
        f = P.create_forest(Ctx(rank), (0, 0, 0) + tuple(float(v) for v in dims), dims, d=d,
                            periodic=per, cells_per_block=(2, 2, 2 if d == 3 else 1))
        got = [[b.id.root, [[list(r.direction), r.block_id.root, r.rank, list(r.shift)]
                            for r in b.neighbors]] for b in f.local_blocks()]
        assert got == spec["blocks"][str(rank)], (dims, rank)


def test_zslab_rank_k_owns_slab_k():
    import paper_1909_13772_b200 as P
    for n in (1, 2, 3, 4, 8):
        for rank in range(n):
            class Ctx:
                pass
            c = Ctx()
            c.rank, c.n_ranks = rank, n
            f = P.create_forest(c, (0, 0, 0, 1, 1, n), (1, 1, n), periodic=(True, True, False),
                                cells_per_block=(4, 4, 4))
            [b] = f.local_blocks()
            assert f.cell_box(b.id) == ((0, 0, 4 * rank), (4, 4, 4 * rank + 4))
