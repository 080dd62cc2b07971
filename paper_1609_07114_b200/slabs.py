"""Row-slab decomposition helpers (host logic of DESIGN.md "Multi-GPU").

Rank g of N owns coarse cell rows [g*ny//N, (g+1)*ny//N) and the Ex edge rows of the same range.
A ROM instance belongs to the slab that contains its footprint plus one-cell ring (R19); an
instance that straddles a slab boundary is a placement error (the generator never emits one).
"""
from __future__ import annotations

import numpy as np


def slab_rows(ny, nranks, rank):
    return rank * ny // nranks, (rank + 1) * ny // nranks


def owned_placements(placements, models, row_begin, row_end):
    """Placements (model, i0, j0) whose footprint + ring rows j0-1 .. j0+by lie in [row_begin, row_end)."""
    if placements is None or len(placements) == 0:
        return np.zeros((0, 3), dtype=np.int32)
    P = np.asarray(placements)
    by = np.array([models[k]["by"] for k in P[:, 0]])
    keep = (P[:, 2] - 1 >= row_begin) & (P[:, 2] + by <= row_end - 1)
    return P[keep]


def check_partition(placements, models, ny, nranks):
    """Every placement is owned by exactly one slab."""
    n = 0
    for g in range(nranks):
        rb, re = slab_rows(ny, nranks, g)
        n += len(owned_placements(placements, models, rb, re))
    return n == (0 if placements is None else len(placements))
