"""Host logic of the fix-up clusters (fdtd_pass_regions; -m "not gpu"):
the regions partition the instances, no two regions' boxes grown by the pass depth meet, each box is
exactly its members' bounding box, instances whose grown blocks meet share a region, and depth 1
keeps one region per instance."""
import numpy as np
import pytest

from inputs import scene as sc


def _meet(a, b, K):
    return a[0] - K < b[0] + b[2] + K and b[0] - K < a[0] + a[2] + K and \
        a[1] - K < b[1] + b[3] + K and b[1] - K < a[1] + a[3] + K


@pytest.mark.parametrize("K", [1, 2, 4])
@pytest.mark.parametrize("seed", [5, 7, 11])
def test_regions_partition_and_separation(K, seed):
    from paper_1609_07114_b200 import pass_regions
    P = sc.place_blocks(192, 192, [(6, 6), (4, 8)], 50, seed, nslabs=1, margin=1, clear=1)
    rects = np.array([[i0, j0, *[(6, 6), (4, 8)][m]] for m, i0, j0 in P], np.int32)
    reg, boxes = pass_regions(rects, P[:, 0], K)
    assert reg.min() >= 0 and reg.max() == len(boxes) - 1
    if K == 1:
        assert len(boxes) == len(P)
    for g, b in enumerate(boxes):
        mem = rects[reg == g]
        assert len(mem) >= 1
        assert b[0] == mem[:, 0].min() and b[1] == mem[:, 1].min()
        assert b[0] + b[2] == (mem[:, 0] + mem[:, 2]).max() and b[1] + b[3] == (mem[:, 1] + mem[:, 3]).max()
        assert b[4] == (len(set(P[reg == g, 0])) > 1)
    if K >= 2:
        for a in range(len(boxes)):
            for c in range(a + 1, len(boxes)):
                assert not _meet(boxes[a], boxes[c], K)
        for a in range(len(rects)):
            for c in range(a + 1, len(rects)):
                if _meet(rects[a], rects[c], K):
                    assert reg[a] == reg[c]


def test_regions_chain_merges_through_bounding_box():
    """An L-shaped pair whose bounding box reaches a third block that neither member meets: the
    iterated merge takes the third block in (its region would otherwise lie inside the pair's
    fix-up region)."""
    from paper_1609_07114_b200 import pass_regions
    K = 4
    rects = np.array([[10, 10, 6, 6], [18, 18, 6, 6], [26, 2, 6, 6]], np.int32)
    assert _meet(rects[0], rects[1], K) and not _meet(rects[0], rects[2], K) and not _meet(rects[1], rects[2], K)
    reg, boxes = pass_regions(rects, [0, 0, 0], K)
    assert len(boxes) == 1 and (reg == 0).all()
