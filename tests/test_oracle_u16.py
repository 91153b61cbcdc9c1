"""Pins of the 16-bit oracle watershed (O10, NEXT f4: 16-bit microCT).

The watershed is defined by comparisons of intensities only (Eq. 1, plateaux and
their BFS P:194-203, minimal plateaux P:316), so it is invariant under any strictly
increasing map of the intensities.  A u16 image with at most 256 distinct values therefore
has exactly the labels the (separately pinned) u8 oracle gives its rank image; hand cases
below fail if 16-bit values were clipped or wrapped to 8 bits."""
import numpy as np
import pytest

import oracle


def _rank_u8(a):
    vals, inv = np.unique(a, return_inverse=True)
    assert vals.size <= 256
    return inv.reshape(a.shape).astype(np.uint8)


@pytest.mark.parametrize("conn,shape", [(4, (3, 17, 23)), (8, (2, 19, 21)), (6, (7, 9, 11)), (26, (5, 8, 9))])
@pytest.mark.parametrize("nlev", [3, 12, 200])
def test_monotone_invariance_vs_u8_oracle(conn, shape, nlev):
    rng = np.random.default_rng(1000 + conn * 7 + nlev)
    table = np.sort(rng.choice(65536, size=nlev, replace=False)).astype(np.uint16)  # spread over 16 bits
    img = table[rng.integers(0, nlev, shape)]
    ndim = 3 if conn in (6, 26) else 2
    lab16, d16, p16, r16 = oracle.watershed(img, conn, ndim=ndim, dumps=True)
    lab8, d8, p8, r8 = oracle.watershed(_rank_u8(img), conn, ndim=ndim, dumps=True)
    assert np.array_equal(lab16, lab8) and np.array_equal(d16, d8) and np.array_equal(p16, p8) and r16 == r8


def test_hand_cases_need_16_bits():
    # 1-D rows (ndim 2, conn 4).  [256, 300, 255]: 256 has no lower neighbour (300 > 256) and
    # is a strict minimum; 300 descends to the smaller of 256 / 255 (Eq. 1) -> voxel 2; the
    # label is the smallest voxel index of the region (C7): [0, 1, 1].  Wrapped to 8 bits
    # ([0, 44, 255]) voxel 1 would descend to voxel 0 instead ([0, 0, 2]).
    a = np.array([[256, 300, 255]], np.uint16)
    assert oracle.watershed(a, 4, ndim=2).tolist() == [[0, 1, 1]]
    # [300, 256, 301, 257, 302]: two minima (256, 257); clipped to 255 all voxels would be
    # one plateau (one region).  301 descends to 256 (the smaller): regions {0,1,2}, {3,4}.
    b = np.array([[300, 256, 301, 257, 302]], np.uint16)
    assert oracle.watershed(b, 4, ndim=2).tolist() == [[0, 0, 0, 3, 3]]
    # full-range extremes: 65535 descends to 0 on both sides; 65534 is a strict minimum
    c = np.array([[65535, 0, 65535, 65534]], np.uint16)
    assert oracle.watershed(c, 4, ndim=2).tolist() == [[0, 0, 0, 3]]
