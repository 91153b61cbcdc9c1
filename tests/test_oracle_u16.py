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


# ---- O11: the 16-bit gradient (x / 65535, q = min(65535, floor(65535 g + 0.5)))
@pytest.mark.parametrize("sigma", [0.0, 0.6, 1.0, 2.0])
@pytest.mark.parametrize("ndim,shape", [(2, (2, 9, 14)), (3, (6, 7, 9))])
def test_u8_widened_by_257_has_the_same_blur_and_gradient(sigma, ndim, shape):
    """img / 255 == (257 img) / 65535 exactly, so blur and g equal the pinned u8 oracle's."""
    rng = np.random.default_rng(int(sigma * 10) + ndim)
    a = rng.integers(0, 256, shape).astype(np.uint8)
    b8, g8, _ = oracle.gradient(a, sigma, ndim=ndim)
    b16, g16, q16 = oracle.gradient(a.astype(np.uint16) * 257, sigma, ndim=ndim)
    assert np.max(np.abs(b8 - b16)) <= 1e-12 and np.max(np.abs(g8 - g16)) <= 1e-12
    assert q16.dtype == np.uint16


@pytest.mark.parametrize("slope", [1, 37, 1234])
def test_ramp_closed_form_16bit(slope):
    """img = slope * x: central and one-sided differences both give g = slope / 65535, so
    q = slope exactly (no blur); with a symmetric normalised blur the ramp is preserved away
    from the clamped ends, so the interior keeps q = slope."""
    n = 48
    img = (np.arange(n, dtype=np.int64) * slope).astype(np.uint16).reshape(1, 1, n)
    _, g, q = oracle.gradient(img, 0.0, ndim=2)
    assert np.all(q == slope)
    assert np.allclose(g, slope / 65535.0, rtol=0, atol=1e-15)
    _, g1, q1 = oracle.gradient(img, 1.0, ndim=2)  # r = 3: x in [4, n - 5] is interior
    assert np.all(q1.ravel()[4:n - 4] == slope)
    vol = np.broadcast_to(img.reshape(1, 1, n), (5, 6, n)).copy()
    _, _, q3 = oracle.gradient(vol, 0.0, ndim=3)  # constant along z and y: d0 = d1 = 0
    assert np.all(q3 == slope)


def test_steep_ramp_clips_at_65535():
    img = np.array([[0, 65535, 0, 65535]], np.uint16)
    _, g, q = oracle.gradient(img, 0.0, ndim=2)
    assert q.tolist() == [[65535, 0, 0, 65535]]  # one-sided ends g = 1; centres (b[x+1]-b[x-1])/2 = 0
    chk = np.array([[0, 65535], [65535, 0]], np.uint16)  # |dx| = |dy| = 1 everywhere: g = sqrt 2
    _, g2, q2 = oracle.gradient(chk, 0.0, ndim=2)
    assert np.allclose(g2, np.sqrt(2.0)) and np.all(q2 == 65535)  # clipped (C10 at 16 bits)


# ---- O12: the 16-bit waterfall (pass heights max(I(p), I(q)) as u16, K of C14)
@pytest.mark.parametrize("conn,shape", [(4, (3, 17, 23)), (8, (2, 19, 21)), (6, (7, 9, 11)), (26, (5, 8, 9))])
@pytest.mark.parametrize("nlev", [4, 40, 256])
def test_waterfall_monotone_invariance_vs_u8_oracle(conn, shape, nlev):
    """The waterfall compares pass heights only (max of two intensities, the per-pair min,
    then K), so a strictly increasing map of the intensities leaves every level unchanged:
    the u16 levels equal the (separately pinned) u8 oracle's on the rank image."""
    rng = np.random.default_rng(2000 + conn * 7 + nlev)
    table = np.sort(rng.choice(65536, size=nlev, replace=False)).astype(np.uint16)
    img = table[rng.integers(0, nlev, shape)]
    ndim = 3 if conn in (6, 26) else 2
    r8 = _rank_u8(img)
    lab = oracle.watershed(img, conn, ndim=ndim)
    lv16, c16 = oracle.waterfall(lab, img, conn, 6, ndim=ndim)
    lv8, c8 = oracle.waterfall(oracle.watershed(r8, conn, ndim=ndim), r8, conn, 6, ndim=ndim)
    assert np.array_equal(lv16, lv8) and list(c16) == list(c8)


@pytest.mark.parametrize("shape,conn,ndim", [((1, 9, 9), 4, 2), ((1, 8, 11), 8, 2), ((3, 4, 5), 6, 3),
                                             ((3, 3, 4), 26, 3)])
def test_waterfall_u16_vs_kruskal_mst(shape, conn, ndim):
    """O8 (independent Kruskal-MST waterfall) on images with many more than 256
    distinct 16-bit values, so no u8 reduction is involved."""
    from paper_literal import as_list, kruskal_waterfall, neighbour_table
    rng = np.random.default_rng(300 + conn)
    nbrs = neighbour_table(shape, conn, ndim)
    for _ in range(30):
        img = rng.integers(0, 65536, size=shape).astype(np.uint16)
        lab = oracle.watershed(img, conn, ndim=ndim)
        lv, counts = oracle.waterfall(lab, img, conn, 6, ndim=ndim)
        ref = kruskal_waterfall(as_list(lab), as_list(img), nbrs, 6)
        for k in range(6):
            assert as_list(lv[k]) == ref[k], k


def test_waterfall_hand_case_needs_16_bits():
    # 1-D [0, 256, 10, 300, 20, 255, 30]: regions {0,1} {2,3} {4,5} {6} (each wall descends to
    # its smaller neighbour, Eq. 1); pass heights 256 (R0-R2), 300 (R2-R4), 255 (R4-R6).  Level
    # 1: R0 and R2 pick 256, R4 and R6 pick 255, the 300 pass is never picked -> {0..3} {4..6}.
    # Clipped to 255 all three passes tie and K's max-label tie-break chains them into one
    # region; wrapped to 8 bits the watershed itself differs.
    a = np.array([[0, 256, 10, 300, 20, 255, 30]], np.uint16)
    lab = oracle.watershed(a, 4, ndim=2)
    assert lab.tolist() == [[0, 0, 2, 2, 4, 4, 6]]
    lv, counts = oracle.waterfall(lab, a, 4, 3, ndim=2)
    assert lv[1].tolist() == [[0, 0, 0, 0, 4, 4, 4]] and lv[2].tolist() == [[0] * 7]
    assert list(counts) == [4, 2, 1]
