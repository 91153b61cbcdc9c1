"""Pins of oracle O9, the paper-literal waterfall by image reconstruction (Alg. 4 steps V-VI +
the watershed re-run per layer, Alg. 5): a 1-D example worked by hand from
the algorithm text (tests/golden/), closed-form special cases, and invariants the paper
states (the transform coarsens until one region per image)."""
import json
import os

import numpy as np
import pytest

import oracle
import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_hand_example_alg4_alg5():
    d = json.load(open(os.path.join(GOLDEN, "waterfall_reconstruct_hand.json")))
    I = np.array([d["image"]], np.uint8)
    lab = oracle.watershed(I, d["conn"], ndim=2)
    assert lab.ravel().tolist() == d["levels"][0]
    lv, counts = oracle.waterfall_reconstruct(lab, I, d["conn"], len(d["levels"]), ndim=2)
    assert lv.reshape(len(d["levels"]), -1).tolist() == d["levels"]
    assert counts.tolist() == d["counts"]


def test_two_basins_merge_at_their_pass():
    """[0, 5, 0]: two basins, both with lowest pass 5; raised to 5 the image is flat."""
    I = np.array([[0, 5, 0]], np.uint8)
    lab = oracle.watershed(I, 4, ndim=2)
    assert lab.ravel().tolist() == [0, 1, 1]  # Eq. 1: the max-index minimum wins the tie
    lv, counts = oracle.waterfall_reconstruct(lab, I, 4, 3, ndim=2)
    assert lv[1].ravel().tolist() == [0, 0, 0] and counts.tolist() == [2, 1, 1]


@pytest.mark.parametrize("conn,ndim", [(4, 2), (6, 3)])
def test_single_region_stays(conn, ndim):
    """A region without neighbours keeps newmin = M: raised to M it stays one region."""
    I = np.full((3, 5, 7), 9, np.uint8) if ndim == 3 else np.full((1, 6, 9), 9, np.uint8)
    lab = oracle.watershed(I, conn, ndim=ndim)
    lv, counts = oracle.waterfall_reconstruct(lab, I, conn, 4, ndim=ndim)
    assert np.all(lv == 0) and counts.tolist() == [1, 1, 1, 1]


def test_batch_images_stay_independent():
    """Batched 2-D images (C18): layer k of the batch = layer k of each image alone."""
    g = synth.random_plateau_image((3, 17, 23), 5, seed=3).numpy()
    lab = oracle.watershed(g, 4, ndim=2)
    lv, _ = oracle.waterfall_reconstruct(lab, g, 4, 4, ndim=2)
    n = 17 * 23
    for b in range(3):
        one = g[b:b + 1]
        l1 = oracle.watershed(one, 4, ndim=2)
        lv1, _ = oracle.waterfall_reconstruct(l1, one, 4, 4, ndim=2)
        assert np.array_equal(lv[:, b], lv1[:, 0] + b * n)


@pytest.mark.parametrize("conn,ndim,shape", [(4, 2, (1, 40, 50)), (8, 2, (1, 33, 41)), (6, 3, (9, 14, 17)),
                                             (26, 3, (7, 11, 13))])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_coarsening_invariants(conn, ndim, shape, seed):
    """Counts never increase (every new basin holds a regional minimum of the raised image,
    which lies on a raised old basin) and reach one region per connected image;
    every layer is canonical (label = smallest voxel index of its region, C7)."""
    g = synth.random_plateau_image(shape, 12, seed=seed + conn).numpy()
    lab = oracle.watershed(g, conn, ndim=ndim)
    NL = 40
    lv, counts = oracle.waterfall_reconstruct(lab, g, conn, NL, ndim=ndim)
    assert all(counts[k + 1] <= counts[k] for k in range(NL - 1))
    assert counts[-1] == 1
    for k in range(NL):
        f = lv[k].ravel()
        first = {}
        for p, l in enumerate(f):
            first.setdefault(l, p)
        assert all(first[l] == l for l in first)
