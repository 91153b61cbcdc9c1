"""Pins for oracle.watershed (O3-O4) — independent of the oracle's own code.

* the paper's worked examples (tests/golden)
* literal Alg. 1 (tests/paper_literal.py) on exhaustive tiny images and random images
* #regions == #regional minima (flood fill), closed-form special cases
"""
import itertools
import json
import os

import numpy as np
import pytest

import oracle
from paper_literal import (alg1_pruf, alg3_balanced, as_list, canonical, count_regional_minima,
                           neighbour_table, step3_iterations)

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def test_sec3_3_worked_example():
    g = _gold("sec3_3_long_plateau.json")
    I = np.array(g["image"], np.uint8).reshape(1, 1, -1)
    nbrs = neighbour_table((1, 1, len(g["image"])), 4, 2)
    tr = {}
    raw = alg1_pruf(as_list(I), nbrs, trace=tr)
    # the literal algorithm reproduces the printed states/iterations (pins the helper)
    assert tr["S1"] == g["states_step1"]
    assert tr["it2"] == g["step2_iterations"]
    assert tr["S2_hist"][g["n"] - 3] == g["states_after_n_minus_2_iterations"]
    assert tr["L2"][1:-1] == g["parent_after_step2"][1:-1]
    # the oracle: parent pointers after step II and the 6/6 split
    lab, dist, ptr, R = oracle.watershed(I, 4, dumps=True)
    assert as_list(ptr) == g["parent_after_step2"]
    assert R == g["n_regions"]
    assert as_list(lab) == [0] * 6 + [6] * 6
    assert canonical(raw) == as_list(lab)


def test_sec3_4_balanced_fixpoint():
    g = _gold("sec3_4_balanced.json")
    hist = alg3_balanced(g["image"], g["block"])
    assert hist[0] == g["states_iter1"]
    assert hist[1] == g["states_iter2"]
    assert hist[2] == g["states_iter3"]
    I = np.array(g["image"], np.uint8).reshape(1, 1, -1)
    _, dist, _, _ = oracle.watershed(I, 4, dumps=True)
    fix = g["states_iter3"]
    # oracle BFS distance == |balanced fixpoint state| on the plateau (P:462 semantics)
    assert as_list(dist)[1:-1] == [abs(s) for s in fix[1:-1]]


def test_fig4_path_reduction_iterations():
    g = _gold("fig4_path_reduction.json")
    assert step3_iterations(g["length"], g["RR"]) == g["changing_iterations"]


def test_spec_step1_examples():
    # constant 5x5: Eq. 1 gives exactly one state-3 pixel, the last index; one region
    I = np.full((1, 5, 5), 7, np.uint8)
    tr = {}
    alg1_pruf(as_list(I), neighbour_table((1, 5, 5), 4, 2), trace=tr)
    assert [p for p, s in enumerate(tr["S1"]) if s == 3] == [24]
    assert set(as_list(oracle.watershed(I, 4))) == {0}
    # strictly increasing ramp: one minimum, one region
    I = np.array([[[1, 2, 3, 4]]], np.uint8)
    assert as_list(oracle.watershed(I, 4)) == [0, 0, 0, 0]
    # single voxel (C4)
    assert as_list(oracle.watershed(np.zeros((1, 1, 1), np.uint8), 4)) == [0]
    assert as_list(oracle.watershed(np.zeros((1, 1, 1), np.uint8), 6)) == [0]


def _exhaustive(shape, conn, ndim, values=3):
    n = int(np.prod(shape))
    imgs = np.array(list(itertools.product(range(values), repeat=n)), np.uint8)
    return imgs.reshape((-1,) + tuple(shape))


@pytest.mark.parametrize("conn", [4, 8])
def test_exhaustive_3x3_vs_literal_alg1(conn):
    imgs = _exhaustive((3, 3), conn, 2)  # 19683 images, one batched oracle call (C18)
    lab = oracle.watershed(imgs, conn, ndim=2)
    nbrs = neighbour_table((1, 3, 3), conn, 2)
    for i in range(imgs.shape[0]):
        raw = alg1_pruf(as_list(imgs[i]), nbrs)
        got = [v - 9 * i for v in as_list(lab[i])]
        assert got == canonical(raw), (conn, imgs[i])


@pytest.mark.parametrize("conn", [6, 26])
def test_exhaustive_2x2x2_vs_literal_alg1(conn):
    imgs = _exhaustive((2, 2, 2), conn, 3)  # 6561 volumes
    nbrs = neighbour_table((2, 2, 2), conn, 3)
    for i in range(imgs.shape[0]):
        lab = oracle.watershed(imgs[i], conn, ndim=3)
        assert as_list(lab) == canonical(alg1_pruf(as_list(imgs[i]), nbrs)), imgs[i]


@pytest.mark.parametrize("shape,conn,ndim", [((1, 1, 40), 4, 2), ((1, 11, 13), 4, 2), ((1, 12, 9), 8, 2),
                                             ((3, 7, 6), 4, 2), ((5, 6, 7), 6, 3), ((4, 5, 6), 26, 3)])
def test_random_vs_literal_alg1_and_minima_count(shape, conn, ndim):
    rng = np.random.default_rng(1234 + conn)
    nbrs = neighbour_table(shape, conn, ndim)
    for trial in range(40):
        levels = int(rng.integers(2, 9))
        I = rng.integers(0, levels, size=shape).astype(np.uint8)
        lab, dist, ptr, R = oracle.watershed(I, conn, ndim=ndim, dumps=True)
        assert as_list(lab) == canonical(alg1_pruf(as_list(I), nbrs))
        assert R == count_regional_minima(as_list(I), nbrs)
        labs = np.asarray(lab).ravel()
        assert np.all(labs <= np.arange(labs.size)) and np.all(labs[labs] == labs)


def test_depth1_volume_equals_2d():
    """C21 (SPEC S:250 is wrong): depth-1 3D with 6-conn == 2D 4-conn; 26 == 8."""
    rng = np.random.default_rng(7)
    for _ in range(60):
        I = rng.integers(0, 4, size=(1, 9, 11)).astype(np.uint8)
        assert np.array_equal(oracle.watershed(I, 6, ndim=3), oracle.watershed(I, 4, ndim=2))
        assert np.array_equal(oracle.watershed(I, 26, ndim=3), oracle.watershed(I, 8, ndim=2))


def test_batch_independence():
    """C18: a batch of 2D images == each image on its own, offset by its base index."""
    rng = np.random.default_rng(3)
    imgs = rng.integers(0, 5, size=(6, 8, 10)).astype(np.uint8)
    lab = oracle.watershed(imgs, 8, ndim=2)
    for b in range(6):
        one = oracle.watershed(imgs[b:b + 1], 8, ndim=2)
        assert np.array_equal(lab[b] - b * 80, one[0])


def test_invalid_arguments():
    with pytest.raises(ValueError):
        oracle.watershed(np.zeros((2, 2, 2), np.uint8), 4, ndim=3)
    with pytest.raises(ValueError):
        oracle.watershed(np.zeros((2, 2, 2), np.uint8), 6, ndim=2)
