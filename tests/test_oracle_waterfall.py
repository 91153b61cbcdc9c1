"""Pins for oracle.waterfall (O6-O7, readings C12-C17): an independent Kruskal-MST waterfall
(O8), a first-principles level-1 rule from brute-force newmin (Alg. 4), a hand-derived
example, and the hierarchy invariants (nesting, monotone counts, halving)."""
import json
import os

import numpy as np
import pytest

import oracle
import synth
from paper_literal import as_list, kruskal_waterfall, level1_by_partner, neighbour_table


def _levels(I, conn, ndim, NL):
    lab = oracle.watershed(I, conn, ndim=ndim)
    lv, counts = oracle.waterfall(lab, I, conn, NL, ndim=ndim)
    return lab, lv, counts


def test_hand_example_1d():
    """[0,3,1,5,10,2,1,7,0]: basins {0,1},{2,3},{4,5,6},{7,8}; pass heights 3 (0|2), 10 (2|4),
    7 (4|7); each basin merges along its lowest pass (C13) -> level 1 {0..3},{4..8}
    (the literal reconstruction would split {4,5,6} instead)."""
    I = np.array([[[0, 3, 1, 5, 10, 2, 1, 7, 0]]], np.uint8)
    lab, lv, counts = _levels(I, 4, 2, 3)
    assert as_list(lab) == [0, 0, 2, 2, 4, 4, 4, 7, 7]
    assert as_list(lv[1]) == [0, 0, 0, 0, 4, 4, 4, 4, 4]
    assert as_list(lv[2]) == [0] * 9
    assert list(counts) == [4, 2, 1]


def test_spec_two_basins():
    """[75, 89, 89, 81] -> two basins whose lowest pass is 89; one region at
    level 1; a single-region image stays as is (C17)."""
    I = np.array([[[75, 89, 89, 81]]], np.uint8)
    lab, lv, counts = _levels(I, 4, 2, 4)
    assert as_list(lab) == [0, 0, 2, 2]
    assert list(counts) == [2, 1, 1, 1]
    I = np.full((1, 4, 4), 9, np.uint8)
    _, lv, counts = _levels(I, 4, 2, 3)
    assert list(counts) == [1, 1, 1] and np.all(lv == 0)


def test_nl1_is_the_watershed():
    I = synth.random_plateau_image((1, 9, 9), 5, seed=3).numpy()
    lab, lv, counts = _levels(I, 8, 2, 1)
    assert lv.shape[0] == 1 and np.array_equal(lv[0], lab)


@pytest.mark.parametrize("shape,conn,ndim", [((1, 9, 9), 4, 2), ((1, 8, 11), 8, 2), ((3, 4, 5), 6, 3),
                                             ((3, 3, 4), 26, 3), ((1, 1, 30), 4, 2)])
def test_kruskal_and_level1_rule(shape, conn, ndim):
    rng = np.random.default_rng(100 + conn)
    nbrs = neighbour_table(shape, conn, ndim)
    for _ in range(60):
        I = rng.integers(0, int(rng.integers(3, 12)), size=shape).astype(np.uint8)
        lab, lv, counts = _levels(I, conn, ndim, 6)
        ref = kruskal_waterfall(as_list(lab), as_list(I), nbrs, 6)
        for k in range(6):
            assert as_list(lv[k]) == ref[k], k
        assert as_list(lv[1]) == level1_by_partner(as_list(lab), as_list(I), nbrs)


def _check_invariants(lv, counts, nimg=1):
    NL = lv.shape[0]
    flat = lv.reshape(NL, -1)
    for k in range(NL):
        u = np.unique(flat[k])
        assert counts[k] == u.size
        assert np.all(flat[k][flat[k]] == flat[k])  # canonical: label is a member index
        assert np.all(flat[k] <= np.arange(flat.shape[1]))
    for k in range(NL - 1):
        # nesting: the map level-k label -> level-(k+1) label is a function
        pairs = np.unique(np.stack([flat[k], flat[k + 1]]), axis=1)
        assert np.unique(pairs[0]).size == pairs.shape[1]
        assert counts[k + 1] <= counts[k]
        if counts[k] > nimg:  # halving (every component merges with >= 1 other)
            assert counts[k + 1] <= counts[k] - (counts[k] - nimg + 1) // 2


@pytest.mark.parametrize("name,shape", [("C1", None), ("C3", (24, 28, 30)), ("C4", (20, 32, 32)),
                                        ("C5", (3, 145, 145)), ("C2", (1, 160, 192))])
def test_invariants_on_config_workloads(name, shape):
    c = synth.CONFIGS[name]
    raw = synth.make_config_image(name, shape=shape).numpy()
    _, _, q = oracle.gradient(raw, c.sigma, ndim=c.ndim)
    lab, lv, counts = _levels(q, c.conn, c.ndim, c.NL)
    _check_invariants(lv, counts, nimg=q.shape[0] if c.ndim == 2 else 1)


def test_table5_ratio_sanity_band():
    """Per-level coarsening on a C1-shaped image vs the paper's Table 5 ratios (5.9-7.4x,
    P:896-916): a loose sanity band only, never a parity value."""
    with open(os.path.join(os.path.dirname(__file__), "golden", "sec5_table5_ratios.json")) as f:
        t5 = json.load(f)
    paper = np.array(t5["column_4096"][:3], float)
    c = synth.CONFIGS["C1"]
    raw = synth.make_config_image("C1").numpy()
    _, _, q = oracle.gradient(raw, c.sigma, ndim=2)
    _, _, counts = _levels(q, 4, 2, 3)
    ours = counts[0] / counts[1]
    assert 0.4 * (paper[0] / paper[1]) < ours < 2.5 * (paper[0] / paper[1])
