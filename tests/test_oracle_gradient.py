"""Pins for oracle.gradient (O1-O2, readings C8-C10): SciPy / NumPy library routines in
fp64 and closed forms.  None of these re-type the oracle's loops."""
import math

import numpy as np
import pytest
import scipy.ndimage as ndi

import oracle


def _scipy_ref(img, sigma, ndim):
    x = img.astype(np.float64) / 255.0
    if ndim == 3:
        b = ndi.gaussian_filter(x, sigma, mode="nearest", truncate=3.0) if sigma > 0 else x
        axes = (0, 1, 2)
    else:  # batch of 2D images: blur and differentiate in-plane only (C18)
        b = np.stack([ndi.gaussian_filter(im, sigma, mode="nearest", truncate=3.0) if sigma > 0 else im
                      for im in x])
        axes = (1, 2)
    s = np.zeros_like(b)
    for ax in axes:
        if b.shape[ax] >= 2:
            s += np.gradient(b, axis=ax, edge_order=1) ** 2
    return b, np.sqrt(s)


@pytest.mark.parametrize("shape,ndim,sigma", [((1, 37, 29), 2, 1.0), ((3, 16, 21), 2, 1.5), ((9, 10, 11), 3, 1.0),
                                              ((7, 12, 5), 3, 0.7), ((1, 30, 1), 2, 1.0), ((1, 13, 17), 2, 0.0)])
def test_matches_scipy_numpy(shape, ndim, sigma):
    rng = np.random.default_rng(11)
    img = rng.integers(0, 256, size=shape).astype(np.uint8)
    blur, grad, q = oracle.gradient(img, sigma, ndim=ndim)
    rb, rg = _scipy_ref(img, sigma, ndim)
    assert np.max(np.abs(blur - rb)) < 1e-12
    assert np.max(np.abs(grad - rg)) < 1e-12
    assert np.array_equal(q, np.minimum(255, np.floor(255 * rg + 0.5)).astype(np.uint8))


def test_closed_forms():
    # constant image -> zero gradient
    _, g, q = oracle.gradient(np.full((1, 20, 20), 93, np.uint8), 1.0)
    assert np.all(g == 0) and np.all(q == 0)
    # linear ramp, slope s per pixel -> interior 255*g == s, any sigma (blur of a
    # linear function is linear away from the clamped border)
    s = 2
    img = (np.arange(64, dtype=np.int64) * s).astype(np.uint8)[None, None, :].repeat(3, 1)
    _, g, q = oracle.gradient(img, 1.0)
    assert np.allclose(255 * g[0, :, 5:-5], s, atol=1e-12)
    assert np.all(q[0, :, 5:-5] == s)
    # unit impulse -> blur = separable product of the sampled, normalised Gaussian
    img = np.zeros((1, 15, 15), np.uint8)
    img[0, 7, 7] = 255
    b, _, _ = oracle.gradient(img, 1.0)
    w = np.exp(-np.arange(-3, 4) ** 2 / 2.0)
    w /= w.sum()
    assert abs(b[0, 7, 7] - w[3] * w[3]) < 1e-15
    assert abs(b[0, 7, 9] - w[3] * w[5]) < 1e-15
    assert b[0, 7, 11] == 0.0  # outside radius r = floor(3*1 + 0.5) = 3
    # sigma = 0 is the identity blur
    rng = np.random.default_rng(0)
    img = rng.integers(0, 256, size=(2, 6, 7)).astype(np.uint8)
    b, _, _ = oracle.gradient(img, 0.0)
    assert np.array_equal(b, img / 255.0)


def test_radius_rule():
    # r = floor(3 sigma + 0.5): sigma=0.5 -> r=2 (reach 2 px), not ceil(1.5)=2 ... sigma=0.4 -> r=1
    img = np.zeros((1, 1, 11), np.uint8)
    img[0, 0, 5] = 255
    b, _, _ = oracle.gradient(img, 0.4)
    assert b[0, 0, 4] > 0 and b[0, 0, 3] == 0.0
    assert math.floor(3 * 0.4 + 0.5) == 1


def test_mirror_symmetry():
    rng = np.random.default_rng(5)
    img = rng.integers(0, 256, size=(6, 7, 8)).astype(np.uint8)
    _, g, _ = oracle.gradient(img, 1.0, ndim=3)
    _, gm, _ = oracle.gradient(img[:, :, ::-1].copy(), 1.0, ndim=3)
    assert np.allclose(g[:, :, ::-1], gm, atol=1e-13)


def test_invalid():
    with pytest.raises(ValueError):
        oracle.gradient(np.zeros((1, 3, 3), np.uint8), -1.0)
