"""GPU parity of ws_watershed_u16 (NEXT f4, 16-bit images) against the 16-bit oracle
(O10), bit-exact labels and region counts; TMA (n2 % 8 == 0) and plain loaders; tiles
spanning several tiles with ragged tails; and u16 == u8 on order-isomorphic images."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu


def _ws():
    import paper_2410_08946_b200 as ws
    return ws


def _img(shape, kind, seed):
    rng = np.random.default_rng(seed)
    if kind == "few":  # plateau-heavy: a dozen levels spread over the 16-bit range
        return (rng.integers(0, 12, shape) * 5417 + 3).astype(np.uint16)
    if kind == "many":  # thousands of levels: plateaux almost only where the field is flat
        return rng.integers(0, 4000, shape).astype(np.uint16)
    # smooth field quantised to 16 bits (the f4 motivation: fine levels, small plateaux)
    f = rng.standard_normal(shape)
    for ax in range(len(shape)):
        f = (f + np.roll(f, 1, ax) + np.roll(f, -1, ax)) / 3
    f = (f - f.min()) / (np.ptp(f) + 1e-12)
    return np.floor(f * 65535).astype(np.uint16)


def _check(img, conn, ndim):
    ws = _ws()
    lab, R = ws.watershed(torch.from_numpy(img).cuda(), conn, ndim=ndim)
    ref, _, _, Rref = oracle.watershed(img, conn, ndim=ndim, dumps=True)
    got = lab.cpu().numpy()
    if not np.array_equal(got, ref):
        bad = np.flatnonzero(got.ravel() != ref.ravel())
        pytest.fail("u16 watershed mismatch at %d voxels, first %s" % (bad.size, bad[:5]))
    assert R == Rref


@pytest.mark.parametrize("kind", ["few", "many", "smooth"])
@pytest.mark.parametrize("conn,ndim,shape", [(6, 3, (19, 21, 70)), (26, 3, (11, 17, 40)), (6, 3, (9, 10, 33)),
                                             (4, 2, (2, 70, 130)), (8, 2, (3, 45, 67))])
def test_u16_parity(kind, conn, ndim, shape):
    _check(_img(shape, kind, hash((kind, conn, shape)) & 0xffff), conn, ndim)


@pytest.mark.parametrize("conn,ndim,shape", [(6, 3, (17, 24, 64)), (8, 2, (2, 64, 128))])
def test_u16_tma_and_plain_loader(conn, ndim, shape, monkeypatch):
    img = _img(shape, "few", 7)
    _check(img, conn, ndim)
    monkeypatch.setenv("WS_NO_TMA", "1")
    _check(img, conn, ndim)


@pytest.mark.parametrize("conn,ndim,shape", [(6, 3, (16, 40, 96)), (26, 3, (9, 16, 48)), (4, 2, (2, 96, 160))])
def test_u16_equals_u8_on_order_isomorphic_images(conn, ndim, shape):
    ws = _ws()
    rng = np.random.default_rng(5)
    img8 = rng.integers(0, 9, shape).astype(np.uint8)
    img16 = (img8.astype(np.uint16) * 7919 + 11).astype(np.uint16)  # strictly increasing map
    l8, r8 = ws.watershed(torch.from_numpy(img8).cuda(), conn, ndim=ndim)
    l16, r16 = ws.watershed(torch.from_numpy(img16).cuda(), conn, ndim=ndim)
    assert r8 == r16 and torch.equal(l8, l16)


def test_u16_edge_cases():
    for img, conn, ndim in [(np.zeros((1, 1, 1), np.uint16), 6, 3), (np.full((3, 5, 7), 65535, np.uint16), 26, 3),
                            (np.arange(64, dtype=np.uint16).reshape(1, 1, 64) * 1000, 4, 2)]:
        _check(img, conn, ndim)
