"""GPU parity of ws_watershed_u16 and ws_waterfall_u16 (NEXT f4, 16-bit images) against
the 16-bit oracles (O10, O12): bit-exact labels, every waterfall level and the region counts;
TMA (n2 % 8 == 0) and plain loaders; several tiles with ragged tails; u16 == u8 on
order-isomorphic images."""
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


def _check(img, conn, ndim, NL=6):
    ws = _ws()
    q = torch.from_numpy(img).cuda()
    lab, R = ws.watershed(q, conn, ndim=ndim)
    ref, _, _, Rref = oracle.watershed(img, conn, ndim=ndim, dumps=True)
    got = lab.cpu().numpy()
    if not np.array_equal(got, ref):
        bad = np.flatnonzero(got.ravel() != ref.ravel())
        pytest.fail("u16 watershed mismatch at %d voxels, first %s" % (bad.size, bad[:5]))
    assert R == Rref
    lv, counts = ws.waterfall(lab, q, conn, NL, ndim=ndim)  # ws_waterfall_u16
    rlv, rcounts = oracle.waterfall(ref, img, conn, NL, ndim=ndim)
    glv = lv.cpu().numpy()
    for k in range(NL):
        if not np.array_equal(glv[k], rlv[k]):
            pytest.fail("u16 waterfall level %d mismatch at %d voxels" % (k, int((glv[k] != rlv[k]).sum())))
    assert list(counts) == [int(c) for c in rcounts]


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
    g8, g16 = torch.from_numpy(img8).cuda(), torch.from_numpy(img16).cuda()
    l8, r8 = ws.watershed(g8, conn, ndim=ndim)
    l16, r16 = ws.watershed(g16, conn, ndim=ndim)
    assert r8 == r16 and torch.equal(l8, l16)
    v8, c8 = ws.waterfall(l8, g8, conn, 6, ndim=ndim)
    v16, c16 = ws.waterfall(l16, g16, conn, 6, ndim=ndim)
    assert c8 == c16 and torch.equal(v8, v16)


@pytest.mark.parametrize("NL", [1, 2, 4, 9])
@pytest.mark.parametrize("conn,ndim,shape", [(6, 3, (12, 40, 72)), (4, 2, (3, 64, 100))])
def test_u16_waterfall_levels(NL, conn, ndim, shape):
    _check(_img(shape, "smooth", 11 + NL), conn, ndim, NL)


def test_u16_waterfall_hand_case():
    """O12's hand case on the GPU: {0..3} {4..6} at level 1, one region at level 2."""
    ws = _ws()
    a = torch.tensor([[[0, 256, 10, 300, 20, 255, 30]]], dtype=torch.uint16).cuda()
    lab, R = ws.watershed(a, 4, ndim=2)
    lv, counts = ws.waterfall(lab, a, 4, 3, ndim=2)
    assert lv[1].cpu().tolist() == [[[0, 0, 0, 0, 4, 4, 4]]] and counts == [4, 2, 1]


def test_u16_edge_cases():
    for img, conn, ndim in [(np.zeros((1, 1, 1), np.uint16), 6, 3), (np.full((3, 5, 7), 65535, np.uint16), 26, 3),
                            (np.arange(64, dtype=np.uint16).reshape(1, 1, 64) * 1000, 4, 2)]:
        _check(img, conn, ndim)


FTOL = 1e-5  # north_star float tolerance (as for the u8 gradient)


@pytest.mark.parametrize("sigma", [0.0, 1.0, 1.7])
@pytest.mark.parametrize("ndim,shape", [(3, (13, 19, 37)), (3, (9, 34, 72)), (2, (2, 45, 70)), (2, (3, 96, 200))])
# 72: aligned word loads (3-D streaming kernel); (3, 96, 200): TMA-staged 2-D tiles (row pitch % 16 == 0)
def test_u16_gradient_parity_and_pipeline(sigma, ndim, shape):
    """ws_gradient_u16 vs O11: floats within 1e-5, q equal except on boundary straddles
    (C11 at 16 bits: |65535 g - (k + 1/2)| <= 65535 tol, off by one); then the watershed of
    the agreed u16 image is bit-exact vs O10."""
    ws = _ws()
    rng = np.random.default_rng(int(sigma * 10) + ndim)
    f = rng.standard_normal(shape)
    img = np.floor((f - f.min()) / (np.ptp(f) + 1e-12) * 65535).astype(np.uint16)
    q, blur, grad = ws.gradient(torch.from_numpy(img).cuda(), sigma, ndim=ndim, verify=True)
    ob, og, oq = oracle.gradient(img, sigma, ndim=ndim)
    assert q.dtype == torch.uint16
    assert np.max(np.abs(blur.cpu().numpy() - ob)) <= FTOL
    assert np.max(np.abs(grad.cpu().numpy() - og)) <= FTOL
    qn = q.cpu().numpy()
    diff = qn != oq
    if diff.any():
        t = 65535.0 * og[diff]
        assert np.all(np.abs(t - np.floor(t) - 0.5) <= 65535 * FTOL), "u16 quantisation mismatch"
        assert np.all(np.abs(qn[diff].astype(int) - oq[diff].astype(int)) == 1)
    conn = 6 if ndim == 3 else 8
    _check(qn, conn, ndim)


def test_u16_gradient_of_widened_u8_matches_u8_floats():
    ws = _ws()
    rng = np.random.default_rng(3)
    a = rng.integers(0, 256, (9, 20, 33)).astype(np.uint8)
    _, b8, g8 = ws.gradient(torch.from_numpy(a).cuda(), 1.0, ndim=3, verify=True)
    _, b16, g16 = ws.gradient(torch.from_numpy(a.astype(np.uint16) * 257).cuda(), 1.0, ndim=3, verify=True)
    assert torch.max(torch.abs(b8 - b16)).item() <= 1e-6 and torch.max(torch.abs(g8 - g16)).item() <= 1e-6
