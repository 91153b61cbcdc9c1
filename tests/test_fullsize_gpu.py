"""Full-size parity (C4: 768 x 1024 x 1024 = 805 Mvoxel, the bench configuration):

  * gradient: exact against the oracle on sampled crops (a voxel's blur + gradient depends
    only on its (2r+3)^3 neighbourhood, so the oracle on a crop with a 4-voxel margin
    reproduces the full-volume value; C11 rule for the u8 image);
  * watershed: properties that hold at any size -- canonical labels (C7), every voxel with
    a strictly lower neighbour has the label of its Eq. 1 target, every
    region holds a voxel without a strictly lower neighbour (its regional minimum);
  * waterfall: nested levels (C13), canonical labels per level (C16), counts non-increasing
    with at least halving while > 1 (every component merges, C14).
Runs the same calls as bench.py (ws.gradient -> ws.watershed -> ws.waterfall NL=6)."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

FTOL = 1e-5
SHAPE = (768, 1024, 1024)
NL = 6


@pytest.fixture(scope="module")
def c4():
    import paper_2410_08946_b200 as ws
    raw = synth.make_config_image("C4", device="cuda", shape=SHAPE)
    q, blur, grad = ws.gradient(raw, 1.0, ndim=3, verify=True)
    lab, R = ws.watershed(q, 6, ndim=3)
    levels, counts = ws.waterfall(lab, q, 6, NL, ndim=3)
    torch.cuda.synchronize()
    return raw, q, blur, grad, lab, R, levels, counts


def test_gradient_sampled_crops(c4):
    raw, q, blur, grad, *_ = c4
    rng = np.random.default_rng(4)
    D, H, W = SHAPE
    M, C = 4, 12  # margin (blur radius 3 + 1 for the central difference), inner crop side
    corners = [(0, 0, 0), (D - C, H - C, W - C)] + [tuple(int(rng.integers(0, s - C + 1)) for s in SHAPE)
                                                   for _ in range(10)]
    for z, y, x in corners:
        z0, y0, x0 = max(z - M, 0), max(y - M, 0), max(x - M, 0)
        z1, y1, x1 = min(z + C + M, D), min(y + C + M, H), min(x + C + M, W)
        crop = raw[z0:z1, y0:y1, x0:x1].cpu().numpy()
        ob, og, oq = oracle.gradient(crop, 1.0, ndim=3)
        sl = (slice(z - z0, z - z0 + C), slice(y - y0, y - y0 + C), slice(x - x0, x - x0 + C))
        gs = (slice(z, z + C), slice(y, y + C), slice(x, x + C))
        assert np.max(np.abs(blur[gs].cpu().numpy() - ob[sl])) <= FTOL
        assert np.max(np.abs(grad[gs].cpu().numpy() - og[sl])) <= FTOL
        qg, qo, go = q[gs].cpu().numpy(), oq[sl], og[sl]
        diff = qg != qo
        if diff.any():
            t = 255.0 * go[diff]
            assert np.all(np.abs(t - np.floor(t) - 0.5) <= 255 * FTOL)


def _shift(a, axis, d, fill):
    """a shifted by d along axis (out-of-volume positions = fill)."""
    out = torch.full_like(a, fill)
    n = a.shape[axis]
    src = [slice(None)] * 3
    dst = [slice(None)] * 3
    if d > 0:
        src[axis], dst[axis] = slice(d, n), slice(0, n - d)
    else:
        src[axis], dst[axis] = slice(0, n + d), slice(-d, n)
    out[tuple(dst)] = a[tuple(src)]
    return out


def test_watershed_properties(c4):
    _, q, _, _, lab, R, _, _ = c4
    _check_watershed_properties(q, lab, R)


def _check_watershed_properties(q, lab, R):
    N = lab.numel()
    idx = torch.arange(N, device="cuda", dtype=torch.int64).view(SHAPE)
    l64 = lab.long()
    assert bool((l64 <= idx).all())                                   # canonical: min index
    flat = lab.view(-1).long()
    assert bool((flat[flat] == flat).all())                           # representative's own label
    I = q.int()
    # Eq. 1 target of every voxel: among the 6 neighbours with the minimum value, the largest
    # index; neighbours in increasing index order are (z-1), (y-1), (x-1), (x+1), (y+1), (z+1)
    order = [(0, -1), (1, -1), (2, -1), (2, 1), (1, 1), (0, 1)]
    best = torch.full_like(I, 1 << 16)  # above every u8 / u16 value
    tgt = torch.full_like(l64, -1)
    for axis, d in order:
        nv = _shift(I, axis, d, 1 << 20)
        nl = _shift(l64, axis, d, -1)
        take = nv <= best                                             # "<=": the last minimum wins
        best = torch.where(take, nv, best)
        tgt = torch.where(take, nl, tgt)
        del nv, nl, take
    lower = best < I
    assert bool((tgt[lower] == l64[lower]).all())                     # descent stays in the region
    reps = flat == torch.arange(N, device="cuda")
    assert int(reps.sum()) == R
    has_min = torch.zeros(N, dtype=torch.bool, device="cuda")
    has_min[flat[~lower.view(-1)]] = True                             # voxels without a lower neighbour
    assert bool(has_min[reps].all())                                  # every region holds a minimum


def test_waterfall_properties(c4):
    *_, lab, R, levels, counts = c4
    N = lab.numel()
    assert counts[0] == R
    ar = torch.arange(N, device="cuda")
    for k in range(1, NL):
        prev, cur = levels[k - 1].view(-1).long(), levels[k].view(-1).long()
        m = torch.full((N,), -1, device="cuda", dtype=torch.int64)
        m[prev] = cur
        assert bool((m[prev] == cur).all())                           # nested: a function of level k-1
        assert bool((cur <= ar).all()) and bool((cur[cur] == cur).all())  # canonical
        assert int((cur == ar).sum()) == counts[k]
        assert counts[k] <= counts[k - 1] and (counts[k - 1] <= 1 or 2 * counts[k] <= counts[k - 1])
    assert torch.equal(levels[0], lab)


# ---- NEXT f4 at the full C4 shape: a 16-bit volume (the u8 volume as the high byte, seeded
# low byte, as in bench.py), ws_gradient_u16 sampled crops vs O11 and the properties of
# ws_watershed_u16 on its gradient
def test_u16_fullsize_gradient_crops_and_watershed():
    import paper_2410_08946_b200 as ws
    raw = synth.make_config_image("C4", device="cuda", shape=SHAPE)
    gen = torch.Generator(device="cuda").manual_seed(4242)
    raw16 = (raw.to(torch.int32) * 256 + torch.randint(0, 256, SHAPE, generator=gen, device="cuda",
                                                       dtype=torch.int32)).to(torch.uint16)
    del raw
    q, blur, grad = ws.gradient(raw16, 1.0, ndim=3, verify=True)
    rng = np.random.default_rng(16)
    D, H, W = SHAPE
    M, C = 4, 10
    corners = [(0, 0, 0), (D - C, H - C, W - C)] + [tuple(int(rng.integers(0, s - C + 1)) for s in SHAPE)
                                                   for _ in range(6)]
    for z, y, x in corners:
        z0, y0, x0 = max(z - M, 0), max(y - M, 0), max(x - M, 0)
        z1, y1, x1 = min(z + C + M, D), min(y + C + M, H), min(x + C + M, W)
        crop = raw16[z0:z1, y0:y1, x0:x1].cpu().numpy()
        ob, og, oq = oracle.gradient(crop, 1.0, ndim=3)
        sl = (slice(z - z0, z - z0 + C), slice(y - y0, y - y0 + C), slice(x - x0, x - x0 + C))
        gs = (slice(z, z + C), slice(y, y + C), slice(x, x + C))
        assert np.max(np.abs(blur[gs].cpu().numpy() - ob[sl])) <= FTOL
        assert np.max(np.abs(grad[gs].cpu().numpy() - og[sl])) <= FTOL
        qg, qo, go = q[gs].cpu().numpy(), oq[sl], og[sl]
        diff = qg != qo
        if diff.any():
            t = 65535.0 * go[diff]
            assert np.all(np.abs(t - np.floor(t) - 0.5) <= 65535 * FTOL)
            assert np.all(np.abs(qg[diff].astype(int) - qo[diff].astype(int)) == 1)
    del blur, grad, raw16
    torch.cuda.empty_cache()
    lab, R = ws.watershed(q, 6, ndim=3)
    _check_watershed_properties(q, lab, R)
