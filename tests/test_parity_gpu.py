"""GPU parity: the CUDA path (through the C ABI) vs the oracle, element by element, on the
same seeded inputs.  Bars: blur/gradient floats within 1e-5 absolute;
the u8 gradient equal except on agreed boundary straddles (C11); watershed labels, step II
intermediates and every waterfall level bit-exact."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

FTOL = 1e-5  # north_star: blur and gradient floats within 1e-5 absolute


def _ws():
    import paper_2410_08946_b200 as ws
    return ws


def agreed_gradient(raw_np, sigma, ndim, dev="cuda"):
    """Run ws_gradient and check it against the oracle under C11; return the agreed image
    (the GPU's bytes, which both sides then share) as (torch cuda u8, numpy u8)."""
    ws = _ws()
    img = torch.from_numpy(raw_np).to(dev)
    q, blur, grad = ws.gradient(img, sigma, ndim=ndim, verify=True)
    ob, og, oq = oracle.gradient(raw_np, sigma, ndim=ndim)
    assert np.max(np.abs(blur.cpu().numpy() - ob)) <= FTOL
    assert np.max(np.abs(grad.cpu().numpy() - og)) <= FTOL
    qn = q.cpu().numpy()
    diff = qn != oq
    if diff.any():  # only boundary straddles may differ (|255 g - (k + 1/2)| <= 255 * tol)
        t = 255.0 * og[diff]
        assert np.all(np.abs(t - np.floor(t) - 0.5) <= 255 * FTOL), "gradient quantisation mismatch"
        assert np.all(np.abs(qn[diff].astype(int) - oq[diff].astype(int)) == 1)
    return q, qn


def check_watershed(q_dev, q_np, conn, ndim):
    ws = _ws()
    lab, R = ws.watershed(q_dev, conn, ndim=ndim)
    ref, dist, ptr, Rref = oracle.watershed(q_np, conn, ndim=ndim, dumps=True)
    got = lab.cpu().numpy()
    if not np.array_equal(got, ref):
        bad = np.flatnonzero(got.ravel() != ref.ravel())
        pytest.fail("watershed mismatch at %d voxels, first %s: got %s want %s" % (
            bad.size, bad[:5], got.ravel()[bad[:5]], ref.ravel()[bad[:5]]))
    assert R == Rref
    return lab, ref


def check_waterfall(lab_dev, q_dev, q_np, ref_lab, conn, ndim, NL):
    ws = _ws()
    lv, counts = ws.waterfall(lab_dev, q_dev, conn, NL, ndim=ndim)
    rlv, rcounts = oracle.waterfall(ref_lab, q_np, conn, NL, ndim=ndim)
    got = lv.cpu().numpy()
    for k in range(NL):
        if not np.array_equal(got[k], rlv[k]):
            bad = np.flatnonzero(got[k].ravel() != rlv[k].ravel())
            pytest.fail("level %d mismatch at %d voxels" % (k, bad.size))
    assert list(counts) == [int(c) for c in rcounts]
    return lv


# ---------------------------------------------------------------- configs, reduced sizes
CASES = [("C1", None), ("C2", (1, 384, 512)), ("C3", (40, 48, 56)), ("C4", (24, 96, 80)),
         ("C5", (6, 145, 145))]


@pytest.mark.parametrize("name,shape", CASES)
def test_pipeline_parity_config(name, shape):
    c = synth.CONFIGS[name]
    raw = synth.make_config_image(name, shape=shape, device="cuda").cpu().numpy()
    q, qn = agreed_gradient(raw, c.sigma, c.ndim)
    lab, ref = check_watershed(q, qn, c.conn, c.ndim)
    check_waterfall(lab, q, qn, ref, c.conn, c.ndim, c.NL)


@pytest.mark.parametrize("conn,ndim,shape", [(4, 2, (3, 37, 61)), (8, 2, (2, 45, 33)), (6, 3, (13, 17, 70)),
                                             (26, 3, (9, 21, 35)), (4, 2, (1, 1, 300)), (6, 3, (1, 23, 29))])
@pytest.mark.parametrize("levels", [2, 4, 16])
def test_random_plateau_images(conn, ndim, shape, levels):
    """Plateau-forcing inputs: random values in {0..levels-1}; every plateau
    kind, several tiles and ragged tails in every axis."""
    g = synth.random_plateau_image(shape, levels, seed=levels * 100 + conn)
    qn = g.numpy()
    q = g.cuda()
    lab, ref = check_watershed(q, qn, conn, ndim)
    check_waterfall(lab, q, qn, ref, conn, ndim, 6)


@pytest.mark.parametrize("conn,ndim,shape", [(4, 2, (2, 33, 47)), (8, 2, (1, 40, 40)), (6, 3, (7, 19, 23)),
                                             (26, 3, (6, 11, 17))])
def test_plateau_intermediates(conn, ndim, shape):
    """T2: step I+II intermediates (BFS distances and parent pointers) exact."""
    ws = _ws()
    g = synth.random_plateau_image(shape, 3, seed=conn)
    dist, parent = ws.plateau_debug(g.cuda(), conn, ndim=ndim)
    _, rdist, rptr, _ = oracle.watershed(g.numpy(), conn, ndim=ndim, dumps=True)
    assert np.array_equal(dist.cpu().numpy(), rdist)
    assert np.array_equal(parent.cpu().numpy().astype(np.int64), rptr)


def test_edge_cases():
    ws = _ws()
    cases = [
        (np.zeros((1, 1, 1), np.uint8), 4, 2),                 # single voxel (C4)
        (np.zeros((1, 1, 1), np.uint8), 26, 3),
        (np.full((1, 50, 70), 3, np.uint8), 8, 2),             # one giant minimal plateau
        (np.full((5, 9, 40), 7, np.uint8), 6, 3),
        (np.arange(4096, dtype=np.int64).reshape(1, 64, 64).astype(np.uint8), 4, 2),  # ramps
        (np.array([[[75] + [89] * 10 + [81]]], np.uint8), 4, 2),  # P:364 example
        (np.array([[[75] + [89] * 3000 + [81]]], np.uint8), 4, 2),  # long plateau (deep BFS)
        (np.tile(np.array([0, 255], np.uint8), 300).reshape(1, 20, 30), 4, 2),  # checkerboard rows
    ]
    # serpentine corridor plateau: long BFS depth across many tiles
    snake = np.full((1, 64, 64), 50, np.uint8)
    snake[0, 1::4, :-1] = 200
    snake[0, 3::4, 1:] = 200
    snake[0, 0, 0] = 1
    cases.append((snake, 4, 2))
    for qn, conn, ndim in cases:
        q = torch.from_numpy(qn).cuda()
        lab, ref = check_watershed(q, qn, conn, ndim)
        check_waterfall(lab, q, qn, ref, conn, ndim, 4)
        check_waterfall(lab, q, qn, ref, conn, ndim, 1)


def test_depth1_volume_matches_2d_on_gpu():
    ws = _ws()
    g = synth.random_plateau_image((1, 31, 45), 4, seed=9).cuda()
    a, _ = ws.watershed(g, 6, ndim=3)
    b, _ = ws.watershed(g, 4, ndim=2)
    assert torch.equal(a, b)


def test_determinism_repeated_runs():
    ws = _ws()
    raw = synth.make_config_image("C4", shape=(16, 64, 64), device="cuda")
    q = ws.gradient(raw, 1.0, ndim=3)
    a, _ = ws.watershed(q, 6)
    la, _ = ws.waterfall(a, q, 6, 6)
    for _ in range(3):
        b, _ = ws.watershed(q, 6)
        lb, _ = ws.waterfall(b, q, 6, 6)
        assert torch.equal(a, b) and torch.equal(la, lb)


def test_segment_host_matches_device_path():
    ws = _ws()
    raw = synth.make_config_image("C3", shape=(20, 30, 40), device="cuda")
    q = ws.gradient(raw, 1.0, ndim=3)
    lab, _ = ws.watershed(q, 6)
    lv, counts = ws.waterfall(lab, q, 6, 6)
    lh, ch = ws.segment_host(q.cpu().contiguous(), 6, 6)
    assert torch.equal(lh, lv.cpu()) and ch == counts


def test_abi_errors_on_device():
    ws = _ws()
    q = torch.zeros((2, 3, 4), dtype=torch.uint8, device="cuda")
    with pytest.raises(ws.WsError, match="WS_ERR_INVALID"):
        ws.watershed(q, 6, ndim=2)      # conn/ndim mismatch
    with pytest.raises(ws.WsError, match="WS_ERR_INVALID"):
        ws.watershed(q, 4, ndim=3)
    lab, _ = ws.watershed(q, 4)
    with pytest.raises(ws.WsError, match="WS_ERR_INVALID"):
        ws.waterfall(lab, q, 4, 0)
    with pytest.raises(ws.WsError, match="WS_ERR_INVALID"):
        ws.gradient(q, -1.0)
    # outputs untouched on error
    out = torch.full((2, 3, 4), -7, dtype=torch.int32, device="cuda")
    with pytest.raises(ws.WsError):
        ws.watershed(q, 8, ndim=3, out=out)
    assert bool((out == -7).all())


@pytest.mark.parametrize("conn,ndim,shape", [(6, 3, (20, 48, 64)), (26, 3, (12, 40, 48)), (4, 2, (2, 96, 128)),
                                             (8, 2, (1, 64, 80))])
def test_tma_and_fallback_loaders_agree(conn, ndim, shape, monkeypatch):
    """Aligned shapes (row pitch % 16 == 0) stage tiles with TMA; WS_NO_TMA=1 forces the plain
    loader.  Both must equal the oracle."""
    ws = _ws()
    g = synth.random_plateau_image(shape, 5, seed=conn + 7)
    qn = g.numpy()
    q = g.cuda()
    lab, ref = check_watershed(q, qn, conn, ndim)
    assert ws.stats()["tma"] == 1
    monkeypatch.setenv("WS_NO_TMA", "1")
    lab2, _ = check_watershed(q, qn, conn, ndim)
    assert ws.stats()["tma"] == 0
    assert torch.equal(lab, lab2)


@pytest.mark.parametrize("NL", [1, 2, 3, 5, 6, 9, 10, 12])
@pytest.mark.parametrize("shape", [(1, 64, 96), (1, 37, 61)])
def test_waterfall_nl_variants(NL, shape):
    """Every NL (level-map strides 4 / 8 / NL-1, vector and scalar level writes, early
    termination once one region is left) against the oracle."""
    g = synth.random_plateau_image(shape, 6, seed=NL)
    qn = g.numpy()
    q = g.cuda()
    lab, ref = check_watershed(q, qn, 8, 2)
    check_waterfall(lab, q, qn, ref, 8, 2, NL)


@pytest.mark.parametrize("sigma", [0.0, 0.4, 0.7, 1.0, 1.3, 2.0])
@pytest.mark.parametrize("shape,ndim", [((20, 40, 96), 3), ((3, 70, 130), 2), ((9, 30, 17), 3)])
def test_gradient_sigmas_and_loaders(sigma, shape, ndim, monkeypatch):
    """Fused tile kernel (radius 1..4, TMA or clamped loads) and the separable fallback
    (radius > 4, sigma = 0) against the oracle under C11."""
    raw = synth.random_plateau_image(shape, 256, seed=int(sigma * 10) + ndim).numpy()
    agreed_gradient(raw, sigma, ndim)
    monkeypatch.setenv("WS_NO_TMA", "1")
    agreed_gradient(raw, sigma, ndim)


@pytest.mark.parametrize("conn", [6, 26])
def test_overflow_fallback_paths(conn):
    """The rare host-side fallbacks of ws_watershed, each against the oracle: i.i.d. noise has
    more than N/16 regions (root-list overflow: the watershed is redone with a larger list);
    a constant volume has every tile-face pair on one minimal plateau (cross-tile pair list
    overflow: full union scan after the chase, then the per-root minima are merged)."""
    gen = torch.Generator().manual_seed(conn)
    noise = torch.randint(0, 256, (12, 40, 64), generator=gen, dtype=torch.uint8)
    const = torch.full((24, 48, 64), 7, dtype=torch.uint8)
    for g in (noise, const):
        qn = g.numpy()
        q = g.cuda()
        lab, ref = check_watershed(q, qn, conn, 3)
        if g is noise and conn == 6:
            assert int(np.unique(ref).size) > ref.size // 16  # the overflow case is exercised
        check_waterfall(lab, q, qn, ref, conn, 3, 4)


@pytest.mark.parametrize("conn,ndim,shape,levels", [(4, 2, (2, 45, 61), 6), (8, 2, (1, 70, 90), 10),
                                                    (6, 3, (11, 37, 70), 8), (26, 3, (9, 21, 35), 16),
                                                    (4, 2, (1, 1, 300), 5)])
def test_waterfall_reconstruct_parity(conn, ndim, shape, levels):
    """ws_waterfall_reconstruct (paper-literal Alg. 4 V-VI + Alg. 5) vs oracle O9: every layer
    bit-exact, counts equal; the input gradient is left untouched."""
    ws = _ws()
    g = synth.random_plateau_image(shape, levels, seed=conn + levels)
    qn = g.numpy()
    q = g.cuda()
    lab, ref = check_watershed(q, qn, conn, ndim)
    NL = 6
    lv, counts = ws.waterfall(lab, q, conn, NL, ndim=ndim, mode="reconstruct")
    rlv, rcounts = oracle.waterfall_reconstruct(ref, qn, conn, NL, ndim=ndim)
    got = lv.cpu().numpy()
    for k in range(NL):
        assert np.array_equal(got[k], rlv[k]), "reconstruct level %d" % k
    assert list(counts) == [int(c) for c in rcounts]
    assert np.array_equal(q.cpu().numpy(), qn)


def test_waterfall_reconstruct_config_c1():
    """C1 (cameraman-like, sigma 1, 4-conn, NL=6) through the literal reconstruction."""
    ws = _ws()
    raw = synth.make_config_image("C1", device="cuda").cpu().numpy()
    q, qn = agreed_gradient(raw, 1.0, 2)
    lab, ref = check_watershed(q, qn, 4, 2)
    lv, counts = ws.waterfall(lab, q, 4, 6, ndim=2, mode="reconstruct")
    rlv, rcounts = oracle.waterfall_reconstruct(ref, qn, 4, 6, ndim=2)
    assert np.array_equal(lv.cpu().numpy(), rlv)
    assert list(counts) == [int(c) for c in rcounts]


@pytest.mark.parametrize("variant", ["pruf_sync", "prw_sync", "apruf_sync"])
@pytest.mark.parametrize("conn,ndim,shape,levels", [(4, 2, (2, 45, 61), 3), (8, 2, (1, 70, 90), 5),
                                                    (6, 3, (11, 37, 70), 4), (26, 3, (9, 21, 35), 3),
                                                    (4, 2, (1, 1, 300), 2), (6, 3, (7, 19, 23), 16)])
def test_paper_variants_parity(variant, conn, ndim, shape, levels):
    """The paper's own one-thread-per-voxel kernels (Alg. 1 PRUF_sync, Alg. 2 PRW step IV,
    APRUF step III) give the oracle's partition and canonical labels exactly."""
    ws = _ws()
    g = synth.random_plateau_image(shape, levels, seed=conn * 7 + levels)
    qn = g.numpy()
    lab, R = ws.watershed(g.cuda(), conn, ndim=ndim, variant=variant)
    ref, _, _, Rref = oracle.watershed(qn, conn, ndim=ndim, dumps=True)
    assert np.array_equal(lab.cpu().numpy(), ref)
    assert R == Rref


# ---------------------------------------------------------------- ws_segment (one call)
def check_segment(q_dev, q_np, conn, ndim, NL):
    """ws_segment == oracle watershed + waterfall: every level (level 0 = the labels) and the
    counts, bit-exact."""
    ws = _ws()
    lv, counts = ws.segment(q_dev, conn, NL, ndim=ndim)
    ref = oracle.watershed(q_np, conn, ndim=ndim)
    rlv, rcounts = oracle.waterfall(ref, q_np, conn, NL, ndim=ndim)
    got = lv.cpu().numpy()
    for k in range(NL):
        if not np.array_equal(got[k], rlv[k]):
            pytest.fail("segment level %d mismatch at %d voxels" % (k, int((got[k] != rlv[k]).sum())))
    assert list(counts) == [int(c) for c in rcounts]


@pytest.mark.parametrize("name,shape", CASES)
def test_segment_parity_config(name, shape):
    c = synth.CONFIGS[name]
    raw = synth.make_config_image(name, shape=shape, device="cuda")
    q = _ws().gradient(raw, c.sigma, ndim=c.ndim)
    check_segment(q, q.cpu().numpy(), c.conn, c.ndim, c.NL)


@pytest.mark.parametrize("conn,ndim,shape", [(4, 2, (3, 37, 61)), (8, 2, (2, 45, 33)), (6, 3, (13, 17, 70)),
                                             (26, 3, (9, 21, 35)), (4, 2, (1, 1, 301)), (6, 3, (1, 23, 29))])
@pytest.mark.parametrize("levels,NL", [(2, 1), (3, 6), (16, 3)])
def test_segment_random_plateau_images(conn, ndim, shape, levels, NL):
    """Plateau-forcing inputs incl. giant minimal plateaux (the chase-first union order: listed
    roots that are not final), ragged tails, N % 4 != 0, NL = 1."""
    g = synth.random_plateau_image(shape, levels, seed=levels * 10 + conn)
    check_segment(g.cuda(), g.numpy(), conn, ndim, NL)


def test_segment_edge_cases():
    for img, conn, ndim in [(np.zeros((1, 1, 1), np.uint8), 6, 3), (np.full((3, 5, 7), 9, np.uint8), 26, 3),
                            (np.arange(64, dtype=np.uint8).reshape(1, 1, 64), 4, 2),
                            (np.zeros((1, 1, 3), np.uint8), 8, 2)]:
        check_segment(torch.from_numpy(img).cuda(), img, conn, ndim, 4)


@pytest.mark.parametrize("name,shape,conn,ndim,NL", [("C1", None, 4, 2, 6), ("C4", (16, 64, 96), 6, 3, 6),
                                                     ("C4", (12, 40, 56), 26, 3, 5)])
def test_segment_small_graph_replay(name, shape, conn, ndim, NL, monkeypatch):
    """ws_segment on small inputs runs sync-free and, from the second call with the same
    buffers, as a replayed CUDA graph: every call (direct, capture, replays, and replays on NEW
    contents of the same input buffer) equals the oracle; the regular path agrees"""
    ws = _ws()
    ctx = ws.Context(0)
    raws = [synth.make_config_image(name, device="cuda", shape=shape)]
    g2 = torch.Generator(device="cpu").manual_seed(7)
    raws.append((raws[0].cpu().to(torch.int32) + torch.randint(0, 40, tuple(raws[0].shape), generator=g2,
                                                              dtype=torch.int32)).clamp(0, 255).to(torch.uint8).cuda())
    q = torch.empty_like(raws[0])
    out = torch.empty((NL,) + tuple(raws[0].shape), dtype=torch.int32, device="cuda")
    for it in range(6):
        raw = raws[0] if it < 4 else raws[1]
        ws.gradient(raw, 1.0, ndim=ndim, out=q)
        lv, counts = ws.segment(q, conn, NL, ndim=ndim, ctx=ctx, out=out)
        torch.cuda.synchronize()
        qn = q.cpu().numpy()
        ref = oracle.watershed(qn, conn, ndim=ndim)
        rlv, rc = oracle.waterfall(ref, qn, conn, NL, ndim=ndim)
        assert np.array_equal(lv.cpu().numpy(), rlv), "call %d" % it
        assert list(counts) == [int(c) for c in rc]
        assert ctx.stats()["kernel_launches"] > 0
    monkeypatch.setenv("WS_NO_SMALL", "1")
    lv2, c2 = ws.segment(q, conn, NL, ndim=ndim)
    assert torch.equal(lv2, out) and list(c2) == list(counts)
