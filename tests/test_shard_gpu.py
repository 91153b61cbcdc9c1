"""z-slab sharding on ONE GPU: K virtual ranks through the in-process
LocalTransport must reproduce the unsharded ws_watershed bit-exactly (T6)."""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


def _run(grad, K, conn=6):
    import paper_2410_08946_b200 as ws
    from paper_2410_08946_b200 import shard
    D = grad.shape[0]
    slabs = shard.make_slabs(D, K)
    tr = shard.LocalTransport(K)
    ctxs = [ws.Context(0) for _ in range(K)]
    grads = [grad[s.e0:s.e1].contiguous() for s in slabs]
    labels, R, rounds = shard.sharded_watershed(tr, ctxs, slabs, grads, conn)
    for c in ctxs:
        c.close()
    return torch.cat(labels, 0), R, rounds


def _check(grad, K, conn=6):
    import paper_2410_08946_b200 as ws
    ref, Rref = ws.watershed(grad, conn)
    got, R, rounds = _run(grad, K, conn)
    if not torch.equal(got, ref):
        bad = (got != ref).nonzero()
        pytest.fail("K=%d: %d voxels differ, first %s got %s want %s" % (
            K, bad.shape[0], bad[0].tolist(), got[tuple(bad[0])].item(), ref[tuple(bad[0])].item()))
    assert R == Rref


@pytest.mark.parametrize("K", [2, 3, 5])
def test_sharded_equals_unsharded_microct(K):
    import paper_2410_08946_b200 as ws
    raw = synth.make_config_image("C4", shape=(40, 64, 96), device="cuda")
    grad = ws.gradient(raw, 1.0, ndim=3)
    _check(grad, K)


@pytest.mark.parametrize("conn", [6, 26])
@pytest.mark.parametrize("K,shape,levels", [(2, (12, 33, 47), 3), (4, (16, 32, 64), 2), (6, (6, 20, 30), 3),
                                            (3, (9, 17, 23), 5)])
def test_sharded_plateau_volumes(K, shape, levels, conn):
    """values in {0..levels-1}: plateaux (minimal and not) crossing every cut; 1-plane slabs;
    26-connectivity adds the diagonal neighbours across every cut."""
    g = synth.random_plateau_image(shape, levels, seed=K * 10 + levels).cuda()
    _check(g, K, conn)


def test_sharded_constant_and_corridor():
    g = torch.full((10, 16, 32), 7, dtype=torch.uint8, device="cuda")   # one minimal plateau over all slabs
    _check(g, 4)
    # a plateau corridor winding through z (deep BFS across slabs), exit at the top
    v = np.full((24, 8, 8), 200, np.uint8)
    v[:, 2:6, 2:6] = 50
    v[23, 4, 4] = 1
    _check(torch.from_numpy(v).cuda(), 4)
    # a knee-like volume
    import paper_2410_08946_b200 as ws
    raw = synth.make_config_image("C3", shape=(30, 40, 48), device="cuda")
    _check(ws.gradient(raw, 1.0, ndim=3), 3)


def _check_segment(grad, K, NL=6, conn=6):
    import paper_2410_08946_b200 as ws
    from paper_2410_08946_b200 import shard
    ref, Rref = ws.watershed(grad, conn)
    rlv, rcounts = ws.waterfall(ref, grad, conn, NL)
    slabs = shard.make_slabs(grad.shape[0], K)
    ctxs = [ws.Context(0) for _ in range(K)]
    labels, levels, counts, R, rounds = shard.sharded_segment(
        shard.LocalTransport(K), ctxs, slabs, [grad[s.e0:s.e1].contiguous() for s in slabs], NL, conn)
    for c in ctxs:
        c.close()
    assert torch.equal(torch.cat(labels, 0), ref) and R == Rref
    got = torch.cat(levels, 1)
    for k in range(NL):
        if not torch.equal(got[k], rlv[k]):
            pytest.fail("K=%d level %d: %d voxels differ" % (K, k, int((got[k] != rlv[k]).sum())))
    assert counts == list(rcounts)


@pytest.mark.parametrize("K", [2, 3, 4])
def test_sharded_waterfall_microct(K):
    import paper_2410_08946_b200 as ws
    raw = synth.make_config_image("C4", shape=(36, 64, 96), device="cuda")
    _check_segment(ws.gradient(raw, 1.0, ndim=3), K)


@pytest.mark.parametrize("conn", [6, 26])
@pytest.mark.parametrize("K,shape,levels,NL", [(2, (10, 24, 40), 4, 6), (5, (5, 16, 32), 3, 4), (3, (12, 20, 28), 6, 9)])
def test_sharded_waterfall_plateaux(K, shape, levels, NL, conn):
    g = synth.random_plateau_image(shape, levels, seed=K + levels).cuda()
    _check_segment(g, K, NL, conn)


@pytest.mark.parametrize("K", [2, 4])
def test_sharded_26conn_microct_and_constant(K):
    """26-connectivity through the whole sharded pipeline on a C4-like volume, and one
    minimal plateau spanning every slab."""
    import paper_2410_08946_b200 as ws
    raw = synth.make_config_image("C4", shape=(24, 48, 64), device="cuda")
    _check_segment(ws.gradient(raw, 1.0, ndim=3), K, 6, 26)
    _check(torch.full((12, 16, 24), 5, dtype=torch.uint8, device="cuda"), K, 26)


@pytest.mark.parametrize("conn2d,conn3d,K", [(8, 26, 3), (4, 6, 4)])
def test_2d_y_band_sharding(conn2d, conn3d, K):
    """NEXT f4, 2-D y-band sharding: an H x W image is the (H, 1, W) volume, whose 26- (6-)
    connectivity is the image's 8- (4-) connectivity and whose linear order is the image's
    (C1, C21), so its z-slabs are y-bands.  The sharded segmentation of the bands must equal
    the unsharded 2-D one."""
    import paper_2410_08946_b200 as ws
    from paper_2410_08946_b200 import shard
    raw = synth.make_config_image("C2", shape=(1, 96, 160), device="cuda")
    q = ws.gradient(raw, 1.0, ndim=2)
    ref, Rref = ws.watershed(q, conn2d, ndim=2)
    rlv, rc = ws.waterfall(ref, q, conn2d, 6, ndim=2)
    H, W = q.shape[1], q.shape[2]
    q3 = q.view(H, 1, W)
    slabs = shard.make_slabs(H, K)
    ctxs = [ws.Context(0) for _ in range(K)]
    labels, levels, counts, R, _ = shard.sharded_segment(
        shard.LocalTransport(K), ctxs, slabs, [q3[s.e0:s.e1].contiguous() for s in slabs], 6, conn3d)
    for c in ctxs:
        c.close()
    assert torch.equal(torch.cat(labels, 0).view(1, H, W), ref) and R == Rref
    assert torch.equal(torch.cat(levels, 1).view(6, 1, H, W), rlv) and counts == list(rc)
