"""GPU parity of the alternative code paths the library selects by size or by an environment
switch (read per call): every variant must give the oracle's labels and levels bit-exactly.

  WS_JUMP_V   step III across tiles: 1 = k_jump, 2 (default) / 4 / 8 = k_jumpv<V>
  WS_NO_EQC   step II rounds restage the I box instead of reading k_relax_first's mask cache
  WS_NO_COOP  step II rounds as per-round launches only (no cooperative loop)
  WS_NO_SMALL ws_segment on a small input through the regular (host-synchronised) path
  WS_GRAD_V1  the v1 streaming gradient kernel instead of v2
"""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

CASES = [(6, 3, (13, 40, 70)), (26, 3, (9, 21, 35)), (4, 2, (3, 70, 97)), (8, 2, (2, 45, 66))]


def _ws():
    import paper_2410_08946_b200 as ws
    return ws


def _check(conn, ndim, shape, levels, seed):
    ws = _ws()
    g = synth.random_plateau_image(shape, levels, seed=seed)
    qn = g.numpy()
    lab, _ = ws.watershed(g.cuda(), conn, ndim=ndim)
    ref = oracle.watershed(qn, conn, ndim=ndim)
    assert np.array_equal(lab.cpu().numpy(), ref)
    lv, counts = ws.segment(g.cuda(), conn, 6, ndim=ndim)
    rlv, rcounts = oracle.waterfall(ref, qn, conn, 6, ndim=ndim)
    assert np.array_equal(lv.cpu().numpy(), rlv)
    assert list(counts) == [int(c) for c in rcounts]


@pytest.mark.parametrize("v", ["1", "2", "4", "8"])
@pytest.mark.parametrize("conn,ndim,shape", CASES)
def test_jump_variants(monkeypatch, v, conn, ndim, shape):
    monkeypatch.setenv("WS_JUMP_V", v)
    _check(conn, ndim, shape, 3, seed=int(v) + conn)


@pytest.mark.parametrize("env", ["WS_NO_EQC", "WS_NO_COOP", "WS_NO_SMALL"])
@pytest.mark.parametrize("conn,ndim,shape", CASES)
def test_switches(monkeypatch, env, conn, ndim, shape):
    monkeypatch.setenv(env, "1")
    _check(conn, ndim, shape, 2, seed=conn)
    _check(conn, ndim, shape, 6, seed=conn + 1)


def test_raw_volume_jump_variants(monkeypatch):
    """A raw (noisy, many single-voxel regions) C4-like volume: the root-dense case that made
    V = 4 slower; every V gives the same labels."""
    ws = _ws()
    raw = synth.make_config_image("C4", shape=(24, 96, 80))
    ref = oracle.watershed(raw.numpy(), 6, ndim=3)
    for v in ("1", "2", "4", "8"):
        monkeypatch.setenv("WS_JUMP_V", v)
        lab, R = ws.watershed(raw.cuda(), 6, ndim=3)
        assert np.array_equal(lab.cpu().numpy(), ref), v


def test_gradient_v1_v2_agree(monkeypatch):
    """v1 and v2 streaming gradient kernels: both within the C11 bar of the oracle."""
    ws = _ws()
    raw = synth.make_config_image("C4", shape=(20, 64, 96))
    _, og, oq = oracle.gradient(raw.numpy(), 1.0, ndim=3)
    for v1 in ("0", "1"):
        monkeypatch.setenv("WS_GRAD_V1", v1)
        q = ws.gradient(raw.cuda(), 1.0, ndim=3).cpu().numpy()
        diff = q != oq
        if diff.any():
            t = 255.0 * og[diff]
            assert np.all(np.abs(t - np.floor(t) - 0.5) <= 255 * 1e-5)


def test_segment_host_async_pipeline():
    """ws_segment_host_async on two contexts / streams (the pipelined e2e of bench.py) gives the
    synchronous call's levels and counts for every volume of a sequence."""
    ws = _ws()
    vols = [synth.random_plateau_image((9, 40, 70), 4, seed=s) for s in range(4)]
    ref = [ws.segment_host(v, 6, 6, ndim=3) for v in vols]
    ctxs = (ws.Context(0), ws.Context(0))
    sts = (torch.cuda.Stream(), torch.cuda.Stream())
    outs = [torch.empty((6,) + tuple(v.shape), dtype=torch.int32, pin_memory=True) for v in vols]
    got = []
    for i, v in enumerate(vols):
        k = i & 1
        sts[k].synchronize()
        _, counts = ws.segment_host(v, 6, 6, ndim=3, ctx=ctxs[k], out=outs[i], stream=sts[k], wait=False)
        got.append(counts)
    for st in sts:
        st.synchronize()
    for (rl, rc), out, c in zip(ref, outs, got):
        assert torch.equal(rl, out) and list(rc) == list(c)
