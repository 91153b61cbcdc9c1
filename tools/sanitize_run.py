"""Small end-to-end run for compute-sanitizer: C1 and a small C4-like volume through
ws_gradient -> ws_watershed -> ws_waterfall (graph and reconstruct), the paper's variants and the
sharded path with a local transport; parity against the oracle at the end."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle
import synth
import paper_2410_08946_b200 as ws
from paper_2410_08946_b200 import shard

for name, shape, conn, nd in (("C1", None, 4, 2), ("C4", (20, 48, 64), 6, 3)):
    raw = synth.make_config_image(name, device="cuda", shape=shape)
    q = ws.gradient(raw, 1.0, ndim=nd)
    lab, R = ws.watershed(q, conn, ndim=nd)
    lv, c = ws.waterfall(lab, q, conn, 6, ndim=nd)
    lv2, c2 = ws.waterfall(lab, q, conn, 6, ndim=nd, mode="reconstruct")
    lab3, _ = ws.watershed(q, conn, ndim=nd, variant="prw_sync")
    qn = q.cpu().numpy()
    ref = oracle.watershed(qn, conn, ndim=nd)
    assert np.array_equal(lab.cpu().numpy(), ref) and np.array_equal(lab3.cpu().numpy(), ref)
    assert np.array_equal(lv.cpu().numpy(), oracle.waterfall(ref, qn, conn, 6, ndim=nd)[0])
    assert np.array_equal(lv2.cpu().numpy(), oracle.waterfall_reconstruct(ref, qn, conn, 6, ndim=nd)[0])
    if nd == 3:
        K = 3
        slabs = shard.make_slabs(q.shape[0], K)
        tr = shard.LocalTransport(K)
        ctxs = [ws.Context() for _ in range(K)]
        grads = [q[s.e0:s.e1].contiguous() for s in slabs]
        labs, levs, counts, Rs, _ = shard.sharded_segment(tr, ctxs, slabs, grads, 6, conn)
        assert np.array_equal(torch.cat(labs).cpu().numpy(), ref)
    print(name, "ok", R, c, c2)

# ws_segment: the regular path, the sync-free small mode and its CUDA-graph replays; the
# library's sharded pipeline with K = 3 thread ranks
for name, shape, conn, nd in (("C1", None, 4, 2), ("C4", (20, 48, 64), 6, 3), ("C4", (12, 32, 40), 26, 3)):
    raw = synth.make_config_image(name, device="cuda", shape=shape)
    q = ws.gradient(raw, 1.0, ndim=nd)
    qn = q.cpu().numpy()
    ref = oracle.watershed(qn, conn, ndim=nd)
    rlv = oracle.waterfall(ref, qn, conn, 6, ndim=nd)[0]
    ctx = ws.Context()
    out = torch.empty((6,) + tuple(q.shape), dtype=torch.int32, device="cuda")
    for _ in range(3):
        lv, _ = ws.segment(q, conn, 6, ndim=nd, ctx=ctx, out=out)
        assert np.array_equal(lv.cpu().numpy(), rlv)
    if nd == 3:
        lvs, _, _ = shard.segment_threads(3, q, 6, conn)
        assert np.array_equal(lvs.cpu().numpy(), rlv)
    print("segment", name, conn, "ok")

# large flat minimal plateaux on 2-D tiles (the row-run / parent-initialised in-tile union)
for conn in (4, 8):
    g2 = synth.random_plateau_image((2, 96, 130), 2, seed=conn).cuda()
    lab2, _ = ws.watershed(g2, conn, ndim=2)
    assert np.array_equal(lab2.cpu().numpy(), oracle.watershed(g2.cpu().numpy(), conn, ndim=2))
    print("plateau2d", conn, "ok")

# 16-bit images (NEXT f4): gradient (streaming kernel and generic path) + watershed
rng = np.random.default_rng(7)
for shape, conn, nd, sig in (((20, 48, 64), 6, 3, 1.0), ((18, 40, 36), 26, 3, 2.0), ((2, 70, 96), 8, 2, 1.0)):
    f = rng.standard_normal(shape)
    img = np.floor((f - f.min()) / (np.ptp(f) + 1e-12) * 65535).astype(np.uint16)
    q16 = ws.gradient(torch.from_numpy(img).cuda(), sig, ndim=nd)
    lab16, R16 = ws.watershed(q16, conn, ndim=nd)
    qn16 = q16.cpu().numpy()
    assert np.array_equal(lab16.cpu().numpy(), oracle.watershed(qn16, conn, ndim=nd))
    print("u16", shape, conn, "ok", R16)
