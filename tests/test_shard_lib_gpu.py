"""The sharded pipeline as ONE library call per rank (ws_segment_sharded, include/ws.h; SURVEY
§8(b)/(e)) must reproduce the unsharded ws_segment bit-exactly (T6): labels and every level.

  - K virtual ranks as threads of one process (ThreadCallbacks transport), K = 1..5, 6- and
    26-connectivity, plateau-heavy volumes with 1-plane slabs;
  - 2 processes on the one GPU over torch.distributed gloo (TorchCallbacks: the multi-process
    control flow of the NCCL deployment, planes staged through host memory);
  - the library's own NCCL transport at world size 1 (communicator creation, the collectives
    on one rank) and ws_ctx_create_sharded (the three plain calls on a sharded context);
  - 16-bit volumes (NEXT f4 u16 sharding: ws_segment_sharded_u16 vs ws_watershed_u16 +
    ws_waterfall_u16), K = 1..3, 6- and 26-connectivity, plateaux across the cuts.
"""
import os
import socket

import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


def _ref(grad, conn, NL):
    import paper_2410_08946_b200 as ws
    lv, counts = ws.segment(grad, conn, NL, ndim=3)
    return lv, list(counts)


def _check(grad, K, conn=6, NL=6):
    from paper_2410_08946_b200 import shard
    ref, rc = _ref(grad, conn, NL)
    got, counts, rounds = shard.segment_threads(K, grad, NL, conn)
    if not torch.equal(got, ref):
        bad = (got != ref).nonzero()
        pytest.fail("K=%d: %d values differ, first %s got %s want %s" % (
            K, bad.shape[0], bad[0].tolist(), got[tuple(bad[0])].item(), ref[tuple(bad[0])].item()))
    assert counts == rc
    assert rounds >= 1


@pytest.mark.parametrize("K", [1, 2, 3, 5])
def test_lib_sharded_microct(K):
    import paper_2410_08946_b200 as ws
    raw = synth.make_config_image("C4", shape=(40, 64, 96), device="cuda")
    _check(ws.gradient(raw, 1.0, ndim=3), K)


@pytest.mark.parametrize("conn", [6, 26])
@pytest.mark.parametrize("K,shape,levels", [(2, (12, 33, 47), 3), (4, (16, 32, 64), 2), (6, (6, 20, 30), 3)])
def test_lib_sharded_plateau_volumes(K, shape, levels, conn):
    g = synth.random_plateau_image(shape, levels, seed=K * 10 + levels).cuda()
    _check(g, K, conn, NL=5)


def test_lib_sharded_constant_and_corridor():
    _check(torch.full((10, 16, 32), 7, dtype=torch.uint8, device="cuda"), 4)
    v = np.full((24, 8, 8), 200, np.uint8)
    v[:, 2:6, 2:6] = 50
    v[-1, 3, 3] = 10
    _check(torch.from_numpy(v).cuda(), 3)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, K, port, grad_cpu, NL, conn, out_path):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=K)
    torch.cuda.set_device(0)
    from paper_2410_08946_b200 import _binding, shard
    s = shard.make_slabs(grad_cpu.shape[0], K)[rank]
    ctx = _binding.Context(0)
    tr = shard._CallbackTransport(shard.TorchCallbacks(), rank, K)
    ge = grad_cpu[s.e0:s.e1].contiguous().cuda()
    lv, counts, rounds = shard.segment_sharded(tr, ctx, s, ge, NL, conn)
    torch.save({"lv": lv.cpu(), "counts": counts, "z0": s.z0}, "%s.%d" % (out_path, rank))
    dist.barrier()
    dist.destroy_process_group()


def test_lib_sharded_two_processes_gloo(tmp_path):
    """world size 2, one process per rank, ranks sharing the GPU; gloo moves the planes"""
    import torch.multiprocessing as mp
    import paper_2410_08946_b200 as ws
    raw = synth.make_config_image("C4", shape=(24, 48, 64), device="cuda")
    grad = ws.gradient(raw, 1.0, ndim=3)
    ref, rc = _ref(grad, 6, 6)
    out = str(tmp_path / "r")
    mp.start_processes(_worker, args=(2, _free_port(), grad.cpu(), 6, 6, out), nprocs=2, join=True,
                       start_method="spawn")
    parts = [torch.load("%s.%d" % (out, r)) for r in range(2)]
    got = torch.cat([p["lv"] for p in parts], dim=1)
    assert torch.equal(got, ref.cpu())
    assert parts[0]["counts"] == rc and parts[1]["counts"] == rc


def test_lib_nccl_transport_world1_and_sharded_context():
    """the library's NCCL communicator (world size 1) and ws_ctx_create_sharded: the plain
    ws_segment / ws_watershed calls on a sharded context run the sharded pipeline"""
    import ctypes
    import torch.distributed as dist
    import paper_2410_08946_b200 as ws
    from paper_2410_08946_b200 import _binding, shard
    raw = synth.make_config_image("C4", shape=(16, 40, 56), device="cuda")
    grad = ws.gradient(raw, 1.0, ndim=3)
    ref, rc = _ref(grad, 26, 4)
    if not dist.is_initialized():
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
        dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        tr = shard.NcclLibTransport(0)
        s = shard.make_slabs(grad.shape[0], 1)[0]
        ctx = _binding.Context(0)
        lv, counts, _ = shard.segment_sharded(tr, ctx, s, grad.contiguous(), 4, 26)
        assert torch.equal(lv, ref) and counts == rc
        lib = _binding.load()
        h = ctypes.c_void_p()
        _binding.check(lib.ws_ctx_create_sharded(0, tr.ptr(), s.c(), ctypes.byref(h)))
        sctx = _binding.Context.__new__(_binding.Context)
        sctx.device, sctx.handle = 0, h
        lv2, c2 = ws.segment(grad, 26, 4, ndim=3, ctx=sctx)
        assert torch.equal(lv2, ref) and list(c2) == rc
        lab, R = ws.watershed(grad, 26, ndim=3, ctx=sctx)
        assert torch.equal(lab, ref[0]) and R == rc[0]
        sctx.close()
        tr.close()
    finally:
        dist.destroy_process_group()


def _ref16(grad, conn, NL):
    import paper_2410_08946_b200 as ws
    lab, R = ws.watershed(grad, conn, ndim=3)
    lv, counts = ws.waterfall(lab, grad, conn, NL, ndim=3)
    assert torch.equal(lv[0], lab)
    return lv, list(counts)


@pytest.mark.parametrize("conn", [6, 26])
@pytest.mark.parametrize("K", [1, 2, 3])
def test_lib_sharded_u16(K, conn):
    """u16 sharding (NEXT f4): the sharded watershed + two-step-reduced 16-bit waterfall equal
    ws_watershed_u16 + ws_waterfall_u16 on the whole volume"""
    import paper_2410_08946_b200 as ws
    from paper_2410_08946_b200 import shard
    raw = synth.make_config_image("C4", shape=(24, 40, 56), device="cuda")
    gen = torch.Generator(device="cuda").manual_seed(11 + K)
    raw16 = (raw.to(torch.int32) * 256 + torch.randint(0, 256, tuple(raw.shape), generator=gen, device="cuda",
                                                        dtype=torch.int32)).to(torch.uint16)
    q16 = ws.gradient(raw16, 1.0, ndim=3)
    assert q16.dtype == torch.uint16
    ref, rc = _ref16(q16, conn, 5)
    got, counts, _ = shard.segment_threads(K, q16, 5, conn)
    assert torch.equal(got, ref)
    assert counts == rc


def test_lib_sharded_u16_plateaux():
    """16-bit values with few levels spread over the range: plateaux (minimal and not) cross
    the cuts; odd plane size"""
    from paper_2410_08946_b200 import shard
    g8 = synth.random_plateau_image((12, 33, 47), 4, seed=5).cuda()
    q16 = (g8.to(torch.int32) * 16000 + 7).to(torch.uint16)
    ref, rc = _ref16(q16, 6, 6)
    got, counts, _ = shard.segment_threads(3, q16, 6, 6)
    assert torch.equal(got, ref) and counts == rc
