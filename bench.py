#!/usr/bin/env python
"""bench.py — throughput of the hot path (ws_watershed + ws_waterfall NL=6) on B200.

Contract (task statement): ``python bench.py --gpus N --steps K --warmup W`` prints ONE JSON
line on rank 0.  A step = one ws_watershed + one ws_waterfall(NL) over the workload's u8
gradient volume, inputs resident in HBM.  Default workload = config C4 (the metric's 805-Mvox
1024x1024x768 microCT-like volume, 6-conn, NL=6, sigma=1 gradient), see DESIGN.md.

  --impl reference   the oracle (oracle/, plain single-threaded C++) on the host cores, on a
                     bounded sample of the same workload (rank 0 only; other ranks exit 0).
N > 1 (torchrun), 3-D 6-connected workloads (default C4): ONE volume in z-slabs over the ranks
("scaling": "strong"): NCCL halo exchange + boundary union-find merge + per-level all_reduce
(paper_2410_08946_b200/shard.py).  Other workloads: one independent volume per rank ("weak").  Timing: CUDA events on the launching
stream, barrier + synchronize on both sides, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Mvoxel/s watershed+NL=6 waterfall (800 Mvox 3D) at 1/2/4/8 B200; % HBM peak"
UNIT = "Mvoxel/s"
PAPER_CONTEXT = ("paper (P:819 Table 3): 4000x4000x50 raw u8 microCT, watershed only, PRUF 6-conn on an "
                 "RTX 3060 Ti: 1357.75 ms = 589 Mvox/s; no waterfall timings are printed (Figs. 9-10 stripped)")

# algorithmic (compulsory) bytes per voxel of each phase's kernel(s), per launch (DESIGN.md
# §6), for the step's ws_segment call; None = graph / list work (no per-voxel pass)
ALG_BYTES = {
    "watershed.init": 5,        # k_relax_first: read I (1) + write L (4)
    "watershed.relax": None,    # active tiles only
    "watershed.select": 9,      # k_resolve: read I + L, write P
    "watershed.jump": 8,        # k_jump: read P, write P
    "watershed.union": None,    # the cross-tile pair list
    "watershed.find": None,     # the root list
    "watershed.relabel": 8,     # k_relabel_seg: read P, write the dense-id image D
    "waterfall.dense_ids": None,  # bitmap scan over N/32 words + the root list
    "waterfall.rag": 5,         # k_rag: read D + I
    "waterfall.materialise": None,  # k_levels: read D + write levels 0..NL-1: 4 + 4 NL
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--shape", default=None, help="override shape, e.g. 64,128,128 (testing only)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-paper-protocol", action="store_true")
    ap.add_argument("--no-other-configs", action="store_true")
    ap.add_argument("--cpu-sample-slices", type=int, default=32)
    ap.add_argument("--ref-sample-slices", type=int, default=4)
    return ap.parse_args()


def load_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def load_traffic():
    """profiles/ncu_traffic.json (tools/make_traffic.py from an ncu launch list of one step):
    per-phase DRAM bytes per launch, the step's total and the sha256 of the library captured;
    `matches_build` says whether that capture is of the library this run loaded."""
    import hashlib
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
    except Exception:
        return {}
    try:
        lib = os.path.join(ROOT, "paper_2410_08946_b200", "libws_b200.so")
        cur = hashlib.sha256(open(lib, "rb").read()).hexdigest()
        prov = d.get("_provenance", {})
        prov["matches_build"] = prov.get("lib_sha256") == cur
        # nvcc output is not byte-reproducible: the source tree the capture was built from is
        # the stable identity (tools/make_traffic.py records the same hash)
        prov["matches_source"] = prov.get("src_sha256") == source_sha256()
        d["_provenance"] = prov
    except Exception:
        pass
    return d


def source_sha256():
    """sha256 over the library sources (csrc/*, include/ws.h), in sorted path order."""
    import glob
    import hashlib
    h = hashlib.sha256()
    files = sorted(glob.glob(os.path.join(ROOT, "paper_2410_08946_b200", "csrc", "*"))) + \
        [os.path.join(ROOT, "include", "ws.h")]
    for fn in files:
        h.update(os.path.basename(fn).encode())
        h.update(open(fn, "rb").read())
    return h.hexdigest()


class Clocks:
    """nvidia-smi sampler for the timed region (B200_PROFILING.md clocks line)."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        self.f.flush()
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            r = [x.strip() for x in r]
            if len(r) < 9:
                continue
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
            except ValueError:
                continue
            for n, v in zip(names, r[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        load = [s for s in sm if mx and s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        # (WS_BENCH_SHARE_GPU=1: every rank on device local % count -- a functional check of
        # the multi-rank path on a box with fewer GPUs; its timings mean nothing)
        if os.environ.get("WS_BENCH_SHARE_GPU") == "1":
            local = local % torch.cuda.device_count()
            torch.cuda.set_device(local)
            dist.init_process_group("gloo")  # NCCL refuses two ranks on one GPU
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(v, world):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def workload(args):
    import synth
    cfg = synth.CONFIGS[args.config]
    shape = tuple(int(s) for s in args.shape.split(",")) if args.shape else cfg.shape
    return cfg, shape


def cpu_oracle_rate(grad_np, cfg, slices):
    """Oracle (single-threaded C++) watershed + waterfall on the first ``slices`` slices of
    the gradient volume: returns (Mvox/s, seconds, sample description)."""
    import oracle
    sub = grad_np[:slices].copy() if cfg.ndim == 3 else grad_np[: max(1, slices)].copy()
    oracle.build()
    t0 = time.perf_counter()
    lab = oracle.watershed(sub, cfg.conn, ndim=cfg.ndim)
    oracle.waterfall(lab, sub, cfg.conn, cfg.NL, ndim=cfg.ndim)
    dt = time.perf_counter() - t0
    return sub.size / dt / 1e6, dt, "first %d slices %s of the same gradient volume (%d voxels)" % (
        sub.shape[0], "x".join(map(str, sub.shape)), sub.size)


def host_cpu():
    """CPU model and core count of the host (reported next to the oracle)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for l in f:
                if l.startswith("model name"):
                    model = l.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return model, os.cpu_count()


def _c5_worker(args):
    import oracle
    q, conn, NL = args
    lab = oracle.watershed(q, conn, ndim=2)
    oracle.waterfall(lab, q, conn, NL, ndim=2)
    return q.size


def c5_parallel_oracle(q_np, conn, NL):
    """The oracle on C5 with one process per host core, a chunk of the independent images each
    (process-parallel C5 oracle).  Returns (Mvox/s, processes, seconds)."""
    import multiprocessing as mp
    import numpy as np
    import oracle
    oracle.build()
    n = os.cpu_count() or 1
    chunks = [c for c in np.array_split(q_np, n) if c.shape[0] > 0]
    with mp.get_context("fork").Pool(len(chunks)) as pool:
        t0 = time.perf_counter()
        total = sum(pool.map(_c5_worker, [(np.ascontiguousarray(c), conn, NL) for c in chunks]))
        dt = time.perf_counter() - t0
    return total / dt / 1e6, len(chunks), dt


def straddle_count(raw_head, q_head, sigma, ndim, sl):
    """C11 on a sample: the oracle's u8 gradient on the first sl slices (computed from sl + 4
    raw slices: blur radius 3 + 1) vs the GPU's; returns (differing voxels, all straddles?)."""
    import numpy as np
    import oracle
    _, og, oq = oracle.gradient(raw_head, sigma, ndim=ndim)
    og, oq = og[:sl], oq[:sl]
    diff = q_head != oq
    t = 255.0 * og[diff]
    ok = bool(np.all(np.abs(t - np.floor(t) - 0.5) <= 255 * 1e-5))
    return int(diff.sum()), ok


def run_reference(args):
    """--impl reference: the oracle as it stands on the host cores, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    import numpy as np
    import torch
    import oracle
    import synth
    cfg, shape = workload(args)
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    sl = max(1, min(args.ref_sample_slices, shape[0]))
    raw = synth.make_config_image(cfg.name, device=dev, shape=shape)[: sl + 8].cpu().numpy()
    _, _, q = oracle.gradient(raw, cfg.sigma, ndim=cfg.ndim)   # untimed input preparation
    grad = np.ascontiguousarray(q[:sl])
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        lab = oracle.watershed(grad, cfg.conn, ndim=cfg.ndim)
        oracle.waterfall(lab, grad, cfg.conn, cfg.NL, ndim=cfg.ndim)
        if i >= args.warmup:
            times.append(time.perf_counter() - t0)
    ms = 1e3 * sum(times) / len(times)
    value = grad.size / (ms / 1e3) / 1e6
    sample = "first %d slices (%s, %d voxels) of the %s workload per step" % (
        sl, "x".join(map(str, grad.shape)), grad.size, cfg.name)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8/i32", "data": "synthetic",
            "config": {"workload": cfg.desc, "shape": list(shape), "conn": cfg.conn, "NL": cfg.NL,
                       "sigma": cfg.sigma, "sample": sample},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_sharded(args, world, rank, cfg, shape):
    """N > 1 on a 3-D 6-connected workload: ONE volume split into z-slabs over the ranks (strong
    scaling), NCCL halo exchange / boundary-table gathers / all_reduce through
    torch.distributed, every compute step in libws_b200 (paper_2410_08946_b200/shard.py)."""
    import torch
    import synth
    import paper_2410_08946_b200 as ws
    from paper_2410_08946_b200 import shard

    dev = torch.device("cuda", torch.cuda.current_device())
    D, H, W = shape
    N = D * H * W
    NL, conn = cfg.NL, cfg.conn
    slabs = shard.make_slabs(D, world)
    s = slabs[rank]
    ctx = ws.Context(dev.index)
    stream = torch.cuda.current_stream(dev)
    # input (untimed): the same seeded volume on every rank; the slab's gradient from raw planes
    # [e0-4, e1+4) (blur radius 3 + 1 for the derivative) is exactly the global gradient
    raw = synth.make_config_image(cfg.name, device=dev, shape=shape)
    r0, r1 = max(0, s.e0 - 4), min(D, s.e1 + 4)
    raw_ext = raw[r0:r1].contiguous()
    del raw
    torch.cuda.empty_cache()
    gfull = torch.empty_like(raw_ext)
    ws.gradient(raw_ext, cfg.sigma, ndim=3, ctx=ctx, out=gfull)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(3):
        ws.gradient(raw_ext, cfg.sigma, ndim=3, ctx=ctx, out=gfull)
    b.record(stream)
    torch.cuda.synchronize()
    grad_ms = max_over_ranks(a.elapsed_time(b) / 3, world)
    grad_ext = gfull[s.e0 - r0:s.e1 - r0].contiguous()
    del gfull, raw_ext
    torch.cuda.empty_cache()
    # the whole sharded pipeline is ONE library call per rank (ws_segment_sharded); planes move
    # through the library's own NCCL communicator (gloo callbacks when ranks share a GPU)
    import torch.distributed as dist
    if dist.get_backend() == "nccl":
        tr = shard.NcclLibTransport(dev.index)
        transport = "ws_transport_nccl (library-owned NCCL communicator)"
    else:
        tr = shard._CallbackTransport(shard.TorchCallbacks(), rank, world)
        transport = "torch.distributed gloo callbacks (ranks sharing a GPU: functional only)"
    levels_own = torch.empty((NL, s.z1 - s.z0) + tuple(shape[1:]), dtype=torch.int32, device=dev)

    def step():
        lv, cts, rnd = shard.segment_sharded(tr, ctx, s, grad_ext, NL, conn, out=levels_own)
        return lv[0], lv, cts, cts[0], rnd

    for _ in range(args.warmup):
        out = step()
    l0 = ctx.stats()["total_launches"]
    clocks = Clocks(dev.index)
    barrier(world)
    torch.cuda.synchronize()
    clocks.start()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        out = step()
    t1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    clk = clocks.stop()
    launches = ctx.stats()["total_launches"] - l0
    ms = max_over_ranks(t0.elapsed_time(t1) / args.steps, world)
    value = N / (ms / 1e3) / 1e6
    labels, levels, counts, R, rounds = out
    peak, peak_src = load_peak()
    own = (s.z1 - s.z0) * H * W
    step_bytes = 38 if NL == 6 else (5 + 9 + 4 * NL)
    achieved = step_bytes * own / (ms / 1e3) / 1e9  # per GPU (the slowest rank bounds the step)
    roofline = {"bound": "hbm", "kernel": "whole sharded step (per GPU slab)", "achieved": achieved, "peak": peak,
                "unit": "GB/s", "frac": achieved / peak, "traffic": None, "alg_bytes_per_voxel": step_bytes,
                "peak_source": peak_src}
    e2e = None
    if not args.no_e2e:
        gh = torch.empty(grad_ext.shape, dtype=torch.uint8, pin_memory=True)
        gh.copy_(grad_ext)
        lh = torch.empty((NL, s.z1 - s.z0, H, W), dtype=torch.int32, pin_memory=True)
        gdev = torch.empty_like(grad_ext)

        def e2e_step():
            gdev.copy_(gh, non_blocking=True)
            lv, _, _ = shard.segment_sharded(tr, ctx, s, gdev, NL, conn, out=levels_own)
            lh.copy_(lv, non_blocking=True)

        e2e_step()
        barrier(world)
        torch.cuda.synchronize()
        a.record(stream)
        for _ in range(args.e2e_steps):
            e2e_step()
        b.record(stream)
        torch.cuda.synchronize()
        barrier(world)
        ems = max_over_ranks(a.elapsed_time(b) / args.e2e_steps, world)
        e2e = {"value": N / (ems / 1e3) / 1e6, "unit": UNIT, "h2d_bytes_per_step": grad_ext.numel() * world,
               "d2h_bytes_per_step": NL * N * 4, "ms_per_step": ems,
               "api": "ws_segment_sharded per rank, host buffers copied in/out inside the timed region"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u8/i32", "data": "synthetic",
            "config": {"workload": cfg.desc, "name": cfg.name, "shape": list(shape), "conn": conn, "NL": NL,
                       "sigma": cfg.sigma, "global_voxels": N, "parallelism": "z-slab x%d (NCCL halo + boundary "
                       "union-find + per-level all_reduce)" % world, "transport": transport,
                       "l2": "inputs larger than L2 (slab grad %.0f MB, levels %.0f MB per GPU)" % (
                           grad_ext.numel() / 1e6, 4 * NL * own / 1e6)},
            "roofline": roofline, "cpu_baseline": None, "e2e": e2e, "gpu_launches": launches, "clocks": clk,
            "gradient_prepass": {"ms": grad_ms, "Mvoxel_per_s": N / (grad_ms / 1e3) / 1e6},
            "input_stats": {"regions": R, "plateau_rounds": rounds, "level_counts": counts},
            "context": PAPER_CONTEXT,
        }
        print(json.dumps(line), flush=True)
    import torch.distributed as dist
    dist.destroy_process_group()
    return 0


def run_ours(args):
    import numpy as np
    import torch
    import synth
    import paper_2410_08946_b200 as ws

    world, rank, local = dist_setup(args)
    cfg, shape = workload(args)
    if world > 1 and cfg.ndim == 3 and cfg.conn in (6, 26):
        return run_sharded(args, world, rank, cfg, shape)
    dev = torch.device("cuda", torch.cuda.current_device())
    N = int(np.prod(shape))
    NL, conn = cfg.NL, cfg.conn
    ctx = ws.Context(dev.index)

    # input generation (untimed): seeded raw volume, one per rank (independent problems)
    raw = synth.make_config_image(cfg.name, device=dev, shape=shape, seed_offset=1000 * rank)
    stream = torch.cuda.current_stream(dev)

    # ---- gradient pre-pass (timed separately; not part of the metric step)
    grad = torch.empty_like(raw)
    for _ in range(2):
        ws.gradient(raw, cfg.sigma, ndim=cfg.ndim, ctx=ctx, out=grad)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    GK = 3
    for _ in range(GK):
        ws.gradient(raw, cfg.sigma, ndim=cfg.ndim, ctx=ctx, out=grad)
    e1.record(stream)
    torch.cuda.synchronize()
    grad_ms = e0.elapsed_time(e1) / GK

    # the paper's own protocol for context ("all images are raw", Table 3): the
    # watershed alone on the RAW volume, 6- and 26-connectivity (3-D configs only)
    paper_protocol = None
    if cfg.ndim == 3 and not args.no_paper_protocol:
        lab_raw = torch.empty(shape, dtype=torch.int32, device=dev)
        paper_protocol = {"workload": "raw u8 volume of the same config, watershed only (ws_watershed)",
                          "paper": {"volume": "4000x4000x50 raw microCT (800 Mvox)", "gpu": "RTX 3060 Ti",
                                    "ms": {"6": 1357.75, "26": 2258.02}, "Mvoxel_per_s": {"6": 589.2, "26": 354.3},
                                    "cite": "P:819, P:823 (Table 3, PRUF)"}}
        for c3 in (6, 26):
            for _ in range(2):
                _, Rraw = ws.watershed(raw, c3, ndim=3, ctx=ctx, out=lab_raw)
            torch.cuda.synchronize()
            e0.record(stream)
            for _ in range(3):
                _, Rraw = ws.watershed(raw, c3, ndim=3, ctx=ctx, out=lab_raw)
            e1.record(stream)
            torch.cuda.synchronize()
            pms = e0.elapsed_time(e1) / 3
            paper_protocol[str(c3)] = {"ms": pms, "Mvoxel_per_s": N / (pms / 1e3) / 1e6, "regions": Rraw}
        # the paper's 128-Mvoxel microCT shape 500x500x512 (207.99 ms 6-conn, 453.55 ms 26-conn
        # PRUF on an RTX 3060 Ti), the same recipe at that shape, raw, watershed only
        r128 = synth.make_config_image(cfg.name, device=dev, shape=(512, 500, 500))
        l128 = torch.empty(r128.shape, dtype=torch.int32, device=dev)
        ctx128 = {"shape": [512, 500, 500], "paper_ms": {"6": 207.99, "26": 453.554}, "cite": "P:819, P:825 (Table 3)"}
        for c3 in (6, 26):
            ws.watershed(r128, c3, ndim=3, ctx=ctx, out=l128)
            torch.cuda.synchronize()
            e0.record(stream)
            for _ in range(5):
                _, R128 = ws.watershed(r128, c3, ndim=3, ctx=ctx, out=l128)
            e1.record(stream)
            torch.cuda.synchronize()
            pms = e0.elapsed_time(e1) / 5
            ctx128[str(c3)] = {"ms": pms, "Mvoxel_per_s": r128.numel() / (pms / 1e3) / 1e6, "regions": R128}
        paper_protocol["raw_500x500x512"] = ctx128
        del r128, l128
        # 16-bit acquisition (NEXT f4): the u8 volume as the high byte, seeded uniform
        # low byte -> ws_watershed_u16 on the same shape, 6-connectivity
        gen = torch.Generator(device=dev).manual_seed(4242 + rank)
        raw16 = (raw.to(torch.int32) * 256 + torch.randint(0, 256, tuple(shape), generator=gen, device=dev,
                                                           dtype=torch.int32)).to(torch.uint16)
        for _ in range(2):
            _, R16 = ws.watershed(raw16, 6, ndim=3, ctx=ctx, out=lab_raw)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(3):
            _, R16 = ws.watershed(raw16, 6, ndim=3, ctx=ctx, out=lab_raw)
        e1.record(stream)
        torch.cuda.synchronize()
        pms = e0.elapsed_time(e1) / 3
        paper_protocol["u16_6"] = {"what": "ws_watershed_u16, raw volume * 256 + seeded uniform low byte",
                                   "ms": pms, "Mvoxel_per_s": N / (pms / 1e3) / 1e6, "regions": R16}
        # the 16-bit pre-pass on that volume (ws_gradient_u16, generic separable path) and the
        # watershed of its 16-bit gradient: finer quantisation, smaller plateaux (f4)
        q16 = torch.empty_like(raw16)
        ws.gradient(raw16, cfg.sigma, ndim=3, ctx=ctx, out=q16)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(3):
            ws.gradient(raw16, cfg.sigma, ndim=3, ctx=ctx, out=q16)
        e1.record(stream)
        torch.cuda.synchronize()
        gms16 = e0.elapsed_time(e1) / 3
        ws.watershed(q16, 6, ndim=3, ctx=ctx, out=lab_raw)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(3):
            _, Rq16 = ws.watershed(q16, 6, ndim=3, ctx=ctx, out=lab_raw)
        e1.record(stream)
        torch.cuda.synchronize()
        wms16 = e0.elapsed_time(e1) / 3
        rounds16 = ctx.stats()["plateau_rounds"]
        lv16 = torch.empty((NL,) + tuple(shape), dtype=torch.int32, device=dev)
        ws.waterfall(lab_raw, q16, 6, NL, ndim=3, ctx=ctx, out=lv16)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(3):
            _, c16 = ws.waterfall(lab_raw, q16, 6, NL, ndim=3, ctx=ctx, out=lv16)
        e1.record(stream)
        torch.cuda.synchronize()
        fms16 = e0.elapsed_time(e1) / 3
        paper_protocol["u16_gradient"] = {"what": "ws_gradient_u16 (sigma of the config), ws_watershed_u16 6-conn, "
                                                  "ws_waterfall_u16 NL=%d" % NL,
                                          "gradient_ms": gms16, "watershed_ms": wms16, "waterfall_ms": fms16,
                                          "Mvoxel_per_s_watershed_waterfall": N / ((wms16 + fms16) / 1e3) / 1e6,
                                          "regions": Rq16, "plateau_rounds": rounds16, "level_counts": list(c16)}
        del lab_raw, raw16, q16, lv16
    sl_cpu = max(1, min(args.cpu_sample_slices, shape[0])) if cfg.ndim == 3 else shape[0]
    raw_head = raw[:sl_cpu + 4].cpu().numpy() if cfg.ndim == 3 else raw.cpu().numpy()
    del raw
    torch.cuda.empty_cache()

    levels = torch.empty((NL,) + tuple(shape), dtype=torch.int32, device=dev)
    labels = levels[0]

    def step():  # ws_segment = ws_watershed + ws_waterfall(NL) in one call (levels[0] = labels)
        ws.segment(grad, conn, NL, ndim=cfg.ndim, ctx=ctx, out=levels)
        s = ctx.stats()
        return s, s

    for _ in range(args.warmup):
        step()
    ctx.set_timing(True)
    clocks = Clocks(dev.index)
    barrier(world)
    torch.cuda.synchronize()
    clocks.start()
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    phase_ms, phase_launch, launches, stats = {}, {}, 0, []
    step_ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    for i in range(args.steps):
        step_ev[i].record(stream)
        s1, s2 = step()
        stats.append((s1, s2))
        for s in ((s1,) if s1 is s2 else (s1, s2)):
            launches += s["kernel_launches"]
            for k, v in s["phases"].items():
                phase_ms[k] = phase_ms.get(k, 0.0) + v["ms"]
                phase_launch[k] = phase_launch.get(k, 0) + v["launches"]
    step_ev[args.steps].record(stream)
    t_end.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    clk = clocks.stop()
    ctx.set_timing(False)
    ms_local = t_start.elapsed_time(t_end) / args.steps
    per_step = [step_ev[i].elapsed_time(step_ev[i + 1]) for i in range(args.steps)]
    step_stats = {"mean": ms_local, "min": min(per_step), "median": statistics.median(per_step),
                  "note": "per-step CUDA events inside the timed region; min = the paper's protocol (P:742)"}
    ms = max_over_ranks(ms_local, world)
    value = N * world / (ms / 1e3) / 1e6

    # ---- roofline of the dominant kernel (phase with the largest share of the step)
    peak, peak_src = load_peak()
    traffic = load_traffic()
    alg = dict(ALG_BYTES)
    alg["waterfall.materialise"] = 4 + 4 * NL
    cand = {k: v for k, v in phase_ms.items() if alg.get(k)}
    dom = max(cand, key=cand.get)
    per_launch_ms = phase_ms[dom] / max(1, phase_launch[dom])
    achieved = alg[dom] * N / (per_launch_ms / 1e3) / 1e9
    tr = traffic.get(dom)
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": tr.get("bytes_per_launch") if tr else None,
                "traffic_source": dict(traffic.get("_provenance", {}), file="profiles/ncu_traffic.json") if tr else None,
                "alg_bytes_per_voxel": alg[dom], "avg_launch_ms": per_launch_ms,
                "share_of_step": phase_ms[dom] / (ms_local * args.steps), "peak_source": peak_src}
    step_bytes = 38 if NL == 6 else (5 + 9 + 4 * NL)
    step_roof = {"alg_bytes_per_voxel": step_bytes, "achieved_GBps": step_bytes * N / (ms / 1e3) / 1e9,
                 "frac": step_bytes * N / (ms / 1e3) / 1e9 / peak}
    if traffic.get("_step") and cfg.name == "C4" and args.shape is None:
        st = traffic["_step"]
        step_roof["measured_dram_bytes_per_voxel"] = st.get("dram_bytes_per_voxel")
        step_roof["amplification_vs_alg"] = st.get("amplification_vs_38B")
        step_roof["measured_source"] = dict(traffic.get("_provenance", {}), file="profiles/ncu_traffic.json")

    # ---- the paper-literal waterfall (Alg. 4 V-VI + watershed per layer,
    # Alg. 5) on the same labels, for context: not the metric (outside the timed region)
    literal = None
    if not args.no_paper_protocol:
        lv2 = torch.empty_like(levels)
        for _ in range(2):
            _, lc = ws.waterfall(labels, grad, conn, NL, ndim=cfg.ndim, ctx=ctx, out=lv2, mode="reconstruct")
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(3):
            _, lc = ws.waterfall(labels, grad, conn, NL, ndim=cfg.ndim, ctx=ctx, out=lv2, mode="reconstruct")
        e1.record(stream)
        torch.cuda.synchronize()
        lms = e0.elapsed_time(e1) / 3
        literal = {"what": "ws_waterfall_reconstruct, NL=%d, on the step's level-0 labels (Alg. 4 V-VI + Alg. 5)" % NL,
                   "ms": lms, "Mvoxel_per_s": N / (lms / 1e3) / 1e6, "level_counts": list(lc)}
        del lv2
        torch.cuda.empty_cache()

    # ---- the paper's own one-thread-per-voxel watershed kernels on the same gradient (SURVEY
    # NEXT f3: the baseline design the tiled ws_watershed replaces), for context
    variants = None
    if not args.no_paper_protocol:
        variants = {"what": "ws_watershed_variant on the step's gradient, same partition as ws_watershed",
                    "tiled_ws_watershed_ms": sum(v for k, v in phase_ms.items() if k.startswith("watershed.")) / args.steps}
        lab_v = torch.empty_like(labels)
        for vname in ("pruf_sync", "prw_sync", "apruf_sync"):
            ws.watershed(grad, conn, ndim=cfg.ndim, ctx=ctx, out=lab_v, variant=vname)
            torch.cuda.synchronize()
            e0.record(stream)
            for _ in range(2):
                _, Rv = ws.watershed(grad, conn, ndim=cfg.ndim, ctx=ctx, out=lab_v, variant=vname)
            e1.record(stream)
            torch.cuda.synchronize()
            vms = e0.elapsed_time(e1) / 2
            variants[vname] = {"ms": vms, "Mvoxel_per_s": N / (vms / 1e3) / 1e6, "regions": Rv,
                               "same_labels": bool(torch.equal(lab_v, labels)),
                               "step2_rounds": ctx.stats()["plateau_rounds"]}
        del lab_v
        torch.cuda.empty_cache()

    # ---- the other configs of BASELINE.json at full size, one GPU (SURVEY §8(d) "also
    # reported"): gradient pre-pass timed separately, then the step; min and median of 5
    others = None
    if world == 1 and not args.no_other_configs and args.shape is None and cfg.name == "C4":
        others = {}
        del labels, levels
        torch.cuda.empty_cache()
        for name in ("C1", "C2", "C3", "C5"):
            oc = synth.CONFIGS[name]
            oraw = synth.make_config_image(name, device=dev)
            og = torch.empty_like(oraw)
            for _ in range(2):
                ws.gradient(oraw, oc.sigma, ndim=oc.ndim, ctx=ctx, out=og)
            torch.cuda.synchronize()
            e0.record(stream)
            for _ in range(3):
                ws.gradient(oraw, oc.sigma, ndim=oc.ndim, ctx=ctx, out=og)
            e1.record(stream)
            torch.cuda.synchronize()
            gms = e0.elapsed_time(e1) / 3
            for oNL in ((oc.NL, 6) if oc.NL != 6 else (6,)):  # C5: NL = 4 and NL = 6
                olev = torch.empty((oNL,) + tuple(oraw.shape), dtype=torch.int32, device=dev)
                for _ in range(2):
                    ws.segment(og, oc.conn, oNL, ndim=oc.ndim, ctx=ctx, out=olev)
                torch.cuda.synchronize()
                times = []
                for _ in range(10):
                    e0.record(stream)
                    _, ocounts = ws.segment(og, oc.conn, oNL, ndim=oc.ndim, ctx=ctx, out=olev)
                    e1.record(stream)
                    torch.cuda.synchronize()
                    times.append(e0.elapsed_time(e1))
                on = oraw.numel()
                med = statistics.median(times)
                sb = 14 + 4 * oNL  # 5 + (9 + 4 NL) algorithmic bytes per voxel
                key = name if oNL == oc.NL else "%s_NL%d" % (name, oNL)
                others[key] = {"workload": oc.desc, "shape": list(oraw.shape), "conn": oc.conn, "NL": oNL,
                               "gradient_ms": gms, "step_ms_min": min(times), "step_ms_median": med,
                               "Mvoxel_per_s": on / (med / 1e3) / 1e6,
                               "Mvoxel_per_s_incl_gradient": on / ((med + gms) / 1e3) / 1e6,
                               "hbm_frac": sb * on / (min(times) / 1e3) / 1e9 / load_peak()[0],
                               "alg_bytes_per_voxel": sb, "regions": ocounts[0], "level_counts": list(ocounts),
                               "launches_per_step": ctx.stats()["kernel_launches"]}
                del olev
            del oraw, og
            torch.cuda.empty_cache()
        levels = torch.empty((NL,) + tuple(shape), dtype=torch.int32, device=dev)
        labels = levels[0]

    # ---- end to end through the public API with HOST buffers (ws_segment_host)
    e2e = None
    if not args.no_e2e:
        gh = torch.empty(shape, dtype=torch.uint8, pin_memory=True)
        gh.copy_(grad)
        lh = torch.empty((NL,) + tuple(shape), dtype=torch.int32, pin_memory=True)
        ws.segment_host(gh, conn, NL, ndim=cfg.ndim, ctx=ctx, out=lh)  # warm
        barrier(world)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.e2e_steps):
            ws.segment_host(gh, conn, NL, ndim=cfg.ndim, ctx=ctx, out=lh)
        b.record(stream)
        torch.cuda.synchronize()
        barrier(world)
        sync_ms = max_over_ranks(a.elapsed_time(b) / args.e2e_steps, world)
        # pipelined: ws_segment_host_async on two contexts / streams, so the levels' PCIe copy of
        # one step overlaps the host-to-device copy and the compute of the next (PCIe is full
        # duplex); every step still copies its input in and its levels out inside the span
        ctx2 = ws.Context(dev.index if dev.index is not None else 0)
        lh2 = torch.empty((NL,) + tuple(shape), dtype=torch.int32, pin_memory=True)
        ctxs, lhs = (ctx, ctx2), (lh, lh2)
        sts = (torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev))
        ws.segment_host(gh, conn, NL, ndim=cfg.ndim, ctx=ctx2, out=lh2)  # warm the second context
        torch.cuda.synchronize()
        psteps = max(args.e2e_steps, 4)
        a.record(stream)
        for st_ in sts:
            st_.wait_event(a)
        for i in range(psteps):
            k = i & 1
            sts[k].synchronize()  # context k's previous copy is done before it is reused
            ws.segment_host(gh, conn, NL, ndim=cfg.ndim, ctx=ctxs[k], out=lhs[k], stream=sts[k], wait=False)
        for st_ in sts:
            stream.wait_stream(st_)
        b.record(stream)
        torch.cuda.synchronize()
        barrier(world)
        ems = max_over_ranks(a.elapsed_time(b) / psteps, world)
        e2e = {"value": N * world / (ems / 1e3) / 1e6, "unit": UNIT, "h2d_bytes_per_step": N,
               "d2h_bytes_per_step": NL * N * 4, "ms_per_step": ems,
               "api": "ws_segment_host_async, two contexts on two streams (pipelined), %d steps" % psteps,
               "pcie_GBps": (N + NL * N * 4) / (ems / 1e3) / 1e9,
               "sync_ms_per_step": sync_ms, "sync_api": "ws_segment_host (one call at a time)",
               "note": "host-to-device grad + device-to-host NL i32 level arrays per step: PCIe-bound "
                       "(the levels are %.1f GB; the device step is %.1f ms; one call at a time %.1f ms, "
                       "pipelined %.1f ms per step)" % (NL * N * 4 / 1e9, ms, sync_ms, ems)}
        del gh, lh, lh2, ctx2

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        gnp = grad.cpu().numpy()
        v, dt, sample = cpu_oracle_rate(gnp, cfg, args.cpu_sample_slices)
        model, ncpu = host_cpu()
        cpu = {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample, "seconds": dt,
               "cpu_model": model, "nproc": ncpu, "note": "single-threaded C++ oracle (-O2), 1 of nproc cores"}
        nst, st_ok = straddle_count(raw_head, gnp[:sl_cpu], cfg.sigma, cfg.ndim, sl_cpu)
        cpu["c11_straddles"] = {"voxels": nst, "all_boundary_straddles": st_ok, "sample_voxels": int(gnp[:sl_cpu].size),
                                "what": "u8 gradient voxels where ws_gradient and the fp64 oracle differ (C11)"}
        del gnp
        if world == 1 and args.shape is None and not args.no_other_configs:
            c5 = synth.CONFIGS["C5"]
            c5raw = synth.make_config_image("C5", device=dev)
            c5q = ws.gradient(c5raw, c5.sigma, ndim=2, ctx=ctx).cpu().numpy()
            pv, pn, pdt = c5_parallel_oracle(c5q, c5.conn, c5.NL)
            cpu["process_parallel_C5"] = {"value": pv, "unit": UNIT, "cores": pn, "seconds": pdt, "NL": c5.NL,
                                          "sample": "the full C5 batch %s, one chunk of images per process" %
                                                    "x".join(map(str, c5q.shape))}
            del c5raw, c5q

    s1, s2 = stats[-1]
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8/i32", "data": "synthetic",
            "config": {"workload": cfg.desc, "name": cfg.name, "shape": list(shape), "conn": conn, "NL": NL,
                       "sigma": cfg.sigma, "global_voxels": N * world,
                       "parallelism": "replicas" if world > 1 else "single",
                       "l2": "inputs larger than L2 (grad %.0f MB, labels %.0f MB, levels %.0f MB)" % (
                           N / 1e6, 4 * N / 1e6, 4 * NL * N / 1e6)},
            "roofline": roofline, "step_roofline": step_roof, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "clocks": clk,
            "gradient_prepass": {"ms": grad_ms, "Mvoxel_per_s": N / (grad_ms / 1e3) / 1e6},
            "paper_protocol_watershed_raw": paper_protocol,
            "paper_literal_waterfall": literal,
            "paper_kernel_variants": variants,
            "step_ms": step_stats,
            "other_configs": others,
            "phases_ms_per_step": {k: v / args.steps for k, v in sorted(phase_ms.items(), key=lambda x: -x[1])},
            "input_stats": {"regions": s1["n_regions"], "edges": s2["n_edges"],
                            "plateau_rounds": s1["plateau_rounds"], "level_counts": s2["level_counts"][:NL],
                            "level_edges": s2["level_edges"][1:NL], "rag_records": s2.get("rag_records"),
                            "rag_global_emits": s2.get("rag_global_emits")},
            "context": PAPER_CONTEXT,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def relaunch_under_torchrun(args):
    """`python bench.py --gpus N` (N > 1) outside torchrun: run the same command as N ranks,
    one process per GPU (the contract's launch), and pass rank 0's line through."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl != "reference":
        return relaunch_under_torchrun(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
