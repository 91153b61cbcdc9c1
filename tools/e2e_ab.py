"""ws_segment_host on the C4 gradient with host buffers: ms per call for WS_D2H_SPLIT settings."""
import os, sys, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth, paper_2410_08946_b200 as ws
raw = synth.make_config_image("C4", device="cuda")
q = ws.gradient(raw, 1.0, ndim=3)
gh = torch.empty(q.shape, dtype=torch.uint8, pin_memory=True); gh.copy_(q)
del raw, q
ctx = ws.Context(0)
lh = torch.empty((6,) + tuple(gh.shape), dtype=torch.int32, pin_memory=True)
ws.segment_host(gh, 6, 6, ndim=3, ctx=ctx, out=lh)
for rep in range(2):
    for sp in ("0", "2", "4", "8"):
        os.environ["WS_D2H_SPLIT"] = sp
        ws.segment_host(gh, 6, 6, ndim=3, ctx=ctx, out=lh)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(3):
            ws.segment_host(gh, 6, 6, ndim=3, ctx=ctx, out=lh)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t) / 3 * 1e3
        print("split", sp, "%.1f ms" % ms, "%.2f GB/s of PCIe" % (20.13e9 / (ms / 1e3) / 1e9), flush=True)
