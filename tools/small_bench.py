"""ws_segment step time on the small configs (no phase timing): min / median of 50."""
import os, statistics, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth, paper_2410_08946_b200 as ws
for name in sys.argv[1:] or ["C1", "C5"]:
    c = synth.CONFIGS[name]
    raw = synth.make_config_image(name, device="cuda")
    q = ws.gradient(raw, c.sigma, ndim=c.ndim)
    ctx = ws.Context(0)
    out = torch.empty((c.NL,) + tuple(q.shape), dtype=torch.int32, device="cuda")
    for _ in range(5):
        ws.segment(q, c.conn, c.NL, ndim=c.ndim, ctx=ctx, out=out)
    torch.cuda.synchronize()
    ts = []
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(50):
        a.record(); _, counts = ws.segment(q, c.conn, c.NL, ndim=c.ndim, ctx=ctx, out=out); b.record()
        torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    print(os.environ.get("TAG", ""), name, "min %.3f median %.3f ms" % (min(ts), statistics.median(ts)),
          "launches", ctx.stats()["kernel_launches"], "counts", list(counts))
