"""ws_watershed on the raw C4 volume (the paper's Table 3 protocol) and on its gradient, per
step III variant (WS_JUMP_V read per call): min of 5."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth, paper_2410_08946_b200 as ws
raw = synth.make_config_image("C4", device="cuda")
q = ws.gradient(raw, 1.0, ndim=3)
ctx = ws.Context(0)
lab = torch.empty(raw.shape, dtype=torch.int32, device="cuda")
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for what, img in (("raw", raw), ("grad", q)):
    for conn in (6, 26):
        for v in ("1", "2", "4"):
            os.environ["WS_JUMP_V"] = v
            ws.watershed(img, conn, ndim=3, ctx=ctx, out=lab)
            ts = []
            for _ in range(5):
                a.record(); _, R = ws.watershed(img, conn, ndim=3, ctx=ctx, out=lab); b.record()
                torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
            st = ctx.stats()
            print(what, conn, "V=%s" % v, "min %.2f ms" % min(ts), "R", R, "union_order", st["union_order"])
