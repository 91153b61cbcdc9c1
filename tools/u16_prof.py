"""ws_waterfall_u16 on the C4-shaped 16-bit volume (bench's f4 context line) between
cudaProfilerStart/Stop, with per-phase timing."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth, paper_2410_08946_b200 as ws
raw = synth.make_config_image("C4", device="cuda")
gen = torch.Generator(device="cuda").manual_seed(4242)
raw16 = (raw.to(torch.int32) * 256 + torch.randint(0, 256, tuple(raw.shape), generator=gen, device="cuda",
                                                   dtype=torch.int32)).to(torch.uint16)
del raw
ctx = ws.Context(0)
q16 = ws.gradient(raw16, 1.0, ndim=3, ctx=ctx)
del raw16
lab, R = ws.watershed(q16, 6, ndim=3, ctx=ctx)
lv = torch.empty((6,) + tuple(q16.shape), dtype=torch.int32, device="cuda")
ws.waterfall(lab, q16, 6, 6, ndim=3, ctx=ctx, out=lv)
torch.cuda.synchronize()
ctx.set_timing(True) if hasattr(ctx, "set_timing") else None
torch.cuda.cudart().cudaProfilerStart()
_, c = ws.waterfall(lab, q16, 6, 6, ndim=3, ctx=ctx, out=lv)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("R", R, "counts", list(c))
