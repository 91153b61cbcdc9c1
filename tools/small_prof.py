"""One ws_segment call of a small config between cudaProfilerStart/Stop (for an ncu launch list:
ncu --profile-from-start off ...).  WS_NO_SMALL=1 forces the regular path."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth, paper_2410_08946_b200 as ws
name = sys.argv[1] if len(sys.argv) > 1 else "C5"
c = synth.CONFIGS[name]
raw = synth.make_config_image(name, device="cuda")
q = ws.gradient(raw, c.sigma, ndim=c.ndim)
ctx = ws.Context(0)
out = torch.empty((c.NL,) + tuple(q.shape), dtype=torch.int32, device="cuda")
for _ in range(3):
    ws.segment(q, c.conn, c.NL, ndim=c.ndim, ctx=ctx, out=out)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
ws.segment(q, c.conn, c.NL, ndim=c.ndim, ctx=ctx, out=out)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print(name, "stats", {k: v for k, v in ctx.stats().items() if k in ("kernel_launches", "plateau_rounds", "n_regions")})
