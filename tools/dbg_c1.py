import sys, torch
sys.path.insert(0, '.')
import synth, paper_2410_08946_b200 as ws
raw = synth.make_config_image("C1", device="cuda")
q = ws.gradient(raw, 1.0, ndim=2); torch.cuda.synchronize(); print("grad ok", flush=True)
for v in ("0", "1"):
    import os; os.environ["WS_NO_TMA"] = v
    try:
        lab, R = ws.watershed(q, 4, ndim=2); torch.cuda.synchronize(); print("ws ok", v, R, flush=True)
        lv, c = ws.waterfall(lab, q, 4, 6, ndim=2); torch.cuda.synchronize(); print("wf ok", v, list(c), flush=True)
    except Exception as e:
        print("ERR", v, e, flush=True); break
