import sys, torch
sys.path.insert(0, '/root/repo')
import synth, paper_2410_08946_b200 as ws
for shape in [(16, 64, 64), (64, 256, 256)]:
    raw = synth.make_config_image("C4", device="cuda", shape=shape)
    q = ws.gradient(raw, 1.0, ndim=3)
    lab, R = ws.watershed(q, 6, ndim=3)
    torch.cuda.synchronize()
    print(shape, R, ws.stats()["union_order"], flush=True)
