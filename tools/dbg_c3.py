import sys, os, torch
sys.path.insert(0, '/root/repo')
import synth, paper_2410_08946_b200 as ws
raw = synth.make_config_image("C3", device="cuda")
q = ws.gradient(raw, 1.0, ndim=3)
torch.cuda.synchronize()
lab, R = ws.watershed(q, 6, ndim=3)
st = ws.stats()
lv, c = ws.segment(q, 6, 6, ndim=3)
st2 = ws.stats()
print(os.environ.get("TAG"), "R", R, "seg R", c[0], "union_order", st["union_order"], st2["union_order"], "rounds", st["plateau_rounds"], st2["plateau_rounds"],
      "mismatch", int((lv[0] != lab).sum()), "qsum", int(q.sum()))
