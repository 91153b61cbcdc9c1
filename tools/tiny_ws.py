import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2410_08946_b200 as ws
shape = tuple(int(x) for x in sys.argv[1].split(",")) if len(sys.argv) > 1 else (1, 64, 64)
conn = int(sys.argv[2]) if len(sys.argv) > 2 else 4
g = synth.random_plateau_image(shape, 4, seed=1).cuda()
lab, R = ws.watershed(g, conn)
torch.cuda.synchronize()
print("ok", R, ws.stats()["tma"])
