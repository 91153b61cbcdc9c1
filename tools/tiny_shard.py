import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2410_08946_b200 as ws
from paper_2410_08946_b200 import shard
K = int(sys.argv[1]) if len(sys.argv) > 1 else 2
g = synth.random_plateau_image((12, 16, 32), 3, seed=1).cuda()
slabs = shard.make_slabs(g.shape[0], K)
ctxs = [ws.Context(0) for _ in range(K)]
labels, R, rounds = shard.sharded_watershed(shard.LocalTransport(K), ctxs, slabs, [g[s.e0:s.e1].contiguous() for s in slabs])
ref, Rref = ws.watershed(g, 6)
print("equal", torch.equal(torch.cat(labels), ref), R, Rref, rounds)
