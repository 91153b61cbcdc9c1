import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2410_08946_b200 as ws
from paper_2410_08946_b200 import shard
K = int(sys.argv[1]) if len(sys.argv) > 1 else 2
shape = tuple(int(x) for x in sys.argv[2].split(",")) if len(sys.argv) > 2 else (40, 64, 96)
raw = synth.make_config_image("C4", shape=shape, device="cuda")
g = ws.gradient(raw, 1.0, ndim=3)
torch.cuda.synchronize()
slabs = shard.make_slabs(g.shape[0], K)
ctxs = [ws.Context(0) for _ in range(K)]
labels, R, rounds = shard.sharded_watershed(shard.LocalTransport(K), ctxs, slabs, [g[s.e0:s.e1].contiguous() for s in slabs])
ref, Rref = ws.watershed(g, 6)
print("equal", torch.equal(torch.cat(labels), ref), R, Rref, rounds)
