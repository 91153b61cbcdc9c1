"""Full-size check of the z-slab sharded path on ONE GPU: K virtual ranks (LocalTransport)
vs the unsharded ws_watershed + ws_waterfall on the same C4 volume.  Prints one JSON line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth
import paper_2410_08946_b200 as ws
from paper_2410_08946_b200 import shard

K = int(sys.argv[1]) if len(sys.argv) > 1 else 8
shape = tuple(int(x) for x in sys.argv[2].split(",")) if len(sys.argv) > 2 else (768, 1024, 1024)
NL = 6
raw = synth.make_config_image("C4", device="cuda", shape=shape)
grad = ws.gradient(raw, 1.0, ndim=3)
del raw
torch.cuda.synchronize()
t = time.time()
ref, R = ws.watershed(grad, 6)
rlv, rc = ws.waterfall(ref, grad, 6, NL)
torch.cuda.synchronize()
t_ref = time.time() - t
slabs = shard.make_slabs(shape[0], K)
ctxs = [ws.Context(0) for _ in range(K)]
grads = [grad[s.e0:s.e1].contiguous() for s in slabs]
for it in range(2):
    torch.cuda.synchronize()
    t = time.time()
    labels, levels, counts, Rs, rounds = shard.sharded_segment(shard.LocalTransport(K), ctxs, slabs, grads, NL)
    torch.cuda.synchronize()
    t_sh = time.time() - t
ok_l = all(torch.equal(labels[i], ref[s.z0:s.z1]) for i, s in enumerate(slabs))
ok_v = all(torch.equal(levels[i], rlv[:, s.z0:s.z1]) for i, s in enumerate(slabs))
print(json.dumps({"K": K, "shape": list(shape), "labels_equal": ok_l, "levels_equal": ok_v, "R": R, "R_sharded": Rs,
                  "counts": rc, "counts_sharded": counts, "plateau_rounds": rounds, "t_unsharded_s": t_ref,
                  "t_sharded_serial_s": t_sh,
                  "note": "K virtual ranks run one after another on one GPU: wall times are not a scaling number"}))
