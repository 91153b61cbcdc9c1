import sys, torch
sys.path.insert(0, '/root/repo')
import synth
from paper_2410_08946_b200 import shard
g = synth.random_plateau_image((12, 33, 47), 3, seed=23).cuda()
lv, c, r = shard.segment_threads(int(sys.argv[1]) if len(sys.argv) > 1 else 2, g, 5, 6)
print("ok", c, r)
