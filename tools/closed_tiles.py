"""Measure the fraction of 32x8x8 tiles whose step II distances are final after the first
in-tile round ("closed": no face pair across the tile border joins two equal-valued plateau
voxels without a lower neighbour).  Analysis only."""
import sys
import torch
sys.path.insert(0, ".")
import synth
import paper_2410_08946_b200 as ws

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
raw = synth.make_config_image(name, device="cuda")
I = ws.gradient(raw, 1.0, ndim=3).int()
D, H, W = I.shape
BIG = 1 << 20
def sh(a, axis, d, fill):
    out = torch.full_like(a, fill); n = a.shape[axis]
    src = [slice(None)] * 3; dst = [slice(None)] * 3
    if d > 0: src[axis], dst[axis] = slice(d, n), slice(0, n - d)
    else: src[axis], dst[axis] = slice(0, n + d), slice(-d, n)
    out[tuple(dst)] = a[tuple(src)]; return out
lower = torch.zeros_like(I, dtype=torch.bool); eq = torch.zeros_like(lower)
for ax in range(3):
    for d in (-1, 1):
        n = sh(I, ax, d, BIG)
        lower |= n < I; eq |= n == I
PL = eq & ~lower
print("plateau-without-lower fraction %.3f" % PL.float().mean().item())
open_t = torch.zeros((D // 8, H // 8, W // 32), dtype=torch.bool, device="cuda")
tile = (8, 8, 32)
for ax in range(3):
    n_pl = sh(PL, ax, 1, False); n_I = sh(I, ax, 1, BIG)
    cross = PL & n_pl & (n_I == I)
    idx = torch.arange(I.shape[ax], device="cuda")
    border = ((idx + 1) % tile[ax] == 0)
    shape = [1, 1, 1]; shape[ax] = -1
    cross &= border.view(shape)
    c = cross.view(D // 8, 8, H // 8, 8, W // 32, 32).any(dim=5).any(dim=3).any(dim=1)
    # the tile on the other side of the face is open as well
    open_t |= c
    other = torch.zeros_like(c)
    sl_src = [slice(None)] * 3; sl_dst = [slice(None)] * 3
    sl_src[ax] = slice(0, c.shape[ax] - 1); sl_dst[ax] = slice(1, c.shape[ax])
    other[tuple(sl_dst)] = c[tuple(sl_src)]
    open_t |= other
print(name, "closed tiles %.3f of %d" % (1 - open_t.float().mean().item(), open_t.numel()))
