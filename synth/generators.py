"""Seeded synthetic workloads shaped like the paper's inputs.

Every generator is deterministic for a given (shape, seed, device): it draws from a
``torch.Generator`` seeded with ``seed``.  CPU and CUDA generators give different bytes for
the same seed, so a consumer always feeds the SAME tensor to both the CUDA path and the
oracle (the tests copy device bytes to the host, never regenerate them).

Structure is built from value noise (a coarse random lattice upsampled with (tri)linear
interpolation), hard-edged shapes and additive Gaussian noise.  No blur, gradient or
watershed arithmetic lives here (those are the method; see ``oracle/`` and the CUDA path).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch
import torch.nn.functional as F

GENERATOR_VERSION = 1


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def _value_noise(shape, cell: float, g: torch.Generator, device) -> torch.Tensor:
    """Value noise in [-1, 1]: a random lattice with spacing ``cell`` voxels, upsampled
    (bi/tri)linearly to ``shape`` (2 or 3 dims)."""
    coarse = [max(2, int(math.ceil(s / cell)) + 1) for s in shape]
    lat = torch.rand(coarse, generator=g, device=device, dtype=torch.float32) * 2 - 1
    mode = "bilinear" if len(shape) == 2 else "trilinear"
    out = F.interpolate(lat[None, None], size=tuple(shape), mode=mode, align_corners=True)
    return out[0, 0]


def _to_u8(x: torch.Tensor) -> torch.Tensor:
    return x.round().clamp_(0, 255).to(torch.uint8)


# --------------------------------------------------------------------------------------
# C1: "cameraman-like" 2D image (Fig. 1 workload shape)
# --------------------------------------------------------------------------------------
def cameraman_like(H: int = 256, W: int = 256, seed: int = 1, device="cpu") -> torch.Tensor:
    g = _gen(seed, device)
    y = torch.arange(H, device=device, dtype=torch.float32)[:, None] / H
    x = torch.arange(W, device=device, dtype=torch.float32)[None, :] / W
    horizon = 0.45
    sky = 200.0 - 50.0 * (y / horizon)
    ground = 110.0 + 14.0 * _value_noise((H, W), max(2.0, H / 16), g, device) \
        + 6.0 * _value_noise((H, W), max(2.0, H / 64), g, device)
    img = torch.where(y < horizon, sky.expand(H, W), ground)
    # light distant buildings on the horizon
    for bx0, bx1, top, val in ((0.05, 0.14, 0.33, 178.0), (0.16, 0.21, 0.37, 184.0),
                               (0.74, 0.86, 0.35, 172.0), (0.88, 0.95, 0.39, 180.0)):
        m = (x >= bx0) & (x < bx1) & (y >= top) & (y < horizon + 0.02)
        img = torch.where(m, torch.full_like(img, val), img)
    # dark figure: head ellipse, torso, camera box, three thin tripod legs
    head = ((x - 0.42) / 0.05) ** 2 + ((y - 0.22) / 0.065) ** 2 <= 1
    torso = ((x - 0.43) / 0.11) ** 2 + ((y - 0.48) / 0.2) ** 2 <= 1
    camera = (x >= 0.52) & (x < 0.62) & (y >= 0.26) & (y < 0.33)
    img = torch.where(torso, torch.full_like(img, 30.0), img)
    img = torch.where(head, torch.full_like(img, 22.0), img)
    img = torch.where(camera, torch.full_like(img, 15.0), img)
    for (x0, x1) in ((0.57, 0.50), (0.57, 0.58), (0.57, 0.66)):
        # leg from (x0, 0.33) to (x1, 0.92), 1.5 px thick
        t = ((y - 0.33) / (0.92 - 0.33)).clamp(0, 1)
        xl = x0 + (x1 - x0) * t
        leg = (y >= 0.33) & (y <= 0.92) & ((x - xl).abs() * W <= 0.9)
        img = torch.where(leg, torch.full_like(img, 45.0), img)
    img = img + 2.0 * torch.randn((H, W), generator=g, device=device)
    return _to_u8(img)[None]  # (1, H, W)


# --------------------------------------------------------------------------------------
# C2: large 2D "synthetic gradient image": alpha-composited discs + value noise + noise
# --------------------------------------------------------------------------------------
def disc_composite(H: int = 8192, W: int = 8192, seed: int = 2, device="cpu",
                   n_discs: int | None = None) -> torch.Tensor:
    g = _gen(seed, device)
    if n_discs is None:
        n_discs = max(8, int(round(4000 * (H * W) / (8192 * 8192))))
    rmax = min(256.0, max(4.0, min(H, W) / 4))
    img = 128.0 + 10.0 * _value_noise((H, W), max(2.0, min(H, W) / 32), g, device)
    u = torch.rand((n_discs, 5), generator=g, device=device, dtype=torch.float64).cpu()
    for i in range(n_discs):
        r = 4.0 * (rmax / 4.0) ** float(u[i, 0])
        cy, cx = float(u[i, 1]) * H, float(u[i, 2]) * W
        val, alpha = 255.0 * float(u[i, 3]), 0.5 + 0.5 * float(u[i, 4])
        y0, y1 = max(0, int(cy - r)), min(H, int(cy + r) + 1)
        x0, x1 = max(0, int(cx - r)), min(W, int(cx + r) + 1)
        if y0 >= y1 or x0 >= x1:
            continue
        yy = torch.arange(y0, y1, device=device, dtype=torch.float32)[:, None] - cy
        xx = torch.arange(x0, x1, device=device, dtype=torch.float32)[None, :] - cx
        m = (yy * yy + xx * xx) <= r * r
        sub = img[y0:y1, x0:x1]
        img[y0:y1, x0:x1] = torch.where(m, sub * (1 - alpha) + alpha * val, sub)
    img = img + 3.0 * torch.randn((H, W), generator=g, device=device)
    return _to_u8(img)[None]


# --------------------------------------------------------------------------------------
# C3: "knee-MRI-like" 3D volume
# --------------------------------------------------------------------------------------
def knee_like(D: int = 512, H: int = 512, W: int = 512, seed: int = 3, device="cpu") -> torch.Tensor:
    g = _gen(seed, device)
    z = torch.linspace(-1, 1, D, device=device)[:, None, None]
    y = torch.linspace(-1, 1, H, device=device)[None, :, None]
    x = torch.linspace(-1, 1, W, device=device)[None, None, :]
    vol = torch.full((D, H, W), 4.0, device=device)
    soft = (x / 0.62) ** 2 + (y / 0.55) ** 2 <= 1
    vol = torch.where(soft, torch.full_like(vol, 90.0), vol)
    # fluid pocket
    fluid = ((x - 0.25) / 0.12) ** 2 + ((y + 0.2) / 0.1) ** 2 + (z / 0.15) ** 2 <= 1
    vol = torch.where(fluid & soft, torch.full_like(vol, 60.0), vol)
    # femur (upper, z<-0.05) and tibia (lower, z>0.05): capped elliptic cylinders
    for zc, sgn in ((-0.05, -1.0), (0.05, 1.0)):
        rad = ((x + 0.02) / 0.3) ** 2 + (y / 0.27) ** 2
        cap = ((z - zc) * sgn >= 0) | (rad + ((z - zc) / 0.25) ** 2 <= 1)
        inside = (rad <= 1) & ((z - zc) * sgn >= -0.25) & cap
        cart = inside & ((z - zc).abs() <= 0.018) | (
            (rad <= 1.0) & ((z - zc) * sgn < 0) & ((z - zc) * sgn > -0.02))
        marrow = (rad <= 0.7) & inside
        vol = torch.where(inside, torch.full_like(vol, 200.0), vol)
        vol = torch.where(marrow, torch.full_like(vol, 140.0), vol)
        vol = torch.where(cart & soft, torch.full_like(vol, 120.0), vol)
    bias = 1.0 + 0.15 * _value_noise((D, H, W), max(2.0, D / 3), g, device)
    vol = vol * bias + 6.0 * torch.randn((D, H, W), generator=g, device=device)
    return _to_u8(vol)


# --------------------------------------------------------------------------------------
# C4: "microCT-like" porous two-phase medium (the metric workload)
# --------------------------------------------------------------------------------------
def microct_like(D: int = 768, H: int = 1024, W: int = 1024, seed: int = 4, device="cpu",
                 cell: float = 4.0, solid_fraction: float = 0.45) -> torch.Tensor:
    """Threshold a correlated random field at its 55% quantile (pore 60 / solid 200) and add
    Gaussian noise sigma=12.  The correlated field is value noise with lattice spacing
    ``cell`` (correlation length ~2.5 voxels like the recipe's sigma_c=2.5)."""
    g = _gen(seed, device)
    field = _value_noise((D, H, W), cell, g, device)
    flat = field.reshape(-1)
    step = max(1, flat.numel() // (1 << 22))
    sample = flat[::step]
    k = max(1, int(round((1.0 - solid_fraction) * sample.numel())))
    thr = sample.kthvalue(k).values
    vol = torch.where(field > thr, 200.0, 60.0)
    del field, flat, sample
    vol += 12.0 * torch.randn((D, H, W), generator=g, device=device)
    return _to_u8(vol)


# --------------------------------------------------------------------------------------
# C5: batch of 145x145 HSI-band-derived images ("compressed image")
# --------------------------------------------------------------------------------------
def hsi_batch(B: int = 1024, H: int = 145, W: int = 145, seed: int = 5, device="cpu",
              n_classes: int = 16, bands: int = 200) -> torch.Tensor:
    g = _gen(seed, device)
    lam = torch.linspace(0, 1, bands, device=device)
    out = torch.empty((B, H, W), dtype=torch.uint8, device=device)
    yy = torch.arange(H, device=device, dtype=torch.float32)[:, None, None]
    xx = torch.arange(W, device=device, dtype=torch.float32)[None, :, None]
    # per-class smooth spectra, band-averaged -> one intensity per class
    coef = torch.rand((n_classes, 3, 3), generator=g, device=device)
    spectra = 60 + 140 * (coef[:, :, 0:1] * torch.sin(
        math.pi * (1 + 3 * coef[:, :, 1:2]) * lam + 6.28 * coef[:, :, 2:3])).mean(1).abs()
    class_val = spectra.mean(-1)  # (n_classes,)
    class_sd = 0.02 * spectra.mean(-1) / math.sqrt(bands) * 10.0
    for b in range(B):
        ns = int(torch.randint(8, 41, (1,), generator=g, device=device))
        sy = torch.rand((ns,), generator=g, device=device) * H
        sx = torch.rand((ns,), generator=g, device=device) * W
        cls = torch.randint(0, n_classes, (ns,), generator=g, device=device)
        d2 = (yy - sy) ** 2 + (xx - sx) ** 2
        lab = cls[d2.argmin(-1)]
        img = class_val[lab] + class_sd[lab] * torch.randn((H, W), generator=g, device=device)
        out[b] = _to_u8(img)
    return out


# --------------------------------------------------------------------------------------
# stress inputs
# --------------------------------------------------------------------------------------
def random_plateau_image(shape, levels: int = 4, seed: int = 0, device="cpu") -> torch.Tensor:
    """i.i.d. values in {0..levels-1}: forces plateaux of every kind."""
    g = _gen(seed, device)
    return torch.randint(0, levels, tuple(shape), generator=g, device=device, dtype=torch.int64).to(torch.uint8)


@dataclass(frozen=True)
class Config:
    name: str
    ndim: int          # 2: (batch, H, W) independent images; 3: volume (D, H, W)
    shape: tuple       # full size (outermost first)
    conn: int
    sigma: float
    NL: int
    seed: int
    desc: str


CONFIGS = {
    "C1": Config("C1", 2, (1, 256, 256), 4, 1.0, 6, 1,
                 "2D 256x256 cameraman-like, 4-conn, sigma=1, NL=6"),
    "C2": Config("C2", 2, (1, 8192, 8192), 8, 1.0, 6, 2,
                 "2D 8192x8192 disc composite, 8-conn, sigma=1, NL=6"),
    "C3": Config("C3", 3, (512, 512, 512), 6, 1.0, 6, 3,
                 "3D 512^3 knee-MRI-like, 6-conn, sigma=1, NL=6"),
    "C4": Config("C4", 3, (768, 1024, 1024), 6, 1.0, 6, 4,
                 "3D 1024x1024x768 microCT-like (805 Mvox), 6-conn, sigma=1, NL=6"),
    "C5": Config("C5", 2, (1024, 145, 145), 4, 1.0, 4, 5,
                 "batch of 1024 145x145 HSI-band-derived images, 4-conn, sigma=1, NL=4"),
}


def make_config_image(name: str, device="cpu", shape=None, seed_offset: int = 0) -> torch.Tensor:
    """Raw u8 input of config ``name`` (optionally at a reduced ``shape``; ``seed_offset``
    gives independent volumes of the same recipe, e.g. one per rank)."""
    c = CONFIGS[name]
    s = tuple(shape) if shape is not None else c.shape
    seed = c.seed + seed_offset
    if name == "C1":
        return cameraman_like(s[1], s[2], seed, device)
    if name == "C2":
        return disc_composite(s[1], s[2], seed, device)
    if name == "C3":
        return knee_like(s[0], s[1], s[2], seed, device)
    if name == "C4":
        return microct_like(s[0], s[1], s[2], seed, device)
    if name == "C5":
        return hsi_batch(s[0], s[1], s[2], seed, device)
    raise KeyError(name)
