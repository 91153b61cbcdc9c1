"""B200-native (sm_100a) hot path of arXiv 2410.08946, "Parallel Watershed Partitioning".

Python API (same names as the C ABI in include/ws.h; argument marshalling only):

    grad_q              = gradient(img, sigma, ndim)             # ws_gradient
    labels, R           = watershed(grad, conn)                  # ws_watershed
    levels, counts      = waterfall(labels, grad, conn, NL)      # ws_waterfall
    levels, counts      = segment(grad, conn, NL)                # ws_segment (both, one call)
    levels_h, counts    = segment_host(grad_host, conn, NL)      # ws_segment_host (host buffers)

Tensors live on a CUDA device (PyTorch is used for device memory and streams only); work is
enqueued on the current torch stream.  ``ndim`` is 2 for (batch, H, W) image stacks (4/8-conn)
and 3 for (D, H, W) volumes (6/26-conn); it defaults from ``conn``.
"""
from __future__ import annotations

import ctypes

import torch

from . import _binding as _b
from ._binding import Context, WsError, default_context  # noqa: F401

__all__ = ["gradient", "watershed", "waterfall", "segment", "segment_host", "plateau_debug", "stats", "Context",
           "WsError", "version"]


def version() -> str:
    return _b.load().ws_version().decode()


def _ndim_for(conn, ndim):
    if ndim is not None:
        return int(ndim)
    return 3 if conn in (6, 26) else 2


def _req(t, dtype, name):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError("%s must be a CUDA tensor" % name)
    if t.dtype != dtype:
        raise TypeError("%s must be %s (got %s)" % (name, dtype, t.dtype))
    if not t.is_contiguous():
        raise ValueError("%s must be contiguous" % name)


def _req_out(t, dtype, shape, like, name):
    """Validate a caller-supplied output tensor before its pointer reaches the library."""
    _req(t, dtype, name)
    if tuple(t.shape) != tuple(shape):
        raise ValueError("%s must have shape %s (got %s)" % (name, tuple(shape), tuple(t.shape)))
    if t.device != like.device:
        raise ValueError("%s must be on %s (got %s)" % (name, like.device, t.device))


def gradient(img: torch.Tensor, sigma: float = 1.0, ndim: int = None, verify: bool = False,
             ctx: Context = None, out: torch.Tensor = None):
    """ws_gradient: u8 image -> agreed u8 gradient image (and fp32 blur/grad if ``verify``).
    A torch.uint16 image runs ws_gradient_u16 (16-bit in, 16-bit gradient out, NEXT f4)."""
    wide = isinstance(img, torch.Tensor) and img.dtype == torch.uint16
    _req(img, torch.uint16 if wide else torch.uint8, "img")
    ndim = ndim if ndim is not None else (3 if img.dim() == 3 and img.shape[0] > 1 else 2)
    ctx = ctx or default_context(img.device.index)
    if out is not None:
        _req_out(out, img.dtype, img.shape, img, "out")
    q = out if out is not None else torch.empty_like(img)
    blur = torch.empty(img.shape, dtype=torch.float32, device=img.device) if verify else None
    grad = torch.empty(img.shape, dtype=torch.float32, device=img.device) if verify else None
    fn = _b.load().ws_gradient_u16 if wide else _b.load().ws_gradient
    _b.check(fn(ctx.handle, _b.ptr(img), _b.dims_of(img.shape, ndim), float(sigma),
                                   _b.ptr(q), _b.ptr(blur), _b.ptr(grad), _b.stream_of(img)))
    return (q, blur, grad) if verify else q


VARIANTS = {"pruf_sync": 0, "prw_sync": 1, "apruf_sync": 2}


def watershed(grad: torch.Tensor, conn: int, ndim: int = None, ctx: Context = None,
              out: torch.Tensor = None, variant: str = None):
    """ws_watershed: canonical labels (int32, shaped like grad) and the region count R.
    variant="pruf_sync" | "prw_sync" | "apruf_sync": the paper's one-thread-per-voxel kernels
    (ws_watershed_variant, Alg. 1 / Alg. 2 / APRUF) instead of the tiled design.
    A torch.uint16 grad runs ws_watershed_u16 (16-bit images, NEXT f4; tiled design only)."""
    wide = isinstance(grad, torch.Tensor) and grad.dtype == torch.uint16
    _req(grad, torch.uint16 if wide else torch.uint8, "grad")
    ndim = _ndim_for(conn, ndim)
    ctx = ctx or default_context(grad.device.index)
    if out is not None:
        _req_out(out, torch.int32, grad.shape, grad, "out")
    labels = out if out is not None else torch.empty(grad.shape, dtype=torch.int32, device=grad.device)
    R = ctypes.c_int64(0)
    if wide:
        if variant is not None:
            raise ValueError("the paper's kernel variants take u8 images")
        _b.check(_b.load().ws_watershed_u16(ctx.handle, _b.ptr(grad), _b.dims_of(grad.shape, ndim), int(conn),
                                            _b.ptr(labels), ctypes.byref(R), _b.stream_of(grad)))
    elif variant is None:
        _b.check(_b.load().ws_watershed(ctx.handle, _b.ptr(grad), _b.dims_of(grad.shape, ndim), int(conn),
                                        _b.ptr(labels), ctypes.byref(R), _b.stream_of(grad)))
    else:
        if variant not in VARIANTS:
            raise ValueError("variant must be one of %s" % sorted(VARIANTS))
        _b.check(_b.load().ws_watershed_variant(ctx.handle, _b.ptr(grad), _b.dims_of(grad.shape, ndim), int(conn),
                                                VARIANTS[variant], _b.ptr(labels), ctypes.byref(R),
                                                _b.stream_of(grad)))
    return labels, R.value


def waterfall(labels: torch.Tensor, grad: torch.Tensor, conn: int, NL: int, ndim: int = None,
              ctx: Context = None, out: torch.Tensor = None, mode: str = "graph"):
    """ws_waterfall: levels (int32 [NL, *shape], level 0 = labels) and per-level counts.
    mode="graph": the nested graph waterfall (C13); mode="reconstruct": the paper-literal
    waterfall by image reconstruction (ws_waterfall_reconstruct, Alg. 4 V-VI + Alg. 5).
    A torch.uint16 grad runs ws_waterfall_u16 (16-bit pass heights, NEXT f4; graph mode)."""
    if mode not in ("graph", "reconstruct"):
        raise ValueError("mode must be 'graph' or 'reconstruct'")
    _req(labels, torch.int32, "labels")
    wide = isinstance(grad, torch.Tensor) and grad.dtype == torch.uint16
    if wide and mode != "graph":
        raise ValueError("the reconstruct waterfall takes u8 images")
    _req(grad, torch.uint16 if wide else torch.uint8, "grad")
    if labels.shape != grad.shape:
        raise ValueError("labels and grad shapes differ")
    ndim = _ndim_for(conn, ndim)
    ctx = ctx or default_context(grad.device.index)
    if labels.device != grad.device:
        raise ValueError("labels and grad must be on the same device")
    if out is not None:
        _req_out(out, torch.int32, (max(int(NL), 1),) + tuple(grad.shape), grad, "out")
    levels = out if out is not None else torch.empty((max(int(NL), 1),) + tuple(grad.shape), dtype=torch.int32,
                                                      device=grad.device)
    counts = (ctypes.c_int64 * max(int(NL), 1))()
    fn = _b.load().ws_waterfall if mode == "graph" else _b.load().ws_waterfall_reconstruct
    if wide:
        fn = _b.load().ws_waterfall_u16
    _b.check(fn(ctx.handle, _b.ptr(labels), _b.ptr(grad), _b.dims_of(grad.shape, ndim), int(conn), int(NL),
                _b.ptr(levels), counts, _b.stream_of(grad)))
    return levels, list(counts)


def segment(grad: torch.Tensor, conn: int, NL: int, ndim: int = None, ctx: Context = None,
            out: torch.Tensor = None):
    """ws_segment: ws_watershed + ws_waterfall(NL) as one call (Alg. 5).  Returns
    (levels int32 [NL, *shape] with levels[0] = the canonical labels, counts)."""
    _req(grad, torch.uint8, "grad")
    ndim = _ndim_for(conn, ndim)
    ctx = ctx or default_context(grad.device.index)
    if out is not None:
        _req_out(out, torch.int32, (max(int(NL), 1),) + tuple(grad.shape), grad, "out")
    levels = out if out is not None else torch.empty((max(int(NL), 1),) + tuple(grad.shape), dtype=torch.int32,
                                                      device=grad.device)
    counts = (ctypes.c_int64 * max(int(NL), 1))()
    _b.check(_b.load().ws_segment(ctx.handle, _b.ptr(grad), _b.dims_of(grad.shape, ndim), int(conn), int(NL),
                                  _b.ptr(levels), counts, _b.stream_of(grad)))
    return levels, list(counts)


def segment_host(grad_host: torch.Tensor, conn: int, NL: int, ndim: int = None, device: int = None,
                 ctx: Context = None, out: torch.Tensor = None, stream: torch.cuda.Stream = None,
                 wait: bool = True):
    """ws_segment_host: HOST u8 gradient -> HOST int32 levels [NL, *shape] (copies inside).
    wait=False calls ws_segment_host_async: the levels are ready once `stream` (default: the
    current stream) is synchronised."""
    if grad_host.is_cuda or grad_host.dtype != torch.uint8 or not grad_host.is_contiguous():
        raise TypeError("grad_host must be a contiguous CPU uint8 tensor")
    ndim = _ndim_for(conn, ndim)
    ctx = ctx or default_context(device)
    if out is not None and (out.is_cuda or out.dtype != torch.int32 or not out.is_contiguous()
                            or tuple(out.shape) != (int(NL),) + tuple(grad_host.shape)):
        raise ValueError("out must be a contiguous CPU int32 tensor of shape %s" % (((int(NL),) + tuple(grad_host.shape)),))
    levels = out if out is not None else torch.empty((int(NL),) + tuple(grad_host.shape), dtype=torch.int32,
                                                      pin_memory=True)
    counts = (ctypes.c_int64 * max(int(NL), 1))()
    st = ctypes.c_void_p((stream or torch.cuda.current_stream(ctx.device)).cuda_stream)
    fn = _b.load().ws_segment_host if wait else _b.load().ws_segment_host_async
    _b.check(fn(ctx.handle, _b.ptr(grad_host), _b.dims_of(grad_host.shape, ndim), int(conn), int(NL), _b.ptr(levels),
                counts, st))
    return levels, list(counts)


def plateau_debug(grad: torch.Tensor, conn: int, ndim: int = None, ctx: Context = None):
    """ws_plateau_debug: (dist, parent) after steps I-II (per-kernel parity, T2)."""
    _req(grad, torch.uint8, "grad")
    ndim = _ndim_for(conn, ndim)
    ctx = ctx or default_context(grad.device.index)
    dist = torch.empty(grad.shape, dtype=torch.int32, device=grad.device)
    parent = torch.empty(grad.shape, dtype=torch.int32, device=grad.device)
    _b.check(_b.load().ws_plateau_debug(ctx.handle, _b.ptr(grad), _b.dims_of(grad.shape, ndim), int(conn),
                                        _b.ptr(dist), _b.ptr(parent), _b.stream_of(grad)))
    return dist, parent


def stats(device: int = None) -> dict:
    """Statistics of the last call on the default context of ``device``."""
    return default_context(device).stats()
