"""ctypes wrapper of the C++ oracle (``oracle/ws_oracle.cpp``).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The product path
(``paper_2410_08946_b200``) never imports it and shares no code with it.

Arrays are numpy; shapes are ``(n0, n1, n2)`` with ``ndim`` 2 (n0 independent 2D images)
or 3 (one volume).  All functions are single-threaded and slow by design.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libws_oracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with g++ (-O2, single-threaded).  Returns the .so path."""
    src = os.path.join(_HERE, "ws_oracle.cpp")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-o", _SO, src])
    return _SO


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        i64, i32, dbl, vp = ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_void_p
        lib.oracle_gradient.argtypes = [vp, i32, i64, i64, i64, dbl, vp, vp, vp]
        lib.oracle_watershed.argtypes = [vp, i32, i64, i64, i64, i32, vp, vp, vp, vp]
        lib.oracle_waterfall.argtypes = [vp, vp, i32, i64, i64, i64, i32, i32, vp, vp]
        lib.oracle_waterfall_reconstruct.argtypes = [vp, vp, i32, i64, i64, i64, i32, i32, vp, vp]
        lib.oracle_watershed_u16.argtypes = lib.oracle_watershed.argtypes
        lib.oracle_waterfall_u16.argtypes = lib.oracle_waterfall.argtypes
        lib.oracle_waterfall_u16.restype = ctypes.c_int
        lib.oracle_gradient_u16.argtypes = lib.oracle_gradient.argtypes
        lib.oracle_gradient_u16.restype = ctypes.c_int
        for f in (lib.oracle_gradient, lib.oracle_watershed, lib.oracle_watershed_u16, lib.oracle_waterfall,
                  lib.oracle_waterfall_reconstruct):
            f.restype = ctypes.c_int
        _lib = lib
    return _lib


def _shape3(a: np.ndarray, ndim: int):
    if a.ndim == 1:
        a = a.reshape(1, 1, -1)
    elif a.ndim == 2:
        a = a.reshape((1,) + a.shape)
    if a.ndim != 3:
        raise ValueError("expected a 1-, 2- or 3-D array")
    if ndim not in (2, 3):
        raise ValueError("ndim must be 2 or 3")
    return np.ascontiguousarray(a), a.shape


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def gradient(img: np.ndarray, sigma: float, ndim: int = None):
    """O1+O2: returns (blur f64, grad f64, grad_q u8), each shaped like ``img``.  A np.uint16
    image uses x / 65535 and 16-bit quantisation (O11, NEXT f4; grad_q u16)."""
    orig = img.shape
    if ndim is None:
        ndim = 3 if img.ndim == 3 else 2
    wide = isinstance(img, np.ndarray) and img.dtype == np.uint16
    a, (n0, n1, n2) = _shape3(np.asarray(img, dtype=np.uint16 if wide else np.uint8), ndim)
    blur = np.empty(a.shape, np.float64)
    grad = np.empty(a.shape, np.float64)
    q = np.empty(a.shape, np.uint16 if wide else np.uint8)
    fn = _load().oracle_gradient_u16 if wide else _load().oracle_gradient
    rc = fn(_p(a), ndim, n0, n1, n2, float(sigma), _p(blur), _p(grad), _p(q))
    if rc != 0:
        raise ValueError("oracle_gradient: invalid arguments")
    return blur.reshape(orig), grad.reshape(orig), q.reshape(orig)


def watershed(grad: np.ndarray, conn: int, ndim: int = None, dumps: bool = False):
    """O3+O4: canonical labels (int32).  With ``dumps`` also (dist int32, ptr int64, R).
    A np.uint16 image runs the same definition on 16-bit intensities (O10, NEXT f4)."""
    orig = grad.shape
    if ndim is None:
        ndim = 3 if conn in (6, 26) else 2
    wide = isinstance(grad, np.ndarray) and grad.dtype == np.uint16
    a, (n0, n1, n2) = _shape3(np.asarray(grad, dtype=np.uint16 if wide else np.uint8), ndim)
    labels = np.empty(a.shape, np.int32)
    dist = np.empty(a.shape, np.int32) if dumps else None
    ptr = np.empty(a.shape, np.int64) if dumps else None
    R = ctypes.c_int64(0)
    fn = _load().oracle_watershed_u16 if wide else _load().oracle_watershed
    rc = fn(_p(a), ndim, n0, n1, n2, int(conn), _p(labels), _p(dist), _p(ptr),
            ctypes.byref(R))
    if rc != 0:
        raise ValueError("oracle_watershed: invalid arguments")
    if dumps:
        return labels.reshape(orig), dist.reshape(orig), ptr.reshape(orig), R.value
    return labels.reshape(orig)


def waterfall(labels: np.ndarray, grad: np.ndarray, conn: int, NL: int, ndim: int = None):
    """O6+O7: (levels int32 [NL, *shape], counts int64 [NL]).  A np.uint16 image uses 16-bit
    pass heights (O12, NEXT f4)."""
    orig = grad.shape
    if ndim is None:
        ndim = 3 if conn in (6, 26) else 2
    wide = isinstance(grad, np.ndarray) and grad.dtype == np.uint16
    g, (n0, n1, n2) = _shape3(np.asarray(grad, dtype=np.uint16 if wide else np.uint8), ndim)
    lab = np.ascontiguousarray(np.asarray(labels, dtype=np.int32).reshape(g.shape))
    levels = np.empty((max(NL, 1),) + g.shape, np.int32)
    counts = np.empty(max(NL, 1), np.int64)
    fn = _load().oracle_waterfall_u16 if wide else _load().oracle_waterfall
    rc = fn(_p(lab), _p(g), ndim, n0, n1, n2, int(conn), int(NL), _p(levels), _p(counts))
    if rc != 0:
        raise ValueError("oracle_waterfall: invalid arguments")
    return levels.reshape((NL,) + orig), counts


def waterfall_reconstruct(labels: np.ndarray, grad: np.ndarray, conn: int, NL: int, ndim: int = None):
    """O9, the paper-literal waterfall (Alg. 4 steps V-VI + watershed per layer, Alg. 5):
    (levels int32 [NL, *shape], counts int64 [NL])."""
    orig = grad.shape
    if ndim is None:
        ndim = 3 if conn in (6, 26) else 2
    g, (n0, n1, n2) = _shape3(np.asarray(grad, dtype=np.uint8), ndim)
    lab = np.ascontiguousarray(np.asarray(labels, dtype=np.int32).reshape(g.shape))
    levels = np.empty((max(NL, 1),) + g.shape, np.int32)
    counts = np.empty(max(NL, 1), np.int64)
    rc = _load().oracle_waterfall_reconstruct(_p(lab), _p(g), ndim, n0, n1, n2, int(conn), int(NL), _p(levels),
                                              _p(counts))
    if rc != 0:
        raise ValueError("oracle_waterfall_reconstruct: invalid arguments")
    return levels.reshape((NL,) + orig), counts
