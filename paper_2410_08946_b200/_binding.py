"""Thin ctypes binding of libws_b200.so (include/ws.h).  Argument marshalling ONLY: every step
of the hot path runs in the library's CUDA kernels.  There is no CPU or PyTorch fallback:
if the shared library is missing or a call fails, this raises."""
from __future__ import annotations

import ctypes
import os
import threading

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(_HERE, "libws_b200.so")

WS_OK, WS_ERR_INVALID, WS_ERR_OOM, WS_ERR_CUDA, WS_ERR_NCCL, WS_ERR_INTERNAL, WS_ERR_LIMIT = range(7)
STATUS_NAMES = {0: "WS_OK", 1: "WS_ERR_INVALID", 2: "WS_ERR_OOM", 3: "WS_ERR_CUDA", 4: "WS_ERR_NCCL",
                5: "WS_ERR_INTERNAL", 6: "WS_ERR_LIMIT"}

# every symbol include/ws.h declares (checked by tests/test_abi.py)
EXPORTS = ("ws_ctx_create", "ws_ctx_destroy", "ws_last_error", "ws_version", "ws_get_stats",
           "ws_ctx_set_timing", "ws_phase_name",
           "ws_gradient", "ws_gradient_u16", "ws_watershed", "ws_watershed_u16", "ws_watershed_variant", "ws_waterfall", "ws_waterfall_u16", "ws_waterfall_reconstruct", "ws_segment", "ws_segment_host", "ws_segment_host_async", "ws_plateau_debug",
           "ws_shard_table_bytes", "ws_shard_plateau", "ws_shard_halo", "ws_shard_local", "ws_shard_merge",
           "ws_shard_relabel", "ws_shard_wf_dense", "ws_shard_wf_btable", "ws_shard_wf_bfill", "ws_shard_wf_begin",
           "ws_shard_wf_step", "ws_shard_wf_end",
           "ws_nccl_unique_id", "ws_transport_nccl_create", "ws_transport_nccl_destroy", "ws_ctx_create_sharded",
           "ws_watershed_sharded", "ws_waterfall_sharded", "ws_segment_sharded", "ws_watershed_sharded_u16",
           "ws_waterfall_sharded_u16", "ws_segment_sharded_u16")


class WsDims(ctypes.Structure):
    _fields_ = [("ndim", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("n0", ctypes.c_int64), ("n1", ctypes.c_int64), ("n2", ctypes.c_int64)]


class WsSlab(ctypes.Structure):
    _fields_ = [("D", ctypes.c_int64), ("z0", ctypes.c_int64), ("z1", ctypes.c_int64), ("e0", ctypes.c_int64),
                ("e1", ctypes.c_int64)]


# ws_transport (include/ws.h): the callbacks of the sharded pipeline
EXCHANGE_FN = ctypes.CFUNCTYPE(ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                               ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p)
ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                ctypes.c_void_p)
ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                                ctypes.c_int32, ctypes.c_void_p)


class WsTransport(ctypes.Structure):
    _fields_ = [("user", ctypes.c_void_p), ("rank", ctypes.c_int32), ("nranks", ctypes.c_int32),
                ("exchange", EXCHANGE_FN), ("allgather", ALLGATHER_FN), ("allreduce", ALLREDUCE_FN)]


class WsStats(ctypes.Structure):
    _fields_ = [("n_voxels", ctypes.c_int64), ("n_regions", ctypes.c_int64), ("n_edges", ctypes.c_int64),
                ("plateau_rounds", ctypes.c_int32), ("waterfall_levels", ctypes.c_int32),
                ("level_counts", ctypes.c_int64 * 16), ("kernel_launches", ctypes.c_int64),
                ("phase_ms", ctypes.c_double * 16), ("phase_launches", ctypes.c_int32 * 16),
                ("tma", ctypes.c_int32), ("reserved0", ctypes.c_int32), ("level_edges", ctypes.c_int64 * 16),
                ("total_launches", ctypes.c_int64), ("union_order", ctypes.c_int32),
                ("root_overflow", ctypes.c_int32), ("lookback_max", ctypes.c_int32),
                ("edge_chunks_max", ctypes.c_int32), ("rag_global_emits", ctypes.c_int64),
                ("rag_records", ctypes.c_int64)]

    def as_dict(self):
        lib = load()
        phases = {}
        for i in range(16):
            name = lib.ws_phase_name(i).decode()
            if name and (self.phase_launches[i] or self.phase_ms[i]):
                phases[name] = {"ms": self.phase_ms[i], "launches": self.phase_launches[i]}
        return {"n_voxels": self.n_voxels, "n_regions": self.n_regions, "n_edges": self.n_edges,
                "plateau_rounds": self.plateau_rounds, "waterfall_levels": self.waterfall_levels,
                "level_counts": list(self.level_counts), "kernel_launches": self.kernel_launches,
                "phases": phases, "tma": self.tma, "level_edges": list(self.level_edges),
                "total_launches": self.total_launches, "union_order": self.union_order,
                "root_overflow": self.root_overflow, "lookback_max": self.lookback_max,
                "edge_chunks_max": self.edge_chunks_max, "rag_global_emits": self.rag_global_emits,
                "rag_records": self.rag_records}


class WsError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__("%s: %s" % (STATUS_NAMES.get(status, status), msg))
        self.status = status


_lib = None
_lock = threading.Lock()


def load(path: str = SO_PATH):
    """Load the CUDA library (raises if it is not built — no fallback)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise ImportError("libws_b200.so not built (%s); run __graft_entry__.build()" % path)
        lib = ctypes.CDLL(path)
        vp, i32, i64, f32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_float
        lib.ws_ctx_create.argtypes = [i32, ctypes.POINTER(vp)]
        lib.ws_ctx_destroy.argtypes = [vp]
        lib.ws_last_error.restype = ctypes.c_char_p
        lib.ws_version.restype = ctypes.c_char_p
        lib.ws_get_stats.argtypes = [vp, ctypes.POINTER(WsStats)]
        lib.ws_ctx_set_timing.argtypes = [vp, i32]
        lib.ws_phase_name.argtypes = [i32]
        lib.ws_phase_name.restype = ctypes.c_char_p
        lib.ws_gradient.argtypes = [vp, vp, WsDims, f32, vp, vp, vp, vp]
        lib.ws_gradient_u16.argtypes = [vp, vp, WsDims, f32, vp, vp, vp, vp]
        lib.ws_watershed.argtypes = [vp, vp, WsDims, i32, vp, vp, vp]
        lib.ws_watershed_u16.argtypes = [vp, vp, WsDims, i32, vp, vp, vp]
        lib.ws_waterfall.argtypes = [vp, vp, vp, WsDims, i32, i32, vp, vp, vp]
        lib.ws_waterfall_reconstruct.argtypes = [vp, vp, vp, WsDims, i32, i32, vp, vp, vp]
        lib.ws_waterfall_u16.argtypes = [vp, vp, vp, WsDims, i32, i32, vp, vp, vp]
        lib.ws_watershed_variant.argtypes = [vp, vp, WsDims, i32, i32, vp, vp, vp]
        lib.ws_segment_host.argtypes = [vp, vp, WsDims, i32, i32, vp, vp, vp]
        lib.ws_segment_host_async.argtypes = [vp, vp, WsDims, i32, i32, vp, vp, vp]
        lib.ws_segment.argtypes = [vp, vp, WsDims, i32, i32, vp, vp, vp]
        lib.ws_plateau_debug.argtypes = [vp, vp, WsDims, i32, vp, vp, vp]
        lib.ws_shard_table_bytes.argtypes = [WsDims]
        lib.ws_shard_table_bytes.restype = ctypes.c_int64
        pi32 = ctypes.POINTER(ctypes.c_int32)
        lib.ws_shard_plateau.argtypes = [vp, vp, WsDims, i32, WsSlab, vp, i32, i32, i32, pi32, vp]
        lib.ws_shard_halo.argtypes = [vp, vp, WsDims, WsSlab, i32, vp, pi32, vp]
        lib.ws_shard_local.argtypes = [vp, vp, vp, WsDims, i32, WsSlab, vp, vp, vp]
        lib.ws_shard_merge.argtypes = [vp, vp, i32, vp, vp, WsDims, WsSlab, vp, vp, vp]
        lib.ws_shard_relabel.argtypes = [vp, vp, vp, vp, WsDims, WsSlab, vp, vp, vp]
        lib.ws_shard_wf_dense.argtypes = [vp, vp, WsDims, WsSlab, i64, vp, vp, vp, vp]
        lib.ws_shard_wf_btable.argtypes = [vp, vp, vp, WsDims, WsSlab, vp, vp]
        lib.ws_shard_wf_bfill.argtypes = [vp, vp, i32, WsDims, WsSlab, vp, vp]
        lib.ws_shard_wf_begin.argtypes = [vp, vp, vp, WsDims, i32, WsSlab, vp, i64, i32, vp, vp]
        lib.ws_shard_wf_step.argtypes = [vp, vp, vp, vp, pi32, vp]
        lib.ws_shard_wf_end.argtypes = [vp, vp, vp, vp, WsDims, i32, WsSlab, vp, vp]
        ptr_t = ctypes.POINTER(WsTransport)
        lib.ws_nccl_unique_id.argtypes = [vp]
        lib.ws_transport_nccl_create.argtypes = [vp, i32, i32, i32, ctypes.POINTER(ptr_t)]
        lib.ws_transport_nccl_destroy.argtypes = [ptr_t]
        lib.ws_ctx_create_sharded.argtypes = [i32, ptr_t, WsSlab, ctypes.POINTER(vp)]
        lib.ws_watershed_sharded.argtypes = [vp, ptr_t, vp, WsDims, WsSlab, i32, vp, ctypes.POINTER(i64), pi32, vp]
        lib.ws_waterfall_sharded.argtypes = [vp, ptr_t, vp, vp, WsDims, WsSlab, i32, i32, vp, vp, vp]
        lib.ws_segment_sharded.argtypes = [vp, ptr_t, vp, WsDims, WsSlab, i32, i32, vp, vp, pi32, vp]
        lib.ws_watershed_sharded_u16.argtypes = lib.ws_watershed_sharded.argtypes
        lib.ws_waterfall_sharded_u16.argtypes = lib.ws_waterfall_sharded.argtypes
        lib.ws_segment_sharded_u16.argtypes = lib.ws_segment_sharded.argtypes
        for name in EXPORTS:
            f = getattr(lib, name)
            if name not in ("ws_last_error", "ws_version", "ws_phase_name", "ws_shard_table_bytes"):
                f.restype = ctypes.c_int
        _lib = lib
        return lib


def check(status):
    if status != WS_OK:
        raise WsError(status, load().ws_last_error().decode(errors="replace"))


class Context:
    """Owns one ws_ctx (device workspace) for one CUDA device."""

    def __init__(self, device: int = None):
        lib = load()
        if device is None:
            device = torch.cuda.current_device()
        self.device = int(device)
        h = ctypes.c_void_p()
        check(lib.ws_ctx_create(self.device, ctypes.byref(h)))
        self.handle = h

    def close(self):
        if getattr(self, "handle", None):
            load().ws_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_timing(self, enable: bool = True):
        check(load().ws_ctx_set_timing(self.handle, 1 if enable else 0))

    def stats(self) -> dict:
        s = WsStats()
        check(load().ws_get_stats(self.handle, ctypes.byref(s)))
        return s.as_dict()


_ctxs = {}


def default_context(device: int = None) -> Context:
    if device is None:
        device = torch.cuda.current_device()
    if device not in _ctxs:
        _ctxs[device] = Context(device)
    return _ctxs[device]


def dims_of(shape, ndim: int) -> WsDims:
    shape = tuple(int(s) for s in shape)
    if len(shape) == 1:
        shape = (1, 1) + shape
    elif len(shape) == 2:
        shape = (1,) + shape
    if len(shape) != 3:
        raise ValueError("expected a 1-, 2- or 3-D tensor, got shape %s" % (shape,))
    return WsDims(int(ndim), 0, *shape)


def ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def stream_of(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)
