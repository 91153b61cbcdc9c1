"""z-slab sharded watershed (north_star: "3D volumes are partitioned along z into slabs across
the 8 GPUs of one box, with NCCL halo exchange over NVLink and a cross-slab boundary
union-find merge").

SPMD orchestration of the ws_shard_* C-ABI phases (every compute step runs in the library's
kernels).  Planes move between ranks through a Transport:

  DistTransport   one process per GPU, torch.distributed (NCCL over NVLink / NVSwitch, or
                  gloo for host-only tests): batched P2P halo planes, all_gather of the
                  boundary tables, all_reduce(max) of the convergence flags;
  LocalTransport  K virtual ranks in ONE process on one device (in-process plane copies) —
                  the single-GPU test bed: sharded(K) must equal the unsharded result.

The code below always iterates over the ranks a process holds (K for LocalTransport, 1 for
DistTransport); collectives take / return one value per held rank.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _binding as _b

HALO = 2  # extended slab: grad planes z0-2 .. z1+1 (step I of the halo plane needs its neighbours)


@dataclass(frozen=True)
class Slab:
    rank: int
    K: int
    D: int
    z0: int
    z1: int
    e0: int
    e1: int

    @property
    def zlo(self):
        return self.z0 - self.e0

    @property
    def zhi(self):
        return self.z1 - self.e0

    def c(self):
        return _b.WsSlab(self.D, self.z0, self.z1, self.e0, self.e1)


def make_slabs(D: int, K: int, halo: int = HALO):
    """Even contiguous z-slabs (each >= 1 plane)."""
    if K < 1 or K > D:
        raise ValueError("need 1 <= K <= D slabs")
    out = []
    for r in range(K):
        z0, z1 = D * r // K, D * (r + 1) // K
        out.append(Slab(r, K, D, z0, z1, max(0, z0 - halo), min(D, z1 + halo)))
    return out


# ------------------------------------------------------------------------- transports
class LocalTransport:
    """K virtual ranks in one process (one device)."""

    def __init__(self, K: int):
        self.K = K
        self.held = list(range(K))

    def exchange(self, send_lo, send_hi):
        """send_lo[i]: rank's first owned plane -> rank-1; send_hi[i]: last plane -> rank+1.
        Returns (recv_below, recv_above) per held rank (None at the volume ends)."""
        K = self.K
        below = [send_hi[r - 1] if r > 0 else None for r in range(K)]
        above = [send_lo[r + 1] if r < K - 1 else None for r in range(K)]
        return below, above

    def allgather(self, xs):
        cat = torch.cat([x.reshape(-1) for x in xs])
        return [cat for _ in xs]

    def allgather_i64(self, vals):
        return [list(vals) for _ in vals]

    def any(self, flags):
        return bool(any(flags))

    def allreduce_min(self, xs):
        m = torch.stack(xs).amin(0)
        return [m for _ in xs]

    def allreduce_max(self, xs):
        m = torch.stack(xs).amax(0)
        return [m for _ in xs]


class DistTransport:
    """One rank per process over torch.distributed (NCCL on GPUs; gloo on CPU).  With gloo,
    device tensors are staged through host memory (a functional test of the multi-process
    path when several ranks share one GPU; NCCL refuses that)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.K = dist.get_world_size(group)
        self.held = [self.rank]
        self.host = dist.get_backend(group) == "gloo"

    def _out(self, t):
        return t.cpu() if (self.host and t is not None) else t

    def exchange(self, send_lo, send_hi):
        dist = self.dist
        r, K = self.rank, self.K
        lo, hi = self._out(send_lo[0]), self._out(send_hi[0])
        ref = lo if lo is not None else hi
        below = torch.empty_like(ref) if r > 0 else None
        above = torch.empty_like(ref) if r < K - 1 else None
        ops = []
        if r > 0:
            ops.append(dist.P2POp(dist.isend, lo, r - 1, self.group))
            ops.append(dist.P2POp(dist.irecv, below, r - 1, self.group))
        if r < K - 1:
            ops.append(dist.P2POp(dist.isend, hi, r + 1, self.group))
            ops.append(dist.P2POp(dist.irecv, above, r + 1, self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        dev = (send_lo[0] if send_lo[0] is not None else send_hi[0]).device
        if self.host:
            below = below.to(dev) if below is not None else None
            above = above.to(dev) if above is not None else None
        return [below], [above]

    def allgather(self, xs):
        x = xs[0].reshape(-1)
        if self.host:
            parts = [torch.empty_like(x, device="cpu") for _ in range(self.K)]
            self.dist.all_gather(parts, x.cpu(), group=self.group)
            return [torch.cat(parts).to(x.device)]
        out = torch.empty(self.K * x.numel(), dtype=x.dtype, device=x.device)
        self.dist.all_gather_into_tensor(out, x, group=self.group)
        return [out]

    def allgather_i64(self, vals):
        dev = "cuda" if torch.cuda.is_available() and self.dist.get_backend(self.group) == "nccl" else "cpu"
        t = torch.tensor([int(vals[0])], dtype=torch.int64, device=dev)
        out = torch.empty(self.K, dtype=torch.int64, device=dev)
        self.dist.all_gather_into_tensor(out, t, group=self.group)
        return [out.cpu().tolist()]

    def any(self, flags):
        dev = "cuda" if torch.cuda.is_available() and self.dist.get_backend(self.group) == "nccl" else "cpu"
        t = torch.tensor([1 if flags[0] else 0], dtype=torch.int32, device=dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return bool(t.item())

    def _allreduce(self, xs, op):
        if self.host and xs[0].is_cuda:
            h = xs[0].cpu()
            self.dist.all_reduce(h, op=op, group=self.group)
            xs[0].copy_(h)
        else:
            self.dist.all_reduce(xs[0], op=op, group=self.group)
        return xs

    def allreduce_min(self, xs):
        return self._allreduce(xs, self.dist.ReduceOp.MIN)

    def allreduce_max(self, xs):
        return self._allreduce(xs, self.dist.ReduceOp.MAX)


# ------------------------------------------------------------------------ watershed
def _dims(slab: Slab, n1: int, n2: int):
    return _b.WsDims(3, 0, slab.e1 - slab.e0, n1, n2)


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def halo_exchange(tr, ctxs, slabs, Ls, n1, n2):
    lib = _b.load()
    plane = n1 * n2
    send_lo = [Ls[i].view(-1)[s.zlo * plane:(s.zlo + 1) * plane].clone() if s.rank > 0 else None
               for i, s in enumerate(slabs)]
    send_hi = [Ls[i].view(-1)[(s.zhi - 1) * plane:s.zhi * plane].clone() if s.rank < s.K - 1 else None
               for i, s in enumerate(slabs)]
    below, above = tr.exchange(send_lo, send_hi)
    ch_lo, ch_hi = [], []
    for i, s in enumerate(slabs):
        for side, buf, out in ((0, below[i], ch_lo), (1, above[i], ch_hi)):
            if buf is None:
                out.append(0)
                continue
            c = ctypes.c_int32(0)
            _b.check(lib.ws_shard_halo(ctxs[i].handle, _b.ptr(Ls[i]), _dims(s, n1, n2), s.c(), side, _b.ptr(buf),
                                       ctypes.byref(c), _stream()))
            out.append(c.value)
    return ch_lo, ch_hi


def sharded_watershed(tr, ctxs, slabs, grads_ext, conn: int = 6, with_nreps: bool = False):
    """grads_ext[i]: u8 (e1-e0, n1, n2) of held slab i.  Returns (labels_own list, R, rounds
    [, owned representative counts])."""
    lib = _b.load()
    n1, n2 = grads_ext[0].shape[1], grads_ext[0].shape[2]
    plane = n1 * n2
    Ls = [torch.empty(g.shape, dtype=torch.int32, device=g.device) for g in grads_ext]
    pend = []
    for i, s in enumerate(slabs):
        p = ctypes.c_int32(0)
        _b.check(lib.ws_shard_plateau(ctxs[i].handle, _b.ptr(grads_ext[i]), _dims(s, n1, n2), conn, s.c(),
                                      _b.ptr(Ls[i]), 0, 0, 0, ctypes.byref(p), _stream()))
        pend.append(p.value)
    ch_lo, ch_hi = halo_exchange(tr, ctxs, slabs, Ls, n1, n2)
    rounds = 1
    while tr.any([pend[i] or ch_lo[i] or ch_hi[i] for i in range(len(slabs))]):
        for i, s in enumerate(slabs):
            p = ctypes.c_int32(0)
            _b.check(lib.ws_shard_plateau(ctxs[i].handle, _b.ptr(grads_ext[i]), _dims(s, n1, n2), conn, s.c(),
                                          _b.ptr(Ls[i]), 1, ch_lo[i], ch_hi[i], ctypes.byref(p), _stream()))
            pend[i] = p.value
        ch_lo, ch_hi = halo_exchange(tr, ctxs, slabs, Ls, n1, n2)
        rounds += 1
    tb = lib.ws_shard_table_bytes(_dims(slabs[0], n1, n2))
    Ps = [torch.empty_like(L) for L in Ls]
    tables = [torch.empty(tb, dtype=torch.uint8, device=L.device) for L in Ls]
    for i, s in enumerate(slabs):
        _b.check(lib.ws_shard_local(ctxs[i].handle, _b.ptr(grads_ext[i]), _b.ptr(Ls[i]), _dims(s, n1, n2), conn,
                                    s.c(), _b.ptr(Ps[i]), _b.ptr(tables[i]), _stream()))
    alltab = tr.allgather(tables)
    K = slabs[0].K
    full = make_slabs(slabs[0].D, K)
    z0s = (ctypes.c_int64 * K)(*[f.z0 for f in full])
    z1s = (ctypes.c_int64 * K)(*[f.z1 for f in full])
    labels, nreps = [], []
    for i, s in enumerate(slabs):
        ec = torch.empty(2 * plane, dtype=torch.int32, device=Ls[i].device)
        _b.check(lib.ws_shard_merge(ctxs[i].handle, _b.ptr(alltab[i]), K, z0s, z1s, _dims(s, n1, n2), s.c(),
                                    _b.ptr(Ls[i]), _b.ptr(ec), _stream()))
        out = torch.empty((s.z1 - s.z0, n1, n2), dtype=torch.int32, device=Ls[i].device)
        nr = ctypes.c_int64(0)
        _b.check(lib.ws_shard_relabel(ctxs[i].handle, _b.ptr(Ps[i]), _b.ptr(Ls[i]), _b.ptr(ec), _dims(s, n1, n2),
                                      s.c(), _b.ptr(out), ctypes.byref(nr), _stream()))
        labels.append(out)
        nreps.append(nr.value)
    R = sum(tr.allgather_i64([nreps[0]])[0]) if isinstance(tr, DistTransport) else sum(nreps)
    if with_nreps:
        return labels, R, rounds, nreps
    return labels, R, rounds


# ------------------------------------------------------------------------ waterfall
def sharded_waterfall(tr, ctxs, slabs, grads_ext, labels_own, nreps, NL: int, conn: int = 6):
    """Graph waterfall (C13) on z-slabs: dense ids by rank order, per-rank RAG (own planes + the
    cut above), per level all_reduce(MIN) of the per-component minima, replicated hook/flatten.
    Returns (levels_own list [NL, z1-z0, n1, n2], counts)."""
    lib = _b.load()
    K = slabs[0].K
    n1, n2 = grads_ext[0].shape[1], grads_ext[0].shape[2]
    plane = n1 * n2
    N = slabs[0].D * plane
    dev = grads_ext[0].device
    cnt_all = tr.allgather_i64([nreps[i] for i in range(len(slabs))])
    R = int(sum(cnt_all[0]))
    dense_of = [torch.empty((s.z1 - s.z0 + 1) * plane, dtype=torch.int32, device=dev) for s in slabs]  # window
    rep_of = [torch.full((R,), -1, dtype=torch.int32, device=dev) for _ in slabs]
    for i, s in enumerate(slabs):
        doff = int(sum(cnt_all[i][:s.rank]))
        c = ctypes.c_int64(0)
        _b.check(lib.ws_shard_wf_dense(ctxs[i].handle, _b.ptr(labels_own[i]), _dims(s, n1, n2), s.c(), doff,
                                       _b.ptr(dense_of[i]), _b.ptr(rep_of[i]), ctypes.byref(c), _stream()))
    rep_of = tr.allreduce_max(rep_of)
    bt = [torch.empty(4 * plane, dtype=torch.int32, device=dev) for _ in slabs]
    for i, s in enumerate(slabs):
        _b.check(lib.ws_shard_wf_btable(ctxs[i].handle, _b.ptr(labels_own[i]), _b.ptr(dense_of[i]), _dims(s, n1, n2),
                                        s.c(), _b.ptr(bt[i]), _stream()))
    allbt = tr.allgather(bt)
    for i, s in enumerate(slabs):
        _b.check(lib.ws_shard_wf_bfill(ctxs[i].handle, _b.ptr(allbt[i]), K, _dims(s, n1, n2), s.c(),
                                       _b.ptr(dense_of[i]), _stream()))
    # labels of the owned planes plus the first plane of the rank above (cut pairs)
    send_lo = [lo[0].contiguous() if s.rank > 0 else None for lo, s in zip(labels_own, slabs)]
    send_hi = [lo[-1].contiguous() if s.rank < K - 1 else None for lo, s in zip(labels_own, slabs)]
    below, above = tr.exchange(send_lo, send_hi)
    labels_ext = []
    for i, s in enumerate(slabs):
        le = torch.zeros((s.e1 - s.e0, n1, n2), dtype=torch.int32, device=dev)
        le[s.zlo:s.zhi] = labels_own[i]
        if above[i] is not None:
            le[s.zhi] = above[i].view(n1, n2)
        labels_ext.append(le)
    best = [torch.empty(R, dtype=torch.int64, device=dev) for _ in slabs]
    for i, s in enumerate(slabs):
        _b.check(lib.ws_shard_wf_begin(ctxs[i].handle, _b.ptr(labels_ext[i]), _b.ptr(grads_ext[i]), _dims(s, n1, n2),
                                       conn, s.c(), _b.ptr(dense_of[i]), R, NL, _b.ptr(best[i]), _stream()))
    best = tr.allreduce_min(best)
    counts = [R]
    more = 1 if (NL > 1 and R > 1) else 0
    cnt = R
    for k in range(1, NL):
        if more:
            # the exchanged minima shrink with the levels: only the current roots' (sorted)
            nxt = [torch.empty(max(cnt, 1), dtype=torch.int64, device=dev) for _ in slabs]
            for i, s in enumerate(slabs):
                c, m = ctypes.c_int64(0), ctypes.c_int32(0)
                _b.check(lib.ws_shard_wf_step(ctxs[i].handle, _b.ptr(best[i]), _b.ptr(nxt[i]), ctypes.byref(c),
                                              ctypes.byref(m), _stream()))
                cnt, more = c.value, m.value
            if more:
                best = tr.allreduce_min([x[:cnt].contiguous() for x in nxt])
        counts.append(cnt)
    levels = []
    for i, s in enumerate(slabs):
        out = torch.empty((NL, s.z1 - s.z0, n1, n2), dtype=torch.int32, device=dev)
        _b.check(lib.ws_shard_wf_end(ctxs[i].handle, _b.ptr(labels_own[i]), _b.ptr(dense_of[i]), _b.ptr(rep_of[i]),
                                     _dims(s, n1, n2), conn, s.c(), _b.ptr(out), _stream()))
        levels.append(out)
    return levels, counts


def sharded_segment(tr, ctxs, slabs, grads_ext, NL: int, conn: int = 6):
    """ws_watershed + ws_waterfall(NL) on z-slabs.  Returns (labels_own, levels_own, counts, R,
    plateau rounds)."""
    labels, R, rounds, nreps = sharded_watershed(tr, ctxs, slabs, grads_ext, conn, with_nreps=True)
    levels, counts = sharded_waterfall(tr, ctxs, slabs, grads_ext, labels, nreps, NL, conn)
    return labels, levels, counts, R, rounds


# ============================================================================ library path
# The sharded pipeline as ONE library call per rank (ws_segment_sharded / ws_watershed_sharded,
# include/ws.h): the control flow above runs inside libws_b200; Python only supplies the
# transport.  NcclLibTransport = the library's own NCCL communicator (production);
# TorchCallbacks / ThreadCallbacks = caller callbacks (multi-process on one GPU with gloo,
# K virtual ranks as threads in one process) for tests.

class _DevBuf:
    """A device pointer as a torch tensor (no copy) through __cuda_array_interface__."""

    def __init__(self, p, n, typestr):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": typestr, "data": (int(p), False),
                                         "version": 3, "strides": None, "stream": None}


_TYPESTR = {torch.uint8: "|u1", torch.int32: "<i4", torch.int64: "<i8"}


def _dev(p, n, dtype=torch.uint8):
    return torch.as_tensor(_DevBuf(p, n, _TYPESTR[dtype]), device="cuda")


def _torch_stream(ptr):
    """the library's stream argument (NULL = the legacy default stream) as a torch stream"""
    return torch.cuda.ExternalStream(ptr) if ptr else torch.cuda.default_stream()


class _CallbackTransport:
    """Wraps an object with exchange / allgather / allreduce methods on device tensors into a
    ws_transport (ctypes callbacks; exceptions become a non-zero status)."""

    def __init__(self, impl, rank: int, nranks: int):
        self.impl = impl

        def ex(user, slo, shi, rb, ra, nbytes, stream):
            try:
                self.impl.exchange(slo, shi, rb, ra, int(nbytes), stream)
                return 0
            except Exception as e:  # noqa: BLE001 - reported through the status
                self.error = e
                return -1

        def ag(user, send, recv, nbytes, stream):
            try:
                self.impl.allgather(send, recv, int(nbytes), stream)
                return 0
            except Exception as e:  # noqa: BLE001
                self.error = e
                return -1

        def ar(user, buf, count, dtype, op, stream):
            try:
                self.impl.allreduce(buf, int(count), int(dtype), int(op), stream)
                return 0
            except Exception as e:  # noqa: BLE001
                self.error = e
                return -1

        self._fns = (_b.EXCHANGE_FN(ex), _b.ALLGATHER_FN(ag), _b.ALLREDUCE_FN(ar))  # keep alive
        self.t = _b.WsTransport(None, int(rank), int(nranks), *self._fns)
        self.error = None

    def ptr(self):
        return ctypes.pointer(self.t)


class ThreadHub:
    """Shared state of K virtual ranks running as threads of one process (one device)."""

    def __init__(self, K: int):
        import threading
        self.K = K
        self.bar = threading.Barrier(K)
        self.slots = [None] * K


class ThreadCallbacks:
    """Collectives among the threads of a ThreadHub: device-to-device copies, ordered by
    synchronising each rank's stream around a barrier."""

    def __init__(self, hub: ThreadHub, rank: int):
        self.hub, self.rank = hub, rank

    def _sync(self, stream):
        _torch_stream(stream).synchronize()

    def exchange(self, slo, shi, rb, ra, n, stream):
        h, r = self.hub, self.rank
        self._sync(stream)
        h.slots[r] = (slo, shi)
        h.bar.wait()
        if rb:
            _dev(rb, n).copy_(_dev(h.slots[r - 1][1], n))
        if ra:
            _dev(ra, n).copy_(_dev(h.slots[r + 1][0], n))
        torch.cuda.synchronize()
        h.bar.wait()

    def allgather(self, send, recv, n, stream):
        h, r = self.hub, self.rank
        self._sync(stream)
        h.slots[r] = send
        h.bar.wait()
        out = _dev(recv, n * h.K)
        for q in range(h.K):
            out[q * n:(q + 1) * n].copy_(_dev(h.slots[q], n))
        torch.cuda.synchronize()
        h.bar.wait()

    def allreduce(self, buf, count, dtype, op, stream):
        h, r = self.hub, self.rank
        dt = torch.int64 if dtype == 1 else torch.int32
        self._sync(stream)
        h.slots[r] = buf
        h.bar.wait()
        parts = torch.stack([_dev(h.slots[q], count, dt) for q in range(h.K)])
        res = parts.amax(0) if op == 1 else parts.amin(0)
        torch.cuda.synchronize()
        h.bar.wait()  # every rank has read every buffer
        _dev(buf, count, dt).copy_(res)
        torch.cuda.synchronize()
        h.bar.wait()


class TorchCallbacks:
    """Collectives over torch.distributed (one rank per process).  gloo: device buffers are
    staged through host memory (several ranks may share one GPU); nccl: device buffers
    directly (on the library's stream)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.rank = dist.get_rank(group)
        self.K = dist.get_world_size(group)
        self.host = dist.get_backend(group) == "gloo"

    def _t(self, p, n, dtype=torch.uint8):
        t = _dev(p, n, dtype)
        return t.cpu() if self.host else t

    def exchange(self, slo, shi, rb, ra, n, stream):
        dist, r = self.dist, self.rank
        es = _torch_stream(stream)
        es.synchronize()
        with torch.cuda.stream(es):
            ops, outs = [], []
            if rb:
                b = self._t(rb, n)
                ops += [dist.P2POp(dist.isend, self._t(slo, n), r - 1, self.group),
                        dist.P2POp(dist.irecv, b, r - 1, self.group)]
                outs.append((rb, b))
            if ra:
                a = self._t(ra, n)
                ops += [dist.P2POp(dist.isend, self._t(shi, n), r + 1, self.group),
                        dist.P2POp(dist.irecv, a, r + 1, self.group)]
                outs.append((ra, a))
            if ops:
                for q in dist.batch_isend_irecv(ops):
                    q.wait()
            if self.host:
                for p, t in outs:
                    _dev(p, n).copy_(t)
        es.synchronize()

    def allgather(self, send, recv, n, stream):
        es = _torch_stream(stream)
        es.synchronize()
        with torch.cuda.stream(es):
            x = self._t(send, n)
            if self.host:
                parts = [torch.empty_like(x) for _ in range(self.K)]
                self.dist.all_gather(parts, x, group=self.group)
                _dev(recv, n * self.K).copy_(torch.cat(parts))
            else:
                self.dist.all_gather_into_tensor(_dev(recv, n * self.K), x, group=self.group)
        es.synchronize()

    def allreduce(self, buf, count, dtype, op, stream):
        dt = torch.int64 if dtype == 1 else torch.int32
        es = _torch_stream(stream)
        es.synchronize()
        with torch.cuda.stream(es):
            x = self._t(buf, count, dt)
            self.dist.all_reduce(x, op=self.dist.ReduceOp.MAX if op == 1 else self.dist.ReduceOp.MIN,
                                 group=self.group)
            if self.host:
                _dev(buf, count, dt).copy_(x)
        es.synchronize()


class NcclLibTransport:
    """The library's NCCL transport (ws_transport_nccl_create): rank 0 makes the unique id, it
    travels to the other ranks over torch.distributed (a CPU object broadcast)."""

    def __init__(self, device: int, group=None):
        import torch.distributed as dist
        lib = _b.load()
        self.rank, self.K = dist.get_rank(group), dist.get_world_size(group)
        uid = ctypes.create_string_buffer(128)
        if self.rank == 0:
            _b.check(lib.ws_nccl_unique_id(uid))
        obj = [bytes(uid.raw) if self.rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        uid = ctypes.create_string_buffer(obj[0], 128)
        self._p = ctypes.POINTER(_b.WsTransport)()
        _b.check(lib.ws_transport_nccl_create(uid, self.rank, self.K, int(device), ctypes.byref(self._p)))

    def ptr(self):
        return self._p

    def close(self):
        if getattr(self, "_p", None):
            _b.load().ws_transport_nccl_destroy(self._p)
            self._p = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def segment_sharded(transport, ctx, slab: Slab, grad_ext, NL: int, conn: int = 6, out=None):
    """ws_segment_sharded on this rank's extended slab grad_ext (u8 (e1-e0, n1, n2)).
    Returns (levels_own [NL, z1-z0, n1, n2], counts (global), step II rounds)."""
    lib = _b.load()
    n1, n2 = grad_ext.shape[1], grad_ext.shape[2]
    if out is None:
        out = torch.empty((NL, slab.z1 - slab.z0, n1, n2), dtype=torch.int32, device=grad_ext.device)
    counts = (ctypes.c_int64 * NL)()
    rounds = ctypes.c_int32(0)
    st = ctypes.c_void_p(torch.cuda.current_stream(grad_ext.device).cuda_stream)
    fn = lib.ws_segment_sharded_u16 if grad_ext.dtype == torch.uint16 else lib.ws_segment_sharded
    s = fn(ctx.handle, transport.ptr(), _b.ptr(grad_ext), _dims(slab, n1, n2), slab.c(), conn, NL,
                               _b.ptr(out), counts, ctypes.byref(rounds), st)
    if s != _b.WS_OK and getattr(transport, "error", None) is not None:
        raise RuntimeError("transport callback failed: %r" % (transport.error,))
    _b.check(s)
    return out, [int(c) for c in counts], rounds.value


def watershed_sharded(transport, ctx, slab: Slab, grad_ext, conn: int = 6, out=None):
    """ws_watershed_sharded: (labels_own [z1-z0, n1, n2], R (global), step II rounds)."""
    lib = _b.load()
    n1, n2 = grad_ext.shape[1], grad_ext.shape[2]
    if out is None:
        out = torch.empty((slab.z1 - slab.z0, n1, n2), dtype=torch.int32, device=grad_ext.device)
    R = ctypes.c_int64(0)
    rounds = ctypes.c_int32(0)
    st = ctypes.c_void_p(torch.cuda.current_stream(grad_ext.device).cuda_stream)
    fn = lib.ws_watershed_sharded_u16 if grad_ext.dtype == torch.uint16 else lib.ws_watershed_sharded
    _b.check(fn(ctx.handle, transport.ptr(), _b.ptr(grad_ext), _dims(slab, n1, n2), slab.c(),
                                      conn, _b.ptr(out), ctypes.byref(R), ctypes.byref(rounds), st))
    return out, R.value, rounds.value


def segment_threads(K: int, grad, NL: int, conn: int = 6):
    """K virtual ranks as threads of this process, each running ws_segment_sharded on its
    slab of the (D, n1, n2) volume grad with ThreadCallbacks.  Returns (levels [NL, D, n1, n2],
    counts, rounds)."""
    import threading
    D, n1, n2 = grad.shape
    slabs = make_slabs(D, K)
    hub = ThreadHub(K)
    res, errs = [None] * K, []
    dev = grad.device

    def run(r):
        try:
            torch.cuda.set_device(dev)
            st = torch.cuda.Stream(dev)
            with torch.cuda.stream(st):
                s = slabs[r]
                from . import _binding
                ctx = _binding.Context(dev.index)
                tr = _CallbackTransport(ThreadCallbacks(hub, r), r, K)
                ge = grad[s.e0:s.e1].contiguous()
                res[r] = segment_sharded(tr, ctx, s, ge, NL, conn)
                st.synchronize()
                ctx.close()
        except Exception as e:  # noqa: BLE001
            errs.append(e)
            hub.bar.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(K)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    levels = torch.cat([res[r][0] for r in range(K)], dim=1)
    return levels, res[0][1], res[0][2]
