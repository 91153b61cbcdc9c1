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
    dense_of = [torch.empty(N, dtype=torch.int32, device=dev) for _ in slabs]
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
        _b.check(lib.ws_shard_wf_bfill(ctxs[i].handle, _b.ptr(allbt[i]), K, _dims(s, n1, n2), _b.ptr(dense_of[i]),
                                       _stream()))
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
