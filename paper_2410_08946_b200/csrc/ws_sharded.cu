// ws_sharded.cu — the z-slab sharded hot path as ONE library call per rank (SURVEY §8(b) "the
// same calls then operate on the local slab", §8(e)): the whole distributed control flow —
// step II rounds with halo exchange until global convergence, boundary-table gather, the
// replicated cross-slab merge, rank-ordered dense ids, the per-level reduction of the
// per-component minima — runs here, on top of the ws_shard_* phase kernels (ws_shard.cu).
// Planes and tables move through a ws_transport (include/ws.h): the built-in NCCL transport
// (NCCL over NVLink / NVSwitch, the library owns the communicator; libnccl is resolved with
// dlopen, so the library has no link-time NCCL dependency), or caller callbacks (torch.
// distributed gloo for multi-process tests on one GPU, in-process threads for K virtual
// ranks).  Readings: DESIGN.md §9; correctness argument SURVEY A13.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "ws_internal.h"

using namespace ws;

// ------------------------------------------------------------------ NCCL by dlopen
namespace {
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi g_nccl;

template <class F>
bool sym(void* h, const char* name, F& f) {
  f = reinterpret_cast<F>(dlsym(h, name));
  return f != nullptr;
}

// the libnccl already loaded by the process (e.g. torch's) is reused: dlopen by soname
ws_status nccl_load() {
  if (g_nccl.h) return WS_OK;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    set_error(WS_ERR_NCCL, "libnccl.so.2 not found: %s", dlerror());
    return WS_ERR_NCCL;
  }
  NcclApi a;
  a.h = h;
  if (!(sym(h, "ncclGetUniqueId", a.GetUniqueId) && sym(h, "ncclCommInitRank", a.CommInitRank) &&
        sym(h, "ncclCommDestroy", a.CommDestroy) && sym(h, "ncclGroupStart", a.GroupStart) &&
        sym(h, "ncclGroupEnd", a.GroupEnd) && sym(h, "ncclSend", a.Send) && sym(h, "ncclRecv", a.Recv) &&
        sym(h, "ncclAllGather", a.AllGather) && sym(h, "ncclAllReduce", a.AllReduce) &&
        sym(h, "ncclGetErrorString", a.GetErrorString))) {
    set_error(WS_ERR_NCCL, "libnccl lacks a required symbol");
    return WS_ERR_NCCL;
  }
  g_nccl = a;
  return WS_OK;
}

struct NcclTransport {
  ws_transport t;  // first member: the public handle points here
  ncclComm_t comm = nullptr;
  int device = 0;
};

int nccl_exchange(void* user, const void* send_lo, const void* send_hi, void* recv_below, void* recv_above,
                  int64_t bytes, void* stream) {
  auto* T = static_cast<NcclTransport*>(user);
  const int r = T->t.rank;
  cudaStream_t st = (cudaStream_t)stream;
  ncclResult_t e = g_nccl.GroupStart();
  if (e == ncclSuccess && recv_below) e = g_nccl.Recv(recv_below, (size_t)bytes, ncclUint8, r - 1, T->comm, st);
  if (e == ncclSuccess && send_lo) e = g_nccl.Send(send_lo, (size_t)bytes, ncclUint8, r - 1, T->comm, st);
  if (e == ncclSuccess && send_hi) e = g_nccl.Send(send_hi, (size_t)bytes, ncclUint8, r + 1, T->comm, st);
  if (e == ncclSuccess && recv_above) e = g_nccl.Recv(recv_above, (size_t)bytes, ncclUint8, r + 1, T->comm, st);
  const ncclResult_t e2 = g_nccl.GroupEnd();
  return (int)(e != ncclSuccess ? e : e2);
}

int nccl_allgather(void* user, const void* send, void* recv, int64_t bytes, void* stream) {
  auto* T = static_cast<NcclTransport*>(user);
  return (int)g_nccl.AllGather(send, recv, (size_t)bytes, ncclUint8, T->comm, (cudaStream_t)stream);
}

int nccl_allreduce(void* user, void* buf, int64_t count, int32_t dtype, int32_t op, void* stream) {
  auto* T = static_cast<NcclTransport*>(user);
  return (int)g_nccl.AllReduce(buf, buf, (size_t)count, dtype == 1 ? ncclInt64 : ncclInt32, op == 1 ? ncclMax : ncclMin,
                               T->comm, (cudaStream_t)stream);
}

// ------------------------------------------------------------------ transport helpers
ws_status tr_fail(int code, const char* what) {
  if (g_nccl.h && g_nccl.GetErrorString && code > 0 && code < 16)
    set_error(WS_ERR_NCCL, "%s failed: %s (%d)", what, g_nccl.GetErrorString((ncclResult_t)code), code);
  else
    set_error(WS_ERR_NCCL, "%s failed (transport status %d)", what, code);
  return WS_ERR_NCCL;
}

#define TR_TRY(call, what)            \
  do {                                \
    const int _c = (call);            \
    if (_c != 0) return tr_fail(_c, what); \
  } while (0)

// the small device scratch of the collectives on host values (ctx->sh_small, pinned mirror)
struct Small {
  int64_t* d;   // device
  int64_t* h;   // pinned host
};

ws_status small_of(ws_ctx* ctx, int K, Small& s) {
  const size_t n = 2 * (size_t)K + 8;
  WS_TRY(ctx->sh_small.ensure(n * sizeof(int64_t), "sharded scratch"));
  if (!ctx->sh_small_h || ctx->sh_small_n < n) {
    if (ctx->sh_small_h) cudaFreeHost(ctx->sh_small_h);
    ctx->sh_small_h = nullptr;
    WS_CUDA(cudaMallocHost(&ctx->sh_small_h, n * sizeof(int64_t)));
    ctx->sh_small_n = n;
  }
  s.d = ctx->sh_small.as<int64_t>();
  s.h = ctx->sh_small_h;
  return WS_OK;
}

// every rank's value v -> out[0..K) (host)
ws_status allgather_i64(const ws_transport* tr, const Small& s, int64_t v, int64_t* out, cudaStream_t st) {
  const int K = tr->nranks;
  s.h[0] = v;
  WS_CUDA(cudaMemcpyAsync(s.d, s.h, sizeof(int64_t), cudaMemcpyHostToDevice, st));
  TR_TRY(tr->allgather(tr->user, s.d, s.d + 1, sizeof(int64_t), st), "allgather");
  WS_CUDA(cudaMemcpyAsync(s.h + 1, s.d + 1, K * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  WS_CUDA(cudaStreamSynchronize(st));
  std::memcpy(out, s.h + 1, K * sizeof(int64_t));
  return WS_OK;
}

// logical OR over the ranks
ws_status any_rank(const ws_transport* tr, const Small& s, bool v, bool* out, cudaStream_t st) {
  s.h[0] = v ? 1 : 0;
  WS_CUDA(cudaMemcpyAsync(s.d, s.h, sizeof(int64_t), cudaMemcpyHostToDevice, st));
  TR_TRY(tr->allreduce(tr->user, s.d, 1, 1, 1, st), "allreduce(max)");
  WS_CUDA(cudaMemcpyAsync(s.h, s.d, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  WS_CUDA(cudaStreamSynchronize(st));
  *out = s.h[0] != 0;
  return WS_OK;
}

ws_status check_transport(const ws_transport* tr, const ws_slab& sl) {
  if (!tr || !tr->exchange || !tr->allgather || !tr->allreduce || tr->nranks < 1 || tr->rank < 0 ||
      tr->rank >= tr->nranks) {
    set_error(WS_ERR_INVALID, "invalid ws_transport (callbacks, rank, nranks)");
    return WS_ERR_INVALID;
  }
  if ((tr->rank == 0) != (sl.z0 == 0) || (tr->rank == tr->nranks - 1) != (sl.z1 == sl.D)) {
    set_error(WS_ERR_INVALID, "slab [%lld, %lld) of D=%lld does not match rank %d of %d", (long long)sl.z0,
              (long long)sl.z1, (long long)sl.D, tr->rank, tr->nranks);
    return WS_ERR_INVALID;
  }
  return WS_OK;
}

// the phases of one pixel type (u8: ws_shard.cu; u16: ws_shard16.cu, NEXT f4)
template <class Px> struct ShardOps;
template <> struct ShardOps<uint8_t> {
  static ws_status first(ws_ctx* c, const uint8_t* I, const Geo& g, int conn, int32_t* L, int* p, cudaStream_t st) {
    return ws::plateau_first_shard(c, I, g, conn, L, p, st);
  }
  static ws_status round(ws_ctx* c, const uint8_t* I, const Geo& g, int conn, int32_t* L, int lo, int hi, int* p,
                         cudaStream_t st) {
    return ws::plateau_round_shard(c, I, g, conn, L, lo, hi, p, st);
  }
  static ws_status halo(ws_ctx* c, int32_t* L, const Geo& g, int side, const int32_t* in, int32_t* ch, cudaStream_t st) {
    return ws::shard_halo(c, L, g, side, in, ch, st);
  }
  static ws_status local(ws_ctx* c, const uint8_t* I, const Geo& g, int conn, int32_t* L, int32_t* P, void* t,
                         cudaStream_t st) {
    return ws::shard_local(c, I, g, conn, L, P, t, st);
  }
  static ws_status merge(ws_ctx* c, const void* t, const int64_t* z0, const int64_t* z1, int K, int r, const Geo& g,
                         int32_t* L, int32_t* ec, cudaStream_t st) {
    return ws::shard_merge(c, t, z0, z1, K, r, g, L, ec, st);
  }
  static ws_status relabel(ws_ctx* c, const int32_t* P, int32_t* L, const int32_t* ec, const Geo& g, int32_t* out,
                           int64_t* nreps, cudaStream_t st) {
    return ws::shard_relabel(c, P, L, ec, g, out, nreps, st);
  }
  static size_t table_bytes(size_t plane) { return ws::shard_table_bytes(plane); }
};
template <> struct ShardOps<uint16_t> {
  static ws_status first(ws_ctx* c, const uint16_t* I, const Geo& g, int conn, int32_t* L, int* p, cudaStream_t st) {
    return ws::px16::plateau_first_shard(c, I, g, conn, L, p, st);
  }
  static ws_status round(ws_ctx* c, const uint16_t* I, const Geo& g, int conn, int32_t* L, int lo, int hi, int* p,
                         cudaStream_t st) {
    return ws::px16::plateau_round_shard(c, I, g, conn, L, lo, hi, p, st);
  }
  static ws_status halo(ws_ctx* c, int32_t* L, const Geo& g, int side, const int32_t* in, int32_t* ch, cudaStream_t st) {
    return ws::px16::shard_halo(c, L, g, side, in, ch, st);
  }
  static ws_status local(ws_ctx* c, const uint16_t* I, const Geo& g, int conn, int32_t* L, int32_t* P, void* t,
                         cudaStream_t st) {
    return ws::px16::shard_local(c, I, g, conn, L, P, t, st);
  }
  static ws_status merge(ws_ctx* c, const void* t, const int64_t* z0, const int64_t* z1, int K, int r, const Geo& g,
                         int32_t* L, int32_t* ec, cudaStream_t st) {
    return ws::px16::shard_merge(c, t, z0, z1, K, r, g, L, ec, st);
  }
  static ws_status relabel(ws_ctx* c, const int32_t* P, int32_t* L, const int32_t* ec, const Geo& g, int32_t* out,
                           int64_t* nreps, cudaStream_t st) {
    return ws::px16::shard_relabel(c, P, L, ec, g, out, nreps, st);
  }
  static size_t table_bytes(size_t plane) { return ws::px16::shard_table_bytes(plane); }
};

// extended-slab geometry (owned planes [zlo, zhi), global offset) with the checks of ws_shard_*
ws_status slab_geo(const ws_dims& d, const ws_slab& sl, Geo* g) {
  const int64_t plane = d.n1 * d.n2;
  if (d.ndim != 3 || d.n0 < 1 || d.n1 < 1 || d.n2 < 1 || !(0 <= sl.e0 && sl.e0 <= sl.z0 && sl.z0 < sl.z1 &&
                                                            sl.z1 <= sl.e1 && sl.e1 <= sl.D) ||
      d.n0 != sl.e1 - sl.e0 || (double)sl.D * (double)plane >= 2147483648.0 || (sl.z0 > 0 && sl.e0 > sl.z0 - 1) ||
      (sl.z1 < sl.D && sl.e1 < sl.z1 + 1)) {
    set_error(WS_ERR_INVALID, "inconsistent slab (D=%lld z=[%lld,%lld) e=[%lld,%lld) n0=%lld)", (long long)sl.D,
              (long long)sl.z0, (long long)sl.z1, (long long)sl.e0, (long long)sl.e1, (long long)d.n0);
    return WS_ERR_INVALID;
  }
  g->n0 = (int)d.n0;
  g->n1 = (int)d.n1;
  g->n2 = (int)d.n2;
  g->plane = (int)plane;
  g->N = (int)(d.n0 * plane);
  g->zlo = (int)(sl.z0 - sl.e0);
  g->zhi = (int)(sl.z1 - sl.e0);
  g->gofs = (int)(sl.e0 * plane);
  return WS_OK;
}

// ------------------------------------------------------------------ the pipeline
// Watershed on the slab: labels_own (i32[(z1-z0) plane], global canonical labels), nreps
// (owned representatives), R (all ranks), rounds (step II rounds).
template <class Px>
ws_status sharded_watershed(ws_ctx* ctx, const ws_transport* tr, const Px* grad_ext, ws_dims d, ws_slab sl,
                            int conn, int32_t* labels_own, int64_t* nreps, int64_t* R, int32_t* rounds,
                            cudaStream_t st) {
  using O = ShardOps<Px>;
  Geo g;
  WS_TRY(slab_geo(d, sl, &g));
  const int K = tr->nranks, r = tr->rank;
  const int64_t plane = d.n1 * d.n2, next = d.n0 * plane;
  const int zlo = (int)(sl.z0 - sl.e0), zhi = (int)(sl.z1 - sl.e0);
  Small s;
  WS_TRY(small_of(ctx, K, s));
  WS_TRY(ctx->sh_L.ensure((size_t)next * 4, "sharded L"));
  WS_TRY(ctx->sh_P.ensure((size_t)next * 4, "sharded P"));
  WS_TRY(ctx->sh_planes.ensure((size_t)plane * 4 * 2, "halo planes"));
  int32_t* L = ctx->sh_L.as<int32_t>();
  int32_t* P = ctx->sh_P.as<int32_t>();
  int32_t* below = ctx->sh_planes.as<int32_t>();
  int32_t* above = below + plane;
  const bool has_lo = r > 0, has_hi = r < K - 1;
  auto halo = [&](int* ch_lo, int* ch_hi) -> ws_status {
    TR_TRY(tr->exchange(tr->user, has_lo ? L + (size_t)zlo * plane : nullptr,
                        has_hi ? L + (size_t)(zhi - 1) * plane : nullptr, has_lo ? below : nullptr,
                        has_hi ? above : nullptr, plane * 4, st),
           "halo exchange");
    *ch_lo = *ch_hi = 0;
    if (has_lo) WS_TRY(O::halo(ctx, L, g, 0, below, ch_lo, st));
    if (has_hi) WS_TRY(O::halo(ctx, L, g, 1, above, ch_hi, st));
    return WS_OK;
  };
  // steps I + II: relaxation rounds until no rank has pending work or a changed halo (the
  // halo planes start defined: the first exchange compares against them)
  if (has_lo) WS_CUDA(cudaMemsetAsync(L + (size_t)(zlo - 1) * plane, 0xFF, plane * 4, st));
  if (has_hi) WS_CUDA(cudaMemsetAsync(L + (size_t)zhi * plane, 0xFF, plane * 4, st));
  int pend = 0, ch_lo = 0, ch_hi = 0;
  WS_TRY(O::first(ctx, grad_ext, g, conn, L, &pend, st));
  WS_TRY(halo(&ch_lo, &ch_hi));
  int nround = 1;
  while (true) {
    bool more = false;
    WS_TRY(any_rank(tr, s, pend || ch_lo || ch_hi, &more, st));
    if (!more) break;
    WS_TRY(O::round(ctx, grad_ext, g, conn, L, ch_lo, ch_hi, &pend, st));
    WS_TRY(halo(&ch_lo, &ch_hi));
    ++nround;
  }
  // pointers, local steps III/IV, boundary tables; replicated merge over the gathered tables
  const int64_t tb = (int64_t)O::table_bytes((size_t)plane);
  WS_TRY(ctx->sh_tab.ensure((size_t)tb, "boundary table"));
  WS_TRY(ctx->sh_alltab.ensure((size_t)tb * K, "gathered boundary tables"));
  WS_TRY(O::local(ctx, grad_ext, g, conn, L, P, ctx->sh_tab.p, st));
  TR_TRY(tr->allgather(tr->user, ctx->sh_tab.p, ctx->sh_alltab.p, tb, st), "allgather(tables)");
  std::vector<int64_t> z0s(K), z1s(K);
  WS_TRY(allgather_i64(tr, s, sl.z0, z0s.data(), st));
  WS_TRY(allgather_i64(tr, s, sl.z1, z1s.data(), st));
  WS_TRY(ctx->sh_ec.ensure((size_t)plane * 2 * 4, "exit labels"));
  for (int q = 0; q < K; ++q)
    if ((q > 0 && z0s[q] != z1s[q - 1]) || z0s[0] != 0 || z1s[K - 1] != sl.D || (q == r && (z0s[q] != sl.z0 || z1s[q] != sl.z1))) {
      set_error(WS_ERR_INVALID, "the ranks' slabs must tile [0, D) in rank order");
      return WS_ERR_INVALID;
    }
  WS_TRY(O::merge(ctx, ctx->sh_alltab.p, z0s.data(), z1s.data(), K, r, g, L, ctx->sh_ec.as<int32_t>(), st));
  WS_TRY(O::relabel(ctx, P, L, ctx->sh_ec.as<int32_t>(), g, labels_own, nreps, st));
  std::vector<int64_t> cnt(K);
  WS_TRY(allgather_i64(tr, s, *nreps, cnt.data(), st));
  int64_t tot = 0;
  for (int64_t c : cnt) tot += c;
  *R = tot;
  *rounds = nround;
  return WS_OK;
}

// Graph waterfall (C13) on the slab: levels_own (i32[NL][(z1-z0) plane]), counts (host i64[NL])
template <class Px>
ws_status sharded_waterfall(ws_ctx* ctx, const ws_transport* tr, const Px* grad_ext, ws_dims d, ws_slab sl,
                            int conn, int NL, const int32_t* labels_own, int64_t nreps, int32_t* levels_own,
                            int64_t* counts, cudaStream_t st) {
  const int K = tr->nranks, r = tr->rank;
  const int64_t plane = d.n1 * d.n2, next = d.n0 * plane;
  const int zlo = (int)(sl.z0 - sl.e0), zhi = (int)(sl.z1 - sl.e0);
  Small s;
  WS_TRY(small_of(ctx, K, s));
  std::vector<int64_t> cnt(K);
  WS_TRY(allgather_i64(tr, s, nreps, cnt.data(), st));
  int64_t R = 0, doff = 0;
  for (int q = 0; q < K; ++q) {
    if (q < r) doff += cnt[q];
    R += cnt[q];
  }
  // dense ids in rank order; rep_of reduced (max) over the ranks (other entries -1)
  WS_TRY(ctx->sh_dense.ensure((size_t)(sl.z1 - sl.z0 + 1) * plane * 4, "dense-id window"));
  WS_TRY(ctx->sh_rep.ensure((size_t)std::max<int64_t>(R, 1) * 4, "rep_of"));
  int32_t* dense_of = ctx->sh_dense.as<int32_t>();
  int32_t* rep_of = ctx->sh_rep.as<int32_t>();
  WS_CUDA(cudaMemsetAsync(rep_of, 0xFF, (size_t)std::max<int64_t>(R, 1) * 4, st));
  int64_t c = 0;
  WS_TRY(ws_shard_wf_dense(ctx, labels_own, d, sl, doff, dense_of, rep_of, &c, st));
  TR_TRY(tr->allreduce(tr->user, rep_of, R, 0, 1, st), "allreduce(rep_of)");
  // dense ids of every label crossing a cut
  WS_TRY(ctx->sh_bt.ensure((size_t)plane * 4 * 4, "boundary dense table"));
  WS_TRY(ctx->sh_allbt.ensure((size_t)plane * 4 * 4 * K, "gathered boundary dense tables"));
  WS_TRY(ws_shard_wf_btable(ctx, labels_own, dense_of, d, sl, ctx->sh_bt.as<int32_t>(), st));
  TR_TRY(tr->allgather(tr->user, ctx->sh_bt.p, ctx->sh_allbt.p, plane * 4 * 4, st), "allgather(dense tables)");
  WS_TRY(ws_shard_wf_bfill(ctx, ctx->sh_allbt.as<int32_t>(), K, d, sl, dense_of, st));
  // labels of the owned planes + the first plane of the rank above (the cut pairs)
  WS_TRY(ctx->sh_lext.ensure((size_t)next * 4, "extended labels"));
  WS_TRY(ctx->sh_planes.ensure((size_t)plane * 4 * 2, "halo planes"));
  int32_t* lext = ctx->sh_lext.as<int32_t>();
  int32_t* below = ctx->sh_planes.as<int32_t>();
  int32_t* above = below + plane;
  const bool has_lo = r > 0, has_hi = r < K - 1;
  const int nown = zhi - zlo;
  TR_TRY(tr->exchange(tr->user, has_lo ? labels_own : nullptr,
                      has_hi ? labels_own + (size_t)(nown - 1) * plane : nullptr, has_lo ? below : nullptr,
                      has_hi ? above : nullptr, plane * 4, st),
         "label plane exchange");
  WS_CUDA(cudaMemsetAsync(lext, 0, (size_t)next * 4, st));
  WS_CUDA(cudaMemcpyAsync(lext + (size_t)zlo * plane, labels_own, (size_t)nown * plane * 4, cudaMemcpyDeviceToDevice,
                          st));
  if (has_hi)
    WS_CUDA(cudaMemcpyAsync(lext + (size_t)zhi * plane, above, (size_t)plane * 4, cudaMemcpyDeviceToDevice, st));
  // RAG + level-1 minima, reduced over the ranks; then the levels
  WS_TRY(ctx->sh_best.ensure((size_t)std::max<int64_t>(R, 1) * 8, "per-component minima"));
  WS_TRY(ctx->sh_nxt.ensure((size_t)std::max<int64_t>(R, 1) * 8, "next minima"));
  int64_t* best = ctx->sh_best.as<int64_t>();
  int64_t* nxt = ctx->sh_nxt.as<int64_t>();
  if constexpr (sizeof(Px) == 1) {
    WS_TRY(ws_shard_wf_begin(ctx, lext, grad_ext, d, conn, sl, dense_of, R, NL, best, st));
    TR_TRY(tr->allreduce(tr->user, best, R, 1, 0, st), "allreduce(min) level 1");
    if (counts) counts[0] = R;
    int more = (NL > 1 && R > 1) ? 1 : 0;
    int64_t cur = R;
    for (int k = 1; k < NL; ++k) {
      if (more) {
        int64_t cc = 0;
        int32_t m = 0;
        WS_TRY(ws_shard_wf_step(ctx, best, nxt, &cc, &m, st));
        cur = cc;
        more = m;
        if (more) {
          TR_TRY(tr->allreduce(tr->user, nxt, cur, 1, 0, st), "allreduce(min) level");
          std::swap(best, nxt);
        }
      }
      if (counts) counts[k] = cur;
    }
  } else {
    // 16-bit: K = (hi, lo) reduced in two steps per level (ws_waterfall.cu shard_wf16_level)
    Geo g;
    WS_TRY(slab_geo(d, sl, &g));
    WS_TRY(shard_wf16_begin(ctx, lext, grad_ext, g, conn, dense_of, R, NL, st));
    if (counts) counts[0] = R;
    int64_t cur = R;
    for (int k = 1; k < NL; ++k) {
      if (cur > 1) {
        WS_TRY(shard_wf16_level(ctx, 0, &cur, st));
        TR_TRY(tr->allreduce(tr->user, ctx->best.p, R, 1, 0, st), "allreduce(min) hi");
        WS_TRY(shard_wf16_level(ctx, 1, &cur, st));
        TR_TRY(tr->allreduce(tr->user, ctx->best_lo.p, R, 0, 0, st), "allreduce(min) lo");
        WS_TRY(shard_wf16_level(ctx, 2, &cur, st));
      }
      if (counts) counts[k] = cur;
    }
  }
  WS_TRY(ws_shard_wf_end(ctx, labels_own, dense_of, rep_of, d, conn, sl, levels_own, st));
  return WS_OK;
}

// owned representatives: labels_own[i] == pofs + i (a region's smallest voxel lies here)
__global__ void k_count_reps(const int32_t* __restrict__ lab, long long n, long long pofs,
                             unsigned long long* __restrict__ cnt) {
  unsigned long long c = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    c += lab[i] == (int32_t)(pofs + i);
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(cnt, c);
}

ws_status check_sharded_args(ws_ctx* ctx, const ws_transport* tr, const void* grad_ext, const ws_dims& d,
                             const ws_slab& sl, int conn, const void* out) {
  if (!ctx) {
    set_error(WS_ERR_INVALID, "ctx is NULL");
    return WS_ERR_INVALID;
  }
  if (!grad_ext || !out) {
    set_error(WS_ERR_INVALID, "NULL argument (grad_ext / output)");
    return WS_ERR_INVALID;
  }
  WS_TRY(check_transport(tr, sl));
  if (d.ndim != 3 || (conn != 6 && conn != 26) || d.n0 != sl.e1 - sl.e0) {
    set_error(WS_ERR_INVALID, "the sharded path takes the extended slab of a 3-D volume, 6- or 26-connectivity");
    return WS_ERR_INVALID;
  }
  return WS_OK;
}
}  // namespace

extern "C" {

ws_status ws_nccl_unique_id(void* out) {
  if (!out) {
    set_error(WS_ERR_INVALID, "out is NULL");
    return WS_ERR_INVALID;
  }
  WS_TRY(nccl_load());
  ncclUniqueId id;
  const ncclResult_t e = g_nccl.GetUniqueId(&id);
  if (e != ncclSuccess) return tr_fail((int)e, "ncclGetUniqueId");
  static_assert(sizeof(ncclUniqueId) == WS_NCCL_ID_BYTES, "ncclUniqueId size");
  std::memcpy(out, &id, sizeof(id));
  return WS_OK;
}

ws_status ws_transport_nccl_create(const void* unique_id, int32_t rank, int32_t nranks, int32_t device,
                                   ws_transport** out) {
  if (!unique_id || !out || nranks < 1 || rank < 0 || rank >= nranks) {
    set_error(WS_ERR_INVALID, "bad arguments (unique_id, rank %d, nranks %d)", rank, nranks);
    return WS_ERR_INVALID;
  }
  WS_TRY(nccl_load());
  WS_CUDA(cudaSetDevice(device));
  auto* T = new (std::nothrow) NcclTransport();
  if (!T) {
    set_error(WS_ERR_OOM, "host allocation failed");
    return WS_ERR_OOM;
  }
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof(id));
  const ncclResult_t e = g_nccl.CommInitRank(&T->comm, nranks, id, rank);
  if (e != ncclSuccess) {
    delete T;
    return tr_fail((int)e, "ncclCommInitRank");
  }
  T->device = device;
  T->t.user = T;
  T->t.rank = rank;
  T->t.nranks = nranks;
  T->t.exchange = nccl_exchange;
  T->t.allgather = nccl_allgather;
  T->t.allreduce = nccl_allreduce;
  *out = &T->t;
  return WS_OK;
}

ws_status ws_transport_nccl_destroy(ws_transport* tr) {
  if (!tr) return WS_OK;
  auto* T = reinterpret_cast<NcclTransport*>(tr);
  if (T->comm && g_nccl.CommDestroy) g_nccl.CommDestroy(T->comm);
  delete T;
  return WS_OK;
}

ws_status ws_ctx_create_sharded(int32_t device, const ws_transport* tr, ws_slab slab, ws_ctx** out) {
  WS_TRY(check_transport(tr, slab));
  WS_TRY(ws_ctx_create(device, out));
  (*out)->sh_tr = *tr;
  (*out)->sh_slab = slab;
  (*out)->sharded = 1;
  return WS_OK;
}

}  // extern "C"

namespace {
template <class Px>
ws_status watershed_sharded_t(ws_ctx* ctx, const ws_transport* tr, const Px* grad_ext, ws_dims dims_ext, ws_slab slab,
                              int32_t connectivity, int32_t* labels_own, int64_t* num_regions, int32_t* rounds,
                              void* stream) {
  WS_TRY(check_sharded_args(ctx, tr, grad_ext, dims_ext, slab, connectivity, labels_own));
  std::memset(&ctx->stats, 0, sizeof(ctx->stats));
  cudaStream_t st = (cudaStream_t)stream;
  int64_t nreps = 0, R = 0;
  int32_t nr = 0;
  WS_TRY(sharded_watershed(ctx, tr, grad_ext, dims_ext, slab, connectivity, labels_own, &nreps, &R, &nr, st));
  if (num_regions) *num_regions = R;
  if (rounds) *rounds = nr;
  ctx->stats.n_regions = R;
  ctx->stats.plateau_rounds = nr;
  return WS_OK;
}

template <class Px>
ws_status segment_sharded_t(ws_ctx* ctx, const ws_transport* tr, const Px* grad_ext, ws_dims dims_ext, ws_slab slab,
                            int32_t connectivity, int32_t NL, int32_t* levels_own, int64_t* counts, int32_t* rounds,
                            void* stream) {
  WS_TRY(check_sharded_args(ctx, tr, grad_ext, dims_ext, slab, connectivity, levels_own));
  if (NL < 1 || NL > 16) {
    set_error(WS_ERR_INVALID, "NL must be in [1, 16] (got %d)", NL);
    return WS_ERR_INVALID;
  }
  std::memset(&ctx->stats, 0, sizeof(ctx->stats));
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t nown = (slab.z1 - slab.z0) * dims_ext.n1 * dims_ext.n2;
  WS_TRY(ctx->sh_lab.ensure((size_t)nown * 4, "slab labels"));
  int64_t nreps = 0, R = 0;
  int32_t nr = 0;
  WS_TRY(sharded_watershed(ctx, tr, grad_ext, dims_ext, slab, connectivity, ctx->sh_lab.as<int32_t>(), &nreps, &R,
                           &nr, st));
  int64_t cts[16] = {};
  WS_TRY(sharded_waterfall(ctx, tr, grad_ext, dims_ext, slab, connectivity, NL, ctx->sh_lab.as<int32_t>(), nreps,
                           levels_own, cts, st));
  WS_CUDA(cudaStreamSynchronize(st));
  if (counts) std::memcpy(counts, cts, (size_t)NL * sizeof(int64_t));
  if (rounds) *rounds = nr;
  ctx->stats.n_regions = R;
  ctx->stats.plateau_rounds = nr;
  for (int k = 0; k < NL; ++k) ctx->stats.level_counts[k] = cts[k];
  return WS_OK;
}

template <class Px>
ws_status waterfall_sharded_t(ws_ctx* ctx, const ws_transport* tr, const int32_t* labels_own, const Px* grad_ext,
                              ws_dims dims_ext, ws_slab slab, int32_t connectivity, int32_t NL, int32_t* levels_own,
                              int64_t* counts, void* stream) {
  WS_TRY(check_sharded_args(ctx, tr, grad_ext, dims_ext, slab, connectivity, levels_own));
  if (!labels_own) {
    set_error(WS_ERR_INVALID, "labels_own is NULL");
    return WS_ERR_INVALID;
  }
  if (NL < 1 || NL > 16) {
    set_error(WS_ERR_INVALID, "NL must be in [1, 16] (got %d)", NL);
    return WS_ERR_INVALID;
  }
  std::memset(&ctx->stats, 0, sizeof(ctx->stats));
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t plane = dims_ext.n1 * dims_ext.n2, nown = (slab.z1 - slab.z0) * plane;
  Small s;
  WS_TRY(small_of(ctx, tr->nranks, s));
  WS_CUDA(cudaMemsetAsync(s.d, 0, sizeof(int64_t), st));
  k_count_reps<<<std::max<long long>(1, std::min<long long>((nown + 255) / 256, ctx->num_sms * 8LL)), 256, 0, st>>>(
      labels_own, nown, slab.z0 * plane, reinterpret_cast<unsigned long long*>(s.d));
  WS_CUDA(cudaMemcpyAsync(s.h, s.d, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  WS_CUDA(cudaStreamSynchronize(st));
  const int64_t nreps = s.h[0];
  int64_t cts[16] = {};
  WS_TRY(sharded_waterfall(ctx, tr, grad_ext, dims_ext, slab, connectivity, NL, labels_own, nreps, levels_own, cts,
                           st));
  WS_CUDA(cudaStreamSynchronize(st));
  if (counts) std::memcpy(counts, cts, (size_t)NL * sizeof(int64_t));
  for (int k = 0; k < NL; ++k) ctx->stats.level_counts[k] = cts[k];
  return WS_OK;
}
}  // namespace

extern "C" {

ws_status ws_watershed_sharded(ws_ctx* ctx, const ws_transport* tr, const uint8_t* grad_ext, ws_dims dims_ext,
                               ws_slab slab, int32_t connectivity, int32_t* labels_own, int64_t* num_regions,
                               int32_t* rounds, void* stream) {
  return watershed_sharded_t(ctx, tr, grad_ext, dims_ext, slab, connectivity, labels_own, num_regions, rounds, stream);
}
ws_status ws_watershed_sharded_u16(ws_ctx* ctx, const ws_transport* tr, const uint16_t* grad_ext, ws_dims dims_ext,
                                   ws_slab slab, int32_t connectivity, int32_t* labels_own, int64_t* num_regions,
                                   int32_t* rounds, void* stream) {
  return watershed_sharded_t(ctx, tr, grad_ext, dims_ext, slab, connectivity, labels_own, num_regions, rounds, stream);
}
ws_status ws_segment_sharded(ws_ctx* ctx, const ws_transport* tr, const uint8_t* grad_ext, ws_dims dims_ext,
                             ws_slab slab, int32_t connectivity, int32_t NL, int32_t* levels_own, int64_t* counts,
                             int32_t* rounds, void* stream) {
  return segment_sharded_t(ctx, tr, grad_ext, dims_ext, slab, connectivity, NL, levels_own, counts, rounds, stream);
}
ws_status ws_segment_sharded_u16(ws_ctx* ctx, const ws_transport* tr, const uint16_t* grad_ext, ws_dims dims_ext,
                                 ws_slab slab, int32_t connectivity, int32_t NL, int32_t* levels_own, int64_t* counts,
                                 int32_t* rounds, void* stream) {
  return segment_sharded_t(ctx, tr, grad_ext, dims_ext, slab, connectivity, NL, levels_own, counts, rounds, stream);
}
ws_status ws_waterfall_sharded(ws_ctx* ctx, const ws_transport* tr, const int32_t* labels_own, const uint8_t* grad_ext,
                               ws_dims dims_ext, ws_slab slab, int32_t connectivity, int32_t NL, int32_t* levels_own,
                               int64_t* counts, void* stream) {
  return waterfall_sharded_t(ctx, tr, labels_own, grad_ext, dims_ext, slab, connectivity, NL, levels_own, counts,
                             stream);
}
ws_status ws_waterfall_sharded_u16(ws_ctx* ctx, const ws_transport* tr, const int32_t* labels_own,
                                   const uint16_t* grad_ext, ws_dims dims_ext, ws_slab slab, int32_t connectivity,
                                   int32_t NL, int32_t* levels_own, int64_t* counts, void* stream) {
  return waterfall_sharded_t(ctx, tr, labels_own, grad_ext, dims_ext, slab, connectivity, NL, levels_own, counts,
                             stream);
}

}  // extern "C"

// ws_watershed / ws_segment / ws_waterfall on a context made by ws_ctx_create_sharded
namespace ws {
ws_status sharded_dispatch_watershed(ws_ctx* ctx, const uint8_t* grad_ext, const ws_dims& d, int conn, int32_t* labels,
                                     int64_t* num_regions, cudaStream_t st) {
  return ws_watershed_sharded(ctx, &ctx->sh_tr, grad_ext, d, ctx->sh_slab, conn, labels, num_regions, nullptr, st);
}
ws_status sharded_dispatch_segment(ws_ctx* ctx, const uint8_t* grad_ext, const ws_dims& d, int conn, int NL,
                                   int32_t* levels, int64_t* counts, cudaStream_t st) {
  return ws_segment_sharded(ctx, &ctx->sh_tr, grad_ext, d, ctx->sh_slab, conn, NL, levels, counts, nullptr, st);
}
ws_status sharded_dispatch_waterfall(ws_ctx* ctx, const int32_t* labels_own, const uint8_t* grad_ext, const ws_dims& d,
                                     int conn, int NL, int32_t* levels, int64_t* counts, cudaStream_t st) {
  return ws_waterfall_sharded(ctx, &ctx->sh_tr, labels_own, grad_ext, d, ctx->sh_slab, conn, NL, levels, counts, st);
}
ws_status sharded_dispatch_watershed_u16(ws_ctx* ctx, const uint16_t* grad_ext, const ws_dims& d, int conn,
                                         int32_t* labels, int64_t* num_regions, cudaStream_t st) {
  return ws_watershed_sharded_u16(ctx, &ctx->sh_tr, grad_ext, d, ctx->sh_slab, conn, labels, num_regions, nullptr, st);
}
ws_status sharded_dispatch_waterfall_u16(ws_ctx* ctx, const int32_t* labels_own, const uint16_t* grad_ext,
                                         const ws_dims& d, int conn, int NL, int32_t* levels, int64_t* counts,
                                         cudaStream_t st) {
  return ws_waterfall_sharded_u16(ctx, &ctx->sh_tr, labels_own, grad_ext, d, ctx->sh_slab, conn, NL, levels, counts,
                                  st);
}
}  // namespace ws
