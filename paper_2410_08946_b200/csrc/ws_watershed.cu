// ws_watershed.cu — steps I-IV of PRUF (Alg. 1) + canonical relabel, sm_100a.
//
// Working array: L (= the caller's `labels` output, i32[N]) in the step II encoding of
// ws_common.cuh; aux (i32[N], context scratch) holds per-root canonical minima.
//
//   k_init      step I  (Alg. 1 l.1-10, Eq. 1)               1 pass
//   k_relax     step II distances (Alg. 3 relaxation)         repeated until no change
//   k_select    step II pointer selection (C6)                1 pass
//   k_jump      step III pointer jumping to roots (l.19-23)   1 pass (per-thread chase)
//   k_union     step IV Union over q > p (l.24-27)            1 pass, lock-free CAS
//   k_find      step IV Find (l.28-29) + canonical atomicMin  1 pass
//   k_relabel   labels = canonical minimum of the root        1 pass
#include "ws_internal.h"

namespace ws {

#define ZLOOP_BEGIN                                                         \
  const int x = blockIdx.x * blockDim.x + threadIdx.x;                      \
  const int y = blockIdx.y * blockDim.y + threadIdx.y;                      \
  if (x >= g.n2 || y >= g.n1) return;                                       \
  for (int z = blockIdx.z; z < g.n0; z += gridDim.z) {                      \
    const int p = z * g.plane + y * g.n2 + x;
#define ZLOOP_END }

// ---------------------------------------------------------------- step I (Alg. 1 l.1-10)
template <int CONN>
__global__ void k_init(const uint8_t* __restrict__ I, int* __restrict__ L, Geo g) {
  ZLOOP_BEGIN
  const int v = I[p];
  int m = 256, q = -1;
#pragma unroll
  for (int i = 0; i < CONN; ++i) {
    if (!nb_in<CONN>(g, z, y, x, i)) continue;
    const int r = p + nb_off<CONN>(g, i);
    const int nv = I[r];
    if (nv <= m) { m = nv; q = r; }  // increasing index order: '<=' keeps the max index (Eq. 1)
  }
  int out;
  if (q < 0 || m > v) out = p;            // S = 1: strict minimum (or a 1-voxel image, C4)
  else if (m < v) out = q;                // S = 0: steepest descent
  else out = enc(DUNREACHED, DIR_NONE);   // S = 2/3: plateau voxel, distance unknown
  L[p] = out;
  ZLOOP_END
}

// --------------------------------------------- step II relaxation (Alg. 3 l.7-8, in place)
// d(p) <- min(d(p), 1 + min_{q in N(p), I(q) = I(p)} d(q)) ; voxels with L >= 0 have d = 0.
// Chaotic in-place relaxation from above converges to the unique BFS fixpoint.
template <int CONN>
__global__ void k_relax(const uint8_t* __restrict__ I, int* L, Geo g, int* changed) {
  ZLOOP_BEGIN
  const int Lp = L[p];
  if (Lp >= 0) continue;
  const int d = dec_d(Lp);
  const int v = I[p];
  int best = d;
#pragma unroll
  for (int i = 0; i < CONN; ++i) {
    if (!nb_in<CONN>(g, z, y, x, i)) continue;
    const int r = p + nb_off<CONN>(g, i);
    if (I[r] != v) continue;
    const int dq = dec_d(L[r]) + 1;
    best = dq < best ? dq : best;
  }
  if (best < d) {
    L[p] = enc(best, DIR_NONE);
    if (best >= DUNREACHED - 1) changed[1] = 1;  // depth limit (WS_ERR_LIMIT)
    changed[0] = 1;
  }
  ZLOOP_END
}

// --------------------------------------------------- step II pointer selection (C5, C6)
// d finite: dir = max-index equal neighbour with d(q) = d - 1.  d unreached (minimal
// plateau): Eq. 1 among equal neighbours; state 2 (q > p) keeps dir, state 3 is a root.
// Only the low 5 bits of L change, so concurrent readers still decode every d.
template <int CONN>
__global__ void k_select(const uint8_t* __restrict__ I, int* L, Geo g) {
  ZLOOP_BEGIN
  const int Lp = L[p];
  if (Lp >= 0) continue;
  const int d = dec_d(Lp);
  const int v = I[p];
  int dir = DIR_NONE;
  if (d != DUNREACHED) {
#pragma unroll
    for (int i = 0; i < CONN; ++i) {
      if (!nb_in<CONN>(g, z, y, x, i)) continue;
      const int r = p + nb_off<CONN>(g, i);
      if (I[r] == v && dec_d(L[r]) == d - 1) dir = i;
    }
  } else {
    int last = -1;
#pragma unroll
    for (int i = 0; i < CONN; ++i) {
      if (!nb_in<CONN>(g, z, y, x, i)) continue;
      if (I[p + nb_off<CONN>(g, i)] == v) last = i;
    }
    dir = (last >= Conn<CONN>::nfwd) ? last : DIR_NONE;  // q > p  <=>  forward half
  }
  L[p] = enc(d, dir);
  ZLOOP_END
}

// -------------------------------------------- step III: follow pointers to the self-loop
// Each thread chases its own path (Alg. 1 l.28-29, APRUF) and writes the root; concurrent
// writes only shortcut paths toward the same root.  Roots also seed aux[root] = root.
template <int CONN>
__global__ void k_jump(int* L, int* __restrict__ aux, Geo g) {
  ZLOOP_BEGIN
  int t = ptr_of<CONN>(g, p, L[p]);
  if (t != p) {
    while (true) {
      const int nt = ptr_of<CONN>(g, t, L[t]);
      if (nt == t) break;
      t = nt;
    }
  } else {
    aux[p] = p;
  }
  L[p] = t;
  ZLOOP_END
}

__device__ __forceinline__ int uf_find(int* L, int x) {
  while (true) {
    const int y = ld_cg(L + x);
    if (y == x) return x;
    x = y;
  }
}

// min-root lock-free union ("setting the smaller label as the parent")
__device__ __forceinline__ void uf_unite(int* L, int a, int b) {
  while (true) {
    a = uf_find(L, a);
    b = uf_find(L, b);
    if (a == b) return;
    if (a > b) { const int t = a; a = b; b = t; }
    const int old = atomicCAS(L + b, b, a);
    if (old == b) return;
  }
}

// ------------------------------------------------ step IV Union (Alg. 1 l.24-27, q > p)
// p is on a minimal plateau  <=>  I(root(p)) == I(p) (the descent path into a regional
// minimum keeps the intensity only inside that minimum's plateau).
template <int CONN>
__global__ void k_union(const uint8_t* __restrict__ I, int* L, Geo g) {
  ZLOOP_BEGIN
  const int v = I[p];
  const int r = ld_cg(L + p);
  if (I[r] != v) continue;
#pragma unroll
  for (int i = Conn<CONN>::nfwd; i < CONN; ++i) {
    if (!nb_in<CONN>(g, z, y, x, i)) continue;
    const int q = p + nb_off<CONN>(g, i);
    if (I[q] != v) continue;
    if (ld_cg(L + q) == ld_cg(L + p)) continue;  // already in the same set
    uf_unite(L, p, q);
  }
  ZLOOP_END
}

// ------------------------------- step IV Find (l.28-29) + canonical minimum per root (C7)
__global__ void k_find(int* L, int* __restrict__ aux, Geo g) {
  ZLOOP_BEGIN
  const int r = uf_find(L, ld_cg(L + p));
  L[p] = r;
  // warp-aggregated atomicMin: lanes sharing a root elect one leader
  const unsigned act = __activemask();
  const unsigned grp = __match_any_sync(act, r);
  const int mn = (int)__reduce_min_sync(grp, (unsigned)p);
  if (mn < r && (__ffs(grp) - 1) == (int)(threadIdx.x + threadIdx.y * blockDim.x) % 32)
    atomicMin(aux + r, mn);
  ZLOOP_END
}

__global__ void k_relabel(int* L, const int* __restrict__ aux, Geo g, unsigned long long* nroots) {
  ZLOOP_BEGIN
  const int c = aux[L[p]];
  L[p] = c;
  const unsigned act = __activemask();
  const unsigned b = __ballot_sync(act, c == p);
  if (nroots && b && (__ffs(act) - 1) == (int)(threadIdx.x + threadIdx.y * blockDim.x) % 32)
    atomicAdd(nroots, (unsigned long long)__popc(b));
  ZLOOP_END
}

// ------------------------------------------------------- debug dump of step I+II (T2)
template <int CONN>
__global__ void k_plateau_dump(const int* __restrict__ L, Geo g, int* dist, int* parent) {
  ZLOOP_BEGIN
  const int Lp = L[p];
  int d, par;
  if (Lp >= 0) {
    d = (Lp == p) ? -1 : 0;
    par = Lp;
  } else {
    const int dd = dec_d(Lp);
    d = dd == DUNREACHED ? -1 : dd;
    par = dd == DUNREACHED ? p : ptr_of<CONN>(g, p, Lp);
  }
  dist[p] = d;
  parent[p] = par;
  ZLOOP_END
}

// --------------------------------------------------------------------------- drivers
template <int CONN>
static ws_status plateau_phase(ws_ctx* ctx, const uint8_t* grad, const Geo& g, int32_t* L, cudaStream_t st) {
  const L3 l = launch3(g);
  WS_TRY(ctx->flags.ensure(256, "flags"));
  int* flag = ctx->flags.as<int>();
  k_init<CONN><<<l.grid, l.block, 0, st>>>(grad, L, g);
  launched(ctx, PH_WS_INIT);
  tmark(ctx, st, PH_WS_INIT);
  int rounds = 0;
  WS_CUDA(cudaMemsetAsync(flag, 0, 2 * sizeof(int), st));
  while (true) {
    WS_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), st));
    k_relax<CONN><<<l.grid, l.block, 0, st>>>(grad, L, g, flag);
    launched(ctx, PH_WS_RELAX);
    ++rounds;
    WS_CUDA(cudaMemcpyAsync(ctx->pinned, flag, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
    WS_CUDA(cudaStreamSynchronize(st));
    const int* h = reinterpret_cast<const int*>(ctx->pinned);
    if (h[1]) {
      set_error(WS_ERR_LIMIT, "a non-minimal plateau is deeper than 2^26-2 voxels");
      return WS_ERR_LIMIT;
    }
    if (!h[0]) break;
  }
  ctx->stats.plateau_rounds = rounds;
  tmark(ctx, st, PH_WS_RELAX);
  k_select<CONN><<<l.grid, l.block, 0, st>>>(grad, L, g);
  launched(ctx, PH_WS_SELECT);
  tmark(ctx, st, PH_WS_SELECT);
  WS_CUDA(cudaGetLastError());
  return WS_OK;
}

template <int CONN>
static ws_status watershed_t(ws_ctx* ctx, const uint8_t* grad, const Geo& g, int32_t* L,
                             int64_t* num_regions, cudaStream_t st) {
  WS_TRY(plateau_phase<CONN>(ctx, grad, g, L, st));
  WS_TRY(ctx->aux.ensure((size_t)g.N * sizeof(int), "aux"));
  int* aux = ctx->aux.as<int>();
  const L3 l = launch3(g);
  k_jump<CONN><<<l.grid, l.block, 0, st>>>(L, aux, g);
  launched(ctx, PH_WS_JUMP);
  tmark(ctx, st, PH_WS_JUMP);
  k_union<CONN><<<l.grid, l.block, 0, st>>>(grad, L, g);
  launched(ctx, PH_WS_UNION);
  tmark(ctx, st, PH_WS_UNION);
  k_find<<<l.grid, l.block, 0, st>>>(L, aux, g);
  launched(ctx, PH_WS_FIND);
  tmark(ctx, st, PH_WS_FIND);
  unsigned long long* nroots = reinterpret_cast<unsigned long long*>(ctx->flags.as<char>() + 64);
  WS_CUDA(cudaMemsetAsync(nroots, 0, sizeof(unsigned long long), st));
  k_relabel<<<l.grid, l.block, 0, st>>>(L, aux, g, nroots);
  launched(ctx, PH_WS_RELABEL);
  tmark(ctx, st, PH_WS_RELABEL);
  WS_CUDA(cudaGetLastError());
  WS_CUDA(cudaMemcpyAsync(ctx->pinned, nroots, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  WS_CUDA(cudaStreamSynchronize(st));
  ctx->stats.n_regions = ctx->pinned[0];
  if (num_regions) *num_regions = ctx->pinned[0];
  return WS_OK;
}

ws_status run_watershed(ws_ctx* ctx, const uint8_t* grad, const Geo& g, int conn, int32_t* labels,
                        int64_t* num_regions, cudaStream_t st) {
  switch (conn) {
    case 4: return watershed_t<4>(ctx, grad, g, labels, num_regions, st);
    case 8: return watershed_t<8>(ctx, grad, g, labels, num_regions, st);
    case 6: return watershed_t<6>(ctx, grad, g, labels, num_regions, st);
    case 26: return watershed_t<26>(ctx, grad, g, labels, num_regions, st);
  }
  set_error(WS_ERR_INVALID, "connectivity must be 4, 8, 6 or 26");
  return WS_ERR_INVALID;
}

template <int CONN>
static ws_status debug_t(ws_ctx* ctx, const uint8_t* grad, const Geo& g, int32_t* dist, int32_t* parent,
                         cudaStream_t st) {
  WS_TRY(ctx->aux.ensure((size_t)g.N * sizeof(int), "aux"));
  int* L = ctx->aux.as<int>();
  WS_TRY(plateau_phase<CONN>(ctx, grad, g, L, st));
  const L3 l = launch3(g);
  k_plateau_dump<CONN><<<l.grid, l.block, 0, st>>>(L, g, dist, parent);
  launched(ctx, PH_WS_SELECT);
  WS_CUDA(cudaGetLastError());
  return WS_OK;
}

ws_status run_plateau_debug(ws_ctx* ctx, const uint8_t* grad, const Geo& g, int conn, int32_t* dist,
                            int32_t* parent, cudaStream_t st) {
  switch (conn) {
    case 4: return debug_t<4>(ctx, grad, g, dist, parent, st);
    case 8: return debug_t<8>(ctx, grad, g, dist, parent, st);
    case 6: return debug_t<6>(ctx, grad, g, dist, parent, st);
    case 26: return debug_t<26>(ctx, grad, g, dist, parent, st);
  }
  set_error(WS_ERR_INVALID, "connectivity must be 4, 8, 6 or 26");
  return WS_ERR_INVALID;
}

}  // namespace ws
