// ws_shard.cu — z-slab sharded watershed, sm_100a kernels.
//
// A rank owns global planes [z0, z1) and holds an EXTENDED slab [e0, e1) = [z0-2, z1+2) ∩ [0, D)
// of grad and of the working label array L (halo planes are filled by the caller's exchanges).
// In extended coordinates the owned planes are [zlo, zhi) and gofs = e0 * plane is the global
// index of extended voxel 0; every pointer value below is a GLOBAL voxel index.
//
//   ws_shard_plateau_first / _round / _halo   step I + distributed step II relaxation
//   ws_shard_local      pointers (k_resolve), local step III with exits (k_jump_shard),
//                       local step IV (k_union_shard), per-root minima, boundary table
//   ws_shard_merge      replicated cross-slab resolution over the gathered boundary tables:
//                       exit chasing, cut-plane union-find of minimal plateaux, canonical minima
//   ws_shard_relabel    canonical labels of the owned voxels
//
// Boundary table of one rank (plane = n1 * n2 voxels, slots s = 0: first owned plane,
// s = 1: last owned plane):
//   term[2][plane]    i32  final LOCAL root (global index) or -1 - e (exit voxel e)
//   rootmin[2][plane] i32  smallest owned voxel index reaching term (if term is a root)
//   exitmin[2][plane] i32  smallest owned voxel index whose terminal is exit e, e in the plane
//                          below z0 (s = 0) / above z1 - 1 (s = 1)   (INT_MAX: none)
//   I[2][plane]       u8   intensity of the voxel
//   rootI[2][plane]   u8   intensity of term (if term is a root)
#include <climits>
#include <vector>

#include "ws_internal.h"

namespace ws {
#ifdef WS_PX16
namespace px16 {  // ws_shard16.cu: the same phases on 16-bit pixels (NEXT f4)
using Px = uint16_t;
#else
using Px = uint8_t;
#endif

constexpr int NTS = 256;

struct Table {  // views into one rank's boundary table
  int* term;
  int* rootmin;
  int* exitmin;
  Px* I;
  Px* rootI;
};

// 2 slots x (term, rootmin, exitmin: 12 B + I, rootI: 2 sizeof(Px)) per plane voxel
__host__ __device__ inline size_t table_bytes(size_t plane) { return plane * (24 + 4 * sizeof(Px)); }

__host__ __device__ inline Table table_view(void* base, size_t plane) {
  Table t;
  char* b = static_cast<char*>(base);
  t.term = reinterpret_cast<int*>(b);
  t.rootmin = reinterpret_cast<int*>(b + plane * 8);
  t.exitmin = reinterpret_cast<int*>(b + plane * 16);
  t.I = reinterpret_cast<Px*>(b + plane * 24);
  t.rootI = reinterpret_cast<Px*>(b + plane * (24 + 2 * sizeof(Px)));
  return t;
}

__device__ __forceinline__ bool own_g(const Geo& g, int t) {  // global index t owned?
  const int l = t - g.gofs;
  return l >= g.zlo * g.plane && l < g.zhi * g.plane;
}

// ------------------------------------------------ step III inside the slab (exits kept)
// P[p] (global) -> terminal: an owned root (P[r] == r) or the first non-owned voxel e
// (stored as -1 - e).  L[root] accumulates INT_MAX - min{p}; exitmin planes the per-exit
// minima (as INT_MAX - p); roots go to the compact list.
__global__ void __launch_bounds__(NTS) k_jump_shard(int* P, int* L, Geo g, int* exitmx, int* roots, int cap,
                                                    int* nroots) {
  __shared__ int sbuf[2048];
  __shared__ int scount, sbase;
  if (threadIdx.x == 0) scount = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int lo = g.zlo * g.plane, hi = g.zhi * g.plane;
  const int stride = gridDim.x * NTS;
  int cnt = 0;  // staged roots: block-uniform (a register, never re-read from scount)
  for (int p0 = lo + blockIdx.x * NTS; p0 < hi; p0 += stride) {
    const int p = p0 + threadIdx.x;
    const bool valid = p < hi;
    int t = -2 - lane, code = 0;
    bool isr = false;
    if (valid) {
      t = P[p];
      if (t < 0) t = -1 - t;                // (never: k_resolve writes pointers only)
      while (true) {
        if (!own_g(g, t)) break;            // exit
        const int nt = P[t - g.gofs];
        if (nt == t) break;                 // root
        if (nt < 0) {                       // another thread already resolved t to an exit
          t = -1 - nt;
          break;
        }
        t = nt;
      }
      const bool ex = !own_g(g, t);
      code = ex ? -1 - t : t;
      if (code != P[p]) P[p] = code;
      isr = (t == p + g.gofs);
      if (ex) {
        const int e = t - g.gofs;           // extended index of the exit voxel
        const int s = e < lo ? 0 : 1;
        atomicMax(exitmx + s * g.plane + (e % g.plane), INT_MAX - (p + g.gofs));
      }
    }
    const int cprev = __shfl_up_sync(0xffffffffu, code, 1);
    if (valid && code >= 0 && (lane == 0 || cprev != code)) atomicMax(L + code - g.gofs, INT_MAX - (p + g.gofs));
    const unsigned rb = __ballot_sync(0xffffffffu, isr);
    if (rb) {
      int base = 0;
      if (lane == 0) base = atomicAdd(&scount, __popc(rb));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (isr) sbuf[base + __popc(rb & ((1u << lane) - 1))] = p + g.gofs;
    }
    cnt += __syncthreads_count(isr);
    if (cnt > 2048 - NTS || p0 + stride >= hi) {
      if (cnt > 0) {
        if (threadIdx.x == 0) sbase = atomicAdd(nroots, cnt);
        __syncthreads();
        for (int i = threadIdx.x; i < cnt; i += NTS)
          if (sbase + i < cap) roots[sbase + i] = sbuf[i];
      }
      __syncthreads();
      if (threadIdx.x == 0) scount = 0;
      __syncthreads();
      cnt = 0;
    }
  }
}

// union-find on P with global values (owned roots only)
__device__ __forceinline__ int sfind(int* P, const Geo& g, int x) {
  while (true) {
    const int y = __ldcg(P + x - g.gofs);
    if (y == x) return x;
    const int z = __ldcg(P + y - g.gofs);
    if (z == y) return y;
    __stcg(P + x - g.gofs, z);
    x = z;
  }
}

__device__ __forceinline__ int sfind_ro(const int* P, const Geo& g, int x) {
  while (true) {
    const int y = __ldcg(P + x - g.gofs);
    if (y == x) return x;
    x = y;
  }
}

// step IV inside the slab on the cross-tile pairs k_resolve listed (global indices)
__global__ void k_union_pairs_shard(int* P, const int2* __restrict__ pairs, int n, Geo g) {
  for (int i = blockIdx.x * NTS + threadIdx.x; i < n; i += gridDim.x * NTS) {
    int a = pairs[i].x, b = pairs[i].y;
    while (true) {
      a = sfind(P, g, a);
      b = sfind(P, g, b);
      if (a == b) break;
      if (a > b) { const int t = a; a = b; b = t; }
      if (atomicCAS(P + b - g.gofs, b, a) == b) break;
    }
  }
}

// step IV inside the slab (fallback when the pair list overflowed): pairs of owned voxels (q > p) on one minimal plateau.  A voxel
// whose terminal is an exit descends out of the slab and is never on a minimal plateau
// (minimal-plateau pointers are kept inside the slab by k_resolve).
template <int CONN>
__global__ void k_union_shard(const Px* __restrict__ I, int* P, Geo g) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= g.n2 || y >= g.n1) return;
  for (int z = g.zlo + blockIdx.z; z < g.zhi; z += gridDim.z) {
    const int p = z * g.plane + y * g.n2 + x;
    const int r = __ldcg(P + p);
    if (r < 0) continue;
    const int v = I[p];
    if (I[r - g.gofs] != v) continue;
#pragma unroll
    for (int i = Conn<CONN>::nfwd; i < CONN; ++i) {
      if (!nb_in<CONN>(g, z, y, x, i)) continue;
      int dz, dy, dx;
      nb_delta(CONN, i, dz, dy, dx);
      if (z + dz >= g.zhi) continue;  // the cut plane is merged by ws_shard_merge
      const int q = p + nb_off<CONN>(g, i);
      if (I[q] != v) continue;
      int a = p + g.gofs, b = q + g.gofs;
      while (true) {
        a = sfind(P, g, a);
        b = sfind(P, g, b);
        if (a == b) break;
        if (a > b) { const int t = a; a = b; b = t; }
        if (atomicCAS(P + b - g.gofs, b, a) == b) break;
      }
    }
  }
}

// fold every listed root's minimum into its final local root
__global__ void k_root_fold(const int* P, int* L, const int* __restrict__ roots, int n, Geo g) {
  for (int i = blockIdx.x * NTS + threadIdx.x; i < n; i += gridDim.x * NTS) {
    const int r = roots[i];
    const int f = sfind_ro(P, g, r);
    if (f != r) atomicMax(L + f - g.gofs, L[r - g.gofs]);
  }
}

// boundary table of the owned first/last planes (+ the exit minima)
__global__ void k_table(const Px* __restrict__ I, const int* P, const int* __restrict__ L,
                        const int* __restrict__ exitmx, Geo g, Table t) {
  const int n = 2 * g.plane;
  for (int i = blockIdx.x * NTS + threadIdx.x; i < n; i += gridDim.x * NTS) {
    const int s = i / g.plane, xy = i % g.plane;
    const int z = s == 0 ? g.zlo : g.zhi - 1;
    const int p = z * g.plane + xy;
    const int c = P[p];
    int term, rmin = INT_MAX;
    Px ri = 0;
    if (c >= 0) {
      term = sfind_ro(P, g, c);
      rmin = INT_MAX - L[term - g.gofs];
      ri = I[term - g.gofs];
    } else {
      term = c;
    }
    t.term[i] = term;
    t.rootmin[i] = rmin;
    t.rootI[i] = ri;
    t.I[i] = I[p];
    const int em = exitmx[i];
    t.exitmin[i] = em > 0 ? INT_MAX - em : INT_MAX;
  }
}

// ---------------------------------------------------------- replicated cross-slab merge
struct Slabs {
  const int* z0;  // [K]
  const int* z1;  // [K]
  int K;
  int plane;
  char* tables;   // K tables, table_bytes(plane) apart
};

// table entry (rank * 2 + slot) * plane + xy of a global voxel lying on a boundary plane
__device__ __forceinline__ long long entry_of(const Slabs& S, int e) {
  const int z = e / S.plane, xy = e % S.plane;
  int lo = 0, hi = S.K - 1;
  while (lo < hi) {  // owner rank: z0[r] <= z < z1[r]
    const int mid = (lo + hi + 1) >> 1;
    if (S.z0[mid] <= z) lo = mid; else hi = mid - 1;
  }
  const int slot = (z == S.z0[lo]) ? 0 : 1;
  return ((long long)lo * 2 + slot) * S.plane + xy;
}

__device__ __forceinline__ Table tab(const Slabs& S, int r) {
  return table_view(S.tables + (size_t)r * table_bytes(S.plane), S.plane);
}

// R0 of every boundary voxel of every rank: chase exits through the tables to a root
__global__ void k_merge_resolve(Slabs S, int* R0) {
  const long long n = (long long)S.K * 2 * S.plane;
  for (long long i = blockIdx.x * (long long)NTS + threadIdx.x; i < n; i += (long long)gridDim.x * NTS) {
    int t = tab(S, (int)(i / (2 * S.plane))).term[i % (2 * S.plane)];
    while (t < 0) {
      const long long e = entry_of(S, -1 - t);
      t = tab(S, (int)(e / (2 * S.plane))).term[e % (2 * S.plane)];
    }
    R0[i] = t;
  }
}

// open-addressing map root -> {parent, canonical minimum}
struct RootMap {
  int* key;
  int* parent;
  int* mn;
  unsigned mask;
};

__device__ __forceinline__ unsigned rm_hash(int k) { return (unsigned)k * 0x9E3779B1u; }

__device__ __forceinline__ unsigned rm_insert(const RootMap& M, int k) {
  unsigned h = rm_hash(k) & M.mask;
  while (true) {
    const int cur = atomicCAS(M.key + h, -1, k);
    if (cur == -1 || cur == k) return h;
    h = (h + 1) & M.mask;
  }
}

__device__ __forceinline__ unsigned rm_slot(const RootMap& M, int k) {
  unsigned h = rm_hash(k) & M.mask;
  while (__ldcg(M.key + h) != k) h = (h + 1) & M.mask;
  return h;
}

__device__ __forceinline__ int rm_find(const RootMap& M, int k) {
  while (true) {
    const int p = __ldcg(M.parent + rm_slot(M, k));
    if (p == k) return k;
    k = p;
  }
}

__global__ void k_merge_insert(const int* R0, long long n, RootMap M) {
  for (long long i = blockIdx.x * (long long)NTS + threadIdx.x; i < n; i += (long long)gridDim.x * NTS) {
    const int k = R0[i];
    const unsigned h = rm_insert(M, k);
    M.parent[h] = k;  // every insert of k writes the same value
  }
}

// cut-plane unions: last plane of rank r vs first plane of rank r + 1 -- the voxel straight
// above (6-connectivity) or the 3 x 3 voxels above (26) -- both on one minimal plateau
// (I equal and I(root) == I: an equal-valued neighbour lies on the same plateau)
__global__ void k_merge_union(Slabs S, const int* R0, RootMap M, int n2, int diag) {
  const long long n = (long long)(S.K - 1) * S.plane;
  const int n1 = S.plane / n2;
  for (long long i = blockIdx.x * (long long)NTS + threadIdx.x; i < n; i += (long long)gridDim.x * NTS) {
    const int r = (int)(i / S.plane), xy = (int)(i % S.plane);
    const Table A = tab(S, r), B = tab(S, r + 1);
    const int ia = S.plane + xy;  // slot 1 of r
    if (A.term[ia] < 0 || A.rootI[ia] != A.I[ia]) continue;
    const int x = xy % n2, y = xy / n2;
    for (int dy = -diag; dy <= diag; ++dy)
      for (int dx = -diag; dx <= diag; ++dx) {
        if ((unsigned)(x + dx) >= (unsigned)n2 || (unsigned)(y + dy) >= (unsigned)n1) continue;
        const int ib = xy + dy * n2 + dx;  // slot 0 of r + 1
        if (A.I[ia] != B.I[ib]) continue;
        int a = R0[(long long)r * 2 * S.plane + ia], b = R0[(long long)(r + 1) * 2 * S.plane + ib];
        while (true) {
          a = rm_find(M, a);
          b = rm_find(M, b);
          if (a == b) break;
          if (a > b) { const int t = a; a = b; b = t; }
          if (atomicCAS(M.parent + rm_slot(M, b), b, a) == b) break;
        }
      }
  }
}

// canonical minima of the merged regions: owned-root minima and exit minima
__global__ void k_merge_min(Slabs S, const int* R0, RootMap M) {
  const long long n = (long long)S.K * 2 * S.plane;
  for (long long i = blockIdx.x * (long long)NTS + threadIdx.x; i < n; i += (long long)gridDim.x * NTS) {
    const int r = (int)(i / (2 * S.plane));
    const int j = (int)(i % (2 * S.plane));
    const Table T = tab(S, r);
    if (T.term[j] >= 0) atomicMin(M.mn + rm_slot(M, rm_find(M, R0[i])), T.rootmin[j]);
    const int em = T.exitmin[j];
    if (em != INT_MAX) {
      const int s = j / S.plane, xy = j % S.plane;
      const int ez = s == 0 ? S.z0[r] - 1 : S.z1[r];
      const long long e = entry_of(S, ez * S.plane + xy);
      atomicMin(M.mn + rm_slot(M, rm_find(M, R0[e])), em);
    }
  }
}

// this rank: canonical label into L[final local root] of every referenced owned root, and
// into exitcanon for every exit plane voxel
__global__ void k_merge_apply(Slabs S, const int* R0, RootMap M, int rank, Geo g, int* L, int* exitcanon) {
  const int n = 2 * S.plane;
  const Table T = tab(S, rank);
  for (int j = blockIdx.x * NTS + threadIdx.x; j < n; j += gridDim.x * NTS) {
    const long long i = (long long)rank * 2 * S.plane + j;
    if (T.term[j] >= 0) L[T.term[j] - g.gofs] = INT_MAX - M.mn[rm_slot(M, rm_find(M, R0[i]))];
    const int s = j / S.plane, xy = j % S.plane;
    const int ez = s == 0 ? S.z0[rank] - 1 : S.z1[rank];
    int c = INT_MAX;
    if (ez >= 0 && (s == 0 ? rank > 0 : rank < S.K - 1)) {
      const long long e = entry_of(S, ez * S.plane + xy);
      c = M.mn[rm_slot(M, rm_find(M, R0[e]))];
    }
    exitcanon[j] = c;
  }
}

// every listed root takes its final root's value; then labels of the owned voxels
__global__ void k_root_spread(const int* P, int* L, const int* __restrict__ roots, int n, Geo g) {
  for (int i = blockIdx.x * NTS + threadIdx.x; i < n; i += gridDim.x * NTS) {
    const int r = roots[i];
    const int f = sfind_ro(P, g, r);
    if (f != r) L[r - g.gofs] = L[f - g.gofs];
  }
}

__global__ void k_relabel_shard(const int* __restrict__ P, const int* __restrict__ L, const int* __restrict__ exitcanon,
                                Geo g, int* __restrict__ out, unsigned long long* nreps) {
  const int lo = g.zlo * g.plane, hi = g.zhi * g.plane;
  for (int p = lo + blockIdx.x * NTS + threadIdx.x; p < hi; p += gridDim.x * NTS) {
    const int t = P[p];
    int c;
    if (t >= 0) {
      c = INT_MAX - L[t - g.gofs];
    } else {
      const int e = -1 - t - g.gofs;
      c = exitcanon[(e < lo ? 0 : g.plane) + e % g.plane];
    }
    out[p - lo] = c;
    const unsigned act = __activemask();
    const unsigned b = __ballot_sync(act, c == p + g.gofs);
    if (b && (threadIdx.x & 31) == __ffs(act) - 1) atomicAdd(nreps, (unsigned long long)__popc(b));
  }
}

// ================================================================== host side
ws_status plateau_first_shard(ws_ctx* ctx, const Px* grad, const Geo& g, int conn, int32_t* L, int* pending,
                              cudaStream_t st);
ws_status plateau_round_shard(ws_ctx* ctx, const Px* grad, const Geo& g, int conn, int32_t* L, int act_lo,
                              int act_hi, int* pending, cudaStream_t st);
ws_status resolve_shard(ws_ctx* ctx, const Px* grad, const Geo& g, int conn, const int32_t* L, int32_t* P,
                        cudaStream_t st);

static int grid_s(long long n, int sms) {
  long long b = (n + NTS - 1) / NTS;
  long long cap = (long long)sms * 8;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

ws_status shard_local(ws_ctx* ctx, const Px* grad, const Geo& g, int conn, int32_t* L, int32_t* P, void* table,
                      cudaStream_t st) {
  WS_TRY(resolve_shard(ctx, grad, g, conn, L, P, st));
  const size_t own = (size_t)(g.zhi - g.zlo) * g.plane;
  const size_t want = own / 16 + 1024;
  if (ctx->roots.bytes / sizeof(int) < want) {
    WS_TRY(ctx->roots.ensure(want * sizeof(int), "roots"));
  }
  size_t cap = ctx->roots.bytes / sizeof(int);
  WS_TRY(ctx->flags.ensure(256, "flags"));
  WS_TRY(ctx->exitmx.ensure((size_t)2 * g.plane * sizeof(int), "exit minima"));
  int* nr = ctx->flags.as<int>() + 8;
  WS_CUDA(cudaMemsetAsync(nr, 0, 2 * sizeof(int), st));  // [0] roots, [1] unused ([2] = pairs, set by pair_out)
  WS_CUDA(cudaMemsetAsync(ctx->exitmx.p, 0, (size_t)2 * g.plane * sizeof(int), st));
  const int gN = grid_s((long long)own, ctx->num_sms);
  k_jump_shard<<<gN, NTS, 0, st>>>(P, L, g, ctx->exitmx.as<int>(), ctx->roots.as<int>(), (int)cap, nr);
  launched(ctx, PH_WS_JUMP);
  WS_CUDA(cudaMemcpyAsync(ctx->pinned, nr, 3 * sizeof(int), cudaMemcpyDeviceToHost, st));  // nr, -, npairs
  WS_CUDA(cudaStreamSynchronize(st));
  int n_roots = reinterpret_cast<const int*>(ctx->pinned)[0];
  const int n_pairs = reinterpret_cast<const int*>(ctx->pinned)[2];
  const int pcap = (int)(ctx->upairs.bytes / sizeof(int2));
  if ((size_t)n_roots > cap) {
    set_error(WS_ERR_LIMIT, "ws_shard_local: more than %zu step III roots in one slab", cap);
    return WS_ERR_LIMIT;
  }
  tmark(ctx, st, PH_WS_JUMP);
  if (n_pairs <= pcap) {
    if (n_pairs > 0) {
      k_union_pairs_shard<<<grid_s(n_pairs, ctx->num_sms), NTS, 0, st>>>(P, ctx->upairs.as<int2>(), n_pairs, g);
      launched(ctx, PH_WS_UNION);
    }
  } else {
    L3 l = launch3(g);
    l.grid.z = (g.zhi - g.zlo) < 65535 ? (g.zhi - g.zlo) : 65535;
    if (conn == 26) k_union_shard<26><<<l.grid, l.block, 0, st>>>(grad, P, g);
    else k_union_shard<6><<<l.grid, l.block, 0, st>>>(grad, P, g);
    launched(ctx, PH_WS_UNION);
  }
  tmark(ctx, st, PH_WS_UNION);
  const int gR = grid_s(n_roots, ctx->num_sms);
  k_root_fold<<<gR, NTS, 0, st>>>(P, L, ctx->roots.as<int>(), n_roots, g);
  k_table<<<grid_s(2LL * g.plane, ctx->num_sms), NTS, 0, st>>>(grad, P, L, ctx->exitmx.as<int>(), g,
                                                                 table_view(table, g.plane));
  launched(ctx, PH_WS_FIND, 2);
  tmark(ctx, st, PH_WS_FIND);
  ctx->stats.n_regions = n_roots;
  ctx->shard_nroots = n_roots;
  ctx->shard_conn = conn;  // ws_shard_merge's cut-plane adjacency
  WS_CUDA(cudaGetLastError());
  return WS_OK;
}

ws_status shard_merge(ws_ctx* ctx, const void* tables, const int64_t* z0s, const int64_t* z1s, int K, int rank,
                      const Geo& g, int32_t* L, int32_t* exitcanon, cudaStream_t st) {
  const size_t tb = table_bytes(g.plane);
  WS_TRY(ctx->mtables.ensure(tb * K, "gathered tables"));
  WS_TRY(ctx->mslabs.ensure(2 * K * sizeof(int), "slab bounds"));
  std::vector<int> zz(2 * K);
  for (int r = 0; r < K; ++r) { zz[r] = (int)z0s[r]; zz[K + r] = (int)z1s[r]; }
  WS_CUDA(cudaMemcpyAsync(ctx->mslabs.p, zz.data(), 2 * K * sizeof(int), cudaMemcpyHostToDevice, st));
  if (tables != ctx->mtables.p)
    WS_CUDA(cudaMemcpyAsync(ctx->mtables.p, tables, tb * K, cudaMemcpyDeviceToDevice, st));
  Slabs S;
  S.z0 = ctx->mslabs.as<int>();
  S.z1 = S.z0 + K;
  S.K = K;
  S.plane = g.plane;
  S.tables = ctx->mtables.as<char>();
  const long long n = (long long)K * 2 * g.plane;
  unsigned cap = 1;
  while (cap < 2 * n) cap <<= 1;
  WS_TRY(ctx->mr0.ensure((size_t)n * sizeof(int), "R0"));
  WS_TRY(ctx->mmap.ensure((size_t)cap * 3 * sizeof(int), "root map"));
  RootMap M;
  M.key = ctx->mmap.as<int>();
  M.parent = M.key + cap;
  M.mn = M.parent + cap;
  M.mask = cap - 1;
  WS_CUDA(cudaMemsetAsync(M.key, 0xFF, (size_t)cap * sizeof(int), st));
  WS_CUDA(cudaMemsetAsync(M.mn, 0x7F, (size_t)cap * sizeof(int), st));
  int* R0 = ctx->mr0.as<int>();
  const int gg = grid_s(n, ctx->num_sms);
  k_merge_resolve<<<gg, NTS, 0, st>>>(S, R0);
  k_merge_insert<<<gg, NTS, 0, st>>>(R0, n, M);
  if (K > 1)
    k_merge_union<<<grid_s((long long)(K - 1) * g.plane, ctx->num_sms), NTS, 0, st>>>(S, R0, M, g.n2,
                                                                                     ctx->shard_conn == 26 ? 1 : 0);
  k_merge_min<<<gg, NTS, 0, st>>>(S, R0, M);
  k_merge_apply<<<grid_s(2LL * g.plane, ctx->num_sms), NTS, 0, st>>>(S, R0, M, rank, g, L, exitcanon);
  launched(ctx, PH_WS_FIND, K > 1 ? 5 : 4);
  WS_CUDA(cudaGetLastError());
  return WS_OK;
}

ws_status shard_relabel(ws_ctx* ctx, const int32_t* P, int32_t* L, const int32_t* exitcanon, const Geo& g,
                        int32_t* labels_own, int64_t* nreps, cudaStream_t st) {
  const int n_roots = ctx->shard_nroots;
  if (n_roots > 0)
    k_root_spread<<<grid_s(n_roots, ctx->num_sms), NTS, 0, st>>>(P, L, ctx->roots.as<int>(), n_roots, g);
  unsigned long long* nr = reinterpret_cast<unsigned long long*>(ctx->flags.as<char>() + 64);
  WS_CUDA(cudaMemsetAsync(nr, 0, sizeof(unsigned long long), st));
  const long long own = (long long)(g.zhi - g.zlo) * g.plane;
  k_relabel_shard<<<grid_s(own, ctx->num_sms), NTS, 0, st>>>(P, L, exitcanon, g, labels_own, nr);
  launched(ctx, PH_WS_RELABEL, 2);
  tmark(ctx, st, PH_WS_RELABEL);
  WS_CUDA(cudaGetLastError());
  if (nreps) {
    WS_CUDA(cudaMemcpyAsync(ctx->pinned, nr, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    WS_CUDA(cudaStreamSynchronize(st));
    *nreps = ctx->pinned[0];
  }
  return WS_OK;
}

// copy a received halo plane into L (side 0: plane zlo - 1, side 1: plane zhi); flag changes
__global__ void k_halo_in(int* L, Geo g, int side, const int* __restrict__ in, int* changed) {
  const int z = side == 0 ? g.zlo - 1 : g.zhi;
  int* dst = L + (size_t)z * g.plane;
  bool ch = false;
  for (int i = blockIdx.x * NTS + threadIdx.x; i < g.plane; i += gridDim.x * NTS) {
    const int v = in[i];
    if (dst[i] != v) {
      dst[i] = v;
      ch = true;
    }
  }
  if (__syncthreads_or(ch) && threadIdx.x == 0) *changed = 1;
}

ws_status shard_halo(ws_ctx* ctx, int32_t* L, const Geo& g, int side, const int32_t* plane_in, int32_t* changed,
                     cudaStream_t st) {
  WS_TRY(ctx->flags.ensure(256, "flags"));
  int* f = ctx->flags.as<int>() + 12;
  WS_CUDA(cudaMemsetAsync(f, 0, sizeof(int), st));
  k_halo_in<<<grid_s(g.plane, ctx->num_sms), NTS, 0, st>>>(L, g, side, plane_in, f);
  WS_CUDA(cudaMemcpyAsync(ctx->pinned, f, sizeof(int), cudaMemcpyDeviceToHost, st));
  WS_CUDA(cudaStreamSynchronize(st));
  *changed = reinterpret_cast<const int*>(ctx->pinned)[0];
  return WS_OK;
}

size_t shard_table_bytes(size_t plane) { return table_bytes(plane); }

#ifdef WS_PX16
}  // namespace px16
#endif
}  // namespace ws
