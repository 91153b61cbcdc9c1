// ws_watershed.cu — steps I-IV of PRUF (Alg. 1) + canonical relabel, sm_100a.
//
// Tile design: the volume is cut into tiles of 2048 voxels
// (3-D 32x8x8, 2-D 64x32) staged in shared memory with a halo.  Intensities are staged as
// 16-bit values with an out-of-volume sentinel (0xFFFF: never lower, never equal), so the
// stencil loops carry no bounds checks.
//
//   k_relax_first  step I classification (Alg. 1 l.1-10) fused with the first round of the
//                  step II distance relaxation (Alg. 3 l.7-8) inside each tile      [all tiles]
//   k_relax_round  further step II rounds, only on tiles whose halo changed       [active tiles]
//   k_resolve      step I/II pointers (Eq. 1; C5/C6 selection) + tile-local pointer
//                  jumping in shared memory (step III inside the tile)  -> P        [all tiles]
//   k_jump         step III across tiles: chase exits to the self-loop roots (l.19-23/28-29);
//                  per-root minimum voxel index (warp-aggregated atomicMax on INT_MAX - p);
//                  compact list of roots
//   k_union        step IV Union over q > p (l.24-27), lock-free min-root CAS on the roots
//   k_root_merge / k_root_label / k_root_store   step IV Find (l.28-29) on the root list only:
//                  canonical label (C7) of every final region, stored into P[root]
//   k_relabel      labels[p] = canonical label of p's root
//
// Arrays: L = the caller's `labels` (i32[N]); during step II it holds the plateau distance
// code of ws_common.cuh (L >= 0: d = 0; L < 0: -1 - (d << 5)).  P = ctx->aux (i32[N]) holds
// pointers from k_resolve on.  From k_jump on, L[r] of a root r holds INT_MAX - (smallest
// voxel index reaching r); all other L entries are dead until k_relabel writes the output.
#include <climits>

#include "ws_internal.h"

namespace ws {

constexpr int NT = 256;
constexpr int INF = DUNREACHED;
using u16 = unsigned short;
constexpr int OOB = 0xFFFF;  // out-of-volume intensity sentinel in shared memory

template <int CONN> struct Tile {
  static constexpr bool is3d = Conn<CONN>::is3d;
  static constexpr int TX = is3d ? 32 : 64;
  static constexpr int TY = is3d ? 8 : 32;
  static constexpr int TZ = is3d ? 8 : 1;
  static constexpr int V = TX * TY * TZ;
  static constexpr int VPT = V / NT;
  static_assert(V % NT == 0, "tile");
};

// shared-memory box of the tile plus a halo of H voxels (no halo across axis 0 in 2-D)
template <int CONN, int H> struct Box {
  using T = Tile<CONN>;
  static constexpr int HZ = T::is3d ? H : 0;
  static constexpr int SX = T::TX + 2 * H, SY = T::TY + 2 * H, SZ = T::TZ + 2 * HZ;
  static constexpr int S = SX * SY * SZ;
  __device__ static constexpr int at(int lz, int ly, int lx) { return ((lz + HZ) * SY + (ly + H)) * SX + (lx + H); }
  __device__ static constexpr int off(int i) {
    int dz = 0, dy = 0, dx = 0;
    nb_delta(CONN, i, dz, dy, dx);
    return (dz * SY + dy) * SX + dx;
  }
};

struct TileCoord {
  int bx, by, bz;  // global coordinates of the tile origin
};

template <int CONN>
__device__ __forceinline__ TileCoord tile_coord(int t, int ntx, int nty) {
  using T = Tile<CONN>;
  TileCoord c;
  c.bx = (t % ntx) * T::TX;
  c.by = ((t / ntx) % nty) * T::TY;
  c.bz = (t / (ntx * nty)) * T::TZ;
  return c;
}

// voxel k of this thread inside the tile: j = threadIdx.x + k * NT (x fastest)
template <int CONN>
__device__ __forceinline__ void my_voxel(int k, int& lx, int& ly, int& lz) {
  using T = Tile<CONN>;
  const int j = threadIdx.x + k * NT;
  lx = j % T::TX;
  ly = (j / T::TX) % T::TY;
  lz = j / (T::TX * T::TY);
}

// row-wise staging: one warp per (sz, sy) row, lanes along x
template <int CONN, int H>
__device__ __forceinline__ void load_I(const uint8_t* __restrict__ I, const Geo& g, const TileCoord& c, u16* sI) {
  using B = Box<CONN, H>;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int r = warp; r < B::SY * B::SZ; r += NT / 32) {
    const int sy = r % B::SY, sz = r / B::SY;
    const int gy = c.by + sy - H, gz = c.bz + sz - B::HZ;
    const bool rowok = (unsigned)gy < (unsigned)g.n1 && (unsigned)gz < (unsigned)g.n0;
    const uint8_t* row = I + ((size_t)(rowok ? gz : 0) * g.plane + (size_t)(rowok ? gy : 0) * g.n2);
#pragma unroll
    for (int sx = lane; sx < B::SX; sx += 32) {
      const int gx = c.bx + sx - H;
      int v = OOB;
      if (rowok && (unsigned)gx < (unsigned)g.n2) v = __ldg(row + gx);
      sI[r * B::SX + sx] = (u16)v;
    }
  }
}

// distances of the tile + 1-voxel halo from the L code (out of the volume: INF, never read)
template <int CONN>
__device__ __forceinline__ void load_D(const int* L, const Geo& g, const TileCoord& c, int* sD) {
  using B = Box<CONN, 1>;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int r = warp; r < B::SY * B::SZ; r += NT / 32) {
    const int sy = r % B::SY, sz = r / B::SY;
    const int gy = c.by + sy - 1, gz = c.bz + sz - B::HZ;
    const bool rowok = (unsigned)gy < (unsigned)g.n1 && (unsigned)gz < (unsigned)g.n0;
    const int* row = L + ((size_t)(rowok ? gz : 0) * g.plane + (size_t)(rowok ? gy : 0) * g.n2);
#pragma unroll
    for (int sx = lane; sx < B::SX; sx += 32) {
      const int gx = c.bx + sx - 1;
      int d = INF;
      if (rowok && (unsigned)gx < (unsigned)g.n2) d = dec_d(row[gx]);
      sD[r * B::SX + sx] = d;
    }
  }
}

// Mark the (up to 26) neighbouring tiles for the next relaxation round.
template <int CONN>
__device__ __forceinline__ void mark_neighbours(int t, int ntx, int nty, int ntz, uint8_t* next, int* any) {
  const int tx = t % ntx, ty = (t / ntx) % nty, tz = t / (ntx * nty);
  const int i = threadIdx.x;
  constexpr int ZR = Tile<CONN>::is3d ? 1 : 0;
  if (i < 27) {
    const int dz = i / 9 - 1, dy = (i / 3) % 3 - 1, dx = i % 3 - 1;
    if ((dz == 0 || ZR) && !(dz == 0 && dy == 0 && dx == 0)) {
      const int x = tx + dx, y = ty + dy, z = tz + dz;
      if ((unsigned)x < (unsigned)ntx && (unsigned)y < (unsigned)nty && (unsigned)z < (unsigned)ntz)
        next[(z * nty + y) * ntx + x] = 1;
    }
  }
  if (i == 0) *any = 1;
}

// in-tile relaxation sweeps until the tile converges (chaotic, in place)
template <int CONN, int H>
__device__ __forceinline__ void relax_tile(int* sD, const int* my, const unsigned* eqm, int* limit) {
  using B = Box<CONN, H>;
  using T = Tile<CONN>;
  while (true) {
    bool ch = false;
#pragma unroll
    for (int k = 0; k < T::VPT; ++k) {
      const unsigned m = eqm[k];
      if (!m) continue;
      const int s = my[k];
      const int cur = sD[s];
      int best = cur;
#pragma unroll
      for (int i = 0; i < CONN; ++i)
        if (m & (1u << i)) best = min(best, sD[s + B::off(i)] + 1);
      if (best < cur) {
        sD[s] = best;
        ch = true;
        if (best >= INF - 1) *limit = 1;
      }
    }
    if (!__syncthreads_or(ch)) break;
  }
}

template <int CONN>
__device__ __forceinline__ bool on_tile_border(int lx, int ly, int lz) {
  using T = Tile<CONN>;
  return lx == 0 || lx == T::TX - 1 || ly == 0 || ly == T::TY - 1 || (T::is3d && (lz == 0 || lz == T::TZ - 1));
}

// ------------------------------------------- step I + first step II round (all tiles)
template <int CONN>
__global__ void __launch_bounds__(NT) k_relax_first(const uint8_t* __restrict__ I, int* __restrict__ L, Geo g,
                                                     int ntx, int nty, int ntz, uint8_t* next,
                                                     uint8_t* hasplat, int* flags) {
  using T = Tile<CONN>;
  using B2 = Box<CONN, 2>;
  using B1 = Box<CONN, 1>;
  __shared__ u16 sI[B2::S];
  __shared__ int sD[B2::S];
  const int t = blockIdx.x;
  const TileCoord c = tile_coord<CONN>(t, ntx, nty);
  load_I<CONN, 2>(I, g, c, sI);
  __syncthreads();
  // classify the tile + 1-voxel halo: lower -> 0, plateau without lower -> INF (Alg. 1 l.3-10)
  for (int s = threadIdx.x; s < B1::S; s += NT) {
    const int sx = s % B1::SX, sy = (s / B1::SX) % B1::SY, sz = s / (B1::SX * B1::SY);
    const int s2 = B2::at(sz - B1::HZ, sy - 1, sx - 1);
    const int v = sI[s2];
    bool lower = false, eq = false;
#pragma unroll
    for (int i = 0; i < CONN; ++i) {
      const int nv = sI[s2 + B2::off(i)];
      lower |= nv < v;
      eq |= nv == v;
    }
    sD[s2] = (v == OOB) ? INF : (lower ? 0 : (eq ? INF : 0));
  }
  __syncthreads();
  int my[T::VPT];
  unsigned eqm[T::VPT];
  bool any_plat = false;
#pragma unroll
  for (int k = 0; k < T::VPT; ++k) {
    int lx, ly, lz;
    my_voxel<CONN>(k, lx, ly, lz);
    my[k] = B2::at(lz, ly, lx);
    const int v = sI[my[k]];
    unsigned m = 0;
    if (v != OOB && sD[my[k]] == INF) {
#pragma unroll
      for (int i = 0; i < CONN; ++i)
        if (sI[my[k] + B2::off(i)] == v) m |= 1u << i;
      any_plat = true;
    }
    eqm[k] = m;
  }
  relax_tile<CONN, 2>(sD, my, eqm, flags + 1);
  bool border = false;
#pragma unroll
  for (int k = 0; k < T::VPT; ++k) {
    int lx, ly, lz;
    my_voxel<CONN>(k, lx, ly, lz);
    if (sI[my[k]] == OOB) continue;
    const int d = sD[my[k]];
    L[(size_t)(c.bz + lz) * g.plane + (size_t)(c.by + ly) * g.n2 + c.bx + lx] = eqm[k] ? enc(d, DIR_NONE) : 0;
    if (eqm[k] && d != INF && on_tile_border<CONN>(lx, ly, lz)) border = true;
  }
  const int hp = __syncthreads_or(any_plat);
  if (threadIdx.x == 0) hasplat[t] = hp ? 1 : 0;
  if (__syncthreads_or(border)) mark_neighbours<CONN>(t, ntx, nty, ntz, next, flags);
}

// ------------------------------------------------ further step II rounds (active tiles)
template <int CONN>
__global__ void __launch_bounds__(NT) k_relax_round(const uint8_t* __restrict__ I, int* __restrict__ L, Geo g,
                                                     int ntx, int nty, int ntz, const uint8_t* cur,
                                                     uint8_t* next, const uint8_t* hasplat, int* flags) {
  using T = Tile<CONN>;
  using B = Box<CONN, 1>;
  const int t = blockIdx.x;
  if (!cur[t] || !hasplat[t]) return;
  __shared__ u16 sI[B::S];
  __shared__ int sD[B::S];
  const TileCoord c = tile_coord<CONN>(t, ntx, nty);
  load_I<CONN, 1>(I, g, c, sI);
  load_D<CONN>(L, g, c, sD);
  __syncthreads();
  int my[T::VPT], d0[T::VPT];
  unsigned eqm[T::VPT];
#pragma unroll
  for (int k = 0; k < T::VPT; ++k) {
    int lx, ly, lz;
    my_voxel<CONN>(k, lx, ly, lz);
    my[k] = B::at(lz, ly, lx);
    const int v = sI[my[k]];
    d0[k] = sD[my[k]];
    unsigned m = 0;
    if (v != OOB && d0[k] > 0) {  // plateau voxel (d >= 1)
#pragma unroll
      for (int i = 0; i < CONN; ++i)
        if (sI[my[k] + B::off(i)] == v) m |= 1u << i;
    }
    eqm[k] = m;
  }
  relax_tile<CONN, 1>(sD, my, eqm, flags + 1);
  bool border = false;
#pragma unroll
  for (int k = 0; k < T::VPT; ++k) {
    if (!eqm[k]) continue;
    const int d = sD[my[k]];
    if (d == d0[k]) continue;
    int lx, ly, lz;
    my_voxel<CONN>(k, lx, ly, lz);
    L[(size_t)(c.bz + lz) * g.plane + (size_t)(c.by + ly) * g.n2 + c.bx + lx] = enc(d, DIR_NONE);
    if (on_tile_border<CONN>(lx, ly, lz)) border = true;
  }
  if (__syncthreads_or(border)) mark_neighbours<CONN>(t, ntx, nty, ntz, next, flags);
}

// ---------------------- pointers (steps I-II) + tile-local pointer jumping (step III)
// DEBUG: write the un-jumped parent and the distance instead (ws_plateau_debug, T2).
template <int CONN, bool DEBUG>
__global__ void __launch_bounds__(NT) k_resolve(const uint8_t* __restrict__ I, const int* __restrict__ L, Geo g,
                                                int ntx, int nty, int* __restrict__ P, int* __restrict__ dist) {
  using T = Tile<CONN>;
  using B = Box<CONN, 1>;
  __shared__ u16 sI[B::S];
  __shared__ int sD[B::S];
  __shared__ short sP[T::V];  // local target, -1 = leaves the tile
  __shared__ int sG[T::V];    // global target when leaving the tile
  const int t = blockIdx.x;
  const TileCoord c = tile_coord<CONN>(t, ntx, nty);
  load_I<CONN, 1>(I, g, c, sI);
  load_D<CONN>(L, g, c, sD);
  __syncthreads();
#pragma unroll
  for (int k = 0; k < T::VPT; ++k) {
    int lx, ly, lz;
    my_voxel<CONN>(k, lx, ly, lz);
    const int j = threadIdx.x + k * NT;
    const int s = B::at(lz, ly, lx);
    const int v = sI[s];
    if (v == OOB) {
      sP[j] = (short)j;
      continue;
    }
    int m = 0x10000, dm = 0;
    unsigned eqm = 0;
#pragma unroll
    for (int i = 0; i < CONN; ++i) {
      const int nv = sI[s + B::off(i)];
      if (nv <= m) { m = nv; dm = i; }  // Eq. 1: max index among the minima
      if (nv == v) eqm |= 1u << i;
    }
    int dir = DIR_NONE, dd = 0;
    bool minimal = (m > v);  // strict single-voxel minimum (or a 1-voxel image, C4)
    if (m < v) {
      dir = dm;                               // steepest descent (S = 0)
    } else if (m == v) {                      // plateau voxel without a lower neighbour
      dd = sD[s];
      if (dd != INF) {                        // non-minimal plateau: BFS parent (C5/C6)
#pragma unroll
        for (int i = 0; i < CONN; ++i)
          if ((eqm & (1u << i)) && sD[s + B::off(i)] == dd - 1) dir = i;
      } else {                                // minimal plateau: state 2 -> q, state 3 -> root
        minimal = true;
        dir = dm >= Conn<CONN>::nfwd ? dm : DIR_NONE;
      }
    }
    const int p = (int)((size_t)(c.bz + lz) * g.plane + (size_t)(c.by + ly) * g.n2 + c.bx + lx);
    if (DEBUG) {
      dist[p] = minimal ? -1 : dd;
      P[p] = (dir == DIR_NONE || minimal) ? p : p + nb_off<CONN>(g, dir);  // oracle: minima are terminals
      continue;
    }
    if (dir == DIR_NONE) {
      sP[j] = (short)j;
    } else {
      int dz, dy, dx;
      nb_delta(CONN, dir, dz, dy, dx);
      const int nx = lx + dx, ny = ly + dy, nz = lz + dz;
      if ((unsigned)nx < (unsigned)T::TX && (unsigned)ny < (unsigned)T::TY && (unsigned)nz < (unsigned)T::TZ) {
        sP[j] = (short)(j + (dz * T::TY + dy) * T::TX + dx);
      } else {
        sP[j] = -1;
        sG[j] = p + nb_off<CONN>(g, dir);
      }
    }
  }
  if (DEBUG) return;
  __syncthreads();
  // tile-local path reduction: follow in-tile pointers to a root or to the tile exit
#pragma unroll
  for (int k = 0; k < T::VPT; ++k) {
    int lx, ly, lz;
    my_voxel<CONN>(k, lx, ly, lz);
    if (sI[B::at(lz, ly, lx)] == OOB) continue;
    int j = threadIdx.x + k * NT;
    int out;
    while (true) {
      const int jn = sP[j];
      if (jn < 0) { out = sG[j]; break; }
      if (jn == j) {
        const int rx = j % T::TX, ry = (j / T::TX) % T::TY, rz = j / (T::TX * T::TY);
        out = (int)((size_t)(c.bz + rz) * g.plane + (size_t)(c.by + ry) * g.n2 + c.bx + rx);
        break;
      }
      j = jn;
    }
    P[(size_t)(c.bz + lz) * g.plane + (size_t)(c.by + ly) * g.n2 + c.bx + lx] = out;
  }
}

// --------------------------- step III across tiles + per-root minimum + root list
// After the chase P[p] = r (a self-loop root).  L[r] accumulates INT_MAX - min{p : P[p] = r}
// with atomicMax: the dead step-II codes left in L are all <= 0 < INT_MAX - p, so no
// initialisation pass is needed.  Each block owns a contiguous chunk of voxels; within a warp
// voxels are consecutive, so the first lane of every run of equal roots holds the run's
// minimum and issues the only atomic for it.  Roots are staged in shared memory and flushed
// to the global list with one atomicAdd per batch.
constexpr int RBUF = 2048;

__global__ void __launch_bounds__(NT) k_jump(int* P, int* __restrict__ L, int N, int chunk, int* roots, int cap,
                                             int* nroots) {
  __shared__ int sbuf[RBUF];
  __shared__ int scount, sbase;
  const int lane = threadIdx.x & 31;
  const int begin = blockIdx.x * chunk;
  const int end = min(N, begin + chunk);
  if (threadIdx.x == 0) scount = 0;
  __syncthreads();
  for (int p0 = begin; p0 < end; p0 += NT) {
    const int p = p0 + threadIdx.x;
    const bool valid = p < end;
    int t = -1 - lane;  // unique per lane when invalid (never equals a neighbour's root)
    if (valid) {
      t = P[p];
      if (t != p) {
        int nt = P[t];
        if (nt != t) {
          do {
            t = nt;
            nt = P[t];
          } while (nt != t);
          P[p] = t;
        }
      }
    }
    const int tprev = __shfl_up_sync(0xffffffffu, t, 1);
    if (valid && (lane == 0 || tprev != t)) atomicMax(L + t, INT_MAX - p);
    const bool isr = valid && t == p;
    const unsigned rb = __ballot_sync(0xffffffffu, isr);
    if (rb) {
      int base = 0;
      if (lane == 0) base = atomicAdd(&scount, __popc(rb));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (isr) sbuf[base + __popc(rb & ((1u << lane) - 1))] = p;
    }
    __syncthreads();
    const int cnt = scount;
    if (cnt > RBUF - NT || p0 + NT >= end) {  // flush the staged roots
      if (threadIdx.x == 0) sbase = atomicAdd(nroots, cnt);
      __syncthreads();
      for (int i = threadIdx.x; i < cnt; i += NT)
        if (sbase + i < cap) roots[sbase + i] = sbuf[i];
      __syncthreads();
      if (threadIdx.x == 0) scount = 0;
      __syncthreads();
    }
  }
}

// rebuild the root list (only if k_jump's list overflowed): roots are P[p] == p
__global__ void k_collect_roots(const int* __restrict__ P, int N, int* roots, int* nroots) {
  for (int p0 = blockIdx.x * NT; p0 < N; p0 += gridDim.x * NT) {
    const int p = p0 + threadIdx.x;
    if (p >= N) break;
    const unsigned act = __activemask();
    const int lane = threadIdx.x & 31;
    const bool isr = P[p] == p;
    const unsigned rb = __ballot_sync(act, isr);
    if (rb) {
      const int leader = __ffs(act) - 1;
      int base = 0;
      if (lane == leader) base = atomicAdd(nroots, __popc(rb));
      base = __shfl_sync(act, base, leader);
      if (isr) roots[base + __popc(rb & ((1u << lane) - 1))] = p;
    }
  }
}

// find with path halving: x -> y -> z becomes x -> z.  Only non-roots are rewritten, and only
// to one of their ancestors, so concurrent finds/unions stay correct.
__device__ __forceinline__ int uf_find(int* P, int x) {
  while (true) {
    const int y = ld_cg(P + x);
    if (y == x) return x;
    const int z = ld_cg(P + y);
    if (z == y) return y;
    __stcg(P + x, z);
    x = z;
  }
}

// min-root lock-free union ("setting the smaller label as the parent")
__device__ __forceinline__ void uf_unite(int* P, int a, int b) {
  while (true) {
    a = uf_find(P, a);
    b = uf_find(P, b);
    if (a == b) return;
    if (a > b) { const int t = a; a = b; b = t; }
    const int old = atomicCAS(P + b, b, a);
    if (old == b) return;
  }
}

#define ZLOOP_BEGIN                                                         \
  const int x = blockIdx.x * blockDim.x + threadIdx.x;                      \
  const int y = blockIdx.y * blockDim.y + threadIdx.y;                      \
  if (x >= g.n2 || y >= g.n1) return;                                       \
  for (int z = blockIdx.z; z < g.n0; z += gridDim.z) {                      \
    const int p = z * g.plane + y * g.n2 + x;
#define ZLOOP_END }

// ------------------------------------------------ step IV Union (Alg. 1 l.24-27, q > p)
// p is on a minimal plateau  <=>  I(root(p)) == I(p): the descent path into a regional
// minimum keeps the intensity only inside that minimum's plateau.
template <int CONN>
__global__ void k_union(const uint8_t* __restrict__ I, int* P, Geo g) {
  ZLOOP_BEGIN
  const int v = I[p];
  const int r = ld_cg(P + p);
  if (I[r] != v) continue;
#pragma unroll
  for (int i = Conn<CONN>::nfwd; i < CONN; ++i) {
    if (!nb_in<CONN>(g, z, y, x, i)) continue;
    const int q = p + nb_off<CONN>(g, i);
    if (I[q] != v) continue;
    if (ld_cg(P + q) == ld_cg(P + p)) continue;  // already in the same set
    uf_unite(P, p, q);
  }
  ZLOOP_END
}

// ------------- step IV Find (l.28-29) on the roots only; canonical labels (C7) per region
// merge: every root folds its minimum into its final root's (atomicMax on INT_MAX - min)
__global__ void k_root_merge(int* P, int* L, const int* __restrict__ roots, int n, unsigned long long* nfinal) {
  for (int i = blockIdx.x * NT + threadIdx.x; i < n; i += gridDim.x * NT) {
    const int r = roots[i];
    const int f = uf_find(P, r);
    if (f != r) atomicMax(L + f, L[r]);
    const unsigned act = __activemask();
    const unsigned b = __ballot_sync(act, f == r);
    if (b && (threadIdx.x & 31) == __ffs(act) - 1) atomicAdd(nfinal, (unsigned long long)__popc(b));
  }
}

// canonical label of every listed root (finds only; no P writes except path halving)
__global__ void k_root_label(int* P, const int* __restrict__ L, const int* __restrict__ roots, int n,
                             int* __restrict__ rootc) {
  for (int i = blockIdx.x * NT + threadIdx.x; i < n; i += gridDim.x * NT)
    rootc[i] = INT_MAX - L[uf_find(P, roots[i])];
}

// P[root] = -1 - canonical label (no finds run any more)
__global__ void k_root_store(int* P, const int* __restrict__ roots, const int* __restrict__ rootc, int n) {
  for (int i = blockIdx.x * NT + threadIdx.x; i < n; i += gridDim.x * NT) P[roots[i]] = -1 - rootc[i];
}

// labels[p] = canonical label of p's step III root
__global__ void __launch_bounds__(NT) k_relabel(const int* __restrict__ P, int* __restrict__ L, int N) {
  for (int p = blockIdx.x * NT + threadIdx.x; p < N; p += gridDim.x * NT) {
    const int t = P[p];
    L[p] = -1 - (t < 0 ? t : __ldg(P + t));
  }
}

// --------------------------------------------------------------------------- drivers
struct TileGrid {
  int ntx, nty, ntz, n;
};

template <int CONN>
static TileGrid tiles_of(const Geo& g) {
  using T = Tile<CONN>;
  TileGrid tg;
  tg.ntx = (g.n2 + T::TX - 1) / T::TX;
  tg.nty = (g.n1 + T::TY - 1) / T::TY;
  tg.ntz = (g.n0 + T::TZ - 1) / T::TZ;
  tg.n = tg.ntx * tg.nty * tg.ntz;
  return tg;
}

static int grid1d(long long n, int sms, int per_sm = 8) {
  long long b = (n + NT - 1) / NT;
  long long cap = (long long)sms * per_sm;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

template <int CONN>
static ws_status plateau_phase(ws_ctx* ctx, const uint8_t* grad, const Geo& g, int32_t* L, const TileGrid& tg,
                               cudaStream_t st) {
  WS_TRY(ctx->flags.ensure(256, "flags"));
  WS_TRY(ctx->tiles.ensure((size_t)tg.n * 3, "tile flags"));
  int* flags = ctx->flags.as<int>();
  uint8_t* cur = ctx->tiles.as<uint8_t>();
  uint8_t* next = cur + tg.n;
  uint8_t* hasplat = next + tg.n;
  WS_CUDA(cudaMemsetAsync(flags, 0, 2 * sizeof(int), st));
  WS_CUDA(cudaMemsetAsync(next, 0, tg.n, st));
  k_relax_first<CONN><<<tg.n, NT, 0, st>>>(grad, L, g, tg.ntx, tg.nty, tg.ntz, next, hasplat, flags);
  launched(ctx, PH_WS_INIT);
  tmark(ctx, st, PH_WS_INIT);
  int rounds = 1;
  while (true) {
    WS_CUDA(cudaMemcpyAsync(ctx->pinned, flags, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
    WS_CUDA(cudaStreamSynchronize(st));
    const int* h = reinterpret_cast<const int*>(ctx->pinned);
    if (h[1]) {
      set_error(WS_ERR_LIMIT, "a non-minimal plateau is deeper than 2^26-2 voxels");
      return WS_ERR_LIMIT;
    }
    if (!h[0]) break;
    if (rounds > g.N + 2) {
      set_error(WS_ERR_INTERNAL, "step II did not converge");
      return WS_ERR_INTERNAL;
    }
    std::swap(cur, next);
    WS_CUDA(cudaMemsetAsync(next, 0, tg.n, st));
    WS_CUDA(cudaMemsetAsync(flags, 0, sizeof(int), st));
    k_relax_round<CONN><<<tg.n, NT, 0, st>>>(grad, L, g, tg.ntx, tg.nty, tg.ntz, cur, next, hasplat, flags);
    launched(ctx, PH_WS_RELAX);
    ++rounds;
  }
  ctx->stats.plateau_rounds = rounds;
  tmark(ctx, st, PH_WS_RELAX);
  WS_CUDA(cudaGetLastError());
  return WS_OK;
}

template <int CONN>
static ws_status watershed_t(ws_ctx* ctx, const uint8_t* grad, const Geo& g, int32_t* L, int64_t* num_regions,
                             cudaStream_t st) {
  const TileGrid tg = tiles_of<CONN>(g);
  WS_TRY(plateau_phase<CONN>(ctx, grad, g, L, tg, st));
  WS_TRY(ctx->aux.ensure((size_t)g.N * sizeof(int), "aux"));
  int* P = ctx->aux.as<int>();
  k_resolve<CONN, false><<<tg.n, NT, 0, st>>>(grad, L, g, tg.ntx, tg.nty, P, nullptr);
  launched(ctx, PH_WS_SELECT);
  tmark(ctx, st, PH_WS_SELECT);

  // step III across tiles + root list
  size_t cap = ctx->roots.bytes / sizeof(int);
  const size_t want = (size_t)g.N / 16 + 1024;
  if (cap < want) {
    WS_TRY(ctx->roots.ensure(want * sizeof(int), "roots"));
    WS_TRY(ctx->rootc.ensure(want * sizeof(int), "root labels"));
    cap = want;
  }
  int* nr = ctx->flags.as<int>() + 8;
  unsigned long long* nfinal = reinterpret_cast<unsigned long long*>(ctx->flags.as<char>() + 64);
  WS_CUDA(cudaMemsetAsync(nr, 0, sizeof(int), st));
  WS_CUDA(cudaMemsetAsync(nfinal, 0, sizeof(unsigned long long), st));
  const int gN = grid1d(g.N, ctx->num_sms);
  const int chunk = (int)((((long long)g.N + gN - 1) / gN + NT - 1) / NT * NT);
  k_jump<<<(g.N + chunk - 1) / chunk, NT, 0, st>>>(P, L, g.N, chunk, ctx->roots.as<int>(), (int)cap, nr);
  launched(ctx, PH_WS_JUMP);
  WS_CUDA(cudaMemcpyAsync(ctx->pinned, nr, sizeof(int), cudaMemcpyDeviceToHost, st));
  WS_CUDA(cudaStreamSynchronize(st));
  const int n_roots = (int)reinterpret_cast<const int*>(ctx->pinned)[0];
  if ((size_t)n_roots > cap) {  // list overflow: grow and rebuild it from P
    WS_TRY(ctx->roots.ensure((size_t)n_roots * sizeof(int), "roots"));
    WS_TRY(ctx->rootc.ensure((size_t)n_roots * sizeof(int), "root labels"));
    WS_CUDA(cudaMemsetAsync(nr, 0, sizeof(int), st));
    k_collect_roots<<<gN, NT, 0, st>>>(P, g.N, ctx->roots.as<int>(), nr);
    launched(ctx, PH_WS_JUMP);
  }
  tmark(ctx, st, PH_WS_JUMP);
  const L3 l = launch3(g);
  k_union<CONN><<<l.grid, l.block, 0, st>>>(grad, P, g);
  launched(ctx, PH_WS_UNION);
  tmark(ctx, st, PH_WS_UNION);
  const int gR = grid1d(n_roots, ctx->num_sms);
  const int* roots = ctx->roots.as<int>();
  k_root_merge<<<gR, NT, 0, st>>>(P, L, roots, n_roots, nfinal);
  k_root_label<<<gR, NT, 0, st>>>(P, L, roots, n_roots, ctx->rootc.as<int>());
  k_root_store<<<gR, NT, 0, st>>>(P, roots, ctx->rootc.as<int>(), n_roots);
  launched(ctx, PH_WS_FIND, 3);
  tmark(ctx, st, PH_WS_FIND);
  k_relabel<<<gN, NT, 0, st>>>(P, L, g.N);
  launched(ctx, PH_WS_RELABEL);
  tmark(ctx, st, PH_WS_RELABEL);
  WS_CUDA(cudaGetLastError());
  WS_CUDA(cudaMemcpyAsync(ctx->pinned, nfinal, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
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
  const TileGrid tg = tiles_of<CONN>(g);
  WS_TRY(plateau_phase<CONN>(ctx, grad, g, L, tg, st));
  k_resolve<CONN, true><<<tg.n, NT, 0, st>>>(grad, L, g, tg.ntx, tg.nty, parent, dist);
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
