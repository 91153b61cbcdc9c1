// ws_watershed.cu — steps I-IV of PRUF (Alg. 1) + canonical relabel, sm_100a.
//
// Tile design: the volume is cut into tiles of 2048 voxels
// (3-D 32x8x8, 2-D 64x32) staged in shared memory with a halo.
//
//   k_relax_first  step I classification (Alg. 1 l.1-10) fused with the first round of the
//                  step II distance relaxation (Alg. 3 l.7-8) inside each tile      [all tiles]
//   k_relax_round  further step II rounds, only on tiles whose halo changed       [active tiles]
//   k_resolve      step I/II pointers (Eq. 1; C5/C6 selection) + tile-local pointer
//                  jumping in shared memory (step III inside the tile)  -> P = aux  [all tiles]
//   k_jump         step III across tiles: chase exits to the self-loop roots (l.19-23/28-29)
//   k_union        step IV Union over q > p (l.24-27), lock-free min-root CAS
//   k_find         step IV Find (l.28-29) + warp-aggregated canonical atomicMin (C7)
//   k_relabel      labels = canonical minimum of the root
//
// Arrays: L = the caller's `labels` (i32[N]); during step II it holds the plateau distance
// code of ws_common.cuh (L >= 0: d = 0; L < 0: -1 - (d << 5)).  P = ctx->aux (i32[N]) holds
// pointers from k_resolve on.  After k_jump, L[r] of every root r is reused as the canonical
// minimum of r's region, and finally L[p] = L[P[p]].
#include "ws_internal.h"

namespace ws {

constexpr int NT = 256;
constexpr int INF = DUNREACHED;

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

// voxel k of this thread inside the tile
template <int CONN>
__device__ __forceinline__ void my_voxel(int k, int& lx, int& ly, int& lz) {
  using T = Tile<CONN>;
  const int j = threadIdx.x + k * NT;
  lx = j % T::TX;
  ly = (j / T::TX) % T::TY;
  lz = j / (T::TX * T::TY);
}

template <int CONN, int H>
__device__ __forceinline__ void load_I(const uint8_t* __restrict__ I, const Geo& g, const TileCoord& c, uint8_t* sI) {
  using B = Box<CONN, H>;
  for (int s = threadIdx.x; s < B::S; s += NT) {
    const int sx = s % B::SX, sy = (s / B::SX) % B::SY, sz = s / (B::SX * B::SY);
    const int gx = c.bx + sx - H, gy = c.by + sy - H, gz = c.bz + sz - B::HZ;
    uint8_t v = 0;
    if ((unsigned)gx < (unsigned)g.n2 && (unsigned)gy < (unsigned)g.n1 && (unsigned)gz < (unsigned)g.n0)
      v = __ldg(I + (size_t)gz * g.plane + (size_t)gy * g.n2 + gx);
    sI[s] = v;
  }
}

// distances of the tile + 1-voxel halo from the L code (out of the volume: INF, never read)
template <int CONN>
__device__ __forceinline__ void load_D(const int* L, const Geo& g, const TileCoord& c, int* sD) {
  using B = Box<CONN, 1>;
  for (int s = threadIdx.x; s < B::S; s += NT) {
    const int sx = s % B::SX, sy = (s / B::SX) % B::SY, sz = s / (B::SX * B::SY);
    const int gx = c.bx + sx - 1, gy = c.by + sy - 1, gz = c.bz + sz - B::HZ;
    int d = INF;
    if ((unsigned)gx < (unsigned)g.n2 && (unsigned)gy < (unsigned)g.n1 && (unsigned)gz < (unsigned)g.n0)
      d = dec_d(L[(size_t)gz * g.plane + (size_t)gy * g.n2 + gx]);
    sD[s] = d;
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

// one in-tile relaxation sweep loop until the tile converges (chaotic, in place)
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
      int best = sD[s];
#pragma unroll
      for (int i = 0; i < CONN; ++i)
        if (m & (1u << i)) {
          const int dq = sD[s + B::off(i)] + 1;
          best = dq < best ? dq : best;
        }
      if (best < sD[s]) {
        sD[s] = best;
        ch = true;
        if (best >= INF - 1) *limit = 1;
      }
    }
    if (!__syncthreads_or(ch)) break;
  }
}

// ------------------------------------------- step I + first step II round (all tiles)
template <int CONN>
__global__ void __launch_bounds__(NT) k_relax_first(const uint8_t* __restrict__ I, int* __restrict__ L, Geo g,
                                                     int ntx, int nty, int ntz, uint8_t* next,
                                                     uint8_t* hasplat, int* flags) {
  using T = Tile<CONN>;
  using B2 = Box<CONN, 2>;
  __shared__ uint8_t sI[B2::S];
  __shared__ int sD[B2::S];
  const int t = blockIdx.x;
  const TileCoord c = tile_coord<CONN>(t, ntx, nty);
  load_I<CONN, 2>(I, g, c, sI);
  __syncthreads();
  // classify the tile + 1-voxel halo: lower -> 0, plateau without lower -> INF (Alg. 1 l.3-10)
  {
    using B1 = Box<CONN, 1>;
    for (int s = threadIdx.x; s < B1::S; s += NT) {
      const int sx = s % B1::SX, sy = (s / B1::SX) % B1::SY, sz = s / (B1::SX * B1::SY);
      const int lx = sx - 1, ly = sy - 1, lz = sz - B1::HZ;
      const int gx = c.bx + lx, gy = c.by + ly, gz = c.bz + lz;
      const int s2 = B2::at(lz, ly, lx);
      if (!((unsigned)gx < (unsigned)g.n2 && (unsigned)gy < (unsigned)g.n1 && (unsigned)gz < (unsigned)g.n0)) {
        sD[s2] = INF;
        continue;
      }
      const int v = sI[s2];
      bool lower = false, eq = false;
#pragma unroll
      for (int i = 0; i < CONN; ++i) {
        if (!nb_in<CONN>(g, gz, gy, gx, i)) continue;
        const int nv = sI[s2 + B2::off(i)];
        lower |= nv < v;
        eq |= nv == v;
      }
      sD[s2] = lower ? 0 : (eq ? INF : 0);
    }
  }
  __syncthreads();
  int my[T::VPT];
  unsigned eqm[T::VPT];
  bool any_plat = false;
#pragma unroll
  for (int k = 0; k < T::VPT; ++k) {
    int lx, ly, lz;
    my_voxel<CONN>(k, lx, ly, lz);
    const int gx = c.bx + lx, gy = c.by + ly, gz = c.bz + lz;
    my[k] = B2::at(lz, ly, lx);
    eqm[k] = 0;
    if (gx < g.n2 && gy < g.n1 && gz < g.n0 && sD[my[k]] == INF) {
      const int v = sI[my[k]];
      unsigned m = 0;
#pragma unroll
      for (int i = 0; i < CONN; ++i)
        if (nb_in<CONN>(g, gz, gy, gx, i) && sI[my[k] + B2::off(i)] == v) m |= 1u << i;
      eqm[k] = m;
      any_plat = true;
    }
  }
  relax_tile<CONN, 2>(sD, my, eqm, flags + 1);
  bool border = false;
#pragma unroll
  for (int k = 0; k < T::VPT; ++k) {
    int lx, ly, lz;
    my_voxel<CONN>(k, lx, ly, lz);
    const int gx = c.bx + lx, gy = c.by + ly, gz = c.bz + lz;
    if (!(gx < g.n2 && gy < g.n1 && gz < g.n0)) continue;
    const int d = sD[my[k]];
    L[(size_t)gz * g.plane + (size_t)gy * g.n2 + gx] = eqm[k] ? enc(d, DIR_NONE) : 0;
    if (eqm[k] && d != INF &&
        (lx == 0 || lx == T::TX - 1 || ly == 0 || ly == T::TY - 1 || (T::is3d && (lz == 0 || lz == T::TZ - 1))))
      border = true;
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
  __shared__ uint8_t sI[B::S];
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
    const int gx = c.bx + lx, gy = c.by + ly, gz = c.bz + lz;
    my[k] = B::at(lz, ly, lx);
    eqm[k] = 0;
    d0[k] = 0;
    if (gx < g.n2 && gy < g.n1 && gz < g.n0 && sD[my[k]] > 0) {  // plateau voxel (d >= 1)
      d0[k] = sD[my[k]];
      const int v = sI[my[k]];
      unsigned m = 0;
#pragma unroll
      for (int i = 0; i < CONN; ++i)
        if (nb_in<CONN>(g, gz, gy, gx, i) && sI[my[k] + B::off(i)] == v) m |= 1u << i;
      eqm[k] = m;
    }
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
    if (lx == 0 || lx == T::TX - 1 || ly == 0 || ly == T::TY - 1 || (T::is3d && (lz == 0 || lz == T::TZ - 1)))
      border = true;
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
  __shared__ uint8_t sI[B::S];
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
    const int gx = c.bx + lx, gy = c.by + ly, gz = c.bz + lz;
    if (!(gx < g.n2 && gy < g.n1 && gz < g.n0)) {
      sP[j] = (short)j;
      continue;
    }
    const int s = B::at(lz, ly, lx);
    const int v = sI[s];
    int m = 256, dm = -1;
    unsigned eqm = 0;
#pragma unroll
    for (int i = 0; i < CONN; ++i) {
      if (!nb_in<CONN>(g, gz, gy, gx, i)) continue;
      const int nv = sI[s + B::off(i)];
      if (nv <= m) { m = nv; dm = i; }  // Eq. 1: max index among the minima
      if (nv == v) eqm |= 1u << i;
    }
    int dir = DIR_NONE, dd = 0;
    if (dm >= 0 && m < v) {
      dir = dm;                               // steepest descent (S = 0)
    } else if (dm >= 0 && m == v) {           // plateau voxel without a lower neighbour
      dd = sD[s];
      if (dd != INF) {                        // non-minimal plateau: BFS parent (C5/C6)
#pragma unroll
        for (int i = 0; i < CONN; ++i)
          if ((eqm & (1u << i)) && sD[s + B::off(i)] == dd - 1) dir = i;
      } else {                                // minimal plateau: state 2 -> q, state 3 -> root
        dir = dm >= Conn<CONN>::nfwd ? dm : DIR_NONE;
      }
    }
    const int p = (int)((size_t)gz * g.plane + (size_t)gy * g.n2 + gx);
    if (DEBUG) {
      const bool term = (dir == DIR_NONE);
      const bool minimal = (dm < 0 || m > v || (m == v && dd == INF));
      dist[p] = minimal ? -1 : dd;
      P[p] = (term || minimal) ? p : p + nb_off<CONN>(g, dir);  // oracle: minimal plateaux are terminals
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
    const int gx = c.bx + lx, gy = c.by + ly, gz = c.bz + lz;
    if (!(gx < g.n2 && gy < g.n1 && gz < g.n0)) continue;
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
    P[(size_t)gz * g.plane + (size_t)gy * g.n2 + gx] = out;
  }
}

// ------------------------------------ step III across tiles: chase to the self-loop
__global__ void k_jump(int* P, int* __restrict__ L, int N) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < N; p += gridDim.x * blockDim.x) {
    int t = P[p];
    if (t == p) {
      L[p] = p;  // root: seed its canonical minimum
      continue;
    }
    int nt = P[t];
    if (nt == t) continue;
    while (true) {
      t = nt;
      nt = P[t];
      if (nt == t) break;
    }
    P[p] = t;
  }
}

__device__ __forceinline__ int uf_find(int* P, int x) {
  while (true) {
    const int y = ld_cg(P + x);
    if (y == x) return x;
    x = y;
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

// ------------------------------- step IV Find (l.28-29) + canonical minimum per root (C7)
__global__ void k_find(int* P, int* __restrict__ L, int N) {
  for (int p0 = blockIdx.x * blockDim.x; p0 < N; p0 += gridDim.x * blockDim.x) {
    const int p = p0 + threadIdx.x;
    if (p >= N) break;
    const int r = uf_find(P, ld_cg(P + p));
    P[p] = r;
    // warp-aggregated atomicMin: lanes sharing a root elect one leader
    const unsigned act = __activemask();
    const unsigned grp = __match_any_sync(act, r);
    const int mn = (int)__reduce_min_sync(grp, (unsigned)p);
    if (mn < r && (__ffs(grp) - 1) == (int)(threadIdx.x & 31)) atomicMin(L + r, mn);
  }
}

__global__ void k_relabel(const int* __restrict__ P, int* L, int N, unsigned long long* nroots) {
  for (int p0 = blockIdx.x * blockDim.x; p0 < N; p0 += gridDim.x * blockDim.x) {
    const int p = p0 + threadIdx.x;
    if (p >= N) break;
    const int c = L[P[p]];  // roots keep L[r] = canonical minimum; other entries are free
    L[p] = c;
    const unsigned act = __activemask();
    const unsigned b = __ballot_sync(act, c == p);
    if (b && (__ffs(act) - 1) == (int)(threadIdx.x & 31)) atomicAdd(nroots, (unsigned long long)__popc(b));
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

static int grid1d(long long n, int sms, int per_sm = 16) {
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
  const int gN = grid1d(g.N, ctx->num_sms);
  k_jump<<<gN, NT, 0, st>>>(P, L, g.N);
  launched(ctx, PH_WS_JUMP);
  tmark(ctx, st, PH_WS_JUMP);
  const L3 l = launch3(g);
  k_union<CONN><<<l.grid, l.block, 0, st>>>(grad, P, g);
  launched(ctx, PH_WS_UNION);
  tmark(ctx, st, PH_WS_UNION);
  k_find<<<gN, NT, 0, st>>>(P, L, g.N);
  launched(ctx, PH_WS_FIND);
  tmark(ctx, st, PH_WS_FIND);
  unsigned long long* nroots = reinterpret_cast<unsigned long long*>(ctx->flags.as<char>() + 64);
  WS_CUDA(cudaMemsetAsync(nroots, 0, sizeof(unsigned long long), st));
  k_relabel<<<gN, NT, 0, st>>>(P, L, g.N, nroots);
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
