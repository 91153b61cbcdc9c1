// ws_watershed.cu — steps I-IV of PRUF (Alg. 1) + canonical relabel, sm_100a.
//
// Tile design: the volume is cut into tiles of 2048 voxels
// (3-D 32x8x8, 2-D 64x32) staged in shared memory with a halo by TMA (zero fill outside the
// volume); tiles whose halo leaves the volume use neighbour-validity masks (BORDER bodies).
// Pixel type Px: u8 here; ws_watershed16.cu compiles this file again with u16 pixels
// (NEXT f4) into namespace ws::px16.
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
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>

#include "ws_internal.h"
#include <cooperative_groups.h>

#include "ws_tile.cuh"

namespace ws {
#ifdef WS_PX16
namespace px16 {
using Px = uint16_t;
#else
using Px = uint8_t;
#endif

constexpr int INF = DUNREACHED;

// decode the staged L box in place into plateau distances (L >= 0: 0; else d)
template <int CONN>
__device__ __forceinline__ void decode_box(int* sD) {
  using T = TL<CONN>;
  for (int s = threadIdx.x; s < T::SL; s += NT) sD[s] = dec_d(sD[s]);
  __syncthreads();
}

template <int CONN>
__device__ __forceinline__ bool on_tile_border(int lx, int ly, int lz) {
  using T = TL<CONN>;
  return lx == 0 || lx == T::TX - 1 || ly == 0 || ly == T::TY - 1 || (T::is3d && (lz == 0 || lz == T::TZ - 1));
}

// Activate a neighbouring tile only where it can gain: a border voxel with distance d whose
// equal-intensity neighbour h across the tile border still holds sD[h] > d + 1 (the value
// loaded at kernel start; distances only decrease, so a stale value never hides a gain).
template <int CONN>
__device__ __forceinline__ bool mark_gains(const int* sD, int s, int d, unsigned m, int lx, int ly, int lz, int t,
                                           int ntx, int nty, uint8_t* next, const Geo& g, const TileCoord& c) {
  using T = TL<CONN>;
  bool any = false;
#pragma unroll
  for (int i = 0; i < CONN; ++i) {
    if (!(m & (1u << i))) continue;
    int dz, dy, dx;
    nb_delta(CONN, i, dz, dy, dx);
    const int ox = (lx + dx < 0) ? -1 : (lx + dx >= T::TX ? 1 : 0);
    const int oy = (ly + dy < 0) ? -1 : (ly + dy >= T::TY ? 1 : 0);
    const int oz = (lz + dz < 0) ? -1 : (lz + dz >= T::TZ ? 1 : 0);
    if ((ox | oy | oz) == 0) continue;
    if (oz != 0) {  // no tile beyond the owned planes (slab halo)
      const int zz = c.bz - g.zlo + oz * T::TZ;
      if (zz < 0 || zz >= g.zhi - g.zlo) continue;
    }
    if (sD[s + T::oL(i)] > d + 1) {
      next[t + (oz * nty + oy) * ntx + ox] = 1;
      any = true;
    }
  }
  return any;
}

// L-box index of this thread's voxel k: s0 + k * KS (voxel k = threadIdx.x + k * NT)
template <int CONN> struct Mine {
  using T = TL<CONN>;
  static constexpr int KS = (T::is3d ? T::SYL * T::SXL : (NT / T::TX) * T::SXL);
  __device__ static int s0() {
    int lx, ly, lz;
    my_voxel<CONN>(0, lx, ly, lz);
    return T::iL(lz, ly, lx);
  }
};

// in-tile relaxation sweeps until the tile converges (chaotic, in place, on sD); returns a
// bitmask of this thread's voxels whose distance decreased
template <int CONN>
__device__ __forceinline__ unsigned relax_tile(int* sD, int s0, const unsigned* eqm, int* limit) {
  using T = TL<CONN>;
  unsigned changed = 0;
  while (true) {
    bool ch = false;
#pragma unroll
    for (int k = 0; k < T::VPT; ++k) {
      const unsigned m = eqm[k];
      if (!m) continue;
      const int s = s0 + k * Mine<CONN>::KS;
      const int cur = sD[s];
      int best = cur;
#pragma unroll
      for (int i = 0; i < CONN; ++i)
        if (m & (1u << i)) best = min(best, sD[s + T::oL(i)] + 1);
      if (best < cur) {
        sD[s] = best;
        ch = true;
        changed |= 1u << k;
        if (best >= INF - 1) *limit = 1;
      }
    }
    if (!__syncthreads_or(ch)) break;
  }
  return changed;
}

// The same relaxation over a compact list of the tile's plateau voxels (typically a few
// percent of the tile): each sweep costs the list length, not 8 checks per thread.  Tiles
// with more than RQCAP plateau voxels use relax_tile.  q.n / q.chg are zeroed by the kernel
// before a __syncthreads.  Returns what relax_tile returns when CHG, else 0.
constexpr int RQCAP = 256;  // measured on C4: 256 > 512 > 1024 (smem -> 8 CTAs per SM)
struct RQ {
  uint2 q[RQCAP];  // x = eqm, y = L-box index | tile voxel index << 16
  unsigned chg[2048 / 32];
  int n;
};
__device__ __forceinline__ void rq_zero(RQ& q) {
  if (threadIdx.x < 2048 / 32) q.chg[threadIdx.x] = 0;
  if (threadIdx.x == 0) q.n = 0;
}

template <int CONN, bool CHG>
__device__ __forceinline__ unsigned relax_tile_q(int* sD, int s0, const unsigned* eqm, int* limit, RQ& q) {
  using T = TL<CONN>;
  unsigned mine = 0;
#pragma unroll
  for (int k = 0; k < T::VPT; ++k)
    if (eqm[k]) mine |= 1u << k;
  const int cnt = __popc(mine), lane = threadIdx.x & 31;
  int inc = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  const int tot = __shfl_sync(0xffffffffu, inc, 31);
  int base = 0;
  if (lane == 31 && tot) base = atomicAdd(&q.n, tot);
  base = __shfl_sync(0xffffffffu, base, 31) + inc - cnt;
#pragma unroll
  for (int k = 0; k < T::VPT; ++k)
    if (mine & (1u << k)) {
      if (base < RQCAP)
        q.q[base] = make_uint2(eqm[k], (unsigned)(s0 + k * Mine<CONN>::KS) | ((unsigned)(threadIdx.x + k * NT) << 16));
      ++base;
    }
  __syncthreads();
  const int n = q.n;
  if (n > RQCAP) return relax_tile<CONN>(sD, s0, eqm, limit);  // uniform over the block
  if (n == 0) return 0;
  unsigned chr = 0;  // bit r: list entry threadIdx.x + r * NT decreased
  while (true) {
    bool ch = false;
#pragma unroll
    for (int r = 0; r < RQCAP / NT; ++r) {
      const int i = threadIdx.x + r * NT;
      if (i >= n) break;
      const uint2 e = q.q[i];
      const int s = e.y & 0xffff;
      const int cur = sD[s];
      int best = cur;
#pragma unroll
      for (int d = 0; d < CONN; ++d)
        if (e.x & (1u << d)) best = min(best, sD[s + T::oL(d)] + 1);
      if (best < cur) {
        sD[s] = best;
        ch = true;
        chr |= 1u << r;
        if (best >= INF - 1) *limit = 1;
      }
    }
    if (!__syncthreads_or(ch)) break;
  }
  if constexpr (!CHG) {
    return 0;
  } else {
    for (; chr; chr &= chr - 1) {
      const int j = q.q[threadIdx.x + (__ffs(chr) - 1) * NT].y >> 16;
      atomicOr(&q.chg[j >> 5], 1u << (j & 31));
    }
    __syncthreads();
    unsigned changed = 0;
#pragma unroll
    for (int k = 0; k < T::VPT; ++k) {
      const int j = threadIdx.x + k * NT;
      if (q.chg[j >> 5] & (1u << (j & 31))) changed |= 1u << k;
    }
    return changed;
  }
}

// write back the changed voxels of this thread and activate neighbouring tiles that gain
template <int CONN>
__device__ __forceinline__ bool write_back(const int* sD, int s0, const unsigned* eqm, unsigned todo, int* L,
                                           const Geo& g, const TileCoord& c, int t, int ntx, int nty,
                                           uint8_t* next) {
  bool marked = false;
#pragma unroll 1
  for (; todo; todo &= todo - 1) {
    const int k = __ffs(todo) - 1;
    int lx, ly, lz;
    my_voxel<CONN>(k, lx, ly, lz);
    const int s = s0 + k * Mine<CONN>::KS;
    const int d = sD[s];
    L[(size_t)(c.bz + lz) * g.plane + (size_t)(c.by + ly) * g.n2 + c.bx + lx] = enc(d, DIR_NONE);
    if (d != INF && on_tile_border<CONN>(lx, ly, lz)) {
      unsigned m = 0;
#pragma unroll
      for (int kk = 0; kk < TL<CONN>::VPT; ++kk)
        if (kk == k) m = eqm[kk];
      marked |= mark_gains<CONN>(sD, s, d, m, lx, ly, lz, t, ntx, nty, next, g, c);
    }
  }
  return marked;
}

// SWAR variant for interior tiles: 4 voxels per 32-bit word of the I box; x-1 / x+1
// neighbours by byte permutation of adjacent words, byte-wise compares (vcmpltu4/vcmpeq4).
template <int CONN>
__device__ __forceinline__ void classify_box_swar(const uint8_t* sI, int* sD) {
  using T = TL<CONN>;
  constexpr int WPR = (T::TX + 8) / 4;                 // words per row: x in [-4, TX+4)
  constexpr int ROWS = (T::TY + 2) * (T::is3d ? T::TZ + 2 : 1);
  for (int job = threadIdx.x; job < ROWS * WPR; job += NT) {
    const int w = job % WPR, r = job / WPR;
    const int ly = r % (T::TY + 2) - 1, lz = T::is3d ? r / (T::TY + 2) - 1 : 0;
    const int x0 = 4 * w - 4;
    const int wb = T::iI(lz, ly, x0);                  // 4-byte aligned (IXO and SXI are multiples of 16)
    const uint32_t C = *reinterpret_cast<const uint32_t*>(sI + wb);
    uint32_t lower = 0, eq = 0;
#pragma unroll
    for (int i = 0; i < CONN; ++i) {
      int dz = 0, dy = 0, dx = 0;
      nb_delta(CONN, i, dz, dy, dx);
      const int ro = wb + (dz * T::SYI + dy) * T::SXI;
      uint32_t nb;
      if (dx == 0) nb = *reinterpret_cast<const uint32_t*>(sI + ro);
      else if (dx < 0)
        nb = __byte_perm(*reinterpret_cast<const uint32_t*>(sI + ro - 4), *reinterpret_cast<const uint32_t*>(sI + ro),
                         0x6543);
      else
        nb = __byte_perm(*reinterpret_cast<const uint32_t*>(sI + ro), *reinterpret_cast<const uint32_t*>(sI + ro + 4),
                         0x4321);
      lower |= __vcmpltu4(nb, C);
      eq |= __vcmpeq4(nb, C);
    }
    const uint32_t plat = eq & ~lower;  // 0xff bytes: plateau voxel without a lower neighbour
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int x = x0 + u;
      if (x < -1 || x > T::TX) continue;
      sD[T::iL(lz, ly, x)] = ((plat >> (8 * u)) & 0xff) ? INF : 0;
    }
  }
}

// step I classification of the tile + 1-voxel halo into sD (L layout):
// lower -> 0, plateau without lower -> INF, strict minimum -> 0 (Alg. 1 l.1-10)
template <int CONN, bool BORDER>
__device__ __forceinline__ void classify_box(const Px* sI, int* sD, const Geo& g, const TileCoord& c) {
  if constexpr (!BORDER && sizeof(Px) == 1) {
    classify_box_swar<CONN>(sI, sD);
    return;
  } else {
  using T = TL<CONN>;
  for (int s = threadIdx.x; s < T::SL; s += NT) {
    const int sx = s % T::SXL, sy = (s / T::SXL) % T::SYL, sz = s / (T::SXL * T::SYL);
    const int lx = sx - T::LXO, ly = sy - T::LYO, lz = sz - T::LZO;
    if (lx < -1 || lx > T::TX) continue;  // alignment padding of the L box
    unsigned vm = (1u << CONN) - 1;
    if (BORDER) {
      const int gx = c.bx + lx, gy = c.by + ly, gz = c.bz + lz;
      if (!((unsigned)gx < (unsigned)g.n2 && (unsigned)gy < (unsigned)g.n1 && (unsigned)gz < (unsigned)g.n0)) {
        sD[s] = INF;
        continue;
      }
      vm = valid_mask<CONN>(g, gz, gy, gx);
    }
    const int si = T::iI(lz, ly, lx);
    const int v = sI[si];
    bool lower = false, eq = false;
#pragma unroll
    for (int i = 0; i < CONN; ++i) {
      if (BORDER && !(vm & (1u << i))) continue;
      const int nv = sI[si + T::oI(i)];
      lower |= nv < v;
      eq |= nv == v;
    }
    sD[s] = lower ? 0 : (eq ? INF : 0);
  }
  }
}

// ------------------------------------------- step I + first step II round (all tiles)
constexpr int EQB = NT * 8;  // equal-mask cache bytes per tile: one 8-byte word per thread (VPT <= 8)

template <int CONN, bool BORDER>
__device__ __forceinline__ void relax_first_body(const Px* sI, int* sD, int* __restrict__ L, const Geo& g,
                                                 const TileCoord& c, int t, int ntx, int nty, uint8_t* next,
                                                 uint8_t* hasplat, int* flags, RQ& q, uint8_t* eqc) {
  using T = TL<CONN>;
  classify_box<CONN, BORDER>(sI, sD, g, c);
  __syncthreads();
  const int s0 = Mine<CONN>::s0();
  unsigned eqm[T::VPT];
  unsigned plat = 0;
#pragma unroll
  for (int k = 0; k < T::VPT; ++k) {
    int lx, ly, lz;
    my_voxel<CONN>(k, lx, ly, lz);
    unsigned m = 0;
    const bool inside = !BORDER || (c.bx + lx < g.n2 && c.by + ly < g.n1 && c.bz + lz < g.zhi);
    if (inside && sD[s0 + k * Mine<CONN>::KS] == INF) {
      const unsigned vm = BORDER ? valid_mask<CONN>(g, c.bz + lz, c.by + ly, c.bx + lx) : (1u << CONN) - 1;
      const int si = T::iI(lz, ly, lx);
      const int v = sI[si];
#pragma unroll
      for (int i = 0; i < CONN; ++i)
        if ((vm & (1u << i)) && sI[si + T::oI(i)] == v) m |= 1u << i;
      plat |= 1u << k;
    }
    eqm[k] = m;
  }
  if constexpr (CONN <= 8) {
    // the equal-neighbour masks of this thread's 8 voxels (one byte each) for the later step II
    // rounds, which then stage only the L box (tile-major, thread-major inside the tile)
    static_assert(T::VPT <= 8, "one 8-byte cache word per thread");
    if (eqc) {
      uint2 w = make_uint2(0u, 0u);
#pragma unroll
      for (int k = 0; k < T::VPT; ++k) {
        if (k < 4) w.x |= eqm[k] << (8 * k);
        else w.y |= eqm[k] << (8 * (k - 4));
      }
      reinterpret_cast<uint2*>(eqc + (size_t)t * EQB)[threadIdx.x] = w;
    }
  }
  relax_tile_q<CONN, false>(sD, s0, eqm, flags + 1, q);
  // every voxel is written once: 0 (d = 0) or the plateau code
#pragma unroll
  for (int k = 0; k < T::VPT; ++k) {
    if (plat & (1u << k)) continue;
    int lx, ly, lz;
    my_voxel<CONN>(k, lx, ly, lz);
    if (BORDER && !(c.bx + lx < g.n2 && c.by + ly < g.n1 && c.bz + lz < g.zhi)) continue;
    L[(size_t)(c.bz + lz) * g.plane + (size_t)(c.by + ly) * g.n2 + c.bx + lx] = 0;
  }
  const bool marked = write_back<CONN>(sD, s0, eqm, plat, L, g, c, t, ntx, nty, next);
  // no block barriers: one idempotent store per warp (hasplat is zeroed by the host)
  const bool lane0 = (threadIdx.x & 31) == 0;
  if (__any_sync(0xffffffffu, plat != 0) && lane0) hasplat[t] = 1;
  if (__any_sync(0xffffffffu, marked) && lane0) flags[0] = 1;
}

template <int CONN>
__global__ void __launch_bounds__(NT) k_relax_first(const __grid_constant__ CUtensorMap mI, int tma,
                                                     const Px* __restrict__ I, int* __restrict__ L, Geo g,
                                                     int ntx, int nty, uint8_t* next, uint8_t* hasplat, int* flags,
                                                     uint8_t* eqc) {
  using T = TL<CONN>;
  __shared__ alignas(128) Px sI[T::SI];
  __shared__ alignas(16) int sD[T::SL];
  __shared__ uint64_t bar;
  __shared__ RQ q;
  int t;
  const TileCoord c = tile_of_block<CONN>(ntx, nty, g, t);
  rq_zero(q);
  stage<CONN>(&mI, nullptr, tma, I, nullptr, g, c, sI, nullptr, &bar);
  if (tile_interior<CONN>(c, g))
    relax_first_body<CONN, false>(sI, sD, L, g, c, t, ntx, nty, next, hasplat, flags, q, eqc);
  else
    relax_first_body<CONN, true>(sI, sD, L, g, c, t, ntx, nty, next, hasplat, flags, q, eqc);
}

// ------------------------------------------------ further step II rounds (active tiles)
template <int CONN, bool BORDER, bool EQC = false>
__device__ __forceinline__ void relax_round_body(const Px* sI, int* sD, int* __restrict__ L, const Geo& g,
                                                 const TileCoord& c, int t, int ntx, int nty, uint8_t* next,
                                                 int* changed_flag, int* limit_flag, RQ& q,
                                                 const uint8_t* eqc = nullptr) {
  using T = TL<CONN>;
  const int s0 = Mine<CONN>::s0();
  unsigned eqm[T::VPT];
  if constexpr (EQC) {  // the masks k_relax_first cached (plateau voxels; 0 elsewhere)
    const uint2 w = reinterpret_cast<const uint2*>(eqc + (size_t)t * EQB)[threadIdx.x];
#pragma unroll
    for (int k = 0; k < T::VPT; ++k) eqm[k] = ((k < 4 ? w.x : w.y) >> (8 * (k & 3))) & 0xffu;
  } else {
#pragma unroll
  for (int k = 0; k < T::VPT; ++k) {
    int lx, ly, lz;
    my_voxel<CONN>(k, lx, ly, lz);
    unsigned m = 0;
    const bool inside = !BORDER || (c.bx + lx < g.n2 && c.by + ly < g.n1 && c.bz + lz < g.zhi);
    if (inside && sD[s0 + k * Mine<CONN>::KS] > 0) {  // plateau voxel (d >= 1)
      const unsigned vm = BORDER ? valid_mask<CONN>(g, c.bz + lz, c.by + ly, c.bx + lx) : (1u << CONN) - 1;
      const int si = T::iI(lz, ly, lx);
      const int v = sI[si];
#pragma unroll
      for (int i = 0; i < CONN; ++i)
        if ((vm & (1u << i)) && sI[si + T::oI(i)] == v) m |= 1u << i;
    }
    eqm[k] = m;
  }
  }
  const unsigned changed = relax_tile_q<CONN, true>(sD, s0, eqm, limit_flag, q);
  const bool marked = write_back<CONN>(sD, s0, eqm, changed, L, g, c, t, ntx, nty, next);
  if (__any_sync(0xffffffffu, marked) && (threadIdx.x & 31) == 0) *changed_flag = 1;  // idempotent, no barrier
}

// EQC: the equal-neighbour masks come from k_relax_first's cache, so only the L box is staged
// (no I box: 9 KB less shared memory and 25 -> 16 KB of box traffic per active tile)
template <int CONN, bool EQC = false>
__global__ void __launch_bounds__(NT) k_relax_round(const __grid_constant__ CUtensorMap mI,
                                                     const __grid_constant__ CUtensorMap mL, int tma,
                                                     const Px* __restrict__ I, int* __restrict__ L, Geo g,
                                                     int ntx, int nty, const uint8_t* cur, uint8_t* next,
                                                     const uint8_t* hasplat, int* flags, const int* list,
                                                     const uint8_t* eqc = nullptr) {
  using T = TL<CONN>;
  const int t = list ? list[blockIdx.x] : blockIdx.x;  // list: the compacted active tiles
  if (!list && (!cur[t] || !hasplat[t])) return;
  __shared__ alignas(128) Px sI[EQC ? 16 : T::SI];
  __shared__ alignas(128) int sD[T::SL];
  __shared__ uint64_t bar;
  __shared__ RQ q;
  const TileCoord c = tile_coord<CONN>(t, ntx, nty, g);
  rq_zero(q);
  stage<CONN>(&mI, &mL, tma, I, L, g, c, EQC ? nullptr : sI, sD, &bar);
  decode_box<CONN>(sD);
  if (tile_interior<CONN>(c, g))
    relax_round_body<CONN, false, EQC>(sI, sD, L, g, c, t, ntx, nty, next, flags, flags + 1, q, eqc);
  else
    relax_round_body<CONN, true, EQC>(sI, sD, L, g, c, t, ntx, nty, next, flags, flags + 1, q, eqc);
}

// All further step II rounds in ONE cooperative launch (no host round trip per round, P:363
// names the per-iteration host loop as the cost).  A grid of co-resident CTAs walks the
// round's active tile list (the k_relax_round body per tile, boxes staged with TMA on one
// mbarrier whose phase flips per tile); grid barrier; the tiles marked for the next round
// (and holding plateau voxels) are compacted into the other list while next[] is cleared;
// grid barrier; every CTA reads the same counts and stops together when no tile changed a
// neighbour or none is active.  Loop state ls (device ints): ls[r & 1] = "a tile marked a
// neighbour in round r", ls[2 + (r & 1)] = length of round r's list, ls[4] = rounds run (0 if
// flags[0] says the previous round changed nothing).  A
// round's slots are reset in the compaction phase of the round before it uses them, when no
// CTA reads or writes them.
template <int CONN, bool EQC = false>
__global__ void __launch_bounds__(NT, 8) k_relax_loop(const __grid_constant__ CUtensorMap mI,
                                                    const __grid_constant__ CUtensorMap mL, int tma,
                                                    const Px* __restrict__ I, int* __restrict__ L, Geo g, int ntx,
                                                    int nty, int ntiles, uint8_t* next, const uint8_t* hasplat,
                                                    int* flags, int* ls, int* list0, int* list1, int max_rounds,
                                                    const uint8_t* eqc) {
  using T = TL<CONN>;
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ alignas(128) Px sI[EQC ? 16 : T::SI];
  __shared__ alignas(128) int sD[T::SL];
  __shared__ uint64_t bar;
  __shared__ RQ q;
  volatile int* vls = ls;
  if (!flags[0] || vls[2] == 0) return;  // the previous round changed no neighbour / no active tile
  if (tma && threadIdx.x == 0) mbar_init(&bar, 1);
  __syncthreads();
  uint32_t phase = 0;
  int r = 0;
  for (;; ++r) {
    const int nact = vls[2 + (r & 1)];
    const int* cl = (r & 1) ? list1 : list0;
    int* nl = (r & 1) ? list0 : list1;
    for (int i = blockIdx.x; i < nact; i += gridDim.x) {
      const int t = cl[i];
      const TileCoord c = tile_coord<CONN>(t, ntx, nty, g);
      rq_zero(q);
      if (tma) {
        if (threadIdx.x == 0) {
          mbar_expect_tx(&bar, (EQC ? 0 : T::SI * (int)sizeof(Px)) + T::SL * 4);
          if (!EQC) tma_load_3d(sI, &mI, c.bx - T::IXO, c.by - T::IYO, c.bz - T::IZO, &bar);
          tma_load_3d(sD, &mL, c.bx - T::LXO, c.by - T::LYO, c.bz - T::LZO, &bar);
        }
        mbar_wait(&bar, phase);
        phase ^= 1u;
      } else {
        stage<CONN>(&mI, &mL, false, I, L, g, c, EQC ? nullptr : sI, sD, &bar);
      }
      decode_box<CONN>(sD);
      if (tile_interior<CONN>(c, g))
        relax_round_body<CONN, false, EQC>(sI, sD, L, g, c, t, ntx, nty, next, ls + (r & 1), flags + 1, q, eqc);
      else
        relax_round_body<CONN, true, EQC>(sI, sD, L, g, c, t, ntx, nty, next, ls + (r & 1), flags + 1, q, eqc);
      __syncthreads();  // the boxes and q are reused by the next tile
    }
    grid.sync();
    // compaction of round r + 1's list; reset the slots round r + 1 uses
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      ls[(r + 1) & 1] = 0;
      ls[2 + (r & 1)] = 0;
    }
    const int lane = threadIdx.x & 31;
    for (int t0 = blockIdx.x * NT; t0 < ntiles; t0 += gridDim.x * NT) {
      const int t = t0 + threadIdx.x;
      bool a = false;
      if (t < ntiles && next[t]) {
        next[t] = 0;
        a = hasplat[t] != 0;
      }
      const unsigned b = __ballot_sync(0xffffffffu, a);
      if (!b) continue;
      int base = 0;
      if (lane == 0) base = atomicAdd(ls + 2 + ((r + 1) & 1), __popc(b));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (a) nl[base + __popc(b & ((1u << lane) - 1))] = t;
    }
    grid.sync();
    if (!vls[r & 1] || vls[2 + ((r + 1) & 1)] == 0 || r + 1 > max_rounds || flags[1]) break;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) ls[4] = r + 1;  // rounds this launch ran
}

// compact list of the tiles of the next round: marked by a neighbour and holding plateau voxels
__global__ void k_tile_list(const uint8_t* __restrict__ next, const uint8_t* __restrict__ hasplat, int n,
                            int* __restrict__ list, int* count) {
  for (int t0 = blockIdx.x * NT; t0 < n; t0 += gridDim.x * NT) {
    const int t = t0 + threadIdx.x;
    const bool a = t < n && next[t] && hasplat[t];
    const unsigned b = __ballot_sync(0xffffffffu, a);
    if (!b) continue;
    const int lane = threadIdx.x & 31;
    int base = 0;
    if (lane == 0) base = atomicAdd(count, __popc(b));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (a) list[base + __popc(b & ((1u << lane) - 1))] = t;
  }
}

// ---------------------- pointers (steps I-II) + tile-local pointer jumping (step III)
// DEBUG: write the un-jumped parent and the distance instead (ws_plateau_debug, T2).
//
// Minimal plateaus (step IV, Alg. 1 l.24-27) are merged inside the tile here: the tile's
// minimal voxels form a shared-memory union-find (min-root, in sG, unused by them otherwise)
// over their in-tile q > p equal pairs, and every minimal voxel points at its in-tile root.
// The q > p pairs that cross the tile face go to a global list for k_union_pairs (about
// 0.1% of the voxels on the paper-like inputs), so step IV never rescans the volume.
constexpr int QCAP = 128;  // per-tile staging of the cross-tile pairs

struct PairOut {
  int2* pairs;   // cross-tile union pairs (global indices)
  int* npairs;   // counter (may exceed cap: the host then runs the full k_union scan)
  int cap;
};

__device__ __forceinline__ int s_find(volatile int* U, int x) {
  while (true) {
    const int y = U[x];
    if (y == x) return x;
    const int z = U[y];
    if (z == y) return y;
    U[x] = z;  // path halving (z is an ancestor of x: benign race)
    x = z;
  }
}

__device__ __forceinline__ void s_unite(int* U, int a, int b) {
  while (true) {
    a = s_find(U, a);
    b = s_find(U, b);
    if (a == b) return;
    if (a > b) { const int t = a; a = b; b = t; }
    if (atomicCAS(U + b, b, a) == b) return;
  }
}

template <int CONN, bool DEBUG, bool BORDER>
__device__ __forceinline__ void resolve_body(const Px* sI, const int* sD, short* sP, int* sG /* aliases sD */, int2* sQ,
                                             int* sQn, int* sQb, const Geo& g, const TileCoord& c,
                                             int* __restrict__ P, int* __restrict__ dist, const PairOut& po) {
  using T = TL<CONN>;
  uint32_t minmask = 0;  // bit k: voxel k of this thread is on a minimal plateau (or a strict minimum)
  // 2-D tiles: minimal-plateau voxels start at their smallest in-tile backward equal neighbour
  // (parent initialisation) and only the other backward neighbours are united -- large flat
  // minimal plateaux (C5, C2) then do not contend for one growing root.  3-D tiles keep every
  // minimal voxel as its own root (C4: fewer instructions in this issue-bound kernel).
  constexpr bool PINIT = false;
  // 2-D tiles use the row runs instead (RUNS; PINIT stays as the measured alternative): a warp
  // holds 32 consecutive voxels of one tile row, a ballot of "equal to my left neighbour" gives
  // every plateau voxel its run start (the run's smallest index) as parent (the first lane of a
  // warp that continues a run links to its left neighbour), and vertical unions are needed only
  // where a run starts: 4-conn, runs R1 (row y) and R2 (row y - 1) overlap => at the leftmost
  // voxel of the overlap one of them starts; 8-conn, they touch => R1's start sees R2 up-left or
  // up, or R2 starts above R1's start or one voxel right of a voxel of R1 (up or up-right)
  constexpr bool RUNS = !Conn<CONN>::is3d;
  constexpr int LEFT = CONN == 4 ? 1 : 3;  // direction (0, 0, -1)
  __shared__ unsigned sStart[RUNS ? T::V / 32 : 1];  // bit: the voxel starts its row run
  uint32_t leqm = 0;     // RUNS: bit k: voxel k is minimal and equal to its in-tile left neighbour
  uint32_t gmask = 0;    // bit k: gk[k] holds sG[j] (stored once sD is dead: sG aliases sD)
  int gk[T::VPT];
#pragma unroll
  for (int k = 0; k < T::VPT; ++k) {
    int lx, ly, lz;
    my_voxel<CONN>(k, lx, ly, lz);
    const int j = threadIdx.x + k * NT;
    if (BORDER && !(c.bx + lx < g.n2 && c.by + ly < g.n1 && c.bz + lz < g.zhi)) {
      // not owned (halo plane of a z-slab, or outside the volume): a tile exit, never a root
      sP[j] = -1;
      gk[k] = (int)((size_t)(c.bz + lz) * g.plane + (size_t)(c.by + ly) * g.n2 + c.bx + lx) + g.gofs;
      gmask |= 1u << k;
      continue;
    }
    const unsigned vm = BORDER ? valid_mask<CONN>(g, c.bz + lz, c.by + ly, c.bx + lx) : (1u << CONN) - 1;
    const int si = T::iI(lz, ly, lx), sl = T::iL(lz, ly, lx);
    const int v = sI[si];
    int m = 1 << (8 * sizeof(Px)), dm = -1;
    unsigned eqm = 0;
#pragma unroll
    for (int i = 0; i < CONN; ++i) {
      if (BORDER && !(vm & (1u << i))) continue;
      const int nv = sI[si + T::oI(i)];
      if (nv <= m) { m = nv; dm = i; }  // Eq. 1: max index among the minima
      if (nv == v) eqm |= 1u << i;
    }
    int dir = DIR_NONE, dd = 0;
    bool minimal = (dm < 0 || m > v);  // strict single-voxel minimum (or a 1-voxel image, C4)
    if (!minimal && m < v) {
      dir = dm;                               // steepest descent (S = 0)
    } else if (!minimal) {                    // plateau voxel without a lower neighbour
      // sD holds the raw step II codes: 0 for d = 0, enc(d, DIR_NONE) = -32 d - 32 for a
      // plateau voxel (INT_MIN = not reached), so the parent test needs no decoding
      const int Lp = sD[sl];
      if (Lp != enc(INF, DIR_NONE)) {         // non-minimal plateau: BFS parent (C5/C6)
        const int want = Lp == enc(1, DIR_NONE) ? 0 : Lp + 32;  // the code of distance d - 1
#pragma unroll
        for (int i = 0; i < CONN; ++i)
          if ((eqm & (1u << i)) && sD[sl + T::oL(i)] == want) dir = i;
        if (DEBUG) dd = dec_d(Lp);
      } else {                                // minimal plateau: merged below
        minimal = true;
      }
    }
    const int p = (int)((size_t)(c.bz + lz) * g.plane + (size_t)(c.by + ly) * g.n2 + c.bx + lx);
    if (DEBUG) {
      dist[p] = minimal ? -1 : dd;
      P[p] = (dir == DIR_NONE || minimal) ? p : p + nb_off<CONN>(g, dir);  // oracle: minima are terminals
      continue;
    }
    if (minimal) {
      minmask |= 1u << k;
      sP[j] = -2;  // root (set after the in-tile union below)
      int par = j;  // union-find parent (local index; RUNS: set with the row ballot below)
      if constexpr (RUNS) {
        if (((eqm >> LEFT) & 1u) && lx > 0) leqm |= 1u << k;
      } else if constexpr (PINIT) {
#pragma unroll
        for (int i = Conn<CONN>::nfwd - 1; i >= 0; --i) {
          int dz, dy, dx;
          nb_delta(CONN, i, dz, dy, dx);
          if ((eqm & (1u << i)) && (unsigned)(lx + dx) < (unsigned)T::TX && (unsigned)(ly + dy) < (unsigned)T::TY &&
              (unsigned)(lz + dz) < (unsigned)T::TZ)
            par = j + (dz * T::TY + dy) * T::TX + dx;
        }
      }
      gk[k] = par;
      gmask |= 1u << k;
    } else {
      int dz, dy, dx;
      nb_delta(CONN, dir, dz, dy, dx);
      const int nx = lx + dx, ny = ly + dy, nz = lz + dz;
      if ((unsigned)nx < (unsigned)T::TX && (unsigned)ny < (unsigned)T::TY && (unsigned)nz < (unsigned)T::TZ) {
        sP[j] = (short)(j + (dz * T::TY + dy) * T::TX + dx);
      } else {
        sP[j] = -1;
        gk[k] = p + nb_off<CONN>(g, dir) + g.gofs;
        gmask |= 1u << k;
      }
    }
  }
  if (DEBUG) return;
  // step IV inside the tile + the cross-tile pairs (q > p: the forward half).  Only
  // the (few) minimal voxels loop; cross-tile pairs are staged in shared memory (sQ) and
  // flushed with one global atomic per tile.
  const bool anymin = __syncthreads_or(minmask != 0);  // sD is dead from here on
#pragma unroll
  for (int k = 0; k < T::VPT; ++k) {
    const int j = threadIdx.x + k * NT;
    int val = gk[k];
    if constexpr (RUNS) {
      const int lane = threadIdx.x & 31;
      const unsigned b = __ballot_sync(0xffffffffu, (leqm >> k) & 1u);
      if (lane == 0) sStart[j >> 5] = ~b;
      if ((leqm >> k) & 1u) {
        const unsigned st = ~b & ((2u << lane) - 1u);  // run starts at or left of me in this warp
        val = st ? j - (lane - (31 - __clz(st))) : (lane ? j - lane : j - 1);
      }
    }
    if (gmask & (1u << k)) sG[j] = val;
  }
  __syncthreads();
  if (anymin) {
    for (uint32_t mm = minmask; mm; mm &= mm - 1) {
      const int k = __ffs(mm) - 1;
      const int j = threadIdx.x + k * NT;
      const int lx = j % T::TX, ly = (j / T::TX) % T::TY, lz = j / (T::TX * T::TY);
      const int si = T::iI(lz, ly, lx);
      const int v = sI[si];
      const unsigned vm = BORDER ? valid_mask<CONN>(g, c.bz + lz, c.by + ly, c.bx + lx) : (1u << CONN) - 1;
      if constexpr (RUNS) {  // vertical: where a run starts
        const bool sj = (sStart[j >> 5] >> (j & 31)) & 1u;
        if (ly > 0) {
          constexpr int UP = CONN == 4 ? 0 : 1;  // direction (0, -1, 0)
          if ((!BORDER || ((vm >> UP) & 1u)) && sI[si + T::oI(UP)] == v) {
            const int u = j - T::TX;
            if (sj || ((sStart[u >> 5] >> (u & 31)) & 1u)) s_unite(sG, j, u);
          }
          if constexpr (CONN == 8) {
            if (sj && lx > 0 && (!BORDER || (vm & 1u)) && sI[si + T::oI(0)] == v)  // up-left
              s_unite(sG, j, j - T::TX - 1);
            if (lx + 1 < T::TX && (!BORDER || (vm & 4u)) && sI[si + T::oI(2)] == v) {  // up-right
              const int u = j - T::TX + 1;
              if ((sStart[u >> 5] >> (u & 31)) & 1u) s_unite(sG, j, u);
            }
          }
        }
      } else if constexpr (PINIT) {  // in-tile backward equal neighbours other than the parent
        bool first = true;
#pragma unroll
        for (int i = 0; i < Conn<CONN>::nfwd; ++i) {
          int dz, dy, dx;
          nb_delta(CONN, i, dz, dy, dx);
          const int nx = lx + dx, ny = ly + dy, nz = lz + dz;
          if (!((unsigned)nx < (unsigned)T::TX && (unsigned)ny < (unsigned)T::TY && (unsigned)nz < (unsigned)T::TZ))
            continue;
          if (BORDER && !(vm & (1u << i))) continue;
          if (sI[si + T::oI(i)] != v) continue;
          if (!first) s_unite(sG, j, j + (dz * T::TY + dy) * T::TX + dx);
          first = false;
        }
      }
#pragma unroll
      for (int i = Conn<CONN>::nfwd; i < CONN; ++i) {
        if (sI[si + T::oI(i)] != v) continue;
        int dz, dy, dx;
        nb_delta(CONN, i, dz, dy, dx);
        const int nx = lx + dx, ny = ly + dy, nz = lz + dz;
        if (BORDER && (!(vm & (1u << i)) || c.bz + nz >= g.zhi)) continue;  // cut plane: ws_shard_merge
        if ((unsigned)nx < (unsigned)T::TX && (unsigned)ny < (unsigned)T::TY && (unsigned)nz < (unsigned)T::TZ) {
          if constexpr (!PINIT && !RUNS) s_unite(sG, j, j + (dz * T::TY + dy) * T::TX + dx);
        } else {
          const int p = (int)((size_t)(c.bz + lz) * g.plane + (size_t)(c.by + ly) * g.n2 + c.bx + lx) + g.gofs;
          const int2 e = make_int2(p, p + nb_off<CONN>(g, i));
          const int s = atomicAdd(sQn, 1);
          if (s < QCAP) {
            sQ[s] = e;
          } else {
            const int gi = atomicAdd(po.npairs, 1);
            if (gi < po.cap) po.pairs[gi] = e;
          }
        }
      }
    }
    __syncthreads();
    const int nq = *sQn < QCAP ? *sQn : QCAP;
    if (threadIdx.x == 0 && nq > 0) *sQb = atomicAdd(po.npairs, nq);
#pragma unroll
    for (int k = 0; k < T::VPT; ++k)
      if ((minmask >> k) & 1) {
        const int j = threadIdx.x + k * NT;
        const int r = s_find(sG, j);
        sP[j] = (short)(r == j ? -2 : r);
      }
    __syncthreads();
    for (int i = threadIdx.x; i < nq; i += NT)
      if (*sQb + i < po.cap) po.pairs[*sQb + i] = sQ[i];
  }  // no minimal voxel: the barrier after the sG stores already orders sP / sG for the walk
  // two in-place pointer-jumping rounds (sP[j] = sP[sP[j]] where that is again an in-tile
  // pointer; a racing reader sees the old or the new value, both ancestors), then the walk
#pragma unroll 1
  for (int round = 0; round < 2; ++round) {
#pragma unroll
    for (int k = 0; k < T::VPT; ++k) {
      const int j = threadIdx.x + k * NT;
      const int jn = sP[j];
      if (jn >= 0) {
        const int jj = sP[jn];
        if (jj >= 0) sP[j] = (short)jj;
      }
    }
    __syncthreads();
  }
  // tile-local path reduction: follow in-tile pointers to a root or to the tile exit (a
  // serial walk per voxel measured faster than pointer doubling with block-wide rounds)
  const int base = (int)((size_t)c.bz * g.plane + (size_t)c.by * g.n2 + c.bx);
#pragma unroll
  for (int k = 0; k < T::VPT; ++k) {
    int lx, ly, lz;
    my_voxel<CONN>(k, lx, ly, lz);
    if (BORDER && !(c.bx + lx < g.n2 && c.by + ly < g.n1 && c.bz + lz < g.zhi)) continue;
    int j = threadIdx.x + k * NT;
    int jn = sP[j];
    while (jn >= 0) {
      j = jn;
      jn = sP[j];
    }
    int out;
    if (jn == -1) {
      out = sG[j];
    } else {
      const int rx = j % T::TX, ry = (j / T::TX) % T::TY, rz = j / (T::TX * T::TY);
      out = base + rz * g.plane + ry * g.n2 + rx + g.gofs;  // global index
    }
    P[base + lz * g.plane + ly * g.n2 + lx] = out;
  }
}

template <int CONN, bool DEBUG>
__global__ void __launch_bounds__(NT) k_resolve(const __grid_constant__ CUtensorMap mI,
                                                const __grid_constant__ CUtensorMap mL, int tma,
                                                const Px* __restrict__ I, const int* __restrict__ L, Geo g,
                                                int ntx, int nty, int* __restrict__ P, int* __restrict__ dist,
                                                PairOut po) {
  using T = TL<CONN>;
  __shared__ alignas(128) Px sI[T::SI];
  __shared__ alignas(128) int sD[T::SL];
  static_assert(T::SL >= T::V, "sG aliases sD");
  __shared__ short sP[T::V];  // local target, -1 = leaves the tile, -2 = root
  __shared__ int2 sQ[QCAP];   // cross-tile step IV pairs
  __shared__ int sQn, sQb;
  __shared__ uint64_t bar;
  int t;
  const TileCoord c = tile_of_block<CONN>(ntx, nty, g, t);
  if (threadIdx.x == 0) sQn = 0;
  stage<CONN>(&mI, &mL, tma, I, L, g, c, sI, sD, &bar);  // raw step II codes (no decoding)
  if (tile_interior<CONN>(c, g))
    resolve_body<CONN, DEBUG, false>(sI, sD, sP, sD, sQ, &sQn, &sQb, g, c, P, dist, po);
  else
    resolve_body<CONN, DEBUG, true>(sI, sD, sP, sD, sQ, &sQn, &sQb, g, c, P, dist, po);
}

// --------------------------- step III across tiles + per-root minimum + root list
// After the chase P[p] = r (a self-loop root).  L[r] accumulates INT_MAX - min{p : P[p] = r}
// with atomicMax: the dead step-II codes left in L are all <= 0 < INT_MAX - p, so no
// initialisation pass is needed.  Grid-stride order keeps every block inside one moving
// window of the volume (the chase targets of neighbouring tiles stay in L2).  Within a warp
// voxels are consecutive, so the first lane of every run of equal roots holds the run's
// minimum and issues the only atomic for it.  Roots are staged in shared memory and flushed
// to the global list with one atomicAdd per batch.
constexpr int RBUF = 2048;

__global__ void __launch_bounds__(NT) k_jump(int* P, int* __restrict__ L, int N, int* roots, int cap,
                                             int* nroots) {
  __shared__ int sbuf[RBUF];
  __shared__ int scount, sbase;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) scount = 0;
  __syncthreads();
  const int stride = gridDim.x * NT;
  int cnt = 0;  // staged roots: block-uniform (a register, never re-read from scount)
  for (int p0 = blockIdx.x * NT; p0 < N; p0 += stride) {
    const int p = p0 + threadIdx.x;
    const bool valid = p < N;
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
    cnt += __syncthreads_count(isr);  // the barrier that orders the appends before the flush
    if (cnt > RBUF - NT || p0 + stride >= N) {  // flush the staged roots
      if (cnt > 0) {
        if (threadIdx.x == 0) sbase = atomicAdd(nroots, cnt);
        __syncthreads();
        for (int i = threadIdx.x; i < cnt; i += NT)
          if (sbase + i < cap) roots[sbase + i] = sbuf[i];
      }
      __syncthreads();
      if (threadIdx.x == 0) scount = 0;
      __syncthreads();
      cnt = 0;
    }
  }
}

// The same with V voxels per thread (p, p + NT, ... of a V NT window): every chase's first
// load and first hop is issued before any is consumed (V times the loads in flight of a
// latency-bound kernel, 1/V of the loop iterations); the rare longer chases (tile exits) follow.
__device__ __forceinline__ int chase_tail(int* P, int p, int t, int nt) {
  // t = P[p] != p and nt = P[t] != t: follow to the root, compress p
  do {
    t = nt;
    nt = P[t];
  } while (nt != t);
  P[p] = t;
  return t;
}

template <int V>
__global__ void __launch_bounds__(NT) k_jumpv(int* P, int* __restrict__ L, int N, int* roots, int cap, int* nroots) {
  constexpr int SB = 2 * V * NT > RBUF ? 2 * V * NT : RBUF;  // staged roots (two iterations' worth)
  __shared__ int sbuf[SB];
  __shared__ int scount, sbase;
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1;
  if (threadIdx.x == 0) scount = 0;
  __syncthreads();
  const int stride = gridDim.x * V * NT;
  int cnt = 0;
  for (int p0 = blockIdx.x * V * NT; p0 < N; p0 += stride) {
    int t[V], n[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int p = p0 + v * NT + threadIdx.x;
      t[v] = p < N ? P[p] : p;
    }
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int p = p0 + v * NT + threadIdx.x;
      n[v] = t[v] != p ? P[t[v]] : t[v];
    }
    int nr = 0;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int p = p0 + v * NT + threadIdx.x;
      const bool valid = p < N;
      if (n[v] != t[v]) t[v] = chase_tail(P, p, t[v], n[v]);
      if (!valid) t[v] = -1 - lane;  // unique per lane (never equals a neighbour's root)
      const int pr = __shfl_up_sync(0xffffffffu, t[v], 1);
      if (valid && (lane == 0 || pr != t[v])) atomicMax(L + t[v], INT_MAX - p);
      const bool isr = valid && t[v] == p;
      const unsigned rb = __ballot_sync(0xffffffffu, isr);
      if (rb) {
        int base = 0;
        if (lane == 0) base = atomicAdd(&scount, __popc(rb));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (isr) sbuf[base + __popc(rb & lt)] = p;
      }
      nr += isr;
    }
    // block-uniform count of the staged roots: every thread reads scount between two barriers
    __syncthreads();
    cnt = scount;
    __syncthreads();
    if (cnt > SB - V * NT || p0 + stride >= N) {  // flush the staged roots
      if (cnt > 0) {
        if (threadIdx.x == 0) sbase = atomicAdd(nroots, cnt);
        __syncthreads();
        for (int i = threadIdx.x; i < cnt; i += NT)
          if (sbase + i < cap) roots[sbase + i] = sbuf[i];
      }
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
__global__ void k_union(const Px* __restrict__ I, int* P, Geo g) {
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

// step IV Union on the cross-tile pairs k_resolve listed (the in-tile ones are merged there)
// nptr != nullptr: the count is k_resolve's device counter (clipped to the list capacity n)
__global__ void k_union_pairs(int* P, const int2* __restrict__ pairs, int n, const int* nptr = nullptr) {
  if (nptr) n = min(*nptr, n);
  for (int i = blockIdx.x * NT + threadIdx.x; i < n; i += gridDim.x * NT) {
    const int2 e = pairs[i];
    if (ld_cg(P + e.x) != ld_cg(P + e.y)) uf_unite(P, e.x, e.y);
  }
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

// fast path (unions before the chase): every listed root is final and L[r] already holds
// INT_MAX - (smallest voxel index of its region); P[r] = -1 - canonical label
// bits != nullptr (ws_segment): also set bit c of the representative bitmap for the canonical
// label c of every listed root (several listed roots of one region set the same bit)
__global__ void k_root_canon(int* P, const int* __restrict__ L, const int* __restrict__ roots, const int* nptr,
                             int cap, unsigned* __restrict__ bits) {
  const int n = min(*nptr, cap);
  for (int i = blockIdx.x * NT + threadIdx.x; i < n; i += gridDim.x * NT) {
    const int r = roots[i];
    const int c = INT_MAX - L[r];
    P[r] = -1 - c;
    if (bits) atomicOr(bits + (c >> 5), 1u << (c & 31));
  }
}

// P[root] = -1 - canonical label (no finds run any more)
__global__ void k_root_store(int* P, const int* __restrict__ roots, const int* __restrict__ rootc, int n,
                             unsigned* __restrict__ bits) {
  for (int i = blockIdx.x * NT + threadIdx.x; i < n; i += gridDim.x * NT) {
    const int c = rootc[i];
    P[roots[i]] = -1 - c;
    if (bits) atomicOr(bits + (c >> 5), 1u << (c & 31));
  }
}

// labels[p] = canonical label of p's step III root
__global__ void __launch_bounds__(NT) k_relabel(const int* __restrict__ P, int* __restrict__ L, int N) {
  for (int p = blockIdx.x * NT + threadIdx.x; p < N; p += gridDim.x * NT) {
    const int t = P[p];
    L[p] = -1 - (t < 0 ? t : __ldg(P + t));
  }
}

// the same, 4 consecutive voxels per thread (16-byte loads and stores; a root shared by
// neighbouring voxels is gathered once)
__device__ __forceinline__ int relabel_one(const int* __restrict__ P, int t) {
  return -1 - (t < 0 ? t : __ldg(P + t));
}

__global__ void __launch_bounds__(NT) k_relabel4(const int* __restrict__ P, int* __restrict__ L, int N) {
  const int n4 = N >> 2;
  const int4* P4 = reinterpret_cast<const int4*>(P);
  int4* L4 = reinterpret_cast<int4*>(L);
  for (int i = blockIdx.x * NT + threadIdx.x; i < n4; i += gridDim.x * NT) {
    const int4 t = __ldg(P4 + i);  // not evict-first: the root entries it gathers share these lines
    int4 o;
    o.x = relabel_one(P, t.x);
    o.y = t.y == t.x ? o.x : relabel_one(P, t.y);
    o.z = t.z == t.y ? o.y : relabel_one(P, t.z);
    o.w = t.w == t.z ? o.z : relabel_one(P, t.w);
    __stcs(L4 + i, o);
  }
  for (int p = 4 * n4 + blockIdx.x * NT + threadIdx.x; p < N; p += gridDim.x * NT) L[p] = relabel_one(P, P[p]);
}

// --------------------------------------------------------------------------- drivers
struct TileGrid {
  int ntx, nty, ntz, n;
};

template <int CONN>
static TileGrid tiles_of(const Geo& g) {
  using T = TL<CONN>;
  TileGrid tg;
  tg.ntx = (g.n2 + T::TX - 1) / T::TX;
  tg.nty = (g.n1 + T::TY - 1) / T::TY;
  tg.ntz = (g.zhi - g.zlo + T::TZ - 1) / T::TZ;
  tg.n = tg.ntx * tg.nty * tg.ntz;
  return tg;
}

static int grid1d(long long n, int sms, int per_sm = 8) {
  long long b = (n + NT - 1) / NT;
  long long cap = (long long)sms * per_sm;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

template <int CONN>
static ws_status plateau_phase(ws_ctx* ctx, const Px* grad, const Geo& g, int32_t* L, const TileGrid& tg,
                               const Maps& mp, cudaStream_t st, bool small = false) {
  WS_TRY(ctx->flags.ensure(256, "flags"));
  WS_TRY(ctx->tiles.ensure((size_t)tg.n * 3, "tile flags"));
  int* flags = ctx->flags.as<int>();
  uint8_t* cur = ctx->tiles.as<uint8_t>();
  uint8_t* next = cur + tg.n;
  uint8_t* hasplat = next + tg.n;
  // two lists (the cooperative loop ping-pongs); sized BEFORE k_tile_list writes the first:
  // a later ensure() may re-allocate (no copy)
  WS_TRY(ctx->tlist.ensure((size_t)tg.n * 2 * sizeof(int), "active tile lists"));
  int* list = ctx->tlist.as<int>();
  const int gl = std::max(1, std::min((tg.n + NT - 1) / NT, ctx->num_sms * 8));
  // the whole flag block (later host reads copy ranges of it; every field is defined)
  WS_CUDA(cudaMemsetAsync(flags, 0, 256, st));
  WS_CUDA(cudaMemsetAsync(next, 0, 2 * (size_t)tg.n, st));  // next and hasplat
  // equal-neighbour mask cache (CONN <= 8: one byte per voxel) so the later rounds stage only
  // the L box; WS_NO_EQC=1 restages the I box
  constexpr bool EQ = CONN <= 8;
  uint8_t* eqc = nullptr;
  {
    const char* ne = getenv("WS_NO_EQC");
    if (EQ && !(ne && ne[0] == '1')) {
      WS_TRY(ctx->eqc.ensure((size_t)tg.n * EQB, "equal-neighbour mask cache"));
      eqc = ctx->eqc.as<uint8_t>();
    }
  }
  k_relax_first<CONN><<<tile_grid(tg.ntx, tg.nty, tg.ntz), NT, 0, st>>>(mp.mI, mp.tma, grad, L, g, tg.ntx, tg.nty, next, hasplat, flags,
                                                                        eqc);
  k_tile_list<<<gl, NT, 0, st>>>(next, hasplat, tg.n, list, flags + 4);
  launched(ctx, PH_WS_INIT, 2);
  tmark(ctx, st, PH_WS_INIT);
  int rounds = 1;
  // Rounds with many active tiles run as k_relax_round launches (one CTA per listed tile);
  // once the list fits one wave of co-resident CTAs, all remaining rounds run in ONE
  // cooperative k_relax_loop launch (no host round trip per round).  A persistent grid
  // walking a long list measured slower than the per-round launches (C4 first round).
  int occ = 0;
  const bool coop = ctx->coop &&
                    cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                        &occ, eqc ? (const void*)k_relax_loop<CONN, EQ> : (const void*)k_relax_loop<CONN, false>, NT,
                        0) == cudaSuccess &&
                    occ > 0;
  const int wave = occ * ctx->num_sms;
  // small inputs (every tile list fits one wave): all rounds after the first in the
  // cooperative kernel straight away, no host read (the depth-limit flag and the round
  // count are read with the call's final counts)
  if (small && coop && tg.n <= wave) {
    int* list1 = list + tg.n;
    int* ls = flags + 20;
    WS_CUDA(cudaMemsetAsync(ls, 0, 5 * sizeof(int), st));
    WS_CUDA(cudaMemcpyAsync(ls + 2, flags + 4, sizeof(int), cudaMemcpyDeviceToDevice, st));
    const int grid = std::max(1, std::min(tg.n, wave));
    CUtensorMap mI = mp.mI, mL = mp.mL;
    int tma = mp.tma, ntx = tg.ntx, nty = tg.nty, ntiles = tg.n, maxr = g.N + 2;
    Geo gg = g;
    int32_t* LL = L;
    const Px* II = grad;
    const uint8_t* ec = eqc;
    void* args[] = {&mI, &mL, &tma, &II, &LL, &gg, &ntx, &nty, &ntiles, &next, &hasplat, &flags, &ls, &list, &list1,
                    &maxr, &ec};
    WS_CUDA(cudaLaunchCooperativeKernel(
        eqc ? (const void*)k_relax_loop<CONN, EQ> : (const void*)k_relax_loop<CONN, false>, dim3(grid), dim3(NT), args, 0,
        st));
    launched(ctx, PH_WS_RELAX);
    ctx->stats.plateau_rounds = -1;  // filled from ls[4] by the final read
    tmark(ctx, st, PH_WS_RELAX);
    WS_CUDA(cudaGetLastError());
    return WS_OK;
  }
  while (true) {
    WS_CUDA(cudaMemcpyAsync(ctx->pinned, flags, 5 * sizeof(int), cudaMemcpyDeviceToHost, st));
    WS_CUDA(cudaStreamSynchronize(st));
    const int* h = reinterpret_cast<const int*>(ctx->pinned);
    if (h[1]) {
      set_error(WS_ERR_LIMIT, "a non-minimal plateau is deeper than 2^26-2 voxels");
      return WS_ERR_LIMIT;
    }
    const int nact = h[4];
    if (!h[0] || nact == 0) break;
    if (rounds > g.N + 2) {
      set_error(WS_ERR_INTERNAL, "step II did not converge");
      return WS_ERR_INTERNAL;
    }
    if (coop && nact <= wave) {
      int* list1 = list + tg.n;
      int* ls = flags + 20;
      // ls[2] = the list k_tile_list just built (its count is flags[4]); ls[0], ls[3] = 0
      WS_CUDA(cudaMemsetAsync(next, 0, tg.n, st));
      WS_CUDA(cudaMemsetAsync(ls, 0, 5 * sizeof(int), st));
      WS_CUDA(cudaMemcpyAsync(ls + 2, flags + 4, sizeof(int), cudaMemcpyDeviceToDevice, st));
      const int grid = std::max(1, std::min(nact, wave));
      CUtensorMap mI = mp.mI, mL = mp.mL;
      int tma = mp.tma, ntx = tg.ntx, nty = tg.nty, ntiles = tg.n, maxr = g.N + 2 - rounds;
      Geo gg = g;
      int32_t* LL = L;
      const Px* II = grad;
      const uint8_t* ec = eqc;
      void* args[] = {&mI, &mL, &tma, &II, &LL, &gg, &ntx, &nty, &ntiles, &next, &hasplat, &flags, &ls, &list, &list1,
                      &maxr, &ec};
      WS_CUDA(cudaLaunchCooperativeKernel(
          eqc ? (const void*)k_relax_loop<CONN, EQ> : (const void*)k_relax_loop<CONN, false>, dim3(grid), dim3(NT), args,
          0, st));
      launched(ctx, PH_WS_RELAX);
      WS_CUDA(cudaMemcpyAsync(ctx->pinned, flags, 25 * sizeof(int), cudaMemcpyDeviceToHost, st));
      WS_CUDA(cudaStreamSynchronize(st));
      if (h[1]) {
        set_error(WS_ERR_LIMIT, "a non-minimal plateau is deeper than 2^26-2 voxels");
        return WS_ERR_LIMIT;
      }
      rounds += h[24];
      if (rounds > g.N + 2) {
        set_error(WS_ERR_INTERNAL, "step II did not converge");
        return WS_ERR_INTERNAL;
      }
      break;
    }
    std::swap(cur, next);
    WS_CUDA(cudaMemsetAsync(next, 0, tg.n, st));
    WS_CUDA(cudaMemsetAsync(flags, 0, 5 * sizeof(int), st));
    if (eqc)
      k_relax_round<CONN, EQ><<<nact, NT, 0, st>>>(mp.mI, mp.mL, mp.tma, grad, L, g, tg.ntx, tg.nty, cur, next, hasplat,
                                                   flags, list, eqc);
    else
      k_relax_round<CONN><<<nact, NT, 0, st>>>(mp.mI, mp.mL, mp.tma, grad, L, g, tg.ntx, tg.nty, cur, next, hasplat,
                                               flags, list);
    k_tile_list<<<gl, NT, 0, st>>>(next, hasplat, tg.n, list, flags + 4);
    launched(ctx, PH_WS_RELAX, 2);
    ++rounds;
  }
  ctx->stats.plateau_rounds = rounds;
  tmark(ctx, st, PH_WS_RELAX);
  WS_CUDA(cudaGetLastError());
  return WS_OK;
}

// step III across tiles: k_jumpv with V voxels per thread (WS_JUMP_V = 1, 2, 4, 8; default 2;
// 1 = the one-voxel k_jump).  Measured on C4 (tools/raw_ab.py): the gradient 20.8 / 19.5 /
// 19.3 ms for V = 1 / 2 / 4, the raw volume (98 M regions, 12 % roots) 18.4 / 18.7 / 24.8 ms
// -- V = 2 is the robust choice.
static ws_status launch_jump(ws_ctx* ctx, int* P, int* L, int N, int cap, int* nr, cudaStream_t st) {
  const char* e = getenv("WS_JUMP_V");
  const int v = e ? atoi(e) : 2;
  int* roots = ctx->roots.as<int>();
  if (v == 1)
    k_jump<<<grid1d(N, ctx->num_sms), NT, 0, st>>>(P, L, N, roots, cap, nr);
  else if (v == 2)
    k_jumpv<2><<<grid1d(N / 2 + 1, ctx->num_sms), NT, 0, st>>>(P, L, N, roots, cap, nr);
  else if (v == 8)
    k_jumpv<8><<<grid1d(N / 8 + 1, ctx->num_sms), NT, 0, st>>>(P, L, N, roots, cap, nr);
  else
    k_jumpv<4><<<grid1d(N / 4 + 1, ctx->num_sms), NT, 0, st>>>(P, L, N, roots, cap, nr);
  WS_CUDA(cudaGetLastError());
  return WS_OK;
}

// cross-tile step IV pair list of k_resolve: ctx->upairs, counter at flags int 10
static ws_status pair_out(ws_ctx* ctx, const Geo& g, PairOut& po, cudaStream_t st) {
  const size_t own = (size_t)(g.zhi - g.zlo) * g.plane;
  const size_t want = own / 8 + 65536;  // plateau-heavy volumes (C3 air) have many face pairs
  if (ctx->upairs.bytes / sizeof(int2) < want) WS_TRY(ctx->upairs.ensure(want * sizeof(int2), "union pairs"));
  WS_TRY(ctx->flags.ensure(256, "flags"));
  po.pairs = ctx->upairs.as<int2>();
  po.npairs = ctx->flags.as<int>() + 10;
  po.cap = (int)(ctx->upairs.bytes / sizeof(int2));
  WS_CUDA(cudaMemsetAsync(po.npairs, 0, sizeof(int), st));
  return WS_OK;
}

// relabel == false (ws_segment): stop before the relabel pass; P = ctx->aux then holds, for
// every voxel, a listed root (or, at a listed root r, P[r] = -1 - canonical label), the
// listed roots are ctx->roots[0 .. ctx->seg_nroots) (a superset of the final roots on the
// chase-first path; every listed root maps to its region's canonical label), and
// ctx->repbits (N/32 + 1 words) has bit c set for every canonical label c.
template <int CONN>
static ws_status watershed_t(ws_ctx* ctx, const Px* grad, const Geo& g, int32_t* L, int64_t* num_regions,
                             cudaStream_t st, bool relabel = true, bool small = false) {
  const TileGrid tg = tiles_of<CONN>(g);
  Maps mp;
  make_maps<CONN>(grad, L, g, mp);
  ctx->stats.tma = mp.tma;
  WS_TRY(plateau_phase<CONN>(ctx, grad, g, L, tg, mp, st, small));
  WS_TRY(ctx->aux.ensure((size_t)g.N * sizeof(int), "aux"));
  int* P = ctx->aux.as<int>();
  PairOut po;
  WS_TRY(pair_out(ctx, g, po, st));
  k_resolve<CONN, false><<<tile_grid(tg.ntx, tg.nty, tg.ntz), NT, 0, st>>>(mp.mI, mp.mL, mp.tma, grad, L, g, tg.ntx, tg.nty, P, nullptr, po);
  launched(ctx, PH_WS_SELECT);
  tmark(ctx, st, PH_WS_SELECT);

  // step IV Union of the minimal plateaus across tile faces FIRST (k_resolve merged them
  // inside the tiles and left every minimal voxel pointing at its in-tile root), then step III
  // across tiles: the chase ends at the FINAL roots, whose minima k_jump folds directly
  size_t cap = ctx->roots.bytes / sizeof(int);
  const size_t want = small ? (size_t)g.N + 1024 : (size_t)g.N / 16 + 1024;  // small: never overflows
  if (cap < want) {
    WS_TRY(ctx->roots.ensure(want * sizeof(int), "roots"));
    WS_TRY(ctx->rootc.ensure(want * sizeof(int), "root labels"));
    cap = ctx->roots.bytes / sizeof(int);
  }
  int* nr = ctx->flags.as<int>() + 8;
  unsigned long long* nfinal = reinterpret_cast<unsigned long long*>(ctx->flags.as<char>() + 64);
  unsigned* bits = nullptr;
  if (!relabel) {
    const size_t nw = (size_t)g.N / 32 + 1;
    WS_TRY(ctx->repbits.ensure(nw * sizeof(unsigned), "representative bitmap"));
    bits = ctx->repbits.as<unsigned>();
    WS_CUDA(cudaMemsetAsync(bits, 0, nw * sizeof(unsigned), st));
  }
  WS_CUDA(cudaMemsetAsync(nr, 0, sizeof(int), st));
  WS_CUDA(cudaMemsetAsync(nfinal, 0, sizeof(unsigned long long), st));
  if (small) {
    // sync-free (ws_segment on small inputs): unions first with the device pair count, the
    // chase, the root labels; a pair-list overflow is detected by the call's final read
    // (which then redoes the call on the regular path)
    k_union_pairs<<<grid1d(std::min<long long>(po.cap, g.N / 8 + 1), ctx->num_sms), NT, 0, st>>>(
        P, po.pairs, po.cap, po.npairs);
    launched(ctx, PH_WS_UNION);
    tmark(ctx, st, PH_WS_UNION);
    WS_TRY(launch_jump(ctx, P, L, g.N, (int)cap, nr, st));
    launched(ctx, PH_WS_JUMP);
    tmark(ctx, st, PH_WS_JUMP);
    k_root_canon<<<grid1d((long long)g.N / 32, ctx->num_sms), NT, 0, st>>>(P, L, ctx->roots.as<int>(), nr, (int)cap,
                                                                          bits);
    launched(ctx, PH_WS_FIND);
    tmark(ctx, st, PH_WS_FIND);
    ctx->stats.union_order = 0;
    WS_CUDA(cudaGetLastError());
    return WS_OK;
  }
  WS_CUDA(cudaMemcpyAsync(ctx->pinned, po.npairs, sizeof(int), cudaMemcpyDeviceToHost, st));
  WS_CUDA(cudaStreamSynchronize(st));
  const int n_pairs = (int)reinterpret_cast<const int*>(ctx->pinned)[0];
  const int gN = grid1d(g.N, ctx->num_sms);
  const int* roots = ctx->roots.as<int>();
  // Unions before the chase put every voxel of a region on its FINAL root; for a giant
  // minimal plateau (many cross-tile pairs, e.g. the air of C3) the chase's per-root minimum
  // atomics would then all hit one address, so such inputs chase first and union after
  bool fast = n_pairs <= po.cap && (long long)n_pairs <= (long long)g.N / 64;
  ctx->stats.union_order = fast ? 0 : (n_pairs <= po.cap ? 1 : 2);
  if (fast) {
    if (n_pairs > 0) {
      k_union_pairs<<<grid1d(n_pairs, ctx->num_sms), NT, 0, st>>>(P, po.pairs, n_pairs);
      launched(ctx, PH_WS_UNION);
    }
    tmark(ctx, st, PH_WS_UNION);
    WS_TRY(launch_jump(ctx, P, L, g.N, (int)cap, nr, st));
    launched(ctx, PH_WS_JUMP);
    tmark(ctx, st, PH_WS_JUMP);
    k_root_canon<<<grid1d((long long)g.N / 32, ctx->num_sms), NT, 0, st>>>(P, L, roots, nr, (int)cap, bits);
    launched(ctx, PH_WS_FIND);
    tmark(ctx, st, PH_WS_FIND);
    if (!relabel) {
      WS_CUDA(cudaMemcpyAsync(ctx->pinned, nr, sizeof(int), cudaMemcpyDeviceToHost, st));
      WS_CUDA(cudaStreamSynchronize(st));
      const int n_roots = reinterpret_cast<const int*>(ctx->pinned)[0];
      if ((size_t)n_roots <= cap) {
        ctx->seg_nroots = n_roots;
        ctx->stats.n_regions = n_roots;
        if (num_regions) *num_regions = n_roots;
        WS_CUDA(cudaGetLastError());
        return WS_OK;
      }
      WS_TRY(ctx->roots.ensure((size_t)n_roots * sizeof(int), "roots"));
      WS_TRY(ctx->rootc.ensure((size_t)n_roots * sizeof(int), "root labels"));
      const ws_status s = watershed_t<CONN>(ctx, grad, g, L, num_regions, st, false);
      ctx->stats.root_overflow = 1;
      return s;
    }
    if (!(reinterpret_cast<uintptr_t>(P) & 15) && !(reinterpret_cast<uintptr_t>(L) & 15))
      k_relabel4<<<grid1d(g.N / 4 + 1, ctx->num_sms), NT, 0, st>>>(P, L, g.N);
    else
      k_relabel<<<gN, NT, 0, st>>>(P, L, g.N);
    launched(ctx, PH_WS_RELABEL);
    tmark(ctx, st, PH_WS_RELABEL);
    WS_CUDA(cudaMemcpyAsync(ctx->pinned, nr, sizeof(int), cudaMemcpyDeviceToHost, st));
    WS_CUDA(cudaStreamSynchronize(st));
    const int n_roots = reinterpret_cast<const int*>(ctx->pinned)[0];
    if ((size_t)n_roots <= cap) {
      ctx->stats.n_regions = n_roots;
      if (num_regions) *num_regions = n_roots;
      WS_CUDA(cudaGetLastError());
      return WS_OK;
    }
    // root list overflow (more than N/16 regions): P no longer holds the roots' self-loops,
    // so the watershed is redone with a list large enough
    WS_TRY(ctx->roots.ensure((size_t)n_roots * sizeof(int), "roots"));
    WS_TRY(ctx->rootc.ensure((size_t)n_roots * sizeof(int), "root labels"));
    const ws_status s = watershed_t<CONN>(ctx, grad, g, L, num_regions, st);
    ctx->stats.root_overflow = 1;
    return s;
  }
  // many cross-tile pairs: chase first (per-root minima on the tiles' roots), then the union
  // (the pair list, or the full q > p scan when it overflowed), then merge the minima into
  // the final roots
  WS_TRY(launch_jump(ctx, P, L, g.N, (int)cap, nr, st));
  launched(ctx, PH_WS_JUMP);
  WS_CUDA(cudaMemcpyAsync(ctx->pinned, nr, sizeof(int), cudaMemcpyDeviceToHost, st));
  WS_CUDA(cudaStreamSynchronize(st));
  const int n_roots = (int)reinterpret_cast<const int*>(ctx->pinned)[0];
  if ((size_t)n_roots > cap) {  // list overflow: grow and rebuild it from P
    ctx->stats.root_overflow = 1;
    WS_TRY(ctx->roots.ensure((size_t)n_roots * sizeof(int), "roots"));
    WS_TRY(ctx->rootc.ensure((size_t)n_roots * sizeof(int), "root labels"));
    WS_CUDA(cudaMemsetAsync(nr, 0, sizeof(int), st));
    k_collect_roots<<<gN, NT, 0, st>>>(P, g.N, ctx->roots.as<int>(), nr);
    launched(ctx, PH_WS_JUMP);
    roots = ctx->roots.as<int>();
  }
  tmark(ctx, st, PH_WS_JUMP);
  if (n_pairs <= po.cap) {
    if (n_pairs > 0) {
      k_union_pairs<<<grid1d(n_pairs, ctx->num_sms), NT, 0, st>>>(P, po.pairs, n_pairs);
      launched(ctx, PH_WS_UNION);
    }
  } else {
    const L3 l = launch3(g);
    k_union<CONN><<<l.grid, l.block, 0, st>>>(grad, P, g);
    launched(ctx, PH_WS_UNION);
  }
  tmark(ctx, st, PH_WS_UNION);
  const int gR = grid1d(n_roots, ctx->num_sms);
  k_root_merge<<<gR, NT, 0, st>>>(P, L, roots, n_roots, nfinal);
  k_root_label<<<gR, NT, 0, st>>>(P, L, roots, n_roots, ctx->rootc.as<int>());
  k_root_store<<<gR, NT, 0, st>>>(P, roots, ctx->rootc.as<int>(), n_roots, bits);
  launched(ctx, PH_WS_FIND, 3);
  tmark(ctx, st, PH_WS_FIND);
  if (!relabel) {
    ctx->seg_nroots = n_roots;
    WS_CUDA(cudaGetLastError());
    WS_CUDA(cudaMemcpyAsync(ctx->pinned, nfinal, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    WS_CUDA(cudaStreamSynchronize(st));
    ctx->stats.n_regions = ctx->pinned[0];
    if (num_regions) *num_regions = ctx->pinned[0];
    return WS_OK;
  }
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

// ------------------------------------------------------------- z-slab sharded phases
// (both pixel types: the 16-bit instantiation shards ws_watershed_u16, NEXT f4)
__global__ void k_mark_layer(uint8_t* cur, int layer, int per_layer) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < per_layer; i += gridDim.x * blockDim.x)
    cur[layer * per_layer + i] = 1;
}

template <int CONN>
static ws_status shard_first_t(ws_ctx* ctx, const Px* grad, const Geo& g, int32_t* L, int* pending,
                               cudaStream_t st) {
  const TileGrid tg = tiles_of<CONN>(g);
  Maps mp;
  make_maps<CONN>(grad, L, g, mp);
  WS_TRY(ctx->flags.ensure(256, "flags"));
  WS_TRY(ctx->tiles.ensure((size_t)tg.n * 3, "tile flags"));
  int* flags = ctx->flags.as<int>();
  uint8_t* a = ctx->tiles.as<uint8_t>();
  uint8_t* hasplat = a + 2 * tg.n;
  WS_CUDA(cudaMemsetAsync(flags, 0, 2 * sizeof(int), st));
  WS_CUDA(cudaMemsetAsync(a, 0, tg.n, st));
  WS_CUDA(cudaMemsetAsync(hasplat, 0, tg.n, st));
  k_relax_first<CONN><<<tile_grid(tg.ntx, tg.nty, tg.ntz), NT, 0, st>>>(mp.mI, mp.tma, grad, L, g, tg.ntx, tg.nty, a, hasplat, flags,
                                                                        nullptr);
  launched(ctx, PH_WS_INIT);
  ctx->shard_tiles = tg.n;
  ctx->shard_flip = 0;  // "next" = buffer 0
  WS_CUDA(cudaMemcpyAsync(ctx->pinned, flags, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
  WS_CUDA(cudaStreamSynchronize(st));
  const int* h = reinterpret_cast<const int*>(ctx->pinned);
  if (h[1]) {
    set_error(WS_ERR_LIMIT, "a non-minimal plateau is deeper than 2^26-2 voxels");
    return WS_ERR_LIMIT;
  }
  *pending = h[0];
  return WS_OK;
}

template <int CONN>
static ws_status shard_round_t(ws_ctx* ctx, const Px* grad, const Geo& g, int32_t* L, int act_lo, int act_hi,
                               int* pending, cudaStream_t st) {
  const TileGrid tg = tiles_of<CONN>(g);
  if (tg.n != ctx->shard_tiles) {
    set_error(WS_ERR_INVALID, "ws_shard_plateau: round called without a matching first phase");
    return WS_ERR_INVALID;
  }
  Maps mp;
  make_maps<CONN>(grad, L, g, mp);
  int* flags = ctx->flags.as<int>();
  uint8_t* cur = ctx->tiles.as<uint8_t>() + (size_t)ctx->shard_flip * tg.n;
  uint8_t* next = ctx->tiles.as<uint8_t>() + (size_t)(1 - ctx->shard_flip) * tg.n;
  uint8_t* hasplat = ctx->tiles.as<uint8_t>() + 2 * (size_t)tg.n;
  const int per = tg.ntx * tg.nty;
  if (act_lo) k_mark_layer<<<(per + 255) / 256, 256, 0, st>>>(cur, 0, per);
  if (act_hi) k_mark_layer<<<(per + 255) / 256, 256, 0, st>>>(cur, tg.ntz - 1, per);
  WS_CUDA(cudaMemsetAsync(next, 0, tg.n, st));
  WS_CUDA(cudaMemsetAsync(flags, 0, 2 * sizeof(int), st));
  k_relax_round<CONN><<<tg.n, NT, 0, st>>>(mp.mI, mp.mL, mp.tma, grad, L, g, tg.ntx, tg.nty, cur, next, hasplat, flags,
                                           nullptr);
  launched(ctx, PH_WS_RELAX);
  ctx->shard_flip = 1 - ctx->shard_flip;
  WS_CUDA(cudaMemcpyAsync(ctx->pinned, flags, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
  WS_CUDA(cudaStreamSynchronize(st));
  const int* h = reinterpret_cast<const int*>(ctx->pinned);
  if (h[1]) {
    set_error(WS_ERR_LIMIT, "a non-minimal plateau is deeper than 2^26-2 voxels");
    return WS_ERR_LIMIT;
  }
  *pending = h[0];
  return WS_OK;
}

ws_status plateau_first_shard(ws_ctx* ctx, const Px* grad, const Geo& g, int conn, int32_t* L, int* pending,
                              cudaStream_t st) {
  if (conn == 6) return shard_first_t<6>(ctx, grad, g, L, pending, st);
  if (conn == 26) return shard_first_t<26>(ctx, grad, g, L, pending, st);
  set_error(WS_ERR_INVALID, "the sharded path supports 6- and 26-connectivity");
  return WS_ERR_INVALID;
}

ws_status plateau_round_shard(ws_ctx* ctx, const Px* grad, const Geo& g, int conn, int32_t* L, int act_lo,
                              int act_hi, int* pending, cudaStream_t st) {
  if (conn == 6) return shard_round_t<6>(ctx, grad, g, L, act_lo, act_hi, pending, st);
  if (conn == 26) return shard_round_t<26>(ctx, grad, g, L, act_lo, act_hi, pending, st);
  set_error(WS_ERR_INVALID, "the sharded path supports 6- and 26-connectivity");
  return WS_ERR_INVALID;
}

template <int CONN>
static ws_status resolve_shard_t(ws_ctx* ctx, const Px* grad, const Geo& g, const int32_t* L, int32_t* P,
                                 cudaStream_t st) {
  const TileGrid tg = tiles_of<CONN>(g);
  Maps mp;
  make_maps<CONN>(grad, L, g, mp);
  PairOut po;
  WS_TRY(pair_out(ctx, g, po, st));
  k_resolve<CONN, false><<<tile_grid(tg.ntx, tg.nty, tg.ntz), NT, 0, st>>>(mp.mI, mp.mL, mp.tma, grad, L, g, tg.ntx, tg.nty, P, nullptr, po);
  launched(ctx, PH_WS_SELECT);
  tmark(ctx, st, PH_WS_SELECT);
  WS_CUDA(cudaGetLastError());
  return WS_OK;
}

ws_status resolve_shard(ws_ctx* ctx, const Px* grad, const Geo& g, int conn, const int32_t* L, int32_t* P,
                        cudaStream_t st) {
  if (conn == 6) return resolve_shard_t<6>(ctx, grad, g, L, P, st);
  if (conn == 26) return resolve_shard_t<26>(ctx, grad, g, L, P, st);
  set_error(WS_ERR_INVALID, "the sharded path supports 6- and 26-connectivity");
  return WS_ERR_INVALID;
}

ws_status run_watershed(ws_ctx* ctx, const Px* grad, const Geo& g, int conn, int32_t* labels,
                        int64_t* num_regions, cudaStream_t st, bool relabel, bool small) {
  switch (conn) {
    case 4: return watershed_t<4>(ctx, grad, g, labels, num_regions, st, relabel, small);
    case 8: return watershed_t<8>(ctx, grad, g, labels, num_regions, st, relabel, small);
    case 6: return watershed_t<6>(ctx, grad, g, labels, num_regions, st, relabel, small);
    case 26: return watershed_t<26>(ctx, grad, g, labels, num_regions, st, relabel, small);
  }
  set_error(WS_ERR_INVALID, "connectivity must be 4, 8, 6 or 26");
  return WS_ERR_INVALID;
}

#ifndef WS_PX16
template <int CONN>
static ws_status debug_t(ws_ctx* ctx, const Px* grad, const Geo& g, int32_t* dist, int32_t* parent,
                         cudaStream_t st) {
  WS_TRY(ctx->aux.ensure((size_t)g.N * sizeof(int), "aux"));
  int* L = ctx->aux.as<int>();
  const TileGrid tg = tiles_of<CONN>(g);
  Maps mp;
  make_maps<CONN>(grad, L, g, mp);
  WS_TRY(plateau_phase<CONN>(ctx, grad, g, L, tg, mp, st));
  k_resolve<CONN, true><<<tile_grid(tg.ntx, tg.nty, tg.ntz), NT, 0, st>>>(mp.mI, mp.mL, mp.tma, grad, L, g, tg.ntx, tg.nty, parent, dist,
                                             PairOut{nullptr, nullptr, 0});
  launched(ctx, PH_WS_SELECT);
  WS_CUDA(cudaGetLastError());
  return WS_OK;
}

ws_status run_plateau_debug(ws_ctx* ctx, const Px* grad, const Geo& g, int conn, int32_t* dist,
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

#endif  // !WS_PX16

#ifdef WS_PX16
}  // namespace px16
#endif
}  // namespace ws
