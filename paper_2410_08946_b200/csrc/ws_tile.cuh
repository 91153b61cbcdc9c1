// ws_tile.cuh — shared tile layout + TMA staging for the tile kernels (watershed, RAG).
#pragma once
#include <cstdlib>
#include <cstring>

#include "ws_internal.h"
#include "ws_tma.cuh"

namespace ws {

constexpr int NT = 256;

// Tile layout.  3-D tiles 32x8x8, 2-D tiles 64x32 (2048 voxels, 8 per thread); 4-connected 2-D
// images use 32x32 tiles (1024 voxels, 4 per thread): less padding on small images (C5's
// 145x145: 18 % instead of 46 %) and twice the CTAs on C1.
//   I box (u8 or u16 pixels):  x in [bx-16, bx+TX+16), y in [by-2, by+TY+2), z in [bz-2, bz+TZ+2) (3-D)
//   L box (i32): x in [bx-4, bx+TX+4),   y in [by-1, by+TY+1), z in [bz-1, bz+TZ+1) (3-D)
// TMA rules (measured on sm_100a): box widths AND the innermost start coordinate must be
// multiples of 16 bytes, hence the wide x halos; 2-D tiles have no halo across axis 0.
template <int CONN> struct TL {
  static constexpr bool is3d = Conn<CONN>::is3d;
  static constexpr int TX = (is3d || CONN == 4) ? 32 : 64;
  static constexpr int TY = is3d ? 8 : 32;
  static constexpr int TZ = is3d ? 8 : 1;
  static constexpr int V = TX * TY * TZ;
  static constexpr int VPT = V / NT;
  static constexpr int IXO = 16, IYO = 2, IZO = is3d ? 2 : 0;
  static constexpr int SXI = TX + 32, SYI = TY + 4, SZI = TZ + 2 * IZO, SI = SXI * SYI * SZI;
  static constexpr int LXO = 4, LYO = 1, LZO = is3d ? 1 : 0;
  static constexpr int SXL = TX + 8, SYL = TY + 2, SZL = TZ + 2 * LZO, SL = SXL * SYL * SZL;
  __device__ static constexpr int iI(int lz, int ly, int lx) { return ((lz + IZO) * SYI + ly + IYO) * SXI + lx + IXO; }
  __device__ static constexpr int iL(int lz, int ly, int lx) { return ((lz + LZO) * SYL + ly + LYO) * SXL + lx + LXO; }
  __device__ static constexpr int oI(int i) {
    int dz = 0, dy = 0, dx = 0;
    nb_delta(CONN, i, dz, dy, dx);
    return (dz * SYI + dy) * SXI + dx;
  }
  __device__ static constexpr int oL(int i) {
    int dz = 0, dy = 0, dx = 0;
    nb_delta(CONN, i, dz, dy, dx);
    return (dz * SYL + dy) * SXL + dx;
  }
  static_assert(V % NT == 0, "tile");
  static_assert((SXI % 16) == 0 && ((SXL * 4) % 16) == 0 && IXO % 16 == 0 && (LXO * 4) % 16 == 0, "TMA");
};

struct TileCoord {
  int bx, by, bz;  // global coordinates of the tile origin
};

// tiles cover the owned planes [zlo, zhi) (the whole volume when unsharded)
template <int CONN>
__device__ __forceinline__ TileCoord tile_coord(int t, int ntx, int nty, const Geo& g) {
  using T = TL<CONN>;
  TileCoord c;
  c.bx = (t % ntx) * T::TX;
  c.by = ((t / ntx) % nty) * T::TY;
  c.bz = g.zlo + (t / (ntx * nty)) * T::TZ;
  return c;
}

// Tile of this CTA.  Kernels with one CTA per tile are launched on a 3-D grid (ntx, nty, ntz)
// (tile_grid below), so the coordinates come from blockIdx without integer division; a
// volume with more than 65535 tile rows or layers falls back to a 1-D grid (gridDim.x != ntx).
// t = the linear tile index (z-major), as tile_coord's.
template <int CONN>
__device__ __forceinline__ TileCoord tile_of_block(int ntx, int nty, const Geo& g, int& t) {
  using T = TL<CONN>;
  if (gridDim.x == (unsigned)ntx) {
    t = ((int)blockIdx.z * nty + (int)blockIdx.y) * ntx + (int)blockIdx.x;
    TileCoord c;
    c.bx = (int)blockIdx.x * T::TX;
    c.by = (int)blockIdx.y * T::TY;
    c.bz = g.zlo + (int)blockIdx.z * T::TZ;
    return c;
  }
  t = (int)blockIdx.x;
  return tile_coord<CONN>(t, ntx, nty, g);
}

static inline dim3 tile_grid(int ntx, int nty, int ntz) {
  if (nty <= 65535 && ntz <= 65535) return dim3((unsigned)ntx, (unsigned)nty, (unsigned)ntz);
  return dim3((unsigned)((long long)ntx * nty * ntz));
}

// the tile and its 2-voxel halo lie inside the volume: no neighbour checks needed
template <int CONN>
__device__ __forceinline__ bool tile_interior(const TileCoord& c, const Geo& g) {
  using T = TL<CONN>;
  return c.bx >= 2 && c.bx + T::TX + 2 <= g.n2 && c.by >= 2 && c.by + T::TY + 2 <= g.n1 &&
         (!T::is3d || (c.bz >= 2 && c.bz + T::TZ + 2 <= g.n0)) &&
         c.bz + T::TZ + (g.zhi < g.n0 ? 1 : 0) <= g.zhi;  // sharded: the top layer is border
}

// voxel k of this thread inside the tile: j = threadIdx.x + k * NT (x fastest)
template <int CONN>
__device__ __forceinline__ void my_voxel(int k, int& lx, int& ly, int& lz) {
  using T = TL<CONN>;
  const int j = threadIdx.x + k * NT;
  lx = j % T::TX;
  ly = (j / T::TX) % T::TY;
  lz = j / (T::TX * T::TY);
}

// neighbour validity mask (bit i: neighbour i inside the volume) of a voxel at global coords
template <int CONN>
__device__ __forceinline__ unsigned valid_mask(const Geo& g, int gz, int gy, int gx) {
  unsigned m = 0;
#pragma unroll
  for (int i = 0; i < CONN; ++i)
    if (nb_in<CONN>(g, gz, gy, gx, i)) m |= 1u << i;
  return m;
}

// box rows [0, ROWS) of width SX starting at global (x0, y0, z0) into dst (row pitch SX),
// zero outside the volume; row r = (z - z0) * SY + (y - y0)
template <class V, int SX, int SY, int ROWS, int RB>
__device__ __forceinline__ void plain_rows(const V* __restrict__ src, const Geo& g, int x0, int y0, int z0, V* dst) {
  constexpr int CH = (SX + 31) / 32, NW = NT / 32;
  const int lane = threadIdx.x & 31;
  for (int r0 = threadIdx.x >> 5; r0 < ROWS; r0 += RB * NW) {
    V v[RB][CH];
#pragma unroll
    for (int u = 0; u < RB; ++u) {
      const int r = r0 + u * NW;
      const int gy = y0 + r % SY, gz = z0 + r / SY;
      const bool rok = r < ROWS && (unsigned)gy < (unsigned)g.n1 && (unsigned)gz < (unsigned)g.n0;
      const V* row = src + ((size_t)gz * g.plane + (size_t)gy * g.n2);
#pragma unroll
      for (int ch = 0; ch < CH; ++ch) {
        const int gx = x0 + lane + 32 * ch;
        v[u][ch] = (rok && lane + 32 * ch < SX && (unsigned)gx < (unsigned)g.n2) ? row[gx] : (V)0;
      }
    }
#pragma unroll
    for (int u = 0; u < RB; ++u) {
      const int r = r0 + u * NW;
      if (r >= ROWS) break;
#pragma unroll
      for (int ch = 0; ch < CH; ++ch)
        if (lane + 32 * ch < SX) dst[r * SX + lane + 32 * ch] = v[u][ch];
    }
  }
}

// Stage the I box (sI may be null: L box only) and optionally the L box (raw L values) into
// shared memory: one
// cp.async.bulk.tensor per box (TMA zero-fills outside the volume), or a plain loader when
// the layout has no tensor map.
template <int CONN, class Px>
__device__ __forceinline__ void stage(const CUtensorMap* mI, const CUtensorMap* mL, bool tma,
                                      const Px* __restrict__ I, const int* __restrict__ L, const Geo& g,
                                      const TileCoord& c, Px* sI, int* sL, uint64_t* bar) {
  using T = TL<CONN>;
  if (tma) {
    if (threadIdx.x == 0) mbar_init(bar, 1);
    __syncthreads();
    if (threadIdx.x == 0) {
      mbar_expect_tx(bar, (sI ? T::SI * (int)sizeof(Px) : 0) + (sL ? T::SL * 4 : 0));
      if (sI) tma_load_3d(sI, mI, c.bx - T::IXO, c.by - T::IYO, c.bz - T::IZO, bar);
      if (sL) tma_load_3d(sL, mL, c.bx - T::LXO, c.by - T::LYO, c.bz - T::LZO, bar);
    }
    mbar_wait(bar, 0);
  } else {
    // plain loader (layouts without a tensor map, e.g. rows not a multiple of 16 bytes): one
    // warp per box row, lanes along x (no per-element index division), zero fill outside;
    // 2-D tiles: 4 rows per warp at a time with all their loads issued before the shared
    // stores (small images such as C5's have no tensor map); 3-D tiles (tensor maps in
    // practice) keep the register-lean row loop
    if constexpr (!T::is3d) {
      if (sI) plain_rows<Px, T::SXI, T::SYI, T::SYI * T::SZI, 4>(I, g, c.bx - T::IXO, c.by - T::IYO, c.bz - T::IZO, sI);
      if (sL) plain_rows<int, T::SXL, T::SYL, T::SYL * T::SZL, 4>(L, g, c.bx - T::LXO, c.by - T::LYO, c.bz - T::LZO, sL);
    } else {
      const int lane = threadIdx.x & 31;
      for (int r = threadIdx.x >> 5; sI && r < T::SYI * T::SZI; r += NT / 32) {
        const int gy = c.by + r % T::SYI - T::IYO, gz = c.bz + r / T::SYI - T::IZO;
        const bool rok = (unsigned)gy < (unsigned)g.n1 && (unsigned)gz < (unsigned)g.n0;
        const Px* row = I + ((size_t)gz * g.plane + (size_t)gy * g.n2);
        for (int sx = lane; sx < T::SXI; sx += 32) {
          const int gx = c.bx + sx - T::IXO;
          sI[r * T::SXI + sx] = (rok && (unsigned)gx < (unsigned)g.n2) ? __ldg(row + gx) : (Px)0;
        }
      }
      if (sL) {
        for (int r = threadIdx.x >> 5; r < T::SYL * T::SZL; r += NT / 32) {
          const int gy = c.by + r % T::SYL - T::LYO, gz = c.bz + r / T::SYL - T::LZO;
          const bool rok = (unsigned)gy < (unsigned)g.n1 && (unsigned)gz < (unsigned)g.n0;
          const int* row = L + ((size_t)gz * g.plane + (size_t)gy * g.n2);
          for (int sx = lane; sx < T::SXL; sx += 32) {
            const int gx = c.bx + sx - T::LXO;
            sL[r * T::SXL + sx] = (rok && (unsigned)gx < (unsigned)g.n2) ? row[gx] : 0;
          }
        }
      }
    }
    __syncthreads();
  }
}


// tensor maps of one call (grad u8 box with a 2-voxel halo, L i32 box with a 1-voxel halo);
// WS_NO_TMA=1 forces the plain loader (tested for parity as well)
struct Maps {
  CUtensorMap mI, mL;
  int tma;
};

template <int CONN, class Px>
static inline void make_maps(const Px* grad, const int* L, const Geo& g, Maps& m) {
  using T = TL<CONN>;
  const char* env = getenv("WS_NO_TMA");
  const bool off = env && env[0] == '1';
  std::memset(&m, 0, sizeof(m));
  const bool a = !off && encode_tmap_3d(&m.mI, (int)sizeof(Px), grad, g, T::SXI, T::SYI, T::SZI);
  const bool b = !off && encode_tmap_3d(&m.mL, 4, L, g, T::SXL, T::SYL, T::SZL);
  m.tma = (a && b) ? 1 : 0;
}


}  // namespace ws
