// ws_common.cuh — shared device helpers of the sm_100a path (never shared with oracle/).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ws {

// Grid geometry: n0 (depth or batch) x n1 x n2, row-major (ws.h).
struct Geo {
  int n0, n1, n2;   // each < 2^31 and n0*n1*n2 < 2^31
  int plane;        // n1 * n2
  int N;
  // z-slab sharding (ws_shard_*): planes [zlo, zhi) of this (extended) volume are owned by
  // the caller, the others are read-only halo; gofs = global linear index of local voxel 0.
  // Unsharded calls: zlo = 0, zhi = n0, gofs = 0.
  int zlo, zhi;
  int gofs;
};

// ------------------------------------------------------------------------------------
// Neighbourhoods.  Index i enumerates the offsets in increasing linear-offset
// order (lexicographic (dz, dy, dx)), so "the last neighbour in scan order" is the
// max-index neighbour (Eq. 1 tie-break, C3).  The forward half (offset > 0) is
// i >= n/2 (only q > p in step IV).
// ------------------------------------------------------------------------------------
template <int CONN> struct Conn {
  static constexpr int n = CONN;
  static constexpr int nfwd = CONN / 2;
  static constexpr bool is3d = (CONN == 6 || CONN == 26);
};

__host__ __device__ constexpr void nb_delta(int conn, int i, int& dz, int& dy, int& dx) {
  if (conn == 4) {  // (0,-1,0) (0,0,-1) (0,0,1) (0,1,0)
    dz = 0; dy = (i == 0) ? -1 : (i == 3) ? 1 : 0; dx = (i == 1) ? -1 : (i == 2) ? 1 : 0;
  } else if (conn == 6) {  // (-1,0,0) (0,-1,0) (0,0,-1) (0,0,1) (0,1,0) (1,0,0)
    dz = (i == 0) ? -1 : (i == 5) ? 1 : 0;
    dy = (i == 1) ? -1 : (i == 4) ? 1 : 0;
    dx = (i == 2) ? -1 : (i == 3) ? 1 : 0;
  } else if (conn == 8) {
    int j = i < 4 ? i : i + 1;  // skip the centre of the 3x3 stencil
    dz = 0; dy = j / 3 - 1; dx = j % 3 - 1;
  } else {  // 26
    int j = i < 13 ? i : i + 1;
    dz = j / 9 - 1; dy = (j / 3) % 3 - 1; dx = j % 3 - 1;
  }
}

// linear offset of direction i
template <int CONN>
__device__ __forceinline__ int nb_off(const Geo& g, int i) {
  int dz, dy, dx;
  nb_delta(CONN, i, dz, dy, dx);
  return dz * g.plane + dy * g.n2 + dx;
}

template <int CONN>
__device__ __forceinline__ bool nb_in(const Geo& g, int z, int y, int x, int i) {
  int dz, dy, dx;
  nb_delta(CONN, i, dz, dy, dx);
  return (unsigned)(z + dz) < (unsigned)g.n0 && (unsigned)(y + dy) < (unsigned)g.n1 &&
         (unsigned)(x + dx) < (unsigned)g.n2;
}

// ------------------------------------------------------------------------------------
// Step II encoding of the label array L (int32).
//   L >= 0 : a resolved pointer (a voxel with a lower neighbour: its Eq. 1 target) or a
//            strict single-voxel minimum (L = p).  Such a voxel has plateau distance 0.
//   L <  0 : a plateau voxel without a lower neighbour, L = -1 - ((d << 5) | dir)
//            d   = BFS distance to the plateau's lower voxels (DUNREACHED = not reached,
//                  i.e. so far / finally a minimal-plateau voxel);
//            dir = chosen neighbour index (31 = none / self root).
// The paper's PRUF_bal also stores distances as negative states.
// ------------------------------------------------------------------------------------
constexpr int DIR_NONE = 31;
constexpr int DUNREACHED = (1 << 26) - 1;

__host__ __device__ __forceinline__ int enc(int d, int dir) { return -1 - ((d << 5) | dir); }
__host__ __device__ __forceinline__ int dec_d(int L) { return L >= 0 ? 0 : ((-1 - L) >> 5); }
__host__ __device__ __forceinline__ int dec_dir(int L) { return (-1 - L) & 31; }

// pointer of voxel v given its L value (decoding the step II encoding)
template <int CONN>
__device__ __forceinline__ int ptr_of(const Geo& g, int v, int Lv) {
  if (Lv >= 0) return Lv;
  int dir = dec_dir(Lv);
  return dir == DIR_NONE ? v : v + nb_off<CONN>(g, dir);
}

// ------------------------------------------------------------------------------------
// Waterfall edge key K (C14): w asc, max(a,b) desc, min(a,b) desc  as ONE u64 whose
// natural order is K: [w:8][~max:28][~min:28].  Requires dense ids < 2^28.
// ------------------------------------------------------------------------------------
constexpr uint32_t IDMASK = (1u << 28) - 1;
__host__ __device__ __forceinline__ uint64_t make_key(uint32_t w, uint32_t a, uint32_t b) {
  uint32_t hi = a > b ? a : b, lo = a > b ? b : a;
  return ((uint64_t)w << 56) | ((uint64_t)(IDMASK - hi) << 28) | (uint64_t)(IDMASK - lo);
}
__host__ __device__ __forceinline__ uint32_t key_hi(uint64_t k) { return IDMASK - (uint32_t)((k >> 28) & IDMASK); }
__host__ __device__ __forceinline__ uint32_t key_lo(uint64_t k) { return IDMASK - (uint32_t)(k & IDMASK); }
constexpr uint64_t KEY_NONE = ~0ull;

// Uncached (L2) loads for data concurrently modified by other CTAs (union-find).
__device__ __forceinline__ int ld_cg(const int* p) { return __ldcg(p); }

}  // namespace ws
