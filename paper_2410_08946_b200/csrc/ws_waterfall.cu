// ws_waterfall.cu — the graph waterfall (C13) over the region adjacency graph, sm_100a.
//
//   k_dense      dense ids: single-pass exclusive scan of [labels(p) == p] with decoupled
//                look-back (prefix-scan compaction); dense_of[label] and rep_of[dense]
//   k_rag        RAG extraction: forward neighbour pairs with different labels, height
//                max(I(p), I(q)), deduplicated per tile in a shared-memory hash with
//                u64 atomicMin on the edge key K (C14) = per-pair minimum (Alg. 4 l.2-7);
//                each unique tile edge also folds into best[] = level-1 min-K edge per region
//   k_hook       level k: every component merges along its min-K edge (min-root CAS union, C16)
//   k_flatten    level k: flatten the previous level's roots only; new root list, counts
//   k_edges      level k >= 2: re-label the live edges to current roots, drop internal ones
//                (compaction), fold the survivors into best[] (per-component min-K edge)
//   k_levelmap   per dense id: the chain comp^k(d) = its level-k root -> canonical label rows
//   k_levels     levels[k][p] = map_k[dense(labels(p))]  (Alg. 5 l.12 output, one pass)
#include <cstdio>

#include "ws_internal.h"
#include "ws_tile.cuh"

namespace ws {

constexpr int NTW = 256;

// ------------------------------------------------------------------ dense ids (scan)
constexpr int DROUND = NTW * 16;      // 4096 voxels per round, 16 consecutive per thread
constexpr int DR = 4;                 // rounds per block
constexpr int DCHUNK = DROUND * DR;   // 16384 voxels per block
constexpr uint64_t ST_AGG = 1ull << 62, ST_PRE = 2ull << 62, ST_MASK = (1ull << 62) - 1;

__device__ __forceinline__ int warp_incl_scan(int v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) >= o) v += t;
  }
  return v;
}

// block-wide exclusive scan of one int per thread (blockDim.x == NTW)
__device__ __forceinline__ int block_excl_scan(int v, int* smem, int& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int inc = warp_incl_scan(v);
  if (lane == 31) smem[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    int s = lane < NTW / 32 ? smem[lane] : 0;
    s = warp_incl_scan(s);
    if (lane < NTW / 32) smem[lane] = s;
  }
  __syncthreads();
  const int base = wid ? smem[wid - 1] : 0;
  total = smem[NTW / 32 - 1];
  __syncthreads();
  return base + inc - v;
}

// Single pass, decoupled look-back: block b (dynamic order) scans its 16384 voxels (thread
// t owns voxels 16t..16t+15 of each 4096-voxel round, so thread order = voxel order and the
// dense ids keep the canonical label order, C14), publishes its aggregate, then warp 0 looks
// back over 32 predecessors at a time until an inclusive prefix is found.
// pofs: label value of a representative at local index 0 (global index of local voxel 0);
// doff: dense id of this call's first representative (z-slab sharding; 0 / 0 otherwise);
// dense_of (sharded) is the slab's window, indexed by label - pofs.
// rk != nullptr (unsharded): instead of dense_of, the rank structure rk[w] = (dense id of the
// first representative at or after voxel 32 w, bit mask of the representatives among voxels
// 32 w .. 32 w + 31) is written: dense(l) = rk[l/32].x + popc(rk[l/32].y & ((1 << l%32) - 1)).
// It holds 8 bytes per 32 voxels, so the lookups of k_dimage stay in L2.
__global__ void __launch_bounds__(NTW) k_dense(const int* __restrict__ labels, int N, int aligned,
                                                unsigned long long* status, int* ticket, int* __restrict__ dense_of,
                                                int* __restrict__ rep_of, int rep_cap, long long* R, int pofs,
                                                int doff, uint2* __restrict__ rk, unsigned long long* depth_max,
                                                int agg_only) {
  __shared__ int sm[32];
  __shared__ int sb;
  __shared__ long long sprefix;
  if (threadIdx.x == 0) sb = atomicAdd(ticket, 1);
  __syncthreads();
  const int b = sb;
  const int lane = threadIdx.x & 31;
  uint64_t fl = 0;
  int ex[DR];
  int total = 0;
#pragma unroll
  for (int r = 0; r < DR; ++r) {
    const int p0 = b * DCHUNK + r * DROUND + threadIdx.x * 16;
    int cnt = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int p = p0 + 4 * j;
      int f0, f1, f2, f3;
      const int q = p + pofs;
      if (aligned && p + 3 < N) {
        const int4 v = __ldg(reinterpret_cast<const int4*>(labels + p));
        f0 = v.x == q; f1 = v.y == q + 1; f2 = v.z == q + 2; f3 = v.w == q + 3;
      } else {
        f0 = (p < N) && __ldg(labels + p) == q;
        f1 = (p + 1 < N) && __ldg(labels + p + 1) == q + 1;
        f2 = (p + 2 < N) && __ldg(labels + p + 2) == q + 2;
        f3 = (p + 3 < N) && __ldg(labels + p + 3) == q + 3;
      }
      const int sh = r * 16 + 4 * j;
      fl |= ((uint64_t)f0 << sh) | ((uint64_t)f1 << (sh + 1)) | ((uint64_t)f2 << (sh + 2)) | ((uint64_t)f3 << (sh + 3));
      cnt += f0 + f1 + f2 + f3;
    }
    int tot;
    ex[r] = block_excl_scan(cnt, sm, tot) + total;
    total += tot;
  }
  if (threadIdx.x < 32) {
    long long prefix = 0;
    if (b == 0) {
      if (lane == 0) atomicExch(status, ST_PRE | (unsigned long long)total);
    } else {
      if (lane == 0) atomicExch(status + b, ST_AGG | (unsigned long long)total);
      int q = b - 1;
      while (true) {
        const int idx = q - lane;
        unsigned long long s = ST_PRE;  // virtual inclusive prefix 0 before block 0
        if (idx >= 0) s = *reinterpret_cast<volatile unsigned long long*>(status + idx);
        const unsigned flag = (unsigned)(s >> 62);
        if (__any_sync(0xffffffffu, flag == 0)) continue;  // a predecessor has not published yet
        const unsigned pre = __ballot_sync(0xffffffffu, flag == 2);
        const int first = pre ? __ffs(pre) - 1 : 31;
        long long v = (lane <= first) ? (long long)(s & ST_MASK) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        prefix += v;
        if (pre) {
          if (lane == 0) atomicMax(depth_max, (unsigned long long)(b - (q - first)));  // blocks looked back
          break;
        }
        q -= 32;
      }
      // (agg_only, a test knob: keep only the aggregate published, so every successor looks
      // back to block 0 across many 32-block windows)
      if (lane == 0 && !agg_only) atomicExch(status + b, ST_PRE | (unsigned long long)(prefix + total));
    }
    if (lane == 0) {
      sprefix = prefix;
      if ((long long)(b + 1) * DCHUNK >= N) *R = prefix + total;
    }
  }
  __syncthreads();
  const int pre = (int)sprefix;
#pragma unroll
  for (int r = 0; r < DR; ++r) {
    int d = pre + ex[r];
    uint32_t m = (uint32_t)((fl >> (r * 16)) & 0xffffu);
    const int p0 = b * DCHUNK + r * DROUND + threadIdx.x * 16;
    if (rk) {  // even thread: voxels 32 w .. 32 w + 15, odd thread: the next 16
      const uint32_t mo = __shfl_down_sync(0xffffffffu, m, 1);
      if (!(threadIdx.x & 1) && p0 < N) rk[p0 >> 5] = make_uint2((unsigned)d, m | (mo << 16));
    }
    while (m) {
      const int u = __ffs(m) - 1;
      m &= m - 1;
      if (!rk) dense_of[p0 + u] = d + doff;  // sharded: the slab's window, index = label - pofs
      if (d < rep_cap) rep_of[d] = p0 + u + pofs;
      ++d;
    }
  }
}

// ------------------------------------------------------------------- dense-id image
// D[p] = dense id of labels[p] (dense_of is indexed by label).  Every later pass of the
// waterfall (RAG, level materialisation) reads D instead of labels, so no per-voxel or
// per-edge dense_of gather remains on the hot path.  Each thread maps 4 consecutive voxels;
// equal neighbours (the common case: regions are runs along x) reuse the previous gather.
// Sharded dense ids (z-slab waterfall): labels in the slab's window [lo, hi) (its own planes
// and the plane above) index the window array; the few labels below it (regions that cross
// the slab's lower cut, all listed in the gathered boundary tables) live in a small
// open-addressing map of 64-bit slots (label << 32 | dense id), empty = ~0.
struct DenseMap {
  const int* win;                   // dense id of label lo + i
  int lo, hi;
  const unsigned long long* fmap;   // foreign labels
  int fbits;                        // log2 of the map's slot count
};

__device__ __forceinline__ uint32_t fmap_hash(int l, int bits) { return ((uint32_t)l * 0x9E3779B1u) >> (32 - bits); }

__device__ __forceinline__ int dense_lookup(const DenseMap& m, int l) {
  if (l >= m.lo && l < m.hi) return __ldg(m.win + (l - m.lo));
  const uint32_t mask = (1u << m.fbits) - 1;
  for (uint32_t h = fmap_hash(l, m.fbits);; h = (h + 1) & mask) {
    const unsigned long long v = __ldg(m.fmap + h);
    if (v == ~0ull) return -1;  // not a label of this slab (never met on valid input)
    if ((int)(v >> 32) == l) return (int)(unsigned)v;
  }
}

// vec == 0 (labels or D not 16-byte aligned): scalar accesses only.
__global__ void __launch_bounds__(NTW) k_dimage(const int* __restrict__ labels, DenseMap m, long long n,
                                                 int* __restrict__ D, int vec) {
  const long long n4 = vec ? n >> 2 : 0;
  const int4* L4 = reinterpret_cast<const int4*>(labels);
  int4* D4 = reinterpret_cast<int4*>(D);
  for (long long i = blockIdx.x * (long long)NTW + threadIdx.x; i < n4; i += (long long)gridDim.x * NTW) {
    const int4 v = __ldcs(L4 + i);
    int4 d;
    d.x = dense_lookup(m, v.x);
    d.y = v.y == v.x ? d.x : dense_lookup(m, v.y);
    d.z = v.z == v.y ? d.y : dense_lookup(m, v.z);
    d.w = v.w == v.z ? d.z : dense_lookup(m, v.w);
    D4[i] = d;
  }
  for (long long p = (n4 << 2) + blockIdx.x * (long long)NTW + threadIdx.x; p < n; p += (long long)gridDim.x * NTW)
    D[p] = dense_lookup(m, labels[p]);
}

// the same from the rank structure of k_dense (unsharded calls)
__device__ __forceinline__ int rank_of(const uint2* __restrict__ rk, int l) {
  const uint2 e = __ldg(rk + (l >> 5));
  return (int)e.x + __popc(e.y & ((1u << (l & 31)) - 1u));
}

__global__ void __launch_bounds__(NTW) k_dimage_rk(const int* __restrict__ labels, const uint2* __restrict__ rk,
                                                    long long n, int* __restrict__ D, int vec) {
  const long long n4 = vec ? n >> 2 : 0;
  const int4* L4 = reinterpret_cast<const int4*>(labels);
  int4* D4 = reinterpret_cast<int4*>(D);
  for (long long i = blockIdx.x * (long long)NTW + threadIdx.x; i < n4; i += (long long)gridDim.x * NTW) {
    const int4 v = __ldcs(L4 + i);
    int4 d;
    d.x = rank_of(rk, v.x);
    d.y = v.y == v.x ? d.x : rank_of(rk, v.y);
    d.z = v.z == v.y ? d.y : rank_of(rk, v.z);
    d.w = v.w == v.z ? d.z : rank_of(rk, v.w);
    D4[i] = d;
  }
  for (long long p = (n4 << 2) + blockIdx.x * (long long)NTW + threadIdx.x; p < n; p += (long long)gridDim.x * NTW)
    D[p] = rank_of(rk, labels[p]);
}

// ------------------------------------------------------------------------ RAG extraction
// One CTA per watershed tile (ws_tile.cuh: 3-D 32x8x8, 2-D 64x32).  The dense-id box and the
// intensity box of the tile + its FORWARD halo (the neighbours q > p) land in shared
// memory with one bulk-tensor copy each.  Then:
//   1. detection: every (voxel p, forward direction f) with D(p) != D(p + f) is a boundary
//      pair; it is appended as a 16-bit record (voxel step k, lane, f) to the warp's staging
//      list with ballot + popc (uniform, no atomics, no divergent work);
//   2. dedup: every warp walks its own list with all lanes (a record's box indices are the
//      warp's base + k * step + lane), re-reads D(p), D(q) and the pass height
//      w = max(I(p), I(q)) from shared memory, and folds the pair into the tile's
//      shared hash (2048 slots, linear probing).  u8 images: one 64-bit slot holds the pair
//      AND its height, [min:28][max:28][w:8]: a CAS inserts it, and a record of a pair
//      already present lowers the height with a 32-bit atomicMin on the slot's low word
//      (whose upper 24 bits are the pair's, equal for all contenders) when its w is below
//      the one just read = the per-pair minimum pass height, Alg. 4 l.2-7.  16-bit images
//      keep the pair key and a 32-bit height in two arrays;
//   3. flush: every unique tile pair becomes its edge key K = [w:8][~max:28][~min:28] (C14),
//      is appended (block scan + one global atomic per tile; thread t owns the slots t,
//      t + NT, ..., so the slot reads are bank-conflict free) and folded into best[] (the
//      level-1 per-region min-K edge, RED atomicMin).
template <int CONN, class Px = uint8_t> struct RL {
  using T = TL<CONN>;
  static constexpr bool is3d = T::is3d;
  static constexpr int TX = T::TX, TY = T::TY, TZ = T::TZ;
  static constexpr int XA = (CONN == 8 || CONN == 26) ? 1 : 0;  // forward half reaches x-1
  static constexpr int YA = (CONN == 26) ? 1 : 0;               // ... and y-1 (across z)
  // boxes start at the tile origin (minus an aligned left margin when XA/YA)
  static constexpr int IXO = XA ? 16 : 0, LXO = XA ? 4 : 0, YO = YA;
  static constexpr int SXI = TX + 16 + IXO, SXL = TX + 4 + LXO, SY = TY + 1 + YA, SZ = is3d ? TZ + 1 : 1;
  static constexpr int SI = SXI * SY * SZ, SL = SXL * SY * SZ;
  static constexpr int HP = 2048;  // pair slots per tile (overflow -> direct global emit)
  static constexpr int HB = 11;    // log2(HP)
  static constexpr bool PACK = sizeof(Px) == 1;  // u8: pair + height in one 64-bit slot
  static constexpr int SLOT = PACK ? 8 : 12;     // bytes per slot (16-bit: key + separate height)
  static constexpr int NF = CONN - Conn<CONN>::nfwd;
  static constexpr int WALL = T::VPT * NF * 32;  // records a warp can produce
  static constexpr int WCAP = WALL < 512 ? WALL : 512;  // per-warp staging list
  static constexpr bool MIDFOLD = WALL > WCAP;           // fold inside the detection loop
  static constexpr int STG = WCAP * (NT / 32);
  __device__ static constexpr int iI(int lz, int ly, int lx) { return (lz * SY + ly + YO) * SXI + lx + IXO; }
  __device__ static constexpr int iL(int lz, int ly, int lx) { return (lz * SY + ly + YO) * SXL + lx + LXO; }
  __device__ static constexpr int oI(int i) {
    int dz = 0, dy = 0, dx = 0;
    nb_delta(CONN, i, dz, dy, dx);
    return (dz * SY + dy) * SXI + dx;
  }
  __device__ static constexpr int oL(int i) {
    int dz = 0, dy = 0, dx = 0;
    nb_delta(CONN, i, dz, dy, dx);
    return (dz * SY + dy) * SXL + dx;
  }
  static_assert((SXI % 16) == 0 && ((SXL * 4) % 16) == 0, "TMA");
  static_assert(T::VPT <= 8 && NF <= 16, "record encoding [k:3][lane:5][f:4]");
  static_assert(WCAP >= NF * 32, "staging list holds one detection step");
  static constexpr int SIA = (SI * (int)sizeof(Px) + 127) / 128 * 128;  // TMA destinations are 128-byte aligned
  static constexpr int SLA = (4 * SL + 127) / 128 * 128;
  static constexpr int SMEM = SIA + SLA + SLOT * HP + 2 * STG;
};

// global-space atomics spelled out: through a generic pointer the compiler may emit ATOM.E
// with a shared-space check (and wait for it) instead of the fire-and-forget RED
__device__ __forceinline__ void red_min_g(uint64_t* p, uint64_t v) {
  asm volatile("red.relaxed.gpu.global.min.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_add_g(unsigned long long* p, unsigned long long v) {
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long atom_add_g(unsigned long long* p, unsigned long long v) {
  unsigned long long r;
  asm volatile("atom.relaxed.gpu.global.add.u64 %0, [%1], %2;" : "=l"(r) : "l"(p), "l"(v) : "memory");
  return r;
}

__device__ __forceinline__ void fold_best(uint64_t* best, uint64_t k) {
  red_min_g(best + key_lo(k), k);
  red_min_g(best + key_hi(k), k);
}

// where the RAG's unique tile edges go (level-1 key list + best[]); emits counts the records
// that bypassed a full tile hash (ws_stats.rag_global_emits)
struct E16;
struct EdgeOut {
  uint64_t* edges;
  unsigned long long* ecount;
  long long cap;
  uint64_t* best;
  unsigned long long* emits;
  E16* e16;                  // 16-bit images: the edge list (w, ids) instead of 64-bit keys (no best[] fold)
  unsigned long long* recs;  // staged boundary records (ws_stats.rag_records), may be null
};

// A waterfall edge of a 16-bit image (ws_waterfall_u16).  K (C14) = (w asc, max desc, min
// desc) on the level-0 dense ids needs 16 + 28 + 28 bits, more than one u64 holds, so it is
// the pair (hi, lo): hi = w << 28 | (IDMASK - max), lo = IDMASK - min; per-component minima
// take two passes (hi, then lo among the edges with the minimum hi).  ca, cb: the endpoints'
// current components.
struct E16 {
  uint64_t hi;
  uint32_t lo;
  int ca, cb, pad;
};
__host__ __device__ __forceinline__ E16 make_e16(uint32_t w, uint32_t a, uint32_t b) {
  const uint32_t mx = a > b ? a : b, mn = a > b ? b : a;
  E16 e;
  e.hi = ((uint64_t)w << 28) | (uint64_t)(IDMASK - mx);
  e.lo = IDMASK - mn;
  e.ca = (int)mn;
  e.cb = (int)mx;
  e.pad = 0;
  return e;
}

__device__ __noinline__ void emit_global(uint32_t w, uint32_t a, uint32_t b, const EdgeOut& eo) {
  const unsigned long long i = atom_add_g(eo.ecount, 1ull);
  if (eo.e16) {
    if ((long long)i < eo.cap) eo.e16[i] = make_e16(w, a, b);
  } else {
    const uint64_t k = make_key(w, a, b);
    if ((long long)i < eo.cap) eo.edges[i] = k;
    fold_best(eo.best, k);
  }
  red_add_g(eo.emits, 1ull);
}

// Box indices of a warp's voxels: voxel k of lane l is D-box index wb.x + k * wb.y + l and
// I-box index wb.z + k * wb.w + l (lanes run along x inside one row of the tile).
template <int CONN, class Px>
__device__ __forceinline__ int4 warp_boxes() {
  using R = RL<CONN, Px>;
  int lx, ly, lz, lx1, ly1, lz1;
  my_voxel<CONN>(0, lx, ly, lz);
  my_voxel<CONN>(1, lx1, ly1, lz1);
  const int lane = threadIdx.x & 31;
  const int l0 = R::iL(lz, ly, lx) - lane, i0 = R::iI(lz, ly, lx) - lane;
  return make_int4(l0, R::iL(lz1, ly1, lx1) - lane - l0, i0, R::iI(lz1, ly1, lx1) - lane - i0);
}

template <int HB>
__device__ __forceinline__ uint32_t pair_hash(uint32_t lo, uint32_t hi) {
  return ((lo * 0x9E3779B1u) ^ (hi * 0x85EBCA77u)) >> (32 - HB);
}

// u8: fold one packed key [min:28][max:28][w:8] into the tile's hash
template <int HB>
__device__ __forceinline__ void fold_key(unsigned long long* pk, unsigned long long key, const EdgeOut& eo) {
  const uint32_t lo = (uint32_t)(key >> 36), hi = (uint32_t)(key >> 8) & IDMASK;
  uint32_t h = pair_hash<HB>(lo, hi);
#pragma unroll 1
  for (int probe = 0; probe < 64; ++probe) {
    unsigned long long cur = pk[h];
    if (cur == KEY_NONE) {
      cur = atomicCAS(pk + h, KEY_NONE, key);
      if (cur == KEY_NONE) return;  // inserted with this key's height
    }
    if ((cur >> 8) == (key >> 8)) {
      // same pair: lower the height (the slot's low word carries the pair's bits 0..23
      // above w, equal for every contender, so a 32-bit min on it is the min of w)
      if ((unsigned)(cur & 0xff) > ((unsigned)key & 0xff))
        atomicMin(reinterpret_cast<unsigned*>(pk + h), (unsigned)key);
      return;
    }
    h = (h + 1) & ((1u << HB) - 1);
  }
  emit_global((unsigned)key & 0xff, lo, hi, eo);  // congested tile
}

// fold one record rec = [k:3][lane:5][f:4] (re-reads the boxes).  u8: as a packed key;
// 16-bit images: key + separate height
template <int CONN, class Px>
__device__ __forceinline__ void fold_rec(unsigned rec, int4 wb, const short* offs, const Px* sI, const int* sD,
                                         unsigned long long* pk, unsigned* pw, const EdgeOut& eo) {
  using R = RL<CONN, Px>;
  const int f = rec & 15, l = (rec >> 4) & 31, k = rec >> 9;
  const int sl = wb.x + k * wb.y + l, si = wb.z + k * wb.w + l;
  const uint32_t dp = (uint32_t)sD[sl], dq = (uint32_t)sD[sl + offs[f]];
  const unsigned w = max((unsigned)sI[si], (unsigned)sI[si + offs[16 + f]]);
  const uint32_t lo = min(dp, dq), hi = max(dp, dq);
  if constexpr (R::PACK) {
    fold_key<R::HB>(pk, ((unsigned long long)lo << 36) | ((unsigned long long)hi << 8) | w, eo);
    return;
  }
  uint32_t h = pair_hash<R::HB>(lo, hi);
  const unsigned long long key = ((unsigned long long)lo << 28) | hi;
#pragma unroll 1
  for (int probe = 0; probe < 64; ++probe) {
    unsigned long long cur = pk[h];
    if (cur == KEY_NONE) cur = atomicCAS(pk + h, KEY_NONE, key);
    if (cur == KEY_NONE || cur == key) {
      atomicMin(pw + h, w);
      return;
    }
    h = (h + 1) & (R::HP - 1);
  }
  emit_global(w, dp, dq, eo);  // congested tile
}

// a warp folds its staged list
template <int CONN, class Px>
__device__ __forceinline__ void fold_warp(const uint16_t* wst, int wcnt, int4 wb, const short* offs, const Px* sI,
                                          const int* sD, unsigned long long* pk, unsigned* pw, const EdgeOut& eo) {
  for (int r = threadIdx.x & 31; r < wcnt; r += 32) fold_rec<CONN, Px>(wst[r], wb, offs, sI, sD, pk, pw, eo);
}

template <int CONN, bool BORDER, class Px>
__device__ __forceinline__ int rag_pairs(const Px* sI, const int* sD, unsigned long long* pk, unsigned* pw,
                                          uint16_t* wst, int4 wb, const short* offs, const Geo& g, const TileCoord& c,
                                          const EdgeOut& eo) {
  using R = RL<CONN, Px>;
  using T = TL<CONN>;
  constexpr int NF = R::NF;
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1;
  int wcnt = 0;
#pragma unroll
  for (int k = 0; k < T::VPT; ++k) {
    int lx, ly, lz;
    my_voxel<CONN>(k, lx, ly, lz);
    const bool own = !BORDER || (c.bx + lx < g.n2 && c.by + ly < g.n1 && c.bz + lz < g.zhi);
    const unsigned vm = !own ? 0u : (BORDER ? valid_mask<CONN>(g, c.bz + lz, c.by + ly, c.bx + lx) : (1u << CONN) - 1);
    const int sl = wb.x + k * wb.y + lane;
    const int dp = sD[sl];
#pragma unroll
    for (int f = 0; f < NF; ++f) {
      const int i = Conn<CONN>::nfwd + f;
      const bool e = ((vm >> i) & 1u) && sD[sl + R::oL(i)] != dp;
      const unsigned b = __ballot_sync(0xffffffffu, e);
      if (e) wst[wcnt + __popc(b & lt)] = (uint16_t)(f | (lane << 4) | (k << 9));
      wcnt += __popc(b);
    }
    if (R::MIDFOLD && wcnt > R::WCAP - NF * 32) {
      if (eo.recs && lane == 0) red_add_g(eo.recs, (unsigned long long)wcnt);
      __syncwarp();
      fold_warp<CONN, Px>(wst, wcnt, wb, offs, sI, sD, pk, pw, eo);
      __syncwarp();
      wcnt = 0;
    }
  }
  return wcnt;
}

template <int CONN, class Px>
__device__ __forceinline__ void rag_load_plain(const int* __restrict__ D, const Px* __restrict__ I, const Geo& g,
                                               const TileCoord& c, Px* sI, int* sD) {
  using R = RL<CONN, Px>;
  // one warp per box row, lanes along x (no per-element index division), zero fill outside
  const int lane = threadIdx.x & 31;
  for (int r = threadIdx.x >> 5; r < R::SY * R::SZ; r += NT / 32) {
    const int gy = c.by + r % R::SY - R::YO, gz = c.bz + r / R::SY;
    const bool rok = (unsigned)gy < (unsigned)g.n1 && (unsigned)gz < (unsigned)g.n0;
    const size_t ro = (size_t)gz * g.plane + (size_t)gy * g.n2;
    for (int sx = lane; sx < R::SXI; sx += 32) {
      const int gx = c.bx + sx - R::IXO;
      sI[r * R::SXI + sx] = (rok && (unsigned)gx < (unsigned)g.n2) ? __ldg(I + ro + gx) : (Px)0;
    }
    for (int sx = lane; sx < R::SXL; sx += 32) {
      const int gx = c.bx + sx - R::LXO;
      sD[r * R::SXL + sx] = (rok && (unsigned)gx < (unsigned)g.n2) ? __ldg(D + ro + gx) : 0;
    }
  }
}

// One CTA per tile t = blockIdx.x (a 1-D grid: CTAs running together hold neighbouring tiles in
// linear order, so the edge list comes out in tile order -- the level loop's per-chunk dedup
// and comp gathers depend on it -- and the best[] atomics of neighbouring CTAs share L2 lines;
// a 3-D grid measured 9.1 -> 11.2 ms).  Thread 0 decodes the tile coordinates (integer
// divisions once per CTA, not per thread) and shares them.
template <int CONN, class Px>
__global__ void __launch_bounds__(NT, 5) k_rag(const __grid_constant__ CUtensorMap mI, const __grid_constant__ CUtensorMap mD,
                                               int tma, const int* __restrict__ D, const Px* __restrict__ I, Geo g,
                                               int ntx, int nty, EdgeOut eo) {
  using R = RL<CONN, Px>;
  extern __shared__ __align__(128) unsigned char rag_smem[];
  Px* sI = reinterpret_cast<Px*>(rag_smem);                                       // R::SI pixels
  int* sD = reinterpret_cast<int*>(rag_smem + R::SIA);                            // R::SL dense ids
  unsigned long long* pk = reinterpret_cast<unsigned long long*>(rag_smem + R::SIA + R::SLA);  // R::HP slots
  unsigned* pw = reinterpret_cast<unsigned*>(pk + R::HP);    // R::HP min pass heights (16-bit images only)
  uint16_t* stg = reinterpret_cast<uint16_t*>(rag_smem + R::SIA + R::SLA + R::SLOT * R::HP);  // staged records
  __shared__ uint64_t bar;
  __shared__ unsigned long long gbase;
  __shared__ int sscan[32];
  __shared__ short offs[32];  // [f]: D-box offset, [16 + f]: I-box offset of forward direction f
  __shared__ TileCoord sc;
  if (threadIdx.x == 0) {
    const TileCoord c0 = tile_coord<CONN>((int)blockIdx.x, ntx, nty, g);
    sc = c0;
    if (tma) {
      mbar_init(&bar, 1);
      mbar_expect_tx(&bar, R::SI * (int)sizeof(Px) + R::SL * 4);
      tma_load_3d(sI, &mI, c0.bx - R::IXO, c0.by - R::YO, c0.bz, &bar);
      tma_load_3d(sD, &mD, c0.bx - R::LXO, c0.by - R::YO, c0.bz, &bar);
    }
  }
  if (threadIdx.x < R::NF) {
    offs[threadIdx.x] = (short)R::oL(Conn<CONN>::nfwd + threadIdx.x);
    offs[16 + threadIdx.x] = (short)R::oI(Conn<CONN>::nfwd + threadIdx.x);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int4 wb = warp_boxes<CONN, Px>();
  uint16_t* wst = stg + warp * R::WCAP;
#pragma unroll
  for (int i = threadIdx.x; i < R::HP; i += NT) {
    pk[i] = KEY_NONE;
    if constexpr (!R::PACK) pw[i] = 0xffffffffu;
  }
  __syncthreads();  // tile coordinates and barrier init visible; hash reset done
  const TileCoord c = sc;
  if (tma) {
    mbar_wait(&bar, 0);
  } else {
    rag_load_plain<CONN, Px>(D, I, g, c, sI, sD);
    __syncthreads();
  }
  // 1. detection into the per-warp lists
  const int n = tile_interior<CONN>(c, g) ? rag_pairs<CONN, false, Px>(sI, sD, pk, pw, wst, wb, offs, g, c, eo)
                                           : rag_pairs<CONN, true, Px>(sI, sD, pk, pw, wst, wb, offs, g, c, eo);
  // 2. dedup: every warp folds its own list
  __syncwarp();
  fold_warp<CONN, Px>(wst, n, wb, offs, sI, sD, pk, pw, eo);
  if (eo.recs && lane == 0) red_add_g(eo.recs, (unsigned long long)n);
  __syncthreads();  // hash complete
  // 3. flush: block scan of the per-thread counts, one global atomic per tile
  constexpr int M = R::HP / NT;  // thread t owns the slots t, t + NT, ... (consecutive lanes,
                                 // consecutive slots: no bank conflicts)
  int cnt = 0;
#pragma unroll
  for (int m = 0; m < M; ++m) cnt += pk[threadIdx.x + m * NT] != KEY_NONE;
  int tot;
  const int ex = block_excl_scan(cnt, sscan, tot);
  if (threadIdx.x == 0) gbase = tot ? atom_add_g(eo.ecount, (unsigned long long)tot) : 0;
  __syncthreads();
  long long i = (long long)gbase + ex;
#pragma unroll
  for (int m = 0; m < M; ++m) {
    const unsigned long long key = pk[threadIdx.x + m * NT];
    if (key == KEY_NONE) continue;
    if constexpr (R::PACK) {
      const uint64_t k = make_key((uint32_t)(key & 0xff), (uint32_t)(key >> 36), (uint32_t)(key >> 8) & IDMASK);
      if (i < eo.cap) eo.edges[i] = k;
      fold_best(eo.best, k);
    } else {
      if (i < eo.cap) eo.e16[i] = make_e16(pw[threadIdx.x + m * NT], (uint32_t)(key >> 28), (uint32_t)(key & IDMASK));
    }
    ++i;
  }
}

// ---------------------------------------------------------------------- level loop
__device__ __forceinline__ int c_find_ro(const int* c, int x) {
  while (true) {
    const int y = ld_cg(c + x);
    if (y == x) return x;
    x = y;
  }
}

__global__ void k_iota(int* a, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = i;
}

// level k: every root c of level k-1 with a min-K edge merges along it (min-root union,
// C16); best[c] is reset for the next level.  roots == nullptr: all c in [0, n).
// Finds are read-only: the chains below the previous level's roots (comp^k(d) = level-k
// root) must survive for k_levelmap, so no path halving here.
__global__ void k_hook(uint64_t* best, int* comp, const int* __restrict__ roots, int n,
                       const unsigned long long* nptr) {
  if (nptr) n = (int)*nptr;  // device-resident count of the previous level's roots
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int c = roots ? roots[i] : i;
    const uint64_t k = best[c];
    if (k == KEY_NONE) continue;  // isolated component (C17)
    best[c] = KEY_NONE;
    int a = (int)key_lo(k), b = (int)key_hi(k);
    while (true) {
      a = c_find_ro(comp, a);
      b = c_find_ro(comp, b);
      if (a == b) break;
      if (a > b) { const int t = a; a = b; b = t; }
      if (atomicCAS(comp + b, b, a) == b) break;
    }
  }
}

// Flatten the previous level's roots onto their level-k roots (read-only finds, then the
// stores; non-root entries keep pointing one level up, so comp^k(d) is d's level-k root)
// and collect the level-k roots (warp-aggregated append, smem-staged per block).
__global__ void __launch_bounds__(NTW) k_flatten(int* comp, const int* __restrict__ roots, int n,
                                                  const unsigned long long* nptr, int* __restrict__ out,
                                                  unsigned long long* nout, uint8_t* __restrict__ lvl, int level) {
  __shared__ int sbuf[2 * NTW];
  __shared__ int scount;
  __shared__ unsigned long long sbase;
  if (nptr) n = (int)*nptr;
  if (threadIdx.x == 0) scount = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  int cnt = 0;  // staged roots: block-uniform (a register, never re-read from scount)
  for (int i0 = blockIdx.x * NTW; i0 < n; i0 += gridDim.x * NTW) {
    const int i = i0 + threadIdx.x;
    int c = -1, r = -1;
    if (i < n) {
      c = roots ? roots[i] : i;
      r = c_find_ro(comp, c);
    }
    const bool isr = (i < n) && r == c;
    const unsigned rb = __ballot_sync(0xffffffffu, isr);
    if (rb) {
      int base = 0;
      if (lane == 0) base = atomicAdd(&scount, __popc(rb));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (isr) sbuf[base + __popc(rb & ((1u << lane) - 1))] = c;
    }
    cnt += __syncthreads_count(isr);
    if (i < n && r != c) {
      comp[c] = r;
      lvl[c] = (uint8_t)level;  // c stops being a root at this level
    }
    if (cnt > NTW || i0 + gridDim.x * NTW >= n) {
      if (cnt > 0) {
        if (threadIdx.x == 0) sbase = atomicAdd(nout, (unsigned long long)cnt);
        __syncthreads();
        for (int j = threadIdx.x; j < cnt; j += NTW) out[sbase + j] = sbuf[j];
      }
      __syncthreads();
      if (threadIdx.x == 0) scount = 0;
      __syncthreads();
      cnt = 0;
    }
  }
}

struct Edge {
  uint64_t k;
  int a, b;  // current component roots
};

// level k >= 2: re-label live edges to the level-(k-1) roots, drop edges inside one component,
// and deduplicate per block chunk by COMPONENT pair in a shared hash (min K per pair: only
// the lowest edge between two components can ever be picked, C14/C15).  Survivors fold into
// best[] (per-component min-K edge) and are appended (one global atomic per block).
// in_keys != nullptr: the input is the level-1 key list (endpoints decoded from K).
constexpr int ECH = 2048;  // edges per block (8 per thread)
constexpr int EHC = 2048;  // shared hash slots (>= ECH distinct pairs: probing always ends; typical load ~26%)

__global__ void __launch_bounds__(NTW) k_edges(const uint64_t* __restrict__ in_keys, const Edge* __restrict__ in,
                                                long long n, const unsigned long long* nptr,
                                                const int* __restrict__ comp, uint64_t* best, Edge* __restrict__ out,
                                                unsigned long long* nout, unsigned long long* chunks_max) {
  extern __shared__ __align__(16) unsigned long long esm[];
  unsigned long long* tp = esm;                         // component pair (lo << 32 | hi)
  unsigned* khi = reinterpret_cast<unsigned*>(esm + EHC);  // min K of the pair: high word,
  unsigned* klo = khi + EHC;                               // then low word (two 32-bit passes)
  __shared__ int sscan[32];
  __shared__ unsigned long long gbase;
  if (nptr) n = (long long)*nptr;  // device-resident count of the previous level's live edges
  constexpr int M = EHC / NTW;     // thread t owns the slots t, t + NTW, ... (no bank conflicts)
  constexpr int J = ECH / NTW;
  if (threadIdx.x == 0 && (long long)blockIdx.x * ECH < n)
    atomicMax(chunks_max, (unsigned long long)((n - 1 - (long long)blockIdx.x * ECH) / ((long long)gridDim.x * ECH) + 1));
#pragma unroll 1
  for (long long e0 = (long long)blockIdx.x * ECH; e0 < n; e0 += (long long)gridDim.x * ECH) {
    for (int i = threadIdx.x; i < EHC; i += NTW) {
      tp[i] = KEY_NONE;
      khi[i] = 0xffffffffu;
      klo[i] = 0xffffffffu;
    }
    __syncthreads();
    // all loads of the chunk first (keys, then the component gathers), then the hash: the
    // loads of a thread are independent and overlap instead of one round trip per edge
    uint64_t kk[J];
    int ca[J], cb[J];
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const long long e = e0 + threadIdx.x + j * NTW;
      kk[j] = KEY_NONE;
      ca[j] = cb[j] = 0;
      if (e < n) {
        if (in_keys) {
          kk[j] = in_keys[e];
          ca[j] = (int)key_lo(kk[j]);
          cb[j] = (int)key_hi(kk[j]);
        } else {
          const Edge ed = in[e];
          kk[j] = ed.k;
          ca[j] = ed.a;
          cb[j] = ed.b;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < J; ++j) {
      ca[j] = __ldg(comp + ca[j]);
      cb[j] = __ldg(comp + cb[j]);
    }
    // pass 1: insert the component pair, fold the high word of K (native 32-bit atomics;
    // a 64-bit shared atomicMin would be a CAS loop)
    int slot[J];
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int a = ca[j], b = cb[j];
      slot[j] = -1;
      if (kk[j] == KEY_NONE || a == b) continue;
      const uint64_t pk = ((uint64_t)(uint32_t)min(a, b) << 32) | (uint32_t)max(a, b);
      uint32_t h = (((uint32_t)(pk >> 32) * 0x9E3779B1u) ^ ((uint32_t)pk * 0x85EBCA77u)) >> 21;  // 11 bits
#pragma unroll 1
      while (true) {
        unsigned long long cur = tp[h];
        if (cur == KEY_NONE) cur = atomicCAS(tp + h, KEY_NONE, (unsigned long long)pk);
        if (cur == KEY_NONE || cur == pk) break;
        h = (h + 1) & (EHC - 1);  // at most ECH pairs in EHC slots: always terminates
      }
      slot[j] = (int)h;
      const unsigned hi = (unsigned)(kk[j] >> 32);
      if (hi < khi[h]) atomicMin(khi + h, hi);
    }
    __syncthreads();
    // pass 2: among the edges with the pair's minimum high word, the minimum low word
#pragma unroll
    for (int j = 0; j < J; ++j)
      if (slot[j] >= 0 && (unsigned)(kk[j] >> 32) == khi[slot[j]]) atomicMin(klo + slot[j], (unsigned)kk[j]);
    __syncthreads();
    int cnt = 0;
#pragma unroll
    for (int m = 0; m < M; ++m) cnt += tp[threadIdx.x + m * NTW] != KEY_NONE;
    int tot;
    const int ex = block_excl_scan(cnt, sscan, tot);
    if (threadIdx.x == 0) gbase = tot ? atomicAdd(nout, (unsigned long long)tot) : 0;
    __syncthreads();
    unsigned long long o = gbase + ex;
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const int sl = threadIdx.x + m * NTW;
      const unsigned long long pk = tp[sl];
      if (pk == KEY_NONE) continue;
      Edge ed;
      ed.k = ((uint64_t)khi[sl] << 32) | klo[sl];
      ed.a = (int)(pk >> 32);
      ed.b = (int)(pk & 0xffffffffu);
      atomicMin((unsigned long long*)(best + ed.a), (unsigned long long)ed.k);
      atomicMin((unsigned long long*)(best + ed.b), (unsigned long long)ed.k);
      out[o++] = ed;
    }
    __syncthreads();  // the chunk's hash is consumed before the next chunk resets it
  }
}

// level map rows: row(d)[k] = canonical label of d's level-k root, k = 0..NL-1 (row[0] = the
// region's own canonical label).  x stays its own root below lvl[x]; from level lvl[x] on,
// comp[x] is its root at that level.
__global__ void k_levelmap(const int* __restrict__ comp, const uint8_t* __restrict__ lvl,
                           const int* __restrict__ rep_of, int R, int NL, int stride, int* __restrict__ levelmap,
                           const unsigned long long* Rdev) {
  if (Rdev) R = (int)*Rdev;
  for (int d = blockIdx.x * blockDim.x + threadIdx.x; d < R; d += gridDim.x * blockDim.x) {
    int x = d;
    int* row = levelmap + (size_t)d * stride;
    if (stride == 4 || stride == 8) {  // the row in registers, written with 16-byte stores
      int r[8];
      r[0] = __ldg(rep_of + d);
#pragma unroll
      for (int k = 1; k < 8; ++k) {
        r[k] = 0;  // padding of the row (read by 16-byte loads)
        if (k < NL) {
          while (__ldg(lvl + x) <= k) x = __ldg(comp + x);
          r[k] = __ldg(rep_of + x);
        }
      }
      reinterpret_cast<int4*>(row)[0] = make_int4(r[0], r[1], r[2], r[3]);
      if (stride == 8) reinterpret_cast<int4*>(row)[1] = make_int4(r[4], r[5], r[6], r[7]);
      continue;
    }
    row[0] = __ldg(rep_of + d);
    for (int k = 1; k < NL; ++k) {
      while (__ldg(lvl + x) <= k) x = __ldg(comp + x);
      row[k] = __ldg(rep_of + x);
    }
    for (int k = NL; k < stride; ++k) row[k] = 0;  // padding of the row (read by 16-byte loads)
  }
}

// --------------------------------------------------------------- level materialisation
// levels[k][p] = row(D[p])[k] for k = 0..NL-1 (Alg. 5 l.12 output, all layers in one pass).
// Tiled (the watershed's 2048-voxel tiles): a region's voxels are processed together, so its
// level-map row (16/32 bytes, one sector) is fetched about once per tile.  Lanes run along x:
// only the first lane of every run of equal dense ids gathers, the others take the row by
// shuffle; along z each lane also reuses its previous row.  Level outputs are streaming
// stores (evict-first).
template <int CONN, int STRIDE>
__global__ void __launch_bounds__(NTW) k_levels(const int* __restrict__ D, const int* __restrict__ levelmap, int NL,
                                                 Geo g, int ntx, int nty, int* __restrict__ levels) {
  using T = TL<CONN>;
  int t;
  const TileCoord c = tile_of_block<CONN>(ntx, nty, g, t);
  const int lane = threadIdx.x & 31;
  const size_t N = (size_t)g.N;
  int prev_d = -1;
  int row[STRIDE];
#pragma unroll
  for (int j = 0; j < STRIDE; ++j) row[j] = 0;
#pragma unroll 1
  for (int k = 0; k < T::VPT; ++k) {
    int lx, ly, lz;
    my_voxel<CONN>(k, lx, ly, lz);
    const int gx = c.bx + lx, gy = c.by + ly, gz = c.bz + lz;
    const bool valid = gx < g.n2 && gy < g.n1 && gz < g.n0;
    const size_t p = (size_t)gz * g.plane + (size_t)gy * g.n2 + gx;
    const int d = valid ? __ldcs(D + p) : -1 - lane;
    const int dup = __shfl_up_sync(0xffffffffu, d, 1);
    const bool head = (lane == 0 || dup != d);
    const bool fetch = valid && head && d != prev_d;
    if (fetch) {
      const int* m = levelmap + (size_t)d * STRIDE;
#pragma unroll
      for (int j = 0; j < STRIDE; j += 4) {
        const int4 v = __ldg(reinterpret_cast<const int4*>(m + j));
        row[j] = v.x; row[j + 1] = v.y; row[j + 2] = v.z; row[j + 3] = v.w;
      }
    }
    const unsigned heads = __ballot_sync(0xffffffffu, head);
    const int src = 31 - __clz(heads & (0xffffffffu >> (31 - lane)));
#pragma unroll
    for (int j = 0; j < STRIDE; ++j) row[j] = __shfl_sync(0xffffffffu, row[j], src);
    prev_d = d;
    if (valid) {
#pragma unroll
      for (int j = 0; j < STRIDE; ++j)
        if (j < NL) __stcs(levels + (size_t)j * N + p, row[j]);
    }
  }
}

// scalar variant for large NL (stride not specialised)
__global__ void k_levels_any(const int* __restrict__ D, const int* __restrict__ levelmap, int NL, int stride,
                             long long N, int* __restrict__ levels) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < N; p += (long long)gridDim.x * blockDim.x) {
    const int* m = levelmap + (size_t)__ldg(D + p) * stride;
    for (int k = 0; k < NL; ++k) levels[(size_t)k * N + p] = __ldg(m + k);
  }
}

// --------------------------------------------------------------------------- driver
template <int CONN, class Px>
static ws_status rag_t(const int* D, const Px* I, const Geo& g, const EdgeOut& eo, cudaStream_t st) {
  using T = TL<CONN>;
  using R = RL<CONN, Px>;
  const int ntx = (g.n2 + T::TX - 1) / T::TX, nty = (g.n1 + T::TY - 1) / T::TY,
            ntz = (g.zhi - g.zlo + T::TZ - 1) / T::TZ;
  Maps mp;
  std::memset(&mp, 0, sizeof(mp));
  const char* env = getenv("WS_NO_TMA");
  const bool off = env && env[0] == '1';
  const bool a = !off && encode_tmap_3d(&mp.mI, (int)sizeof(Px), I, g, R::SXI, R::SY, R::SZ);
  const bool b = !off && encode_tmap_3d(&mp.mL, 4, D, g, R::SXL, R::SY, R::SZ);
  mp.tma = (a && b) ? 1 : 0;
  // one tile per CTA (a persistent grid interleaves distant tiles in the edge list and
  // measured slower overall)
  const int grid = ntx * nty * ntz;
  WS_CUDA(cudaFuncSetAttribute(k_rag<CONN, Px>, cudaFuncAttributeMaxDynamicSharedMemorySize, R::SMEM));
  k_rag<CONN, Px><<<grid, NT, R::SMEM, st>>>(mp.mI, mp.mL, mp.tma, D, I, g, ntx, nty, eo);
  WS_CUDA(cudaGetLastError());
  return WS_OK;
}

template <class Px>
static ws_status rag(int conn, const int* D, const Px* I, const Geo& g, const EdgeOut& eo, cudaStream_t st) {
  switch (conn) {
    case 4: return rag_t<4, Px>(D, I, g, eo, st);
    case 8: return rag_t<8, Px>(D, I, g, eo, st);
    case 6: return rag_t<6, Px>(D, I, g, eo, st);
    case 26: return rag_t<26, Px>(D, I, g, eo, st);
  }
  return WS_ERR_INVALID;
}

static int grid_for(long long n, int sms, int per_sm = 16) {
  long long b = (n + 255) / 256;
  long long cap = (long long)sms * per_sm;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

static ws_status read_i64(ws_ctx* ctx, const void* dptr, int64_t* out, cudaStream_t st) {
  WS_CUDA(cudaMemcpyAsync(ctx->pinned, dptr, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  WS_CUDA(cudaStreamSynchronize(st));
  *out = ctx->pinned[0];
  return WS_OK;
}

// dense ids of the representatives among n labels starting at global index pofs
static ws_status wf_dense(ws_ctx* ctx, const int32_t* labels, int n, int pofs, int doff, int* dense_of,
                          int64_t* count, cudaStream_t st, uint2* rk = nullptr) {
  const int nb = (n + DCHUNK - 1) / DCHUNK;
  if (!ctx->pathc.p) {
    WS_TRY(ctx->pathc.ensure(4 * sizeof(unsigned long long), "path counters"));
    WS_CUDA(cudaMemsetAsync(ctx->pathc.p, 0, 4 * sizeof(unsigned long long), st));
  }
  WS_TRY(ctx->blockcnt.ensure((size_t)nb * sizeof(unsigned long long), "scan status"));
  char* fl = ctx->flags.as<char>();
  long long* dR = reinterpret_cast<long long*>(fl + 128);
  int* ticket = reinterpret_cast<int*>(fl + 148);
  size_t rep_cap = ctx->rep_of.bytes / sizeof(int);
  if (rep_cap < (size_t)n / 16 + 1024) {
    WS_TRY(ctx->rep_of.ensure(((size_t)n / 16 + 1024) * sizeof(int), "rep_of"));
    rep_cap = ctx->rep_of.bytes / sizeof(int);
  }
  const char* knob = getenv("WS_TEST_LOOKBACK");  // test only: force look-backs to block 0
  const int agg_only = knob && knob[0] == '1';
  for (int attempt = 0; attempt < 2; ++attempt) {
    WS_CUDA(cudaMemsetAsync(ctx->blockcnt.p, 0, (size_t)nb * sizeof(unsigned long long), st));
    WS_CUDA(cudaMemsetAsync(ticket, 0, sizeof(int), st));
    k_dense<<<nb, NTW, 0, st>>>(labels, n, !(reinterpret_cast<uintptr_t>(labels) & 15),
                                ctx->blockcnt.as<unsigned long long>(), ticket, dense_of, ctx->rep_of.as<int>(),
                                (int)rep_cap, dR, pofs, doff, rk, ctx->pathc.as<unsigned long long>(), agg_only);
    launched(ctx, PH_WF_DENSE);
    WS_TRY(read_i64(ctx, dR, count, st));
    if ((size_t)*count <= rep_cap) break;
    WS_TRY(ctx->rep_of.ensure((size_t)*count * sizeof(int), "rep_of"));
    rep_cap = ctx->rep_of.bytes / sizeof(int);
  }
  tmark(ctx, st, PH_WF_DENSE);
  return WS_OK;
}

// device-resident level counters (ctx->lvcount): [k] = roots after level k, [LVC + k] = live
// edges entering level k (k < LVC); the level loop runs without host round trips
constexpr int LVC = 64;

// level-loop buffers for R regions; best[] = KEY_NONE, comp = iota, lvl = 0xFF
static ws_status wf_alloc(ws_ctx* ctx, int64_t R, int NL, cudaStream_t st) {
  if (R > (long long)IDMASK) {
    set_error(WS_ERR_LIMIT, "ws_waterfall: %lld regions exceed the 2^28-1 edge-key limit", (long long)R);
    return WS_ERR_LIMIT;
  }
  if (R < 1) {
    set_error(WS_ERR_INVALID, "ws_waterfall: labels are not a canonical labelling (no representative)");
    return WS_ERR_INVALID;
  }
  const int stride = NL <= 4 ? 4 : (NL <= 8 ? 8 : NL);  // row = canonical label at levels 0..NL-1
  WS_TRY(ctx->comp.ensure((size_t)R * sizeof(int), "comp"));
  WS_TRY(ctx->best.ensure((size_t)R * sizeof(uint64_t), "best"));
  WS_TRY(ctx->levelmap.ensure((size_t)R * stride * sizeof(int), "levelmap"));
  WS_TRY(ctx->rootsA.ensure((size_t)R * sizeof(int), "level roots A"));
  WS_TRY(ctx->rootsB.ensure((size_t)R * sizeof(int), "level roots B"));
  WS_TRY(ctx->lvl.ensure((size_t)R, "demotion levels"));
  WS_TRY(ctx->lvcount.ensure(2 * LVC * sizeof(unsigned long long), "level counters"));
  WS_CUDA(cudaMemsetAsync(ctx->lvcount.p, 0, 2 * LVC * sizeof(unsigned long long), st));
  WS_CUDA(cudaMemsetAsync(ctx->best.p, 0xFF, (size_t)R * sizeof(uint64_t), st));
  WS_CUDA(cudaMemsetAsync(ctx->lvl.p, 0xFF, (size_t)R, st));
  k_iota<<<grid_for(R, ctx->num_sms), 256, 0, st>>>(ctx->comp.as<int>(), (int)R);
  launched(ctx, PH_WF_LEVELS);
  ctx->wf.R = R;
  ctx->wf.Rdev = nullptr;
  ctx->wf.NL = NL;
  ctx->wf.stride = stride;
  return WS_OK;
}

// RAG edges of the owned planes, tile-deduplicated, folded into best[] (level-1 minima).
// First the dense-id image D of the owned planes and the plane above (the forward halo) is
// written into ctx->dimg (same layout as labels).
// Px = u16 (ws_waterfall_u16): the unique tile edges go to ctx->edges as E16 records (no
// best[] fold; the u16 level loop takes its minima in two passes).
template <class Px = uint8_t>
static ws_status wf_rag(ws_ctx* ctx, const int32_t* labels, const Px* I, const Geo& g, int conn,
                        const int* dense_of, cudaStream_t st, const uint2* rk = nullptr, bool small = false) {
  constexpr size_t ESZ = sizeof(Px) == 1 ? sizeof(uint64_t) : sizeof(E16);
  unsigned long long* ecount = reinterpret_cast<unsigned long long*>(ctx->flags.as<char>() + 136);
  unsigned long long* pathc = ctx->pathc.as<unsigned long long>();
  WS_TRY(ctx->dimg.ensure((size_t)g.N * sizeof(int), "dense-id image"));
  int* D = ctx->dimg.as<int>();
  if (!labels) {  // ws_segment: the relabel pass already wrote D
    ctx->wf.dofs = 0;
  } else {
    const int z1 = g.zhi < g.n0 ? g.zhi + 1 : g.zhi;
    const size_t o = (size_t)g.zlo * g.plane;
    const long long n = (long long)(z1 - g.zlo) * g.plane;
    const bool al = !(reinterpret_cast<uintptr_t>(labels + o) & 15) && !(reinterpret_cast<uintptr_t>(D + o) & 15);
    if (rk) {  // unsharded: the rank structure of k_dense
      k_dimage_rk<<<grid_for(al ? n / 4 + 1 : n, ctx->num_sms), NTW, 0, st>>>(labels + o, rk, n, D + o, al ? 1 : 0);
    } else {
      const DenseMap m{dense_of, ctx->wf.dlo, ctx->wf.dhi, ctx->fmap.as<unsigned long long>(), ctx->wf.fbits};
      k_dimage<<<grid_for(al ? n / 4 + 1 : n, ctx->num_sms), NTW, 0, st>>>(labels + o, m, n, D + o, al ? 1 : 0);
    }
    launched(ctx, PH_WF_DENSE);
    ctx->wf.dofs = (long long)o;
  }
  tmark(ctx, st, PH_WF_DENSE);
  const long long own = (long long)(g.zhi - g.zlo) * g.plane;
  long long cap = (long long)(ctx->edges.bytes / ESZ);
  // small (sync-free ws_segment): every boundary record fits, the count stays on the device
  const long long want = small ? own * (conn - conn / 2) + 4096 : own / 4 + 4096;
  if (cap < want) {
    WS_TRY(ctx->edges.ensure((size_t)want * ESZ, "edges"));
    cap = want;
  }
  // The edge count of a congested input varies slightly from run to run (tiles whose pair
  // hash overflows emit their records directly), so a retry gets headroom and repeats until
  // the list fits; best[] is reset before every repeat.
  int64_t E = 0;
  for (int attempt = 0;; ++attempt) {
    WS_CUDA(cudaMemsetAsync(ecount, 0, sizeof(unsigned long long), st));
    WS_CUDA(cudaMemsetAsync(pathc + 2, 0, 2 * sizeof(unsigned long long), st));
    WS_TRY(rag<Px>(conn, D, I, g,
                   EdgeOut{ctx->edges.as<uint64_t>(), ecount, cap, ctx->best.as<uint64_t>(), pathc + 2,
                           sizeof(Px) == 1 ? nullptr : ctx->edges.as<E16>(), pathc + 3}, st));
    launched(ctx, PH_WF_RAG);
    if (small) {
      E = cap;  // a bound; k_edges reads the count from ecount
      break;
    }
    WS_TRY(read_i64(ctx, ecount, &E, st));
    if (E <= cap) break;
    if (attempt >= 4) {
      set_error(WS_ERR_INTERNAL, "ws_waterfall: edge list does not fit after %d attempts", attempt + 1);
      return WS_ERR_INTERNAL;
    }
    cap = E + E / 4 + 4096;
    WS_TRY(ctx->edges.ensure((size_t)cap * ESZ, "edges"));
    WS_CUDA(cudaMemsetAsync(ctx->best.p, 0xFF, (size_t)ctx->wf.R * sizeof(uint64_t), st));
  }
  tmark(ctx, st, PH_WF_RAG);
  ctx->stats.n_edges = E;
  ctx->stats.n_regions = ctx->wf.R;
  constexpr size_t LSZ = sizeof(Px) == 1 ? sizeof(Edge) : sizeof(E16);
  WS_TRY(ctx->ebufA.ensure((size_t)(E > 0 ? E : 1) * LSZ, "edge buffer A"));
  WS_TRY(ctx->ebufB.ensure((size_t)(E > 0 ? E : 1) * LSZ, "edge buffer B"));
  ctx->wf.E = E;
  ctx->wf.ne_in = E;
  ctx->wf.nr_in = ctx->wf.R;
  ctx->wf.prev = ctx->wf.R;
  ctx->wf.lv = 0;
  ctx->wf.k = 1;
  ctx->wf.eflip = 0;
  ctx->wf.rflip = -1;  // level 1 hooks every region
  ctx->wf.Edev = small ? ecount : nullptr;
  return WS_OK;
}

// Level k = ctx->wf.k: hook + flatten (+ the live edges of level k + 1 when `edges_next`).
// Counts stay on the device; nothing here synchronises.
static ws_status wf_level(ws_ctx* ctx, bool edges_next, cudaStream_t st) {
  WSState& w = ctx->wf;
  const int k = w.k;
  unsigned long long* cnt = ctx->lvcount.as<unsigned long long>();
  int* comp = ctx->comp.as<int>();
  uint64_t* best = ctx->best.as<uint64_t>();
  int* rA = ctx->rootsA.as<int>();
  int* rB = ctx->rootsB.as<int>();
  int* rin = w.rflip < 0 ? nullptr : (w.rflip == 0 ? rA : rB);
  int* rout = (w.rflip == 0) ? rB : rA;
  const unsigned long long* nin = rin ? cnt + (k - 1) : w.Rdev;  // level 1: all R regions
  k_hook<<<grid_for(w.R, ctx->num_sms), 256, 0, st>>>(best, comp, rin, (int)w.R, nin);
  k_flatten<<<grid_for(w.R, ctx->num_sms, 8), NTW, 0, st>>>(comp, rin, (int)w.R, nin, rout, cnt + k,
                                                             ctx->lvl.as<uint8_t>(), k);
  launched(ctx, PH_WF_LEVELS, 2);
  w.rflip = (rout == rA) ? 0 : 1;
  w.k = k + 1;
  if (!edges_next || k + 1 >= LVC) return WS_OK;
  // level k + 1 minima from the live edges (level 2 reads the level-1 key list)
  Edge* ein = (k == 1) ? nullptr : (w.eflip == 0 ? ctx->ebufB.as<Edge>() : ctx->ebufA.as<Edge>());
  Edge* eout = (w.eflip == 0) ? ctx->ebufA.as<Edge>() : ctx->ebufB.as<Edge>();
  if (w.E > 0) {
    const int esmem = EHC * 16;
    WS_CUDA(cudaFuncSetAttribute(k_edges, cudaFuncAttributeMaxDynamicSharedMemorySize, esmem));
    // one wave of resident CTAs walking the chunks (no partial last wave)
    int& occ = ctx->edges_occ;  // per context (per device), computed once
    if (!occ) WS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_edges, NTW, esmem));
    const long long chunks = (w.E + ECH - 1) / ECH;
    const int grid = (int)std::min<long long>(chunks, (long long)ctx->num_sms * std::max(1, occ));
    k_edges<<<grid, NTW, esmem, st>>>(k == 1 ? ctx->edges.as<uint64_t>() : nullptr, ein, w.E,
                                      k == 1 ? w.Edev : cnt + LVC + k, comp, best, eout, cnt + LVC + k + 1,
                                      ctx->pathc.as<unsigned long long>() + 1);
    launched(ctx, PH_WF_LEVELS);
  }
  w.eflip = 1 - w.eflip;  // eout becomes the next input
  return WS_OK;
}

// host copy of the device level counters of levels 1..k_last; region counts, the last level
// that merged, per-level edge counts
static ws_status wf_read_counts(ws_ctx* ctx, int k_last, int64_t* counts, cudaStream_t st) {
  WSState& w = ctx->wf;
  static_assert(2 * LVC <= 256, "pinned scratch");
  WS_CUDA(cudaMemcpyAsync(ctx->pinned, ctx->lvcount.p, 2 * LVC * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                          st));
  WS_CUDA(cudaMemcpyAsync(ctx->pinned + 2 * LVC, ctx->pathc.p, 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                          st));
  WS_CUDA(cudaStreamSynchronize(st));
  const unsigned long long* h = reinterpret_cast<const unsigned long long*>(ctx->pinned);
  ctx->stats.lookback_max = (int32_t)h[2 * LVC];
  ctx->stats.edge_chunks_max = (int32_t)h[2 * LVC + 1];
  ctx->stats.rag_global_emits = (int64_t)h[2 * LVC + 2];
  ctx->stats.rag_records = (int64_t)h[2 * LVC + 3];
  long long prev = w.R;
  for (int k = 1; k <= k_last && k < LVC; ++k) {
    const long long c = (long long)h[k];
    if (c < prev) w.lv = k;
    prev = c;
    if (counts) counts[k] = c;
    if (k < 16) ctx->stats.level_counts[k] = c;
    if (k >= 2 && k < 16) ctx->stats.level_edges[k] = (long long)h[LVC + k];
  }
  w.prev = prev;
  return WS_OK;
}

// sharded level step (ws_shard_wf_step): best[] holds all ranks' minima; the count of the
// level is read back (the host decides whether another level follows)
static ws_status wf_step(ws_ctx* ctx, int64_t* count, int* more, cudaStream_t st) {
  WSState& w = ctx->wf;
  const int k = w.k;
  if (k >= LVC) {
    set_error(WS_ERR_LIMIT, "ws_waterfall: more than %d levels", LVC - 1);
    return WS_ERR_LIMIT;
  }
  const long long prev = k == 1 ? w.R : w.prev;
  WS_TRY(wf_level(ctx, k + 1 < w.NL, st));
  int64_t c[LVC] = {};
  WS_TRY(wf_read_counts(ctx, k, c, st));
  *count = c[k];
  *more = (k + 1 < w.NL && c[k] > 1 && c[k] < prev) ? 1 : 0;
  return WS_OK;
}

// level maps (replicated) + level arrays of the voxels of the dense-id image D (n0 planes of g)
static ws_status wf_finish(ws_ctx* ctx, const int32_t* D, const Geo& g, int conn, int32_t* levels, cudaStream_t st) {
  WSState& w = ctx->wf;
  const int NL = w.NL, stride = w.stride;
  ctx->stats.waterfall_levels = w.lv;
  int* levelmap = ctx->levelmap.as<int>();
  k_levelmap<<<grid_for(w.R, ctx->num_sms), 256, 0, st>>>(ctx->comp.as<int>(), ctx->lvl.as<uint8_t>(),
                                                           ctx->rep_of.as<int>(), (int)w.R, NL, stride, levelmap,
                                                           w.Rdev);
  launched(ctx, PH_WF_LEVELS);
  tmark(ctx, st, PH_WF_LEVELS);
  const int N = g.N;
  const int gN = grid_for(N, ctx->num_sms);
  // (a linear 4-voxels-per-thread variant with 16-byte stores measured 6.0 vs 4.7 ms on C4:
  // the tiled kernel shares each gathered row across the lanes of a run and along z)
  if (stride == 4 || stride == 8) {
    const bool is3d = (conn == 6 || conn == 26);
    const int TX = is3d ? TL<6>::TX : TL<4>::TX, TY = is3d ? TL<6>::TY : TL<4>::TY, TZ = is3d ? TL<6>::TZ : TL<4>::TZ;
    const int ntx = (g.n2 + TX - 1) / TX, nty = (g.n1 + TY - 1) / TY, ntz = (g.zhi - g.zlo + TZ - 1) / TZ;
    if (is3d && stride == 4) k_levels<6, 4><<<tile_grid(ntx, nty, ntz), NTW, 0, st>>>(D, levelmap, NL, g, ntx, nty, levels);
    else if (is3d) k_levels<6, 8><<<tile_grid(ntx, nty, ntz), NTW, 0, st>>>(D, levelmap, NL, g, ntx, nty, levels);
    else if (stride == 4) k_levels<4, 4><<<tile_grid(ntx, nty, ntz), NTW, 0, st>>>(D, levelmap, NL, g, ntx, nty, levels);
    else k_levels<4, 8><<<tile_grid(ntx, nty, ntz), NTW, 0, st>>>(D, levelmap, NL, g, ntx, nty, levels);
  } else {
    k_levels_any<<<gN, NTW, 0, st>>>(D, levelmap, NL, stride, N, levels);
  }
  launched(ctx, PH_WF_MATERIALISE);
  tmark(ctx, st, PH_WF_MATERIALISE);
  WS_CUDA(cudaGetLastError());
  return WS_OK;
}

ws_status run_waterfall(ws_ctx* ctx, const int32_t* labels, const uint8_t* I, const Geo& g, int conn, int NL,
                        int32_t* levels, int64_t* counts, cudaStream_t st) {
  if (NL > LVC) {
    set_error(WS_ERR_LIMIT, "ws_waterfall: NL must be <= %d", LVC);
    return WS_ERR_LIMIT;
  }
  WS_TRY(ctx->flags.ensure(256, "flags"));
  WS_TRY(ctx->aux.ensure((size_t)g.N * sizeof(int), "aux"));
  WS_TRY(ctx->pathc.ensure(4 * sizeof(unsigned long long), "path counters"));
  WS_CUDA(cudaMemsetAsync(ctx->pathc.p, 0, 4 * sizeof(unsigned long long), st));
  int* dense_of = ctx->aux.as<int>();
  int64_t R = 0;
  WS_TRY(ctx->rank.ensure(((size_t)g.N / 32 + 1) * sizeof(uint2), "dense rank structure"));
  uint2* rk = ctx->rank.as<uint2>();
  WS_TRY(wf_dense(ctx, labels, g.N, 0, 0, dense_of, &R, st, rk));
  WS_TRY(wf_alloc(ctx, R, NL, st));
  WS_TRY(wf_rag(ctx, labels, I, g, conn, dense_of, st, rk));
  if (counts) counts[0] = R;
  ctx->stats.level_counts[0] = R;
  ctx->stats.level_edges[1] = ctx->wf.E;
  // all levels are enqueued back to back (a level without merges leaves everything as is);
  // the counts are read once, after the level arrays are enqueued
  for (int k = 1; k < NL; ++k) WS_TRY(wf_level(ctx, k + 1 < NL, st));
  WS_TRY(wf_finish(ctx, ctx->dimg.as<int>(), g, conn, levels, st));
  if (NL > 1) WS_TRY(wf_read_counts(ctx, NL - 1, counts, st));
  ctx->stats.waterfall_levels = ctx->wf.lv;
  return WS_OK;
}

// exclusive scan of the nb block counts in place (one block); total -> bc[nb]
__global__ void __launch_bounds__(NTW) k_scan_counts(int* bc, int nb) {
  __shared__ int sm[32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int b0 = 0; b0 < nb; b0 += NTW) {
    const int i = b0 + threadIdx.x;
    const int v = i < nb ? bc[i] : 0;
    int tot;
    const int ex = block_excl_scan(v, sm, tot);
    if (i < nb) bc[i] = carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) bc[nb] = carry;
}

// ------------------------------------------------------ ws_segment (watershed + waterfall)
// One procedure, as Alg. 5: the watershed stops before its relabel pass, the
// dense ids come from the root list instead of a scan over the labels, and ONE relabel pass
// writes the dense-id image D; k_levels then writes all NL levels from the level-map rows:
//   (watershed) k_root_canon / k_root_store set bit c of the representative bitmap for the
//               canonical label c of every listed root (C7)
//   k_rank_sum / k_scan_counts / k_rank_write   reduce-then-scan over the N/32 bitmap words:
//               rk[w] = (reps before voxel 32 w, bits of word w) -> dense(c) = rank of c
//               (dense ids keep the canonical label order, C14)
//   k_relabel_seg D[p] = dense id of p's region (= rank of its canonical label in the
//               bitmap); the representative voxels write rep_of[dense] = canonical label
// then the RAG, the level loop and k_levels exactly as ws_waterfall.
constexpr int RKW = 16;            // bitmap words per thread
constexpr int RKB = NTW * RKW;     // words per block

__global__ void __launch_bounds__(NTW) k_rank_sum(const unsigned* __restrict__ bits, int nw, int* __restrict__ bsum) {
  __shared__ int sm[32];
  const int w0 = blockIdx.x * RKB + threadIdx.x * RKW;
  int c = 0;
#pragma unroll
  for (int j = 0; j < RKW; ++j)
    if (w0 + j < nw) c += __popc(__ldg(bits + w0 + j));
  int tot;
  block_excl_scan(c, sm, tot);
  if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(NTW) k_rank_write(const unsigned* __restrict__ bits, int nw,
                                                    const int* __restrict__ bsum, uint2* __restrict__ rk) {
  __shared__ int sm[32];
  const int w0 = blockIdx.x * RKB + threadIdx.x * RKW;
  unsigned v[RKW];
  int c = 0;
#pragma unroll
  for (int j = 0; j < RKW; ++j) {
    v[j] = w0 + j < nw ? __ldg(bits + w0 + j) : 0u;
    c += __popc(v[j]);
  }
  int tot;
  int base = bsum[blockIdx.x] + block_excl_scan(c, sm, tot);
#pragma unroll
  for (int j = 0; j < RKW; ++j) {
    if (w0 + j < nw) rk[w0 + j] = make_uint2((unsigned)base, v[j]);
    base += __popc(v[j]);
  }
}

// 4 consecutive voxels per thread.  P[p] = t >= 0 (a listed root) or -1 - canonical label (p
// listed); d = rank of the canonical label c in the bitmap (one P and one rk gather per run
// of equal roots; c lies a few planes behind p, so the rk window stays in L2).  The
// representative voxel p == c also writes rep_of[d] = c.
__device__ __forceinline__ int seg_canon(const int* __restrict__ P, int t) { return -1 - (t < 0 ? t : __ldg(P + t)); }

__global__ void __launch_bounds__(NTW) k_relabel_seg(const int* __restrict__ P, const uint2* __restrict__ rk, int N,
                                                     int* __restrict__ D, int* __restrict__ rep_of) {
  const int n4 = N >> 2;
  const int4* P4 = reinterpret_cast<const int4*>(P);
  for (int i = blockIdx.x * NTW + threadIdx.x; i < n4; i += gridDim.x * NTW) {
    const int4 t = __ldg(P4 + i);  // not evict-first: the root entries it gathers share these lines
    const int p = 4 * i;
    int4 c, d;
    c.x = seg_canon(P, t.x);
    c.y = (t.y == t.x && t.x >= 0) ? c.x : seg_canon(P, t.y);
    c.z = (t.z == t.y && t.y >= 0) ? c.y : seg_canon(P, t.z);
    c.w = (t.w == t.z && t.z >= 0) ? c.z : seg_canon(P, t.w);
    d.x = rank_of(rk, c.x);
    d.y = c.y == c.x ? d.x : rank_of(rk, c.y);
    d.z = c.z == c.y ? d.y : rank_of(rk, c.z);
    d.w = c.w == c.z ? d.z : rank_of(rk, c.w);
    __stcs(reinterpret_cast<int4*>(D) + i, d);  // evict-first: keep L2 for the root gathers of P
    if (c.x == p) rep_of[d.x] = p;
    if (c.y == p + 1) rep_of[d.y] = p + 1;
    if (c.z == p + 2) rep_of[d.z] = p + 2;
    if (c.w == p + 3) rep_of[d.w] = p + 3;
  }
  for (int p = 4 * n4 + blockIdx.x * NTW + threadIdx.x; p < N; p += gridDim.x * NTW) {
    const int c = seg_canon(P, P[p]);
    const int d = rank_of(rk, c);
    D[p] = d;
    if (c == p) rep_of[d] = p;
  }
}

__global__ void k_store_count(const int* __restrict__ src, unsigned long long* dst) { *dst = (unsigned long long)*src; }

static void begin_call_stats(ws_ctx* ctx, const Geo& g) {
  std::memset(&ctx->stats, 0, sizeof(ctx->stats));
  ctx->stats.n_voxels = g.N;
}

// Inputs small enough that every list can be sized from N (the sync-free mode of ws_segment:
// no host round trip until the final counts; a list that still overflowed is caught by the
// final read, and the call then reruns on the regular path)
static bool segment_small(const Geo& g, int conn) {
  const char* e = getenv("WS_NO_SMALL");
  if (e && e[0] == '1') return false;
  const long long nf = conn - conn / 2;
  return (long long)g.N * nf <= (1ll << 27);
}

static ws_status seg_small_finish(ws_ctx* ctx, const uint8_t* I, const Geo& g, int conn, int NL, int32_t* levels,
                                  int64_t* counts, cudaStream_t st);

// enqueue == true (small only): stop after enqueuing the final device-to-host copies (no
// synchronisation: the sequence can be captured as a graph); seg_small_finish reads them
static ws_status run_segment_impl(ws_ctx* ctx, const uint8_t* I, const Geo& g, int conn, int NL, int32_t* levels,
                                  int64_t* counts, cudaStream_t st, bool small, bool enqueue = false) {
  // steps I-IV: every voxel points at a listed root, listed roots hold -1 - canonical label,
  // the representative bitmap is set
  WS_TRY(run_watershed(ctx, I, g, conn, levels, nullptr, st, false, small));
  const int* P = ctx->aux.as<int>();
  WS_TRY(ctx->flags.ensure(256, "flags"));
  WS_TRY(ctx->pathc.ensure(4 * sizeof(unsigned long long), "path counters"));
  WS_CUDA(cudaMemsetAsync(ctx->pathc.p, 0, 4 * sizeof(unsigned long long), st));
  const int nw = g.N / 32 + 1;
  const int nb = (nw + RKB - 1) / RKB;
  WS_TRY(ctx->rank.ensure((size_t)nw * sizeof(uint2), "dense rank structure"));
  WS_TRY(ctx->blockcnt.ensure((size_t)(nb + 1) * sizeof(int), "rank block sums"));
  const unsigned* bits = ctx->repbits.as<unsigned>();
  int* bsum = ctx->blockcnt.as<int>();
  uint2* rk = ctx->rank.as<uint2>();
  k_rank_sum<<<nb, NTW, 0, st>>>(bits, nw, bsum);
  k_scan_counts<<<1, NTW, 0, st>>>(bsum, nb);
  k_rank_write<<<nb, NTW, 0, st>>>(bits, nw, bsum, rk);
  launched(ctx, PH_WF_DENSE, 3);
  int64_t R;
  if (small) {
    R = g.N;  // a bound: the level loop reads R from the device
    WS_TRY(wf_alloc(ctx, R, NL, st));
    unsigned long long* Rd = ctx->lvcount.as<unsigned long long>();  // slot 0 (levels use 1..)
    k_store_count<<<1, 1, 0, st>>>(bsum + nb, Rd);
    launched(ctx, PH_WF_DENSE);
    ctx->wf.Rdev = Rd;
  } else {
    WS_CUDA(cudaMemcpyAsync(ctx->pinned, bsum + nb, sizeof(int), cudaMemcpyDeviceToHost, st));
    WS_CUDA(cudaStreamSynchronize(st));
    R = reinterpret_cast<const int*>(ctx->pinned)[0];
    ctx->stats.n_regions = R;
    WS_TRY(wf_alloc(ctx, R, NL, st));
  }
  WS_TRY(ctx->rep_of.ensure((size_t)R * sizeof(int), "rep_of"));
  WS_TRY(ctx->dimg.ensure((size_t)g.N * sizeof(int), "dense-id image"));
  int* D = ctx->dimg.as<int>();
  tmark(ctx, st, PH_WF_DENSE);
  k_relabel_seg<<<grid_for(g.N / 4 + 1, ctx->num_sms), NTW, 0, st>>>(P, rk, g.N, D, ctx->rep_of.as<int>());
  launched(ctx, PH_WS_RELABEL);
  tmark(ctx, st, PH_WS_RELABEL);
  const unsigned long long* Rdev = ctx->wf.Rdev;
  WS_TRY(wf_rag<uint8_t>(ctx, nullptr, I, g, conn, nullptr, st, nullptr, small));
  ctx->wf.Rdev = Rdev;
  for (int k = 1; k < NL; ++k) WS_TRY(wf_level(ctx, k + 1 < NL, st));
  WS_TRY(wf_finish(ctx, D, g, conn, levels, st));
  if (!small) {
    if (counts) counts[0] = R;
    ctx->stats.level_counts[0] = R;
    ctx->stats.level_edges[1] = ctx->wf.E;
    if (NL > 1) WS_TRY(wf_read_counts(ctx, NL - 1, counts, st));
    ctx->stats.waterfall_levels = ctx->wf.lv;
    return WS_OK;
  }
  // the one host read of the sync-free mode: flags (step II depth limit, pair count, rounds,
  // edge count), R, the level counters and the code-path counters
  char* hp = reinterpret_cast<char*>(ctx->pinned);
  WS_CUDA(cudaMemcpyAsync(hp, ctx->flags.p, 256, cudaMemcpyDeviceToHost, st));
  WS_CUDA(cudaMemcpyAsync(hp + 256, ctx->lvcount.p, 2 * LVC * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  WS_CUDA(cudaMemcpyAsync(hp + 256 + 2 * LVC * 8, ctx->pathc.p, 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                          st));
  if (enqueue) return WS_OK;
  return seg_small_finish(ctx, I, g, conn, NL, levels, counts, st);
}

static ws_status seg_small_finish(ws_ctx* ctx, const uint8_t* I, const Geo& g, int conn, int NL, int32_t* levels,
                                  int64_t* counts, cudaStream_t st) {
  WS_CUDA(cudaStreamSynchronize(st));
  const char* hp = reinterpret_cast<const char*>(ctx->pinned);
  int64_t R;
  const int* fi = reinterpret_cast<const int*>(hp);
  const unsigned long long* lv = reinterpret_cast<const unsigned long long*>(hp + 256);
  const unsigned long long* pc = reinterpret_cast<const unsigned long long*>(hp + 256 + 2 * LVC * 8);
  if (fi[1]) {
    set_error(WS_ERR_LIMIT, "a non-minimal plateau is deeper than 2^26-2 voxels");
    return WS_ERR_LIMIT;
  }
  const long long npairs = fi[10], pcap = (long long)(ctx->upairs.bytes / sizeof(int2));
  const unsigned long long E = *reinterpret_cast<const unsigned long long*>(hp + 136);
  if (npairs > pcap || (long long)E > ctx->wf.E) return run_segment_impl(ctx, I, g, conn, NL, levels, counts, st, false);
  R = (int64_t)lv[0];
  ctx->stats.n_regions = R;
  ctx->stats.n_edges = (int64_t)E;
  if (ctx->stats.plateau_rounds < 0) ctx->stats.plateau_rounds = 1 + fi[24];  // the cooperative rounds
  ctx->stats.level_counts[0] = R;
  ctx->stats.level_edges[1] = (int64_t)E;
  ctx->stats.edge_chunks_max = (int32_t)pc[1];
  ctx->stats.rag_global_emits = (int64_t)pc[2];
  ctx->stats.rag_records = (int64_t)pc[3];
  if (counts) counts[0] = R;
  long long prev = R;
  ctx->wf.lv = 0;
  for (int k = 1; k < NL && k < LVC; ++k) {
    const long long c = (long long)lv[k];
    if (c < prev) ctx->wf.lv = k;
    prev = c;
    if (counts) counts[k] = c;
    if (k < 16) ctx->stats.level_counts[k] = c;
    if (k >= 2 && k < 16) ctx->stats.level_edges[k] = (long long)lv[LVC + k];
  }
  ctx->wf.prev = prev;
  ctx->stats.waterfall_levels = ctx->wf.lv;
  return WS_OK;
}

ws_status run_segment(ws_ctx* ctx, const uint8_t* I, const Geo& g, int conn, int NL, int32_t* levels,
                      int64_t* counts, cudaStream_t st) {
  if (NL > LVC) {
    set_error(WS_ERR_LIMIT, "ws_segment: NL must be <= %d", LVC);
    return WS_ERR_LIMIT;
  }
  if ((reinterpret_cast<uintptr_t>(levels) & 15) != 0) {
    set_error(WS_ERR_INVALID, "ws_segment: levels must be 16-byte aligned");
    return WS_ERR_INVALID;
  }
  const bool small = segment_small(g, conn) && ctx->coop;
  if (!small) return run_segment_impl(ctx, I, g, conn, NL, levels, counts, st, false);
  // small: replay the captured call while the arguments stay the same; capture it on the
  // second call with these arguments (the first one sized every workspace buffer, so the
  // capture allocates nothing); per-phase timing keeps the direct path
  ws_ctx::SegGraph& G = ctx->sg;
  const bool same = G.I == I && G.levels == levels && G.st == st && G.n0 == g.n0 && G.n1 == g.n1 &&
                    G.n2 == g.n2 && G.conn == conn && G.NL == NL && G.last_call == ctx->calls - 1;
  const char* ng = getenv("WS_NO_GRAPH");
  const bool graphs = !(ng && ng[0] == '1') && !ctx->timing && !G.failed;
  if (!same) {
    if (G.exec) cudaGraphExecDestroy(G.exec);
    G = ws_ctx::SegGraph();
    G.I = I;
    G.levels = levels;
    G.st = st;
    G.n0 = g.n0;
    G.n1 = g.n1;
    G.n2 = g.n2;
    G.conn = conn;
    G.NL = NL;
  }
  G.last_call = ctx->calls;
  if (graphs && G.exec) {
    WS_CUDA(cudaGraphLaunch(G.exec, st));
    ctx->stats.kernel_launches = G.launches;
    ctx->stats.plateau_rounds = -1;
    ctx->stats.union_order = 0;
    ctx->total_launches += G.launches;
    return seg_small_finish(ctx, I, g, conn, NL, levels, counts, st);
  }
  if (graphs && G.seen >= 1) {
    cudaGraph_t graph = nullptr;
    const int64_t l0 = ctx->stats.kernel_launches;
    if (!ctx->cap_st) cudaStreamCreateWithFlags(&ctx->cap_st, cudaStreamNonBlocking);
    const cudaError_t eb = ctx->cap_st ? cudaStreamBeginCapture(ctx->cap_st, cudaStreamCaptureModeRelaxed)
                                       : cudaErrorInvalidResourceHandle;
    if (eb == cudaSuccess) {
      const ws_status s = run_segment_impl(ctx, I, g, conn, NL, levels, counts, ctx->cap_st, true, true);
      const cudaError_t e = cudaStreamEndCapture(ctx->cap_st, &graph);
      if (getenv("WS_DEBUG_GRAPH"))
        fprintf(stderr, "ws_segment capture: status %d (%s) end %s\n", (int)s, ws_last_error(), cudaGetErrorString(e));
      if (s == WS_OK && e == cudaSuccess && graph &&
          cudaGraphInstantiate(&G.exec, graph, 0) == cudaSuccess) {
        cudaGraphDestroy(graph);
        G.launches = ctx->stats.kernel_launches - l0;
        WS_CUDA(cudaGraphLaunch(G.exec, st));
        return seg_small_finish(ctx, I, g, conn, NL, levels, counts, st);
      }
      if (graph) cudaGraphDestroy(graph);
    }
    if (getenv("WS_DEBUG_GRAPH")) fprintf(stderr, "ws_segment capture failed (begin %s)\n", cudaGetErrorString(eb));
    (void)cudaGetLastError();  // capture unsupported here: stay on the direct path
    G.exec = nullptr;
    G.failed = 1;
    begin_call_stats(ctx, g);
  }
  ++G.seen;
  return run_segment_impl(ctx, I, g, conn, NL, levels, counts, st, true);
}

// ------------------------------------------------- 16-bit waterfall (ws_waterfall_u16)
// Level k = 1..NL-1 on the E16 list of level k-1 (level 1: the RAG list, endpoints = dense
// ids): k_e16_live re-labels both endpoints to the current components (one comp hop: the
// previous level's roots were flattened onto their new roots), drops internal edges, appends
// the survivors and folds hi into best[c]; k_e16_lo folds lo among the edges whose hi is the
// component's minimum; k_hook16 merges every component along (hi, lo) = its min-K edge (C14,
// min-root union C16); k_flatten as for u8.  Counts stay on the device.
__global__ void __launch_bounds__(NTW) k_e16_live(const E16* __restrict__ in, long long n,
                                                   const unsigned long long* nptr, const int* __restrict__ comp,
                                                   uint64_t* best_hi, E16* __restrict__ out, unsigned long long* nout) {
  if (nptr) n = (long long)*nptr;
  const int lane = threadIdx.x & 31;
  for (long long i0 = blockIdx.x * (long long)NTW; i0 < n; i0 += (long long)gridDim.x * NTW) {
    const long long i = i0 + threadIdx.x;
    E16 e;
    bool live = false;
    if (i < n) {
      e = in[i];
      e.ca = __ldg(comp + e.ca);
      e.cb = __ldg(comp + e.cb);
      live = e.ca != e.cb;
    }
    const unsigned b = __ballot_sync(0xffffffffu, live);
    if (!b) continue;
    unsigned long long base = 0;
    if (lane == __ffs(b) - 1) base = atomicAdd(nout, (unsigned long long)__popc(b));
    base = __shfl_sync(0xffffffffu, base, __ffs(b) - 1);
    if (live) {
      out[base + __popc(b & ((1u << lane) - 1))] = e;
      atomicMin((unsigned long long*)(best_hi + e.ca), (unsigned long long)e.hi);
      atomicMin((unsigned long long*)(best_hi + e.cb), (unsigned long long)e.hi);
    }
  }
}

__global__ void __launch_bounds__(NTW) k_e16_lo(const E16* __restrict__ list, const unsigned long long* nptr,
                                                 const uint64_t* __restrict__ best_hi, unsigned* best_lo) {
  const long long n = (long long)*nptr;
  for (long long i = blockIdx.x * (long long)NTW + threadIdx.x; i < n; i += (long long)gridDim.x * NTW) {
    const E16 e = list[i];
    if (__ldcg(reinterpret_cast<const unsigned long long*>(best_hi) + e.ca) == e.hi) atomicMin(best_lo + e.ca, e.lo);
    if (__ldcg(reinterpret_cast<const unsigned long long*>(best_hi) + e.cb) == e.hi) atomicMin(best_lo + e.cb, e.lo);
  }
}

__global__ void k_hook16(uint64_t* best_hi, unsigned* best_lo, int* comp, const int* __restrict__ roots, int n,
                         const unsigned long long* nptr) {
  if (nptr) n = (int)*nptr;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int c = roots ? roots[i] : i;
    const uint64_t hi = best_hi[c];
    if (hi == KEY_NONE) continue;  // isolated component (C17)
    const unsigned lo = best_lo[c];
    best_hi[c] = KEY_NONE;
    best_lo[c] = 0xffffffffu;
    int a = (int)(IDMASK - lo), b = (int)(IDMASK - (uint32_t)(hi & IDMASK));
    while (true) {
      a = c_find_ro(comp, a);
      b = c_find_ro(comp, b);
      if (a == b) break;
      if (a > b) { const int t = a; a = b; b = t; }
      if (atomicCAS(comp + b, b, a) == b) break;
    }
  }
}

ws_status run_waterfall_u16(ws_ctx* ctx, const int32_t* labels, const uint16_t* I, const Geo& g, int conn, int NL,
                            int32_t* levels, int64_t* counts, cudaStream_t st) {
  if (NL > LVC) {
    set_error(WS_ERR_LIMIT, "ws_waterfall_u16: NL must be <= %d", LVC);
    return WS_ERR_LIMIT;
  }
  WS_TRY(ctx->flags.ensure(256, "flags"));
  WS_TRY(ctx->aux.ensure((size_t)g.N * sizeof(int), "aux"));
  WS_TRY(ctx->pathc.ensure(4 * sizeof(unsigned long long), "path counters"));
  WS_CUDA(cudaMemsetAsync(ctx->pathc.p, 0, 4 * sizeof(unsigned long long), st));
  int64_t R = 0;
  WS_TRY(ctx->rank.ensure(((size_t)g.N / 32 + 1) * sizeof(uint2), "dense rank structure"));
  uint2* rk = ctx->rank.as<uint2>();
  WS_TRY(wf_dense(ctx, labels, g.N, 0, 0, ctx->aux.as<int>(), &R, st, rk));
  WS_TRY(wf_alloc(ctx, R, NL, st));
  WS_TRY(ctx->best_lo.ensure((size_t)R * sizeof(unsigned), "best lo"));
  WS_CUDA(cudaMemsetAsync(ctx->best_lo.p, 0xFF, (size_t)R * sizeof(unsigned), st));
  WS_TRY(wf_rag<uint16_t>(ctx, labels, I, g, conn, nullptr, st, rk));
  if (counts) counts[0] = R;
  ctx->stats.level_counts[0] = R;
  ctx->stats.level_edges[1] = ctx->wf.E;
  WSState& w = ctx->wf;
  unsigned long long* cnt = ctx->lvcount.as<unsigned long long>();
  int* comp = ctx->comp.as<int>();
  uint64_t* best_hi = ctx->best.as<uint64_t>();
  unsigned* best_lo = ctx->best_lo.as<unsigned>();
  int* rA = ctx->rootsA.as<int>();
  int* rB = ctx->rootsB.as<int>();
  const E16* ein = ctx->edges.as<E16>();
  const int ge = grid_for(w.E, ctx->num_sms, 8);
  for (int k = 1; k < NL; ++k) {
    E16* eout = (k & 1) ? ctx->ebufA.as<E16>() : ctx->ebufB.as<E16>();
    int* rin = k == 1 ? nullptr : ((k & 1) ? rB : rA);  // roots of level k-1 (level 1: all R)
    int* rout = (k & 1) ? rA : rB;
    const unsigned long long* nin = k == 1 ? nullptr : cnt + (k - 1);
    k_e16_live<<<ge, NTW, 0, st>>>(ein, w.E, k == 1 ? nullptr : cnt + LVC + k - 1, comp, best_hi, eout,
                                   cnt + LVC + k);
    k_e16_lo<<<ge, NTW, 0, st>>>(eout, cnt + LVC + k, best_hi, best_lo);
    k_hook16<<<grid_for(R, ctx->num_sms), 256, 0, st>>>(best_hi, best_lo, comp, rin, (int)R, nin);
    k_flatten<<<grid_for(R, ctx->num_sms, 8), NTW, 0, st>>>(comp, rin, (int)R, nin, rout, cnt + k,
                                                           ctx->lvl.as<uint8_t>(), k);
    launched(ctx, PH_WF_LEVELS, 4);
    ein = eout;
  }
  WS_CUDA(cudaGetLastError());
  WS_TRY(wf_finish(ctx, ctx->dimg.as<int>(), g, conn, levels, st));
  if (NL > 1) WS_TRY(wf_read_counts(ctx, NL - 1, counts, st));
  for (int k = 1; k < NL && k < 16; ++k) ctx->stats.level_edges[k] = (long long)reinterpret_cast<const unsigned long long*>(ctx->pinned)[LVC + k];
  ctx->stats.waterfall_levels = ctx->wf.lv;
  return WS_OK;
}

// ------------------------------------------------------------- z-slab sharded waterfall
// boundary dense table: for the first/last owned plane, (label, dense id if the label's
// representative is owned here else -1); every region crossing a cut crosses its owner's
// boundary plane, so the gathered tables give every rank the dense id of every foreign label
__global__ void k_wf_btable(const int* __restrict__ labels_own, int nplanes, int plane, int pofs_lo, int pofs_hi,
                            const int* __restrict__ dense_of, int* out) {
  for (int i = blockIdx.x * NTW + threadIdx.x; i < 2 * plane; i += gridDim.x * NTW) {
    const int s = i / plane, xy = i % plane;
    const int z = s == 0 ? 0 : nplanes - 1;
    const int l = labels_own[(size_t)z * plane + xy];
    out[i] = l;
    out[2 * plane + i] = (l >= pofs_lo && l < pofs_hi) ? dense_of[l - pofs_lo] : -1;
  }
}

// every gathered (label, dense id) with a dense id: into the slab's window, or into the
// foreign map if below it (a label of a region crossing the lower cut); others are not met here
__global__ void k_wf_bfill(const int* __restrict__ tabs, int K, int plane, int* win, int lo, int hi,
                           unsigned long long* fmap, int fbits) {
  const long long n = (long long)K * 2 * plane;
  const uint32_t mask = (1u << fbits) - 1;
  for (long long i = blockIdx.x * (long long)NTW + threadIdx.x; i < n; i += (long long)gridDim.x * NTW) {
    const long long r = i / (2 * plane), j = i % (2 * plane);
    const int* t = tabs + r * 4 * plane;
    const int d = t[2 * plane + j];
    if (d < 0) continue;
    const int l = t[j];
    if (l >= lo && l < hi) {
      win[l - lo] = d;
    } else if (l < lo) {
      const unsigned long long v = ((unsigned long long)(unsigned)l << 32) | (unsigned)d;
      for (uint32_t h = fmap_hash(l, fbits);; h = (h + 1) & mask) {
        const unsigned long long cur = atomicCAS(fmap + h, ~0ull, v);
        if (cur == ~0ull || (int)(cur >> 32) == l) break;  // inserted / already there (same d)
      }
    }
  }
}

ws_status shard_wf_dense(ws_ctx* ctx, const int32_t* labels_own, int n, int pofs, int doff, int* dense_of,
                         int* rep_of_global, int64_t* count, cudaStream_t st) {
  WS_TRY(ctx->flags.ensure(256, "flags"));
  WS_TRY(ctx->pathc.ensure(4 * sizeof(unsigned long long), "path counters"));
  WS_CUDA(cudaMemsetAsync(ctx->pathc.p, 0, 4 * sizeof(unsigned long long), st));
  WS_TRY(wf_dense(ctx, labels_own, n, pofs, doff, dense_of, count, st));
  if (*count > 0)
    WS_CUDA(cudaMemcpyAsync(rep_of_global + doff, ctx->rep_of.p, (size_t)*count * sizeof(int),
                            cudaMemcpyDeviceToDevice, st));
  return WS_OK;
}

ws_status shard_wf_btable(ws_ctx* ctx, const int32_t* labels_own, int nplanes, int plane, int pofs, const int* dense_of,
                          int32_t* out, cudaStream_t st) {
  k_wf_btable<<<grid_for(2LL * plane, ctx->num_sms), NTW, 0, st>>>(labels_own, nplanes, plane, pofs,
                                                                   pofs + nplanes * plane, dense_of, out);
  launched(ctx, PH_WF_DENSE);
  WS_CUDA(cudaGetLastError());
  return WS_OK;
}

ws_status shard_wf_bfill(ws_ctx* ctx, const int32_t* tabs, int K, int plane, int lo, int hi, int* dense_of,
                         cudaStream_t st) {
  int bits = 4;
  while ((1ll << bits) < 4ll * plane) ++bits;  // 2 planes of foreign labels at most, load <= 1/2
  WS_TRY(ctx->fmap.ensure(((size_t)1 << bits) * sizeof(unsigned long long), "foreign dense-id map"));
  WS_CUDA(cudaMemsetAsync(ctx->fmap.p, 0xFF, ((size_t)1 << bits) * sizeof(unsigned long long), st));
  ctx->wf.dlo = lo;
  ctx->wf.dhi = hi;
  ctx->wf.fbits = bits;
  k_wf_bfill<<<grid_for((long long)K * 2 * plane, ctx->num_sms), NTW, 0, st>>>(tabs, K, plane, dense_of, lo, hi,
                                                                              ctx->fmap.as<unsigned long long>(), bits);
  launched(ctx, PH_WF_DENSE);
  WS_CUDA(cudaGetLastError());
  return WS_OK;
}

// keys leave / enter the library sign-flipped (K ^ 2^63): the order of K as int64, so the
// transport's all_reduce(MIN) on int64 is the per-component minimum
__global__ void k_flip_copy(uint64_t* dst, const uint64_t* __restrict__ src, long long n) {
  for (long long i = blockIdx.x * (long long)NTW + threadIdx.x; i < n; i += (long long)gridDim.x * NTW)
    dst[i] = src[i] ^ (1ull << 63);
}

ws_status shard_wf_begin(ws_ctx* ctx, const int32_t* labels_ext, const uint8_t* I_ext, const Geo& g, int conn,
                         const int* dense_of, int64_t R, int NL, uint64_t* best_out, cudaStream_t st) {
  WS_TRY(ctx->flags.ensure(256, "flags"));
  WS_TRY(wf_alloc(ctx, R, NL, st));
  WS_TRY(wf_rag(ctx, labels_ext, I_ext, g, conn, dense_of, st));
  ctx->stats.level_counts[0] = R;
  ctx->stats.level_edges[1] = ctx->wf.E;
  k_flip_copy<<<grid_for(R, ctx->num_sms), NTW, 0, st>>>(best_out, ctx->best.as<uint64_t>(), R);
  WS_CUDA(cudaGetLastError());
  return WS_OK;
}

// Sharded levels exchange only the minima of the CURRENT roots, in increasing dense-id order
// (every rank holds the same replicated union-find, so the order is the same on all ranks):
// level 1 = all R regions (identity), then the roots of each level, compacted by a
// deterministic scan over comp (comp[c] == c <=> c is a root).
constexpr int SCH = 2048;  // entries per compaction block

__global__ void __launch_bounds__(NTW) k_root_count(const int* __restrict__ comp, int R, int* __restrict__ bc) {
  const int b0 = blockIdx.x * SCH;
  int c = 0;
  for (int i = b0 + threadIdx.x; i < min(b0 + SCH, R); i += NTW) c += comp[i] == i;
  __shared__ int sm[32];
  int tot;
  block_excl_scan(c, sm, tot);
  if (threadIdx.x == 0) bc[blockIdx.x] = tot;
}

// sorted roots and the flipped minima of this rank at them
__global__ void __launch_bounds__(NTW) k_root_scatter(const int* __restrict__ comp, int R, const int* __restrict__ bc,
                                                       int* __restrict__ sroots, uint64_t* __restrict__ best_out,
                                                       const uint64_t* __restrict__ best) {
  const int b0 = blockIdx.x * SCH;
  __shared__ int sm[32];
  int base = bc[blockIdx.x];
  for (int i0 = b0; i0 < min(b0 + SCH, R); i0 += NTW) {
    const int i = i0 + threadIdx.x;
    const bool r = i < R && comp[i] == i;
    int tot;
    const int ex = block_excl_scan(r ? 1 : 0, sm, tot);
    if (r) {
      sroots[base + ex] = i;
      best_out[base + ex] = best[i] ^ (1ull << 63);
    }
    base += tot;
  }
}

__global__ void k_best_scatter(uint64_t* best, const int* __restrict__ sroots, const uint64_t* __restrict__ best_in,
                               int n) {
  for (int i = blockIdx.x * NTW + threadIdx.x; i < n; i += gridDim.x * NTW) best[sroots[i]] = best_in[i] ^ (1ull << 63);
}

ws_status shard_wf_step(ws_ctx* ctx, const uint64_t* best_in, uint64_t* best_out, int64_t* count, int* more,
                        cudaStream_t st) {
  const long long R = ctx->wf.R;
  WS_TRY(ctx->sroots.ensure((size_t)R * sizeof(int), "sorted level roots"));
  const int nb = (int)((R + SCH - 1) / SCH);
  WS_TRY(ctx->sblocks.ensure((size_t)(nb + 1) * sizeof(int), "root compaction counts"));
  int* sr = ctx->sroots.as<int>();
  if (ctx->wf.k == 1) {  // level 1: the minima of all R regions, in dense-id order
    k_flip_copy<<<grid_for(R, ctx->num_sms), NTW, 0, st>>>(ctx->best.as<uint64_t>(), best_in, R);
  } else {
    const int n = (int)ctx->wf.sorted_n;
    if (n > 0) k_best_scatter<<<grid_for(n, ctx->num_sms), NTW, 0, st>>>(ctx->best.as<uint64_t>(), sr, best_in, n);
  }
  WS_TRY(wf_step(ctx, count, more, st));
  if (*more) {
    int* bc = ctx->sblocks.as<int>();
    k_root_count<<<nb, NTW, 0, st>>>(ctx->comp.as<int>(), (int)R, bc);
    k_scan_counts<<<1, NTW, 0, st>>>(bc, nb);
    k_root_scatter<<<nb, NTW, 0, st>>>(ctx->comp.as<int>(), (int)R, bc, sr, best_out, ctx->best.as<uint64_t>());
    launched(ctx, PH_WF_LEVELS, 3);
    ctx->wf.sorted_n = *count;  // the roots of this level are the next level's components
  }
  WS_CUDA(cudaGetLastError());
  return WS_OK;
}

// ---------------------------------------- z-slab sharded 16-bit waterfall (u16 sharding)
// The per-component minimum of K = (hi, lo) (make_e16) is reduced over the ranks in two
// steps per level, as on one GPU: the minimum hi of every component (all ranks' live edges,
// all_reduce MIN), then the minimum lo among the edges with that hi (all_reduce MIN); both
// travel sign-flipped (x ^ top bit) so unsigned order is the transport's signed order.  The
// union-find over dense ids is replicated (k_hook16 / k_flatten on every rank, same result).
__global__ void k_flip32(unsigned* a, long long n) {
  for (long long i = blockIdx.x * (long long)NTW + threadIdx.x; i < n; i += (long long)gridDim.x * NTW)
    a[i] ^= 0x80000000u;
}

ws_status shard_wf16_begin(ws_ctx* ctx, const int32_t* labels_ext, const uint16_t* I_ext, const Geo& g, int conn,
                           const int* dense_of, int64_t R, int NL, cudaStream_t st) {
  if (NL > LVC) {
    set_error(WS_ERR_LIMIT, "ws_waterfall_u16: NL must be <= %d", LVC);
    return WS_ERR_LIMIT;
  }
  WS_TRY(ctx->flags.ensure(256, "flags"));
  WS_TRY(ctx->pathc.ensure(4 * sizeof(unsigned long long), "path counters"));
  WS_CUDA(cudaMemsetAsync(ctx->pathc.p, 0, 4 * sizeof(unsigned long long), st));
  WS_TRY(wf_alloc(ctx, R, NL, st));
  WS_TRY(ctx->best_lo.ensure((size_t)R * sizeof(unsigned), "best lo"));
  WS_CUDA(cudaMemsetAsync(ctx->best_lo.p, 0xFF, (size_t)R * sizeof(unsigned), st));
  WS_TRY(wf_rag<uint16_t>(ctx, labels_ext, I_ext, g, conn, dense_of, st));
  ctx->stats.level_counts[0] = R;
  ctx->stats.level_edges[1] = ctx->wf.E;
  return WS_OK;
}

// level k = ctx->wf.k, step 0: live edges + local minimum hi, flipped for the reduction
// (exchange buffer: ctx->best, R x i64); step 1: local minimum lo among the edges with the
// reduced hi, flipped (ctx->best_lo, R x i32); step 2: hook + flatten, *count = components
// after the level (host)
ws_status shard_wf16_level(ws_ctx* ctx, int step, int64_t* count, cudaStream_t st) {
  WSState& w = ctx->wf;
  const int k = w.k;
  const int64_t R = w.R;
  unsigned long long* cnt = ctx->lvcount.as<unsigned long long>();
  uint64_t* best_hi = ctx->best.as<uint64_t>();
  unsigned* best_lo = ctx->best_lo.as<unsigned>();
  E16* eout = (k & 1) ? ctx->ebufA.as<E16>() : ctx->ebufB.as<E16>();
  const int ge = grid_for(std::max<int64_t>(w.E, 1), ctx->num_sms, 8);
  if (step == 0) {
    const E16* ein = k == 1 ? ctx->edges.as<E16>() : ((k & 1) ? ctx->ebufB.as<E16>() : ctx->ebufA.as<E16>());
    k_e16_live<<<ge, NTW, 0, st>>>(ein, w.E, k == 1 ? nullptr : cnt + LVC + k - 1, ctx->comp.as<int>(), best_hi, eout,
                                   cnt + LVC + k);
    k_flip_copy<<<grid_for(R, ctx->num_sms), NTW, 0, st>>>(best_hi, best_hi, R);
    launched(ctx, PH_WF_LEVELS, 2);
  } else if (step == 1) {
    k_flip_copy<<<grid_for(R, ctx->num_sms), NTW, 0, st>>>(best_hi, best_hi, R);
    k_e16_lo<<<ge, NTW, 0, st>>>(eout, cnt + LVC + k, best_hi, best_lo);
    k_flip32<<<grid_for(R, ctx->num_sms), NTW, 0, st>>>(best_lo, R);
    launched(ctx, PH_WF_LEVELS, 3);
  } else {
    k_flip32<<<grid_for(R, ctx->num_sms), NTW, 0, st>>>(best_lo, R);
    int* rA = ctx->rootsA.as<int>();
    int* rB = ctx->rootsB.as<int>();
    int* rin = k == 1 ? nullptr : ((k & 1) ? rB : rA);  // roots of level k-1 (level 1: all R)
    int* rout = (k & 1) ? rA : rB;
    const unsigned long long* nin = k == 1 ? nullptr : cnt + (k - 1);
    k_hook16<<<grid_for(R, ctx->num_sms), 256, 0, st>>>(best_hi, best_lo, ctx->comp.as<int>(), rin, (int)R, nin);
    k_flatten<<<grid_for(R, ctx->num_sms, 8), NTW, 0, st>>>(ctx->comp.as<int>(), rin, (int)R, nin, rout, cnt + k,
                                                           ctx->lvl.as<uint8_t>(), k);
    launched(ctx, PH_WF_LEVELS, 3);
    int64_t c[LVC] = {};
    WS_TRY(wf_read_counts(ctx, k, c, st));
    *count = c[k];
    w.k = k + 1;
  }
  WS_CUDA(cudaGetLastError());
  return WS_OK;
}

ws_status shard_wf_end(ws_ctx* ctx, const int32_t* labels_own, const Geo& gown, int conn, const int* dense_of,
                       const int* rep_of_global, int32_t* levels_own, cudaStream_t st) {
  (void)labels_own;
  (void)dense_of;  // the owned planes' dense ids are in ctx->dimg (written by shard_wf_begin)
  WS_TRY(ctx->rep_of.ensure((size_t)ctx->wf.R * sizeof(int), "rep_of"));
  WS_CUDA(cudaMemcpyAsync(ctx->rep_of.p, rep_of_global, (size_t)ctx->wf.R * sizeof(int), cudaMemcpyDeviceToDevice, st));
  return wf_finish(ctx, ctx->dimg.as<int>() + ctx->wf.dofs, gown, conn, levels_own, st);
}

}  // namespace ws
