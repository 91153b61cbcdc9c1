// ws_waterfall.cu — the graph waterfall (C13) over the region adjacency graph, sm_100a.
//
//   k_rep_count / k_scan_blocks / k_rep_assign   dense ids: exclusive scan of
//                                                [labels(p) == p] (prefix-scan compaction)
//   k_rag        RAG extraction: forward neighbour pairs with different labels, height
//                max(I(p), I(q)), deduplicated per tile in a shared-memory hash
//                with u64 atomicMin on the edge key K (C14) = per-pair minimum (Alg. 4 l.2-7)
//   per level k: k_best_reset, k_edge_min (per-component min-K edge, u64 atomicMin),
//                k_hook (min-root CAS union along the picks, C16), k_flatten (+ level map)
//   k_levels     levels[k][p] = map_k[dense(labels(p))]  (Alg. 5 l.12 output, one pass)
#include "ws_internal.h"

namespace ws {

constexpr int SCAN_CHUNK = 4096;  // voxels per block in the representative scan
constexpr int SCAN_THREADS = 256;

__device__ __forceinline__ int warp_incl_scan(int v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) >= o) v += t;
  }
  return v;
}

// block-wide exclusive scan of one int per thread (blockDim.x == SCAN_THREADS)
__device__ __forceinline__ int block_excl_scan(int v, int* smem, int& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int inc = warp_incl_scan(v);
  if (lane == 31) smem[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    int s = lane < SCAN_THREADS / 32 ? smem[lane] : 0;
    s = warp_incl_scan(s);
    if (lane < SCAN_THREADS / 32) smem[lane] = s;
  }
  __syncthreads();
  const int base = wid ? smem[wid - 1] : 0;
  total = smem[SCAN_THREADS / 32 - 1];
  __syncthreads();
  return base + inc - v;
}

__global__ void k_rep_count(const int* __restrict__ labels, int N, int* __restrict__ blockcnt) {
  __shared__ int sm[32];
  const int base = blockIdx.x * SCAN_CHUNK;
  int c = 0;
  for (int i = threadIdx.x; i < SCAN_CHUNK; i += SCAN_THREADS) {
    const int p = base + i;
    if (p < N && __ldg(labels + p) == p) ++c;
  }
  int total;
  block_excl_scan(c, sm, total);
  if (threadIdx.x == 0) blockcnt[blockIdx.x] = total;
}

// single block: in-place exclusive scan of blockcnt[0..nb), total -> *R
__global__ void k_scan_blocks(int* blockcnt, int nb, long long* R) {
  __shared__ int sm[32];
  int carry = 0;
  for (int base = 0; base < nb; base += SCAN_THREADS) {
    const int i = base + threadIdx.x;
    const int v = i < nb ? blockcnt[i] : 0;
    int total;
    const int ex = block_excl_scan(v, sm, total);
    if (i < nb) blockcnt[i] = carry + ex;
    carry += total;
  }
  if (threadIdx.x == 0) *R = carry;
}

__global__ void k_rep_assign(const int* __restrict__ labels, int N, const int* __restrict__ blockoff,
                             int* __restrict__ dense_of, int* __restrict__ rep_of) {
  __shared__ int sm[32];
  const int base = blockIdx.x * SCAN_CHUNK;
  int off = blockoff[blockIdx.x];
  for (int i0 = 0; i0 < SCAN_CHUNK; i0 += SCAN_THREADS) {
    const int p = base + i0 + threadIdx.x;
    const int f = (p < N && __ldg(labels + p) == p) ? 1 : 0;
    int total;
    const int ex = block_excl_scan(f, sm, total);
    if (f) {
      dense_of[p] = off + ex;
      rep_of[off + ex] = p;
    }
    off += total;
  }
}

// ------------------------------------------------------------------------ RAG extraction
constexpr int RAG_TZ = 4;           // tile = 32 x 8 x RAG_TZ voxels (3-D), 32 x 8 (2-D)
constexpr int HCAP = 2048;          // shared hash slots (u64)
constexpr uint64_t PAIRMASK = (1ull << 56) - 1;

__device__ __forceinline__ void emit_global(uint64_t k, uint64_t* edges, unsigned long long* ecount,
                                            long long cap) {
  const unsigned long long i = atomicAdd(ecount, 1ull);
  if ((long long)i < cap) edges[i] = k;
}

__device__ __forceinline__ void hash_insert(uint64_t* tab, uint64_t k, uint64_t* edges,
                                            unsigned long long* ecount, long long cap) {
  const uint64_t pair = k & PAIRMASK;
  uint32_t h = (uint32_t)(pair * 0x9E3779B97F4A7C15ull >> 40) & (HCAP - 1);
  for (int probe = 0; probe < 64; ++probe) {
    uint64_t cur = tab[h];
    if (cur == KEY_NONE) {
      cur = atomicCAS((unsigned long long*)(tab + h), (unsigned long long)KEY_NONE, (unsigned long long)k);
      if (cur == KEY_NONE) return;
    }
    if ((cur & PAIRMASK) == pair) {  // same region pair: keep the lower pass (min K)
      atomicMin((unsigned long long*)(tab + h), (unsigned long long)k);
      return;
    }
    h = (h + 1) & (HCAP - 1);
  }
  emit_global(k, edges, ecount, cap);  // table congested: emit undeduplicated (still correct)
}

template <int CONN>
__global__ void __launch_bounds__(256) k_rag(const int* __restrict__ labels, const uint8_t* __restrict__ I,
                                             const int* __restrict__ dense_of, Geo g, uint64_t* __restrict__ edges,
                                             unsigned long long* ecount, long long cap) {
  __shared__ uint64_t tab[HCAP];
  __shared__ int nloc;
  __shared__ unsigned long long gbase;
  const int tid = threadIdx.x + threadIdx.y * blockDim.x;
  for (int i = tid; i < HCAP; i += 256) tab[i] = KEY_NONE;
  if (tid == 0) nloc = 0;
  __syncthreads();
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  constexpr int TZ = Conn<CONN>::is3d ? RAG_TZ : 1;
  const int z0 = blockIdx.z * TZ;
  if (x < g.n2 && y < g.n1) {
    for (int z = z0; z < z0 + TZ && z < g.n0; ++z) {
      const int p = z * g.plane + y * g.n2 + x;
      const int lp = __ldg(labels + p);
      const int vp = __ldg(I + p);
      int dp = -1;
#pragma unroll
      for (int i = Conn<CONN>::nfwd; i < CONN; ++i) {
        if (!nb_in<CONN>(g, z, y, x, i)) continue;
        const int q = p + nb_off<CONN>(g, i);
        const int lq = __ldg(labels + q);
        if (lq == lp) continue;
        if (dp < 0) dp = __ldg(dense_of + lp);
        const int dq = __ldg(dense_of + lq);
        const int w = max(vp, (int)__ldg(I + q));
        hash_insert(tab, make_key((uint32_t)w, (uint32_t)dp, (uint32_t)dq), edges, ecount, cap);
      }
    }
  }
  __syncthreads();
  // flush the tile's unique edges: local slot numbers, one global atomic per block
  int myidx[HCAP / 256];
#pragma unroll
  for (int j = 0; j < HCAP / 256; ++j) {
    const uint64_t k = tab[tid + j * 256];
    myidx[j] = (k != KEY_NONE) ? atomicAdd(&nloc, 1) : -1;
  }
  __syncthreads();
  if (tid == 0) gbase = atomicAdd(ecount, (unsigned long long)nloc);
  __syncthreads();
#pragma unroll
  for (int j = 0; j < HCAP / 256; ++j) {
    if (myidx[j] >= 0) {
      const long long i = (long long)gbase + myidx[j];
      if (i < cap) edges[i] = tab[tid + j * 256];
    }
  }
}

// ---------------------------------------------------------------------- level loop
__global__ void k_iota(int* a, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = i;
}

__global__ void k_best_reset(uint64_t* best, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) best[i] = KEY_NONE;
}

// per-component min-K outgoing edge; internal edges are marked dead
__global__ void k_edge_min(uint64_t* __restrict__ edges, long long E, const int* __restrict__ comp,
                           uint64_t* __restrict__ best) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < E; e += (long long)gridDim.x * blockDim.x) {
    const uint64_t k = edges[e];
    if (k == KEY_NONE) continue;
    const int ca = __ldg(comp + key_lo(k)), cb = __ldg(comp + key_hi(k));
    if (ca == cb) { edges[e] = KEY_NONE; continue; }
    atomicMin((unsigned long long*)(best + ca), (unsigned long long)k);
    atomicMin((unsigned long long*)(best + cb), (unsigned long long)k);
  }
}

// find with path halving (see ws_watershed.cu uf_find)
__device__ __forceinline__ int c_find(int* c, int x) {
  while (true) {
    const int y = ld_cg(c + x);
    if (y == x) return x;
    const int z = ld_cg(c + y);
    if (z == y) return y;
    __stcg(c + x, z);
    x = z;
  }
}

__global__ void k_hook(const uint64_t* __restrict__ best, int* comp, int n) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    const uint64_t k = best[c];
    if (k == KEY_NONE) continue;  // non-roots and isolated components (C17)
    int a = (int)key_lo(k), b = (int)key_hi(k);
    while (true) {  // min-root union (C16)
      a = c_find(comp, a);
      b = c_find(comp, b);
      if (a == b) break;
      if (a > b) { const int t = a; a = b; b = t; }
      if (atomicCAS(comp + b, b, a) == b) break;
    }
  }
}

// read-only find: k_flatten must not path-halve, or a halving store could land after the
// owner's flattening store and leave a non-root parent behind
__device__ __forceinline__ int c_find_ro(const int* c, int x) {
  while (true) {
    const int y = ld_cg(c + x);
    if (y == x) return x;
    x = y;
  }
}

__global__ void k_flatten(int* comp, int n, const int* __restrict__ rep_of, int* __restrict__ levelmap,
                          int stride, int col, unsigned long long* nroots) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    const int r = c_find_ro(comp, c);
    comp[c] = r;
    levelmap[(size_t)c * stride + col] = __ldg(rep_of + r);
    const unsigned act = __activemask();
    const unsigned b = __ballot_sync(act, r == c);
    if (b && (threadIdx.x & 31) == (unsigned)(__ffs(act) - 1)) atomicAdd(nroots, (unsigned long long)__popc(b));
  }
}

__global__ void k_copy_col(int* levelmap, int n, int stride, int from, int to) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x)
    levelmap[(size_t)c * stride + to] = levelmap[(size_t)c * stride + from];
}

// --------------------------------------------------------------- level materialisation
__global__ void k_levels(const int* __restrict__ labels, const int* __restrict__ dense_of,
                         const int* __restrict__ levelmap, int NL, long long N, int* __restrict__ levels) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < N; p += (long long)gridDim.x * blockDim.x) {
    const int l = __ldg(labels + p);
    levels[p] = l;
    if (NL > 1) {
      const int* m = levelmap + (size_t)__ldg(dense_of + l) * (NL - 1);
      for (int k = 1; k < NL; ++k) levels[k * N + p] = __ldg(m + k - 1);
    }
  }
}

// --------------------------------------------------------------------------- driver
template <int CONN>
static ws_status rag_t(const int* labels, const uint8_t* I, const int* dense_of, const Geo& g, uint64_t* edges,
                       unsigned long long* ecount, long long cap, cudaStream_t st) {
  dim3 block(32, 8, 1);
  constexpr int TZ = Conn<CONN>::is3d ? RAG_TZ : 1;
  const int gz = (g.n0 + TZ - 1) / TZ;
  if (gz > 65535) {
    set_error(WS_ERR_LIMIT, "ws_waterfall: axis 0 too long for the RAG launch (%d tiles)", gz);
    return WS_ERR_LIMIT;
  }
  dim3 grid((g.n2 + 31) / 32, (g.n1 + 7) / 8, gz);
  k_rag<CONN><<<grid, block, 0, st>>>(labels, I, dense_of, g, edges, ecount, cap);
  WS_CUDA(cudaGetLastError());
  return WS_OK;
}

static ws_status rag(int conn, const int* labels, const uint8_t* I, const int* dense_of, const Geo& g,
                     uint64_t* edges, unsigned long long* ecount, long long cap, cudaStream_t st) {
  switch (conn) {
    case 4: return rag_t<4>(labels, I, dense_of, g, edges, ecount, cap, st);
    case 8: return rag_t<8>(labels, I, dense_of, g, edges, ecount, cap, st);
    case 6: return rag_t<6>(labels, I, dense_of, g, edges, ecount, cap, st);
    case 26: return rag_t<26>(labels, I, dense_of, g, edges, ecount, cap, st);
  }
  return WS_ERR_INVALID;
}

static int grid_for(long long n, int sms) {
  long long b = (n + 255) / 256;
  long long cap = (long long)sms * 16;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

ws_status run_waterfall(ws_ctx* ctx, const int32_t* labels, const uint8_t* I, const Geo& g, int conn, int NL,
                        int32_t* levels, int64_t* counts, cudaStream_t st) {
  const int N = g.N;
  const int nb = (N + SCAN_CHUNK - 1) / SCAN_CHUNK;
  WS_TRY(ctx->flags.ensure(256, "flags"));
  WS_TRY(ctx->aux.ensure((size_t)N * sizeof(int), "aux"));
  WS_TRY(ctx->blockcnt.ensure((size_t)nb * sizeof(int), "blockcnt"));
  int* dense_of = ctx->aux.as<int>();
  int* blockcnt = ctx->blockcnt.as<int>();
  long long* dR = reinterpret_cast<long long*>(ctx->flags.as<char>() + 128);
  unsigned long long* ecount = reinterpret_cast<unsigned long long*>(ctx->flags.as<char>() + 136);
  unsigned long long* nroots = reinterpret_cast<unsigned long long*>(ctx->flags.as<char>() + 144);

  // dense ids (prefix-scan compaction of the representatives)
  k_rep_count<<<nb, SCAN_THREADS, 0, st>>>(labels, N, blockcnt);
  k_scan_blocks<<<1, SCAN_THREADS, 0, st>>>(blockcnt, nb, dR);
  launched(ctx, PH_WF_DENSE, 2);
  WS_CUDA(cudaMemcpyAsync(ctx->pinned, dR, sizeof(long long), cudaMemcpyDeviceToHost, st));
  WS_CUDA(cudaStreamSynchronize(st));
  const long long R = ctx->pinned[0];
  if (R > (long long)IDMASK) {
    set_error(WS_ERR_LIMIT, "ws_waterfall: %lld regions exceed the 2^28-1 edge-key limit", R);
    return WS_ERR_LIMIT;
  }
  if (R < 1) {
    set_error(WS_ERR_INVALID, "ws_waterfall: labels are not a canonical labelling (no representative)");
    return WS_ERR_INVALID;
  }
  const int stride = NL > 1 ? NL - 1 : 1;
  WS_TRY(ctx->rep_of.ensure((size_t)R * sizeof(int), "rep_of"));
  WS_TRY(ctx->comp.ensure((size_t)R * sizeof(int), "comp"));
  WS_TRY(ctx->best.ensure((size_t)R * sizeof(uint64_t), "best"));
  WS_TRY(ctx->levelmap.ensure((size_t)R * stride * sizeof(int), "levelmap"));
  int* rep_of = ctx->rep_of.as<int>();
  int* comp = ctx->comp.as<int>();
  uint64_t* best = ctx->best.as<uint64_t>();
  int* levelmap = ctx->levelmap.as<int>();
  k_rep_assign<<<nb, SCAN_THREADS, 0, st>>>(labels, N, blockcnt, dense_of, rep_of);
  launched(ctx, PH_WF_DENSE);
  tmark(ctx, st, PH_WF_DENSE);

  // RAG edges, tile-deduplicated; grow the buffer and redo on overflow
  long long cap = (long long)(ctx->edges.bytes / sizeof(uint64_t));
  long long want = (long long)N / 4 + 4096;
  if (cap < want) {
    WS_TRY(ctx->edges.ensure((size_t)want * sizeof(uint64_t), "edges"));
    cap = want;
  }
  long long E = 0;
  for (int attempt = 0; attempt < 2; ++attempt) {
    WS_CUDA(cudaMemsetAsync(ecount, 0, sizeof(unsigned long long), st));
    WS_TRY(rag(conn, labels, I, dense_of, g, ctx->edges.as<uint64_t>(), ecount, cap, st));
    launched(ctx, PH_WF_RAG);
    WS_CUDA(cudaMemcpyAsync(ctx->pinned, ecount, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    WS_CUDA(cudaStreamSynchronize(st));
    E = ctx->pinned[0];
    if (E <= cap) break;
    WS_TRY(ctx->edges.ensure((size_t)E * sizeof(uint64_t), "edges"));
    cap = E;
  }
  tmark(ctx, st, PH_WF_RAG);
  ctx->stats.n_edges = E;
  ctx->stats.n_regions = R;
  uint64_t* edges = ctx->edges.as<uint64_t>();

  const int gR = grid_for(R, ctx->num_sms), gE = grid_for(E, ctx->num_sms);
  k_iota<<<gR, 256, 0, st>>>(comp, (int)R);
  launched(ctx, PH_WF_LEVELS);
  long long prev = R;
  int lv = 0;
  if (counts) counts[0] = R;
  ctx->stats.level_counts[0] = R;
  for (int k = 1; k < NL; ++k) {
    if (k >= 2 && (prev == 1 || lv < k - 1)) {  // converged: the hierarchy is constant from here (C17)
      k_copy_col<<<gR, 256, 0, st>>>(levelmap, (int)R, stride, k - 2, k - 1);
      launched(ctx, PH_WF_LEVELS);
      if (counts) counts[k] = prev;
      if (k < 16) ctx->stats.level_counts[k] = prev;
      continue;
    }
    k_best_reset<<<gR, 256, 0, st>>>(best, (int)R);
    k_edge_min<<<gE, 256, 0, st>>>(edges, E, comp, best);
    k_hook<<<gR, 256, 0, st>>>(best, comp, (int)R);
    WS_CUDA(cudaMemsetAsync(nroots, 0, sizeof(unsigned long long), st));
    k_flatten<<<gR, 256, 0, st>>>(comp, (int)R, rep_of, levelmap, stride, k - 1, nroots);
    launched(ctx, PH_WF_LEVELS, 4);
    WS_CUDA(cudaMemcpyAsync(ctx->pinned, nroots, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    WS_CUDA(cudaStreamSynchronize(st));
    const long long cnt = ctx->pinned[0];
    if (counts) counts[k] = cnt;
    if (k < 16) ctx->stats.level_counts[k] = cnt;
    if (cnt < prev) lv = k;
    prev = cnt;
  }
  ctx->stats.waterfall_levels = lv;
  tmark(ctx, st, PH_WF_LEVELS);
  const int gN = grid_for(N, ctx->num_sms);
  k_levels<<<gN, 256, 0, st>>>(labels, dense_of, levelmap, NL, N, levels);
  launched(ctx, PH_WF_MATERIALISE);
  tmark(ctx, st, PH_WF_MATERIALISE);
  WS_CUDA(cudaGetLastError());
  return WS_OK;
}

}  // namespace ws
