// ws_internal.h — host-side internals shared by the translation units of libws_b200.so.
#pragma once
#include <cstddef>
#include <cstdint>
#include <string>

#include <cuda_runtime.h>

#include "../../include/ws.h"
#include "ws_common.cuh"

namespace ws {

// Status carrier for internal functions (converted to ws_status at the ABI).
struct Err {
  ws_status st = WS_OK;
  bool ok() const { return st == WS_OK; }
};

void set_error(ws_status st, const char* fmt, ...);
ws_status cuda_fail(cudaError_t e, const char* where);

#define WS_CUDA(call)                                             \
  do {                                                            \
    cudaError_t e__ = (call);                                     \
    if (e__ != cudaSuccess) return ::ws::cuda_fail(e__, #call);   \
  } while (0)

#define WS_TRY(call)                       \
  do {                                     \
    ws_status s__ = (call);                \
    if (s__ != WS_OK) return s__;          \
  } while (0)

// A growable device buffer owned by the context.
struct Buf {
  void* p = nullptr;
  size_t bytes = 0;
  ws_status ensure(size_t want, const char* name);
  void release();
  template <class T> T* as() const { return static_cast<T*>(p); }
};

}  // namespace ws

// waterfall level-loop state (ws_waterfall.cu); persists across the sharded phase calls
struct WSState {
  int64_t R = 0, E = 0, ne_in = 0, nr_in = 0, prev = 0;
  long long dofs = 0;  // offset of the owned planes in ctx->dimg
  long long sorted_n = 0;  // sharded: length of the exchanged minima (current roots, sorted)
  int NL = 1, stride = 4, lv = 0, k = 1, eflip = 0, rflip = -1;
  // sync-free ws_segment (small inputs): R and E stay on the device (R, E above are bounds)
  const unsigned long long* Rdev = nullptr;
  const unsigned long long* Edev = nullptr;
  // sharded dense ids: the slab's label window [dlo, dhi) and the foreign map (ctx->fmap)
  int dlo = 0, dhi = 0, fbits = 4;
};

struct ws_ctx {
  int device = 0;
  int num_sms = 148;
  int coop = 0;       // cooperative launches available (the device-side step II loop); WS_NO_COOP=1 disables
  int edges_occ = 0;  // resident k_edges CTAs per SM (queried once per context)
  ws::Buf aux;        // i32[N]   union-find canonical minima / dense ids (indexed by label)
  ws::Buf tmpA, tmpB; // f32[N]   gradient pre-pass intermediates
  ws::Buf flags;      // small device counters / flags
  ws::Buf tiles;      // u8[3 * ntiles] step II active-tile flags
  ws::Buf tlist;      // i32[ntiles]  compacted active tiles of the next step II round
  ws::Buf roots;      // i32[cap]  step III roots (self-loops), compact list
  ws::Buf upairs;     // int2[cap] step IV pairs crossing a tile face (k_resolve -> k_union_pairs)
  ws::Buf eqc;        // u8[ntiles * 2048] step II equal-neighbour masks (k_relax_first -> later rounds)
  ws::Buf rootc;      // i32[cap]  canonical label per listed root
  ws::Buf blockcnt;   // per-block look-back status words of the dense-id scan
  ws::Buf edges;      // u64[cap] RAG edge keys (level 1)
  ws::Buf ebufA, ebufB;   // compacted live edges (key + current endpoints), ping-pong
  ws::Buf rootsA, rootsB; // level roots lists, ping-pong
  ws::Buf lvl;            // u8[R] level at which a component stops being a root
  // z-slab sharding state
  ws::Buf exitmx;         // i32[2*plane] per-exit minima (INT_MAX - p)
  ws::Buf mtables, mslabs, mr0, mmap;  // replicated merge: gathered tables, bounds, R0, root map
  WSState wf;
  int64_t total_launches = 0;
  int shard_nroots = 0;
  int seg_nroots = 0;     // ws_segment: listed roots left by the watershed (ctx->roots)
  ws::Buf repbits;        // u32[N/32+1] ws_segment: bit c set <=> c is a canonical label
  ws::Buf fmap;           // u64 slots: foreign labels -> dense ids (sharded waterfall)
  int shard_conn = 6;     // connectivity of the last ws_shard_local (6 or 26)
  int shard_tiles = 0;    // tile count of the current sharded plateau phase
  int shard_flip = 0;     // which tile-flag buffer holds "next"
  ws::Buf comp;       // i32[R]   component parent (union-find over dense ids)
  ws::Buf best;       // u64[R]   per-component min-K edge (u16: the hi word of K)
  ws::Buf best_lo;    // u32[R]   u16 waterfall: the lo word of the per-component min-K edge
  ws::Buf rep_of;     // i32[R]   dense id -> canonical voxel label
  ws::Buf levelmap;   // i32[R*stride]  canonical label of each dense id at levels 0..NL-1
  ws::Buf dimg;       // i32[N]   dense id of every voxel's label (waterfall)
  ws::Buf sroots, sblocks;  // sharded waterfall: sorted roots of the level, compaction block counts
  ws::Buf rank;       // uint2[N/32+1] dense-id rank structure (k_dense, unsharded)
  ws::Buf wimg;       // u8[N]    reconstructed image (paper-literal waterfall)
  ws::Buf vstate;     // u8[2N]   states S, S' of the paper's one-thread-per-voxel variants
  ws::Buf nmin;       // u32[N]   255 - newmin per label (paper-literal waterfall)
  ws::Buf lvcount;    // i64[NL]  device-side region counts
  ws::Buf pathc;      // u64[4]   code-path counters of the waterfall (look-back depth, k_edges chunks, RAG emits)
  ws::Buf h_grad, h_labels, h_levels;  // device copies used by ws_segment_host
  // sharded pipeline (ws_sharded.cu): transport + slab of a ws_ctx_create_sharded context and
  // the per-rank working buffers of ws_watershed_sharded / ws_segment_sharded
  int sharded = 0;
  ws_transport sh_tr{};
  ws_slab sh_slab{};
  ws::Buf sh_L, sh_P, sh_planes, sh_tab, sh_alltab, sh_ec, sh_lab, sh_dense, sh_rep, sh_bt, sh_allbt, sh_lext, sh_best,
      sh_nxt, sh_small;
  int64_t* sh_small_h = nullptr;
  size_t sh_small_n = 0;
  int64_t* pinned = nullptr;           // small pinned host scratch (flags / counts)
  // ws_segment on small inputs: the sync-free call captured once as a CUDA graph and replayed
  // while the arguments stay the same (ws_waterfall.cu run_segment)
  struct SegGraph {
    const void* I = nullptr;
    void* levels = nullptr;
    cudaStream_t st = nullptr;
    int n0 = 0, n1 = 0, n2 = 0, conn = 0, NL = 0;
    int seen = 0;             // calls with this key so far (the buffers are sized after one)
    int failed = 0;           // capture unsupported: stay direct
    int64_t launches = 0;     // kernels in the graph
    int64_t last_call = -2;   // ctx->calls at its last use: any other call in between (it may
                              // re-allocate a workspace buffer the graph refers to) drops it
    cudaGraphExec_t exec = nullptr;
  } sg;
  cudaStream_t cap_st = nullptr;  // capture stream (the caller's may be the legacy stream)
  int64_t calls = 0;          // API calls on this context (begin_call)
  ws_stats stats{};
  // per-phase CUDA-event timing (ws_ctx_set_timing)
  bool timing = false;
  static constexpr int MAXEV = 64;
  cudaEvent_t ev[MAXEV] = {};
  int ev_phase[MAXEV] = {};
  int ev_n = 0;
};

namespace ws {

// phases of ws_stats.phase_ms (names in ws_api.cu)
enum Phase {
  PH_GRAD_BLUR = 0, PH_GRAD_MAG, PH_WS_INIT, PH_WS_RELAX, PH_WS_SELECT, PH_WS_JUMP, PH_WS_UNION,
  PH_WS_FIND, PH_WS_RELABEL, PH_WF_DENSE, PH_WF_RAG, PH_WF_LEVELS, PH_WF_MATERIALISE, PH_COPY
};

// timing marks: tbegin() at the start of a call; tmark(ph) closes the segment since the
// previous mark and attributes it to phase ph; tfinish() accumulates the segments.
void tbegin(ws_ctx* ctx, cudaStream_t st);
void tmark(ws_ctx* ctx, cudaStream_t st, int phase);
void tfinish(ws_ctx* ctx);
inline void launched(ws_ctx* ctx, int phase, int n = 1) {
  ctx->total_launches += n;
  ctx->stats.kernel_launches += n;
  ctx->stats.phase_launches[phase] += n;
}

// launch helpers (ws_gradient.cu, ws_watershed.cu, ws_waterfall.cu); each returns WS_OK or a
// CUDA error status and counts its launches into ctx->stats.kernel_launches.
ws_status run_gradient(ws_ctx* ctx, const uint8_t* img, const Geo& g, int is3d, float sigma,
                       uint8_t* grad_q, float* blur_f32, float* grad_f32, cudaStream_t st);
// ws_watershed / ws_segment on a ws_ctx_create_sharded context (ws_sharded.cu)
ws_status sharded_dispatch_watershed(ws_ctx* ctx, const uint8_t* grad_ext, const ws_dims& d, int conn, int32_t* labels,
                                     int64_t* num_regions, cudaStream_t st);
ws_status sharded_dispatch_segment(ws_ctx* ctx, const uint8_t* grad_ext, const ws_dims& d, int conn, int NL,
                                   int32_t* levels, int64_t* counts, cudaStream_t st);
ws_status sharded_dispatch_waterfall(ws_ctx* ctx, const int32_t* labels_own, const uint8_t* grad_ext, const ws_dims& d,
                                     int conn, int NL, int32_t* levels, int64_t* counts, cudaStream_t st);
ws_status sharded_dispatch_watershed_u16(ws_ctx* ctx, const uint16_t* grad_ext, const ws_dims& d, int conn,
                                         int32_t* labels, int64_t* num_regions, cudaStream_t st);
ws_status sharded_dispatch_waterfall_u16(ws_ctx* ctx, const int32_t* labels_own, const uint16_t* grad_ext,
                                         const ws_dims& d, int conn, int NL, int32_t* levels, int64_t* counts,
                                         cudaStream_t st);
ws_status run_watershed(ws_ctx* ctx, const uint8_t* grad, const Geo& g, int conn,
                        int32_t* labels, int64_t* num_regions, cudaStream_t st, bool relabel = true,
                        bool small = false);
ws_status run_gradient_u16(ws_ctx* ctx, const uint16_t* img, const Geo& g, int is3d, float sigma,
                           uint16_t* grad_q, float* blur_f32, float* grad_f32, cudaStream_t st);
namespace px16 {  // ws_watershed16.cu / ws_shard16.cu: the same watershed on u16 pixels
ws_status run_watershed(ws_ctx* ctx, const uint16_t* grad, const Geo& g, int conn, int32_t* labels,
                        int64_t* num_regions, cudaStream_t st, bool relabel = true, bool small = false);
ws_status plateau_first_shard(ws_ctx* ctx, const uint16_t* grad, const Geo& g, int conn, int32_t* L, int* pending,
                              cudaStream_t st);
ws_status plateau_round_shard(ws_ctx* ctx, const uint16_t* grad, const Geo& g, int conn, int32_t* L, int act_lo,
                              int act_hi, int* pending, cudaStream_t st);
ws_status shard_halo(ws_ctx* ctx, int32_t* L, const Geo& g, int side, const int32_t* plane_in, int32_t* changed,
                     cudaStream_t st);
ws_status shard_local(ws_ctx* ctx, const uint16_t* grad, const Geo& g, int conn, int32_t* L, int32_t* P, void* table,
                      cudaStream_t st);
ws_status shard_merge(ws_ctx* ctx, const void* tables, const int64_t* z0s, const int64_t* z1s, int K, int rank,
                      const Geo& g, int32_t* L, int32_t* exitcanon, cudaStream_t st);
ws_status shard_relabel(ws_ctx* ctx, const int32_t* P, int32_t* L, const int32_t* exitcanon, const Geo& g,
                        int32_t* labels_own, int64_t* nreps, cudaStream_t st);
size_t shard_table_bytes(size_t plane);
}
ws_status run_plateau_debug(ws_ctx* ctx, const uint8_t* grad, const Geo& g, int conn,
                            int32_t* dist, int32_t* parent, cudaStream_t st);
// z-slab sharded watershed phases (ws_shard.cu / ws_watershed.cu)
ws_status plateau_first_shard(ws_ctx* ctx, const uint8_t* grad, const Geo& g, int conn, int32_t* L, int* pending,
                              cudaStream_t st);
ws_status plateau_round_shard(ws_ctx* ctx, const uint8_t* grad, const Geo& g, int conn, int32_t* L, int act_lo,
                              int act_hi, int* pending, cudaStream_t st);
ws_status shard_halo(ws_ctx* ctx, int32_t* L, const Geo& g, int side, const int32_t* plane_in, int32_t* changed,
                     cudaStream_t st);
ws_status shard_local(ws_ctx* ctx, const uint8_t* grad, const Geo& g, int conn, int32_t* L, int32_t* P, void* table,
                      cudaStream_t st);
ws_status shard_merge(ws_ctx* ctx, const void* tables, const int64_t* z0s, const int64_t* z1s, int K, int rank,
                      const Geo& g, int32_t* L, int32_t* exitcanon, cudaStream_t st);
ws_status shard_relabel(ws_ctx* ctx, const int32_t* P, int32_t* L, const int32_t* exitcanon, const Geo& g,
                        int32_t* labels_own, int64_t* nreps, cudaStream_t st);
size_t shard_table_bytes(size_t plane);  // boundary table bytes of one rank (u8 pixels)

ws_status shard_wf_dense(ws_ctx* ctx, const int32_t* labels_own, int n, int pofs, int doff, int* dense_of,
                         int* rep_of_global, int64_t* count, cudaStream_t st);
ws_status shard_wf_btable(ws_ctx* ctx, const int32_t* labels_own, int nplanes, int plane, int pofs, const int* dense_of,
                          int32_t* out, cudaStream_t st);
ws_status shard_wf_bfill(ws_ctx* ctx, const int32_t* tabs, int K, int plane, int lo, int hi, int* dense_of,
                         cudaStream_t st);
ws_status shard_wf_begin(ws_ctx* ctx, const int32_t* labels_ext, const uint8_t* I_ext, const Geo& g, int conn,
                         const int* dense_of, int64_t R, int NL, uint64_t* best_out, cudaStream_t st);
ws_status shard_wf_step(ws_ctx* ctx, const uint64_t* best_in, uint64_t* best_out, int64_t* count, int* more,
                        cudaStream_t st);
ws_status shard_wf16_begin(ws_ctx* ctx, const int32_t* labels_ext, const uint16_t* I_ext, const Geo& g, int conn,
                           const int* dense_of, int64_t R, int NL, cudaStream_t st);
ws_status shard_wf16_level(ws_ctx* ctx, int step, int64_t* count, cudaStream_t st);
ws_status shard_wf_end(ws_ctx* ctx, const int32_t* labels_own, const Geo& gown, int conn, const int* dense_of,
                       const int* rep_of_global, int32_t* levels_own, cudaStream_t st);

ws_status run_waterfall(ws_ctx* ctx, const int32_t* labels, const uint8_t* grad, const Geo& g,
                        int conn, int NL, int32_t* levels, int64_t* counts, cudaStream_t st);
ws_status run_segment(ws_ctx* ctx, const uint8_t* grad, const Geo& g, int conn, int NL, int32_t* levels,
                      int64_t* counts, cudaStream_t st);
ws_status run_waterfall_u16(ws_ctx* ctx, const int32_t* labels, const uint16_t* grad, const Geo& g,
                            int conn, int NL, int32_t* levels, int64_t* counts, cudaStream_t st);
ws_status run_watershed_variant(ws_ctx* ctx, const uint8_t* grad, const Geo& g, int conn, int variant,
                                int32_t* labels, int64_t* num_regions, cudaStream_t st);
ws_status run_waterfall_reconstruct(ws_ctx* ctx, const int32_t* labels, const uint8_t* grad, const Geo& g, int conn,
                                    int NL, int32_t* levels, int64_t* counts, cudaStream_t st);

// TMA tensor map for a row-major (n0, n1, n2) array of `esize`-byte elements with box
// {bx, by, bz} (x fastest).  Returns false when the layout cannot be described (global
// address or row pitch not 16-byte aligned); the caller then uses the fallback loader.
bool encode_tmap_3d(void* map /* CUtensorMap* */, int esize, const void* base, const Geo& g, unsigned bx,
                    unsigned by, unsigned bz);

// 3-D launch geometry: block (32, 8, 1), grid over (n2, n1, min(n0, 65535)); kernels loop z.
struct L3 {
  dim3 grid, block;
};
#define ZLOOP_BEGIN_R                                                       \
  const int x = blockIdx.x * blockDim.x + threadIdx.x;                      \
  const int y = blockIdx.y * blockDim.y + threadIdx.y;                      \
  if (x >= g.n2 || y >= g.n1) return;                                       \
  for (int z = blockIdx.z; z < g.n0; z += gridDim.z) {                      \
    const int p = z * g.plane + y * g.n2 + x;
#define ZLOOP_END_R }

inline L3 launch3(const Geo& g, int bx = 32, int by = 8) {
  L3 l;
  l.block = dim3(bx, by, 1);
  l.grid = dim3((g.n2 + bx - 1) / bx, (g.n1 + by - 1) / by, g.n0 < 65535 ? g.n0 : 65535);
  return l;
}

}  // namespace ws
