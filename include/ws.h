/* =====================================================================================
 *  ws.h — C ABI of the B200-native (sm_100a) hot path of arXiv 2410.08946,
 *  "Parallel Watershed Partitioning: GPU-Based Hierarchical Image Segmentation".
 *
 *  The three calls follow the paper's statement of the problem (BASELINE.json north_star):
 *    ws_gradient (img, dims, sigma)           -> agreed u8 gradient-magnitude image
 *    ws_watershed(grad, dims, connectivity)   -> canonical watershed labels
 *    ws_waterfall(labels, grad, NL)           -> NL nested hierarchical label levels
 *
 *  Citation keys: P:n = PAPER.md line n (arXiv 2410.08946 LaTeX source); Cn = reading n in
 *  DESIGN.md "Readings" (= SURVEY.md §8(c)).
 *
 *  Conventions shared by every call
 *  --------------------------------
 *  - All array pointers are DEVICE pointers owned by the caller (e.g. torch tensors); the
 *    library never frees or retains them past the call.  Exception: ws_segment_host takes
 *    HOST pointers (see there).
 *  - Layout: row-major, last axis fastest (C1).  Linear voxel index
 *      p = (z * n1 + y) * n2 + x,   N = n0 * n1 * n2  (must be < 2^31).
 *  - dims.ndim == 2: n0 independent 2-D images of n1 x n2 (a batch; no adjacency across
 *    axis 0, C18).  1-D images are 2-D images with n1 == 1.
 *    dims.ndim == 3: one volume of depth n0.
 *  - connectivity: 4 or 8 with ndim 2 (von Neumann / Moore), 6 or 26 with ndim 3.
 *    Neighbourhoods are clipped at the border, the centre excluded (C2).
 *  - stream: a cudaStream_t passed as void*; NULL = the legacy default stream.  Work is
 *    enqueued on it.  ws_watershed and ws_waterfall synchronise the stream internally (they
 *    read convergence flags and sizes back), ws_gradient does not.
 *  - Errors: every argument is validated before any launch; on error nothing is written to
 *    any output and a message is available from ws_last_error() (thread-local).  No C++
 *    exception or abort crosses the ABI.
 *  - Determinism: outputs are bit-identical across runs ("fully deterministic").
 * ===================================================================================== */
#ifndef WS_B200_H
#define WS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum ws_status {
  WS_OK = 0,
  WS_ERR_INVALID = 1,  /* bad dims / connectivity / NL / sigma / NULL pointer          */
  WS_ERR_OOM = 2,      /* workspace allocation failed                                   */
  WS_ERR_CUDA = 3,     /* a CUDA runtime error (message has the CUDA error string)      */
  WS_ERR_NCCL = 4,     /* a transport (NCCL or caller callback) of the sharded path failed */
  WS_ERR_INTERNAL = 5, /* an internal consistency check failed                          */
  WS_ERR_LIMIT = 6     /* a documented size limit was exceeded (message says which)     */
} ws_status;

typedef struct ws_dims {
  int32_t ndim;     /* 2 (batch of images) or 3 (volume)                                  */
  int32_t reserved; /* must be 0                                                          */
  int64_t n0;       /* ndim 2: number of images (>= 1); ndim 3: depth                     */
  int64_t n1;       /* height                                                             */
  int64_t n2;       /* width (fastest axis)                                               */
} ws_dims;

/* Opaque context: owns the device scratch workspace (grown on demand, freed by destroy)
 * and the statistics of the last call.  One context per device; not thread-safe. */
typedef struct ws_ctx ws_ctx;

#define WS_NUM_PHASES 16

typedef struct ws_stats {
  int64_t n_voxels;
  int64_t n_regions;          /* R of the last ws_watershed / ws_waterfall               */
  int64_t n_edges;            /* RAG edge records after tile-local dedup (ws_waterfall)   */
  int32_t plateau_rounds;     /* step II global relaxation rounds (ws_watershed)          */
  int32_t waterfall_levels;   /* levels actually iterated (stops early once R == 1)       */
  int64_t level_counts[16];   /* regions per level (first min(NL,16) levels)              */
  int64_t kernel_launches;    /* kernels launched by the last call                        */
  /* per-phase device time of the last call, CUDA events on the call's stream; filled only
   * when timing is enabled (ws_ctx_set_timing).  Phase names: ws_phase_name(i). */
  double phase_ms[WS_NUM_PHASES];
  int32_t phase_launches[WS_NUM_PHASES];
  int32_t tma;                /* 1 if the tile kernels staged their boxes with TMA         */
  int32_t reserved0;
  int64_t level_edges[16];    /* live RAG edge records entering each waterfall level       */
  int64_t total_launches;     /* kernels launched by this context since its creation       */
  /* size-dependent code paths the last call took (the full-size parity tests assert them) */
  int32_t union_order;        /* ws_watershed step IV: 0 = cross-tile pair list before the chase,
                                 1 = chase first + pair list (many pairs: giant minimal plateaux),
                                 2 = chase first + full k_union scan (pair list overflow)        */
  int32_t root_overflow;      /* ws_watershed: 1 if the step III root list overflowed (rebuilt) */
  int32_t lookback_max;       /* ws_waterfall: deepest look-back (blocks) of the dense-id scan   */
  int32_t edge_chunks_max;    /* ws_waterfall: most edge chunks one k_edges block walked         */
  int64_t rag_global_emits;   /* ws_waterfall: RAG records emitted past a full tile pair hash    */
  int64_t rag_records;        /* ws_waterfall: boundary records the RAG staged after run merging  */
} ws_stats;

ws_status ws_ctx_create(int32_t device, ws_ctx** out);
ws_status ws_ctx_destroy(ws_ctx* ctx);
const char* ws_last_error(void);
const char* ws_version(void);
/* Statistics of the most recent call on ctx (copied into *out). */
ws_status ws_get_stats(const ws_ctx* ctx, ws_stats* out);
/* Enable (1) / disable (0) per-phase CUDA-event timing in ws_stats.phase_ms. */
ws_status ws_ctx_set_timing(ws_ctx* ctx, int32_t enable);
/* Name of phase i (0 <= i < WS_NUM_PHASES), "" if unused. */
const char* ws_phase_name(int32_t i);

/* ws_gradient — the stencil pre-pass (Fig. 2: "input image smoothing and
 * use of gradient magnitude image are optional").
 *   b    = G_sigma * (img / 255): separable sampled Gaussian, radius r = floor(3 sigma + 0.5),
 *          normalised weights, clamp-to-edge; sigma == 0 is the identity (C8).
 *          ndim 3 blurs along all three axes, ndim 2 along n1 and n2 of each image.
 *   g    = || grad b ||_2 with central differences inside and one-sided differences at the
 *          ends, 0 along an axis of length 1 (C9).
 *   grad_q[p] = min(255, floor(255 g + 0.5))  (C10, the agreed integer image, C11).
 * Arguments: img u8[N] (in), grad_q u8[N] (out, required), blur_f32 / grad_f32 f32[N]
 * (out, optional "verify mode", may be NULL).  Arithmetic is fp32.
 * Errors: WS_ERR_INVALID for bad dims, sigma < 0 or sigma > 20, NULL img/grad_q. */
ws_status ws_gradient(ws_ctx* ctx, const uint8_t* img, ws_dims dims, float sigma,
                      uint8_t* grad_q, float* blur_f32, float* grad_f32, void* stream);

/* ws_gradient_u16 — ws_gradient on a 16-bit image (NEXT f4; microCT volumes are often
 * 16-bit): b = G_sigma * (img / 65535) with the same Gaussian (C8) and differences
 * (C9); grad_q[p] = min(65535, floor(65535 g + 0.5)) (C10 at 16 bits: finer levels, smaller
 * plateaux).  A u8 image widened by x257 has exactly the same b and g.
 * Arguments: img u16[N] (in), grad_q u16[N] (out, required), blur_f32 / grad_f32 f32[N]
 * (optional verify mode), all 2-byte aligned.  Arithmetic is fp32: with r = floor(3 sigma
 * + 0.5) in 1..4 the kernels of ws_gradient run on u16 pixels (volumes: streaming kernel,
 * 2-D: tile kernel), other cases separable passes through two f32[N] workspace arrays.
 * Errors: as ws_gradient. */
ws_status ws_gradient_u16(ws_ctx* ctx, const uint16_t* img, ws_dims dims, float sigma,
                          uint16_t* grad_q, float* blur_f32, float* grad_f32, void* stream);

/* ws_watershed — steps I-IV of PRUF (Alg. 1) + canonical relabel.
 *   Step I   steepest-descent pointer, Eq. 1: among the minimal neighbours
 *            the one with the largest index (C3).
 *   Step II  non-minimal plateaux: BFS distance from the plateau's lower voxels, parent =
 *            max-index equal neighbour one step closer (Sync semantics P:194-203, C5/C6),
 *            computed by tile-local relaxation (the PRUF_bal mechanism, Alg. 3)
 *            followed by a pointer-selection pass.
 *   Step III pointer jumping to the self-loop roots (Alg. 1 l.19-23 / l.28-29).
 *   Step IV  min-root lock-free union-find over adjacent minimal-plateau voxels.
 *   Output   labels[p] = smallest linear index in p's catchment basin (C7).
 * Arguments: grad u8[N] (in), labels i32[N] (out; also used as the working pointer array),
 * num_regions (HOST i64, optional, may be NULL).
 * Errors: WS_ERR_INVALID (dims/conn mismatch, NULL), WS_ERR_LIMIT (a non-minimal plateau
 * deeper than 2^26-2 voxels). */
ws_status ws_watershed(ws_ctx* ctx, const uint8_t* grad, ws_dims dims, int32_t connectivity,
                       int32_t* labels, int64_t* num_regions, void* stream);

/* ws_watershed_u16 — ws_watershed on a 16-bit image (NEXT f4; microCT volumes are often
 * 16-bit; the paper's headline protocol runs on raw images).  Identical
 * definition, steps and output; intensities compare as unsigned 16-bit values.
 * Arguments: grad u16[N] (in, 2-byte aligned), labels i32[N] (out), num_regions (HOST i64,
 * optional).  TMA staging needs a 16-byte aligned grad and n2 % 8 == 0, else a plain loader
 * runs (same result).  Unsharded only (the ws_shard_* calls take u8).
 * Errors: as ws_watershed. */
ws_status ws_watershed_u16(ws_ctx* ctx, const uint16_t* grad, ws_dims dims, int32_t connectivity,
                           int32_t* labels, int64_t* num_regions, void* stream);

/* ws_watershed_variant — the paper's own one-thread-per-voxel watershed kernels (SURVEY NEXT
 * f3), the baseline for the tiled ws_watershed; every variant yields the same partition
 * and the same canonical labels (C7):
 *   WS_VARIANT_PRUF_SYNC   Alg. 1 as written: step I, Jacobi step II (S -> S',
 *                          host loop until no change), step III by RR = 6 jumps
 *                          per launch until no change, step IV Union + Find.
 *   WS_VARIANT_PRW_SYNC    step IV of Alg. 2: min-merging of representatives +
 *                          path reduction, repeated until no change.
 *   WS_VARIANT_APRUF_SYNC  step III replaced by one independent Find per voxel.
 * Arguments as ws_watershed; errors as ws_watershed plus WS_ERR_INVALID for an unknown
 * variant. */
enum { WS_VARIANT_PRUF_SYNC = 0, WS_VARIANT_PRW_SYNC = 1, WS_VARIANT_APRUF_SYNC = 2 };
ws_status ws_watershed_variant(ws_ctx* ctx, const uint8_t* grad, ws_dims dims, int32_t connectivity,
                               int32_t variant, int32_t* labels, int64_t* num_regions, void* stream);

/* ws_waterfall — the hierarchical segmentation as the graph waterfall (C13):
 *   RAG edges {a, b} between adjacent regions with height max(I(p), I(q)), per pair
 *   the minimum (Alg. 4 l.2-7); strict edge order K = (w asc, max(a,b) desc, min(a,b) desc)
 *   on level-0 canonical labels (C14).  Level k = 1..NL-1: every component of level k-1
 *   merges along its min-K outgoing edge (min-root union-find, C16); isolated components
 *   stay (C17).
 *   levels[k*N + p] = smallest linear index of p's level-k region; levels[0..N) = labels.
 * Arguments: labels i32[N] (in; MUST be canonical ws_watershed output for the same grad,
 * dims and connectivity), grad u8[N] (in), NL >= 1 levels including level 0 (C12),
 * levels i32[NL*N] (out, level-major), counts (HOST i64[NL], optional).
 * Errors: WS_ERR_INVALID (dims/conn/NL, NULL), WS_ERR_LIMIT (more than 2^28-1 regions). */
ws_status ws_waterfall(ws_ctx* ctx, const int32_t* labels, const uint8_t* grad, ws_dims dims,
                       int32_t connectivity, int32_t NL, int32_t* levels, int64_t* counts,
                       void* stream);

/* ws_waterfall_u16 — ws_waterfall on a 16-bit image (NEXT f4): the same graph waterfall
 * (C13) with 16-bit pass heights max(I(p), I(q)) and the same strict order K (C14).
 * K needs 16 + 28 + 28 bits, so per-component minima take two passes (the high word
 * w << 28 | ~max, then ~min among the edges with the minimum high word).
 * Arguments as ws_waterfall; labels MUST be canonical ws_watershed_u16 output for the same
 * grad; grad u16[N] (in, 2-byte aligned).
 * Errors: as ws_waterfall. */
ws_status ws_waterfall_u16(ws_ctx* ctx, const int32_t* labels, const uint16_t* grad, ws_dims dims,
                           int32_t connectivity, int32_t NL, int32_t* levels, int64_t* counts, void* stream);

/* ws_waterfall_reconstruct — the paper's own waterfall by image reconstruction (Sec. 4,
 * P:593-656), single GPU.  Level 0 = labels on I_0 = grad; level k = 1..NL-1:
 *   Step V   newmin(l) = M = 255 (reading C23), then for every p and q in N(p) with
 *            L(q) != L(p): newmin(L(p)) = min(newmin(L(p)), max(I(p), I(q)))  (Alg. 4 l.1-7)
 *   Step VI  I_k(p) = max(I_{k-1}(p), newmin(L_{k-1}(p)))                    (Alg. 4 l.8-12)
 *   then L_k = ws_watershed(I_k) (Alg. 5 l.4-8), canonical labels (C7).
 *   Unlike the graph waterfall (C13) the layers are NOT nested.
 * Arguments as ws_waterfall: labels i32[N] (in, canonical ws_watershed output of grad), grad
 * u8[N] (in, not modified: the raised images live in the context), NL >= 1, levels
 * i32[NL*N] (out, level-major; levels[0..N) = labels), counts (HOST i64[NL], optional).
 * Errors: WS_ERR_INVALID (dims/conn/NL, NULL), WS_ERR_LIMIT as ws_watershed. */
ws_status ws_waterfall_reconstruct(ws_ctx* ctx, const int32_t* labels, const uint8_t* grad, ws_dims dims,
                                   int32_t connectivity, int32_t NL, int32_t* levels, int64_t* counts,
                                   void* stream);

/* ws_segment — ws_watershed followed by ws_waterfall as ONE call (Alg. 5 is one procedure,
 * P:629-656): identical outputs, fewer full-volume passes.  The watershed stops before its
 * relabel; dense region ids come from the root list (a scan over a bitmap of the canonical
 * labels, N/32 words, instead of a scan over the labels); one pass writes level 0 and the
 * dense-id image; the level pass writes levels 1..NL-1.
 * Arguments: grad u8[N] (in), NL >= 1 (C12), levels i32[NL*N] (out, level-major, 16-byte
 * aligned; levels[0..N) = the canonical watershed labels), counts (HOST i64[NL], optional).
 * Errors: as ws_watershed and ws_waterfall. */
ws_status ws_segment(ws_ctx* ctx, const uint8_t* grad, ws_dims dims, int32_t connectivity, int32_t NL,
                     int32_t* levels, int64_t* counts, void* stream);

/* ws_segment_host — the end-to-end user call on HOST buffers: copies grad (host, ideally
 * pinned) to the device, runs ws_segment, copies levels back to the host (host i32[NL*N]).
 * Device buffers come from the context workspace.  Synchronous. */
ws_status ws_segment_host(ws_ctx* ctx, const uint8_t* grad_host, ws_dims dims,
                          int32_t connectivity, int32_t NL, int32_t* levels_host,
                          int64_t* counts, void* stream);

/* ws_segment_host_async — ws_segment_host without the final wait: it returns once the levels'
 * device-to-host copy is ENQUEUED on `stream` (counts are complete at return: the call reads
 * them back before enqueuing the copy).  levels_host is written when the stream reaches the copy
 * and must stay valid until then; the caller synchronises `stream` before reading it.  Two
 * contexts on two streams pipeline a sequence of volumes: the PCIe copy of one volume's levels
 * overlaps the host-to-device copy and the compute of the next (PCIe is full duplex).  The
 * context's workspace holds the levels until the copy is done: do not reuse the context before
 * synchronising `stream`.  Errors: as ws_segment_host. */
ws_status ws_segment_host_async(ws_ctx* ctx, const uint8_t* grad_host, ws_dims dims,
                                int32_t connectivity, int32_t NL, int32_t* levels_host,
                                int64_t* counts, void* stream);

/* ws_plateau_debug — intermediate of step II for per-kernel parity tests (T2):
 *   dist[p] = 0 for voxels with a lower neighbour, the BFS distance on non-minimal plateaux,
 *             -1 on minimal plateaux (regional minima, incl. strict single-voxel minima);
 *   parent[p] = the step-I/II pointer of p (p itself on minimal plateaux).
 * Arguments: grad u8[N] (in), dist i32[N] (out), parent i32[N] (out). */
ws_status ws_plateau_debug(ws_ctx* ctx, const uint8_t* grad, ws_dims dims, int32_t connectivity,
                           int32_t* dist, int32_t* parent, void* stream);

/* ==================================================================================
 * z-slab sharding (north_star: "3D volumes are partitioned along z into slabs across the 8
 * GPUs of one box, with NCCL halo exchange over NVLink and a cross-slab boundary union-find
 * merge").  Volumes (ndim 3), 6- or 26-connectivity.  Rank r of K owns global planes
 * [z0, z1) and holds an EXTENDED slab [e0, e1) = [max(0, z0-2), min(D, z1+2)) of grad and of
 * the working array L_ext (i32); every dims argument below is the extended slab
 * (n0 = e1 - e0, n1, n2).  The caller moves the planes between ranks (NCCL through
 * torch.distributed, or in-process copies) between the calls; the library computes.
 * Result: identical labels to ws_watershed on the whole volume (global voxel indices).
 * ================================================================================== */
typedef struct ws_slab {
  int64_t D;        /* global depth                                                        */
  int64_t z0, z1;   /* owned planes [z0, z1)                                                */
  int64_t e0, e1;   /* extended planes held by the caller                                   */
} ws_slab;

/* bytes of one rank's boundary table (ws_shard_local output, ws_shard_merge input) */
int64_t ws_shard_table_bytes(ws_dims dims_ext);

/* step I + one step II relaxation round on the owned planes (Alg. 1 l.1-18 / Alg. 3).
 * phase 0: first round (classification + relaxation; halo planes of L_ext need not be set).
 * phase 1: a further round on the active tiles; act_lo / act_hi re-activate the first / last
 *          owned tile layer after the halo plane below / above changed.
 * pending (HOST): 1 if this rank has work for another round.  L_ext halo planes: the plane
 * just outside the owned range on each side must hold the neighbour's L values (phase 1). */
ws_status ws_shard_plateau(ws_ctx* ctx, const uint8_t* grad_ext, ws_dims dims_ext, int32_t connectivity,
                           ws_slab slab, int32_t* L_ext, int32_t phase, int32_t act_lo, int32_t act_hi,
                           int32_t* pending, void* stream);
/* copy a neighbour's boundary plane of L (plane_in, i32[n1*n2], device) into the halo plane
 * below (side 0: z0 - 1) or above (side 1: z1) of L_ext; changed (HOST) = 1 if it differed */
ws_status ws_shard_halo(ws_ctx* ctx, int32_t* L_ext, ws_dims dims_ext, ws_slab slab, int32_t side,
                        const int32_t* plane_in, int32_t* changed, void* stream);
/* pointers (steps I-II), local step III (chains leaving the slab stop at an exit), local
 * step IV, per-root minima; writes P_ext (i32, owned planes) and this rank's boundary table */
ws_status ws_shard_local(ws_ctx* ctx, const uint8_t* grad_ext, int32_t* L_ext, ws_dims dims_ext,
                         int32_t connectivity, ws_slab slab, int32_t* P_ext, void* table, void* stream);
/* replicated cross-slab merge over the K gathered tables (tables_all: K tables back to back,
 * device; z0s/z1s: HOST i64[K] owned plane ranges, ascending): chase exits, union minimal
 * plateaux across every cut plane, canonical minima; writes this rank's root labels into
 * L_ext and exitcanon (i32[2*n1*n2], device) */
ws_status ws_shard_merge(ws_ctx* ctx, const void* tables_all, int32_t nranks, const int64_t* z0s,
                         const int64_t* z1s, ws_dims dims_ext, ws_slab slab, int32_t* L_ext, int32_t* exitcanon,
                         void* stream);
/* canonical labels of the owned voxels -> labels_own (i32[(z1-z0)*n1*n2]); nreps (HOST,
 * optional) = owned voxels that are their region's smallest index (for dense-id offsets) */
ws_status ws_shard_relabel(ws_ctx* ctx, const int32_t* P_ext, int32_t* L_ext, const int32_t* exitcanon,
                           ws_dims dims_ext, ws_slab slab, int32_t* labels_own, int64_t* nreps, void* stream);

/* z-slab sharded waterfall (same slabs; labels_own = ws_shard_relabel output).
 * Dense ids follow the rank order: doff = owned representatives (ws_shard_relabel nreps) of
 * all lower ranks; R = all ranks' total.  dense_of: the slab's WINDOW of dense ids, i32[(z1 -
 * z0 + 1) * n1 * n2] (device): entry i = dense id of global label z0*n1*n2 + i (the owned
 * planes and the plane above; sparse: only labels met by this rank are written).  Labels
 * below the window (regions crossing the lower cut, at most two planes of them) are kept in
 * a small map in the context (filled by ws_shard_wf_bfill), so no rank holds a global-size
 * array.  rep_of: i32[R] (device); this
 * rank writes its segment [doff, doff + count), the caller reduces (max) it over ranks with
 * the other entries at -1.  btable: i32[4*n1*n2]: (label, dense id if owned here else -1) of
 * the first and last owned plane; ws_shard_wf_bfill gives every rank the dense ids of all
 * labels crossing a cut.  Per-component minima travel as i64 = K ^ 2^63 (all_reduce MIN). */
ws_status ws_shard_wf_dense(ws_ctx* ctx, const int32_t* labels_own, ws_dims dims_ext, ws_slab slab, int64_t doff,
                            int32_t* dense_of, int32_t* rep_of, int64_t* count, void* stream);
ws_status ws_shard_wf_btable(ws_ctx* ctx, const int32_t* labels_own, const int32_t* dense_of, ws_dims dims_ext,
                             ws_slab slab, int32_t* btable, void* stream);
ws_status ws_shard_wf_bfill(ws_ctx* ctx, const int32_t* btables_all, int32_t nranks, ws_dims dims_ext,
                            ws_slab slab, int32_t* dense_of, void* stream);
/* RAG of the owned planes plus the cut pairs with the rank above (labels_ext: owned planes and
 * the plane above, extended layout); best_out: i64[R] this rank's level-1 minima */
ws_status ws_shard_wf_begin(ws_ctx* ctx, const int32_t* labels_ext, const uint8_t* grad_ext, ws_dims dims_ext,
                            int32_t connectivity, ws_slab slab, const int32_t* dense_of, int64_t R, int32_t NL,
                            int64_t* best_out, void* stream);
/* one level: best_in = all ranks' minima (reduced) of the current components -- level 1: all R
 * regions in dense-id order (ws_shard_wf_begin's output); later levels: the previous level's
 * roots in increasing dense id (the same order on every rank: the union-find is replicated);
 * count (HOST) = regions after the level; more (HOST) = 1 if another level follows, then
 * best_out[0..count) = this rank's minima at this level's roots in increasing dense id
 * (best_out must hold the previous count) */
ws_status ws_shard_wf_step(ws_ctx* ctx, const int64_t* best_in, int64_t* best_out, int64_t* count, int32_t* more,
                           void* stream);
/* level maps + the NL level arrays of the owned voxels: levels_own i32[NL][(z1-z0)*n1*n2] */
ws_status ws_shard_wf_end(ws_ctx* ctx, const int32_t* labels_own, const int32_t* dense_of, const int32_t* rep_of,
                          ws_dims dims_ext, int32_t connectivity, ws_slab slab, int32_t* levels_own, void* stream);

/* ==================================================================================
 * The sharded pipeline as ONE call per rank ("ctx created with
 * ws_ctx_create_sharded(...); the same three calls then operate on the local slab").  The
 * whole distributed control flow of DESIGN.md §9 runs inside the library on top of the
 * ws_shard_* phases above: step II rounds with a halo-plane exchange after each until no rank
 * has work (an all-reduce of the pending flags), the all-gather of the boundary tables and
 * the replicated merge, rank-ordered dense ids (all-gather of the representative counts,
 * all-reduce(max) of rep_of, all-gather of the boundary dense tables), the cut-plane label
 * exchange, and per waterfall level an all-reduce(min) of the per-component minima.
 * Rank r of K owns the planes [z0, z1) of slab (the ranks' slabs tile [0, D) in rank order);
 * grad_ext is the u8 EXTENDED slab [e0, e1) (dims_ext.n0 = e1 - e0, the planes z0-1 and z1
 * must be present when they exist: e0 <= z0-1, e1 >= z1+1); results are the owned planes
 * with GLOBAL canonical labels, identical to the unsharded call (determinism).
 *
 * Collectives go through a ws_transport: three callbacks, each enqueued on / ordered with
 * `stream` (device buffers; the callback returns 0 on success, anything else fails the call
 * with WS_ERR_NCCL).  The library provides an NCCL transport (ws_transport_nccl_create:
 * NCCL over NVLink / NVSwitch, the communicator owned by the library, libnccl.so.2 resolved at
 * run time); callers may supply their own (e.g. torch.distributed / gloo for multi-process
 * tests with several ranks on one GPU, threads for virtual ranks in one process).
 * ================================================================================== */
#define WS_NCCL_ID_BYTES 128
typedef struct ws_transport {
  void* user;        /* passed back to every callback                                      */
  int32_t rank;      /* this rank                                                          */
  int32_t nranks;    /* K                                                                  */
  /* send_lo (this rank's first owned plane) to rank-1 and send_hi (last) to rank+1; receive
   * rank-1's last plane into recv_below and rank+1's first into recv_above; `bytes` each;
   * NULL where the neighbour does not exist */
  int32_t (*exchange)(void* user, const void* send_lo, const void* send_hi, void* recv_below, void* recv_above,
                      int64_t bytes, void* stream);
  /* recv = the K ranks' `bytes`-byte send blocks in rank order */
  int32_t (*allgather)(void* user, const void* send, void* recv, int64_t bytes, void* stream);
  /* in place over `count` elements; dtype 0 = i32, 1 = i64; op 0 = min, 1 = max */
  int32_t (*allreduce)(void* user, void* buf, int64_t count, int32_t dtype, int32_t op, void* stream);
} ws_transport;

/* NCCL transport: rank 0 makes the unique id (WS_NCCL_ID_BYTES bytes, HOST), the caller
 * broadcasts it to the other ranks (e.g. over the torch.distributed store), every rank then
 * creates its transport (collective: all ranks must call).  Errors: WS_ERR_NCCL (libnccl
 * missing, NCCL failure), WS_ERR_INVALID. */
ws_status ws_nccl_unique_id(void* out);
ws_status ws_transport_nccl_create(const void* unique_id, int32_t rank, int32_t nranks, int32_t device,
                                   ws_transport** out);
ws_status ws_transport_nccl_destroy(ws_transport* tr);

/* A context bound to a transport and a slab (the transport must outlive it): ws_watershed,
 * ws_waterfall and ws_segment on it take the EXTENDED slab dims/grad and write the owned
 * planes (labels i32[(z1-z0)*n1*n2], levels i32[NL][(z1-z0)*n1*n2]); counts / num_regions
 * are global.  Volumes only, 6- or 26-connectivity. */
ws_status ws_ctx_create_sharded(int32_t device, const ws_transport* transport, ws_slab slab, ws_ctx** out);

/* the same with an explicit transport (any context); rounds (HOST, optional) = step II rounds */
ws_status ws_watershed_sharded(ws_ctx* ctx, const ws_transport* transport, const uint8_t* grad_ext,
                               ws_dims dims_ext, ws_slab slab, int32_t connectivity, int32_t* labels_own,
                               int64_t* num_regions, int32_t* rounds, void* stream);
ws_status ws_waterfall_sharded(ws_ctx* ctx, const ws_transport* transport, const int32_t* labels_own,
                               const uint8_t* grad_ext, ws_dims dims_ext, ws_slab slab, int32_t connectivity,
                               int32_t NL, int32_t* levels_own, int64_t* counts, void* stream);
ws_status ws_segment_sharded(ws_ctx* ctx, const ws_transport* transport, const uint8_t* grad_ext, ws_dims dims_ext,
                             ws_slab slab, int32_t connectivity, int32_t NL, int32_t* levels_own, int64_t* counts,
                             int32_t* rounds, void* stream);
/* 16-bit images (NEXT f4): the same on u16 gradients -- the watershed of
 * ws_watershed_u16 and the graph waterfall of ws_waterfall_u16 (K = (w:16, ~max, ~min); its
 * per-component minima are reduced over the ranks in two steps per level, the 16-bit height
 * and the larger label first, then the smaller label among those).  grad_ext 2-byte aligned;
 * ws_watershed_u16 / ws_waterfall_u16 on a sharded context run these. */
ws_status ws_watershed_sharded_u16(ws_ctx* ctx, const ws_transport* transport, const uint16_t* grad_ext,
                                   ws_dims dims_ext, ws_slab slab, int32_t connectivity, int32_t* labels_own,
                                   int64_t* num_regions, int32_t* rounds, void* stream);
ws_status ws_waterfall_sharded_u16(ws_ctx* ctx, const ws_transport* transport, const int32_t* labels_own,
                                   const uint16_t* grad_ext, ws_dims dims_ext, ws_slab slab, int32_t connectivity,
                                   int32_t NL, int32_t* levels_own, int64_t* counts, void* stream);
ws_status ws_segment_sharded_u16(ws_ctx* ctx, const ws_transport* transport, const uint16_t* grad_ext,
                                 ws_dims dims_ext, ws_slab slab, int32_t connectivity, int32_t NL, int32_t* levels_own,
                                 int64_t* counts, int32_t* rounds, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* WS_B200_H */
