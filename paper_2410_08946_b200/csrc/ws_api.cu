// ws_api.cu — the C ABI (include/ws.h): validation, context/workspace, error reporting.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <new>

#include <cuda.h>

#include <cstdlib>

#include "ws_internal.h"

namespace ws {

static thread_local char g_err[512] = "";

void set_error(ws_status st, const char* fmt, ...) {
  (void)st;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

ws_status cuda_fail(cudaError_t e, const char* where) {
  set_error(WS_ERR_CUDA, "CUDA error %s (%s) at %s", cudaGetErrorName(e), cudaGetErrorString(e), where);
  return e == cudaErrorMemoryAllocation ? WS_ERR_OOM : WS_ERR_CUDA;
}

// Grows with 1/8 headroom: sizes that vary slightly from call to call (edge counts) must not
// re-allocate (cudaFree synchronises the device) on every call.
ws_status Buf::ensure(size_t want, const char* name) {
  if (want <= bytes) return WS_OK;
  if (p) cudaFree(p);
  p = nullptr;
  bytes = 0;
  if (want == 0) return WS_OK;
  const size_t grow = want + want / 8;
  cudaError_t e = cudaMalloc(&p, grow);
  if (e == cudaSuccess) want = grow;
  else {
    (void)cudaGetLastError();
    e = cudaMalloc(&p, want);
  }
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    p = nullptr;
    set_error(WS_ERR_OOM, "cannot allocate %zu bytes of device workspace for %s", want, name);
    return WS_ERR_OOM;
  }
  bytes = want;
  return WS_OK;
}

void Buf::release() {
  if (p) cudaFree(p);
  p = nullptr;
  bytes = 0;
}

// dims + connectivity validation (ws.h "Errors")
static ws_status check_dims(const ws_dims& d, Geo* g) {
  if (d.ndim != 2 && d.ndim != 3) {
    set_error(WS_ERR_INVALID, "dims.ndim must be 2 or 3 (got %d)", d.ndim);
    return WS_ERR_INVALID;
  }
  if (d.reserved != 0) {
    set_error(WS_ERR_INVALID, "dims.reserved must be 0");
    return WS_ERR_INVALID;
  }
  if (d.n0 < 1 || d.n1 < 1 || d.n2 < 1) {
    set_error(WS_ERR_INVALID, "dims must be >= 1 (got %lld x %lld x %lld)", (long long)d.n0, (long long)d.n1,
              (long long)d.n2);
    return WS_ERR_INVALID;
  }
  const double n = (double)d.n0 * (double)d.n1 * (double)d.n2;
  if (n >= 2147483648.0) {
    set_error(WS_ERR_INVALID, "N = %.0f voxels: must be < 2^31 (i32 labels)", n);
    return WS_ERR_INVALID;
  }
  g->n0 = (int)d.n0;
  g->n1 = (int)d.n1;
  g->n2 = (int)d.n2;
  g->plane = g->n1 * g->n2;
  g->N = g->plane * g->n0;
  g->zlo = 0;
  g->zhi = g->n0;
  g->gofs = 0;
  return WS_OK;
}

static ws_status check_conn(const ws_dims& d, int conn) {
  const bool ok = (d.ndim == 2 && (conn == 4 || conn == 8)) || (d.ndim == 3 && (conn == 6 || conn == 26));
  if (!ok) {
    set_error(WS_ERR_INVALID, "connectivity %d does not match ndim %d (2-D: 4|8, 3-D: 6|26)", conn, d.ndim);
    return WS_ERR_INVALID;
  }
  return WS_OK;
}

static ws_status check_ctx(ws_ctx* ctx) {
  if (!ctx) {
    set_error(WS_ERR_INVALID, "ctx is NULL");
    return WS_ERR_INVALID;
  }
  WS_CUDA(cudaSetDevice(ctx->device));
  return WS_OK;
}

static ws_status null_arg(const char* name) {
  set_error(WS_ERR_INVALID, "%s must not be NULL", name);
  return WS_ERR_INVALID;
}

static void begin_call(ws_ctx* ctx, const Geo& g) {
  ++ctx->calls;
  std::memset(&ctx->stats, 0, sizeof(ctx->stats));
  ctx->stats.n_voxels = g.N;
}

void tbegin(ws_ctx* ctx, cudaStream_t st) {
  ctx->ev_n = 0;
  if (!ctx->timing) return;
  cudaEventRecord(ctx->ev[0], st);
  ctx->ev_phase[0] = -1;
  ctx->ev_n = 1;
}

void tmark(ws_ctx* ctx, cudaStream_t st, int phase) {
  if (!ctx->timing || ctx->ev_n == 0 || ctx->ev_n >= ws_ctx::MAXEV) return;
  cudaEventRecord(ctx->ev[ctx->ev_n], st);
  ctx->ev_phase[ctx->ev_n] = phase;
  ++ctx->ev_n;
}

void tfinish(ws_ctx* ctx) {
  if (!ctx->timing || ctx->ev_n < 2) return;
  cudaEventSynchronize(ctx->ev[ctx->ev_n - 1]);
  for (int i = 1; i < ctx->ev_n; ++i) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, ctx->ev[i - 1], ctx->ev[i]) == cudaSuccess)
      ctx->stats.phase_ms[ctx->ev_phase[i]] += ms;
  }
  (void)cudaGetLastError();
  ctx->ev_n = 0;
}

typedef CUresult (*PfnEncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PfnEncodeTiled encode_fn() {
  static PfnEncodeTiled fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PfnEncodeTiled>(p);
    (void)cudaGetLastError();
  }
  return fn;
}

bool encode_tmap_3d(void* map, int esize, const void* base, const Geo& g, unsigned bx, unsigned by, unsigned bz) {
  PfnEncodeTiled fn = encode_fn();
  if (!fn) return false;
  const size_t pitch = (size_t)g.n2 * esize, plane = pitch * g.n1;
  if ((reinterpret_cast<uintptr_t>(base) & 15) || (pitch & 15) || (plane & 15)) return false;
  cuuint64_t dims[3] = {(cuuint64_t)g.n2, (cuuint64_t)g.n1, (cuuint64_t)g.n0};
  cuuint64_t strides[2] = {(cuuint64_t)pitch, (cuuint64_t)plane};
  cuuint32_t box[3] = {bx, by, bz};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(reinterpret_cast<CUtensorMap*>(map),
                  esize == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                  : esize == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16 : CU_TENSOR_MAP_DATA_TYPE_INT32, 3,
                  const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

static const char* kPhaseNames[WS_NUM_PHASES] = {
    "gradient.blur", "gradient.magnitude", "watershed.init", "watershed.relax", "watershed.select",
    "watershed.jump", "watershed.union", "watershed.find", "watershed.relabel", "waterfall.dense_ids",
    "waterfall.rag", "waterfall.levels", "waterfall.materialise", "copy", "", ""};

}  // namespace ws

using namespace ws;

extern "C" {

const char* ws_last_error(void) { return g_err; }
const char* ws_version(void) { return "ws_b200 0.1 (sm_100a)"; }

ws_status ws_ctx_create(int32_t device, ws_ctx** out) {
  if (!out) return null_arg("out");
  *out = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || device < 0 || device >= n) {
    set_error(WS_ERR_CUDA, "no CUDA device %d (%d visible%s%s)", device, n, e != cudaSuccess ? ": " : "",
              e != cudaSuccess ? cudaGetErrorString(e) : "");
    (void)cudaGetLastError();
    return WS_ERR_CUDA;
  }
  WS_CUDA(cudaSetDevice(device));
  ws_ctx* c = new (std::nothrow) ws_ctx();
  if (!c) {
    set_error(WS_ERR_OOM, "host allocation failed");
    return WS_ERR_OOM;
  }
  c->device = device;
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  cudaDeviceGetAttribute(&c->coop, cudaDevAttrCooperativeLaunch, device);
  {
    const char* nc = getenv("WS_NO_COOP");
    if (nc && nc[0] == '1') c->coop = 0;
  }
  e = cudaMallocHost(&c->pinned, 256 * sizeof(int64_t));
  if (e != cudaSuccess) {
    delete c;
    return cuda_fail(e, "cudaMallocHost");
  }
  *out = c;
  return WS_OK;
}

ws_status ws_ctx_destroy(ws_ctx* ctx) {
  if (!ctx) return WS_OK;
  cudaSetDevice(ctx->device);
  ws::Buf* bufs[] = {&ctx->aux, &ctx->tmpA, &ctx->tmpB, &ctx->flags, &ctx->tiles, &ctx->roots, &ctx->rootc, &ctx->blockcnt, &ctx->edges, &ctx->ebufA, &ctx->ebufB, &ctx->rootsA, &ctx->rootsB, &ctx->lvl,
                     &ctx->comp, &ctx->best, &ctx->rep_of, &ctx->levelmap, &ctx->lvcount,
                     &ctx->h_grad, &ctx->h_labels, &ctx->h_levels, &ctx->dimg, &ctx->sroots, &ctx->sblocks, &ctx->rank, &ctx->wimg, &ctx->vstate, &ctx->nmin, &ctx->tlist, &ctx->upairs, &ctx->eqc, &ctx->exitmx,
                     &ctx->mtables, &ctx->mslabs, &ctx->mr0, &ctx->mmap, &ctx->pathc, &ctx->best_lo, &ctx->repbits,
                     &ctx->sh_L, &ctx->sh_P, &ctx->sh_planes, &ctx->sh_tab, &ctx->sh_alltab, &ctx->sh_ec, &ctx->sh_lab,
                     &ctx->sh_dense, &ctx->sh_rep, &ctx->sh_bt, &ctx->sh_allbt, &ctx->sh_lext, &ctx->sh_best,
                     &ctx->sh_nxt, &ctx->sh_small, &ctx->fmap};
  for (auto* b : bufs) b->release();
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  if (ctx->sh_small_h) cudaFreeHost(ctx->sh_small_h);
  if (ctx->sg.exec) cudaGraphExecDestroy(ctx->sg.exec);
  if (ctx->cap_st) cudaStreamDestroy(ctx->cap_st);
  for (int i = 0; i < ws_ctx::MAXEV; ++i)
    if (ctx->ev[i]) cudaEventDestroy(ctx->ev[i]);
  delete ctx;
  return WS_OK;
}

const char* ws_phase_name(int32_t i) { return (i >= 0 && i < WS_NUM_PHASES) ? kPhaseNames[i] : ""; }

ws_status ws_ctx_set_timing(ws_ctx* ctx, int32_t enable) {
  WS_TRY(check_ctx(ctx));
  if (enable && !ctx->ev[0]) {
    for (int i = 0; i < ws_ctx::MAXEV; ++i) WS_CUDA(cudaEventCreate(&ctx->ev[i]));
  }
  ctx->timing = enable != 0;
  return WS_OK;
}

ws_status ws_get_stats(const ws_ctx* ctx, ws_stats* out) {
  if (!ctx || !out) return null_arg("ctx/out");
  *out = ctx->stats;
  out->total_launches = ctx->total_launches;
  return WS_OK;
}

ws_status ws_gradient(ws_ctx* ctx, const uint8_t* img, ws_dims dims, float sigma, uint8_t* grad_q,
                      float* blur_f32, float* grad_f32, void* stream) {
  WS_TRY(check_ctx(ctx));
  Geo g;
  WS_TRY(check_dims(dims, &g));
  if (!(sigma >= 0.f) || sigma > 20.f) {
    set_error(WS_ERR_INVALID, "sigma must be in [0, 20] (got %g)", (double)sigma);
    return WS_ERR_INVALID;
  }
  if (!img) return null_arg("img");
  if (!grad_q) return null_arg("grad_q");
  begin_call(ctx, g);
  tbegin(ctx, (cudaStream_t)stream);
  ws_status s = run_gradient(ctx, img, g, dims.ndim == 3, sigma, grad_q, blur_f32, grad_f32, (cudaStream_t)stream);
  tfinish(ctx);
  return s;
}

ws_status ws_gradient_u16(ws_ctx* ctx, const uint16_t* img, ws_dims dims, float sigma, uint16_t* grad_q,
                          float* blur_f32, float* grad_f32, void* stream) {
  WS_TRY(check_ctx(ctx));
  Geo g;
  WS_TRY(check_dims(dims, &g));
  if (!(sigma >= 0.f) || sigma > 20.f) {
    set_error(WS_ERR_INVALID, "sigma must be in [0, 20] (got %g)", (double)sigma);
    return WS_ERR_INVALID;
  }
  if (!img) return null_arg("img");
  if (!grad_q) return null_arg("grad_q");
  if ((reinterpret_cast<uintptr_t>(img) | reinterpret_cast<uintptr_t>(grad_q)) & 1) {
    set_error(WS_ERR_INVALID, "img and grad_q must be 2-byte aligned");
    return WS_ERR_INVALID;
  }
  begin_call(ctx, g);
  tbegin(ctx, (cudaStream_t)stream);
  ws_status s =
      run_gradient_u16(ctx, img, g, dims.ndim == 3, sigma, grad_q, blur_f32, grad_f32, (cudaStream_t)stream);
  tfinish(ctx);
  return s;
}

ws_status ws_watershed(ws_ctx* ctx, const uint8_t* grad, ws_dims dims, int32_t connectivity, int32_t* labels,
                       int64_t* num_regions, void* stream) {
  WS_TRY(check_ctx(ctx));
  Geo g;
  WS_TRY(check_dims(dims, &g));
  WS_TRY(check_conn(dims, connectivity));
  if (!grad) return null_arg("grad");
  if (!labels) return null_arg("labels");
  begin_call(ctx, g);
  if (ctx->sharded) return sharded_dispatch_watershed(ctx, grad, dims, connectivity, labels, num_regions, (cudaStream_t)stream);
  tbegin(ctx, (cudaStream_t)stream);
  ws_status s = run_watershed(ctx, grad, g, connectivity, labels, num_regions, (cudaStream_t)stream);
  tfinish(ctx);
  return s;
}

ws_status ws_watershed_u16(ws_ctx* ctx, const uint16_t* grad, ws_dims dims, int32_t connectivity,
                           int32_t* labels, int64_t* num_regions, void* stream) {
  WS_TRY(check_ctx(ctx));
  Geo g;
  WS_TRY(check_dims(dims, &g));
  WS_TRY(check_conn(dims, connectivity));
  if (!grad) return null_arg("grad");
  if (!labels) return null_arg("labels");
  if (reinterpret_cast<uintptr_t>(grad) & 1) {
    set_error(WS_ERR_INVALID, "grad must be 2-byte aligned");
    return WS_ERR_INVALID;
  }
  begin_call(ctx, g);
  if (ctx->sharded)
    return sharded_dispatch_watershed_u16(ctx, grad, dims, connectivity, labels, num_regions, (cudaStream_t)stream);
  tbegin(ctx, (cudaStream_t)stream);
  ws_status s = px16::run_watershed(ctx, grad, g, connectivity, labels, num_regions, (cudaStream_t)stream);
  tfinish(ctx);
  return s;
}

ws_status ws_waterfall(ws_ctx* ctx, const int32_t* labels, const uint8_t* grad, ws_dims dims, int32_t connectivity,
                       int32_t NL, int32_t* levels, int64_t* counts, void* stream) {
  WS_TRY(check_ctx(ctx));
  Geo g;
  WS_TRY(check_dims(dims, &g));
  WS_TRY(check_conn(dims, connectivity));
  if (NL < 1) {
    set_error(WS_ERR_INVALID, "NL must be >= 1 (got %d)", NL);
    return WS_ERR_INVALID;
  }
  if (!labels) return null_arg("labels");
  if (!grad) return null_arg("grad");
  if (!levels) return null_arg("levels");
  if (ctx->sharded) {
    begin_call(ctx, g);
    return sharded_dispatch_waterfall(ctx, labels, grad, dims, connectivity, NL, levels, counts, (cudaStream_t)stream);
  }
  begin_call(ctx, g);
  tbegin(ctx, (cudaStream_t)stream);
  ws_status s = run_waterfall(ctx, labels, grad, g, connectivity, NL, levels, counts, (cudaStream_t)stream);
  tfinish(ctx);
  return s;
}

ws_status ws_waterfall_u16(ws_ctx* ctx, const int32_t* labels, const uint16_t* grad, ws_dims dims, int32_t connectivity,
                           int32_t NL, int32_t* levels, int64_t* counts, void* stream) {
  WS_TRY(check_ctx(ctx));
  Geo g;
  WS_TRY(check_dims(dims, &g));
  WS_TRY(check_conn(dims, connectivity));
  if (NL < 1) {
    set_error(WS_ERR_INVALID, "NL must be >= 1 (got %d)", NL);
    return WS_ERR_INVALID;
  }
  if (!labels) return null_arg("labels");
  if (!grad) return null_arg("grad");
  if (!levels) return null_arg("levels");
  if (reinterpret_cast<uintptr_t>(grad) & 1) {
    set_error(WS_ERR_INVALID, "grad must be 2-byte aligned");
    return WS_ERR_INVALID;
  }
  begin_call(ctx, g);
  if (ctx->sharded)
    return sharded_dispatch_waterfall_u16(ctx, labels, grad, dims, connectivity, NL, levels, counts,
                                          (cudaStream_t)stream);
  tbegin(ctx, (cudaStream_t)stream);
  ws_status s = run_waterfall_u16(ctx, labels, grad, g, connectivity, NL, levels, counts, (cudaStream_t)stream);
  tfinish(ctx);
  return s;
}

ws_status ws_watershed_variant(ws_ctx* ctx, const uint8_t* grad, ws_dims dims, int32_t connectivity, int32_t variant,
                               int32_t* labels, int64_t* num_regions, void* stream) {
  WS_TRY(check_ctx(ctx));
  Geo g;
  WS_TRY(check_dims(dims, &g));
  WS_TRY(check_conn(dims, connectivity));
  if (variant != WS_VARIANT_PRUF_SYNC && variant != WS_VARIANT_PRW_SYNC && variant != WS_VARIANT_APRUF_SYNC) {
    set_error(WS_ERR_INVALID, "unknown watershed variant %d", variant);
    return WS_ERR_INVALID;
  }
  if (!grad) return null_arg("grad");
  if (!labels) return null_arg("labels");
  begin_call(ctx, g);
  tbegin(ctx, (cudaStream_t)stream);
  ws_status s = run_watershed_variant(ctx, grad, g, connectivity, variant, labels, num_regions, (cudaStream_t)stream);
  tfinish(ctx);
  return s;
}

ws_status ws_waterfall_reconstruct(ws_ctx* ctx, const int32_t* labels, const uint8_t* grad, ws_dims dims,
                                   int32_t connectivity, int32_t NL, int32_t* levels, int64_t* counts, void* stream) {
  WS_TRY(check_ctx(ctx));
  Geo g;
  WS_TRY(check_dims(dims, &g));
  WS_TRY(check_conn(dims, connectivity));
  if (NL < 1) {
    set_error(WS_ERR_INVALID, "NL must be >= 1 (got %d)", NL);
    return WS_ERR_INVALID;
  }
  if (!labels) return null_arg("labels");
  if (!grad) return null_arg("grad");
  if (!levels) return null_arg("levels");
  begin_call(ctx, g);
  tbegin(ctx, (cudaStream_t)stream);
  ws_status s = run_waterfall_reconstruct(ctx, labels, grad, g, connectivity, NL, levels, counts, (cudaStream_t)stream);
  tfinish(ctx);
  return s;
}

ws_status ws_segment(ws_ctx* ctx, const uint8_t* grad, ws_dims dims, int32_t connectivity, int32_t NL,
                     int32_t* levels, int64_t* counts, void* stream) {
  WS_TRY(check_ctx(ctx));
  Geo g;
  WS_TRY(check_dims(dims, &g));
  WS_TRY(check_conn(dims, connectivity));
  if (NL < 1) {
    set_error(WS_ERR_INVALID, "NL must be >= 1 (got %d)", NL);
    return WS_ERR_INVALID;
  }
  if (!grad) return null_arg("grad");
  if (!levels) return null_arg("levels");
  begin_call(ctx, g);
  if (ctx->sharded) return sharded_dispatch_segment(ctx, grad, dims, connectivity, NL, levels, counts, (cudaStream_t)stream);
  tbegin(ctx, (cudaStream_t)stream);
  ws_status s = run_segment(ctx, grad, g, connectivity, NL, levels, counts, (cudaStream_t)stream);
  tfinish(ctx);
  return s;
}

static ws_status segment_host_impl(ws_ctx* ctx, const uint8_t* grad_host, ws_dims dims, int32_t connectivity,
                                   int32_t NL, int32_t* levels_host, int64_t* counts, void* stream, bool wait) {
  WS_TRY(check_ctx(ctx));
  Geo g;
  WS_TRY(check_dims(dims, &g));
  WS_TRY(check_conn(dims, connectivity));
  if (NL < 1) {
    set_error(WS_ERR_INVALID, "NL must be >= 1 (got %d)", NL);
    return WS_ERR_INVALID;
  }
  if (!grad_host) return null_arg("grad_host");
  if (!levels_host) return null_arg("levels_host");
  cudaStream_t st = (cudaStream_t)stream;
  const size_t N = (size_t)g.N;
  WS_TRY(ctx->h_grad.ensure(N, "segment grad"));
  WS_TRY(ctx->h_levels.ensure(N * (size_t)NL * sizeof(int32_t), "segment levels"));
  begin_call(ctx, g);
  tbegin(ctx, st);
  WS_CUDA(cudaMemcpyAsync(ctx->h_grad.p, grad_host, N, cudaMemcpyHostToDevice, st));
  tmark(ctx, st, PH_COPY);
  WS_TRY(run_segment(ctx, ctx->h_grad.as<uint8_t>(), g, connectivity, NL, ctx->h_levels.as<int32_t>(), counts, st));
  WS_CUDA(cudaMemcpyAsync(levels_host, ctx->h_levels.p, N * (size_t)NL * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  tmark(ctx, st, PH_COPY);
  if (!wait) return WS_OK;  // the caller synchronises the stream (per-phase timing not collected)
  WS_CUDA(cudaStreamSynchronize(st));
  tfinish(ctx);
  return WS_OK;
}

ws_status ws_segment_host(ws_ctx* ctx, const uint8_t* grad_host, ws_dims dims, int32_t connectivity, int32_t NL,
                          int32_t* levels_host, int64_t* counts, void* stream) {
  return segment_host_impl(ctx, grad_host, dims, connectivity, NL, levels_host, counts, stream, true);
}

ws_status ws_segment_host_async(ws_ctx* ctx, const uint8_t* grad_host, ws_dims dims, int32_t connectivity,
                                int32_t NL, int32_t* levels_host, int64_t* counts, void* stream) {
  return segment_host_impl(ctx, grad_host, dims, connectivity, NL, levels_host, counts, stream, false);
}

ws_status ws_plateau_debug(ws_ctx* ctx, const uint8_t* grad, ws_dims dims, int32_t connectivity, int32_t* dist,
                           int32_t* parent, void* stream) {
  WS_TRY(check_ctx(ctx));
  Geo g;
  WS_TRY(check_dims(dims, &g));
  WS_TRY(check_conn(dims, connectivity));
  if (!grad) return null_arg("grad");
  if (!dist || !parent) return null_arg("dist/parent");
  begin_call(ctx, g);
  ws_status s = run_plateau_debug(ctx, grad, g, connectivity, dist, parent, (cudaStream_t)stream);
  ctx->ev_n = 0;
  return s;
}

// ------------------------------------------------------------------ z-slab sharding
static ws_status check_slab(const ws_dims& d, const ws_slab& sl, int conn, Geo* g) {
  WS_TRY(check_dims(d, g));
  if (d.ndim != 3 || (conn != 6 && conn != 26)) {
    set_error(WS_ERR_INVALID, "the sharded path supports 3-D volumes with 6- or 26-connectivity");
    return WS_ERR_INVALID;
  }
  const int64_t plane = d.n1 * d.n2;
  if (!(0 <= sl.e0 && sl.e0 <= sl.z0 && sl.z0 < sl.z1 && sl.z1 <= sl.e1 && sl.e1 <= sl.D) ||
      d.n0 != sl.e1 - sl.e0 || (double)sl.D * (double)plane >= 2147483648.0 ||
      (sl.z0 > 0 && sl.e0 > sl.z0 - 1) || (sl.z1 < sl.D && sl.e1 < sl.z1 + 1)) {
    set_error(WS_ERR_INVALID, "inconsistent slab (D=%lld z=[%lld,%lld) e=[%lld,%lld) n0=%lld)", (long long)sl.D,
              (long long)sl.z0, (long long)sl.z1, (long long)sl.e0, (long long)sl.e1, (long long)d.n0);
    return WS_ERR_INVALID;
  }
  g->zlo = (int)(sl.z0 - sl.e0);
  g->zhi = (int)(sl.z1 - sl.e0);
  g->gofs = (int)(sl.e0 * plane);
  return WS_OK;
}

int64_t ws_shard_table_bytes(ws_dims d) { return (int64_t)d.n1 * d.n2 * 28; }

ws_status ws_shard_plateau(ws_ctx* ctx, const uint8_t* grad_ext, ws_dims dims, int32_t conn, ws_slab slab,
                           int32_t* L_ext, int32_t phase, int32_t act_lo, int32_t act_hi, int32_t* pending,
                           void* stream) {
  WS_TRY(check_ctx(ctx));
  Geo g;
  WS_TRY(check_slab(dims, slab, conn, &g));
  if (!grad_ext || !L_ext || !pending) return null_arg("grad_ext/L_ext/pending");
  begin_call(ctx, g);
  int pend = 0;
  ws_status s = phase == 0 ? plateau_first_shard(ctx, grad_ext, g, conn, L_ext, &pend, (cudaStream_t)stream)
                           : plateau_round_shard(ctx, grad_ext, g, conn, L_ext, act_lo, act_hi, &pend,
                                                 (cudaStream_t)stream);
  *pending = pend;
  return s;
}

ws_status ws_shard_halo(ws_ctx* ctx, int32_t* L_ext, ws_dims dims, ws_slab slab, int32_t side,
                        const int32_t* plane_in, int32_t* changed, void* stream) {
  WS_TRY(check_ctx(ctx));
  Geo g;
  WS_TRY(check_slab(dims, slab, 6, &g));
  if (!L_ext || !plane_in || !changed) return null_arg("L_ext/plane_in/changed");
  if ((side == 0 && g.zlo < 1) || (side == 1 && g.zhi >= g.n0) || (side != 0 && side != 1)) {
    set_error(WS_ERR_INVALID, "no halo plane on side %d", side);
    return WS_ERR_INVALID;
  }
  return shard_halo(ctx, L_ext, g, side, plane_in, changed, (cudaStream_t)stream);
}

ws_status ws_shard_local(ws_ctx* ctx, const uint8_t* grad_ext, int32_t* L_ext, ws_dims dims, int32_t conn,
                         ws_slab slab, int32_t* P_ext, void* table, void* stream) {
  WS_TRY(check_ctx(ctx));
  Geo g;
  WS_TRY(check_slab(dims, slab, conn, &g));
  if (!grad_ext || !L_ext || !P_ext || !table) return null_arg("grad_ext/L_ext/P_ext/table");
  begin_call(ctx, g);
  return shard_local(ctx, grad_ext, g, conn, L_ext, P_ext, table, (cudaStream_t)stream);
}

ws_status ws_shard_merge(ws_ctx* ctx, const void* tables_all, int32_t nranks, const int64_t* z0s, const int64_t* z1s,
                         ws_dims dims, ws_slab slab, int32_t* L_ext, int32_t* exitcanon, void* stream) {
  WS_TRY(check_ctx(ctx));
  Geo g;
  WS_TRY(check_slab(dims, slab, 6, &g));
  if (!tables_all || !z0s || !z1s || !L_ext || !exitcanon) return null_arg("tables/z0s/z1s/L_ext/exitcanon");
  int rank = -1;
  for (int r = 0; r < nranks; ++r) {
    if (r > 0 && z0s[r] != z1s[r - 1]) {
      set_error(WS_ERR_INVALID, "slabs must tile [0, D) in order");
      return WS_ERR_INVALID;
    }
    if (z0s[r] == slab.z0 && z1s[r] == slab.z1) rank = r;
  }
  if (rank < 0 || nranks < 1 || z0s[0] != 0 || z1s[nranks - 1] != slab.D) {
    set_error(WS_ERR_INVALID, "slab not among the nranks slabs / slabs do not cover [0, D)");
    return WS_ERR_INVALID;
  }
  return shard_merge(ctx, tables_all, z0s, z1s, nranks, rank, g, L_ext, exitcanon, (cudaStream_t)stream);
}

ws_status ws_shard_relabel(ws_ctx* ctx, const int32_t* P_ext, int32_t* L_ext, const int32_t* exitcanon, ws_dims dims,
                           ws_slab slab, int32_t* labels_own, int64_t* nreps, void* stream) {
  WS_TRY(check_ctx(ctx));
  Geo g;
  WS_TRY(check_slab(dims, slab, 6, &g));
  if (!P_ext || !L_ext || !exitcanon || !labels_own) return null_arg("P_ext/L_ext/exitcanon/labels_own");
  return shard_relabel(ctx, P_ext, L_ext, exitcanon, g, labels_own, nreps, (cudaStream_t)stream);
}

ws_status ws_shard_wf_dense(ws_ctx* ctx, const int32_t* labels_own, ws_dims dims, ws_slab slab, int64_t doff,
                            int32_t* dense_of, int32_t* rep_of, int64_t* count, void* stream) {
  WS_TRY(check_ctx(ctx));
  Geo g;
  WS_TRY(check_slab(dims, slab, 6, &g));
  if (!labels_own || !dense_of || !rep_of || !count) return null_arg("labels_own/dense_of/rep_of/count");
  begin_call(ctx, g);
  const int n = (g.zhi - g.zlo) * g.plane;
  return shard_wf_dense(ctx, labels_own, n, (int)(slab.z0 * g.plane), (int)doff, dense_of, rep_of, count,
                        (cudaStream_t)stream);
}

ws_status ws_shard_wf_btable(ws_ctx* ctx, const int32_t* labels_own, const int32_t* dense_of, ws_dims dims,
                             ws_slab slab, int32_t* btable, void* stream) {
  WS_TRY(check_ctx(ctx));
  Geo g;
  WS_TRY(check_slab(dims, slab, 6, &g));
  if (!labels_own || !dense_of || !btable) return null_arg("labels_own/dense_of/btable");
  return shard_wf_btable(ctx, labels_own, g.zhi - g.zlo, g.plane, (int)(slab.z0 * g.plane), dense_of, btable,
                         (cudaStream_t)stream);
}

ws_status ws_shard_wf_bfill(ws_ctx* ctx, const int32_t* btables_all, int32_t nranks, ws_dims dims, ws_slab slab,
                            int32_t* dense_of, void* stream) {
  WS_TRY(check_ctx(ctx));
  Geo g;
  WS_TRY(check_slab(dims, slab, 6, &g));
  if (!btables_all || !dense_of || nranks < 1) return null_arg("btables_all/dense_of");
  return shard_wf_bfill(ctx, btables_all, nranks, g.plane, (int)(slab.z0 * g.plane), (int)((slab.z1 + 1) * g.plane),
                        dense_of, (cudaStream_t)stream);
}

ws_status ws_shard_wf_begin(ws_ctx* ctx, const int32_t* labels_ext, const uint8_t* grad_ext, ws_dims dims,
                            int32_t conn, ws_slab slab, const int32_t* dense_of, int64_t R, int32_t NL,
                            int64_t* best_out, void* stream) {
  WS_TRY(check_ctx(ctx));
  Geo g;
  WS_TRY(check_slab(dims, slab, conn, &g));
  if (!labels_ext || !grad_ext || !dense_of || !best_out) return null_arg("labels_ext/grad_ext/dense_of/best_out");
  if (NL < 1) {
    set_error(WS_ERR_INVALID, "NL must be >= 1 (got %d)", NL);
    return WS_ERR_INVALID;
  }
  begin_call(ctx, g);
  return shard_wf_begin(ctx, labels_ext, grad_ext, g, conn, dense_of, R, NL,
                        reinterpret_cast<uint64_t*>(best_out), (cudaStream_t)stream);
}

ws_status ws_shard_wf_step(ws_ctx* ctx, const int64_t* best_in, int64_t* best_out, int64_t* count, int32_t* more,
                           void* stream) {
  WS_TRY(check_ctx(ctx));
  if (!best_in || !best_out || !count || !more) return null_arg("best_in/best_out/count/more");
  int m = 0;
  ws_status s = shard_wf_step(ctx, reinterpret_cast<const uint64_t*>(best_in), reinterpret_cast<uint64_t*>(best_out),
                              count, &m, (cudaStream_t)stream);
  *more = m;
  return s;
}

ws_status ws_shard_wf_end(ws_ctx* ctx, const int32_t* labels_own, const int32_t* dense_of, const int32_t* rep_of,
                          ws_dims dims, int32_t conn, ws_slab slab, int32_t* levels_own, void* stream) {
  WS_TRY(check_ctx(ctx));
  Geo g;
  WS_TRY(check_slab(dims, slab, conn, &g));
  if (!labels_own || !dense_of || !rep_of || !levels_own) return null_arg("labels_own/dense_of/rep_of/levels_own");
  Geo go = g;  // the owned planes as their own volume (labels_own / levels_own layout)
  go.n0 = g.zhi - g.zlo;
  go.N = go.n0 * go.plane;
  go.zlo = 0;
  go.zhi = go.n0;
  go.gofs = 0;
  return shard_wf_end(ctx, labels_own, go, conn, dense_of, rep_of, levels_own, (cudaStream_t)stream);
}

}  // extern "C"
