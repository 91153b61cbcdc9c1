// ws_variants.cu — the paper's own watershed kernels, one thread per voxel, as written in
// Alg. 1 (PRUF_sync), Alg. 2 (PRW step IV) and APRUF
// (step III by Find): SURVEY NEXT f3.  They are the baseline the tiled design of
// ws_watershed.cu is measured against; all give the same partition, and the
// output is canonicalised (C7) like ws_watershed's.
//
//   k_v_init      step I (Alg. 1 l.1-10): q = max-index minimal neighbour (Eq. 1); states 0-3
//   k_v_plateau   step II (l.11-18), Jacobi S -> S', the state-0 neighbour of equal value with
//                 the largest index (C5); host loop until no change
//   k_v_jump      step III (l.19-23): up to RR = 6 jumps per launch; host loop until no change
//   k_v_findall   APRUF step III / PRUF l.28-29: L(p) = Find(L, p), independently per thread
//   k_v_union     PRUF step IV (l.24-27): min-root Union over q > p with S(p), S(q) >= 2
//   k_v_prw       PRW step IV (Alg. 2 l.19-31): min-merging of the two labels' representatives,
//                 then path reduction; host loop until no change
//   k_v_canon_*   canonical labels: smallest voxel index per final root
#include <climits>

#include "ws_internal.h"

namespace ws {

constexpr int RR = 6;

template <int CONN>
__global__ void k_v_init(const uint8_t* __restrict__ I, Geo g, int* __restrict__ L, uint8_t* __restrict__ S) {
  ZLOOP_BEGIN_R
  const int v = I[p];
  int q = -1, m = 256;
#pragma unroll
  for (int i = 0; i < CONN; ++i) {  // neighbours in increasing index order: "<=" keeps the last
    if (!nb_in<CONN>(g, z, y, x, i)) continue;
    const int r = p + nb_off<CONN>(g, i);
    const int w = I[r];
    if (w <= m) { m = w; q = r; }
  }
  if (q < 0 || m > v) { L[p] = p; S[p] = 1; }  // empty N(p) (C4) or strict minimum
  else if (m < v) { L[p] = q; S[p] = 0; }
  else if (q > p) { L[p] = q; S[p] = 2; }
  else { L[p] = p; S[p] = 3; }
  ZLOOP_END_R
}

template <int CONN>
__global__ void k_v_plateau(const uint8_t* __restrict__ I, Geo g, int* __restrict__ L, const uint8_t* __restrict__ S,
                            uint8_t* __restrict__ S2, int* changed) {
  ZLOOP_BEGIN_R
  const int s = S[p];
  int q = -1;
  if (s >= 2) {
    const int v = I[p];
#pragma unroll
    for (int i = 0; i < CONN; ++i) {
      if (!nb_in<CONN>(g, z, y, x, i)) continue;
      const int r = p + nb_off<CONN>(g, i);
      if (S[r] == 0 && I[r] == v) q = r;  // the largest index (C5)
    }
  }
  if (q >= 0) {
    L[p] = q;
    S2[p] = 0;
    *changed = 1;
  } else {
    S2[p] = (uint8_t)s;
  }
  ZLOOP_END_R
}

__global__ void k_v_jump(int* L, long long N, int* changed) {
  bool ch = false;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < N; p += (long long)gridDim.x * blockDim.x) {
    int l = L[p];
    for (int i = 0; i < RR; ++i) {
      const int ll = L[l];
      if (ll == l) break;
      l = ll;
      ch = true;
    }
    L[p] = l;
  }
  if (__syncthreads_or(ch) && threadIdx.x == 0) *changed = 1;
}

__device__ __forceinline__ int v_find(const int* L, int x) {
  while (true) {
    const int y = __ldcg(L + x);
    if (y == x) return x;
    x = y;
  }
}

__global__ void k_v_findall(int* L, long long N) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < N; p += (long long)gridDim.x * blockDim.x)
    L[p] = v_find(L, (int)p);
}

template <int CONN>
__global__ void k_v_union(Geo g, int* L, const uint8_t* __restrict__ S) {
  ZLOOP_BEGIN_R
  if (S[p] < 2) continue;
#pragma unroll
  for (int i = Conn<CONN>::nfwd; i < CONN; ++i) {  // q > p
    if (!nb_in<CONN>(g, z, y, x, i)) continue;
    const int q = p + nb_off<CONN>(g, i);
    if (S[q] < 2) continue;
    int a = p, b = q;
    while (true) {
      a = v_find(L, a);
      b = v_find(L, b);
      if (a == b) break;
      if (a > b) { const int t = a; a = b; b = t; }
      if (atomicCAS(L + b, b, a) == b) break;
    }
  }
  ZLOOP_END_R
}

// PRW step IV (Alg. 2): merge the representatives' labels towards the minimum (atomicMin:
// the two assignments of l.23-24 without lost updates), then reduce the path of p
template <int CONN>
__global__ void k_v_prw(Geo g, int* L, const uint8_t* __restrict__ S, int* changed) {
  ZLOOP_BEGIN_R
  bool ch = false;
  if (S[p] >= 2) {
#pragma unroll
    for (int i = Conn<CONN>::nfwd; i < CONN; ++i) {
      if (!nb_in<CONN>(g, z, y, x, i)) continue;
      const int q = p + nb_off<CONN>(g, i);
      if (S[q] < 2) continue;
      const int lp = __ldcg(L + p), lq = __ldcg(L + q);
      while (true) {
        const int a = __ldcg(L + lp), b = __ldcg(L + lq);
        if (a == b) break;
        const int m = min(a, b);
        atomicMin(L + lp, m);
        atomicMin(L + lq, m);
        ch = true;
      }
    }
  }
  while (true) {
    const int l = __ldcg(L + p), ll = __ldcg(L + l);
    if (l == ll) break;
    atomicMin(L + p, ll);
    ch = true;
  }
  if (ch) *changed = 1;
  ZLOOP_END_R
}

__global__ void k_v_canon_min(const int* __restrict__ L, long long N, int* __restrict__ canon) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < N; p += (long long)gridDim.x * blockDim.x)
    atomicMin(canon + L[p], (int)p);
}

__global__ void k_v_canon_apply(int* L, const int* __restrict__ canon, long long N, unsigned long long* R) {
  unsigned long long c = 0;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < N; p += (long long)gridDim.x * blockDim.x) {
    const int cl = canon[L[p]];
    c += cl == p;
    L[p] = cl;
  }
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(R, c);
}

__global__ void k_v_fill(int* a, long long n, int v) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    a[i] = v;
}

static ws_status read_flag(ws_ctx* ctx, int* dflag, int* out, cudaStream_t st) {
  WS_CUDA(cudaMemcpyAsync(ctx->pinned, dflag, sizeof(int), cudaMemcpyDeviceToHost, st));
  WS_CUDA(cudaStreamSynchronize(st));
  *out = reinterpret_cast<const int*>(ctx->pinned)[0];
  return WS_OK;
}

template <int CONN>
static ws_status variant_t(ws_ctx* ctx, const uint8_t* grad, const Geo& g, int variant, int32_t* L,
                           int64_t* num_regions, cudaStream_t st) {
  const long long N = g.N;
  WS_TRY(ctx->flags.ensure(256, "flags"));
  WS_TRY(ctx->vstate.ensure((size_t)2 * N, "variant states"));
  WS_TRY(ctx->aux.ensure((size_t)N * sizeof(int), "aux"));
  uint8_t* S = ctx->vstate.as<uint8_t>();
  uint8_t* S2 = S + N;
  int* flag = ctx->flags.as<int>() + 40;
  unsigned long long* R = reinterpret_cast<unsigned long long*>(ctx->flags.as<char>() + 192);
  const L3 l = launch3(g);
  const int g1 = std::max(1, (int)std::min<long long>((N + 255) / 256, (long long)ctx->num_sms * 16));
  k_v_init<CONN><<<l.grid, l.block, 0, st>>>(grad, g, L, S);
  launched(ctx, PH_WS_INIT);
  tmark(ctx, st, PH_WS_INIT);
  int rounds = 0, ch = 1;
  while (ch) {  // step II
    WS_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), st));
    k_v_plateau<CONN><<<l.grid, l.block, 0, st>>>(grad, g, L, S, S2, flag);
    launched(ctx, PH_WS_RELAX);
    std::swap(S, S2);
    ++rounds;
    WS_TRY(read_flag(ctx, flag, &ch, st));
  }
  ctx->stats.plateau_rounds = rounds;
  tmark(ctx, st, PH_WS_RELAX);
  if (variant == WS_VARIANT_APRUF_SYNC) {  // step III by independent Finds (l.28-29)
    k_v_findall<<<g1, 256, 0, st>>>(L, N);
    launched(ctx, PH_WS_JUMP);
  } else {
    ch = 1;
    while (ch) {  // step III (l.19-23), RR jumps per launch
      WS_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), st));
      k_v_jump<<<g1, 256, 0, st>>>(L, N, flag);
      launched(ctx, PH_WS_JUMP);
      WS_TRY(read_flag(ctx, flag, &ch, st));
    }
  }
  tmark(ctx, st, PH_WS_JUMP);
  if (variant == WS_VARIANT_PRW_SYNC) {  // step IV of PRW (Alg. 2), until no change
    ch = 1;
    while (ch) {
      WS_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), st));
      k_v_prw<CONN><<<l.grid, l.block, 0, st>>>(g, L, S, flag);
      launched(ctx, PH_WS_UNION);
      WS_TRY(read_flag(ctx, flag, &ch, st));
    }
    tmark(ctx, st, PH_WS_UNION);
  } else {  // step IV of PRUF: Union, then Find for every voxel
    k_v_union<CONN><<<l.grid, l.block, 0, st>>>(g, L, S);
    launched(ctx, PH_WS_UNION);
    tmark(ctx, st, PH_WS_UNION);
    k_v_findall<<<g1, 256, 0, st>>>(L, N);
    launched(ctx, PH_WS_FIND);
    tmark(ctx, st, PH_WS_FIND);
  }
  // canonical labels (C7)
  int* canon = ctx->aux.as<int>();
  k_v_fill<<<g1, 256, 0, st>>>(canon, N, INT_MAX);
  k_v_canon_min<<<g1, 256, 0, st>>>(L, N, canon);
  WS_CUDA(cudaMemsetAsync(R, 0, sizeof(unsigned long long), st));
  k_v_canon_apply<<<g1, 256, 0, st>>>(L, canon, N, R);
  launched(ctx, PH_WS_RELABEL, 3);
  tmark(ctx, st, PH_WS_RELABEL);
  WS_CUDA(cudaGetLastError());
  WS_CUDA(cudaMemcpyAsync(ctx->pinned, R, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  WS_CUDA(cudaStreamSynchronize(st));
  ctx->stats.n_regions = (int64_t)ctx->pinned[0];
  if (num_regions) *num_regions = (int64_t)ctx->pinned[0];
  return WS_OK;
}

ws_status run_watershed_variant(ws_ctx* ctx, const uint8_t* grad, const Geo& g, int conn, int variant,
                                int32_t* labels, int64_t* num_regions, cudaStream_t st) {
  switch (conn) {
    case 4: return variant_t<4>(ctx, grad, g, variant, labels, num_regions, st);
    case 8: return variant_t<8>(ctx, grad, g, variant, labels, num_regions, st);
    case 6: return variant_t<6>(ctx, grad, g, variant, labels, num_regions, st);
    case 26: return variant_t<26>(ctx, grad, g, variant, labels, num_regions, st);
  }
  set_error(WS_ERR_INVALID, "connectivity must be 4, 8, 6 or 26");
  return WS_ERR_INVALID;
}

}  // namespace ws
