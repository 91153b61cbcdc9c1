// ws_reconstruct.cu — the paper-literal waterfall by image reconstruction:
// Alg. 4 steps V-VI between watershed applications (Alg. 5).
//
//   k_newmin   step V: for every voxel p with a neighbour q in another region,
//              newmin(L(p)) = min(newmin(L(p)), max(I(p), I(q)))  (stored as 255 - newmin with
//              a RED max, so a zero memset initialises newmin to M = 255, reading C23)
//   k_raise    step VI: I(p) = max(I(p), newmin(L(p)))
//   then the full watershed (ws_watershed.cu) of the raised image gives the next layer.
// newmin is indexed by the canonical label (a voxel index), so no compaction is needed.
#include <climits>

#include "ws_internal.h"

namespace ws {

constexpr int NTR = 256;

template <int CONN>
__global__ void __launch_bounds__(NTR) k_newmin(const int* __restrict__ L, const uint8_t* __restrict__ I, Geo g,
                                                unsigned* __restrict__ nm) {
  ZLOOP_BEGIN_R
  const int l = L[p];
  const unsigned v = I[p];
  unsigned m = 256;
#pragma unroll
  for (int i = 0; i < CONN; ++i) {
    if (!nb_in<CONN>(g, z, y, x, i)) continue;
    const int q = p + nb_off<CONN>(g, i);
    if (L[q] != l) m = min(m, max(v, (unsigned)I[q]));
  }
  if (m < 256) atomicMax(nm + l, 255u - m);
  ZLOOP_END_R
}

__global__ void k_raise(const int* __restrict__ L, uint8_t* __restrict__ I, const unsigned* __restrict__ nm,
                        long long N) {
  for (long long p = blockIdx.x * (long long)NTR + threadIdx.x; p < N; p += (long long)gridDim.x * NTR) {
    const unsigned nmin = 255u - nm[L[p]];
    if (I[p] < nmin) I[p] = (uint8_t)nmin;
  }
}

__global__ void k_count_reps(const int* __restrict__ L, long long N, unsigned long long* R) {
  unsigned long long c = 0;
  for (long long p = blockIdx.x * (long long)NTR + threadIdx.x; p < N; p += (long long)gridDim.x * NTR)
    c += L[p] == p;
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(R, c);
}

template <int CONN>
static void newmin_t(const int* L, const uint8_t* I, const Geo& g, unsigned* nm, cudaStream_t st) {
  const L3 l = launch3(g);
  k_newmin<CONN><<<l.grid, l.block, 0, st>>>(L, I, g, nm);
}

ws_status run_waterfall_reconstruct(ws_ctx* ctx, const int32_t* labels, const uint8_t* grad, const Geo& g, int conn,
                                    int NL, int32_t* levels, int64_t* counts, cudaStream_t st) {
  const size_t N = (size_t)g.N;
  WS_TRY(ctx->flags.ensure(256, "flags"));
  WS_TRY(ctx->wimg.ensure(N, "reconstructed image"));
  WS_TRY(ctx->nmin.ensure(N * sizeof(unsigned), "new minima"));
  uint8_t* Iw = ctx->wimg.as<uint8_t>();
  unsigned* nm = ctx->nmin.as<unsigned>();
  unsigned long long* R0 = reinterpret_cast<unsigned long long*>(ctx->flags.as<char>() + 200);
  WS_CUDA(cudaMemcpyAsync(Iw, grad, N, cudaMemcpyDeviceToDevice, st));
  WS_CUDA(cudaMemcpyAsync(levels, labels, N * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
  WS_CUDA(cudaMemsetAsync(R0, 0, sizeof(unsigned long long), st));
  const int gN = std::max(1, std::min((int)((N + NTR - 1) / NTR), ctx->num_sms * 16));
  k_count_reps<<<gN, NTR, 0, st>>>(labels, (long long)N, R0);
  launched(ctx, PH_WF_DENSE);
  WS_CUDA(cudaMemcpyAsync(ctx->pinned, R0, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  WS_CUDA(cudaStreamSynchronize(st));
  int64_t R = (int64_t)ctx->pinned[0];
  if (counts) counts[0] = R;
  ctx->stats.level_counts[0] = R;
  int lv = 0;
  for (int k = 1; k < NL; ++k) {
    const int32_t* prev = levels + (size_t)(k - 1) * N;
    int32_t* cur = levels + (size_t)k * N;
    WS_CUDA(cudaMemsetAsync(nm, 0, N * sizeof(unsigned), st));  // newmin = M = 255
    switch (conn) {
      case 4: newmin_t<4>(prev, Iw, g, nm, st); break;
      case 8: newmin_t<8>(prev, Iw, g, nm, st); break;
      case 6: newmin_t<6>(prev, Iw, g, nm, st); break;
      default: newmin_t<26>(prev, Iw, g, nm, st); break;
    }
    k_raise<<<gN, NTR, 0, st>>>(prev, Iw, nm, (long long)N);
    launched(ctx, PH_WF_LEVELS, 2);
    tmark(ctx, st, PH_WF_LEVELS);
    int64_t Rk = 0;
    WS_TRY(run_watershed(ctx, Iw, g, conn, cur, &Rk, st));
    if (counts) counts[k] = Rk;
    if (k < 16) ctx->stats.level_counts[k] = Rk;
    if (Rk < R) lv = k;
    R = Rk;
  }
  ctx->stats.waterfall_levels = lv;
  ctx->stats.n_regions = ctx->stats.level_counts[0];
  WS_CUDA(cudaGetLastError());
  return WS_OK;
}

}  // namespace ws
