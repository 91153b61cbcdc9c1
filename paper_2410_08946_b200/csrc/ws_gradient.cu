// ws_gradient.cu — the stencil pre-pass: Gaussian blur (C8) + gradient magnitude (C9) +
// quantisation to the agreed u8 image (C10).  P:91-94, Fig. 2 caption P:159.
//
// v1 design: one separable pass per blurred axis (fp32, clamp-to-edge) through fp32 scratch,
// then one fused gradient + quantise pass.  HBM-bound; see DESIGN.md §Kernels.
#include "ws_internal.h"

namespace ws {

constexpr int RMAX = 60;  // sigma <= 20  ->  r = floor(3 sigma + 0.5) <= 60
__constant__ float c_w[2 * RMAX + 1];

template <class Tin>
__device__ __forceinline__ float load_norm(const Tin* in, size_t i);
template <>
__device__ __forceinline__ float load_norm<uint8_t>(const uint8_t* in, size_t i) {
  return (float)__ldg(in + i) / 255.0f;
}
template <>
__device__ __forceinline__ float load_norm<float>(const float* in, size_t i) {
  return __ldg(in + i);
}

// out = (1-D Gaussian along `axis`) * in ; axis 0 = n0, 1 = n1, 2 = n2.
template <class Tin>
__global__ void k_blur_axis(const Tin* __restrict__ in, float* __restrict__ out, Geo g, int axis, int r) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= g.n2 || y >= g.n1) return;
  const int len = axis == 0 ? g.n0 : axis == 1 ? g.n1 : g.n2;
  const int stride = axis == 0 ? g.plane : axis == 1 ? g.n2 : 1;
  for (int z = blockIdx.z; z < g.n0; z += gridDim.z) {
    const int c = axis == 0 ? z : axis == 1 ? y : x;
    const size_t p = (size_t)z * g.plane + (size_t)y * g.n2 + x;
    float acc = 0.f;
    for (int i = -r; i <= r; ++i) {
      int k = c + i;
      k = k < 0 ? 0 : (k >= len ? len - 1 : k);
      acc = fmaf(c_w[i + r], load_norm<Tin>(in, p + (ptrdiff_t)(k - c) * stride), acc);
    }
    out[p] = acc;
  }
}

template <class Tin>
__device__ __forceinline__ float deriv(const Tin* b, size_t p, int c, int len, int stride) {
  if (len < 2) return 0.f;
  if (c == 0) return load_norm<Tin>(b, p + stride) - load_norm<Tin>(b, p);
  if (c == len - 1) return load_norm<Tin>(b, p) - load_norm<Tin>(b, p - stride);
  return 0.5f * (load_norm<Tin>(b, p + stride) - load_norm<Tin>(b, p - stride));
}

template <class Tin>
__global__ void k_gradmag(const Tin* __restrict__ b, Geo g, int is3d, uint8_t* __restrict__ q,
                          float* __restrict__ blur_out, float* __restrict__ grad_out) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= g.n2 || y >= g.n1) return;
  for (int z = blockIdx.z; z < g.n0; z += gridDim.z) {
    const size_t p = (size_t)z * g.plane + (size_t)y * g.n2 + x;
    float s = 0.f;
    if (is3d) {
      float d = deriv<Tin>(b, p, z, g.n0, g.plane);
      s = fmaf(d, d, s);
    }
    float d1 = deriv<Tin>(b, p, y, g.n1, g.n2);
    s = fmaf(d1, d1, s);
    float d2 = deriv<Tin>(b, p, x, g.n2, 1);
    s = fmaf(d2, d2, s);
    const float gm = sqrtf(s);
    const float qq = floorf(fmaf(255.0f, gm, 0.5f));
    q[p] = (uint8_t)(qq > 255.f ? 255.f : qq);
    if (blur_out) blur_out[p] = load_norm<Tin>(b, p);
    if (grad_out) grad_out[p] = gm;
  }
}

ws_status run_gradient(ws_ctx* ctx, const uint8_t* img, const Geo& g, int is3d, float sigma,
                       uint8_t* grad_q, float* blur_f32, float* grad_f32, cudaStream_t st) {
  L3 l = launch3(g);
  if (sigma == 0.f) {
    k_gradmag<uint8_t><<<l.grid, l.block, 0, st>>>(img, g, is3d, grad_q, blur_f32, grad_f32);
    launched(ctx, PH_GRAD_MAG);
    tmark(ctx, st, PH_GRAD_MAG);
    WS_CUDA(cudaGetLastError());
    return WS_OK;
  }
  const int r = (int)floor(3.0 * (double)sigma + 0.5);
  float w[2 * RMAX + 1];
  double ws = 0, wd[2 * RMAX + 1];
  for (int i = -r; i <= r; ++i) { wd[i + r] = exp(-(double)i * i / (2.0 * sigma * (double)sigma)); ws += wd[i + r]; }
  for (int i = 0; i <= 2 * r; ++i) w[i] = (float)(wd[i] / ws);
  WS_CUDA(cudaMemcpyToSymbolAsync(c_w, w, sizeof(float) * (2 * r + 1), 0, cudaMemcpyHostToDevice, st));
  const size_t nb = (size_t)g.N * sizeof(float);
  WS_TRY(ctx->tmpA.ensure(nb, "gradient scratch A"));
  WS_TRY(ctx->tmpB.ensure(nb, "gradient scratch B"));
  float* A = ctx->tmpA.as<float>();
  float* B = ctx->tmpB.as<float>();
  const float* fin;
  if (is3d) {
    k_blur_axis<uint8_t><<<l.grid, l.block, 0, st>>>(img, A, g, 0, r);
    k_blur_axis<float><<<l.grid, l.block, 0, st>>>(A, B, g, 1, r);
    k_blur_axis<float><<<l.grid, l.block, 0, st>>>(B, A, g, 2, r);
    fin = A;
    launched(ctx, PH_GRAD_BLUR, 3);
  } else {
    k_blur_axis<uint8_t><<<l.grid, l.block, 0, st>>>(img, A, g, 1, r);
    k_blur_axis<float><<<l.grid, l.block, 0, st>>>(A, B, g, 2, r);
    fin = B;
    launched(ctx, PH_GRAD_BLUR, 2);
  }
  tmark(ctx, st, PH_GRAD_BLUR);
  k_gradmag<float><<<l.grid, l.block, 0, st>>>(fin, g, is3d, grad_q, blur_f32, grad_f32);
  launched(ctx, PH_GRAD_MAG);
  tmark(ctx, st, PH_GRAD_MAG);
  WS_CUDA(cudaGetLastError());
  return WS_OK;
}

}  // namespace ws
