// Probe: TMA 3-D u8 box loads on sm_100a (param-space vs global descriptor; box vs dims).
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../paper_2410_08946_b200/csrc/ws_tma.cuh"
using namespace ws;

template <int SX, int SY, int SZ>
__global__ void k_probe(const __grid_constant__ CUtensorMap m, const CUtensorMap* gm, int use_global, int x, int y, int z, int* out) {
  __shared__ alignas(128) uint8_t s[SX * SY * SZ];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) mbar_init(&bar, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(&bar, SX * SY * SZ);
    tma_load_3d(s, use_global ? gm : &m, x, y, z, &bar);
  }
  mbar_wait(&bar, 0);
  if (threadIdx.x == 0) { int acc = 0; for (int i = 0; i < SX * SY * SZ; ++i) acc += s[i]; out[0] = acc; }
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  int only = argc > 1 ? atoi(argv[1]) : -1;
  void* p; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  Enc enc = (Enc)p;
  for (int trial = 0; trial < 6; ++trial) {
    if (only >= 0 && trial != only) continue;
    int n2 = trial < 2 ? 1024 : 64, n1 = trial < 2 ? 1024 : 64, n0 = 16;
    uint8_t* d; cudaMalloc(&d, (size_t)n2 * n1 * n0); cudaMemset(d, 1, (size_t)n2 * n1 * n0);
    CUtensorMap m;
    cuuint64_t dims[3] = {(cuuint64_t)n2, (cuuint64_t)n1, (cuuint64_t)n0};
    cuuint64_t str[2] = {(cuuint64_t)n2, (cuuint64_t)n2 * n1};
    cuuint32_t box[3] = {48, 12, 12}, es[3] = {1, 1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUtensorMap* gm; cudaMalloc(&gm, sizeof(CUtensorMap)); cudaMemcpy(gm, &m, sizeof(m), cudaMemcpyHostToDevice);
    int* out; cudaMalloc(&out, 4); cudaMemset(out, 0, 4);
    int use_global = trial & 1;
    int X = atoi(argv[2]), Y = atoi(argv[3]), Z = atoi(argv[4]);
    k_probe<48, 12, 12><<<1, 128>>>(m, gm, use_global, X, Y, Z, out);
    cudaError_t e = cudaDeviceSynchronize();
    int h = -1; cudaMemcpy(&h, out, 4, cudaMemcpyDeviceToHost);
    printf("xyz=%s,%s,%s trial %d n2=%d global=%d encode=%d err=%s sum=%d (expect in-bounds count)\n", argv[2],argv[3],argv[4],trial, n2, use_global, (int)r,
           cudaGetErrorString(e), h);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
