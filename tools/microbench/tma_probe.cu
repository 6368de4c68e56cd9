// Probe which TMA 3D box shapes load correctly on this part (one config per process).
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_2511_11890_b200/csrc/tma.cuh"
using namespace hb;
__global__ void k(const __grid_constant__ CUtensorMap m, int bytes, int x, int y, int z, float* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    mbar_expect_tx(&bar, bytes);
    tma_load_3d(sm, &m, x, y, z, &bar);
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  if (threadIdx.x == 0) { float s = 0; for (int i = 0; i < bytes; i++) s += sm[i]; out[0] = s; }
}
int main(int argc, char** argv) {
  int es = atoi(argv[1]), bx = atoi(argv[2]), by = atoi(argv[3]);
  int nx = atoi(argv[4]), ny = atoi(argv[5]), nz = 4, x = atoi(argv[6]), y = atoi(argv[7]);
  int stat_smem = argc > 8 ? atoi(argv[8]) : 0;
  void* d; cudaMalloc(&d, (size_t)nx * ny * nz * es); cudaMemset(d, 1, (size_t)nx * ny * nz * es);
  float* o; cudaMalloc(&o, 4);
  CUtensorMap m;
  CUtensorMapDataType dt = es == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : (es == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16 : CU_TENSOR_MAP_DATA_TYPE_UINT8);
  bool ok = make_tmap_3d(&m, d, dt, es, nx, ny, nz, bx, by);
  int bytes = bx * by * es;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  k<<<1, 32, bytes + 256>>>(m, bytes, x, y, 1, o);
  cudaError_t e = cudaDeviceSynchronize();
  float h = 0; cudaMemcpy(&h, o, 4, cudaMemcpyDeviceToHost);
  printf("es=%d box=%dx%d n=%dx%d at (%d,%d) enc=%d -> %s sum=%g\n", es, bx, by, nx, ny, x, y, ok, cudaGetErrorString(e), h);
  return 0;
}
