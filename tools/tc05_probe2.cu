// Probe 2: the k_sigma_tc TMA pattern in isolation: 5-D fp32 maps with plane/kz/atom dims, SWIZZLE_128B,
// 8 loads per stage into a 2-stage ring with full/empty mbarriers, a consumer warp releasing stages.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <vector>
#include <cstdlib>
#include "../paper_1912_10024_b200/csrc/tma.cuh"
using namespace qt;
constexpr int AP = 128 * 32, BP = 80 * 32, STG = 4 * (AP + BP);
__global__ void k(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB, int nst, int mode, float* out) {
  extern __shared__ uint8_t sm[];
  float* st = (float*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(st + 2 * STG);
  uint64_t* empty = full + 2;
  if (threadIdx.x == 0) { for (int s = 0; s < 2; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); } fence_barrier_init(); }
  __syncthreads();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0 && lane == 0) {
    if (mode & 4) { prefetch_tmap(&tA); prefetch_tmap(&tB); }
    for (int g = 0; g < nst; ++g) {
      const int slot = g % 2;
      if (g >= 2) mbar_wait(&empty[slot], ((g / 2) - 1) & 1);
      float* sa = st + ((mode & 256) ? 0 : slot * STG); float* sb = sa + 4 * AP;
      const int np = (mode & 2) ? 1 : 4;
      const int z = (mode & 1) ? 0 : 1;
      const int useB = (mode & 8) ? 0 : 1;
      mbar_arrive_expect_tx(&full[slot], np * (AP + useB * BP) * 4);
      for (int p = 0; p < np; ++p) {
        if (mode & 2048) tma_load_4d(sa + p * AP, &tA, (g % 3) * 5, 0, z * p, z * (g % 3), &full[slot]);
        else tma_load_5d(sa + p * AP, &tA, (g % 3) * 5, 0, z * p, z * (g % 3), z * (g % 16), &full[slot]);
        if (useB) tma_load_5d(sb + p * BP, &tB, 0, 0, z * p, z * (g % 3), z * (g % 7), &full[slot]);
      }
    }
  } else if (warp == 1 && lane == 0) {
    float s = 0;
    for (int g = 0; g < nst; ++g) {
      const int slot = g % 2;
      mbar_wait(&full[slot], (g / 2) & 1);
      if (!(mode & 128)) s += st[slot * STG + 5] + st[slot * STG + 4 * AP + 7];
      mbar_arrive(&empty[slot]);
    }
    out[0] = s;
  }
  __syncwarp();
  __syncthreads();
}
int main(int argc, char** argv) {
  const int MODE = atoi(argv[1]);
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
  const size_t nA = (size_t)16 * 3 * 4 * 128 * 32, nB = (size_t)7 * 3 * 4 * 80 * 32;
  float *dA, *dB, *dO; cudaMalloc(&dA, nA * 4); cudaMalloc(&dB, nB * 4); cudaMalloc(&dO, 4);
  cudaMemset(dA, 0, nA * 4); cudaMemset(dB, 0, nB * 4);
  CUtensorMap tA, tB; const cuuint32_t es[5] = {1, 1, 1, 1, 1};
  const bool simple = MODE & 16;
  cuuint64_t dA0 = simple ? 64 : 32;
  { cuuint64_t dims[5] = {dA0, 128, simple ? 1ull : 4ull, simple ? 1ull : 3ull, simple ? 1ull : 16ull}; cuuint64_t str[4] = {dA0 * 4, dA0 * 4 * 128, dA0 * 4 * 128 * 4, dA0 * 4 * 128 * 12}; cuuint32_t box[5] = {32, 128, 1, 1, 1};
    printf("encA %d\n", enc(&tA, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, dA, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, (MODE & 1024) ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)); }
  { cuuint64_t dims[5] = {32, 80, 4, 3, 7}; cuuint64_t str[4] = {128, 80 * 128, 4 * 80 * 128, 3 * 4 * 80 * 128}; cuuint32_t box[5] = {32, 80, 1, 1, 1};
    printf("encB %d\n", enc(&tB, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, dB, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)); }
  const int smem = 2 * STG * 4 + 1024 + 256 + ((MODE & 512) ? 4096 : 0);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int mode : {MODE}) for (int threads : {64}) {
    k<<<(MODE & 64) ? 1 : 2, threads, smem>>>(tA, tB, argc > 2 ? atoi(argv[2]) : 10, mode, dO);
    printf("mode %d threads %d: %s\n", mode, threads, cudaGetErrorString(cudaDeviceSynchronize()));
  }
  return 0;
}
