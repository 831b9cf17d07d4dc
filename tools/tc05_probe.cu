// Probe: one CTA computes C[128][N] = A[128][K] · B[N][K]^T with tcgen05.mma kind::tf32 (K-major, SW128 TMA
// tiles), accumulator in TMEM, 4 warps read it back. Checks against a host reference on tf32-truncated
// inputs. Also checks the negate-A bit and descriptor K-advance (+32 B per 8 tf32).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "../paper_1912_10024_b200/csrc/tc05.cuh"
#ifdef SW64
constexpr int KC = 16;
__device__ __forceinline__ uint64_t desc_sw(const void* p) {
  const uint32_t a = qt::smem_u32(p);
  uint64_t d = 0;
  d |= (uint64_t)((a >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;
  return d;
}
#define SWZ CU_TENSOR_MAP_SWIZZLE_64B
#else
constexpr int KC = 32;
#define desc_sw umma_desc_k128
#define SWZ CU_TENSOR_MAP_SWIZZLE_128B
#endif
using namespace qt;
#ifndef PN
#define PN 64
#endif
#ifndef PCOLS
#define PCOLS 64
#endif
constexpr int M = 128, N = PN, K = 64;   // K = 2 swizzle chunks of 32

#ifdef P5D
#define TLOAD(d, m, c) tma_load_5d(d, m, c, 0, 0, 0, 0, &bar_load)
#else
#define TLOAD(d, m, c) tma_load_4d(d, m, c, 0, 0, 0, &bar_load)
#endif
__global__ void probe(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB, float* C, int neg) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  float* sA = (float*)base;
  float* sB = (float*)(base + (K / KC) * M * KC * 4);
  __shared__ uint64_t bar_load, bar_mma;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) tmem_alloc<PCOLS>(&tbase);
  if (threadIdx.x == 32) { mbar_init(&bar_load, 1); mbar_init(&bar_mma, 1); fence_barrier_init(); }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tm = tbase;
  if (threadIdx.x == 32) {
    mbar_arrive_expect_tx(&bar_load, (M + N) * K * 4);
    for (int c = 0; c < K / KC; ++c) {
      TLOAD(sA + c * M * KC, &tA, c * KC);
      TLOAD(sB + c * N * KC, &tB, c * KC);
    }
    mbar_wait(&bar_load, 0);
    tc_fence_after();
    const uint32_t idesc = umma_idesc_tf32(M, N, neg != 0, false);
    for (int k = 0; k < K / 8; ++k) {
      const int c = k / (KC / 8), kk = k % (KC / 8);
      const uint64_t ad = desc_sw((uint8_t*)(sA + c * M * KC) + kk * 32);
      const uint64_t bd = desc_sw((uint8_t*)(sB + c * N * KC) + kk * 32);
      umma_tf32(tm, ad, bd, idesc, k > 0);
    }
    umma_commit(&bar_mma);
  }
  __syncwarp();
  if (warp < 4) {
    mbar_wait(&bar_mma, 0);
    tc_fence_after();
    const int row = warp * 32 + lane;
    for (int c0 = 0; c0 < N; c0 += 16) {
      float v[16];
      tmem_ld16(tm + ((warp * 32) << 16) + c0, v);
      for (int i = 0; i < 16; ++i) C[row * N + c0 + i] = v[i];
    }
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (warp == 0) tmem_dealloc<PCOLS>(tm);
}

static float tf32t(float x) { unsigned u; memcpy(&u, &x, 4); u &= ~0x1FFFu; float y; memcpy(&y, &u, 4); return y; }

int main() {
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
  std::vector<float> A(M * K), B(N * K), C(M * N);
  srand(1);
  for (auto& x : A) x = (rand() / (float)RAND_MAX - 0.5f);
  for (auto& x : B) x = (rand() / (float)RAND_MAX - 0.5f);
  float *dA, *dB, *dC; cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dC, C.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice); cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  CUtensorMap tA, tB;
  const cuuint32_t es[5] = {1, 1, 1, 1, 1};
#ifdef P5D
  const int RANK = 5;
#else
  const int RANK = 4;
#endif
  { cuuint64_t dims[5] = {K, M, 1, 1, 1}; cuuint64_t str[4] = {K * 4, M * K * 4, M * K * 4, M * K * 4}; cuuint32_t box[5] = {KC, M, 1, 1, 1};
    CUresult r = enc(&tA, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, RANK, dA, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, SWZ, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE); printf("encA %d\n", r); }
  { cuuint64_t dims[5] = {K, N, 1, 1, 1}; cuuint64_t str[4] = {K * 4, N * K * 4, N * K * 4, N * K * 4}; cuuint32_t box[5] = {KC, N, 1, 1, 1};
    CUresult r = enc(&tB, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, RANK, dB, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, SWZ, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE); printf("encB %d\n", r); }
  const int smem = 1024 + (M + N) * K * 4;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int neg = 0; neg < 2; ++neg) {
    probe<<<1, 160, smem>>>(tA, tB, dC, neg);
    cudaError_t e = cudaDeviceSynchronize(); printf("kernel: %s\n", cudaGetErrorString(e)); if (e) return 1;
    cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0;
    for (int i = 0; i < M; ++i) for (int j = 0; j < N; ++j) {
      double r = 0; for (int k = 0; k < K; ++k) r += (double)tf32t(A[i * K + k]) * tf32t(B[j * K + k]);
      if (neg) r = -r;
      maxerr = fmax(maxerr, fabs(r - C[i * N + j])); maxref = fmax(maxref, fabs(r));
    }
    printf("neg=%d max|err| %.3e  max|ref| %.3e  C[0][0]=%f C[127][63]=%f\n", neg, maxerr, maxref, C[0], C[M * N - 1]);
  }
  return 0;
}
