// Legacy warp-level MMA throughput on sm_100a: mma.sync m16n8k8 tf32 (f32 accumulate) and m16n8k16 bf16.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){fprintf(stderr,"CUDA %s @%d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

template <int NACC>
__global__ void tf32_loop(float* out, int iters) {
  unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  float c[NACC][4] = {};
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int k = 0; k < NACC; ++k)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[k][0]), "+f"(c[k][1]), "+f"(c[k][2]), "+f"(c[k][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  float s = 0;
  for (int k = 0; k < NACC; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
  if (s == 1234.5f) out[0] = s;
}
template <int NACC>
__global__ void bf16_loop(float* out, int iters) {
  unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  float c[NACC][4] = {};
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int k = 0; k < NACC; ++k)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[k][0]), "+f"(c[k][1]), "+f"(c[k][2]), "+f"(c[k][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  float s = 0;
  for (int k = 0; k < NACC; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
  if (s == 1234.5f) out[0] = s;
}
int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  float* d; CK(cudaMalloc(&d, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int threads : {256, 512}) for (int bps : {1, 2, 4}) {
    const int blocks = sms * bps, iters = 4000;
    float best = 1e30f;
    tf32_loop<8><<<blocks, threads>>>(d, 10); CK(cudaDeviceSynchronize());
    for (int r = 0; r < 3; ++r) { cudaEventRecord(e0); tf32_loop<8><<<blocks, threads>>>(d, iters); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }
    const double fl = 2.0 * 16 * 8 * 8 * 8.0 * iters * (threads / 32) * blocks;
    printf("{\"test\":\"mma_sync_tf32_m16n8k8\",\"threads\":%d,\"blocks\":%d,\"tflops\":%.1f}\n", threads, blocks, fl / best / 1e9);
    best = 1e30f;
    bf16_loop<8><<<blocks, threads>>>(d, 10); CK(cudaDeviceSynchronize());
    for (int r = 0; r < 3; ++r) { cudaEventRecord(e0); bf16_loop<8><<<blocks, threads>>>(d, iters); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }
    const double fl2 = 2.0 * 16 * 8 * 16 * 8.0 * iters * (threads / 32) * blocks;
    printf("{\"test\":\"mma_sync_bf16_m16n8k16\",\"threads\":%d,\"blocks\":%d,\"tflops\":%.1f}\n", threads, blocks, fl2 / best / 1e9);
  }
  return 0;
}
