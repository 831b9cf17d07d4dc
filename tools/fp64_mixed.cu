// Do DMMA (tensor pipe) and DFMA (fp64 pipe) run concurrently on sm_100a? Warps of even index run an
// m8n8k4 f64 MMA loop, odd warps a DFMA loop; compare with each half alone (other half idle).
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){fprintf(stderr,"CUDA %s @%d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

__global__ void mixed(double* out, int it_mma, int it_fma, int mode) {
  const int w = threadIdx.x >> 5;
  double s = 0;
  if ((w & 1) == 0 && (mode & 1)) {
    double a = 1.0 + threadIdx.x * 1e-12, b = 0.999999;
    double c[4][2] = {};
    for (int it = 0; it < it_mma; ++it)
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int k = 0; k < 4; ++k)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                       : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
    for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
  }
  if ((w & 1) == 1 && (mode & 2)) {
    double acc[8];
    for (int c = 0; c < 8; ++c) acc[c] = threadIdx.x * 1e-9 + c;
    for (int it = 0; it < it_fma; ++it)
#pragma unroll
      for (int u = 0; u < 16; ++u)
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[c] = fma(acc[c], 1.0000001, 1e-7);
    for (int c = 0; c < 8; ++c) s += acc[c];
  }
  if (s == 12345.678) out[0] = s;
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double* d; CK(cudaMalloc(&d, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int threads = 512, blocks = sms * 2;
  for (int fma_it : {500, 1000, 2000, 4000}) {
    const int mma_it = 1000;
    float t[4];
    for (int mode = 1; mode <= 3; ++mode) {
      mixed<<<blocks, threads>>>(d, 10, 10, mode); CK(cudaDeviceSynchronize());
      float best = 1e30f;
      for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0); mixed<<<blocks, threads>>>(d, mma_it, fma_it, mode); cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      t[mode] = best;
    }
    const double half = (threads / 64) * (double)blocks;   // warps per role
    const double fl_mma = 2.0 * 256 * 8 * 4 * (double)mma_it * half;
    const double fl_fma = 2.0 * 8 * 16 * (double)fma_it * half * 32;
    printf("{\"fma_it\":%d,\"ms_dmma_only\":%.3f,\"ms_dfma_only\":%.3f,\"ms_both\":%.3f,\"tf_dmma_only\":%.2f,"
           "\"tf_dfma_only\":%.2f,\"tf_both\":%.2f}\n", fma_it, t[1], t[2], t[3], fl_mma / t[1] / 1e9,
           fl_fma / t[2] / 1e9, (fl_mma + fl_fma) / t[3] / 1e9);
  }
  return 0;
}
