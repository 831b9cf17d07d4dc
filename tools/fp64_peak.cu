// FP64 peak microbenchmark for B200 (sm_100a): DFMA pipe vs DMMA (mma.sync m8n8k4 f64).
// Prints one JSON line per test. Used to pick the roofline denominator.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){fprintf(stderr,"CUDA %s @%d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

template<int CH>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x * 1e-9 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int c = 0; c < CH; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

template<int NACC>
__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-12, b = 0.999999;
  double c[NACC][2];
#pragma unroll
  for (int k = 0; k < NACC; ++k) { c[k][0] = 0; c[k][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int k = 0; k < NACC; ++k)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < NACC; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int sms = p.multiProcessorCount;
  printf("{\"device\":\"%s\",\"sms\":%d,\"cc\":\"%d.%d\",\"l2_mb\":%.1f,\"smem_optin_kb\":%zu}\n", p.name, sms, p.major, p.minor,
         p.l2CacheSize / 1048576.0, p.sharedMemPerBlockOptin / 1024);
  double* d; CK(cudaMalloc(&d, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  // DFMA: 8 chains x 16 unroll per iter per thread
  for (int threads : {256, 512}) for (int bps : {2, 4, 8}) {
    int blocks = sms * bps; int iters = 4000;
    dfma_loop<8><<<blocks, threads>>>(d, 10, 1.0000001, 1e-7); CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0); dfma_loop<8><<<blocks, threads>>>(d, iters, 1.0000001, 1e-7); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double fl = 2.0 * 8 * 16 * (double)iters * threads * blocks;
    printf("{\"test\":\"dfma\",\"threads\":%d,\"blocks\":%d,\"ms\":%.3f,\"tflops\":%.3f}\n", threads, blocks, best, fl / best / 1e9);
  }
  // sustained DFMA ~3 s
  {
    int threads = 256, blocks = sms * 4, iters = 4000; cudaEventRecord(e0);
    int reps = 0; float ms = 0;
    while (ms < 3000) { dfma_loop<8><<<blocks, threads>>>(d, iters, 1.0000001, 1e-7); ++reps;
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); }
    double fl = 2.0 * 8 * 16 * (double)iters * threads * blocks * reps;
    printf("{\"test\":\"dfma_sustained\",\"reps\":%d,\"ms\":%.1f,\"tflops\":%.3f}\n", reps, ms, fl / ms / 1e9);
  }
  for (int threads : {128, 256, 512}) for (int bps : {2, 4, 8}) {
    int blocks = sms * bps, iters = 2000;
    dmma_loop<4><<<blocks, threads>>>(d, 10); CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0); dmma_loop<4><<<blocks, threads>>>(d, iters); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double fl = 2.0 * 256 * 8 * 4 * (double)iters * (threads / 32) * blocks;
    printf("{\"test\":\"dmma_m8n8k4\",\"threads\":%d,\"blocks\":%d,\"ms\":%.3f,\"tflops\":%.3f}\n", threads, blocks, best, fl / best / 1e9);
  }
  {
    int threads = 256, blocks = sms * 4, iters = 2000; cudaEventRecord(e0);
    int reps = 0; float ms = 0;
    while (ms < 3000) { dmma_loop<4><<<blocks, threads>>>(d, iters); ++reps;
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); }
    double fl = 2.0 * 256 * 8 * 4 * (double)iters * (threads / 32) * blocks * reps;
    printf("{\"test\":\"dmma_sustained\",\"reps\":%d,\"ms\":%.1f,\"tflops\":%.3f}\n", reps, ms, fl / ms / 1e9);
  }
  return 0;
}
