// common.cuh — small device helpers shared by the libqtsse kernels (product side only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace qt {

// FP64 tensor-core MMA, m8n8k4 (SASS: DMMA.8x8x4). Fragment layout (PTX ISA, mma.m8n8k4 .f64):
//   A (8x4, row):  a = A[lane>>2][lane&3]
//   B (4x8, col):  b = B[lane&3][lane>>2]
//   C/D (8x8):     c0,c1 = C[lane>>2][2*(lane&3) + {0,1}]
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// complex 8x8x4 step on split accumulators: C += A*B with A = (ar, ai), B = (br, bi)
struct CAcc {
  double r0, r1, i0, i1;
};
__device__ __forceinline__ void cmma(CAcc& c, double ar, double ai, double nai, double br, double bi) {
  dmma(c.r0, c.r1, ar, br);
  dmma(c.r0, c.r1, nai, bi);
  dmma(c.i0, c.i1, ar, bi);
  dmma(c.i0, c.i1, ai, br);
}

// Gauss 3M complex product on three real accumulators: T1 += Ar·Br, T2 += Ai·Bi,
// T3 += (Ar+Ai)(Br+Bi); value = (T1 - T2) + i (T3 - T1 - T2). as = ar + ai (computed once per A fragment).
struct C3Acc {
  double t1[2] = {0.0, 0.0}, t2[2] = {0.0, 0.0}, t3[2] = {0.0, 0.0};
  __device__ __forceinline__ double2 value(int k) const {
    return make_double2(t1[k] - t2[k], (t3[k] - t1[k]) - t2[k]);
  }
};
__device__ __forceinline__ void cmma3(C3Acc& c, double ar, double ai, double as, double br, double bi) {
  dmma(c.t1[0], c.t1[1], ar, br);
  dmma(c.t2[0], c.t2[1], ai, bi);
  dmma(c.t3[0], c.t3[1], as, br + bi);
}

// same with the B-side sum bs = br + bi precomputed
__device__ __forceinline__ void cmma3s(C3Acc& c, double ar, double ai, double as, double br, double bi, double bs) {
  dmma(c.t1[0], c.t1[1], ar, br);
  dmma(c.t2[0], c.t2[1], ai, bi);
  dmma(c.t3[0], c.t3[1], as, bs);
}

// 16-byte async global->shared copy; src_valid == false zero-fills the destination.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool src_valid) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int sz = src_valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ void cfma(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}

__device__ __forceinline__ void cfma(float2& acc, float2 a, float2 b) {
  acc.x = fmaf(a.x, b.x, acc.x);
  acc.x = fmaf(-a.y, b.y, acc.x);
  acc.y = fmaf(a.x, b.y, acc.y);
  acc.y = fmaf(a.y, b.x, acc.y);
}
// complex type of a real type (double2 / float2), conversions from / to double2
template <class R> struct Cx;
template <> struct Cx<double> {
  using T = double2;
  __device__ static T zero() { return make_double2(0.0, 0.0); }
  __device__ static T from(double2 v) { return v; }
  __device__ static double2 wide(T v) { return v; }
};
template <> struct Cx<float> {
  using T = float2;
  __device__ static T zero() { return make_float2(0.f, 0.f); }
  __device__ static T from(double2 v) { return make_float2((float)v.x, (float)v.y); }
  __device__ static double2 wide(T v) { return make_double2((double)v.x, (double)v.y); }
};

__host__ __device__ inline int64_t imod(int64_t x, int64_t n) {
  int64_t r = x % n;
  return r < 0 ? r + n : r;
}

// ---- work lists (built on the host in qt_sse_plan) ----
// Σ is source-organized: one item = a source atom b and up to 8 (FP32 mode: 14) of the pairs (a,s) with nbr[a][s] == b.
struct SigPair {
  int32_t a;      // destination atom (local output index space: a - a_lo)
  int32_t s;      // slot of b in nbr[a]
  int32_t r;      // slot of a in nbr[b]
  int32_t a_in;   // destination atom in the input window
};
struct SigItem {
  int32_t b_in;   // source atom in the input window
  int32_t npair;  // 1..8 (FP32 mode: 1..14)
  int32_t pair0;  // index into the SigPair list
  int32_t b;      // source atom (global)
};
// Π is destination-organized: one item = a destination atom a and up to 8 (FP32 mode: 14) of its valid slots.
struct PiPair {
  int32_t s, b_in, r, a_in;
};
struct PiItem {
  int32_t a_out;  // output atom (a - a_lo)
  int32_t a_in;   // atom in the input window
  int32_t npair;
  int32_t pair0;
};

constexpr int kMaxPairs = 8;   // pairs per item -> 9*8 = 72 rows = 9 m-fragments
constexpr int kMaxEpt = 4;     // energies per Σ tile for small items (1 pair: 2 m-fragments per energy)
constexpr int kRows = 72;
constexpr int kWarps = 9;
constexpr int kThreads = kWarps * 32;

}  // namespace qt
