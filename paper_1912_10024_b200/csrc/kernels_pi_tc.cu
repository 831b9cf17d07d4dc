// kernels_pi_tc.cu — Π≷ correlation (Eq. 4) in the FP32 mixed-precision mode on the
// tcgen05 tensor cores (kind::tf32; see kernels_sigma_tc.cu for the operand split and the 12-UMMA complex step).
//
// Same reformulation as k_pi_contract (kernels_pi.cu): Π^{ij}_{a,s+1}(qz,m) = scale · Σ_{kz,E,xy}
// W_t^{ij}(kz,E)[xy] · G_a(kz+qz−h, E+s_m)[xy], as the UMMA
//   D[row][m] = Σ_k A[row][k] · B[m][k],  row = (t, ij) of ≤ 14 pairs of destination atom a (M = 128 TMEM
//   lanes), m = frequency (N = 80), k = (kz, E, xy) flattened with the xy row padded to NNp = 4⌈Norb²/4⌉.
// A = the split planes of W (written K-major by k_pi_w_tc, an FP32 sandwich on FP32-rounded inputs). B = G_a: row m starts
// s_m energies later in the same flattened (E, xy) sequence, i.e. B is a TMA view with row stride NNp over a
// copy of G_a padded with zero energies past NE (R7), so every K-chunk of 32 is one box per plane.
// Precision: the tensor core's FP32 accumulation loses ~1 ulp per addition (its error grows linearly with the
// number of products: 8e-5 relative after ~3,600 complex products), so each TMEM accumulator only sums one
// segment of kSegChunks K-chunks (128 products); the 20 epilogue warps then add the segment into FP64
// registers (thread = one row x 16 frequencies) while the MMAs fill the other TMEM buffer, and store
// scale·Π once per tile.
#include "kernels_decl.cuh"
#include "tc05.cuh"
#include "tma.cuh"

#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

namespace qt {

#define UMMA_DESC(p) (kPKC == 16 ? umma_desc_k64(p) : umma_desc_k128(p))
constexpr int kPM = 128;                 // UMMA M: rows (t, ij), 9·14 = 126 used
constexpr int kPN = 80;                  // UMMA N: shift columns ((Nω−1)·shift_step + 1 <= 80 in this mode)
#ifndef QT_PI_KC
#define QT_PI_KC 32
#endif
constexpr int kPKC = QT_PI_KC;           // K per stage: one 64-byte (16) or 128-byte (32) swizzle row of fp32
constexpr int kPStages = kPKC == 16 ? 4 : 2;
constexpr int kPAPlane = kPM * kPKC;
constexpr int kPBPlane = kPN * kPKC;
constexpr int kPStage = 4 * (kPAPlane + kPBPlane);
constexpr uint32_t kPStageBytes = kPStage * 4;
constexpr int kPBufCols = 256;
constexpr int kSegChunks = 128 / kPKC;   // chunks per FP32 accumulation segment (128 products per accumulator)
constexpr int kPEpiWarps = 20;           // epilogue warps: 4 TMEM lane quarters x 5 groups of 16 frequencies
constexpr int kPCols = 16;               // frequencies per epilogue thread (FP64 accumulators)
constexpr int kPThreads = (2 + kPEpiWarps) * 32;
constexpr size_t kPSmem = (size_t)kPStages * kPStageBytes + 1024 + 256;
static_assert(kPSmem <= 227 * 1024, "shared memory");

__device__ __forceinline__ float tf32_rna_p(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
__device__ __forceinline__ void split3_p(double x, float& hi, float& lo) {   // both terms rounded (unbiased)
  hi = tf32_rna_p((float)x);
  lo = tf32_rna_p((float)(x - (double)hi));
}

// G^X (paper layout [Nkz][NE][Nwin][NN], complex128) -> Gp[a][kz][plane][Epad][NNp] fp32 split planes
// (re_hi, re_lo, im_hi, im_lo); energies >= NE and xy >= NN are zero.
__global__ void __launch_bounds__(256) k_relayout_pi_tc(const double2* __restrict__ G, float* __restrict__ out,
                                                        int64_t Nkz, int64_t NE, int64_t Epad, int64_t Nwin, int NN,
                                                        int NNp) {
  const int64_t a = blockIdx.x / Nkz, kz = blockIdx.x % Nkz;
  float* o = out + (a * Nkz + kz) * 4 * Epad * NNp;
  const int64_t n = Epad * NNp;
  for (int64_t idx = threadIdx.x; idx < n; idx += blockDim.x) {
    const int64_t e = idx / NNp;
    const int xy = (int)(idx - e * NNp);
    double2 v = make_double2(0.0, 0.0);
    if (e < NE && xy < NN) v = __ldg(G + ((kz * NE + e) * Nwin + a) * NN + xy);
    float h, l;
    split3_p(v.x, h, l);
    o[idx] = h;
    o[n + idx] = l;
    split3_p(v.y, h, l);
    o[2 * n + idx] = h;
    o[3 * n + idx] = l;
  }
}

cudaError_t launch_relayout_pi_tc(const double2* G, float* out, int64_t Nkz, int64_t NE, int64_t Epad, int64_t Nwin, int NN,
                                  int NNp, cudaStream_t st) {
  if (Nkz * Nwin == 0) return cudaSuccess;
  k_relayout_pi_tc<<<(unsigned)(Nkz * Nwin), 256, 0, st>>>(G, out, Nkz, NE, Epad, Nwin, NN, NNp);
  return cudaGetLastError();
}

// W_p^{ij}(kz,E)[x][y] = (∇_jH_{as} G^Y_b(kz,E) ∇_iH_{br})[y][x] (FP32 arithmetic on FP32-rounded inputs; the
// same order as k_pi_w) written as split planes
// Wp[il][plane][row = t·9+ij][k = (kz·NE + E)·NNp + x·Norb + y]; xy padding columns are zero. One CTA per
// (item, kz, group of 4 pairs), looping over energy pairs.
#ifndef QT_PIWTC_P
#define QT_PIWTC_P 4
#endif
#ifndef QT_PIWTC_T
#define QT_PIWTC_T 256
#endif
constexpr int kTWPairs = QT_PIWTC_P;
constexpr int kTWThreads = QT_PIWTC_T;
constexpr int kTWE = 2;

template <int NO>
__global__ void __launch_bounds__(kTWThreads, 512 / kTWThreads) k_pi_w_tc(PiWArgs A, float* __restrict__ Wp, int NNp) {
  constexpr int NN = NO * NO;
  extern __shared__ __align__(16) float2 w_sm[];
  float2* Hl = w_sm;                           // [kTWPairs][3][NN]  ∇_jH_{as}
  float2* Hr = Hl + kTWPairs * 3 * NN;         // [kTWPairs][3][NN]  ∇_iH_{br}
  double2* Gb = reinterpret_cast<double2*>(Hr + kTWPairs * 3 * NN);   // [2][kTWPairs][kTWE][NN] (FP64, cp.async)
  float2* T = reinterpret_cast<float2*>(Gb + 2 * kTWPairs * kTWE * NN); // [kTWPairs][kTWE][3][NN]
  constexpr int NG = (kTcPiPairs + kTWPairs - 1) / kTWPairs;
  const int grp = blockIdx.x % NG;
  const int64_t r = blockIdx.x / NG;
  const int kz = (int)(r % A.Nkz);
  const int64_t item = A.i0 + r / A.Nkz;
  const PiItem it = A.items[item];
  const int t0 = grp * kTWPairs;
  const int P = min(kTWPairs, it.npair - t0);
  if (P <= 0) return;
  for (int idx = threadIdx.x; idx < P * 3 * NN; idx += blockDim.x) {
    const int t = idx / (3 * NN), rem = idx - t * 3 * NN;
    const PiPair pr = A.pairs[it.pair0 + t0 + t];
    Hl[idx] = Cx<float>::from(A.dH[((int64_t)pr.a_in * A.Nb + pr.s) * 3 * NN + rem]);
    Hr[idx] = Cx<float>::from(A.dH[((int64_t)pr.b_in * A.Nb + pr.r) * 3 * NN + rem]);
  }
  const int KwB = ((A.NEo * NNp + kPKC - 1) / kPKC) * kPKC;       // per-kz block (whole K-chunks, zero tail)
  const int64_t K = (int64_t)A.Nkz * KwB;                          // row length (energies from E0)
  const int64_t plane = (int64_t)kTcPiRows * K;
  float* Wi = Wp + (item - A.i0) * 4 * plane;
  auto prefetch = [&](int e0, double2* dst) {
    const int ne = min(kTWE, A.NEo - e0);
    for (int idx = threadIdx.x; idx < P * ne * NN; idx += blockDim.x) {
      const int t = idx / (ne * NN), rem = idx - t * ne * NN;
      const int b_in = A.pairs[it.pair0 + t0 + t].b_in;
      const int e = rem / NN, uv = rem - e * NN;
      cp_async16(dst + t * kTWE * NN + rem, A.GY + (((int64_t)kz * A.NE + A.E0 + e0 + e) * A.Nwin + b_in) * NN + uv, true);
    }
    cp_async_commit();
  };
  prefetch(0, Gb);
  for (int e0 = 0, itr = 0; e0 < A.NEo; e0 += kTWE, ++itr) {
    const int ne = min(kTWE, A.NEo - e0);
    const double2* Gc = Gb + (itr & 1) * kTWPairs * kTWE * NN;
    if (e0 + kTWE < A.NEo) {
      prefetch(e0 + kTWE, Gb + ((itr + 1) & 1) * kTWPairs * kTWE * NN);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    for (int u = threadIdx.x; u < P * ne * 3 * NO; u += blockDim.x) {   // T_i = G_b ∇_iH_{br}
      const int q = u % NO, r1 = u / NO, i = r1 % 3, r2 = r1 / 3, e = r2 % ne, t = r2 / ne;
      float2 g[NO], s[NO];
#pragma unroll
      for (int k = 0; k < NO; ++k) {
        g[k] = Cx<float>::from(Gc[(t * kTWE + e) * NN + q * NO + k]);
        s[k] = make_float2(0.f, 0.f);
      }
      const float2* h = Hr + (t * 3 + i) * NN;
#pragma unroll
      for (int k = 0; k < NO; ++k)
#pragma unroll
        for (int x = 0; x < NO; ++x) cfma(s[x], g[k], h[k * NO + x]);
      float2* o = T + ((t * kTWE + e) * 3 + i) * NN + q * NO;
#pragma unroll
      for (int x = 0; x < NO; ++x) o[x] = s[x];
    }
    __syncthreads();
    for (int u = threadIdx.x; u < P * ne * 9 * NO; u += blockDim.x) {   // W^{ij}[x][y] = Σ_q ∇_jH[y][q] T_i[q][x]
      const int y = u % NO, r1 = u / NO, ij = r1 % 9, r2 = r1 / 9, e = r2 % ne, t = r2 / ne;
      const int i = ij / 3, j = ij - 3 * i;
      float2 hrow[NO], s[NO];
#pragma unroll
      for (int k = 0; k < NO; ++k) {
        hrow[k] = Hl[(t * 3 + j) * NN + y * NO + k];
        s[k] = make_float2(0.f, 0.f);
      }
      const float2* tt = T + ((t * kTWE + e) * 3 + i) * NN;
#pragma unroll
      for (int q = 0; q < NO; ++q)
#pragma unroll
        for (int x = 0; x < NO; ++x) cfma(s[x], hrow[q], tt[q * NO + x]);
      float* o = Wi + (int64_t)((t0 + t) * 9 + ij) * K + (int64_t)kz * KwB + (int64_t)(e0 + e) * NNp + y;
#pragma unroll
      for (int x = 0; x < NO; ++x) {
        const float hr = tf32_rna_p(s[x].x), hi_ = tf32_rna_p(s[x].y);
        o[x * NO] = hr;
        o[plane + x * NO] = tf32_rna_p(s[x].x - hr);
        o[2 * plane + x * NO] = hi_;
        o[3 * plane + x * NO] = tf32_rna_p(s[x].y - hi_);
      }
    }
    if constexpr (true) {   // zero the xy padding columns of these energies
      const int npad = NNp - NN;
      for (int u = threadIdx.x; u < P * ne * 9 * npad * 4; u += blockDim.x) {
        const int c = u % npad, r1 = u / npad, pl = r1 % 4, r2 = r1 / 4, ij = r2 % 9, r3 = r2 / 9, e = r3 % ne,
                  t = r3 / ne;
        Wi[pl * plane + (int64_t)((t0 + t) * 9 + ij) * K + (int64_t)kz * KwB + (int64_t)(e0 + e) * NNp + NN + c] = 0.0f;
      }
    }
  }
  // zero the K tail of each of the group's rows for this kz (positions NEo·NNp .. KwB of the kz block)
  for (int u = threadIdx.x; u < P * 9 * 4 * (KwB - A.NEo * NNp); u += blockDim.x) {
    const int w = KwB - A.NEo * NNp;
    const int c = u % w, r1 = u / w, pl = r1 % 4, row = r1 / 4;
    Wi[pl * plane + (int64_t)(t0 * 9 + row) * K + (int64_t)kz * KwB + A.NEo * NNp + c] = 0.0f;
  }
}

template <int NO>
static cudaError_t launch_pi_w_tc_no(const PiWArgs& a, float* Wp, int NNp, int64_t nitems, cudaStream_t st) {
  const int smem = (6 + 3 * kTWE) * kTWPairs * NO * NO * 8 + 2 * kTWE * kTWPairs * NO * NO * 16;
  cudaError_t e = cudaFuncSetAttribute(k_pi_w_tc<NO>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  constexpr int NG = (kTcPiPairs + kTWPairs - 1) / kTWPairs;
  k_pi_w_tc<NO><<<(unsigned)(nitems * a.Nkz * NG), kTWThreads, smem, st>>>(a, Wp, NNp);
  return cudaGetLastError();
}

cudaError_t launch_pi_w_tc(const PiWArgs& a, float* Wp, int NNp, int64_t nitems, cudaStream_t st) {
  if (nitems * a.Nkz == 0) return cudaSuccess;
  switch (a.Norb) {
    case 1: return launch_pi_w_tc_no<1>(a, Wp, NNp, nitems, st);
    case 2: return launch_pi_w_tc_no<2>(a, Wp, NNp, nitems, st);
    case 3: return launch_pi_w_tc_no<3>(a, Wp, NNp, nitems, st);
    case 4: return launch_pi_w_tc_no<4>(a, Wp, NNp, nitems, st);
    case 5: return launch_pi_w_tc_no<5>(a, Wp, NNp, nitems, st);
    case 6: return launch_pi_w_tc_no<6>(a, Wp, NNp, nitems, st);
    case 7: return launch_pi_w_tc_no<7>(a, Wp, NNp, nitems, st);
    case 8: return launch_pi_w_tc_no<8>(a, Wp, NNp, nitems, st);
    case 9: return launch_pi_w_tc_no<9>(a, Wp, NNp, nitems, st);
    case 10: return launch_pi_w_tc_no<10>(a, Wp, NNp, nitems, st);
    default: return cudaErrorInvalidValue;
  }
}

// ---------------------------------------------------------------- the tcgen05 correlation
struct PiTcArgs {
  const PiItem* items;   // chunk's items (index il)
  const PiPair* pairs;
  double2* Pi;
  double2 scale;
  int64_t ntiles, Nout, Nb;
  int NE, Nkz, Nqz, h, Nw, shift0, NNp, nch;   // nch = K-chunks per kz
  int NWv, step;                                // shift columns c < NWv; column c is frequency c / step if c % step == 0
  int accumulate;                               // add into Π (later energy sub-ranges) instead of overwriting
  int E0, NEo;                                  // this rank's energies: window [E0, E0 + NEo)
};

__global__ void __launch_bounds__(kPThreads, 1)
    k_pi_contract_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, PiTcArgs A) {
  extern __shared__ uint8_t smem_raw[];
  float* stages = reinterpret_cast<float*>(smem_raw + ((-smem_u32(smem_raw)) & 1023u));
  uint64_t* full = reinterpret_cast<uint64_t*>(stages + kPStages * kPStage);
  uint64_t* empty = full + kPStages;
  uint64_t* tfull = empty + kPStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tbase = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 1) tmem_alloc<512>(tbase);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kPStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], kPEpiWarps);
    }
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = *tbase;
  const int nck = A.Nkz * A.nch;                              // chunks per tile
  const int nseg = (nck + kSegChunks - 1) / kSegChunks;

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      prefetch_tmap(&tmA);
      prefetch_tmap(&tmB);
      uint32_t g = 0;
      for (int64_t t = blockIdx.x; t < A.ntiles; t += gridDim.x) {
        const int qz = (int)(t % A.Nqz);
        const int il = (int)(t / A.Nqz);
        const PiItem item = A.items[il];
        for (int c = 0; c < nck; ++c, ++g) {
          const int kz = c / A.nch, kc = (c - kz * A.nch) * kPKC;
          const int k2 = (int)imod(kz + qz - A.h, A.Nkz);      // kz + qz (R5)
          const uint32_t slot = g % kPStages;
          if (g >= kPStages) mbar_wait(&empty[slot], ((g / kPStages) - 1) & 1);
          mbar_arrive_expect_tx(&full[slot], kPStageBytes);
          float* sa = stages + slot * kPStage;
          float* sb = sa + 4 * kPAPlane;
          for (int p = 0; p < 4; ++p) {
            tma_load_4d(sa + p * kPAPlane, &tmA, kz * A.nch * kPKC + kc, 0, p, il, &full[slot]);
            tma_load_5d(sb + p * kPBPlane, &tmB, (A.shift0 + A.E0) * A.NNp + kc, 0, p, k2, item.a_in, &full[slot]);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- UMMA issuer
    if (lane == 0) {
      const uint32_t id_pos = umma_idesc_tf32(kPM, kPN, false, false);
      const uint32_t id_neg = umma_idesc_tf32(kPM, kPN, true, false);
      uint32_t g = 0, sc = 0;
      for (int64_t t = blockIdx.x; t < A.ntiles; t += gridDim.x) {
        for (int sg = 0; sg < nseg; ++sg, ++sc) {
          const uint32_t buf = sc & 1;
          if (sc >= 2) mbar_wait(&tempty[buf], ((sc / 2) - 1) & 1);
          tc_fence_after();
          const uint32_t dre = tm + buf * kPBufCols, dim = dre + kPN;
          bool acc = false;
          const int c1 = min(nck, (sg + 1) * kSegChunks);
          for (int c = sg * kSegChunks; c < c1; ++c, ++g) {
            const uint32_t slot = g % kPStages;
            mbar_wait(&full[slot], (g / kPStages) & 1);
            tc_fence_after();
            const float* sa = stages + slot * kPStage;
            const float* sb = sa + 4 * kPAPlane;
#pragma unroll 1
            for (int kk = 0; kk < kPKC / 8; ++kk) {
              const uint64_t arh = UMMA_DESC(sa + 0 * kPAPlane + kk * 8);
              const uint64_t arl = UMMA_DESC(sa + 1 * kPAPlane + kk * 8);
              const uint64_t aih = UMMA_DESC(sa + 2 * kPAPlane + kk * 8);
              const uint64_t ail = UMMA_DESC(sa + 3 * kPAPlane + kk * 8);
              const uint64_t brh = UMMA_DESC(sb + 0 * kPBPlane + kk * 8);
              const uint64_t brl = UMMA_DESC(sb + 1 * kPBPlane + kk * 8);
              const uint64_t bih = UMMA_DESC(sb + 2 * kPBPlane + kk * 8);
              const uint64_t bil = UMMA_DESC(sb + 3 * kPBPlane + kk * 8);
              umma_tf32(dre, arh, brh, id_pos, acc);
              umma_tf32(dre, arh, brl, id_pos, true);
              umma_tf32(dre, arl, brh, id_pos, true);
              umma_tf32(dre, aih, bih, id_neg, true);
              umma_tf32(dre, aih, bil, id_neg, true);
              umma_tf32(dre, ail, bih, id_neg, true);
              umma_tf32(dim, arh, bih, id_pos, acc);
              umma_tf32(dim, arh, bil, id_pos, true);
              umma_tf32(dim, arl, bih, id_pos, true);
              umma_tf32(dim, aih, brh, id_pos, true);
              umma_tf32(dim, aih, brl, id_pos, true);
              umma_tf32(dim, ail, brh, id_pos, true);
              acc = true;
            }
            umma_commit(&empty[slot]);
          }
          umma_commit(&tfull[buf]);
        }
      }
    }
  } else {
    // ---------------- epilogue: FP64 accumulation of the segments, Π[qz][m][a][slot][ij] = scale · Σ_seg D
    const int quarter = warp & 3;                 // TMEM lane quarter (tcgen05.ld rule: warp % 4)
    const int cg = (warp - 2) >> 2;               // frequency group: m in [cg·16, cg·16 + 16)
    const int row = quarter * 32 + lane;
    uint32_t sc = 0;
    for (int64_t t = blockIdx.x; t < A.ntiles; t += gridDim.x) {
      const int qz = (int)(t % A.Nqz);
      const int il = (int)(t / A.Nqz);
      const PiItem item = A.items[il];
      double ar[kPCols], ai[kPCols];
#pragma unroll
      for (int i = 0; i < kPCols; ++i) ar[i] = ai[i] = 0.0;
      for (int sg = 0; sg < nseg; ++sg, ++sc) {
        const uint32_t buf = sc & 1;
        mbar_wait(&tfull[buf], (sc / 2) & 1);
        tc_fence_after();
        const uint32_t taddr = tm + ((uint32_t)(quarter * 32) << 16) + buf * kPBufCols + cg * kPCols;
        float v[kPCols];
        tmem_ld16(taddr, v);
#pragma unroll
        for (int i = 0; i < kPCols; ++i) ar[i] += (double)v[i];
        tmem_ld16(taddr + kPN, v);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[buf]);   // buffer free: the registers hold this segment
#pragma unroll
        for (int i = 0; i < kPCols; ++i) ai[i] += (double)v[i];
      }
      const int tp = row / 9, ij = row - 9 * tp;
      if (tp < item.npair) {
        const int slot = A.pairs[item.pair0 + tp].s + 1;
        const int64_t base = ((int64_t)item.a_out * (A.Nb + 1) + slot) * 9 + ij;
        const int64_t mstride = A.Nout * (A.Nb + 1) * 9;
#pragma unroll
        for (int i = 0; i < kPCols; ++i) {
          const int c = cg * kPCols + i, m = c / A.step;
          if (c < A.NWv && c == m * A.step) {
            double2* o = A.Pi + ((int64_t)qz * A.Nw + m) * mstride + base;
            double2 v = make_double2(A.scale.x * ar[i] - A.scale.y * ai[i], A.scale.x * ai[i] + A.scale.y * ar[i]);
            if (A.accumulate) {
              v.x += o->x;
              v.y += o->y;
            }
            *o = v;
          }
        }
      }
    }
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tm);
  }
}

cudaError_t make_tmap_f32_sw128(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
                                const uint32_t* box);

// Wp: [nitems][4][128][Kw] (Kw = Nkz·NE·NNp); Gp: [Nwin][Nkz][4][Epad][NNp].
cudaError_t launch_pi_contract_tc(const PiCArgs& a, const float* Wp, const float* Gp, int64_t Epad, int NNp, int64_t nitems,
                                  cudaStream_t st) {
  cudaError_t ea = cudaFuncSetAttribute(k_pi_contract_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPSmem);
  if (ea != cudaSuccess) return ea;
  if (a.NWv > kPN || nitems == 0) return a.NWv > kPN ? cudaErrorInvalidValue : cudaSuccess;
  const int KwB = ((a.NEo * NNp + kPKC - 1) / kPKC) * kPKC;
  const uint64_t Kw = (uint64_t)a.Nkz * KwB;
  CUtensorMap tmA, tmB;
  {
    const uint64_t dims[4] = {Kw, kPM, 4, (uint64_t)nitems};
    const uint64_t strides[3] = {Kw * 4, kPM * Kw * 4, 4ull * kPM * Kw * 4};
    const uint32_t box[4] = {kPKC, kPM, 1, 1};
    cudaError_t e = make_tmap_f32_sw128(&tmA, Wp, 4, dims, strides, box);
    if (e != cudaSuccess) return e;
  }
  {
    // B rows m: element k of row m at (shift0 + m)·NNp + k of the (atom, kz', plane) block; inner extent stops
    // before the last row could leave the block (energies >= NE read the zero padding)
    const uint64_t blk = (uint64_t)Epad * NNp;
    const uint64_t dims[5] = {(uint64_t)(Epad - kPN) * NNp, kPN, 4, (uint64_t)a.Nkz, (uint64_t)a.Nwin};
    const uint64_t strides[4] = {(uint64_t)NNp * 4, blk * 4, 4 * blk * 4, (uint64_t)a.Nkz * 4 * blk * 4};
    const uint32_t box[5] = {kPKC, kPN, 1, 1, 1};
    cudaError_t e = make_tmap_f32_sw128(&tmB, Gp, 5, dims, strides, box);
    if (e != cudaSuccess) return e;
  }
  PiTcArgs p;
  p.items = a.items + a.i0;
  p.pairs = a.pairs;
  p.Pi = a.Pi;
  p.scale = a.scale;
  p.ntiles = nitems * a.Nqz;
  p.Nout = a.Nout;
  p.Nb = a.Nb;
  p.NE = a.NE;
  p.Nkz = a.Nkz;
  p.Nqz = a.Nqz;
  p.h = a.h;
  p.Nw = a.Nw;
  p.shift0 = a.shift0;
  p.NWv = a.NWv;
  p.step = a.step;
  p.accumulate = a.accumulate;
  p.NNp = NNp;
  // chunks per kz: energies E < NE - shift0 have in-window terms (R7)
  p.E0 = a.E0;
  p.NEo = a.NEo;
  p.nch = KwB / kPKC;   // every chunk of the kz block: the W tail past NEo·NNp is zero, energies past NE read zero G rows
  int dev = 0, nsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int64_t grid = std::min<int64_t>(p.ntiles, nsm);
  k_pi_contract_tc<<<(unsigned)grid, kPThreads, kPSmem, st>>>(tmA, tmB, p);
  return cudaGetLastError();
}

}  // namespace qt
