// kernels_sigma_tc.cu — Σ≷ D-contraction (Eq. 3) in the FP32 mixed-precision mode
// (QT_PREC_FP32_MIXED; §4.4: reduced-precision products,
// wide accumulation) on the 5th-generation tensor cores: tcgen05.mma kind::tf32, accumulators in TMEM.
//
// Same contraction as k_sigma (Gt^{ij}_t(kz,E) = Σ_{q,d} C^{ij}_t(q,d) · G_b(kz−q+h, E+d)), transposed so
// the Norb² entries of G are the UMMA M dimension:
//   D[rc][n] = Σ_k A[rc][k] · B[n][k],  A = G_b rows E+d (a Hankel window; K-major copy of G with E
//   contiguous, so the window is one TMA box whose out-of-range energies are zero-filled = reading R7),
//   B = the item's coefficient rows n = (t, ij) (72, padded to N = 80).
// Precision: every operand is split x ≈ hi + lo with hi = tf32(x), lo = tf32(x − hi) ("3xTF32"), and a real
// product is hi·hi + hi·lo + lo·hi (relative error ~2^-21); complex products use four real products
// (Re = ArBr − AiBi via the UMMA negate-A bit, Im = ArBi + AiBr): 12 UMMAs per 8-wide k-step. FP32
// accumulation in TMEM over SEGMENTS of kTcSegChunks K-chunks (128 shifts; the tensor core's FP32 accumulation
// error grows with the number of additions into one accumulator: 1.3e-5 per block after K = 987 products at
// the cfg4 shape with one accumulator per tile), the segments summed by the epilogue in FP32 registers with
// round-to-nearest adds; the epilogue stores the FP32 Gt scratch and the ∇H sandwich (k_sigma_sand<_, float>)
// runs in FP32, adding into the FP64 Σ.
//
// Warp roles (persistent CTA per SM, 576 threads): warp 0 = TMA producer, warp 1 = UMMA issuer (+ TMEM
// allocation), warps 2..17 = epilogue (TMEM lane quarter warp%4: rc rows 32·(warp%4) ..; column group
// (warp-2)/4: 32 of the 128 coefficient rows). Two TMEM accumulator buffers (Re|Im = 256 columns each)
// alternate between segments, so the epilogue drains one segment while the MMAs fill the next.
#include "kernels_decl.cuh"
#include "tc05.cuh"
#include "tma.cuh"

#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

namespace qt {

constexpr int kTcM = kTcRowsA;                   // UMMA M: Norb² entries of a G block (Norb <= 11)
constexpr int kTcN = kTcRows;                    // UMMA N: the item's <= 126 coefficient rows (14 pairs)
constexpr int kTcKC = 16;                        // shifts per stage: one 64-byte swizzle row of fp32
constexpr int kTcStages = 3;
constexpr int kTcAPlane = kTcM * kTcKC;          // floats per A plane tile (8 KB)
constexpr int kTcBPlane = kTcN * kTcKC;          // floats per B plane tile (8 KB)
constexpr int kTcStage = 4 * (kTcAPlane + kTcBPlane);
constexpr uint32_t kTcStageBytes = kTcStage * 4;
constexpr int kTcBufCols = 256;                  // TMEM columns per accumulator buffer (Re: 0..127, Im: 128..255)
constexpr int kTcSegChunks = 8;                  // K-chunks per TMEM accumulation segment (128 shifts)
constexpr int kTcEpiWarps = 16;                  // epilogue warps: 4 TMEM lane quarters x 4 groups of 32 columns
constexpr int kTcThreads = (2 + kTcEpiWarps) * 32;
constexpr size_t kTcSmem = (size_t)kTcStages * kTcStageBytes + 1024 + 256;
static_assert(kTcSmem <= 227 * 1024, "shared memory");

// ---------------------------------------------------------------- operand preparation
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
// x (FP64) -> (hi, lo): hi = tf32(x), lo = tf32(x - hi), both rounded to nearest (a truncated lo would bias
// every hi·lo product the same way; rounded, the split error ~2^-22 |x| is unbiased)
__device__ __forceinline__ void split3(double x, float& hi, float& lo) {
  hi = tf32_rna((float)x);
  lo = tf32_rna((float)(x - (double)hi));
}

// G (paper layout [Nkz][NE][Nwin][NN], complex128) -> Gtp[a][kz][plane][rc < kTcRowsA][NEp] fp32, planes
// (re_hi, re_lo, im_hi, im_lo); rows rc >= NN and energies >= NE are zero (every TMA box lies inside
// the tensor: NEp >= 32 and 128 rows).
__global__ void __launch_bounds__(256) k_relayout_tc(const double2* __restrict__ G, float* __restrict__ out,
                                                     int64_t Nkz, int64_t NE, int64_t NEp, int64_t Nwin, int NN,
                                                     int64_t a0) {
  __shared__ float tile[4][32][33];
  const int64_t a = a0 + blockIdx.x / Nkz, kz = blockIdx.x % Nkz;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 x 8
  float* o = out + (a * Nkz + kz) * 4 * (int64_t)kTcRowsA * NEp;
  for (int64_t e0 = 0; e0 < NEp; e0 += 32) {
    for (int r0 = 0; r0 < kTcRowsA; r0 += 32) {
      __syncthreads();
      for (int j = ty; j < 32; j += 8) {   // read: e = e0 + j, rc = r0 + tx (rc contiguous)
        const int64_t e = e0 + j;
        const int rc = r0 + tx;
        double2 v = make_double2(0.0, 0.0);
        if (e < NE && rc < NN) v = __ldg(G + ((kz * NE + e) * Nwin + a) * NN + rc);
        float h, l;
        split3(v.x, h, l);
        tile[0][j][tx] = h;
        tile[1][j][tx] = l;
        split3(v.y, h, l);
        tile[2][j][tx] = h;
        tile[3][j][tx] = l;
      }
      __syncthreads();
      for (int j = ty; j < 32; j += 8) {   // write: rc = r0 + j, e = e0 + tx (e contiguous)
        const int rc = r0 + j;
        const int64_t e = e0 + tx;
        if (e < NEp) {
#pragma unroll
          for (int p = 0; p < 4; ++p) o[((int64_t)p * kTcRowsA + rc) * NEp + e] = tile[p][tx][j];
        }
      }
    }
  }
}

cudaError_t launch_relayout_tc(const double2* G, float* out, int64_t Nkz, int64_t NE, int64_t NEp, int64_t Nwin, int NN,
                               int64_t a0, int64_t a1, cudaStream_t st) {
  if (Nkz * (a1 - a0) <= 0) return cudaSuccess;
  k_relayout_tc<<<(unsigned)(Nkz * (a1 - a0)), 256, 0, st>>>(G, out, Nkz, NE, NEp, Nwin, NN, a0);
  return cudaGetLastError();
}

// Coefficient planes: coef[il][q][s][plane][row n < 80][k < Kp] fp32 holding C(d = k - s), i.e. the shift
// index d (energy shift d - Dmax) delayed by s = 0..3: a TMA box must start on a 16-byte boundary, so the
// tile of energy E reads the G window from the aligned row E - Dmax + 32c - s (s = (E - Dmax) mod 4) and the
// copy of the coefficients delayed by the same s. Values: the Eq. 3 four-term combination
// C^{ij}(q, -s_m) = Dc^X_{ij}, C^{ij}(q, +s_m) = Dc^Y_{ji} (readings R2, R3); rows n >= 9·npair and
// d outside [0, Dwin) are zero.
__global__ void k_sigma_coef_tc(CoefArgs A, int Kp) {
  // one thread per (item, q, row n, shift d < Kp): forms C(d) once and stores it at k = d + s of each delay s
  // (thread d = k also zeroes the leading slots k < s); every store is coalesced over the warp's consecutive d
  const int64_t per_item = A.Nqz * (int64_t)kTcN * Kp;
  const int64_t total = A.nitems * per_item;
  const int64_t pp0 = A.items[A.item0].pair0;
  float* out = reinterpret_cast<float*>(A.coef);
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int d = (int)(idx % Kp);
    int64_t r = idx / Kp;
    const int n = (int)(r % kTcN);
    r /= kTcN;
    const int64_t q = r % A.Nqz;
    const int64_t il = r / A.Nqz;
    const SigItem item = A.items[A.item0 + il];
    const int t = n / 9, ij = n - 9 * t;
    double2 c = make_double2(0.0, 0.0);
    if (t < item.npair && d < A.Dwin) {
      const int64_t dd = d - A.Dmax, ad = dd < 0 ? -dd : dd;
      if (ad >= A.shift0 && ad <= A.Dmax && (ad - A.shift0) % A.step == 0) {
        const SigPair pr = A.pairs[item.pair0 - pp0 + t];
        const int64_t b = item.b_in, m = (ad - A.shift0) / A.step, ns = A.Nb + 1;
        const double2* D = dd < 0 ? A.DX : A.DY;
        const int e = dd < 0 ? ij : (ij % 3) * 3 + ij / 3;
        const int64_t base = (q * A.Nw + m) * A.Nwin;
        const double2 dba = D[((base + b) * ns + pr.r + 1) * 9 + e];
        const double2 dbb = D[((base + b) * ns + 0) * 9 + e];
        const double2 daa = D[((base + pr.a_in) * ns + 0) * 9 + e];
        const double2 dab = D[((base + pr.a_in) * ns + pr.s + 1) * 9 + e];
        c.x = ((dba.x - dbb.x) - daa.x) + dab.x;
        c.y = ((dba.y - dbb.y) - daa.y) + dab.y;
      }
    }
    float v[4];
    split3(c.x, v[0], v[1]);
    split3(c.y, v[2], v[3]);
    float* o = out + ((il * A.Nqz + q) * 16 * kTcN + n) * (int64_t)Kp;   // [s][plane][n][k] below
#pragma unroll
    for (int sh = 0; sh < 4; ++sh) {
      const int k = d + sh;
      if (k < Kp) {
#pragma unroll
        for (int p = 0; p < 4; ++p) o[(int64_t)(sh * 4 + p) * kTcN * Kp + k] = v[p];
      }
      if (d < sh) {   // leading slots k < s of delay s hold C(k - s), k - s < 0: zero
#pragma unroll
        for (int p = 0; p < 4; ++p) o[(int64_t)(sh * 4 + p) * kTcN * Kp + d] = 0.0f;
      }
    }
  }
}

cudaError_t launch_sigma_coef_tc(const CoefArgs& a, int Kp, cudaStream_t st) {
  const int64_t total = a.nitems * a.Nqz * kTcN * Kp;
  if (total == 0) return cudaSuccess;
  int64_t g = (total + 255) / 256;
  if (g > 148 * 32) g = 148 * 32;
  k_sigma_coef_tc<<<(int)g, 256, 0, st>>>(a, Kp);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- the tcgen05 contraction
struct TcTile {
  int il, kz, E, dlo, dhi, sh, c0, nchunk, nst;
  SigItem item;
};
__device__ __forceinline__ TcTile tc_tile(const SigmaArgs& A, int64_t t) {
  TcTile T;
  T.E = A.E0 + (int)(t % A.NEo);              // output energy (window coordinates)
  T.kz = (int)((t / A.NEo) % A.Nkz);
  T.il = (int)(t / ((int64_t)A.NEo * A.Nkz));
  T.item = A.items[T.il];
  // shifts d (energy E + d - Dmax) inside the window (R7). Chunk c covers d = 32c - sh + j, j < 32, with
  // sh = (E - Dmax) mod 4, so its G rows start at the 16-byte aligned row E - Dmax + 32c - sh.
  T.dlo = max(0, A.Dmax - T.E);
  T.dhi = min(A.Dwin, A.Dmax - T.E + A.NE);
  T.sh = (int)imod(T.E - A.Dmax, 4);
  T.c0 = (T.dlo + T.sh) / kTcKC;
  T.nchunk = (T.dhi + T.sh + kTcKC - 1) / kTcKC - T.c0;
  T.nst = A.Nqz * T.nchunk;
  return T;
}

__global__ void __launch_bounds__(kTcThreads, 1)
    k_sigma_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, SigmaArgs A) {
  extern __shared__ uint8_t smem_raw[];
  float* stages = reinterpret_cast<float*>(smem_raw + ((-smem_u32(smem_raw)) & 1023u));
  uint64_t* full = reinterpret_cast<uint64_t*>(stages + kTcStages * kTcStage);
  uint64_t* empty = full + kTcStages;
  uint64_t* tfull = empty + kTcStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tbase = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 1) tmem_alloc<512>(tbase);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kTcStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], kTcEpiWarps);
    }
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = *tbase;

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      prefetch_tmap(&tmA);
      prefetch_tmap(&tmB);
      uint32_t g = 0;
      for (int64_t t = blockIdx.x; t < A.ntiles; t += gridDim.x) {
        const TcTile T = tc_tile(A, t);
        for (int q = 0; q < A.Nqz; ++q) {
          const int kp = (int)imod(T.kz - q + A.h, A.Nkz);       // kz - qz (R4, R5)
          for (int c = 0; c < T.nchunk; ++c, ++g) {
            const uint32_t slot = g % kTcStages;
            if (g >= kTcStages) mbar_wait(&empty[slot], ((g / kTcStages) - 1) & 1);
            float* sa = stages + slot * kTcStage;
            float* sb = sa + 4 * kTcAPlane;
            const int kc = (T.c0 + c) * kTcKC;                           // B column of this chunk
            const int row = T.E - A.Dmax + kc - T.sh;                     // first G row (multiple of 4)
            mbar_arrive_expect_tx(&full[slot], kTcStageBytes);
            for (int p = 0; p < 4; ++p) {
              tma_load_5d(sa + p * kTcAPlane, &tmA, row, 0, p, kp, T.item.b_in, &full[slot]);
              tma_load_5d(sb + p * kTcBPlane, &tmB, kc, 0, T.sh * 4 + p, q, T.il, &full[slot]);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- UMMA issuer (one thread): each segment of kTcSegChunks chunks into the next buffer
    if (lane == 0) {
      const uint32_t id_pos = umma_idesc_tf32(kTcM, kTcN, false, false);
      const uint32_t id_neg = umma_idesc_tf32(kTcM, kTcN, true, false);
      uint32_t g = 0, sc = 0;
      for (int64_t t = blockIdx.x; t < A.ntiles; t += gridDim.x) {
        const TcTile T = tc_tile(A, t);
        const int nck = A.Nqz * T.nchunk;
        const int nseg = (nck + kTcSegChunks - 1) / kTcSegChunks;
        for (int sg = 0; sg < nseg; ++sg, ++sc) {
          const uint32_t buf = sc & 1;
          if (sc >= 2) mbar_wait(&tempty[buf], ((sc / 2) - 1) & 1);
          tc_fence_after();
          const uint32_t dre = tm + buf * kTcBufCols, dim = dre + kTcN;
          bool acc = false;
          const int cend = min(nck, (sg + 1) * kTcSegChunks);
          for (int ci = sg * kTcSegChunks; ci < cend; ++ci, ++g) {
            const int c = ci % T.nchunk;
            const uint32_t slot = g % kTcStages;
            mbar_wait(&full[slot], (g / kTcStages) & 1);
            tc_fence_after();
            const float* sa = stages + slot * kTcStage;
            const float* sb = sa + 4 * kTcAPlane;
            // k-steps of 8 shifts j with 16(c0+c) + j in [dlo + sh, dhi + sh)
            const int kc = (T.c0 + c) * kTcKC;
            const int k_lo = max(0, T.dlo + T.sh - kc) / 8, k_hi = min(kTcKC, T.dhi + T.sh - kc + 7) / 8;
            for (int kk = k_lo; kk < k_hi; ++kk) {
              const uint64_t arh = umma_desc_k64(sa + 0 * kTcAPlane + kk * 8);
              const uint64_t arl = umma_desc_k64(sa + 1 * kTcAPlane + kk * 8);
              const uint64_t aih = umma_desc_k64(sa + 2 * kTcAPlane + kk * 8);
              const uint64_t ail = umma_desc_k64(sa + 3 * kTcAPlane + kk * 8);
              const uint64_t brh = umma_desc_k64(sb + 0 * kTcBPlane + kk * 8);
              const uint64_t brl = umma_desc_k64(sb + 1 * kTcBPlane + kk * 8);
              const uint64_t bih = umma_desc_k64(sb + 2 * kTcBPlane + kk * 8);
              const uint64_t bil = umma_desc_k64(sb + 3 * kTcBPlane + kk * 8);
              // Re += Ar·Br − Ai·Bi
              umma_tf32(dre, arh, brh, id_pos, acc);
              umma_tf32(dre, arh, brl, id_pos, true);
              umma_tf32(dre, arl, brh, id_pos, true);
              umma_tf32(dre, aih, bih, id_neg, true);
              umma_tf32(dre, aih, bil, id_neg, true);
              umma_tf32(dre, ail, bih, id_neg, true);
              // Im += Ar·Bi + Ai·Br
              umma_tf32(dim, arh, bih, id_pos, acc);
              umma_tf32(dim, arh, bil, id_pos, true);
              umma_tf32(dim, arl, bih, id_pos, true);
              umma_tf32(dim, aih, brh, id_pos, true);
              umma_tf32(dim, aih, brl, id_pos, true);
              umma_tf32(dim, ail, brh, id_pos, true);
              acc = true;
            }
            umma_commit(&empty[slot]);   // frees the stage when these MMAs complete
          }
          umma_commit(&tfull[buf]);      // segment ready for the epilogue
        }
      }
    }
  } else {
    // ---------------- epilogue: segments (FP32, TMEM) summed in registers, then the FP32 Gt scratch
    const int quarter = warp & 3;
    const int cg = (warp - 2) >> 2;             // coefficient rows n in [cg·32, cg·32 + 32)
    const int rc = quarter * 32 + lane;
    uint32_t sc = 0;
    for (int64_t t = blockIdx.x; t < A.ntiles; t += gridDim.x) {
      const TcTile T = tc_tile(A, t);
      const int nck = A.Nqz * T.nchunk;
      const int nseg = (nck + kTcSegChunks - 1) / kTcSegChunks;
      float re[32], im[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) re[i] = im[i] = 0.f;
      for (int sg = 0; sg < nseg; ++sg, ++sc) {
        const uint32_t buf = sc & 1;
        mbar_wait(&tfull[buf], (sc / 2) & 1);
        tc_fence_after();
        const uint32_t taddr = tm + ((uint32_t)(quarter * 32) << 16) + buf * kTcBufCols + cg * 32;
        float v[16];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          tmem_ld16(taddr + 16 * h, v);
#pragma unroll
          for (int i = 0; i < 16; ++i) re[16 * h + i] += v[i];
          tmem_ld16(taddr + kTcN + 16 * h, v);
#pragma unroll
          for (int i = 0; i < 16; ++i) im[16 * h + i] += v[i];
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[buf]);   // buffer free: the registers hold this segment
      }
      const int rows = 9 * T.item.npair;
      if (rc < A.NN) {
        float2* out = reinterpret_cast<float2*>(A.Gt) +
                      (((int64_t)T.il * A.Nkz + T.kz) * A.NEo + T.E - A.E0) * A.rows * A.gt_ld + rc;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int n = cg * 32 + i;
          if (n < rows) out[(int64_t)n * A.gt_ld] = make_float2(re[i], im[i]);
        }
      }
    }
  }
  __syncwarp();   // reconverge the single-lane roles before the CTA barrier
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tm);
  }
}

cudaError_t make_tmap_f32_sw128(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
                                const uint32_t* box) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return cudaErrorNotSupported;
  auto fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  const uint32_t estr[5] = {1, 1, 1, 1, 1};
  // swizzle span = the box's inner row (16 fp32 = 64 B for Σ, 32 fp32 = 128 B for Π)
  const CUtensorMapSwizzle sw = box[0] * 4 == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B;
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, (cuuint32_t)rank, const_cast<void*>(base), dims, strides, box,
                  estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS && getenv("QT_DEBUG"))
    fprintf(stderr, "qt_sse: cuTensorMapEncodeTiled (fp32, rank %d, dims %llu x %llu, box %u x %u) failed: %d\n", rank,
            (unsigned long long)dims[0], (unsigned long long)dims[1], box[0], box[1], (int)r);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// Gtp: [Nwin][Nkz][4][128][NEp] fp32; coef: [nitems][Nqz][4 delays][4 planes][80][Kp] fp32.
cudaError_t launch_sigma_tc(const SigmaArgs& a, const float* Gtp, int64_t NEp, const float* coef, int Kp, int64_t nitems,
                            cudaStream_t st) {
  cudaError_t ea = cudaFuncSetAttribute(k_sigma_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTcSmem);
  if (ea != cudaSuccess) return ea;
  if (a.NN > kTcM || NEp < kTcKC || Kp < kTcKC || (Kp & 31)) return cudaErrorInvalidValue;
  CUtensorMap tmA, tmB;
  {
    const uint64_t NN = (uint64_t)kTcRowsA;
    const uint64_t dims[5] = {(uint64_t)NEp, NN, 4, (uint64_t)a.Nkz, (uint64_t)a.Nwin};
    const uint64_t strides[4] = {(uint64_t)NEp * 4, NN * NEp * 4, 4 * NN * NEp * 4, (uint64_t)a.Nkz * 4 * NN * NEp * 4};
    const uint32_t box[5] = {kTcKC, kTcM, 1, 1, 1};
    cudaError_t e = make_tmap_f32_sw128(&tmA, Gtp, 5, dims, strides, box);
    if (e != cudaSuccess) return e;
  }
  {
    const uint64_t dims[5] = {(uint64_t)Kp, kTcN, 16, (uint64_t)a.Nqz, (uint64_t)nitems};
    const uint64_t strides[4] = {(uint64_t)Kp * 4, (uint64_t)kTcN * Kp * 4, 16ull * kTcN * Kp * 4,
                                 (uint64_t)a.Nqz * 16 * kTcN * Kp * 4};
    const uint32_t box[5] = {kTcKC, kTcN, 1, 1, 1};
    cudaError_t e = make_tmap_f32_sw128(&tmB, coef, 5, dims, strides, box);
    if (e != cudaSuccess) return e;
  }
  SigmaArgs b = a;
  b.ntiles = nitems * a.Nkz * a.NEo;
  if (b.ntiles == 0) return cudaSuccess;
  int dev = 0, nsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int64_t grid = std::min<int64_t>(b.ntiles, nsm);
  k_sigma_tc<<<(unsigned)grid, kTcThreads, kTcSmem, st>>>(tmA, tmB, b);
  return cudaGetLastError();
}

}  // namespace qt
