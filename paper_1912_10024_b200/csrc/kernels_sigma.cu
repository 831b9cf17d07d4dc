// kernels_sigma.cu — Σ≷ (Eq. 3) on sm_100a.
//
// Reformulation (exact up to rounding): for a pair p = (a,s), b = nbr[a][s],
//   Gt_p^{ij}(kz,E) = Σ_{q,d} C_p^{ij}(q,d) · G_b(kz-q+h, E+d)              (D-contraction)
//   Σ_a(kz,E)      = scale · Σ_s Σ_i ∇_iH_{as} ( Σ_j Gt_p^{ij} ∇_jH_{br} )     (sandwich + neighbour sum)
// with C_p^{ij}(q,-s_m) = Dc^X_{ij}(q,m), C_p^{ij}(q,+s_m) = Dc^Y_{ji}(q,m), 0 otherwise (R2, R3).
// The contraction is a GEMM with rows (pair t, ij) — the ≤8 pairs sharing one source atom b,
// 72 rows = 9 DMMA m-fragments — columns rc (Norb² orbital entries of G_b) and K = (q, d):
// the G operand is a Hankel window of G_b rows E+d. It runs on FP64 tensor cores
// (mma.sync m8n8k4 -> DMMA.8x8x4), staged through shared memory with cp.async.
#include "kernels_decl.cuh"

namespace qt {

// C_p^{ij}(q, dd) with d = dd - Dmax: the four-term D combination of Eq. 3.
__global__ void k_sigma_coef(CoefArgs A) {
  const int64_t total = A.npairs * 9 * A.Nqz * A.DWp;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t dd = idx % A.DWp, t = idx / A.DWp;
    int64_t q = t % A.Nqz;
    t /= A.Nqz;
    int ij = (int)(t % 9);
    int64_t p = t / 9;
    const SigPair pr = A.pairs[p];
    const int64_t b = A.items[A.pair_item[p]].b_in;
    int64_t d = dd - A.Dmax;
    double2 v = make_double2(0.0, 0.0);
    int64_t ad = d < 0 ? -d : d;
    if (ad >= A.shift0 && ad <= A.Dmax && (ad - A.shift0) % A.step == 0) {
      int64_t m = (ad - A.shift0) / A.step;
      // absorption (E - ħω): Dc^X_{ij}; emission (E + ħω): Dc^Y_{ji} (reading R3)
      const double2* D = d < 0 ? A.DX : A.DY;
      int e = d < 0 ? ij : (ij % 3) * 3 + ij / 3;
      const int64_t base = (q * A.Nw + m) * A.Nwin;
      const int64_t ns = A.Nb + 1;
      double2 dba = D[((base + b) * ns + pr.r + 1) * 9 + e];
      double2 dbb = D[((base + b) * ns + 0) * 9 + e];
      double2 daa = D[((base + pr.a_in) * ns + 0) * 9 + e];
      double2 dab = D[((base + pr.a_in) * ns + pr.s + 1) * 9 + e];
      v.x = ((dba.x - dbb.x) - daa.x) + dab.x;
      v.y = ((dba.y - dbb.y) - daa.y) + dab.y;
    }
    A.coef[idx] = v;
  }
}

template <int NF>
struct SigmaCfg {
  static constexpr int NP = 8 * NF;                 // padded Norb² (n-fragments of 8)
  static constexpr int NPS = NP + 2;                // row stride: conflict-free B-fragment LDS.128
  static constexpr int KC = 16;                     // d values per pipeline stage
  static constexpr int KCP = 20;                    // coef row stride: conflict-free A-fragment LDS.128
  static constexpr int STAGES = NF > 13 ? 2 : 3;
  static constexpr int G_STAGE = KC * NPS;
  static constexpr int C_STAGE = kRows * KCP;
  static constexpr int PIPE = STAGES * (G_STAGE + C_STAGE);
  static constexpr int GT = kRows * NPS;
  static constexpr int REGION1 = PIPE > GT ? PIPE : GT;
  static constexpr int VS = kMaxPairs * 3 * NP;
  static constexpr size_t SMEM = (size_t)(REGION1 + VS) * sizeof(double2);
};

// cp.async variant, used for Norb = 11, 12 (Norb² rows too wide for one TMA box; see kernels_sigma_tma.cu).
// One CTA = (item: source atom b + ≤8 pairs, kz, E). 9 warps; warp w owns m-fragment w (rows 8w..8w+7)
// and all NF n-fragments.
template <int NF>
__global__ void __launch_bounds__(kThreads, 1) k_sigma_cp(SigmaArgs A) {
  using C = SigmaCfg<NF>;
  extern __shared__ __align__(16) double2 smem[];
  double2* Gs = smem;
  double2* Cs = smem + C::STAGES * C::G_STAGE;
  __shared__ SigPair pairs_s[kMaxPairs];

  const int64_t blk = blockIdx.x;
  const int E = (int)(blk % A.NE);
  const int kz = (int)((blk / A.NE) % A.Nkz);
  const int64_t it = blk / ((int64_t)A.NE * A.Nkz);
  const SigItem item = A.items[it];
  const int P = item.npair;
  if (threadIdx.x < P) pairs_s[threadIdx.x] = A.pairs[item.pair0 + threadIdx.x];

  // K range: d with E+d in [0,NE) (reading R7), rounded to the k=4 DMMA step.
  int dd_lo = max(0, A.Dmax - E), dd_hi = min(A.Dwin, A.Dmax - E + A.NE);
  dd_lo &= ~3;
  dd_hi = (dd_hi + 3) & ~3;
  const int nchunk = (dd_hi - dd_lo + C::KC - 1) / C::KC;
  const int nst = A.Nqz * nchunk;
  const int NN = A.NN;

  auto load_stage = [&](int slot, int st) {
    const int q = st / nchunk, c = st % nchunk;
    const int dd0 = dd_lo + c * C::KC;
    const int kc = min(C::KC, dd_hi - dd0);
    const int kp = (int)imod(kz - q + A.h, A.Nkz);   // kz - qz (R4, R5)
    double2* gs = Gs + slot * C::G_STAGE;
    for (int idx = threadIdx.x; idx < kc * NN; idx += kThreads) {
      const int kk = idx / NN, rc = idx - kk * NN;
      const int Ep = E - A.Dmax + dd0 + kk;
      const bool v = (Ep >= 0) && (Ep < A.NE);     // outside the window: zero-filled row (R7)
      const double2* src = v ? A.G + (((int64_t)kp * A.NE + Ep) * A.Nwin + item.b_in) * NN + rc : A.G;
      cp_async16(gs + kk * C::NPS + rc, src, v);
    }
    double2* cs = Cs + slot * C::C_STAGE;
    for (int idx = threadIdx.x; idx < 9 * P * kc; idx += kThreads) {
      const int row = idx / kc, kk = idx - row * kc;
      const int t = row / 9, ij = row - 9 * t;
      const double2* src = A.coef + (((int64_t)(item.pair0 - A.cp0 + t) * 9 + ij) * A.Nqz + q) * A.DWp + dd0 + kk;
      cp_async16(cs + row * C::KCP + kk, src, true);
    }
  };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool active = warp * 8 < 9 * P;
  CAcc acc[NF];
#pragma unroll
  for (int f = 0; f < NF; ++f) acc[f] = CAcc{0.0, 0.0, 0.0, 0.0};

#pragma unroll
  for (int s = 0; s < C::STAGES - 1; ++s) {
    if (s < nst) load_stage(s, s);
    cp_async_commit();
  }
  for (int st = 0; st < nst; ++st) {
    cp_async_wait<C::STAGES - 2>();
    __syncthreads();
    {
      const int nx = st + C::STAGES - 1;
      if (nx < nst) load_stage(nx % C::STAGES, nx);
      cp_async_commit();
    }
    if (active) {
      const int slot = st % C::STAGES;
      const int dd0 = dd_lo + (st % nchunk) * C::KC;
      const int kc = min(C::KC, dd_hi - dd0);
      const double2* gs = Gs + slot * C::G_STAGE + (lane & 3) * C::NPS + (lane >> 2);
      const double2* cs = Cs + slot * C::C_STAGE + (warp * 8 + (lane >> 2)) * C::KCP + (lane & 3);
#pragma unroll
      for (int k4 = 0; k4 < C::KC; k4 += 4) {
        if (k4 < kc) {
          const double2 a = cs[k4];
          const double na = -a.y;
          const double2* gb = gs + k4 * C::NPS;
#pragma unroll
          for (int f = 0; f < NF; ++f) {
            const double2 b = gb[f * 8];
            cmma(acc[f], a.x, a.y, na, b.x, b.y);
          }
        }
      }
    }
  }
  cp_async_wait<0>();
  __syncthreads();

  // ---- epilogue 1: Gt (72 x NP) -> shared memory (aliases the pipeline buffers)
  double2* Gt = smem;
  if (active) {
    const int row = warp * 8 + (lane >> 2);
#pragma unroll
    for (int f = 0; f < NF; ++f) {
      const int col = f * 8 + 2 * (lane & 3);
      Gt[row * C::NPS + col] = make_double2(acc[f].r0, acc[f].i0);
      Gt[row * C::NPS + col + 1] = make_double2(acc[f].r1, acc[f].i1);
    }
  }
  __syncthreads();

  // ---- epilogue 2: V^i_t = Σ_j Gt^{ij}_t · ∇_jH_{b r_t}
  const int No = A.Norb;
  double2* Vs = smem + C::REGION1;
  for (int idx = threadIdx.x; idx < P * 3 * NN; idx += kThreads) {
    const int t = idx / (3 * NN), rem = idx - t * 3 * NN, i = rem / NN, xy = rem - i * NN;
    const int x = xy / No, y = xy - x * No;
    const SigPair pr = pairs_s[t];
    double2 s = make_double2(0.0, 0.0);
    for (int j = 0; j < 3; ++j) {
      const double2* g = Gt + (t * 9 + i * 3 + j) * C::NPS + x * No;
      const double2* hr = A.dH + (((int64_t)item.b_in * A.Nb + pr.r) * 3 + j) * NN + y;
      for (int v = 0; v < No; ++v) cfma(s, g[v], __ldg(hr + v * No));
    }
    Vs[(t * 3 + i) * NN + xy] = s;
  }
  __syncthreads();

  // ---- epilogue 3: S_t = Σ_i ∇_iH_{a_t s_t} · V^i_t; Σ_a += scale · S_t (R8)
  for (int idx = threadIdx.x; idx < P * NN; idx += kThreads) {
    const int t = idx / NN, xy = idx - t * NN, x = xy / No, y = xy - x * No;
    const SigPair pr = pairs_s[t];
    double2 s = make_double2(0.0, 0.0);
    for (int i = 0; i < 3; ++i) {
      const double2* hl = A.dH + (((int64_t)pr.a_in * A.Nb + pr.s) * 3 + i) * NN + x * No;
      const double2* v = Vs + (t * 3 + i) * NN + y;
      for (int u = 0; u < No; ++u) cfma(s, __ldg(hl + u), v[u * No]);
    }
    const double2 r = cmul(A.scale, s);
    double* dst = reinterpret_cast<double*>(A.Sig + (((int64_t)kz * A.NE + E) * A.Nout + pr.a) * NN + xy);
    atomicAdd(dst, r.x);
    atomicAdd(dst + 1, r.y);
  }
}

// ---------------------------------------------------------------- launchers
cudaError_t launch_sigma_coef(const CoefArgs& a, cudaStream_t st) {
  int64_t total = a.npairs * 9 * a.Nqz * a.DWp;
  if (total == 0) return cudaSuccess;
  int64_t g = (total + 255) / 256;
  if (g > 148 * 32) g = 148 * 32;
  k_sigma_coef<<<(int)g, 256, 0, st>>>(a);
  return cudaGetLastError();
}

template <int NF>
static cudaError_t launch_sigma_nf(const SigmaArgs& a, int64_t nitems, cudaStream_t st) {
  using C = SigmaCfg<NF>;
  cudaError_t ea = cudaFuncSetAttribute(k_sigma_cp<NF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
  if (ea != cudaSuccess) return ea;
  int64_t nblk = nitems * a.NE * a.Nkz;
  if (nblk == 0) return cudaSuccess;
  if (nblk > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  k_sigma_cp<NF><<<(unsigned)nblk, kThreads, C::SMEM, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_sigma_cp(const SigmaArgs& a, int64_t nitems, cudaStream_t st) {
  switch ((a.NN + 7) / 8) {
    case 16: return launch_sigma_nf<16>(a, nitems, st);
    case 18: return launch_sigma_nf<18>(a, nitems, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace qt
