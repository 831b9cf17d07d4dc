// kernels_pi.cu — Π≷ (Eq. 4) on sm_100a.
//
// Reformulation (exact up to rounding), for a pair p = (a,s), b = nbr[a][s]:
//   W_p^{ij}(kz,E)[x][y] = (∇_jH_{as} · G^Y_b(kz,E) · ∇_iH_{br})[y][x]          (sandwich, k_pi_w)
//   Π^X_{a,s+1}^{ij}(qz,m) = scale · Σ_{kz,E} Σ_{xy} W_p^{ij}(kz,E)[xy] · G^X_a(kz+qz-h, E+s_m)[xy]
// (cyclic trace: tr{∇_iH_ba G_a ∇_jH_ab G_b} = Σ_xy G_a[x][y] (∇_jH_ab G_b ∇_iH_ba)[y][x]).
// The correlation is a GEMM with rows (pair t, ij) — ≤8 pairs of one destination atom a,
// 72 rows = 9 DMMA m-fragments — columns m and K = (kz, E, xy); the G_a operand is a Hankel
// window (rows E+s_m), held in a shared-memory ring buffer that advances one row per E.
// Π_{a,0} = Σ_s Π_{a,s+1} (R9) is formed by k_pi_self.
#include "kernels_decl.cuh"

namespace qt {

// W^{ij}[x][y] = Σ_q ∇_jH_{as}[y][q] · T_i[q][x],  T_i = G^Y_b · ∇_iH_{br}
__global__ void __launch_bounds__(256) k_pi_w(PiWArgs A) {
  extern __shared__ __align__(16) double2 sm[];
  const int NN = A.NN, No = A.Norb;
  double2* Gb = sm;                 // [kEB][NN]
  double2* Hl = Gb + kEB * NN;      // [3][NN]  ∇_jH_{as}
  double2* Hr = Hl + 3 * NN;        // [3][NN]  ∇_iH_{br}
  double2* T = Hr + 3 * NN;         // [kEB][3][NN]
  const int64_t blk = blockIdx.x;
  const int eb = (int)(blk % A.nEB);
  const int kz = (int)((blk / A.nEB) % A.Nkz);
  const int64_t pl = blk / ((int64_t)A.nEB * A.Nkz);
  const PiPair pr = A.pairs[A.p0 + pl];
  const int e0 = eb * kEB;
  const int ne = min(kEB, A.NE - e0);
  for (int idx = threadIdx.x; idx < kEB * NN; idx += blockDim.x) {
    const int e = idx / NN, uv = idx - e * NN;
    Gb[idx] = e < ne ? A.GY[(((int64_t)kz * A.NE + e0 + e) * A.Nwin + pr.b_in) * NN + uv] : make_double2(0.0, 0.0);
  }
  for (int idx = threadIdx.x; idx < 3 * NN; idx += blockDim.x) {
    Hl[idx] = A.dH[((int64_t)pr.a_in * A.Nb + pr.s) * 3 * NN + idx];
    Hr[idx] = A.dH[((int64_t)pr.b_in * A.Nb + pr.r) * 3 * NN + idx];
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < ne * 3 * NN; idx += blockDim.x) {
    const int e = idx / (3 * NN), rem = idx - e * 3 * NN, i = rem / NN, qx = rem - i * NN;
    const int q = qx / No, x = qx - q * No;
    double2 s = make_double2(0.0, 0.0);
    const double2* g = Gb + e * NN + q * No;
    const double2* h = Hr + i * NN + x;
    for (int p = 0; p < No; ++p) cfma(s, g[p], h[p * No]);
    T[idx] = s;
  }
  __syncthreads();
  double2* out = A.W + (((pl * A.Nkz + kz) * A.NE) + e0) * 9 * NN;
  for (int idx = threadIdx.x; idx < ne * 9 * NN; idx += blockDim.x) {
    const int e = idx / (9 * NN), rem = idx - e * 9 * NN, ij = rem / NN, xy = rem - ij * NN;
    const int i = ij / 3, j = ij - 3 * i, x = xy / No, y = xy - x * No;
    double2 s = make_double2(0.0, 0.0);
    const double2* hl = Hl + j * NN + y * No;
    const double2* t = T + (e * 3 + i) * NN + x;
    for (int q = 0; q < No; ++q) cfma(s, hl[q], t[q * No]);
    out[idx] = s;
  }
}

struct PiCfg {
  static constexpr int XC = 20;       // xy values per step (5 DMMA k-steps)
  static constexpr int XCP = 20;      // row stride (conflict-free fragment LDS.128)
  static constexpr int STAGES = 4;
  static constexpr int A_STAGE = kRows * XCP;
};

// One CTA = (item: destination atom a + ≤8 pairs, qz). Warp w owns m-fragment w and all m columns.
template <int NFM>
__global__ void __launch_bounds__(kThreads, 1) k_pi_contract(PiCArgs A) {
  using C = PiCfg;
  extern __shared__ __align__(16) double2 smem[];
  double2* As = smem;                                   // [STAGES][72][XCP]
  double2* rings = smem + C::STAGES * C::A_STAGE;       // [nring][ring_rows][XCP]
  __shared__ PiPair pairs_s[kMaxPairs];

  const int64_t blk = blockIdx.x;
  const int qz = (int)(blk % A.Nqz);
  const PiItem item = A.items[A.i0 + blk / A.Nqz];
  const int P = item.npair;
  if (threadIdx.x < P) pairs_s[threadIdx.x] = A.pairs[item.pair0 + threadIdx.x];
  __syncthreads();

  const int NN = A.NN, R = A.ring_rows;
  const int nxc = (NN + C::XC - 1) / C::XC;
  const int e_end = A.NE - A.shift0;   // E with at least one in-window E + s_m (R7)
  const int64_t nsteps = e_end > 0 ? (int64_t)A.Nkz * nxc * e_end : 0;

  auto load_step = [&](int slot, int64_t g) {
    const int64_t seg = g / e_end;
    const int e = (int)(g - seg * e_end);
    const int kz = (int)(seg / nxc), xc = (int)(seg - (int64_t)kz * nxc);
    const int xy0 = xc * C::XC;
    double2* as = As + slot * C::A_STAGE;
    for (int idx = threadIdx.x; idx < 9 * P * C::XC; idx += kThreads) {
      const int row = idx / C::XC, c = idx - row * C::XC;
      const int t = row / 9, ij = row - 9 * t;
      const bool v = xy0 + c < NN;
      const int64_t pl = item.pair0 + t - A.p0;
      const double2* src = v ? A.W + (((pl * A.Nkz + kz) * A.NE + e) * 9 + ij) * NN + xy0 + c : A.W;
      cp_async16(as + row * C::XCP + c, src, v);
    }
    const int k2 = (int)imod(kz + qz - A.h, A.Nkz);     // kz + qz (R5)
    double2* ring = rings + (int)(seg % A.nring) * R * C::XCP;
    const int m_lo = e == 0 ? 0 : A.NWP - 1;              // prime the window, then one new row per E
    const int nrow = A.NWP - m_lo;
    for (int idx = threadIdx.x; idx < nrow * C::XC; idx += kThreads) {
      const int mr = idx / C::XC, c = idx - mr * C::XC;
      const int ep = e + A.shift0 + m_lo + mr;
      const bool v = (ep < A.NE) && (xy0 + c < NN);
      const double2* src = v ? A.GX + (((int64_t)k2 * A.NE + ep) * A.Nwin + item.a_in) * NN + xy0 + c : A.GX;
      cp_async16(ring + (ep % R) * C::XCP + c, src, v);
    }
  };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool active = warp * 8 < 9 * P;
  CAcc acc[NFM];
#pragma unroll
  for (int f = 0; f < NFM; ++f) acc[f] = CAcc{0.0, 0.0, 0.0, 0.0};

#pragma unroll
  for (int s = 0; s < C::STAGES - 1; ++s) {
    if (s < nsteps) load_step(s, s);
    cp_async_commit();
  }
  for (int64_t g = 0; g < nsteps; ++g) {
    cp_async_wait<C::STAGES - 2>();
    __syncthreads();
    {
      const int64_t nx = g + C::STAGES - 1;
      if (nx < nsteps) load_step((int)(nx % C::STAGES), nx);
      cp_async_commit();
    }
    if (active) {
      const int64_t seg = g / e_end;
      const int e = (int)(g - seg * e_end);
      const int slot = (int)(g % C::STAGES);
      const double2* ring = rings + (int)(seg % A.nring) * R * C::XCP;
      const double2* as = As + slot * C::A_STAGE + (warp * 8 + (lane >> 2)) * C::XCP + (lane & 3);
      // column fragments with at least one in-window E + s_m
      const int nf = min(NFM, (A.NE - e - A.shift0 + 7) >> 3);
      int rowoff[NFM];
#pragma unroll
      for (int f = 0; f < NFM; ++f) rowoff[f] = ((e + A.shift0 + f * 8 + (lane >> 2)) % R) * C::XCP + (lane & 3);
#pragma unroll
      for (int k4 = 0; k4 < C::XC; k4 += 4) {
        const double2 a = as[k4];
        const double na = -a.y;
#pragma unroll
        for (int f = 0; f < NFM; ++f) {
          if (f < nf) {
            const double2 b = ring[rowoff[f] + k4];
            cmma(acc[f], a.x, a.y, na, b.x, b.y);
          }
        }
      }
    }
  }
  cp_async_wait<0>();

  if (active) {
    const int row = warp * 8 + (lane >> 2);
    const int t = row / 9, ij = row - 9 * t;
    if (t < P) {
      const int slot = pairs_s[t].s + 1;
#pragma unroll
      for (int f = 0; f < NFM; ++f) {
        const int m0 = f * 8 + 2 * (lane & 3);
        if (m0 < A.Nw)
          A.Pi[(((int64_t)qz * A.Nw + m0) * A.Nout + item.a_out) * (A.Nb + 1) * 9 + slot * 9 + ij] =
              cmul(A.scale, make_double2(acc[f].r0, acc[f].i0));
        if (m0 + 1 < A.Nw)
          A.Pi[(((int64_t)qz * A.Nw + m0 + 1) * A.Nout + item.a_out) * (A.Nb + 1) * 9 + slot * 9 + ij] =
              cmul(A.scale, make_double2(acc[f].r1, acc[f].i1));
      }
    }
  }
}

// Π_{a,0} = Σ_{valid s} Π_{a,s+1} (reading R9); empty slots are set to 0 (R12).
__global__ void k_pi_self(PiSelfArgs A) {
  const int64_t total = A.Nqz * A.Nw * A.Nout * 9;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int ij = (int)(idx % 9);
    const int64_t blkid = idx / 9;            // (qz, m, a_out)
    const int64_t a = blkid % A.Nout;
    double2* base = A.Pi + blkid * (A.Nb + 1) * 9;
    double2 s = make_double2(0.0, 0.0);
    for (int64_t t = 0; t < A.Nb; ++t) {
      if (A.nbr[(a + A.a_off) * A.Nb + t] >= 0) {
        const double2 v = base[(t + 1) * 9 + ij];
        s.x += v.x;
        s.y += v.y;
      } else {
        base[(t + 1) * 9 + ij] = make_double2(0.0, 0.0);
      }
    }
    base[ij] = s;
  }
}

// ---------------------------------------------------------------- launchers
cudaError_t launch_pi_w(const PiWArgs& a, int64_t npairs_chunk, cudaStream_t st) {
  int64_t nblk = npairs_chunk * a.Nkz * a.nEB;
  if (nblk == 0) return cudaSuccess;
  size_t smem = (size_t)(kEB * a.NN + 6 * a.NN + kEB * 3 * a.NN) * sizeof(double2);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_pi_w, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  k_pi_w<<<(unsigned)nblk, 256, smem, st>>>(a);
  return cudaGetLastError();
}

size_t pi_contract_smem(int nring, int ring_rows) {
  return (size_t)(PiCfg::STAGES * PiCfg::A_STAGE + nring * ring_rows * PiCfg::XCP) * sizeof(double2);
}

template <int NFM>
static cudaError_t launch_pi_nfm(const PiCArgs& a, int64_t nitems, cudaStream_t st) {
  size_t smem = pi_contract_smem(a.nring, a.ring_rows);
  cudaError_t e = cudaFuncSetAttribute(k_pi_contract<NFM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int64_t nblk = nitems * a.Nqz;
  if (nblk == 0) return cudaSuccess;
  k_pi_contract<NFM><<<(unsigned)nblk, kThreads, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_pi_contract(const PiCArgs& a, int64_t nitems, cudaStream_t st) {
  switch (a.NWP / 8) {
    case 1: return launch_pi_nfm<1>(a, nitems, st);
    case 2: return launch_pi_nfm<2>(a, nitems, st);
    case 3: return launch_pi_nfm<3>(a, nitems, st);
    case 4: return launch_pi_nfm<4>(a, nitems, st);
    case 5: return launch_pi_nfm<5>(a, nitems, st);
    case 6: return launch_pi_nfm<6>(a, nitems, st);
    case 7: return launch_pi_nfm<7>(a, nitems, st);
    case 8: return launch_pi_nfm<8>(a, nitems, st);
    case 9: return launch_pi_nfm<9>(a, nitems, st);
    case 10: return launch_pi_nfm<10>(a, nitems, st);
    case 11: return launch_pi_nfm<11>(a, nitems, st);
    case 12: return launch_pi_nfm<12>(a, nitems, st);
    case 13: return launch_pi_nfm<13>(a, nitems, st);
    case 14: return launch_pi_nfm<14>(a, nitems, st);
    case 15: return launch_pi_nfm<15>(a, nitems, st);
    case 16: return launch_pi_nfm<16>(a, nitems, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_pi_self(const PiSelfArgs& a, cudaStream_t st) {
  int64_t total = a.Nqz * a.Nw * a.Nout * 9;
  if (total == 0) return cudaSuccess;
  int64_t g = (total + 255) / 256;
  if (g > 148 * 32) g = 148 * 32;
  k_pi_self<<<(int)g, 256, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace qt
