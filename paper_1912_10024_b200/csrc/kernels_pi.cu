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
#include "tma.cuh"

namespace qt {

// W^{ij}[x][y] = Σ_q ∇_jH_{as}[y][q] · T_i[q][x],  T_i = G^Y_b · ∇_iH_{br}   (the Π sandwich)
// One CTA per (work item, kz, half of the item's pairs), looping over energy pairs. Compile-time Norb;
// T-threads own a row (t, e, i, q) of T_i = G^Y_b ∇_iH_{br}, W-threads own a column set (t, e, i, j, y):
// W^{ij}[x][y] = Σ_q ∇_jH_{as}[y][q] T_i[q][x] for all x. The W block of (item, kz, E) is 72 contiguous
// rows per 20-wide xy chunk; each thread's stores fill part of it (L2 merges the partial lines).
#ifndef QT_PIW_P
#define QT_PIW_P 2
#endif
#ifndef QT_PIW_T
#define QT_PIW_T 128
#endif
constexpr int kWPairs = QT_PIW_P;
constexpr int kWThreads = QT_PIW_T;
constexpr int kWGroups = (kMaxPairs + kWPairs - 1) / kWPairs;   // CTAs per (item, kz)
constexpr int kWE = 2;

template <int NO>
__global__ void __launch_bounds__(kWThreads, 512 / kWThreads) k_pi_w(PiWArgs A) {
  constexpr int NN = NO * NO;
  extern __shared__ __align__(16) double2 w_sm[];
  double2* Hl = w_sm;                          // [kWPairs][3][NN]  ∇_jH_{as}
  double2* Hr = Hl + kWPairs * 3 * NN;         // [kWPairs][3][NN]  ∇_iH_{br}
  double2* Gb = Hr + kWPairs * 3 * NN;         // [2 buffers][kWPairs][kWE][NN]
  double2* T = Gb + 2 * kWPairs * kWE * NN;    // [kWPairs][kWE][3][NN]
  const int half = blockIdx.x % kWGroups;
  const int64_t r = blockIdx.x / kWGroups;
  const int kz = (int)(r % A.Nkz);
  const int64_t item = A.i0 + r / A.Nkz;
  const PiItem it = A.items[item];
  const int t0 = half * kWPairs;
  const int P = min(kWPairs, it.npair - t0);
  if (P <= 0) return;
  for (int idx = threadIdx.x; idx < P * 3 * NN; idx += blockDim.x) {
    const int t = idx / (3 * NN), rem = idx - t * 3 * NN;
    const PiPair pr = A.pairs[it.pair0 + t0 + t];
    Hl[idx] = A.dH[((int64_t)pr.a_in * A.Nb + pr.s) * 3 * NN + rem];
    Hr[idx] = A.dH[((int64_t)pr.b_in * A.Nb + pr.r) * 3 * NN + rem];
  }
  constexpr int XC = 20;                       // = PiCfg::XC
  constexpr int NXC = (NN + XC - 1) / XC;
  const int64_t wblk = ((item - A.i0) * A.Nkz + kz) * (int64_t)NXC * A.NEo * kRows * XC;   // W: energies from E0
  double2* Wdst = A.W + wblk;
  // G_b(kz, e0 .. e0+kWE-1) of the group's pairs: cp.async into one of two buffers, one step ahead
  auto prefetch = [&](int e0, double2* dst) {
    const int ne = min(kWE, A.NEo - e0);
    for (int idx = threadIdx.x; idx < P * ne * NN; idx += blockDim.x) {
      const int t = idx / (ne * NN), rem = idx - t * ne * NN;
      const int b_in = A.pairs[it.pair0 + t0 + t].b_in;
      const int e = rem / NN, uv = rem - e * NN;
      cp_async16(dst + t * kWE * NN + rem, A.GY + (((int64_t)kz * A.NE + A.E0 + e0 + e) * A.Nwin + b_in) * NN + uv, true);
    }
    cp_async_commit();
  };
  prefetch(0, Gb);
  for (int e0 = 0, itr = 0; e0 < A.NEo; e0 += kWE, ++itr) {
    const int ne = min(kWE, A.NEo - e0);
    const double2* Gc = Gb + (itr & 1) * kWPairs * kWE * NN;
    if (e0 + kWE < A.NEo) {
      prefetch(e0 + kWE, Gb + ((itr + 1) & 1) * kWPairs * kWE * NN);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    // T_i(t, e)[q][x] = Σ_p G_b[q][p] ∇_iH_{br}[p][x]
    for (int u = threadIdx.x; u < P * ne * 3 * NO; u += blockDim.x) {
      const int q = u % NO, r1 = u / NO, i = r1 % 3, r2 = r1 / 3, e = r2 % ne, t = r2 / ne;
      double2 g[NO], s[NO];
#pragma unroll
      for (int k = 0; k < NO; ++k) {
        g[k] = Gc[(t * kWE + e) * NN + q * NO + k];
        s[k] = make_double2(0.0, 0.0);
      }
      const double2* h = Hr + (t * 3 + i) * NN;
#pragma unroll
      for (int k = 0; k < NO; ++k)
#pragma unroll
        for (int x = 0; x < NO; ++x) cfma(s[x], g[k], h[k * NO + x]);
      double2* o = T + ((t * kWE + e) * 3 + i) * NN + q * NO;
#pragma unroll
      for (int x = 0; x < NO; ++x) o[x] = s[x];
    }
    __syncthreads();
    // W^{ij}(t, e)[x][y] = Σ_q ∇_jH_{as}[y][q] T_i[q][x]
    for (int u = threadIdx.x; u < P * ne * 9 * NO; u += blockDim.x) {
      const int y = u % NO, r1 = u / NO, ij = r1 % 9, r2 = r1 / 9, e = r2 % ne, t = r2 / ne;
      const int i = ij / 3, j = ij - 3 * i;
      double2 hrow[NO], s[NO];
#pragma unroll
      for (int k = 0; k < NO; ++k) {
        hrow[k] = Hl[(t * 3 + j) * NN + y * NO + k];
        s[k] = make_double2(0.0, 0.0);
      }
      const double2* tt = T + ((t * kWE + e) * 3 + i) * NN;
#pragma unroll
      for (int q = 0; q < NO; ++q)
#pragma unroll
        for (int x = 0; x < NO; ++x) cfma(s[x], hrow[q], tt[q * NO + x]);
      // W layout [xy chunk][E][72 rows][XC]: each Π stage reads one contiguous block
#pragma unroll
      for (int x = 0; x < NO; ++x) {
        const int xy = x * NO + y, xc = xy / XC, c = xy - xc * XC;
        const int64_t o = (((int64_t)xc * A.NEo + e0 + e) * kRows + (t0 + t) * 9 + ij) * XC + c;
        Wdst[o] = s[x];
      }
    }
  }
}

// W sandwich, warp-per-energy form (Norb <= 10): CTA = (pair, kz), warp w owns energies e ≡ w (mod kW2Warps).
// Phase 1, lane (i, q): row q of T_i = G^Y_b(E) ∇_iH_{br} (G_b row from global;
// ∇_iH_{br} broadcast from shared memory) into the warp's T buffer. Phase 2, lane (j, y): row y of
// ∇_jH_{as} held in registers, W^{ij}[x][y] = Σ_q ∇_jH_{as}[y][q] T_i[q][x] for i, x (T broadcast), stored
// straight to the W scratch. Only __syncwarp between the phases; 12·Norb³ complex MACs per (pair, kz, E).
constexpr int kW2Warps = 4;

template <int NO>
__global__ void __launch_bounds__(kW2Warps * 32) k_pi_w2(PiWArgs A) {
  constexpr int NN = NO * NO, NNP = NN + 2;
  constexpr int XC = 20, NXC = (NN + XC - 1) / XC;
  static_assert(3 * NO <= 32, "lanes (i, q) / (j, y)");
  extern __shared__ __align__(16) double2 w2_sm[];
  double2* Hr = w2_sm;                          // [3][NNP]  ∇_iH_{br}
  double2* Tw = Hr + 3 * NNP;                   // [kW2Warps][3][NNP]
  const int kz = (int)(blockIdx.x % A.Nkz);
  const int64_t pg = A.p0 + blockIdx.x / A.Nkz;                 // pair (global index)
  const int64_t item = A.pair_item[pg];
  const PiItem it = A.items[item];
  const PiPair pr = A.pairs[pg];
  const int t = (int)(pg - it.pair0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int idx = threadIdx.x; idx < 3 * NN; idx += blockDim.x) {
    const int i = idx / NN, rc = idx - i * NN;
    Hr[i * NNP + rc] = A.dH[((int64_t)pr.b_in * A.Nb + pr.r) * 3 * NN + idx];
  }
  const bool act = lane < 3 * NO;
  const int hi = min(lane / NO, 2), lo = lane % NO;   // phase 1: (i, q); phase 2: (j, y)
  double2 hl[NO];                                      // row y of ∇_jH_{as}
#pragma unroll
  for (int k = 0; k < NO; ++k) hl[k] = A.dH[((int64_t)pr.a_in * A.Nb + pr.s) * 3 * NN + hi * NN + lo * NO + k];
  __syncthreads();
  double2* T = Tw + warp * 3 * NNP;
  const double2* hr = Hr + hi * NNP;
  double2* Wb = A.W + ((item - A.i0) * A.Nkz + kz) * (int64_t)NXC * A.NEo * kRows * XC;
  // row q = lo of G^Y_b(kz, E0 + e) (latency covered by the other warps: up to 8 CTAs of 4 warps per SM)
  const double2* gsrc = A.GY + (((int64_t)kz * A.NE + A.E0) * A.Nwin + pr.b_in) * NN + lo * NO;
  const int64_t gstep = (int64_t)A.Nwin * NN;   // one energy
  for (int e = warp; e < A.NEo; e += kW2Warps) {
    double2 g[NO];
#pragma unroll
    for (int p = 0; p < NO; ++p) g[p] = __ldg(gsrc + e * gstep + p);
    // phase 1: T_i[q][x] = Σ_p G_b[q][p] ∇_iH_{br}[p][x]
    double2 tr[NO];
#pragma unroll
    for (int x = 0; x < NO; ++x) tr[x] = make_double2(0.0, 0.0);
#pragma unroll
    for (int p = 0; p < NO; ++p)
#pragma unroll
      for (int x = 0; x < NO; ++x) cfma(tr[x], g[p], hr[p * NO + x]);
    if (act) {
#pragma unroll
      for (int x = 0; x < NO; ++x) T[hi * NNP + lo * NO + x] = tr[x];
    }
    __syncwarp();
    // phase 2: W^{ij}[x][y] = Σ_q ∇_jH_{as}[y][q] T_i[q][x]; row (t, i, j), column xy = x·Norb + y
#pragma unroll 1
    for (int i = 0; i < 3; ++i) {
      double2 w[NO], wm[NO];   // split accumulators: four independent FMA chains per complex element
#pragma unroll
      for (int x = 0; x < NO; ++x) w[x] = wm[x] = make_double2(0.0, 0.0);
      const double2* ti = T + i * NNP;
#pragma unroll
      for (int q = 0; q < NO; ++q)
#pragma unroll
        for (int x = 0; x < NO; ++x) {
          const double2 b = ti[q * NO + x];
          w[x].x = fma(hl[q].x, b.x, w[x].x);
          wm[x].x = fma(hl[q].y, b.y, wm[x].x);
          w[x].y = fma(hl[q].x, b.y, w[x].y);
          wm[x].y = fma(hl[q].y, b.x, wm[x].y);
        }
#pragma unroll
      for (int x = 0; x < NO; ++x) {
        w[x].x -= wm[x].x;
        w[x].y += wm[x].y;
      }
      if (act) {
        const int row = t * 9 + i * 3 + hi;
#pragma unroll
        for (int x = 0; x < NO; ++x) {
          const int xy = x * NO + lo, xc = xy / XC, c = xy - xc * XC;
          Wb[(((int64_t)xc * A.NEo + e) * kRows + row) * XC + c] = w[x];
        }
      }
    }
    __syncwarp();   // T is rewritten by the next energy
  }
}

// ---------------------------------------------------------------- Π correlation: TMA / mbarrier pipeline
// Stage = (kz, E0..E0+EC-1, xy0..xy0+XC-1): the W tile [EC][72][XC] (one contiguous 1-D bulk copy) and the G_a window
// rows E0+s_0 .. E0+EC-1+s_{NWP-1} (4-D TMA box; rows >= NE zero-filled: reading R7). Warp 18 produces;
// warps 0..17 consume (warp w: m-fragment w%9 of the rows (t,ij), half of the m-column fragments).
#ifndef QT_PI_EC
#define QT_PI_EC 1
#endif
#ifndef QT_PI_STAGES
#define QT_PI_STAGES 3
#endif
struct PiCfg {
  static constexpr int XC = 20;      // xy per stage: 5 DMMA k-steps; row stride 80 words ≡ 16 (mod 32)
  static constexpr int EC = QT_PI_EC;   // energies per stage
  static constexpr int STAGES = QT_PI_STAGES;   // (two for Nω windows > 88 shifts: PiTma::STAGES)
  static constexpr int W_STAGE = EC * kRows * XC;
  static constexpr int NCONS = 18;
  static constexpr int THREADS = (NCONS + 1) * 32;
};

template <int NFM>
struct PiTma {
  static constexpr int NWP = NFM * 8;
  static constexpr int GROWS = PiCfg::EC + NWP - 1;
  static constexpr int G_STAGE = ((GROWS * PiCfg::XC) + 7) & ~7;       // 128-byte multiple
  static constexpr int GS_STAGE = ((GROWS * PiCfg::XC / 2) + 7) & ~7;  // Re+Im of the G window (doubles)
  static constexpr int STAGE = PiCfg::W_STAGE + G_STAGE + GS_STAGE;
  static constexpr uint32_t STAGE_BYTES = (PiCfg::W_STAGE + GROWS * PiCfg::XC) * 16 + GROWS * PiCfg::XC * 8;
  static constexpr int NF0 = (NFM + 1) / 2, NF1 = NFM / 2;
  // three stages of (W tile + G window + Re+Im) fit up to 11 column fragments (88 shifts); wider windows take two
  static constexpr int STAGES = (size_t)PiCfg::STAGES * STAGE * 16 + 2 * PiCfg::STAGES * 8 + 128 <= 227 * 1024
                                    ? PiCfg::STAGES : 2;
  static constexpr size_t SMEM = (size_t)STAGES * STAGE * 16 + 2 * STAGES * 8 + 128;
  static_assert(SMEM <= 227 * 1024, "shared memory");
};

// Complex k-step over N column fragments with Gauss's 3-multiplication form: per fragment
// T1 += Ar·Br, T2 += Ai·Bi, T3 += (Ar+Ai)(Br+Bi) (three real DMMAs instead of four); the complex
// result is Re = T1 - T2, Im = T3 - T1 - T2 (formed once, in the epilogue). The B-side Re+Im (one per
// fragment) comes precomputed from shared memory; the A-side one (one per k-step, shared by all the
// warp's fragments) is one DADD per 3·N DMMAs, cheaper than storing and streaming a W sum plane.
// Fragment f of the warp is column fragment f0 + f·stride: `fs` = stride·8·XC elements between them.
template <int N>
__device__ __forceinline__ void pi_kstep(C3Acc* acc, double2 a, double as, const double2* gb, const double* sb, int fs) {
#pragma unroll
  for (int f = 0; f < N; ++f) {
    const double2 b = gb[f * fs];
    cmma3s(acc[f], a.x, a.y, as, b.x, b.y, sb[f * fs]);
  }
}

// DMMA work of one stage (EC energies) for one warp owning nfa column fragments f0, f0 + stride, ..
// (nfa <= NFW). rem = NE - E0 - shift0: energy E0+el has in-window columns m < rem - el; column fragments
// without any are skipped.
template <int NFW, int STRIDE = 0>   // STRIDE > 0: compile-time fragment stride (immediate smem offsets)
__device__ __forceinline__ void pi_stage(C3Acc* acc, const double2* ws, const double2* gs,
                                         const double* gss, int rem, int nel, int f0, int stride_rt, int nfa) {
  static_assert(NFW > 0, "empty fragment range");
  using C = PiCfg;
  const int stride = STRIDE > 0 ? STRIDE : stride_rt;
  const int fs = stride * 8 * C::XC;
#pragma unroll
  for (int el = 0; el < C::EC; ++el) {
    const int ncol = el < nel ? (rem - el + 7) >> 3 : 0;         // column fragments with columns < rem - el
    const int nfe = min(nfa, max(0, (ncol - f0 + stride - 1) / stride));
    const double2* w = ws + el * kRows * C::XC;
    const double2* g = gs + el * C::XC;
    const double* gsm = gss + el * C::XC;
    if (nfe == NFW) {
#pragma unroll
      for (int k4 = 0; k4 < C::XC; k4 += 4) {
        const double2 a = w[k4];
        pi_kstep<NFW>(acc, a, a.x + a.y, g + k4, gsm + k4, fs);
      }
    } else if (nfe > 0) {
#pragma unroll
      for (int k4 = 0; k4 < C::XC; k4 += 4) {
        const double2 a = w[k4];
        const double as = a.x + a.y;
#pragma unroll
        for (int f = 0; f < NFW; ++f) {
          if (f < nfe) {
            const double2 b = g[k4 + f * fs];
            cmma3s(acc[f], a.x, a.y, as, b.x, b.y, gsm[k4 + f * fs]);
          }
        }
      }
    }
  }
}

template <int NFM>
__global__ void __launch_bounds__(PiCfg::THREADS, 1)
    k_pi_contract(const __grid_constant__ CUtensorMap tmG, const __grid_constant__ CUtensorMap tmGS, PiCArgs A) {
  using C = PiCfg;
  using T = PiTma<NFM>;
  extern __shared__ uint8_t smem_raw[];
  double2* smem = reinterpret_cast<double2*>(smem_raw + ((-smem_u32(smem_raw)) & 127u));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + T::STAGES * T::STAGE);
  uint64_t* empty = full + T::STAGES;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t blk = blockIdx.x;
  const int qz = (int)(blk % A.Nqz);
  const int il = (int)(blk / A.Nqz);
  const PiItem item = A.items[A.i0 + il];
  const int P = item.npair;
  const int NN = A.NN;
  const int nxc = (NN + C::XC - 1) / C::XC;
  const int e_end = min(A.NEo, A.NE - A.shift0 - A.E0);   // energies E0 + e with an in-window E + s_m (R7)
  const int nec = e_end > 0 ? (e_end + C::EC - 1) / C::EC : 0;
  const int nst = A.Nkz * nxc * nec;

  if (tid == 0) {
    for (int s = 0; s < T::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::NCONS);
    }
    fence_barrier_init();
  }
  __syncthreads();

  // Roles: warp -> (row fragment mi of the item's F = ceil(9P/8) active ones, column fragments f0, f0 + Wp,
  // ..). Full items (F = 9): Wp = 2 warps per row fragment, placed by a role table so the 5-fragment (lower)
  // warps fill sub-partitions 2, 3 and the 4-fragment ones 0, 1 (warp w issues on sub-partition w % 4):
  // DMMA work per sub-partition 21/20/20/20 for NFM = 9. Small items (the remainder of an atom's pairs,
  // e.g. 2 of 34: F = 3) spread the column fragments over Wp = 18 / F warps per row fragment instead of
  // leaving 18 - 2F warps idle: the tile takes ceil(NFM/Wp) fragment-times instead of ceil(NFM/2).
  // Column fragments are interleaved (stride Wp), so the out-of-window cut at large E (R7) removes work
  // from every warp alike.
  constexpr int kPiRole[18] = {8, 10, 0, 1, 9, 12, 2, 3, 11, 14, 4, 5, 13, 16, 6, 7, 15, 17};
  const int Fr = (9 * P + 7) / 8;
  const int Wp = Fr >= 9 ? 2 : C::NCONS / Fr;
  int mi = 0, f0 = 0;
  if (warp < C::NCONS) {
    if (Fr >= 9) {
      const int role = kPiRole[warp];
      mi = role % 9;
      f0 = role >= 9 ? 1 : 0;
    } else {
      mi = warp / Wp;
      f0 = warp - mi * Wp;
    }
  }
  const int nfa = f0 < NFM ? (NFM - f0 + Wp - 1) / Wp : 0;   // column fragments of this warp (<= NF0)
  C3Acc acc[T::NF0];
#pragma unroll
  for (int f = 0; f < T::NF0; ++f) acc[f] = C3Acc{};

  if (warp == C::NCONS) {
    if (lane == 0) {
      prefetch_tmap(&tmG);
      prefetch_tmap(&tmGS);
      int kz = 0, xc = 0, ec = 0;
      for (int st = 0; st < nst; ++st) {
        const int slot = st % T::STAGES;
        if (st >= T::STAGES) mbar_wait(&empty[slot], ((st / T::STAGES) - 1) & 1);
        mbar_arrive_expect_tx(&full[slot], T::STAGE_BYTES);
        double2* ws = smem + slot * T::STAGE;
        const int k2 = (int)imod(kz + qz - A.h, A.Nkz);   // kz + qz (R5)
        const int64_t woff = ((((int64_t)il * A.Nkz + kz) * nxc + xc) * A.NEo + ec * C::EC) * kRows * C::XC;
        bulk_load(ws, A.W + woff, C::W_STAGE * 16, &full[slot]);
        tma_load_4d(ws + C::W_STAGE, &tmG, 2 * xc * C::XC, item.a_in, A.E0 + ec * C::EC + A.shift0, k2, &full[slot]);
        tma_load_4d(ws + C::W_STAGE + T::G_STAGE, &tmGS, xc * C::XC, A.E0 + ec * C::EC + A.shift0, k2, item.a_in,
                    &full[slot]);
        if (++ec == nec) {
          ec = 0;
          if (++xc == nxc) {
            xc = 0;
            ++kz;
          }
        }
      }
    }
  } else {
    const bool active = warp < C::NCONS && mi < Fr && nfa > 0;
    int ec = 0;
    for (int st = 0; st < nst; ++st) {
      const int slot = st % T::STAGES;
      mbar_wait(&full[slot], (st / T::STAGES) & 1);
      if (active) {
        const int aoff = (mi * 8 + (lane >> 2)) * C::XC + (lane & 3);
        const int boff = (f0 * 8 + (lane >> 2)) * C::XC + (lane & 3);
        const double2* st0 = smem + slot * T::STAGE;
        const double2* ws = st0 + aoff;
        const double2* gs = st0 + C::W_STAGE + boff;
        const double* gss = reinterpret_cast<const double*>(st0 + C::W_STAGE + T::G_STAGE) + boff;
        const int rem = A.NE - A.E0 - ec * C::EC - A.shift0;
        const int nel = e_end - ec * C::EC;                     // energies of this stage inside the chunk's range
        // compile-time fragment counts for the common cases (full-speed unrolled path), guarded otherwise
        if (Wp == 2 && nfa == T::NF0) {
          pi_stage<T::NF0, 2>(acc, ws, gs, gss, rem, nel, f0, Wp, nfa);
        } else if (Wp == 2 && nfa == T::NF0 - 1) {
          if constexpr (T::NF0 > 1) pi_stage<(T::NF0 > 1 ? T::NF0 - 1 : 1), 2>(acc, ws, gs, gss, rem, nel, f0, Wp, nfa);
        } else if (nfa == 1) {
          pi_stage<1>(acc, ws, gs, gss, rem, nel, f0, Wp, nfa);
        } else if (nfa == 2) {
          if constexpr (T::NF0 >= 2) pi_stage<2>(acc, ws, gs, gss, rem, nel, f0, Wp, nfa);
        } else if (nfa == 3) {
          if constexpr (T::NF0 >= 3) pi_stage<3>(acc, ws, gs, gss, rem, nel, f0, Wp, nfa);
        } else {
          pi_stage<T::NF0>(acc, ws, gs, gss, rem, nel, f0, Wp, nfa);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
      if (++ec == nec) ec = 0;
    }
    if (active) {
      const int row = mi * 8 + (lane >> 2);
      const int t = row / 9, ij = row - 9 * t;
      if (t < P) {
        const int slot = A.pairs[item.pair0 + t].s + 1;
        const int64_t base = (int64_t)item.a_out * (A.Nb + 1) * 9 + slot * 9 + ij;
#pragma unroll
        for (int f = 0; f < T::NF0; ++f) {
          if (f < nfa) {
            const int c0 = (f0 + Wp * f) * 8 + 2 * (lane & 3);   // shift columns c0, c0 + 1 (shift0 + c)
#pragma unroll
            for (int k = 0; k < 2; ++k) {
              const int c = c0 + k, m = c / A.step;
              if (c < A.NWv && c == m * A.step) {
                double2* o = A.Pi + ((int64_t)qz * A.Nw + m) * A.Nout * (A.Nb + 1) * 9 + base;
                double2 v = cmul(A.scale, acc[f].value(k));
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
    }
  }
}

cudaError_t make_tmap_f64(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
                          const uint32_t* box);

template <int NFM>
static cudaError_t launch_pi_nfm(const PiCArgs& a, cudaStream_t st) {
  using T = PiTma<NFM>;
  cudaError_t ea = cudaFuncSetAttribute(k_pi_contract<NFM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)T::SMEM);
  if (ea != cudaSuccess) return ea;
  const uint64_t NN = (uint64_t)a.NN;
  CUtensorMap tmG, tmGS;
  {
    const uint64_t NS = (NN + 1) & ~1ull;
    const uint64_t dims[4] = {NN, (uint64_t)a.NE, (uint64_t)a.Nkz, (uint64_t)a.Nwin};
    const uint64_t strides[3] = {NS * 8, (uint64_t)a.NE * NS * 8, (uint64_t)a.Nkz * a.NE * NS * 8};
    const uint32_t box[4] = {PiCfg::XC, (uint32_t)T::GROWS, 1, 1};
    cudaError_t e = make_tmap_f64(&tmGS, a.GXsum, 4, dims, strides, box);
    if (e != cudaSuccess) return e;
  }
  {   // G^X window in the paper layout [Nkz][NE][Nwin][NN]: box = the GROWS-energy Hankel window of one atom
    const uint64_t dims[4] = {2 * NN, (uint64_t)a.Nwin, (uint64_t)a.NE, (uint64_t)a.Nkz};
    const uint64_t strides[3] = {NN * 16, (uint64_t)a.Nwin * NN * 16, (uint64_t)a.NE * a.Nwin * NN * 16};
    const uint32_t box[4] = {2 * PiCfg::XC, 1, (uint32_t)T::GROWS, 1};
    cudaError_t e = make_tmap_f64(&tmG, a.GX, 4, dims, strides, box);
    if (e != cudaSuccess) return e;
  }
  const int64_t nblk = a.nitems * a.Nqz;
  if (nblk == 0) return cudaSuccess;
  k_pi_contract<NFM><<<(unsigned)nblk, PiCfg::THREADS, T::SMEM, st>>>(tmG, tmGS, a);
  return cudaGetLastError();
}

cudaError_t launch_pi_contract(const PiCArgs& a, int64_t /*nitems*/, cudaStream_t st) {
  switch (a.NWP / 8) {
    case 1: return launch_pi_nfm<1>(a, st);
    case 2: return launch_pi_nfm<2>(a, st);
    case 3: return launch_pi_nfm<3>(a, st);
    case 4: return launch_pi_nfm<4>(a, st);
    case 5: return launch_pi_nfm<5>(a, st);
    case 6: return launch_pi_nfm<6>(a, st);
    case 7: return launch_pi_nfm<7>(a, st);
    case 8: return launch_pi_nfm<8>(a, st);
    case 9: return launch_pi_nfm<9>(a, st);
    case 10: return launch_pi_nfm<10>(a, st);
    case 11: return launch_pi_nfm<11>(a, st);
    case 12: return launch_pi_nfm<12>(a, st);
    case 13: return launch_pi_nfm<13>(a, st);
    case 14: return launch_pi_nfm<14>(a, st);
    case 15: return launch_pi_nfm<15>(a, st);
    case 16: return launch_pi_nfm<16>(a, st);
    default: return cudaErrorInvalidValue;
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
template <int NO>
static cudaError_t launch_pi_w_no(const PiWArgs& a, int64_t nitems, cudaStream_t st) {
  const int smem = (6 + 2 * kWE + 3 * kWE) * kWPairs * NO * NO * 16;
  cudaError_t e = cudaFuncSetAttribute(k_pi_w<NO>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  k_pi_w<NO><<<(unsigned)(nitems * a.Nkz * kWGroups), kWThreads, smem, st>>>(a);
  return cudaGetLastError();
}

template <int NO>
static cudaError_t launch_pi_w2_no(const PiWArgs& a, cudaStream_t st) {
  const int smem = (1 + kW2Warps) * 3 * (NO * NO + 2) * 16;
  cudaError_t e = cudaFuncSetAttribute(k_pi_w2<NO>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  k_pi_w2<NO><<<(unsigned)(a.npairs * a.Nkz), kW2Warps * 32, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_pi_w(const PiWArgs& a, int64_t nitems_chunk, cudaStream_t st) {
  if (nitems_chunk * a.Nkz == 0) return cudaSuccess;
#ifndef QT_PIW_OLD
  switch (a.Norb) {   // warp-per-energy form
    case 1: return launch_pi_w2_no<1>(a, st);
    case 2: return launch_pi_w2_no<2>(a, st);
    case 3: return launch_pi_w2_no<3>(a, st);
    case 4: return launch_pi_w2_no<4>(a, st);
    case 5: return launch_pi_w2_no<5>(a, st);
    case 6: return launch_pi_w2_no<6>(a, st);
    case 7: return launch_pi_w2_no<7>(a, st);
    case 8: return launch_pi_w2_no<8>(a, st);
    case 9: return launch_pi_w2_no<9>(a, st);
    case 10: return launch_pi_w2_no<10>(a, st);
    default: break;
  }
#endif
  switch (a.Norb) {
    case 1: return launch_pi_w_no<1>(a, nitems_chunk, st);
    case 2: return launch_pi_w_no<2>(a, nitems_chunk, st);
    case 3: return launch_pi_w_no<3>(a, nitems_chunk, st);
    case 4: return launch_pi_w_no<4>(a, nitems_chunk, st);
    case 5: return launch_pi_w_no<5>(a, nitems_chunk, st);
    case 6: return launch_pi_w_no<6>(a, nitems_chunk, st);
    case 7: return launch_pi_w_no<7>(a, nitems_chunk, st);
    case 8: return launch_pi_w_no<8>(a, nitems_chunk, st);
    case 9: return launch_pi_w_no<9>(a, nitems_chunk, st);
    case 10: return launch_pi_w_no<10>(a, nitems_chunk, st);
    case 11: return launch_pi_w_no<11>(a, nitems_chunk, st);
    case 12: return launch_pi_w_no<12>(a, nitems_chunk, st);
    default: return cudaErrorInvalidValue;
  }
}

// one CTA per (window atom, kz): Re + Im of the NE x NN block of G^X (paper layout) into the atom-major sum plane
// (the B-side sum of the Gauss 3M product, so the DMMA consumers need no DADD); atoms a0 + blockIdx / Nkz
__global__ void __launch_bounds__(256) k_relayout(const double2* __restrict__ in, double* __restrict__ osum, int64_t Nkz,
                                                  int64_t NE, int64_t Nwin, int64_t NN, int64_t a0) {
  const int64_t a = a0 + blockIdx.x / Nkz, kz = blockIdx.x % Nkz;
  const int64_t NS = (NN + 1) & ~int64_t(1);   // sum-plane row stride: even, so TMA strides are 16-byte multiples
  double* os = osum + (a * Nkz + kz) * NE * NS;
  const double2* src = in + (kz * NE * Nwin + a) * NN;
  const int64_t n = NE * NN;
  for (int64_t idx = threadIdx.x; idx < n; idx += blockDim.x) {
    const int64_t e = idx / NN, uv = idx - e * NN;
    const double2 v = __ldg(src + e * Nwin * NN + uv);
    os[e * NS + uv] = v.x + v.y;
  }
}

cudaError_t launch_relayout(const double2* in, double* osum, int64_t Nkz, int64_t NE, int64_t Nwin, int64_t NN, int64_t a0,
                            int64_t a1, cudaStream_t st) {
  if (Nkz * (a1 - a0) <= 0) return cudaSuccess;
  k_relayout<<<(unsigned)(Nkz * (a1 - a0)), 256, 0, st>>>(in, osum, Nkz, NE, Nwin, NN, a0);
  return cudaGetLastError();
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
