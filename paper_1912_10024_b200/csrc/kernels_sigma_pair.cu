// kernels_sigma_pair.cu — the Σ D-contraction of k_sigma (Eq. 3) with TWO energies per tile
// for items of >= 4 pairs and Norb 9..11, where Norb² is not a multiple of 8.
//
// k_sigma's GEMM has N = Norb² columns per energy, rounded up to DMMA n-fragments of 8 (100 -> 104 for Norb 10).
// Consecutive energies E, E+1 share the coefficient tile and the Hankel G rows (energy E+1 reads the same rows
// shifted by one), so their columns can be flattened into one GEMM of 2·Norb² columns: column c = 2·rc + e is
// entry rc of G_b(E + e + d), i.e. shared-memory row k + e. 200 columns are 25 fragments (no padding for Norb 10);
// each thread's accumulator pair (c, c + 1) is (rc, E) and (rc, E + 1). A tile is (item, kz, energy pair,
// column quarter); each quarter's columns come from one TMA box of KC + 1 rows x its rc range. Everything
// else — producer warp, 18 consumer warps, Gauss-3M DMMA, 4-stage mbarrier ring, role tables, k-step trimming
// to the energy window (R7), Gt scratch layout — is k_sigma's.
//
// Items of 1..3 pairs fill only F = ceil(9n/8) = 2..4 of the 9 m-fragments; like k_sigma's multi-energy tiles
// they take ept = 9/F consecutive energy PAIRS per tile (m-fragment group g = mi / F serves energies E + 2g and
// E + 2g + 1: shared-memory rows k + 2g + e of one taller TMA box of KC + 2·ept − 1 rows; tiles of the other
// energy pairs are empty), so every item of a chunk runs here and k_sigma is not launched in pair mode.
#include "kernels_decl.cuh"
#include "tma.cuh"

#include <cudaTypedefs.h>

#include <algorithm>

namespace qt {

cudaError_t make_tmap_f64(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
                          const uint32_t* box);

template <int NN>
struct SigPairCfg {
  static constexpr int NFP = (2 * NN + 7) / 8;        // column fragments of an energy pair
  static constexpr int QMAX = (NFP + 3) / 4;          // fragments of the widest quarter
  static constexpr int RQ = 4 * QMAX;                 // rc per quarter (max)
  static constexpr int NPSG = RQ + 1 + ((RQ + 1) % 2 == 0 ? 1 : 0);   // odd complex row stride: conflict-free B loads
  static constexpr int NPSS = ((RQ + 2) + 7) / 8 * 8 + 2;             // ≡ 2 (mod 8) doubles: Re+Im row stride
  static constexpr int KC = 16;
  static constexpr int ROWS = KC + 1;                 // G rows per stage: energy E + 1 reads one row further
  static constexpr int KCP = kCoefKCP;
#ifndef QT_PAIR_STAGES
#define QT_PAIR_STAGES 4
#endif
  static constexpr int STAGES = QT_PAIR_STAGES;
  static constexpr int EPT_MAX = 4;                  // energy pairs per tile for items of 1 pair (F = 2)
  static constexpr int ROWS_M = KC + 2 * EPT_MAX - 1; // G rows per stage of a multi-energy-pair tile
  static constexpr int G_STAGE = (ROWS_M * NPSG + 7) & ~7;            // complex (room for the taller box)
  static constexpr int S_STAGE = ((ROWS_M * NPSS + 1) / 2 + 7) & ~7;  // complex units of the double plane
  static constexpr int C_STAGE = kRows * KCP;
  static constexpr int STAGE = G_STAGE + S_STAGE + C_STAGE;
  static constexpr uint32_t STAGE_BYTES = ROWS * NPSG * 16 + ROWS * NPSS * 8 + C_STAGE * 16;
  __host__ __device__ static constexpr uint32_t stage_bytes_m(int F) {
    return ROWS_M * NPSG * 16 + ROWS_M * NPSS * 8 + F * 8 * KCP * 16;
  }
  static constexpr int PIPE = STAGES * STAGE;
  static constexpr int NCONS = 18;
  static constexpr int THREADS = (NCONS + 1) * 32;
  static constexpr int TMAXW = (QMAX + 1) / 2;
  static constexpr size_t SMEM = (size_t)PIPE * 16 + 2 * STAGES * 8 + 128;
  static_assert((NPSG * 16) % 16 == 0 && (NPSS * 8) % 16 == 0, "TMA box rows are 16-byte multiples");
  static_assert(2 * NPSG <= 256 && NPSS <= 256, "TMA box width");
  static_assert(SMEM <= 227 * 1024, "shared memory");
  __host__ __device__ static constexpr int qfrags(int q) { return NFP / 4 + (q < NFP % 4 ? 1 : 0); }
  __host__ __device__ static constexpr int qfirst(int q) { return q * (NFP / 4) + min(q, NFP % 4); }
};

template <int NFW, int NPSG, int KC>
__device__ __forceinline__ void sigma_pair_stage(C3Acc* acc, const double2* gs, const double* ss, const double2* cs, int klo,
                                                 int khi, int ssrow) {
#pragma unroll
  for (int k4 = 0; k4 < KC; k4 += 4) {
    if (k4 >= klo && k4 < khi) {
      const double2 a = cs[k4];
      const double as = reinterpret_cast<const double*>(cs - (threadIdx.x & 3))[32 + k4 + (threadIdx.x & 3)];
      const double2* gb = gs + k4 * NPSG;
      const double* sb = ss + k4 * ssrow;
#pragma unroll
      for (int f = 0; f < NFW; ++f) cmma3s(acc[f], a.x, a.y, as, gb[f * 4].x, gb[f * 4].y, sb[f * 4]);
    }
  }
}

struct PairTile {
  SigItem item;
  int E, kz, Q, il, dc_lo, nchunk, nst, lo, hi, F, ept;
  bool skip;   // energy pair served by its group's first tile
};

template <int KC>
__device__ __forceinline__ PairTile pair_tile(const SigmaArgs& A, int64_t t) {
  PairTile T;
  const int NP = (A.NEo + 1) / 2;
  T.Q = (int)((t + t / gridDim.x) & 3);   // the quarter rotates between a CTA's rounds (quarters differ in work)
  t >>= 2;
  T.E = A.E0 + 2 * (int)(t % NP);
  T.kz = (int)((t / NP) % A.Nkz);
  T.il = (int)(t / ((int64_t)NP * A.Nkz));
  T.item = A.items[T.il];
  // items of n <= 3 pairs: F = ceil(9n/8) m-fragments, ept = 9/F energy pairs per tile (tiles of the other
  // energy pairs of the group are empty)
  T.F = (9 * T.item.npair + 7) / 8;
  T.ept = T.item.npair >= 4 ? 1 : 9 / T.F;
  T.skip = ((T.E - A.E0) / 2) % T.ept != 0;
  T.lo = max(0, A.Dmax - (T.E + 2 * T.ept - 1));   // union of the windows of E .. E + 2·ept − 1 (R7)
  T.hi = min(A.Dwin, A.Dmax - T.E + A.NE);
  T.dc_lo = T.lo / KC;
  T.nchunk = (T.hi + KC - 1) / KC - T.dc_lo;
  T.nst = T.skip ? 0 : A.Nqz * T.nchunk;
  return T;
}

template <int NN>
__global__ void __launch_bounds__(SigPairCfg<NN>::THREADS, 1)
    k_sigma_pair(const __grid_constant__ CUtensorMap tmG, const __grid_constant__ CUtensorMap tmS,
                 const __grid_constant__ CUtensorMap tmGm, const __grid_constant__ CUtensorMap tmSm, SigmaArgs A) {
  using C = SigPairCfg<NN>;
  extern __shared__ uint8_t smem_raw[];
  double2* smem = reinterpret_cast<double2*>(smem_raw + ((-smem_u32(smem_raw)) & 127u));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::PIPE);
  uint64_t* empty = full + C::STAGES;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::NCONS);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == C::NCONS) {
    // ---------------- producer: G rows E-Dmax+16dc .. +16 (one box per quarter), their Re+Im, the coefficient tile
    if (lane == 0) {
      prefetch_tmap(&tmG);
      prefetch_tmap(&tmS);
      prefetch_tmap(&tmGm);
      prefetch_tmap(&tmSm);
      uint32_t g = 0;
      for (int64_t t = blockIdx.x; t < A.ntiles; t += gridDim.x) {
        const PairTile T = pair_tile<C::KC>(A, t);
        const int rq0 = 4 * C::qfirst(T.Q);
        int q = 0, c = 0;
        for (int st = 0; st < T.nst; ++st, ++g) {
          const uint32_t slot = g % C::STAGES;
          if (g >= C::STAGES) mbar_wait(&empty[slot], ((g / C::STAGES) - 1) & 1);
          const bool multi = T.ept > 1;
          mbar_arrive_expect_tx(&full[slot], multi ? C::stage_bytes_m(T.F) : C::STAGE_BYTES);
          const int dc = T.dc_lo + c;
          const int kp = (int)imod(T.kz - q + A.h, A.Nkz);          // kz - qz (R4, R5)
          double2* gs = smem + slot * C::STAGE;
          const int r0 = T.E - A.Dmax + dc * C::KC;
          tma_load_4d(gs, multi ? &tmGm : &tmG, 2 * rq0, T.item.b_in, r0, kp, &full[slot]);
          tma_load_4d(gs + C::G_STAGE, multi ? &tmSm : &tmS, rq0, r0, kp, T.item.b_in, &full[slot]);
          bulk_load(gs + C::G_STAGE + C::S_STAGE, A.coef + (((int64_t)T.il * A.Nqz + q) * A.ndc + dc) * C::C_STAGE,
                    (multi ? T.F * 8 : kRows) * C::KCP * 16, &full[slot]);
          if (++c == T.nchunk) {
            c = 0;
            ++q;
          }
        }
      }
    }
    return;
  }

  // ---------------- consumers: roles as in k_sigma (see its comment)
  constexpr int kRoleA[18] = {9, 14, 1, 5, 10, 15, 2, 6, 11, 16, 3, 7, 12, 17, 4, 8, 13, 0};
  constexpr int kRoleB[18] = {9, 12, 15, 16, 10, 13, 4, 17, 11, 14, 5, 7, 0, 2, 6, 8, 1, 3};
  const int roleA = kRoleA[warp], roleB = kRoleB[warp];
  uint32_t g = 0;
  for (int64_t t = blockIdx.x; t < A.ntiles; t += gridDim.x) {
    const PairTile T = pair_tile<C::KC>(A, t);
    if (T.skip) continue;   // (no stages, and its energies' Gt is written by the group's first tile)
    const int nfq = C::qfrags(T.Q), fq0 = C::qfirst(T.Q);
    const bool split_b = (nfq % 2 == 0) && nfq / 2 + 1 == C::TMAXW;
    const int role = split_b ? roleB : roleA;
    const int mi = role % 9, qq = role / 9;
    const int n0 = split_b ? nfq / 2 + 1 : (nfq + 1) / 2;
    const int nfw = qq ? nfq - n0 : n0;
    const int f0 = qq ? n0 : 0;
    const int eg = mi / T.F, ml = mi - eg * T.F;     // energy pair E + 2·eg, m-fragment ml of the item's rows
    const int row = ml * 8 + (lane >> 2);
    const bool active = eg < T.ept && T.E + 2 * eg - A.E0 < A.NEo && ml * 8 < 9 * T.item.npair && nfw > 0;
    // this lane's B element: column 8·f + (lane>>2) -> rc offset 4·f + (lane>>3), energy e = (lane>>2) & 1
    const int n = lane >> 2, e = n & 1;
    const int boffg = ((lane & 3) + e + 2 * eg) * C::NPSG + (n >> 1) + 4 * f0;
    const int boffs = ((lane & 3) + e + 2 * eg) * C::NPSS + (n >> 1) + 4 * f0;
    C3Acc acc[C::TMAXW];
#pragma unroll
    for (int f = 0; f < C::TMAXW; ++f) acc[f] = C3Acc{};
    int c = 0;
    for (int st = 0; st < T.nst; ++st, ++g) {
      const uint32_t slot = g % C::STAGES;
      mbar_wait(&full[slot], (g / C::STAGES) & 1);
      if (active) {
        const int d0 = (T.dc_lo + c) * C::KC;
        const int klo = max(0, T.lo - d0) & ~3, khi = min(C::KC, T.hi - d0);
        const double2* gs = smem + slot * C::STAGE + boffg;
        const double* ss = reinterpret_cast<const double*>(smem + slot * C::STAGE + C::G_STAGE) + boffs;
        const double2* cs = smem + slot * C::STAGE + C::G_STAGE + C::S_STAGE + row * C::KCP + (lane & 3);
        if (nfw == C::TMAXW) {
          sigma_pair_stage<C::TMAXW, C::NPSG, C::KC>(acc, gs, ss, cs, klo, khi, C::NPSS);
        } else if (nfw == C::TMAXW - 1) {
          if constexpr (C::TMAXW > 1) sigma_pair_stage<C::TMAXW - 1, C::NPSG, C::KC>(acc, gs, ss, cs, klo, khi, C::NPSS);
        } else {
          if constexpr (C::TMAXW > 2) sigma_pair_stage<C::TMAXW - 2, C::NPSG, C::KC>(acc, gs, ss, cs, klo, khi, C::NPSS);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
      if (++c == T.nchunk) c = 0;
    }
    if (active && row < 9 * T.item.npair) {
      // accumulator pair = columns 2·rc + {0, 1} = (rc, E) and (rc, E + 1)
      const int Eg = T.E + 2 * eg;
      double2* out0 = A.Gt + ((((int64_t)T.il * A.Nkz + T.kz) * A.NEo + Eg - A.E0) * A.rows + row) * A.gt_ld;
      const bool second = Eg + 1 - A.E0 < A.NEo;
      double2* out1 = out0 + (int64_t)A.rows * A.gt_ld;
#pragma unroll
      for (int f = 0; f < C::TMAXW; ++f) {
        if (f < nfw) {
          const int rc = 4 * (fq0 + f0 + f) + (lane & 3);
          if (rc < NN) {
            out0[rc] = acc[f].value(0);
            if (second) out1[rc] = acc[f].value(1);
          }
        }
      }
    }
  }
}

template <int NN>
static cudaError_t launch_sigma_pair_nn(const SigmaArgs& a, int64_t nitems, cudaStream_t st) {
  using C = SigPairCfg<NN>;
  cudaError_t ea = cudaFuncSetAttribute(k_sigma_pair<NN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
  if (ea != cudaSuccess) return ea;
  CUtensorMap tmG, tmS, tmGm, tmSm;
  for (int m = 0; m < 2; ++m) {
    const uint32_t rows = m ? C::ROWS_M : C::ROWS;
    {   // G^X window in the paper layout [Nkz][NE][Nwin][NN]: box = `rows` energies of one atom, one quarter's rc range
      const uint64_t dims[4] = {2ull * NN, (uint64_t)a.Nwin, (uint64_t)a.NE, (uint64_t)a.Nkz};
      const uint64_t strides[3] = {(uint64_t)NN * 16, (uint64_t)a.Nwin * NN * 16, (uint64_t)a.NE * a.Nwin * NN * 16};
      const uint32_t box[4] = {2 * C::NPSG, 1, rows, 1};
      cudaError_t e = make_tmap_f64(m ? &tmGm : &tmG, a.G, 4, dims, strides, box);
      if (e != cudaSuccess) return e;
    }
    {
      const uint64_t NS = (NN + 1) & ~1ull;
      const uint64_t dims[4] = {(uint64_t)NN, (uint64_t)a.NE, (uint64_t)a.Nkz, (uint64_t)a.Nwin};
      const uint64_t strides[3] = {NS * 8, (uint64_t)a.NE * NS * 8, (uint64_t)a.Nkz * a.NE * NS * 8};
      const uint32_t box[4] = {C::NPSS, rows, 1, 1};
      cudaError_t e = make_tmap_f64(m ? &tmSm : &tmS, a.Gsum, 4, dims, strides, box);
      if (e != cudaSuccess) return e;
    }
  }
  SigmaArgs b = a;
  b.ntiles = nitems * ((a.NEo + 1) / 2) * a.Nkz * 4;
  if (b.ntiles == 0) return cudaSuccess;
  int dev = 0, nsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int64_t grid = std::min<int64_t>(b.ntiles, nsm);
  k_sigma_pair<NN><<<(unsigned)grid, C::THREADS, C::SMEM, st>>>(tmG, tmS, tmGm, tmSm, b);
  return cudaGetLastError();
}

bool sigma_pair_supported(int Norb) { return Norb >= 9 && Norb <= 11; }

cudaError_t launch_sigma_pair(const SigmaArgs& a, int64_t nitems, cudaStream_t st) {
  switch (a.Norb) {
    case 9: return launch_sigma_pair_nn<81>(a, nitems, st);
    case 10: return launch_sigma_pair_nn<100>(a, nitems, st);
    case 11: return launch_sigma_pair_nn<121>(a, nitems, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace qt
