// kernels_sigma_tma.cu — Σ≷ D-contraction + sandwich (Eq. 3), warp-specialized
// TMA / mbarrier pipeline for sm_100a (Norb <= 12).
//
// Reformulation (exact up to rounding): for a pair p = (a,s), b = nbr[a][s],
//   Gt_p^{ij}(kz,E) = Σ_{q,d} C_p^{ij}(q,d) · G_b(kz-q+h, E+d)              (D-contraction, k_sigma)
//   Σ_a(kz,E)      = scale · Σ_s Σ_i ∇_iH_{as} ( Σ_j Gt_p^{ij} ∇_jH_{br} )     (sandwich + neighbour sum)
// with C_p^{ij}(q,-s_m) = Dc^X_{ij}(q,m), C_p^{ij}(q,+s_m) = Dc^Y_{ji}(q,m), 0 otherwise (R2, R3).
// The contraction is a GEMM with rows (pair t, ij) — the ≤ 8 pairs sharing one source atom b, 72 rows = 9 DMMA
// m-fragments — columns rc (the Norb² entries of G_b) and K = (q, d): the G operand is a Hankel window of G_b
// rows E+d. The kernel is organized so that the FP64 tensor pipe never waits on block-wide barriers:
//   warp 18          : producer. One elected lane issues, per stage, three bulk loads: the G_b rows
//                      E-Dmax+d0 .. +KC straight from the caller's G window in the paper layout (a 4-D box of
//                      one atom x KC energies; TMA zero-fills rows outside [0,NE): reading R7, and the padding
//                      columns Norb²..NPS), the same rows of the Re+Im plane, and the 72 x KCP coefficient tile.
//   warps 0..17      : consumers. Warp w owns m-fragment w%9 and half of the n-fragments; it waits on the
//                      stage's `full` mbarrier, runs DMMA.8x8x4, and releases the stage on `empty`.
// Gt tiles go to the chunk's scratch; the sandwich kernels below add ∇H·Gt·∇H into Σ_a.
#include "kernels_decl.cuh"
#include "tma.cuh"

#include <cudaTypedefs.h>

#include <algorithm>

namespace qt {

// Coefficient tiles for the TMA path: coef[il][q][dc][row = t*9+ij][k], d = 16*dc + k - Dmax (k < 16;
// k = 16..19 and rows t >= P are zero padding). Same values as k_sigma_coef (Eq. 3 four-term
// combination; absorption Dc^X_{ij}, emission Dc^Y_{ji}: readings R2, R3).
__global__ void k_sigma_coef_tiled(CoefArgs A) {
  constexpr int KCP = kCoefKCP;
  const int64_t per_item = A.Nqz * A.ndc * kRows * KCP;
  const int64_t total = A.nitems * per_item;
  const int64_t pp0 = A.items[A.item0].pair0;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(idx % KCP);
    int64_t r = idx / KCP;
    const int row = (int)(r % kRows);
    r /= kRows;
    const int64_t dc = r % A.ndc;
    r /= A.ndc;
    const int64_t q = r % A.Nqz;
    const int64_t il = r / A.Nqz;
    const SigItem item = A.items[A.item0 + il];
    const int t = row / 9, ij = row - 9 * t;
    // slot k < 16: coefficient dd = 16*dc + k; slots 16..23 hold the Re+Im sums of coefficients
    // 2(k-16) and 2(k-16)+1 (Gauss 3M A-side operand); slots 24..27 are padding
    const bool is_sum = QT_SIG_CSUM && k >= 16 && k < 24;
    double2 v = make_double2(0.0, 0.0);
    for (int h = 0; h < (is_sum ? 2 : 1); ++h) {
    const int64_t dd = 16 * dc + (is_sum ? 2 * (k - 16) + h : k);
    double2 c = make_double2(0.0, 0.0);
    if ((k < 16 || is_sum) && t < item.npair && dd < A.Dwin) {
      const int64_t d = dd - A.Dmax, ad = d < 0 ? -d : d;
      if (ad >= A.shift0 && ad <= A.Dmax && (ad - A.shift0) % A.step == 0) {
        const SigPair pr = A.pairs[item.pair0 - pp0 + t];
        const int64_t b = item.b_in, m = (ad - A.shift0) / A.step, ns = A.Nb + 1;
        const double2* D = d < 0 ? A.DX : A.DY;
        const int e = d < 0 ? ij : (ij % 3) * 3 + ij / 3;
        const int64_t base = (q * A.Nw + m) * A.Nwin;
        const double2 dba = D[((base + b) * ns + pr.r + 1) * 9 + e];
        const double2 dbb = D[((base + b) * ns + 0) * 9 + e];
        const double2 daa = D[((base + pr.a_in) * ns + 0) * 9 + e];
        const double2 dab = D[((base + pr.a_in) * ns + pr.s + 1) * 9 + e];
        c.x = ((dba.x - dbb.x) - daa.x) + dab.x;
        c.y = ((dba.y - dbb.y) - daa.y) + dab.y;
      }
    }
    if (is_sum) {
      (h == 0 ? v.x : v.y) = c.x + c.y;
    } else {
      v = c;
    }
    }
    A.coef[idx] = v;
  }
}

cudaError_t launch_sigma_coef_tiled(const CoefArgs& a, cudaStream_t st) {
  const int64_t total = a.nitems * a.Nqz * a.ndc * kRows * kCoefKCP;
  if (total == 0) return cudaSuccess;
  int64_t g = (total + 255) / 256;
  if (g > 148 * 32) g = 148 * 32;
  k_sigma_coef_tiled<<<(int)g, 256, 0, st>>>(a);
  return cudaGetLastError();
}

template <int NF>
struct SigTmaCfg {
  static constexpr int NFH0 = (NF + 1) / 2;  // n-fragments of column half 0
  static constexpr int NFH1 = NF / 2;        // n-fragments of column half 1
  static constexpr int NPS = NFH0 * 8 + 2;   // ≡ 2 (mod 8): conflict-free B-fragment LDS.128
  static constexpr int KC = 16;              // d values per stage (4 DMMA k-steps)
  static constexpr int KCP = kCoefKCP;       // tiled coef row (see kernels_decl.cuh); ≡ 4 (mod 8)
#ifndef QT_SIG_STAGES
#define QT_SIG_STAGES 4
#endif
  // Norb 11, 12 (NF = 16, 18): a stage is 61 KB, three fit next to each other
  static constexpr int STAGES = NF > 13 ? 3 : QT_SIG_STAGES;
  static constexpr int G_STAGE = KC * NPS;   // complex elements
  static constexpr int S_STAGE = (KC * NPS / 2 + 7) & ~7;   // Re+Im plane of the G rows (doubles), complex units
  static constexpr int C_STAGE = kRows * KCP;
  static constexpr int STAGE = G_STAGE + S_STAGE + C_STAGE;
  static constexpr uint32_t STAGE_BYTES = (G_STAGE + C_STAGE) * 16 + KC * NPS * 8;
  static constexpr int PIPE = STAGES * STAGE;
  static constexpr int NCONS = 18;           // consumer warps: (m-fragment, half of the half-tile's n-frags)
  static constexpr int THREADS = (NCONS + 1) * 32;
  static constexpr int TMAXW = (NFH0 + 1) / 2;   // n-fragments per consumer warp (max)
  static constexpr size_t SMEM = (size_t)PIPE * 16 + 2 * STAGES * 8 + 128;
  // Multi-energy stages (items of <= 3 pairs, see sig_ept): G rows for up to kMaxEpt energies (Hankel:
  // energy E+e reads the same rows shifted by e) and a coefficient tile of <= 32 rows.
  static constexpr int GROWS_M = KC + kMaxEpt - 1;
  static constexpr int G_STAGE_M = (GROWS_M * NPS + 7) & ~7;
  static constexpr int S_STAGE_M = ((GROWS_M * NPS + 1) / 2 + 7) & ~7;
  __host__ __device__ static constexpr uint32_t stage_bytes_m(int F) { return GROWS_M * NPS * 24 + F * 8 * KCP * 16; }
  static_assert(G_STAGE_M + S_STAGE_M + 32 * KCP <= STAGE, "multi-energy stage fits");
  static_assert(2 * NPS <= 256, "TMA box width");
  static_assert((G_STAGE * 16) % 128 == 0 && (STAGE * 16) % 128 == 0, "TMA destination alignment");
  static_assert(SMEM <= 227 * 1024, "shared memory");
};

// One stage of DMMA work for a consumer warp with NFW n-fragments (Gauss 3M complex product: three
// real DMMAs per complex 8x8x4 step, see C3Acc).
template <int NFW, int NPS, int KC>
__device__ __forceinline__ void sigma_stage(C3Acc* acc, const double2* gs, const double* ss, const double2* cs, int klo,
                                            int khi) {
  static_assert(NFW > 0, "empty fragment range");
#pragma unroll
  for (int k4 = 0; k4 < KC; k4 += 4) {
    if (k4 >= klo && k4 < khi) {   // k-steps whose 4 shifts all lie outside the tile's energy window are skipped
      const double2 a = cs[k4];
#if QT_SIG_CSUM
      const double as = reinterpret_cast<const double*>(cs - (threadIdx.x & 3))[32 + k4 + (threadIdx.x & 3)];
#else
      const double as = a.x + a.y;
#endif
      const double2* gb = gs + k4 * NPS;
      const double* sb = ss + k4 * NPS;
#pragma unroll
      for (int f = 0; f < NFW; ++f) cmma3s(acc[f], a.x, a.y, as, gb[f * 8].x, gb[f * 8].y, sb[f * 8]);
    }
  }
}

struct SigTile {
  SigItem item;
  int E, kz, ch, il, dc_lo, nchunk, nst, F, ept;
  int lo, hi;   // shifts d (window index) with E + e + d - Dmax in [0, NE) for some energy e < ept of the tile
  bool skip;
};

template <int KC>
__device__ __forceinline__ SigTile sig_tile(const SigmaArgs& A, int64_t t) {
  SigTile T;
  // Column half alternates between a CTA's consecutive tiles (the two halves differ in work; with an
  // even grid, ch = t & 1 would give every CTA the same half for the whole launch).
  T.ch = (int)((t ^ (t / gridDim.x)) & 1);
  t >>= 1;
  T.E = A.E0 + (int)(t % A.NEo);              // output energy (window coordinates)
  T.kz = (int)((t / A.NEo) % A.Nkz);
  T.il = (int)(t / ((int64_t)A.NEo * A.Nkz));
  T.item = A.items[T.il];
  // An item of n pairs fills F = ceil(9n/8) of the 9 m-fragments; small items process ept = 9/F
  // consecutive energies per tile (tiles with E % ept != 0 are empty), one energy per group of F.
  T.F = (9 * T.item.npair + 7) / 8;
  T.ept = min(kMaxEpt, 9 / T.F);
  T.skip = ((T.E - A.E0) % T.ept) != 0;
  // K range: shifts d = 16*dc + k - Dmax with E+e+d in [0,NE) for some e < ept (R7), in whole 16-shift
  // chunks (rows outside the window are zero-filled by TMA; shifts beyond the table are zero coefficients).
  T.lo = max(0, A.Dmax - (T.E + T.ept - 1));
  T.hi = min(A.Dwin, A.Dmax - T.E + A.NE);
  T.dc_lo = T.lo / KC;
  const int dc_hi = (T.hi + KC - 1) / KC;
  T.nchunk = dc_hi - T.dc_lo;
  T.nst = T.skip ? 0 : A.Nqz * T.nchunk;
  return T;
}

// Persistent: CTA c processes tiles c, c + gridDim.x, ... with tile = (item, kz, E, column half).
// The producer streams stages across tile boundaries; consumers store each finished tile of Gt
// (complex, from the 3M accumulators) to the chunk's scratch [item][kz][E][72][Norb²].
template <int NF>
__global__ void __launch_bounds__(SigTmaCfg<NF>::THREADS, 1)
    k_sigma(const __grid_constant__ CUtensorMap tmG, const __grid_constant__ CUtensorMap tmS,
            const __grid_constant__ CUtensorMap tmGm, const __grid_constant__ CUtensorMap tmSm, SigmaArgs A) {
  using C = SigTmaCfg<NF>;
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
    // ---------------- producer
    if (lane == 0) {
      prefetch_tmap(&tmG);
      prefetch_tmap(&tmS);
      prefetch_tmap(&tmGm);
      prefetch_tmap(&tmSm);
      uint32_t g = 0;
      for (int64_t t = blockIdx.x; t < A.ntiles; t += gridDim.x) {
        const SigTile T = sig_tile<C::KC>(A, t);
        int q = 0, c = 0;
        for (int st = 0; st < T.nst; ++st, ++g) {
          const uint32_t slot = g % C::STAGES;
          if (g >= C::STAGES) mbar_wait(&empty[slot], ((g / C::STAGES) - 1) & 1);
          const bool multi = T.ept > 1;
          mbar_arrive_expect_tx(&full[slot], multi ? C::stage_bytes_m(T.F) : C::STAGE_BYTES);
          const int dc = T.dc_lo + c;
          const int kp = (int)imod(T.kz - q + A.h, A.Nkz);          // kz - qz (R4, R5)
          double2* gs = smem + slot * C::STAGE;
          const int soff = multi ? C::G_STAGE_M : C::G_STAGE;
          const int coff = soff + (multi ? C::S_STAGE_M : C::S_STAGE);
          const int r0 = T.E - A.Dmax + dc * C::KC;
          tma_load_4d(gs, multi ? &tmGm : &tmG, T.ch * C::NFH0 * 16, T.item.b_in, r0, kp, &full[slot]);
          tma_load_4d(gs + soff, multi ? &tmSm : &tmS, T.ch * C::NFH0 * 8, r0, kp, T.item.b_in, &full[slot]);
          bulk_load(gs + coff, A.coef + (((int64_t)T.il * A.Nqz + q) * A.ndc + dc) * C::C_STAGE,
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

  // ---------------- consumers: warp -> role (m-fragment mi, part q of the half-tile's n-fragments).
  // Warp w issues on sub-partition w % 4; sub-partitions 0, 1 hold 5 consumer warps, 2, 3 hold 4. The
  // role tables balance the DMMA work per sub-partition (the slowest one paces the CTA's pipeline):
  //  kRoleA, split (ceil, floor): all 9 q=1 warps (fewer fragments) on the 5-warp sub-partitions,
  //          e.g. Norb=10 half 0 (4+3 fragments) -> 15/16/16/16;
  //  kRoleB, split (n/2+1, n/2-1) for an even fragment count n: 3+3+1+2 q=1 warps,
  //          e.g. Norb=10 half 1 (4+2 fragments) -> 14/14/14/12 instead of 15/15/12/12.
  constexpr int kRoleA[18] = {9, 14, 1, 5, 10, 15, 2, 6, 11, 16, 3, 7, 12, 17, 4, 8, 13, 0};
  constexpr int kRoleB[18] = {9, 12, 15, 16, 10, 13, 4, 17, 11, 14, 5, 7, 0, 2, 6, 8, 1, 3};
  const int roleA = kRoleA[warp], roleB = kRoleB[warp];
  uint32_t g = 0;
  for (int64_t t = blockIdx.x; t < A.ntiles; t += gridDim.x) {
    const SigTile T = sig_tile<C::KC>(A, t);
    if (T.skip) continue;
    const int nfh = T.ch ? C::NFH1 : C::NFH0;
    const bool split_b = (nfh % 2 == 0) && nfh / 2 + 1 == C::TMAXW;
    const int role = split_b ? roleB : roleA;
    const int mi = role % 9, q = role / 9;
    const int n0 = split_b ? nfh / 2 + 1 : (nfh + 1) / 2;
    const int nfw = q ? nfh - n0 : n0;
    const int f0 = q ? n0 : 0;
    const int e = mi / T.F, ml = mi - e * T.F;      // energy E+e, m-fragment ml of the item's rows
    const int row = ml * 8 + (lane >> 2);
    const bool active = e < T.ept && T.E - A.E0 + e < A.NEo && nfw > 0;
    const bool multi = T.ept > 1;
    const int soff = multi ? C::G_STAGE_M : C::G_STAGE;
    const int coff = soff + (multi ? C::S_STAGE_M : C::S_STAGE);
    C3Acc acc[C::TMAXW];
#pragma unroll
    for (int f = 0; f < C::TMAXW; ++f) acc[f] = C3Acc{};
    int c = 0;
    for (int st = 0; st < T.nst; ++st, ++g) {
      const uint32_t slot = g % C::STAGES;
      mbar_wait(&full[slot], (g / C::STAGES) & 1);
      if (active) {
        // k-step range of this chunk: shifts 16·dc + k in [lo, hi), in whole DMMA k-steps of 4
        const int d0 = (T.dc_lo + c) * C::KC;
        const int klo = max(0, T.lo - d0) & ~3, khi = min(C::KC, T.hi - d0);
        const int boff = ((lane & 3) + e) * C::NPS + (lane >> 2) + f0 * 8;
        const double2* gs = smem + slot * C::STAGE + boff;
        const double* ss = reinterpret_cast<const double*>(smem + slot * C::STAGE + soff) + boff;
        const double2* cs = smem + slot * C::STAGE + coff + row * C::KCP + (lane & 3);
        if (nfw == C::TMAXW) {
          sigma_stage<C::TMAXW, C::NPS, C::KC>(acc, gs, ss, cs, klo, khi);
        } else if (nfw == C::TMAXW - 1) {
          if constexpr (C::TMAXW > 1) sigma_stage<C::TMAXW - 1, C::NPS, C::KC>(acc, gs, ss, cs, klo, khi);
        } else {
          if constexpr (C::TMAXW > 2) sigma_stage<C::TMAXW - 2, C::NPS, C::KC>(acc, gs, ss, cs, klo, khi);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
      if (++c == T.nchunk) c = 0;
    }
    if (active && row < 9 * T.item.npair) {
      double2* out = A.Gt + ((((int64_t)T.il * A.Nkz + T.kz) * A.NEo + T.E - A.E0 + e) * A.rows + row) * A.gt_ld;
#pragma unroll
      for (int f = 0; f < C::TMAXW; ++f) {
        if (f < nfw) {
          const int col = (T.ch * C::NFH0 + f0 + f) * 8 + 2 * (lane & 3);
          if (col < A.NN) out[col] = acc[f].value(0);
          if (col + 1 < A.NN) out[col + 1] = acc[f].value(1);
        }
      }
    }
  }
}

// ---------------------------------------------------------------- Σ sandwich + neighbour sum
// Σ_a(kz,E) += scale · Σ_{i,j} ∇_iH_{as} Gt^{ij} ∇_jH_{br} for every pair of the chunk (Eq. 3 outer products, R8),
// associated as S = Σ_j U^j ∇_jH_{br} with U^j = Σ_i ∇_iH_{as} Gt^{ij} (12·Norb³ complex MACs per (pair, kz, E)).
// CTA = (pair, kz): one producer warp streams the pair's 9 Gt rows of each energy from the scratch into a ring of
// shared-memory slots (9 bulk copies per energy, padded row stride: conflict-free broadcasts; mbarrier
// full/empty per slot; the ring is deeper than the consumer warps, so the next energies are in flight while
// every warp computes); each consumer warp owns whole energies: lane (j, x) = (lane / Norb, lane % Norb) forms
// row x of U^j (Norb² · 3 MACs) and of S_j = U^j ∇_jH_{br} (Norb² MACs) in registers, the three S_j rows are
// summed with two shuffles and the j = 0 lanes add scale·S into Σ_a with RED.F64 (other CTAs hold the atom's
// other pairs). No block-wide barrier after the ∇H load, no intermediate in shared memory.
#ifndef QT_SAND_W
#define QT_SAND_W 12
#endif
#ifndef QT_SAND_SPLIT
#define QT_SAND_SPLIT 1
#endif
#ifndef QT_SAND_S
#define QT_SAND_S 14
#endif
#ifndef QT_SAND_PF
#define QT_SAND_PF 0
#endif
#ifndef QT_SAND_KU
#define QT_SAND_KU 2
#endif
constexpr int kSandKU = QT_SAND_KU;   // unroll of the sandwich's k loop (loads of the next k in flight)
// FP32 Gt (the mixed mode): half the bytes per slot, so the ring can be deeper
#ifndef QT_SAND_WF
#define QT_SAND_WF 12
#endif
#ifndef QT_SAND_SF
#define QT_SAND_SF 14
#endif

template <int NO, class R>
struct SandCfg {
  using C2 = typename Cx<R>::T;
  static constexpr bool F32 = sizeof(R) == 4;
  static constexpr int NN = NO * NO;
  static constexpr int NNE = (int)(((size_t)NN * sizeof(C2) + 15) / 16 * 16 / sizeof(C2));   // row, 16-byte multiple
  static constexpr int NNP = NNE + 16 / (int)sizeof(C2);   // padded slot row: j = 0,1,2 rows on distinct banks
  static constexpr uint32_t ROWB = (uint32_t)(NNE * sizeof(C2));   // bytes copied per row (the scratch's gt_ld)
  static constexpr int SLOT = 9 * NNP;         // C2 per slot (rows (i,j) of one energy)
  static constexpr int HSZ = 3 * NNP;          // C2 per ∇H triple
  static constexpr int WARPS = F32 ? QT_SAND_WF : QT_SAND_W;   // consumer warps per CTA (energies e ≡ w mod WARPS)
  // Gt ring: SLOTS - WARPS energies prefetched (the FP32 ring as deep as 220 KB allows, up to QT_SAND_SF)
  static constexpr int SLOTS_FIT = (int)((220 * 1024 - 2 * HSZ * sizeof(C2)) / (SLOT * sizeof(C2) + 16));
  static constexpr int SLOTS = F32 ? (QT_SAND_SF < SLOTS_FIT ? QT_SAND_SF : SLOTS_FIT) : QT_SAND_S;
  static_assert(SLOTS > WARPS, "ring deeper than the consumer warps");
  static constexpr size_t SMEM = ((size_t)SLOTS * SLOT + 2 * HSZ) * sizeof(C2) + 2 * SLOTS * 8;
  static_assert(SMEM <= 227 * 1024, "shared memory");
  static_assert(3 * NO <= 32, "lanes (j, x)");
};

template <int NO, class R>
__global__ void __launch_bounds__((SandCfg<NO, R>::WARPS + 1) * 32) k_sigma_sand(SigmaArgs A) {
  using Cf = SandCfg<NO, R>;
  constexpr int kSandWarps = Cf::WARPS, kSandSlots = Cf::SLOTS;
  using C2 = typename Cf::C2;
  constexpr int NN = Cf::NN, NNP = Cf::NNP;
  extern __shared__ __align__(128) double2 sand_raw[];
  C2* ring = reinterpret_cast<C2*>(sand_raw);   // pointer casts only: the loads stay LDS (no generic addressing)
  C2* Hl = ring + kSandSlots * Cf::SLOT;   // [3][NNP]  ∇_iH_{as}
  C2* Hr = Hl + Cf::HSZ;                   // [3][NNP]  ∇_jH_{br}
  uint64_t* full = reinterpret_cast<uint64_t*>(Hr + Cf::HSZ);
  uint64_t* empty = full + kSandSlots;
  const int kz = (int)(blockIdx.x % A.Nkz);
  const int64_t pg = A.cp0 + blockIdx.x / A.Nkz;   // pair (global index)
  const int il = A.pair_item[pg] - (int)A.item0;    // chunk-relative item
  const SigItem item = A.items[il];
  const SigPair pr = A.pairs[pg];
  const int t = (int)(pg - item.pair0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kSandSlots; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_barrier_init();
  }
  for (int idx = threadIdx.x; idx < 3 * NN; idx += blockDim.x) {
    const int i = idx / NN, rc = idx - i * NN;
    Hl[i * NNP + rc] = Cx<R>::from(A.dH[((int64_t)pr.a_in * A.Nb + pr.s) * 3 * NN + idx]);
    Hr[i * NNP + rc] = Cx<R>::from(A.dH[((int64_t)item.b_in * A.Nb + pr.r) * 3 * NN + idx]);
  }
  __syncthreads();
  const int ld = A.gt_ld;   // Gt row stride: 16-byte multiple (bulk copies)
  const C2* gsrc = reinterpret_cast<const C2*>(A.Gt) + ((int64_t)il * A.Nkz + kz) * A.NEo * A.rows * ld + t * 9 * ld;
  if (warp == kSandWarps) {
    // ---------------- producer: energy e -> slot e % kSandSlots
    if (lane == 0) {
      for (int e = 0; e < A.NEo; ++e) {
        const int slot = e % kSandSlots;
        if (e >= kSandSlots) mbar_wait(&empty[slot], ((e / kSandSlots) - 1) & 1);
        const C2* src = gsrc + (int64_t)e * A.rows * ld;
        if (QT_SAND_PF > 0 && e + QT_SAND_PF < A.NEo)   // the pair's 9 rows are contiguous: one L2 prefetch
          bulk_prefetch_l2(src + (int64_t)QT_SAND_PF * A.rows * ld, 9 * ld * (uint32_t)sizeof(C2));
        if (ld == NNP) {   // scratch rows already padded like the slot: one copy (the per-copy cost dominates)
          mbar_arrive_expect_tx(&full[slot], 9 * NNP * (uint32_t)sizeof(C2));
          bulk_load(ring + slot * Cf::SLOT, src, 9 * NNP * (uint32_t)sizeof(C2), &full[slot]);
        } else {
          mbar_arrive_expect_tx(&full[slot], 9 * Cf::ROWB);
          for (int r = 0; r < 9; ++r)
            bulk_load(ring + slot * Cf::SLOT + r * NNP, src + r * ld, Cf::ROWB, &full[slot]);
        }
      }
    }
    return;
  }
  // ---------------- consumers
  const int j = min(lane / NO, 2), x = lane % NO;
  const bool act = lane < 3 * NO;
  const C2* hr = Hr + j * NNP;
  for (int e = warp; e < A.NEo; e += kSandWarps) {
    const int slot = e % kSandSlots;
    mbar_wait(&full[slot], (e / kSandSlots) & 1);
    const C2* g = ring + slot * Cf::SLOT;
    C2 u[NO];
#pragma unroll
    for (int v = 0; v < NO; ++v) u[v] = Cx<R>::zero();
#if QT_SAND_SPLIT
    // split accumulators: u = (Σ hr·gr − Σ hi·gi, Σ hr·gi + Σ hi·gr) with the four real sums in independent
    // FMA chains (the two FMAs of one complex MAC no longer depend on each other)
    C2 um[NO];
#pragma unroll
    for (int v = 0; v < NO; ++v) um[v] = Cx<R>::zero();
#endif
#pragma unroll 1
    for (int i = 0; i < 3; ++i) {   // (i, k) loops rolled: keeps the kernel inside the instruction cache
      const C2* gr = g + (i * 3 + j) * NNP;
      const C2* hl = Hl + i * NNP + x * NO;
#pragma unroll kSandKU
      for (int k = 0; k < NO; ++k) {
        const C2 h = hl[k];
#pragma unroll
        for (int v = 0; v < NO; ++v) {
#if QT_SAND_SPLIT
          const C2 b = gr[k * NO + v];
          u[v].x = fma(h.x, b.x, u[v].x);
          um[v].x = fma(h.y, b.y, um[v].x);
          u[v].y = fma(h.x, b.y, u[v].y);
          um[v].y = fma(h.y, b.x, um[v].y);
#else
          cfma(u[v], h, gr[k * NO + v]);
#endif
        }
      }
    }
#if QT_SAND_SPLIT
#pragma unroll
    for (int v = 0; v < NO; ++v) {
      u[v].x -= um[v].x;
      u[v].y += um[v].y;
    }
#endif
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);   // the slot's rows are in registers now
    C2 sv[NO];
#pragma unroll
    for (int y = 0; y < NO; ++y) sv[y] = Cx<R>::zero();
#pragma unroll
    for (int v = 0; v < NO; ++v)
#pragma unroll
      for (int y = 0; y < NO; ++y) cfma(sv[y], u[v], hr[v * NO + y]);
    // S = S_0 + S_1 + S_2: lanes (1, x) and (2, x) -> lane (0, x)
#pragma unroll
    for (int y = 0; y < NO; ++y) {
      double2 w = Cx<R>::wide(sv[y]);
      if (!act) w = make_double2(0.0, 0.0);
      const double ax = __shfl_down_sync(0xffffffffu, w.x, NO), ay = __shfl_down_sync(0xffffffffu, w.y, NO);
      const double bx = __shfl_down_sync(0xffffffffu, w.x, 2 * NO), by = __shfl_down_sync(0xffffffffu, w.y, 2 * NO);
      if (lane < NO) {
        const double2 tot = make_double2((w.x + ax) + bx, (w.y + ay) + by);
        const double2 rr = cmul(A.scale, tot);
        double* out = reinterpret_cast<double*>(A.Sig + (((int64_t)kz * A.NEs + A.Es0 + e) * A.Nout + pr.a) * NN + x * NO + y);
        atomicAdd(out, rr.x);
        atomicAdd(out + 1, rr.y);
      }
    }
  }
}

// ---------------------------------------------------------------- deterministic Σ sandwich (QT_FLAG_DETERMINISTIC)
// Destination-organized: one CTA per (destination atom with pairs in the chunk, kz) runs the sandwich of each of
// the atom's pairs in a fixed order and adds scale·S into Σ_a with plain loads and stores (each Σ element is
// updated by the same thread for every pair, and chunks run in a fixed order), so the neighbour sum of Eq. 3
// has one summation order and Σ is bitwise reproducible — no floating-point atomics.
constexpr int kSandThreads = 128;
constexpr int kSandE = 2;   // energies per iteration
constexpr int kSandY = 5;   // S columns per thread

template <int NO, class R>
__global__ void __launch_bounds__(kSandThreads) k_sigma_sand_det(SigmaArgs A) {
  using C2 = typename Cx<R>::T;
  constexpr int NN = NO * NO;
  extern __shared__ __align__(16) double2 det_raw[];
  C2* sm = reinterpret_cast<C2*>(det_raw);
  C2* Hr = sm;                  // [3][NN]  ∇_jH_{br}
  C2* Hl = Hr + 3 * NN;         // [3][NN]  ∇_iH_{as}
  C2* Vs = Hl + 3 * NN;         // [kSandE][3][NN]
  const int kz = (int)(blockIdx.x % A.Nkz);
  const int4 ent = A.det_atoms[blockIdx.x / A.Nkz];
  constexpr int NYG = (NO + kSandY - 1) / kSandY;
  for (int q = 0; q < ent.z; ++q) {
    const int2 pi = A.det_pairs[ent.y + q];
    const SigItem item = A.items[pi.x];
    const SigPair pr = A.pairs[item.pair0 + pi.y];
    __syncthreads();   // the previous pair's V and H are no longer read
    for (int idx = threadIdx.x; idx < 3 * NN; idx += blockDim.x) {
      Hr[idx] = Cx<R>::from(A.dH[((int64_t)item.b_in * A.Nb + pr.r) * 3 * NN + idx]);
      Hl[idx] = Cx<R>::from(A.dH[((int64_t)pr.a_in * A.Nb + pr.s) * 3 * NN + idx]);
    }
    const C2* gbase = reinterpret_cast<const C2*>(A.Gt) + ((int64_t)pi.x * A.Nkz + kz) * A.NEo * A.rows * A.gt_ld;
    for (int e0 = 0; e0 < A.NEo; e0 += kSandE) {
      __syncthreads();
      for (int u = threadIdx.x; u < kSandE * 3 * NO; u += blockDim.x) {   // V rows (e, i, x)
        const int x = u % NO, r1 = u / NO, i = r1 % 3, e = r1 / 3;
        if (e0 + e >= A.NEo) continue;
        C2 s[NO];
#pragma unroll
        for (int y = 0; y < NO; ++y) s[y] = Cx<R>::zero();
        const C2* g = gbase + ((int64_t)(e0 + e) * A.rows + pi.y * 9 + i * 3) * A.gt_ld + x * NO;
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          C2 gv[NO];
#pragma unroll
          for (int v = 0; v < NO; ++v) gv[v] = g[j * A.gt_ld + v];
          const C2* hr = Hr + j * NN;
#pragma unroll
          for (int v = 0; v < NO; ++v)
#pragma unroll
            for (int y = 0; y < NO; ++y) cfma(s[y], gv[v], hr[v * NO + y]);
        }
        C2* vo = Vs + (e * 3 + i) * NN + x * NO;
#pragma unroll
        for (int y = 0; y < NO; ++y) vo[y] = s[y];
      }
      __syncthreads();
      for (int u = threadIdx.x; u < kSandE * NO * NYG; u += blockDim.x) {   // S units (e, x, y group)
        const int yg = u % NYG, r0 = u / NYG, x = r0 % NO, e = r0 / NO;
        if (e0 + e >= A.NEo) continue;
        const int y0 = yg * kSandY;
        C2 s[kSandY];
#pragma unroll
        for (int y = 0; y < kSandY; ++y) s[y] = Cx<R>::zero();
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          const C2* hl = Hl + i * NN + x * NO;
          const C2* v = Vs + (e * 3 + i) * NN + y0;
#pragma unroll
          for (int k = 0; k < NO; ++k) {
            const C2 h = hl[k];
#pragma unroll
            for (int y = 0; y < kSandY; ++y)
              if (y0 + y < NO) cfma(s[y], h, v[k * NO + y]);
          }
        }
        double2* out = A.Sig + (((int64_t)kz * A.NEs + A.Es0 + e0 + e) * A.Nout + ent.x) * NN + x * NO + y0;
#pragma unroll
        for (int y = 0; y < kSandY; ++y) {
          if (y0 + y < NO) {
            const double2 rr = cmul(A.scale, Cx<R>::wide(s[y]));
            double2 o = out[y];
            o.x += rr.x;
            o.y += rr.y;
            out[y] = o;
          }
        }
      }
    }
  }
}

template <int NO, class R>
static cudaError_t launch_sand_det_nr(const SigmaArgs& a, cudaStream_t st) {
  const int smem = (2 + kSandE) * 3 * NO * NO * (int)sizeof(typename Cx<R>::T);
  cudaError_t e = cudaFuncSetAttribute(k_sigma_sand_det<NO, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  k_sigma_sand_det<NO, R><<<(unsigned)(a.n_det * a.Nkz), kSandThreads, smem, st>>>(a);
  return cudaGetLastError();
}
template <int NO>
static cudaError_t launch_sand_det_no(const SigmaArgs& a, cudaStream_t st) {
  return a.gt_f32 ? launch_sand_det_nr<NO, float>(a, st) : launch_sand_det_nr<NO, double>(a, st);
}

cudaError_t launch_sigma_sand_det(const SigmaArgs& a, cudaStream_t st) {
  if (a.n_det * a.Nkz == 0) return cudaSuccess;
  switch (a.Norb) {
    case 1: return launch_sand_det_no<1>(a, st);
    case 2: return launch_sand_det_no<2>(a, st);
    case 3: return launch_sand_det_no<3>(a, st);
    case 4: return launch_sand_det_no<4>(a, st);
    case 5: return launch_sand_det_no<5>(a, st);
    case 6: return launch_sand_det_no<6>(a, st);
    case 7: return launch_sand_det_no<7>(a, st);
    case 8: return launch_sand_det_no<8>(a, st);
    case 9: return launch_sand_det_no<9>(a, st);
    case 10: return launch_sand_det_no<10>(a, st);
    case 11: return launch_sand_det_no<11>(a, st);
    case 12: return launch_sand_det_no<12>(a, st);
    default: return cudaErrorInvalidValue;
  }
}

// ---------------------------------------------------------------- host: tensor maps + launch
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// FP64 tiled map of rank 1..5; dims/box innermost first, strides in bytes for dims 1..rank-1.
cudaError_t make_tmap_f64(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
                          const uint32_t* box) {
  auto fn = encode_fn();
  if (!fn) return cudaErrorNotSupported;
  const uint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, (cuuint32_t)rank, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int NF>
static cudaError_t launch_sigma_tma_nf(const SigmaArgs& a, int64_t nitems, cudaStream_t st) {
  using C = SigTmaCfg<NF>;
  // function attributes are per device context: set on every launch (cheap) instead of once per process
  cudaError_t ea = cudaFuncSetAttribute(k_sigma<NF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
  if (ea != cudaSuccess) return ea;
  CUtensorMap tmG, tmS, tmGm, tmSm;
  const uint64_t NN = (uint64_t)a.NN;
  for (int m = 0; m < 2; ++m) {
    const uint32_t rows = m ? C::GROWS_M : C::KC;
    {   // G^X window in the paper layout [Nkz][NE][Nwin][NN]: box = KC (or GROWS) energies of one atom
      const uint64_t dims[4] = {2 * NN, (uint64_t)a.Nwin, (uint64_t)a.NE, (uint64_t)a.Nkz};
      const uint64_t strides[3] = {NN * 16, (uint64_t)a.Nwin * NN * 16, (uint64_t)a.NE * a.Nwin * NN * 16};
      const uint32_t box[4] = {2 * C::NPS, 1, rows, 1};
      cudaError_t e = make_tmap_f64(m ? &tmGm : &tmG, a.G, 4, dims, strides, box);
      if (e != cudaSuccess) return e;
    }
    {
      const uint64_t NS = (NN + 1) & ~1ull;   // even row stride of the Re+Im plane
      const uint64_t dims[4] = {NN, (uint64_t)a.NE, (uint64_t)a.Nkz, (uint64_t)a.Nwin};
      const uint64_t strides[3] = {NS * 8, (uint64_t)a.NE * NS * 8, (uint64_t)a.Nkz * a.NE * NS * 8};
      const uint32_t box[4] = {C::NPS, rows, 1, 1};
      cudaError_t e = make_tmap_f64(m ? &tmSm : &tmS, a.Gsum, 4, dims, strides, box);
      if (e != cudaSuccess) return e;
    }
  }
  SigmaArgs b = a;
  b.ntiles = nitems * a.NEo * a.Nkz * 2;
  if (b.ntiles == 0) return cudaSuccess;
  int dev = 0, nsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int64_t grid = std::min<int64_t>(b.ntiles, nsm) & ~int64_t(1);   // even: sig_tile pairs t = 2u, 2u+1 in one round
  k_sigma<NF><<<(unsigned)grid, C::THREADS, C::SMEM, st>>>(tmG, tmS, tmGm, tmSm, b);
  return cudaGetLastError();
}

template <int NO, class R>
static cudaError_t launch_sand_nr(const SigmaArgs& a, int64_t /*nitems*/, cudaStream_t st) {
  using Cf = SandCfg<NO, R>;
  cudaError_t e = cudaFuncSetAttribute(k_sigma_sand<NO, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cf::SMEM);
  if (e != cudaSuccess) return e;
  k_sigma_sand<NO, R><<<(unsigned)(a.npairs_chunk * a.Nkz), (Cf::WARPS + 1) * 32, Cf::SMEM, st>>>(a);
  return cudaGetLastError();
}
// FP64 Gt scratch (72-row items) or, in the FP32 mixed mode (128-row items), FP32 Gt and an FP32 sandwich
template <int NO>
static cudaError_t launch_sand_no(const SigmaArgs& a, int64_t nitems, cudaStream_t st) {
  return a.gt_f32 ? launch_sand_nr<NO, float>(a, nitems, st) : launch_sand_nr<NO, double>(a, nitems, st);
}

cudaError_t launch_sigma_sand(const SigmaArgs& a, int64_t nitems, cudaStream_t st) {
  if (nitems * a.Nkz == 0) return cudaSuccess;
  switch (a.Norb) {
    case 1: return launch_sand_no<1>(a, nitems, st);
    case 2: return launch_sand_no<2>(a, nitems, st);
    case 3: return launch_sand_no<3>(a, nitems, st);
    case 4: return launch_sand_no<4>(a, nitems, st);
    case 5: return launch_sand_no<5>(a, nitems, st);
    case 6: return launch_sand_no<6>(a, nitems, st);
    case 7: return launch_sand_no<7>(a, nitems, st);
    case 8: return launch_sand_no<8>(a, nitems, st);
    case 9: return launch_sand_no<9>(a, nitems, st);
    case 10: return launch_sand_no<10>(a, nitems, st);
    default: return cudaErrorInvalidValue;   // Norb 11, 12 (3·Norb > 32 lanes): the destination-ordered kernel
  }
}

cudaError_t launch_sigma(const SigmaArgs& a, int64_t nitems, cudaStream_t st) {
  switch ((a.NN + 7) / 8) {
    case 1: return launch_sigma_tma_nf<1>(a, nitems, st);
    case 2: return launch_sigma_tma_nf<2>(a, nitems, st);
    case 4: return launch_sigma_tma_nf<4>(a, nitems, st);
    case 5: return launch_sigma_tma_nf<5>(a, nitems, st);
    case 7: return launch_sigma_tma_nf<7>(a, nitems, st);
    case 8: return launch_sigma_tma_nf<8>(a, nitems, st);
    case 11: return launch_sigma_tma_nf<11>(a, nitems, st);
    case 13: return launch_sigma_tma_nf<13>(a, nitems, st);
    case 16: return launch_sigma_tma_nf<16>(a, nitems, st);   // Norb 11
    case 18: return launch_sigma_tma_nf<18>(a, nitems, st);   // Norb 12 (the paper's FinFET basis)
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace qt
