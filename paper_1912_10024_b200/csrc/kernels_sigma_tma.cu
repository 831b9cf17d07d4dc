// kernels_sigma_tma.cu — Σ≷ D-contraction + sandwich (Eq. 3), warp-specialized
// TMA / mbarrier pipeline for sm_100a (Norb <= 10).
//
// Same GEMM as kernels_sigma.cu (rows (pair t, ij): 72 = 9 DMMA m-fragments; columns rc = Norb²;
// K = (q, d) with a Hankel G_b operand), reorganized so that the FP64 tensor pipe never waits on
// block-wide barriers or address arithmetic:
//   warp 18          : producer. One elected lane issues, per stage, two cp.async.bulk.tensor loads:
//                      the G_b rows E-Dmax+d0 .. +KC from the atom-major copy of G (one contiguous block;
//                      TMA zero-fills rows outside [0,NE): reading R7,
//                      and the padding columns Norb²..NPS) and the 72 x KCP coefficient tile.
//   warps 0..17      : consumers. Warp w owns m-fragment w%9 and half of the n-fragments; it waits on the
//                      stage's `full` mbarrier, runs DMMA.8x8x4, and releases the stage on `empty`.
// Epilogue (all warps): Gt -> smem, V^i = Σ_j Gt^{ij} ∇_jH_{br}, S = Σ_i ∇_iH_{as} V^i, Σ_a += scale·S.
#include "kernels_decl.cuh"
#include "tma.cuh"

#include <cudaTypedefs.h>

namespace qt {

template <int NF>
struct SigTmaCfg {
  static constexpr int NP = 8 * NF;
  static constexpr int NPS = NP + 2;        // ≡ 2 (mod 8): conflict-free B-fragment LDS.128
  static constexpr int KC = 16;             // d values per stage (4 DMMA k-steps)
  static constexpr int KCP = 20;            // ≡ 4 (mod 8): conflict-free A-fragment LDS.128
  static constexpr int STAGES = 4;
  static constexpr int G_STAGE = KC * NPS;  // complex elements
  static constexpr int C_STAGE = kRows * KCP;
  static constexpr int STAGE = G_STAGE + C_STAGE;
  static constexpr uint32_t STAGE_BYTES = STAGE * 16;
  static constexpr int PIPE = STAGES * STAGE;
  static constexpr int GT = kRows * NPS;
  static constexpr int VS = kMaxPairs * 3 * NP;
  static constexpr int HR = kMaxPairs * 3 * NP;
  static constexpr int EPI = GT + VS + HR;
  static constexpr int REGION = PIPE > EPI ? PIPE : EPI;
  static constexpr int NCONS = 18;          // consumer warps
  static constexpr int THREADS = (NCONS + 1) * 32;
  static constexpr int NF0 = (NF + 1) / 2;  // n-fragments of warps 0..8
  static constexpr int NF1 = NF / 2;        // n-fragments of warps 9..17
  static constexpr size_t SMEM = (size_t)REGION * 16 + 2 * STAGES * 8 + kMaxPairs * sizeof(SigPair) + 128;
  static_assert(2 * NPS <= 256, "TMA box width");
  static_assert((G_STAGE * 16) % 128 == 0 && (STAGE * 16) % 128 == 0, "TMA destination alignment");
};

// One stage of DMMA work for a warp: NFW n-fragments, kc/4 k-steps. Complex product on split
// accumulators, ordered so the two DMMAs that update the same accumulator are never adjacent and only
// two B fragments are live: (re·re, re·im) for fragment f, then (-im·im, im·re) for fragment f-1.
template <int NFW, int NPS, int KC>
__device__ __forceinline__ void sigma_stage(CAcc* acc, const double2* gs, const double2* cs, int kc) {
  static_assert(NFW > 0, "empty fragment range");
#pragma unroll
  for (int k4 = 0; k4 < KC; k4 += 4) {
    if (k4 < kc) {
      const double2 a = cs[k4];
      const double2* gb = gs + k4 * NPS;
      double2 bp = gb[0];
      dmma(acc[0].r0, acc[0].r1, a.x, bp.x);
      dmma(acc[0].i0, acc[0].i1, a.x, bp.y);
#pragma unroll
      for (int f = 1; f < NFW; ++f) {
        const double2 b = gb[f * 8];
        dmma(acc[f].r0, acc[f].r1, a.x, b.x);
        dmma(acc[f].i0, acc[f].i1, a.x, b.y);
        dmma(acc[f - 1].r0, acc[f - 1].r1, -a.y, bp.y);
        dmma(acc[f - 1].i0, acc[f - 1].i1, a.y, bp.x);
        bp = b;
      }
      dmma(acc[NFW - 1].r0, acc[NFW - 1].r1, -a.y, bp.y);
      dmma(acc[NFW - 1].i0, acc[NFW - 1].i1, a.y, bp.x);
    }
  }
}

template <int NF>
__global__ void __launch_bounds__(SigTmaCfg<NF>::THREADS, 1)
    k_sigma(const __grid_constant__ CUtensorMap tmG, const __grid_constant__ CUtensorMap tmC, SigmaArgs A) {
  using C = SigTmaCfg<NF>;
  extern __shared__ uint8_t smem_raw[];
  double2* smem = reinterpret_cast<double2*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::REGION);
  uint64_t* empty = full + C::STAGES;
  SigPair* pairs_s = reinterpret_cast<SigPair*>(empty + C::STAGES);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t blk = blockIdx.x;
  const int E = (int)(blk % A.NE);
  const int kz = (int)((blk / A.NE) % A.Nkz);
  const SigItem item = A.items[blk / ((int64_t)A.NE * A.Nkz)];
  const int P = item.npair;

  // K range: d with E+d in [0,NE) (R7), rounded to the k=4 step; chunks of KC per q.
  int dd_lo = max(0, A.Dmax - E), dd_hi = min(A.Dwin, A.Dmax - E + A.NE);
  dd_lo &= ~3;
  dd_hi = (dd_hi + 3) & ~3;
  const int nchunk = (dd_hi - dd_lo + C::KC - 1) / C::KC;
  const int nst = A.Nqz * nchunk;

  if (tid == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::NCONS);
    }
    fence_barrier_init();
  }
  if (tid < P) pairs_s[tid] = A.pairs[item.pair0 + tid];
  __syncthreads();

  // Warp -> (m-fragment, n-half). Warp w runs on SM sub-partition w % 4; the 6-fragment halves go to
  // the sub-partitions with 5 consumer warps and the 7-fragment halves to those with 4, so the DMMA
  // counts per sub-partition are 30/31/28/28 (vs 33/32/26/26 for the naive w%9, w/9 split).
  constexpr int kRole[18] = {9, 14, 1, 5, 10, 15, 2, 6, 11, 16, 3, 7, 12, 17, 4, 8, 13, 0};
  const int role = warp < C::NCONS ? kRole[warp] : 0;
  const int mi = role % 9;
  const bool upper = role >= 9;
  const int f0 = upper ? C::NF0 : 0;
  CAcc acc[C::NF0];
#pragma unroll
  for (int f = 0; f < C::NF0; ++f) acc[f] = CAcc{0.0, 0.0, 0.0, 0.0};

  if (warp == C::NCONS) {
    // ---------------- producer
    if (lane == 0) {
      prefetch_tmap(&tmG);
      prefetch_tmap(&tmC);
      int q = 0, c = 0;
      for (int st = 0; st < nst; ++st) {
        const int slot = st & (C::STAGES - 1);
        if (st >= C::STAGES) mbar_wait(&empty[slot], ((st / C::STAGES) - 1) & 1);
        static_assert((C::STAGES & (C::STAGES - 1)) == 0, "power-of-two stage count");
        mbar_arrive_expect_tx(&full[slot], C::STAGE_BYTES);
        const int dd0 = dd_lo + c * C::KC;
        const int kp = (int)imod(kz - q + A.h, A.Nkz);          // kz - qz (R4, R5)
        double2* gs = smem + slot * C::STAGE;
        tma_load_4d(gs, &tmG, 0, E - A.Dmax + dd0, kp, item.b_in, &full[slot]);
        tma_load_4d(gs + C::G_STAGE, &tmC, 2 * dd0, q, 0, (int)(item.pair0 - A.cp0), &full[slot]);
        if (++c == nchunk) {
          c = 0;
          ++q;
        }
      }
    }
  } else {
    // ---------------- consumers
    const bool active = mi * 8 < 9 * P;
    int c = 0;
    for (int st = 0; st < nst; ++st) {
      const int slot = st & (C::STAGES - 1);
      mbar_wait(&full[slot], (st / C::STAGES) & 1);
      if (active) {
        const int kc = min(C::KC, dd_hi - (dd_lo + c * C::KC));
        const double2* gs = smem + slot * C::STAGE + (lane & 3) * C::NPS + (lane >> 2) + f0 * 8;
        const double2* cs = smem + slot * C::STAGE + C::G_STAGE + (mi * 8 + (lane >> 2)) * C::KCP + (lane & 3);
        if (upper) {
          if constexpr (C::NF1 > 0) sigma_stage<C::NF1, C::NPS, C::KC>(acc, gs, cs, kc);
        } else {
          sigma_stage<C::NF0, C::NPS, C::KC>(acc, gs, cs, kc);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
      if (++c == nchunk) c = 0;
    }
  }
  __syncthreads();   // every stage consumed; the pipeline buffers are free

  // ---- epilogue 1: Gt (72 x NP) -> shared memory; ∇_jH_{b r_t} -> shared memory
  double2* Gt = smem;
  double2* Vs = smem + C::GT;
  double2* Hr = Vs + C::VS;
  const int NN = A.NN, No = A.Norb;
  if (warp < C::NCONS && mi * 8 < 9 * P) {
    const int row = mi * 8 + (lane >> 2);
    const int nfw = upper ? C::NF1 : C::NF0;
#pragma unroll
    for (int f = 0; f < C::NF0; ++f) {
      if (f < nfw) {
        const int col = (f0 + f) * 8 + 2 * (lane & 3);
        Gt[row * C::NPS + col] = make_double2(acc[f].r0, acc[f].i0);
        Gt[row * C::NPS + col + 1] = make_double2(acc[f].r1, acc[f].i1);
      }
    }
  }
  for (int idx = tid; idx < P * 3 * NN; idx += C::THREADS) {
    const int t = idx / (3 * NN), rem = idx - t * 3 * NN;
    Hr[t * 3 * C::NP + rem] = A.dH[((int64_t)item.b_in * A.Nb + pairs_s[t].r) * 3 * NN + rem];
  }
  __syncthreads();

  // Register-blocked sandwich: each thread owns a 2 x YB output block (rows x, x+1; columns y0..y0+YB-1).
  constexpr int YB = 5;
  const int nxb = (No + 1) >> 1, nyb = (No + YB - 1) / YB;
  // ---- epilogue 2: V^i_t = Σ_j Gt^{ij}_t · ∇_jH_{b r_t}
  for (int idx = tid; idx < P * 3 * nxb * nyb; idx += C::THREADS) {
    const int yb = idx % nyb, r1 = idx / nyb, xb = r1 % nxb, ti = r1 / nxb;   // ti = t*3 + i
    const int t = ti / 3, i = ti - 3 * t, x0 = 2 * xb, y0 = yb * YB;
    double2 s[2][YB];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int w = 0; w < YB; ++w) s[u][w] = make_double2(0.0, 0.0);
    for (int j = 0; j < 3; ++j) {
      const double2* g0 = Gt + (t * 9 + i * 3 + j) * C::NPS + x0 * No;
      const double2* hr = Hr + t * 3 * C::NP + j * NN + y0;
      for (int v = 0; v < No; ++v) {
        const double2 ga = g0[v], gb = (x0 + 1 < No) ? g0[No + v] : make_double2(0.0, 0.0);
#pragma unroll
        for (int w = 0; w < YB; ++w) {
          const double2 h = (y0 + w < No) ? hr[v * No + w] : make_double2(0.0, 0.0);
          cfma(s[0][w], ga, h);
          cfma(s[1][w], gb, h);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int w = 0; w < YB; ++w)
        if (x0 + u < No && y0 + w < No) Vs[ti * C::NP + (x0 + u) * No + y0 + w] = s[u][w];
  }
  __syncthreads();
  // ∇_iH_{a_t s_t} -> shared memory (reuses the Gt region)
  double2* Hl = smem;
  for (int idx = tid; idx < P * 3 * NN; idx += C::THREADS) {
    const int t = idx / (3 * NN), rem = idx - t * 3 * NN;
    const SigPair pr = pairs_s[t];
    Hl[t * 3 * C::NP + rem] = A.dH[((int64_t)pr.a_in * A.Nb + pr.s) * 3 * NN + rem];
  }
  __syncthreads();

  // ---- epilogue 3: S_t = Σ_i ∇_iH_{a_t s_t} · V^i_t; Σ_a += scale · S_t (R8)
  for (int idx = tid; idx < P * nxb * nyb; idx += C::THREADS) {
    const int yb = idx % nyb, r1 = idx / nyb, xb = r1 % nxb, t = r1 / nxb;
    const int x0 = 2 * xb, y0 = yb * YB;
    double2 s[2][YB];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int w = 0; w < YB; ++w) s[u][w] = make_double2(0.0, 0.0);
    for (int i = 0; i < 3; ++i) {
      const double2* hl = Hl + t * 3 * C::NP + i * NN + x0 * No;
      const double2* v = Vs + (t * 3 + i) * C::NP + y0;
      for (int u = 0; u < No; ++u) {
        const double2 ha = hl[u], hb = (x0 + 1 < No) ? hl[No + u] : make_double2(0.0, 0.0);
#pragma unroll
        for (int w = 0; w < YB; ++w) {
          const double2 vv = (y0 + w < No) ? v[u * No + w] : make_double2(0.0, 0.0);
          cfma(s[0][w], ha, vv);
          cfma(s[1][w], hb, vv);
        }
      }
    }
    const SigPair pr = pairs_s[t];
    double2* out = A.Sig + (((int64_t)kz * A.NE + E) * A.Nout + pr.a) * NN;
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int w = 0; w < YB; ++w)
        if (x0 + u < No && y0 + w < No) {
          const double2 r = cmul(A.scale, s[u][w]);
          double* dst = reinterpret_cast<double*>(out + (x0 + u) * No + y0 + w);
          atomicAdd(dst, r.x);
          atomicAdd(dst + 1, r.y);
        }
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
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_sigma<NF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  CUtensorMap tmG, tmC;
  const uint64_t NN = (uint64_t)a.NN;
  {
    const uint64_t dims[4] = {2 * NN, (uint64_t)a.NE, (uint64_t)a.Nkz, (uint64_t)a.Nwin};
    const uint64_t strides[3] = {NN * 16, (uint64_t)a.NE * NN * 16, (uint64_t)a.Nkz * a.NE * NN * 16};
    const uint32_t box[4] = {2 * C::NPS, C::KC, 1, 1};
    cudaError_t e = make_tmap_f64(&tmG, a.Gam, 4, dims, strides, box);
    if (e != cudaSuccess) return e;
  }
  {
    const uint64_t D = (uint64_t)a.DWp;
    const uint64_t dims[4] = {2 * D, (uint64_t)a.Nqz, 9, (uint64_t)a.npairs_chunk};
    const uint64_t strides[3] = {D * 16, (uint64_t)a.Nqz * D * 16, 9ull * a.Nqz * D * 16};
    const uint32_t box[4] = {2 * C::KCP, 1, 9, kMaxPairs};
    cudaError_t e = make_tmap_f64(&tmC, a.coef, 4, dims, strides, box);
    if (e != cudaSuccess) return e;
  }
  const int64_t nblk = nitems * a.NE * a.Nkz;
  if (nblk == 0) return cudaSuccess;
  if (nblk > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  k_sigma<NF><<<(unsigned)nblk, C::THREADS, C::SMEM, st>>>(tmG, tmC, a);
  return cudaGetLastError();
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
    default: return launch_sigma_cp(a, nitems, st);   // Norb 11, 12
  }
}

}  // namespace qt
