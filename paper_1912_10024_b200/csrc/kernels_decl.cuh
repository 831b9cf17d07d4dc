// kernels_decl.cuh — launcher declarations (definitions in kernels_sigma_tma.cu, kernels_sigma_tc.cu, kernels_pi.cu,
// kernels_pi_tc.cu).
#pragma once
#include "common.cuh"

namespace qt {

struct CoefArgs {
  const double2* DX;
  const double2* DY;
  const SigPair* pairs;
  const SigItem* items;
  const int32_t* pair_item;
  double2* coef;
  int64_t npairs, Nw, Nwin, Nb, Nqz, DWp;
  int Dmax, shift0, step;   // shifts s_m = shift0 + m·step; other |d| in the window get zero coefficients
  // tiled layout (TMA path): [item - item0][q][dc][72 rows (t,ij)][kCoefKCP], d = 16*dc + k - Dmax
  bool tiled;
  int64_t item0, nitems, ndc, Dwin;
};

// Tiled Σ coefficient row (k_sigma_coef_tiled -> k_sigma): 16 coefficients, then (QT_SIG_CSUM) their
// Re+Im sums in 8 complex slots, then padding to a row length ≡ 4 (mod 8) complex (conflict-free A loads).
#ifndef QT_SIG_CSUM
#define QT_SIG_CSUM 1
#endif
constexpr int kCoefKCP = QT_SIG_CSUM ? 28 : 20;

struct SigmaArgs {
  const double2* G;      // G^X window, paper layout [Nkz][NE][Nwin][NN] (TMA boxes read it in place)
  const double* Gsum;    // Re + Im of G^X, atom-major [Nwin][Nkz][NE][NN rounded up to even] (k_relayout)
  const double2* coef;   // coefficient table of the current chunk: pair index p - cp0
  const double2* dH;
  const SigItem* items;  // the chunk's items (items[0] = global item item0)
  const SigPair* pairs;
  const int32_t* pair_item;   // pair (global index) -> item (global index)
  int64_t item0;
  double2* Sig;
  double2* Gt;           // Gt scratch of the chunk [item][kz][E][72][NN] (TMA path)
  double2 scale;
  int64_t Nwin, Nout, Nb, DWp, cp0, npairs_chunk, ntiles;
  int NE, Nkz, Nqz, h, Norb, NN, Dmax, Dwin, ndc;
  int rows;              // Gt rows per (item, kz, E) block: 72 (items of <= 8 pairs) or 128 (FP32 mode, <= 14)
  int E0, NEo;           // outputs for window energies [E0, E0 + NEo) (NE = the G window; a sub-range of the rank's
                         // energies when the scratch is split by energy)
  int NEs, Es0;          // Σ tensor: NEs energies per kz; this launch's energies start at Σ energy Es0
  int gt_f32;            // Gt scratch holds float2 (FP32 mixed mode: k_sigma_tc -> FP32 sandwich)
  int gt_ld;             // Gt scratch row stride in elements: Norb² rounded up to a 16-byte multiple
  // QT_FLAG_DETERMINISTIC: destination lists of the chunk — entry = {a_out, first, count, -} into det_pairs
  // {il (chunk-relative item), t (pair in item)}, pairs in a fixed order; one CTA sums an atom's pairs
  const int4* det_atoms;
  const int2* det_pairs;
  int64_t n_det;
};

struct PiWArgs {
  const double2* GY;          // G^Y window, paper layout [Nkz][NE][Nwin][NN]
  const double2* dH;
  const PiPair* pairs;
  const PiItem* items;
  const int32_t* pair_item;   // pair -> item
  double2* W;                 // [item - i0][Nkz][xy chunk][NE][72 rows (t,ij)][20]
  int64_t p0, i0, Nwin, Nb;
  int64_t npairs;             // pairs of the chunk [p0, p0 + npairs) (k_pi_w2: one CTA per (pair, kz))
  int NE, Nkz, Norb, NN, nEB;
  int E0, NEo;                // energies of this rank's Π sum: window energies [E0, E0 + NEo)
};

struct PiCArgs {
  const double2* GX;     // G^X window, paper layout [Nkz][NE][Nwin][NN]
  const double* GXsum;   // Re + Im of G^X, atom-major [Nwin][Nkz][NE][NN rounded up to even]
  const double2* W;
  const PiItem* items;
  const PiPair* pairs;
  double2* Pi;
  double2 scale;
  int64_t i0, nitems, Nwin, Nout, Nb;
  int NE, Nkz, Nqz, h, NN, Nw, NWP, shift0;
  int NWv, step;         // GEMM columns = every shift shift0 + c (c < NWv); column c is frequency m = c / step
                         // when c % step == 0 (shift_step > 1: the other columns are computed and dropped)
  int E0, NEo;           // energies of this rank's Π sum: window energies [E0, E0 + NEo)
  int accumulate;        // add into Π (later energy sub-ranges of a chunk) instead of overwriting
};

struct PiSelfArgs {
  double2* Pi;
  const int32_t* nbr;
  int64_t Nout, Nb, Nqz, Nw, a_off;
};

constexpr int kEB = 4;

cudaError_t launch_sigma_coef_tiled(const CoefArgs& a, cudaStream_t st);
cudaError_t launch_sigma(const SigmaArgs& a, int64_t nitems, cudaStream_t st);
// energy-pair form of the Σ contraction for items of >= 4 pairs (kernels_sigma_pair.cu)
bool sigma_pair_supported(int Norb);
cudaError_t launch_sigma_pair(const SigmaArgs& a, int64_t nitems, cudaStream_t st);
cudaError_t launch_sigma_sand(const SigmaArgs& a, int64_t nitems, cudaStream_t st);
cudaError_t launch_sigma_sand_det(const SigmaArgs& a, cudaStream_t st);   // QT_FLAG_DETERMINISTIC
// FP32 mixed-precision Σ contraction (tcgen05 kind::tf32; kernels_sigma_tc.cu). Coefficient planes
// [item][q][4 planes][kTcRows][Kp] fp32; G planes [Nwin][Nkz][4][kTcRowsA][NEp] fp32.
constexpr int kTcRows = 128;    // FP32-mode Σ items: <= 14 pairs (126 coefficient rows) = UMMA N
constexpr int kTcPiPairs = 14;   // FP32-mode Π items: <= 14 pairs of one destination atom (126 of 128 UMMA rows)
constexpr int kTcPiRows = 128;
constexpr int kTcRowsA = 128;   // G plane rows (Norb² padded to the UMMA M)
cudaError_t launch_relayout_tc(const double2* G, float* out, int64_t Nkz, int64_t NE, int64_t NEp, int64_t Nwin, int NN,
                               int64_t a0, int64_t a1, cudaStream_t st);
cudaError_t launch_sigma_coef_tc(const CoefArgs& a, int Kp, cudaStream_t st);
cudaError_t launch_relayout_pi_tc(const double2* G, float* out, int64_t Nkz, int64_t NE, int64_t Epad, int64_t Nwin, int NN,
                                  int NNp, cudaStream_t st);
cudaError_t launch_pi_w_tc(const PiWArgs& a, float* Wp, int NNp, int64_t nitems, cudaStream_t st);
cudaError_t launch_pi_contract_tc(const PiCArgs& a, const float* Wp, const float* Gp, int64_t Epad, int NNp, int64_t nitems,
                                  cudaStream_t st);
cudaError_t launch_sigma_tc(const SigmaArgs& a, const float* Gtp, int64_t NEp, const float* coef, int Kp, int64_t nitems,
                            cudaStream_t st);
cudaError_t launch_pi_w(const PiWArgs& a, int64_t npairs_chunk, cudaStream_t st);
cudaError_t launch_pi_contract(const PiCArgs& a, int64_t nitems, cudaStream_t st);
cudaError_t launch_pi_self(const PiSelfArgs& a, cudaStream_t st);
// Re + Im of G [Nkz][NE][Nwin][NN] (paper layout) for window atoms [a0, a1) -> osum [Nwin][Nkz][NE][NN even]
// (the B-side sums of the Gauss 3M products, so the DMMA consumers issue no FP64 adds)
cudaError_t launch_relayout(const double2* in, double* osum, int64_t Nkz, int64_t NE, int64_t Nwin, int64_t NN,
                            int64_t a0, int64_t a1, cudaStream_t st);

}  // namespace qt
