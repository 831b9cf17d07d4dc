/* qt_sse.h — C ABI of libqtsse.so, the B200 (sm_100a) electron-phonon scattering
 * self-energy (SSE) hot path of Ziogas et al., SC19 (arXiv 1912.10024).
 *
 * The library evaluates, for X ∈ {<,>} and Y the other one:
 *   Σ^X_aa(kz,E)  — Eq. 3, PAPER.md P:355-365 (electron SSE, diagonal atom blocks)
 *   Π^X_ab(ω,qz)  — Eq. 4, PAPER.md P:366-375 (phonon SSE, self + N_b neighbour blocks)
 * from the tensors of PAPER.md P:386-397, with the readings R1-R20 of DESIGN.md §3:
 *   Σ^X[kz][E][a] = scale_Σ · Σ_{s,qz,m} Σ_{i,j} ∇_iH_{ab} ·
 *        ( Dc^X_{ij}(qz,m) G^X_b(kz-qz, E-s_m) + Dc^Y_{ji}(qz,m) G^X_b(kz-qz, E+s_m) ) · ∇_jH_{ba}
 *   Dc^X_{ij}(qz,m) = D^X[qz][m][b][r+1] - D^X[qz][m][b][0] - D^X[qz][m][a][0] + D^X[qz][m][a][s+1]
 *   Π^X[qz][m][a][s+1]_{ij} = scale_Π · Σ_{kz,E} tr{ ∇_iH_{ba} G^X_a(kz+qz, E+s_m) ∇_jH_{ab} G^Y_b(kz,E) }
 *   Π^X[qz][m][a][0] = Σ_s Π^X[qz][m][a][s+1]
 * where b = nbr[a][s], r = the slot of a in nbr[b], s_m = shift0 + m·shift_step (ħω_m/ΔE),
 * kz-qz ↦ (kz-qz+h) mod Nkz, kz+qz ↦ (kz+qz-h) mod Nkz, h = Nkz/2, and energies
 * outside [0,NE) contribute nothing (zero extension, never clamped).
 *
 * Tensors (all complex128, interleaved (re,im), row-major, 16-byte aligned):
 *   G≷, Σ≷ : [Nkz][NE][Na][Norb][Norb]
 *   D≷, Π≷ : [Nqz][Nw][Na][Nb+1][3][3]      (slot 0 = self, slot s+1 = neighbour s)
 *   dH     : [Na][Nb][3][Norb][Norb]        dH[a][s][i] = ∇_i H_{a, nbr[a][s]}
 *   neighbors (host, int32): [Na][Nb], -1 = empty slot; must be symmetric.
 *
 * Multi-GPU (nranks > 1): the ranks form a Ta x TE grid (the paper's Ta x TE tiling),
 * rank = ta·TE + te. QT_SHARD_ATOM is Ta = nranks (TE = 1), QT_SHARD_ENERGY is TE = nranks (Ta = 1),
 * QT_SHARD_2D takes Ta = desc.grid_atoms (TE = nranks / Ta). Rank (ta, te) owns the atoms
 * [a_lo, a_hi) (slab ta of contiguous atoms balanced by pair count) and the energies [e_lo, e_hi)
 * (slab te balanced by per-energy work), and every pointer holds the rank's LOCAL WINDOW
 * (see qt_sse_query / qt_sse_shard_info):
 *   G≷  : [Nkz][ew_hi-ew_lo][w_hi-w_lo][Norb][Norb]   owned block + halo (window atoms x window energies)
 *   D≷  : [Nqz][Nw][w_hi-w_lo][Nb+1][3][3]            owned atoms + atom halo
 *   dH  : [w_hi-w_lo][Nb][3][Norb][Norb]
 *   Σ≷  : [Nkz][e_hi-e_lo][a_hi-a_lo][Norb][Norb]      owned block only
 *   Π≷  : [Nqz][Nw][pa_hi-pa_lo][Nb+1][3][3]          Π sums over all energies: with TE > 1 the TE ranks of
 *         an atom slab each own one sub-slab [pa_lo, pa_hi) of it and receive the sum of the slab's partial
 *         sums by ncclReduce (overlapped with the next sub-slab's compute); a plan without a communicator
 *         ("loopback": one process emulating a rank) returns this rank's PARTIAL sum over its own energies
 *         for the whole atom slab, pa = [a_lo, a_hi).
 * The window is the halo contract: the OWNED region of G≷/D≷ is input (read only); the HALO region
 * (window entries owned by other ranks) is written by the library's NCCL exchange (qt_sse_sigma_pi and
 * qt_sse_halo_exchange) before it is read. This keeps one G window per rank instead of an owned copy plus
 * a second, library-owned window (the difference decides whether BASELINE cfg4/cfg5 fit).
 *
 * Ownership: the caller owns every tensor; outputs are OVERWRITTEN (never accumulated); apart from the
 * halo region above, inputs are never modified. The plan owns its device workspace, work lists, halo
 * staging, Π partial buffers, its communicators and its communication stream.
 * Execution: calls are stream-ordered and asynchronous on `stream`; argument and launch errors are
 * returned synchronously; asynchronous device faults surface as QT_ERR_CUDA and asynchronous NCCL
 * failures (ncclCommGetAsyncError) as QT_ERR_NCCL on a later call or on qt_sse_query. Calls of one plan on
 * different streams are ordered by the plan (each call waits for the previous one's completion event).
 * No exceptions cross the ABI. One plan per host thread. A plan is reusable with new tensor pointers of the
 * same dimensions.
 */
#ifndef QT_SSE_H
#define QT_SSE_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  QT_OK = 0,
  QT_ERR_INVALID_ARG = 1,   /* bad dims, neighbour table, grid, null/misaligned/aliased pointer          */
  QT_ERR_UNSUPPORTED = 2,   /* Norb > 12 (> 10 in FP32 mode), (Nω−1)·shift_step + 1 > 128 (80) shifts    */
  QT_ERR_OUT_OF_MEMORY = 3,
  QT_ERR_CUDA = 4,
  QT_ERR_NCCL = 5,
  QT_ERR_INTERNAL = 6
} qt_status;

typedef enum { QT_PREC_FP64 = 0, QT_PREC_FP32_MIXED = 1 } qt_precision;
typedef enum { QT_SHARD_NONE = 0, QT_SHARD_ENERGY = 1, QT_SHARD_ATOM = 2, QT_SHARD_2D = 3 } qt_shard;

/* desc.flags */
#define QT_FLAG_DETERMINISTIC 1u   /* Σ neighbour sum in a fixed order (no floating-point atomics): the FP64 */
                                   /* result is bitwise reproducible run to run; slower sandwich             */

typedef struct {
  int64_t Na, Nb, Norb, N3D, NE, Nw, Nkz, Nqz; /* paper symbols; N3D must be 3; Nkz == Nqz                    */
  int32_t shift0, shift_step;                  /* ħω_m/ΔE = shift0 + m·shift_step; shift0, shift_step ≥ 1     */
  qt_precision precision;                      /* QT_PREC_FP64, or QT_PREC_FP32_MIXED (Norb <= 10): both      */
                                               /* contractions on tcgen05 (kind::tf32, operands split hi+lo,  */
                                               /* TMEM segments of 128 products summed in registers: Σ FP32, */
                                               /* Π FP64), the ∇H sandwiches in FP32; ≤1e-5 per block (§8(f) */
                                               /* NEXT(1), §4.4)                           */
  qt_shard shard;                              /* QT_SHARD_NONE, or with nranks > 1 ATOM / ENERGY / 2D        */
  int32_t rank, nranks;
  const void* nccl_unique_id;                  /* host ptr to a 128-byte ncclUniqueId (nranks > 1), or NULL:  */
                                               /* loopback plan (no exchange, partial Π; see above)           */
  size_t workspace_limit;                      /* bytes of device scratch the plan may use; 0 = auto          */
  int32_t grid_atoms;                          /* QT_SHARD_2D: Ta (divides nranks); ignored otherwise         */
  uint32_t flags;                              /* QT_FLAG_*                                                   */
} qt_sse_desc;

typedef struct qt_sse_plan_s* qt_sse_plan_t;

typedef struct {
  int64_t a_lo, a_hi;       /* atoms whose Σ this rank computes (outputs)                              */
  int64_t w_lo, w_hi;       /* atom window of this rank's input tensors (owned + halo)                 */
  int64_t npairs;           /* valid (a,s) pairs with a in [a_lo,a_hi)                                  */
  size_t workspace_bytes;   /* device bytes owned by the plan                                           */
  double flops_sigma;       /* algorithmic FP64 flops of one qt_sse_sigma call (both X)                 */
  double flops_pi;          /* algorithmic FP64 flops of one qt_sse_pi call (both X)                    */
  double halo_bytes;        /* bytes received per exchange (G≷ + D≷ halo)                               */
  int64_t e_lo, e_hi;       /* output energies of this rank                                             */
  int64_t ew_lo, ew_hi;     /* energy window of this rank's G inputs: [e_lo - Dmax, e_hi + Dmax) ∩ [0,NE) */
  int64_t pa_lo, pa_hi;     /* atoms of this rank's Π output                                            */
  int32_t Ta, TE, ta, te;   /* rank grid and this rank's coordinates                                    */
  double reduce_bytes;      /* bytes this rank sends in the Π reduction per qt_sse_pi call              */
  double mem_bytes;         /* device bytes per rank: caller tensors (window inputs, outputs) + plan    */
  double flops_sigma_pair;  /* the part of flops_sigma's D-contraction run by the energy-pair kernel
                               (k_sigma_pair: FP64, Norb 9..11, items of >= 4 pairs); 0 otherwise      */
} qt_sse_info;

/* Validates desc + neighbours, builds the work lists, allocates the workspace. With an NCCL unique id and
 * nranks > 1 the call is collective over the ranks (creates the communicators). */
qt_status qt_sse_plan(const qt_sse_desc* desc, const int32_t* neighbors_host, void* cuda_stream,
                      qt_sse_plan_t* plan_out);

/* Σ^<, Σ^> (Eq. 3) from window inputs whose halo is already filled. scale = complex ∫dħω/2π weight
 * (default i·ΔE/2π, R8). */
qt_status qt_sse_sigma(qt_sse_plan_t plan, const void* dH, const void* G_less, const void* G_gtr,
                       const void* D_less, const void* D_gtr, double scale_re, double scale_im,
                       void* Sig_less, void* Sig_gtr, void* cuda_stream);

/* Π^<, Π^> (Eq. 4) from window inputs whose halo is already filled (TE > 1 with a communicator: the
 * partial sums are reduced to the sub-slab owners). scale = complex ∫dE/2π weight (default -i·ΔE/2π). */
qt_status qt_sse_pi(qt_sse_plan_t plan, const void* dH, const void* G_less, const void* G_gtr,
                    double scale_re, double scale_im, void* Pi_less, void* Pi_gtr, void* cuda_stream);

/* The whole hot path in one call: halo exchange (nranks > 1 with a communicator)
 * on the plan's communication stream, overlapped with the work that reads no halo entry (interior source
 * atoms, owned-atom re-layout, coefficient tables); Σ≷ and Π≷ sharing one re-layout of G≷; the Π
 * reduction (TE > 1) overlapped with the next sub-slab. Same results as halo_exchange + sigma + pi. */
qt_status qt_sse_sigma_pi(qt_sse_plan_t plan, const void* dH, void* G_less, void* G_gtr, void* D_less,
                          void* D_gtr, double sig_scale_re, double sig_scale_im, double pi_scale_re,
                          double pi_scale_im, void* Sig_less, void* Sig_gtr, void* Pi_less, void* Pi_gtr,
                          void* cuda_stream);

/* End-to-end call on HOST buffers (pinned or pageable) holding the window inputs and the outputs:
 * copies inputs to device buffers owned by the plan, runs qt_sse_sigma_pi, copies Σ≷, Π≷ back,
 * and synchronizes `cuda_stream` before returning. */
qt_status qt_sse_execute_host(qt_sse_plan_t plan, const void* dH, const void* G_less, const void* G_gtr,
                              const void* D_less, const void* D_gtr, double sig_scale_re, double sig_scale_im,
                              double pi_scale_re, double pi_scale_im, void* Sig_less, void* Sig_gtr,
                              void* Pi_less, void* Pi_gtr, void* cuda_stream);

qt_status qt_sse_query(qt_sse_plan_t plan, qt_sse_info* out);

/* Halo exchange alone (nranks > 1 with a communicator): fills the halo region of the window buffers from
 * their owners — G≷ boxes (window atoms x window energies owned by a peer) and, with Ta > 1, D≷ atom halos —
 * with one grouped ncclSend/ncclRecv round on `cuda_stream` (energy-only splits send the contiguous energy
 * ranges in place; atom splits pack). Owned entries are only read. QT_OK with nranks == 1;
 * QT_ERR_UNSUPPORTED for a loopback plan; QT_ERR_NCCL on NCCL failure. */
qt_status qt_sse_halo_exchange(qt_sse_plan_t plan, void* G_less, void* G_gtr, void* D_less, void* D_gtr,
                               void* cuda_stream);

/* Writes a fresh 128-byte ncclUniqueId into out128 (call on one rank, broadcast to the others). */
qt_status qt_sse_nccl_unique_id(void* out128);

void qt_sse_destroy(qt_sse_plan_t plan);   /* NULL-safe; frees workspace, streams, events, NCCL comms */
const char* qt_sse_status_string(qt_status s);

/* Host-only (no device needed): algorithmic flop counts for desc + neighbours (the rank's share when
 * nranks > 1): out[0] Σ contraction, out[1] Σ sandwich, out[2] Π sandwich, out[3] Π contraction
 * (both X, 8 real flops per complex multiply-add, in-window valid-pair work only). */
qt_status qt_sse_count_flops(const qt_sse_desc* desc, const int32_t* neighbors_host, double out[4]);

/* Host-only (no device needed): the qt_sse_info a plan for desc (incl. rank/nranks) would report:
 * owned atoms/energies, windows, Π sub-slab, pairs, flops, halo and reduction bytes, and mem_bytes, the
 * device footprint per rank (caller window tensors + outputs + the plan's allocations for
 * desc.workspace_limit, or the automatic workspace cap of min(48 GiB, Σ/Π scratch need) when 0). */
qt_status qt_sse_shard_info(const qt_sse_desc* desc, const int32_t* neighbors_host, qt_sse_info* out);

/* Number of this library's kernel launches issued since load (for bench accounting). */
uint64_t qt_sse_launch_count(void);

/* Per-kernel timing: while enabled, every launch of `plan` is bracketed by CUDA events
 * recorded on the launching stream. qt_sse_timing_read synchronizes those events and
 * returns, per kernel kind (QT_K_*), the summed milliseconds and launch counts since the
 * last reset, then clears them. */
enum { QT_K_SIGMA_COEF = 0, QT_K_SIGMA = 1, QT_K_PI_W = 2, QT_K_PI_CONTRACT = 3, QT_K_PI_SELF = 4,
       QT_K_RELAYOUT = 5, QT_K_HALO = 6, QT_K_SIGMA_SAND = 7, QT_K_SIGMA_PAIR = 8, QT_K_NKINDS = 9 };
/* QT_K_SIGMA = k_sigma (multi-energy tiles) or k_sigma_tc (FP32 mode); QT_K_SIGMA_PAIR = k_sigma_pair. */
qt_status qt_sse_timing_enable(qt_sse_plan_t plan, int enable);
qt_status qt_sse_timing_read(qt_sse_plan_t plan, double ms[QT_K_NKINDS], int64_t launches[QT_K_NKINDS]);

#ifdef __cplusplus
}
#endif
#endif
