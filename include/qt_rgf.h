/* qt_rgf.h — C ABI of the recursive Green's Function (RGF) solver in libqtsse.so: the GF phase that feeds
 * the SSE (§3 Eq. 1, and the RGF paragraph P:343-350).
 *
 * For every point p of a batch (an (E, kz) pair of the electron map or an (ω, qz) pair of the phonon map) the
 * block-tridiagonal matrix A_p = E·S(kz) − H(kz) − Σ^R(E,kz) (phonons: ω²·I − Φ(qz) − Π^R) with bnum diagonal
 * blocks of size bs defines (Eq. 1)
 *     G^R = A^{-1},     G^≷ = G^R · Σ^≷ · G^A,   G^A = (G^R)†,
 * and the solver returns the DIAGONAL BLOCKS of G^R, G^<, G^> (what the SSE needs) by one forward
 * pass over the blocks (left-connected g^R_n = (A_nn − A_{n,n−1} g^R_{n−1} A_{n−1,n})^{-1},
 * g^≷_n = g^R_n (Σ^≷_n + A_{n,n−1} g^≷_{n−1} A_{n,n−1}†) g^R_n†) and one backward pass
 * (G^R_n = g^R_n + X_n G^R_{n+1} A_{n+1,n} g^R_n,  G^≷_n = g^≷_n + X_n G^≷_{n+1} X_n† + Y_n − Y_n†,
 *  X_n = g^R_n A_{n,n+1},  Y_n = X_n G^R_{n+1} A_{n+1,n} g^≷_n). The backward lesser/greater step is exact when
 * the couplings are Hermitian (A_{n+1,n} = A_{n,n+1}†: real energy, Hermitian H and S, block-diagonal Σ^R) and
 * Σ^≷ is anti-Hermitian per block (reading R21); the solver does not check this.
 *
 * Tensors (device pointers, complex128 interleaved, row-major, 16-byte aligned):
 *   Ad       [P][bnum][bs][bs]     diagonal blocks A_nn
 *   Au       [P][bnum-1][bs][bs]   upper blocks A_{n,n+1}
 *   Al       [P][bnum-1][bs][bs]   lower blocks A_{n+1,n}
 *   Sl, Sg   [P][bnum][bs][bs]     diagonal blocks of Σ^<, Σ^>
 *   GRd, GLd, GGd [P][bnum][bs][bs]  outputs: diagonal blocks of G^R, G^<, G^> (overwritten)
 * Ownership: the caller owns every tensor; inputs are never modified; the plan owns its scratch (the
 * left-connected g^R, g^<, g^> of every block, temporaries, LU pivots) and its cuBLAS handle.
 * Execution: stream-ordered and asynchronous on `stream`; argument / launch errors are returned synchronously;
 * a singular pivot block is reported by qt_rgf_check_info (after synchronizing) as the first failing
 * (point, block), reading the getrf info the solver keeps on the device.
 */
#ifndef QT_RGF_H
#define QT_RGF_H
#include <stddef.h>
#include <stdint.h>

#include "qt_sse.h"   /* qt_status */

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int64_t P;      /* points in the batch                     */
  int64_t bnum;   /* diagonal blocks ("bnum")          */
  int64_t bs;     /* block size = Na·Norb / bnum             */
} qt_rgf_desc;

typedef struct qt_rgf_plan_s* qt_rgf_plan_t;

/* Validates the sizes (all > 0, bs <= 4096), allocates the scratch, creates the cuBLAS handle. */
qt_status qt_rgf_plan(const qt_rgf_desc* desc, void* cuda_stream, qt_rgf_plan_t* plan_out);

/* Diagonal blocks of G^R, G^<, G^> for every point (Eq. 1 by RGF, see above). */
qt_status qt_rgf_solve(qt_rgf_plan_t plan, const void* Ad, const void* Au, const void* Al, const void* Sl,
                       const void* Sg, void* GRd, void* GLd, void* GGd, void* cuda_stream);

/* Synchronizes `cuda_stream`; QT_OK if every block inversion of the last solve was regular, else
 * QT_ERR_INVALID_ARG with the first singular (point, block) in *point, *block. */
qt_status qt_rgf_check_info(qt_rgf_plan_t plan, void* cuda_stream, int64_t* point, int64_t* block);

/* Host-only: flops of one solve — out[0] = the executed dense count (complex GEMMs and inversions at 8 real
 * flops per complex multiply-add), out[1] = the paper's RGF model 8·(26·bnum − 25)·bs³ per point. */
qt_status qt_rgf_count_flops(const qt_rgf_desc* desc, double out[2]);

void qt_rgf_destroy(qt_rgf_plan_t plan);   /* NULL-safe */

#ifdef __cplusplus
}
#endif
#endif
