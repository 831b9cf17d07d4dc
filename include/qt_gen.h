/* qt_gen.h — seeded synthetic-input generator for the SSE hot path.
 *
 * This module is the ONLY code shared (by contract, not by linkage) between the
 * CPU oracle side and the CUDA product side: qtgen/gen_host.c implements it on
 * the host, qtgen/gen_dev.cu implements the same counter-based generator on the
 * device, and a GPU test checks the two bit-for-bit. It holds none of the
 * method's arithmetic (no Eq. 3 / Eq. 4 term is formed here): it only draws
 * numbers and imposes the input-structure invariants the paper and SPEC state
 * for the tensors (SURVEY.md §8(d) "Input structure"):
 *   - G≷ blocks anti-Hermitian (PAPER.md P:386-389 tensor shape),
 *   - D≷ anti-Hermitian as a full (atom,dir) matrix (slot 0 = self, R11),
 *   - ∇H_ba = (∇H_ab)†.
 *
 * Value of draw `idx` of tensor `id`:
 *   z = splitmix64(seed ^ (id * 0x9E3779B97F4A7C15) ^ idx)
 *   random : x = (z >> 11) * 2^-53 * 2 - 1            in [-1, 1)
 *   integer: x = (double)(z % 5) - 2                   in {-2..2} (pin P2)
 * Complex element with flat index f takes re = x(2f), im = x(2f+1).
 *
 * Modes (QTGEN_*): RANDOM, INTEGER, DELTA (D only: neighbour slots = I3/2 at
 * (qz = floor(Nqz/2), m = delta_m), everything else 0; pin P3), PHYSICAL (the
 * wide-dynamic-range envelope of SURVEY.md §8(d) "Modes", for the FP32 mode's
 * accuracy):
 *   G<(E) = i·f(E)·A,  G>(E) = -i·g(E)·A,  A = X X† / Norb  (Hermitian PSD),
 *   X the block's random draws of tensor ID_GL (X_rk = complex draw at flat
 *   index r·Norb + k; the same X for G< and G>, so both share one A),
 *   f(E) = 1 / (1 + 2^t), g(E) = 1 / (1 + 2^-t), t = floor(40·e / NE) - 20
 *   (a Fermi-like ladder over the energy grid: f spans 1 .. 2^-19, g = 1 - f
 *   up to rounding, computed without cancellation);
 *   ∇H: random draws scaled by the neighbour shell of the slot the draw is
 *   owned by: slots 0-3 ×1, 4-15 ×0.3, 16-27 ×0.1, 28+ ×0.03 (diamond shells
 *   of 4 / 12 / 12 / 6 neighbours, qtgen/geometry.py);
 *   D: as RANDOM.
 * Every PHYSICAL value is formed in a fixed order of IEEE-rounded +, ×, ÷
 * (no contraction; ldexp exact), so host and device agree bit for bit. A_cr is
 * conj(A_rc) exactly, so G stays exactly anti-Hermitian.
 *
 * Layouts (row-major, complex128 interleaved re,im):
 *   G  [Nkz][NE][Na][Norb][Norb]
 *   D  [Nqz][Nw][Na][Nb+1][3][3]
 *   dH [Na][Nb][3][Norb][Norb]           (dH[a][s][i] = ∇_i H_{a, nbr[a][s]})
 * Sub-range fills write only e in [e_lo,e_hi) / a in [a_lo,a_hi) into a dense
 * buffer of shape [..][e_hi-e_lo][a_hi-a_lo][..]; the draw index is always the
 * GLOBAL one, so shards on different ranks see the same values.
 */
#ifndef QT_GEN_H
#define QT_GEN_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum { QTGEN_RANDOM = 0, QTGEN_INTEGER = 1, QTGEN_DELTA = 2, QTGEN_ZERO = 3, QTGEN_PHYSICAL = 4 };
enum { QTGEN_ID_DH = 1, QTGEN_ID_GL = 2, QTGEN_ID_GG = 3, QTGEN_ID_DL = 4, QTGEN_ID_DG = 5 };

/* ---- host (qtgen/libqtgen_host.so, OpenMP) ---- */
void qtgen_host_G(uint64_t seed, int id, int mode, int64_t Nkz, int64_t NE, int64_t Na, int64_t Norb,
                  int64_t e_lo, int64_t e_hi, int64_t a_lo, int64_t a_hi, double* out);
void qtgen_host_D(uint64_t seed, int id, int mode, int64_t Nqz, int64_t Nw, int64_t Na, int64_t Nb,
                  const int32_t* nbr, int64_t delta_m, int64_t a_lo, int64_t a_hi, double* out);
void qtgen_host_dH(uint64_t seed, int id, int mode, int64_t Na, int64_t Nb, int64_t Norb,
                   const int32_t* nbr, double* out);

/* ---- device (qtgen/libqtgen_dev.so); pointers are device pointers, nbr too;
 *      stream is a cudaStream_t (void* to keep this header CUDA-free).
 *      Returns 0 on success, a cudaError_t value otherwise. ---- */
int qtgen_dev_G(uint64_t seed, int id, int mode, int64_t Nkz, int64_t NE, int64_t Na, int64_t Norb,
                int64_t e_lo, int64_t e_hi, int64_t a_lo, int64_t a_hi, double* out, void* stream);
int qtgen_dev_D(uint64_t seed, int id, int mode, int64_t Nqz, int64_t Nw, int64_t Na, int64_t Nb,
                const int32_t* nbr_dev, int64_t delta_m, int64_t a_lo, int64_t a_hi, double* out, void* stream);
int qtgen_dev_dH(uint64_t seed, int id, int mode, int64_t Na, int64_t Nb, int64_t Norb,
                 const int32_t* nbr_dev, double* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif
