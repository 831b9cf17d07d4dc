/* oracle.c — CPU ORACLE for the electron-phonon scattering self-energies.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. The product path
 * (paper_1912_10024_b200/, libqtsse.so) never links, loads or calls it, and it
 * shares no code with the CUDA path (no headers, helpers or tables).
 *
 * What it computes: Eq. 3 (Σ≷) and Eq. 4 (Π≷)
 * literally, as plain nested loops over output blocks, one matrix product at a
 * time, with the readings R1-R19 of SURVEY.md §8(c) / DESIGN.md §3:
 *   Σ^X_aa(kz,E) = scale_Σ · Σ_{s, qz, m} Σ_{i,j} [
 *        Dc^X_{ij}(qz,m) · ∇_iH_{ab} G^X_bb(kz-qz, E - ħω_m) ∇_jH_{ba}      (absorption)
 *      + Dc^Y_{ji}(qz,m) · ∇_iH_{ab} G^X_bb(kz-qz, E + ħω_m) ∇_jH_{ba} ]    (emission, R2/R3)
 *   Dc^X_{ij} = D^X_ba - D^X_bb - D^X_aa + D^X_ab   (the four-term combination of Eq. 3)
 *   Π^X_ab(qz,ω_m) = scale_Π · Σ_{kz,E} tr{∇_iH_ba G^X_aa(E+ħω_m, kz+qz) ∇_jH_ab G^Y_bb(E,kz)}
 *   Π^X_aa = Σ_{l∈N(a)} (same summand with b := l)          (R9)
 * X ∈ {<,>}, Y = the other one. b = nbr[a][s], r = reverse slot (nbr[b][r] = a).
 * Momentum indices (R5): h = floor(Nkz/2); kz-qz -> (kz-qz+h) mod Nkz,
 * kz+qz -> (kz+qz-h) mod Nkz. Energies: ħω_m/ΔE = s_m = shift0 + m*shift_step
 * (R6); E±ħω outside [0,NE) contributes nothing (R7). The ∫dħω/2π and ∫dE/2π
 * rectangle-rule weights are folded into the complex scale factors (R8), applied
 * once at the end. ∇H_ba is read from the tensor at (b, r) (R10).
 *
 * Arithmetic: explicit re/im products in double (built with -ffp-contract=off),
 * each output element accumulated in long double. No blocking, fusion or
 * reordering beyond the loops of the definitions above.
 * Parity pins: tests/test_oracle_*.py (brute force, integer-exact, D=δ, linearity,
 * anti-Hermiticity, window edges, kz covariance, Π self slot, impulses, relabel).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int64_t Na, Nb, Norb, NE, Nw, Nkz, Nqz;
  int64_t shift0, shift_step;
} or_dims;

typedef struct { double re, im; } cplx;

static inline cplx cmul(cplx a, cplx b) {
  cplx c;
  c.re = a.re * b.re - a.im * b.im;
  c.im = a.re * b.im + a.im * b.re;
  return c;
}

/* C = A @ B for n×n complex row-major matrices (plain triple loop). */
static void matmul(const cplx* A, const cplx* B, cplx* C, int64_t n) {
  for (int64_t x = 0; x < n; ++x)
    for (int64_t y = 0; y < n; ++y) {
      double re = 0.0, im = 0.0;
      for (int64_t u = 0; u < n; ++u) {
        cplx p = cmul(A[x * n + u], B[u * n + y]);
        re += p.re;
        im += p.im;
      }
      C[x * n + y].re = re;
      C[x * n + y].im = im;
    }
}

static int64_t mod(int64_t x, int64_t n) { int64_t r = x % n; return r < 0 ? r + n : r; }

/* reverse slot: r with nbr[b][r] == a, or -1 */
static int64_t rev_of(const int32_t* nbr, int64_t Nb, int64_t b, int64_t a) {
  for (int64_t t = 0; t < Nb; ++t) if (nbr[b * Nb + t] == a) return t;
  return -1;
}

/* pointers to blocks */
static const cplx* Gblk(const double* G, const or_dims* d, int64_t k, int64_t e, int64_t a) {
  return (const cplx*)G + ((k * d->NE + e) * d->Na + a) * d->Norb * d->Norb;
}
static const cplx* Dblk(const double* D, const or_dims* d, int64_t q, int64_t m, int64_t a, int64_t slot) {
  return (const cplx*)D + (((q * d->Nw + m) * d->Na + a) * (d->Nb + 1) + slot) * 9;
}
static const cplx* dHblk(const double* dH, const or_dims* d, int64_t a, int64_t s, int64_t i) {
  return (const cplx*)dH + ((a * d->Nb + s) * 3 + i) * d->Norb * d->Norb;
}

/* One Σ^X block (kz, e, a), Eq. 3. X = 0 (<) or 1 (>).
 * GX = G^X, DX = D^X, DY = D^Y. out: Norb×Norb complex. */
static void sigma_block(const or_dims* d, const int32_t* nbr, const double* dH, const double* GX,
                        const double* DX, const double* DY, cplx scale, int64_t kz, int64_t e, int64_t a,
                        double* out) {
  const int64_t n = d->Norb, nn = n * n, h = d->Nkz / 2;
  long double* acc = (long double*)calloc(2 * nn, sizeof(long double));
  cplx* T = (cplx*)malloc(nn * sizeof(cplx));
  cplx* U = (cplx*)malloc(nn * sizeof(cplx));
  for (int64_t s = 0; s < d->Nb; ++s) {                 /* Σ over neighbours b of a (R1) */
    int64_t b = nbr[a * d->Nb + s];
    if (b < 0) continue;                                 /* empty slot (R12) */
    int64_t r = rev_of(nbr, d->Nb, b, a);
    for (int64_t qz = 0; qz < d->Nqz; ++qz) {
      int64_t kp = mod(kz - qz + h, d->Nkz);             /* kz - qz (R4, R5) */
      for (int64_t m = 0; m < d->Nw; ++m) {
        int64_t sm = d->shift0 + m * d->shift_step;      /* ħω_m / ΔE (R6) */
        for (int term = 0; term < 2; ++term) {           /* 0: E-ħω with D^X; 1: E+ħω with D^Y, transposed (R2, R3) */
          int64_t ep = term == 0 ? e - sm : e + sm;
          if (ep < 0 || ep >= d->NE) continue;           /* outside the energy window (R7) */
          const double* Dsel = term == 0 ? DX : DY;
          const cplx* Dba = Dblk(Dsel, d, qz, m, b, r + 1);
          const cplx* Dbb = Dblk(Dsel, d, qz, m, b, 0);
          const cplx* Daa = Dblk(Dsel, d, qz, m, a, 0);
          const cplx* Dab = Dblk(Dsel, d, qz, m, a, s + 1);
          cplx Dc[9];
          for (int t = 0; t < 9; ++t) {                  /* D_ba - D_bb - D_aa + D_ab (Eq. 3) */
            Dc[t].re = Dba[t].re - Dbb[t].re - Daa[t].re + Dab[t].re;
            Dc[t].im = Dba[t].im - Dbb[t].im - Daa[t].im + Dab[t].im;
          }
          const cplx* Gb = Gblk(GX, d, kp, ep, b);
          for (int64_t i = 0; i < 3; ++i)
            for (int64_t j = 0; j < 3; ++j) {
              cplx c = term == 0 ? Dc[i * 3 + j] : Dc[j * 3 + i];
              matmul(dHblk(dH, d, a, s, i), Gb, T, n);   /* ∇_iH_ab · G_bb */
              matmul(T, dHblk(dH, d, b, r, j), U, n);    /* · ∇_jH_ba */
              for (int64_t t = 0; t < nn; ++t) {
                cplx p = cmul(c, U[t]);
                acc[2 * t] += p.re;
                acc[2 * t + 1] += p.im;
              }
            }
        }
      }
    }
  }
  for (int64_t t = 0; t < nn; ++t) {                     /* single final multiply by the scale (R8) */
    double re = (double)acc[2 * t], im = (double)acc[2 * t + 1];
    out[2 * t] = scale.re * re - scale.im * im;
    out[2 * t + 1] = scale.re * im + scale.im * re;
  }
  free(acc); free(T); free(U);
}

/* Π^X summand for pair (a, s) accumulated into acc3 (9 complex, long double), Eq. 4. */
static void pi_pair_accumulate(const or_dims* d, const int32_t* nbr, const double* dH, const double* GX,
                               const double* GY, int64_t qz, int64_t m, int64_t a, int64_t s, long double* acc3) {
  const int64_t n = d->Norb, nn = n * n, h = d->Nkz / 2;
  int64_t b = nbr[a * d->Nb + s];
  if (b < 0) return;
  int64_t r = rev_of(nbr, d->Nb, b, a);
  int64_t sm = d->shift0 + m * d->shift_step;
  cplx* T1 = (cplx*)malloc(nn * sizeof(cplx));
  cplx* T2 = (cplx*)malloc(nn * sizeof(cplx));
  cplx* T3 = (cplx*)malloc(nn * sizeof(cplx));
  for (int64_t kz = 0; kz < d->Nkz; ++kz) {
    int64_t k2 = mod(kz + qz - h, d->Nkz);               /* kz + qz (R5) */
    for (int64_t e = 0; e < d->NE; ++e) {
      int64_t e2 = e + sm;                               /* E + ħω (R7: drop if outside) */
      if (e2 < 0 || e2 >= d->NE) continue;
      const cplx* Ga = Gblk(GX, d, k2, e2, a);          /* G^X_aa(E+ħω, kz+qz) (R13) */
      const cplx* Gb = Gblk(GY, d, kz, e, b);           /* G^Y_bb(E, kz) */
      for (int64_t i = 0; i < 3; ++i)
        for (int64_t j = 0; j < 3; ++j) {
          matmul(dHblk(dH, d, b, r, i), Ga, T1, n);      /* ∇_iH_ba · G_aa */
          matmul(T1, dHblk(dH, d, a, s, j), T2, n);      /* · ∇_jH_ab */
          matmul(T2, Gb, T3, n);                         /* · G_bb */
          long double tre = 0.0L, tim = 0.0L;
          for (int64_t x = 0; x < n; ++x) { tre += T3[x * n + x].re; tim += T3[x * n + x].im; }  /* tr{} */
          acc3[2 * (i * 3 + j)] += tre;
          acc3[2 * (i * 3 + j) + 1] += tim;
        }
    }
  }
  free(T1); free(T2); free(T3);
}

/* One Π^X block (qz, m, a, slot); slot 0 = self (R9, R11), slot s+1 = neighbour s. */
static void pi_block(const or_dims* d, const int32_t* nbr, const double* dH, const double* GX, const double* GY,
                     cplx scale, int64_t qz, int64_t m, int64_t a, int64_t slot, double* out) {
  long double acc3[18];
  for (int t = 0; t < 18; ++t) acc3[t] = 0.0L;
  if (slot == 0) {
    for (int64_t s = 0; s < d->Nb; ++s) pi_pair_accumulate(d, nbr, dH, GX, GY, qz, m, a, s, acc3);
  } else {
    pi_pair_accumulate(d, nbr, dH, GX, GY, qz, m, a, slot - 1, acc3);
  }
  for (int t = 0; t < 9; ++t) {
    double re = (double)acc3[2 * t], im = (double)acc3[2 * t + 1];
    out[2 * t] = scale.re * re - scale.im * im;
    out[2 * t + 1] = scale.re * im + scale.im * re;
  }
}

/* ---------------- exported entry points (ctypes; tests/bench only) ---------------- */

/* Σ blocks listed in blk[nblk][4] = (X, kz, e, a); out[nblk][Norb][Norb] complex. */
void oracle_sigma_blocks(const or_dims* d, const int32_t* nbr, const double* dH, const double* G_less,
                         const double* G_gtr, const double* D_less, const double* D_gtr, double scale_re,
                         double scale_im, int64_t nblk, const int64_t* blk, double* out) {
  cplx sc = {scale_re, scale_im};
  const int64_t nn = d->Norb * d->Norb;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t q = 0; q < nblk; ++q) {
    const int64_t* B = blk + 4 * q;
    int X = (int)B[0];
    sigma_block(d, nbr, dH, X == 0 ? G_less : G_gtr, X == 0 ? D_less : D_gtr, X == 0 ? D_gtr : D_less, sc, B[1],
                B[2], B[3], out + 2 * nn * q);
  }
}

/* Π blocks listed in blk[nblk][5] = (X, qz, m, a, slot); out[nblk][3][3] complex. */
void oracle_pi_blocks(const or_dims* d, const int32_t* nbr, const double* dH, const double* G_less,
                      const double* G_gtr, double scale_re, double scale_im, int64_t nblk, const int64_t* blk,
                      double* out) {
  cplx sc = {scale_re, scale_im};
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t q = 0; q < nblk; ++q) {
    const int64_t* B = blk + 5 * q;
    int X = (int)B[0];
    pi_block(d, nbr, dH, X == 0 ? G_less : G_gtr, X == 0 ? G_gtr : G_less, sc, B[1], B[2], B[3], B[4],
             out + 18 * q);
  }
}

/* Full tensors: Σ≷ [Nkz][NE][Na][Norb][Norb], Π≷ [Nqz][Nw][Na][Nb+1][3][3]. */
void oracle_sigma(const or_dims* d, const int32_t* nbr, const double* dH, const double* G_less, const double* G_gtr,
                  const double* D_less, const double* D_gtr, double scale_re, double scale_im, double* S_less,
                  double* S_gtr) {
  cplx sc = {scale_re, scale_im};
  const int64_t nn = d->Norb * d->Norb, per = d->Nkz * d->NE * d->Na;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t q = 0; q < 2 * per; ++q) {
    int X = (int)(q / per);
    int64_t t = q % per, a = t % d->Na, e = (t / d->Na) % d->NE, kz = t / (d->Na * d->NE);
    sigma_block(d, nbr, dH, X == 0 ? G_less : G_gtr, X == 0 ? D_less : D_gtr, X == 0 ? D_gtr : D_less, sc, kz, e,
                a, (X == 0 ? S_less : S_gtr) + 2 * nn * t);
  }
}

void oracle_pi(const or_dims* d, const int32_t* nbr, const double* dH, const double* G_less, const double* G_gtr,
               double scale_re, double scale_im, double* P_less, double* P_gtr) {
  cplx sc = {scale_re, scale_im};
  const int64_t ns = d->Nb + 1, per = d->Nqz * d->Nw * d->Na * ns;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t q = 0; q < 2 * per; ++q) {
    int X = (int)(q / per);
    int64_t t = q % per, slot = t % ns, a = (t / ns) % d->Na, m = (t / (ns * d->Na)) % d->Nw,
            qz = t / (ns * d->Na * d->Nw);
    pi_block(d, nbr, dH, X == 0 ? G_less : G_gtr, X == 0 ? G_gtr : G_less, sc, qz, m, a, slot,
             (X == 0 ? P_less : P_gtr) + 18 * t);
  }
}
