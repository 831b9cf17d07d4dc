/* gen_host.c — host implementation of include/qt_gen.h (see that header for the
 * value/structure contract). Input generation only: no SSE arithmetic here.
 * gen_dev.cu implements the same generator on the device; tests check they
 * agree bit-for-bit. Build: gcc -O2 -fopenmp -ffp-contract=off -shared -fPIC. */
#include "qt_gen.h"
#include <math.h>
#include <stddef.h>

static inline uint64_t sm64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
static inline double draw(uint64_t seed, int id, int mode, uint64_t idx) {
  uint64_t z = sm64(seed ^ ((uint64_t)id * 0x9E3779B97F4A7C15ULL) ^ idx);
  if (mode == QTGEN_INTEGER) return (double)(int64_t)(z % 5ULL) - 2.0;
  return (double)(z >> 11) * 0x1.0p-53 * 2.0 - 1.0;
}
/* slot of a in nbr[b][:], -1 if absent */
static inline int rev_slot(const int32_t* nbr, int64_t Nb, int64_t b, int64_t a) {
  for (int64_t t = 0; t < Nb; ++t) if (nbr[b * Nb + t] == (int32_t)a) return (int)t;
  return -1;
}

/* PHYSICAL envelope (see qt_gen.h): occupation factor of energy e for tensor id (f for G<, g for G>) */
static inline double occupation(int id, int64_t e, int64_t NE) {
  const int t = (int)((40 * e) / NE) - 20;
  return 1.0 / (1.0 + ldexp(1.0, id == QTGEN_ID_GL ? t : -t));
}
static inline double shell_scale(int64_t slot) {
  return slot < 4 ? 1.0 : slot < 16 ? 0.3 : slot < 28 ? 0.1 : 0.03;
}

void qtgen_host_G(uint64_t seed, int id, int mode, int64_t Nkz, int64_t NE, int64_t Na, int64_t Norb,
                  int64_t e_lo, int64_t e_hi, int64_t a_lo, int64_t a_hi, double* out) {
  const int64_t ne = e_hi - e_lo, na = a_hi - a_lo, nn = Norb * Norb;
  const int64_t nblk = Nkz * ne * na;
#pragma omp parallel for schedule(static)
  for (int64_t q = 0; q < nblk; ++q) {
    int64_t k = q / (ne * na), rem = q % (ne * na), e = e_lo + rem / na, a = a_lo + rem % na;
    double* o = out + 2 * nn * q;
    if (mode == QTGEN_ZERO) { for (int64_t t = 0; t < 2 * nn; ++t) o[t] = 0.0; continue; }
    uint64_t base = (uint64_t)(((k * NE + e) * Na + a) * nn);
    if (mode == QTGEN_PHYSICAL) {
      const double occ = occupation(id, e, NE);
      for (int64_t r = 0; r < Norb; ++r)
        for (int64_t c = 0; c < Norb; ++c) {
          double are = 0.0, aim = 0.0;   /* A_rc = sum_k X_rk conj(X_ck) */
          for (int64_t kk = 0; kk < Norb; ++kk) {
            uint64_t fx = base + (uint64_t)(r * Norb + kk), fy = base + (uint64_t)(c * Norb + kk);
            double xr = draw(seed, QTGEN_ID_GL, QTGEN_RANDOM, 2 * fx), xi = draw(seed, QTGEN_ID_GL, QTGEN_RANDOM, 2 * fx + 1);
            double yr = draw(seed, QTGEN_ID_GL, QTGEN_RANDOM, 2 * fy), yi = draw(seed, QTGEN_ID_GL, QTGEN_RANDOM, 2 * fy + 1);
            are = are + (xr * yr + xi * yi);
            aim = aim + (xi * yr - xr * yi);
          }
          are = are / (double)Norb;
          aim = aim / (double)Norb;
          if (id == QTGEN_ID_GL) { /* i f A */
            o[2 * (r * Norb + c)] = -(occ * aim);
            o[2 * (r * Norb + c) + 1] = occ * are;
          } else {                 /* -i g A */
            o[2 * (r * Norb + c)] = occ * aim;
            o[2 * (r * Norb + c) + 1] = -(occ * are);
          }
        }
      continue;
    }
    for (int64_t r = 0; r < Norb; ++r)
      for (int64_t c = 0; c < Norb; ++c) {
        uint64_t f_rc = base + (uint64_t)(r * Norb + c), f_cr = base + (uint64_t)(c * Norb + r);
        double xr_rc = draw(seed, id, mode, 2 * f_rc), xi_rc = draw(seed, id, mode, 2 * f_rc + 1);
        double xr_cr = draw(seed, id, mode, 2 * f_cr), xi_cr = draw(seed, id, mode, 2 * f_cr + 1);
        /* G = (X - X^dagger)/2 */
        o[2 * (r * Norb + c)] = (xr_rc - xr_cr) * 0.5;
        o[2 * (r * Norb + c) + 1] = (xi_rc + xi_cr) * 0.5;
      }
  }
}

void qtgen_host_D(uint64_t seed, int id, int mode, int64_t Nqz, int64_t Nw, int64_t Na, int64_t Nb,
                  const int32_t* nbr, int64_t delta_m, int64_t a_lo, int64_t a_hi, double* out) {
  const int64_t na = a_hi - a_lo, ns = Nb + 1;
  const int64_t nblk = Nqz * Nw * na * ns;
  const int64_t h = Nqz / 2;
#pragma omp parallel for schedule(static)
  for (int64_t q = 0; q < nblk; ++q) {
    int64_t slot = q % ns, t1 = q / ns, a = a_lo + t1 % na, t2 = t1 / na, m = t2 % Nw, qz = t2 / Nw;
    double* o = out + 18 * q;
    for (int t = 0; t < 18; ++t) o[t] = 0.0;
    if (mode == QTGEN_ZERO) continue;
    if (mode == QTGEN_DELTA) {
      if (slot > 0 && nbr[a * Nb + slot - 1] >= 0 && qz == h && m == delta_m)
        for (int i = 0; i < 3; ++i) o[2 * (i * 3 + i)] = 0.5;
      continue;
    }
    if (slot == 0) { /* self block: (Y - Y^dagger)/2 */
      uint64_t base = (uint64_t)((((qz * Nw + m) * Na + a) * ns + 0) * 9);
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
          uint64_t fij = base + i * 3 + j, fji = base + j * 3 + i;
          o[2 * (i * 3 + j)] = (draw(seed, id, mode, 2 * fij) - draw(seed, id, mode, 2 * fji)) * 0.5;
          o[2 * (i * 3 + j) + 1] = (draw(seed, id, mode, 2 * fij + 1) + draw(seed, id, mode, 2 * fji + 1)) * 0.5;
        }
      continue;
    }
    int64_t b = nbr[a * Nb + slot - 1];
    if (b < 0) continue;
    if (a < b) { /* Z drawn at (a, slot) */
      uint64_t base = (uint64_t)((((qz * Nw + m) * Na + a) * ns + slot) * 9);
      for (int t = 0; t < 9; ++t) { o[2 * t] = draw(seed, id, mode, 2 * (base + t)); o[2 * t + 1] = draw(seed, id, mode, 2 * (base + t) + 1); }
    } else { /* D_{a,b} = -(D_{b,a})^dagger, D_{b,a} = Z drawn at (b, rev+1) */
      int r = rev_slot(nbr, Nb, b, a);
      uint64_t base = (uint64_t)((((qz * Nw + m) * Na + b) * ns + (r + 1)) * 9);
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
          uint64_t f = base + j * 3 + i;
          o[2 * (i * 3 + j)] = -draw(seed, id, mode, 2 * f);
          o[2 * (i * 3 + j) + 1] = draw(seed, id, mode, 2 * f + 1);
        }
    }
  }
}

void qtgen_host_dH(uint64_t seed, int id, int mode, int64_t Na, int64_t Nb, int64_t Norb,
                   const int32_t* nbr, double* out) {
  const int64_t nn = Norb * Norb, nblk = Na * Nb * 3;
#pragma omp parallel for schedule(static)
  for (int64_t q = 0; q < nblk; ++q) {
    int64_t i = q % 3, s = (q / 3) % Nb, a = q / (3 * Nb);
    double* o = out + 2 * nn * q;
    for (int64_t t = 0; t < 2 * nn; ++t) o[t] = 0.0;
    if (mode == QTGEN_ZERO) continue;
    int64_t b = nbr[a * Nb + s];
    if (b < 0) continue;
    if (a < b) {
      uint64_t base = (uint64_t)(((a * Nb + s) * 3 + i) * nn);
      const double sc = mode == QTGEN_PHYSICAL ? shell_scale(s) : 1.0;
      for (int64_t t = 0; t < nn; ++t) {
        o[2 * t] = sc * draw(seed, id, mode, 2 * (base + t));
        o[2 * t + 1] = sc * draw(seed, id, mode, 2 * (base + t) + 1);
      }
    } else { /* dH_{a,b} = (dH_{b,a})^dagger */
      int r = rev_slot(nbr, Nb, b, a);
      uint64_t base = (uint64_t)(((b * Nb + r) * 3 + i) * nn);
      const double sc = mode == QTGEN_PHYSICAL ? shell_scale(r) : 1.0;
      for (int64_t x = 0; x < Norb; ++x)
        for (int64_t y = 0; y < Norb; ++y) {
          uint64_t f = base + y * Norb + x;
          o[2 * (x * Norb + y)] = sc * draw(seed, id, mode, 2 * f);
          o[2 * (x * Norb + y) + 1] = -(sc * draw(seed, id, mode, 2 * f + 1));
        }
    }
  }
}
