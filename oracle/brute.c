/* brute.c — scalarized brute-force evaluation of Eq. 3 / Eq. 4 for TINY inputs.
 *
 * TEST INFRASTRUCTURE ONLY (pin P1 for the oracle: "equals a
 * scalarized six-nested-loop oracle"). Written independently of oracle.c: no
 * matrix helpers, every output element is one flat sum over all summation
 * indices of products of scalar tensor entries, with its own index arithmetic.
 * Readings R1-R19 as in oracle.c.
 *   Σ^X[kz][e][a][x][y] = scale Σ_{s,qz,m,±,i,j,u,v} c^±_{ij} dH[a][s][i][x][u] G^X[k'][e∓s_m][b][u][v] dH[b][r][j][v][y]
 *   Π^X[qz][m][a][s+1][i][j] = scale Σ_{kz,e,x,y,u,v} dH[b][r][i][x][y] G^X[k2][e+s_m][a][y][u] dH[a][s][j][u][v] G^Y[kz][e][b][v][x]
 */
#include <stdint.h>

typedef struct {
  int64_t Na, Nb, Norb, NE, Nw, Nkz, Nqz;
  int64_t shift0, shift_step;
} br_dims;

#define RE(p, f) ((p)[2 * (f)])
#define IM(p, f) ((p)[2 * (f) + 1])

static int64_t g_idx(const br_dims* d, int64_t k, int64_t e, int64_t a, int64_t u, int64_t v) {
  return (((k * d->NE + e) * d->Na + a) * d->Norb + u) * d->Norb + v;
}
static int64_t d_idx(const br_dims* d, int64_t q, int64_t m, int64_t a, int64_t slot, int64_t i, int64_t j) {
  return ((((q * d->Nw + m) * d->Na + a) * (d->Nb + 1) + slot) * 3 + i) * 3 + j;
}
static int64_t h_idx(const br_dims* d, int64_t a, int64_t s, int64_t i, int64_t x, int64_t y) {
  return (((a * d->Nb + s) * 3 + i) * d->Norb + x) * d->Norb + y;
}
static int64_t wrap(int64_t x, int64_t n) { while (x < 0) x += n; while (x >= n) x -= n; return x; }

void brute_sigma(const br_dims* d, const int32_t* nbr, const double* dH, const double* GL, const double* GG,
                 const double* DL, const double* DG, double sre, double sim, double* SL, double* SG) {
  const int64_t n = d->Norb;
  for (int X = 0; X < 2; ++X) {
    const double* G = X ? GG : GL;
    const double* Dm = X ? DG : DL;   /* D used with E - ħω */
    const double* Dp = X ? DL : DG;   /* D used (transposed) with E + ħω */
    double* S = X ? SG : SL;
    for (int64_t kz = 0; kz < d->Nkz; ++kz)
      for (int64_t e = 0; e < d->NE; ++e)
        for (int64_t a = 0; a < d->Na; ++a)
          for (int64_t x = 0; x < n; ++x)
            for (int64_t y = 0; y < n; ++y) {
              long double ar = 0, ai = 0;
              for (int64_t s = 0; s < d->Nb; ++s) {
                int64_t b = nbr[a * d->Nb + s];
                if (b < 0) continue;
                int64_t r = -1;
                for (int64_t t = 0; t < d->Nb; ++t) if (nbr[b * d->Nb + t] == a) r = t;
                for (int64_t qz = 0; qz < d->Nqz; ++qz)
                  for (int64_t m = 0; m < d->Nw; ++m)
                    for (int pm = -1; pm <= 1; pm += 2) {
                      int64_t ep = e + pm * (d->shift0 + m * d->shift_step);
                      if (ep < 0 || ep >= d->NE) continue;
                      int64_t kp = wrap(kz - qz + d->Nkz / 2, d->Nkz);
                      const double* Dq = pm < 0 ? Dm : Dp;
                      for (int64_t i = 0; i < 3; ++i)
                        for (int64_t j = 0; j < 3; ++j) {
                          int64_t ii = pm < 0 ? i : j, jj = pm < 0 ? j : i;
                          double cr = RE(Dq, d_idx(d, qz, m, b, r + 1, ii, jj)) - RE(Dq, d_idx(d, qz, m, b, 0, ii, jj)) -
                                      RE(Dq, d_idx(d, qz, m, a, 0, ii, jj)) + RE(Dq, d_idx(d, qz, m, a, s + 1, ii, jj));
                          double ci = IM(Dq, d_idx(d, qz, m, b, r + 1, ii, jj)) - IM(Dq, d_idx(d, qz, m, b, 0, ii, jj)) -
                                      IM(Dq, d_idx(d, qz, m, a, 0, ii, jj)) + IM(Dq, d_idx(d, qz, m, a, s + 1, ii, jj));
                          for (int64_t u = 0; u < n; ++u)
                            for (int64_t v = 0; v < n; ++v) {
                              int64_t f1 = h_idx(d, a, s, i, x, u), f2 = g_idx(d, kp, ep, b, u, v),
                                      f3 = h_idx(d, b, r, j, v, y);
                              long double h1r = RE(dH, f1), h1i = IM(dH, f1), gr = RE(G, f2), gi = IM(G, f2),
                                          h3r = RE(dH, f3), h3i = IM(dH, f3);
                              long double pr = h1r * gr - h1i * gi, pi = h1r * gi + h1i * gr;
                              long double qr = pr * h3r - pi * h3i, qi = pr * h3i + pi * h3r;
                              ar += cr * qr - ci * qi;
                              ai += cr * qi + ci * qr;
                            }
                        }
                    }
              }
              int64_t f = g_idx(d, kz, e, a, x, y);
              RE(S, f) = (double)(sre * ar - sim * ai);
              IM(S, f) = (double)(sre * ai + sim * ar);
            }
  }
}

void brute_pi(const br_dims* d, const int32_t* nbr, const double* dH, const double* GL, const double* GG, double sre,
              double sim, double* PL, double* PG) {
  const int64_t n = d->Norb;
  for (int X = 0; X < 2; ++X) {
    const double* GX = X ? GG : GL;
    const double* GY = X ? GL : GG;
    double* P = X ? PG : PL;
    for (int64_t qz = 0; qz < d->Nqz; ++qz)
      for (int64_t m = 0; m < d->Nw; ++m)
        for (int64_t a = 0; a < d->Na; ++a) {
          long double self_r[9] = {0}, self_i[9] = {0};
          for (int64_t s = 0; s < d->Nb; ++s) {
            int64_t b = nbr[a * d->Nb + s];
            for (int64_t i = 0; i < 3; ++i)
              for (int64_t j = 0; j < 3; ++j) {
                long double ar = 0, ai = 0;
                if (b >= 0) {
                  int64_t r = -1;
                  for (int64_t t = 0; t < d->Nb; ++t) if (nbr[b * d->Nb + t] == a) r = t;
                  for (int64_t kz = 0; kz < d->Nkz; ++kz) {
                    int64_t k2 = wrap(kz + qz - d->Nkz / 2, d->Nkz);
                    for (int64_t e = 0; e < d->NE; ++e) {
                      int64_t e2 = e + d->shift0 + m * d->shift_step;
                      if (e2 >= d->NE) continue;
                      for (int64_t x = 0; x < n; ++x)
                        for (int64_t y = 0; y < n; ++y)
                          for (int64_t u = 0; u < n; ++u)
                            for (int64_t v = 0; v < n; ++v) {
                              int64_t f1 = h_idx(d, b, r, i, x, y), f2 = g_idx(d, k2, e2, a, y, u),
                                      f3 = h_idx(d, a, s, j, u, v), f4 = g_idx(d, kz, e, b, v, x);
                              long double p1r = RE(dH, f1), p1i = IM(dH, f1);
                              long double p2r = p1r * RE(GX, f2) - p1i * IM(GX, f2), p2i = p1r * IM(GX, f2) + p1i * RE(GX, f2);
                              long double p3r = p2r * RE(dH, f3) - p2i * IM(dH, f3), p3i = p2r * IM(dH, f3) + p2i * RE(dH, f3);
                              ar += p3r * RE(GY, f4) - p3i * IM(GY, f4);
                              ai += p3r * IM(GY, f4) + p3i * RE(GY, f4);
                            }
                    }
                  }
                }
                int64_t f = d_idx(d, qz, m, a, s + 1, i, j);
                RE(P, f) = (double)(sre * ar - sim * ai);
                IM(P, f) = (double)(sre * ai + sim * ar);
                self_r[i * 3 + j] += ar;
                self_i[i * 3 + j] += ai;
              }
          }
          for (int t = 0; t < 9; ++t) {
            int64_t f = d_idx(d, qz, m, a, 0, t / 3, t % 3);
            RE(P, f) = (double)(sre * self_r[t] - sim * self_i[t]);
            IM(P, f) = (double)(sre * self_i[t] + sim * self_r[t]);
          }
        }
  }
}
