// gen_dev.cu — device implementation of include/qt_gen.h (same counter-based
// generator as gen_host.c, written separately; tests check bit-for-bit equality).
// Input generation only: no SSE arithmetic here. One thread per complex element.
#include "qt_gen.h"
#include <cuda_runtime.h>

namespace {
__device__ __forceinline__ uint64_t sm64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double draw(uint64_t seed, int id, int mode, uint64_t idx) {
  uint64_t z = sm64(seed ^ ((uint64_t)id * 0x9E3779B97F4A7C15ULL) ^ idx);
  if (mode == QTGEN_INTEGER) return (double)(int64_t)(z % 5ULL) - 2.0;
  return __dmul_rn(__dmul_rn((double)(z >> 11), 0x1.0p-53), 2.0) - 1.0;
}
__device__ __forceinline__ int rev_slot(const int32_t* nbr, int64_t Nb, int64_t b, int64_t a) {
  for (int64_t t = 0; t < Nb; ++t) if (nbr[b * Nb + t] == (int32_t)a) return (int)t;
  return -1;
}

// PHYSICAL envelope (see qt_gen.h); same expressions as gen_host.c, every operation explicitly rounded
__device__ __forceinline__ double occupation(int id, int64_t e, int64_t NE) {
  const int t = (int)((40 * e) / NE) - 20;
  return __ddiv_rn(1.0, __dadd_rn(1.0, ldexp(1.0, id == QTGEN_ID_GL ? t : -t)));
}
__device__ __forceinline__ double shell_scale(int64_t slot) {
  return slot < 4 ? 1.0 : slot < 16 ? 0.3 : slot < 28 ? 0.1 : 0.03;
}

__global__ void k_gen_G(uint64_t seed, int id, int mode, int64_t NE, int64_t Na, int64_t Norb,
                        int64_t e_lo, int64_t ne, int64_t a_lo, int64_t na, int64_t total, double2* out) {
  const int64_t nn = Norb * Norb;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t rc = t % nn, blk = t / nn;
    int64_t a = a_lo + blk % na, e = e_lo + (blk / na) % ne, k = blk / (na * ne);
    if (mode == QTGEN_ZERO) { out[t] = make_double2(0.0, 0.0); continue; }
    int64_t r = rc / Norb, c = rc % Norb;
    uint64_t base = (uint64_t)(((k * NE + e) * Na + a) * nn);
    if (mode == QTGEN_PHYSICAL) {
      double are = 0.0, aim = 0.0;
      for (int64_t kk = 0; kk < Norb; ++kk) {
        uint64_t fx = base + (uint64_t)(r * Norb + kk), fy = base + (uint64_t)(c * Norb + kk);
        double xr = draw(seed, QTGEN_ID_GL, QTGEN_RANDOM, 2 * fx), xi = draw(seed, QTGEN_ID_GL, QTGEN_RANDOM, 2 * fx + 1);
        double yr = draw(seed, QTGEN_ID_GL, QTGEN_RANDOM, 2 * fy), yi = draw(seed, QTGEN_ID_GL, QTGEN_RANDOM, 2 * fy + 1);
        are = __dadd_rn(are, __dadd_rn(__dmul_rn(xr, yr), __dmul_rn(xi, yi)));
        aim = __dadd_rn(aim, __dsub_rn(__dmul_rn(xi, yr), __dmul_rn(xr, yi)));
      }
      are = __ddiv_rn(are, (double)Norb);
      aim = __ddiv_rn(aim, (double)Norb);
      const double occ = occupation(id, e, NE);
      out[t] = id == QTGEN_ID_GL ? make_double2(-__dmul_rn(occ, aim), __dmul_rn(occ, are))
                                 : make_double2(__dmul_rn(occ, aim), -__dmul_rn(occ, are));
      continue;
    }
    uint64_t f_rc = base + (uint64_t)(r * Norb + c), f_cr = base + (uint64_t)(c * Norb + r);
    double xr_rc = draw(seed, id, mode, 2 * f_rc), xi_rc = draw(seed, id, mode, 2 * f_rc + 1);
    double xr_cr = draw(seed, id, mode, 2 * f_cr), xi_cr = draw(seed, id, mode, 2 * f_cr + 1);
    out[t] = make_double2(__dmul_rn(__dsub_rn(xr_rc, xr_cr), 0.5), __dmul_rn(__dadd_rn(xi_rc, xi_cr), 0.5));
  }
}

__global__ void k_gen_D(uint64_t seed, int id, int mode, int64_t Nqz, int64_t Nw, int64_t Na, int64_t Nb,
                        const int32_t* nbr, int64_t delta_m, int64_t a_lo, int64_t na, int64_t total, double2* out) {
  const int64_t ns = Nb + 1, h = Nqz / 2;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t ij = t % 9, q = t / 9;
    int64_t slot = q % ns, t1 = q / ns, a = a_lo + t1 % na, t2 = t1 / na, m = t2 % Nw, qz = t2 / Nw;
    int64_t i = ij / 3, j = ij % 3;
    double2 v = make_double2(0.0, 0.0);
    if (mode == QTGEN_ZERO) {
    } else if (mode == QTGEN_DELTA) {
      if (slot > 0 && nbr[a * Nb + slot - 1] >= 0 && qz == h && m == delta_m && i == j) v.x = 0.5;
    } else if (slot == 0) {
      uint64_t base = (uint64_t)((((qz * Nw + m) * Na + a) * ns + 0) * 9);
      uint64_t fij = base + i * 3 + j, fji = base + j * 3 + i;
      v.x = __dmul_rn(__dsub_rn(draw(seed, id, mode, 2 * fij), draw(seed, id, mode, 2 * fji)), 0.5);
      v.y = __dmul_rn(__dadd_rn(draw(seed, id, mode, 2 * fij + 1), draw(seed, id, mode, 2 * fji + 1)), 0.5);
    } else {
      int64_t b = nbr[a * Nb + slot - 1];
      if (b >= 0) {
        if (a < b) {
          uint64_t f = (uint64_t)((((qz * Nw + m) * Na + a) * ns + slot) * 9) + ij;
          v.x = draw(seed, id, mode, 2 * f); v.y = draw(seed, id, mode, 2 * f + 1);
        } else {
          int r = rev_slot(nbr, Nb, b, a);
          uint64_t f = (uint64_t)((((qz * Nw + m) * Na + b) * ns + (r + 1)) * 9) + j * 3 + i;
          v.x = -draw(seed, id, mode, 2 * f); v.y = draw(seed, id, mode, 2 * f + 1);
        }
      }
    }
    out[t] = v;
  }
}

__global__ void k_gen_dH(uint64_t seed, int id, int mode, int64_t Na, int64_t Nb, int64_t Norb,
                         const int32_t* nbr, int64_t total, double2* out) {
  const int64_t nn = Norb * Norb;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t xy = t % nn, q = t / nn;
    int64_t i = q % 3, s = (q / 3) % Nb, a = q / (3 * Nb);
    int64_t x = xy / Norb, y = xy % Norb;
    double2 v = make_double2(0.0, 0.0);
    int64_t b = nbr[a * Nb + s];
    if (mode != QTGEN_ZERO && b >= 0) {
      if (a < b) {
        uint64_t f = (uint64_t)(((a * Nb + s) * 3 + i) * nn) + xy;
        const double sc = mode == QTGEN_PHYSICAL ? shell_scale(s) : 1.0;
        v.x = __dmul_rn(sc, draw(seed, id, mode, 2 * f)); v.y = __dmul_rn(sc, draw(seed, id, mode, 2 * f + 1));
      } else {
        int r = rev_slot(nbr, Nb, b, a);
        uint64_t f = (uint64_t)(((b * Nb + r) * 3 + i) * nn) + y * Norb + x;
        const double sc = mode == QTGEN_PHYSICAL ? shell_scale(r) : 1.0;
        v.x = __dmul_rn(sc, draw(seed, id, mode, 2 * f)); v.y = -__dmul_rn(sc, draw(seed, id, mode, 2 * f + 1));
      }
    }
    out[t] = v;
  }
}

inline int grid_for(int64_t total) {
  int64_t g = (total + 255) / 256;
  return (int)(g > 148 * 64 ? 148 * 64 : (g < 1 ? 1 : g));
}
}  // namespace

extern "C" int qtgen_dev_G(uint64_t seed, int id, int mode, int64_t Nkz, int64_t NE, int64_t Na, int64_t Norb,
                           int64_t e_lo, int64_t e_hi, int64_t a_lo, int64_t a_hi, double* out, void* stream) {
  int64_t total = Nkz * (e_hi - e_lo) * (a_hi - a_lo) * Norb * Norb;
  if (total <= 0) return 0;
  k_gen_G<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>(seed, id, mode, NE, Na, Norb, e_lo, e_hi - e_lo, a_lo,
                                                             a_hi - a_lo, total, (double2*)out);
  return (int)cudaGetLastError();
}
extern "C" int qtgen_dev_D(uint64_t seed, int id, int mode, int64_t Nqz, int64_t Nw, int64_t Na, int64_t Nb,
                           const int32_t* nbr_dev, int64_t delta_m, int64_t a_lo, int64_t a_hi, double* out, void* stream) {
  int64_t total = Nqz * Nw * (a_hi - a_lo) * (Nb + 1) * 9;
  if (total <= 0) return 0;
  k_gen_D<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>(seed, id, mode, Nqz, Nw, Na, Nb, nbr_dev, delta_m, a_lo,
                                                             a_hi - a_lo, total, (double2*)out);
  return (int)cudaGetLastError();
}
extern "C" int qtgen_dev_dH(uint64_t seed, int id, int mode, int64_t Na, int64_t Nb, int64_t Norb,
                            const int32_t* nbr_dev, double* out, void* stream) {
  int64_t total = Na * Nb * 3 * Norb * Norb;
  if (total <= 0) return 0;
  k_gen_dH<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>(seed, id, mode, Na, Nb, Norb, nbr_dev, total,
                                                              (double2*)out);
  return (int)cudaGetLastError();
}
