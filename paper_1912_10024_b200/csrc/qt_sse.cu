// qt_sse.cu — C ABI of libqtsse.so (include/qt_sse.h): plan validation, the Ta x TE rank grid, work lists,
// workspace, halo exchange and Π reduction scheduling, and the stream-ordered kernel sequence for Σ≷ (Eq. 3,
// PAPER.md P:355-365) and Π≷ (Eq. 4).
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <atomic>
#include <cstring>
#include <new>
#include <vector>

#include "common.cuh"
#include "qt_sse.h"
#include "halo.cuh"

#include "kernels_decl.cuh"

#ifndef QT_SIG_PAIR
#define QT_SIG_PAIR 1
#endif
// smallest item (pairs) the energy-pair kernel takes in pair mode; 1 = every item (its multi-energy-pair tiles
// for items of 1..3 pairs), 4 = items of 1..3 pairs on k_sigma's multi-energy tiles
#ifndef QT_PAIR_MIN
#define QT_PAIR_MIN 1
#endif
constexpr int kPairMinPairs = QT_PAIR_MIN;

using namespace qt;

static std::atomic<uint64_t> g_launches{0};
namespace qt {
void count_launches(uint64_t n) { g_launches.fetch_add(n); }   // the RGF solver's own kernels (rgf.cu)
}

namespace {

// ---------------------------------------------------------------- host-only layout of one rank
// Everything a plan needs that does not touch the device: the rank's place in the Ta x TE grid (the paper's
// Ta x TE tiling), its owned atoms/energies and input windows, the work lists, the workspace chunks,
// the halo boxes per peer and the footprint. Built identically by qt_sse_plan and the host-only queries.
struct Geom {
  int Ta = 1, TE = 1, ta = 0, te = 0;
  int64_t a_lo = 0, a_hi = 0, w_lo = 0, w_hi = 0;   // owned atoms, atom window
  int64_t e_lo = 0, e_hi = 0, ew_lo = 0, ew_hi = 0; // owned energies, energy window
  int64_t pa_lo = 0, pa_hi = 0;                     // Π output atoms
};

struct PiGroup {            // Π output group: atoms [lo, hi) of the owned slab
  int64_t lo = 0, hi = 0;
  int root = -1;            // TE-communicator rank receiving the reduced group (-1: written in place)
  std::vector<int64_t> chunks;   // item bounds
};

struct SigChunk {
  int64_t i0 = 0, i1 = 0;
  int64_t det_off = 0, det_n = 0;   // QT_FLAG_DETERMINISTIC: the chunk's destination-atom entries
  int64_t nfull = 0;                 // leading items of >= 4 pairs (k_sigma_pair in pair mode)
  bool coef_halo = false;   // the coefficient tables read D of halo atoms
  bool g_halo = false;      // the contraction reads G entries of the halo
};

struct Layout {
  qt_sse_desc d{};
  Geom g;
  int64_t NN = 0, h = 0, Dmax = 0, Dwin = 0, DWp = 0, NWv = 0, NWP = 0;
  int64_t Nwin = 0, Nout = 0, NEw = 0, NEo = 0, E0 = 0;
  bool fp32 = false, sig_tma = true, reduce = false;
  bool sig_pair_mode = false;   // items of >= 4 pairs on the energy-pair contraction (k_sigma_pair)
  std::vector<int32_t> nbr_win;
  std::vector<SigItem> sig_items;
  std::vector<SigPair> sig_pairs;
  std::vector<int32_t> sig_pair_item;
  std::vector<PiItem> pi_items;
  std::vector<PiPair> pi_pairs;
  std::vector<int32_t> pi_pair_item;
  std::vector<SigChunk> sig_chunks;
  bool det = false;
  std::vector<int4> det_atoms;   // {a_out, first pair entry, count, 0}
  std::vector<int2> det_pairs;   // {chunk-relative item, pair in item}
  std::vector<PiGroup> groups;
  int64_t n_interior_items = 0;
  int64_t sig_rows = kRows, ndc = 0, NNp = 0, Epad = 0, NEp = 0, Kp = 0;
  int64_t gt_ld = 0;   // Gt scratch row stride (elements)
  int64_t sig_ec = 0, pi_ec = 0;   // energies per Σ / Π scratch sub-range (= NEo unless the workspace is small)
  size_t ws_bytes = 0, gt_offset = 0, part_bytes = 0;
  std::vector<HaloPeer> peers;
  size_t send_total = 0, recv_total = 0;
  double flops[4] = {0, 0, 0, 0};
  double npairs = 0;
  size_t gs_elems() const { return (size_t)d.Nkz * NEw * Nwin * ((NN + 1) & ~int64_t(1)); }
  size_t gtp_elems() const { return (size_t)Nwin * d.Nkz * 4 * kTcRowsA * NEp; }
  size_t gpi_elems() const { return (size_t)Nwin * d.Nkz * 4 * Epad * NNp; }
  double halo_recv = 0, reduce_bytes = 0;
};

qt_status validate_desc(const qt_sse_desc* d) {
  if (!d) return QT_ERR_INVALID_ARG;
  if (d->Na <= 0 || d->Nb <= 0 || d->Norb <= 0 || d->NE <= 0 || d->Nw <= 0 || d->Nkz <= 0 || d->Nqz <= 0)
    return QT_ERR_INVALID_ARG;
  if (d->N3D != 3 || d->Nkz != d->Nqz) return QT_ERR_INVALID_ARG;
  if (d->shift0 < 1 || d->shift_step < 1) return QT_ERR_INVALID_ARG;     // S:287 grid alignment
  if (d->Na > (1LL << 30) || d->Nb > 4096 || d->NE > (1LL << 24)) return QT_ERR_INVALID_ARG;
  if (d->nranks < 1 || d->rank < 0 || d->rank >= d->nranks) return QT_ERR_INVALID_ARG;
  if (d->shard == QT_SHARD_2D && (d->grid_atoms < 1 || d->nranks % d->grid_atoms != 0)) return QT_ERR_INVALID_ARG;
  if (d->flags & ~QT_FLAG_DETERMINISTIC) return QT_ERR_INVALID_ARG;
  if (d->precision != QT_PREC_FP64 && d->precision != QT_PREC_FP32_MIXED) return QT_ERR_UNSUPPORTED;
  const int64_t nwv = (d->Nw - 1) * d->shift_step + 1;   // Π columns: every shift between s_0 and s_{Nω-1}
  if (d->precision == QT_PREC_FP32_MIXED && (d->Norb > 10 || nwv > 80))   // UMMA M = Norb² <= 128, N <= 80
    return QT_ERR_UNSUPPORTED;
  if (d->Norb > 12 || nwv > 128) return QT_ERR_UNSUPPORTED;
  if (d->nranks > 1 && d->shard == QT_SHARD_NONE) return QT_ERR_UNSUPPORTED;
  return QT_OK;
}

// neighbour table: in range, no self, no duplicates, symmetric
qt_status validate_nbr(const qt_sse_desc* d, const int32_t* nbr) {
  if (!nbr) return QT_ERR_INVALID_ARG;
  const int64_t Na = d->Na, Nb = d->Nb;
  for (int64_t a = 0; a < Na; ++a)
    for (int64_t s = 0; s < Nb; ++s) {
      int32_t b = nbr[a * Nb + s];
      if (b < -1 || b >= Na || b == a) return QT_ERR_INVALID_ARG;
      if (b < 0) continue;
      int cnt = 0, back = 0;
      for (int64_t t = 0; t < Nb; ++t) {
        if (nbr[a * Nb + t] == b) ++cnt;
        if (nbr[(int64_t)b * Nb + t] == a) ++back;
      }
      if (cnt != 1 || back != 1) return QT_ERR_INVALID_ARG;
    }
  return QT_OK;
}

int64_t rev_slot(const int32_t* nbr, int64_t Nb, int64_t b, int64_t a) {
  for (int64_t t = 0; t < Nb; ++t)
    if (nbr[b * Nb + t] == a) return t;
  return -1;
}

int64_t shift_of(const qt_sse_desc* d, int64_t m) { return d->shift0 + m * d->shift_step; }

// valid (E, m) counts over output energies [e_lo, e_hi): V- = #{E - s_m >= 0}, V+ = #{E + s_m < NE}
void window_counts(const qt_sse_desc* d, double* vm, double* vp, int64_t e_lo, int64_t e_hi) {
  double a = 0, b = 0;
  for (int64_t e = e_lo; e < e_hi; ++e)
    for (int64_t m = 0; m < d->Nw; ++m) {
      const int64_t sm = shift_of(d, m);
      if (e - sm >= 0) a += 1;
      if (e + sm < d->NE) b += 1;
    }
  *vm = a;
  *vp = b;
}

// algorithmic flops of the output energies [e_lo, e_hi) for npairs valid pairs (SURVEY §8(d) F_alg)
void count_flops(const qt_sse_desc* d, double npairs, double out[4], int64_t e_lo, int64_t e_hi) {
  double vm, vp;
  window_counts(d, &vm, &vp, e_lo, e_hi);
  const double NN = (double)d->Norb * d->Norb, No3 = NN * d->Norb;
  out[0] = 2.0 * d->Nkz * d->Nqz * npairs * (vm + vp) * 9.0 * NN * 8.0;
  out[1] = 2.0 * d->Nkz * (double)(e_hi - e_lo) * npairs * 12.0 * No3 * 8.0;
  out[2] = out[1];
  out[3] = 2.0 * d->Nkz * d->Nqz * npairs * vp * 9.0 * NN * 8.0;
}

// cut a cumulative weight table into n contiguous ranges; range k
void cut_range(const std::vector<double>& cum, int n, int k, int64_t* lo, int64_t* hi) {
  const int64_t N = (int64_t)cum.size() - 1;
  auto cut = [&](int j) -> int64_t {
    const double target = cum[N] * j / n;
    return (int64_t)(std::lower_bound(cum.begin(), cum.end(), target) - cum.begin());
  };
  *lo = k == 0 ? 0 : cut(k);
  *hi = k == n - 1 ? N : cut(k + 1);
  if (*hi < *lo) *hi = *lo;
}

// atom slab k of n over [lo0, hi0): contiguous, balanced by valid-pair count (+1 per atom)
void atom_slab(const qt_sse_desc* d, const int32_t* nbr, int64_t lo0, int64_t hi0, int n, int k, int64_t* lo,
               int64_t* hi) {
  std::vector<double> cum(hi0 - lo0 + 1, 0.0);
  for (int64_t a = lo0; a < hi0; ++a) {
    int c = 0;
    for (int64_t s = 0; s < d->Nb; ++s) c += nbr[a * d->Nb + s] >= 0;
    cum[a - lo0 + 1] = cum[a - lo0] + c + 1;
  }
  cut_range(cum, n, k, lo, hi);
  *lo += lo0;
  *hi += lo0;
}

// energy slab k of n (the paper's T_E tiling), balanced by the Σ/Π work per energy (valid shifts +
// sandwich); its input window is [lo - Dmax, hi + Dmax) ∩ [0, NE)
void energy_slab(const qt_sse_desc* d, int n, int k, int64_t* lo, int64_t* hi, int64_t* wlo, int64_t* whi) {
  std::vector<double> cum(d->NE + 1, 0.0);
  const int64_t Dmax = shift_of(d, d->Nw - 1);
  for (int64_t e = 0; e < d->NE; ++e) {
    double w = 1.0;
    for (int64_t m = 0; m < d->Nw; ++m) {
      const int64_t sm = shift_of(d, m);
      w += (e - sm >= 0) + 2.0 * (e + sm < d->NE);   // Σ absorption + emission, Π correlation
    }
    cum[e + 1] = cum[e] + w;
  }
  cut_range(cum, n, k, lo, hi);
  *wlo = std::max<int64_t>(0, *lo - Dmax);
  *whi = std::min<int64_t>(d->NE, *hi + Dmax);
}

void grid_of(const qt_sse_desc* d, int* Ta, int* TE) {
  if (d->nranks == 1) {
    *Ta = *TE = 1;
  } else if (d->shard == QT_SHARD_ENERGY) {
    *Ta = 1;
    *TE = d->nranks;
  } else if (d->shard == QT_SHARD_2D) {
    *Ta = d->grid_atoms;
    *TE = d->nranks / d->grid_atoms;
  } else {
    *Ta = d->nranks;
    *TE = 1;
  }
}

// geometry of rank r; `reduce` = the Π partial sums are reduced to sub-slab owners (communicator, TE > 1)
Geom geom_of(const qt_sse_desc* d, const int32_t* nbr, int r, bool reduce) {
  Geom g;
  grid_of(d, &g.Ta, &g.TE);
  g.ta = r / g.TE;
  g.te = r % g.TE;
  atom_slab(d, nbr, 0, d->Na, g.Ta, g.ta, &g.a_lo, &g.a_hi);
  g.w_lo = g.a_lo;
  g.w_hi = g.a_hi;
  for (int64_t a = g.a_lo; a < g.a_hi; ++a)
    for (int64_t s = 0; s < d->Nb; ++s) {
      const int32_t b = nbr[a * d->Nb + s];
      if (b < 0) continue;
      g.w_lo = std::min<int64_t>(g.w_lo, b);
      g.w_hi = std::max<int64_t>(g.w_hi, b + 1);
    }
  energy_slab(d, g.TE, g.te, &g.e_lo, &g.e_hi, &g.ew_lo, &g.ew_hi);
  if (reduce && g.TE > 1) {
    atom_slab(d, nbr, g.a_lo, g.a_hi, g.TE, g.te, &g.pa_lo, &g.pa_hi);
  } else {
    g.pa_lo = g.a_lo;
    g.pa_hi = g.a_hi;
  }
  return g;
}

size_t d_block_bytes(const qt_sse_desc& d) { return (size_t)d.Nqz * d.Nw * (d.Nb + 1) * 9 * 16; }   // per atom

// Builds everything host-side for `rank` (reduce: a communicator will exist).
qt_status build_layout(const qt_sse_desc* desc, const int32_t* nbr, bool reduce, size_t ws_budget, Layout* L,
                       bool strict = true) {
  L->d = *desc;
  const qt_sse_desc& d = L->d;
  L->NN = d.Norb * d.Norb;
  L->h = d.Nkz / 2;
  L->Dmax = shift_of(&d, d.Nw - 1);
  L->Dwin = 2 * L->Dmax + 1;
  L->DWp = (L->Dwin + 3) & ~3LL;
  L->NWv = (d.Nw - 1) * d.shift_step + 1;
  L->NWP = (L->NWv + 7) & ~7LL;
  L->fp32 = d.precision == QT_PREC_FP32_MIXED;
  L->g = geom_of(&d, nbr, d.rank, reduce);
  const Geom& g = L->g;
  // Σ sandwich: the warp-per-energy kernel needs 3·Norb <= 32 lanes; Norb 11, 12 (and QT_FLAG_DETERMINISTIC) use the
  // destination-ordered kernel, whose per-chunk destination lists are built below
  L->det = (d.flags & QT_FLAG_DETERMINISTIC) != 0 || d.Norb > 10;
  L->reduce = reduce && g.TE > 1;
  L->Nwin = g.w_hi - g.w_lo;
  L->Nout = g.a_hi - g.a_lo;
  L->NEw = g.ew_hi - g.ew_lo;
  L->NEo = g.e_hi - g.e_lo;
  L->E0 = g.e_lo - g.ew_lo;
  L->nbr_win.assign(L->Nwin * d.Nb, -1);
  for (int64_t a = g.w_lo; a < g.w_hi; ++a)
    for (int64_t s = 0; s < d.Nb; ++s) {
      int32_t b = nbr[a * d.Nb + s];
      if (b >= g.w_lo && b < g.w_hi) L->nbr_win[(a - g.w_lo) * d.Nb + s] = (int32_t)(b - g.w_lo);
    }

  // Σ work list: source-organized. For each source atom b, its reverse pairs (a,s) with a owned; interior
  // sources (b owned: no halo read in the contraction or the coefficient tables) first, then halo sources.
  const size_t scap = L->fp32 ? kTcPiPairs : kMaxPairs;   // 126 / 72 GEMM rows
  auto add_source = [&](int64_t b) {
    std::vector<SigPair> mine;
    for (int64_t r = 0; r < d.Nb; ++r) {
      int32_t a = nbr[b * d.Nb + r];
      if (a < 0 || a < g.a_lo || a >= g.a_hi) continue;
      SigPair q;
      q.a = (int32_t)(a - g.a_lo);
      q.a_in = (int32_t)(a - g.w_lo);
      q.s = (int32_t)rev_slot(nbr, d.Nb, a, b);
      q.r = (int32_t)r;
      mine.push_back(q);
    }
    for (size_t k = 0; k < mine.size(); k += scap) {
      SigItem it;
      it.b_in = (int32_t)(b - g.w_lo);
      it.b = (int32_t)b;
      it.npair = (int32_t)std::min<size_t>(scap, mine.size() - k);
      it.pair0 = (int32_t)L->sig_pairs.size();
      for (int t = 0; t < it.npair; ++t) {
        L->sig_pairs.push_back(mine[k + t]);
        L->sig_pair_item.push_back((int32_t)L->sig_items.size());
      }
      L->sig_items.push_back(it);
    }
  };
  for (int64_t b = g.a_lo; b < g.a_hi; ++b) add_source(b);
  L->n_interior_items = (int64_t)L->sig_items.size();
  for (int64_t b = g.w_lo; b < g.w_hi; ++b)
    if (b < g.a_lo || b >= g.a_hi) add_source(b);
  // Within the interior and the halo sources, items of >= 4 pairs first (full-height tiles before the
  // multi-energy-pair tiles of the small items; with QT_PAIR_MIN = 4 the small items run k_sigma instead), then
  // the pair list rebuilt in item order so every chunk's pairs stay contiguous.
  L->sig_pair_mode = !L->fp32 && sigma_pair_supported((int)d.Norb) && QT_SIG_PAIR;
  if (L->sig_pair_mode) {
    auto full_first = [](const SigItem& x) { return x.npair >= 4; };
    std::stable_partition(L->sig_items.begin(), L->sig_items.begin() + L->n_interior_items, full_first);
    std::stable_partition(L->sig_items.begin() + L->n_interior_items, L->sig_items.end(), full_first);
    std::vector<SigPair> pairs;
    std::vector<int32_t> pair_item;
    pairs.reserve(L->sig_pairs.size());
    for (size_t i = 0; i < L->sig_items.size(); ++i) {
      SigItem& it = L->sig_items[i];
      const int32_t p0 = (int32_t)pairs.size();
      for (int t = 0; t < it.npair; ++t) {
        pairs.push_back(L->sig_pairs[it.pair0 + t]);
        pair_item.push_back((int32_t)i);
      }
      it.pair0 = p0;
    }
    L->sig_pairs.swap(pairs);
    L->sig_pair_item.swap(pair_item);
  }

  // Π groups: one per output owner (sub-slabs of the owned atoms when the partial sums are reduced)
  if (L->reduce) {
    for (int j = 0; j < g.TE; ++j) {
      PiGroup G;
      atom_slab(&d, nbr, g.a_lo, g.a_hi, g.TE, j, &G.lo, &G.hi);
      G.root = j;
      L->groups.push_back(G);
    }
  } else {
    PiGroup G;
    G.lo = g.a_lo;
    G.hi = g.a_hi;
    L->groups.push_back(G);
  }
  // Π work list: destination-organized. For each owned atom a, its valid slots in items of <= 8 (14) pairs;
  // a_out is relative to the atom's group.
  std::vector<int64_t> group_item0;
  for (const PiGroup& G : L->groups) {
    group_item0.push_back((int64_t)L->pi_items.size());
    for (int64_t a = G.lo; a < G.hi; ++a) {
      std::vector<PiPair> mine;
      for (int64_t s = 0; s < d.Nb; ++s) {
        int32_t b = nbr[a * d.Nb + s];
        if (b < 0) continue;
        PiPair q;
        q.s = (int32_t)s;
        q.b_in = (int32_t)(b - g.w_lo);
        q.r = (int32_t)rev_slot(nbr, d.Nb, b, a);
        q.a_in = (int32_t)(a - g.w_lo);
        mine.push_back(q);
      }
      for (size_t k = 0; k < mine.size(); k += scap) {
        PiItem it;
        it.a_out = (int32_t)(a - G.lo);
        it.a_in = (int32_t)(a - g.w_lo);
        it.npair = (int32_t)std::min<size_t>(scap, mine.size() - k);
        it.pair0 = (int32_t)L->pi_pairs.size();
        for (int t = 0; t < it.npair; ++t) {
          L->pi_pairs.push_back(mine[k + t]);
          L->pi_pair_item.push_back((int32_t)L->pi_items.size());
        }
        L->pi_items.push_back(it);
      }
    }
  }
  group_item0.push_back((int64_t)L->pi_items.size());
  L->npairs = (double)L->pi_pairs.size();
  count_flops(&d, L->npairs, L->flops, g.e_lo, g.e_hi);

  // workspace (shared by the Σ coefficient tables + Gt scratch and the Π W scratch; calls are serialized)
  L->sig_rows = L->fp32 ? kTcRows : kRows;
  // Gt row stride = the Σ sandwich's padded shared-memory row (Norb² rounded to 16 bytes + 16 bytes), so one bulk
  // copy moves a pair's 9 rows of an energy into its ring slot with the bank-conflict padding in place
  L->gt_ld = L->fp32 ? ((L->NN + 1) & ~int64_t(1)) + 2 : L->NN + 1;
  const size_t gt_e = (size_t)d.Nkz * L->sig_rows * std::max<int64_t>((L->NN + 19) / 20 * 20, L->gt_ld) *
                      (L->fp32 ? sizeof(float2) : sizeof(double2));   // Gt (and Π W) scratch per item and energy
  L->NNp = (L->NN + 3) & ~int64_t(3);
  L->Epad = L->NEw + d.shift0 + 80 + 1;
  // W scratch of one item for ne energies (FP32: split planes with each kz row padded to whole 32-chunks)
  auto w_item = [&](int64_t ne) -> size_t {
    return L->fp32 ? (size_t)4 * kTcPiRows * d.Nkz * (((ne * L->NNp + 31) / 32) * 32) * sizeof(float) : gt_e * ne;
  };
  L->NEp = std::max<int64_t>(32, (L->NEw + 3) & ~int64_t(3));   // TMA boxes (32 wide) must lie inside the tensor
  L->Kp = (L->Dwin + 3 + 31) & ~int64_t(31);                      // delayed coefficient rows, whole 32-chunks
  L->sig_tma = true;   // every Norb <= 12 runs the TMA / mbarrier contraction
  L->ndc = (L->Dwin + 15) / 16;
  const size_t coef_item_t = L->fp32 ? (size_t)d.Nqz * 16 * kTcRows * L->Kp * sizeof(float)
                                     : (size_t)d.Nqz * L->ndc * kRows * kCoefKCP * sizeof(double2);
  const int64_t n_sig_items = (int64_t)L->sig_items.size(), n_pi_items = (int64_t)L->pi_items.size();
  const size_t need_min = coef_item_t + std::max(gt_e, w_item(1)) + 512;
  const size_t full = std::max((coef_item_t + gt_e * L->NEo) * n_sig_items + 512, w_item(L->NEo) * n_pi_items);
  size_t budget = std::max(ws_budget, need_min);
  L->ws_bytes = std::max<size_t>(std::min(budget, full), 256);
  // Enough parallel work per launch: >= 2 waves of k_pi_contract CTAs (one per item and qz) and of sandwich CTAs
  // (one per pair and kz). When the workspace cannot hold the scratch of that many items for all energies, the
  // chunks are split by energy as well (Σ outputs are disjoint per energy; Π sub-ranges accumulate).
  const int64_t waves = 2 * 148;
  const int64_t pairs_per_item = L->fp32 ? kTcPiPairs : kMaxPairs;
  const int64_t min_pi = std::min<int64_t>(std::max<int64_t>(1, n_pi_items), (waves + d.Nqz - 1) / d.Nqz);
  const int64_t min_sig = std::min<int64_t>(std::max<int64_t>(1, n_sig_items),
                                            (waves + d.Nkz * pairs_per_item - 1) / (d.Nkz * pairs_per_item));
  L->pi_ec = L->NEo;
  while (L->pi_ec > 1 && w_item(L->pi_ec) * min_pi > L->ws_bytes) L->pi_ec = (L->pi_ec + 1) / 2;
  L->sig_ec = L->NEo;
  while (L->sig_ec > 1 && (coef_item_t + gt_e * L->sig_ec) * min_sig + 512 > L->ws_bytes) L->sig_ec = (L->sig_ec + 1) / 2;

  // Π chunks inside each group (each chunk's W scratch for pi_ec energies fits the workspace)
  {
    const int64_t cap = std::max<int64_t>(1, (int64_t)(L->ws_bytes / w_item(L->pi_ec)));
    for (size_t gi = 0; gi < L->groups.size(); ++gi) {
      PiGroup& G = L->groups[gi];
      const int64_t i0 = group_item0[gi], i1 = group_item0[gi + 1];
      G.chunks.push_back(i0);
      for (int64_t i = i0 + cap; i < i1; i += cap) G.chunks.push_back(i);
      G.chunks.push_back(i1);
    }
    // Inside each chunk, items of more pairs first (k_pi_contract / sandwich CTAs are issued in item order: the
    // long CTAs start in the first waves and the short remainder items fill the tail), then the pair list rebuilt
    // in item order (each chunk's pairs stay one contiguous range).
    for (const PiGroup& G : L->groups)
      for (size_t k = 0; k + 1 < G.chunks.size(); ++k)
        std::stable_sort(L->pi_items.begin() + G.chunks[k], L->pi_items.begin() + G.chunks[k + 1],
                         [](const PiItem& x, const PiItem& y) { return x.npair > y.npair; });
    std::vector<PiPair> pairs;
    std::vector<int32_t> pair_item;
    pairs.reserve(L->pi_pairs.size());
    pair_item.reserve(L->pi_pairs.size());
    for (size_t i = 0; i < L->pi_items.size(); ++i) {
      PiItem& it = L->pi_items[i];
      const int32_t p0 = (int32_t)pairs.size();
      for (int t = 0; t < it.npair; ++t) {
        pairs.push_back(L->pi_pairs[it.pair0 + t]);
        pair_item.push_back((int32_t)i);
      }
      it.pair0 = p0;
    }
    L->pi_pairs.swap(pairs);
    L->pi_pair_item.swap(pair_item);
  }
  // Σ chunks: per item a tiled coefficient block [q][16-shift chunk][72][kCoefKCP] + its Gt scratch for sig_ec
  // energies. Workspace = [coef | Gt]. A chunk never mixes interior and halo sources.
  {
    const size_t gt_item = gt_e * L->sig_ec;
    size_t coef_acc = 0, gt_acc = 0, coef_max = 0;
    SigChunk c;
    c.i0 = 0;
    auto close = [&](int64_t i) {
      c.i1 = i;
      c.nfull = 0;
      if (L->sig_pair_mode)
        while (c.i0 + c.nfull < c.i1 && L->sig_items[c.i0 + c.nfull].npair >= kPairMinPairs) ++c.nfull;
      const bool halo_src = c.i0 >= L->n_interior_items;
      c.coef_halo = halo_src && g.Ta > 1;
      c.g_halo = halo_src || g.TE > 1;
      if (c.i1 > c.i0) L->sig_chunks.push_back(c);
      c.i0 = i;
      coef_max = std::max(coef_max, coef_acc);
      coef_acc = gt_acc = 0;
    };
    for (size_t i = 0; i < L->sig_items.size(); ++i) {
      const size_t cu = coef_item_t;
      if ((int64_t)i == L->n_interior_items && gt_acc + coef_acc > 0) close((int64_t)i);
      if (gt_acc > 0 && coef_acc + cu + gt_acc + gt_item + 256 > L->ws_bytes) close((int64_t)i);
      coef_acc += cu;
      gt_acc += gt_item;
    }
    close((int64_t)L->sig_items.size());
    L->gt_offset = (coef_max + 255) & ~size_t(255);
  }
  if (L->det) {   // per chunk: destination atoms (ascending) and their pairs in (item, slot) order
    for (SigChunk& c : L->sig_chunks) {
      std::vector<std::vector<int2>> by_atom(L->Nout);
      for (int64_t i = c.i0; i < c.i1; ++i) {
        const SigItem& it = L->sig_items[i];
        for (int t = 0; t < it.npair; ++t) by_atom[L->sig_pairs[it.pair0 + t].a].push_back(make_int2((int)(i - c.i0), t));
      }
      c.det_off = (int64_t)L->det_atoms.size();
      for (int64_t a = 0; a < L->Nout; ++a) {
        if (by_atom[a].empty()) continue;
        L->det_atoms.push_back(make_int4((int)a, (int)L->det_pairs.size(), (int)by_atom[a].size(), 0));
        L->det_pairs.insert(L->det_pairs.end(), by_atom[a].begin(), by_atom[a].end());
      }
      c.det_n = (int64_t)L->det_atoms.size() - c.det_off;
    }
  }
  if (L->reduce) {
    int64_t mx = 0;
    for (const PiGroup& G : L->groups) mx = std::max(mx, G.hi - G.lo);
    L->part_bytes = (size_t)mx * d_block_bytes(d);
    for (const PiGroup& G : L->groups)
      if (G.root != g.te) L->reduce_bytes += 2.0 * (double)(G.hi - G.lo) * d_block_bytes(d);
  }

  // halo boxes per peer: G≷ = (my window ∩ their owned block), D≷ (Ta > 1) from the peer of my energy row
  if (d.nranks > 1) {
    const size_t gb = (size_t)L->NN * 16, db = d_block_bytes(d) / (d.Nqz * d.Nw);   // per (kz,e,atom) / (q,m,atom)
    for (int r = 0; r < d.nranks; ++r) {
      if (r == d.rank) continue;
      const Geom o = geom_of(&d, nbr, r, reduce);
      HaloPeer hp;
      hp.rank = r;
      auto box = [](int64_t lo1, int64_t hi1, int64_t lo2, int64_t hi2, int64_t* lo, int64_t* n) {
        *lo = std::max(lo1, lo2);
        *n = std::max<int64_t>(0, std::min(hi1, hi2) - *lo);
      };
      int64_t ra0, rna, re0, rne, sa0, sna, se0, sne;
      box(g.w_lo, g.w_hi, o.a_lo, o.a_hi, &ra0, &rna);
      box(g.ew_lo, g.ew_hi, o.e_lo, o.e_hi, &re0, &rne);
      box(g.a_lo, g.a_hi, o.w_lo, o.w_hi, &sa0, &sna);
      box(g.e_lo, g.e_hi, o.ew_lo, o.ew_hi, &se0, &sne);
      if (rna && rne) {
        hp.recv_g = {re0 - g.ew_lo, rne, ra0 - g.w_lo, rna};
      }
      if (sna && sne) {
        hp.send_g = {se0 - g.ew_lo, sne, sa0 - g.w_lo, sna};
      }
      if (g.Ta > 1 && o.te == g.te) {
        if (rna) hp.recv_d = {0, 1, ra0 - g.w_lo, rna};
        if (sna) hp.send_d = {0, 1, sa0 - g.w_lo, sna};
      }
      hp.recv_bytes = 2 * ((size_t)d.Nkz * hp.recv_g.ne * hp.recv_g.na * gb + (size_t)d.Nqz * d.Nw * hp.recv_d.na * db);
      hp.send_bytes = 2 * ((size_t)d.Nkz * hp.send_g.ne * hp.send_g.na * gb + (size_t)d.Nqz * d.Nw * hp.send_d.na * db);
      if (!hp.recv_bytes && !hp.send_bytes) continue;
      // energy-only splits (Ta == 1): the G boxes are Nkz contiguous runs of the window, sent in place
      hp.direct = g.Ta == 1;
      if (!hp.direct) {
        hp.recv_off = L->recv_total;
        hp.send_off = L->send_total;
        L->recv_total += hp.recv_bytes;
        L->send_total += hp.send_bytes;
      }
      L->halo_recv += (double)hp.recv_bytes;
      L->peers.push_back(hp);
    }
  }
  return QT_OK;
}

// footprint of one rank: caller tensors (window inputs, owned outputs) + the plan's device allocations
double footprint(const Layout& L) {
  const qt_sse_desc& d = L.d;
  const double c16 = 16.0;
  double caller = 2.0 * d.Nkz * L.NEw * L.Nwin * L.NN * c16 + 2.0 * L.Nwin * (double)d_block_bytes(d) +
                  (double)L.Nwin * d.Nb * 3 * L.NN * c16 + 2.0 * d.Nkz * L.NEo * L.Nout * L.NN * c16 +
                  2.0 * (L.g.pa_hi - L.g.pa_lo) * (double)d_block_bytes(d);
  double plan = (double)L.ws_bytes + (1 << 20) + (double)L.send_total + (double)L.recv_total + 2.0 * L.part_bytes;
  if (L.fp32)
    plan += 2.0 * L.gtp_elems() * 4 + (double)L.gpi_elems() * 4;
  else
    plan += 2.0 * L.gs_elems() * 8;
  plan += (double)(L.sig_items.size() * sizeof(SigItem) + L.sig_pairs.size() * (sizeof(SigPair) + 4) +
                   L.pi_items.size() * sizeof(PiItem) + L.pi_pairs.size() * (sizeof(PiPair) + 4) + L.nbr_win.size() * 4);
  return caller + plan;
}

constexpr size_t kAutoWsCap = (size_t)48 << 30;

}  // namespace

struct qt_sse_plan_s {
  Layout L;
  // device
  int device = 0;
  int32_t* d_nbr_win = nullptr;
  SigItem* d_sig_items = nullptr;
  SigPair* d_sig_pairs = nullptr;
  int32_t* d_sig_pair_item = nullptr;
  PiItem* d_pi_items = nullptr;
  PiPair* d_pi_pairs = nullptr;
  int32_t* d_pi_pair_item = nullptr;
  int4* d_det_atoms = nullptr;
  int2* d_det_pairs = nullptr;
  double2* ws = nullptr;
  double* ws_gs = nullptr;      // FP64: Re + Im planes of G^<, G^> [2][Nwin][Nkz][NEw][NN rounded up to even]
  float* ws_gtp = nullptr;      // FP32 mode: split G planes [2][Nwin][Nkz][4][128][NEp]
  float* ws_gpi = nullptr;      // FP32 mode: split G^X planes for Π [Nwin][Nkz][4][Epad][NNp] (one X at a time)
  double2* part[2] = {nullptr, nullptr};   // Π partial sums of one group (TE > 1 with a communicator)
  // host-execute staging
  void* h_dev = nullptr;
  size_t h_dev_bytes = 0;
  cudaStream_t xstream = nullptr;   // copy-back stream of qt_sse_execute_host
  cudaEvent_t ev_out[4] = {nullptr, nullptr, nullptr, nullptr};   // Σ^<, Σ^>, Π^<, Π^> complete
  // communication
  void* comm = nullptr;         // all ranks
  void* comm_e = nullptr;       // the TE ranks of this atom slab (Π reduction)
  cudaStream_t cstream = nullptr;
  cudaEvent_t ev_in = nullptr, ev_halo = nullptr, ev_part[2] = {nullptr, nullptr}, ev_red[2] = {nullptr, nullptr};
  bool red_pending[2] = {false, false};
  char* sendbuf = nullptr;
  char* recvbuf = nullptr;
  // call ordering across streams
  cudaEvent_t ev_done = nullptr;
  cudaStream_t last_stream = nullptr;
  bool has_last = false;
  // per-kernel timing (qt_sse_timing_*)
  bool timing = false;
  std::vector<cudaEvent_t> ev_pool;
  struct Rec { int kind; cudaEvent_t a, b; };
  std::vector<Rec> recs;
  size_t ev_used = 0;
};

namespace {

qt_status cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return QT_OK;
  if (e == cudaErrorMemoryAllocation) return QT_ERR_OUT_OF_MEMORY;
  return QT_ERR_CUDA;
}
// a failed kernel launch: the status, plus (with QT_DEBUG set in the environment) the CUDA error on stderr
qt_status launch_fail(int kind, cudaError_t e, int line) {
  static const bool dbg = getenv("QT_DEBUG") != nullptr;
  if (dbg) fprintf(stderr, "qt_sse: launch of kernel kind %d failed (qt_sse.cu:%d): %s\n", kind, line, cudaGetErrorString(e));
  return cuda_status(e);
}
#define QT_CUDA(call)                              \
  do {                                             \
    cudaError_t e_ = (call);                       \
    if (e_ != cudaSuccess) return cuda_status(e_); \
  } while (0)
#define QT_TRY(call)                  \
  do {                                \
    qt_status s_ = (call);            \
    if (s_ != QT_OK) return s_;       \
  } while (0)
cudaEvent_t take_event(qt_sse_plan_s* p) {
  if (p->ev_used == p->ev_pool.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    p->ev_pool.push_back(e);
  }
  return p->ev_pool[p->ev_used++];
}
#define QT_LAUNCH(kind, call)                                            \
  do {                                                                   \
    g_launches.fetch_add(1);                                             \
    cudaEvent_t ea_ = nullptr, eb_ = nullptr;                            \
    if (p->timing) {                                                     \
      ea_ = take_event(p);                                               \
      eb_ = take_event(p);                                               \
      if (ea_ && eb_) cudaEventRecord(ea_, cs);                          \
    }                                                                    \
    cudaError_t e_ = (call);                                             \
    if (e_ != cudaSuccess) return launch_fail(kind, e_, __LINE__);       \
    if (ea_ && eb_) {                                                    \
      cudaEventRecord(eb_, cs);                                          \
      p->recs.push_back({kind, ea_, eb_});                               \
    }                                                                    \
  } while (0)

bool aligned16(const void* q) { return q != nullptr && (reinterpret_cast<uintptr_t>(q) & 15) == 0; }

// asynchronous NCCL failures of earlier calls (ncclCommGetAsyncError) -> QT_ERR_NCCL
qt_status nccl_check(const qt_sse_plan_s* p) {
  if (p->comm && nccl_async_error(p->comm)) return QT_ERR_NCCL;
  if (p->comm_e && nccl_async_error(p->comm_e)) return QT_ERR_NCCL;
  return QT_OK;
}

// every call: order after the plan's previous call when it ran on another stream (the calls share scratch)
qt_status call_begin(qt_sse_plan_s* p, cudaStream_t cs) {
  QT_TRY(nccl_check(p));
  if (p->has_last && p->last_stream != cs) QT_CUDA(cudaStreamWaitEvent(cs, p->ev_done, 0));
  return QT_OK;
}
qt_status call_end(qt_sse_plan_s* p, cudaStream_t cs) {
  QT_CUDA(cudaEventRecord(p->ev_done, cs));
  p->last_stream = cs;
  p->has_last = true;
  return QT_OK;
}

// sum planes (FP64) / split planes (FP32) of the window atoms [a0, a1) of both G^X
qt_status relayout_sigma(qt_sse_plan_s* p, const void* GL, const void* GG, int64_t a0, int64_t a1, cudaStream_t cs) {
  const Layout& L = p->L;
  const qt_sse_desc& d = L.d;
  if (a1 <= a0) return QT_OK;
  if (L.fp32) {
    QT_LAUNCH(QT_K_RELAYOUT, launch_relayout_tc((const double2*)GL, p->ws_gtp, d.Nkz, L.NEw, L.NEp, L.Nwin, (int)L.NN, a0, a1, cs));
    QT_LAUNCH(QT_K_RELAYOUT, launch_relayout_tc((const double2*)GG, p->ws_gtp + L.gtp_elems(), d.Nkz, L.NEw, L.NEp, L.Nwin,
                                                (int)L.NN, a0, a1, cs));
  } else {
    QT_LAUNCH(QT_K_RELAYOUT, launch_relayout((const double2*)GL, p->ws_gs, d.Nkz, L.NEw, L.Nwin, L.NN, a0, a1, cs));
    QT_LAUNCH(QT_K_RELAYOUT, launch_relayout((const double2*)GG, p->ws_gs + L.gs_elems(), d.Nkz, L.NEw, L.Nwin, L.NN, a0, a1, cs));
  }
  return QT_OK;
}

// Σ^X (Eq. 3) over the Σ chunks; with `halo` set the stream waits for it (and re-lays-out the halo part of
// G) before the first chunk that reads halo data.
qt_status run_sigma(qt_sse_plan_s* p, const void* dH, const void* GL, const void* GG, const void* DL, const void* DG,
                    double sre, double sim, void* SL, void* SG, cudaStream_t cs, cudaEvent_t halo, bool* halo_done,
                    cudaEvent_t* done_x = nullptr) {
  const Layout& L = p->L;
  const qt_sse_desc& d = L.d;
  const size_t sig_bytes = (size_t)d.Nkz * L.NEo * L.Nout * L.NN * sizeof(double2);
  auto wait_halo = [&](bool need) -> qt_status {
    if (!need || *halo_done) return QT_OK;
    if (halo) QT_CUDA(cudaStreamWaitEvent(cs, halo, 0));
    if (L.g.TE > 1 || !halo) {
      QT_TRY(relayout_sigma(p, GL, GG, 0, L.Nwin, cs));   // energy halo: every atom's window
    } else {
      QT_TRY(relayout_sigma(p, GL, GG, 0, L.g.a_lo - L.g.w_lo, cs));
      QT_TRY(relayout_sigma(p, GL, GG, L.g.a_hi - L.g.w_lo, L.Nwin, cs));
    }
    *halo_done = true;
    return QT_OK;
  };
  for (int X = 0; X < 2; ++X) {
    void* S = X == 0 ? SL : SG;
    QT_CUDA(cudaMemsetAsync(S, 0, sig_bytes, cs));
    for (const SigChunk& ch : L.sig_chunks) {
      const int64_t i0 = ch.i0, i1 = ch.i1;
      const int64_t pp0 = L.sig_items[i0].pair0;
      const int64_t pp1 = L.sig_items[i1 - 1].pair0 + L.sig_items[i1 - 1].npair;
      QT_TRY(wait_halo(ch.coef_halo));
      CoefArgs ca;
      ca.DX = (const double2*)(X == 0 ? DL : DG);
      ca.DY = (const double2*)(X == 0 ? DG : DL);
      ca.pairs = p->d_sig_pairs + pp0;
      ca.items = p->d_sig_items;
      ca.pair_item = p->d_sig_pair_item + pp0;
      ca.coef = p->ws;
      ca.npairs = pp1 - pp0;
      ca.Nw = d.Nw;
      ca.Nwin = L.Nwin;
      ca.Nb = d.Nb;
      ca.Nqz = d.Nqz;
      ca.DWp = L.DWp;
      ca.Dmax = (int)L.Dmax;
      ca.shift0 = d.shift0;
      ca.step = d.shift_step;
      ca.tiled = L.sig_tma;
      ca.item0 = i0;
      ca.nitems = i1 - i0;
      ca.ndc = L.ndc;
      ca.Dwin = L.Dwin;
      QT_LAUNCH(QT_K_SIGMA_COEF, L.fp32 ? launch_sigma_coef_tc(ca, (int)L.Kp, cs) : launch_sigma_coef_tiled(ca, cs));
      QT_TRY(wait_halo(ch.g_halo));
      SigmaArgs sa;
      sa.G = (const double2*)(X == 0 ? GL : GG);
      sa.Gsum = p->ws_gs ? p->ws_gs + (X == 0 ? 0 : L.gs_elems()) : nullptr;
      sa.coef = p->ws;
      sa.Gt = reinterpret_cast<double2*>(reinterpret_cast<char*>(p->ws) + L.gt_offset);
      sa.cp0 = pp0;
      sa.npairs_chunk = pp1 - pp0;
      sa.dH = (const double2*)dH;
      sa.items = p->d_sig_items + i0;
      sa.pairs = p->d_sig_pairs;
      sa.pair_item = p->d_sig_pair_item;
      sa.item0 = i0;
      sa.Sig = (double2*)S;
      sa.scale = make_double2(sre, sim);
      sa.Nwin = L.Nwin;
      sa.Nout = L.Nout;
      sa.Nb = d.Nb;
      sa.DWp = L.DWp;
      sa.NE = (int)L.NEw;
      sa.E0 = (int)L.E0;
      sa.NEo = (int)L.NEo;
      sa.NEs = (int)L.NEo;
      sa.Es0 = 0;
      sa.Nkz = (int)d.Nkz;
      sa.Nqz = (int)d.Nqz;
      sa.h = (int)L.h;
      sa.Norb = (int)d.Norb;
      sa.NN = (int)L.NN;
      sa.Dmax = (int)L.Dmax;
      sa.ndc = (int)L.ndc;
      sa.Dwin = (int)L.Dwin;
      sa.rows = (int)L.sig_rows;
      sa.gt_f32 = L.fp32 ? 1 : 0;
      sa.gt_ld = (int)L.gt_ld;
      sa.ntiles = 0;
      sa.det_atoms = p->d_det_atoms ? p->d_det_atoms + ch.det_off : nullptr;
      sa.det_pairs = p->d_det_pairs;
      sa.n_det = ch.det_n;
      for (int64_t e0 = 0; e0 < L.NEo; e0 += L.sig_ec) {   // energy sub-ranges of the Gt scratch (usually one)
        sa.E0 = (int)(L.E0 + e0);
        sa.NEo = (int)std::min<int64_t>(L.sig_ec, L.NEo - e0);
        sa.Es0 = (int)e0;
        if (L.fp32) {
          QT_LAUNCH(QT_K_SIGMA, launch_sigma_tc(sa, p->ws_gtp + (X == 0 ? 0 : L.gtp_elems()), L.NEp,
                                                reinterpret_cast<const float*>(p->ws), (int)L.Kp, i1 - i0, cs));
        } else if (L.sig_pair_mode) {
          // items [i0, i0 + nfull): energy-pair tiles; the rest: k_sigma (Gt scratch offset by nfull items)
          if (ch.nfull > 0) QT_LAUNCH(QT_K_SIGMA_PAIR, launch_sigma_pair(sa, ch.nfull, cs));
          if (i1 - i0 > ch.nfull) {
            SigmaArgs sb = sa;
            sb.items = sa.items + ch.nfull;
            sb.coef = sa.coef + (int64_t)ch.nfull * d.Nqz * L.ndc * kRows * kCoefKCP;   // tiles per chunk item
            sb.Gt = sa.Gt + (int64_t)ch.nfull * d.Nkz * sa.NEo * sa.rows * sa.gt_ld;
            QT_LAUNCH(QT_K_SIGMA, launch_sigma(sb, i1 - i0 - ch.nfull, cs));
          }
        } else {
          QT_LAUNCH(QT_K_SIGMA, launch_sigma(sa, i1 - i0, cs));
        }
        if (L.det) {
          QT_LAUNCH(QT_K_SIGMA_SAND, launch_sigma_sand_det(sa, cs));
        } else {
          QT_LAUNCH(QT_K_SIGMA_SAND, launch_sigma_sand(sa, i1 - i0, cs));
        }
      }
    }
    if (done_x) QT_CUDA(cudaEventRecord(done_x[X], cs));   // Σ^X complete (qt_sse_execute_host copies it back)
  }
  return QT_OK;
}

// Π^X (Eq. 4): per group, W sandwiches + correlation per chunk, the self slot, and (TE > 1 with a
// communicator) an ncclReduce of the group's partial sums to its owner on the communication stream, while
// the compute stream continues with the next group (two partial buffers).
qt_status run_pi(qt_sse_plan_s* p, const void* dH, const void* GL, const void* GG, double sre, double sim, void* PL,
                 void* PG, cudaStream_t cs, cudaEvent_t* done_x = nullptr) {
  const Layout& L = p->L;
  const qt_sse_desc& d = L.d;
  int nb = 0;   // partial buffer toggle
  for (int X = 0; X < 2; ++X) {
    const double2* GX = (const double2*)(X == 0 ? GL : GG);
    const double2* GY = (const double2*)(X == 0 ? GG : GL);
    double2* P = (double2*)(X == 0 ? PL : PG);
    if (L.fp32)
      QT_LAUNCH(QT_K_RELAYOUT, launch_relayout_pi_tc(GX, p->ws_gpi, d.Nkz, L.NEw, L.Epad, L.Nwin, (int)L.NN, (int)L.NNp, cs));
    for (const PiGroup& G : L.groups) {
      const int64_t nga = G.hi - G.lo;
      double2* target = P;
      int buf = -1;
      if (L.reduce) {
        buf = nb;
        nb ^= 1;
        if (p->red_pending[buf]) {   // the reduction that last read this buffer must be done
          QT_CUDA(cudaStreamWaitEvent(cs, p->ev_red[buf], 0));
          p->red_pending[buf] = false;
        }
        target = p->part[buf];
      }
      for (size_t c = 0; c + 1 < G.chunks.size(); ++c) {
        const int64_t i0 = G.chunks[c], i1 = G.chunks[c + 1];
        if (i1 <= i0) continue;
        const int64_t pp0 = L.pi_items[i0].pair0;
        for (int64_t e0 = 0; e0 < L.NEo; e0 += L.pi_ec) {   // energy sub-ranges of the W scratch (usually one)
        const int64_t ne = std::min<int64_t>(L.pi_ec, L.NEo - e0);
        PiWArgs wa;
        wa.GY = GY;
        wa.dH = (const double2*)dH;
        wa.pairs = p->d_pi_pairs;
        wa.items = p->d_pi_items;
        wa.pair_item = p->d_pi_pair_item;
        wa.W = p->ws;
        wa.p0 = pp0;
        wa.i0 = i0;
        wa.npairs = L.pi_items[i1 - 1].pair0 + L.pi_items[i1 - 1].npair - pp0;
        wa.Nwin = L.Nwin;
        wa.Nb = d.Nb;
        wa.NE = (int)L.NEw;
        wa.E0 = (int)(L.E0 + e0);
        wa.NEo = (int)ne;
        wa.Nkz = (int)d.Nkz;
        wa.Norb = (int)d.Norb;
        wa.NN = (int)L.NN;
        wa.nEB = (int)((L.NEw + kEB - 1) / kEB);
        if (L.fp32) {
          QT_LAUNCH(QT_K_PI_W, launch_pi_w_tc(wa, reinterpret_cast<float*>(p->ws), (int)L.NNp, i1 - i0, cs));
        } else {
          QT_LAUNCH(QT_K_PI_W, launch_pi_w(wa, i1 - i0, cs));
        }
        PiCArgs ca;
        ca.GX = GX;
        ca.W = p->ws;
        ca.GXsum = p->ws_gs ? p->ws_gs + (X == 0 ? 0 : L.gs_elems()) : nullptr;
        ca.items = p->d_pi_items;
        ca.pairs = p->d_pi_pairs;
        ca.Pi = target;
        ca.scale = make_double2(sre, sim);
        ca.i0 = i0;
        ca.nitems = i1 - i0;
        ca.Nwin = L.Nwin;
        ca.Nout = nga;
        ca.Nb = d.Nb;
        ca.NE = (int)L.NEw;
        ca.E0 = (int)(L.E0 + e0);
        ca.NEo = (int)ne;
        ca.accumulate = e0 > 0 ? 1 : 0;
        ca.Nkz = (int)d.Nkz;
        ca.Nqz = (int)d.Nqz;
        ca.h = (int)L.h;
        ca.NN = (int)L.NN;
        ca.Nw = (int)d.Nw;
        ca.NWv = (int)L.NWv;
        ca.NWP = (int)L.NWP;
        ca.shift0 = d.shift0;
        ca.step = d.shift_step;
        if (L.fp32) {
          QT_LAUNCH(QT_K_PI_CONTRACT, launch_pi_contract_tc(ca, reinterpret_cast<const float*>(p->ws), p->ws_gpi, L.Epad,
                                                            (int)L.NNp, i1 - i0, cs));
        } else {
          QT_LAUNCH(QT_K_PI_CONTRACT, launch_pi_contract(ca, i1 - i0, cs));
        }
        }
      }
      PiSelfArgs sa;
      sa.Pi = target;
      sa.nbr = p->d_nbr_win;
      sa.Nout = nga;
      sa.Nb = d.Nb;
      sa.Nqz = d.Nqz;
      sa.Nw = d.Nw;
      sa.a_off = G.lo - L.g.w_lo;
      QT_LAUNCH(QT_K_PI_SELF, launch_pi_self(sa, cs));
      if (L.reduce) {   // Π is a sum over energies: the group's owner receives the sum of the TE partials
        QT_CUDA(cudaEventRecord(p->ev_part[buf], cs));
        QT_CUDA(cudaStreamWaitEvent(p->cstream, p->ev_part[buf], 0));
        const size_t n = (size_t)nga * d_block_bytes(d) / sizeof(double);
        if (nccl_reduce_sum(p->comm_e, reinterpret_cast<const double*>(target), reinterpret_cast<double*>(P), n, G.root,
                            p->cstream) != 0)
          return QT_ERR_NCCL;
        QT_CUDA(cudaEventRecord(p->ev_red[buf], p->cstream));
        p->red_pending[buf] = true;
      }
    }
    if (done_x && !L.reduce) QT_CUDA(cudaEventRecord(done_x[X], cs));   // Π^X complete (no pending reduction)
  }
  for (int b = 0; b < 2; ++b)
    if (p->red_pending[b]) {
      QT_CUDA(cudaStreamWaitEvent(cs, p->ev_red[b], 0));
      p->red_pending[b] = false;
    }
  return QT_OK;
}

// halo exchange on `st`: pack (atom splits) -> one grouped send/recv round -> unpack into the window halo
qt_status exchange(qt_sse_plan_s* p, void* GL, void* GG, void* DL, void* DG, cudaStream_t st) {
  const Layout& L = p->L;
  const qt_sse_desc& d = L.d;
  cudaStream_t cs = st;   // for QT_LAUNCH
  void* gt[2] = {GL, GG};
  void* dt[2] = {DL, DG};
  const int64_t ginner = L.NN * 16, dinner = (int64_t)(d.Nb + 1) * 9 * 16;
  for (const HaloPeer& h : L.peers) {
    if (h.direct) continue;
    size_t off = h.send_off;
    for (int x = 0; x < 2; ++x) {
      const HaloBox& b = h.send_g;
      QT_LAUNCH(QT_K_HALO, launch_pack(gt[x], p->sendbuf + off, d.Nkz, L.NEw, b.e0, b.ne, L.Nwin, b.a0, b.na, ginner, false, cs));
      off += (size_t)d.Nkz * b.ne * b.na * ginner;
    }
    for (int x = 0; x < 2; ++x) {
      const HaloBox& b = h.send_d;
      QT_LAUNCH(QT_K_HALO, launch_pack(dt[x], p->sendbuf + off, d.Nqz * d.Nw, 1, 0, b.na ? 1 : 0, L.Nwin, b.a0, b.na, dinner,
                                       false, cs));
      off += (size_t)d.Nqz * d.Nw * b.na * dinner;
    }
  }
  const int64_t kzstride = L.NEw * L.Nwin * ginner;   // bytes per kz of the G window
  if (nccl_exchange(p->comm, L.peers, p->sendbuf, p->recvbuf, gt, d.Nkz, kzstride, L.Nwin * ginner, cs) != 0)
    return QT_ERR_NCCL;
  for (const HaloPeer& h : L.peers) {
    if (h.direct) continue;
    size_t off = h.recv_off;
    for (int x = 0; x < 2; ++x) {
      const HaloBox& b = h.recv_g;
      QT_LAUNCH(QT_K_HALO, launch_pack(p->recvbuf + off, gt[x], d.Nkz, L.NEw, b.e0, b.ne, L.Nwin, b.a0, b.na, ginner, true, cs));
      off += (size_t)d.Nkz * b.ne * b.na * ginner;
    }
    for (int x = 0; x < 2; ++x) {
      const HaloBox& b = h.recv_d;
      QT_LAUNCH(QT_K_HALO, launch_pack(p->recvbuf + off, dt[x], d.Nqz * d.Nw, 1, 0, b.na ? 1 : 0, L.Nwin, b.a0, b.na, dinner,
                                       true, cs));
      off += (size_t)d.Nqz * d.Nw * b.na * dinner;
    }
  }
  return QT_OK;
}

template <typename T>
qt_status upload(T** dst, const std::vector<T>& v, cudaStream_t st) {
  if (v.empty()) return QT_OK;
  QT_CUDA(cudaMalloc(dst, v.size() * sizeof(T)));
  QT_CUDA(cudaMemcpyAsync(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st));
  return QT_OK;
}

qt_status check_ptrs(std::initializer_list<const void*> ins, std::initializer_list<const void*> outs) {
  for (const void* q : ins)
    if (!aligned16(q)) return QT_ERR_INVALID_ARG;
  for (const void* o : outs) {
    if (!aligned16(o)) return QT_ERR_INVALID_ARG;
    for (const void* q : ins)
      if (q == o) return QT_ERR_INVALID_ARG;
  }
  std::vector<const void*> o(outs);
  for (size_t i = 0; i < o.size(); ++i)
    for (size_t j = i + 1; j < o.size(); ++j)
      if (o[i] == o[j]) return QT_ERR_INVALID_ARG;
  return QT_OK;
}

}  // namespace

extern "C" qt_status qt_sse_nccl_unique_id(void* out128) {
  if (!out128) return QT_ERR_INVALID_ARG;
  return nccl_unique_id(out128) == 0 ? QT_OK : QT_ERR_NCCL;
}

extern "C" const char* qt_sse_status_string(qt_status s) {
  switch (s) {
    case QT_OK: return "ok";
    case QT_ERR_INVALID_ARG: return "invalid argument";
    case QT_ERR_UNSUPPORTED: return "unsupported configuration";
    case QT_ERR_OUT_OF_MEMORY: return "out of device memory";
    case QT_ERR_CUDA: return "CUDA error";
    case QT_ERR_NCCL: return "NCCL error";
    case QT_ERR_INTERNAL: return "internal error";
  }
  return "unknown status";
}

extern "C" uint64_t qt_sse_launch_count(void) { return g_launches.load(); }

extern "C" qt_status qt_sse_count_flops(const qt_sse_desc* desc, const int32_t* nbr, double out[4]) {
  qt_status st = validate_desc(desc);
  if (st == QT_ERR_UNSUPPORTED) st = QT_OK;   // counting does not depend on kernel limits
  if (st != QT_OK) return st;
  if (!out) return QT_ERR_INVALID_ARG;
  if ((st = validate_nbr(desc, nbr)) != QT_OK) return st;
  const Geom g = geom_of(desc, nbr, desc->rank, false);
  double np = 0;
  for (int64_t a = g.a_lo; a < g.a_hi; ++a)
    for (int64_t s = 0; s < desc->Nb; ++s) np += nbr[a * desc->Nb + s] >= 0;
  count_flops(desc, np, out, g.e_lo, g.e_hi);
  return QT_OK;
}

static void fill_info(const Layout& L, size_t ws_total, qt_sse_info* o) {
  const Geom& g = L.g;
  o->a_lo = g.a_lo;
  o->a_hi = g.a_hi;
  o->w_lo = g.w_lo;
  o->w_hi = g.w_hi;
  o->npairs = (int64_t)L.npairs;
  o->workspace_bytes = ws_total;
  o->flops_sigma = L.flops[0] + L.flops[1];
  o->flops_pi = L.flops[2] + L.flops[3];
  o->halo_bytes = L.halo_recv;
  o->e_lo = g.e_lo;
  o->e_hi = g.e_hi;
  o->ew_lo = g.ew_lo;
  o->ew_hi = g.ew_hi;
  o->pa_lo = g.pa_lo;
  o->pa_hi = g.pa_hi;
  o->Ta = g.Ta;
  o->TE = g.TE;
  o->ta = g.ta;
  o->te = g.te;
  o->reduce_bytes = L.reduce_bytes;
  o->mem_bytes = footprint(L);
  int64_t np_pair = 0;
  if (L.sig_pair_mode)
    for (const SigItem& it : L.sig_items)
      if (it.npair >= kPairMinPairs) np_pair += it.npair;
  o->flops_sigma_pair = L.sig_pairs.empty() ? 0.0 : L.flops[0] * (double)np_pair / (double)L.sig_pairs.size();
}

extern "C" qt_status qt_sse_shard_info(const qt_sse_desc* desc, const int32_t* nbr, qt_sse_info* o) {
  qt_status st = validate_desc(desc);
  if (st == QT_ERR_UNSUPPORTED) st = QT_OK;
  if (st != QT_OK) return st;
  if (!o) return QT_ERR_INVALID_ARG;
  if ((st = validate_nbr(desc, nbr)) != QT_OK) return st;
  Layout* L = new (std::nothrow) Layout();
  if (!L) return QT_ERR_OUT_OF_MEMORY;
  // a sharded description is reported as the communicator-backed plan it describes
  const bool reduce = desc->nranks > 1;
  st = build_layout(desc, nbr, reduce, desc->workspace_limit ? desc->workspace_limit : kAutoWsCap, L, false);
  if (st == QT_OK) {
    size_t gsb = L->fp32 ? 2 * L->gtp_elems() * 4 + L->gpi_elems() * 4 : 2 * L->gs_elems() * 8;
    fill_info(*L, L->ws_bytes + gsb, o);
  }
  delete L;
  return st;
}

extern "C" void qt_sse_destroy(qt_sse_plan_t p) {
  if (!p) return;
  if (p->has_last) cudaEventSynchronize(p->ev_done);
  cudaFree(p->d_nbr_win);
  cudaFree(p->d_sig_items);
  cudaFree(p->d_sig_pairs);
  cudaFree(p->d_sig_pair_item);
  cudaFree(p->d_pi_items);
  cudaFree(p->d_pi_pairs);
  cudaFree(p->d_pi_pair_item);
  cudaFree(p->d_det_atoms);
  cudaFree(p->d_det_pairs);
  cudaFree(p->ws);
  cudaFree(p->ws_gs);
  cudaFree(p->ws_gtp);
  cudaFree(p->ws_gpi);
  cudaFree(p->part[0]);
  cudaFree(p->part[1]);
  cudaFree(p->sendbuf);
  cudaFree(p->recvbuf);
  nccl_comm_destroy(p->comm_e);
  nccl_comm_destroy(p->comm);
  if (p->xstream) cudaStreamSynchronize(p->xstream);
  cudaFree(p->h_dev);
  if (p->xstream) cudaStreamDestroy(p->xstream);
  for (cudaEvent_t e : p->ev_out)
    if (e) cudaEventDestroy(e);
  cudaEvent_t evs[] = {p->ev_in, p->ev_halo, p->ev_part[0], p->ev_part[1], p->ev_red[0], p->ev_red[1], p->ev_done};
  for (cudaEvent_t e : evs)
    if (e) cudaEventDestroy(e);
  if (p->cstream) cudaStreamDestroy(p->cstream);
  for (cudaEvent_t e : p->ev_pool) cudaEventDestroy(e);
  delete p;
}

extern "C" qt_status qt_sse_plan(const qt_sse_desc* desc, const int32_t* nbr, void* stream, qt_sse_plan_t* out) {
  if (!out) return QT_ERR_INVALID_ARG;
  *out = nullptr;
  qt_status st = validate_desc(desc);
  if (st != QT_OK) return st;
  if ((st = validate_nbr(desc, nbr)) != QT_OK) return st;
  cudaStream_t cs = (cudaStream_t)stream;
  qt_sse_plan_s* p = new (std::nothrow) qt_sse_plan_s();
  if (!p) return QT_ERR_OUT_OF_MEMORY;
  cudaGetDevice(&p->device);
  const bool have_comm = desc->nranks > 1 && desc->nccl_unique_id != nullptr;
  size_t budget = desc->workspace_limit;
  if (budget == 0) {
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) {
      delete p;
      return QT_ERR_CUDA;
    }
    budget = std::min<size_t>((size_t)(fr * 0.6), kAutoWsCap);
  }
  if ((st = build_layout(desc, nbr, have_comm, budget, &p->L)) != QT_OK) {
    delete p;
    return st;
  }
  Layout& L = p->L;
  auto fail = [&](qt_status s) {
    qt_sse_destroy(p);
    return s;
  };
  qt_status s2;
  if ((s2 = upload(&p->d_nbr_win, L.nbr_win, cs)) != QT_OK || (s2 = upload(&p->d_sig_items, L.sig_items, cs)) != QT_OK ||
      (s2 = upload(&p->d_sig_pairs, L.sig_pairs, cs)) != QT_OK ||
      (s2 = upload(&p->d_sig_pair_item, L.sig_pair_item, cs)) != QT_OK ||
      (s2 = upload(&p->d_pi_items, L.pi_items, cs)) != QT_OK || (s2 = upload(&p->d_pi_pairs, L.pi_pairs, cs)) != QT_OK ||
      (s2 = upload(&p->d_pi_pair_item, L.pi_pair_item, cs)) != QT_OK ||
      (s2 = upload(&p->d_det_atoms, L.det_atoms, cs)) != QT_OK || (s2 = upload(&p->d_det_pairs, L.det_pairs, cs)) != QT_OK)
    return fail(s2);
  if ((!L.fp32 && cudaMalloc(&p->ws_gs, 2 * L.gs_elems() * sizeof(double)) != cudaSuccess) ||
      (L.fp32 && cudaMalloc(&p->ws_gtp, 2 * L.gtp_elems() * sizeof(float)) != cudaSuccess) ||
      (L.fp32 && cudaMalloc(&p->ws_gpi, L.gpi_elems() * sizeof(float)) != cudaSuccess))
    return fail(QT_ERR_OUT_OF_MEMORY);
  // the odd-NN padding element of each sum-plane row is never written by k_relayout: keep it a finite zero
  if (p->ws_gs && cudaMemsetAsync(p->ws_gs, 0, 2 * L.gs_elems() * sizeof(double), cs) != cudaSuccess)
    return fail(QT_ERR_CUDA);
  if (cudaEventCreateWithFlags(&p->ev_done, cudaEventDisableTiming) != cudaSuccess) return fail(QT_ERR_CUDA);
  if (have_comm) {
    if ((L.send_total && cudaMalloc(&p->sendbuf, L.send_total) != cudaSuccess) ||
        (L.recv_total && cudaMalloc(&p->recvbuf, L.recv_total) != cudaSuccess))
      return fail(QT_ERR_OUT_OF_MEMORY);
    if (L.reduce && (cudaMalloc(&p->part[0], L.part_bytes) != cudaSuccess || cudaMalloc(&p->part[1], L.part_bytes) != cudaSuccess))
      return fail(QT_ERR_OUT_OF_MEMORY);
    if (cudaStreamCreateWithFlags(&p->cstream, cudaStreamNonBlocking) != cudaSuccess) return fail(QT_ERR_CUDA);
    cudaEvent_t* evs[] = {&p->ev_in, &p->ev_halo, &p->ev_part[0], &p->ev_part[1], &p->ev_red[0], &p->ev_red[1]};
    for (cudaEvent_t* e : evs)
      if (cudaEventCreateWithFlags(e, cudaEventDisableTiming) != cudaSuccess) return fail(QT_ERR_CUDA);
    if (nccl_comm_init(&p->comm, desc->nranks, desc->nccl_unique_id, desc->rank) != 0) return fail(QT_ERR_NCCL);
    if (L.g.TE > 1 && nccl_comm_split(p->comm, L.g.ta, L.g.te, &p->comm_e) != 0) return fail(QT_ERR_NCCL);
  }
  // + slack: the last Π stage of a chunk may read one energy block past the chunk (its results are unused)
  if (cudaMalloc(&p->ws, L.ws_bytes + (1 << 20)) != cudaSuccess) return fail(QT_ERR_OUT_OF_MEMORY);
  // zero once: padding columns of the Π W tiles are never written and must hold finite values
  if (cudaMemsetAsync(p->ws, 0, L.ws_bytes + (1 << 20), cs) != cudaSuccess) return fail(QT_ERR_CUDA);
  if (cudaStreamSynchronize(cs) != cudaSuccess) return fail(QT_ERR_CUDA);
  *out = p;
  return QT_OK;
}

extern "C" qt_status qt_sse_query(qt_sse_plan_t p, qt_sse_info* o) {
  if (!p || !o) return QT_ERR_INVALID_ARG;
  const Layout& L = p->L;
  size_t gsb = L.fp32 ? 2 * L.gtp_elems() * 4 + L.gpi_elems() * 4 : 2 * L.gs_elems() * 8;
  fill_info(L, L.ws_bytes + gsb + L.send_total + L.recv_total + 2 * L.part_bytes, o);
  QT_TRY(nccl_check(p));
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? QT_OK : cuda_status(e);
}

extern "C" qt_status qt_sse_sigma(qt_sse_plan_t p, const void* dH, const void* GL, const void* GG, const void* DL,
                                  const void* DG, double sre, double sim, void* SL, void* SG, void* stream) {
  if (!p) return QT_ERR_INVALID_ARG;
  QT_TRY(check_ptrs({dH, GL, GG, DL, DG}, {SL, SG}));
  cudaStream_t cs = (cudaStream_t)stream;
  QT_TRY(call_begin(p, cs));
  QT_TRY(relayout_sigma(p, GL, GG, 0, p->L.Nwin, cs));
  bool done = true;
  QT_TRY(run_sigma(p, dH, GL, GG, DL, DG, sre, sim, SL, SG, cs, nullptr, &done));
  return call_end(p, cs);
}

extern "C" qt_status qt_sse_pi(qt_sse_plan_t p, const void* dH, const void* GL, const void* GG, double sre,
                               double sim, void* PL, void* PG, void* stream) {
  if (!p) return QT_ERR_INVALID_ARG;
  QT_TRY(check_ptrs({dH, GL, GG}, {PL, PG}));
  cudaStream_t cs = (cudaStream_t)stream;
  QT_TRY(call_begin(p, cs));
  if (!p->L.fp32) QT_TRY(relayout_sigma(p, GL, GG, 0, p->L.Nwin, cs));   // Re+Im planes of G^X_a (Π correlation)
  QT_TRY(run_pi(p, dH, GL, GG, sre, sim, PL, PG, cs));
  return call_end(p, cs);
}

static qt_status sigma_pi_impl(qt_sse_plan_t p, const void* dH, void* GL, void* GG, void* DL, void* DG, double ssre,
                               double ssim, double psre, double psim, void* SL, void* SG, void* PL, void* PG, void* stream,
                               cudaEvent_t* sig_done, cudaEvent_t* pi_done);

extern "C" qt_status qt_sse_sigma_pi(qt_sse_plan_t p, const void* dH, void* GL, void* GG, void* DL, void* DG,
                                     double ssre, double ssim, double psre, double psim, void* SL, void* SG, void* PL,
                                     void* PG, void* stream) {
  return sigma_pi_impl(p, dH, GL, GG, DL, DG, ssre, ssim, psre, psim, SL, SG, PL, PG, stream, nullptr, nullptr);
}

static qt_status sigma_pi_impl(qt_sse_plan_t p, const void* dH, void* GL, void* GG, void* DL, void* DG, double ssre,
                               double ssim, double psre, double psim, void* SL, void* SG, void* PL, void* PG, void* stream,
                               cudaEvent_t* sig_done, cudaEvent_t* pi_done) {
  if (!p) return QT_ERR_INVALID_ARG;
  QT_TRY(check_ptrs({dH, GL, GG, DL, DG}, {SL, SG, PL, PG}));
  cudaStream_t cs = (cudaStream_t)stream;
  QT_TRY(call_begin(p, cs));
  const Layout& L = p->L;
  cudaEvent_t halo = nullptr;
  bool halo_done = true;
  if (p->comm && !L.peers.empty()) {
    // the exchange runs on the communication stream once the caller's inputs are ready (stream order)
    QT_CUDA(cudaEventRecord(p->ev_in, cs));
    QT_CUDA(cudaStreamWaitEvent(p->cstream, p->ev_in, 0));
    QT_TRY(exchange(p, GL, GG, DL, DG, p->cstream));
    QT_CUDA(cudaEventRecord(p->ev_halo, p->cstream));
    halo = p->ev_halo;
    halo_done = false;
    if (L.g.TE == 1) QT_TRY(relayout_sigma(p, GL, GG, L.g.a_lo - L.g.w_lo, L.g.a_hi - L.g.w_lo, cs));   // owned atoms
  } else {
    QT_TRY(relayout_sigma(p, GL, GG, 0, L.Nwin, cs));
  }
  QT_TRY(run_sigma(p, dH, GL, GG, DL, DG, ssre, ssim, SL, SG, cs, halo, &halo_done, sig_done));
  if (!halo_done) {   // no Σ chunk read the halo (e.g. no pairs): Π still needs it
    QT_CUDA(cudaStreamWaitEvent(cs, halo, 0));
    QT_TRY(relayout_sigma(p, GL, GG, 0, L.Nwin, cs));
  }
  QT_TRY(run_pi(p, dH, GL, GG, psre, psim, PL, PG, cs, pi_done));
  return call_end(p, cs);
}

extern "C" qt_status qt_sse_execute_host(qt_sse_plan_t p, const void* dH, const void* GL, const void* GG,
                                         const void* DL, const void* DG, double ssre, double ssim, double psre,
                                         double psim, void* SL, void* SG, void* PL, void* PG, void* stream) {
  if (!p || !dH || !GL || !GG || !DL || !DG || !SL || !SG || !PL || !PG) return QT_ERR_INVALID_ARG;
  cudaStream_t cs = (cudaStream_t)stream;
  const Layout& L = p->L;
  const qt_sse_desc& d = L.d;
  const size_t b_dH = (size_t)L.Nwin * d.Nb * 3 * L.NN * 16;
  const size_t b_G = (size_t)d.Nkz * L.NEw * L.Nwin * L.NN * 16;
  const size_t b_D = (size_t)L.Nwin * d_block_bytes(d);
  const size_t b_S = (size_t)d.Nkz * L.NEo * L.Nout * L.NN * 16;
  const size_t b_P = (size_t)(L.g.pa_hi - L.g.pa_lo) * d_block_bytes(d);
  const size_t total = b_dH + 2 * b_G + 2 * b_D + 2 * b_S + 2 * b_P;
  if (p->h_dev_bytes < total) {
    if (p->has_last) cudaEventSynchronize(p->ev_done);
    cudaFree(p->h_dev);
    p->h_dev = nullptr;
    p->h_dev_bytes = 0;
    QT_CUDA(cudaMalloc(&p->h_dev, total));
    p->h_dev_bytes = total;
  }
  char* base = (char*)p->h_dev;
  char *ddH = base, *dGL = ddH + b_dH, *dGG = dGL + b_G, *dDL = dGG + b_G, *dDG = dDL + b_D;
  char *dSL = dDG + b_D, *dSG = dSL + b_S, *dPL = dSG + b_S, *dPG = dPL + b_P;
  QT_CUDA(cudaMemcpyAsync(ddH, dH, b_dH, cudaMemcpyHostToDevice, cs));
  QT_CUDA(cudaMemcpyAsync(dGL, GL, b_G, cudaMemcpyHostToDevice, cs));
  QT_CUDA(cudaMemcpyAsync(dGG, GG, b_G, cudaMemcpyHostToDevice, cs));
  QT_CUDA(cudaMemcpyAsync(dDL, DL, b_D, cudaMemcpyHostToDevice, cs));
  QT_CUDA(cudaMemcpyAsync(dDG, DG, b_D, cudaMemcpyHostToDevice, cs));
  // Σ^<, Σ^> and (without a pending Π reduction) Π^< are copied back on a second stream as soon as each is complete,
  // overlapped with the remaining compute; Π^> (and reduced Π) after the call
  if (!p->xstream) {
    QT_CUDA(cudaStreamCreateWithFlags(&p->xstream, cudaStreamNonBlocking));
    for (cudaEvent_t& e : p->ev_out) QT_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  cudaEvent_t* sig_done = p->ev_out;
  cudaEvent_t* pi_done = p->ev_out + 2;
  QT_TRY(sigma_pi_impl(p, ddH, dGL, dGG, dDL, dDG, ssre, ssim, psre, psim, dSL, dSG, dPL, dPG, stream, sig_done, pi_done));
  void* hS[2] = {SL, SG};
  const char* dS[2] = {dSL, dSG};
  for (int x = 0; x < 2; ++x) {
    QT_CUDA(cudaStreamWaitEvent(p->xstream, sig_done[x], 0));
    QT_CUDA(cudaMemcpyAsync(hS[x], dS[x], b_S, cudaMemcpyDeviceToHost, p->xstream));
  }
  if (!L.reduce) {
    QT_CUDA(cudaStreamWaitEvent(p->xstream, pi_done[0], 0));
    QT_CUDA(cudaMemcpyAsync(PL, dPL, b_P, cudaMemcpyDeviceToHost, p->xstream));
  } else {
    QT_CUDA(cudaMemcpyAsync(PL, dPL, b_P, cudaMemcpyDeviceToHost, cs));
  }
  QT_CUDA(cudaMemcpyAsync(PG, dPG, b_P, cudaMemcpyDeviceToHost, cs));
  QT_CUDA(cudaStreamSynchronize(cs));
  QT_CUDA(cudaStreamSynchronize(p->xstream));
  QT_TRY(nccl_check(p));
  return QT_OK;
}

extern "C" qt_status qt_sse_halo_exchange(qt_sse_plan_t p, void* GL, void* GG, void* DL, void* DG, void* stream) {
  if (!p) return QT_ERR_INVALID_ARG;
  if (p->L.d.nranks == 1) return QT_OK;
  if (!p->comm) return QT_ERR_UNSUPPORTED;   // loopback plan (no NCCL unique id)
  QT_TRY(check_ptrs({GL, GG, DL, DG}, {}));
  cudaStream_t cs = (cudaStream_t)stream;
  QT_TRY(call_begin(p, cs));
  QT_TRY(exchange(p, GL, GG, DL, DG, cs));
  return call_end(p, cs);
}

extern "C" qt_status qt_sse_timing_enable(qt_sse_plan_t p, int enable) {
  if (!p) return QT_ERR_INVALID_ARG;
  p->timing = enable != 0;
  return QT_OK;
}

extern "C" qt_status qt_sse_timing_read(qt_sse_plan_t p, double ms[QT_K_NKINDS], int64_t launches[QT_K_NKINDS]) {
  if (!p || !ms || !launches) return QT_ERR_INVALID_ARG;
  for (int k = 0; k < QT_K_NKINDS; ++k) {
    ms[k] = 0.0;
    launches[k] = 0;
  }
  for (const auto& r : p->recs) {
    QT_CUDA(cudaEventSynchronize(r.b));
    float t = 0.f;
    QT_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
    ms[r.kind] += t;
    launches[r.kind] += 1;
  }
  p->recs.clear();
  p->ev_used = 0;
  return QT_OK;
}
