// qt_sse.cu — C ABI of libqtsse.so (include/qt_sse.h): plan validation, work lists,
// workspace, and the stream-ordered kernel sequence for Σ≷ (Eq. 3) and Π≷ (Eq. 4).
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

using namespace qt;

static std::atomic<uint64_t> g_launches{0};

struct qt_sse_plan_s {
  qt_sse_desc d{};
  int64_t NN = 0, h = 0, Dmax = 0, Dwin = 0, DWp = 0, NWP = 0;
  int64_t a_lo = 0, a_hi = 0, w_lo = 0, w_hi = 0, Nwin = 0, Nout = 0;
  std::vector<int32_t> nbr;          // global [Na][Nb]
  std::vector<int32_t> nbr_win;      // window [Nwin][Nb] (local indices, -1 outside/empty)
  // device
  int32_t* d_nbr_win = nullptr;
  SigItem* d_sig_items = nullptr;
  SigPair* d_sig_pairs = nullptr;
  int32_t* d_sig_pair_item = nullptr;
  PiItem* d_pi_items = nullptr;
  PiPair* d_pi_pairs = nullptr;
  int32_t* d_pi_pair_item = nullptr;
  std::vector<SigItem> sig_items;
  std::vector<PiItem> pi_items;
  int64_t n_sig_pairs = 0, n_pi_pairs = 0;
  // chunks: item ranges [lo, hi) and their pair ranges
  std::vector<int64_t> sig_chunks, pi_chunks;   // item boundaries
  double2* ws = nullptr;
  size_t ws_bytes = 0;
  double2* ws_g = nullptr;      // atom-major copies of G^<, G^> [2][Nwin][Nkz][NE][NN]
  double* ws_gs = nullptr;      // their Re + Im planes [2][Nwin][Nkz][NE][NN rounded up to even]
  bool fp32 = false;            // QT_PREC_FP32_MIXED: Σ contraction on tcgen05 (kind::tf32, 3xTF32 split)
  float* ws_gtp = nullptr;      // FP32 mode: split G planes [2][Nwin][Nkz][4][NN][NEp]
  float* ws_gpi = nullptr;      // FP32 mode: split G^X planes for Π [Nwin][Nkz][4][Epad][NNp] (one X at a time)
  int64_t Epad = 0, NNp = 0;
  int64_t sig_rows = kRows;     // Gt rows per (item, kz, E): 72, or 128 in FP32 mode (items of <= 14 pairs)
  // energy window of this rank's inputs [ew_lo, ew_hi) (NEw energies; all of [0, NE) unless energy-sharded)
  // and its output energies [e_lo, e_hi) = window energies [E0, E0 + NEo)
  int64_t e_lo = 0, e_hi = 0, ew_lo = 0, ew_hi = 0, NEw = 0, NEo = 0, E0 = 0;
  bool eshard = false;
  size_t gpi_elems() const { return (size_t)Nwin * d.Nkz * 4 * Epad * NNp; }
  int64_t NEp = 0, Kp = 0;      // FP32 mode: energy row length (multiple of 4), coefficient row length
  size_t gtp_elems() const { return (size_t)Nwin * d.Nkz * 4 * kTcRowsA * NEp; }
  size_t gs_elems() const { return (size_t)d.Nkz * NEw * Nwin * ((NN + 1) & ~int64_t(1)); }
  size_t gt_offset = 0;         // byte offset of the Σ Gt scratch inside ws
  bool sig_tma = true;          // Norb <= 10: TMA/3M k_sigma + separate sandwich
  int64_t ndc = 0;              // 16-shift chunks of the Σ coefficient window
  size_t g_elems = 0;
  double flops[4] = {0, 0, 0, 0};
  // host-execute staging
  void* h_dev = nullptr;
  size_t h_dev_bytes = 0;
  // atom-halo exchange (nranks > 1)
  void* comm = nullptr;
  std::vector<HaloPeer> peers;
  char* sendbuf = nullptr;
  char* recvbuf = nullptr;
  size_t send_total = 0, recv_total = 0;
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
#define QT_CUDA(call)                           \
  do {                                          \
    cudaError_t e_ = (call);                    \
    if (e_ != cudaSuccess) return cuda_status(e_); \
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
    if (e_ != cudaSuccess) return launch_fail(kind, e_, __LINE__);      \
    if (ea_ && eb_) {                                                    \
      cudaEventRecord(eb_, cs);                                          \
      p->recs.push_back({kind, ea_, eb_});                               \
    }                                                                    \
  } while (0)

bool aligned16(const void* p) { return p != nullptr && (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

qt_status validate_desc(const qt_sse_desc* d) {
  if (!d) return QT_ERR_INVALID_ARG;
  if (d->Na <= 0 || d->Nb <= 0 || d->Norb <= 0 || d->NE <= 0 || d->Nw <= 0 || d->Nkz <= 0 || d->Nqz <= 0)
    return QT_ERR_INVALID_ARG;
  if (d->N3D != 3 || d->Nkz != d->Nqz) return QT_ERR_INVALID_ARG;
  if (d->shift0 < 1 || d->shift_step < 1) return QT_ERR_INVALID_ARG;     // S:287 grid alignment
  if (d->Na > (1LL << 30) || d->Nb > 4096) return QT_ERR_INVALID_ARG;
  if (d->precision != QT_PREC_FP64 && d->precision != QT_PREC_FP32_MIXED) return QT_ERR_UNSUPPORTED;
  if (d->precision == QT_PREC_FP32_MIXED && (d->Norb > 10 || d->Nw > 80))   // UMMA M = Norb² <= 128, N = Nω <= 80
    return QT_ERR_UNSUPPORTED;
  if (d->Norb > 12 || d->shift_step != 1 || d->Nw > 128) return QT_ERR_UNSUPPORTED;
  if (d->nranks < 1 || d->rank < 0 || d->rank >= d->nranks) return QT_ERR_INVALID_ARG;
  if (d->nranks > 1 && d->shard != QT_SHARD_ATOM && d->shard != QT_SHARD_ENERGY) return QT_ERR_UNSUPPORTED;
  if (d->shard == QT_SHARD_ENERGY && d->Norb > 10) return QT_ERR_UNSUPPORTED;   // the TMA / tcgen05 paths only
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

// valid (E, m) counts: V- = #{E - s_m >= 0}, V+ = #{E + s_m < NE}
void window_counts(const qt_sse_desc* d, double* vm, double* vp, int64_t e_lo = 0, int64_t e_hi = -1) {
  double a = 0, b = 0;
  if (e_hi < 0) e_hi = d->NE;
  for (int64_t e = e_lo; e < e_hi; ++e)
    for (int64_t m = 0; m < d->Nw; ++m) {
      int64_t sm = d->shift0 + m * d->shift_step;
      if (e - sm >= 0) a += 1;
      if (e + sm < d->NE) b += 1;
    }
  *vm = a;
  *vp = b;
}

// algorithmic flops of the output energies [e_lo, e_hi) (default: all) for npairs valid pairs
void count_flops(const qt_sse_desc* d, double npairs, double out[4], int64_t e_lo = 0, int64_t e_hi = -1) {
  double vm, vp;
  if (e_hi < 0) e_hi = d->NE;
  window_counts(d, &vm, &vp, e_lo, e_hi);
  const double NN = (double)d->Norb * d->Norb, No3 = NN * d->Norb;
  out[0] = 2.0 * d->Nkz * d->Nqz * npairs * (vm + vp) * 9.0 * NN * 8.0;
  out[1] = 2.0 * d->Nkz * (double)(e_hi - e_lo) * npairs * 12.0 * No3 * 8.0;
  out[2] = out[1];
  out[3] = 2.0 * d->Nkz * d->Nqz * npairs * vp * 9.0 * NN * 8.0;
}

// Atom ranges of a rank for atom sharding: contiguous owned slabs balanced by valid-pair count.
void owned_range(const qt_sse_desc* d, const int32_t* nbr, int64_t* lo, int64_t* hi) {
  if (d->nranks == 1) {
    *lo = 0;
    *hi = d->Na;
    return;
  }
  std::vector<double> cum(d->Na + 1, 0.0);
  for (int64_t a = 0; a < d->Na; ++a) {
    int c = 0;
    for (int64_t s = 0; s < d->Nb; ++s) c += nbr[a * d->Nb + s] >= 0;
    cum[a + 1] = cum[a] + c + 1;
  }
  auto cut = [&](int r) -> int64_t {
    double target = cum[d->Na] * r / d->nranks;
    return (int64_t)(std::lower_bound(cum.begin(), cum.end(), target) - cum.begin());
  };
  *lo = d->rank == 0 ? 0 : cut(d->rank);
  *hi = d->rank == d->nranks - 1 ? d->Na : cut(d->rank + 1);
}

// Energy sharding (the paper's T_E tiling): rank r owns output energies [e_lo, e_hi), split by the
// Σ/Π work per energy (valid shifts + sandwich), and reads the window [e_lo - Dmax, e_hi + Dmax) ∩ [0, NE).
void energy_range(const qt_sse_desc* d, int r, int64_t* lo, int64_t* hi, int64_t* wlo, int64_t* whi) {
  std::vector<double> cum(d->NE + 1, 0.0);
  const int64_t Dmax = d->shift0 + (d->Nw - 1) * d->shift_step;
  for (int64_t e = 0; e < d->NE; ++e) {
    double w = 1.0;
    for (int64_t m = 0; m < d->Nw; ++m) {
      const int64_t sm = d->shift0 + m * d->shift_step;
      w += (e - sm >= 0) + 2.0 * (e + sm < d->NE);   // Σ absorption + emission, Π correlation
    }
    cum[e + 1] = cum[e] + w;
  }
  auto cut = [&](int k) -> int64_t {
    const double target = cum[d->NE] * k / d->nranks;
    return (int64_t)(std::lower_bound(cum.begin(), cum.end(), target) - cum.begin());
  };
  *lo = r == 0 ? 0 : cut(r);
  *hi = r == d->nranks - 1 ? d->NE : cut(r + 1);
  *wlo = std::max<int64_t>(0, *lo - Dmax);
  *whi = std::min<int64_t>(d->NE, *hi + Dmax);
}

// input window of a rank: its owned atoms plus every neighbour of them (contiguous hull)
void rank_window(const qt_sse_desc* d, const int32_t* nbr, int r, int64_t* a_lo, int64_t* a_hi, int64_t* w_lo,
                 int64_t* w_hi) {
  qt_sse_desc e = *d;
  e.rank = r;
  owned_range(&e, nbr, a_lo, a_hi);
  *w_lo = *a_lo;
  *w_hi = *a_hi;
  for (int64_t a = *a_lo; a < *a_hi; ++a)
    for (int64_t s = 0; s < d->Nb; ++s) {
      const int32_t b = nbr[a * d->Nb + s];
      if (b < 0) continue;
      *w_lo = std::min<int64_t>(*w_lo, b);
      *w_hi = std::max<int64_t>(*w_hi, b + 1);
    }
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
  int64_t lo = 0, hi = desc->Na, e_lo = 0, e_hi = desc->NE, wlo, whi;
  if (desc->shard == QT_SHARD_ENERGY && desc->nranks > 1)
    energy_range(desc, desc->rank, &e_lo, &e_hi, &wlo, &whi);   // all atoms, this rank's energies
  else
    owned_range(desc, nbr, &lo, &hi);
  double np = 0;
  for (int64_t a = lo; a < hi; ++a)
    for (int64_t s = 0; s < desc->Nb; ++s) np += nbr[a * desc->Nb + s] >= 0;
  count_flops(desc, np, out, e_lo, e_hi);
  return QT_OK;
}

extern "C" qt_status qt_sse_shard_info(const qt_sse_desc* desc, const int32_t* nbr, qt_sse_info* o) {
  qt_status st = validate_desc(desc);
  if (st == QT_ERR_UNSUPPORTED) st = QT_OK;
  if (st != QT_OK) return st;
  if (!o) return QT_ERR_INVALID_ARG;
  if ((st = validate_nbr(desc, nbr)) != QT_OK) return st;
  const bool eshard = desc->shard == QT_SHARD_ENERGY && desc->nranks > 1;
  if (eshard) {
    o->a_lo = o->w_lo = 0;
    o->a_hi = o->w_hi = desc->Na;
    energy_range(desc, desc->rank, &o->e_lo, &o->e_hi, &o->ew_lo, &o->ew_hi);
  } else {
    rank_window(desc, nbr, desc->rank, &o->a_lo, &o->a_hi, &o->w_lo, &o->w_hi);
    o->e_lo = o->ew_lo = 0;
    o->e_hi = o->ew_hi = desc->NE;
  }
  double np = 0;
  for (int64_t a = o->a_lo; a < o->a_hi; ++a)
    for (int64_t s = 0; s < desc->Nb; ++s) np += nbr[a * desc->Nb + s] >= 0;
  double f[4];
  count_flops(desc, np, f, o->e_lo, o->e_hi);
  o->npairs = (int64_t)np;
  o->workspace_bytes = 0;
  o->flops_sigma = f[0] + f[1];
  o->flops_pi = f[2] + f[3];
  double recv = 0;
  const double per_atom = 2.0 * desc->Nkz * desc->NE * desc->Norb * desc->Norb * 16 +
                          2.0 * desc->Nqz * desc->Nw * (desc->Nb + 1) * 9 * 16;
  const double per_e = 2.0 * desc->Nkz * desc->Na * desc->Norb * desc->Norb * 16;
  for (int r = 0; eshard && r < desc->nranks; ++r) {
    if (r == desc->rank) continue;
    int64_t elo, ehi, wlo, whi;
    energy_range(desc, r, &elo, &ehi, &wlo, &whi);
    recv += std::max<int64_t>(0, std::min(o->ew_hi, ehi) - std::max(o->ew_lo, elo)) * per_e;
  }
  for (int r = 0; !eshard && r < desc->nranks; ++r) {
    if (r == desc->rank) continue;
    int64_t alo, ahi, wlo, whi;
    rank_window(desc, nbr, r, &alo, &ahi, &wlo, &whi);
    recv += std::max<int64_t>(0, std::min(o->w_hi, ahi) - std::max(o->w_lo, alo)) * per_atom;
  }
  o->halo_bytes = recv;
  return QT_OK;
}

extern "C" void qt_sse_destroy(qt_sse_plan_t p) {
  if (!p) return;
  cudaFree(p->d_nbr_win);
  cudaFree(p->d_sig_items);
  cudaFree(p->d_sig_pairs);
  cudaFree(p->d_sig_pair_item);
  cudaFree(p->d_pi_items);
  cudaFree(p->d_pi_pairs);
  cudaFree(p->d_pi_pair_item);
  cudaFree(p->ws);
  cudaFree(p->ws_g);
  cudaFree(p->ws_gs);
  cudaFree(p->ws_gtp);
  cudaFree(p->ws_gpi);
  cudaFree(p->sendbuf);
  cudaFree(p->recvbuf);
  nccl_comm_destroy(p->comm);
  cudaFree(p->h_dev);
  for (cudaEvent_t e : p->ev_pool) cudaEventDestroy(e);
  delete p;
}

template <typename T>
static qt_status upload(T** dst, const std::vector<T>& v, cudaStream_t st) {
  if (v.empty()) return QT_OK;
  QT_CUDA(cudaMalloc(dst, v.size() * sizeof(T)));
  QT_CUDA(cudaMemcpyAsync(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st));
  return QT_OK;
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
  p->d = *desc;
  const qt_sse_desc& d = p->d;
  p->NN = d.Norb * d.Norb;
  p->h = d.Nkz / 2;
  p->Dmax = d.shift0 + (d.Nw - 1) * d.shift_step;
  p->Dwin = 2 * p->Dmax + 1;
  p->DWp = (p->Dwin + 3) & ~3LL;
  p->NWP = (d.Nw + 7) & ~7LL;
  p->nbr.assign(nbr, nbr + d.Na * d.Nb);
  p->eshard = d.shard == QT_SHARD_ENERGY && d.nranks > 1;
  if (p->eshard) {
    // energy sharding: all atoms, an energy window; halo = window energies owned by peers (G only: D and
    // ∇H do not depend on energy and are replicated)
    p->a_lo = p->w_lo = 0;
    p->a_hi = p->w_hi = d.Na;
    energy_range(&d, d.rank, &p->e_lo, &p->e_hi, &p->ew_lo, &p->ew_hi);
    const size_t per_e = 2 * (size_t)d.Nkz * d.Na * d.Norb * d.Norb * 16;
    for (int r = 0; r < d.nranks; ++r) {
      if (r == d.rank) continue;
      int64_t elo, ehi, wlo, whi;
      energy_range(&d, r, &elo, &ehi, &wlo, &whi);
      HaloPeer h;
      h.rank = r;
      const int64_t rl = std::max(p->ew_lo, elo), rh = std::min(p->ew_hi, ehi);
      const int64_t sl = std::max(p->e_lo, wlo), sh = std::min(p->e_hi, whi);
      h.recv_lo = rl - p->ew_lo;
      h.recv_n = std::max<int64_t>(0, rh - rl);
      h.send_lo = sl - p->ew_lo;
      h.send_n = std::max<int64_t>(0, sh - sl);
      h.recv_bytes = h.recv_n * per_e;
      h.send_bytes = h.send_n * per_e;
      h.recv_off = p->recv_total;
      h.send_off = p->send_total;
      p->recv_total += h.recv_bytes;
      p->send_total += h.send_bytes;
      if (h.recv_n || h.send_n) p->peers.push_back(h);
    }
  } else {
    rank_window(&d, nbr, d.rank, &p->a_lo, &p->a_hi, &p->w_lo, &p->w_hi);
    p->e_lo = p->ew_lo = 0;
    p->e_hi = p->ew_hi = d.NE;
  }
  p->NEw = p->ew_hi - p->ew_lo;
  p->NEo = p->e_hi - p->e_lo;
  p->E0 = p->e_lo - p->ew_lo;
  // halo exchange plan: receive window atoms owned by peers, send owned atoms in the peers' windows
  if (d.nranks > 1 && !p->eshard) {
    const size_t per_atom = 2 * (size_t)d.Nkz * d.NE * d.Norb * d.Norb * 16 + 2 * (size_t)d.Nqz * d.Nw * (d.Nb + 1) * 9 * 16;
    for (int r = 0; r < d.nranks; ++r) {
      if (r == d.rank) continue;
      int64_t alo, ahi, wlo, whi;
      rank_window(&d, nbr, r, &alo, &ahi, &wlo, &whi);
      HaloPeer h;
      h.rank = r;
      const int64_t rl = std::max(p->w_lo, alo), rh = std::min(p->w_hi, ahi);
      const int64_t sl = std::max(p->a_lo, wlo), sh = std::min(p->a_hi, whi);
      h.recv_lo = rl - p->w_lo;
      h.recv_n = std::max<int64_t>(0, rh - rl);
      h.send_lo = sl - p->w_lo;
      h.send_n = std::max<int64_t>(0, sh - sl);
      h.recv_bytes = h.recv_n * per_atom;
      h.send_bytes = h.send_n * per_atom;
      h.recv_off = p->recv_total;
      h.send_off = p->send_total;
      p->recv_total += h.recv_bytes;
      p->send_total += h.send_bytes;
      if (h.recv_n || h.send_n) p->peers.push_back(h);
    }
  }
  p->Nwin = p->w_hi - p->w_lo;
  p->Nout = p->a_hi - p->a_lo;
  p->nbr_win.assign(p->Nwin * d.Nb, -1);
  for (int64_t a = p->w_lo; a < p->w_hi; ++a)
    for (int64_t s = 0; s < d.Nb; ++s) {
      int32_t b = nbr[a * d.Nb + s];
      if (b >= p->w_lo && b < p->w_hi) p->nbr_win[(a - p->w_lo) * d.Nb + s] = (int32_t)(b - p->w_lo);
    }

  // Σ work list: source-organized. For each source atom b, its reverse pairs (a,s) with a owned.
  std::vector<SigPair> sp;
  std::vector<int32_t> sp_item;
  for (int64_t b = p->w_lo; b < p->w_hi; ++b) {
    std::vector<SigPair> mine;
    for (int64_t r = 0; r < d.Nb; ++r) {
      int32_t a = nbr[b * d.Nb + r];
      if (a < 0 || a < p->a_lo || a >= p->a_hi) continue;
      SigPair q;
      q.a = (int32_t)(a - p->a_lo);
      q.a_in = (int32_t)(a - p->w_lo);
      q.s = (int32_t)rev_slot(nbr, d.Nb, a, b);
      q.r = (int32_t)r;
      mine.push_back(q);
    }
    const size_t scap = d.precision == QT_PREC_FP32_MIXED ? kTcPiPairs : kMaxPairs;   // 126 / 72 GEMM rows
    for (size_t k = 0; k < mine.size(); k += scap) {
      SigItem it;
      it.b_in = (int32_t)(b - p->w_lo);
      it.b = (int32_t)b;
      it.npair = (int32_t)std::min<size_t>(scap, mine.size() - k);
      it.pair0 = (int32_t)sp.size();
      for (int t = 0; t < it.npair; ++t) {
        sp.push_back(mine[k + t]);
        sp_item.push_back((int32_t)p->sig_items.size());
      }
      p->sig_items.push_back(it);
    }
  }
  p->n_sig_pairs = (int64_t)sp.size();
  // Π work list: destination-organized. For each owned atom a, its valid slots in chunks of 8.
  std::vector<PiPair> pp;
  std::vector<int32_t> pp_item;
  for (int64_t a = p->a_lo; a < p->a_hi; ++a) {
    std::vector<PiPair> mine;
    for (int64_t s = 0; s < d.Nb; ++s) {
      int32_t b = nbr[a * d.Nb + s];
      if (b < 0) continue;
      PiPair q;
      q.s = (int32_t)s;
      q.b_in = (int32_t)(b - p->w_lo);
      q.r = (int32_t)rev_slot(nbr, d.Nb, b, a);
      q.a_in = (int32_t)(a - p->w_lo);
      mine.push_back(q);
    }
    const size_t cap = d.precision == QT_PREC_FP32_MIXED ? kTcPiPairs : kMaxPairs;   // 126 / 72 GEMM rows
    for (size_t k = 0; k < mine.size(); k += cap) {
      PiItem it;
      it.a_out = (int32_t)(a - p->a_lo);
      it.a_in = (int32_t)(a - p->w_lo);
      it.npair = (int32_t)std::min<size_t>(cap, mine.size() - k);
      it.pair0 = (int32_t)pp.size();
      for (int t = 0; t < it.npair; ++t) {
        pp.push_back(mine[k + t]);
        pp_item.push_back((int32_t)p->pi_items.size());
      }
      p->pi_items.push_back(it);
    }
  }
  p->n_pi_pairs = (int64_t)pp.size();
  count_flops(&d, (double)p->n_pi_pairs, p->flops, p->e_lo, p->e_hi);

  // workspace (shared by Σ coefficient tables and Π W scratch; the two calls never overlap)
  const size_t coef_per_pair = (size_t)9 * d.Nqz * p->DWp * sizeof(double2);
  // Π W scratch per item: complex tiles (FP64 mode) or four fp32 split planes (FP32 mode)
  p->sig_rows = d.precision == QT_PREC_FP32_MIXED ? kTcRows : kRows;   // Gt rows per (item, kz, E)
  const size_t gt_per_item = (size_t)d.Nkz * p->NEo * p->sig_rows * ((p->NN + 19) / 20) * 20 *
                             (d.precision == QT_PREC_FP32_MIXED ? sizeof(float2) : sizeof(double2));
  p->NNp = (p->NN + 3) & ~int64_t(3);
  p->Epad = p->NEw + d.shift0 + 80 + 1;
  const size_t w_per_item = d.precision == QT_PREC_FP32_MIXED
                                ? (size_t)4 * kTcPiRows * d.Nkz * (((p->NEo * p->NNp + 31) / 32) * 32) * sizeof(float)
                                : gt_per_item;
  size_t budget = d.workspace_limit;
  if (budget == 0) {
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) {
      qt_sse_destroy(p);
      return QT_ERR_CUDA;
    }
    budget = std::min<size_t>((size_t)(fr * 0.6), (size_t)48 << 30);
  }
  p->fp32 = d.precision == QT_PREC_FP32_MIXED;
  p->NEp = std::max<int64_t>(32, (p->NEw + 3) & ~int64_t(3));   // TMA boxes (32 wide) must lie inside the tensor
  p->Kp = (p->Dwin + 3 + 31) & ~int64_t(31);   // delayed coefficient rows (d + s, s <= 3), whole 32-chunks
  const size_t coef_item_t = p->fp32 ? (size_t)d.Nqz * 16 * kTcRows * p->Kp * sizeof(float)
                                     : (size_t)d.Nqz * ((p->Dwin + 15) / 16) * kRows * kCoefKCP * sizeof(double2);
  const size_t need_min = std::max(coef_per_pair * kMaxPairs, coef_item_t) + w_per_item + 512;
  if (budget < need_min) budget = need_min;
  const size_t full = std::max((coef_per_pair * kMaxPairs + coef_item_t + w_per_item) * p->sig_items.size() + 512,
                               w_per_item * p->pi_items.size());
  p->ws_bytes = std::max<size_t>(std::min(budget, full), 256);
  // chunk item ranges so that each chunk's pairs fit the workspace
  // chunk item ranges so that each chunk's scratch fits the workspace (Σ: per pair; Π: per item)
  auto make_chunks = [&](auto& items, size_t per_unit, bool per_pair, std::vector<int64_t>& bounds) {
    const int64_t cap = (int64_t)(p->ws_bytes / per_unit);
    bounds.clear();
    bounds.push_back(0);
    int64_t acc = 0;
    for (size_t i = 0; i < items.size(); ++i) {
      const int64_t u = per_pair ? items[i].npair : 1;
      if (acc + u > cap) {
        bounds.push_back((int64_t)i);
        acc = 0;
      }
      acc += u;
    }
    bounds.push_back((int64_t)items.size());
  };
  make_chunks(p->pi_items, w_per_item, false, p->pi_chunks);
  // Σ chunks. TMA path (Norb <= 10): per item a tiled coefficient block [q][16-shift chunk][72][kCoefKCP] +
  // its Gt scratch; cp.async path (Norb 11, 12): per pair coefficient rows. Workspace = [coef | Gt].
  {
    p->sig_tma = d.Norb <= 10;
    p->ndc = (p->Dwin + 15) / 16;
    const size_t coef_item = coef_item_t;
    const size_t gt_item = p->sig_tma ? gt_per_item : 0;
    p->sig_chunks.clear();
    p->sig_chunks.push_back(0);
    size_t coef_acc = 0, gt_acc = 0, coef_max = 0;
    for (size_t i = 0; i < p->sig_items.size(); ++i) {
      const size_t cu = p->sig_tma ? coef_item : (size_t)p->sig_items[i].npair * coef_per_pair;
      if (gt_acc > 0 && coef_acc + cu + gt_acc + gt_item + 256 > p->ws_bytes) {
        p->sig_chunks.push_back((int64_t)i);
        coef_max = std::max(coef_max, coef_acc);
        coef_acc = 0;
        gt_acc = 0;
      }
      coef_acc += cu;
      gt_acc += gt_item == 0 ? 1 : gt_item;
    }
    coef_max = std::max(coef_max, coef_acc);
    p->sig_chunks.push_back((int64_t)p->sig_items.size());
    p->gt_offset = (coef_max + 255) & ~size_t(255);
  }

  qt_status s2;
  if ((s2 = upload(&p->d_nbr_win, p->nbr_win, cs)) != QT_OK || (s2 = upload(&p->d_sig_items, p->sig_items, cs)) != QT_OK ||
      (s2 = upload(&p->d_sig_pairs, sp, cs)) != QT_OK || (s2 = upload(&p->d_sig_pair_item, sp_item, cs)) != QT_OK ||
      (s2 = upload(&p->d_pi_items, p->pi_items, cs)) != QT_OK || (s2 = upload(&p->d_pi_pairs, pp, cs)) != QT_OK ||
      (s2 = upload(&p->d_pi_pair_item, pp_item, cs)) != QT_OK) {
    qt_sse_destroy(p);
    return s2;
  }
  p->g_elems = (size_t)d.Nkz * p->NEw * p->Nwin * p->NN;
  if (cudaMalloc(&p->ws_g, 2 * p->g_elems * sizeof(double2)) != cudaSuccess ||
      cudaMalloc(&p->ws_gs, 2 * p->gs_elems() * sizeof(double)) != cudaSuccess ||
      (p->fp32 && cudaMalloc(&p->ws_gtp, 2 * p->gtp_elems() * sizeof(float)) != cudaSuccess) ||
      (p->fp32 && cudaMalloc(&p->ws_gpi, p->gpi_elems() * sizeof(float)) != cudaSuccess)) {
    qt_sse_destroy(p);
    return QT_ERR_OUT_OF_MEMORY;
  }
  // the odd-NN padding element of each sum-plane row is never written by k_relayout: keep it a finite zero
  if (cudaMemsetAsync(p->ws_gs, 0, 2 * p->gs_elems() * sizeof(double), cs) != cudaSuccess) {
    qt_sse_destroy(p);
    return QT_ERR_CUDA;
  }
  if (d.nranks > 1 && d.nccl_unique_id) {
    if ((p->send_total && cudaMalloc(&p->sendbuf, p->send_total) != cudaSuccess) ||
        (p->recv_total && cudaMalloc(&p->recvbuf, p->recv_total) != cudaSuccess)) {
      qt_sse_destroy(p);
      return QT_ERR_OUT_OF_MEMORY;
    }
    if (nccl_comm_init(&p->comm, d.nranks, d.nccl_unique_id, d.rank) != 0) {
      qt_sse_destroy(p);
      return QT_ERR_NCCL;
    }
  }
  // + slack: the last Π stage of a chunk may read one energy block past the chunk (its results are unused)
  if (cudaMalloc(&p->ws, p->ws_bytes + (1 << 20)) != cudaSuccess) {
    qt_sse_destroy(p);
    return QT_ERR_OUT_OF_MEMORY;
  }
  // zero once: padding columns of the Π W tiles are never written and must hold finite values
  if (cudaMemsetAsync(p->ws, 0, p->ws_bytes + (1 << 20), cs) != cudaSuccess) {
    qt_sse_destroy(p);
    return QT_ERR_CUDA;
  }
  if (cudaStreamSynchronize(cs) != cudaSuccess) {
    qt_sse_destroy(p);
    return QT_ERR_CUDA;
  }
  *out = p;
  return QT_OK;
}

extern "C" qt_status qt_sse_query(qt_sse_plan_t p, qt_sse_info* o) {
  if (!p || !o) return QT_ERR_INVALID_ARG;
  o->a_lo = p->a_lo;
  o->a_hi = p->a_hi;
  o->w_lo = p->w_lo;
  o->w_hi = p->w_hi;
  o->npairs = p->n_pi_pairs;
  o->workspace_bytes = p->ws_bytes + 2 * p->g_elems * sizeof(double2) + 2 * p->gs_elems() * sizeof(double);
  o->flops_sigma = p->flops[0] + p->flops[1];
  o->flops_pi = p->flops[2] + p->flops[3];
  o->halo_bytes = (double)p->recv_total;
  o->e_lo = p->e_lo;
  o->e_hi = p->e_hi;
  o->ew_lo = p->ew_lo;
  o->ew_hi = p->ew_hi;
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? QT_OK : cuda_status(e);
}

extern "C" qt_status qt_sse_sigma(qt_sse_plan_t p, const void* dH, const void* GL, const void* GG, const void* DL,
                                  const void* DG, double sre, double sim, void* SL, void* SG, void* stream) {
  if (!p) return QT_ERR_INVALID_ARG;
  const void* ins[] = {dH, GL, GG, DL, DG};
  for (const void* q : ins)
    if (!aligned16(q)) return QT_ERR_INVALID_ARG;
  if (!aligned16(SL) || !aligned16(SG) || SL == SG) return QT_ERR_INVALID_ARG;
  for (const void* q : ins)
    if (q == SL || q == SG) return QT_ERR_INVALID_ARG;
  cudaStream_t cs = (cudaStream_t)stream;
  const qt_sse_desc& d = p->d;
  const size_t sig_bytes = (size_t)d.Nkz * p->NEo * p->Nout * p->NN * sizeof(double2);
  if (p->fp32) {
    QT_LAUNCH(QT_K_RELAYOUT, launch_relayout_tc((const double2*)GL, p->ws_gtp, d.Nkz, p->NEw, p->NEp, p->Nwin, (int)p->NN, cs));
    QT_LAUNCH(QT_K_RELAYOUT, launch_relayout_tc((const double2*)GG, p->ws_gtp + p->gtp_elems(), d.Nkz, p->NEw, p->NEp, p->Nwin,
                                                (int)p->NN, cs));
  } else {
    QT_LAUNCH(QT_K_RELAYOUT, launch_relayout((const double2*)GL, p->ws_g, p->ws_gs, d.Nkz, p->NEw, p->Nwin, p->NN, cs));
    QT_LAUNCH(QT_K_RELAYOUT, launch_relayout((const double2*)GG, p->ws_g + p->g_elems, p->ws_gs + p->gs_elems(), d.Nkz, p->NEw, p->Nwin, p->NN, cs));
  }
  for (int X = 0; X < 2; ++X) {
    void* S = X == 0 ? SL : SG;
    QT_CUDA(cudaMemsetAsync(S, 0, sig_bytes, cs));
    for (size_t c = 0; c + 1 < p->sig_chunks.size(); ++c) {
      const int64_t i0 = p->sig_chunks[c], i1 = p->sig_chunks[c + 1];
      if (i1 <= i0) continue;
      const int64_t pp0 = p->sig_items[i0].pair0;
      const int64_t pp1 = p->sig_items[i1 - 1].pair0 + p->sig_items[i1 - 1].npair;
      CoefArgs ca;
      ca.DX = (const double2*)(X == 0 ? DL : DG);
      ca.DY = (const double2*)(X == 0 ? DG : DL);
      ca.pairs = p->d_sig_pairs + pp0;
      ca.items = p->d_sig_items;
      ca.pair_item = p->d_sig_pair_item + pp0;
      ca.coef = p->ws;
      ca.npairs = pp1 - pp0;
      ca.Nw = d.Nw;
      ca.Nwin = p->Nwin;
      ca.Nb = d.Nb;
      ca.Nqz = d.Nqz;
      ca.DWp = p->DWp;
      ca.Dmax = (int)p->Dmax;
      ca.shift0 = d.shift0;
      ca.tiled = p->sig_tma;
      ca.item0 = i0;
      ca.nitems = i1 - i0;
      ca.ndc = p->ndc;
      ca.Dwin = p->Dwin;
      QT_LAUNCH(QT_K_SIGMA_COEF, p->fp32      ? launch_sigma_coef_tc(ca, (int)p->Kp, cs)
                                 : p->sig_tma ? launch_sigma_coef_tiled(ca, cs)
                                              : launch_sigma_coef(ca, cs));
      SigmaArgs sa;
      sa.G = (const double2*)(X == 0 ? GL : GG);
      sa.Gam = p->ws_g + (X == 0 ? 0 : p->g_elems);
      sa.Gsum = p->ws_gs + (X == 0 ? 0 : p->gs_elems());
      sa.coef = p->ws;
      sa.Gt = reinterpret_cast<double2*>(reinterpret_cast<char*>(p->ws) + p->gt_offset);
      sa.cp0 = pp0;
      sa.npairs_chunk = pp1 - pp0;
      sa.dH = (const double2*)dH;
      sa.items = p->d_sig_items + i0;
      sa.pairs = p->d_sig_pairs;
      sa.Sig = (double2*)S;
      sa.scale = make_double2(sre, sim);
      sa.Nwin = p->Nwin;
      sa.Nout = p->Nout;
      sa.Nb = d.Nb;
      sa.DWp = p->DWp;
      sa.NE = (int)p->NEw;
      sa.E0 = (int)p->E0;
      sa.NEo = (int)p->NEo;
      sa.Nkz = (int)d.Nkz;
      sa.Nqz = (int)d.Nqz;
      sa.h = (int)p->h;
      sa.Norb = (int)d.Norb;
      sa.NN = (int)p->NN;
      sa.Dmax = (int)p->Dmax;
      sa.ndc = (int)p->ndc;
      sa.Dwin = (int)p->Dwin;
      sa.rows = (int)p->sig_rows;
      sa.gt_f32 = p->fp32 ? 1 : 0;
      if (p->fp32) {
        QT_LAUNCH(QT_K_SIGMA, launch_sigma_tc(sa, p->ws_gtp + (X == 0 ? 0 : p->gtp_elems()), p->NEp,
                                              reinterpret_cast<const float*>(p->ws), (int)p->Kp, i1 - i0, cs));
      } else {
        QT_LAUNCH(QT_K_SIGMA, launch_sigma(sa, i1 - i0, cs));
      }
      QT_LAUNCH(QT_K_SIGMA_SAND, launch_sigma_sand(sa, i1 - i0, cs));
    }
  }
  return QT_OK;
}

extern "C" qt_status qt_sse_pi(qt_sse_plan_t p, const void* dH, const void* GL, const void* GG, double sre,
                               double sim, void* PL, void* PG, void* stream) {
  if (!p) return QT_ERR_INVALID_ARG;
  const void* ins[] = {dH, GL, GG};
  for (const void* q : ins)
    if (!aligned16(q)) return QT_ERR_INVALID_ARG;
  if (!aligned16(PL) || !aligned16(PG) || PL == PG) return QT_ERR_INVALID_ARG;
  for (const void* q : ins)
    if (q == PL || q == PG) return QT_ERR_INVALID_ARG;
  cudaStream_t cs = (cudaStream_t)stream;
  const qt_sse_desc& d = p->d;
  QT_LAUNCH(QT_K_RELAYOUT, launch_relayout((const double2*)GL, p->ws_g, p->ws_gs, d.Nkz, p->NEw, p->Nwin, p->NN, cs));
  QT_LAUNCH(QT_K_RELAYOUT, launch_relayout((const double2*)GG, p->ws_g + p->g_elems, p->ws_gs + p->gs_elems(), d.Nkz, p->NEw, p->Nwin, p->NN, cs));
  for (int X = 0; X < 2; ++X) {
    const double2* GXam = p->ws_g + (X == 0 ? 0 : p->g_elems);
    const double2* GY = (const double2*)(X == 0 ? GG : GL);
    double2* P = (double2*)(X == 0 ? PL : PG);
    if (p->fp32)
      QT_LAUNCH(QT_K_RELAYOUT, launch_relayout_pi_tc((const double2*)(X == 0 ? GL : GG), p->ws_gpi, d.Nkz, p->NEw, p->Epad,
                                                     p->Nwin, (int)p->NN, (int)p->NNp, cs));
    for (size_t c = 0; c + 1 < p->pi_chunks.size(); ++c) {
      const int64_t i0 = p->pi_chunks[c], i1 = p->pi_chunks[c + 1];
      if (i1 <= i0) continue;
      const int64_t pp0 = p->pi_items[i0].pair0;
      const int64_t pp1 = p->pi_items[i1 - 1].pair0 + p->pi_items[i1 - 1].npair;
      PiWArgs wa;
      wa.GY = GY;
      wa.GYam = p->ws_g + (X == 0 ? p->g_elems : 0);
      wa.dH = (const double2*)dH;
      wa.pairs = p->d_pi_pairs;
      wa.items = p->d_pi_items;
      wa.pair_item = p->d_pi_pair_item;
      wa.W = p->ws;
      wa.p0 = pp0;
      wa.i0 = i0;
      wa.Nwin = p->Nwin;
      wa.Nb = d.Nb;
      wa.NE = (int)p->NEw;
      wa.E0 = (int)p->E0;
      wa.NEo = (int)p->NEo;
      wa.Nkz = (int)d.Nkz;
      wa.Norb = (int)d.Norb;
      wa.NN = (int)p->NN;
      wa.nEB = (int)((p->NEw + kEB - 1) / kEB);
      if (p->fp32) {
        QT_LAUNCH(QT_K_PI_W, launch_pi_w_tc(wa, reinterpret_cast<float*>(p->ws), (int)p->NNp, i1 - i0, cs));
      } else {
        QT_LAUNCH(QT_K_PI_W, launch_pi_w(wa, i1 - i0, cs));
      }
      PiCArgs ca;
      ca.GX = GXam;
      ca.W = p->ws;
      ca.GXsum = p->ws_gs + (X == 0 ? 0 : p->gs_elems());
      ca.items = p->d_pi_items;
      ca.pairs = p->d_pi_pairs;
      ca.Pi = P;
      ca.scale = make_double2(sre, sim);
      ca.i0 = i0;
      ca.nitems = i1 - i0;
      ca.Nwin = p->Nwin;
      ca.Nout = p->Nout;
      ca.Nb = d.Nb;
      ca.NE = (int)p->NEw;
      ca.E0 = (int)p->E0;
      ca.NEo = (int)p->NEo;
      ca.Nkz = (int)d.Nkz;
      ca.Nqz = (int)d.Nqz;
      ca.h = (int)p->h;
      ca.NN = (int)p->NN;
      ca.Nw = (int)d.Nw;
      ca.NWP = (int)p->NWP;
      ca.shift0 = d.shift0;
      if (p->fp32) {
        QT_LAUNCH(QT_K_PI_CONTRACT, launch_pi_contract_tc(ca, reinterpret_cast<const float*>(p->ws), p->ws_gpi, p->Epad,
                                                          (int)p->NNp, i1 - i0, cs));
      } else {
        QT_LAUNCH(QT_K_PI_CONTRACT, launch_pi_contract(ca, i1 - i0, cs));
      }
    }
    PiSelfArgs sa;
    sa.Pi = P;
    sa.nbr = p->d_nbr_win;
    sa.Nout = p->Nout;
    sa.Nb = d.Nb;
    sa.Nqz = d.Nqz;
    sa.Nw = d.Nw;
    sa.a_off = p->a_lo - p->w_lo;
    QT_LAUNCH(QT_K_PI_SELF, launch_pi_self(sa, cs));
    if (p->eshard) {   // Π is a sum over energies: add the ranks' partial sums (NCCL over NVLink)
      if (!p->comm) return QT_ERR_UNSUPPORTED;
      const size_t n = (size_t)d.Nqz * d.Nw * p->Nout * (d.Nb + 1) * 9 * 2;
      if (nccl_allreduce_sum(p->comm, reinterpret_cast<double*>(P), n, cs) != 0) return QT_ERR_NCCL;
    }
  }
  return QT_OK;
}

extern "C" qt_status qt_sse_execute_host(qt_sse_plan_t p, const void* dH, const void* GL, const void* GG,
                                         const void* DL, const void* DG, double ssre, double ssim, double psre,
                                         double psim, void* SL, void* SG, void* PL, void* PG, void* stream) {
  if (!p || !dH || !GL || !GG || !DL || !DG || !SL || !SG || !PL || !PG) return QT_ERR_INVALID_ARG;
  cudaStream_t cs = (cudaStream_t)stream;
  const qt_sse_desc& d = p->d;
  const size_t b_dH = (size_t)p->Nwin * d.Nb * 3 * p->NN * 16;
  const size_t b_G = (size_t)d.Nkz * p->NEw * p->Nwin * p->NN * 16;
  const size_t b_D = (size_t)d.Nqz * d.Nw * p->Nwin * (d.Nb + 1) * 9 * 16;
  const size_t b_S = (size_t)d.Nkz * p->NEo * p->Nout * p->NN * 16;
  const size_t b_P = (size_t)d.Nqz * d.Nw * p->Nout * (d.Nb + 1) * 9 * 16;
  const size_t total = b_dH + 2 * b_G + 2 * b_D + 2 * b_S + 2 * b_P;
  if (p->h_dev_bytes < total) {
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
  qt_status st = qt_sse_sigma(p, ddH, dGL, dGG, dDL, dDG, ssre, ssim, dSL, dSG, stream);
  if (st != QT_OK) return st;
  st = qt_sse_pi(p, ddH, dGL, dGG, psre, psim, dPL, dPG, stream);
  if (st != QT_OK) return st;
  QT_CUDA(cudaMemcpyAsync(SL, dSL, b_S, cudaMemcpyDeviceToHost, cs));
  QT_CUDA(cudaMemcpyAsync(SG, dSG, b_S, cudaMemcpyDeviceToHost, cs));
  QT_CUDA(cudaMemcpyAsync(PL, dPL, b_P, cudaMemcpyDeviceToHost, cs));
  QT_CUDA(cudaMemcpyAsync(PG, dPG, b_P, cudaMemcpyDeviceToHost, cs));
  QT_CUDA(cudaStreamSynchronize(cs));
  return QT_OK;
}

extern "C" qt_status qt_sse_halo_exchange(qt_sse_plan_t p, void* GL, void* GG, void* DL, void* DG, void* stream) {
  if (!p) return QT_ERR_INVALID_ARG;
  if (p->d.nranks == 1) return QT_OK;
  if (!p->comm) return QT_ERR_UNSUPPORTED;   // planned without an NCCL unique id
  void* ts[4] = {GL, GG, DL, DG};
  for (void* t : ts)
    if (!aligned16(t)) return QT_ERR_INVALID_ARG;
  cudaStream_t cs = (cudaStream_t)stream;
  const qt_sse_desc& d = p->d;
  // atom sharding: G≷ [Nkz·NE][atoms][NN] and D≷ [Nqz·Nω][atoms][Nb+1][9] along atoms; energy sharding:
  // G≷ [Nkz][energies][Na·NN] along energies (D≷ replicated)
  const int nt = p->eshard ? 2 : 4;
  const int64_t outer[4] = {p->eshard ? d.Nkz : d.Nkz * d.NE, p->eshard ? d.Nkz : d.Nkz * d.NE, d.Nqz * d.Nw,
                            d.Nqz * d.Nw};
  const int64_t inner[4] = {p->eshard ? d.Na * p->NN * 16 : p->NN * 16, p->eshard ? d.Na * p->NN * 16 : p->NN * 16,
                            (d.Nb + 1) * 9 * 16, (d.Nb + 1) * 9 * 16};
  const int64_t span = p->eshard ? p->NEw : p->Nwin;
  for (const HaloPeer& h : p->peers) {
    size_t off = h.send_off;
    for (int k = 0; k < nt; ++k) {
      QT_LAUNCH(QT_K_HALO, launch_pack(ts[k], p->sendbuf + off, outer[k], span, h.send_lo, h.send_n, inner[k], false, cs));
      off += (size_t)outer[k] * h.send_n * inner[k];
    }
  }
  if (nccl_exchange(p->comm, p->peers, p->sendbuf, p->recvbuf, cs) != 0) return QT_ERR_NCCL;
  for (const HaloPeer& h : p->peers) {
    size_t off = h.recv_off;
    for (int k = 0; k < nt; ++k) {
      QT_LAUNCH(QT_K_HALO, launch_pack(p->recvbuf + off, ts[k], outer[k], span, h.recv_lo, h.recv_n, inner[k], true, cs));
      off += (size_t)outer[k] * h.recv_n * inner[k];
    }
  }
  return QT_OK;
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
