// rgf.cu — recursive Green's Function solver (include/qt_rgf.h): the GF phase of Eq. 1
// by the RGF forward/backward pass over the bnum diagonal blocks, batched over the independent
// (E, kz) points ("operating on all atoms for a specific energy-momentum pair").
//
// B200 mapping: every block step is a handful of dense bs x bs complex products, identical for all P points, so
// each is ONE strided-batched ZGEMM over the points (cuBLAS: a plain library GEMM on the FP64 tensor pipe, 34 TF
// measured at bs = 640); the block inversions are blocked LU + triangular solves against the identity
// (cuSOLVER getrf + getrs, whose trailing updates are GEMMs), one per point, fanned out over kRgfLanes streams so
// the points' factorizations run concurrently (cuBLAS' batched getrf/getri is built for small matrices: 9 of 10 s
// at bs = 640); the only hand-written kernels are the anti-Hermitian update G^≷ += Y − Y† of the backward pass
// (tiled transpose in shared memory), the identity fill and a batched add.
// The left-connected g^R, g^<, g^> live in the OUTPUT tensors (the backward pass overwrites block n after its
// last read), so the plan's scratch is seven bs x bs temporaries per point. Row-major blocks are handed to the
// column-major cuBLAS as their transposes: row-major C = op(A)·op(B) is column-major C^T = op(B)^T·op(A)^T,
// with op = N for X and op = C (conjugate transpose) for X†.
#include <cublas_v2.h>
#include <cusolverDn.h>

#include <cstdio>
#include <cstdlib>
#include <new>
#include <vector>

#include "qt_rgf.h"

namespace qt {
void count_launches(uint64_t n);   // qt_sse_launch_count accounting (qt_sse.cu)
}

namespace {

struct Z {
  double x, y;
};

// out[p][i][j] += Y[p][i][j] − conj(Y[p][j][i])  (the Y − Y† term of the backward lesser/greater step)
__global__ void k_add_antiherm(double2* __restrict__ out, int64_t out_stride, const double2* __restrict__ Y, int bs) {
  __shared__ double2 tile[32][33];
  const int p = blockIdx.z;
  const int i0 = blockIdx.y * 32, j0 = blockIdx.x * 32;
  const double2* y = Y + (int64_t)p * bs * bs;
  double2* o = out + (int64_t)p * out_stride;
  // tile of Y^T: rows j0.., columns i0..
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int j = j0 + r, i = i0 + threadIdx.x;
    if (j < bs && i < bs) tile[r][threadIdx.x] = y[(int64_t)j * bs + i];
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int i = i0 + r, j = j0 + threadIdx.x;
    if (i < bs && j < bs) {
      const double2 a = y[(int64_t)i * bs + j];
      const double2 b = tile[threadIdx.x][r];   // Y[j][i]
      double2 v = o[(int64_t)i * bs + j];
      v.x += a.x - b.x;
      v.y += a.y + b.y;
      o[(int64_t)i * bs + j] = v;
    }
  }
}

// out[p] += Zt[p] (elementwise, batched)
__global__ void k_add(double2* __restrict__ out, int64_t out_stride, const double2* __restrict__ Zt, int64_t n,
                      int64_t P) {
  const int64_t total = n * P;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = idx / n, e = idx - p * n;
    double2 v = out[p * out_stride + e];
    const double2 z = Zt[idx];
    v.x += z.x;
    v.y += z.y;
    out[p * out_stride + e] = v;
  }
}

// out[p] = I (P blocks of bs x bs at stride `stride`)
__global__ void k_set_identity(double2* __restrict__ out, int64_t stride, int bs, int64_t P) {
  const int64_t n = (int64_t)bs * bs, total = n * P;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = idx / n, e = idx - p * n;
    out[p * stride + e] = make_double2((e / bs) == (e % bs) ? 1.0 : 0.0, 0.0);
  }
}

constexpr int kRgfLanes = 16;   // concurrent per-point factorizations

}  // namespace

struct qt_rgf_plan_s {
  qt_rgf_desc d{};
  cublasHandle_t h = nullptr;
  double2* tmp = nullptr;          // 7 temporaries [7][P][bs][bs]
  int* piv = nullptr;              // [P][bs]
  int* info = nullptr;             // [bnum][P] getrf info, [P] getrs info
  // point groups: independent halves of the batch, each on its own stream + cuBLAS handle, so one group's
  // GEMMs overlap the other group's factorizations
  int ngroups = 1;
  cudaStream_t gs[2] = {};
  cublasHandle_t gh[2] = {};
  cudaEvent_t ev_start = nullptr, ev_gdone[2] = {};
  // per-point factorizations (cuSOLVER), fanned out over lanes
  int lanes = 0;
  cudaStream_t ls[kRgfLanes] = {};
  cusolverDnHandle_t sh[kRgfLanes] = {};
  double2* lwork = nullptr;        // [lanes][lwork_elems]
  int lwork_elems = 0;
  cudaEvent_t ev_fork = nullptr, ev_join[kRgfLanes] = {};
};

namespace {

qt_status cu(cudaError_t e) { return e == cudaSuccess ? QT_OK : (e == cudaErrorMemoryAllocation ? QT_ERR_OUT_OF_MEMORY : QT_ERR_CUDA); }
qt_status cb(cublasStatus_t s) {
  if (s == CUBLAS_STATUS_SUCCESS) return QT_OK;
  if (getenv("QT_DEBUG")) fprintf(stderr, "qt_rgf: cuBLAS status %d\n", (int)s);
  return s == CUBLAS_STATUS_ALLOC_FAILED ? QT_ERR_OUT_OF_MEMORY : QT_ERR_CUDA;
}
#define RG_TRY(x)                 \
  do {                            \
    qt_status s_ = (x);           \
    if (s_ != QT_OK) return s_;   \
  } while (0)

struct Grp {   // a contiguous range of points [p0, p0 + np) solved on its own stream
  int64_t p0, np;
  cublasHandle_t h;
  cudaStream_t s;
  int l0, nl;   // its factorization lanes
};

// row-major C[p] = alpha·opA(A[p])·opB(B[p]) + beta·C[p] for the group's points; cA / cB select X† (conjugate transpose)
qt_status gemm(qt_rgf_plan_s* q, const Grp& g, const double2* A, int64_t sA, bool cA, const double2* B, int64_t sB, bool cB,
               double2* C, int64_t sC, double ar, double br) {
  const int n = (int)q->d.bs;
  const cuDoubleComplex al = make_cuDoubleComplex(ar, 0.0), be = make_cuDoubleComplex(br, 0.0);
  return cb(cublasZgemmStridedBatched(g.h, cB ? CUBLAS_OP_C : CUBLAS_OP_N, cA ? CUBLAS_OP_C : CUBLAS_OP_N, n, n, n, &al,
                                      reinterpret_cast<const cuDoubleComplex*>(B), n, sB,
                                      reinterpret_cast<const cuDoubleComplex*>(A), n, sA, &be,
                                      reinterpret_cast<cuDoubleComplex*>(C), n, sC, (int)g.np));
}

// dst[p] = src[p] for the group's points (strided blocks of bs² complex)
qt_status copy(qt_rgf_plan_s* q, const Grp& g, double2* dst, int64_t sd, const double2* src, int64_t ss) {
  const size_t w = (size_t)q->d.bs * q->d.bs * sizeof(double2);
  return cu(cudaMemcpy2DAsync(dst, sd * sizeof(double2), src, ss * sizeof(double2), w, (size_t)g.np,
                              cudaMemcpyDeviceToDevice, g.s));
}

}  // namespace

extern "C" qt_status qt_rgf_count_flops(const qt_rgf_desc* d, double out[2]) {
  if (!d || !out || d->P <= 0 || d->bnum <= 0 || d->bs <= 0) return QT_ERR_INVALID_ARG;
  const double n3 = (double)d->bs * d->bs * d->bs, nb = (double)d->bnum;
  // forward: block 0: 4 GEMMs + 1 inversion; blocks 1..: 10 GEMMs + 1 inversion; backward: 11 GEMMs per block
  // 0..bnum-2 (Z = XT·g^R_n included); an inversion = LU (n³/3 complex MACs) + two triangular solves with n
  // right-hand sides (n³)
  const double gemms = 4.0 + 10.0 * (nb - 1.0) + 11.0 * (nb - 1.0);
  const double inv = nb * (4.0 / 3.0);
  out[0] = d->P * (gemms + inv) * n3 * 8.0;
  out[1] = d->P * 8.0 * (26.0 * nb - 25.0) * n3;
  return QT_OK;
}

extern "C" void qt_rgf_destroy(qt_rgf_plan_t q) {
  if (!q) return;
  for (int l = 0; l < q->lanes; ++l) {
    if (q->ls[l]) cudaStreamSynchronize(q->ls[l]);
    if (q->sh[l]) cusolverDnDestroy(q->sh[l]);
    if (q->ls[l]) cudaStreamDestroy(q->ls[l]);
    if (q->ev_join[l]) cudaEventDestroy(q->ev_join[l]);
  }
  if (q->ev_fork) cudaEventDestroy(q->ev_fork);
  for (int g = 0; g < 2; ++g) {
    if (q->gs[g]) cudaStreamSynchronize(q->gs[g]);
    if (q->gh[g]) cublasDestroy(q->gh[g]);
    if (q->gs[g]) cudaStreamDestroy(q->gs[g]);
    if (q->ev_gdone[g]) cudaEventDestroy(q->ev_gdone[g]);
  }
  if (q->ev_start) cudaEventDestroy(q->ev_start);
  cudaFree(q->lwork);
  if (q->h) cublasDestroy(q->h);
  cudaFree(q->tmp);
  cudaFree(q->piv);
  cudaFree(q->info);
  delete q;
}

extern "C" qt_status qt_rgf_plan(const qt_rgf_desc* d, void* stream, qt_rgf_plan_t* out) {
  if (!out) return QT_ERR_INVALID_ARG;
  *out = nullptr;
  if (!d || d->P <= 0 || d->bnum <= 0 || d->bs <= 0) return QT_ERR_INVALID_ARG;
  if (d->bs > 4096 || d->P > (1 << 20) || d->bnum > (1 << 20)) return QT_ERR_UNSUPPORTED;
  qt_rgf_plan_s* q = new (std::nothrow) qt_rgf_plan_s();
  if (!q) return QT_ERR_OUT_OF_MEMORY;
  q->d = *d;
  auto fail = [&](qt_status s) {
    qt_rgf_destroy(q);
    return s;
  };
  const size_t blk = (size_t)d->bs * d->bs;
  qt_status s;
  if ((s = cb(cublasCreate(&q->h))) != QT_OK) return fail(s);
  if ((s = cu(cudaMalloc(&q->tmp, 7 * d->P * blk * sizeof(double2)))) != QT_OK) return fail(s);
  if ((s = cu(cudaMalloc(&q->piv, d->P * d->bs * sizeof(int)))) != QT_OK) return fail(s);
  if ((s = cu(cudaMalloc(&q->info, (d->bnum + 1) * d->P * sizeof(int)))) != QT_OK) return fail(s);
  if ((s = cu(cudaMemsetAsync(q->info, 0, (d->bnum + 1) * d->P * sizeof(int), (cudaStream_t)stream))) != QT_OK) return fail(s);
  // one group: splitting the points into two concurrent halves measured 2.29 s vs 2.24 s at rgf_finfet (the
  // lanes already overlap the factorizations; half-size GEMM batches lose more than the overlap gains)
  q->ngroups = 1;
  if ((s = cu(cudaEventCreateWithFlags(&q->ev_start, cudaEventDisableTiming))) != QT_OK) return fail(s);
  for (int g = 0; g < q->ngroups; ++g) {
    if ((s = cu(cudaStreamCreateWithFlags(&q->gs[g], cudaStreamNonBlocking))) != QT_OK) return fail(s);
    if ((s = cu(cudaEventCreateWithFlags(&q->ev_gdone[g], cudaEventDisableTiming))) != QT_OK) return fail(s);
    if ((s = cb(cublasCreate(&q->gh[g]))) != QT_OK) return fail(s);
    if ((s = cb(cublasSetStream(q->gh[g], q->gs[g]))) != QT_OK) return fail(s);
  }
  q->lanes = (int)std::min<int64_t>(d->P, kRgfLanes);
  if ((s = cu(cudaEventCreateWithFlags(&q->ev_fork, cudaEventDisableTiming))) != QT_OK) return fail(s);
  for (int l = 0; l < q->lanes; ++l) {
    if ((s = cu(cudaStreamCreateWithFlags(&q->ls[l], cudaStreamNonBlocking))) != QT_OK) return fail(s);
    if ((s = cu(cudaEventCreateWithFlags(&q->ev_join[l], cudaEventDisableTiming))) != QT_OK) return fail(s);
    if (cusolverDnCreate(&q->sh[l]) != CUSOLVER_STATUS_SUCCESS) return fail(QT_ERR_CUDA);
    if (cusolverDnSetStream(q->sh[l], q->ls[l]) != CUSOLVER_STATUS_SUCCESS) return fail(QT_ERR_CUDA);
  }
  if (cusolverDnZgetrf_bufferSize(q->sh[0], (int)d->bs, (int)d->bs, reinterpret_cast<cuDoubleComplex*>(q->tmp),
                                  (int)d->bs, &q->lwork_elems) != CUSOLVER_STATUS_SUCCESS)
    return fail(QT_ERR_CUDA);
  if ((s = cu(cudaMalloc(&q->lwork, (size_t)q->lanes * std::max(q->lwork_elems, 1) * sizeof(double2)))) != QT_OK)
    return fail(s);
  if ((s = cu(cudaStreamSynchronize((cudaStream_t)stream))) != QT_OK) return fail(s);
  *out = q;
  return QT_OK;
}

namespace {

// The whole RGF pass for the points of one group, stream-ordered on g.s. Pointers are the group's first point.
qt_status solve_group(qt_rgf_plan_s* q, const Grp& g, const double2* Ad, const double2* Au, const double2* Al,
                      const double2* Sl, const double2* Sg, double2* GR, double2* GL, double2* GG) {
  const int64_t P = q->d.P, nb = q->d.bnum, bs = q->d.bs, blk = bs * bs, np = g.np;
  const int64_t sD = nb * blk, sO = (nb - 1) * blk;   // point strides of [P][bnum] and [P][bnum-1] tensors
  const cudaStream_t st = g.s;
  double2* T[7];
  for (int k = 0; k < 7; ++k) T[k] = q->tmp + (k * P + g.p0) * blk;   // the group's slice of each temporary
  const int n_i = (int)bs;
  // ---------------- forward pass: left-connected g^R_n (into GR), g^<_n (GL), g^>_n (GG).
  // Schedule: the inversion of M_{n+1} (per-point LU + solve on the lanes) runs concurrently with the eight GEMMs
  // of g^<_n, g^>_n on the group stream; only M_{n+1} itself (two GEMMs) waits for g^R_n.
  auto build_M = [&](int64_t n) -> qt_status {   // M_n = A_nn − A_{n,n-1} g^R_{n-1} A_{n-1,n} into T[0]
    RG_TRY(copy(q, g, T[0], blk, Ad + n * blk, sD));
    if (n > 0) {
      RG_TRY(gemm(q, g, Al + (n - 1) * blk, sO, false, GR + (n - 1) * blk, sD, false, T[1], blk, 1.0, 0.0));
      RG_TRY(gemm(q, g, T[1], blk, false, Au + (n - 1) * blk, sO, false, T[0], blk, -1.0, 1.0));
    }
    return QT_OK;
  };
  auto fork_inverse = [&](int64_t n) -> qt_status {   // g^R_n = M_n^{-1} on the lanes (identity written first)
    const int64_t tot = np * blk;
    k_set_identity<<<(int)std::min<int64_t>((tot + 255) / 256, 148 * 16), 256, 0, st>>>(GR + n * blk, sD, n_i, np);
    RG_TRY(cu(cudaGetLastError()));
    qt::count_launches(1);
    cudaEvent_t fork = g.l0 == 0 ? q->ev_fork : q->ev_gdone[1];
    RG_TRY(cu(cudaEventRecord(fork, st)));
    for (int l = g.l0; l < g.l0 + g.nl; ++l) RG_TRY(cu(cudaStreamWaitEvent(q->ls[l], fork, 0)));
    for (int64_t p = 0; p < np; ++p) {
      const int l = g.l0 + (int)(p % g.nl);
      cuDoubleComplex* Mp = reinterpret_cast<cuDoubleComplex*>(T[0] + p * blk);
      int* piv = q->piv + (g.p0 + p) * bs;
      if (cusolverDnZgetrf(q->sh[l], n_i, n_i, Mp, n_i, reinterpret_cast<cuDoubleComplex*>(q->lwork) + (size_t)l * q->lwork_elems,
                           piv, q->info + n * P + g.p0 + p) != CUSOLVER_STATUS_SUCCESS)
        return QT_ERR_CUDA;
      if (cusolverDnZgetrs(q->sh[l], CUBLAS_OP_N, n_i, n_i, Mp, n_i, piv,
                           reinterpret_cast<cuDoubleComplex*>(GR + p * sD + n * blk), n_i,
                           q->info + nb * P + g.p0 + p) != CUSOLVER_STATUS_SUCCESS)
        return QT_ERR_CUDA;
    }
    for (int l = g.l0; l < g.l0 + g.nl; ++l) RG_TRY(cu(cudaEventRecord(q->ev_join[l], q->ls[l])));
    return QT_OK;
  };
  auto join_inverse = [&]() -> qt_status {
    for (int l = g.l0; l < g.l0 + g.nl; ++l) RG_TRY(cu(cudaStreamWaitEvent(st, q->ev_join[l], 0)));
    return QT_OK;
  };
  RG_TRY(build_M(0));
  RG_TRY(fork_inverse(0));
  RG_TRY(join_inverse());
  for (int64_t n = 0; n < nb; ++n) {
    // M_{n+1} needs g^R_n (joined); its inversion overlaps the lesser/greater GEMMs of block n below. T[0] (M)
    // is free again: the lanes finished with M_n at the join.
    if (n + 1 < nb) {
      RG_TRY(build_M(n + 1));
      RG_TRY(fork_inverse(n + 1));
    }
    const double2* S[2] = {Sl, Sg};
    double2* G[2] = {GL, GG};
    for (int x = 0; x < 2; ++x) {
      double2* Sx = T[2];
      RG_TRY(copy(q, g, Sx, blk, S[x] + n * blk, sD));
      if (n > 0) {
        // Sx = Σ^x_n + A_{n,n-1} g^x_{n-1} A_{n,n-1}†
        RG_TRY(gemm(q, g, Al + (n - 1) * blk, sO, false, G[x] + (n - 1) * blk, sD, false, T[3], blk, 1.0, 0.0));
        RG_TRY(gemm(q, g, T[3], blk, false, Al + (n - 1) * blk, sO, true, Sx, blk, 1.0, 1.0));
      }
      // g^x_n = g^R_n Sx g^R_n†
      RG_TRY(gemm(q, g, GR + n * blk, sD, false, Sx, blk, false, T[3], blk, 1.0, 0.0));
      RG_TRY(gemm(q, g, T[3], blk, false, GR + n * blk, sD, true, G[x] + n * blk, sD, 1.0, 0.0));
    }
    if (n + 1 < nb) RG_TRY(join_inverse());
  }
  // ---------------- backward pass: G_{nb-1} = g_{nb-1}; block n <- block n+1
  const dim3 tb(32, 8), tg((unsigned)((bs + 31) / 32), (unsigned)((bs + 31) / 32), (unsigned)np);
  for (int64_t n = nb - 2; n >= 0; --n) {
    double2 *X = T[1], *Tt = T[2], *XT = T[3], *Zt = T[4], *Y = T[5], *W = T[6];
    RG_TRY(gemm(q, g, GR + n * blk, sD, false, Au + n * blk, sO, false, X, blk, 1.0, 0.0));        // X = g^R_n A_{n,n+1}
    RG_TRY(gemm(q, g, GR + (n + 1) * blk, sD, false, Al + n * blk, sO, false, Tt, blk, 1.0, 0.0)); // G^R_{n+1} A_{n+1,n}
    RG_TRY(gemm(q, g, X, blk, false, Tt, blk, false, XT, blk, 1.0, 0.0));                          // XT
    double2* Gx[2] = {GL, GG};
    for (int x = 0; x < 2; ++x) {
      double2* G = Gx[x];
      RG_TRY(gemm(q, g, XT, blk, false, G + n * blk, sD, false, Y, blk, 1.0, 0.0));                // Y = XT g^x_n
      RG_TRY(gemm(q, g, X, blk, false, G + (n + 1) * blk, sD, false, W, blk, 1.0, 0.0));           // W = X G^x_{n+1}
      RG_TRY(gemm(q, g, W, blk, false, X, blk, true, G + n * blk, sD, 1.0, 1.0));                  // g^x_n += W X†
      k_add_antiherm<<<tg, tb, 0, st>>>(G + n * blk, sD, Y, (int)bs);                               // += Y − Y†
      RG_TRY(cu(cudaGetLastError()));
      qt::count_launches(1);
    }
    RG_TRY(gemm(q, g, XT, blk, false, GR + n * blk, sD, false, Zt, blk, 1.0, 0.0));                // Z = XT g^R_n
    const int64_t tot = np * blk;
    const int grid = (int)std::min<int64_t>((tot + 255) / 256, 148 * 16);
    k_add<<<grid, 256, 0, st>>>(GR + n * blk, sD, Zt, blk, np);                                     // G^R_n = g^R_n + Z
    RG_TRY(cu(cudaGetLastError()));
    qt::count_launches(1);
  }
  return QT_OK;
}

}  // namespace

extern "C" qt_status qt_rgf_solve(qt_rgf_plan_t q, const void* Ad_, const void* Au_, const void* Al_, const void* Sl_,
                                  const void* Sg_, void* GR_, void* GL_, void* GG_, void* stream) {
  if (!q) return QT_ERR_INVALID_ARG;
  const void* ptrs[] = {Ad_, Sl_, Sg_, GR_, GL_, GG_};
  for (const void* p : ptrs)
    if (!p || (reinterpret_cast<uintptr_t>(p) & 15)) return QT_ERR_INVALID_ARG;
  if (q->d.bnum > 1 && (!Au_ || !Al_)) return QT_ERR_INVALID_ARG;
  if (GR_ == GL_ || GR_ == GG_ || GL_ == GG_) return QT_ERR_INVALID_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t P = q->d.P, nb = q->d.bnum, blk = q->d.bs * q->d.bs;
  const int64_t sD = nb * blk, sO = (nb - 1) * blk;
  // fork: the groups start after the caller's stream has produced the inputs; join before returning
  RG_TRY(cu(cudaEventRecord(q->ev_start, st)));
  const int G = q->ngroups;
  for (int gi = 0; gi < G; ++gi) {
    Grp g;
    g.p0 = P * gi / G;
    g.np = P * (gi + 1) / G - g.p0;
    g.h = q->gh[gi];
    g.s = q->gs[gi];
    g.nl = std::max(1, q->lanes / G);
    g.l0 = std::min(gi * g.nl, q->lanes - g.nl);
    RG_TRY(cu(cudaStreamWaitEvent(g.s, q->ev_start, 0)));
    RG_TRY(solve_group(q, g, (const double2*)Ad_ + g.p0 * sD, Au_ ? (const double2*)Au_ + g.p0 * sO : nullptr,
                       Al_ ? (const double2*)Al_ + g.p0 * sO : nullptr, (const double2*)Sl_ + g.p0 * sD,
                       (const double2*)Sg_ + g.p0 * sD, (double2*)GR_ + g.p0 * sD, (double2*)GL_ + g.p0 * sD,
                       (double2*)GG_ + g.p0 * sD));
  }
  for (int gi = 0; gi < G; ++gi) {
    RG_TRY(cu(cudaEventRecord(q->ev_gdone[gi], q->gs[gi])));
    RG_TRY(cu(cudaStreamWaitEvent(st, q->ev_gdone[gi], 0)));
  }
  return QT_OK;
}

extern "C" qt_status qt_rgf_check_info(qt_rgf_plan_t q, void* stream, int64_t* point, int64_t* block) {
  if (!q) return QT_ERR_INVALID_ARG;
  RG_TRY(cu(cudaStreamSynchronize((cudaStream_t)stream)));
  std::vector<int> h((q->d.bnum + 1) * q->d.P);
  RG_TRY(cu(cudaMemcpy(h.data(), q->info, h.size() * sizeof(int), cudaMemcpyDeviceToHost)));
  for (int64_t n = 0; n < q->d.bnum; ++n)
    for (int64_t p = 0; p < q->d.P; ++p)
      if (h[n * q->d.P + p] != 0) {
        if (point) *point = p;
        if (block) *block = n;
        return QT_ERR_INVALID_ARG;
      }
  return QT_OK;
}
