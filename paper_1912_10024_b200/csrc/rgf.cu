// rgf.cu — recursive Green's Function solver (include/qt_rgf.h): the GF phase of Eq. 1
// by the RGF forward/backward pass over the bnum diagonal blocks, batched over the independent
// (E, kz) points ("operating on all atoms for a specific energy-momentum pair").
//
// B200 mapping: every block step is a handful of dense bs x bs complex products, identical for all P points, so
// each is ONE strided-batched ZGEMM over the points (cuBLAS: a plain library GEMM on the FP64 tensor pipe), the
// block inversions are batched LU + inverse (cublasZgetrfBatched / getriBatched), and the only hand-written
// kernel is the anti-Hermitian update G^≷ += Y − Y† of the backward pass (tiled transpose in shared memory).
// The left-connected g^R, g^<, g^> live in the OUTPUT tensors (the backward pass overwrites block n after its
// last read), so the plan's scratch is seven bs x bs temporaries per point. Row-major blocks are handed to the
// column-major cuBLAS as their transposes: row-major C = op(A)·op(B) is column-major C^T = op(B)^T·op(A)^T,
// with op = N for X and op = C (conjugate transpose) for X†.
#include <cublas_v2.h>

#include <cstdio>
#include <cstdlib>
#include <new>
#include <vector>

#include "qt_rgf.h"

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

}  // namespace

struct qt_rgf_plan_s {
  qt_rgf_desc d{};
  cublasHandle_t h = nullptr;
  double2* tmp = nullptr;          // 7 temporaries [7][P][bs][bs]
  int* piv = nullptr;              // [P][bs]
  int* info = nullptr;             // [bnum][P] getrf info, [P] getri info
  double2** ptrM = nullptr;        // [P] -> temporary M
  double2** ptrG = nullptr;        // [bnum][P] -> block n of the G^R output (set per solve)
  std::vector<double2*> hptrG;
  const void* last_GR = nullptr;
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

// row-major C[p] = alpha·opA(A[p])·opB(B[p]) + beta·C[p] for p < P; conjA / conjB select X† (conjugate transpose)
qt_status gemm(qt_rgf_plan_s* q, const double2* A, int64_t sA, bool cA, const double2* B, int64_t sB, bool cB, double2* C,
               int64_t sC, double ar, double br) {
  const int n = (int)q->d.bs;
  const cuDoubleComplex al = make_cuDoubleComplex(ar, 0.0), be = make_cuDoubleComplex(br, 0.0);
  return cb(cublasZgemmStridedBatched(q->h, cB ? CUBLAS_OP_C : CUBLAS_OP_N, cA ? CUBLAS_OP_C : CUBLAS_OP_N, n, n, n, &al,
                                      reinterpret_cast<const cuDoubleComplex*>(B), n, sB,
                                      reinterpret_cast<const cuDoubleComplex*>(A), n, sA, &be,
                                      reinterpret_cast<cuDoubleComplex*>(C), n, sC, (int)q->d.P));
}

// dst[p] = src[p] for p < P (strided blocks of bs² complex)
qt_status copy(qt_rgf_plan_s* q, double2* dst, int64_t sd, const double2* src, int64_t ss, cudaStream_t st) {
  const size_t w = (size_t)q->d.bs * q->d.bs * sizeof(double2);
  return cu(cudaMemcpy2DAsync(dst, sd * sizeof(double2), src, ss * sizeof(double2), w, (size_t)q->d.P,
                              cudaMemcpyDeviceToDevice, st));
}

}  // namespace

extern "C" qt_status qt_rgf_count_flops(const qt_rgf_desc* d, double out[2]) {
  if (!d || !out || d->P <= 0 || d->bnum <= 0 || d->bs <= 0) return QT_ERR_INVALID_ARG;
  const double n3 = (double)d->bs * d->bs * d->bs, nb = (double)d->bnum;
  // forward: block 0: 4 GEMMs + 1 inversion; blocks 1..: 10 GEMMs + 1 inversion; backward: 10 GEMMs + 1 add-GEMM
  // per block 0..bnum-2 (Z = XT·g^R_n included); an LU (≈ n³/3 complex MACs... counted as getrf 1/3 + getri 2/3 = n³)
  const double gemms = 4.0 + 10.0 * (nb - 1.0) + 11.0 * (nb - 1.0);
  const double inv = nb * 1.0;
  out[0] = d->P * (gemms + inv) * n3 * 8.0;
  out[1] = d->P * 8.0 * (26.0 * nb - 25.0) * n3;
  return QT_OK;
}

extern "C" void qt_rgf_destroy(qt_rgf_plan_t q) {
  if (!q) return;
  if (q->h) cublasDestroy(q->h);
  cudaFree(q->tmp);
  cudaFree(q->piv);
  cudaFree(q->info);
  cudaFree(q->ptrM);
  cudaFree(q->ptrG);
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
  if ((s = cu(cudaMalloc(&q->ptrM, d->P * sizeof(double2*)))) != QT_OK) return fail(s);
  if ((s = cu(cudaMalloc(&q->ptrG, d->bnum * d->P * sizeof(double2*)))) != QT_OK) return fail(s);
  std::vector<double2*> pm(d->P);
  for (int64_t p = 0; p < d->P; ++p) pm[p] = q->tmp + p * blk;   // temporary 0 = M
  if ((s = cu(cudaMemcpyAsync(q->ptrM, pm.data(), d->P * sizeof(double2*), cudaMemcpyHostToDevice, (cudaStream_t)stream))) != QT_OK)
    return fail(s);
  if ((s = cu(cudaStreamSynchronize((cudaStream_t)stream))) != QT_OK) return fail(s);
  *out = q;
  return QT_OK;
}

extern "C" qt_status qt_rgf_solve(qt_rgf_plan_t q, const void* Ad_, const void* Au_, const void* Al_, const void* Sl_,
                                  const void* Sg_, void* GR_, void* GL_, void* GG_, void* stream) {
  if (!q) return QT_ERR_INVALID_ARG;
  const void* ptrs[] = {Ad_, Sl_, Sg_, GR_, GL_, GG_};
  for (const void* p : ptrs)
    if (!p || (reinterpret_cast<uintptr_t>(p) & 15)) return QT_ERR_INVALID_ARG;
  if (q->d.bnum > 1 && (!Au_ || !Al_)) return QT_ERR_INVALID_ARG;
  if (GR_ == GL_ || GR_ == GG_ || GL_ == GG_) return QT_ERR_INVALID_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  RG_TRY(cb(cublasSetStream(q->h, st)));
  const int64_t P = q->d.P, nb = q->d.bnum, bs = q->d.bs, blk = bs * bs;
  const double2* Ad = (const double2*)Ad_;
  const double2* Au = (const double2*)Au_;
  const double2* Al = (const double2*)Al_;
  const double2* Sl = (const double2*)Sl_;
  const double2* Sg = (const double2*)Sg_;
  double2* GR = (double2*)GR_;
  double2* GL = (double2*)GL_;
  double2* GG = (double2*)GG_;
  const int64_t sD = nb * blk, sO = (nb - 1) * blk;   // point strides of [P][bnum] and [P][bnum-1] tensors
  double2* T[7];
  for (int k = 0; k < 7; ++k) T[k] = q->tmp + k * P * blk;   // T[0] = M (pointer array ptrM)
  // pointer array of the G^R output blocks (inverse destinations), rebuilt when the output moves
  if (q->last_GR != GR_) {
    q->hptrG.resize(nb * P);
    for (int64_t n = 0; n < nb; ++n)
      for (int64_t p = 0; p < P; ++p) q->hptrG[n * P + p] = GR + p * sD + n * blk;
    RG_TRY(cu(cudaMemcpyAsync(q->ptrG, q->hptrG.data(), nb * P * sizeof(double2*), cudaMemcpyHostToDevice, st)));
    q->last_GR = GR_;
  }
  const int n_i = (int)bs;
  // ---------------- forward pass: left-connected g^R_n (into GR), g^<_n (GL), g^>_n (GG)
  for (int64_t n = 0; n < nb; ++n) {
    double2* M = T[0];
    RG_TRY(copy(q, M, blk, Ad + n * blk, sD, st));
    if (n > 0) {
      // T1 = A_{n,n-1} g^R_{n-1};  M = A_nn − T1 A_{n-1,n}
      RG_TRY(gemm(q, Al + (n - 1) * blk, sO, false, GR + (n - 1) * blk, sD, false, T[1], blk, 1.0, 0.0));
      RG_TRY(gemm(q, T[1], blk, false, Au + (n - 1) * blk, sO, false, M, blk, -1.0, 1.0));
    }
    // g^R_n = M^{-1}: batched LU in place, inverse into block n of GR
    RG_TRY(cb(cublasZgetrfBatched(q->h, n_i, reinterpret_cast<cuDoubleComplex**>(q->ptrM), n_i, q->piv, q->info + n * P,
                                  (int)P)));
    RG_TRY(cb(cublasZgetriBatched(q->h, n_i, reinterpret_cast<const cuDoubleComplex* const*>(q->ptrM), n_i, q->piv,
                                  reinterpret_cast<cuDoubleComplex**>(q->ptrG + n * P), n_i, q->info + nb * P, (int)P)));
    const double2* S[2] = {Sl, Sg};
    double2* G[2] = {GL, GG};
    for (int x = 0; x < 2; ++x) {
      double2* Sx = T[2];
      RG_TRY(copy(q, Sx, blk, S[x] + n * blk, sD, st));
      if (n > 0) {
        // Sx = Σ^x_n + A_{n,n-1} g^x_{n-1} A_{n,n-1}†
        RG_TRY(gemm(q, Al + (n - 1) * blk, sO, false, G[x] + (n - 1) * blk, sD, false, T[3], blk, 1.0, 0.0));
        RG_TRY(gemm(q, T[3], blk, false, Al + (n - 1) * blk, sO, true, Sx, blk, 1.0, 1.0));
      }
      // g^x_n = g^R_n Sx g^R_n†
      RG_TRY(gemm(q, GR + n * blk, sD, false, Sx, blk, false, T[3], blk, 1.0, 0.0));
      RG_TRY(gemm(q, T[3], blk, false, GR + n * blk, sD, true, G[x] + n * blk, sD, 1.0, 0.0));
    }
  }
  // ---------------- backward pass: G_{nb-1} = g_{nb-1}; block n <- block n+1
  const dim3 tb(32, 8), tg((unsigned)((bs + 31) / 32), (unsigned)((bs + 31) / 32), (unsigned)P);
  for (int64_t n = nb - 2; n >= 0; --n) {
    double2 *X = T[1], *Tt = T[2], *XT = T[3], *Zt = T[4], *Y = T[5], *W = T[6];
    RG_TRY(gemm(q, GR + n * blk, sD, false, Au + n * blk, sO, false, X, blk, 1.0, 0.0));        // X = g^R_n A_{n,n+1}
    RG_TRY(gemm(q, GR + (n + 1) * blk, sD, false, Al + n * blk, sO, false, Tt, blk, 1.0, 0.0)); // G^R_{n+1} A_{n+1,n}
    RG_TRY(gemm(q, X, blk, false, Tt, blk, false, XT, blk, 1.0, 0.0));                          // XT
    const double2* Gx[2] = {GL, GG};
    for (int x = 0; x < 2; ++x) {
      double2* G = const_cast<double2*>(Gx[x]);
      RG_TRY(gemm(q, XT, blk, false, G + n * blk, sD, false, Y, blk, 1.0, 0.0));                // Y = XT g^x_n
      RG_TRY(gemm(q, X, blk, false, G + (n + 1) * blk, sD, false, W, blk, 1.0, 0.0));           // W = X G^x_{n+1}
      RG_TRY(gemm(q, W, blk, false, X, blk, true, G + n * blk, sD, 1.0, 1.0));                  // g^x_n += W X†
      k_add_antiherm<<<tg, tb, 0, st>>>(G + n * blk, sD, Y, (int)bs);                            // += Y − Y†
      RG_TRY(cu(cudaGetLastError()));
    }
    RG_TRY(gemm(q, XT, blk, false, GR + n * blk, sD, false, Zt, blk, 1.0, 0.0));                // Z = XT g^R_n
    const int64_t tot = P * blk;
    const int grid = (int)std::min<int64_t>((tot + 255) / 256, 148 * 16);
    k_add<<<grid, 256, 0, st>>>(GR + n * blk, sD, Zt, blk, P);                                   // G^R_n = g^R_n + Z
    RG_TRY(cu(cudaGetLastError()));
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
