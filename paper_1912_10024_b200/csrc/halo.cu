// halo.cu — atom-sharded multi-GPU support: NCCL point-to-point exchange of the neighbour halo.
//
// Atom sharding is the paper's Ta tiling (T_E = 1): rank r owns the contiguous atom
// slab [a_lo(r), a_hi(r)) and computes Σ/Π for it; Eq. 3/4 also read G/D of the neighbour atoms, which
// (atoms are sorted along the transport axis) lie in a contiguous window [w_lo(r), w_hi(r)). Before a
// qt_sse_sigma/qt_sse_pi pair, each rank receives the window atoms owned by other ranks. On one node the
// peers are NVSwitch-connected, so this is one grouped ncclSend/ncclRecv round (no Alltoallv, no
// reduction: outputs are owner-computed).
#include <nccl.h>

#include "halo.cuh"

namespace qt {

// dst[o][k][u] = src[o][lo + k][u], o < outer, k < n atoms, u < inner16 (16-byte units)
__global__ void k_pack(const uint4* __restrict__ src, uint4* __restrict__ dst, int64_t outer, int64_t nwin,
                       int64_t lo, int64_t n, int64_t inner16) {
  const int64_t total = outer * n * inner16;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = i % inner16, r = i / inner16, k = r % n, o = r / n;
    dst[i] = src[(o * nwin + lo + k) * inner16 + u];
  }
}
__global__ void k_unpack(const uint4* __restrict__ src, uint4* __restrict__ dst, int64_t outer, int64_t nwin,
                         int64_t lo, int64_t n, int64_t inner16) {
  const int64_t total = outer * n * inner16;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = i % inner16, r = i / inner16, k = r % n, o = r / n;
    dst[(o * nwin + lo + k) * inner16 + u] = src[i];
  }
}

static int grid_for(int64_t total) {
  int64_t g = (total + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 16));
}

cudaError_t launch_pack(const void* src, void* dst, int64_t outer, int64_t nwin, int64_t lo, int64_t n,
                        int64_t inner_bytes, bool unpack, cudaStream_t st) {
  const int64_t inner16 = inner_bytes / 16, total = outer * n * inner16;
  if (total == 0) return cudaSuccess;
  if (unpack)
    k_unpack<<<grid_for(total), 256, 0, st>>>((const uint4*)src, (uint4*)dst, outer, nwin, lo, n, inner16);
  else
    k_pack<<<grid_for(total), 256, 0, st>>>((const uint4*)src, (uint4*)dst, outer, nwin, lo, n, inner16);
  return cudaGetLastError();
}

int nccl_unique_id(void* out128) {
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return 1;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  memcpy(out128, &id, sizeof(id));
  return 0;
}

int nccl_comm_init(void** comm, int nranks, const void* id128, int rank) {
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  ncclComm_t c;
  if (ncclCommInitRank(&c, nranks, id, rank) != ncclSuccess) return 1;
  *comm = c;
  return 0;
}

void nccl_comm_destroy(void* comm) {
  if (comm) ncclCommDestroy((ncclComm_t)comm);
}

// one grouped round of byte sends/receives; peers with 0 bytes are skipped
int nccl_exchange(void* comm, const std::vector<HaloPeer>& peers, const char* sendbuf, char* recvbuf,
                  cudaStream_t st) {
  if (ncclGroupStart() != ncclSuccess) return 1;
  for (const HaloPeer& h : peers) {
    if (h.send_bytes && ncclSend(sendbuf + h.send_off, h.send_bytes, ncclChar, h.rank, (ncclComm_t)comm, st) != ncclSuccess)
      return 1;
    if (h.recv_bytes && ncclRecv(recvbuf + h.recv_off, h.recv_bytes, ncclChar, h.rank, (ncclComm_t)comm, st) != ncclSuccess)
      return 1;
  }
  if (ncclGroupEnd() != ncclSuccess) return 1;
  return 0;
}

// in-place sum over ranks (energy sharding: each rank's Π holds the partial sum over its energies)
int nccl_allreduce_sum(void* comm, double* buf, size_t count, cudaStream_t st) {
  return ncclAllReduce(buf, buf, count, ncclDouble, ncclSum, (ncclComm_t)comm, st) == ncclSuccess ? 0 : 1;
}

}  // namespace qt
