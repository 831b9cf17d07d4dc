// halo.cu — multi-GPU support: NCCL exchange of the input halo and the Π reduction.
//
// The ranks form the paper's Ta x TE grid: rank (ta, te) owns atom slab ta x energy slab te
// and computes Σ/Π for it. Eq. 3 reads G_b(E ± ħω) and D of the neighbour atoms, Eq. 4 reads G_b and G_a(E + ħω),
// so a rank's input window is its block plus an atom halo (the neighbour shells; atoms are sorted along the
// transport axis, so the window is contiguous) and an energy halo of Dmax = the largest ħω/ΔE on each side.
// Before the contractions each rank receives the window entries owned by other ranks: on one node the peers are
// NVSwitch-connected, so this is one grouped ncclSend/ncclRecv round (the paper's four Alltoallv become
// point-to-point boxes). Π sums over all energies: with TE > 1 its partial sums are reduced (ncclReduce) to the
// owner of each sub-slab.
#include <nccl.h>

#include "halo.cuh"

namespace qt {

__global__ void k_pack(const uint4* __restrict__ src, uint4* __restrict__ dst, int64_t outer, int64_t span_e,
                       int64_t e0, int64_t ne, int64_t span_a, int64_t a0, int64_t na, int64_t inner16, bool unpack) {
  const int64_t total = outer * ne * na * inner16;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = i % inner16;
    int64_t r = i / inner16;
    const int64_t a = r % na;
    r /= na;
    const int64_t e = r % ne, o = r / ne;
    const int64_t w = ((o * span_e + e0 + e) * span_a + a0 + a) * inner16 + u;
    if (unpack)
      dst[w] = src[i];
    else
      dst[i] = src[w];
  }
}

static int grid_for(int64_t total) {
  int64_t g = (total + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 16));
}

cudaError_t launch_pack(const void* src, void* dst, int64_t outer, int64_t span_e, int64_t e0, int64_t ne, int64_t span_a,
                        int64_t a0, int64_t na, int64_t inner_bytes, bool unpack, cudaStream_t st) {
  const int64_t inner16 = inner_bytes / 16, total = outer * ne * na * inner16;
  if (total == 0) return cudaSuccess;
  k_pack<<<grid_for(total), 256, 0, st>>>((const uint4*)src, (uint4*)dst, outer, span_e, e0, ne, span_a, a0, na, inner16,
                                          unpack);
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

// collective over `comm`: ranks with the same color form a new communicator, ordered by key
int nccl_comm_split(void* comm, int color, int key, void** out) {
  ncclComm_t c = nullptr;
  if (ncclCommSplit((ncclComm_t)comm, color, key, &c, nullptr) != ncclSuccess) return 1;
  *out = c;
  return 0;
}

void nccl_comm_destroy(void* comm) {
  if (comm) ncclCommDestroy((ncclComm_t)comm);
}

// an asynchronous failure of an earlier operation (network, peer, internal), not "still in progress"
bool nccl_async_error(void* comm) {
  ncclResult_t r = ncclSuccess;
  if (ncclCommGetAsyncError((ncclComm_t)comm, &r) != ncclSuccess) return true;
  return r != ncclSuccess && r != ncclInProgress;
}

int nccl_exchange(void* comm, const std::vector<HaloPeer>& peers, const char* sendbuf, char* recvbuf, void* const gwin[2],
                  int64_t Nkz, int64_t kz_bytes, int64_t e_bytes, cudaStream_t st) {
  ncclComm_t c = (ncclComm_t)comm;
  if (ncclGroupStart() != ncclSuccess) return 1;
  int bad = 0;
  for (const HaloPeer& h : peers) {
    if (h.direct) {
      for (int x = 0; x < 2 && !bad; ++x)
        for (int64_t kz = 0; kz < Nkz && !bad; ++kz) {
          char* base = static_cast<char*>(gwin[x]) + kz * kz_bytes;
          if (h.send_g.ne)
            bad |= ncclSend(base + h.send_g.e0 * e_bytes, (size_t)(h.send_g.ne * e_bytes), ncclChar, h.rank, c, st) !=
                   ncclSuccess;
          if (h.recv_g.ne)
            bad |= ncclRecv(base + h.recv_g.e0 * e_bytes, (size_t)(h.recv_g.ne * e_bytes), ncclChar, h.rank, c, st) !=
                   ncclSuccess;
        }
    } else {
      if (h.send_bytes)
        bad |= ncclSend(sendbuf + h.send_off, h.send_bytes, ncclChar, h.rank, c, st) != ncclSuccess;
      if (h.recv_bytes)
        bad |= ncclRecv(recvbuf + h.recv_off, h.recv_bytes, ncclChar, h.rank, c, st) != ncclSuccess;
    }
    if (bad) break;
  }
  // always close the group, also after a failed enqueue (an open group would capture the next NCCL call)
  if (ncclGroupEnd() != ncclSuccess) return 1;
  return bad;
}

int nccl_reduce_sum(void* comm, const double* send, double* recv, size_t count, int root, cudaStream_t st) {
  return ncclReduce(send, recv, count, ncclDouble, ncclSum, root, (ncclComm_t)comm, st) == ncclSuccess ? 0 : 1;
}

}  // namespace qt
