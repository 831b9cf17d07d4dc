// halo.cuh — declarations for the multi-GPU support (halo.cu): halo boxes, pack kernels, NCCL wrappers.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstring>
#include <vector>

namespace qt {

// a box of window entries: energies [e0, e0 + ne) x atoms [a0, a0 + na) (window-local); D boxes use ne = 1
struct HaloBox {
  int64_t e0 = 0, ne = 0, a0 = 0, na = 0;
};

struct HaloPeer {
  int rank = -1;
  HaloBox send_g, recv_g;   // G≷ entries this rank sends (owned) / receives (halo)
  HaloBox send_d, recv_d;   // D≷ atom halo (atom splits only; na = 0 otherwise)
  bool direct = false;      // energy-only split: G boxes are Nkz contiguous runs, sent/received in place
  size_t send_off = 0, send_bytes = 0, recv_off = 0, recv_bytes = 0;   // staging offsets (packed peers)
};

// dst[o][e][a][u] = src[o][e0 + e][a0 + a][u] (or the reverse with unpack), o < outer, e < ne, a < na,
// u < inner_bytes / 16; src spans [outer][span_e][span_a][inner]
cudaError_t launch_pack(const void* src, void* dst, int64_t outer, int64_t span_e, int64_t e0, int64_t ne, int64_t span_a,
                        int64_t a0, int64_t na, int64_t inner_bytes, bool unpack, cudaStream_t st);
int nccl_unique_id(void* out128);
int nccl_comm_init(void** comm, int nranks, const void* id128, int rank);
int nccl_comm_split(void* comm, int color, int key, void** out);
void nccl_comm_destroy(void* comm);
bool nccl_async_error(void* comm);
// one grouped send/recv round: packed peers from/to the staging buffers, direct peers from/to the G windows
// gwin[2] in place (kz_bytes = bytes per kz of a window, e_bytes = bytes per energy row of all window atoms)
int nccl_exchange(void* comm, const std::vector<HaloPeer>& peers, const char* sendbuf, char* recvbuf, void* const gwin[2],
                  int64_t Nkz, int64_t kz_bytes, int64_t e_bytes, cudaStream_t st);
int nccl_reduce_sum(void* comm, const double* send, double* recv, size_t count, int root, cudaStream_t st);

}  // namespace qt
