// halo.cuh — declarations for the atom-halo exchange (halo.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstring>
#include <vector>

namespace qt {

struct HaloPeer {
  int rank;
  int64_t send_lo, send_n;   // atoms this rank sends (window-local index of the first, count)
  int64_t recv_lo, recv_n;   // atoms this rank receives (window-local)
  size_t send_off, send_bytes, recv_off, recv_bytes;
};

cudaError_t launch_pack(const void* src, void* dst, int64_t outer, int64_t nwin, int64_t lo, int64_t n,
                        int64_t inner_bytes, bool unpack, cudaStream_t st);
int nccl_unique_id(void* out128);
int nccl_comm_init(void** comm, int nranks, const void* id128, int rank);
void nccl_comm_destroy(void* comm);
int nccl_exchange(void* comm, const std::vector<HaloPeer>& peers, const char* sendbuf, char* recvbuf,
                  cudaStream_t st);
int nccl_allreduce_sum(void* comm, double* buf, size_t count, cudaStream_t st);

}  // namespace qt
