// tc05.cuh — tcgen05 (5th-gen tensor core) helpers for sm_100a: TMEM allocation, UMMA shared-memory and
// instruction descriptors (kind::tf32), MMA issue / commit, TMEM -> register loads. Raw PTX; the
// descriptor bit layouts follow the sm_100 UMMA descriptor definition (K-major, 128-byte swizzle:
// 8-row x 128-byte atoms, SBO = 1024 B between 8-row groups, LBO unused (1), version 1).
#pragma once
#include <stdint.h>

#include "tma.cuh"

namespace qt {

// ---- TMEM allocation (one warp, .sync.aligned); the base address is written to shared memory
template <int kCols>
__device__ __forceinline__ void tmem_alloc(uint32_t* smem_dst) {
  static_assert(kCols >= 32 && kCols <= 512 && (kCols & (kCols - 1)) == 0, "TMEM columns: power of 2 in [32,512]");
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(smem_dst)),
               "n"(kCols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
}
template <int kCols>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "n"(kCols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

// ---- shared-memory matrix descriptor: K-major operand tile [rows][32 x 4-byte] written by TMA with
// CU_TENSOR_MAP_SWIZZLE_128B (tile base 1024-byte aligned). Advancing K by 8 tf32 = +32 bytes of start address.
__device__ __forceinline__ uint64_t umma_desc_k128(const void* smem_tile) {
  const uint32_t a = smem_u32(smem_tile);
  uint64_t d = 0;
  d |= (uint64_t)((a >> 4) & 0x3FFF);          // start address  [0,14)
  d |= (uint64_t)1 << 16;                      // LBO (unused for swizzled K-major) [16,30)
  d |= (uint64_t)(1024 >> 4) << 32;            // SBO = 1024 B    [32,46)
  d |= (uint64_t)1 << 46;                      // version = 1     [46,48)
  d |= (uint64_t)2 << 61;                      // layout: SWIZZLE_128B [61,64)
  return d;
}

// same for a tile [rows][16 x 4-byte] written with CU_TENSOR_MAP_SWIZZLE_64B (8-row x 64-byte atoms, SBO 512 B,
// base 512-byte aligned); K advances by 8 tf32 = +32 bytes within the 64-byte row
__device__ __forceinline__ uint64_t umma_desc_k64(const void* smem_tile) {
  const uint32_t a = smem_u32(smem_tile);
  uint64_t d = 0;
  d |= (uint64_t)((a >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;                      // layout: SWIZZLE_64B
  return d;
}

// ---- instruction descriptor, kind::tf32: D f32, A/B tf32, both K-major, M x N, optional negation
__host__ __device__ constexpr uint32_t umma_idesc_tf32(int M, int N, bool neg_a = false, bool neg_b = false) {
  return (1u << 4)                          // c_format = F32
         | (2u << 7) | (2u << 10)           // a_format = b_format = TF32
         | ((neg_a ? 1u : 0u) << 13) | ((neg_b ? 1u : 0u) << 14)
         | (0u << 15) | (0u << 16)          // a_major = b_major = K
         | ((uint32_t)(N >> 3) << 17)       // n_dim
         | ((uint32_t)(M >> 4) << 24);      // m_dim
}

// D[tmem] (+)= A[smem] · B[smem]^T   (single thread issues for the CTA)
__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, bool acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"((uint32_t)acc)
      : "memory");
}

// arrive on `bar` when all previously issued tcgen05.mma of this thread have completed
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}

// TMEM -> registers: this warp's 32 lanes (lane quarter warp%4), 16 consecutive 32-bit columns each
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// TMEM -> registers: 20 consecutive 32-bit columns (x16 + x4)
__device__ __forceinline__ void tmem_ld20(uint32_t taddr, float* v) {
  uint32_t r[20];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19])
               : "r"(taddr + 16));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 20; ++i) v[i] = __uint_as_float(r[i]);
}

}  // namespace qt
