// tcgen05 (5th-generation tensor core) helpers for sm_100a: TMEM allocation, shared-memory matrix and
// instruction descriptors, the single-thread MMA issue, commit-to-mbarrier and the TMEM -> register load.
// Encodings follow the PTX ISA for tcgen05 (the same bit layout CUTLASS's cute/arch/mma_sm100_desc.hpp
// spells out as UMMA::SmemDescriptor / UMMA::InstrDescriptor).
#pragma once
#include <cstdint>

namespace loki {
namespace umma {

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// Shared-memory matrix descriptor of a K-major operand tile whose rows are one swizzle atom wide
// (rb = 64 or 128 bytes, TMA SWIZZLE_64B / SWIZZLE_128B) and stacked at rb bytes: core matrices of 8 rows,
// stride byte offset 8 * rb, leading byte offset unused for K-major swizzled layouts (1 by convention),
// version 1 (sm_100), layout type 4 (64B) / 2 (128B).  The tile base must be 1024-byte aligned; a K
// step inside the atom advances the start address by its byte offset.
__device__ __forceinline__ uint64_t smem_desc_kmajor(uint32_t saddr, int rb) {
  const uint64_t start = (uint64_t)((saddr >> 4) & 0x3FFFu);
  const uint64_t lbo = 1ull;
  const uint64_t sbo = (uint64_t)(((8u * (uint32_t)rb) >> 4) & 0x3FFFu);
  const uint64_t layout = rb == 128 ? 2ull : 4ull;
  return start | (lbo << 16) | (sbo << 32) | (1ull << 46) | (layout << 61);
}

// Instruction descriptor, kind::f16: A = B = bf16, D = f32, both K-major, M x N.
__host__ __device__ constexpr uint32_t idesc_bf16_f32(int M, int N) {
  return (1u << 4)                      // D format f32
         | (1u << 7)                    // A format bf16
         | (1u << 10)                   // B format bf16
         | ((uint32_t)(N >> 3) << 17)   // N / 8
         | ((uint32_t)(M >> 4) << 24);  // M / 16
}

// D[tmem] (+)= A[smem] * B[smem]^T, issued by one thread for the CTA.
__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                         bool accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"((uint32_t)accumulate)
      : "memory");
}

// The mbarrier completes (one arrival) once every tcgen05 operation this thread issued before it is done.
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_addr(bar))
               : "memory");
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// Whole-warp TMEM allocation of `ncols` (a power of two >= 32) columns; the address lands in *dst (smem).
__device__ __forceinline__ void alloc(uint32_t* dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(dst)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

// 32 TMEM lanes x 16 columns of 32 bits -> 16 registers per thread (thread i <- lane base + i).
__device__ __forceinline__ void ld_32x32b_x16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// generic-proxy shared-memory writes (an operand tile built by threads) made visible to the tensor core
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

}  // namespace umma
}  // namespace loki
