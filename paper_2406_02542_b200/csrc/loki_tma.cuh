// TMA / mbarrier / shared-memory helpers shared by the TMA decode kernels
// (loki_decode_tma.cu, loki_pipe.cu).
#pragma once

#include <cuda.h>
#include <cstdio>

#include "loki_common.cuh"
#include "loki_internal.h"

namespace loki {
namespace tma {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* bar, unsigned parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Bounded wait: a transfer that never lands is reported and trapped (the
// kernel dies with an error) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  if (mbar_try(bar, parity)) return;
  for (unsigned long long n = 0;; ++n) {
    if (mbar_try(bar, parity)) return;
    if (n > (1ull << 26)) {
      printf("loki: mbarrier wait timeout block %d warp %d bar %p parity %u\n", (int)blockIdx.x,
             (int)(threadIdx.x >> 5), bar, parity);
      __trap();
    }
  }
}
__device__ __forceinline__ void tma_box4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::
          "r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* map, int col, int r0, int r1, int r2, int r3,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
      "%5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
      : "memory");
}
// Shared-memory operands as 32-bit addresses.  TMA instructions take uniform registers: operands that ptxas
// cannot prove warp-uniform cost a per-instruction waterfall loop (ELECT, R2UR.BROADCAST, BRA.U.ANY), so
// callers broadcast them from lane 0 first (__shfl_sync(~0u, x, 0) results are known uniform).
__device__ __forceinline__ void tma_gather4_u(uint32_t dst, const CUtensorMap* map, int col, int r0, int r1, int r2,
                                              int r3, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
      "%5, %6}], [%7];" ::"r"(dst),
      "l"(map), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_box4d_u(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::
          "r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
      : "memory");
}
// Called by every lane of a warp: the operands are broadcast from lane 0 (warp-uniform for ptxas) and lane 0
// arms the barrier and issues the box
__device__ __forceinline__ void tma_box4d_warp(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                               uint64_t* bar, unsigned bytes) {
  const uint32_t ds = __shfl_sync(0xffffffffu, smem_u32(dst), 0);
  const uint32_t bs = __shfl_sync(0xffffffffu, smem_u32(bar), 0);
  c1 = __shfl_sync(0xffffffffu, c1, 0);
  c2 = __shfl_sync(0xffffffffu, c2, 0);
  c3 = __shfl_sync(0xffffffffu, c3, 0);
  if ((threadIdx.x & 31) == 0) {
    mbar_expect_tx(bar, bytes);
    tma_box4d_u(ds, map, c0, c1, c2, c3, bs);
  }
}
__device__ __forceinline__ void prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

// VEC elements of a row chunk held in shared memory
template <typename T, int VEC>
__device__ __forceinline__ void lds_chunk(const uint8_t* p, float (&x)[VEC]) {
  if constexpr (sizeof(T) == 2) {
    static_assert(VEC == 8 || VEC == 4, "bf16 chunk");
    if constexpr (VEC == 8) {
      const uint4 u = *reinterpret_cast<const uint4*>(p);
      const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        x[2 * i] = __uint_as_float(w[i] << 16);
        x[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
      }
    } else {
      const uint2 u = *reinterpret_cast<const uint2*>(p);
      x[0] = __uint_as_float(u.x << 16);
      x[1] = __uint_as_float(u.x & 0xFFFF0000u);
      x[2] = __uint_as_float(u.y << 16);
      x[3] = __uint_as_float(u.y & 0xFFFF0000u);
    }
  } else {
    static_assert(VEC == 4, "fp32 chunk");
    const float4 u = *reinterpret_cast<const float4*>(p);
    x[0] = u.x;
    x[1] = u.y;
    x[2] = u.z;
    x[3] = u.w;
  }
}


__device__ __forceinline__ long long globaltimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
template <typename P>
__device__ __forceinline__ void trace(const P& p, int k) {
  if (p.trace != nullptr && threadIdx.x == 0 && !((p.debug & 4) && k > 0)) p.trace[(size_t)blockIdx.x * 8 + k] = globaltimer();
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Ring position: slot and parity advance together (no division in the loop).
struct RingPos {
  int slot = 0;
  unsigned phase = 0;
  int count = 0;  // uses of the ring so far
  int nst;
  __device__ __forceinline__ explicit RingPos(int n) : nst(n) {}
  __device__ __forceinline__ void advance(int n) {
    count += n;
    slot += n;
    while (slot >= nst) {
      slot -= nst;
      phase ^= 1u;
    }
  }
  // the slot at this position held an earlier transfer that its consumer must release first
  __device__ __forceinline__ bool reused() const { return count >= nst; }
};

template <int W>
__device__ __forceinline__ float sum_lanes(float v) {
#pragma unroll
  for (int off = W >> 1; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

}  // namespace tma
}  // namespace loki
