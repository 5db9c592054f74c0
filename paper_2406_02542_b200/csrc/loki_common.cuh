// Shared device helpers for the Loki sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include <mutex>

#include "loki_b200.h"

namespace loki {

// Kernel attributes are per device: a per-device high-water mark of the dynamic
// shared memory attribute (and the non-portable cluster flag), set under a lock
// so concurrent callers and several GPUs in one process are safe.  Steady-state
// launches find the attribute already set and never call into the driver (which
// also keeps the call out of CUDA-graph capture).
struct KernelAttrs {
  static constexpr int kDevs = 64;
  std::mutex mu;
  size_t smem[kDevs] = {};
  bool nonportable[kDevs] = {};
  cudaError_t ensure(const void* kern, size_t bytes, bool nonportable_cluster = false) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kDevs) dev = kDevs - 1;
    std::lock_guard<std::mutex> lock(mu);
    if (bytes > smem[dev]) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
      if (e != cudaSuccess) return e;
      smem[dev] = bytes;
    }
    if (nonportable_cluster && !nonportable[dev]) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
      nonportable[dev] = true;
    }
    return cudaSuccess;
  }
  // resident CTAs per SM at `bytes` of dynamic smem (cached per device: the plan asks on every call)
  size_t occ_smem[kDevs] = {};
  int occ[kDevs] = {};
  int occupancy(const void* kern, int threads, size_t bytes) {
    if (ensure(kern, bytes) != cudaSuccess) return 0;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kDevs) dev = kDevs - 1;
    {
      std::lock_guard<std::mutex> lock(mu);
      if (occ_smem[dev] == bytes && occ[dev] > 0) return occ[dev];
    }
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, threads, bytes) != cudaSuccess) return 0;
    std::lock_guard<std::mutex> lock(mu);
    occ_smem[dev] = bytes;
    occ[dev] = n;
    return n;
  }
};

constexpr int kWarp = 32;

// ---------------------------------------------------------------- element IO
// Caches hold fp32 (exact reference semantics) or bf16 (HBM-halving) rows.
template <typename T> struct Elem;

template <> struct Elem<float> {
  static constexpr int kBytes = 4;
  __device__ __forceinline__ static float to_f(float x) { return x; }
  __device__ __forceinline__ static float from_f(float x) { return x; }
};

template <> struct Elem<__nv_bfloat16> {
  static constexpr int kBytes = 2;
  __device__ __forceinline__ static float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
  __device__ __forceinline__ static __nv_bfloat16 from_f(float x) { return __float2bfloat16_rn(x); }
};

// Streaming read-only vector loads: keep the once-read KV bytes out of L1.
__device__ __forceinline__ uint4 ldg_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ uint2 ldg_nc_v2(const void* p) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t ldg_nc_u32(const void* p) {
  uint32_t r;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ uint16_t ldg_nc_u16(const void* p) {
  uint16_t r;
  asm volatile("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(r) : "l"(p));
  return r;
}

// A VEC-element chunk of a row held as raw 32-bit words.
template <typename T, int VEC> struct Chunk {
  static constexpr int kBytes = VEC * Elem<T>::kBytes;
  static constexpr int kWords = (kBytes + 3) / 4;
  uint32_t w[kWords];

  __device__ __forceinline__ void load(const T* p) {
    if constexpr (kBytes == 16) {
      uint4 v = ldg_nc_v4(p);
      w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
    } else if constexpr (kBytes == 8) {
      uint2 v = ldg_nc_v2(p);
      w[0] = v.x; w[1] = v.y;
    } else if constexpr (kBytes == 4) {
      w[0] = ldg_nc_u32(p);
    } else {
      static_assert(kBytes == 2, "chunk size");
      w[0] = ldg_nc_u16(p);
    }
  }
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int i = 0; i < kWords; ++i) w[i] = 0u;
  }
  __device__ __forceinline__ float get(int i) const {
    if constexpr (sizeof(T) == 4) {
      return __uint_as_float(w[i]);
    } else {
      uint32_t word = w[i >> 1];
      uint32_t bits = (i & 1) ? (word & 0xFFFF0000u) : (word << 16);
      return __uint_as_float(bits);
    }
  }
};

// ---------------------------------------------------------------- ordering
// Order-preserving fp32 -> uint32 key: larger float <=> larger key.  -0.0 is
// canonicalised to +0.0 first because the reference treats them as ties
// (np.partition / == compare, linalg.py:110-113).  NaN is undefined (the
// reference itself returns fewer than k indices on NaN).
__device__ __forceinline__ uint32_t order_key(float f) {
  uint32_t u = __float_as_uint(f);
  if (u == 0x80000000u) u = 0u;
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key_to_float(uint32_t k) {
  uint32_t u = (k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k;
  return __uint_as_float(u);
}

// ---------------------------------------------------------------- budgets
// k = clamp(floor(f * n + 0.5), 1, n) exactly as Python evaluates it
// (attention.py:40-46): one rounded fp64 multiply, one rounded fp64 add, no
// FMA contraction.
__host__ __device__ __forceinline__ int resolve_fraction(double f, int n) {
#ifdef __CUDA_ARCH__
  double x = __dadd_rn(__dmul_rn(f, (double)n), 0.5);
#else
  volatile double prod = f * (double)n;
  double x = prod + 0.5;
#endif
  long long r = (long long)floor(x);
  if (r < 1) r = 1;
  if (r > n) r = n;
  return (int)r;
}

__device__ __forceinline__ int warp_id() { return threadIdx.x >> 5; }
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

template <typename T>
__device__ __forceinline__ T warp_sum_width(T v, int width) {
  for (int off = width >> 1; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

__host__ __device__ __forceinline__ int next_pow2(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}
__host__ __device__ __forceinline__ int ceil_div(int a, int b) { return (a + b - 1) / b; }
__host__ __device__ __forceinline__ size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

}  // namespace loki
