// K0: rotary + PCA transform of the new token's query / key and the cache
// append (attention.py:188-206 loki_attention lines :201-203, and
// attention.py:316-341 transform_step for both RotaryComposition orders).
//
// One CTA per (KV head, group of kBatch batches) loads that head's P once
// (64 KB fp32 at D = 128, L2-resident across heads) and applies it to the
// (G query + 1 key) vectors of each batch in the group.  RoPE is evaluated in
// fp64 with explicitly rounded products (no FMA contraction), exactly like
// the reference's numpy expression rope.py:47-55, then cast to fp32.
#include "loki_common.cuh"
#include "loki_internal.h"

namespace loki {
namespace {

constexpr int kBatch = 2;
constexpr int kThreads = 128;
constexpr int kVecChunk = 8;
constexpr int kSmemPMaxD = 128;  // P [D][D] fp32 staged on chip up to D = 128 (64 KB)

// rope.py:47-55: out[:h] = lo*cos - hi*sin ; out[h:] = lo*sin + hi*cos (fp64)
__device__ __forceinline__ void rope_pair(double lo, double hi, double theta, double& olo, double& ohi) {
  double s, c;
  sincos(theta, &s, &c);
  olo = __dsub_rn(__dmul_rn(lo, c), __dmul_rn(hi, s));
  ohi = __dadd_rn(__dmul_rn(lo, s), __dmul_rn(hi, c));
}

template <typename T, bool P_SMEM>
__global__ void __launch_bounds__(kThreads) append_kernel(
    const float* __restrict__ q_raw, const float* __restrict__ k_raw, const float* __restrict__ v_new,
    const float* __restrict__ P, int64_t P_head_stride, const double* __restrict__ inv_freq,
    const int64_t* __restrict__ positions, int rope_mode, T* __restrict__ K, T* __restrict__ V,
    loki_kv_geom g, const int32_t* __restrict__ rows, float* __restrict__ q_hat_out) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const int hk = blockIdx.x;
  const int b0 = blockIdx.y * kBatch;
  const int D = g.D, half = D / 2;
  const int G = g.Hq / g.Hkv;
  const int nb = min(kBatch, g.B - b0);
  const int per_b = (q_raw ? G : 0) + 1;  // vectors per batch: G queries then the key
  const int nv = nb * per_b;
  float* Ps = reinterpret_cast<float*>(smem_raw);           // [D][D] when P_SMEM
  float* x = Ps + (P_SMEM && P ? (size_t)D * D : 0);       // [nv][D]
  float* y = x + (size_t)nv * D;                            // [nv][D]
  const float* Ph = P ? P + (size_t)hk * P_head_stride : nullptr;

  // PDL: everything above overlaps the previous kernel; inputs are read below
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (P_SMEM && Ph) {  // stage this head's P with 16-byte loads (L2-resident across batches)
    const int n4 = D * D / 4;
    const float4* src = reinterpret_cast<const float4*>(Ph);
    float4* dst = reinterpret_cast<float4*>(Ps);
    for (int i = threadIdx.x; i < n4; i += kThreads) dst[i] = __ldg(src + i);
  }
  // gather inputs; rotate first when the composition is rotate-then-project
  for (int i = threadIdx.x; i < nv * D; i += kThreads) {
    const int v = i / D, col = i % D;
    const int bl = v / per_b, slot = v % per_b;
    const int bb = b0 + bl;
    const float* src = (slot < per_b - 1)
                           ? q_raw + ((size_t)bb * g.Hq + (size_t)hk * G + slot) * D
                           : k_raw + ((size_t)bb * g.Hkv + hk) * D;
    if (rope_mode == LOKI_ROPE_ROTATE_THEN_PROJECT) {
      if (col < half) {
        const double pos = (double)(positions ? positions[bb] : (rows ? rows[bb] : 0));
        const double theta = pos * inv_freq[col];
        double olo, ohi;
        rope_pair((double)src[col], (double)src[col + half], theta, olo, ohi);
        x[v * D + col] = (float)olo;
        x[v * D + col + half] = (float)ohi;
      }
    } else {
      x[v * D + col] = src[col];
    }
  }
  __syncthreads();

  // y = x @ P (fp32 accumulate in index order, like the reference's float32 matmul)
  for (int col = threadIdx.x; col < D; col += kThreads) {
    for (int v0 = 0; v0 < nv; v0 += kVecChunk) {
      float acc[kVecChunk];
#pragma unroll
      for (int u = 0; u < kVecChunk; ++u) acc[u] = 0.f;
      if (Ph) {
#pragma unroll 4
        for (int i = 0; i < D; ++i) {
          const float pij = P_SMEM ? Ps[i * D + col] : __ldg(Ph + (size_t)i * D + col);
#pragma unroll
          for (int u = 0; u < kVecChunk; ++u)
            if (v0 + u < nv) acc[u] = fmaf(x[(v0 + u) * D + i], pij, acc[u]);
        }
      } else {
#pragma unroll
        for (int u = 0; u < kVecChunk; ++u)
          if (v0 + u < nv) acc[u] = x[(v0 + u) * D + col];
      }
#pragma unroll
      for (int u = 0; u < kVecChunk; ++u)
        if (v0 + u < nv) y[(v0 + u) * D + col] = acc[u];
    }
  }
  __syncthreads();

  if (rope_mode == LOKI_ROPE_PROJECT_THEN_ROTATE) {
    for (int i = threadIdx.x; i < nv * half; i += kThreads) {
      const int v = i / half, col = i % half;
      const int bb = b0 + v / per_b;
      const double pos = (double)(positions ? positions[bb] : (rows ? rows[bb] : 0));
      double olo, ohi;
      rope_pair((double)y[v * D + col], (double)y[v * D + col + half], pos * inv_freq[col], olo, ohi);
      x[v * D + col] = (float)olo;  // reuse x as the output staging buffer
      x[v * D + col + half] = (float)ohi;
    }
    __syncthreads();
    y = x;
  }

  for (int i = threadIdx.x; i < nv * D; i += kThreads) {
    const int v = i / D, col = i % D;
    const int bl = v / per_b, slot = v % per_b;
    const int bb = b0 + bl;
    if (slot < per_b - 1) {
      q_hat_out[((size_t)bb * g.Hq + (size_t)hk * G + slot) * D + col] = y[i];
    } else {
      const int row = rows ? rows[bb] : 0;
      const size_t off = (size_t)bb * g.stride_b + (size_t)hk * g.stride_h + (size_t)row * g.stride_s + col;
      K[off] = Elem<T>::from_f(y[i]);
      if (v_new) V[off] = Elem<T>::from_f(v_new[((size_t)bb * g.Hkv + hk) * D + col]);
    }
  }
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <typename T, bool P_SMEM>
cudaError_t launch_append_t(dim3 grid, size_t smem, cudaStream_t st, const float* q_raw, const float* k_raw,
                            const float* v_new, const float* P, int64_t P_head_stride, const double* inv_freq,
                            const int64_t* positions, int rope_mode, void* K, void* V, const loki_kv_geom& g,
                            const int32_t* rows, float* q_hat_out) {
  auto kern = append_kernel<T, P_SMEM>;
  static size_t smem_set = 0;
  if (smem > smem_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    smem_set = smem;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, q_raw, k_raw, v_new, P, P_head_stride, inv_freq, positions, rope_mode,
                            static_cast<T*>(K), static_cast<T*>(V), g, rows, q_hat_out);
}

}  // namespace

cudaError_t launch_append(const float* q_raw, const float* k_raw, const float* v_new, const float* P,
                          int64_t P_head_stride, const double* inv_freq, const int64_t* positions,
                          int rope_mode, void* K, void* V, const loki_kv_geom& g, const int32_t* rows,
                          float* q_hat_out, cudaStream_t st) {
  const int G = g.Hq / g.Hkv;
  const int per_b = (q_raw ? G : 0) + 1;
  const bool p_smem = P != nullptr && g.D <= kSmemPMaxD && (reinterpret_cast<uintptr_t>(P) % 16) == 0 &&
                      (P_head_stride % 4) == 0 && (g.D % 4) == 0;
  const size_t smem = (size_t)2 * kBatch * per_b * g.D * sizeof(float) +
                      (p_smem ? (size_t)g.D * g.D * sizeof(float) : 0);
  dim3 grid((unsigned)g.Hkv, (unsigned)ceil_div(g.B, kBatch));
  cudaError_t e;
  if (g.dtype == LOKI_DTYPE_BF16)
    e = p_smem ? launch_append_t<__nv_bfloat16, true>(grid, smem, st, q_raw, k_raw, v_new, P, P_head_stride,
                                                       inv_freq, positions, rope_mode, K, V, g, rows, q_hat_out)
               : launch_append_t<__nv_bfloat16, false>(grid, smem, st, q_raw, k_raw, v_new, P, P_head_stride,
                                                        inv_freq, positions, rope_mode, K, V, g, rows, q_hat_out);
  else
    e = p_smem ? launch_append_t<float, true>(grid, smem, st, q_raw, k_raw, v_new, P, P_head_stride, inv_freq,
                                               positions, rope_mode, K, V, g, rows, q_hat_out)
               : launch_append_t<float, false>(grid, smem, st, q_raw, k_raw, v_new, P, P_head_stride, inv_freq,
                                                positions, rope_mode, K, V, g, rows, q_hat_out);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace loki
