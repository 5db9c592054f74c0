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
constexpr int kThreads = 512;  // r02: 128 -> 512 threads, the matvec split over row blocks (C2 K0 12.7 us alone)
constexpr int kVecChunk = 8;
constexpr int kSmemPMaxD = 128;  // P [D][D] fp32 staged on chip up to D = 128 (64 KB)

// Row blocks of the K0 matvec: the largest power of two KS with KS * D <= kThreads that divides D.
__host__ __device__ constexpr int row_blocks(int D) {
  int ks = 1;
  while (2 * ks * D <= kThreads && D % (2 * ks) == 0) ks *= 2;
  return ks;
}

// rope.py:47-55: out[:h] = lo*cos - hi*sin ; out[h:] = lo*sin + hi*cos (fp64)
__device__ __forceinline__ void rope_pair(double lo, double hi, double theta, double& olo, double& ohi) {
  double s, c;
  sincos(theta, &s, &c);
  olo = __dsub_rn(__dmul_rn(lo, c), __dmul_rn(hi, s));
  ohi = __dadd_rn(__dmul_rn(lo, s), __dmul_rn(hi, c));
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <typename T, bool P_SMEM>
__global__ void __launch_bounds__(kThreads) append_kernel(
    const float* __restrict__ q_raw, const float* __restrict__ k_raw, const float* __restrict__ v_new,
    const float* __restrict__ P, int64_t P_head_stride, const double* __restrict__ inv_freq,
    const int64_t* __restrict__ positions, int rope_mode, T* __restrict__ K, T* __restrict__ V,
    loki_kv_geom g, const int32_t* __restrict__ rows, float* __restrict__ q_hat_out) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t p_bar;
  const int hk = blockIdx.x;
  const int b0 = blockIdx.y * kBatch;
  const int D = g.D, half = D / 2;
  const int G = g.Hq / g.Hkv;
  const int nb = min(kBatch, g.B - b0);
  const int per_b = (q_raw ? G : 0) + 1;  // vectors per batch: G queries then the key
  const int nv = nb * per_b;
  const int nv4 = (nv + 3) & ~3;          // padded to whole float4 groups of vectors
  float* Ps = reinterpret_cast<float*>(smem_raw);           // [D][D] when P_SMEM
  float* x = Ps + (P_SMEM && P ? (size_t)D * D : 0);       // [nv4][D], zero padded
  float* y = x + (size_t)nv4 * D;                           // [nv4][D]
  const float* Ph = P ? P + (size_t)hk * P_head_stride : nullptr;

  // P is a constant of the layer: its bulk copy starts before the PDL wait, so
  // it overlaps the tail of the previous kernel
  const bool stage_p = P_SMEM && Ph != nullptr;
  if (stage_p && threadIdx.x == 0) {
    const uint32_t bytes = (uint32_t)(D * D * sizeof(float));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&p_bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&p_bar)), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(Ps)),
        "l"(Ph), "r"(bytes), "r"(smem_addr(&p_bar))
        : "memory");
  }
  // every thread waits on p_bar below: none may touch it before thread 0 has initialised it
  // (compute-sanitizer racecheck / synccheck, r02)
  if (stage_p) __syncthreads();
  // PDL: inputs (the previous layer's products in a real model) are read below
  asm volatile("griddepcontrol.wait;" ::: "memory");

  // gather inputs; rotate first when the composition is rotate-then-project
  for (int i = threadIdx.x; i < nv4 * D; i += kThreads) {
    const int v = i / D, col = i % D;
    if (v >= nv) {
      x[i] = 0.f;
      continue;
    }
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
  if (stage_p) {
    uint32_t ok = 0;
    while (!ok)
      asm volatile(
          "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(ok)
          : "r"(smem_addr(&p_bar))
          : "memory");
  }
  __syncthreads();

  // y = x @ P: thread (col, kq) accumulates rows [kq R, (kq + 1) R) of P for column col (fp32, index
  // order), the KS partial sums are then added in kq order; four vectors per pass, float4 broadcast reads
  // of x.  (KS = kThreads / D row blocks: the dependent FMA chain is D / KS long instead of D.)
  const int KS = row_blocks(D);
  const int R = D / KS;
  float* part = y + (size_t)nv4 * D;  // [KS][nv4][D]
  for (int t = threadIdx.x; t < KS * D; t += kThreads) {
    const int col = t % D, kq = t / D;
    const int i_lo = kq * R, i_hi = i_lo + R;
    for (int v0 = 0; v0 < nv4; v0 += 4) {
      float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
      if (Ph && ((D & 3) || (R & 3))) {  // odd widths: plain scalar walk
        for (int i = i_lo; i < i_hi; ++i) {
          const float pij = P_SMEM ? Ps[i * D + col] : __ldg(Ph + (size_t)i * D + col);
          a0 = fmaf(x[(v0 + 0) * D + i], pij, a0);
          a1 = fmaf(x[(v0 + 1) * D + i], pij, a1);
          a2 = fmaf(x[(v0 + 2) * D + i], pij, a2);
          a3 = fmaf(x[(v0 + 3) * D + i], pij, a3);
        }
      } else if (Ph) {
#pragma unroll 4
        for (int i = i_lo; i < i_hi; i += 4) {
          float p4[4];
#pragma unroll
          for (int t4 = 0; t4 < 4; ++t4)
            p4[t4] = P_SMEM ? Ps[(i + t4) * D + col] : __ldg(Ph + (size_t)(i + t4) * D + col);
          const float4 x0 = *reinterpret_cast<const float4*>(x + (v0 + 0) * D + i);
          const float4 x1 = *reinterpret_cast<const float4*>(x + (v0 + 1) * D + i);
          const float4 x2 = *reinterpret_cast<const float4*>(x + (v0 + 2) * D + i);
          const float4 x3 = *reinterpret_cast<const float4*>(x + (v0 + 3) * D + i);
          a0 = fmaf(x0.w, p4[3], fmaf(x0.z, p4[2], fmaf(x0.y, p4[1], fmaf(x0.x, p4[0], a0))));
          a1 = fmaf(x1.w, p4[3], fmaf(x1.z, p4[2], fmaf(x1.y, p4[1], fmaf(x1.x, p4[0], a1))));
          a2 = fmaf(x2.w, p4[3], fmaf(x2.z, p4[2], fmaf(x2.y, p4[1], fmaf(x2.x, p4[0], a2))));
          a3 = fmaf(x3.w, p4[3], fmaf(x3.z, p4[2], fmaf(x3.y, p4[1], fmaf(x3.x, p4[0], a3))));
        }
      } else if (kq == 0) {
        a0 = x[(v0 + 0) * D + col];
        a1 = x[(v0 + 1) * D + col];
        a2 = x[(v0 + 2) * D + col];
        a3 = x[(v0 + 3) * D + col];
      }
      float* pp = part + ((size_t)kq * nv4 + v0) * D + col;
      pp[0] = a0;
      pp[D] = a1;
      pp[2 * D] = a2;
      pp[3 * D] = a3;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nv4 * D; i += kThreads) {  // partial sums in row-block order
    float acc = part[i];
    for (int kq = 1; kq < KS; ++kq) acc += part[(size_t)kq * nv4 * D + i];
    y[i] = acc;
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
  static KernelAttrs attrs;
  {
    cudaError_t e = attrs.ensure(reinterpret_cast<const void*>(kern), smem);
    if (e != cudaSuccess) return e;
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
                      (P_head_stride % 4) == 0;
  const size_t nv4 = ((size_t)kBatch * per_b + 3) & ~(size_t)3;
  const size_t ks = (size_t)row_blocks(g.D);  // row blocks of the matvec (partial sums on chip)
  const size_t smem = (size_t)(2 + ks) * nv4 * g.D * sizeof(float) + (p_smem ? (size_t)g.D * g.D * sizeof(float) : 0);
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
