// Function-level kernels behind the reference's standalone L1/L2 API:
//   gathered_score_kernel       kernels.py:244-261
//   gathered / dense weighted sum kernels.py:264-294 (fixed-order split reduce,
//                               the deterministic analogue of :163-181)
//   softmax_row                 linalg.py:76-92 (fp64 internally)
//   rope_apply / rope_apply_rows rope.py:38-75 (fp64)
//   _index_status               kernels.py:48-60
// These serve direct calls of those functions; the decode hot path is the
// fused kernel in loki_decode.cu.
#include <math_constants.h>

#include "loki_common.cuh"
#include "loki_internal.h"

namespace loki {
namespace {

template <typename T>
__device__ __forceinline__ float load_elem(const void* base, size_t off) {
  return Elem<T>::to_f(reinterpret_cast<const T*>(base)[off]);
}

// one warp per gathered row, lanes across the head dimension
template <typename T>
__global__ void gathered_scores_kernel(const float* __restrict__ Q, int M, const void* __restrict__ K,
                                       int64_t ks, int D, const int64_t* __restrict__ idx, int n,
                                       float* __restrict__ out) {
  const int warps = blockDim.x / 32;
  const int j = blockIdx.x * warps + warp_id();
  if (j >= n) return;
  const size_t row = (size_t)idx[j] * ks;
  for (int i = 0; i < M; ++i) {
    float acc = 0.f;
    for (int t = lane_id(); t < D; t += 32) acc = fmaf(Q[(size_t)i * D + t], load_elem<T>(K, row + t), acc);
    acc = warp_sum_width(acc, 32);
    if (lane_id() == 0) out[(size_t)i * n + j] = acc;
  }
}

// partial[s, t] = sum over rows of split s (ascending) of w[j] V[row_j, t]
template <typename T>
__global__ void wsum_partial_kernel(const float* __restrict__ w, const void* __restrict__ V, int64_t vs,
                                    int D, const int64_t* __restrict__ idx, int n, int per_split,
                                    float* __restrict__ partial) {
  const int s = blockIdx.y;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= D) return;
  const int j0 = s * per_split, j1 = min(n, j0 + per_split);
  float acc = 0.f;
  for (int j = j0; j < j1; ++j) {
    const size_t row = idx ? (size_t)idx[j] : (size_t)j;
    acc = fmaf(w[j], load_elem<T>(V, row * vs + t), acc);
  }
  partial[(size_t)s * D + t] = acc;
}

__global__ void wsum_reduce_kernel(const float* __restrict__ partial, int nsplit, int D, float* __restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= D) return;
  float acc = 0.f;
  for (int s = 0; s < nsplit; ++s) acc += partial[(size_t)s * D + t];
  out[t] = acc;
}

template <int NT>
__device__ double block_reduce_d(double v, bool is_max, double* scratch) {
  for (int off = 16; off > 0; off >>= 1) {
    const double o = __shfl_xor_sync(0xffffffffu, v, off);
    v = is_max ? fmax(v, o) : v + o;
  }
  __syncthreads();
  if (lane_id() == 0) scratch[warp_id()] = v;
  __syncthreads();
  double r = scratch[0];
  for (int i = 1; i < NT / 32; ++i) r = is_max ? fmax(r, scratch[i]) : r + scratch[i];
  return r;
}

template <int NT>
__global__ void __launch_bounds__(NT) softmax_rows_kernel(const float* __restrict__ x, int n, int64_t stride,
                                                          float* __restrict__ out) {
  __shared__ double scratch[NT / 32];
  const float* row = x + (size_t)blockIdx.x * stride;
  float* dst = out + (size_t)blockIdx.x * stride;
  double mx = -CUDART_INF;
  for (int j = threadIdx.x; j < n; j += NT) mx = fmax(mx, (double)row[j]);
  mx = block_reduce_d<NT>(mx, true, scratch);
  double sum = 0.0;
  for (int j = threadIdx.x; j < n; j += NT) sum += exp((double)row[j] - mx);
  sum = block_reduce_d<NT>(sum, false, scratch);
  for (int j = threadIdx.x; j < n; j += NT) dst[j] = (float)(exp((double)row[j] - mx) / sum);
}

template <typename IO>
__global__ void rope_kernel(const IO* __restrict__ x, IO* __restrict__ out, int64_t n_rows, int D,
                            const int64_t* __restrict__ positions, const double* __restrict__ inv_freq) {
  const int half = D / 2;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_rows * half) return;
  const int64_t r = i / half;
  const int c = (int)(i % half);
  const double theta = (double)positions[r] * inv_freq[c];
  double s, co;
  sincos(theta, &s, &co);
  const double lo = (double)x[r * D + c], hi = (double)x[r * D + c + half];
  out[r * D + c] = (IO)__dsub_rn(__dmul_rn(lo, co), __dmul_rn(hi, s));
  out[r * D + c + half] = (IO)__dadd_rn(__dmul_rn(lo, s), __dmul_rn(hi, co));
}

// first violation (in index order) wins, as in the reference's serial loop
__global__ void index_status_kernel(const int64_t* __restrict__ idx, int n, int64_t bound,
                                    int32_t* __restrict__ status) {
  __shared__ unsigned long long first;
  if (threadIdx.x == 0) first = ~0ull;
  __syncthreads();
  if (n > 0 && (idx[0] < 0 || idx[n - 1] >= bound)) {
    if (threadIdx.x == 0) *status = 2;
    return;
  }
  for (int j = 1 + threadIdx.x; j < n; j += blockDim.x) {
    unsigned long long code = ~0ull;
    if (idx[j] <= idx[j - 1]) code = ((unsigned long long)j << 2) | 1ull;
    else if (idx[j] >= bound) code = ((unsigned long long)j << 2) | 2ull;
    if (code != ~0ull) atomicMin(&first, code);
  }
  __syncthreads();
  if (threadIdx.x == 0) *status = (first == ~0ull) ? 0 : (int32_t)(first & 3ull);
}

}  // namespace

cudaError_t launch_gathered_scores(const float* Q, int M, const void* K, int64_t ks, int dtype, int D,
                                   const int64_t* idx, int n, float* out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int threads = 256, warps = threads / 32;
  const unsigned blocks = (unsigned)ceil_div(n, warps);
  if (dtype == LOKI_DTYPE_BF16)
    gathered_scores_kernel<__nv_bfloat16><<<blocks, threads, 0, st>>>(Q, M, K, ks, D, idx, n, out);
  else
    gathered_scores_kernel<float><<<blocks, threads, 0, st>>>(Q, M, K, ks, D, idx, n, out);
  return cudaGetLastError();
}

cudaError_t launch_weighted_sum(const float* w, const void* V, int64_t vs, int dtype, int D, const int64_t* idx,
                                int n, float* out, float* partial, int nsplit, cudaStream_t st) {
  const int per_split = ceil_div(n > 0 ? n : 1, nsplit);
  const int threads = D < 128 ? 32 * ceil_div(D, 32) : 128;
  dim3 grid((unsigned)ceil_div(D, threads), (unsigned)nsplit);
  if (dtype == LOKI_DTYPE_BF16)
    wsum_partial_kernel<__nv_bfloat16><<<grid, threads, 0, st>>>(w, V, vs, D, idx, n, per_split, partial);
  else
    wsum_partial_kernel<float><<<grid, threads, 0, st>>>(w, V, vs, D, idx, n, per_split, partial);
  wsum_reduce_kernel<<<(unsigned)ceil_div(D, threads), threads, 0, st>>>(partial, nsplit, D, out);
  return cudaGetLastError();
}

cudaError_t launch_softmax_rows(const float* x, int64_t rows, int n, int64_t stride, float* out, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  softmax_rows_kernel<256><<<(unsigned)rows, 256, 0, st>>>(x, n, stride, out);
  return cudaGetLastError();
}

cudaError_t launch_rope(const void* x, void* out, int io_dtype, int64_t n_rows, int D, const int64_t* positions,
                        const double* inv_freq, cudaStream_t st) {
  const int64_t work = n_rows * (D / 2);
  if (work <= 0) return cudaSuccess;
  const unsigned blocks = (unsigned)((work + 255) / 256);
  if (io_dtype == LOKI_DTYPE_F64)
    rope_kernel<double><<<blocks, 256, 0, st>>>(static_cast<const double*>(x), static_cast<double*>(out), n_rows, D,
                                                positions, inv_freq);
  else
    rope_kernel<float><<<blocks, 256, 0, st>>>(static_cast<const float*>(x), static_cast<float*>(out), n_rows, D,
                                               positions, inv_freq);
  return cudaGetLastError();
}

cudaError_t launch_index_status(const int64_t* idx, int n, int64_t bound, int32_t* status, cudaStream_t st) {
  index_status_kernel<<<1, 1024, 0, st>>>(idx, n, bound, status);
  return cudaGetLastError();
}

}  // namespace loki

// ---------------------------------------------------------------- row projection
// out[b, h, s, :] = x[b, h, s, :] . P[h / G]  (fp32 accumulate in index order):
// the PCA transform of whole caches / query blocks (the batched form of the
// k @ P / q @ P products of attention.py:201-202, e.g. for a prefill or an
// HF cache update).  One CTA per (b, h, 32-row block); P[h / G] staged in
// shared memory; I/O dtype f32 or bf16.
namespace loki {
namespace {

template <typename TI, typename TO>
__global__ void __launch_bounds__(128) project_rows_kernel(const TI* __restrict__ x, const float* __restrict__ P,
                                                          TO* __restrict__ out, int H, int S, int D, int G,
                                                          int64_t x_sb, int64_t x_sh, int64_t x_ss, int64_t o_sb,
                                                          int64_t o_sh, int64_t o_ss) {
  extern __shared__ float ps[];  // [D][D] then [32][D] rows
  const int bh = blockIdx.x, b = bh / H, h = bh % H;
  const int s0 = blockIdx.y * 32;
  const float* Ph = P + (size_t)(h / G) * D * D;
  float* xs = ps + (size_t)D * D;
  for (int i = threadIdx.x; i < D * D; i += blockDim.x) ps[i] = Ph[i];
  const int rows = min(32, S - s0);
  for (int i = threadIdx.x; i < rows * D; i += blockDim.x) {
    const int r = i / D, c = i % D;
    xs[i] = Elem<TI>::to_f(x[b * x_sb + h * x_sh + (int64_t)(s0 + r) * x_ss + c]);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < rows * D; i += blockDim.x) {
    const int r = i / D, c = i % D;
    float acc = 0.f;
    for (int t = 0; t < D; ++t) acc = fmaf(xs[r * D + t], ps[t * D + c], acc);
    out[b * o_sb + h * o_sh + (int64_t)(s0 + r) * o_ss + c] = Elem<TO>::from_f(acc);
  }
}

}  // namespace

cudaError_t launch_project_rows(const void* x, int x_dtype, const float* P, void* out, int out_dtype, int B, int H,
                                int S, int D, int G, const int64_t* xs, const int64_t* os, cudaStream_t st) {
  if (B == 0 || S == 0) return cudaSuccess;
  const size_t smem = (size_t)(D * D + 32 * D) * sizeof(float);
  dim3 grid((unsigned)(B * H), (unsigned)ceil_div(S, 32));
#define LOKI_PR(TI, TO)                                                                                      \
  do {                                                                                                       \
    auto k = project_rows_kernel<TI, TO>;                                                                    \
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);        \
    if (e != cudaSuccess) return e;                                                                          \
    k<<<grid, 128, smem, st>>>(static_cast<const TI*>(x), P, static_cast<TO*>(out), H, S, D, G, xs[0], xs[1], \
                               xs[2], os[0], os[1], os[2]);                                                  \
    return cudaGetLastError();                                                                               \
  } while (0)
  if (x_dtype == LOKI_DTYPE_BF16 && out_dtype == LOKI_DTYPE_BF16) LOKI_PR(__nv_bfloat16, __nv_bfloat16);
  if (x_dtype == LOKI_DTYPE_BF16 && out_dtype == LOKI_DTYPE_F32) LOKI_PR(__nv_bfloat16, float);
  if (x_dtype == LOKI_DTYPE_F32 && out_dtype == LOKI_DTYPE_BF16) LOKI_PR(float, __nv_bfloat16);
  LOKI_PR(float, float);
#undef LOKI_PR
}

}  // namespace loki
