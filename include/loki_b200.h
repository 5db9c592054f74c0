/*
 * loki_b200.h -- C ABI of the B200-native Loki decode-attention library
 * (libloki_b200.so, sm_100a).
 *
 * This is the drop-in boundary for the hot path named by BASELINE.json's
 * north star: the reference (`lokiattn`, a pure-Python/numba package) has no
 * FFI, so each entry point below replaces one reference Python function of
 * the path (file:line under /root/reference/pkg/src/lokiattn/).  The Python
 * package `paper_2406_02542_b200` binds these symbols with ctypes and mirrors
 * the reference API (same names, argument meaning and exception classes).
 *
 * Conventions
 *   - Every function returns loki_status; on failure loki_last_error()
 *     returns a thread-local message.  Argument errors are detected on the
 *     host before any launch, like the reference raising before compute.
 *   - All tensor pointers are DEVICE pointers; the caller owns all memory
 *     (query loki_decode_workspace_bytes for scratch).  No hidden allocation
 *     on the hot path; calls are asynchronous on `stream` (a cudaStream_t,
 *     NULL = legacy default stream).
 *   - KV caches are [B, Hkv, S_cap, D] with explicit element strides and a
 *     contiguous D axis, in fp32 (LOKI_DTYPE_F32 == the LKD1 dtype byte 0,
 *     dataio.py:43) or bf16.  Query heads map to KV heads as h -> h / (Hq/Hkv).
 *   - Internal / exported indices are int32 (function-level gathers take the
 *     reference's int64 indices).
 */
#ifndef LOKI_B200_H_
#define LOKI_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LOKI_ABI_VERSION 1

typedef int32_t loki_status;
#define LOKI_OK 0
#define LOKI_ERR_SHAPE 1       /* errors.py:20  ShapeError  */
#define LOKI_ERR_BUDGET 2      /* errors.py:24  BudgetError */
#define LOKI_ERR_INDEX 3       /* kernels.py:72 / linalg.py:137 IndexError */
#define LOKI_ERR_DOMAIN 4      /* errors.py:28  DomainError */
#define LOKI_ERR_CUDA 5        /* CUDA runtime / launch failure */
#define LOKI_ERR_UNSUPPORTED 6 /* shape outside the compiled kernel envelope */

#define LOKI_DTYPE_F32 0
#define LOKI_DTYPE_BF16 1
#define LOKI_DTYPE_F64 2 /* loki_rope I/O only (rope.py keeps the input dtype) */

/* attention.py:309-313 RotaryComposition, plus "no rotary" (loki_attention,
 * attention.py:188-206) and "rotary only" (rope_apply, rope.py:38-55). */
#define LOKI_ROPE_NONE 0
#define LOKI_ROPE_ROTATE_THEN_PROJECT 1
#define LOKI_ROPE_PROJECT_THEN_ROTATE 2

/* select modes of loki_decode */
#define LOKI_SELECT_TOPK 0     /* attention.py:166-185 loki_rank_and_attend      */
#define LOKI_SELECT_ALL 1      /* attention.py:137-142 vanilla_attention (dense) */
#define LOKI_SELECT_INDICES 2  /* kernels.py:244-279 gathered score/sum on given indices */
#define LOKI_SELECT_NONE 3     /* kernels.py:223-241 sliced_score_kernel only    */
/* Opt-in GQA mode (hard part 3): the Hq/Hkv query heads of a KV group share ONE selection of k
 * rows, ranked on the group's summed leading-d scores sum_g q_g[:d] . K_hat[j, :d]; every head then
 * attends over that selection exactly.  Composition of reference primitives: sliced_score_kernel on the
 * [G, D] query block (kernels.py:223-241) summed over the group -> topk_indices (linalg.py:95-118) ->
 * per-head attention.py:180-184.  Same as LOKI_SELECT_TOPK when Hq == Hkv.  bf16 caches, TMA-addressable
 * geometry (else LOKI_ERR_UNSUPPORTED).  Diagnostics: every head of a group reports the same indices
 * and the group score as its approx_scores. */
#define LOKI_SELECT_TOPK_SHARED 4

typedef struct loki_kv_geom {
  int32_t B, Hq, Hkv, D, S_cap;
  int32_t dtype;                        /* LOKI_DTYPE_F32 / LOKI_DTYPE_BF16 */
  int64_t stride_b, stride_h, stride_s; /* element strides of K and V */
} loki_kv_geom;

typedef struct loki_decode_args {
  const float* q_hat;      /* [B, Hq, D] fp32 contiguous, already in the PCA basis */
  const void* K;           /* rotated key cache  K_hat (KvCache.keys, attention.py:85-89) */
  const void* V;           /* value cache                (KvCache.values, attention.py:91-95) */
  loki_kv_geom g;
  const int32_t* lens;     /* [B] device: cached rows per batch, new token included */
  int32_t S_max;           /* upper bound of lens[] (<= S_cap): sizes the launch.  A row whose len
                              exceeds S_max attends over its first S_max rows only (a replayed graph
                              keeps its S_max: plan it at S_cap for a cache that grows) */
  int32_t d;               /* ranking columns, 1 <= d <= D (attention.py:176-177) */
  double k_f;              /* k_b = clamp(floor(k_f * len_b + 0.5), 1, len_b) (attention.py:40-46) */
  int32_t k_fixed;         /* > 0: use this k for every row instead (must be <= every len_b) */
  int32_t select_mode;     /* LOKI_SELECT_* */
  const float* ext_scores; /* optional [B, Hq, S_cap] fp32: rank these instead of approx scores */
  const int32_t* ext_idx;  /* SELECT_INDICES: ascending [B, Hq, idx_stride], k_b valid per row */
  int64_t idx_stride;      /* row stride of ext_idx / idx_out / weights_out */
  float* out;              /* [B, Hq, D] fp32 attention output; NULL = rank only */
  int32_t* idx_out;        /* optional [B, Hq, idx_stride]: LokiDiagnostics.indices */
  float* approx_out;       /* optional [B, Hq, S_cap]:     LokiDiagnostics.approx_scores */
  float* weights_out;      /* optional [B, Hq, idx_stride]: LokiDiagnostics.weights */
  void* workspace;
  size_t workspace_bytes;
  int32_t cluster_override; /* 0 = auto; else CTAs per (b, kv head): 1,2,4,8,16 */
} loki_decode_args;

/* ---------------------------------------------------------------- library */
const char* loki_last_error(void);
int32_t loki_abi_version(void);
/* LOKI_OK iff `device` is an sm_100 part this library was compiled for. */
loki_status loki_device_check(int32_t device);

/* ---------------------------------------------------------------- hot path */

/* Fused decode attention: approx scores -> top-k -> sparse exact attention.
 * Replaces attention.py:166-185 loki_rank_and_attend (and, with the select
 * modes above, vanilla_attention :137-142, sliced_score_kernel kernels.py:223,
 * topk_indices linalg.py:95 on given scores, and the gathered score + softmax
 * + weighted-sum chain kernels.py:244-279 / linalg.py:76-92). */
loki_status loki_decode(const loki_decode_args* args, void* stream);

/* Phase timing: the launches of one loki_decode step separately, for a plan that splits
 * the layer (S_max >= 8192 bf16, or group-shared selection).  launches = 1: the A launch only (approximate
 * scores over the leading d columns + the top-k selection, kernels.py:223-241 + linalg.py:95-118);
 * 2: the B launch only (gathered exact scores, softmax, weighted sum and the merge, kernels.py:244-279 +
 * linalg.py:76-92) -- it consumes the selections a preceding launches = 1 call left in the workspace;
 * 3: both (== loki_decode).  Same arguments and workspace as loki_decode; LOKI_ERR_UNSUPPORTED for
 * single-launch plans.  Not a serving entry point. */
loki_status loki_decode_phase(const loki_decode_args* args, int32_t launches, void* stream);

/* Scratch bytes loki_decode needs for `args` (0 for on-chip plans).
 * The workspace must be ZERO-FILLED before its first use (cudaMemset); every
 * launch leaves it zero-filled again (the persistent kernel's ticket counter,
 * per-unit arrival counters and histograms reset themselves), so one
 * workspace serves any number of launches on one stream.  Do not share one
 * workspace between launches that may run concurrently. */
loki_status loki_decode_workspace_bytes(const loki_decode_args* args, size_t* bytes);

/* Launch plan chosen for `args`: CTAs per unit (cluster kernels), 0 for the
 * persistent pipe kernel (one launch) or -2 for split pipe layers (an A-only and
 * a B-only launch); rows per CTA / chunk; dynamic smem. */
loki_status loki_decode_plan(const loki_decode_args* args, int32_t* ctas_per_unit,
                             int32_t* rows_per_cta, size_t* smem_bytes);

/* Key append with optional rotary + PCA transform (K0).
 * Replaces attention.py:188-206 (q @ P, k @ P, cache.append, :201-203) and
 * attention.py:316-341 transform_step (both RotaryComposition orders).
 *   q_raw  [B, Hq, D] fp32 or NULL      -> q_hat_out [B, Hq, D] fp32
 *   k_raw  [B, Hkv, D] fp32             -> K cache row rows[b] (dtype of g)
 *   v_new  [B, Hkv, D] fp32 or NULL     -> V cache row rows[b]
 *   P      [Hkv, D, D] fp32 row-major (columns = principal directions,
 *          calibration.py:117-123); P_head_stride 0 = one P for all heads;
 *          NULL with LOKI_ROPE_NONE = identity (plain append).
 *   inv_freq [D/2] fp64 = base ** (-2i/D) (rope.py:34), NULL when rope_mode NONE
 *   positions [B] int64 rotary position of the new token, NULL = rows[b]
 *   rows   [B] int32 destination row per batch (NULL = row 0). */
loki_status loki_append_kv(const float* q_raw, const float* k_raw, const float* v_new,
                           const float* P, int64_t P_head_stride, const double* inv_freq,
                           const int64_t* positions, int32_t rope_mode, void* K, void* V,
                           loki_kv_geom g, const int32_t* rows, float* q_hat_out, void* stream);

/* ---------------------------------------------------------------- function level */

/* kernels.py:244-261 gathered_score_kernel: out[i, j] = Q[i, :] . K[idx[j], :]
 * Q [M, D] fp32; K rows with row stride k_row_stride (elements); idx int64 [n]
 * ascending and in range (validated by the caller, kernels.py:63-73). */
loki_status loki_gathered_scores(const float* Q, int32_t M, const void* K, int64_t k_row_stride,
                                 int32_t dtype, int32_t D, const int64_t* idx, int32_t n,
                                 float* out, void* stream);

/* kernels.py:264-294 gathered / dense weighted sum: out = sum_j w[j] V[idx[j], :]
 * (idx NULL = dense rows 0..n-1).  `partial` is caller scratch of
 * loki_weighted_sum_workspace(n, D) bytes, reduced in fixed order. */
loki_status loki_weighted_sum(const float* w, const void* V, int64_t v_row_stride, int32_t dtype,
                              int32_t D, const int64_t* idx, int32_t n, float* out, void* partial,
                              size_t partial_bytes, void* stream);
size_t loki_weighted_sum_workspace(int32_t n, int32_t D);

/* linalg.py:76-92 softmax_row over each row of x [rows, n] (row stride `stride`);
 * fp64 max / exp / sum like the reference, fp32 out. */
loki_status loki_softmax_rows(const float* x, int64_t rows, int32_t n, int64_t stride, float* out,
                              void* stream);

/* rope.py:38-75 rope_apply / rope_apply_rows: row i of x [n_rows, D] rotates to
 * positions[i]; fp64 rotation, output in the input dtype (F32 or F64). */
loki_status loki_rope(const void* x, void* out, int32_t io_dtype, int64_t n_rows, int32_t D,
                      const int64_t* positions, const double* inv_freq, void* stream);

/* kernels.py:48-60 _index_status on device: *status = 0 ascending and in
 * [0, bound), 1 not strictly ascending, 2 out of range. */
loki_status loki_index_status(const int64_t* idx, int32_t n, int64_t bound, int32_t* status,
                              void* stream);

/* Batched PCA transform (the k @ P / q @ P products of attention.py:201-202
 * and transform_step's projection, attention.py:316-341, for whole blocks):
 *   out[b, h, s, :] = x[b, h, s, :] . P[h / G]
 * x, out: [B, H, S, D] with element strides {b, h, s} (D contiguous), dtype
 * f32 or bf16 each; P [H / G, D, D] fp32 row-major (calibration.py:117-123).
 * fp32 accumulation in index order.  D <= 128. */
loki_status loki_project_rows(const void* x, int32_t x_dtype, const int64_t* x_strides, const float* P,
                              void* out, int32_t out_dtype, const int64_t* out_strides, int32_t B, int32_t H,
                              int32_t S, int32_t D, int32_t G, void* stream);

/* Diagnostics: subsequent TMA-path loki_decode launches whose grid fits in
 * max_ctas record eight %globaltimer stamps per CTA into buf [max_ctas][8]
 * (start, phase 1 done, radix passes done, tie counts exchanged, selection
 * emitted, union built, phase 3 done, end).  NULL disables. */
loki_status loki_set_phase_trace(int64_t* buf, int32_t max_ctas);

#ifdef __cplusplus
}
#endif

#endif /* LOKI_B200_H_ */
