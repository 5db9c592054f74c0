// Internal (non-ABI) declarations shared by the Loki CUDA translation units.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "loki_b200.h"

namespace loki {

// Kernel parameters of the fused decode kernel (loki_decode.cu).
struct FusedParams {
  const float* q_hat;        // [B, Hq, D] fp32
  const void* K;             // cache base pointers, element type per dtype
  const void* V;
  int64_t sb, sh, ss;        // element strides (batch, kv head, row)
  int B, Hq, Hkv, G, D, S_cap;
  const int32_t* lens;       // [B] cache lengths
  int d;
  double k_f;
  int k_fixed;
  int select_mode;           // 0 radix, 1 all, 2 external idx, 3 scores only
  const float* ext_scores;   // [B, Hq, S_cap] or null
  const int32_t* ext_idx;    // [B, Hq, idx_stride] or null
  int64_t idx_stride;
  float* out;
  int32_t* idx_out;
  float* approx_out;
  float* weights_out;
  int C;                     // CTAs per unit == cluster size
  int Lmax;                  // max rows per CTA slice
  uint32_t* keys_ws;         // global key store when it does not fit on chip
  int off_keys, off_sel, off_union, off_hist, off_merge, off_final, off_misc;
  float qscale;              // log2(e) / sqrt(D)
  int slice_align;           // slice length is a multiple of this (phase-1 tile rows)
  // TMA variant: ring of nst stages of stage_bytes at off_ring, mbarriers at off_bars
  int nst, stage_bytes, off_ring, off_bars;
  int r1, dbox;              // phase-1 box: r1 rows x dbox leading columns
  int r3;                    // phase-3 stage: r3 gathered rows of K and of V
  long long unit_rows;       // rows per (b, kv head) in the 2-D gather view (= S_cap)
  long long* trace;          // optional [grid][8] %globaltimer stamps at phase boundaries
  int debug;                 // LOKI_DEBUG bits (tuning experiments only): 1 = dense rows via gather4
};

// Phase-trace buffer installed by loki_set_phase_trace (diagnostics only).
extern long long* g_phase_trace;
extern int g_phase_trace_ctas;

struct Plan {
  int C = 1;
  int Lmax = 1;
  int G_T = 1;
  bool fast = false;
  bool tma = false;
  bool keys_in_smem = true;
  size_t smem = 0;
  size_t workspace = 0;
  int dtype = LOKI_DTYPE_F32;
};

// Opaque 128-byte TMA descriptors (CUtensorMap) built on the host.
struct alignas(64) TmaDesc {
  unsigned char bytes[128];
};

constexpr int kTmaWarps = 8;  // every warp streams through its own ring
constexpr int kTmaThreads = kTmaWarps * 32;

size_t fused_layout(int G_T, int NT, int D, int Lmax, bool keys_in_smem, FusedParams* p);
size_t fused_tma_layout(int G_T, int NT, int D, int Lmax, bool keys_in_smem, int nst, int stage_bytes,
                        FusedParams* p);
cudaError_t launch_fused(const FusedParams& p, const Plan& plan, cudaStream_t st);
bool tma_supported(int dtype, int D, int G_T);
cudaError_t launch_fused_tma(const FusedParams& p, const Plan& plan, const TmaDesc* maps, cudaStream_t st);
// Encode the five descriptors (lead boxes, K/V row gathers, K/V row boxes);
// false if TMA cannot address the cache.
bool encode_tma(const void* K, const void* V, const loki_kv_geom& g, int dbox, int r1, int r3, TmaDesc* maps);

// K0 transform / append (loki_append.cu)
cudaError_t launch_append(const float* q_raw, const float* k_raw, const float* v_new,
                          const float* P, int64_t P_head_stride, const double* inv_freq,
                          const int64_t* positions, int rope_mode, void* K, void* V,
                          const loki_kv_geom& g, const int32_t* rows, float* q_hat_out,
                          cudaStream_t st);

// function-level kernels (loki_kernels.cu)
cudaError_t launch_gathered_scores(const float* Q, int M, const void* K, int64_t k_row_stride, int dtype,
                                   int D, const int64_t* idx, int n, float* out, cudaStream_t st);
cudaError_t launch_weighted_sum(const float* w, const void* V, int64_t v_row_stride, int dtype, int D,
                                const int64_t* idx, int n, float* out, float* partial, int nsplit,
                                cudaStream_t st);
cudaError_t launch_softmax_rows(const float* x, int64_t rows, int n, int64_t stride, float* out,
                                cudaStream_t st);
cudaError_t launch_rope(const void* x, void* out, int io_dtype, int64_t n_rows, int D,
                        const int64_t* positions, const double* inv_freq, cudaStream_t st);
cudaError_t launch_index_status(const int64_t* idx, int n, int64_t bound, int32_t* status, cudaStream_t st);

}  // namespace loki
