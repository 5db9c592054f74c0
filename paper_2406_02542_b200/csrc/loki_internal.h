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
  const int32_t* lens;       // [B] cache lengths (clamped to S_max: the plan covers S_max rows per unit)
  int S_max;
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
  long long row_sb, row_sh;  // the 2-D gather view: row of (b, kv head, s) = b * row_sb + h * row_sh + s
  long long* trace;          // optional [grid][8] %globaltimer stamps at phase boundaries
  int debug;                 // LOKI_DEBUG bits (tuning experiments only): 1 = dense rows via gather4
};

// Persistent pipelined decode (loki_pipe.cu): a grid of resident CTAs draws
// tickets from one global counter; ticket -> work item
//   A(u, c)  phase 1 of chunk c of unit u (approx scores -> keys, histogram);
//            the last A arriver of a unit runs its top-k selection
//   B(u, q)  phase 3 over rows [q * Lc, (q + 1) * Lc) of unit u: picks its
//            selected rows from the keys and the published thresholds, gathers
//            them, online softmax -> partial state; the last B arriver merges.
// B(u, *) tickets come `lag` units after A(u, *), so other CTAs keep HBM busy
// while a unit's selection runs.  The workspace must be zero on first use;
// every launch leaves it zero again (counters / histograms self-reset).
// Key-stream buffers of the warp-specialised A launch's select group (16 KB each): the key passes are
// L2-latency bound, so four chunks are kept in flight (r02: two left a 32K-key pass at ~7 GB/s).
constexpr int kSelNB = 4;
// ... in use: four for per-head groups (G passes per unit), two for G = 1 (its shared memory goes to a
// fourth stream stage instead: r02, TGT)
__host__ __device__ constexpr int sel_nb(int G_T) { return G_T > 1 ? kSelNB : 2; }

struct PipeParams {
  const float* q_hat;  // [B, Hq, D]
  int B, Hq, Hkv, G, D, S_cap;
  const int32_t* lens;  // [B] cache lengths, clamped to S_max (the ticket space covers S_max rows per unit)
  int S_max;
  int d;
  double k_f;
  int k_fixed;
  int64_t idx_stride;
  float* out;
  int32_t* idx_out;
  float* approx_out;
  float* weights_out;
  float qscale;  // log2(e) / sqrt(D)
  int nst, stage_bytes, off_ring, off_bars, off_hist, off_ents;
  int r1, dbox, r3;
  long long row_sb, row_sh;  // the 2-D gather view: row of (b, kv head, s) = b * row_sb + h * row_sh + s
  int units, Lc, nA, lag, hbits, cand_cap;  // Lc / nA: B-part rows / B parts per unit
  int La, nAa;       // A-chunk rows / A chunks per unit (La >= Lc: phase-1 items are not overhead-bound)
  long long n_tickets;
  int split_k;       // 1: phase 3 gathers K columns [d, D) only and reuses the phase-1 partial score
  int mma;           // 1: tensor-core phase 3 (bf16 caches): 8-row stages of 128B-swizzled row halves
  int lead_swz;      // 64 / 128: lead rows of that many bytes, TMA-swizzled, one lane per row (G == 1); 0: off
  uint32_t* ctrl;    // [2 + 4 * units]: ticket, exits, then per unit {A arrivals, B arrivals, ready, -}
  uint32_t* hist;    // [units][G][1 << hbits]
  uint32_t* keys;    // [units][G][kstride] order keys of the approx scores
  int kstride;       // S_cap rounded up to a multiple of 4 (uint4 scans)
  unsigned long long* tcs;  // [units][G] selection thresholds on composite keys
  uint32_t* poff;    // [units][G][2 nA] idx_out offset of each half part (idx_out only)
  float* part;       // [units][2 nA][G][D + 2] per-part (acc[D], m, l); tail units use half parts
  float* logits;     // [units][G][S_cap] exact logits (weights_out only) or null
  int spec;          // 1: A items publish boundary-bin candidates (selection skips the key scan)
  int ccap;          // candidate capacity per (unit, head)
  unsigned long long* cbuf;  // [units][G][ccap] candidate composites
  uint32_t* ccnt;    // [units][G] candidate counts (zero between launches)
  uint32_t* cwin;    // [units][G][nA] each chunk's bin window lo | hi << 16
  long long* trace;  // optional [n_tickets][4] {start, end, sm | kind << 16 | block << 32, tail start}
  int debug;
  int halves;
  // lists mode (single-chunk units): the A item keeps the unit's keys on chip ([G][La] words at
  // off_kchip), selects there and publishes the ordered entries (head mask << 24 | row) of every
  // selected row to sel[u] plus each half part's entry offset to loff[u][0 .. 2 nA]; B items copy
  // their slice instead of re-deriving it from the keys
  int lists;
  int off_kchip;
  int off_cand, cand_bytes;  // warp-specialised A launch: the select group's candidate buffers
  long long spin_ns;  // B items trap after waiting this long for their unit's selection (0: never)
  uint32_t* sel;     // [units][sel_stride] (aliases keys: entries are written in place over a unit's keys)
  int sel_stride;    // words between units' entry lists: kstride x key arrays per unit in the A launch
  // group-shared selection (LOKI_SELECT_TOPK_SHARED): the query heads of a KV group share one selection,
  // made on the group's summed query (sum_g q_g[:d] . K[j, :d]); the A launch runs it as a G = 1 problem
  // (its params carry G = 1, shared = the group size), the B launch attends every head (full masks)
  int shared;
  int umma;          // per-head GQA A launch: phase 1 on tcgen05 (128-row tiles, TMEM accumulators)
  int ust;           // ... its tile stages
  int off_qt;        // ... its query-term operand tile in shared memory
  int dense;         // 1: SELECT_ALL on the B-only launch -- every row of every part, no A launch, no flags
  float* ml;         // [units][G][2] merged (max, sum) per head (lists mode with weights_out only)
  uint32_t* loff;    // [units][2 nA + 1]        // B parts in halves: 2 every unit, 1 tail units only (grouping then depends on #units), 0 none
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

// The cache as one 2-D [rows, D] row space for TMA row gathers: row of (b, h, s)
// = b * sb + h * sh + s.  ok == false when the strides are not whole rows or the
// space needs more than 2^31 rows (then the LDG kernels serve the call).
struct RowSpace {
  long long sb = 0, sh = 0, total = 0;
  bool ok = false;
};
RowSpace row_space(const loki_kv_geom& g);

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
cudaError_t launch_project_rows(const void* x, int x_dtype, const float* P, void* out, int out_dtype, int B, int H,
                                int S, int D, int G, const int64_t* xs, const int64_t* os, cudaStream_t st);

// persistent pipelined decode (loki_pipe.cu)
size_t pipe_layout(int G_T, PipeParams* p);
bool pipe_supported(int dtype, int D, int G_T);
// lead boxes {dbox, r1} (64 B promotion), K row gathers of columns [kcol0, D), V row gathers
bool encode_pipe_tma(const void* K, const void* V, const loki_kv_geom& g, int dbox, int r1, int kcol0, bool mma,
                     int lead_swz, TmaDesc* maps);
// big: 2x larger chunks (compiled for G == 1 only; long sequences amortise per-item latency)
// mode 0: one launch; 1 / 2: the A-only / B-only halves of a split layer (MHA bf16)
cudaError_t launch_pipe(const PipeParams& p, int dtype, int G_T, int grid, size_t smem, const TmaDesc* maps,
                        cudaStream_t st, bool big, int mode = 0);
int pipe_ctas_per_sm(int dtype, int D, int G_T, size_t smem, bool big, int mode = 0);
// warp-specialised A launch of split MHA bf16 layers (lead rows of 64 / 128 B), one unit per item: sets the
// layout offsets in *p (ring, bars, double-buffered histograms, on-chip keys or the key stream's buffers,
// candidates) and returns its bytes.  onchip: keys on chip + lists mode; else keys in the workspace
size_t pipe_select_layout(PipeParams* p, bool onchip, int G_T = 1);
cudaError_t launch_pipe_weights(const PipeParams& p, cudaStream_t st);
int pipe_select_ctas_per_sm(int dtype, int lead_rb, bool onchip, size_t smem, int G_T = 1);
cudaError_t launch_pipe_select(const PipeParams& p, int dtype, bool onchip, int grid, size_t smem,
                               const TmaDesc* maps, cudaStream_t st, int G_T = 1);
int pipe_warps();
// 128-row blocks per warp in a B part (Lc = blocks * 128 * warps), shared by kernel and host
__host__ __device__ constexpr int pipe_blocks_per_warp(int G_T, bool big) {
  return G_T == 1 ? (big ? 8 : 4) : (G_T == 8 ? 1 : 2);
}

}  // namespace loki
