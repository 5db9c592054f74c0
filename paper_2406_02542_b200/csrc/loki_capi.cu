// C ABI entry points (include/loki_b200.h): host-side validation with the
// reference's error classes and messages, launch planning, dispatch.
#include <math.h>
#include <stdlib.h>
#include <stdarg.h>
#include <stdio.h>

#include <string>

#include "loki_common.cuh"
#include "loki_internal.h"
#include <cstring>

namespace loki {
long long* g_phase_trace = nullptr;
int g_phase_trace_ctas = 0;
}  // namespace loki

namespace {

thread_local std::string g_last_error;

loki_status fail(loki_status code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

loki_status cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return LOKI_OK;
  (void)cudaGetLastError();  // a rejected launch must not resurface as the next call's error
  return fail(LOKI_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

int sm_count() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) return 148;
  return n;
}

bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

constexpr int kThreads = 256;
constexpr size_t kSmemPreferred = 100 * 1024;
constexpr size_t kSmemMax = 200 * 1024;
// the warp-specialised A launch: one CTA per SM with (almost) the whole SM's shared memory -- 227 KB opt-in
// less the kernel's static shared memory (PipeShared and friends)
constexpr size_t kSmemSelMax = 224 * 1024;

int k_for(const loki_decode_args* a, int S) {
  if (a->select_mode == LOKI_SELECT_ALL) return S;
  if (a->k_fixed > 0) return a->k_fixed < S ? a->k_fixed : S;
  return loki::resolve_fraction(a->k_f, S);
}

loki_status validate(const loki_decode_args* a) {
  if (a == nullptr) return fail(LOKI_ERR_SHAPE, "null argument block");
  const loki_kv_geom& g = a->g;
  if (g.B < 1 || g.Hq < 1 || g.Hkv < 1 || g.D < 1 || g.S_cap < 1)
    return fail(LOKI_ERR_SHAPE, "invalid geometry B=%d Hq=%d Hkv=%d D=%d S_cap=%d", g.B, g.Hq, g.Hkv, g.D, g.S_cap);
  if (g.Hq % g.Hkv != 0)
    return fail(LOKI_ERR_SHAPE, "query heads %d are not a multiple of kv heads %d", g.Hq, g.Hkv);
  if (g.Hq / g.Hkv > 8) return fail(LOKI_ERR_UNSUPPORTED, "group size %d > 8", g.Hq / g.Hkv);
  if (g.D > 256) return fail(LOKI_ERR_UNSUPPORTED, "head dim %d > 256", g.D);
  if (g.dtype != LOKI_DTYPE_F32 && g.dtype != LOKI_DTYPE_BF16)
    return fail(LOKI_ERR_UNSUPPORTED, "cache dtype code %d", g.dtype);
  if (a->S_max < 1) return fail(LOKI_ERR_SHAPE, "attention needs at least one cached token");
  if (a->S_max > g.S_cap) return fail(LOKI_ERR_SHAPE, "S_max %d exceeds cache capacity %d", a->S_max, g.S_cap);
  if (a->lens == nullptr) return fail(LOKI_ERR_SHAPE, "lens is required");
  if (a->select_mode < 0 || a->select_mode > 4) return fail(LOKI_ERR_DOMAIN, "select_mode %d", a->select_mode);
  const bool ranks = a->select_mode == LOKI_SELECT_TOPK || a->select_mode == LOKI_SELECT_TOPK_SHARED;
  if (a->select_mode == LOKI_SELECT_TOPK_SHARED && a->ext_scores != nullptr)
    return fail(LOKI_ERR_UNSUPPORTED, "group-shared selection ranks its own approximate scores");
  const bool computes_scores = a->ext_scores == nullptr && (ranks || a->select_mode == LOKI_SELECT_NONE);
  const bool attends = a->out != nullptr;
  if (computes_scores || attends) {
    if (a->q_hat == nullptr || a->K == nullptr) return fail(LOKI_ERR_SHAPE, "q_hat and K are required");
    if (g.stride_s < g.D || g.stride_h < 0 || g.stride_b < 0)
      return fail(LOKI_ERR_SHAPE, "cache strides (%lld, %lld, %lld) do not hold rows of %d",
                  (long long)g.stride_b, (long long)g.stride_h, (long long)g.stride_s, g.D);
  }
  if (attends && a->V == nullptr) return fail(LOKI_ERR_SHAPE, "V is required");
  if (computes_scores && (a->d < 1 || a->d > g.D)) return fail(LOKI_ERR_BUDGET, "d=%d outside [1, %d]", a->d, g.D);
  if (a->select_mode != LOKI_SELECT_ALL && a->select_mode != LOKI_SELECT_NONE) {
    if (a->k_fixed > a->S_max) return fail(LOKI_ERR_BUDGET, "k=%d outside [1, %d]", a->k_fixed, a->S_max);
    if (a->k_fixed <= 0 && !(a->k_f > 0.0 && a->k_f <= 1.0))
      return fail(LOKI_ERR_DOMAIN, "budget fraction must lie in (0, 1], got %g", a->k_f);
  }
  if (a->select_mode == LOKI_SELECT_NONE && a->approx_out == nullptr && !attends)
    return fail(LOKI_ERR_SHAPE, "scores-only call without approx_out");
  if (a->select_mode == LOKI_SELECT_NONE && attends)
    return fail(LOKI_ERR_SHAPE, "scores-only call cannot attend");
  if (a->select_mode == LOKI_SELECT_INDICES && a->ext_idx == nullptr)
    return fail(LOKI_ERR_SHAPE, "external index lists are required");
  if (ranks && !attends && a->idx_out == nullptr && a->approx_out == nullptr)
    return fail(LOKI_ERR_SHAPE, "ranking-only call without outputs");
  const bool needs_stride = a->ext_idx || a->idx_out || a->weights_out;
  if (needs_stride) {
    const int kmax = k_for(a, a->S_max);
    if (a->idx_stride < kmax)
      return fail(LOKI_ERR_SHAPE, "idx_stride %lld < k %d", (long long)a->idx_stride, kmax);
  }
  return LOKI_OK;
}

// Tuning knobs (LOKI_PIPE_*, LOKI_TMA_*, LOKI_DEBUG, ...) are honoured only with LOKI_TUNING=1, so a
// deployment's launch plan cannot change silently with its environment.
bool tuning_enabled() {
  const char* v = getenv("LOKI_TUNING");
  return v != nullptr && *v != '\0' && *v != '0';
}

int env_int(const char* name, int dflt) {
  if (!tuning_enabled()) return dflt;
  const char* v = getenv(name);
  if (v == nullptr || *v == '\0') return dflt;
  return atoi(v);
}

int stage_bytes_cfg() { return env_int("LOKI_TMA_STAGE_KB", 4) * 1024; }
size_t smem_tma_target() { return (size_t)env_int("LOKI_SMEM_KB", 112) * 1024; }  // 112 KB: two CTAs per SM

struct TmaGeom {
  int vec, dbox, r1, r3;
};

// TMA plan pieces for (dtype, D, d, G_T); false when the layout is outside
// what the TMA kernel handles.
bool tma_geom(const loki_decode_args* a, int G_T, TmaGeom* t, int stage_bytes = 0) {
  const loki_kv_geom& g = a->g;
  const int e = g.dtype == LOKI_DTYPE_BF16 ? 2 : 4;
  const int vec = g.dtype == LOKI_DTYPE_BF16 ? (G_T == 8 ? 4 : 8) : 4;
  if ((g.D * e) % 16 != 0 || g.D / vec > 32 || g.D % vec != 0) return false;
  const int per16 = 16 / e;
  const int d = a->d < 1 ? 1 : a->d;
  const int dbox = loki::ceil_div(d, per16) * per16;
  if (dbox > g.D && a->select_mode != LOKI_SELECT_ALL) return false;
  // a stage is digested by one warp: phase 1 in passes of 4 x rpw1 rows,
  // phase 3 in passes of 2 x rpw3 rows; gather4 needs multiples of 4 rows
  const int rpw1 = 32 / loki::next_pow2(dbox / vec);
  const int kStageBytes = stage_bytes > 0 ? stage_bytes : stage_bytes_cfg();
  int r1 = kStageBytes / (dbox * e);
  if (r1 > 256) r1 = 256;
  r1 = r1 / (4 * rpw1) * (4 * rpw1);
  const int rpw3 = 32 / loki::next_pow2(g.D / vec);
  int unit3 = 2 * rpw3;
  while (unit3 % 4) unit3 *= 2;
  int r3 = kStageBytes / (2 * g.D * e);
  if (r3 > 32) r3 = 32;  // the producer warp resolves one gathered row per lane
  r3 = r3 / unit3 * unit3;
  if (r1 < 4 * rpw1 || r3 < unit3) return false;
  t->vec = vec;
  t->dbox = dbox;
  t->r1 = r1;
  t->r3 = r3;
  return true;
}

loki_status make_plan(const loki_decode_args* a, loki::Plan* plan, loki::FusedParams* p, TmaGeom* tg) {
  const loki_kv_geom& g = a->g;
  const int G = g.Hq / g.Hkv;
  const int units = g.B * g.Hkv;
  plan->G_T = loki::next_pow2(G);
  plan->dtype = g.dtype;
  const int vec = (g.dtype == LOKI_DTYPE_BF16) ? (plan->G_T == 8 ? 4 : 8) : 4;
  const size_t ebytes = g.dtype == LOKI_DTYPE_BF16 ? 2 : 4;
  const size_t vbytes = (size_t)vec * ebytes;
  plan->fast = (g.D % vec == 0) && (g.D / vec <= 32) && (g.stride_s % vec == 0) && (g.stride_h % vec == 0) &&
               (g.stride_b % vec == 0) && (a->K == nullptr || aligned(a->K, vbytes)) &&
               (a->V == nullptr || aligned(a->V, vbytes));

  // TMA path: cache reachable as one 2-D [rows, D] row space (any whole-row head / batch strides), 16 B aligned
  const loki::RowSpace rs = loki::row_space(g);
  plan->tma = env_int("LOKI_TMA", 1) != 0 && a->K != nullptr && a->V != nullptr && a->ext_scores == nullptr &&
              rs.ok && aligned(a->K, 16) && aligned(a->V, 16) && (g.stride_s * ebytes) % 16 == 0 &&
              loki::tma_supported(g.dtype, g.D, plan->G_T) && tma_geom(a, plan->G_T, tg);
  const int kStageBytes = stage_bytes_cfg();
  const int NTt = loki::kTmaThreads;
  const int align = plan->tma ? tg->r1 : 1;
  const int nst_env = env_int("LOKI_TMA_STAGES", 0);
  auto Lfor = [&](int c) { return loki::ceil_div(loki::ceil_div(a->S_max, c), align) * align; };
  // TMA: as many ring stages as fit next to the slice state in the per-CTA budget
  auto stages_for = [&](int L, bool keys_smem) {
    if (nst_env > 0) return nst_env;
    loki::FusedParams tmp{};
    const size_t base = loki::fused_tma_layout(plan->G_T, NTt, g.D, L, keys_smem, 0, kStageBytes, &tmp);
    const long long per = (long long)kStageBytes * loki::kTmaWarps;  // one stage in every warp's ring
    const long long n = base >= smem_tma_target() ? 0 : (long long)((smem_tma_target() - base) / per);
    return (int)(n > 8 ? 8 : n);
  };
  auto smem_for = [&](int L, bool keys_smem) {
    loki::FusedParams tmp{};
    return plan->tma ? loki::fused_tma_layout(plan->G_T, NTt, g.D, L, keys_smem, stages_for(L, keys_smem) < 2 ? 2 : stages_for(L, keys_smem), kStageBytes, &tmp)
                     : loki::fused_layout(plan->G_T, kThreads, g.D, L, keys_smem, &tmp);
  };
  const size_t preferred = plan->tma ? smem_tma_target() : kSmemPreferred;
  const int target = 4 * sm_count();
  int C = 0;
  bool keys_smem = true;
  const int cov = a->cluster_override > 0 ? a->cluster_override : env_int("LOKI_CLUSTER", 0);
  if (cov > 0) {
    C = cov;
    if (C != 1 && C != 2 && C != 4 && C != 8 && C != 16)
      return fail(LOKI_ERR_DOMAIN, "cluster_override %d not in {1,2,4,8,16}", C);
    keys_smem = smem_for(Lfor(C), true) <= kSmemMax;
  } else {
    for (int c = 1; c <= 16; c *= 2) {
      const int L = Lfor(c);
      if (L > 65535) continue;
      if (smem_for(L, true) > preferred) continue;
      if (units * c >= target || L <= 256 || c == 16) {
        C = c;
        break;
      }
    }
    if (C == 0) {
      C = 16;
      keys_smem = smem_for(Lfor(16), true) <= kSmemMax;
    }
  }
  int nst = plan->tma ? stages_for(Lfor(C), keys_smem) : 0;
  if (plan->tma && nst < 2) nst = 2;
  const int L = Lfor(C);
  if (L > 65535) return fail(LOKI_ERR_UNSUPPORTED, "sequence %d too long for %d CTAs per unit", a->S_max, C);
  plan->C = C;
  plan->Lmax = L < 1 ? 1 : L;
  plan->keys_in_smem = keys_smem;
  plan->smem = plan->tma ? loki::fused_tma_layout(plan->G_T, NTt, g.D, plan->Lmax, keys_smem, nst, kStageBytes, p)
                         : loki::fused_layout(plan->G_T, kThreads, g.D, plan->Lmax, keys_smem, p);
  if (plan->smem > kSmemMax) return fail(LOKI_ERR_UNSUPPORTED, "shared memory plan %zu bytes", plan->smem);
  plan->workspace = keys_smem ? 0 : (size_t)units * C * plan->G_T * plan->Lmax * 4;
  p->slice_align = align;
  if (plan->tma) {
    p->r1 = tg->r1;
    p->dbox = tg->dbox;
    p->r3 = tg->r3;
    p->row_sb = rs.sb;
    p->row_sh = rs.sh;
  }
  return LOKI_OK;
}


// ---------------------------------------------------------------- pipelined plan
struct PipePlan {
  loki::PipeParams p{};
  TmaGeom tg{};
  int G_T = 1;
  int G_Ta = 1;  // group size the A launch is instantiated for (1 for group-shared selection)
  bool mode3 = false;  // the opt-in on-chip lists A launch (LOKI_LISTS)
  loki::PipeParams blay{};  // group-shared: the B-only launch's shared-memory layout (no histogram)
  size_t smem_b = 0;
  bool big = false;
  bool split = false;  // A-only launch + B-only launch (MHA bf16)
  bool ws_select = false;  // the A launch is the warp-specialised pipe_select_kernel (layout in sel_layout)
  bool ws_onchip = false;  // ... with the keys on chip (lists mode)
  int ws_groups = 1;       // ... its key arrays per unit (per-head GQA: the group size)
  loki::PipeParams sel_layout{};
  int grid = 0, grid1 = 0, grid2 = 0;
  size_t smem1 = 0;
  size_t smem = 0;
  size_t ws = 0;
  size_t off_hist = 0, off_keys = 0, off_tcs = 0, off_poff = 0, off_part = 0, off_spec = 0, off_logits = 0;
  size_t off_loff = 0, off_ml = 0;
};

// The persistent pipelined kernel (loki_pipe.cu) serves the attending TOPK
// path whenever the cache is TMA-addressable; false -> cluster kernels.
bool pipe_eligible(const loki_decode_args* a) {
  const loki_kv_geom& g = a->g;
  const int G_T = loki::next_pow2(g.Hq / g.Hkv);
  const size_t e = g.dtype == LOKI_DTYPE_BF16 ? 2 : 4;
  const loki::RowSpace rs = loki::row_space(g);
  // dense decode (SELECT_ALL) runs as a B-only launch over every row when no diagnostics are asked for
  const bool dense = a->select_mode == LOKI_SELECT_ALL && g.dtype == LOKI_DTYPE_BF16 && a->idx_out == nullptr &&
                     a->approx_out == nullptr && a->weights_out == nullptr && env_int("LOKI_PIPE_DENSE", 1) != 0;
  return env_int("LOKI_PIPE", 1) != 0 &&
         (a->select_mode == LOKI_SELECT_TOPK || a->select_mode == LOKI_SELECT_TOPK_SHARED || dense) &&
         a->ext_scores == nullptr &&
         a->out != nullptr && a->K != nullptr && a->V != nullptr && rs.ok && aligned(a->K, 16) &&
         aligned(a->V, 16) && (g.stride_s * e) % 16 == 0 &&
         a->S_max < (1 << 24) && loki::pipe_supported(g.dtype, g.D, G_T) && a->cluster_override == 0;
}

loki_status make_pipe_plan(const loki_decode_args* a, PipePlan* pl);

// Group-shared selection with one query head per KV head is plain per-head selection; with groups it
// exists only on the pipe path (no cluster-kernel fallback).
const loki_decode_args* canonical_mode(const loki_decode_args* a, loki_decode_args* tmp) {
  if (a->select_mode != LOKI_SELECT_TOPK_SHARED || a->g.Hq != a->g.Hkv) return a;
  *tmp = *a;
  tmp->select_mode = LOKI_SELECT_TOPK;
  return tmp;
}

// Small batches (B <= 4, MHA, bf16, up to 32K rows): one thread-block cluster of C CTAs per unit (phase 1 in
// lockstep, DSMEM radix select, gather, DSMEM merge) beats the persistent pipe, whose per-unit selection is
// serial -- r02 sweep (tools/one_layer.py): B = 1, S = 4K 35.8 -> 24.1 us (C = 8); B = 1, S = 32K 148 -> 70;
// B = 2, S = 8K 108 -> 42 (C = 4); B = 4, S = 8K 131 -> 79 (C = 4); B = 8 breaks even.  C depends on B
// only, so KV-head shards of a layer run the same per-unit plan (bit-identical).
const loki_decode_args* small_batch_plan(const loki_decode_args* a, loki_decode_args* tmp) {
  const loki_kv_geom& g = a->g;
  if (a->select_mode != LOKI_SELECT_TOPK || a->cluster_override != 0 || g.Hq != g.Hkv ||
      g.dtype != LOKI_DTYPE_BF16 || g.B > 4 || a->S_max > 32768 || a->ext_scores != nullptr ||
      env_int("LOKI_SMALL_CLUSTER", 1) == 0)
    return a;
  *tmp = *a;
  tmp->cluster_override = g.B == 1 ? 8 : 4;
  return tmp;
}

loki_status shared_unsupported(const loki_decode_args* a) {
  if (!pipe_eligible(a))
    return fail(LOKI_ERR_UNSUPPORTED, "group-shared selection needs a TMA-addressable cache (16 B aligned rows)");
  PipePlan pl;
  const loki_status s = make_pipe_plan(a, &pl);
  return s != LOKI_OK ? s : fail(LOKI_ERR_UNSUPPORTED, "group-shared selection: no pipe plan");
}

loki_status make_pipe_plan(const loki_decode_args* a_in, PipePlan* pl) {
  // dense decode: B-only launch over every row; the (unused) lead-column geometry is planned for d = 32
  const bool dense = a_in->select_mode == LOKI_SELECT_ALL;
  loki_decode_args ad = *a_in;
  if (dense) ad.d = a_in->g.D < 32 ? a_in->g.D : 32;
  const loki_decode_args* a = &ad;
  const loki_kv_geom& g = a->g;
  const int G = g.Hq / g.Hkv;
  const int G_T = loki::next_pow2(G);
  const int units = g.B * g.Hkv;
  const int e = g.dtype == LOKI_DTYPE_BF16 ? 2 : 4;
  pl->G_T = G_T;
  const bool shared = a->select_mode == LOKI_SELECT_TOPK_SHARED;  // (G > 1: canonical_mode maps G == 1 to TOPK)
  if (shared && g.dtype != LOKI_DTYPE_BF16) return fail(LOKI_ERR_UNSUPPORTED, "group-shared selection needs bf16 caches");
  // tensor-core phase 3 (bf16): 16-row stages of K and V (64 * D bytes)
  const bool mma = g.dtype == LOKI_DTYPE_BF16;  // bf16 caches: tensor-core phase 3 (compiled in, not optional)
  const int stage = mma ? 32 * g.D : env_int("LOKI_PIPE_STAGE_KB", 4) * 1024;
  if (!tma_geom(a, G_T, &pl->tg, stage)) return fail(LOKI_ERR_UNSUPPORTED, "pipe: TMA geometry");
  loki::PipeParams& p = pl->p;
  p.mma = mma ? 1 : 0;
  p.nst = env_int("LOKI_PIPE_STAGES", 2);
  p.stage_bytes = stage;
  p.r1 = pl->tg.r1;
  p.dbox = pl->tg.dbox;
  p.r3 = pl->tg.r3;
  p.hbits = G_T <= 2 ? 11 : (G_T == 4 ? 10 : 9);
  const int d = a->d < 1 ? 1 : a->d;
  const int vec = pl->tg.vec;
  // split-K: phase 3 skips the lead columns and adds the phase-1 partial score.  Tensor-core path: compiled
  // for d = 32 of D = 128 (128 B + 64 B K pieces); the partial scores take Lc words of shared memory per
  // head, so not with the 8192-row chunks
  // (r01: no gain on the tensor-core path at C2, 210.5 vs 211.3 us, and 16 KB more smem: opt-in there)
  p.shared = shared ? G : 0;
  p.dense = dense ? 1 : 0;
  p.split_k = !shared && env_int("LOKI_SPLITK", mma ? 0 : 1) != 0 && d < g.D &&
              (mma ? (d == 32 && g.D == 128 && G_T <= 4) : (d % vec == 0 && ((g.D - d) * e) % 32 == 0));
  if (mma) p.r3 = 8;
  // one lane per lead row when the row is a TMA swizzle span (64 / 128 B) and r1 covers whole lanes
  const int lead_rb = p.dbox * e;
  // G == 1: one lane per lead row (r1 % 64); G >= 2 (bf16): tensor-core scores on 16-row blocks
  const bool lead_ok = (lead_rb == 64 || lead_rb == 128) && env_int("LOKI_LEAD_LPR", 1) != 0 &&
                       (G_T == 1 ? p.r1 % (lead_rb == 64 ? 64 : 32) == 0 : (g.dtype == LOKI_DTYPE_BF16 && p.r1 % 16 == 0));
  p.lead_swz = lead_ok ? lead_rb : 0;
  if (g.dtype == LOKI_DTYPE_BF16 && G_T >= 2 && p.lead_swz == 0)  // bf16 groups need the tensor-core lead path
    return fail(LOKI_ERR_UNSUPPORTED, "pipe: bf16 query groups need 64 / 128 B lead rows (d = %d)", d);
  // chunk = part: kNB 128-row blocks per warp in the B-item row scan (loki_pipe.cu)
  // MHA at long sequences: 2x larger chunks (fewer per-item latency bubbles; r01: TGT 683 -> 658 us,
  // C2 213 -> 219 us, so only from 16K rows on)
  // (r02, split layers with entry lists: from 8K rows too -- C2 step 177.2 -> 172.5 us/layer)
  pl->big = G_T == 1 && env_int("LOKI_PIPE_BIG", a->S_max >= 8192 ? 1 : 0) != 0;
  if (pl->big && mma) p.split_k = 0;
  const int kNB = loki::pipe_blocks_per_warp(G_T, pl->big);
  int Lc = kNB * 128 * loki::pipe_warps();
  // group-shared selection publishes entry lists (unless diagnostic weights need the key path): B parts
  // then copy their slice instead of re-deriving it from the keys, so their size is free of the key-scan
  // register arrays -- MHA-sized parts (a k-fraction of the rows is selected, whatever the group size)
  const bool shared_lists = shared && env_int("LOKI_GLOBAL_LISTS", 1) != 0;
  // per-head groups in split layers publish union lists too (head masks per entry)
  const bool head_lists = !shared && !dense && G_T > 1 && g.dtype == LOKI_DTYPE_BF16 && a->S_max >= 8192 &&
                          env_int("LOKI_PIPE_SPLIT", 1) != 0 && env_int("LOKI_HEAD_LISTS", 1) != 0;
  const bool lists_plan = shared_lists || head_lists;
  if (lists_plan) Lc = env_int("LOKI_LISTS_LC", a->S_max >= 16384 ? 8192 : 4096);
  if (dense) Lc = env_int("LOKI_DENSE_LC", a->S_max >= 8192 ? 8192 : 4096);
  if (Lc % p.r1 != 0) return fail(LOKI_ERR_UNSUPPORTED, "pipe: chunk %d vs box rows %d", Lc, p.r1);
  p.Lc = Lc;
  p.nA = loki::ceil_div(a->S_max, Lc);
  // A chunks of >= 4096 rows: small GQA parts would make phase-1 items overhead-bound
  p.La = env_int("LOKI_PIPE_LA", Lc >= 4096 ? Lc : 4096);
  if (p.La < Lc && env_int("LOKI_PIPE_LA", 0) == 0) p.La = Lc;
  if (p.La % p.r1 != 0) return fail(LOKI_ERR_UNSUPPORTED, "pipe: chunk %d vs box rows %d", p.La, p.r1);
  p.nAa = loki::ceil_div(a->S_max, p.La);
  p.units = units;
  // speculative boundary-bin candidates (ranking-free path only: idx_out needs per-part counts)
  p.spec = env_int("LOKI_SPEC", 0) != 0 && G_T <= 4 && a->idx_out == nullptr && p.La == p.Lc;  // opt-in (net loss)
  p.ccap = a->S_max / 4 > 2048 ? a->S_max / 4 : 2048;
  pl->smem = loki::pipe_layout(G_T, &p);
  if (shared || dense || head_lists) {  // the B-only launch keeps no histogram: its own, smaller layout
    pl->blay = p;
    pl->blay.hbits = 0;
    pl->smem_b = loki::pipe_layout(G_T, &pl->blay);
  }
  const size_t ring = (size_t)loki::pipe_warps() * p.nst * p.stage_bytes;
  if ((size_t)loki::pipe_warps() * G_T * (g.D + 2) * 4 > ring || p.cand_cap < 256)
    return fail(LOKI_ERR_UNSUPPORTED, "pipe: ring of %zu bytes too small", ring);
  if (pl->smem > kSmemMax) return fail(LOKI_ERR_UNSUPPORTED, "pipe: shared memory plan %zu bytes", pl->smem);
  const int occ = loki::pipe_ctas_per_sm(g.dtype, g.D, G_T, pl->smem, pl->big);
  if (occ < 1) return fail(LOKI_ERR_UNSUPPORTED, "pipe: kernel does not fit on an SM (%zu B smem)", pl->smem);
  // r01: split layers beat the single launch on MHA bf16 (C2 212 -> 205 us, TGT 626 -> 603 us)
  // (short sequences keep one launch: S = 4K 125 vs 137 us split)
  // (r01: GQA too, C3 866 -> 742, C4 989 -> 875, C5s 4445 -> 3468 us)
  pl->split = (shared || dense || env_int("LOKI_PIPE_SPLIT", a->S_max >= 8192 ? 1 : 0) != 0) &&
              g.dtype == LOKI_DTYPE_BF16 && !p.spec;
  if (dense && !pl->split) return fail(LOKI_ERR_UNSUPPORTED, "pipe: dense decode needs the B-only launch");
  pl->G_Ta = shared ? 1 : G_T;  // group-shared: the A launch ranks once per unit (a G = 1 problem)
  if (pl->split) {  // the A-only launch needs no B-item entry region
    pl->smem1 = (size_t)p.off_ents + 1024;
    const int occ1 = loki::pipe_ctas_per_sm(g.dtype, g.D, pl->G_Ta, pl->smem1, pl->big, 1);
    const int occ2 = loki::pipe_ctas_per_sm(g.dtype, g.D, G_T, pl->smem_b > 0 ? pl->smem_b : pl->smem, pl->big, 2);
    if (occ1 < 1 || occ2 < 1) pl->split = false;
    // A chunks of >= 8192 rows (r01: C2 197.9 -> 193.0 us); the A launch has no lag to feed.  Groups of 8:
    // >= 32768 rows (fewer arrivals into the serial 8-head selection; r01 C5s 3398 -> 3232 us,
    // tools/c5s_sweep.sh).  Groups of 4: >= 16384 rows once the units alone fill an A wave (C4 877 -> 863 us,
    // tools/la_big.sh; C3, 256 units, loses 1.2 % with them and keeps 8192)
    const int GA = pl->G_Ta;
    const int la_min = GA == 8 ? 32768 : (GA == 4 && units >= sm_count() * occ1 ? 16384 : 8192);
    if (env_int("LOKI_PIPE_LA", 0) == 0 && p.La < la_min) {
      p.La = la_min;
      p.nAa = loki::ceil_div(a->S_max, p.La);
    }
    const int a_ctas = env_int("LOKI_PIPE_A_CTAS", occ1);
    pl->grid1 = sm_count() * (a_ctas < occ1 ? (a_ctas < 1 ? 1 : a_ctas) : occ1);
    pl->grid2 = sm_count() * occ2;
  }
  // B parts as halves (2: every unit; 1: the tail units, which shortens the drain; 0: none).  r01 sweep
  // (tools/halves_check.sh, one launch): every-unit halves help groups and small batches (GQA S = 4K
  // 186 -> 166 us, B = 1 48 -> 40, B = 4 73 -> 70) but not B = 16 MHA (137 -> 136, S = 2K 95 -> 101);
  // split layers lose from either (TGT 597 / 593 / 641 us).  The default depends on G, B and S only, so a
  // KV-head shard groups its partial states exactly like one launch (bit-identical).  Tail
  // halves (1) are faster still at one launch (S = 4K 137 -> 125 us, B = 4 73 -> 57) but the tail is a
  // set of units, so shards then agree to rounding only: opt-in
  p.halves = env_int("LOKI_PIPE_HALVES", pl->split ? 0 : ((G >= 2 || g.B <= 4) ? 2 : 0));
  // few units: smaller A chunks, so phase 1 spreads over the grid -- at least 128 A items for one launch,
  // one A-launch wave for split layers (r01, tools/la_small.sh: B = 1, S = 4K 39.8 -> 35.4 us; B = 2,
  // S = 8K 95.7 -> 81.4 us; B = 4, S = 4K keeps 4096-row chunks: 66.8 vs 71.6 us at 1024; GQA B = 1, S = 32K
  // 209 -> 176 us).  MHA: at most 8 chunks per unit (B = 1, S = 32K: 16 chunks 144 us vs 138 at 4)
  if (env_int("LOKI_PIPE_LA", 0) == 0) {
    const long long target = pl->split ? (long long)pl->grid1 : 128;
    while ((long long)units * p.nAa < target && p.La >= 2048 && (p.La / 2) % p.r1 == 0 &&
           (pl->G_Ta > 1 || p.nAa < 8)) {
      p.La /= 2;
      p.nAa = loki::ceil_div(a->S_max, p.La);
    }
  }
  // lists mode: single-chunk units select on chip and publish ordered entry lists (no global keys, no
  // histogram merge, no L2 key re-stream; B items copy their slice).  Needs the unit's keys on chip next
  // to the ring: the A-only launch of a split layer carries them in place of the B-entry region
  p.lists = 0;
  // group-shared selection always runs here: its selection is a G = 1 problem on the summed query (one lane
  // per lead row, so the G = 1 box rule applies), whatever the number of units
  const bool g1_lead = (p.lead_swz == 64 || p.lead_swz == 128) && p.r1 % (p.lead_swz == 64 ? 64 : 32) == 0;
  // per-head groups (bf16, tensor-core lead path): the same launch with G key arrays in the workspace,
  // the select group taking the heads in turn; B items re-derive the union from the keys
  const bool gqa_ws = G_T > 1 && !shared && g.dtype == LOKI_DTYPE_BF16 && (p.lead_swz == 64 || p.lead_swz == 128) &&
                      env_int("LOKI_SELECT_WS_GQA", 1) != 0;
  if (pl->split && !dense && ((G_T == 1 || shared) ? g1_lead : gqa_ws) && !p.spec && !p.split_k &&
      env_int("LOKI_SELECT_WS", 1) != 0 && units >= env_int("LOKI_WS_MIN_UNITS", G_T > 1 ? 96 : sm_count())) {
    // (query groups from 96 units: C5s' 128 units, shared 898 -> 837 us, per-head 2683 -> 2511 us, even with
    // 20 SMs idle in the A launch -- the chunked launch's serial per-unit selection costs more)
    // The warp-specialised A launch (one 16-warp CTA per SM, one whole unit per item): a stream group
    // streams unit i's lead columns while a select group selects unit i - 1, so the selection never
    // idles the loads.  Units of <= 8192 rows keep their keys on chip and publish ordered entry lists
    // (lists mode); longer ones keep the keys in the workspace and publish the threshold.
    loki::PipeParams ps = p;
    ps.La = loki::ceil_div(a->S_max, p.r1) * p.r1;
    ps.nAa = 1;
    // Entry lists need power-of-two half parts; diagnostic weights need the keys left in the workspace
    // (the merge re-derives each head's selection from them), so such calls keep the key path
    const bool pow2 = ((p.Lc / 2) & (p.Lc / 2 - 1)) == 0;
    const int GS = gqa_ws ? G_T : 1;  // key arrays / histograms per unit in the A launch
    // on-chip keys up to 8192 rows; group-shared layers up to 16384 (with two stream stages: C4 shared
    // 358.6 -> 340.5 us; MHA at 16K loses with two stages, 307.6 -> 368.0 us at B = 16)
    const bool onchip = GS == 1 && ps.La <= env_int("LOKI_ONCHIP_ROWS", shared ? 16384 : 8192) && pow2;
    // ring stages per stream warp: 3 where they fit (r02: 2 -> 3 TGT 591 -> 566 us, C2 177 -> 174 us; 4 measured
    // no faster at TGT, 567 vs 566 us), else 2
    size_t sw = 0;
    int ow = 0;
    for (int nst = env_int("LOKI_SELECT_STAGES", 3); nst >= 2 && ow < 1; --nst) {
      ps.nst = nst;
      sw = loki::pipe_select_layout(&ps, onchip, GS);
      ow = sw <= kSmemSelMax ? loki::pipe_select_ctas_per_sm(g.dtype, p.lead_swz, onchip, sw, GS) : 0;
    }
    if (ow >= 1) {
      p.La = ps.La;
      p.nAa = 1;
      // (units whose keys stay in the workspace publish lists too: the select group streams them back once
      // more and writes the entries in place, so B items copy slices instead of re-deriving them)
      p.lists = (onchip || (pow2 && lists_plan)) ? 1 : 0;
      // key mode (tuning): on-chip selection publishes only the threshold, B items scan the workspace keys
      if (onchip && !shared && a->idx_out == nullptr && env_int("LOKI_WS_KEYS", 0) != 0) p.lists = 0;
      pl->ws_groups = GS;
      if (GS > 1 && env_int("LOKI_UMMA", 1) != 0) {  // per-head phase 1 on tcgen05: 128-row tile stages
        const int tile = 128 * p.dbox * 2;
        int ust = (int)(((size_t)loki::pipe_warps() * ps.nst * ps.stage_bytes) / (size_t)tile);
        ust = ust > 8 ? 8 : ust;
        if (ust >= 2 && 2 * ust + 4 <= loki::pipe_warps() * ps.nst && 128 % p.r1 == 0) {
          ps.umma = 1;
          ps.ust = ust;
        }
      }
      pl->ws_select = true;
      pl->ws_onchip = onchip;
      pl->sel_layout = ps;
      pl->smem1 = sw;
      pl->grid1 = sm_count() * ow;
      // MHA: leave some SMs to the B launch from the layer's start -- B CTAs there drain the first selected
      // units while the A launch streams (r02 sweep, LOKI_SELECT_GRID after the faster on-chip selection: C2
      // 148 -> 138 A CTAs, attention 165.9 -> 162.7 us; TGT 148 -> 120, 550.4 -> 545.9 us; group-shared GQA
      // does not gain: C4 shared 343 -> 359 us at 136)
      if (G_T == 1 && !shared && ow == 1 && units >= 2 * sm_count())
        pl->grid1 = sm_count() - (a->S_max >= 32768 ? sm_count() * 3 / 16 : sm_count() / 16 + 1);
      const int g1 = env_int("LOKI_SELECT_GRID", 0);  // tuning: fewer A CTAs leave SMs to the B launch
      if (g1 > 0 && g1 < pl->grid1) pl->grid1 = g1;
    }
  }
  if (shared && !g1_lead)  // (few units: the chunked A-only launch with G = 1 items, MODE 1)
    return fail(LOKI_ERR_UNSUPPORTED, "group-shared selection: lead rows of %d B in %d-row boxes", p.lead_swz, p.r1);
  if (pl->split && !pl->ws_select && lists_plan && ((p.Lc / 2) & (p.Lc / 2 - 1)) == 0)
    p.lists = 1;  // the last A arriver's selection also emits the unit's entry list (select_unit)
  if (lists_plan && !p.lists) return fail(LOKI_ERR_UNSUPPORTED, "pipe: list plan without a split layer");
  const size_t kchip = (size_t)G_T * p.La * 4;
  if (!pl->ws_select && pl->split && G_T == 1 && !pl->big && env_int("LOKI_LISTS", 0) != 0 && p.nAa == 1 &&
      !p.spec && !p.split_k && a->idx_out == nullptr && a->weights_out == nullptr &&
      ((p.Lc / 2) & (p.Lc / 2 - 1)) == 0 && p.Lc / 2 >= 4) {
    // MODE 3 (opt-in): the A-only launch selects on chip, the keys in place of the B-entry region
    const size_t s1 = (size_t)p.off_ents + kchip + 1024;
    const int o1 = loki::pipe_ctas_per_sm(g.dtype, g.D, G_T, s1, pl->big, 3);
    if (s1 <= kSmemMax && o1 >= 1) {
      p.lists = 1;
      pl->mode3 = true;
      p.off_kchip = p.off_ents;
      pl->smem1 = s1;
      const int a_ctas = env_int("LOKI_PIPE_A_CTAS", o1);
      pl->grid1 = sm_count() * (a_ctas < o1 ? (a_ctas < 1 ? 1 : a_ctas) : o1);
    }
  }
  const int per_sm = env_int("LOKI_PIPE_CTAS_PER_SM", occ);
  pl->grid = sm_count() * (per_sm < occ ? (per_sm < 1 ? 1 : per_sm) : occ);
  // B tickets trail A tickets by enough work to cover a unit's selection, which walks the G heads in turn
  // (r01 sweeps, tools/lag_sweep.sh: MHA best at 4.0; G = 4 at 7-10; G = 8 (C5s) at 32)
  const double lagx = env_int("LOKI_PIPE_LAG_X10", G == 1 ? 40 : (G <= 4 ? 25 * G : 40 * G)) / 10.0;
  const int nb_slot = (p.halves == 2 ? 2 : 1) * p.nA;  // B tickets per unit
  const int per_slot = (p.nAa + nb_slot) > 2 * p.nA ? (p.nAa + nb_slot) : 2 * p.nA;
  int lag = (int)ceil(lagx * pl->grid / (double)(p.nAa + nb_slot));
  p.lag = lag < 1 ? 1 : (lag > units ? units : lag);
  p.n_tickets = (long long)(units + p.lag) * per_slot;
  // workspace: ctrl | hist | keys | sel | part | logits
  const int HB = 1 << p.hbits;
  size_t off = loki::align_up((size_t)(2 + 4 * (size_t)units + 2) * 4, 256);  // + split-layer B counters
  pl->off_hist = off;
  off = loki::align_up(off + (size_t)units * G * HB * 4, 256);
  pl->off_keys = off;
  p.kstride = loki::ceil_div(g.S_cap, 4) * 4;
  p.sel_stride = p.kstride * (shared ? 1 : G);  // entry lists overwrite a unit's (first) key array
  off = loki::align_up(off + (size_t)units * G * p.kstride * 4, 256);
  pl->off_tcs = off;
  off = loki::align_up(off + (size_t)units * G * 8, 256);
  pl->off_poff = off;
  if (a->idx_out != nullptr) off = loki::align_up(off + (size_t)units * G * 2 * p.nA * 4, 256);
  pl->off_part = off;
  off = loki::align_up(off + (size_t)units * 2 * p.nA * G * (g.D + 2) * 4, 256);  // full or half parts
  pl->off_spec = off;
  if (p.spec) {
    off = loki::align_up(off + (size_t)units * G * p.ccap * 8, 256);  // cbuf
    off = loki::align_up(off + (size_t)units * G * 4, 256);           // ccnt (zeroed, self-resetting)
    off = loki::align_up(off + (size_t)units * G * p.nA * 4, 256);    // cwin
  }
  pl->off_logits = off;
  if (a->weights_out != nullptr) off = loki::align_up(off + (size_t)units * G * g.S_cap * 4, 256);
  pl->off_loff = off;
  if (p.lists) off = loki::align_up(off + (size_t)units * (2 * p.nA + 1) * 4, 256);
  pl->off_ml = off;
  if (p.lists && a->weights_out != nullptr) off = loki::align_up(off + (size_t)units * G * 2 * 4, 256);
  pl->ws = off;
  return LOKI_OK;
}

// phases: bit 0 the A-only launch, bit 1 the B-only launch (split plans; both = the decode step).
// `cached_maps`: the four tensor maps of an earlier call with identical arguments (plan cache).
loki_status run_pipe(const loki_decode_args* a, PipePlan& pl, void* stream, int phases = 3,
                     const loki::TmaDesc* cached_maps = nullptr, loki::TmaDesc* maps_out = nullptr) {
  const loki_kv_geom& g = a->g;
  if (a->workspace == nullptr || a->workspace_bytes < pl.ws)
    return fail(LOKI_ERR_SHAPE, "workspace of %zu bytes required", pl.ws);
  loki::PipeParams& p = pl.p;
  uint8_t* ws = static_cast<uint8_t*>(a->workspace);
  p.q_hat = a->q_hat;
  p.B = g.B;
  p.Hq = g.Hq;
  p.Hkv = g.Hkv;
  p.G = g.Hq / g.Hkv;
  p.D = g.D;
  p.S_cap = g.S_cap;
  p.lens = a->lens;
  p.S_max = a->S_max;
  p.d = a->d < 1 ? 1 : a->d;
  p.k_f = a->k_f;
  p.k_fixed = a->k_fixed;
  p.idx_stride = a->idx_stride;
  p.out = a->out;
  p.idx_out = a->idx_out;
  p.approx_out = a->approx_out;
  p.weights_out = a->weights_out;
  p.qscale = (float)(1.4426950408889634 / sqrt((double)g.D));
  {
    const loki::RowSpace rs = loki::row_space(g);
    p.row_sb = rs.sb;
    p.row_sh = rs.sh;
  }
  p.ctrl = reinterpret_cast<uint32_t*>(ws);
  p.hist = reinterpret_cast<uint32_t*>(ws + pl.off_hist);
  p.keys = reinterpret_cast<uint32_t*>(ws + pl.off_keys);
  p.tcs = reinterpret_cast<unsigned long long*>(ws + pl.off_tcs);
  p.poff = a->idx_out ? reinterpret_cast<uint32_t*>(ws + pl.off_poff) : nullptr;
  if (p.spec) {
    size_t o = pl.off_spec;
    p.cbuf = reinterpret_cast<unsigned long long*>(ws + o);
    o = loki::align_up(o + (size_t)p.units * p.G * p.ccap * 8, 256);
    p.ccnt = reinterpret_cast<uint32_t*>(ws + o);
    o = loki::align_up(o + (size_t)p.units * p.G * 4, 256);
    p.cwin = reinterpret_cast<uint32_t*>(ws + o);
  }
  p.part = reinterpret_cast<float*>(ws + pl.off_part);
  p.logits = a->weights_out ? reinterpret_cast<float*>(ws + pl.off_logits) : nullptr;
  p.sel = p.lists ? p.keys : nullptr;
  p.loff = p.lists ? reinterpret_cast<uint32_t*>(ws + pl.off_loff) : nullptr;
  p.ml = (p.lists && a->weights_out) ? reinterpret_cast<float*>(ws + pl.off_ml) : nullptr;
  p.debug = env_int("LOKI_DEBUG", 0);
  p.spin_ns = (long long)env_int("LOKI_SPIN_S", 20) * 1000000000LL;  // sanitizer runs raise it
  p.trace = (loki::g_phase_trace != nullptr && p.n_tickets * 4 <= (long long)loki::g_phase_trace_ctas * 8)
                ? loki::g_phase_trace : nullptr;
  loki::TmaDesc maps[4];
  if (cached_maps != nullptr) {
    for (int i = 0; i < 4; ++i) maps[i] = cached_maps[i];
  } else if (!loki::encode_pipe_tma(a->K, a->V, g, p.dbox, p.r1, p.split_k ? p.d : 0, p.mma != 0, p.lead_swz,
                                    maps)) {
    return fail(LOKI_ERR_CUDA, "cuTensorMapEncodeTiled rejected the cache geometry");
  }
  if (maps_out != nullptr)
    for (int i = 0; i < 4; ++i) maps_out[i] = maps[i];
  cudaError_t e = cudaSuccess;
  if (!pl.split && phases != 3) return fail(LOKI_ERR_UNSUPPORTED, "single-launch plan: phases run together");
  if (pl.split) {
    loki::PipeParams pa = p, pb = p;
    pa.n_tickets = (long long)p.units * p.nAa;
    if (p.shared) pa.G = 1;  // the A launch selects once per unit, on the group's summed query
    // units whose B parts run as halves (short drain, opt-in: the grouping of the partial states then
    // depends on the number of units, so KV-head shards would not be bit-identical to one launch)
    int tail = p.halves == 2 ? p.units
               : p.halves ? (int)ceil(env_int("LOKI_PIPE_TAIL_X10", 2) / 10.0 * pl.grid2 / p.nA) : 0;
    pb.lag = tail > p.units ? p.units : tail;
    pb.n_tickets = (long long)(p.units - pb.lag) * p.nA + (long long)pb.lag * 2 * p.nA;
    // trace rows: the A launch's tickets, then the B launch's (diagnostics only)
    const bool fits = loki::g_phase_trace != nullptr &&
                      (pa.n_tickets + pb.n_tickets) * 4 <= (long long)loki::g_phase_trace_ctas * 8;
    pa.trace = fits ? loki::g_phase_trace : nullptr;
    pb.trace = fits ? loki::g_phase_trace + pa.n_tickets * 4 : nullptr;
    if (!(phases & 1) || p.dense) {  // (dense decode: no A launch)
    } else if (pl.ws_select) {
      pa.off_ring = pl.sel_layout.off_ring;
      pa.off_bars = pl.sel_layout.off_bars;
      pa.off_hist = pl.sel_layout.off_hist;
      pa.off_kchip = pl.sel_layout.off_kchip;
      pa.off_cand = pl.sel_layout.off_cand;
      pa.cand_bytes = pl.sel_layout.cand_bytes;
      pa.nst = pl.sel_layout.nst;
      pa.umma = pl.sel_layout.umma;
      pa.ust = pl.sel_layout.ust;
      pa.off_qt = pl.sel_layout.off_qt;
      e = loki::launch_pipe_select(pa, g.dtype, pl.ws_onchip, pl.grid1, pl.smem1, maps,
                                   static_cast<cudaStream_t>(stream), pl.ws_groups);
    } else {
      e = loki::launch_pipe(pa, g.dtype, pl.G_Ta, pl.grid1, pl.smem1, maps, static_cast<cudaStream_t>(stream), pl.big,
                            pl.mode3 ? 3 : 1);
    }
    size_t smem2 = pl.smem;
    if (pl.smem_b > 0) {
      pb.off_ring = pl.blay.off_ring;
      pb.off_bars = pl.blay.off_bars;
      pb.off_hist = pl.blay.off_hist;
      pb.off_ents = pl.blay.off_ents;
      smem2 = pl.smem_b;
    }
    if (e == cudaSuccess && (phases & 2))
      e = loki::launch_pipe(pb, g.dtype, pl.G_T, pl.grid2, smem2, maps, static_cast<cudaStream_t>(stream), pl.big, 2);
  } else {
    e = loki::launch_pipe(p, g.dtype, pl.G_T, pl.grid, pl.smem, maps, static_cast<cudaStream_t>(stream), pl.big);
  }
  if (e == cudaSuccess && (phases & 2) && p.lists && a->weights_out != nullptr)  // diagnostics: weights from lists
    e = loki::launch_pipe_weights(p, static_cast<cudaStream_t>(stream));
  if (e == cudaSuccess) e = cudaGetLastError();
  return cuda_status(e, "loki_decode (pipe) launch");
}

}  // namespace

extern "C" {

const char* loki_last_error(void) { return g_last_error.c_str(); }

int32_t loki_abi_version(void) { return LOKI_ABI_VERSION; }

loki_status loki_device_check(int32_t device) {
  cudaDeviceProp prop;
  cudaError_t e = cudaGetDeviceProperties(&prop, device);
  if (e != cudaSuccess) return cuda_status(e, "cudaGetDeviceProperties");
  if (prop.major != 10 || prop.minor != 0)
    return fail(LOKI_ERR_UNSUPPORTED, "device %d is sm_%d%d; libloki_b200 is built for sm_100a", device,
                prop.major, prop.minor);
  return LOKI_OK;
}

loki_status loki_decode_workspace_bytes(const loki_decode_args* a, size_t* bytes) {
  loki_status s = validate(a);
  if (s != LOKI_OK) return s;
  loki_decode_args a1, a2;
  a = small_batch_plan(canonical_mode(a, &a1), &a2);
  {
    PipePlan pl;
    if (pipe_eligible(a) && make_pipe_plan(a, &pl) == LOKI_OK) {
      *bytes = pl.ws;
      return LOKI_OK;
    }
  }
  if (a->select_mode == LOKI_SELECT_TOPK_SHARED) return shared_unsupported(a);
  loki::Plan plan;
  loki::FusedParams p{};
  TmaGeom tg{};
  s = make_plan(a, &plan, &p, &tg);
  if (s != LOKI_OK) return s;
  *bytes = plan.workspace;
  return LOKI_OK;
}

loki_status loki_decode_plan(const loki_decode_args* a, int32_t* ctas_per_unit, int32_t* rows_per_cta,
                             size_t* smem_bytes) {
  loki_status s = validate(a);
  if (s != LOKI_OK) return s;
  loki_decode_args a1, a2;
  a = small_batch_plan(canonical_mode(a, &a1), &a2);
  PipePlan pl;
  if (pipe_eligible(a) && make_pipe_plan(a, &pl) == LOKI_OK) {  // persistent grid: 0 (-2: split, two launches)
    if (ctas_per_unit) *ctas_per_unit = pl.split ? -2 : 0;
    if (rows_per_cta) *rows_per_cta = pl.p.Lc;
    if (smem_bytes) *smem_bytes = pl.smem;
    return LOKI_OK;
  }
  if (a->select_mode == LOKI_SELECT_TOPK_SHARED) return shared_unsupported(a);
  loki::Plan plan;
  loki::FusedParams p{};
  TmaGeom tg{};
  s = make_plan(a, &plan, &p, &tg);
  if (s != LOKI_OK) return s;
  if (ctas_per_unit) *ctas_per_unit = plan.C;
  if (rows_per_cta) *rows_per_cta = plan.Lmax;
  if (smem_bytes) *smem_bytes = plan.smem;
  return LOKI_OK;
}

loki_status loki_decode_phase(const loki_decode_args* a, int32_t launches, void* stream) {
  loki_status s = validate(a);
  if (s != LOKI_OK) return s;
  loki_decode_args a1, a2;
  a = small_batch_plan(canonical_mode(a, &a1), &a2);
  if (launches < 1 || launches > 3) return fail(LOKI_ERR_DOMAIN, "launches %d not in {1, 2, 3}", launches);
  PipePlan pl;
  if (!pipe_eligible(a)) return fail(LOKI_ERR_UNSUPPORTED, "phase launches exist on the pipe path only");
  s = make_pipe_plan(a, &pl);
  if (s != LOKI_OK) return s;
  return run_pipe(a, pl, stream, launches);
}

// Per-thread cache of recent pipe plans and their tensor maps, keyed by the argument block's bytes and
// the device: a serving loop (LokiDecoder, the HF cache, eager replays) calls with identical arguments every
// step, so the planning, occupancy queries and four cuTensorMapEncodeTiled calls run once.  Tuning mode
// (LOKI_TUNING=1: the plan may follow the environment) bypasses it.
struct PlanCacheEntry {
  bool valid = false;
  int dev = -1;
  loki_decode_args a{};
  PipePlan pl;
  loki::TmaDesc maps[4];
};
constexpr int kPlanCache = 8;
thread_local PlanCacheEntry g_plan_cache[kPlanCache];
thread_local int g_plan_next = 0;

loki_status loki_decode(const loki_decode_args* a_in, void* stream) {
  loki_status s = validate(a_in);
  if (s != LOKI_OK) return s;
  const bool cacheable = !tuning_enabled() && loki::g_phase_trace == nullptr;
  int dev = 0;
  if (cacheable && cudaGetDevice(&dev) == cudaSuccess) {
    for (PlanCacheEntry& e : g_plan_cache)
      if (e.valid && e.dev == dev && std::memcmp(&e.a, a_in, sizeof(loki_decode_args)) == 0)
        return run_pipe(&e.a, e.pl, stream, 3, e.maps);
  }
  loki_decode_args a1, a2;
  const loki_decode_args* a = small_batch_plan(canonical_mode(a_in, &a1), &a2);
  {
    PipePlan pl;
    if (pipe_eligible(a) && make_pipe_plan(a, &pl) == LOKI_OK) {
      if (!cacheable || a != a_in) return run_pipe(a, pl, stream);
      PlanCacheEntry& e = g_plan_cache[g_plan_next];
      e.valid = false;
      const loki_status r = run_pipe(a, pl, stream, 3, nullptr, e.maps);
      if (r == LOKI_OK) {
        e.a = *a_in;
        e.dev = dev;
        e.pl = pl;
        e.valid = true;
        g_plan_next = (g_plan_next + 1) % kPlanCache;
      }
      return r;
    }
  }
  if (a->select_mode == LOKI_SELECT_TOPK_SHARED) return shared_unsupported(a);
  loki::Plan plan;
  loki::FusedParams p{};
  TmaGeom tg{};
  s = make_plan(a, &plan, &p, &tg);
  if (s != LOKI_OK) return s;
  if (plan.workspace > 0 && (a->workspace == nullptr || a->workspace_bytes < plan.workspace))
    return fail(LOKI_ERR_SHAPE, "workspace of %zu bytes required", plan.workspace);
  const loki_kv_geom& g = a->g;
  p.q_hat = a->q_hat;
  p.K = a->K;
  p.V = a->V;
  p.sb = g.stride_b;
  p.sh = g.stride_h;
  p.ss = g.stride_s;
  p.B = g.B;
  p.Hq = g.Hq;
  p.Hkv = g.Hkv;
  p.G = g.Hq / g.Hkv;
  p.D = g.D;
  p.S_cap = g.S_cap;
  p.lens = a->lens;
  p.S_max = a->S_max;
  p.d = a->d < 1 ? 1 : a->d;
  p.k_f = a->k_f;
  p.k_fixed = a->k_fixed;
  p.select_mode = a->select_mode;
  p.ext_scores = a->ext_scores;
  p.ext_idx = a->ext_idx;
  p.idx_stride = a->idx_stride;
  p.out = a->out;
  p.idx_out = a->idx_out;
  p.approx_out = a->approx_out;
  p.weights_out = a->weights_out;
  p.C = plan.C;
  p.Lmax = plan.Lmax;
  p.keys_ws = plan.keys_in_smem ? nullptr : static_cast<uint32_t*>(a->workspace);
  p.debug = env_int("LOKI_DEBUG", 0);
  p.trace = (loki::g_phase_trace != nullptr && g.B * g.Hkv * plan.C <= loki::g_phase_trace_ctas)
                ? loki::g_phase_trace : nullptr;
  p.qscale = (float)(1.4426950408889634 / sqrt((double)g.D));
  cudaError_t e;
  if (plan.tma) {
    loki::TmaDesc maps[5];
    if (!loki::encode_tma(a->K, a->V, g, tg.dbox, tg.r1, tg.r3, maps))
      return fail(LOKI_ERR_CUDA, "cuTensorMapEncodeTiled rejected the cache geometry");
    e = loki::launch_fused_tma(p, plan, maps, static_cast<cudaStream_t>(stream));
  } else {
    e = loki::launch_fused(p, plan, static_cast<cudaStream_t>(stream));
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  return cuda_status(e, "loki_decode launch");
}

loki_status loki_append_kv(const float* q_raw, const float* k_raw, const float* v_new, const float* P,
                           int64_t P_head_stride, const double* inv_freq, const int64_t* positions,
                           int32_t rope_mode, void* K, void* V, loki_kv_geom g, const int32_t* rows,
                           float* q_hat_out, void* stream) {
  if (g.B < 1 || g.Hq < 1 || g.Hkv < 1 || g.D < 1 || g.S_cap < 1 || g.Hq % g.Hkv != 0)
    return fail(LOKI_ERR_SHAPE, "invalid geometry B=%d Hq=%d Hkv=%d D=%d", g.B, g.Hq, g.Hkv, g.D);
  if (g.Hq / g.Hkv > 8) return fail(LOKI_ERR_UNSUPPORTED, "group size %d > 8", g.Hq / g.Hkv);
  if (g.D > 256) return fail(LOKI_ERR_UNSUPPORTED, "head dim %d > 256", g.D);
  if (g.dtype != LOKI_DTYPE_F32 && g.dtype != LOKI_DTYPE_BF16)
    return fail(LOKI_ERR_UNSUPPORTED, "cache dtype code %d", g.dtype);
  if (rope_mode < LOKI_ROPE_NONE || rope_mode > LOKI_ROPE_PROJECT_THEN_ROTATE)
    return fail(LOKI_ERR_DOMAIN, "rope_mode %d", rope_mode);
  if (rope_mode != LOKI_ROPE_NONE && (inv_freq == nullptr || g.D % 2 != 0))
    return fail(LOKI_ERR_SHAPE, "head_dim must be a positive even number, got %d", g.D);
  if (k_raw == nullptr || K == nullptr) return fail(LOKI_ERR_SHAPE, "k_raw and K are required");
  if (v_new != nullptr && V == nullptr) return fail(LOKI_ERR_SHAPE, "V is required with v_new");
  if (q_raw != nullptr && q_hat_out == nullptr) return fail(LOKI_ERR_SHAPE, "q_hat_out is required with q_raw");
  cudaError_t e = loki::launch_append(q_raw, k_raw, v_new, P, P_head_stride, inv_freq, positions, rope_mode, K, V,
                                      g, rows, q_hat_out, static_cast<cudaStream_t>(stream));
  return cuda_status(e, "loki_append_kv launch");
}

loki_status loki_gathered_scores(const float* Q, int32_t M, const void* K, int64_t k_row_stride, int32_t dtype,
                                 int32_t D, const int64_t* idx, int32_t n, float* out, void* stream) {
  if (M < 1 || D < 1 || n < 0 || k_row_stride < D) return fail(LOKI_ERR_SHAPE, "invalid gathered-score shape");
  if (dtype != LOKI_DTYPE_F32 && dtype != LOKI_DTYPE_BF16) return fail(LOKI_ERR_UNSUPPORTED, "dtype %d", dtype);
  cudaError_t e = loki::launch_gathered_scores(Q, M, K, k_row_stride, dtype, D, idx, n, out,
                                               static_cast<cudaStream_t>(stream));
  return cuda_status(e, "loki_gathered_scores launch");
}

size_t loki_weighted_sum_workspace(int32_t n, int32_t D) {
  const int nsplit = loki::ceil_div(n > 0 ? n : 1, 256);
  return (size_t)nsplit * (D > 0 ? D : 1) * sizeof(float);
}

loki_status loki_weighted_sum(const float* w, const void* V, int64_t v_row_stride, int32_t dtype, int32_t D,
                              const int64_t* idx, int32_t n, float* out, void* partial, size_t partial_bytes,
                              void* stream) {
  if (D < 1 || n < 0 || v_row_stride < D) return fail(LOKI_ERR_SHAPE, "invalid weighted-sum shape");
  if (dtype != LOKI_DTYPE_F32 && dtype != LOKI_DTYPE_BF16) return fail(LOKI_ERR_UNSUPPORTED, "dtype %d", dtype);
  if (partial == nullptr || partial_bytes < loki_weighted_sum_workspace(n, D))
    return fail(LOKI_ERR_SHAPE, "partial workspace of %zu bytes required", loki_weighted_sum_workspace(n, D));
  const int nsplit = loki::ceil_div(n > 0 ? n : 1, 256);
  cudaError_t e = loki::launch_weighted_sum(w, V, v_row_stride, dtype, D, idx, n, out, static_cast<float*>(partial),
                                            nsplit, static_cast<cudaStream_t>(stream));
  return cuda_status(e, "loki_weighted_sum launch");
}

loki_status loki_softmax_rows(const float* x, int64_t rows, int32_t n, int64_t stride, float* out, void* stream) {
  if (n < 1) return fail(LOKI_ERR_SHAPE, "softmax_row expects a nonempty vector");
  if (rows < 0 || stride < n) return fail(LOKI_ERR_SHAPE, "invalid softmax shape");
  cudaError_t e = loki::launch_softmax_rows(x, rows, n, stride, out, static_cast<cudaStream_t>(stream));
  return cuda_status(e, "loki_softmax_rows launch");
}

loki_status loki_rope(const void* x, void* out, int32_t io_dtype, int64_t n_rows, int32_t D,
                      const int64_t* positions, const double* inv_freq, void* stream) {
  if (D <= 0 || D % 2 != 0) return fail(LOKI_ERR_SHAPE, "head_dim must be a positive even number, got %d", D);
  if (io_dtype != LOKI_DTYPE_F32 && io_dtype != LOKI_DTYPE_F64)
    return fail(LOKI_ERR_UNSUPPORTED, "rope dtype %d", io_dtype);
  if (n_rows < 0 || positions == nullptr || inv_freq == nullptr) return fail(LOKI_ERR_SHAPE, "invalid rope arguments");
  cudaError_t e = loki::launch_rope(x, out, io_dtype, n_rows, D, positions, inv_freq,
                                    static_cast<cudaStream_t>(stream));
  return cuda_status(e, "loki_rope launch");
}

loki_status loki_set_phase_trace(int64_t* buf, int32_t max_ctas) {
  loki::g_phase_trace = reinterpret_cast<long long*>(buf);
  loki::g_phase_trace_ctas = buf ? max_ctas : 0;
  return LOKI_OK;
}

loki_status loki_project_rows(const void* x, int32_t x_dtype, const int64_t* x_strides, const float* P,
                              void* out, int32_t out_dtype, const int64_t* out_strides, int32_t B, int32_t H,
                              int32_t S, int32_t D, int32_t G, void* stream) {
  if (B < 0 || H < 1 || S < 0 || D < 1 || G < 1 || H % G != 0)
    return fail(LOKI_ERR_SHAPE, "invalid projection shape B=%d H=%d S=%d D=%d G=%d", B, H, S, D, G);
  if (D > 128) return fail(LOKI_ERR_UNSUPPORTED, "projection head dim %d > 128", D);
  if ((x_dtype != LOKI_DTYPE_F32 && x_dtype != LOKI_DTYPE_BF16) ||
      (out_dtype != LOKI_DTYPE_F32 && out_dtype != LOKI_DTYPE_BF16))
    return fail(LOKI_ERR_UNSUPPORTED, "projection dtypes %d -> %d", x_dtype, out_dtype);
  if (x == nullptr || P == nullptr || out == nullptr || x_strides == nullptr || out_strides == nullptr)
    return fail(LOKI_ERR_SHAPE, "null projection argument");
  cudaError_t e = loki::launch_project_rows(x, x_dtype, P, out, out_dtype, B, H, S, D, G, x_strides, out_strides,
                                            static_cast<cudaStream_t>(stream));
  return cuda_status(e, "loki_project_rows launch");
}

loki_status loki_index_status(const int64_t* idx, int32_t n, int64_t bound, int32_t* status, void* stream) {
  if (n < 0 || status == nullptr) return fail(LOKI_ERR_SHAPE, "invalid index-status arguments");
  cudaError_t e = loki::launch_index_status(idx, n, bound, status, static_cast<cudaStream_t>(stream));
  return cuda_status(e, "loki_index_status launch");
}

}  // extern "C"
