// Building blocks shared by the fused Loki decode kernels (LDG and TMA
// variants): per-CTA context, cluster-wide radix top-k with the reference's
// tie rule, ordered compaction, and the fixed-order softmax-state merge.
#pragma once

#include <cooperative_groups.h>
#include <cstdio>
#include <math_constants.h>

#include "loki_common.cuh"
#include "loki_internal.h"

namespace loki {
namespace fused {

namespace cg = cooperative_groups;

constexpr int kRadixBins = 256;
constexpr int kMaxG = 8;

struct MiscState {
  uint32_t prefix[kMaxG];
  int32_t krem[kMaxG];
  int32_t done[kMaxG];
  uint32_t T[kMaxG];
  long long gt[kMaxG];
  int32_t cnt_gt[kMaxG];
  int32_t cnt_eq[kMaxG];
  int32_t tie_take[kMaxG];
  int32_t sel_off[kMaxG];
  int32_t ext_p0[kMaxG];
  int32_t ext_p1[kMaxG];
  int32_t scan_a[2][32];
  int32_t scan_b[2][32];
  float gm[kMaxG];
  float gl[kMaxG];
  int32_t lgt[kMaxG];   // local keys strictly above the threshold (from histograms)
  int32_t leq[kMaxG];   // local keys equal to the exact threshold
  int32_t ncand[2];     // candidate list lengths (single-head fast path)
  int32_t n_union;      // rows gathered in phase 3 (single-head fast path)
  int32_t wcnt[2][32];  // per-warp counts of the ordered emission
  long long probe[16];  // LOKI_DEBUG & 8: clock64 stamps of block 0 (tuning only)
};

// Exclusive prefix of `pred` over the block in thread order, plus the total.
template <int NT>
__device__ __forceinline__ int block_scan_pred(bool pred, int* total, int32_t* scratch) {
  constexpr int NW = NT / 32;
  const int lane = lane_id(), w = warp_id();
  const unsigned bal = __ballot_sync(0xffffffffu, pred);
  const int in_warp = __popc(bal & ((1u << lane) - 1u));
  if (lane == 0) scratch[w] = __popc(bal);
  __syncthreads();
  int before = 0, tot = 0;
#pragma unroll
  for (int i = 0; i < NW; ++i) {
    const int c = scratch[i];
    before += (i < w) ? c : 0;
    tot += c;
  }
  *total = tot;
  return before + in_warp;
}

// Histogram update.  Plain shared-memory atomics: on B200 this beat
// match.any-based warp aggregation (phase 1 26.6 -> 19.7 us per CTA slice,
// profiles/r01_phase_trace.md).
__device__ __forceinline__ void hist_add(uint32_t* hist, bool active, uint32_t bin) {
  if (active) atomicAdd(&hist[bin], 1u);
}

// (m, l) <- (m, l) (+) (m2, l2) in the log2 domain; s1 / s2 rescale the accumulators.
__device__ __forceinline__ void merge_state(float& m, float& l, float m2, float l2, float& s1, float& s2) {
  const float mn = fmaxf(m, m2);
  s1 = (m == -CUDART_INF_F) ? 0.f : exp2f(m - mn);
  s2 = (m2 == -CUDART_INF_F) ? 0.f : exp2f(m2 - mn);
  l = l * s1 + l2 * s2;
  m = mn;
}

#define LOKI_PROBE(ms, k)                                                  \
  do {                                                                     \
    if ((p.debug & 8) && threadIdx.x == 0) (ms)->probe[(k)] = clock64();  \
  } while (0)

__device__ __forceinline__ void dbg_stamp(const FusedParams& p, int slot) {
  if ((p.debug & 4) && p.trace != nullptr && threadIdx.x == 0) {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[(size_t)blockIdx.x * 8 + slot] = t;
  }
}

// Per-CTA view of its (batch, KV head) unit and cache slice.
struct Ctx {
  int C, rank, b, hk, G, D, Lmax, S, kb, s0, s1, n_local;
  bool select_all, need_keys;
  size_t qrow0;
  uint32_t* keys;
  uint8_t* selmask;
  uint16_t* uni;
  uint32_t* hist;   // [2][G_T][256]
  uint32_t* ghist;  // [G_T][256]
  float* part;      // [NW][G_T][D + 2]
  float* fin;       // [G_T][D + 2]
  MiscState* ms;
};

// Fills the context; returns false when the unit has no rows (the whole
// cluster leaves together: S is uniform per unit).
template <int G_T>
__device__ __forceinline__ bool make_ctx(const FusedParams& p, uint8_t* smem, int rank, Ctx& c) {
  c.C = p.C;
  c.rank = rank;
  const int unit = blockIdx.x / p.C;
  c.b = unit / p.Hkv;
  c.hk = unit % p.Hkv;
  c.G = p.G;
  c.D = p.D;
  c.Lmax = p.Lmax;
  int S = p.lens[c.b];
  S = S > p.S_max ? p.S_max : S;  // S_max <= S_cap (host); slices are sized for S_max rows
  c.S = S;
  if (S <= 0) return false;
  int kb;
  if (p.select_mode == 1) kb = S;
  else if (p.k_fixed > 0) kb = p.k_fixed < S ? p.k_fixed : S;
  else kb = resolve_fraction(p.k_f, S);
  c.kb = kb;
  // slices are whole phase-1 tiles (host sizes Lmax with the same rule)
  const int L = ceil_div(ceil_div(S, p.C), p.slice_align) * p.slice_align;
  c.s0 = min(rank * L, S);
  c.s1 = min(c.s0 + L, S);
  c.n_local = c.s1 - c.s0;
  c.select_all = (p.select_mode == 1) || ((p.select_mode == 0 || p.select_mode == 2) && kb == S);
  c.need_keys = (p.select_mode == 0) && !c.select_all;
  c.qrow0 = (size_t)c.b * p.Hq + (size_t)c.hk * c.G;
  c.keys = p.keys_ws ? p.keys_ws + (size_t)blockIdx.x * G_T * p.Lmax : reinterpret_cast<uint32_t*>(smem + p.off_keys);
  c.selmask = smem + p.off_sel;
  c.uni = reinterpret_cast<uint16_t*>(smem + p.off_union);
  c.hist = reinterpret_cast<uint32_t*>(smem + p.off_hist);
  c.ghist = c.hist + 2 * G_T * kRadixBins;
  c.part = reinterpret_cast<float*>(smem + p.off_merge);
  c.fin = reinterpret_cast<float*>(smem + p.off_final);
  c.ms = reinterpret_cast<MiscState*>(smem + p.off_misc);
  return true;
}

template <int NT, int G_T>
__device__ __forceinline__ void init_state(const Ctx& c) {
  const int tid = threadIdx.x;
  for (int i = tid; i < G_T * kRadixBins; i += NT) c.hist[i] = 0u;
  for (int i = tid; i < c.Lmax; i += NT) c.selmask[i] = 0;
  if (tid < kMaxG) {
    c.ms->prefix[tid] = 0u;
    c.ms->krem[tid] = c.kb;
    c.ms->done[tid] = (tid >= c.G) ? 1 : 0;
  }
}

// Phase 1 from externally supplied fp32 scores (topk_indices on given scores).
template <int NT>
__device__ __forceinline__ void keys_from_scores(const FusedParams& p, const Ctx& c) {
  const int tid = threadIdx.x;
  for (int g = 0; g < c.G; ++g) {
    const float* src = p.ext_scores + (c.qrow0 + g) * (size_t)p.S_cap;
    for (int j0 = 0; j0 < c.n_local; j0 += NT) {
      const int j = j0 + tid;
      const bool ok = j < c.n_local;
      const float s = ok ? src[c.s0 + j] : 0.f;
      const uint32_t key = order_key(s);
      if (ok) c.keys[g * c.Lmax + j] = key;
      if (c.need_keys) hist_add(c.hist + g * kRadixBins, ok, key >> 24);
    }
  }
}

// Phase 2, single query head per unit (MHA).  Same selection as the generic
// path below, cheaper:
//   - each radix pass scans only the keys that still match the prefix: pass 1
//     compacts the pass-0 matches into `uni`, pass 2 the pass-1 matches into
//     the (still unused) merge scratch when they fit;
//   - the counts above / at the threshold come from the local histograms, so
//     no extra scan over the slice;
//   - the ordered emission writes the phase-3 gather list and idx_out directly
//     (two passes over warp-contiguous row ranges, one block barrier).
// Exact end of the single-head radix select once at most 256 keys match
// the prefix cluster-wide: every CTA publishes its candidate keys and its
// count of keys above the prefix, one cluster barrier, then every CTA ranks
// the (small) candidate union itself -- the threshold, the tie split and the
// per-rank offsets follow without further barriers.
template <int NT>
__device__ void exact_finish(const FusedParams& p, const Ctx& c, cg::cluster_group& cluster, int shift, int level,
                             int r0, int r1, const uint16_t* segA, const uint16_t* segB, int nA, int nB) {
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = lane_id(), w = warp_id();
  MiscState* ms = c.ms;
  const uint32_t mask = 0xFFFFFFFFu << shift;
  const uint32_t pre = ms->prefix[0];
  const unsigned lt = (1u << lane) - 1u;
  const int n_src = level == 0 ? (r1 - r0) : (level == 1 ? nA : nB);
  auto key_at = [&](int i) {
    const int j = level == 0 ? r0 + i : (level == 1 ? (int)segA[i] : (int)segB[i]);
    return c.keys[j];
  };
  // publish: candidate keys into ghist[0, n) in warp order
  int cnt = 0;
  for (int i0 = 0; i0 < n_src; i0 += 32) {
    const int i = i0 + lane;
    cnt += __popc(__ballot_sync(0xffffffffu, i < n_src && (key_at(i) & mask) == pre));
  }
  if (lane == 0) ms->wcnt[0][w] = cnt;
  __syncthreads();
  int off = 0, tot = 0;
  for (int ww = 0; ww < NW; ++ww) {
    off += ww < w ? ms->wcnt[0][ww] : 0;
    tot += ms->wcnt[0][ww];
  }
  for (int i0 = 0; i0 < n_src; i0 += 32) {
    const int i = i0 + lane;
    const uint32_t key = i < n_src ? key_at(i) : 0u;
    const bool m = i < n_src && (key & mask) == pre;
    const unsigned bal = __ballot_sync(0xffffffffu, m);
    if (m) c.ghist[off + __popc(bal & lt)] = key;
    off += __popc(bal);
  }
  if (tid == 0) ms->ncand[0] = tot;
  cluster.sync();
  // gather every rank's candidates (and their rank) into local scratch
  uint32_t* ck = c.hist;                   // keys   [<= 256]
  uint32_t* cr = c.hist + kRadixBins;      // owner  [<= 256]
  int offs[17];
  int ntot = 0;
  for (int r = 0; r < c.C; ++r) {
    offs[r] = ntot;
    ntot += cluster.map_shared_rank(ms, r)->ncand[0];
  }
  offs[c.C] = ntot;
  for (int i = tid; i < ntot; i += NT) {
    int r = 0;
    while (offs[r + 1] <= i) ++r;
    ck[i] = cluster.map_shared_rank(c.ghist, r)[i - offs[r]];
    cr[i] = (uint32_t)r;
  }
  if (tid < c.C) ms->wcnt[1][tid] = cluster.map_shared_rank(ms, tid)->cnt_gt[0];
  __syncthreads();
  // the krem-th largest candidate is the exact threshold T
  const int krem = ms->krem[0];
  for (int i = tid; i < ntot; i += NT) {
    const uint32_t x = ck[i];
    int g = 0, e = 0;
    for (int t = 0; t < ntot; ++t) {
      g += ck[t] > x;
      e += ck[t] == x;
    }
    if (g < krem && krem <= g + e) ms->T[0] = x;
  }
  __syncthreads();
  if (tid == 0) {
    const uint32_t T = ms->T[0];
    int above_T = 0;
    for (int t = 0; t < ntot; ++t) above_T += ck[t] > T;
    const int need = krem - above_T;  // threshold ties still to take, lowest rank first
    int eq_before = 0, sel_before = 0, take = 0;
    for (int r = 0; r <= c.rank; ++r) {
      int gt_r = ms->wcnt[1][r], eq_r = 0;
      for (int t = offs[r]; t < offs[r + 1]; ++t) {
        gt_r += ck[t] > T;
        eq_r += ck[t] == T;
      }
      int tk = need - eq_before;  // ties at T go to the lowest ranks (lowest indices) first
      tk = tk < 0 ? 0 : (tk > eq_r ? eq_r : tk);
      if (r < c.rank) {
        sel_before += gt_r + tk;
        eq_before += eq_r;
      } else {
        take = tk;
        ms->lgt[0] = gt_r;
        ms->leq[0] = eq_r;
      }
    }
    ms->done[0] = 2;
    ms->gt[0] = (long long)T;
    ms->tie_take[0] = take;
    ms->sel_off[0] = sel_before;
    ms->n_union = ms->lgt[0] + take;
  }
  __syncthreads();
}

template <int NT>
__device__ void select_single(const FusedParams& p, const Ctx& c, cg::cluster_group& cluster) {
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = lane_id(), w = warp_id();
  MiscState* ms = c.ms;
  const int n_local = c.n_local;
  const uint32_t* keys = c.keys;
  const unsigned lt = (1u << lane) - 1u;
  // warp w owns the contiguous rows [w * Rw, w * Rw + Rw) and private segments of
  // the candidate lists (no cross-warp atomics): listA in `uni`, listB in the merge scratch
  const int Rw = ceil_div(ceil_div(n_local, NW), 32) * 32;
  const int r0 = min(w * Rw, n_local), r1 = min(r0 + Rw, n_local);
  uint16_t* segA = c.uni + w * Rw;
  const int capBw = (NW * (c.D + 2) * 2) / NW;  // uint16 entries per warp in the merge scratch
  uint16_t* segB = reinterpret_cast<uint16_t*>(c.part) + w * capBw;
  int nA = 0, nB = 0;  // this warp's list lengths (warp-uniform)
  int level = 0;       // 0: scan rows, 1: scan segA, 2: scan segB
  bool exact = false;  // threshold found by exact_finish (counts already exchanged)
  if (tid == 0) {
    ms->cnt_gt[0] = 0;     // running count of local keys above the prefix
    ms->lgt[1] = n_local;  // local keys matching the prefix so far
  }
  __syncthreads();
  LOKI_PROBE(ms, 0);
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = 24 - 8 * pass;
    uint32_t* hcur = c.hist + (pass & 1) * kRadixBins;
    if (pass > 0) {
      const uint32_t hi_mask = 0xFFFFFFFFu << (shift + 8);
      const uint32_t pre = ms->prefix[0];
      // compact the keys matching the prefix: pass 1 -> segA, pass 2 -> segB when it surely fits
      const int to = (pass == 1) ? 1 : ((pass == 2 && ms->lgt[1] <= capBw) ? 2 : 0);
      uint16_t* dst = to == 1 ? segA : segB;
      const int n_src = level == 0 ? (r1 - r0) : (level == 1 ? nA : nB);
      int nd = 0;
      constexpr int U = 4;  // independent keys in flight per lane
      for (int i0 = 0; i0 < n_src; i0 += 32 * U) {
        int jj[U];
        uint32_t kk[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int i = i0 + u * 32 + lane;
          jj[u] = i < n_src ? (level == 0 ? r0 + i : (level == 1 ? (int)segA[i] : (int)segB[i])) : -1;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) kk[u] = jj[u] >= 0 ? keys[jj[u]] : 0u;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const bool m = jj[u] >= 0 && ((kk[u] & hi_mask) == pre);
          if (m) atomicAdd(&hcur[(kk[u] >> shift) & 0xFFu], 1u);
          if (to) {
            const unsigned bal = __ballot_sync(0xffffffffu, m);
            if (m) dst[nd + __popc(bal & lt)] = (uint16_t)jj[u];
            nd += __popc(bal);
          }
        }
      }
      if (to == 1) { nA = nd; level = 1; }
      if (to == 2) { nB = nd; level = 2; }
    }
    LOKI_PROBE(ms, 1 + 4 * pass);
    // cluster.sync also orders this CTA's histogram writes for every thread
    cluster.sync();
    LOKI_PROBE(ms, 2 + 4 * pass);
    // merge the C ranks' histograms, one bin per thread (DSMEM loads in parallel);
    // the other buffer was last read remotely two passes ago, before this
    // pass's cluster barrier: clear it for the next pass at the same time
    for (int i = tid; i < kRadixBins; i += NT) {
      uint32_t sum = 0;
      for (int r = 0; r < c.C; ++r) sum += cluster.map_shared_rank(hcur, r)[i];
      c.ghist[i] = sum;
      c.hist[((pass + 1) & 1) * kRadixBins + i] = 0u;
    }
    __syncthreads();
    LOKI_PROBE(ms, 3 + 4 * (pass & 1));
    if (w == 0 && !ms->done[0]) {
      const int krem = ms->krem[0];
      uint32_t cnt[8], lc[8];
      uint32_t lsum = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {  // lane 0 holds the top bins 255..248
        const int bin = 255 - (lane * 8 + i);
        lc[i] = hcur[bin];
        cnt[i] = c.ghist[bin];
        lsum += cnt[i];
      }
      uint32_t incl = lsum;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += t;
      }
      const uint32_t excl = incl - lsum;
      const bool here = (excl < (uint32_t)krem) && ((uint32_t)krem <= incl);
      const int L = __ffs(__ballot_sync(0xffffffffu, here)) - 1;
      int istar = 0;
      uint32_t above = excl;
      if (lane == L) {
        for (; istar < 8; ++istar) {
          if (above + cnt[istar] >= (uint32_t)krem) break;
          above += cnt[istar];
        }
      }
      istar = __shfl_sync(0xffffffffu, istar, L);
      // local keys strictly above the chosen bin, and in it
      uint32_t up = 0, at = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (lane < L || (lane == L && i < istar)) up += lc[i];
        if (lane == L && i == istar) at = lc[i];
      }
      up = __reduce_add_sync(0xffffffffu, up);
      at = __reduce_add_sync(0xffffffffu, at);
      if (lane == L) {
        const uint32_t bin = 255u - (uint32_t)(lane * 8 + istar);
        const int rem = krem - (int)above;
        const uint32_t pre = ms->prefix[0] | (bin << shift);
        ms->prefix[0] = pre;
        ms->krem[0] = rem;
        const int lgt = ms->cnt_gt[0] + (int)up;
        const int lmatch = (int)at;
        ms->cnt_gt[0] = lgt;
        ms->lgt[1] = lmatch;  // size of the next candidate list
        ms->ncand[1] = (int)cnt[istar];  // cluster-wide keys matching the new prefix
        if ((int)cnt[istar] == rem) {  // the whole boundary bin is in: no tie to break
          ms->done[0] = 1;
          ms->gt[0] = (long long)pre - 1;
          ms->T[0] = 0u;
          ms->krem[0] = 0;
          ms->lgt[0] = lgt + lmatch;
          ms->leq[0] = 0;
        } else if (pass == 3) {
          ms->done[0] = 2;  // exact threshold key with ties to fill
          ms->gt[0] = (long long)pre;
          ms->T[0] = pre;
          ms->lgt[0] = lgt;
          ms->leq[0] = lmatch;
        }
      }
    }
    __syncthreads();
    LOKI_PROBE(ms, 4 + 4 * (pass & 1));
    if (!ms->done[0] && ms->ncand[1] <= kRadixBins) {
      // few candidates left cluster-wide: finish exactly from the candidate keys
      exact_finish<NT>(p, c, cluster, shift, level, r0, r1, segA, segB, nA, nB);
      exact = true;
      break;
    }
    if (pass == 0) dbg_stamp(p, 1);
    if (pass == 1) dbg_stamp(p, 4);
    if (pass == 2) dbg_stamp(p, 5);
    if (pass == 3) dbg_stamp(p, 6);
    if (ms->done[0]) break;
  }
  if (p.trace != nullptr && tid == 0 && !(p.debug & 4)) {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[(size_t)blockIdx.x * 8 + 2] = t;
  }
  if (!exact) {
  cluster.sync();  // every CTA's counts visible
  if (tid == 0) {
    const int need = ms->krem[0];
    int eq_before = 0, sel_before = 0;
    for (int r = 0; r < c.rank; ++r) {
      MiscState* rs = cluster.map_shared_rank(ms, r);
      const int eq = rs->leq[0];
      int take = need - eq_before;
      take = take < 0 ? 0 : (take > eq ? eq : take);
      sel_before += rs->lgt[0] + take;
      eq_before += eq;
    }
    int take = need - eq_before;
    const int eq = ms->leq[0];
    take = take < 0 ? 0 : (take > eq ? eq : take);
    ms->tie_take[0] = take;
    ms->sel_off[0] = sel_before;
    ms->n_union = ms->lgt[0] + take;
  }
  __syncthreads();
  }
  if (p.trace != nullptr && tid == 0 && !(p.debug & 4)) {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[(size_t)blockIdx.x * 8 + 3] = t;
  }
  dbg_stamp(p, 7);

  LOKI_PROBE(ms, 9);
  // ordered emission over the warp's rows, four keys per lane per step
  const long long gt = ms->gt[0];
  const uint32_t Tk = ms->T[0];
  const int take = ms->tie_take[0];
  const bool ties = ms->done[0] == 2 && take > 0;
  const bool partial = ties && take < ms->leq[0];  // only then do tie ranks matter
  int cg_ = 0, ct = 0;
  for (int j0 = r0; j0 < r1; j0 += 128) {
    const int jb = j0 + 4 * lane;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int j = jb + e;
      const uint32_t key = j < r1 ? keys[j] : 0u;
      cg_ += (j < r1 && (long long)key > gt);
      ct += (j < r1 && ties && key == Tk);
    }
  }
  cg_ = __reduce_add_sync(0xffffffffu, cg_);
  ct = __reduce_add_sync(0xffffffffu, ct);
  if (lane == 0) {
    ms->wcnt[0][w] = cg_;
    ms->wcnt[1][w] = ct;
  }
  __syncthreads();
  int pos = 0, tseen = 0;
  for (int ww = 0; ww < w; ++ww) {
    const int tw = ms->wcnt[1][ww];
    int tk = take - tseen;
    tk = tk < 0 ? 0 : (tk > tw ? tw : tk);
    pos += ms->wcnt[0][ww] + tk;
    tseen += tw;
  }
  int32_t* dsti = p.idx_out ? p.idx_out + c.qrow0 * p.idx_stride + ms->sel_off[0] : nullptr;
  for (int j0 = r0; j0 < r1; j0 += 128) {
    const int jb = j0 + 4 * lane;
    bool g1[4], t1[4];
    int nt = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int j = jb + e;
      const uint32_t key = j < r1 ? keys[j] : 0u;
      g1[e] = j < r1 && (long long)key > gt;
      t1[e] = j < r1 && ties && key == Tk;
      nt += t1[e];
    }
    bool sel[4];
    int ns = 0, tin = 0;
    if (partial) {
      // ties before this lane's first key, in row order
      tin = nt;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, tin, off);
        if (lane >= off) tin += t;
      }
      int trank = tseen + tin - nt;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        sel[e] = g1[e] || (t1[e] && trank < take);
        trank += t1[e];
        ns += sel[e];
      }
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        sel[e] = g1[e] || t1[e];
        ns += sel[e];
      }
    }
    int sin = ns;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, sin, off);
      if (lane >= off) sin += t;
    }
    int q = pos + sin - ns;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (sel[e]) {
        const int j = jb + e;
        c.uni[q] = (uint16_t)j;
        c.selmask[j] = 1;  // phase-3 head mask and the weights emission
        if (dsti) dsti[q] = c.s0 + j;
        ++q;
      }
    }
    pos += __shfl_sync(0xffffffffu, sin, 31);
    if (partial) tseen += __shfl_sync(0xffffffffu, tin, 31);
  }
  __syncthreads();
  LOKI_PROBE(ms, 10);
  if ((p.debug & 8) && threadIdx.x == 0 && blockIdx.x == 0) {
    printf("loki select probe (cycles from start): scan1 %lld | p0: sync %lld merge %lld dec %lld | p1: scan %lld sync %lld merge %lld dec %lld | exact %lld emit %lld | cand %d\n",
           ms->probe[1] - ms->probe[0], ms->probe[2] - ms->probe[1], ms->probe[3] - ms->probe[2],
           ms->probe[4] - ms->probe[3], ms->probe[5] - ms->probe[4], ms->probe[6] - ms->probe[5],
           ms->probe[7] - ms->probe[6], ms->probe[8] - ms->probe[7], ms->probe[9] - ms->probe[8],
           ms->probe[10] - ms->probe[9], ms->ncand[1]);
  }
}

// Phase 2: cluster-wide MSB radix select of each head's k_b largest keys
// (linalg.py:95-118: everything above the threshold, threshold ties
// lowest-index-first), then the ordered emission of selmask bits and the
// ascending idx_out; also the external-index and select-all selections.
// Every CTA of the cluster sees the same merged histograms, so all decisions
// (and the number of cluster barriers) agree.
template <int NT, int G_T>
__device__ void select_phase(const FusedParams& p, const Ctx& c, cg::cluster_group& cluster) {
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = lane_id(), w = warp_id();
  MiscState* ms = c.ms;
  const int G = c.G, Lmax = c.Lmax, n_local = c.n_local;
  uint32_t* keys = c.keys;
  if (G_T == 1 && c.need_keys) {
    select_single<NT>(p, c, cluster);
  } else if (c.need_keys) {
    for (int pass = 0; pass < 4; ++pass) {
      const int shift = 24 - 8 * pass;
      const uint32_t* hcur = c.hist + (pass & 1) * G_T * kRadixBins;
      if (pass > 0) {
        uint32_t* hnew = c.hist + (pass & 1) * G_T * kRadixBins;
        const uint32_t hi_mask = 0xFFFFFFFFu << (shift + 8);
        for (int g = 0; g < G; ++g) {
          if (ms->done[g]) continue;
          const uint32_t pre = ms->prefix[g];
          for (int j = tid; j < n_local; j += NT) {
            const uint32_t key = keys[g * Lmax + j];
            if ((key & hi_mask) == pre) atomicAdd(&hnew[g * kRadixBins + ((key >> shift) & 0xFFu)], 1u);
          }
        }
      }
      cluster.sync();
      for (int i = tid; i < G * kRadixBins; i += NT) {
        uint32_t s = 0;
        for (int r = 0; r < c.C; ++r) s += cluster.map_shared_rank(const_cast<uint32_t*>(hcur), r)[i];
        c.ghist[i] = s;
      }
      __syncthreads();
      for (int g = w; g < G; g += NW) {  // one warp per query head
        if (ms->done[g]) continue;
        const int krem = ms->krem[g];
        uint32_t cnt[8];
        uint32_t lsum = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {  // lane 0 holds the top bins 255..248
          cnt[i] = c.ghist[g * kRadixBins + 255 - (lane * 8 + i)];
          lsum += cnt[i];
        }
        uint32_t incl = lsum;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const uint32_t t = __shfl_up_sync(0xffffffffu, incl, off);
          if (lane >= off) incl += t;
        }
        const uint32_t excl = incl - lsum;
        const bool here = (excl < (uint32_t)krem) && ((uint32_t)krem <= incl);
        const unsigned who = __ballot_sync(0xffffffffu, here);
        if (here && lane == __ffs(who) - 1) {
          uint32_t above = excl;
          int i = 0;
          for (; i < 8; ++i) {
            if (above + cnt[i] >= (uint32_t)krem) break;
            above += cnt[i];
          }
          const uint32_t bin = 255u - (uint32_t)(lane * 8 + i);
          const int rem = krem - (int)above;
          const uint32_t pre = ms->prefix[g] | (bin << shift);
          ms->prefix[g] = pre;
          ms->krem[g] = rem;
          if ((int)cnt[i] == rem) {  // the whole boundary bin is in: no tie to break
            ms->done[g] = 1;
            ms->gt[g] = (long long)pre - 1;
            ms->T[g] = 0u;
            ms->krem[g] = 0;
          } else if (pass == 3) {
            ms->done[g] = 2;  // exact threshold key with ties to fill
            ms->gt[g] = (long long)pre;
            ms->T[g] = pre;
          }
        }
      }
      __syncthreads();
      bool all_done = true;
      for (int g = 0; g < G; ++g) all_done &= (ms->done[g] != 0);
      if (all_done) break;
      if (pass < 3) {
        uint32_t* hnext = c.hist + ((pass + 1) & 1) * G_T * kRadixBins;
        for (int i = tid; i < G_T * kRadixBins; i += NT) hnext[i] = 0u;
        __syncthreads();
      }
    }

    if (p.trace != nullptr && tid == 0) {
      long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      p.trace[(size_t)blockIdx.x * 8 + 2] = t;
    }
    if (tid < kMaxG) {
      ms->cnt_gt[tid] = 0;
      ms->cnt_eq[tid] = 0;
    }
    __syncthreads();
    for (int g = 0; g < G; ++g) {
      const long long gt = ms->gt[g];
      const uint32_t Tk = ms->T[g];
      const bool ties = ms->done[g] == 2;
      int cgt = 0, ce = 0;
      for (int j = tid; j < n_local; j += NT) {
        const uint32_t key = keys[g * Lmax + j];
        cgt += ((long long)key > gt);
        ce += (ties && key == Tk);
      }
      cgt = __reduce_add_sync(0xffffffffu, cgt);
      ce = __reduce_add_sync(0xffffffffu, ce);
      if (lane == 0) {
        atomicAdd(&ms->cnt_gt[g], cgt);
        atomicAdd(&ms->cnt_eq[g], ce);
      }
    }
    cluster.sync();  // every CTA's counts visible
    if (tid < G) {
      const int g = tid;
      const int need = ms->krem[g];
      int eq_before = 0, sel_before = 0;
      for (int r = 0; r < c.rank; ++r) {
        MiscState* rs = cluster.map_shared_rank(ms, r);
        const int eq = rs->cnt_eq[g];
        int take = need - eq_before;
        take = take < 0 ? 0 : (take > eq ? eq : take);
        sel_before += rs->cnt_gt[g] + take;
        eq_before += eq;
      }
      int take = need - eq_before;
      const int eq = ms->cnt_eq[g];
      take = take < 0 ? 0 : (take > eq ? eq : take);
      ms->tie_take[g] = take;
      ms->sel_off[g] = sel_before;
    }
    __syncthreads();
    if (p.trace != nullptr && tid == 0) {
      long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      p.trace[(size_t)blockIdx.x * 8 + 3] = t;
    }

    const bool ordered = (p.idx_out != nullptr);
    for (int g = 0; g < G; ++g) {
      const long long gt = ms->gt[g];
      const uint32_t Tk = ms->T[g];
      const int take = ms->tie_take[g];
      const bool ties = ms->done[g] == 2;
      const bool partial_ties = ties && take > 0 && take < ms->cnt_eq[g];
      const bool all_ties = ties && take > 0 && take == ms->cnt_eq[g];
      int32_t* dst = p.idx_out ? p.idx_out + (c.qrow0 + g) * p.idx_stride + ms->sel_off[g] : nullptr;
      if (!ordered && !partial_ties) {
        for (int j = tid; j < n_local; j += NT) {
          const uint32_t key = keys[g * Lmax + j];
          if ((long long)key > gt || (all_ties && key == Tk)) c.selmask[j] |= (uint8_t)(1u << g);
        }
        __syncthreads();
        continue;
      }
      int ties_seen = 0, emitted = 0, buf = 0;
      for (int j0 = 0; j0 < n_local; j0 += NT) {
        const int j = j0 + tid;
        const uint32_t key = j < n_local ? keys[g * Lmax + j] : 0u;
        bool sel = (j < n_local) && ((long long)key > gt);
        if (ties) {
          const bool is_tie = (j < n_local) && key == Tk;
          if (partial_ties) {
            int tot;
            const int rk = block_scan_pred<NT>(is_tie, &tot, ms->scan_a[buf]);
            sel |= is_tie && (ties_seen + rk < take);
            ties_seen += tot;
          } else {
            sel |= is_tie && all_ties;
          }
        }
        int tot;
        const int pos = block_scan_pred<NT>(sel, &tot, ms->scan_b[buf]);
        if (sel) {
          c.selmask[j] |= (uint8_t)(1u << g);
          if (dst) dst[emitted + pos] = c.s0 + j;
        }
        emitted += tot;
        buf ^= 1;
      }
      __syncthreads();
    }
  } else if (p.select_mode == 2 && !c.select_all) {
    if (tid < G) {  // locate this slice inside each head's ascending index list
      const int32_t* lst = p.ext_idx + (c.qrow0 + tid) * p.idx_stride;
      int lo = 0, hi = c.kb;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (lst[mid] < c.s0) lo = mid + 1; else hi = mid;
      }
      const int p0 = lo;
      hi = c.kb;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (lst[mid] < c.s1) lo = mid + 1; else hi = mid;
      }
      ms->ext_p0[tid] = p0;
      ms->ext_p1[tid] = lo;
      ms->sel_off[tid] = p0;
    }
    __syncthreads();
    for (int g = 0; g < G; ++g) {
      const int32_t* lst = p.ext_idx + (c.qrow0 + g) * p.idx_stride;
      for (int j = ms->ext_p0[g] + tid; j < ms->ext_p1[g]; j += NT) {
        c.selmask[lst[j] - c.s0] |= (uint8_t)(1u << g);
        if (p.idx_out) p.idx_out[(c.qrow0 + g) * p.idx_stride + j] = lst[j];
      }
      __syncthreads();
    }
  } else if (c.select_all) {
    if (p.idx_out != nullptr)
      for (int g = 0; g < G; ++g) {
        int32_t* dst = p.idx_out + (c.qrow0 + g) * p.idx_stride;
        for (int j = tid; j < n_local; j += NT) dst[c.s0 + j] = c.s0 + j;
      }
    if (tid < G) ms->sel_off[tid] = c.s0;
    __syncthreads();
  }
}

// Union of the group's selections, ascending (identity when selecting all).
template <int NT>
__device__ __forceinline__ int build_union(const Ctx& c) {
  if (c.select_all) return c.n_local;
  if (c.G == 1 && c.need_keys) return c.ms->n_union;  // emitted directly by select_single
  int emitted = 0, buf = 0;
  for (int j0 = 0; j0 < c.n_local; j0 += NT) {
    const int j = j0 + threadIdx.x;
    const bool sel = (j < c.n_local) && c.selmask[j] != 0;
    int tot;
    const int pos = block_scan_pred<NT>(sel, &tot, c.ms->scan_a[buf]);
    if (sel) c.uni[emitted + pos] = (uint16_t)j;
    emitted += tot;
    buf ^= 1;
  }
  __syncthreads();
  return emitted;
}

// Merge per-lane online-softmax states (lanes that share columns, warps,
// then cluster ranks, always in fixed order), write the output rows, and
// emit the softmax weights of the selection when requested.
// Lane layout: row slot r = lane / LPR, column group sl = lane % LPR; lane
// owns columns (sl + c * LPR) * VEC + v.
template <int NT, int G_T, int NCH, int VEC>
__device__ void merge_and_write(const FusedParams& p, const Ctx& c, cg::cluster_group& cluster,
                                float (&m)[G_T], float (&l)[G_T], float (&acc)[G_T][NCH][VEC], int LPR,
                                int nch, bool want_logits) {
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = lane_id(), w = warp_id();
  const int r = lane / LPR, sl = lane % LPR;
  const int G = c.G, D = c.D;
#pragma unroll
  for (int g = 0; g < G_T; ++g) {
    for (int off = LPR; off < 32; off <<= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, m[g], off);
      const float l2 = __shfl_xor_sync(0xffffffffu, l[g], off);
      float s1, s2;
      merge_state(m[g], l[g], m2, l2, s1, s2);
#pragma unroll
      for (int cc = 0; cc < NCH; ++cc)
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
          const float a2 = __shfl_xor_sync(0xffffffffu, acc[g][cc][v], off);
          acc[g][cc][v] = acc[g][cc][v] * s1 + a2 * s2;
        }
    }
  }
  const int ldp = D + 2;
  if (r == 0) {
#pragma unroll
    for (int g = 0; g < G_T; ++g) {
      if (g >= G) break;
      float* dst = c.part + ((size_t)w * G_T + g) * ldp;
#pragma unroll
      for (int cc = 0; cc < NCH; ++cc)
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
          const int col = (sl + cc * LPR) * VEC + v;
          if (cc < nch && col < D) dst[col] = acc[g][cc][v];
        }
      if (sl == 0) {
        dst[D] = m[g];
        dst[D + 1] = l[g];
      }
    }
  }
  __syncthreads();
  for (int i = tid; i < G * D; i += NT) {
    const int g = i / D, col = i % D;
    float mm = -CUDART_INF_F, ll = 0.f, aa = 0.f;
    for (int ww = 0; ww < NW; ++ww) {
      const float* src = c.part + ((size_t)ww * G_T + g) * ldp;
      float s1, s2;
      merge_state(mm, ll, src[D], src[D + 1], s1, s2);
      aa = aa * s1 + src[col] * s2;
    }
    c.fin[g * ldp + col] = aa;
    if (col == 0) {
      c.fin[g * ldp + D] = mm;
      c.fin[g * ldp + D + 1] = ll;
    }
  }
  if (c.C > 1) cluster.sync();
  else __syncthreads();
  if (tid < G) {  // every rank derives the global (M, L) in the same order
    float mm = -CUDART_INF_F, ll = 0.f;
    for (int rr = 0; rr < c.C; ++rr) {
      const float* f = cluster.map_shared_rank(c.fin, rr) + tid * ldp;
      float s1, s2;
      merge_state(mm, ll, f[D], f[D + 1], s1, s2);
    }
    c.ms->gm[tid] = mm;
    c.ms->gl[tid] = ll;
  }
  if (c.rank == 0) {
    for (int i = tid; i < G * D; i += NT) {
      const int g = i / D, col = i % D;
      float mm = -CUDART_INF_F, ll = 0.f, aa = 0.f;
      for (int rr = 0; rr < c.C; ++rr) {
        const float* f = cluster.map_shared_rank(c.fin, rr) + g * ldp;
        float s1, s2;
        merge_state(mm, ll, f[D], f[D + 1], s1, s2);
        aa = aa * s1 + f[col] * s2;
      }
      p.out[(c.qrow0 + g) * D + col] = ll > 0.f ? aa / ll : 0.f;
    }
  }
  if (c.C > 1) cluster.sync();
  else __syncthreads();

  if (want_logits) {  // softmax weights of the selection, ascending index order
    for (int g = 0; g < G; ++g) {
      const float M = c.ms->gm[g];
      const float invL = 1.f / c.ms->gl[g];
      float* dst = p.weights_out + (c.qrow0 + g) * p.idx_stride + c.ms->sel_off[g];
      int emitted = 0, buf = 0;
      for (int j0 = 0; j0 < c.n_local; j0 += NT) {
        const int j = j0 + tid;
        const bool sel = (j < c.n_local) && (c.select_all || (c.selmask[j] >> g) & 1u);
        int tot;
        const int pos = block_scan_pred<NT>(sel, &tot, c.ms->scan_a[buf]);
        if (sel) dst[emitted + pos] = exp2f(__uint_as_float(c.keys[g * c.Lmax + j]) - M) * invL;
        emitted += tot;
        buf ^= 1;
      }
      __syncthreads();
    }
  }
}

}  // namespace fused
}  // namespace loki
