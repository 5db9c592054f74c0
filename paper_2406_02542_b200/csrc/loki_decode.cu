// Fused Loki decode attention for sm_100a.
//
// One thread-block cluster of C CTAs owns one (batch b, KV head) unit and the
// G query heads that share it (G = Hq / Hkv; G = 1 for MHA).  CTA `rank`
// owns the contiguous cache slice [rank*L, rank*L + L) with L = ceil(S_b / C).
// Everything between the query and the output stays on chip:
//
//   phase 1  approx scores   (kernels.py:223-241 sliced_score_kernel)
//            leading-d columns of the rotated K cache, 128-bit streaming loads,
//            fp32 accumulate; scores become order-preserving uint32 keys in
//            shared memory; pass-0 radix histogram built on the fly.
//   phase 2  top-k           (linalg.py:95-118 topk_indices)
//            cluster-wide MSB radix select (4 x 8-bit digits, histograms merged
//            through distributed shared memory), exact tie rule: everything
//            above the threshold, threshold ties lowest-index-first, ascending.
//   phase 3  sparse exact attention (kernels.py:244-279 + linalg.py:76-92)
//            gathers only the selected full rows of K and V (one pass over the
//            union of the G heads' selections), online softmax in fp32, per-CTA
//            partials merged in fixed order: warp -> CTA -> cluster (DSMEM).
//
// select_mode: 0 radix top-k, 1 all rows (dense decode, attention.py:137-142),
// 2 external ascending index lists (gathered attention on a given selection),
// 3 scores only.  Reduction orders are fixed, so results are bit-identical
// run to run for a fixed launch plan.
#include <cooperative_groups.h>
#include <math_constants.h>

#include "loki_common.cuh"
#include "loki_internal.h"

namespace cg = cooperative_groups;

namespace loki {

struct Plan;  // loki_internal.h

namespace {

constexpr int kRadixBins = 256;
constexpr int kMaxG = 8;
constexpr int kUnroll = 4;

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
  int32_t n_union;
  float gm[kMaxG];
  float gl[kMaxG];
};

// Ordered block-wide compaction helper: returns the exclusive prefix of `pred`
// over all threads of the block (in thread order) and the block total.
template <int NT>
__device__ __forceinline__ int block_scan_pred(bool pred, int* total, int32_t* scratch) {
  constexpr int NW = NT / 32;
  const int lane = lane_id(), w = warp_id();
  unsigned bal = __ballot_sync(0xffffffffu, pred);
  int in_warp = __popc(bal & ((1u << lane) - 1u));
  if (lane == 0) scratch[w] = __popc(bal);
  __syncthreads();
  int before = 0, tot = 0;
#pragma unroll
  for (int i = 0; i < NW; ++i) {
    int c = scratch[i];
    before += (i < w) ? c : 0;
    tot += c;
  }
  *total = tot;
  return before + in_warp;
}

// Histogram update with warp-level aggregation of equal bins (the leading
// digit of fp32 score keys concentrates on a few exponent values).
__device__ __forceinline__ void hist_add(uint32_t* hist, bool active, uint32_t bin) {
  unsigned m = __ballot_sync(0xffffffffu, active);
  if (active) {
    unsigned peers = __match_any_sync(m, bin);
    if ((int)(__ffs(peers) - 1) == lane_id()) atomicAdd(&hist[bin], (uint32_t)__popc(peers));
  }
}

__device__ __forceinline__ void merge_state(float& m, float& l, float m2, float l2, float& s1, float& s2) {
  float mn = fmaxf(m, m2);
  s1 = (m == -CUDART_INF_F) ? 0.f : exp2f(m - mn);
  s2 = (m2 == -CUDART_INF_F) ? 0.f : exp2f(m2 - mn);
  l = l * s1 + l2 * s2;
  m = mn;
}

}  // namespace

template <typename T, int G_T, int VEC, int NCH, int NT>
__global__ void __launch_bounds__(NT) fused_decode_kernel(const FusedParams p) {
  constexpr int NW = NT / 32;
  extern __shared__ __align__(16) uint8_t smem[];
  cg::cluster_group cluster = cg::this_cluster();

  const int C = p.C;
  const int rank = (int)cluster.block_rank();
  const int unit = blockIdx.x / C;
  const int b = unit / p.Hkv, hk = unit % p.Hkv;
  const int G = p.G, D = p.D, Lmax = p.Lmax;
  const int tid = threadIdx.x, lane = lane_id(), w = warp_id();

  int S = p.lens[b];
  S = S > p.S_cap ? p.S_cap : S;
  if (S <= 0) return;  // whole cluster leaves together (uniform per unit)

  int kb;
  if (p.select_mode == 1) kb = S;
  else if (p.k_fixed > 0) kb = p.k_fixed < S ? p.k_fixed : S;
  else kb = resolve_fraction(p.k_f, S);

  const int L = ceil_div(S, C);
  const int s0 = rank * L;
  const int s1 = min(s0 + L, S);
  const int n_local = s1 > s0 ? s1 - s0 : 0;

  const bool select_all = (p.select_mode == 1) || ((p.select_mode == 0 || p.select_mode == 2) && kb == S);
  const bool need_keys = (p.select_mode == 0) && !select_all;
  const bool need_scores = need_keys || (p.approx_out != nullptr);

  uint32_t* keys = p.keys_ws ? p.keys_ws + (size_t)blockIdx.x * G_T * Lmax
                             : reinterpret_cast<uint32_t*>(smem + p.off_keys);
  uint8_t* selmask = smem + p.off_sel;
  uint16_t* uni = reinterpret_cast<uint16_t*>(smem + p.off_union);
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem + p.off_hist);  // [2][G_T][256]
  uint32_t* ghist = hist + 2 * G_T * kRadixBins;                     // [G_T][256]
  float* part = reinterpret_cast<float*>(smem + p.off_merge);        // [NW][G_T][D+2]
  float* fin = reinterpret_cast<float*>(smem + p.off_final);         // [G_T][D+2]
  MiscState* ms = reinterpret_cast<MiscState*>(smem + p.off_misc);

  const T* Kb = reinterpret_cast<const T*>(p.K) + (size_t)b * p.sb + (size_t)hk * p.sh;
  const T* Vb = reinterpret_cast<const T*>(p.V) + (size_t)b * p.sb + (size_t)hk * p.sh;
  const size_t qrow0 = (size_t)b * p.Hq + (size_t)hk * G;  // first query head row of the unit

  for (int i = tid; i < G_T * kRadixBins; i += NT) hist[i] = 0u;
  for (int i = tid; i < Lmax; i += NT) selmask[i] = 0;
  if (tid < kMaxG) {
    ms->prefix[tid] = 0u;
    ms->krem[tid] = kb;
    ms->done[tid] = (tid >= G) ? 1 : 0;
  }
  __syncthreads();

  // ------------------------------------------------------------ phase 1
  if (need_scores) {
    if (p.ext_scores != nullptr) {
      for (int g = 0; g < G; ++g) {
        const float* src = p.ext_scores + (qrow0 + g) * (size_t)p.S_cap;
        for (int j0 = 0; j0 < n_local; j0 += NT) {
          const int j = j0 + tid;
          const bool ok = j < n_local;
          float s = ok ? src[s0 + j] : 0.f;
          uint32_t key = order_key(s);
          if (ok) keys[g * Lmax + j] = key;
          if (need_keys) hist_add(hist + g * kRadixBins, ok, key >> 24);
        }
      }
    } else {
      const int d = p.d;
      const int nch1 = ceil_div(d, VEC);                      // 16-byte chunks holding columns < d
      const int LPR1 = NCH == 1 ? next_pow2(nch1) : 32;       // lanes per row
      const int RPW1 = 32 / LPR1;
      const int r = lane / LPR1, sl = lane % LPR1;
      float q1[G_T][NCH][VEC];
#pragma unroll
      for (int g = 0; g < G_T; ++g)
#pragma unroll
        for (int c = 0; c < NCH; ++c)
#pragma unroll
          for (int v = 0; v < VEC; ++v) {
            const int col = (sl + c * LPR1) * VEC + v;
            q1[g][c][v] = (g < G && col < d) ? p.q_hat[(qrow0 + g) * D + col] : 0.f;
          }
      const int step = NW * kUnroll * RPW1;
      for (int row0 = s0 + w * kUnroll * RPW1; row0 < s1; row0 += step) {
        Chunk<T, VEC> ch[kUnroll][NCH];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const int row = row0 + u * RPW1 + r;
#pragma unroll
          for (int c = 0; c < NCH; ++c) {
            const int ci = sl + c * LPR1;
            if (row < s1 && ci < nch1) ch[u][c].load(Kb + (size_t)row * p.ss + ci * VEC);
            else ch[u][c].zero();
          }
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const int row = row0 + u * RPW1 + r;
          const bool writer = (sl == 0) && (row < s1);
#pragma unroll
          for (int g = 0; g < G_T; ++g) {
            float acc = 0.f;
#pragma unroll
            for (int c = 0; c < NCH; ++c)
#pragma unroll
              for (int v = 0; v < VEC; ++v) {
                const int col = (sl + c * LPR1) * VEC + v;
                const float x = ch[u][c].get(v);
                acc = fmaf(q1[g][c][v], col < d ? x : 0.f, acc);
              }
            acc = warp_sum_width(acc, LPR1);
            if (g < G) {
              const uint32_t key = order_key(acc);
              if (writer) {
                keys[g * Lmax + (row - s0)] = key;
                if (p.approx_out) p.approx_out[(qrow0 + g) * (size_t)p.S_cap + row] = acc;
              }
              if (need_keys) hist_add(hist + g * kRadixBins, writer, key >> 24);
            }
          }
        }
      }
    }
  }
  __syncthreads();

  // ------------------------------------------------------------ phase 2
  if (need_keys) {
    // All CTAs of the cluster see identical merged histograms, so every
    // decision below (and therefore the number of cluster barriers) agrees.
    for (int pass = 0; pass < 4; ++pass) {
      const int shift = 24 - 8 * pass;
      const uint32_t* hcur = hist + (pass & 1) * G_T * kRadixBins;
      if (pass > 0) {
        uint32_t* hnew = hist + (pass & 1) * G_T * kRadixBins;
        const uint32_t hi_mask = 0xFFFFFFFFu << (shift + 8);
        for (int g = 0; g < G; ++g) {
          if (ms->done[g]) continue;
          const uint32_t pre = ms->prefix[g];
          for (int j0 = 0; j0 < n_local; j0 += NT) {
            const int j = j0 + tid;
            const uint32_t key = j < n_local ? keys[g * Lmax + j] : 0u;
            const bool ok = (j < n_local) && ((key & hi_mask) == pre);
            if (ok) atomicAdd(&hnew[g * kRadixBins + ((key >> shift) & 0xFFu)], 1u);
          }
        }
      }
      cluster.sync();
      for (int i = tid; i < G * kRadixBins; i += NT) {
        uint32_t s = 0;
        for (int c = 0; c < C; ++c) s += cluster.map_shared_rank(const_cast<uint32_t*>(hcur), c)[i];
        ghist[i] = s;
      }
      __syncthreads();
      // one warp per query head finds the bin holding the k-th largest key
      for (int g = w; g < G; g += NW) {
        if (ms->done[g]) continue;
        const int krem = ms->krem[g];
        uint32_t cnt[8];
        uint32_t lsum = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {  // lane 0 holds the top bins 255..248
          cnt[i] = ghist[g * kRadixBins + 255 - (lane * 8 + i)];
          lsum += cnt[i];
        }
        uint32_t incl = lsum;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          uint32_t t = __shfl_up_sync(0xffffffffu, incl, off);
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
        uint32_t* hnext = hist + ((pass + 1) & 1) * G_T * kRadixBins;
        for (int i = tid; i < G_T * kRadixBins; i += NT) hnext[i] = 0u;
        __syncthreads();
      }
    }

    // local counts above the threshold / at the threshold
    if (tid < kMaxG) { ms->cnt_gt[tid] = 0; ms->cnt_eq[tid] = 0; }
    __syncthreads();
    for (int g = 0; g < G; ++g) {
      const long long gt = ms->gt[g];
      const uint32_t Tk = ms->T[g];
      const bool ties = ms->done[g] == 2;
      int cg_ = 0, ce = 0;
      for (int j = tid; j < n_local; j += NT) {
        const uint32_t key = keys[g * Lmax + j];
        cg_ += ((long long)key > gt);
        ce += (ties && key == Tk);
      }
      cg_ = __reduce_add_sync(0xffffffffu, cg_);
      ce = __reduce_add_sync(0xffffffffu, ce);
      if (lane == 0) {
        atomicAdd(&ms->cnt_gt[g], cg_);
        atomicAdd(&ms->cnt_eq[g], ce);
      }
    }
    cluster.sync();  // counts of every CTA visible
    if (tid < G) {
      const int g = tid;
      const int need = ms->krem[g];
      int eq_before = 0, sel_before = 0;
      for (int c = 0; c < rank; ++c) {
        MiscState* rs = cluster.map_shared_rank(ms, c);
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

    // ordered emission of each head's selection: selmask bit + ascending idx_out
    const bool ordered = (p.idx_out != nullptr);
    for (int g = 0; g < G; ++g) {
      const long long gt = ms->gt[g];
      const uint32_t Tk = ms->T[g];
      const int take = ms->tie_take[g];
      const bool ties = ms->done[g] == 2;
      const bool partial_ties = ties && take > 0 && take < ms->cnt_eq[g];
      const bool all_ties = ties && take > 0 && take == ms->cnt_eq[g];
      const int off = ms->sel_off[g];
      int32_t* dst = p.idx_out ? p.idx_out + (qrow0 + g) * p.idx_stride + off : nullptr;
      if (!ordered && !partial_ties) {
        for (int j = tid; j < n_local; j += NT) {
          const uint32_t key = keys[g * Lmax + j];
          if ((long long)key > gt || (all_ties && key == Tk)) selmask[j] |= (uint8_t)(1u << g);
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
          selmask[j] |= (uint8_t)(1u << g);
          if (dst) dst[emitted + pos] = s0 + j;
        }
        emitted += tot;
        buf ^= 1;
      }
      __syncthreads();
    }
  } else if (p.select_mode == 2 && !select_all) {
    if (tid < G) {  // locate this slice inside each head's ascending index list
      const int32_t* lst = p.ext_idx + (qrow0 + tid) * p.idx_stride;
      int lo = 0, hi = kb;
      while (lo < hi) { int mid = (lo + hi) >> 1; if (lst[mid] < s0) lo = mid + 1; else hi = mid; }
      const int p0 = lo;
      hi = kb;
      while (lo < hi) { int mid = (lo + hi) >> 1; if (lst[mid] < s1) lo = mid + 1; else hi = mid; }
      ms->ext_p0[tid] = p0;
      ms->ext_p1[tid] = lo;
      ms->sel_off[tid] = p0;
    }
    __syncthreads();
    for (int g = 0; g < G; ++g) {
      const int32_t* lst = p.ext_idx + (qrow0 + g) * p.idx_stride;
      for (int j = ms->ext_p0[g] + tid; j < ms->ext_p1[g]; j += NT) {
        const int row = lst[j] - s0;
        selmask[row] |= (uint8_t)(1u << g);
        if (p.idx_out) p.idx_out[(qrow0 + g) * p.idx_stride + j] = lst[j];
      }
      __syncthreads();
    }
  } else if (select_all && p.idx_out != nullptr) {
    for (int g = 0; g < G; ++g) {
      int32_t* dst = p.idx_out + (qrow0 + g) * p.idx_stride;
      for (int j = tid; j < n_local; j += NT) dst[s0 + j] = s0 + j;
    }
    if (tid < G) ms->sel_off[tid] = s0;
  } else if (select_all) {
    if (tid < G) ms->sel_off[tid] = s0;
  }

  if (p.out == nullptr) {
    if (C > 1) cluster.sync();  // keep smem alive for remote readers above
    return;
  }

  // union of the group's selections, ascending (identity when selecting all)
  int n_rows = n_local;
  if (!select_all) {
    int emitted = 0, buf = 0;
    for (int j0 = 0; j0 < n_local; j0 += NT) {
      const int j = j0 + tid;
      const bool sel = (j < n_local) && selmask[j] != 0;
      int tot;
      const int pos = block_scan_pred<NT>(sel, &tot, ms->scan_a[buf]);
      if (sel) uni[emitted + pos] = (uint16_t)j;
      emitted += tot;
      buf ^= 1;
    }
    n_rows = emitted;
    __syncthreads();
  }

  // ------------------------------------------------------------ phase 3
  {
    const int nch3 = NCH == 1 ? 1 : ceil_div(D, 32);
    const int LPR3 = NCH == 1 ? next_pow2(D / VEC) : 32;
    const int RPW3 = 32 / LPR3;
    const int r = lane / LPR3, sl = lane % LPR3;
    const uint8_t full_mask = (uint8_t)((1u << G) - 1u);
    const bool want_logits = p.weights_out != nullptr;

    float q3[G_T][NCH][VEC];
    float acc[G_T][NCH][VEC];
    float m[G_T], l[G_T];
#pragma unroll
    for (int g = 0; g < G_T; ++g) {
      m[g] = -CUDART_INF_F;
      l[g] = 0.f;
#pragma unroll
      for (int c = 0; c < NCH; ++c)
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
          const int col = (sl + c * LPR3) * VEC + v;
          q3[g][c][v] = (g < G && col < D && c < nch3) ? p.q_hat[(qrow0 + g) * D + col] * p.qscale : 0.f;
          acc[g][c][v] = 0.f;
        }
    }

    const int step = NW * kUnroll * RPW3;
    for (int base = w * kUnroll * RPW3; base < n_rows; base += step) {
      Chunk<T, VEC> kc[kUnroll][NCH];
      Chunk<T, VEC> vc[kUnroll][NCH];
      int jrow[kUnroll];
      uint8_t msk[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int t = base + u * RPW3 + r;
        const bool ok = t < n_rows;
        const int j = ok ? (select_all ? t : (int)uni[t]) : 0;
        jrow[u] = j;
        msk[u] = ok ? (select_all ? full_mask : selmask[j]) : (uint8_t)0;
        const size_t roff = (size_t)(s0 + j) * p.ss;
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          const int ci = sl + c * LPR3;
          if (ok && c < nch3 && ci * VEC < D) {
            kc[u][c].load(Kb + roff + ci * VEC);
            vc[u][c].load(Vb + roff + ci * VEC);
          } else {
            kc[u][c].zero();
            vc[u][c].zero();
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
#pragma unroll
        for (int g = 0; g < G_T; ++g) {
          float x = 0.f;
#pragma unroll
          for (int c = 0; c < NCH; ++c)
#pragma unroll
            for (int v = 0; v < VEC; ++v) x = fmaf(q3[g][c][v], kc[u][c].get(v), x);
          x = warp_sum_width(x, LPR3);
          if (msk[u] & (1u << g)) {
            if (want_logits && sl == 0) keys[g * Lmax + jrow[u]] = __float_as_uint(x);
            const float mn = fmaxf(m[g], x);
            const float sc = exp2f(m[g] - mn);  // m = -inf -> 0
            const float pe = exp2f(x - mn);
            l[g] = l[g] * sc + pe;
            m[g] = mn;
#pragma unroll
            for (int c = 0; c < NCH; ++c)
#pragma unroll
              for (int v = 0; v < VEC; ++v) acc[g][c][v] = fmaf(pe, vc[u][c].get(v), acc[g][c][v] * sc);
          }
        }
      }
    }

    // merge the row slots of the warp (lanes differing only in slot bits)
#pragma unroll
    for (int g = 0; g < G_T; ++g) {
      for (int off = LPR3; off < 32; off <<= 1) {
        const float m2 = __shfl_xor_sync(0xffffffffu, m[g], off);
        const float l2 = __shfl_xor_sync(0xffffffffu, l[g], off);
        float s1, s2;
        merge_state(m[g], l[g], m2, l2, s1, s2);
#pragma unroll
        for (int c = 0; c < NCH; ++c)
#pragma unroll
          for (int v = 0; v < VEC; ++v) {
            const float a2 = __shfl_xor_sync(0xffffffffu, acc[g][c][v], off);
            acc[g][c][v] = acc[g][c][v] * s1 + a2 * s2;
          }
      }
    }
    const int ldp = D + 2;
    if (r == 0) {
#pragma unroll
      for (int g = 0; g < G_T; ++g) {
        if (g >= G) break;
        float* dst = part + ((size_t)w * G_T + g) * ldp;
#pragma unroll
        for (int c = 0; c < NCH; ++c)
#pragma unroll
          for (int v = 0; v < VEC; ++v) {
            const int col = (sl + c * LPR3) * VEC + v;
            if (c < nch3 && col < D) dst[col] = acc[g][c][v];
          }
        if (sl == 0) { dst[D] = m[g]; dst[D + 1] = l[g]; }
      }
    }
    __syncthreads();
    // CTA merge over warps in fixed order
    for (int i = tid; i < G * D; i += NT) {
      const int g = i / D, col = i % D;
      float mm = -CUDART_INF_F, ll = 0.f, aa = 0.f;
      for (int ww = 0; ww < NW; ++ww) {
        const float* src = part + ((size_t)ww * G_T + g) * ldp;
        float s1, s2;
        merge_state(mm, ll, src[D], src[D + 1], s1, s2);
        aa = aa * s1 + src[col] * s2;
      }
      fin[g * ldp + col] = aa;
      if (col == 0) { fin[g * ldp + D] = mm; fin[g * ldp + D + 1] = ll; }
    }
    if (C > 1) cluster.sync();
    else __syncthreads();

    // cluster merge in rank order; every rank derives the global (M, L)
    if (tid < G) {
      float mm = -CUDART_INF_F, ll = 0.f;
      for (int c = 0; c < C; ++c) {
        const float* f = cluster.map_shared_rank(fin, c) + tid * ldp;
        float s1, s2;
        merge_state(mm, ll, f[D], f[D + 1], s1, s2);
      }
      ms->gm[tid] = mm;
      ms->gl[tid] = ll;
    }
    if (rank == 0) {
      for (int i = tid; i < G * D; i += NT) {
        const int g = i / D, col = i % D;
        float mm = -CUDART_INF_F, ll = 0.f, aa = 0.f;
        for (int c = 0; c < C; ++c) {
          const float* f = cluster.map_shared_rank(fin, c) + g * ldp;
          float s1, s2;
          merge_state(mm, ll, f[D], f[D + 1], s1, s2);
          aa = aa * s1 + f[col] * s2;
        }
        p.out[(qrow0 + g) * D + col] = ll > 0.f ? aa / ll : 0.f;
      }
    }
    if (C > 1) cluster.sync();
    else __syncthreads();

    // softmax weights of the selection, in ascending index order
    if (want_logits) {
      for (int g = 0; g < G; ++g) {
        const float M = ms->gm[g];
        const float invL = 1.f / ms->gl[g];
        float* dst = p.weights_out + (qrow0 + g) * p.idx_stride + ms->sel_off[g];
        int emitted = 0, buf = 0;
        for (int j0 = 0; j0 < n_local; j0 += NT) {
          const int j = j0 + tid;
          const bool sel = (j < n_local) && (select_all || (selmask[j] >> g) & 1u);
          int tot;
          const int pos = block_scan_pred<NT>(sel, &tot, ms->scan_a[buf]);
          if (sel) dst[emitted + pos] = exp2f(__uint_as_float(keys[g * Lmax + j]) - M) * invL;
          emitted += tot;
          buf ^= 1;
        }
        __syncthreads();
      }
    }
  }
}

// ---------------------------------------------------------------- host side

size_t fused_layout(int G_T, int NT, int D, int Lmax, bool keys_in_smem, FusedParams* p) {
  const int NW = NT / 32;
  size_t off = 0;
  const size_t keys = keys_in_smem ? (size_t)G_T * Lmax * 4 : 0;
  p->off_keys = (int)off; off = align_up(off + keys, 16);
  p->off_sel = (int)off; off = align_up(off + (size_t)Lmax, 16);
  p->off_union = (int)off; off = align_up(off + (size_t)Lmax * 2, 16);
  p->off_hist = (int)off; off = align_up(off + (size_t)3 * G_T * kRadixBins * 4, 16);
  p->off_merge = (int)off; off = align_up(off + (size_t)NW * G_T * (D + 2) * 4, 16);
  p->off_final = (int)off; off = align_up(off + (size_t)G_T * (D + 2) * 4, 16);
  p->off_misc = (int)off; off = align_up(off + sizeof(MiscState), 16);
  return off;
}

template <typename T, int G_T, int VEC, int NCH, int NT>
static cudaError_t launch_t(const FusedParams& p, int units, size_t smem, cudaStream_t st) {
  auto kern = fused_decode_kernel<T, G_T, VEC, NCH, NT>;
  // attributes are process-wide per kernel: set them once (also keeps them out
  // of CUDA-graph capture on the steady-state path)
  static size_t smem_set = 0;
  static bool nonportable_set = false;
  cudaError_t e;
  if (smem > smem_set) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    smem_set = smem;
  }
  if (p.C > 8 && !nonportable_set) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    nonportable_set = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(units * p.C));
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)p.C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, p);
}

template <typename T, int VEC>
static cudaError_t dispatch_g(const FusedParams& p, int G_T, bool fast, int units, size_t smem, cudaStream_t st) {
  constexpr int NT = 256;
  if (fast) {
    switch (G_T) {
      case 1: return launch_t<T, 1, VEC, 1, NT>(p, units, smem, st);
      case 2: return launch_t<T, 2, VEC, 1, NT>(p, units, smem, st);
      case 4: return launch_t<T, 4, VEC, 1, NT>(p, units, smem, st);
      default: break;
    }
  } else {
    switch (G_T) {
      case 1: return launch_t<T, 1, 1, 8, NT>(p, units, smem, st);
      case 2: return launch_t<T, 2, 1, 8, NT>(p, units, smem, st);
      case 4: return launch_t<T, 4, 1, 8, NT>(p, units, smem, st);
      case 8: return launch_t<T, 8, 1, 8, NT>(p, units, smem, st);
      default: break;
    }
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_fused(const FusedParams& p, const Plan& plan, cudaStream_t st) {
  const int units = p.B * p.Hkv;
  if (plan.dtype == LOKI_DTYPE_BF16) {
    if (plan.fast && plan.G_T == 8) return launch_t<__nv_bfloat16, 8, 4, 1, 256>(p, units, plan.smem, st);
    return plan.fast ? dispatch_g<__nv_bfloat16, 8>(p, plan.G_T, true, units, plan.smem, st)
                     : dispatch_g<__nv_bfloat16, 1>(p, plan.G_T, false, units, plan.smem, st);
  }
  if (plan.fast && plan.G_T == 8) return launch_t<float, 8, 4, 1, 256>(p, units, plan.smem, st);
  return plan.fast ? dispatch_g<float, 4>(p, plan.G_T, true, units, plan.smem, st)
                   : dispatch_g<float, 1>(p, plan.G_T, false, units, plan.smem, st);
}

}  // namespace loki
