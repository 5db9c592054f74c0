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
#include "loki_fused.cuh"

namespace loki {

using namespace fused;

namespace {
constexpr int kUnroll = 4;
}

// LDG variant: any dtype / head dim / stride layout the TMA variant cannot
// address (loki_decode_tma.cu is the fast path).
template <typename T, int G_T, int VEC, int NCH, int NT>
__global__ void __launch_bounds__(NT) fused_decode_kernel(const FusedParams p) {
  constexpr int NW = NT / 32;
  extern __shared__ __align__(16) uint8_t smem[];
  cg::cluster_group cluster = cg::this_cluster();
  Ctx c;
  if (!make_ctx<G_T>(p, smem, (int)cluster.block_rank(), c)) return;
  const int G = c.G, D = c.D, Lmax = c.Lmax;
  const int lane = lane_id(), w = warp_id();
  const int s0 = c.s0, s1 = c.s1;
  const T* Kb = reinterpret_cast<const T*>(p.K) + (size_t)c.b * p.sb + (size_t)c.hk * p.sh;
  const T* Vb = reinterpret_cast<const T*>(p.V) + (size_t)c.b * p.sb + (size_t)c.hk * p.sh;
  init_state<NT, G_T>(c);
  __syncthreads();

  // ------------------------------------------------------------ phase 1
  const bool need_scores = c.need_keys || (p.approx_out != nullptr);
  if (need_scores) {
    if (p.ext_scores != nullptr) {
      keys_from_scores<NT>(p, c);
    } else {
      const int d = p.d;
      const int nch1 = ceil_div(d, VEC);                 // VEC-element chunks holding columns < d
      const int LPR1 = NCH == 1 ? next_pow2(nch1) : 32;  // lanes per row
      const int RPW1 = 32 / LPR1;
      const int r = lane / LPR1, sl = lane % LPR1;
      float q1[G_T][NCH][VEC];
#pragma unroll
      for (int g = 0; g < G_T; ++g)
#pragma unroll
        for (int cc = 0; cc < NCH; ++cc)
#pragma unroll
          for (int v = 0; v < VEC; ++v) {
            const int col = (sl + cc * LPR1) * VEC + v;
            q1[g][cc][v] = (g < G && col < d) ? p.q_hat[(c.qrow0 + g) * D + col] : 0.f;
          }
      const int step = NW * kUnroll * RPW1;
      for (int row0 = s0 + w * kUnroll * RPW1; row0 < s1; row0 += step) {
        Chunk<T, VEC> ch[kUnroll][NCH];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const int row = row0 + u * RPW1 + r;
#pragma unroll
          for (int cc = 0; cc < NCH; ++cc) {
            const int ci = sl + cc * LPR1;
            if (row < s1 && ci < nch1) ch[u][cc].load(Kb + (size_t)row * p.ss + ci * VEC);
            else ch[u][cc].zero();
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
            for (int cc = 0; cc < NCH; ++cc)
#pragma unroll
              for (int v = 0; v < VEC; ++v) {
                const int col = (sl + cc * LPR1) * VEC + v;
                const float x = ch[u][cc].get(v);
                acc = fmaf(q1[g][cc][v], col < d ? x : 0.f, acc);
              }
            acc = warp_sum_width(acc, LPR1);
            if (g < G) {
              const uint32_t key = order_key(acc);
              if (writer) {
                c.keys[g * Lmax + (row - s0)] = key;
                if (p.approx_out) p.approx_out[(c.qrow0 + g) * (size_t)p.S_cap + row] = acc;
              }
              if (c.need_keys) hist_add(c.hist + g * kRadixBins, writer, key >> 24);
            }
          }
        }
      }
    }
  }
  __syncthreads();

  // ------------------------------------------------------------ phase 2
  select_phase<NT, G_T>(p, c, cluster);
  if (p.out == nullptr) {
    if (c.C > 1) cluster.sync();  // keep shared memory alive for remote readers
    return;
  }
  const int n_rows = build_union<NT>(c);

  // ------------------------------------------------------------ phase 3
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
    for (int cc = 0; cc < NCH; ++cc)
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        const int col = (sl + cc * LPR3) * VEC + v;
        q3[g][cc][v] = (g < G && col < D && cc < nch3) ? p.q_hat[(c.qrow0 + g) * D + col] * p.qscale : 0.f;
        acc[g][cc][v] = 0.f;
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
      const int j = ok ? (c.select_all ? t : (int)c.uni[t]) : 0;
      jrow[u] = j;
      msk[u] = ok ? (c.select_all ? full_mask : c.selmask[j]) : (uint8_t)0;
      const size_t roff = (size_t)(s0 + j) * p.ss;
#pragma unroll
      for (int cc = 0; cc < NCH; ++cc) {
        const int ci = sl + cc * LPR3;
        if (ok && cc < nch3 && ci * VEC < D) {
          kc[u][cc].load(Kb + roff + ci * VEC);
          vc[u][cc].load(Vb + roff + ci * VEC);
        } else {
          kc[u][cc].zero();
          vc[u][cc].zero();
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
#pragma unroll
      for (int g = 0; g < G_T; ++g) {
        float x = 0.f;
#pragma unroll
        for (int cc = 0; cc < NCH; ++cc)
#pragma unroll
          for (int v = 0; v < VEC; ++v) x = fmaf(q3[g][cc][v], kc[u][cc].get(v), x);
        x = warp_sum_width(x, LPR3);
        if (msk[u] & (1u << g)) {
          if (want_logits && sl == 0) c.keys[g * Lmax + jrow[u]] = __float_as_uint(x);
          const float mn = fmaxf(m[g], x);
          const float sc = exp2f(m[g] - mn);  // m = -inf -> 0
          const float pe = exp2f(x - mn);
          l[g] = l[g] * sc + pe;
          m[g] = mn;
#pragma unroll
          for (int cc = 0; cc < NCH; ++cc)
#pragma unroll
            for (int v = 0; v < VEC; ++v) acc[g][cc][v] = fmaf(pe, vc[u][cc].get(v), acc[g][cc][v] * sc);
        }
      }
    }
  }
  merge_and_write<NT, G_T, NCH, VEC>(p, c, cluster, m, l, acc, LPR3, nch3, want_logits);
}

// ---------------------------------------------------------------- host side

size_t fused_layout(int G_T, int NT, int D, int Lmax, bool keys_in_smem, FusedParams* p) {
  const int NW = NT / 32;
  size_t off = 0;
  const size_t keys = keys_in_smem ? (size_t)G_T * Lmax * 4 : 0;
  p->off_keys = (int)off; off = align_up(off + keys, 16);
  p->off_sel = (int)off; off = align_up(off + (size_t)Lmax, 16);
  p->off_union = (int)off; off = align_up(off + align_up((size_t)Lmax, 1024) * 2, 16);
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
  static KernelAttrs attrs;
  cudaError_t e = attrs.ensure(reinterpret_cast<const void*>(kern), smem, p.C > 8);
  if (e != cudaSuccess) return e;
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
