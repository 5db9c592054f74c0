// Fused Loki decode attention, TMA variant (the hot path on sm_100a).
//
// Same three phases and cluster decomposition as loki_decode.cu, but every
// byte of the KV cache moves through the Tensor Memory Accelerator into a
// shared-memory ring of `nst` stages guarded by mbarriers, so the bytes in
// flight are decoupled from registers:
//
//   phase 1  one 4-D box per stage: r1 rows x dbox leading columns of the
//            rotated K cache, L2 promotion 64 B -- exactly the d*S*e
//            algorithmic bytes (LDG of 64 of every 256 B drags in the whole
//            128 B line: tools/l2probe.cu, profiles/r01_l2probe.txt);
//   phase 3  tile::gather4 of the selected rows: r3 rows of K and r3 rows of V
//            per stage, rows addressed through a 2-D [B*Hkv*S_cap, D] view.
//
// Stage recycling: all warps consume a stage, __syncthreads, then one thread
// re-arms its mbarrier and issues the next transfer into it.  Launched with
// programmatic stream serialization: the prologue overlaps the K0 append
// kernel and griddepcontrol.wait orders the reads after it.
#include <cuda.h>
#include <cstdio>

#include "loki_fused.cuh"
#include "loki_tma.cuh"

namespace loki {

using namespace fused;

namespace {

using namespace tma;

// Phase-1 stage consumed by ONE warp: r1 rows x dbox leading columns, LPR1
// lanes per row; per-row score -> order key (+ approx diagnostics, pass-0 histogram).
template <typename T, int G_T, int VEC, int LPR1>
__device__ __forceinline__ void consume_lead(const FusedParams& p, const Ctx& c, const uint8_t* tile, int i0,
                                             int rows_here, const float (&q1)[G_T][VEC], int lane) {
  constexpr int E = sizeof(T);
  constexpr int RPW1 = 32 / LPR1;
  constexpr int U = 4;  // independent rows in flight per lane
  const int row_bytes = p.dbox * E;
  const int nch1 = p.dbox / VEC;
  const int r = lane / LPR1, sl = lane % LPR1;
  const bool lane_on = sl < nch1;
  const int passes = p.r1 / RPW1;  // host: r1 % (U * RPW1) == 0
  for (int ps = 0; ps < passes; ps += U) {
    float x[U][VEC];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int rr = (ps + u) * RPW1 + r;
      if (lane_on) lds_chunk<T, VEC>(tile + rr * row_bytes + sl * VEC * E, x[u]);
      else
#pragma unroll
        for (int v = 0; v < VEC; ++v) x[u][v] = 0.f;
    }
#pragma unroll
    for (int g = 0; g < G_T; ++g) {
      float acc[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        acc[u] = 0.f;
#pragma unroll
        for (int v = 0; v < VEC; ++v) acc[u] = fmaf(q1[g][v], x[u][v], acc[u]);
        acc[u] = sum_lanes<LPR1>(acc[u]);
      }
      if (g < c.G) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int rr = (ps + u) * RPW1 + r;
          const bool writer = (sl == 0) && (rr < rows_here);
          const uint32_t key = order_key(acc[u]);
          if (writer) {
            c.keys[g * c.Lmax + i0 + rr] = key;
            if (p.approx_out) p.approx_out[(c.qrow0 + g) * (size_t)p.S_cap + c.s0 + i0 + rr] = acc[u];
          }
          if (c.need_keys) hist_add(c.hist + g * kRadixBins, writer, key >> 24);
        }
      }
    }
  }
}

}  // namespace

// Every warp is its own producer: warp w owns a private ring of `nsw`
// stages (mbarriers wbar[w][*]); its lane 0 issues the TMA transfers for the
// work items assigned to w (phase-1 boxes i = w, w + NW, ...; phase-3 stages
// st = w, w + NW, ...), the whole warp digests them, and lane 0 re-arms the
// slot for the warp's next item.  No cross-warp synchronisation inside the
// streaming phases, and NW warps keep TMA requests in flight (the gather4
// issue rate of a single thread is far below one SM's share of HBM).
template <typename T, int G_T, int VEC, int D_T, int NW>
__global__ void __launch_bounds__(NW * 32) fused_decode_tma_kernel(
    const FusedParams p, const __grid_constant__ CUtensorMap lead_map, const __grid_constant__ CUtensorMap krow_map,
    const __grid_constant__ CUtensorMap vrow_map, const __grid_constant__ CUtensorMap kbox_map,
    const __grid_constant__ CUtensorMap vbox_map) {
  constexpr int NT = NW * 32;
  constexpr int E = sizeof(T);
  constexpr int LPR3 = D_T / VEC;  // lanes per gathered row
  constexpr int RPW3 = 32 / LPR3;
  constexpr int ROWB = D_T * E;
  static_assert(LPR3 >= 1 && LPR3 <= 32 && (LPR3 & (LPR3 - 1)) == 0, "row layout");
  extern __shared__ __align__(128) uint8_t smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const int tid = threadIdx.x, lane = lane_id(), w = warp_id();
  const int nsw = p.nst, SB = p.stage_bytes;  // stages per warp, bytes per stage
  uint8_t* wring = smem + p.off_ring + (size_t)w * nsw * SB;
  uint64_t* wbar = reinterpret_cast<uint64_t*>(smem + p.off_bars) + (size_t)w * nsw;
  if (lane == 0) {
    for (int s = 0; s < nsw; ++s) mbar_init(&wbar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid == 0) {
    prefetch_desc(&lead_map);
    prefetch_desc(&krow_map);
    prefetch_desc(&vrow_map);
    prefetch_desc(&kbox_map);
    prefetch_desc(&vbox_map);
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");  // K0's q_hat / appended row are visible
  // the next layer's K0 may be scheduled into the tail of this grid (it stages
  // its P, then waits for this grid to complete before reading activations)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  trace(p, 0);

  Ctx c;
  if (!make_ctx<G_T>(p, smem, (int)cluster.block_rank(), c)) return;
  const int G = c.G, D = D_T;
  init_state<NT, G_T>(c);
  __syncthreads();
  RingPos rp(nsw);  // this warp's ring: uses so far, slot, parity

  // ------------------------------------------------------------ phase 1
  const bool need_scores = c.need_keys || (p.approx_out != nullptr);
  if (need_scores && p.ext_scores != nullptr) {
    keys_from_scores<NT>(p, c);
  } else if (need_scores) {
    const int R1 = p.r1;
    const int nbox = ceil_div(c.n_local, R1);
    const unsigned box_bytes = (unsigned)(R1 * p.dbox * E);
    const int mine = nbox > w ? ceil_div(nbox - w, NW) : 0;  // boxes w, w + NW, ...
    auto issue = [&](int k, const RingPos& at) {  // every lane (tma_box4d_warp: warp-uniform operands)
      tma_box4d_warp(wring + at.slot * SB, &lead_map, 0, c.s0 + (w + k * NW) * R1, c.hk, c.b, &wbar[at.slot],
                     box_bytes);
    };
    {
      RingPos q = rp;
      for (int k = 0; k < nsw && k < mine; ++k, q.advance(1)) issue(k, q);
    }
    const int nch1 = p.dbox / VEC;
    const int LPR1 = next_pow2(nch1);
    const int sl = lane % LPR1;
    float q1[G_T][VEC];
#pragma unroll
    for (int g = 0; g < G_T; ++g)
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        const int col = sl * VEC + v;
        q1[g][v] = (g < G && col < p.d && sl < nch1) ? p.q_hat[(c.qrow0 + g) * D + col] : 0.f;
      }
    for (int k = 0; k < mine; ++k, rp.advance(1)) {
      mbar_wait(&wbar[rp.slot], rp.phase);
      const uint8_t* tile = wring + rp.slot * SB;
      const int i = w + k * NW;
      const int rows_here = min(R1, c.n_local - i * R1);
      switch (LPR1) {
        case 1: consume_lead<T, G_T, VEC, 1>(p, c, tile, i * R1, rows_here, q1, lane); break;
        case 2: consume_lead<T, G_T, VEC, 2>(p, c, tile, i * R1, rows_here, q1, lane); break;
        case 4: consume_lead<T, G_T, VEC, 4>(p, c, tile, i * R1, rows_here, q1, lane); break;
        case 8: consume_lead<T, G_T, VEC, 8>(p, c, tile, i * R1, rows_here, q1, lane); break;
        case 16: consume_lead<T, G_T, VEC, 16>(p, c, tile, i * R1, rows_here, q1, lane); break;
        default: consume_lead<T, G_T, VEC, 32>(p, c, tile, i * R1, rows_here, q1, lane); break;
      }
      __syncwarp();  // every lane is done with the slot before it is refilled
      if (k + nsw < mine) issue(k + nsw, rp);
    }
  }
  __syncthreads();
  trace(p, 1);

  // ------------------------------------------------------------ phase 2
  select_phase<NT, G_T>(p, c, cluster);
  if (p.out == nullptr) {
    if (c.C > 1) cluster.sync();
    return;
  }
  trace(p, 4);
  const int n_rows = build_union<NT>(c);
  trace(p, 5);

  // ------------------------------------------------------------ phase 3
  const int R3 = p.r3;
  const int nstage = ceil_div(n_rows, R3);
  const unsigned stage_bytes = (unsigned)(2 * R3 * ROWB);
  const bool want_logits = p.weights_out != nullptr;
  const bool gather = !c.select_all || (p.debug & 1);
  const int row_base = (int)((long long)c.b * p.row_sb + (long long)c.hk * p.row_sh) + c.s0;
  const int mine = nstage > w ? ceil_div(nstage - w, NW) : 0;  // stages w, w + NW, ...
  // all lanes call issue (the row indices are spread over the lanes); lane 0 issues
  auto issue = [&](int k, const RingPos& at) {
    const int st = w + k * NW;
    uint8_t* dst = wring + at.slot * SB;
    if (lane == 0) mbar_expect_tx(&wbar[at.slot], stage_bytes);
    // warp-uniform TMA operands (tma_gather4_u): no per-instruction waterfall loop
    const uint32_t ds = __shfl_sync(0xffffffffu, smem_u32(dst), 0);
    const uint32_t bs = __shfl_sync(0xffffffffu, smem_u32(&wbar[at.slot]), 0);
    if (!gather) {
      if (lane == 0) {
        tma_box4d(dst, &kbox_map, 0, c.s0 + st * R3, c.hk, c.b, &wbar[at.slot]);
        tma_box4d(dst + R3 * ROWB, &vbox_map, 0, c.s0 + st * R3, c.hk, c.b, &wbar[at.slot]);
      }
    } else {
      int row = -1;  // lane t < R3 resolves row t of the stage; -1 = out of bounds, zero-filled
      const int u = st * R3 + lane;
      if (lane < R3 && u < n_rows) row = row_base + (c.select_all ? u : (int)c.uni[u]);
      for (int qq = 0; qq < R3 / 4; ++qq) {
        const int r0 = __shfl_sync(0xffffffffu, row, 4 * qq);
        const int r1 = __shfl_sync(0xffffffffu, row, 4 * qq + 1);
        const int r2 = __shfl_sync(0xffffffffu, row, 4 * qq + 2);
        const int r3 = __shfl_sync(0xffffffffu, row, 4 * qq + 3);
        if (lane == 0) {
          tma_gather4_u(ds + qq * 4 * ROWB, &krow_map, 0, r0, r1, r2, r3, bs);
          tma_gather4_u(ds + R3 * ROWB + qq * 4 * ROWB, &vrow_map, 0, r0, r1, r2, r3, bs);
        }
      }
    }
  };
  {
    RingPos q = rp;
    for (int k = 0; k < nsw && k < mine; ++k, q.advance(1)) issue(k, q);
  }
  float acc[G_T][1][VEC];
  float m[G_T], l[G_T];
#pragma unroll
  for (int g = 0; g < G_T; ++g) {
    m[g] = -CUDART_INF_F;
    l[g] = 0.f;
#pragma unroll
    for (int v = 0; v < VEC; ++v) acc[g][0][v] = 0.f;
  }
  {
    const int r = lane / LPR3, sl = lane % LPR3;
    const uint8_t full_mask = (uint8_t)((1u << G) - 1u);
    float q3[G_T][VEC];
#pragma unroll
    for (int g = 0; g < G_T; ++g)
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        const int col = sl * VEC + v;
        q3[g][v] = (g < G && col < D) ? p.q_hat[(c.qrow0 + g) * D + col] * p.qscale : 0.f;
      }
    constexpr int U = 2;  // rows per lane slot whose logits are formed before the softmax updates
    for (int k = 0; k < mine; ++k, rp.advance(1)) {
      mbar_wait(&wbar[rp.slot], rp.phase);
      const int st = w + k * NW;
      const uint8_t* kt = wring + rp.slot * SB;
      const uint8_t* vt = kt + R3 * ROWB;
      for (int ps = 0; ps < R3 / RPW3; ps += U) {  // host: (R3 / RPW3) % U == 0
        float x[U][G_T];
        int jr[U];
        uint8_t msk[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int rr = (ps + u) * RPW3 + r;
          const int t = st * R3 + rr;
          const bool ok = t < n_rows;
          const int j = ok ? (c.select_all ? t : (int)c.uni[t]) : 0;
          jr[u] = j;
          msk[u] = ok ? (c.select_all ? full_mask : c.selmask[j]) : (uint8_t)0;
          float kx[VEC];
          lds_chunk<T, VEC>(kt + rr * ROWB + sl * VEC * E, kx);
#pragma unroll
          for (int g = 0; g < G_T; ++g) {
            float s = 0.f;
#pragma unroll
            for (int v = 0; v < VEC; ++v) s = fmaf(q3[g][v], kx[v], s);
            x[u][g] = sum_lanes<LPR3>(s);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int rr = (ps + u) * RPW3 + r;
          float vx[VEC];
          lds_chunk<T, VEC>(vt + rr * ROWB + sl * VEC * E, vx);
#pragma unroll
          for (int g = 0; g < G_T; ++g) {
            if (msk[u] & (1u << g)) {
              const float xv = x[u][g];
              if (want_logits && sl == 0) c.keys[g * c.Lmax + jr[u]] = __float_as_uint(xv);
              const float mn = fmaxf(m[g], xv);
              const float sc = exp2f(m[g] - mn);
              const float pe = exp2f(xv - mn);
              l[g] = l[g] * sc + pe;
              m[g] = mn;
#pragma unroll
              for (int v = 0; v < VEC; ++v) acc[g][0][v] = fmaf(pe, vx[v], acc[g][0][v] * sc);
            }
          }
        }
      }
      __syncwarp();
      if (k + nsw < mine) issue(k + nsw, rp);
    }
  }
  trace(p, 6);
  merge_and_write<NT, G_T, 1, VEC>(p, c, cluster, m, l, acc, LPR3, 1, want_logits);
  trace(p, 7);
}

// ---------------------------------------------------------------- host side

size_t fused_tma_layout(int G_T, int NT, int D, int Lmax, bool keys_in_smem, int nsw, int stage_bytes,
                        FusedParams* p) {
  const int nw = NT / 32;
  size_t off = fused_layout(G_T, NT, D, Lmax, keys_in_smem, p);
  off = align_up(off, 128);
  p->off_ring = (int)off;
  off += (size_t)nw * nsw * stage_bytes;  // one private ring of nsw stages per warp
  p->off_bars = (int)off;
  off = align_up(off + (size_t)nw * nsw * 8, 16);  // one mbarrier per stage
  p->nst = nsw;
  p->stage_bytes = stage_bytes;
  return off;
}

namespace {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(f);
  }
  return fn;
}

bool encode4d(EncodeTiledFn enc, TmaDesc* out, const void* base, const loki_kv_geom& g, int box0, int box1,
              CUtensorMapL2promotion promo, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_NONE) {
  const size_t e = g.dtype == LOKI_DTYPE_BF16 ? 2 : 4;
  const CUtensorMapDataType dt =
      g.dtype == LOKI_DTYPE_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  // size-1 dimensions may carry any stride in a torch view; give TMA the packed one
  const int64_t sh = g.Hkv == 1 ? (int64_t)g.S_cap * g.stride_s : g.stride_h;
  const int64_t sb = g.B == 1 ? (int64_t)g.Hkv * sh : g.stride_b;
  cuuint64_t dims[4] = {(cuuint64_t)g.D, (cuuint64_t)g.S_cap, (cuuint64_t)g.Hkv, (cuuint64_t)g.B};
  cuuint64_t str[3] = {(cuuint64_t)(g.stride_s * e), (cuuint64_t)(sh * e), (cuuint64_t)(sb * e)};
  cuuint32_t box[4] = {(cuuint32_t)box0, (cuuint32_t)box1, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(reinterpret_cast<CUtensorMap*>(out->bytes), dt, 4, const_cast<void*>(base), dims, str, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, swz, promo,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool encode_rows(EncodeTiledFn enc, TmaDesc* out, const void* base, const loki_kv_geom& g, int width = 0,
                 int swizzle = 0, CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_128B) {
  const size_t e = g.dtype == LOKI_DTYPE_BF16 ? 2 : 4;
  const CUtensorMapDataType dt =
      g.dtype == LOKI_DTYPE_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  cuuint64_t dims[2] = {(cuuint64_t)g.D, (cuuint64_t)row_space(g).total};
  cuuint64_t str[1] = {(cuuint64_t)(g.stride_s * e)};
  cuuint32_t box[2] = {(cuuint32_t)(width > 0 ? width : g.D), 1};
  cuuint32_t es[2] = {1, 1};
  return enc(reinterpret_cast<CUtensorMap*>(out->bytes), dt, 2, const_cast<void*>(base), dims, str, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE,
             swizzle == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : (swizzle == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE),
             promo,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

RowSpace row_space(const loki_kv_geom& g) {
  RowSpace r;
  const long long ss = g.stride_s;
  // size-1 dimensions may carry any stride in a torch view: give them the packed one
  const long long sh = g.Hkv == 1 ? (long long)g.S_cap * ss : (long long)g.stride_h;
  const long long sb = g.B == 1 ? (long long)g.Hkv * sh : (long long)g.stride_b;
  if (ss < g.D || sh % ss != 0 || sb % ss != 0 || sh < (long long)g.S_cap * ss || sb < 0) return r;
  r.sh = sh / ss;
  r.sb = sb / ss;
  r.total = (long long)(g.B - 1) * r.sb + (long long)(g.Hkv - 1) * r.sh + g.S_cap;
  r.ok = r.total < (1LL << 31);
  return r;
}

bool encode_tma(const void* K, const void* V, const loki_kv_geom& g, int dbox, int r1, int r3, TmaDesc* maps) {
  EncodeTiledFn enc = encode_fn();
  if (enc == nullptr) return false;
  // [0] phase-1 boxes {dbox, r1} of K with 64 B promotion (exact leading-column bytes)
  // [1], [2] row gathers of K / V; [3], [4] contiguous boxes {D, r3} of K / V (dense)
  return encode4d(enc, &maps[0], K, g, dbox, r1, CU_TENSOR_MAP_L2_PROMOTION_L2_64B) &&
         encode_rows(enc, &maps[1], K, g) && encode_rows(enc, &maps[2], V, g) &&
         encode4d(enc, &maps[3], K, g, g.D, r3, CU_TENSOR_MAP_L2_PROMOTION_L2_128B) &&
         encode4d(enc, &maps[4], V, g, g.D, r3, CU_TENSOR_MAP_L2_PROMOTION_L2_128B);
}

bool encode_pipe_tma(const void* K, const void* V, const loki_kv_geom& g, int dbox, int r1, int kcol0,
                     bool mma, int lead_swz, TmaDesc* maps) {
  EncodeTiledFn enc = encode_fn();
  if (enc == nullptr) return false;
  const CUtensorMapSwizzle ls = lead_swz == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                               : (lead_swz == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE);
  if (!encode4d(enc, &maps[0], K, g, dbox, r1, CU_TENSOR_MAP_L2_PROMOTION_L2_64B, ls)) return false;
  if (mma) {  // tensor-core phase 3: 128 B row pieces 128B-swizzled, a trailing 64 B K piece 64B-swizzled
    // split-K reads K from column d: 64 B promotion fetches exactly the sectors after the lead columns
    const CUtensorMapL2promotion kp = kcol0 > 0 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B : CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
    return encode_rows(enc, &maps[1], K, g, 64, 128, kp) && encode_rows(enc, &maps[2], V, g, 64, 128) &&
           encode_rows(enc, &maps[3], K, g, 32, 64, CU_TENSOR_MAP_L2_PROMOTION_L2_64B);
  }
  return encode_rows(enc, &maps[1], K, g, g.D - kcol0) && encode_rows(enc, &maps[2], V, g) &&
         encode_rows(enc, &maps[3], K, g);
}

template <typename T, int G_T, int VEC, int D_T>
static cudaError_t launch_tma_t(const FusedParams& p, int units, size_t smem, const TmaDesc* maps,
                                cudaStream_t st) {
  constexpr int NW = kTmaWarps;
  auto kern = fused_decode_tma_kernel<T, G_T, VEC, D_T, NW>;
  static KernelAttrs attrs;
  cudaError_t e = attrs.ensure(reinterpret_cast<const void*>(kern), smem, p.C > 8);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(units * p.C));
  cfg.blockDim = dim3(NW * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)p.C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  const CUtensorMap* m = reinterpret_cast<const CUtensorMap*>(maps);
  return cudaLaunchKernelEx(&cfg, kern, p, m[0], m[1], m[2], m[3], m[4]);
}

template <typename T, int D_T>
static cudaError_t dispatch_tma_g(const FusedParams& p, const Plan& plan, const TmaDesc* maps, cudaStream_t st) {
  constexpr bool kBf16 = sizeof(T) == 2;
  const int units = p.B * p.Hkv;
  switch (plan.G_T) {
    case 1: return launch_tma_t<T, 1, kBf16 ? 8 : 4, D_T>(p, units, plan.smem, maps, st);
    case 2: return launch_tma_t<T, 2, kBf16 ? 8 : 4, D_T>(p, units, plan.smem, maps, st);
    case 4: return launch_tma_t<T, 4, kBf16 ? 8 : 4, D_T>(p, units, plan.smem, maps, st);
    case 8:
      if constexpr (D_T / 4 <= 32) return launch_tma_t<T, 8, 4, D_T>(p, units, plan.smem, maps, st);
      break;
    default: break;
  }
  return cudaErrorInvalidValue;
}

bool tma_supported(int dtype, int D, int G_T) {
  const int vec = dtype == LOKI_DTYPE_BF16 ? (G_T == 8 ? 4 : 8) : 4;
  return (D == 64 || D == 128 || D == 256) && D / vec <= 32 && G_T <= 8;
}

cudaError_t launch_fused_tma(const FusedParams& p, const Plan& plan, const TmaDesc* maps, cudaStream_t st) {
  if (plan.dtype == LOKI_DTYPE_BF16) {
    switch (p.D) {
      case 64: return dispatch_tma_g<__nv_bfloat16, 64>(p, plan, maps, st);
      case 128: return dispatch_tma_g<__nv_bfloat16, 128>(p, plan, maps, st);
      case 256: return dispatch_tma_g<__nv_bfloat16, 256>(p, plan, maps, st);
      default: break;
    }
  } else {
    switch (p.D) {
      case 64: return dispatch_tma_g<float, 64>(p, plan, maps, st);
      case 128: return dispatch_tma_g<float, 128>(p, plan, maps, st);
      default: break;
    }
  }
  return cudaErrorInvalidValue;
}

}  // namespace loki
