// Persistent, dynamically scheduled Loki decode attention -- the TOPK hot
// path on sm_100a (attention.py:166-185 loki_rank_and_attend, batched).
//
// Why not one cluster per (batch, KV head) unit (loki_decode_tma.cu): there
// every resident CTA runs phase 1 -> selection -> phase 3 -> merge in
// lockstep, so HBM idles while the whole GPU selects (profiles/r01_summary.md:
// 53 % of the roofline).  Here a grid of resident CTAs draws tickets from one
// global counter and each ticket is a work item:
//
//   A(u, c)  phase 1 over chunk c of unit u: TMA boxes of the leading d
//            columns (L2 promotion 64 B: exactly d*S*e DRAM bytes), approx
//            scores (kernels.py:223-241) -> order keys in an L2-resident
//            workspace + a (1 << hbits)-bin histogram of their top bits.  The
//            LAST A arriver of the unit runs the unit's top-k selection
//            (linalg.py:95-118) and publishes the ascending union list.
//   B(u, q)  phase 3 over part q of that list: tile::gather4 of the selected
//            K and V rows, exact logits / sqrt(D), online softmax and V
//            accumulation (kernels.py:244-279, linalg.py:76-92) -> a partial
//            (m, l, acc) state.  The LAST B arriver merges the parts in fixed
//            order and writes the output row.
//
// B tickets of unit u are issued `lag` units after its A tickets, so while
// one CTA selects, the others keep streaming.  Items are 256 KB - 1 MB of HBM
// traffic, so the tail of the grid is short and there is no wave
// quantisation.  Everything is deterministic: selections are exact, partial
// states are merged in fixed order (warps, then parts).
//
// Selection on 64-bit composite keys (order_key(score) << 32 | ~row): all
// composites are distinct and "the k largest composites" is exactly the
// reference's rule -- every score above the threshold, then threshold ties
// lowest row first.  MSB radix select: the first digit comes from the
// histogram built during phase 1; further digits are resolved over the
// candidates (compacted to shared memory once they fit).
#pragma once
#include <cuda.h>

#include <type_traits>

#include "loki_fused.cuh"
#include "loki_tma.cuh"
#include "loki_umma.cuh"

namespace loki {

namespace {

using namespace tma;
using fused::kMaxG;
using fused::merge_state;

#ifndef LOKI_PIPE_WARPS
#define LOKI_PIPE_WARPS 8
#endif
constexpr int kPW = LOKI_PIPE_WARPS;  // warps per CTA; every warp streams through its own TMA ring
constexpr int kPT = kPW * 32;

struct PipeShared {
  unsigned next_ticket;
  int last;
  long long t_sel;
  int fb_bin;
  unsigned fb_above, fb_cnt;
  int scan[kPW];
  int ncand, ncand_first;
  unsigned long long tsel;
  unsigned long long Tc[kMaxG];
  int wcnt[kPW][kMaxG + 1];
  float gm[kMaxG], gl[kMaxG];
};

// Thread groups the selection helpers run on: the whole CTA, or a warp group of
// a warp-specialised CTA (its own named barrier; the other group keeps going).
struct CtaGroup {
  static constexpr int kThreads = kPT, kWarps = kPW;
  __device__ __forceinline__ static int tid() { return threadIdx.x; }
  __device__ __forceinline__ static int warp() { return threadIdx.x >> 5; }
  __device__ __forceinline__ static void sync() { __syncthreads(); }
};
template <int FIRST_WARP, int NWARPS, int BAR_ID>
struct WarpGroup {
  static constexpr int kThreads = NWARPS * 32, kWarps = NWARPS;
  __device__ __forceinline__ static int tid() { return (int)threadIdx.x - FIRST_WARP * 32; }
  __device__ __forceinline__ static int warp() { return ((int)threadIdx.x >> 5) - FIRST_WARP; }
  __device__ __forceinline__ static void sync() {
    asm volatile("bar.sync %0, %1;" ::"n"(BAR_ID), "n"(NWARPS * 32) : "memory");
  }
};

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// generic-proxy shared-memory writes ordered before later TMA (async-proxy) writes
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ unsigned long long comp_key(uint32_t key, int j) {
  return ((unsigned long long)key << 32) | (unsigned long long)(~(uint32_t)j);
}

// ---- tensor-core helpers (phase 3 on bf16 caches)
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
// d += a (16x16 bf16, row) * b (16x8 bf16, col), fp32 accumulate
__device__ __forceinline__ void mma_bf16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// {lo -> bits 0..15, hi -> bits 16..31}, round to nearest even
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
// x = hi + lo with hi, lo bf16 (relative error of hi + lo ~ 2^-17)
__device__ __forceinline__ float bf16_hi(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }
__device__ __forceinline__ float bf16_lo(float x) { return x - bf16_hi(x); }
// 16 B chunk c of row r inside a 128B-swizzled block of 128 B rows (TMA SWIZZLE_128B)
__device__ __forceinline__ uint32_t swz128(uint32_t base, int r, int c) {
  return base + (uint32_t)(r * 128) + (uint32_t)(((c ^ (r & 7)) << 4));
}

__device__ __forceinline__ int k_of(const PipeParams& p, int S) {
  if (S <= 0) return 0;
  return p.k_fixed > 0 ? (p.k_fixed < S ? p.k_fixed : S) : resolve_fraction(p.k_f, S);
}

// Group-wide inclusive scan of one value per thread, in thread order.
// Query heads of a unit: the group size, also for the A launch of a group-shared layer (whose params
// carry G = 1 and shared = the group size).
__device__ __forceinline__ int unit_heads(const PipeParams& p) { return p.shared > 1 ? p.shared : p.G; }
// Head mask of a selected row in an entry list: every head of the group in shared mode.
__device__ __forceinline__ unsigned shared_mask(const PipeParams& p) {
  return p.shared > 1 ? (1u << p.shared) - 1u : 1u;
}

// Column c of the query that ranks a unit's rows: q_hat[qrow0] itself, or (group-shared selection)
// q_0 + q_1 + ... + q_{gs-1} summed in that fixed order in fp32.  Out of line: an inlined loop with a
// runtime trip count inside the callers' unrolled column loops multiplied their code size (r02: the
// A launch's kernel grew 5x and ran 40 us slower at C2).
__device__ __noinline__ float group_q(const PipeParams& p, size_t qrow0, int gs, int c) {
  float a = p.q_hat[qrow0 * p.D + c];
  for (int g = 1; g < gs; ++g) a += p.q_hat[(qrow0 + g) * p.D + c];
  return a;
}

template <typename Grp = CtaGroup>
__device__ __forceinline__ unsigned block_incl_scan(unsigned v, PipeShared& sh, unsigned* total) {
  const int lane = lane_id(), w = Grp::warp();
  unsigned x = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const unsigned t = __shfl_up_sync(0xffffffffu, x, off);
    if (lane >= off) x += t;
  }
  if (lane == 31) sh.scan[w] = (int)x;
  Grp::sync();
  unsigned before = 0, tot = 0;
#pragma unroll
  for (int i = 0; i < Grp::kWarps; ++i) {
    const unsigned c = (unsigned)sh.scan[i];
    before += i < w ? c : 0u;
    tot += c;
  }
  Grp::sync();
  *total = tot;
  return before + x;
}

// The bin holding the need-th largest element: largest b with
// sum_{i>b} h[i] < need <= sum_{i>=b} h[i] -> sh.fb_bin / fb_above / fb_cnt.
template <typename Grp = CtaGroup>
__device__ void find_bin(const uint32_t* h, int nbins, unsigned need, PipeShared& sh) {
  const int tid = Grp::tid();
  const int per = nbins > Grp::kThreads ? nbins / Grp::kThreads : 1;  // nbins is a power of two
  const int hi = nbins - tid * per;                                    // this thread owns bins [hi - per, hi)
  unsigned s = 0;
  if (hi > 0)
    for (int i = 0; i < per; ++i) s += h[hi - 1 - i];
  unsigned tot;
  const unsigned incl = block_incl_scan<Grp>(s, sh, &tot);
  const unsigned excl = incl - s;
  if (hi > 0 && excl < need && need <= incl) {
    unsigned acc = excl;
    for (int i = 0; i < per; ++i) {
      const int b = hi - 1 - i;
      if (acc + h[b] >= need) {
        sh.fb_bin = b;
        sh.fb_above = acc;
        sh.fb_cnt = h[b];
        break;
      }
      acc += h[b];
    }
  }
  Grp::sync();
}

// Warp-aggregated append of `c` to dst when `m` (order within dst is irrelevant).
__device__ __forceinline__ void append_if(bool m, unsigned long long c, unsigned long long* dst, int* counter) {
  const int lane = lane_id();
  const unsigned bal = __ballot_sync(0xffffffffu, m);
  int base = 0;
  if (lane == 0 && bal) base = atomicAdd(counter, __popc(bal));
  base = __shfl_sync(0xffffffffu, base, 0);
  if (m) dst[base + __popc(bal & ((1u << lane) - 1u))] = c;
}

// ------------------------------------------------------------------ selection
// Scans over a unit's keys are latency-bound L2 reads: every lane keeps
// kSU uint4 loads (16 rows) in flight.  Warp w owns the contiguous rows
// [ra, rb) (128-row aligned) so the emission can be ordered.
constexpr int kSU = 4;

__device__ __forceinline__ uint4 ld_keys4(const uint32_t* k, int j) {
  return __ldcg(reinterpret_cast<const uint4*>(k + j));
}
__device__ __forceinline__ uint32_t u4_at(const uint4& v, int e) {
  return e == 0 ? v.x : (e == 1 ? v.y : (e == 2 ? v.z : v.w));
}


__device__ __forceinline__ int warp_excl_scan(int v, int* total) {
  const int lane = lane_id();
  int x = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, x, off);
    if (lane >= off) x += t;
  }
  *total = __shfl_sync(0xffffffffu, x, 31);
  return x - v;
}

// Keys of one head streamed through shared memory: two buffers of kCK keys
// filled by cp.async.bulk (one L2 round trip per chunk, the next chunk in
// flight while this one is scanned).  `sbar` are two mbarriers owned by the
// selection; `sphase` holds their parity bits (identical in every thread).
constexpr int kCK = 4096;  // keys per chunk (16 KB)
constexpr int kSpecW = 2;  // speculative candidate window: boundary-bin estimate +- kSpecW bins

struct KeyStream {
  const uint32_t* src;
  int S, kstride;
  uint32_t* buf;  // [2][kCK]
  uint64_t* sbar;
  unsigned* sphase;
  int nchunk;
  __device__ void issue(int c) const {
    if (threadIdx.x == 0 && c < nchunk) {
      const int base = c * kCK;
      int rows = min(kCK, kstride - base);
      const unsigned bytes = (unsigned)(((rows * 4) + 15) & ~15);
      uint64_t* bar = &sbar[c & 1];
      mbar_expect_tx(bar, bytes);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(buf + (c & 1) * kCK)),
          "l"(src + base), "r"(bytes), "r"(smem_u32(bar))
          : "memory");
    }
  }
  // chunks 0 and 1 in flight (call once per pass, before run)
  __device__ void start() const {
    if (threadIdx.x == 0) asm volatile("fence.proxy.async.global;" ::: "memory");  // keys were stored by generic st
    issue(0);
    issue(1);
  }
  // wait for the chunks start() issued without reading them
  __device__ void drain() const {
    for (int c = 0; c < 2 && c < nchunk; ++c) {
      mbar_wait(&sbar[c], (*sphase >> c) & 1u);
      *sphase ^= 1u << c;
    }
    __syncthreads();
  }
  // f(j0, keys, n): rows [j0, j0 + n) of the chunk in shared memory; every thread calls
  template <typename F>
  __device__ void run(F&& f) const {
    for (int c = 0; c < nchunk; ++c) {
      const int bi = c & 1;
      mbar_wait(&sbar[bi], (*sphase >> bi) & 1u);
      *sphase ^= 1u << bi;
      f(c * kCK, buf + bi * kCK, min(kCK, S - c * kCK));
      __syncthreads();  // every thread is done with buffer bi before it is refilled
      issue(c + 2);
    }
  }
};

// LOKI_DEBUG & 16 (tuning only): %globaltimer at selection checkpoints, [units][8] at trace + 2^21
template <typename Grp = CtaGroup>
__device__ __forceinline__ void sel_stamp(const PipeParams& p, int u, int k) {
  if ((p.debug & 16) && p.trace != nullptr && Grp::tid() == 0) p.trace[(1 << 21) + (size_t)u * 8 + k] = globaltimer();
}

// Threshold of each head's top-k in unit u on 64-bit composite keys: the
// last A arriver reads the level-0 histogram, compacts the boundary-bin rows
// into shared memory with one pass over the keys (further histogram levels
// only if they do not fit), narrows them (radix passes, then a direct rank
// once <= 256 remain) and publishes tcs[u][g].  With idx_out it also
// publishes each part's output offset (rows above the boundary per part +
// candidates kept).
template <typename Grp, int NB = 2>
__device__ void emit_lists_global(const PipeParams& p, int u, int S, unsigned long long Tc, uint32_t* kbuf,
                                  uint64_t* sbar, unsigned& sphase, PipeShared& sh);
template <typename Grp, int G_T, int NB = 2, int CKE = kCK>
__device__ void emit_lists_global_heads(const PipeParams& p, int u, int S, uint32_t* kbuf, uint64_t* sbar,
                                        unsigned& sphase, PipeShared& sh);

template <int G_T>
__device__ void select_unit(const PipeParams& p, int u, int S, uint8_t* ring, uint32_t* hist, uint64_t* sbar,
                            unsigned& sphase, PipeShared& sh) {
  const int tid = threadIdx.x, lane = lane_id(), w = warp_id();
  const int G = p.G, hb = p.hbits, HB = 1 << hb;
  uint32_t* cu = p.ctrl + 2 + 4 * (size_t)u;
  const int kb = k_of(p, S);
  const int cap = p.cand_cap;
  const bool offsets = p.idx_out != nullptr;
  uint32_t* kbuf = reinterpret_cast<uint32_t*>(ring);
  unsigned long long* candA = reinterpret_cast<unsigned long long*>(ring + 2 * kCK * 4);
  unsigned long long* candB = candA + cap;
  unsigned long long* candC = candB + cap;
  const int Lh = p.Lc / 2;                      // idx_out offsets at half-part granularity
  const int nhp = ceil_div(S > 0 ? S : 1, Lh);
  const int nparts_a = ceil_div(S > 0 ? S : 1, p.La);
  for (int g = 0; g < G; ++g) {
    const uint32_t* keys = p.keys + ((size_t)u * G + g) * p.kstride;
    uint32_t* gh = p.hist + ((size_t)u * G + g) * HB;
    // per half part; group-shared selection: the one list's offsets serve (and are copied to) every head
    uint32_t* poff = offsets ? p.poff + ((size_t)u * unit_heads(p) + g) * 2 * p.nA : nullptr;
    KeyStream ks{keys, S, p.kstride, kbuf, sbar, &sphase, ceil_div(S, kCK)};
    if (g == 0) sel_stamp(p, u, 0);
    const bool spec = p.spec && !offsets;
    if (kb > 0 && !spec) ks.start();  // prefetch: the compaction pass below almost always runs
    for (int i = tid; i < HB; i += kPT) {
      hist[i] = __ldcg(&gh[i]);
      gh[i] = 0u;  // ready for the next launch
    }
    if (offsets)
      for (int q = tid; q < nhp; q += kPT) poff[q] = 0u;
    __syncthreads();
    if (kb == 0) {
      if (tid == 0) p.tcs[(size_t)u * G + g] = ~0ull;
      continue;
    }
    find_bin(hist, HB, (unsigned)kb, sh);
    if (g == 0) sel_stamp(p, u, 1);
    unsigned long long P = (unsigned long long)sh.fb_bin;
    int nb = hb;
    unsigned need = (unsigned)kb - sh.fb_above, cnt = sh.fb_cnt;
    int ncand = 0;
    bool listed = false, started = !spec;
    if (spec) {
      const size_t ug = (size_t)u * G + g;
      const unsigned total = __ldcg(&p.ccnt[ug]);
      if (tid == 0) sh.ncand = (total <= (unsigned)p.ccap && cnt <= (unsigned)cap) ? 1 : 0;
      __syncthreads();
      for (int q = tid; q < nparts_a; q += kPT) {
        const uint32_t wv = __ldcg(&p.cwin[ug * p.nA + q]);
        if (P < (wv & 0xFFFFu) || P > (wv >> 16)) sh.ncand = 0;  // a chunk's window misses the boundary bin
      }
      __syncthreads();
      const bool use = sh.ncand != 0;
      __syncthreads();
      if (tid == 0) {
        sh.ncand = 0;
        p.ccnt[ug] = 0u;  // ready for the next launch
      }
      __syncthreads();
      if (use) {
        const unsigned long long* cb = p.cbuf + ug * p.ccap;
        for (int i0 = 0; i0 < (int)total; i0 += 4 * kPT) {
          unsigned long long cv[4];
#pragma unroll
          for (int x = 0; x < 4; ++x) {
            const int i = i0 + x * kPT + tid;
            cv[x] = i < (int)total ? __ldcg(&cb[i]) : 0ull;
          }
#pragma unroll
          for (int x = 0; x < 4; ++x) {
            const int i = i0 + x * kPT + tid;
            append_if(i < (int)total && (cv[x] >> (64 - nb)) == P, cv[x], candA, &sh.ncand);
          }
        }
        __syncthreads();
        ncand = sh.ncand;
        if (tid == 0) sh.ncand_first = ncand;
        listed = (unsigned)ncand == cnt;  // always true when the windows cover the bin
      }
    }
    for (; !listed;) {
      if (!started) ks.start();
      started = false;
      if (cnt <= (unsigned)cap) {  // compact the rows matching P (and count the rows above P per part)
        if (tid == 0) sh.ncand = 0;
        __syncthreads();
        const unsigned long long Pc = P;
        const int sh64 = 64 - nb;
        ks.run([&](int j0, const uint32_t* kc, int nrow) {
          for (int i0 = 0; i0 < nrow; i0 += 4 * kPT) {
            const int il = i0 + 4 * tid;
            const uint4 kk = *reinterpret_cast<const uint4*>(kc + il);
            int above = 0;
            bool any = false;
            if (nb <= 32) {  // prefix inside the 32-bit key: cheap tests, composites only for candidates
              const int s32 = 32 - nb;
              const uint32_t P32 = (uint32_t)Pc;
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const bool ok = il + e < nrow;
                const uint32_t pre = u4_at(kk, e) >> s32;
                above += (ok && pre > P32) ? 1 : 0;
                any |= ok && pre == P32;
              }
            } else {
              any = true;
#pragma unroll
              for (int e = 0; e < 4; ++e)
                above += (il + e < nrow && (comp_key(u4_at(kk, e), j0 + il + e) >> sh64) > Pc) ? 1 : 0;
            }
            if (__any_sync(0xffffffffu, any)) {
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const unsigned long long c = comp_key(u4_at(kk, e), j0 + il + e);
                append_if(il + e < nrow && (c >> sh64) == Pc, c, candA, &sh.ncand);
              }
            }
            if (offsets) {  // a warp's 128 rows lie inside one half part (Lc / 2 % 128 == 0)
              above = __reduce_add_sync(0xffffffffu, above);
              const int jw = j0 + i0 + 128 * w;
              if (lane == 0 && above) atomicAdd(&poff[jw / Lh], (uint32_t)above);
            }
          }
        });
        ncand = sh.ncand;
        if (tid == 0) sh.ncand_first = ncand;
        listed = true;
        break;
      }
      if (cnt == need) {  // exact boundary bin, too large to list: drain the prefetched chunks
        ks.drain();
        break;
      }
      // one more histogram level over every row matching P
      const int bits = min(hb, 64 - nb);
      for (int i = tid; i < (1 << bits); i += kPT) hist[i] = 0u;
      __syncthreads();
      const unsigned long long Pc = P;
      const int sh64 = 64 - nb;
      ks.run([&](int j0, const uint32_t* kc, int nrow) {
        for (int i = tid; i < nrow; i += kPT) {
          const unsigned long long c = comp_key(kc[i], j0 + i);
          if ((c >> sh64) == Pc) atomicAdd(&hist[(c >> (sh64 - bits)) & ((1ull << bits) - 1)], 1u);
        }
      });
      find_bin(hist, 1 << bits, need, sh);
      P = (P << bits) | (unsigned long long)sh.fb_bin;
      nb += bits;
      need -= sh.fb_above;
      cnt = sh.fb_cnt;
    }
    unsigned long long Tc;
    if (g == 0) sel_stamp(p, u, 2);
    if ((p.debug & 16) && p.trace != nullptr && tid == 0 && g == 0) p.trace[(1 << 21) + (size_t)u * 8 + 7] = ncand;
    if (listed) {  // narrow inside shared memory; candA stays intact for the part counts
      const unsigned long long* src = candA;
      unsigned long long* dst = candB;
      while (cnt != need && ncand > 256) {
        const int bits = min(8, 64 - nb);
        for (int i = tid; i < (1 << bits); i += kPT) hist[i] = 0u;
        __syncthreads();
        for (int i = tid; i < ncand; i += kPT)
          atomicAdd(&hist[(src[i] >> (64 - nb - bits)) & ((1ull << bits) - 1)], 1u);
        __syncthreads();
        find_bin(hist, 1 << bits, need, sh);
        P = (P << bits) | (unsigned long long)sh.fb_bin;
        nb += bits;
        need -= sh.fb_above;
        cnt = sh.fb_cnt;
        if (cnt == need) break;
        if (tid == 0) sh.ncand = 0;
        __syncthreads();
        for (int i0 = 0; i0 < ncand; i0 += kPT) {
          const int i = i0 + tid;
          const unsigned long long c = i < ncand ? src[i] : 0ull;
          append_if(i < ncand && (c >> (64 - nb)) == P, c, dst, &sh.ncand);
        }
        __syncthreads();
        ncand = sh.ncand;
        src = dst;
        dst = (dst == candB) ? candC : candB;
      }
      if (g == 0) sel_stamp(p, u, 3);
      if (cnt == need) {
        Tc = nb >= 64 ? P : (P << (64 - nb));
      } else {  // <= 256 distinct candidates: the need-th largest by direct rank
        for (int ci = tid; ci < ncand; ci += kPT) {
          const unsigned long long c = src[ci];
          unsigned rank = 0;
          for (int i = 0; i < ncand; ++i) rank += src[i] > c;
          if (rank == need - 1) sh.tsel = c;
        }
        __syncthreads();
        Tc = sh.tsel;
      }
      if (offsets) {  // kept candidates per part
        const int n0 = sh.ncand_first;
        for (int i = tid; i < n0; i += kPT) {
          const unsigned long long c = candA[i];
          if (c >= Tc) atomicAdd(&poff[(int)(~(uint32_t)c) / Lh], 1u);
        }
      }
    } else {
      Tc = nb >= 64 ? P : (P << (64 - nb));
      if (offsets) {  // counting pass: rows >= Tc per part
        ks.start();
        ks.run([&](int j0, const uint32_t* kc, int nrow) {
          for (int i0 = 0; i0 < nrow; i0 += kPT) {
            const int i = i0 + tid;
            const bool on = i < nrow && comp_key(kc[i], j0 + i) >= Tc;
            const int c = __popc(__ballot_sync(0xffffffffu, on));
            if (lane == 0 && c) atomicAdd(&poff[(j0 + i0 + 32 * w) / Lh], (uint32_t)c);
          }
        });
      }
    }
    if (g == 0) sel_stamp(p, u, 4);
    if (tid == 0) p.tcs[(size_t)u * G + g] = Tc;
    if (offsets) {  // counts -> exclusive offsets (one warp)
      __syncthreads();
      if (w == 0) {
        unsigned run = 0;
        for (int q0 = 0; q0 < nhp; q0 += 32) {
          const int q = q0 + lane;
          const unsigned v = q < nhp ? __ldcg(&poff[q]) : 0u;
          unsigned x = v;
#pragma unroll
          for (int off = 1; off < 32; off <<= 1) {
            const unsigned t = __shfl_up_sync(0xffffffffu, x, off);
            if (lane >= off) x += t;
          }
          if (q < nhp) {
            poff[q] = run + x - v;
            for (int gg = 1; gg < p.shared; ++gg) poff[(size_t)gg * 2 * p.nA + q] = run + x - v;
          }
          run += __shfl_sync(0xffffffffu, x, 31);
        }
      }
    }
    __syncthreads();
  }
  if (p.lists) {  // lists mode: the unit's ordered entries for the B items
    __syncthreads();
    if constexpr (G_T == 1)
      emit_lists_global<CtaGroup>(p, u, S, __ldcg(&p.tcs[u]), reinterpret_cast<uint32_t*>(ring), sbar, sphase, sh);
    else
      emit_lists_global_heads<CtaGroup, G_T, 2, (G_T * 1024 > kCK ? G_T * 1024 : kCK)>(  // (the whole ring)
          p, u, S, reinterpret_cast<uint32_t*>(ring), sbar, sphase, sh);
  }
  if (tid == 0) cu[0] = 0u;  // A arrivals: ready for the next launch
  sel_stamp(p, u, 5);
  __syncthreads();
  if (tid == 0) {  // the barrier makes every thread's writes visible to thread 0; its release publishes them
    __threadfence();
    st_release(&cu[2], 1u);
  }
  sel_stamp(p, u, 6);
}

// Selection of a single-chunk unit with everything on chip: the unit's keys
// ([G][kst] in shared memory) and its complete level-0 histogram are where the
// A item left them, so the threshold costs no L2 round trip.  Same composite-key
// rule as select_unit (linalg.py:95-118): the boundary bin's rows are compacted
// into `scratch` (the idle TMA ring) when they fit, else narrowed by further
// histogram levels over the on-chip keys; radix passes over the candidates, then
// a direct rank once <= 256 remain.  Thresholds -> sh.Tc[g].
template <int G_T, typename Grp = CtaGroup>
__device__ void select_onchip(const PipeParams& p, int u, int S, const uint32_t* ks, int kst, uint32_t* hist,
                              uint8_t* scratch, int scratch_bytes, PipeShared& sh) {
  const int tid = Grp::tid();
  const int G = p.G, hb = p.hbits, HB = 1 << hb;
  const int kb = k_of(p, S);
  const int cap = scratch_bytes / 16;
  unsigned long long* candA = reinterpret_cast<unsigned long long*>(scratch);
  unsigned long long* candB = candA + cap;
  for (int g = 0; g < G; ++g) {
    const uint32_t* kg = ks + (size_t)g * kst;
    uint32_t* h = hist + g * HB;  // consumed by find_bin, then reused for deeper levels
    if (kb <= 0 || kb >= S) {     // nothing / everything selected
      if (tid == 0) sh.Tc[g] = kb <= 0 ? ~0ull : 0ull;
      continue;
    }
    find_bin<Grp>(h, HB, (unsigned)kb, sh);
    if (g == 0) sel_stamp<Grp>(p, u, 1);
    unsigned long long P = (unsigned long long)sh.fb_bin;
    int nb = hb;
    unsigned need = (unsigned)kb - sh.fb_above, cnt = sh.fb_cnt;
    int ncand = 0;
    bool listed = false;
    for (;;) {
      if (cnt == need) break;  // the whole boundary prefix is selected
      const int sh64 = 64 - nb;
      if (cnt <= (unsigned)cap) {  // compact the rows matching P
        if (tid == 0) sh.ncand = 0;
        Grp::sync();
        const int lane = lane_id();
        // (r02: eight uint4 groups per thread per round, one warp scan and one shared atomic per warp and round
        // -- the per-128-row scan + atomic chain made this pass 4.2 us at 8K rows)
        constexpr int U = 8;
        for (int i0 = 0; i0 < S; i0 += 4 * U * Grp::kThreads) {
          uint4 kk[U];
          unsigned hit[U];
          int c = 0;
#pragma unroll
          for (int v = 0; v < U; ++v) {
            const int il = i0 + 4 * (tid + v * Grp::kThreads);
            kk[v] = make_uint4(0u, 0u, 0u, 0u);
            if (il < S) kk[v] = *reinterpret_cast<const uint4*>(kg + il);  // kst % 4 == 0, rows past S masked
            hit[v] = 0u;
#pragma unroll
            for (int e = 0; e < 4; ++e)
              hit[v] |= (il + e < S && (comp_key(u4_at(kk[v], e), il + e) >> sh64) == P ? 1u : 0u) << e;
            c += __popc(hit[v]);
          }
          if (__any_sync(0xffffffffu, c != 0)) {  // one shared atomic per warp, then order-free writes
            int tot;
            const int ex = warp_excl_scan(c, &tot);
            int at = 0;
            if (lane == 0) at = atomicAdd(&sh.ncand, tot);
            at = __shfl_sync(0xffffffffu, at, 0) + ex;
#pragma unroll
            for (int v = 0; v < U; ++v) {
              const int il = i0 + 4 * (tid + v * Grp::kThreads);
#pragma unroll
              for (int e = 0; e < 4; ++e)
                if ((hit[v] >> e) & 1u) candA[at++] = comp_key(u4_at(kk[v], e), il + e);
            }
          }
        }
        Grp::sync();
        ncand = sh.ncand;
        listed = true;
        break;
      }
      // one more histogram level over the rows matching P
      const int bits = min(hb, 64 - nb);
      for (int i = tid; i < (1 << bits); i += Grp::kThreads) h[i] = 0u;
      Grp::sync();
      for (int i = tid; i < S; i += Grp::kThreads) {
        const unsigned long long c = comp_key(kg[i], i);
        if ((c >> sh64) == P) atomicAdd(&h[(c >> (sh64 - bits)) & ((1ull << bits) - 1)], 1u);
      }
      Grp::sync();
      find_bin<Grp>(h, 1 << bits, need, sh);
      P = (P << bits) | (unsigned long long)sh.fb_bin;
      nb += bits;
      need -= sh.fb_above;
      cnt = sh.fb_cnt;
    }
    unsigned long long Tc = nb >= 64 ? P : (P << (64 - nb));
    if (g == 0) sel_stamp<Grp>(p, u, 2);
    if ((p.debug & 16) && p.trace != nullptr && tid == 0 && g == 0) p.trace[(1 << 21) + (size_t)u * 8 + 7] = ncand;
    if (listed && cnt != need) {
      const unsigned long long* src = candA;
      unsigned long long* dst = candB;
      while (ncand > 32) {
        const int bits = min(8, 64 - nb);
        for (int i = tid; i < (1 << bits); i += Grp::kThreads) h[i] = 0u;
        Grp::sync();
        for (int i = tid; i < ncand; i += Grp::kThreads) atomicAdd(&h[(src[i] >> (64 - nb - bits)) & ((1ull << bits) - 1)], 1u);
        Grp::sync();
        find_bin<Grp>(h, 1 << bits, need, sh);
        P = (P << bits) | (unsigned long long)sh.fb_bin;
        nb += bits;
        need -= sh.fb_above;
        cnt = sh.fb_cnt;
        if (cnt == need) break;
        if (tid == 0) sh.ncand = 0;
        Grp::sync();
        for (int i0 = 0; i0 < ncand; i0 += Grp::kThreads) {
          const int i = i0 + tid;
          const unsigned long long c = i < ncand ? src[i] : 0ull;
          append_if(i < ncand && (c >> (64 - nb)) == P, c, dst, &sh.ncand);
        }
        Grp::sync();
        ncand = sh.ncand;
        unsigned long long* was = const_cast<unsigned long long*>(src);
        src = dst;
        dst = was;
      }
      if (cnt == need) {
        Tc = nb >= 64 ? P : (P << (64 - nb));
      } else {  // <= 32 distinct candidates, one per lane of warp 0: the need-th largest by rank
        if (tid < 32) {
          const unsigned long long c = tid < ncand ? src[tid] : 0ull;
          unsigned rank = 0;
          for (int i = 0; i < ncand; ++i) rank += __shfl_sync(0xffffffffu, c, i) > c;
          if (tid < ncand && rank == need - 1) sh.tsel = c;
        }
        Grp::sync();
        Tc = sh.tsel;
      }
    }
    if (g == 0) sel_stamp<Grp>(p, u, 3);
    if (tid == 0) sh.Tc[g] = Tc;
    Grp::sync();
  }
  Grp::sync();
}

// Ordered emission of a single-chunk unit's selection: entries (head mask << 24
// | row) of every row some head of the group selected, ascending, to p.sel[u],
// plus the entry offset of every half part (Lc / 2 rows) to p.loff[u] -- the B
// items read their part's slice instead of re-deriving it from the keys.  Warp w
// owns the contiguous rows [w S8, (w + 1) S8): a counting pass (ballots), one
// block exclusive scan of the warp totals, then an ordered writing pass.
template <int G_T, typename Grp = CtaGroup>
__device__ void emit_lists(const PipeParams& p, int u, int S, const uint32_t* ks, int kst, PipeShared& sh) {
  const int lane = lane_id(), w = Grp::warp();
  const int G = p.G;
  const int lhs = 31 - __clz(p.Lc / 2);  // Lc / 2 is a power of two
  uint32_t* dst = p.sel + (size_t)u * p.sel_stride;
  uint32_t* lo = p.loff + (size_t)u * (2 * p.nA + 1);
  unsigned long long Tc[G_T];
#pragma unroll
  for (int g = 0; g < G_T; ++g) Tc[g] = g < G ? sh.Tc[g] : ~0ull;
  const unsigned one = G_T == 1 ? shared_mask(p) : 1u;  // G = 1 lists: a selected row serves the whole group
  // diagnostics (G = 1 lists): entry order is each head's ascending index order
  int32_t* idx_dst = nullptr;
  int nh = 0;
  if (G_T == 1 && p.idx_out != nullptr) {
    nh = unit_heads(p);
    idx_dst = p.idx_out + ((size_t)(u / p.Hkv) * p.Hq + (size_t)(u % p.Hkv) * nh) * p.idx_stride;
  }
  // warp w: rows [r0, r1), 128 per pass (4 per lane, one uint4 of keys per head)
  const int S8 = ceil_div(ceil_div(S > 0 ? S : 1, Grp::kWarps), 128) * 128;
  const int r0 = min(S, w * S8), r1 = min(S, r0 + S8);
  auto masks = [&](int j, unsigned (&m)[4]) -> int {
#pragma unroll
    for (int e = 0; e < 4; ++e) m[e] = 0u;
    if (j < r1) {
#pragma unroll
      for (int g = 0; g < G_T; ++g) {
        if (g < G) {
          const uint4 kk = *reinterpret_cast<const uint4*>(ks + (size_t)g * kst + j);
#pragma unroll
          for (int e = 0; e < 4; ++e)
            m[e] |= (j + e < r1 && comp_key(u4_at(kk, e), j + e) >= Tc[g] ? one : 0u) << g;
        }
      }
    }
    return (m[0] != 0u) + (m[1] != 0u) + (m[2] != 0u) + (m[3] != 0u);
  };
  unsigned cnt = 0;
  for (int j0 = r0; j0 < r1; j0 += 128) {
    unsigned m[4];
    cnt += __reduce_add_sync(0xffffffffu, (unsigned)masks(j0 + 4 * lane, m));
  }
  if (lane == 0) sh.scan[w] = (int)cnt;
  Grp::sync();
  unsigned base = 0, total = 0;
#pragma unroll
  for (int i = 0; i < Grp::kWarps; ++i) {
    base += i < w ? (unsigned)sh.scan[i] : 0u;
    total += (unsigned)sh.scan[i];
  }
  for (int j0 = r0; j0 < r1; j0 += 128) {
    const int j = j0 + 4 * lane;
    unsigned m[4];
    const int c = masks(j, m);
    int wt;
    unsigned at = base + (unsigned)warp_excl_scan(c, &wt);
    if (j < r1 && (j & ((1 << lhs) - 1)) == 0) lo[j >> lhs] = at;  // entries before row j
    if (idx_dst != nullptr) {  // diagnostics: the same ascending rows, for every head of the unit
      unsigned a2 = at;
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (m[e]) {
          for (int g = 0; g < nh; ++g) idx_dst[(size_t)g * p.idx_stride + a2] = j + e;
          ++a2;
        }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (m[e]) dst[at++] = (m[e] << 24) | (uint32_t)(j + e);
    base += (unsigned)wt;
  }
  if (Grp::tid() == 0)
    for (int q = S > 0 ? ((S + (1 << lhs) - 1) >> lhs) : 0; q <= 2 * p.nA; ++q) lo[q] = total;
  Grp::sync();  // sh.scan is reused by the next block scan
}

// Single-pass ordered emission for a G = 1 (MHA or group-shared) unit whose keys are on chip (r02): warp w owns
// rows [w S8, (w + 1) S8) in 1024-row segments, lane L the 32 contiguous rows [32 L, 32 L + 32) of each segment,
// read as eight uint4 groups in a lane-rotated order (conflict-free) into a 32-bit hit mask; one warp scan per
// segment and one block scan of the warp totals give every lane its ascending entry positions.  Same entries,
// offsets and diagnostics as emit_lists<1> (two passes, a scan every 128 rows: 5.9 us at 8K rows).
template <typename Grp>
__device__ void emit_lists_g1(const PipeParams& p, int u, int S, const uint32_t* ks, PipeShared& sh) {
  constexpr int SEGMAX = 2;  // segments per warp (S8 <= 2048: on-chip units of <= 16384 rows)
  const int lane = lane_id(), w = Grp::warp();
  const int lhs = 31 - __clz(p.Lc / 2);  // Lc / 2 is a power of two (>= 32)
  uint32_t* dst = p.sel + (size_t)u * p.sel_stride;
  uint32_t* lo = p.loff + (size_t)u * (2 * p.nA + 1);
  const unsigned long long Tc = sh.Tc[0];
  const uint32_t full = shared_mask(p) << 24;
  int32_t* idx_dst = nullptr;
  int nh = 0;
  if (p.idx_out != nullptr) {
    nh = unit_heads(p);
    idx_dst = p.idx_out + ((size_t)(u / p.Hkv) * p.Hq + (size_t)(u % p.Hkv) * nh) * p.idx_stride;
  }
  const int S8 = ceil_div(ceil_div(S > 0 ? S : 1, Grp::kWarps), 1024) * 1024;
  const int r0 = min(S, w * S8), r1 = min(S, r0 + S8);
  unsigned m[SEGMAX];
  int ex[SEGMAX], segoff[SEGMAX];
  int wtot = 0;
#pragma unroll
  for (int sg = 0; sg < SEGMAX; ++sg) {
    const int rb = r0 + sg * 1024 + 32 * lane;
    m[sg] = 0u;
    if (sg * 1024 < S8) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int ci = (i + lane) & 7;  // lane-rotated group: the 8 lanes of a phase hit distinct banks
        const int j = rb + 4 * ci;
        if (j < r1) {
          const uint4 kk = *reinterpret_cast<const uint4*>(ks + j);
          unsigned h4 = 0u;
#pragma unroll
          for (int e = 0; e < 4; ++e) h4 |= (j + e < r1 && comp_key(u4_at(kk, e), j + e) >= Tc ? 1u : 0u) << e;
          m[sg] |= h4 << (4 * ci);
        }
      }
    }
    int t;
    ex[sg] = warp_excl_scan(__popc(m[sg]), &t);
    segoff[sg] = wtot;
    wtot += t;
  }
  if (lane == 0) sh.scan[w] = wtot;
  Grp::sync();
  unsigned base = 0, total = 0;
#pragma unroll
  for (int i = 0; i < Grp::kWarps; ++i) {
    base += i < w ? (unsigned)sh.scan[i] : 0u;
    total += (unsigned)sh.scan[i];
  }
#pragma unroll
  for (int sg = 0; sg < SEGMAX; ++sg) {
    const int rb = r0 + sg * 1024 + 32 * lane;
    unsigned at = base + (unsigned)(segoff[sg] + ex[sg]);
    if (sg * 1024 < S8 && rb < r1 && (rb & ((1 << lhs) - 1)) == 0) lo[rb >> lhs] = at;  // entries before row rb
    unsigned mm = m[sg];
    while (mm != 0u) {
      const int b = __ffs(mm) - 1;
      mm &= mm - 1u;
      if (idx_dst != nullptr)
        for (int g = 0; g < nh; ++g) idx_dst[(size_t)g * p.idx_stride + at] = rb + b;
      dst[at++] = full | (uint32_t)(rb + b);
    }
  }
  if (Grp::tid() == 0)
    for (int q = S > 0 ? ((S + (1 << lhs) - 1) >> lhs) : 0; q <= 2 * p.nA; ++q) lo[q] = total;
  Grp::sync();  // sh.scan is reused by the next block scan
}

// ------------------------------------------------------------------ item A
template <typename T, int G_T, int VEC, int LPR1>
__device__ __forceinline__ void lead_consume(const PipeParams& p, const uint8_t* tile, int rows_here,
                                             const float (&q1)[G_T][VEC], int G, uint32_t* keys0, size_t kst,
                                             uint32_t* kl, float* approx0, uint32_t* hist, int HB, int hshift) {
  constexpr int E = sizeof(T);
  constexpr int RPW1 = 32 / LPR1;
  constexpr int U = G_T >= 4 ? 2 : 4;  // independent rows in flight per lane (register budget: 2 CTAs / SM)
  const int lane = lane_id();
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
      if (g < G) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int rr = (ps + u) * RPW1 + r;
          if (sl == 0 && rr < rows_here) {
            const uint32_t key = order_key(acc[u]);
            keys0[(size_t)g * kst + rr] = key;
            if (kl != nullptr) kl[g * p.Lc + rr] = key;
            if (approx0 != nullptr) approx0[(size_t)g * p.S_cap + rr] = acc[u];
            atomicAdd(&hist[g * HB + (key >> hshift)], 1u);
          }
        }
      }
    }
  }
}

__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ unsigned long long pk2(uint32_t lo, uint32_t hi) {
  return ((unsigned long long)hi << 32) | lo;
}

// Phase-1 stage consumed by ONE warp with one lane per row (single query
// head): RB-byte lead rows, TMA-swizzled (64 B: chunk ^ (row >> 1 & 3); 128 B:
// chunk ^ (row & 7)) so the 16 B row reads are conflict-free; packed fp32 FMA
// (two partial sums, any order is inside the fp32 tie band); the key and
// approx stores are coalesced.
template <typename T, int RB>
__device__ __forceinline__ void lead_consume_lpr(const PipeParams& p, const uint8_t* tile, int rows_here,
                                                 const unsigned long long (&q2)[RB / (2 * sizeof(T))], uint32_t* keys0,
                                                 uint32_t* kl, float* approx0, uint32_t* hist, int hshift) {
  constexpr int NCH = RB / 16;
  constexpr int RIF = RB == 64 ? 2 : 1;  // rows in flight per lane (register budget)
  const int lane = lane_id();
  for (int r0 = 0; r0 < p.r1; r0 += 32 * RIF) {
    uint4 v[RIF][NCH];
#pragma unroll
    for (int i = 0; i < RIF; ++i) {
      const int rr = r0 + 32 * i + lane;
      const int sw = RB == 64 ? ((rr >> 1) & 3) : (rr & 7);
#pragma unroll
      for (int c = 0; c < NCH; ++c)
        v[i][c] = *reinterpret_cast<const uint4*>(tile + rr * RB + ((c ^ sw) << 4));
    }
#pragma unroll
    for (int i = 0; i < RIF; ++i) {
      unsigned long long acc = 0ull;
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        const uint32_t wv[4] = {v[i][c].x, v[i][c].y, v[i][c].z, v[i][c].w};
        if constexpr (sizeof(T) == 2) {
#pragma unroll
          for (int e = 0; e < 4; ++e) acc = ffma2(pk2(wv[e] << 16, wv[e] & 0xFFFF0000u), q2[c * 4 + e], acc);
        } else {
#pragma unroll
          for (int e = 0; e < 2; ++e) acc = ffma2(pk2(wv[2 * e], wv[2 * e + 1]), q2[c * 2 + e], acc);
        }
      }
      const float sc = __uint_as_float((uint32_t)acc) + __uint_as_float((uint32_t)(acc >> 32));
      const int rr = r0 + 32 * i + lane;
      if (rr < rows_here) {
        const uint32_t key = order_key(sc);
        keys0[rr] = key;
        if (kl != nullptr) kl[rr] = key;
        if (approx0 != nullptr) approx0[rr] = sc;
        atomicAdd(&hist[key >> hshift], 1u);
      }
    }
  }
}

// Phase-1 stage consumed by ONE warp on the tensor cores (bf16 caches, query
// groups G >= 2: scores[rows x G] = K_lead[rows x dbox] . Q[dbox x G] is a real
// contraction).  q is split into three bf16 terms (hi + mid + lo == the fp32
// value), one mma n-tile each, so a lane sums its own three fragments: the
// scores carry fp32-level error, inside the tie band of the selection parity
// (SURVEY 8c O4).  Lead rows are RB = 64 / 128 B, TMA-swizzled.  Lane
// (g8, t4) holds rows {g8, g8 + 8} x heads {2 t4, 2 t4 + 1} of each 16-row block.
template <int RB, int G_T>
__device__ __forceinline__ void lead_consume_mma(const PipeParams& p, const uint8_t* tile, int rows_here,
                                                 const uint32_t (&qf)[3][4][2], int G, uint32_t* keys0, size_t kst,
                                                 uint32_t* kl, float* approx0, uint32_t* hist, int HB, int hshift) {
  constexpr int KS = RB / 32;  // k-steps of 16 bf16 columns
  const int lane = lane_id();
  const int g8 = lane >> 2, t4 = lane & 3;
  const uint32_t tb = smem_u32(tile);
  const int rA = (lane & 7) | (((lane >> 3) & 1) << 3);
  const int cA = (lane >> 4) & 1;
  for (int b0 = 0; b0 < p.r1; b0 += 16) {
    float S[3][4];
#pragma unroll
    for (int t = 0; t < 3; ++t)
#pragma unroll
      for (int i = 0; i < 4; ++i) S[t][i] = 0.f;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int r = b0 + rA, c = 2 * ks + cA;
      const int sw = RB == 64 ? ((r >> 1) & 3) : (r & 7);
      uint32_t a[4];
      ldsm_x4(tb + (uint32_t)(r * RB + ((c ^ sw) << 4)), a);
#pragma unroll
      for (int t = 0; t < 3; ++t) mma_bf16(S[t], a, qf[t][ks][0], qf[t][ks][1]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int rr = b0 + g8 + (i >> 1) * 8;
      const int h = 2 * t4 + (i & 1);
      if (h < G && rr < rows_here) {
        const float sc = (S[0][i] + S[1][i]) + S[2][i];
        const uint32_t key = order_key(sc);
        keys0[(size_t)h * kst + rr] = key;
        if (kl != nullptr) kl[h * p.Lc + rr] = key;
        if (approx0 != nullptr) approx0[(size_t)h * p.S_cap + rr] = sc;
        atomicAdd(&hist[h * HB + (key >> hshift)], 1u);
      }
    }
  }
}

template <typename T, int G_T, int VEC, bool ONCHIP = false>
__device__ int item_A(const PipeParams& p, const CUtensorMap* lead_map, int u, int c, uint8_t* ring,
                       uint8_t* wring, uint64_t* wbar, uint32_t* hist, uint32_t* kloc, uint32_t* kchip,
                       uint64_t* sbar, unsigned& sphase, RingPos& rp, PipeShared& sh) {
  constexpr int E = sizeof(T);
  const int tid = threadIdx.x, lane = lane_id(), w = warp_id();
  const int nsw = p.nst, SB = p.stage_bytes;
  const int b = u / p.Hkv, hk = u % p.Hkv, G = p.G;
  int S = p.lens[b];
  S = S < 0 ? 0 : (S > p.S_max ? p.S_max : S);  // the ticket space covers S_max <= S_cap rows
  const int nparts = ceil_div(S > 0 ? S : 1, p.La);
  if (c >= nparts) return 0;  // past this unit's length: not an arrival
  const int row0 = c * p.La;
  const int n = max(0, min(S - row0, p.La));
  const int HB = 1 << p.hbits, hshift = 32 - p.hbits;
  // a single-chunk unit (lists mode, the A-only launch) keeps its keys on chip and selects right here
  const bool onchip = ONCHIP && nparts == 1;
  for (int i = tid; i < G * HB; i += kPT) hist[i] = 0u;
  __syncthreads();
  if (n > 0) {
    const int R1 = p.r1;
    const int nbox = ceil_div(n, R1);
    const unsigned box_bytes = (unsigned)(R1 * p.dbox * E);
    const int mine = nbox > w ? ceil_div(nbox - w, kPW) : 0;  // boxes w, w + kPW, ...
    auto issue = [&](int k, const RingPos& at) {
      mbar_expect_tx(&wbar[at.slot], box_bytes);
      tma_box4d(wring + at.slot * SB, lead_map, 0, row0 + (w + k * kPW) * R1, hk, b, &wbar[at.slot]);
    };
    if (lane == 0) {
      RingPos q = rp;
      for (int k = 0; k < nsw && k < mine; ++k, q.advance(1)) issue(k, q);
    }
    const int gs = unit_heads(p);  // G, or the group whose summed query ranks the rows (shared mode, G = 1 here)
    const size_t qrow0 = (size_t)b * p.Hq + (size_t)hk * gs;
    const int nch1 = p.dbox / VEC;
    const int LPR1 = next_pow2(nch1);
    const int sl = lane % LPR1;
    float q1[G_T][VEC];
#pragma unroll
    for (int g = 0; g < G_T; ++g)
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        const int col = sl * VEC + v;
        q1[g][v] = (g < G && col < p.d && sl < nch1) ? p.q_hat[(qrow0 + g) * p.D + col] : 0.f;
      }
    uint32_t* keys_u = onchip ? kchip : p.keys + (size_t)u * G * p.kstride + row0;
    const size_t kst = onchip ? (size_t)p.La : (size_t)p.kstride;  // head stride of the key rows
    // spec: the chunk's keys also stay in shared memory ([G][Lc], the idle B-item entry region)
    auto kl0 = [&](int box) -> uint32_t* { return p.spec ? kloc + box * p.r1 : nullptr; };
    float* approx_u = p.approx_out ? p.approx_out + qrow0 * p.S_cap + row0 : nullptr;
    constexpr int E = sizeof(T);
    bool consumed = false;
    if constexpr (sizeof(T) == 2 && G_T >= 2) {
      if (p.lead_swz != 0) {  // tensor-core scores for the query group
        uint32_t qf[3][4][2];   // [part][k-step][reg]: B operand, k = 16 ks + 2 t4 + {0, 1, 8, 9}, n = head
        const int g8 = lane >> 2, t4 = lane & 3;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          float v[4], r1v[4], r2v[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int dim = 16 * ks + 2 * t4 + (i & 1) + (i >> 1) * 8;
            v[i] = (g8 < G && dim < p.d) ? p.q_hat[(qrow0 + g8) * p.D + dim] : 0.f;
            r1v[i] = v[i] - bf16_hi(v[i]);
            r2v[i] = r1v[i] - bf16_hi(r1v[i]);
          }
          qf[0][ks][0] = pack_bf16(v[0], v[1]);
          qf[0][ks][1] = pack_bf16(v[2], v[3]);
          qf[1][ks][0] = pack_bf16(r1v[0], r1v[1]);
          qf[1][ks][1] = pack_bf16(r1v[2], r1v[3]);
          qf[2][ks][0] = pack_bf16(r2v[0], r2v[1]);
          qf[2][ks][1] = pack_bf16(r2v[2], r2v[3]);
        }
        for (int k = 0; k < mine; ++k, rp.advance(1)) {
          mbar_wait(&wbar[rp.slot], rp.phase);
          const uint8_t* tile = wring + rp.slot * SB;
          const int i = w + k * kPW;
          const int rows_here = min(R1, n - i * R1);
          uint32_t* k0 = keys_u + i * R1;
          float* a0 = approx_u ? approx_u + i * R1 : nullptr;
          if (p.lead_swz == 64)
            lead_consume_mma<64, G_T>(p, tile, rows_here, qf, G, k0, kst, kl0(i), a0, hist, HB, hshift);
          else
            lead_consume_mma<128, G_T>(p, tile, rows_here, qf, G, k0, kst, kl0(i), a0, hist, HB, hshift);
          __syncwarp();
          if (lane == 0 && k + nsw < mine) issue(k + nsw, rp);
        }
        consumed = true;
      }
    }
    if (consumed || (sizeof(T) == 2 && G_T >= 2)) {  // (bf16 groups always take the tensor-core path: host)
    } else if (G_T == 1 && p.lead_swz != 0) {  // one lane per row (swizzled lead rows)
      // q as fp32 pairs, sized to the lead row so only the live half of a wider array is kept
      auto run = [&](auto rbc) {
        constexpr int RB = decltype(rbc)::value;
        constexpr int Q2 = RB / (2 * E);
        unsigned long long q2[Q2];
#pragma unroll
        for (int j = 0; j < Q2; ++j) {
          const int c0 = 2 * j, c1 = 2 * j + 1;
          const float a = c0 < p.d ? p.q_hat[qrow0 * p.D + c0] : 0.f;
          const float bq = c1 < p.d ? p.q_hat[qrow0 * p.D + c1] : 0.f;
          q2[j] = pk2(__float_as_uint(a), __float_as_uint(bq));
        }
        if (gs > 1) {  // group-shared selection: rank on the group's summed query
#pragma unroll
          for (int j = 0; j < Q2; ++j) {
            const int c0 = 2 * j, c1 = 2 * j + 1;
            const float a = c0 < p.d ? group_q(p, qrow0, gs, c0) : 0.f;
            const float bq = c1 < p.d ? group_q(p, qrow0, gs, c1) : 0.f;
            q2[j] = pk2(__float_as_uint(a), __float_as_uint(bq));
          }
        }
        for (int k = 0; k < mine; ++k, rp.advance(1)) {
          mbar_wait(&wbar[rp.slot], rp.phase);
          const uint8_t* tile = wring + rp.slot * SB;
          const int i = w + k * kPW;
          const int rows_here = min(R1, n - i * R1);
          uint32_t* k0 = keys_u + i * R1;
          float* a0 = approx_u ? approx_u + i * R1 : nullptr;
          lead_consume_lpr<T, RB>(p, tile, rows_here, q2, k0, kl0(i), a0, hist, hshift);
          __syncwarp();
          if (lane == 0 && k + nsw < mine) issue(k + nsw, rp);
        }
      };
      if (p.lead_swz == 64) run(std::integral_constant<int, 64>{});
      else run(std::integral_constant<int, 128>{});
    } else if constexpr (!(sizeof(T) == 2 && G_T >= 2))
    for (int k = 0; k < mine; ++k, rp.advance(1)) {
      mbar_wait(&wbar[rp.slot], rp.phase);
      const uint8_t* tile = wring + rp.slot * SB;
      const int i = w + k * kPW;
      const int rows_here = min(R1, n - i * R1);
      uint32_t* k0 = keys_u + i * R1;
      float* a0 = approx_u ? approx_u + i * R1 : nullptr;
      switch (LPR1) {
        case 1: lead_consume<T, G_T, VEC, 1>(p, tile, rows_here, q1, G, k0, kst, kl0(i), a0, hist, HB, hshift); break;
        case 2: lead_consume<T, G_T, VEC, 2>(p, tile, rows_here, q1, G, k0, kst, kl0(i), a0, hist, HB, hshift); break;
        case 4: lead_consume<T, G_T, VEC, 4>(p, tile, rows_here, q1, G, k0, kst, kl0(i), a0, hist, HB, hshift); break;
        case 8: lead_consume<T, G_T, VEC, 8>(p, tile, rows_here, q1, G, k0, kst, kl0(i), a0, hist, HB, hshift); break;
        case 16: lead_consume<T, G_T, VEC, 16>(p, tile, rows_here, q1, G, k0, kst, kl0(i), a0, hist, HB, hshift); break;
        default: lead_consume<T, G_T, VEC, 32>(p, tile, rows_here, q1, G, k0, kst, kl0(i), a0, hist, HB, hshift); break;
      }
      __syncwarp();  // every lane is done with the slot before it is refilled
      if (lane == 0 && k + nsw < mine) issue(k + nsw, rp);
    }
  }
  __syncthreads();
  if (p.shared > 1 && p.approx_out != nullptr && n > 0) {  // diagnostics: every head reports the group score
    const size_t r0 = ((size_t)b * p.Hq + (size_t)hk * p.shared) * p.S_cap + row0;
    for (int g = 1; g < p.shared; ++g)
      for (int j = tid; j < n; j += kPT) p.approx_out[r0 + (size_t)g * p.S_cap + j] = p.approx_out[r0 + j];
    __syncthreads();
  }
  if (p.spec && n > 0) {
    // Speculative candidates (SURVEY 8(a) R7 made cheap): this chunk is a sample of the unit, so the
    // unit's boundary bin is near the chunk's own k * n / S quantile.  Rows within kSpecW bins of
    // it go to a per-(unit, head) list; the selection uses the list when every chunk's window holds
    // the true boundary bin and falls back to scanning all keys otherwise.
    const int kb = k_of(p, S);
    const unsigned lt = (1u << lane) - 1u;
    for (int g = 0; g < G; ++g) {
      int kq = (int)(((long long)kb * n + S / 2) / S);
      kq = kq < 1 ? 1 : (kq > n ? n : kq);
      find_bin(hist + g * HB, HB, (unsigned)kq, sh);
      const int lo = max(0, sh.fb_bin - kSpecW), hi = min(HB - 1, sh.fb_bin + kSpecW);
      const size_t ug = (size_t)u * G + g;
      if (tid == 0) p.cwin[ug * p.nA + c] = (uint32_t)lo | ((uint32_t)hi << 16);
      unsigned long long* cb = p.cbuf + ug * p.ccap;
      for (int j0 = 0; j0 < n; j0 += kPT) {
        const int j = j0 + tid;
        const uint32_t key = j < n ? kloc[g * p.Lc + j] : 0u;
        const int bin = (int)(key >> hshift);
        const bool m = j < n && bin >= lo && bin <= hi;
        const unsigned bal = __ballot_sync(0xffffffffu, m);
        unsigned base = 0;
        if (lane == 0 && bal) base = atomicAdd(&p.ccnt[ug], (unsigned)__popc(bal));
        base = __shfl_sync(0xffffffffu, base, 0);
        const unsigned at = base + __popc(bal & lt);
        if (m && at < (unsigned)p.ccap) cb[at] = comp_key(key, row0 + j);
      }
    }
  }
  if constexpr (ONCHIP) if (onchip) {
    if (p.trace != nullptr && tid == 0) sh.t_sel = globaltimer();
    sel_stamp(p, u, 0);
    select_onchip<G_T>(p, u, S, kchip, p.La, hist, ring, p.nst * kPW * p.stage_bytes, sh);
    sel_stamp(p, u, 4);
    emit_lists<G_T>(p, u, S, kchip, p.La, sh);
    sel_stamp(p, u, 5);
    if (tid == 0) {  // every thread's list stores precede the release (barrier, then a gpu-scope fence)
      __threadfence();
      st_release(&p.ctrl[2 + 4 * (size_t)u + 2], 1u);
    }
    sel_stamp(p, u, 6);
    return 3;
  }
  uint32_t* gh = p.hist + (size_t)u * G * HB;
  for (int i = tid; i < G * HB; i += kPT) {
    const uint32_t v = hist[i];
    if (v) atomicAdd(&gh[i], v);
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    sh.last = atomicAdd(&p.ctrl[2 + 4 * (size_t)u], 1u) == (unsigned)nparts - 1u;
    if (sh.last) __threadfence();
  }
  __syncthreads();
  if (sh.last) {
    if (p.trace != nullptr && tid == 0) sh.t_sel = globaltimer();
    select_unit<G_T>(p, u, S, ring, hist, sbar, sphase, sh);
    return 3;
  }
  return 1;
}

// ------------------------------------------------------------------ item B
template <int G_T>
__device__ void merge_unit(const PipeParams& p, int u, int S, PipeShared& sh) {
  const int tid = threadIdx.x, lane = lane_id(), w = warp_id();
  const int G = p.G, D = p.D, ldp = D + 2;
  uint32_t* cu = p.ctrl + 2 + 4 * (size_t)u;
  const size_t qrow0 = ((size_t)(u / p.Hkv) * p.Hq) + (size_t)(u % p.Hkv) * G;
  // half-size B parts: every unit (halves == 2) or the tail units (halves == 1)
  const bool split = p.halves == 2 || (p.halves == 1 && u + p.lag >= p.units);
  const int nparts = ceil_div(S > 0 ? S : 1, p.Lc) * (split ? 2 : 1);
  const float* part = p.part + (size_t)u * 2 * p.nA * G * ldp;
  for (int i = tid; i < G * D; i += kPT) {
    const int g = i / D, col = i % D;
    float mm = -CUDART_INF_F, ll = 0.f, aa = 0.f;
    for (int q = 0; q < nparts; ++q) {
      const float* f = part + ((size_t)q * G + g) * ldp;
      float s1, s2;
      merge_state(mm, ll, __ldcg(&f[D]), __ldcg(&f[D + 1]), s1, s2);
      aa = aa * s1 + __ldcg(&f[col]) * s2;
    }
    p.out[(qrow0 + g) * D + col] = ll > 0.f ? aa / ll : 0.f;
    if (col == 0) {
      sh.gm[g] = mm;
      sh.gl[g] = ll;
    }
  }
  __syncthreads();
  if (p.weights_out != nullptr && p.lists) {  // lists mode: pipe_weights_kernel finishes the weights
    if (tid < G) {
      p.ml[((size_t)u * G + tid) * 2] = sh.gm[tid];
      p.ml[((size_t)u * G + tid) * 2 + 1] = sh.gl[tid];
    }
  } else if (p.weights_out != nullptr) {  // softmax weights of each head's selection, ascending rows
    const unsigned lt = (1u << lane) - 1u;
    const int Gk = (G_T > 1 && p.shared > 1) ? 1 : G;  // group-shared: one key array and threshold per unit
    for (int g = 0; g < G; ++g) {
      const int gk = Gk == 1 ? 0 : g;
      const unsigned long long Tc = __ldcg(&p.tcs[(size_t)u * Gk + gk]);
      const uint32_t* keys = p.keys + ((size_t)u * Gk + gk) * p.kstride;
      const float M = sh.gm[g], invL = 1.f / sh.gl[g];
      const float* lg = p.logits + ((size_t)u * G + g) * p.S_cap;
      float* dst = p.weights_out + (qrow0 + g) * p.idx_stride;
      unsigned emitted = 0;
      for (int j0 = 0; j0 < S; j0 += kPT) {
        const int j = j0 + tid;
        const bool on = j < S && comp_key(__ldcg(&keys[j]), j) >= Tc;
        const unsigned bal = __ballot_sync(0xffffffffu, on);
        if (lane == 0) sh.wcnt[w][0] = __popc(bal);
        __syncthreads();
        unsigned before = 0, tot = 0;
        for (int ww = 0; ww < kPW; ++ww) {
          before += ww < w ? sh.wcnt[ww][0] : 0;
          tot += sh.wcnt[ww][0];
        }
        if (on) dst[emitted + before + __popc(bal & lt)] = exp2f(__ldcg(&lg[j]) - M) * invL;
        emitted += tot;
        __syncthreads();
      }
    }
  }
  if (tid == 0) {
    cu[1] = 0u;
    cu[2] = 0u;
  }
}

template <typename T, int G_T, int VEC, int D_T>
__device__ void stream_B_simt(const PipeParams& p, const CUtensorMap* krow_map, const CUtensorMap* vrow_map, int u,
                              int n, int row_base, size_t qrow0, const uint32_t* ents, const float* apx, uint8_t* wring,
                              uint64_t* wbar, RingPos& rp, float* wpart) {
  constexpr int E = sizeof(T);
  constexpr int LPR3 = D_T / VEC;  // lanes per V row
  constexpr int RPW3 = 32 / LPR3;
  constexpr int ROWB = D_T * E;
  const int lane = lane_id(), w = warp_id();
  const int nsw = p.nst, SB = p.stage_bytes;
  const int G = p.G, D = D_T;
  const bool split = p.split_k != 0;
  const int kcol0 = split ? p.d : 0;  // first gathered K column
  const int KW = D - kcol0;           // gathered K columns
  const int KROWB = KW * E;
  const int R3 = p.r3;
  const int nstage = ceil_div(n, R3);
  const unsigned stage_bytes = (unsigned)(R3 * (KROWB + ROWB));
  const bool want_logits = p.weights_out != nullptr;
  const int mine = nstage > w ? ceil_div(nstage - w, kPW) : 0;  // stages w, w + kPW, ...
  auto issue = [&](int k, const RingPos& at) {
    const int st = w + k * kPW;
    uint8_t* dst = wring + at.slot * SB;
    if (lane == 0) mbar_expect_tx(&wbar[at.slot], stage_bytes);
    int row = -1;  // lane t < R3 resolves row t of the stage; -1 = out of bounds, zero-filled
    const int t = st * R3 + lane;
    if (lane < R3 && t < n) row = row_base + (int)(ents[t] & 0xFFFFFFu);
    for (int qq = 0; qq < R3 / 4; ++qq) {
      const int a0 = __shfl_sync(0xffffffffu, row, 4 * qq);
      const int a1 = __shfl_sync(0xffffffffu, row, 4 * qq + 1);
      const int a2 = __shfl_sync(0xffffffffu, row, 4 * qq + 2);
      const int a3 = __shfl_sync(0xffffffffu, row, 4 * qq + 3);
      if (lane == 0) {
        tma_gather4(dst + qq * 4 * KROWB, krow_map, kcol0, a0, a1, a2, a3, &wbar[at.slot]);
        tma_gather4(dst + R3 * KROWB + qq * 4 * ROWB, vrow_map, 0, a0, a1, a2, a3, &wbar[at.slot]);
      }
    }
  };
  {
    RingPos qp = rp;
    for (int k = 0; k < nsw && k < mine; ++k, qp.advance(1)) issue(k, qp);
  }
  float acc[G_T][VEC];
  float m[G_T], l[G_T];
#pragma unroll
  for (int g = 0; g < G_T; ++g) {
    m[g] = -CUDART_INF_F;
    l[g] = 0.f;
#pragma unroll
    for (int v = 0; v < VEC; ++v) acc[g][v] = 0.f;
  }
  const int r = lane / LPR3, sl = lane % LPR3;
  const bool k_on = sl * VEC < KW;
  float q3[G_T][VEC];
#pragma unroll
  for (int g = 0; g < G_T; ++g)
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      const int col = kcol0 + sl * VEC + v;
      q3[g][v] = (g < G && k_on && col < D) ? p.q_hat[(qrow0 + g) * D + col] * p.qscale : 0.f;
    }
  constexpr int U = 2;  // rows per lane slot whose logits are formed before the softmax updates
  for (int k = 0; k < mine; ++k, rp.advance(1)) {
    mbar_wait(&wbar[rp.slot], rp.phase);
    const int st = w + k * kPW;
    const uint8_t* kt = wring + rp.slot * SB;
    const uint8_t* vt = kt + R3 * KROWB;
    for (int ps = 0; ps < R3 / RPW3; ps += U) {  // host: (R3 / RPW3) % U == 0
      float x[U][G_T];
      int jr[U];
      unsigned msk[U];
#pragma unroll
      for (int uu = 0; uu < U; ++uu) {
        const int rr = (ps + uu) * RPW3 + r;
        const int t = st * R3 + rr;
        const bool ok = t < n;
        const uint32_t e = ok ? ents[t] : 0u;
        jr[uu] = (int)(e & 0xFFFFFFu);
        msk[uu] = e >> 24;
        float kx[VEC];
        if (k_on) lds_chunk<T, VEC>(kt + rr * KROWB + sl * VEC * E, kx);
        else
#pragma unroll
          for (int v = 0; v < VEC; ++v) kx[v] = 0.f;
#pragma unroll
        for (int g = 0; g < G_T; ++g) {
          float s = 0.f;
#pragma unroll
          for (int v = 0; v < VEC; ++v) s = fmaf(q3[g][v], kx[v], s);
          s = sum_lanes<LPR3>(s);
          if (split && ok && g < G) s += apx[g * p.Lc + t];
          x[uu][g] = s;
        }
      }
#pragma unroll
      for (int uu = 0; uu < U; ++uu) {
        const int rr = (ps + uu) * RPW3 + r;
        float vx[VEC];
        lds_chunk<T, VEC>(vt + rr * ROWB + sl * VEC * E, vx);
#pragma unroll
        for (int g = 0; g < G_T; ++g) {
          if (msk[uu] & (1u << g)) {
            const float xv = x[uu][g];
            if (want_logits && sl == 0) p.logits[((size_t)u * G + g) * p.S_cap + jr[uu]] = xv;
            const float mn = fmaxf(m[g], xv);
            const float sc = exp2f(m[g] - mn);
            const float pe = exp2f(xv - mn);
            l[g] = l[g] * sc + pe;
            m[g] = mn;
#pragma unroll
            for (int v = 0; v < VEC; ++v) acc[g][v] = fmaf(pe, vx[v], acc[g][v] * sc);
          }
        }
      }
    }
    __syncwarp();
    if (k + nsw < mine) issue(k + nsw, rp);
  }

  // merge lanes sharing columns, then warps in fixed order, into this part's state
#pragma unroll
  for (int g = 0; g < G_T; ++g) {
    for (int off = LPR3; off < 32; off <<= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, m[g], off);
      const float l2 = __shfl_xor_sync(0xffffffffu, l[g], off);
      float s1, s2;
      merge_state(m[g], l[g], m2, l2, s1, s2);
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        const float a2 = __shfl_xor_sync(0xffffffffu, acc[g][v], off);
        acc[g][v] = acc[g][v] * s1 + a2 * s2;
      }
    }
  }
  const int ldp = D + 2;
  __syncthreads();
  if (r == 0) {
#pragma unroll
    for (int g = 0; g < G_T; ++g) {
      if (g >= G) break;
      float* dstp = wpart + ((size_t)w * G_T + g) * ldp;
#pragma unroll
      for (int v = 0; v < VEC; ++v) dstp[sl * VEC + v] = acc[g][v];
      if (sl == 0) {
        dstp[D] = m[g];
        dstp[D + 1] = l[g];
      }
    }
  }
}

// Phase 3 on the tensor cores (bf16 caches).  A stage is 8 gathered rows
// (4 KB at D = 128: many small stages keep 16 warps per SM issuing gathers,
// tools/gatherbench.cu), 128B/64B-swizzled by TMA so ldmatrix is conflict-free:
//   V   as 128 B row halves (NH x 1 KB), then
//   K   columns [kc0, D): `ka` 128 B pieces (1 KB each) + `kb` 64 B piece (512 B).
// kc0 = 0, or d with split-K: the phase-1 partial score q[:d].K[:d] (from the
// keys) is added to the logit and the leading d columns are not fetched again.
// Per stage, with the 8 rows as M rows 0..7 of m16n8k16 (rows 8..15 zero):
//   S^T[8 x 8] = K[8 x D'] . Qc[D' x 8]  and  O^T[D x 8] += V^T[D x 8] . P^T[8 x 8]
// MHA (G = 1, kc0 = 0) folds the head dimension's upper half into the idle rows instead (kFold): M rows
// 8..15 of q.K are the same 8 rows' dims [D/2, D) against query columns 2..3 (hi / lo of q[D/2:]), and the
// k rows 8..15 of P.V are the stage rows again against the upper dims, P in columns 2..3 -- every mma
// does useful work, half as many mmas per row (r03).
// (fp32 accumulate).  Columns carry (head, hi / lo part): q * qscale and the
// softmax weights are split into two bf16 terms, so both products keep ~2^-17
// relative accuracy.  G <= 4: column 2h + part;  G == 8: columns = heads, hi
// and lo in two mmas.
template <int G_T, int D_T, int KC0>
__device__ void stream_B_mma(const PipeParams& p, const CUtensorMap* krow_map, const CUtensorMap* vrow_map,
                             const CUtensorMap* krow64_map, int u, int n, int row_base, size_t qrow0,
                             const uint32_t* ents, const float* apx, uint8_t* wring, uint64_t* wbar, RingPos& rp,
                             float* wpart) {
  constexpr int NH = D_T / 64;             // 128 B row halves of V
  constexpr int KS = D_T / 16;             // max k-steps of q.K == m-tiles of P.V
  constexpr int R = 8;                     // rows per stage
  constexpr int HW = R * 128;              // bytes of one 128 B-row block (one swizzle atom)
  constexpr int NHL = G_T == 8 ? 2 : 1;    // heads per lane
  constexpr bool kSplitCols = G_T < 8;
  const int lane = lane_id(), w = warp_id();
  const int G = p.G;
  const int nsw = p.nst, SB = p.stage_bytes;
  const int g8 = lane >> 2, t4 = lane & 3;
  constexpr bool split = KC0 > 0;
  constexpr int kc0 = KC0;                 // first gathered K column (compile time: keeps the loops static)
  constexpr int ka = (D_T - kc0) / 64, kbp = ((D_T - kc0) % 64) / 32;  // K pieces: 128 B and 64 B
  constexpr int KSK = (D_T - kc0) / 16;    // k-steps of q.K over the gathered columns
  const int nstage = ceil_div(n, R);
  const unsigned stage_bytes = (unsigned)(R * (D_T + (D_T - kc0)) * 2);
  const bool want_logits = p.weights_out != nullptr;
  const int mine = nstage > w ? ceil_div(nstage - w, kPW) : 0;  // stages w, w + kPW, ...
  auto issue = [&](int k, const RingPos& at) {
    const int st = w + k * kPW;
    uint8_t* dst = wring + at.slot * SB;
    if (lane == 0) mbar_expect_tx(&wbar[at.slot], stage_bytes);
    int row = -1;  // -1: out of bounds, zero-filled
    const int t = st * R + lane;
    if (lane < R && t < n) row = row_base + (int)(ents[t] & 0xFFFFFFu);
    // warp-uniform operands (tma_gather4_u): no per-instruction waterfall loop around the TMA issues
    const uint32_t ds = __shfl_sync(0xffffffffu, smem_u32(dst), 0);
    const uint32_t bs = __shfl_sync(0xffffffffu, smem_u32(&wbar[at.slot]), 0);
#pragma unroll
    for (int qq = 0; qq < R / 4; ++qq) {
      const int a0 = __shfl_sync(0xffffffffu, row, 4 * qq);
      const int a1 = __shfl_sync(0xffffffffu, row, 4 * qq + 1);
      const int a2 = __shfl_sync(0xffffffffu, row, 4 * qq + 2);
      const int a3 = __shfl_sync(0xffffffffu, row, 4 * qq + 3);
      if (lane == 0) {
#pragma unroll
        for (int h = 0; h < NH; ++h)
          tma_gather4_u(ds + h * HW + qq * 512, vrow_map, 64 * h, a0, a1, a2, a3, bs);
#pragma unroll
        for (int j = 0; j < ka; ++j)
          tma_gather4_u(ds + (NH + j) * HW + qq * 512, krow_map, kc0 + 64 * j, a0, a1, a2, a3, bs);
        if constexpr (kbp > 0)
          tma_gather4_u(ds + (NH + ka) * HW + qq * 256, krow64_map, D_T - 32, a0, a1, a2, a3, bs);
      }
    }
  };
  {
    RingPos qp = rp;
    for (int k = 0; k < nsw && k < mine; ++k, qp.advance(1)) issue(k, qp);
  }
  // B operand of S^T = K . Qc: lane holds Qc[16 ks + 2 t4 + {0, 1, 8, 9}][g8]
  // (kFold: column g8 = 2 half + part holds q[half * D / 2 + 16 ks + ...], half in {0, 1}; KF k-steps)
  constexpr bool kFold = G_T == 1 && KC0 == 0;
  constexpr int KF = kFold ? KS / 2 : KS;  // k-steps of q.K == m-tiles of P.V
  uint32_t qb[KS][2], ql[G_T == 8 ? KS : 1][2];
#pragma unroll
  for (int ks = 0; ks < KS; ++ks) {
    const int k0 = kFold ? (g8 >> 1) * (D_T / 2) + 16 * ks + 2 * t4 : kc0 + 16 * ks + 2 * t4;
    const int head = kFold ? (g8 < 4 && ks < KF ? 0 : G) : (kSplitCols ? (g8 >> 1) : g8);
    float v[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int dim = k0 + (i & 1) + (i >> 1) * 8;
      v[i] = (head < G && ks < KSK) ? p.q_hat[(qrow0 + head) * D_T + dim] * p.qscale : 0.f;
    }
    if (kSplitCols) {
      const bool lo = g8 & 1;
#pragma unroll
      for (int i = 0; i < 4; ++i) v[i] = lo ? bf16_lo(v[i]) : v[i];
      qb[ks][0] = pack_bf16(v[0], v[1]);
      qb[ks][1] = pack_bf16(v[2], v[3]);
    } else {
      qb[ks][0] = pack_bf16(v[0], v[1]);
      qb[ks][1] = pack_bf16(v[2], v[3]);
      ql[ks][0] = pack_bf16(bf16_lo(v[0]), bf16_lo(v[1]));
      ql[ks][1] = pack_bf16(bf16_lo(v[2]), bf16_lo(v[3]));
    }
  }
  float O[KS][4];
#pragma unroll
  for (int mt = 0; mt < KS; ++mt)
#pragma unroll
    for (int i = 0; i < 4; ++i) O[mt][i] = 0.f;
  float m[NHL], l[NHL];
#pragma unroll
  for (int j = 0; j < NHL; ++j) {
    m[j] = -CUDART_INF_F;
    l[j] = 0.f;
  }
  const int rX = lane & 7;            // ldmatrix.x2 row (lanes 0..15 address two 8x8 matrices)
  const int cX = (lane >> 3) & 1;     // second matrix: +8 columns (K) / +8 dims (V)
  for (int k = 0; k < mine; ++k, rp.advance(1)) {
    mbar_wait(&wbar[rp.slot], rp.phase);
    const int st = w + k * kPW;
    const uint32_t sb = smem_u32(wring + rp.slot * SB);
    float S[4] = {0.f, 0.f, 0.f, 0.f}, S2[4] = {0.f, 0.f, 0.f, 0.f};
    if constexpr (kFold) {  // x4: rows 0..7 x {dims [16 ks, +16), dims [D/2 + 16 ks, +16)}
      const int hiX = (lane >> 3) & 1, khX = lane >> 4;
#pragma unroll
      for (int ks = 0; ks < KF; ++ks) {
        const int dim0 = hiX * (D_T / 2) + 16 * ks + 8 * khX;
        uint32_t a[4];
        asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
                     : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3])
                     : "r"(swz128(sb + (NH + (dim0 >> 6)) * HW, rX, (dim0 & 63) >> 3)));
        mma_bf16((ks & 1) ? S2 : S, a, qb[ks][0], qb[ks][1]);
      }
    }
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      if constexpr (!kFold) {
        if (ks >= KSK) continue;
        uint32_t addr;
        if (ks < 4 * ka) {  // 128 B piece ks / 4
          addr = swz128(sb + (NH + (ks >> 2)) * HW, rX, ((ks & 3) << 1) | cX);
        } else {            // trailing 64 B piece (64B swizzle: chunk ^ (row >> 1 & 3))
          const int c = ((ks - 4 * ka) << 1) | cX;
          addr = sb + (NH + ka) * HW + rX * 64 + ((c ^ ((rX >> 1) & 3)) << 4);
        }
        uint32_t a2[2];
        asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0, %1}, [%2];"
                     : "=r"(a2[0]), "=r"(a2[1])
                     : "r"(addr));
        const uint32_t a[4] = {a2[0], 0u, a2[1], 0u};
        if (kSplitCols) {  // two accumulators (even / odd k-steps): half the dependent mma chain
          mma_bf16((ks & 1) ? S2 : S, a, qb[ks][0], qb[ks][1]);
        } else {
          mma_bf16(S, a, qb[ks][0], qb[ks][1]);
          mma_bf16(S2, a, ql[ks][0], ql[ks][1]);
        }
      }
    }
    const int tA = st * R + g8;
    const uint32_t eA = tA < n ? ents[tA] : 0u;
    float x[NHL], pr[NHL], sc[NHL];
#pragma unroll
    for (int j = 0; j < NHL; ++j) {
      // (kFold: lane t4 = 0 holds row g8's lower-half sum, t4 = 1 the upper half (M row g8 + 8, columns
      // 2..3); both lanes then carry the row's score and the same softmax state)
      const int head = kFold ? (t4 < 2 ? 0 : G) : (kSplitCols ? t4 : 2 * t4 + j);
      if constexpr (kFold) {
        x[j] = t4 == 0 ? (S[0] + S2[0]) + (S[1] + S2[1]) : (S[2] + S2[2]) + (S[3] + S2[3]);
        x[j] += __shfl_xor_sync(0xffffffffu, x[j], 1);
      } else {
        x[j] = kSplitCols ? (S[0] + S2[0]) + (S[1] + S2[1]) : S[j] + S2[j];
      }
      const bool ok = head < G && ((eA >> (24 + head)) & 1u);
      if (split && ok) x[j] += apx[head * p.Lc + tA];  // phase-1 partial over the first d columns
      float tm = ok ? x[j] : -CUDART_INF_F;
      tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, 4));
      tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, 8));
      tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, 16));
      const float mn = fmaxf(m[j], tm);
      sc[j] = (mn == -CUDART_INF_F) ? 1.f : exp2f(m[j] - mn);
      pr[j] = ok ? exp2f(x[j] - mn) : 0.f;
      l[j] = l[j] * sc[j] + pr[j];
      m[j] = mn;
      if (want_logits && ok && (!kFold || t4 == 0)) p.logits[((size_t)u * G + head) * p.S_cap + (eA & 0xFFFFFFu)] = x[j];
    }
    bool same = true;
#pragma unroll
    for (int j = 0; j < NHL; ++j) same &= sc[j] == 1.f;
    if (!__all_sync(0xffffffffu, same)) {
#pragma unroll
      for (int mt = 0; mt < KF; ++mt) {
        O[mt][0] *= sc[0];
        O[mt][2] *= sc[0];
        O[mt][1] *= sc[NHL - 1];
        O[mt][3] *= sc[NHL - 1];
      }
    }
    // B operand P^T: lane holds P[rows 2 t4, 2 t4 + 1][column g8] (rows 8..15 do not exist);
    // (row r, lane head slot) lives in lane r * 4 + head slot
    const int src0 = (2 * t4) * 4 + (kFold ? 0 : (g8 >> 1)), src1 = src0 + 4;
    uint32_t pb, pl = 0u;
    if constexpr (kFold) {  // k rows 0..7: P in columns 0..1; k rows 8..15 (same rows, upper dims): columns 2..3
      const float v0 = __shfl_sync(0xffffffffu, pr[0], src0);
      const float v1 = __shfl_sync(0xffffffffu, pr[0], src1);
      const bool lo = g8 & 1;
      const uint32_t pk = pack_bf16(lo ? bf16_lo(v0) : v0, lo ? bf16_lo(v1) : v1);
      pb = g8 < 2 ? pk : 0u;
      pl = (g8 == 2 || g8 == 3) ? pk : 0u;
#pragma unroll
      for (int mt = 0; mt < KF; ++mt) {  // x4.trans: V^T dims [16 mt, +16) and [D/2 + 16 mt, +16) of rows 0..7
        const int dim = 16 * mt + (cX << 3) + (lane >> 4) * (D_T / 2);
        uint32_t a[4];
        asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
                     : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3])
                     : "r"(swz128(sb + (dim >> 6) * HW, rX, (dim & 63) >> 3)));
        mma_bf16(O[mt], a, pb, pl);
      }
      __syncwarp();
      if (k + nsw < mine) issue(k + nsw, rp);
      continue;
    } else if (kSplitCols) {
      const float v0 = __shfl_sync(0xffffffffu, pr[0], src0);
      const float v1 = __shfl_sync(0xffffffffu, pr[0], src1);
      const bool lo = g8 & 1;
      pb = pack_bf16(lo ? bf16_lo(v0) : v0, lo ? bf16_lo(v1) : v1);
    } else {
      const bool odd = g8 & 1;  // column g8 = head; element j = head & 1 of the source lane
      const float a0 = __shfl_sync(0xffffffffu, pr[0], src0), b0 = __shfl_sync(0xffffffffu, pr[NHL - 1], src0);
      const float a1 = __shfl_sync(0xffffffffu, pr[0], src1), b1 = __shfl_sync(0xffffffffu, pr[NHL - 1], src1);
      const float v0 = odd ? b0 : a0, v1 = odd ? b1 : a1;
      pb = pack_bf16(v0, v1);
      pl = pack_bf16(bf16_lo(v0), bf16_lo(v1));
    }
#pragma unroll
    for (int mt = 0; mt < KS; ++mt) {
      const int dim = 16 * mt + (cX << 3);
      uint32_t a2[2];
      asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0, %1}, [%2];"
                   : "=r"(a2[0]), "=r"(a2[1])
                   : "r"(swz128(sb + (dim >> 6) * HW, rX, (dim & 63) >> 3)));
      const uint32_t a[4] = {a2[0], a2[1], 0u, 0u};
      mma_bf16(O[mt], a, pb, 0u);
      if (!kSplitCols) mma_bf16(O[mt], a, pl, 0u);
    }
    __syncwarp();
    if (k + nsw < mine) issue(k + nsw, rp);
  }
#pragma unroll
  for (int j = 0; j < NHL; ++j) {
    l[j] += __shfl_xor_sync(0xffffffffu, l[j], 4);
    l[j] += __shfl_xor_sync(0xffffffffu, l[j], 8);
    l[j] += __shfl_xor_sync(0xffffffffu, l[j], 16);
  }
  __syncthreads();  // wpart aliases the ring: every warp has drained its slots
#pragma unroll
  for (int j = 0; j < NHL; ++j) {
    const int head = kSplitCols ? t4 : 2 * t4 + j;
    if (kFold && t4 < 2) {  // lane t4 holds output dims t4 * D / 2 + [0, D / 2)
      float* dstp = wpart + (size_t)w * (D_T + 2) + t4 * (D_T / 2);
#pragma unroll
      for (int mt = 0; mt < KF; ++mt) {
        dstp[16 * mt + g8] = O[mt][0] + O[mt][1];
        dstp[16 * mt + g8 + 8] = O[mt][2] + O[mt][3];
      }
      if (g8 == 0 && t4 == 0) {
        dstp[D_T] = m[j];
        dstp[D_T + 1] = l[j];
      }
    } else if (!kFold && head < G) {
      float* dstp = wpart + ((size_t)w * G_T + head) * (D_T + 2);
#pragma unroll
      for (int mt = 0; mt < KS; ++mt) {
        if (kSplitCols) {
          dstp[16 * mt + g8] = O[mt][0] + O[mt][1];
          dstp[16 * mt + g8 + 8] = O[mt][2] + O[mt][3];
        } else {
          dstp[16 * mt + g8] = O[mt][j];
          dstp[16 * mt + g8 + 8] = O[mt][2 + j];
        }
      }
      if (g8 == 0) {
        dstp[D_T] = m[j];
        dstp[D_T + 1] = l[j];
      }
    }
  }
}

// B(u, q): rows [q * Lc, (q + 1) * Lc).  kNB 128-row blocks per warp.
template <typename T, int G_T, int VEC, int D_T, bool BIG>
__device__ int item_B(const PipeParams& p, const CUtensorMap* krow_map, const CUtensorMap* vrow_map,
                      const CUtensorMap* krow64_map, int u, int q, int half, uint8_t* ring, uint8_t* wring, uint64_t* wbar, uint32_t* ents, RingPos& rp,
                      PipeShared& sh) {
  constexpr int E = sizeof(T);
  constexpr int LPR3 = D_T / VEC;  // lanes per V row
  constexpr int RPW3 = 32 / LPR3;
  constexpr int ROWB = D_T * E;
  constexpr int kNB = pipe_blocks_per_warp(G_T, BIG);  // Lc == kNB * 128 * kPW (host)
  const int tid = threadIdx.x, lane = lane_id(), w = warp_id();
  const int nsw = p.nst, SB = p.stage_bytes;
  const int b = u / p.Hkv, hk = u % p.Hkv, G = p.G, D = D_T;
  int S = p.lens[b];
  S = S < 0 ? 0 : (S > p.S_max ? p.S_max : S);  // the ticket space covers S_max <= S_cap rows
  const int nparts = ceil_div(S > 0 ? S : 1, p.Lc);
  if (q >= nparts) return 0;  // past this unit's length: not an arrival
  // full part q = rows [q Lc, (q + 1) Lc); the tail units' half parts (half = 0 / 1) cover Lc / 2 rows each
  const int span = half < 0 ? p.Lc : p.Lc / 2;
  const int row0 = q * p.Lc + (half > 0 ? span : 0);
  const int nrows = max(0, min(S - row0, span));
  const int pidx = half < 0 ? q : 2 * q + half;             // partial-state slot
  const int narrive = half < 0 ? nparts : 2 * nparts;     // B items of this unit
  uint32_t* cu = p.ctrl + 2 + 4 * (size_t)u;
  if (tid == 0 && !p.dense) {
    // a unit's selection is published by a CTA that is already running, so the wait always ends; the
    // guard turns a broken invariant into an error instead of a hung GPU (p.spin_ns, 0 = no guard)
    unsigned spins = 0;
    long long t_start = 0;
    while (ld_acquire(&cu[2]) == 0u) {
      __nanosleep(64);
      if ((++spins & 1023u) == 0u && p.spin_ns > 0) {
        const long long now = globaltimer();
        if (t_start == 0) t_start = now;
        else if (now - t_start > p.spin_ns) {
          printf("loki pipe: unit %d never became ready (block %d)\n", u, (int)blockIdx.x);
          __trap();
        }
      }
    }
  }
  if (p.trace != nullptr && tid == 0) sh.t_sel = globaltimer();  // ready observed (trace: wait vs work)
  __syncthreads();
  const bool split = p.split_k != 0;
  const size_t qrow0 = (size_t)b * p.Hq + (size_t)hk * G;
  float* apx = reinterpret_cast<float*>(ents + p.Lc);  // [G][Lc] phase-1 partial logits, log2 domain
  // this part's selected rows, ascending, with head masks: one L2 round trip for the keys
  int n = 0;
  if (p.dense) {  // dense decode (vanilla_attention): every row of the part, every head
    const uint32_t full = ((1u << G) - 1u) << 24;
    n = nrows;
    for (int i = tid; i < n; i += kPT) ents[i] = full | (uint32_t)(row0 + i);
  } else if (nrows > 0 && p.lists) {  // the A item published this unit's ordered entries and their part offsets
    const uint32_t* lo = p.loff + (size_t)u * (2 * p.nA + 1);
    const int h0 = half < 0 ? 2 * q : 2 * q + half;
    const int e0 = (int)__ldcg(&lo[h0]);
    n = (int)__ldcg(&lo[h0 + (half < 0 ? 2 : 1)]) - e0;
    const uint32_t* src = p.sel + (size_t)u * p.sel_stride + e0;
    for (int i = tid; i < n; i += kPT) ents[i] = __ldcg(&src[i]);
  } else if (nrows > 0) {
    // group-shared selection: one key array and one threshold per unit; a selected row serves every head
    const int Gk = (G_T > 1 && p.shared > 1) ? 1 : G;
    const uint32_t* kbase = p.keys + (size_t)u * Gk * p.kstride;
    unsigned long long Tc[G_T];
#pragma unroll
    for (int g = 0; g < G_T; ++g) Tc[g] = g < Gk ? __ldcg(&p.tcs[(size_t)u * Gk + g]) : ~0ull;
    const int wr0 = row0 + w * kNB * 128;  // this warp's rows [wr0, wr0 + kNB * 128)
    const int rend = row0 + nrows;
    uint4 kk[kNB][G_T];
#pragma unroll
    for (int bq = 0; bq < kNB; ++bq) {
      const int jb = wr0 + bq * 128 + 4 * lane;
#pragma unroll
      for (int g = 0; g < G_T; ++g)
        kk[bq][g] = (g < Gk && jb < rend) ? ld_keys4(kbase + (size_t)g * p.kstride, jb) : make_uint4(0u, 0u, 0u, 0u);
    }
    unsigned m[kNB][4];
    int ns = 0;
#pragma unroll
    for (int bq = 0; bq < kNB; ++bq)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int j = wr0 + bq * 128 + 4 * lane + e;
        unsigned mm = 0;
#pragma unroll
        for (int g = 0; g < G_T; ++g)
          if (g < Gk && j < rend && comp_key(u4_at(kk[bq][g], e), j) >= Tc[g]) mm |= 1u << g;
        if (G_T > 1 && Gk != G && mm) mm = (1u << G) - 1u;
        m[bq][e] = mm;
        ns += mm != 0;
      }
    int wtot;
    const int lpos = warp_excl_scan(ns, &wtot);
    if (lane == 0) sh.wcnt[w][0] = wtot;
    __syncthreads();
    int pos = lpos;
    for (int ww = 0; ww < kPW; ++ww) {
      pos += ww < w ? sh.wcnt[ww][0] : 0;
      n += sh.wcnt[ww][0];
    }
    // lane order inside a warp: block-major (bq), then lane, then e
    int bpos[kNB];
    {
      int acc = 0;
#pragma unroll
      for (int bq = 0; bq < kNB; ++bq) {
        int c = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) c += m[bq][e] != 0;
        int tot;
        const int ex = warp_excl_scan(c, &tot);
        bpos[bq] = pos - lpos + acc + ex;  // warp base + earlier blocks + earlier lanes
        acc += tot;
      }
    }
#pragma unroll
    for (int bq = 0; bq < kNB; ++bq) {
      int qd = bpos[bq];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (m[bq][e]) {
          const int j = wr0 + bq * 128 + 4 * lane + e;
          ents[qd] = (m[bq][e] << 24) | (uint32_t)j;
          if (split)
#pragma unroll
            for (int g = 0; g < G_T; ++g)
              if (g < G) apx[g * p.Lc + qd] = key_to_float(u4_at(kk[bq][g], e)) * p.qscale;
          ++qd;
        }
      }
    }
    if (p.idx_out != nullptr) {  // per-head ascending indices at the part's published offset
#pragma unroll
      for (int g = 0; g < G_T; ++g) {
        if (g >= G) break;
        int cg = 0;
#pragma unroll
        for (int bq = 0; bq < kNB; ++bq)
#pragma unroll
          for (int e = 0; e < 4; ++e) cg += (m[bq][e] >> g) & 1u;
        const int gtot = __reduce_add_sync(0xffffffffu, cg);
        if (lane == 0) sh.wcnt[w][1 + g] = gtot;
      }
      __syncthreads();
#pragma unroll
      for (int g = 0; g < G_T; ++g) {
        if (g >= G) break;
        int base = (int)__ldcg(&p.poff[((size_t)u * G + g) * 2 * p.nA + row0 / (p.Lc / 2)]);
        for (int ww = 0; ww < w; ++ww) base += sh.wcnt[ww][1 + g];
        int32_t* dst = p.idx_out + (qrow0 + g) * p.idx_stride;
#pragma unroll
        for (int bq = 0; bq < kNB; ++bq) {
          int c = 0;
#pragma unroll
          for (int e = 0; e < 4; ++e) c += (m[bq][e] >> g) & 1u;
          int tot;
          int qd = base + warp_excl_scan(c, &tot);
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if ((m[bq][e] >> g) & 1u) dst[qd++] = wr0 + bq * 128 + 4 * lane + e;
          base += tot;
        }
      }
    }
  }
  __syncthreads();

  const int ldp = D + 2;
  float* wpart = reinterpret_cast<float*>(ring);  // [kPW][G_T][D + 2]; every ring slot has been consumed
  const int row_base = (int)((long long)b * p.row_sb + (long long)hk * p.row_sh);
  if constexpr (sizeof(T) == 2) {  // bf16: always the tensor-core phase 3 (host sets p.mma)
    if constexpr (D_T == 128 && G_T <= 4) {
      if (p.split_k)  // host: split-K on the tensor-core path means d == 32
        stream_B_mma<G_T, D_T, 32>(p, krow_map, vrow_map, krow64_map, u, n, row_base, qrow0, ents, apx, wring, wbar,
                                   rp, wpart);
      else
        stream_B_mma<G_T, D_T, 0>(p, krow_map, vrow_map, krow64_map, u, n, row_base, qrow0, ents, apx, wring, wbar,
                                  rp, wpart);
    } else {
      stream_B_mma<G_T, D_T, 0>(p, krow_map, vrow_map, krow64_map, u, n, row_base, qrow0, ents, apx, wring, wbar, rp,
                                wpart);
    }
  }
  else
    stream_B_simt<T, G_T, VEC, D_T>(p, krow_map, vrow_map, u, n, row_base, qrow0, ents, apx, wring, wbar, rp, wpart);
  __syncthreads();
  float* gpart = p.part + (((size_t)u * 2 * p.nA + pidx) * G) * ldp;
  for (int i = tid; i < G * ldp; i += kPT) {
    const int g = i / ldp, col = i % ldp;
    float mm = -CUDART_INF_F, ll = 0.f, aa = 0.f;
    for (int ww = 0; ww < kPW; ++ww) {
      const float* src = wpart + ((size_t)ww * G_T + g) * ldp;
      float s1, s2;
      merge_state(mm, ll, src[D], src[D + 1], s1, s2);
      if (col < D) aa = aa * s1 + src[col] * s2;
    }
    gpart[(size_t)g * ldp + col] = col < D ? aa : (col == D ? mm : ll);
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    sh.last = atomicAdd(&cu[1], 1u) == (unsigned)narrive - 1u;
    if (sh.last) __threadfence();
  }
  __syncthreads();
  if (sh.last) {
    if (p.trace != nullptr && tid == 0) sh.t_sel = globaltimer();
    merge_unit<G_T>(p, u, S, sh);
    return 4;
  }
  return 2;
}

// ------------------------------------------------------------------ kernel
// MODE 0: one launch interleaves A and B tickets (lag).  Split layers (MODE 1 then MODE 2,
// MHA bf16): an A-only launch (phase 1 + selection, 3 CTAs / SM) and a B-only launch (phase 3 +
// merge) that starts as A CTAs retire, gated by the per-unit ready flags; it waits for the A
// grid before it exits, so "B complete" implies "A complete" for whatever follows.
template <typename T, int G_T, int VEC, int D_T, bool BIG, int MODE = 0>
__global__ void __launch_bounds__(kPT, MODE == 1 ? 3 : 2) pipe_decode_kernel(const PipeParams p,
                                                          const __grid_constant__ CUtensorMap lead_map,
                                                          const __grid_constant__ CUtensorMap krow_map,
                                                          const __grid_constant__ CUtensorMap vrow_map,
                                                          const __grid_constant__ CUtensorMap krow64_map) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  __shared__ PipeShared sh;
  // 1024 B alignment: the tensor-core path reads 128B-swizzled TMA tiles
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int tid = threadIdx.x, lane = lane_id(), w = warp_id();
  const int nsw = p.nst;
  uint8_t* ring = smem + p.off_ring;
  uint8_t* wring = ring + (size_t)w * nsw * p.stage_bytes;
  uint64_t* wbar = reinterpret_cast<uint64_t*>(smem + p.off_bars) + (size_t)w * nsw;
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem + p.off_hist);
  uint32_t* ents = reinterpret_cast<uint32_t*>(smem + p.off_ents);
  uint32_t* kchip = reinterpret_cast<uint32_t*>(smem + p.off_kchip);  // lists mode: a unit's keys [G][La]
  uint64_t* sbar = reinterpret_cast<uint64_t*>(smem + p.off_bars) + (size_t)kPW * nsw;  // selection key stream
  unsigned sphase = 0u;
  if (lane == 0) {
    for (int s = 0; s < nsw; ++s) mbar_init(&wbar[s], 1);
    if (w == 0) {
      mbar_init(&sbar[0], 1);
      mbar_init(&sbar[1], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid == 0) {
    prefetch_desc(&lead_map);
    prefetch_desc(&krow_map);
    prefetch_desc(&vrow_map);
    prefetch_desc(&krow64_map);
  }
  // MODE 2 reads only what the ready flags publish (and K0's products, complete before the A grid
  // passed its own wait): it does not wait for the A grid here
  if constexpr (MODE != 2) asm volatile("griddepcontrol.wait;" ::: "memory");  // K0's q_hat / appended rows
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  uint32_t* tk = MODE == 2 ? p.ctrl + 2 + 4 * (size_t)p.units : p.ctrl;  // ticket / exit counters
  if (tid == 0) sh.next_ticket = atomicAdd(&tk[0], 1u);
  __syncthreads();
  RingPos rp(nsw);
  if constexpr (MODE != 0) {
    // MODE 1: tickets = A(u, c); MODE 2: full B parts of units [0, units - tail), then half parts
    const int tailU = p.lag;  // (MODE 2: units whose parts run as halves)
    const long long nfull = (long long)(p.units - tailU) * p.nA;
    for (;;) {
      const unsigned t = sh.next_ticket;
      __syncthreads();
      if ((long long)t >= p.n_tickets) {
        if (tid == 0 && atomicAdd(&tk[1], 1u) == gridDim.x - 1u) {  // last CTA out resets the counters
          atomicExch(&tk[0], 0u);
          atomicExch(&tk[1], 0u);
        }
        break;
      }
      if (tid == 0) sh.next_ticket = atomicAdd(&tk[0], 1u);
      const long long t0 = (p.trace != nullptr) ? globaltimer() : 0;
      int kind = 0;
      if constexpr (MODE == 3) {
        kind = item_A<T, G_T, VEC, true>(p, &lead_map, (int)(t / (unsigned)p.nAa), (int)(t % (unsigned)p.nAa), ring, wring,
                                  wbar, hist, ents, kchip, sbar, sphase, rp, sh);
      } else if constexpr (MODE == 1) {
        kind = item_A<T, G_T, VEC>(p, &lead_map, (int)(t / (unsigned)p.nAa), (int)(t % (unsigned)p.nAa), ring, wring, wbar,
                            hist, ents, kchip, sbar, sphase, rp, sh);
      } else {
        if ((long long)t < nfull) {
          kind = item_B<T, G_T, VEC, D_T, BIG>(p, &krow_map, &vrow_map, &krow64_map, (int)(t / (unsigned)p.nA),
                                               (int)(t % (unsigned)p.nA), -1, ring, wring, wbar, ents, rp, sh);
        } else {
          const long long tt = t - nfull;
          const int r = (int)(tt % (2 * p.nA));
          kind = item_B<T, G_T, VEC, D_T, BIG>(p, &krow_map, &vrow_map, &krow64_map,
                                        p.units - tailU + (int)(tt / (2 * p.nA)), r >> 1, r & 1, ring, wring, wbar,
                                        ents, rp, sh);
        }
      }
      fence_proxy_async();
      __syncthreads();
      if (p.trace != nullptr && tid == 0) {  // split layers: the host gives each launch its own trace rows
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        long long* tr = p.trace + (size_t)t * 4;
        tr[0] = t0;
        tr[1] = globaltimer();
        tr[2] = (long long)smid | ((long long)kind << 16) | ((long long)blockIdx.x << 32);
        tr[3] = (kind >= 2) ? sh.t_sel : 0;
      }
    }
    if constexpr (MODE == 2) asm volatile("griddepcontrol.wait;" ::: "memory");
    return;
  }
  // slot = A(u, 0..nAa-1), B(u - lag, 0..nA-1); tail slots (no A left): 2 nA half-size B items
  const int per_slot = max(p.nAa + (p.halves == 2 ? 2 : 1) * p.nA, 2 * p.nA);
  for (;;) {
    const unsigned t = sh.next_ticket;
    __syncthreads();
    if ((long long)t >= p.n_tickets) {
      if (tid == 0 && atomicAdd(&p.ctrl[1], 1u) == gridDim.x - 1u) {  // last CTA out resets the counters
        atomicExch(&p.ctrl[0], 0u);
        atomicExch(&p.ctrl[1], 0u);
      }
      break;
    }
    if (tid == 0) sh.next_ticket = atomicAdd(&p.ctrl[0], 1u);  // prefetched; read after the item's barriers
    const long long t0 = (p.trace != nullptr) ? globaltimer() : 0;
    const int slot = (int)(t / (unsigned)per_slot), r = (int)(t % (unsigned)per_slot);
    int kind = 0;
    if (slot >= p.units) {  // tail slot: no A items left, B items (half-size with p.halves)
      if (p.halves ? r < 2 * p.nA : r < p.nA)
        kind = item_B<T, G_T, VEC, D_T, BIG>(p, &krow_map, &vrow_map, &krow64_map, slot - p.lag,
                                      p.halves ? r >> 1 : r, p.halves ? (r & 1) : -1, ring, wring, wbar, ents,
                                      rp, sh);
    } else if (r < p.nAa) {
      kind = item_A<T, G_T, VEC>(p, &lead_map, slot, r, ring, wring, wbar, hist, ents, kchip, sbar, sphase, rp, sh);
    } else if (slot >= p.lag && r < p.nAa + (p.halves == 2 ? 2 * p.nA : p.nA)) {
      const int rb = r - p.nAa;
      kind = item_B<T, G_T, VEC, D_T, BIG>(p, &krow_map, &vrow_map, &krow64_map, slot - p.lag,
                                      p.halves == 2 ? rb >> 1 : rb, p.halves == 2 ? (rb & 1) : -1, ring, wring,
                                      wbar, ents, rp, sh);
    }
    fence_proxy_async();  // this item's generic shared-memory writes precede the next item's TMA writes
    __syncthreads();
    if (p.trace != nullptr && tid == 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      long long* tr = p.trace + (size_t)t * 4;
      tr[0] = t0;
      tr[1] = globaltimer();
      tr[2] = (long long)smid | ((long long)kind << 16) | ((long long)blockIdx.x << 32);
      tr[3] = (kind >= 2) ? sh.t_sel : 0;
    }
  }
}


// Keys of one unit streamed from L2 through two shared buffers of kCK keys
// (cp.async.bulk, the next chunk in flight while this one is scanned), run by a
// thread group.  `sbar` are the group's two mbarriers, `sphase` their parities.
template <typename Grp, int NB = 2, int CK = kCK>
struct KeyStreamG {
  const uint32_t* src;
  int S, kstride;
  uint32_t* buf;  // [NB][CK]
  uint64_t* sbar;  // [NB]
  unsigned* sphase;
  int nchunk;
  __device__ void issue(int c) const {
    if (Grp::tid() == 0 && c < nchunk) {
      const int base = c * CK;
      const int rows = min(CK, kstride - base);
      const unsigned bytes = (unsigned)(((rows * 4) + 15) & ~15);
      uint64_t* bar = &sbar[c % NB];
      mbar_expect_tx(bar, bytes);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(buf + (c % NB) * CK)),
          "l"(src + base), "r"(bytes), "r"(smem_u32(bar))
          : "memory");
    }
  }
  __device__ void start() const {
    if (Grp::tid() == 0) asm volatile("fence.proxy.async.global;" ::: "memory");  // keys came from generic stores
    for (int c = 0; c < NB; ++c) issue(c);
  }
  // the chunks start() put in flight but run() never consumed (an early exit): wait them out
  __device__ void drain() const {
    for (int c = 0; c < NB && c < nchunk; ++c) {
      mbar_wait(&sbar[c], (*sphase >> c) & 1u);
      *sphase ^= 1u << c;
    }
    Grp::sync();
  }
  template <typename F>
  __device__ void run(F&& f) const {
    for (int c = 0; c < nchunk; ++c) {
      const int bi = c % NB;
      mbar_wait(&sbar[bi], (*sphase >> bi) & 1u);
      *sphase ^= 1u << bi;
      f(c * CK, buf + bi * CK, min(CK, S - c * CK));
      Grp::sync();  // the whole group is done with buffer bi before it is refilled
      issue(c + NB);
    }
  }
};

// Selection of a whole unit (one head) whose level-0 histogram is on chip but
// whose keys are in the L2-resident workspace (too many rows to keep on chip):
// the select group of the warp-specialised A launch, for long MHA sequences.
// Same composite-key rule as select_unit / select_onchip; publishes tcs[u].
template <typename Grp, int NB = 2, int CK = kCK>
__device__ void select_global(const PipeParams& p, int u, int S, uint32_t* h, uint32_t* kbuf, uint64_t* sbar,
                              unsigned& sphase, uint8_t* scratch, int scratch_bytes, PipeShared& sh, int g = 0) {
  const size_t ug = (size_t)u * p.G + g;  // this (unit, head)'s keys and threshold (per-head GQA: G heads in turn)
  const int tid = Grp::tid(), lane = lane_id();
  const int hb = p.hbits, HB = 1 << hb;
  const int kb = k_of(p, S);
  const int cap = scratch_bytes / 16;
  unsigned long long* candA = reinterpret_cast<unsigned long long*>(scratch);
  unsigned long long* candB = candA + cap;
  const uint32_t* keys = p.keys + ug * p.kstride;
  const KeyStreamG<Grp, NB, CK> ks{keys, S, p.kstride, kbuf, sbar, &sphase, ceil_div(S > 0 ? S : 1, CK)};
  unsigned long long Tc;
  if (kb <= 0 || kb >= S) {
    Tc = kb <= 0 ? ~0ull : 0ull;
  } else {
    ks.start();  // the compaction pass below almost always runs
    bool started = true;
    find_bin<Grp>(h, HB, (unsigned)kb, sh);
    sel_stamp<Grp>(p, u, 1);
    unsigned long long P = (unsigned long long)sh.fb_bin;
    int nb = hb;
    unsigned need = (unsigned)kb - sh.fb_above, cnt = sh.fb_cnt;
    int ncand = 0;
    bool listed = false;
    for (;;) {
      if (cnt == need) break;
      if (!started) ks.start();
      started = false;
      const int sh64 = 64 - nb;
      if (cnt <= (unsigned)cap) {  // compact the rows matching P
        if (tid == 0) sh.ncand = 0;
        Grp::sync();
        ks.run([&](int j0, const uint32_t* kc, int nrow) {
          // (r02: the chunk's U uint4 groups per thread first, then one warp scan and one shared atomic per warp
          // and chunk -- as select_onchip; a scan + atomic chain per 128 rows made this pass ~18 us at 32K rows)
          constexpr int U = CK / (4 * Grp::kThreads) > 0 ? CK / (4 * Grp::kThreads) : 1;
          for (int i0 = 0; i0 < nrow; i0 += 4 * U * Grp::kThreads) {
            uint4 kk[U];
            unsigned hit[U];
            int c = 0;
#pragma unroll
            for (int v = 0; v < U; ++v) {
              const int il = i0 + 4 * (tid + v * Grp::kThreads);
              kk[v] = make_uint4(0u, 0u, 0u, 0u);
              if (il < nrow) kk[v] = *reinterpret_cast<const uint4*>(kc + il);
              hit[v] = 0u;
#pragma unroll
              for (int e = 0; e < 4; ++e)
                hit[v] |= (il + e < nrow && (comp_key(u4_at(kk[v], e), j0 + il + e) >> sh64) == P ? 1u : 0u) << e;
              c += __popc(hit[v]);
            }
            if (__any_sync(0xffffffffu, c != 0)) {
              int tot;
              const int ex = warp_excl_scan(c, &tot);
              int at = 0;
              if (lane == 0) at = atomicAdd(&sh.ncand, tot);
              at = __shfl_sync(0xffffffffu, at, 0) + ex;
#pragma unroll
              for (int v = 0; v < U; ++v) {
                const int il = i0 + 4 * (tid + v * Grp::kThreads);
#pragma unroll
                for (int e = 0; e < 4; ++e)
                  if ((hit[v] >> e) & 1u) candA[at++] = comp_key(u4_at(kk[v], e), j0 + il + e);
              }
            }
          }
        });
        ncand = sh.ncand;
        listed = true;
        break;
      }
      // one more histogram level over the rows matching P
      const int bits = min(hb, 64 - nb);
      for (int i = tid; i < (1 << bits); i += Grp::kThreads) h[i] = 0u;
      Grp::sync();
      ks.run([&](int j0, const uint32_t* kc, int nrow) {
        for (int i = tid; i < nrow; i += Grp::kThreads) {
          const unsigned long long c = comp_key(kc[i], j0 + i);
          if ((c >> sh64) == P) atomicAdd(&h[(c >> (sh64 - bits)) & ((1ull << bits) - 1)], 1u);
        }
      });
      find_bin<Grp>(h, 1 << bits, need, sh);
      P = (P << bits) | (unsigned long long)sh.fb_bin;
      nb += bits;
      need -= sh.fb_above;
      cnt = sh.fb_cnt;
    }
    if (started) ks.drain();  // the prefetched chunks were never consumed: drain them before the buffers are reused
    sel_stamp<Grp>(p, u, 2);
    Tc = nb >= 64 ? P : (P << (64 - nb));
    if (listed && cnt != need) {
      const unsigned long long* src = candA;
      unsigned long long* dst = candB;
      while (ncand > 32) {
        const int bits = min(8, 64 - nb);
        for (int i = tid; i < (1 << bits); i += Grp::kThreads) h[i] = 0u;
        Grp::sync();
        for (int i = tid; i < ncand; i += Grp::kThreads)
          atomicAdd(&h[(src[i] >> (64 - nb - bits)) & ((1ull << bits) - 1)], 1u);
        Grp::sync();
        find_bin<Grp>(h, 1 << bits, need, sh);
        P = (P << bits) | (unsigned long long)sh.fb_bin;
        nb += bits;
        need -= sh.fb_above;
        cnt = sh.fb_cnt;
        if (cnt == need) break;
        if (tid == 0) sh.ncand = 0;
        Grp::sync();
        for (int i0 = 0; i0 < ncand; i0 += Grp::kThreads) {
          const int i = i0 + tid;
          const unsigned long long c = i < ncand ? src[i] : 0ull;
          append_if(i < ncand && (c >> (64 - nb)) == P, c, dst, &sh.ncand);
        }
        Grp::sync();
        ncand = sh.ncand;
        unsigned long long* was = const_cast<unsigned long long*>(src);
        src = dst;
        dst = was;
      }
      if (cnt == need) {
        Tc = nb >= 64 ? P : (P << (64 - nb));
      } else {  // <= 32 candidates, one per lane of the group's first warp: the need-th largest by rank
        if (tid < 32) {
          const unsigned long long c = tid < ncand ? src[tid] : 0ull;
          unsigned rank = 0;
          for (int i = 0; i < ncand; ++i) rank += __shfl_sync(0xffffffffu, c, i) > c;
          if (tid < ncand && rank == need - 1) sh.tsel = c;
        }
        Grp::sync();
        Tc = sh.tsel;
      }
    }
    sel_stamp<Grp>(p, u, 3);
  }
  if (p.poff != nullptr && !p.lists) {  // diagnostics (key path): each half part's offset into the index lists
    const int half = p.Lc / 2, nh = 2 * p.nA;
    uint32_t* cnt = h;  // the histogram is free again
    for (int i = tid; i < nh; i += Grp::kThreads) cnt[i] = 0u;
    Grp::sync();
    if (kb >= S) {
      for (int i = tid; i < nh; i += Grp::kThreads) cnt[i] = (unsigned)max(0, min(S - i * half, half));
    } else if (kb > 0) {
      ks.start();
      ks.run([&](int j0, const uint32_t* kc, int nrow) {
        for (int i = tid; i < nrow; i += Grp::kThreads)
          if (comp_key(kc[i], j0 + i) >= Tc) atomicAdd(&cnt[(j0 + i) / half], 1u);
      });
    }
    Grp::sync();
    if (tid == 0) {  // group-shared: the one selection's offsets serve every head of the group
      const size_t r0 = p.shared > 1 ? (size_t)u * p.shared : ug;
      const int nr = p.shared > 1 ? p.shared : 1;
      unsigned run = 0;
      for (int i = 0; i < nh; ++i) {
        for (int r = 0; r < nr; ++r) p.poff[(r0 + r) * nh + i] = run;
        run += cnt[i];
      }
    }
    Grp::sync();
  }
  if (tid == 0) p.tcs[ug] = Tc;
  Grp::sync();
}

// Ordered emission (lists mode) for a unit whose keys are in the L2-resident workspace: the keys stream
// back through the group's two chunk buffers; every selected row (composite key >= Tc) becomes an
// entry (head mask << 24 | row), ascending, written IN PLACE over the keys (an entry's position never
// exceeds its row, and rows are consumed chunk by chunk ahead of the writes; the chunks in flight lie
// past every position written), plus each half part's entry offset in p.loff[u] and, for diagnostics,
// the heads' ascending index rows.  One selection per unit: G = 1, or group-shared (every head's mask).
template <typename Grp, int NB>
__device__ void emit_lists_global(const PipeParams& p, int u, int S, unsigned long long Tc, uint32_t* kbuf,
                                  uint64_t* sbar, unsigned& sphase, PipeShared& sh) {
  constexpr int PER = kCK / Grp::kThreads;  // contiguous keys per thread and chunk
  const int tid = Grp::tid();
  const int lhs = 31 - __clz(p.Lc / 2);     // Lc / 2 is a power of two (>= PER)
  uint32_t* keys = p.keys + (size_t)u * p.sel_stride;  // (== the unit's keys: one array per unit here)
  uint32_t* lo = p.loff + (size_t)u * (2 * p.nA + 1);
  const unsigned full = shared_mask(p) << 24;
  int32_t* idx_dst = nullptr;
  int nh = 0;
  if (p.idx_out != nullptr) {
    nh = unit_heads(p);
    idx_dst = p.idx_out + ((size_t)(u / p.Hkv) * p.Hq + (size_t)(u % p.Hkv) * nh) * p.idx_stride;
  }
  unsigned base = 0;
  if (S > 0) {
    const KeyStreamG<Grp, NB> ks{keys, S, p.kstride, kbuf, sbar, &sphase, ceil_div(S, kCK)};
    ks.start();
    ks.run([&](int j0, const uint32_t* kc, int nrow) {
      const int t0 = tid * PER;
      unsigned m = 0;
#pragma unroll
      for (int e4 = 0; e4 < PER; e4 += 4) {  // 16-byte loads: a lane's PER keys are contiguous
        const uint4 kk = *reinterpret_cast<const uint4*>(kc + t0 + e4);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int j = t0 + e4 + e;
          m |= (j < nrow && comp_key(u4_at(kk, e), j0 + j) >= Tc ? 1u : 0u) << (e4 + e);
        }
      }
      const unsigned c = __popc(m);
      unsigned tot;
      unsigned at = base + block_incl_scan<Grp>(c, sh, &tot) - c;
      const int r0 = j0 + t0;
      if (t0 < nrow && (r0 & ((1 << lhs) - 1)) == 0) lo[r0 >> lhs] = at;  // entries before row r0
#pragma unroll
      for (int e = 0; e < PER; ++e)
        if ((m >> e) & 1u) {
          if (idx_dst != nullptr)
            for (int g = 0; g < nh; ++g) idx_dst[(size_t)g * p.idx_stride + at] = r0 + e;
          keys[at++] = full | (uint32_t)(r0 + e);
        }
      base += tot;
    });
  }
  if (tid == 0)
    for (int q = S > 0 ? ((S + (1 << lhs) - 1) >> lhs) : 0; q <= 2 * p.nA; ++q) lo[q] = base;
  Grp::sync();
}

// Ordered emission for per-head groups (G_T > 1, keys in the workspace): the G key arrays of a unit stream
// back together (chunks of kCK / G_T rows per head in one buffer), every row some head selected becomes
// an entry (head mask << 24 | row), ascending, written in place over the unit's head-0 keys (same rule
// as emit_lists_global: positions never pass their rows, the chunks in flight lie beyond), plus the half
// parts' entry offsets and, for diagnostics, each head's own ascending index row.
template <typename Grp, int G_T, int NB, int CKE>
__device__ void emit_lists_global_heads(const PipeParams& p, int u, int S, uint32_t* kbuf, uint64_t* sbar,
                                        unsigned& sphase, PipeShared& sh) {
  constexpr int C = CKE / G_T;              // rows per chunk (one buffer holds G_T x C keys)
  constexpr int PER = C / Grp::kThreads;    // contiguous rows per thread and chunk
  static_assert(PER >= 4 && PER % 4 == 0, "a thread's rows are read as whole uint4 groups");
  const int tid = Grp::tid();
  const int G = p.G;
  const int lhs = 31 - __clz(p.Lc / 2);
  uint32_t* dst = p.sel + (size_t)u * p.sel_stride;  // == the unit's head-0 keys
  const uint32_t* keys = p.keys + (size_t)u * G * p.kstride;
  uint32_t* lo = p.loff + (size_t)u * (2 * p.nA + 1);
  unsigned long long Tc[G_T];
#pragma unroll
  for (int g = 0; g < G_T; ++g) Tc[g] = g < G ? __ldcg(&p.tcs[(size_t)u * G + g]) : ~0ull;
  int32_t* idx0 = p.idx_out != nullptr
                      ? p.idx_out + ((size_t)(u / p.Hkv) * p.Hq + (size_t)(u % p.Hkv) * G) * p.idx_stride
                      : nullptr;
  const int nchunk = ceil_div(S > 0 ? S : 1, C);
  auto issue = [&](int c) {
    if (tid == 0 && c < nchunk) {
      const int base = c * C;
      const int rows = min(C, p.kstride - base);
      const unsigned bytes = (unsigned)(((rows * 4) + 15) & ~15);
      uint64_t* bar = &sbar[c % NB];
      mbar_expect_tx(bar, bytes * (unsigned)G);
      for (int g = 0; g < G; ++g)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(kbuf + (c % NB) * CKE + g * C)),
            "l"(keys + (size_t)g * p.kstride + base), "r"(bytes), "r"(smem_u32(bar))
            : "memory");
    }
  };
  unsigned base = 0, hbase[G_T];
#pragma unroll
  for (int g = 0; g < G_T; ++g) hbase[g] = 0u;
  if (S > 0) {
    if (tid == 0) asm volatile("fence.proxy.async.global;" ::: "memory");  // keys came from generic stores
    for (int c = 0; c < NB; ++c) issue(c);
    for (int c = 0; c < nchunk; ++c) {
      const int bi = c % NB;
      mbar_wait(&sbar[bi], (sphase >> bi) & 1u);
      sphase ^= 1u << bi;
      const uint32_t* kc = kbuf + bi * CKE;
      const int j0 = c * C, t0 = tid * PER;
      const int nrow = min(C, S - j0);
      unsigned m[PER];
      unsigned cnt = 0;
#pragma unroll
      for (int e = 0; e < PER; ++e) m[e] = 0u;
#pragma unroll
      for (int g = 0; g < G_T; ++g) {
        if (g >= G) break;
#pragma unroll
        for (int e4 = 0; e4 < PER; e4 += 4) {  // 16-byte loads: a lane's PER keys are contiguous
          const uint4 kk = *reinterpret_cast<const uint4*>(kc + g * C + t0 + e4);
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (t0 + e4 + e < nrow && comp_key(u4_at(kk, e), j0 + t0 + e4 + e) >= Tc[g]) m[e4 + e] |= 1u << g;
        }
      }
#pragma unroll
      for (int e = 0; e < PER; ++e) cnt += m[e] != 0u;
      unsigned tot;
      unsigned at = base + block_incl_scan<Grp>(cnt, sh, &tot) - cnt;
      const int r0 = j0 + t0;
      if (t0 < nrow && (r0 & ((1 << lhs) - 1)) == 0) lo[r0 >> lhs] = at;
      if (idx0 != nullptr) {  // diagnostics: each head's ascending rows at its own positions
#pragma unroll
        for (int g = 0; g < G_T; ++g) {
          if (g >= G) break;
          unsigned cg = 0;
#pragma unroll
          for (int e = 0; e < PER; ++e) cg += (m[e] >> g) & 1u;
          unsigned tg;
          unsigned pg = hbase[g] + block_incl_scan<Grp>(cg, sh, &tg) - cg;
#pragma unroll
          for (int e = 0; e < PER; ++e)
            if ((m[e] >> g) & 1u) idx0[(size_t)g * p.idx_stride + pg++] = r0 + e;
          hbase[g] += tg;
        }
      }
#pragma unroll
      for (int e = 0; e < PER; ++e)
        if (m[e]) dst[at++] = (m[e] << 24) | (uint32_t)(r0 + e);
      base += tot;
      Grp::sync();  // the group is done with buffer bi (and its writes precede later chunks') before the refill
      issue(c + NB);
    }
  }
  if (tid == 0)
    for (int q = S > 0 ? ((S + (1 << lhs) - 1) >> lhs) : 0; q <= 2 * p.nA; ++q) lo[q] = base;
  Grp::sync();
}

// Per-head GQA phase 1 on the 5th-generation tensor cores (tcgen05, TMEM accumulators): the stream group
// of the warp-specialised A launch runs it as a warp-specialised pipeline over 128-row tiles of a unit --
//   warp 0 (one lane): TMA producer, the tile's lead boxes into a ring of p.ust tile stages;
//   warp 1 (one lane): MMA issuer, D[128 x N] = K_lead[128 x d] . Qt[N x d]^T per tile (d / 16 tcgen05.mma,
//     kind::f16, bf16 x bf16 -> f32 in TMEM, two accumulators), committing to the ring's empty barrier and
//     the accumulator's full barrier;
//   warps 4-7: epilogue, tcgen05.ld of their 32-row TMEM lane quadrant, the score of head g = term 0 +
//     term 1 + term 2 (q split into three bf16 terms, columns t * G_T + g, so the score keeps fp32-level
//     error) -> order key -> the head's key array and histogram.
// `tc` counts the tiles this CTA has processed (barrier phases continue across units).
template <int RB, int G_T>
__device__ void stream_unit_umma(const PipeParams& p, const CUtensorMap* lead_map, int bb, int hk, int n,
                                 size_t qrow0, uint32_t* keys, uint32_t* hist, int HB, int hshift, uint8_t* smem,
                                 uint64_t* bars, uint32_t tmem, uint32_t& tc) {
  constexpr int E = 2;
  constexpr int TR = 128;                            // rows per tile (the MMA's M)
  constexpr int NCOL = (3 * G_T + 15) / 16 * 16;     // N: three query terms per head, padded to 16
  constexpr uint32_t IDESC = umma::idesc_bf16_f32(TR, NCOL);
  const int lane = lane_id(), w = warp_id();
  const int NS = p.ust;
  const int R1 = p.r1;
  const int tile_bytes = TR * RB;
  const int ntile = ceil_div(n, TR);
  uint8_t* tiles = smem + p.off_ring;                // [NS][TR][RB], 1024-byte aligned tiles
  uint8_t* qt = smem + p.off_qt;                     // [NCOL][RB] K-major query terms
  uint64_t* fullb = bars;
  uint64_t* emptyb = bars + NS;
  uint64_t* tfull = bars + 2 * NS;
  uint64_t* tempty = bars + 2 * NS + 2;
  // the B operand: row r = term t (r / G_T) of head g (r % G_T), swizzled like the TMA tiles
  for (int i = threadIdx.x; i < NCOL * (RB / 2); i += kPT) {
    const int r = i / (RB / 2), c = i % (RB / 2);
    const int t = r / G_T, g = r % G_T;
    float v = 0.f;
    if (t < 3 && g < p.G && c < p.d) {
      const float x = p.q_hat[(qrow0 + g) * p.D + c];
      const float r1 = x - bf16_hi(x);
      v = t == 0 ? x : (t == 1 ? r1 : r1 - bf16_hi(r1));
    }
    const int sw = RB == 64 ? ((r >> 1) & 3) : (r & 7);
    *reinterpret_cast<__nv_bfloat16*>(qt + r * RB + ((((c * E) >> 4) ^ sw) << 4) + ((c * E) & 15)) =
        __float2bfloat16_rn(v);
  }
  umma::fence_async_smem();
  WarpGroup<0, kPW, 1>::sync();  // (the stream group's barrier)
  if (w == 0 && lane == 0) {  // ---- TMA producer
    for (int t = 0; t < ntile; ++t) {
      const uint32_t q = tc + (uint32_t)t;
      const int slot = (int)(q % (uint32_t)NS);
      if (q >= (uint32_t)NS) mbar_wait(&emptyb[slot], ((q / NS) - 1u) & 1u);
      const int rows = min(TR, n - t * TR);
      const int nb = ceil_div(rows, R1);
      mbar_expect_tx(&fullb[slot], (unsigned)(nb * R1 * RB));
      for (int i = 0; i < nb; ++i)
        tma_box4d(tiles + slot * tile_bytes + i * R1 * RB, lead_map, 0, t * TR + i * R1, hk, bb, &fullb[slot]);
    }
  } else if (w == 1 && lane == 0) {  // ---- MMA issuer
    const uint32_t qa = umma::smem_addr(qt);
    for (int t = 0; t < ntile; ++t) {
      const uint32_t q = tc + (uint32_t)t;
      const int slot = (int)(q % (uint32_t)NS), acc = (int)(q & 1u);
      mbar_wait(&fullb[slot], (q / NS) & 1u);
      if (q >= 2u) mbar_wait(&tempty[acc], ((q >> 1) - 1u) & 1u);
      umma::fence_after();
      const uint32_t ta = umma::smem_addr(tiles + slot * tile_bytes);
#pragma unroll
      for (int ks = 0; ks < RB / 32; ++ks)
        umma::mma_bf16(tmem + (uint32_t)(acc * NCOL), umma::smem_desc_kmajor(ta + 32 * ks, RB),
                       umma::smem_desc_kmajor(qa + 32 * ks, RB), IDESC, ks > 0);
      umma::commit(&emptyb[slot]);
      umma::commit(&tfull[acc]);
    }
  } else if (w >= 4) {  // ---- epilogue: TMEM lane quadrant w % 4
    const int ew = w - 4;
    for (int t = 0; t < ntile; ++t) {
      const uint32_t q = tc + (uint32_t)t;
      const int acc = (int)(q & 1u);
      mbar_wait(&tfull[acc], (q >> 1) & 1u);
      umma::fence_after();
      uint32_t v[NCOL];
      const uint32_t ta = tmem + (uint32_t)(acc * NCOL) + ((uint32_t)(ew * 32) << 16);
#pragma unroll
      for (int c0 = 0; c0 < NCOL; c0 += 16) umma::ld_32x32b_x16(ta + c0, *reinterpret_cast<uint32_t(*)[16]>(v + c0));
      umma::wait_ld();
      umma::fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      const int row = t * TR + ew * 32 + lane;
      if (row < n) {
#pragma unroll
        for (int g = 0; g < G_T; ++g) {
          if (g < p.G) {
            const float sc = (__uint_as_float(v[g]) + __uint_as_float(v[G_T + g])) + __uint_as_float(v[2 * G_T + g]);
            const uint32_t key = order_key(sc);
            keys[(size_t)g * p.kstride + row] = key;
            if (p.approx_out != nullptr) p.approx_out[(qrow0 + g) * p.S_cap + row] = sc;
            atomicAdd(&hist[g * HB + (key >> hshift)], 1u);
          }
        }
      }
    }
  }
  tc += (uint32_t)ntile;
}

// ------------------------------------------------------------------ warp-specialised A launch
// Split layers whose units are one A chunk (lists mode, MHA): a 16-warp CTA per
// SM runs phase 1 and the selection as a two-stage pipeline over units.
//   stream group (warps 0-7): draws a unit, streams its lead columns through the
//     per-warp TMA rings, keeps the order keys and the level-0 histogram on chip
//     in one of two buffers, hands the buffer over and starts the next unit;
//   select group (warps 8-15): selects on the handed-over buffer (select_onchip),
//     publishes the ordered entry lists (emit_lists) and the unit's ready flag,
//     returns the buffer.
// So the selection never stalls the HBM stream (the old A item streamed, then
// selected with the SM's loads idle).  Hand-over is two mbarriers per buffer
// (full: stream -> select, empty: select -> stream).
using StreamGrp = WarpGroup<0, kPW, 1>;
using SelectGrp = WarpGroup<kPW, kPW, 2>;

// ONCHIP: the unit's keys stay in shared memory (double-buffered [2][La]) and the
// select group also emits the ordered entry lists (lists mode); else (long
// sequences) the stream group writes the keys to the L2-resident workspace, the
// select group streams them back (select_global) and publishes the threshold.
// G_T > 1 (per-head GQA, workspace keys): the stream group scores the G heads on the tensor cores
// (lead_consume_mma) into G key arrays and G histograms; the select group selects the heads in turn.
template <typename T, int RB, bool ONCHIP, int G_T = 1>
__global__ void __launch_bounds__(2 * kPT, 1) pipe_select_kernel(const PipeParams p,
                                                                 const __grid_constant__ CUtensorMap lead_map) {
  static_assert(G_T == 1 || !ONCHIP, "per-head groups keep their keys in the workspace");
  constexpr int E = sizeof(T);
  constexpr int Q2 = RB / (2 * E);
  extern __shared__ __align__(128) uint8_t smem_raw[];
  __shared__ PipeShared sh;
  __shared__ int item_u[2];
  __shared__ unsigned s_ticket;
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int lane = lane_id(), wid = warp_id();
  const int nsw = p.nst, SB = p.stage_bytes;
  const int HB = 1 << p.hbits, hshift = 32 - p.hbits;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.off_bars);
  uint64_t* full = bars + (size_t)kPW * nsw;  // [2]
  uint64_t* empty = full + 2;                 // [2]
  uint64_t* sbar = empty + 2;                 // [kSelNB] the select group's key stream (!ONCHIP)
  uint32_t* hist2 = reinterpret_cast<uint32_t*>(smem + p.off_hist);   // [2][G_T][HB]
  uint32_t* kbuf2 = reinterpret_cast<uint32_t*>(smem + p.off_kchip);  // ONCHIP: [2][La]; else [kSelNB][kCK]
  uint8_t* cand = smem + p.off_cand;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kPW * nsw; ++i) mbar_init(&bars[i], 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&empty[b], 1);
    }
    for (int b = 0; b < kSelNB; ++b) mbar_init(&sbar[b], 1);
    if constexpr (G_T > 1) {  // tcgen05 phase 1: the accumulators' empty barriers take the 4 epilogue warps
      if (p.umma) {
        mbar_init(&bars[2 * p.ust + 2], 4);
        mbar_init(&bars[2 * p.ust + 3], 4);
      }
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    prefetch_desc(&lead_map);
  }
  __shared__ uint32_t tmem_base;
  if constexpr (G_T > 1) {
    if (p.umma && wid == 0) umma::alloc(&tmem_base, 2 * ((3 * G_T + 15) / 16 * 16) <= 32 ? 32u : 64u);
  }
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");  // K0's q_hat / appended rows
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if (wid < kPW) {  // ---------------- stream group
    const int w = wid, tid = StreamGrp::tid();
    uint8_t* wring = smem + p.off_ring + (size_t)w * nsw * SB;
    uint64_t* wbar = bars + (size_t)w * nsw;
    RingPos rp(nsw);
    uint32_t utc = 0;  // tcgen05 path: tiles processed (barrier phases run on across units)
    for (int i = 0;; ++i) {
      const int b = i & 1;
      if (i >= 2) mbar_wait(&empty[b], ((i >> 1) - 1) & 1u);  // the select group is done with buffer b
      if (tid == 0) s_ticket = atomicAdd(&p.ctrl[0], 1u);
      StreamGrp::sync();
      const unsigned t = s_ticket;
      StreamGrp::sync();  // s_ticket is rewritten next round only after this
      if ((long long)t >= p.n_tickets) {
        if (tid == 0) {
          item_u[b] = -1;
          mbar_arrive(&full[b]);
          if (atomicAdd(&p.ctrl[1], 1u) == gridDim.x - 1u) {  // last CTA out resets the counters
            atomicExch(&p.ctrl[0], 0u);
            atomicExch(&p.ctrl[1], 0u);
          }
        }
        break;
      }
      const int u = (int)t;
      const int bb = u / p.Hkv, hk = u % p.Hkv;
      int S = p.lens[bb];
      S = S < 0 ? 0 : (S > p.S_max ? p.S_max : S);
      uint32_t* hist = hist2 + (size_t)b * G_T * HB;
      uint32_t* keys = ONCHIP ? kbuf2 + (size_t)b * p.La : p.keys + (size_t)u * p.G * p.kstride;
      // on-chip selection without entry lists: the keys also go to the workspace for the B items
      uint32_t* kglob = (ONCHIP && !p.lists) ? p.keys + (size_t)u * p.kstride : nullptr;
      for (int j = tid; j < G_T * HB; j += kPT) hist[j] = 0u;
      StreamGrp::sync();
      const int n = S < p.La ? S : p.La;
      if (n > 0) {
        const int R1 = p.r1;
        const int nbox = ceil_div(n, R1);
        const unsigned box_bytes = (unsigned)(R1 * p.dbox * E);
        const int mine = nbox > w ? ceil_div(nbox - w, kPW) : 0;
        auto issue = [&](int k, const RingPos& at) {
          mbar_expect_tx(&wbar[at.slot], box_bytes);
          tma_box4d(wring + at.slot * SB, &lead_map, 0, (w + k * kPW) * R1, hk, bb, &wbar[at.slot]);
        };
        if (lane == 0 && !(G_T > 1 && p.umma)) {  // (the tcgen05 path has its own producer)
          RingPos q = rp;
          for (int k = 0; k < nsw && k < mine; ++k, q.advance(1)) issue(k, q);
        }
        const int gs = unit_heads(p);  // 1, the group size, or the group whose summed query ranks (shared)
        const size_t qrow0 = (size_t)bb * p.Hq + (size_t)hk * gs;
        if constexpr (G_T > 1) {
          if (p.umma) {  // per-head GQA phase 1 on tcgen05 (tiles of 128 rows, TMEM accumulators)
            stream_unit_umma<RB, G_T>(p, &lead_map, bb, hk, n, qrow0, keys, hist, HB, hshift, smem, bars, tmem_base,
                                      utc);
          } else {  // per-head GQA: G heads on mma.sync (q in three bf16 terms)
          uint32_t qf[3][4][2];
          const int g8 = lane >> 2, t4 = lane & 3;
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            float v[4], r1v[4], r2v[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int dim = 16 * ks + 2 * t4 + (i & 1) + (i >> 1) * 8;
              v[i] = (g8 < p.G && dim < p.d) ? p.q_hat[(qrow0 + g8) * p.D + dim] : 0.f;
              r1v[i] = v[i] - bf16_hi(v[i]);
              r2v[i] = r1v[i] - bf16_hi(r1v[i]);
            }
            qf[0][ks][0] = pack_bf16(v[0], v[1]);
            qf[0][ks][1] = pack_bf16(v[2], v[3]);
            qf[1][ks][0] = pack_bf16(r1v[0], r1v[1]);
            qf[1][ks][1] = pack_bf16(r1v[2], r1v[3]);
            qf[2][ks][0] = pack_bf16(r2v[0], r2v[1]);
            qf[2][ks][1] = pack_bf16(r2v[2], r2v[3]);
          }
          float* approx_u = p.approx_out ? p.approx_out + qrow0 * p.S_cap : nullptr;
          for (int k = 0; k < mine; ++k, rp.advance(1)) {
            mbar_wait(&wbar[rp.slot], rp.phase);
            const int box = w + k * kPW;
            const int rows_here = min(R1, n - box * R1);
            lead_consume_mma<RB, G_T>(p, wring + rp.slot * SB, rows_here, qf, p.G, keys + box * R1, p.kstride,
                                      nullptr, approx_u ? approx_u + box * R1 : nullptr, hist, HB, hshift);
            __syncwarp();
            if (lane == 0 && k + nsw < mine) issue(k + nsw, rp);
          }
          }
        } else {
        unsigned long long q2[Q2];
#pragma unroll
        for (int j = 0; j < Q2; ++j) {  // (independent loads, all in flight together)
          const int c0 = 2 * j, c1 = 2 * j + 1;
          const float a = c0 < p.d ? p.q_hat[qrow0 * p.D + c0] : 0.f;
          const float bq = c1 < p.d ? p.q_hat[qrow0 * p.D + c1] : 0.f;
          q2[j] = pk2(__float_as_uint(a), __float_as_uint(bq));
        }
        if (gs > 1) {  // group-shared selection: rank on the group's summed query
#pragma unroll
          for (int j = 0; j < Q2; ++j) {
            const int c0 = 2 * j, c1 = 2 * j + 1;
            const float a = c0 < p.d ? group_q(p, qrow0, gs, c0) : 0.f;
            const float bq = c1 < p.d ? group_q(p, qrow0, gs, c1) : 0.f;
            q2[j] = pk2(__float_as_uint(a), __float_as_uint(bq));
          }
        }
        float* approx_u = p.approx_out ? p.approx_out + qrow0 * p.S_cap : nullptr;
        for (int k = 0; k < mine; ++k, rp.advance(1)) {
          mbar_wait(&wbar[rp.slot], rp.phase);
          const int box = w + k * kPW;
          const int rows_here = min(R1, n - box * R1);
          lead_consume_lpr<T, RB>(p, wring + rp.slot * SB, rows_here, q2, keys + box * R1,
                                  kglob != nullptr ? kglob + box * R1 : nullptr,
                                  approx_u ? approx_u + box * R1 : nullptr, hist, hshift);
          __syncwarp();
          if (lane == 0 && k + nsw < mine) issue(k + nsw, rp);
        }
        }
      }
      StreamGrp::sync();  // every key and histogram count of this unit is in shared memory
      if (p.approx_out != nullptr && p.shared > 1) {  // diagnostics: each head of the group reports the group score
        const size_t r0 = ((size_t)bb * p.Hq + (size_t)hk * p.shared) * p.S_cap;
        for (int g = 1; g < p.shared; ++g)
          for (int j = tid; j < n; j += kPT) p.approx_out[r0 + (size_t)g * p.S_cap + j] = p.approx_out[r0 + j];
      }
      if (tid == 0) {
        item_u[b] = u;
        mbar_arrive(&full[b]);  // release: the select group acquires through the barrier phase
      }
    }
    if constexpr (G_T > 1) {
      if (p.umma) {  // every tile's MMAs and TMEM loads are done: free the accumulators
        StreamGrp::sync();
        if (w == 0) umma::dealloc(tmem_base, 2 * ((3 * G_T + 15) / 16 * 16) <= 32 ? 32u : 64u);
      }
    }
  } else {  // ---------------- select group
    const int tid = SelectGrp::tid();
    unsigned sphase = 0u;
    for (int i = 0;; ++i) {
      const int b = i & 1;
      mbar_wait(&full[b], (i >> 1) & 1u);
      const int u = item_u[b];
      if (u < 0) break;
      int S = p.lens[u / p.Hkv];
      S = S < 0 ? 0 : (S > p.S_max ? p.S_max : S);
      const uint32_t* keys = kbuf2 + (size_t)b * p.La;
      const long long t0 = (p.trace != nullptr) ? globaltimer() : 0;
      sel_stamp<SelectGrp>(p, u, 0);
      if constexpr (G_T > 1) {  // per-head GQA: the G heads in turn, then the union emission
        // (r02: the heads on four 2-warp sub-groups at once measured no faster -- the passes are bound by
        // the select threads' per-key work, not by L2 latency)
        for (int g = 0; g < p.G; ++g)
          select_global<SelectGrp, sel_nb(G_T)>(p, u, S, hist2 + ((size_t)b * G_T + g) * HB, kbuf2, sbar, sphase, cand,
                                           p.cand_bytes, sh, g);
        sel_stamp<SelectGrp>(p, u, 4);
        if (p.lists)
          emit_lists_global_heads<SelectGrp, G_T, 2, sel_nb(G_T) * kCK / 2>(p, u, S, kbuf2, sbar, sphase, sh);
      } else if constexpr (ONCHIP) {
        select_onchip<1, SelectGrp>(p, u, S, keys, p.La, hist2 + (size_t)b * HB, cand, p.cand_bytes, sh);
        sel_stamp<SelectGrp>(p, u, 4);
        if (p.lists) {
          if (p.La <= 16384)
            emit_lists_g1<SelectGrp>(p, u, S, keys, sh);  // ends with a group barrier
          else
            emit_lists<1, SelectGrp>(p, u, S, keys, p.La, sh);
        } else if (tid == 0) {  // key mode: the B items re-derive their rows from the workspace keys
          p.tcs[u] = sh.Tc[0];
        }
      } else {
        select_global<SelectGrp, sel_nb(G_T)>(p, u, S, hist2 + (size_t)b * HB, kbuf2, sbar, sphase, cand, p.cand_bytes,
                                         sh);
        sel_stamp<SelectGrp>(p, u, 4);
        if (p.lists) emit_lists_global<SelectGrp, sel_nb(G_T)>(p, u, S, p.tcs[u], kbuf2, sbar, sphase, sh);
      }
      sel_stamp<SelectGrp>(p, u, 5);
      if (tid == 0) {
        // the buffer is free as soon as the group's barrier has passed: hand it back first (the stream group
        // waits on it when the selection is the longer side, C2); then the release store, cumulative over the
        // group's list stores ordered by that barrier (no separate fence: st.release.gpu is one)
        mbar_arrive(&empty[b]);
        st_release(&p.ctrl[2 + 4 * (size_t)u + 2], 1u);
        if (p.trace != nullptr) {  // one row per unit: {select start, end, smid | kind 3, select start}
          unsigned smid;
          asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
          long long* tr = p.trace + (size_t)u * 4;
          tr[0] = t0;
          tr[1] = globaltimer();
          tr[2] = (long long)smid | (3LL << 16) | ((long long)blockIdx.x << 32);
          tr[3] = t0;
        }
      }
      sel_stamp<SelectGrp>(p, u, 6);
    }
  }
}

// LokiDiagnostics.weights of a lists-mode launch: head g's weights follow its own ascending rows -- the
// entries whose mask has bit g -- weight exp2(logit - M) / L with the head's merged (M, L).  Diagnostics
// only: a separate small launch keeps this code out of the B items' register budget.
__global__ void __launch_bounds__(256) pipe_weights_kernel(const PipeParams p) {
  __shared__ unsigned wsum[8];
  const int u = blockIdx.x, g = blockIdx.y;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t* sel = p.sel + (size_t)u * p.sel_stride;
  const int total = (int)p.loff[(size_t)u * (2 * p.nA + 1) + 2 * p.nA];
  const float M = p.ml[((size_t)u * p.G + g) * 2], invL = 1.f / p.ml[((size_t)u * p.G + g) * 2 + 1];
  const float* lg = p.logits + ((size_t)u * p.G + g) * p.S_cap;
  const size_t qrow = (size_t)(u / p.Hkv) * p.Hq + (size_t)(u % p.Hkv) * p.G + g;
  float* dst = p.weights_out + qrow * p.idx_stride;
  unsigned base = 0;
  for (int i0 = 0; i0 < total; i0 += 256) {
    const int i = i0 + threadIdx.x;
    const uint32_t e = i < total ? sel[i] : 0u;
    const bool on = i < total && ((e >> (24 + g)) & 1u);
    const unsigned bal = __ballot_sync(0xffffffffu, on);
    if (lane == 0) wsum[w] = __popc(bal);
    __syncthreads();
    unsigned before = 0, tot = 0;
    for (int k = 0; k < 8; ++k) {
      before += k < w ? wsum[k] : 0u;
      tot += wsum[k];
    }
    if (on) dst[base + before + __popc(bal & ((1u << lane) - 1u))] = exp2f(lg[e & 0xFFFFFFu] - M) * invL;
    base += tot;
    __syncthreads();
  }
}

}  // namespace


template <typename T, int G_T, int VEC, int D_T, bool BIG, int MODE>
KernelAttrs& pipe_attrs() {  // one per instantiation, shared by the launch and the occupancy query
  static KernelAttrs a;
  return a;
}

template <typename T, int G_T, int VEC, int D_T, bool BIG, int MODE = 0>
inline cudaError_t launch_pipe_t(const PipeParams& p, int grid, size_t smem, const TmaDesc* maps, cudaStream_t st) {
  auto kern = pipe_decode_kernel<T, G_T, VEC, D_T, BIG, MODE>;
  {
    cudaError_t e = pipe_attrs<T, G_T, VEC, D_T, BIG, MODE>().ensure(reinterpret_cast<const void*>(kern), smem);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kPT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const CUtensorMap* m = reinterpret_cast<const CUtensorMap*>(maps);
  return cudaLaunchKernelEx(&cfg, kern, p, m[0], m[1], m[2], m[3]);
}

template <typename T, int G_T, int VEC, int D_T, bool BIG, int MODE = 0>
inline int occupancy_t(size_t smem) {
  auto kern = pipe_decode_kernel<T, G_T, VEC, D_T, BIG, MODE>;
  return pipe_attrs<T, G_T, VEC, D_T, BIG, MODE>().occupancy(reinterpret_cast<const void*>(kern), kPT, smem);
}


// One (dtype, head dim) slice of the instantiations; each slice is compiled in
// its own translation unit (loki_pipe_inst_*.cu) so the build runs in parallel.
template <typename T, int DT>
cudaError_t pipe_launch_dt(const PipeParams& p, int G_T, int grid, size_t smem, const TmaDesc* maps, cudaStream_t st,
                           bool big, int mode) {
  constexpr int V = sizeof(T) == 2 ? 8 : 4;
  if constexpr (sizeof(T) == 2) {  // split layers: bf16 caches
    if (mode == 3) {  // A-only launch with on-chip selection (lists mode: MHA, single-chunk units)
      if (G_T == 1 && !big) return launch_pipe_t<T, 1, V, DT, false, 3>(p, grid, smem, maps, st);
      return cudaErrorInvalidValue;
    }
    if (mode != 0) {
      switch (G_T) {
        case 1:
          if (mode == 1)
            return big ? launch_pipe_t<T, 1, V, DT, true, 1>(p, grid, smem, maps, st)
                       : launch_pipe_t<T, 1, V, DT, false, 1>(p, grid, smem, maps, st);
          return big ? launch_pipe_t<T, 1, V, DT, true, 2>(p, grid, smem, maps, st)
                     : launch_pipe_t<T, 1, V, DT, false, 2>(p, grid, smem, maps, st);
        case 2:
          return mode == 1 ? launch_pipe_t<T, 2, V, DT, false, 1>(p, grid, smem, maps, st)
                           : launch_pipe_t<T, 2, V, DT, false, 2>(p, grid, smem, maps, st);
        case 4:
          return mode == 1 ? launch_pipe_t<T, 4, V, DT, false, 1>(p, grid, smem, maps, st)
                           : launch_pipe_t<T, 4, V, DT, false, 2>(p, grid, smem, maps, st);
        case 8:
          if constexpr (DT != 256)
            return mode == 1 ? launch_pipe_t<T, 8, 4, DT, false, 1>(p, grid, smem, maps, st)
                             : launch_pipe_t<T, 8, 4, DT, false, 2>(p, grid, smem, maps, st);
          break;
        default: break;
      }
      return cudaErrorInvalidValue;
    }
  }
  if (mode != 0) return cudaErrorInvalidValue;
  switch (G_T) {
    case 1:
      return big ? launch_pipe_t<T, 1, V, DT, true>(p, grid, smem, maps, st)
                 : launch_pipe_t<T, 1, V, DT, false>(p, grid, smem, maps, st);
    case 2: return launch_pipe_t<T, 2, V, DT, false>(p, grid, smem, maps, st);
    case 4: return launch_pipe_t<T, 4, V, DT, false>(p, grid, smem, maps, st);
    case 8:
      if constexpr (!(sizeof(T) == 2 && DT == 256)) return launch_pipe_t<T, 8, 4, DT, false>(p, grid, smem, maps, st);
      break;
    default: break;
  }
  return cudaErrorInvalidValue;
}
template <typename T, int DT>
int pipe_occ_dt(int G_T, size_t smem, bool big, int mode) {
  constexpr int V = sizeof(T) == 2 ? 8 : 4;
  if constexpr (sizeof(T) == 2) {
    if (mode == 3) return (G_T == 1 && !big) ? occupancy_t<T, 1, V, DT, false, 3>(smem) : 0;
    if (mode != 0) {
      switch (G_T) {
        case 1:
          if (mode == 1) return big ? occupancy_t<T, 1, V, DT, true, 1>(smem) : occupancy_t<T, 1, V, DT, false, 1>(smem);
          return big ? occupancy_t<T, 1, V, DT, true, 2>(smem) : occupancy_t<T, 1, V, DT, false, 2>(smem);
        case 2: return mode == 1 ? occupancy_t<T, 2, V, DT, false, 1>(smem) : occupancy_t<T, 2, V, DT, false, 2>(smem);
        case 4: return mode == 1 ? occupancy_t<T, 4, V, DT, false, 1>(smem) : occupancy_t<T, 4, V, DT, false, 2>(smem);
        case 8:
          if constexpr (DT != 256)
            return mode == 1 ? occupancy_t<T, 8, 4, DT, false, 1>(smem) : occupancy_t<T, 8, 4, DT, false, 2>(smem);
          break;
        default: break;
      }
      return 0;
    }
  }
  if (mode != 0) return 0;
  switch (G_T) {
    case 1: return big ? occupancy_t<T, 1, V, DT, true>(smem) : occupancy_t<T, 1, V, DT, false>(smem);
    case 2: return occupancy_t<T, 2, V, DT, false>(smem);
    case 4: return occupancy_t<T, 4, V, DT, false>(smem);
    case 8:
      if constexpr (!(sizeof(T) == 2 && DT == 256)) return occupancy_t<T, 8, 4, DT, false>(smem);
      break;
    default: break;
  }
  return 0;
}

#define LOKI_PIPE_SLICE(NAME, T, DT)                                                                        \
  cudaError_t pipe_launch_##NAME(const PipeParams& p, int G_T, int grid, size_t smem, const TmaDesc* maps,  \
                                 cudaStream_t st, bool big, int mode) {                                     \
    return pipe_launch_dt<T, DT>(p, G_T, grid, smem, maps, st, big, mode);                                  \
  }                                                                                                         \
  int pipe_occ_##NAME(int G_T, size_t smem, bool big, int mode) {                                           \
    return pipe_occ_dt<T, DT>(G_T, smem, big, mode);                                                        \
  }

}  // namespace loki
