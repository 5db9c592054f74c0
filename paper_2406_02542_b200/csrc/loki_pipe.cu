// Persistent pipelined Loki decode: host side (layout, dispatch).  The kernel
// itself lives in loki_pipe_impl.cuh; its instantiations are split across the
// loki_pipe_inst_*.cu translation units.
#include "loki_pipe_impl.cuh"

namespace loki {

cudaError_t pipe_launch_bf16_64(const PipeParams&, int, int, size_t, const TmaDesc*, cudaStream_t, bool, int);
int pipe_occ_bf16_64(int, size_t, bool, int);
cudaError_t pipe_launch_bf16_128(const PipeParams&, int, int, size_t, const TmaDesc*, cudaStream_t, bool, int);
int pipe_occ_bf16_128(int, size_t, bool, int);
cudaError_t pipe_launch_bf16_256(const PipeParams&, int, int, size_t, const TmaDesc*, cudaStream_t, bool, int);
int pipe_occ_bf16_256(int, size_t, bool, int);
cudaError_t pipe_launch_f32_64(const PipeParams&, int, int, size_t, const TmaDesc*, cudaStream_t, bool, int);
int pipe_occ_f32_64(int, size_t, bool, int);
cudaError_t pipe_launch_f32_128(const PipeParams&, int, int, size_t, const TmaDesc*, cudaStream_t, bool, int);
int pipe_occ_f32_128(int, size_t, bool, int);


int pipe_warps() { return kPW; }

size_t pipe_layout(int G_T, PipeParams* p) {
  size_t off = 0;
  p->off_ring = 0;
  off += (size_t)kPW * p->nst * p->stage_bytes;
  p->off_bars = (int)off;
  off = align_up(off + (size_t)(kPW * p->nst + 2) * 8, 16);
  p->off_hist = (int)off;
  const int hb = p->hbits > 8 ? p->hbits : 8;
  off = align_up(off + (size_t)G_T * (1u << hb) * 4, 16);
  p->off_ents = (int)off;
  const size_t ents_words = (size_t)p->Lc * (1 + (p->split_k ? G_T : 0));
  const size_t spec_words = p->spec ? (size_t)p->Lc * G_T : 0;
  off = align_up(off + 4 * (ents_words > spec_words ? ents_words : spec_words), 128);
  off += 1024;  // slack for aligning the dynamic shared memory base to 1024 B
  // ring during a selection: two key chunks of kCK keys, then three u64 candidate buffers
  const long long rest = (long long)kPW * p->nst * p->stage_bytes - 2LL * kCK * 4;
  p->cand_cap = rest > 0 ? (int)(rest / 24) : 0;
  return off;
}

bool pipe_supported(int dtype, int D, int G_T) {
  if (dtype == LOKI_DTYPE_BF16) return (D == 64 || D == 128 || (D == 256 && G_T <= 4)) && G_T <= 8;
  return (D == 64 || D == 128) && G_T <= 8;
}

int pipe_ctas_per_sm(int dtype, int D, int G_T, size_t smem, bool big, int mode) {
  if (dtype == LOKI_DTYPE_BF16) {
    if (D == 64) return pipe_occ_bf16_64(G_T, smem, big, mode);
    if (D == 128) return pipe_occ_bf16_128(G_T, smem, big, mode);
    if (D == 256) return pipe_occ_bf16_256(G_T, smem, big, mode);
  } else {
    if (D == 64) return pipe_occ_f32_64(G_T, smem, big, mode);
    if (D == 128) return pipe_occ_f32_128(G_T, smem, big, mode);
  }
  return 0;
}

size_t pipe_select_layout(PipeParams* p, bool onchip, int G_T) {
  size_t off = 0;
  p->off_ring = 0;
  off += (size_t)kPW * p->nst * p->stage_bytes;
  p->off_bars = (int)off;
  off = align_up(off + (size_t)(kPW * p->nst + 4 + kSelNB) * 8, 16);
  p->off_hist = (int)off;
  off = align_up(off + 2 * (size_t)G_T * (1u << p->hbits) * 4, 128);  // [2][G_T][HB]
  p->off_kchip = (int)off;  // on-chip keys [2][La], or the key stream's chunk buffers [kSelNB][kCK]
  off = align_up(off + (onchip ? 2 * (size_t)p->La : (size_t)sel_nb(G_T) * kCK) * 4, 128);
  p->off_cand = (int)off;
  p->cand_bytes = (onchip ? 16 : 32) * 1024;  // boundary-bin candidates, two buffers; more -> histogram levels
  off += (size_t)p->cand_bytes;
  if (G_T > 1) {  // tcgen05 phase 1: the query-term operand tile [N][lead row] (1024-byte aligned)
    off = align_up(off, 1024);
    p->off_qt = (int)off;
    off += (size_t)((3 * G_T + 15) / 16 * 16) * (size_t)(p->dbox * 2);
  }
  return off + 1024;  // slack for aligning the dynamic shared memory base to 1024 B
}

template <int RB, bool ONCHIP, int G_T>
KernelAttrs& select_attrs() {
  static KernelAttrs a;
  return a;
}

template <int RB, bool ONCHIP, int G_T>
static int select_occ(size_t smem) {
  return select_attrs<RB, ONCHIP, G_T>().occupancy(
      reinterpret_cast<const void*>(pipe_select_kernel<__nv_bfloat16, RB, ONCHIP, G_T>), 2 * kPT, smem);
}

template <int RB, bool ONCHIP, int G_T>
static cudaError_t launch_select_t(const PipeParams& p, int grid, size_t smem, const TmaDesc* maps, cudaStream_t st) {
  auto kern = pipe_select_kernel<__nv_bfloat16, RB, ONCHIP, G_T>;
  cudaError_t e = select_attrs<RB, ONCHIP, G_T>().ensure(reinterpret_cast<const void*>(kern), smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(2 * kPT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const CUtensorMap* m = reinterpret_cast<const CUtensorMap*>(maps);
  return cudaLaunchKernelEx(&cfg, kern, p, m[0]);
}

// Instantiations: G = 1 (MHA, group-shared) with on-chip or workspace keys; per-head groups of 2 / 4 / 8
// with workspace keys.  op = 0: occupancy for `smem`; op = 1: launch.
template <int RB>
static int select_dispatch(int op, bool onchip, int G_T, const PipeParams* p, int grid, size_t smem,
                           const TmaDesc* maps, cudaStream_t st, cudaError_t* err) {
#define LOKI_SEL(ONC, G)                                                          \
  {                                                                               \
    if (op == 0) return select_occ<RB, ONC, G>(smem);                             \
    *err = launch_select_t<RB, ONC, G>(*p, grid, smem, maps, st);                 \
    return 0;                                                                     \
  }
  if (G_T == 1) {
    if (onchip) LOKI_SEL(true, 1)
    LOKI_SEL(false, 1)
  }
  if (!onchip) {
    if (G_T == 2) LOKI_SEL(false, 2)
    if (G_T == 4) LOKI_SEL(false, 4)
    if (G_T == 8) LOKI_SEL(false, 8)
  }
#undef LOKI_SEL
  *err = cudaErrorInvalidValue;
  return 0;
}

int pipe_select_ctas_per_sm(int dtype, int lead_rb, bool onchip, size_t smem, int G_T) {
  if (dtype != LOKI_DTYPE_BF16) return 0;
  cudaError_t e = cudaSuccess;
  if (lead_rb == 64) return select_dispatch<64>(0, onchip, G_T, nullptr, 0, smem, nullptr, nullptr, &e);
  if (lead_rb == 128) return select_dispatch<128>(0, onchip, G_T, nullptr, 0, smem, nullptr, nullptr, &e);
  return 0;
}

cudaError_t launch_pipe_select(const PipeParams& p, int dtype, bool onchip, int grid, size_t smem,
                               const TmaDesc* maps, cudaStream_t st, int G_T) {
  if (dtype != LOKI_DTYPE_BF16) return cudaErrorInvalidValue;
  cudaError_t e = cudaErrorInvalidValue;
  if (p.lead_swz == 64) select_dispatch<64>(1, onchip, G_T, &p, grid, smem, maps, st, &e);
  else if (p.lead_swz == 128) select_dispatch<128>(1, onchip, G_T, &p, grid, smem, maps, st, &e);
  return e;
}

cudaError_t launch_pipe_weights(const PipeParams& p, cudaStream_t st) {
  pipe_weights_kernel<<<dim3((unsigned)p.units, (unsigned)p.G), 256, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_pipe(const PipeParams& p, int dtype, int G_T, int grid, size_t smem, const TmaDesc* maps,
                        cudaStream_t st, bool big, int mode) {
  if (dtype == LOKI_DTYPE_BF16) {
    if (p.D == 64) return pipe_launch_bf16_64(p, G_T, grid, smem, maps, st, big, mode);
    if (p.D == 128) return pipe_launch_bf16_128(p, G_T, grid, smem, maps, st, big, mode);
    if (p.D == 256) return pipe_launch_bf16_256(p, G_T, grid, smem, maps, st, big, mode);
  } else {
    if (p.D == 64) return pipe_launch_f32_64(p, G_T, grid, smem, maps, st, big, mode);
    if (p.D == 128) return pipe_launch_f32_128(p, G_T, grid, smem, maps, st, big, mode);
  }
  return cudaErrorInvalidValue;
}

}  // namespace loki
