// TMA streaming microbenchmark (not part of the library): achievable HBM
// bandwidth of the Loki access patterns with NO compute, as a function of
// warps per CTA, ring stages per warp and CTAs per SM.
//   mode 0: gather4 of sorted random rows (25 % of 4096-row regions), full 256 B rows
//   mode 1: same rows as two 128 B halves, SWIZZLE_128B (the tensor-core layout)
//   mode 2: 4-D-style lead boxes: 64 B of every 256 B row (L2 promotion 64 B)
//   mode 3: contiguous 256 B rows (dense)
//   mode 4: gather4 of 512 B rows (K and V rows interleaved: one selected row = K row + V row)
//   mode 5: the interleaved rows of mode 4 fetched as the kernel's B items do: four 128 B swizzled halves
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gb tools/gatherbench.cu -lcuda
//   /tmp/gb <mode> <warps> <stages> <stage_kb> <ctas_per_sm>
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));        \
      return 1;                                                                \
    }                                                                          \
  } while (0)

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t* b) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(b))); }
__device__ __forceinline__ void bar_tx(uint64_t* b, unsigned n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, unsigned ph) {
  asm volatile(
      "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(su(b)),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void g4(void* dst, const CUtensorMap* m, int col, int r0, int r1, int r2, int r3, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
      "%5, %6}], [%7];" ::"r"(su(dst)),
      "l"(m), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(su(b))
      : "memory");
}
__device__ __forceinline__ void box2(void* dst, const CUtensorMap* m, int c0, int c1, uint64_t* b) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
                   "r"(su(dst)),
               "l"(m), "r"(c0), "r"(c1), "r"(su(b))
               : "memory");
}

struct Args {
  int mode, nst, sb, items, rows_per_item, sel_per_item;
  const int* idx;  // [items][sel_per_item] sorted rows (absolute)
  unsigned* ticket;
};

__global__ void bench(Args a, const __grid_constant__ CUtensorMap full, const __grid_constant__ CUtensorMap half,
                      const __grid_constant__ CUtensorMap lead, const __grid_constant__ CUtensorMap wide, const __grid_constant__ CUtensorMap whalf) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (su(smem_raw) & 1023u)) & 1023u);
  __shared__ int s_item;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint8_t* ring = smem + (size_t)w * a.nst * a.sb;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)nw * a.nst * a.sb) + w * a.nst;
  if (lane == 0)
    for (int s = 0; s < a.nst; ++s) bar_init(&bars[s]);
  __syncwarp();
  int slot = 0;
  unsigned phase = 0;
  int used = 0;
  // rows per stage: mode 0 sb/256, mode 1 sb/256 (two halves), mode 2 sb/64 lead rows, mode 3 sb/256
  const int rps = (a.mode == 2) ? a.sb / 64 : (a.mode >= 4 ? a.sb / 512 : a.sb / 256);
  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(a.ticket, 1);
    __syncthreads();
    const int it = s_item;
    __syncthreads();
    if (it >= a.items) break;
    const int nrows = (a.mode != 2 && a.mode != 3) ? a.sel_per_item : a.rows_per_item;
    const int nstage = (nrows + rps - 1) / rps;
    const int* idx = a.idx + (size_t)it * a.sel_per_item;
    const int base = it * a.rows_per_item;
    auto issue = [&](int st, int sl) {
      uint8_t* dst = ring + sl * a.sb;
      if (lane == 0) bar_tx(&bars[sl], (unsigned)a.sb);
      if (a.mode == 2 || a.mode == 3) {
        if (lane == 0) {
          if (a.mode == 2) box2(dst, &lead, 0, base + st * rps, &bars[sl]);
          else box2(dst, &full, 0, base + st * rps, &bars[sl]);
        }
        return;
      }
      int row = -1;
      if (lane < rps && st * rps + lane < nrows) row = idx[st * rps + lane];
      for (int q = 0; q < rps / 4; ++q) {
        const int r0 = __shfl_sync(~0u, row, 4 * q), r1 = __shfl_sync(~0u, row, 4 * q + 1);
        const int r2 = __shfl_sync(~0u, row, 4 * q + 2), r3 = __shfl_sync(~0u, row, 4 * q + 3);
        if (lane == 0) {
          if (a.mode == 4) {
            g4(dst + q * 2048, &wide, 0, r0, r1, r2, r3, &bars[sl]);
          } else if (a.mode == 5) {
            for (int hh = 0; hh < 4; ++hh) g4(dst + hh * rps * 128 + q * 512, &whalf, 64 * hh, r0, r1, r2, r3, &bars[sl]);
          } else if (a.mode == 0) {
            g4(dst + q * 1024, &full, 0, r0, r1, r2, r3, &bars[sl]);
          } else {
            g4(dst + q * 512, &half, 0, r0, r1, r2, r3, &bars[sl]);
            g4(dst + rps * 128 + q * 512, &half, 64, r0, r1, r2, r3, &bars[sl]);
          }
        }
      }
    };
    const int mine = nstage > w ? (nstage - w + nw - 1) / nw : 0;
    {
      int s2 = slot;
      for (int k = 0; k < a.nst && k < mine; ++k) {
        issue(w + k * nw, s2);
        s2 = (s2 + 1) % a.nst;
      }
    }
    for (int k = 0; k < mine; ++k) {
      bar_wait(&bars[slot], phase);
      __syncwarp();
      if (k + a.nst < mine) issue(w + (k + a.nst) * nw, slot);
      if (++slot == a.nst) {
        slot = 0;
        phase ^= 1u;
      }
      ++used;
    }
  }
  if (threadIdx.x == 0 && blockIdx.x == 0 && used < 0) printf("%d\n", used);
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0;
  const int nw = argc > 2 ? atoi(argv[2]) : 8;
  const int nst = argc > 3 ? atoi(argv[3]) : 2;
  const int sb = (argc > 4 ? atoi(argv[4]) : 8) * 1024;
  const int per_sm = argc > 5 ? atoi(argv[5]) : 2;
  const size_t total_rows = (size_t)1 << 24;  // 16 M rows x 256 B = 4 GiB
  const int rows_per_item = mode == 2 ? 4096 : 4096;
  const int items = (int)(total_rows / rows_per_item);
  const int sel = rows_per_item / 4;
  uint8_t* buf;
  const size_t row_bytes = mode >= 4 ? 512 : 256;
  CK(cudaMalloc(&buf, total_rows * row_bytes));
  CK(cudaMemset(buf, 1, total_rows * row_bytes));
  std::vector<int> h((size_t)items * sel);
  std::mt19937 rng(1);
  std::vector<int> perm(rows_per_item);
  for (int i = 0; i < rows_per_item; ++i) perm[i] = i;
  for (int it = 0; it < items; ++it) {
    std::shuffle(perm.begin(), perm.end(), rng);
    std::vector<int> s(perm.begin(), perm.begin() + sel);
    std::sort(s.begin(), s.end());
    for (int j = 0; j < sel; ++j) h[(size_t)it * sel + j] = it * rows_per_item + s[j];
  }
  int* idx;
  unsigned* ticket;
  CK(cudaMalloc(&idx, h.size() * 4));
  CK(cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&ticket, 4));
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  EncFn enc = (EncFn)fn;
  CUtensorMap full, half, lead, wide, whalf;
  cuuint64_t wdims[2] = {256, total_rows};
  cuuint64_t wstr[1] = {512};
  cuuint32_t bwide[2] = {256, 1};
  cuuint64_t dims[2] = {128, total_rows};
  cuuint64_t str[1] = {256};
  cuuint32_t es[2] = {1, 1};
  cuuint32_t bfull[2] = {128, mode == 3 ? (cuuint32_t)(sb / 256) : 1u};
  cuuint32_t bhalf[2] = {64, 1};
  cuuint32_t blead[2] = {32, (cuuint32_t)std::min(256, sb / 64)};
  if (enc(&full, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, bfull, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ||
      enc(&half, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, bhalf, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ||
      enc(&lead, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, blead, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_64B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ||
      enc(&wide, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, wdims, wstr, bwide, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ||
      enc(&whalf, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, wdims, wstr, bhalf, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)) {
    printf("encode failed\n");
    return 1;
  }
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t smem = (size_t)nw * nst * sb + nw * nst * 8 + 1024;
  CK(cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, bench, nw * 32, smem));
  const int cps = std::min(per_sm, occ);
  Args a{mode, nst, sb, items, rows_per_item, sel, idx, ticket};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    CK(cudaMemset(ticket, 0, 4));
    cudaEventRecord(e0);
    bench<<<sms * cps, nw * 32, smem>>>(a, full, half, lead, wide, whalf);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = std::min(best, ms);
  }
  CK(cudaGetLastError());
  double bytes = mode >= 4 ? (double)items * sel * 512 : (mode == 0 || mode == 1) ? (double)items * sel * 256 : (mode == 2 ? (double)total_rows * 64 : (double)total_rows * 256);
  printf("mode %d warps %d stages %d stage_kb %d ctas/sm %d (occ %d): %.1f us, %.0f GB/s\n", mode, nw, nst, sb / 1024, cps,
         occ, best * 1e3, bytes / (best * 1e-3) / 1e9);
  return 0;
}
