// Micro-probe of DRAM over-fetch for the two Loki access patterns on B200:
//   lead:   64 B (the leading d = 32 bf16 columns) of every 256 B row
//   gather: full 256 B rows / 64 B segments at sorted random 25 % positions
// for LDG flavours, TMA 2-D boxes (with / without L2 promotion) and bulk
// copies.  Run under ncu (dram__bytes_read.sum) to see what the memory system
// fetches.  Not part of the library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2probe tools/l2probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint4 ld_nc(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

// 4 lanes x 16 B per 256 B row, 8 rows per warp instruction, unrolled 8
__global__ void lead_kernel(const uint8_t* buf, size_t rows, unsigned* sink) {
  const size_t lane = threadIdx.x & 31;
  const size_t warp = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const size_t nwarps = (gridDim.x * (size_t)blockDim.x) >> 5;
  unsigned acc = 0;
  for (size_t r0 = warp * 64; r0 < rows; r0 += nwarps * 64) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = ld_nc(buf + (r0 + u * 8 + lane / 4) * 256 + (lane % 4) * 16);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678u) *sink = acc;
}

__global__ void stream_kernel(const uint8_t* buf, size_t bytes, unsigned* sink) {
  const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  const size_t n = gridDim.x * (size_t)blockDim.x;
  unsigned acc = 0;
  for (size_t i = tid * 16; i < bytes; i += n * 16 * 4) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      size_t o = i + (size_t)u * n * 16;
      v[u] = o < bytes ? ld_nc(buf + o) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) acc ^= v[u].x ^ v[u].w;
  }
  if (acc == 0x12345678u) *sink = acc;
}

template <int SEG>
__global__ void gather_kernel(const uint8_t* buf, const uint32_t* idx, size_t n, size_t stride, unsigned* sink) {
  constexpr int LPR = SEG / 16;
  constexpr int RPW = 32 / LPR;
  const size_t lane = threadIdx.x & 31;
  const size_t warp = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const size_t nwarps = (gridDim.x * (size_t)blockDim.x) >> 5;
  unsigned acc = 0;
  for (size_t j0 = warp * RPW * 8; j0 < n; j0 += nwarps * RPW * 8) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      size_t j = j0 + u * RPW + lane / LPR;
      v[u] = j < n ? ld_nc(buf + (size_t)idx[j] * stride + (lane % LPR) * 16) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].w;
  }
  if (acc == 0x12345678u) *sink = acc;
}

// ---------------------------------------------------------------- TMA / bulk
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(bar)), "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" :: "r"((unsigned)__cvta_generic_to_shared(bar)), "r"(phase));
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      :: "r"((unsigned)__cvta_generic_to_shared(dst)), "l"(map), "r"(x), "r"(y),
         "r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ void bulk_1d(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      :: "r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes),
         "r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
}

constexpr int kBoxRows = 256, kStages = 4;

// each CTA streams boxes of [256 rows x 32 bf16] through a 4-stage ring
__global__ void tma_lead_kernel(const __grid_constant__ CUtensorMap map, int rows, unsigned* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t bar[kStages];
  const int boxes = rows / kBoxRows;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  unsigned acc = 0;
  int it = 0;
  int issued = 0;
  int my0 = blockIdx.x;
  // prologue
  if (threadIdx.x == 0)
    for (int s = 0; s < kStages && my0 + s * (int)gridDim.x < boxes; ++s) {
      mbar_expect(&bar[s], kBoxRows * 64);
      tma_2d(sm + s * kBoxRows * 64, &map, 0, (my0 + s * gridDim.x) * kBoxRows, &bar[s]);
      ++issued;
    }
  for (int b = my0; b < boxes; b += gridDim.x, ++it) {
    const int s = it % kStages;
    mbar_wait(&bar[s], (it / kStages) & 1);
    acc ^= reinterpret_cast<const unsigned*>(sm + s * kBoxRows * 64)[threadIdx.x];
    __syncthreads();
    const int nb = b + kStages * gridDim.x;
    if (threadIdx.x == 0 && nb < boxes) {
      mbar_expect(&bar[s], kBoxRows * 64);
      tma_2d(sm + s * kBoxRows * 64, &map, 0, nb * kBoxRows, &bar[s]);
    }
  }
  if (acc == 0x12345678u) *sink = acc;
}

// bulk-copy gather: one elected thread per warp issues SEG-byte copies of 32 rows
template <int SEG>
__global__ void bulk_gather_kernel(const uint8_t* buf, const uint32_t* idx, size_t n, size_t stride, unsigned* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t bar[8][2];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* wbuf = sm + (size_t)w * 2 * 32 * SEG;
  if (lane == 0) {
    mbar_init(&bar[w][0], 1);
    mbar_init(&bar[w][1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  const size_t warp = blockIdx.x * (blockDim.x / 32) + w;
  const size_t nwarps = gridDim.x * (blockDim.x / 32);
  unsigned acc = 0;
  int it = 0;
  for (size_t j0 = warp * 32; j0 < n; j0 += nwarps * 32, ++it) {
    const int s = it & 1;
    const int cnt = (int)min((size_t)32, n - j0);
    if (lane == 0) mbar_expect(&bar[w][s], cnt * SEG);
    __syncwarp();
    if (lane < cnt) bulk_1d(wbuf + (s * 32 + lane) * SEG, buf + (size_t)idx[j0 + lane] * stride, SEG, &bar[w][s]);
    mbar_wait(&bar[w][s], (it >> 1) & 1);
    acc ^= reinterpret_cast<const unsigned*>(wbuf + s * 32 * SEG)[lane];
    __syncwarp();
  }
  if (acc == 0x12345678u) *sink = acc;
}

// TMA gather4: 32 selected rows per stage via 8 gather4 (lanes 0..7 of warp 0), 4-stage ring
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* map, int col, int r0, int r1, int r2, int r3,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
      :: "r"((unsigned)__cvta_generic_to_shared(dst)), "l"(map), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
         "r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
}

__global__ void tma_gather_kernel(const __grid_constant__ CUtensorMap map, const uint32_t* idx, int n, unsigned* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t bar[kStages];
  constexpr int R = 32, ROWB = 256, STB = R * ROWB;
  const int chunks = (n + R - 1) / R;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  auto issue = [&](int c, int s) {
    const int lane = threadIdx.x;
    if (lane == 0) mbar_expect(&bar[s], STB);
    __syncwarp(0xff);
    const int j = c * R + lane * 4;
    int r[4];
    for (int t = 0; t < 4; ++t) r[t] = (j + t < n) ? (int)idx[j + t] : -1;
    tma_gather4(sm + s * STB + lane * 4 * ROWB, &map, 0, r[0], r[1], r[2], r[3], &bar[s]);
  };
  unsigned acc = 0;
  int it = 0;
  if (threadIdx.x < 8)
    for (int s = 0; s < kStages && (int)blockIdx.x + s * (int)gridDim.x < chunks; ++s) issue(blockIdx.x + s * gridDim.x, s);
  for (int c = blockIdx.x; c < chunks; c += gridDim.x, ++it) {
    const int s = it % kStages;
    mbar_wait(&bar[s], (it / kStages) & 1);
    acc ^= reinterpret_cast<const unsigned*>(sm + s * STB)[threadIdx.x];
    __syncthreads();
    const int nc = c + kStages * gridDim.x;
    if (threadIdx.x < 8 && nc < chunks) issue(nc, s);
  }
  if (acc == 0x12345678u) *sink = acc;
}

// cp.async (LDGSTS) gather of 256 B rows, per-warp 4-stage ring of 8 rows
__global__ void cpasync_gather_kernel(const uint8_t* buf, const uint32_t* idx, size_t n, unsigned* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int RW = 8, ST = 4;  // rows per warp stage, stages
  uint8_t* wb = sm + (size_t)w * ST * RW * 256;
  const size_t warp = blockIdx.x * (blockDim.x / 32) + w;
  const size_t nwarps = gridDim.x * (blockDim.x / 32);
  unsigned acc = 0;
  size_t it = 0;
  auto issue = [&](size_t j0, int s) {
    for (int q = 0; q < 4; ++q) {  // 8 rows x 256 B = 128 chunks of 16 B, 4 per lane
      const int ch = q * 32 + lane;
      const int row = ch / 16, off = (ch % 16) * 16;
      const size_t j = j0 + row;
      const uint8_t* src = buf + (size_t)(j < n ? idx[j] : idx[0]) * 256 + off;
      unsigned dst = (unsigned)__cvta_generic_to_shared(wb + (s * RW + row) * 256 + off);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(dst), "l"(src));
    }
    asm volatile("cp.async.commit_group;");
  };
  size_t j = warp * RW;
  for (int s = 0; s < ST - 1; ++s) { if (j + s * nwarps * RW < n) issue(j + s * nwarps * RW, s); else asm volatile("cp.async.commit_group;"); }
  for (; j < n; j += nwarps * RW, ++it) {
    const int s = it % ST;
    const size_t jn = j + (ST - 1) * nwarps * RW;
    if (jn < n) issue(jn, (it + ST - 1) % ST); else asm volatile("cp.async.commit_group;");
    asm volatile("cp.async.wait_group 3;");
    __syncwarp();
    acc ^= reinterpret_cast<const unsigned*>(wb + s * RW * 256)[lane];
    __syncwarp();
  }
  asm volatile("cp.async.wait_all;");
  if (acc == 0x12345678u) *sink = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const size_t rows = (size_t)16 << 20;  // 16 M rows x 256 B = 4 GiB
  const size_t bytes = rows * 256;
  uint8_t* buf;
  unsigned* sink;
  CK(cudaMalloc(&buf, bytes));
  CK(cudaMalloc(&sink, 4));
  CK(cudaMemset(buf, 1, bytes));
  std::vector<uint32_t> h;
  std::mt19937 rng(1);
  for (uint32_t r = 0; r < rows; ++r)
    if ((rng() & 3u) == 0) h.push_back(r);
  uint32_t* idx;
  CK(cudaMalloc(&idx, h.size() * 4));
  CK(cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](const char* name, double useful, auto launch) {
    launch();
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); exit(1); }
    cudaEventRecord(a);
    for (int i = 0; i < 5; ++i) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-30s %8.1f us  useful %7.1f MB  %7.1f GB/s useful\n", name, ms * 200.0, useful / 1e6,
           useful / (ms / 5 * 1e-3) / 1e9);
  };
  const int grid = 148 * 8, block = 256;
  const double lead = rows * 64.0;
  timeit("lead64 ldg.nc", lead, [&] { lead_kernel<<<grid, block>>>(buf, rows, sink); });
  timeit("stream same bytes", lead, [&] { stream_kernel<<<grid, block>>>(buf, (size_t)lead, sink); });
  timeit("stream 4GiB", bytes, [&] { stream_kernel<<<grid, block>>>(buf, bytes, sink); });

  EncodeFn encode = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q));
  for (int promo = 0; promo < 4; ++promo) {
    CUtensorMap map;
    cuuint64_t dims[2] = {128, (cuuint64_t)rows};
    cuuint64_t strides[1] = {256};
    cuuint32_t box[2] = {32, kBoxRows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        (CUtensorMapL2promotion)promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
    char nm[64];
    snprintf(nm, sizeof(nm), "lead64 tma promo=%d", promo);
    const int smem = kStages * kBoxRows * 64;
    cudaFuncSetAttribute(tma_lead_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    timeit(nm, lead, [&] { tma_lead_kernel<<<148 * 3, 256, smem>>>(map, (int)rows, sink); });
  }
  timeit("gather 256B rows ldg", h.size() * 256.0, [&] { gather_kernel<256><<<grid, block>>>(buf, idx, h.size(), 256, sink); });
  timeit("gather 64B segs ldg", h.size() * 64.0, [&] { gather_kernel<64><<<grid, block>>>(buf, idx, h.size(), 64, sink); });
  timeit("gather 128B segs ldg", h.size() * 128.0, [&] { gather_kernel<128><<<grid, block>>>(buf, idx, h.size(), 128, sink); });
  {
    const int smem = 8 * 2 * 32 * 64;
    cudaFuncSetAttribute(bulk_gather_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    timeit("gather 64B segs bulk", h.size() * 64.0, [&] { bulk_gather_kernel<64><<<grid, block, smem>>>(buf, idx, h.size(), 64, sink); });
    const int smem2 = 8 * 2 * 32 * 256;
    cudaFuncSetAttribute(bulk_gather_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2);
    timeit("gather 256B rows bulk", h.size() * 256.0, [&] { bulk_gather_kernel<256><<<148 * 2, block, smem2>>>(buf, idx, h.size(), 256, sink); });
  }

  {
    CUtensorMap gmap;
    cuuint64_t dims[2] = {128, (cuuint64_t)rows};
    cuuint64_t strides[1] = {256};
    cuuint32_t box[2] = {128, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = encode(&gmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("gather encode failed %d\n", (int)r); return 1; }
    const int smem = kStages * 32 * 256;
    cudaFuncSetAttribute(tma_gather_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int occ : {2, 4, 6})
      timeit(occ == 2 ? "gather 256B tma4 x2" : occ == 4 ? "gather 256B tma4 x4" : "gather 256B tma4 x6",
             h.size() * 256.0, [&] { tma_gather_kernel<<<148 * occ, 256, smem>>>(gmap, idx, (int)h.size(), sink); });
    const int smem2 = 8 * 4 * 8 * 256;
    cudaFuncSetAttribute(cpasync_gather_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2);
    for (int occ : {2, 3})
      timeit(occ == 2 ? "gather 256B cp.async x2" : "gather 256B cp.async x3", h.size() * 256.0,
             [&] { cpasync_gather_kernel<<<148 * occ, 256, smem2>>>(buf, idx, h.size(), sink); });
  }
  CK(cudaDeviceSynchronize());
  return 0;
}
