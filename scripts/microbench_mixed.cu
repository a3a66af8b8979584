// Microbenchmark (diagnostics, GPU box): ingress of one stage of 64 gathered
// A^T rows x 256 tokens (32 KB, 128-B swizzled MN-major chunks) when the rows
// are split between TMA tile::gather4 (rows [0, R), issued by one thread) and
// 16-byte cp.async (rows [R, 64), 12 warps), both completing on the same
// mbarrier -- do the two paths add up?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lcuda -o mb_mixed microbench_mixed.cu
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "../paper_2402_10876_b200/csrc/sm100_ptx.cuh"

using namespace tw;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int kStage = 32768;
constexpr int kSt = 4;
constexpr int kNRows = 1536;
constexpr int kCpWarps = 12;

// warp 0: consumer (lane 0) ; warp 1: TMA issuer (lane 0) ; warps 2..: cp.async
__global__ void mixed_ring(const __grid_constant__ CUtensorMap gmap, const __half* at, int64_t ld,
                           const int* rows, int M, int iters, int R, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[kSt], empty[kSt];
  __shared__ int s_rows[kNRows];
  for (int i = threadIdx.x; i < kNRows; i += blockDim.x) s_rows[i] = rows[i];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ncp = 32 * kCpWarps;
  if (tid == 0) {
    for (int s = 0; s < kSt; ++s) {
      mbar_init(&full[s], ncp);
      mbar_init(&empty[s], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const long long t0 = clock64();
  auto rowbase = [&](int it) { return ((it + blockIdx.x * 7) * 64) % (kNRows - 64); };
  auto tokbase = [&](int it) { return ((it * 3 + blockIdx.x) * 256) % M; };
  if (warp == 0) {
    if (lane == 0)
      for (int it = 0; it < iters; ++it) {
        const int stage = it % kSt;
        mbar_wait(&full[stage], (it / kSt) & 1);
        mbar_arrive(&empty[stage]);
      }
  } else if (warp >= 2 && warp < 2 + kCpWarps) {
    const int t = tid - 64;
    for (int it = 0; it < iters; ++it) {
      const int stage = it % kSt;
      mbar_wait(&empty[stage], ((it / kSt) & 1) ^ 1u);
      const int kb = rowbase(it), m0 = tokbase(it);
      const uint32_t base = smem_u32(smem + stage * kStage);
      for (int c = t; c < (64 - R) * 32; c += ncp) {
        const int r = R + (c >> 5), j = c & 31;
        const int row = s_rows[kb + r];
        const uint32_t dst = base + (j >> 3) * 8192 + r * 128 + (((j & 7) ^ (r & 7)) << 4);
        cp_async_16(dst, at + static_cast<int64_t>(row) * ld + m0 + j * 8, 16);
      }
      if (lane == 0 && R > 0) {
        // this warp's share of the R/4 x 4 gather4 boxes
        const int cw = warp - 2;
        int mine = 0;
        for (int g = cw; g < R; g += kCpWarps) ++mine;
        if (mine) {
          asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(
                           smem_u32(&full[stage])),
                       "r"(mine * 512)
                       : "memory");
          for (int g = cw; g < R; g += kCpWarps) {  // g = (r4 / 4) * 4 + ch
            const int r4 = (g >> 2) * 4, ch = g & 3;
            const int* rr = s_rows + kb + r4;
            tma_gather4(smem + stage * kStage + ch * 8192 + r4 * 128, &gmap, &full[stage],
                        m0 + ch * 64, rr[0], rr[1], rr[2], rr[3]);
          }
        }
      }
      cp_async_mbar_arrive_noinc(&full[stage]);
    }
  }
  __syncthreads();
  if (tid == 0) cycles[blockIdx.x] = clock64() - t0;
}

int main() {
  const int K = 3072, M = 8192, iters = 300;
  std::vector<int> rows(K);
  for (int i = 0; i < K; ++i) rows[i] = i;
  std::mt19937 rng(1);
  std::shuffle(rows.begin(), rows.end(), rng);
  rows.resize(kNRows);
  std::sort(rows.begin(), rows.end());
  __half* at;
  int* drows;
  long long* cyc;
  CK(cudaMalloc(&at, (size_t)K * M * 2));
  CK(cudaMemset(at, 0, (size_t)K * M * 2));
  CK(cudaMalloc(&drows, kNRows * 4));
  CK(cudaMemcpy(drows, rows.data(), kNRows * 4, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&cyc, 148 * 8));
  void* fn;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  auto encode = (CUresult(*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill))fn;
  CUtensorMap gmap;
  cuuint64_t dims[2] = {(cuuint64_t)M, (cuuint64_t)K};
  cuuint64_t strides[1] = {(cuuint64_t)M * 2};
  cuuint32_t gbox[2] = {64, 1}, es[2] = {1, 1};
  encode(&gmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, at, dims, strides, gbox, es,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int smem = kSt * kStage + 1024;
  CK(cudaFuncSetAttribute(mixed_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int R : {0, 8, 16, 24, 32, 48, 64}) {
    float ms = 0;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      mixed_ring<<<148, 32 * (2 + kCpWarps), smem>>>(gmap, at, M, drows, M, iters, R, cyc);
      cudaEventRecord(e1);
      CK(cudaDeviceSynchronize());
      cudaEventElapsedTime(&ms, e0, e1);
    }
    std::vector<long long> c(148);
    CK(cudaMemcpy(c.data(), cyc, 148 * 8, cudaMemcpyDeviceToHost));
    std::sort(c.begin(), c.end());
    const double bytes = 148.0 * iters * kStage;
    printf("gather4 rows %2d / cp.async rows %2d : %8.1f GB/s  %6.1f B/cyc/SM (median)\n", R,
           64 - R, bytes / ms / 1e6, (double)iters * kStage / c[74]);
  }
  return 0;
}
