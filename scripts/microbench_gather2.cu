// Microbenchmark (diagnostics, GPU box): ingress of one 32 KB stage
// ([64 gathered A^T rows] x [256 tokens], 128-B swizzled MN-major chunks) with
//   * dense TMA 2-D boxes (4 x {64 tok, 64 rows})      -- upper bound
//   * TMA tile::gather4 (64 requests), indices in smem, I issuing threads
//   * cp.async 16 B, indices in smem, W warps
// for grid = 148 and 96 CTAs.  Consumer: the ring slot is recycled as soon as
// its bytes have landed (no MMA).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lcuda -o mb_gather2 microbench_gather2.cu
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
constexpr int kSt = 6;  // max stages (runtime nst <= kSt)
constexpr int kNRows = 1536;

__device__ __forceinline__ void load_rows(int* s_rows, const int* rows) {
  for (int i = threadIdx.x; i < kNRows; i += blockDim.x) s_rows[i] = rows[i];
}

// mode 0 dense TMA, 1 gather4
__global__ void tma_ring(const __grid_constant__ CUtensorMap map, const int* rows, int M,
                         int iters, int issuers, int mode, long long* cycles, int nst) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar[kSt];
  __shared__ int s_rows[kNRows];
  load_rows(s_rows, rows);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < nst; ++s) mbar_init(&bar[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  const long long t0 = clock64();
  if (lane == 0 && warp < issuers) {
    for (int it = 0; it < iters + nst; ++it) {
      const int stage = it % nst;
      if (it >= nst) mbar_wait(&bar[stage], ((it / nst) - 1) & 1);
      if (it >= iters) continue;
      if (warp == 0) mbar_arrive_expect_tx(&bar[stage], kStage);
      const int kb = ((it + blockIdx.x * 7) * 64) % (kNRows - 64);
      const int m0 = ((it * 3 + blockIdx.x) * 256) % M;
      uint8_t* dst = smem + stage * kStage;
      if (mode == 0) {
        for (int ch = warp; ch < 4; ch += issuers)
          tma_load_2d(dst + ch * 8192, &map, &bar[stage], m0 + ch * 64, s_rows[kb]);
      } else {
        for (int g = warp; g < 64; g += issuers) {
          const int ch = g >> 4, r4 = (g & 15) * 4;
          const int* rr = s_rows + kb + r4;
          tma_gather4(dst + ch * 8192 + r4 * 128, &map, &bar[stage], m0 + ch * 64, rr[0], rr[1],
                      rr[2], rr[3]);
        }
      }
    }
  }
  __syncthreads();
  if (tid == 0) cycles[blockIdx.x] = clock64() - t0;
}

__global__ void cp_ring(const __half* at, int64_t ld, const int* rows, int M, int iters,
                        long long* cycles, int nst) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ int s_rows[kNRows];
  load_rows(s_rows, rows);
  __syncthreads();
  const int tid = threadIdx.x, nthr = blockDim.x;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int stage = it % nst;
    const int kb = ((it + blockIdx.x * 7) * 64) % (kNRows - 64);
    const int m0 = ((it * 3 + blockIdx.x) * 256) % M;
    const uint32_t base = smem_u32(smem + stage * kStage);
    // 64 rows x 32 16-byte chunks (256 tokens); consecutive threads take
    // consecutive chunks of one row (512 contiguous bytes per row)
    for (int c = tid; c < 2048; c += nthr) {
      const int r = c >> 5, j = c & 31;
      const int row = s_rows[kb + r];
      const uint32_t dst = base + (j >> 3) * 8192 + r * 128 + (((j & 7) ^ (r & 7)) << 4);
      cp_async_16(dst, at + static_cast<int64_t>(row) * ld + m0 + j * 8, 16);
    }
    asm volatile("cp.async.commit_group;");
    if (nst <= 2) asm volatile("cp.async.wait_group 0;" ::: "memory");
    else if (nst <= 4) asm volatile("cp.async.wait_group 2;" ::: "memory");
    else asm volatile("cp.async.wait_group 4;" ::: "memory");
  }
  asm volatile("cp.async.wait_group 0;");
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
  CUtensorMap dmap, gmap;
  cuuint64_t dims[2] = {(cuuint64_t)M, (cuuint64_t)K};
  cuuint64_t strides[1] = {(cuuint64_t)M * 2};
  cuuint32_t dbox[2] = {64, 64}, gbox[2] = {64, 1}, es[2] = {1, 1};
  encode(&dmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, at, dims, strides, dbox, es,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  encode(&gmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, at, dims, strides, gbox, es,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int smem = kSt * kStage + 1024;
  CK(cudaFuncSetAttribute(tma_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(cp_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  char name[64];
  for (int nst : {2, 4, 6}) for (int grid : {148, 96}) {
    auto report = [&](const char* name) {
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      std::vector<long long> c(grid);
      CK(cudaMemcpy(c.data(), cyc, grid * 8, cudaMemcpyDeviceToHost));
      std::sort(c.begin(), c.end());
      const double bytes = (double)grid * iters * kStage;
      printf("grid %3d %-26s %8.1f GB/s  %6.1f B/cyc/SM (median)\n", grid, name,
             bytes / ms / 1e6, (double)iters * kStage / c[grid / 2]);
    };
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      tma_ring<<<grid, 128, smem>>>(dmap, drows, M, iters, 1, 0, cyc, nst);
      cudaEventRecord(e1);
      CK(cudaDeviceSynchronize());
    }
    snprintf(name, 64, "dense tma 2d st%d", nst);
    report(name);
    for (int is : {8}) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        tma_ring<<<grid, 32 * std::max(is, 4), smem>>>(gmap, drows, M, iters, is, 1, cyc, nst);
        cudaEventRecord(e1);
        CK(cudaDeviceSynchronize());
      }
      snprintf(name, 64, "gather4 %d issuers st%d", is, nst);
      report(name);
    }
    for (int w : {4, 8, 16}) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        cp_ring<<<grid, 32 * w, smem>>>(at, M, drows, M, iters, cyc, nst);
        cudaEventRecord(e1);
        CK(cudaDeviceSynchronize());
      }
      snprintf(name, 64, "cp.async %d warps st%d", w, nst);
      report(name);
    }
  }
  return 0;
}
