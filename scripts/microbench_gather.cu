// Microbenchmark (diagnostics, GPU box): achievable row-gather bandwidth into
// shared memory on sm_100a for the TW activation gather (64 kept rows x 128
// tokens x fp16 = 16 KB per stage), comparing
//   (a) cp.async 16-byte chunks issued by W warps,
//   (b) TMA tile::gather4 (4 rows x 64 tokens per request) issued by 1..W threads,
//   (c) dense TMA 2-D tiles (64 rows x 64 tokens) as the upper reference.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mb microbench_gather.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>

#include "../paper_2402_10876_b200/csrc/sm100_ptx.cuh"

using namespace tw;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int kStageBytes = 16384;
constexpr int kStages = 8;

__global__ void gather_cpasync(const __half* at, int64_t ld, const int* rows, int nrows, int M,
                               int iters, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x, nthr = blockDim.x;
  long long t0 = clock64();
  int stage = 0;
  for (int it = 0; it < iters; ++it) {
    const int kb = (it * 64 + blockIdx.x * 64) % (nrows - 64);
    const int m0 = ((it + blockIdx.x) * 128) % M;
    const uint32_t base = smem_u32(smem + stage * kStageBytes);
    for (int c = tid; c < 1024; c += nthr) {
      const int r = c >> 4, j = c & 15;
      const int row = rows[kb + r];
      const uint32_t dst = base + (j >> 3) * 8192 + r * 128 + (((j & 7) ^ (r & 7)) << 4);
      cp_async_16(dst, at + (int64_t)row * ld + m0 + j * 8, 16);
    }
    asm volatile("cp.async.commit_group;");
    asm volatile("cp.async.wait_group 6;");
    stage = (stage + 1) % kStages;
  }
  asm volatile("cp.async.wait_group 0;");
  __syncthreads();
  if (tid == 0) cycles[blockIdx.x] = clock64() - t0;
}

__global__ void gather_tma4(const __grid_constant__ CUtensorMap map, const int* rows, int nrows,
                            int M, int iters, int issuers, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[kStages];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&bar[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  long long t0 = clock64();
  const int warp = tid >> 5, lane = tid & 31;
  const int per = 32 / issuers;
  if (lane == 0 && warp < issuers) {
    for (int it = 0; it < iters; ++it) {
      const int stage = it % kStages;
      if (it >= kStages) mbar_wait(&bar[stage], ((it / kStages) - 1) & 1);
      if (warp == 0) mbar_arrive_expect_tx(&bar[stage], kStageBytes);
      const int kb = (it * 64 + blockIdx.x * 64) % (nrows - 64);
      const int m0 = ((it + blockIdx.x) * 128) % M;
      for (int g = warp * per; g < (warp + 1) * per; ++g) {
        const int half = g >> 4, r4 = (g & 15) * 4;
        const int* rr = rows + kb + r4;
        tma_gather4(smem + stage * kStageBytes + half * 8192 + r4 * 128, &map, &bar[stage],
                    m0 + half * 64, rr[0], rr[1], rr[2], rr[3]);
      }
    }
    for (int it = iters; it < iters + kStages; ++it) {
      const int stage = it % kStages;
      if (it >= kStages && warp == 0) mbar_wait(&bar[stage], ((it / kStages) - 1) & 1);
    }
  }
  __syncthreads();
  if (tid == 0) cycles[blockIdx.x] = clock64() - t0;
}

__global__ void gather_hybrid(const __grid_constant__ CUtensorMap map, const __half* at, int64_t ld,
                              const int* rows, int nrows, int M, int iters, int tma_warps,
                              long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[kStages];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&bar[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  long long t0 = clock64();
  const int warp = tid >> 5, lane = tid & 31;
  const int cp_threads = blockDim.x - 32 * tma_warps;
  int stage = 0;
  for (int it = 0; it < iters + kStages; ++it) {
    stage = it % kStages;
    const int kb = (it * 64 + blockIdx.x * 64) % (nrows - 64);
    const int m0 = ((it + blockIdx.x) * 128) % M;
    if (warp < tma_warps) {
      if (lane == 0) {
        if (it >= kStages) mbar_wait(&bar[stage], ((it / kStages) - 1) & 1);
        if (it < iters) {
          if (warp == 0) mbar_arrive_expect_tx(&bar[stage], kStageBytes / 2);
          // rows 32..63 via gather4: 8 row-groups x 2 halves = 16 requests
          const int per = 16 / tma_warps;
          for (int g = warp * per; g < (warp + 1) * per; ++g) {
            const int half = g >> 3, r4 = 32 + (g & 7) * 4;
            const int* rr = rows + kb + r4;
            tma_gather4(smem + stage * kStageBytes + half * 8192 + r4 * 128, &map, &bar[stage],
                        m0 + half * 64, rr[0], rr[1], rr[2], rr[3]);
          }
        }
      }
    } else if (it < iters) {
      const int t = tid - 32 * tma_warps;
      const uint32_t base = smem_u32(smem + stage * kStageBytes);
      for (int c = t; c < 512; c += cp_threads) {   // rows 0..31
        const int r = c >> 4, j = c & 15;
        const int row = rows[kb + r];
        const uint32_t dst = base + (j >> 3) * 8192 + r * 128 + (((j & 7) ^ (r & 7)) << 4);
        cp_async_16(dst, at + (int64_t)row * ld + m0 + j * 8, 16);
      }
      asm volatile("cp.async.commit_group;");
      asm volatile("cp.async.wait_group 6;");
    }
  }
  asm volatile("cp.async.wait_group 0;");
  __syncthreads();
  if (tid == 0) cycles[blockIdx.x] = clock64() - t0;
}

// Decoupled hybrid: warps [0, cw) run an independent cp.async gather ring in
// smem half 0; lane 0 of warps [cw, cw+tw) run an independent gather4 ring in
// smem half 1.  Reports combined bytes.
__global__ void gather_hybrid2(const __grid_constant__ CUtensorMap map, const __half* at, int64_t ld,
                               const int* rows, int nrows, int M, int iters, int cw, int tw_,
                               long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[4];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < 4; ++s) mbar_init(&bar[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  long long t0 = clock64();
  const int warp = tid >> 5, lane = tid & 31;
  if (warp < cw) {
    for (int it = 0; it < iters; ++it) {
      const int stage = it % 4;
      const int kb = (it * 64 + blockIdx.x * 64) % (nrows - 64);
      const int m0 = ((it + blockIdx.x) * 128) % M;
      const uint32_t base = smem_u32(smem + stage * kStageBytes);
      for (int c = tid; c < 1024; c += 32 * cw) {
        const int r = c >> 4, j = c & 15;
        const int row = rows[kb + r];
        const uint32_t dst = base + (j >> 3) * 8192 + r * 128 + (((j & 7) ^ (r & 7)) << 4);
        cp_async_16(dst, at + (int64_t)row * ld + m0 + j * 8, 16);
      }
      asm volatile("cp.async.commit_group;");
      asm volatile("cp.async.wait_group 2;");
    }
    asm volatile("cp.async.wait_group 0;");
  } else if (warp < cw + tw_ && lane == 0) {
    const int w = warp - cw;
    const int per = 32 / tw_;
    for (int it = 0; it < iters + 4; ++it) {
      const int stage = it % 4;
      if (it >= 4) mbar_wait(&bar[stage], ((it / 4) - 1) & 1);
      if (it >= iters) continue;
      if (w == 0) mbar_arrive_expect_tx(&bar[stage], kStageBytes);
      const int kb = (it * 64 + blockIdx.x * 64 + 777) % (nrows - 64);
      const int m0 = ((it + blockIdx.x + 3) * 128) % M;
      for (int g = w * per; g < (w + 1) * per; ++g) {
        const int half = g >> 4, r4 = (g & 15) * 4;
        const int* rr = rows + kb + r4;
        tma_gather4(smem + (4 + stage) * kStageBytes + half * 8192 + r4 * 128, &map, &bar[stage],
                    m0 + half * 64, rr[0], rr[1], rr[2], rr[3]);
      }
    }
  }
  __syncthreads();
  if (tid == 0) cycles[blockIdx.x] = clock64() - t0;
}

__global__ void dense_tma(const __grid_constant__ CUtensorMap map, int nrows, int M, int iters,
                          long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[kStages];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&bar[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  long long t0 = clock64();
  if (tid == 0) {
    for (int it = 0; it < iters + kStages; ++it) {
      const int stage = it % kStages;
      if (it >= kStages) mbar_wait(&bar[stage], ((it / kStages) - 1) & 1);
      if (it >= iters) continue;
      mbar_arrive_expect_tx(&bar[stage], kStageBytes);
      const int kb = (it * 64 + blockIdx.x * 64) % (nrows - 64);
      const int m0 = ((it + blockIdx.x) * 128) % M;
      tma_load_2d(smem + stage * kStageBytes, &map, &bar[stage], m0, kb);
      tma_load_2d(smem + stage * kStageBytes + 8192, &map, &bar[stage], m0 + 64, kb);
    }
  }
  __syncthreads();
  if (tid == 0) cycles[blockIdx.x] = clock64() - t0;
}

int main() {
  const int K = 3072, M = 8192, nrows = 1536, iters = 400, grid = 148;
  std::vector<int> rows(K);
  for (int i = 0; i < K; ++i) rows[i] = i;
  std::mt19937 rng(1);
  std::shuffle(rows.begin(), rows.end(), rng);
  rows.resize(nrows);
  std::sort(rows.begin(), rows.end());
  __half* at;
  int* drows;
  long long* cyc;
  CK(cudaMalloc(&at, (size_t)K * M * 2));
  CK(cudaMemset(at, 0, (size_t)K * M * 2));
  CK(cudaMalloc(&drows, nrows * 4));
  CK(cudaMemcpy(drows, rows.data(), nrows * 4, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&cyc, grid * 8));
  void* fn;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  auto encode = (CUresult(*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill))fn;
  CUtensorMap gmap, dmap;
  cuuint64_t dims[2] = {(cuuint64_t)M, (cuuint64_t)K};
  cuuint64_t str[1] = {(cuuint64_t)M * 2};
  cuuint32_t gbox[2] = {64, 1}, dbox[2] = {64, 64}, es[2] = {1, 1};
  encode(&gmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, at, dims, str, gbox, es,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  encode(&dmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, at, dims, str, dbox, es,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int smem = kStages * kStageBytes + 1024;
  CK(cudaFuncSetAttribute(gather_cpasync, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(gather_tma4, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(gather_hybrid, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(dense_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto report = [&](const char* name) {
    std::vector<long long> c(grid);
    CK(cudaMemcpy(c.data(), cyc, grid * 8, cudaMemcpyDeviceToHost));
    std::sort(c.begin(), c.end());
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = (double)grid * iters * kStageBytes;
    printf("%-28s %8.1f GB/s  %6.1f B/cyc/SM (median cycles %lld)\n", name, bytes / ms / 1e6,
           (double)iters * kStageBytes / c[grid / 2], c[grid / 2]);
  };
  for (int w : {4, 8, 16}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      gather_cpasync<<<grid, 32 * w, smem>>>(at, M, drows, nrows, M, iters, cyc);
      cudaEventRecord(e1);
      CK(cudaDeviceSynchronize());
    }
    char name[64];
    snprintf(name, 64, "cp.async %d warps", w);
    report(name);
  }
  for (int issuers : {1, 2, 4, 8, 16, 32}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      gather_tma4<<<grid, 32 * std::max(issuers, 8), smem>>>(gmap, drows, nrows, M, iters, issuers, cyc);
      cudaEventRecord(e1);
      CK(cudaDeviceSynchronize());
    }
    char name[64];
    snprintf(name, 64, "tma gather4 %d issuers", issuers);
    report(name);
  }
  CK(cudaFuncSetAttribute(gather_hybrid2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  for (int tw_ : {4, 8, 16}) {
    for (int cw : {8, 16}) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        gather_hybrid2<<<grid, 32 * (tw_ + cw), smem>>>(gmap, at, M, drows, nrows, M, iters, cw, tw_, cyc);
        cudaEventRecord(e1);
        CK(cudaDeviceSynchronize());
      }
      // both rings move iters stages each: report 2x bytes
      std::vector<long long> c(grid);
      CK(cudaMemcpy(c.data(), cyc, grid * 8, cudaMemcpyDeviceToHost));
      std::sort(c.begin(), c.end());
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("hybrid2 tma %2d + cp %2d warps  %8.1f GB/s  %6.1f B/cyc/SM\n", tw_, cw,
             2.0 * grid * iters * kStageBytes / ms / 1e6, 2.0 * iters * kStageBytes / c[grid / 2]);
    }
  }
  for (int tw_ : {2, 4, 8}) {
    for (int cw : {4, 8}) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        gather_hybrid<<<grid, 32 * (tw_ + cw), smem>>>(gmap, at, M, drows, nrows, M, iters, tw_, cyc);
        cudaEventRecord(e1);
        CK(cudaDeviceSynchronize());
      }
      char name[64];
      snprintf(name, 64, "hybrid tma %d + cp %d warps", tw_, cw);
      report(name);
    }
  }
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    dense_tma<<<grid, 128, smem>>>(dmap, K, M, iters, cyc);
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
  }
  report("dense tma 2d");
  return 0;
}
