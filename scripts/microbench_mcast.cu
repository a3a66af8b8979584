// Microbenchmark (diagnostics, GPU box): does TMA multicast raise per-SM
// ingress above the unicast cap?  Each CTA of a cluster of `csz` receives a
// full 32 KB stage per iteration; with multicast, each CTA requests only
// 1/csz of it (one box slice) and the TMA unit delivers the slice to every
// CTA of the cluster.  Unicast baseline: each CTA requests all 32 KB itself.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lcuda -o mb_mcast microbench_mcast.cu
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2402_10876_b200/csrc/sm100_ptx.cuh"

using namespace tw;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int kStage = 32768;
constexpr int kSt = 4;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, uint32_t rank) {
  asm volatile(
      "{\n .reg .b32 ra;\n mapa.shared::cluster.u32 ra, %0, %1;\n"
      " mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n}" ::"r"(smem_u32(bar)),
      "r"(rank)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* map, uint64_t* bar,
                                               int32_t c0, int32_t c1, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}

// mode 0: unicast (each CTA loads its full stage: 4 boxes of {64 tok, 64 rows})
// mode 1: multicast (CTA r loads boxes r, r + csz, ... and multicasts them)
// spin on test_wait (no suspend hint): a remote (cluster) arrival may not
// wake a thread suspended in try_wait promptly
__device__ __forceinline__ void mbar_spin(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tSPIN_%=:\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra SPIN_%=;\n\t}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}

__device__ __forceinline__ void mbar_arrive_remote_relaxed(uint64_t* bar, uint32_t rank) {
  asm volatile(
      "{\n .reg .b32 ra;\n mapa.shared::cluster.u32 ra, %0, %1;\n"
      " mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [ra];\n}" ::"r"(smem_u32(bar)),
      "r"(rank)
      : "memory");
}

__global__ void ring(const __grid_constant__ CUtensorMap map, int M, int K, int iters, int csz,
                     int mode, long long* cycles, int share) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[kSt], empty[kSt];
  const int tid = threadIdx.x;
  const uint32_t rank = csz > 1 ? cluster_rank() : 0;
  const int cluster_id = blockIdx.x / (csz * (share > 0 ? share : 1));
  if (tid == 0) {
    for (int s = 0; s < kSt; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], (mode == 1 || mode == 3) ? csz : 1);  // mode 2: multicast, local release only (raw delivery rate; racy by design)
    }
    fence_barrier_init();
  }
  if (csz > 1) cluster_sync(); else __syncthreads();
  const long long t0 = clock64();
  if (tid == 0) {
    for (int it = 0; it < iters; ++it) {
      const int stage = it % kSt;
      if (it >= kSt) {
        if (mode == 3) mbar_spin(&empty[stage], ((it / kSt) - 1) & 1);
        else mbar_wait(&empty[stage], ((it / kSt) - 1) & 1);
      }
      mbar_arrive_expect_tx(&full[stage], kStage);
      // same tile for the whole cluster (that is what multicast shares)
      int kb = ((it + cluster_id * 7) * 64) % (K - 64);
      if (share < 0) kb = (kb + 1) % (K - 64);                 // unaligned start row
      if (share < -1) kb = (kb * 37 + (kb >> 6) * 11) % (K - 64); // scattered start rows
      const int m0 = ((it * 3 + cluster_id) * 256) % M;
      uint8_t* dst = smem + stage * kStage;
      if (mode == 0) {
        for (int ch = 0; ch < 4; ++ch) tma_load_2d(dst + ch * 8192, &map, &full[stage], m0 + ch * 64, kb);
      } else {
        for (int ch = rank; ch < 4; ch += csz)
          tma_load_2d_mc(dst + ch * 8192, &map, &full[stage], m0 + ch * 64, kb,
                         static_cast<uint16_t>((1u << csz) - 1));
      }
    }
  } else if (tid == 32) {
    // consumer: recycle the slot once it landed (in every CTA of the cluster)
    for (int it = 0; it < iters; ++it) {
      const int stage = it % kSt;
      mbar_wait(&full[stage], (it / kSt) & 1);
      if (mode == 3) {
        for (int r = 0; r < csz; ++r) mbar_arrive_remote_relaxed(&empty[stage], r);
      } else if (mode == 1) {
        for (int r = 0; r < csz; ++r) mbar_arrive_remote(&empty[stage], r);
      } else if (mode == 2) {
        mbar_arrive(&empty[stage]);
      } else {
        mbar_arrive(&empty[stage]);
      }
    }
  }
  __syncthreads();
  if (tid == 0) cycles[blockIdx.x] = clock64() - t0;
  if (csz > 1) cluster_sync();
}

int main() {
  const int K = 3072, M = 8192, iters = 400;
  __half* at;
  long long* cyc;
  CK(cudaMalloc(&at, (size_t)K * M * 2));
  CK(cudaMemset(at, 0, (size_t)K * M * 2));
  CK(cudaMalloc(&cyc, 160 * 8));
  void* fn;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  auto encode = (CUresult(*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill))fn;
  CUtensorMap dmap;
  cuuint64_t dims[2] = {(cuuint64_t)M, (cuuint64_t)K};
  cuuint64_t strides[1] = {(cuuint64_t)M * 2};
  cuuint32_t dbox[2] = {64, 64}, es[2] = {1, 1};
  encode(&dmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, at, dims, strides, dbox, es,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int smem = kSt * kStage + 1024;
  CK(cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(ring, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int share : {1, -1, -2}) for (int csz : {1, 2, 4}) {
    for (int mode : {0, 1, 2, 3}) {
      if (mode >= 1 && csz == 1) continue;
      if (share > 1 && mode == 1) continue;
      const int grid = 148 / csz * csz;
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(64);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = csz;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      float ms = 0;
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        CK(cudaLaunchKernelEx(&cfg, ring, dmap, M, K, iters, csz, mode, cyc, share));
        cudaEventRecord(e1);
        CK(cudaDeviceSynchronize());
        cudaEventElapsedTime(&ms, e0, e1);
      }
      std::vector<long long> c(grid);
      CK(cudaMemcpy(c.data(), cyc, grid * 8, cudaMemcpyDeviceToHost));
      std::sort(c.begin(), c.end());
      const double bytes = (double)grid * iters * kStage;  // bytes landed in smem
      printf("share %2d cluster %d %-10s grid %3d  %8.1f GB/s landed  %6.1f B/cyc/SM landed (median)\n",
             share, csz, mode == 3 ? "mc-relax+spin" : mode == 2 ? "mc-local" : mode ? "multicast" : "unicast", grid, bytes / ms / 1e6,
             (double)iters * kStage / c[grid / 2]);
      (void)share;
    }
  }
  return 0;
}
