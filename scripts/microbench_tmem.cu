// Microbenchmark (diagnostics, GPU box): tcgen05.ld throughput from TMEM to
// registers for the epilogue shapes, with W warps (lane quadrant = warp % 4).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mb_tmem microbench_tmem.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>

#include "../paper_2402_10876_b200/csrc/sm100_ptx.cuh"

using namespace tw;

__device__ __forceinline__ void ld_x64(uint32_t taddr, uint32_t (&r)[64]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x64.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,"
      "%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,"
      "%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]),
        "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]),
        "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]),
        "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]), "=r"(r[49]),
        "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]),
        "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]),
        "=r"(r[62]), "=r"(r[63])
      : "r"(taddr));
}

template <int X>
__global__ void tmem_read(int iters, long long* cycles, float* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    tmem_alloc(&slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t base = slot + (static_cast<uint32_t>((warp & 3) * 32) << 16);
  float acc = 0.f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    for (int c = 0; c < 256; c += X) {
      if (X == 16) {
        uint32_t r[16];
        tmem_ld_32x32b_x16(base + c, r);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 16; ++i) acc += __uint_as_float(r[i]);
      } else if (X == 32) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(base + c, r);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) acc += __uint_as_float(r[i]);
      } else {
        uint32_t r[64];
        ld_x64(base + c, r);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 64; ++i) acc += __uint_as_float(r[i]);
      }
    }
  }
  long long t1 = clock64();
  if (lane == 0) cycles[blockIdx.x * 32 + warp] = t1 - t0;
  if (acc == 12345.f) sink[0] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(slot, 512);
}

int main() {
  long long* cyc;
  float* sink;
  cudaMalloc(&cyc, 148 * 32 * 8);
  cudaMalloc(&sink, 4);
  const int iters = 200;
  for (int warps : {4, 8, 16}) {
    for (int x : {16, 32, 64}) {
      cudaMemset(cyc, 0, 148 * 32 * 8);
      if (x == 16) tmem_read<16><<<148, 32 * warps>>>(iters, cyc, sink);
      if (x == 32) tmem_read<32><<<148, 32 * warps>>>(iters, cyc, sink);
      if (x == 64) tmem_read<64><<<148, 32 * warps>>>(iters, cyc, sink);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      std::vector<long long> c(148 * 32);
      cudaMemcpy(c.data(), cyc, c.size() * 8, cudaMemcpyDeviceToHost);
      long long mx = 0;
      for (int b = 0; b < 148; ++b)
        for (int w = 0; w < warps; ++w) mx = std::max(mx, c[b * 32 + w]);
      // each warp reads 32 lanes x 256 cols x 4 B per iteration
      const double bytes = (double)warps * iters * 32 * 256 * 4;
      printf("warps %2d  x%-2d  %8.1f B/cycle/SM  (%lld cycles, %.0f cycles per 4 KB warp load)\n",
             warps, x, bytes / mx, mx, (double)mx / (iters * (256.0 / x)) / (x / 32.0));
    }
  }
  return 0;
}
