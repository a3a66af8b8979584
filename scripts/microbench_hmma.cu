// Warp-level tensor-core and ldmatrix rates on one B200 SM partition set.
// Diagnostic for the K2m design (tw_aux.cu): cycles per mma.sync m16n8k16
// (f16 -> f32) per SM, cycles per ldmatrix.x4.trans per SM, and both
// interleaved, with W warps per CTA and one CTA per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_hmma microbench_hmma.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                    uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, "
      "{%8, %9}, {%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldsm(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                     uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

template <int MODE>
__global__ void bench(int iters, float* out, long long* cyc) {
  __shared__ __align__(128) uint16_t sm[64 * 64];
  for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) sm[i] = (uint16_t)(i * 7);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm);
  // lane: row lane % 8 of matrix lane / 8, conflict-free (XOR swizzle)
  const uint32_t row = (lane & 7) + 8 * ((lane >> 4) & 1);
  uint32_t addr = base + row * 128 + ((((lane >> 3) & 1) ^ (row & 7)) << 4);
  float acc[4][4] = {};
  uint32_t a[4] = {lane, lane * 3u, lane * 5u, lane * 7u};
  const uint32_t b0 = 0x3c003c00u, b1 = 0x3c003c00u;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      if (MODE != 0) ldsm(addr + (uint32_t)(s * 32), a[0], a[1], a[2], a[3]);
      if (MODE != 1) mma(acc[s], a[0], a[1], a[2], a[3], b0, b1);
    }
  }
  long long t1 = clock64();
  float sum = 0;
  for (int s = 0; s < 4; ++s)
    for (int i = 0; i < 4; ++i) sum += acc[s][i];
  sum += a[0] + a[1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = sum;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  long long* cyc;
  cudaMalloc(&out, sms * 1024 * sizeof(float));
  cudaMalloc(&cyc, sms * sizeof(long long));
  const int iters = 4096;
  for (int mode = 0; mode < 3; ++mode)
    for (int warps : {4, 8, 16, 32}) {
      void (*k)(int, float*, long long*) = mode == 0 ? bench<0> : mode == 1 ? bench<1> : bench<2>;
      k<<<sms, warps * 32>>>(iters, out, cyc);
      k<<<sms, warps * 32>>>(iters, out, cyc);
      cudaDeviceSynchronize();
      long long c = 0;
      cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
      const double ops = (double)iters * 4 * warps;  // per SM
      printf("%-12s warps=%2d  cycles/op/SM=%.3f  (%s)\n",
             mode == 0 ? "mma only" : mode == 1 ? "ldsm only" : "ldsm+mma", warps, c / ops,
             mode == 1 ? "ldmatrix.x4.trans" : "m16n8k16 f16->f32");
    }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
