// CUDA-core FMA rates per SM on B200 for the K2 design (tw_aux.cu):
// fma.rn.f32.f16 (FHFMA: 16-bit operands, fp32 accumulator), fma.rn.f32
// (FFMA) and fma.rn.f32x2 (packed FFMA2), 32 warps per SM, 8 independent
// accumulator chains per thread.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_fma microbench_fma.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void bench(int iters, float* out, long long* cyc, float seed) {
  float acc[8];
  for (int i = 0; i < 8; ++i) acc[i] = seed * (threadIdx.x + i);
  const uint16_t h = 0x3c01, v = 0x3bff;
  const float fa = 1.0001f, fb = 0.9999f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) {
        asm volatile("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(acc[i]) : "h"(h), "h"(v));
      } else if (MODE == 1) {
        asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(acc[i]) : "f"(fa), "f"(fb));
      } else if (i % 2 == 0) {
        uint64_t d, a, b;
        asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(acc[i]), "f"(acc[i + 1]));
        asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "f"(fa), "f"(fa));
        asm("mov.b64 %0, {%1, %2};" : "=l"(b) : "f"(fb), "f"(fb));
        asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b));
        asm("mov.b64 {%0, %1}, %2;" : "=f"(acc[i]), "=f"(acc[i + 1]) : "l"(d));
      }
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
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
  const char* names[3] = {"fma.rn.f32.f16 (FHFMA)", "fma.rn.f32 (FFMA)", "fma.rn.f32x2 (FFMA2)"};
  for (int mode = 0; mode < 3; ++mode) {
    void (*k)(int, float*, long long*, float) = mode == 0 ? bench<0> : mode == 1 ? bench<1> : bench<2>;
    k<<<sms, 1024>>>(iters, out, cyc, 1e-3f);
    k<<<sms, 1024>>>(iters, out, cyc, 1e-3f);
    cudaDeviceSynchronize();
    long long c = 0;
    cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
    const double fmas = (double)iters * 8 * 1024;  // per SM (lane FMAs)
    printf("%-24s lane-FMAs per cycle per SM = %.1f\n", names[mode], fmas / c);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
