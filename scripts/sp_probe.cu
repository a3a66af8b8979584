// Pins the tcgen05.mma.sp (kind::f16, 2:4 A operand) conventions the TVW
// path relies on: compressed K-major SW128 A, MN-major SW128 B, metadata in
// tensor memory.  One CTA, M = 128, N = 64 tokens, K = 64 logical (two sparse
// MMAs of K = 32); integer-valued fp16 data so the product is exact.  Several
// candidate metadata layouts are written and each result is compared with the
// dense host product; the one with error 0 is the layout the kernels use.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I.. -o sp_probe sp_probe.cu
#include <cuda_fp16.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_2402_10876_b200/csrc/sm100_ptx.cuh"

using namespace tw;

constexpr int M = 128, N = 64, KL = 128;  // logical K (4 sparse MMAs)
constexpr int KC = KL / 2;               // compressed K

__device__ __forceinline__ void umma_sp(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                        uint32_t e, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], %1, %2, [%5], %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(e)
      : "memory");
}

__global__ void probe(const __half* a_c, const __half* b, const uint32_t* meta, float* d,
                      int meta_cols, int packed) {
  __shared__ __align__(1024) uint8_t sA[M * 128];
  __shared__ __align__(1024) uint8_t sB[KL * 128];
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // A: row r = 128 B (SW128, K-major), compressed elements 0..31 in chunks 0..3
  for (int i = tid; i < M * 8; i += blockDim.x) {
    const int r = i / 8, c = i % 8;  // 16-byte chunk c of row r (8 halves)
    uint4 v = make_uint4(0, 0, 0, 0);
    if (c < KC / 8) v = *reinterpret_cast<const uint4*>(a_c + r * KC + c * 8);
    *reinterpret_cast<uint4*>(sA + r * 128 + ((c ^ (r & 7)) * 16)) = v;
  }
  // B: row k = 64 tokens = 128 B (SW128, MN-major)
  for (int i = tid; i < KL * 8; i += blockDim.x) {
    const int k = i / 8, c = i % 8;
    *reinterpret_cast<uint4*>(sB + k * 128 + ((c ^ (k & 7)) * 16)) =
        *reinterpret_cast<const uint4*>(b + k * N + c * 8);
  }
  if (warp == 0) tmem_alloc(&s_tmem, 128);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  // metadata: columns 64 .. 64 + meta_cols - 1, lane quadrant of this warp
  for (int c = 0; c < meta_cols; ++c) {
    const uint32_t v = meta[c * 128 + warp * 32 + lane];
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(
                     tmem + ((uint32_t)(warp * 32) << 16) + 64 + (packed ? c : 4 * c)),
                 "r"(v)
                 : "memory");
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    const uint32_t idesc = umma_idesc_f16(M, N, 0, 0, 1) | (1u << 2);  // sparse
    for (int i = 0; i < KL / 32; ++i) {
      const uint64_t ad = umma_desc_sw128(smem_u32(sA) + i * 32, 16, 1024);
      const uint64_t bd = umma_desc_sw128(smem_u32(sB) + i * 32 * 128, 8192, 1024);
      if (packed)  // metadata of MMA i in column 64 + i: even base, id2 = i % 2
        umma_sp(tmem, ad, bd, idesc | (uint32_t)(i & 1), tmem + 64 + (i & ~1), i > 0);
      else
        umma_sp(tmem, ad, bd, idesc, tmem + 64 + 4 * i, i > 0);
    }
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  uint32_t r[32];
  for (int h = 0; h < 2; ++h) {
    tmem_ld_32x32b_x32(tmem + ((uint32_t)(warp * 32) << 16) + h * 32, r);
    tmem_ld_wait();
    for (int j = 0; j < 32; ++j) d[(warp * 32 + lane) * N + h * 32 + j] = __uint_as_float(r[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 128);
}

int main(int argc, char** argv) {
  const int only = argc > 1 ? atoi(argv[1]) : -1;
  const int bmask = argc > 2 ? atoi(argv[2]) : 0;
  const int packed = argc > 3 ? atoi(argv[3]) : 0;
  srand(7);
  std::vector<float> ad(M * KL, 0.f), bd(KL * N);
  std::vector<__half> ac(M * KC), bh(KL * N);
  std::vector<uint8_t> nib(M * (KL / 4));  // per row, per 4-group: idx0 | idx1 << 2
  for (int r = 0; r < M; ++r)
    for (int g = 0; g < KL / 4; ++g) {
      int i0 = rand() % 4, i1 = rand() % 3;
      if (i1 >= i0) ++i1;
      if (i0 > i1) std::swap(i0, i1);
      const float v0 = (float)(rand() % 7 - 3), v1 = (float)(rand() % 7 - 3);
      ad[r * KL + 4 * g + i0] = v0;
      ad[r * KL + 4 * g + i1] = v1;
      ac[r * KC + 2 * g] = __float2half(v0);
      ac[r * KC + 2 * g + 1] = __float2half(v1);
      nib[r * (KL / 4) + g] = (uint8_t)(i0 | (i1 << 2));
    }
  for (int i = 0; i < KL * N; ++i) {
    bd[i] = (float)(rand() % 5 - 2);
    const int k = i / N;
    if ((bmask == 1 && k % 32 >= 16) || (bmask == 2 && k % 32 < 16)) bd[i] = 0.f;
    bh[i] = __float2half(bd[i]);
  }
  std::vector<float> ref(M * N, 0.f);
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      float s = 0;
      for (int k = 0; k < KL; ++k) s += ad[m * KL + k] * bd[k * N + n];
      ref[m * N + n] = s;
    }
  __half *dac, *db;
  uint32_t* dmeta;
  float* dd;
  cudaMalloc(&dac, ac.size() * 2);
  cudaMalloc(&db, bh.size() * 2);
  cudaMalloc(&dmeta, 4 * 128 * 4);
  cudaMalloc(&dd, M * N * 4);
  cudaMemcpy(dac, ac.data(), ac.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(db, bh.data(), bh.size() * 2, cudaMemcpyHostToDevice);
  // candidate layouts: meta[col][lane], one column per MMA (K = 32 logical)
  const char* names[] = {
      "H1 lane=m%8+16(m/16)+8(k/16), bits 16((m/8)%2)+k%16",
      "H2 lane=m, bits k%32 (8 nibbles)",
      "H3 H1 with swapped nibble halves",
      "H4 lane=m%8+16(m/16)+8((m/8)%2), bits k%32",
      "H5 H1 with m%8 rows 2 and 4 swapped"};
  for (int h = 0; h < 5; ++h) {
    if (only >= 0 && h != only) continue;
    std::vector<uint32_t> meta(4 * 128, 0);
    for (int mma = 0; mma < KL / 32; ++mma)
      for (int m = 0; m < M; ++m)
        for (int kk = 0; kk < 32; kk += 4) {
          const int g = (mma * 32 + kk) / 4;
          uint32_t v = nib[m * (KL / 4) + g];
          if (h == 2) v = ((v & 3) << 2) | (v >> 2);
          int lane, bit;
          if (h == 0 || h == 2 || h == 4) {
            static const int sw[8] = {0, 1, 4, 3, 2, 5, 6, 7};
            lane = (h == 4 ? sw[m % 8] : m % 8) + 16 * (m / 16) + 8 * (kk / 16);
            bit = 16 * ((m / 8) % 2) + (kk % 16);
          } else if (h == 1) {
            lane = m;
            bit = kk;
          } else {
            lane = (m % 8) + 16 * (m / 16) + 8 * ((m / 8) % 2);
            bit = kk;
          }
          meta[mma * 128 + lane] |= v << bit;
        }
    cudaMemcpy(dmeta, meta.data(), meta.size() * 4, cudaMemcpyHostToDevice);
    cudaMemset(dd, 0, M * N * 4);
    probe<<<1, 128>>>(dac, db, dmeta, dd, KL / 32, packed);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> got(M * N);
    cudaMemcpy(got.data(), dd, M * N * 4, cudaMemcpyDeviceToHost);
    double err = 0;
    int bad = 0;
    for (int i = 0; i < M * N; ++i) {
      const double x = fabs(got[i] - ref[i]);
      err = x > err ? x : err;
      bad += x > 0;
    }
    printf("%-55s max|err| = %g  mismatches = %d  (%s)\n", names[h], err, bad,
           cudaGetErrorString(e));
    // rows with any mismatch, by m % 16 and m / 16
    int byr[16] = {0}, byq[8] = {0};
    for (int m = 0; m < M; ++m) {
      int b = 0;
      for (int n = 0; n < N; ++n) b += got[m * N + n] != ref[m * N + n];
      if (b) { byr[m % 16]++; byq[m / 16]++; }
    }
    printf("  bad rows by m%%16:");
    for (int i = 0; i < 16; ++i) printf(" %d", byr[i]);
    printf("   by m/16:");
    for (int i = 0; i < 8; ++i) printf(" %d", byq[i]);
    printf("\n");
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
