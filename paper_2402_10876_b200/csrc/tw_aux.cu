// Auxiliary kernels around K1:
//   K2  tw_residual_kernel   -- TEW overlay SpMM (reference executor.py:196-203)
//   K4  transpose_cast_kernel-- A (M x K) -> A^T (K x M) + dtype cast
//       (the reference's as_matrix/astype copies, core.py:32-43, executor.py:158)
//       build_payload_kernel -- CTO packed payload (formats.py:200) -> padded
//                               fp16/bf16 K-major tiles the TMA reads
#include "tw_kernels.cuh"

#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>

namespace tw {

namespace {

__device__ __forceinline__ float load_as_float(const void* p, int32_t dtype, int64_t i) {
  if (dtype == kF32) return static_cast<const float*>(p)[i];
  if (dtype == kF16) return __half2float(static_cast<const __half*>(p)[i]);
  return __bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]);
}

__device__ __forceinline__ void store_from_float(void* p, int32_t dtype, int64_t i, float v) {
  if (dtype == kF32) {
    static_cast<float*>(p)[i] = v;
  } else if (dtype == kF16) {
    static_cast<__half*>(p)[i] = __float2half_rn(v);
  } else {
    static_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn(v);
  }
}

// Each thread owns two consecutive tokens of one overlay column; the column's
// (row, value) list is walked in ascending row order (CSC order of
// patterns.py:145-214).  Reads of A^T rows are 32-lane coalesced.
constexpr int kResThreads = 128;
constexpr int kResTokens = 2 * kResThreads;

__global__ void __launch_bounds__(kResThreads)
    tw_residual_kernel(const ResidualArgs args) {
  const int col = blockIdx.y;
  const int64_t m = static_cast<int64_t>(blockIdx.x) * kResTokens + 2 * threadIdx.x;
  if (m >= args.M) return;
  const bool pair = (m + 1) < args.M;
  const int lo = args.col_start[col];
  const int hi = args.col_start[col + 1];
  float acc0 = 0.f, acc1 = 0.f;
  if (args.in_dtype == kF16 && pair && (args.ld_at % 2 == 0)) {
    const __half* at = static_cast<const __half*>(args.at);
    for (int e = lo; e < hi; ++e) {
      const float v = __ldg(args.vals + e);
      const int64_t r = __ldg(args.rows + e);
      const float2 a = __half22float2(*reinterpret_cast<const __half2*>(at + r * args.ld_at + m));
      acc0 = fmaf(a.x, v, acc0);
      acc1 = fmaf(a.y, v, acc1);
    }
  } else {
    for (int e = lo; e < hi; ++e) {
      const float v = __ldg(args.vals + e);
      const int64_t r = __ldg(args.rows + e);
      acc0 = fmaf(load_as_float(args.at, args.in_dtype, r * args.ld_at + m), v, acc0);
      if (pair) acc1 = fmaf(load_as_float(args.at, args.in_dtype, r * args.ld_at + m + 1), v, acc1);
    }
  }
  const int64_t base = static_cast<int64_t>(args.out_rows[col]) * args.ld_out + m;
  if (args.accumulate[col]) {
    acc0 += load_as_float(args.out, args.out_dtype, base);
    if (pair) acc1 += load_as_float(args.out, args.out_dtype, base + 1);
  }
  store_from_float(args.out, args.out_dtype, base, acc0);
  if (pair) store_from_float(args.out, args.out_dtype, base + 1, acc1);
}

// 32 x 32 shared-memory transpose with dtype conversion.
__global__ void transpose_cast_kernel(const void* a, int32_t a_dtype, int64_t M, int64_t K,
                                      int64_t lda, void* at, int32_t at_dtype, int64_t ld_at) {
  __shared__ float tile[32][33];
  const int64_t k0 = static_cast<int64_t>(blockIdx.x) * 32;
  const int64_t m0 = static_cast<int64_t>(blockIdx.y) * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t m = m0 + i, k = k0 + threadIdx.x;
    tile[i][threadIdx.x] = (m < M && k < K) ? load_as_float(a, a_dtype, m * lda + k) : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t k = k0 + i, m = m0 + threadIdx.x;
    if (k < K && m < M) store_from_float(at, at_dtype, k * ld_at + m, tile[threadIdx.x][i]);
  }
}

// dst[(s*BN + c) * Kp + r] = payload of sub-tile s, column c, kept row r
// (zero for padding slots r >= K'_i and padded columns c >= width).
__global__ void build_payload_kernel(const PayloadArgs args) {
  const int s = blockIdx.y;
  const SubTile d = args.subtiles[s];
  const int64_t per = static_cast<int64_t>(args.bn) * args.Kp;
  const int64_t base = static_cast<int64_t>(d.pay_row) * args.Kp;
  const int64_t src0 = args.src_base[s];
  const int ld = args.src_ld[s];
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < per;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i / args.Kp);
    const int r = static_cast<int>(i - static_cast<int64_t>(c) * args.Kp);
    float v = 0.f;
    if (c < d.width && r < ld) v = args.src[src0 + static_cast<int64_t>(c) * ld + r];
    store_from_float(args.dst, args.dst_dtype, base + i, v);
  }
}

}  // namespace

cudaError_t launch_tw_residual(const ResidualArgs& args, cudaStream_t stream) {
  if (args.n_cols <= 0 || args.M <= 0) return cudaSuccess;
  dim3 grid(static_cast<unsigned>((args.M + kResTokens - 1) / kResTokens),
            static_cast<unsigned>(args.n_cols));
  tw_residual_kernel<<<grid, kResThreads, 0, stream>>>(args);
  return cudaGetLastError();
}

cudaError_t launch_transpose_cast(const void* a, int32_t a_dtype, int64_t M, int64_t K,
                                  int64_t lda, void* at, int32_t at_dtype, int64_t ld_at,
                                  cudaStream_t stream) {
  if (M <= 0 || K <= 0) return cudaSuccess;
  dim3 grid(static_cast<unsigned>((K + 31) / 32), static_cast<unsigned>((M + 31) / 32));
  dim3 block(32, 8);
  transpose_cast_kernel<<<grid, block, 0, stream>>>(a, a_dtype, M, K, lda, at, at_dtype, ld_at);
  return cudaGetLastError();
}

cudaError_t launch_build_payload(const PayloadArgs& args, cudaStream_t stream) {
  if (args.n_sub <= 0) return cudaSuccess;
  const int64_t per = static_cast<int64_t>(args.bn) * args.Kp;
  unsigned gx = static_cast<unsigned>((per + 255) / 256);
  if (gx > 1024) gx = 1024;
  dim3 grid(gx, static_cast<unsigned>(args.n_sub));
  build_payload_kernel<<<grid, 256, 0, stream>>>(args);
  return cudaGetLastError();
}

}  // namespace tw
