// Auxiliary kernels around K1:
//   K2  tw_residual_kernel   -- TEW overlay SpMM (reference executor.py:196-203)
//   K4  transpose_cast_kernel-- A (M x K) -> A^T (K x M) + dtype cast
//       (the reference's as_matrix/astype copies, core.py:32-43, executor.py:158)
//       build_payload_kernel -- CTO packed payload (formats.py:200) -> padded
//                               fp16/bf16 K-major tiles the TMA reads
#include "sm100_ptx.cuh"
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

// K2 -- TEW overlay SpMM, C'^T[urow(c)] (+)= sum_{(r, v) in column c} v * A^T[r].
//
// Every overlay row r of A^T is shared by many overlay columns (nnz/col is
// 11-46 at the BERT shapes while K is 768-3072), so reading A^T rows per nnz
// from L2 would move nnz * M * 2 bytes (580 MB for BERT 768x3072) through the
// SMs.  Instead a CTA stages the A^T block of its T tokens for ALL K rows in
// shared memory (16-bit, K * T * 2 bytes) together with the packed
// (row, value) list of its column group (4 bytes per nnz: row << 16 | 16-bit
// value in the compute dtype, the same rounding the TW payload gets), and
// walks the columns from there: a group of T/4 lanes per column, 4 tokens per
// lane, per nnz one broadcast 4-byte list load, one 8-byte A^T load, two
// conversions and two packed fma.rn.f32x2.  Columns are visited in
// descending-nnz order (host-sorted) so the lane groups of a warp finish
// together.  Each column's list is in ascending row order (CSC order of
// patterns.py:145-214); fp32 accumulation, then one coalesced
// read-modify-write of the TW result (accumulate = 1) or a plain store
// (residual-only column).  Geometry (T, column groups) comes from
// residual_geometry(); shapes that do not fit fall back to the direct kernel.
constexpr int kResThreads = 512;
constexpr int kResWarps = kResThreads / 32;
constexpr int kResSmem = 200 * 1024;

__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(reinterpret_cast<uint64_t&>(d))
      : "l"(reinterpret_cast<const uint64_t&>(a)), "l"(reinterpret_cast<const uint64_t&>(b)),
        "l"(reinterpret_cast<const uint64_t&>(c)));
  return d;
}

__device__ __forceinline__ float2 h2_to_f2(uint32_t u, bool bf) {
  if (bf) return make_float2(__uint_as_float(u << 16), __uint_as_float(u & 0xFFFF0000u));
  return __half22float2(*reinterpret_cast<const __half2*>(&u));
}

__device__ __forceinline__ float h_to_f(uint32_t h16, bool bf) {
  return bf ? __uint_as_float(h16 << 16) : __half2float(__ushort_as_half(static_cast<uint16_t>(h16)));
}

template <int T>
__global__ void __launch_bounds__(kResThreads)
    tw_residual_kernel(const ResidualArgs args, int col_groups) {
  extern __shared__ __align__(16) uint8_t res_smem[];
  uint16_t* sA = reinterpret_cast<uint16_t*>(res_smem);                  // [K][T]
  uint32_t* sRV = reinterpret_cast<uint32_t*>(res_smem + args.K * T * 2);  // group's list
  constexpr int kLanesPerCol = T / 4;
  constexpr int kColsPerWarp = 32 / kLanesPerCol;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * T;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint16_t* at = static_cast<const uint16_t*>(args.at);
  const int K = args.K;
  const bool bf = args.in_dtype == kBF16;
  const int64_t rem = args.M - t0;
  const int ntok = rem < T ? static_cast<int>(rem) : T;
  // column group g: processed columns [c0, c1), nnz [e0, e1)
  const int g = blockIdx.y;
  const int c0 = static_cast<int>(static_cast<int64_t>(g) * args.n_cols / col_groups);
  const int c1 = static_cast<int>(static_cast<int64_t>(g + 1) * args.n_cols / col_groups);
  const int e0 = __ldg(args.col_start + c0), e1 = __ldg(args.col_start + c1);
  // stage the (row, value) list and A^T[:, t0:t0+T] (zero past M) with
  // cp.async so every load of the CTA is in flight at once
  {
    const int n4 = (e1 - e0);
    const bool al = ((e0 & 3) == 0);
    const int nvec = al ? n4 / 4 : 0;
    for (int i = threadIdx.x; i < nvec; i += kResThreads)
      cp_async_16(smem_u32(sRV + 4 * i), args.rv + e0 + 4 * i, 16);
    for (int i = 4 * nvec + threadIdx.x; i < n4; i += kResThreads) sRV[i] = __ldg(args.rv + e0 + i);
  }
  if (T % 8 == 0 && args.ld_at % 8 == 0) {
    constexpr int per_row = T / 8;
    for (int i = threadIdx.x; i < K * per_row; i += kResThreads) {
      const int r = i / per_row, j = (i - r * per_row) * 8;
      const int valid = ntok - j;
      const uint32_t bytes = valid >= 8 ? 16u : (valid > 0 ? static_cast<uint32_t>(valid) * 2 : 0u);
      cp_async_16(smem_u32(sA + r * T + j), bytes ? at + r * args.ld_at + t0 + j : at, bytes);
    }
  } else {
    for (int i = threadIdx.x; i < K * T; i += kResThreads) {
      const int r = i / T, j = i - r * T;
      sA[i] = j < ntok ? at[r * args.ld_at + t0 + j] : static_cast<uint16_t>(0);
    }
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  const int sub = lane / kLanesPerCol;
  const int tok = (lane - sub * kLanesPerCol) * 4;
  const uint16_t* sAt = sA + tok;
  for (int col = c0 + warp * kColsPerWarp + sub; col < c1; col += kResWarps * kColsPerWarp) {
    const int lo = __ldg(args.col_start + col) - e0, hi = __ldg(args.col_start + col + 1) - e0;
    float2 acc0 = make_float2(0.f, 0.f), acc1 = make_float2(0.f, 0.f);
#pragma unroll 4
    for (int e = lo; e < hi; ++e) {
      const uint32_t q = sRV[e];
      const uint2 a = *reinterpret_cast<const uint2*>(sAt + (q >> 16) * T);
      const float v = h_to_f(q & 0xFFFFu, bf);
      const float2 vv = make_float2(v, v);
      acc0 = fma2(h2_to_f2(a.x, bf), vv, acc0);
      acc1 = fma2(h2_to_f2(a.y, bf), vv, acc1);
    }
    if (tok >= ntok) continue;
    const int64_t base = static_cast<int64_t>(__ldg(args.out_rows + col)) * args.ld_out + t0 + tok;
    const bool accum = __ldg(args.accumulate + col) != 0;
    const float o[4] = {acc0.x, acc0.y, acc1.x, acc1.y};
    if (args.out_dtype != kF32 && tok + 4 <= ntok && base % 4 == 0) {
      // 8-byte read-modify-write of 4 16-bit outputs
      uint2* p = reinterpret_cast<uint2*>(static_cast<uint16_t*>(args.out) + base);
      uint2 cur = accum ? *p : make_uint2(0u, 0u);
      float f[4];
      const float2 lo2 = h2_to_f2(cur.x, args.out_dtype == kBF16);
      const float2 hi2 = h2_to_f2(cur.y, args.out_dtype == kBF16);
      f[0] = lo2.x + o[0]; f[1] = lo2.y + o[1]; f[2] = hi2.x + o[2]; f[3] = hi2.y + o[3];
      if (args.out_dtype == kF16) {
        const __half2 x = __floats2half2_rn(f[0], f[1]), y = __floats2half2_rn(f[2], f[3]);
        cur = make_uint2(*reinterpret_cast<const uint32_t*>(&x), *reinterpret_cast<const uint32_t*>(&y));
      } else {
        const __nv_bfloat162 x = __floats2bfloat162_rn(f[0], f[1]);
        const __nv_bfloat162 y = __floats2bfloat162_rn(f[2], f[3]);
        cur = make_uint2(*reinterpret_cast<const uint32_t*>(&x), *reinterpret_cast<const uint32_t*>(&y));
      }
      *p = cur;
      continue;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (tok + i >= ntok) break;
      float w = o[i];
      if (accum) w += load_as_float(args.out, args.out_dtype, base + i);
      store_from_float(args.out, args.out_dtype, base + i, w);
    }
  }
}

// Fallback (A^T block does not fit): rows read from global per nnz.
__global__ void __launch_bounds__(256)
    tw_residual_direct_kernel(const ResidualArgs args) {
  const int col = blockIdx.y;
  const int64_t m = static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x;
  if (m >= args.M) return;
  const int lo = args.col_start[col], hi = args.col_start[col + 1];
  float acc = 0.f;
  for (int e = lo; e < hi; ++e)
    acc = fmaf(load_as_float(args.at, args.in_dtype, args.rows[e] * args.ld_at + m), args.vals[e],
               acc);
  const int64_t base = static_cast<int64_t>(args.out_rows[col]) * args.ld_out + m;
  if (args.accumulate[col]) acc += load_as_float(args.out, args.out_dtype, base);
  store_from_float(args.out, args.out_dtype, base, acc);
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

bool residual_geometry(int32_t K, int64_t max_group_nnz_bytes_per_group1, int* T_out,
                       int* groups_out) {
  // largest T whose A^T block leaves room for the (row, value) list split into
  // as few column groups as possible (list bytes = 4 * nnz)
  for (int T : {64, 32, 16, 8}) {
    const int64_t a_bytes = static_cast<int64_t>(K) * T * 2;
    if (a_bytes > kResSmem / 2) continue;
    const int64_t budget = kResSmem - a_bytes;
    const int64_t groups = (max_group_nnz_bytes_per_group1 + budget - 1) / budget;
    *T_out = T;
    *groups_out = static_cast<int>(std::max<int64_t>(1, groups));
    return true;
  }
  return false;
}

template <int T>
static cudaError_t launch_res(const ResidualArgs& args, cudaStream_t stream) {
  const int blocks = static_cast<int>((args.M + T - 1) / T);
  // smem: A^T block + the largest column group's list (host-checked bound)
  const size_t smem = static_cast<size_t>(args.K) * T * 2 + static_cast<size_t>(args.max_group_nnz) * 4;
  cudaError_t e = cudaFuncSetAttribute(tw_residual_kernel<T>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  dim3 grid(static_cast<unsigned>(blocks), static_cast<unsigned>(args.col_groups));
  tw_residual_kernel<T><<<grid, kResThreads, smem, stream>>>(args, args.col_groups);
  return cudaGetLastError();
}

cudaError_t launch_tw_residual(const ResidualArgs& args, cudaStream_t stream) {
  if (args.n_cols <= 0 || args.M <= 0) return cudaSuccess;
  switch (args.rv ? args.block_tokens : 0) {
    case 64: return launch_res<64>(args, stream);
    case 32: return launch_res<32>(args, stream);
    case 16: return launch_res<16>(args, stream);
    case 8: return launch_res<8>(args, stream);
    default: break;
  }
  dim3 grid(static_cast<unsigned>((args.M + 255) / 256), static_cast<unsigned>(args.n_cols));
  tw_residual_direct_kernel<<<grid, 256, 0, stream>>>(args);
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
