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
#include <cstdlib>

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
// Replaces the per-column overlay loop of gemm_tew (executor.py:196-203).
// Every overlay row of A^T is shared by many overlay columns (nnz/col is
// 11-46 at the BERT shapes while K is 768-3072, and the overlay covers every
// row), so a CTA stages the A^T block of T tokens for ALL K rows in shared
// memory (16-bit, K * T * 2 bytes) and serves every overlay column of its
// column range from there: 2 bytes of shared-memory traffic per FMA and ~1x
// A^T of L2 reads for the staging.
//
// Grid = (token blocks, column splits), one 32-warp CTA per SM; T is as
// large as shared memory allows so the column lists (re-read per block) are
// amortised.  After one barrier the warps walk their columns independently:
// a lane group of L lanes per column (8 tokens per lane and one 16-byte
// shared load per entry; 16 tokens and two loads for T = 64), 32 / L columns
// per warp step, columns in descending-nnz order (host) so the groups of a
// warp finish together.  Each lane group fetches its column's packed entries
// (16-bit value, rounded like the TW payload, << 16 | the row's offset in the
// staged block in 16-byte units) in groups of L, two groups ahead; one
// fma.rn.f32.f16 (FHFMA: 16-bit operands, fp32 accumulator, no conversions)
// per token, fp32 accumulation in the list order (the CSC rows of
// patterns.py:145-214, interleaved by bank class on the host, tw_capi.cu),
// then one read-modify-write of the TW result (accumulate = 1) or a plain
// store (residual-only column).
constexpr int kResThreads = 1024;  // 32 warps: one CTA per SM, 64 registers per thread
constexpr int kResWarps = kResThreads / 32;

__device__ __forceinline__ float2 h2_to_f2(uint32_t u, bool bf) {
  if (bf) return make_float2(__uint_as_float(u << 16), __uint_as_float(u & 0xFFFF0000u));
  return __half22float2(*reinterpret_cast<const __half2*>(&u));
}

// acc + a * v with 16-bit a, v and fp32 accumulation (FHFMA: the product is
// exact in fp32, one rounding -- identical to widening first).
template <bool kBf>
__device__ __forceinline__ float fma_h(uint16_t a, uint16_t v, float acc) {
  float d;
  if (kBf)
    asm("fma.rn.f32.bf16 %0, %1, %2, %3;" : "=f"(d) : "h"(a), "h"(v), "f"(acc));
  else
    asm("fma.rn.f32.f16 %0, %1, %2, %3;" : "=f"(d) : "h"(a), "h"(v), "f"(acc));
  return d;
}

// acc[0..7] += 8 packed 16-bit a (uint4) * v
template <bool kBf>
__device__ __forceinline__ void fma8(float (&acc)[8], const uint4& a, uint16_t v) {
  const uint32_t w[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint16_t lo, hi;
    asm("mov.b32 {%0, %1}, %2;" : "=h"(lo), "=h"(hi) : "r"(w[i]));
    acc[2 * i] = fma_h<kBf>(lo, v, acc[2 * i]);
    acc[2 * i + 1] = fma_h<kBf>(hi, v, acc[2 * i + 1]);
  }
}


// two fp32 values rounded to a packed 16-bit pair (x: low half)
template <bool kBf>
__device__ __forceinline__ uint32_t pack2(float x, float y) {
  if (kBf) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(x, y);
    return *reinterpret_cast<const uint32_t*>(&h);
  }
  const __half2 h = __floats2half2_rn(x, y);
  return *reinterpret_cast<const uint32_t*>(&h);
}

// 4 outputs out[bs..bs+3] = o (+ src[ps..ps+3] when ps >= 0: the TW result),
// 16-bit or fp32, tail-masked by n.
__device__ __forceinline__ void residual_store4(const ResidualArgs& args, int64_t bs, int n,
                                                const void* src, int64_t ps, float o0, float o1,
                                                float o2, float o3) {
  const bool obf = args.out_dtype == kBF16;
  const bool accum = ps >= 0;
  if (args.vec_ok && n >= 4 && bs % 4 == 0 && (!accum || ps % 4 == 0)) {
    if (args.out_dtype != kF32) {
      uint2* p = reinterpret_cast<uint2*>(static_cast<uint16_t*>(args.out) + bs);
      const uint2 prev =
          accum ? *reinterpret_cast<const uint2*>(static_cast<const uint16_t*>(src) + ps)
                : make_uint2(0u, 0u);
      const float2 lo2 = h2_to_f2(prev.x, obf), hi2 = h2_to_f2(prev.y, obf);
      const float f0 = lo2.x + o0, f1 = lo2.y + o1, f2 = hi2.x + o2, f3 = hi2.y + o3;
      uint2 w;
      if (!obf) {
        const __half2 x = __floats2half2_rn(f0, f1), y = __floats2half2_rn(f2, f3);
        w = make_uint2(*reinterpret_cast<const uint32_t*>(&x), *reinterpret_cast<const uint32_t*>(&y));
      } else {
        const __nv_bfloat162 x = __floats2bfloat162_rn(f0, f1);
        const __nv_bfloat162 y = __floats2bfloat162_rn(f2, f3);
        w = make_uint2(*reinterpret_cast<const uint32_t*>(&x), *reinterpret_cast<const uint32_t*>(&y));
      }
      *p = w;
    } else {
      float4* p = reinterpret_cast<float4*>(static_cast<float*>(args.out) + bs);
      const float4 prev =
          accum ? *reinterpret_cast<const float4*>(static_cast<const float*>(src) + ps)
                : make_float4(0.f, 0.f, 0.f, 0.f);
      *p = make_float4(prev.x + o0, prev.y + o1, prev.z + o2, prev.w + o3);
    }
    return;
  }
  const float o[4] = {o0, o1, o2, o3};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (i < n) {
      float w = o[i];
      if (accum) w += load_as_float(src, args.out_dtype, ps + i);
      store_from_float(args.out, args.out_dtype, bs + i, w);
    }
  }
}

// One CTA of K2: token block bx, column split by.  TPL tokens per lane: 8
// (one 16-byte chunk of a staged row per entry) or 16 (two chunks, T = 64:
// half the lanes per column, so the per-column work around the FMAs --
// metadata, entry broadcast, the output read-modify-write -- is spread over
// twice the products; odd columns of a warp step read their second chunk
// first, so each of the two loads of a warp covers all 32 banks).
template <int T, bool kBf, int TPL = 8, int NT = kResThreads>
__device__ __forceinline__ void residual_body(const ResidualArgs& args, const int bx,
                                              const int by) {
  extern __shared__ __align__(16) uint8_t res_smem[];
  uint16_t* sA = reinterpret_cast<uint16_t*>(res_smem);  // [K][T]
  constexpr int kH = TPL / 8;     // 16-byte chunks per lane and entry
  constexpr int L = T / TPL;      // lanes per column
  constexpr int kCols = 32 / L;   // columns per warp step
  static_assert(kH == 1 || kH == 2, "8 or 16 tokens per lane");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint16_t* at = static_cast<const uint16_t*>(args.at);
  const int K = args.K;
  const int sub = lane / L;
  const int tl = lane - sub * L;
  const int swp = kH == 2 ? (sub & 1) : 0;
  // tokens of the first (and second) chunk this lane reads
  const int tokA = tl * TPL + 8 * swp, tokB = tl * TPL + 8 * (1 - swp);
  const int64_t t0 = static_cast<int64_t>(bx) * T;
  const int64_t rem = args.M - t0;
  const int ntok = rem < T ? static_cast<int>(rem) : T;
  // this CTA's columns: split y of the descending-nnz order (by nnz)
  const int c0 = args.group_first[by], c1 = args.group_first[by + 1];
  // launched with programmatic dependent launch after K1: the TW result (and,
  // in a chain, A^T) is complete and visible only after this wait
  grid_dependency_wait();
  {
    constexpr int per_row = T / 8;
    // row K stays zero: padding entries (row K, value 0) add exactly 0
    for (int i = threadIdx.x; i < (K + 1) * per_row; i += NT) {
      const int r = i / per_row, j = (i - r * per_row) * 8;
      const int valid = r < K ? ntok - j : 0;
      const uint32_t bytes = valid >= 8 ? 16u : (valid > 0 ? static_cast<uint32_t>(valid) * 2 : 0u);
      cp_async_16(smem_u32(sA + r * T + j), bytes ? at + r * args.ld_at + t0 + j : at, bytes);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
  }
  // the next kernel may launch; it waits for this grid before touching data
  grid_launch_dependents();
  constexpr int kStep = kCols * (NT / 32);
  constexpr int G = L;  // entries per group (one per lane of the column)
  // entries: 16-bit value << 16 | row offset in 16-byte units (row * T / 8)
  const uint32_t zrow = static_cast<uint32_t>(K) * (T / 8);
  const uint8_t* sAa = reinterpret_cast<const uint8_t*>(sA + tokA);
  const uint8_t* sAb = reinterpret_cast<const uint8_t*>(sA + tokB);
  // whole blocks with 16-bit outputs of the input type and 16-byte aligned
  // rows (t0 is a multiple of T, pitches of 8 elements): one 16-byte
  // read-modify-write per chunk, the TW result added with FHFMA (x * 1 + acc:
  // exact product, one rounding, as widening and adding)
  const bool fast = args.vec_ok && args.out_dtype == (kBf ? kBF16 : kF16) && ntok == T &&
                    args.ld_out % 8 == 0 && (!args.src || args.ld_src % 8 == 0);
  const uint16_t one = kBf ? 0x3f80u : 0x3c00u;
  uint16_t* out16 = static_cast<uint16_t*>(args.out);
  const void* src = args.src ? args.src : args.out;
  const uint16_t* src16 = static_cast<const uint16_t*>(src);
  int cs = c0 + warp * kCols;
  // columns past c1 read the (zero-row) padding at the start of the lists
  int4 m = cs + sub < c1 ? __ldg(args.meta + cs + sub) : make_int4(0, 0, 0, 0);
  // Entry groups: lane tl of a column holds entry tl of each group and the
  // group is broadcast with shuffles -- except for 32-token blocks (4 lanes
  // per column, 8 tokens each), where every lane loads its column's whole
  // group with one 16-byte load (the shuffles share the MIO queue with the
  // shared-memory loads: 41.3 -> 39.3 us on 3072 x 768; with 16 tokens per
  // lane the extra registers cost more than the shuffles).  The current
  // column's first two groups are loaded here; later columns' at the end of
  // the previous step, so their latency overlaps its stores and the next
  // step's setup.
  constexpr bool kGL = G == 4 && TPL == 8;
  uint32_t c = 0, n1 = 0;
  uint4 c4 = make_uint4(0u, 0u, 0u, 0u), n4 = c4;
  const uint4 z4 = make_uint4(zrow, zrow, zrow, zrow);
  if constexpr (kGL) {
    c4 = __ldg(reinterpret_cast<const uint4*>(args.rv + m.x));
    n4 = __ldg(reinterpret_cast<const uint4*>(args.rv + m.x + G));
  } else {
    c = __ldg(args.rv + m.x + tl);
    n1 = __ldg(args.rv + m.x + tl + L);
  }
  for (; cs < c1; cs += kStep) {
    const int col = cs + sub;
    // the next step's metadata, one step ahead
    const int4 mn = col + kStep < c1 ? __ldg(args.meta + col + kStep) : make_int4(0, 0, 0, 0);
    const bool incol = col < c1;
    const int64_t bs0 = static_cast<int64_t>(m.z) * args.ld_out + t0;
    // the TW result of a kept column (workspace row m.w - 1, else the out row
    // itself); -1: residual-only column
    const int64_t ps0 = args.acc_all ? bs0
                        : m.w == 0 ? -1
                        : args.src ? static_cast<int64_t>(m.w - 1) * args.ld_src + t0
                                   : bs0;
    const int maxlen = __reduce_max_sync(0xffffffffu, m.y);
    float aa[8], ab[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) aa[i] = ab[i] = 0.f;
    // one entry: its staged row (one or two chunks) times its value
    auto entry = [&](uint32_t q) {
      // PRMT (zero-extended low half) + IMAD: the chunk address
      const uint32_t off = __byte_perm(q, 0u, 0x4410) * 16u;
      const uint16_t v = static_cast<uint16_t>(q >> 16);
      fma8<kBf>(aa, *reinterpret_cast<const uint4*>(sAa + off), v);
      if constexpr (kH == 2) fma8<kBf>(ab, *reinterpret_cast<const uint4*>(sAb + off), v);
    };
    // entry groups: lane tl holds entry tl of a group;
    // groups gi + 1, gi + 2 are in flight while gi is consumed.  Lists are
    // padded to whole groups with zero-row entries (row K of the block is
    // zero) and a lane group past its list substitutes them, so the entry
    // loop has no branches.
    int eo = 0;
    if constexpr (kGL) {
      // the column's lanes share the address of each group load
      const uint4* lq = reinterpret_cast<const uint4*>(args.rv + m.x);
      for (; eo + G <= maxlen; eo += G) {
        const uint4 f4 = __ldg(lq + 2);
        ++lq;
        if (eo >= m.y) c4 = z4;
        entry(c4.x);
        entry(c4.y);
        entry(c4.z);
        entry(c4.w);
        c4 = n4;
        n4 = f4;
      }
      if (eo < maxlen) {
        if (eo >= m.y) c4 = z4;
        const int cnt = maxlen - eo;
        entry(c4.x);
        if (cnt > 1) entry(c4.y);
        if (cnt > 2) entry(c4.z);
      }
      c4 = __ldg(reinterpret_cast<const uint4*>(args.rv + mn.x));
      n4 = __ldg(reinterpret_cast<const uint4*>(args.rv + mn.x + G));
    } else {
    const uint32_t* lp = args.rv + m.x + tl;
    for (; eo + G <= maxlen; eo += G) {
      const uint32_t f = __ldg(lp + 2 * L);
      lp += L;
      if (eo >= m.y) c = zrow;
#pragma unroll
      for (int j = 0; j < G; ++j) entry(L == 1 ? c : __shfl_sync(0xffffffffu, c, j, L));
      c = n1;
      n1 = f;
    }
    // the warp's last, partial group stops at its longest list (warp-uniform
    // count): the padding entries past it are not computed
    if (eo < maxlen) {
      if (eo >= m.y) c = zrow;
      const int cnt = maxlen - eo;
      int j = 0;
      if (L >= 8 && cnt >= 4) {
        // four entries unrolled (their shared loads in flight together), the
        // rest one by one
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) entry(__shfl_sync(0xffffffffu, c, jj, L));
        j = 4;
      }
#pragma unroll 1
      for (; j < cnt; ++j) entry(L == 1 ? c : __shfl_sync(0xffffffffu, c, j, L));
    }
    // the next column's first two entry groups, in flight during the stores
    c = __ldg(args.rv + mn.x + tl);
    n1 = __ldg(args.rv + mn.x + tl + L);
    }
    if (fast) {
      if (incol) {
        // the TW result is read here, not before the entry loop: holding it
        // across the loop costs registers the loop's loads in flight need
        if (ps0 >= 0) {
          fma8<kBf>(aa, *reinterpret_cast<const uint4*>(src16 + ps0 + tokA), one);
          if constexpr (kH == 2) fma8<kBf>(ab, *reinterpret_cast<const uint4*>(src16 + ps0 + tokB), one);
        }
        uint16_t* orow = out16 + bs0;
        *reinterpret_cast<uint4*>(orow + tokA) =
            make_uint4(pack2<kBf>(aa[0], aa[1]), pack2<kBf>(aa[2], aa[3]),
                       pack2<kBf>(aa[4], aa[5]), pack2<kBf>(aa[6], aa[7]));
        if constexpr (kH == 2)
          *reinterpret_cast<uint4*>(orow + tokB) =
              make_uint4(pack2<kBf>(ab[0], ab[1]), pack2<kBf>(ab[2], ab[3]),
                         pack2<kBf>(ab[4], ab[5]), pack2<kBf>(ab[6], ab[7]));
      }
    } else {
#pragma unroll
      for (int h = 0; h < kH; ++h) {
        const int tk = h ? tokB : tokA;
        const float* ac = h ? ab : aa;
        if (!incol || tk >= ntok) continue;
        const int64_t bs = bs0 + tk;
        const int64_t ps = ps0 < 0 ? -1 : ps0 + tk;
        residual_store4(args, bs, ntok - tk, src, ps, ac[0], ac[1], ac[2], ac[3]);
        if (tk + 4 < ntok)
          residual_store4(args, bs + 4, ntok - tk - 4, src, ps < 0 ? -1 : ps + 4, ac[4], ac[5],
                          ac[6], ac[7]);
      }
    }
    m = mn;
  }
}

template <int T, bool kBf, int TPL, int NT = kResThreads>
__global__ void __launch_bounds__(NT, 1)
    tw_residual_kernel(const __grid_constant__ ResidualArgs args) {
  residual_body<T, kBf, TPL, NT>(args, blockIdx.x, blockIdx.y);
}

// K2 of several layers in one launch (the TEW grouped step): layer p owns
// CTAs [cta0[p], cta0[p + 1]), n_blocks x n_groups of them; its token block
// size picks the body (64 for K <= 1536, 32 up to K = 3072).
template <bool kBf>
__global__ void __launch_bounds__(kResThreads, 1)
    tw_residual_group_kernel(const __grid_constant__ ResidualGroupArgs g) {
  int p = 0;
  while (p + 1 < g.n && static_cast<int>(blockIdx.x) >= g.cta0[p + 1]) ++p;
  const ResidualArgs& a = g.args[p];
  const int local = static_cast<int>(blockIdx.x) - g.cta0[p];
  const int bx = local % a.n_blocks, by = local / a.n_blocks;
  if (a.tokens_per_lane == 16) {
    residual_body<64, kBf, 16>(a, bx, by);
    return;
  }
  switch (a.block_tokens) {
    case 64: residual_body<64, kBf>(a, bx, by); break;
    case 32: residual_body<32, kBf>(a, bx, by); break;
    default: residual_body<16, kBf>(a, bx, by); break;
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
  if (args.accumulate[col] || args.acc_all) acc += load_as_float(args.out, args.out_dtype, base);
  store_from_float(args.out, args.out_dtype, base, acc);
}

// ct[u] = src[src_row[u]] or 0: the caller's tile product placed at the union
// rows (GemmOutput.expand + re-condense of executor.py:194-203, on the device).
// Also the row permutation of a natural-order A^T into a plan's row-run
// layout (TwPlan.prepare(at=...)): 16-byte copies when rows are aligned.
__global__ void scatter_rows_kernel(const uint8_t* src, int64_t ld_src, const int32_t* src_row,
                                    uint8_t* dst, int64_t ld_dst, int64_t M, int esz, int vec) {
  const int u = blockIdx.y;
  const int sr = __ldg(src_row + u);
  const int64_t bytes = M * esz;
  uint8_t* d = dst + static_cast<int64_t>(u) * ld_dst * esz;
  const uint8_t* s = sr >= 0 ? src + static_cast<int64_t>(sr) * ld_src * esz : nullptr;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t step = static_cast<int64_t>(gridDim.x) * blockDim.x;
  if (vec) {
    for (int64_t i = t0; i < bytes / 16; i += step)
      reinterpret_cast<uint4*>(d)[i] = s ? reinterpret_cast<const uint4*>(s)[i] : make_uint4(0, 0, 0, 0);
    return;
  }
  for (int64_t i = t0; i < bytes; i += step) d[i] = s ? s[i] : 0;
}

// 32 x 32 shared-memory transpose with dtype conversion (general fallback).
__global__ void transpose_cast_kernel(const void* a, int32_t a_dtype, int64_t M, int64_t K,
                                      int64_t lda, void* at, int32_t at_dtype, int64_t ld_at,
                                      const int32_t* out_row) {
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
    if (k < K && m < M) {
      const int64_t ko = out_row ? __ldg(out_row + k) : k;
      store_from_float(at, at_dtype, ko * ld_at + m, tile[threadIdx.x][i]);
    }
  }
}

// fp32 plans: A (M x K, any dtype) -> [A_hi^T; A_lo^T] (2K x M fp16),
// hi = fp16(a), lo = fp16(a - hi): the hi/lo operand pair of the split
// product (tw_capi.cu, plan creation).
__global__ void transpose_split_kernel(const void* a, int32_t a_dtype, int64_t M, int64_t K,
                                       int64_t lda, __half* at, int64_t ld_at) {
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
    if (k < K && m < M) {
      const float v = tile[threadIdx.x][i];
      const __half hi = __float2half_rn(v);
      at[k * ld_at + m] = hi;
      at[(k + K) * ld_at + m] = __float2half_rn(v - __half2float(hi));
    }
  }
}

// 16-bit -> 16-bit (same type) tile transpose, 64 tokens x KT k per CTA,
// 16-byte loads and stores: each thread first issues all its row loads
// (KT / 32 of them, in flight together), then writes 8 consecutive m of a
// row of A^T per 16-byte store.  Needs M, K, lda, ld_at multiples of 8 and
// 16-byte aligned bases.  out_row (optional) permutes the A^T rows (the
// plan's row-run layout).
template <int KT>
__global__ void __launch_bounds__(256) transpose16_kernel(const uint16_t* a, int64_t M, int64_t K,
                                                          int64_t lda, uint16_t* at,
                                                          int64_t ld_at, const int32_t* out_row) {
  constexpr int kChunks = KT / 8;                 // 16-byte chunks per tile row of A
  constexpr int kItems = 64 * kChunks / 256;      // per thread, both phases
  // [m][k] with the 8-element k-chunk index XOR-swizzled by m / 8, so the
  // column reads of the second phase hit 8 different banks
  __shared__ __align__(16) uint16_t tile[64][KT];
  const int64_t k0 = static_cast<int64_t>(blockIdx.x) * KT;
  const int64_t m0 = static_cast<int64_t>(blockIdx.y) * 64;
  const int t = threadIdx.x;
  uint4 v[kItems];
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const int idx = t + r * 256;
    const int mi = idx / kChunks, kc = idx % kChunks;
    const int64_t m = m0 + mi, k = k0 + kc * 8;
    v[r] = (m < M && k < K) ? *reinterpret_cast<const uint4*>(a + m * lda + k)
                            : make_uint4(0u, 0u, 0u, 0u);
  }
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const int idx = t + r * 256;
    const int mi = idx / kChunks, kc = idx % kChunks;
    *reinterpret_cast<uint4*>(&tile[mi][(kc ^ (mi >> 3)) * 8]) = v[r];
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const int idx = t + r * 256;
    const int ki = idx >> 3, mc = idx & 7;
    const int64_t k = k0 + ki, m = m0 + mc * 8;
    if (k >= K || m >= M) continue;
    const int col = ((ki >> 3) ^ mc) * 8 + (ki & 7);
    const int64_t ko = out_row ? __ldg(out_row + k) : k;
    uint32_t w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
      w[j] = static_cast<uint32_t>(tile[mc * 8 + 2 * j][col]) |
             (static_cast<uint32_t>(tile[mc * 8 + 2 * j + 1][col]) << 16);
    *reinterpret_cast<uint4*>(at + ko * ld_at + m) = make_uint4(w[0], w[1], w[2], w[3]);
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

int residual_block_tokens(int32_t K, int* ctas_per_sm) {
  // T tokens per CTA (8 per lane): the largest block (K + 1) * T * 2 bytes
  // of at most ~200 KB, so the column lists (re-read once per block) are
  // amortised over as many tokens as shared memory allows; one 32-warp CTA
  // per SM hides the list loads
  constexpr int64_t kMaxBlock = 200 * 1024;
  for (int T : {64, 32, 16}) {
    const int64_t bytes = static_cast<int64_t>(K + 1) * T * 2;
    if (bytes <= kMaxBlock) {
      *ctas_per_sm = 1;
      return T;
    }
  }
  *ctas_per_sm = 0;
  return 0;
}

template <int T, bool kBf, int TPL, int NT = kResThreads>
static cudaError_t launch_res_t(const ResidualArgs& args, cudaStream_t stream) {
  const size_t smem = static_cast<size_t>(args.K + 1) * T * 2;
  // the dynamic shared-memory limit is raised once per device (to the
  // largest block any K allows), not on every launch
  static uint64_t configured = 0;  // bit per device ordinal
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev >= 64 || !(configured >> dev & 1u)) {
    e = cudaFuncSetAttribute(tw_residual_kernel<T, kBf, TPL, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(200 * 1024 + 2 * T));
    if (e != cudaSuccess) return e;
    if (dev < 64) configured |= uint64_t{1} << dev;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(args.n_blocks), static_cast<unsigned>(args.n_groups));
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  // programmatic dependent launch: K2's CTAs start as K1's leave (the
  // kernel waits with griddepcontrol.wait before reading anything)
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, tw_residual_kernel<T, kBf, TPL, NT>, args);
}

template <int T, int TPL = 8, int NT = kResThreads>
static cudaError_t launch_res(const ResidualArgs& args, cudaStream_t stream) {
  return args.in_dtype == kBF16 ? launch_res_t<T, true, TPL, NT>(args, stream)
                                : launch_res_t<T, false, TPL, NT>(args, stream);
}

cudaError_t launch_tw_residual_group(const ResidualGroupArgs& g, cudaStream_t stream) {
  if (g.n < 1 || g.n > kMaxResGroup) return cudaErrorInvalidValue;
  size_t smem = 0;
  bool bf = false;
  for (int p = 0; p < g.n; ++p) {
    const ResidualArgs& a = g.args[p];
    if (!a.rv || a.block_tokens <= 0) return cudaErrorInvalidValue;  // staged kernels only
    smem = std::max(smem, static_cast<size_t>(a.K + 1) * a.block_tokens * 2);
    bf = a.in_dtype == kBF16;
    if ((a.in_dtype == kBF16) != (g.args[0].in_dtype == kBF16)) return cudaErrorInvalidValue;
  }
  const int grid = g.cta0[g.n];
  if (grid <= 0) return cudaSuccess;
  static uint64_t configured = 0;  // bit per device ordinal (both dtypes)
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev >= 64 || !(configured >> dev & 1u)) {
    for (auto* k : {tw_residual_group_kernel<false>, tw_residual_group_kernel<true>}) {
      e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024 + 128);
      if (e != cudaSuccess) return e;
    }
    if (dev < 64) configured |= uint64_t{1} << dev;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(kResThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return bf ? cudaLaunchKernelEx(&cfg, tw_residual_group_kernel<true>, g)
            : cudaLaunchKernelEx(&cfg, tw_residual_group_kernel<false>, g);
}

cudaError_t launch_tw_residual(const ResidualArgs& args, cudaStream_t stream) {
  if (args.n_cols <= 0 || args.M <= 0) return cudaSuccess;
  switch (args.rv ? args.block_tokens : 0) {
    case 64:
      return args.tokens_per_lane == 16 ? launch_res<64, 16>(args, stream)
                                        : launch_res<64>(args, stream);
    case 32: return launch_res<32>(args, stream);
    case 16: return launch_res<16>(args, stream);
    default: break;
  }
  dim3 grid(static_cast<unsigned>((args.M + 255) / 256), static_cast<unsigned>(args.n_cols));
  tw_residual_direct_kernel<<<grid, 256, 0, stream>>>(args);
  return cudaGetLastError();
}

// Split-K reduction (tw_capi.cu, kSplitKMaxTokens): one thread per 4 tokens
// of a row, the partials summed in split order, launched with programmatic
// dependent launch after K1 (waits before reading the partials).
__global__ void __launch_bounds__(256) splitk_reduce_kernel(const __grid_constant__ SplitKArgs a) {
  grid_dependency_wait();
  const int r = blockIdx.y;
  const int t = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (r >= a.rows || t >= a.M) return;
  const float* src = a.ws + static_cast<int64_t>(r) * a.ld_ws + t;
  float4 acc = *reinterpret_cast<const float4*>(src);
  for (int j = 1; j < a.splits; ++j) {
    const float4 v = *reinterpret_cast<const float4*>(src + j * a.split_stride);
    acc.x += v.x;
    acc.y += v.y;
    acc.z += v.z;
    acc.w += v.w;
  }
  const int64_t orow = a.rowmap ? __ldg(a.rowmap + r) : r;
  const int64_t o = orow * a.ld_out + t;
  const float f[4] = {acc.x, acc.y, acc.z, acc.w};
  const int n = a.M - t < 4 ? a.M - t : 4;
  for (int i = 0; i < n; ++i) store_from_float(a.out, a.out_dtype, o + i, f[i]);
}

cudaError_t launch_splitk_reduce(const SplitKArgs& a, cudaStream_t stream) {
  if (a.rows <= 0 || a.M <= 0) return cudaSuccess;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>((a.M + 1023) / 1024), static_cast<unsigned>(a.rows));
  cfg.blockDim = dim3(256);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, splitk_reduce_kernel, a);
}

cudaError_t launch_transpose_cast(const void* a, int32_t a_dtype, int64_t M, int64_t K,
                                  int64_t lda, void* at, int32_t at_dtype, int64_t ld_at,
                                  const int32_t* out_row, cudaStream_t stream) {
  if (M <= 0 || K <= 0) return cudaSuccess;
  const bool fast = a_dtype == at_dtype && a_dtype != kF32 && M % 8 == 0 && K % 8 == 0 &&
                    lda % 8 == 0 && ld_at % 8 == 0 &&
                    reinterpret_cast<uintptr_t>(a) % 16 == 0 && reinterpret_cast<uintptr_t>(at) % 16 == 0;
  if (fast) {
    // 64 x 128 tiles (4 loads in flight per thread) unless K is small
    if (K >= 128 && !getenv("TW_T64")) {
      dim3 grid(static_cast<unsigned>((K + 127) / 128), static_cast<unsigned>((M + 63) / 64));
      transpose16_kernel<128><<<grid, 256, 0, stream>>>(static_cast<const uint16_t*>(a), M, K,
                                                        lda, static_cast<uint16_t*>(at), ld_at,
                                                        out_row);
    } else {
      dim3 grid(static_cast<unsigned>((K + 63) / 64), static_cast<unsigned>((M + 63) / 64));
      transpose16_kernel<64><<<grid, 256, 0, stream>>>(static_cast<const uint16_t*>(a), M, K, lda,
                                                       static_cast<uint16_t*>(at), ld_at, out_row);
    }
    return cudaGetLastError();
  }
  dim3 grid(static_cast<unsigned>((K + 31) / 32), static_cast<unsigned>((M + 31) / 32));
  dim3 block(32, 8);
  transpose_cast_kernel<<<grid, block, 0, stream>>>(a, a_dtype, M, K, lda, at, at_dtype, ld_at,
                                                     out_row);
  return cudaGetLastError();
}

cudaError_t launch_scatter_rows(const void* src, int64_t ld_src, const int32_t* src_row,
                                int32_t n_rows, void* dst, int64_t ld_dst, int64_t M, int esz,
                                cudaStream_t stream) {
  if (n_rows <= 0 || M <= 0) return cudaSuccess;
  const int64_t bytes = M * esz;
  const int vec = bytes % 16 == 0 && (ld_src * esz) % 16 == 0 && (ld_dst * esz) % 16 == 0 &&
                  reinterpret_cast<uintptr_t>(src) % 16 == 0 &&
                  reinterpret_cast<uintptr_t>(dst) % 16 == 0;
  const int64_t items = vec ? bytes / 16 : bytes;
  unsigned gx = static_cast<unsigned>(std::min<int64_t>((items + 255) / 256, 64));
  dim3 grid(gx, static_cast<unsigned>(n_rows));
  scatter_rows_kernel<<<grid, 256, 0, stream>>>(static_cast<const uint8_t*>(src), ld_src, src_row,
                                                static_cast<uint8_t*>(dst), ld_dst, M, esz, vec);
  return cudaGetLastError();
}

cudaError_t launch_transpose_split(const void* a, int32_t a_dtype, int64_t M, int64_t K,
                                   int64_t lda, void* at, int64_t ld_at, cudaStream_t stream) {
  if (M <= 0 || K <= 0) return cudaSuccess;
  dim3 grid(static_cast<unsigned>((K + 31) / 32), static_cast<unsigned>((M + 31) / 32));
  transpose_split_kernel<<<grid, dim3(32, 8), 0, stream>>>(a, a_dtype, M, K, lda,
                                                           static_cast<__half*>(at), ld_at);
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
