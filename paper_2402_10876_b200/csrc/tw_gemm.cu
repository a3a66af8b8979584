// K1 -- tw_gather_gemm: one persistent, warp-specialised sm_100a kernel over
// every (column tile, 128-token block) work unit of a TW layer.
//
// Replaces the reference's per-tile CPU loop (executor.py:121-177 gemm_cto /
// _tile_product / _mac_kernel and the threaded lanes of execute_batched,
// executor.py:230-265):
//   C'[:, cols_i] = A[:, kept_rows_i] . P_i        for every tile i
// computed as  C'^T tile (BN x 128 tokens) = P_i^T . A^T[kept_rows_i, tokens].
//
// Roles (256 threads, 1 CTA per SM):
//   warp 0      TMA producer: 32 lanes each issue one tile::gather4 (4 kept
//               rows x 64 tokens) of A^T per stage; lane 0 adds the payload box.
//   warp 1      MMA issuer: one thread issues tcgen05.mma.kind::f16
//               (M=128 tokens, N=BN tile columns, K=16) into a TMEM accumulator.
//   warp 2      TMEM allocator (2*BN columns: double-buffered accumulators).
//   warps 4-7   epilogue: tcgen05.ld -> convert -> store C'^T rows (optionally
//               scattered through rowmap for the TEW union layout).
//
// Shared memory per stage: A = 2 x [64 k][128 B] (MN-major, 128-B swizzle),
// B = [BN cols][128 B] (K-major, 128-B swizzle) -- the CTO transposed payload
// layout of formats.py:200 is exactly this K-major B operand.
#include "sm100_ptx.cuh"
#include "tw_kernels.cuh"

#include <cuda_bf16.h>
#include <cuda_fp16.h>

namespace tw {

namespace {

constexpr int kThreads = 256;
constexpr int kAHalfBytes = 64 * kBK * 2;      // 64 tokens x 64 rows x 2 B = 8 KB
constexpr int kABytes = 2 * kAHalfBytes;       // 16 KB per stage

template <int BN>
struct Cfg {
  static constexpr int kBBytes = BN * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStages = (BN >= 256) ? 4 : (BN >= 128 ? 6 : 8);
  static constexpr int kBarrierBytes = (2 * kStages + 4) * 8 + 16;
  static constexpr int kSmemBytes = kStages * kStageBytes + kBarrierBytes + 1024;
  static constexpr uint32_t kTmemCols = 2 * BN;
};

__device__ __forceinline__ void store_out(void* out, int32_t dtype, int64_t off, float v) {
  if (dtype == kF32) {
    static_cast<float*>(out)[off] = v;
  } else if (dtype == kF16) {
    static_cast<__half*>(out)[off] = __float2half_rn(v);
  } else {
    static_cast<__nv_bfloat16*>(out)[off] = __float2bfloat16_rn(v);
  }
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    tw_gather_gemm_kernel(const __grid_constant__ CUtensorMap map_at,
                          const __grid_constant__ CUtensorMap map_pay, const GemmArgs args,
                          uint32_t idesc) {
  using C = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::kStages * kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    fence_barrier_init();
    fence_proxy_async_smem();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_at);
    tma_prefetch_desc(&map_pay);
  }
  if (warp == 2) {
    tmem_alloc(tmem_slot, C::kTmemCols);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int n_units = args.n_units;
  const int n_sub = args.n_sub;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    int stage = 0;
    uint32_t phase = 0;
    const int grp = lane & 15;   // which 4-row group of the 64-row stage
    const int half = lane >> 4;  // which 64-token half of the 128-token block
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      const int mb = u / n_sub;
      const SubTile d = args.subtiles[args.order[u - mb * n_sub]];
      const int32_t* idx = args.rowidx + static_cast<int64_t>(d.idx_row) * args.Kp;
      const int tok0 = mb * kBM + half * 64;
      for (int ks = 0; ks < d.kp_steps; ++ks) {
        mbar_wait(&empty[stage], phase ^ 1u);
        if (lane == 0) mbar_arrive_expect_tx(&full[stage], C::kStageBytes);
        __syncwarp();
        const int4 r = __ldg(reinterpret_cast<const int4*>(idx + ks * kBK + grp * 4));
        uint8_t* dst = sA + stage * kABytes + half * kAHalfBytes + grp * 4 * 128;
        tma_gather4(dst, &map_at, &full[stage], tok0, r.x, r.y, r.z, r.w);
        if (lane == 0) {
          tma_load_2d(sB + stage * C::kBBytes, &map_pay, &full[stage], ks * kBK, d.pay_row);
        }
        if (++stage == C::kStages) {
          stage = 0;
          phase ^= 1u;
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int j = 0;
      for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++j) {
        const int mb = u / n_sub;
        const SubTile d = args.subtiles[args.order[u - mb * n_sub]];
        const int acc = j & 1;
        mbar_wait(&tempty[acc], ((j >> 1) & 1) ^ 1u);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int ks = 0; ks < d.kp_steps; ++ks) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + stage * kABytes);
          const uint32_t b0 = smem_u32(sB + stage * C::kBBytes);
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk) {
            // A: MN-major SW128, LBO = 8 KB between 64-token halves, SBO = 1 KB
            //    between 8-row K groups; 16 K rows = 2 KB per MMA.
            // B: K-major SW128, SBO = 1 KB between 8-column groups; 16 K = 32 B.
            const uint64_t adesc = umma_desc_sw128(a0 + kk * 2048, kAHalfBytes, 1024);
            const uint64_t bdesc = umma_desc_sw128(b0 + kk * 32, 16, 1024);
            umma_f16(d_tmem, adesc, bdesc, idesc, (ks | kk) != 0);
          }
          umma_commit(&empty[stage]);
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1u;
          }
        }
        umma_commit(&tfull[acc]);
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    int j = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++j) {
      const int mb = u / n_sub;
      const SubTile d = args.subtiles[args.order[u - mb * n_sub]];
      const int acc = j & 1;
      mbar_wait(&tfull[acc], (j >> 1) & 1);
      tc_fence_after();
      const int m = mb * kBM + q * 32 + lane;
      const bool live = m < args.M;
      const uint32_t t0 = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN;
      for (int c0 = 0; c0 < d.width; c0 += 16) {
        uint32_t r[16];
        tmem_ld_32x32b_x16(t0 + c0, r);
        tmem_ld_wait();
        if (live) {
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            const int col = c0 + c;
            if (col < d.width) {
              const int crow = d.out_row + col;
              const int orow = args.rowmap ? __ldg(args.rowmap + crow) : crow;
              store_out(args.out, args.out_dtype,
                        static_cast<int64_t>(orow) * args.ld_out + m, __uint_as_float(r[c]));
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::kTmemCols);
  }
}

template <int BN>
cudaError_t launch_bn(const CUtensorMap& map_at, const CUtensorMap& map_pay, const GemmArgs& args,
                      int in_dtype, int grid, cudaStream_t stream) {
  using C = Cfg<BN>;
  const uint32_t idesc =
      umma_idesc_f16(kBM, BN, in_dtype == kBF16 ? 1u : 0u, /*a MN-major*/ 1u, /*b K-major*/ 0u);
  tw_gather_gemm_kernel<BN><<<grid, kThreads, C::kSmemBytes, stream>>>(map_at, map_pay, args,
                                                                       idesc);
  return cudaGetLastError();
}

template <int BN>
cudaError_t configure_bn() {
  return cudaFuncSetAttribute(tw_gather_gemm_kernel<BN>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<BN>::kSmemBytes);
}

}  // namespace

cudaError_t configure_gemm_kernels() {
  cudaError_t e = configure_bn<32>();
  if (e == cudaSuccess) e = configure_bn<64>();
  if (e == cudaSuccess) e = configure_bn<128>();
  if (e == cudaSuccess) e = configure_bn<256>();
  return e;
}

cudaError_t launch_tw_gather_gemm(const CUtensorMap& map_at, const CUtensorMap& map_pay,
                                  const GemmArgs& args, int bn, int in_dtype, int grid,
                                  cudaStream_t stream) {
  if (args.n_units <= 0) return cudaSuccess;
  switch (bn) {
    case 32: return launch_bn<32>(map_at, map_pay, args, in_dtype, grid, stream);
    case 64: return launch_bn<64>(map_at, map_pay, args, in_dtype, grid, stream);
    case 128: return launch_bn<128>(map_at, map_pay, args, in_dtype, grid, stream);
    case 256: return launch_bn<256>(map_at, map_pay, args, in_dtype, grid, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace tw
