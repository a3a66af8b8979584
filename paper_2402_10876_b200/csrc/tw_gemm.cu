// K1 -- tw_gemm_kernel: one persistent, warp-specialised sm_100a kernel over
// every (column tile, 256-token block) work unit of a TW layer.
//
// Replaces the reference's per-tile CPU loop (executor.py:121-177 gemm_cto /
// _tile_product / _mac_kernel and the threaded lanes of execute_batched,
// executor.py:230-265):
//   C'[:, cols_i] = A[:, kept_rows_i] . P_i        for every tile i
// computed transposed, one UMMA tile per unit:
//   C'^T[cols_i, tokens] (128 x 256) = P_i^T (128 x K') . X[runs_i, tokens] (K' x 256)
// with the payload P_i^T as the K-major A operand (exactly the CTO transposed
// payload layout of formats.py:200) and the plan's grouped input X (tile i's
// kept rows are a few contiguous runs, see tw_capi.cu) as the MN-major B
// operand.  TMEM lanes are output columns and TMEM columns are tokens, so an
// epilogue thread holds a contiguous segment of one C'^T row.
//
// Work decomposition.  A unit is (tn-token block, 128-column sub-tile), tn in
// {64, 128, 192, 256} chosen per launch by the host so the units fill the SMs;
// its k-steps (64 kept rows each) are stages.  Units are strided over the
// persistent CTAs; optionally (TW_STREAMK=1, tn = 256) the CTA-major stage
// list is cut into equal ranges (stream-K): a unit cut by a range boundary is
// split in two, the lower CTA publishes its head k-steps as an fp32 partial,
// the higher CTA adds it in its epilogue.  CTAs walk their range backwards so
// a CTA only waits on a lower-numbered CTA that published first.
//
// Roles (1 CTA per SM):
//   warp 0      payload producer: one TMA box per stage (128 cols x 64 k).
//   warp 1      TMEM allocator (2 x 256 columns: double-buffered accumulators)
//               and MMA issuer: one thread, tcgen05.mma.kind::f16 M=128 N=tn K=16.
//   warps 4..   gather producers (kGatherWGs warpgroups): the tile's 64 kept
//               A^T rows of a stage, each row's tn tokens (512 contiguous bytes
//               for tn = 256) as 16-byte cp.async into the 128-B swizzled
//               MN-major layout; gather indices are prefetched one stage ahead
//               in registers.  A^T is read where it lies: no repacked copy.
//   last 8      epilogue: warp w owns TMEM lanes 32*(w%4).. (output columns)
//               and token half; tcgen05.ld -> fp16/bf16/fp32 -> swizzled smem
//               tile -> one TMA 2-D store per 32 x 32 block (16-byte stores for
//               the TEW row scatter through rowmap and ragged sub-tiles).
//
// Shared memory per stage: payload [128 cols][128 B] K-major SW128 (16 KB) and
// X [4 x 64-token chunks][64 k][128 B] MN-major SW128 (32 KB); 4 stages.
#include "sm100_ptx.cuh"
#include "tw_kernels.cuh"

#include <cuda_bf16.h>
#include <cuda_fp16.h>

namespace tw {

namespace {

#ifndef TW_GATHER_WARPGROUPS
#define TW_GATHER_WARPGROUPS 3
#endif
constexpr int kGatherWGs = TW_GATHER_WARPGROUPS;
constexpr int kPayloadWarp = 0;
constexpr int kMmaWarp = 1;
constexpr int kGatherWarp0 = 4;
constexpr int kGatherWarps = 4 * kGatherWGs;
constexpr int kEpilogueWarp0 = kGatherWarp0 + kGatherWarps;
constexpr int kEpilogueWarps = 8;
constexpr int kThreads = 32 * (kEpilogueWarp0 + kEpilogueWarps);
constexpr int kTileN = kTN;                          // max tokens per unit (UMMA N)
constexpr int kChunkBytes = 64 * kBK * 2;            // 64 tokens x 64 rows x 2 B = 8 KB
constexpr int kXBytes = (kTileN / 64) * kChunkBytes; // 32 KB per stage
constexpr int kPBytes = kBN * kBK * 2;               // 16 KB per stage
constexpr int kStageBytes = kXBytes + kPBytes;
constexpr int kStages = 4;
constexpr int kMaxSmemSub = 32;                      // sub-tile table cached in smem up to this
constexpr int kSubBytes = kMaxSmemSub * static_cast<int>(sizeof(SubTile));
constexpr int kBarrierBytes = 256;
constexpr int kStgBytes = 4096;                      // per epilogue warp: [32 rows][128 B]
constexpr int kSmemBytes =
    kStages * kStageBytes + kEpilogueWarps * kStgBytes + kBarrierBytes + kSubBytes + 1024;
constexpr uint32_t kTmemCols = 2 * kTileN;           // double-buffered 128 x 256 fp32
constexpr int kEpiBarrier = 2;                       // named barrier id of the epilogue warps
constexpr int kEpiThreads = 32 * kEpilogueWarps;
static_assert(kSmemBytes <= 227 * 1024, "shared memory budget");
static_assert(kEpilogueWarp0 % 4 == 0, "epilogue warps must start a warpgroup (TMEM lane quadrants)");

// Sub-tile table in visiting order (smem copy when small enough).
struct Tables {
  const SubTile* sub;
  int n_sub;
  __device__ __forceinline__ const SubTile& get(int i) const { return sub[i]; }
  // index j with sub[j].stage_off <= rem < sub[j].stage_off + sub[j].kp_steps
  __device__ __forceinline__ int find(int rem) const {
    int lo = 0, hi = n_sub - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (sub[mid].stage_off <= rem) lo = mid; else hi = mid - 1;
    }
    return lo;
  }
};

enum SegKind : int { kSegFull = 0, kSegHead = 1, kSegTail = 2 };

struct Seg {
  int mb, sub, ks0, ks1, kind;
  SubTile d;
};

// Deterministic per-CTA segment sequence, identical in every role.
//   unit mode  (split == 0): units blockIdx.x, +gridDim.x, ... whole.
//   stream-K   (split == 1): stage range [lo, hi) of the CTA-major stage list,
//                            walked backwards segment by segment.
struct SegWalker {
  int64_t lo, g;  // stream-K cursor
  int u;          // unit-mode cursor
  __device__ __forceinline__ void init(const GemmArgs& a) {
    if (a.split) {
      const int64_t T = static_cast<int64_t>(a.n_mblk) * a.spm;
      lo = T * blockIdx.x / gridDim.x;
      g = T * (blockIdx.x + 1) / gridDim.x;
    } else {
      u = blockIdx.x;
    }
  }
  __device__ __forceinline__ bool next(const GemmArgs& a, const Tables& t, Seg& s) {
    if (a.split) {
      if (g <= lo) return false;
      const int64_t h = g - 1;
      s.mb = static_cast<int>(h / a.spm);
      const int rem = static_cast<int>(h - static_cast<int64_t>(s.mb) * a.spm);
      s.sub = t.find(rem);
      s.d = t.get(s.sub);
      const int64_t u0 = static_cast<int64_t>(s.mb) * a.spm + s.d.stage_off;
      const int64_t s0 = u0 > lo ? u0 : lo;
      s.ks0 = static_cast<int>(s0 - u0);
      s.ks1 = static_cast<int>(g - u0);
      const bool head = s.ks0 == 0, tail = s.ks1 == s.d.kp_steps;
      s.kind = (head && tail) ? kSegFull : (head ? kSegHead : kSegTail);
      g = s0;
      return true;
    }
    if (u >= a.n_units) return false;
    s.mb = u / a.n_sub;
    s.sub = u - s.mb * a.n_sub;
    s.d = t.get(s.sub);
    s.ks0 = 0;
    s.ks1 = s.d.kp_steps;
    s.kind = kSegFull;
    u += gridDim.x;
    return true;
  }
};

__device__ __forceinline__ void st_release_gpu(int32_t* p, int32_t v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ int32_t ld_acquire_gpu(const int32_t* p) {
  int32_t v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint32_t pack2(float a, float b, int32_t dtype) {
  if (dtype == kF16) {
    const __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&h);
  }
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

// Epilogue of one accumulator quarter: the warp's 32 output rows (columns
// q*32.. of the tile) x tokens [tok0, tok0 + 128), in 4 chunks of 32 tokens.
// Per chunk: tcgen05.ld (next chunk in flight), optional stream-K partial add,
// convert, then either
//   * stage [32 rows][32 tok] in this warp's swizzled smem tile and issue one
//     TMA 2-D store (condensed output, all 32 rows inside the sub-tile), or
//   * 16-byte stores of each thread's row segment (TEW row scatter through
//     rowmap, ragged sub-tiles, misaligned outputs).
__device__ __forceinline__ void epilogue_rows(const GemmArgs& args, const CUtensorMap* map_out,
                                              uint8_t* stg, uint32_t t0, int lane, int orow,
                                              bool row_live, bool warp_full, int row0_tma,
                                              int tok0, int ntok, const float* add) {
  const bool do_store = !(args.flags & kFlagSkipStore);
  const int esz = args.out_dtype == kF32 ? 4 : 2;
  const bool use_tma = do_store && args.use_tma_store && warp_full;
  uint8_t* row_base =
      static_cast<uint8_t*>(args.out) + static_cast<int64_t>(orow) * args.ld_out * esz;
  if (ntok <= 0) return;
#pragma unroll 1
  for (int c = 0; c < ntok; c += 32) {
    // one 32-token chunk of the row, converted in place in the load registers
    uint32_t w[32];
    tmem_ld_32x32b_x32(t0 + c, w);
    tmem_ld_wait();
    if (add) {
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        const float4 p = __ldcg(reinterpret_cast<const float4*>(add + c + i));
        w[i] = __float_as_uint(__uint_as_float(w[i]) + p.x);
        w[i + 1] = __float_as_uint(__uint_as_float(w[i + 1]) + p.y);
        w[i + 2] = __float_as_uint(__uint_as_float(w[i + 2]) + p.z);
        w[i + 3] = __float_as_uint(__uint_as_float(w[i + 3]) + p.w);
      }
    }
    if (!do_store) continue;
    const int tok = tok0 + c;
    if (tok >= args.M) continue;
    if (esz == 2) {
      // packed row segment: 16 words (element pairs); w[i] <- (w[2i], w[2i+1])
#pragma unroll
      for (int i = 0; i < 16; ++i)
        w[i] = pack2(__uint_as_float(w[2 * i]), __uint_as_float(w[2 * i + 1]), args.out_dtype);
    }
    if (use_tma) {
      // the TMA store that last read this staging tile must be done with it
      if (lane == 0) bulk_wait_read<0>();
      __syncwarp();
      // row `lane` of the tile; 16-byte chunk index XOR-swizzled to match the
      // tensor map (SWIZZLE_64B for 64-byte rows, SWIZZLE_128B for 128-byte)
      if (esz == 4) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          *reinterpret_cast<uint4*>(stg + lane * 128 + ((j ^ (lane & 7)) << 4)) =
              make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          *reinterpret_cast<uint4*>(stg + lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4)) =
              make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_2d(map_out, stg, tok, row0_tma);
        bulk_commit();
      }
      continue;
    }
    if (!row_live) continue;
    const bool full = args.vec_ok && tok + 32 <= args.M;
    if (esz == 4) {
      float* dst = reinterpret_cast<float*>(row_base) + tok;
      if (full) {
#pragma unroll
        for (int i = 0; i < 32; i += 4)
          *reinterpret_cast<uint4*>(dst + i) = make_uint4(w[i], w[i + 1], w[i + 2], w[i + 3]);
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (tok + i < args.M) dst[i] = __uint_as_float(w[i]);
      }
    } else {
      uint16_t* dst = reinterpret_cast<uint16_t*>(row_base) + tok;
      if (full) {
#pragma unroll
        for (int i = 0; i < 16; i += 4)
          *reinterpret_cast<uint4*>(dst + 2 * i) = make_uint4(w[i], w[i + 1], w[i + 2], w[i + 3]);
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          if (tok + 2 * i < args.M) dst[2 * i] = static_cast<uint16_t>(w[i] & 0xFFFFu);
          if (tok + 2 * i + 1 < args.M) dst[2 * i + 1] = static_cast<uint16_t>(w[i] >> 16);
        }
      }
    }
  }
}

// Stream-K head segment: raw fp32 accumulator row -> workspace [128 cols][256 tok].
__device__ __forceinline__ void epilogue_partial_row(float* ws_row, uint32_t t0, int tok_half) {
  uint32_t r[32];
#pragma unroll 1
  for (int c = 0; c < 128; c += 32) {
    tmem_ld_32x32b_x32(t0 + c, r);
    tmem_ld_wait();
    float* dst = ws_row + tok_half * 128 + c;
#pragma unroll
    for (int i = 0; i < 32; i += 4)
      __stcg(reinterpret_cast<float4*>(dst + i),
             make_float4(__uint_as_float(r[i]), __uint_as_float(r[i + 1]),
                         __uint_as_float(r[i + 2]), __uint_as_float(r[i + 3])));
  }
}

__global__ void __launch_bounds__(kThreads, 1)
    tw_gemm_kernel(const __grid_constant__ CUtensorMap map_pay,
                   const __grid_constant__ CUtensorMap map_out, const GemmArgs args,
                   uint32_t idesc) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned base derived by offset so the compiler keeps the shared
  // address space (plain LDS/STS instead of generic loads)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sX = smem;                                 // [kStages][kXBytes]
  uint8_t* sP = smem + kStages * kXBytes;             // [kStages][kPBytes]
  uint8_t* sStg = smem + kStages * kStageBytes;       // [kEpilogueWarps][kStgBytes]
  uint8_t* bar_region = sStg + kEpilogueWarps * kStgBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(bar_region);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  SubTile* sub_smem = reinterpret_cast<SubTile*>(bar_region + kBarrierBytes);
  long long* trace = args.trace ? args.trace + static_cast<int64_t>(blockIdx.x) * 4096 : nullptr;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int32_t flags = args.flags;

  Tables tab{args.subtiles, args.n_sub};
  if (args.n_sub <= kMaxSmemSub) {
    for (int i = threadIdx.x; i < args.n_sub; i += kThreads) sub_smem[i] = args.subtiles[i];
    tab.sub = sub_smem;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      // payload TMA (expect_tx arrival) + one arrival per gather warp
      mbar_init(&full[s], 1 + kGatherWarps);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kEpilogueWarps);
    }
    fence_barrier_init();
    fence_proxy_async_smem();
  }
  if (warp == kPayloadWarp && lane == 0) {
    tma_prefetch_desc(&map_pay);
    if (args.use_tma_store) tma_prefetch_desc(&map_out);
  }
  if (warp == kMmaWarp) {
    tmem_alloc(tmem_slot, kTmemCols);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // Everything above (barriers, TMEM, descriptor prefetch, tables) overlaps the
  // previous kernel's tail under programmatic dependent launch; inputs and
  // outputs are only touched after the previous grid has completed.
  grid_dependency_wait();
  grid_launch_dependents();
  if (trace && threadIdx.x == 0) {
    trace[3072] = clock64();
    trace[3074] = static_cast<long long>(globaltimer_ns());
  }

  const int tn = args.tn;
  SegWalker walk;
  walk.init(args);
  Seg sg;

  if (warp == kPayloadWarp) {
    // ---------------------------------------------------- payload producer
    if (lane == 0) {
      int gs = 0;
      while (walk.next(args, tab, sg)) {
        for (int ks = sg.ks0; ks < sg.ks1; ++ks, ++gs) {
          const int stage = gs % kStages;
          mbar_wait(&empty[stage], ((gs / kStages) & 1) ^ 1u);
          mbar_arrive_expect_tx(&full[stage], kPBytes);
          tma_load_2d(sP + stage * kPBytes, &map_pay, &full[stage], ks * kBK, sg.d.pay_row);
        }
      }
    }
  } else if (warp >= kGatherWarp0 && warp < kEpilogueWarp0) {
    // ----------------------------------------------------- gather producers
    // Warp pw loads rows pw, pw + kGatherWarps, ... of every stage; lane l
    // copies tokens [8l, 8l + 8) of the row (zero-filled past M and for the
    // padding slots, index -1).  Lane i holds the index of the warp's i-th row
    // for the NEXT stage (one stage of prefetch hides the table latency).
    const int pw = warp - kGatherWarp0;
    const bool lane_on = lane * 8 < tn && !(flags & kFlagSkipA);
    const char* xa = static_cast<const char*>(args.x);
    const int my_row = pw + kGatherWarps * lane;  // row slot this lane indexes
    auto load_idx = [&](const Seg& g, int ks) -> int {
      return my_row < kBK
                 ? __ldg(args.gidx + static_cast<int64_t>(g.d.idx_row) * args.kp + ks * kBK +
                         my_row)
                 : -1;
    };
    bool have = walk.next(args, tab, sg);
    int ks = have ? sg.ks0 : 0;
    int idx_next = have ? load_idx(sg, ks) : -1;
    int gs = 0, prev_stage = -1;
    while (have) {
      const int idx_cur = idx_next;
      const int m0 = sg.mb * tn;
      // advance to the next stage and prefetch its indices
      Seg nsg = sg;
      int nks = ks + 1;
      bool nhave = true;
      if (nks >= sg.ks1) {
        nhave = walk.next(args, tab, nsg);
        nks = nhave ? nsg.ks0 : 0;
      }
      if (nhave) idx_next = load_idx(nsg, nks);
      const int stage = gs % kStages;
      mbar_wait(&empty[stage], ((gs / kStages) & 1) ^ 1u);
      const uint32_t xs = smem_u32(sX + stage * kXBytes) + (lane >> 3) * kChunkBytes;
      const int tok = m0 + lane * 8;
      const int tb = max(0, min(8, args.M - tok)) * 2;
#pragma unroll
      for (int i = 0; i < (kBK + kGatherWarps - 1) / kGatherWarps; ++i) {
        const int r = pw + i * kGatherWarps;
        const int row = __shfl_sync(0xffffffffu, idx_cur, i);
        if (r < kBK && lane_on) {
          const uint32_t bytes = row >= 0 ? static_cast<uint32_t>(tb) : 0u;
          const char* src = bytes ? xa + (static_cast<int64_t>(row) * args.ld_x + tok) * 2 : xa;
          cp_async_16(xs + r * 128 + (((lane & 7) ^ (r & 7)) << 4), src, bytes);
        }
      }
      cp_async_commit();
      if (prev_stage >= 0) {
        cp_async_wait<1>();
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[prev_stage]);
      }
      prev_stage = stage;
      ++gs;
      sg = nsg;
      ks = nks;
      have = nhave;
    }
    if (prev_stage >= 0) {
      cp_async_wait<0>();
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[prev_stage]);
    }
  } else if (warp == kMmaWarp) {
    // ---------------------------------------------------------- MMA issuer
    if (lane == 0) {
      int gs = 0;
      int j = 0;
      while (walk.next(args, tab, sg)) {
        const int acc = j & 1;
        mbar_wait(&tempty[acc], ((j >> 1) & 1) ^ 1u);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * kTileN;
        for (int ks = sg.ks0; ks < sg.ks1; ++ks, ++gs) {
          const int stage = gs % kStages;
          mbar_wait(&full[stage], (gs / kStages) & 1);
          if (trace && gs < 1024) trace[1024 + gs] = clock64();
          tc_fence_after();
          const uint32_t p0 = smem_u32(sP + stage * kPBytes);
          const uint32_t x0 = smem_u32(sX + stage * kXBytes);
          if (!(flags & kFlagSkipMma)) {
#pragma unroll
            for (int kk = 0; kk < kBK / 16; ++kk) {
              // A = payload: K-major SW128, SBO = 1 KB between 8-column groups,
              //     16 K = 32 B per MMA.
              // B = X: MN-major SW128, LBO = 8 KB between 64-token chunks,
              //     SBO = 1 KB between 8-row K groups, 16 K rows = 2 KB per MMA.
              const uint64_t adesc = umma_desc_sw128(p0 + kk * 32, 16, 1024);
              const uint64_t bdesc = umma_desc_sw128(x0 + kk * 2048, kChunkBytes, 1024);
              umma_f16(d_tmem, adesc, bdesc, idesc, (ks != sg.ks0) || (kk != 0));
            }
          }
          umma_commit(&empty[stage]);
        }
        umma_commit(&tfull[acc]);
        ++j;
      }
    }
  } else if (warp >= kEpilogueWarp0) {
    // ------------------------------------------------------------ epilogue
    // Warp w owns TMEM lanes 32*(w%4).. (output columns c of the tile) and
    // token half h of the unit.
    const int q = warp & 3;
    const int h = (warp - kEpilogueWarp0) >> 2;
    const int c = q * 32 + lane;  // output column within the 128-wide sub-tile
    const int ntok = min(128, tn - h * 128);
    const int64_t ws_slot = static_cast<int64_t>(kBN) * kTileN;
    int j = 0;
    while (walk.next(args, tab, sg)) {
      const int acc = j & 1;
      mbar_wait(&tfull[acc], (j >> 1) & 1);
      tc_fence_after();
      if (trace && warp == kEpilogueWarp0 && lane == 0 && j < 256) trace[2048 + 2 * j] = clock64();
      const uint32_t t0 =
          tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * kTileN + h * 128;
      const bool row_live = c < sg.d.width;
      const bool warp_full = q * 32 + 32 <= sg.d.width && args.rowmap == nullptr;
      const int crow = sg.d.out_row + c;
      const int orow = row_live ? (args.rowmap ? __ldg(args.rowmap + crow) : crow) : 0;
      const int tok0 = sg.mb * tn + h * 128;
      uint8_t* stg = sStg + (warp - kEpilogueWarp0) * kStgBytes;
      if (sg.kind == kSegHead) {
        // publish the head partial for the next CTA, which finishes this unit
        epilogue_partial_row(args.ws + blockIdx.x * ws_slot + static_cast<int64_t>(c) * kTileN,
                             t0, h);
        __threadfence();
        named_bar_sync(kEpiBarrier, kEpiThreads);
        if (warp == kEpilogueWarp0 && lane == 0) st_release_gpu(args.ws_flags + blockIdx.x, 1);
      } else {
        const float* add = nullptr;
        if (sg.kind == kSegTail) {
          // wait for the lower CTA's head partial of this unit
          if (warp == kEpilogueWarp0 && lane == 0)
            while (ld_acquire_gpu(args.ws_flags + blockIdx.x - 1) == 0) __nanosleep(64);
          named_bar_sync(kEpiBarrier, kEpiThreads);
          add = args.ws + (blockIdx.x - 1) * ws_slot + static_cast<int64_t>(c) * kTileN + h * 128;
        }
        epilogue_rows(args, &map_out, stg, t0, lane, orow, row_live, warp_full,
                      sg.d.out_row + q * 32, tok0, ntok, add);
        if (sg.kind == kSegTail) {
          named_bar_sync(kEpiBarrier, kEpiThreads);
          if (warp == kEpilogueWarp0 && lane == 0) args.ws_flags[blockIdx.x - 1] = 0;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (trace && warp == kEpilogueWarp0 && lane == 0 && j < 256) {
        trace[2048 + 2 * j + 1] = clock64();
        trace[3075] = static_cast<long long>(globaltimer_ns());
      }
      ++j;
    }
    if (lane == 0) bulk_wait_all<0>();  // TMA stores finished with shared memory
  }

  tc_fence_before();
  __syncthreads();
  if (trace && threadIdx.x == 0) trace[3073] = clock64();
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc(tmem_base, kTmemCols);
  }
}

}  // namespace

cudaError_t configure_gemm_kernels() {
  return cudaFuncSetAttribute(tw_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              kSmemBytes);
}

cudaError_t launch_tw_gemm(const CUtensorMap& map_pay, const CUtensorMap& map_out,
                           const GemmArgs& args, int in_dtype, int grid, cudaStream_t stream) {
  if (args.n_units <= 0) return cudaSuccess;
  if (args.tn < 64 || args.tn > kTileN || args.tn % 64 != 0) return cudaErrorInvalidValue;
  const uint32_t idesc = umma_idesc_f16(kBN, args.tn, in_dtype == kBF16 ? 1u : 0u,
                                        /*a (payload) K-major*/ 0u, /*b (X) MN-major*/ 1u);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, tw_gemm_kernel, map_pay, map_out, args, idesc);
}

}  // namespace tw
