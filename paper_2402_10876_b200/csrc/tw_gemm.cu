// K1 -- tw_gather_gemm: one persistent, warp-specialised sm_100a kernel over
// every (column tile, 128-token block) work unit of a TW layer.
//
// Replaces the reference's per-tile CPU loop (executor.py:121-177 gemm_cto /
// _tile_product / _mac_kernel and the threaded lanes of execute_batched,
// executor.py:230-265):
//   C'[:, cols_i] = A[:, kept_rows_i] . P_i        for every tile i
// computed as  C'^T tile (BN x 128 tokens) = P_i^T . A^T[kept_rows_i, tokens].
//
// Work decomposition.  A unit is (128-token block, sub-tile); its k-steps
// (64 kept rows each) are stages.  With more units than SMs the kernel runs
// stream-K: the CTA-major list of all stages is cut into gridDim.x equal
// ranges, so every SM gets the same number of MMA stages whatever the unit
// count (BERT 768x768 has 192 units for 148 SMs).  A unit cut by a range
// boundary is split in two: the lower CTA computes its head k-steps first and
// publishes an fp32 partial; the higher CTA finishes the tail k-steps last,
// adds the partial in its epilogue and stores.  CTAs walk their range
// backwards so a CTA only ever waits on a lower-numbered CTA that published
// first (no dependence on co-residency beyond in-order dispatch).
//
// Roles (1 CTA per SM):
//   warps 0..P-1  producers, kGroups stage-interleaved groups.  kGatherCpAsync
//                 (default): cp.async 16-byte chunks of the kept A^T rows into
//                 the 128-B swizzled layout; kGatherTma4: tile::gather4 (4 kept
//                 rows x 64 tokens per request).  The group's thread 0 adds the
//                 payload box with a TMA tile load.
//   warp P        TMEM allocator (2*BN columns, double-buffered accumulators) and
//                 MMA issuer: one thread issues tcgen05.mma.kind::f16
//                 (M=128 tokens, N=BN tile columns, K=16).
//   warp P+1      index warp: streams each stage's 64 gather indices into an
//                 8-slot smem ring with 1-D bulk copies, ahead of the producers.
//   warps P+4..   epilogue (4 warps): tcgen05.ld -> convert -> C'^T rows via
//                 TMA 2-D stores (condensed) or 16-byte stores (TEW row scatter,
//                 ragged chunks); stream-K partials in fp32.
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

#ifndef TW_PRODUCER_WARPS
#define TW_PRODUCER_WARPS 8
#endif
#ifndef TW_PRODUCER_GROUPS
#define TW_PRODUCER_GROUPS 2
#endif
constexpr int kProducerWarps = TW_PRODUCER_WARPS;
constexpr int kGroups = TW_PRODUCER_GROUPS;          // stage-interleaved producer groups
constexpr int kGroupWarps = kProducerWarps / kGroups;
constexpr int kGroupThreads = 32 * kGroupWarps;
constexpr int kMmaWarp = kProducerWarps;             // also allocates TMEM
constexpr int kIdxWarp = kProducerWarps + 1;         // streams gather lists into the ring
constexpr int kEpilogueWarp0 = kProducerWarps + 4;   // 4 warps, warp % 4 == TMEM quadrant
constexpr int kThreads = 32 * (kEpilogueWarp0 + 4);
constexpr int kAHalfBytes = 64 * kBK * 2;            // 64 tokens x 64 rows x 2 B = 8 KB
constexpr int kABytes = 2 * kAHalfBytes;             // 16 KB per stage
constexpr int kEpiCols = 32;                         // columns per epilogue chunk
constexpr int kEpiWarpBytes = 4096;                  // 2 x [32 cols][32 tok] 16-bit or 1 x fp32
constexpr int kEpiBytes = 4 * kEpiWarpBytes;
constexpr int kRowsPerThread = kBK * 16 / kGroupThreads;  // cp.async chunks / thread / stage
constexpr int kGatherPerWarp = 32 / kGroupWarps;          // gather4 requests / warp / stage
constexpr int kIdxSlots = 8;                         // gather-index ring (stages of lookahead)
constexpr int kIdxBytes = kIdxSlots * kBK * 4;
constexpr int kMaxSmemSub = 256;                     // sub-tile table cached in smem up to this
constexpr int kSubBytes = kMaxSmemSub * static_cast<int>(sizeof(SubTile));
constexpr int kBarrierBytes = 512;
constexpr int kEpiBarrier = 2;                       // named barrier id of the epilogue warps
static_assert(kRowsPerThread % 4 == 0, "rows per thread must allow int4 index loads");
static_assert(kGroupWarps * kGroups == kProducerWarps, "groups must split the producer warps");

template <int BN>
struct Cfg {
  static constexpr int kBBytes = BN * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStages = (BN >= 256) ? 4 : (BN >= 128 ? 6 : 8);
  static constexpr int kSmemBytes =
      kStages * kStageBytes + kBarrierBytes + kIdxBytes + kEpiBytes + kSubBytes + 1024;
  static constexpr uint32_t kTmemCols = 2 * BN;
  // Every stage slot must always be filled by the same producer group: a slot
  // shared by two groups lets one group lap its empty barrier by two phases
  // (parity ABA) and overwrite data the MMA has not consumed yet.
  static_assert(kStages % kGroups == 0, "stage slots must map to a fixed producer group");
};

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

// Epilogue of one accumulator: TMEM -> registers (+ stream-K partial) ->
// per-warp smem staging [32 cols][32 tokens] -> C'^T.  Whole 32-row chunks of a
// condensed output leave through one TMA 2-D store; ragged chunks, TEW row
// scatter and misaligned outputs use 16-byte (or scalar) stores.
template <int ESZ>
__device__ __forceinline__ void epilogue_store(const GemmArgs& args, const CUtensorMap* map_out,
                                               uint8_t* stg, uint32_t t0, const SubTile& d,
                                               int mtile, int lane, int q, const float* add,
                                               int& chunk_ctr) {
  constexpr int kRow = 32 * ESZ;           // staged bytes per output row
  constexpr int kCpr = kRow / 16;          // 16-byte chunks per row
  constexpr int kPer16 = 16 / ESZ;         // tokens per 16-byte chunk
  constexpr int kBufs = ESZ == 2 ? 2 : 1;  // staging buffers per warp
  const bool do_store = !(args.flags & kFlagSkipStore);
  const bool tma_ok = args.use_tma_store && args.rowmap == nullptr;
  uint32_t r[kEpiCols];
  tmem_ld_32x32b_x32(t0, r);
  for (int c0 = 0; c0 < d.width; c0 += kEpiCols) {
    uint8_t* buf = stg + (chunk_ctr % kBufs) * (kEpiCols * kRow);
    ++chunk_ctr;
    // the TMA store that last read this buffer must be done with it
    if (lane == 0) bulk_wait_read<kBufs - 1>();
    __syncwarp();
    tmem_ld_wait();
    float v[kEpiCols];
#pragma unroll
    for (int c = 0; c < kEpiCols; ++c) v[c] = __uint_as_float(r[c]);
    if (add) {
      const float* src = add + static_cast<int64_t>(c0) * kBM + q * 32 + lane;
#pragma unroll
      for (int c = 0; c < kEpiCols; ++c) v[c] += __ldcg(src + c * kBM);
    }
    if (c0 + kEpiCols < d.width) tmem_ld_32x32b_x32(t0 + c0 + kEpiCols, r);
    if (ESZ == 4) {
      float* st = reinterpret_cast<float*>(buf);
#pragma unroll
      for (int c = 0; c < kEpiCols; ++c) st[c * 32 + lane] = v[c];
    } else if (args.out_dtype == kF16) {
      __half* st = reinterpret_cast<__half*>(buf);
#pragma unroll
      for (int c = 0; c < kEpiCols; ++c) st[c * 32 + lane] = __float2half_rn(v[c]);
    } else {
      __nv_bfloat16* st = reinterpret_cast<__nv_bfloat16*>(buf);
#pragma unroll
      for (int c = 0; c < kEpiCols; ++c) st[c * 32 + lane] = __float2bfloat16_rn(v[c]);
    }
    const int ncols = min(kEpiCols, d.width - c0);
    if (do_store && tma_ok && ncols == kEpiCols) {
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_2d(map_out, buf, mtile, d.out_row + c0);
        bulk_commit();
      }
    } else {
      __syncwarp();
      if (do_store) {
#pragma unroll 4
        for (int id = lane; id < ncols * kCpr; id += 32) {
          const int c = id / kCpr;
          const int part = id % kCpr;
          const int crow = d.out_row + c0 + c;
          const int orow = args.rowmap ? __ldg(args.rowmap + crow) : crow;
          const int tok = mtile + part * kPer16;
          const uint8_t* src = buf + c * kRow + part * 16;
          uint8_t* dst = static_cast<uint8_t*>(args.out) +
                         (static_cast<int64_t>(orow) * args.ld_out + tok) * ESZ;
          if (args.vec_ok && tok + kPer16 <= args.M) {
            *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(src);
          } else {
            for (int e = 0; e < kPer16 && tok + e < args.M; ++e)
#pragma unroll
              for (int b = 0; b < ESZ; ++b) dst[e * ESZ + b] = src[e * ESZ + b];
          }
        }
      }
      __syncwarp();
    }
  }
}

// Stream-K head segment: raw fp32 accumulator -> workspace slot [BN][128 tok].
template <int BN>
__device__ __forceinline__ void epilogue_partial(float* ws, uint8_t* stg, uint32_t t0, int lane,
                                                 int q) {
  float* st = reinterpret_cast<float*>(stg);
  for (int c0 = 0; c0 < BN; c0 += kEpiCols) {
    uint32_t r[kEpiCols];
    tmem_ld_32x32b_x32(t0 + c0, r);
    tmem_ld_wait();
    __syncwarp();
#pragma unroll
    for (int c = 0; c < kEpiCols; ++c) st[c * 32 + lane] = __uint_as_float(r[c]);
    __syncwarp();
    // 32 rows x 128 B, 8 x 16 B per row
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int id = lane + 32 * i;
      const int c = id >> 3, part = id & 7;
      const uint4 val = *reinterpret_cast<const uint4*>(st + c * 32 + part * 4);
      __stcg(reinterpret_cast<uint4*>(ws + static_cast<int64_t>(c0 + c) * kBM + q * 32 + part * 4),
             val);
    }
  }
}

template <int BN, int MODE>
__global__ void __launch_bounds__(kThreads, 1)
    tw_gather_gemm_kernel(const __grid_constant__ CUtensorMap map_at,
                          const __grid_constant__ CUtensorMap map_pay,
                          const __grid_constant__ CUtensorMap map_out, const GemmArgs args,
                          uint32_t idesc) {
  using C = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned base derived by offset so the compiler keeps the shared
  // address space (plain LDS/STS instead of generic loads)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::kStages * kABytes;
  uint8_t* bar_region = smem + C::kStages * C::kStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(bar_region);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;
  uint64_t* tempty = tfull + 2;
  uint64_t* idx_full = tempty + 2;
  uint64_t* idx_empty = idx_full + kIdxSlots;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(idx_empty + kIdxSlots);
  int32_t* idx_ring = reinterpret_cast<int32_t*>(bar_region + kBarrierBytes);
  uint8_t* epi = bar_region + kBarrierBytes + kIdxBytes;
  SubTile* sub_smem = reinterpret_cast<SubTile*>(epi + kEpiBytes);
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
    // cp.async mode: one producer group's arrivals + 1 expect_tx arrival (payload box)
    const uint32_t full_count = MODE == kGatherCpAsync ? kGroupThreads + 1 : 1;
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], full_count);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    for (int i = 0; i < kIdxSlots; ++i) {
      mbar_init(&idx_full[i], 1);
      mbar_init(&idx_empty[i], kGroupWarps);
    }
    fence_barrier_init();
    fence_proxy_async_smem();
  }
  if (warp == 0 && lane == 0) {
    if (MODE == kGatherTma4) tma_prefetch_desc(&map_at);
    tma_prefetch_desc(&map_pay);
    if (args.use_tma_store) tma_prefetch_desc(&map_out);
  }
  if (warp == kMmaWarp) {
    tmem_alloc(tmem_slot, C::kTmemCols);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (trace && threadIdx.x == 0) trace[3072] = clock64();

  SegWalker walk;
  walk.init(args);
  Seg sg;

  if (warp < kProducerWarps) {
    // ------------------------------------------------------------ producers
    // Stage gs belongs to group gs % kGroups (kStages % kGroups == 0, so a stage
    // slot always has the same owner), so one group's fixed per-stage
    // latency (barrier waits, index load, address math, copy issue) overlaps
    // the other groups' stages.
    const int grp = warp / kGroupWarps;
    const int gwarp = warp % kGroupWarps;
    const int gtid = threadIdx.x % kGroupThreads;
    const __half* at = static_cast<const __half*>(args.at);
    // cp.async mapping: thread gtid copies token chunk j of kRowsPerThread
    // consecutive k rows starting at r0 (indices read as int4 vectors)
    const int j = gtid & 15;
    const int r0 = (gtid >> 4) * kRowsPerThread;
    int gs = 0;
    while (walk.next(args, tab, sg)) {
      const int m0 = sg.mb * kBM;
      for (int ks = sg.ks0; ks < sg.ks1; ++ks, ++gs) {
        if (gs % kGroups != grp) continue;
        const int stage = gs % C::kStages;
        const uint32_t phase = (gs / C::kStages) & 1;
        const int slot = gs % kIdxSlots;
        const int32_t* ring = idx_ring + slot * kBK;
        mbar_wait(&idx_full[slot], (gs / kIdxSlots) & 1);
        int rows[kRowsPerThread];
        int4 g4[kGatherPerWarp];
        if (MODE == kGatherCpAsync) {
#pragma unroll
          for (int v = 0; v < kRowsPerThread / 4; ++v) {
            const int4 rv = *reinterpret_cast<const int4*>(ring + r0 + 4 * v);
            rows[4 * v + 0] = rv.x;
            rows[4 * v + 1] = rv.y;
            rows[4 * v + 2] = rv.z;
            rows[4 * v + 3] = rv.w;
          }
        } else if (lane == 0) {
#pragma unroll
          for (int g = 0; g < kGatherPerWarp; ++g)
            g4[g] = *reinterpret_cast<const int4*>(ring + ((gwarp * kGatherPerWarp + g) & 15) * 4);
        }
        mbar_wait(&empty[stage], phase ^ 1u);
        if (MODE == kGatherCpAsync) {
          if (gtid == 0) {
            mbar_arrive_expect_tx(&full[stage], C::kBBytes);
            tma_load_2d(sB + stage * C::kBBytes, &map_pay, &full[stage], ks * kBK, sg.d.pay_row);
          }
          if (!(flags & kFlagSkipA)) {
            // The destination follows the 128-byte swizzle (chunk ^= row & 7)
            // that the UMMA descriptor expects.  Padding rows (== K) and tokens
            // >= M are zero-filled (src-size 0).
            const uint32_t a_base = smem_u32(sA + stage * kABytes);
            const int tok = m0 + j * 8;
            const bool tok_ok = tok < args.M;
            const __half* tok_base = at + tok;
#pragma unroll
            for (int i = 0; i < kRowsPerThread; ++i) {
              const int r = r0 + i;
              const bool ok = tok_ok && rows[i] < args.K;
              const uint32_t dst =
                  a_base + (j >> 3) * kAHalfBytes + r * 128 + (((j & 7) ^ (r & 7)) << 4);
              const __half* src = ok ? tok_base + static_cast<int64_t>(rows[i]) * args.ld_at : at;
              cp_async_16(dst, src, ok ? 16u : 0u);
            }
          }
          cp_async_mbar_arrive_noinc(&full[stage]);
        } else {
          // TMA tile::gather4: 32 requests of (4 kept rows x 64 tokens) per
          // stage, issued by lane 0 of each warp of the owning group.  Padding
          // rows (== K) are out of bounds and zero-filled by the TMA unit.
          const uint32_t bytes = (flags & kFlagSkipA) ? C::kBBytes : C::kStageBytes;
          if (gtid == 0) {
            mbar_arrive_expect_tx(&full[stage], bytes);
            tma_load_2d(sB + stage * C::kBBytes, &map_pay, &full[stage], ks * kBK, sg.d.pay_row);
          }
          if (lane == 0 && !(flags & kFlagSkipA)) {
#pragma unroll
            for (int g = 0; g < kGatherPerWarp; ++g) {
              const int q4 = gwarp * kGatherPerWarp + g;  // 0..31
              const int half = q4 >> 4;                   // 64-token half
              const int r4 = (q4 & 15) * 4;               // first of 4 k rows
              uint8_t* dst = sA + stage * kABytes + half * kAHalfBytes + r4 * 128;
              tma_gather4(dst, &map_at, &full[stage], m0 + half * 64, g4[g].x, g4[g].y, g4[g].z,
                          g4[g].w);
            }
          }
        }
        // the indices are consumed (the copies above used them): free the slot
        __syncwarp();
        if (lane == 0) mbar_arrive(&idx_empty[slot]);
      }
    }
  } else if (warp == kIdxWarp) {
    // ---------------------------------------------------------- index warp
    if (lane == 0) {
      int gs = 0;
      while (walk.next(args, tab, sg)) {
        const int32_t* src = args.rowidx + static_cast<int64_t>(sg.d.idx_row) * args.Kp;
        for (int ks = sg.ks0; ks < sg.ks1; ++ks, ++gs) {
          const int slot = gs % kIdxSlots;
          mbar_wait(&idx_empty[slot], ((gs / kIdxSlots) & 1) ^ 1u);
          mbar_arrive_expect_tx(&idx_full[slot], kBK * 4);
          bulk_load(idx_ring + slot * kBK, src + ks * kBK, kBK * 4, &idx_full[slot]);
        }
      }
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
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int ks = sg.ks0; ks < sg.ks1; ++ks, ++gs) {
          const int stage = gs % C::kStages;
          mbar_wait(&full[stage], (gs / C::kStages) & 1);
          tc_fence_after();
          if (MODE == kGatherCpAsync) fence_proxy_async_smem();  // generic -> async proxy
          const uint32_t a0 = smem_u32(sA + stage * kABytes);
          const uint32_t b0 = smem_u32(sB + stage * C::kBBytes);
          if (!(flags & kFlagSkipMma)) {
#pragma unroll
            for (int kk = 0; kk < kBK / 16; ++kk) {
              // A: MN-major SW128, LBO = 8 KB between 64-token halves, SBO = 1 KB
              //    between 8-row K groups; 16 K rows = 2 KB per MMA.
              // B: K-major SW128, SBO = 1 KB between 8-column groups; 16 K = 32 B.
              const uint64_t adesc = umma_desc_sw128(a0 + kk * 2048, kAHalfBytes, 1024);
              const uint64_t bdesc = umma_desc_sw128(b0 + kk * 32, 16, 1024);
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
    // Warp q owns TMEM lanes (= tokens) [32q, 32q+32).
    const int q = warp & 3;
    uint8_t* stg = epi + q * kEpiWarpBytes;
    const int64_t ws_slot = static_cast<int64_t>(BN) * kBM;
    int j = 0;
    int chunk_ctr = 0;
    while (walk.next(args, tab, sg)) {
      const int acc = j & 1;
      mbar_wait(&tfull[acc], (j >> 1) & 1);
      tc_fence_after();
      if (trace && q == 0 && lane == 0 && j < 256) trace[2048 + 2 * j] = clock64();
      const int mtile = sg.mb * kBM + q * 32;
      const uint32_t t0 = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN;
      if (sg.kind == kSegHead) {
        // publish the head partial for the next CTA, which finishes this unit
        epilogue_partial<BN>(args.ws + blockIdx.x * ws_slot, stg, t0, lane, q);
        __threadfence();
        named_bar_sync(kEpiBarrier, 128);
        if (q == 0 && lane == 0) st_release_gpu(args.ws_flags + blockIdx.x, 1);
      } else {
        const float* add = nullptr;
        if (sg.kind == kSegTail) {
          // wait for the lower CTA's head partial of this unit
          if (q == 0 && lane == 0)
            while (ld_acquire_gpu(args.ws_flags + blockIdx.x - 1) == 0) __nanosleep(64);
          named_bar_sync(kEpiBarrier, 128);
          add = args.ws + (blockIdx.x - 1) * ws_slot;
        }
        if (args.out_dtype == kF32)
          epilogue_store<4>(args, &map_out, stg, t0, sg.d, mtile, lane, q, add, chunk_ctr);
        else
          epilogue_store<2>(args, &map_out, stg, t0, sg.d, mtile, lane, q, add, chunk_ctr);
        if (sg.kind == kSegTail) {
          named_bar_sync(kEpiBarrier, 128);
          if (q == 0 && lane == 0) args.ws_flags[blockIdx.x - 1] = 0;  // re-arm for the next launch
        }
      }
      tc_fence_before();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (trace && q == 0 && lane == 0 && j < 256) trace[2048 + 2 * j + 1] = clock64();
      ++j;
    }
    if (lane == 0) bulk_wait_all<0>();  // TMA stores finished with shared memory
  }

  tc_fence_before();
  __syncthreads();
  if (trace && threadIdx.x == 0) trace[3073] = clock64();
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::kTmemCols);
  }
}

template <int BN, int MODE>
cudaError_t launch_bn(const CUtensorMap& map_at, const CUtensorMap& map_pay,
                      const CUtensorMap& map_out, const GemmArgs& args, int in_dtype, int grid,
                      cudaStream_t stream) {
  using C = Cfg<BN>;
  const uint32_t idesc =
      umma_idesc_f16(kBM, BN, in_dtype == kBF16 ? 1u : 0u, /*a MN-major*/ 1u, /*b K-major*/ 0u);
  tw_gather_gemm_kernel<BN, MODE><<<grid, kThreads, C::kSmemBytes, stream>>>(
      map_at, map_pay, map_out, args, idesc);
  return cudaGetLastError();
}

template <int BN>
cudaError_t configure_bn() {
  cudaError_t e = cudaFuncSetAttribute(tw_gather_gemm_kernel<BN, kGatherTma4>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       Cfg<BN>::kSmemBytes);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(tw_gather_gemm_kernel<BN, kGatherCpAsync>,
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
                                  const CUtensorMap& map_out, const GemmArgs& args_in,
                                  const void* at, int64_t ld_at, int bn, int in_dtype,
                                  int gather_mode, int grid, cudaStream_t stream) {
  if (args_in.n_units <= 0) return cudaSuccess;
  GemmArgs args = args_in;
  args.at = at;
  args.ld_at = ld_at;
  const bool cp = gather_mode == kGatherCpAsync;
#define TW_LAUNCH(BNV)                                                                     \
  return cp ? launch_bn<BNV, kGatherCpAsync>(map_at, map_pay, map_out, args, in_dtype, grid, \
                                             stream)                                        \
            : launch_bn<BNV, kGatherTma4>(map_at, map_pay, map_out, args, in_dtype, grid, stream)
  switch (bn) {
    case 32: TW_LAUNCH(32);
    case 64: TW_LAUNCH(64);
    case 128: TW_LAUNCH(128);
    case 256: TW_LAUNCH(256);
    default: return cudaErrorInvalidValue;
  }
#undef TW_LAUNCH
}

}  // namespace tw
