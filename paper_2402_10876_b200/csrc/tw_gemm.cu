// K1 -- tw_gemm_kernel: one persistent, warp-specialised sm_100a kernel over
// every (column sub-tile, token range) of a TW layer.
//
// Replaces the reference's per-tile CPU loop (executor.py:121-177 gemm_cto /
// _tile_product / _mac_kernel and the threaded lanes of execute_batched,
// executor.py:230-265):
//   C'[:, cols_i] = A[:, kept_rows_i] . P_i        for every tile i
// computed transposed, one UMMA tile per unit:
//   C'^T[cols_i, tokens] (128 x n) = P_i^T (128 x K') . A^T[kept_rows_i, tokens] (K' x n)
// with the payload P_i^T as the K-major A operand (the CTO transposed payload
// layout of formats.py:200, zero-padded to whole 64-row k-steps) and the
// gathered A^T rows as the MN-major B operand.  TMEM lanes are output columns
// and TMEM columns are tokens, so an epilogue thread holds a contiguous segment
// of one C'^T row.
//
// Work decomposition (the reference's LPT lanes, executor.py:206-227, become
// a static balanced split).  When the layer has no more 128-column sub-tiles
// than SMs ("owner" mode), every CTA owns ONE sub-tile and a contiguous token
// range: sub-tile s gets c_s CTAs with c_s proportional to its k-steps
// (host-side largest-remainder split, tw_capi.cu), and its tokens are cut into
// c_s ranges on 16-token boundaries.  A range is processed in units of <= 256
// tokens (UMMA N = the unit's tokens rounded up to 16).  When the sub-tile's
// payload fits in shared memory (<= kResSteps k-steps, e.g. every K = 768
// BERT layer) it is loaded ONCE per CTA ("resident" kernel) -- before the
// programmatic-dependent-launch wait, since it does not depend on the
// previous kernel -- and only the activations stream; otherwise each stage
// carries its payload slice ("streamed" kernel).  Layers with more sub-tiles
// than SMs fall back to 256-token units strided over the CTAs (streamed).
//
// Per-SM ingress (L2 -> SMEM) of gathered rows is the bound of this kernel
// (scripts/microbench_gather2.cu: ~30-38 B/cycle/SM for scattered rows vs
// ~58 for aligned TMA boxes), so the design minimises bytes per SM: payload
// residency removes the payload re-reads, and the balanced split keeps the
// busiest SM close to the mean.
//
// Roles (1 CTA per SM, 896 threads; 16 gather warps measured ~7% faster than
// 12 and equal to 20):
//   warp 0      payload producer (TMA 2-D boxes of 128 cols x 64 k, SW128).
//   warp 1      TMEM allocator (2 x 256 columns: double-buffered accumulators)
//               and MMA issuer: one thread, tcgen05.mma.kind::f16 M=128 N=n K=16.
//   warps 4-19  gather producers: each stage is 64 kept A^T rows x n tokens as
//               16-byte cp.async into the 128-B swizzled MN-major layout; row
//               indices are prefetched one stage ahead in registers; every
//               thread's copies arrive on the stage barrier asynchronously
//               (cp.async.mbarrier.arrive.noinc).  A^T is read where it lies.
//   warps 20-27 epilogue: warp w owns TMEM lanes 32*(w%4).. (output columns)
//               and one 128-token half; tcgen05.ld -> fp16/bf16 -> swizzled
//               smem -> TMA 2-D store per 32 x 32 block (16-byte stores for the
//               TEW row scatter, ragged sub-tiles, partial blocks, fp32 out).
#include "sm100_ptx.cuh"
#include "tw_kernels.cuh"

#include <cuda_bf16.h>
#include <cuda_fp16.h>

namespace tw {

namespace {

constexpr int kPayloadWarp = 0;
constexpr int kMmaWarp = 1;
constexpr int kGatherWarp0 = 4;
constexpr int kGatherWarps = 16;
constexpr int kGatherThreads = 32 * kGatherWarps;
constexpr int kEpilogueWarp0 = kGatherWarp0 + kGatherWarps;
constexpr int kEpilogueWarps = 8;
constexpr int kThreads = 32 * (kEpilogueWarp0 + kEpilogueWarps);
constexpr int kTileN = kTN;                          // max tokens per unit (UMMA N)
constexpr int kChunkBytes = 64 * kBK * 2;            // 64 tokens x 64 rows x 2 B = 8 KB
constexpr int kXBytes = (kTileN / 64) * kChunkBytes; // 32 KB per stage
constexpr int kPBytes = kBN * kBK * 2;               // 16 KB per k-step of payload
constexpr int kMaxSmemSub = 32;                      // strided mode: sub-tile table in smem
constexpr int kStgBytes = 2048;                      // per epilogue warp: 2 x [32 rows][32 B]
constexpr uint32_t kTmemCols = 2 * kTileN;           // double-buffered 128 x 256 fp32
constexpr int kMaxItems = (kBK * kTileN / 8 + kGatherThreads - 1) / kGatherThreads;
static_assert(kEpilogueWarp0 % 4 == 0, "epilogue warps must start a warpgroup (TMEM lane quadrants)");

template <bool kRes>
struct Cfg {
  static constexpr int kStages = kRes ? 3 : 4;
  static constexpr int kStageBytes = kXBytes + (kRes ? 0 : kPBytes);
  static constexpr int kPayloadRegion = kRes ? kResSteps * kPBytes : 0;
  static constexpr int kBarrierBytes = 256;
  static constexpr int kSubBytes = kRes ? 0 : kMaxSmemSub * static_cast<int>(sizeof(SubTile));
  // owner mode: the owned sub-tile's whole gather list, staged once
  static constexpr int kIdxCap = kRes ? kResSteps * kBK : 64 * kBK;
  static constexpr int kIdxBytes = kIdxCap * 4;
  static constexpr int kSmemBytes = kStages * kStageBytes + kPayloadRegion +
                                    kEpilogueWarps * kStgBytes + kBarrierBytes + kSubBytes +
                                    kIdxBytes + 1024;
  static_assert(kSmemBytes <= 227 * 1024, "shared memory budget");
  static_assert(2 * kStages + kResSteps + 4 + 3 <= kBarrierBytes / 8, "barrier region");
};

// One unit of work: sub-tile d over tokens [ub, ue).
struct Seg {
  int sub, ub, ue;
  SubTile d;
};

// Deterministic per-CTA unit sequence, identical in every role.
struct Walker {
  // owner mode: this CTA's sub-tile and token range (host work table)
  int b, e, nu, i, usz;
  SubTile d;
  // strided mode
  int u;
  const SubTile* tab;

  int ncta;  // CTAs of this launch (strided mode stride)

  __device__ __forceinline__ void init(const GemmArgs& a, const CtaWork* mine, int cta, int nctas,
                                       const SubTile* table) {
    tab = table;
    i = 0;
    ncta = nctas;
    if (a.owner) {
      const CtaWork& w = *mine;
      d.kp_steps = w.kp_steps;
      d.k0 = w.k0;
      d.idx_row = w.idx_row;
      d.pay_row = w.pay_row;
      d.width = w.width;
      d.out_row = w.out_row;
      b = w.b;
      e = w.e;
      usz = w.usz;
      nu = usz > 0 ? (e - b + usz - 1) / usz : 0;
    } else {
      u = cta;
    }
  }
  __device__ __forceinline__ bool next(const GemmArgs& a, Seg& g) {
    if (a.owner) {
      if (i >= nu) return false;
      g.sub = 0;
      g.ub = b + i * usz;
      g.ue = min(e, g.ub + usz);
      g.d = d;
      ++i;
      return true;
    }
    if (u >= a.n_units) return false;
    // units in sub-tile groups of a.sub_group (host: the group's payloads
    // plus the token blocks one wave touches fit in L2), token-block-major
    // inside a group; one group = the whole layer when sub_group >= n_sub
    const int n_mb = (a.M + kTileN - 1) / kTileN;
    const int sg = a.sub_group;
    const int grp = u / (n_mb * sg);
    const int local = u - grp * n_mb * sg;
    const int sz = min(sg, a.n_sub - grp * sg);
    const int mb = local / sz;
    g.sub = grp * sg + (local - mb * sz);
    g.ub = mb * kTileN;
    g.ue = min(a.M, g.ub + kTileN);
    g.d = tab[g.sub];
    u += ncta;
    return true;
  }
};

__device__ __forceinline__ uint32_t pack2(float a, float b, int32_t dtype) {
  if (dtype == kF16) {
    const __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&h);
  }
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

// Keeps the compiler from hoisting reads of tcgen05.ld destinations above
// the tcgen05.wait::ld that completes them.
__device__ __forceinline__ void reg_fence(uint32_t (&w)[16]) {
#pragma unroll
  for (int i = 0; i < 16; ++i) asm volatile("" : "+r"(w[i]));
}

// Epilogue of one accumulator quarter: the warp's 32 output rows (columns
// q*32.. of the sub-tile) x tokens [tok0, tok0 + ntok), in pieces of 16
// tokens; tokens >= lim belong to another CTA (or are past M) and are never
// written.  The next piece's tcgen05.ld is issued as soon as the current one
// is packed, so TMEM latency overlaps the stores.  16-bit condensed output
// leaves through TMA 2-D stores of [32 rows][16 tokens] from two 1 KB staging
// buffers used alternately (sbuf), so filling one overlaps the bulk read of
// the other; otherwise 16-byte / scalar stores of each thread's row segment.
__device__ __forceinline__ void epilogue_rows(const GemmArgs& args, const CUtensorMap* map_out,
                                              uint8_t* stg, int& sbuf, bool dbl, uint32_t t0,
                                              int lane, int orow, bool row_live, bool warp_full,
                                              int row0_tma, int tok0, int ntok, int lim) {
  const bool do_store = !(args.flags & kFlagSkipStore);
  const int esz = args.out_dtype == kF32 ? 4 : 2;
  uint8_t* row_base =
      static_cast<uint8_t*>(args.out) + static_cast<int64_t>(orow) * args.ld_out * esz;
  if (ntok <= 0) return;
  uint32_t w[16];
  tmem_ld_32x32b_x16(t0, w);
#pragma unroll 1
  for (int c = 0; c < ntok; c += 16) {
    tmem_ld_wait();
    reg_fence(w);
    const bool more = c + 16 < ntok;
    const int tok = tok0 + c;
    const bool live = do_store && tok < lim;
    const bool whole = tok + 16 <= lim;
    if (esz == 4) {
      if (live && row_live) {
        float* dst = reinterpret_cast<float*>(row_base) + tok;
        if (args.vec_ok && whole) {
#pragma unroll
          for (int i = 0; i < 16; i += 4)
            *reinterpret_cast<uint4*>(dst + i) = make_uint4(w[i], w[i + 1], w[i + 2], w[i + 3]);
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (tok + i < lim) dst[i] = __uint_as_float(w[i]);
        }
      }
      if (more) tmem_ld_32x32b_x16(t0 + c + 16, w);
      continue;
    }
    // packed row segment: 8 words (element pairs)
    uint32_t pk[8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
      pk[i] = pack2(__uint_as_float(w[2 * i]), __uint_as_float(w[2 * i + 1]), args.out_dtype);
    if (more) tmem_ld_32x32b_x16(t0 + c + 16, w);
    if (!live) continue;
    if (args.use_tma_store && warp_full && whole) {
      // the store that last read this buffer (two stores ago; the previous
      // one with a single buffer) must be done
      if (lane == 0) {
        if (dbl) bulk_wait_read<1>(); else bulk_wait_read<0>();
      }
      __syncwarp();
      uint8_t* buf = stg + sbuf * 1024;
      // row `lane` = 32 bytes, 16-byte halves XOR-swizzled (SWIZZLE_32B)
#pragma unroll
      for (int j = 0; j < 2; ++j)
        *reinterpret_cast<uint4*>(buf + lane * 32 + ((j ^ ((lane >> 2) & 1)) << 4)) =
            make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_2d(map_out, buf, tok, row0_tma);
        bulk_commit();
      }
      if (dbl) sbuf ^= 1;
      continue;
    }
    if (!row_live) continue;
    uint16_t* dst = reinterpret_cast<uint16_t*>(row_base) + tok;
    if (args.vec_ok && whole) {
#pragma unroll
      for (int i = 0; i < 8; i += 4)
        *reinterpret_cast<uint4*>(dst + 2 * i) = make_uint4(pk[i], pk[i + 1], pk[i + 2], pk[i + 3]);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (tok + 2 * i < lim) dst[2 * i] = static_cast<uint16_t>(pk[i] & 0xFFFFu);
        if (tok + 2 * i + 1 < lim) dst[2 * i + 1] = static_cast<uint16_t>(pk[i] >> 16);
      }
    }
  }
}

// One unit's epilogue for one warp: TMEM quadrant q (output columns
// q*32..), token part `part` of `nparts` (multiples of 16 tokens).
__device__ __forceinline__ void epilogue_unit(const GemmArgs& args, const CUtensorMap* map_out,
                                              const Seg& sg, uint32_t tmem_base, int acc,
                                              int tile_n, int q, int lane, int part, int nparts,
                                              uint8_t* stg, int& sbuf, bool dbl) {
  const int n = (sg.ue - sg.ub + 15) & ~15;
  const int per = ((n + nparts - 1) / nparts + 15) & ~15;  // tokens per part
  const int tlo = part * per;
  const int ntok = min(per, n - tlo);
  if (ntok <= 0) return;
  const int c = q * 32 + lane;  // output column within the 128-wide sub-tile
  const uint32_t t0 = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * tile_n + tlo;
  const bool row_live = c < sg.d.width;
  const bool warp_full = q * 32 + 32 <= sg.d.width && args.rowmap == nullptr;
  const int crow = sg.d.out_row + c;
  const int orow = row_live ? (args.rowmap ? __ldg(args.rowmap + crow) : crow) : 0;
  epilogue_rows(args, map_out, stg, sbuf, dbl, t0, lane, orow, row_live, warp_full,
                sg.d.out_row + q * 32, sg.ub + tlo, ntok, sg.ue);
}

// The kernel body for one CTA of one layer: CTA `cta` of `ncta`, its
// owner-mode work entry at `work` (this CTA's own).  Called by tw_gemm_kernel (one layer per
// launch) and tw_gemm_group_kernel (several independent layers in one
// launch); the tensor maps and args live in kernel parameter space.
template <bool kRes, bool kPair>
__device__ __forceinline__ void gemm_body(const CUtensorMap& map_pay, const CUtensorMap& map_out,
                                          const RunMaps& run_maps, const GemmArgs& args,
                                          const CtaWork* work, const int cta, const int ncta,
                                          const int tslot) {
  using C = Cfg<kRes>;
  constexpr int kStages = C::kStages;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned base derived by offset so the compiler keeps the shared
  // address space (plain LDS/STS instead of generic loads)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  // paired units (kPair: streamed run path, args.pair set by the host): 2
  // ring slots of [2 units][kXBytes] A^T + the payload
  constexpr bool pair = !kRes && kPair;
  constexpr int nst = pair ? 2 : kStages;                // ring slots in use
  constexpr int xstride = pair ? 2 * kXBytes : kXBytes;  // A^T bytes per slot
  static_assert(kRes || 2 * (2 * kXBytes + kPBytes) <= kStages * (kXBytes + kPBytes),
                "paired ring fits the streamed ring");
  uint8_t* sX = smem;                                    // [nst][xstride]
  uint8_t* sP = smem + nst * xstride;                    // streamed: [nst][kPBytes]
                                                         // resident: [kResSteps][kPBytes]
  uint8_t* sStg = smem + kStages * C::kStageBytes + C::kPayloadRegion;
  uint8_t* bar_region = sStg + kEpilogueWarps * kStgBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(bar_region);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint64_t* pfull = tempty + 2;  // resident payload, one barrier per k-step
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pfull + kResSteps);
  // completes once per kernel, when the last unit's accumulator is full: the
  // gather warps then join that unit's epilogue (a parity wait on tfull could
  // alias an earlier phase)
  uint64_t* jbar = pfull + kResSteps + 1;
  // sparse plans: the four metadata writers (one per TMEM lane quadrant) are done
  uint64_t* mfull = jbar + 1;
  SubTile* sub_smem = reinterpret_cast<SubTile*>(bar_region + C::kBarrierBytes);
  int32_t* sIdx = reinterpret_cast<int32_t*>(bar_region + C::kBarrierBytes + C::kSubBytes);
  long long* trace = args.trace ? args.trace + static_cast<int64_t>(tslot) * 4096 : nullptr;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int32_t flags = args.flags;
  // Run path, streamed kernel: the gather warps have nothing to gather, so
  // they join the epilogue (24 warps instead of 8, the extra 16 staging in
  // the unused gather-list region) -- the epilogue is a fixed ~4K-cycle cost
  // per unit that a CTA with one or two units cannot hide.
  const bool wide_epi = !kRes && args.runs;
  constexpr int kWideEpi = kEpilogueWarps + kGatherWarps;

  // Everything up to the role split reads only plan constants (tables, gather
  // lists, payload), so it overlaps the previous kernel's tail under
  // programmatic dependent launch; activations are read and outputs written
  // only after grid_dependency_wait() in the gather and epilogue roles.
  // sparse plans: the metadata writers (epilogue warps 0-3, one per TMEM
  // lane quadrant) load the owned sub-tile's metadata now, so the loads
  // overlap the prologue (and, under PDL, the previous kernel's tail)
  uint32_t meta_v[32];
  const bool meta_writer = args.sparse && !(args.flags & kFlagSkipMeta) && warp >= kEpilogueWarp0 &&
                           warp < kEpilogueWarp0 + 4;
  if (meta_writer) {
    const CtaWork& w = *work;
    const int n = w.usz > 0 ? 2 * w.kp_steps : 0;
    const uint32_t* mp = args.meta + static_cast<int64_t>(w.pay_row / kBN) * args.meta_cols * 128 +
                         (warp & 3) * 32 + lane;
#pragma unroll
    for (int i = 0; i < 32; ++i) meta_v[i] = i < n ? __ldg(mp + i * 128) : 0u;
  }
  const SubTile* tab = args.subtiles;
  if (!kRes && !args.owner && args.n_sub <= kMaxSmemSub) {
    for (int i = threadIdx.x; i < args.n_sub; i += kThreads) sub_smem[i] = args.subtiles[i];
    tab = sub_smem;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      // streamed: payload TMA (expect_tx arrival); both: one cp.async
      // arrival per gather thread
      // streamed: payload TMA (expect_tx arrival); cp.async path: one
      // arrival per gather thread; run path: the box issuer's one arrival
      mbar_init(&full[s], args.runs ? 1 : (kRes ? 0 : 1) + kGatherThreads);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], wide_epi ? kWideEpi : kEpilogueWarps);
    }
    for (int k = 0; k < kResSteps; ++k) mbar_init(&pfull[k], 1);
    mbar_init(jbar, 1);
    mbar_init(mfull, 4);
    fence_barrier_init();
    fence_proxy_async_smem();
  }
  if (warp == kPayloadWarp && lane == 0) {
    tma_prefetch_desc(&map_pay);
    if (args.use_tma_store) tma_prefetch_desc(&map_out);
  }
  if (args.runs && warp == kPayloadWarp && lane < kRunMaps) tma_prefetch_desc(&run_maps.m[lane]);
  if (warp == kMmaWarp) {
    tmem_alloc(tmem_slot, kTmemCols);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  grid_launch_dependents();
  if (trace && threadIdx.x == 0) {
    trace[3072] = clock64();
    trace[3074] = static_cast<long long>(globaltimer_ns());
  }

  Walker walk;
  walk.init(args, work, cta, ncta, tab);
  Seg sg;

  if (warp == kPayloadWarp) {
    // ---------------------------------------------------- payload producer
    if (kRes && lane == 0) {
      // the owned sub-tile's whole payload, once, paced with the first
      // unit's activation stages (k-step ks is requested when stage ks may
      // be filled) so the first stages are not queued behind all of it; on
      // the run path this warp also fills the stages, so no pacing
      Walker w0 = walk;
      Seg s0;
      if (w0.next(args, s0)) {
        const bool skip_p = flags & kFlagSkipP;
        // sparse payload: one 64-column box holds 2 stages (128 K' rows, 2:4)
        const int nbox = args.sparse ? (s0.d.kp_steps + 1) / 2 : s0.d.kp_steps;
        for (int ks = 0; ks < nbox; ++ks) {
          if (!args.runs) mbar_wait(&empty[ks % kStages], ((ks / kStages) & 1) ^ 1u);
          if (skip_p) {
            mbar_arrive(&pfull[ks]);
            continue;
          }
          mbar_arrive_expect_tx(&pfull[ks], kPBytes);
          tma_load_2d(sP + ks * kPBytes, &map_pay, &pfull[ks], (s0.d.k0 + ks) * kBK, s0.d.pay_row);
        }
      }
    }
    if (args.runs) {
      // Run path: each stage is a few dense TMA boxes of consecutive A^T
      // rows (plan row layout) x 64 tokens, one box per lane; lane 0 also
      // streams the payload slice (streamed kernel).
      grid_dependency_wait();  // A^T may be written by the previous kernel
      int gs = 0;
      while (walk.next(args, sg)) {
        const int n = (sg.ue - sg.ub + 15) & ~15;
        const int chunks = (n + 63) >> 6;
        // paired units: the next unit (same sub-tile, same stages) rides along
        int ub2 = 0, chunks2 = 0;
        if (pair) {
          Walker w2 = walk;
          Seg s2;
          if (w2.next(args, s2)) {
            walk = w2;
            ub2 = s2.ub;
            chunks2 = (((s2.ue - s2.ub + 15) & ~15) + 63) >> 6;
          }
        }
        const int32_t* bf =
            args.box_first + static_cast<int64_t>(sg.d.idx_row) * args.box_stride + sg.d.k0;
        int b0 = __ldg(bf), b1 = __ldg(bf + 1);
        for (int ks = 0; ks < sg.d.kp_steps; ++ks, ++gs) {
          const int stage = gs % nst;
          const int nb0 = ks + 1 < sg.d.kp_steps ? __ldg(bf + ks + 1) : 0;
          const int nb1 = ks + 1 < sg.d.kp_steps ? __ldg(bf + ks + 2) : 0;
          const uint32_t e = b0 + lane < b1 ? __ldg(args.boxes + b0 + lane) : 0u;
          mbar_wait(&empty[stage], ((gs / nst) & 1) ^ 1u);
          if (trace && lane == 0 && gs < 1024) {
            trace[gs] = clock64();
            trace[3076] += b1 - b0;
          }
          const bool skip_p = kRes || (flags & kFlagSkipP);
          const bool skip_a = flags & kFlagSkipA;
          if (lane == 0) {
            mbar_arrive_expect_tx(&full[stage],
                                  (skip_p ? 0u : static_cast<uint32_t>(kPBytes)) +
                                      (skip_a ? 0u : static_cast<uint32_t>((chunks + chunks2) * kBK * 128)));
            if (!skip_p)
              tma_load_2d(sP + stage * kPBytes, &map_pay, &full[stage], (sg.d.k0 + ks) * kBK,
                          sg.d.pay_row);
          }
          __syncwarp();
          for (int j = b0 + lane, jj = 0; j < b1 && !skip_a; j += 32, jj += 32) {
            const uint32_t ej = jj == 0 ? e : __ldg(args.boxes + j);
            const int slot = static_cast<int>(ej & 63u), code = static_cast<int>((ej >> 6) & 7u);
            const int32_t pos = static_cast<int32_t>(ej >> 9);
            uint8_t* dst = sX + stage * xstride + slot * 128;
            for (int c = 0; c < chunks; ++c)
              tma_load_2d(dst + c * kChunkBytes, &run_maps.m[code], &full[stage], sg.ub + c * 64, pos);
            for (int c = 0; c < chunks2; ++c)
              tma_load_2d(dst + kXBytes + c * kChunkBytes, &run_maps.m[code], &full[stage],
                          ub2 + c * 64, pos);
          }
          b0 = nb0;
          b1 = nb1;
        }
      }
    } else if (!kRes && lane == 0) {
      int gs = 0;
      while (walk.next(args, sg)) {
        for (int ks = 0; ks < sg.d.kp_steps; ++ks, ++gs) {
          const int stage = gs % kStages;
          mbar_wait(&empty[stage], ((gs / kStages) & 1) ^ 1u);
          if (trace && gs < 1024) trace[gs] = clock64();
          if (flags & kFlagSkipP) {
            mbar_arrive(&full[stage]);
            continue;
          }
          if (args.sparse == 1) {  // the stage's 32 compressed columns (2:4), 64-B swizzle
            mbar_arrive_expect_tx(&full[stage], kPBytes / 2);
            tma_load_2d(sP + stage * kPBytes, &map_pay, &full[stage], ks * (kBK / 2), sg.d.pay_row);
          } else if (args.sparse == 2) {  // the 64-column SW128 box holding this stage's half
            mbar_arrive_expect_tx(&full[stage], kPBytes);
            tma_load_2d(sP + stage * kPBytes, &map_pay, &full[stage], (ks >> 1) * kBK, sg.d.pay_row);
          } else {
            mbar_arrive_expect_tx(&full[stage], kPBytes);
            tma_load_2d(sP + stage * kPBytes, &map_pay, &full[stage], (sg.d.k0 + ks) * kBK,
                        sg.d.pay_row);
          }
        }
      }
    }
  } else if (warp >= kGatherWarp0 && warp < kEpilogueWarp0 && !args.runs) {
    // ----------------------------------------------------- gather producers
    // A stage is kBK kept rows x n tokens = kBK * n / 8 16-byte items; item i
    // is row i / cpr, 16-byte chunk i % cpr (cpr = n / 8), so every lane is
    // busy for any n.  Thread t copies items t, t + kGatherThreads, ...;
    // kept-row indices of the next stage are prefetched in registers.  Copies
    // are zero-filled past M and for padding slots (index -1).  Each thread's
    // cp.async completion arrives on full[stage] asynchronously (noinc), so
    // every stage can be in flight at once without blocking the warp (a
    // per-warp arrival after cp.async.wait_group measured 20% slower); the MMA
    // thread fences the generic -> async proxy after its wait.
    const int gt = threadIdx.x - 32 * kGatherWarp0;
    const bool skip_a = flags & kFlagSkipA;
    const char* xa = static_cast<const char*>(args.x);
    int slot_row[kMaxItems], slot_chunk[kMaxItems];
    uint32_t slot_dst[kMaxItems];
    int cpr = -1;
    auto layout = [&](int n) {  // item -> (row, chunk, smem offset) for n tokens
      if ((n >> 3) == cpr) return;
      cpr = n >> 3;
#pragma unroll
      for (int i = 0; i < kMaxItems; ++i) {
        const int it = gt + i * kGatherThreads;
        const int r = it / cpr, c = it - r * cpr;
        slot_row[i] = it < kBK * cpr ? r : -1;
        slot_chunk[i] = c;
        slot_dst[i] = (c >> 3) * kChunkBytes + r * 128 + (((c & 7) ^ (r & 7)) << 4);
      }
    };
    auto unit_n = [](const Seg& g) { return (g.ue - g.ub + 15) & ~15; };
    // Gather lists live in shared memory, so a stage's row indices are a
    // shared load away (indices prefetched from global only one stage ahead
    // let their L2 latency pace the whole gather).  Owner mode with a list
    // that fits: the owned sub-tile's whole list, staged once (plan
    // constants: before the dependency wait).  Otherwise chunks of kChunkSt
    // stages in two alternating buffers, refilled at chunk boundaries; every
    // gather thread walks the same units and stages, so the named barriers
    // line up.
    constexpr int kChunkSt = C::kIdxCap / (2 * kBK);
    bool have = walk.next(args, sg);
    const bool whole = args.owner && have && sg.d.kp_steps * kBK <= C::kIdxCap;
    auto stage_chunk = [&](const Seg& g, int c) {  // stages [c * kChunkSt, ...) -> buffer c & 1
      const int first = c * kChunkSt * kBK;
      const int n = min(kChunkSt, g.d.kp_steps - c * kChunkSt) * kBK;
      const int32_t* src = args.gidx + static_cast<int64_t>(g.d.idx_row) * args.kp + g.d.k0 * kBK + first;
      int32_t* dst = sIdx + (c & 1) * kChunkSt * kBK;
      for (int i = gt; i < n; i += kGatherThreads) dst[i] = __ldg(src + i);
    };
    auto begin_unit = [&](const Seg& g) {
      if (whole) return;
      named_bar_sync(1, kGatherThreads);  // everyone is done with the old lists
      stage_chunk(g, 0);
      if (g.d.kp_steps > kChunkSt) stage_chunk(g, 1);
      named_bar_sync(1, kGatherThreads);
    };
    if (whole) {
      const int32_t* src = args.gidx + static_cast<int64_t>(sg.d.idx_row) * args.kp + sg.d.k0 * kBK;
      for (int i = gt; i < sg.d.kp_steps * kBK; i += kGatherThreads) sIdx[i] = __ldg(src + i);
      named_bar_sync(1, kGatherThreads);
    }
    auto load_idx = [&](int ks, int (&idx)[kMaxItems]) {
      const int32_t* src =
          whole ? sIdx + ks * kBK
                : sIdx + ((ks / kChunkSt) & 1) * kChunkSt * kBK + (ks % kChunkSt) * kBK;
#pragma unroll
      for (int i = 0; i < kMaxItems; ++i) idx[i] = slot_row[i] >= 0 ? src[slot_row[i]] : -1;
    };
    int ks = 0;
    int idx[kMaxItems];
    if (have) {
      begin_unit(sg);
      layout(unit_n(sg));
      load_idx(0, idx);
    }
    grid_dependency_wait();  // A^T may be written by the previous kernel
    int gs = 0;
    int units = 0;
    Seg last = sg;
    while (have) {
      const int stage = gs % kStages;
      mbar_wait(&empty[stage], ((gs / kStages) & 1) ^ 1u);
      const uint32_t xs = smem_u32(sX + stage * kXBytes);
      if (!skip_a) {
        const int m0 = sg.ub;
#pragma unroll
        for (int i = 0; i < kMaxItems; ++i) {
          if (slot_row[i] < 0) continue;
          const int tok = m0 + slot_chunk[i] * 8;
          const int row = idx[i];
          const uint32_t bytes =
              row >= 0 ? static_cast<uint32_t>(max(0, min(8, args.M - tok)) * 2) : 0u;
          const char* src = bytes ? xa + (static_cast<int64_t>(row) * args.ld_x + tok) * 2 : xa;
          cp_async_16(xs + slot_dst[i], src, bytes);
        }
      }
      cp_async_mbar_arrive_noinc(&full[stage]);
      ++gs;
      // advance and prefetch the next stage's indices (consumed after the
      // next empty-slot wait, which hides their latency)
      if (++ks >= sg.d.kp_steps) {
        last = sg;
        ++units;
        have = walk.next(args, sg);
        ks = 0;
        if (have) {
          begin_unit(sg);
          layout(unit_n(sg));
        }
      } else if (!whole && ks % kChunkSt == 0) {
        // entering chunk c: chunk c - 1 is done everywhere; refill its
        // buffer with chunk c + 1 (read only after the next boundary's barrier)
        named_bar_sync(1, kGatherThreads);
        const int c = ks / kChunkSt;
        if ((c + 1) * kChunkSt < sg.d.kp_steps) stage_chunk(sg, c + 1);
      }
      if (have) load_idx(ks, idx);
    }
    // The CTA's last unit: nothing is left to gather, and once its
    // accumulator is full every ring slot has been consumed, so the gather
    // warps join its epilogue (6 token parts per quadrant instead of 2),
    // staging in ring slot memory.  This shortens the exposed tail.
    if (units > 0) {
      const int j = units - 1;
      const int ew = kEpilogueWarps + (warp - kGatherWarp0);
      // released by the dedicated epilogue warps once the last accumulator
      // is full (a parity wait on tfull could alias an earlier phase)
      mbar_wait(jbar, 0);
      tc_fence_after();
      int sbuf = 0;
      epilogue_unit(args, &map_out, last, tmem_base, j & 1, kTileN, warp & 3, lane, ew >> 2,
                    kWideEpi / 4, sX + (ew - kEpilogueWarps) * kStgBytes, sbuf, true);
      if (lane == 0) bulk_wait_all<0>();
    }
  } else if (warp >= kGatherWarp0 && warp < kEpilogueWarp0 && kRes && args.runs) {
    // Run path with a resident payload: nothing to gather, but the dedicated
    // epilogue warps still count on these warps for the last unit's token
    // parts (see below), staged in the drained ring slots as on the cp.async
    // path.
    int units = 0;
    Seg last;
    while (walk.next(args, sg)) {
      last = sg;
      ++units;
    }
    grid_dependency_wait();  // the previous kernel may still read our output buffer
    if (units > 0) {
      const int j = units - 1;
      const int ew = kEpilogueWarps + (warp - kGatherWarp0);
      mbar_wait(jbar, 0);
      tc_fence_after();
      int sbuf = 0;
      epilogue_unit(args, &map_out, last, tmem_base, j & 1, kTileN, warp & 3, lane, ew >> 2,
                    kWideEpi / 4, sX + (ew - kEpilogueWarps) * kStgBytes, sbuf, true);
      if (lane == 0) bulk_wait_all<0>();
    }
  } else if (warp == kMmaWarp) {
    // ---------------------------------------------------------- MMA issuer
    if (lane == 0) {
      const uint32_t in_fmt = args.in_dtype == kBF16 ? 1u : 0u;
      const bool sparse = args.sparse;
      int gs = 0;
      int j = 0;
      if (sparse && !(flags & kFlagSkipMeta)) {  // the CTA's metadata is in tensor memory
        mbar_wait(mfull, 0);
        tc_fence_after();
      }
      while (walk.next(args, sg)) {
        const int acc = j & 1;
        const uint32_t idesc = umma_idesc_f16(kBN, (sg.ue - sg.ub + 15) & ~15, in_fmt,
                                              /*a (payload) K-major*/ 0u, /*b (A^T) MN-major*/ 1u) |
                               (sparse ? 4u : 0u);
        // paired units: the next unit's MMAs follow each stage's into the
        // other accumulator (j is even here, so that is accumulator 1)
        bool two = false;
        uint32_t idesc2 = 0;
        if (pair) {
          Walker w2 = walk;
          Seg s2;
          if (w2.next(args, s2)) {
            walk = w2;
            two = true;
            idesc2 = umma_idesc_f16(kBN, (s2.ue - s2.ub + 15) & ~15, in_fmt, 0u, 1u);
          }
        }
        mbar_wait(&tempty[acc], ((j >> 1) & 1) ^ 1u);
        if (two) mbar_wait(&tempty[acc ^ 1], (((j + 1) >> 1) & 1) ^ 1u);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * kTileN;
        for (int ks = 0; ks < sg.d.kp_steps; ++ks, ++gs) {
          const int stage = gs % nst;
          if (kRes) mbar_wait(&pfull[sparse ? ks >> 1 : ks], 0);
          mbar_wait(&full[stage], (gs / nst) & 1);
          if (trace && gs < 1024) trace[1024 + gs] = clock64();
          tc_fence_after();
          if (!args.runs) fence_proxy_async_smem();  // cp.async (generic proxy) writes -> tcgen05 reads
          const uint32_t x0 = smem_u32(sX + stage * xstride);
          if (sparse && !(flags & kFlagSkipMma)) {
            // two tcgen05.mma.sp of K = 32 logical rows: A = this stage's 32
            // compressed columns (64 B of the 128-B SW128 row of box ks / 2,
            // 32 B = 16 compressed per MMA), B = 32 gathered rows (4 KB),
            // metadata in column kMetaCol0 + 2 ks + h (pair base + id2 = h)
            // (streamed: the stage's own 64-B swizzled slice, 512-B atoms)
            const uint32_t pa = kRes ? smem_u32(sP + (ks >> 1) * kPBytes) + (ks & 1) * 64
                                : args.sparse == 2 ? smem_u32(sP + stage * kPBytes) + (ks & 1) * 64
                                                   : smem_u32(sP + stage * kPBytes);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const uint64_t adesc = (kRes || args.sparse == 2) ? umma_desc_sw128(pa + h * 32, 16, 1024)
                                                                : umma_desc_sw64(pa + h * 32, 16, 512);
              const uint64_t bdesc = umma_desc_sw128(x0 + h * 4096, kChunkBytes, 1024);
              umma_f16_sp(d_tmem, adesc, bdesc, idesc | static_cast<uint32_t>(h),
                          tmem_base + kMetaCol0 + 2 * ks, (ks != 0) || (h != 0));
            }
          }
          const uint32_t p0 = smem_u32(sP + (kRes ? ks : stage) * kPBytes);
          if (!sparse && !(flags & kFlagSkipMma)) {
#pragma unroll
            for (int kk = 0; kk < kBK / 16; ++kk) {
              // A = payload: K-major SW128, SBO = 1 KB between 8-column groups,
              //     16 K = 32 B per MMA.
              // B = A^T rows: MN-major SW128, LBO = 8 KB between 64-token
              //     chunks, SBO = 1 KB between 8-row K groups, 16 K rows = 2 KB.
              const uint64_t adesc = umma_desc_sw128(p0 + kk * 32, 16, 1024);
              const uint64_t bdesc = umma_desc_sw128(x0 + kk * 2048, kChunkBytes, 1024);
              umma_f16(d_tmem, adesc, bdesc, idesc, (ks != 0) || (kk != 0));
            }
            if (two) {
              const uint32_t d2 = tmem_base + (acc ^ 1) * kTileN;
#pragma unroll
              for (int kk = 0; kk < kBK / 16; ++kk) {
                const uint64_t adesc = umma_desc_sw128(p0 + kk * 32, 16, 1024);
                const uint64_t bdesc = umma_desc_sw128(x0 + kXBytes + kk * 2048, kChunkBytes, 1024);
                umma_f16(d2, adesc, bdesc, idesc2, (ks != 0) || (kk != 0));
              }
            }
          }
          umma_commit(&empty[stage]);
        }
        umma_commit(&tfull[acc]);
        if (two) umma_commit(&tfull[acc ^ 1]);
        j += two ? 2 : 1;
      }
    }
  } else if (warp >= kEpilogueWarp0 || (wide_epi && warp >= kGatherWarp0)) {
    // ------------------------------------------------------------ epilogue
    // Epilogue warp ew owns TMEM lanes 32*(ew%4).. (output columns c of the
    // sub-tile) and token part ew/4 of the unit (2 parts, or 6 with the
    // gather warps joining on the run path).  ew % 4 == warp % 4 because both
    // warp ranges start on a warpgroup boundary.
    const int ew = warp >= kEpilogueWarp0 ? warp - kEpilogueWarp0
                                          : kEpilogueWarps + (warp - kGatherWarp0);
    const int parts = (wide_epi ? kWideEpi : kEpilogueWarps) / 4;
    const int q = warp & 3;
    const int part = ew >> 2;
    // 2 x 1 KB double-buffered staging for the 8 dedicated warps; 1 KB in the
    // gather-list region for the gather warps
    const bool dbl = ew < kEpilogueWarps;
    uint8_t* stg = dbl ? sStg + ew * kStgBytes
                       : reinterpret_cast<uint8_t*>(sIdx) + (ew - kEpilogueWarps) * 1024;
    int sbuf = 0;
    if (meta_writer) {
      // sparse MMA metadata of the owned sub-tile (loaded before the prologue,
      // plan constants): column kMetaCol0 + i for MMA i, this warp's 32 TMEM
      // lanes, all 32 columns in one store; one arrival per quadrant on mfull
      tmem_st_32x32b_x32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + kMetaCol0, meta_v);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(mfull);
    }
    grid_dependency_wait();  // the previous kernel may still read our output buffer
    int j = 0;
    Walker ahead = walk;  // one unit ahead: is the current unit the last?
    Seg nxt;
    bool more = ahead.next(args, nxt);
    while (walk.next(args, sg)) {
      more = ahead.next(args, nxt);
      const int acc = j & 1;
      mbar_wait(&tfull[acc], (j >> 1) & 1);
      // last unit of a non-wide epilogue: release the gather warps into it
      if (!more && !wide_epi && ew == 0 && lane == 0) mbar_arrive(jbar);
      tc_fence_after();
      if (trace && warp == kEpilogueWarp0 && lane == 0 && j < 256) trace[2048 + 2 * j] = clock64();
      // the gather warps share the last unit of the cp.async path (and every
      // unit of the run path)
      const int nparts = (wide_epi || !more) ? kWideEpi / 4 : parts;
      epilogue_unit(args, &map_out, sg, tmem_base, acc, kTileN, q, lane, part, nparts, stg, sbuf,
                    dbl);
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

template <bool kRes, bool kPair>
__global__ void __launch_bounds__(kThreads, 1)
    tw_gemm_kernel(const __grid_constant__ CUtensorMap map_pay,
                   const __grid_constant__ CUtensorMap map_out,
                   const __grid_constant__ RunMaps run_maps, const __grid_constant__ GemmArgs args,
                   const __grid_constant__ WorkTable work) {
  gemm_body<kRes, kPair>(map_pay, map_out, run_maps, args, work.w + blockIdx.x, blockIdx.x,
                         gridDim.x, blockIdx.x);
}

// Several independent layers in ONE launch (TwPlanGroup): layer p owns CTAs
// [cta0[p], cta0[p + 1]) -- its SM share -- and runs the resident or the
// streamed body as it would alone.  One launch per step instead of a fork /
// join over streams, so programmatic dependent launch chains consecutive
// steps like consecutive layers.
__global__ void __launch_bounds__(kThreads, 1)
    tw_gemm_group_kernel(const __grid_constant__ GroupArgs g, const __grid_constant__ WorkTable work) {
  // CTA b runs CTA cta_local[b] of plan cta_plan[b]; its owner work entry is
  // work.w[b] (the host orders the CTAs heaviest first across plans)
  const int b = static_cast<int>(blockIdx.x);
  const int p = g.cta_plan[b];
  const int cta = g.cta_local[b];
  const int ncta = g.plan_ctas[p];
  if (g.resident[p])
    gemm_body<true, false>(g.map_pay[p], g.map_out[p], g.run_maps[p], g.args[p], work.w + b, cta,
                           ncta, b);
  else if (g.args[p].pair)
    gemm_body<false, true>(g.map_pay[p], g.map_out[p], g.run_maps[p], g.args[p], work.w + b, cta,
                           ncta, b);
  else
    gemm_body<false, false>(g.map_pay[p], g.map_out[p], g.run_maps[p], g.args[p], work.w + b, cta,
                            ncta, b);
}

}  // namespace

constexpr int kGroupSmemBytes =
    Cfg<true>::kSmemBytes > Cfg<false>::kSmemBytes ? Cfg<true>::kSmemBytes : Cfg<false>::kSmemBytes;

cudaError_t configure_gemm_kernels() {
  cudaError_t e = cudaFuncSetAttribute(tw_gemm_kernel<true, false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       Cfg<true>::kSmemBytes);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(tw_gemm_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           Cfg<false>::kSmemBytes);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(tw_gemm_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           Cfg<false>::kSmemBytes);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(tw_gemm_group_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              kGroupSmemBytes);
}

cudaError_t launch_tw_gemm_group(const GroupArgs& g, const WorkTable& work, int grid,
                                 cudaStream_t stream) {
  if (grid <= 0) return cudaSuccess;
  if (g.n < 1 || g.n > kMaxGroup || grid > kMaxCtas) return cudaErrorInvalidValue;
  for (int p = 0; p < g.n; ++p)
    if (g.resident[p] && !g.args[p].owner) return cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kGroupSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g.args[0].flags & kFlagNoPdl ? 0 : 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, tw_gemm_group_kernel, g, work);
}

cudaError_t launch_tw_gemm(const CUtensorMap& map_pay, const CUtensorMap& map_out,
                           const RunMaps& run_maps, const GemmArgs& args, const WorkTable& work,
                           bool resident, int grid, cudaStream_t stream) {
  if (grid <= 0) return cudaSuccess;
  if (resident && !args.owner) return cudaErrorInvalidValue;
  if (args.owner && grid > kMaxCtas) return cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = resident ? Cfg<true>::kSmemBytes : Cfg<false>::kSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = args.flags & kFlagNoPdl ? 0 : 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (resident)
    return cudaLaunchKernelEx(&cfg, tw_gemm_kernel<true, false>, map_pay, map_out, run_maps, args,
                              work);
  if (args.pair)
    return cudaLaunchKernelEx(&cfg, tw_gemm_kernel<false, true>, map_pay, map_out, run_maps, args,
                              work);
  return cudaLaunchKernelEx(&cfg, tw_gemm_kernel<false, false>, map_pay, map_out, run_maps, args,
                            work);
}

}  // namespace tw
