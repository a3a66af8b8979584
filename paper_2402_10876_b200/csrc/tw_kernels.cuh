// Shared host/device definitions of the TW device weight format and the
// kernel launchers.  See DESIGN.md "Data layout in HBM".
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace tw {

enum DType : int32_t { kF32 = 0, kF16 = 1, kBF16 = 2 };

constexpr int kTN = 256;  // tokens per work unit            (UMMA N, TMEM columns)
constexpr int kBN = 128;  // output columns per sub-tile     (UMMA M, TMEM lanes)
constexpr int kBK = 64;   // kept rows per stage   (one 128-byte swizzle row of 16-bit data)

// One 128-column slice of a TW tile (UMMA M).  Tiles of width <= 128 are one
// sub-tile (narrower ones zero-padded); wider tiles (g > 128) are split into
// column slices sharing the row runs.
struct SubTile {
  int32_t kp_steps;   // stages of this tile: ceil(padded kept rows / kBK)
  int32_t idx_row;    // row of the gather-index table (one per TW tile)
  int32_t pay_row;    // first payload row in the payload tensor (kBN rows per sub-tile)
  int32_t width;      // live output columns of this slice (<= kBN)
  int32_t out_row;    // first condensed output column == row of C'^T
  int32_t kept;       // K'_i (kept rows), for accounting and LPT ordering
  int32_t stage_off;  // first stage of this sub-tile inside one token block
  int32_t k0;         // first k-step (split-K: a CTA owns stages [k0, k0 + kp_steps))
  int32_t pad1, pad2, pad3, pad4;
};

// Resident-payload kernel: a sub-tile's whole payload (<= kResSteps k-steps,
// i.e. K' <= 448) stays in shared memory for all of the CTA's tokens.
constexpr int kResSteps = 7;

// Owner mode: the whole assignment of every CTA (its sub-tile and token
// range), computed on the host per call and passed as a kernel parameter so
// a CTA starts its pipeline without dependent global loads.
constexpr int kMaxCtas = 160;
struct CtaWork {
  int32_t kp_steps, idx_row, pay_row, width, out_row;  // the owned sub-tile
  int32_t b, e;                                        // token range [b, e)
  int32_t usz;                                         // tokens per unit (0 = idle CTA)
  int32_t k0;                                          // first k-step (split-K), else 0
};
struct WorkTable {
  CtaWork w[kMaxCtas];
};

struct GemmArgs {
  const SubTile* subtiles;  // [n_sub] in visiting order (LPT)
  const void* x;            // activations A^T [K][ld_x] (tokens contiguous), fp16/bf16
  int64_t ld_x;             // elements between A^T rows (multiple of 8)
  const int32_t* gidx;      // [n_tiles][kp] kept rows of every tile, -1 = zero padding
  int32_t kp;               // gather-table row length (multiple of kBK)
  int32_t in_dtype;         // kF16 / kBF16 (activations and payload)
  const int32_t* rowmap;    // [n_cond] condensed col -> output row; nullptr = identity
  void* out;                // C'^T, rows = output columns, M contiguous
  int64_t ld_out;           // elements between output rows
  int32_t out_dtype;        // DType
  int32_t M;
  int32_t n_sub;
  int32_t n_units;          // strided mode: n_sub * ceil(M / kTN)
  int32_t sub_group;        // strided mode: sub-tiles per L2-resident group (>= 1)
  int32_t owner;            // 1 = one sub-tile + token range per CTA (WorkTable), 0 = strided units
  int32_t flags;            // diagnostics (kFlag*); 0 in production
  int32_t vec_ok;           // output rows 16-byte aligned: vector stores allowed
  int32_t vec32_ok;         // output rows 32-byte aligned: 32-byte (full-sector) stores
  int32_t use_tma_store;    // map_out valid (16-bit output): 32 x 16 blocks via TMA stores
  long long* trace;         // optional per-CTA clock64 trace (4096 entries per CTA)
  // row-run path (x in the plan's permuted row layout): activation stages are
  // dense TMA boxes listed per (tile, stage) instead of cp.async gathers
  int32_t runs;
  const int32_t* box_first; // [n_tiles][box_stride]
  const uint32_t* boxes;    // slot | log2(rows) << 6 | position << 9
  int32_t box_stride;
  // TVW on the sparse tensor cores (owner mode, resident payload): the payload
  // holds two of every four K' rows per output column (2:4 along K'), and
  // every tcgen05.mma.sp (K = 32 logical) reads its metadata from one TMEM
  // column kMetaCol0 + i, loaded once per CTA from meta
  int32_t sparse;
  const uint32_t* meta;     // [n_sub][meta_cols][128] u32, TMEM lane order (tw_capi.cu)
  int32_t meta_cols;        // sparse MMAs per sub-tile (2 per 64-row stage)
  // paired units (owner mode, streamed payload, run path): two consecutive
  // units of the CTA's sub-tile share every payload stage (2 ring slots of
  // payload + both units' A^T boxes; accumulators 0 and 1)
  int32_t pair;
};
constexpr int kSparseMaxTokens = 224;  // sparse units: accumulators at 0 / 256, metadata at 480
constexpr int kMetaCol0 = 480;         // 4-aligned; 32 columns = 16 stages (K' <= 1024)

// Tensor maps over the permuted A^T for box heights 1, 2, 4, ..., 64 rows
// (64 tokens wide, 128-byte swizzle).
constexpr int kRunMaps = 7;
struct RunMaps {
  CUtensorMap m[kRunMaps];
};

// Diagnostic switches (profiling only; results are wrong when set).
constexpr int32_t kFlagSkipA = 1;       // do not load the activations
constexpr int32_t kFlagSkipStore = 2;   // do not write the output
constexpr int32_t kFlagSkipMma = 4;     // do not issue tcgen05.mma
constexpr int32_t kFlagNoPdl = 8;       // launch without programmatic dependent launch (timing only)
constexpr int32_t kFlagSkipP = 16;      // do not load the payload
constexpr int32_t kFlagSkipMeta = 32;   // sparse: no metadata load / wait

// K1: persistent warp-specialised TW GEMM (tcgen05 + TMA + cp.async gather).
//   map_pay : payload [n_sub * kBN][Kp], box {64 k, kBN rows}, 128-B swizzle
//   map_out : C'^T (16-bit), box {16 tokens, 32 rows}, 32-B swizzle
//   resident: payload held in shared memory (owner mode, kp_steps <= kResSteps)
cudaError_t launch_tw_gemm(const CUtensorMap& map_pay, const CUtensorMap& map_out,
                           const RunMaps& run_maps, const GemmArgs& args, const WorkTable& work,
                           bool resident, int grid, cudaStream_t stream);

// Raise the dynamic shared-memory limit of every K1 instance (call once per
// device before launching or capturing).
cudaError_t configure_gemm_kernels();

// K1 for several independent layers in one launch (TwPlanGroup): CTA b
// runs CTA cta_local[b] of layer cta_plan[b] (plan_ctas[p] CTAs in all), its
// owner-mode work entry at position b of the shared work table.
constexpr int kMaxGroup = 4;
struct GroupArgs {
  CUtensorMap map_pay[kMaxGroup];
  CUtensorMap map_out[kMaxGroup];
  RunMaps run_maps[kMaxGroup];
  GemmArgs args[kMaxGroup];
  int32_t plan_ctas[kMaxGroup];
  int32_t resident[kMaxGroup];
  int32_t n;
  int8_t cta_plan[kMaxCtas];
  uint8_t cta_local[kMaxCtas];
};
cudaError_t launch_tw_gemm_group(const GroupArgs& g, const WorkTable& work, int grid,
                                 cudaStream_t stream);

// K2: TEW residual, C'^T[urow(c)] (+)= sum_r A^T[r] * v over overlay column c.
constexpr int kMaxColGroups = 64;
struct ResidualArgs {
  const void* at;           // activations A^T [K][ld_at]
  int64_t ld_at;
  int32_t in_dtype;
  const int32_t* col_start; // [n_cols + 1] CSC pointers (columns in descending-nnz order)
  const int32_t* rows;      // [nnz] K rows            (direct kernel)
  const float* vals;        // [nnz]                   (direct kernel)
  const uint32_t* rv;       // [nnz] 16-bit value << 16 | row * T / 8 (16-byte units); nullptr = direct kernel
  const int32_t* out_rows;  // [n_cols] output row (union position)
  const int32_t* accumulate;// [n_cols] 1 = add onto TW result, 0 = overwrite
  const int4* meta;         // [n_cols] {first entry, entries, out row, source row + 1 (0: none)}
  const void* src;          // workspace mode: K1's condensed C'^T (source rows), else nullptr
  int64_t ld_src;           //   (nullptr: the TW result is read back from the out row itself)
  void* out;
  int64_t ld_out;
  int32_t out_dtype;
  int32_t M;
  int32_t n_cols;
  int32_t K;                // rows of A^T
  int32_t block_tokens;     // T: tokens of the staged A^T block (0 = direct kernel)
  int32_t tokens_per_lane;  // 8, or 16 (T = 64 only): lists grouped by T / tokens_per_lane
  int32_t n_blocks;         // ceil(M / T): grid.x
  int32_t n_groups;         // nnz-balanced column splits: grid.y
  int32_t vec_ok;           // out (and src) bases and pitches 16-byte aligned: vector I/O allowed
  int32_t acc_all;          // every column adds onto its out row (caller's tile output already
                            // scattered there: gemm_tew(tile_output=...), executor.py:194)
  int32_t group_first[kMaxColGroups + 1];  // first column of every split
};
cudaError_t launch_tw_residual(const ResidualArgs& args, cudaStream_t stream);

// K2 of several layers in one launch: layer p owns CTAs [cta0[p], cta0[p+1])
// (its n_blocks x n_groups grid, flattened); staged (block_tokens > 0) only.
constexpr int kMaxResGroup = 4;
struct ResidualGroupArgs {
  ResidualArgs args[kMaxResGroup];
  int32_t cta0[kMaxResGroup + 1];
  int32_t n;
};
cudaError_t launch_tw_residual_group(const ResidualGroupArgs& g, cudaStream_t stream);

// Split-K (small M): out[rowmap ? rowmap[r] : r][t] = sum over j < splits of
// ws[j * split_stride + r * ld_ws + t] (fp32, in order j = 0, 1, ...), for
// rows r < rows and tokens t < M, converted to out_dtype.
struct SplitKArgs {
  const float* ws;
  int32_t splits;
  int64_t split_stride;
  int64_t ld_ws;
  int32_t rows;
  int32_t M;
  void* out;
  int64_t ld_out;
  int32_t out_dtype;
  const int32_t* rowmap;
};
cudaError_t launch_splitk_reduce(const SplitKArgs& a, cudaStream_t stream);

// ct[u] = src[src_row[u]] (or 0 where src_row[u] < 0) for u < n_rows, M tokens,
// element size esz (the caller's tile product scattered to the union rows).
cudaError_t launch_scatter_rows(const void* src, int64_t ld_src, const int32_t* src_row,
                                int32_t n_rows, void* dst, int64_t ld_dst, int64_t M, int esz,
                                cudaStream_t stream);
// Token-block size of the staged SpMM for K rows (0 = direct kernel) and the
// number of resident CTAs per SM it allows.
int residual_block_tokens(int32_t K, int* ctas_per_sm);

// K4: A (M x K, row-major, lda) -> A^T (K x M, ld_at) with a dtype cast.
// out_row (optional, [K]): A column k lands in A^T row out_row[k] (plan row layout).
cudaError_t launch_transpose_cast(const void* a, int32_t a_dtype, int64_t M, int64_t K,
                                  int64_t lda, void* at, int32_t at_dtype, int64_t ld_at,
                                  const int32_t* out_row, cudaStream_t stream);

// fp32 plans: A (M x K) -> [fp16(A)^T; fp16(A - fp16(A))^T] (2K x M fp16).
cudaError_t launch_transpose_split(const void* a, int32_t a_dtype, int64_t M, int64_t K,
                                   int64_t lda, void* at, int64_t ld_at, cudaStream_t stream);

// Payload build: packed transposed fp32 CTO payload -> padded [n_sub*kBN][Kp] fp16/bf16
// (kept-row order, as formats.py:200 stores it).
struct PayloadArgs {
  const float* src;          // packed CTO payload (per tile: width x kept, kept contiguous)
  const int64_t* src_base;   // [n_sub] offset of the sub-tile's first column in src
  const int32_t* src_ld;     // [n_sub] kept rows of the tile (row length in src)
  const SubTile* subtiles;
  void* dst;
  int32_t dst_dtype;
  int32_t bn;
  int32_t Kp;
  int32_t n_sub;
};
cudaError_t launch_build_payload(const PayloadArgs& args, cudaStream_t stream);

}  // namespace tw
