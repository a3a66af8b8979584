// Shared host/device definitions of the TW device weight format and the
// kernel launchers.  See DESIGN.md "Data layout in HBM".
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace tw {

enum DType : int32_t { kF32 = 0, kF16 = 1, kBF16 = 2 };

constexpr int kBM = 128;  // tokens per work unit  (UMMA M, TMEM lanes)
constexpr int kBK = 64;   // kept rows per stage   (one 128-byte swizzle row of 16-bit data)

// One UMMA-N slice of a TW tile.  Tiles of width <= 256 are one sub-tile;
// wider tiles (g > 256) are split into column slices sharing the gather list.
struct SubTile {
  int32_t kp_steps;  // ceil(K'_i / kBK): pipeline stages of this tile
  int32_t idx_row;   // row of the gather-index table (one per TW tile)
  int32_t pay_row;   // first payload row in the payload tensor (BN rows per sub-tile)
  int32_t width;     // live output columns of this slice (<= BN)
  int32_t out_row;   // first condensed output column == row of C'^T
  int32_t kept;      // K'_i (kept rows), for accounting
  int32_t stage_off; // first stage of this sub-tile inside one 128-token block
  int32_t pad1;
};

struct GemmArgs {
  const int32_t* rowidx;    // [n_tiles][Kp] original K-row ids; padding = K (TMA OOB -> zeros)
  const SubTile* subtiles;  // [n_sub] in visiting order inside one m-block (LPT)
  const int32_t* rowmap;    // [n_cond] condensed col -> output row; nullptr = identity
  void* out;                // C'^T, rows = output columns, M contiguous
  int64_t ld_out;           // elements between output rows
  int32_t out_dtype;        // DType
  int32_t M;
  int32_t Kp;               // padded gather-list length (multiple of kBK)
  int32_t n_sub;
  int32_t n_mblk;
  int32_t n_units;          // n_sub * n_mblk
  int32_t flags;            // diagnostics (kFlag*); 0 in production
  int32_t K;                // original rows of A^T (gather sentinel)
  const void* at;           // A^T base (cp.async gather path)
  int64_t ld_at;            // A^T row pitch in elements
  int32_t spm;              // stages per 128-token block (sum of kp_steps)
  int32_t split;            // 1 = stream-K ranges, 0 = whole units strided by gridDim.x
  float* ws;                // stream-K partials, gridDim.x x [BN][128] fp32
  int32_t* ws_flags;        // gridDim.x publish flags (0 between launches)
  int32_t vec_ok;           // output rows 16-byte aligned: vector stores allowed
  int32_t use_tma_store;    // map_out is valid (condensed output via TMA 2-D stores)
  long long* trace;         // optional per-CTA clock64 trace (4096 entries per CTA)
};

// Diagnostic switches (profiling only; results are wrong when set).
constexpr int32_t kFlagSkipA = 1;       // do not load the gathered activations
constexpr int32_t kFlagSkipStore = 2;   // do not write the output
constexpr int32_t kFlagSkipMma = 4;     // do not issue tcgen05.mma

// How the activation rows are gathered into shared memory.
enum GatherMode : int32_t { kGatherTma4 = 0, kGatherCpAsync = 1 };

// K1: persistent warp-specialised gather GEMM (tcgen05 + TMA gather4).
// bn in {32, 64, 128, 256}; in_dtype kF16 or kBF16.
cudaError_t launch_tw_gather_gemm(const CUtensorMap& map_at, const CUtensorMap& map_pay,
                                  const CUtensorMap& map_out, const GemmArgs& args,
                                  const void* at, int64_t ld_at, int bn, int in_dtype,
                                  int gather_mode, int grid, cudaStream_t stream);

// Raise the dynamic shared-memory limit of every K1 instance (call once per
// device before launching or capturing).
cudaError_t configure_gemm_kernels();

// K2: TEW residual, C'^T[urow(c)] (+)= sum_r A^T[r] * v over overlay column c.
struct ResidualArgs {
  const void* at;           // A^T, K x M (ld_at)
  int64_t ld_at;
  int32_t in_dtype;
  const int32_t* col_start; // [n_cols + 1] CSC pointers into rows / vals
  const int32_t* rows;      // [nnz]
  const float* vals;        // [nnz]
  const int32_t* out_rows;  // [n_cols] output row (union position)
  const int32_t* accumulate;// [n_cols] 1 = add onto TW result, 0 = overwrite
  void* out;
  int64_t ld_out;
  int32_t out_dtype;
  int32_t M;
  int32_t n_cols;
};
cudaError_t launch_tw_residual(const ResidualArgs& args, cudaStream_t stream);

// K4: A (M x K, row-major, lda) -> A^T (K x M, ld_at) with a dtype cast.
cudaError_t launch_transpose_cast(const void* a, int32_t a_dtype, int64_t M, int64_t K,
                                  int64_t lda, void* at, int32_t at_dtype, int64_t ld_at,
                                  cudaStream_t stream);

// Payload build: packed transposed fp32 CTO payload -> padded [n_sub*BN][Kp] fp16/bf16.
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
