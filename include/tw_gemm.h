/*
 * tw_gemm.h -- C ABI of the B200-native TW / TEW sparse matmul
 * (libtwgemm.so, built from paper_2402_10876_b200/csrc for sm_100a).
 *
 * The reference (tilesparse 0.1.0, pure Python) has no FFI; its boundary for
 * this path is the Python call surface of executor.py / formats.py.  Each
 * entry point below names the reference function it replaces; the Python
 * shim in paper_2402_10876_b200/executor.py keeps the reference signatures
 * and calls these through ctypes.
 *
 * Conventions
 *   - Plain C types only: host pointers for weights/encodings, device
 *     pointers for activations/outputs, cudaStream_t passed as void*.
 *   - Activations enter the GEMM as A^T: k rows x m tokens, tokens
 *     contiguous, pitch ld_at (ld_at % 8 == 0, 16-byte aligned base), in the
 *     plan's compute dtype -- the layout the GEMM itself writes (C'^T), so a
 *     layer's output feeds the next layer without a copy.  tw_transpose_cast
 *     converts a row-major A (m x k, any dtype).  Outputs are C'^T: one row
 *     per output column, tokens contiguous, pitch ld_ct.
 *   - Stream-ordered, no host synchronisation inside tw_gemm / tw_gemm_tew /
 *     tw_transpose_cast, so they are CUDA-graph capturable.
 *   - Every function returns a status code; tw_last_error() gives the
 *     thread-local message of the last failure.
 */
#ifndef TW_GEMM_H_
#define TW_GEMM_H_

#include <stdint.h>
#include <stddef.h>

#if defined(__GNUC__)
#define TW_API __attribute__((visibility("default")))
#else
#define TW_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes: mirror tilesparse.errors (errors.py:4-17) and the CLI exit
 * codes (cli.py:40-45). */
#define TW_OK 0
#define TW_ERR_INVALID_INPUT 2   /* InvalidInputError                     */
#define TW_ERR_CONTRACT 3        /* ContractViolationError                */
#define TW_ERR_CORRUPT 4         /* CorruptEncodingError (CLI exit 2)     */
#define TW_ERR_CUDA 5            /* CUDA / driver failure (no reference)  */

/* Element types. */
#define TW_F32 0
#define TW_F16 1
#define TW_BF16 2

/* Activation row layouts (tw_gemm_ex). */
#define TW_LAYOUT_NATURAL 0        /* A^T rows in original K order             */
#define TW_LAYOUT_PLAN 1           /* the plan's row order (tw_plan_prepare)   */

/* Sub-tile visiting order inside each token block
 * (executor.py:206-227 schedule_tiles strategies). */
#define TW_SCHEDULE_LPT 0          /* descending surviving K'             */
#define TW_SCHEDULE_ROUND_ROBIN 1  /* tile order                          */

typedef struct tw_plan tw_plan;

typedef struct tw_plan_info {
  int32_t k, n, g;            /* original dims and tile width            */
  int32_t n_tiles;            /* TW tiles                                */
  int32_t n_sub;              /* UMMA-N slices (== n_tiles when g <= 256) */
  int32_t bn;                 /* output columns per sub-tile (UMMA M)    */
  int32_t kp;                 /* padded gather-list length               */
  int32_t n_condensed;        /* N' = sum of tile widths                 */
  int32_t n_union;            /* |TW cols U overlay cols| (TEW), else N' */
  int32_t compute_dtype;      /* TW_F16 | TW_BF16                        */
  int64_t nnz;                /* overlay entries (0 when none)           */
  int64_t kept_macs_per_token;/* sum_i width_i * K'_i (+ nnz for TEW)    */
  int32_t sm_count;           /* SMs of the plan's device                */
  int32_t has_overlay;
  int32_t row_runs;           /* 1: the plan has a permuted row layout in
                                 which every tile's kept rows form runs     */
  int32_t row_copies;         /* rows of the plan layout = row_copies * k
                                 (one row order per group of tiles)         */
  int32_t sm_budget;          /* SMs K1 uses (tw_plan_set_sm_budget)     */
  int64_t stage_work;         /* sum over sub-tiles of 64-row k-steps: the
                                 per-token cost model of the work split     */
  int32_t sparse_payload;     /* 1: every tile's payload is 2:4 along K'
                                 (TVW, patterns.py:645-717) and K1 runs it on
                                 tcgen05.mma.sp from a compressed resident
                                 copy (TW_NO_SPARSE=1: dense tensor cores)  */
  int32_t splitk_max;         /* split-K for small m: most CTAs per sub-tile
                                 (0: never; see tw_gemm)                     */
  int32_t splitk_max_tokens;  /* ... used when m <= this on tiles of at least
                                 splitk_min_steps 64-row stages             */
  int32_t splitk_min_steps;
} tw_plan_info;

/* Build a device plan from a CTO encoding held in host memory.
 * Replaces: formats.CtoEncoding (formats.py:82-181) as consumed by
 * executor.gemm_cto (executor.py:149-177).  Validates exactly what
 * gemm_cto validates (offset decode of tile_rows / tile_cols, columns
 * strictly increasing across tiles -> TW_ERR_CORRUPT), converts the fp32
 * payload to compute_dtype on the device and builds the gather lists.
 *   row_offsets: n_tiles x max_rows u32, col_offsets: n_tiles x max_cols u32,
 *   payload: sum(row_counts[i]*col_counts[i]) fp32, per tile transposed
 *            (width x kept rows, kept rows contiguous; formats.py:200).
 * row_runs = 1 lets the plan choose a permuted row layout in which every
 * tile's kept rows form runs (tiles' K' then follow that order; see
 * tw_plan_prepare / tw_gemm_ex); 0 keeps ascending kept-row order.
 * Synchronises `stream` before returning. */
TW_API int tw_plan_create_cto(tw_plan** out, int32_t k, int32_t n, int32_t g, int32_t n_tiles,
                       const uint32_t* row_counts, const uint32_t* col_counts,
                       const uint32_t* row_offsets, int32_t max_rows,
                       const uint32_t* col_offsets, int32_t max_cols, const float* payload,
                       int32_t compute_dtype, int32_t schedule, int32_t row_runs, void* stream);

/* tw_plan_create_cto with the chained-layer options:
 *   row_groups [n_groups + 1]: bounds 0 = b_0 < ... < b_n = k of row groups;
 *     the row-run permutation (row_runs = 1) then only reorders rows inside
 *     each group (NULL: unconstrained).  Pass the previous layer's
 *     tw_plan_output_groups so that its epilogue can write this plan's layout.
 *   out_row_of_cond [N']: the C'^T row each condensed column is written to;
 *     it may only permute rows inside each 128-column sub-tile block (free:
 *     the payload rows are reordered), so a layer writes its output directly
 *     in the next layer's row-run order (NULL: condensed order).
 * tw_plan_condensed_columns then reports the original column of every output
 * row in that order. */
TW_API int tw_plan_create_cto_ex(tw_plan** out, int32_t k, int32_t n, int32_t g, int32_t n_tiles,
                                 const uint32_t* row_counts, const uint32_t* col_counts,
                                 const uint32_t* row_offsets, int32_t max_rows,
                                 const uint32_t* col_offsets, int32_t max_cols,
                                 const float* payload, int32_t compute_dtype, int32_t schedule,
                                 int32_t row_runs, const int32_t* row_groups, int32_t n_groups,
                                 const int32_t* out_row_of_cond, void* stream);

/* Row blocks of C'^T written by one sub-tile each (host buffer of n_sub + 1
 * ascending bounds): the groups tw_plan_create_cto_ex may permute within. */
TW_API int tw_plan_output_groups(const tw_plan* plan, int32_t* bounds);

/* Device-native plan file "TWP1": the plan as the kernels
 * read it (validated structure, merged tiles, row-run layout and box tables,
 * fp16/bf16 payload), so tw_plan_load only uploads -- no CTO validation,
 * merging, row ordering or payload conversion.  The CTO1 artifact
 * (formats.py:239-304) stays the interchange format.
 * tw_plan_save: *len in = buffer capacity (buf may be NULL to query), out =
 * bytes needed; a plan with an overlay cannot be saved (attach it after
 * loading).  tw_plan_load validates every index against the plan's dims
 * (TW_ERR_CORRUPT otherwise) and synchronises `stream`. */
TW_API int tw_plan_save(const tw_plan* plan, void* buf, uint64_t* len);
TW_API int tw_plan_load(tw_plan** out, const void* buf, uint64_t len, void* stream);

/* Attach a TEW overlay (CSC, int64 like patterns.SparseOverlay,
 * patterns.py:145-214).  Replaces the overlap/dims checks of
 * executor.gemm_tew (executor.py:186-193): dims mismatch -> TW_ERR_INVALID_INPUT,
 * an entry on a payload slot -> TW_ERR_CONTRACT.  Computes the union column
 * layout of the TEW output (executor.py:201-203). */
TW_API int tw_plan_attach_overlay(tw_plan* plan, int32_t k, int32_t n, int64_t nnz,
                           const int64_t* col_ptr, const int64_t* row_idx, const float* values,
                           void* stream);

TW_API int tw_plan_get_info(const tw_plan* plan, tw_plan_info* info);

/* Number of SMs the plan's product kernel (K1) may occupy (0 = all of the
 * device).  With a budget below the SM count, several plans launched on
 * concurrent streams run side by side (a grouped step over independent
 * layers, paper_2402_10876_b200.TwPlanGroup); the work split over the
 * budget mirrors the LPT balancing of executor.py:206-227. */
TW_API int tw_plan_set_sm_budget(tw_plan* plan, int32_t sms);

/* Cost model of the work split for `sms` SMs (0 = all) and m tokens,
 * without changing the plan: the busiest CTA's token x 64-row-stage count
 * and its number of units (used to choose SM shares, TwPlanGroup). */
TW_API int tw_plan_estimate(const tw_plan* plan, int32_t sms, int64_t m, int64_t* stage_tokens,
                            int32_t* units);

/* Output column maps (host buffers sized n_condensed / n_union):
 * original column id of every row of C'^T. */
TW_API int tw_plan_condensed_columns(const tw_plan* plan, int32_t* out_cols);
TW_API int tw_plan_union_columns(const tw_plan* plan, int32_t* out_cols);

/* TW product, condensed: ct[N' x m] = (A . W_tw)^T from at = A^T [k x m].
 * Replaces: executor.gemm_cto (executor.py:149-177), gemm_tile_sparse
 * (executor.py:135-146) and execute_batched (executor.py:230-265); all three
 * are bit-identical on the GPU as in the reference.
 * Small m (<= 128 tokens) on plans with long tiles (>= 16 64-row stages) runs
 * split-K: the stages over several CTAs, fp32 partials in a workspace the
 * plan owns, summed by a second kernel.  Like a cuBLAS handle's workspace,
 * that workspace serves one launch at a time, so calls on one plan must be
 * ordered (one stream, or events between streams); TW_SPLITK=0 turns it off. */
TW_API int tw_gemm(const tw_plan* plan, const void* at, int64_t m, int64_t ld_at, void* ct,
                   int64_t ld_ct, int32_t out_dtype, void* stream);

/* Several independent TW layers in ONE K1 launch (TwPlanGroup): plan i
   runs on its SM share (tw_plan_set_sm_budget; the shares must sum to at
   most the GPU) over xs[i] (layout x_layouts[i], NULL = all natural) into
   cts[i]; all with M tokens and out_dtype.  Bit-identical to n tw_gemm_ex
   calls.  Replaces the reference's threaded lanes over independent products
   (execute_batched, executor.py:230-265) at the step level. */
TW_API int tw_gemm_group(const tw_plan* const* plans, int32_t n, const void* const* xs,
                         const int64_t* ld_xs, const int32_t* x_layouts, void* const* cts,
                         const int64_t* ld_cts, int64_t m, int32_t out_dtype, void* stream);

/* TEW for several independent plans (each with an overlay): K1 of all of
   them in one launch (into workspaces[i] when tw_plan_tew_workspace_bytes
   asks for one, else straight into the union rows), then every plan's K2 on
   the same stream.  Bit-identical to n tw_gemm_tew_ex calls with the same
   workspaces. */
TW_API int tw_gemm_tew_group(const tw_plan* const* plans, int32_t n, const void* const* xs,
                             const int64_t* ld_xs, const int32_t* x_layouts, void* const* cts,
                             const int64_t* ld_cts, void* const* workspaces,
                             const uint64_t* ws_bytes, int64_t m, int32_t out_dtype,
                             void* stream);

/* tw_gemm with the activation row layout given: TW_LAYOUT_NATURAL (A^T rows
 * in K order, kept rows gathered with cp.async) or TW_LAYOUT_PLAN (A^T as
 * tw_plan_prepare writes it; on plans with row_runs, every stage is a few
 * dense TMA boxes).  Both layouts give bit-identical results. */
TW_API int tw_gemm_ex(const tw_plan* plan, const void* at, int64_t m, int64_t ld_at, void* ct,
                      int64_t ld_ct, int32_t out_dtype, int32_t at_layout, void* stream);

/* A (m x k row-major, pitch lda, any dtype) -> A^T in the plan's row layout and
 * compute dtype (row_copies * k rows x m, pitch ld_at): tw_transpose_cast plus
 * the plan's row permutation(s).  Replaces the as_matrix / astype copies (core.py:32-43,
 * executor.py:158) for inputs of this plan. */
TW_API int tw_plan_prepare(const tw_plan* plan, const void* a, int32_t a_dtype, int64_t m,
                           int64_t lda, void* at, int64_t ld_at, void* stream);

/* A natural-order A^T (k x m, pitch ld_at, compute dtype) -> the plan's row
 * layout (row_copies * k x m, pitch ld_x): row perm[p] copied to position p
 * (a plain copy for plans without row runs).  The device form of
 * tw_plan_row_order for callers that already hold A^T. */
TW_API int tw_plan_permute_rows(const tw_plan* plan, const void* at, int64_t m, int64_t ld_at,
                                void* x, int64_t ld_x, void* stream);

/* Original K row held at each position of the plan's row layout (host buffer
 * of row_copies * k entries; the identity when row_runs == 0). */
TW_API int tw_plan_row_order(const tw_plan* plan, int32_t* out_rows);

/* TEW product over the union columns: ct[|union| x M].
 * Replaces: executor.gemm_tew (executor.py:180-203). */
TW_API int tw_gemm_tew(const tw_plan* plan, const void* at, int64_t m, int64_t ld_at, void* ct,
                       int64_t ld_ct, int32_t out_dtype, void* stream);

/* tw_gemm_tew with a caller-owned workspace of tw_plan_tew_workspace_bytes()
 * bytes (16-byte aligned): K1 writes the condensed TW result there with its
 * TMA epilogue and K2 scatters every column to its union row while adding the
 * residual (faster than K1 scattering union rows itself).  A size of 0 means
 * the plan does not use one (workspace may then be NULL). */
TW_API int tw_plan_tew_workspace_bytes(const tw_plan* plan, int64_t m, int32_t out_dtype,
                                       uint64_t* bytes);
TW_API int tw_gemm_tew_ws(const tw_plan* plan, const void* at, int64_t m, int64_t ld_at,
                          void* ct, int64_t ld_ct, int32_t out_dtype, void* workspace,
                          uint64_t ws_bytes, void* stream);

/* tw_gemm_tew_ws with the activation layout of tw_gemm_ex: TW_LAYOUT_PLAN
 * reads A^T in the plan's row-run order (tw_plan_prepare) in both K1 and K2
 * (the overlay rows are remapped to layout positions at attach time), so a
 * TEW layer gets the dense-TMA row runs too.  Results are bit-identical to
 * tw_gemm_tew_ws on the natural-order A^T.
 * Replaces: executor.gemm_tew (executor.py:180-203). */
TW_API int tw_gemm_tew_ex(const tw_plan* plan, const void* at, int64_t m, int64_t ld_at,
                          void* ct, int64_t ld_ct, int32_t out_dtype, void* workspace,
                          uint64_t ws_bytes, int32_t x_layout, void* stream);

/* TEW product on a tile product the caller already holds (K2 only; the TW
 * GEMM is not run again).  Replaces the tile_output path of executor.gemm_tew
 * (executor.py:180-203, `tile_out = tile_output if ... else ...` at line 194):
 * the tile product is expanded to the original columns, the overlay added and
 * the result re-condensed to the union columns.
 *   tile_ct (ld_tile): the tile product as C^T rows (one row per column of the
 *     caller's GemmOutput.column_map, tokens contiguous), in out_dtype.
 *   tile_row_of_union: host array [n_union]: row of tile_ct holding union
 *     column u, or -1 (that column starts from zero).  NULL means tile_ct rows
 *     are this plan's condensed columns (tw_plan_condensed_columns order).
 * With NULL the call is stream-ordered and graph-capturable; with a map it
 * uploads the map and synchronises `stream` once. */
TW_API int tw_gemm_tew_reuse(const tw_plan* plan, const void* at, int64_t m, int64_t ld_at,
                             const void* tile_ct, int64_t ld_tile,
                             const int32_t* tile_row_of_union, void* ct, int64_t ld_ct,
                             int32_t out_dtype, int32_t at_layout, void* stream);

/* A (m x k row-major, pitch lda, a_dtype) -> A^T (k x m, pitch ld_at, at_dtype).
 * Replaces the float32/float64 carrier copies of core.as_matrix
 * (core.py:32-43) and executor.py:158 on the device; the per-tile column
 * gather a64[:, rows] of executor.py:121-124 happens inside tw_gemm. */
TW_API int tw_transpose_cast(const void* a, int32_t a_dtype, int64_t m, int64_t k, int64_t lda,
                      void* at, int32_t at_dtype, int64_t ld_at, void* stream);

TW_API void tw_plan_destroy(tw_plan* plan);

/* Diagnostics only: device buffer of (grid x 4096) int64 that K1 fills with
 * clock64() timestamps per pipeline stage (nullptr disables).  Not for
 * production use; see scripts/ktrace.py. */
TW_API void tw_debug_set_trace(void* dev_buffer);

/* Thread-local message of the last failing call ("" if none). */
TW_API const char* tw_last_error(void);

/* ABI version (major * 100 + minor). */
TW_API int32_t tw_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* TW_GEMM_H_ */
