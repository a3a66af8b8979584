// C ABI (include/tw_gemm.h): host-side validation of CTO encodings and
// overlays, construction of the device weight format (padded fp16/bf16
// payload + per-tile gather lists), TMA descriptor encoding, work-unit sizing
// and kernel dispatch.  All numerics run in the kernels of tw_gemm.cu /
// tw_aux.cu; nothing here computes on the CPU beyond index bookkeeping.
#include "../../include/tw_gemm.h"
#include "tw_kernels.cuh"

#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <iterator>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

using namespace tw;

namespace {

thread_local std::string g_last_error;
long long* g_trace = nullptr;  // diagnostics: per-CTA clock64 trace buffer

int fail(int status, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return status;
}

#define TW_CUDA(expr)                                                                    \
  do {                                                                                   \
    cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess)                                                               \
      return fail(TW_ERR_CUDA, "%s failed: %s", #expr, cudaGetErrorString(_e));          \
  } while (0)

// ------------------------------------------------------- driver entry point
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 2-D tensor map over a row-major [rows][cols] matrix (cols contiguous).
// swizzle: 0 = none, 32 / 64 / 128 = that many bytes.
int make_map_2d(CUtensorMap* map, const void* base, int32_t dtype, uint64_t cols, uint64_t rows,
                uint64_t pitch_elems, uint32_t box_cols, uint32_t box_rows, int swizzle = 128) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fail(TW_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (driver too old?)");
  const CUtensorMapDataType dt = dtype == kBF16  ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                 : dtype == kF32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                                 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  const uint64_t esz = dtype == kF32 ? 4 : 2;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {pitch_elems * esz};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swizzle == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                  : swizzle == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                  : swizzle == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                  : CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(TW_ERR_INVALID_INPUT,
                "cuTensorMapEncodeTiled failed (%d): cols=%llu rows=%llu pitch=%llu", (int)r,
                (unsigned long long)cols, (unsigned long long)rows,
                (unsigned long long)pitch_elems);
  return TW_OK;
}

int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return (v && *v) ? atoi(v) : dflt;
}

int sm_count_of_current_device(int* out) {
  int dev = 0;
  TW_CUDA(cudaGetDevice(&dev));
  TW_CUDA(cudaDeviceGetAttribute(out, cudaDevAttrMultiProcessorCount, dev));
  return TW_OK;
}

template <class T>
int upload(T** dptr, const std::vector<T>& host, cudaStream_t s) {
  *dptr = nullptr;
  if (host.empty()) return TW_OK;
  TW_CUDA(cudaMalloc(reinterpret_cast<void**>(dptr), host.size() * sizeof(T)));
  TW_CUDA(cudaMemcpyAsync(*dptr, host.data(), host.size() * sizeof(T), cudaMemcpyHostToDevice, s));
  return TW_OK;
}

int32_t round_up(int32_t v, int32_t a) { return (v + a - 1) / a * a; }

// IEEE binary16 / bfloat16 bits of a float, round to nearest even.
uint32_t float_to_half_bits(float f) {
  const __half h = __float2half_rn(f);
  return (uint32_t)__half_as_ushort(h);
}
uint32_t float_to_bf16_bits(float f) {
  const __nv_bfloat16 h = __float2bfloat16_rn(f);
  return (uint32_t)__bfloat16_as_ushort(h);
}

}  // namespace

struct TwLaunch {  // everything a K1 launch needs besides the plan constants
  GemmArgs a;
  WorkTable work;
  RunMaps maps;
  CUtensorMap map_out;
  int grid = 0;
  bool resident = false;
  bool sparse = false;  // tcgen05.mma.sp on the compressed payload
  bool sparse_resident = false;
  // split-K (small M): K1 wrote S fp32 partial products into the plan's
  // workspace; splitk_reduce sums them into the caller's output
  int splitk = 0;
  SplitKArgs red{};
};

struct tw_plan;
struct LaunchEnv;

struct tw_plan {
  int32_t k = 0, n = 0, g = 0, n_tiles = 0, n_sub = 0, bn = 0, kp = 0, n_cond = 0;
  int32_t dtype = kF16, schedule = TW_SCHEDULE_LPT, sm_count = 0;
  bool split = false;  // fp32 compute as fp16 hi/lo pairs: A^T has 2k rows
  int32_t k_rows() const { return split ? 2 * k : k; }  // rows of the kernels' A^T
  std::vector<SubTile> subtiles;
  std::vector<int32_t> cond_cols;        // condensed col -> original col
  std::vector<int32_t> tile_of_col;      // original col -> tile (or -1)
  std::vector<std::vector<uint8_t>> tile_rows;  // per tile: K flags
  std::vector<int32_t> tile_first_cond;  // per tile: first condensed column
  int64_t kept_macs = 0;
  bool owner = false;                    // n_sub <= SMs: one sub-tile per CTA
  bool resident = false;                 // owner and every payload fits in smem
  std::vector<int32_t> cta_first;        // owner mode: [n_sub + 1]
  int32_t sm_budget = 0;                 // SMs K1 may use (<= sm_count; tw_plan_set_sm_budget)
  std::vector<double> tile_cost;         // owner split weight per tile (run path)
  // last launch geometry (run_tw): reused while the key matches
  mutable std::mutex launch_mu;
  mutable bool cache_valid = false;
  mutable TwLaunch cache;
  struct Key {
    const void* x; int64_t m, ld_x; void* ct; int64_t ld_ct; int32_t out_dtype;
    const int32_t* rowmap; int64_t out_rows; bool plan_layout; int32_t budget;
    int flags, no_tma_store, strided, force_owner, gran, split1, run_max_units, no_sparse,
        sparse_resident, splitk, pair;
    long long* trace;
    bool operator==(const Key& o) const { return std::memcmp(this, &o, sizeof(Key)) == 0; }
  };
  mutable Key cache_key;
  // row-run layout: A^T rows permuted so each tile's kept rows form a few
  // runs; position p holds original row perm[p] (empty = not used)
  bool runs = false;
  int32_t row_copies = 1;                // G copies of A^T (one per tile group)
  std::vector<int32_t> perm, inv;        // [G * k]: position -> row, copy g: row -> position
  int32_t box_stride = 0;                // stages per tile + 1
  // host copies of the device tables (tw_plan_save / tw_plan_load)
  std::vector<int32_t> h_gidx, h_gidx_pos, h_box_first;
  std::vector<uint32_t> h_boxes;
  // device
  SubTile* d_subtiles = nullptr;
  int32_t* d_perm = nullptr;             // [k] position -> original row
  int32_t* d_inv = nullptr;              // [k] original row -> position
  int32_t* d_box_first = nullptr;        // [n_tiles][box_stride] first box of every stage
  int32_t* d_gidx_pos = nullptr;         // [n_tiles][kp] kept rows as layout positions
  uint32_t* d_boxes = nullptr;           // slot | log2(rows) << 6 | position << 9
  int32_t* d_gidx = nullptr;  // [n_tiles][kp] kept rows, -1 padded
  void* d_payload = nullptr;
  CUtensorMap map_pay;
  // TVW on the sparse tensor cores: every tile's payload is 2:4 along K'
  // (two nonzeros in each group of four kept rows, K' order); compressed
  // payload [n_sub * bn][kpc] and per-MMA metadata (tw_gemm.cu, sparse MMA)
  bool sparse = false;
  int32_t kpc = 0, meta_cols = 0;
  void* d_payload_sp = nullptr;
  uint32_t* d_meta = nullptr;
  CUtensorMap map_pay_sp;               // resident kernel: 64-column boxes (2 stages), SW128
  CUtensorMap map_pay_sp64;             // streamed kernel: 32-column slices (1 stage), SW64
  // TEW overlay
  bool has_overlay = false;
  int64_t nnz = 0;
  std::vector<int32_t> union_cols;
  int32_t n_ov_cols = 0;                // overlay columns with entries (listed first)
  int32_t n_ov_cols_all = 0;            // + kept columns without entries (workspace mode)
  // device overlay arrays; replaced as a whole by tw_plan_attach_overlay
  // (built into a fresh set first, so a failed attach leaves the old one)
  struct OvDev {
    int32_t* union_rowmap = nullptr;    // condensed col -> union position
    int32_t* start = nullptr;
    int32_t* rows = nullptr;
    float* vals = nullptr;
    int32_t* out = nullptr;
    int32_t* acc = nullptr;
    int4* meta = nullptr;               // K2 per column: {first entry, entries, out row, src row + 1}
    uint32_t* rv = nullptr;             // K2 lists: 16-bit value << 16 | staged-row offset
    int32_t* rows_pos = nullptr;        // row-run plans: rows as layout positions (copy 0)
    uint32_t* rv_pos = nullptr;         // row-run plans: rv as layout positions (copy 0)
    void release() {
      for (void* q : {(void*)union_rowmap, (void*)start, (void*)rows, (void*)vals, (void*)out,
                      (void*)acc, (void*)meta, (void*)rv, (void*)rows_pos, (void*)rv_pos})
        if (q) cudaFree(q);
      *this = OvDev{};
    }
  } ov;
  int32_t ov_block_tokens = 0, ov_ctas_per_sm = 0, ov_tpl = 8;
  // split-K workspace for small M: up to splitk_max partial products of
  // n_cond rows x kSplitKMaxTokens fp32 (allocated at plan creation)
  float* d_splitws = nullptr;
  int32_t splitk_max = 0;
  std::vector<int32_t> ov_start;       // host copy of the K2 column pointers

  ~tw_plan() {
    for (void* p : {(void*)d_subtiles, (void*)d_gidx, d_payload, (void*)d_perm, (void*)d_inv,
                    (void*)d_box_first, (void*)d_boxes, (void*)d_gidx_pos, d_payload_sp,
                    (void*)d_meta, (void*)d_splitws})
      if (p) cudaFree(p);
    ov.release();
  }
};

// Owner-mode split over the plan's SM budget G: sub-tile s gets c_s CTAs,
// c_s proportional to its per-token cost, largest remainder, at least one
// each.  Mirrors the LPT balancing of executor.py:206-227.  Plans with more
// sub-tiles than G run the strided decomposition instead.
namespace {
constexpr uint32_t kTwpMagic = 0x31505754u;  // "TWP1"
constexpr uint32_t kTwpVersion = 1;

struct Writer {
  std::vector<uint8_t> b;
  template <class T> void pod(const T& v) {
    const uint8_t* p = reinterpret_cast<const uint8_t*>(&v);
    b.insert(b.end(), p, p + sizeof(T));
  }
  template <class T> void vec(const std::vector<T>& v) {
    pod<uint64_t>(v.size());
    const uint8_t* p = reinterpret_cast<const uint8_t*>(v.data());
    b.insert(b.end(), p, p + v.size() * sizeof(T));
  }
};

struct Reader {
  const uint8_t* p;
  size_t n, off = 0;
  bool ok = true;
  template <class T> T pod() {
    T v{};
    if (off + sizeof(T) > n) { ok = false; return v; }
    std::memcpy(&v, p + off, sizeof(T));
    off += sizeof(T);
    return v;
  }
  template <class T> std::vector<T> vec(uint64_t max_elems = (1ull << 34)) {
    const uint64_t len = pod<uint64_t>();
    std::vector<T> v;
    if (!ok || len > max_elems || off + len * sizeof(T) > n) { ok = false; return v; }
    v.resize(len);
    std::memcpy(v.data(), p + off, len * sizeof(T));
    off += len * sizeof(T);
    return v;
  }
};
}  // namespace

static std::vector<int32_t> split_counts(const tw_plan* plan, int G);

// Split-K for small M (tokens <= kSplitKMaxTokens): one CTA per sub-tile would
// leave most SMs idle while each active CTA streams every stage of its
// sub-tile at one SM's ingress rate (profiles/r2_k1_stage_ingress.txt), so the
// stages of every sub-tile are spread over S CTAs instead, each writing an
// fp32 partial product, and a second kernel sums the S partials in order.
// Measured (scripts/splitk_probe.py): 3072 x 768 (43 k-steps) at M = 1 / 128:
// 13.3 -> 8.0 / 14.5 -> 11.1 us; on 9-step sub-tiles (1024^2, 768 x 3072) it
// only pays below ~20 tokens, and at M = 256 it loses everywhere.
constexpr int64_t kSplitKMaxTokens = 128;
constexpr int kSplitKMinSteps = 16;
constexpr int kSplitKMaxSplits = 16;
constexpr int64_t kSplitKMaxWsBytes = 64ll << 20;

static int splitk_splits(const tw_plan* p, int budget) {
  if (p->n_sub < 1 || p->subtiles.empty()) return 0;
  int min_steps = 1 << 30;
  for (const SubTile& st : p->subtiles) min_steps = std::min(min_steps, (int)st.kp_steps);
  return std::min({min_steps, budget / p->n_sub, kSplitKMaxSplits});
}

// Optional: without the workspace (too large, or the allocation fails) the
// plan simply never splits.
static int alloc_splitk_ws(tw_plan* plan) {
  const int S = splitk_splits(plan, plan->sm_count);
  if (S < 2 || plan->n_cond > 65535) return TW_OK;  // reduce grid: one row per grid.y
  const int64_t bytes = (int64_t)S * plan->n_cond * kSplitKMaxTokens * 4;
  if (bytes > kSplitKMaxWsBytes) return TW_OK;
  if (cudaMalloc(&plan->d_splitws, (size_t)bytes) != cudaSuccess) {
    (void)cudaGetLastError();
    plan->d_splitws = nullptr;
    return TW_OK;
  }
  plan->splitk_max = S;
  return TW_OK;
}

static void owner_split(tw_plan* plan) {
  const int G = plan->sm_budget;
  plan->cta_first.clear();
  plan->owner = plan->n_sub <= G && G <= kMaxCtas;
  plan->resident = false;
  if (!plan->owner) return;
  const std::vector<int32_t> c = split_counts(plan, G);
  plan->cta_first.assign(plan->n_sub + 1, 0);
  for (int i = 0; i < plan->n_sub; ++i) plan->cta_first[i + 1] = plan->cta_first[i] + c[i];
  int max_steps = 0;
  for (const SubTile& st : plan->subtiles) max_steps = std::max(max_steps, (int)st.kp_steps);
  plan->resident = max_steps <= kResSteps && !env_int("TW_NO_RESIDENT", 0);
}

// CTAs per sub-tile for G SMs (owner mode): proportional to the per-token
// cost weights, largest remainder, at least one each.
static std::vector<int32_t> split_counts(const tw_plan* plan, int G) {
  // weight (per token): k-steps, or (row-run plans) the stages' TMA issue
  // cost, plus a fixed per-unit share for the epilogue and pipeline fill,
  // which dominates short-K' sub-tiles (TEW 768x3072 keeps K' = 1 on one
  // tile: proportional-to-k-steps gave it 2 CTAs for all 8192 tokens)
  std::vector<int32_t> c(plan->n_sub, 1);
  std::vector<double> wt(plan->n_sub);
  double w = 0;
  for (int i = 0; i < plan->n_sub; ++i) {
    const SubTile& st = plan->subtiles[i];
    wt[i] = plan->runs ? plan->tile_cost[st.idx_row] + env_int("TW_RUN_FIX", 48)
                       : (double)st.kp_steps + 3.0;
    w += wt[i];
  }
  std::vector<std::pair<double, int>> frac;
  int used = 0;
  for (int i = 0; i < plan->n_sub; ++i) {
    const double q = (double)G * wt[i] / w;
    c[i] = std::max(1, (int)q);
    used += c[i];
    frac.push_back({q - (int)q, i});
  }
  std::stable_sort(frac.begin(), frac.end(),
                   [](const std::pair<double, int>& a, const std::pair<double, int>& b) {
                     return a.first > b.first;
                   });
  for (size_t t = 0; used < G && t < frac.size(); ++t, ++used) c[frac[t].second] += 1;
  while (used > G) {  // only when the max(1, .) floor overshot
    int big = (int)(std::max_element(c.begin(), c.end()) - c.begin());
    c[big] -= 1;
    --used;
  }
  return c;
}

extern "C" {

const char* tw_last_error(void) { return g_last_error.c_str(); }

int32_t tw_abi_version(void) { return 421; }

int tw_plan_create_cto(tw_plan** out, int32_t k, int32_t n, int32_t g, int32_t n_tiles,
                       const uint32_t* row_counts, const uint32_t* col_counts,
                       const uint32_t* row_offsets, int32_t max_rows,
                       const uint32_t* col_offsets, int32_t max_cols, const float* payload,
                       int32_t compute_dtype, int32_t schedule, int32_t row_runs, void* stream) {
  return tw_plan_create_cto_ex(out, k, n, g, n_tiles, row_counts, col_counts, row_offsets,
                               max_rows, col_offsets, max_cols, payload, compute_dtype, schedule,
                               row_runs, nullptr, 0, nullptr, stream);
}

int tw_plan_create_cto_ex(tw_plan** out, int32_t k, int32_t n, int32_t g, int32_t n_tiles,
                          const uint32_t* row_counts, const uint32_t* col_counts,
                          const uint32_t* row_offsets, int32_t max_rows,
                          const uint32_t* col_offsets, int32_t max_cols, const float* payload,
                          int32_t compute_dtype, int32_t schedule, int32_t row_runs,
                          const int32_t* row_groups, int32_t n_groups,
                          const int32_t* out_row_of_cond, void* stream) {
  g_last_error.clear();
  if (!out) return fail(TW_ERR_INVALID_INPUT, "out is null");
  *out = nullptr;
  if (k < 1 || n < 1 || g < 1) return fail(TW_ERR_INVALID_INPUT, "dims must be >= 1");
  // row groups (chained layout): bounds 0 = b0 < b1 < ... < b_n = k; the
  // row-run permutation then only moves rows within their group
  std::vector<int32_t> grp_of;
  if (row_groups) {
    if (n_groups < 1 || row_groups[0] != 0 || row_groups[n_groups] != k)
      return fail(TW_ERR_INVALID_INPUT, "row groups must cover [0, k) from 0 to k");
    grp_of.resize(k);
    for (int32_t gi = 0; gi < n_groups; ++gi) {
      if (row_groups[gi + 1] <= row_groups[gi])
        return fail(TW_ERR_INVALID_INPUT, "row group bounds must be strictly increasing");
      for (int32_t r = row_groups[gi]; r < row_groups[gi + 1]; ++r) grp_of[r] = gi;
    }
  }
  if (compute_dtype != kF16 && compute_dtype != kBF16 && compute_dtype != kF32)
    return fail(TW_ERR_INVALID_INPUT, "compute dtype must be fp16, bf16 or fp32");
  const bool split = compute_dtype == kF32;  // fp32 operands as fp16 hi + lo pairs
  if (split && (row_groups || out_row_of_cond))
    return fail(TW_ERR_INVALID_INPUT, "chained layouts need fp16 / bf16 compute");
  if (schedule != TW_SCHEDULE_LPT && schedule != TW_SCHEDULE_ROUND_ROBIN)
    return fail(TW_ERR_INVALID_INPUT, "unknown schedule %d", schedule);
  // CtoEncoding.__post_init__ (formats.py:94-127)
  if (n_tiles < 1) return fail(TW_ERR_CORRUPT, "encoding must contain at least one tile");
  if (!row_counts || !col_counts || !row_offsets || !col_offsets || !payload)
    return fail(TW_ERR_INVALID_INPUT, "null encoding array");
  uint32_t max_h = 0, max_w = 0;
  for (int i = 0; i < n_tiles; ++i) {
    if (row_counts[i] < 1 || col_counts[i] < 1)
      return fail(TW_ERR_CORRUPT, "every tile must keep at least one row and one column");
    max_h = std::max(max_h, row_counts[i]);
    max_w = std::max(max_w, col_counts[i]);
  }
  if ((uint32_t)max_rows < max_h)
    return fail(TW_ERR_CORRUPT, "row offsets narrower than the largest row count");
  if ((uint32_t)max_cols < max_w)
    return fail(TW_ERR_CORRUPT, "col offsets narrower than the largest col count");

  auto plan = new tw_plan();
  std::unique_ptr<tw_plan> guard(plan);
  plan->k = k;
  plan->n = n;
  plan->g = g;
  plan->n_tiles = n_tiles;
  plan->dtype = split ? kF16 : compute_dtype;  // what the kernels read
  plan->split = split;
  plan->schedule = schedule;
  if (int st = sm_count_of_current_device(&plan->sm_count)) return st;
  TW_CUDA(configure_gemm_kernels());
  cudaStream_t s = static_cast<cudaStream_t>(stream);

  // decode offsets: tile_rows / tile_cols (formats.py:138-158) and the column
  // order check of gemm_cto (executor.py:478-480)
  plan->tile_of_col.assign(n, -1);
  plan->tile_rows.resize(n_tiles);
  std::vector<std::vector<int32_t>> rows(n_tiles);
  int64_t prev_col = -1;
  for (int i = 0; i < n_tiles; ++i) {
    const uint32_t h = row_counts[i], w = col_counts[i];
    rows[i].resize(h);
    plan->tile_rows[i].assign(k, 0);
    int64_t prev = -1;
    for (uint32_t j = 0; j < h; ++j) {
      const int64_t r = (int64_t)j + row_offsets[(int64_t)i * max_rows + j];
      if (r <= prev || r >= k)
        return fail(TW_ERR_CORRUPT,
                    "tile %d: reconstructed rows are not strictly increasing within [0, %d)", i,
                    k);
      rows[i][j] = (int32_t)r;
      plan->tile_rows[i][r] = 1;
      prev = r;
    }
    plan->tile_first_cond.push_back((int32_t)plan->cond_cols.size());
    int64_t prevc = -1;
    for (uint32_t j = 0; j < w; ++j) {
      const int64_t c = (int64_t)j + col_offsets[(int64_t)i * max_cols + j];
      if (c <= prevc || c >= n)
        return fail(TW_ERR_CORRUPT,
                    "tile %d: reconstructed cols are not strictly increasing within [0, %d)", i,
                    n);
      if (c <= prev_col)
        return fail(TW_ERR_CORRUPT, "tile column ranges overlap or are out of order");
      plan->cond_cols.push_back((int32_t)c);
      plan->tile_of_col[c] = i;
      prevc = c;
      prev_col = c;
    }
    plan->kept_macs += (int64_t)h * w;
  }
  plan->n_cond = (int32_t)plan->cond_cols.size();

  // Narrow tiles (width <= 64) leave most of the 128-row UMMA M idle and
  // gather their kept rows once per tile.  Consecutive narrow tiles are
  // therefore merged into 128-column virtual tiles over the UNION of their
  // kept rows, the payload zero-filled where a tile does not keep a row: one
  // gather and one full-width MMA serve the whole group (2 x G = 64 at 50 %
  // rows: 0.75 K rows gathered instead of 2 x 0.5 K, at full M).  The
  // condensed column order is unchanged; the reference's tile structure
  // stays in tile_rows / tile_of_col (overlay checks) and kept_macs.
  int nt = n_tiles;
  std::vector<uint32_t> rc(row_counts, row_counts + n_tiles), cc(col_counts, col_counts + n_tiles);
  std::vector<int32_t> tfc = plan->tile_first_cond;
  const float* pay_in = payload;
  std::vector<float> pay_merged;
  // fp32 operands (compute dtype TW_F32): every value is split into an fp16
  // pair, hi = fp16(v) and lo = fp16(v - hi), and the product runs on the
  // fp16 tensor cores as A.W ~ A_hi.W_hi + A_hi.W_lo + A_lo.W_hi (the dropped
  // A_lo.W_lo is ~2^-22 relative): the activations enter as 2K rows
  // [A_hi^T; A_lo^T] (tw_plan_prepare) and every tile gathers its kept rows
  // three times -- row r with W_hi, row r again with W_lo, row K + r with
  // W_hi.  Same kernels; 3x the MACs; fp32-class accuracy on fp32 inputs.
  std::vector<float> pay_split;
  if (split) {
    if (2 * (int64_t)k >= (1 << 30)) return fail(TW_ERR_INVALID_INPUT, "k too large for fp32 split");
    int64_t pb = 0, total = 0;
    for (int i = 0; i < n_tiles; ++i) total += 3 * (int64_t)row_counts[i] * col_counts[i];
    pay_split.resize(std::max<int64_t>(total, 1));
    int64_t ob = 0;
    for (int i = 0; i < n_tiles; ++i) {
      const int32_t h = (int32_t)row_counts[i], w = (int32_t)col_counts[i];
      for (int32_t c = 0; c < w; ++c)
        for (int32_t j = 0; j < h; ++j) {
          const float v = payload[pb + (int64_t)c * h + j];
          const float hi = __half2float(__float2half_rn(v));
          const float lo = __half2float(__float2half_rn(v - hi));
          float* dst = pay_split.data() + ob + (int64_t)c * 3 * h;
          dst[j] = hi;
          dst[h + j] = lo;
          dst[2 * h + j] = hi;
        }
      std::vector<int32_t> r3(rows[i]);
      r3.insert(r3.end(), rows[i].begin(), rows[i].end());
      for (int32_t r : rows[i]) r3.push_back(r + k);
      rows[i].swap(r3);
      rc[i] = 3 * (uint32_t)h;
      pb += (int64_t)h * w;
      ob += 3 * (int64_t)h * w;
    }
    pay_in = pay_split.data();
  }
  {
    uint32_t wmax = 0;
    for (int i = 0; i < n_tiles; ++i) wmax = std::max(wmax, col_counts[i]);
    int gs = 1;
    while (gs * 2 * (int)wmax <= kBN) gs *= 2;
    if (gs > 1 && n_tiles > 1 && !split && !env_int("TW_NO_MERGE", 0)) {
      std::vector<int64_t> pb(n_tiles + 1, 0);
      for (int i = 0; i < n_tiles; ++i) pb[i + 1] = pb[i] + (int64_t)row_counts[i] * col_counts[i];
      const int nv = (n_tiles + gs - 1) / gs;
      std::vector<std::vector<int32_t>> vrows(nv);
      std::vector<uint32_t> vrc(nv), vcc(nv, 0);
      std::vector<int32_t> vtfc(nv);
      std::vector<int32_t> pos(k, -1);
      for (int v = 0; v < nv; ++v) {
        const int t0 = v * gs, t1 = std::min(n_tiles, t0 + gs);
        std::vector<int32_t> u;
        for (int t = t0; t < t1; ++t) u.insert(u.end(), rows[t].begin(), rows[t].end());
        std::sort(u.begin(), u.end());
        u.erase(std::unique(u.begin(), u.end()), u.end());
        vrows[v] = u;
        vrc[v] = (uint32_t)u.size();
        vtfc[v] = plan->tile_first_cond[t0];
        for (int t = t0; t < t1; ++t) vcc[v] += col_counts[t];
      }
      int64_t total = 0;
      for (int v = 0; v < nv; ++v) total += (int64_t)vrc[v] * vcc[v];
      pay_merged.assign(total, 0.0f);
      int64_t base = 0;
      for (int v = 0; v < nv; ++v) {
        const int t0 = v * gs, t1 = std::min(n_tiles, t0 + gs);
        const int32_t hv = (int32_t)vrc[v];
        for (int32_t j = 0; j < hv; ++j) pos[vrows[v][j]] = j;
        int32_t col = 0;
        for (int t = t0; t < t1; ++t) {
          const int32_t h = (int32_t)row_counts[t], w = (int32_t)col_counts[t];
          for (int32_t c = 0; c < w; ++c, ++col)
            for (int32_t j = 0; j < h; ++j)
              pay_merged[base + (int64_t)col * hv + pos[rows[t][j]]] =
                  payload[pb[t] + (int64_t)c * h + j];
        }
        base += (int64_t)hv * vcc[v];
      }
      nt = nv;
      rc.swap(vrc);
      cc.swap(vcc);
      tfc.swap(vtfc);
      rows.swap(vrows);
      pay_in = pay_merged.data();
    }
  }

  // gather lists: each tile's kept rows padded with -1 to whole stages
  int32_t kp = kBK;
  for (int i = 0; i < nt; ++i) kp = std::max(kp, round_up((int32_t)rc[i], kBK));
  plan->kp = kp;

  // Row-run layout.  Ordering the rows of A^T by their tile-membership
  // signature (Gray-code order of the set of tiles that keep the row) turns
  // every tile's kept rows into a handful of runs of consecutive positions,
  // which dense TMA boxes fetch at the full TMA rate instead of 16-byte
  // cp.async gathers.  That works for up to ~6 tiles; layers with more tiles
  // split them into G <= 4 contiguous groups, each with its own row order and
  // its own copy of A^T (the plan layout is then G x K rows).  The tiles' K'
  // order becomes position order (payload columns reordered to match), so
  // the natural-layout cp.async path and the run path accumulate in the same
  // order and stay bit-identical.  Used when the boxes per 64-row stage stay
  // few.
  const float* pay_src = pay_in;
  std::vector<float> pay_re;
  std::vector<int32_t> box_first;
  std::vector<uint32_t> boxes;
  std::vector<double> tile_cost(nt, 0.0);  // owner split weight (run path)
  // More than one copy (layers with > 6 tiles) measured no faster than the
  // gather on BERT 768x3072 (G = 3: 21.0 vs 20.9 us), so it is opt-in.
  const int max_copies = grp_of.empty() ? std::max(1, std::min(4, env_int("TW_RUN_COPIES", 1))) : 1;
  const double run_stage_w = env_int("TW_RUN_STAGE_W", 8);
  // TVW payloads (prune_tvw, patterns.py:645-717: 2:4 down every payload
  // column in K' order) can run on tcgen05.mma.sp (TW_SPARSE=1 at plan
  // creation) when the metadata fits its 32 TMEM columns (K' <= 1024: 2
  // sparse MMAs per 64-row stage).  The 2:4 groups are defined in K' order,
  // so such plans keep the natural row order (no row-run permutation).  Opt-in:
  // the kernel is bound by activation ingress, so halving the payload bytes
  // does not pay for losing the row-run TMA boxes or 256-token units on the
  // BERT shapes (profiles/r2_tvw_sparse.txt)
  bool sp_ok = !split && kp / kBK <= 16 && env_int("TW_SPARSE", 0) && !env_int("TW_NO_SPARSE", 0);
  for (int i = 0; i < nt && sp_ok; ++i) {
    const int32_t h = (int32_t)rc[i], w = (int32_t)cc[i];
    const float* t = pay_in;
    int64_t off = 0;
    for (int j = 0; j < i; ++j) off += (int64_t)rc[j] * cc[j];
    t += off;
    for (int32_t c = 0; c < w && sp_ok; ++c)
      for (int32_t g0 = 0; g0 < h && sp_ok; g0 += 4) {
        int nz = 0;
        for (int32_t j = g0; j < std::min(h, g0 + 4); ++j) nz += t[(int64_t)c * h + j] != 0.0f;
        sp_ok = nz <= 2;
      }
  }
  if (row_runs && !split && !sp_ok && k < (1 << 20) && !env_int("TW_NO_RUNS", 0)) {
    const int stride = kp / kBK + 1;
    for (int G = (nt + 5) / 6; G <= max_copies && G <= nt; ++G) {
      const int per = (nt + G - 1) / G;  // tiles per group
      if ((int64_t)G * k >= (1 << 23)) break;
      std::vector<int32_t> perm((size_t)G * k), inv((size_t)G * k);
      std::vector<std::vector<int32_t>> order(nt);
      std::vector<int32_t> bf((size_t)nt * stride, 0);
      std::vector<uint32_t> bx;
      std::vector<double> cost(nt, 0.0);
      int64_t stages = 0;
      for (int gi = 0; gi < G; ++gi) {
        const int t0 = gi * per, t1 = std::min(nt, t0 + per);
        const int nt = t1 - t0;
        if (nt <= 0) break;
        std::vector<int32_t> sig(k, 0);
        for (int i = t0; i < t1; ++i)
          for (int32_t r : rows[i]) sig[r] |= 1 << (i - t0);
        std::vector<int32_t> gray_rank(1 << nt);
        for (int v = 0; v < (1 << nt); ++v) gray_rank[v ^ (v >> 1)] = v;
        int32_t* pg = perm.data() + (size_t)gi * k;
        int32_t* ig = inv.data() + (size_t)gi * k;
        std::iota(pg, pg + k, 0);
        if (grp_of.empty())
          std::stable_sort(pg, pg + k, [&](int32_t x, int32_t y) {
            return gray_rank[sig[x]] < gray_rank[sig[y]];
          });
        else  // chained layout: Gray order inside each row group, groups in place
          std::stable_sort(pg, pg + k, [&](int32_t x, int32_t y) {
            return grp_of[x] != grp_of[y] ? grp_of[x] < grp_of[y]
                                           : gray_rank[sig[x]] < gray_rank[sig[y]];
          });
        for (int32_t q = 0; q < k; ++q) ig[pg[q]] = gi * k + q;  // global layout position
        for (int i = t0; i < t1; ++i) {
          const int32_t h = (int32_t)rows[i].size();
          order[i].resize(h);
          std::iota(order[i].begin(), order[i].end(), 0);
          std::stable_sort(order[i].begin(), order[i].end(), [&](int32_t x, int32_t y) {
            return ig[rows[i][x]] < ig[rows[i][y]];
          });
          const int nst = round_up(h, kBK) / kBK;
          for (int st = 0; st < nst; ++st) {
            const size_t nb0 = bx.size();
            bf[(size_t)i * stride + st] = (int32_t)nb0;
            // slots [64 st, 64 st + 64): maximal runs of consecutive
            // positions, then the padding (positions past the whole G x K
            // layout, zero-filled by the TMA); each run is cut into
            // power-of-two boxes
            int slot = st * kBK;
            const int end = st * kBK + kBK;
            while (slot < end) {
              int len = 1;
              int32_t p0 = slot < h ? ig[rows[i][order[i][slot]]] : G * k;
              if (slot < h) {
                while (slot + len < end && slot + len < h &&
                       ig[rows[i][order[i][slot + len]]] == p0 + len)
                  ++len;
              } else {
                len = end - slot;
              }
              int done = 0;
              while (done < len) {
                int hb = 64;
                while (hb > len - done) hb >>= 1;
                int code = 0;
                while ((1 << code) < hb) ++code;
                bx.push_back((uint32_t)((slot + done) - st * kBK) | ((uint32_t)code << 6) |
                             ((uint32_t)(p0 + done) << 9));
                done += hb;
              }
              slot += len;
            }
            cost[i] += run_stage_w + (double)(bx.size() - nb0);  // per-stage cost: fixed + per box
            ++stages;
          }
          for (int st = nst; st < stride; ++st) bf[(size_t)i * stride + st] = (int32_t)bx.size();
        }
      }
      const double per_stage = stages ? (double)bx.size() / (double)stages : 1e9;
      if (per_stage > (!grp_of.empty() ? 8.0 : G == 1 ? 4.0 : 3.0)) continue;
      plan->runs = true;
      plan->row_copies = G;
      plan->perm = perm;
      plan->inv = inv;
      plan->box_stride = stride;
      box_first.swap(bf);
      boxes.swap(bx);
      tile_cost.swap(cost);
      // K' order = position order: rows and payload columns follow
      int64_t total = 0;
      for (int i = 0; i < nt; ++i) total += (int64_t)rc[i] * cc[i];
      pay_re.resize(std::max<int64_t>(total, 1));
      int64_t base = 0;
      for (int i = 0; i < nt; ++i) {
        const int32_t h = (int32_t)rc[i], w = (int32_t)cc[i];
        std::vector<int32_t> r2(h);
        for (int32_t j = 0; j < h; ++j) r2[j] = rows[i][order[i][j]];
        rows[i].swap(r2);
        for (int32_t c = 0; c < w; ++c)
          for (int32_t j = 0; j < h; ++j)
            pay_re[base + (int64_t)c * h + j] = pay_in[base + (int64_t)c * h + order[i][j]];
        base += (int64_t)h * w;
      }
      pay_src = pay_re.data();
      break;
    }
  }
  std::vector<int32_t> gidx((size_t)nt * kp, -1);
  for (int i = 0; i < nt; ++i)
    std::copy(rows[i].begin(), rows[i].end(), gidx.begin() + (size_t)i * kp);

  // sub-tiles (128-column UMMA-M slices) and payload sources
  const int bn = kBN;
  plan->bn = bn;
  std::vector<SubTile> subs;
  std::vector<int64_t> src_base;
  std::vector<int32_t> src_ld;
  int64_t pbase = 0;
  for (int i = 0; i < nt; ++i) {
    const int32_t h = (int32_t)rc[i], w = (int32_t)cc[i];
    for (int32_t c0 = 0; c0 < w; c0 += bn) {
      SubTile st{};
      st.kp_steps = round_up(h, kBK) / kBK;
      st.idx_row = i;
      st.width = std::min(bn, w - c0);
      st.out_row = tfc[i] + c0;
      st.kept = h;
      subs.push_back(st);
      src_base.push_back(pbase + (int64_t)c0 * h);
      src_ld.push_back(h);
    }
    pbase += (int64_t)h * w;
  }
  plan->n_sub = (int32_t)subs.size();

  // Output row order (chained layout): condensed column c is written to
  // C'^T row out_row_of_cond[c].  Only permutations inside each sub-tile's
  // row block are allowed -- they cost nothing, the payload rows of the
  // sub-tile (UMMA M = TMEM lanes = output rows) are reordered instead.
  std::vector<float> pay_out;
  if (out_row_of_cond) {
    const int32_t nc = plan->n_cond;
    std::vector<int32_t> inv(nc, -1);
    for (int32_t c = 0; c < nc; ++c) {
      const int32_t r = out_row_of_cond[c];
      if (r < 0 || r >= nc || inv[r] >= 0)
        return fail(TW_ERR_INVALID_INPUT, "output order must be a permutation of the %d columns", nc);
      inv[r] = c;
    }
    pay_out.assign(pay_src, pay_src + pbase);
    for (size_t si = 0; si < subs.size(); ++si) {
      const SubTile& st = subs[si];
      const int i = st.idx_row;
      const int32_t h = (int32_t)rc[i];
      const int64_t tile_base = src_base[si] - (int64_t)(st.out_row - tfc[i]) * h;
      for (int32_t j = 0; j < st.width; ++j) {
        const int32_t c = inv[st.out_row + j];
        if (c < st.out_row || c >= st.out_row + st.width)
          return fail(TW_ERR_INVALID_INPUT,
                      "output order may only permute rows inside a 128-column sub-tile block");
        std::copy(pay_src + tile_base + (int64_t)(c - tfc[i]) * h,
                  pay_src + tile_base + (int64_t)(c - tfc[i] + 1) * h,
                  pay_out.begin() + tile_base + (int64_t)(st.out_row + j - tfc[i]) * h);
      }
    }
    std::vector<int32_t> cond2(nc);
    for (int32_t r = 0; r < nc; ++r) cond2[r] = plan->cond_cols[inv[r]];
    plan->cond_cols.swap(cond2);
    pay_src = pay_out.data();
  }
  std::vector<int32_t> order(plan->n_sub);
  std::iota(order.begin(), order.end(), 0);
  if (schedule == TW_SCHEDULE_LPT) {
    // executor.py:526 sorts tiles by (-macs, index); per token block the
    // MACs of a sub-tile are proportional to K' * width
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
      return (int64_t)subs[a].kept * subs[a].width > (int64_t)subs[b].kept * subs[b].width;
    });
  }
  // device table in visiting order with stage offsets and payload rows
  std::vector<int64_t> base2(plan->n_sub);
  std::vector<int32_t> ld2(plan->n_sub);
  int32_t off = 0;
  for (int i = 0; i < plan->n_sub; ++i) {
    plan->subtiles.push_back(subs[order[i]]);
    SubTile& st = plan->subtiles.back();
    st.stage_off = off;
    st.pay_row = i * bn;
    off += st.kp_steps;
    base2[i] = src_base[order[i]];
    ld2[i] = src_ld[order[i]];
  }
  (void)off;

  plan->tile_cost = tile_cost;
  plan->sm_budget = plan->sm_count;
  owner_split(plan);
  if (int st = alloc_splitk_ws(plan)) return st;

  plan->h_gidx = gidx;
  if (int st = upload(&plan->d_subtiles, plan->subtiles, s)) return st;
  if (int st = upload(&plan->d_gidx, gidx, s)) return st;
  if (plan->runs) {
    // the same lists as layout positions: the cp.async gather on a
    // plan-layout A^T (many units per CTA, where TMA boxes lose)
    std::vector<int32_t> gpos(gidx.size(), -1);
    for (int i = 0; i < nt; ++i) {
      const int g = std::min(plan->row_copies - 1, i / ((nt + plan->row_copies - 1) / plan->row_copies));
      for (size_t j = 0; j < rows[i].size(); ++j)
        gpos[(size_t)i * kp + j] = plan->inv[(size_t)g * k + rows[i][j]];
    }
    if (int st = upload(&plan->d_gidx_pos, gpos, s)) return st;
    if (int st = upload(&plan->d_perm, plan->perm, s)) return st;
    if (int st = upload(&plan->d_inv, plan->inv, s)) return st;
    if (int st = upload(&plan->d_box_first, box_first, s)) return st;
    if (int st = upload(&plan->d_boxes, boxes, s)) return st;
    plan->h_gidx_pos = gpos;
    plan->h_box_first = box_first;
    plan->h_boxes = boxes;
  }

  int64_t* d_src_base = nullptr;
  int32_t* d_src_ld = nullptr;
  float* d_src = nullptr;
  if (int st = upload(&d_src_base, base2, s)) return st;
  if (int st = upload(&d_src_ld, ld2, s)) return st;
  TW_CUDA(cudaMalloc(&d_src, std::max<int64_t>(pbase, 1) * sizeof(float)));
  TW_CUDA(cudaMemcpyAsync(d_src, pay_src, pbase * sizeof(float), cudaMemcpyHostToDevice, s));
  const size_t pay_bytes = (size_t)plan->n_sub * bn * kp * 2;
  TW_CUDA(cudaMalloc(&plan->d_payload, pay_bytes));
  PayloadArgs pa{d_src, d_src_base, d_src_ld, plan->d_subtiles, plan->d_payload,
                 plan->dtype, bn, kp, plan->n_sub};
  TW_CUDA(launch_build_payload(pa, s));
  TW_CUDA(cudaStreamSynchronize(s));
  cudaFree(d_src);
  cudaFree(d_src_base);
  cudaFree(d_src_ld);
  if (int st = make_map_2d(&plan->map_pay, plan->d_payload, plan->dtype, kp,
                           (uint64_t)plan->n_sub * bn, kp, kBK, bn))
    return st;
  if (sp_ok && bn == kBN) {
    // Compressed payload: per output column, the two values of each group of
    // four K' rows in K' order (a group with fewer nonzeros keeps zeros at
    // unused positions), K-major like the dense payload, kpc = K'_max / 2
    // rounded to whole 64-column boxes (one box = 2 stages).  Metadata: one
    // u32 per (sparse MMA i = 32 K' rows, TMEM lane); lane m % 8 + 16 (m / 16)
    // + 8 (k / 16) of row m = output column holds the 4-bit group codes
    // idx0 | idx1 << 2 of 16 K' rows at bit 16 ((m / 8) % 2) + k % 16
    // (scripts/sp_probe.cu, exact against a dense product).
    const int32_t kpc = round_up(kp / 2, kBK);
    const int32_t mcols = 2 * (kp / kBK);
    const bool bf = plan->dtype == kBF16;
    std::vector<uint16_t> pay_sp((size_t)plan->n_sub * bn * kpc, 0);
    std::vector<uint32_t> meta((size_t)plan->n_sub * mcols * 128, 0);
    for (int i = 0; i < plan->n_sub; ++i) {
      const SubTile& st = plan->subtiles[i];
      const int32_t h = ld2[i];
      for (int32_t c = 0; c < bn; ++c) {
        const float* col = c < st.width ? pay_src + base2[i] + (int64_t)c * h : nullptr;
        uint16_t* dst = pay_sp.data() + ((size_t)i * bn + c) * kpc;
        for (int32_t g0 = 0; g0 < kp; g0 += 4) {
          int pos[2] = {0, 1}, np = 0;
          for (int32_t j = 0; j < 4 && col; ++j)
            if (g0 + j < h && col[g0 + j] != 0.0f) pos[np++] = j;
          if (np == 1) {  // pair the nonzero with an unused position, idx0 < idx1
            if (pos[0] == 3) { pos[1] = 3; pos[0] = 2; } else { pos[1] = pos[0] + 1; }
          }
          for (int e = 0; e < 2; ++e) {
            const int32_t j = g0 + pos[e];
            const float v = col && j < h ? col[j] : 0.0f;
            dst[g0 / 2 + e] = (uint16_t)(bf ? float_to_bf16_bits(v) : float_to_half_bits(v));
          }
          const uint32_t nib = (uint32_t)pos[0] | (uint32_t)pos[1] << 2;
          const int32_t mi = g0 / 32, kk = g0 % 32;
          const int lane = c % 8 + 16 * (c / 16) + 8 * (kk / 16);
          const int bit = 16 * ((c / 8) % 2) + kk % 16;
          meta[((size_t)i * mcols + mi) * 128 + lane] |= nib << bit;
        }
      }
    }
    TW_CUDA(cudaMalloc(&plan->d_payload_sp, pay_sp.size() * 2));
    TW_CUDA(cudaMemcpyAsync(plan->d_payload_sp, pay_sp.data(), pay_sp.size() * 2,
                            cudaMemcpyHostToDevice, s));
    if (int st = upload(&plan->d_meta, meta, s)) return st;
    TW_CUDA(cudaStreamSynchronize(s));
    if (int st = make_map_2d(&plan->map_pay_sp, plan->d_payload_sp, plan->dtype, kpc,
                             (uint64_t)plan->n_sub * bn, kpc, kBK, bn))
      return st;
    if (int st = make_map_2d(&plan->map_pay_sp64, plan->d_payload_sp, plan->dtype, kpc,
                             (uint64_t)plan->n_sub * bn, kpc, kBK / 2, bn, 64))
      return st;
    plan->sparse = true;
    plan->kpc = kpc;
    plan->meta_cols = mcols;
  }
  plan->union_cols = plan->cond_cols;
  *out = guard.release();
  return TW_OK;
}

// ------------------------------------------------------------------ TWP1
// Device-native plan file: everything tw_plan_create_cto
// derives from a CTO encoding -- the validated column / row structure, the
// merged tiles, the row-run layout and box tables, the owner weights and the
// fp16/bf16 payload exactly as the kernels read it -- so a plan loads with
// plain uploads instead of re-validating, re-merging, re-permuting and
// re-converting the encoding (the CTO1 artifact, formats.py:239-304, stays
// the interchange format; this is its cached GPU form).

int tw_plan_save(const tw_plan* p, void* buf, uint64_t* len) {
  g_last_error.clear();
  if (!p || !len) return fail(TW_ERR_INVALID_INPUT, "null argument");
  if (p->has_overlay) return fail(TW_ERR_INVALID_INPUT, "save the plan before attaching an overlay");
  Writer w;
  w.pod(kTwpMagic);
  w.pod(kTwpVersion);
  for (int32_t v : {p->k, p->n, p->g, p->n_tiles, p->n_sub, p->bn, p->kp, p->n_cond, p->dtype,
                    p->schedule, (int32_t)p->runs, p->row_copies, p->box_stride,
                    (int32_t)p->split})
    w.pod(v);
  w.pod(p->kept_macs);
  w.vec(p->subtiles);
  w.vec(p->cond_cols);
  w.vec(p->tile_of_col);
  w.vec(p->tile_first_cond);
  std::vector<int32_t> counts, rows;
  for (const auto& flags : p->tile_rows) {
    int32_t c = 0;
    for (int32_t r = 0; r < p->k; ++r)
      if (flags[r]) { rows.push_back(r); ++c; }
    counts.push_back(c);
  }
  w.vec(counts);
  w.vec(rows);
  w.vec(p->h_gidx);
  w.vec(p->h_gidx_pos);
  w.vec(p->perm);
  w.vec(p->inv);
  w.vec(p->h_box_first);
  w.vec(p->h_boxes);
  w.vec(p->tile_cost);
  std::vector<uint8_t> pay((size_t)p->n_sub * p->bn * p->kp * 2);
  TW_CUDA(cudaMemcpy(pay.data(), p->d_payload, pay.size(), cudaMemcpyDeviceToHost));
  w.vec(pay);
  const uint64_t need = w.b.size();
  if (buf && *len >= need) std::memcpy(buf, w.b.data(), need);
  const bool small = buf && *len < need;
  *len = need;
  if (small) return fail(TW_ERR_INVALID_INPUT, "buffer too small: %llu bytes needed",
                         (unsigned long long)need);
  return TW_OK;
}

int tw_plan_load(tw_plan** out, const void* buf, uint64_t len, void* stream) {
  g_last_error.clear();
  if (!out || !buf) return fail(TW_ERR_INVALID_INPUT, "null argument");
  *out = nullptr;
  Reader r{static_cast<const uint8_t*>(buf), (size_t)len};
  if (r.pod<uint32_t>() != kTwpMagic) return fail(TW_ERR_CORRUPT, "not a TWP1 plan file");
  if (r.pod<uint32_t>() != kTwpVersion) return fail(TW_ERR_CORRUPT, "unsupported TWP1 version");
  auto plan = new tw_plan();
  std::unique_ptr<tw_plan> guard(plan);
  int32_t runs = 0, split = 0;
  for (int32_t* f : {&plan->k, &plan->n, &plan->g, &plan->n_tiles, &plan->n_sub, &plan->bn,
                     &plan->kp, &plan->n_cond, &plan->dtype, &plan->schedule, &runs,
                     &plan->row_copies, &plan->box_stride, &split})
    *f = r.pod<int32_t>();
  plan->runs = runs != 0;
  plan->split = split != 0;
  plan->kept_macs = r.pod<int64_t>();
  plan->subtiles = r.vec<SubTile>();
  plan->cond_cols = r.vec<int32_t>();
  plan->tile_of_col = r.vec<int32_t>();
  plan->tile_first_cond = r.vec<int32_t>();
  const std::vector<int32_t> counts = r.vec<int32_t>();
  const std::vector<int32_t> rows = r.vec<int32_t>();
  plan->h_gidx = r.vec<int32_t>();
  plan->h_gidx_pos = r.vec<int32_t>();
  plan->perm = r.vec<int32_t>();
  plan->inv = r.vec<int32_t>();
  plan->h_box_first = r.vec<int32_t>();
  plan->h_boxes = r.vec<uint32_t>();
  plan->tile_cost = r.vec<double>();
  const std::vector<uint8_t> pay = r.vec<uint8_t>();
  // structural validation (a corrupt file must not reach the kernels)
  const bool dims_ok = r.ok && plan->k >= 1 && plan->n >= 1 && plan->n_tiles >= 1 &&
                       plan->n_sub == (int32_t)plan->subtiles.size() && plan->bn == kBN &&
                       plan->kp >= kBK && plan->kp % kBK == 0 &&
                       (plan->dtype == kF16 || plan->dtype == kBF16) &&
                       (int32_t)plan->cond_cols.size() == plan->n_cond &&
                       (int32_t)plan->tile_of_col.size() == plan->n &&
                       (int32_t)counts.size() == plan->n_tiles &&
                       pay.size() == (size_t)plan->n_sub * kBN * plan->kp * 2 &&
                       plan->h_gidx.size() % (size_t)plan->kp == 0;
  if (!dims_ok) return fail(TW_ERR_CORRUPT, "TWP1 file is truncated or inconsistent");
  const int32_t nt = (int32_t)(plan->h_gidx.size() / plan->kp);
  for (const SubTile& st : plan->subtiles)
    if (st.idx_row < 0 || st.idx_row >= nt || st.kp_steps < 1 || st.kp_steps * kBK > plan->kp ||
        st.width < 1 || st.width > kBN || st.out_row < 0 || st.out_row + st.width > plan->n_cond ||
        st.pay_row < 0 || st.pay_row + kBN > plan->n_sub * kBN)
      return fail(TW_ERR_CORRUPT, "TWP1 sub-tile table out of range");
  for (int32_t v : plan->h_gidx)
    if (v < -1 || v >= plan->k_rows()) return fail(TW_ERR_CORRUPT, "TWP1 gather list out of range");
  if (plan->runs) {
    const int64_t rows_l = (int64_t)plan->k * plan->row_copies;
    if ((int64_t)plan->perm.size() != rows_l || (int64_t)plan->inv.size() != rows_l ||
        plan->h_gidx_pos.size() != plan->h_gidx.size() ||
        (int64_t)plan->h_box_first.size() != (int64_t)nt * plan->box_stride ||
        (int32_t)plan->tile_cost.size() != nt)
      return fail(TW_ERR_CORRUPT, "TWP1 row-run tables inconsistent");
    for (int32_t v : plan->perm)
      if (v < 0 || v >= plan->k) return fail(TW_ERR_CORRUPT, "TWP1 row order out of range");
    for (int32_t v : plan->h_gidx_pos)
      if (v < -1 || v >= rows_l) return fail(TW_ERR_CORRUPT, "TWP1 gather positions out of range");
    for (int32_t v : plan->h_box_first)
      if (v < 0 || v > (int32_t)plan->h_boxes.size())
        return fail(TW_ERR_CORRUPT, "TWP1 box table out of range");
    for (uint32_t b : plan->h_boxes)
      if ((int64_t)(b >> 9) > rows_l || (b & 63u) + (1u << ((b >> 6) & 7u)) > 64u)
        return fail(TW_ERR_CORRUPT, "TWP1 box out of range");
  }
  plan->tile_rows.assign(plan->n_tiles, std::vector<uint8_t>(plan->k, 0));
  size_t pos = 0;
  for (int32_t i = 0; i < plan->n_tiles; ++i) {
    if (counts[i] < 1 || pos + counts[i] > rows.size())
      return fail(TW_ERR_CORRUPT, "TWP1 tile rows inconsistent");
    for (int32_t j = 0; j < counts[i]; ++j, ++pos) {
      const int32_t row = rows[pos];
      if (row < 0 || row >= plan->k) return fail(TW_ERR_CORRUPT, "TWP1 tile row out of range");
      plan->tile_rows[i][row] = 1;
    }
  }
  if (int st = sm_count_of_current_device(&plan->sm_count)) return st;
  TW_CUDA(configure_gemm_kernels());
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (SubTile& st : plan->subtiles) st.k0 = 0;  // written per launch (split-K) only
  if (int st = upload(&plan->d_subtiles, plan->subtiles, s)) return st;
  if (int st = upload(&plan->d_gidx, plan->h_gidx, s)) return st;
  if (plan->runs) {
    if (int st = upload(&plan->d_gidx_pos, plan->h_gidx_pos, s)) return st;
    if (int st = upload(&plan->d_perm, plan->perm, s)) return st;
    if (int st = upload(&plan->d_inv, plan->inv, s)) return st;
    if (int st = upload(&plan->d_box_first, plan->h_box_first, s)) return st;
    if (int st = upload(&plan->d_boxes, plan->h_boxes, s)) return st;
  }
  TW_CUDA(cudaMalloc(&plan->d_payload, pay.size()));
  TW_CUDA(cudaMemcpyAsync(plan->d_payload, pay.data(), pay.size(), cudaMemcpyHostToDevice, s));
  TW_CUDA(cudaStreamSynchronize(s));
  if (int st = make_map_2d(&plan->map_pay, plan->d_payload, plan->dtype, plan->kp,
                           (uint64_t)plan->n_sub * kBN, plan->kp, kBK, kBN))
    return st;
  plan->sm_budget = plan->sm_count;
  if (plan->tile_cost.size() < (size_t)nt) plan->tile_cost.resize(nt, 0.0);
  owner_split(plan);
  if (int st = alloc_splitk_ws(plan)) return st;
  plan->union_cols = plan->cond_cols;
  *out = guard.release();
  return TW_OK;
}

int tw_plan_attach_overlay(tw_plan* p, int32_t k, int32_t n, int64_t nnz, const int64_t* col_ptr,
                           const int64_t* row_idx, const float* values, void* stream) {
  g_last_error.clear();
  if (!p) return fail(TW_ERR_INVALID_INPUT, "plan is null");
  if (k != p->k || n != p->n)
    return fail(TW_ERR_INVALID_INPUT, "overlay dims (%d, %d) do not match weights (%d, %d)", k,
                n, p->k, p->n);
  if (nnz < 0 || !col_ptr || (nnz > 0 && (!row_idx || !values)))
    return fail(TW_ERR_INVALID_INPUT, "malformed overlay arrays");
  if (col_ptr[0] != 0 || col_ptr[n] != nnz)
    return fail(TW_ERR_INVALID_INPUT, "malformed overlay column pointers");
  // overlap check of gemm_tew (executor.py:190-193) + union (executor.py:201-203)
  std::vector<int32_t> ov_cols;
  for (int32_t c = 0; c < n; ++c) {
    const int64_t lo = col_ptr[c], hi = col_ptr[c + 1];
    if (hi < lo)
      return fail(TW_ERR_INVALID_INPUT, "overlay column pointers must be non-decreasing");
    if (hi == lo) continue;
    ov_cols.push_back(c);
    const int t = p->tile_of_col[c];
    for (int64_t e = lo; e < hi; ++e) {
      const int64_t r = row_idx[e];
      if (r < 0 || r >= k || (e > lo && r <= row_idx[e - 1]))
        return fail(TW_ERR_INVALID_INPUT,
                    "overlay rows must be strictly increasing within a column");
      if (t >= 0 && p->tile_rows[t][r])
        return fail(TW_ERR_CONTRACT, "overlay entries overlap tile payload positions");
    }
  }
  std::vector<int32_t> uni;
  std::set_union(p->cond_cols.begin(), p->cond_cols.end(), ov_cols.begin(), ov_cols.end(),
                 std::back_inserter(uni));
  std::vector<int32_t> pos_of(n, -1);
  for (size_t i = 0; i < uni.size(); ++i) pos_of[uni[i]] = (int32_t)i;
  std::vector<int32_t> rowmap(p->n_cond);
  for (int32_t i = 0; i < p->n_cond; ++i) rowmap[i] = pos_of[p->cond_cols[i]];
  // K2 visits overlay columns in descending-nnz order (lane groups of a warp
  // then finish together); results do not depend on the order.
  std::stable_sort(ov_cols.begin(), ov_cols.end(), [&](int32_t a, int32_t b) {
    return col_ptr[a + 1] - col_ptr[a] > col_ptr[b + 1] - col_ptr[b];
  });
  // Workspace mode (tw_gemm_tew_ws): K1 writes the condensed TW result to a
  // scratch C'^T with its fast TMA epilogue and K2 moves every kept column
  // to its union row, adding the residual; kept columns without overlay
  // entries ride at the end of the list (0 entries: a plain copy).
  std::vector<int32_t> cond_of(n, -1);
  for (int32_t i = 0; i < p->n_cond; ++i) cond_of[p->cond_cols[i]] = i;
  const int32_t n_with_entries = (int32_t)ov_cols.size();
  for (int32_t c : p->cond_cols)
    if (col_ptr[c + 1] == col_ptr[c]) ov_cols.push_back(c);
  std::vector<int32_t> start(1, 0), rows, out_rows, acc, src_cond;
  std::vector<float> vals;
  for (int32_t c : ov_cols) {
    for (int64_t e = col_ptr[c]; e < col_ptr[c + 1]; ++e) {
      rows.push_back((int32_t)row_idx[e]);
      vals.push_back(values[e]);
    }
    if (p->split) {
      // fp32 plans: v.a ~ v_hi.a_hi + v_lo.a_hi + v_hi.a_lo (rows r, r, k + r)
      const size_t b = rows.size() - (size_t)(col_ptr[c + 1] - col_ptr[c]);
      const size_t e1 = rows.size();
      for (size_t e = b; e < e1; ++e) {
        const float hi = __half2float(__float2half_rn(vals[e]));
        const float lo = __half2float(__float2half_rn(vals[e] - hi));
        vals[e] = hi;
        rows.push_back(rows[e]);
        vals.push_back(lo);
        rows.push_back(rows[e] + k);
        vals.push_back(hi);
      }
    }
    start.push_back((int32_t)rows.size());
    out_rows.push_back(pos_of[c]);
    acc.push_back(p->tile_of_col[c] >= 0 ? 1 : 0);
    src_cond.push_back(cond_of[c]);
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // new device arrays go into a fresh set, swapped in only when every upload
  // succeeded (a failure frees them and leaves the plan's previous overlay)
  struct Guard {
    tw_plan::OvDev d;
    bool keep = false;
    ~Guard() { if (!keep) d.release(); }
  } ng;
  tw_plan::OvDev& nd = ng.d;
  if (int st = upload(&nd.union_rowmap, rowmap, s)) return st;
  if (int st = upload(&nd.start, start, s)) return st;
  if (int st = upload(&nd.rows, rows, s)) return st;
  if (int st = upload(&nd.vals, vals, s)) return st;
  if (int st = upload(&nd.out, out_rows, s)) return st;
  if (int st = upload(&nd.acc, acc, s)) return st;
  // Row-run plans: K2 reads A^T in the plan layout too (tw_gemm_tew_ex with
  // TW_LAYOUT_PLAN), through copy 0's positions (p->inv[r] < k).
  if (p->runs) {
    std::vector<int32_t> rows_pos(rows.size());
    for (size_t e = 0; e < rows.size(); ++e) rows_pos[e] = p->inv[rows[e]];
    if (int st = upload(&nd.rows_pos, rows_pos, s)) return st;
  }
  // K2 geometry: A^T block of T tokens for all K rows in shared memory;
  // packed (row, value) lists need row < 2^16.  Each column's list starts on
  // a group boundary and is zero-padded to whole groups of L entries
  // (L = T / 8 lanes per column), so every lane fetches its next entry with
  // one 4-byte load (1 instead of 2 per lane: less padding, 11.5 entries per
  // column on BERT).
  int32_t new_block_tokens = 0, new_ctas_per_sm = 0, new_tpl = 8;
  const int32_t kr = p->k_rows();  // rows of the kernels' A^T (2k for fp32 plans)
  if (kr < 65535 && !ov_cols.empty() && !env_int("TW_RESIDUAL_DIRECT", 0)) {
    int cps = 0;
    const int T = residual_block_tokens(kr, &cps);
    if (T > 0) {
      new_block_tokens = T;
      new_ctas_per_sm = cps;
      // entries per group = lanes per column: T / 8 (8 tokens per lane), or
      // T / 16 with 16 tokens per lane (T = 64)
      new_tpl = (T == 64 && env_int("TW_K2_TPL", 16) == 16) ? 16 : 8;
      const int G = T / new_tpl;
      const int row16 = T / 8;  // staged row length in 16-byte units
      std::vector<uint32_t> rv;
      std::vector<int4> meta(ov_cols.size());
      // Shared-memory bank classes: a staged row is T * 2 bytes, so
      // C = 64 / T rows share one 128-byte line and row r sits in class
      // r % C of it.  The kCols columns of a warp step read entry j of their
      // lists in one 16-byte load each; entries of random rows pile onto
      // some classes (30 % extra wavefronts measured at T = 32).  So each
      // column's list is interleaved by class (the row order within a class
      // kept), starting at class (column % kCols) % C: entry j of a warp step
      // then covers the classes evenly.  Classes follow the row the kernel
      // reads (layout position on row-run plans); the natural-order list uses
      // the same entry order, so both paths stay bit-identical.
      const int C = std::max(1, 64 / T), kCols = 32 / G;
      std::vector<int32_t> order;
      std::vector<std::vector<int32_t>> cls(C);
      for (size_t i = 0; i < ov_cols.size(); ++i) {
        const int32_t n = start[i + 1] - start[i];
        // w: condensed source row + 1 of a TW-kept column (0: residual only)
        meta[i] = make_int4((int32_t)rv.size(), n, out_rows[i], src_cond[i] + 1);
        order.clear();
        if (C > 1) {
          for (auto& q : cls) q.clear();
          for (int32_t e = start[i]; e < start[i + 1]; ++e) {
            const int32_t r = p->runs ? p->inv[rows[e]] : rows[e];
            cls[r % C].push_back(e);
          }
          std::vector<size_t> head(C, 0);
          // 16 tokens per lane: odd columns read their chunks in the other
          // order, so the class alternates per column pair
          int c = (int)((i % (size_t)kCols) / (new_tpl == 16 ? 2 : 1)) % C;
          for (int32_t t = 0; t < n; ++t) {
            while (head[c] >= cls[c].size()) c = (c + 1) % C;
            order.push_back(cls[c][head[c]++]);
            c = (c + 1) % C;
          }
        } else {
          for (int32_t e = start[i]; e < start[i + 1]; ++e) order.push_back(e);
        }
        for (int32_t e : order)
          rv.push_back(((uint32_t)rows[e] << 16) |
                       (p->dtype == kBF16 ? float_to_bf16_bits(vals[e]) : float_to_half_bits(vals[e])));
        while (rv.size() % G) rv.push_back((uint32_t)kr << 16);  // zero row, value 0
      }
      // A lane group keeps prefetching (two groups ahead) until the longest
      // list of its warp is done, so the lists at the end need that much
      // zero-row padding behind them.
      int32_t max_len = 0;
      for (size_t i = 0; i < ov_cols.size(); ++i) max_len = std::max(max_len, start[i + 1] - start[i]);
      rv.resize(rv.size() + ((size_t)(max_len + G - 1) / G + 2) * G, (uint32_t)kr << 16);
      // device form: value << 16 | row offset in 16-byte units of the staged
      // block (row * T * 2 / 16 < 2^16 since the block is <= 200 KB), so K2
      // forms the shared-memory address with one mask and one shift-add
      auto device_form = [row16](std::vector<uint32_t> v) {
        for (uint32_t& x : v) x = ((x & 0xffffu) << 16) | ((x >> 16) * (uint32_t)row16);
        return v;
      };
      if (int st = upload(&nd.rv, device_form(rv), s)) return st;
      if (int st = upload(&nd.meta, meta, s)) return st;
      if (p->runs) {
        for (uint32_t& x : rv)  // zero row k stays k (the staged block's appended row)
          if ((int32_t)(x >> 16) < k) x = ((uint32_t)p->inv[x >> 16] << 16) | (x & 0xffffu);
        if (int st = upload(&nd.rv_pos, device_form(rv), s)) return st;
      }
    }
  }
  TW_CUDA(cudaStreamSynchronize(s));
  p->ov.release();
  p->ov = nd;
  ng.keep = true;
  p->ov_block_tokens = new_block_tokens;
  p->ov_tpl = new_tpl;
  p->ov_ctas_per_sm = new_ctas_per_sm;
  p->ov_start = start;
  p->union_cols = uni;
  p->n_ov_cols = n_with_entries;
  p->n_ov_cols_all = (int32_t)ov_cols.size();
  p->nnz = nnz;
  p->has_overlay = true;
  return TW_OK;
}

int tw_plan_set_sm_budget(tw_plan* p, int32_t sms) {
  g_last_error.clear();
  if (!p) return fail(TW_ERR_INVALID_INPUT, "plan is null");
  if (sms < 0) return fail(TW_ERR_INVALID_INPUT, "sm budget must be >= 0");
  const int32_t b = sms == 0 ? p->sm_count : std::min(sms, p->sm_count);
  if (b != p->sm_budget) {
    p->sm_budget = b;
    owner_split(p);
  }
  return TW_OK;
}

int tw_plan_estimate(const tw_plan* p, int32_t sms, int64_t m, int64_t* stage_tokens,
                     int32_t* units) {
  if (!p || !stage_tokens || !units || m < 1) return fail(TW_ERR_INVALID_INPUT, "bad argument");
  const int G = sms <= 0 ? p->sm_count : std::min<int>(sms, p->sm_count);
  int64_t worst = 0;
  int32_t wu = 0;
  if (p->n_sub <= G && G <= kMaxCtas) {
    const std::vector<int32_t> c = split_counts(p, G);
    const int64_t ch = (m + 63) / 64;
    for (int s = 0; s < p->n_sub; ++s) {
      const int64_t len = ((ch + c[s] - 1) / c[s]) * 64;  // busiest CTA of the sub-tile
      const int64_t st = len * p->subtiles[s].kp_steps;
      const int32_t u = (int32_t)((len + kTN - 1) / kTN);
      if (st > worst) { worst = st; wu = u; }
    }
  } else {
    const int64_t n_units = (int64_t)p->n_sub * ((m + kTN - 1) / kTN);
    int32_t max_steps = 0;
    for (const SubTile& st : p->subtiles) max_steps = std::max(max_steps, st.kp_steps);
    wu = (int32_t)((n_units + G - 1) / G);
    worst = (int64_t)wu * kTN * max_steps;
  }
  *stage_tokens = worst;
  *units = wu;
  return TW_OK;
}

int tw_plan_get_info(const tw_plan* p, tw_plan_info* info) {
  if (!p || !info) return fail(TW_ERR_INVALID_INPUT, "null argument");
  info->k = p->k;
  info->n = p->n;
  info->g = p->g;
  info->n_tiles = p->n_tiles;
  info->n_sub = p->n_sub;
  info->bn = p->bn;
  info->kp = p->kp;
  info->n_condensed = p->n_cond;
  info->n_union = (int32_t)p->union_cols.size();
  info->compute_dtype = p->split ? kF32 : p->dtype;
  info->nnz = p->nnz;
  info->kept_macs_per_token = p->kept_macs + p->nnz;
  info->sm_count = p->sm_count;
  info->has_overlay = p->has_overlay ? 1 : 0;
  info->row_runs = p->runs ? 1 : 0;
  info->row_copies = p->runs ? p->row_copies : p->split ? 2 : 1;
  info->sm_budget = p->sm_budget;
  info->sparse_payload = p->sparse ? 1 : 0;
  info->splitk_max = p->d_splitws ? p->splitk_max : 0;
  info->splitk_max_tokens = (int32_t)kSplitKMaxTokens;
  info->splitk_min_steps = kSplitKMinSteps;
  int64_t steps = 0;
  for (const SubTile& st : p->subtiles) steps += st.kp_steps;
  info->stage_work = steps;
  return TW_OK;
}

int tw_plan_output_groups(const tw_plan* p, int32_t* bounds) {
  if (!p || !bounds) return fail(TW_ERR_INVALID_INPUT, "null argument");
  std::vector<int32_t> starts;
  for (const SubTile& st : p->subtiles) starts.push_back(st.out_row);
  std::sort(starts.begin(), starts.end());
  for (size_t i = 0; i < starts.size(); ++i) bounds[i] = starts[i];
  bounds[starts.size()] = p->n_cond;
  return TW_OK;
}

int tw_plan_condensed_columns(const tw_plan* p, int32_t* out) {
  if (!p || !out) return fail(TW_ERR_INVALID_INPUT, "null argument");
  std::copy(p->cond_cols.begin(), p->cond_cols.end(), out);
  return TW_OK;
}

int tw_plan_union_columns(const tw_plan* p, int32_t* out) {
  if (!p || !out) return fail(TW_ERR_INVALID_INPUT, "null argument");
  std::copy(p->union_cols.begin(), p->union_cols.end(), out);
  return TW_OK;
}

static int check_dtype(int32_t d) {
  if (d != kF32 && d != kF16 && d != kBF16)
    return fail(TW_ERR_INVALID_INPUT, "unknown dtype %d", d);
  return TW_OK;
}

static int check_io(const tw_plan* p, const void* x, int64_t m, int64_t ld_x, const void* ct,
                    int64_t ld_ct, int32_t out_dtype) {
  if (!p || !x || !ct) return fail(TW_ERR_INVALID_INPUT, "null argument");
  if (m < 1 || m > INT32_MAX) return fail(TW_ERR_INVALID_INPUT, "m must be in [1, 2^31)");
  if (ld_x < m || ld_x % 8 != 0)
    return fail(TW_ERR_INVALID_INPUT, "ld_at (%lld) must be >= m and a multiple of 8",
                (long long)ld_x);
  if (reinterpret_cast<uintptr_t>(x) % 16 != 0)
    return fail(TW_ERR_INVALID_INPUT, "A^T base must be 16-byte aligned");
  if (ld_ct < m) return fail(TW_ERR_INVALID_INPUT, "ld_ct must be >= m");
  return check_dtype(out_dtype);
}

// Diagnostic environment switches that shape a launch,
// read on every call (getenv is cheap) so tests can flip them per call.
struct LaunchEnv {
  int flags, no_tma_store, strided, force_owner, gran, split1, run_max_units, no_sparse,
      sparse_resident, splitk, pair;
  long long* trace;
  bool operator==(const LaunchEnv& o) const {
    return flags == o.flags && no_tma_store == o.no_tma_store && strided == o.strided &&
           force_owner == o.force_owner && gran == o.gran && split1 == o.split1 &&
           run_max_units == o.run_max_units && no_sparse == o.no_sparse &&
           sparse_resident == o.sparse_resident && splitk == o.splitk && pair == o.pair &&
           trace == o.trace;
  }
};

static LaunchEnv read_launch_env() {
  LaunchEnv e;
  e.flags = env_int("TW_DEBUG_FLAGS", 0);
  e.no_tma_store = env_int("TW_NO_TMA_STORE", 0);
  e.strided = env_int("TW_STRIDED", 0);
  e.force_owner = env_int("TW_OWNER", 0);
  e.gran = env_int("TW_GRAN", 64);
  e.split1 = env_int("TW_SPLIT1", 0) != 0;
  e.run_max_units = env_int("TW_RUN_MAX_UNITS", 16);
  // bit 0: TW_NO_SPARSE; bit 1: TW_SPARSE_SW128 (diagnostic payload variant)
  e.no_sparse = (env_int("TW_NO_SPARSE", 0) ? 1 : 0) | (env_int("TW_SPARSE_SW128", 0) ? 2 : 0);
  e.sparse_resident = env_int("TW_SPARSE_RESIDENT", 0);
  // split-K for small M: -1 = when M <= kSplitKMaxTokens, 0 = never, 1 = forced
  e.splitk = env_int("TW_SPLITK", -1);
  // paired units on streamed run-path plans (two units share each payload stage)
  e.pair = env_int("TW_PAIR", 0);
  e.trace = g_trace;
  return e;
}

static int build_tw_launch(const tw_plan* p, const void* x, int64_t m, int64_t ld_x, void* ct,
                           int64_t ld_ct, int32_t out_dtype, const int32_t* rowmap,
                           int64_t out_rows, bool plan_layout, const LaunchEnv& env,
                           TwLaunch& L) {
  GemmArgs& a = L.a;
  a = GemmArgs{};
  a.subtiles = p->d_subtiles;
  a.x = x;
  a.ld_x = ld_x;
  a.gidx = p->d_gidx;
  a.kp = p->kp;
  a.in_dtype = p->dtype;
  a.rowmap = rowmap;
  a.out = ct;
  a.ld_out = ld_ct;
  a.out_dtype = out_dtype;
  a.M = (int32_t)m;
  a.n_sub = p->n_sub;
  a.flags = env.flags;
  a.trace = g_trace;
  const int esz = out_dtype == kF32 ? 4 : 2;
  a.vec_ok = ((ld_ct * esz) % 16 == 0 && reinterpret_cast<uintptr_t>(ct) % 16 == 0) ? 1 : 0;
  a.vec32_ok = ((ld_ct * esz) % 32 == 0 && reinterpret_cast<uintptr_t>(ct) % 32 == 0) ? 1 : 0;
  // condensed 16-bit output: 32 x 16 blocks leave through TMA 2-D stores
  CUtensorMap& map_out = L.map_out;
  std::memset(&map_out, 0, sizeof(map_out));
  a.use_tma_store = 0;
  if (esz == 2 && a.vec_ok && rowmap == nullptr && !env.no_tma_store) {
    if (make_map_2d(&map_out, ct, out_dtype, (uint64_t)m, (uint64_t)out_rows, (uint64_t)ld_ct,
                    16, 32, 32) == TW_OK)
      a.use_tma_store = 1;
    g_last_error.clear();
  }
  // Owner mode (one sub-tile + token range per CTA) whenever the sub-tiles fit
  // on the SMs; otherwise 256-token units strided over the CTAs.
  int& grid = L.grid;
  WorkTable& work = L.work;
  std::memset(&work, 0, sizeof(work));  // the cached launch is rebuilt in place
  bool owner = p->owner && !env.strided;
  // sparse tensor-core path: owner mode with the compressed payload resident
  int max_steps_all = 0;
  for (const SubTile& st : p->subtiles) max_steps_all = std::max(max_steps_all, (int)st.kp_steps);
  // (metadata: 2 TMEM columns per stage, loaded once per CTA -> owner mode);
  // the compressed payload streams with each stage (4-stage ring) unless
  // TW_SPARSE_RESIDENT=1 keeps it resident (3 stages: measured slower)
  const bool sparse = p->sparse && owner && !(env.no_sparse & 1);
  L.sparse = sparse;
  L.sparse_resident = sparse && env.sparse_resident &&
                      (max_steps_all + 1) / 2 <= kResSteps;
  if (owner && !p->resident && !sparse && !env.force_owner) {
    // Streamed payload: both modes re-stream a sub-tile's payload per unit,
    // so pick the one whose busiest CTA does less (k-steps x tokens).
    int64_t own = 0, max_steps = 0;
    for (int sidx = 0; sidx < p->n_sub; ++sidx) {
      const int c = p->cta_first[sidx + 1] - p->cta_first[sidx];
      const int64_t toks = ((m + c - 1) / c + 63) / 64 * 64;
      own = std::max<int64_t>(own, (int64_t)p->subtiles[sidx].kp_steps * toks);
      max_steps = std::max<int64_t>(max_steps, p->subtiles[sidx].kp_steps);
    }
    const int64_t units = (int64_t)p->n_sub * ((m + kTN - 1) / kTN);
    const int64_t strided = (units + p->sm_budget - 1) / p->sm_budget * kTN * max_steps;
    if (strided < own) owner = false;
  }
  // split-K for small M (see kSplitKMaxTokens): S CTAs per sub-tile, each a
  // contiguous range of its k-steps, one unit of all M tokens, fp32 partial
  // products into the plan's workspace (partial j of condensed row r at row
  // j * n_cond + r); splitk_reduce then writes the caller's output
  L.splitk = 0;
  int S = 0;
  if (p->d_splitws && !sparse && m <= kSplitKMaxTokens &&
      (env.splitk > 0 || (env.splitk < 0 && max_steps_all >= kSplitKMinSteps)))
    S = std::min(splitk_splits(p, p->sm_budget), (int)p->splitk_max);
  if (S >= 2) {
    a.owner = 1;
    grid = p->n_sub * S;
    const int64_t ldw = (m + 15) / 16 * 16;
    const int32_t usz = (int32_t)std::min<int64_t>(kTN, (m + 63) / 64 * 64);
    for (int sidx = 0; sidx < p->n_sub; ++sidx) {
      const SubTile& st = p->subtiles[sidx];
      for (int j = 0; j < S; ++j) {
        CtaWork& w = work.w[sidx * S + j];
        const int k0 = st.kp_steps * j / S, k1 = st.kp_steps * (j + 1) / S;
        w.kp_steps = k1 - k0;
        w.k0 = k0;
        w.idx_row = st.idx_row;
        w.pay_row = st.pay_row;
        w.width = st.width;
        w.out_row = j * p->n_cond + st.out_row;
        w.b = 0;
        w.e = (int32_t)m;
        w.usz = usz;
      }
    }
    a.out = p->d_splitws;
    a.ld_out = ldw;
    a.out_dtype = kF32;
    a.rowmap = nullptr;
    a.vec_ok = 1;
    a.vec32_ok = 1;
    a.use_tma_store = 0;
    L.splitk = S;
    SplitKArgs& r = L.red;
    r.ws = p->d_splitws;
    r.splits = S;
    r.split_stride = (int64_t)p->n_cond * ldw;
    r.ld_ws = ldw;
    r.rows = p->n_cond;
    r.M = (int32_t)m;
    r.out = ct;
    r.ld_out = ld_ct;
    r.out_dtype = out_dtype;
    r.rowmap = rowmap;
  } else if (owner) {
    a.owner = 1;
    int gran = env.gran;
    if (gran != 16 && gran != 32 && gran != 64) gran = 64;
    const bool split_single = env.split1;
    grid = p->cta_first.back();
    if (grid > kMaxCtas) return fail(TW_ERR_INVALID_INPUT, "owner grid %d > %d", grid, kMaxCtas);
    // CTA j of sub-tile s (c_s CTAs): tokens cut into c_s ranges on `gran`
    // boundaries, processed in units of <= kTN tokens with the remainder last
    // (shortest final epilogue); split_single halves a one-unit range so the
    // first half's epilogue overlaps the second half's mainloop.
    const int64_t ch = (m + gran - 1) / gran;
    for (int sidx = 0; sidx < p->n_sub; ++sidx) {
      const SubTile& st = p->subtiles[sidx];
      const int c0 = p->cta_first[sidx], c = p->cta_first[sidx + 1] - c0;
      for (int j = 0; j < c; ++j) {
        CtaWork& w = work.w[c0 + j];
        w.kp_steps = st.kp_steps;
        w.idx_row = st.idx_row;
        w.pay_row = st.pay_row;
        w.width = st.width;
        w.out_row = st.out_row;
        const int64_t b = (int64_t)j * ch / c * gran;
        const int64_t e = std::min<int64_t>(m, (int64_t)(j + 1) * ch / c * gran);
        const int64_t len = std::max<int64_t>(0, e - b);
        // sparse: the metadata sits in TMEM columns 480-511, inside the second
        // accumulator buffer (256-511), so units that can land there (every
        // odd unit of a CTA with two or more) stop at kSparseMaxTokens; a
        // one-unit range keeps the full 256 tokens in buffer 0
        const int64_t cap = sparse && len > kTN ? kSparseMaxTokens : kTN;
        int64_t n = (len + cap - 1) / cap;
        if (split_single && n == 1 && len >= 2 * gran) n = 2;
        w.b = (int32_t)b;
        w.e = (int32_t)std::max(b, e);
        w.usz = n > 0 ? (int32_t)std::min<int64_t>(cap, ((len + n - 1) / n + gran - 1) / gran * gran)
                      : 0;
      }
    }
  } else {
    a.owner = 0;
    a.n_units = (int32_t)(p->n_sub * ((m + kTN - 1) / kTN));
    grid = std::min(a.n_units, p->sm_budget);
    // L2-aware unit order: a wave of `grid` units touches sg payloads and
    // about grid / sg token blocks of A^T; choose the largest sg whose
    // working set fits in ~3/4 of L2 (126 MB), so payloads and A^T blocks
    // are fetched from DRAM about once per group instead of once per wave
    // (configs[4]: 64 payloads of 2 MB = all of L2 when every wave touches
    // every sub-tile)
    const double l2 = 0.85 * 126e6;
    const double pay_b = (double)kBN * p->kp * 2;                 // one sub-tile's payload
    const double blk_b = (double)p->k * p->row_copies * kTN * 2;  // one token block of A^T
    int sg = p->n_sub;
    if (!env_int("TW_NO_SUBGROUP", 0)) {
      // working set of one wave: sg payloads + the ~grid / sg token blocks
      auto ws = [&](int g) { return g * pay_b + (std::ceil((double)grid / g) + 1.0) * blk_b; };
      int best = p->n_sub;
      for (int g = p->n_sub; g >= 1; --g)
        if (ws(g) < ws(best)) best = g;
      while (sg > 1 && ws(sg) > l2) --sg;  // the largest group that fits ...
      if (ws(sg) > l2) sg = best;          // ... else the smallest working set
      // prefer whole waves of distinct sub-tiles: round down to a divisor-friendly size
      if (sg < p->n_sub) {
        const int ngrp = (p->n_sub + sg - 1) / sg;
        sg = (p->n_sub + ngrp - 1) / ngrp;
      }
    }
    a.sub_group = std::max(1, sg);
  }
  bool& resident = L.resident;
  resident = a.owner && (sparse ? L.sparse_resident : p->resident);
  if (sparse) {
    // 1: 32-column SW64 payload slices per stage; 2 (TW_SPARSE_SW128=1,
    // diagnostics): the 64-column SW128 box per stage, half of it used
    a.sparse = (env.no_sparse & 2) ? 2 : 1;
    a.meta = p->d_meta;
    a.meta_cols = p->meta_cols;
  }
  // Plan-layout input: TMA row runs unless a CTA has many units.  Runs win
  // where the gather is L2->SM-bound (3072x768 21.4 -> 17.3 us; VGG conv4_2
  // at 6 units per CTA 218 -> 160 us); on long HBM-streaming ranges (VGG
  // conv1_2: 85 units per CTA) the per-chunk TMA boxes revisit each DRAM row
  // four times and the cp.async gather by layout position is faster
  // (545 vs 860 us).  Row runs with <= 2 units per CTA
  // stream the payload: the TMA boxes need the deeper 4 x 48 KB ring more
  // than the payload needs residency (768^2: 9.3 -> 8.7 us).
  bool use_runs = false;
  int64_t min_units = 0;  // owner mode: fewest units of an active CTA
  if (plan_layout && p->runs) {
    int64_t max_units = 0;
    if (a.owner) {
      min_units = INT64_MAX;
      for (int i = 0; i < grid; ++i)
        if (work.w[i].usz > 0) {
          const int64_t u = (work.w[i].e - work.w[i].b + work.w[i].usz - 1) / work.w[i].usz;
          max_units = std::max<int64_t>(max_units, u);
          min_units = std::min<int64_t>(min_units, u);
        }
      if (min_units == INT64_MAX) min_units = 0;
    } else {
      max_units = (a.n_units + grid - 1) / grid;
    }
    use_runs = max_units <= env.run_max_units;
    if (use_runs && max_units <= 2) resident = false;
    if (!use_runs) a.gidx = p->d_gidx_pos;
  }
  // row-run path: x is in the plan's permuted row layout
  RunMaps& run_maps = L.maps;
  std::memset(&run_maps, 0, sizeof(run_maps));
  a.runs = 0;
  if (use_runs) {
    a.runs = 1;
    a.box_first = p->d_box_first;
    a.boxes = p->d_boxes;
    a.box_stride = p->box_stride;
    for (int c = 0; c < kRunMaps && a.runs; ++c)
      if (make_map_2d(&run_maps.m[c], x, p->dtype, (uint64_t)m,
                      (uint64_t)p->k * p->row_copies, (uint64_t)ld_x, 64, 1u << c, 128) != TW_OK)
        return TW_ERR_INVALID_INPUT;
  }
  // paired units: owner CTAs (one sub-tile each) on the streamed run path
  // (every active CTA has two units or more: a single unit gains nothing and
  // would only run on the shallower 2-slot ring)
  a.pair = (env.pair && a.owner && !resident && a.runs && !sparse && !L.splitk && min_units >= 2)
               ? 1 : 0;
  return TW_OK;
}

// K1 launch with the per-call host work (tensor-map encodes, the owner-mode
// work table, the row-run decision) cached per plan for the last geometry:
// repeated calls on the same buffers (a serving loop, the reference API in a
// loop) pay only the launch.
// The plan's cached launch for this geometry (built on a key miss); the
// caller holds p->launch_mu.
static int get_launch(const tw_plan* p, const void* x, int64_t m, int64_t ld_x, void* ct,
                      int64_t ld_ct, int32_t out_dtype, const int32_t* rowmap, int64_t out_rows,
                      bool plan_layout, const LaunchEnv& env, const TwLaunch** out) {
  tw_plan::Key key;
  std::memset(&key, 0, sizeof(key));  // padding too: keys compare with memcmp
  key.x = x; key.m = m; key.ld_x = ld_x; key.ct = ct; key.ld_ct = ld_ct;
  key.out_dtype = out_dtype; key.rowmap = rowmap; key.out_rows = out_rows;
  key.plan_layout = plan_layout; key.budget = p->sm_budget;
  key.flags = env.flags; key.no_tma_store = env.no_tma_store; key.strided = env.strided;
  key.force_owner = env.force_owner; key.gran = env.gran; key.split1 = env.split1;
  key.run_max_units = env.run_max_units; key.no_sparse = env.no_sparse;
  key.sparse_resident = env.sparse_resident; key.splitk = env.splitk; key.pair = env.pair;
  key.trace = env.trace;
  if (!(p->cache_valid && p->cache_key == key)) {
    p->cache_valid = false;
    if (int st = build_tw_launch(p, x, m, ld_x, ct, ld_ct, out_dtype, rowmap, out_rows,
                                 plan_layout, env, p->cache))
      return st;
    p->cache_key = key;
    p->cache_valid = true;
  }
  *out = &p->cache;
  return TW_OK;
}

// The payload tensor map a launch reads (dense, or the compressed sparse one).
static const CUtensorMap& launch_payload_map(const tw_plan* p, const TwLaunch& L) {
  return !L.sparse                         ? p->map_pay
         : (L.resident || L.a.sparse == 2) ? p->map_pay_sp
                                           : p->map_pay_sp64;
}

static int run_tw(const tw_plan* p, const void* x, int64_t m, int64_t ld_x, void* ct,
                  int64_t ld_ct, int32_t out_dtype, const int32_t* rowmap, int64_t out_rows,
                  cudaStream_t s, bool plan_layout = false) {
  const LaunchEnv env = read_launch_env();
  std::lock_guard<std::mutex> lock(p->launch_mu);
  const TwLaunch* Lp = nullptr;
  if (int st = get_launch(p, x, m, ld_x, ct, ld_ct, out_dtype, rowmap, out_rows, plan_layout, env,
                          &Lp))
    return st;
  const TwLaunch& L = *Lp;
  if (env.flags & 64) return TW_OK;  // diagnostics: host work only, no launch
  TW_CUDA(launch_tw_gemm(launch_payload_map(p, L), L.map_out, L.maps, L.a, L.work, L.resident,
                         L.grid, s));
  if (L.splitk) TW_CUDA(launch_splitk_reduce(L.red, s));
  return TW_OK;
}

int tw_gemm(const tw_plan* p, const void* x, int64_t m, int64_t ld_x, void* ct, int64_t ld_ct,
            int32_t out_dtype, void* stream) {
  g_last_error.clear();
  if (int st = check_io(p, x, m, ld_x, ct, ld_ct, out_dtype)) return st;
  return run_tw(p, x, m, ld_x, ct, ld_ct, out_dtype, nullptr, p->n_cond,
                static_cast<cudaStream_t>(stream));
}

// K1 of n independent plans in one launch; outs[i] (ld_outs[i]) receive plan
// i's condensed C'^T, or with tew_scatter its union rows (the overlay's
// rowmap), exactly as run_tw would write them.
static int group_k1(const tw_plan* const* plans, int32_t n, const void* const* xs,
                    const int64_t* ld_xs, const int32_t* x_layouts, void* const* outs,
                    const int64_t* ld_outs, const bool* tew_scatter, int64_t m, int32_t out_dtype,
                    cudaStream_t stream) {
  if (!plans || !xs || !ld_xs || !outs || !ld_outs || n < 1)
    return fail(TW_ERR_INVALID_INPUT, "null argument");
  if (n > kMaxGroup) return fail(TW_ERR_INVALID_INPUT, "at most %d plans per group launch", kMaxGroup);
  LaunchEnv env = read_launch_env();
  env.splitk = 0;  // one launch for every plan: no second (reduce) kernel per plan
  GroupArgs g;
  std::memset(&g, 0, sizeof(g));
  WorkTable work;
  std::memset(&work, 0, sizeof(work));
  int grid = 0;
  // (plan, local CTA, estimated work): CTAs are launched heaviest first, so
  // under programmatic dependent launch -- where a step's CTAs take SMs in
  // launch order as the previous step's free them -- the longest ones start
  // earliest
  struct CtaRef { int p, c; double w; CtaWork work; bool owner; };
  std::vector<CtaRef> ctas;
  for (int i = 0; i < n; ++i) {
    const tw_plan* p = plans[i];
    if (int st = check_io(p, xs[i], m, ld_xs[i], outs[i], ld_outs[i], out_dtype)) return st;
    const int32_t lay = x_layouts ? x_layouts[i] : TW_LAYOUT_NATURAL;
    if (lay != TW_LAYOUT_NATURAL && lay != TW_LAYOUT_PLAN)
      return fail(TW_ERR_INVALID_INPUT, "unknown activation layout %d", lay);
    if (lay == TW_LAYOUT_PLAN && !p->runs)
      return fail(TW_ERR_INVALID_INPUT, "plan %d has no row-run layout", i);
    for (int j = 0; j < i; ++j)
      if (plans[j] == p) return fail(TW_ERR_INVALID_INPUT, "a plan may appear once per group launch");
    const bool scatter = tew_scatter && tew_scatter[i];
    std::lock_guard<std::mutex> lock(p->launch_mu);
    const TwLaunch* Lp = nullptr;
    if (int st = get_launch(p, xs[i], m, ld_xs[i], outs[i], ld_outs[i], out_dtype,
                            scatter ? p->ov.union_rowmap : nullptr,
                            scatter ? (int64_t)p->union_cols.size() : p->n_cond,
                            lay == TW_LAYOUT_PLAN, env, &Lp))
      return st;
    const TwLaunch& L = *Lp;
    if (grid + L.grid > kMaxCtas || L.grid > 255)
      return fail(TW_ERR_INVALID_INPUT, "group launch needs %d CTAs (> %d): set SM budgets",
                  grid + L.grid, kMaxCtas);
    g.map_pay[i] = launch_payload_map(p, L);
    g.map_out[i] = L.map_out;
    g.run_maps[i] = L.maps;
    g.args[i] = L.a;
    g.resident[i] = L.resident ? 1 : 0;
    g.plan_ctas[i] = L.grid;
    for (int c = 0; c < L.grid; ++c) {
      double w = 0.0;
      if (L.a.owner) {
        const CtaWork& cw = L.work.w[c];
        const int units = cw.usz > 0 ? (cw.e - cw.b + cw.usz - 1) / cw.usz : 0;
        w = (double)(cw.e - cw.b) * cw.kp_steps + 3000.0 / 4.0 * units;  // group.py cost model
      }
      // the work entry is copied while the plan's launch cache is locked
      ctas.push_back({i, c, w, L.a.owner ? L.work.w[c] : CtaWork{}, L.a.owner != 0});
    }
    grid += L.grid;
  }
  if (!env_int("TW_GROUP_PLAN_ORDER", 0))
    std::stable_sort(ctas.begin(), ctas.end(),
                     [](const CtaRef& a, const CtaRef& b) { return a.w > b.w; });
  for (int b = 0; b < grid; ++b) {
    const CtaRef& r = ctas[b];
    g.cta_plan[b] = (int8_t)r.p;
    g.cta_local[b] = (uint8_t)r.c;
    if (r.owner) work.w[b] = r.work;
  }
  g.n = n;
  if (env.flags & 64) return TW_OK;
  TW_CUDA(launch_tw_gemm_group(g, work, grid, stream));
  return TW_OK;
}

int tw_gemm_group(const tw_plan* const* plans, int32_t n, const void* const* xs,
                  const int64_t* ld_xs, const int32_t* x_layouts, void* const* cts,
                  const int64_t* ld_cts, int64_t m, int32_t out_dtype, void* stream) {
  g_last_error.clear();
  return group_k1(plans, n, xs, ld_xs, x_layouts, cts, ld_cts, nullptr, m, out_dtype,
                  static_cast<cudaStream_t>(stream));
}

static int launch_k2(const tw_plan* p, const void* x, int64_t m, int64_t ld_x, void* ct,
                     int64_t ld_ct, int32_t out_dtype, const void* src, int64_t ld_src,
                     int32_t n_cols, const int4* meta, bool acc_all, cudaStream_t s,
                     bool plan_layout);
static void build_k2_args(const tw_plan* p, const void* x, int64_t m, int64_t ld_x, void* ct,
                          int64_t ld_ct, int32_t out_dtype, const void* src, int64_t ld_src,
                          int32_t n_cols, const int4* meta, bool acc_all, bool plan_layout,
                          ResidualArgs& r);

int tw_gemm_tew_group(const tw_plan* const* plans, int32_t n, const void* const* xs,
                      const int64_t* ld_xs, const int32_t* x_layouts, void* const* cts,
                      const int64_t* ld_cts, void* const* workspaces, const uint64_t* ws_bytes,
                      int64_t m, int32_t out_dtype, void* stream) {
  g_last_error.clear();
  if (!plans || !cts || !ld_cts || n < 1 || n > kMaxGroup)
    return fail(TW_ERR_INVALID_INPUT, "bad group arguments");
  // K1 of every plan in one launch -- into its workspace (condensed, TMA
  // epilogue) when it needs one, else straight into its union rows -- then
  // K2 of every plan, one after another on the same stream (each K2 takes
  // the whole GPU; programmatic dependent launch chains them)
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::vector<void*> k1_out(n);
  std::vector<int64_t> k1_ld(n);
  std::vector<uint8_t> scatter(n);
  for (int i = 0; i < n; ++i) {
    const tw_plan* p = plans[i];
    if (!p || !p->has_overlay) return fail(TW_ERR_INVALID_INPUT, "plan %d has no overlay", i);
    uint64_t need = 0;
    if (int st = tw_plan_tew_workspace_bytes(p, m, out_dtype, &need)) return st;
    void* ws = need && workspaces ? workspaces[i] : nullptr;
    if (need && (!ws || !ws_bytes || ws_bytes[i] < need || reinterpret_cast<uintptr_t>(ws) % 16))
      return fail(TW_ERR_INVALID_INPUT, "plan %d: workspace must hold %llu bytes, 16-byte aligned",
                  i, (unsigned long long)need);
    k1_out[i] = ws ? ws : cts[i];
    k1_ld[i] = ws ? (m + 7) / 8 * 8 : ld_cts[i];
    scatter[i] = ws ? 0 : 1;
  }
  bool scb[kMaxGroup];
  for (int i = 0; i < n; ++i) scb[i] = scatter[i] != 0;
  if (int st = group_k1(plans, n, xs, ld_xs, x_layouts, k1_out.data(), k1_ld.data(), scb, m,
                        out_dtype, s))
    return st;
  // K2 of every plan: one launch over all of them when every plan has the
  // staged kernel (CTAs of all layers fill the waves together), else one
  // launch per plan
  ResidualGroupArgs rg;
  std::memset(&rg, 0, sizeof(rg));
  bool grouped = n <= kMaxResGroup && !env_int("TW_K2_PER_LAYER", 0);
  // Layers enter the launch heaviest CTA first (CTAs are dispatched in index
  // order as SMs free up, so the long ones must not come last: BERT TEW,
  // 768x3072 / 3072x768 / 768^2 CTAs of ~34 / ~20 / ~11 us, packs 84 -> 75 us
  // in a list-scheduling model); each CTA's work ~ its entries x tokens.
  std::vector<int> order(n);
  std::vector<double> cta_work(n, 0.0);
  for (int i = 0; i < n; ++i) {
    order[i] = i;
    const tw_plan* p = plans[i];
    if (p && p->ov_block_tokens > 0 && !p->ov_start.empty())
      cta_work[i] = (double)p->ov_start.back() * p->ov_block_tokens;
  }
  if (!env_int("TW_GROUP_PLAN_ORDER", 0))
    std::stable_sort(order.begin(), order.end(),
                     [&](int x, int y) { return cta_work[x] > cta_work[y]; });
  for (int j = 0; j < n; ++j) {
    const int i = order[j];
    const tw_plan* p = plans[i];
    if (int st = check_io(p, xs[i], m, ld_xs[i], cts[i], ld_cts[i], out_dtype)) return st;
    const bool plan_layout = x_layouts && x_layouts[i] == TW_LAYOUT_PLAN;
    const bool ws = !scatter[i];
    build_k2_args(p, xs[i], m, ld_xs[i], cts[i], ld_cts[i], out_dtype, ws ? k1_out[i] : nullptr,
                  ws ? k1_ld[i] : 0, ws ? p->n_ov_cols_all : p->n_ov_cols, nullptr, false,
                  plan_layout, rg.args[j]);
    const ResidualArgs& a = rg.args[j];
    if (!a.rv || a.block_tokens <= 0 || a.n_cols <= 0 ||
        (a.in_dtype == kBF16) != (rg.args[0].in_dtype == kBF16))
      grouped = false;
    rg.cta0[j + 1] = rg.cta0[j] + (a.n_cols > 0 ? a.n_blocks * a.n_groups : 0);
  }
  rg.n = n;
  if (grouped) {
    TW_CUDA(launch_tw_residual_group(rg, s));
    return TW_OK;
  }
  for (int i = 0; i < n; ++i) TW_CUDA(launch_tw_residual(rg.args[i], s));
  return TW_OK;
}

int tw_gemm_ex(const tw_plan* p, const void* x, int64_t m, int64_t ld_x, void* ct, int64_t ld_ct,
               int32_t out_dtype, int32_t x_layout, void* stream) {
  g_last_error.clear();
  if (int st = check_io(p, x, m, ld_x, ct, ld_ct, out_dtype)) return st;
  if (x_layout != TW_LAYOUT_NATURAL && x_layout != TW_LAYOUT_PLAN)
    return fail(TW_ERR_INVALID_INPUT, "unknown activation layout %d", x_layout);
  return run_tw(p, x, m, ld_x, ct, ld_ct, out_dtype, nullptr, p->n_cond,
                static_cast<cudaStream_t>(stream), x_layout == TW_LAYOUT_PLAN);
}

int tw_plan_prepare(const tw_plan* p, const void* a, int32_t a_dtype, int64_t m, int64_t lda,
                    void* at, int64_t ld_at, void* stream) {
  g_last_error.clear();
  if (!p || !a || !at) return fail(TW_ERR_INVALID_INPUT, "null argument");
  if (m < 1 || lda < p->k || ld_at < m) return fail(TW_ERR_INVALID_INPUT, "bad prepare geometry");
  if (int st = check_dtype(a_dtype)) return st;
  if (p->split) {  // A -> [A_hi^T; A_lo^T]
    TW_CUDA(launch_transpose_split(a, a_dtype, m, p->k, lda, at, ld_at,
                                   static_cast<cudaStream_t>(stream)));
    return TW_OK;
  }
  for (int gi = 0; gi < (p->runs ? p->row_copies : 1); ++gi)
    TW_CUDA(launch_transpose_cast(a, a_dtype, m, p->k, lda, at, p->dtype, ld_at,
                                  p->runs ? p->d_inv + (size_t)gi * p->k : nullptr,
                                  static_cast<cudaStream_t>(stream)));
  return TW_OK;
}

int tw_plan_permute_rows(const tw_plan* p, const void* at, int64_t m, int64_t ld_at, void* x,
                         int64_t ld_x, void* stream) {
  g_last_error.clear();
  if (!p || !at || !x) return fail(TW_ERR_INVALID_INPUT, "null argument");
  if (m < 1 || ld_at < m || ld_x < m) return fail(TW_ERR_INVALID_INPUT, "bad permute geometry");
  if (p->split) return fail(TW_ERR_INVALID_INPUT, "fp32 plans take A (m x k), see tw_plan_prepare");
  const int64_t rows = (int64_t)p->k * (p->runs ? p->row_copies : 1);
  if (!p->runs) {
    TW_CUDA(cudaMemcpy2DAsync(x, ld_x * 2, at, ld_at * 2, m * 2, p->k, cudaMemcpyDeviceToDevice,
                              static_cast<cudaStream_t>(stream)));
    return TW_OK;
  }
  TW_CUDA(launch_scatter_rows(at, ld_at, p->d_perm, (int32_t)rows, x, ld_x, m, 2,
                              static_cast<cudaStream_t>(stream)));
  return TW_OK;
}

int tw_plan_row_order(const tw_plan* p, int32_t* out_rows) {
  if (!p || !out_rows) return fail(TW_ERR_INVALID_INPUT, "null argument");
  const int64_t n = (int64_t)p->k * (p->runs ? p->row_copies : 1);
  for (int64_t i = 0; i < n; ++i) out_rows[i] = p->runs ? p->perm[i] : (int32_t)i;
  return TW_OK;
}

// K2 over n_cols columns of the plan's overlay lists.  src (ld_src): the
// condensed TW result the kept columns read (workspace mode), nullptr = the
// out rows themselves; meta overrides the plan's per-column table; acc_all:
// every column adds onto its out row.
// K2's arguments for n_cols columns of the plan's overlay lists (see
// launch_k2).
static void build_k2_args(const tw_plan* p, const void* x, int64_t m, int64_t ld_x, void* ct,
                          int64_t ld_ct, int32_t out_dtype, const void* src, int64_t ld_src,
                          int32_t n_cols, const int4* meta, bool acc_all, bool plan_layout,
                          ResidualArgs& r) {
  r = ResidualArgs{};
  r.at = x;
  r.ld_at = ld_x;
  r.in_dtype = p->dtype;
  r.col_start = p->ov.start;
  r.rows = plan_layout ? p->ov.rows_pos : p->ov.rows;
  r.vals = p->ov.vals;
  r.out_rows = p->ov.out;
  r.meta = meta ? meta : p->ov.meta;
  r.accumulate = p->ov.acc;
  r.out = ct;
  r.ld_out = ld_ct;
  r.out_dtype = out_dtype;
  r.M = (int32_t)m;
  r.n_cols = n_cols;
  r.src = src;
  r.ld_src = ld_src;
  r.K = p->k_rows();
  r.acc_all = acc_all ? 1 : 0;
  const int esz = out_dtype == kF32 ? 4 : 2;
  auto al16 = [](const void* q, int64_t ld, int e) {
    return reinterpret_cast<uintptr_t>(q) % 16 == 0 && (ld * e) % 16 == 0;
  };
  r.vec_ok = al16(ct, ld_ct, esz) && (!src || al16(src, ld_src, esz)) ? 1 : 0;
  r.rv = plan_layout ? p->ov.rv_pos : p->ov.rv;
  r.block_tokens = p->ov_block_tokens;
  r.tokens_per_lane = p->ov_tpl;
  if (r.block_tokens > 0) {
    // grid = token blocks x column splits; splits (nnz-balanced runs of the
    // descending-nnz column order) are added only to round the number of
    // CTAs up to whole waves of resident CTAs
    const int T = r.block_tokens;
    const int64_t sms = p->sm_count;
    r.n_blocks = (int32_t)((m + T - 1) / T);
    int best = 1;
    double best_eff = 0.0;
    for (int ng = 1; ng <= 4 && ng <= r.n_cols; ++ng) {
      // CTAs are scheduled as slots free, so the busiest SM does about
      // ceil(ctas / SMs) CTAs of 1 / ng of a block's work; each extra split
      // re-stages the A^T block
      const int64_t ctas = (int64_t)r.n_blocks * ng;
      const int64_t per_sm = (ctas + sms - 1) / sms;
      const double eff = (double)ctas / (double)(per_sm * sms) / (1.0 + 0.1 * (ng - 1));
      if (eff > best_eff + 1e-9) {
        best_eff = eff;
        best = ng;
      }
    }
    r.n_groups = best;
    const int64_t total = p->ov_start.back();
    int c = 0;
    r.group_first[0] = 0;
    for (int g = 1; g < r.n_groups; ++g) {
      const int64_t target = total * g / r.n_groups;
      while (c < r.n_cols && p->ov_start[c] < target) ++c;
      r.group_first[g] = std::max(c, r.group_first[g - 1]);
    }
    r.group_first[r.n_groups] = r.n_cols;
  }
}

static int launch_k2(const tw_plan* p, const void* x, int64_t m, int64_t ld_x, void* ct,
                     int64_t ld_ct, int32_t out_dtype, const void* src, int64_t ld_src,
                     int32_t n_cols, const int4* meta, bool acc_all, cudaStream_t s,
                     bool plan_layout) {
  ResidualArgs r;
  build_k2_args(p, x, m, ld_x, ct, ld_ct, out_dtype, src, ld_src, n_cols, meta, acc_all,
                plan_layout, r);
  TW_CUDA(launch_tw_residual(r, s));
  return TW_OK;
}

static int run_tew(const tw_plan* p, const void* x, int64_t m, int64_t ld_x, void* ct,
                   int64_t ld_ct, int32_t out_dtype, void* ws, int64_t ld_ws, cudaStream_t s,
                   bool plan_layout = false) {
  // TW_TEW_PARTS (diagnostics): 1 = K1 only, 2 = K2 only, otherwise both
  const int parts = env_int("TW_TEW_PARTS", 3);
  if (parts != 2) {
    if (ws) {
      if (int st = run_tw(p, x, m, ld_x, ws, ld_ws, out_dtype, nullptr, p->n_cond, s, plan_layout))
        return st;
    } else if (int st = run_tw(p, x, m, ld_x, ct, ld_ct, out_dtype, p->ov.union_rowmap,
                               (int64_t)p->union_cols.size(), s, plan_layout)) {
      return st;
    }
  }
  if (parts == 1) return TW_OK;
  return launch_k2(p, x, m, ld_x, ct, ld_ct, out_dtype, ws, ld_ws,
                   ws ? p->n_ov_cols_all : p->n_ov_cols, nullptr, false, s, plan_layout);
}

int tw_gemm_tew(const tw_plan* p, const void* x, int64_t m, int64_t ld_x, void* ct,
                int64_t ld_ct, int32_t out_dtype, void* stream) {
  g_last_error.clear();
  if (int st = check_io(p, x, m, ld_x, ct, ld_ct, out_dtype)) return st;
  if (!p->has_overlay) return fail(TW_ERR_INVALID_INPUT, "plan has no overlay attached");
  return run_tew(p, x, m, ld_x, ct, ld_ct, out_dtype, nullptr, 0, static_cast<cudaStream_t>(stream));
}

int tw_plan_tew_workspace_bytes(const tw_plan* p, int64_t m, int32_t out_dtype, uint64_t* bytes) {
  if (!p || !bytes) return fail(TW_ERR_INVALID_INPUT, "null argument");
  if (int st = check_dtype(out_dtype)) return st;
  const uint64_t ld = (uint64_t)((m + 7) / 8 * 8);
  *bytes = (p->has_overlay && p->ov_block_tokens > 0)
               ? (uint64_t)p->n_cond * ld * (out_dtype == kF32 ? 4u : 2u)
               : 0u;
  return TW_OK;
}

int tw_gemm_tew_ws(const tw_plan* p, const void* x, int64_t m, int64_t ld_x, void* ct,
                   int64_t ld_ct, int32_t out_dtype, void* workspace, uint64_t ws_bytes,
                   void* stream) {
  g_last_error.clear();
  if (int st = check_io(p, x, m, ld_x, ct, ld_ct, out_dtype)) return st;
  if (!p->has_overlay) return fail(TW_ERR_INVALID_INPUT, "plan has no overlay attached");
  uint64_t need = 0;
  if (int st = tw_plan_tew_workspace_bytes(p, m, out_dtype, &need)) return st;
  void* ws = need ? workspace : nullptr;  // 0 bytes: the scatter path needs none
  if (need && (!workspace || ws_bytes < need || reinterpret_cast<uintptr_t>(workspace) % 16))
    return fail(TW_ERR_INVALID_INPUT, "workspace must hold %llu bytes, 16-byte aligned",
                (unsigned long long)need);
  return run_tew(p, x, m, ld_x, ct, ld_ct, out_dtype, ws, (m + 7) / 8 * 8,
                 static_cast<cudaStream_t>(stream));
}

int tw_gemm_tew_ex(const tw_plan* p, const void* x, int64_t m, int64_t ld_x, void* ct,
                   int64_t ld_ct, int32_t out_dtype, void* workspace, uint64_t ws_bytes,
                   int32_t x_layout, void* stream) {
  g_last_error.clear();
  if (int st = check_io(p, x, m, ld_x, ct, ld_ct, out_dtype)) return st;
  if (!p->has_overlay) return fail(TW_ERR_INVALID_INPUT, "plan has no overlay attached");
  if (x_layout != TW_LAYOUT_NATURAL && x_layout != TW_LAYOUT_PLAN)
    return fail(TW_ERR_INVALID_INPUT, "unknown activation layout %d", x_layout);
  const bool plan_layout = x_layout == TW_LAYOUT_PLAN;
  if (plan_layout && !p->runs) return fail(TW_ERR_INVALID_INPUT, "this plan has no row-run layout");
  uint64_t need = 0;
  if (int st = tw_plan_tew_workspace_bytes(p, m, out_dtype, &need)) return st;
  void* ws = need ? workspace : nullptr;
  if (need && (!workspace || ws_bytes < need || reinterpret_cast<uintptr_t>(workspace) % 16))
    return fail(TW_ERR_INVALID_INPUT, "workspace must hold %llu bytes, 16-byte aligned",
                (unsigned long long)need);
  return run_tew(p, x, m, ld_x, ct, ld_ct, out_dtype, ws, (m + 7) / 8 * 8,
                 static_cast<cudaStream_t>(stream), plan_layout);
}

int tw_gemm_tew_reuse(const tw_plan* p, const void* x, int64_t m, int64_t ld_x,
                      const void* tile_ct, int64_t ld_tile, const int32_t* tile_row_of_union,
                      void* ct, int64_t ld_ct, int32_t out_dtype, int32_t x_layout, void* stream) {
  g_last_error.clear();
  if (int st = check_io(p, x, m, ld_x, ct, ld_ct, out_dtype)) return st;
  if (!p->has_overlay) return fail(TW_ERR_INVALID_INPUT, "plan has no overlay attached");
  if (!tile_ct || ld_tile < m) return fail(TW_ERR_INVALID_INPUT, "tile product must be given, ld >= m");
  if (x_layout != TW_LAYOUT_NATURAL && x_layout != TW_LAYOUT_PLAN)
    return fail(TW_ERR_INVALID_INPUT, "unknown activation layout %d", x_layout);
  const bool plan_layout = x_layout == TW_LAYOUT_PLAN;
  if (plan_layout && !p->runs) return fail(TW_ERR_INVALID_INPUT, "this plan has no row-run layout");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int esz = out_dtype == kF32 ? 4 : 2;
  const int32_t nu = (int32_t)p->union_cols.size();
  if (!tile_row_of_union && p->ov_block_tokens > 0) {
    // the tile product is in this plan's condensed column order: K2 alone in
    // workspace mode, reading it as the kept columns' source rows
    return launch_k2(p, x, m, ld_x, ct, ld_ct, out_dtype, tile_ct, ld_tile, p->n_ov_cols_all,
                     nullptr, false, s, plan_layout);
  }
  // general: scatter the caller's rows to the union rows (zeros where the
  // tile product has no such column), then K2 adds every overlay column
  std::vector<int32_t> map(nu, -1);
  if (tile_row_of_union) {
    for (int32_t u = 0; u < nu; ++u) map[u] = tile_row_of_union[u];
  } else {
    std::vector<int32_t> cond_of(p->n, -1);
    for (int32_t i = 0; i < p->n_cond; ++i) cond_of[p->cond_cols[i]] = i;
    for (int32_t u = 0; u < nu; ++u) map[u] = cond_of[p->union_cols[u]];
  }
  int32_t* d_map = nullptr;
  TW_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_map), (size_t)nu * sizeof(int32_t), s));
  cudaError_t e = cudaMemcpyAsync(d_map, map.data(), (size_t)nu * sizeof(int32_t),
                                  cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = launch_scatter_rows(tile_ct, ld_tile, d_map, nu, ct, ld_ct, m, esz, s);
  // the host vector must outlive the (pageable, staged) copy
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFreeAsync(d_map, s);
  if (e != cudaSuccess) return fail(TW_ERR_CUDA, "tile product scatter failed: %s", cudaGetErrorString(e));
  return launch_k2(p, x, m, ld_x, ct, ld_ct, out_dtype, nullptr, 0, p->n_ov_cols, nullptr, true, s,
                   plan_layout);
}

int tw_transpose_cast(const void* a, int32_t a_dtype, int64_t m, int64_t k, int64_t lda, void* at,
                      int32_t at_dtype, int64_t ld_at, void* stream) {
  g_last_error.clear();
  if (!a || !at) return fail(TW_ERR_INVALID_INPUT, "null argument");
  if (m < 1 || k < 1 || lda < k || ld_at < m)
    return fail(TW_ERR_INVALID_INPUT, "bad transpose geometry");
  if (int st = check_dtype(a_dtype)) return st;
  if (int st = check_dtype(at_dtype)) return st;
  TW_CUDA(launch_transpose_cast(a, a_dtype, m, k, lda, at, at_dtype, ld_at, nullptr,
                                static_cast<cudaStream_t>(stream)));
  return TW_OK;
}

void tw_plan_destroy(tw_plan* p) { delete p; }

void tw_debug_set_trace(void* dev_buffer) { g_trace = static_cast<long long*>(dev_buffer); }

}  // extern "C"
