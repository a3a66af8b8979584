/*
 * TEST INFRASTRUCTURE ONLY -- CPU oracle for the TW / TEW matmul.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path never does.
 *
 * Plain-C restatement of the reference kernel:
 *   _mac_kernel    pkg/src/tilesparse/executor.py:27-37  (fp64, k strictly ascending)
 *   _tile_product  executor.py:121-124                  (gather A[:, kept_rows])
 *   gemm_cto       executor.py:149-177                  (rows/cols = position + offset)
 *   gemm_tew       executor.py:194-200                  (tile product + per-column overlay)
 *
 * Bit-exactness argument: the reference multiplies float32 values widened to
 * float64 (exact: 24+24 < 53 mantissa bits) and adds the products in
 * ascending kept-row order into a float64 accumulator starting at 0.  The loop
 * below performs the same additions in the same order; fma contraction cannot
 * change the result because each product is exact in float64.
 *
 * Threads split the output rows (tokens); each output element is still a
 * single sequential sum, so results are independent of the thread count.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  const float* a;          /* M x K row-major fp32 */
  int64_t m, k;
  int32_t n_tiles;
  const uint32_t* row_counts, *col_counts, *row_offsets, *col_offsets;
  int32_t max_rows, max_cols;
  const float* payload;    /* packed, per tile transposed: width x kept */
  double* out;             /* M x N' row-major fp64 */
  int64_t n_cond;
  int64_t m_lo, m_hi;
} job_t;

static void* run_rows(void* arg) {
  job_t* j = (job_t*)arg;
  int64_t pbase = 0, col0 = 0;
  for (int32_t t = 0; t < j->n_tiles; ++t) {
    const int64_t h = j->row_counts[t], w = j->col_counts[t];
    const uint32_t* offs = j->row_offsets + (int64_t)t * j->max_rows;
    for (int64_t m = j->m_lo; m < j->m_hi; ++m) {
      const float* arow = j->a + m * j->k;
      double* orow = j->out + m * j->n_cond + col0;
      for (int64_t c = 0; c < w; ++c) {
        const float* p = j->payload + pbase + c * h; /* payload_t row c */
        double acc = 0.0;
        for (int64_t i = 0; i < h; ++i) {
          const int64_t r = i + (int64_t)offs[i];
          acc += (double)arow[r] * (double)p[i];
        }
        orow[c] = acc;
      }
    }
    pbase += h * w;
    col0 += w;
  }
  return NULL;
}

/* out[M x N'] = gemm_cto(a, enc) in fp64.  Returns 0 on success. */
int tw_oracle_gemm_cto(const float* a, int64_t m, int64_t k, int32_t n_tiles,
                       const uint32_t* row_counts, const uint32_t* col_counts,
                       const uint32_t* row_offsets, int32_t max_rows,
                       const uint32_t* col_offsets, int32_t max_cols, const float* payload,
                       double* out, int32_t threads) {
  int64_t n_cond = 0;
  for (int32_t t = 0; t < n_tiles; ++t) n_cond += col_counts[t];
  if (m <= 0) return 0;
  if (threads > m) threads = (int32_t)m;
  if (threads < 1) threads = 1;
  pthread_t* tid = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  job_t* jobs = (job_t*)calloc((size_t)threads, sizeof(job_t));
  if (!tid || !jobs) return 1;
  for (int32_t i = 0; i < threads; ++i) {
    job_t* j = &jobs[i];
    j->a = a; j->m = m; j->k = k; j->n_tiles = n_tiles;
    j->row_counts = row_counts; j->col_counts = col_counts;
    j->row_offsets = row_offsets; j->col_offsets = col_offsets;
    j->max_rows = max_rows; j->max_cols = max_cols; j->payload = payload;
    j->out = out; j->n_cond = n_cond;
    j->m_lo = m * i / threads; j->m_hi = m * (i + 1) / threads;
  }
  for (int32_t i = 1; i < threads; ++i) pthread_create(&tid[i], NULL, run_rows, &jobs[i]);
  run_rows(&jobs[0]);
  for (int32_t i = 1; i < threads; ++i) pthread_join(tid[i], NULL);
  free(tid);
  free(jobs);
  return 0;
}

/* full[M x N] += overlay product (executor.py:197-200), sequential over the
 * column's rows in CSC order. */
int tw_oracle_overlay_add(const float* a, int64_t m, int64_t k, int64_t n,
                          const int64_t* col_ptr, const int64_t* row_idx, const float* vals,
                          double* full) {
  for (int64_t c = 0; c < n; ++c) {
    const int64_t lo = col_ptr[c], hi = col_ptr[c + 1];
    if (lo == hi) continue;
    for (int64_t mm = 0; mm < m; ++mm) {
      const float* arow = a + mm * k;
      double acc = 0.0;
      for (int64_t e = lo; e < hi; ++e) acc += (double)arow[row_idx[e]] * (double)vals[e];
      full[mm * n + c] += acc;
    }
  }
  return 0;
}
