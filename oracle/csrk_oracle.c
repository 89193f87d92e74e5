/*
 * csrk_oracle.c -- CPU restatement of the reference csrk SpMV path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the checker and the CPU baseline:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  The product (paper_2203_05096_b200)
 * never links or calls it.
 *
 * Each function restates one reference function (file:line under
 * /root/reference/pkg/src/csrk/).  Arithmetic is IEEE double with the
 * multiply and the add rounded separately (build with -ffp-contract=off),
 * which is what numpy's `vals * x[cols]` followed by `acc += ...` does.
 * The oracle is pinned against the reference's own outputs by
 * tests/golden (tests/test_oracle.py).
 */
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* kernels.py:97-114 spmv_csr_ref and kernels.py:117-147 _rows_spmv: every
 * row is acc = 0.0; acc += vals[p] * x[col[p]] left to right. */
static double row_serial(const uint32_t *row_ptr, const uint32_t *col_idx,
                         const double *vals, const double *x, int64_t r) {
  double acc = 0.0;
  for (uint32_t p = row_ptr[r]; p < row_ptr[r + 1]; ++p) {
    const double prod = vals[p] * x[col_idx[p]];
    acc = acc + prod;
  }
  return acc;
}

void oracle_spmv_serial(int64_t n_rows, const uint32_t *row_ptr,
                        const uint32_t *col_idx, const double *vals,
                        const double *x, double *y) {
  for (int64_t r = 0; r < n_rows; ++r)
    y[r] = row_serial(row_ptr, col_idx, vals, x, r);
}

/* kernels.py:150-182 _static_chunks + _grouped_spmv, used by spmv_csr2
 * (groups = super-rows, kernels.py:185-206) and spmv_csr3 (groups =
 * super-super-rows, row offsets sr_ptr[ssr_ptr], kernels.py:209-221):
 * the group range is split into `workers` contiguous near-equal chunks
 * (numpy linspace bounds), each chunk summed row by row.  group_rows holds
 * the first row of every group plus the end (n_groups + 1 entries). */
void oracle_spmv_grouped(int64_t n_groups, const int64_t *group_rows,
                         const uint32_t *row_ptr, const uint32_t *col_idx,
                         const double *vals, const double *x, double *y,
                         int workers) {
  if (workers < 1) workers = 1;
  int64_t parts = n_groups < workers ? n_groups : workers;
  if (parts < 1) parts = 1;
#pragma omp parallel for schedule(static, 1) num_threads(workers)
  for (int64_t c = 0; c < parts; ++c) {
    /* linspace(0, count, parts + 1) cast to int64 truncates */
    const int64_t g0 = (int64_t)((double)n_groups * (double)c / (double)parts);
    const int64_t g1 =
        (int64_t)((double)n_groups * (double)(c + 1) / (double)parts);
    for (int64_t r = group_rows[g0]; r < group_rows[g1]; ++r)
      y[r] = row_serial(row_ptr, col_idx, vals, x, r);
  }
}

/* kernels.py:264-324: nonzero p of a row goes to temp[(p - start) % nx];
 * lanes are zero-padded to the next power of two and combined by the
 * halving tree buf[i] += buf[i + stride]. */
void oracle_spmv_strided(int64_t n_rows, const uint32_t *row_ptr,
                         const uint32_t *col_idx, const double *vals,
                         const double *x, double *y, int nx) {
  int size = 1;
  while (size < nx) size <<= 1;
  double buf[1024];
  for (int64_t r = 0; r < n_rows; ++r) {
    for (int i = 0; i < size; ++i) buf[i] = 0.0;
    int lane = 0;
    for (uint32_t p = row_ptr[r]; p < row_ptr[r + 1]; ++p) {
      const double prod = vals[p] * x[col_idx[p]];
      buf[lane] = buf[lane] + prod;
      if (++lane == nx) lane = 0;
    }
    if (nx > 1)
      for (int stride = size / 2; stride > 0; stride /= 2)
        for (int i = 0; i < stride; ++i) buf[i] = buf[i] + buf[i + stride];
    y[r] = buf[0];
  }
}

/* format.py:318-344 _permute_symmetric: new row i is old row inv[i] with
 * columns renamed by fwd and sorted ascending (insertion sort: columns are
 * unique, so any sort gives the lexsort answer). */
void oracle_permute_symmetric(int64_t n, const uint32_t *row_ptr,
                              const uint32_t *col_idx, const double *vals,
                              const int64_t *fwd, const int64_t *inv,
                              uint32_t *out_ptr, uint32_t *out_cols,
                              double *out_vals) {
  out_ptr[0] = 0;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t src = inv[i];
    out_ptr[i + 1] = out_ptr[i] + (row_ptr[src + 1] - row_ptr[src]);
  }
  for (int64_t i = 0; i < n; ++i) {
    const int64_t src = inv[i];
    const uint32_t s = row_ptr[src], len = row_ptr[src + 1] - s;
    uint32_t *c = out_cols + out_ptr[i];
    double *v = out_vals + out_ptr[i];
    for (uint32_t j = 0; j < len; ++j) {
      const uint32_t key = (uint32_t)fwd[col_idx[s + j]];
      const double val = vals[s + j];
      uint32_t k = j;
      while (k > 0 && c[k - 1] > key) {
        c[k] = c[k - 1];
        v[k] = v[k - 1];
        --k;
      }
      c[k] = key;
      v[k] = val;
    }
  }
}

/* format.py:396-409: out[i] = in[idx[i]] */
void oracle_gather(int64_t n, const double *in, const int64_t *idx,
                   double *out) {
  for (int64_t i = 0; i < n; ++i) out[i] = in[idx[i]];
}

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
