/* Oracle CSC products -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
 *
 * C restatement of the reference's compiled kernels
 * (/root/reference/pkg/src/conegrad/_kernels/_csc.pyx:17-50): entry k of
 * column j contributes values[k]*x[j] to row row_idx[k]; both products
 * accumulate in storage order, so results are bit-identical to the
 * reference's Cython and NumPy backends.  Built by oracle/Makefile with the
 * same -O2 the reference's setup.py uses, without FMA contraction. */
#include <stdint.h>
#include <string.h>

void oracle_csc_spmv(int64_t nrows, int64_t ncols, const int64_t *col_ptr,
                     const int64_t *row_idx, const double *values,
                     const double *x, double *out) {
  memset(out, 0, (size_t)nrows * sizeof(double));
  for (int64_t j = 0; j < ncols; ++j) {
    const double xj = x[j];
    for (int64_t k = col_ptr[j]; k < col_ptr[j + 1]; ++k) {
      const double prod = values[k] * xj;
      out[row_idx[k]] += prod;
    }
  }
}

void oracle_csc_spmv_adjoint(int64_t ncols, const int64_t *col_ptr,
                             const int64_t *row_idx, const double *values,
                             const double *y, double *out) {
  for (int64_t j = 0; j < ncols; ++j) {
    double acc = 0.0;
    for (int64_t k = col_ptr[j]; k < col_ptr[j + 1]; ++k) {
      const double prod = values[k] * y[row_idx[k]];
      acc += prod;
    }
    out[j] = acc;
  }
}
