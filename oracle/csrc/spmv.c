/* Plain CSR sparse matrix-vector product y = A x for the oracle-assembled matrix
 * (PAPER eq:matrixbasedop P:224-227; the paper's sparse baseline P:921-931) --
 * TEST / BASELINE INFRASTRUCTURE ONLY (see oracle/__init__.py).  One FMA per stored
 * entry, rows split statically over `nthreads` OpenMP threads.  No code shared with
 * the CUDA path. */
#include <stdint.h>
#include <omp.h>

void oracle_spmv_csr(int64_t nrows, const int64_t *rp, const int32_t *col, const double *val, const double *x,
                     double *y, int nthreads) {
  int64_t i;
#pragma omp parallel for schedule(static) num_threads(nthreads)
  for (i = 0; i < nrows; ++i) {
    double s = 0.0;
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) s += val[k] * x[col[k]];
    y[i] = s;
  }
}

int oracle_max_threads(void) { return omp_get_max_threads(); }
