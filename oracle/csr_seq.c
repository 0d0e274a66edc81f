/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.  Never linked into, loaded by, or called
 * from the product package (paper_2105_07544_b200).  Only tests/, the smoke()
 * check in __graft_entry__.py and bench.py's cpu_baseline / --impl reference
 * legs may load this file's shared object.
 *
 * Restatement of the third-party kernel the reference's SpMV bottoms out in:
 * mpkrylov `spmv` (pkg/src/mpkrylov/sparse.py:190-206) calls
 * `scipy.sparse.csr_matrix.dot`, i.e. SciPy sparsetools `csr_matvec`
 * (scipy 1.18.1 in the survey container; not vendored under /root/reference).
 * Its published algorithm: for every row, start a running sum at zero (the
 * output vector is freshly zeroed), add value*x[col] for the row's stored
 * entries in storage order, rounding after every multiply and every add in
 * the value dtype, and store the sum.  Indices are 32-bit in SciPy; we take
 * 64-bit and it makes no difference to the arithmetic.
 *
 * Compile with -ffp-contract=off so the multiply-add pairs are never fused.
 */
#include <stdint.h>

void oracle_spmv_f64(int64_t n, const int64_t *row_ptr, const int64_t *col_idx,
                     const double *val, const double *x, double *y)
{
    for (int64_t r = 0; r < n; ++r) {
        double acc = 0.0;
        for (int64_t p = row_ptr[r]; p < row_ptr[r + 1]; ++p) {
            double prod = val[p] * x[col_idx[p]];
            acc = acc + prod;
        }
        y[r] = acc;
    }
}

void oracle_spmv_f32(int64_t n, const int64_t *row_ptr, const int64_t *col_idx,
                     const float *val, const float *x, float *y)
{
    for (int64_t r = 0; r < n; ++r) {
        float acc = 0.0f;
        for (int64_t p = row_ptr[r]; p < row_ptr[r + 1]; ++p) {
            float prod = val[p] * x[col_idx[p]];
            acc = acc + prod;
        }
        y[r] = acc;
    }
}
