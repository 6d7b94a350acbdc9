/* oracle/o1.c -- O1, the plain serial definition of y = A x.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header or constant with the CUDA path (paper_2203_02530_b200/).
 *
 * What it follows: PAPER.md §III-A (sec:dag) P:271-275 -- "A rank's y entries
 * can then be computed as the sum of a local and remote matrix-vector
 * multiplication y_L = A_L x_L and y_R = A_R x_R", i.e. the plain product
 * y_i = sum_j a_ij x_j over the stored nonzeros of row i.  SURVEY.md §8(c) O1:
 * rows ascending, entries in stored order, fp64 accumulation starting at +0.0,
 * product and sum rounded separately (built with -O2 -ffp-contract=off, no
 * fast-math).  fp32 inputs are upcast to fp64 by the caller.
 */
#include <stdint.h>
#include <math.h>

/* y[i] = sum_{p=rowptr[i]-rowptr[0]}^{rowptr[i+1]-rowptr[0]-1} val[p]*x[col[p]] */
void o1_spmv(int64_t n_rows, const int64_t* rowptr, const int32_t* col,
             const double* val, const double* x, double* y)
{
    const int64_t base = rowptr[0];
    for (int64_t i = 0; i < n_rows; ++i) {
        double acc = 0.0;
        for (int64_t p = rowptr[i] - base; p < rowptr[i + 1] - base; ++p) {
            double prod = val[p] * x[col[p]];
            acc = acc + prod;
        }
        y[i] = acc;
    }
}

/* The same loop on a sample of rows: y_s[k] = row rows[k] of A x. */
void o1_spmv_rows(int64_t n_sample, const int64_t* rows, const int64_t* rowptr,
                  const int32_t* col, const double* val, const double* x, double* y_s)
{
    const int64_t base = rowptr[0];
    for (int64_t k = 0; k < n_sample; ++k) {
        const int64_t i = rows[k];
        double acc = 0.0;
        for (int64_t p = rowptr[i] - base; p < rowptr[i + 1] - base; ++p) {
            double prod = val[p] * x[col[p]];
            acc = acc + prod;
        }
        y_s[k] = acc;
    }
}

/* s[i] = sum_p |val[p] * x[col[p]]| -- the scale of the north_star tolerance
 * |y_gpu - y_ref| <= 1e-12 * sum_j |a_ij x_j| (BASELINE.json north_star). */
void o1_absdot(int64_t n_rows, const int64_t* rowptr, const int32_t* col,
               const double* val, const double* x, double* s)
{
    const int64_t base = rowptr[0];
    for (int64_t i = 0; i < n_rows; ++i) {
        double acc = 0.0;
        for (int64_t p = rowptr[i] - base; p < rowptr[i + 1] - base; ++p)
            acc = acc + fabs(val[p] * x[col[p]]);
        s[i] = acc;
    }
}

/* "the same plain loop with #pragma omp parallel for
 * schedule(static) over rows on all host cores" -- the CPU baseline on every
 * core.  Each row is still summed by one thread in stored order, so y is
 * bitwise that of o1_spmv. */
#include <omp.h>
void o1_spmv_omp(int64_t n_rows, const int64_t* rowptr, const int32_t* col,
                 const double* val, const double* x, double* y)
{
    const int64_t base = rowptr[0];
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n_rows; ++i) {
        double acc = 0.0;
        for (int64_t p = rowptr[i] - base; p < rowptr[i + 1] - base; ++p) {
            double prod = val[p] * x[col[p]];
            acc = acc + prod;
        }
        y[i] = acc;
    }
}

int o1_omp_threads(void) { return omp_get_max_threads(); }
