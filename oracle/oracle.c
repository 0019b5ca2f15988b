/*
 * oracle/oracle.c -- the CPU oracle for msRep's hot path (arXiv 2209.07552).
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the C-ABI library
 * libmsrep.so and its Python binding) may include, link, load or call this
 * file.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may use it.  It shares no code, header, table or
 * helper with paper_2209_07552_b200/csrc/.
 *
 * Plain, slow, single-threaded, obviously-correct C99.  Built with
 *   gcc -O2 -ffp-contract=off -fno-fast-math
 * so every floating-point operation is the one written here (no FMA
 * contraction).  Indices are 0-based (reading R1: the paper's
 * algorithms are 1-based and their i = 1..np loop would skip part 0).
 *
 * Citations: "P:a-b" = /root/reference/PAPER.md lines a-b, "S:a-b" = SPEC.md.
 *
 * Precision (reading R13): values are fp64 or fp32 storage; every
 * sum is accumulated in fp64 and rounded once to the storage type at the end.
 * For fp32 data the product (double)a*(double)x is exact (24+24 < 53 bits).
 *
 * Pins (tests/test_oracle_*.py): fixture E and every SPEC worked value,
 * identity / permutation / diagonal / 27-point-stencil closed forms, numpy
 * dense brute force, bit-exact conversion round trips, exhaustive balance
 * and merge-of-partition identities.  No function below is "parity unpinned".
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

#define OR_F64 0
#define OR_F32 1

/* ------------------------------------------------------------------------ */
/* scalar access helpers for the two storage types                          */
/* ------------------------------------------------------------------------ */
static double get_val(const void *a, int dtype, int64_t k)
{
    if (dtype == OR_F64) return ((const double *)a)[k];
    return (double)((const float *)a)[k];
}

static void put_val(void *a, int dtype, int64_t k, double v)
{
    if (dtype == OR_F64) ((double *)a)[k] = v;
    else ((float *)a)[k] = (float)v;
}

static size_t vsize(int dtype) { return dtype == OR_F64 ? 8 : 4; }

/* ------------------------------------------------------------------------ */
/* Format conversions (Sec. 2.1).  Stable counting sort;  */
/* values are copied byte-for-byte (bit-exact).                              */
/* ------------------------------------------------------------------------ */

/* COO (any order) -> CSR.  Entries with equal row keep their input order, so
 * a row-sorted (ties by column) COO gives column-sorted rows. */
void or_coo_to_csr(int64_t m, int64_t nnz, const int64_t *row_idx,
                   const int32_t *col_idx, const void *val, int dtype,
                   int64_t *row_ptr, int32_t *out_col, void *out_val)
{
    size_t vs = vsize(dtype);
    int64_t *next = (int64_t *)malloc((size_t)(m + 1) * sizeof(int64_t));
    for (int64_t r = 0; r <= m; r++) row_ptr[r] = 0;
    for (int64_t k = 0; k < nnz; k++) row_ptr[row_idx[k] + 1] += 1;   /* count */
    for (int64_t r = 0; r < m; r++) row_ptr[r + 1] += row_ptr[r];     /* prefix */
    for (int64_t r = 0; r <= m; r++) next[r] = row_ptr[r];
    for (int64_t k = 0; k < nnz; k++) {                               /* place */
        int64_t d = next[row_idx[k]]++;
        out_col[d] = col_idx[k];
        memcpy((char *)out_val + (size_t)d * vs, (const char *)val + (size_t)k * vs, vs);
    }
    free(next);
}

/* CSR -> COO (row-sorted, ties by the CSR order within the row). */
void or_csr_to_coo(int64_t m, const int64_t *row_ptr, int64_t *row_idx)
{
    for (int64_t r = 0; r < m; r++)
        for (int64_t j = row_ptr[r]; j < row_ptr[r + 1]; j++) row_idx[j] = r;
}

/* CSR (m x n) -> CSC (m x n): "CSC of A = CSR of A^T".  Counting sort
 * by column; within a column, rows come out ascending because CSR is walked
 * row by row. */
void or_csr_to_csc(int64_t m, int64_t n, const int64_t *row_ptr,
                   const int32_t *col_idx, const void *val, int dtype,
                   int64_t *col_ptr, int32_t *out_row, void *out_val)
{
    size_t vs = vsize(dtype);
    int64_t nnz = row_ptr[m];
    int64_t *next = (int64_t *)malloc((size_t)(n + 1) * sizeof(int64_t));
    for (int64_t c = 0; c <= n; c++) col_ptr[c] = 0;
    for (int64_t k = 0; k < nnz; k++) col_ptr[col_idx[k] + 1] += 1;
    for (int64_t c = 0; c < n; c++) col_ptr[c + 1] += col_ptr[c];
    for (int64_t c = 0; c <= n; c++) next[c] = col_ptr[c];
    for (int64_t r = 0; r < m; r++) {
        for (int64_t j = row_ptr[r]; j < row_ptr[r + 1]; j++) {
            int64_t d = next[col_idx[j]]++;
            out_row[d] = (int32_t)r;
            memcpy((char *)out_val + (size_t)d * vs, (const char *)val + (size_t)j * vs, vs);
        }
    }
    free(next);
}

/* CSC -> COO in column order (col_idx expanded from col_ptr). */
void or_csc_to_coo(int64_t n, const int64_t *col_ptr, int64_t *col_idx)
{
    for (int64_t c = 0; c < n; c++)
        for (int64_t j = col_ptr[c]; j < col_ptr[c + 1]; j++) col_idx[j] = c;
}

/* ------------------------------------------------------------------------ */
/* Reference SpMV, y = alpha*A*x + beta*y (Alg. 1).      */
/* Reading R2: Alg. 1 prints the update inside the inner loop; the operation  */
/* it names is y_i = alpha * sum_j a_ij x_j + beta * y_i, applied once.       */
/* Reading R12 (BLAS convention): beta == 0 -> y_in is not read;              */
/* alpha == 0 -> y = beta*y_in and neither A nor x is read.                  */
/* ------------------------------------------------------------------------ */
static double finish(double alpha, double acc, double beta, const void *y, int dtype, int64_t i)
{
    double r = alpha * acc;
    if (beta != 0.0) r = r + beta * get_val(y, dtype, i);
    return r;
}

/* Alg. 1: rows in order, nonzeros left to right. */
void or_spmv_csr(int64_t m, const int64_t *row_ptr, const int32_t *col_idx,
                 const void *val, int dtype, const void *x, void *y,
                 double alpha, double beta)
{
    for (int64_t i = 0; i < m; i++) {
        double acc = 0.0;
        if (alpha != 0.0) {
            for (int64_t j = row_ptr[i]; j < row_ptr[i + 1]; j++)
                acc = acc + get_val(val, dtype, j) * get_val(x, dtype, col_idx[j]);
        }
        put_val(y, dtype, i, finish(alpha, acc, beta, y, dtype, i));
    }
}

/* CSC: "switch the role of x and y" -- scatter column by column into
 * a zeroed accumulator, then y = alpha*acc + beta*y_in. */
void or_spmv_csc(int64_t m, int64_t n, const int64_t *col_ptr, const int32_t *row_idx,
                 const void *val, int dtype, const void *x, void *y,
                 double alpha, double beta)
{
    double *acc = (double *)calloc((size_t)(m > 0 ? m : 1), sizeof(double));
    if (alpha != 0.0) {
        for (int64_t c = 0; c < n; c++)
            for (int64_t j = col_ptr[c]; j < col_ptr[c + 1]; j++)
                acc[row_idx[j]] = acc[row_idx[j]] + get_val(val, dtype, j) * get_val(x, dtype, c);
    }
    for (int64_t i = 0; i < m; i++) put_val(y, dtype, i, finish(alpha, acc[i], beta, y, dtype, i));
    free(acc);
}

/* COO: "only one loop for all the nnz non-zero elements", triplet
 * order. */
void or_spmv_coo(int64_t m, int64_t nnz, const int64_t *row_idx, const int32_t *col_idx,
                 const void *val, int dtype, const void *x, void *y,
                 double alpha, double beta)
{
    double *acc = (double *)calloc((size_t)(m > 0 ? m : 1), sizeof(double));
    if (alpha != 0.0) {
        for (int64_t k = 0; k < nnz; k++)
            acc[row_idx[k]] = acc[row_idx[k]] + get_val(val, dtype, k) * get_val(x, dtype, col_idx[k]);
    }
    for (int64_t i = 0; i < m; i++) put_val(y, dtype, i, finish(alpha, acc[i], beta, y, dtype, i));
    free(acc);
}

/* Per-row error scale for the tolerance check:
 * bound_i = |alpha| * sum_j |a_ij * x_j| + |beta * y_in_i|. */
void or_row_bound_csr(int64_t m, const int64_t *row_ptr, const int32_t *col_idx,
                      const void *val, int dtype, const void *x, const void *y_in,
                      double alpha, double beta, double *bound)
{
    for (int64_t i = 0; i < m; i++) {
        double s = 0.0;
        for (int64_t j = row_ptr[i]; j < row_ptr[i + 1]; j++)
            s = s + fabs(get_val(val, dtype, j) * get_val(x, dtype, col_idx[j]));
        double b = fabs(alpha) * s;
        if (beta != 0.0) b = b + fabs(beta * get_val(y_in, dtype, i));
        bound[i] = b;
    }
}

/* ------------------------------------------------------------------------ */
/* nnz split, Alg. 2 lines 2-3: b_i = floor(i*nnz/np), 0<=i<=np. */
/* ------------------------------------------------------------------------ */
void or_nnz_boundaries(int64_t nnz, int64_t np, int64_t *b)
{
    for (int64_t i = 0; i <= np; i++) b[i] = (i * nnz) / np;
}

/* Row/column-block split of the paper's "Baseline" (Sec. 5.1: "the
 * input matrix is partitioned in either row blocks (for CSR and COO) or column
 * blocks (for CSC) without considering the distribution of non-zero
 * elements"): part i holds the whole rows (columns) [floor(i*m/np),
 * floor((i+1)*m/np)), i.e. b_i = ptr[floor(i*m/np)]. */
void or_block_boundaries(int64_t m, const int64_t *ptr, int64_t np, int64_t *b)
{
    for (int64_t i = 0; i <= np; i++) b[i] = ptr[(i * m) / np];
}

/* The same row-block split on a row-sorted COO: b_i = number of nonzeros whose
 * row is below floor(i*m/np), counted by a linear scan. */
void or_block_boundaries_coo(int64_t m, int64_t nnz, const int64_t *row_idx, int64_t np, int64_t *b)
{
    for (int64_t i = 0; i <= np; i++) {
        int64_t r = (i * m) / np, k = 0;
        while (k < nnz && row_idx[k] < r) k++;
        b[i] = k;
    }
}

/* Two-level split (Sec. 4.2, P:567 and Fig. 2level): level 1 cuts
 * [0,nnz) among NUMA groups in proportion to their part (GPU) counts,
 * c_g = floor(D_g*nnz/D) with D_g the prefix sum of the group sizes; level 2
 * cuts each group's range among its parts with the floor rule,
 * b = c_g + floor(i*(c_{g+1}-c_g)/d_g).  Writes np+1 boundaries, np = D. */
void or_two_level_boundaries(int64_t nnz, int64_t ngroups, const int64_t *sizes, int64_t *b)
{
    int64_t D = 0;
    for (int64_t g = 0; g < ngroups; g++) D += sizes[g];
    int64_t Dg = 0, w = 0;
    for (int64_t g = 0; g < ngroups; g++) {
        int64_t c0 = (Dg * nnz) / D, c1 = ((Dg + sizes[g]) * nnz) / D;
        for (int64_t i = 0; i < sizes[g]; i++) b[w++] = c0 + (i * (c1 - c0)) / sizes[g];
        Dg += sizes[g];
    }
    b[w] = nnz;
}

/* The workload-imbalance cost model behind Fig. 6: a
 * memory-bound SpMV's time is set by the part with the most nonzeros, so the
 * throughput of a plan relative to a perfectly balanced one is
 * (sum_i nnz_i / np) / max_i nnz_i. */
double or_relative_throughput(int64_t np, const int64_t *b)
{
    int64_t mx = 0;
    for (int64_t i = 0; i < np; i++)
        if (b[i + 1] - b[i] > mx) mx = b[i + 1] - b[i];
    if (mx == 0) return 1.0;
    return ((double)(b[np] - b[0]) / (double)np) / (double)mx;
}

/* Strict owner of nonzero position idx: the unique r with
 * ptr[r] <= idx < ptr[r+1] (reading R3).  LINEAR scan on purpose:
 * the library uses a binary search, so this is an independent check. */
int64_t or_owner_linear(int64_t m, const int64_t *ptr, int64_t idx)
{
    for (int64_t r = 0; r < m; r++)
        if (ptr[r] <= idx && idx < ptr[r + 1]) return r;
    return -1;
}

/* Descriptor of one part (mirrors msrep_part_desc field-for-field but is a
 * separate definition: the oracle shares no header with the library). */
typedef struct {
    int64_t start_idx, end_idx;     /* inclusive (Alg. 2 l.2-3); empty: start == end+1 */
    int64_t start_row, end_row;     /* start_col/end_col for pCSC; -1,-1 if empty     */
    int32_t start_flag;             /* first row/col shared with an earlier part      */
    int32_t pad_;
    int64_t owned_begin, owned_end; /* [R_i, R_{i+1}) rows this part writes (R9)      */
} or_part;

/* Alg. 2 (CSR->pCSR) and Alg. 4 (CSC->pCSC): the same
 * computation over a pointer array ptr[0..m] (row_ptr or col_ptr).
 *   start_row = BinarySearch(ptr, start_idx)  -> strict owner (R3), linear here
 *   start_flag = start_idx > ptr[start_row]   (Alg. 2 l.6)
 *   local_ptr[k] = clamp(ptr[start_row+k], start_idx, end_idx+1) - start_idx,
 *                  k = 0..end_row-start_row+1 (Alg. 2 l.11-12; reading R5)
 *   owned range R_i = smallest r with ptr[r] >= b_i, R_0 = 0, R_np = m (R9).
 * local_out receives, for each part in order, its end_row-start_row+2 local
 * pointers (1 entry [0] for an empty part); returns total entries written. */
int64_t or_partition_ptr_b(int64_t m, const int64_t *ptr, int64_t np, const int64_t *b,
                           or_part *parts, int64_t *local_out);

int64_t or_partition_ptr(int64_t m, const int64_t *ptr, int64_t np,
                         or_part *parts, int64_t *local_out)
{
    int64_t *b = (int64_t *)malloc((size_t)(np + 1) * sizeof(int64_t));
    or_nnz_boundaries(ptr[m], np, b);
    int64_t w = or_partition_ptr_b(m, ptr, np, b, parts, local_out);
    free(b);
    return w;
}

/* Alg. 2 / Alg. 4 lines 4-12 for given part boundaries b[0..np] (nnz split or
 * the Baseline's row/column blocks). */
int64_t or_partition_ptr_b(int64_t m, const int64_t *ptr, int64_t np, const int64_t *b,
                           or_part *parts, int64_t *local_out)
{
    int64_t w = 0;
    for (int64_t i = 0; i < np; i++) {
        or_part *p = &parts[i];
        p->start_idx = b[i];
        p->end_idx = b[i + 1] - 1;
        p->pad_ = 0;
        /* owned range (reading R9) */
        if (i == 0) p->owned_begin = 0;
        else {
            int64_t r = 0;
            while (r < m && ptr[r] < b[i]) r++;
            p->owned_begin = r;
        }
        if (i == np - 1) p->owned_end = m;
        else {
            int64_t r = 0;
            while (r < m && ptr[r] < b[i + 1]) r++;
            p->owned_end = r;
        }
        if (b[i] == b[i + 1]) {               /* empty part (reading R11) */
            p->start_row = -1; p->end_row = -1; p->start_flag = 0;
            if (local_out) local_out[w] = 0;
            w += 1;
            continue;
        }
        p->start_row = or_owner_linear(m, ptr, p->start_idx);
        p->end_row = or_owner_linear(m, ptr, p->end_idx);
        p->start_flag = p->start_idx > ptr[p->start_row] ? 1 : 0;
        for (int64_t k = 0; k <= p->end_row - p->start_row + 1; k++) {
            int64_t v = ptr[p->start_row + k];
            if (v < p->start_idx) v = p->start_idx;
            if (v > p->end_idx + 1) v = p->end_idx + 1;
            if (local_out) local_out[w] = v - p->start_idx;
            w += 1;
        }
    }
    return w;
}

/* Alg. 6 (COO->pCOO) on a row-sorted COO.  Reading R8: the paper's
 * BinarySearch on "A.row_ptr" (COO has none) becomes start_row =
 * row_idx[start_idx], end_row = row_idx[end_idx], start_flag = start_idx > 0
 * && row_idx[start_idx-1] == row_idx[start_idx]; owned_begin =
 * row_idx[b_i - 1] + 1 (R_0 = 0), owned_end = next part's owned_begin (R_np=m). */
void or_partition_coo_b(int64_t m, const int64_t *row_idx, int64_t np, const int64_t *b, or_part *parts);

void or_partition_coo(int64_t m, int64_t nnz, const int64_t *row_idx, int64_t np, or_part *parts)
{
    int64_t *b = (int64_t *)malloc((size_t)(np + 1) * sizeof(int64_t));
    or_nnz_boundaries(nnz, np, b);
    or_partition_coo_b(m, row_idx, np, b, parts);
    free(b);
}

/* Alg. 6 for given part boundaries b[0..np]. */
void or_partition_coo_b(int64_t m, const int64_t *row_idx, int64_t np, const int64_t *b, or_part *parts)
{
    for (int64_t i = 0; i < np; i++) {
        or_part *p = &parts[i];
        p->start_idx = b[i];
        p->end_idx = b[i + 1] - 1;
        p->pad_ = 0;
        p->owned_begin = (i == 0) ? 0 : (b[i] == 0 ? 0 : row_idx[b[i] - 1] + 1);
        if (i == np - 1) p->owned_end = m;
        else p->owned_end = (b[i + 1] == 0) ? 0 : row_idx[b[i + 1] - 1] + 1;
        if (b[i] == b[i + 1]) { p->start_row = -1; p->end_row = -1; p->start_flag = 0; continue; }
        p->start_row = row_idx[p->start_idx];
        p->end_row = row_idx[p->end_idx];
        p->start_flag = (p->start_idx > 0 && row_idx[p->start_idx - 1] == row_idx[p->start_idx]) ? 1 : 0;
    }
}

/* ------------------------------------------------------------------------ */
/* The partitioned executor: per-part PURE products, then  */
/* a beta-deferred merge.  Reading R6: Alg. 3/7's printed fix-up ("tmp =      */
/* y[start_row]; y <- py; y -= tmp*beta") double-counts; instead every part   */
/* computes pure sums and alpha, beta are applied exactly once per row.       */
/* Reading R7: Alg. 5's truncated "y =" is y = alpha * sum_i py_i + beta*y.   */
/* ------------------------------------------------------------------------ */

/* Row formats (pCSR, pCOO): part i produces seg_i[r] for r in
 * [start_row, end_row] over its own nonzeros only (Alg. 3 l.4-7).
 * Merge (Sec. 4.3): y_r = alpha * (sum over the parts
 * covering r, in part order) + beta * y_in_r; rows no part covers (empty
 * rows) get alpha*0 + beta*y_in. */
void or_exec_csr(int64_t m, const int64_t *row_ptr, const int32_t *col_idx,
                 const void *val, int dtype, const void *x, void *y,
                 double alpha, double beta, int64_t np)
{
    or_part *parts = (or_part *)malloc((size_t)np * sizeof(or_part));
    int64_t nloc = or_partition_ptr(m, row_ptr, np, parts, NULL);
    int64_t *loc = (int64_t *)malloc((size_t)nloc * sizeof(int64_t));
    or_partition_ptr(m, row_ptr, np, parts, loc);
    double *sum = (double *)calloc((size_t)(m > 0 ? m : 1), sizeof(double));
    int64_t w = 0;
    for (int64_t i = 0; i < np; i++) {
        or_part *p = &parts[i];
        if (p->start_row < 0) { w += 1; continue; }
        int64_t rows = p->end_row - p->start_row + 1;
        const int64_t *lp = loc + w;
        for (int64_t k = 0; k < rows; k++) {       /* csrSpMVKernel on the view */
            double seg = 0.0;
            if (alpha != 0.0)
                for (int64_t j = lp[k]; j < lp[k + 1]; j++) {
                    int64_t g = p->start_idx + j;  /* val = A.csr[start_idx] (Alg. 3 l.4) */
                    seg = seg + get_val(val, dtype, g) * get_val(x, dtype, col_idx[g]);
                }
            sum[p->start_row + k] = sum[p->start_row + k] + seg;   /* merge, part order */
        }
        w += rows + 1;
    }
    for (int64_t r = 0; r < m; r++) put_val(y, dtype, r, finish(alpha, sum[r], beta, y, dtype, r));
    free(sum); free(loc); free(parts);
}

void or_exec_coo(int64_t m, int64_t nnz, const int64_t *row_idx, const int32_t *col_idx,
                 const void *val, int dtype, const void *x, void *y,
                 double alpha, double beta, int64_t np)
{
    or_part *parts = (or_part *)malloc((size_t)np * sizeof(or_part));
    or_partition_coo(m, nnz, row_idx, np, parts);
    double *sum = (double *)calloc((size_t)(m > 0 ? m : 1), sizeof(double));
    for (int64_t i = 0; i < np; i++) {
        or_part *p = &parts[i];
        if (p->start_row < 0) continue;
        int64_t rows = p->end_row - p->start_row + 1;
        double *seg = (double *)calloc((size_t)rows, sizeof(double));
        if (alpha != 0.0)
            for (int64_t k = p->start_idx; k <= p->end_idx; k++)
                seg[row_idx[k] - p->start_row] = seg[row_idx[k] - p->start_row]
                    + get_val(val, dtype, k) * get_val(x, dtype, col_idx[k]);
        for (int64_t k = 0; k < rows; k++) sum[p->start_row + k] = sum[p->start_row + k] + seg[k];
        free(seg);
    }
    for (int64_t r = 0; r < m; r++) put_val(y, dtype, r, finish(alpha, sum[r], beta, y, dtype, r));
    free(sum); free(parts);
}

/* Unsorted COO (Sec. 3.2.3): "if the elements are unsorted ... elements in a
 * particular partition can spread among the entire matrix".  The nnz split is by position in the
 * given triplet order (Alg. 6 l.2-3, b_i = floor(i*nnz/np)); a part's rows are not contiguous, so
 * its descriptor reports the smallest and largest row it touches (reading R25), no flag and no
 * owned rows, and -- as the paper says for this case -- the merge is the column-style one: every
 * part produces a full-length partial y (like pCSC), summed in part order. */
void or_partition_coo_unsorted(int64_t nnz, const int64_t *row_idx, int64_t np, or_part *parts)
{
    int64_t *b = (int64_t *)malloc((size_t)(np + 1) * sizeof(int64_t));
    or_nnz_boundaries(nnz, np, b);
    for (int64_t i = 0; i < np; i++) {
        or_part *p = &parts[i];
        p->start_idx = b[i];
        p->end_idx = b[i + 1] - 1;
        p->pad_ = 0;
        p->start_flag = 0;
        p->owned_begin = 0;
        p->owned_end = 0;
        p->start_row = -1;
        p->end_row = -1;
        for (int64_t k = b[i]; k < b[i + 1]; k++) {
            if (p->start_row < 0 || row_idx[k] < p->start_row) p->start_row = row_idx[k];
            if (p->end_row < 0 || row_idx[k] > p->end_row) p->end_row = row_idx[k];
        }
    }
    free(b);
}

void or_exec_coo_unsorted(int64_t m, int64_t nnz, const int64_t *row_idx, const int32_t *col_idx,
                          const void *val, int dtype, const void *x, void *y,
                          double alpha, double beta, int64_t np)
{
    or_part *parts = (or_part *)malloc((size_t)np * sizeof(or_part));
    or_partition_coo_unsorted(nnz, row_idx, np, parts);
    double *sum_y = (double *)calloc((size_t)(m > 0 ? m : 1), sizeof(double));
    double *py = (double *)malloc((size_t)(m > 0 ? m : 1) * sizeof(double));
    for (int64_t i = 0; i < np; i++) {
        for (int64_t r = 0; r < m; r++) py[r] = 0.0;
        if (alpha != 0.0)
            for (int64_t k = parts[i].start_idx; k <= parts[i].end_idx; k++)
                py[row_idx[k]] = py[row_idx[k]] + get_val(val, dtype, k) * get_val(x, dtype, col_idx[k]);
        for (int64_t r = 0; r < m; r++) sum_y[r] = sum_y[r] + py[r];   /* sum_y += py[i] */
    }
    for (int64_t r = 0; r < m; r++) put_val(y, dtype, r, finish(alpha, sum_y[r], beta, y, dtype, r));
    free(py); free(sum_y); free(parts);
}

/* Column format (pCSC, Alg. 5; Sec. 4.3): part i
 * scatters its columns' nonzeros into its own full-length py_i; the merge is
 * sum_y = sum_i py_i (part order), y = alpha*sum_y + beta*y_in. */
void or_exec_csc(int64_t m, int64_t n, const int64_t *col_ptr, const int32_t *row_idx,
                 const void *val, int dtype, const void *x, void *y,
                 double alpha, double beta, int64_t np)
{
    or_part *parts = (or_part *)malloc((size_t)np * sizeof(or_part));
    int64_t nloc = or_partition_ptr(n, col_ptr, np, parts, NULL);
    int64_t *loc = (int64_t *)malloc((size_t)nloc * sizeof(int64_t));
    or_partition_ptr(n, col_ptr, np, parts, loc);
    double *sum_y = (double *)calloc((size_t)(m > 0 ? m : 1), sizeof(double));
    double *py = (double *)malloc((size_t)(m > 0 ? m : 1) * sizeof(double));
    int64_t w = 0;
    for (int64_t i = 0; i < np; i++) {
        or_part *p = &parts[i];
        for (int64_t r = 0; r < m; r++) py[r] = 0.0;
        if (p->start_row >= 0) {
            int64_t cols = p->end_row - p->start_row + 1;
            const int64_t *lp = loc + w;
            if (alpha != 0.0)
                for (int64_t k = 0; k < cols; k++)
                    for (int64_t j = lp[k]; j < lp[k + 1]; j++) {
                        int64_t g = p->start_idx + j;
                        py[row_idx[g]] = py[row_idx[g]]
                            + get_val(val, dtype, g) * get_val(x, dtype, p->start_row + k);
                    }
            w += cols + 1;
        } else {
            w += 1;
        }
        for (int64_t r = 0; r < m; r++) sum_y[r] = sum_y[r] + py[r];   /* sum_y += py[i] */
    }
    for (int64_t r = 0; r < m; r++) put_val(y, dtype, r, finish(alpha, sum_y[r], beta, y, dtype, r));
    free(py); free(sum_y); free(loc); free(parts);
}

/* merge_parts_to_csr: rebuild the global row_ptr from the parts'
 * descriptors and local pointers alone.  row_ptr[r+1] - row_ptr[r] is the sum
 * over the parts covering r of (local[k+1] - local[k]).  Used by the
 * merge-of-partition round-trip invariant. */
void or_merge_parts_to_ptr(int64_t m, int64_t np, const or_part *parts,
                           const int64_t *local, int64_t *ptr_out)
{
    int64_t *len = (int64_t *)calloc((size_t)(m > 0 ? m : 1), sizeof(int64_t));
    int64_t w = 0;
    for (int64_t i = 0; i < np; i++) {
        const or_part *p = &parts[i];
        if (p->start_row < 0) { w += 1; continue; }
        int64_t rows = p->end_row - p->start_row + 1;
        for (int64_t k = 0; k < rows; k++) len[p->start_row + k] += local[w + k + 1] - local[w + k];
        w += rows + 1;
    }
    ptr_out[0] = 0;
    for (int64_t r = 0; r < m; r++) ptr_out[r + 1] = ptr_out[r] + len[r];
    free(len);
}

/* ------------------------------------------------------------------------ */
/* Conjugate gradient (Hestenes & Stiefel 1952, the textbook algorithm) for a */
/* symmetric positive definite CSR matrix, the iterative-solver application   */
/* of SpMV (Sec. 6).  fp64 throughout; A*p by or_spmv_csr (alpha=1,    */
/* beta=0).  x0 in x; stops when ||r|| <= tol*||b|| or after maxit iterations */
/* (the residual is tested after every iteration).  Writes the iteration      */
/* count and ||r||/||b||.                                                      */
/* ------------------------------------------------------------------------ */
void or_cg_csr(int64_t m, const int64_t *row_ptr, const int32_t *col_idx, const double *val,
               const double *b, double *x, double tol, int64_t maxit, int64_t *iters, double *relres)
{
    double *r = (double *)malloc((size_t)(m > 0 ? m : 1) * sizeof(double));
    double *p = (double *)malloc((size_t)(m > 0 ? m : 1) * sizeof(double));
    double *ap = (double *)malloc((size_t)(m > 0 ? m : 1) * sizeof(double));
    or_spmv_csr(m, row_ptr, col_idx, val, OR_F64, x, ap, 1.0, 0.0);      /* ap = A x0 */
    double rs = 0.0, bn = 0.0;
    for (int64_t i = 0; i < m; i++) {
        r[i] = b[i] - ap[i];
        p[i] = r[i];
        rs += r[i] * r[i];
        bn += b[i] * b[i];
    }
    int64_t it = 0;
    while (!(rs <= tol * tol * bn) && it < maxit) {
        it++;
        or_spmv_csr(m, row_ptr, col_idx, val, OR_F64, p, ap, 1.0, 0.0);  /* ap = A p */
        double pap = 0.0;
        for (int64_t i = 0; i < m; i++) pap += p[i] * ap[i];
        double alpha = rs / pap, rs_new = 0.0;
        for (int64_t i = 0; i < m; i++) {
            x[i] += alpha * p[i];
            r[i] -= alpha * ap[i];
            rs_new += r[i] * r[i];
        }
        if (rs_new <= tol * tol * bn) { rs = rs_new; break; }
        double beta = rs_new / rs;
        for (int64_t i = 0; i < m; i++) p[i] = r[i] + beta * p[i];
        rs = rs_new;
    }
    *iters = it;
    *relres = bn > 0.0 ? sqrt(rs / bn) : sqrt(rs);
    free(r); free(p); free(ap);
}
