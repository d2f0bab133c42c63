/*
 * ktune_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's CPU algorithms for the SpMV hot
 * path (Xabclib/OpenATLib "ktune", /root/reference/proj/include/ktune/).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load this; the product (libktb) never links or calls it.
 *
 * Parity of this restatement is pinned against the reference itself: the
 * reference headers are compiled by oracle/Makefile into oracle/_ref/ and
 * tests/golden/ holds vectors produced by that build (tests/golden/make_golden.py).
 *
 * Conventions follow the reference: index_t = int64 (common.hpp:13), values
 * fp64, every accumulation strictly left to right, no FMA contraction
 * (built with -ffp-contract=off so results are bitwise equal to the
 * reference compiled with its default x86-64 flags).
 */
#ifndef KTUNE_ORACLE_H
#define KTUNE_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error codes: 0 ok, otherwise an index into ko_error_message(). */
const char* ko_error_message(int code);

/* csr.hpp:38-54 CsrMatrix::validate / SymCsrMatrix::validate */
int ko_validate(int64_t n, const int64_t* row_ptr, int64_t nnz, const int64_t* col_idx,
                int upper_only);

/* csr.hpp:69-78 spmv_ref */
void ko_spmv_ref(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                 const double* values, const double* x, double* y);

/* csr.hpp:88-123 expand_symmetric: count pass, then fill pass. */
int64_t ko_expand_symmetric_nnz(int64_t n, const int64_t* row_ptr, const int64_t* col_idx);
void ko_expand_symmetric(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                         const double* values, int64_t* out_row_ptr, int64_t* out_col_idx,
                         double* out_values);

/* partition.hpp:28-55 build_row_partition. scheme 0 = row_based, 1 = nnz_balanced. */
int ko_build_row_partition(const int64_t* row_ptr, int64_t n, int num_workers, int scheme,
                           int64_t* boundaries /* num_workers+1 */);

/* partition.hpp:73-96 build_reduction_regions */
void ko_build_reduction_regions(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                                int num_workers, const int64_t* boundaries, int64_t* lo,
                                int64_t* hi);

/* bss.hpp:34-69 build_bss_plan: ko_bss_count returns total_slices and the
 * clamped jl; ko_bss_fill writes the arrays (caller-allocated). */
int ko_bss_count(int64_t n, const int64_t* row_ptr, int64_t jl, int64_t* jl_eff,
                 int64_t* total_slices);
void ko_bss_fill(int64_t n, const int64_t* row_ptr, int64_t jl_eff, int64_t* slice_start,
                 int64_t* slice_len, int64_t* slice_row, int64_t* lane_slice_ptr,
                 int64_t* row_slice_ptr, uint8_t* row_start_flag);

/* spmv.hpp:74-86 (U1/U2 row blocks) */
void ko_spmv_row_blocks(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                        const double* values, int num_workers, const int64_t* boundaries,
                        const double* x, double* y);

/* spmv.hpp:127-166 (U3 branchless slice loop / U4 flag scan) + :91-101 combine */
void ko_spmv_bss(int u4, int64_t n, const int64_t* col_idx, const double* values, int64_t jl,
                 const int64_t* slice_start, const int64_t* slice_len,
                 const int64_t* lane_slice_ptr, const int64_t* row_slice_ptr,
                 const uint8_t* row_start_flag, const double* x, double* sums, double* y);

/* spmv.hpp:180-234 spmv_sym (S1/S2/S3). kernel 0=s1,1=s2,2=s3. pool_size is
 * the WorkerPool size (reduction chunk count, spmv.hpp:222). scratch holds
 * num_workers*n doubles; contents on entry are irrelevant except where the
 * reference would read stale data (it never does). */
void ko_spmv_sym(int kernel, int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                 const double* values, int num_workers, const int64_t* boundaries,
                 const int64_t* lo, const int64_t* hi, int pool_size, const double* x,
                 double* y, double* scratch);

/* lanczos.hpp:17-29 detail::seeded_vector (splitmix64 -> U[-1,1)) */
void ko_seeded_vector(int64_t n, uint64_t seed, double* out);
/* autotune.hpp:188-196 detail::probe_vector (LCG -> [0.5,1.5)) */
void ko_probe_vector(int64_t n, double* out);
/* autotune.hpp:198-204 detail::outputs_match */
int ko_outputs_match(int64_t n, const double* y, const double* ref);

/* common.hpp:33-60 serial BLAS-1 */
double ko_dot(int64_t n, const double* a, const double* b);
double ko_norm2(int64_t n, const double* a);

/* gmres.hpp:16-173 restarted GMRES(m) with MGS (ortho.hpp:88-94), x0 = 0,
 * no preconditioner, no restart adaptation. The operator is spmv_ref on the
 * given CSR. history (max_iters doubles) receives the recurrence residuals. */
typedef struct {
    int64_t iterations;
    int64_t restarts;
    int64_t spmv_calls;
    int converged;
    int breakdown;
    int fault_convergence;
    double recurrence_residual;
    double true_residual;
} ko_gmres_result;

int ko_gmres_mgs(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                 const double* values, const double* b, int64_t m, double tol,
                 int64_t max_iters, double* x, double* history, ko_gmres_result* res);

/* ilu0.hpp:23-69 ilu0_factorize on the pattern of A (in place on a copy of
 * values): diag_ptr[n] and values[nnz] receive the combined L\U factors.
 * Returns 0, or -(1 + i) for "structurally missing diagonal in row i", or
 * (1 + i) for "zero pivot at row i" (the reference's first raise). */
int64_t ko_ilu0_factorize(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                          double* values, int64_t* diag_ptr);
/* ilu0.hpp:73-87 ilu0_apply: forward (unit L) then backward (U) sweeps. */
void ko_ilu0_apply(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                   const double* values, const int64_t* diag_ptr, const double* r, double* z);

#ifdef __cplusplus
}
#endif

#endif
