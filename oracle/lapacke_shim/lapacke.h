/* Minimal LAPACKE prototypes so the reference umbrella headers that include
 * dense_eig.hpp compile in this image (no lapacke.h is installed).
 * libktune_ref.so calls neither; libktune_ref_eig.so (the reference's Lanczos)
 * calls LAPACKE_dsteqr, resolved from the OpenBLAS the python env bundles
 * (oracle/Makefile). TEST INFRASTRUCTURE. */
#pragma once
typedef int lapack_int;
#define LAPACK_ROW_MAJOR 101
#define LAPACK_COL_MAJOR 102
extern "C" {
lapack_int LAPACKE_dsteqr(int matrix_layout, char compz, lapack_int n, double* d, double* e,
                          double* z, lapack_int ldz);
lapack_int LAPACKE_dgeev(int matrix_layout, char jobvl, char jobvr, lapack_int n, double* a,
                         lapack_int lda, double* wr, double* wi, double* vl, lapack_int ldvl,
                         double* vr, lapack_int ldvr);
}
