/* Test-infrastructure shim: LAPACKE prototypes (LP64) for the bundled OpenBLAS.
 * Not product code. */
#pragma once
#ifdef __cplusplus
extern "C" {
#endif
typedef int lapack_int;
#define LAPACK_ROW_MAJOR 101
#define LAPACK_COL_MAJOR 102
lapack_int LAPACKE_dpotrf(int, char, lapack_int, double*, lapack_int);
lapack_int LAPACKE_dsytrf(int, char, lapack_int, double*, lapack_int, lapack_int*);
lapack_int LAPACKE_dgesdd(int, char, lapack_int, lapack_int, double*, lapack_int, double*,
                          double*, lapack_int, double*, lapack_int);
lapack_int LAPACKE_dgesvd(int, char, char, lapack_int, lapack_int, double*, lapack_int, double*,
                          double*, lapack_int, double*, lapack_int, double*);
lapack_int LAPACKE_dsyev(int, char, char, lapack_int, double*, lapack_int, double*);
#ifdef __cplusplus
}
#endif
