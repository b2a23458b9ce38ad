/* Test-infrastructure shim: CBLAS prototypes for the OpenBLAS shared object
 * bundled in the image (opencv_python_headless.libs, LP64).  Only the entry
 * points the reference calls are declared.  Not product code. */
#pragma once
#ifdef __cplusplus
extern "C" {
#endif
enum CBLAS_ORDER { CblasRowMajor = 101, CblasColMajor = 102 };
enum CBLAS_TRANSPOSE { CblasNoTrans = 111, CblasTrans = 112, CblasConjTrans = 113 };
enum CBLAS_UPLO { CblasUpper = 121, CblasLower = 122 };
enum CBLAS_DIAG { CblasNonUnit = 131, CblasUnit = 132 };
enum CBLAS_SIDE { CblasLeft = 141, CblasRight = 142 };
void cblas_dgemm(enum CBLAS_ORDER, enum CBLAS_TRANSPOSE, enum CBLAS_TRANSPOSE, int, int, int,
                 double, const double*, int, const double*, int, double, double*, int);
void cblas_dtrsm(enum CBLAS_ORDER, enum CBLAS_SIDE, enum CBLAS_UPLO, enum CBLAS_TRANSPOSE,
                 enum CBLAS_DIAG, int, int, double, const double*, int, double*, int);
void cblas_dgemv(enum CBLAS_ORDER, enum CBLAS_TRANSPOSE, int, int, double, const double*, int,
                 const double*, int, double, double*, int);
void cblas_dtrsv(enum CBLAS_ORDER, enum CBLAS_UPLO, enum CBLAS_TRANSPOSE, enum CBLAS_DIAG, int,
                 const double*, int, double*, int);
double cblas_ddot(int, const double*, int, const double*, int);
void cblas_daxpy(int, double, const double*, int, double*, int);
double cblas_dnrm2(int, const double*, int);
void cblas_dscal(int, double, double*, int);
#ifdef __cplusplus
}
#endif
