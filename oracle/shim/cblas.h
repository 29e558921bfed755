/* Minimal CBLAS declarations so the reference (/root/reference/proj) compiles
 * against the LP64 OpenBLAS 0.3.15 that ships inside the image's
 * opencv_python_headless wheel (it exports unprefixed cblas_* symbols).
 * Only the four GEMM entry points the reference calls are declared
 * (reference proj/src/contraction.cpp:46-72, proj/src/bench.cpp:53-68).
 * Test infrastructure only: used to build oracle/_ref, never the product. */
#ifndef QTNG_ORACLE_CBLAS_SHIM_H
#define QTNG_ORACLE_CBLAS_SHIM_H
#ifdef __cplusplus
extern "C" {
#endif

enum CBLAS_ORDER { CblasRowMajor = 101, CblasColMajor = 102 };
enum CBLAS_TRANSPOSE { CblasNoTrans = 111, CblasTrans = 112, CblasConjTrans = 113 };

void cblas_sgemm(enum CBLAS_ORDER order, enum CBLAS_TRANSPOSE ta, enum CBLAS_TRANSPOSE tb,
                 int m, int n, int k, float alpha, const float* a, int lda,
                 const float* b, int ldb, float beta, float* c, int ldc);
void cblas_dgemm(enum CBLAS_ORDER order, enum CBLAS_TRANSPOSE ta, enum CBLAS_TRANSPOSE tb,
                 int m, int n, int k, double alpha, const double* a, int lda,
                 const double* b, int ldb, double beta, double* c, int ldc);
void cblas_cgemm(enum CBLAS_ORDER order, enum CBLAS_TRANSPOSE ta, enum CBLAS_TRANSPOSE tb,
                 int m, int n, int k, const void* alpha, const void* a, int lda,
                 const void* b, int ldb, const void* beta, void* c, int ldc);
void cblas_zgemm(enum CBLAS_ORDER order, enum CBLAS_TRANSPOSE ta, enum CBLAS_TRANSPOSE tb,
                 int m, int n, int k, const void* alpha, const void* a, int lda,
                 const void* b, int ldb, const void* beta, void* c, int ldc);

#ifdef __cplusplus
}
#endif
#endif
