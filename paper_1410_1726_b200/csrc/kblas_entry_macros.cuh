// kblas_entry_macros.cuh — the BLAS-style extern "C" entry points of one
// precision (sync, _async, _offset, _offset_async, _mgpu, _mgpu_async), as
// macros expanded by kblas_<p>.cu.
#pragma once
#include "kblas_impl.cuh"

#define KB_GEMV(P, T)                                                                                        \
  int kblas_##P##gemv(char trans, int m, int n, T alpha, const T *dA, int lda, const T *dx, int incx, T beta,   \
                      T *dy, int incy) {                                                                       \
    return gemv_entry<T>(trans, m, n, alpha, dA, lda, dx, incx, beta, dy, incy, 0, 0, 0);                      \
  }                                                                                                            \
  int kblas_##P##gemv_async(char trans, int m, int n, T alpha, const T *dA, int lda, const T *dx, int incx,    \
                            T beta, T *dy, int incy, cudaStream_t s) {                                         \
    return gemv_entry<T>(trans, m, n, alpha, dA, lda, dx, incx, beta, dy, incy, 0, 0, s);                      \
  }                                                                                                            \
  int kblas_##P##gemv_offset(char trans, int m, int n, T alpha, const T *dA, int lda, const T *dx, int incx,   \
                             T beta, T *dy, int incy, int offset_r, int offset_c) {                            \
    return gemv_entry<T>(trans, m, n, alpha, dA, lda, dx, incx, beta, dy, incy, offset_r, offset_c, 0);        \
  }                                                                                                            \
  int kblas_##P##gemv_offset_async(char trans, int m, int n, T alpha, const T *dA, int lda, const T *dx,       \
                                   int incx, T beta, T *dy, int incy, int offset_r, int offset_c,             \
                                   cudaStream_t s) {                                                           \
    return gemv_entry<T>(trans, m, n, alpha, dA, lda, dx, incx, beta, dy, incy, offset_r, offset_c, s);        \
  }                                                                                                            \
  int kblas_##P##gemv_mgpu(char trans, int m, int n, T alpha, T *const *dA, int lda, T *const *dx, int incx,   \
                           T beta, T *const *dy, int incy, int ngpus, int nb, const int *device_ids) {         \
    char t = (char)(trans | 0x20);                                                                             \
    if (t != 'n' && t != 't' && t != 'c') return -1;                                                           \
    if (m < 0) return -2;                                                                                      \
    if (n < 0) return -3;                                                                                      \
    if (lda < std::max(1, m)) return -6;                                                                       \
    if (incx != 1) return -8;                                                                                  \
    if (incy != 1) return -11;                                                                                 \
    return mgpu_entry<T>(true, t, false, m, n, alpha, dA, lda, dx, beta, dy, ngpus, nb, device_ids);          \
  }                                                                                                            \
  int kblas_##P##gemv_mgpu_async(char trans, int m, int n, T alpha, T *const *dA, int lda, T *const *dx,      \
                                 int incx, T beta, T *const *dy, int incy, int ngpus, int nb,                 \
                                 const int *device_ids, cudaStream_t const *streams) {                        \
    char t = (char)(trans | 0x20);                                                                             \
    if (t != 'n' && t != 't' && t != 'c') return -1;                                                           \
    if (m < 0) return -2;                                                                                      \
    if (n < 0) return -3;                                                                                      \
    if (lda < std::max(1, m)) return -6;                                                                       \
    if (incx != 1) return -8;                                                                                  \
    if (incy != 1) return -11;                                                                                 \
    if (streams == nullptr) return -16;                                                                        \
    return mgpu_entry<T>(true, t, false, m, n, alpha, dA, lda, dx, beta, dy, ngpus, nb, device_ids, streams); \
  }

#define KB_SYMV(NAME, T, HERM)                                                                                \
  int kblas_##NAME(char uplo, int n, T alpha, const T *dA, int lda, const T *dx, int incx, T beta, T *dy,      \
                   int incy) {                                                                                 \
    return symv_entry<T>(uplo, HERM, n, alpha, dA, lda, dx, incx, beta, dy, incy, 0, 0);                       \
  }                                                                                                            \
  int kblas_##NAME##_async(char uplo, int n, T alpha, const T *dA, int lda, const T *dx, int incx, T beta,     \
                           T *dy, int incy, cudaStream_t s) {                                                  \
    return symv_entry<T>(uplo, HERM, n, alpha, dA, lda, dx, incx, beta, dy, incy, 0, s);                       \
  }                                                                                                            \
  int kblas_##NAME##_offset(char uplo, int n, T alpha, const T *dA, int lda, const T *dx, int incx, T beta,    \
                            T *dy, int incy, int offset) {                                                     \
    return symv_entry<T>(uplo, HERM, n, alpha, dA, lda, dx, incx, beta, dy, incy, offset, 0);                  \
  }                                                                                                            \
  int kblas_##NAME##_offset_async(char uplo, int n, T alpha, const T *dA, int lda, const T *dx, int incx,      \
                                  T beta, T *dy, int incy, int offset, cudaStream_t s) {                       \
    return symv_entry<T>(uplo, HERM, n, alpha, dA, lda, dx, incx, beta, dy, incy, offset, s);                  \
  }                                                                                                            \
  int kblas_##NAME##_mgpu(char uplo, int n, T alpha, T *const *dA, int lda, T *const *dx, int incx, T beta,    \
                          T *const *dy, int incy, int ngpus, int nb, const int *device_ids) {                  \
    const char u = (char)(uplo | 0x20);                                                                        \
    if (u != 'l' && u != 'u') return -1;                                                                       \
    if (n < 0) return -2;                                                                                      \
    if (lda < std::max(1, n)) return -5;                                                                       \
    if (incx != 1) return -7;                                                                                  \
    if (incy != 1) return -10;                                                                                 \
    return mgpu_entry<T>(false, u, HERM, n, n, alpha, dA, lda, dx, beta, dy, ngpus, nb, device_ids);          \
  }                                                                                                            \
  int kblas_##NAME##_mgpu_async(char uplo, int n, T alpha, T *const *dA, int lda, T *const *dx, int incx,      \
                                T beta, T *const *dy, int incy, int ngpus, int nb, const int *device_ids,     \
                                cudaStream_t const *streams) {                                                 \
    const char u = (char)(uplo | 0x20);                                                                        \
    if (u != 'l' && u != 'u') return -1;                                                                       \
    if (n < 0) return -2;                                                                                      \
    if (lda < std::max(1, n)) return -5;                                                                       \
    if (incx != 1) return -7;                                                                                  \
    if (incy != 1) return -10;                                                                                 \
    if (streams == nullptr) return -14;                                                                        \
    return mgpu_entry<T>(false, u, HERM, n, n, alpha, dA, lda, dx, beta, dy, ngpus, nb, device_ids, streams); \
  }
