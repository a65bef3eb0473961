/*
 * streamed.c — C restatement of the reference oracle, TEST INFRASTRUCTURE.
 *
 * Restates blockmv/reference.py:39-59 (naive_gemv, naive_symv_hemv) in
 * wide precision (double / double complex, reference.py:15-16) without
 * materialising the mirrored dense matrix (reference.py:19-36 builds
 * ~5 matrix-sized temporaries, which does not fit for N >= 32k).  Each
 * stored column is streamed once: for SYMV/HEMV every stored element
 * a(i,j) contributes a(i,j) x_j to y_i and op(a(i,j)) x_i to y_j, with
 * op = conj for Hermitian and the Hermitian diagonal read as real
 * (reference.py:33-35).  Columns are split over OpenMP threads with
 * thread-private accumulators, summed at the end.
 *
 * Used by tests/ (large-N checks), bench.py's cpu_baseline and the
 * `--impl reference` CPU arm.  Never linked into the product.
 *
 * Element codes: 's' float, 'd' double, 'c' float complex, 'z' double
 * complex (interleaved re, im).  alpha / beta / y_out are wide: double[2]
 * per element (imaginary part 0 for real precisions).
 */
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static inline void ld_elem(char p, const void *A, long long k, double *re, double *im) {
  switch (p) {
    case 's': *re = ((const float *)A)[k]; *im = 0.0; break;
    case 'd': *re = ((const double *)A)[k]; *im = 0.0; break;
    case 'c': *re = ((const float *)A)[2 * k]; *im = ((const float *)A)[2 * k + 1]; break;
    default: *re = ((const double *)A)[2 * k]; *im = ((const double *)A)[2 * k + 1]; break;
  }
}

static int nthreads_of(int want) {
#ifdef _OPENMP
  return want > 0 ? want : omp_get_max_threads();
#else
  (void)want;
  return 1;
#endif
}

/* y_out[i] = alpha * acc[i] + beta * y[i]  (beta == 0: y not read) */
static void finish(char p, long long len, const double *alpha, const double *beta, const void *y,
                   const double *acc, double *y_out) {
  const int bz = beta[0] == 0.0 && beta[1] == 0.0;
  for (long long i = 0; i < len; ++i) {
    double ar = acc[2 * i], ai = acc[2 * i + 1];
    double r = alpha[0] * ar - alpha[1] * ai, im = alpha[0] * ai + alpha[1] * ar;
    if (!bz) {
      double yr, yi;
      ld_elem(p, y, i, &yr, &yi);
      r += beta[0] * yr - beta[1] * yi;
      im += beta[0] * yi + beta[1] * yr;
    }
    y_out[2 * i] = r;
    y_out[2 * i + 1] = im;
  }
}

/* naive_gemv (reference.py:39-50), op in {n, t, c}. */
int oracle_gemv(char p, char trans, int m, int n, const double *alpha, const void *A, long long lda,
                const void *x, const double *beta, const void *y, double *y_out, int nthreads) {
  const int nt = nthreads_of(nthreads);
  const long long ylen = (trans == 'n') ? m : n;
  double *acc = (double *)calloc((size_t)ylen * 2, sizeof(double));
  if (!acc) return 1;
  if (trans == 'n') {
    double *priv = (double *)calloc((size_t)nt * m * 2, sizeof(double));
    if (!priv) { free(acc); return 1; }
#pragma omp parallel num_threads(nt)
    {
      int t = 0;
#ifdef _OPENMP
      t = omp_get_thread_num();
#endif
      double *yb = priv + (size_t)t * m * 2;
#pragma omp for schedule(static)
      for (int j = 0; j < n; ++j) {
        double xr, xi;
        ld_elem(p, x, j, &xr, &xi);
        for (int i = 0; i < m; ++i) {
          double ar, ai;
          ld_elem(p, A, (long long)j * lda + i, &ar, &ai);
          yb[2 * i] += ar * xr - ai * xi;
          yb[2 * i + 1] += ar * xi + ai * xr;
        }
      }
    }
    for (int t = 0; t < nt; ++t)
      for (long long i = 0; i < 2LL * m; ++i) acc[i] += priv[(size_t)t * m * 2 + i];
    free(priv);
  } else {
    const int cj = trans == 'c';
#pragma omp parallel for schedule(static) num_threads(nt)
    for (int j = 0; j < n; ++j) {
      double sr = 0.0, si = 0.0;
      for (int i = 0; i < m; ++i) {
        double ar, ai, xr, xi;
        ld_elem(p, A, (long long)j * lda + i, &ar, &ai);
        if (cj) ai = -ai;
        ld_elem(p, x, i, &xr, &xi);
        sr += ar * xr - ai * xi;
        si += ar * xi + ai * xr;
      }
      acc[2 * j] = sr;
      acc[2 * j + 1] = si;
    }
  }
  finish(p, ylen, alpha, beta, y, acc, y_out);
  free(acc);
  return 0;
}

/* naive_symv_hemv (reference.py:53-59) from the stored triangle. */
int oracle_symv(char p, char uplo, int herm, int n, const double *alpha, const void *A, long long lda,
                const void *x, const double *beta, const void *y, double *y_out, int nthreads) {
  const int nt = nthreads_of(nthreads);
  const int lower = uplo == 'l';
  double *priv = (double *)calloc((size_t)nt * n * 2, sizeof(double));
  double *acc = (double *)calloc((size_t)n * 2, sizeof(double));
  if (!priv || !acc) { free(priv); free(acc); return 1; }
#pragma omp parallel num_threads(nt)
  {
    int t = 0;
#ifdef _OPENMP
    t = omp_get_thread_num();
#endif
    double *yb = priv + (size_t)t * n * 2;
#pragma omp for schedule(dynamic, 16)
    for (int j = 0; j < n; ++j) {
      double xjr, xji;
      ld_elem(p, x, j, &xjr, &xji);
      double dr, di;
      ld_elem(p, A, (long long)j * lda + j, &dr, &di);
      if (herm) di = 0.0;
      double sr = dr * xjr - di * xji, si = dr * xji + di * xjr;
      const int i0 = lower ? j + 1 : 0, i1 = lower ? n : j;
      for (int i = i0; i < i1; ++i) {
        double ar, ai, xr, xi;
        ld_elem(p, A, (long long)j * lda + i, &ar, &ai);
        ld_elem(p, x, i, &xr, &xi);
        yb[2 * i] += ar * xjr - ai * xji;
        yb[2 * i + 1] += ar * xji + ai * xjr;
        const double br = ar, bi = herm ? -ai : ai;
        sr += br * xr - bi * xi;
        si += br * xi + bi * xr;
      }
      yb[2 * j] += sr;
      yb[2 * j + 1] += si;
    }
  }
  for (int t = 0; t < nt; ++t)
    for (long long i = 0; i < 2LL * n; ++i) acc[i] += priv[(size_t)t * n * 2 + i];
  finish(p, n, alpha, beta, y, acc, y_out);
  free(priv);
  free(acc);
  return 0;
}

/* ||A_dense||_inf of the mirrored matrix (row sums of |a|) for the
 * tolerance bound (reference.py:62-66, test_acceptance.py:94). */
double oracle_symv_norm_inf(char p, char uplo, int herm, int n, const void *A, long long lda) {
  double *rs = (double *)calloc((size_t)n, sizeof(double));
  if (!rs) return -1.0;
  const int lower = uplo == 'l';
  for (int j = 0; j < n; ++j) {
    double dr, di;
    ld_elem(p, A, (long long)j * lda + j, &dr, &di);
    if (herm) di = 0.0;
    rs[j] += __builtin_sqrt(dr * dr + di * di);
    const int i0 = lower ? j + 1 : 0, i1 = lower ? n : j;
    for (int i = i0; i < i1; ++i) {
      double ar, ai;
      ld_elem(p, A, (long long)j * lda + i, &ar, &ai);
      const double a = __builtin_sqrt(ar * ar + ai * ai);
      rs[i] += a;
      rs[j] += a;
    }
  }
  double mx = 0.0;
  for (int i = 0; i < n; ++i) mx = rs[i] > mx ? rs[i] : mx;
  free(rs);
  return mx;
}

int oracle_max_threads(void) { return nthreads_of(0); }
