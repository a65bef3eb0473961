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
 * thread-private accumulators, summed at the end in thread order.
 *
 * Element sources.  The operand is read either from memory (a column-major
 * host buffer) or REGENERATED from a counter-based generator, so N = 60k /
 * 100k operands (28-160 GB) need no host copy at all (SURVEY §8c "panel-
 * streamed restatement ... regenerate the panel from (seed, block col)",
 * BASELINE.md §3.3).  The generator is stateless: element (i, j) of an
 * operand generated with (seed, gen_ld) at offset (ro, co) is
 *     u(k) = (splitmix64((seed << 36) + k) >> 11) * 2^-52 - 1,
 *     k = (j + co) * gen_ld + (i + ro)        real types,
 *     re = u(2k), im = u(2k + 1)              complex types,
 * rounded to float for s / c.  Every step is exact in IEEE double, so the
 * tests' torch restatement (oracle/gen.py) produces bit-identical device
 * operands; the value depends only on (seed, global row, global column),
 * not on the block-column layout, so mgpu panels regenerate per block
 * column j from (seed, j).
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

/* ------------------------------------------------------------ generator */
static inline unsigned long long mix64(unsigned long long z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

static inline double gen_u(unsigned long long seed, unsigned long long k) {
  return (double)(mix64((seed << 36) + k) >> 11) * 0x1.0p-52 - 1.0;
}

/* element (i, j) of the generated operand */
static inline void gen_elem(char p, unsigned long long seed, long long k, double *re, double *im) {
  switch (p) {
    case 's': *re = (double)(float)gen_u(seed, (unsigned long long)k); *im = 0.0; break;
    case 'd': *re = gen_u(seed, (unsigned long long)k); *im = 0.0; break;
    case 'c':
      *re = (double)(float)gen_u(seed, 2ULL * k);
      *im = (double)(float)gen_u(seed, 2ULL * k + 1);
      break;
    default: *re = gen_u(seed, 2ULL * k); *im = gen_u(seed, 2ULL * k + 1); break;
  }
}

/* where the operand's elements come from */
typedef struct {
  char p;
  const void *A;          /* memory source when non-NULL */
  long long lda;
  unsigned long long seed; /* generated source otherwise */
  long long gen_ld, ro, co;
} Src;

static inline void src_elem(const Src *s, long long i, long long j, double *re, double *im) {
  if (s->A)
    ld_elem(s->p, s->A, j * s->lda + i, re, im);
  else
    gen_elem(s->p, s->seed, (j + s->co) * s->gen_ld + (i + s->ro), re, im);
}

static int nthreads_of(int want) {
#ifdef _OPENMP
  return want > 0 ? want : omp_get_max_threads();
#else
  (void)want;
  return 1;
#endif
}

static inline int thread_id(void) {
#ifdef _OPENMP
  return omp_get_thread_num();
#else
  return 0;
#endif
}

static inline double cabs2(double r, double i) { return __builtin_sqrt(r * r + i * i); }

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

static double max_of(const double *v, long long n) {
  double mx = 0.0;
  for (long long i = 0; i < n; ++i) mx = v[i] > mx ? v[i] : mx;
  return mx;
}

/* naive_gemv (reference.py:39-50), op in {n, t, c}.  norm_out (optional):
 * ||op(A)||_inf, the row sums of |op(A)| (reference.py:62-66). */
static int gemv_src(const Src *S, char trans, int m, int n, const double *alpha, const void *x,
                    const double *beta, const void *y, double *y_out, int nthreads, double *norm_out) {
  const char p = S->p;
  const int nt = nthreads_of(nthreads);
  const long long ylen = (trans == 'n') ? m : n;
  double *acc = (double *)calloc((size_t)ylen * 2 + 1, sizeof(double));
  double *rs = (double *)calloc((size_t)ylen + 1, sizeof(double));
  if (!acc || !rs) { free(acc); free(rs); return 1; }
  if (trans == 'n') {
    double *priv = (double *)calloc((size_t)nt * m * 3 + 1, sizeof(double));
    if (!priv) { free(acc); free(rs); return 1; }
#pragma omp parallel num_threads(nt)
    {
      double *yb = priv + (size_t)thread_id() * m * 3;
      double *ab = yb + 2 * (size_t)m;
#pragma omp for schedule(static)
      for (int j = 0; j < n; ++j) {
        double xr, xi;
        ld_elem(p, x, j, &xr, &xi);
        for (int i = 0; i < m; ++i) {
          double ar, ai;
          src_elem(S, i, j, &ar, &ai);
          yb[2 * i] += ar * xr - ai * xi;
          yb[2 * i + 1] += ar * xi + ai * xr;
          if (norm_out) ab[i] += cabs2(ar, ai);
        }
      }
    }
    for (int t = 0; t < nt; ++t) {
      const double *yb = priv + (size_t)t * m * 3;
      for (long long i = 0; i < 2LL * m; ++i) acc[i] += yb[i];
      for (long long i = 0; i < m; ++i) rs[i] += yb[2 * m + i];
    }
    free(priv);
  } else {
    const int cj = trans == 'c';
#pragma omp parallel for schedule(static) num_threads(nt)
    for (int j = 0; j < n; ++j) {
      double sr = 0.0, si = 0.0, sa = 0.0;
      for (int i = 0; i < m; ++i) {
        double ar, ai, xr, xi;
        src_elem(S, i, j, &ar, &ai);
        if (cj) ai = -ai;
        ld_elem(p, x, i, &xr, &xi);
        sr += ar * xr - ai * xi;
        si += ar * xi + ai * xr;
        if (norm_out) sa += cabs2(ar, ai);
      }
      acc[2 * j] = sr;
      acc[2 * j + 1] = si;
      rs[j] = sa;
    }
  }
  finish(p, ylen, alpha, beta, y, acc, y_out);
  if (norm_out) *norm_out = max_of(rs, ylen);
  free(acc);
  free(rs);
  return 0;
}

/* naive_symv_hemv (reference.py:53-59) from the stored triangle.  norm_out
 * (optional): ||A_dense||_inf of the mirrored matrix (reference.py:19-36,
 * 62-66; test_acceptance.py:94). */
static int symv_src(const Src *S, char uplo, int herm, int n, const double *alpha, const void *x,
                    const double *beta, const void *y, double *y_out, int nthreads, double *norm_out) {
  const char p = S->p;
  const int nt = nthreads_of(nthreads);
  const int lower = uplo == 'l';
  double *priv = (double *)calloc((size_t)nt * n * 3 + 1, sizeof(double));
  double *acc = (double *)calloc((size_t)n * 2 + 1, sizeof(double));
  double *rs = (double *)calloc((size_t)n + 1, sizeof(double));
  if (!priv || !acc || !rs) { free(priv); free(acc); free(rs); return 1; }
#pragma omp parallel num_threads(nt)
  {
    double *yb = priv + (size_t)thread_id() * n * 3;
    double *ab = yb + 2 * (size_t)n;
#pragma omp for schedule(dynamic, 16)
    for (int j = 0; j < n; ++j) {
      double xjr, xji;
      ld_elem(p, x, j, &xjr, &xji);
      double dr, di;
      src_elem(S, j, j, &dr, &di);
      if (herm) di = 0.0;
      double sr = dr * xjr - di * xji, si = dr * xji + di * xjr;
      double sa = cabs2(dr, di);
      const int i0 = lower ? j + 1 : 0, i1 = lower ? n : j;
      for (int i = i0; i < i1; ++i) {
        double ar, ai, xr, xi;
        src_elem(S, i, j, &ar, &ai);
        ld_elem(p, x, i, &xr, &xi);
        yb[2 * i] += ar * xjr - ai * xji;
        yb[2 * i + 1] += ar * xji + ai * xjr;
        const double br = ar, bi = herm ? -ai : ai;
        sr += br * xr - bi * xi;
        si += br * xi + bi * xr;
        if (norm_out) {
          const double a = cabs2(ar, ai);
          ab[i] += a;
          sa += a;
        }
      }
      yb[2 * j] += sr;
      yb[2 * j + 1] += si;
      if (norm_out) ab[j] += sa;
    }
  }
  for (int t = 0; t < nt; ++t) {
    const double *yb = priv + (size_t)t * n * 3;
    for (long long i = 0; i < 2LL * n; ++i) acc[i] += yb[i];
    for (long long i = 0; i < n; ++i) rs[i] += yb[2 * (size_t)n + i];
  }
  finish(p, n, alpha, beta, y, acc, y_out);
  if (norm_out) *norm_out = max_of(rs, n);
  free(priv);
  free(acc);
  free(rs);
  return 0;
}

/* ------------------------------------------------ memory-source entries */
int oracle_gemv(char p, char trans, int m, int n, const double *alpha, const void *A, long long lda,
                const void *x, const double *beta, const void *y, double *y_out, int nthreads) {
  const Src S = {p, A, lda, 0, 0, 0, 0};
  return gemv_src(&S, trans, m, n, alpha, x, beta, y, y_out, nthreads, NULL);
}

int oracle_symv(char p, char uplo, int herm, int n, const double *alpha, const void *A, long long lda,
                const void *x, const double *beta, const void *y, double *y_out, int nthreads) {
  const Src S = {p, A, lda, 0, 0, 0, 0};
  return symv_src(&S, uplo, herm, n, alpha, x, beta, y, y_out, nthreads, NULL);
}

/* ||A_dense||_inf of the mirrored matrix (row sums of |a|) for the
 * tolerance bound (reference.py:62-66, test_acceptance.py:94). */
double oracle_symv_norm_inf(char p, char uplo, int herm, int n, const void *A, long long lda) {
  double *rs = (double *)calloc((size_t)n + 1, sizeof(double));
  if (!rs) return -1.0;
  const int lower = uplo == 'l';
  for (int j = 0; j < n; ++j) {
    double dr, di;
    ld_elem(p, A, (long long)j * lda + j, &dr, &di);
    if (herm) di = 0.0;
    rs[j] += cabs2(dr, di);
    const int i0 = lower ? j + 1 : 0, i1 = lower ? n : j;
    for (int i = i0; i < i1; ++i) {
      double ar, ai;
      ld_elem(p, A, (long long)j * lda + i, &ar, &ai);
      const double a = cabs2(ar, ai);
      rs[i] += a;
      rs[j] += a;
    }
  }
  const double mx = max_of(rs, n);
  free(rs);
  return mx;
}

/* --------------------------------------------- generated-source entries */
/* GEMV on the m x n operand generated with (seed, gen_ld) at (ro, co). */
int oracle_gemv_gen(char p, char trans, int m, int n, unsigned long long seed, long long gen_ld, long long ro,
                    long long co, const double *alpha, const void *x, const double *beta, const void *y,
                    double *y_out, double *norm_out, int nthreads) {
  const Src S = {p, NULL, 0, seed, gen_ld, ro, co};
  return gemv_src(&S, trans, m, n, alpha, x, beta, y, y_out, nthreads, norm_out);
}

/* SYMV / HEMV on the diagonal n x n block at (off, off) of the generated
 * operand; only the stored triangle is generated. */
int oracle_symv_gen(char p, char uplo, int herm, int n, unsigned long long seed, long long gen_ld, long long off,
                    const double *alpha, const void *x, const double *beta, const void *y, double *y_out,
                    double *norm_out, int nthreads) {
  const Src S = {p, NULL, 0, seed, gen_ld, off, off};
  return symv_src(&S, uplo, herm, n, alpha, x, beta, y, y_out, nthreads, norm_out);
}

/* Materialise the generated m x n operand (at (ro, co)) into a column-major
 * buffer of the element type with leading dimension ld_out. */
int oracle_gen_fill(char p, int m, int n, unsigned long long seed, long long gen_ld, long long ro, long long co,
                    void *out, long long ld_out, int nthreads) {
  const int nt = nthreads_of(nthreads);
#pragma omp parallel for schedule(static) num_threads(nt)
  for (int j = 0; j < n; ++j) {
    for (int i = 0; i < m; ++i) {
      double re, im;
      gen_elem(p, seed, ((long long)j + co) * gen_ld + (i + ro), &re, &im);
      const long long k = (long long)j * ld_out + i;
      switch (p) {
        case 's': ((float *)out)[k] = (float)re; break;
        case 'd': ((double *)out)[k] = re; break;
        case 'c': ((float *)out)[2 * k] = (float)re; ((float *)out)[2 * k + 1] = (float)im; break;
        default: ((double *)out)[2 * k] = re; ((double *)out)[2 * k + 1] = im; break;
      }
    }
  }
  return 0;
}

/* Only the stored triangle ('l': i >= j, 'u': i <= j) of the generated
 * n x n operand, into a column-major buffer: the other triangle is never
 * touched (the bench's host operand for N = 100000 backs only those pages). */
int oracle_gen_fill_tri(char p, char uplo, int n, unsigned long long seed, long long gen_ld, void *out,
                        long long ld_out, int nthreads) {
  const int nt = nthreads_of(nthreads);
  const int lower = uplo == 'l';
#pragma omp parallel for schedule(dynamic, 64) num_threads(nt)
  for (int j = 0; j < n; ++j) {
    const int i0 = lower ? j : 0, i1 = lower ? n : j + 1;
    for (int i = i0; i < i1; ++i) {
      double re, im;
      gen_elem(p, seed, (long long)j * gen_ld + i, &re, &im);
      const long long k = (long long)j * ld_out + i;
      switch (p) {
        case 's': ((float *)out)[k] = (float)re; break;
        case 'd': ((double *)out)[k] = re; break;
        case 'c': ((float *)out)[2 * k] = (float)re; ((float *)out)[2 * k + 1] = (float)im; break;
        default: ((double *)out)[2 * k] = re; ((double *)out)[2 * k + 1] = im; break;
      }
    }
  }
  return 0;
}

int oracle_max_threads(void) { return nthreads_of(0); }
