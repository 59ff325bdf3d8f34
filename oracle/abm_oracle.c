/*
 * abm_oracle.c — CPU restatement of the reference ABM solver in C.
 * TEST INFRASTRUCTURE ONLY: used by tests/ as a fast checker at sizes the
 * NumPy oracle is too slow for, and by bench.py's `--impl reference` /
 * cpu_baseline legs as the timed CPU implementation ("port") with all host
 * threads.  The product path never links or calls it.
 *
 * Follows /root/reference/pkg/src/fodeabm:
 *   solve loop      serial.py:150-170 (predictor 153-157, corrector 160-168)
 *   chunked sums    parallel/reduction.py:98-136: the history range of each
 *                   step is split into contiguous per-thread spans whose
 *                   partials are folded in ascending span order (the
 *                   reduction engine's deterministic combine, :296-325)
 *   rhs             systems.py:64-73,101-123 and the BASELINE systems of
 *                   paper_1611_08678_b200/systems.py, same operator order
 *                   (compiled with -ffp-contract=off: no FMA contraction)
 * Weights are inputs (the precompute_weights seam, serial.py:130).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { SYS_CONSTANT = 0, SYS_POWER_LAW, SYS_LINEAR, SYS_HINDMARSH_ROSE, SYS_LORENZ, SYS_CHEN, SYS_ROSSLER,
       SYS_FINANCIAL };

static void rhs_eval(int sys, const double* p, int d, double t, const double* y, double* f) {
  switch (sys) {
    case SYS_CONSTANT:
      for (int i = 0; i < d; ++i) f[i] = p[i];
      break;
    case SYS_POWER_LAW:
      f[0] = t > 0.0 ? p[0] * pow(t, p[1]) : 0.0;
      break;
    case SYS_LINEAR:
      for (int i = 0; i < d; ++i) f[i] = p[0] * y[i];
      break;
    case SYS_HINDMARSH_ROSE: {
      const double x = y[0], yy = y[1], z = y[2], x2 = x * x;
      f[0] = yy - p[0] * x2 * x + p[1] * x2 - z + p[7];
      f[1] = p[2] - p[3] * x2 - yy;
      f[2] = p[4] * (p[5] * (x - p[6]) - z);
    } break;
    case SYS_LORENZ: {
      const double x = y[0], yy = y[1], z = y[2];
      f[0] = p[0] * (yy - x);
      f[1] = x * (p[1] - z) - yy;
      f[2] = x * yy - p[2] * z;
    } break;
    case SYS_CHEN: {
      const double x = y[0], yy = y[1], z = y[2];
      f[0] = p[0] * (yy - x);
      f[1] = (p[2] - p[0]) * x - x * z + p[2] * yy;
      f[2] = x * yy - p[1] * z;
    } break;
    case SYS_ROSSLER: {
      const double x = y[0], yy = y[1], z = y[2];
      f[0] = -yy - z;
      f[1] = x + p[0] * yy;
      f[2] = p[1] + z * (x - p[2]);
    } break;
    case SYS_FINANCIAL: {
      const double x = y[0], yy = y[1], z = y[2];
      f[0] = z + (yy - p[0]) * x;
      f[1] = 1.0 - p[1] * yy - x * x;
      f[2] = -x - p[2] * z;
    } break;
  }
}

static int all_finite(const double* v, int d) {
  for (int i = 0; i < d; ++i)
    if (!isfinite(v[i])) return 0;
  return 1;
}

/* partial sums over k in [k0, k1): P += rb[N-n+k] f_k ; C += ra[N-n+k] f_k (k>=1) */
static void span_sums(int d, const double* fT, int64_t stride, const double* rb, const double* ra, int64_t N,
                      int64_t n, int64_t k0, int64_t k1, double* P, double* C) {
  for (int c = 0; c < d; ++c) {
    const double* fr = fT + c * stride;
    double p8[8] = {0}, c8[8] = {0};
    const double* wb = rb + (N - n);
    const double* wa = ra + (N - n);
    int64_t k = k0;
    int64_t kc = k0 < 1 ? 1 : k0; /* corrector starts at k = 1 */
    /* predictor-only head k = 0 */
    if (k < kc && k < k1) {
      p8[0] += wb[k] * fr[k];
      k = kc;
    }
    for (; k + 8 <= k1; k += 8)
      for (int j = 0; j < 8; ++j) {
        p8[j] += wb[k + j] * fr[k + j];
        c8[j] += wa[k + j] * fr[k + j];
      }
    for (; k < k1; ++k) {
      p8[0] += wb[k] * fr[k];
      c8[0] += wa[k] * fr[k];
    }
    P[c] = ((p8[0] + p8[1]) + (p8[2] + p8[3])) + ((p8[4] + p8[5]) + (p8[6] + p8[7]));
    C[c] = ((c8[0] + c8[1]) + (c8[2] + c8[3])) + ((c8[4] + c8[5]) + (c8[6] + c8[7]));
  }
}

/*
 * Returns 0 on success, 1 on a non-finite rhs (err_step / err_t set: the
 * loop index n and t=(n+1)h, serial.py:157-168; step 0 / t 0 for f(0,y0)).
 * Y, Fc: (N+1) x d row-major outputs.  nthreads <= 0 -> all OpenMP threads.
 */
int abm_oracle_solve(int sys, const double* params, int d, double alpha, const double* y0, double h,
                     int64_t N, double ha, double ig, const double* b, const double* a, const double* c,
                     double* Y, double* Fc, int nthreads, int64_t* err_step, double* err_t) {
  (void)alpha;
  const int64_t stride = N + 1;
  double* fT = (double*)malloc(sizeof(double) * d * stride);
  double* rb = (double*)malloc(sizeof(double) * stride);
  double* ra = (double*)malloc(sizeof(double) * stride);
  for (int64_t i = 0; i <= N; ++i) {
    rb[N - i] = b[i];
    ra[N - i] = a[i];
  }
  int T = 1;
#ifdef _OPENMP
  T = nthreads > 0 ? nthreads : omp_get_max_threads();
#endif
  double* part = (double*)calloc((size_t)T * 2 * 8, sizeof(double));
  double f0[8], buf[8], yp[8], y1[8];
  int status = 0;
  for (int i = 0; i < d; ++i) Y[i] = y0[i];
  rhs_eval(sys, params, d, 0.0, y0, f0);
  if (!all_finite(f0, d)) {
    *err_step = 0;
    *err_t = 0.0;
    free(fT); free(rb); free(ra); free(part);
    return 1;
  }
  for (int i = 0; i < d; ++i) fT[i * stride] = f0[i];

#pragma omp parallel num_threads(T) shared(status)
  {
    int tid = 0;
#ifdef _OPENMP
    tid = omp_get_thread_num();
#endif
    for (int64_t n = 0; n < N; ++n) {
      /* contiguous spans of [0, n] per thread, folded in ascending order */
      const int64_t len = n + 1;
      const int64_t q = len / T, r = len % T;
      const int64_t k0 = tid * q + (tid < r ? tid : r);
      const int64_t k1 = k0 + q + (tid < r ? 1 : 0);
      double* mine = part + (size_t)tid * 16;
      if (k1 > k0)
        span_sums(d, fT, stride, rb, ra, N, n, k0, k1, mine, mine + 8);
      else
        memset(mine, 0, sizeof(double) * 16);
#pragma omp barrier
#pragma omp single
      {
        if (!status) {
          const double t1 = (double)(n + 1) * h;
          double P[8], C[8];
          for (int cc = 0; cc < d; ++cc) {
            P[cc] = part[cc];
            C[cc] = part[8 + cc];
          }
          for (int t = 1; t < T; ++t)
            for (int cc = 0; cc < d; ++cc) {
              P[cc] += part[t * 16 + cc];
              C[cc] += part[t * 16 + 8 + cc];
            }
          for (int cc = 0; cc < d; ++cc) yp[cc] = P[cc] * ha + y0[cc];
          rhs_eval(sys, params, d, t1, yp, buf);
          if (!all_finite(buf, d)) {
            status = 1;
            *err_step = n;
            *err_t = t1;
          } else {
            for (int cc = 0; cc < d; ++cc) {
              double v = c[n] * f0[cc];
              if (n >= 1) v += C[cc];
              v += ig * buf[cc];
              y1[cc] = v * ha + y0[cc];
            }
            rhs_eval(sys, params, d, t1, y1, buf);
            if (!all_finite(buf, d)) {
              status = 1;
              *err_step = n;
              *err_t = t1;
            } else {
              for (int cc = 0; cc < d; ++cc) {
                Y[(n + 1) * d + cc] = y1[cc];
                fT[cc * stride + n + 1] = buf[cc];
              }
            }
          }
        }
      } /* implicit barrier */
      if (status) break;
    }
  }
  if (!status)
    for (int64_t i = 0; i <= N; ++i)
      for (int cc = 0; cc < d; ++cc) Fc[i * d + cc] = fT[cc * stride + i];
  free(fT);
  free(rb);
  free(ra);
  free(part);
  return status;
}

int abm_oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
