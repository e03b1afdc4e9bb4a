/*
 * rbffd_oracle.c -- CPU restatement of the reference hot path.  TEST
 * INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py, and only as the checker or
 * the CPU baseline, never as part of the product path.
 *
 * Restates, from /root/reference/pkg/src/rbffd/solver.py:
 *   orc_step_kernel    <- _step_kernel        :294-311  (numba @njit(parallel=True))
 *   orc_run_time_loop  <- run_time_loop loop  :190-225  (flags, residual, swap /
 *                                                        copy-back, steady break,
 *                                                        timeout)
 * The numba kernel compiles to scalar fmul/fadd with no contraction
 * (SURVEY.md A.3); this file is built with -ffp-contract=off and no fast-math
 * so gcc emits the same separately rounded operations in the same order.
 * Parallelism mirrors numba's prange over row chunks (OpenMP), which cannot
 * change any bit because each row is computed by exactly one thread.
 *
 * Parity of this oracle is PINNED: tests/test_oracle.py checks it bit-for-bit
 * against the fixtures tests/golden/make_golden.py recorded from the
 * unmodified reference (numba 0.65.0).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>
#include <stdlib.h>
#include <time.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OK 0
#define ORC_INSTABILITY 4
#define ORC_TIMEOUT 5

static int64_t chunk_count(int64_t n_rows, int64_t chunk) {  /* solver.py:290-291 */
  int64_t c = (n_rows + chunk - 1) / chunk;
  return c > 1 ? c : 1;
}

/* solver.py:294-311 */
void orc_step_kernel(const double* u1, double* u2, const int64_t* interior, const int64_t* rows,
                     const double* weights, const double* f_int, double dt, int64_t n_rows,
                     int32_t width, int64_t chunk, uint8_t* flags, int32_t nthreads) {
  const int64_t n_chunks = (n_rows + chunk - 1) / chunk;
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
#endif
  for (int64_t c = 0; c < n_chunks; ++c) {
    const int64_t lo = c * chunk;
    const int64_t hi = lo + chunk < n_rows ? lo + chunk : n_rows;
    int bad = 0;
    for (int64_t k = lo; k < hi; ++k) {
      double acc = 0.0;
      const double* w = weights + k * width;
      const int64_t* r = rows + k * width;
      for (int32_t j = 0; j < width; ++j) acc += w[j] * u1[r[j]];
      const double value = u1[interior[k]] + dt * (f_int[k] + acc);
      u2[interior[k]] = value;
      if (!isfinite(value)) bad = 1;
    }
    flags[c] = bad ? 1 : 0;
  }
  (void)nthreads;
}

/* float(np.max(np.abs(a - b))) with numpy's NaN propagation */
static double max_abs_diff(const double* a, const double* b, int64_t n, int32_t nthreads) {
  double m = 0.0;
  int nan_seen = 0;
#ifdef _OPENMP
#pragma omp parallel for reduction(max : m) reduction(| : nan_seen) num_threads(nthreads > 0 ? nthreads : 1)
#endif
  for (int64_t i = 0; i < n; ++i) {
    const double d = fabs(a[i] - b[i]);
    if (d != d) nan_seen |= 1;
    else if (d > m) m = d;
  }
  (void)nthreads;
  return nan_seen ? NAN : m;
}

static double max_abs(const double* a, int64_t n) {
  double m = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double d = fabs(a[i]);
    if (d != d) return NAN;
    if (d > m) m = d;
  }
  return m;
}

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/*
 * solver.py:186-225 with the host prep (apply_dirichlet, forcing, auto dt)
 * done by the caller: u0 = the initial field, f_int = forcing at interior.
 * On return `field` holds u1 after the loop (solver.py:227), or the failing
 * step's u2 on ORC_INSTABILITY (then *max_abs_out = max|u2|, solver.py:201).
 */
int orc_run_time_loop(int64_t N, int64_t n_rows, int32_t width, const int64_t* interior,
                      const int64_t* rows, const double* weights, const double* f_int,
                      const double* u0, double dt, int64_t steps, int32_t steady, double tol,
                      int64_t max_steps, int32_t copy_back, int64_t chunk, int32_t nthreads,
                      double* field, int64_t* steps_done_out, double* residual_out,
                      int32_t* has_residual_out, int64_t* bad_step_out, double* max_abs_out,
                      double* seconds_out) {
  double* u1 = (double*)malloc(sizeof(double) * (size_t)N);
  double* u2 = (double*)malloc(sizeof(double) * (size_t)N);
  uint8_t* flags = (uint8_t*)calloc((size_t)chunk_count(n_rows, chunk), 1);
  if (!u1 || !u2 || !flags) {
    free(u1); free(u2); free(flags);
    return -1;
  }
  memcpy(u1, u0, sizeof(double) * (size_t)N);
  memcpy(u2, u0, sizeof(double) * (size_t)N);
  const int64_t limit = steady ? max_steps : steps;
  const int64_t nc = chunk_count(n_rows, chunk);
  int has_res = 0;
  double residual = 0.0;
  int64_t steps_done = 0;
  int rc = ORC_OK;
  const double t0 = now_s();
  for (int64_t step = 0; step < limit; ++step) {
    orc_step_kernel(u1, u2, interior, rows, weights, f_int, dt, n_rows, width, chunk, flags, nthreads);
    int any = 0;
    for (int64_t c = 0; c < nc; ++c) any |= flags[c];
    if (any) {
      memcpy(field, u2, sizeof(double) * (size_t)N);
      *max_abs_out = max_abs(u2, N);
      *bad_step_out = step;
      rc = ORC_INSTABILITY;
      break;
    }
    steps_done = step + 1;
    if (steady || steps_done == limit) {
      residual = max_abs_diff(u2, u1, N, nthreads) / dt;
      has_res = 1;
    }
    if (copy_back) {
      memcpy(u1, u2, sizeof(double) * (size_t)N);
    } else {
      double* t = u1; u1 = u2; u2 = t;
    }
    if (steady && residual <= tol) break;
  }
  *seconds_out = now_s() - t0;
  if (rc == ORC_OK) {
    memcpy(field, u1, sizeof(double) * (size_t)N);
    *bad_step_out = -1;
    if (steady && steps_done == max_steps && (!has_res || residual > tol)) rc = ORC_TIMEOUT;
  }
  *steps_done_out = steps_done;
  *residual_out = residual;
  *has_residual_out = has_res;
  free(u1); free(u2); free(flags);
  return rc;
}

int orc_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
