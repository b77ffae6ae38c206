/* CPU ORACLE — test infrastructure only (tests/, smoke(), bench.py's CPU
 * baseline leg); never linked into the product.
 *
 * C restatement of the reference's CPU evaluation of the stencil programs:
 * frontend/oracle.py evaluate_program (pkg/src/sdfgkit/frontend/oracle.py:
 * 126-156 exec_assign, 205-262 eval_expr) evaluates each slice statement as
 * whole-array numpy ops, left to right, into a temporary, then assigns.
 * Per element that is exactly the scalar expression below in source order,
 * so with -ffp-contract=off this is bitwise identical to the numpy oracle.
 * Points are independent within a statement, so OpenMP over planes/rows does
 * not change any result.
 *
 *   jacobi_2d (pkg/tests/corpus/jacobi_2d.dpy):
 *     B[1:-1,1:-1] = 0.2*(A[c] + A[w] + A[e] + A[s] + A[n]) ; then A from B
 *   heat_3d (programs/heat_3d.dpy):
 *     B = 0.125*(A[i+1]-2A+A[i-1]) + 0.125*(A[j+1]-2A+A[j-1])
 *       + 0.125*(A[k+1]-2A+A[k-1]) + A ; then A from B
 */
#include <stddef.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static void jac_sweep(const double *restrict a, double *restrict b, long n) {
#pragma omp parallel for schedule(static)
  for (long i = 1; i < n - 1; ++i)
    for (long j = 1; j < n - 1; ++j) {
      const double *r = a + i * n;
      double v = r[j] + r[j - 1];
      v = v + r[j + 1];
      v = v + a[(i + 1) * n + j];
      v = v + a[(i - 1) * n + j];
      b[i * n + j] = 0.2 * v;
    }
}

void oracle_jacobi_2d(double *A, double *B, long n, long tsteps, int threads) {
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#endif
  for (long t = 1; t < tsteps; ++t) {
    jac_sweep(A, B, n);
    jac_sweep(B, A, n);
  }
}

static void heat_sweep(const double *restrict a, double *restrict b, long n) {
  const long s0 = n * n, s1 = n;
#pragma omp parallel for schedule(static)
  for (long i = 1; i < n - 1; ++i)
    for (long j = 1; j < n - 1; ++j)
      for (long k = 1; k < n - 1; ++k) {
        const long c = i * s0 + j * s1 + k;
        const double ac = a[c];
        double x = a[c + s0] - 2.0 * ac;
        x = x + a[c - s0];
        double y = a[c + s1] - 2.0 * ac;
        y = y + a[c - s1];
        double z = a[c + 1] - 2.0 * ac;
        z = z + a[c - 1];
        double v = 0.125 * x + 0.125 * y;
        v = v + 0.125 * z;
        b[c] = v + ac;
      }
}

void oracle_heat_3d(double *A, double *B, long n, long tsteps, int threads) {
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#endif
  for (long t = 1; t < tsteps; ++t) {
    heat_sweep(A, B, n);
    heat_sweep(B, A, n);
  }
}

/* one sweep each, for bounded CPU-baseline samples */
void oracle_heat_3d_sweeps(double *A, double *B, long n, long sweeps, int threads) {
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#endif
  for (long s = 0; s < sweeps; ++s) {
    if (s & 1) heat_sweep(B, A, n);
    else heat_sweep(A, B, n);
  }
}
