/*
 * ORACLE / TEST INFRASTRUCTURE ONLY -- never linked into the product path.
 *
 * Plain-C restatement of the reference's cyclic complex Jacobi sweep
 * (reference pkg/src/chfsi/_jacobi.py:14-80, `sweep_loop`, numba-JIT there).
 * Same sweep order, pivot-skip threshold and rotation formulas, so on the
 * same input it reproduces the reference's eigenvalues/eigenvectors.
 *
 * H and V are row-major n x n complex128 (interleaved re, im), as the
 * reference passes a C-order copy (linalg.py:309) and np.eye (C-order).
 * Compiled with -ffp-contract=off so no FMA contraction changes rounding.
 */
#include <math.h>

#define RE(a, i, j, n) (a)[2 * ((i) * (n) + (j))]
#define IM(a, i, j, n) (a)[2 * ((i) * (n) + (j)) + 1]

static double off_norm(int n, const double* h) {
  double off2 = 0.0;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      if (i != j) {
        const double xr = RE(h, i, j, n), xi = IM(h, i, j, n);
        off2 += xr * xr + xi * xi;
      }
  return sqrt(off2);
}

/* returns 1 when converged; *sweeps_done = sweeps performed (_jacobi.py:21-80) */
int oracle_jacobi_sweeps(int n, double* h, double* v, int vrows, int max_sweeps, double off_tol,
                         int* sweeps_done) {
  int sweeps = 0;
  while (sweeps < max_sweeps) {
    if (off_norm(n, h) <= off_tol) {
      *sweeps_done = sweeps;
      return 1;
    }
    const double skip = off_tol / (2.0 * n);
    for (int p = 0; p < n - 1; ++p) {
      for (int q = p + 1; q < n; ++q) {
        const double ar = RE(h, p, q, n), ai = IM(h, p, q, n);
        const double mag = hypot(ar, ai);
        if (mag <= skip) continue;
        const double app = RE(h, p, p, n), aqq = RE(h, q, q, n);
        const double tau = (aqq - app) / (2.0 * mag);
        double t;
        if (tau >= 0.0)
          t = 1.0 / (tau + sqrt(1.0 + tau * tau));
        else
          t = -1.0 / (-tau + sqrt(1.0 + tau * tau));
        const double c = 1.0 / sqrt(1.0 + t * t);
        const double s = t * c;
        const double ur = ar / mag, ui = ai / mag;   /* u = apq / |apq| */
        const double sur = s * ur, sui = s * ui;     /* su = s u */
        const double scr = s * ur, sci = -(s * ui);  /* suc = s conj(u) */
        for (int j = 0; j < n; ++j) { /* rows p, q */
          const double hpr = RE(h, p, j, n), hpi = IM(h, p, j, n);
          const double hqr = RE(h, q, j, n), hqi = IM(h, q, j, n);
          RE(h, p, j, n) = c * hpr - (sur * hqr - sui * hqi);
          IM(h, p, j, n) = c * hpi - (sur * hqi + sui * hqr);
          RE(h, q, j, n) = (scr * hpr - sci * hpi) + c * hqr;
          IM(h, q, j, n) = (scr * hpi + sci * hpr) + c * hqi;
        }
        for (int i = 0; i < n; ++i) { /* columns p, q */
          const double hpr = RE(h, i, p, n), hpi = IM(h, i, p, n);
          const double hqr = RE(h, i, q, n), hqi = IM(h, i, q, n);
          RE(h, i, p, n) = c * hpr - (scr * hqr - sci * hqi);
          IM(h, i, p, n) = c * hpi - (scr * hqi + sci * hqr);
          RE(h, i, q, n) = (sur * hpr - sui * hpi) + c * hqr;
          IM(h, i, q, n) = (sur * hpi + sui * hpr) + c * hqi;
        }
        const double dd = t * mag;
        RE(h, p, p, n) = app - dd; IM(h, p, p, n) = 0.0;
        RE(h, q, q, n) = aqq + dd; IM(h, q, q, n) = 0.0;
        RE(h, p, q, n) = 0.0; IM(h, p, q, n) = 0.0;
        RE(h, q, p, n) = 0.0; IM(h, q, p, n) = 0.0;
        for (int i = 0; i < vrows; ++i) {
          const double vpr = RE(v, i, p, n), vpi = IM(v, i, p, n);
          const double vqr = RE(v, i, q, n), vqi = IM(v, i, q, n);
          RE(v, i, p, n) = c * vpr - (scr * vqr - sci * vqi);
          IM(v, i, p, n) = c * vpi - (scr * vqi + sci * vqr);
          RE(v, i, q, n) = (sur * vpr - sui * vpi) + c * vqr;
          IM(v, i, q, n) = (sur * vpi + sui * vpr) + c * vqi;
        }
      }
    }
    ++sweeps;
  }
  *sweeps_done = sweeps;
  return off_norm(n, h) <= off_tol;
}
