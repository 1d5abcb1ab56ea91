/*
 * ORACLE (test infrastructure only - never the product path).
 *
 * Plain-C, single-threaded restatement of the reference hot kernel
 * tdbem._kernels._core.pair_block_contributions
 * (/root/reference/pkg/src/tdbem/_kernels/_core.pyx:47-159, helpers :19-44),
 * point loop, table evaluation and accumulation order kept as in the Cython
 * source so the result agrees with the compiled reference to rounding.
 * Built by oracle/Makefile into oracle/liboracle.so; called from tests/ and
 * from bench.py's cpu_baseline leg only.  Pinned against the reference's own
 * outputs in tests/golden/pair_contrib.npz (tests/test_oracle_golden.py).
 *
 * Signature = tdb_pair_block_contributions (include/tdb.h).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/tdb.h"

static const double INV4PI = 1.0 / (4.0 * 3.14159265358979323846264338327950288);

/* _core.pyx:53-60 */
static double clenshaw(const double* c, int deg, double x) {
  double b1 = 0.0, b2 = 0.0, tmp;
  for (int k = deg; k > 0; --k) {
    tmp = 2.0 * x * b1 - b2 + c[k];
    b2 = b1;
    b1 = tmp;
  }
  return x * b1 - b2 + c[0];
}

/* _core.pyx:63-78 */
static double eval_table(const TdbPsiPack* pk, int t, double a) {
  const double lo = pk->lo[t], width = pk->width[t];
  const int64_t nsub = pk->nsub[t];
  const double hi = lo + nsub * width;
  if (a < lo || a > hi) return 0.0;
  int64_t idx = (int64_t)((a - lo) / width);
  if (idx > nsub - 1) idx = nsub - 1;
  double x = 2.0 * (a - lo - idx * width) / width - 1.0;
  if (x < -1.0) x = -1.0;
  else if (x > 1.0) x = 1.0;
  return clenshaw(pk->coeffs + ((int64_t)t * pk->max_nsub + idx) * (pk->deg + 1), pk->deg, x);
}

int oracle_pair_block_contributions(const double* cx, const double* cy, const double* a2x,
                                    const double* a2y, const double* ndot, const double* curly,
                                    const double* curlx, const double* xhat, const double* yhat,
                                    const double* wq, int64_t npair, int64_t nq,
                                    const TdbPsiPack* pk, double* out) {
  const int np1 = pk->p + 1;
  const int nt = 2 * np1 * np1;
  const double delta = pk->delta;
  double amin = 1e300, amax = -1e300;
  /* union of the table supports in offset space (_core.pyx:122-135) */
  for (int t = 0; t < nt; ++t) {
    if (!pk->active[t]) continue;
    const double thi = pk->lo[t] + pk->nsub[t] * pk->width[t];
    if (pk->fold[t]) {
      if (-thi < amin) amin = -thi;
    } else if (pk->lo[t] < amin) {
      amin = pk->lo[t];
    }
    if (thi > amax) amax = thi;
  }
  memset(out, 0, sizeof(double) * (size_t)npair * np1 * np1 * 9);
  double* shx = (double*)malloc(sizeof(double) * 3 * (size_t)(nq > 0 ? nq : 1));
  double* shy = (double*)malloc(sizeof(double) * 3 * (size_t)(nq > 0 ? nq : 1));
  if (!shx || !shy) {
    free(shx);
    free(shy);
    return TDB_E_NOMEM;
  }
  for (int64_t q = 0; q < nq; ++q) {
    shx[3 * q] = 1.0 - xhat[2 * q];
    shx[3 * q + 1] = xhat[2 * q] - xhat[2 * q + 1];
    shx[3 * q + 2] = xhat[2 * q + 1];
    shy[3 * q] = 1.0 - yhat[2 * q];
    shy[3 * q + 1] = yhat[2 * q] - yhat[2 * q + 1];
    shy[3 * q + 2] = yhat[2 * q + 1];
  }
  for (int64_t p = 0; p < npair; ++p) {
    const double* X = cx + 9 * p;
    const double* Y = cy + 9 * p;
    const double nd = ndot[p];
    double cdot[3][3];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b)
        cdot[a][b] = curly[9 * p + 3 * a] * curlx[9 * p + 3 * b] +
                     curly[9 * p + 3 * a + 1] * curlx[9 * p + 3 * b + 1] +
                     curly[9 * p + 3 * a + 2] * curlx[9 * p + 3 * b + 2];
    double* o = out + (size_t)p * np1 * np1 * 9;
    for (int64_t q = 0; q < nq; ++q) {
      const double x0 = xhat[2 * q], x1 = xhat[2 * q + 1];
      const double y0 = yhat[2 * q], y1 = yhat[2 * q + 1];
      const double X0 = X[0] + x0 * (X[3] - X[0]) + x1 * (X[6] - X[3]);
      const double X1 = X[1] + x0 * (X[4] - X[1]) + x1 * (X[7] - X[4]);
      const double X2 = X[2] + x0 * (X[5] - X[2]) + x1 * (X[8] - X[5]);
      const double Y0 = Y[0] + y0 * (Y[3] - Y[0]) + y1 * (Y[6] - Y[3]);
      const double Y1 = Y[1] + y0 * (Y[4] - Y[1]) + y1 * (Y[7] - Y[4]);
      const double Y2 = Y[2] + y0 * (Y[5] - Y[2]) + y1 * (Y[8] - Y[5]);
      const double r = sqrt((X0 - Y0) * (X0 - Y0) + (X1 - Y1) * (X1 - Y1) + (X2 - Y2) * (X2 - Y2));
      const double av = r + delta;
      if (av < amin || av > amax) continue;
      const double common = INV4PI * a2x[p] * a2y[p] * wq[q] / r;
      const double aa = fabs(av);
      for (int m2 = 0; m2 < np1; ++m2)
        for (int m1 = 0; m1 < np1; ++m1) {
          const int t = (m2 * np1 + m1) * 2;
          double psi = 0.0, psit = 0.0;
          for (int tt = t; tt < t + 2; ++tt) {
            double cp;
            if (!pk->active[tt]) continue;
            if (pk->fold[tt]) {
              cp = eval_table(pk, tt, aa);
              cp = av >= 0.0 ? pk->sp[tt] * cp : pk->sn[tt] * cp;
            } else {
              cp = eval_table(pk, tt, av);
            }
            if (tt == t) psi = cp;
            else psit = cp;
          }
          if (psi == 0.0 && psit == 0.0) continue;
          psi = common * psi * nd;
          psit = common * psit;
          double* ob = o + (m2 * np1 + m1) * 9;
          for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b)
              ob[3 * a + b] += psi * shy[3 * q + a] * shx[3 * q + b] + psit * cdot[a][b];
        }
    }
  }
  free(shx);
  free(shy);
  return TDB_OK;
}
