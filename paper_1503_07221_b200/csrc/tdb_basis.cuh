// Temporal basis on the device (restating temporal_basis.py:105-260 of this
// package, itself pinned to the reference's tables): the smooth cutoff f and its
// first two derivatives, Legendre factors, and the canonical prototypes of the
// first / inner / last time steps with derivatives 0, 1, 2.
#pragma once

#include <cuda_runtime.h>

namespace tdb {

constexpr double kBasisTClamp = 1.0 - 1e-14;                  // temporal_basis.py:47
constexpr double kBasisCErf = 1.1283791670955125738961589031;  // 2 / sqrt(pi)

// f(t) = (1 + erf(2 atanh t)) / 2 on (-1, 1), 0 left, 1 right; f', f''
__device__ __forceinline__ void cutoff012(double t, double& f0, double& f1, double& f2) {
  const double tc = fmin(fmax(t, -kBasisTClamp), kBasisTClamp);
  const double s = atanh(tc);
  const double g = exp(-4.0 * s * s);
  f0 = t >= 1.0 ? 1.0 : (t <= -1.0 ? 0.0 : 0.5 * erf(2.0 * s) + 0.5);
  const double q = 1.0 - tc * tc;
  const bool in = fabs(t) < 1.0 && g > 0.0;
  f1 = in ? kBasisCErf * g / q : 0.0;
  f2 = in ? kBasisCErf * g * (2.0 * tc - 8.0 * s) / (q * q) : 0.0;
}

// P_m, P_m', P_m'' (Bonnet)
__device__ __forceinline__ void legendre012(int m, double x, double& P, double& D1, double& D2) {
  double p0 = 1.0, d0 = 0.0, e0 = 0.0;
  if (m == 0) {
    P = p0, D1 = d0, D2 = e0;
    return;
  }
  double p1 = x, d1 = 1.0, e1 = 0.0;
  for (int k = 2; k <= m; ++k) {
    const double a = (2.0 * k - 1.0) / k, b = (k - 1.0) / k;
    const double p2 = a * x * p1 - b * p0;
    const double d2 = a * (p1 + x * d1) - b * d0;
    const double e2 = a * (2.0 * d1 + x * e1) - b * e0;
    p0 = p1, d0 = d1, e0 = e1;
    p1 = p2, d1 = d2, e1 = e2;
  }
  P = p1, D1 = d1, D2 = e1;
}

// Canonical prototype of order m (kind 0 first, 1 inner, 2 last) at offset u:
// b(u), b'(u), b''(u) (zero outside the support, temporal_basis.py:196-260)
__device__ inline void basis012(int kind, int m, double dt, double u, double& b0, double& b1, double& b2) {
  b0 = b1 = b2 = 0.0;
  if (kind == 1) {
    if (u <= 0.0 || u >= 2.0 * dt) return;
    const double c = 2.0 / dt;
    double r0, r1, r2, f0, f1, f2;
    if (u <= dt) {
      cutoff012(c * u - 1.0, f0, f1, f2);
      r0 = f0, r1 = f1 * c, r2 = f2 * c * c;
    } else {
      cutoff012(c * (u - dt) - 1.0, f0, f1, f2);
      r0 = 1.0 - f0, r1 = -(f1 * c), r2 = -(f2 * c * c);
    }
    double P, D1, D2;
    legendre012(m, u / dt - 1.0, P, D1, D2);
    b0 = r0 * P;
    b1 = r1 * P + r0 * D1 / dt;
    b2 = r2 * P + 2.0 * r1 * D1 / dt + r0 * D2 / (dt * dt);
    return;
  }
  const double c = 2.0 / dt, x = c * u - 1.0;
  double P, D1, D2, f0, f1, f2;
  legendre012(m, x, P, D1, D2);
  cutoff012(x, f0, f1, f2);
  if (kind == 2) {
    if (u <= 0.0 || u > dt) return;
    b0 = f0 * P;
    b1 = c * (f1 * P + f0 * D1);
    b2 = c * c * (f2 * P + 2.0 * f1 * D1 + f0 * D2);
    return;
  }
  if (u <= 0.0 || u >= dt) return;
  const double g0 = 1.0 - f0, g1 = -c * f1, g2 = -c * c * f2;
  const double q0 = (u / dt) * (u / dt), q1 = 2.0 * u / (dt * dt), q2 = 2.0 / (dt * dt);
  b0 = 8.0 * g0 * q0 * P;
  b1 = 8.0 * (g1 * q0 * P + g0 * q1 * P + g0 * q0 * D1 * c);
  b2 = 8.0 * (g2 * q0 * P + g0 * q2 * P + g0 * q0 * D2 * c * c + 2.0 * g1 * q1 * P + 2.0 * g1 * q0 * D1 * c +
              2.0 * g0 * q1 * D1 * c);
}

}  // namespace tdb
