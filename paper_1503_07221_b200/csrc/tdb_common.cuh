// Shared device helpers: error plumbing, Clenshaw evaluation of the packed
// piecewise-Chebyshev psi/psi~ tables, warp reductions.  sm_100a, FP64 SIMT.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "../../include/tdb.h"

namespace tdb {

constexpr double kInv4Pi = 1.0 / (4.0 * 3.14159265358979323846264338327950288);
constexpr int kWarp = 32;

void set_error(const std::string& msg);

#define TDB_CUDA_CHECK(expr)                                                  \
  do {                                                                        \
    cudaError_t _e = (expr);                                                  \
    if (_e != cudaSuccess) {                                                  \
      ::tdb::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));   \
      return _e == cudaErrorMemoryAllocation ? TDB_E_NOMEM : TDB_E_CUDA;      \
    }                                                                         \
  } while (0)

#define TDB_REQUIRE(cond, msg)       \
  do {                               \
    if (!(cond)) {                   \
      ::tdb::set_error(msg);         \
      return TDB_E_INVALID;          \
    }                                \
  } while (0)

// Clenshaw recurrence sum_k c_k T_k(x), degree DEG, coefficients contiguous.
// Two independent tables are evaluated together for ILP (psi and psi~).
template <int DEG>
__device__ __forceinline__ void clenshaw2(const double* __restrict__ c0,
                                          const double* __restrict__ c1,
                                          double x0, double x1, double& v0,
                                          double& v1) {
  const double y0 = 2.0 * x0, y1 = 2.0 * x1;
  double b1a = c0[DEG], b2a = 0.0;
  double b1b = c1[DEG], b2b = 0.0;
#pragma unroll
  for (int k = DEG - 1; k >= 1; --k) {
    double ta = fma(y0, b1a, c0[k] - b2a);
    double tb = fma(y1, b1b, c1[k] - b2b);
    b2a = b1a;
    b1a = ta;
    b2b = b1b;
    b1b = tb;
  }
  v0 = fma(x0, b1a, c0[0] - b2a);
  v1 = fma(x1, b1b, c1[0] - b2b);
}

__device__ __forceinline__ double clenshaw_dyn(const double* __restrict__ c, int deg, double x) {
  const double y = 2.0 * x;
  double b1 = 0.0, b2 = 0.0;
  for (int k = deg; k >= 1; --k) {
    double t = fma(y, b1, c[k] - b2);
    b2 = b1;
    b1 = t;
  }
  return fma(x, b1, c[0] - b2);
}

// Subinterval index and local coordinate of offset a in table [lo, lo+nsub*w]
// (_core.pyx:63-78): idx = min(floor((a-lo)/w), nsub-1), x clamped to [-1, 1].
__device__ __forceinline__ int cheb_locate(double a, double lo, double w, double inv_w,
                                           int nsub, double& x) {
  const double t = (a - lo) * inv_w;
  int idx = (int)t;
  idx = idx > nsub - 1 ? nsub - 1 : idx;
  const double xl = 2.0 * (a - lo - (double)idx * w) * inv_w - 1.0;
  x = fmin(fmax(xl, -1.0), 1.0);  // xl is never NaN here: same result as the compares
  return idx;
}

// Full warp all-reduce (xor butterfly; identical result in every lane, fixed order).
__device__ __forceinline__ double warp_allsum(double v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace tdb
