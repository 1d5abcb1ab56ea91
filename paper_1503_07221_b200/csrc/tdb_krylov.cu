// Device-side pieces of the restarted / flexible GMRES cycle (reference
// solvers.py:172-223 _gmres_cycle_raw) that otherwise force a host round trip
// per Arnoldi step: the Hessenberg column update with Givens rotations, the
// convergence / breakdown decisions, and the final triangular solve + update.
//
// With these, a fixed-iteration inner solve of the recursive block
// preconditioner (solvers.py:276-320) runs without host synchronisation and the
// whole preconditioner application is captured once in a CUDA graph
// (paper_1503_07221_b200/solvers.py).  Early exit is emulated on the device:
// after `done` is set, every later step's Givens update is a no-op and the
// final update uses only the k_done columns the reference would have used.
//
// Cycle state (doubles): see TDB_KS_* in include/tdb.h.
#include <cuda_runtime.h>

#include <cmath>

#include "tdb_common.cuh"
#include "tdb_internal.h"

using namespace tdb;

namespace {

__global__ void k_krylov_init(double* st, const double* beta, double tol_rel, double* g) {
  const double b = *beta;
  const double tol_abs = tol_rel * b;  // x0 = 0: ||b|| = ||r0|| = beta
  st[TDB_KS_DONE] = (b <= tol_abs) ? 1.0 : 0.0;
  st[TDB_KS_KDONE] = 0.0;
  st[TDB_KS_BREAKDOWN] = 0.0;
  st[TDB_KS_TOL_ABS] = tol_abs;
  st[TDB_KS_BETA] = b;
  st[TDB_KS_CONVERGED] = (b <= tol_abs) ? 1.0 : 0.0;
  g[0] = b;
}

// Step k of the cycle: hcol[0..k+1] = (h_0k .. h_kk, ||w||).  Mirrors the
// reference's Givens bookkeeping line by line (solvers.py:196-215).
__global__ void k_krylov_givens(double* st, int k, const double* hcol, double* H, int ldh, double* cs,
                                double* sn, double* g) {
  if (st[TDB_KS_DONE] != 0.0) return;
  double* col = H + k;  // H[i][k] = H[i * ldh + k]
  for (int i = 0; i <= k + 1; ++i) col[i * ldh] = hcol[i];
  const double hk = hcol[k + 1];
  for (int j = 0; j < k; ++j) {
    const double a = col[j * ldh], b = col[(j + 1) * ldh];
    const double t = cs[j] * a + sn[j] * b;
    col[(j + 1) * ldh] = -sn[j] * a + cs[j] * b;
    col[j * ldh] = t;
  }
  const double hkk = col[k * ldh], hk1 = col[(k + 1) * ldh];
  const double denom = hypot(hkk, hk1);
  cs[k] = denom > 0.0 ? hkk / denom : 1.0;
  sn[k] = denom > 0.0 ? hk1 / denom : 0.0;
  col[k * ldh] = denom;
  g[k + 1] = -sn[k] * g[k];
  g[k] = cs[k] * g[k];
  col[(k + 1) * ldh] = 0.0;
  st[TDB_KS_KDONE] = (double)(k + 1);
  if (fabs(g[k + 1]) <= st[TDB_KS_TOL_ABS]) {
    st[TDB_KS_DONE] = 1.0;
    st[TDB_KS_CONVERGED] = 1.0;
  } else if (hk <= 1e-14 * st[TDB_KS_BETA]) {
    st[TDB_KS_DONE] = 1.0;
    st[TDB_KS_BREAKDOWN] = 1.0;
  }
}

// x = x0 + Z[:kd]^T y with H[:kd, :kd] y = g[:kd] (back substitution, every CTA
// redundantly: kd <= restart, a few hundred flops).
__global__ void k_krylov_update(double* x, const double* x0, const double* Z, long long ldz, long long n,
                                const double* st, const double* H, int ldh, const double* g, int m) {
  extern __shared__ double sy[];
  const int kd = (int)st[TDB_KS_KDONE];
  if (threadIdx.x == 0) {
    for (int i = kd - 1; i >= 0; --i) {
      double s = g[i];
      for (int j = i + 1; j < kd; ++j) s -= H[i * ldh + j] * sy[j];
      sy[i] = s / H[i * ldh + i];
    }
  }
  __syncthreads();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double v = x0 ? x0[i] : 0.0;
    for (int j = 0; j < kd; ++j) v = fma(sy[j], Z[j * ldz + i], v);
    x[i] = v;
  }
}

// Fold a cycle's breakdown-without-convergence into a sticky error word.
__global__ void k_krylov_flag(const double* st, double* err) {
  if (st[TDB_KS_BREAKDOWN] != 0.0 && st[TDB_KS_CONVERGED] == 0.0) *err = 1.0;
}

}  // namespace

extern "C" {

int tdb_krylov_init(double* state, const double* beta, double tol_rel, double* g, void* stream) {
  TDB_REQUIRE(state && beta && g, "krylov_init: NULL argument");
  k_krylov_init<<<1, 1, 0, (cudaStream_t)stream>>>(state, beta, tol_rel, g);
  TDB_CUDA_CHECK(cudaGetLastError());
  return TDB_OK;
}

int tdb_krylov_givens(double* state, int32_t k, const double* hcol, double* H, int32_t ldh, double* cs,
                      double* sn, double* g, void* stream) {
  TDB_REQUIRE(state && hcol && H && cs && sn && g && k >= 0 && ldh > k, "krylov_givens: bad argument");
  k_krylov_givens<<<1, 1, 0, (cudaStream_t)stream>>>(state, k, hcol, H, ldh, cs, sn, g);
  TDB_CUDA_CHECK(cudaGetLastError());
  return TDB_OK;
}

int tdb_krylov_update(double* x, const double* x0, const double* Z, int64_t ldz, int64_t n, const double* state,
                      const double* H, int32_t ldh, const double* g, int32_t m, void* stream) {
  TDB_REQUIRE(x && Z && state && H && g && n >= 0 && m >= 1 && m <= 4096, "krylov_update: bad argument");
  const int threads = 256;
  const long long blocks = std::min<long long>((n + threads - 1) / threads, 148LL * 8);
  if (blocks <= 0) return TDB_OK;
  k_krylov_update<<<(int)blocks, threads, (size_t)m * sizeof(double), (cudaStream_t)stream>>>(
      x, x0, Z, ldz, n, state, H, ldh, g, m);
  TDB_CUDA_CHECK(cudaGetLastError());
  return TDB_OK;
}

int tdb_krylov_flag(const double* state, double* err, void* stream) {
  TDB_REQUIRE(state && err, "krylov_flag: NULL argument");
  k_krylov_flag<<<1, 1, 0, (cudaStream_t)stream>>>(state, err);
  TDB_CUDA_CHECK(cudaGetLastError());
  return TDB_OK;
}

}  // extern "C"
