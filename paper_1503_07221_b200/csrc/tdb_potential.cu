// Retarded double-layer potential at off-boundary points.
//
// Replaces tdbem.potential.eval_double_layer / eval_total_field
// (/root/reference/pkg/src/tdbem/potential.py:53-126):
//   u(x, t) = -(1/4pi) sum_e sum_q w_q 2|e| (n_e.(x - y)/r) (phi(y, t - r)/r^2 + phi_t(y, t - r)/r)
// with r = |x - y|, phi(y, s) = sum_i b_i(s) sum_a shape_a(y) alpha[i][tri_e[a]] over
// the basis functions whose (open) support contains the retarded time s
// (potential.py:84-94), and the q_near rule on triangles closer than twice their
// longest edge to x (potential.py:67-76, distance bitwise as the reference's).
//
// One CTA per (point, time); threads stride over (triangle, rule point); the
// temporal basis b_i, b_i' (temporal_basis.py canonical prototypes: erf cutoff,
// Legendre factors) is evaluated in closed form only for the 1-3 time steps whose
// support can contain s; the CTA sum is a fixed-order block reduction.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "tdb_basis.cuh"
#include "tdb_common.cuh"
#include "tdb_geometry.cuh"
#include "tdb_internal.h"

namespace tdb {
namespace {

struct DlpArgs {
  int E, M, N, p;
  double dt;
  const double* corners;  // (E,3,3)
  const double* normals;  // (E,3)
  const double* a2;       // (E,) 2 |e|
  const int* tri;         // (E,3)
  const double* alpha;    // (L, M) density coefficients
  int nqf, nqn;
  const double* rule;     // far then near: x1, x2, w per point (3 * (nqf + nqn))
  long long npts;
  const double* points;   // (npts, 3)
  const double* times;    // (ntimes,)
  double* out;            // (ntimes, npts)
};

constexpr int kDlpThreads = 256;

__global__ void __launch_bounds__(kDlpThreads) k_dlp(DlpArgs a) {
  const long long pt = blockIdx.x % a.npts;
  const long long ti = blockIdx.x / a.npts;
  const V3 X = {a.points[3 * pt], a.points[3 * pt + 1], a.points[3 * pt + 2]};
  const double t = a.times[ti];
  const int np1 = a.p + 1;
  const double dt = a.dt;
  double acc = 0.0;
  for (int e = threadIdx.x; e < a.E; e += kDlpThreads) {
    const V3 c0 = corner(a.corners, e, 0), c1 = corner(a.corners, e, 1), c2 = corner(a.corners, e, 2);
    const double diam = fmax(fmax(enorm(vsub(c0, c1)), enorm(vsub(c1, c2))), enorm(vsub(c2, c0)));
    const bool near = pt_tri(X, c0, c1, c2) < 2.0 * diam;
    const int nq = near ? a.nqn : a.nqf;
    const double* R = a.rule + 3 * (near ? a.nqf : 0);
    const V3 e1 = sub(c1, c0), e2 = sub(c2, c1);
    const double nx = a.normals[3 * e], ny = a.normals[3 * e + 1], nz = a.normals[3 * e + 2];
    const double ar = a.a2[e];
    const int v0 = a.tri[3 * e], v1 = a.tri[3 * e + 1], v2 = a.tri[3 * e + 2];
    double sum_e = 0.0;
    for (int q = 0; q < nq; ++q) {
      const double x1 = R[3 * q], x2 = R[3 * q + 1], w = R[3 * q + 2];
      const double dx = X.x - (c0.x + x1 * e1.x + x2 * e2.x);
      const double dy = X.y - (c0.y + x1 * e1.y + x2 * e2.y);
      const double dz = X.z - (c0.z + x1 * e1.z + x2 * e2.z);
      const double r = sqrt(dx * dx + dy * dy + dz * dz);
      const double tret = t - r;
      if (tret <= 0.0) continue;  // every support starts at t >= 0
      const double sh0 = 1.0 - x1, sh1 = x1 - x2, sh2 = x2;
      // time steps whose support can contain tret: inner k covers ((k-2)dt, k dt)
      const int kc = (int)floor(tret / dt);
      double phi = 0.0, phit = 0.0;
      for (int k = max(1, kc); k <= min(a.N, kc + 3); ++k) {
        const int kind = k == 1 ? 0 : (k == a.N ? 2 : 1);
        const double o = kind == 0 ? 0.0 : (kind == 2 ? (double)(a.N - 2) * dt : (double)(k - 2) * dt);
        const double hi = o + (kind == 1 ? 2.0 * dt : dt);
        if (!(tret > o && tret < hi)) continue;  // potential.py:86-88 (open interval)
        for (int m = 0; m < np1; ++m) {
          const double* al = a.alpha + (long long)((k - 1) * np1 + m) * a.M;
          const double dof = sh0 * al[v0] + sh1 * al[v1] + sh2 * al[v2];
          double b0, b1, b2;
          basis012(kind, m, dt, tret - o, b0, b1, b2);
          phi = fma(b0, dof, phi);
          phit = fma(b1, dof, phit);
        }
      }
      const double ndotd = nx * dx + ny * dy + nz * dz;
      sum_e = fma(w * ndotd / r, phi / (r * r) + phit / r, sum_e);
    }
    acc = fma(ar, sum_e, acc);
  }
  // fixed-order block reduction
  __shared__ double red[kDlpThreads / 32];
  acc = warp_allsum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kDlpThreads / 32; ++w) s += red[w];
    a.out[ti * a.npts + pt] = -kInv4Pi * s;
  }
}

}  // namespace
}  // namespace tdb

using namespace tdb;

extern "C" int tdb_dlp_eval(TdbContext* ctx, const TdbMesh* mesh, double T, int32_t N, int32_t p,
                            const double* coeffs, int64_t npts, const double* points, int64_t ntimes,
                            const double* times, int32_t nq_far, const double* far_xhat, const double* far_w,
                            int32_t nq_near, const double* near_xhat, const double* near_w, double* out) {
  TDB_REQUIRE(ctx && mesh && coeffs && points && times && out && far_xhat && far_w && near_xhat && near_w,
              "dlp: NULL argument");
  TDB_REQUIRE(T > 0.0 && N >= 3 && p >= 0 && p <= 8, "dlp: bad time grid");
  TDB_REQUIRE(npts >= 0 && ntimes >= 0 && nq_far >= 1 && nq_near >= 1, "dlp: bad sizes");
  if (npts == 0 || ntimes == 0) return TDB_OK;
  TDB_CUDA_CHECK(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  const long long E = mesh->num_triangles, M = mesh->num_vertices, L = (long long)N * (p + 1);
  std::vector<int> tri(3 * E);
  for (long long i = 0; i < 3 * E; ++i) tri[i] = (int)mesh->triangles[i];
  std::vector<double> rule;
  for (int q = 0; q < nq_far; ++q) rule.insert(rule.end(), {far_xhat[2 * q], far_xhat[2 * q + 1], far_w[q]});
  for (int q = 0; q < nq_near; ++q) rule.insert(rule.end(), {near_xhat[2 * q], near_xhat[2 * q + 1], near_w[q]});
  struct Buf {
    void* p = nullptr;
    ~Buf() { dev_free(p); }
  } bc, bn, ba, bt, bal, br, bp, btm, bo;
  auto up = [&](Buf& b, const void* h, size_t bytes) -> int {
    TDB_CUDA_CHECK(dev_malloc(&b.p, bytes));
    if (h) TDB_CUDA_CHECK(cudaMemcpyAsync(b.p, h, bytes, cudaMemcpyHostToDevice, st));
    return TDB_OK;
  };
  int rc;
  if ((rc = up(bc, mesh->corners, 9 * E * sizeof(double)))) return rc;
  if ((rc = up(bn, mesh->normals, 3 * E * sizeof(double)))) return rc;
  if ((rc = up(ba, mesh->a2, E * sizeof(double)))) return rc;
  if ((rc = up(bt, tri.data(), 3 * E * sizeof(int)))) return rc;
  if ((rc = up(bal, coeffs, L * M * sizeof(double)))) return rc;
  if ((rc = up(br, rule.data(), rule.size() * sizeof(double)))) return rc;
  if ((rc = up(bp, points, 3 * npts * sizeof(double)))) return rc;
  if ((rc = up(btm, times, ntimes * sizeof(double)))) return rc;
  if ((rc = up(bo, nullptr, npts * ntimes * sizeof(double)))) return rc;
  DlpArgs a;
  a.E = (int)E;
  a.M = (int)M;
  a.N = N;
  a.p = p;
  a.dt = T / (N - 1);  // TimeGrid.dt (temporal_basis.py:67)
  a.corners = (const double*)bc.p;
  a.normals = (const double*)bn.p;
  a.a2 = (const double*)ba.p;
  a.tri = (const int*)bt.p;
  a.alpha = (const double*)bal.p;
  a.nqf = nq_far;
  a.nqn = nq_near;
  a.rule = (const double*)br.p;
  a.npts = npts;
  a.points = (const double*)bp.p;
  a.times = (const double*)btm.p;
  a.out = (double*)bo.p;
  const long long blocks = npts * ntimes;
  TDB_REQUIRE(blocks < (1LL << 31), "dlp: too many (point, time) pairs per call");
  k_dlp<<<(unsigned)blocks, kDlpThreads, 0, st>>>(a);
  TDB_CUDA_CHECK(cudaGetLastError());
  TDB_CUDA_CHECK(cudaMemcpyAsync(out, bo.p, npts * ntimes * sizeof(double), cudaMemcpyDeviceToHost, st));
  TDB_CUDA_CHECK(cudaStreamSynchronize(st));
  return TDB_OK;
}
