// psi / psi~ prototype tables on the device.
//
// Replaces the quadrature loop of PrototypeTables.build / _node_values
// (/root/reference/pkg/src/tdbem/kernel_weights.py:243-295; this package's
// kernel_weights.py:186-244): for every table subinterval and Chebyshev-Lobatto
// node alpha, the defining integrals
//   psi  = int b_i''(u - alpha) bdot_k(u) du,   psi~ = int b_i(u - alpha) bdot_k(u) du
// over 32-point Gauss panels whose ends are affine in alpha (split at dt
// multiples, ceil(4 len/dt) sub-panels).  The panel structure is decided on the
// host at each subinterval midpoint exactly as the host build does; this kernel
// evaluates every (subinterval, node) integral, one thread each.  The 17 x 17
// Lobatto -> Chebyshev transform stays on the host.
#include <cuda_runtime.h>

#include <algorithm>

#include "tdb_basis.cuh"
#include "tdb_common.cuh"
#include "tdb_internal.h"

namespace tdb {
namespace {

constexpr int kMaxP1 = 4;  // p <= 3

struct TabArgs {
  int nsub, nnodes, nq, np1;
  double dt;
  const int* kinds;        // (nsub, 2): kind_i (ansatz), kind_k (test); 0 first, 1 inner, 2 last
  const double* a0w;       // (nsub, 2): subinterval start, width
  const double* nodes;     // (nnodes,) Lobatto nodes on [-1, 1]
  const int* pptr;         // (nsub + 1,) panel ranges
  const double* panels;    // (npanels, 5): e0 = c0 + s0 a, e1 = c1 + s1 a, n_split
  const double* xq;        // (nq,)
  const double* wq;
  double* out;             // (nsub, 2, np1, np1, nnodes)
};

__global__ void k_table_nodes(TabArgs a) {
  const long long n_total = (long long)a.nsub * a.nnodes;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n_total;
       i += (long long)gridDim.x * blockDim.x) {
    const int sub = (int)(i / a.nnodes), nd = (int)(i % a.nnodes);
    const int ki = a.kinds[2 * sub], kk = a.kinds[2 * sub + 1];
    const double a0 = a.a0w[2 * sub], width = a.a0w[2 * sub + 1];
    const double alpha = a0 + 0.5 * width * (a.nodes[nd] + 1.0);
    const int np1 = a.np1;
    double s2[kMaxP1][kMaxP1] = {}, s0[kMaxP1][kMaxP1] = {};
    for (int pn = a.pptr[sub]; pn < a.pptr[sub + 1]; ++pn) {
      const double* P = a.panels + 5 * pn;
      const double ua = P[0] + P[1] * alpha, ub = P[2] + P[3] * alpha;
      const int ns = (int)P[4];
      for (int j = 0; j < ns; ++j) {
        const double qa = ua + (ub - ua) * ((double)j / ns);
        const double qb = ua + (ub - ua) * ((double)(j + 1) / ns);
        const double h = 0.5 * (qb - qa);
        const double mid = 0.5 * (qa + qb);
        const double hw = fmax(h, 0.0);
        for (int q = 0; q < a.nq; ++q) {
          const double U = mid + h * a.xq[q];
          const double W = hw * a.wq[q];
          const double S = U - alpha;
          double test[kMaxP1], d0[kMaxP1], d2[kMaxP1];
          for (int m = 0; m < np1; ++m) {
            double b0, b1, b2;
            basis012(kk, m, a.dt, U, b0, b1, b2);
            test[m] = W * b1;
            basis012(ki, m, a.dt, S, b0, b1, b2);
            d0[m] = b0;
            d2[m] = b2;
          }
          for (int m1 = 0; m1 < np1; ++m1)
            for (int m2 = 0; m2 < np1; ++m2) {
              s2[m1][m2] = fma(d2[m1], test[m2], s2[m1][m2]);
              s0[m1][m2] = fma(d0[m1], test[m2], s0[m1][m2]);
            }
        }
      }
    }
    for (int m1 = 0; m1 < np1; ++m1)
      for (int m2 = 0; m2 < np1; ++m2) {
        a.out[((((long long)sub * 2 + 0) * np1 + m1) * np1 + m2) * a.nnodes + nd] = s2[m1][m2];
        a.out[((((long long)sub * 2 + 1) * np1 + m1) * np1 + m2) * a.nnodes + nd] = s0[m1][m2];
      }
  }
}

}  // namespace
}  // namespace tdb

using namespace tdb;

extern "C" int tdb_table_node_values(TdbContext* ctx, double dt, int32_t p, int32_t nsub, const int32_t* kinds,
                                     const double* a0w, int32_t nnodes, const double* nodes, const int32_t* pptr,
                                     const double* panels, int32_t nq, const double* xq, const double* wq,
                                     double* out) {
  TDB_REQUIRE(ctx && kinds && a0w && nodes && pptr && panels && xq && wq && out, "tables: NULL argument");
  TDB_REQUIRE(dt > 0.0 && p >= 0 && p < kMaxP1 && nsub >= 1 && nnodes >= 1 && nq >= 1, "tables: bad argument");
  TDB_CUDA_CHECK(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  const int np1 = p + 1;
  const long long npanels = pptr[nsub];
  const size_t out_n = (size_t)nsub * 2 * np1 * np1 * nnodes;
  struct Buf {
    void* p = nullptr;
    ~Buf() { dev_free(p); }
  } bk, ba, bn, bp, bpn, bx, bw, bo;
  auto up = [&](Buf& b, const void* h, size_t bytes) -> int {
    TDB_CUDA_CHECK(dev_malloc(&b.p, std::max<size_t>(bytes, 8)));
    if (h && bytes) TDB_CUDA_CHECK(cudaMemcpyAsync(b.p, h, bytes, cudaMemcpyHostToDevice, st));
    return TDB_OK;
  };
  int rc;
  if ((rc = up(bk, kinds, 2 * (size_t)nsub * sizeof(int)))) return rc;
  if ((rc = up(ba, a0w, 2 * (size_t)nsub * sizeof(double)))) return rc;
  if ((rc = up(bn, nodes, (size_t)nnodes * sizeof(double)))) return rc;
  if ((rc = up(bp, pptr, ((size_t)nsub + 1) * sizeof(int)))) return rc;
  if ((rc = up(bpn, panels, 5 * (size_t)npanels * sizeof(double)))) return rc;
  if ((rc = up(bx, xq, (size_t)nq * sizeof(double)))) return rc;
  if ((rc = up(bw, wq, (size_t)nq * sizeof(double)))) return rc;
  if ((rc = up(bo, nullptr, out_n * sizeof(double)))) return rc;
  TabArgs a;
  a.nsub = nsub;
  a.nnodes = nnodes;
  a.nq = nq;
  a.np1 = np1;
  a.dt = dt;
  a.kinds = (const int*)bk.p;
  a.a0w = (const double*)ba.p;
  a.nodes = (const double*)bn.p;
  a.pptr = (const int*)bp.p;
  a.panels = (const double*)bpn.p;
  a.xq = (const double*)bx.p;
  a.wq = (const double*)bw.p;
  a.out = (double*)bo.p;
  const long long n = (long long)nsub * nnodes;
  k_table_nodes<<<(int)std::min<long long>((n + 127) / 128, 148LL * 8), 128, 0, st>>>(a);
  TDB_CUDA_CHECK(cudaGetLastError());
  TDB_CUDA_CHECK(cudaMemcpyAsync(out, bo.p, out_n * sizeof(double), cudaMemcpyDeviceToHost, st));
  TDB_CUDA_CHECK(cudaStreamSynchronize(st));
  return TDB_OK;
}
