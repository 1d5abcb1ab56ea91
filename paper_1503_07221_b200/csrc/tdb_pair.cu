// Drop-in pair_block_contributions on the GPU (one block position, host buffers).
//
// Contract of tdbem._kernels.pair_block_contributions
// (/root/reference/pkg/src/tdbem/_kernels/__init__.py:1-34, _core.pyx:47-159):
// per pair P and rule point q, X = cx0 + x1 (cx1-cx0) + x2 (cx2-cx1), same for Y,
// r = |X - Y|, a = r + delta; points with a outside the union of the active
// table supports are skipped; common = a2x a2y w / (4 pi r);
//   out[P,m2,m1,a,b] += common nd psi shy[a] shx[b] + common psi~ (curly[a].curlx[b]).
// Here the point sum is factorised as nd * S[a][b] + cdot[a][b] * s with
// S = sum common psi shy shx and s = sum common psi~ (the NumPy twin's form,
// _fallback.py:263-273); the difference to the Cython loop is rounding only.
//
// One warp per pair; lanes stride over the rule points; deterministic xor
// butterfly reduction.  Tables stay in global memory (L1-resident): this entry
// exists for parity with the reference plugin, the throughput path is
// tdb_assembly.cu.

#include <cuda_runtime.h>

#include <vector>

#include "tdb_common.cuh"

namespace tdb {

struct PackDev {
  int np1, nt, deg, max_nsub;
  double delta, amin, amax;
  const double* lo;
  const double* width;
  const double* inv_w;
  const int* nsub;
  const double* coeffs;
  const double* sp;
  const double* sn;
  const unsigned char* fold;
  const unsigned char* active;
};

template <int P>
__global__ void __launch_bounds__(256) pair_contrib_kernel(
    const double* __restrict__ cx, const double* __restrict__ cy,
    const double* __restrict__ a2x, const double* __restrict__ a2y,
    const double* __restrict__ ndot, const double* __restrict__ curly,
    const double* __restrict__ curlx, const double* __restrict__ xhat,
    const double* __restrict__ yhat, const double* __restrict__ wq, long long npair,
    long long nq, PackDev pk, double* __restrict__ out) {
  constexpr int NP1 = P + 1;
  constexpr int NM = NP1 * NP1;
  constexpr int NACC = 10 * NM;
  const int lane = threadIdx.x & 31;
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long pr = warp; pr < npair; pr += nwarps) {
    const double* X = cx + 9 * pr;
    const double* Y = cy + 9 * pr;
    const double e1x = X[3] - X[0], e1y = X[4] - X[1], e1z = X[5] - X[2];
    const double e2x = X[6] - X[3], e2y = X[7] - X[4], e2z = X[8] - X[5];
    const double f1x = Y[3] - Y[0], f1y = Y[4] - Y[1], f1z = Y[5] - Y[2];
    const double f2x = Y[6] - Y[3], f2y = Y[7] - Y[4], f2z = Y[8] - Y[5];
    const double scale = kInv4Pi * a2x[pr] * a2y[pr];
    double acc[NACC];
#pragma unroll
    for (int k = 0; k < NACC; ++k) acc[k] = 0.0;
    for (long long q = lane; q < nq; q += 32) {
      const double x1 = xhat[2 * q], x2 = xhat[2 * q + 1];
      const double y1 = yhat[2 * q], y2 = yhat[2 * q + 1];
      const double dx = (X[0] + x1 * e1x + x2 * e2x) - (Y[0] + y1 * f1x + y2 * f2x);
      const double dy = (X[1] + x1 * e1y + x2 * e2y) - (Y[1] + y1 * f1y + y2 * f2y);
      const double dz = (X[2] + x1 * e1z + x2 * e2z) - (Y[2] + y1 * f1z + y2 * f2z);
      const double r = sqrt(dx * dx + dy * dy + dz * dz);
      const double av = r + pk.delta;
      if (av < pk.amin || av > pk.amax) continue;
      const double c = scale * wq[q] / r;
      const double shx0 = 1.0 - x1, shx1 = x1 - x2, shx2 = x2;
      const double shy[3] = {1.0 - y1, y1 - y2, y2};
      const double aa = fabs(av);
#pragma unroll
      for (int m = 0; m < NM; ++m) {
        double v[2];
#pragma unroll
        for (int v_ = 0; v_ < 2; ++v_) {
          const int t = 2 * m + v_;
          double val = 0.0;
          if (pk.active[t]) {
            const double a = pk.fold[t] ? aa : av;
            const double lo = pk.lo[t];
            const int ns = pk.nsub[t];
            if (a >= lo && a <= lo + ns * pk.width[t]) {
              double x;
              const int idx = cheb_locate(a, lo, pk.width[t], pk.inv_w[t], ns, x);
              val = clenshaw_dyn(pk.coeffs + ((long long)t * pk.max_nsub + idx) * (pk.deg + 1),
                                 pk.deg, x);
              if (pk.fold[t]) val *= (av >= 0.0 ? pk.sp[t] : pk.sn[t]);
            }
          }
          v[v_] = val;
        }
        const double cp = c * v[0];
        const double u0 = cp * shy[0], u1 = cp * shy[1], u2 = cp * shy[2];
        double* S = acc + 10 * m;
        S[0] = fma(u0, shx0, S[0]);
        S[1] = fma(u0, shx1, S[1]);
        S[2] = fma(u0, shx2, S[2]);
        S[3] = fma(u1, shx0, S[3]);
        S[4] = fma(u1, shx1, S[4]);
        S[5] = fma(u1, shx2, S[5]);
        S[6] = fma(u2, shx0, S[6]);
        S[7] = fma(u2, shx1, S[7]);
        S[8] = fma(u2, shx2, S[8]);
        S[9] = fma(c, v[1], S[9]);
      }
    }
#pragma unroll
    for (int k = 0; k < NACC; ++k) acc[k] = warp_allsum(acc[k]);
    // curl dots cdot[a][b] = curly[a] . curlx[b]; output lane i -> (m, a, b)
    const double nd = ndot[pr];
    for (int i = lane; i < 9 * NM; i += 32) {
      const int m = i / 9, ab = i % 9, a = ab / 3, b = ab % 3;
      const double* cyv = curly + 9 * pr + 3 * a;
      const double* cxv = curlx + 9 * pr + 3 * b;
      const double cd = cyv[0] * cxv[0] + cyv[1] * cxv[1] + cyv[2] * cxv[2];
      double Sab = 0.0, s = 0.0;
#pragma unroll
      for (int k = 0; k < NACC; ++k) {
        Sab = (k == 10 * m + ab) ? acc[k] : Sab;
        s = (k == 10 * m + 9) ? acc[k] : s;
      }
      out[9 * NM * pr + i] = nd * Sab + cd * s;
    }
  }
}

}  // namespace tdb

using namespace tdb;

namespace {

struct DevBuf {
  void* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

template <typename T>
int upload(DevBuf& b, const T* host, size_t n) {
  if (n == 0) n = 1;
  TDB_CUDA_CHECK(cudaMalloc(&b.p, n * sizeof(T)));
  if (host) TDB_CUDA_CHECK(cudaMemcpy(b.p, host, n * sizeof(T), cudaMemcpyHostToDevice));
  return TDB_OK;
}

}  // namespace

extern "C" int tdb_pair_block_contributions(const double* cx, const double* cy,
                                            const double* a2x, const double* a2y,
                                            const double* ndot, const double* curly,
                                            const double* curlx, const double* xhat,
                                            const double* yhat, const double* wq,
                                            int64_t npair, int64_t nq,
                                            const TdbPsiPack* pack, double* out) {
  TDB_REQUIRE(pack != nullptr, "pack is NULL");
  TDB_REQUIRE(npair >= 0 && nq >= 0, "negative size");
  TDB_REQUIRE(pack->p >= 0 && pack->p <= 3, "pair_block_contributions: p must be in 0..3");
  TDB_REQUIRE(pack->deg >= 0 && pack->max_nsub >= 1, "invalid table shape");
  const int np1 = pack->p + 1;
  const int nt = 2 * np1 * np1;
  const size_t nout = (size_t)npair * np1 * np1 * 9;
  if (npair == 0) return TDB_OK;
  if (nq == 0) {
    for (size_t i = 0; i < nout; ++i) out[i] = 0.0;
    return TDB_OK;
  }
  // union of active supports in offset space (_core.pyx:122-135)
  double amin = 1e300, amax = -1e300;
  std::vector<double> inv_w(nt);
  std::vector<int> nsub(nt);
  for (int t = 0; t < nt; ++t) {
    inv_w[t] = 1.0 / pack->width[t];
    nsub[t] = (int)pack->nsub[t];
    if (!pack->active[t]) continue;
    const double thi = pack->lo[t] + pack->nsub[t] * pack->width[t];
    if (pack->fold[t]) {
      if (-thi < amin) amin = -thi;
    } else if (pack->lo[t] < amin) {
      amin = pack->lo[t];
    }
    if (thi > amax) amax = thi;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    set_error("no CUDA device visible");
    return TDB_E_NODEVICE;
  }
  DevBuf dcx, dcy, da2x, da2y, dnd, dcuy, dcux, dxh, dyh, dw, dout;
  DevBuf dlo, dwid, dinv, dns, dco, dsp, dsn, dfo, dac;
  int rc;
#define UP(buf, ptr, n)                      \
  if ((rc = upload(buf, ptr, n)) != TDB_OK) \
    return rc;
  UP(dcx, cx, 9 * (size_t)npair);
  UP(dcy, cy, 9 * (size_t)npair);
  UP(da2x, a2x, (size_t)npair);
  UP(da2y, a2y, (size_t)npair);
  UP(dnd, ndot, (size_t)npair);
  UP(dcuy, curly, 9 * (size_t)npair);
  UP(dcux, curlx, 9 * (size_t)npair);
  UP(dxh, xhat, 2 * (size_t)nq);
  UP(dyh, yhat, 2 * (size_t)nq);
  UP(dw, wq, (size_t)nq);
  UP(dout, (const double*)nullptr, nout);
  UP(dlo, pack->lo, nt);
  UP(dwid, pack->width, nt);
  UP(dinv, inv_w.data(), nt);
  UP(dns, nsub.data(), nt);
  UP(dco, pack->coeffs, (size_t)nt * pack->max_nsub * (pack->deg + 1));
  UP(dsp, pack->sp, nt);
  UP(dsn, pack->sn, nt);
  UP(dfo, pack->fold, nt);
  UP(dac, pack->active, nt);
#undef UP
  PackDev pk;
  pk.np1 = np1;
  pk.nt = nt;
  pk.deg = pack->deg;
  pk.max_nsub = pack->max_nsub;
  pk.delta = pack->delta;
  pk.amin = amin;
  pk.amax = amax;
  pk.lo = (const double*)dlo.p;
  pk.width = (const double*)dwid.p;
  pk.inv_w = (const double*)dinv.p;
  pk.nsub = (const int*)dns.p;
  pk.coeffs = (const double*)dco.p;
  pk.sp = (const double*)dsp.p;
  pk.sn = (const double*)dsn.p;
  pk.fold = (const unsigned char*)dfo.p;
  pk.active = (const unsigned char*)dac.p;
  const int threads = 256;
  long long blocks = (npair + 7) / 8;
  if (blocks > 148 * 64) blocks = 148 * 64;
#define LAUNCH(PP)                                                                       \
  pair_contrib_kernel<PP><<<(unsigned)blocks, threads>>>(                                \
      (const double*)dcx.p, (const double*)dcy.p, (const double*)da2x.p,                 \
      (const double*)da2y.p, (const double*)dnd.p, (const double*)dcuy.p,                \
      (const double*)dcux.p, (const double*)dxh.p, (const double*)dyh.p,                 \
      (const double*)dw.p, npair, nq, pk, (double*)dout.p)
  switch (pack->p) {
    case 0: LAUNCH(0); break;
    case 1: LAUNCH(1); break;
    case 2: LAUNCH(2); break;
    default: LAUNCH(3); break;
  }
#undef LAUNCH
  TDB_CUDA_CHECK(cudaGetLastError());
  TDB_CUDA_CHECK(cudaMemcpy(out, dout.p, nout * sizeof(double), cudaMemcpyDeviceToHost));
  return TDB_OK;
}
