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
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>
#include <cmath>
#include <cstdlib>

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

// One fused Arnoldi step after the matvec (thread-block cluster, DSMEM reductions):
//   two classical Gram-Schmidt passes  h_p = V[0..k] w,  w -= V[0..k]^T h_p  (CGS2),
//   hcol[0..k] = h_1 + h_2, hcol[k+1] = ||w||, then (optionally) the Givens step of
//   k_krylov_givens and V[k+1] = w / ||w||.
// Each CTA owns a contiguous slice of the vector; a partial sum is reduced
// warp -> CTA (shared memory) -> cluster (every CTA reads all ranks' partials
// through distributed shared memory in rank order), so every CTA holds the same
// coefficients (deterministic, no atomics) and the step is one launch.
constexpr int kArnThreads = 256;
constexpr int kArnMaxK = 64;  // restart lengths up to 64
constexpr int kArnMaxCluster = 16;  // non-portable cluster size used by the launcher

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(kArnThreads) k_krylov_arnoldi(const double* __restrict__ V, long long ldv,
                                                               long long n, int k, double* __restrict__ w,
                                                               double* hcol, double* st, double* H, int ldh,
                                                               double* cs, double* sn, double* g,
                                                               double* vnext) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int crank = (int)cl.block_rank(), csize = (int)cl.num_blocks();
  constexpr int NW = kArnThreads / 32;
  __shared__ double red[kArnMaxK + 1][NW];
  __shared__ double cta[2][kArnMaxK + 1];  // double-buffered: pass p uses cta[p & 1]
  __shared__ double h[kArnMaxK + 1], hs[kArnMaxK + 1];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const long long per = (n + csize - 1) / csize;
  const long long lo = (long long)crank * per, hi = min(n, lo + per);
  const int nj = k + 1;
  for (int j = tid; j < nj; j += kArnThreads) hs[j] = 0.0;
  // passes 0, 1: CGS; pass 2: the norm of w (nj = 1 "coefficient")
  for (int pass = 0; pass < 3; ++pass) {
    const int nc = pass < 2 ? nj : 1;
    double* cb = cta[pass & 1];
    // up to 8 coefficients per sweep of the slice (independent accumulators and
    // warp reductions: the dependent-latency chain is one sweep, not k + 1)
    for (int jb = 0; jb < nc; jb += 8) {
      double loc[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) loc[u] = 0.0;
      if (pass < 2) {
        const double* vb = V + (long long)jb * ldv;
        const int nu = min(8, nc - jb);
        for (long long i = lo + tid; i < hi; i += kArnThreads) {
          const double wi = w[i];
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (u < nu) loc[u] = fma(vb[(long long)u * ldv + i], wi, loc[u]);
        }
      } else {
        for (long long i = lo + tid; i < hi; i += kArnThreads) loc[0] = fma(w[i], w[i], loc[0]);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const double r_ = warp_sum(loc[u]);
        if (lane == 0 && jb + u < nc) red[jb + u][wid] = r_;
      }
    }
    __syncthreads();
    for (int j = tid; j < nc; j += kArnThreads) {
      double s_ = 0.0;
#pragma unroll
      for (int q = 0; q < NW; ++q) s_ += red[j][q];
      cb[j] = s_;
    }
    cl.sync();
    for (int j = tid; j < nc; j += kArnThreads) {
      // every rank's partial loaded first (independent DSMEM loads in flight),
      // then summed in rank order
      double pr[kArnMaxCluster];
#pragma unroll
      for (int r = 0; r < kArnMaxCluster; ++r) pr[r] = r < csize ? *cl.map_shared_rank(cb + j, r) : 0.0;
      double s_ = 0.0;
#pragma unroll
      for (int r = 0; r < kArnMaxCluster; ++r)
        if (r < csize) s_ += pr[r];
      h[j] = s_;
      if (pass < 2) hs[j] += s_;
    }
    __syncthreads();
    if (pass < 2)
      for (long long i = lo + tid; i < hi; i += kArnThreads) {
        double acc = 0.0;
        for (int j = 0; j < nj; ++j) acc = fma(V[(long long)j * ldv + i], h[j], acc);
        w[i] -= acc;
      }
    __syncthreads();
  }
  const double hk = sqrt(h[0]);
  if (crank == 0 && tid == 0) {
    for (int j = 0; j < nj; ++j) hcol[j] = hs[j];
    hcol[nj] = hk;
  }
  if (H != nullptr && crank == 0) {
    // the Givens step of k_krylov_givens (same arithmetic), with the rotations
    // staged in shared memory and the rotated column carried in registers: one
    // thread, no dependent global round trips
    __shared__ double s_cs[kArnMaxK], s_sn[kArnMaxK];
    __shared__ double s_g;
    __shared__ int s_done;
    for (int j = tid; j < k; j += kArnThreads) {
      s_cs[j] = cs[j];
      s_sn[j] = sn[j];
    }
    if (tid == 0) {
      s_done = st[TDB_KS_DONE] != 0.0;
      s_g = g[k];
    }
    __syncthreads();
    if (tid == 0 && !s_done) {
      double* col = H + k;
      double a = hs[0];
      for (int j = 0; j < k; ++j) {
        const double b = hs[j + 1];
        const double t = s_cs[j] * a + s_sn[j] * b;
        a = -s_sn[j] * a + s_cs[j] * b;
        col[j * ldh] = t;
      }
      const double hkk = a, hk1 = hk;
      const double denom = hypot(hkk, hk1);
      const double c = denom > 0.0 ? hkk / denom : 1.0;
      const double sg = denom > 0.0 ? hk1 / denom : 0.0;
      cs[k] = c;
      sn[k] = sg;
      col[k * ldh] = denom;
      const double gk = s_g;
      g[k + 1] = -sg * gk;
      g[k] = c * gk;
      col[(k + 1) * ldh] = 0.0;
      st[TDB_KS_KDONE] = (double)(k + 1);
      if (fabs(-sg * gk) <= st[TDB_KS_TOL_ABS]) {
        st[TDB_KS_DONE] = 1.0;
        st[TDB_KS_CONVERGED] = 1.0;
      } else if (hk <= 1e-14 * st[TDB_KS_BETA]) {
        st[TDB_KS_DONE] = 1.0;
        st[TDB_KS_BREAKDOWN] = 1.0;
      }
    }
  }
  if (vnext != nullptr) {
    const double inv = 1.0 / hk;
    for (long long i = lo + tid; i < hi; i += kArnThreads) vnext[i] = w[i] * inv;
  }
  cl.sync();  // peers may still read this CTA's partials
}

// ---- grid-wide Arnoldi step (long vectors) -----------------------------------
// The cluster kernel above keeps a step in one launch but uses at most 16 SMs; for
// long vectors (the quarter-range inner solves of the preconditioner: 1e5 entries,
// the outer cycle: 4e5) the step runs as four full-grid launches instead, each CTA
// streaming its slice of V and w: dots -> (update, dots) -> (update, norm) ->
// (Givens, normalise).  Per-CTA partials are summed by the last CTA to finish
// (threadfence + ticket), in CTA order: deterministic, no host round trip, capturable.
constexpr int kArnGridThreads = 256;
constexpr int kArnK1 = kArnMaxK + 1;

struct ArnWs {
  double* part;       // [G][kArnK1] per-CTA partial sums
  double* h;          // [3][kArnK1]: pass-1 and pass-2 coefficients, ||w||^2
  unsigned* counter;  // CTAs done with the current reduction
  int G;
};

__device__ __forceinline__ void arn_slice(long long n, int G, long long& lo, long long& hi) {
  const long long per = (n + G - 1) / G;
  lo = (long long)blockIdx.x * per;
  hi = min(n, lo + per);
}

// this CTA's partial sums of V[j] . w (j < nc) or w . w (norm) -> part[blockIdx.x][*]
__device__ void arn_partials(const double* __restrict__ V, long long ldv, int nc, bool norm,
                             const double* __restrict__ w, long long lo, long long hi, double* part) {
  constexpr int NW = kArnGridThreads / 32;
  __shared__ double red[kArnK1][NW];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int jb = 0; jb < nc; jb += 8) {
    double loc[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) loc[u] = 0.0;
    if (!norm) {
      const double* vb = V + (long long)jb * ldv;
      const int nu = min(8, nc - jb);
      for (long long i = lo + tid; i < hi; i += kArnGridThreads) {
        const double wi = w[i];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (u < nu) loc[u] = fma(vb[(long long)u * ldv + i], wi, loc[u]);
      }
    } else {
      for (long long i = lo + tid; i < hi; i += kArnGridThreads) loc[0] = fma(w[i], w[i], loc[0]);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double r_ = warp_sum(loc[u]);
      if (lane == 0 && jb + u < nc) red[jb + u][wid] = r_;
    }
  }
  __syncthreads();
  for (int j = tid; j < nc; j += kArnGridThreads) {
    double s_ = 0.0;
#pragma unroll
    for (int q = 0; q < NW; ++q) s_ += red[j][q];
    part[(long long)blockIdx.x * kArnK1 + j] = s_;
  }
}

// the last CTA to arrive sums the partials in CTA order into hout
__device__ void arn_last_reduce(const ArnWs& ws, int nc, double* hout) {
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(ws.counter, 1u) == (unsigned)(gridDim.x - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int j = threadIdx.x; j < nc; j += kArnGridThreads) {
    double s_ = 0.0;
    for (int b = 0; b < (int)gridDim.x; ++b) s_ += __ldcg(ws.part + (long long)b * kArnK1 + j);
    hout[j] = s_;
  }
  if (threadIdx.x == 0) *ws.counter = 0u;
}

__global__ void __launch_bounds__(kArnGridThreads) k_arn_dots(const double* __restrict__ V, long long ldv, long long n,
                                                             int nj, const double* __restrict__ w, ArnWs ws) {
  long long lo, hi;
  arn_slice(n, gridDim.x, lo, hi);
  arn_partials(V, ldv, nj, false, w, lo, hi, ws.part);
  arn_last_reduce(ws, nj, ws.h);
}

// w -= V^T h[src]; then the next pass's partials (dots into h[1], or the norm into h[2])
__global__ void __launch_bounds__(kArnGridThreads) k_arn_update(const double* __restrict__ V, long long ldv,
                                                               long long n, int nj, double* __restrict__ w, ArnWs ws,
                                                               int src, int norm) {
  __shared__ double h[kArnK1];
  for (int j = threadIdx.x; j < nj; j += kArnGridThreads) h[j] = __ldcg(ws.h + src * kArnK1 + j);
  __syncthreads();
  long long lo, hi;
  arn_slice(n, gridDim.x, lo, hi);
  for (long long i = lo + threadIdx.x; i < hi; i += kArnGridThreads) {
    double acc = 0.0;
    for (int j = 0; j < nj; ++j) acc = fma(V[(long long)j * ldv + i], h[j], acc);
    w[i] -= acc;
  }
  __syncthreads();  // this CTA's w slice is final before its own partials read it
  arn_partials(V, ldv, norm ? 1 : nj, norm != 0, w, lo, hi, ws.part);
  arn_last_reduce(ws, norm ? 1 : nj, ws.h + (norm ? 2 : 1) * kArnK1);
}

// hcol = (h1 + h2, ||w||), the Givens step of k_krylov_givens (CTA 0), V[k+1] = w / ||w||
__global__ void __launch_bounds__(kArnGridThreads) k_arn_finish(ArnWs ws, long long n, int k, const double* __restrict__ w,
                                                               double* hcol, double* st, double* H, int ldh, double* cs,
                                                               double* sn, double* g, double* vnext) {
  const int nj = k + 1;
  const double hk = sqrt(__ldcg(ws.h + 2 * kArnK1));
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double hs[kArnK1];
    for (int j = 0; j < nj; ++j) {
      hs[j] = __ldcg(ws.h + j) + __ldcg(ws.h + kArnK1 + j);
      hcol[j] = hs[j];
    }
    hcol[nj] = hk;
    if (H != nullptr && st[TDB_KS_DONE] == 0.0) {
      double* col = H + k;
      double a = hs[0];
      for (int j = 0; j < k; ++j) {
        const double b = hs[j + 1];
        const double t = cs[j] * a + sn[j] * b;
        a = -sn[j] * a + cs[j] * b;
        col[j * ldh] = t;
      }
      const double denom = hypot(a, hk);
      const double c = denom > 0.0 ? a / denom : 1.0;
      const double sg = denom > 0.0 ? hk / denom : 0.0;
      cs[k] = c;
      sn[k] = sg;
      col[k * ldh] = denom;
      const double gk = g[k];
      g[k + 1] = -sg * gk;
      g[k] = c * gk;
      col[(k + 1) * ldh] = 0.0;
      st[TDB_KS_KDONE] = (double)(k + 1);
      if (fabs(-sg * gk) <= st[TDB_KS_TOL_ABS]) {
        st[TDB_KS_DONE] = 1.0;
        st[TDB_KS_CONVERGED] = 1.0;
      } else if (hk <= 1e-14 * st[TDB_KS_BETA]) {
        st[TDB_KS_DONE] = 1.0;
        st[TDB_KS_BREAKDOWN] = 1.0;
      }
    }
  }
  if (vnext != nullptr) {
    const double inv = 1.0 / hk;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
      vnext[i] = w[i] * inv;
  }
}

// per-device workspace of the grid-wide step (allocated on the first eager call; a
// call inside a stream capture before that uses the cluster kernel)
struct ArnWsCache {
  std::mutex mu;
  ArnWs ws[64] = {};
};
ArnWsCache& arn_cache() {
  static ArnWsCache* c = new ArnWsCache();
  return *c;
}

}  // namespace

extern "C" {

int tdb_krylov_arnoldi(const double* V, int64_t ldv, int64_t n, int32_t k, double* w, double* hcol, double* state,
                       double* H, int32_t ldh, double* cs, double* sn, double* g, double* vnext, void* stream) {
  TDB_REQUIRE(V && w && hcol && n > 0 && k >= 0 && k < kArnMaxK, "krylov_arnoldi: bad argument");
  TDB_REQUIRE(H == nullptr || (state && cs && sn && g && ldh > k), "krylov_arnoldi: bad Givens arguments");
  // the non-portable cluster size is a per-device function attribute: set it once per
  // device (bit set under a mutex; a second GPU in the same process gets its own call)
  static std::mutex mu;
  static unsigned long long done = 0ull;
  int dev = 0;
  TDB_CUDA_CHECK(cudaGetDevice(&dev));
  {
    std::lock_guard<std::mutex> g_(mu);
    if (dev < 64 && !((done >> dev) & 1ull)) {
      TDB_CUDA_CHECK(cudaFuncSetAttribute(k_krylov_arnoldi, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      done |= 1ull << dev;
    }
  }
  cudaStream_t cs_ = (cudaStream_t)stream;
  static const long long grid_min_n = [] {
    const char* e = std::getenv("TDB_ARNOLDI_GRID_MIN_N");
    return e ? std::atoll(e) : 32768LL;
  }();
  if (n >= grid_min_n && dev < 64) {
    ArnWsCache& C = arn_cache();
    ArnWs ws{};
    {
      std::lock_guard<std::mutex> g_(C.mu);
      ws = C.ws[dev];
      if (ws.part == nullptr) {
        cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
        TDB_CUDA_CHECK(cudaStreamIsCapturing(cs_, &cap));
        if (cap == cudaStreamCaptureStatusNone) {
          int sms = 148;
          cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
          ws.G = 2 * sms;
          void *pp = nullptr, *ph = nullptr, *pc = nullptr;
          if (dev_malloc(&pp, (size_t)ws.G * kArnK1 * sizeof(double)) != cudaSuccess ||
              dev_malloc(&ph, 3 * kArnK1 * sizeof(double)) != cudaSuccess ||
              dev_malloc(&pc, sizeof(unsigned)) != cudaSuccess) {
            set_error("krylov_arnoldi: workspace allocation failed");
            return TDB_E_NOMEM;
          }
          TDB_CUDA_CHECK(cudaMemset(pc, 0, sizeof(unsigned)));
          ws.part = static_cast<double*>(pp);
          ws.h = static_cast<double*>(ph);
          ws.counter = static_cast<unsigned*>(pc);
          C.ws[dev] = ws;
        }
      }
    }
    if (ws.part != nullptr) {
      const int G = (int)std::min<long long>(ws.G, std::max<long long>(1, n / 1024));
      k_arn_dots<<<G, kArnGridThreads, 0, cs_>>>(V, (long long)ldv, (long long)n, k + 1, w, ws);
      k_arn_update<<<G, kArnGridThreads, 0, cs_>>>(V, (long long)ldv, (long long)n, k + 1, w, ws, 0, 0);
      k_arn_update<<<G, kArnGridThreads, 0, cs_>>>(V, (long long)ldv, (long long)n, k + 1, w, ws, 1, 1);
      k_arn_finish<<<G, kArnGridThreads, 0, cs_>>>(ws, (long long)n, (int)k, w, hcol, state, H, (int)ldh, cs, sn, g,
                                                   vnext);
      TDB_CUDA_CHECK(cudaGetLastError());
      return TDB_OK;
    }
  }
  const int csize = 16;
  // cluster of up to 16 CTAs (one per SM), at least ~512 elements per CTA
  int cls = (int)std::min<long long>(csize, std::max<long long>(1, n / 512));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cls);
  cfg.blockDim = dim3(kArnThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cls;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  TDB_CUDA_CHECK(cudaLaunchKernelEx(&cfg, k_krylov_arnoldi, V, (long long)ldv, (long long)n, (int)k, w, hcol, state,
                                    H, (int)ldh, cs, sn, g, vnext));
  return TDB_OK;
}


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
