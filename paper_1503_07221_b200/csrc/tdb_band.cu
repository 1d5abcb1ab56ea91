// Lag-band tiles: the block-Toeplitz part of the matvec on the FP64 tensor cores (p = 0).
//
// Replaces the lag-reused part of BlockHessenbergMatrix.matvec (/root/reference/
// pkg/src/tdbem/block_system.py:180-216, a SciPy CSR SpMV per logical block
// position).  The inner family's stored blocks A_s (lag d_s = d_0 + s) act as
//     Y[j][kt] += sum_s sum_l A_s[j][l] X[l][kt - d_s]     (kt over the plan's rows)
// i.e. for every (test vertex j, column vertex l) a short 1-D correlation over
// the contiguous band of lags whose light cone the dof pair touches.
//
// Storage (built once per family, on first use): tiles of 8 test rows (Morton
// order, row block J) x 4 consecutive lags (S-tile: s = 4S .. 4S+3) for ONE column
// vertex l, in the mma.m8n8k4 A-fragment order (lane = 4 * row + lag).  Tiles are
// sorted (J, l, S).  The dof pair's lag band is contiguous and neighbouring rows
// have neighbouring bands, so the tiles are ~80% full (the (j, l)-tiled layout of
// round 1 was ~50%, and re-gathered x per tile).
//
// Matvec: the B operand of tile (J, l, S) at time tile u is a Hankel window of
// ONE row of the vertex-major iterate: B[k][n] = X[l][kt0 + n - d_0 - 4S - k], so
// lane (n = lane / 4, k = lane % 4) reads xt[l][off0 - 4S - k + n + 8u] - a
// broadcast-heavy, L1-resident load (all S-tiles of (J, l) reuse the row).  One
// CTA = (row block J, part of J's tile list); its warps split the time tiles and
// walk the same tiles (A fragments from L1 after the first warp).  Columns outside
// the plan's range are zero pads of xt; positions outside the plan (or whose
// logical mask is not the full band, e.g. the light-cone tie lag) are masked off
// per lane and handled by the CSR kernel.  Part partials are summed in part order
// (deterministic) and added to y after the CSR kernel has written it.
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <string>

#include "tdb_band.h"
#include "tdb_common.cuh"
#include "tdb_internal.h"

namespace tdb {

namespace {

__global__ void k_band_keys(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                            long long nrows_total, int nrows, int V, int nS, const int* __restrict__ rinv,
                            unsigned long long* __restrict__ keys, long long* __restrict__ ids) {
  const int lane = threadIdx.x & 31;
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long row = warp; row < nrows_total; row += nw) {
    const int s = (int)(row / nrows);
    const int jp = rinv[(int)(row % nrows)];
    const int64_t e0 = indptr[row], e1 = indptr[row + 1];
    const unsigned sub = (unsigned)((jp & 7) * 4 + (s & 3));
    for (int64_t e = e0 + lane; e < e1; e += 32) {
      const unsigned long long k =
          ((unsigned long long)(jp >> 3) * (unsigned long long)V + (unsigned long long)indices[e]) *
              (unsigned long long)nS + (unsigned long long)(s >> 2);
      keys[e] = (k << 5) | sub;
      ids[e] = e;
    }
  }
}

__global__ void k_band_heads(const unsigned long long* __restrict__ keys, long long n, int* __restrict__ head) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    head[i] = (i == 0 || (keys[i] >> 5) != (keys[i - 1] >> 5)) ? 1 : 0;
}

__global__ void k_band_fill(const unsigned long long* __restrict__ keys, const long long* __restrict__ ids,
                            const int* __restrict__ tid_incl, long long n, int V, int nS,
                            const double* __restrict__ data, int32_t* __restrict__ col, int32_t* __restrict__ stile,
                            double* __restrict__ val, int* __restrict__ tile_rb) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long t = tid_incl[i] - 1;
    const unsigned long long k = keys[i] >> 5;
    val[t * 32 + (keys[i] & 31u)] = data[ids[i]];
    if (i == 0 || (keys[i - 1] >> 5) != k) {
      stile[t] = (int32_t)(k % (unsigned long long)nS);
      const unsigned long long jl = k / (unsigned long long)nS;
      col[t] = (int32_t)(jl % (unsigned long long)V);
      tile_rb[t] = (int)(jl / (unsigned long long)V);
    }
  }
}

__global__ void k_band_rbptr(const int* __restrict__ tile_rb, long long ntiles, int nRB, int64_t* __restrict__ rbptr) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k <= nRB; k += (long long)gridDim.x * blockDim.x) {
    long long lo = 0, hi = ntiles;
    while (lo < hi) {
      const long long mid = (lo + hi) >> 1;
      if (tile_rb[mid] < (int)k) lo = mid + 1; else hi = mid;
    }
    rbptr[k] = lo;
  }
}

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// One CTA = (row block J, part); warp w owns time tiles [w TT, w TT + TT).  Two
// tiles per step: both tiles' A and B loads are issued before their DMMAs.
template <int TT>
__global__ void __launch_bounds__(kBandMaxWarps * 32) k_band_mv(BandMvArgs a) {
  extern __shared__ unsigned bm_act[];  // (nS,) active-lag bits of each S-tile
  for (int i = threadIdx.x; i < a.nS; i += blockDim.x) bm_act[i] = __ldg(a.s_act + i);
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int J = blockIdx.x / a.P, part = blockIdx.x % a.P;
  const int g = lane >> 2, k = lane & 3;
  const int t0 = w * TT;
  double acc[TT][2];
#pragma unroll
  for (int u = 0; u < TT; ++u) acc[u][0] = acc[u][1] = 0.0;
  const long long r0 = __ldg(a.rbptr + J), r1 = __ldg(a.rbptr + J + 1);
  const long long q0 = r0 + (r1 - r0) * part / a.P, q1 = r0 + (r1 - r0) * (part + 1) / a.P;
  const double* xl = a.xt + (a.off0 - k + g + 8 * t0);
  const unsigned kbit = 1u << k;
  for (long long pb = q0; pb < q1; pb += 32) {
    const int n = (int)min(32LL, q1 - pb);
    int my_l = 0, my_S = 0;
    unsigned my_act = 0u;
    if (lane < n) {
      my_l = __ldg(a.col + pb + lane);
      my_S = __ldg(a.stile + pb + lane);
      my_act = bm_act[my_S];
    }
    unsigned live = __ballot_sync(0xffffffffu, my_act != 0u);
    while (live) {
      const int i1 = __ffs(live) - 1;
      live &= live - 1;
      const int i2 = live ? __ffs(live) - 1 : -1;
      if (i2 >= 0) live &= live - 1;
      const int l1 = __shfl_sync(0xffffffffu, my_l, i1), S1 = __shfl_sync(0xffffffffu, my_S, i1);
      const unsigned c1 = __shfl_sync(0xffffffffu, my_act, i1);
      const int l2 = __shfl_sync(0xffffffffu, my_l, i2 < 0 ? i1 : i2);
      const int S2 = __shfl_sync(0xffffffffu, my_S, i2 < 0 ? i1 : i2);
      const unsigned c2 = __shfl_sync(0xffffffffu, my_act, i2 < 0 ? i1 : i2);
      double av1 = __ldg(a.val + (pb + i1) * 32 + lane);
      double av2 = i2 >= 0 ? __ldg(a.val + (pb + i2) * 32 + lane) : 0.0;
      const double* x1 = xl + (long long)l1 * a.xs - 4 * S1;
      const double* x2 = xl + (long long)l2 * a.xs - 4 * S2;
      double b1[TT], b2[TT];
#pragma unroll
      for (int u = 0; u < TT; ++u) {
        b1[u] = __ldg(x1 + 8 * u);
        b2[u] = __ldg(x2 + 8 * u);
      }
      if (!(c1 & kbit)) av1 = 0.0;
      if (i2 < 0 || !(c2 & kbit)) av2 = 0.0;
#pragma unroll
      for (int u = 0; u < TT; ++u) dmma884(acc[u][0], acc[u][1], av1, b1[u]);
#pragma unroll
      for (int u = 0; u < TT; ++u) dmma884(acc[u][0], acc[u][1], av2, b2[u]);
    }
  }
  // partial tile rows of this part: ypart[part][8 J + g][8 (t0 + u) + 2 k + {0, 1}]
  double* yp = a.ypart + ((long long)part * a.nRB * 8 + 8LL * J + g) * a.ldy + 8 * t0 + 2 * k;
#pragma unroll
  for (int u = 0; u < TT; ++u)
    if (t0 + u < a.nT) *reinterpret_cast<double2*>(yp + 8 * u) = make_double2(acc[u][0], acc[u][1]);
}

// y[(kt - rlo) nrows + j] += sum over parts (in part order) for kt in the band rows
__global__ void k_band_reduce(BandMvArgs a) {
  const long long total = (long long)a.nrows * a.nkt;
  const long long pstride = (long long)a.nRB * 8 * a.ldy;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int jp = (int)(idx / a.nkt), c = (int)(idx % a.nkt);
    const double* src = a.ypart + (long long)jp * a.ldy + c;
    double s = 0.0;
    for (int q = 0; q < a.P; ++q) s += __ldcg(src + q * pstride);
    a.y[(long long)(a.ktlo - a.rlo + c) * a.nrows + __ldg(a.rperm + jp)] += s;
  }
}

template <int TT>
int launch_tt(const BandMvArgs& a, cudaStream_t st) {
  const size_t smem = (size_t)a.nS * sizeof(unsigned);
  k_band_mv<TT><<<(unsigned)((long long)a.nRB * a.P), a.W * 32, smem, st>>>(a);
  TDB_CUDA_CHECK(cudaGetLastError());
  return TDB_OK;
}

}  // namespace

int band_build(TdbSystem* sys, int f) {
  if ((int)sys->band.size() != sys->F) sys->band.assign(sys->F, BandStore{});
  BandStore& b = sys->band[f];
  if (b.built) return TDB_OK;
  if (b.failed) {
    set_error("band tiles: an earlier build of this family failed");
    return TDB_E_NOMEM;
  }
  TDB_REQUIRE(sys->p == 0, "band tiles: built for p = 0 only");
  cudaStream_t st = sys->ctx->stream;
  const int NR = sys->nrows, nRB = sys->nRB, V = (int)sys->V;
  FamilyStore& fs = sys->fam[f];
  const int nS = (fs.npos + 3) / 4;
  const long long n = fs.nnz;
  unsigned long long *k0 = nullptr, *k1 = nullptr;
  long long *i0 = nullptr, *i1 = nullptr;
  int *head = nullptr, *tile_rb = nullptr;
  void* tmp = nullptr;
  auto release = [&]() {
    dev_free(k0);
    dev_free(k1);
    dev_free(i0);
    dev_free(i1);
    dev_free(head);
    dev_free(tile_rb);
    dev_free(tmp);
  };
  auto fail = [&](cudaError_t e) {
    release();
    dev_free(b.rbptr);
    dev_free(b.col);
    dev_free(b.stile);
    dev_free(b.val);
    b.rbptr = nullptr;
    b.col = b.stile = nullptr;
    b.val = nullptr;
    b.failed = true;  // sticky: later plans go straight to CSR
    set_error(std::string("band tiles build: ") + cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? TDB_E_NOMEM : TDB_E_CUDA;
  };
#define TRY(expr)                       \
  do {                                  \
    cudaError_t e_ = (expr);            \
    if (e_ != cudaSuccess) return fail(e_); \
  } while (0)
  TRY(dev_malloc((void**)&b.rbptr, (size_t)(nRB + 1) * sizeof(int64_t)));
  b.nS = nS;
  if (n == 0) {
    TRY(cudaMemsetAsync(b.rbptr, 0, (size_t)(nRB + 1) * sizeof(int64_t), st));
    TRY(dev_malloc((void**)&b.col, sizeof(int32_t)));
    TRY(dev_malloc((void**)&b.stile, sizeof(int32_t)));
    TRY(dev_malloc((void**)&b.val, 32 * sizeof(double)));
    TRY(cudaStreamSynchronize(st));
    b.built = true;
    return TDB_OK;
  }
  TRY(dev_malloc((void**)&k0, n * sizeof(unsigned long long)));
  TRY(dev_malloc((void**)&k1, n * sizeof(unsigned long long)));
  TRY(dev_malloc((void**)&i0, n * sizeof(long long)));
  TRY(dev_malloc((void**)&i1, n * sizeof(long long)));
  TRY(dev_malloc((void**)&head, n * sizeof(int)));
  k_band_keys<<<148 * 16, 256, 0, st>>>(fs.indptr, fs.indices, (long long)fs.npos * NR, NR, V, nS, sys->d_rinv,
                                        k0, i0);
  TRY(cudaGetLastError());
  int end_bit = 5;
  {
    const unsigned long long maxkey = (unsigned long long)nRB * (unsigned long long)V * (unsigned long long)nS;
    while (end_bit < 64 && (maxkey >> (end_bit - 5)) != 0) ++end_bit;
  }
  size_t tb = 0, tb2 = 0;
  TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb, k0, k1, i0, i1, n, 0, end_bit, st));
  TRY(cub::DeviceScan::InclusiveSum(nullptr, tb2, head, head, n, st));
  TRY(dev_malloc(&tmp, std::max(tb, tb2)));
  TRY(cub::DeviceRadixSort::SortPairs(tmp, tb, k0, k1, i0, i1, n, 0, end_bit, st));
  k_band_heads<<<148 * 16, 256, 0, st>>>(k1, n, head);
  TRY(cudaGetLastError());
  TRY(cub::DeviceScan::InclusiveSum(tmp, tb2, head, head, n, st));
  int nt = 0;
  TRY(cudaMemcpyAsync(&nt, head + n - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  TRY(cudaStreamSynchronize(st));
  b.ntiles = nt;
  b.nnz = n;
  TRY(dev_malloc((void**)&b.col, (size_t)nt * sizeof(int32_t)));
  TRY(dev_malloc((void**)&b.stile, (size_t)nt * sizeof(int32_t)));
  TRY(dev_malloc((void**)&b.val, (size_t)nt * 32 * sizeof(double)));
  TRY(dev_malloc((void**)&tile_rb, (size_t)nt * sizeof(int)));
  TRY(cudaMemsetAsync(b.val, 0, (size_t)nt * 32 * sizeof(double), st));
  k_band_fill<<<148 * 16, 256, 0, st>>>(k1, i1, head, n, V, nS, fs.data, b.col, b.stile, b.val, tile_rb);
  TRY(cudaGetLastError());
  k_band_rbptr<<<(nRB + 256) / 256, 256, 0, st>>>(tile_rb, nt, nRB, b.rbptr);
  TRY(cudaGetLastError());
  TRY(cudaStreamSynchronize(st));
  release();
#undef TRY
  b.built = true;
  return TDB_OK;
}

int band_mv_tiles(const BandMvArgs& a, cudaStream_t st) {
  switch (a.TT) {
    case 1: return launch_tt<1>(a, st);
    case 2: return launch_tt<2>(a, st);
    case 3: return launch_tt<3>(a, st);
    case 4: return launch_tt<4>(a, st);
    case 5: return launch_tt<5>(a, st);
    default: return launch_tt<6>(a, st);
  }
}

int band_mv_reduce(const BandMvArgs& a, cudaStream_t st) {
  const long long total = (long long)a.nrows * a.nkt;
  k_band_reduce<<<(unsigned)std::max<long long>(1, std::min<long long>((total + 255) / 256, 148 * 8)), 256, 0, st>>>(a);
  TDB_CUDA_CHECK(cudaGetLastError());
  return TDB_OK;
}

}  // namespace tdb
