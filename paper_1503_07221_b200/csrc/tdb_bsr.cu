// Tensor-core (FP64 DMMA) block-Toeplitz matvec for p = 0.
//
// Replaces the inner loop of BlockHessenbergMatrix.matvec (/root/reference/pkg/
// src/tdbem/block_system.py:197-215: per logical block position, y_kt += A_k x_it
// with a SciPy CSR SpMV).  Every stored lag block A_t is applied to all block
// rows kt that reuse it at once, as a sparse x dense product
//     Y[j][kt] += sum_l A_t[j][l] X[l][kt - d_t]       (kt in the term's mask)
// i.e. a batched dense contraction: A_t is kept as 8 x 4 tiles (dofs in Morton
// order, ~50% of tile slots non-zero, tools/fill_probe.py) and each tile is the
// A operand of `mma.sync.m8n8k4.f64` against an 8-time-step panel of X (the B
// operand, 4 vertices x 8 block columns), accumulating an 8 x 8 tile of Y in
// registers.  One A tile load serves all time panels of the warp (8 per warp).
//
// Fragments (PTX ISA, mma.m8n8k4 .f64): A[g][t] and B[t][g] with g = lane >> 2,
// t = lane & 3; D holds Y[g][2t], Y[g][2t+1].
//
// Work: CTA = (row block rb, time-tile group kg) with kBsrWarps warps; warp w
// takes every kBsrWarps-th tile of every term (balanced, fixed), UNR tiles' A/B
// loads in flight per step; the warps' partial tiles are summed through shared
// memory in warp order (deterministic).
//
// Status: opt-in (TDB_MV_BSR=1).  Parity-tested, DMMA runs at the FP64 peak in
// isolation (tools/micro/dmma_bench.cu: 37 TFLOP/s), but the per-tile B gathers
// from L2 leave this kernel 1.4-2.2x slower than the CSR lanes-over-time kernel
// (tdb_matvec.cu) on configs 2 and 4, so CSR is the default.
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "tdb_bsr.h"
#include "tdb_common.cuh"
#include "tdb_internal.h"

namespace tdb {

namespace {

// ---- BSR build: CSR rows (s, jl) -> sorted (s, rb, cb, sub) keys -> tiles ----
__global__ void k_bsr_keys(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                           long long nrows_total, int nrows, const int* __restrict__ rinv,
                           const int* __restrict__ vinv, int nRB, int nCB, unsigned long long* __restrict__ keys,
                           long long* __restrict__ ids) {
  const int lane = threadIdx.x & 31;
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long row = warp; row < nrows_total; row += nw) {
    const long long s = row / nrows;
    const int jl = (int)(row % nrows);
    const int jp = rinv[jl];
    const unsigned long long rbkey = (unsigned long long)(s * nRB + (jp >> 3)) * (unsigned long long)nCB;
    const int64_t e0 = indptr[row], e1 = indptr[row + 1];
    for (int64_t e = e0 + lane; e < e1; e += 32) {
      const int lp = vinv[indices[e]];
      const unsigned sub = (unsigned)((jp & 7) * 4 + (lp & 3));
      keys[e] = ((rbkey + (unsigned)(lp >> 2)) << 5) | sub;
      ids[e] = e;
    }
  }
}

__global__ void k_bsr_heads(const unsigned long long* __restrict__ keys, long long n, int* __restrict__ head) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    head[i] = (i == 0 || (keys[i] >> 5) != (keys[i - 1] >> 5)) ? 1 : 0;
}

// tid[i] = inclusive scan of heads - 1
__global__ void k_bsr_fill(const unsigned long long* __restrict__ keys, const long long* __restrict__ ids,
                           const int* __restrict__ tid_incl, long long n, int nCB, const double* __restrict__ data,
                           int32_t* __restrict__ col, double* __restrict__ val,
                           unsigned long long* __restrict__ tile_rb) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long t = tid_incl[i] - 1;
    const unsigned long long k = keys[i] >> 5;
    val[t * 32 + (keys[i] & 31u)] = data[ids[i]];
    if (i == 0 || (keys[i - 1] >> 5) != k) {
      col[t] = (int32_t)(k % (unsigned long long)nCB);
      tile_rb[t] = k / (unsigned long long)nCB;
    }
  }
}

// rbptr[k] = first tile whose (position, row block) key is >= k
__global__ void k_bsr_rbptr(const unsigned long long* __restrict__ tile_rb, long long ntiles, long long nkeys,
                            int64_t* __restrict__ rbptr) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k <= nkeys; k += (long long)gridDim.x * blockDim.x) {
    long long lo = 0, hi = ntiles;
    while (lo < hi) {
      const long long mid = (lo + hi) >> 1;
      if (tile_rb[mid] < (unsigned long long)k) lo = mid + 1; else hi = mid;
    }
    rbptr[k] = lo;
  }
}

}  // namespace

int bsr_build(TdbSystem* sys) {
  if (sys->bsr_built) return TDB_OK;
  cudaStream_t st = sys->ctx->stream;
  TDB_REQUIRE(sys->p == 0, "bsr: tensor-core storage is built for p = 0 only");
  const int NR = sys->nrows, nRB = sys->nRB, nCB = sys->nCB;
  sys->bsr.assign(sys->F, BsrStore{});
  for (int f = 0; f < sys->F; ++f) {
    FamilyStore& fs = sys->fam[f];
    BsrStore& b = sys->bsr[f];
    const long long n = fs.nnz;
    const long long nkeys = (long long)fs.npos * nRB;
    TDB_CUDA_CHECK(cudaMalloc(&b.rbptr, (nkeys + 1) * sizeof(int64_t)));
    if (n == 0) {
      TDB_CUDA_CHECK(cudaMemsetAsync(b.rbptr, 0, (nkeys + 1) * sizeof(int64_t), st));
      TDB_CUDA_CHECK(cudaMalloc(&b.col, sizeof(int32_t)));
      TDB_CUDA_CHECK(cudaMalloc(&b.val, 32 * sizeof(double)));
      continue;
    }
    unsigned long long *k0 = nullptr, *k1 = nullptr, *tile_rb = nullptr;
    long long *i0 = nullptr, *i1 = nullptr;
    int* head = nullptr;
    void* tmp = nullptr;
    size_t tb = 0, tb2 = 0;
    auto release = [&]() {
      cudaFree(k0);
      cudaFree(k1);
      cudaFree(i0);
      cudaFree(i1);
      cudaFree(head);
      cudaFree(tmp);
      cudaFree(tile_rb);
    };
#define TRY(expr)                                                  \
  do {                                                             \
    cudaError_t e_ = (expr);                                       \
    if (e_ != cudaSuccess) {                                       \
      release();                                                   \
      set_error(std::string("bsr build: ") + cudaGetErrorString(e_)); \
      return e_ == cudaErrorMemoryAllocation ? TDB_E_NOMEM : TDB_E_CUDA; \
    }                                                              \
  } while (0)
    TRY(cudaMalloc(&k0, n * sizeof(unsigned long long)));
    TRY(cudaMalloc(&k1, n * sizeof(unsigned long long)));
    TRY(cudaMalloc(&i0, n * sizeof(long long)));
    TRY(cudaMalloc(&i1, n * sizeof(long long)));
    TRY(cudaMalloc(&head, n * sizeof(int)));
    const long long rows_total = (long long)fs.npos * NR;
    k_bsr_keys<<<148 * 16, 256, 0, st>>>(fs.indptr, fs.indices, rows_total, NR, sys->d_rinv, sys->d_vinv, nRB, nCB,
                                         k0, i0);
    TRY(cudaGetLastError());
    int end_bit = 5;
    {
      const unsigned long long maxkey = (unsigned long long)nkeys * (unsigned long long)nCB;
      while (end_bit < 64 && (maxkey >> (end_bit - 5)) != 0) ++end_bit;
    }
    TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb, k0, k1, i0, i1, n, 0, end_bit, st));
    TRY(cub::DeviceScan::InclusiveSum(nullptr, tb2, head, head, n, st));
    TRY(cudaMalloc(&tmp, std::max(tb, tb2)));
    TRY(cub::DeviceRadixSort::SortPairs(tmp, tb, k0, k1, i0, i1, n, 0, end_bit, st));
    k_bsr_heads<<<148 * 16, 256, 0, st>>>(k1, n, head);
    TRY(cudaGetLastError());
    TRY(cub::DeviceScan::InclusiveSum(tmp, tb2, head, head, n, st));
    int nt = 0;
    TRY(cudaMemcpyAsync(&nt, head + n - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
    TRY(cudaStreamSynchronize(st));
    b.ntiles = nt;
    TRY(cudaMalloc(&b.col, (size_t)nt * sizeof(int32_t)));
    TRY(cudaMalloc(&b.val, (size_t)nt * 32 * sizeof(double)));
    TRY(cudaMalloc(&tile_rb, (size_t)nt * sizeof(unsigned long long)));
    TRY(cudaMemsetAsync(b.val, 0, (size_t)nt * 32 * sizeof(double), st));
    k_bsr_fill<<<148 * 16, 256, 0, st>>>(k1, i1, head, n, nCB, fs.data, b.col, b.val, tile_rb);
    TRY(cudaGetLastError());
    k_bsr_rbptr<<<(int)std::min<long long>((nkeys + 256) / 256, 148 * 16), 256, 0, st>>>(tile_rb, nt, nkeys, b.rbptr);
    TRY(cudaGetLastError());
    TRY(cudaStreamSynchronize(st));
    release();
#undef TRY
  }
  sys->bsr_built = true;
  return TDB_OK;
}

// ---- DMMA matvec ----------------------------------------------------------
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// CTA = (row block rb, time-tile group kg); warp w = term group w (kBsrWarps groups),
// T 8-time tiles per warp.  The group partials are summed through shared memory
// in warp order (deterministic) and written to y (reference layout).
template <int T>
__global__ void __launch_bounds__(kBsrWarps * 32, 2) k_bsr_mv(BsrMvArgs a) {
  extern __shared__ double red[];  // [kBsrWarps][T][64]
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int gq = lane >> 2, tq = lane & 3;  // fragment row / column group
  const int rb = blockIdx.x % a.nRB, kg = blockIdx.x / a.nRB;
  const int tile0 = kg * T;  // first 8-time tile of this CTA
  double acc[T][2];
#pragma unroll
  for (int u = 0; u < T; ++u) acc[u][0] = acc[u][1] = 0.0;
  // every warp takes every kBsrWarps-th tile of every term: balanced and fixed
  const int nterms = __ldg(a.group_begin + kBsrWarps);
  for (int t = 0; t < nterms; ++t) {
    const int f = __ldg(a.term_f + t), s = __ldg(a.term_s + t), d = __ldg(a.term_d + t);
    const BsrFam fam = a.fam[f];
    const long long rk = (long long)s * a.nRB + rb;
    const long long p0 = __ldg(fam.rbptr + rk) + wid, p1 = __ldg(fam.rbptr + rk + 1);
    if (p0 >= p1) continue;
    // this lane's B column n = gq: block row kt = rlo + 8 (tile0 + u) + gq
    const unsigned* mask = a.term_mask + (long long)t * a.words;
    int off[T];
    unsigned act = 0u;
#pragma unroll
    for (int u = 0; u < T; ++u) {
      const int r = 8 * (tile0 + u) + gq;
      const int kt = a.rlo + r;
      bool ok = r < a.nr;
      if (ok) ok = (__ldg(mask + ((kt - 1) >> 5)) >> ((kt - 1) & 31)) & 1u;
      off[u] = ok ? (kt - d - a.clo) : a.nc;  // column nc of Xp is a zero pad
      if (__any_sync(0xffffffffu, ok)) act |= 1u << u;
    }
    if (act == 0u) continue;
    const double* __restrict__ xp = a.xp + (long long)tq * a.xs;
    constexpr int W = kBsrWarps;
    for (long long pb = p0; pb < p1; pb += 32 * W) {
      const int n = (int)min(32LL, (p1 - pb + W - 1) / W);
      // column blocks of this warp's next <= 32 tiles: one load, broadcast by shuffle
      const int my_cb = lane < n ? __ldg(fam.col + pb + (long long)W * lane) : 0;
      // UNR tiles per step: all their A and B loads are issued before any DMMA
      constexpr int UNR = T >= 8 ? 2 : (T >= 4 ? 4 : 8);
      for (int i0 = 0; i0 < n; i0 += UNR) {
        double av[UNR], bv[UNR][T];
#pragma unroll
        for (int k = 0; k < UNR; ++k) {
          const bool ok = i0 + k < n;
          const long long p = pb + (long long)W * (ok ? i0 + k : i0);
          av[k] = ok ? __ldg(fam.val + p * 32 + lane) : 0.0;
          const long long rowo = (long long)__shfl_sync(0xffffffffu, my_cb, ok ? i0 + k : i0) * 4 * a.xs;
#pragma unroll
          for (int u = 0; u < T; ++u) bv[k][u] = ((act >> u) & 1u) ? __ldg(xp + rowo + off[u]) : 0.0;
        }
#pragma unroll
        for (int k = 0; k < UNR; ++k)
#pragma unroll
          for (int u = 0; u < T; ++u)
            if ((act >> u) & 1u) dmma884(acc[u][0], acc[u][1], av[k], bv[k][u]);
      }
    }
  }
#pragma unroll
  for (int u = 0; u < T; ++u) {
    red[(wid * T + u) * 64 + 2 * lane] = acc[u][0];
    red[(wid * T + u) * 64 + 2 * lane + 1] = acc[u][1];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < T * 64; e += blockDim.x) {
    double sum = 0.0;
#pragma unroll
    for (int ww = 0; ww < kBsrWarps; ++ww) sum += red[ww * T * 64 + e];
    const int u = e >> 6, q = e & 63, ln = q >> 1, i = q & 1;
    const int jp = 8 * rb + (ln >> 2);
    const int r = 8 * (tile0 + u) + 2 * (ln & 3) + i;
    if (jp < a.nrows && r < a.nr) a.y[(long long)r * a.nrows + __ldg(a.rperm + jp)] = sum;
  }
}

int bsr_mv_launch(const BsrMvArgs& a, cudaStream_t st) {
  const unsigned ctas = (unsigned)((long long)a.nRB * a.KG);
  switch (a.T) {
    case 1: k_bsr_mv<1><<<ctas, kBsrWarps * 32, (size_t)kBsrWarps * 1 * 64 * 8, st>>>(a); break;
    case 2: k_bsr_mv<2><<<ctas, kBsrWarps * 32, (size_t)kBsrWarps * 2 * 64 * 8, st>>>(a); break;
    case 4: k_bsr_mv<4><<<ctas, kBsrWarps * 32, (size_t)kBsrWarps * 4 * 64 * 8, st>>>(a); break;
    default: k_bsr_mv<8><<<ctas, kBsrWarps * 32, (size_t)kBsrWarps * 8 * 64 * 8, st>>>(a); break;
  }
  TDB_CUDA_CHECK(cudaGetLastError());
  return TDB_OK;
}

}  // namespace tdb
