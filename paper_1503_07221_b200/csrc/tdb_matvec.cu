// Block Hessenberg / block Toeplitz matvec on device-resident canonical blocks.
//
// Replaces BlockHessenbergMatrix.matvec (/root/reference/pkg/src/tdbem/
// block_system.py:180-216): y = A[rows, cols] x over the logical block
// positions, each resolved to its canonical stored block (canonical_position
// :54-66) with the structural zero test (:153-160) applied per logical
// position by the caller-provided term masks.
//
// Layout trick: the time axis is the long axis.  Vectors are transposed to
// "vertex-major" xt[l][time] so that one stored entry (j, l, v) of a lag block
// multiplies a contiguous strip x[l][kt - d] over all logical kt of that lag:
// a warp owns test vertex j, lanes own block rows kt (lane + 32 c), and each
// stored entry is read ONCE per matvec (broadcast), however many logical
// positions reuse it (Toeplitz SpMM, intensity ~ N/6 flop/B).  Positions are
// split into G groups (partial outputs, summed in fixed order) only to give
// the grid enough warps on small meshes.

#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "tdb_common.cuh"
#include "tdb_internal.h"

namespace tdb {

constexpr int kMaxRowChunks = 12;  // rows per plan <= 12 * 32 = 384 block rows

struct FamCsr {
  const int64_t* indptr;
  const int32_t* indices;
  const double* data;
};

struct MvArgs {
  int M, NP1, NM;
  int nrows;                // owned test-vertex rows (warps per group)
  int rlo, nr, clo, nc;     // block ranges
  int words;
  int G;
  const FamCsr* fam;
  const int* term_f;
  const int* term_s;
  const int* term_d;
  const unsigned* term_mask;
  const int* group_begin;   // (G+1,) term ranges
  const double* xt;         // [M][nc*NP1]
  double* ypart;            // [G][M][nr*NP1]
};

__global__ void k_transpose_in(const double* __restrict__ x, double* __restrict__ xt, int M,
                               int ncols, const long long* __restrict__ xmap, long long xstride) {
  // x[xmap[l] + c*xstride] -> xt[l*ncols + c], c = (block col)*NP1 + m1
  __shared__ double tile[32][33];
  const int c0 = blockIdx.y * 32, l0 = blockIdx.x * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int c = c0 + k, l = l0 + threadIdx.x;
    if (c < ncols && l < M)
      tile[k][threadIdx.x] = x[(xmap ? xmap[l] : (long long)l) + (long long)c * xstride];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int l = l0 + k, c = c0 + threadIdx.x;
    if (c < ncols && l < M) xt[(long long)l * ncols + c] = tile[threadIdx.x][k];
  }
}

template <int NP1>
__global__ void __launch_bounds__(256) k_matvec(MvArgs a) {
  constexpr int NM = NP1 * NP1;
  const int lane = threadIdx.x & 31;
  const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  if (w >= (long long)a.nrows * a.G) return;
  const int j = (int)(w % a.nrows), g = (int)(w / a.nrows);  // j = local row
  const int ncol = a.nc * NP1;
  double acc[kMaxRowChunks][NP1];
#pragma unroll
  for (int c = 0; c < kMaxRowChunks; ++c)
#pragma unroll
    for (int m = 0; m < NP1; ++m) acc[c][m] = 0.0;
  const int nchunks = (a.nr + 31) >> 5;
  for (int t = a.group_begin[g]; t < a.group_begin[g + 1]; ++t) {
    const FamCsr fc = a.fam[a.term_f[t]];
    const int s = a.term_s[t], d = a.term_d[t];
    const unsigned* mask = a.term_mask + (long long)t * a.words;
    // lane validity per row chunk (bit kt-1)
    unsigned valid = 0;
#pragma unroll
    for (int c = 0; c < kMaxRowChunks; ++c) {
      if (c < nchunks) {
        const int kt = a.rlo + lane + 32 * c;
        const bool v = (lane + 32 * c < a.nr) && ((mask[(kt - 1) >> 5] >> ((kt - 1) & 31)) & 1u);
        valid |= (v ? 1u : 0u) << c;
      }
    }
    if (__ballot_sync(0xffffffffu, valid != 0) == 0) continue;
    const long long row = (long long)s * a.nrows + j;
    const int64_t e0 = fc.indptr[row], e1 = fc.indptr[row + 1];
    for (int64_t e = e0; e < e1; ++e) {
      const int l = fc.indices[e];
      double v[NM];
#pragma unroll
      for (int m = 0; m < NM; ++m) v[m] = fc.data[e * NM + m];
      const double* xl = a.xt + (long long)l * ncol;
#pragma unroll
      for (int c = 0; c < kMaxRowChunks; ++c) {
        if ((valid >> c) & 1u) {
          const int kt = a.rlo + lane + 32 * c;
          const double* xv = xl + (kt - d - a.clo) * NP1;
#pragma unroll
          for (int m1 = 0; m1 < NP1; ++m1) {
            const double xm = xv[m1];
#pragma unroll
            for (int m2 = 0; m2 < NP1; ++m2) acc[c][m2] = fma(v[m2 * NP1 + m1], xm, acc[c][m2]);
          }
        }
      }
    }
  }
  double* yp = a.ypart + ((long long)g * a.nrows + j) * (a.nr * NP1);
#pragma unroll
  for (int c = 0; c < kMaxRowChunks; ++c) {
    const int r = lane + 32 * c;
    if (c < nchunks && r < a.nr)
#pragma unroll
      for (int m = 0; m < NP1; ++m) yp[r * NP1 + m] = acc[c][m];
  }
}

__global__ void k_reduce_out(const double* __restrict__ ypart, double* __restrict__ y, int M, int nrow,
                             int G) {
  // y[c*M + j] = sum_g ypart[g][j][c]; c = (block row)*NP1 + m2
  __shared__ double tile[32][33];
  const int c0 = blockIdx.y * 32, j0 = blockIdx.x * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int j = j0 + k, c = c0 + threadIdx.x;
    double s = 0.0;
    if (j < M && c < nrow)
      for (int g = 0; g < G; ++g) s += ypart[((long long)g * M + j) * nrow + c];
    tile[k][threadIdx.x] = s;
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int c = c0 + k, j = j0 + threadIdx.x;
    if (j < M && c < nrow) y[(long long)c * M + j] = tile[threadIdx.x][k];
  }
}

}  // namespace tdb

using namespace tdb;

struct TdbMatvecPlan {
  TdbSystem* sys = nullptr;
  MvArgs args{};
  long long* d_xmap = nullptr;
  long long xstride = 0;
  FamCsr* d_fam = nullptr;
  int* d_ints = nullptr;       // term_f, term_s, term_d, group_begin
  unsigned* d_mask = nullptr;
  double* d_xt = nullptr;
  double* d_ypart = nullptr;
  double bytes = 0.0, flops = 0.0;
};

extern "C" int tdb_matvec_plan_destroy(TdbMatvecPlan* p) {
  if (!p) return TDB_OK;
  cudaFree(p->d_fam);
  cudaFree(p->d_ints);
  cudaFree(p->d_mask);
  cudaFree(p->d_xt);
  cudaFree(p->d_ypart);
  cudaFree(p->d_xmap);
  delete p;
  return TDB_OK;
}

extern "C" int tdb_matvec_plan_create(TdbSystem* sys, const TdbMatvecDesc* d, TdbMatvecPlan** out) {
  TDB_REQUIRE(sys && d && out, "NULL argument");
  TDB_REQUIRE(d->rlo >= 1 && d->rhi >= d->rlo && d->rhi <= d->N, "bad row range");
  TDB_REQUIRE(d->clo >= 1 && d->chi >= d->clo && d->chi <= d->N, "bad column range");
  TDB_REQUIRE(d->rhi - d->rlo + 1 <= kMaxRowChunks * 32, "matvec: more than 384 block rows");
  TDB_REQUIRE(d->words == (d->N + 31) / 32, "matvec: words must be ceil(N/32)");
  TDB_REQUIRE(d->nterms >= 0, "negative term count");
  TDB_CUDA_CHECK(cudaSetDevice(sys->ctx->device));
  const int M = (int)sys->V, NP1 = sys->np1, NM = sys->nm, NR = sys->nrows;
  TdbMatvecPlan* p = new TdbMatvecPlan();
  p->sys = sys;
  const int nt = d->nterms;
  // work per term, for grouping and for the roofline bookkeeping
  std::vector<long long> tnnz(nt);
  std::vector<std::vector<int64_t>> famptr(sys->F);
  double bytes = 0.0, flops = 0.0;
  for (int t = 0; t < nt; ++t) {
    const int f = d->term_family[t], s = d->term_pos[t];
    if (f < 0 || f >= sys->F || s < 0 || s >= sys->fam[f].npos) {
      delete p;
      set_error("matvec: term references a missing family/position");
      return TDB_E_INVALID;
    }
    int64_t b[2];
    cudaMemcpy(b, sys->fam[f].indptr + (long long)s * NR, sizeof(int64_t), cudaMemcpyDeviceToHost);
    cudaMemcpy(b + 1, sys->fam[f].indptr + (long long)(s + 1) * NR, sizeof(int64_t), cudaMemcpyDeviceToHost);
    tnnz[t] = b[1] - b[0];
    int nlog = 0;
    for (int w = 0; w < d->words; ++w) nlog += __builtin_popcount(d->term_mask[(long long)t * d->words + w]);
    bytes += (double)tnnz[t] * (8.0 * NM + 4.0);
    flops += 2.0 * NM * (double)tnnz[t] * nlog;
  }
  const int nr = d->rhi - d->rlo + 1, nc = d->chi - d->clo + 1;
  bytes += 8.0 * ((double)nr * NR + (double)nc * M) * NP1;
  p->bytes = bytes;
  p->flops = flops;
  // groups: enough warps to fill the chip on small meshes
  const int want_warps = sys->ctx->num_sms * 32;
  int G = std::max(1, std::min(nt, (want_warps + NR - 1) / NR));
  G = std::min(G, 64);
  std::vector<int> gb(G + 1, nt);
  {
    long long total = 0;
    for (long long v : tnnz) total += v;
    long long acc = 0;
    int g = 0;
    gb[0] = 0;
    for (int t = 0; t < nt && g < G - 1; ++t) {
      acc += tnnz[t];
      if (acc * G >= total * (g + 1)) gb[++g] = t + 1;
    }
    for (int k = g + 1; k <= G; ++k) gb[k] = nt;
  }
  std::vector<FamCsr> fam(sys->F);
  for (int f = 0; f < sys->F; ++f) fam[f] = {sys->fam[f].indptr, sys->fam[f].indices, sys->fam[f].data};
  std::vector<int> ints;
  ints.insert(ints.end(), d->term_family, d->term_family + nt);
  ints.insert(ints.end(), d->term_pos, d->term_pos + nt);
  ints.insert(ints.end(), d->term_d, d->term_d + nt);
  ints.insert(ints.end(), gb.begin(), gb.end());
  cudaStream_t st = sys->ctx->stream;
#define ALLOC_COPY(dst, src, n, T)                                                                 \
  do {                                                                                             \
    size_t nn = std::max<size_t>(1, (size_t)(n));                                                  \
    if (cudaMalloc((void**)&(dst), nn * sizeof(T)) != cudaSuccess) {                              \
      tdb_matvec_plan_destroy(p);                                                                  \
      set_error("matvec plan: cudaMalloc failed");                                                 \
      return TDB_E_NOMEM;                                                                          \
    }                                                                                              \
    if ((n) > 0 && (src) != nullptr)                                                               \
      cudaMemcpyAsync((dst), (src), (size_t)(n) * sizeof(T), cudaMemcpyHostToDevice, st);          \
  } while (0)
  ALLOC_COPY(p->d_fam, fam.data(), sys->F, FamCsr);
  ALLOC_COPY(p->d_ints, ints.data(), ints.size(), int);
  ALLOC_COPY(p->d_mask, d->term_mask, (size_t)nt * d->words, unsigned);
  ALLOC_COPY(p->d_xt, (const double*)nullptr, (size_t)M * nc * NP1, double);
  ALLOC_COPY(p->d_ypart, (const double*)nullptr, (size_t)G * NR * nr * NP1, double);
  if (d->x_map) ALLOC_COPY(p->d_xmap, reinterpret_cast<const long long*>(d->x_map), M, long long);
  p->xstride = d->x_map ? d->x_stride : M;
#undef ALLOC_COPY
  TDB_CUDA_CHECK(cudaStreamSynchronize(st));
  MvArgs& a = p->args;
  a.M = M;
  a.nrows = NR;
  a.NP1 = NP1;
  a.NM = NM;
  a.rlo = d->rlo;
  a.nr = nr;
  a.clo = d->clo;
  a.nc = nc;
  a.words = d->words;
  a.G = G;
  a.fam = p->d_fam;
  a.term_f = p->d_ints;
  a.term_s = p->d_ints + nt;
  a.term_d = p->d_ints + 2 * nt;
  a.group_begin = p->d_ints + 3 * nt;
  a.term_mask = p->d_mask;
  a.xt = p->d_xt;
  a.ypart = p->d_ypart;
  *out = p;
  return TDB_OK;
}

extern "C" int tdb_matvec_plan_work(const TdbMatvecPlan* p, double* bytes, double* flops) {
  TDB_REQUIRE(p != nullptr, "NULL plan");
  if (bytes) *bytes = p->bytes;
  if (flops) *flops = p->flops;
  return TDB_OK;
}

extern "C" int tdb_matvec(TdbMatvecPlan* p, const double* x, double* y) {
  TDB_REQUIRE(p && x && y, "NULL argument");
  const MvArgs& a = p->args;
  cudaStream_t st = p->sys->ctx->stream;
  const int ncols = a.nc * a.NP1, nrows = a.nr * a.NP1;
  {
    dim3 blk(32, 8), grd((a.M + 31) / 32, (ncols + 31) / 32);
    k_transpose_in<<<grd, blk, 0, st>>>(x, p->d_xt, a.M, ncols, p->d_xmap, p->xstride);
  }
  {
    const long long warps = (long long)a.nrows * a.G;
    const int blocks = (int)((warps * 32 + 255) / 256);
    switch (a.NP1) {
      case 1: k_matvec<1><<<blocks, 256, 0, st>>>(a); break;
      case 2: k_matvec<2><<<blocks, 256, 0, st>>>(a); break;
      case 3: k_matvec<3><<<blocks, 256, 0, st>>>(a); break;
      default: k_matvec<4><<<blocks, 256, 0, st>>>(a); break;
    }
  }
  {
    dim3 blk(32, 8), grd((a.nrows + 31) / 32, (nrows + 31) / 32);
    k_reduce_out<<<grd, blk, 0, st>>>(p->d_ypart, y, a.nrows, nrows, a.G);
  }
  TDB_CUDA_CHECK(cudaGetLastError());
  return TDB_OK;
}
