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
#include <cstdlib>
#include <vector>

#include "tdb_band.h"
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
  const FamCsr* term_csr;   // (nterms,) the term's CSR with indptr at its position's first row
  const int* term_f;
  const int* term_s;
  const int* term_d;
  const unsigned* term_mask;
  const int* term_kt;       // (nterms, 4): block rows of a "single" term, padded with 0;
                            // kt[0] == -1 marks a lag term, 0 an empty mask
  const int* group_begin;   // (G+1,) term ranges
  const double* xt;         // [M][xs]: row l = x[l][block col][m1], then NP1 zeros
  int xs;                   // row stride of xt = nc*NP1 + NP1
  double* ypart;            // [G][M][nr*NP1]
  double* y;                // output, time-major y[(block row)*NP1 + m][row]
  unsigned* row_done;       // [nrows] groups finished per row (reset by the last one)
};

__global__ void k_transpose_in(const double* __restrict__ x, double* __restrict__ xt, int M,
                               int ncols, int xs, const long long* __restrict__ xmap, long long xstride) {
  // x[xmap[l] + c*xstride] -> xt[l*xs + c], c = (block col)*NP1 + m1 (pad columns stay 0)
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
    if (c < ncols && l < M) xt[(long long)l * xs + c] = tile[threadIdx.x][k];
  }
}

// ---- asynchronous staging of a warp's CSR stream (cp.async, double-buffered) ----
__device__ __forceinline__ void cp_async4(void* smem, const void* g) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* g) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

template <int NM>
struct MvStage {
#ifndef TDB_MV_CAP1
#define TDB_MV_CAP1 256
#endif
  static constexpr int CAP = NM <= 1 ? TDB_MV_CAP1 : NM <= 4 ? 128 : 64;  // entries per buffer
  static constexpr size_t BYTES = 2 * (size_t)CAP * (4 + 8 * NM);
};

// One chunk of a CSR row segment: term t, entries [b, b + n) (n <= CAP).
struct MvChunk {
  int t, n;
  int64_t b;
};

// Producer cursor over the warp's (term, row j) CSR segments, split into chunks.
struct MvCursor {
  int t, te;           // next term to open, end of the group's term range
  int cur;             // term of the open segment
  int64_t e, e1;       // remaining entries of the open segment
  int64_t ne0, ne1;    // prefetched row bounds of term t (valid if t < te)
};

template <int NM>
__device__ __forceinline__ void mv_row_bounds(const MvArgs& a, int t, int j, int64_t& e0, int64_t& e1) {
  const FamCsr* fc = a.term_csr + t;  // one dependent level less than family -> position
  const long long row = j;
  const int kt0 = __ldg(a.term_kt + 4 * t);
  if (kt0 == 0) {  // empty mask: nothing to do
    e0 = e1 = 0;
    return;
  }
  const int64_t* ip = fc->indptr;
  e0 = __ldg(ip + row);
  e1 = __ldg(ip + row + 1);
}

template <int NM>
__device__ __forceinline__ bool mv_next_chunk(const MvArgs& a, int j, MvCursor& c, MvChunk& out) {
  constexpr int CAP = MvStage<NM>::CAP;
  while (c.e >= c.e1) {
    if (c.t >= c.te) return false;
    c.cur = c.t;
    c.e = c.ne0;
    c.e1 = c.ne1;
    ++c.t;
    if (c.t < c.te) mv_row_bounds<NM>(a, c.t, j, c.ne0, c.ne1);  // look one term ahead
  }
  out.t = c.cur;
  out.b = c.e;
  out.n = (int)min((int64_t)CAP, c.e1 - c.e);
  c.e += out.n;
  return true;
}

template <int NM>
__device__ __forceinline__ void mv_stage(const MvArgs& a, const MvChunk& ch, int* s_idx, double* s_val, int lane) {
  const FamCsr* fc = a.term_csr + ch.t;
  const int32_t* gi = fc->indices + ch.b;
  const double* gv = fc->data + ch.b * NM;
  for (int q = lane; q < ch.n; q += 32) cp_async4(s_idx + q, gi + q);
  for (int q = lane; q < ch.n * NM; q += 32) cp_async8(s_val + q, gv + q);
}

// Two inner loops, chosen per term (warp-uniform):
//  * "lag" terms (a stored block reused at > kSpmvMaxKt block rows, the
//    Toeplitz part): lanes own block rows kt.  Each staged entry (column l,
//    value v) is broadcast from shared memory and multiplies the x strip
//    xt[l][kt - d] of every valid lane; U entries' strips are loaded before any
//    FMA (U * NC * NP1 independent loads in flight).  Invalid block rows load 0.
//  * "single" terms (boundary blocks used at <= kSpmvMaxKt block rows, e.g. the
//    first block column and last block row): lanes own entries (CSR SpMV, each
//    entry read once), partial sums reduced with a fixed xor butterfly and added
//    by the lane that owns the output block row.
// The CSR stream (column indices + values) of the warp's terms is staged into
// shared memory with cp.async one chunk ahead, so the HBM latency of the matrix
// stream overlaps the FMAs of the previous chunk.  Accumulation order is fixed
// by the plan (deterministic run to run).
constexpr int kSpmvMaxKt = 4;

template <int NP1, int NC>
struct MvShape {
  static constexpr int NM = NP1 * NP1;
  static constexpr int LOADS = NC * NP1;
#ifndef TDB_MV_LOADS_IN_FLIGHT
#define TDB_MV_LOADS_IN_FLIGHT 8
#endif
  static constexpr int U0 = TDB_MV_LOADS_IN_FLIGHT / LOADS;
  static constexpr int U = U0 >= 8 ? 8 : U0 >= 4 ? 4 : U0 >= 2 ? 2 : 1;
};

template <int NP1, int NC>
__device__ __forceinline__ void mv_single_chunk(const MvArgs& a, int t, int n, const int* s_idx,
                                                const double* s_val, int lane, double (&acc)[NC][NP1]) {
  constexpr int NM = NP1 * NP1;
  const int4 k4 = __ldg(reinterpret_cast<const int4*>(a.term_kt) + t);
  const int kts[4] = {k4.x, k4.y, k4.z, k4.w};
  const int d = __ldg(a.term_d + t);
  // 32-bit element offsets (row l * xs + column) and one IMAD.WIDE.U32 per load;
  // block rows outside the mask read the zero pad column and are never reduced
  const unsigned xs = (unsigned)a.xs, zpad = xs - NP1;
  bool on[kSpmvMaxKt];
  unsigned xo[kSpmvMaxKt];
#pragma unroll
  for (int k = 0; k < kSpmvMaxKt; ++k) {
    on[k] = kts[k] > 0;
    xo[k] = on[k] ? (unsigned)((kts[k] - d - a.clo) * NP1) : zpad;
  }
  const double* __restrict__ xt = a.xt;
  double part[kSpmvMaxKt][NP1];
#pragma unroll
  for (int k = 0; k < kSpmvMaxKt; ++k)
#pragma unroll
    for (int m = 0; m < NP1; ++m) part[k][m] = 0.0;
#pragma unroll 4
  for (int q = lane; q < n; q += 32) {
    const unsigned rowo = (unsigned)s_idx[q] * xs;
    double v[NM];
#pragma unroll
    for (int m = 0; m < NM; ++m) v[m] = s_val[q * NM + m];
#pragma unroll
    for (int k = 0; k < kSpmvMaxKt; ++k) {
      if (on[k]) {  // warp-uniform
#pragma unroll
        for (int m1 = 0; m1 < NP1; ++m1) {
          const double xv = __ldg(xt + (rowo + xo[k] + m1));
#pragma unroll
          for (int m2 = 0; m2 < NP1; ++m2) part[k][m2] = fma(v[m2 * NP1 + m1], xv, part[k][m2]);
        }
      }
    }
  }
#pragma unroll
  for (int k = 0; k < kSpmvMaxKt; ++k) {
    if (!on[k]) continue;  // warp-uniform
    const int r = kts[k] - a.rlo, owner = r & 31, chunk = r >> 5;
#pragma unroll
    for (int m2 = 0; m2 < NP1; ++m2) {
      const double sum = warp_allsum(part[k][m2]);
#pragma unroll
      for (int c = 0; c < NC; ++c)
        if (c == chunk && lane == owner) acc[c][m2] += sum;
    }
  }
}

template <int NP1, int NC>
__device__ __forceinline__ void mv_lag_chunk(const MvArgs& a, int t, int n, const int* s_idx, const double* s_val,
                                             int lane, double (&acc)[NC][NP1]) {
  using S = MvShape<NP1, NC>;
  constexpr int NM = S::NM, U = S::U;
  const int d = __ldg(a.term_d + t);
  const unsigned* mask = a.term_mask + (long long)t * a.words;
  // lane validity per row chunk (bit kt-1).  Invalid lanes point at the zero
  // pad that ends every xt row, so loads and FMAs need no predicate and every
  // address is one 32-bit add + one IMAD.WIDE.U32.
  const unsigned xs = (unsigned)a.xs;
  unsigned offc[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int kt = a.rlo + lane + 32 * c;
    const bool ok = (lane + 32 * c < a.nr) && ((__ldg(mask + ((kt - 1) >> 5)) >> ((kt - 1) & 31)) & 1u);
    offc[c] = ok ? (unsigned)((kt - d - a.clo) * NP1) : xs - NP1;
  }
  const double* __restrict__ xt = a.xt;
  // n is padded to a multiple of U by the caller (weight 0, a real column)
  for (int i = 0; i < n; i += U) {
    double xr[U][NC][NP1];
    double v[U][NM];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const unsigned xo = (unsigned)s_idx[i + u] * xs;
#pragma unroll
      for (int m = 0; m < NM; ++m) v[u][m] = s_val[(i + u) * NM + m];
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int m1 = 0; m1 < NP1; ++m1) xr[u][c][m1] = __ldg(xt + (xo + offc[c] + m1));
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
          for (int m1 = 0; m1 < NP1; ++m1)
#pragma unroll
            for (int m2 = 0; m2 < NP1; ++m2) acc[c][m2] = fma(v[u][m2 * NP1 + m1], xr[u][c][m1], acc[c][m2]);
  }
}

template <int NP1, int NC>
#ifndef TDB_MV_MIN_BLOCKS
#define TDB_MV_MIN_BLOCKS 16
#endif
#ifndef TDB_MV_MIN_BLOCKS_NC1
#define TDB_MV_MIN_BLOCKS_NC1 16
#endif
__global__ void __launch_bounds__(32, NC <= 1 ? TDB_MV_MIN_BLOCKS_NC1 : TDB_MV_MIN_BLOCKS) k_matvec(MvArgs a) {
  // one warp per CTA: the warp index is blockIdx.x, so every loop bound below is
  // provably warp-uniform (plain SHFL / no divergence handling)
  constexpr int NM = NP1 * NP1;
  constexpr int CAP = MvStage<NM>::CAP;
  extern __shared__ __align__(16) unsigned char mv_smem[];
  double* s_val = reinterpret_cast<double*>(mv_smem);          // [2][CAP*NM]
  int* s_idx = reinterpret_cast<int*>(s_val + 2 * CAP * NM);   // [2][CAP]
  const int lane = threadIdx.x;
  const long long w = blockIdx.x;
  const int j = (int)(w % a.nrows), g = (int)(w / a.nrows);  // j = local row
  double acc[NC][NP1];
#pragma unroll
  for (int c = 0; c < NC; ++c)
#pragma unroll
    for (int m = 0; m < NP1; ++m) acc[c][m] = 0.0;
  MvCursor cur;
  cur.t = __ldg(a.group_begin + g);
  cur.te = __ldg(a.group_begin + g + 1);
  cur.cur = -1;
  cur.e = cur.e1 = 0;
  cur.ne0 = cur.ne1 = 0;
  if (cur.t < cur.te) mv_row_bounds<NM>(a, cur.t, j, cur.ne0, cur.ne1);
  MvChunk c0, c1;
  bool h0 = mv_next_chunk<NM>(a, j, cur, c0);
  if (h0) mv_stage<NM>(a, c0, s_idx, s_val, lane);
  cp_async_commit();
  bool h1 = h0 && mv_next_chunk<NM>(a, j, cur, c1);
  if (h1) mv_stage<NM>(a, c1, s_idx + CAP, s_val + CAP * NM, lane);
  cp_async_commit();
  int buf = 0;
  while (h0) {
    cp_async_wait1();
    __syncwarp();
    int* bi = s_idx + buf * CAP;
    double* bv = s_val + buf * CAP * NM;
    if (__ldg(a.term_kt + 4 * c0.t) > 0) {
      mv_single_chunk<NP1, NC>(a, c0.t, c0.n, bi, bv, lane, acc);
    } else {
      constexpr int U = MvShape<NP1, NC>::U;
      const int nU = (c0.n + U - 1) / U * U;  // pad: weight 0 on the chunk's first column
      for (int q = c0.n + lane; q < nU; q += 32) {
        bi[q] = bi[0];
#pragma unroll
        for (int m = 0; m < NM; ++m) bv[q * NM + m] = 0.0;
      }
      __syncwarp();
      mv_lag_chunk<NP1, NC>(a, c0.t, nU, bi, bv, lane, acc);
    }
    __syncwarp();
    c0 = c1;
    h0 = h1;
    h1 = h1 && mv_next_chunk<NM>(a, j, cur, c1);
    if (h1) mv_stage<NM>(a, c1, s_idx + buf * CAP, s_val + buf * CAP * NM, lane);
    cp_async_commit();
    buf ^= 1;
  }
  // Partial rows of the G term groups are summed in group order by the warp that
  // finishes row j last (threadfence reduction: deterministic, no extra launch).
  if (a.G == 1) {
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int r = lane + 32 * c;
      if (r < a.nr)
#pragma unroll
        for (int m = 0; m < NP1; ++m) a.y[(long long)(r * NP1 + m) * a.nrows + j] = acc[c][m];
    }
    return;
  }
  double* yp = a.ypart + ((long long)g * a.nrows + j) * (a.nr * NP1);
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int r = lane + 32 * c;
    if (r < a.nr)
#pragma unroll
      for (int m = 0; m < NP1; ++m) yp[r * NP1 + m] = acc[c][m];
  }
  __threadfence();
  unsigned prev = 0;
  if (lane == 0) prev = atomicAdd(a.row_done + j, 1u);
  prev = __shfl_sync(0xffffffffu, prev, 0);
  if (prev != (unsigned)(a.G - 1)) return;
  __threadfence();
  const double* ypj = a.ypart + (long long)j * (a.nr * NP1);
  const long long gstride = (long long)a.nrows * (a.nr * NP1);
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int r = lane + 32 * c;
    if (r < a.nr) {
#pragma unroll
      for (int m = 0; m < NP1; ++m) {
        double s = 0.0;
        for (int gg = 0; gg < a.G; ++gg) s += __ldcg(ypj + gg * gstride + r * NP1 + m);
        a.y[(long long)(r * NP1 + m) * a.nrows + j] = s;
      }
    }
  }
  if (lane == 0) a.row_done[j] = 0u;
}

template <int NP1, int NC>
static void launch_mv_nc(const MvArgs& a, int nchunks, int blocks, cudaStream_t st) {
  if constexpr (NC < kMaxRowChunks) {
    if (nchunks > NC) return launch_mv_nc<NP1, NC + 1>(a, nchunks, blocks, st);
  }
  constexpr size_t smem = MvStage<NP1 * NP1>::BYTES;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_matvec<NP1, NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_matvec<NP1, NC><<<blocks, 32, smem, st>>>(a);
}

// ---- single-term SpMV (p = 0): the boundary blocks of a band plan --------------
// Plans whose lag terms all go to the band tiles keep only "single" CSR terms:
// boundary-family blocks each applied at <= kSpmvMaxKt block rows (first block
// column, last block row, singletons).  One warp per output row (kt, j): it walks
// that row's single items in plan order, lanes over the CSR entries (4 entries
// per lane in flight (8 measured slower), coalesced 4/8-byte streams), x read from the time-major
// iterate (one block column = M doubles, L1/L2 resident), a fixed xor-butterfly
// reduction, and ONE plain store y[kt][j] = sum (rows without items get 0; the
// band partials are added afterwards by k_band_reduce).  Deterministic.
struct SpmvItem {
  int64_t rowptr;  // offset of the item's (position, row 0) in its family's indptr
  int fam, col;    // family, block column of x relative to the plan's clo
};

struct SpmvArgs {
  int nrows, nkt;                     // owned rows, output block rows of the plan
  const int* kt_ptr;                  // (nkt + 1,) items of output row kt
  const SpmvItem* items;
  const FamCsr* fam;
  const double* x;
  const long long* xmap;              // NULL: x[c * M + l]
  long long xstride;
  int M;
  double* y;                          // y[kt_local * nrows + j]
};

__global__ void __launch_bounds__(256) k_spmv_single(SpmvArgs a) {
  const int lane = threadIdx.x & 31;
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  if (warp >= (long long)a.nkt * a.nrows) return;
  const int kt = (int)(warp / a.nrows), j = (int)(warp % a.nrows);
  double sum = 0.0;
  for (int it = a.kt_ptr[kt]; it < a.kt_ptr[kt + 1]; ++it) {
    const SpmvItem m = a.items[it];
    const FamCsr F = a.fam[m.fam];
    const int64_t e0 = __ldg(F.indptr + m.rowptr + j), e1 = __ldg(F.indptr + m.rowptr + j + 1);
    const double* xc = a.x + (long long)m.col * a.xstride;
    double acc = 0.0;
    int64_t e = e0 + lane;
    for (; e + 96 < e1; e += 128) {
      const int l0 = __ldg(F.indices + e), l1 = __ldg(F.indices + e + 32), l2 = __ldg(F.indices + e + 64),
                l3 = __ldg(F.indices + e + 96);
      const double v0 = __ldg(F.data + e), v1 = __ldg(F.data + e + 32), v2 = __ldg(F.data + e + 64),
                   v3 = __ldg(F.data + e + 96);
      const double x0 = __ldg(xc + (a.xmap ? a.xmap[l0] : l0)), x1 = __ldg(xc + (a.xmap ? a.xmap[l1] : l1));
      const double x2 = __ldg(xc + (a.xmap ? a.xmap[l2] : l2)), x3 = __ldg(xc + (a.xmap ? a.xmap[l3] : l3));
      acc = fma(v0, x0, acc);
      acc = fma(v1, x1, acc);
      acc = fma(v2, x2, acc);
      acc = fma(v3, x3, acc);
    }
    for (; e < e1; e += 32) {
      const int l0 = __ldg(F.indices + e);
      acc = fma(__ldg(F.data + e), __ldg(xc + (a.xmap ? a.xmap[l0] : l0)), acc);
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    sum += acc;
  }
  if (lane == 0) a.y[(long long)kt * a.nrows + j] = sum;
}

}  // namespace tdb

using namespace tdb;

struct TdbMatvecPlan {
  TdbSystem* sys = nullptr;
  MvArgs args{};
  long long* d_xmap = nullptr;
  long long xstride = 0;
  FamCsr* d_fam = nullptr;
  FamCsr* d_tcsr = nullptr;
  int* d_ints = nullptr;       // term_f, term_s, term_d, group_begin
  unsigned* d_mask = nullptr;
  double* d_xt = nullptr;
  double* d_ypart = nullptr;
  unsigned* d_done = nullptr;
  double bytes = 0.0, flops = 0.0;
  // p = 0 lag-band tensor-core path for the inner family's regular lag terms (tdb_band.cu)
  bool band = false;
  int n_tiled = 0, n_csr = 0, n_csr_all = 0;
  // the band kernel runs on its own stream, concurrently with the CSR kernel
  cudaStream_t tst = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  BandMvArgs bargs{};
  int band_cols = 0, band_c0 = 0, band_padl = 0;  // inner columns of x copied into xt, first one, pad
  unsigned* d_sact = nullptr;
  double* d_bxt = nullptr;
  double* d_bypart = nullptr;
  // single-term SpMV replacing the CSR kernel when every non-band term is a single term
  bool spmv = false;
  SpmvArgs sargs{};
  int* d_ktptr = nullptr;
  SpmvItem* d_items = nullptr;
  FamCsr* d_sfam = nullptr;
};

extern "C" int tdb_matvec_plan_destroy(TdbMatvecPlan* p) {
  if (!p) return TDB_OK;
  cudaDeviceSynchronize();  // the system may already be gone: no p->sys access here
  if (p->tst) cudaStreamDestroy(p->tst);
  if (p->ev_fork) cudaEventDestroy(p->ev_fork);
  if (p->ev_join) cudaEventDestroy(p->ev_join);
  dev_free(p->d_sact);
  dev_free(p->d_bxt);
  dev_free(p->d_bypart);
  dev_free(p->d_ktptr);
  dev_free(p->d_items);
  dev_free(p->d_sfam);
  dev_free(p->d_fam);
  dev_free(p->d_tcsr);
  dev_free(p->d_ints);
  dev_free(p->d_mask);
  dev_free(p->d_xt);
  dev_free(p->d_ypart);
  dev_free(p->d_done);
  dev_free(p->d_xmap);
  delete p;
  return TDB_OK;
}

static int plan_create_impl(TdbSystem* sys, const TdbMatvecDesc* d, TdbMatvecPlan** out) {
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
  std::vector<double> tcost(nt);
  std::vector<int> term_kt(4 * (size_t)nt, 0);
  std::vector<std::vector<int64_t>> famptr(sys->F);
  double bytes = 0.0, flops = 0.0;
  for (int t = 0; t < nt; ++t) {
    const int f = d->term_family[t], s = d->term_pos[t];
    if (f < 0 || f >= sys->F || s < 0 || s >= sys->fam[f].npos) {
      delete p;
      set_error("matvec: term references a missing family/position");
      return TDB_E_INVALID;
    }
    std::vector<int64_t>& fp = famptr[f];
    if (fp.empty()) {  // one D2H copy of each referenced family's row pointers
      fp.resize((size_t)sys->fam[f].npos * NR + 1);
      TDB_CUDA_CHECK(cudaMemcpy(fp.data(), sys->fam[f].indptr, fp.size() * sizeof(int64_t),
                                cudaMemcpyDeviceToHost));
    }
    tnnz[t] = fp[(size_t)(s + 1) * NR] - fp[(size_t)s * NR];
    int nlog = 0;
    for (int w = 0; w < d->words; ++w) nlog += __builtin_popcount(d->term_mask[(long long)t * d->words + w]);
    bytes += (double)tnnz[t] * (8.0 * NM + 4.0);
    flops += 2.0 * NM * (double)tnnz[t] * nlog;
    int* k4 = &term_kt[4 * (size_t)t];
    if (nlog <= kSpmvMaxKt) {
      int q = 0;
      for (int kt = 1; kt <= d->N; ++kt)
        if ((d->term_mask[(long long)t * d->words + ((kt - 1) >> 5)] >> ((kt - 1) & 31)) & 1u) {
          if (kt < d->rlo || kt > d->rhi) {
            delete p;
            set_error("matvec: term mask has a block row outside the plan's row range");
            return TDB_E_INVALID;
          }
          k4[q++] = kt;
        }
      tcost[t] = (double)tnnz[t] * (10.0 + 3.0 * nlog) / 32.0;
    } else {
      k4[0] = -1;
      tcost[t] = (double)tnnz[t] * (3.0 + 3.0 * ((d->rhi - d->rlo + 32) / 32) * NP1);
    }
  }
  const int nr = d->rhi - d->rlo + 1, nc = d->chi - d->clo + 1;
  bytes += 8.0 * ((double)nr * NR + (double)nc * M) * NP1;
  p->bytes = bytes;
  p->flops = flops;
  p->n_csr_all = nt;
  // groups: enough warps to fill the chip on small meshes
  static const int warps_per_sm = [] {
    const char* e = std::getenv("TDB_MV_WARPS_PER_SM");
    return e ? std::max(1, std::atoi(e)) : 48;
  }();
  const int want_warps = sys->ctx->num_sms * warps_per_sm;
  int G = std::max(1, std::min(nt, (want_warps + NR - 1) / NR));
  G = std::min(G, 64);
  std::vector<int> gb(G + 1, nt);
  {
    double total = 0;
    for (double v : tcost) total += v;
    double acc = 0;
    int g = 0;
    gb[0] = 0;
    for (int t = 0; t < nt && g < G - 1; ++t) {
      acc += tcost[t];
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
  const size_t kt_off = (ints.size() + 3) & ~size_t(3);  // 16-byte aligned int4 rows
  ints.resize(kt_off, 0);
  ints.insert(ints.end(), term_kt.begin(), term_kt.end());
  cudaStream_t st = sys->ctx->stream;
#define ALLOC_COPY(dst, src, n, T)                                                                 \
  do {                                                                                             \
    size_t nn = std::max<size_t>(1, (size_t)(n));                                                  \
    if (dev_malloc((void**)&(dst), nn * sizeof(T)) != cudaSuccess) {                              \
      tdb_matvec_plan_destroy(p);                                                                  \
      set_error("matvec plan: cudaMalloc failed");                                                 \
      return TDB_E_NOMEM;                                                                          \
    }                                                                                              \
    if ((n) > 0 && (src) != nullptr)                                                               \
      cudaMemcpyAsync((dst), (src), (size_t)(n) * sizeof(T), cudaMemcpyHostToDevice, st);          \
  } while (0)
  std::vector<FamCsr> tcsr(std::max(1, nt));
  for (int t = 0; t < nt; ++t) {
    const FamilyStore& fs_ = sys->fam[d->term_family[t]];
    tcsr[t] = {fs_.indptr + (size_t)d->term_pos[t] * NR, fs_.indices, fs_.data};
  }
  ALLOC_COPY(p->d_fam, fam.data(), sys->F, FamCsr);
  ALLOC_COPY(p->d_tcsr, tcsr.data(), nt, FamCsr);
  ALLOC_COPY(p->d_ints, ints.data(), ints.size(), int);
  ALLOC_COPY(p->d_mask, d->term_mask, (size_t)nt * d->words, unsigned);
  ALLOC_COPY(p->d_xt, (const double*)nullptr, (size_t)M * (nc + 1) * NP1, double);
  cudaMemsetAsync(p->d_xt, 0, (size_t)M * (nc + 1) * NP1 * sizeof(double), st);  // zero pads
  ALLOC_COPY(p->d_ypart, (const double*)nullptr, (size_t)G * NR * nr * NP1, double);
  ALLOC_COPY(p->d_done, (const unsigned*)nullptr, (size_t)NR, unsigned);
  cudaMemsetAsync(p->d_done, 0, (size_t)NR * sizeof(unsigned), st);
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
  a.term_csr = p->d_tcsr;
  a.term_f = p->d_ints;
  a.term_s = p->d_ints + nt;
  a.term_d = p->d_ints + 2 * nt;
  a.group_begin = p->d_ints + 3 * nt;
  a.term_kt = p->d_ints + kt_off;
  a.term_mask = p->d_mask;
  a.xt = p->d_xt;
  a.xs = (nc + 1) * NP1;
  a.ypart = p->d_ypart;
  a.row_done = p->d_done;
  *out = p;
  return TDB_OK;
}

// Regular lag terms of the inner (Toeplitz) family -> lag-band DMMA tiles
// (tdb_band.cu); every other term (boundary blocks, the light-cone tie lag whose
// logical mask is not the full band, and all terms when p > 0) -> the CSR kernel
// above, which writes y first; the band partials are added after it.
extern "C" int tdb_matvec_plan_create(TdbSystem* sys, const TdbMatvecDesc* d, TdbMatvecPlan** out) {
  TDB_REQUIRE(sys && d && out, "NULL argument");
  static const bool band_on = [] {
    const char* e = std::getenv("TDB_MV_BAND");
    return !(e && std::atoi(e) == 0);
  }();
  const int nt = d->nterms;
  if (!band_on || sys->np1 != 1 || nt <= 0 || d->words != (d->N + 31) / 32) return plan_create_impl(sys, d, out);
  const int N = d->N;
  std::vector<int> nlog(nt, 0), cnt(sys->F, 0);
  for (int t = 0; t < nt; ++t) {
    const int f = d->term_family[t];
    if (f < 0 || f >= sys->F || d->term_pos[t] < 0 || d->term_pos[t] >= sys->fam[f].npos)
      return plan_create_impl(sys, d, out);  // reports the error
    for (int w = 0; w < d->words; ++w) nlog[t] += __builtin_popcount(d->term_mask[(long long)t * d->words + w]);
    if (nlog[t] > kSpmvMaxKt) ++cnt[f];
  }
  const int tf = (int)(std::max_element(cnt.begin(), cnt.end()) - cnt.begin());
  if (cnt[tf] < 2) return plan_create_impl(sys, d, out);
  // band rows / columns: the inner block rows and columns of the plan's ranges
  const int ktlo = std::max(d->rlo, 2), kthi = std::min(d->rhi, N - 1);
  const int itlo = std::max(d->clo, 2), ithi = std::min(d->chi, N - 1);
  if (ktlo > kthi || itlo > ithi) return plan_create_impl(sys, d, out);
  const int npos = sys->fam[tf].npos;
  // lag of each position: must be d0 + s (the family's positions are consecutive lags)
  int d0 = 0;
  bool have_d0 = false, consecutive = true;
  for (int t = 0; t < nt; ++t)
    if (d->term_family[t] == tf) {
      const int dd = d->term_d[t] - d->term_pos[t];
      if (!have_d0) {
        d0 = dd;
        have_d0 = true;
      } else if (dd != d0) {
        consecutive = false;
      }
    }
  if (!consecutive) return plan_create_impl(sys, d, out);
  std::vector<int> term_of(npos, -1);
  std::vector<char> to_tile(nt, 0);
  double useful = 0.0;
  int s_irr = -1;
  std::vector<unsigned> irr_bits(kIrrWords, 0u);
  for (int t = 0; t < nt; ++t) {
    if (d->term_family[t] != tf || term_of[d->term_pos[t]] >= 0) continue;
    // regular: the logical mask is exactly {kt in band rows : kt - d in band columns};
    // one term whose mask is a strict subset of that (the light-cone tie lag, whose
    // zero test is decided per logical position) rides along with a row mask
    const unsigned* mk = d->term_mask + (long long)t * d->words;
    bool regular = true, subset = true;
    int n = 0;
    for (int kt = 1; kt <= N; ++kt) {
      const bool want = kt >= ktlo && kt <= kthi && kt - d->term_d[t] >= itlo && kt - d->term_d[t] <= ithi;
      const bool have = (mk[(kt - 1) >> 5] >> ((kt - 1) & 31)) & 1u;
      regular &= want == have;
      subset &= want || !have;
      n += have;
    }
    if (n == 0 || !subset) continue;
    if (!regular) {
      if (s_irr >= 0 || kthi - ktlo + 1 > 32 * kIrrWords) continue;
      s_irr = d->term_pos[t];
      for (int kt = ktlo; kt <= kthi; ++kt)
        if ((mk[(kt - 1) >> 5] >> ((kt - 1) & 31)) & 1u) irr_bits[(kt - ktlo) >> 5] |= 1u << ((kt - ktlo) & 31);
    }
    term_of[d->term_pos[t]] = t;
    to_tile[t] = 1;
    useful += n;
  }
  const int nkt = kthi - ktlo + 1, nT = (nkt + 7) / 8;
  int ntiled = 0;
  for (int s_ = 0; s_ < npos; ++s_) ntiled += term_of[s_] >= 0;
  static const double min_eff = [] {
    const char* e = std::getenv("TDB_BAND_MIN_EFF");
    return e ? std::atof(e) : 0.25;
  }();
  if (ntiled < 2 || useful < min_eff * (double)ntiled * nT * 8) return plan_create_impl(sys, d, out);
  if (band_build(sys, tf) != TDB_OK) {  // e.g. no room for the tile copy: CSR for every term
    cudaGetLastError();
    return plan_create_impl(sys, d, out);
  }
  // the CSR plan of the remaining terms
  std::vector<int> cf, cs, cd;
  std::vector<unsigned> cm;
  for (int t = 0; t < nt; ++t) {
    if (to_tile[t]) continue;
    cf.push_back(d->term_family[t]);
    cs.push_back(d->term_pos[t]);
    cd.push_back(d->term_d[t]);
    cm.insert(cm.end(), d->term_mask + (long long)t * d->words, d->term_mask + (long long)(t + 1) * d->words);
  }
  TdbMatvecDesc dc = *d;
  dc.nterms = (int)cf.size();
  dc.term_family = cf.data();
  dc.term_pos = cs.data();
  dc.term_d = cd.data();
  dc.term_mask = cm.data();
  TdbMatvecPlan* p = nullptr;
  int rc = plan_create_impl(sys, &dc, &p);
  if (rc != TDB_OK) return rc;
  {  // every remaining term a single term: one warp per output row instead of the CSR kernel
    static const bool spmv_on = [] {
      const char* e = std::getenv("TDB_MV_SPMV");
      return !(e && std::atoi(e) == 0);
    }();
    bool all_single = spmv_on && sys->np1 == 1;
    for (int t = 0; t < nt && all_single; ++t)
      if (!to_tile[t] && nlog[t] > kSpmvMaxKt) all_single = false;
    if (all_single) {
      const int nr = d->rhi - d->rlo + 1;
      std::vector<int> ktptr(nr + 1, 0);
      std::vector<SpmvItem> items;
      for (int r = 0; r < nr; ++r) {
        const int kt = d->rlo + r;
        for (size_t q = 0; q < cf.size(); ++q) {
          const unsigned* mk = cm.data() + q * d->words;
          if (!((mk[(kt - 1) >> 5] >> ((kt - 1) & 31)) & 1u)) continue;
          items.push_back(SpmvItem{(int64_t)cs[q] * sys->nrows, cf[q], kt - cd[q] - d->clo});
        }
        ktptr[r + 1] = (int)items.size();
      }
      cudaStream_t st0 = sys->ctx->stream;
      if (dev_malloc((void**)&p->d_ktptr, ktptr.size() * sizeof(int)) != cudaSuccess ||
          dev_malloc((void**)&p->d_items, std::max<size_t>(1, items.size()) * sizeof(SpmvItem)) != cudaSuccess) {
        tdb_matvec_plan_destroy(p);
        set_error("matvec plan: cudaMalloc failed");
        return TDB_E_NOMEM;
      }
      TDB_CUDA_CHECK(cudaMemcpyAsync(p->d_ktptr, ktptr.data(), ktptr.size() * sizeof(int), cudaMemcpyHostToDevice, st0));
      if (!items.empty())
        TDB_CUDA_CHECK(cudaMemcpyAsync(p->d_items, items.data(), items.size() * sizeof(SpmvItem),
                                       cudaMemcpyHostToDevice, st0));
      TDB_CUDA_CHECK(cudaStreamSynchronize(st0));
      SpmvArgs& sa = p->sargs;
      sa.nrows = sys->nrows;
      sa.nkt = nr;
      sa.kt_ptr = p->d_ktptr;
      sa.items = p->d_items;
      sa.fam = p->args.fam;
      sa.xmap = p->d_xmap;
      sa.xstride = p->xstride;
      sa.M = (int)sys->V;
      p->spmv = true;
    }
  }
  // algorithmic bytes / flops of the tiled terms (canonical CSR figures, as for the rest)
  {
    std::vector<int64_t> fp((size_t)npos * sys->nrows + 1);
    TDB_CUDA_CHECK(cudaMemcpy(fp.data(), sys->fam[tf].indptr, fp.size() * sizeof(int64_t), cudaMemcpyDeviceToHost));
    for (int t = 0; t < nt; ++t)
      if (to_tile[t]) {
        const double nnz = (double)(fp[(size_t)(d->term_pos[t] + 1) * sys->nrows] - fp[(size_t)d->term_pos[t] * sys->nrows]);
        p->bytes += nnz * 12.0;
        p->flops += 2.0 * nnz * nlog[t];
      }
  }
  const BandStore& bs = sys->band[tf];
  const int act_words = (npos + 31) / 32 + 1, V = (int)sys->V, nRB = sys->nRB;
  std::vector<unsigned> sact(act_words, 0u);
  for (int s_ = 0; s_ < npos; ++s_)
    if (term_of[s_] >= 0) sact[s_ >> 5] |= 1u << (s_ & 31);
  // the records of this plan's active lags only, masks and valid time tiles baked in
  // (cached per plan signature)
  const BandTile* view_tiles = nullptr;
  const int64_t* view_rbptr = nullptr;
  long long view_ntiles = 0;
  if (band_view(sys, tf, sact, itlo + d0 - ktlo, ithi + d0 - ktlo, nT, &view_tiles, &view_rbptr, &view_ntiles) !=
      TDB_OK) {
    tdb_matvec_plan_destroy(p);
    return TDB_E_NOMEM;
  }
  // time tiles per warp ~3 (more warps per CTA: B-load parallelism), at most 8 warps
  // (measured on config 4: 3 for the 40-row ranges of the preconditioner, 5 for longer ones)
  static const int tt_env = [] {
    const char* e = std::getenv("TDB_BAND_TT");
    return e ? std::max(1, std::min(6, std::atoi(e))) : 0;
  }();
  // short plans (<= 6 time tiles): one warp covers every time tile and reads its records
  // straight from global memory (k_band_direct); TDB_BAND_DIRECT=0 keeps the ring kernel
  static const bool direct_env = [] {
    const char* e = std::getenv("TDB_BAND_DIRECT");
    return !(e && std::atoi(e) == 0);
  }();
  static const int direct_max_nt = [] {  // direct kernel up to this many time tiles (0: never)
    const char* e = std::getenv("TDB_BAND_DIRECT_NT");
    // config 4: longer plans are faster on the ring kernel (half range 1.09 vs 1.29 ms,
    // full 2.42 vs 3.05 ms); the short ones on the direct kernel (quarter 0.28 vs 0.33 ms)
    return e ? std::atoi(e) : 6;
  }();
  const bool direct = direct_env && nT <= direct_max_nt && nT <= 48 && !tt_env;
  const int tt_target = tt_env ? tt_env : (nT <= 6 ? 3 : 5);
  // direct units: the fewest warps (1, 2, 4, 8) with at most 6 time tiles each
  static const int direct_tt = [] {  // most time tiles per direct warp
    const char* e = std::getenv("TDB_BAND_DIRECT_TT");
    return e ? std::max(1, std::min(6, std::atoi(e))) : 6;
  }();
  int Wd = 1;
  while (Wd < 8 && (nT + Wd - 1) / Wd > direct_tt) Wd *= 2;
  const int W = direct ? Wd : std::max(1, std::min(kBandMaxWarps, (nT + tt_target - 1) / tt_target));
  const int TT = (nT + W - 1) / W;
  if (TT > 6) {  // more than 384 block rows: not instantiated
    tdb_matvec_plan_destroy(p);
    return plan_create_impl(sys, d, out);
  }
  // xt column of (kt, lag d): PADL + (kt - d - itlo); off0 = column of (ktlo + n, d0 + 4 S + k) + 4 S + k - n
  const int base = ktlo - itlo - d0;
  const int padl = std::max(0, npos + 2 - base);  // window start lags s0 <= npos - 1
  const int off0 = padl + base;
  const int ncols = ithi - itlo + 1;
  int xs = std::max(padl + ncols, off0 + 8 * W * TT + 8);
  xs = (xs + 1) & ~1;
  const long long tiles_per_rb = view_ntiles / std::max(1, nRB);
  // stage size: 16 records for 1-2 warps per CTA (twice the resident CTAs), else 32;
  // parts per row block: as many CTAs as fit on the SMs at once (shared-memory ring)
  const int chunk = W <= 2 ? 16 : kBandChunk;
  static const int band_ctas_env = [] {
    const char* e = std::getenv("TDB_BAND_CTAS_PER_SM");
    return e ? std::max(1, std::atoi(e)) : 0;
  }();
  const int band_ctas = band_ctas_env ? band_ctas_env
                                      : std::max(1, std::min(16, (int)((200 * 1024) / band_smem_bytes((npos + 31) / 32 + 1, chunk))));
  // one wave: nRB * P <= SMs x resident CTAs (a partial second wave is a pure tail)
  // (direct plans: ~32 warps per SM, at least 16 records per warp)
  static const int direct_wps = [] {  // direct plans: warps per SM the parts are sized for
    const char* e = std::getenv("TDB_BAND_DIRECT_WPS");
    return e ? std::max(1, std::atoi(e)) : 48;  // config 4 quarter range: 16 -> 0.320, 32 -> 0.285, 48 -> 0.280 ms
  }();
  const int P = direct ? (int)std::max<long long>(
                             1, std::min<long long>({64LL, ((long long)sys->ctx->num_sms * direct_wps) / std::max(1, nRB * W),
                                                     tiles_per_rb / 16}))
                       : (int)std::max<long long>(
                             1, std::min<long long>({64LL, ((long long)sys->ctx->num_sms * band_ctas) / std::max(1, nRB),
                                                     tiles_per_rb / (2 * chunk)}));
  const int ldy = 8 * W * TT;
  cudaStream_t st = sys->ctx->stream;
  const size_t xt_n = (size_t)V * xs;
  const size_t yp_n = (size_t)P * nRB * 8 * ldy;
#define ALLOC_COPY3(dst, src, n, T_)                                                               \
  do {                                                                                             \
    size_t nn = std::max<size_t>(1, (size_t)(n));                                                  \
    if (dev_malloc((void**)&(dst), nn * sizeof(T_)) != cudaSuccess) {                             \
      tdb_matvec_plan_destroy(p);                                                                  \
      set_error("matvec plan: cudaMalloc failed");                                                 \
      return TDB_E_NOMEM;                                                                          \
    }                                                                                              \
    if ((n) > 0 && (src) != nullptr)                                                               \
      cudaMemcpyAsync((dst), (src), (size_t)(n) * sizeof(T_), cudaMemcpyHostToDevice, st);         \
  } while (0)
  ALLOC_COPY3(p->d_sact, sact.data(), act_words, unsigned);
  ALLOC_COPY3(p->d_bypart, (const double*)nullptr, yp_n, double);
  ALLOC_COPY3(p->d_bxt, (const double*)nullptr, xt_n, double);
  cudaMemsetAsync(p->d_bxt, 0, xt_n * sizeof(double), st);  // zero pads (never written again)
#undef ALLOC_COPY3
  TDB_CUDA_CHECK(cudaStreamSynchronize(st));
  BandMvArgs& ba = p->bargs;
  ba.nRB = nRB;
  ba.P = P;
  ba.nT = nT;
  ba.TT = TT;
  ba.W = W;
  ba.nrows = sys->nrows;
  ba.act_words = act_words;
  ba.chunk = chunk;
  ba.direct = direct ? 1 : 0;
  ba.ktlo = ktlo;
  ba.nkt = nkt;
  ba.rlo = d->rlo;
  ba.off0 = off0;
  ba.dt0 = itlo + d0 - ktlo;
  ba.dt1 = ithi + d0 - ktlo;
  ba.xs = xs;
  ba.ldy = ldy;
  ba.tiles = view_tiles;
  ba.rbptr = view_rbptr;
  ba.s_irr = s_irr;
  for (int w_ = 0; w_ < kIrrWords; ++w_) ba.irr_mask[w_] = irr_bits[w_];
  ba.s_act = p->d_sact;
  ba.rperm = sys->d_rperm;
  ba.xt = p->d_bxt;
  ba.ypart = p->d_bypart;
  p->band_cols = ncols;
  p->band_c0 = itlo - d->clo;
  p->band_padl = padl;
  if (cudaStreamCreateWithFlags(&p->tst, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&p->ev_join, cudaEventDisableTiming) != cudaSuccess) {
    tdb_matvec_plan_destroy(p);
    set_error("matvec plan: stream/event creation failed");
    return TDB_E_CUDA;
  }
  p->band = true;
  p->n_tiled = nt - (int)cf.size();
  p->n_csr = (int)cf.size();
  *out = p;
  return TDB_OK;
}

extern "C" int tdb_matvec_plan_kind(const TdbMatvecPlan* p, int32_t* tiled_terms, int32_t* csr_terms) {
  TDB_REQUIRE(p != nullptr, "NULL plan");
  if (tiled_terms) *tiled_terms = p->band ? p->n_tiled : 0;
  if (csr_terms) *csr_terms = p->band ? p->n_csr : p->n_csr_all;
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
  const int ncols = a.nc * a.NP1;
  // The band kernel runs on the plan's own stream, concurrently with the boundary-term
  // kernel (event fork / join; inside a CUDA-graph capture, e.g. the recursive
  // preconditioner, the fork becomes two parallel graph branches).  TDB_MV_FORK=0 keeps
  // both on the caller's stream.
  static const bool fork_on = [] {
    const char* e = std::getenv("TDB_MV_FORK");
    return !(e && std::atoi(e) == 0);
  }();
  const bool fork = p->band && fork_on;
  if (p->band) {
    cudaStream_t bst = st;
    if (fork) {
      TDB_CUDA_CHECK(cudaEventRecord(p->ev_fork, st));
      TDB_CUDA_CHECK(cudaStreamWaitEvent(p->tst, p->ev_fork, 0));
      bst = p->tst;
    }
    // inner columns of x -> vertex-major rows of xt at column padl (pads stay zero)
    dim3 blk(32, 8), grd((a.M + 31) / 32, (p->band_cols + 31) / 32);
    k_transpose_in<<<grd, blk, 0, bst>>>(x + (long long)p->band_c0 * p->xstride, p->d_bxt + p->band_padl, a.M,
                                         p->band_cols, p->bargs.xs, p->d_xmap, p->xstride);
    TDB_CUDA_CHECK(cudaGetLastError());
    p->bargs.y = y;
    int rc = band_mv_tiles(p->bargs, bst);
    if (rc) return rc;
    if (fork) TDB_CUDA_CHECK(cudaEventRecord(p->ev_join, p->tst));
  }
  if (p->spmv) {
    p->sargs.x = x;
    p->sargs.y = y;
    const long long warps = (long long)p->sargs.nkt * p->sargs.nrows;
    k_spmv_single<<<(unsigned)((warps + 7) / 8), 256, 0, st>>>(p->sargs);
    TDB_CUDA_CHECK(cudaGetLastError());
  } else {
    dim3 blk(32, 8), grd((a.M + 31) / 32, (ncols + 31) / 32);
    k_transpose_in<<<grd, blk, 0, st>>>(x, p->d_xt, a.M, ncols, a.xs, p->d_xmap, p->xstride);
  }
  p->args.y = y;
  if (!p->spmv) {
    const long long warps = (long long)a.nrows * a.G;
    const int blocks = (int)warps;
    const int nchunks = (a.nr + 31) >> 5;
    switch (a.NP1) {
      case 1: launch_mv_nc<1, 1>(a, nchunks, blocks, st); break;
      case 2: launch_mv_nc<2, 1>(a, nchunks, blocks, st); break;
      case 3: launch_mv_nc<3, 1>(a, nchunks, blocks, st); break;
      default: launch_mv_nc<4, 1>(a, nchunks, blocks, st); break;
    }
  }
  TDB_CUDA_CHECK(cudaGetLastError());
  if (p->band) {  // (join,) then the band partials are added to the CSR kernel's y in part order
    if (fork) TDB_CUDA_CHECK(cudaStreamWaitEvent(st, p->ev_join, 0));
    return band_mv_reduce(p->bargs, st);
  }
  return TDB_OK;
}
