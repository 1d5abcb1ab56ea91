// Toeplitz-ordered tensor-core (FP64 DMMA) matvec for the lag-reused family, p = 0.
//
// Replaces the lag-term part of BlockHessenbergMatrix.matvec (/root/reference/
// pkg/src/tdbem/block_system.py:197-215, a SciPy CSR SpMV per logical block
// position): a stored inner block A_s (lag d_s) is applied at every block row kt
// of its term mask at once,
//     Y[j][kt] += sum_l A_s[j][l] X[l][kt - d_s].
//
// Storage: the family's blocks as 8 x 4 tiles (dofs in Morton order, A-fragment
// layout), sorted by (row block J, column block L, position s).  All lags of one
// (J, L) pair are adjacent, so the 4 x (time) strip of x that feeds their B
// operands is fetched from L2 once and then served from L1 for every lag; in
// position-major order (tdb_bsr.cu) every tile re-gathered its strip from L2.
//
// Kernel: one warp = (row block J, time group tg, part g).  The warp holds the
// 8 x 8 Y tiles of TT consecutive 8-step time tiles in registers (DMMA D
// fragments) and walks a contiguous share of J's tiles: one coalesced A-fragment
// load per tile, then per active time tile one B load (lane (g, t) reads
// X[4L + t][kt(g) - d_s], or the zero column when kt(g) is outside the term's
// mask: per-plan table in shared memory) and one mma.sync.m8n8k4.f64; tiles of
// positions outside the plan are skipped by a warp ballot, and the next tile's
// loads are issued before the current tile's DMMAs.  The G parts' partial tiles
// are summed in part order by k_tbsr_reduce and added to y (written before by the
// CSR kernel for the other terms): deterministic run to run.
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <string>

#include "tdb_bsr.h"
#include "tdb_common.cuh"
#include "tdb_internal.h"

namespace tdb {

namespace {

__global__ void k_tbsr_keys(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                            long long nrows_total, int nrows, int npos, const int* __restrict__ rinv,
                            const int* __restrict__ vinv, int nCB, unsigned long long* __restrict__ keys,
                            long long* __restrict__ ids) {
  const int lane = threadIdx.x & 31;
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long row = warp; row < nrows_total; row += nw) {
    const long long s = row / nrows;
    const int jl = (int)(row % nrows);
    const int jp = rinv[jl];
    const int64_t e0 = indptr[row], e1 = indptr[row + 1];
    for (int64_t e = e0 + lane; e < e1; e += 32) {
      const int lp = vinv[indices[e]];
      const unsigned sub = (unsigned)((jp & 7) * 4 + (lp & 3));
      const unsigned long long k =
          ((unsigned long long)(jp >> 3) * (unsigned long long)nCB + (unsigned long long)(lp >> 2)) *
              (unsigned long long)npos + (unsigned long long)s;
      keys[e] = (k << 5) | sub;
      ids[e] = e;
    }
  }
}

__global__ void k_tbsr_heads(const unsigned long long* __restrict__ keys, long long n, int* __restrict__ head) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    head[i] = (i == 0 || (keys[i] >> 5) != (keys[i - 1] >> 5)) ? 1 : 0;
}

__global__ void k_tbsr_fill(const unsigned long long* __restrict__ keys, const long long* __restrict__ ids,
                            const int* __restrict__ tid_incl, long long n, int nCB, int npos,
                            const double* __restrict__ data, int32_t* __restrict__ col, int32_t* __restrict__ pos,
                            double* __restrict__ val, int* __restrict__ tile_rb) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long t = tid_incl[i] - 1;
    const unsigned long long k = keys[i] >> 5;
    val[t * 32 + (keys[i] & 31u)] = data[ids[i]];
    if (i == 0 || (keys[i - 1] >> 5) != k) {
      pos[t] = (int32_t)(k % (unsigned long long)npos);
      const unsigned long long rc = k / (unsigned long long)npos;
      col[t] = (int32_t)(rc % (unsigned long long)nCB);
      tile_rb[t] = (int)(rc / (unsigned long long)nCB);
    }
  }
}

__global__ void k_tbsr_rbptr(const int* __restrict__ tile_rb, long long ntiles, int nRB, int64_t* __restrict__ rbptr) {
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

constexpr int kTbsrWarps = 4;  // warps per CTA (same time group)

struct TbsrTile {
  int s, cb;
  unsigned act;
  long long p;
};

// B fragments of one tile: lane (g, t) reads X[4 cb + t][off(s, u, g)]; the offset
// table points inactive (row, lag) combinations at the zero column of xp
template <int TT>
__device__ __forceinline__ void tbsr_load(const TbsrMvArgs& a, const int* __restrict__ s_off, const double* xq,
                                          const TbsrTile& t, int gq, int lane, double& av, double (&bv)[TT]) {
  av = __ldg(a.val + t.p * 32 + lane);
  const double* xr = xq + (long long)t.cb * 4 * a.xs;
  const int2* so = reinterpret_cast<const int2*>(s_off + (t.s * 8 + gq) * TT);
#pragma unroll
  for (int u = 0; u < TT; u += 2) {
    const int2 o = so[u >> 1];
    bv[u] = __ldg(xr + (unsigned)o.x);
    bv[u + 1] = __ldg(xr + (unsigned)o.y);
  }
}

// Cursor over a warp's tile range: batches of 32 tiles (coalesced column /
// position loads), live tiles (position in the plan) picked by ballot.  Warp-uniform.
struct TbsrCursor {
  long long pb, q1;
  int my_cb, my_s;
  unsigned my_act, live;
};

__device__ __forceinline__ bool tbsr_next(const TbsrMvArgs& a, const unsigned* s_act, int lane, TbsrCursor& c,
                                          TbsrTile& t) {
  while (c.live == 0u) {
    if (c.pb >= c.q1) return false;
    const int n = (int)min(32LL, c.q1 - c.pb);
    c.my_cb = lane < n ? __ldg(a.col + c.pb + lane) : 0;
    c.my_s = lane < n ? __ldg(a.pos + c.pb + lane) : 0;
    c.my_act = lane < n ? s_act[c.my_s] : 0u;
    c.live = __ballot_sync(0xffffffffu, c.my_act != 0u);
    c.pb += 32;
  }
  const int i = __ffs(c.live) - 1;
  c.live &= c.live - 1;
  t.s = __shfl_sync(0xffffffffu, c.my_s, i);
  t.cb = __shfl_sync(0xffffffffu, c.my_cb, i);
  t.act = __shfl_sync(0xffffffffu, c.my_act, i);
  t.p = c.pb - 32 + i;
  return true;
}

template <int TT>
__global__ void __launch_bounds__(kTbsrWarps * 32) k_tbsr_mv(TbsrMvArgs a) {
  extern __shared__ __align__(16) int tb_smem[];
  int* s_off = tb_smem;                                                    // [npos][8 (g)][TT]
  unsigned* s_act = reinterpret_cast<unsigned*>(s_off + a.npos * TT * 8);  // [npos]
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int tg = blockIdx.x % a.ntg;
  const long long jg = (long long)(blockIdx.x / a.ntg) * kTbsrWarps + wid;  // (J, g)
  {
    const int* go = a.off_tab + (long long)tg * a.npos * TT * 8;
    for (int i = threadIdx.x; i < a.npos * TT * 8; i += blockDim.x) s_off[i] = __ldg(go + i);
    for (int i = threadIdx.x; i < a.npos; i += blockDim.x) s_act[i] = __ldg(a.act_tab + (long long)tg * a.npos + i);
  }
  __syncthreads();
  if (jg >= (long long)a.nRB * a.G) return;
  const int J = (int)(jg / a.G), g = (int)(jg % a.G);
  const int gq = lane >> 2, tq = lane & 3;
  double acc[TT][2];
#pragma unroll
  for (int u = 0; u < TT; ++u) acc[u][0] = acc[u][1] = 0.0;
  const long long r0 = __ldg(a.rbptr + J), r1 = __ldg(a.rbptr + J + 1);
  const long long q0 = r0 + (r1 - r0) * g / a.G, q1 = r0 + (r1 - r0) * (g + 1) / a.G;
  const double* xq = a.xp + (long long)tq * a.xs;
  // Software pipeline over the warp's live tiles (tiles whose position is a lag
  // term of this plan), ping-pong buffers A / B: the next tile's A and B loads are
  // in flight while the current tile's DMMAs issue (no register copies).
  TbsrCursor cs{q0, q1, 0, 0, 0u, 0u};
  TbsrTile tA, tB;
  double avA, avB, bvA[TT], bvB[TT];
  bool hA = tbsr_next(a, s_act, lane, cs, tA);
  if (hA) tbsr_load<TT>(a, s_off, xq, tA, gq, lane, avA, bvA);
  while (hA) {
    const bool hB = tbsr_next(a, s_act, lane, cs, tB);
    if (hB) tbsr_load<TT>(a, s_off, xq, tB, gq, lane, avB, bvB);
#pragma unroll
    for (int u = 0; u < TT; ++u) dmma884(acc[u][0], acc[u][1], avA, bvA[u]);
    if (!hB) break;
    hA = tbsr_next(a, s_act, lane, cs, tA);
    if (hA) tbsr_load<TT>(a, s_off, xq, tA, gq, lane, avA, bvA);
#pragma unroll
    for (int u = 0; u < TT; ++u) dmma884(acc[u][0], acc[u][1], avB, bvB[u]);
  }
  // partial tiles of the G parts: summed in part order by k_tbsr_reduce
  const long long key = (long long)J * a.ntg + tg;
  double2* yp = reinterpret_cast<double2*>(a.ypart + (key * a.G + g) * (TT * 64));
#pragma unroll
  for (int u = 0; u < TT; ++u) yp[u * 32 + lane] = make_double2(acc[u][0], acc[u][1]);
}

__global__ void k_tbsr_reduce(TbsrMvArgs a) {
  const int TT64 = a.TT * 64;
  const long long total = (long long)a.nRB * a.ntg * TT64;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long key = idx / TT64;
    const int e = (int)(idx % TT64);
    const double* src = a.ypart + key * a.G * TT64 + e;
    double sum = 0.0;
    for (int gg = 0; gg < a.G; ++gg) sum += __ldcg(src + (long long)gg * TT64);
    const int J = (int)(key / a.ntg), tg = (int)(key % a.ntg);
    const int u = e >> 6, q = e & 63, ln = q >> 1, ii = q & 1;
    const int jp = 8 * J + (ln >> 2);
    const int r = 8 * (tg * a.TT + u) + 2 * (ln & 3) + ii;
    if (jp < a.nrows && r < a.nr) a.y[(long long)r * a.nrows + __ldg(a.rperm + jp)] += sum;
  }
}

template <int TT>
static int launch_tt(const TbsrMvArgs& a, cudaStream_t st, bool reduce) {
  const size_t smem = (size_t)a.npos * (TT * 8 + 1) * sizeof(int);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_tbsr_mv<TT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  const long long ctas = (((long long)a.nRB * a.G + kTbsrWarps - 1) / kTbsrWarps) * a.ntg;
  k_tbsr_mv<TT><<<(unsigned)ctas, kTbsrWarps * 32, smem, st>>>(a);
  TDB_CUDA_CHECK(cudaGetLastError());
  if (!reduce) return TDB_OK;
  const long long total = (long long)a.nRB * a.ntg * TT * 64;
  k_tbsr_reduce<<<(unsigned)std::min<long long>((total + 255) / 256, 148 * 8), 256, 0, st>>>(a);
  TDB_CUDA_CHECK(cudaGetLastError());
  return TDB_OK;
}

}  // namespace

int tbsr_build(TdbSystem* sys, int f) {
  if ((int)sys->tbsr.size() != sys->F) sys->tbsr.assign(sys->F, TbsrStore{});
  TbsrStore& b = sys->tbsr[f];
  if (b.built) return TDB_OK;
  TDB_REQUIRE(sys->p == 0, "tbsr: tensor-core storage is built for p = 0 only");
  cudaStream_t st = sys->ctx->stream;
  const int NR = sys->nrows, nRB = sys->nRB, nCB = sys->nCB;
  FamilyStore& fs = sys->fam[f];
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
#define TRY(expr)                                                      \
  do {                                                                 \
    cudaError_t e_ = (expr);                                           \
    if (e_ != cudaSuccess) {                                           \
      release();                                                       \
      set_error(std::string("tbsr build: ") + cudaGetErrorString(e_)); \
      return e_ == cudaErrorMemoryAllocation ? TDB_E_NOMEM : TDB_E_CUDA; \
    }                                                                  \
  } while (0)
  TRY(dev_malloc((void**)&b.rbptr, (size_t)(nRB + 1) * sizeof(int64_t)));
  if (n == 0) {
    TRY(cudaMemsetAsync(b.rbptr, 0, (size_t)(nRB + 1) * sizeof(int64_t), st));
    TRY(dev_malloc((void**)&b.col, sizeof(int32_t)));
    TRY(dev_malloc((void**)&b.pos, sizeof(int32_t)));
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
  const long long rows_total = (long long)fs.npos * NR;
  k_tbsr_keys<<<148 * 16, 256, 0, st>>>(fs.indptr, fs.indices, rows_total, NR, fs.npos, sys->d_rinv, sys->d_vinv,
                                        nCB, k0, i0);
  TRY(cudaGetLastError());
  int end_bit = 5;
  {
    const unsigned long long maxkey = (unsigned long long)nRB * (unsigned long long)nCB * (unsigned long long)fs.npos;
    while (end_bit < 64 && (maxkey >> (end_bit - 5)) != 0) ++end_bit;
  }
  size_t tb = 0, tb2 = 0;
  TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb, k0, k1, i0, i1, n, 0, end_bit, st));
  TRY(cub::DeviceScan::InclusiveSum(nullptr, tb2, head, head, n, st));
  TRY(dev_malloc(&tmp, std::max(tb, tb2)));
  TRY(cub::DeviceRadixSort::SortPairs(tmp, tb, k0, k1, i0, i1, n, 0, end_bit, st));
  k_tbsr_heads<<<148 * 16, 256, 0, st>>>(k1, n, head);
  TRY(cudaGetLastError());
  TRY(cub::DeviceScan::InclusiveSum(tmp, tb2, head, head, n, st));
  int nt = 0;
  TRY(cudaMemcpyAsync(&nt, head + n - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  TRY(cudaStreamSynchronize(st));
  b.ntiles = nt;
  TRY(dev_malloc((void**)&b.col, (size_t)nt * sizeof(int32_t)));
  TRY(dev_malloc((void**)&b.pos, (size_t)nt * sizeof(int32_t)));
  TRY(dev_malloc((void**)&b.val, (size_t)nt * 32 * sizeof(double)));
  TRY(dev_malloc((void**)&tile_rb, (size_t)nt * sizeof(int)));
  TRY(cudaMemsetAsync(b.val, 0, (size_t)nt * 32 * sizeof(double), st));
  k_tbsr_fill<<<148 * 16, 256, 0, st>>>(k1, i1, head, n, nCB, fs.npos, fs.data, b.col, b.pos, b.val, tile_rb);
  TRY(cudaGetLastError());
  k_tbsr_rbptr<<<(nRB + 256) / 256, 256, 0, st>>>(tile_rb, nt, nRB, b.rbptr);
  TRY(cudaGetLastError());
  TRY(cudaStreamSynchronize(st));
  release();
#undef TRY
  b.built = true;
  return TDB_OK;
}

int tbsr_mv_tiles(const TbsrMvArgs& a, cudaStream_t st, bool reduce) {
  switch (a.TT) {
    case 2: return launch_tt<2>(a, st, reduce);
    case 4: return launch_tt<4>(a, st, reduce);
    case 6: return launch_tt<6>(a, st, reduce);
    case 8: return launch_tt<8>(a, st, reduce);
    case 10: return launch_tt<10>(a, st, reduce);
    default: return launch_tt<12>(a, st, reduce);
  }
}

int tbsr_mv_reduce(const TbsrMvArgs& a, cudaStream_t st) {
  const long long total = (long long)a.nRB * a.ntg * a.TT * 64;
  k_tbsr_reduce<<<(unsigned)std::min<long long>((total + 255) / 256, 148 * 8), 256, 0, st>>>(a);
  TDB_CUDA_CHECK(cudaGetLastError());
  return TDB_OK;
}

int tbsr_mv_launch(const TbsrMvArgs& a, cudaStream_t st) { return tbsr_mv_tiles(a, st, true); }

}  // namespace tdb
