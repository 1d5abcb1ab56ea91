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
// order, row block J) x 4 consecutive lags for ONE column vertex l, starting at
// the first lag of the (J, l) band (so the 4-lag windows follow the band, not a
// fixed grid), in the mma.m8n8k4 A-fragment order (lane = 4 * row + lag) with the
// (l, first lag) header in the same 272-byte record.  Records are sorted (J, l, lag).
//
// Matvec: the B operand of tile (J, l, s0) at time tile u is a Hankel window of
// ONE row of the vertex-major iterate: B[k][n] = X[l][kt0 + n - d_0 - s0 - k], so
// lane (n = lane / 4, k = lane % 4) reads xt[l][off0 - s0 - k + n + 8u] - an
// L1-resident load (all lag windows of (J, l) reuse the row).  One CTA = (row block
// J, part of J's tile list): its tile records stream HBM -> shared memory through a
// 3-stage ring of cp.async.bulk copies completing on mbarriers (one elected
// thread produces), and its warps split the time tiles over the same staged
// records (each record read from HBM once).  Columns outside the plan's range are
// zero pads of xt; positions outside the plan (or whose logical mask is not the
// full band, e.g. the light-cone tie lag) are masked off per lane and handled by
// the CSR kernel.  Part partials are summed in part order (deterministic) and
// added to y after the CSR kernel has written it.
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <string>

#include "tdb_async.cuh"
#include "tdb_band.h"
#include "tdb_common.cuh"
#include "tdb_internal.h"

namespace tdb {

namespace {

// pass 1 keys: ((J V + l) << 7 | s) << 3 | r  (entries of one (row block, column) adjacent, by lag)
__global__ void k_band_keys(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                            long long nrows_total, int nrows, int V, const int* __restrict__ rinv,
                            unsigned long long* __restrict__ keys, long long* __restrict__ ids) {
  const int lane = threadIdx.x & 31;
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long row = warp; row < nrows_total; row += nw) {
    const int s = (int)(row / nrows);
    const int jp = rinv[(int)(row % nrows)];
    const int64_t e0 = indptr[row], e1 = indptr[row + 1];
    for (int64_t e = e0 + lane; e < e1; e += 32) {
      const unsigned long long jl = (unsigned long long)(jp >> 3) * (unsigned long long)V + (unsigned long long)indices[e];
      keys[e] = (((jl << 7) | (unsigned long long)s) << 3) | (unsigned long long)(jp & 7);
      ids[e] = e;
    }
  }
}

// segment (row block, column) starts: seg[i] = i at a segment head, else 0 (max-scanned next)
__global__ void k_band_seg(const unsigned long long* __restrict__ keys, long long n, long long* __restrict__ seg) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    seg[i] = (i == 0 || (keys[i] >> 10) != (keys[i - 1] >> 10)) ? i : 0;
}

// tile heads: a new (row block, column) segment or a new 4-lag window from the segment's first lag
__global__ void k_band_heads(const unsigned long long* __restrict__ keys, const long long* __restrict__ seg, long long n,
                             int* __restrict__ head) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int s0 = (int)((keys[seg[i]] >> 3) & 127u);
    const int t = ((int)((keys[i] >> 3) & 127u) - s0) >> 2;
    int h = 1;
    if (i > 0 && seg[i] == seg[i - 1]) h = t != ((((int)((keys[i - 1] >> 3) & 127u)) - s0) >> 2);
    head[i] = h;
  }
}

__global__ void k_band_fill(const unsigned long long* __restrict__ keys, const long long* __restrict__ ids,
                            const long long* __restrict__ seg, const int* __restrict__ tid_incl, long long n, int V,
                            const double* __restrict__ data, BandTile* __restrict__ tiles, int* __restrict__ tile_rb) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long t = tid_incl[i] - 1;
    const unsigned long long k = keys[i];
    const int sst = (int)((keys[seg[i]] >> 3) & 127u);
    const int s = (int)((k >> 3) & 127u);
    const int r = (int)(k & 7u);
    const int w0 = sst + ((s - sst) & ~3);
    tiles[t].v[r * 4 + (s - w0)] = data[ids[i]];
    if (i == 0 || tid_incl[i - 1] != tid_incl[i]) {
      const unsigned long long jl = k >> 10;
      tiles[t].l = (int32_t)(jl % (unsigned long long)V);
      tiles[t].s0 = w0;
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

// per-plan view: the records whose 4-lag window meets the plan's active positions
__device__ __forceinline__ unsigned act4_g(const unsigned* act, int s0) {
  const int w = s0 >> 5, b = s0 & 31;
  const unsigned long long v = ((unsigned long long)act[w + 1] << 32) | act[w];
  return (unsigned)(v >> b) & 0xFu;
}

// time tiles t of the plan holding a valid block row for the window's lags:
// ceil((dt0 + s0 - 7) / 8) <= t <= floor((dt1 + s0 + 3) / 8), clipped to [0, nT)
__device__ __forceinline__ void band_trange(int dt0, int dt1, int nT, int s0, int& lo, int& hi) {
  lo = max(0, (dt0 + s0 + 8 * 1024) / 8 - 1024);
  hi = min(nT - 1, (dt1 + s0 + 3 + 8 * 1024) / 8 - 1024);
}

__global__ void k_band_flag(const BandTile* __restrict__ tiles, long long n, const unsigned* __restrict__ act, int dt0,
                            int dt1, int nT, int* __restrict__ flag) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    const int s0 = tiles[t].s0;
    int lo, hi;
    band_trange(dt0, dt1, nT, s0, lo, hi);
    flag[t] = act4_g(act, s0) != 0u && lo <= hi;
  }
}

// the view's record: A values of lags outside the plan zeroed, the plan's valid time-tile
// range in the header (pad0 = lo | hi << 8), so the kernel does no per-tile mask work
__global__ void k_band_scatter(const BandTile* __restrict__ tiles, long long n, const int* __restrict__ flag,
                               const long long* __restrict__ pos, const unsigned* __restrict__ act, int dt0, int dt1,
                               int nT, BandTile* __restrict__ out) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    if (!flag[t]) continue;
    BandTile r = tiles[t];
    const unsigned c = act4_g(act, r.s0);
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (!((c >> (i & 3)) & 1u)) r.v[i] = 0.0;
    int lo, hi;
    band_trange(dt0, dt1, nT, r.s0, lo, hi);
    r.pad0 = lo | (hi << 8);
    out[pos[t]] = r;
  }
}

__global__ void k_band_rbview(const int64_t* __restrict__ rbptr, int nRB, const long long* __restrict__ pos,
                              int64_t* __restrict__ out) {
  for (int J = blockIdx.x * blockDim.x + threadIdx.x; J <= nRB; J += gridDim.x * blockDim.x) out[J] = pos[rbptr[J]];
}

__global__ void k_flag_to_ll(const int* __restrict__ f, long long n, long long* __restrict__ o) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t <= n; t += (long long)gridDim.x * blockDim.x)
    o[t] = t < n ? f[t] : 0;
}

struct MaxLL {
  __device__ __forceinline__ long long operator()(long long a, long long b) const { return a > b ? a : b; }
};

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// active-lag bits of positions s0 .. s0 + 3
__device__ __forceinline__ unsigned act4(const unsigned* act, int s0) {
  const int w = s0 >> 5, b = s0 & 31;
  const unsigned long long v = ((unsigned long long)act[w + 1] << 32) | act[w];
  return (unsigned)(v >> b) & 0xFu;
}

// One CTA = (row block J, part); warp w owns time tiles [w TT, w TT + TT).  Tile
// records arrive in shared memory by bulk copy (kBandStages-deep ring); two tiles
// per step, both tiles' B loads issued before their DMMAs; time tiles without a
// valid row for the tile's lags (the Toeplitz triangle) are skipped.
template <int TT>
__global__ void __launch_bounds__(kBandMaxWarps * 32) k_band_mv(BandMvArgs a) {
  extern __shared__ __align__(128) unsigned char bm_smem[];
  const int CH = a.chunk;  // tile records per stage
  BandTile* stg = reinterpret_cast<BandTile*>(bm_smem);  // [kBandStages][CH]
  unsigned long long* full = reinterpret_cast<unsigned long long*>(stg + kBandStages * CH);
  unsigned long long* empty = full + kBandStages;
  unsigned* act = reinterpret_cast<unsigned*>(empty + kBandStages);  // [act_words + 1]
  unsigned* irr = act + a.act_words + 1;                              // [kIrrWords]
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (int i = tid; i <= a.act_words; i += blockDim.x) act[i] = i < a.act_words ? __ldg(a.s_act + i) : 0u;
  for (int i = tid; i < kIrrWords; i += blockDim.x) irr[i] = a.irr_mask[i];
  const int J = blockIdx.x / a.P, part = blockIdx.x % a.P;
  const long long r0 = __ldg(a.rbptr + J), r1 = __ldg(a.rbptr + J + 1);
  const long long q0 = r0 + (r1 - r0) * part / a.P, q1 = r0 + (r1 - r0) * (part + 1) / a.P;
  const int nchunks = (int)((q1 - q0 + CH - 1) / CH);
  if (tid == 0) {
    for (int i = 0; i < kBandStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], a.W);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (tid == 0)
    for (int c = 0; c < min(kBandStages, nchunks); ++c) {
      const long long qb = q0 + (long long)c * CH;
      const unsigned bytes = (unsigned)(min((long long)CH, q1 - qb) * sizeof(BandTile));
      mbar_arrive_expect_tx(&full[c], bytes);
      bulk_g2s(stg + c * CH, a.tiles + qb, bytes, &full[c]);
    }
  const int g = lane >> 2, k = lane & 3;
  // warp w owns the contiguous time tiles t = t0 + u (adjacent B windows share L1 sectors)
  const int t0 = w * TT;
  double acc[TT][2];
#pragma unroll
  for (int u = 0; u < TT; ++u) acc[u][0] = acc[u][1] = 0.0;
  const double* xl = a.xt + (a.off0 - k + g + 8 * t0);
  // one pair of tile records: header, A fragments (masked by the plan's lags), B windows
  struct PairRegs {
    int lo1, hi1, lo2, hi2;
    double av1, av2;
    double b1[TT], b2[TT];
  };
  auto load_pair = [&](const BandTile* T, int i, int n, PairRegs& R) {
    const bool two = i + 1 < n;
    const int4 h1 = *reinterpret_cast<const int4*>(&T[i].l);
    const int4 h2 = two ? *reinterpret_cast<const int4*>(&T[i + 1].l) : h1;
    const int l1 = h1.x, s1 = h1.y, l2 = h2.x, s2 = h2.y;
    // valid time tiles of the record for this plan (baked into the view's header)
    R.lo1 = (h1.z & 0xff) - t0;
    R.hi1 = (h1.z >> 8) - t0;
    R.lo2 = (h2.z & 0xff) - t0;
    R.hi2 = two ? (h2.z >> 8) - t0 : -1;
    R.av1 = T[i].v[lane];
    R.av2 = two ? T[i + 1].v[lane] : 0.0;
    const double* x1 = xl + (long long)l1 * a.xs - s1;
    const double* x2 = xl + (long long)l2 * a.xs - s2;
#pragma unroll
    for (int u = 0; u < TT; ++u) {
      R.b1[u] = __ldg(x1 + 8 * u);
      R.b2[u] = __ldg(x2 + 8 * u);
    }
    // the light-cone tie lag: only the block rows of its logical mask (per lane / row)
    if (a.s_irr >= s1 && a.s_irr < s1 + 4 && k == a.s_irr - s1) {
#pragma unroll
      for (int u = 0; u < TT; ++u) {
        const int r = 8 * (t0 + u) + g;
        if (!((irr[r >> 5] >> (r & 31)) & 1u)) R.b1[u] = 0.0;
      }
    }
    if (a.s_irr >= s2 && a.s_irr < s2 + 4 && k == a.s_irr - s2) {
#pragma unroll
      for (int u = 0; u < TT; ++u) {
        const int r = 8 * (t0 + u) + g;
        if (!((irr[r >> 5] >> (r & 31)) & 1u)) R.b2[u] = 0.0;
      }
    }
  };
  auto mma_pair = [&](const PairRegs& R) {
#pragma unroll
    for (int u = 0; u < TT; ++u)
      if (u >= R.lo1 && u <= R.hi1) dmma884(acc[u][0], acc[u][1], R.av1, R.b1[u]);
#pragma unroll
    for (int u = 0; u < TT; ++u)
      if (u >= R.lo2 && u <= R.hi2) dmma884(acc[u][0], acc[u][1], R.av2, R.b2[u]);
  };
  for (int c = 0; c < nchunks; ++c) {
    const int st = c % kBandStages;
    const unsigned ph = (unsigned)(c / kBandStages) & 1u;
    mbar_wait(&full[st], ph);
    const BandTile* T = stg + st * CH;
    const int n = (int)min((long long)CH, q1 - (q0 + (long long)c * CH));
    // software pipeline: the next pair's loads are in flight during this pair's DMMAs
    PairRegs RA, RB;
    load_pair(T, 0, n, RA);
    for (int i = 0; i < n; i += 4) {
      if (i + 2 < n) load_pair(T, i + 2, n, RB);
      mma_pair(RA);
      if (i + 2 >= n) break;
      if (i + 4 < n) load_pair(T, i + 4, n, RA);
      mma_pair(RB);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    if (tid == 0 && c + kBandStages < nchunks) {  // refill this stage once every warp released it
      mbar_wait(&empty[st], ph);
      const long long qb = q0 + (long long)(c + kBandStages) * CH;
      const unsigned bytes = (unsigned)(min((long long)CH, q1 - qb) * sizeof(BandTile));
      mbar_arrive_expect_tx(&full[st], bytes);
      bulk_g2s(stg + st * CH, a.tiles + qb, bytes, &full[st]);
    }
  }
  // partial tile rows of this part: ypart[part][8 J + g][8 (t0 + u) + 2 k + {0, 1}]
  double* yp = a.ypart + ((long long)part * a.nRB * 8 + 8LL * J + g) * a.ldy + 8 * t0 + 2 * k;
#pragma unroll
  for (int u = 0; u < TT; ++u)
    if (t0 + u < a.nT) *reinterpret_cast<double2*>(yp + 8 * u) = make_double2(acc[u][0], acc[u][1]);
}

// Direct variant: a unit = (row block J, part) is W adjacent warps, each covering TT of
// the time tiles; every warp reads the unit's records straight from global memory
// (coalesced 256-byte A fragment + broadcast header; the other warps of the unit hit
// L1), the next step's records prefetched during this step's B loads and DMMAs.  No
// shared-memory ring, no barriers.  Same DMMA sequence per accumulator as k_band_mv<TT>.
#ifndef TDB_DIRECT_UNROLL
#define TDB_DIRECT_UNROLL 3
#endif
constexpr int kDirectWarps = 8;   // warps per CTA: 8 / W units of W warps (W = 1, 2, 4, 8 time groups)
constexpr int kDirectUnroll = TDB_DIRECT_UNROLL;  // records per step (the next step's are prefetched)
template <int TT>
__global__ void __launch_bounds__(kDirectWarps * 32) k_band_direct(BandMvArgs a) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // the W warps of a unit (adjacent in the CTA) read the same records (L1) for their own time tiles
  const long long unit = (long long)blockIdx.x * (kDirectWarps / a.W) + wid / a.W;
  const int t0 = (wid % a.W) * TT;
  if (unit >= (long long)a.nRB * a.P) return;
  const int J = (int)(unit / a.P), part = (int)(unit % a.P);
  const long long r0 = __ldg(a.rbptr + J), r1 = __ldg(a.rbptr + J + 1);
  const long long q0 = r0 + (r1 - r0) * part / a.P, q1 = r0 + (r1 - r0) * (part + 1) / a.P;
  const int g = lane >> 2, k = lane & 3;
  double acc[TT][2];
#pragma unroll
  for (int u = 0; u < TT; ++u) acc[u][0] = acc[u][1] = 0.0;
  const double* xl = a.xt + (a.off0 - k + g + 8 * t0);
  // software pipeline: the next batch's headers and A fragments are in flight during this
  // batch's B loads and DMMAs
  int4 hn[kDirectUnroll];
  double an[kDirectUnroll];
  auto fetch = [&](long long i) {
#pragma unroll
    for (int v = 0; v < kDirectUnroll; ++v) {
      const BandTile* T = a.tiles + (i + v < q1 ? i + v : q1 - 1);
      hn[v] = __ldg(reinterpret_cast<const int4*>(&T->l));
      an[v] = __ldg(&T->v[lane]);
    }
  };
  if (q0 < q1) fetch(q0);
  for (long long i = q0; i < q1; i += kDirectUnroll) {
    int lo[kDirectUnroll], hi[kDirectUnroll];
    double av[kDirectUnroll], b[kDirectUnroll][TT];
#pragma unroll
    for (int v = 0; v < kDirectUnroll; ++v) {
      const int4 h = hn[v];
      lo[v] = (h.z & 0xff) - t0;
      hi[v] = i + v < q1 ? (h.z >> 8) - t0 : -1;
      av[v] = an[v];
      const double* x = xl + (long long)h.x * a.xs - h.y;
#pragma unroll
      for (int u = 0; u < TT; ++u) b[v][u] = __ldg(x + 8 * u);
      // the light-cone tie lag: only the block rows of its logical mask (per lane / row)
      if (a.s_irr >= h.y && a.s_irr < h.y + 4) {  // warp-uniform
        if (k == a.s_irr - h.y) {
#pragma unroll
          for (int u = 0; u < TT; ++u) {
            const int r = 8 * (t0 + u) + g;
            if (!((a.irr_mask[r >> 5] >> (r & 31)) & 1u)) b[v][u] = 0.0;
          }
        }
      }
    }
    if (i + kDirectUnroll < q1) fetch(i + kDirectUnroll);
#pragma unroll
    for (int v = 0; v < kDirectUnroll; ++v)
#pragma unroll
      for (int u = 0; u < TT; ++u)
        if (u >= lo[v] && u <= hi[v]) dmma884(acc[u][0], acc[u][1], av[v], b[v][u]);
  }
  double* yp = a.ypart + ((long long)part * a.nRB * 8 + 8LL * J + g) * a.ldy + 8 * t0 + 2 * k;
#pragma unroll
  for (int u = 0; u < TT; ++u)
    if (t0 + u < a.nT) *reinterpret_cast<double2*>(yp + 8 * u) = make_double2(acc[u][0], acc[u][1]);
}

template <int TT>
int launch_direct(const BandMvArgs& a, cudaStream_t st) {
  const long long units = (long long)a.nRB * a.P, per_cta = kDirectWarps / a.W;
  k_band_direct<TT><<<(unsigned)((units + per_cta - 1) / per_cta), kDirectWarps * 32, 0, st>>>(a);
  TDB_CUDA_CHECK(cudaGetLastError());
  return TDB_OK;
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
  const size_t smem = band_smem_bytes(a.act_words, a.chunk);
  if (smem > 48 * 1024)
    TDB_CUDA_CHECK(cudaFuncSetAttribute(k_band_mv<TT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_band_mv<TT><<<(unsigned)((long long)a.nRB * a.P), a.W * 32, smem, st>>>(a);
  TDB_CUDA_CHECK(cudaGetLastError());
  return TDB_OK;
}

}  // namespace

size_t band_smem_bytes(int act_words, int chunk) {
  return (size_t)kBandStages * chunk * sizeof(BandTile) + 2 * kBandStages * sizeof(unsigned long long) +
         (size_t)(act_words + 1 + kIrrWords) * sizeof(unsigned);
}

int band_build(TdbSystem* sys, int f) {
  if ((int)sys->band.size() != sys->F) sys->band.assign(sys->F, BandStore{});
  BandStore& b = sys->band[f];
  if (b.built) return TDB_OK;
  if (b.failed) {
    set_error("band tiles: an earlier build of this family failed");
    return TDB_E_NOMEM;
  }
  TDB_REQUIRE(sys->p == 0, "band tiles: built for p = 0 only");
  FamilyStore& fs = sys->fam[f];
  TDB_REQUIRE(fs.npos <= 124, "band tiles: at most 124 positions per family");
  cudaStream_t st = sys->ctx->stream;
  const int NR = sys->nrows, nRB = sys->nRB, V = (int)sys->V;
  const long long n = fs.nnz;
  unsigned long long *k0 = nullptr, *k1 = nullptr;
  long long *i0 = nullptr, *i1 = nullptr, *seg = nullptr;
  int *head = nullptr, *tile_rb = nullptr;
  void* tmp = nullptr;
  auto release = [&]() {
    dev_free(k0);
    dev_free(k1);
    dev_free(i0);
    dev_free(i1);
    dev_free(seg);
    dev_free(head);
    dev_free(tile_rb);
    dev_free(tmp);
    k0 = k1 = nullptr;
    i0 = i1 = seg = nullptr;
    head = tile_rb = nullptr;
    tmp = nullptr;
  };
  auto fail = [&](cudaError_t e) {
    release();
    dev_free(b.rbptr);
    dev_free(b.tiles);
    b.rbptr = nullptr;
    b.tiles = nullptr;
    b.failed = true;  // sticky: later plans go straight to CSR without retrying
    set_error(std::string("band tiles build: ") + cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? TDB_E_NOMEM : TDB_E_CUDA;
  };
#define TRY(expr)                           \
  do {                                      \
    cudaError_t e_ = (expr);                \
    if (e_ != cudaSuccess) return fail(e_); \
  } while (0)
  TRY(dev_malloc((void**)&b.rbptr, (size_t)(nRB + 1) * sizeof(int64_t)));
  if (n == 0) {
    TRY(cudaMemsetAsync(b.rbptr, 0, (size_t)(nRB + 1) * sizeof(int64_t), st));
    TRY(dev_malloc((void**)&b.tiles, sizeof(BandTile)));
    TRY(cudaStreamSynchronize(st));
    b.built = true;
    return TDB_OK;
  }
  TRY(dev_malloc((void**)&k0, n * sizeof(unsigned long long)));
  TRY(dev_malloc((void**)&k1, n * sizeof(unsigned long long)));
  TRY(dev_malloc((void**)&i0, n * sizeof(long long)));
  TRY(dev_malloc((void**)&i1, n * sizeof(long long)));
  TRY(dev_malloc((void**)&seg, n * sizeof(long long)));
  TRY(dev_malloc((void**)&head, n * sizeof(int)));
  k_band_keys<<<148 * 16, 256, 0, st>>>(fs.indptr, fs.indices, (long long)fs.npos * NR, NR, V, sys->d_rinv, k0, i0);
  TRY(cudaGetLastError());
  int end_bit = 10;
  {
    const unsigned long long maxjl = (unsigned long long)nRB * (unsigned long long)V;
    while (end_bit < 64 && (maxjl >> (end_bit - 10)) != 0) ++end_bit;
  }
  size_t tb = 0, tb2 = 0, tb3 = 0;
  TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb, k0, k1, i0, i1, n, 0, end_bit, st));
  TRY(cub::DeviceScan::InclusiveSum(nullptr, tb2, head, head, n, st));
  TRY(cub::DeviceScan::InclusiveScan(nullptr, tb3, seg, seg, MaxLL(), n, st));
  TRY(dev_malloc(&tmp, std::max(tb, std::max(tb2, tb3))));
  TRY(cub::DeviceRadixSort::SortPairs(tmp, tb, k0, k1, i0, i1, n, 0, end_bit, st));
  k_band_seg<<<148 * 16, 256, 0, st>>>(k1, n, seg);
  TRY(cudaGetLastError());
  TRY(cub::DeviceScan::InclusiveScan(tmp, tb3, seg, seg, MaxLL(), n, st));
  k_band_heads<<<148 * 16, 256, 0, st>>>(k1, seg, n, head);
  TRY(cudaGetLastError());
  TRY(cub::DeviceScan::InclusiveSum(tmp, tb2, head, head, n, st));
  int nt = 0;
  TRY(cudaMemcpyAsync(&nt, head + n - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  TRY(cudaStreamSynchronize(st));
  b.ntiles = nt;
  b.nnz = n;
  TRY(dev_malloc((void**)&b.tiles, (size_t)nt * sizeof(BandTile)));
  TRY(dev_malloc((void**)&tile_rb, (size_t)nt * sizeof(int)));
  TRY(cudaMemsetAsync(b.tiles, 0, (size_t)nt * sizeof(BandTile), st));
  k_band_fill<<<148 * 16, 256, 0, st>>>(k1, i1, seg, head, n, V, fs.data, b.tiles, tile_rb);
  TRY(cudaGetLastError());
  k_band_rbptr<<<(nRB + 256) / 256, 256, 0, st>>>(tile_rb, nt, nRB, b.rbptr);
  TRY(cudaGetLastError());
  TRY(cudaStreamSynchronize(st));
  release();
#undef TRY
  b.built = true;
  return TDB_OK;
}

// Records of family f restricted to the active positions `act` (bit s set: position s is
// a band term), order kept; cached per active set (the recursive preconditioner reuses a
// handful of ranges).  A quarter-range plan then streams only its lags' records.
int band_view(TdbSystem* sys, int f, const std::vector<unsigned>& act, int dt0, int dt1, int nT,
              const BandTile** tiles, const int64_t** rbptr, long long* ntiles) {
  BandStore& b = sys->band[f];
  for (const BandView& v : b.views)
    if (v.act == act && v.dt0 == dt0 && v.dt1 == dt1 && v.nT == nT) {
      *ntiles = v.ntiles;
      *tiles = v.tiles;
      *rbptr = v.rbptr;
      return TDB_OK;
    }
  cudaStream_t st = sys->ctx->stream;
  const long long n = b.ntiles;
  const int nRB = sys->nRB;
  BandView v;
  v.act = act;
  v.dt0 = dt0;
  v.dt1 = dt1;
  v.nT = nT;
  int* flag = nullptr;
  long long* pos = nullptr;
  unsigned* dact = nullptr;
  void* tmp = nullptr;
  size_t tb = 0;
  auto release = [&]() {
    dev_free(flag);
    dev_free(pos);
    dev_free(dact);
    dev_free(tmp);
  };
#define TRY(expr)                                                            \
  do {                                                                       \
    cudaError_t e_ = (expr);                                                 \
    if (e_ != cudaSuccess) {                                                 \
      release();                                                             \
      dev_free(v.tiles);                                                     \
      dev_free(v.rbptr);                                                     \
      set_error(std::string("band view: ") + cudaGetErrorString(e_));        \
      return e_ == cudaErrorMemoryAllocation ? TDB_E_NOMEM : TDB_E_CUDA;     \
    }                                                                        \
  } while (0)
  TRY(dev_malloc((void**)&flag, (size_t)std::max(1LL, n) * sizeof(int)));
  TRY(dev_malloc((void**)&pos, (size_t)(n + 1) * sizeof(long long)));
  TRY(dev_malloc((void**)&dact, act.size() * sizeof(unsigned)));
  TRY(cudaMemcpyAsync(dact, act.data(), act.size() * sizeof(unsigned), cudaMemcpyHostToDevice, st));
  if (n > 0) {
    k_band_flag<<<148 * 8, 256, 0, st>>>(b.tiles, n, dact, dt0, dt1, nT, flag);
    TRY(cudaGetLastError());
  }
  k_flag_to_ll<<<148 * 8, 256, 0, st>>>(flag, n, pos);
  TRY(cudaGetLastError());
  TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb, pos, pos, n + 1, st));
  TRY(dev_malloc(&tmp, tb));
  TRY(cub::DeviceScan::ExclusiveSum(tmp, tb, pos, pos, n + 1, st));
  long long nsel = 0;
  TRY(cudaMemcpyAsync(&nsel, pos + n, sizeof(long long), cudaMemcpyDeviceToHost, st));
  TRY(cudaStreamSynchronize(st));
  TRY(dev_malloc((void**)&v.tiles, (size_t)std::max(1LL, nsel) * sizeof(BandTile)));
  TRY(dev_malloc((void**)&v.rbptr, (size_t)(nRB + 1) * sizeof(int64_t)));
  if (n > 0) {
    k_band_scatter<<<148 * 8, 256, 0, st>>>(b.tiles, n, flag, pos, dact, dt0, dt1, nT, v.tiles);
    TRY(cudaGetLastError());
  }
  k_band_rbview<<<(nRB + 256) / 256, 256, 0, st>>>(b.rbptr, nRB, pos, v.rbptr);
  TRY(cudaGetLastError());
  TRY(cudaStreamSynchronize(st));
  release();
#undef TRY
  v.ntiles = nsel;
  b.views.push_back(v);
  *tiles = v.tiles;
  *rbptr = v.rbptr;
  *ntiles = nsel;
  return TDB_OK;
}

int band_mv_tiles(const BandMvArgs& a, cudaStream_t st) {
  if (a.direct) {  // W in {1, 2, 4, 8}, TT <= 6
    switch (a.TT) {
      case 1: return launch_direct<1>(a, st);
      case 2: return launch_direct<2>(a, st);
      case 3: return launch_direct<3>(a, st);
      case 4: return launch_direct<4>(a, st);
      case 5: return launch_direct<5>(a, st);
      default: return launch_direct<6>(a, st);
    }
  }
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
