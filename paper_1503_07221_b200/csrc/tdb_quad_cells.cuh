// Regular (non-touching) pairs: "cell owner" quadrature.  Included by
// tdb_assembly.cu after k_quad (uses its QuadArgs / QFam / reduce-scatter).
//
// Same integrand, rule points and table arithmetic as k_quad (the reference's
// pair_block_contributions, _core.pyx:47-159, summed per pair and position), but the
// work is laid out around the table instead of around the position:
//
//   * k_quad gathers one coefficient row per (point, position) evaluation from shared
//     memory, ~180 B per evaluation: the LSU return path (128 B/clk/SM) runs at 75%
//     while the FP64 pipe idles at 32% (profiles/r02/ncu_quad_cfg4_r02d_summary.txt).
//   * Every table of a family lives on a dt-aligned grid of C = 32 cells per time step
//     and the positions of a family are one time step apart, so a rule point at
//     distance r sits in the same cell column j = floor(32 frac(r / dt)) at every
//     position, one dt-span of the table support further per lag.
//   * The pair's 256 points are sorted by column and cut into column-pure sub-runs of 5.
//     Per dt span m of the support, every lane takes one sub-run, loads the coefficient
//     row of its cell (m, j) into REGISTERS once and evaluates its 5 points against it
//     (position s = floor(r / dt) + kappa - m).  Per evaluation the LSU delivers the
//     point (12 B), the position's table offset (8 B), a fifth of a coefficient row
//     (~40 B) and takes the two table values (16 B) instead of a 180 B row.
//   * The values land in G[m][q] (q = rule point).  The regular rule is the tensor
//     product of a 16-point triangle rule with itself, so the shape products are
//     contracted per unit as shy_a * sum_ix (c g0)[ix, iy] shx_b[ix]: lane = (iy, half
//     of ix), 8 fused multiply-adds per table per lane, four units per step; the warp sum
//     exchanges whole register sets in its first two levels (set u of a lane holds unit
//     si + (u ^ lane bits 4-3): no selects) and ends with an 8-lane reduce-scatter.
//     Summation order differs from k_quad's r-sorted order (deterministic, fixed per lane,
//     independent of the pair's position window); everything else is the same arithmetic.
//
// Families that do not fit this grid (p > 0, a different cell count, non-uniform lags,
// table values that do not vanish at the support ends) and the singular cases stay on
// k_quad (QuadArgs::cell_mask tells it which (regular pair, family) work is done here).
#pragma once

constexpr int kCellWarps = 8;
constexpr int kCellSpans = 4;   // dt spans of a table support (passes per family), max
constexpr int kCellPerDt = 32;  // table cells per time step
// The pair's points are sorted by cell column and cut into column-pure sub-runs of
// kCellSub (columns padded to a multiple of it): at most (256 + 4 * 32) / 5 = 76
// sub-runs, kept transposed ([entry][sub-run], consecutive lanes read consecutive words).
// Measured at config 4 (k_quad_cells ms): 4 -> 641, 5 -> 624, 6 -> 641, 8 -> 797: the time
// follows the evaluation slots per lane (rounds x kCellSub: 12, 11.8, 12, 16).
#ifndef TDB_CELL_SUB
#define TDB_CELL_SUB 5
#endif
constexpr int kCellSub = TDB_CELL_SUB;
constexpr int kCellSubRuns = (kChunk + (kCellSub - 1) * 32) / kCellSub + 1;
// per-warp scratch: sorted r (FP64), sorted q | column << 8 | n << 13, G[span][q] = (psi, psi~), counters
constexpr int kCellScratchBytes = (kCellSub * kCellSubRuns * 12 + kCellSpans * kChunk * 16 + 32 * 4 + 15) / 16 * 16;
static_assert(kChunk == 256, "the cell-owner kernel packs the rule point index in 8 bits");

// Coefficient rows of the cell-owner launch: one 16-byte aligned record per table cell,
// [7 x (psi, psi~) FP64 head][D - 6 x (psi, psi~) FP32 tail][pad], an odd number of
// 16-byte words (rows of neighbouring cells start in different bank groups).
__host__ __device__ constexpr int cell_row_words(int D) { return (7 + (D - 6 + 1) / 2) | 1; }

template <int D>
struct CellRow {
  double2 a[7];
  float2 b[D - 6];
  double roww;
  __device__ __forceinline__ void load(const double2* __restrict__ rows, int row, double w) {
    const double2* p = rows + row * cell_row_words(D);
#pragma unroll
    for (int k = 0; k < 7; ++k) a[k] = p[k];
#pragma unroll
    for (int k = 0; k < (D - 6) / 2; ++k) {
      const double2 t = p[7 + k];
      b[2 * k] = make_float2(__int_as_float(__double2loint(t.x)), __int_as_float(__double2hiint(t.x)));
      b[2 * k + 1] = make_float2(__int_as_float(__double2loint(t.y)), __int_as_float(__double2hiint(t.y)));
    }
    roww = (double)row * w;
  }
};

// (psi, psi~) of one table pair from register-resident coefficients: the arithmetic of
// eval_pair<2, ., D, 7> (Estrin FP64 head, packed FP32 Horner tail).
template <int D>
__device__ __forceinline__ void cell_poly(const CellRow<D>& c, double x, double& v0, double& v1) {
  const double2(&a)[7] = c.a;
  const double x2 = x * x, x4 = x2 * x2;
  const double qa0 = fma(a[1].x, x, a[0].x), qa1 = fma(a[3].x, x, a[2].x), qa2 = fma(a[5].x, x, a[4].x);
  const double qb0 = fma(a[1].y, x, a[0].y), qb1 = fma(a[3].y, x, a[2].y), qb2 = fma(a[5].y, x, a[4].y);
  const double ra0 = fma(qa1, x2, qa0), ra1 = fma(a[6].x, x2, qa2);
  const double rb0 = fma(qb1, x2, qb0), rb1 = fma(a[6].y, x2, qb2);
  v0 = fma(ra1, x4, ra0);
  v1 = fma(rb1, x4, rb0);
  const float xf = (float)x;
  const float2 xx = make_float2(xf, xf);
  float2 tt = c.b[D - 7];
#pragma unroll
  for (int k = D - 8; k >= 0; --k) tt = ffma2(tt, xx, c.b[k]);
  const double x7 = x4 * x2 * x;
  v0 = fma(x7, (double)tt.x, v0);
  v1 = fma(x7, (double)tt.y, v1);
}

// Family constants of stage 1 (warp-uniform).
struct CellFam {
  double amin, amax, lo, inv_w2;  // inv_w2 = 2 / w
  int abs_mask;        // |a| as a mask on the high word (fold families)
  unsigned sp1, sn1;   // sign bit of the tables for a >= 0 / a < 0
};

// NE points of one sub-run (entries e0 .. e0 + NE - 1) against the row in `cr`.
template <int D, int NE>
__device__ __forceinline__ void cell_evals(const CellFam& cf, const CellRow<D>& cr, const double* __restrict__ sdel,
                                           const double* __restrict__ s_r, const int* __restrict__ s_q,
                                           double2* __restrict__ Gm, int u, int e0, bool live, int koff,
                                           unsigned ucnt, int sg, unsigned& n_act) {
  double r[NE], delta[NE];
  int qi[NE];
  bool valid[NE];
#pragma unroll
  for (int i = 0; i < NE; ++i) {
    r[i] = s_r[(e0 + i) * kCellSubRuns + u];
    qi[i] = live ? s_q[(e0 + i) * kCellSubRuns + u] : (int)0x80000000u;  // idle lanes: like a pad entry
  }
#pragma unroll
  for (int i = 0; i < NE; ++i) {
    const unsigned sr = (unsigned)((qi[i] >> 13) + koff);  // position relative to the pair's window
    valid[i] = sr < ucnt;
    delta[i] = sdel[valid[i] ? sr : 0u];
  }
#pragma unroll
  for (int i = 0; i < NE; ++i) {
    const double av = r[i] + delta[i];
    const bool act = valid[i] && av >= cf.amin && av <= cf.amax;
    n_act += act ? 1u : 0u;
    const int avh = __double2hiint(av);
    const double aa = __hiloint2double(avh & cf.abs_mask, __double2loint(av));
    // cheb_locate's local coordinate with the sub-run's row for idx (equal to it except
    // within roundoff of a cell edge, where the two pieces agree to 1e-16)
    // (2 t) inv_w - 1 == fma(t, 2 inv_w, -1) bit for bit (the doubling is exact)
    const double x = fma(aa - cf.lo - cr.roww, cf.inv_w2, -1.0);
    double v0, v1;
    cell_poly<D>(cr, x, v0, v1);
    v0 = __hiloint2double(__double2hiint(v0) ^ sg, __double2loint(v0));
    v1 = __hiloint2double(__double2hiint(v1) ^ sg, __double2loint(v1));
    // two predicated stores (measured 2% faster than selecting the values first)
    if (qi[i] >= 0) {
      double2* g = Gm + (qi[i] & 255);
      if (act) *g = make_double2(v0, v1);
      else *g = make_double2(0.0, 0.0);
    }
  }
}

// Stage 1 of one family: per dt span m of the support, round by round every lane takes
// one column-pure sub-run of points, loads the coefficient row of its (span, column)
// cell into registers and evaluates its points against it (independent evaluations,
// interleaved by the compiler: the kernel runs two warps per scheduler and lives on
// instruction-level parallelism).
template <int D>
__device__ __forceinline__ void cell_family(const QFam& fd, const double2* __restrict__ rows,
                                            const double* __restrict__ sdel, const double* __restrict__ s_r,
                                            const int* __restrict__ s_q, double2* __restrict__ G, int nsr,
                                            int lane, int w_lo, unsigned ucnt, double dt, int n_min, int n_max,
                                            unsigned& n_act) {
  CellFam cf;
  cf.amin = fd.amin;
  cf.amax = fd.amax;
  cf.lo = fd.lo;
  cf.inv_w2 = 2.0 * fd.inv_w;
  const double w = fd.w;
  const int nsub = fd.nsub, nspan = fd.cell_M;
  const bool fold = fd.fold != 0;
  cf.abs_mask = fold ? 0x7fffffff : -1;
  cf.sp1 = (fd.sp_neg & 1u) << 31;
  cf.sn1 = (fd.sn_neg & 1u) << 31;
  for (int m = 0; m < nspan; ++m) {
    const int koff = fd.cell_kappa - m - w_lo;
    // no point of the pair has its span-m position inside the window (position batches,
    // lag-sharded systems): nothing of this span is read by stage 2
    if (n_max + koff < 0 || n_min + koff >= (int)ucnt) continue;
    double2* Gm = G + m * kChunk;
    // sign of the tables on this span (a < 0 on the spans below zero; where a span meets
    // a = 0 the two signs differ only for an odd table, which vanishes there)
    const int sg = (int)(cf.amin + ((double)m + 0.5) * dt < 0.0 ? cf.sn1 : cf.sp1);
#pragma unroll 1
    for (int u0 = 0; u0 < nsr; u0 += 32) {
      // a last round of at most 6 sub-runs (a third of the pairs end on 1-2 of them) is
      // spread one point per lane instead of one sub-run per lane
      const bool wide = u0 > 0 && nsr - u0 <= 32 / kCellSub;  // warp-uniform
      const int mine = wide ? u0 + lane / kCellSub : u0 + lane;
      const bool live = mine < nsr;
      const int u = live ? mine : 0;
      CellRow<D> cr;
      {
        const int c = m * kCellPerDt + ((s_q[u] >> 8) & 31);  // cell on the a axis, from amin
        cr.load(rows, fold ? (c < nsub ? nsub - 1 - c : c - nsub) : c, w);
      }
      if (wide)
        cell_evals<D, 1>(cf, cr, sdel, s_r, s_q, Gm, u, lane % kCellSub, live, koff, ucnt, sg, n_act);
      else
        cell_evals<D, kCellSub>(cf, cr, sdel, s_r, s_q, Gm, u, 0, live, koff, ucnt, sg, n_act);
    }
  }
}

__global__ void __launch_bounds__(kCellWarps * 32, 1) k_quad_cells(QuadArgs a) {
  constexpr int NACC = 10;
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ __align__(16) double smem[];
  double* sblob = smem;
  double* sdelta = sblob + (a.blob_doubles + 1) / 2 * 2;
  char* swarp = reinterpret_cast<char*>(sdelta + (a.delta_doubles + 1) / 2 * 2);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  char* mine = swarp + (size_t)wid * kCellScratchBytes;
  double2* G = reinterpret_cast<double2*>(mine);
  double* s_r = reinterpret_cast<double*>(G + kCellSpans * kChunk);
  int* s_q = reinterpret_cast<int*>(s_r + kCellSub * kCellSubRuns);
  unsigned* bins = reinterpret_cast<unsigned*>(s_q + kCellSub * kCellSubRuns);
  for (int i = threadIdx.x; i < a.blob_doubles; i += blockDim.x) sblob[i] = a.blob[i];
  for (int fi = 0; fi < a.fam_count; ++fi)
    for (int i = threadIdx.x; i < a.fam[fi].npos; i += blockDim.x)
      sdelta[a.fam[fi].delta_off + i] = a.fam[fi].delta[i];
  __syncthreads();

  // rule constants of this lane's points q = lane + 32 k: x index 2 k + (lane >> 4), y index lane & 15
  const RuleDev& R = a.rules[0];
  const double y1 = R.y1[lane], y2 = R.y2[lane];
  const double shy0 = 1.0 - y1, shy1 = y1 - y2, shy2 = y2;

  const unsigned E = (unsigned)a.E;
  const long long E2 = a.npair;
  const double inv_dt = a.inv_dt;
  unsigned long long my_in = 0, my_pairs = 0;

  // pair index two ahead, pair header (corners, plan entries) one ahead of the work
  struct Header {
    double d;  // lanes 0-8 / 9-17: corners of ex / ey, 18 / 19: twice their areas
    FRange fr;
    int units, cs;
    long long base;
  };
  auto grab = [&]() {
    long long v = 0;
    if (lane == 0) v = (long long)atomicAdd(a.work, 1ULL);
    return __shfl_sync(FULL, v, 0);
  };
  auto load_header = [&](long long Pp, Header& h) {
    h.d = 0.0;
    h.fr = FRange{0, 0};
    h.units = 0;
    h.cs = 0;
    h.base = 0;
    if (Pp < E2) {
      h.units = a.units[Pp];
      h.cs = a.pcase[Pp];
      h.base = a.pair_base[Pp];
      const unsigned ex = (unsigned)Pp % E;
      const int ey = a.tt[(unsigned)Pp / E];
      if (lane < 9) h.d = a.corners[9 * (long long)ex + lane];
      else if (lane < 18) h.d = a.corners[9 * (long long)ey + lane - 9];
      else if (lane == 18) h.d = a.a2[ex];
      else if (lane == 19) h.d = a.a2[ey];
      if (lane < a.fam_count) h.fr = a.frange[(long long)a.fam_ids[lane] * E2 + Pp];
    }
  };
  long long P0 = grab();
  Header pre;
  load_header(P0, pre);
  long long P1 = grab();

  while (P0 < E2) {
    const Header cur = pre;
    P0 = P1;
    load_header(P0, pre);
    P1 = grab();
    if (cur.units == 0 || cur.cs != 0) continue;
    if (__ballot_sync(FULL, (cur.fr.lo_cnt >> 16) != 0) == 0u) continue;
    my_pairs += lane == 0 ? 1ULL : 0ULL;
    V3 X0, X1, X2, Y0, Y1, Y2;
    X0.x = __shfl_sync(FULL, cur.d, 0); X0.y = __shfl_sync(FULL, cur.d, 1); X0.z = __shfl_sync(FULL, cur.d, 2);
    X1.x = __shfl_sync(FULL, cur.d, 3); X1.y = __shfl_sync(FULL, cur.d, 4); X1.z = __shfl_sync(FULL, cur.d, 5);
    X2.x = __shfl_sync(FULL, cur.d, 6); X2.y = __shfl_sync(FULL, cur.d, 7); X2.z = __shfl_sync(FULL, cur.d, 8);
    Y0.x = __shfl_sync(FULL, cur.d, 9); Y0.y = __shfl_sync(FULL, cur.d, 10); Y0.z = __shfl_sync(FULL, cur.d, 11);
    Y1.x = __shfl_sync(FULL, cur.d, 12); Y1.y = __shfl_sync(FULL, cur.d, 13); Y1.z = __shfl_sync(FULL, cur.d, 14);
    Y2.x = __shfl_sync(FULL, cur.d, 15); Y2.y = __shfl_sync(FULL, cur.d, 16); Y2.z = __shfl_sync(FULL, cur.d, 17);
    const V3 e1 = sub(X1, X0), e2 = sub(X2, X1), f1 = sub(Y1, Y0), f2 = sub(Y2, Y1);
    const double scale = kInv4Pi * __shfl_sync(FULL, cur.d, 18) * __shfl_sync(FULL, cur.d, 19);

    // geometry of the lane's points (k_quad's arithmetic), their time-step index n and cell column j
    double ck[kNK], rk[kNK];
    int nj[kNK];  // column | n << 5
    bins[lane] = 0u;
    __syncwarp();
    const double yx = Y0.x + y1 * f1.x + y2 * f2.x, yy = Y0.y + y1 * f1.y + y2 * f2.y,
                 yz = Y0.z + y1 * f1.z + y2 * f2.z;
#pragma unroll
    for (int k = 0; k < kNK; ++k) {
      const double x1 = R.x1[lane + 32 * k], x2 = R.x2[lane + 32 * k];
      const double dx = (X0.x + x1 * e1.x + x2 * e2.x) - yx;
      const double dy = (X0.y + x1 * e1.y + x2 * e2.y) - yy;
      const double dz = (X0.z + x1 * e1.z + x2 * e2.z) - yz;
      rk[k] = sqrt(dx * dx + dy * dy + dz * dz);
      ck[k] = scale * R.w[lane + 32 * k] / rk[k];
      const double u = rk[k] * inv_dt;
      const int n = (int)u;
      const int j = min(kCellPerDt - 1, (int)((u - (double)n) * (double)kCellPerDt));
      nj[k] = j | (n << 5);
      atomicAdd(bins + j, 1u);
    }
    __syncwarp();
    int n_min = nj[0] >> 5, n_max = n_min;  // time-step range of the pair's points
#pragma unroll
    for (int k = 1; k < kNK; ++k) {
      n_min = min(n_min, nj[k] >> 5);
      n_max = max(n_max, nj[k] >> 5);
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      n_min = min(n_min, __shfl_xor_sync(FULL, n_min, o));
      n_max = max(n_max, __shfl_xor_sync(FULL, n_max, o));
    }
    int nsr;  // sub-runs of the pair
    {  // columns -> column-pure sub-runs (the order inside a column is free: stage 1
       // stores by rule point, stage 2 sums in rule-point order)
      const int cnt = (int)bins[lane];
      const int mine_sr = (cnt + kCellSub - 1) / kCellSub;
      int incl = mine_sr;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += v;
      }
      nsr = __shfl_sync(FULL, incl, 31);
      const int first = (incl - mine_sr) * kCellSub;  // first slot of column `lane`
      __syncwarp();
      bins[lane] = (unsigned)first;
      for (int p = cnt; p < mine_sr * kCellSub; ++p) {  // pads of the column's last sub-run
        const int slot = first + p;
        s_q[(slot % kCellSub) * kCellSubRuns + slot / kCellSub] = (int)0x80000000u | (lane << 8);
      }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < kNK; ++k) {
        const int slot = (int)atomicAdd(bins + (nj[k] & 31), 1u);
        const int at = (slot % kCellSub) * kCellSubRuns + slot / kCellSub;
        s_r[at] = rk[k];
        s_q[at] = (nj[k] << 8) | (lane + 32 * k);
      }
      __syncwarp();
    }

    for (int fi = 0; fi < a.fam_count; ++fi) {
      FRange fr;
      fr.foff = __shfl_sync(FULL, cur.fr.foff, fi);
      fr.lo_cnt = __shfl_sync(FULL, cur.fr.lo_cnt, fi);
      const int ucnt = fr.lo_cnt >> 16, s_lo = fr.lo_cnt & 0xffff;
      if (ucnt == 0) continue;
      const QFam& fd = a.fam[fi];
      const double2* rows = reinterpret_cast<const double2*>(sblob + fd.coeff_off);
      const double* sdel = sdelta + fd.delta_off + s_lo;
      unsigned n_act = 0;
      // (every grid family is stored with degree-16 rows: one loop body in the instruction cache)
      cell_family<16>(fd, rows, sdel, s_r, s_q, G, nsr, lane, s_lo, (unsigned)ucnt, a.dt, n_min, n_max, n_act);
      my_in += n_act;
      __syncwarp();

      // stage 2: per unit, contract the table values with the weights and shape functions
      double cx[kNK][3];
      int mk[kNK];  // span of point k at the window's first position
#pragma unroll
      for (int k = 0; k < kNK; ++k) {
        const double x1 = R.x1[lane + 32 * k], x2 = R.x2[lane + 32 * k];
        cx[k][0] = ck[k] * (1.0 - x1);
        cx[k][1] = ck[k] * (x1 - x2);
        cx[k][2] = ck[k] * x2;
        mk[k] = (nj[k] >> 5) + fd.cell_kappa - s_lo;
      }
      const unsigned nspan = (unsigned)fd.cell_M;
      double* dst = a.part + (cur.base + fr.foff) * NACC;
      const double2* Gq = G + lane;
      // Four units per step.  Register set u of a lane holds unit si + (u ^ h), h = lane
      // bits 4-3: the first two levels of the warp sum exchange whole sets (no selects),
      // after them the 8 lanes sharing h hold the 10 partial values of unit si + h.
      const int h = (lane >> 3) & 3;
      for (int si = 0; si < ucnt; si += 4) {
        double tb[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u) tb[u][0] = tb[u][1] = tb[u][2] = tb[u][3] = 0.0;
#pragma unroll
        for (int k = 0; k < kNK; ++k) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int unit = si + (u ^ h);
            const unsigned m = (unsigned)(mk[k] - unit);
            double2 g = make_double2(0.0, 0.0);
            if (m < nspan && unit < ucnt) g = Gq[m * kChunk + 32 * k];
            tb[u][0] = fma(g.x, cx[k][0], tb[u][0]);
            tb[u][1] = fma(g.x, cx[k][1], tb[u][1]);
            tb[u][2] = fma(g.x, cx[k][2], tb[u][2]);
            tb[u][3] = fma(g.y, ck[k], tb[u][3]);
          }
        }
        double acc[4][NACC];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          // explicitly rounded products: a product fused into the first exchange's add
          // would make the sum depend on which lane of a pair keeps the unit
          acc[u][0] = __dmul_rn(shy0, tb[u][0]);
          acc[u][1] = __dmul_rn(shy0, tb[u][1]);
          acc[u][2] = __dmul_rn(shy0, tb[u][2]);
          acc[u][3] = __dmul_rn(shy1, tb[u][0]);
          acc[u][4] = __dmul_rn(shy1, tb[u][1]);
          acc[u][5] = __dmul_rn(shy1, tb[u][2]);
          acc[u][6] = __dmul_rn(shy2, tb[u][0]);
          acc[u][7] = __dmul_rn(shy2, tb[u][1]);
          acc[u][8] = __dmul_rn(shy2, tb[u][2]);
          acc[u][9] = tb[u][3];
        }
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int i = 0; i < NACC; ++i) acc[u][i] += __shfl_xor_sync(FULL, acc[u ^ 2][i], 16);
#pragma unroll
        for (int i = 0; i < NACC; ++i) acc[0][i] += __shfl_xor_sync(FULL, acc[1][i], 8);
        // the 8 lanes of a group: reduce-scatter of the 10 values (5, 3, 2 per level)
        double w1[5], w2[3], w3[2];
        rs_level<NACC, 4>(acc[0], w1, lane & 4);
        rs_level<5, 2>(w1, w2, lane & 2);
        rs_level<3, 1>(w2, w3, lane & 1);
        int base = 0, n = NACC;
        {
          const int H[3] = {5, 3, 2};
#pragma unroll
          for (int l = 0; l < 3; ++l) {
            const bool hi = (lane >> (2 - l)) & 1;
            if (hi) {
              base += H[l];
              n = n > H[l] ? n - H[l] : 0;
            } else {
              n = n < H[l] ? n : H[l];
            }
          }
        }
        const int unit = si + h;
        if (unit < ucnt) {
          if (n > 0) dst[(long long)unit * NACC + base] = w3[0];
          if (n > 1) dst[(long long)unit * NACC + base + 1] = w3[1];
        }
      }
      __syncwarp();
    }
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) my_in += __shfl_xor_sync(FULL, my_in, o);
  if (lane == 0) {
    atomicAdd(a.n_in, my_in);
    atomicAdd(a.n_in + 34, my_in);  // this kernel's share (TdbStats::n_in_cells)
    atomicAdd(a.n_in + 35, my_pairs);
  }
}
