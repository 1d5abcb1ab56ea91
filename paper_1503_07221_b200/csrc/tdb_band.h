// Lag-band tensor-core (FP64 DMMA) tiles of the block-Toeplitz matvec (tdb_band.cu); internal.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "tdb_internal.h"

namespace tdb {

constexpr int kBandMaxWarps = 8;  // time-group warps per CTA

struct BandMvArgs {
  int nRB, P, nT, TT, W;  // row blocks, parts per row block, 8-step time tiles, tiles per warp, warps per CTA
  int nrows, nS;          // owned rows, S-tiles (4 positions each)
  int ktlo, nkt, rlo;     // band rows kt in [ktlo, ktlo + nkt); y row index kt - rlo
  int off0, xs;           // xt column of (kt = ktlo, lag d_0) and row stride
  int ldy;                // ypart row stride (>= 8 nT)
  const int32_t* col;
  const int32_t* stile;
  const double* val;
  const int64_t* rbptr;
  const unsigned* s_act;  // (nS,) bit k: position 4 S + k is a band term of this plan
  const int* rperm;       // Morton row -> local row
  const double* xt;       // [V][xs] vertex-major x of the plan's inner columns, zero pads
  double* ypart;          // [P][nRB * 8][ldy]
  double* y;
};

int band_build(TdbSystem* sys, int f);
int band_mv_tiles(const BandMvArgs& a, cudaStream_t st);   // tile kernel -> ypart
int band_mv_reduce(const BandMvArgs& a, cudaStream_t st);  // y += sum of parts (ordered)

}  // namespace tdb
