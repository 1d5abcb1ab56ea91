// Lag-band tensor-core (FP64 DMMA) tiles of the block-Toeplitz matvec (tdb_band.cu); internal.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "tdb_internal.h"

namespace tdb {

constexpr int kBandMaxWarps = 8;  // time-group warps per CTA
constexpr int kBandChunk = 32;    // tile records per bulk-copy stage (wide plans; 16 for 1-2 warps)
constexpr int kBandStages = 3;    // stages of the shared-memory ring
constexpr int kIrrWords = 13;     // block-row bits of the irregular (tie) lag: 8 x 6 x 8 tiles max

struct BandMvArgs {
  int nRB, P, nT, TT, W;  // row blocks, parts per row block, 8-step time tiles, tiles per warp, warps per CTA
  int nrows, act_words;   // owned rows, words of the active-position bit set
  int chunk;              // tile records per pipeline stage
  int direct;             // short plan: k_band_direct (one warp per (row block, part), no smem ring)
  int ktlo, nkt, rlo;     // band rows kt in [ktlo, ktlo + nkt); y row index kt - rlo
  int off0, xs;           // xt column of (kt = ktlo, lag d_0) and row stride
  int dt0, dt1;           // itlo + d_0 - ktlo, ithi + d_0 - ktlo: valid rows of lag d_0 + s are
                          // ktlo + [dt0 + s, dt1 + s]
  int ldy;                // ypart row stride (>= 8 nT)
  const BandTile* tiles;
  const int64_t* rbptr;
  const unsigned* s_act;  // (act_words,) bit s: position s is a band term of this plan
  int s_irr;              // position whose logical mask is a strict subset of the band rows
                          // (the light-cone tie lag), -1 if none
  unsigned irr_mask[kIrrWords];  // its valid block rows: bit r <-> kt = ktlo + r
  const int* rperm;       // Morton row -> local row
  const double* xt;       // [V][xs] vertex-major x of the plan's inner columns, zero pads
  double* ypart;          // [P][nRB * 8][ldy]
  double* y;
};

int band_build(TdbSystem* sys, int f);
// the records of family f for one plan signature (active positions, valid-row offsets
// dt0 / dt1, time tiles nT): lags outside the plan zeroed, records without a valid time
// tile dropped, the valid time-tile range in each header; cached per signature
int band_view(TdbSystem* sys, int f, const std::vector<unsigned>& act, int dt0, int dt1, int nT,
              const BandTile** tiles, const int64_t** rbptr, long long* ntiles);
int band_mv_tiles(const BandMvArgs& a, cudaStream_t st);   // tile kernel -> ypart
size_t band_smem_bytes(int act_words, int chunk);
int band_mv_reduce(const BandMvArgs& a, cudaStream_t st);  // y += sum of parts (ordered)

}  // namespace tdb
