// Tensor-core (FP64 DMMA) matvec on 8 x 4 BSR tiles (tdb_bsr.cu); internal.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "tdb_internal.h"

namespace tdb {

constexpr int kBsrWarps = 8;  // warps (= term groups) per CTA

struct BsrFam {
  const int32_t* col;
  const double* val;
  const int64_t* rbptr;
};

struct BsrMvArgs {
  int nrows, nRB, KG, T;  // T: 8-time tiles per CTA (1, 2, 4 or 8)
  int rlo, nr, clo, nc;
  int words;
  const BsrFam* fam;
  const int* term_f;
  const int* term_s;
  const int* term_d;
  const unsigned* term_mask;
  const int* group_begin;
  const int* rperm;      // Morton row -> local row
  const double* xp;      // [nCB*4][xs] permuted, transposed x (zero pad rows/columns)
  int xs;
  double* y;
};

// Toeplitz-ordered tiles of one family (tdb_tbsr.cu)
struct TbsrMvArgs {
  int nRB, G, ntg, TT, npos;
  int nrows, nr;
  const int32_t* col;
  const int32_t* pos;
  const double* val;
  const int64_t* rbptr;
  const int* off_tab;        // [ntg][npos][8 (g)][TT] column offset in xp (nc = zero column)
  const unsigned* act_tab;   // [ntg][npos] active time tiles of the position's term
  const int* rperm;
  const double* xp;          // [nCB*4][xs] permuted, transposed x
  int xs;
  double* ypart;             // [nRB * ntg][G][TT * 64]
  double* y;
};

int tbsr_build(TdbSystem* sys, int f);
int tbsr_mv_launch(const TbsrMvArgs& a, cudaStream_t st);              // tiles + ordered reduce
int tbsr_mv_tiles(const TbsrMvArgs& a, cudaStream_t st, bool reduce);  // tile kernel (optionally + reduce)
int tbsr_mv_reduce(const TbsrMvArgs& a, cudaStream_t st);              // ordered reduce into y

int bsr_build(TdbSystem* sys);
int bsr_mv_launch(const BsrMvArgs& a, cudaStream_t st);

}  // namespace tdb
