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

int bsr_build(TdbSystem* sys);
int bsr_mv_launch(const BsrMvArgs& a, cudaStream_t st);

}  // namespace tdb
