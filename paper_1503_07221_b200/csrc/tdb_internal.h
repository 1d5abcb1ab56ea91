// Internal (non-ABI) structures shared by the CUDA translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "../../include/tdb.h"

namespace tdb {

constexpr int kMaxTables = 32;   // nt = 2 (p+1)^2, p <= 3
constexpr int kMaxFamilies = 16;
constexpr int kDeg = 16;         // Chebyshev degree of the fast path (PrototypeTables default)
#ifndef TDB_CHUNK
#define TDB_CHUNK 256
#endif
constexpr int kChunk = TDB_CHUNK;  // rule points per warp work item (tuning variants: -DTDB_CHUNK)

// One table family on the device (all tables share domain/nsub/fold).
struct FamDev {
  int npos, nsub, nt, fold;
  int coeff_off;   // offset (doubles) of this family's coefficients in the launch blob
  int coef_global; // 1: read `coeffs` (global, transposed layout) instead of the smem blob
  int deg;         // polynomial degree kept (Chebyshev tail below 3e-15 of the table max dropped)
  int khead;       // monomials 0..khead-1 in FP64, khead..deg in FP32 (float tail)
  int tail_off;    // doubles from the head start to the FP32 tail block
  int pad_;
  double lo, w, inv_w, amin, amax;
  double sp[kMaxTables], sn[kMaxTables];
  const double* delta;
  const double* slo;
  const double* shi;
  const double* coeffs;  // global copy, rows [sub][k][t] (head FP64 + FP32 tail)
};

struct RuleDev {
  long long nq;
  int nitems;  // ceil(nq / kChunk)
  int pad_;
  const double* x1;
  const double* x2;
  const double* y1;
  const double* y2;
  const double* w;
};

// Admissible position range of one (family, pair): s in [s_lo, s_lo + cnt),
// partial-slot offset foff within the pair.
struct FRange {
  int foff;
  int lo_cnt;  // s_lo | (cnt << 16)
};

// One lag-band tile record (tdb_band.cu): 8 test rows (Morton row block J) x 4
// consecutive positions s0 .. s0+3 of ONE column vertex l, A-fragment order
// (v[4 * row + (s - s0)]), header in the same 16-byte-aligned record (bulk copies).
struct __align__(16) BandTile {
  double v[32];
  int32_t l, s0, pad0, pad1;
};

// The records of a BandStore whose lag window meets a set of active positions.
struct BandView {
  std::vector<unsigned> act;  // active-position bit set (key, with dt0 / dt1 / nT)
  int dt0 = 0, dt1 = 0, nT = 0;
  long long ntiles = 0;
  BandTile* tiles = nullptr;
  int64_t* rbptr = nullptr;
};

// One family's stored blocks as lag-band tiles, sorted (J, l, s0).
struct BandStore {
  bool built = false, failed = false;
  long long ntiles = 0, nnz = 0;
  BandTile* tiles = nullptr;  // (ntiles,)
  int64_t* rbptr = nullptr;   // (nRB + 1,)
  std::vector<BandView> views;  // per-plan restrictions (tdb_band.cu band_view)
};

struct FamilyStore {
  int npos = 0;
  int split_R = 1, split_D = kDeg, split_K = kDeg + 1;  // evaluation split chosen at create
  long long nnz = 0;
  int64_t* indptr = nullptr;   // npos * M + 1
  int32_t* indices = nullptr;  // nnz
  double* data = nullptr;      // nnz * (p+1)^2
  // device copies of the position tables
  double* delta = nullptr;
  double* slo = nullptr;
  double* shi = nullptr;
  double* coeffs = nullptr;
};

}  // namespace tdb

namespace tdb {
// caching device allocator (tdb_context.cu): freed blocks are reused by later
// systems / plans; release only after the owning stream is idle
cudaError_t dev_malloc(void** out, size_t bytes);
void dev_free(void* p);
void dev_pool_trim();
}  // namespace tdb

struct TdbContext {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
};

struct AsmWorkspace;
void tdb_workspace_free(struct TdbSystem* sys);

struct TdbSystem {
  TdbContext* ctx = nullptr;
  AsmWorkspace* ws = nullptr;
  int p = 0, np1 = 1, nm = 1, nacc = 10, F = 0;
  long long E = 0, V = 0;
  int nrows = 0;  // owned test-vertex rows (== V for a full system)
  // mesh
  double* corners = nullptr;
  double* a2 = nullptr;
  double* normals = nullptr;
  double* curls = nullptr;
  int* tri = nullptr;
  int* star_off = nullptr;
  int* star_ids = nullptr;
  // families
  std::vector<tdb::FamilyStore> fam;
  std::vector<tdb::FamDev> famdev_host;
  tdb::FamDev* famdev = nullptr;
  // Morton orders for the tensor-core matvec (built at create time):
  // vperm[new] = old vertex, vinv[old] = new; rperm[new] = old local row, rinv[old] = new
  std::vector<int> vperm, vinv, rperm, rinv;
  int* d_vperm = nullptr;
  int* d_vinv = nullptr;
  int* d_rperm = nullptr;
  int* d_rinv = nullptr;
  int nRB = 0, nCB = 0;  // ceil(nrows / 8), ceil(V / 4)
  std::vector<tdb::BandStore> band;  // per family, built on first use by a matvec plan
  TdbStats stats{};
};
