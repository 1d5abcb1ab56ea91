/*
 * tdb.h - C ABI of the B200-native lag-block assembly + block Hessenberg matvec
 * for the space-time Galerkin TDBIE (arXiv:1503.07221).
 *
 * Every entry point returns int: TDB_OK (0) or a negative TDB_E* code;
 * tdb_last_error() gives a thread-local message.  No C++ exceptions and no
 * torch types cross this boundary; arrays are plain pointers + sizes, all
 * float64 C-contiguous unless stated.  Pointers named *_dev are device
 * pointers; all others are host pointers owned by the caller.
 *
 * Reference interfaces replaced (paths under /root/reference/pkg/src/tdbem/):
 *   tdb_pair_block_contributions  <- _kernels/__init__.py:1-34 dispatch
 *                                    (_core.pyx:47-159, _fallback.py:46-81)
 *   tdb_system_assemble           <- block_system.py:228-275 assemble_system
 *                                    + assembly.py:240-306 assemble_subblocks
 *   tdb_system_copy_family        <- the CSR lists of BlockHessenbergMatrix
 *                                    .unique_blocks (block_system.py:145)
 *   tdb_matvec (+ plan)           <- block_system.py:180-216 matvec(x, rows, cols)
 *   tdb_krylov_*                  <- solvers.py:189-222 (_gmres_cycle_raw's Givens
 *                                    bookkeeping and final update, on the device)
 *   tdb_dlp_eval                  <- potential.py:53-126 eval_double_layer /
 *                                    eval_total_field
 *   tdb_rhs_*                     <- assembly.py:314-355 assemble_rhs (contraction)
 *   tdb_table_node_values         <- kernel_weights.py:243-295 PrototypeTables.build
 */
#ifndef TDB_H_
#define TDB_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TDB_ABI_VERSION 1

enum {
  TDB_OK = 0,
  TDB_E_INVALID = -1,   /* bad argument / shape (ValueError) */
  TDB_E_CUDA = -2,      /* CUDA runtime failure (RuntimeError) */
  TDB_E_NOMEM = -3,     /* device allocation failed (MemoryError) */
  TDB_E_NODEVICE = -4,  /* no CUDA device visible (RuntimeError) */
  TDB_E_UNSUPPORTED = -5
};

/* Packed psi / psi~ tables of one block position (assembly.py:68-127 PsiPack).
 * nt = 2 (p+1)^2 tables, index t = (m2 (p+1) + m1) * 2 + {0: psi, 1: psi~}.
 * coeffs is (nt, max_nsub, deg+1). */
typedef struct TdbPsiPack {
  int32_t p;
  int32_t deg;
  int32_t max_nsub;
  int32_t reserved;
  double delta;
  const double* lo;       /* (nt,) */
  const double* width;    /* (nt,) */
  const int64_t* nsub;    /* (nt,) */
  const double* coeffs;   /* (nt, max_nsub, deg+1) */
  const double* sp;       /* (nt,) sign for a >= 0 (folded tables) */
  const double* sn;       /* (nt,) sign for a < 0 */
  const uint8_t* fold;    /* (nt,) */
  const uint8_t* active;  /* (nt,) */
} TdbPsiPack;

/* Drop-in for tdbem._kernels.pair_block_contributions.
 * cx, cy (npair,3,3) chart corners; a2x, a2y, ndot (npair,); curly, curlx
 * (npair,3,3); xhat, yhat (nq,2); wq (nq,).  out (npair,p+1,p+1,3,3) is
 * written (not accumulated): out[P,m2,m1,a,b] = contribution of pair P to
 * sub-block (m2,m1) at (row = y chart vertex a, col = x chart vertex b).
 * Host pointers; the call copies to the current device and synchronises. */
int tdb_pair_block_contributions(const double* cx, const double* cy,
                                 const double* a2x, const double* a2y,
                                 const double* ndot, const double* curly,
                                 const double* curlx, const double* xhat,
                                 const double* yhat, const double* wq,
                                 int64_t npair, int64_t nq,
                                 const TdbPsiPack* pack, double* out);

/* ---- device-resident system ------------------------------------------- */

typedef struct TdbMesh {
  int64_t num_vertices;
  int64_t num_triangles;
  const double* corners;   /* (E,3,3) */
  const double* a2;        /* (E,) twice the triangle area */
  const double* normals;   /* (E,3) */
  const double* curls;     /* (E,3,3) n x grad(hat_a) */
  const int64_t* triangles;/* (E,3) */
  const int64_t* star_off; /* (V+1,) vertex -> triangles CSR, ascending ids */
  const int64_t* star_ids; /* (3E,) */
} TdbMesh;

/* One table family = all canonical block positions sharing (ansatz kind,
 * test kind): identical tables, only delta differs.  Positions
 * are listed in lag order so that slo and shi are non-decreasing. */
typedef struct TdbFamily {
  int32_t npos;
  int32_t reserved;
  const double* delta;     /* (npos,) canonical_origin(it) - canonical_origin(kt) */
  const double* slo;       /* (npos,) psi_support lower end */
  const double* shi;       /* (npos,) psi_support upper end */
  TdbPsiPack pack;         /* delta field ignored */
} TdbFamily;

typedef struct TdbRule {
  int64_t nq;
  const double* xhat;      /* (nq,2) */
  const double* yhat;      /* (nq,2) */
  const double* w;         /* (nq,) */
} TdbRule;

enum { TDB_CASE_REGULAR = 0, TDB_CASE_COINCIDENT = 1, TDB_CASE_EDGE = 2, TDB_CASE_VERTEX = 3 };

typedef struct TdbAssemblyDesc {
  int32_t p;
  int32_t num_families;
  const TdbFamily* families;
  TdbRule rules[4];        /* indexed by TDB_CASE_* */
  /* Row block (multi-GPU sharding): assemble only the test-vertex
   * rows listed (strictly increasing); 0 = all vertices.  Pairs are restricted
   * to test triangles in the owned rows' stars; CSR rows follow `rows`. */
  int64_t num_rows;
  const int64_t* rows;
} TdbAssemblyDesc;

typedef struct TdbStats {
  int64_t units;           /* admissible (pair, position) units */
  int64_t items;           /* warp work items of the quadrature kernel */
  int64_t n_in;            /* (unit, point) evaluations inside the table support */
  int64_t n_geom;          /* rule points whose geometry was evaluated */
  int64_t nnz_total;       /* stored entries over all families */
  double ms_plan;          /* pair bounds + admissible ranges + scans */
  double ms_quad;          /* quadrature kernel(s) */
  double ms_finalize;      /* singular item reduction */
  double ms_pattern;       /* CSR pattern + compensated gather */
  double ms_total;
  int64_t units_case[4];   /* units per pair case (regular, coincident, edge, vertex) */
  int64_t pairs_case[4];   /* pairs with >= 1 unit, per case */
  int64_t launches;        /* kernel launches issued by the last tdb_system_run */
  int64_t units_primary;   /* units whose test triangle's first vertex is an owned row:
                              summed over row blocks = the global unit count */
  /* share of the regular-pair kernel (k_quad_cells) in ms_quad / n_in, pairs it took */
  double ms_quad_cells;
  int64_t n_in_cells;
  int64_t pairs_cells;
} TdbStats;

typedef struct TdbContext TdbContext;
typedef struct TdbSystem TdbSystem;

int tdb_abi_version(void);
/* Device blocks freed by destroyed systems / plans are cached for reuse (up to
 * 8 GB); this returns them to the driver. */
int tdb_release_cached_memory(void);
/* Measured FP64 throughput of the device (TFLOP/s): the better of a DFMA
 * (2 flops per lane) and a DMMA m8n8k4 (512 flops per warp) microbenchmark of
 * independent chains over all SMs, best of `repeats`. */
int tdb_fp64_peak(TdbContext* ctx, int repeats, double* tflops);
const char* tdb_last_error(void);
int tdb_device_count(int* count);

int tdb_ctx_create(int device, TdbContext** out);
int tdb_ctx_destroy(TdbContext* ctx);
/* stream used by all stream-ordered calls on this context (0 = legacy default) */
int tdb_ctx_set_stream(TdbContext* ctx, void* cuda_stream);

/* SurfaceMesh.tri_distance_bounds rows (mesh.py:146-153, :357-391) on the
 * device: tmin (exact triangle distance, 0 for touching pairs) and tmax (max
 * corner distance) of triangles rows[r] x every triangle, (nrows, E) each,
 * bit-identical to the reference's numpy evaluation order.  Only the mesh's
 * corners and triangles are read. */
int tdb_tri_distance_bounds(TdbContext* ctx, const TdbMesh* mesh, int64_t nrows,
                            const int64_t* rows, double* tmin, double* tmax);

/* Upload the mesh, tables and rules (host inputs), size every device buffer
 * (pair plan, work items, partials, CSR patterns); no values yet. */
int tdb_system_create(TdbContext* ctx, const TdbMesh* mesh,
                      const TdbAssemblyDesc* desc, TdbSystem** out);
/* (Re)compute all blocks on the device from the resident inputs: pair plan,
 * quadrature, singular item reduction, CSR pattern + compensated gather.
 * Stream-ordered without host round trips; synchronises once at the end to
 * publish TdbStats. */
int tdb_system_run(TdbSystem* sys);
/* tdb_system_create + tdb_system_run */
int tdb_system_assemble(TdbContext* ctx, const TdbMesh* mesh,
                        const TdbAssemblyDesc* desc, TdbSystem** out);
int tdb_system_destroy(TdbSystem* sys);
int tdb_system_stats(const TdbSystem* sys, TdbStats* out);
/* nnz of family f (stored pattern incl. explicit zeros) */
int tdb_system_family_nnz(const TdbSystem* sys, int32_t f, int64_t* nnz);
/* Admissible (pair, position) units of every position of family f (npos,),
 * i.e. len(block_pattern(mesh, grid, kt, it).element_pairs) of the reference
 * (assembly.py:167-184) over this system's test triangles; valid after a run. */
int tdb_system_position_units(TdbSystem* sys, int32_t f, int64_t* units);
/* Evaluation split family f runs with (introspection; chosen at create so every
 * table stays within 3e-15 of its max of the reference's Clenshaw value):
 * subintervals refined R-fold, monomial degree D, monomials k < K in FP64 and
 * K <= k <= D in FP32 (K = D + 1: all FP64). */
int tdb_system_family_split(const TdbSystem* sys, int32_t f, int32_t* R, int32_t* D, int32_t* K);
/* D2H copy of family f: indptr (npos*nrows+1,) int64 with rows (s, local row r);
 * indices (nnz,) int32 columns; data (nnz,(p+1)^2) */
int tdb_system_copy_family(const TdbSystem* sys, int32_t f, int64_t* indptr,
                           int32_t* indices, double* data);
/* Device pointers of family f (valid until tdb_system_destroy). */
int tdb_system_family_device(const TdbSystem* sys, int32_t f,
                             const int64_t** indptr_dev,
                             const int32_t** indices_dev,
                             const double** data_dev);


/* ---- block Hessenberg matvec (block_system.py:180-216) ------------------
 * A matvec plan fixes the inclusive 1-based block ranges rows = [rlo, rhi],
 * cols = [clo, chi] and the list of "terms": one per stored (family f,
 * position s) that any logical block position (kt, it) in range resolves to,
 * with d = kt - it constant per term and a bitmask over kt (bit kt-1 of
 * word (kt-1)/32) of the logical positions that are structurally non-zero
 * (is_zero_position, block_system.py:153-160, evaluated by the caller).
 * Vectors are time-major as in the reference: entry ((k-1)(p+1)+m)*M + j
 * relative to the range start.  tdb_matvec is stream-ordered on the
 * context's stream and deterministic (fixed summation order). */
typedef struct TdbMatvecDesc {
  int32_t N;
  int32_t rlo, rhi, clo, chi;
  int32_t nterms;
  int32_t words;            /* mask words per term = ceil(N / 32) */
  int32_t reserved;
  const int32_t* term_family;
  const int32_t* term_pos;
  const int32_t* term_d;
  const uint32_t* term_mask; /* (nterms, words) */
  /* Layout of x (optional): entry (vertex l, column c) is x[x_map[l] + c*x_stride].
   * NULL x_map = the reference's time-major layout (x_map[l] = l, stride M).
   * A multi-GPU caller passes the all-gathered rank-major layout
   * [rank][column][rows_per_rank] with x_map[l] = owner*ncols*stride + local. */
  int64_t x_stride;
  const int64_t* x_map;      /* (M,) */
} TdbMatvecDesc;

typedef struct TdbMatvecPlan TdbMatvecPlan;

int tdb_matvec_plan_create(TdbSystem* sys, const TdbMatvecDesc* desc, TdbMatvecPlan** out);
int tdb_matvec_plan_destroy(TdbMatvecPlan* plan);
/* y_dev[(rhi-rlo+1)(p+1) * nrows] = A[rows, cols] x_dev (device pointers); y is
 * time-major over the system's owned test-vertex rows (all M for a full system). */
int tdb_matvec(TdbMatvecPlan* plan, const double* x_dev, double* y_dev);
/* canonical stored bytes and logical flops of one application of this plan */
int tdb_matvec_plan_work(const TdbMatvecPlan* plan, double* algorithmic_bytes, double* flops);
/* how the plan applies its terms: *tiled_terms lag terms on the FP64 tensor-core
 * tiles (tdb_tbsr.cu), *csr_terms on the CSR kernel (tdb_matvec.cu).  Introspection
 * only (no counterpart in the reference, whose matvec is block_system.py:180-216). */
int tdb_matvec_plan_kind(const TdbMatvecPlan* plan, int32_t* tiled_terms, int32_t* csr_terms);

/* ---- device-side GMRES cycle bookkeeping (solvers.py:172-223) ------------
 * Replaces the per-Arnoldi-step host round trip of _gmres_cycle_raw
 * (reference solvers.py:189-215: Hessenberg column, Givens rotations,
 * convergence and breakdown tests) and the final solve_triangular + Z^T y
 * update (:217-222) for fixed-iteration inner solves, so a whole preconditioner
 * application can be captured in a CUDA graph.  All pointers are device
 * pointers; `stream` is a cudaStream_t (NULL = legacy default stream).
 * state: TDB_KS_NSTATE doubles.  H is (m+1) x ldh row-major. */
#define TDB_KS_DONE 0
#define TDB_KS_KDONE 1
#define TDB_KS_BREAKDOWN 2
#define TDB_KS_TOL_ABS 3
#define TDB_KS_BETA 4
#define TDB_KS_CONVERGED 5
#define TDB_KS_NSTATE 8
/* beta: device scalar ||b|| (x0 = 0); tol_abs = tol_rel * beta; g[0] = beta */
int tdb_krylov_init(double* state, const double* beta, double tol_rel, double* g, void* stream);
/* step k: hcol[0..k+1] = (V_j . w for j <= k, ||w||) */
int tdb_krylov_givens(double* state, int32_t k, const double* hcol, double* H, int32_t ldh, double* cs,
                      double* sn, double* g, void* stream);
/* x[0..n) = x0 + sum_{j < k_done} y_j Z[j*ldz + i], H[:k_done,:k_done] y = g (x0 may be NULL) */
int tdb_krylov_update(double* x, const double* x0, const double* Z, int64_t ldz, int64_t n, const double* state,
                      const double* H, int32_t ldh, const double* g, int32_t m, void* stream);
/* *err = 1 if the cycle broke down without converging (BreakdownError) */
int tdb_krylov_flag(const double* state, double* err, void* stream);
/* One fused Arnoldi step after the matvec w = A z: w is orthogonalised against the rows V[0..k] (row stride ldv) by
 * two classical Gram-Schmidt passes, hcol[0..k+1] = (coefficients, ||w||).  If
 * H != NULL the Givens step of tdb_krylov_givens follows; if vnext != NULL it
 * receives w / ||w||.  Replaces the MGS loop of solvers.py:189-194. k < 64.
 * n < 32768 (TDB_ARNOLDI_GRID_MIN_N): one launch of a <= 16-CTA thread-block
 * cluster; longer vectors: four full-grid launches (per-CTA partials summed in
 * CTA order by the last CTA, so the result is deterministic). */
int tdb_krylov_arnoldi(const double* V, int64_t ldv, int64_t n, int32_t k, double* w, double* hcol, double* state,
                       double* H, int32_t ldh, double* cs, double* sn, double* g, double* vnext, void* stream);

/* ---- retarded double-layer potential (potential.py:53-126) ---------------
 * out[t * npts + x] = u(points[x], times[t]) for the density coefficients
 * coeffs (L = N (p+1) rows of M vertex values, the solver's layout); the far /
 * near triangle rules are (x1, x2) chart nodes + weights of triangle_rule(q).
 * Host buffers; computed on the context's device.  Replaces
 * tdbem.potential.eval_double_layer for a batch of points and times. */
int tdb_dlp_eval(TdbContext* ctx, const TdbMesh* mesh, double T, int32_t N, int32_t p, const double* coeffs,
                 int64_t npts, const double* points, int64_t ntimes, const double* times, int32_t nq_far,
                 const double* far_xhat, const double* far_w, int32_t nq_near, const double* near_xhat,
                 const double* near_w, double* out);

/* ---- right-hand side contraction (assembly.py:314-355) -------------------
 * Device pointers.  G: rows j0 .. j0+nj-1 of the datum g(X_p, t_j) at the P
 * regular-rule points (node-major, row stride P).  Stage 1 writes
 * H[j][l] = sum_{q in vptr[l]..vptr[l+1]} vw[q] G[j][vpts[q]] (vertex gather of the
 * shape-weighted rule points); stage 2 writes out[k*M + l] = sum_{j in
 * kptr[k]..kptr[k+1]} w[j] H[j][l] (the time nodes of basis k are contiguous). */
int tdb_rhs_vertex_gather(const double* G, int64_t j0, int64_t nj, int64_t P, const int64_t* vptr, const int32_t* vpts,
                          const double* vw, int64_t M, double* H, void* stream);
int tdb_rhs_time_sum(const double* H, const int64_t* kptr, const double* w, int64_t L, int64_t M, double* out,
                     void* stream);

/* ---- psi / psi~ prototype tables (kernel_weights.py:243-295) --------------
 * Node integrals of every table subinterval: for subinterval s (kinds[2s] =
 * ansatz kind, kinds[2s+1] = test kind: 0 first, 1 inner, 2 last; a0w[2s],
 * a0w[2s+1] = start, width) and Lobatto node n, out[(((s*2 + v)*(p+1) + m1)*(p+1)
 * + m2)*nnodes + n] = the v = 0 (psi: b_i'') / v = 1 (psi~: b_i) integral against
 * the test basis' time derivative over the panels pptr[s]..pptr[s+1] (5 doubles
 * each: c0, s0, c1, s1, n_split; ends c + s*alpha).  Host buffers. */
int tdb_table_node_values(TdbContext* ctx, double dt, int32_t p, int32_t nsub, const int32_t* kinds, const double* a0w,
                          int32_t nnodes, const double* nodes, const int32_t* pptr, const double* panels, int32_t nq,
                          const double* xq, const double* wq, double* out);

#ifdef __cplusplus
}
#endif
#endif /* TDB_H_ */
