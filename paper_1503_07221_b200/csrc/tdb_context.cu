// Context / system lifecycle and the C ABI wrappers (include/tdb.h).
#include <cuda_runtime.h>

#include <string>

#include "tdb_common.cuh"
#include "tdb_internal.h"

namespace tdb {
static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }
}  // namespace tdb

int tdb_system_create_impl(TdbContext* ctx, const TdbMesh* mesh, const TdbAssemblyDesc* desc,
                           TdbSystem* sys);
int tdb_system_run_impl(TdbSystem* sys);
int tdb_fp64_peak_impl(TdbContext* ctx, int repeats, double* tflops);
int tdb_tri_bounds_impl(TdbContext* ctx, const TdbMesh* mesh, int64_t nrows, const int64_t* rows,
                        double* tmin, double* tmax);

using namespace tdb;

extern "C" {

int tdb_abi_version(void) { return TDB_ABI_VERSION; }

const char* tdb_last_error(void) { return g_last_error.c_str(); }

int tdb_fp64_peak(TdbContext* ctx, int repeats, double* tflops) {
  TDB_REQUIRE(ctx && tflops, "NULL argument");
  TDB_CUDA_CHECK(cudaSetDevice(ctx->device));
  return tdb_fp64_peak_impl(ctx, repeats, tflops);
}

int tdb_device_count(int* count) {
  TDB_REQUIRE(count != nullptr, "count is NULL");
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) n = 0;
  *count = n;
  return TDB_OK;
}

int tdb_ctx_create(int device, TdbContext** out) {
  TDB_REQUIRE(out != nullptr, "out is NULL");
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    set_error("no CUDA device visible");
    return TDB_E_NODEVICE;
  }
  TDB_REQUIRE(device >= 0 && device < n, "device index out of range");
  TDB_CUDA_CHECK(cudaSetDevice(device));
  TdbContext* c = new TdbContext();
  c->device = device;
  c->stream = nullptr;
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  *out = c;
  return TDB_OK;
}

int tdb_ctx_destroy(TdbContext* ctx) {
  delete ctx;
  return TDB_OK;
}

int tdb_ctx_set_stream(TdbContext* ctx, void* stream) {
  TDB_REQUIRE(ctx != nullptr, "ctx is NULL");
  ctx->stream = static_cast<cudaStream_t>(stream);
  return TDB_OK;
}

int tdb_system_destroy(TdbSystem* sys) {
  if (!sys) return TDB_OK;
  if (sys->ctx) cudaSetDevice(sys->ctx->device);
  tdb_workspace_free(sys);
  cudaFree(sys->corners);
  cudaFree(sys->a2);
  cudaFree(sys->normals);
  cudaFree(sys->curls);
  cudaFree(sys->tri);
  cudaFree(sys->star_off);
  cudaFree(sys->star_ids);
  cudaFree(sys->famdev);
  for (auto& f : sys->fam) {
    cudaFree(f.indptr);
    cudaFree(f.indices);
    cudaFree(f.data);
    cudaFree(f.delta);
    cudaFree(f.slo);
    cudaFree(f.shi);
  }
  for (auto& b : sys->bsr) {
    cudaFree(b.col);
    cudaFree(b.val);
    cudaFree(b.rbptr);
  }
  cudaFree(sys->d_vperm);
  cudaFree(sys->d_vinv);
  cudaFree(sys->d_rperm);
  cudaFree(sys->d_rinv);
  delete sys;
  return TDB_OK;
}

int tdb_system_create(TdbContext* ctx, const TdbMesh* mesh, const TdbAssemblyDesc* desc,
                      TdbSystem** out) {
  TDB_REQUIRE(ctx && mesh && desc && out, "NULL argument");
  TDB_CUDA_CHECK(cudaSetDevice(ctx->device));
  TdbSystem* sys = new TdbSystem();
  sys->ctx = ctx;
  int rc = tdb_system_create_impl(ctx, mesh, desc, sys);
  if (rc != TDB_OK) {
    tdb_system_destroy(sys);
    return rc;
  }
  *out = sys;
  return TDB_OK;
}

int tdb_system_run(TdbSystem* sys) {
  TDB_REQUIRE(sys != nullptr, "NULL system");
  TDB_CUDA_CHECK(cudaSetDevice(sys->ctx->device));
  return tdb_system_run_impl(sys);
}

int tdb_system_assemble(TdbContext* ctx, const TdbMesh* mesh, const TdbAssemblyDesc* desc,
                        TdbSystem** out) {
  int rc = tdb_system_create(ctx, mesh, desc, out);
  if (rc != TDB_OK) return rc;
  rc = tdb_system_run(*out);
  if (rc != TDB_OK) {
    tdb_system_destroy(*out);
    *out = nullptr;
  }
  return rc;
}

int tdb_tri_distance_bounds(TdbContext* ctx, const TdbMesh* mesh, int64_t nrows,
                            const int64_t* rows, double* tmin, double* tmax) {
  TDB_REQUIRE(ctx && mesh && (nrows == 0 || (rows && tmin && tmax)), "NULL argument");
  TDB_CUDA_CHECK(cudaSetDevice(ctx->device));
  return tdb_tri_bounds_impl(ctx, mesh, nrows, rows, tmin, tmax);
}

int tdb_system_stats(const TdbSystem* sys, TdbStats* out) {
  TDB_REQUIRE(sys && out, "NULL argument");
  *out = sys->stats;
  return TDB_OK;
}

int tdb_system_family_nnz(const TdbSystem* sys, int32_t f, int64_t* nnz) {
  TDB_REQUIRE(sys && nnz, "NULL argument");
  TDB_REQUIRE(f >= 0 && f < sys->F, "family index out of range");
  *nnz = sys->fam[f].nnz;
  return TDB_OK;
}

int tdb_system_copy_family(const TdbSystem* sys, int32_t f, int64_t* indptr, int32_t* indices,
                           double* data) {
  TDB_REQUIRE(sys != nullptr, "NULL system");
  TDB_REQUIRE(f >= 0 && f < sys->F, "family index out of range");
  const FamilyStore& fs = sys->fam[f];
  TDB_CUDA_CHECK(cudaSetDevice(sys->ctx->device));
  const size_t nrows = (size_t)fs.npos * sys->nrows;
  if (indptr)
    TDB_CUDA_CHECK(cudaMemcpy(indptr, fs.indptr, (nrows + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost));
  if (indices && fs.nnz)
    TDB_CUDA_CHECK(cudaMemcpy(indices, fs.indices, fs.nnz * sizeof(int32_t), cudaMemcpyDeviceToHost));
  if (data && fs.nnz)
    TDB_CUDA_CHECK(cudaMemcpy(data, fs.data, fs.nnz * sys->nm * sizeof(double), cudaMemcpyDeviceToHost));
  return TDB_OK;
}

int tdb_system_family_device(const TdbSystem* sys, int32_t f, const int64_t** indptr_dev,
                             const int32_t** indices_dev, const double** data_dev) {
  TDB_REQUIRE(sys != nullptr, "NULL system");
  TDB_REQUIRE(f >= 0 && f < sys->F, "family index out of range");
  if (indptr_dev) *indptr_dev = sys->fam[f].indptr;
  if (indices_dev) *indices_dev = sys->fam[f].indices;
  if (data_dev) *data_dev = sys->fam[f].data;
  return TDB_OK;
}

}  // extern "C"
