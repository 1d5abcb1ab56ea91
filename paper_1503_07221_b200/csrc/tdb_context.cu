// Context / system lifecycle and the C ABI wrappers (include/tdb.h).
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "tdb_common.cuh"
#include "tdb_internal.h"

namespace tdb {
static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }

// ---- caching device allocator --------------------------------------------
// Repeated assemble/destroy cycles (the public API builds a fresh system per
// call) would otherwise pay cudaMalloc/cudaFree of GB-sized workspaces every
// time.  Freed blocks are kept per device (size-rounded, at most kPoolCap bytes
// cached) and reused best-fit; an allocation failure releases the cache and
// retries.  Callers release blocks only after their stream is idle.
namespace {
constexpr size_t kPoolCap = 8ull << 30;
struct Pool {
  std::mutex mu;
  std::unordered_map<void*, std::pair<size_t, int>> live;  // ptr -> (bytes, device)
  std::map<std::pair<int, size_t>, std::vector<void*>> cached;  // (device, bytes) -> blocks
  size_t cached_bytes = 0;
};
Pool& pool() {
  static Pool* p = new Pool();  // never destroyed (may be used during process teardown)
  return *p;
}
size_t round_bytes(size_t b) {
  if (b <= (1u << 20)) return (b + 511) & ~size_t(511);
  return (b + (2u << 20) - 1) & ~size_t((2u << 20) - 1);
}
void trim_locked(Pool& P) {
  for (auto& kv : P.cached)
    for (void* q : kv.second) cudaFree(q);
  P.cached.clear();
  P.cached_bytes = 0;
}
}  // namespace

cudaError_t dev_malloc(void** out, size_t bytes) {
  Pool& P = pool();
  int dev = 0;
  cudaGetDevice(&dev);
  const size_t b = round_bytes(bytes == 0 ? 1 : bytes);
  std::lock_guard<std::mutex> g(P.mu);
  auto it = P.cached.lower_bound({dev, b});
  if (it != P.cached.end() && it->first.first == dev && it->first.second <= b + b / 4 && !it->second.empty()) {
    void* q = it->second.back();
    const size_t have = it->first.second;
    it->second.pop_back();
    if (it->second.empty()) P.cached.erase(it);
    P.cached_bytes -= have;
    P.live[q] = {have, dev};
    *out = q;
    return cudaSuccess;
  }
  cudaError_t e = cudaMalloc(out, b);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    trim_locked(P);
    e = cudaMalloc(out, b);
  }
  if (e == cudaSuccess) P.live[*out] = {b, dev};
  return e;
}

void dev_free(void* q) {
  if (!q) return;
  Pool& P = pool();
  std::lock_guard<std::mutex> g(P.mu);
  auto it = P.live.find(q);
  if (it == P.live.end()) {  // not ours
    cudaFree(q);
    return;
  }
  const size_t b = it->second.first;
  const int dev = it->second.second;
  P.live.erase(it);
  if (P.cached_bytes + b > kPoolCap) {
    cudaFree(q);
    return;
  }
  P.cached[{dev, b}].push_back(q);
  P.cached_bytes += b;
}

void dev_pool_trim() {
  Pool& P = pool();
  std::lock_guard<std::mutex> g(P.mu);
  trim_locked(P);
}
}  // namespace tdb

int tdb_system_create_impl(TdbContext* ctx, const TdbMesh* mesh, const TdbAssemblyDesc* desc,
                           TdbSystem* sys);
int tdb_system_run_impl(TdbSystem* sys);
int tdb_fp64_peak_impl(TdbContext* ctx, int repeats, double* tflops);
int tdb_position_units_impl(TdbSystem* sys, int f, int64_t* out);
int tdb_tri_bounds_impl(TdbContext* ctx, const TdbMesh* mesh, int64_t nrows, const int64_t* rows,
                        double* tmin, double* tmax);

using namespace tdb;

extern "C" {

int tdb_abi_version(void) { return TDB_ABI_VERSION; }

int tdb_release_cached_memory(void) {
  dev_pool_trim();
  return TDB_OK;
}

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
  if (sys->ctx) {
    cudaSetDevice(sys->ctx->device);
    cudaStreamSynchronize(sys->ctx->stream);  // blocks go back to the pool
  }
  tdb_workspace_free(sys);
  dev_free(sys->corners);
  dev_free(sys->a2);
  dev_free(sys->normals);
  dev_free(sys->curls);
  dev_free(sys->tri);
  dev_free(sys->star_off);
  dev_free(sys->star_ids);
  dev_free(sys->famdev);
  for (auto& f : sys->fam) {
    dev_free(f.indptr);
    dev_free(f.indices);
    dev_free(f.data);
    dev_free(f.delta);
    dev_free(f.slo);
    dev_free(f.shi);
  }
  for (auto& b : sys->band) {
    dev_free(b.tiles);
    dev_free(b.rbptr);
    for (auto& v : b.views) {
      dev_free(v.tiles);
      dev_free(v.rbptr);
    }
  }
  dev_free(sys->d_vperm);
  dev_free(sys->d_vinv);
  dev_free(sys->d_rperm);
  dev_free(sys->d_rinv);
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

int tdb_system_position_units(TdbSystem* sys, int32_t f, int64_t* units) {
  TDB_REQUIRE(sys && units, "NULL argument");
  TDB_REQUIRE(f >= 0 && f < sys->F, "family index out of range");
  TDB_CUDA_CHECK(cudaSetDevice(sys->ctx->device));
  return tdb_position_units_impl(sys, f, units);
}

int tdb_system_family_split(const TdbSystem* sys, int32_t f, int32_t* R, int32_t* D, int32_t* K) {
  TDB_REQUIRE(sys && R && D && K, "NULL argument");
  TDB_REQUIRE(f >= 0 && f < sys->F, "family index out of range");
  *R = sys->fam[f].split_R;
  *D = sys->fam[f].split_D;
  *K = sys->fam[f].split_K;
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
