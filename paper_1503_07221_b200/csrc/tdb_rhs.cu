// Right-hand side contraction on the device.
//
// Replaces the inner loops of tdbem.assembly.assemble_rhs
// (/root/reference/pkg/src/tdbem/assembly.py:314-355):
//   b[(k-1) M + l] = sum_{time nodes j of basis k} w_j sum_{rule points p on l's star} s_{p,l} g(X_p, t_j)
// G = g(X, t_j) is evaluated by the caller on the device (node-major rows).  Two
// deterministic passes (no atomics):
//   stage 1  H[j][l] = sum_p s_{p,l} G[j][p]      (vertex gather of rule points, CSR)
//   stage 2  b[k][l] = sum_{j in nodes(k)} w_j H[j][l]   (the nodes of k are contiguous)
#include <cuda_runtime.h>

#include <algorithm>

#include "tdb_common.cuh"
#include "tdb_internal.h"

namespace {

__global__ void k_rhs_vertex(const double* __restrict__ G, long long j0, long long nj, long long P,
                             const long long* __restrict__ vptr, const int* __restrict__ vpts,
                             const double* __restrict__ vw, long long M, double* __restrict__ H) {
  const long long n = nj * M;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long j = i / M, l = i % M;
    const double* g = G + j * P;
    double s = 0.0;
    for (long long q = vptr[l]; q < vptr[l + 1]; ++q) s = fma(vw[q], g[vpts[q]], s);
    H[(j0 + j) * M + l] = s;
  }
}

__global__ void k_rhs_time(const double* __restrict__ H, const long long* __restrict__ kptr,
                           const double* __restrict__ w, long long L, long long M, double* __restrict__ out) {
  const long long n = L * M;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long k = i / M, l = i % M;
    double s = 0.0;
    for (long long j = kptr[k]; j < kptr[k + 1]; ++j) s = fma(w[j], H[j * M + l], s);
    out[i] = s;
  }
}

}  // namespace

extern "C" {

int tdb_rhs_vertex_gather(const double* G, int64_t j0, int64_t nj, int64_t P, const int64_t* vptr, const int32_t* vpts,
                          const double* vw, int64_t M, double* H, void* stream) {
  TDB_REQUIRE(G && vptr && vpts && vw && H && nj >= 0 && P >= 0 && M > 0 && j0 >= 0, "rhs_vertex_gather: bad argument");
  if (nj == 0) return TDB_OK;
  const long long n = nj * M;
  const int blocks = (int)std::min<long long>((n + 255) / 256, 148LL * 16);
  k_rhs_vertex<<<blocks, 256, 0, (cudaStream_t)stream>>>(G, j0, nj, P, (const long long*)vptr, vpts, vw, M, H);
  TDB_CUDA_CHECK(cudaGetLastError());
  return TDB_OK;
}

int tdb_rhs_time_sum(const double* H, const int64_t* kptr, const double* w, int64_t L, int64_t M, double* out,
                     void* stream) {
  TDB_REQUIRE(H && kptr && w && out && L > 0 && M > 0, "rhs_time_sum: bad argument");
  const long long n = L * M;
  const int blocks = (int)std::min<long long>((n + 255) / 256, 148LL * 16);
  k_rhs_time<<<blocks, 256, 0, (cudaStream_t)stream>>>(H, (const long long*)kptr, w, L, M, out);
  TDB_CUDA_CHECK(cudaGetLastError());
  return TDB_OK;
}

}  // extern "C"
