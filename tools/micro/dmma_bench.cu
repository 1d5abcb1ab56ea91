// DMMA (mma.sync m8n8k4 f64) vs DFMA throughput microbenchmark.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int NACC>
__global__ void k_dmma(double* out, int iters) {
  double acc[NACC][2];
  for (int i = 0; i < NACC; ++i) acc[i][0] = acc[i][1] = threadIdx.x * 1e-3;
  double a = 1.0 + threadIdx.x * 1e-6, b = 0.999;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) dmma(acc[i][0], acc[i][1], a, b);
  }
  double s = 0;
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int NACC>
__global__ void k_dfma(double* out, int iters) {
  double acc[NACC];
  for (int i = 0; i < NACC; ++i) acc[i] = threadIdx.x * 1e-3;
  double a = 1.0 + threadIdx.x * 1e-6, b = 0.999;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = fma(acc[i], b, a);
  }
  double s = 0;
  for (int i = 0; i < NACC; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double* out;
  cudaMalloc(&out, 148 * 8 * 1024 * sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps : {4, 8, 16}) {
    const int iters = 20000;
    k_dmma<8><<<148 * 2, warps * 32>>>(out, 100);
    cudaEventRecord(e0);
    k_dmma<8><<<148 * 2, warps * 32>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256 * 8 * (double)iters * 148 * 2 * warps;
    printf("DMMA m8n8k4: %2d warps/CTA x 2 CTA/SM: %.2f TFLOP/s (%.3f ms)\n", warps, flops / ms / 1e9, ms);
    k_dfma<8><<<148 * 2, warps * 32>>>(out, 100);
    cudaEventRecord(e0);
    k_dfma<8><<<148 * 2, warps * 32>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 8 * (double)iters * 148 * 2 * warps * 32;
    printf("DFMA       : %2d warps/CTA x 2 CTA/SM: %.2f TFLOP/s (%.3f ms)\n", warps, flops / ms / 1e9, ms);
  }
  printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
