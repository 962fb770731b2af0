// DMMA / DFMA interleaving on B200: throughput of DMMA-only, DFMA-only, mixed
// (independent), and DMMA results consumed by DFMA (dependent).
#include <cuda_runtime.h>
#include <stdio.h>
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
template <int MODE, int NF>
__global__ void k(double* out, int iters) {
  double c[8][2], f[8];
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.9999999;
  for (int i = 0; i < 8; ++i) { c[i][0] = c[i][1] = i; f[i] = i; }
  for (int it = 0; it < iters; ++it) {
    if (MODE != 1)
#pragma unroll
      for (int i = 0; i < 8; ++i) dmma(c[i], a, b);
    if (MODE == 1 || MODE == 2)
#pragma unroll
      for (int j = 0; j < NF; ++j) f[j % 8] = fma(f[j % 8], b, a);
    if (MODE == 3)  // consume accumulators with DFMA (dependent)
#pragma unroll
      for (int j = 0; j < NF; ++j) f[j % 8] = fma(c[j % 8][j & 1], b, f[j % 8]);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + f[i];
  if (s == 1.2345) out[0] = s;
}
template <int MODE, int NF>
float run(double* d, int warps, int iters) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<MODE, NF><<<148, warps * 32>>>(d, 10);
  cudaEventRecord(e0);
  k<MODE, NF><<<148, warps * 32>>>(d, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); return ms;
}
int main() {
  double* d; cudaMalloc(&d, 64);
  const int it = 20000;
  for (int w : {8, 16}) {
    float t0 = run<0, 8>(d, w, it);
    float t1 = run<1, 8>(d, w, it);
    float t2 = run<2, 8>(d, w, it);
    float t3 = run<3, 8>(d, w, it);
    float t1b = run<1, 32>(d, w, it);
    float t2b = run<2, 32>(d, w, it);
    printf("warps/SM %d: DMMAx8 %.3f ms | DFMAx8 %.3f | mixed 8+8 %.3f | dependent 8+8 %.3f | DFMAx32 %.3f | mixed 8+32 %.3f\n",
           w, t0, t1, t2, t3, t1b, t2b);
  }
  return 0;
}
