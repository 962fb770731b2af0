// FP64 tensor-core (DMMA, mma.sync m8n8k4 f64) throughput on B200 vs DFMA.
#include <cuda_runtime.h>
#include <stdio.h>
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
template <int ACC>
__global__ void dmma_tput(double* out, int iters) {
  double c[ACC][2];
  double a = 1.0 + threadIdx.x * 1e-6, b = 0.999999;
#pragma unroll
  for (int i = 0; i < ACC; ++i) c[i][0] = c[i][1] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) dmma(c[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[0] = s;
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  double* d; cudaMalloc(&d, 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int warps : {4, 8, 16, 32}) {
    const int iters = 20000, blocks = p.multiProcessorCount;
    dmma_tput<8><<<blocks, warps * 32>>>(d, 10);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    dmma_tput<8><<<blocks, warps * 32>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 256 * 8 * (double)iters * warps * blocks;
    printf("DMMA m8n8k4 f64, %d warps/SM x 8 acc: %.2f TFLOP/s  (%s)\n", warps, fl / ms / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
