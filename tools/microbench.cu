// Microbenchmarks for the roofline denominators of the PIF kernels on B200
// (DESIGN.md "Roofline"): FP64 DFMA throughput and latency, shared-memory
// broadcast LDS rate, native fp64 global reduction (REDG.ADD.F64) rate into an
// L2-resident array, and fp64 shared-memory atomicAdd (CAS loop) rate.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/microbench.cu -o /tmp/mb
#include <cuda_runtime.h>
#include <stdio.h>

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e = (x);                                                   \
    if (e != cudaSuccess) {                                                \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      return 1;                                                            \
    }                                                                      \
  } while (0)

template <int CHAINS>
__global__ void dfma_tput(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void dfma_latency(double* out, int iters, double a, double b, long long* cyc) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    x = fma(x, a, b);
    x = fma(x, a, b);
    x = fma(x, a, b);
    x = fma(x, a, b);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (x == 12345.678) out[0] = x;
}

__global__ void redg_rate(double* grid, int mask, int iters) {
  unsigned idx = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u;
  for (int it = 0; it < iters; ++it) {
    atomicAdd(grid + ((idx + it * 97u) & mask), 1.0);
  }
}

__global__ void smem_atomic_rate(double* out, int iters) {
  __shared__ double s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = 0;
  __syncthreads();
  unsigned idx = threadIdx.x * 37u;
  for (int it = 0; it < iters; ++it) atomicAdd(&s[(idx + it * 131u) & 4095], 1.0);
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = s[0];
}

__global__ void lds_bcast_rate(double* out, int iters) {
  __shared__ double s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = i;
  __syncthreads();
  double acc0 = 0, acc1 = 0;
  int base = 0;
  for (int it = 0; it < iters; ++it) {
    double2 v = *reinterpret_cast<double2*>(&s[(base) & 1022]);
    acc0 += v.x;
    acc1 += v.y;
    base += 2;
  }
  if (acc0 + acc1 == 1.2345) out[0] = acc0;
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  int sms = p.multiProcessorCount;
  printf("device %s SMs %d\n", p.name, sms);
  double* d;
  CK(cudaMalloc(&d, 64 << 20));
  long long* cyc;
  CK(cudaMalloc(&cyc, 4096 * sizeof(long long)));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  // DFMA throughput: 8 chains x iters per thread
  {
    const int iters = 20000, threads = 256, blocks = sms * 8;
    dfma_tput<8><<<blocks, threads>>>(d, 10, 1.0000001, 1e-9);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dfma_tput<8><<<blocks, threads>>>(d, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * iters * (double)threads * blocks;
    printf("DFMA throughput: %.2f TFLOP/s (%.1f DFMA/clk/SM at %d MHz)\n", fl / ms / 1e9,
           fl / 2 / (ms * 1e-3) / sms / (p.clockRate * 1e3), p.clockRate / 1000);
  }
  for (int ch : {1, 2, 4}) {
    const int iters = 20000, threads = 256, blocks = sms * 8;
    cudaEventRecord(e0);
    if (ch == 1) dfma_tput<1><<<blocks, threads>>>(d, iters, 1.0000001, 1e-9);
    if (ch == 2) dfma_tput<2><<<blocks, threads>>>(d, iters, 1.0000001, 1e-9);
    if (ch == 4) dfma_tput<4><<<blocks, threads>>>(d, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * ch * iters * (double)threads * blocks;
    printf("DFMA %d chains x 64 warps/SM: %.2f TFLOP/s\n", ch, fl / ms / 1e9);
  }
  {
    const int iters = 10000;
    dfma_latency<<<1, 32>>>(d, iters, 1.0000001, 1e-9, cyc);
    CK(cudaDeviceSynchronize());
    long long c;
    cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
    printf("DFMA dependent latency: %.2f cycles\n", (double)c / (4.0 * iters));
  }
  // REDG f64 into an L2-resident 2 MB grid (random addresses)
  {
    const int iters = 256, threads = 256, blocks = sms * 16;
    const int mask = (1 << 18) - 1;  // 2 MB of doubles
    CK(cudaMemset(d, 0, 8 << 18));
    redg_rate<<<blocks, threads>>>(d, mask, 4);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    redg_rate<<<blocks, threads>>>(d, mask, iters);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double n = (double)iters * threads * blocks;
    printf("REDG.ADD.F64 (2 MB L2-resident, scattered): %.3g atomics/s\n", n / (ms * 1e-3));
  }
  {
    const int iters = 2048, threads = 256, blocks = sms * 4;
    cudaEventRecord(e0);
    smem_atomic_rate<<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double n = (double)iters * threads * blocks;
    printf("shared fp64 atomicAdd (CAS loop): %.3g atomics/s\n", n / (ms * 1e-3));
  }
  {
    const int iters = 100000, threads = 256, blocks = sms * 8;
    cudaEventRecord(e0);
    lds_bcast_rate<<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double n = (double)iters * (threads / 32) * blocks;
    printf("LDS.128 broadcast: %.2f warp-instr/clk/SM\n", n / (ms * 1e-3) / sms / (p.clockRate * 1e3));
  }
  return 0;
}
