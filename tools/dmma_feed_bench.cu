// How fast can a warp feed DMMA (mma.sync m8n8k4 f64) from shared memory?
// Models the k_interp_push inner loop: per k-step one A element (psi_x * psi_y,
// two LDS + DMUL) and NT*3 = 6 B fragments from a 75 KB smem tile.
//   V0: B from registers (A from smem)        -- upper bound
//   V1: one LDS.64 per DMMA (current kernel)
//   V2: two m-tiles per pass: each B LDS.64 feeds 2 DMMAs
//   V3: one LDS.128 per 2 DMMAs (B of n-tiles 0 and 1 adjacent per lane)
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/dmma_feed_bench.cu -o tools/dmma_feed_bench
#include <cuda_runtime.h>
#include <stdio.h>

constexpr int KS = 49, NT = 2, NW = 16, SX = 20;
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

template <int V>
__global__ void __launch_bounds__(512, 1) feed(double* out, int reps) {
  extern __shared__ double sm[];
  double* gB = sm;                         // [KS][NT][3][32]
  double* psi = sm + KS * NT * 3 * 32;     // [NW][2][8][SX] px / py rows
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, gr = lane >> 2, tq = lane & 3;
  for (int i = threadIdx.x; i < KS * NT * 3 * 32 + NW * 2 * 8 * SX * 2; i += blockDim.x)
    sm[i] = 1.0 + 1e-9 * i;
  __syncthreads();
  const double* px = psi + wid * 2 * 8 * SX * 2 + gr * SX;
  const double* py = px + 8 * SX;
  const double* px2 = py + 8 * SX;
  const double* py2 = px2 + 8 * SX;
  constexpr int MT = V == 2 ? 2 : 1;
  double acc[MT][NT][3][2];
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int d = 0; d < 3; ++d) acc[m][nt][d][0] = acc[m][nt][d][1] = 0.0;
    int cx = tq, cy = 0;
#pragma unroll 2
    for (int ks = 0; ks < KS; ++ks) {
      const double a = px[cx] * py[cy];
      const double a2 = V == 2 ? px2[cx] * py2[cy] : 0.0;
      cx += 4;
      if (cx >= 14) { cx -= 14; cy += 1; }
      if (V == 3) {
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const double2 b = *reinterpret_cast<const double2*>(gB + ((ks * 3 + d) * 32 + lane) * 2);
          dmma(acc[0][0][d], a, b.x);
          dmma(acc[0][1][d], a, b.y);
        }
      } else {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            const double b = V == 0 ? 0.5 + 1e-9 * (nt * 3 + d) : gB[((ks * NT + nt) * 3 + d) * 32 + lane];
            dmma(acc[0][nt][d], a, b);
            if (V == 2) dmma(acc[MT - 1][nt][d], a2, b);
          }
      }
    }
    double s = 0;
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int d = 0; d < 3; ++d) s += acc[m][nt][d][0] + acc[m][nt][d][1];
    if (s == 1.2345) out[threadIdx.x] = s;
  }
}

template <int V>
void run(const char* name, int sms, int warps = 8, int per_sm = 2) {
  const size_t smem = (KS * NT * 3 * 32 + NW * 2 * 8 * SX * 2) * sizeof(double);
  cudaFuncSetAttribute(feed<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  double* d;
  cudaMalloc(&d, 4096);
  const int reps = 400, blocks = per_sm * sms;
  feed<V><<<blocks, 32 * warps, smem>>>(d, 2);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  feed<V><<<blocks, 32 * warps, smem>>>(d, reps);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const int MT = V == 2 ? 2 : 1;
  const double fl = 2.0 * 256 * KS * NT * 3 * MT * (double)reps * warps * blocks;
  printf("%-34s %2d warps x %d CTA/SM: %.2f TFLOP/s (%s, smem %zu B)\n", name, warps, per_sm, fl / ms / 1e9,
         cudaGetErrorString(cudaGetLastError()), smem);
  cudaFree(d);
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  for (int w : {4, 8, 16}) {
    run<0>("V0 B in registers", sms, w, 1);
    run<1>("V1 LDS.64 per DMMA (interp)", sms, w, 1);
    run<2>("V2 2 m-tiles per B LDS.64", sms, w, 1);
    run<3>("V3 LDS.128 per 2 DMMA", sms, w, 1);
  }
  return 0;
}
