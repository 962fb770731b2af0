// a11: CIC-PIC deposit and gather+push (reading R14);
// a12: parareal correction + stopping norms (eq. parareal_correction P:154-161,
// eq. stop_criteria); the test-only push and a finiteness check.
#include "pif_internal.cuh"

namespace pif {

__device__ __forceinline__ void cic_1d(double x, double inv_h, int Ng, int& i0, int& i1,
                                       double& w0, double& w1) {
  double s = x * inv_h;
  double fi = floor(s);
  double f = s - fi;
  int i = (int)fi;
  i0 = ((i % Ng) + Ng) % Ng;
  i1 = i0 + 1 == Ng ? 0 : i0 + 1;
  w0 = 1.0 - f;
  w1 = f;
}

// rho_p += W_pj (the q / h^3 factor is applied in the Poisson kernel).
__global__ void k_cic_deposit(const double* __restrict__ x, int64_t stride, int64_t n, int Ng,
                              double inv_h, double* __restrict__ grid) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  int i0[3], i1[3];
  double w0[3], w1[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) cic_1d(x[d * stride + j], inv_h, Ng, i0[d], i1[d], w0[d], w1[d]);
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    int ix = (c & 4) ? i1[0] : i0[0];
    int iy = (c & 2) ? i1[1] : i0[1];
    int iz = (c & 1) ? i1[2] : i0[2];
    double wt = ((c & 4) ? w1[0] : w0[0]) * ((c & 2) ? w1[1] : w0[1]) * ((c & 1) ? w1[2] : w0[2]);
    atomicAdd(grid + ((int64_t)ix * Ng + iy) * Ng + iz, wt);
  }
}

// Shared-memory deposit for small grids (N_g <= 32, the C5 coarse grid): the
// grid's z range is cut into NZC chunks of ZC planes (N_g^2 ZC doubles <= 128 KB
// of shared memory); blockIdx.y = chunk.  A CTA accumulates the weights of its
// particles (grid-stride over blockIdx.x) that land in its chunk in shared
// memory, then flushes the chunk with one REDG.ADD.F64 per non-zero node: 8
// global atomics per particle become 8 shared ones plus N_g^2 ZC global ones
// per CTA, and no two particles contend in L2.
__global__ void __launch_bounds__(512) k_cic_deposit_smem(const double* __restrict__ x, int64_t stride,
                                                          int64_t n, int Ng, int ZC, double inv_h,
                                                          double* __restrict__ grid) {
  extern __shared__ double tile[];
  const int z0 = blockIdx.y * ZC;
  const int nt = Ng * Ng * ZC;
  for (int i = threadIdx.x; i < nt; i += blockDim.x) tile[i] = 0.0;
  __syncthreads();
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    int i0[3], i1[3];
    double w0[3], w1[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) cic_1d(x[d * stride + j], inv_h, Ng, i0[d], i1[d], w0[d], w1[d]);
#pragma unroll
    for (int cz = 0; cz < 2; ++cz) {
      const int iz = (cz ? i1[2] : i0[2]) - z0;
      if (iz < 0 || iz >= ZC) continue;
      const double wz = cz ? w1[2] : w0[2];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int ix = (c & 2) ? i1[0] : i0[0];
        const int iy = (c & 1) ? i1[1] : i0[1];
        const double wt = ((c & 2) ? w1[0] : w0[0]) * ((c & 1) ? w1[1] : w0[1]) * wz;
        atomicAdd(&tile[(ix * Ng + iy) * ZC + iz], wt);
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nt; i += blockDim.x) {
    const double val = tile[i];
    if (val != 0.0) {
      const int iz = i % ZC, xy = i / ZC;
      atomicAdd(grid + (int64_t)xy * Ng + z0 + iz, val);
    }
  }
}

// E on the nodes interleaved, {E_x, E_y, E_z, 0} per node (one 32-byte sector):
// the gather's 8 nodes x 3 components become 8 sector reads instead of 24.
__global__ void k_pic_interleave(const double* __restrict__ g3, int64_t npts, double4* __restrict__ gi) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < npts;
       j += (int64_t)gridDim.x * blockDim.x)
    gi[j] = make_double4(g3[j], g3[npts + j], g3[2 * npts + j], 0.0);
}

__global__ void k_cic_gather_push(const double4* __restrict__ gi, double* __restrict__ x,
                                  double* __restrict__ v, int64_t stride, int64_t n, int Ng,
                                  double inv_h, PushArgs P) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  double x0 = x[j], x1 = x[stride + j], x2 = x[2 * stride + j];
  int i0[3], i1[3];
  double w0[3], w1[3];
  cic_1d(x0, inv_h, Ng, i0[0], i1[0], w0[0], w1[0]);
  cic_1d(x1, inv_h, Ng, i0[1], i1[1], w0[1], w1[1]);
  cic_1d(x2, inv_h, Ng, i0[2], i1[2], w0[2], w1[2]);
  double E0 = 0, E1 = 0, E2 = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    int ix = (c & 4) ? i1[0] : i0[0];
    int iy = (c & 2) ? i1[1] : i0[1];
    int iz = (c & 1) ? i1[2] : i0[2];
    double wt = ((c & 4) ? w1[0] : w0[0]) * ((c & 2) ? w1[1] : w0[1]) * ((c & 1) ? w1[2] : w0[2]);
    const double2* node = reinterpret_cast<const double2*>(gi + ((int64_t)ix * Ng + iy) * Ng + iz);
    const double2 exy = __ldg(node);
    const double ez = __ldg(reinterpret_cast<const double*>(node + 1));
    E0 += wt * exy.x;
    E1 += wt * exy.y;
    E2 += wt * ez;
  }
  double v0 = v[j], v1 = v[stride + j], v2 = v[2 * stride + j];
  push_particle(x0, x1, x2, v0, v1, v2, E0, E1, E2, P);
  x[j] = x0;
  x[stride + j] = x1;
  x[2 * stride + j] = x2;
  v[j] = v0;
  v[stride + j] = v1;
  v[2 * stride + j] = v2;
}

__global__ void k_push_only(double* __restrict__ x, double* __restrict__ v,
                            const double* __restrict__ E, int64_t stride, int64_t n, PushArgs P) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  double x0 = x[j], x1 = x[stride + j], x2 = x[2 * stride + j];
  double v0 = v[j], v1 = v[stride + j], v2 = v[2 * stride + j];
  push_particle(x0, x1, x2, v0, v1, v2, E[j], E[stride + j], E[2 * stride + j], P);
  x[j] = x0;
  x[stride + j] = x1;
  x[2 * stride + j] = x2;
  v[j] = v0;
  v[stride + j] = v1;
  v[2 * stride + j] = v2;
}

// Canonical states: [x0..|x1..|x2..|v0..|v1..|v2..], 6n doubles.
// U = F + Gn - Go (x wrapped, R17); partial sums of
// {|mi(Gn.x - Go.x)|^2, |Gn.x|^2, |Gn.v - Go.v|^2, |Gn.v|^2} (eq. stop_criteria).
__device__ __forceinline__ void block_sum4_m(double a[4], double* __restrict__ dst) {
  __shared__ double sh[4][32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a[q] += __shfl_xor_sync(0xffffffffu, a[q], o);
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < 4; ++q) sh[q][wid] = a[q];
  __syncthreads();
  if (threadIdx.x == 0)
    for (int q = 0; q < 4; ++q) {
      double s = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sh[q][w];
      dst[q] = s;
    }
}

__global__ void __launch_bounds__(256) k_correct_norms(const double* __restrict__ F,
                                                       const double* __restrict__ Gn,
                                                       const double* __restrict__ Go,
                                                       double* __restrict__ U, int64_t n, double L,
                                                       double* __restrict__ partials) {
  double a[4] = {0, 0, 0, 0};
  const int64_t tot = 3 * n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot;
       i += (int64_t)gridDim.x * blockDim.x) {
    // positions
    double gn = Gn[i], go = Go[i];
    double ux = (F[i] + gn) - go;
    if (U) U[i] = wrapL(ux, L);
    double d = gn - go;
    d = d - L * rint(d / L);
    a[0] += d * d;
    a[1] += gn * gn;
    // velocities
    double hn = Gn[tot + i], ho = Go[tot + i];
    if (U) U[tot + i] = (F[tot + i] + hn) - ho;
    double e = hn - ho;
    a[2] += e * e;
    a[3] += hn * hn;
  }
  block_sum4_m(a, partials + 4 * blockIdx.x);
}

__global__ void __launch_bounds__(256) k_reduce4(const double* __restrict__ partials, int nparts,
                                                 double* __restrict__ out4) {
  double a[4] = {0, 0, 0, 0};
  for (int i = threadIdx.x; i < nparts; i += blockDim.x)
#pragma unroll
    for (int q = 0; q < 4; ++q) a[q] += partials[4 * i + q];
  block_sum4_m(a, out4);
}

// flag <- 1 if any a[i] is non-finite; L > 0: also wrap a[i] into [0, L) in
// place (positions given outside the periodic box, any number of periods).
__global__ void k_check_finite(double* __restrict__ a, int64_t count, double L, int* flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double y = a[i];
    if (!isfinite(y)) atomicExch(flag, 1);
    else if (L > 0.0 && !(y >= 0.0 && y < L)) a[i] = wrapL(y, L);
  }
}

// fp64 <-> fp32 staging for the fp32 density all-reduce (PIF_FLAG_FP32_ALLREDUCE)
__global__ void k_convert(double* __restrict__ d, float* __restrict__ f, int64_t count, int to_float) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (to_float) f[i] = (float)d[i];
    else d[i] = (double)f[i];
  }
}

static inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

cudaError_t launch_convert(double* d, float* f, int64_t count, bool to_float, cudaStream_t st) {
  k_convert<<<kReduceBlocks, 256, 0, st>>>(d, f, count, to_float ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_cic_deposit(const double* x, int64_t stride, int64_t n, int Ng, double inv_h,
                               double* grid, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
#ifndef PIF_CIC_SMEM
#define PIF_CIC_SMEM 1
#endif
  if (PIF_CIC_SMEM && Ng <= 32) {
    const int ZC = Ng < 16 ? Ng : 16, NZC = Ng / ZC;
    const size_t smem = (size_t)Ng * Ng * ZC * sizeof(double);
    static DevCache cache;
    int ctas = 0;  // resident 512-thread CTAs on the device
    cudaError_t e = dev_cached(cache, ctas, [&](int dev, int& val) {
      int sms = 0, per = 0;
      cudaError_t r = cudaFuncSetAttribute(k_cic_deposit_smem, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)(32 * 32 * 16 * sizeof(double)));
      if (r == cudaSuccess) r = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      if (r == cudaSuccess)
        r = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_cic_deposit_smem, 512, 32 * 32 * 16 * sizeof(double));
      val = sms * (per > 0 ? per : 1);
      return r;
    });
    if (e != cudaSuccess) return e;
    // enough particles per CTA that the chunk flush (Ng^2 ZC REDG) stays small
    int64_t bx = std::min<int64_t>((n + 8191) / 8192, std::max(1, ctas / NZC));
    k_cic_deposit_smem<<<dim3((unsigned)bx, NZC), 512, smem, st>>>(x, stride, n, Ng, ZC, inv_h, grid);
    return cudaGetLastError();
  }
  k_cic_deposit<<<nblk(n, 256), 256, 0, st>>>(x, stride, n, Ng, inv_h, grid);
  return cudaGetLastError();
}
cudaError_t launch_cic_gather_push(const double* grid3, double* grid4, double* x, double* v,
                                   int64_t stride, int64_t n, int Ng, double inv_h, const PushArgs& P,
                                   cudaStream_t st) {
  const int64_t npts = (int64_t)Ng * Ng * Ng;
  k_pic_interleave<<<nblk(npts, 256) < 1184 ? nblk(npts, 256) : 1184, 256, 0, st>>>(grid3, npts,
                                                                                  (double4*)grid4);
  if (n > 0)
    k_cic_gather_push<<<nblk(n, 256), 256, 0, st>>>((const double4*)grid4, x, v, stride, n, Ng, inv_h, P);
  return cudaGetLastError();
}
cudaError_t launch_push_only(double* x, double* v, const double* E, int64_t stride, int64_t n,
                             const PushArgs& P, cudaStream_t st) {
  if (n > 0) k_push_only<<<nblk(n, 256), 256, 0, st>>>(x, v, E, stride, n, P);
  return cudaGetLastError();
}
cudaError_t launch_correct_norms(const double* F, const double* Gn, const double* Go, double* U,
                                 int64_t n, double L, double* partials, double* out4,
                                 cudaStream_t st) {
  k_correct_norms<<<kReduceBlocks, 256, 0, st>>>(F, Gn, Go, U, n, L, partials);
  k_reduce4<<<1, 256, 0, st>>>(partials, kReduceBlocks, out4);
  return cudaGetLastError();
}
cudaError_t launch_check_finite(double* a, int64_t count, double wrap_L, int* flag, cudaStream_t st) {
  k_check_finite<<<kReduceBlocks, 256, 0, st>>>(a, count, wrap_L, flag);
  return cudaGetLastError();
}

}  // namespace pif
