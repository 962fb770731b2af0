// a3 deconvolve/truncate, a5 Poisson + type-2 pre-correction + Hermitian pad,
// field-energy and particle-moment reductions, PIC Poisson.
//
// Spectral layouts (cuFFT D2Z of a row-major [x][y][z] real n^3 array):
// spec[(ix * n + iy) * (n/2+1) + iz], mode m_d = i_d for i_d < n/2 else i_d - n
// (x, y); m_z = iz >= 0.  The mode box kept on device is the Hermitian half
// box mx, my in [-N/2, N/2], mz in [0, N/2]: box[((mx+N/2)*(N+1) + my+N/2)*(N/2+1) + mz]
// (reading R2: the (N+1)^2 (N/2+1) box holds every K_N mode and its partner).
#include <math.h>

#include "pif_internal.cuh"

namespace pif {

template <typename C2>
__device__ __forceinline__ C2 cplx(double re, double im) {
  if constexpr (sizeof(C2) == 8) return make_float2((float)re, (float)im);
  else return make_double2(re, im);
}

__device__ __forceinline__ int64_t spec_index(int mx, int my, int mz, int n) {
  int ix = mx < 0 ? mx + n : mx;
  int iy = my < 0 ? my + n : my;
  return ((int64_t)ix * n + iy) * (n / 2 + 1) + mz;
}

// rho_tilde_k = scale * F[k] / (psi^(kx) psi^(ky) psi^(kz))   (type-1 deconvolution;
// scale = q / L^3 gives eq. scatter_pif without S_k).
__global__ void k_extract_box(const double2* __restrict__ spec, int n, int N,
                              const double* __restrict__ cor, double scale,
                              double2* __restrict__ box) {
  const int H = N / 2, NB = N + 1, NZ = H + 1;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)NB * NB * NZ) return;
  int mz = (int)(i % NZ);
  int my = (int)((i / NZ) % NB) - H;
  int mx = (int)(i / ((int64_t)NZ * NB)) - H;
  double2 f = spec[spec_index(mx, my, mz, n)];
  double c = scale * cor[mx + H] * cor[my + H] * cor[mz + H];
  box[i] = make_double2(f.x * c, f.y * c);
}

// omega_k = (1[k in K_N] + 1[-k in K_N]) / 2 on [-N/2, N/2]^3 (reading R2).
__device__ __forceinline__ double completion_weight(int mx, int my, int mz, int H) {
  bool in = (mx < H) && (my < H) && (mz < H) && (mx >= -H) && (my >= -H) && (mz >= -H);
  bool neg = (mx > -H) && (my > -H) && (mz > -H) && (mx <= H) && (my <= H) && (mz <= H);
  return 0.5 * ((in ? 1.0 : 0.0) + (neg ? 1.0 : 0.0));
}

// G_d[k] = omega_k S_k E_{d,k} / psi^(k), E_{d,k} = -i k_d S_k rho_tilde_k / |k|^2,
// k = 0 -> 0 (eq. gather_pif); zero outside the box.
template <typename C2>
__global__ void k_poisson_pad(const double2* __restrict__ box, int n, int N, double L,
                              const double* __restrict__ cor, const double* __restrict__ S,
                              C2* __restrict__ G3) {
  const int H = N / 2, NB = N + 1, NZ = H + 1, nz = n / 2 + 1;
  const int64_t tot = (int64_t)n * n * nz;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= tot) return;
  int iz = (int)(i % nz);
  int iy = (int)((i / nz) % n);
  int ix = (int)(i / ((int64_t)nz * n));
  int mx = ix < n / 2 ? ix : ix - n;
  int my = iy < n / 2 ? iy : iy - n;
  int mz = iz;
  double2 g0 = make_double2(0.0, 0.0), g1 = g0, g2 = g0;
  if (mx >= -H && mx <= H && my >= -H && my <= H && mz <= H && (mx | my | mz) != 0) {
    double2 r = box[((int64_t)(mx + H) * NB + (my + H)) * NZ + mz];
    const double k0 = 2.0 * M_PI / L;
    double kx = k0 * mx, ky = k0 * my, kz = k0 * mz;
    double Sk = S[mx + H] * S[my + H] * S[mz + H];
    double w = completion_weight(mx, my, mz, H);
    // coefficient multiplying (-i k_d) rho_tilde: omega S_k^2 / (|k|^2 psi^)
    double f = w * Sk * Sk * cor[mx + H] * cor[my + H] * cor[mz + H] / (kx * kx + ky * ky + kz * kz);
    // -i k (a + ib) = k b - i k a
    g0 = make_double2(f * kx * r.y, -f * kx * r.x);
    g1 = make_double2(f * ky * r.y, -f * ky * r.x);
    g2 = make_double2(f * kz * r.y, -f * kz * r.x);
  }
  G3[i] = cplx<C2>(g0.x, g0.y);
  G3[tot + i] = cplx<C2>(g1.x, g1.y);
  G3[2 * tot + i] = cplx<C2>(g2.x, g2.y);
}

// Debug type-1 output on K_N in (mx, my, mz) row-major order, no scale.
__global__ void k_debug_extract_KN(const double2* __restrict__ spec, int n, int N,
                                   const double* __restrict__ cor, double2* __restrict__ out) {
  const int H = N / 2;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)N * N * N) return;
  int mz = (int)(i % N) - H;
  int my = (int)((i / N) % N) - H;
  int mx = (int)(i / ((int64_t)N * N)) - H;
  double c = cor[mx + H] * cor[my + H] * cor[mz + H];
  double2 f;
  if (mz >= 0) {
    f = spec[spec_index(mx, my, mz, n)];
  } else {  // F[-m] = conj(F[m]) for a real grid
    int ax = -mx, ay = -my;
    ax = ax >= n / 2 ? ax - n : ax;  // -(-N/2) = N/2 stays N/2 (n >= 2N)
    ay = ay >= n / 2 ? ay - n : ay;
    double2 g = spec[spec_index(ax, ay, -mz, n)];
    f = make_double2(g.x, -g.y);
  }
  out[i] = make_double2(f.x * c, f.y * c);
}

// Debug type-2 input: c on K_N -> G (component 0) = c^box / psi^ on the half
// spectrum, c^box_k = (c_k 1[k in K_N] + conj(c_{-k}) 1[-k in K_N]) / 2 (R2).
template <typename C2>
__global__ void k_debug_pad_KN(const double2* __restrict__ c, int n, int N,
                               const double* __restrict__ cor, C2* __restrict__ G3) {
  const int H = N / 2, nz = n / 2 + 1;
  const int64_t tot = (int64_t)n * n * nz;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= tot) return;
  int iz = (int)(i % nz);
  int iy = (int)((i / nz) % n);
  int ix = (int)(i / ((int64_t)nz * n));
  int mx = ix < n / 2 ? ix : ix - n;
  int my = iy < n / 2 ? iy : iy - n;
  int mz = iz;
  double2 g = make_double2(0.0, 0.0);
  if (mx >= -H && mx <= H && my >= -H && my <= H && mz <= H) {
    double re = 0.0, im = 0.0;
    if (mx < H && my < H && mz < H) {
      double2 a = c[((int64_t)(mx + H) * N + (my + H)) * N + (mz + H)];
      re += a.x;
      im += a.y;
    }
    if (mx > -H && my > -H && mz > -H) {
      double2 a = c[((int64_t)(-mx + H) * N + (-my + H)) * N + (-mz + H)];
      re += a.x;
      im -= a.y;
    }
    double f = 0.5 * cor[mx + H] * cor[my + H] * cor[mz + H];
    g = make_double2(re * f, im * f);
  }
  G3[i] = cplx<C2>(g.x, g.y);
  G3[tot + i] = cplx<C2>(0.0, 0.0);
  G3[2 * tot + i] = cplx<C2>(0.0, 0.0);
}

// W_d = (L^3/2) sum_{K_N} |E_{d,k}|^2 = (L^3/2) sum_box omega_k |E_{d,k}|^2, the box
// sum over mz < 0 folded onto mz > 0 (factor 2).  out4 = {W0, W1, W2, Re rho_0}.
// One CTA, fixed summation order (deterministic).
__global__ void __launch_bounds__(1024) k_field_energy(const double2* __restrict__ box, int N,
                                                       double L, const double* __restrict__ S,
                                                       double* __restrict__ out4) {
  const int H = N / 2, NB = N + 1, NZ = H + 1;
  const int64_t tot = (int64_t)NB * NB * NZ;
  double a0 = 0, a1 = 0, a2 = 0;
  const double k0 = 2.0 * M_PI / L;
  for (int64_t i = threadIdx.x; i < tot; i += blockDim.x) {
    int mz = (int)(i % NZ);
    int my = (int)((i / NZ) % NB) - H;
    int mx = (int)(i / ((int64_t)NZ * NB)) - H;
    if ((mx | my | mz) == 0) continue;
    double2 r = box[i];
    double kx = k0 * mx, ky = k0 * my, kz = k0 * mz, k2 = kx * kx + ky * ky + kz * kz;
    double Sk = S[mx + H] * S[my + H] * S[mz + H];
    double e = Sk * Sk * (r.x * r.x + r.y * r.y) / (k2 * k2);
    double w = completion_weight(mx, my, mz, H) * (mz > 0 ? 2.0 : 1.0);
    a0 += w * kx * kx * e;
    a1 += w * ky * ky * e;
    a2 += w * kz * kz * e;
  }
  __shared__ double sh[3][32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a0 += __shfl_xor_sync(0xffffffffu, a0, o);
    a1 += __shfl_xor_sync(0xffffffffu, a1, o);
    a2 += __shfl_xor_sync(0xffffffffu, a2, o);
  }
  if (lane == 0) {
    sh[0][wid] = a0;
    sh[1][wid] = a1;
    sh[2][wid] = a2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s0 = 0, s1 = 0, s2 = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      s0 += sh[0][w];
      s1 += sh[1][w];
      s2 += sh[2][w];
    }
    const double f = 0.5 * L * L * L;
    out4[0] = f * s0;
    out4[1] = f * s1;
    out4[2] = f * s2;
    out4[3] = box[((int64_t)H * NB + H) * NZ].x;
  }
}

// Block partial sums of 4 quantities, then one CTA folds the partials in
// fixed order (deterministic two-pass reduction).
__device__ __forceinline__ void block_sum4(double a[4], double* __restrict__ dst) {
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
  if (threadIdx.x == 0) {
    for (int q = 0; q < 4; ++q) {
      double s = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sh[q][w];
      dst[q] = s;
    }
  }
}

__global__ void __launch_bounds__(256) k_reduce_partials(const double* __restrict__ partials,
                                                         int nparts, double* __restrict__ out4) {
  double a[4] = {0, 0, 0, 0};
  for (int i = threadIdx.x; i < nparts; i += blockDim.x)
#pragma unroll
    for (int q = 0; q < 4; ++q) a[q] += partials[4 * i + q];
  block_sum4(a, out4);
}

// {sum |v|^2, sum vx, sum vy, sum vz}
__global__ void __launch_bounds__(256) k_particle_moments(const double* __restrict__ v,
                                                          int64_t stride, int64_t n,
                                                          double* __restrict__ partials) {
  double a[4] = {0, 0, 0, 0};
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    double v0 = v[j], v1 = v[stride + j], v2 = v[2 * stride + j];
    a[0] += v0 * v0 + v1 * v1 + v2 * v2;
    a[1] += v0;
    a[2] += v1;
    a[3] += v2;
  }
  block_sum4(a, partials + 4 * blockIdx.x);
}

// PIC grid field energy (h^3/2) sum_p |E_p|^2 per component -> partials
__global__ void __launch_bounds__(256) k_grid_energy(const double* __restrict__ g3, int64_t npts,
                                                     double* __restrict__ partials) {
  double a[4] = {0, 0, 0, 0};
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < npts;
       j += (int64_t)gridDim.x * blockDim.x) {
    double e0 = g3[j], e1 = g3[npts + j], e2 = g3[2 * npts + j];
    a[0] += e0 * e0;
    a[1] += e1 * e1;
    a[2] += e2 * e2;
  }
  block_sum4(a, partials + 4 * blockIdx.x);
}

// PIC Poisson (reading R15): E_hat_d = -i k_d rho_hat / |k|^2 * scale,
// zero at k = 0 and on Nyquist planes (m_d = -Ng/2, i.e. index Ng/2).
__global__ void k_pic_poisson(const double2* __restrict__ spec, int Ng, double L, double scale,
                              double2* __restrict__ G3) {
  const int nz = Ng / 2 + 1;
  const int64_t tot = (int64_t)Ng * Ng * nz;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= tot) return;
  int iz = (int)(i % nz);
  int iy = (int)((i / nz) % Ng);
  int ix = (int)(i / ((int64_t)nz * Ng));
  double2 g0 = make_double2(0.0, 0.0), g1 = g0, g2 = g0;
  bool nyq = ix == Ng / 2 || iy == Ng / 2 || iz == Ng / 2;
  if (!nyq && (ix | iy | iz) != 0) {
    int mx = ix < Ng / 2 ? ix : ix - Ng;
    int my = iy < Ng / 2 ? iy : iy - Ng;
    const double k0 = 2.0 * M_PI / L;
    double kx = k0 * mx, ky = k0 * my, kz = k0 * iz;
    double f = scale / (kx * kx + ky * ky + kz * kz);
    double2 r = spec[i];
    g0 = make_double2(f * kx * r.y, -f * kx * r.x);
    g1 = make_double2(f * ky * r.y, -f * ky * r.x);
    g2 = make_double2(f * kz * r.y, -f * kz * r.x);
  }
  G3[i] = g0;
  G3[tot + i] = g1;
  G3[2 * tot + i] = g2;
}

static inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

cudaError_t launch_extract_box(const double2* spec, int n, int N, const double* cor, double scale,
                               double2* box, cudaStream_t st) {
  int64_t tot = (int64_t)(N + 1) * (N + 1) * (N / 2 + 1);
  k_extract_box<<<nblk(tot, 256), 256, 0, st>>>(spec, n, N, cor, scale, box);
  return cudaGetLastError();
}
cudaError_t launch_poisson_pad(const double2* box, int n, int N, double L, const double* cor,
                               const double* S, void* G3, bool fp32, cudaStream_t st) {
  int64_t tot = (int64_t)n * n * (n / 2 + 1);
  if (fp32) k_poisson_pad<<<nblk(tot, 256), 256, 0, st>>>(box, n, N, L, cor, S, (float2*)G3);
  else k_poisson_pad<<<nblk(tot, 256), 256, 0, st>>>(box, n, N, L, cor, S, (double2*)G3);
  return cudaGetLastError();
}
cudaError_t launch_debug_extract_KN(const double2* spec, int n, int N, const double* cor,
                                    double2* out, cudaStream_t st) {
  int64_t tot = (int64_t)N * N * N;
  k_debug_extract_KN<<<nblk(tot, 256), 256, 0, st>>>(spec, n, N, cor, out);
  return cudaGetLastError();
}
cudaError_t launch_debug_pad_KN(const double2* c, int n, int N, const double* cor, void* G3,
                                bool fp32, cudaStream_t st) {
  int64_t tot = (int64_t)n * n * (n / 2 + 1);
  if (fp32) k_debug_pad_KN<<<nblk(tot, 256), 256, 0, st>>>(c, n, N, cor, (float2*)G3);
  else k_debug_pad_KN<<<nblk(tot, 256), 256, 0, st>>>(c, n, N, cor, (double2*)G3);
  return cudaGetLastError();
}
cudaError_t launch_field_energy(const double2* box, int N, double L, const double* S,
                                double* out4, cudaStream_t st) {
  k_field_energy<<<1, 1024, 0, st>>>(box, N, L, S, out4);
  return cudaGetLastError();
}
cudaError_t launch_particle_moments(const double* v, int64_t stride, int64_t n, double* partials,
                                    double* out4, cudaStream_t st) {
  k_particle_moments<<<kReduceBlocks, 256, 0, st>>>(v, stride, n, partials);
  k_reduce_partials<<<1, 256, 0, st>>>(partials, kReduceBlocks, out4);
  return cudaGetLastError();
}
cudaError_t launch_grid_energy(const double* grid3, int64_t npts, double h3, double* partials,
                               double* out4, cudaStream_t st) {
  (void)h3;
  k_grid_energy<<<kReduceBlocks, 256, 0, st>>>(grid3, npts, partials);
  k_reduce_partials<<<1, 256, 0, st>>>(partials, kReduceBlocks, out4);
  return cudaGetLastError();
}
cudaError_t launch_pic_poisson(const double2* spec, int Ng, double L, double scale, double2* G3,
                               cudaStream_t st) {
  int64_t tot = (int64_t)Ng * Ng * (Ng / 2 + 1);
  k_pic_poisson<<<nblk(tot, 256), 256, 0, st>>>(spec, Ng, L, scale, G3);
  return cudaGetLastError();
}

}  // namespace pif
