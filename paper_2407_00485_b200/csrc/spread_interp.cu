// a1 (type-1 spread) and a7+a8 (type-2 interpolation fused with the push).
//
// Tile-owned design: one CTA per brick of b^3 cells;
// thread (tx, ty) owns the z-column (T0x+tx, T0y+ty, T0z .. T0z+R-1) of the
// brick's R^3 tile.  Spreading accumulates each column in R registers over all
// particles of the brick (no shared-memory atomics -- fp64 smem atomicAdd is a
// CAS loop on sm_100a) and flushes the tile once with native fp64 global
// reductions (REDG.ADD.F64 resolved in L2).  Interpolation holds the three
// field components of the column in registers and reduces the per-column
// partial sums of each particle across the CTA.
//
// Separable ES weights (reading R12): psi_d[t] = psi(T0_d + t - x~_d) inside
// the particle's w-point window, 0 outside, computed once per particle and
// staged in shared memory.
#include "pif_internal.cuh"

namespace pif {

constexpr int kChunk = 64;  // particles staged per shared-memory round

template <int R>
struct TileSmem {
  double psi[kChunk][3][R];
  double xs[kChunk][3];
  int rel[kChunk][3];
  double str[kChunk];
};

template <int R>
__device__ __forceinline__ void brick_origin(const Brick& g, int brick, int T0[3]) {
  int bz = brick % g.nb, by = (brick / g.nb) % g.nb, bx = brick / (g.nb * g.nb);
  T0[0] = bx * g.b - g.hw;
  T0[1] = by * g.b - g.hw;
  T0[2] = bz * g.b - g.hw;
}

// Stage positions and ES weights of particles [base, base+cnt) of the sorted
// arrays into shared memory.  Ends with __syncthreads().
template <int R, bool HAS_S>
__device__ __forceinline__ void stage_chunk(TileSmem<R>& sm, const double* __restrict__ x,
                                            int64_t stride, const double* __restrict__ s,
                                            int64_t base, int cnt, const Brick& g,
                                            const int T0[3]) {
  const int tid = threadIdx.x;
  if (tid < cnt) {
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      double xs = x[d * stride + base + tid] * g.scale;
      int a = anchor_of(xs, g);
      sm.xs[tid][d] = xs;
      sm.rel[tid][d] = a - g.hw - T0[d];
    }
    if (HAS_S) sm.str[tid] = s[base + tid];
  }
  __syncthreads();
  const double two_over_w = 2.0 / g.w;
  for (int it = tid; it < cnt * 3 * R; it += blockDim.x) {
    int p = it / (3 * R);
    int rem = it - p * 3 * R;
    int d = rem / R;
    int t = rem - d * R;
    int r = t - sm.rel[p][d];
    double val = 0.0;
    if (r >= 0 && r < g.w) val = es_kernel((double)(T0[d] + t) - sm.xs[p][d], two_over_w, g.beta);
    sm.psi[p][d][t] = val;
  }
  __syncthreads();
}

template <int R, bool HAS_S>
__global__ void __launch_bounds__(((R * R + 31) / 32) * 32)
    k_spread(const double* __restrict__ x, int64_t stride, const double* __restrict__ s,
             double s_uniform, const int* __restrict__ offsets, Brick g, double* __restrict__ grid) {
  __shared__ TileSmem<R> sm;
  const int brick = blockIdx.x;
  const int64_t start = offsets[brick], end = offsets[brick + 1];
  if (start == end) return;
  int T0[3];
  brick_origin<R>(g, brick, T0);
  const int tid = threadIdx.x;
  const bool col = tid < R * R;
  const int tx = col ? tid % R : 0, ty = col ? tid / R : 0;
  double acc[R];
#pragma unroll
  for (int z = 0; z < R; ++z) acc[z] = 0.0;

  for (int64_t base = start; base < end; base += kChunk) {
    const int cnt = (int)min((int64_t)kChunk, end - base);
    stage_chunk<R, HAS_S>(sm, x, stride, s, base, cnt, g, T0);
    if (col) {
      for (int p = 0; p < cnt; ++p) {
        double c = sm.psi[p][0][tx] * sm.psi[p][1][ty];
        if (HAS_S) c *= sm.str[p];
#pragma unroll
        for (int z = 0; z < R; ++z) acc[z] = fma(c, sm.psi[p][2][z], acc[z]);
      }
    }
    __syncthreads();
  }
  if (!col) return;
  const int n = g.n;
  const int gx = ((T0[0] + tx) % n + n) % n;
  const int gy = ((T0[1] + ty) % n + n) % n;
  double* colp = grid + ((int64_t)gx * n + gy) * n;
#pragma unroll
  for (int z = 0; z < R; ++z) {
    if (acc[z] != 0.0) {
      int gz = ((T0[2] + z) % n + n) % n;
      atomicAdd(colp + gz, acc[z] * s_uniform);
    }
  }
}

template <int R>
__global__ void __launch_bounds__(((R * R + 31) / 32) * 32, 1)
    k_interp_push(const double* __restrict__ grid3, double* __restrict__ x,
                  double* __restrict__ v, int64_t stride, const int* __restrict__ id,
                  double* __restrict__ Eout, const int* __restrict__ offsets, Brick g, PushArgs P) {
  constexpr int NW = ((R * R + 31) / 32);
  __shared__ TileSmem<R> sm;
  __shared__ double red[kChunk][NW][3];
  const int brick = blockIdx.x;
  const int64_t start = offsets[brick], end = offsets[brick + 1];
  if (start == end) return;
  int T0[3];
  brick_origin<R>(g, brick, T0);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const bool col = tid < R * R;
  const int tx = col ? tid % R : 0, ty = col ? tid / R : 0;
  const int n = g.n;
  const int64_t n3 = (int64_t)n * n * n;
  double g0[R], g1[R], g2[R];
  {
    const int gx = ((T0[0] + tx) % n + n) % n;
    const int gy = ((T0[1] + ty) % n + n) % n;
    const int64_t cb = ((int64_t)gx * n + gy) * n;
#pragma unroll
    for (int z = 0; z < R; ++z) {
      int gz = ((T0[2] + z) % n + n) % n;
      g0[z] = col ? grid3[cb + gz] : 0.0;
      g1[z] = col ? grid3[n3 + cb + gz] : 0.0;
      g2[z] = col ? grid3[2 * n3 + cb + gz] : 0.0;
    }
  }
  for (int64_t base = start; base < end; base += kChunk) {
    const int cnt = (int)min((int64_t)kChunk, end - base);
    stage_chunk<R, false>(sm, x, stride, nullptr, base, cnt, g, T0);
    for (int p = 0; p < cnt; ++p) {
      double c = sm.psi[p][0][tx] * sm.psi[p][1][ty];
      double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
      for (int z = 0; z < R; ++z) {
        double pz = sm.psi[p][2][z];
        s0 = fma(pz, g0[z], s0);
        s1 = fma(pz, g1[z], s1);
        s2 = fma(pz, g2[z], s2);
      }
      s0 *= c;
      s1 *= c;
      s2 *= c;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        s0 += __shfl_xor_sync(0xffffffffu, s0, o);
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
      }
      if (lane == 0) {
        red[p][wid][0] = s0;
        red[p][wid][1] = s1;
        red[p][wid][2] = s2;
      }
    }
    __syncthreads();
    if (tid < cnt) {
      double E0 = 0.0, E1 = 0.0, E2 = 0.0;
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        E0 += red[tid][w][0];
        E1 += red[tid][w][1];
        E2 += red[tid][w][2];
      }
      const int64_t j = base + tid;
      if (Eout) {
        const int64_t k = id[j];
        Eout[k] = E0;
        Eout[stride + k] = E1;
        Eout[2 * stride + k] = E2;
      }
      if (P.kicks > 0 || P.drift) {
        double x0 = x[j], x1 = x[stride + j], x2 = x[2 * stride + j];
        double v0 = v[j], v1 = v[stride + j], v2 = v[2 * stride + j];
        push_particle(x0, x1, x2, v0, v1, v2, E0, E1, E2, P);
        x[j] = x0;
        x[stride + j] = x1;
        x[2 * stride + j] = x2;
        v[j] = v0;
        v[stride + j] = v1;
        v[2 * stride + j] = v2;
      }
    }
    __syncthreads();
  }
}

static int tile_threads(int R) { return ((R * R + 31) / 32) * 32; }

cudaError_t launch_spread(const double* x, int64_t stride, const double* s, double s_uniform,
                          const int* offsets, const Brick& g, double* grid, cudaStream_t st) {
  const unsigned nbr = (unsigned)((int64_t)g.nb * g.nb * g.nb);
  const int T = tile_threads(g.R);
#define PIF_SPREAD(RR)                                                                        \
  if (s)                                                                                      \
    k_spread<RR, true><<<nbr, T, 0, st>>>(x, stride, s, s_uniform, offsets, g, grid);         \
  else                                                                                        \
    k_spread<RR, false><<<nbr, T, 0, st>>>(x, stride, s, s_uniform, offsets, g, grid);
  switch (g.R) {
    case 8: PIF_SPREAD(8) break;
    case 12: PIF_SPREAD(12) break;
    case 16: PIF_SPREAD(16) break;
    default: return cudaErrorInvalidValue;
  }
#undef PIF_SPREAD
  return cudaGetLastError();
}

cudaError_t launch_interp_push(const double* grid3, double* x, double* v, int64_t stride,
                               const int* id, double* Eout, const int* offsets, const Brick& g,
                               const PushArgs& P, cudaStream_t st) {
  const unsigned nbr = (unsigned)((int64_t)g.nb * g.nb * g.nb);
  const int T = tile_threads(g.R);
  switch (g.R) {
    case 8: k_interp_push<8><<<nbr, T, 0, st>>>(grid3, x, v, stride, id, Eout, offsets, g, P); break;
    case 12: k_interp_push<12><<<nbr, T, 0, st>>>(grid3, x, v, stride, id, Eout, offsets, g, P); break;
    case 16: k_interp_push<16><<<nbr, T, 0, st>>>(grid3, x, v, stride, id, Eout, offsets, g, P); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace pif
