// a7+a8 for small kernel widths (w <= 6: eps >= ~1e-5, the coarse propagator
// of parareal): the type-2 interpolation fused with the
// push on the vector pipes, fp64 or fp32 (PIF_FLAG_FP32, "single precision"
// of P:553-554).
//
// Why not the DMMA kernels here: at w = 5 an 8-particle m-tile contracts over
// only 7 k-steps x 3 DMMAs, so the per-m-tile staging (psi rows in shared
// memory, window reduction, cursor, push on 8 of 32 lanes) dominates and the
// DMMA path reached 0.19 of the FP64 peak.  Here one thread owns
// one particle: psi_x, psi_y, psi_z (w values each) stay in registers, the
// sub-brick tile of the three field components sits in shared memory (one
// CTA per interpolation item), and
//   E_d(x_j) = sum_{ix,iy} psi_x[ix] psi_y[iy] sum_iz psi_z[iz] g_d[ix][iy][iz]
// costs w^3 node loads (fp64: LDS.128 {g_x, g_y} + LDS.64 g_z; fp32: one
// LDS.128 {g_x, g_y, g_z, 0}) and 3 w^3 + 4 w^2 FMAs per particle.  Particles
// are sorted by (sub-brick, xy-cell), so the lanes of a warp mostly read the
// same node at the same time (shared-memory broadcast).
#include <type_traits>

#include "pif_internal.cuh"

namespace pif {

template <typename T>
__device__ __forceinline__ void cp_async_t(T* smem, const T* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  if constexpr (sizeof(T) == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(gmem) : "memory");
}

// grid3: the three field grids [3][n^3] in T (fp32 plans run the inverse FFT
// in single precision, so the grid is already float).  Persistent over items
// (grid-stride), the tile of the next item loading (cp.async) while the current
// one is computed.  Tile node (cx, cy, cz) at cx PX + cy PY + cz: {g_x, g_y} in
// gxy, g_z in gz -- per node and lane 2 + 1 shared-memory wavefronts in fp32,
// 4 + 2 in fp64 (the load width sets the wavefront count; lanes of a warp that
// share a cell read the same node).  PY = RZ + 1, PX = RY PY + 1: with sparse
// particles (lanes in different cells) the node addresses of a warp spread over
// the banks instead of repeating every 128 bytes.
template <typename T, int W, int RX, int RY, int RZ, typename HC>
__global__ void __launch_bounds__(128) k_interp_push_simt(const T* __restrict__ grid3,
                                                          double* __restrict__ x,
                                                          double* __restrict__ v, int64_t stride,
                                                          const int* __restrict__ id,
                                                          double* __restrict__ Eout, const Sched Sc,
                                                          Brick g, const __grid_constant__ HC hc,
                                                          PushArgs P) {
  constexpr int NN = RX * RY * RZ;
  constexpr int PY = RZ + 1, PX = RY * PY + 1, NP = RX * PX;
  using T2 = typename std::conditional<sizeof(T) == 4, float2, double2>::type;
  __shared__ __align__(16) T2 gxy[2][NP];
  __shared__ __align__(16) T gz[2][NP];
  const int total = Sc.ioff[Sc.nkeys];
  const int M = g.m[0] * g.m[1] * g.m[2];
  const int n = g.n;
  const int64_t n3 = (int64_t)n * n * n;
  // item -> particle range and tile origin (keys are (brick, sub-brick, xy-cell) / C)
  auto decode = [&](int item, int& start, int& end, int T0[3]) {
    const int4 e = Sc.iitems[item];
    start = e.y;
    end = e.z;
    const int sub = e.x / g.C, brick = sub / M, sk = sub % M;
    const int bz = brick % g.NB[2], by = (brick / g.NB[2]) % g.NB[1], bx = brick / (g.NB[2] * g.NB[1]);
    const int sz = sk % g.m[2], sy = (sk / g.m[2]) % g.m[1], sx = sk / (g.m[2] * g.m[1]);
    T0[0] = bx * g.sb[0] - g.hw + sx * g.ib[0];
    T0[1] = by * g.sb[1] - g.hw + sy * g.ib[1];
    T0[2] = bz * g.sb[2] - g.hw + sz * g.ib[2];
  };
  auto load_tile = [&](int buf, const int T0[3]) {
    for (int i = threadIdx.x; i < NN; i += blockDim.x) {
      const int cz = i % RZ, cy = (i / RZ) % RY, cx = i / (RZ * RY);
      int gx = T0[0] + cx, gy = T0[1] + cy, gzz = T0[2] + cz;
      gx = gx < 0 ? gx + n : (gx >= n ? gx - n : gx);
      gy = gy < 0 ? gy + n : (gy >= n ? gy - n : gy);
      gzz = gzz < 0 ? gzz + n : (gzz >= n ? gzz - n : gzz);
      const int64_t o = ((int64_t)gx * n + gy) * n + gzz;
      const int t = cx * PX + cy * PY + cz;
      cp_async_t(&gxy[buf][t].x, grid3 + o);
      cp_async_t(&gxy[buf][t].y, grid3 + n3 + o);
      cp_async_t(&gz[buf][t], grid3 + 2 * n3 + o);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  int item = blockIdx.x;
  if (item >= total) return;
  int start, end, T0[3];
  decode(item, start, end, T0);
  load_tile(0, T0);
  const double flo = g.odd ? -0.5 : 0.0;
  for (int buf = 0; item < total; item += gridDim.x, buf ^= 1) {
    int nstart = 0, nend = 0, nT0[3] = {0, 0, 0};
    if (item + (int)gridDim.x < total) {
      decode(item + gridDim.x, nstart, nend, nT0);
      load_tile(buf ^ 1, nT0);  // buffer buf ^ 1 was released by the barrier below
    } else {
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncthreads();
    const T2* txy = gxy[buf];
    const T* tz = gz[buf];
    int j = start + threadIdx.x;
    double xr[3] = {0.0, 0.0, 0.0};
    if (j < end) {
      const int64_t sj = src_of(P.perm, j);
      xr[0] = x[sj], xr[1] = x[stride + sj], xr[2] = x[2 * stride + sj];
    }
    for (; j < end; j += blockDim.x) {
      // positions of this thread's next particle in flight during this one
      const int jn = j + blockDim.x;
      double xn[3] = {0.0, 0.0, 0.0};
      if (jn < end) {
        const int64_t sn = src_of(P.perm, jn);
        xn[0] = x[sn], xn[1] = x[stride + sn], xn[2] = x[2 * stride + sn];
      }
      int rel[3];
      T px[W], py[W], pz[W];
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        double xs = xr[d] * g.scale;
        const int a = anchor_of(xs, g);
        const double f = xs - (double)a;
        rel[d] = a - g.hw - T0[d];
        const T s = (T)(2.0 * (f - flo) - 1.0);
        if (d == 0) psi_regs<T, W>(px, s, f, hc, g);
        else if (d == 1) psi_regs<T, W>(py, s, f, hc, g);
        else psi_regs<T, W>(pz, s, f, hc, g);
      }
      T E0 = 0, E1 = 0, E2 = 0;
      const int base = rel[0] * PX + rel[1] * PY + rel[2];
#pragma unroll
      for (int ix = 0; ix < W; ++ix) {
#pragma unroll
        for (int iy = 0; iy < W; ++iy) {
          const int nb = base + ix * PX + iy * PY;
          T t0 = 0, t1 = 0, t2 = 0;
#pragma unroll
          for (int iz = 0; iz < W; ++iz) {
            const T2 q = txy[nb + iz];
            const T r = tz[nb + iz];
            t0 = fma(pz[iz], q.x, t0);
            t1 = fma(pz[iz], q.y, t1);
            t2 = fma(pz[iz], r, t2);
          }
          const T wxy = px[ix] * py[iy];
          E0 = fma(wxy, t0, E0);
          E1 = fma(wxy, t1, E1);
          E2 = fma(wxy, t2, E2);
        }
      }
      const int64_t sj = src_of(P.perm, j);
      if (Eout) {
        const int64_t k = id[sj];
        Eout[k] = (double)E0;
        Eout[stride + k] = (double)E1;
        Eout[2 * stride + k] = (double)E2;
      }
      if (P.kicks > 0 || P.drift) {
        double v0 = v[sj], v1 = v[stride + sj], v2 = v[2 * stride + sj];
        push_particle(xr[0], xr[1], xr[2], v0, v1, v2, (double)E0, (double)E1, (double)E2, P);
        double* const xo = P.xo ? P.xo : x;
        double* const vo = P.vo ? P.vo : v;
        xo[j] = xr[0];
        xo[stride + j] = xr[1];
        xo[2 * stride + j] = xr[2];
        vo[j] = v0;
        vo[stride + j] = v1;
        vo[2 * stride + j] = v2;
        if (P.ido) P.ido[j] = id[sj];
      }
      xr[0] = xn[0];
      xr[1] = xn[1];
      xr[2] = xn[2];
    }
    __syncthreads();  // tile buf is rewritten by the load two items ahead
    start = nstart;
    end = nend;
    T0[0] = nT0[0];
    T0[1] = nT0[1];
    T0[2] = nT0[2];
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}

template <typename T, int W, int RX, int RY, int RZ, typename HC>
static cudaError_t simt_launch(const T* grid3, double* x, double* v, int64_t stride, const int* id,
                               double* Eout, const Sched& S, const Brick& g, const HC& hc,
                               const PushArgs& P, cudaStream_t st) {
  static DevCache cache;
  int ctas = 0;  // resident CTAs on the device
  cudaError_t e = dev_cached(cache, ctas, [&](int dev, int& val) {
    int sms = 0, per = 0;
    cudaError_t r = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (r == cudaSuccess)
      r = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_interp_push_simt<T, W, RX, RY, RZ, HC>, 128, 0);
    val = sms * per;
    return r;
  });
  if (e != cudaSuccess) return e;
  const int64_t grid = std::min<int64_t>(S.max_i, 2 * (int64_t)ctas);
  if (grid > 0)
    k_interp_push_simt<T, W, RX, RY, RZ, HC><<<(unsigned)grid, 128, 0, st>>>(grid3, x, v, stride, id, Eout, S, g, hc, P);
  return cudaGetLastError();
}

bool simt_interp_supported(const Brick& g) {
  return (g.w <= 5 && ((g.RI[0] == 8 && g.RI[1] == 8 && g.RI[2] == 8) ||
                       (g.w == 5 && g.RI[0] == 6 && g.RI[1] == 6 && g.RI[2] == 8))) ||
         (g.w == 6 && g.RI[0] == 12 && g.RI[1] == 12 && g.RI[2] == 12);
}

template <typename T, typename HC>
static cudaError_t simt_dispatch(const T* grid3, double* x, double* v, int64_t stride, const int* id,
                                 double* Eout, const Sched& S, const Brick& g, const HC& hc,
                                 const PushArgs& P, cudaStream_t st) {
  const bool t888 = g.RI[0] == 8 && g.RI[1] == 8 && g.RI[2] == 8;
  switch (g.w) {
    case 2: if (t888) return simt_launch<T, 2, 8, 8, 8>(grid3, x, v, stride, id, Eout, S, g, hc, P, st); break;
    case 3: if (t888) return simt_launch<T, 3, 8, 8, 8>(grid3, x, v, stride, id, Eout, S, g, hc, P, st); break;
    case 4: if (t888) return simt_launch<T, 4, 8, 8, 8>(grid3, x, v, stride, id, Eout, S, g, hc, P, st); break;
    case 5:
      if (t888) return simt_launch<T, 5, 8, 8, 8>(grid3, x, v, stride, id, Eout, S, g, hc, P, st);
      if (g.RI[0] == 6 && g.RI[1] == 6 && g.RI[2] == 8)
        return simt_launch<T, 5, 6, 6, 8>(grid3, x, v, stride, id, Eout, S, g, hc, P, st);
      break;
    case 6:  // fp32 only (the fp64 12^3 double-buffered tile exceeds 48 KB)
      if constexpr (sizeof(T) == 4)
        if (g.RI[0] == 12 && g.RI[1] == 12 && g.RI[2] == 12)
          return simt_launch<T, 6, 12, 12, 12>(grid3, x, v, stride, id, Eout, S, g, hc, P, st);
      break;
    default: break;
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_interp_push_simt(const void* grid3, double* x, double* v, int64_t stride,
                                    const int* id, double* Eout, const Sched& S, const Brick& g,
                                    const Horner& hc, const HornerF& hcf, bool fp32, const PushArgs& P,
                                    cudaStream_t st) {
  if (fp32) return simt_dispatch<float>((const float*)grid3, x, v, stride, id, Eout, S, g, hcf, P, st);
  return simt_dispatch<double>((const double*)grid3, x, v, stride, id, Eout, S, g, hc, P, st);
}

}  // namespace pif
