// a1 (type-1 spread) and a7+a8 (type-2 interpolation fused with the push) on
// the FP64 tensor cores (DMMA, mma.sync.m8n8k4.f64; 37 TFLOP/s measured on
// B200 -- tcgen05 has no f64 kind).
//
// Tile-owned design: the upsampled grid is cut into
// sub-bricks of ib cells (interpolation CTAs) grouped m at a time into bricks
// (spreading CTAs); particles are counting-sorted brick-major so a brick's
// particles are the concatenation of its sub-bricks'.  A CTA owns the
// RX x RY x RZ tile that covers every w-point window of its cells.  With
// columns c = (cx, cy) (c = cy*RX + cx) and separable ES weights
// psi_x[p][cx] psi_y[p][cy] psi_z[p][z] (reading R12; zero outside the
// particle's window) both transforms are dense contractions over the tile:
//
//   spread:  G[c][z]   += sum_p W[c][p] psi_z[p][z],  W[c][p] = psi_x[p][cx] psi_y[p][cy]
//            (M = columns, N = z, K = particles; the tile lives in the MMA
//            accumulators over all particles of the brick and is flushed once
//            with native fp64 global reductions, REDG.ADD.F64, into the
//            L2-resident grid -- no shared-memory atomics, which are CAS loops
//            for fp64 on sm_100a);
//   interp:  T_d[p][c]  = sum_z psi_z[p][z] g_d[z][c]     (M = particles, N = columns,
//            K = z; the 3 field components of the tile stay in registers as B
//            fragments for the whole sub-brick), then
//            E_d[p] = sum_c W[c][p] T_d[p][c] on the vector pipe, reduced over
//            the 4 lanes of a fragment row and over the warps in shared memory.
//
// Fragment layouts of m8n8k4.f64 (lane l, g = l >> 2, t = l & 3):
//   A (8x4, row): A[g][t];  B (4x8, col): B[t][g];  C (8x8): C[g][2t], C[g][2t+1].
#include "pif_internal.cuh"

namespace pif {

constexpr int kChunk = 64;  // particles staged per shared-memory round (multiple of 8)

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ int wrapi(int i, int n) { return ((i % n) + n) % n; }

// psi row strides (doubles): S == 4 or 12 (mod 16) so that the 4 particle rows
// read by one half-warp fragment load (4 consecutive doubles each) fall in
// disjoint banks.
template <int R>
struct RowStride {
  static constexpr int v = R <= 8 ? 12 : (R <= 16 ? 20 : ((R + 11) / 16) * 16 + 4);
};

template <int RX, int RY, int RZ>
struct Psi {
  double px[kChunk][RowStride<RX>::v];
  double py[kChunk][RowStride<RY>::v];
  double pz[kChunk][RowStride<(RZ + 7) / 8 * 8>::v];  // z rows zero-padded to a multiple of 8
  double xs[kChunk][3];
  int rel[kChunk][3];
  double str[kChunk];
};

// Decode a spread brick (sub == false) or interpolation sub-brick (sub == true)
// from the CTA index into its tile origin T0 (grid points) and particle range.
__device__ __forceinline__ void tile_of(const Brick& g, int cta, bool sub, int T0[3],
                                        const int* __restrict__ offsets, int64_t& start,
                                        int64_t& end) {
  const int M = g.m[0] * g.m[1] * g.m[2];
  int brick = sub ? cta / M : cta;
  int bz = brick % g.NB[2], by = (brick / g.NB[2]) % g.NB[1], bx = brick / (g.NB[2] * g.NB[1]);
  T0[0] = bx * g.sb[0] - g.hw;
  T0[1] = by * g.sb[1] - g.hw;
  T0[2] = bz * g.sb[2] - g.hw;
  if (sub) {
    int s = cta % M;
    int sz = s % g.m[2], sy = (s / g.m[2]) % g.m[1], sx = s / (g.m[2] * g.m[1]);
    T0[0] += sx * g.ib[0];
    T0[1] += sy * g.ib[1];
    T0[2] += sz * g.ib[2];
    start = offsets[cta];
    end = offsets[cta + 1];
  } else {
    start = offsets[brick * M];
    end = offsets[(brick + 1) * M];
  }
}

// Thread tid < cnt: record particle tid's grid coordinate and window offset.
template <int RX, int RY, int RZ>
__device__ __forceinline__ void stage_position(Psi<RX, RY, RZ>& sm, int tid, const double xr[3],
                                               const Brick& g, const int T0[3]) {
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    double xs = xr[d] * g.scale;
    int a = anchor_of(xs, g);
    sm.xs[tid][d] = xs;
    sm.rel[tid][d] = a - g.hw - T0[d];
  }
}

// ES weights of the chunk's particles (positions already staged); particles
// cnt .. pad-1 get zero rows.  One item per (dimension, particle): the w window
// weights by per-node Horner polynomials (edge nodes exactly), zeros elsewhere
// in the tile row.  Starts and ends with __syncthreads().
template <int RX, int RY, int RZ>
__device__ __forceinline__ void stage_psi(Psi<RX, RY, RZ>& sm, int cnt, int pad, const Brick& g,
                                          const int T0[3], const Horner& hc) {
  __syncthreads();
  const double two_over_w = 2.0 / g.w;
  const double flo = g.odd ? -0.5 : 0.0;
  const int w = g.w;
  for (int it = threadIdx.x; it < 3 * pad; it += blockDim.x) {
    const int d = it / pad, p = it - d * pad;
    const int R = d == 0 ? RX : (d == 1 ? RY : (RZ + 7) / 8 * 8);
    double* row = d == 0 ? sm.px[p] : (d == 1 ? sm.py[p] : sm.pz[p]);
    if (p >= cnt) {
      for (int u = 0; u < R; ++u) row[u] = 0.0;
      continue;
    }
    const int rel = sm.rel[p][d];
    const int T0d = d == 0 ? T0[0] : (d == 1 ? T0[1] : T0[2]);
    const double f = sm.xs[p][d] - (double)(rel + g.hw + T0d);  // x~ - anchor
    const double sv = 2.0 * (f - flo) - 1.0;
    for (int u = 0; u < rel; ++u) row[u] = 0.0;
    for (int u = rel + w; u < R; ++u) row[u] = 0.0;
    row[rel] = es_kernel((double)(-g.hw) - f, two_over_w, g.beta);
    row[rel + w - 1] = es_kernel((double)(w - 1 - g.hw) - f, two_over_w, g.beta);
    // interior nodes 1 .. w-2, four independent Horner chains at a time
    for (int k0 = 1; k0 < w - 1; k0 += 4) {
      double acc[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] = hc.a[min(k0 + q, 15)][kHornerDeg];
#pragma unroll
      for (int j = kHornerDeg - 1; j >= 0; --j)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[q] = fma(acc[q], sv, hc.a[min(k0 + q, 15)][j]);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (k0 + q < w - 1) row[rel + k0 + q] = acc[q];
    }
  }
  __syncthreads();
}

// ------------------------------------------------------------------ spread --
template <int RX, int RY, int RZ>
struct SpreadCfg {
  static constexpr int NCT = RX * RY / 8;         // column tiles (of 8)
  static constexpr int CT = NCT % 4 == 0 ? 4 : 3; // column tiles per warp
  static constexpr int NW = NCT / CT;             // warps
  static constexpr int ZT = (RZ + 7) / 8;         // z tiles of 8 (psi_z rows zero-padded)
  static_assert(RX * RY % 8 == 0 && NCT % CT == 0, "tile shape");
};

template <int RX, int RY, int RZ, bool HAS_S>
__global__ void __launch_bounds__(32 * SpreadCfg<RX, RY, RZ>::NW)
    k_spread(const double* __restrict__ x, int64_t stride, const double* __restrict__ s,
             double s_uniform, const int* __restrict__ offsets, Brick g,
             const __grid_constant__ Horner hc, double* __restrict__ grid) {
  using C = SpreadCfg<RX, RY, RZ>;
  __shared__ Psi<RX, RY, RZ> sm;
  int T0[3];
  int64_t start, end;
  tile_of(g, blockIdx.x, false, T0, offsets, start, end);
  if (start == end) return;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int gr = lane >> 2, tq = lane & 3;
  // A-fragment rows: column c = (wid*CT + ct)*8 + gr
  int acx[C::CT], acy[C::CT];
#pragma unroll
  for (int ct = 0; ct < C::CT; ++ct) {
    int c = (wid * C::CT + ct) * 8 + gr;
    acx[ct] = c % RX;
    acy[ct] = c / RX;
  }
  double acc[C::CT][C::ZT][2];
#pragma unroll
  for (int ct = 0; ct < C::CT; ++ct)
#pragma unroll
    for (int zt = 0; zt < C::ZT; ++zt) acc[ct][zt][0] = acc[ct][zt][1] = 0.0;

  for (int64_t base = start; base < end; base += kChunk) {
    const int cnt = (int)min((int64_t)kChunk, end - base);
    const int pad = (cnt + 3) & ~3;
    if (tid < cnt) {
      double xr[3] = {x[base + tid], x[stride + base + tid], x[2 * stride + base + tid]};
      stage_position(sm, tid, xr, g, T0);
      if (HAS_S) sm.str[tid] = s[base + tid];
    }
    stage_psi(sm, cnt, pad, g, T0, hc);
    for (int p0 = 0; p0 < pad; p0 += 4) {
      const int pl = p0 + tq;  // K index of this lane's A and B elements
      double b[C::ZT];
#pragma unroll
      for (int zt = 0; zt < C::ZT; ++zt) b[zt] = sm.pz[pl][zt * 8 + gr];
      double sp = 1.0;
      if (HAS_S) sp = pl < cnt ? sm.str[pl] : 0.0;
#pragma unroll
      for (int ct = 0; ct < C::CT; ++ct) {
        double a = sm.px[pl][acx[ct]] * sm.py[pl][acy[ct]];
        if (HAS_S) a *= sp;
#pragma unroll
        for (int zt = 0; zt < C::ZT; ++zt) dmma(acc[ct][zt], a, b[zt]);
      }
    }
    __syncthreads();
  }
  // flush: C[g][2t+i] = G[column (wid*CT+ct)*8 + gr][z = zt*8 + 2t + i]
  const int n = g.n;
#pragma unroll
  for (int ct = 0; ct < C::CT; ++ct) {
    double* colp = grid + ((int64_t)wrapi(T0[0] + acx[ct], n) * n + wrapi(T0[1] + acy[ct], n)) * n;
#pragma unroll
    for (int zt = 0; zt < C::ZT; ++zt)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const double val = acc[ct][zt][i];
        const int z = zt * 8 + 2 * tq + i;
        if (z < RZ && val != 0.0) atomicAdd(colp + wrapi(T0[2] + z, n), val * s_uniform);
      }
  }
}

// ------------------------------------------------------------ interp+push --
template <int RX, int RY, int RZ>
struct InterpCfg {
  static constexpr int NCT = RX * RY / 8;         // column tiles (of 8)
  static constexpr int CT = NCT % 4 == 0 ? 4 : 3; // column tiles per warp
  static constexpr int NW = NCT / CT;             // warps
  static constexpr int KS = RZ / 4;               // k steps (z) per MMA chain
  static_assert(RX * RY % 8 == 0 && NCT % CT == 0 && RZ % 4 == 0, "tile shape");
};

template <int RX, int RY, int RZ>
struct InterpSmem {
  Psi<RX, RY, RZ> psi;
  double red[kChunk][InterpCfg<RX, RY, RZ>::NW][3];
};

template <int RX, int RY, int RZ>
__global__ void __launch_bounds__(32 * InterpCfg<RX, RY, RZ>::NW)
    k_interp_push(const double* __restrict__ grid3, double* __restrict__ x,
                  double* __restrict__ v, int64_t stride, const int* __restrict__ id,
                  double* __restrict__ Eout, const int* __restrict__ offsets, Brick g,
                  const __grid_constant__ Horner hc, PushArgs P) {
  using C = InterpCfg<RX, RY, RZ>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  InterpSmem<RX, RY, RZ>& S = *reinterpret_cast<InterpSmem<RX, RY, RZ>*>(smem_raw);
  Psi<RX, RY, RZ>& sm = S.psi;
  int T0[3];
  int64_t start, end;
  tile_of(g, blockIdx.x, true, T0, offsets, start, end);
  if (start == end) return;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int gr = lane >> 2, tq = lane & 3;
  const int n = g.n;
  const int64_t n3 = (int64_t)n * n * n;
  // B fragments: B[k = tq][col = gr] = g_d[z = ks*4 + tq][c = (wid*CT+ct)*8 + gr]
  double gb[C::CT][C::KS][3];
#pragma unroll
  for (int ct = 0; ct < C::CT; ++ct) {
    int c = (wid * C::CT + ct) * 8 + gr;
    const int64_t cb = ((int64_t)wrapi(T0[0] + c % RX, n) * n + wrapi(T0[1] + c / RX, n)) * n;
#pragma unroll
    for (int ks = 0; ks < C::KS; ++ks) {
      int gz = wrapi(T0[2] + ks * 4 + tq, n);
      gb[ct][ks][0] = grid3[cb + gz];
      gb[ct][ks][1] = grid3[n3 + cb + gz];
      gb[ct][ks][2] = grid3[2 * n3 + cb + gz];
    }
  }
  // C-fragment columns of this lane: c = (wid*CT+ct)*8 + 2*tq + i
  int ccx[C::CT][2], ccy[C::CT][2];
#pragma unroll
  for (int ct = 0; ct < C::CT; ++ct)
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      int c = (wid * C::CT + ct) * 8 + 2 * tq + i;
      ccx[ct][i] = c % RX;
      ccy[ct][i] = c / RX;
    }

  // x, v of the next chunk are prefetched into registers during the MMA phase
  double xn[3] = {0, 0, 0}, vn[3] = {0, 0, 0};
  auto fetch = [&](int64_t b, int c) {
    if (tid < c) {
      const int64_t j = b + tid;
      xn[0] = x[j];
      xn[1] = x[stride + j];
      xn[2] = x[2 * stride + j];
      if (v) {
        vn[0] = v[j];
        vn[1] = v[stride + j];
        vn[2] = v[2 * stride + j];
      }
    }
  };
  fetch(start, (int)min((int64_t)kChunk, end - start));
  for (int64_t base = start; base < end; base += kChunk) {
    const int cnt = (int)min((int64_t)kChunk, end - base);
    const int pad = (cnt + 7) & ~7;
    double xr[3] = {xn[0], xn[1], xn[2]}, vr[3] = {vn[0], vn[1], vn[2]};
    if (tid < cnt) stage_position(sm, tid, xr, g, T0);
    stage_psi(sm, cnt, pad, g, T0, hc);
    if (base + kChunk < end) fetch(base + kChunk, (int)min((int64_t)kChunk, end - base - kChunk));
    // Software-pipelined over m-tiles of 8 particles: the DMMAs of tile i+1 are
    // issued before the vector-pipe stage 2 of tile i consumes its accumulators.
    auto mma_tile = [&](int p0, double (&acc)[C::CT][3][2]) {
#pragma unroll
      for (int ct = 0; ct < C::CT; ++ct)
#pragma unroll
        for (int d = 0; d < 3; ++d) acc[ct][d][0] = acc[ct][d][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < C::KS; ++ks) {
        const double a = sm.pz[p0 + gr][ks * 4 + tq];  // A[g][t] = psi_z[p0+g][z]
#pragma unroll
        for (int ct = 0; ct < C::CT; ++ct)
#pragma unroll
          for (int d = 0; d < 3; ++d) dmma(acc[ct][d], a, gb[ct][ks][d]);
      }
    };
    auto stage2 = [&](int p0, const double (&acc)[C::CT][3][2]) {
      const int p = p0 + gr;
      double e0 = 0.0, e1 = 0.0, e2 = 0.0;
#pragma unroll
      for (int ct = 0; ct < C::CT; ++ct)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const double W = sm.px[p][ccx[ct][i]] * sm.py[p][ccy[ct][i]];
          e0 = fma(W, acc[ct][0][i], e0);
          e1 = fma(W, acc[ct][1][i], e1);
          e2 = fma(W, acc[ct][2][i], e2);
        }
#pragma unroll
      for (int o = 1; o <= 2; o <<= 1) {
        e0 += __shfl_xor_sync(0xffffffffu, e0, o);
        e1 += __shfl_xor_sync(0xffffffffu, e1, o);
        e2 += __shfl_xor_sync(0xffffffffu, e2, o);
      }
      if (tq == 0) {
        S.red[p][wid][0] = e0;
        S.red[p][wid][1] = e1;
        S.red[p][wid][2] = e2;
      }
    };
    {
      double accA[C::CT][3][2], accB[C::CT][3][2];
      mma_tile(0, accA);
      int p0 = 0;
      for (; p0 + 16 <= pad; p0 += 16) {
        mma_tile(p0 + 8, accB);
        stage2(p0, accA);
        if (p0 + 16 < pad) mma_tile(p0 + 16, accA);
        stage2(p0 + 8, accB);
      }
      if (p0 < pad) stage2(p0, accA);  // pad % 16 == 8: last tile pending in accA
    }
    __syncthreads();
    if (tid < cnt) {
      double E0 = 0.0, E1 = 0.0, E2 = 0.0;
#pragma unroll
      for (int w = 0; w < C::NW; ++w) {
        E0 += S.red[tid][w][0];
        E1 += S.red[tid][w][1];
        E2 += S.red[tid][w][2];
      }
      const int64_t j = base + tid;
      if (Eout) {
        const int64_t k = id[j];
        Eout[k] = E0;
        Eout[stride + k] = E1;
        Eout[2 * stride + k] = E2;
      }
      if (P.kicks > 0 || P.drift) {
        push_particle(xr[0], xr[1], xr[2], vr[0], vr[1], vr[2], E0, E1, E2, P);
        x[j] = xr[0];
        x[stride + j] = xr[1];
        x[2 * stride + j] = xr[2];
        v[j] = vr[0];
        v[stride + j] = vr[1];
        v[2 * stride + j] = vr[2];
      }
    }
    __syncthreads();
  }
}

cudaError_t launch_spread(const double* x, int64_t stride, const double* s, double s_uniform,
                          const int* offsets, const Brick& g, const Horner& hc, double* grid,
                          cudaStream_t st) {
  const unsigned nbr = (unsigned)((int64_t)g.NB[0] * g.NB[1] * g.NB[2]);
#define PIF_SPREAD(A, B, Cz)                                                                  \
  if (g.RS[0] == A && g.RS[1] == B && g.RS[2] == Cz) {                                        \
    const int T = 32 * SpreadCfg<A, B, Cz>::NW;                                               \
    if (s)                                                                                    \
      k_spread<A, B, Cz, true><<<nbr, T, 0, st>>>(x, stride, s, s_uniform, offsets, g, hc, grid); \
    else                                                                                      \
      k_spread<A, B, Cz, false><<<nbr, T, 0, st>>>(x, stride, s, s_uniform, offsets, g, hc, grid); \
    return cudaGetLastError();                                                                \
  }
  PIF_SPREAD(8, 8, 8)
  PIF_SPREAD(12, 12, 12)
  PIF_SPREAD(16, 16, 16)
#undef PIF_SPREAD
  return cudaErrorInvalidValue;
}

template <int A, int B, int Cz>
static cudaError_t interp_launch(unsigned nsub, const double* grid3, double* x, double* v,
                                 int64_t stride, const int* id, double* Eout, const int* offsets,
                                 const Brick& g, const Horner& hc, const PushArgs& P,
                                 cudaStream_t st) {
  const int T = 32 * InterpCfg<A, B, Cz>::NW;
  const size_t smem = sizeof(InterpSmem<A, B, Cz>);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_interp_push<A, B, Cz>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  k_interp_push<A, B, Cz><<<nsub, T, smem, st>>>(grid3, x, v, stride, id, Eout, offsets, g, hc, P);
  return cudaGetLastError();
}

cudaError_t launch_interp_push(const double* grid3, double* x, double* v, int64_t stride,
                               const int* id, double* Eout, const int* offsets, const Brick& g,
                               const Horner& hc, const PushArgs& P, cudaStream_t st) {
  const unsigned nsub = (unsigned)g.nkeys;
#define PIF_INTERP(A, B, Cz)                                                                   \
  if (g.RI[0] == A && g.RI[1] == B && g.RI[2] == Cz)                                           \
    return interp_launch<A, B, Cz>(nsub, grid3, x, v, stride, id, Eout, offsets, g, hc, P, st);
  PIF_INTERP(8, 8, 8)
  PIF_INTERP(12, 12, 12)
  PIF_INTERP(16, 14, 16)
  PIF_INTERP(16, 16, 16)
#undef PIF_INTERP
  return cudaErrorInvalidValue;
}

}  // namespace pif
