// Internal declarations of the PIF library (not part of the ABI).
// Citations: P:n = PAPER.md line n; Rn = reading n of DESIGN.md.
#pragma once
#include <cuda_runtime.h>
#include <cufft.h>
#include <stdint.h>

#include <algorithm>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/pif.h"

namespace pif {

// ---------------------------------------------------------------- physics --
struct Phys {
  double L, qm, Q;
  double B[3];
  double A[9];
  double c[3];
};

// Geometry of the tile-owned spreading / interpolation kernels.  The upsampled
// periodic grid n^3 is cut into interpolation sub-bricks of ib[d] cells; m[d]
// sub-bricks per dimension form a spreading brick of sb[d] = m[d] ib[d] cells.
// A CTA owns the tile covering every window of its cells: RI = ib + w - 1
// (interpolation) or RS = sb + w - 1 (spreading) points per dimension.  A
// particle's window is the w grid points [a - hw, a - hw + w) around its anchor
// a (round(x~) for odd w, floor(x~) for even w), hw = (w - 1) / 2, so that
// |g - x~| <= w / 2 on the whole window.  Sort key (brick-major):
// key = (brick * (m0 m1 m2) + sub-brick-in-brick) * C + xy-cell-in-sub-brick.
struct Brick {
  int n;         // upsampled grid points per dimension
  int w;         // kernel width (grid points)
  int hw;        // (w - 1) / 2
  int odd;       // w odd
  int ib[3];     // cells per interpolation sub-brick
  int m[3];      // sub-bricks per spreading brick
  int sb[3];     // cells per spreading brick
  int NB[3];     // spreading bricks per dimension = ceil(n / sb)
  int C;         // sort keys per sub-brick: 1, or ib0 ib1 (its xy-cells; slab interp)
  int RI[3];     // interpolation tile points
  int RS[3];     // spreading tile points
  int64_t nkeys; // number of sub-bricks = NB0 NB1 NB2 m0 m1 m2
  double scale;  // n / L (grid units per length)
  double beta;   // ES shape parameter
  float rsb[3];  // 1 / sb, 1 / ib (binning: floor(a / d) = (int)((a + 1/2) / d) in fp32,
  float rib[3];  //  exact for a < 2^16, d <= 64: the quotient is >= 1/(2d) from an integer)
};

// Piecewise-polynomial ES kernel: for a particle
// with fractional offset f = x~ - a (f in [-1/2, 1/2) for odd w, [0, 1) for even
// w) the window node k (grid point a - hw + k) has weight psi(k - hw - f) =
// P_k(s), s = 2 (f - f_lo) - 1 in [-1, 1], with P_k a degree-kHornerDeg
// Chebyshev interpolant in monomial form (max error ~5e-15 on interior nodes).
// The two edge nodes k = 0, w-1 carry the sqrt singularity of psi at |t| = w/2;
// their fit error is ~0.05 eps (w >= 5), below the NUFFT error budget, so they
// are polynomials too (exact for w <= 4, spread_interp.cu:horner_sym).  Passed by value as a __grid_constant__ kernel
// parameter: every lane of a warp reads the same coefficient (constant cache).
constexpr int kHornerDeg = 14;
struct Horner {
  double a[16][kHornerDeg + 1];  // a[k][j]: coefficient of s^j for node k
};
struct HornerF {  // the same coefficients rounded to fp32 (PIF_FLAG_FP32 interpolation)
  float a[16][kHornerDeg + 1];
};

// Anchor cell of coordinate xs (grid units) with the window rule above; xs is
// shifted by -n / +n when the anchor wraps so that g - xs stays the true offset.
__device__ __forceinline__ int anchor_of(double& xs, const Brick& g) {
  int a = g.odd ? (int)floor(xs + 0.5) : (int)floor(xs);
  if (a >= g.n) {
    a -= g.n;
    xs -= g.n;
  } else if (a < 0) {
    a += g.n;
    xs += g.n;
  }
  return a;
}

// Exponential-of-semicircle kernel psi(t) = exp(beta (sqrt(1 - (2t/w)^2) - 1)),
// |t| <= w/2 (reading R12; FINUFFT's kernel, P:135 via refs).
__device__ __forceinline__ double es_kernel(double t, double two_over_w, double beta) {
  double z = t * two_over_w;
  double r = 1.0 - z * z;
  return r > 0.0 ? exp(beta * (sqrt(r) - 1.0)) : (r == 0.0 ? exp(-beta) : 0.0);
}

// psi[k] = psi_ES(k - hw - f) for the w window nodes, from the per-node
// polynomials in s (spread_interp.cu:horner_sym, here into registers; used by interp_simt.cu and
// the fp32 staging of spread_interp.cu:k_spread_warp): node
// w-1-k at s is node k at -s, so each pair costs one even/odd Horner split.
template <typename T, int W, typename HC>
__device__ __forceinline__ void psi_regs(T (&p)[W], T s, double f, const HC& hc, const Brick& g) {
  constexpr int NPAIR = W / 2;
  constexpr int P0 = W <= 4 ? 1 : 0;  // edge nodes exact for w <= 4 (fit error 0.25 eps)
  const T s2 = s * s;
#pragma unroll
  for (int i = P0; i < NPAIR; ++i) {
    T e = (T)hc.a[i][kHornerDeg], o = (T)hc.a[i][kHornerDeg - 1];
#pragma unroll
    for (int j = kHornerDeg / 2 - 1; j >= 0; --j) {
      e = fma(e, s2, (T)hc.a[i][2 * j]);
      if (j < kHornerDeg / 2 - 1) o = fma(o, s2, (T)hc.a[i][2 * j + 1]);
    }
    p[i] = fma(s, o, e);
    p[W - 1 - i] = fma(-s, o, e);
  }
  if (W & 1) {
    T e = (T)hc.a[W / 2][kHornerDeg];
#pragma unroll
    for (int j = kHornerDeg / 2 - 1; j >= 0; --j) e = fma(e, s2, (T)hc.a[W / 2][2 * j]);
    p[W / 2] = e;
  }
  if (P0) {
    const double tw = 2.0 / W;
    p[0] = (T)es_kernel((double)(-g.hw) - f, tw, g.beta);
    p[W - 1] = (T)es_kernel((double)(W - 1 - g.hw) - f, tw, g.beta);
  }
}

// x - L floor(x / L), L itself mapped to 0.  For 0 <= x < L, x / L rounds to at
// most 1 - 2^-53 (x <= L - ulp(L)), so floor(x / L) = 0 and the result is x:
// the division (a ~10-instruction FP64 sequence) runs only for crossing particles.
__device__ __forceinline__ double wrapL(double x, double L) {
  if (x >= 0.0 && x < L) return x;
  double y = x - L * floor(x / L);
  return y >= L ? 0.0 : y;
}

// Boris half kick of size dt/2 (reading R7): h = dt/4 * q/m.
__device__ __forceinline__ void kick_half(double& vx, double& vy, double& vz, double Ex, double Ey,
                                          double Ez, double h, double tx, double ty, double tz,
                                          double sx, double sy, double sz, bool magnetic) {
  double mx = vx + h * Ex, my = vy + h * Ey, mz = vz + h * Ez;
  if (magnetic) {
    double px = mx + (my * tz - mz * ty);
    double py = my + (mz * tx - mx * tz);
    double pz = mz + (mx * ty - my * tx);
    mx = mx + (py * sz - pz * sy);
    my = my + (pz * sx - px * sz);
    mz = mz + (px * sy - py * sx);
  }
  vx = mx + h * Ex;
  vy = my + h * Ey;
  vz = mz + h * Ez;
}

// Push parameters shared by all push kernels.
struct PushArgs {
  double L, dt, h;          // h = dt/4 * q/m
  double t[3], s[3];        // Boris vectors
  double A[9], c[3];        // E_ext = A x + c
  int magnetic, has_ext;
  int kicks;                // 0, 1 or 2 half kicks
  int drift;                // 1: x <- wrap(x + dt v)
  // Sort fused into the push (pif_api.cu:sort_particles): perm != null -- the
  // particle at sorted position j is x[perm[j]] (the input arrays stay in the
  // previous order), and the pushed x, v and its id go to xo, vo, ido at j (the
  // other buffers).  perm == null: in place at j.
  const int* perm;
  double* xo;
  double* vo;
  int* ido;
};
// Source index of sorted position j.
__device__ __forceinline__ int64_t src_of(const int* perm, int64_t j) { return perm ? (int64_t)perm[j] : j; }

__device__ __forceinline__ void push_particle(double& x0, double& x1, double& x2, double& v0,
                                              double& v1, double& v2, double E0, double E1,
                                              double E2, const PushArgs& P) {
  if (P.has_ext) {
    E0 += P.A[0] * x0 + P.A[1] * x1 + P.A[2] * x2 + P.c[0];
    E1 += P.A[3] * x0 + P.A[4] * x1 + P.A[5] * x2 + P.c[1];
    E2 += P.A[6] * x0 + P.A[7] * x1 + P.A[8] * x2 + P.c[2];
  }
  bool mag = P.magnetic != 0;
  for (int k = 0; k < P.kicks; ++k)
    kick_half(v0, v1, v2, E0, E1, E2, P.h, P.t[0], P.t[1], P.t[2], P.s[0], P.s[1], P.s[2], mag);
  if (P.drift) {
    x0 = wrapL(x0 + P.dt * v0, P.L);
    x1 = wrapL(x1 + P.dt * v1, P.L);
    x2 = wrapL(x2 + P.dt * v2, P.L);
  }
}

// Per-step work schedule of the brick kernels: particle ranges of the sorted
// arrays (offsets over sub-brick keys) cut into work items of at most kSpreadItem
// (spread, per brick) / kInterpItem (interp, per sub-brick) particles, so a
// crowded brick (e.g. the Penning cloud) is shared by several CTAs.  Item =
// {brick, start, end, 0} (spread) / {key, start, end, first m-tile} (interp);
// *_off are exclusive prefix sums over keys
// (spread items attributed to the first key of their brick); totals at [nkeys].
constexpr int kSpreadItem = 4096;
constexpr int kInterpItem = 1024;
struct Sched {
  int* offsets;  // [nkeys + 1]
  int* soff;     // [nkeys + 1]
  int* ioff;     // [nkeys + 1]
  int* moff;     // [nkeys + 1] interpolation cost (m-tiles + brick loads) before each key
  int4* sitems;  // [max_s]
  int4* iitems;  // [max_i]
  int4* iinfo;   // [max_i] decoded interp item: {bx, by, bz, sx | sy << 16}
  int* part;     // [sched_part_ints(nkeys)] scan scratch
  int64_t nkeys, max_s, max_i;
  int* ctr;      // [16] work counters of the dynamically scheduled kernels (zeroed by their launchers)
};
// blocks of the schedule scan (kSchedT bricks each; >= 1)
#ifndef PIF_SCHED_T
#define PIF_SCHED_T 64
#endif
constexpr int kSchedT = PIF_SCHED_T;  // bricks per schedule-scan block (one thread each)
inline unsigned nblk_sched(int64_t nkeys, int64_t M) {
  const int64_t b = (nkeys / M + kSchedT - 1) / kSchedT;
  return (unsigned)(b < 1 ? 1 : b);
}
// ints of scan scratch (Sched::part) for up to nkeys keys
inline size_t sched_part_ints(int64_t nkeys) { return 4 * ((size_t)nkeys / kSchedT + 2); }
inline int64_t sched_max_s(int64_t nkeys, int64_t M, int64_t n) { return nkeys / M + n / kSpreadItem + 1; }
inline int64_t sched_max_i(int64_t nkeys, int64_t n) { return nkeys + n / kInterpItem + 1; }

// Per-device one-time launch setup: cudaFuncSetAttribute applies to the current
// device only and the persistent grids are sized from its SM count, so the
// result is cached per device (thread-safe).
struct DevCache {
  std::mutex mu;
  int val[64] = {};
};
template <typename F>
inline cudaError_t dev_cached(DevCache& dc, int& out, F&& init) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  std::lock_guard<std::mutex> lk(dc.mu);
  if (!dc.val[dev]) {
    int v = 0;
    e = init(dev, v);
    if (e != cudaSuccess) return e;
    if (v < 1) return cudaErrorInvalidConfiguration;
    dc.val[dev] = v;
  }
  out = dc.val[dev];
  return cudaSuccess;
}

// -------------------------------------------------------------- launchers --
// All launchers enqueue on `st` and return cudaGetLastError().
cudaError_t launch_bin_count(const double* x, int64_t stride, int64_t n, const Brick& g, int* key,
                             int* rank, int* counts, cudaStream_t st);
cudaError_t launch_schedule(const int* counts, const Sched& S, const Brick& g, int M, int C,
                            cudaStream_t st);
// keys per spreading brick
inline int keys_per_brick(const Brick& g) { return g.m[0] * g.m[1] * g.m[2] * g.C; }
// Physical counting sort (perm[offsets[key] + rank] = j, then gathers of x, v,
// id and the optional strengths s; v / s may be null).
cudaError_t launch_gather_sorted(const double* x, const double* v, const int* id, const double* s,
                                 int64_t stride, int64_t n, const int* key, const int* rank,
                                 const int* offsets, int* perm, double* x2, double* v2, int* id2,
                                 double* s2, cudaStream_t st);
// perm[offsets[key] + rank] = j only (the fused sort: spread and interp+push read
// through perm, the push writes the sorted copy, PushArgs::perm)
cudaError_t launch_scatter_index(int64_t n, const int* key, const int* rank, const int* offsets,
                                 int* perm, cudaStream_t st);
// hcf != null (fp32 plans): the warp-owned dense-tile spread evaluates the ES
// weights from the fp32 coefficients in single precision (stored as fp64)
cudaError_t launch_spread(const double* x, const int* perm, int64_t stride, const double* s,
                          double s_uniform, const Sched& S, const Brick& g, const Horner& hc,
                          const HornerF* hcf, double* grid, cudaStream_t st);
cudaError_t launch_interp_push(const double* grid3, double* x, double* v, int64_t stride,
                               const int* id, double* Eout, const Sched& S, const Brick& g,
                               const Horner& hc, const PushArgs& P, cudaStream_t st);
// Vector-pipe interpolation + push for small widths (interp_simt.cu): w <= 5
// on the 8^3 / 6x6x8 tiles, w = 6 on 12^3; fp64 or fp32 (PIF_FLAG_FP32).
bool simt_interp_supported(const Brick& g);
// grid3: [3][n^3] double, or float for fp32 plans (single-precision inverse FFT).
cudaError_t launch_interp_push_simt(const void* grid3, double* x, double* v, int64_t stride,
                                    const int* id, double* Eout, const Sched& S, const Brick& g,
                                    const Horner& hc, const HornerF& hcf, bool fp32, const PushArgs& P,
                                    cudaStream_t st);
cudaError_t launch_extract_box(const double2* spec, int n, int N, const double* cor, double scale,
                               double2* box, cudaStream_t st);
// G3: 3 half spectra, double2 or (fp32) float2 for a single-precision inverse FFT.
cudaError_t launch_poisson_pad(const double2* box, int n, int N, double L, const double* cor,
                               const double* S, void* G3, bool fp32, cudaStream_t st);
cudaError_t launch_debug_extract_KN(const double2* spec, int n, int N, const double* cor,
                                    double2* out, cudaStream_t st);
cudaError_t launch_debug_pad_KN(const double2* c, int n, int N, const double* cor, void* G3,
                                bool fp32, cudaStream_t st);
cudaError_t launch_field_energy(const double2* box, int N, double L, const double* S,
                                double* out4, cudaStream_t st);
cudaError_t launch_particle_moments(const double* v, int64_t stride, int64_t n, double* partials,
                                    double* out4, cudaStream_t st);
cudaError_t launch_cic_deposit(const double* x, int64_t stride, int64_t n, int Ng, double inv_h,
                               double* grid, cudaStream_t st);
cudaError_t launch_pic_poisson(const double2* spec, int Ng, double L, double scale, double2* G3,
                               cudaStream_t st);
// grid4: [Ng^3][4] scratch for the interleaved field (one 32-byte sector per node)
cudaError_t launch_cic_gather_push(const double* grid3, double* grid4, double* x, double* v,
                                   int64_t stride, int64_t n, int Ng, double inv_h, const PushArgs& P,
                                   cudaStream_t st);
cudaError_t launch_grid_energy(const double* grid3, int64_t npts, double h3, double* partials,
                               double* out4, cudaStream_t st);
cudaError_t launch_push_only(double* x, double* v, const double* E, int64_t stride, int64_t n,
                             const PushArgs& P, cudaStream_t st);
cudaError_t launch_scatter_by_id(const double* x, const double* v, const int* id, int64_t stride,
                                 int64_t n, double* xo, double* vo, cudaStream_t st);
cudaError_t launch_iota(int* id, int64_t n, cudaStream_t st);
cudaError_t launch_correct_norms(const double* F, const double* Gn, const double* Go, double* U,
                                 int64_t n, double L, double* partials, double* out4,
                                 cudaStream_t st);
cudaError_t launch_convert(double* d, float* f, int64_t count, bool to_float, cudaStream_t st);
// flag <- 1 on any non-finite a[i]; wrap_L > 0 also wraps a[i] into [0, wrap_L).
cudaError_t launch_check_finite(double* a, int64_t count, double wrap_L, int* flag, cudaStream_t st);

constexpr int kReduceBlocks = 592;  // 4 x 148 SMs

// ---------------------------------------- parareal pipeline protocol (host) --
// Buffer ids of one time slice: input U_t, F(U_t), G(U_t^k), G(U_t^{k+1}), U_{t+1}.
enum { PB_U = 0, PB_F = 1, PB_GOLD = 2, PB_GNEW = 3, PB_UNEXT = 4 };
struct ProtocolOps {
  void* user;
  pif_status (*store_initial)(void* user, int dst);               // current state -> dst (t == 0)
  pif_status (*propagate)(void* user, int which, int src, int dst); // 0 = F, 1 = G
  pif_status (*correct)(void* user, int F, int Gn, int Go, int U, double* ex, double* ev);
  pif_status (*send)(void* user, int buf, double flag);            // to t + 1
  pif_status (*recv)(void* user, int buf, double* flag);           // from t - 1
  pif_status (*guard)(void* user);  // later writes must wait for in-flight sends
};
struct ProtocolResult {
  int iterations = 0, retired_at = -1, final_buf = 0;
  std::vector<double> ex, ev;
};
pif_status run_pipeline(int t, int T, int max_iter, double tol, const ProtocolOps& ops,
                        ProtocolResult& res);
}  // namespace pif
