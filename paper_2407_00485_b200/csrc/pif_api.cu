// C ABI of the PIF library (include/pif.h): context, NUFFT plans, workspace,
// the step loop (a0..a8 of SURVEY.md Sec. 8a), diagnostics, parareal driver
// (fine/coarse propagation, correction, NCCL hand-off) and test-only exports.
#include <math.h>
#include <nccl.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <functional>
#include <cmath>
#include <string>
#include <thread>
#include <type_traits>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "pif_internal.cuh"

using namespace pif;

namespace {

thread_local std::string g_err;

pif_status fail(pif_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

#define CU(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(PIF_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));      \
  } while (0)
#define CUFFT(call)                                                                       \
  do {                                                                                    \
    cufftResult r_ = (call);                                                              \
    if (r_ != CUFFT_SUCCESS)                                                              \
      return fail(PIF_ERR_CUDA, std::string(#call) + ": cufft error " + std::to_string((int)r_)); \
  } while (0)
#define NC(call)                                                                          \
  do {                                                                                    \
    ncclResult_t r_ = (call);                                                             \
    if (r_ != ncclSuccess)                                                                \
      return fail(PIF_ERR_NCCL, std::string(#call) + ": " + ncclGetErrorString(r_));      \
  } while (0)
#define TRY(call)                 \
  do {                            \
    pif_status s_ = (call);       \
    if (s_ != PIF_OK) return s_;  \
  } while (0)

// Every entry point that touches device state runs on the context's device and
// restores the caller's current device on return.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) == cudaSuccess && prev != dev) cudaSetDevice(dev);
    else prev = -1;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// Temporary device buffers outside the workspace (debug exports, parareal
// states): stream-ordered allocations freed on every exit path.
struct DevBufs {
  cudaStream_t st;
  std::vector<void*> v;
  explicit DevBufs(cudaStream_t s) : st(s) {}
  template <typename T>
  cudaError_t alloc(T** p, size_t bytes) {
    void* q = nullptr;
    cudaError_t e = cudaMallocAsync(&q, bytes, st);
    if (e != cudaSuccess) return e;
    v.push_back(q);
    *p = static_cast<T*>(q);
    return cudaSuccess;
  }
  ~DevBufs() {
    for (void* q : v) cudaFreeAsync(q, st);
    if (!v.empty()) cudaStreamSynchronize(st);
  }
};

// ---------------------------------------------------------------------------
// NUFFT parameters (reading R12): w = ceil(-log10(eps/10)), beta = c(w) w, n =
// smallest power of two >= max(2N, 2w); ES kernel and its Fourier transform
// psi^(xi) = int psi(t) cos(xi t) dt by Gauss-Legendre quadrature.
// ---------------------------------------------------------------------------
int es_width(double tol) {
  int w = (int)std::ceil(-std::log10(tol / 10.0) - 1e-9);
  return std::min(16, std::max(2, w));
}
double es_beta(int w) {
  double c = w == 2 ? 2.20 : w == 3 ? 2.26 : w == 4 ? 2.38 : 2.30;
  return c * w;
}
double es_host(double t, double w, double beta) {
  double z = 2.0 * t / w;
  double r = 1.0 - z * z;
  return r >= 0.0 ? std::exp(beta * (std::sqrt(r) - 1.0)) : 0.0;
}
void gauss_legendre(int q, std::vector<double>& x, std::vector<double>& wt) {
  x.resize(q);
  wt.resize(q);
  for (int i = 0; i < q; ++i) {
    double z = std::cos(M_PI * (i + 0.75) / (q + 0.5)), dp = 1.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = z;
      for (int k = 2; k <= q; ++k) {
        double p2 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      dp = q * (z * p1 - p0) / (z * z - 1.0);
      double dz = p1 / dp;
      z -= dz;
      if (std::fabs(dz) < 1e-16) break;
    }
    {
      double p0 = 1.0, p1 = z;
      for (int k = 2; k <= q; ++k) {
        double p2 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      dp = q * (z * p1 - p0) / (z * z - 1.0);
    }
    x[i] = z;
    wt[i] = 2.0 / ((1.0 - z * z) * dp * dp);
  }
}
double es_hat(double xi, int w, double beta) {
  static thread_local std::vector<double> gx, gw;
  if (gx.empty()) gauss_legendre(200, gx, gw);
  double half = 0.5 * w, s = 0.0;
  for (size_t i = 0; i < gx.size(); ++i) {
    double t = 0.5 * half * (gx[i] + 1.0);  // [0, w/2]
    s += gw[i] * es_host(t, w, beta) * std::cos(xi * t);
  }
  return 2.0 * 0.5 * half * s;  // even integrand: 2 * int_0^{w/2}
}

enum { PH_SORT = 0, PH_SPREAD, PH_FFT_FWD, PH_BOX, PH_ALLREDUCE, PH_POISSON, PH_FFT_INV,
       PH_INTERP_PUSH, PH_PIC_DEPOSIT, PH_PIC_GATHER_PUSH, PH_OTHER, PH_COUNT };
static_assert(PH_COUNT == PIF_NPHASES, "phase count");

// Chebyshev interpolation of psi(k - hw - f) on f in [f_lo, f_lo + 1) at
// kHornerDeg + 1 Chebyshev nodes of s = 2 (f - f_lo) - 1, converted to monomial
// coefficients in s (three-term recurrence of T_j).
void horner_fit(int w, double beta, Horner& hc) {
  const int D = kHornerDeg, hw = (w - 1) / 2;
  const double flo = (w & 1) ? -0.5 : 0.0;
  memset(&hc, 0, sizeof(hc));
  std::vector<double> sn(D + 1), cheb(D + 1);
  for (int i = 0; i <= D; ++i) sn[i] = std::cos(M_PI * (i + 0.5) / (D + 1));
  for (int k = 0; k < w; ++k) {
    std::vector<double> val(D + 1);
    for (int i = 0; i <= D; ++i) {
      double f = flo + 0.5 * (sn[i] + 1.0);
      val[i] = es_host(k - hw - f, w, beta);
    }
    for (int j = 0; j <= D; ++j) {
      double acc = 0;
      for (int i = 0; i <= D; ++i) acc += val[i] * std::cos(M_PI * j * (i + 0.5) / (D + 1));
      cheb[j] = acc * (j == 0 ? 1.0 : 2.0) / (D + 1);
    }
    // monomial coefficients: sum_j cheb[j] T_j(s)
    std::vector<double> Tm1(D + 1, 0.0), T0(D + 1, 0.0), T1(D + 1, 0.0), mono(D + 1, 0.0);
    T0[0] = 1.0;  // T_0
    for (int j = 0; j <= D; ++j) {
      const std::vector<double>& Tj = (j == 0) ? T0 : T1;
      for (int q = 0; q <= D; ++q) mono[q] += cheb[j] * Tj[q];
      // advance: T_{j+1} = 2 s T_j - T_{j-1}
      std::vector<double> nxt(D + 1, 0.0);
      if (j == 0) {
        nxt[1] = 1.0;  // T_1 = s
        Tm1 = T0;
      } else {
        for (int q = 0; q < D; ++q) nxt[q + 1] += 2.0 * T1[q];
        for (int q = 0; q <= D; ++q) nxt[q] -= Tm1[q];
        Tm1 = T1;
      }
      T1 = nxt;
    }
    for (int q = 0; q <= D; ++q) hc.a[k][q] = mono[q];
  }
}

struct Plan {
  bool valid = false;
  bool fp32_ar = false;  // PIF_FLAG_FP32_ALLREDUCE
  bool fp32 = false;     // PIF_FLAG_FP32: fp32 interpolation
  bool simt = false;     // interpolation on the vector pipes (interp_simt.cu)
  HornerF hcf{};
  void* ar32 = nullptr;  // fp32 staging buffer of the all-reduced density
  Horner hc{};
  int kind = 0, N = 0, order = 1;
  double tol = 0, dt = 0;
  Brick g{};
  int64_t nbricks = 0;
  int n = 0;  // FFT grid points per dim (PIF: upsampled n; PIC: Ng)
  double* grid = nullptr;
  double2* spec = nullptr;
  double2* G3 = nullptr;
  double* grid3 = nullptr;
  double* grid4 = nullptr;  // PIC: interleaved field [n^3][4]
  double2* box = nullptr;
  double* cor = nullptr;  // 1/psi^(2 pi m / n), m in [-N/2, N/2]
  double* S = nullptr;    // S(k_m), m in [-N/2, N/2]
  std::vector<double> hcor, hS;
  cufftHandle fwd = 0, inv = 0;
  size_t wfwd = 0, winv = 0;
  int64_t box_elems() const { return (int64_t)(N + 1) * (N + 1) * (N / 2 + 1); }
  int64_t grid_pts() const { return (int64_t)n * n * n; }
  int64_t spec_elems() const { return (int64_t)n * n * (n / 2 + 1); }
};

}  // namespace

struct pif_ctx_s {
  Phys ph{};
  Plan plan[2];
  int64_t Nglob = 0, first = 0, nloc = 0;
  double q = 0, m = 0;
  int device = 0, rank = 0, world = 1, space_size = 1, time_size = 1, s_idx = 0, t_idx = 0;
  cudaStream_t st = nullptr;
  ncclComm_t comm_world = nullptr, comm_space = nullptr, comm_time = nullptr;
  // parareal hand-off t -> t+1 travels on comm_tp[t % 2]: a rank's sends and
  // receives never share a communicator, so sends can run on st_comm while the
  // next fine propagation runs on st.
  ncclComm_t comm_tp[2] = {nullptr, nullptr};
  cudaStream_t st_comm = nullptr;
  cudaEvent_t ev_ready = nullptr, ev_sent = nullptr;
  bool nccl_broken = false;  // communicators aborted (async error / timeout)
  // parareal states (outside the workspace, include/pif.h): allocated by the
  // first pif_parareal, reused by later calls of the same size, freed by
  // pif_finalize -- a fresh multi-GB allocation per call costs seconds of page
  // mapping inside the timed parareal window
  std::vector<double*> pstates;
  size_t pstate_doubles = 0;
  // workspace
  void* ws = nullptr;
  size_t ws_bytes = 0;
  double *xA = nullptr, *vA = nullptr, *xB = nullptr, *vB = nullptr;
  int *idA = nullptr, *idB = nullptr, *key = nullptr, *rnk = nullptr, *perm = nullptr, *counts = nullptr,
      *offsets = nullptr, *flag = nullptr, *ctr = nullptr, *soff = nullptr, *ioff = nullptr, *moff = nullptr, *spart = nullptr;
  int4 *sitems = nullptr, *iitems = nullptr, *iinfo = nullptr;
  int64_t max_s = 1, max_i = 1;
  double *partials = nullptr, *red = nullptr;
  void* fft_work = nullptr;
  int64_t max_bins = 1;
  // time level
  bool has_state = false, pending = false, box_fresh = false;
  int pending_plan = 0;
  double* host_red = nullptr;  // pinned 8 doubles
  // phase profiling (pif_profile): event pairs per phase, launch counter
  bool prof = false;
  std::vector<cudaEvent_t> ev[PIF_NPHASES];
  size_t ev_used[PIF_NPHASES] = {};
  int64_t launches = 0;
};

namespace {

// Walk the workspace layout (256-byte aligned buffers).  base == nullptr: size
// only, the context is not touched (so a size query or a failed
// pif_set_workspace never clobbers live buffer pointers); otherwise the
// context's buffer pointers are assigned from base.
size_t layout(pif_ctx c, char* base) {
  const bool assign = base != nullptr;
  size_t off = 0;
  auto take = [&](auto& dst, size_t bytes) {
    off = (off + 255) & ~(size_t)255;
    if (assign) dst = reinterpret_cast<std::remove_reference_t<decltype(dst)>>(base + off);
    off += bytes;
  };
  const int64_t n = std::max<int64_t>(c->nloc, 1);
  take(c->xA, 3 * n * sizeof(double));
  take(c->vA, 3 * n * sizeof(double));
  take(c->xB, 3 * n * sizeof(double));
  take(c->vB, 3 * n * sizeof(double));
  take(c->idA, n * sizeof(int));
  take(c->idB, n * sizeof(int));
  take(c->key, n * sizeof(int));
  take(c->rnk, n * sizeof(int));
  take(c->perm, n * sizeof(int));
  take(c->counts, c->max_bins * sizeof(int));
  take(c->offsets, (c->max_bins + 1) * sizeof(int));
  take(c->soff, (c->max_bins + 1) * sizeof(int));
  take(c->ioff, (c->max_bins + 1) * sizeof(int));
  take(c->moff, (c->max_bins + 1) * sizeof(int));
  take(c->spart, sched_part_ints(c->max_bins) * sizeof(int));
  int64_t max_s = 1, max_i = 1;
  for (int i = 0; i < 2; ++i) {
    const Plan& p = c->plan[i];
    if (!p.valid || p.kind != PIF_PROP_PIF_NUFFT) continue;
    const int64_t M = keys_per_brick(p.g);
    max_s = std::max(max_s, sched_max_s(p.nbricks, M, n));
    max_i = std::max(max_i, sched_max_i(p.nbricks, n));
  }
  if (assign) {
    c->max_s = max_s;
    c->max_i = max_i;
  }
  take(c->sitems, max_s * sizeof(int4));
  take(c->iitems, max_i * sizeof(int4));
  take(c->iinfo, max_i * sizeof(int4));
  take(c->flag, 64);
  take(c->ctr, 64);
  take(c->partials, 4 * kReduceBlocks * sizeof(double));
  take(c->red, 16 * sizeof(double));
  size_t fw = 0;
  for (int i = 0; i < 2; ++i) {
    Plan& p = c->plan[i];
    if (!p.valid) continue;
    fw = std::max(fw, std::max(p.wfwd, p.winv));
    take(p.grid, p.grid_pts() * sizeof(double));
    take(p.spec, p.spec_elems() * sizeof(double2));
    take(p.G3, 3 * p.spec_elems() * sizeof(double2));
    take(p.grid3, 3 * p.grid_pts() * sizeof(double));
    if (p.fp32_ar)
      take(p.ar32, (p.kind == PIF_PROP_PIF_NUFFT ? 2 * p.box_elems() : p.grid_pts()) * sizeof(float));
    if (p.kind == PIF_PROP_PIC_CIC) take(p.grid4, 4 * p.grid_pts() * sizeof(double));
    if (p.kind == PIF_PROP_PIF_NUFFT) {
      take(p.box, p.box_elems() * sizeof(double2));
      take(p.cor, (p.N + 1) * sizeof(double));
      take(p.S, (p.N + 1) * sizeof(double));
    }
  }
  take(c->fft_work, std::max<size_t>(fw, 256));
  return off + 256;
}

pif_status make_plan(pif_ctx c, int which, const pif_propagator* pr) {
  Plan& p = c->plan[which];
  if (pr->dt <= 0 || !std::isfinite(pr->dt)) return fail(PIF_ERR_ARG, "dt must be > 0");
  if (pr->spline_order < 1) return fail(PIF_ERR_ARG, "spline_order must be >= 1");
  p.kind = pr->kind;
  p.N = pr->n;
  p.order = pr->spline_order;
  p.fp32_ar = (pr->flags & PIF_FLAG_FP32_ALLREDUCE) != 0;
  p.fp32 = (pr->flags & PIF_FLAG_FP32) != 0;
  p.tol = pr->tol;
  p.dt = pr->dt;
  const double L = c->ph.L;
  if (pr->kind == PIF_PROP_PIF_NUFFT) {
    if (pr->n < 2 || pr->n % 2 || pr->n > 256) return fail(PIF_ERR_ARG, "PIF n must be even in [2, 256]");
    if (!(pr->tol >= 1e-15 && pr->tol < 1e-1)) return fail(PIF_ERR_ARG, "tol must be in [1e-15, 1e-1)");
    int w = es_width(pr->tol);
    int n = 2;
    while (n < std::max(2 * pr->n, 2 * w)) n *= 2;
    // Tile shapes (DMMA needs RZ % 8 == 0 for spreading and
    // (RX RY) % 32 == 0).  w = 13 (eps = 1e-12): interpolation tiles 16x14x16
    // over 4x2x4-cell sub-bricks, spreading tiles 16^3 over 4^3-cell bricks.
    // Small tiles waste fewer FMAs on padding but carry fewer particles per CTA;
    // below ~4 (w = 8; 8 per cell: dense 2.14e9 vs 12^3 1.23e9 particles/s, 2 per
    // cell: 12^3 better) / ~8 (w = 5) particles per upsampled cell the per-CTA
    // overheads win, so the larger tiles are kept there (measured).
#ifndef PIF_W8_PPC
#define PIF_W8_PPC 4.0
#endif
#ifndef PIF_W5_PPC
#define PIF_W5_PPC 8.0
#endif
    const double ppc = (double)c->nloc / ((double)n * n * n);
    int RI[3], m[3] = {1, 1, 1};
    if (w == 5 && ppc >= PIF_W5_PPC) { RI[0] = RI[1] = 6; RI[2] = 8; m[0] = m[1] = 2; }      // spread 8^3
    else if (w <= 5) { RI[0] = RI[1] = RI[2] = 8; }
    else if (w == 8 && ppc >= PIF_W8_PPC) { RI[0] = RI[1] = 10; RI[2] = 8; m[0] = m[1] = 3; }  // spread 16x16x8
    else if (w <= 9) { RI[0] = RI[1] = RI[2] = 12; }
    else if (w == 13) { RI[0] = 14; RI[1] = 14; RI[2] = 16; m[0] = m[1] = 2; }
    else { RI[0] = RI[1] = RI[2] = 16; }
    Brick& g = p.g;
    g.n = n;
    g.w = w;
    g.hw = (w - 1) / 2;
    g.odd = w & 1;
    g.nkeys = 1;
    for (int d = 0; d < 3; ++d) {
      g.RI[d] = RI[d];
      g.ib[d] = RI[d] - w + 1;
      g.m[d] = m[d];
      g.sb[d] = g.ib[d] * m[d];
      g.RS[d] = g.sb[d] + w - 1;
      g.NB[d] = (n + g.sb[d] - 1) / g.sb[d];
      g.rsb[d] = 1.0f / (float)g.sb[d];
      g.rib[d] = 1.0f / (float)g.ib[d];
      g.nkeys *= (int64_t)g.NB[d] * m[d];
    }
    // slab interpolation tiles: keys down to the xy-cells of a sub-brick, so an
    // m-tile of 8 consecutive particles usually shares one cell and its window
    // (w = 13: 13 x 13 columns instead of the tile's 14 x 14)
#ifndef PIF_CELL_KEYS
#ifdef PIF_NO_SLAB
#define PIF_CELL_KEYS 0
#else
#define PIF_CELL_KEYS 1
#endif
#endif
    const bool slab = (RI[0] == 14 && RI[1] == 14 && RI[2] == 16) || (RI[0] == 10 && RI[1] == 10 && RI[2] == 8) ||
                      (RI[0] == 6 && RI[1] == 6 && RI[2] == 8);
    g.C = (PIF_CELL_KEYS && slab && m[2] == 1) ? g.ib[0] * g.ib[1] : 1;
    g.nkeys *= g.C;
    g.scale = n / L;
    g.beta = es_beta(w);
    horner_fit(w, g.beta, p.hc);
    for (int k = 0; k < 16; ++k)
      for (int j = 0; j <= kHornerDeg; ++j) p.hcf.a[k][j] = (float)p.hc.a[k][j];
    // small widths: the per-particle vector kernel (w <= 5; w = 6 in fp32)
    p.simt = simt_interp_supported(g) && (w <= 5 || p.fp32);
    if (p.fp32 && !p.simt) return fail(PIF_ERR_ARG, "PIF_FLAG_FP32 needs tol >= 1e-5");
    p.n = n;
    p.nbricks = g.nkeys;
    c->max_bins = std::max(c->max_bins, p.nbricks);
    const int H = p.N / 2;
    p.hcor.resize(p.N + 1);
    p.hS.resize(p.N + 1);
    const double h = L / p.N;
    for (int m = -H; m <= H; ++m) {
      p.hcor[m + H] = 1.0 / es_hat(2.0 * M_PI * m / n, w, g.beta);
      double k = 2.0 * M_PI * m / L, u = 0.5 * k * h;
      double sinc = m == 0 ? 1.0 : std::sin(u) / u;
      p.hS[m + H] = std::pow(sinc, p.order + 1);  // S(k) = sinc^(m+1)(k h / 2), R3/R4
    }
  } else if (pr->kind == PIF_PROP_PIC_CIC) {
    if (pr->n < 4 || pr->n % 2 || pr->n > 512) return fail(PIF_ERR_ARG, "PIC n must be even in [4, 512]");
    if (pr->spline_order != 1) return fail(PIF_ERR_ARG, "PIC supports spline_order 1 (CIC) only");
    p.n = pr->n;
  } else {
    return fail(PIF_ERR_ARG, "unknown propagator kind");
  }
  const int n = p.n;
  CUFFT(cufftCreate(&p.fwd));
  CUFFT(cufftSetAutoAllocation(p.fwd, 0));
  CUFFT(cufftMakePlan3d(p.fwd, n, n, n, CUFFT_D2Z, &p.wfwd));
  CUFFT(cufftCreate(&p.inv));
  CUFFT(cufftSetAutoAllocation(p.inv, 0));
  int dims[3] = {n, n, n};
  // fp32 plans: the three inverse transforms in single precision (C2R), whose
  // float grids feed the fp32 interpolation directly
  CUFFT(cufftMakePlanMany(p.inv, 3, dims, nullptr, 1, 0, nullptr, 1, 0, p.fp32 ? CUFFT_C2R : CUFFT_Z2D, 3,
                          &p.winv));
  CUFFT(cufftSetStream(p.fwd, c->st));
  CUFFT(cufftSetStream(p.inv, c->st));
  p.valid = true;
  return PIF_OK;
}

// Host-only argument validation (no CUDA calls), so bad input fails fast.
pif_status validate_prop(const pif_propagator* pr) {
  if (!(pr->dt > 0) || !std::isfinite(pr->dt)) return fail(PIF_ERR_ARG, "dt must be > 0");
  if (pr->spline_order < 1) return fail(PIF_ERR_ARG, "spline_order must be >= 1");
  if (pr->kind == PIF_PROP_PIF_NUFFT) {
    if (pr->n < 2 || pr->n % 2 || pr->n > 256) return fail(PIF_ERR_ARG, "PIF n must be even in [2, 256]");
    if (!(pr->tol >= 1e-15 && pr->tol < 1e-1)) return fail(PIF_ERR_ARG, "tol must be in [1e-15, 1e-1)");
    if ((pr->flags & PIF_FLAG_FP32) && !(pr->tol >= 1e-5))
      return fail(PIF_ERR_ARG, "PIF_FLAG_FP32 needs tol >= 1e-5");
  } else if (pr->kind == PIF_PROP_PIC_CIC) {
    if (pr->n < 4 || pr->n % 2 || pr->n > 512) return fail(PIF_ERR_ARG, "PIC n must be even in [4, 512]");
    if (pr->spline_order != 1) return fail(PIF_ERR_ARG, "PIC supports spline_order 1 (CIC) only");
    if (pr->flags & PIF_FLAG_FP32) return fail(PIF_ERR_ARG, "PIF_FLAG_FP32 applies to PIF propagators");
  } else {
    return fail(PIF_ERR_ARG, "unknown propagator kind");
  }
  return PIF_OK;
}

// The three inverse transforms G3 -> grid3 (fp64, or fp32 for PIF_FLAG_FP32).
cufftResult inverse_fft(const Plan& p) {
  if (p.fp32) return cufftExecC2R(p.inv, (cufftComplex*)p.G3, (cufftReal*)p.grid3);
  return cufftExecZ2D(p.inv, (cufftDoubleComplex*)p.G3, p.grid3);
}

// Fused type-2 interpolation + push of plan p (tensor-core or vector kernel).
cudaError_t interp_push(pif_ctx c, const Plan& p, double* x, double* v, int64_t stride, const int* id,
                        double* Eout, const Sched& S, const PushArgs& P) {
  if (p.simt)
    return launch_interp_push_simt(p.grid3, x, v, stride, id, Eout, S, p.g, p.hc, p.hcf, p.fp32, P, c->st);
  return launch_interp_push(p.grid3, x, v, stride, id, Eout, S, p.g, p.hc, P, c->st);
}

PushArgs push_args(pif_ctx c, const Plan& p, int kicks, int drift) {
  PushArgs P{};
  P.L = c->ph.L;
  P.dt = p.dt;
  P.h = 0.25 * p.dt * c->ph.qm;
  P.magnetic = (c->ph.B[0] != 0 || c->ph.B[1] != 0 || c->ph.B[2] != 0);
  double t2 = 0;
  for (int d = 0; d < 3; ++d) {
    P.t[d] = P.h * c->ph.B[d];
    t2 += P.t[d] * P.t[d];
  }
  for (int d = 0; d < 3; ++d) P.s[d] = 2.0 * P.t[d] / (1.0 + t2);
  P.has_ext = 0;
  for (int i = 0; i < 9; ++i) {
    P.A[i] = c->ph.A[i];
    if (P.A[i] != 0) P.has_ext = 1;
  }
  for (int d = 0; d < 3; ++d) {
    P.c[d] = c->ph.c[d];
    if (P.c[d] != 0) P.has_ext = 1;
  }
  P.kicks = kicks;
  P.drift = drift;
  return P;
}

pif_status need_ready(pif_ctx c) {
  if (!c) return fail(PIF_ERR_ARG, "null context");
  if (!c->ws) return fail(PIF_ERR_STATE, "workspace not set (pif_set_workspace)");
  if (!c->has_state) return fail(PIF_ERR_STATE, "state not set (pif_set_state)");
  return PIF_OK;
}

// Phase events (only when profiling is on): a start/stop pair per phase call.
pif_status ph_mark(pif_ctx c, int ph) {
  if (!c->prof) return PIF_OK;
  auto& v = c->ev[ph];
  if (c->ev_used[ph] == v.size()) {
    cudaEvent_t e;
    CU(cudaEventCreate(&e));
    v.push_back(e);
  }
  CU(cudaEventRecord(v[c->ev_used[ph]++], c->st));
  return PIF_OK;
}
// Each phase: CUDA events when profiling is on (pif_profile) and an NVTX range
// (header-only NVTX v3: free unless a tool such as nsys / ncu attaches).
const char* const kPhaseName[PH_COUNT] = {"pif.sort", "pif.spread", "pif.fft_fwd", "pif.box",
                                          "pif.allreduce", "pif.poisson", "pif.fft_inv", "pif.interp_push",
                                          "pif.pic_deposit", "pif.pic_gather_push", "pif.other"};
#define PH(ph, body)                 \
  do {                               \
    nvtxRangePushA(kPhaseName[ph]);  \
    TRY(ph_mark(c, ph));             \
    body;                            \
    TRY(ph_mark(c, ph));             \
    nvtxRangePop();                  \
  } while (0)

Sched sched_of(pif_ctx c, const Plan& p) {
  const int64_t M = keys_per_brick(p.g);
  return Sched{c->offsets, c->soff, c->ioff, c->moff, c->sitems, c->iitems, c->iinfo, c->spart, p.nbricks,
               sched_max_s(p.nbricks, M, c->nloc), sched_max_i(p.nbricks, c->nloc), c->ctr};
}

// a0: counting sort of the working particles (xA, vA, idA) by brick of plan p.
// fused (PIF_FUSED_SORT): only the permutation perm[sorted j] = current index is
// built; the spread reads x through it and the interpolation + push reads x, v,
// id through it and writes the pushed particles in sorted order into xB, vB,
// idB (then swapped in) -- the separate gather pass (~108 B per particle of HBM
// traffic) disappears.  Otherwise the particles are gathered here.
#ifndef PIF_FUSED_SORT
#define PIF_FUSED_SORT 1
#endif
pif_status sort_particles(pif_ctx c, Plan& p, bool fused) {
  const int64_t n = c->nloc;
  CU(cudaMemsetAsync(c->counts, 0, p.nbricks * sizeof(int), c->st));
  CU(launch_bin_count(c->xA, n, n, p.g, c->key, c->rnk, c->counts, c->st));
  CU(launch_schedule(c->counts, sched_of(c, p), p.g, keys_per_brick(p.g), p.g.C, c->st));
  if (fused) {
    CU(launch_scatter_index(n, c->key, c->rnk, c->offsets, c->perm, c->st));
    return PIF_OK;
  }
  CU(launch_gather_sorted(c->xA, c->vA, c->idA, nullptr, n, n, c->key, c->rnk, c->offsets, c->perm,
                          c->xB, c->vB, c->idB, nullptr, c->st));
  std::swap(c->xA, c->xB);
  std::swap(c->vA, c->vB);
  std::swap(c->idA, c->idB);
  return PIF_OK;
}

// Sum the density buffer (count doubles) over the space group: fp64, or fp32
// (PIF_FLAG_FP32_ALLREDUCE) through the plan's float staging buffer.
pif_status density_allreduce(pif_ctx c, Plan& p, double* buf, int64_t count) {
  if (!p.fp32_ar) {
    NC(ncclAllReduce(buf, buf, count, ncclDouble, ncclSum, c->comm_space, c->st));
    return PIF_OK;
  }
  CU(launch_convert(buf, (float*)p.ar32, count, true, c->st));
  NC(ncclAllReduce(p.ar32, p.ar32, count, ncclFloat, ncclSum, c->comm_space, c->st));
  CU(launch_convert(buf, (float*)p.ar32, count, false, c->st));
  return PIF_OK;
}

// One field solve of plan `which` at the current positions followed by the
// fused interpolation + push (kicks half kicks, optional drift).
pif_status solve_and_push(pif_ctx c, int which, int kicks, int drift) {
  Plan& p = c->plan[which];
  const int64_t n = c->nloc;
  PushArgs P = push_args(c, p, kicks, drift);
  if (p.kind == PIF_PROP_PIF_NUFFT) {
    // a push (kicks or drift) writes the sorted copy; a field-only solve (the
    // diagnostics' box) leaves the particles where they are
    const bool push = kicks > 0 || drift;
    const bool fused = PIF_FUSED_SORT && push;
    const int* perm = fused ? c->perm : nullptr;
    PH(PH_SORT, TRY(sort_particles(c, p, fused)));
    PH(PH_SPREAD, {
      CU(cudaMemsetAsync(p.grid, 0, p.grid_pts() * sizeof(double), c->st));
      CU(launch_spread(c->xA, perm, n, nullptr, 1.0, sched_of(c, p), p.g, p.hc,
                        p.fp32 ? &p.hcf : nullptr, p.grid, c->st));
    });
    PH(PH_FFT_FWD, CUFFT(cufftExecD2Z(p.fwd, p.grid, (cufftDoubleComplex*)p.spec)));
    const double L = c->ph.L;
    PH(PH_BOX, CU(launch_extract_box(p.spec, p.n, p.N, p.cor, c->q / (L * L * L), p.box, c->st)));
    if (c->space_size > 1)
      PH(PH_ALLREDUCE, TRY(density_allreduce(c, p, (double*)p.box, 2 * p.box_elems())));
    PH(PH_POISSON, CU(launch_poisson_pad(p.box, p.n, p.N, L, p.cor, p.S, p.G3, p.fp32, c->st)));
    PH(PH_FFT_INV, CUFFT(inverse_fft(p)));
    if (fused) {
      P.perm = c->perm;
      P.xo = c->xB;
      P.vo = c->vB;
      P.ido = c->idB;
    }
    if (push) PH(PH_INTERP_PUSH, CU(interp_push(c, p, c->xA, c->vA, n, c->idA, nullptr, sched_of(c, p), P)));
    if (fused) {
      std::swap(c->xA, c->xB);
      std::swap(c->vA, c->vB);
      std::swap(c->idA, c->idB);
    }
    // own kernels: bin, schedule (reduce, partials, apply, fill), sort (index
    // scatter [+ gather]), spread, extract, poisson, interp_push (cuFFT not counted)
    c->launches += 9 + (fused ? 0 : 1) + (push ? 1 : 0);
    c->box_fresh = (which == 0) && !drift;
  } else {
    const int Ng = p.n;
    const double h = c->ph.L / Ng;
    PH(PH_PIC_DEPOSIT, {
      CU(cudaMemsetAsync(p.grid, 0, p.grid_pts() * sizeof(double), c->st));
      CU(launch_cic_deposit(c->xA, n, n, Ng, 1.0 / h, p.grid, c->st));
    });
    if (c->space_size > 1)
      PH(PH_ALLREDUCE, TRY(density_allreduce(c, p, p.grid, p.grid_pts())));
    PH(PH_FFT_FWD, CUFFT(cufftExecD2Z(p.fwd, p.grid, (cufftDoubleComplex*)p.spec)));
    double scale = c->q / (h * h * h) / (double)p.grid_pts();
    PH(PH_POISSON, CU(launch_pic_poisson(p.spec, Ng, c->ph.L, scale, p.G3, c->st)));
    PH(PH_FFT_INV, CUFFT(cufftExecZ2D(p.inv, (cufftDoubleComplex*)p.G3, p.grid3)));
    c->launches += 2;
    if (kicks > 0 || drift) {
      PH(PH_PIC_GATHER_PUSH, CU(launch_cic_gather_push(p.grid3, p.grid4, c->xA, c->vA, n, n, Ng, 1.0 / h,
                                                       P, c->st)));
      c->launches += 2;
    }
    c->box_fresh = (which == 0) && !drift;
  }
  return PIF_OK;
}

pif_status materialize(pif_ctx c) {
  if (!c->pending) return PIF_OK;
  TRY(solve_and_push(c, c->pending_plan, 1, 0));
  c->pending = false;
  return PIF_OK;
}

pif_status step_internal(pif_ctx c, int which, int64_t nsteps) {
  if (nsteps <= 0) return PIF_OK;
  if (c->pending && c->pending_plan != which) TRY(materialize(c));
  for (int64_t s = 0; s < nsteps; ++s) {
    TRY(solve_and_push(c, which, c->pending ? 2 : 1, 1));
    c->pending = true;
    c->pending_plan = which;
  }
  c->box_fresh = false;
  return PIF_OK;
}

// Failure detection for the multi-process paths: abort every communicator of
// the context (pending NCCL kernels then return), after which the context only
// accepts pif_finalize.
void abort_comms(pif_ctx c) {
  ncclComm_t* all[] = {&c->comm_tp[0], &c->comm_tp[1], &c->comm_space, &c->comm_time, &c->comm_world};
  for (ncclComm_t* p : all)
    if (*p) {
      ncclCommAbort(*p);
      *p = nullptr;
    }
  c->nccl_broken = true;
}

double nccl_timeout_s() {
  const char* e = getenv("PIF_NCCL_TIMEOUT_S");
  const double t = e ? atof(e) : 0.0;
  return t > 0 ? t : 600.0;
}

// Wait for stream st.  world == 1: cudaStreamSynchronize.  Otherwise poll the
// stream and every communicator's asynchronous error state, so that an NCCL
// error or a peer that never answers (no progress for PIF_NCCL_TIMEOUT_S
// seconds, default 600) aborts the communicators and returns PIF_ERR_NCCL
// instead of hanging every later slice of the parareal pipeline.
pif_status sync_stream(pif_ctx c, cudaStream_t st) {
  if (c->world == 1) {
    CU(cudaStreamSynchronize(st));
    return PIF_OK;
  }
  if (c->nccl_broken) return fail(PIF_ERR_NCCL, "communicators were aborted by an earlier NCCL failure");
  const double t0 = std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
  const double limit = nccl_timeout_s();
  for (unsigned spin = 0;; ++spin) {
    const cudaError_t e = cudaStreamQuery(st);
    if (e == cudaSuccess) return PIF_OK;
    if (e != cudaErrorNotReady) return fail(PIF_ERR_CUDA, std::string("stream: ") + cudaGetErrorString(e));
    if ((spin & 255) != 255) continue;
    ncclComm_t comms[] = {c->comm_world, c->comm_space, c->comm_time, c->comm_tp[0], c->comm_tp[1]};
    for (ncclComm_t cm : comms) {
      if (!cm) continue;
      ncclResult_t ae = ncclSuccess;
      if (ncclCommGetAsyncError(cm, &ae) == ncclSuccess && ae != ncclSuccess && ae != ncclInProgress) {
        abort_comms(c);
        return fail(PIF_ERR_NCCL, std::string("asynchronous NCCL error: ") + ncclGetErrorString(ae));
      }
    }
    const double t = std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
    if (t - t0 > limit) {
      abort_comms(c);
      return fail(PIF_ERR_NCCL, "NCCL watchdog: no progress for " + std::to_string(limit) +
                                    " s (lost peer?); communicators aborted");
    }
    std::this_thread::yield();
  }
}

// PIF_ERR_NUMERIC check of (a, na) and (b, nb) (b may be null) with one
// synchronisation.  wrap_L > 0: a holds positions, wrapped into [0, L) in place
// (inputs outside the periodic box are legal; anchor_of needs [0, L)).
pif_status check_state(pif_ctx c, double* a, int64_t na, const double* b, int64_t nb, double wrap_L,
                       const char* what) {
  CU(cudaMemsetAsync(c->flag, 0, sizeof(int), c->st));
  CU(launch_check_finite(a, na, wrap_L, c->flag, c->st));
  if (b) CU(launch_check_finite(const_cast<double*>(b), nb, 0.0, c->flag, c->st));
  CU(cudaMemcpyAsync(&c->host_red[12], c->flag, sizeof(int), cudaMemcpyDeviceToHost, c->st));
  TRY(sync_stream(c, c->st));
  int bad = 0;
  memcpy(&bad, &c->host_red[12], sizeof(int));
  if (bad) return fail(PIF_ERR_NUMERIC, std::string("non-finite values in ") + what);
  return PIF_OK;
}

// Canonical-order state buffer: [x(3n) | v(3n) | flag(1)] doubles.
struct State {
  double* p = nullptr;
};

pif_status load_state(pif_ctx c, const double* s) {
  const int64_t n = c->nloc;
  CU(cudaMemcpyAsync(c->xA, s, 3 * n * sizeof(double), cudaMemcpyDeviceToDevice, c->st));
  CU(cudaMemcpyAsync(c->vA, s + 3 * n, 3 * n * sizeof(double), cudaMemcpyDeviceToDevice, c->st));
  CU(launch_iota(c->idA, n, c->st));
  c->pending = false;
  c->box_fresh = false;
  c->has_state = true;
  return PIF_OK;
}

pif_status store_state(pif_ctx c, double* s) {
  TRY(materialize(c));
  const int64_t n = c->nloc;
  CU(launch_scatter_by_id(c->xA, c->vA, c->idA, n, n, s, s + 3 * n, c->st));
  return PIF_OK;
}

double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

// ============================================================================
extern "C" {

const char* pif_last_error(void) { return g_err.c_str(); }

pif_status pif_nccl_unique_id(void* out128) {
  if (!out128) return fail(PIF_ERR_ARG, "null output");
  ncclUniqueId id;
  NC(ncclGetUniqueId(&id));
  memcpy(out128, &id, sizeof(id));
  return PIF_OK;
}

pif_status pif_init(const pif_physics* phys, const pif_propagator* fine,
                    const pif_propagator* coarse, int64_t n_particles_global,
                    const pif_dist* dist, pif_ctx* out) {
  if (!phys || !fine || !dist || !out) return fail(PIF_ERR_ARG, "null argument");
  if (!(phys->L > 0) || !std::isfinite(phys->L)) return fail(PIF_ERR_ARG, "L must be > 0");
  if (phys->total_charge == 0 || !std::isfinite(phys->total_charge))
    return fail(PIF_ERR_ARG, "total_charge must be nonzero");
  if (n_particles_global < 1 || n_particles_global > (int64_t)1 << 31)
    return fail(PIF_ERR_ARG, "n_particles_global must be in [1, 2^31]");
  if (dist->world < 1 || dist->rank < 0 || dist->rank >= dist->world || dist->space_size < 1 ||
      dist->world % dist->space_size)
    return fail(PIF_ERR_CONFIG, "bad process layout (space_size must divide world)");
  if (dist->world > 1 && !dist->nccl_id) return fail(PIF_ERR_ARG, "nccl_id required for world > 1");
  TRY(validate_prop(fine));
  if (coarse) TRY(validate_prop(coarse));
  if (coarse && fine->kind == PIF_PROP_PIF_NUFFT && coarse->kind == PIF_PROP_PIF_NUFFT &&
      coarse->tol < fine->tol)
    return fail(PIF_ERR_CONFIG, "coarse tolerance must be >= fine tolerance");
  pif_ctx c = new pif_ctx_s();
  c->ph.L = phys->L;
  c->ph.qm = phys->q_over_m;
  c->ph.Q = phys->total_charge;
  for (int d = 0; d < 3; ++d) {
    c->ph.B[d] = phys->B_ext[d];
    c->ph.c[d] = phys->E_ext_c[d];
  }
  for (int i = 0; i < 9; ++i) c->ph.A[i] = phys->E_ext_A[i];
  c->Nglob = n_particles_global;
  c->q = phys->total_charge / (double)n_particles_global;      // R6
  c->m = std::fabs(phys->total_charge) / (double)n_particles_global;
  c->device = dist->device;
  c->rank = dist->rank;
  c->world = dist->world;
  c->space_size = dist->space_size;
  c->time_size = dist->world / dist->space_size;
  c->s_idx = dist->rank % dist->space_size;
  c->t_idx = dist->rank / dist->space_size;
  c->st = (cudaStream_t)dist->stream;
  pif_partition(n_particles_global, c->space_size, c->s_idx, &c->first, &c->nloc);
  auto bail = [&](pif_status s) {
    std::string msg = g_err;
    pif_finalize(c);
    g_err = msg;
    return s;
  };
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || c->device < 0 || c->device >= ndev) {
    delete c;
    return fail(PIF_ERR_CUDA, std::string("no CUDA device ") + std::to_string(dist->device) + ": " +
                                  cudaGetErrorString(e));
  }
  DeviceGuard dg(c->device);
  pif_status s = make_plan(c, 0, fine);
  if (s != PIF_OK) return bail(s);
  if (coarse) {
    s = make_plan(c, 1, coarse);
    if (s != PIF_OK) return bail(s);
  }
  e = cudaMallocHost(&c->host_red, 16 * sizeof(double));
  if (e != cudaSuccess) {
    fail(PIF_ERR_CUDA, std::string("cudaMallocHost: ") + cudaGetErrorString(e));
    return bail(PIF_ERR_CUDA);
  }
  if (c->world > 1) {
    ncclUniqueId id;
    memcpy(&id, dist->nccl_id, sizeof(id));
    ncclResult_t r = ncclCommInitRank(&c->comm_world, c->world, id, c->rank);
    if (r != ncclSuccess) {
      fail(PIF_ERR_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
      return bail(PIF_ERR_NCCL);
    }
    // space group: same time index; time group: same space index.
    r = ncclCommSplit(c->comm_world, c->t_idx, c->s_idx, &c->comm_space, nullptr);
    if (r == ncclSuccess) r = ncclCommSplit(c->comm_world, c->s_idx, c->t_idx, &c->comm_time, nullptr);
    if (r == ncclSuccess && c->time_size > 1) {
      r = ncclCommSplit(c->comm_time, 0, c->t_idx, &c->comm_tp[0], nullptr);
      if (r == ncclSuccess) r = ncclCommSplit(c->comm_time, 0, c->t_idx, &c->comm_tp[1], nullptr);
    }
    if (r != ncclSuccess) {
      fail(PIF_ERR_NCCL, std::string("ncclCommSplit: ") + ncclGetErrorString(r));
      return bail(PIF_ERR_NCCL);
    }
  }
  if (c->time_size > 1) {
    e = cudaStreamCreateWithFlags(&c->st_comm, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_ready, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_sent, cudaEventDisableTiming);
    if (e != cudaSuccess) {
      fail(PIF_ERR_CUDA, std::string("comm stream: ") + cudaGetErrorString(e));
      return bail(PIF_ERR_CUDA);
    }
    // Establish the t -> t+1 peer connections now (NCCL connects lazily on the
    // first send/recv), so that pif_parareal's timing excludes setup.
    double* tmp = nullptr;
    e = cudaMalloc(&tmp, 2 * sizeof(double));
    if (e != cudaSuccess) {
      fail(PIF_ERR_CUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e));
      return bail(PIF_ERR_CUDA);
    }
    const int t = c->t_idx, T = c->time_size;
    ncclResult_t r = ncclGroupStart();
    if (r == ncclSuccess && t + 1 < T) r = ncclSend(tmp, 1, ncclDouble, t + 1, c->comm_tp[t % 2], c->st);
    if (r == ncclSuccess && t > 0) r = ncclRecv(tmp + 1, 1, ncclDouble, t - 1, c->comm_tp[(t + 1) % 2], c->st);
    ncclResult_t r2 = ncclGroupEnd();
    if (r == ncclSuccess) r = r2;
    e = cudaStreamSynchronize(c->st);
    cudaFree(tmp);
    if (r != ncclSuccess || e != cudaSuccess) {
      fail(PIF_ERR_NCCL, "parareal peer warm-up failed");
      return bail(PIF_ERR_NCCL);
    }
  }
  *out = c;
  return PIF_OK;
}

pif_status pif_partition(int64_t n_global, int32_t space_size, int32_t s_idx, int64_t* first,
                         int64_t* count) {
  if (!first || !count || n_global < 0 || space_size < 1 || s_idx < 0 || s_idx >= space_size)
    return fail(PIF_ERR_ARG, "bad partition arguments");
  const int64_t base = n_global / space_size, rem = n_global % space_size;
  *count = base + (s_idx < rem ? 1 : 0);
  *first = s_idx * base + std::min<int64_t>(s_idx, rem);
  return PIF_OK;
}

pif_status pif_local_count(pif_ctx c, int64_t* first, int64_t* count) {
  if (!c || !first || !count) return fail(PIF_ERR_ARG, "null argument");
  *first = c->first;
  *count = c->nloc;
  return PIF_OK;
}

pif_status pif_workspace_size(pif_ctx c, size_t* bytes) {
  if (!c || !bytes) return fail(PIF_ERR_ARG, "null argument");
  *bytes = layout(c, nullptr);
  return PIF_OK;
}

pif_status pif_set_workspace(pif_ctx c, void* dptr, size_t bytes) {
  if (!c || !dptr) return fail(PIF_ERR_ARG, "null argument");
  if ((uintptr_t)dptr % 256) return fail(PIF_ERR_ARG, "workspace must be 256-byte aligned");
  size_t need = layout(c, nullptr);
  if (bytes < need) return fail(PIF_ERR_OOM, "workspace too small: need " + std::to_string(need));
  DeviceGuard dg(c->device);
  TRY(sync_stream(c, c->st));  // nothing in flight may use the old workspace
  layout(c, (char*)dptr);
  c->ws = dptr;
  c->ws_bytes = bytes;
  for (int i = 0; i < 2; ++i) {
    Plan& p = c->plan[i];
    if (!p.valid) continue;
    CUFFT(cufftSetWorkArea(p.fwd, c->fft_work));
    CUFFT(cufftSetWorkArea(p.inv, c->fft_work));
    if (p.kind == PIF_PROP_PIF_NUFFT) {
      CU(cudaMemcpyAsync(p.cor, p.hcor.data(), (p.N + 1) * sizeof(double), cudaMemcpyHostToDevice, c->st));
      CU(cudaMemcpyAsync(p.S, p.hS.data(), (p.N + 1) * sizeof(double), cudaMemcpyHostToDevice, c->st));
    }
  }
  TRY(sync_stream(c, c->st));
  c->has_state = false;
  return PIF_OK;
}

pif_status pif_set_state(pif_ctx c, const double* x, const double* v, int64_t n_local,
                         int on_device) {
  if (!c || !x || !v) return fail(PIF_ERR_ARG, "null argument");
  if (!c->ws) return fail(PIF_ERR_STATE, "workspace not set");
  if (n_local != c->nloc) return fail(PIF_ERR_ARG, "n_local mismatch: expected " + std::to_string(c->nloc));
  DeviceGuard dg(c->device);
  const size_t b = 3 * n_local * sizeof(double);
  cudaMemcpyKind k = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  CU(cudaMemcpyAsync(c->xA, x, b, k, c->st));
  CU(cudaMemcpyAsync(c->vA, v, b, k, c->st));
  CU(launch_iota(c->idA, n_local, c->st));
  c->has_state = false;
  TRY(check_state(c, c->xA, 3 * n_local, c->vA, 3 * n_local, c->ph.L, "the input state"));
  c->has_state = true;
  c->pending = false;
  c->box_fresh = false;
  return PIF_OK;
}

pif_status pif_get_state(pif_ctx c, double* x, double* v, int64_t n_local, int on_device) {
  TRY(need_ready(c));
  if (!x || !v) return fail(PIF_ERR_ARG, "null argument");
  if (n_local != c->nloc) return fail(PIF_ERR_ARG, "n_local mismatch");
  DeviceGuard dg(c->device);
  TRY(materialize(c));
  const int64_t n = c->nloc;
  CU(launch_scatter_by_id(c->xA, c->vA, c->idA, n, n, c->xB, c->vB, c->st));
  TRY(check_state(c, c->xB, 3 * n, c->vB, 3 * n, 0.0, "the state"));
  cudaMemcpyKind k = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  CU(cudaMemcpyAsync(x, c->xB, 3 * n * sizeof(double), k, c->st));
  CU(cudaMemcpyAsync(v, c->vB, 3 * n * sizeof(double), k, c->st));
  if (!on_device) TRY(sync_stream(c, c->st));
  return PIF_OK;
}

pif_status pif_step(pif_ctx c, int which, int64_t n_steps) {
  TRY(need_ready(c));
  if (which < 0 || which > 1 || !c->plan[which].valid) return fail(PIF_ERR_ARG, "no such propagator");
  if (n_steps < 0) return fail(PIF_ERR_ARG, "n_steps must be >= 0");
  if (c->nccl_broken) return fail(PIF_ERR_NCCL, "communicators were aborted by an earlier NCCL failure");
  DeviceGuard dg(c->device);
  return step_internal(c, which, n_steps);
}

pif_status pif_field_energy(pif_ctx c, double W[3], double* kinetic, double momentum[3],
                            double* charge_err) {
  TRY(need_ready(c));
  if (!W || !kinetic || !momentum || !charge_err) return fail(PIF_ERR_ARG, "null argument");
  DeviceGuard dg(c->device);
  TRY(materialize(c));
  Plan& p = c->plan[0];
  if (!c->box_fresh) TRY(solve_and_push(c, 0, 0, 0));
  const double L = c->ph.L;
  if (p.kind == PIF_PROP_PIF_NUFFT) {
    CU(launch_field_energy(p.box, p.N, L, p.S, c->red, c->st));
  } else {
    const double h = L / p.n;
    CU(launch_grid_energy(p.grid3, p.grid_pts(), h * h * h, c->partials, c->red, c->st));
  }
  CU(launch_particle_moments(c->vA, c->nloc, c->nloc, c->partials, c->red + 4, c->st));
  if (c->space_size > 1)
    NC(ncclAllReduce(c->red + 4, c->red + 4, 4, ncclDouble, ncclSum, c->comm_space, c->st));
  CU(cudaMemcpyAsync(c->host_red, c->red, 8 * sizeof(double), cudaMemcpyDeviceToHost, c->st));
  TRY(sync_stream(c, c->st));
  const double* r = c->host_red;
  if (p.kind == PIF_PROP_PIF_NUFFT) {
    for (int d = 0; d < 3; ++d) W[d] = r[d];
    *charge_err = std::fabs(L * L * L * r[3] - c->ph.Q) / std::fabs(c->ph.Q);
  } else {
    const double h = L / p.n;
    for (int d = 0; d < 3; ++d) W[d] = 0.5 * h * h * h * r[d];
    *charge_err = 0.0;
  }
  *kinetic = 0.5 * c->m * r[4];
  for (int d = 0; d < 3; ++d) momentum[d] = c->m * r[5 + d];
  for (int q = 0; q < 8; ++q)
    if (!std::isfinite(r[q])) return fail(PIF_ERR_NUMERIC, "non-finite field energy / moments");
  return PIF_OK;
}

pif_status pif_get_rho(pif_ctx c, double* out) {
  TRY(need_ready(c));
  if (!out) return fail(PIF_ERR_ARG, "null argument");
  Plan& p = c->plan[0];
  if (p.kind != PIF_PROP_PIF_NUFFT) return fail(PIF_ERR_CONFIG, "fine propagator is not PIF");
  DeviceGuard dg(c->device);
  TRY(materialize(c));
  if (!c->box_fresh) TRY(solve_and_push(c, 0, 0, 0));
  CU(cudaMemcpyAsync(out, p.box, p.box_elems() * sizeof(double2), cudaMemcpyDeviceToHost, c->st));
  TRY(sync_stream(c, c->st));
  return PIF_OK;
}

pif_status pif_plan_info(pif_ctx c, int which, int32_t* w, double* beta, int32_t* n_up) {
  if (!c || which < 0 || which > 1 || !c->plan[which].valid) return fail(PIF_ERR_ARG, "bad plan");
  const Plan& p = c->plan[which];
  if (w) *w = p.kind == PIF_PROP_PIF_NUFFT ? p.g.w : 2;
  if (beta) *beta = p.kind == PIF_PROP_PIF_NUFFT ? p.g.beta : 0.0;
  if (n_up) *n_up = p.n;
  return PIF_OK;
}

// ---------------------------------------------------------------- parareal --
// One parareal window [t0, t1] with n_slices slices (the body of pif_parareal).
static pif_status parareal_window(pif_ctx c, double t0, double t1, int32_t n_slices,
                                  int32_t max_iter, double stop_tol, pif_parareal_report* rep) {
  const double dT = (t1 - t0) / n_slices;
  const int64_t nf = llround(dT / c->plan[0].dt), ng = llround(dT / c->plan[1].dt);
  if (nf < 1 || ng < 1 || std::fabs(nf * c->plan[0].dt - dT) > 1e-9 * dT ||
      std::fabs(ng * c->plan[1].dt - dT) > 1e-9 * dT)
    return fail(PIF_ERR_CONFIG, "slice length must be an integer multiple of both dt");
  const int64_t n = c->nloc, SZ = 6 * n + 1;
  const double L = c->ph.L;
  double tt0 = now();
  double t_fine = 0, t_coarse = 0, t_comm = 0, t_coarse0 = 0;
  for (int i = 0; i < max_iter * n_slices; ++i) rep->err_x[i] = rep->err_v[i] = NAN;
  for (int i = 0; i < n_slices; ++i) rep->retired_at[i] = -1;

  // Parareal states live outside the workspace (include/pif.h): stream-ordered
  // allocations released on every exit path.
  DevBufs bufs(c->st);
  if (c->pstate_doubles != (size_t)SZ) {
    TRY(sync_stream(c, c->st));
    for (double* q : c->pstates) cudaFree(q);
    c->pstates.clear();
    c->pstate_doubles = (size_t)SZ;
  }
  size_t next_state = 0;
  auto alloc = [&](double** p) -> pif_status {
    if (next_state == c->pstates.size()) {
      double* q = nullptr;
      CU(cudaMalloc(&q, SZ * sizeof(double)));
      c->pstates.push_back(q);
    }
    *p = c->pstates[next_state++];
    CU(cudaMemsetAsync(*p, 0, SZ * sizeof(double), c->st));
    return PIF_OK;
  };
  auto timed = [&](double& acc, auto fn) -> pif_status {
    TRY(sync_stream(c, c->st));
    double a = now();
    pif_status s = fn();
    if (s != PIF_OK) return s;
    TRY(sync_stream(c, c->st));
    acc += now() - a;
    return PIF_OK;
  };
  // propagate canonical state src -> canonical dst with plan `which`
  auto propagate = [&](int which, const double* src, double* dst) -> pif_status {
    TRY(load_state(c, src));
    TRY(step_internal(c, which, which == 0 ? nf : ng));
    TRY(store_state(c, dst));
    return PIF_OK;
  };
  // correction + norms; errors (e_x, e_v) summed over the space group
  auto correct = [&](const double* F, const double* Gn, const double* Go, double* U, double& ex,
                     double& ev) -> pif_status {
    CU(launch_correct_norms(F, Gn, Go, U, n, L, c->partials, c->red, c->st));
    if (c->space_size > 1) NC(ncclAllReduce(c->red, c->red, 4, ncclDouble, ncclSum, c->comm_space, c->st));
    CU(cudaMemcpyAsync(c->host_red, c->red, 4 * sizeof(double), cudaMemcpyDeviceToHost, c->st));
    TRY(sync_stream(c, c->st));
    const double* r = c->host_red;
    ex = r[1] > 0 ? std::sqrt(r[0] / r[1]) : std::sqrt(r[0]);
    ev = r[3] > 0 ? std::sqrt(r[2] / r[3]) : std::sqrt(r[2]);
    if (!std::isfinite(ex) || !std::isfinite(ev))
      return fail(PIF_ERR_NUMERIC, "non-finite parareal state (stopping norms)");
    return PIF_OK;
  };

  pif_status st = PIF_OK;
  int iterations = 0;
  if (c->time_size == 1) {
    // ---------------- reference schedule: all slices on this rank ----------
    std::vector<double*> U(n_slices + 1), Gold(n_slices);
    double *Fcur, *Fnext, *Gnew;
    for (auto& p : U) if ((st = alloc(&p)) != PIF_OK) return st;
    for (auto& p : Gold) if ((st = alloc(&p)) != PIF_OK) return st;
    if ((st = alloc(&Fcur)) || (st = alloc(&Fnext)) || (st = alloc(&Gnew))) return st;
    std::vector<char> changed(n_slices, 1), retired(n_slices, 0);
    st = store_state(c, U[0]);
    // iteration 0: serial coarse sweep
    for (int s = 0; s < n_slices && st == PIF_OK; ++s) {
      st = timed(t_coarse0, [&] { return propagate(1, U[s], Gold[s]); });
      changed[s] = 0;
      if (st == PIF_OK) {
        cudaError_t e = cudaMemcpyAsync(U[s + 1], Gold[s], SZ * sizeof(double), cudaMemcpyDeviceToDevice, c->st);
        if (e != cudaSuccess) st = fail(PIF_ERR_CUDA, cudaGetErrorString(e));
        if (s + 1 < n_slices) changed[s + 1] = 1;
      }
    }
    for (int k = 0; k < max_iter && st == PIF_OK; ++k) {
      int r0 = 0;
      while (r0 < n_slices && retired[r0]) ++r0;
      if (r0 == n_slices) break;
      iterations = k + 1;
      st = timed(t_fine, [&] { return propagate(0, U[r0], Fcur); });
      for (int s = r0; s < n_slices && st == PIF_OK; ++s) {
        if (s + 1 < n_slices) st = timed(t_fine, [&] { return propagate(0, U[s + 1], Fnext); });
        if (st != PIF_OK) break;
        double* Gn = Gold[s];
        if (changed[s]) {
          st = timed(t_coarse, [&] { return propagate(1, U[s], Gnew); });
          if (st != PIF_OK) break;
          Gn = Gnew;
        }
        double ex = 0, ev = 0;
        st = correct(Fcur, Gn, Gold[s], U[s + 1], ex, ev);
        if (st != PIF_OK) break;
        if (s + 1 < n_slices) changed[s + 1] = 1;
        changed[s] = 0;
        if (Gn == Gnew) std::swap(Gold[s], Gnew);
        rep->err_x[k * n_slices + s] = ex;
        rep->err_v[k * n_slices + s] = ev;
        if (ex <= stop_tol && ev <= stop_tol && (s == 0 || retired[s - 1])) {
          retired[s] = 1;
          rep->retired_at[s] = k + 1;
        }
        std::swap(Fcur, Fnext);
      }
    }
    if (st == PIF_OK) st = load_state(c, U[n_slices]);
    int conv = 1;
    for (int s = 0; s < n_slices; ++s) conv &= retired[s];
    rep->converged = conv;
  } else {
    // ---------------- pipelined: slice t_idx on this time rank -------------
    // The protocol (protocol.cu) is host logic; the operations below bind its
    // buffer ids to device states and NCCL.
    const int t = c->t_idx, T = c->time_size;
    double* buf[5];
    for (auto& p : buf)
      if ((st = alloc(&p)) != PIF_OK) return st;
    struct GpuOps {
      pif_ctx c;
      double** buf;
      int t;
      int64_t n, SZ;
      double *t_fine, *t_coarse, *t_comm, *t_coarse0;
      bool first_coarse;
      std::function<pif_status(int, const double*, double*)> propagate;
      std::function<pif_status(const double*, const double*, const double*, double*, double&, double&)> correct;
      std::function<pif_status(double&, std::function<pif_status()>)> timed;
    };
    GpuOps G{c, buf, t, n, SZ, &t_fine, &t_coarse, &t_comm, &t_coarse0, true, propagate, correct,
             [&](double& acc, std::function<pif_status()> fn) { return timed(acc, fn); }};
    CU(cudaEventRecord(c->ev_sent, c->st));
    ProtocolOps ops;
    ops.user = &G;
    ops.store_initial = [](void* u, int dst) -> pif_status {
      auto* g = static_cast<GpuOps*>(u);
      return store_state(g->c, g->buf[dst]);
    };
    ops.propagate = [](void* u, int which, int src, int dst) -> pif_status {
      auto* g = static_cast<GpuOps*>(u);
      double& acc = which == 0 ? *g->t_fine : (g->first_coarse ? *g->t_coarse0 : *g->t_coarse);
      if (which == 1) g->first_coarse = false;
      return g->timed(acc, [&] { return g->propagate(which, g->buf[src], g->buf[dst]); });
    };
    ops.correct = [](void* u, int f, int gn, int go, int un, double* ex, double* ev) -> pif_status {
      auto* g = static_cast<GpuOps*>(u);
      return g->correct(g->buf[f], g->buf[gn], g->buf[go], g->buf[un], *ex, *ev);
    };
    // send on the comm stream, ordered after the producer on st; guard() makes
    // later writes into a sent buffer wait for ev_sent.
    ops.send = [](void* u, int b, double flag) -> pif_status {
      auto* g = static_cast<GpuOps*>(u);
      pif_ctx c = g->c;
      CU(cudaMemcpyAsync(g->buf[b] + 6 * g->n, &flag, sizeof(double), cudaMemcpyHostToDevice, c->st));
      CU(cudaEventRecord(c->ev_ready, c->st));
      CU(cudaStreamWaitEvent(c->st_comm, c->ev_ready, 0));
      NC(ncclSend(g->buf[b], g->SZ, ncclDouble, g->t + 1, c->comm_tp[g->t % 2], c->st_comm));
      CU(cudaEventRecord(c->ev_sent, c->st_comm));
      return PIF_OK;
    };
    ops.recv = [](void* u, int b, double* flag) -> pif_status {
      auto* g = static_cast<GpuOps*>(u);
      pif_ctx c = g->c;
      return g->timed(*g->t_comm, [&]() -> pif_status {
        NC(ncclRecv(g->buf[b], g->SZ, ncclDouble, g->t - 1, c->comm_tp[(g->t + 1) % 2], c->st));
        CU(cudaMemcpyAsync(&c->host_red[8], g->buf[b] + 6 * g->n, sizeof(double),
                           cudaMemcpyDeviceToHost, c->st));
        TRY(sync_stream(c, c->st));
        *flag = c->host_red[8];
        return PIF_OK;
      });
    };
    ops.guard = [](void* u) -> pif_status {
      auto* g = static_cast<GpuOps*>(u);
      CU(cudaStreamWaitEvent(g->c->st, g->c->ev_sent, 0));
      return PIF_OK;
    };
    ProtocolResult pr;
    st = run_pipeline(t, T, max_iter, stop_tol, ops, pr);
    iterations = pr.iterations;
    double* Unext = buf[pr.final_buf];
    std::vector<double>& myx = pr.ex;
    std::vector<double>& myv = pr.ev;
    int my_ret = pr.retired_at;
    if (c->st_comm) {
      pif_status s2 = sync_stream(c, c->st_comm);
      if (st == PIF_OK) st = s2;
    }
    if (st == PIF_OK) st = load_state(c, Unext);
    // gather the report over the time group (small)
    if (st == PIF_OK && max_iter > 0) {
      double* d = nullptr;
      const int64_t rowsz = 2 * (int64_t)max_iter + 2;
      CU(bufs.alloc(&d, rowsz * (T + 1) * sizeof(double)));
      std::vector<double> row(rowsz);
      for (int k = 0; k < max_iter; ++k) {
        row[k] = myx[k];
        row[max_iter + k] = myv[k];
      }
      row[2 * max_iter] = my_ret;
      row[2 * max_iter + 1] = iterations;
      CU(cudaMemcpyAsync(d, row.data(), rowsz * sizeof(double), cudaMemcpyHostToDevice, c->st));
      NC(ncclAllGather(d, d + rowsz, rowsz, ncclDouble, c->comm_time, c->st));
      std::vector<double> all(rowsz * T);
      CU(cudaMemcpyAsync(all.data(), d + rowsz, rowsz * T * sizeof(double), cudaMemcpyDeviceToHost, c->st));
      TRY(sync_stream(c, c->st));
      int conv = 1;
      iterations = 0;
      for (int s = 0; s < T; ++s) {
        const double* r = &all[s * rowsz];
        for (int k = 0; k < max_iter; ++k) {
          rep->err_x[k * n_slices + s] = r[k];
          rep->err_v[k * n_slices + s] = r[max_iter + k];
        }
        rep->retired_at[s] = (int)r[2 * max_iter];
        conv &= rep->retired_at[s] > 0;
        iterations = std::max(iterations, (int)r[2 * max_iter + 1]);
      }
      rep->converged = conv;
    }
  }
  if (st != PIF_OK) return st;
  rep->iterations = iterations;
  rep->t_coarse0 = t_coarse0;
  rep->t_fine = t_fine;
  rep->t_coarse = t_coarse;
  rep->t_comm = t_comm;
  rep->t_total = now() - tt0;
  return PIF_OK;
}

pif_status pif_parareal(pif_ctx c, double t0, double t1, int32_t n_slices, int32_t max_iter,
                        double stop_tol, int32_t n_blocks, pif_parareal_report* rep) {
  TRY(need_ready(c));
  if (!rep || !rep->retired_at || !rep->err_x || !rep->err_v) return fail(PIF_ERR_ARG, "null report");
  if (!c->plan[1].valid) return fail(PIF_ERR_CONFIG, "parareal needs a coarse propagator");
  if (n_slices < 1 || max_iter < 0 || !(t1 > t0) || n_blocks < 1)
    return fail(PIF_ERR_ARG, "bad slices / iterations / interval / blocks");
  if (c->time_size > 1 && n_slices != c->time_size)
    return fail(PIF_ERR_CONFIG, "n_slices must equal the number of time ranks");
  DeviceGuard dg(c->device);
  // Multi-block parareal (reading R22): n_blocks equal windows solved
  // one after the other, each by parareal with n_slices slices; the final state
  // of a window (on the last time rank) seeds the next window on every rank.
  const double W = (t1 - t0) / n_blocks;
  int total_iter = 0, all_conv = 1;
  double tf = 0, tg = 0, tg0 = 0, tc = 0, tt = 0;
  for (int b = 0; b < n_blocks; ++b) {
    TRY(parareal_window(c, t0 + b * W, (b + 1 == n_blocks) ? t1 : t0 + (b + 1) * W, n_slices,
                        max_iter, stop_tol, rep));
    total_iter += rep->iterations;
    all_conv &= rep->converged;
    tf += rep->t_fine;
    tg += rep->t_coarse;
    tg0 += rep->t_coarse0;
    tc += rep->t_comm;
    tt += rep->t_total;
    if (c->time_size > 1 && b + 1 < n_blocks) {
      // hand U_{n_slices} of this window from the last time rank to all time ranks
      double t0c = now();
      const int64_t n = c->nloc;
      // a parareal state buffer of the finished window (its final state is
      // already in the context) carries the hand-off
      double* buf = c->pstates.empty() ? nullptr : c->pstates[0];
      if (!buf) return fail(PIF_ERR_STATE, "no parareal state buffer for the window hand-off");
      if (c->t_idx == c->time_size - 1) TRY(store_state(c, buf));
      NC(ncclBroadcast(buf, buf, 6 * n, ncclDouble, c->time_size - 1, c->comm_time, c->st));
      TRY(load_state(c, buf));
      TRY(sync_stream(c, c->st));
      tc += now() - t0c;
      tt += now() - t0c;
    }
  }
  rep->iterations = total_iter;  // summed over windows; per-slice fields are the last window's
  rep->converged = all_conv;
  rep->t_fine = tf;
  rep->t_coarse = tg;
  rep->t_coarse0 = tg0;
  rep->t_comm = tc;
  rep->t_total = tt;
  return PIF_OK;
}

pif_status pif_comm_info(pif_ctx c, int32_t* world_nranks, int32_t* space_nranks,
                        int32_t* time_nranks) {
  if (!c || !world_nranks || !space_nranks || !time_nranks) return fail(PIF_ERR_ARG, "null argument");
  *world_nranks = *space_nranks = *time_nranks = 1;
  if (c->world == 1) return PIF_OK;
  if (c->nccl_broken) return fail(PIF_ERR_NCCL, "communicators were aborted by an earlier NCCL failure");
  int a = 0, b = 0, d = 0;
  NC(ncclCommCount(c->comm_world, &a));
  NC(ncclCommCount(c->comm_space, &b));
  NC(ncclCommCount(c->comm_time, &d));
  *world_nranks = a;
  *space_nranks = b;
  *time_nranks = d;
  return PIF_OK;
}

pif_status pif_profile(pif_ctx c, int enable) {
  if (!c) return fail(PIF_ERR_ARG, "null context");
  c->prof = enable != 0;
  return PIF_OK;
}

pif_status pif_profile_read(pif_ctx c, double* phase_ms, int32_t n_phases, int64_t* launches,
                            int reset) {
  if (!c || !phase_ms || !launches || n_phases < PIF_NPHASES)
    return fail(PIF_ERR_ARG, "need phase_ms[PIF_NPHASES] and launches");
  DeviceGuard dg(c->device);
  TRY(sync_stream(c, c->st));
  for (int ph = 0; ph < PIF_NPHASES; ++ph) {
    double acc = 0;
    for (size_t i = 0; i + 1 < c->ev_used[ph]; i += 2) {
      float ms = 0;
      CU(cudaEventElapsedTime(&ms, c->ev[ph][i], c->ev[ph][i + 1]));
      acc += ms;
    }
    phase_ms[ph] = acc;
    if (reset) c->ev_used[ph] = 0;
  }
  for (int ph = PIF_NPHASES; ph < n_phases; ++ph) phase_ms[ph] = 0;
  *launches = c->launches;
  if (reset) c->launches = 0;
  return PIF_OK;
}

pif_status pif_finalize(pif_ctx c) {
  if (!c) return PIF_OK;
  DeviceGuard dg(c->device);
  for (int ph = 0; ph < PIF_NPHASES; ++ph)
    for (cudaEvent_t e : c->ev[ph]) cudaEventDestroy(e);
  for (int i = 0; i < 2; ++i) {
    if (c->plan[i].fwd) cufftDestroy(c->plan[i].fwd);
    if (c->plan[i].inv) cufftDestroy(c->plan[i].inv);
  }
  for (int i = 0; i < 2; ++i)
    if (c->comm_tp[i]) ncclCommDestroy(c->comm_tp[i]);
  if (c->ev_ready) cudaEventDestroy(c->ev_ready);
  if (c->ev_sent) cudaEventDestroy(c->ev_sent);
  if (c->st_comm) cudaStreamDestroy(c->st_comm);
  if (c->comm_space) ncclCommDestroy(c->comm_space);
  if (c->comm_time) ncclCommDestroy(c->comm_time);
  if (c->comm_world) ncclCommDestroy(c->comm_world);
  if (c->host_red) cudaFreeHost(c->host_red);
  for (double* q : c->pstates) cudaFree(q);
  delete c;
  return PIF_OK;
}

// ------------------------------------------------------------- debug/tests --
// Device buffers of a debug transform on n particles: positions (and
// strengths) in caller order, their sorted copies, and the sort / schedule
// arrays of plan p -- the production bin, schedule and gather sort.
struct DebugSort {
  double *x = nullptr, *x2 = nullptr, *s = nullptr, *s2 = nullptr;
  int *id = nullptr, *id2 = nullptr, *key = nullptr, *rk = nullptr, *perm = nullptr, *counts = nullptr;
  Sched S{};
};
static pif_status debug_sort(pif_ctx c, const Plan& p, DevBufs& B, const double* x, const double* s,
                             int64_t n, DebugSort& D) {
  const int64_t K = p.nbricks, M = keys_per_brick(p.g);
  const int64_t ms = sched_max_s(K, M, n), mi = sched_max_i(K, n);
  CU(B.alloc(&D.x, 3 * n * sizeof(double)));
  CU(B.alloc(&D.x2, 3 * n * sizeof(double)));
  if (s) {
    CU(B.alloc(&D.s, n * sizeof(double)));
    CU(B.alloc(&D.s2, n * sizeof(double)));
  }
  CU(B.alloc(&D.id, 5 * n * sizeof(int)));
  D.id2 = D.id + n;
  D.key = D.id + 2 * n;
  D.rk = D.id + 3 * n;
  D.perm = D.id + 4 * n;
  int* ib = nullptr;
  const size_t ints = K + 5 * (K + 1) + sched_part_ints(K) + 16;
  CU(B.alloc(&ib, ints * sizeof(int)));
  int4* items = nullptr;
  CU(B.alloc(&items, (ms + 2 * mi) * sizeof(int4)));
  D.counts = ib;
  D.S = Sched{ib + K, ib + 2 * K + 1, ib + 3 * K + 2, ib + 4 * K + 3, items, items + ms, items + ms + mi,
              ib + 5 * K + 5, K, ms, mi, ib + ints - 16};
  CU(cudaMemcpyAsync(D.x, x, 3 * n * sizeof(double), cudaMemcpyHostToDevice, c->st));
  if (s) CU(cudaMemcpyAsync(D.s, s, n * sizeof(double), cudaMemcpyHostToDevice, c->st));
  CU(launch_iota(D.id, n, c->st));
  CU(cudaMemsetAsync(D.counts, 0, K * sizeof(int), c->st));
  CU(launch_bin_count(D.x, n, n, p.g, D.key, D.rk, D.counts, c->st));
  CU(launch_schedule(D.counts, D.S, p.g, (int)M, p.g.C, c->st));
  CU(launch_gather_sorted(D.x, nullptr, D.id, D.s, n, n, D.key, D.rk, D.S.offsets, D.perm, D.x2,
                          nullptr, D.id2, D.s2, c->st));
  return PIF_OK;
}

static pif_status debug_args(pif_ctx c, int which, int64_t n) {
  if (!c || n < 1) return fail(PIF_ERR_ARG, "null argument / empty input");
  if (!c->ws) return fail(PIF_ERR_STATE, "workspace not set");
  if (which < 0 || which > 1 || !c->plan[which].valid || c->plan[which].kind != PIF_PROP_PIF_NUFFT)
    return fail(PIF_ERR_ARG, "not a PIF propagator");
  return PIF_OK;
}

pif_status pif_debug_type1(pif_ctx c, int which, const double* x, int64_t n, const double* s,
                           double* out) {
  TRY(debug_args(c, which, n));
  if (!x || !s || !out) return fail(PIF_ERR_ARG, "null argument");
  DeviceGuard dg(c->device);
  Plan& p = c->plan[which];
  const int64_t N3 = (int64_t)p.N * p.N * p.N;
  DevBufs B(c->st);
  DebugSort D;
  TRY(debug_sort(c, p, B, x, s, n, D));
  double2* dout = nullptr;
  CU(B.alloc(&dout, N3 * sizeof(double2)));
  CU(cudaMemsetAsync(p.grid, 0, p.grid_pts() * sizeof(double), c->st));
  CU(launch_spread(D.x2, nullptr, n, D.s2, 1.0, D.S, p.g, p.hc, p.fp32 ? &p.hcf : nullptr, p.grid, c->st));
  CUFFT(cufftExecD2Z(p.fwd, p.grid, (cufftDoubleComplex*)p.spec));
  CU(launch_debug_extract_KN(p.spec, p.n, p.N, p.cor, dout, c->st));
  CU(cudaMemcpyAsync(out, dout, N3 * sizeof(double2), cudaMemcpyDeviceToHost, c->st));
  TRY(sync_stream(c, c->st));
  return PIF_OK;
}

pif_status pif_debug_type2(pif_ctx c, int which, const double* cin, const double* x, int64_t n,
                           double* out) {
  TRY(debug_args(c, which, n));
  if (!x || !cin || !out) return fail(PIF_ERR_ARG, "null argument");
  DeviceGuard dg(c->device);
  Plan& p = c->plan[which];
  const int64_t N3 = (int64_t)p.N * p.N * p.N;
  DevBufs B(c->st);
  DebugSort D;
  TRY(debug_sort(c, p, B, x, nullptr, n, D));
  double *E = nullptr;
  double2* dc = nullptr;
  CU(B.alloc(&E, 3 * n * sizeof(double)));
  CU(B.alloc(&dc, N3 * sizeof(double2)));
  CU(cudaMemcpyAsync(dc, cin, N3 * sizeof(double2), cudaMemcpyHostToDevice, c->st));
  CU(launch_debug_pad_KN(dc, p.n, p.N, p.cor, p.G3, p.fp32, c->st));
  CUFFT(inverse_fft(p));
  PushArgs P = push_args(c, p, 0, 0);
  CU(interp_push(c, p, D.x2, nullptr, n, D.id2, E, D.S, P));
  CU(cudaMemcpyAsync(out, E, n * sizeof(double), cudaMemcpyDeviceToHost, c->st));
  TRY(sync_stream(c, c->st));
  return PIF_OK;
}

pif_status pif_debug_push(pif_ctx c, int which, double* x, double* v, const double* E, int64_t n,
                          int kicks, int drift) {
  if (!c || !x || !v || !E || n < 1) return fail(PIF_ERR_ARG, "null argument");
  if (which < 0 || which > 1 || !c->plan[which].valid) return fail(PIF_ERR_ARG, "no such propagator");
  if (kicks < 0 || kicks > 2) return fail(PIF_ERR_ARG, "kicks must be 0, 1 or 2");
  DeviceGuard dg(c->device);
  DevBufs B(c->st);
  double* d = nullptr;
  CU(B.alloc(&d, 9 * n * sizeof(double)));
  CU(cudaMemcpyAsync(d, x, 3 * n * sizeof(double), cudaMemcpyHostToDevice, c->st));
  CU(cudaMemcpyAsync(d + 3 * n, v, 3 * n * sizeof(double), cudaMemcpyHostToDevice, c->st));
  CU(cudaMemcpyAsync(d + 6 * n, E, 3 * n * sizeof(double), cudaMemcpyHostToDevice, c->st));
  PushArgs P = push_args(c, c->plan[which], kicks, drift);
  CU(launch_push_only(d, d + 3 * n, d + 6 * n, n, n, P, c->st));
  CU(cudaMemcpyAsync(x, d, 3 * n * sizeof(double), cudaMemcpyDeviceToHost, c->st));
  CU(cudaMemcpyAsync(v, d + 3 * n, 3 * n * sizeof(double), cudaMemcpyDeviceToHost, c->st));
  TRY(sync_stream(c, c->st));
  return PIF_OK;
}

}  // extern "C"
