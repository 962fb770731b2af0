/*
 * pif.h -- C ABI of the B200-native Particle-in-Fourier (PIF) step and its
 * parareal driver (arXiv 2407.00485).
 *
 * Citations: P:n = /root/reference/PAPER.md line n (section/equation named).
 *
 * The library computes, per timestep of a PIF propagator (Sec. "Particle-in-
 * Fourier method"):
 *   type-1 NUFFT   rho_k = (q S_k / L^3) sum_j exp(-i k.x_j)     eq. scatter_pif
 *   Poisson        E_k   = -i k rho_k / |k|^2, rho_0 := 0
 *   type-2 NUFFT   E(x_j) = Re sum_{k in K_N} E_k S_k exp(i k.x_j) eq. gather_pif
 *   push           KDK velocity Verlet / Boris
 * with K_N = (2 pi / L) {-N/2 .. N/2-1}^3 (reading R1 of DESIGN.md), and the
 * CIC particle-in-cell propagator of Sec. "Particle-in-cell method"
 * as the alternative coarse propagator; pif_parareal runs the
 * parareal iteration of eq. parareal_correction with the stopping
 * rule of eq. stop_criteria and the local exit of P:692-693.
 *
 * Units: q_e = -1, m_e = 1, eps0 = 1.  N_p equal macro-particles with
 * charge q = Q_e / N_p_global and mass m = |Q_e| / N_p_global (reading R6).
 *
 * Layouts: particle arrays are SoA float64, x[3][n] then v[3][n] (x[d*n+j]).
 * Positions live in [0, L)^3.  Spectra for the debug exports are interleaved
 * complex float64 (re, im), row-major over (mx, my, mz), each from -N/2 to
 * N/2-1.
 *
 * Ownership: every pointer passed in is BORROWED -- the library never frees it.
 * Device memory used by pif_step is one caller-allocated workspace
 * (pif_workspace_size / pif_set_workspace; the Python binding allocates it as
 * a torch uint8 tensor).  Outside it: pif_parareal's states -- (2 n_slices +
 * 4) states of (6 n_local + 1) doubles with time_size == 1, 5 states per time
 * rank otherwise -- are allocated (cudaMalloc) by the first call, reused by
 * later calls with the same n_local and freed by pif_finalize; the debug
 * exports allocate their input / sort buffers stream-ordered (cudaMallocAsync)
 * and release them before returning, on every exit path.  The
 * context handle is library-owned (pif_finalize releases it).  Every call runs
 * on the context's device (pif_dist.device) and restores the caller's current
 * device before returning.
 *
 * Streams: all device work is ordered on pif_dist.stream (a cudaStream_t,
 * NULL = legacy default stream).  pif_step is asynchronous; pif_set_state /
 * pif_get_state with host pointers, pif_field_energy, pif_parareal and the
 * debug exports synchronise the stream before returning.
 *
 * Errors: every call returns pif_status.  On error the message is available
 * from pif_last_error() (thread-local, valid until the next call on the same
 * thread) and the context is left as it was before the call, except for
 * PIF_ERR_CUDA / PIF_ERR_NCCL after which the context must be finalised.
 */
#ifndef PIF_H_
#define PIF_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pif_ctx_s* pif_ctx;

typedef enum {
  PIF_OK = 0,
  PIF_ERR_ARG = 1,     /* null pointer, size mismatch, N odd or < 2, tol out of [1e-15,1e-1), dt <= 0, L <= 0 */
  PIF_ERR_CONFIG = 2,  /* inconsistent configuration (see each call) */
  PIF_ERR_NUMERIC = 3, /* non-finite value detected: checked by pif_set_state (input),
                          pif_get_state, pif_field_energy and each parareal correction */
  PIF_ERR_CUDA = 4,    /* CUDA runtime / cuFFT error (message has the code) */
  PIF_ERR_NCCL = 5,    /* NCCL error, asynchronous NCCL error, or the watchdog: a synchronising
                          call saw no progress for PIF_NCCL_TIMEOUT_S seconds (environment,
                          default 600; a lost peer).  The communicators are then aborted and
                          the context only accepts pif_finalize. */
  PIF_ERR_OOM = 6,     /* workspace too small */
  PIF_ERR_STATE = 7    /* call out of order (e.g. step before set_state / set_workspace) */
} pif_status;

typedef enum { PIF_PROP_PIF_NUFFT = 0, PIF_PROP_PIC_CIC = 1 } pif_prop_kind;
#define PIF_FLAG_FP32_ALLREDUCE 1
#define PIF_FLAG_FP32 2

/* One propagator (fine F or coarse G of Sec. "Parareal for PIF"). */
typedef struct {
  int32_t kind;         /* pif_prop_kind */
  int32_t n;            /* PIF: Fourier modes per dimension N (even, >= 2, <= 256);
                           PIC: grid points per dimension N_g (even, >= 4, <= 512) */
  int32_t spline_order; /* B-spline order m >= 1 of the shape function: S_k = prod_d
                           sinc^(m+1)(k_d h / 2), h = L / n.
                           PIC supports m = 1 (CIC) only. */
  int32_t flags;        /* bit 0 PIF_FLAG_FP32_ALLREDUCE: all-reduce the density (PIF rho_hat
                           box / PIC grid) over the space group in fp32 instead of fp64 --
                           halves the communication, the "single precision for the density
                           field" of P:553-554 (meant for coarse propagators).
                           bit 1 PIF_FLAG_FP32: single-precision coarse propagator (P:553-554,
                           "future work"): the inverse FFT (C2R) and the type-2 interpolation
                           (grid tile, kernel weights, accumulation) run in fp32 on the vector
                           pipe; the spread accumulates in fp64 (DMMA) with its kernel weights
                           evaluated in fp32 on the dense tiles; positions, velocities, the
                           push, the forward FFT and the Poisson solve stay fp64.  PIF kind
                           only, tol >= 1e-5 (w <= 6; fp32 rounding ~1e-7 stays far inside
                           10 eps), else PIF_ERR_ARG.  0 = default. */
  double tol;           /* PIF: NUFFT tolerance eps in [1e-15, 1e-1); ignored for PIC */
  double dt;            /* timestep > 0 */
} pif_propagator;

/* Physical problem (eq. Vlasov). */
typedef struct {
  double L;            /* side of the periodic cube [0, L)^3, > 0 */
  double q_over_m;     /* q_e / m_e (-1 in normalised units) */
  double total_charge; /* Q_e != 0 */
  double B_ext[3];     /* constant magnetic field */
  double E_ext_A[9];   /* E_ext(x) = A x + c, A row-major (eq. penning_ext_efield) */
  double E_ext_c[3];
} pif_physics;

/* Process layout.  world = space_size * time_size ranks, rank = t * space_size + s:
   space rank s owns particle block s (particle decomposition, rho_k
   allreduce over the space group); time rank t owns parareal slice t. */
typedef struct {
  int32_t device;      /* CUDA device ordinal */
  int32_t rank, world; /* 0 <= rank < world */
  int32_t space_size;  /* divides world */
  const void* nccl_id; /* 128-byte ncclUniqueId identical on all ranks; NULL iff world == 1 */
  void* stream;        /* cudaStream_t */
} pif_dist;

/* Create a context.  fine must be PIF or PIC; coarse may be NULL (no parareal).
   n_particles_global = N_p over all space ranks; n_local of this rank is
   pif_local_count().  Returns PIF_ERR_ARG / PIF_ERR_CONFIG on bad input. */
pif_status pif_init(const pif_physics* phys, const pif_propagator* fine,
                    const pif_propagator* coarse, int64_t n_particles_global,
                    const pif_dist* dist, pif_ctx* out);

/* Particles owned by this rank: contiguous block [first, first + count) of the
   global index range (space rank s gets N_p/space_size, the first N_p%space_size
   ranks one more). */
pif_status pif_local_count(pif_ctx ctx, int64_t* first, int64_t* count);

/* Host-only partition rule used by pif_init (no CUDA): space rank s of
   space_size owns [first, first + count) of n_global particles. */
pif_status pif_partition(int64_t n_global, int32_t space_size, int32_t s_idx, int64_t* first,
                         int64_t* count);

/* Device workspace: bytes needed (256-byte aligned base required), then hand
   over a caller-owned device buffer that outlives the context's use. */
pif_status pif_workspace_size(pif_ctx ctx, size_t* bytes);
pif_status pif_set_workspace(pif_ctx ctx, void* dptr, size_t bytes);

/* Copy the local state in ([3][n_local] SoA each).  on_device = 1: CUDA
   pointers; 0: host pointers (pinned or pageable).  Positions outside the
   periodic box are wrapped into [0, L)^3 (x - L floor(x / L)), so any finite
   input is legal.  Resets the time level.  Synchronises; PIF_ERR_NUMERIC (and
   no state) if any value is non-finite. */
pif_status pif_set_state(pif_ctx ctx, const double* x, const double* v, int64_t n_local,
                         int on_device);
/* Copy the local state out at an integer time level, in the ORIGINAL particle
   order of pif_set_state (completes a pending half kick, see pif_step). */
pif_status pif_get_state(pif_ctx ctx, double* x, double* v, int64_t n_local, int on_device);

/* Advance n_steps >= 0 steps of propagator `which` (0 = fine, 1 = coarse) by
   Strang KDK: v <- K(dt/2, E(x)); x <- wrap(x + dt v); v <- K(dt/2, E(x)).
   One field solve per step: the closing half kick of a step and the opening
   half kick of the next share E(x_{n+1}); the last closing kick is applied
   lazily (by pif_get_state, pif_field_energy, a switch of propagator, or the
   next pif_step).  Asynchronous on the stream. */
pif_status pif_step(pif_ctx ctx, int which, int64_t n_steps);

/* Diagnostics at the current integer time level of the fine propagator
   (P:607): W[d] = (L^3/2) sum_{k in K_N} |E_{d,k}|^2, kinetic =
   sum m|v|^2/2, momentum = sum m v, charge_err = |L^3 rho_0 - Q_e| / |Q_e|
   (rho_0 before background removal).  PIC fine: W from the grid spectrum,
   charge_err = 0.  Synchronises; reduces over the space group. */
pif_status pif_field_energy(pif_ctx ctx, double W[3], double* kinetic, double momentum[3],
                            double* charge_err);

/* Density spectrum at the current integer time level (fine PIF propagator):
   rho_tilde_k = (q / L^3) sum_j exp(-i k.x_j) (eq. scatter_pif without S_k, before
   background removal, summed over the space group) on the Hermitian half box
   mx, my in [-N/2, N/2], mz in [0, N/2]: out[2*(((mx+N/2)*(N+1) + my+N/2)*(N/2+1) + mz)]
   = (re, im); host pointer of 2 (N+1)^2 (N/2+1) doubles.  Synchronises. */
pif_status pif_get_rho(pif_ctx ctx, double* out);

/* Parareal report; arrays are caller-allocated. */
typedef struct {
  int32_t iterations;  /* correction iterations run (>= 1 when max_iter >= 1) */
  int32_t converged;   /* 1 if every slice retired */
  int32_t* retired_at; /* [n_slices]: 1-based iteration after which slice n retired, -1 if never */
  double* err_x;       /* [max_iter * n_slices]: e_x of eq. stop_criteria, NaN if frozen */
  double* err_v;       /* [max_iter * n_slices] */
  double t_coarse0, t_fine, t_coarse, t_comm, t_total; /* seconds on this rank */
} pif_parareal_report;

/* Parareal over [t0, t1] with n_slices time slices, starting from the current
   state, ending with the state U_{n_slices} at t1 (on every time rank the
   context holds the U_{t+1} of its own slice; the final state is on the last
   time rank).  F = fine propagator, G = coarse, dT = (t1-t0)/n_slices must be an
   integer multiple of both dt's (relative tolerance 1e-9) -> PIF_ERR_CONFIG.
   Stopping: slice n retires after the first iteration with e_x, e_v <= stop_tol
   and slice n-1 retired; retired slices are frozen.
   time_size == 1: all slices run serially on this rank (reference schedule);
   time_size > 1: n_slices must equal time_size (one slice per time rank,
   states passed by NCCL send/recv).  n_blocks >= 1: multi-block parareal
   (reading R22) -- [t0, t1] is cut into n_blocks equal windows
   solved one after the other, each by parareal with n_slices slices, the final
   state of a window seeding the next (broadcast from the last time rank).  The
   report then holds the total iterations over windows, converged = all windows
   converged, summed timings, and retired_at / err_x / err_v of the last window.
   Synchronises. */
pif_status pif_parareal(pif_ctx ctx, double t0, double t1, int32_t n_slices, int32_t max_iter,
                        double stop_tol, int32_t n_blocks, pif_parareal_report* report);

pif_status pif_finalize(pif_ctx ctx);
const char* pif_last_error(void);

/* NCCL unique id (128 bytes) for rank 0 to broadcast before pif_init. */
pif_status pif_nccl_unique_id(void* out128);

/* Plan parameters chosen for a propagator (NUFFT: kernel width w, ES shape
   beta, upsampled grid n). */
pif_status pif_plan_info(pif_ctx ctx, int which, int32_t* w, double* beta, int32_t* n_up);

/* Communicator sizes as NCCL reports them (ncclCommCount): world, space group
   (rho_hat all-reduce) and time group (parareal hand-off); 1, 1, 1 when
   world == 1.  Host-only query. */
pif_status pif_comm_info(pif_ctx ctx, int32_t* world_nranks, int32_t* space_nranks,
                         int32_t* time_nranks);

/* Phase profiling (tracing).  While enabled, every phase of a step is bracketed
   by CUDA events on the stream (no synchronisation).  pif_profile_read
   synchronises, returns the summed device time in ms per phase since the last
   reset -- phase_ms[PIF_NPHASES] in the order sort, spread, fft_fwd, box
   (deconvolve/truncate), allreduce, poisson (+pad), fft_inv, interp_push,
   pic_deposit, pic_gather_push, other -- and the number of the library's own
   kernels launched (cuFFT / NCCL kernels not counted).  In a step that pushes,
   "sort" is the bin count, schedule and permutation only: the reorder itself
   happens inside the spread (permuted reads) and interp_push (permuted reads,
   sorted writes).  reset != 0 clears both. */
#define PIF_NPHASES 11
pif_status pif_profile(pif_ctx ctx, int enable);
pif_status pif_profile_read(pif_ctx ctx, double* phase_ms, int32_t n_phases, int64_t* launches,
                            int reset);

/* ---- test-only exports: host pointers, synchronous, use `which`'s NUFFT plan.
   type1: out_k = sum_j s_j exp(-i k.x_j) for k in K_N (no 1/L^3, no S_k).
   type2: out_j = Re sum_{k in K_N} c_k exp(+i k.x_j) for arbitrary complex c_k
          on K_N, through the same Hermitian completion and C2R path as the
          step (reading R2).  x: [3][n] in [0, L). out/c: 2*N^3 doubles. */
pif_status pif_debug_type1(pif_ctx ctx, int which, const double* x, int64_t n, const double* s,
                           double* out);
pif_status pif_debug_type2(pif_ctx ctx, int which, const double* c, const double* x, int64_t n,
                           double* out);

/* Test-only: one push with a given field (no field solve): for each particle,
   E_tot = E[:,j] + E_ext(x_j); v <- K(dt/2,E_tot) applied `kicks` (1 or 2) times;
   if drift: x <- wrap(x + dt v).  Host pointers, in place. */
pif_status pif_debug_push(pif_ctx ctx, int which, double* x, double* v, const double* E, int64_t n,
                          int kicks, int drift);

/* Test-only: run the pipelined parareal protocol of time slice t of T (the
   host logic of pif_parareal with time_size > 1: iteration-0 coarse sweep,
   F / receive / G / correction / send per iteration, retirement when the
   slice's e_x, e_v <= tol and its predecessor retired, frozen inputs once the
   predecessor retired) over caller-supplied operations on buffer ids
   0 = U_t, 1 = F(U_t), 2 = G_old, 3 = G_new, 4 = U_{t+1}.  Callbacks return 0
   on success.  Outputs: iterations run, retired_at (1-based, -1 never),
   err_x/err_v[max_iter] (NaN where not run), final_buf = id holding U_{t+1}. */
typedef struct {
  void* user;
  int (*store_initial)(void* user, int dst);
  int (*propagate)(void* user, int which, int src, int dst);
  int (*correct)(void* user, int f, int gn, int go, int u, double* ex, double* ev);
  int (*send)(void* user, int buf, double flag);
  int (*recv)(void* user, int buf, double* flag);
} pif_protocol_ops;
pif_status pif_debug_parareal_protocol(int32_t t, int32_t T, int32_t max_iter, double tol,
                                       const pif_protocol_ops* ops, int32_t* iterations,
                                       int32_t* retired_at, double* err_x, double* err_v,
                                       int32_t* final_buf);

#ifdef __cplusplus
}
#endif
#endif /* PIF_H_ */
