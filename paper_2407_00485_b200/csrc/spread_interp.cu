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
#include <type_traits>

#include "pif_internal.cuh"

namespace pif {


#ifndef PIF_SPREAD_MINB
#define PIF_SPREAD_MINB 3  // 3 CTAs/SM (shared memory allows 3 for the 16^3 tile)
#endif
#ifndef PIF_CHUNK
#define PIF_CHUNK 128
#endif
constexpr int kChunk = PIF_CHUNK;    // spread: particles staged per shared-memory round

#ifdef PIF_DMMA_NONVOLATILE
#define PIF_DMMA_ASM asm
#else
#define PIF_DMMA_ASM asm volatile
#endif
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  PIF_DMMA_ASM("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ int wrapi(int i, int n) { return ((i % n) + n) % n; }

// 8-byte asynchronous global -> shared copy (LDGSTS; no register staging).
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
// 8-byte cp.async that writes zeros (reads nothing) when !valid.
__device__ __forceinline__ void cp_async8_zfill(void* smem, const void* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(sa), "l"(gmem), "r"(valid ? 8 : 0)
               : "memory");
}

// Bulk asynchronous reduction shared -> global (TMA, .add.f64), `cnt` doubles;
// addresses 16-byte aligned, cnt even.  Completion: cp.async.bulk groups.
__device__ __forceinline__ void bulk_reduce_add_f64(double* gdst, const double* ssrc, int cnt) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(ssrc);
  asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;" ::"l"(gdst),
               "r"(sa), "r"(cnt * 8)
               : "memory");
}

// mbarrier (shared memory, CTA scope).
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, int count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
// arrive on b once every cp.async this thread issued so far has landed
__device__ __forceinline__ void cp_async_mbar_arrive(unsigned long long* b) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared.b64 [%0];" ::"r"(smem_u32(b)) : "memory");
}
// Wait for completion of the phase with the given parity.  Bounded: a protocol
// error traps (kernel error) after ~10 s instead of hanging the device.
__device__ __forceinline__ void mbar_wait(unsigned long long* b, int parity) {
  unsigned done = 0;
  long long t0 = 0;
  for (int spin = 0;; ++spin) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    if (done) return;
    // the clock is read once per 256 polls (a spinning warp shares its SMSP's
    // issue slots with the MMA warps)
    if ((spin & 255) == 0) {
      if (spin == 0) t0 = clock64();
      else if (clock64() - t0 > 20000000000LL) __trap();
    }
  }
}

// psi row strides (doubles): S == 4 or 12 (mod 16) so that the 4 particle rows
// read by one half-warp fragment load (4 consecutive doubles each) fall in
// disjoint banks.
template <int R>
struct RowStride {
  static constexpr int v = R <= 8 ? 12 : (R <= 16 ? 20 : ((R + 11) / 16) * 16 + 4);
};

// Column tiles of 8 of a spreading tile: ceil(RX RY / 8), or more (padded) when
// that gives more column tiles per warp (PIF_SPREAD_NCT13 for the 10x10 tile)
#ifndef PIF_SPREAD_NCT13
#define PIF_SPREAD_NCT13 13
#endif
__host__ __device__ constexpr int spread_nct(int RX, int RY) {
  return (RX * RY + 7) / 8 == 13 ? PIF_SPREAD_NCT13 : (RX * RY + 7) / 8;
}
// py entries past RY that padded columns c >= RX RY read (A = 0 there)
__host__ __device__ constexpr int spread_pad_rows(int RX, int RY) {
  return (spread_nct(RX, RY) * 8 + RX - 1) / RX - RY;
}

// Spread staging, node-major: px[node][particle] (py with the rows the padded
// columns read, pz zero-padded to a multiple of 8 nodes).  A staging warp's
// lanes write consecutive particles of one node (conflict-free; the earlier
// particle-major rows, stride 4 mod 16, put 4 lanes on every bank: 16 M / 356 M
// store conflicts at C2 / C5 fine), and the row stride S = CH + 4 (4 mod 16)
// keeps the A and B fragment reads (4 particles x 4 consecutive nodes per
// half-warp) on distinct banks.
template <int RX, int RY, int RZ, int CH = kChunk>
struct Psi {
  static constexpr int S = CH + 4;
  static constexpr int PY = RY + spread_pad_rows(RX, RY);
  static constexpr int ZP = (RZ + 7) / 8 * 8;
  double px[RX][S];
  double py[PY][S];
  double pz[ZP][S];
  double xs[CH][3];
  int rel[CH][3];
  double str[CH];
};

// Decode a work item: spread (sub == false) = {brick, start, end}; interpolation
// (sub == true) = {sub-brick key, start, end}; returns false past the last item.
__device__ __forceinline__ bool tile_of(const Brick& g, const Sched& S, bool sub, int64_t item,
                                        int T0[3], int64_t& start, int64_t& end) {
  const int4 it = sub ? S.iitems[item] : S.sitems[item];
  start = it.y;
  end = it.z;
  const int M = g.m[0] * g.m[1] * g.m[2];
  const int brick = sub ? it.x / M : it.x;
  int bz = brick % g.NB[2], by = (brick / g.NB[2]) % g.NB[1], bx = brick / (g.NB[2] * g.NB[1]);
  T0[0] = bx * g.sb[0] - g.hw;
  T0[1] = by * g.sb[1] - g.hw;
  T0[2] = bz * g.sb[2] - g.hw;
  if (sub) {
    int sk = it.x % M;
    int sz = sk % g.m[2], sy = (sk / g.m[2]) % g.m[1], sx = sk / (g.m[2] * g.m[1]);
    T0[0] += sx * g.ib[0];
    T0[1] += sy * g.ib[1];
    T0[2] += sz * g.ib[2];
  }
  return start < end;
}

// Thread tid < cnt: record particle tid's grid coordinate and window offset.
template <int RX, int RY, int RZ, int CH>
__device__ __forceinline__ void stage_position(Psi<RX, RY, RZ, CH>& sm, int tid, const double xr[3],
                                               const Brick& g, const int T0[3]) {
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    double xs = xr[d] * g.scale;
    int a = anchor_of(xs, g);
    sm.xs[tid][d] = xs;
    sm.rel[tid][d] = a - g.hw - T0[d];
  }
}

// One psi row: the w window weights of a particle at row[rel .. rel + w), by the per-node
// polynomials P_k(s) in s = 2 (f - flo) - 1, using the evenness of the ES kernel:
// with hw = (w - 1) / 2, node w-1-k at s equals node k at -s, so one split
// P_k(s) = E_k(s^2) + s O_k(s^2) gives both nodes of a pair (7 dependent steps,
// ~15 FMAs per pair instead of 14 steps and 30 FMAs); the centre node of an odd
// w is even in s (E only).  All pairs are evaluated in one pass: the FP64 pipe
// is shared with the DMMAs, so dependent steps, not FMAs, set the latency.
template <int NPAIR, bool CENTER, int ST = 1>
__device__ __forceinline__ void horner_sym(double* row, int rel, double f, double sv,
                                           const Horner& hc, const Brick& g, double two_over_w) {
  constexpr int w = 2 * NPAIR + 2 + (CENTER ? 1 : 0);
  // Edge nodes: their polynomial fit error is ~0.05 eps for w >= 5 (degree 14,
  // e.g. 5e-14 at w = 13, 4e-9 at w = 8, 3e-6 at w = 5), so they join the pairs;
  // small widths (w <= 4, fit error up to 0.25 eps) evaluate them exactly.
#ifdef PIF_EXACT_EDGES
  constexpr int P0 = 1;
#else
  constexpr int P0 = w <= 4 ? 1 : 0;
#endif
  if (P0) {
    row[rel * ST] = es_kernel((double)(-g.hw) - f, two_over_w, g.beta);
    row[(rel + w - 1) * ST] = es_kernel((double)(w - 1 - g.hw) - f, two_over_w, g.beta);
  }
  constexpr int NP = NPAIR + 1 - P0;         // polynomial pairs: nodes (P0 + i, w - 1 - P0 - i)
  constexpr int NE = NP + (CENTER ? 1 : 0);  // even parts (+ the centre node of an odd w)
  const double s2 = sv * sv;
  double e[NE + 1], o[NP + 1];  // (+1: may be empty)
#pragma unroll
  for (int i = 0; i < NE; ++i) e[i] = hc.a[P0 + i][kHornerDeg];
#pragma unroll
  for (int i = 0; i < NP; ++i) o[i] = hc.a[P0 + i][kHornerDeg - 1];
#pragma unroll
  for (int j = kHornerDeg / 2 - 1; j >= 0; --j) {
#pragma unroll
    for (int i = 0; i < NE; ++i) e[i] = fma(e[i], s2, hc.a[P0 + i][2 * j]);
    if (j < kHornerDeg / 2 - 1)
#pragma unroll
      for (int i = 0; i < NP; ++i) o[i] = fma(o[i], s2, hc.a[P0 + i][2 * j + 1]);
  }
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    row[(rel + P0 + i) * ST] = fma(sv, o[i], e[i]);
    row[(rel + w - 1 - P0 - i) * ST] = fma(-sv, o[i], e[i]);
  }
  if (CENTER) row[(rel + P0 + NP) * ST] = e[NP];
}

// The w weights at row[(rel + k) ST], k < w (ST: element stride of the row).
template <int ST = 1>
__device__ __forceinline__ void psi_row(double* row, int rel, double f, double sv,
                                        const Horner& hc, const Brick& g, double two_over_w) {
  switch (g.w) {  // uniform
#define PIF_W(W) \
  case W: horner_sym<(W - 2) / 2, (W & 1) == 1, ST>(row, rel, f, sv, hc, g, two_over_w); break;
    PIF_W(2) PIF_W(3) PIF_W(4) PIF_W(5) PIF_W(6) PIF_W(7) PIF_W(8) PIF_W(9)
    PIF_W(10) PIF_W(11) PIF_W(12) PIF_W(13) PIF_W(14) PIF_W(15) PIF_W(16)
#undef PIF_W
    default: break;
  }
}

// ES weights of the chunk's particles (positions already staged); particles
// cnt .. pad-1 get zero rows.  One item per (dimension, particle): the w window
// weights by per-node Horner polynomials (edge nodes exactly), zeros elsewhere
// in the tile row.  Starts and ends with __syncthreads().
template <int RX, int RY, int RZ, int CH>
__device__ __forceinline__ void stage_psi(Psi<RX, RY, RZ, CH>& sm, int cnt, int pad, const Brick& g,
                                          const int T0[3], const Horner& hc) {
  __syncthreads();
  const double two_over_w = 2.0 / g.w;
  const double flo = g.odd ? -0.5 : 0.0;
  const int w = g.w;
  using PS = Psi<RX, RY, RZ, CH>;
  constexpr int S = PS::S;
  // item = (dimension, particle): a warp's lanes share the dimension and write
  // consecutive particles of each node (node-major rows, see Psi)
  for (int it = threadIdx.x; it < 3 * pad; it += blockDim.x) {
    const int d = it / pad, p = it - d * pad;
    const int R = d == 0 ? RX : (d == 1 ? PS::PY : PS::ZP);
    double* col = d == 0 ? &sm.px[0][p] : (d == 1 ? &sm.py[0][p] : &sm.pz[0][p]);
    if (p >= cnt) {
      for (int u = 0; u < R; ++u) col[u * S] = 0.0;
      continue;
    }
    const int rel = sm.rel[p][d];
    const int T0d = d == 0 ? T0[0] : (d == 1 ? T0[1] : T0[2]);
    const double f = sm.xs[p][d] - (double)(rel + g.hw + T0d);  // x~ - anchor
    for (int u = 0; u < rel; ++u) col[u * S] = 0.0;
    for (int u = rel + w; u < R; ++u) col[u * S] = 0.0;  // (py: through the padded-column rows)
    const double sv = 2.0 * (f - flo) - 1.0;
    psi_row<S>(col, rel, f, sv, hc, g, two_over_w);
  }
  __syncthreads();
}

// ------------------------------------------------------------------ spread --
template <int RX, int RY, int RZ>
struct SpreadCfg {
  static constexpr int NCT = spread_nct(RX, RY);   // column tiles (of 8; the last ones may be padded)
  // column tiles per warp: 4 (or 5, 3) when that leaves >= 4 warps, else 1
  static constexpr int CT = (NCT % 4 == 0 && NCT >= 16) ? 4
                            : (NCT % 5 == 0 && NCT >= 20) ? 5
                            : (NCT % 3 == 0 && NCT >= 12) ? 3 : 1;
  static constexpr int NW = NCT / CT;             // warps
  static constexpr int ZT = (RZ + 7) / 8;         // z tiles of 8 (psi_z rows zero-padded)
  static constexpr bool PADC = NCT * 8 != RX * RY;  // padded columns c >= RX RY (A = 0: py rows >= RY)
  // TMA bulk-reduce flush: [column][z] tile rows of RZ doubles.  Used for the
  // 16-deep brick tiles (128-byte rows; C2 spread 0.675 -> 0.668 ms, C4 5.31 ->
  // 5.29 ms); the small sub-brick tiles (8-deep rows, many more items) measured
  // slower with it (C5 coarse 4.44 -> 4.60, C5 fine 8.62 -> 8.86 ms)
#ifndef PIF_SPREAD_BULK
#define PIF_SPREAD_BULK 1
#endif
  static constexpr bool BULK = PIF_SPREAD_BULK && RZ >= 16 && RZ % 2 == 0;
  // resident CTAs per SM the register budget must allow: small tiles (5 warps)
  // fit 5 by shared memory, and the register allocation decides between 3 and 4
  static constexpr int MINB = NW <= 5 ? 4 : PIF_SPREAD_MINB;
  static_assert(!BULK || (RX + RY + spread_pad_rows(RX, RY) + (RZ + 7) / 8 * 8) * (kChunk + 4) >= RX * RY * RZ,
                "the bulk-flush tile reuses the psi rows");
  static_assert(NCT % CT == 0, "tile shape");
};

// SUB: one CTA per interpolation item (a sub-brick's particles, tile RI)
// instead of per brick (tile RS): fewer padded FMAs per particle, more
// REDG.ADD.F64 per particle in the flush.
template <int RX, int RY, int RZ, bool HAS_S, bool SUB>
__global__ void __launch_bounds__(32 * SpreadCfg<RX, RY, RZ>::NW, SpreadCfg<RX, RY, RZ>::MINB)
    k_spread(const double* __restrict__ x, const int* __restrict__ perm, int64_t stride,
             const double* __restrict__ s,
             double s_uniform, const Sched Sc, Brick g,
             const __grid_constant__ Horner hc, double* __restrict__ grid) {
  using C = SpreadCfg<RX, RY, RZ>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Psi<RX, RY, RZ>& sm = *reinterpret_cast<Psi<RX, RY, RZ>*>(smem_raw);
  const int total = SUB ? Sc.ioff[Sc.nkeys] : Sc.soff[Sc.nkeys];
  // dynamically scheduled items: the first gridDim.x by block index, the rest
  // from the work counter Sc.ctr[0] (the grid is sized from the occupancy; crowded
  // and empty bricks differ by orders of magnitude in cost)
  __shared__ int next_item;
  for (int item = blockIdx.x; item < total;) {
  // claim the next item now: the counter's round trip overlaps this item
  int claimed = 0;
  if (threadIdx.x == 0) claimed = gridDim.x + atomicAdd(Sc.ctr, 1);
  do {  // one item (break: empty item)
  int T0[3];
  int64_t start, end;
  if (SUB) {
    const int4 e = Sc.iitems[item];
    const int4 f = Sc.iinfo[item];  // {bx, by, bz, sx | sy << 16}
    start = e.y;
    end = e.z;
    T0[0] = f.x * g.sb[0] - g.hw + (f.w & 0xffff) * g.ib[0];
    T0[1] = f.y * g.sb[1] - g.hw + (f.w >> 16) * g.ib[1];
    T0[2] = f.z * g.sb[2] - g.hw;
    if (start >= end) break;
  } else if (!tile_of(g, Sc, false, item, T0, start, end)) break;
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
    for (int q = tid; q < cnt; q += blockDim.x) {
      const int64_t sq = src_of(perm, base + q);
      double xr[3] = {x[sq], x[stride + sq], x[2 * stride + sq]};
      stage_position(sm, q, xr, g, T0);
      if (HAS_S) sm.str[q] = s[base + q];
    }
    stage_psi(sm, cnt, pad, g, T0, hc);
    for (int p0 = 0; p0 < pad; p0 += 4) {
      const int pl = p0 + tq;  // K index of this lane's A and B elements
      double b[C::ZT];
#pragma unroll
      for (int zt = 0; zt < C::ZT; ++zt) b[zt] = sm.pz[zt * 8 + gr][pl];
      double sp = 1.0;
      if (HAS_S) sp = pl < cnt ? sm.str[pl] : 0.0;
#pragma unroll
      for (int ct = 0; ct < C::CT; ++ct) {
        double a = sm.px[acx[ct]][pl] * sm.py[acy[ct]][pl];
        if (HAS_S) a *= sp;
#pragma unroll
        for (int zt = 0; zt < C::ZT; ++zt) dmma(acc[ct][zt], a, b[zt]);
      }
    }
    __syncthreads();
  }
  // flush: C[g][2t+i] = G[column (wid*CT+ct)*8 + gr][z = zt*8 + 2t + i]
  const int n = g.n;
  if (C::BULK && (T0[2] & 1) == 0) {
    // TMA bulk reduction (cp.reduce.async.bulk .add.f64, SASS UBLKRED): the tile
    // goes to shared memory as [column][z] rows -- a column's z run is
    // contiguous in the grid (z fastest) -- and each row is added to the grid
    // by one bulk operation (two where it wraps the periodic z boundary)
    // instead of RZ scalar REDG.ADD.F64.  Rows must be 16-byte aligned: RZ even
    // (compile time) and an even tile origin T0z (n even keeps its parity).
    // (The last chunk loop iteration ended with a barrier: psi is free.)
    double* tile = &sm.px[0][0];
#pragma unroll
    for (int ct = 0; ct < C::CT; ++ct) {
      const int col = acy[ct] * RX + acx[ct];
#pragma unroll
      for (int zt = 0; zt < C::ZT; ++zt)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int z = zt * 8 + 2 * tq + i;
          if (z < RZ && (!C::PADC || acy[ct] < RY)) tile[col * RZ + z] = acc[ct][zt][i] * s_uniform;
        }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> async-proxy reads
    __syncthreads();
    const int gz0 = wrapi(T0[2], n);
    const int seg = RZ < n - gz0 ? RZ : n - gz0;
    for (int row = threadIdx.x; row < RX * RY; row += blockDim.x) {
      const int cx = row % RX, cy = row / RX;
      double* col = grid + ((int64_t)wrapi(T0[0] + cx, n) * n + wrapi(T0[1] + cy, n)) * n;
      const double* src = tile + row * RZ;
      bulk_reduce_add_f64(col + gz0, src, seg);
      if (seg < RZ) bulk_reduce_add_f64(col, src + seg, RZ - seg);
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // smem reads done before reuse
  } else
#pragma unroll
  for (int ct = 0; ct < C::CT; ++ct) {
    double* colp = grid + ((int64_t)wrapi(T0[0] + acx[ct], n) * n + wrapi(T0[1] + acy[ct], n)) * n;
#pragma unroll
    for (int zt = 0; zt < C::ZT; ++zt)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const double val = acc[ct][zt][i];
        const int z = zt * 8 + 2 * tq + i;
        if (z < RZ && val != 0.0 && (!C::PADC || acy[ct] < RY))
          atomicAdd(colp + wrapi(T0[2] + z, n), val * s_uniform);
      }
  }
  } while (0);
  if (threadIdx.x == 0) next_item = claimed;
  __syncthreads();
  item = next_item;
  __syncthreads();
  }
}

// ------------------------------------------------- spread, warp-owned items --
// The sub-brick tiles (10x10x8 at w = 8, 6x6x8 at w = 5) with one WARP per
// interpolation item instead of one CTA: the warp stages the psi rows of 32
// particles at a time (lane = particle, all three dimensions) into its own
// shared-memory rows and runs the k loop over ALL column tiles of the tile, so
// there is no CTA barrier, and the A operand of a column tile,
// W[c][p] = psi_x[cx][p] psi_y[cy][p], reuses one factor across tiles: the
// columns of a tile are chosen so that, per lane, one of cx / cy is the same in
// every tile of a group (WTile), loaded once per k step.  Shared-memory loads
// per DMMA: 17 / 13 (10x10) and 7 / 5 (6x6) instead of 3 (two A factors + B) --
// the CTA kernel above is shared-memory bound at these tiles (ncu, C5 fine: LSU
// 85 %).  Accumulators stay in registers for the whole item (flush: one
// REDG.ADD.F64 per tile node, as above).
template <int RX, int RY>
struct WTile;
template <>
struct WTile<10, 10> {
  // tiles 0-9: row cy = ct, cx = gr (px[gr] shared); 10, 11: column cx = 8, 9,
  // cy = gr (py[gr] shared); 12: the 2 x 2 corner (cx, cy >= 8) on rows 0-3
  static constexpr int NCT = 13;
  __host__ __device__ static constexpr int group(int ct) { return ct < 10 ? 0 : (ct < 12 ? 1 : 2); }
  __device__ static bool col(int ct, int gr, int& cx, int& cy) {
    if (ct < 10) { cx = gr; cy = ct; return true; }
    if (ct < 12) { cx = 8 + ct - 10; cy = gr; return true; }
    cx = 8 + (gr & 1);
    cy = 8 + ((gr >> 1) & 1);
    return gr < 4;
  }
};
template <>
struct WTile<6, 6> {
  // tiles 0-4: rows 0-5 of the fragment cx = gr, cy = ct (px[gr] shared); rows
  // 6, 7 take the last row cy = 5, cx = 2 ct + gr - 6 (py[5] shared), tiles 0-2
  static constexpr int NCT = 5;
  __host__ __device__ static constexpr int group(int) { return 0; }
  __device__ static bool col(int ct, int gr, int& cx, int& cy) {
    if (gr < 6) { cx = gr; cy = ct; return true; }
    cx = 2 * ct + gr - 6;
    cy = 5;
    return ct <= 2;
  }
};

// The w weights in fp32 (fp32 plans, eps >= 1e-5: the weights' ~1e-7 relative
// error is far below eps) at row[(rel + k) ST]: the Horner chains run on the
// FP32 pipe instead of the FP64 datapath the DMMAs use.
template <int ST>
__device__ __forceinline__ void psi_row_f32(double* row, int rel, double f, double sv,
                                            const HornerF& hc, const Brick& g) {
  switch (g.w) {  // uniform
#define PIF_W(W)                                                          \
  case W: {                                                               \
    float pv[W];                                                          \
    psi_regs<float, W>(pv, (float)sv, f, hc, g);                          \
    _Pragma("unroll") for (int k = 0; k < W; ++k) row[(rel + k) * ST] = pv[k]; \
  } break;
    PIF_W(2) PIF_W(3) PIF_W(4) PIF_W(5) PIF_W(6) PIF_W(7) PIF_W(8)
#undef PIF_W
    default: break;
  }
}

template <int RX, int RY, int RZ>
struct SpreadWCfg {
  using TP = WTile<RX, RY>;
  static constexpr int NCT = TP::NCT;
  static constexpr int ZT = (RZ + 7) / 8;
  static constexpr int MP = 32;                 // particles per staging round (lane = particle)
  static constexpr int S = MP + 4;              // node-major row stride (4 mod 16)
  static constexpr int ZR = RX + RY;            // the zero row (padded columns)
  static constexpr int OZ = RX + RY + 1;        // first psi_z row
  static constexpr int ROWS = OZ + ZT * 8;
  static constexpr int NW = 4;                  // warps per CTA (each on its own items)
  static constexpr int MINB = NCT > 8 ? 5 : 7;  // resident CTAs per SM (registers, no spills)
};

template <int RX, int RY, int RZ, bool HAS_S, typename HC>
__global__ void __launch_bounds__(32 * SpreadWCfg<RX, RY, RZ>::NW, SpreadWCfg<RX, RY, RZ>::MINB)
    k_spread_warp(const double* __restrict__ x, const int* __restrict__ perm, int64_t stride,
                  const double* __restrict__ s,
                  double s_uniform, const Sched Sc, Brick g,
                  const __grid_constant__ HC hc, double* __restrict__ grid) {
  using C = SpreadWCfg<RX, RY, RZ>;
  using TP = typename C::TP;
  constexpr int S = C::S;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* const Q = reinterpret_cast<double*>(smem_raw) + wid * (C::ROWS * S);
  const int gr = lane >> 2, tq = lane & 3;
  const int n = g.n, w = g.w;
  const double two_over_w = 2.0 / w;
  const double flo = g.odd ? -0.5 : 0.0;
  // zero row (never written again)
  if (lane < S) Q[C::ZR * S + lane] = 0.0;
  if (lane + 32 < S) Q[C::ZR * S + lane + 32] = 0.0;
  // per-lane A rows: tile ct reads T[ct] (node-major row offset) and, in groups
  // 0 / 1, the shared factor H0 / H1; group 2 reads both factors per tile
  int toff[C::NCT], goff[C::NCT];
  int h0 = C::ZR * S, h1 = C::ZR * S;
#pragma unroll
  for (int ct = 0; ct < C::NCT; ++ct) {
    // shared factor of this lane in the tile's group: the coordinate that is
    // the same in the group's first two tiles (a one-tile group: px)
    int first = -1, second = -1;
#pragma unroll
    for (int u = 0; u < C::NCT; ++u)
      if (TP::group(u) == TP::group(ct)) {
        if (first < 0) first = u;
        else if (second < 0) second = u;
      }
    int cx, cy, fx, fy, sx = 0, sy = 0;
    const bool ok = TP::col(ct, gr, cx, cy);
    TP::col(first, gr, fx, fy);
    if (second >= 0) TP::col(second, gr, sx, sy);
    const bool share_x = second < 0 || fx == sx;
    const int hrow = share_x ? cx : RX + cy;
    const int trow = share_x ? RX + cy : cx;
    toff[ct] = ok ? trow * S : C::ZR * S;
    goff[ct] = TP::group(ct) == 2 ? hrow * S : 0;
    if (TP::group(ct) == 0 && ct == first) h0 = hrow * S;
    if (TP::group(ct) == 1 && ct == first) h1 = hrow * S;
  }
  const int total = Sc.ioff[Sc.nkeys];
  int item = blockIdx.x * C::NW + wid;
  while (item < total) {
    int claimed = 0;
    if (lane == 0) claimed = gridDim.x * C::NW + atomicAdd(Sc.ctr, 1);
    const int4 e = Sc.iitems[item];
    const int4 f = Sc.iinfo[item];  // {bx, by, bz, sx | sy << 16}
    const int64_t start = e.y, end = e.z;
    int T0[3];
    T0[0] = f.x * g.sb[0] - g.hw + (f.w & 0xffff) * g.ib[0];
    T0[1] = f.y * g.sb[1] - g.hw + (f.w >> 16) * g.ib[1];
    T0[2] = f.z * g.sb[2] - g.hw;
    double acc[C::NCT][C::ZT][2];
#pragma unroll
    for (int ct = 0; ct < C::NCT; ++ct)
#pragma unroll
      for (int zt = 0; zt < C::ZT; ++zt) acc[ct][zt][0] = acc[ct][zt][1] = 0.0;
    double xr[3] = {0.0, 0.0, 0.0}, sr = 0.0;
    if (start + lane < end) {
#pragma unroll
      for (int d = 0; d < 3; ++d) xr[d] = x[d * stride + src_of(perm, start + lane)];
      if (HAS_S) sr = s[start + lane];
    }
    for (int64_t base = start; base < end; base += C::MP) {
      const int cnt = (int)min((int64_t)C::MP, end - base);
      __syncwarp();  // the previous round's k loop is done with Q
      // lane = particle: the psi rows of all three dimensions (zeros outside the
      // window and for lanes past cnt)
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const int R = d == 0 ? RX : (d == 1 ? RY : C::ZT * 8);
        double* col = Q + (d == 0 ? 0 : (d == 1 ? RX : C::OZ)) * S + lane;
        int rel = R;
        double fr = 0.0;
        if (lane < cnt) {
          double xs = xr[d] * g.scale;
          const int a = anchor_of(xs, g);
          rel = a - g.hw - T0[d];
          fr = xs - (double)a;
        }
        for (int u = 0; u < R; ++u)
          if (u < rel || u >= rel + w) col[u * S] = 0.0;
        if (lane < cnt) {
          const double sv = 2.0 * (fr - flo) - 1.0;
          if constexpr (std::is_same<HC, HornerF>::value) psi_row_f32<S>(col, rel, fr, sv, hc, g);
          else psi_row<S>(col, rel, fr, sv, hc, g, two_over_w);
          if (HAS_S && d == 2)
            for (int u = 0; u < w; ++u) col[(rel + u) * S] *= sr;
        }
      }
      // prefetch the next round's positions (consumed after this k loop)
      if (base + C::MP + lane < end) {
#pragma unroll
        for (int d = 0; d < 3; ++d) xr[d] = x[d * stride + src_of(perm, base + C::MP + lane)];
        if (HAS_S) sr = s[base + C::MP + lane];
      }
      __syncwarp();
      const int pad = (cnt + 3) & ~3;
#pragma unroll 2
      for (int p0 = 0; p0 < pad; p0 += 4) {
        const int pl = p0 + tq;
        double b[C::ZT];
#pragma unroll
        for (int zt = 0; zt < C::ZT; ++zt) b[zt] = Q[(C::OZ + zt * 8 + gr) * S + pl];
        const double H0 = Q[h0 + pl];
        const double H1 = Q[h1 + pl];
#pragma unroll
        for (int ct = 0; ct < C::NCT; ++ct) {
          const double t = Q[toff[ct] + pl];
          const double hv = TP::group(ct) == 0 ? H0 : (TP::group(ct) == 1 ? H1 : Q[goff[ct] + pl]);
          const double a = hv * t;
#pragma unroll
          for (int zt = 0; zt < C::ZT; ++zt) dmma(acc[ct][zt], a, b[zt]);
        }
      }
    }
    // flush: C[gr][2 tq + i] = G[column TP::col(ct, gr)][z = 8 zt + 2 tq + i]
#pragma unroll
    for (int ct = 0; ct < C::NCT; ++ct) {
      int cx, cy;
      if (!TP::col(ct, gr, cx, cy)) continue;
      double* colp = grid + ((int64_t)wrapi(T0[0] + cx, n) * n + wrapi(T0[1] + cy, n)) * n;
#pragma unroll
      for (int zt = 0; zt < C::ZT; ++zt)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const double val = acc[ct][zt][i];
          const int z = zt * 8 + 2 * tq + i;
          if (z < RZ && val != 0.0) atomicAdd(colp + wrapi(T0[2] + z, n), val * s_uniform);
        }
    }
    item = __shfl_sync(0xffffffffu, claimed, 0);
  }
}

// ------------------------------------------------------------ interp+push --
// "K = columns" formulation: every warp owns whole m-tiles of 8 particles and
// contracts over all tile columns,
//   T_d[p][z] = sum_c W[p][c] g_d[c][z],   W[p][c] = psi_x[p][cx] psi_y[p][cy]
// (M = particles, K = columns, N = z), with the g tile in shared memory in
// B-fragment order (one conflict-free LDS.64 per DMMA) and A formed by one DMUL
// per fragment element.  Stage 2, E_d[p] = sum_z psi_z[p][z] T_d[p][z], is 16
// values per particle inside the warp, and the warp pushes its own particles.
//
// Persistent and warp-specialised: one producer warp streams the g tiles of the
// CTA's items (blockIdx.x, + gridDim.x, ...) into a ring of NBUF tile buffers
// with cp.async, completion signalled on mbarriers full[b]; NW consumer warps walk the CTA's
// concatenated m-tile sequence round-robin, each with its own x, v cp.async
// double buffer and psi rows (24 lanes = 8 particles x 3 dimensions, Horner
// groups warp-uniform), and release a tile buffer (empty[b]) once past its item.
// No CTA barrier after setup: a warp done with item k starts on item k+1 while
// others finish k, and the tile of item k+1 loads during item k.  DMMA and DFMA
// share the FP64 pipe on B200 (profiles/r1_dmma_mix.log): the vector work is
// ~7 % of the MMA FMAs.
template <int RX, int RY, int RZ>
struct InterpCfg {
  static constexpr int NC = RX * RY;       // tile columns (K)
  static constexpr int KS = NC / 4;        // k steps
  static constexpr int NT = (RZ + 7) / 8;  // z n-tiles of 8 (psi_z rows zero-padded)
  static constexpr int ZP = NT * 8;        // padded z extent
  // warp-private psi rows: px[8][SX] at 0, py[8][SY] at OY, pz[8][SZ] at OZ.
  // Row strides = 4 or 12 (mod 16) doubles keep the A-fragment reads
  // conflict-free; the 1 / 2 double offsets of py / pz put the 24 staging lanes'
  // row writes (particle p of x, y, z) in different banks.
  static constexpr int SX = RowStride<RX>::v, SY = RowStride<RY>::v, SZ = RowStride<ZP>::v;
  static constexpr int OY = 8 * SX + 1, OZ = OY + 8 * SY + 1;
  static constexpr int WP = OZ + 8 * SZ;   // psi doubles per warp (even: 16-byte aligned)
  static constexpr int GB = KS * NT * 3 * 32;  // doubles per g-tile buffer
  // consumer warps: as many as fit (<= 16) next to a double-buffered tile in
  // the 227 KB of dynamic shared memory a CTA may use; then as many tile
  // buffers as fit (<= 8: small tiles carry few particles, so the producer must
  // run several items ahead of the consumers)
  static constexpr int BYTES = 232448 - 16 * 8;  // minus the mbarriers
  static constexpr int BUDGET = BYTES / 8 - 2 * GB;
  static constexpr int NWFIT = BUDGET / (WP + 96);
  static constexpr int NW = NWFIT < 16 ? NWFIT : 16;
  static constexpr int NBFIT = (BYTES / 8 - NW * (WP + 96)) / GB;
  static constexpr int NBUF = NBFIT < 8 ? NBFIT : 8;
  // producer warps: small tiles carry few particles per loaded byte, so one
  // warp's copy issue rate would bound the kernel; they split the k steps
  static constexpr int NP = GB * 8 <= 24576 ? 4 : 1;
  static_assert(NC % 4 == 0, "tile columns must be a multiple of 4");
  static_assert(OZ % 2 == 0 && WP % 2 == 0, "pz rows are read as double2");
  static_assert(NW >= 4, "tile too large for the persistent interpolation kernel");
};

template <int RX, int RY, int RZ>
struct InterpSmem {
  using C = InterpCfg<RX, RY, RZ>;
  double gB[C::NBUF][C::KS][C::NT][3][32];  // B fragments, ring of tile buffers
  double psi[C::NW][C::WP];                 // per-warp psi rows
  double xv[C::NW][2][6][8];                // per-warp x, v double buffer (cp.async)
  unsigned long long full[C::NBUF], empty[C::NBUF];
};

// An interpolation item of this CTA (the k-th: item blockIdx.x + k gridDim.x)
// and its m-tiles [base, base + m) in the CTA's concatenated sequence.
struct ItemCursor {
  int k, base, m;
  int64_t start, end;
  int T0[3];
};

__device__ __forceinline__ void cursor_load(ItemCursor& it, const Brick& g, const Sched& Sc) {
  const int4 e = Sc.iitems[blockIdx.x + (int64_t)it.k * gridDim.x];
  it.start = e.y;
  it.end = e.z;
  it.m = (int)((e.z - e.y + 7) >> 3);
  const int M = g.m[0] * g.m[1] * g.m[2];
  const int brick = e.x / M, sk = e.x % M;
  const int bz = brick % g.NB[2], by = (brick / g.NB[2]) % g.NB[1], bx = brick / (g.NB[2] * g.NB[1]);
  const int sz = sk % g.m[2], sy = (sk / g.m[2]) % g.m[1], sx = sk / (g.m[2] * g.m[1]);
  it.T0[0] = bx * g.sb[0] - g.hw + sx * g.ib[0];
  it.T0[1] = by * g.sb[1] - g.hw + sy * g.ib[1];
  it.T0[2] = bz * g.sb[2] - g.hw + sz * g.ib[2];
}

template <int RX, int RY, int RZ>
__global__ void __launch_bounds__(32 * (InterpCfg<RX, RY, RZ>::NW + InterpCfg<RX, RY, RZ>::NP), 1)
    k_interp_push(const double* __restrict__ grid3, double* __restrict__ x,
                  double* __restrict__ v, int64_t stride, const int* __restrict__ id,
                  double* __restrict__ Eout, const Sched Sc, Brick g,
                  const __grid_constant__ Horner hc, PushArgs P) {
  using C = InterpCfg<RX, RY, RZ>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  InterpSmem<RX, RY, RZ>& S = *reinterpret_cast<InterpSmem<RX, RY, RZ>*>(smem_raw);
  const int total = Sc.ioff[Sc.nkeys];
  const int G = gridDim.x;
  const int nitems = (int)blockIdx.x < total ? (total - (int)blockIdx.x + G - 1) / G : 0;
  if (nitems == 0) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int n = g.n;
  const int64_t n3 = (int64_t)n * n * n;
  if (threadIdx.x == 0)
    for (int b = 0; b < C::NBUF; ++b) {
      mbar_init(&S.full[b], 32 * C::NP);
      mbar_init(&S.empty[b], C::NW);
    }
  __syncthreads();

  if (wid >= C::NW) {
    // ---- producer: g tile of item k -> gB[k % NBUF], stored lane-permuted:
    // B[t][g] = g_d[c = 4 ks + t][z = 8 nt + g] at gB[.][ks][nt][d][e],
    // e = 16 (g >> 2) + 4 t + (g & 3): each half-warp of a fragment read (g = 0..3
    // or 4..7) hits 16 distinct 8-byte bank slots, and the stores come in
    // 128-byte blocks of 4 columns x 4 z (lane = (h = g >> 2, t, zq = g & 3)).
    const int h = (lane >> 4) & 1, t = (lane >> 2) & 3, zq = lane & 3;
    const int eoff = (h << 4) | (t << 2) | zq;
    ItemCursor it;
    for (it.k = 0; it.k < nitems; ++it.k) {
      const int b = it.k % C::NBUF;
      if (it.k >= C::NBUF) mbar_wait(&S.empty[b], (it.k / C::NBUF - 1) & 1);
      cursor_load(it, g, Sc);
      int gz[C::NT];
      bool zin[C::NT];
#pragma unroll
      for (int nt = 0; nt < C::NT; ++nt) {
        const int zl = 8 * nt + 4 * h + zq;
        const int z = it.T0[2] + zl;
        gz[nt] = z < 0 ? z + n : (z >= n ? z - n : z);
        zin[nt] = zl < RZ;
      }
      const int pw = wid - C::NW;  // this producer's k steps: pw, pw + NP, ...
      int cx = (4 * pw + t) % RX, cy = (4 * pw + t) / RX;
      for (int ks = pw; ks < C::KS; ks += C::NP) {
        int gx = it.T0[0] + cx, gy = it.T0[1] + cy;
        gx = gx < 0 ? gx + n : (gx >= n ? gx - n : gx);
        gy = gy < 0 ? gy + n : (gy >= n ? gy - n : gy);
        const double* src = grid3 + ((int64_t)gx * n + gy) * n;
#pragma unroll
        for (int nt = 0; nt < C::NT; ++nt)
#pragma unroll
          for (int d = 0; d < 3; ++d)
            cp_async8_zfill(&S.gB[b][ks][nt][d][eoff], src + d * n3 + gz[nt], zin[nt]);
        cx += (4 * C::NP) % RX;
        cy += (4 * C::NP) / RX;
        if (cx >= RX) {
          cx -= RX;
          cy += 1;
        }
      }
      cp_async_mbar_arrive(&S.full[b]);
    }
    cp_async_wait_all();
    return;
  }

  // ---- consumers
  const int gr = lane >> 2, tq = lane & 3;
  const int lperm = ((gr >> 2) << 4) | (tq << 2) | (gr & 3);  // this lane's B-fragment entry
  double* const wpsi = S.psi[wid];
  double (*const xv)[6][8] = S.xv[wid];
  const double two_over_w = 2.0 / g.w;
  const double flo = g.odd ? -0.5 : 0.0;

  // cursor c: the item of the m-tile being computed; passing an item releases
  // its tile buffer (after its tile is known to have landed, so that this warp's
  // arrivals on empty[b] stay in phase order).  Cursor pf: x, v prefetch.
  ItemCursor c, pf;
  c.k = pf.k = 0;
  c.base = pf.base = 0;
  cursor_load(c, g, Sc);
  pf = c;
  auto pp = c;  // perm prefetch cursor (fused sort)
  auto advance = [&](ItemCursor& it, int q, bool release) {
    while (it.k < nitems && q >= it.base + it.m) {
      if (release) {
        mbar_wait(&S.full[it.k % C::NBUF], (it.k / C::NBUF) & 1);
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.empty[it.k % C::NBUF]);
      }
      it.base += it.m;
      if (++it.k < nitems) cursor_load(it, g, Sc);
    }
    return it.k < nitems;
  };
  // x, v of m-tile q -> xv[buf] (one cp.async group, possibly empty)
  // fused sort: the source index of this lane's particle (p = lane & 7) of an
  // m-tile, loaded one prefetch ahead (cursor pp) so that its latency does not
  // stall the cp.async issue
  auto perm_of = [&](int q) -> int {
    int r = 0;
    if (P.perm && advance(pp, q, false)) {
      const int64_t b = pp.start + 8 * (int64_t)(q - pp.base) + (lane & 7);
      if (b < pp.end) r = P.perm[b];
    }
    return r;
  };
  auto prefetch = [&](int buf, int q, int ps) {
    if (advance(pf, q, false)) {
      const int64_t b = pf.start + 8 * (int64_t)(q - pf.base);
      const int cnt = (int)min((int64_t)8, pf.end - b);
      for (int u = lane; u < 48; u += 32) {
        const int comp = u >> 3, p = u & 7;
        if (p < cnt) {
          const int64_t sj = P.perm ? (int64_t)ps : b + p;
          if (comp < 3) cp_async8(&xv[buf][comp][p], x + comp * stride + sj);
          else if (v) cp_async8(&xv[buf][comp][p], v + (comp - 3) * stride + sj);
        }
      }
    }
    cp_async_commit();
  };
  // psi rows of the current m-tile (cnt particles): lane = (particle p,
  // dimension d) for lanes < 24; zero row, then the w window weights (edge
  // nodes exactly, interior nodes by Horner groups of 4: warp-uniform constants)
  auto stage = [&](int buf, int cnt) {
    if (lane < 24) {
      const int p = lane & 7, d = lane >> 3;
      const int R = d == 0 ? RX : (d == 1 ? RY : C::ZP);
      double* row = wpsi + (d == 0 ? p * C::SX : (d == 1 ? C::OY + p * C::SY : C::OZ + p * C::SZ));
#pragma unroll
      for (int u = 0; u < (RX > C::ZP ? RX : (RY > C::ZP ? RY : C::ZP)); ++u)
        if (u < R) row[u] = 0.0;
      if (p < cnt) {
        const int w = g.w;
        const int T0d = d == 0 ? c.T0[0] : (d == 1 ? c.T0[1] : c.T0[2]);
        double xs = xv[buf][d][p] * g.scale;
        const int a = anchor_of(xs, g);
        const double f = xs - (double)a;
        double* wrow = row + (a - g.hw - T0d);
        const double sv = 2.0 * (f - flo) - 1.0;
        psi_row(wrow, 0, f, sv, hc, g, two_over_w);
      }
    }
  };

  int buf = 0;
  prefetch(0, wid, perm_of(wid));
  int pn = perm_of(wid + C::NW);
  for (int q = wid; advance(c, q, true); q += C::NW, buf ^= 1) {
    const int64_t b = c.start + 8 * (int64_t)(q - c.base);
    const int cnt = (int)min((int64_t)8, c.end - b);
    prefetch(buf ^ 1, q + C::NW, pn);  // xv[buf ^ 1] was released by the previous m-tile
    pn = perm_of(q + 2 * C::NW);
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncwarp();
    stage(buf, cnt);
    const int tb = c.k % C::NBUF;
    mbar_wait(&S.full[tb], (c.k / C::NBUF) & 1);  // g tile of this item landed
    __syncwarp();                            // psi rows visible to the warp
    double acc[C::NT][3][2];
#pragma unroll
    for (int nt = 0; nt < C::NT; ++nt)
#pragma unroll
      for (int d = 0; d < 3; ++d) acc[nt][d][0] = acc[nt][d][1] = 0.0;
    const double* pxr = wpsi + gr * C::SX;
    const double* pyr = wpsi + C::OY + gr * C::SY;
    const double* gBt = &S.gB[tb][0][0][0][0] + lperm;
    int cx = tq % RX, cy = tq / RX;  // column c = 4 ks + tq, advanced incrementally
#pragma unroll 2
    for (int ks = 0; ks < C::KS; ++ks) {
      const double a = pxr[cx] * pyr[cy];  // A[g][t] = W[p][4ks+t]
      cx += 4;
      if (cx >= RX) {
        cx -= RX;
        cy += 1;
      }
#pragma unroll
      for (int nt = 0; nt < C::NT; ++nt)
#pragma unroll
        for (int d = 0; d < 3; ++d) dmma(acc[nt][d], a, gBt[((ks * C::NT + nt) * 3 + d) * 32]);
    }
    // stage 2: C[g][2t+i] = T_d[p][z = 8nt + 2t + i]
    double e0 = 0.0, e1 = 0.0, e2 = 0.0;
    const double* pzr = wpsi + C::OZ + gr * C::SZ;
#pragma unroll
    for (int nt = 0; nt < C::NT; ++nt) {
      const double2 wz = *reinterpret_cast<const double2*>(pzr + 8 * nt + 2 * tq);
      e0 = fma(wz.x, acc[nt][0][0], fma(wz.y, acc[nt][0][1], e0));
      e1 = fma(wz.x, acc[nt][1][0], fma(wz.y, acc[nt][1][1], e1));
      e2 = fma(wz.x, acc[nt][2][0], fma(wz.y, acc[nt][2][1], e2));
    }
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {
      e0 += __shfl_xor_sync(0xffffffffu, e0, o);
      e1 += __shfl_xor_sync(0xffffffffu, e1, o);
      e2 += __shfl_xor_sync(0xffffffffu, e2, o);
    }
    if (tq == 0 && gr < cnt) {
      const int64_t j = b + gr, sj = src_of(P.perm, j);
      if (Eout) {
        const int64_t k = id[sj];
        Eout[k] = e0;
        Eout[stride + k] = e1;
        Eout[2 * stride + k] = e2;
      }
      if (P.kicks > 0 || P.drift) {
        double x0 = xv[buf][0][gr], x1 = xv[buf][1][gr], x2 = xv[buf][2][gr];
        double v0 = xv[buf][3][gr], v1 = xv[buf][4][gr], v2 = xv[buf][5][gr];
        push_particle(x0, x1, x2, v0, v1, v2, e0, e1, e2, P);
        double* const xo = P.xo ? P.xo : x;
        double* const vo = P.vo ? P.vo : v;
        xo[j] = x0;
        xo[stride + j] = x1;
        xo[2 * stride + j] = x2;
        vo[j] = v0;
        vo[stride + j] = v1;
        vo[2 * stride + j] = v2;
        if (P.ido) P.ido[j] = id[sj];
      }
    }
    __syncwarp();  // psi rows and xv[buf] are rewritten for the next m-tile
  }
  cp_async_wait_all();
}

// ------------------------------------------------ interp+push, slab ring --
// The same contraction as k_interp_push, but the g tile of an item is read from
// a ring of z-slabs of its BRICK (the spreading brick: BX x BY columns, SBZ z
// rows = one sub-brick height, 3 components) instead of a private copy per item.
// Each CTA takes a contiguous run of items in key order (brick-major, bz fastest,
// balanced by m-tile count, Sched::moff), so the items of one brick share its
// RZ / SBZ slabs and the next brick along z needs only one new slab: the producer warp
// loads 1/4 of a tile per brick step (w = 13) and runs up to NS - RZ / SBZ slabs
// ahead of the consumers, with the smem of ~1.8 tiles instead of 2.
//
// Virtual slab numbers: item k of the CTA uses slabs V_k .. V_k + NSZ - 1 (ring
// slot = v % NS), V_0 = 0; the next item of the same brick keeps V, the next
// brick of the same (bx, by) column at bz' > bz shifts V by min(bz' - bz, NSZ),
// anything else by NSZ (all slabs new).  Protocol: full[k % ND] -- the
// producer's cp.async of every slab item k needs have landed; done[k % ND] --
// every consumer warp has passed item k.  The producer overwrites a slot only
// after done[] of the last item that used it, and never runs more than ND items
// ahead (done[k - ND]), so the parity waits never alias.
//
// Slab layout: [cy * CS + cx][d][r] (r < SBZ rows), CS = 18 for BX = 16: the
// B-fragment reads (lane (g, t): tile row 8 nt + g, sub-window column 4 ks + t)
// are conflict-free for every sub-brick offset (checked exhaustively).
template <int RX, int RY, int RZ, int BX, int BY, int SBZ, int CSX, int ZR>
struct SlabCfg {
  using I = InterpCfg<RX, RY, RZ>;
  static constexpr int KS = I::KS, NT = I::NT;
  static constexpr int SX = I::SX, SY = I::SY, SZ = I::SZ, OY = I::OY, OZ = I::OZ, WP = I::WP;
  static constexpr int CS = CSX;                    // columns per brick row (>= BX)
  // doubles per slab: BY (+ ZR padding) rows; one-row slabs (SBZ = 1) are padded
  // to 4 (mod 16) so that the 4 slabs of a half-warp's fragment rows fall in
  // different banks (conflict pattern checked exhaustively)
  static constexpr int ZROW = ZR;                   // + a padding row per slab (bank spread)
  static constexpr int SLAB0 = (BY + ZROW) * CS * 3 * SBZ;
  static constexpr int SLAB = SBZ == 1 ? SLAB0 + ((20 - SLAB0 % 16) % 16) : SLAB0;
  static constexpr int NSZ = RZ / SBZ;              // slabs per tile
  static constexpr int ND = 16;                     // full / done barrier ring
#ifndef PIF_SLAB_NS
#define PIF_SLAB_NS 6
#endif
  // slab ring: a tile plus the lookahead (brick steps along z)
  static constexpr int NS = NSZ == 4 ? PIF_SLAB_NS : (SBZ == 1 ? NSZ + 4 : NSZ + 2);
  static_assert(ZR == 1 || NS * (BY * CSX * 3 * SBZ) * 8 + 8 * (WP + 96) * 16 <= 232448 - 512,
                "ring too large");
#ifndef PIF_SLAB_NW
#define PIF_SLAB_NW 16
#endif
#ifndef PIF_SLAB_MT2
#define PIF_SLAB_MT2 1
#endif
  // m-unit: MT m-tiles of 8 particles contracted together over ONE window (the
  // union of their cells), sharing every B fragment load and the per-unit
  // cursor / prefetch / window work.  MT = 2 for the 1-row slabs (w = 8: 16 k
  // steps x 3 DMMAs per m-tile, so the per-m-tile work dominated), else 1.
  static constexpr int MT = (SBZ == 1 && PIF_SLAB_MT2) ? 2 : 1;
  static constexpr int MP = 8 * MT;                 // particles per m-unit
  static constexpr int OYM = MP * SX + 1, OZM = OYM + MP * SY + 1;
  static constexpr int WPM = OZM + MP * SZ;         // psi doubles per warp
  static_assert(OZM % 2 == 0 && WPM % 2 == 0, "pz rows are read as double2");
  static constexpr int BYTES = 232448 - 2 * ND * 8 - 64;
  static constexpr int NWFIT = (BYTES / 8 - NS * SLAB) / (WPM + 12 * MP);
#ifndef PIF_SLAB_NW1
#define PIF_SLAB_NW1 16  // one-row slabs (w = 8 dense) with 16-particle m-units: 16 measured
                         // 1.3 % faster than 18 (the shared-memory fit) and 6 % faster than 14
                         // (with 8-particle m-tiles 20 was best, 2.4 % ahead of 24)
#endif
  static constexpr int NWCAP = SBZ == 1 ? PIF_SLAB_NW1 : PIF_SLAB_NW;
  static constexpr int NW = NWFIT < NWCAP ? NWFIT : NWCAP;
  // psi rows are zero-filled to FILL entries (px < RX, py <= RY: the padded
  // columns of a window's last k step, pz < ZP)
  static constexpr int FILL0 = RX > RY + 1 ? RX : RY + 1;
  static constexpr int FILL = FILL0 > I::ZP ? FILL0 : I::ZP;
  static_assert(FILL <= SX && FILL <= SY && FILL <= SZ, "psi row strides");
  static_assert(CS >= BX, "brick row");
  static_assert(RZ % SBZ == 0 && RZ % 8 == 0 && (SBZ == 1 || SBZ == 4), "slab rows");
  static_assert(NS > NSZ, "slab ring must hold a tile plus lookahead");
  static_assert(NW >= 8, "slab ring too large");
};

template <int RX, int RY, int RZ, int BX, int BY, int SBZ, int CSX, int ZR>
struct SlabSmem {
  using C = SlabCfg<RX, RY, RZ, BX, BY, SBZ, CSX, ZR>;
  double slab[C::NS][C::SLAB];
  double psi[C::NW][C::WPM];
  double xv[C::NW][2][6][C::MP];
  unsigned long long full[C::ND], done[C::ND];
  int range[2];
};

// Item k of this CTA's run (global index lo + k): particle range, tile origin,
// sub-brick column offset and virtual slab number (needs the previous item's
// brick coordinates: call in order of k).
struct SlabCursor {
  int k, base, m;
  int64_t start, end;
  int T0[3];
  int ox, oy, V;
  int bcol, bz;  // brick column (bx * NB1 + by) and bz of item k
};

template <int NSZ, int MP = 8>
__device__ __forceinline__ void slab_cursor_load(SlabCursor& it, int lo, const Brick& g,
                                                 const Sched& Sc) {
  const int4 e = Sc.iitems[lo + it.k];
  const int4 f = Sc.iinfo[lo + it.k];  // {bx, by, bz, sx | sy << 16}
  it.start = e.y;
  it.end = e.z;
  it.m = (int)((e.z - e.y + MP - 1) / MP);
  const int bx = f.x, by = f.y, bz = f.z, sx = f.w & 0xffff, sy = f.w >> 16;
  const int bcol = bx * g.NB[1] + by;
  it.ox = sx * g.ib[0];
  it.oy = sy * g.ib[1];
  it.T0[0] = bx * g.sb[0] - g.hw + it.ox;
  it.T0[1] = by * g.sb[1] - g.hw + it.oy;
  it.T0[2] = bz * g.sb[2] - g.hw;
  if (it.k == 0) it.V = 0;
  else if (bcol == it.bcol && bz == it.bz) {
  } else if (bcol == it.bcol && bz > it.bz) it.V += min(bz - it.bz, NSZ);
  else it.V += NSZ;
  it.bcol = bcol;
  it.bz = bz;
}

template <int RX, int RY, int RZ, int BX, int BY, int SBZ, int CSX, int ZR>
__global__ void __launch_bounds__(32 * (SlabCfg<RX, RY, RZ, BX, BY, SBZ, CSX, ZR>::NW + 1), 1)
    k_interp_push_slab(const double* __restrict__ grid3, double* __restrict__ x,
                       double* __restrict__ v, int64_t stride, const int* __restrict__ id,
                       double* __restrict__ Eout, const Sched Sc, Brick g,
                       const __grid_constant__ Horner hc, PushArgs P) {
  using C = SlabCfg<RX, RY, RZ, BX, BY, SBZ, CSX, ZR>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SlabSmem<RX, RY, RZ, BX, BY, SBZ, CSX, ZR>& S = *reinterpret_cast<SlabSmem<RX, RY, RZ, BX, BY, SBZ, CSX, ZR>*>(smem_raw);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int n = g.n;
  const int64_t n3 = (int64_t)n * n * n;
  if (threadIdx.x == 0) {
    // contiguous item run of this CTA: items whose first m-tile lies in
    // [b M / G, (b + 1) M / G), M = all m-tiles (iitems[].w, increasing)
    const int total = Sc.ioff[Sc.nkeys];
    const int64_t Mt = Sc.moff[Sc.nkeys];
    int r[2];
    for (int q = 0; q < 2; ++q) {
      const int64_t target = (int64_t)(blockIdx.x + q) * Mt / gridDim.x;
      int a = 0, b = total;  // first item with first m-tile >= target
      while (a < b) {
        const int mid = (a + b) >> 1;
        if ((int64_t)Sc.iitems[mid].w < target) a = mid + 1;
        else b = mid;
      }
      r[q] = (blockIdx.x + q == gridDim.x) ? total : a;
    }
    S.range[0] = r[0];
    S.range[1] = r[1];
    for (int b = 0; b < C::ND; ++b) {
      mbar_init(&S.full[b], 32);
      mbar_init(&S.done[b], C::NW);
    }
  }
  __syncthreads();
  const int lo = S.range[0], nitems = S.range[1] - S.range[0];
  if (nitems <= 0) return;

  if (wid == C::NW) {
    // ---- producer: the new slabs of item k -> ring slots, then full[k].
    // Lane = (column j of 8, row r of 4): a 32-byte z run of one (column, d).
    constexpr int RQ = SBZ < 4 ? SBZ : 4;   // rows per instruction
    constexpr int CQ = 32 / RQ;             // columns per instruction
    const int r0 = lane % RQ, j0 = lane / RQ;
    int lastuse[C::NS];
#pragma unroll
    for (int s2 = 0; s2 < C::NS; ++s2) lastuse[s2] = -1;
    int loaded = 0;
    SlabCursor it;
    it.V = 0;
    it.bcol = it.bz = -1;
    for (it.k = 0; it.k < nitems; ++it.k) {
      slab_cursor_load<C::NSZ>(it, lo, g, Sc);
      if (it.k >= C::ND) mbar_wait(&S.done[(it.k - C::ND) % C::ND], ((it.k - C::ND) / C::ND) & 1);
      for (int vs = max(loaded, it.V); vs < it.V + C::NSZ; ++vs) {
        const int slot = vs % C::NS;
        int j = -1;
#pragma unroll
        for (int s2 = 0; s2 < C::NS; ++s2)
          if (s2 == slot) j = lastuse[s2];
        if (j >= 0 && j > it.k - C::ND) mbar_wait(&S.done[j % C::ND], (j / C::ND) & 1);
        const int i = vs - it.V;  // slab of the tile: rows T0z + i SBZ ..
        double* dst = S.slab[slot];
        const int Bx0 = it.T0[0] - it.ox, By0 = it.T0[1] - it.oy;
        for (int rq = 0; rq < SBZ; rq += RQ) {
          const int r = rq + r0;
          int gz = it.T0[2] + i * SBZ + r;
          gz = gz < 0 ? gz + n : (gz >= n ? gz - n : gz);
          for (int c0 = 0; c0 < BX * BY; c0 += CQ) {
            const int cc = c0 + j0;
            if (cc < BX * BY) {
              const int cy = cc / BX, cx = cc - cy * BX;
              int gx = Bx0 + cx, gy = By0 + cy;
              gx = gx < 0 ? gx + n : (gx >= n ? gx - n : gx);
              gy = gy < 0 ? gy + n : (gy >= n ? gy - n : gy);
              const double* src = grid3 + ((int64_t)gx * n + gy) * n + gz;
              double* d0 = dst + ((cy * C::CS + cx) * 3) * SBZ + r;
#pragma unroll
              for (int d = 0; d < 3; ++d) cp_async8(d0 + d * SBZ, src + d * n3);
            }
          }
        }
      }
      loaded = max(loaded, it.V + C::NSZ);
#pragma unroll
      for (int s2 = 0; s2 < C::NS; ++s2) {
        const int off = (s2 - it.V % C::NS + C::NS) % C::NS;  // slot s2 = (V + off) % NS
        if (off < C::NSZ) lastuse[s2] = it.k;
      }
      cp_async_mbar_arrive(&S.full[it.k % C::ND]);
    }
    cp_async_wait_all();
    return;
  }

  // ---- consumers (as k_interp_push; B fragments from the slab ring)
  const int gr = lane >> 2, tq = lane & 3;
  double* const wpsi = S.psi[wid];
  double (*const xv)[6][C::MP] = S.xv[wid];
  constexpr int MT = C::MT, MP = C::MP;
  const double two_over_w = 2.0 / g.w;
  const double flo = g.odd ? -0.5 : 0.0;
  SlabCursor c, pf;
  c.k = pf.k = 0;
  c.base = pf.base = 0;
  c.V = 0;
  c.bcol = c.bz = -1;
  slab_cursor_load<C::NSZ, MP>(c, lo, g, Sc);
  pf = c;
  auto pp = c;  // perm prefetch cursor (fused sort)
  auto advance = [&](SlabCursor& it, int q, bool release) {
    while (it.k < nitems && q >= it.base + it.m) {
      if (release) {
        mbar_wait(&S.full[it.k % C::ND], (it.k / C::ND) & 1);
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.done[it.k % C::ND]);
      }
      it.base += it.m;
      if (++it.k < nitems) slab_cursor_load<C::NSZ, MP>(it, lo, g, Sc);
    }
    return it.k < nitems;
  };
  // fused sort: the source index of this lane's particle (p = lane & 7) of an
  // m-tile, loaded one prefetch ahead (cursor pp) so that its latency does not
  // stall the cp.async issue
  auto perm_of = [&](int q) -> int {
    int r = 0;
    if (P.perm && advance(pp, q, false)) {
      const int64_t b = pp.start + MP * (int64_t)(q - pp.base) + (lane % MP);
      if (b < pp.end) r = P.perm[b];
    }
    return r;
  };
  auto prefetch = [&](int buf, int q, int ps) {
    if (advance(pf, q, false)) {
      const int64_t b = pf.start + MP * (int64_t)(q - pf.base);
      const int cnt = (int)min((int64_t)MP, pf.end - b);
      for (int u = lane; u < 6 * MP; u += 32) {
        const int comp = u / MP, p = u % MP;
        if (p < cnt) {
          const int64_t sj = P.perm ? (int64_t)ps : b + p;
          if (comp < 3) cp_async8(&xv[buf][comp][p], x + comp * stride + sj);
          else if (v) cp_async8(&xv[buf][comp][p], v + (comp - 3) * stride + sj);
        }
      }
    }
    cp_async_commit();
  };
  // psi rows of the current m-tile relative to ITS window: the m-tile's particles
  // (sorted by xy-cell, Brick::C) span cells ox_m .. ox_m + ex_x of the
  // sub-brick in x (same in y), so the window is (w + ex_x) x (w + ex_y) columns
  // from column (ox_m, oy_m) of the sub-brick tile -- 13 x 13 when all 8 share a
  // cell.  Rows are zero outside the window up to C::FILL entries.
  int ox_m = 0, oy_m = 0, ex_x = 0, ex_y = 0;
  // (m-unit of MT m-tiles: lane = (particle p of m-tile r, dimension d), the
  // window is the union over the unit's MP particles)
  auto stage = [&](int buf, int cnt) {
    const int p = lane & 7, d = lane >> 3;
    const int T0d = d == 0 ? c.T0[0] : (d == 1 ? c.T0[1] : c.T0[2]);
    bool valid[MT];
    int rel[MT];
    double f[MT];
    int mn = 1 << 20, mx = -1;
#pragma unroll
    for (int r = 0; r < MT; ++r) {
      valid[r] = lane < 24 && 8 * r + p < cnt;
      rel[r] = 0;
      f[r] = 0.0;
      if (valid[r]) {
        double xs = xv[buf][d][8 * r + p] * g.scale;
        const int a = anchor_of(xs, g);
        f[r] = xs - (double)a;
        rel[r] = a - g.hw - T0d;
        mn = min(mn, rel[r]);
        mx = max(mx, rel[r]);
      }
    }
#pragma unroll
    for (int o = 1; o <= 4; o <<= 1) {
      mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    ox_m = __shfl_sync(0xffffffffu, mn, 0);
    oy_m = __shfl_sync(0xffffffffu, mn, 8);
    ex_x = __shfl_sync(0xffffffffu, mx, 0) - ox_m;
    ex_y = __shfl_sync(0xffffffffu, mx, 8) - oy_m;
    // zero fill, then the weights.  One-row slabs (w = 8): the warp's psi rows
    // with contiguous 16-byte stores (C5 fine interp 12.67 -> 12.41 ms); w = 13:
    // per staging lane and row (the cooperative fill measured 0.5 % slower)
    if constexpr (SBZ == 1) {
#pragma unroll
      for (int i = lane; i < C::WPM / 2; i += 32) reinterpret_cast<double2*>(wpsi)[i] = make_double2(0.0, 0.0);
      __syncwarp();
    }
#pragma unroll
    for (int r = 0; r < MT; ++r) {
      const int pr = 8 * r + p;
      double* row = wpsi + (d == 0 ? pr * C::SX : (d == 1 ? C::OYM + pr * C::SY : C::OZM + pr * C::SZ));
      if (SBZ != 1 && lane < 24) {
#pragma unroll
        for (int u = 0; u < C::FILL; ++u) row[u] = 0.0;
      }
      if (valid[r]) {
        const double sv = 2.0 * (f[r] - flo) - 1.0;
        psi_row(row + rel[r] - (d == 0 ? ox_m : (d == 1 ? oy_m : 0)), 0, f[r], sv, hc, g, two_over_w);
      }
    }
  };

  int buf = 0;
  prefetch(0, wid, perm_of(wid));
  int pn = perm_of(wid + C::NW);
  for (int q = wid; advance(c, q, true); q += C::NW, buf ^= 1) {
    const int64_t b = c.start + MP * (int64_t)(q - c.base);
    const int cnt = (int)min((int64_t)MP, c.end - b);
    prefetch(buf ^ 1, q + C::NW, pn);
    pn = perm_of(q + 2 * C::NW);
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncwarp();
    stage(buf, cnt);
    mbar_wait(&S.full[c.k % C::ND], (c.k / C::ND) & 1);  // every slab of this item landed
    __syncwarp();
    // this lane's B-fragment rows: tile row zl = 8 nt + gr -> slab zl / SBZ, row zl % SBZ
    const double* Pb[C::NT];
#pragma unroll
    for (int nt = 0; nt < C::NT; ++nt) {
      const int zl = 8 * nt + gr;
      Pb[nt] = &S.slab[(c.V + zl / SBZ) % C::NS][0] + (zl % SBZ) +
               ((c.oy + oy_m) * C::CS + c.ox + ox_m) * 3 * SBZ;
    }
    const int RXm = g.w + ex_x, RYm = g.w + ex_y;  // m-tile window (<= RX x RY)
    const int KSm = (RXm * RYm + 3) >> 2;
    double acc[MT][C::NT][3][2];
#pragma unroll
    for (int r = 0; r < MT; ++r)
#pragma unroll
      for (int nt = 0; nt < C::NT; ++nt)
#pragma unroll
        for (int d = 0; d < 3; ++d) acc[r][nt][d][0] = acc[r][nt][d][1] = 0.0;
    const double* pxr[MT];
    const double* pyr[MT];
#pragma unroll
    for (int r = 0; r < MT; ++r) {
      pxr[r] = wpsi + (8 * r + gr) * C::SX;
      pyr[r] = wpsi + C::OYM + (8 * r + gr) * C::SY;
    }
    int cx = tq, cy = 0;  // column 4 ks + tq of the window (RXm >= 4)
    // B offset (cy CS + cx) 3 SBZ kept incrementally: + 4 columns per k step,
    // + (CS - RXm) columns at a window-row wrap.  Used for the 1-row slabs
    // (w = 8: C5 fine interp 14.15 -> 14.02 ms); the 4-row slabs (w = 13)
    // measured slower with it (C2 1.433 -> 1.489 ms), so they keep the
    // recomputed offset below.
    if constexpr (SBZ == 1) {
    int off = cx * 3 * SBZ;
    const int wrap_off = (C::CS - RXm) * 3 * SBZ;
#pragma unroll 2
    for (int ks = 0; ks < KSm - 1; ++ks) {
      double a[MT];
#pragma unroll
      for (int r = 0; r < MT; ++r) a[r] = pxr[r][cx] * pyr[r][cy];
      const int o = off;
      cx += 4;
      off += 4 * 3 * SBZ;
      if (cx >= RXm) {
        cx -= RXm;
        cy += 1;
        off += wrap_off;
      }
#pragma unroll
      for (int nt = 0; nt < C::NT; ++nt)
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const double bb = Pb[nt][o + d * SBZ];
#pragma unroll
          for (int r = 0; r < MT; ++r) dmma(acc[r][nt][d], a[r], bb);
        }
    }
    } else {
#pragma unroll 2
    for (int ks = 0; ks < KSm - 1; ++ks) {
      double a[MT];
#pragma unroll
      for (int r = 0; r < MT; ++r) a[r] = pxr[r][cx] * pyr[r][cy];
      const int off = (cy * C::CS + cx) * 3 * SBZ;
      cx += 4;
      if (cx >= RXm) {
        cx -= RXm;
        cy += 1;
      }
#pragma unroll
      for (int nt = 0; nt < C::NT; ++nt)
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const double bb = Pb[nt][off + d * SBZ];
#pragma unroll
          for (int r = 0; r < MT; ++r) dmma(acc[r][nt][d], a[r], bb);
        }
    }
    }
    {
      // last k step: columns past the window (cy == RYm) have A = 0 (py rows are
      // zero-filled past the window) and read B from the window's last row, so
      // every B operand is landed data of this item's slabs (no read outside them)
      double a[MT];
#pragma unroll
      for (int r = 0; r < MT; ++r) a[r] = pxr[r][cx] * pyr[r][cy];
      const int off = ((cy < RYm ? cy : RYm - 1) * C::CS + cx) * 3 * SBZ;
#pragma unroll
      for (int nt = 0; nt < C::NT; ++nt)
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const double bb = Pb[nt][off + d * SBZ];
#pragma unroll
          for (int r = 0; r < MT; ++r) dmma(acc[r][nt][d], a[r], bb);
        }
    }
    // lanes tq = r hold (after the xor reduction every tq lane does) the field
    // of particle 8 r + gr; lane tq = r < MT pushes it
    double e0 = 0.0, e1 = 0.0, e2 = 0.0;
#pragma unroll
    for (int r = 0; r < MT; ++r) {
      double f0 = 0.0, f1 = 0.0, f2 = 0.0;
      const double* pzr = wpsi + C::OZM + (8 * r + gr) * C::SZ;
#pragma unroll
      for (int nt = 0; nt < C::NT; ++nt) {
        const double2 wz = *reinterpret_cast<const double2*>(pzr + 8 * nt + 2 * tq);
        f0 = fma(wz.x, acc[r][nt][0][0], fma(wz.y, acc[r][nt][0][1], f0));
        f1 = fma(wz.x, acc[r][nt][1][0], fma(wz.y, acc[r][nt][1][1], f1));
        f2 = fma(wz.x, acc[r][nt][2][0], fma(wz.y, acc[r][nt][2][1], f2));
      }
#pragma unroll
      for (int o = 1; o <= 2; o <<= 1) {
        f0 += __shfl_xor_sync(0xffffffffu, f0, o);
        f1 += __shfl_xor_sync(0xffffffffu, f1, o);
        f2 += __shfl_xor_sync(0xffffffffu, f2, o);
      }
      if (tq == r) {
        e0 = f0;
        e1 = f1;
        e2 = f2;
      }
    }
    const int pq = 8 * tq + gr;  // this lane's particle in the m-unit (tq < MT)
    if (tq < MT && pq < cnt) {
      const int64_t j = b + pq, sj = src_of(P.perm, j);
      if (Eout) {
        const int64_t k = id[sj];
        Eout[k] = e0;
        Eout[stride + k] = e1;
        Eout[2 * stride + k] = e2;
      }
      if (P.kicks > 0 || P.drift) {
        double x0 = xv[buf][0][pq], x1 = xv[buf][1][pq], x2 = xv[buf][2][pq];
        double v0 = xv[buf][3][pq], v1 = xv[buf][4][pq], v2 = xv[buf][5][pq];
        push_particle(x0, x1, x2, v0, v1, v2, e0, e1, e2, P);
        double* const xo = P.xo ? P.xo : x;
        double* const vo = P.vo ? P.vo : v;
        xo[j] = x0;
        xo[stride + j] = x1;
        xo[2 * stride + j] = x2;
        vo[j] = v0;
        vo[stride + j] = v1;
        vo[2 * stride + j] = v2;
        if (P.ido) P.ido[j] = id[sj];
      }
    }
    __syncwarp();
  }
  cp_async_wait_all();
}

template <int A, int B, int Cz, bool SUB = false>
static cudaError_t spread_launch(unsigned nbr, const double* x, const int* perm, int64_t stride,
                                 const double* s,
                                 double s_uniform, const Sched& offsets, const Brick& g,
                                 const Horner& hc, double* grid, cudaStream_t st) {
  const int T = 32 * SpreadCfg<A, B, Cz>::NW;
  const size_t smem = sizeof(Psi<A, B, Cz, kChunk>);
  static DevCache cache;
  int ctas = 0;  // resident CTAs on the device
  cudaError_t e = dev_cached(cache, ctas, [&](int dev, int& v) {
    int sms = 0, per = 0;
    cudaError_t r = cudaFuncSetAttribute(k_spread<A, B, Cz, true, SUB>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (r == cudaSuccess)
      r = cudaFuncSetAttribute(k_spread<A, B, Cz, false, SUB>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (r == cudaSuccess) r = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (r == cudaSuccess)
      r = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_spread<A, B, Cz, false, SUB>, T, smem);
    v = sms * per;
    return r;
  });
  if (e != cudaSuccess) return e;
  // an item bound of up to ~n_keys CTAs (most of them empty) -> 2 waves of
  // resident CTAs striding over the items
#ifndef PIF_SPREAD_WAVES
#define PIF_SPREAD_WAVES 2
#endif
  if ((int64_t)nbr > PIF_SPREAD_WAVES * (int64_t)ctas) nbr = PIF_SPREAD_WAVES * ctas;
  cudaError_t e0 = cudaMemsetAsync(offsets.ctr, 0, sizeof(int), st);
  if (e0 != cudaSuccess) return e0;
  if (s)
    k_spread<A, B, Cz, true, SUB><<<nbr, T, smem, st>>>(x, perm, stride, s, s_uniform, offsets, g, hc, grid);
  else
    k_spread<A, B, Cz, false, SUB><<<nbr, T, smem, st>>>(x, perm, stride, s, s_uniform, offsets, g, hc, grid);
  return cudaGetLastError();
}

#ifndef PIF_SPREAD_WARP
#define PIF_SPREAD_WARP 1
#endif
template <int A, int B, int Cz, typename HC>
static cudaError_t spread_warp_launch(unsigned nitems, const double* x, const int* perm, int64_t stride,
                                      const double* s,
                                      double s_uniform, const Sched& offsets, const Brick& g,
                                      const HC& hc, double* grid, cudaStream_t st) {
  using C = SpreadWCfg<A, B, Cz>;
  const int T = 32 * C::NW;
  const size_t smem = sizeof(double) * C::NW * C::ROWS * C::S;
  static DevCache cache;
  int ctas = 0;  // resident CTAs on the device
  cudaError_t e = dev_cached(cache, ctas, [&](int dev, int& v) {
    int sms = 0, per = 0;
    cudaError_t r = cudaFuncSetAttribute(k_spread_warp<A, B, Cz, true, HC>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (r == cudaSuccess)
      r = cudaFuncSetAttribute(k_spread_warp<A, B, Cz, false, HC>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (r == cudaSuccess) r = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (r == cudaSuccess)
      r = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_spread_warp<A, B, Cz, false, HC>, T, smem);
    v = sms * per;
    return r;
  });
  if (e != cudaSuccess) return e;
  unsigned nbr = (nitems + C::NW - 1) / C::NW;
  if ((int64_t)nbr > (int64_t)ctas) nbr = ctas;  // persistent: one wave, items claimed by warps
  if (nbr == 0) return cudaSuccess;
  cudaError_t e0 = cudaMemsetAsync(offsets.ctr, 0, sizeof(int), st);
  if (e0 != cudaSuccess) return e0;
  if (s)
    k_spread_warp<A, B, Cz, true, HC><<<nbr, T, smem, st>>>(x, perm, stride, s, s_uniform, offsets, g, hc, grid);
  else
    k_spread_warp<A, B, Cz, false, HC><<<nbr, T, smem, st>>>(x, perm, stride, s, s_uniform, offsets, g, hc, grid);
  return cudaGetLastError();
}

#ifndef PIF_SPREAD_F32PSI
#define PIF_SPREAD_F32PSI 1
#endif
cudaError_t launch_spread(const double* x, const int* perm, int64_t stride, const double* s,
                          double s_uniform, const Sched& offsets, const Brick& g, const Horner& hc,
                          const HornerF* hcf, double* grid, cudaStream_t st) {
  const unsigned ni = (unsigned)offsets.max_i;
  if (PIF_SPREAD_WARP && g.C > 1 && g.RI[0] == 10 && g.RI[1] == 10 && g.RI[2] == 8)
    return (PIF_SPREAD_F32PSI && hcf)
               ? spread_warp_launch<10, 10, 8>(ni, x, perm, stride, s, s_uniform, offsets, g, *hcf, grid, st)
               : spread_warp_launch<10, 10, 8>(ni, x, perm, stride, s, s_uniform, offsets, g, hc, grid, st);
  if (PIF_SPREAD_WARP && g.C > 1 && g.RI[0] == 6 && g.RI[1] == 6 && g.RI[2] == 8)
    return (PIF_SPREAD_F32PSI && hcf)
               ? spread_warp_launch<6, 6, 8>(ni, x, perm, stride, s, s_uniform, offsets, g, *hcf, grid, st)
               : spread_warp_launch<6, 6, 8>(ni, x, perm, stride, s, s_uniform, offsets, g, hc, grid, st);
  // dense w = 8 / w = 5 plans (>= 12 / 8 particles per cell, cell keys): spread
  // over the interpolation sub-bricks with the interpolation tile (10x10x8 /
  // 6x6x8 instead of 16x16x8 / 8^3: 2.6x / 1.8x fewer padded FMAs), the extra
  // REDG flush per particle being small at that density
  if (g.C > 1 && g.RI[0] == 10 && g.RI[1] == 10 && g.RI[2] == 8)
    return spread_launch<10, 10, 8, true>((unsigned)offsets.max_i, x, perm, stride, s, s_uniform, offsets,
                                          g, hc, grid, st);
  if (g.C > 1 && g.RI[0] == 6 && g.RI[1] == 6 && g.RI[2] == 8)
    return spread_launch<6, 6, 8, true>((unsigned)offsets.max_i, x, perm, stride, s, s_uniform, offsets,
                                        g, hc, grid, st);
  const unsigned nbr = (unsigned)offsets.max_s;  // upper bound on spread items
#define PIF_SPREAD(A, B, Cz)                                        \
  if (g.RS[0] == A && g.RS[1] == B && g.RS[2] == Cz)                \
    return spread_launch<A, B, Cz>(nbr, x, perm, stride, s, s_uniform, offsets, g, hc, grid, st);
  PIF_SPREAD(8, 8, 8)
  PIF_SPREAD(12, 12, 12)
  PIF_SPREAD(16, 16, 16)
#undef PIF_SPREAD
  return cudaErrorInvalidValue;
}

template <int A, int B, int Cz>
static cudaError_t interp_launch(unsigned nsub, const double* grid3, double* x, double* v,
                                 int64_t stride, const int* id, double* Eout, const Sched& offsets,
                                 const Brick& g, const Horner& hc, const PushArgs& P,
                                 cudaStream_t st) {
  const int T = 32 * (InterpCfg<A, B, Cz>::NW + InterpCfg<A, B, Cz>::NP);
  const size_t smem = sizeof(InterpSmem<A, B, Cz>);
  static DevCache cache;
  int ctas = 0;  // persistent grid: SMs x resident CTAs per SM
  cudaError_t e = dev_cached(cache, ctas, [&](int dev, int& v) {
    int sms = 0, per = 0;
    cudaError_t r = cudaFuncSetAttribute(k_interp_push<A, B, Cz>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (r == cudaSuccess) r = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (r == cudaSuccess)
      r = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_interp_push<A, B, Cz>, T, smem);
    v = sms * per;
    return r;
  });
  if (e != cudaSuccess) return e;
  const unsigned grid = nsub < (unsigned)ctas ? nsub : (unsigned)ctas;
  if (grid == 0) return cudaSuccess;
  k_interp_push<A, B, Cz><<<grid, T, smem, st>>>(grid3, x, v, stride, id, Eout, offsets, g, hc, P);
  return cudaGetLastError();
}

template <int A, int B, int Cz, int BX, int BY, int SBZ, int CSX, int ZR>
static cudaError_t interp_slab_launch(unsigned nsub, const double* grid3, double* x, double* v,
                                      int64_t stride, const int* id, double* Eout,
                                      const Sched& offsets, const Brick& g, const Horner& hc,
                                      const PushArgs& P, cudaStream_t st) {
  using C = SlabCfg<A, B, Cz, BX, BY, SBZ, CSX, ZR>;
  const int T = 32 * (C::NW + 1);
  const size_t smem = sizeof(SlabSmem<A, B, Cz, BX, BY, SBZ, CSX, ZR>);
  static DevCache cache;
  int sms = 0;
  cudaError_t e = dev_cached(cache, sms, [&](int dev, int& v) {
    int n_sm = 0, per = 0;
    cudaError_t r = cudaFuncSetAttribute(k_interp_push_slab<A, B, Cz, BX, BY, SBZ, CSX, ZR>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (r == cudaSuccess) r = cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    if (r == cudaSuccess)
      r = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_interp_push_slab<A, B, Cz, BX, BY, SBZ, CSX, ZR>,
                                                        T, smem);
    v = per >= 1 ? n_sm : 0;
    return r;
  });
  if (e != cudaSuccess) return e;
  // persistent: one CTA per SM, each with a contiguous run of items
  const unsigned grid = nsub < (unsigned)sms ? nsub : (unsigned)sms;
  if (grid == 0) return cudaSuccess;
  k_interp_push_slab<A, B, Cz, BX, BY, SBZ, CSX, ZR><<<grid, T, smem, st>>>(grid3, x, v, stride, id, Eout,
                                                                   offsets, g, hc, P);
  return cudaGetLastError();
}

cudaError_t launch_interp_push(const double* grid3, double* x, double* v, int64_t stride,
                               const int* id, double* Eout, const Sched& offsets, const Brick& g,
                               const Horner& hc, const PushArgs& P, cudaStream_t st) {
  const unsigned nsub = (unsigned)offsets.max_i;  // upper bound on interp items
#ifndef PIF_NO_SLAB
  // slab-ring kernels (column strides CSX from the bank-conflict search)
#define PIF_SLAB(A, B, Cz, BX, BY, SBZ, CSX, ZR)                                                \
  if (g.RI[0] == A && g.RI[1] == B && g.RI[2] == Cz && g.RS[0] == BX && g.RS[1] == BY &&       \
      g.ib[2] == SBZ && g.m[2] == 1 && (g.C == 1 || g.C == g.ib[0] * g.ib[1]))                 \
    return interp_slab_launch<A, B, Cz, BX, BY, SBZ, CSX, ZR>(nsub, grid3, x, v, stride, id, Eout,  \
                                                              offsets, g, hc, P, st);
  PIF_SLAB(14, 14, 16, 16, 16, 4, 17, 0)  // w = 13: ring of 6 slabs without zero rows
  PIF_SLAB(10, 10, 8, 16, 16, 1, 17, 1)   // w = 8, dense
#undef PIF_SLAB
#endif
#define PIF_INTERP(A, B, Cz)                                                                   \
  if (g.RI[0] == A && g.RI[1] == B && g.RI[2] == Cz)                                           \
    return interp_launch<A, B, Cz>(nsub, grid3, x, v, stride, id, Eout, offsets, g, hc, P, st);
  if (g.C != 1) return cudaErrorInvalidValue;  // cell keys need the slab kernel
  PIF_INTERP(12, 12, 12)
  PIF_INTERP(16, 16, 16)
#undef PIF_INTERP
  return cudaErrorInvalidValue;
}

}  // namespace pif
