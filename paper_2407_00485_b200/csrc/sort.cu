// a0: bin particles by brick and counting-sort them physically (SoA x, v, id).
// Not a method step (cuFINUFFT bins internally); it gives the brick
// kernels contiguous, coalesced particle ranges per CTA.
#include "pif_internal.cuh"

namespace pif {

__global__ void k_bin_count(const double* __restrict__ x, int64_t stride, int64_t n, Brick g,
                            int* __restrict__ key, int* __restrict__ rank,
                            int* __restrict__ counts) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  int B[3], S[3], Q[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    double xs = x[d * stride + j] * g.scale;
    int a = anchor_of(xs, g);
    // a / sb, r / ib without the integer-division sequences (Brick::rsb)
    B[d] = (int)(((float)a + 0.5f) * g.rsb[d]);
    const int r = a - B[d] * g.sb[d];
    S[d] = (int)(((float)r + 0.5f) * g.rib[d]);
    Q[d] = r - S[d] * g.ib[d];
  }
  int k = ((B[0] * g.NB[1] + B[1]) * g.NB[2] + B[2]) * (g.m[0] * g.m[1] * g.m[2]) +
          (S[0] * g.m[1] + S[1]) * g.m[2] + S[2];
  // C > 1: xy-cell of the sub-brick, snake order (consecutive cells adjacent)
  if (g.C > 1) k = k * g.C + Q[0] * g.ib[1] + ((Q[0] & 1) ? g.ib[1] - 1 - Q[1] : Q[1]);
  key[j] = k;
  // warp-aggregated rank: one atomic per distinct key in the warp (sorted-ish
  // input and crowded bricks give many equal keys per warp)
  const unsigned act = __activemask();
  const unsigned peers = __match_any_sync(act, k);
  const int leader = __ffs(peers) - 1;
  const int lane = threadIdx.x & 31;
  int base = 0;
  if (lane == leader) base = atomicAdd(&counts[k], __popc(peers));
  base = __shfl_sync(peers, base, leader);
  rank[j] = base + __popc(peers & ((1u << lane) - 1u));
}

// Exclusive scans of (counts, spread items, interp items, interpolation cost)
// over keys, three passes over bricks (one thread = one brick = M consecutive
// keys, blocks of kSchedT bricks): per-block totals, one-CTA scan of the block
// totals, per-block scan + writes.  Interp items cover groups of C consecutive
// keys (one sub-brick; C > 1 when keys are its xy-cells).  offsets[k]: first
// particle of key k; ioff[k] (k a group's first key): first interp item of the
// group; soff[k] (k a brick's first key): first spread item of the brick (other
// keys: the end of their brick's / group's items); moff[k] (group first key):
// interpolation cost before the group, in m-tiles of 8 particles plus
// kBrickCost per non-empty brick (the persistent interpolation kernel balances
// its CTAs' item runs by it); [nkeys] = totals.
constexpr int kQ = 4;  // scanned quantities
// Cost of a non-empty brick's slab loads in the interpolation kernel, in m-tiles
// (sparse regions: one m-tile per brick would otherwise look free)
#ifndef PIF_SLAB_BRICK_COST
#define PIF_SLAB_BRICK_COST 6  // A/B: C4 interp 10.95 -> 10.85 ms vs 12; 3 / 0: 12.7 / 14.5 ms
#endif
constexpr int kBrickCost = PIF_SLAB_BRICK_COST;

__device__ __forceinline__ void brick_sums(const int* __restrict__ counts, int64_t i0, int M,
                                           int C, int a[kQ]) {
  int bs = 0, it = 0, mt = 0;
  for (int m = 0; m < M; m += C) {
    int gc = 0;
    for (int q = 0; q < C; ++q) gc += counts[i0 + m + q];
    bs += gc;
    it += (gc + kInterpItem - 1) / kInterpItem;
    mt += (gc + 7) >> 3;
  }
  a[0] = bs;
  a[1] = (bs + kSpreadItem - 1) / kSpreadItem;
  a[2] = it;
  a[3] = mt + (bs > 0 ? kBrickCost : 0);
}

// Block-wide exclusive scan of kQ ints (blockDim.x == kSchedT); returns the
// block totals in tot.
__device__ __forceinline__ void block_scan(const int a[kQ], int ex[kQ], int tot[kQ]) {
  __shared__ int sh[kQ][kSchedT / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int incl[kQ];
#pragma unroll
  for (int q = 0; q < kQ; ++q) {
    int v = a[q];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += u;
    }
    incl[q] = v;
    if (lane == 31) sh[q][wid] = v;
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < kQ; ++q) {
    int before = 0, all = 0;
#pragma unroll
    for (int w = 0; w < kSchedT / 32; ++w) {
      const int x = sh[q][w];
      if (w < wid) before += x;
      all += x;
    }
    ex[q] = incl[q] - a[q] + before;
    tot[q] = all;
  }
}

__global__ void __launch_bounds__(kSchedT) k_sched_reduce(const int* __restrict__ counts, Sched S,
                                                          int M, int C) {
  const int64_t nb = S.nkeys / M, br = blockIdx.x * (int64_t)kSchedT + threadIdx.x;
  int a[kQ] = {0, 0, 0, 0}, ex[kQ], tot[kQ];
  if (br < nb) brick_sums(counts, br * M, M, C, a);
  block_scan(a, ex, tot);
  if (threadIdx.x == 0)
    for (int q = 0; q < kQ; ++q) S.part[kQ * blockIdx.x + q] = tot[q];
}

// In place: part[kQ b + q] <- sum of part[kQ b' + q] over b' < b (one CTA).
__global__ void __launch_bounds__(1024) k_sched_partials(Sched S, int nblk) {
  __shared__ int sh[kQ][32];
  const int T = blockDim.x, t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int per = (nblk + T - 1) / T, lo = min(nblk, t * per), hi = min(nblk, lo + per);
  int a[kQ] = {0, 0, 0, 0};
  for (int i = lo; i < hi; ++i)
    for (int q = 0; q < kQ; ++q) a[q] += S.part[kQ * i + q];
  int incl[kQ];
#pragma unroll
  for (int q = 0; q < kQ; ++q) {
    int v = a[q];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += u;
    }
    incl[q] = v;
    if (lane == 31) sh[q][wid] = v;
  }
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int q = 0; q < kQ; ++q) {
      int w = lane < (T >> 5) ? sh[q][lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += u;
      }
      sh[q][lane] = w;
    }
  }
  __syncthreads();
  int ex[kQ];
#pragma unroll
  for (int q = 0; q < kQ; ++q) ex[q] = incl[q] - a[q] + (wid > 0 ? sh[q][wid - 1] : 0);
  for (int i = lo; i < hi; ++i)
    for (int q = 0; q < kQ; ++q) {
      const int x = S.part[kQ * i + q];
      S.part[kQ * i + q] = ex[q];
      ex[q] += x;
    }
}

__global__ void __launch_bounds__(kSchedT) k_sched_apply(const int* __restrict__ counts, Sched S,
                                                         int M, int C) {
  const int64_t nk = S.nkeys, nb = nk / M, br = blockIdx.x * (int64_t)kSchedT + threadIdx.x;
  int a[kQ] = {0, 0, 0, 0}, ex[kQ], tot[kQ];
  if (br < nb) brick_sums(counts, br * M, M, C, a);
  block_scan(a, ex, tot);
  if (br >= nb) return;
#pragma unroll
  for (int q = 0; q < kQ; ++q) ex[q] += S.part[kQ * blockIdx.x + q];
  const int64_t i = br * M;
  S.soff[i] = ex[1];
  ex[1] += a[1];
  if (a[0] > 0) ex[3] += kBrickCost;  // before the brick's first item
  for (int m = 0; m < M; m += C) {
    int gc = 0;
    for (int q = 0; q < C; ++q) {
      const int c = counts[i + m + q];
      S.offsets[i + m + q] = ex[0] + gc;
      if (m + q) S.soff[i + m + q] = ex[1];
      gc += c;
    }
    S.ioff[i + m] = ex[2];
    S.moff[i + m] = ex[3];
    ex[0] += gc;
    ex[2] += (gc + kInterpItem - 1) / kInterpItem;
    ex[3] += (gc + 7) >> 3;
    for (int q = 1; q < C; ++q) {
      S.ioff[i + m + q] = ex[2];
      S.moff[i + m + q] = ex[3];
    }
  }
  if (br == nb - 1) {
    S.offsets[nk] = ex[0];
    S.soff[nk] = ex[1];
    S.ioff[nk] = ex[2];
    S.moff[nk] = ex[3];
  }
}

// One thread per key: (first key of a group) the interp items of the group,
// and (first key of a brick) the spread items of the brick.
__global__ void k_schedule_fill(Sched S, Brick g, int M, int C) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= S.nkeys) return;
  const int a = S.offsets[k];
  if (k % C == 0) {
    const int b = S.offsets[k + C];
    int it = S.ioff[k];
    // decoded brick / sub-brick coordinates (the slab kernel's item cursors then
    // need no integer divisions)
    const int Ms = g.m[0] * g.m[1] * g.m[2];
    const int brick = (int)(k / M), sk = (int)((k / C) % Ms);
    const int bz = brick % g.NB[2], by = (brick / g.NB[2]) % g.NB[1], bx = brick / (g.NB[2] * g.NB[1]);
    const int sy = (sk / g.m[2]) % g.m[1], sx = sk / (g.m[2] * g.m[1]);
    const int4 info = make_int4(bx, by, bz, sx | (sy << 16));
    // .w = the item's cost offset (m-tiles, key order)
    for (int s0 = a; s0 < b; s0 += kInterpItem) {
      S.iinfo[it] = info;
      S.iitems[it++] = make_int4((int)k, s0, min(b, s0 + kInterpItem), S.moff[k] + ((s0 - a) >> 3));
    }
  }
  if (k % M == 0) {
    const int e = S.offsets[k + M];
    int si = S.soff[k];
    for (int s0 = a; s0 < e; s0 += kSpreadItem)
      S.sitems[si++] = make_int4((int)(k / M), s0, min(e, s0 + kSpreadItem), 0);
  }
}

// Physical sort by gather: perm[dst] = src (a 4-byte scatter), then every
// array is gathered in destination order -- coalesced writes, and the
// reads stay near-sequential because particles move less than a cell per step
// (the partial-sector writes of a 52-byte-per-particle scatter are avoided).
__global__ void k_scatter_index(int64_t n, const int* __restrict__ key,
                                const int* __restrict__ rank, const int* __restrict__ offsets,
                                int* __restrict__ perm) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  perm[offsets[key[j]] + rank[j]] = (int)j;
}

// v / s (per-particle strengths of the debug type-1 export) may be null.
__global__ void k_gather_sorted(const double* __restrict__ x, const double* __restrict__ v,
                                const int* __restrict__ id, const double* __restrict__ s,
                                int64_t stride, int64_t n, const int* __restrict__ perm,
                                double* __restrict__ x2, double* __restrict__ v2,
                                int* __restrict__ id2, double* __restrict__ s2) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t j = perm[i];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    x2[d * stride + i] = x[d * stride + j];
    if (v) v2[d * stride + i] = v[d * stride + j];
  }
  id2[i] = id[j];
  if (s) s2[i] = s[j];
}

__global__ void k_iota(int* id, int64_t n) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j < n) id[j] = (int)j;
}

// dst (canonical order) <- src (sorted order) by particle id.
__global__ void k_scatter_by_id(const double* __restrict__ x, const double* __restrict__ v,
                                const int* __restrict__ id, int64_t stride, int64_t n,
                                double* __restrict__ xo, double* __restrict__ vo) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  int64_t k = id[j];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    xo[d * stride + k] = x[d * stride + j];
    vo[d * stride + k] = v[d * stride + j];
  }
}

static inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

cudaError_t launch_bin_count(const double* x, int64_t stride, int64_t n, const Brick& g, int* key,
                             int* rank, int* counts, cudaStream_t st) {
  if (n > 0) k_bin_count<<<nblk(n, 256), 256, 0, st>>>(x, stride, n, g, key, rank, counts);
  return cudaGetLastError();
}
cudaError_t launch_schedule(const int* counts, const Sched& S, const Brick& g, int M, int C,
                            cudaStream_t st) {
  const unsigned nsb = nblk_sched(S.nkeys, M);
  k_sched_reduce<<<nsb, kSchedT, 0, st>>>(counts, S, M, C);
  k_sched_partials<<<1, 1024, 0, st>>>(S, (int)nsb);
  k_sched_apply<<<nsb, kSchedT, 0, st>>>(counts, S, M, C);
  k_schedule_fill<<<nblk(S.nkeys, 256), 256, 0, st>>>(S, g, M, C);
  return cudaGetLastError();
}
cudaError_t launch_gather_sorted(const double* x, const double* v, const int* id, const double* s,
                                 int64_t stride, int64_t n, const int* key, const int* rank,
                                 const int* offsets, int* perm, double* x2, double* v2, int* id2,
                                 double* s2, cudaStream_t st) {
  if (n > 0) {
    k_scatter_index<<<nblk(n, 256), 256, 0, st>>>(n, key, rank, offsets, perm);
    k_gather_sorted<<<nblk(n, 256), 256, 0, st>>>(x, v, id, s, stride, n, perm, x2, v2, id2, s2);
  }
  return cudaGetLastError();
}
cudaError_t launch_scatter_index(int64_t n, const int* key, const int* rank, const int* offsets,
                                 int* perm, cudaStream_t st) {
  if (n > 0) k_scatter_index<<<nblk(n, 256), 256, 0, st>>>(n, key, rank, offsets, perm);
  return cudaGetLastError();
}
cudaError_t launch_iota(int* id, int64_t n, cudaStream_t st) {
  if (n > 0) k_iota<<<nblk(n, 256), 256, 0, st>>>(id, n);
  return cudaGetLastError();
}
cudaError_t launch_scatter_by_id(const double* x, const double* v, const int* id, int64_t stride,
                                 int64_t n, double* xo, double* vo, cudaStream_t st) {
  if (n > 0) k_scatter_by_id<<<nblk(n, 256), 256, 0, st>>>(x, v, id, stride, n, xo, vo);
  return cudaGetLastError();
}

}  // namespace pif
