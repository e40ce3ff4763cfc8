// bl_attr.cuh -- step a5 of SURVEY.md §8(a) on its own: the CSR attraction
// plus neighbour correction S_i = sum_{j in N(i)} (d^(a-1)/K + C K^2 d^(r-1))
// Δ_ij (§2.2; the if/else of Alg. 2, reading C2) for a
// range of vertices (bl_forces with BL_ATTRACTION_ONLY), and
// the same CSR walk for the edge-uniformity metric (§3.7).
//
// The work is L2 gathers (4 B colidx + 8 B coordinate per CSR entry) over a
// degree distribution from 0 to ~16k (C5: 81 % of the rows have <= 8
// entries, 74 % of the entries are in rows of > 64), so the rows are cut by
// degree class (bla_kernel) into warp items that each keep 8 loads per lane
// in flight.  Every sum has a fixed order: bitwise-reproducible results.
#pragma once
#include "bl_kernel.cuh"
#include "bl_rows.h"

#define BLA_NT 256
#define BLA_LONG 64     // rows above this many entries are cut into chunks
#define BLA_CHUNK 256   // entries per long-row chunk (8 per lane)

// COO row ids of the CSR entries (row[k] = i for rowptr[i] <= k < rowptr[i+1])
// -- kept for the stress / NP metrics' host helpers
__global__ void bla_coo_rows(const int *rowptr, int n, int *row) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    for (int k = rowptr[i]; k < rowptr[i + 1]; ++k) row[k] = i;
}


// attraction coefficient x Δ for one entry (reading C15), fp32 as the layout
template <bool FAST>
__device__ __forceinline__ void bla_term(const BLKParams &p, float2 ci, float2 cj, float rep,
                                         float &sx, float &sy) {
  const float dx = cj.x - ci.x, dy = cj.y - ci.y;
  const float d2 = fmaf(dx, dx, fmaf(dy, dy, BL_EPS2));
  const float rs = bl_rsqrt(d2);
  const float coef = bl_model_coef<FAST>(p, d2, rs, rep);
  sx = fmaf(coef, dx, sx);
  sy = fmaf(coef, dy, sy);
}

// a5 alone over [p.first, p.first + p.count): f_out[v - first] = S_v.
// Items (one warp each), from degree classes built once per context:
//   class 1 (deg <= 8):   32 rows per item, one lane per row, its <= 8
//                         entries loaded before any is used;
//   class 2 (9..64):      4 rows per item, 8 lanes per row (<= 8 entries per
//                         lane), fixed 3-step butterfly;
//   long rows (> 64):     one 256-entry chunk per item, lane-strided, warp
//                         butterfly -> lpart[chunk]; after a grid barrier a
//                         warp per long row adds its chunks (lane-strided,
//                         butterfly: a fixed order; one fence per block, not
//                         per chunk).
// Rows outside the range are skipped.
#define BLA_BPS 5  // blocks per SM (co-resident: the cooperative launch)
template <bool FAST>
__global__ void __launch_bounds__(BLA_NT, BLA_BPS)
    bla_kernel(BLKParams p, const int *__restrict__ cls1, int n1, const int *__restrict__ cls2,
               int n2, const BLAChunk *__restrict__ chunks, int nchunks, float2 *lpart,
               const int2 *__restrict__ lrow, int nlong, unsigned *bar, unsigned bar_target) {
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * BLA_NT) >> 5;
  const int w0 = (blockIdx.x * BLA_NT + threadIdx.x) >> 5;
  const float rep = (p.flags & 1u) ? 0.f : p.ck2;
  const int lo = p.first, hi = p.first + p.count;
  const int g1 = (n1 + 31) >> 5, g2 = (n2 + 3) >> 2;
  const float2 *__restrict__ xy = p.xy;
  for (int item = w0; item < g1 + g2 + nchunks; item += nw) {
    if (item < g1) {
      const int r = item * 32 + lane;
      const int v = r < n1 ? __ldg(cls1 + r) : -1;
      const bool mine = v >= lo && v < hi;
      int k0 = 0, deg = 0;
      if (mine) {
        k0 = __ldg(p.rowptr + v);
        deg = __ldg(p.rowptr + v + 1) - k0;
      }
      int j[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) j[u] = u < deg ? __ldg(p.colidx + k0 + u) : -1;
      const float2 ci = mine ? __ldg(xy + v) : make_float2(0.f, 0.f);
      float2 cj[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) cj[u] = j[u] >= 0 ? __ldg(xy + j[u]) : ci;
      float sx = 0.f, sy = 0.f;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (j[u] >= 0) bla_term<FAST>(p, ci, cj[u], rep, sx, sy);
      if (mine) p.f_out[v - lo] = make_float2(sx, sy);
    } else if (item < g1 + g2) {
      const int sl = lane & 7;
      const int r = (item - g1) * 4 + (lane >> 3);
      const int v = r < n2 ? __ldg(cls2 + r) : -1;
      const bool mine = v >= lo && v < hi;
      int k0 = 0, deg = 0;
      if (mine) {
        k0 = __ldg(p.rowptr + v);
        deg = __ldg(p.rowptr + v + 1) - k0;
      }
      int j[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = sl + 8 * u;
        j[u] = e < deg ? __ldg(p.colidx + k0 + e) : -1;
      }
      const float2 ci = mine ? __ldg(xy + v) : make_float2(0.f, 0.f);
      float2 cj[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) cj[u] = j[u] >= 0 ? __ldg(xy + j[u]) : ci;
      float sx = 0.f, sy = 0.f;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (j[u] >= 0) bla_term<FAST>(p, ci, cj[u], rep, sx, sy);
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) {
        sx += __shfl_xor_sync(0xffffffffu, sx, o);
        sy += __shfl_xor_sync(0xffffffffu, sy, o);
      }
      if (mine && sl == 0) p.f_out[v - lo] = make_float2(sx, sy);
    } else {
      const int c = item - g1 - g2;
      const BLAChunk ch = chunks[c];
      if (ch.v < lo || ch.v >= hi) continue;
      int j[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int k = ch.k0 + lane + 32 * u;
        j[u] = k < ch.k1 ? __ldg(p.colidx + k) : -1;
      }
      const float2 ci = __ldg(xy + ch.v);
      float2 cj[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) cj[u] = j[u] >= 0 ? __ldg(xy + j[u]) : ci;
      float sx = 0.f, sy = 0.f;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (j[u] >= 0) bla_term<FAST>(p, ci, cj[u], rep, sx, sy);
      sx = bl_warp_sum0(sx);
      sy = bl_warp_sum0(sy);
      if (lane == 0) lpart[c] = make_float2(sx, sy);
    }
  }
  if (nlong == 0) return;
  // grid barrier (cooperative launch; monotone counter, target from the
  // host), then one warp per long row: its chunk partials in a fixed order
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("fence.acq_rel.gpu;\n\tred.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    while ((int)(bl_ld_acquire(bar) - bar_target) < 0) {
    }
  }
  __syncthreads();
  for (int li = w0; li < nlong; li += nw) {
    const int2 lr = lrow[li];
    const int v = chunks[lr.x].v;
    if (v < lo || v >= hi) continue;
    float tx = 0.f, ty = 0.f;
    for (int c = lane; c < lr.y; c += 32) {
      const float2 q = __ldcg(lpart + lr.x + c);
      tx += q.x;
      ty += q.y;
    }
    tx = bl_warp_sum0(tx);
    ty = bl_warp_sum0(ty);
    if (lane == 0) p.f_out[v - lo] = make_float2(tx, ty);
  }
}

// Edge uniformity (§3.7; M2) in ONE pass: each undirected edge once (j > i),
// the rows cut into warp items by degree class as in bla_kernel, fp64
// lengths of the fp32 coordinates folded into a
// per-lane shifted sums (shift K = the lane's first length: S = sum (l - K),
// Q = sum (l - K)^2, no division per edge) turned into a (count, mean, M2)
// state once, merged by Chan's formula in a fixed order (warp butterfly, a
// tree over the warps, a tree over the blocks in bla_eu_final): EU =
// sqrt(M2 / m) / mean (the two-pass oracle's value to rounding).  Bitwise
// reproducible (fixed grid, fixed merge order).
struct BLAWelford {
  double n, mean, m2;
};
__device__ __forceinline__ BLAWelford bla_merge(BLAWelford a, BLAWelford b) {
  if (b.n == 0.0) return a;
  if (a.n == 0.0) return b;
  const double n = a.n + b.n, d = b.mean - a.mean;
  BLAWelford r;
  r.n = n;
  r.mean = a.mean + d * (b.n / n);
  r.m2 = a.m2 + b.m2 + d * d * (a.n * b.n / n);
  return r;
}

__device__ __forceinline__ void bla_eu_edge(float2 ci, float2 cj, double &cnt, double &K,
                                            double &S, double &Q) {
  const double dx = (double)cj.x - (double)ci.x, dy = (double)cj.y - (double)ci.y;
  const double l = sqrt(dx * dx + dy * dy);
  if (cnt == 0.0) K = l;
  cnt += 1.0;
  const double d = l - K;
  S += d;
  Q += d * d;
}

// the rows cut by degree class as bla_kernel; each undirected edge once (j > v)
__device__ __forceinline__ BLAWelford bla_block_merge(BLAWelford w, double *shw);

__global__ void __launch_bounds__(BLA_NT, BLA_BPS)
    bla_eu_kernel(const int *__restrict__ rowptr, const int *__restrict__ colidx,
                  const float2 *__restrict__ xy, const int *__restrict__ cls1, int n1,
                  const int *__restrict__ cls2, int n2, const BLAChunk *__restrict__ chunks,
                  int nchunks, double *part, unsigned *done, double *stats) {
  __shared__ double shw[3 * (BLA_NT / 32)];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = (gridDim.x * BLA_NT) >> 5;
  const int w0 = (blockIdx.x * BLA_NT + threadIdx.x) >> 5;
  const int g1 = (n1 + 31) >> 5, g2 = (n2 + 3) >> 2;
  double cnt = 0.0, K = 0.0, S = 0.0, Q = 0.0;
  for (int item = w0; item < g1 + g2 + nchunks; item += nw) {
    int v = -1, kb = 0, ke = 0, step = 1;
    if (item < g1) {
      const int r = item * 32 + lane;
      if (r < n1) {
        v = __ldg(cls1 + r);
        kb = __ldg(rowptr + v);
        ke = __ldg(rowptr + v + 1);
      }
    } else if (item < g1 + g2) {
      const int r = (item - g1) * 4 + (lane >> 3);
      if (r < n2) {
        v = __ldg(cls2 + r);
        kb = __ldg(rowptr + v) + (lane & 7);
        ke = __ldg(rowptr + v + 1);
      }
      step = 8;
    } else {
      const BLAChunk ch = chunks[item - g1 - g2];
      v = ch.v;
      kb = ch.k0 + lane;
      ke = ch.k1;
      step = 32;
    }
    int j[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int k = kb + step * u;
      j[u] = k < ke ? __ldg(colidx + k) : -1;
      if (j[u] <= v) j[u] = -1;  // each undirected edge once
    }
    const float2 ci = v >= 0 ? __ldg(xy + v) : make_float2(0.f, 0.f);
    float2 cj[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) cj[u] = j[u] >= 0 ? __ldg(xy + j[u]) : ci;
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (j[u] >= 0) bla_eu_edge(ci, cj[u], cnt, K, S, Q);
  }
  BLAWelford w = {0.0, 0.0, 0.0};
  if (cnt > 0.0) {
    w.n = cnt;
    w.mean = K + S / cnt;
    w.m2 = fmax(0.0, Q - S * (S / cnt));
  }
  const BLAWelford a = bla_block_merge(w, shw);
  __shared__ int last;
  if (threadIdx.x == 0) {
    part[3 * blockIdx.x] = a.n;
    part[3 * blockIdx.x + 1] = a.mean;
    part[3 * blockIdx.x + 2] = a.m2;
    __threadfence();
    last = atomicAdd(done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  // the last block: the per-block states, thread t over blocks t, t + NT, ...
  // in order, then the same fixed block merge; resets the counter
  __threadfence();
  BLAWelford b = {0.0, 0.0, 0.0};
  for (int k = threadIdx.x; k < (int)gridDim.x; k += BLA_NT)
    b = bla_merge(b, {__ldcg(part + 3 * k), __ldcg(part + 3 * k + 1), __ldcg(part + 3 * k + 2)});
  const BLAWelford r = bla_block_merge(b, shw);
  if (threadIdx.x == 0) {
    stats[0] = r.n;
    stats[1] = r.mean;
    stats[2] = r.m2;
    stats[4] = (r.n > 0.0 && r.mean > 0.0) ? sqrt(r.m2 / r.n) / r.mean : 0.0;
    *done = 0u;
  }
}

// fixed-order block merge of per-thread states: warp butterfly (lane 0's
// result is deterministic), then a tree over the warps; valid on thread 0
__device__ __forceinline__ BLAWelford bla_block_merge(BLAWelford w, double *shw) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    BLAWelford b;
    b.n = __shfl_xor_sync(0xffffffffu, w.n, o);
    b.mean = __shfl_xor_sync(0xffffffffu, w.mean, o);
    b.m2 = __shfl_xor_sync(0xffffffffu, w.m2, o);
    w = lane < (lane ^ o) ? bla_merge(w, b) : bla_merge(b, w);
  }
  __syncthreads();
  if (lane == 0) {
    shw[3 * warp] = w.n;
    shw[3 * warp + 1] = w.mean;
    shw[3 * warp + 2] = w.m2;
  }
  __syncthreads();
  BLAWelford a = {0.0, 0.0, 0.0};
  if (threadIdx.x < 32) {
    const int k = lane < BLA_NT / 32 ? lane : 0;
    if (lane < BLA_NT / 32) a = {shw[3 * k], shw[3 * k + 1], shw[3 * k + 2]};
#pragma unroll
    for (int o = 1; o < BLA_NT / 32; o <<= 1) {
      BLAWelford b;
      b.n = __shfl_down_sync(0xffffffffu, a.n, o);
      b.mean = __shfl_down_sync(0xffffffffu, a.mean, o);
      b.m2 = __shfl_down_sync(0xffffffffu, a.m2, o);
      if ((lane & (2 * o - 1)) == 0) a = bla_merge(a, b);
    }
  }
  return a;
}

