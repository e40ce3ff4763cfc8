// bl_metrics.cuh -- the layout quality metrics of §3.7
// on sm_100a (device side; readings M1-M4 of DESIGN.md §3).
//
//   edge uniformity (M2): one entry-parallel pass over the CSR (edges i < j
//     once; bla_eu_kernel in bl_attr.cuh), fp64 per-lane Welford states
//     merged in a fixed order;
//   stress (M1): multi-source BFS, 256 sources per group as one 256-bit
//     mask per vertex, pull-based levels inside ONE cooperative kernel over
//     the degree classes of bla_kernel (grid barrier per level); every newly
//     reached (source, vertex) pair at hop distance L adds |D|/L and
//     |D|^2/L^2 to fp64 accumulators, so the scale-optimised stress comes out
//     in closed form (s* = A/B, ST = s*^2 B - 2 s* A + N) without storing a
//     distance matrix;
//   neighbourhood preservation (M3): queries with kk = min(deg, n-1) <= 256
//     (bln_np_fast): one scan of all vertices per warp for 8 (kk <= 32) or 2
//     queries, a shared-memory candidate buffer per query behind a threshold
//     on the (d2 bits, id) key; larger kk (blm_np_kernel): one CTA per query,
//     radix select (4 x 8-bit passes, warp-aggregated shared-memory
//     histograms) of the kk-th smallest fp32 squared distance, ties resolved
//     by vertex id with a second select over ids; then the Jaccard of N(i)
//     with the layout-nearest set.
// All reductions have a fixed order: results are bitwise reproducible.
#pragma once
#include "bl_kernel.cuh"
#include "bl_rows.h"

#define BLM_NT 256
#define BLM_NW (BLM_NT / 32)

// fixed-order block sum of a double (warp butterfly, then warps in order)
__device__ __forceinline__ double blm_block_sum(double v, double *sh_warp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) sh_warp[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sh_warp[w];
  return s;  // valid on thread 0
}

// ---------------------------------------------------------------- EU (M2)
// One entry-parallel pass with per-lane Welford states (bla_eu_kernel and
// bla_eu_final in bl_attr.cuh).

// Fixed-order sum of x[0..count) by ONE block of BLM_RT threads: thread t
// sums x[t], x[t + BLM_RT], ... in order, then a fixed pairwise tree in
// shared memory -- parallel (no single-thread loop over thousands of
// partials: that cost 37 us per EU pass) and bitwise reproducible.
#define BLM_RT 1024
template <typename V>
__device__ __forceinline__ V blm_fixed_sum(const V *x, long long count, V *sh) {
  V a = V(0);
  for (long long i = threadIdx.x; i < count; i += BLM_RT) a += x[i];
  sh[threadIdx.x] = a;
  __syncthreads();
  for (int w = BLM_RT / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  const V r = sh[0];
  __syncthreads();
  return r;
}

// stats[pass * 2 + {0, 1}] = fixed-order sums over the parts; after pass 1,
// stats[4] = EU = sqrt(sum (l - mu)^2 / (|E| mu^2))
__global__ void __launch_bounds__(BLM_RT) blm_reduce_parts(const double2 *part, int nparts,
                                                           double *stats, int pass) {
  __shared__ double sh[BLM_RT];
  double s = 0.0, c = 0.0;
  {
    double a = 0.0, b = 0.0;
    for (int i = threadIdx.x; i < nparts; i += BLM_RT) {
      a += part[i].x;
      b += part[i].y;
    }
    sh[threadIdx.x] = a;
    __syncthreads();
    for (int w = BLM_RT / 2; w > 0; w >>= 1) {
      if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
      __syncthreads();
    }
    s = sh[0];
    __syncthreads();
    sh[threadIdx.x] = b;
    __syncthreads();
    for (int w = BLM_RT / 2; w > 0; w >>= 1) {
      if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
      __syncthreads();
    }
    c = sh[0];
  }
  if (threadIdx.x == 0) {
    stats[2 * pass] = s;
    stats[2 * pass + 1] = c;
    if (pass == 1) {
      const double m = stats[1], mu = m > 0.0 ? stats[0] / m : 0.0;
      stats[4] = (m > 0.0 && mu > 0.0) ? sqrt(s / (m * mu * mu)) : 0.0;
    }
  }
}

// ---------------------------------------------------------------- stress (M1)
// Multi-source BFS, BLM_SW x 64 = 256 sources per group: one 256-bit mask per
// vertex (vis, and the frontiers cur / nxt), pull-based levels inside ONE
// cooperative kernel.  A level walks the rows by the degree classes of
// bla_kernel (bl_attr.cuh; built once per context): class 1 (deg <= 8) one
// lane per row, class 2 (9..64) 8 lanes per row (OR butterfly), long rows in
// 256-entry warp chunks whose OR partials are combined by one warp per long
// row after a mid-level grid barrier.  A row whose vertex has already been
// reached from every source of the group is skipped.  Every gather is one
// 256-bit load (one 32 B sector).  OR is exact in any order; the fp64 pair
// terms of each newly reached (source, vertex) are added by a fixed thread in
// a fixed order (words, then bits ascending), so the result is bitwise
// reproducible.
#define BLM_SW 4
#define BLM_GS (64 * BLM_SW)
struct BLMStressParams {
  int n, nsrc;
  const int *rowptr, *colidx;
  const float2 *xy;
  const int *sources;   // [nsrc] (device)
  unsigned long long *vis, *frontA, *frontB;  // [n * BLM_SW]
  unsigned long long *lmask;                  // [nchunks * BLM_SW] long-row chunk ORs
  const int *cls1, *cls2;
  int n1, n2, nchunks, nlong;
  const BLAChunk *chunks;
  const int2 *lrow;
  double *accA, *accB;  // [G * NT] per-thread partials (fixed mapping)
  unsigned long long *accN;
  int *flag;            // [3] per-level 'new pairs' flags, rotating
  unsigned *bar;
  unsigned long long *work;  // [G * NT] CSR entries examined per thread; [G * NT] levels
};

struct BLMMask {
  unsigned long long w[BLM_SW];
};
__device__ __forceinline__ BLMMask blm_ld(const unsigned long long *p) {
  BLMMask m;
  asm volatile("ld.global.cg.v4.u64 {%0,%1,%2,%3}, [%4];"
               : "=l"(m.w[0]), "=l"(m.w[1]), "=l"(m.w[2]), "=l"(m.w[3])
               : "l"(p));
  return m;
}
__device__ __forceinline__ void blm_st(unsigned long long *p, const BLMMask &m) {
  asm volatile("st.global.cg.v4.u64 [%0], {%1,%2,%3,%4};" ::"l"(p), "l"(m.w[0]), "l"(m.w[1]),
               "l"(m.w[2]), "l"(m.w[3])
               : "memory");
}
__device__ __forceinline__ bool blm_is_full(const BLMMask &v, const BLMMask &full) {
  bool f = true;
#pragma unroll
  for (int w = 0; w < BLM_SW; ++w) f &= v.w[w] == full.w[w];
  return f;
}
__device__ __forceinline__ void blm_or(BLMMask &a, const BLMMask &b) {
#pragma unroll
  for (int w = 0; w < BLM_SW; ++w) a.w[w] |= b.w[w];
}
// acc |= cur[j[u]] for the valid entries, two rounds of 4 loads in flight
__device__ __forceinline__ void blm_gather8(const unsigned long long *cur, const int *j, BLMMask &acc) {
#pragma unroll
  for (int h = 0; h < 8; h += 4) {
    BLMMask m[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (j[h + u] >= 0) m[u] = blm_ld(cur + (size_t)j[h + u] * BLM_SW);
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (j[h + u] >= 0) blm_or(acc, m[u]);
  }
}
// OR over the lanes of groups of `width` lanes (butterfly; exact)
__device__ __forceinline__ void blm_or_lanes(BLMMask &a, int width) {
  for (int o = width >> 1; o > 0; o >>= 1)
#pragma unroll
    for (int w = 0; w < BLM_SW; ++w) a.w[w] |= __shfl_xor_sync(0xffffffffu, a.w[w], o);
}
// the pair terms of the newly reached (source, v) pairs in word w of nb
__device__ __forceinline__ void blm_pairs(unsigned long long m, int w, float2 cv, double invL,
                                          const float2 *src_xy, double &A, double &B,
                                          unsigned long long &N) {
  while (m) {  // bits in increasing order: fixed accumulation order
    const int k = 64 * w + __ffsll((long long)m) - 1;
    m &= m - 1ull;
    const double dx = (double)cv.x - (double)src_xy[k].x;
    const double dy = (double)cv.y - (double)src_xy[k].y;
    const double l2 = dx * dx + dy * dy;
    A += sqrt(l2) * invL;
    B += l2 * invL * invL;
    ++N;
  }
}

__global__ void __launch_bounds__(BLM_NT, 2) blm_stress_kernel(BLMStressParams p) {
  __shared__ float2 src_xy[BLM_GS];
  __shared__ int unit_dummy;
  const int G = gridDim.x, tid = blockIdx.x * BLM_NT + threadIdx.x, GT = G * BLM_NT;
  const int lane = threadIdx.x & 31;
  const int nw = GT >> 5, w0 = tid >> 5;
  const int g1 = (p.n1 + 31) >> 5, g2 = (p.n2 + 3) >> 2, nitems = g1 + g2 + p.nchunks;
  unsigned bar_target = 0;
  double A = 0.0, B = 0.0;
  unsigned long long N = 0, examined = 0, levels = 0;
  for (int g0 = 0; g0 < p.nsrc; g0 += BLM_GS) {
    const int gs = min(BLM_GS, p.nsrc - g0);
    // init the group: no vertex visited except the sources
    const BLMMask zero = {};
    for (int v = tid; v < p.n; v += GT) {
      blm_st(p.vis + (size_t)v * BLM_SW, zero);
      blm_st(p.frontA + (size_t)v * BLM_SW, zero);
    }
    for (int t = threadIdx.x; t < BLM_GS; t += BLM_NT)
      src_xy[t] = t < gs ? p.xy[p.sources[g0 + t]] : make_float2(0.f, 0.f);
    if (tid == 0) p.flag[0] = p.flag[1] = p.flag[2] = 0;
    bl_grid_sync(p.bar, bar_target, &unit_dummy);
    if (tid < gs) {
      const int s = p.sources[g0 + tid];
      atomicOr(p.vis + (size_t)s * BLM_SW + (tid >> 6), 1ull << (tid & 63));
      atomicOr(p.frontA + (size_t)s * BLM_SW + (tid >> 6), 1ull << (tid & 63));
    }
    bl_grid_sync(p.bar, bar_target, &unit_dummy);
    BLMMask full;
#pragma unroll
    for (int w = 0; w < BLM_SW; ++w) {
      const int bits = min(64, max(0, gs - 64 * w));
      full.w[w] = bits == 64 ? ~0ull : ((1ull << bits) - 1ull);
    }
    unsigned long long *cur = p.frontA, *nxt = p.frontB;
    for (int L = 1;; ++L) {
      const double invL = 1.0 / (double)L;
      bool any = false;
      for (int item = w0; item < nitems; item += nw) {
        if (item < g1 + g2) {
          // class 1: one lane per row (sub = 0, width 1); class 2: 8 lanes
          // per row, sub-lane sub takes entries sub, sub + 8, ...
          const bool c1 = item < g1;
          const int r = c1 ? item * 32 + lane : (item - g1) * 4 + (lane >> 3);
          const int sub = c1 ? 0 : (lane & 7), stp = c1 ? 1 : 8;
          const int v = c1 ? (r < p.n1 ? __ldg(p.cls1 + r) : -1) : (r < p.n2 ? __ldg(p.cls2 + r) : -1);
          BLMMask vv = full, acc = {};
          int deg = 0, k0 = 0;
          if (v >= 0) {
            vv = blm_ld(p.vis + (size_t)v * BLM_SW);
            if (!blm_is_full(vv, full)) {
              k0 = __ldg(p.rowptr + v);
              deg = __ldg(p.rowptr + v + 1) - k0;
            }
          }
          int j[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int e = sub + stp * u;
            j[u] = e < deg ? __ldg(p.colidx + k0 + e) : -1;
          }
          blm_gather8(cur, j, acc);
          if (sub == 0) examined += (unsigned long long)deg;
          if (!c1) blm_or_lanes(acc, 8);
          if (v >= 0 && sub == 0) {
            BLMMask nb;
            bool hit = false;
#pragma unroll
            for (int w = 0; w < BLM_SW; ++w) {
              nb.w[w] = acc.w[w] & ~vv.w[w];
              hit |= nb.w[w] != 0ull;
            }
            blm_st(nxt + (size_t)v * BLM_SW, nb);
            if (hit) {
              BLMMask nv;
#pragma unroll
              for (int w = 0; w < BLM_SW; ++w) nv.w[w] = vv.w[w] | nb.w[w];
              blm_st(p.vis + (size_t)v * BLM_SW, nv);
              any = true;
              const float2 cv = p.xy[v];
#pragma unroll
              for (int w = 0; w < BLM_SW; ++w) blm_pairs(nb.w[w], w, cv, invL, src_xy, A, B, N);
            }
          }
        } else {
          // a long-row chunk: OR of its <= 256 entries -> lmask[c]
          const int c = item - g1 - g2;
          const BLAChunk ch = p.chunks[c];
          const BLMMask vv = blm_ld(p.vis + (size_t)ch.v * BLM_SW);
          BLMMask acc = {};
          if (!blm_is_full(vv, full)) {
            int j[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const int k = ch.k0 + lane + 32 * u;
              j[u] = k < ch.k1 ? __ldg(p.colidx + k) : -1;
            }
            blm_gather8(cur, j, acc);
            if (lane == 0) examined += (unsigned long long)(ch.k1 - ch.k0);
            blm_or_lanes(acc, 32);
          }
          if (lane == 0) blm_st(p.lmask + (size_t)c * BLM_SW, acc);
        }
      }
      if (p.nlong > 0) {
        // the long rows: one warp each ORs its chunk partials, lanes 0..3
        // take one word of the newly reached set each
        bl_grid_sync(p.bar, bar_target, &unit_dummy);
        for (int li = w0; li < p.nlong; li += nw) {
          const int2 lr = p.lrow[li];
          const int v = p.chunks[lr.x].v;
          BLMMask acc = {};
          for (int c = lane; c < lr.y; c += 32) blm_or(acc, blm_ld(p.lmask + (size_t)(lr.x + c) * BLM_SW));
          blm_or_lanes(acc, 32);
          const BLMMask vv = blm_ld(p.vis + (size_t)v * BLM_SW);
          BLMMask nb;
          bool hit = false;
#pragma unroll
          for (int w = 0; w < BLM_SW; ++w) {
            nb.w[w] = acc.w[w] & ~vv.w[w];
            hit |= nb.w[w] != 0ull;
          }
          __syncwarp();
          if (lane == 0) {
            blm_st(nxt + (size_t)v * BLM_SW, nb);
            if (hit) {
              BLMMask nv;
#pragma unroll
              for (int w = 0; w < BLM_SW; ++w) nv.w[w] = vv.w[w] | nb.w[w];
              blm_st(p.vis + (size_t)v * BLM_SW, nv);
            }
          }
          if (hit && lane < BLM_SW) {
            any = true;
            const float2 cv = p.xy[v];
            unsigned long long mw = 0ull;
#pragma unroll
            for (int w = 0; w < BLM_SW; ++w)
              if (w == lane) mw = nb.w[w];
            blm_pairs(mw, lane, cv, invL, src_xy, A, B, N);
          }
        }
      }
      if (any) p.flag[L % 3] = 1;
      // slot (L+1)%3 was last read after barrier L-2: everyone is past it
      if (tid == 0) p.flag[(L + 1) % 3] = 0;
      ++levels;
      bl_grid_sync(p.bar, bar_target, &unit_dummy);
      const int more = __ldcg(p.flag + (L % 3));
      unsigned long long *t = cur;
      cur = nxt;
      nxt = t;
      if (!more) break;
    }
    bl_grid_sync(p.bar, bar_target, &unit_dummy);  // before the next group rewrites vis
  }
  p.accA[tid] = A;
  p.accB[tid] = B;
  p.accN[tid] = N;
  p.work[tid] = examined;
  if (tid == 0) p.work[GT] = levels;
}

// final fixed-order sums of the per-thread partials and the closed form of
// the scale-optimised stress (M1): out4 = (ST, s*, A, B), outN = pairs
__global__ void __launch_bounds__(BLM_RT) blm_stress_reduce(
    const double *accA, const double *accB, const unsigned long long *accN,
    const unsigned long long *work, int count, double *out4, unsigned long long *outN) {
  __shared__ double shd[BLM_RT];
  __shared__ unsigned long long shu[BLM_RT];
  const double A = blm_fixed_sum(accA, count, shd);
  const double B = blm_fixed_sum(accB, count, shd);
  const unsigned long long N = blm_fixed_sum(accN, count, shu);
  const unsigned long long W = blm_fixed_sum(work, count, shu);
  if (threadIdx.x == 0) {
    outN[1] = W;            // CSR entries examined (all groups, all levels)
    outN[2] = work[count];  // BFS levels (all groups)
    const double sc = B > 0.0 ? A / B : 0.0;
    out4[0] = sc * sc * B - 2.0 * sc * A + (double)N;
    out4[1] = sc;
    out4[2] = A;
    out4[3] = B;
    *outN = N;
  }
}

// ---------------------------------------------------------------- NP (M3)
__device__ __forceinline__ unsigned blm_d2bits(float2 a, float2 b) {
  const float dx = __fsub_rn(b.x, a.x), dy = __fsub_rn(b.y, a.y);
  return __float_as_uint(__fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy)));  // >= 0: order-preserving
}

// Radix select over the keys of the n-1 other vertices: returns the k-th
// smallest (1-based) value of key(l) = (byte pass order) where key is the
// d2 bits (mode 0) or the vertex id among those with d2 bits == tau (mode 1).
// *below receives how many keys are smaller than the result.
__device__ unsigned blm_select(const float2 *xy, int n, int i, float2 ci, int k, int mode,
                               unsigned tau, unsigned *hist, unsigned *shv, unsigned *below) {
  const int lane = threadIdx.x & 31;
  unsigned prefix = 0, pmask = 0;
  int need = k;  // rank within the current candidate set
  unsigned less = 0;
  for (int pass = 3; pass >= 0; --pass) {
    const int sft = 8 * pass;
    for (int d = threadIdx.x; d < 256; d += blockDim.x) hist[d] = 0;
    __syncthreads();
    for (int l0 = 0; l0 < n; l0 += blockDim.x) {
      const int l = l0 + threadIdx.x;
      bool act = false;
      unsigned key = 0;
      if (l < n && l != i) {
        const unsigned d2 = blm_d2bits(ci, xy[l]);
        if (mode == 0) {
          key = d2;
          act = true;
        } else if (d2 == tau) {
          key = (unsigned)l;
          act = true;
        }
        if (act && (key & pmask) != prefix) act = false;
      }
      const unsigned am = __ballot_sync(0xffffffffu, act);
      if (act) {
        const unsigned dig = (key >> sft) & 255u;
        const unsigned peers = __match_any_sync(am, dig);
        if ((peers & ((1u << lane) - 1u)) == 0u) atomicAdd(&hist[dig], __popc(peers));
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned acc = 0, d = 0;
      for (; d < 256; ++d) {
        if (acc + hist[d] >= (unsigned)need) break;
        acc += hist[d];
      }
      shv[0] = d;
      shv[1] = acc;
    }
    __syncthreads();
    const unsigned d = shv[0];
    need -= (int)shv[1];
    less += shv[1];
    prefix |= d << sft;
    pmask |= 255u << sft;
    __syncthreads();
  }
  *below = less;
  return prefix;
}

__global__ void __launch_bounds__(512, 1) blm_np_kernel(const int *rowptr, const int *colidx,
                                                        const float2 *xy, int n, const int *queries,
                                                        const int *slots, int nq, double *jac) {
  __shared__ unsigned hist[256];
  __shared__ unsigned shv[2];
  __shared__ int sh_m[16];
  for (int tt = blockIdx.x; tt < nq; tt += gridDim.x) {
    const int t = slots[tt];  // the query's index in the caller's list
    const int i = queries ? queries[t] : t;
    const int k = rowptr[i + 1] - rowptr[i];
    if (k == 0) {
      if (threadIdx.x == 0) jac[t] = -1.0;
      continue;
    }
    const float2 ci = xy[i];
    const int kk = min(k, n - 1);
    unsigned below = 0;
    const unsigned tau = blm_select(xy, n, i, ci, kk, 0, 0u, hist, shv, &below);
    // number of ties with d2 == tau that are taken, ties by vertex id
    const int r = kk - (int)below;
    unsigned id_cut = 0xffffffffu;
    {
      // count ties; if all of them fit no id selection is needed
      __syncthreads();
      if (threadIdx.x == 0) shv[0] = 0;
      __syncthreads();
      unsigned c = 0;
      for (int l = threadIdx.x; l < n; l += blockDim.x)
        if (l != i && blm_d2bits(ci, xy[l]) == tau) ++c;
      atomicAdd(&shv[0], c);
      __syncthreads();
      const unsigned ties = shv[0];
      __syncthreads();
      if ((int)ties > r) {
        unsigned b2 = 0;
        id_cut = blm_select(xy, n, i, ci, r, 1, tau, hist, shv, &b2);
      }
    }
    // m = |N(i) n nearest-k|: neighbours with (d2, id) <= (tau, id_cut)
    int m = 0;
    for (int e = rowptr[i] + threadIdx.x; e < rowptr[i + 1]; e += blockDim.x) {
      const int j = colidx[e];
      const unsigned d2 = blm_d2bits(ci, xy[j]);
      m += (d2 < tau || (d2 == tau && (unsigned)j <= id_cut)) ? 1 : 0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m += __shfl_xor_sync(0xffffffffu, m, o);
    if ((threadIdx.x & 31) == 0) sh_m[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
      int tot = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += sh_m[w];
      jac[t] = (double)tot / (double)(2 * k - tot);
    }
    __syncthreads();
  }
}

// NP fast path for queries with deg <= KMAX (C5: 95 % of the vertices):
// a warp owns QW queries and scans all n vertices once, 32 per step (one
// coalesced 8-byte load per lane shared by its QW queries).  Per query it
// keeps a shared-memory buffer of candidate keys (d2 bits << 32 | id: the
// (d2, id) order of reading M3, unique per vertex) and a threshold tau = the
// d2 bits of the kk-th smallest key buffered so far.  The scan visits ids in
// increasing order, so every buffered id is smaller than the current one and
// a later vertex can beat the kk-th key only with d2 < tau: the hot test is
// one compare.  A buffer nearing CAP is cut to its kk smallest keys by rank
// (keys are distinct: ranks are a permutation, written in sorted order).
// After the scan T = the kk-th smallest key and m = |{j in N(i): key(j) <=
// T}|, the same decisions as the radix path and the oracle.
#define BLN_NT 256
#define BLN_TAU0 0x7f800001u  // above +inf's bits, below NaN's: every non-NaN d2 passes
struct BLNCut {
  int cnt;
  unsigned tau;
};
template <int CAP>
__device__ __noinline__ BLNCut bln_cut(unsigned long long *buf, int cnt, int kk) {
  // rank of each entry among the cnt buffered keys; keep ranks < kk
  constexpr int PER = CAP / 32;  // entries per lane
  const int lane = threadIdx.x & 31;
  unsigned long long key[PER];
  int rank[PER];
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int e = lane + 32 * u;
    key[u] = e < cnt ? buf[e] : ~0ull;
    rank[u] = 0;
  }
  for (int f = 0; f < cnt; ++f) {
    const unsigned long long kf = buf[f];
#pragma unroll
    for (int u = 0; u < PER; ++u) rank[u] += kf < key[u] ? 1 : 0;
  }
  __syncwarp();
#pragma unroll
  for (int u = 0; u < PER; ++u)
    if (lane + 32 * u < cnt && rank[u] < kk) buf[rank[u]] = key[u];
  __syncwarp();
  BLNCut r;
  r.cnt = min(cnt, kk);
  r.tau = cnt >= kk ? min((unsigned)(buf[kk - 1] >> 32), BLN_TAU0) : BLN_TAU0;
  return r;
}

template <int QW, int CAP>
__global__ void __launch_bounds__(BLN_NT, 2) bln_np_fast(const int *__restrict__ rowptr,
                                                      const int *__restrict__ colidx,
                                                      const float2 *__restrict__ xy, int n,
                                                      const int *__restrict__ queries,
                                                      const int *__restrict__ slots, int nfast,
                                                      double *jac) {
  extern __shared__ unsigned long long bln_buf[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gw = blockIdx.x * (BLN_NT / 32) + warp;
  const int t0 = gw * QW;
  if (t0 >= nfast) return;
  unsigned long long *buf = bln_buf + (size_t)warp * QW * CAP;
  float2 cq[QW];
  int qid[QW], kk[QW], cnt[QW];
  unsigned tau[QW];
#pragma unroll
  for (int q = 0; q < QW; ++q) {
    const int t = min(t0 + q, nfast - 1);  // a short last warp repeats its last query
    qid[q] = queries ? __ldg(queries + __ldg(slots + t)) : __ldg(slots + t);
    cq[q] = __ldg(xy + qid[q]);
    kk[q] = min(__ldg(rowptr + qid[q] + 1) - __ldg(rowptr + qid[q]), n - 1);
    cnt[q] = 0;
    tau[q] = kk[q] > 0 ? BLN_TAU0 : 0u;  // deg 0: nothing to select
  }
  const unsigned lt = (1u << lane) - 1u;
  bl_f2 CQ[QW];
#pragma unroll
  for (int q = 0; q < QW; ++q) CQ[q] = f2pack(cq[q].x, cq[q].y);
  const float qnan = __int_as_float(0x7fffffff);
  // four 32-vertex steps per round, the next round's points loaded while
  // this round's are tested (lanes past n see a NaN point: its d2 bits
  // exceed every threshold)
  float2 nx[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) nx[u] = 32 * u + lane < n ? __ldg(xy + 32 * u + lane) : make_float2(qnan, qnan);
  for (int base0 = 0; base0 < n; base0 += 128) {
    float2 cur4[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      cur4[u] = nx[u];
      const int pn = base0 + 128 + 32 * u + lane;
      nx[u] = pn < n ? __ldg(xy + pn) : make_float2(qnan, qnan);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int pidx = base0 + 32 * u + lane;
      const float2 pt = cur4[u];
      const bl_f2 P = f2pack(pt.x, pt.y);
      unsigned d2[QW];
      bool any = false;
#pragma unroll
      for (int q = 0; q < QW; ++q) {
        // blm_d2bits(cq, pt) with packed ops: (dx, dy) = pt - cq, then
        // dx*dx + dy*dy, each operation rounded separately as the scalar form
        const bl_f2 D = f2sub(P, CQ[q]);
        float sx, sy;
        f2unpack(f2mul(D, D), sx, sy);
        d2[q] = __float_as_uint(__fadd_rn(sx, sy));
        any |= d2[q] < tau[q];
      }
      if (!__any_sync(0xffffffffu, any)) continue;  // the common case
      unsigned need = 0;
#pragma unroll
      for (int q = 0; q < QW; ++q) {
        const bool pass = d2[q] < tau[q];
        const unsigned b = __ballot_sync(0xffffffffu, pass);
        if (b) {
          // the query itself enters as the largest key (~0): never among the
          // kk smallest of the >= kk real keys the buffer ends with
          if (pass)
            buf[q * CAP + cnt[q] + __popc(b & lt)] =
                pidx == qid[q] ? ~0ull : (((unsigned long long)d2[q] << 32) | (unsigned)pidx);
          cnt[q] += __popc(b);
          if (cnt[q] > CAP - 32) need |= 1u << q;
        }
      }
      if (need) {
#pragma unroll
        for (int q = 0; q < QW; ++q)
          if (need >> q & 1u) {
            const BLNCut c = bln_cut<CAP>(buf + q * CAP, cnt[q], kk[q]);
            cnt[q] = c.cnt;
            tau[q] = c.tau;
          }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < QW; ++q) {
    if (t0 + q >= nfast) break;
    const int i = qid[q], k0 = __ldg(rowptr + i), k = __ldg(rowptr + i + 1) - k0;
    if (k == 0) {
      if (lane == 0) jac[__ldg(slots + t0 + q)] = -1.0;
      continue;
    }
    bln_cut<CAP>(buf + q * CAP, cnt[q], kk[q]);  // the kk smallest keys, sorted
    const unsigned long long T = buf[q * CAP + kk[q] - 1];
    int m = 0;
    for (int e = lane; e < k; e += 32) {
      const int j = __ldg(colidx + k0 + e);
      const unsigned long long kj = ((unsigned long long)blm_d2bits(cq[q], __ldg(xy + j)) << 32) | (unsigned)j;
      m += kj <= T ? 1 : 0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m += __shfl_xor_sync(0xffffffffu, m, o);
    if (lane == 0) jac[__ldg(slots + t0 + q)] = (double)m / (double)(2 * k - m);
  }
}

// NP = mean of the non-negative per-query Jaccards (fixed-order sums)
__global__ void __launch_bounds__(BLM_RT) blm_np_reduce(const double *jac, int nq, double *out,
                                                        int *counted) {
  __shared__ double shd[BLM_RT];
  __shared__ int shi[BLM_RT];
  double a = 0.0;
  int k = 0;
  for (int t = threadIdx.x; t < nq; t += BLM_RT)
    if (jac[t] >= 0.0) {
      a += jac[t];
      ++k;
    }
  shd[threadIdx.x] = a;
  shi[threadIdx.x] = k;
  __syncthreads();
  for (int w = BLM_RT / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) {
      shd[threadIdx.x] += shd[threadIdx.x + w];
      shi[threadIdx.x] += shi[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const int c = shi[0];
    *out = c ? shd[0] / c : 0.0;
    *counted = c;
  }
}
