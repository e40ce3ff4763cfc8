// bl_metrics.cuh -- the layout quality metrics of §3.7
// on sm_100a (device side; readings M1-M4 of DESIGN.md §3).
//
//   edge uniformity (M2): one entry-parallel pass over the CSR (edges i < j
//     once; bla_eu_kernel in bl_attr.cuh), fp64 per-lane Welford states
//     merged in a fixed order;
//   stress (M1): multi-source BFS, 64 sources per group as one uint64 bitmask
//     per vertex, pull-based levels inside ONE cooperative kernel (grid barrier
//     per level); every newly reached (source, vertex) pair at hop distance L
//     adds |D|/L and |D|^2/L^2 to fp64 accumulators, so the scale-optimised
//     stress comes out in closed form (s* = A/B, ST = s*^2 B - 2 s* A + N)
//     without storing a distance matrix;
//   neighbourhood preservation (M3): one CTA per query vertex i; radix
//     select (4 x 8-bit passes, warp-aggregated shared-memory histograms) of
//     the deg(i)-th smallest fp32 squared distance, ties resolved by vertex id
//     with a second select over ids, then the Jaccard of N(i) with the
//     layout-nearest set.
// All reductions have a fixed order: results are bitwise reproducible.
#pragma once
#include "bl_kernel.cuh"

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
struct BLMStressParams {
  int n, nsrc;
  const int *rowptr, *colidx;
  const float2 *xy;
  const int *sources;   // [nsrc] (device)
  unsigned long long *vis, *frontA, *frontB;
  double *accA, *accB;  // [G * NT] per-thread partials (fixed mapping)
  unsigned long long *accN;
  int *flag;            // [3] per-level 'new pairs' flags, rotating
  unsigned *bar;
  unsigned long long *work;  // [G * NT] CSR entries examined per thread; [G * NT] levels
};

__global__ void __launch_bounds__(BLM_NT, 1) blm_stress_kernel(BLMStressParams p) {
  __shared__ float2 src_xy[64];
  __shared__ int unit_dummy;
  const int G = gridDim.x, tid = blockIdx.x * BLM_NT + threadIdx.x, GT = G * BLM_NT;
  unsigned bar_target = 0;
  double A = 0.0, B = 0.0;
  unsigned long long N = 0, examined = 0, levels = 0;
  for (int g0 = 0; g0 < p.nsrc; g0 += 64) {
    const int gs = min(64, p.nsrc - g0);
    // init the group: no vertex visited except the sources
    for (int v = tid; v < p.n; v += GT) {
      p.vis[v] = 0ull;
      p.frontA[v] = 0ull;
    }
    if (threadIdx.x < 64) src_xy[threadIdx.x] = threadIdx.x < gs ? p.xy[p.sources[g0 + threadIdx.x]] : make_float2(0.f, 0.f);
    if (tid == 0) p.flag[0] = p.flag[1] = p.flag[2] = 0;
    bl_grid_sync(p.bar, bar_target, &unit_dummy);
    if (tid < gs) {
      const int s = p.sources[g0 + tid];
      atomicOr(p.vis + s, 1ull << tid);
      atomicOr(p.frontA + s, 1ull << tid);
    }
    bl_grid_sync(p.bar, bar_target, &unit_dummy);
    const unsigned long long full = gs == 64 ? ~0ull : ((1ull << gs) - 1ull);
    unsigned long long *cur = p.frontA, *nxt = p.frontB;
    for (int L = 1;; ++L) {
      for (int v = tid; v < p.n; v += GT) {
        const unsigned long long vv = __ldcg(p.vis + v);
        unsigned long long nb = 0ull;
        if (vv != full) {
          unsigned long long acc = 0ull;
          const int k0 = p.rowptr[v], k1 = p.rowptr[v + 1];
          for (int k = k0; k < k1; ++k) acc |= __ldcg(cur + p.colidx[k]);
          examined += (unsigned long long)(k1 - k0);
          nb = acc & ~vv;
        }
        nxt[v] = nb;
        if (nb) {
          p.vis[v] = vv | nb;
          p.flag[L % 3] = 1;
          const float2 cv = p.xy[v];
          const double invL = 1.0 / (double)L;
          unsigned long long m = nb;
          while (m) {  // bits in increasing order: fixed accumulation order
            const int k = __ffsll((long long)m) - 1;
            m &= m - 1ull;
            const double dx = (double)cv.x - (double)src_xy[k].x;
            const double dy = (double)cv.y - (double)src_xy[k].y;
            const double l2 = dx * dx + dy * dy;
            A += sqrt(l2) * invL;
            B += l2 * invL * invL;
            ++N;
          }
        }
      }
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
                                                        int nq, double *jac) {
  __shared__ unsigned hist[256];
  __shared__ unsigned shv[2];
  __shared__ int sh_m[16];
  for (int t = blockIdx.x; t < nq; t += gridDim.x) {
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
