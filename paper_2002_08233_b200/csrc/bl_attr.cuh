// bl_attr.cuh -- step a5 of SURVEY.md §8(a) on its own: the CSR attraction
// plus neighbour correction S_i = sum_{j in N(i)} (d^(a-1)/K + C K^2 d^(r-1))
// Δ_ij (§2.2; the if/else of Alg. 2, reading C2) for a
// range of vertices, as a standalone high-occupancy kernel (bl_forces with
// BL_ATTRACTION_ONLY).
//
// The work is L2-latency-bound gathers (4 B colidx + 8 B coordinate per CSR
// entry), so the kernel is built for memory-level parallelism: 256 threads
// with a small register budget (8 CTAs = 64 warps per SM), a warp takes TWO
// attraction items (<= 128 entries each: 8 entries per lane) and issues all 8
// colidx loads, then all 8 coordinate gathers, before using any.  Pass 1
// writes one partial per item (fixed lane order + butterfly); pass 2 sums a
// vertex's items in item order (fixed): bitwise-reproducible results that
// equal the persistent kernel's item sums.
#pragma once
#include "bl_kernel.cuh"

#define BLA_NT 256

template <bool FAST>
__global__ void __launch_bounds__(BLA_NT, 8) bla_items_kernel(BLKParams p, int ib, int ie) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * BLA_NT + threadIdx.x) >> 5;
  const int GW = (gridDim.x * BLA_NT) >> 5;
  const float rep = (p.flags & 1u) ? 0.f : p.ck2;
  for (int it0 = ib + 2 * gw; it0 < ie; it0 += 2 * GW) {
    int v[2], k1[2];
    float2 ci[2];
    int jj[8];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int it = it0 + h;
      const bool ok = it < ie;
      v[h] = ok ? __ldg(p.item_v + it) : 0;
      const int k0 = ok ? __ldg(p.item_k0 + it) : 0;
      k1[h] = ok ? __ldg(p.item_k0 + it + 1) : 0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = k0 + lane + 32 * u;
        jj[4 * h + u] = k < k1[h] ? __ldg(p.colidx + k) : -1;
      }
    }
    float2 cj[8];
#pragma unroll
    for (int h = 0; h < 2; ++h) ci[h] = __ldcg(p.xy + v[h]);
#pragma unroll
    for (int u = 0; u < 8; ++u) cj[u] = jj[u] >= 0 ? __ldcg(p.xy + jj[u]) : make_float2(0.f, 0.f);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float sx = 0.f, sy = 0.f;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int w = 4 * h + u;
        if (jj[w] < 0) continue;
        const float dx = cj[w].x - ci[h].x, dy = cj[w].y - ci[h].y;
        const float d2 = fmaf(dx, dx, fmaf(dy, dy, BL_EPS2));
        const float rs = bl_rsqrt(d2);
        const float coef = bl_model_coef<FAST>(p, d2, rs, rep);
        sx = fmaf(coef, dx, sx);
        sy = fmaf(coef, dy, sy);
      }
      sx = bl_warp_sum0(sx);
      sy = bl_warp_sum0(sy);
      if (lane == 0 && it0 + h < ie) p.attr[it0 + h - ib] = make_float2(sx, sy);
    }
  }
}

// S_v = sum of v's items in item order, v in [first, first + count)
__global__ void __launch_bounds__(BLA_NT) bla_sum_kernel(BLKParams p) {
  const int ib = __ldg(p.item_ptr + p.first);
  for (int v = p.first + blockIdx.x * BLA_NT + threadIdx.x; v < p.first + p.count;
       v += gridDim.x * BLA_NT) {
    const int a0 = __ldg(p.item_ptr + v) - ib, a1 = __ldg(p.item_ptr + v + 1) - ib;
    float sx = 0.f, sy = 0.f;
    for (int a = a0; a < a1; ++a) {
      const float2 q = __ldcg(p.attr + a);
      sx += q.x;
      sy += q.y;
    }
    p.f_out[v - p.first] = make_float2(sx, sy);
  }
}
