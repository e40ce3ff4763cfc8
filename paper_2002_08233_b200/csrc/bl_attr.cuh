// bl_attr.cuh -- step a5 of SURVEY.md §8(a) on its own: the CSR attraction
// plus neighbour correction S_i = sum_{j in N(i)} (d^(a-1)/K + C K^2 d^(r-1))
// Δ_ij (§2.2; the if/else of Alg. 2, reading C2) for a
// range of vertices, as standalone entry-parallel kernels (bl_forces with
// BL_ATTRACTION_ONLY).
//
// The work is L2-latency-bound gathers (4 B colidx + 8 B coordinate per CSR
// entry) over a degree distribution from 0 to ~16k, so it is cut by ENTRIES,
// not by rows: lane L of a warp owns the 8 consecutive entries k = 8m .. 8m+7
// (m = 32 w + L), loads their COO row ids and columns as two 16-byte vectors
// each, gathers the 16 coordinates, and sums its entries row by row in entry
// order; every (lane, row) segment writes one partial at the index of its
// first entry -- a row start or a multiple of 8.  Pass 2 (one warp per
// vertex) sums the partials of row i -- at rowptr[i] and at the multiples of
// 8 inside the row -- lane-strided in order, then a fixed butterfly.  Every
// sum has a fixed order: bitwise-reproducible results.  256 threads with a
// 64-register budget: 32 warps per SM, 16 gathers in flight per lane.
#pragma once
#include "bl_kernel.cuh"

#define BLA_NT 256

// COO row ids of the CSR entries (row[k] = i for rowptr[i] <= k < rowptr[i+1])
__global__ void bla_coo_rows(const int *rowptr, int n, int *row) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    for (int k = rowptr[i]; k < rowptr[i + 1]; ++k) row[k] = i;
}

template <bool FAST>
__global__ void __launch_bounds__(BLA_NT, 4) bla_edge_kernel(BLKParams p, const int *__restrict__ row,
                                                             int e0, int e1, float2 *part) {
  const int T = gridDim.x * BLA_NT;
  const float rep = (p.flags & 1u) ? 0.f : p.ck2;
  for (int m = e0 / 8 + blockIdx.x * BLA_NT + threadIdx.x; 8 * m < e1; m += T) {
    const int k0 = 8 * m;
    int r[8], j[8];
    if (k0 >= e0 && k0 + 8 <= e1) {  // aligned full group: two 16-byte vectors each
      const int4 a = __ldg(reinterpret_cast<const int4 *>(row + k0));
      const int4 b = __ldg(reinterpret_cast<const int4 *>(row + k0 + 4));
      const int4 c = __ldg(reinterpret_cast<const int4 *>(p.colidx + k0));
      const int4 d = __ldg(reinterpret_cast<const int4 *>(p.colidx + k0 + 4));
      r[0] = a.x; r[1] = a.y; r[2] = a.z; r[3] = a.w; r[4] = b.x; r[5] = b.y; r[6] = b.z; r[7] = b.w;
      j[0] = c.x; j[1] = c.y; j[2] = c.z; j[3] = c.w; j[4] = d.x; j[5] = d.y; j[6] = d.z; j[7] = d.w;
    } else {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int k = k0 + u;
        const bool ok = k >= e0 && k < e1;
        r[u] = ok ? __ldg(row + k) : -1;
        j[u] = ok ? __ldg(p.colidx + k) : 0;
      }
    }
    float2 ci[8], cj[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      ci[u] = r[u] >= 0 ? __ldcg(p.xy + r[u]) : make_float2(0.f, 0.f);
      cj[u] = r[u] >= 0 ? __ldcg(p.xy + j[u]) : make_float2(0.f, 0.f);
    }
    float sx = 0.f, sy = 0.f;
    int start = -1;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (r[u] < 0) continue;
      if (start < 0) start = k0 + u;
      const float dx = cj[u].x - ci[u].x, dy = cj[u].y - ci[u].y;
      const float d2 = fmaf(dx, dx, fmaf(dy, dy, BL_EPS2));
      const float rs = bl_rsqrt(d2);
      const float coef = bl_model_coef<FAST>(p, d2, rs, rep);
      sx = fmaf(coef, dx, sx);
      sy = fmaf(coef, dy, sy);
      if (u == 7 || r[u + 1] != r[u]) {  // the (lane, row) segment ends here
        part[start] = make_float2(sx, sy);
        sx = sy = 0.f;
        start = -1;
      }
    }
  }
}

// pass 2: S_v for v in [first, first + count): the partials of row v at
// rowptr[v] and at every multiple of 8 inside the row, lane-strided in order,
// then the fixed butterfly
__global__ void __launch_bounds__(BLA_NT) bla_row_sum_kernel(BLKParams p, const float2 *part) {
  const int lane = threadIdx.x & 31;
  const int W = (gridDim.x * BLA_NT) >> 5;
  for (int v = p.first + ((blockIdx.x * BLA_NT + threadIdx.x) >> 5); v < p.first + p.count;
       v += W) {
    const int a = __ldg(p.rowptr + v), e = __ldg(p.rowptr + v + 1);
    // partial positions: a, then 8 ceil((a+1)/8), +8, ... < e
    const int g0 = (a + 8) & ~7;               // first multiple of 8 > a
    const int np = a < e ? 1 + (e > g0 ? (e - g0 + 7) / 8 : 0) : 0;
    float sx = 0.f, sy = 0.f;
    for (int t = lane; t < np; t += 32) {
      const float2 q = __ldcg(part + (t == 0 ? a : g0 + 8 * (t - 1)));
      sx += q.x;
      sy += q.y;
    }
    sx = bl_warp_sum0(sx);
    sy = bl_warp_sum0(sy);
    if (lane == 0) p.f_out[v - p.first] = make_float2(sx, sy);
  }
}
