// bl_cluster.cuh -- the exact BatchLayout (Alg. 2) for
// small graphs on ONE thread-block cluster (sm_100a, device side).
//
// On small graphs every dependent batch has little work (C1: 256 x 1,023
// pairs) and the whole-GPU persistent kernel spends ~8 us per batch on its
// grid barrier and L2 round trips.  Here a single cluster of CS CTAs (16,
// non-portable, or 8) keeps a FULL copy of the coordinates in each CTA's
// shared memory and exchanges only the batch's new coordinates through
// distributed shared memory, with one hardware cluster barrier per batch:
//
//   per batch t, CTA r owns the slice of <= 64 batch targets
//   [lo + r sl, lo + (r+1) sl):
//     A  attraction + neighbour correction of its targets (one warp per
//        target, CSR from L2, neighbour coordinates from the local copy)
//     B  all-pairs repulsion: thread k takes target k mod cnt and source chunk
//        k / cnt (all 512 threads busy), packed f32x2 sweep of the local copy
//     C  fixed-order combine, f = S - C K^2 R, normalised fp64 step,
//        the new coordinates go to xy (HBM) and to every CTA's pend[t & 1]
//        (st.shared::cluster through map_shared_rank)
//     cluster barrier (release/acquire)
//     D  every CTA applies the batch's bt new coordinates to its own copy
//   Coordinates are frozen during a batch because nobody writes a copy before
//   the barrier; the next batch sees the update.  Energy:
//   per-CTA fp64 sums in target order, exchanged through DSMEM at the end of
//   an iteration and summed in rank order by every CTA (identical tol
//   decisions).  Bitwise reproducible.
#pragma once
#include <cooperative_groups.h>

#include "bl_kernel.cuh"

namespace blc_cg = cooperative_groups;

#define BLC_NT 512
#define BLC_NW (BLC_NT / 32)
#define BLC_SLICE_MAX 64  // batch targets per CTA
#define BLC_CS_MAX 16
#define BLC_TMAX 4  // batch targets per thread in the sweep (template T <= 4)

struct BLCParams {
  int n, b, nb, iters, max_batches;
  unsigned flags;
  float ck2, invK;
  double step0, cooling, tol;
  int amode, rmode;
  float a_half, r_half;
  int n4;  // float4 slots of the local copy: ceil(n / 2)
  int nnz;
  int csr_smem;  // 1: rowptr and colidx are copied into shared memory too
  float2 *xy;
  const int *rowptr, *colidx;
  double *energy;
  int *iters_done;
};

// dynamic shared memory, in order: src4[n4] float4 | pend[2][b] float2 |
// red[NT * TMAX] float2 | attr[SLICE_MAX] float2 | q[SLICE_MAX] double |
// ecl[2][CS_MAX] double
__host__ __device__ inline size_t blc_smem_bytes(int n4, int b) {
  return (size_t)n4 * 16 + (size_t)2 * b * 8 + (size_t)BLC_NT * BLC_TMAX * 8 +
         (size_t)BLC_SLICE_MAX * 8 + (size_t)BLC_SLICE_MAX * 8 + (size_t)2 * BLC_CS_MAX * 8;
}

template <int BLC_T, int TP>
__global__ void __launch_bounds__(BLC_NT, 1) bl_cluster_kernel(BLCParams p) {
  blc_cg::cluster_group cl = blc_cg::this_cluster();
  const int CS = (int)cl.num_blocks(), r = (int)cl.block_rank();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  extern __shared__ float4 blc_smem[];
  float4 *src4 = blc_smem;
  float2 *pend = reinterpret_cast<float2 *>(src4 + p.n4);
  float2 *red = pend + 2 * p.b;
  float2 *attr = red + BLC_NT * BLC_TMAX;
  double *qv = reinterpret_cast<double *>(attr + BLC_SLICE_MAX);
  double *ecl = qv + BLC_SLICE_MAX;
  int *s_rp = reinterpret_cast<int *>(ecl + 2 * BLC_CS_MAX);  // [n+1] (csr_smem)
  int *s_ci = s_rp + p.n + 1;                                  // [nnz]
  const int *rowptr = p.rowptr, *colidx = p.colidx;
  if (p.csr_smem) {
    for (int k = threadIdx.x; k <= p.n; k += BLC_NT) s_rp[k] = p.rowptr[k];
    for (int k = threadIdx.x; k < p.nnz; k += BLC_NT) s_ci[k] = p.colidx[k];
    rowptr = s_rp;
    colidx = s_ci;
  }

  // the local copy of all coordinates (odd n: a far dummy pads the last slot)
  for (int k = threadIdx.x; k < 2 * p.n4; k += BLC_NT)
    bl_src_set(src4, k, k < p.n ? p.xy[k] : make_float2(1e30f, 1e30f));
  cl.sync();  // every CTA runs before any DSMEM traffic

  const int full4 = p.n >> 1;  // slots [0, full4) hold two real sources
  const float rep = (p.flags & 1u) ? 0.f : p.ck2;
  double step = p.step0, e_prev = 0.0;
  int batches = 0, done = 0;
  bool stop = false;
  for (int it = 0; it < p.iters && !stop; ++it) {
    double e_it = 0.0;  // thread 0
    for (int t = 0; t < p.nb; ++t) {
      const int lo = t * p.b, bt = min(p.b, p.n - lo);
      const int sl = (bt + CS - 1) / CS;
      const int my0 = min(bt, r * sl), cnt = min(bt, my0 + sl) - my0;
      // A: attraction (+ removal of the neighbour's repulsion, the if/else of
      // Alg. 2) of my targets, one warp per target
      for (int j = warp; j < cnt; j += BLC_NW) {
        const int v = lo + my0 + j;
        const float2 ci = bl_src_get(src4, v);
        float sx = 0.f, sy = 0.f;
        auto scan_row = [&](auto fast) {
          for (int k = rowptr[v] + lane; k < rowptr[v + 1]; k += 32) {
            const float2 cj = bl_src_get(src4, colidx[k]);
            const float dx = cj.x - ci.x, dy = cj.y - ci.y;
            const float d2 = fmaf(dx, dx, fmaf(dy, dy, BL_EPS2));
            const float rs = bl_rsqrt(d2);
            const float coef = bl_model_coef<decltype(fast)::value>(p, d2, rs, rep);
            sx = fmaf(coef, dx, sx);
            sy = fmaf(coef, dy, sy);
          }
        };
        if (p.amode == 0 && p.rmode == 0) scan_row(std::true_type{});
        else scan_row(std::false_type{});
        sx = bl_warp_sum0(sx);
        sy = bl_warp_sum0(sy);
        if (lane == 0) attr[j] = make_float2(sx, sy);
      }
      // B: repulsion.  Targets in groups of BLC_T (registers, ILP); thread k
      // works on group k mod ng over source chunk k / ng of nch = NT / ng
      // chunks: all 512 threads busy whatever the slice size
      const int ng = (cnt + BLC_T - 1) / BLC_T;
      const int nch = ng > 0 ? BLC_NT / ng : 1;
      if (cnt > 0 && (int)threadIdx.x < nch * ng) {
        const int gi = threadIdx.x % ng, ch = threadIdx.x / ng;
        float tx[BLC_T], ty[BLC_T];
        bl_f2 AX[BLC_T], AY[BLC_T];
#pragma unroll
        for (int k = 0; k < BLC_T; ++k) {
          const int j = gi * BLC_T + k;
          // missing targets sit far away: every term underflows to 0
          const float2 tc = j < cnt ? bl_src_get(src4, lo + my0 + j) : make_float2(1e30f, 1e30f);
          tx[k] = tc.x;
          ty[k] = tc.y;
          AX[k] = AY[k] = f2pack(0.f, 0.f);
        }
        const int s0 = (int)((long long)p.n4 * ch / nch);
        const int s1 = (int)((long long)p.n4 * (ch + 1) / nch);
        bl_sweep_range<BLC_T, TP>(src4, s0, s1, full4, tx, ty, AX, AY, p.r_half);
#pragma unroll
        for (int k = 0; k < BLC_T; ++k) {
          const int j = gi * BLC_T + k;
          float a0, a1, b0, b1;
          f2unpack(AX[k], a0, a1);
          f2unpack(AY[k], b0, b1);
          if (j < cnt) red[ch * cnt + j] = make_float2(a0 + a1, b0 + b1);
        }
      }
      __syncthreads();
      // C: combine, update, publish to every CTA of the cluster
      float2 *pend_t = pend + (t & 1) * p.b;
      // few chunks: one thread per target; many chunks: one warp per target
      // (lanes strided, then the butterfly); fixed order either way
      const bool by_warp = nch > 32;
      for (int j = by_warp ? warp : (int)threadIdx.x; j < cnt; j += by_warp ? BLC_NW : BLC_NT) {
        const int v = lo + my0 + j;
        float rx = 0.f, ry = 0.f;
        if (by_warp) {
          for (int ch = lane; ch < nch; ch += 32) {
            const float2 q = red[ch * cnt + j];
            rx += q.x;
            ry += q.y;
          }
          rx = bl_warp_sum0(rx);
          ry = bl_warp_sum0(ry);
        } else {
          for (int ch = 0; ch < nch; ++ch) {
            const float2 q = red[ch * cnt + j];
            rx += q.x;
            ry += q.y;
          }
        }
        if (!by_warp || lane == 0) {
          const float2 S = attr[j];
          const float fx = fmaf(-p.ck2, rx, S.x), fy = fmaf(-p.ck2, ry, S.y);
          const double q = (double)fx * fx + (double)fy * fy;
          float2 cv = bl_src_get(src4, v);
          if (q > 0.0) {
            const double sc = step / sqrt(q);
            cv.x = (float)((double)cv.x + sc * fx);
            cv.y = (float)((double)cv.y + sc * fy);
          }
          qv[j] = q;
          p.xy[v] = cv;
          for (int rr = 0; rr < CS; ++rr) cl.map_shared_rank(pend_t, rr)[my0 + j] = cv;
        }
      }
      __syncthreads();
      if (threadIdx.x == 0)
        for (int j = 0; j < cnt; ++j) e_it += qv[j];  // target order
      ++batches;
      const bool last = t == p.nb - 1;
      const bool mb = p.max_batches > 0 && batches >= p.max_batches;
      if ((last || mb) && threadIdx.x == 0)
        for (int rr = 0; rr < CS; ++rr) cl.map_shared_rank(ecl, rr)[(it & 1) * BLC_CS_MAX + r] = e_it;
      cl.sync();
      // D: the batch's new coordinates into the local copy
      for (int i = threadIdx.x; i < bt; i += BLC_NT) bl_src_set(src4, lo + i, pend_t[i]);
      __syncthreads();
      if (last || mb) {
        double E = 0.0;
        for (int rr = 0; rr < CS; ++rr) E += ecl[(it & 1) * BLC_CS_MAX + rr];  // rank order
        if (r == 0 && threadIdx.x == 0) p.energy[it] = E;
        if (mb) {
          stop = true;
          break;
        }
        done = it + 1;
        if (p.tol > 0.0 && it > 0 && fabs(E - e_prev) < p.tol) {
          stop = true;
          break;
        }
        e_prev = E;
      }
    }
    step = step * p.cooling;
  }
  if (r == 0 && threadIdx.x == 0) *p.iters_done = done;
  cl.sync();  // no CTA exits while others may still write into its memory
}
