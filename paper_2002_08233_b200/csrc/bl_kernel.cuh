// bl_kernel.cuh -- the persistent sm_100a BatchLayout kernel (device side).
//
// One cooperative launch walks every dependent minibatch of every iteration
// of Alg. 2.  Per batch t = [lo, hi):
//
//   phase R  (all CTAs)  -- a4 + a5 of SURVEY.md §8(a)
//     * attraction items: edge-parallel over the batch's contiguous CSR slice
//       [rowptr[lo], rowptr[hi]) in items of <= BL_ECH entries, each gathering
//       xy[colidx[k]] through L2 and summing (d/K)·Δ + C K^2·Δ/d^2 (the
//       spring term f_a·û of §2.2 with f_a = d^2/K, plus the removal of that
//       neighbour's repulsion, so adjacent pairs attract only: the if/else of
//       Alg. 2, reading C2).
//     * all-pairs repulsion: CTA c holds its owned sources {v : v ≡ c mod G}
//       resident in shared memory for the whole call; every warp sweeps a
//       sub-range of them against 32·T register-blocked batch targets,
//       R_i += Δ_ij / d_ij^2 (branch-free: d^2 = Δx^2 + Δy^2 + 1e-30 makes the
//       self pair and coincident pairs contribute exactly 0, reading C3/C4;
//       1/d^2 on the SFU via rcp.approx.ftz).  Per-CTA partials go to
//       part[target][c] after a fixed-order in-CTA combine.
//   grid barrier
//   phase U  (owner CTA of each target)  -- a6 + a7
//     * f_i = S_i - C K^2 · Σ_c part[i][c] in fixed order; c_i += Step·f/||f||
//       (no move if f = 0, reading C5); xy in HBM and the owner's
//       shared copy are updated; ||f||^2 accumulates in fp64 per warp.
//   grid barrier
//
// Coordinates are frozen within a batch because nobody writes xy
// during phase R; the next batch sees the update (Fig. 2 caption P:644)
// because phase U precedes the next barrier.  Every sum has a fixed order,
// so runs are bitwise reproducible.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define BL_NT 512          // threads per CTA (16 warps)
#define BL_NW (BL_NT / 32)
#define BL_ECH 128         // CSR entries per attraction item
#define BL_EPS2 1e-30f     // self/coincident-pair guard folded into d^2

struct BLKParams {
  int n, b, nb, iters, max_batches;
  unsigned flags;
  float ck2, invK;
  double step0, cooling, tol;
  int chunk4;            // float4 slots (2 sources each) per CTA chunk
  int forces_mode, first, count;
  float2 *xy;
  const int *rowptr, *colidx;
  const int *item_ptr, *item_v, *item_k0;
  float2 *part;          // [b][G]
  float2 *attr;          // [max items per batch]
  double *e_cta;         // [2][G]
  double *energy;        // [iters]
  int *iters_done;
  unsigned *bar;
  float2 *f_out;
  // optional phase profile (nullptr = off): [0..7] CTA-0 phase cycle sums,
  // [8 + c] CTA c's cycles from phase-R start to barrier-1 arrival
  unsigned long long *prof;
};

__device__ __forceinline__ float bl_rcp(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float bl_rsqrt(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ unsigned bl_ld_acquire(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Sense-free monotone grid barrier: the counter only grows; barrier k of a
// launch completes when it reaches k·G.  Requires co-residency (cooperative
// launch).  Thread 0 fences the CTA's writes (gpu scope) before arriving.
__device__ __forceinline__ void bl_grid_sync(unsigned *bar, unsigned &target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    target += gridDim.x;
    __threadfence();
    atomicAdd(bar, 1u);
    while ((int)(bl_ld_acquire(bar) - target) < 0) {
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ float bl_warp_sum0(float v) {
  // fixed butterfly; lane 0's value is deterministic run to run
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Phase profiler: thread 0 of each CTA marks phase boundaries (clock64).
struct BLProf {
  unsigned long long acc[8];
  long long last;
  bool on;
  __device__ void init(const BLKParams &p) {
    on = p.prof != nullptr && threadIdx.x == 0;
    for (int i = 0; i < 8; ++i) acc[i] = 0;
    last = on ? clock64() : 0;
  }
  __device__ __forceinline__ void mark(int slot) {
    if (on) {
      const long long t = clock64();
      acc[slot] += (unsigned long long)(t - last);
      last = t;
    }
  }
  __device__ void flush(const BLKParams &p) {
    if (!on) return;
    if (blockIdx.x == 0)
      for (int i = 0; i < 8; ++i) p.prof[i] = acc[i];
    p.prof[8 + blockIdx.x] = acc[0] + acc[1] + acc[2];
  }
};

// ---------------------------------------------------------------- phase R
template <int T>
__device__ __forceinline__ void bl_phase_R(const BLKParams &p, int lo, int bt, const float4 *src4,
                                           float2 *red, BLProf &pf) {
  const int G = gridDim.x, c = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // (1) attraction items of this batch, spread over all warps of the grid
  {
    const int ib = __ldg(p.item_ptr + lo), ie = __ldg(p.item_ptr + lo + bt);
    const int GW = G * BL_NW;
    for (int it = ib + c * BL_NW + warp; it < ie; it += GW) {
      const int v = __ldg(p.item_v + it);
      const int k0 = __ldg(p.item_k0 + it);
      const int k1 = min(k0 + BL_ECH, __ldg(p.rowptr + v + 1));
      const float2 ci = __ldcg(p.xy + v);
      float sx = 0.f, sy = 0.f;
      const float rep = (p.flags & 1u) ? 0.f : p.ck2;
#pragma unroll 4
      for (int k = k0 + lane; k < k1; k += 32) {
        const int j = __ldg(p.colidx + k);
        const float2 cj = __ldcg(p.xy + j);
        const float dx = cj.x - ci.x, dy = cj.y - ci.y;
        const float d2 = fmaf(dx, dx, fmaf(dy, dy, BL_EPS2));
        const float rs = bl_rsqrt(d2);
        const float d = d2 * rs;
        const float coef = fmaf(rep * rs, rs, d * p.invK);
        sx = fmaf(coef, dx, sx);
        sy = fmaf(coef, dy, sy);
      }
      sx = bl_warp_sum0(sx);
      sy = bl_warp_sum0(sy);
      if (lane == 0) p.attr[it - ib] = make_float2(sx, sy);
    }
  }
  pf.mark(0);

  // (2) repulsion: units = (target tile of 32·T, sub-range of the chunk)
  const int ntt = (bt + 32 * T - 1) / (32 * T);
  const int nsub = ntt <= BL_NW ? BL_NW / ntt : 1;
  const int nunits = ntt * nsub;
  for (int u = warp; u < nunits; u += BL_NW) {
    const int tile = u % ntt, sub = u / ntt;
    const int s0 = (int)(((long long)p.chunk4 * sub) / nsub);
    const int s1 = (int)(((long long)p.chunk4 * (sub + 1)) / nsub);
    float tx[T], ty[T], ax[T], ay[T];
#pragma unroll
    for (int k = 0; k < T; ++k) {
      const int idx = tile * 32 * T + k * 32 + lane;
      float2 t = make_float2(0.f, 0.f);
      if (idx < bt) t = __ldcg(p.xy + lo + idx);
      tx[k] = t.x;
      ty[k] = t.y;
      ax[k] = 0.f;
      ay[k] = 0.f;
    }
#pragma unroll 2
    for (int s = s0; s < s1; ++s) {
      const float4 q = src4[s];  // two sources, broadcast to the warp
#pragma unroll
      for (int k = 0; k < T; ++k) {
        const float dx0 = q.x - tx[k], dy0 = q.y - ty[k];
        const float dx1 = q.z - tx[k], dy1 = q.w - ty[k];
        const float r0 = bl_rcp(fmaf(dx0, dx0, fmaf(dy0, dy0, BL_EPS2)));
        const float r1 = bl_rcp(fmaf(dx1, dx1, fmaf(dy1, dy1, BL_EPS2)));
        ax[k] = fmaf(dx0, r0, ax[k]);
        ay[k] = fmaf(dy0, r0, ay[k]);
        ax[k] = fmaf(dx1, r1, ax[k]);
        ay[k] = fmaf(dy1, r1, ay[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < T; ++k) {
      const int idx = tile * 32 * T + k * 32 + lane;
      if (idx < bt) {
        if (nsub == 1)
          p.part[(size_t)idx * G + c] = make_float2(ax[k], ay[k]);
        else
          red[sub * (ntt * 32 * T) + idx] = make_float2(ax[k], ay[k]);
      }
    }
  }
  pf.mark(1);
  if (nsub > 1) {
    __syncthreads();
    for (int idx = threadIdx.x; idx < bt; idx += BL_NT) {
      float2 acc = red[idx];
      for (int s = 1; s < nsub; ++s) {
        const float2 v = red[s * (ntt * 32 * T) + idx];
        acc.x += v.x;
        acc.y += v.y;
      }
      p.part[(size_t)idx * G + c] = acc;
    }
  }
  pf.mark(2);
}

// ---------------------------------------------------------------- phase U
// Owner CTA c handles v in [lo, lo+bt) with v ≡ c (mod G); warp w takes the
// w-th, (w+NW)-th, ... of them.  Returns nothing; accumulates e_acc (lane 0).
__device__ __forceinline__ void bl_phase_U(const BLKParams &p, int lo, int bt, double stepd,
                                           float2 *src, double &e_acc) {
  const int G = gridDim.x, c = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int v0 = lo + ((c - lo % G) + G) % G;
  const int ib = __ldg(p.item_ptr + lo);
  for (int v = v0 + warp * G; v < lo + bt; v += BL_NW * G) {
    const int local = v - lo;
    float rx = 0.f, ry = 0.f;
    for (int cc = lane; cc < G; cc += 32) {
      const float2 q = __ldcg(p.part + (size_t)local * G + cc);
      rx += q.x;
      ry += q.y;
    }
    rx = bl_warp_sum0(rx);
    ry = bl_warp_sum0(ry);
    if (lane == 0) {
      float sx = 0.f, sy = 0.f;
      const int a0 = __ldg(p.item_ptr + v), a1 = __ldg(p.item_ptr + v + 1);
      for (int a = a0; a < a1; ++a) {
        const float2 q = __ldcg(p.attr + (a - ib));
        sx += q.x;
        sy += q.y;
      }
      const float fx = fmaf(-p.ck2, rx, sx);
      const float fy = fmaf(-p.ck2, ry, sy);
      if (p.forces_mode) {
        p.f_out[v - p.first] = make_float2(fx, fy);
      } else {
        const double q = (double)fx * fx + (double)fy * fy;
        if (q > 0.0) {
          const double s = stepd / sqrt(q);
          float2 cv = src[(v - c) / G];  // the owner's resident copy of xy[v]
          cv.x = (float)((double)cv.x + s * fx);
          cv.y = (float)((double)cv.y + s * fy);
          p.xy[v] = cv;
          src[(v - c) / G] = cv;
        }
        e_acc += q;
      }
    }
  }
}

template <int T>
__global__ void __launch_bounds__(BL_NT, 1) bl_layout_kernel(BLKParams p) {
  extern __shared__ float4 bl_smem[];
  float4 *src4 = bl_smem;
  float2 *src = reinterpret_cast<float2 *>(bl_smem);
  float2 *red = reinterpret_cast<float2 *>(bl_smem + p.chunk4);
  __shared__ double e_warp[BL_NW];

  const int G = gridDim.x, c = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned bar_target = 0;
  BLProf pf;
  pf.init(p);

  // resident source chunk: owned vertices c, c+G, ...; pad with far dummies
  // (Δ ~ 1e30 -> d^2 = inf -> 1/d^2 = 0 -> contributes exactly 0)
  for (int k = threadIdx.x; k < 2 * p.chunk4; k += BL_NT) {
    const long long v = (long long)c + (long long)k * G;
    src[k] = v < p.n ? __ldcg(p.xy + v) : make_float2(1e30f, 1e30f);
  }
  __syncthreads();

  if (p.forces_mode) {
    double e_dummy = 0.0;
    bl_phase_R<T>(p, p.first, p.count, src4, red, pf);
    bl_grid_sync(p.bar, bar_target);
    bl_phase_U(p, p.first, p.count, 0.0, src, e_dummy);
    return;
  }

  double step = p.step0;
  double e_acc = 0.0;
  double e_prev = 0.0;
  int batches = 0;
  int it = 0;
  bool stop = false;
  for (; it < p.iters && !stop; ++it) {
    e_acc = 0.0;
    for (int t = 0; t < p.nb; ++t) {
      const int lo = t * p.b;
      const int bt = min(p.b, p.n - lo);
      bl_phase_R<T>(p, lo, bt, src4, red, pf);
      bl_grid_sync(p.bar, bar_target);
      pf.mark(3);
      bl_phase_U(p, lo, bt, step, src, e_acc);
      pf.mark(4);
      ++batches;
      const bool last = (t == p.nb - 1);
      if (p.max_batches > 0 && batches >= p.max_batches) stop = true;
      if (last || stop) {
        if (lane == 0) e_warp[warp] = e_acc;
        __syncthreads();
        if (threadIdx.x == 0) {
          double e = 0.0;
          for (int w = 0; w < BL_NW; ++w) e += e_warp[w];
          p.e_cta[(it & 1) * G + c] = e;
        }
      }
      bl_grid_sync(p.bar, bar_target);
      pf.mark(5);
      if (last || stop) {
        // every CTA reduces the per-CTA energies in the same order, so the
        // convergence decision is identical everywhere
        double E = 0.0;
        for (int cc = 0; cc < G; ++cc) E += __ldcg(p.e_cta + (it & 1) * G + cc);
        if (c == 0 && threadIdx.x == 0) p.energy[it] = E;
        if (!stop && p.tol > 0.0 && it > 0 && fabs(E - e_prev) < p.tol) {
          if (c == 0 && threadIdx.x == 0) *p.iters_done = it + 1;
          pf.flush(p);
          return;
        }
        e_prev = E;
      }
      if (stop) break;
    }
    if (!stop) step = step * p.cooling;
  }
  if (c == 0 && threadIdx.x == 0) *p.iters_done = stop ? it - 1 : it;
  pf.mark(6);
  pf.flush(p);
}
