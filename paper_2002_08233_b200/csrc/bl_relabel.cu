// bl_relabel.cu -- batch randomisation (§4.3.3; readings R1-R2 of
// DESIGN.md §3) by relabelling: iteration `it` runs in POSITION space, where
// position i holds vertex pi_it(i).  There the randomised batches
// pi_it(t b .. t b + b - 1) are the contiguous position ranges every
// sequential driver (asynchronous, latency, pipelined) is built for, so the
// iteration is one plain launch of the layout kernel on
//   xyP[i]      = xy[pi_it(i)]
//   rowptrP     = exclusive scan of deg(pi_it(i))
//   colidxP[..] = pi_it^-1(neighbour), rows in their CSR order
// built here by ONE cooperative kernel per iteration (which first scatters
// the previous iteration's xyP back to vertex space).  O(n + nnz) per
// iteration against the iteration's O(n^2) pairs: 47 MB of traffic at C5.
#include "bl_ctx.h"

#define BLR_NT 1024

struct BLRelabelParams {
  int n, nnz, shuf_h, it, unperm;
  unsigned long long seed;
  // convergence: before iteration it >= 2, |E[it-1] - E[it-2]| < tol
  // stops the run -- every CTA takes the same decision from the same two
  // values; *stop = it + 1 makes every later launch of the call a no-op (the
  // stopping launch itself must finish its scatter in every CTA, hence the
  // iteration number: its own CTAs that start late do not take it for theirs)
  double tol;
  const double *energy;
  int *stop, *iters_done;
  const int *rowptr, *colidx;
  int *piv, *inv, *rowptrP, *colidxP, *cta_sum;
  float2 *xy, *xyP;
  unsigned *bar;
};

// exclusive block scan of one int per thread (BLR_NT threads); *total <- sum
__device__ __forceinline__ int blr_block_scan(int v, int *wsum, int *total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int w = wsum[lane];
    int wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    wsum[lane] = wi - w;  // exclusive warp offsets
    if (lane == 31) *total = wi;
  }
  __syncthreads();
  const int r = wsum[warp] + incl - v;
  __syncthreads();  // wsum / total are reused by the next tile
  return r;
}

__global__ void __launch_bounds__(BLR_NT, 1) bl_relabel_kernel(BLRelabelParams p) {
  __shared__ unsigned long long pkey[4];
  __shared__ int wsum[32];
  __shared__ int s_total, s_dummy;
  const int G = gridDim.x, c = blockIdx.x, tid = threadIdx.x;
  unsigned target = 0;
  if (p.stop) {  // stopped by an earlier iteration's launch
    const int sv = *(const volatile int *)p.stop;
    if (sv != 0 && sv <= p.it) return;
  }
  // A: the previous iteration's coordinates back to vertex space
  if (p.unperm) {
    for (int i = c * BLR_NT + tid; i < p.n; i += G * BLR_NT) p.xy[__ldcg(p.piv + i)] = __ldcg(p.xyP + i);
    if (p.tol > 0.0 && p.it >= 2 &&
        fabs(__ldcg(p.energy + p.it - 1) - __ldcg(p.energy + p.it - 2)) < p.tol) {
      // (no CTA reads stop after this point in this launch; later launches do)
      if (c == 0 && tid == 0) {
        *p.iters_done = p.it;
        __threadfence();
        *p.stop = p.it + 1;
      }
      return;
    }
    bl_grid_sync(p.bar, target, &s_dummy);
  }
  const BLPerm P = bl_perm_make(p.seed, p.shuf_h, p.n, p.it, pkey);  // pi_it (R1)
  __syncthreads();
  // B: pi_it and its inverse, the coordinates and degrees in position order
  // (contiguous positions per CTA, for the scan)
  const int chunk = (p.n + G - 1) / G;
  const int lo = min(p.n, c * chunk), hi = min(p.n, lo + chunk);
  int dsum = 0;
  for (int i = lo + tid; i < hi; i += BLR_NT) {
    const int v = bl_perm(P, i);
    p.piv[i] = v;
    p.inv[v] = i;
    p.xyP[i] = __ldcg(p.xy + v);
    const int d = __ldg(p.rowptr + v + 1) - __ldg(p.rowptr + v);
    p.rowptrP[i] = d;
    dsum += d;
  }
  {
    int tot;
    (void)blr_block_scan(dsum, wsum, &s_total);
    tot = s_total;
    if (tid == 0) p.cta_sum[c] = tot;
  }
  bl_grid_sync(p.bar, target, &s_dummy);
  // C: rowptrP = exclusive scan (CTA offset from the per-CTA sums, then tiles)
  int base = 0;
  {
    int part = 0;
    for (int cc = tid; cc < c; cc += BLR_NT) part += __ldcg(p.cta_sum + cc);
    (void)blr_block_scan(part, wsum, &s_total);
    base = s_total;
  }
  const int e0 = base;
  for (int t0 = lo; t0 < hi; t0 += BLR_NT) {
    const int i = t0 + tid;
    const int d = i < hi ? p.rowptrP[i] : 0;
    const int ex = blr_block_scan(d, wsum, &s_total);
    const int tot = s_total;
    if (i < hi) p.rowptrP[i] = base + ex;
    base += tot;
    __syncthreads();  // s_total is rewritten by the next tile
  }
  if (c == G - 1 && tid == 0) p.rowptrP[p.n] = p.nnz;
  __syncthreads();  // this CTA's rowptrP[lo, hi) is visible to all its threads
  // D: the CSR entries of this CTA's positions, one entry per thread step:
  // entry e belongs to the last position i in [lo, hi) with rowptrP[i] <= e
  const int e1 = base;
  for (int e = e0 + tid; e < e1; e += BLR_NT) {
    int a = lo, b = hi - 1;
    while (a < b) {
      const int m = (a + b + 1) >> 1;
      if (p.rowptrP[m] <= e) a = m;
      else b = m - 1;
    }
    const int v = p.piv[a];
    const int k = __ldg(p.rowptr + v) + (e - p.rowptrP[a]);
    p.colidxP[e] = __ldcg(p.inv + __ldg(p.colidx + k));
  }
}

// the last iteration's coordinates back to vertex space; iters_done <- iters
__global__ void bl_unrelabel_kernel(int n, const int *piv, const float2 *xyP, float2 *xy,
                                    int *iters_done, int iters, const int *stop) {
  if (stop && *(const volatile int *)stop) return;  // scattered back by the stopping launch
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    xy[__ldcg(piv + i)] = __ldcg(xyP + i);
  if (blockIdx.x == 0 && threadIdx.x == 0) *iters_done = iters;
}

bl_status bl_relabel_alloc(bl_ctx *h) {
  if (h->d_piv) return BL_OK;
  const size_t n = (size_t)h->n, nz = std::max<size_t>(1, (size_t)h->nnz);
  if (cudaMalloc((void **)&h->d_piv, sizeof(int) * n) != cudaSuccess ||
      cudaMalloc((void **)&h->d_inv, sizeof(int) * n) != cudaSuccess ||
      cudaMalloc((void **)&h->d_rowptrP, sizeof(int) * (n + 1)) != cudaSuccess ||
      cudaMalloc((void **)&h->d_colidxP, sizeof(int) * nz) != cudaSuccess ||
      cudaMalloc((void **)&h->d_xyP, sizeof(float2) * n) != cudaSuccess ||
      cudaMalloc((void **)&h->d_rl_sum, sizeof(int) * (size_t)h->num_sms) != cudaSuccess ||
      cudaMalloc((void **)&h->d_rl_bar, sizeof(unsigned)) != cudaSuccess ||
      cudaMalloc((void **)&h->d_rl_iters, sizeof(int)) != cudaSuccess ||
      cudaMalloc((void **)&h->d_rl_stop, sizeof(int)) != cudaSuccess)
    return bl_fail(h, BL_ENOMEM, "cudaMalloc relabel buffers");
  return BL_OK;
}

void bl_relabel_free(bl_ctx *h) {
  cudaFree(h->d_piv);
  cudaFree(h->d_inv);
  cudaFree(h->d_rowptrP);
  cudaFree(h->d_colidxP);
  cudaFree(h->d_xyP);
  cudaFree(h->d_rl_sum);
  cudaFree(h->d_rl_bar);
  cudaFree(h->d_rl_iters);
  cudaFree(h->d_rl_stop);
}

// Position space of iteration `it` from the vertex-space xy (unperm: xyP of
// the previous iteration is scattered back to xy first).
bl_status bl_relabel_launch(bl_ctx *h, float2 *xy, unsigned long long seed, int shuf_h, int it,
                            int unperm, double tol, cudaStream_t st) {
  BLRelabelParams k{};
  k.n = h->n;
  k.nnz = h->nnz;
  k.shuf_h = shuf_h;
  k.it = it;
  k.unperm = unperm;
  k.seed = seed;
  k.rowptr = h->d_rowptr;
  k.colidx = h->d_colidx;
  k.piv = h->d_piv;
  k.inv = h->d_inv;
  k.rowptrP = h->d_rowptrP;
  k.colidxP = h->d_colidxP;
  k.cta_sum = h->d_rl_sum;
  k.xy = xy;
  k.xyP = h->d_xyP;
  k.bar = h->d_rl_bar;
  k.tol = tol;
  k.energy = h->d_energy;
  k.stop = tol > 0.0 ? h->d_rl_stop : nullptr;
  k.iters_done = h->d_iters_done;
  BL_CUDA(h, cudaMemsetAsync(h->d_rl_bar, 0, sizeof(unsigned), st));
  void *args[] = {&k};
  BL_CUDA(h, cudaLaunchCooperativeKernel((void *)bl_relabel_kernel, dim3(h->num_sms), dim3(BLR_NT),
                                         args, 0, st));
  return BL_OK;
}

bl_status bl_unrelabel_launch(bl_ctx *h, float2 *xy, int iters, bool tol_stop, cudaStream_t st) {
  bl_unrelabel_kernel<<<h->num_sms, BLR_NT, 0, st>>>(h->n, h->d_piv, h->d_xyP, xy, h->d_iters_done,
                                                    iters, tol_stop ? h->d_rl_stop : nullptr);
  BL_CUDA(h, cudaGetLastError());
  return BL_OK;
}
