// bl_metrics.cu -- host side of the §3.7 quality metrics of the
// C-ABI (include/bl.h); kernels in bl_metrics.cuh.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "bl_ctx.h"
#include "bl_metrics.cuh"

#define fail bl_fail

// ------------------------------------------------------------------ metrics
// Quality metrics of §3.7 (csrc/bl_metrics.cuh).  Synchronous on the stream.
namespace {
// context-owned scratch slot (bl_ctx::m_scr): a view that frees nothing
struct DevBuf {
  void *p = nullptr;
  template <typename T>
  T *as() { return reinterpret_cast<T *>(p); }
};
enum {
  S_EU_PART, S_EU_STATS, S_ST_SRC, S_ST_VIS, S_ST_FA, S_ST_FB, S_ST_AA, S_ST_AB, S_ST_AN,
  S_ST_FLAG, S_ST_BAR, S_ST_OUT4, S_ST_OUTN, S_NP_Q, S_NP_JAC, S_NP_OUT, S_NP_CNT, S_EU_ROW,
  S_ST_WORK, S_ST_LMASK, S_NP_SLOTS
};
cudaError_t scratch(bl_ctx *h, int slot, size_t bytes, DevBuf &buf) {
  bytes = std::max<size_t>(bytes, 16);
  if (h->m_cap[slot] < bytes) {
    cudaFree(h->m_scr[slot]);
    h->m_scr[slot] = nullptr;
    h->m_cap[slot] = 0;
    cudaError_t e = cudaMalloc(&h->m_scr[slot], bytes);
    if (e != cudaSuccess) return e;
    h->m_cap[slot] = bytes;
  }
  buf.p = h->m_scr[slot];
  return cudaSuccess;
}
// events around a metric call's kernels: their GPU time -> m_counters[2]
cudaError_t mark(bl_ctx *h, int k, cudaStream_t st) {
  if (!h->m_ev[k]) {
    cudaError_t e = cudaEventCreate(&h->m_ev[k]);
    if (e != cudaSuccess) return e;
  }
  return cudaEventRecord(h->m_ev[k], st);
}
void record_time(bl_ctx *h) {
  float ms = 0.f;
  if (h->m_ev[0] && h->m_ev[1] && cudaEventElapsedTime(&ms, h->m_ev[0], h->m_ev[1]) == cudaSuccess)
    h->m_counters[2] = (long long)(ms * 1e6);
}
}  // namespace

#define BLM_ALLOC(h, slot, buf, bytes)                                                        \
  do {                                                                                       \
    cudaError_t e_ = scratch((h), (slot), (bytes), (buf));                                   \
    if (e_ != cudaSuccess) return fail((h), BL_ENOMEM, "cudaMalloc: %s", cudaGetErrorString(e_)); \
  } while (0)

extern "C" bl_status bl_edge_uniformity(bl_ctx *h, const float *d_xy, double *eu, void *cuda_stream) {
  if (!h || !d_xy || !eu) return bl_fail(h, BL_EINVAL, "NULL argument");
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const int nb = bl_eu_blocks(h);
  DevBuf part, stats;
  BLM_ALLOC(h, S_EU_PART, part, sizeof(double) * 3 * nb);
  BLM_ALLOC(h, S_EU_STATS, stats, sizeof(double) * 8);
  const float2 *xy = reinterpret_cast<const float2 *>(d_xy);
  const int launches = 1;
  BL_CUDA(h, mark(h, 0, st));
  // one pass over the rows by degree class with per-lane shifted sums merged
  // in a fixed order (bla_eu_kernel, bl_attr.cuh; its last block merges)
  {
    bl_status s = bl_eu_launch(h, xy, nb, part.as<double>(), stats.as<double>(), st);
    if (s != BL_OK) return s;
  }
  BL_CUDA(h, cudaGetLastError());
  BL_CUDA(h, mark(h, 1, st));
  BL_CUDA(h, cudaMemcpyAsync(eu, stats.as<double>() + 4, sizeof(double), cudaMemcpyDeviceToHost, st));
  BL_CUDA(h, cudaStreamSynchronize(st));
  record_time(h);
  h->launches = launches;
  return BL_OK;
}

extern "C" bl_status bl_stress(bl_ctx *h, const float *d_xy, const int32_t *sources, int32_t nsrc,
                               double *stress, double *scale, long long *pairs,
                               long long *unreachable, void *cuda_stream) {
  if (!h || !d_xy || !stress) return bl_fail(h, BL_EINVAL, "NULL argument");
  const int n = h->n;
  if (sources) {
    if (nsrc < 1) return bl_fail(h, BL_EINVAL, "nsrc < 1");
    for (int32_t t = 0; t < nsrc; ++t)
      if (sources[t] < 0 || sources[t] >= n) return bl_fail(h, BL_EINVAL, "source %d out of range", sources[t]);
  } else {
    nsrc = n;
  }
  cudaStream_t st = (cudaStream_t)cuda_stream;
  std::vector<int32_t> src(nsrc);
  for (int32_t t = 0; t < nsrc; ++t) src[t] = sources ? sources[t] : t;
  {
    bl_status s = bl_long_rows(h);  // the degree classes (bl_attr.cu)
    if (s != BL_OK) return s;
  }
  int occ = 0;
  BL_CUDA(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, blm_stress_kernel, BLM_NT, 0));
  const int G = h->num_sms * std::max(1, std::min(occ, 4));
  const size_t vb = sizeof(unsigned long long) * BLM_SW * (size_t)n;
  DevBuf d_src, vis, fa, fb, aA, aB, aN, flag, bar, out4, outN, lmask;
  BLM_ALLOC(h, S_ST_SRC, d_src, sizeof(int32_t) * nsrc);
  BLM_ALLOC(h, S_ST_VIS, vis, vb);
  BLM_ALLOC(h, S_ST_FA, fa, vb);
  BLM_ALLOC(h, S_ST_FB, fb, vb);
  BLM_ALLOC(h, S_ST_LMASK, lmask, sizeof(unsigned long long) * BLM_SW * (size_t)std::max(1, h->la_nchunks));
  BLM_ALLOC(h, S_ST_AA, aA, sizeof(double) * G * BLM_NT);
  BLM_ALLOC(h, S_ST_AB, aB, sizeof(double) * G * BLM_NT);
  BLM_ALLOC(h, S_ST_AN, aN, sizeof(unsigned long long) * G * BLM_NT);
  BLM_ALLOC(h, S_ST_FLAG, flag, sizeof(int) * 3);
  BLM_ALLOC(h, S_ST_BAR, bar, sizeof(unsigned));
  BLM_ALLOC(h, S_ST_OUT4, out4, sizeof(double) * 4);
  BLM_ALLOC(h, S_ST_OUTN, outN, sizeof(unsigned long long) * 4);
  DevBuf work;
  BLM_ALLOC(h, S_ST_WORK, work, sizeof(unsigned long long) * ((size_t)G * BLM_NT + 1));
  BL_CUDA(h, cudaMemcpyAsync(d_src.p, src.data(), sizeof(int32_t) * nsrc, cudaMemcpyHostToDevice, st));
  BL_CUDA(h, cudaMemsetAsync(bar.p, 0, sizeof(unsigned), st));
  BLMStressParams k{};
  k.n = n;
  k.nsrc = nsrc;
  k.rowptr = h->d_rowptr;
  k.colidx = h->d_colidx;
  k.xy = reinterpret_cast<const float2 *>(d_xy);
  k.sources = d_src.as<int>();
  k.vis = vis.as<unsigned long long>();
  k.frontA = fa.as<unsigned long long>();
  k.frontB = fb.as<unsigned long long>();
  k.lmask = lmask.as<unsigned long long>();
  k.cls1 = h->d_la_cls;
  k.cls2 = h->d_la_cls + h->la_n1;
  k.n1 = h->la_n1;
  k.n2 = h->la_n2;
  k.nchunks = h->la_nchunks;
  k.nlong = h->la_nlong;
  k.chunks = h->d_la_chunks;
  k.lrow = h->d_la_lrow;
  k.accA = aA.as<double>();
  k.accB = aB.as<double>();
  k.accN = aN.as<unsigned long long>();
  k.flag = flag.as<int>();
  k.bar = bar.as<unsigned>();
  k.work = work.as<unsigned long long>();
  void *args[] = {&k};
  BL_CUDA(h, mark(h, 0, st));
  BL_CUDA(h, cudaLaunchCooperativeKernel((void *)blm_stress_kernel, dim3(G), dim3(BLM_NT), args, 0, st));
  blm_stress_reduce<<<1, BLM_RT, 0, st>>>(k.accA, k.accB, k.accN, k.work, G * BLM_NT,
                                      out4.as<double>(), outN.as<unsigned long long>());
  BL_CUDA(h, cudaGetLastError());
  BL_CUDA(h, mark(h, 1, st));
  double o[4];
  unsigned long long NW[3] = {0, 0, 0};
  BL_CUDA(h, cudaMemcpyAsync(o, out4.p, sizeof o, cudaMemcpyDeviceToHost, st));
  BL_CUDA(h, cudaMemcpyAsync(NW, outN.p, sizeof NW, cudaMemcpyDeviceToHost, st));
  BL_CUDA(h, cudaStreamSynchronize(st));
  const unsigned long long N = NW[0];
  record_time(h);
  h->m_counters[0] = (long long)NW[2];
  h->m_counters[1] = (long long)NW[1];
  *stress = o[0];
  if (scale) *scale = o[1];
  if (pairs) *pairs = (long long)N;
  if (unreachable) *unreachable = (long long)nsrc * (n - 1) - (long long)N;
  h->launches = 2;
  return BL_OK;
}

extern "C" bl_status bl_neighborhood_preservation(bl_ctx *h, const float *d_xy,
                                                  const int32_t *queries, int32_t nq, double *np,
                                                  int32_t *counted, void *cuda_stream) {
  if (!h || !d_xy || !np) return bl_fail(h, BL_EINVAL, "NULL argument");
  const int n = h->n;
  if (queries) {
    if (nq < 1) return bl_fail(h, BL_EINVAL, "nq < 1");
    for (int32_t t = 0; t < nq; ++t)
      if (queries[t] < 0 || queries[t] >= n) return bl_fail(h, BL_EINVAL, "query %d out of range", queries[t]);
  } else {
    nq = n;
  }
  cudaStream_t st = (cudaStream_t)cuda_stream;
  // route each query by kk = min(deg, n - 1): the one-scan threshold kernels
  // for kk <= 32 (8 queries per warp) and kk <= 256 (two per warp), the radix
  // select for the rest (bln_np_fast / blm_np_kernel, bl_metrics.cuh)
  constexpr int K1 = 32, CAP1 = 128, QW1 = 8, K2 = 256, CAP2 = 512, QW2 = 2;
  std::vector<int32_t> slots(nq);
  int n1 = 0, n2 = 0, n3 = 0;
  {
    std::vector<int32_t> s2, s3;
    for (int32_t t = 0; t < nq; ++t) {
      const int i = queries ? queries[t] : t;
      const int kk = std::min(h->rowptr_host[i + 1] - h->rowptr_host[i], n - 1);
      if (kk <= K1) slots[n1++] = t;
      else if (kk <= K2) s2.push_back(t);
      else s3.push_back(t);
    }
    n2 = (int)s2.size();
    n3 = (int)s3.size();
    std::copy(s2.begin(), s2.end(), slots.begin() + n1);
    std::copy(s3.begin(), s3.end(), slots.begin() + n1 + n2);
  }
  DevBuf d_q, jac, out, cnt, d_slots;
  if (queries) {
    BLM_ALLOC(h, S_NP_Q, d_q, sizeof(int32_t) * nq);
    BL_CUDA(h, cudaMemcpyAsync(d_q.p, queries, sizeof(int32_t) * nq, cudaMemcpyHostToDevice, st));
  }
  BLM_ALLOC(h, S_NP_SLOTS, d_slots, sizeof(int32_t) * nq);
  BL_CUDA(h, cudaMemcpyAsync(d_slots.p, slots.data(), sizeof(int32_t) * nq, cudaMemcpyHostToDevice, st));
  BLM_ALLOC(h, S_NP_JAC, jac, sizeof(double) * nq);
  BLM_ALLOC(h, S_NP_OUT, out, sizeof(double));
  BLM_ALLOC(h, S_NP_CNT, cnt, sizeof(int));
  const float2 *xy = reinterpret_cast<const float2 *>(d_xy);
  const int *qp = queries ? d_q.as<int>() : nullptr, *sp = d_slots.as<int>();
  const size_t sm1 = sizeof(unsigned long long) * (BLN_NT / 32) * QW1 * CAP1;
  const size_t sm2 = sizeof(unsigned long long) * (BLN_NT / 32) * QW2 * CAP2;
  BL_CUDA(h, cudaFuncSetAttribute(bln_np_fast<QW1, CAP1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1));
  BL_CUDA(h, cudaFuncSetAttribute(bln_np_fast<QW2, CAP2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2));
  int launches = 1;
  BL_CUDA(h, mark(h, 0, st));
  if (n1) {
    const int per = (BLN_NT / 32) * QW1;
    bln_np_fast<QW1, CAP1><<<(n1 + per - 1) / per, BLN_NT, sm1, st>>>(h->d_rowptr, h->d_colidx, xy, n, qp,
                                                                     sp, n1, jac.as<double>());
    ++launches;
  }
  if (n2) {
    const int per = (BLN_NT / 32) * QW2;
    bln_np_fast<QW2, CAP2><<<(n2 + per - 1) / per, BLN_NT, sm2, st>>>(h->d_rowptr, h->d_colidx, xy, n, qp,
                                                                     sp + n1, n2, jac.as<double>());
    ++launches;
  }
  if (n3) {
    blm_np_kernel<<<2 * h->num_sms, 512, 0, st>>>(h->d_rowptr, h->d_colidx, xy, n, qp, sp + n1 + n2, n3,
                                                  jac.as<double>());
    ++launches;
  }
  blm_np_reduce<<<1, BLM_RT, 0, st>>>(jac.as<double>(), nq, out.as<double>(), cnt.as<int>());
  BL_CUDA(h, cudaGetLastError());
  BL_CUDA(h, mark(h, 1, st));
  int c = 0;
  BL_CUDA(h, cudaMemcpyAsync(np, out.p, sizeof(double), cudaMemcpyDeviceToHost, st));
  BL_CUDA(h, cudaMemcpyAsync(&c, cnt.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  BL_CUDA(h, cudaStreamSynchronize(st));
  if (counted) *counted = c;
  record_time(h);
  h->launches = launches;
  return BL_OK;
}
