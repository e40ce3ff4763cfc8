// bl_attr.cu -- host side of the standalone CSR walks (bl_attr.cuh): step a5
// alone (bl_forces with BL_ATTRACTION_ONLY) and the edge-uniformity passes.
#include "bl_ctx.h"
#include "bl_attr.cuh"

// COO row ids of the CSR (built once per context; the stress / NP helpers)
bl_status bl_coo_rows(bl_ctx *h, cudaStream_t st) {
  if (h->d_coo_row) return BL_OK;
  if (cudaMalloc((void **)&h->d_coo_row, sizeof(int) * std::max<size_t>(8, (size_t)h->nnz + 8)) !=
      cudaSuccess)
    return bl_fail(h, BL_ENOMEM, "cudaMalloc COO rows");
  bla_coo_rows<<<h->num_sms * 8, BLA_NT, 0, st>>>(h->d_rowptr, h->n, h->d_coo_row);
  if (cudaGetLastError() != cudaSuccess) return bl_fail(h, BL_ECUDA, "COO rows kernel");
  return BL_OK;
}

// Degree classes of the rows (bla_kernel), built once per context from the
// host copy of rowptr: class 1 (deg <= 8) and class 2 (9..BLA_LONG) vertex
// lists, and the long rows cut into BLA_CHUNK-entry chunks with per long row
// its (first chunk, chunk count).
bl_status bl_long_rows(bl_ctx *h) {
  if (h->la_ready) return BL_OK;
  std::vector<BLAChunk> ch;
  std::vector<int2> lr;
  std::vector<int> c1, c2;
  for (int v = 0; v < h->n; ++v) {
    const int k0 = h->rowptr_host[v], k1 = h->rowptr_host[v + 1];
    if (k1 - k0 <= 8) {
      c1.push_back(v);
      continue;
    }
    if (k1 - k0 <= BLA_LONG) {
      c2.push_back(v);
      continue;
    }
    const int li = (int)lr.size();
    lr.push_back(make_int2((int)ch.size(), (k1 - k0 + BLA_CHUNK - 1) / BLA_CHUNK));
    for (int k = k0; k < k1; k += BLA_CHUNK) ch.push_back({v, k, std::min(k + BLA_CHUNK, k1), li});
  }
  h->la_nchunks = (int)ch.size();
  h->la_nlong = (int)lr.size();
  h->la_n1 = (int)c1.size();
  h->la_n2 = (int)c2.size();
  const size_t nc = std::max<size_t>(1, ch.size()), nl = std::max<size_t>(1, lr.size());
  if (cudaMalloc((void **)&h->d_la_chunks, sizeof(BLAChunk) * nc) != cudaSuccess ||
      cudaMalloc((void **)&h->d_la_lrow, sizeof(int2) * nl) != cudaSuccess ||
      cudaMalloc((void **)&h->d_la_lpart, sizeof(float2) * nc) != cudaSuccess ||
      cudaMalloc((void **)&h->d_la_cls, sizeof(int) * (c1.size() + c2.size() + 1)) != cudaSuccess ||
      cudaMalloc((void **)&h->d_la_bar, 2 * sizeof(unsigned)) != cudaSuccess ||
      cudaMemset(h->d_la_bar, 0, 2 * sizeof(unsigned)) != cudaSuccess)
    return bl_fail(h, BL_ENOMEM, "cudaMalloc row classes");
  if ((!ch.empty() && cudaMemcpy(h->d_la_chunks, ch.data(), sizeof(BLAChunk) * ch.size(),
                                 cudaMemcpyHostToDevice) != cudaSuccess) ||
      (!lr.empty() && cudaMemcpy(h->d_la_lrow, lr.data(), sizeof(int2) * lr.size(),
                                 cudaMemcpyHostToDevice) != cudaSuccess) ||
      (!c1.empty() && cudaMemcpy(h->d_la_cls, c1.data(), sizeof(int) * c1.size(),
                                 cudaMemcpyHostToDevice) != cudaSuccess) ||
      (!c2.empty() && cudaMemcpy(h->d_la_cls + c1.size(), c2.data(), sizeof(int) * c2.size(),
                                 cudaMemcpyHostToDevice) != cudaSuccess))
    return bl_fail(h, BL_ECUDA, "row class upload");
  h->la_ready = true;
  return BL_OK;
}

// bla_kernel: one cooperative launch (the long rows' sums after its grid
// barrier; the counter is monotone, la_bar_base tracks its target)
bl_status bl_attr_launch(bl_ctx *h, const BLKParams &k, cudaStream_t st) {
  bl_status s = bl_long_rows(h);
  if (s != BL_OK) return s;
  const int blocks = h->num_sms * BLA_BPS;  // co-resident (48 registers per thread)
  const int *c1 = h->d_la_cls, *c2 = h->d_la_cls + h->la_n1;
  BLKParams kk = k;
  int n1 = h->la_n1, n2 = h->la_n2, nch = h->la_nchunks, nlong = h->la_nlong;
  BLAChunk *chunks = h->d_la_chunks;
  float2 *lpart = h->d_la_lpart;
  int2 *lrow = h->d_la_lrow;
  unsigned *bar = h->d_la_bar;
  h->la_bar_base += (unsigned)blocks;
  unsigned target = h->la_bar_base;
  void *args[] = {&kk, &c1, &n1, &c2, &n2, &chunks, &nch, &lpart, &lrow, &nlong, &bar, &target};
  void *fn = (k.amode == 0 && k.rmode == 0) ? (void *)bla_kernel<true> : (void *)bla_kernel<false>;
  if (cudaLaunchCooperativeKernel(fn, dim3(blocks), dim3(BLA_NT), args, 0, st) != cudaSuccess)
    return bl_fail(h, BL_ECUDA, "attraction kernel");
  h->launches = 1;
  return BL_OK;
}

int bl_eu_blocks(const bl_ctx *h) { return BLA_BPS * h->num_sms; }

// edge uniformity: one pass over the degree classes, the last block merges
// (d_la_bar[1] = its arrival counter, reset by that block)
bl_status bl_eu_launch(bl_ctx *h, const float2 *xy, int blocks, double *part, double *stats,
                       cudaStream_t st) {
  bl_status s = bl_long_rows(h);
  if (s != BL_OK) return s;
  const int *c1 = h->d_la_cls, *c2 = h->d_la_cls + h->la_n1;
  bla_eu_kernel<<<blocks, BLA_NT, 0, st>>>(h->d_rowptr, h->d_colidx, xy, c1, h->la_n1, c2,
                                          h->la_n2, h->d_la_chunks, h->la_nchunks, part,
                                          h->d_la_bar + 1, stats);
  if (cudaGetLastError() != cudaSuccess) return bl_fail(h, BL_ECUDA, "edge-uniformity kernels");
  return BL_OK;
}
