// bl_attr.cu -- host launch of the standalone step-a5 kernels (bl_attr.cuh):
// bl_forces with BL_ATTRACTION_ONLY.
#include "bl_ctx.h"
#include "bl_attr.cuh"

// COO row ids of the CSR (built once per context; also used by the EU metric)
bl_status bl_coo_rows(bl_ctx *h, cudaStream_t st) {
  if (h->d_coo_row) return BL_OK;
  if (cudaMalloc((void **)&h->d_coo_row, sizeof(int) * std::max<size_t>(8, (size_t)h->nnz + 8)) !=
      cudaSuccess)
    return bl_fail(h, BL_ENOMEM, "cudaMalloc COO rows");
  bla_coo_rows<<<h->num_sms * 8, BLA_NT, 0, st>>>(h->d_rowptr, h->n, h->d_coo_row);
  if (cudaGetLastError() != cudaSuccess) return bl_fail(h, BL_ECUDA, "COO rows kernel");
  return BL_OK;
}

bl_status bl_attr_launch(bl_ctx *h, const BLKParams &k, cudaStream_t st) {
  bl_status s = bl_coo_rows(h, st);
  if (s != BL_OK) return s;
  if (!h->d_apart &&
      cudaMalloc((void **)&h->d_apart, sizeof(float2) * std::max<size_t>(8, (size_t)h->nnz + 8)) !=
          cudaSuccess)
    return bl_fail(h, BL_ENOMEM, "cudaMalloc attraction partials");
  const int e0 = h->rowptr_host[k.first], e1 = h->rowptr_host[k.first + k.count];
  if (e1 > e0) {
    const int groups = (e1 + 7) / 8 - e0 / 8;
    const int blocks = std::max(1, std::min(h->num_sms * 4, (groups + BLA_NT - 1) / BLA_NT));
    if (k.amode == 0 && k.rmode == 0)
      bla_edge_kernel<true><<<blocks, BLA_NT, 0, st>>>(k, h->d_coo_row, e0, e1, h->d_apart);
    else
      bla_edge_kernel<false><<<blocks, BLA_NT, 0, st>>>(k, h->d_coo_row, e0, e1, h->d_apart);
  }
  const int sblocks = std::max(1, std::min(h->num_sms * 16, (k.count * 32 + BLA_NT - 1) / BLA_NT));
  bla_row_sum_kernel<<<sblocks, BLA_NT, 0, st>>>(k, h->d_apart);
  if (cudaGetLastError() != cudaSuccess) return bl_fail(h, BL_ECUDA, "attraction kernels");
  return BL_OK;
}
