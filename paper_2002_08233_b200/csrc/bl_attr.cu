// bl_attr.cu -- host launch of the standalone step-a5 kernels (bl_attr.cuh):
// bl_forces with BL_ATTRACTION_ONLY.
#include "bl_ctx.h"
#include "bl_attr.cuh"

cudaError_t bl_attr_launch(const BLKParams &k, cudaStream_t st, int ib, int ie, int num_sms) {
  const int items = ie - ib;
  if (items > 0) {
    const int blocks = std::min(num_sms * 8, (items + 2 * (BLA_NT / 32) - 1) / (2 * (BLA_NT / 32)));
    if (k.amode == 0 && k.rmode == 0)
      bla_items_kernel<true><<<std::max(1, blocks), BLA_NT, 0, st>>>(k, ib, ie);
    else
      bla_items_kernel<false><<<std::max(1, blocks), BLA_NT, 0, st>>>(k, ib, ie);
  }
  const int sblocks = std::max(1, std::min(num_sms * 8, (k.count + BLA_NT - 1) / BLA_NT));
  bla_sum_kernel<<<sblocks, BLA_NT, 0, st>>>(k);
  return cudaGetLastError();
}
