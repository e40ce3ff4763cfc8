// bl_bh.cu -- instantiation of the BatchLayoutBH kernel (bl_bh.cuh) in its
// own translation unit (parallel builds).
#include "bl_ctx.h"
#include "bl_bh.cuh"

void *bl_bh_kernel_fn() { return (void *)bl_bh_kernel<BH_NT>; }
size_t bl_bh_smem_bytes() { return sizeof(BHShared); }
int bl_bh_threads() { return BH_NT; }
