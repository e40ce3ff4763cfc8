// bl_exact_v4.cu -- instantiations of the exact whole-GPU kernel
// bl_layout_kernel<NT, T, TP> (bl_kernel.cuh); one translation unit per
// group so that libbl builds in parallel (paper_2002_08233_b200/_build.py).
#include "bl_ctx.h"

extern const BLVariant bl_exact_v4[] = {
    {256, 16, 6, (void *)bl_layout_kernel<256, 16, 6>},
};
extern const int bl_exact_v4_count = 1;
