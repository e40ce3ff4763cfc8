// bl_exact_v3.cu -- instantiations of the exact whole-GPU kernel
// bl_layout_kernel<NT, T, TP> (bl_kernel.cuh); one translation unit per
// group so that libbl builds in parallel (paper_2002_08233_b200/_build.py).
#include "bl_ctx.h"

extern const BLVariant bl_exact_v3[] = {
    {1024, 4, 1, (void *)bl_layout_kernel<1024, 4, 1>},
    {1024, 4, 2, (void *)bl_layout_kernel<1024, 4, 2>},
    {1024, 2, 1, (void *)bl_layout_kernel<1024, 2, 1>},
};
extern const int bl_exact_v3_count = 3;
