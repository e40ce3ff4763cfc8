// bl_exact_v0.cu -- instantiations of the exact whole-GPU kernel
// bl_layout_kernel<NT, T, TP> (bl_kernel.cuh); one translation unit per
// group so that libbl builds in parallel (paper_2002_08233_b200/_build.py).
#include "bl_ctx.h"

extern const BLVariant bl_exact_v0[] = {
    {512, 8, 2, (void *)bl_layout_kernel<512, 8, 2>},
    {512, 8, -1, (void *)bl_layout_kernel<512, 8, -1>},
    {512, 8, 1, (void *)bl_layout_kernel<512, 8, 1>},
};
extern const int bl_exact_v0_count = 3;
