// bl_exact_v1.cu -- instantiations of the exact whole-GPU kernel
// bl_layout_kernel<NT, T, TP> (bl_kernel.cuh); one translation unit per
// group so that libbl builds in parallel (paper_2002_08233_b200/_build.py).
#include "bl_ctx.h"

extern const BLVariant bl_exact_v1[] = {
    {512, 8, 3, (void *)bl_layout_kernel<512, 8, 3>},
    {512, 8, 4, (void *)bl_layout_kernel<512, 8, 4>},
    {512, 4, 2, (void *)bl_layout_kernel<512, 4, 2>},
    {512, 4, 1, (void *)bl_layout_kernel<512, 4, 1>},
    {512, 2, 1, (void *)bl_layout_kernel<512, 2, 1>},
    {512, 1, 1, (void *)bl_layout_kernel<512, 1, 1>},
};
extern const int bl_exact_v1_count = 6;
