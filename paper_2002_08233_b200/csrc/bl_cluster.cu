// bl_cluster.cu -- instantiations of the single-cluster exact kernel
// (bl_cluster.cuh) in their own translation unit (parallel builds).
#include "bl_ctx.h"
#include "bl_cluster.cuh"

// tt: 0/1/2 = 1/2/4 register-blocked targets; rmode: 0 r = -1, else general r
void *bl_cluster_kernel_fn(int tt, int rmode) {
  static void *fns[3][2] = {{(void *)bl_cluster_kernel<1, 0>, (void *)bl_cluster_kernel<1, -1>},
                            {(void *)bl_cluster_kernel<2, 0>, (void *)bl_cluster_kernel<2, -1>},
                            {(void *)bl_cluster_kernel<4, 0>, (void *)bl_cluster_kernel<4, -1>}};
  return fns[tt][rmode ? 1 : 0];
}
