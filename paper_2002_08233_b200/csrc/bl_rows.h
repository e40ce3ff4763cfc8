// bl_rows.h -- the degree-class work items shared by the CSR walks
// (bla_kernel / bla_eu_kernel in bl_attr.cuh, the stress BFS in
// bl_metrics.cuh); built once per context by bl_long_rows (bl_attr.cu).
#pragma once

// one long-row chunk: vertex, entry range, index of the long row
struct BLAChunk {
  int v, k0, k1, li;
};
