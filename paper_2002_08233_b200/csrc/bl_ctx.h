// bl_ctx.h -- the context behind the opaque bl_ctx handle of include/bl.h,
// shared by the host translation units of libbl (bl_api.cu, bl_metrics.cu).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../../include/bl.h"
#include "bl_kernel.cuh"

struct bl_ctx {
  int32_t n = 0, nnz = 0;
  int device = 0, num_sms = 0;
  int G = 0;  // grid size of the persistent kernel
  int NT = 512; // threads per CTA
  int T = 4;  // register-blocked targets per thread
  int TP = 0; // of which use the paired reciprocal (bl_sweep)
  // device CSR + items
  int *d_rowptr = nullptr, *d_colidx = nullptr;
  int *d_item_ptr = nullptr, *d_item_v = nullptr, *d_item_k0 = nullptr;
  int *d_split_ptr = nullptr;  // items of split vertices below v (BatchLayoutBH)
  int4 *d_sitems = nullptr;    // those items: {item, vertex, k0, k1}
  std::vector<int> item_ptr;  // host copy (per-batch maxima)
  std::vector<int> rowptr_host;  // host copy of rowptr (entry ranges)
  int *d_coo_row = nullptr;      // COO row id per CSR entry (metric helpers)
  // long-row chunks of the standalone CSR walks (a5 alone, EU; bl_attr.cu)
  bool la_ready = false;
  int la_nchunks = 0, la_nlong = 0, la_n1 = 0, la_n2 = 0;
  struct BLAChunk *d_la_chunks = nullptr;
  int2 *d_la_lrow = nullptr;
  float2 *d_la_lpart = nullptr;
  int *d_la_cls = nullptr;  // class-1 then class-2 vertex lists
  unsigned *d_la_bar = nullptr;  // grid-barrier counter of bla_kernel (monotone)
  unsigned la_bar_base = 0;
  int n_items = 0;
  int n_long_rows = 0;  // rows of more than BL_LCOOP entries
  // scratch
  float2 *d_part = nullptr;
  size_t part_cap = 0;  // float2 elements
  float2 *d_pend = nullptr;
  size_t pend_cap = 0;
  float2 *d_attr = nullptr;
  size_t attr_cap = 0;
  double *d_e_cta = nullptr;
  double *d_energy = nullptr;
  size_t energy_cap = 0;
  int *d_iters_done = nullptr;
  unsigned *d_bar = nullptr;
  unsigned long long *d_prof = nullptr;  // BL_PROFILE=1: phase profile
  bool prof = false;
  float2 *d_xy_host_path = nullptr;  // staging for bl_layout (host xy)
  size_t xy_cap = 0;
  // state of the last call
  cudaStream_t last_stream = nullptr;    // stream of the last call (any kind)
  cudaStream_t layout_stream = nullptr;  // stream of the last layout call (bl_energy)
  int32_t last_iters = 0;
  bool have_layout = false;
  int32_t launches = 0;
  std::string err;
  char kname[64] = {0};
  char kname_last[64] = {0};  // the kernel the last layout call launched
  const char *driver_last = "";  // its batch sequencing (bl_driver_name)
  // BatchLayoutBH scratch (allocated on first use, sized by n)
  bool bh_ready = false;
  unsigned *d_keyA = nullptr, *d_keyB = nullptr, *d_hist = nullptr;
  int *d_valA = nullptr, *d_valB = nullptr, *d_cnt = nullptr, *d_off = nullptr, *d_blk = nullptr;
  int *d_nnodes = nullptr;
  float4 *d_bbox = nullptr, *d_nodeA = nullptr;
  float2 *d_snap = nullptr, *d_fb = nullptr;
  size_t fb_cap = 0;
  int4 *d_nodeB = nullptr, *d_nodeC = nullptr;
  double2 *d_nsum = nullptr;
  unsigned long long *d_visits = nullptr;
  bool last_bh = false;
  float2 *d_attr_bh = nullptr;
  unsigned *d_aflag = nullptr;
  uint4 *d_attr_ll = nullptr;  // BH split-row partials with in-word flags (layout mode)
  float2 *d_cellf = nullptr;  // BH per-iteration precomputation
  int *d_nleaf = nullptr, *d_leafv = nullptr;
  // checked builds (-DBL_CHECKED): violation record and phase stamps
  unsigned *d_chk = nullptr, *d_part_st = nullptr, *d_pend_st = nullptr, *d_xy_st = nullptr;
  size_t part_st_cap = 0, pend_st_cap = 0;
  // batch randomisation by relabelling (bl_relabel.cu): pi_it, its inverse and
  // the position-space CSR / coordinates of the current iteration
  int *d_piv = nullptr, *d_inv = nullptr, *d_rowptrP = nullptr, *d_colidxP = nullptr;
  int *d_rl_sum = nullptr, *d_rl_iters = nullptr, *d_rl_stop = nullptr;
  unsigned *d_rl_bar = nullptr;
  float2 *d_xyP = nullptr;
  // quality-metric scratch: grown on first use, kept for the context's life
  // (no allocation inside a metric call after the first)
  void *m_scr[24] = {nullptr};
  size_t m_cap[24] = {0};
  long long m_counters[4] = {0, 0, 0, 0};  // bl_debug_counters
  cudaEvent_t m_ev[2] = {nullptr, nullptr};  // GPU time of the last metric call
};


// record the message (on h, or for bl_create) and return s
bl_status bl_fail(bl_ctx *h, bl_status s, const char *fmt, ...);

#define BL_CUDA(h, call)                                                                    \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      return bl_fail((h), e_ == cudaErrorMemoryAllocation ? BL_ENOMEM : BL_ECUDA, "%s: %s (%s:%d)", \
                  #call, cudaGetErrorString(e_), __FILE__, __LINE__);                       \
  } while (0)


// kernel tables: each lives in its own translation unit (parallel builds)
struct BLVariant {
  int NT, T, TP;
  void *fn;
};
const BLVariant *bl_exact_variants(int *count);     // bl_exact_*.cu
void *bl_bh_kernel_fn();                            // bl_bh.cu
size_t bl_bh_smem_bytes();
int bl_bh_threads();
void *bl_cluster_kernel_fn(int tt, int rmode);      // bl_cluster.cu
// bl_attr.cu: step a5 alone (bl_forces + BL_ATTRACTION_ONLY, one launch), the
// edge-uniformity passes, the COO row ids of the CSR (metric helpers)
bl_status bl_attr_launch(bl_ctx *h, const BLKParams &k, cudaStream_t st);
bl_status bl_coo_rows(bl_ctx *h, cudaStream_t st);
bl_status bl_long_rows(bl_ctx *h);  // degree classes of the rows (bl_attr.cu), built once
bl_status bl_eu_launch(bl_ctx *h, const float2 *xy, int blocks, double *part, double *stats,
                       cudaStream_t st);
int bl_eu_blocks(const bl_ctx *h);  // grid of the edge-uniformity kernel
// bl_relabel.cu: position space of one randomised iteration (one cooperative
// launch), and the final scatter back to vertex space
bl_status bl_relabel_alloc(bl_ctx *h);
void bl_relabel_free(bl_ctx *h);
bl_status bl_relabel_launch(bl_ctx *h, float2 *xy, unsigned long long seed, int shuf_h, int it,
                            int unperm, double tol, cudaStream_t st);
bl_status bl_unrelabel_launch(bl_ctx *h, float2 *xy, int iters, bool tol_stop, cudaStream_t st);
