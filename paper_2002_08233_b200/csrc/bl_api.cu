// bl_api.cu -- host side of libbl: the C-ABI declared in include/bl.h.
//
// Context = device copy of the CSR + the attraction item lists +
// all scratch.  Each layout call is ONE cooperative launch of the persistent
// kernel in bl_kernel.cuh (the paper forks OpenMP once per batch, P:961-966;
// here the dependent batches are walked on the device with grid barriers).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/bl.h"
#include "bl_ctx.h"
#include "bl_bh.cuh"
#include "bl_cluster.cuh"

#ifndef BL_DEFAULT_NT
#define BL_DEFAULT_NT 512
#endif
#ifndef BL_DEFAULT_T
#define BL_DEFAULT_T 8
#endif
#ifndef BL_DEFAULT_TP
#define BL_DEFAULT_TP 1
#endif

static thread_local std::string g_create_err;

bl_status bl_fail(bl_ctx *h, bl_status s, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (h)
    h->err = buf;
  else
    g_create_err = buf;
  return s;
}

extern "C" void bl_params_default(bl_params *p) {
  if (!p) return;
  p->iters = 600;
  p->batch = 256;
  p->K = 1.0f;
  p->C = 1.0f;
  p->step0 = 1.0;
  p->cooling = 0.999;
  p->tol = 0.0;
  p->max_batches = 0;
  p->flags = 0;
  p->algo = BL_ALGO_EXACT;
  p->theta = 1.2f;
  p->a = 2.0f;
  p->r = -1.0f;
  p->shuffle_seed = 0;
}

// (a, r)-energy model codes shared by both kernels (reading C15)
static void model_codes(const bl_params *p, int *amode, int *rmode, float *a_half, float *r_half) {
  *amode = p->a == 2.0f ? 0 : p->a == 1.0f ? 1 : p->a == 0.0f ? 2 : p->a == 3.0f ? 3 : 4;
  *rmode = p->r == -1.0f ? 0 : 1;
  *a_half = 0.5f * (p->a - 1.0f);
  *r_half = 0.5f * (p->r - 1.0f);
}

extern "C" const char *bl_status_string(bl_status s) {
  switch (s) {
    case BL_OK: return "BL_OK";
    case BL_EINVAL: return "BL_EINVAL: invalid argument";
    case BL_ENOMEM: return "BL_ENOMEM: out of memory";
    case BL_ECUDA: return "BL_ECUDA: CUDA error";
    case BL_ESTATE: return "BL_ESTATE: invalid call order";
  }
  return "unknown bl_status";
}

extern "C" const char *bl_last_error(const bl_ctx *h) {
  return h ? h->err.c_str() : g_create_err.c_str();
}

extern "C" int32_t bl_last_launch_count(const bl_ctx *h) { return h ? h->launches : 0; }

extern "C" const char *bl_driver_name(const bl_ctx *h) { return h ? h->driver_last : ""; }

// Checked builds (libbl_checked.so, -DBL_CHECKED): copy the
// violation record of the last exact whole-GPU launch (out[0] = violations,
// out[1] = first code, out[2..4] = its details).  Returns 1 in a checked
// build, 0 in the production library (nothing recorded), -1 on error.
extern "C" int32_t bl_debug_check(bl_ctx *h, uint32_t *out) {
  if (!h || !out) return -1;
#ifdef BL_CHECKED
  for (int i = 0; i < 8; ++i) out[i] = 0;
  if (!h->d_chk) return 1;
  if (cudaStreamSynchronize(h->last_stream) != cudaSuccess) return -1;
  if (cudaMemcpy(out, h->d_chk, sizeof(unsigned) * 5, cudaMemcpyDeviceToHost) != cudaSuccess)
    return -1;
  return 1;
#else
  for (int i = 0; i < 8; ++i) out[i] = 0;
  return 0;
#endif
}

// Work counters (measurement aid): out[0] = BFS levels summed over the
// 64-source groups and out[1] = CSR entries examined by the last bl_stress
// call; out[2] = GPU time (ns) of the last metric call's kernels.
extern "C" int32_t bl_debug_counters(const bl_ctx *h, int64_t *out) {
  if (!h || !out) return -1;
  for (int i = 0; i < 4; ++i) out[i] = h->m_counters[i];
  return 4;
}

extern "C" const char *bl_kernel_name(const bl_ctx *h) {
  return h ? (h->kname_last[0] ? h->kname_last : h->kname) : "";
}

// Debug aid (declared in bl.h): phase profile of the last launch when the
// context was created with BL_PROFILE=1 (bench.py --prof).
extern "C" int32_t bl_debug_profile(bl_ctx *h, unsigned long long *out, int32_t len) {
  if (!h || !h->d_prof || !out) return 0;
  const int m = std::min<int>(len, 16 + h->G);
  if (cudaMemcpy(out, h->d_prof, sizeof(unsigned long long) * m, cudaMemcpyDeviceToHost) != cudaSuccess)
    return 0;
  return m;
}

// static shared memory of the layout kernel (BLShared + locals), reserved
// out of the opt-in maximum before the dynamic buffers are sized
static const int kStaticSmemReserve = (int)sizeof(BLShared) + 1024;

static int env_int(const char *name, int def) {
  const char *s = getenv(name);
  return (s && *s) ? atoi(s) : def;
}

static int red_cap_for(int chunk4) {
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const long long room =
      (long long)optin - 1024 - kStaticSmemReserve - (long long)bl_smem_bytes(chunk4, 0);
  long long cap = room / 8;
  const long long mx = env_int("BL_RED_CAP", BL_RED_MAX);  // tuning override
  if (cap > mx) cap = mx;
  return (int)cap;
}

static int chunk4_for(int n, int G) {
  const int per = (n + G - 1) / G;  // owned sources per CTA (max)
  return std::max(1, (per + 1) / 2);
}


// Kernel variants (NT threads per CTA, T targets per thread, TP of them
// paired-reciprocal), instantiated in bl_exact_*.cu.  NT x registers is one
// SM's register file: 512 x 128, 768 x 80, 1024 x 64.
extern const BLVariant bl_exact_v0[], bl_exact_v1[], bl_exact_v2[], bl_exact_v3[], bl_exact_v4[];
extern const int bl_exact_v0_count, bl_exact_v1_count, bl_exact_v2_count, bl_exact_v3_count,
    bl_exact_v4_count;
// v0: <512,8,2> (default), <512,8,-1> (general repulsion exponent r, reading
// C15); v1: other 512-thread blockings; v2: 768 threads; v3: 1024 threads;
// v4: <256,16,6> (8 warps x 16 targets: best at 2^20 vertices, not at C5)
const BLVariant *bl_exact_variants(int *count) {
  static std::vector<BLVariant> all;
  if (all.empty()) {
    const BLVariant *t[] = {bl_exact_v0, bl_exact_v1, bl_exact_v2, bl_exact_v3, bl_exact_v4};
    const int c[] = {bl_exact_v0_count, bl_exact_v1_count, bl_exact_v2_count, bl_exact_v3_count,
                     bl_exact_v4_count};
    for (int k = 0; k < 5; ++k) all.insert(all.end(), t[k], t[k] + c[k]);
  }
  *count = (int)all.size();
  return all.data();
}

static const BLVariant *find_variant(int NT, int T, int TP) {
  int cnt = 0;
  const BLVariant *v = bl_exact_variants(&cnt);
  for (int i = 0; i < cnt; ++i)
    if (v[i].NT == NT && v[i].T == T && v[i].TP == TP) return &v[i];
  return nullptr;
}

extern "C" int32_t bl_max_vertices(void) {
  int dev = 0, sms = 0, optin = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
    return 0;
  const long long room =
      (long long)optin - 2048 - kStaticSmemReserve - (long long)bl_smem_bytes(0, BL_RED_MIN);
  const long long per = room / (long long)sizeof(float4) * 2;
  const long long n = per * sms;
  return (int32_t)std::min<long long>(n, 0x7fffffff);
}

extern "C" bl_status bl_create(int32_t n, const int32_t *rowptr, const int32_t *colidx,
                               bl_ctx **out) {
  if (!out) return bl_fail(nullptr, BL_EINVAL, "out is NULL");
  *out = nullptr;
  if (n < 1) return bl_fail(nullptr, BL_EINVAL, "n must be >= 1 (got %d)", n);
  if (!rowptr) return bl_fail(nullptr, BL_EINVAL, "rowptr is NULL");
  if (rowptr[0] != 0) return bl_fail(nullptr, BL_EINVAL, "rowptr[0] != 0");
  for (int32_t i = 0; i < n; ++i)
    if (rowptr[i + 1] < rowptr[i]) return bl_fail(nullptr, BL_EINVAL, "rowptr decreases at %d", i);
  const int32_t nnz = rowptr[n];
  if (nnz > 0 && !colidx) return bl_fail(nullptr, BL_EINVAL, "colidx is NULL");
  for (int32_t i = 0; i < n; ++i) {
    for (int32_t k = rowptr[i]; k < rowptr[i + 1]; ++k) {
      const int32_t j = colidx[k];
      if (j < 0 || j >= n) return bl_fail(nullptr, BL_EINVAL, "colidx[%d]=%d out of range", k, j);
      if (j == i) return bl_fail(nullptr, BL_EINVAL, "self loop at vertex %d", i);
      if (k > rowptr[i] && colidx[k - 1] >= j)
        return bl_fail(nullptr, BL_EINVAL, "row %d not strictly ascending", i);
    }
  }
  // symmetry: every (i, j) has (j, i) -- binary search in row j
  for (int32_t i = 0; i < n; ++i) {
    for (int32_t k = rowptr[i]; k < rowptr[i + 1]; ++k) {
      const int32_t j = colidx[k];
      if (!std::binary_search(colidx + rowptr[j], colidx + rowptr[j + 1], i))
        return bl_fail(nullptr, BL_EINVAL, "not symmetric: (%d,%d) without (%d,%d)", i, j, j, i);
    }
  }
  const int32_t nmax = bl_max_vertices();
  if (nmax <= 0) return bl_fail(nullptr, BL_ECUDA, "no usable CUDA device");
  if (n > nmax)
    return bl_fail(nullptr, BL_EINVAL, "n=%d exceeds the resident design limit %d", n, nmax);

  bl_ctx *h = new (std::nothrow) bl_ctx();
  if (!h) return bl_fail(nullptr, BL_ENOMEM, "host allocation failed");
  h->n = n;
  h->nnz = nnz;
  h->rowptr_host.assign(rowptr, rowptr + (size_t)n + 1);
  auto bad = [&](bl_status s) {
    g_create_err = h->err;
    bl_destroy(h);
    return s;
  };
  if (cudaGetDevice(&h->device) != cudaSuccess ||
      cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, h->device) != cudaSuccess)
    return bad(bl_fail(h, BL_ECUDA, "no CUDA device"));
  h->NT = env_int("BL_NT", BL_DEFAULT_NT);
  h->T = env_int("BL_T", BL_DEFAULT_T);
  h->TP = env_int("BL_TP", BL_DEFAULT_TP);
  if (!find_variant(h->NT, h->T, h->TP)) {
    h->NT = BL_DEFAULT_NT;
    h->T = BL_DEFAULT_T;
    h->TP = BL_DEFAULT_TP;
  }
  snprintf(h->kname, sizeof h->kname, "bl_layout_kernel<%d,%d,%d>", h->NT, h->T, h->TP);

  // attraction items: ceil(deg(v)/ECH) per vertex, in vertex order
  h->item_ptr.assign((size_t)n + 1, 0);
  for (int32_t v = 0; v < n; ++v) {
    const int deg = rowptr[v + 1] - rowptr[v];
    h->item_ptr[v + 1] = h->item_ptr[v] + (deg + BL_ECH - 1) / BL_ECH;
  }
  h->n_items = h->item_ptr[n];
  h->n_long_rows = 0;  // rows of more than BL_LCOOP entries (latency driver's cooperative walk)
  for (int32_t v = 0; v < n; ++v) h->n_long_rows += rowptr[v + 1] - rowptr[v] > BL_LCOOP ? 1 : 0;
  // BatchLayoutBH: the items of split vertices (rows of more than one item)
  // as one list in vertex order, {item, vertex, k0, k1} each, with split_ptr[v]
  // = the number of them below vertex v: a batch's edge-parallel pass walks
  // split_ptr[lo] .. split_ptr[hi] only, and its inputs are prefetchable
  std::vector<int> split_ptr((size_t)n + 1, 0);
  std::vector<int4> sitems;
  for (int32_t v = 0; v < n; ++v) {
    const int cnt = h->item_ptr[v + 1] - h->item_ptr[v];
    split_ptr[v + 1] = split_ptr[v] + (cnt > 1 ? cnt : 0);
    if (cnt > 1)
      for (int a = h->item_ptr[v]; a < h->item_ptr[v + 1]; ++a) {
        const int k0 = rowptr[v] + (a - h->item_ptr[v]) * BL_ECH;
        sitems.push_back(make_int4(a, v, k0, std::min(k0 + BL_ECH, (int)rowptr[v + 1])));
      }
  }
  // item_k0 has a sentinel: item_k0[n_items] = nnz, so item a ends at item_k0[a + 1]
  std::vector<int> item_v(std::max(1, h->n_items)), item_k0((size_t)h->n_items + 1, nnz);
  for (int32_t v = 0; v < n; ++v)
    for (int a = h->item_ptr[v]; a < h->item_ptr[v + 1]; ++a) {
      item_v[a] = v;
      item_k0[a] = rowptr[v] + (a - h->item_ptr[v]) * BL_ECH;
    }

#define ALLOC(ptr, bytes)                                                  \
  do {                                                                     \
    cudaError_t e_ = cudaMalloc((void **)&(ptr), (bytes));                 \
    if (e_ != cudaSuccess) return bad(bl_fail(h, BL_ENOMEM, "cudaMalloc %s: %s", #ptr, cudaGetErrorString(e_))); \
  } while (0)
  ALLOC(h->d_rowptr, sizeof(int) * ((size_t)n + 1));
  ALLOC(h->d_colidx, sizeof(int) * std::max<size_t>(1, nnz));
  ALLOC(h->d_item_ptr, sizeof(int) * ((size_t)n + 1));
  ALLOC(h->d_split_ptr, sizeof(int) * ((size_t)n + 1));
  ALLOC(h->d_sitems, sizeof(int4) * std::max<size_t>(1, sitems.size()));
  ALLOC(h->d_item_v, sizeof(int) * item_v.size());
  ALLOC(h->d_item_k0, sizeof(int) * item_k0.size());
  ALLOC(h->d_iters_done, sizeof(int));
  ALLOC(h->d_bar, sizeof(unsigned));
#undef ALLOC
  auto cp = [&](void *dst, const void *src, size_t bytes) {
    return cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice);
  };
  if (cp(h->d_rowptr, rowptr, sizeof(int) * ((size_t)n + 1)) != cudaSuccess ||
      (nnz > 0 && cp(h->d_colidx, colidx, sizeof(int) * (size_t)nnz) != cudaSuccess) ||
      cp(h->d_item_ptr, h->item_ptr.data(), sizeof(int) * ((size_t)n + 1)) != cudaSuccess ||
      cp(h->d_split_ptr, split_ptr.data(), sizeof(int) * ((size_t)n + 1)) != cudaSuccess ||
      (!sitems.empty() &&
       cp(h->d_sitems, sitems.data(), sizeof(int4) * sitems.size()) != cudaSuccess) ||
      cp(h->d_item_v, item_v.data(), sizeof(int) * item_v.size()) != cudaSuccess ||
      cp(h->d_item_k0, item_k0.data(), sizeof(int) * item_k0.size()) != cudaSuccess)
    return bad(bl_fail(h, BL_ECUDA, "CSR upload failed"));

  // grid: one CTA per SM (BL_CTAS_PER_SM overrides), capped by occupancy
  const int per_sm = std::max(1, env_int("BL_CTAS_PER_SM", 1));
  h->G = h->num_sms * per_sm;
  h->prof = env_int("BL_PROFILE", 0) != 0;
  if (h->prof && cudaMalloc((void **)&h->d_prof, sizeof(unsigned long long) * (16 + h->G)) != cudaSuccess)
    return bad(bl_fail(h, BL_ENOMEM, "profile buffer"));
  *out = h;
  return BL_OK;
}

extern "C" void bl_destroy(bl_ctx *h) {
  if (!h) return;
  cudaFree(h->d_rowptr);
  cudaFree(h->d_colidx);
  cudaFree(h->d_item_ptr);
  cudaFree(h->d_split_ptr);
  cudaFree(h->d_sitems);
  cudaFree(h->d_item_v);
  cudaFree(h->d_item_k0);
  cudaFree(h->d_part);
  cudaFree(h->d_attr);
  cudaFree(h->d_pend);
  cudaFree(h->d_e_cta);
  cudaFree(h->d_energy);
  cudaFree(h->d_iters_done);
  cudaFree(h->d_bar);
  cudaFree(h->d_prof);
  cudaFree(h->d_xy_host_path);
  cudaFree(h->d_keyA);
  cudaFree(h->d_keyB);
  cudaFree(h->d_hist);
  cudaFree(h->d_valA);
  cudaFree(h->d_valB);
  cudaFree(h->d_cnt);
  cudaFree(h->d_off);
  cudaFree(h->d_blk);
  cudaFree(h->d_nnodes);
  cudaFree(h->d_bbox);
  cudaFree(h->d_nodeA);
  cudaFree(h->d_snap);
  cudaFree(h->d_fb);
  cudaFree(h->d_nodeB);
  cudaFree(h->d_nodeC);
  cudaFree(h->d_nsum);
  cudaFree(h->d_visits);
  cudaFree(h->d_attr_bh);
  cudaFree(h->d_aflag);
  cudaFree(h->d_attr_ll);
  cudaFree(h->d_cellf);
  cudaFree(h->d_nleaf);
  cudaFree(h->d_leafv);
  for (void *q : h->m_scr) cudaFree(q);
  for (cudaEvent_t e : h->m_ev)
    if (e) cudaEventDestroy(e);
  cudaFree(h->d_coo_row);
  cudaFree(h->d_la_chunks);
  cudaFree(h->d_la_lrow);
  cudaFree(h->d_la_lpart);
  cudaFree(h->d_la_cls);
  cudaFree(h->d_la_bar);
  bl_relabel_free(h);
  cudaFree(h->d_chk);
  cudaFree(h->d_part_st);
  cudaFree(h->d_pend_st);
  cudaFree(h->d_xy_st);
  delete h;
}

static bl_status check_params(bl_ctx *h, const bl_params *p) {
  if (!p) return bl_fail(h, BL_EINVAL, "params is NULL");
  if (p->iters < 0) return bl_fail(h, BL_EINVAL, "iters < 0");
  if (p->batch < 1) return bl_fail(h, BL_EINVAL, "batch < 1");
  if (!(p->K > 0.f) || !std::isfinite(p->K)) return bl_fail(h, BL_EINVAL, "K must be > 0");
  if (!(p->C >= 0.f) || !std::isfinite(p->C)) return bl_fail(h, BL_EINVAL, "C must be >= 0");
  if (!(p->step0 > 0.0) || !std::isfinite(p->step0)) return bl_fail(h, BL_EINVAL, "step0 must be > 0");
  if (!(p->cooling > 0.0 && p->cooling <= 1.0)) return bl_fail(h, BL_EINVAL, "cooling must be in (0,1]");
  if (!(p->tol >= 0.0) || !std::isfinite(p->tol)) return bl_fail(h, BL_EINVAL, "tol must be >= 0");
  if (p->flags & ~(uint32_t)(BL_REPULSE_NEIGHBORS | BL_ATTRACTION_ONLY))
    return bl_fail(h, BL_EINVAL, "unknown flags");
  if ((p->flags & BL_ATTRACTION_ONLY) && p->algo != BL_ALGO_EXACT)
    return bl_fail(h, BL_EINVAL, "BL_ATTRACTION_ONLY needs BL_ALGO_EXACT");
  if (p->algo != BL_ALGO_EXACT && p->algo != BL_ALGO_BH) return bl_fail(h, BL_EINVAL, "unknown algo");
  if (p->algo == BL_ALGO_BH && (!(p->theta >= 0.f) || !std::isfinite(p->theta)))
    return bl_fail(h, BL_EINVAL, "theta must be >= 0");
  if (!(p->a >= 0.f && p->a <= 4.f)) return bl_fail(h, BL_EINVAL, "a must be in [0, 4]");
  if (!(p->r >= -3.f && p->r < 1.f)) return bl_fail(h, BL_EINVAL, "r must be in [-3, 1)");
  if (p->shuffle_seed && p->algo != BL_ALGO_EXACT)
    return bl_fail(h, BL_EINVAL, "shuffle_seed (batch randomisation) needs BL_ALGO_EXACT");
  if (p->shuffle_seed && h && std::min(p->batch, h->n) > BL_TGT_CAP)
    return bl_fail(h, BL_EINVAL, "shuffle_seed needs batch <= %d", BL_TGT_CAP);
  return BL_OK;
}

template <typename P>
static bl_status grow(bl_ctx *h, P *&ptr, size_t &cap, size_t need) {
  if (need <= cap) return BL_OK;
  cudaFree(ptr);
  ptr = nullptr;
  cap = 0;
  cudaError_t e = cudaMalloc((void **)&ptr, need * sizeof(P));
  if (e != cudaSuccess) return bl_fail(h, BL_ENOMEM, "cudaMalloc scratch: %s", cudaGetErrorString(e));
  cap = need;
  return BL_OK;
}

static int max_items_per_batch(const bl_ctx *h, int b, int first, int count) {
  int mx = 1;
  for (int lo = first; lo < first + count; lo += b) {
    const int hi = std::min(lo + b, first + count);
    mx = std::max(mx, h->item_ptr[hi] - h->item_ptr[lo]);
  }
  return mx;
}

// Launch the persistent kernel.  forces_mode: one "batch" [first, first+count)
// whose forces are written to f_out instead of being applied.
// rl (batch randomisation by relabelling, bl_relabel.cu): one iteration in
// position space -- the CSR, energy slot and iteration counter it names
// replace the context's, shuffle_seed is ignored (the batches are contiguous
// there); rl->probe only reports which driver the launch would take.
struct BLRelabelRun {
  const int *rowptr, *colidx;
  double *energy;
  int *iters_done;
  int probe;      // in: 1 = no launch, out: pipelined
  int pipelined;  // out: BLKParams::pipelined of this (n, b)
  int it;         // iteration (checked builds: the violation record is zeroed at it = 0 only)
  const int *stop_in;  // tol > 0: device flag that turns the launch into a no-op
};
static bl_status launch(bl_ctx *h, float2 *d_xy, const bl_params *p, cudaStream_t st,
                        int forces_mode, int first, int count, float2 *f_out,
                        BLRelabelRun *rl = nullptr) {
  const int n = h->n;
  const int b = forces_mode ? std::max(1, count) : std::min(p->batch, n);
  const int G = h->G;
  bl_status s;
  const bool attr_only = forces_mode && (p->flags & BL_ATTRACTION_ONLY);
  if (!attr_only && (s = grow(h, h->d_part, h->part_cap, (size_t)3 * b * G)) != BL_OK) return s;
  if ((s = grow(h, h->d_pend, h->pend_cap, (size_t)2 * b)) != BL_OK) return s;
  const int mi = forces_mode ? max_items_per_batch(h, b, first, count)
                             : max_items_per_batch(h, b, 0, n);
  if ((s = grow(h, h->d_attr, h->attr_cap, (size_t)mi)) != BL_OK) return s;
  if (!h->d_e_cta) {
    size_t cap = 0;
    if ((s = grow(h, h->d_e_cta, cap, (size_t)2 * G)) != BL_OK) return s;
  }
  // the energy trace belongs to the last layout call (bl_energy): forces mode
  // neither writes nor reallocates it
  if (!forces_mode &&
      (s = grow(h, h->d_energy, h->energy_cap, (size_t)std::max(1, p->iters))) != BL_OK)
    return s;

  BLKParams k{};
  k.n = n;
  k.b = b;
  k.nb = (n + b - 1) / b;
  k.iters = p->iters;
  k.max_batches = p->max_batches;
  k.flags = p->flags;
  k.ck2 = p->C * p->K * p->K;
  k.invK = 1.0f / p->K;
  k.step0 = p->step0;
  k.cooling = p->cooling;
  k.tol = p->tol;
  k.chunk4 = chunk4_for(n, G);
  k.forces_mode = forces_mode;
  k.attr_only = attr_only ? 1 : 0;
  k.first = first;
  k.count = count;
  k.xy = d_xy;
  k.rowptr = rl ? rl->rowptr : h->d_rowptr;
  k.colidx = rl ? rl->colidx : h->d_colidx;
  k.item_ptr = h->d_item_ptr;
  k.item_v = h->d_item_v;
  k.item_k0 = h->d_item_k0;
  k.part = h->d_part;
  k.pend = h->d_pend;
  // one barrier per batch needs >= 4 batches per iteration,
  // targets within the staging buffer, an even batch and 16-byte aligned
  // coordinates (16-byte cp.async of target pairs)
  // kernel variant: r != -1 -> <512,8,-1> (two MUFU per pair);
  // latency-bound batches (b <= 512 and
  // b n <= BL_SMALL_PAIRS, default 2^24) -> <512,2,1>: 64-target tiles and
  // >= 4-slot sub-ranges spread each batch's small sweep over all 16 warps
  // instead of a few long units (measured: C2 -17 %, C3 b=256 -29 %, C4 -23 %
  // per batch vs <512,8,2>; C3 b=1024 +34 %: its 16 tiles keep the wide one);
  // else <512,8,1> (round 2, with the unroll-4 sweep, same box: C5 -1.9 %,
  // C6 -3.3 % time vs <512,8,2>; C6 used <256,16,6> before, now 3.3 % slower
  // than <512,8,1>).  BL_NT / BL_T / BL_TP (read at bl_create) pin a variant.
  model_codes(p, &k.amode, &k.rmode, &k.a_half, &k.r_half);
  const long long bn = (long long)b * n;
  const bool user_variant = getenv("BL_NT") || getenv("BL_T") || getenv("BL_TP");
  const bool small_b = !user_variant && b <= 512 &&
                       bn <= (long long)env_int("BL_SMALL_PAIRS", 1 << 24);
  const BLVariant *vt = k.rmode != 0 ? find_variant(512, 8, -1)
                        : small_b && !attr_only ? find_variant(512, 2, 1)
                                              : find_variant(h->NT, h->T, h->TP);
  // batch randomisation (readings R1-R2): the two-barrier driver (its phase U
  // takes batch positions, not owned vertices)
  k.shuf_seed = (forces_mode || rl) ? 0ull : (unsigned long long)p->shuffle_seed;
  k.shuf_h = 1;
  while ((1LL << (2 * k.shuf_h)) < (long long)n) ++k.shuf_h;
  k.pipelined = !forces_mode && k.shuf_seed == 0 && k.nb >= 4 && b <= BL_TGT_CAP && (b % 2) == 0 &&
                (b + G - 1) / G <= BL_ETASK_MAX &&
                red_cap_for(chunk4_for(n, G)) / (((b + 32 * vt->T - 1) / (32 * vt->T)) * 32 * vt->T) >= 2 && (((uintptr_t)d_xy) & 15) == 0 &&
                env_int("BL_PIPELINE", 1) != 0;
  k.part_nbuf = 2;
  k.attr = h->d_attr;
  k.e_cta = h->d_e_cta;
  k.energy = rl ? rl->energy : h->d_energy;
  k.iters_done = rl ? rl->iters_done : h->d_iters_done;
  k.stop_in = rl ? rl->stop_in : nullptr;
  k.bar = h->d_bar;
  k.f_out = f_out;
  k.prof = h->d_prof;
  if (rl) {
    rl->pipelined = k.pipelined;
    // the two-barrier driver's phase U walks the vertex-space items
    if (rl->probe || !k.pipelined) return BL_OK;
  }

  if (attr_only) {
    // step a5 alone: the standalone high-occupancy kernels (bl_attr.cuh)
    model_codes(p, &k.amode, &k.rmode, &k.a_half, &k.r_half);
    if ((s = bl_attr_launch(h, k, st)) != BL_OK) return s;
    snprintf(h->kname_last, sizeof h->kname_last, "bla_kernel");
    h->driver_last = "standalone";
    return BL_OK;
  }
  k.red_cap = red_cap_for(k.chunk4);
  k.guided = env_int("BL_GUIDED", 2);
  k.min_unit4 = std::max(1, env_int("BL_MIN_UNIT4", small_b ? 4 : BL_MIN_UNIT4));
  void *kfn = vt->fn;
  // asynchronous phases (bl_run_async) when each half of the partial buffer
  // still holds >= 2 sub-ranges of the batch's target tiles, and the batch's
  // pair work is not tiny with wide tiles (measured, same box, round 1 with
  // <512,8,2>: C5 +13 %, C3 b=1024 +10 %, C4 +2 %, C3 b=256 -16 %, C2 -22 %;
  // round 2 with the <512,2,1> small-batch variant, async beats pipelined
  // everywhere: C2 6.6 vs 7.4 us, C3 b=256 6.5 vs 7.4, C4 8.8 vs 10.1 per
  // batch).  BL_ASYNC=1 / 0 forces it on / off.
  const int async_env = env_int("BL_ASYNC", -1);
  const bool async_auto = vt->T <= 2 || bn >= (1LL << 22);
  if (k.pipelined && (async_env == 1 || (async_env < 0 && async_auto)) &&
      (b + 32 * vt->T - 1) / (32 * vt->T) <= BL_NTT_MAX &&
      k.red_cap / 2 / (((b + 32 * vt->T - 1) / (32 * vt->T)) * 32 * vt->T) >= 2) {
    k.pipelined = 2;
    k.part_nbuf = 3;
    // fewer, flatter units than the pipelined driver's tail-minimising
    // quadratic profile: with no phase-end barrier the tail is overlapped, and
    // each unit's overhead (target loads, partial stores, combine) counts
    // (measured at C5: 6 sub-ranges, linear profile 0.90 vs 8 quadratic 0.88;
    // round 2 with <512,8,1>: equal sizes 0.2 % faster than linear)
    k.guided = env_int("BL_GUIDED", 0);
    k.nsub_max = std::max(2, env_int("BL_NSUB", 6));
    k.spin_max = (unsigned)std::max(32, env_int("BL_SPIN", 512));
    k.afence_gpu = env_int("BL_AFENCE", 0);
    // only what two phases of nsub_max sub-ranges use: the rest of the shared
    // memory goes back to L1 (update-task gathers, partial rows)
    const int tile_slots = ((b + 32 * vt->T - 1) / (32 * vt->T)) * 32 * vt->T;
    k.red_cap = std::min(k.red_cap, 2 * k.nsub_max * tile_slots);
  }
  // latency driver (bl_run_lat): updater warps = owned vertices per batch
  // per CTA (<= half the warps), every tile's clean sub-ranges plus one in
  // each half of red.  The default where the pair work per batch is small
  // (b n <= BL_SMALL_PAIRS, 2^24): measured same box vs the asynchronous
  // driver, us per dependent batch: C2 6.17 -> 4.28, C3 b=256 5.83 -> 4.21,
  // C3 b=1024 10.95 -> 7.36, C4 8.54 -> 6.72.  BL_LAT=1 / 0
  // forces it on / off; BL_ASYNC=0/1 (pipelined / asynchronous) also turns
  // it off.
  {
    const int lat_env = env_int("BL_LAT", -1);
    const bool lat_auto = lat_env < 0 && async_env < 0 &&
                          bn <= (long long)env_int("BL_SMALL_PAIRS", 1 << 24);
    const int ntt = (b + 32 * vt->T - 1) / (32 * vt->T);
    const int U = (b + G - 1) / G;
    const int red_lat = red_cap_for(k.chunk4);
    const bool lat_ok = k.pipelined && U <= vt->NT / 64 && ntt <= BL_NTT_MAX &&
                        red_lat / 2 / (ntt * 32 * vt->T) >= 2 && n >= 2 * G;
    if (lat_ok && (lat_env == 1 || lat_auto)) {
      k.pipelined = 3;
      k.part_nbuf = 2;
      k.red_cap = red_lat;
      k.guided = env_int("BL_GUIDED", 1);
      k.nsub_max = std::max(2, env_int("BL_NSUB", 6));
    }
  }
#ifdef BL_CHECKED
  // checked build: zeroed violation record and stamps for this launch
  if (!h->d_chk) {
    if (cudaMalloc((void **)&h->d_chk, sizeof(unsigned) * 8) != cudaSuccess ||
        cudaMalloc((void **)&h->d_xy_st, sizeof(unsigned) * (size_t)n) != cudaSuccess)
      return bl_fail(h, BL_ENOMEM, "checked-build buffers");
  }
  if ((s = grow(h, h->d_part_st, h->part_st_cap, (size_t)3 * b * G)) != BL_OK) return s;
  if ((s = grow(h, h->d_pend_st, h->pend_st_cap, (size_t)2 * b)) != BL_OK) return s;
  if (!rl || rl->it == 0) BL_CUDA(h, cudaMemsetAsync(h->d_chk, 0, sizeof(unsigned) * 8, st));
  BL_CUDA(h, cudaMemsetAsync(h->d_xy_st, 0, sizeof(unsigned) * (size_t)n, st));
  BL_CUDA(h, cudaMemsetAsync(h->d_part_st, 0, sizeof(unsigned) * h->part_st_cap, st));
  BL_CUDA(h, cudaMemsetAsync(h->d_pend_st, 0, sizeof(unsigned) * h->pend_st_cap, st));
  k.chk = h->d_chk;
  k.part_st = h->d_part_st;
  k.pend_st = h->d_pend_st;
  k.xy_st = h->d_xy_st;
  k.jitter = (unsigned)env_int("BL_JITTER", 0);
  k.chk_break = env_int("BL_CHK_BREAK", 0);
#endif
  // long CSR rows in update tasks: 8 gathers in flight per lane on the async
  // driver (measured +1.4 % at C5, -1..2 % on the latency-bound configs with
  // sequential batches, whose hubs sit in the first batches); with relabelled
  // randomised batches every batch holds hub rows (BL_LONG8 overrides)
  k.long8 = env_int("BL_LONG8", (k.pipelined == 2 || rl) ? 1 : 0);
  // latency driver: long rows walked by all updater warps together where the
  // graph has enough of them to meet one in most batches (>= one row of more
  // than BL_LCOOP entries per 8 batches; measured same box: C4 1,157 -> 1,295
  // it/s, relabelled C4 1.29 -> 0.94 ms per iteration; the hub-free configs
  // keep the plain instance, which the walk would cost 6 %)
  k.lcoop = vt->T <= 2 ? env_int("BL_LCOOP", (long long)h->n_long_rows * 8 >= k.nb ? 1 : 0) : 0;
  const size_t smem = bl_smem_bytes(k.chunk4, k.red_cap);
  snprintf(h->kname_last, sizeof h->kname_last, "bl_layout_kernel<%d,%d,%d>", vt->NT, vt->T, vt->TP);
  h->driver_last = forces_mode ? "two-barrier"
                   : k.pipelined == 3 ? "latency"
                   : k.pipelined == 2 ? "async"
                   : k.pipelined      ? "pipelined"
                                      : "two-barrier";
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return bl_fail(h, BL_ECUDA, "smem attribute (%zu B): %s", smem, cudaGetErrorString(e));
  int occ = 0;
  BL_CUDA(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, vt->NT, smem));
  if (occ * h->num_sms < G)
    return bl_fail(h, BL_ECUDA, "cooperative grid %d exceeds residency %d x %d SMs", G, occ, h->num_sms);

  BL_CUDA(h, cudaMemsetAsync(h->d_bar, 0, sizeof(unsigned), st));
  // forces mode never writes iters_done: leave the last layout call's count
  // (and its energy trace) to bl_energy
  if (!forces_mode) BL_CUDA(h, cudaMemsetAsync(k.iters_done, 0, sizeof(int), st));
  if (h->d_prof) BL_CUDA(h, cudaMemsetAsync(h->d_prof, 0, sizeof(unsigned long long) * (16 + G), st));
  void *args[] = {&k};
  BL_CUDA(h, cudaLaunchCooperativeKernel(kfn, dim3(G), dim3(vt->NT), args, smem, st));
  h->launches = 1;
  return BL_OK;
}

// BatchLayoutBH: one cooperative launch of bl_bh_kernel (csrc/bl_bh.cuh).
static bl_status launch_bh(bl_ctx *h, float2 *d_xy, const bl_params *p, cudaStream_t st,
                           int forces_mode, int first, int count, float2 *f_out) {
  const int n = h->n, G = h->num_sms;
  const int b = forces_mode ? std::max(1, count) : std::min(p->batch, n);
  bl_status s;
  if (!h->bh_ready) {
    const size_t cap = (size_t)17 * n + 1;  // <= 17 nodes per sorted position
#define ALLOC(ptr, cnt)                                                                       \
  do {                                                                                        \
    cudaError_t e_ = cudaMalloc((void **)&(ptr), sizeof(*(ptr)) * (size_t)(cnt));             \
    if (e_ != cudaSuccess) return bl_fail(h, BL_ENOMEM, "cudaMalloc %s: %s", #ptr, cudaGetErrorString(e_)); \
  } while (0)
    ALLOC(h->d_keyA, n);
    ALLOC(h->d_keyB, n);
    ALLOC(h->d_valA, n);
    ALLOC(h->d_valB, n);
    ALLOC(h->d_hist, 256 * G);
    ALLOC(h->d_bbox, G);
    ALLOC(h->d_cnt, n);
    ALLOC(h->d_off, n + 1);
    ALLOC(h->d_blk, G);
    ALLOC(h->d_snap, n);
    ALLOC(h->d_nodeA, cap);
    ALLOC(h->d_nodeB, cap);
    ALLOC(h->d_nodeC, cap);
    ALLOC(h->d_nsum, cap);
    ALLOC(h->d_nnodes, 1);
    ALLOC(h->d_visits, G);
    ALLOC(h->d_attr_bh, std::max(1, h->n_items));
    ALLOC(h->d_aflag, std::max(1, h->n_items));
    ALLOC(h->d_attr_ll, std::max(1, h->n_items));
    ALLOC(h->d_cellf, n);
    ALLOC(h->d_nleaf, n);
    ALLOC(h->d_leafv, (size_t)n * BH_LCAP);
#undef ALLOC
    h->bh_ready = true;
  }
  if ((s = grow(h, h->d_fb, h->fb_cap, (size_t)2 * b)) != BL_OK) return s;  // pend[2][b]
  if (!h->d_e_cta) {
    size_t cap = 0;
    if ((s = grow(h, h->d_e_cta, cap, (size_t)2 * G)) != BL_OK) return s;
  }
  if (!forces_mode &&
      (s = grow(h, h->d_energy, h->energy_cap, (size_t)std::max(1, p->iters))) != BL_OK)
    return s;
  BHKParams k{};
  k.n = n;
  k.b = b;
  k.nb = (n + b - 1) / b;
  k.iters = p->iters;
  k.max_batches = p->max_batches;
  k.ck2 = p->C * p->K * p->K;
  k.invK = 1.0f / p->K;
  const float th = p->theta;
  k.theta2 = th * th;  // fp32, as the oracle (reading B7)
  model_codes(p, &k.amode, &k.rmode, &k.a_half, &k.r_half);
  k.step0 = p->step0;
  k.cooling = p->cooling;
  k.tol = p->tol;
  k.forces_mode = forces_mode;
  k.first = first;
  k.count = count;
  k.xy = d_xy;
  k.rowptr = h->d_rowptr;
  k.colidx = h->d_colidx;
  k.keyA = h->d_keyA;
  k.keyB = h->d_keyB;
  k.valA = h->d_valA;
  k.valB = h->d_valB;
  k.hist = h->d_hist;
  k.bbox = h->d_bbox;
  k.cnt = h->d_cnt;
  k.off = h->d_off;
  k.blk = h->d_blk;
  k.snap = h->d_snap;
  k.nodeA = h->d_nodeA;
  k.nodeB = h->d_nodeB;
  k.nodeC = h->d_nodeC;
  k.nsum = h->d_nsum;
  k.nnodes = h->d_nnodes;
  k.pend = h->d_fb;
  k.prof = h->d_prof;
  k.item_ptr = h->d_item_ptr;
  k.item_v = h->d_item_v;
  k.item_k0 = h->d_item_k0;
  k.attr = h->d_attr_bh;
  k.aflag = h->d_aflag;
  k.attr_ll = h->d_attr_ll;
  k.cellf = h->d_cellf;
  k.nleaf = h->d_nleaf;
  k.leafv = h->d_leafv;
  k.precompute = !forces_mode && env_int("BL_BH_PRE", 1) != 0;
  k.pre2 = env_int("BL_BH_PRE2", 1) != 0;
  k.split_ptr = h->d_split_ptr;
  k.sitems = h->d_sitems;
  k.e_cta = h->d_e_cta;
  k.energy = h->d_energy;
  k.iters_done = h->d_iters_done;
  k.bar = h->d_bar;
  k.f_out = f_out;
  k.visits = h->d_visits;
  void *kfn = bl_bh_kernel_fn();
  const size_t smem = bl_bh_smem_bytes();
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return bl_fail(h, BL_ECUDA, "bh smem attribute (%zu B): %s", smem, cudaGetErrorString(e));
  int occ = 0;
  BL_CUDA(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, bl_bh_threads(), smem));
  if (occ < 1) return bl_fail(h, BL_ECUDA, "bh kernel does not fit an SM");
  BL_CUDA(h, cudaMemsetAsync(h->d_bar, 0, sizeof(unsigned), st));
  if (!forces_mode) BL_CUDA(h, cudaMemsetAsync(h->d_iters_done, 0, sizeof(int), st));
  BL_CUDA(h, cudaMemsetAsync(h->d_visits, 0, sizeof(unsigned long long) * G, st));
  BL_CUDA(h, cudaMemsetAsync(h->d_aflag, 0, sizeof(unsigned) * std::max(1, h->n_items), st));
  if (!forces_mode && k.pre2)
    BL_CUDA(h, cudaMemsetAsync(h->d_attr_ll, 0, sizeof(uint4) * std::max(1, h->n_items), st));
  void *args[] = {&k};
  BL_CUDA(h, cudaLaunchCooperativeKernel(kfn, dim3(G), dim3(bl_bh_threads()), args, smem, st));
  h->launches = 1;
  h->last_bh = true;
  return BL_OK;
}

// Small graphs: the exact method on one thread-block cluster (bl_cluster.cuh)
// when a batch's work is small enough that the whole-GPU kernel's per-batch
// grid barrier dominates (b n <= BL_CLUSTER_PAIRS, default 6e5: the measured
// crossover against the latency driver on B200) and the
// coordinates fit every CTA's shared memory.  Returns BL_OK and sets *used.
// rl: one relabelled iteration (see launch).
static bl_status launch_cluster(bl_ctx *h, float2 *d_xy, const bl_params *p, cudaStream_t st,
                                bool *used, BLRelabelRun *rl = nullptr) {
  *used = false;
  const int n = h->n, b = std::min(p->batch, n);
  if (env_int("BL_CLUSTER", 1) == 0) return BL_OK;
  if (p->shuffle_seed) return BL_OK;  // randomised batches: relabelled, else the two-barrier driver
  // crossover against the latency driver, re-measured in round 2 on grids
  // (scripts/cluster_vs_lat.py, us per batch cluster / latency): b n = 262k
  // 3.2 / 4.2, 352k 3.5 / 3.7, 512k 3.9 / 4.0, 704k 4.3 / 3.8, 1.05M 5.0-6.6 /
  // 3.8-4.2 (round 1, against the pipelined driver: 1e6)
  const long long pairs_max = env_int("BL_CLUSTER_PAIRS", 600000);
  if ((long long)b * n > pairs_max) return BL_OK;
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const int n4 = (n + 1) / 2;
  size_t smem = blc_smem_bytes(n4, b);
  if (smem + 2048 > (size_t)optin) return BL_OK;
  // the CSR too, when it fits (one L2 round trip less per row per batch)
  const size_t csr_bytes = sizeof(int) * ((size_t)n + 1 + (size_t)h->nnz);
  const bool csr_smem = smem + csr_bytes + 2048 <= (size_t)optin;
  if (csr_smem) smem += csr_bytes;
  int amode, rmode;
  float a_half, r_half;
  model_codes(p, &amode, &rmode, &a_half, &r_half);
  // cluster size: 16 (non-portable) if the device can co-schedule it, else 8
  int CS = 0;
  const int tsel = env_int("BL_CLUSTER_T", 0);  // 0: by slice size
  for (int cs : {16, 8}) {
    const int sl = (b + cs - 1) / cs;
    if (sl > BLC_SLICE_MAX) continue;
    const int tt = tsel == 1 ? 0 : tsel == 2 ? 1 : tsel == 4 ? 2 : (sl <= 16 ? 0 : 1);
    void *kfn = bl_cluster_kernel_fn(tt, rmode);
    if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      continue;
    if (cs > 8 && cudaFuncSetAttribute(kfn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
      continue;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(BLC_NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, kfn, &cfg) != cudaSuccess || nclusters < 1) {
      cudaGetLastError();
      continue;
    }
    CS = cs;
    if (rl && rl->probe) {
      *used = true;
      return BL_OK;
    }
    bl_status s;
    if ((s = grow(h, h->d_energy, h->energy_cap, (size_t)std::max(1, p->iters))) != BL_OK) return s;
    BLCParams k{};
    k.n = n;
    k.b = b;
    k.nb = (n + b - 1) / b;
    k.iters = p->iters;
    k.max_batches = p->max_batches;
    k.flags = p->flags;
    k.ck2 = p->C * p->K * p->K;
    k.invK = 1.0f / p->K;
    k.step0 = p->step0;
    k.cooling = p->cooling;
    k.tol = p->tol;
    k.amode = amode;
    k.rmode = rmode;
    k.a_half = a_half;
    k.r_half = r_half;
    k.n4 = n4;
    k.nnz = h->nnz;
    k.csr_smem = csr_smem ? 1 : 0;
    k.xy = d_xy;
    k.rowptr = rl ? rl->rowptr : h->d_rowptr;
    k.colidx = rl ? rl->colidx : h->d_colidx;
    k.energy = rl ? rl->energy : h->d_energy;
    k.iters_done = rl ? rl->iters_done : h->d_iters_done;
    BL_CUDA(h, cudaMemsetAsync(k.iters_done, 0, sizeof(int), st));
    void *args[] = {&k};
    BL_CUDA(h, cudaLaunchKernelExC(&cfg, kfn, args));
    h->launches = 1;
    snprintf(h->kname_last, sizeof h->kname_last, "bl_cluster_kernel<%d,%d> x%d", 1 << tt,
             rmode ? -1 : 0, CS);
    h->driver_last = "cluster";
    *used = true;
    return BL_OK;
  }
  (void)CS;
  return BL_OK;
}

extern "C" bl_status bl_last_visits(bl_ctx *h, unsigned long long *visits) {
  if (!h || !visits) return bl_fail(h, BL_EINVAL, "NULL argument");
  *visits = 0;
  if (!h->last_bh || !h->d_visits) return BL_OK;
  BL_CUDA(h, cudaStreamSynchronize(h->last_stream));
  std::vector<unsigned long long> v(h->num_sms);
  BL_CUDA(h, cudaMemcpy(v.data(), h->d_visits, sizeof(unsigned long long) * v.size(),
                        cudaMemcpyDeviceToHost));
  for (auto x : v) *visits += x;
  return BL_OK;
}

// Batch randomisation by relabelling (bl_relabel.cu): every
// iteration is one relabel launch + one plain launch of the layout kernel in
// position space, with whatever sequential driver (asynchronous, latency,
// pipelined) the size takes.  Taken when the whole-GPU kernel would run one of
// those drivers; BL_SHUFFLE_RELABEL=0 turns it off.  tol > 0 stays a
// device-side decision: the relabel launch of iteration it >= 2 tests
// |E[it-1] - E[it-2]| < tol in every CTA alike, books iters_done = it and
// sets a flag that makes the remaining launches of the call no-ops (the
// layout kernel checks BLKParams::stop_in first); the single-cluster kernel
// has no such check, so tol > 0 takes the whole-GPU kernel.
// max_batches: the iteration that exhausts the budget gets the rest of it.  The Step of iteration it is
// step0 cooling^it by the same repeated fp64 product as in the kernel.
static bl_status layout_relabel(bl_ctx *h, float2 *d_xy, const bl_params *p, cudaStream_t st,
                                bool *used) {
  *used = false;
  if (!p->shuffle_seed || p->algo != BL_ALGO_EXACT || env_int("BL_SHUFFLE_RELABEL", 1) == 0)
    return BL_OK;
  bl_status s = bl_relabel_alloc(h);
  if (s != BL_OK) return s;
  bl_params q = *p;
  q.iters = 1;
  q.shuffle_seed = 0;
  q.max_batches = 0;
  q.tol = 0.0;  // the stop rule runs between the launches
  const bool tol_stop = p->tol > 0.0;
  BLRelabelRun rl{h->d_rowptrP, h->d_colidxP, nullptr, h->d_rl_iters, 1, 0, 0, nullptr};
  bool cluster = false;
  if (!tol_stop && (s = launch_cluster(h, h->d_xyP, &q, st, &cluster, &rl)) != BL_OK) return s;
  if (!cluster) {
    if ((s = launch(h, h->d_xyP, &q, st, 0, 0, 0, nullptr, &rl)) != BL_OK) return s;
    if (!rl.pipelined) return BL_OK;
  }
  if ((s = grow(h, h->d_energy, h->energy_cap, (size_t)std::max(1, p->iters))) != BL_OK) return s;
  int shuf_h = 1;
  while ((1LL << (2 * shuf_h)) < (long long)h->n) ++shuf_h;
  rl.probe = 0;
  rl.stop_in = tol_stop ? h->d_rl_stop : nullptr;
  if (tol_stop) BL_CUDA(h, cudaMemsetAsync(h->d_rl_stop, 0, sizeof(int), st));
  double step = p->step0;
  int launches = 0, done = 0;
  const int b = std::min(p->batch, h->n);
  const long long nb = (h->n + b - 1) / b;
  for (int it = 0; it < p->iters; ++it) {
    const long long left = p->max_batches > 0 ? p->max_batches - it * nb : nb + 1;
    if ((s = bl_relabel_launch(h, d_xy, (unsigned long long)p->shuffle_seed, shuf_h, it, it > 0,
                               p->tol, st)) != BL_OK)
      return s;
    q.step0 = step;
    q.max_batches = left <= nb ? (int)left : 0;  // the budget ends inside this iteration
    rl.energy = h->d_energy + it;
    rl.it = it;
    s = cluster ? launch_cluster(h, h->d_xyP, &q, st, &cluster, &rl)
                : launch(h, h->d_xyP, &q, st, 0, 0, 0, nullptr, &rl);
    if (s != BL_OK) return s;
    launches += 2;
    if (left <= nb) break;  // iters_done counts completed iterations (as every driver)
    done = it + 1;
    step = step * p->cooling;
  }
  if ((s = bl_unrelabel_launch(h, d_xy, done, tol_stop, st)) != BL_OK) return s;
  h->launches = launches + 1;
  const std::string d = h->driver_last;
  h->driver_last = d == "async"     ? "relabel+async"
                   : d == "latency" ? "relabel+latency"
                   : d == "cluster" ? "relabel+cluster"
                                    : "relabel+pipelined";
  *used = true;
  return BL_OK;
}

extern "C" bl_status bl_layout_device(bl_ctx *h, float *d_xy, const bl_params *p, void *cuda_stream) {
  if (!h) return bl_fail(nullptr, BL_EINVAL, "handle is NULL");
  h->launches = 0;
  bl_status s = check_params(h, p);
  if (s != BL_OK) return s;
  if (!d_xy) return bl_fail(h, BL_EINVAL, "d_xy is NULL");
  if (((uintptr_t)d_xy) & 7) return bl_fail(h, BL_EINVAL, "d_xy must be 8-byte aligned");
  if (p->flags & BL_ATTRACTION_ONLY) return bl_fail(h, BL_EINVAL, "BL_ATTRACTION_ONLY is for bl_forces");
  cudaStream_t st = (cudaStream_t)cuda_stream;
  h->last_stream = st;
  h->layout_stream = st;
  h->last_iters = p->iters;
  if (p->iters == 0) {
    h->have_layout = false;
    return BL_OK;
  }
  h->last_bh = false;
  snprintf(h->kname_last, sizeof h->kname_last, "%s", p->algo == BL_ALGO_BH ? "bl_bh_kernel<512>" : h->kname);
  h->driver_last = p->algo == BL_ALGO_BH ? "bh" : "";
  bool clustered = false;
  if (p->algo == BL_ALGO_EXACT && p->shuffle_seed) {
    s = layout_relabel(h, reinterpret_cast<float2 *>(d_xy), p, st, &clustered);
    if (s != BL_OK) return s;
  }
  if (p->algo == BL_ALGO_EXACT && !clustered) {
    s = launch_cluster(h, reinterpret_cast<float2 *>(d_xy), p, st, &clustered);
    if (s != BL_OK) return s;
  }
  if (!clustered)
    s = p->algo == BL_ALGO_BH ? launch_bh(h, reinterpret_cast<float2 *>(d_xy), p, st, 0, 0, 0, nullptr)
                              : launch(h, reinterpret_cast<float2 *>(d_xy), p, st, 0, 0, 0, nullptr);
  if (s != BL_OK) return s;
  h->have_layout = true;
  return BL_OK;
}

extern "C" bl_status bl_layout(bl_ctx *h, float *xy, const bl_params *p, int32_t *iters_done) {
  if (!h) return bl_fail(nullptr, BL_EINVAL, "handle is NULL");
  bl_status s = check_params(h, p);
  if (s != BL_OK) return s;
  if (!xy) return bl_fail(h, BL_EINVAL, "xy is NULL");
  for (int32_t i = 0; i < 2 * h->n; ++i)
    if (!std::isfinite(xy[i])) return bl_fail(h, BL_EINVAL, "non-finite coordinate at %d", i);
  if ((s = grow(h, h->d_xy_host_path, h->xy_cap, (size_t)h->n)) != BL_OK) return s;
  cudaStream_t st = nullptr;
  BL_CUDA(h, cudaMemcpyAsync(h->d_xy_host_path, xy, sizeof(float2) * h->n, cudaMemcpyHostToDevice, st));
  s = bl_layout_device(h, reinterpret_cast<float *>(h->d_xy_host_path), p, st);
  if (s != BL_OK) return s;
  BL_CUDA(h, cudaMemcpyAsync(xy, h->d_xy_host_path, sizeof(float2) * h->n, cudaMemcpyDeviceToHost, st));
  BL_CUDA(h, cudaStreamSynchronize(st));
  BL_CUDA(h, cudaGetLastError());
  if (iters_done) {
    int d = 0;
    if (p->iters > 0) BL_CUDA(h, cudaMemcpy(&d, h->d_iters_done, sizeof(int), cudaMemcpyDeviceToHost));
    *iters_done = d;
  }
  return BL_OK;
}

extern "C" bl_status bl_energy(bl_ctx *h, double *e_last, double *trace, int32_t trace_len,
                               int32_t *n_written, int32_t *iters_done) {
  if (!h) return bl_fail(nullptr, BL_EINVAL, "handle is NULL");
  if (trace_len < 0) return bl_fail(h, BL_EINVAL, "trace_len < 0");
  if (!h->have_layout) return bl_fail(h, BL_ESTATE, "no layout call has run an iteration");
  BL_CUDA(h, cudaStreamSynchronize(h->layout_stream));
  int d = 0;
  BL_CUDA(h, cudaMemcpy(&d, h->d_iters_done, sizeof(int), cudaMemcpyDeviceToHost));
  if (iters_done) *iters_done = d;
  const int avail = std::min(d, h->last_iters);
  if (n_written) *n_written = 0;
  if (trace && trace_len > 0 && avail > 0) {
    const int m = std::min(avail, trace_len);
    BL_CUDA(h, cudaMemcpy(trace, h->d_energy, sizeof(double) * m, cudaMemcpyDeviceToHost));
    if (n_written) *n_written = m;
  }
  if (e_last) {
    if (avail == 0) return bl_fail(h, BL_ESTATE, "no completed iteration");
    BL_CUDA(h, cudaMemcpy(e_last, h->d_energy + (avail - 1), sizeof(double), cudaMemcpyDeviceToHost));
  }
  return BL_OK;
}

extern "C" bl_status bl_forces(bl_ctx *h, const float *d_xy, int32_t first, int32_t count,
                               float *d_f_out, const bl_params *p, void *cuda_stream) {
  if (!h) return bl_fail(nullptr, BL_EINVAL, "handle is NULL");
  h->launches = 0;
  bl_status s = check_params(h, p);
  if (s != BL_OK) return s;
  if (!d_xy || !d_f_out) return bl_fail(h, BL_EINVAL, "NULL pointer");
  if (first < 0 || count < 0 || first > h->n - count)
    return bl_fail(h, BL_EINVAL, "range [%d, %d+%d) outside [0, %d)", first, first, count, h->n);
  if (count == 0) return BL_OK;
  h->last_stream = (cudaStream_t)cuda_stream;
  h->last_bh = false;
  float2 *xy2 = const_cast<float2 *>(reinterpret_cast<const float2 *>(d_xy));
  if (p->algo == BL_ALGO_BH)
    return launch_bh(h, xy2, p, (cudaStream_t)cuda_stream, 1, first, count,
                     reinterpret_cast<float2 *>(d_f_out));
  return launch(h, xy2, p, (cudaStream_t)cuda_stream, 1, first, count,
                reinterpret_cast<float2 *>(d_f_out));
}

