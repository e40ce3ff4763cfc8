// bl_bh.cuh -- BatchLayoutBH on sm_100a: Barnes-Hut repulsion (device side).
//
// Alg. S3 of the supplement with the quadtree of Alg. S1
// and the traversal of Alg. S2, §3.5.
// One persistent cooperative kernel per call walks, for every iteration:
//
//   build (from the coordinates at the iteration start, reading B5):
//     B0  bounding box (grid min/max) -> D = max extent (Alg. S3 line 7)
//     B1  16+16-bit Morton codes in fp32 (reading B6/B7)
//     B2  stable LSD radix sort of (code, vertex id), 4 x 8-bit passes:
//         per-CTA digit histograms, a fixed-order prefix, and a stable
//         in-CTA scatter ranked with __match_any_sync (Alg. S3 line 6)
//     B3  node enumeration: position i of the sorted order starts the
//         segments of levels delta(i)+1 .. (until it is alone), delta = common
//         Morton prefix (in 2-bit digits) with its predecessor; a scan of the
//         per-position counts gives every node its PRE-ORDER index
//     B4  node records: level, start, count (galloping search for the end of
//         the segment), skip pointer (= index of the first node after the
//         subtree = offset of the segment end), children lists
//     B5  centroids bottom-up, level 15 -> 0, fp64 sums of the children in
//         digit order (identical arithmetic to the oracle, reading B7)
//   minibatches (Alg. S3 lines 12-24), per batch:
//     F   one warp per batch vertex: CSR attraction with the live
//         coordinates + Barnes-Hut repulsion by a warp-wide frontier
//         traversal (all frontier nodes of a level tested by the 32 lanes in
//         parallel; MAC in fp32 exactly as the oracle; leaves use the live
//         coordinates; a lane whose children overflow the frontier walks that
//         subtree alone with the skip pointers) -> fb[batch]
//     grid barrier
//     U   owner update c += Step f/||f||, energy in fp64 (fixed order)
//     grid barrier
#pragma once
#include "bl_kernel.cuh"

#define BH_NT 512
#define BH_NW (BH_NT / 32)
#define BH_FCAP 512  // frontier entries per buffer per warp

struct BHKParams {
  int n, b, nb, iters, max_batches;
  float ck2, invK, theta2;
  double step0, cooling, tol;
  int forces_mode, first, count;
  float2 *xy;
  const int *rowptr, *colidx;
  unsigned *keyA, *keyB;
  int *valA, *valB;
  unsigned *hist;     // [256][G]
  float4 *bbox;       // [G]
  int *cnt;           // [n] node count per sorted position, then exclusive offsets
  int *off;           // [n + 1]
  int *blk;           // [G]
  float2 *snap;       // [n] sorted snapshot coordinates
  float4 *nodeA;      // [cap] centroid x, y, D_L^2, count
  int4 *nodeB;        // [cap] level | nchild << 8 | leaf << 16, start, count, skip
  int4 *nodeC;        // [cap] children (-1 padded)
  double2 *nsum;      // [cap] fp64 coordinate sums
  int *nnodes;        // [1]
  float2 *fb;         // [b] forces of the running batch
  double *e_cta;      // [G]
  double *energy;     // [iters]
  int *iters_done;
  unsigned *bar;
  float2 *f_out;
  unsigned long long *visits;  // [G] node visits per CTA (for the roofline)
};

struct BHShared {
  unsigned hist[256];
  unsigned base[256];
  unsigned wcnt[BH_NW][256];
  int frontier[BH_NW][2][BH_FCAP];
  float4 red4[BH_NW];
  double e_warp[BH_NW];
  int scan[BH_NW];
  float D;
  float xmin, ymin, scale;
  int degenerate;
};

__device__ __forceinline__ unsigned bh_interleave(unsigned qx, unsigned qy) {
  // spread the 16 bits of qx to the even bits, qy to the odd bits
  auto spread = [](unsigned v) {
    v &= 0xFFFFu;
    v = (v | (v << 8)) & 0x00FF00FFu;
    v = (v | (v << 4)) & 0x0F0F0F0Fu;
    v = (v | (v << 2)) & 0x33333333u;
    v = (v | (v << 1)) & 0x55555555u;
    return v;
  };
  return spread(qx) | (spread(qy) << 1);
}

__device__ __forceinline__ unsigned bh_quant(float x, float xmin, float scale, int degenerate) {
  if (degenerate) return 0u;
  const float t = __fmul_rn(__fsub_rn(x, xmin), scale);  // no contraction (reading B7)
  float fl = floorf(t);
  fl = fminf(fmaxf(fl, 0.0f), 65535.0f);
  return (unsigned)fl;
}

// common Morton prefix of two codes in 2-bit digits (16 if equal)
__device__ __forceinline__ int bh_delta(unsigned a, unsigned b) {
  const unsigned x = a ^ b;
  return x == 0u ? 16 : (__clz(x) >> 1);
}

__device__ __forceinline__ unsigned bh_prefix(unsigned code, int L) {
  return L == 0 ? 0u : (L >= 16 ? code : (code >> (32 - 2 * L)));
}

// chunk of the vertex / position range owned by CTA c
__device__ __forceinline__ void bh_chunk(int n, int &lo, int &hi) {
  const int G = gridDim.x, c = blockIdx.x;
  const int per = (n + G - 1) / G;
  lo = min(n, c * per);
  hi = min(n, lo + per);
}

// Block-wide exclusive scan of one int per thread (fixed order); returns the
// block total through *total.
__device__ __forceinline__ int bh_block_scan(int v, BHShared &sh, int *total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh.scan[warp] = x;
  __syncthreads();
  int wpre = 0, tot = 0;
  for (int w = 0; w < BH_NW; ++w) {
    const int s = sh.scan[w];
    if (w < warp) wpre += s;
    tot += s;
  }
  __syncthreads();
  *total = tot;
  return wpre + x - v;
}

// ---------------------------------------------------------------- build
template <int NT>
__device__ void bh_build_tree(const BHKParams &p, BHShared &sh, unsigned &bar_target,
                              int *unit_dummy) {
  const int G = gridDim.x, c = blockIdx.x, n = p.n;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int lo, hi;
  bh_chunk(n, lo, hi);

  // B0: bounding box
  {
    float xmn = INFINITY, xmx = -INFINITY, ymn = INFINITY, ymx = -INFINITY;
    for (int v = lo + threadIdx.x; v < hi; v += NT) {
      const float2 q = __ldcg(p.xy + v);
      xmn = fminf(xmn, q.x);
      xmx = fmaxf(xmx, q.x);
      ymn = fminf(ymn, q.y);
      ymx = fmaxf(ymx, q.y);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      xmn = fminf(xmn, __shfl_xor_sync(0xffffffffu, xmn, o));
      xmx = fmaxf(xmx, __shfl_xor_sync(0xffffffffu, xmx, o));
      ymn = fminf(ymn, __shfl_xor_sync(0xffffffffu, ymn, o));
      ymx = fmaxf(ymx, __shfl_xor_sync(0xffffffffu, ymx, o));
    }
    if (lane == 0) sh.red4[warp] = make_float4(xmn, xmx, ymn, ymx);
    __syncthreads();
    if (threadIdx.x == 0) {
      float4 r = sh.red4[0];
      for (int w = 1; w < BH_NW; ++w) {
        r.x = fminf(r.x, sh.red4[w].x);
        r.y = fmaxf(r.y, sh.red4[w].y);
        r.z = fminf(r.z, sh.red4[w].z);
        r.w = fmaxf(r.w, sh.red4[w].w);
      }
      p.bbox[c] = r;
    }
  }
  bl_grid_sync(p.bar, bar_target, unit_dummy);
  if (threadIdx.x == 0) {
    float4 r = __ldcg(p.bbox);
    for (int cc = 1; cc < G; ++cc) {
      const float4 q = __ldcg(p.bbox + cc);
      r.x = fminf(r.x, q.x);
      r.y = fmaxf(r.y, q.y);
      r.z = fminf(r.z, q.z);
      r.w = fmaxf(r.w, q.w);
    }
    const float ex = __fsub_rn(r.y, r.x), ey = __fsub_rn(r.w, r.z);
    const float D = ex > ey ? ex : ey;  // Alg. S3 line 7
    sh.D = D;
    sh.xmin = r.x;
    sh.ymin = r.z;
    sh.degenerate = !(D > 0.0f);
    sh.scale = sh.degenerate ? 0.0f : __fdiv_rn(65536.0f, D);
  }
  __syncthreads();

  // B1: codes of the owned chunk (input order = vertex id order)
  for (int v = lo + threadIdx.x; v < hi; v += NT) {
    const float2 q = __ldcg(p.xy + v);
    p.keyA[v] = bh_interleave(bh_quant(q.x, sh.xmin, sh.scale, sh.degenerate),
                              bh_quant(q.y, sh.ymin, sh.scale, sh.degenerate));
    p.valA[v] = v;
  }
  __syncthreads();

  // B2: stable LSD radix sort, 4 passes of 8 bits
  unsigned *kin = p.keyA, *kout = p.keyB;
  int *vin = p.valA, *vout = p.valB;
  for (int pass = 0; pass < 4; ++pass) {
    const int sft = 8 * pass;
    for (int d = threadIdx.x; d < 256; d += NT) sh.hist[d] = 0;
    __syncthreads();
    for (int v = lo + threadIdx.x; v < hi; v += NT) atomicAdd(&sh.hist[(kin[v] >> sft) & 255u], 1u);
    __syncthreads();
    for (int d = threadIdx.x; d < 256; d += NT) p.hist[d * G + c] = sh.hist[d];
    bl_grid_sync(p.bar, bar_target, unit_dummy);
    // global base of each digit for this CTA: digits below + CTAs below
    {
      unsigned tot = 0, pre = 0;
      const int d = threadIdx.x;
      if (d < 256) {
        for (int cc = 0; cc < G; ++cc) {
          const unsigned h = __ldcg(p.hist + d * G + cc);
          if (cc < c) pre += h;
          tot += h;
        }
      }
      int total;
      const int ex = bh_block_scan(d < 256 ? (int)tot : 0, sh, &total);
      if (d < 256) sh.base[d] = (unsigned)ex + pre;
    }
    __syncthreads();
    // stable scatter in tiles of NT consecutive elements
    for (int t0 = lo; t0 < hi; t0 += NT) {
      const int v = t0 + threadIdx.x;
      const bool act = v < hi;
      unsigned key = 0, dig = 0;
      int val = 0;
      if (act) {
        key = kin[v];
        val = vin[v];
        dig = (key >> sft) & 255u;
      }
      for (int d = threadIdx.x; d < BH_NW * 256; d += NT) (&sh.wcnt[0][0])[d] = 0;
      __syncthreads();
      const unsigned amask = __ballot_sync(0xffffffffu, act);
      unsigned peers = 0, rank = 0;
      if (act) {
        peers = __match_any_sync(amask, dig);
        rank = __popc(peers & ((1u << lane) - 1u));
        if (rank == 0) sh.wcnt[warp][dig] = __popc(peers);
      }
      __syncthreads();
      // per digit: exclusive prefix over warps, then advance the base
      if (threadIdx.x < 256) {
        const int d = threadIdx.x;
        unsigned acc = 0;
        for (int w = 0; w < BH_NW; ++w) {
          const unsigned x = sh.wcnt[w][d];
          sh.wcnt[w][d] = acc;
          acc += x;
        }
        sh.hist[d] = acc;  // tile count of digit d
      }
      __syncthreads();
      if (act) {
        const unsigned pos = sh.base[dig] + sh.wcnt[warp][dig] + rank;
        kout[pos] = key;
        vout[pos] = val;
      }
      __syncthreads();
      if (threadIdx.x < 256) sh.base[threadIdx.x] += sh.hist[threadIdx.x];
      __syncthreads();
    }
    bl_grid_sync(p.bar, bar_target, unit_dummy);
    unsigned *tk = kin;
    kin = kout;
    kout = tk;
    int *tv = vin;
    vin = vout;
    vout = tv;
  }
  // sorted (code, id) are in keyA / valA (4 passes)

  // B3: node counts per sorted position, snapshot in sorted order
  int my = 0;
  for (int i = lo + threadIdx.x; i < hi; i += NT) {
    const unsigned ki = __ldcg(p.keyA + i);
    const int di = i == 0 ? -1 : bh_delta(__ldcg(p.keyA + i - 1), ki);
    const int dn = i == n - 1 ? -1 : bh_delta(ki, __ldcg(p.keyA + i + 1));
    const int L0 = di + 1;
    int cnt = 0;
    if (L0 <= 16) cnt = dn >= L0 ? min(dn + 1, 16) - L0 + 1 : 1;
    p.cnt[i] = cnt;
    p.snap[i] = __ldcg(p.xy + __ldcg(p.valA + i));
    my += cnt;
  }
  {
    int total;
    bh_block_scan(my, sh, &total);
    if (threadIdx.x == 0) p.blk[c] = total;
  }
  bl_grid_sync(p.bar, bar_target, unit_dummy);
  // exclusive offsets: CTAs below, then this CTA's positions in order.  Each
  // thread owns a contiguous run of the chunk so the scan is over runs.
  {
    int before = 0, all = 0;
    for (int cc = 0; cc < G; ++cc) {
      const int s = __ldcg(p.blk + cc);
      if (cc < c) before += s;
      all += s;
    }
    const int len = hi - lo;
    const int per = (len + NT - 1) / NT;
    const int a = lo + threadIdx.x * per, e = min(hi, a + per);
    int run = 0;
    for (int i = a; i < e; ++i) run += __ldcg(p.cnt + i);
    int total;
    int pre = bh_block_scan(run, sh, &total) + before;
    for (int i = a; i < e; ++i) {
      p.off[i] = pre;
      pre += __ldcg(p.cnt + i);
    }
    if (c == 0 && threadIdx.x == 0) {
      p.off[n] = all;
      *p.nnodes = all;
    }
  }
  bl_grid_sync(p.bar, bar_target, unit_dummy);

  // B4: node records (level, start, count, skip) and leaf sums
  const int Nn = __ldcg(p.nnodes);
  for (int i = lo + threadIdx.x; i < hi; i += NT) {
    const int cnt = __ldcg(p.cnt + i);
    if (cnt == 0) continue;
    const unsigned ki = __ldcg(p.keyA + i);
    const int di = i == 0 ? -1 : bh_delta(__ldcg(p.keyA + i - 1), ki);
    const int L0 = di + 1;
    const int k0 = __ldcg(p.off + i);
    int e = i + 1;  // segment ends, computed from the deepest level up
    for (int L = L0 + cnt - 1; L >= L0; --L) {
      // end of the level-L segment starting at i: first j with another prefix
      const unsigned pk = bh_prefix(ki, L);
      if (e < n && bh_prefix(__ldcg(p.keyA + e), L) == pk) {
        int step = 1, a = e;  // keyA[a] has prefix pk
        int b = e + 1;
        while (b < n && bh_prefix(__ldcg(p.keyA + b), L) == pk) {
          a = b;
          step <<= 1;
          b = a + step;
        }
        if (b > n) b = n;
        // invariant: prefix(a) == pk, b == n or prefix(b) != pk
        while (b - a > 1) {
          const int m = (a + b) >> 1;
          if (bh_prefix(__ldcg(p.keyA + m), L) == pk) a = m;
          else b = m;
        }
        e = b;
      }
      const int count = e - i;
      const int k = k0 + (L - L0);
      const int skip = e >= n ? Nn : __ldcg(p.off + e);
      const bool leaf = count == 1 || L == 16;
      p.nodeB[k] = make_int4(L | ((leaf ? 1 : 0) << 16), i, count, skip);
      if (leaf) {
        double sx = 0.0, sy = 0.0;
        for (int s = i; s < e; ++s) {
          const float2 q = __ldcg(p.snap + s);
          sx = sx + (double)q.x;
          sy = sy + (double)q.y;
        }
        p.nsum[k] = make_double2(sx, sy);
        p.nodeA[k] = make_float4((float)(sx / count), (float)(sy / count), 0.f, (float)count);
        p.nodeC[k] = make_int4(-1, -1, -1, -1);
      }
    }
  }
  bl_grid_sync(p.bar, bar_target, unit_dummy);

  // B4': children lists of internal nodes (pre-order: first child k+1, then
  // follow the children's skip pointers up to the parent's skip)
  for (int k = c * NT + threadIdx.x; k < Nn; k += G * NT) {
    int4 B = __ldcg(p.nodeB + k);
    if (B.x & (1 << 16)) continue;
    int ch[4] = {-1, -1, -1, -1};
    int m = 0, t = k + 1;
    while (t < B.w && m < 4) {
      ch[m++] = t;
      t = __ldcg(p.nodeB + t).w;
    }
    p.nodeC[k] = make_int4(ch[0], ch[1], ch[2], ch[3]);
    B.x |= m << 8;
    p.nodeB[k] = B;
  }
  bl_grid_sync(p.bar, bar_target, unit_dummy);

  // B5: centroids bottom-up (Alg. S1 line 11), fp64 sums in digit order
  const float D = sh.D;
  for (int L = 15; L >= 0; --L) {
    for (int k = c * NT + threadIdx.x; k < Nn; k += G * NT) {
      const int4 B = __ldcg(p.nodeB + k);
      if ((B.x & 0xff) != L || (B.x & (1 << 16))) continue;
      const int4 C4 = __ldcg(p.nodeC + k);
      const int chs[4] = {C4.x, C4.y, C4.z, C4.w};
      double sx = 0.0, sy = 0.0;
      for (int q = 0; q < 4; ++q) {
        if (chs[q] < 0) break;
        const double2 s = __ldcg(p.nsum + chs[q]);
        sx = sx + s.x;
        sy = sy + s.y;
      }
      p.nsum[k] = make_double2(sx, sy);
      const float DL = ldexpf(D, -L);
      p.nodeA[k] = make_float4((float)(sx / (double)B.z), (float)(sy / (double)B.z),
                               __fmul_rn(DL, DL), (float)B.z);
    }
    bl_grid_sync(p.bar, bar_target, unit_dummy);
  }
}

// ---------------------------------------------------------------- forces
// Exact repulsive terms of a leaf's vertices against vertex v at (qx, qy),
// live coordinates (reading B5/B8/B9).
__device__ __forceinline__ void bh_leaf_terms(const BHKParams &p, const int4 &B, int v, float qx,
                                              float qy, float &fx, float &fy) {
  for (int s = B.y; s < B.y + B.z; ++s) {
    const int j = __ldcg(p.valA + s);
    if (j == v) continue;
    const float2 cj = __ldcg(p.xy + j);
    const float dx = cj.x - qx, dy = cj.y - qy;
    const float d2 = fmaf(dx, dx, dy * dy);
    if (d2 > 0.f) {
      const float r = p.ck2 / d2;
      fx = fmaf(-r, dx, fx);
      fy = fmaf(-r, dy, fy);
    }
  }
}

// MAC of Alg. S2 in fp32 with separately rounded operations (reading B7).
// Returns true and accumulates the count-weighted centroid term if accepted.
__device__ __forceinline__ bool bh_mac(const BHKParams &p, const float4 &A, float qx, float qy,
                                       float &fx, float &fy) {
  const float dx = __fsub_rn(A.x, qx), dy = __fsub_rn(A.y, qy);
  const float d2 = __fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy));
  if (!(__fmul_rn(p.theta2, d2) > A.z)) return false;
  const float r = A.w * p.ck2 / d2;
  fx = fmaf(-r, dx, fx);
  fy = fmaf(-r, dy, fy);
  return true;
}

// One lane walks the subtree below node k (k's own MAC already failed) with
// the skip pointers: no stack.
__device__ __forceinline__ void bh_walk_subtree(const BHKParams &p, int k, int v, float qx, float qy,
                                                float &fx, float &fy, unsigned long long &vis) {
  const int end = __ldcg(p.nodeB + k).w;
  int t = k + 1;
  while (t < end) {
    const int4 B = __ldcg(p.nodeB + t);
    ++vis;
    if (B.x & (1 << 16)) {
      bh_leaf_terms(p, B, v, qx, qy, fx, fy);
      t = B.w;
    } else if (bh_mac(p, __ldcg(p.nodeA + t), qx, qy, fx, fy)) {
      t = B.w;
    } else {
      t = t + 1;
    }
  }
}

// Force of vertex v (one warp): CSR attraction + Barnes-Hut repulsion.
// Returns the warp-summed force on every lane.
__device__ __forceinline__ float2 bh_force_warp(const BHKParams &p, BHShared &sh, int v,
                                                unsigned long long &vis) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float2 cv = __ldcg(p.xy + v);
  float fx = 0.f, fy = 0.f;
  // attraction f_a = d^2/K along the unit vector (Alg. S3 lines 15-17)
  const int k0 = __ldg(p.rowptr + v), k1 = __ldg(p.rowptr + v + 1);
  for (int k = k0 + lane; k < k1; k += 32) {
    const float2 cj = __ldcg(p.xy + __ldg(p.colidx + k));
    const float dx = cj.x - cv.x, dy = cj.y - cv.y;
    const float d2 = fmaf(dx, dx, dy * dy);
    if (d2 > 0.f) {
      const float d = sqrtf(d2);
      fx = fmaf(d * p.invK, dx, fx);
      fy = fmaf(d * p.invK, dy, fy);
    }
  }
  // repulsion: frontier traversal from the root (Alg. S2)
  int *cur = sh.frontier[warp][0], *nxt = sh.frontier[warp][1];
  int ncur = 1;
  if (lane == 0) cur[0] = 0;
  __syncwarp();
  while (ncur > 0) {
    int nnext = 0;
    for (int base = 0; base < ncur; base += 32) {
      const int idx = base + lane;
      const int k = idx < ncur ? cur[idx] : -1;
      int m = 0;
      int4 kids = make_int4(-1, -1, -1, -1);
      if (k >= 0) {
        const int4 B = __ldcg(p.nodeB + k);
        ++vis;
        if (B.x & (1 << 16)) {
          bh_leaf_terms(p, B, v, cv.x, cv.y, fx, fy);
        } else if (!bh_mac(p, __ldcg(p.nodeA + k), cv.x, cv.y, fx, fy)) {
          m = (B.x >> 8) & 0xff;
          kids = __ldcg(p.nodeC + k);
        }
      }
      int incl = m;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const int pos = nnext + incl - m;
      const bool fits = pos + m <= BH_FCAP;
      if (m > 0) {
        if (fits) {
          const int ks[4] = {kids.x, kids.y, kids.z, kids.w};
          for (int q = 0; q < m; ++q) nxt[pos + q] = ks[q];
        } else {
          bh_walk_subtree(p, k, v, cv.x, cv.y, fx, fy, vis);  // frontier full
        }
      }
      // entries written: the fitting lanes form a prefix of the warp
      nnext = max(nnext, (int)__reduce_max_sync(0xffffffffu, (unsigned)(fits ? pos + m : 0)));
    }
    __syncwarp();
    int *t = cur;
    cur = nxt;
    nxt = t;
    ncur = nnext;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    fx += __shfl_xor_sync(0xffffffffu, fx, o);
    fy += __shfl_xor_sync(0xffffffffu, fy, o);
  }
  return make_float2(fx, fy);
}

// Alg. S3's iterations: tree per iteration, then the dependent minibatches.
template <int NT>
__device__ void bh_run_batches(const BHKParams &p, BHShared &sh, unsigned &bar_target,
                               int *unit_dummy_ptr, unsigned long long &vis) {
  const int G = gridDim.x, c = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gw = c * BH_NW + warp, GW = G * BH_NW;
  double step = p.step0, e_prev = 0.0, e_acc = 0.0;
  int batches = 0, done = 0;
  bool stop = false;
  for (int it = 0; it < p.iters && !stop; ++it) {
    bh_build_tree<NT>(p, sh, bar_target, unit_dummy_ptr);  // Alg. S3 lines 5-8
    e_acc = 0.0;
    for (int t = 0; t < p.nb; ++t) {
      const int lo = t * p.b, bt = min(p.b, p.n - lo);
      // F: forces of the batch, coordinates frozen (lines 13-20)
      for (int i = gw; i < bt; i += GW) {
        const float2 f = bh_force_warp(p, sh, lo + i, vis);
        if (lane == 0) p.fb[i] = f;
      }
      bl_grid_sync(p.bar, bar_target, unit_dummy_ptr);
      // U: owner update (lines 21-24); CTA c owns batch entries c, c+G, ...
      for (int i = c + G * threadIdx.x; i < bt; i += G * NT) {
        const float2 f = __ldcg(p.fb + i);
        const double q = (double)f.x * f.x + (double)f.y * f.y;
        if (q > 0.0) {
          const double s = step / sqrt(q);
          float2 cv = __ldcg(p.xy + lo + i);
          cv.x = (float)((double)cv.x + s * f.x);
          cv.y = (float)((double)cv.y + s * f.y);
          p.xy[lo + i] = cv;
        }
        e_acc += q;
      }
      ++batches;
      const bool last = t == p.nb - 1;
      const bool mb = p.max_batches > 0 && batches >= p.max_batches;
      if (last || mb) {
        double e = e_acc;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
        if (lane == 0) sh.e_warp[warp] = e;
        __syncthreads();
        if (threadIdx.x == 0) {
          double s = 0.0;
          for (int w = 0; w < BH_NW; ++w) s += sh.e_warp[w];
          p.e_cta[c] = s;
        }
      }
      bl_grid_sync(p.bar, bar_target, unit_dummy_ptr);
      if (last || mb) {
        // every CTA sums the per-CTA energies in the same order, so the tol
        // decision is identical everywhere
        double E = 0.0;
        for (int cc = 0; cc < G; ++cc) E += __ldcg(p.e_cta + cc);
        if (c == 0 && threadIdx.x == 0) p.energy[it] = E;
        if (mb) {
          stop = true;
          break;
        }
        done = it + 1;
        if (p.tol > 0.0 && it > 0 && fabs(E - e_prev) < p.tol) {
          stop = true;
          break;
        }
        e_prev = E;
      }
    }
    step = step * p.cooling;
  }
  if (c == 0 && threadIdx.x == 0) *p.iters_done = done;
}

// ---------------------------------------------------------------- kernel
template <int NT>
__global__ void __launch_bounds__(NT, 1) bl_bh_kernel(BHKParams p) {
  extern __shared__ __align__(16) unsigned char bh_smem[];
  BHShared &sh = *reinterpret_cast<BHShared *>(bh_smem);
  __shared__ int unit_dummy;
  const int G = gridDim.x, c = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned bar_target = 0;
  unsigned long long vis = 0;
  const int gw = c * BH_NW + warp, GW = G * BH_NW;

  if (p.forces_mode) {
    bh_build_tree<NT>(p, sh, bar_target, &unit_dummy);
    for (int t = gw; t < p.count; t += GW) {
      const float2 f = bh_force_warp(p, sh, p.first + t, vis);
      if (lane == 0) p.f_out[t] = f;
    }
  } else {
    bh_run_batches<NT>(p, sh, bar_target, &unit_dummy, vis);
  }

  // visits: per-CTA totals (deterministic sum later on the host)
  unsigned long long vsum = vis;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) vsum += __shfl_xor_sync(0xffffffffu, vsum, o);
  if (lane == 0) atomicAdd(p.visits + c, vsum);
}
