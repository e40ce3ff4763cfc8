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
#define BH_TOP_LEVEL 4  // tree levels 0..4 are copied to shared memory per CTA
#define BH_TOP_MAX 352  // >= 1 + 4 + 16 + 64 + 256
#ifndef BH_LCAP
#define BH_LCAP 32      // leaf vertices recorded per query (a multiple of 32: BH_LPL per lane)
#endif
#define BH_LPL (BH_LCAP / 32)

struct BHKParams {
  int n, b, nb, iters, max_batches;
  float ck2, invK, theta2;
  int amode, rmode;       // (a, r)-energy model, as BLKParams (reading C15)
  float a_half, r_half;
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
  double *e_cta;      // [G]
  double *energy;     // [iters]
  int *iters_done;
  unsigned *bar;
  float2 *f_out;
  unsigned long long *visits;  // [G] node visits per CTA (for the roofline)
  float2 *pend;                // [2][b] new coordinates of the last two batches
  // per-iteration precomputation (layout mode): the MAC decisions and the
  // accepted cells' terms depend only on the iteration-start tree and the
  // query's own position, which does not move before its batch (reading B5),
  // so each vertex's cell sum and its list of leaf vertices are computed once
  // per iteration for all n vertices at once; a batch then adds the leaf
  // terms at the live coordinates.  nleaf < 0: list overflow, the batch
  // traverses the tree for that vertex as before.
  float2 *cellf;               // [n]
  int *nleaf;                  // [n]
  int *leafv;                  // [n][BH_LCAP]
  int precompute;              // 1: use the above
  int pre2;                    // 1: batch inputs prefetched across the grid barrier (bh_prefetch)
  // attraction of high-degree ("split") vertices, edge-parallel: rows cut in
  // items of <= BL_ECH entries (the context's item lists), one partial per
  // item, published with a release flag stamped with the batch number
  const int *item_ptr, *item_v, *item_k0;
  const int *split_ptr;        // [n + 1] items of split vertices below v
  const int4 *sitems;          // those items in vertex order: {item, vertex, k0, k1}
  float2 *attr;                // [n_items]
  unsigned *aflag;             // [n_items]
  uint4 *attr_ll;              // [n_items] layout mode with pre2: {fx bits, stamp, fy bits,
                               // stamp} -- two 8-byte words that each carry their own flag
                               // (no release fence between value and flag: one L2 trip less
                               // on the split vertex's critical path)
  unsigned long long *prof;    // optional phase profile (BL_PROFILE=1)
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
  // the top of the tree (levels <= BH_TOP_LEVEL) in BFS order, per CTA: every
  // query starts there, so its records come from shared memory instead of
  // one L2 round trip per level after each grid barrier (which invalidates
  // L1).  Node references: r >= 0 global pre-order index, r < 0 top slot -r-1
  float4 topA[BH_TOP_MAX];
  int4 topB[BH_TOP_MAX];
  int4 topK[BH_TOP_MAX];  // child refs (internal) or (vertex id, -, -, -) (leaf)
  int topG[BH_TOP_MAX];   // global index
  int ntop;
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
                              int *unit_dummy, BLProf &pf) {
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
  if (threadIdx.x < 32) {  // one warp, lanes strided over the CTAs (min/max: exact)
    float4 r = make_float4(INFINITY, -INFINITY, INFINITY, -INFINITY);
    for (int cc = lane; cc < G; cc += 32) {
      const float4 q = __ldcg(p.bbox + cc);
      r.x = fminf(r.x, q.x);
      r.y = fmaxf(r.y, q.y);
      r.z = fminf(r.z, q.z);
      r.w = fmaxf(r.w, q.w);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      r.x = fminf(r.x, __shfl_xor_sync(0xffffffffu, r.x, o));
      r.y = fmaxf(r.y, __shfl_xor_sync(0xffffffffu, r.y, o));
      r.z = fminf(r.z, __shfl_xor_sync(0xffffffffu, r.z, o));
      r.w = fmaxf(r.w, __shfl_xor_sync(0xffffffffu, r.w, o));
    }
    if (lane == 0) {
      const float ex = __fsub_rn(r.y, r.x), ey = __fsub_rn(r.w, r.z);
      const float D = ex > ey ? ex : ey;  // Alg. S3 line 7
      sh.D = D;
      sh.xmin = r.x;
      sh.ymin = r.z;
      sh.degenerate = !(D > 0.0f);
      sh.scale = sh.degenerate ? 0.0f : __fdiv_rn(65536.0f, D);
    }
  }
  __syncthreads();
  pf.mark(0);

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
    // global base of each digit for this CTA: digits below + CTAs below.
    // Warp w handles digits 16w..16w+15, lanes strided over the CTAs (all
    // loads in flight at once); integer sums, so the order is immaterial.
    {
      for (int j = 0; j < 256 / BH_NW; ++j) {
        const int d = warp * (256 / BH_NW) + j;
        unsigned tot = 0, pre = 0;
        for (int cc = lane; cc < G; cc += 32) {
          const unsigned h = __ldcg(p.hist + d * G + cc);
          tot += h;
          if (cc < c) pre += h;
        }
        tot = __reduce_add_sync(0xffffffffu, tot);
        pre = __reduce_add_sync(0xffffffffu, pre);
        if (lane == 0) {
          sh.hist[d] = tot;
          sh.base[d] = pre;
        }
      }
      __syncthreads();
      int total;
      const int d = threadIdx.x;
      const int ex = bh_block_scan(d < 256 ? (int)sh.hist[d] : 0, sh, &total);
      if (d < 256) sh.base[d] += (unsigned)ex;
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
  pf.mark(1);

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
    unsigned bf = 0, al = 0;
    for (int cc = lane; cc < G; cc += 32) {
      const unsigned s = (unsigned)__ldcg(p.blk + cc);
      if (cc < c) bf += s;
      al += s;
    }
    const int before = (int)__reduce_add_sync(0xffffffffu, bf);
    const int all = (int)__reduce_add_sync(0xffffffffu, al);
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
        p.nodeC[k] = make_int4(-1, -1, -1, count == 1 ? __ldcg(p.valA + i) : -1);
      }
    }
  }
  bl_grid_sync(p.bar, bar_target, unit_dummy);

  // B4': children lists of internal nodes (pre-order: child 0 is k+1, the
  // next ones follow the children's skip pointers up to the parent's skip);
  // stored as (c1, c2, c3, -1)
  for (int k = c * NT + threadIdx.x; k < Nn; k += G * NT) {
    int4 B = __ldcg(p.nodeB + k);
    if (B.x & (1 << 16)) continue;
    int ch[4] = {-1, -1, -1, -1};
    int m = 0, t = k + 1;
    while (t < B.w && m < 4) {
      ch[m++] = t;
      t = __ldcg(p.nodeB + t).w;
    }
    p.nodeC[k] = make_int4(ch[1], ch[2], ch[3], -1);
    B.x |= m << 8;
    p.nodeB[k] = B;
  }
  bl_grid_sync(p.bar, bar_target, unit_dummy);

  pf.mark(2);
  // B5: centroids bottom-up (Alg. S1 line 11), fp64 sums in digit order
  const float D = sh.D;
  // each thread owns the nodes k = tid + j G NT; the levels of its first
  // BH_CPT nodes are read ONCE (the level loop used to re-read every node's
  // record at each of the 16 levels: 16 x Nn x 16 B of L2 traffic, 113 us at
  // C5), nodes beyond that window take the scanning path
  constexpr int BH_CPT = 8;
  const int stride = G * NT, tid0 = c * NT + threadIdx.x;
  int lv[BH_CPT];
#pragma unroll
  for (int j = 0; j < BH_CPT; ++j) {
    const int k = tid0 + j * stride;
    lv[j] = -1;
    if (k < Nn) {
      const int bx = __ldcg(&p.nodeB[k].x);
      if (!(bx & (1 << 16))) lv[j] = bx & 0xff;
    }
  }
  auto centroid = [&](int k, const int4 &B, int L) {
    const int4 C4 = __ldcg(p.nodeC + k);
    const int chs[4] = {k + 1, C4.x, C4.y, C4.z};
    const int m = (B.x >> 8) & 0xff;
    double sx = 0.0, sy = 0.0;
    for (int q = 0; q < m; ++q) {
      const double2 s = __ldcg(p.nsum + chs[q]);
      sx = sx + s.x;
      sy = sy + s.y;
    }
    p.nsum[k] = make_double2(sx, sy);
    const float DL = ldexpf(D, -L);
    p.nodeA[k] = make_float4((float)(sx / (double)B.z), (float)(sy / (double)B.z),
                             __fmul_rn(DL, DL), (float)B.z);
  };
  for (int L = 15; L >= 0; --L) {
#pragma unroll
    for (int j = 0; j < BH_CPT; ++j)
      if (lv[j] == L) {
        const int k = tid0 + j * stride;
        centroid(k, __ldcg(p.nodeB + k), L);
      }
    for (int k = tid0 + BH_CPT * stride; k < Nn; k += stride) {
      const int4 B = __ldcg(p.nodeB + k);
      if ((B.x & 0xff) != L || (B.x & (1 << 16))) continue;
      centroid(k, B, L);
    }
    bl_grid_sync(p.bar, bar_target, unit_dummy);
  }
  // B6: the top of the tree into shared memory (warp 0 of each CTA, BFS)
  if (warp == 0) {
    int n_top = 1, head = 0;
    if (lane == 0) sh.topG[0] = 0;
    __syncwarp();
    while (head < n_top) {
      const int i = head + lane;
      int m = 0;
      int4 B = make_int4(0, 0, 0, 0), C = make_int4(-1, -1, -1, -1);
      int g = 0;
      if (i < n_top) {
        g = sh.topG[i];
        B = __ldcg(p.nodeB + g);
        C = __ldcg(p.nodeC + g);
        sh.topA[i] = __ldcg(p.nodeA + g);
        sh.topB[i] = B;
        const bool leaf = B.x & (1 << 16);
        if (!leaf && (B.x & 0xff) < BH_TOP_LEVEL) m = (B.x >> 8) & 0xff;
      }
      int incl = m;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const int pos = n_top + incl - m;
      if (i < n_top) {
        const int kids[4] = {g + 1, C.x, C.y, C.z};
        int4 K;
        if (B.x & (1 << 16)) {
          K = make_int4(C.w, -1, -1, -1);
        } else if (m > 0) {  // children are top slots pos .. pos+m-1
          for (int q = 0; q < m; ++q) sh.topG[pos + q] = kids[q];
          K = make_int4(-(pos + 1), m > 1 ? -(pos + 2) : -1, m > 2 ? -(pos + 3) : -1,
                        m > 3 ? -(pos + 4) : -1);
        } else {  // children stay global
          K = make_int4(kids[0], kids[1], kids[2], kids[3]);
        }
        sh.topK[i] = K;
      }
      const int added = __shfl_sync(0xffffffffu, incl, 31);
      head = min(n_top, head + 32);
      n_top += added;
      __syncwarp();
    }
    if (lane == 0) sh.ntop = n_top;
  }
  __syncthreads();
  pf.mark(3);
}

// ---------------------------------------------------------------- forces
// Tree records are read with plain (L1-cacheable) loads: they are written in
// the build phase before a grid barrier whose acquire orders them, and the
// top of the tree is shared by every query of the SM.
struct BHNode {
  float4 A;  // centroid x, y, D_L^2, count
  int4 B;    // level | nchild << 8 | leaf << 16, start, count, skip
  int4 C;    // children 1..3 (child 0 is k+1), vertex id of a single leaf
};
__device__ __forceinline__ BHNode bh_load(const BHKParams &p, int k) {
  BHNode nd;
  nd.A = p.nodeA[k];
  nd.B = p.nodeB[k];
  nd.C = p.nodeC[k];
  return nd;
}
// A node by reference (shared top slot or global index): its record, its
// child references, its global index.
struct BHRefNode {
  BHNode nd;
  int kids[4];
  int g;
};
__device__ __forceinline__ BHRefNode bh_load_ref(const BHKParams &p, const BHShared &sh, int r) {
  BHRefNode x;
  if (r < 0) {
    const int i = -r - 1;
    x.nd.A = sh.topA[i];
    x.nd.B = sh.topB[i];
    const int4 K = sh.topK[i];
    x.nd.C = make_int4(-1, -1, -1, K.x);  // vertex id of a leaf in .w
    x.kids[0] = K.x;
    x.kids[1] = K.y;
    x.kids[2] = K.z;
    x.kids[3] = K.w;
    x.g = sh.topG[i];
  } else {
    x.nd = bh_load(p, r);
    x.kids[0] = r + 1;
    x.kids[1] = x.nd.C.x;
    x.kids[2] = x.nd.C.y;
    x.kids[3] = x.nd.C.z;
    x.g = r;
  }
  return x;
}

// Live coordinate of vertex j (reading B5): batch `pl` vertices [plo, phi)
// hold their new coordinates in pend (committed to xy one batch later).
__device__ __forceinline__ float2 bh_live(const BHKParams &p, int j, int plo, int phi,
                                          const float2 *pend) {
  return (j >= plo && j < phi) ? __ldcg(pend + (j - plo)) : __ldcg(p.xy + j);
}

// Repulsion weight of Δ at squared distance d2: C K^2 d^(r-1) (reading C15)
__device__ __forceinline__ float bh_rep_weight(const BHKParams &p, float d2) {
  return p.rmode == 0 ? p.ck2 / d2 : p.ck2 * bl_pow_d2(d2, p.r_half);
}

// Exact repulsive terms of a leaf's vertices against vertex v at (qx, qy)
// (readings B5/B8/B9).
__device__ __forceinline__ void bh_leaf_terms(const BHKParams &p, const BHNode &nd, int v, float qx,
                                              float qy, int plo, int phi, const float2 *pend,
                                              float &fx, float &fy) {
  const int cnt = nd.B.z;
  for (int s = 0; s < cnt; ++s) {
    const int j = cnt == 1 ? nd.C.w : __ldcg(p.valA + nd.B.y + s);
    if (j == v) continue;
    const float2 cj = bh_live(p, j, plo, phi, pend);
    const float dx = cj.x - qx, dy = cj.y - qy;
    const float d2 = fmaf(dx, dx, dy * dy);
    if (d2 > 0.f) {
      const float r = bh_rep_weight(p, d2);
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
  const float r = A.w * bh_rep_weight(p, d2);
  fx = fmaf(-r, dx, fx);
  fy = fmaf(-r, dy, fy);
  return true;
}

// One lane walks the subtree below node k (k's own MAC already failed) with
// the skip pointers: no stack.
__device__ __forceinline__ void bh_walk_subtree(const BHKParams &p, int k, int end, int v, float qx,
                                                float qy, int plo, int phi, const float2 *pend,
                                                float &fx, float &fy, unsigned long long &vis) {
  int t = k + 1;
  while (t < end) {
    const BHNode nd = bh_load(p, t);
    ++vis;
    if (nd.B.x & (1 << 16)) {
      bh_leaf_terms(p, nd, v, qx, qy, plo, phi, pend, fx, fy);
      t = nd.B.w;
    } else if (bh_mac(p, nd.A, qx, qy, fx, fy)) {
      t = nd.B.w;
    } else {
      t = t + 1;
    }
  }
}

// Attraction sum over CSR entries [k0, k1) of vertex v at cv (one warp,
// lanes strided, fixed butterfly): f_a = d^2/K along the unit vector
// (Alg. S3 lines 15-17), live neighbour coordinates.
// one CSR entry's attraction f_a(d)/d = d^(a-1)/K along Δ = cj - cv
__device__ __forceinline__ void bh_attr_term(const BHKParams &p, float2 cj, float2 cv, float &fx,
                                             float &fy) {
  const float dx = cj.x - cv.x, dy = cj.y - cv.y;
  const float d2 = fmaf(dx, dx, dy * dy);
  if (d2 > 0.f) {
    float at;
    switch (p.amode) {
      case 0: at = sqrtf(d2); break;
      case 1: at = 1.f; break;
      case 2: at = rsqrtf(d2); break;
      case 3: at = d2; break;
      default: at = bl_pow_d2(d2, p.a_half);
    }
    fx = fmaf(at * p.invK, dx, fx);
    fy = fmaf(at * p.invK, dy, fy);
  }
}
__device__ __forceinline__ void bh_attr_lane(const BHKParams &p, int k0, int k1, float2 cv,
                                             int plo, int phi, const float2 *pend, float &fx,
                                             float &fy) {
  const int lane = threadIdx.x & 31;
  for (int k = k0 + lane; k < k1; k += 32)
    bh_attr_term(p, bh_live(p, __ldg(p.colidx + k), plo, phi, pend), cv, fx, fy);
}
__device__ __forceinline__ float2 bh_attr_range(const BHKParams &p, int k0, int k1, float2 cv,
                                                int plo, int phi, const float2 *pend) {
  float fx = 0.f, fy = 0.f;
  bh_attr_lane(p, k0, k1, cv, plo, phi, pend, fx, fy);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    fx += __shfl_xor_sync(0xffffffffu, fx, o);
    fy += __shfl_xor_sync(0xffffffffu, fy, o);
  }
  return make_float2(fx, fy);
}

// Items of the split vertices in [vlo, vhi): warp gw of GW computes items
// gw, gw + GW, ... and publishes each partial with a release flag.
__device__ __forceinline__ void bh_attr_items(const BHKParams &p, int vlo, int vhi, int gw, int GW,
                                              unsigned stamp, int plo, int phi,
                                              const float2 *pend) {
  const int lane = threadIdx.x & 31;
  const int ib = __ldg(p.item_ptr + vlo), ie = __ldg(p.item_ptr + vhi);
  for (int it = ib + gw; it < ie; it += GW) {
    const int v = __ldg(p.item_v + it);
    if (__ldg(p.item_ptr + v + 1) - __ldg(p.item_ptr + v) <= 1) continue;  // inline vertex
    const int k0 = __ldg(p.item_k0 + it);
    const int k1 = min(k0 + BL_ECH, __ldg(p.rowptr + v + 1));
    const float2 f = bh_attr_range(p, k0, k1, __ldcg(p.xy + v), plo, phi, pend);
    if (lane == 0) {
      p.attr[it] = f;
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p.aflag + it), "r"(stamp) : "memory");
    }
  }
}

// Sum of the published item partials of split vertex v (waits for them).
__device__ __forceinline__ uint2 bh_ld_relaxed_v2(const void *q) {
  uint2 r;
  asm volatile("ld.relaxed.gpu.global.v2.u32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(q) : "memory");
  return r;
}
__device__ __forceinline__ void bh_st_relaxed_v2(void *q, unsigned a, unsigned b) {
  asm volatile("st.relaxed.gpu.global.v2.u32 [%0], {%1, %2};" ::"l"(q), "r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ float2 bh_attr_gather(const BHKParams &p, int v, unsigned stamp) {
  const int lane = threadIdx.x & 31;
  const int a0 = __ldg(p.item_ptr + v), a1 = __ldg(p.item_ptr + v + 1);
  float fx = 0.f, fy = 0.f;
  const bool ll = p.pre2 && !p.forces_mode;
  for (int a = a0 + lane; a < a1; a += 32) {
    float2 q;
    if (ll) {
      // each 8-byte word is written by one store: (value, stamp) arrive together
      uint2 w0, w1;
      for (;;) {
        w0 = bh_ld_relaxed_v2(&p.attr_ll[a].x);
        w1 = bh_ld_relaxed_v2(&p.attr_ll[a].z);
        if (w0.y == stamp && w1.y == stamp) break;
        __nanosleep(20);
      }
      q = make_float2(__uint_as_float(w0.x), __uint_as_float(w1.x));
    } else {
      while (bl_ld_acquire(p.aflag + a) != stamp) __nanosleep(20);
      q = __ldcg(p.attr + a);
    }
    fx += q.x;
    fy += q.y;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    fx += __shfl_xor_sync(0xffffffffu, fx, o);
    fy += __shfl_xor_sync(0xffffffffu, fy, o);
  }
  return make_float2(fx, fy);
}

// Force of vertex v (one warp): CSR attraction + Barnes-Hut repulsion.
// Returns the warp-summed force on every lane.
__device__ __forceinline__ float2 bh_force_warp(const BHKParams &p, BHShared &sh, int v, float2 cv,
                                                int plo, int phi, const float2 *pend,
                                                unsigned stamp, unsigned long long &vis) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float fx = 0.f, fy = 0.f;
  const bool split = __ldg(p.item_ptr + v + 1) - __ldg(p.item_ptr + v) > 1;
  // repulsion: frontier traversal from the root (Alg. S2)
  int *cur = sh.frontier[warp][0], *nxt = sh.frontier[warp][1];
  int ncur = 1;
  if (lane == 0) cur[0] = -1;  // the root, top slot 0
  __syncwarp();
  while (ncur > 0) {
    int nnext = 0;
    for (int base = 0; base < ncur; base += 32) {
      const int idx = base + lane;
      const bool has = idx < ncur;
      const int r = has ? cur[idx] : 0;
      int m = 0;
      BHRefNode x;
      if (has) {
        x = bh_load_ref(p, sh, r);
        ++vis;
        if (x.nd.B.x & (1 << 16)) {
          bh_leaf_terms(p, x.nd, v, cv.x, cv.y, plo, phi, pend, fx, fy);
        } else if (!bh_mac(p, x.nd.A, cv.x, cv.y, fx, fy)) {
          m = (x.nd.B.x >> 8) & 0xff;
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
          nxt[pos] = x.kids[0];
          if (m > 1) nxt[pos + 1] = x.kids[1];
          if (m > 2) nxt[pos + 2] = x.kids[2];
          if (m > 3) nxt[pos + 3] = x.kids[3];
        } else {
          bh_walk_subtree(p, x.g, x.nd.B.w, v, cv.x, cv.y, plo, phi, pend, fx, fy, vis);  // full
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
  // attraction f_a = d^2/K along the unit vector (Alg. S3 lines 15-17):
  // inline for short rows, else the published item partials
  const float2 fa = split ? bh_attr_gather(p, v, stamp)
                          : bh_attr_range(p, __ldg(p.rowptr + v), __ldg(p.rowptr + v + 1), cv,
                                          plo, phi, pend);
  return make_float2(fx + fa.x, fy + fa.y);
}

// Per-iteration precomputation for all n queries (one per thread, queries in
// Morton order so a warp's lanes walk similar paths): the full Alg. S2 walk
// with the skip pointers from the root; accepted cells accumulate into
// cellf[v] (fixed per iteration, reading B5), leaf vertices are recorded
// (at most BH_LCAP; more -> nleaf = -1 and the batch traverses for v).
// Node visits are counted here for every recorded query.
__device__ __forceinline__ void bh_precompute(const BHKParams &p, unsigned long long &vis) {
  const int G = gridDim.x, c = blockIdx.x;
  const int Nn = __ldcg(p.nnodes);
  for (int s = c * blockDim.x + threadIdx.x; s < p.n; s += G * blockDim.x) {
    const int v = __ldcg(p.valA + s);
    const float2 q = __ldcg(p.xy + v);
    float fx = 0.f, fy = 0.f;
    int nl = 0;
    unsigned long long vv = 0;
    int *lst = p.leafv + (size_t)v * BH_LCAP;
    int t = 0;
    while (t < Nn) {
      const BHNode nd = bh_load(p, t);
      ++vv;
      if (nd.B.x & (1 << 16)) {
        const int cnt = nd.B.z;
        for (int k = 0; k < cnt; ++k) {
          const int j = cnt == 1 ? nd.C.w : __ldcg(p.valA + nd.B.y + k);
          if (j == v) continue;
          if (nl < BH_LCAP) lst[nl] = j;
          ++nl;
        }
        t = nd.B.w;
      } else if (bh_mac(p, nd.A, q.x, q.y, fx, fy)) {
        t = nd.B.w;
      } else {
        t = t + 1;
      }
    }
    const bool ok = nl <= BH_LCAP;
    p.cellf[v] = make_float2(fx, fy);
    p.nleaf[v] = ok ? nl : -1;
    if (ok) vis += vv;
  }
}

// Force of vertex v (one warp) from its precomputed cell sum and leaf list:
// the leaf terms at the live coordinates (one leaf vertex per lane) +
// attraction.  Returns the warp-summed force on every lane.
__device__ __forceinline__ float2 bh_force_pre(const BHKParams &p, int v, float2 cv, int nl,
                                               int plo, int phi, const float2 *pend,
                                               unsigned stamp) {
  const int lane = threadIdx.x & 31;
  // first-level loads of both chains together: the leaf ids and the row bounds
  int j[BH_LPL];
#pragma unroll
  for (int u = 0; u < BH_LPL; ++u)
    j[u] = lane + 32 * u < nl ? __ldcg(p.leafv + (size_t)v * BH_LCAP + lane + 32 * u) : -1;
  const int ip0 = __ldg(p.item_ptr + v), ip1 = __ldg(p.item_ptr + v + 1);
  const int k0 = __ldg(p.rowptr + v), k1 = __ldg(p.rowptr + v + 1);
  const float2 cf = __ldcg(p.cellf + v);
  const bool split = ip1 - ip0 > 1;
  // per-lane sums of both chains, one reduction at the end
  float fx = 0.f, fy = 0.f, ax = 0.f, ay = 0.f;
  float2 cj[BH_LPL];
#pragma unroll
  for (int u = 0; u < BH_LPL; ++u) cj[u] = j[u] >= 0 ? bh_live(p, j[u], plo, phi, pend) : cv;
  if (!split) bh_attr_lane(p, k0, k1, cv, plo, phi, pend, ax, ay);
#pragma unroll
  for (int u = 0; u < BH_LPL; ++u)
    if (j[u] >= 0) {
      const float dx = cj[u].x - cv.x, dy = cj[u].y - cv.y;
      const float d2 = fmaf(dx, dx, dy * dy);
      if (d2 > 0.f) {
        const float r = bh_rep_weight(p, d2);
        fx = fmaf(-r, dx, fx);
        fy = fmaf(-r, dy, fy);
      }
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    fx += __shfl_xor_sync(0xffffffffu, fx, o);
    fy += __shfl_xor_sync(0xffffffffu, fy, o);
    ax += __shfl_xor_sync(0xffffffffu, ax, o);
    ay += __shfl_xor_sync(0xffffffffu, ay, o);
  }
  if (split) {
    const float2 g = bh_attr_gather(p, v, stamp);
    ax = g.x;
    ay = g.y;
  }
  return make_float2(fx + cf.x + ax, fy + cf.y + ay);
}

// Everything about a batch vertex that is constant within the iteration --
// its own coordinate (it does not move before its batch, reading B5), its
// precomputed cell sum and leaf list, its row bounds and first 32 neighbour
// ids -- loaded for the warp's first vertex of the NEXT batch between the
// arrival at the grid barrier and the wait, so that after the barrier only
// the live coordinates (leaf vertices, neighbours) are one L2 trip away.
// Before: four dependent trips per batch after three of the item pass.
struct BHPre {
  int valid, v, nl, j[BH_LPL], ip0, ip1, k0, k1, col;
  float2 cv, cf;
};
__device__ __forceinline__ void bh_prefetch(const BHKParams &p, int lo, int bt, BHPre &o) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int i = warp * gridDim.x + blockIdx.x;
  o.valid = p.precompute && i < bt;
  if (!o.valid) return;
  const int v = lo + i;
  o.v = v;
  o.cv = __ldcg(p.xy + v);
  o.nl = __ldcg(p.nleaf + v);
#pragma unroll
  for (int u = 0; u < BH_LPL; ++u)  // entries >= nl: masked by the user
    o.j[u] = __ldcg(p.leafv + (size_t)v * BH_LCAP + lane + 32 * u);
  o.ip0 = __ldg(p.item_ptr + v);
  o.ip1 = __ldg(p.item_ptr + v + 1);
  o.k0 = __ldg(p.rowptr + v);
  o.k1 = __ldg(p.rowptr + v + 1);
  o.cf = __ldcg(p.cellf + v);
  o.col = o.k0 + lane < o.k1 ? __ldg(p.colidx + o.k0 + lane) : -1;
}
// The edge-parallel pass over the split rows of a batch (layout mode): split
// item s of the batch goes to warp BH_NW-1 - s / G of CTA s mod G -- the warps
// that hold no batch vertex while b <= G BH_NW / 2 -- so the pass runs beside
// the forces instead of before them.  A warp's first item of the NEXT batch
// (ids, row range, the vertex's own coordinate, its <= BL_ECH neighbour ids)
// is prefetched with the batch vertex's inputs (bh_prefetch).
#define BH_IPL (BL_ECH / 32)
struct BHItemPre {
  int valid, sib, sie;  // the batch's split items [sib, sie)
  int4 it;              // this warp's first one: {item, vertex, k0, k1}
  int col[BH_IPL];
  float2 cv;
};
__device__ __forceinline__ int bh_item_rank() {
  return (BH_NW - 1 - (int)(threadIdx.x >> 5)) * gridDim.x + blockIdx.x;
}
__device__ __forceinline__ void bh_prefetch_item(const BHKParams &p, int lo, int bt, BHItemPre &o) {
  const int lane = threadIdx.x & 31;
  o.sib = __ldg(p.split_ptr + lo);
  o.sie = __ldg(p.split_ptr + lo + bt);
  const int s = o.sib + bh_item_rank();
  o.valid = s < o.sie;
  if (!o.valid) return;
  o.it = __ldg(p.sitems + s);
  o.cv = __ldcg(p.xy + o.it.y);
#pragma unroll
  for (int u = 0; u < BH_IPL; ++u) {
    const int k = o.it.z + lane + 32 * u;
    o.col[u] = k < o.it.w ? __ldg(p.colidx + k) : -1;
  }
}
// publish one item's partial (release flag stamped with the batch)
__device__ __forceinline__ void bh_item_publish(const BHKParams &p, int a, float fx, float fy,
                                                unsigned stamp) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    fx += __shfl_xor_sync(0xffffffffu, fx, o);
    fy += __shfl_xor_sync(0xffffffffu, fy, o);
  }
  if ((threadIdx.x & 31) == 0) {
    bh_st_relaxed_v2(&p.attr_ll[a].x, __float_as_uint(fx), stamp);
    bh_st_relaxed_v2(&p.attr_ll[a].z, __float_as_uint(fy), stamp);
  }
}
__device__ __forceinline__ void bh_items_batch(const BHKParams &p, const BHItemPre &o, unsigned stamp,
                                               int plo, int phi, const float2 *pend) {
  const int GW = gridDim.x * BH_NW;
  int s = o.sib + bh_item_rank();
  if (o.valid) {  // the prefetched item: only the live coordinates are loaded here
    float2 cj[BH_IPL];
#pragma unroll
    for (int u = 0; u < BH_IPL; ++u)
      cj[u] = o.col[u] >= 0 ? bh_live(p, o.col[u], plo, phi, pend) : o.cv;
    float fx = 0.f, fy = 0.f;
#pragma unroll
    for (int u = 0; u < BH_IPL; ++u)
      if (o.col[u] >= 0) bh_attr_term(p, cj[u], o.cv, fx, fy);
    bh_item_publish(p, o.it.x, fx, fy, stamp);
    s += GW;
  }
  for (; s < o.sie; s += GW) {
    const int4 it = __ldg(p.sitems + s);
    float fx = 0.f, fy = 0.f;
    bh_attr_lane(p, it.z, it.w, __ldcg(p.xy + it.y), plo, phi, pend, fx, fy);
    bh_item_publish(p, it.x, fx, fy, stamp);
  }
}

// bh_force_pre on prefetched inputs: the same terms in the same order.
__device__ __forceinline__ float2 bh_force_pre2(const BHKParams &p, const BHPre &o, int plo, int phi,
                                                const float2 *pend, unsigned stamp) {
  const int lane = threadIdx.x & 31;
  const bool split = o.ip1 - o.ip0 > 1;
  const float2 cv = o.cv;
  float fx = 0.f, fy = 0.f, ax = 0.f, ay = 0.f;
  int j[BH_LPL];
  float2 cj[BH_LPL], cn = cv;
#pragma unroll
  for (int u = 0; u < BH_LPL; ++u) {
    j[u] = lane + 32 * u < o.nl ? o.j[u] : -1;
    cj[u] = j[u] >= 0 ? bh_live(p, j[u], plo, phi, pend) : cv;
  }
  if (!split && o.col >= 0) cn = bh_live(p, o.col, plo, phi, pend);
  if (!split) {
    if (o.col >= 0) bh_attr_term(p, cn, cv, ax, ay);
    bh_attr_lane(p, o.k0 + 32, o.k1, cv, plo, phi, pend, ax, ay);
  }
#pragma unroll
  for (int u = 0; u < BH_LPL; ++u)
    if (j[u] >= 0) {
      const float dx = cj[u].x - cv.x, dy = cj[u].y - cv.y;
      const float d2 = fmaf(dx, dx, dy * dy);
      if (d2 > 0.f) {
        const float r = bh_rep_weight(p, d2);
        fx = fmaf(-r, dx, fx);
        fy = fmaf(-r, dy, fy);
      }
    }
#pragma unroll
  for (int o2 = 16; o2 > 0; o2 >>= 1) {
    fx += __shfl_xor_sync(0xffffffffu, fx, o2);
    fy += __shfl_xor_sync(0xffffffffu, fy, o2);
    ax += __shfl_xor_sync(0xffffffffu, ax, o2);
    ay += __shfl_xor_sync(0xffffffffu, ay, o2);
  }
  if (split) {
    const float2 g = bh_attr_gather(p, o.v, stamp);
    ax = g.x;
    ay = g.y;
  }
  return make_float2(fx + o.cf.x + ax, fy + o.cf.y + ay);
}

// Fixed-order sum of the G per-CTA fp64 energies by one warp (identical in
// every CTA, so the tol decision is too).
__device__ __forceinline__ double bh_energy_sum(const BHKParams &p) {
  const int G = gridDim.x, lane = threadIdx.x & 31;
  double e = 0.0;
  for (int cc = lane; cc < G; cc += 32) e += __ldcg(p.e_cta + cc);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
  return e;
}

// Alg. S3's iterations: tree per iteration, then the dependent minibatches
// with ONE grid barrier each.  Phase t: every warp computes the force of its
// batch-t vertex and writes the new coordinate to pend[t & 1] (not to xy:
// other warps still read batch t's frozen coordinates); meanwhile batch t-1's
// new coordinates are committed from pend to xy, and readers take batch t-1
// vertices from pend.  The last batch of an iteration is committed before the
// next tree is built (its own barrier).
template <int NT>
__device__ void bh_run_batches(const BHKParams &p, BHShared &sh, unsigned &bar_target,
                               int *unit_dummy_ptr, unsigned long long &vis, BLProf &pf) {
  const int G = gridDim.x, c = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gw = c * BH_NW + warp, GW = G * BH_NW;
  double step = p.step0, e_prev = 0.0;
  int batches = 0, done = 0;
  bool stop = false;
  int plo = 0, phi = 0;  // batch whose new coordinates are still in pend
  for (int it = 0; it < p.iters && !stop; ++it) {
    if (phi > plo) {  // commit the previous iteration's last batch
      const float2 *pd = p.pend + (size_t)(((batches - 1) & 1) * p.b);
      for (int i = c * NT + threadIdx.x; i < phi - plo; i += G * NT) p.xy[plo + i] = __ldcg(pd + i);
      plo = phi = 0;
      bl_grid_sync(p.bar, bar_target, unit_dummy_ptr);
    }
    pf.mark(4);
    bh_build_tree<NT>(p, sh, bar_target, unit_dummy_ptr, pf);  // Alg. S3 lines 5-8
    if (p.precompute) {
      bh_precompute(p, vis);
      bl_grid_sync(p.bar, bar_target, unit_dummy_ptr);
      pf.mark(7);
    }
    double e_acc = 0.0;
    const int pre_on = p.pre2;
    BHPre pre;
    pre.valid = 0;
    BHItemPre ipre;
    ipre.valid = 0;
    if (pre_on) {
      bh_prefetch(p, 0, min(p.b, p.n), pre);
      bh_prefetch_item(p, 0, min(p.b, p.n), ipre);
    }
    for (int t = 0; t < p.nb; ++t) {
      const int lo = t * p.b, bt = min(p.b, p.n - lo);
      float2 *pend_t = p.pend + (size_t)((batches & 1) * p.b);
      const float2 *pend_prev = p.pend + (size_t)(((batches - 1) & 1) * p.b);
      // commit batch t-1 (nobody reads its xy entries in this phase): by the
      // upper half of every CTA's warps, which hold no batch vertex while
      // b <= G BH_NW / 2 (CTAs 0 and 1 alone used to do it, ahead of their
      // own vertices' forces: 0.4 us on the batch's critical path)
      if (pre_on) {
        for (int i = c * (NT / 2) + (int)threadIdx.x - NT / 2; threadIdx.x >= NT / 2 && i < phi - plo;
             i += G * (NT / 2))
          p.xy[plo + i] = __ldcg(pend_prev + i);
      } else {
        for (int i = c * NT + threadIdx.x; i < phi - plo; i += G * NT)
          p.xy[plo + i] = __ldcg(pend_prev + i);
      }
      // F: forces of batch t against frozen coordinates (lines 13-20), then
      // the update (lines 21-24) into pend.  Long CSR rows first, edge-
      // parallel over all warps (no warp waits before its items are done);
      // skipped when the batch has no split row.
      const unsigned stamp = (unsigned)batches + 1u;
#ifdef BH_FINE_TS
      pf.mark(0);  // commit
#endif
      if (pre_on) bh_items_batch(p, ipre, stamp, plo, phi, pend_prev);
      else bh_attr_items(p, lo, lo + bt, gw, GW, stamp, plo, phi, pend_prev);
#ifdef BH_FINE_TS
      pf.mark(1);  // item pass
#endif
      // batch entry i -> CTA i mod G, warp i / G: the queries spread over
      // all SMs (b = 1024 on 148 SMs: ~7 concurrent traversals per SM)
      for (int i = warp * G + c; i < bt; i += GW) {
        const int v = lo + i;
        const bool fast = pre.valid && i == warp * G + c && pre.nl >= 0;
        float2 cv, f;
        if (fast) {
          cv = pre.cv;
          f = bh_force_pre2(p, pre, plo, phi, pend_prev, stamp);
        } else {
          cv = __ldcg(p.xy + v);
          const int nl = p.precompute ? __ldcg(p.nleaf + v) : -1;
          f = nl >= 0 ? bh_force_pre(p, v, cv, nl, plo, phi, pend_prev, stamp)
                      : bh_force_warp(p, sh, v, cv, plo, phi, pend_prev, stamp, vis);
        }
        if (lane == 0) {
          const double q = (double)f.x * f.x + (double)f.y * f.y;
          float2 nv = cv;
          if (q > 0.0) {
            const double s = step / sqrt(q);
            nv.x = (float)((double)cv.x + s * f.x);
            nv.y = (float)((double)cv.y + s * f.y);
          }
          pend_t[i] = nv;
          e_acc += q;
        }
      }
#ifdef BH_FINE_TS
      pf.mark(2);  // force + update of this warp's vertices
#endif
      ++batches;
      const bool last = t == p.nb - 1;
      const bool mb = p.max_batches > 0 && batches >= p.max_batches;
      if (last || mb) {
        double e = e_acc;  // only lane 0 of each warp holds a value
        if (lane == 0) sh.e_warp[warp] = e;
        __syncthreads();
        if (threadIdx.x == 0) {
          double s = 0.0;
          for (int w = 0; w < BH_NW; ++w) s += sh.e_warp[w];
          p.e_cta[c] = s;
        }
      }
      pf.mark(5);
      // grid barrier, split: the next batch's iteration-constant inputs are
      // loaded between the arrival and the wait
      __syncthreads();
      if (threadIdx.x == 0) {
        bar_target += gridDim.x;
        asm volatile("fence.acq_rel.gpu;\n\tred.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(p.bar)
                     : "memory");
      }
      pre.valid = 0;
      ipre.valid = 0;
      if (pre_on && !last && !mb) {
        const int lo2 = lo + p.b, bt2 = min(p.b, p.n - lo2);
        bh_prefetch(p, lo2, bt2, pre);
        bh_prefetch_item(p, lo2, bt2, ipre);
      }
      if (threadIdx.x == 0)
        while ((int)(bl_ld_acquire(p.bar) - bar_target) < 0) {
        }
      __syncthreads();
      pf.mark(6);
      plo = lo;
      phi = lo + bt;
      if (last || mb) {
        // identical fixed-order sum in every CTA -> identical tol decision
        const double E = bh_energy_sum(p);
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
  // commit the last batch (the kernel ends: no reader left)
  if (phi > plo) {
    const float2 *pd = p.pend + (size_t)(((batches - 1) & 1) * p.b);
    for (int i = c * NT + threadIdx.x; i < phi - plo; i += G * NT) p.xy[plo + i] = __ldcg(pd + i);
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
  BLProf pf;
  pf.on = p.prof != nullptr && threadIdx.x == 0;
  for (int i = 0; i < 8; ++i) pf.acc[i] = 0;
  pf.last = pf.on ? clock64() : 0;

  if (p.forces_mode) {
    bh_build_tree<NT>(p, sh, bar_target, &unit_dummy, pf);
    bh_attr_items(p, p.first, p.first + p.count, gw, GW, 1u, 0, 0, p.pend);
    for (int t = gw; t < p.count; t += GW) {
      const int v = p.first + t;
      const float2 f = bh_force_warp(p, sh, v, __ldcg(p.xy + v), 0, 0, p.pend, 1u, vis);
      if (lane == 0) p.f_out[t] = f;
    }
  } else {
    bh_run_batches<NT>(p, sh, bar_target, &unit_dummy, vis, pf);
  }
  if (pf.on) {
    if (c == 0)
      for (int i = 0; i < 8; ++i) p.prof[i] = pf.acc[i];
    p.prof[8 + c] = pf.acc[5];
  }

  // visits: per-CTA totals (deterministic sum later on the host)
  unsigned long long vsum = vis;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) vsum += __shfl_xor_sync(0xffffffffu, vsum, o);
  if (lane == 0) atomicAdd(p.visits + c, vsum);
}
