/*
 * bl_oracle_bh.h -- oracle of BatchLayoutBH (Barnes-Hut repulsion), fp64,
 * included once by bl_oracle.c.  TEST INFRASTRUCTURE ONLY (see bl_oracle.c).
 *
 * Follows the supplement's algorithms step by step:
 *   Alg. S3 (BatchLayoutBH): per iteration, bounding box,
 *     D = max extent, Morton sort, constructBHT; then the minibatch loop with
 *     CSR attraction + calcRepulsiveForce, batch update, energy, cooling.
 *   Alg. S1 (constructBHT): recursive four-way split of a
 *     Morton-contiguous range, diameter halved per level, centroid from the
 *     children.
 *   Alg. S2 (calcRepulsiveForce): MAC theta > D/d at a node (d =
 *     distance from the query to the node's centroid) accepts the centroid;
 *     otherwise recurse into children, exact pair terms at leaves.
 *   §3.5: Warren-Salmon hashed quadtree, Morton (Z) order, MAC,
 *     theta = 1.2.
 *
 * Readings (B1-B9):
 *   B1 Alg. S2's accepted branch says f_a; it is the repulsive force f_r.
 *   B2 an accepted centroid stands for all `count` vertices of the node: the
 *      term is count * f_r(d) * u (standard Barnes-Hut mass weighting).
 *   B3 Alg. S3's "f = f - rf" is read so that f = attraction + repulsion, the
 *      f(i, c) of §2.2; adjacent pairs attract AND repel (Alg. S3 adds the
 *      tree repulsion over all vertices), i.e. REPULSE_NEIGHBORS semantics.
 *   B4 "re-scale c in bounding box" = compute the box; coordinates unchanged.
 *   B5 the tree (cells, centroids) is built once per iteration from the
 *      coordinates at the iteration start; leaf terms use the live (current,
 *      batch-frozen) coordinates of the leaf's vertices, so theta = 0 is
 *      exactly the exact method (with REPULSE_NEIGHBORS) for any batch size.
 *   B6 quantisation: 16 bits per axis, q = floor((x - xmin) * (65536 / D))
 *      clamped to 65535 (0 if D = 0); code bit 2k = qx bit k, bit 2k+1 = qy
 *      bit k; level-L digit = bits (31-2L, 30-2L); children in digit order.
 *      A range still holding >1 vertex at level 16 (identical codes) is a
 *      multi-vertex leaf, summed exactly.  Stable sort: ties by vertex id.
 *   B7 decisions that turn floating point into structure (codes, MAC) are
 *      taken in fp32, the precision of the kernel's coordinates, with
 *      separately rounded operations: the box, D, codes and centroids come
 *      from the fp32 rounding of the coordinates; the MAC is
 *      theta^2 * (dx*dx + dy*dy) > (D / 2^L)^2 in fp32.  Centroids: fp64 sums
 *      of fp32 coordinates over the children in digit order, divided by the
 *      count in fp64, rounded to fp32.  Force terms are fp64.
 *   B8 an internal node is tested against the MAC, the root included; the
 *      query's own vertex inside an accepted centroid is not removed (the
 *      paper's MAC as written); at a leaf the query vertex itself is skipped.
 *   B9 coincident pairs (d = 0) contribute nothing (reading C4).
 */

typedef struct {
  int level, start, count, nchild, child[4];
  double sx, sy;  /* fp64 sums of the fp32 coordinates of the node's vertices */
  float cx, cy;   /* centroid, rounded to fp32 (B7) */
} bh_node;

typedef struct {
  int n, nn, cap;
  bh_node *node;
  uint32_t *code;  /* sorted Morton codes */
  int *perm;       /* vertex ids in Morton order */
  float *sx, *sy;  /* fp32 snapshot coordinates in Morton order */
  float D;         /* root diameter (fp32) */
} bh_tree;

static uint32_t bh_interleave(uint32_t qx, uint32_t qy) {
  uint32_t c = 0;
  for (int k = 0; k < 16; ++k) {
    c |= ((qx >> k) & 1u) << (2 * k);
    c |= ((qy >> k) & 1u) << (2 * k + 1);
  }
  return c;
}

/* B6/B7: fp32 quantisation of one coordinate */
static uint32_t bh_quant(float x, float xmin, float scale, int degenerate) {
  if (degenerate) return 0;
  const float t = (x - xmin) * scale;
  float fl = floorf(t);
  if (fl < 0.0f) fl = 0.0f;
  if (fl > 65535.0f) fl = 65535.0f;
  return (uint32_t)fl;
}

typedef struct {
  uint32_t code;
  int id;
} bh_key;

static int bh_key_cmp(const void *a, const void *b) {
  const bh_key *x = (const bh_key *)a, *y = (const bh_key *)b;
  if (x->code != y->code) return x->code < y->code ? -1 : 1;
  return (x->id > y->id) - (x->id < y->id); /* stable: ties by vertex id */
}

/* Alg. S1 constructBHT on the Morton-contiguous range [lo, hi) at level L.
 * Returns the node's index (pre-order: parent before children). */
static int bh_construct(bh_tree *t, int lo, int hi, int L) {
  const int idx = t->nn++;
  bh_node nd;
  memset(&nd, 0, sizeof nd);
  nd.level = L;
  nd.start = lo;
  nd.count = hi - lo;
  if (nd.count == 1 || L == 16) {
    /* leaf: one vertex, or the multi-vertex leaf of identical codes (B6) */
    double sx = 0, sy = 0;
    for (int k = lo; k < hi; ++k) {
      sx = sx + (double)t->sx[k];
      sy = sy + (double)t->sy[k];
    }
    nd.sx = sx;
    nd.sy = sy;
  } else {
    /* the four cells of the next level, in digit order (B6) */
    const int shift = 30 - 2 * L;
    int a = lo;
    double sx = 0, sy = 0;
    for (uint32_t q = 0; q < 4; ++q) {
      int b = a;
      while (b < hi && ((t->code[b] >> shift) & 3u) == q) ++b;
      if (b > a) {
        const int ch = bh_construct(t, a, b, L + 1);
        nd.child[nd.nchild++] = ch;
        sx = sx + t->node[ch].sx; /* centroid from the children (Alg. S1 l.11) */
        sy = sy + t->node[ch].sy;
      }
      a = b;
    }
    nd.sx = sx;
    nd.sy = sy;
  }
  nd.cx = (float)(nd.sx / (double)nd.count);
  nd.cy = (float)(nd.sy / (double)nd.count);
  t->node[idx] = nd;
  return idx;
}

/* Alg. S3 lines 5-8: box, D, Morton sort, tree -- from the fp32 rounding of
 * the coordinates xy (B5, B7).  Returns 0, or -1 on allocation failure. */
static int bh_tree_build(bh_tree *t, int32_t n, const float *xy) {
  memset(t, 0, sizeof *t);
  t->n = n;
  t->cap = 17 * n + 1; /* at most 17 nodes per vertex (a chain of 17 levels) */
  t->node = (bh_node *)malloc(sizeof(bh_node) * (size_t)t->cap);
  t->code = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)n);
  t->perm = (int *)malloc(sizeof(int) * (size_t)n);
  t->sx = (float *)malloc(sizeof(float) * (size_t)n);
  t->sy = (float *)malloc(sizeof(float) * (size_t)n);
  bh_key *keys = (bh_key *)malloc(sizeof(bh_key) * (size_t)n);
  if (!t->node || !t->code || !t->perm || !t->sx || !t->sy || !keys) {
    free(keys);
    return -1;
  }
  float xmin = xy[0], xmax = xy[0], ymin = xy[1], ymax = xy[1];
  for (int32_t i = 1; i < n; ++i) {
    xmin = fminf(xmin, xy[2 * i]);
    xmax = fmaxf(xmax, xy[2 * i]);
    ymin = fminf(ymin, xy[2 * i + 1]);
    ymax = fmaxf(ymax, xy[2 * i + 1]);
  }
  const float ex = xmax - xmin, ey = ymax - ymin;
  t->D = ex > ey ? ex : ey; /* Alg. S3 line 7 */
  const int degenerate = !(t->D > 0.0f);
  const float scale = degenerate ? 0.0f : 65536.0f / t->D;
  for (int32_t i = 0; i < n; ++i) {
    keys[i].code = bh_interleave(bh_quant(xy[2 * i], xmin, scale, degenerate),
                                 bh_quant(xy[2 * i + 1], ymin, scale, degenerate));
    keys[i].id = i;
  }
  qsort(keys, (size_t)n, sizeof(bh_key), bh_key_cmp); /* Alg. S3 line 6 */
  for (int32_t k = 0; k < n; ++k) {
    t->code[k] = keys[k].code;
    t->perm[k] = keys[k].id;
    t->sx[k] = xy[2 * keys[k].id];
    t->sy[k] = xy[2 * keys[k].id + 1];
  }
  free(keys);
  bh_construct(t, 0, n, 0); /* Alg. S3 line 8 */
  return 0;
}

static void bh_tree_free(bh_tree *t) {
  free(t->node);
  free(t->code);
  free(t->perm);
  free(t->sx);
  free(t->sy);
}

/* Alg. S2 calcRepulsiveForce for query vertex i at live position (xi, yi).
 * c = live coordinates (fp64).  Accumulates into (fx, fy); counts visits. */
static void bh_repulse(const bh_tree *t, int r, int32_t i, double xi, double yi, const double *c,
                       double ck2, float theta2, double *fx, double *fy, long long *visits) {
  const bh_node *nd = &t->node[r];
  ++*visits;
  if (nd->nchild == 0) {
    /* leaf: exact pair terms with the live coordinates (B5, B8, B9) */
    for (int k = nd->start; k < nd->start + nd->count; ++k) {
      const int j = t->perm[k];
      if (j == i) continue;
      const double dx = c[2 * j] - xi, dy = c[2 * j + 1] - yi;
      const double d2 = dx * dx + dy * dy;
      if (d2 == 0) continue;
      if (g_model_r == -1.0) {
        *fx = *fx - ck2 * dx / d2; /* f_r(d) * (c_j - c_i)/d, f_r = -CK^2/d */
        *fy = *fy - ck2 * dy / d2;
      } else {
        const double d = sqrt(d2), w = ck2 * pow(d, g_model_r) / d; /* f_r = -CK^2 d^r */
        *fx = *fx - w * dx;
        *fy = *fy - w * dy;
      }
    }
    return;
  }
  /* MAC in fp32 (B7): theta > D_L/d  <=>  theta^2 d^2 > D_L^2 */
  const float qx = (float)xi, qy = (float)yi;
  const float ddx = nd->cx - qx, ddy = nd->cy - qy;
  const float dd2 = ddx * ddx + ddy * ddy;
  const float DL = ldexpf(t->D, -nd->level);
  if (theta2 * dd2 > DL * DL) {
    /* accepted: count x f_r at the centroid (B1, B2) */
    const double dx = (double)nd->cx - xi, dy = (double)nd->cy - yi;
    const double d2 = dx * dx + dy * dy;
    if (d2 > 0) {
      if (g_model_r == -1.0) {
        *fx = *fx - (double)nd->count * ck2 * dx / d2;
        *fy = *fy - (double)nd->count * ck2 * dy / d2;
      } else {
        const double d = sqrt(d2), w = (double)nd->count * ck2 * pow(d, g_model_r) / d;
        *fx = *fx - w * dx;
        *fy = *fy - w * dy;
      }
    }
    return;
  }
  for (int k = 0; k < nd->nchild; ++k)
    bh_repulse(t, nd->child[k], i, xi, yi, c, ck2, theta2, fx, fy, visits);
}

/* f(i, c) of Alg. S3 lines 13-19: attraction over N(i) with the live
 * coordinates plus the tree repulsion (B3). */
static void bh_force(int32_t n, const int32_t *rowptr, const int32_t *colidx, const double *c,
                     const bh_tree *t, int32_t i, double K, double ck2, float theta2, double *fx_out,
                     double *fy_out, long long *visits) {
  (void)n;
  double fx = 0, fy = 0;
  const double xi = c[2 * i], yi = c[2 * i + 1];
  for (int32_t k = rowptr[i]; k < rowptr[i + 1]; ++k) {
    const int32_t j = colidx[k];
    const double dx = c[2 * j] - xi, dy = c[2 * j + 1] - yi;
    const double d = sqrt(dx * dx + dy * dy);
    if (d == 0) continue;
    const double fa = f_attr_f64(d, K); /* f_a = ||c_i - c_j||^a / K */
    fx = fx + fa * dx / d;
    fy = fy + fa * dy / d;
  }
  double rx = 0, ry = 0;
  if (t->nn > 0) bh_repulse(t, 0, i, xi, yi, c, ck2, theta2, &rx, &ry, visits);
  *fx_out = fx + rx;
  *fy_out = fy + ry;
}

static float *bh_round_f32(int32_t n, const double *c) {
  float *f = (float *)malloc(sizeof(float) * 2 * (size_t)n);
  if (f)
    for (int64_t k = 0; k < 2 * (int64_t)n; ++k) f[k] = (float)c[k];
  return f;
}

/* Forces of vertices [first, first+count): tree from snap (fp32), live
 * coordinates `live` (fp64).  f_out: 2*count.  visits (nullable): total
 * nodes visited. */
int oracle_bh_forces(int32_t n, const int32_t *rowptr, const int32_t *colidx, const float *snap,
                     const double *live, int32_t first, int32_t count, double K, double C,
                     double theta, double *f_out, long long *visits) {
  if (n < 1 || first < 0 || count < 0 || first + count > n || !(theta >= 0)) return -1;
  bh_tree t;
  if (bh_tree_build(&t, n, snap) != 0) {
    bh_tree_free(&t);
    return -1;
  }
  const float th = (float)theta, theta2 = th * th;
  long long v = 0;
  for (int32_t k = 0; k < count; ++k)
    bh_force(n, rowptr, colidx, live, &t, first + k, K, C * K * K, theta2, &f_out[2 * k],
             &f_out[2 * k + 1], &v);
  if (visits) *visits = v;
  bh_tree_free(&t);
  return 0;
}

/* Alg. S3 BatchLayoutBH.  Same conventions as oracle_layout (xy in/out fp64,
 * energy[iters], max_batches, tol). */
int oracle_bh_layout(int32_t n, const int32_t *rowptr, const int32_t *colidx, double *xy,
                     int32_t iters, int32_t batch, double K, double C, double step0,
                     double cooling, double theta, int32_t max_batches, double tol,
                     double *energy, int32_t *iters_done, long long *visits) {
  if (n < 1 || iters < 0 || batch < 1 || !(theta >= 0)) return -1;
  if (batch > n) batch = n;
  double *ct = (double *)malloc(sizeof(double) * 2 * (size_t)batch);
  if (!ct) return -1;
  const float th = (float)theta, theta2 = th * th;
  const double ck2 = C * K * K;
  double step = step0, E_prev = 0;
  int32_t batches_done = 0, it_done = 0;
  int stop = 0;
  long long v = 0;
  for (int32_t it = 0; it < iters && !stop; ++it) {
    double E = 0; /* Alg. S3 line 4 */
    float *snap = bh_round_f32(n, xy);
    bh_tree t;
    if (!snap || bh_tree_build(&t, n, snap) != 0) {
      free(snap);
      free(ct);
      return -1;
    }
    for (int32_t lo = 0; lo < n; lo += batch) { /* line 12 */
      const int32_t hi = lo + batch < n ? lo + batch : n;
      for (int32_t i = lo; i < hi; ++i) /* lines 13-20, coordinates frozen */
        bh_force(n, rowptr, colidx, xy, &t, i, K, ck2, theta2, &ct[2 * (i - lo)],
                 &ct[2 * (i - lo) + 1], &v);
      for (int32_t i = lo; i < hi; ++i) { /* lines 21-24 */
        const double fx = ct[2 * (i - lo)], fy = ct[2 * (i - lo) + 1];
        const double q = fx * fx + fy * fy;
        if (q > 0) {
          const double nrm = sqrt(q);
          xy[2 * i] = xy[2 * i] + step * (fx / nrm);
          xy[2 * i + 1] = xy[2 * i + 1] + step * (fy / nrm);
        }
        E = E + q;
      }
      ++batches_done;
      if (max_batches > 0 && batches_done >= max_batches) {
        stop = 1;
        if (energy) energy[it] = E;
        break;
      }
    }
    bh_tree_free(&t);
    free(snap);
    if (!stop) {
      if (energy) energy[it] = E;
      ++it_done;
      step = step * cooling;
      if (tol > 0 && it > 0 && fabs(E - E_prev) < tol) break;
      E_prev = E;
    }
  }
  free(ct);
  if (iters_done) *iters_done = it_done;
  if (visits) *visits = v;
  return 0;
}

/* The tree of Alg. S1 for pins: node arrays in pre-order (cap entries at
 * most; returns the node count, or -1).  child: 4 ints per node (-1 pads).
 * codes/perm: n entries.  D_out: root diameter. */
int oracle_bh_tree(int32_t n, const float *xy, int32_t cap, int32_t *level, int32_t *start,
                   int32_t *count, int32_t *nchild, int32_t *child, float *cx, float *cy,
                   uint32_t *codes, int32_t *perm, float *D_out) {
  if (n < 1) return -1;
  bh_tree t;
  if (bh_tree_build(&t, n, xy) != 0) {
    bh_tree_free(&t);
    return -1;
  }
  if (t.nn > cap) {
    bh_tree_free(&t);
    return -1;
  }
  for (int k = 0; k < t.nn; ++k) {
    level[k] = t.node[k].level;
    start[k] = t.node[k].start;
    count[k] = t.node[k].count;
    nchild[k] = t.node[k].nchild;
    for (int q = 0; q < 4; ++q) child[4 * k + q] = q < t.node[k].nchild ? t.node[k].child[q] : -1;
    cx[k] = t.node[k].cx;
    cy[k] = t.node[k].cy;
  }
  for (int32_t k = 0; k < n; ++k) {
    codes[k] = t.code[k];
    perm[k] = t.perm[k];
  }
  *D_out = t.D;
  const int nn = t.nn;
  bh_tree_free(&t);
  return nn;
}
