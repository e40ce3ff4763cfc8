/*
 * bl_oracle_metrics.h -- oracle of the layout quality metrics of §3.7
 * (PAPER.md P:841-857), included once by bl_oracle.c.  TEST INFRASTRUCTURE
 * ONLY.  Readings M1-M5:
 *   M1 Stress: ST = sum over ordered pairs (i, j), i != j, j reachable
 *      from i, of w_ij (s ||c_i - c_j|| - d_ij)^2, w_ij = 1/d_ij^2, d_ij = BFS
 *      hop distance; "the reported value is the minimum value achievable
 *      after scaling the layout" -> s* = sum w d ||D|| / sum w ||D||^2 in
 *      closed form.  Unreachable pairs are excluded and counted.  A source
 *      subset S (all vertices by default) restricts i to S (sampling).
 *   M2 Edge uniformity: sqrt(sum_e (l_e - l_mu)^2 / (|E| l_mu^2)),
 *      each undirected edge once (i < j), two passes in fp64.
 *   M3 Neighborhood preservation: the paper gives no formula; for
 *      each vertex i with k = deg(i) > 0, the k layout-nearest other vertices
 *      (squared distance in fp32 with separately rounded operations, ties by
 *      vertex id) are compared with N(i) by Jaccard |A n B| / |A u B|; NP =
 *      mean over those vertices (SPEC.md S:475-494's reading).  A query subset
 *      restricts the mean.
 *   M4 fp64 accumulation throughout; the NP selection in fp32 (the kernel's
 *      precision, it decides set membership).
 */

/* M1: BFS from each source in S; accumulates A = sum ||D||/d, B = sum
 * ||D||^2/d^2, N = pairs (w d^2 = 1), so ST(s) = s^2 B - 2 s A + N. */
int oracle_stress(int32_t n, const int32_t *rowptr, const int32_t *colidx, const float *xy,
                  const int32_t *sources, int32_t nsrc, double *stress, double *scale,
                  long long *pairs, long long *unreachable) {
  if (n < 1 || nsrc < 0) return -1;
  int32_t *dist = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
  int32_t *queue = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
  if (!dist || !queue) {
    free(dist);
    free(queue);
    return -1;
  }
  double A = 0, B = 0;
  long long N = 0, U = 0;
  const int32_t ns = sources ? nsrc : n;
  for (int32_t t = 0; t < ns; ++t) {
    const int32_t s = sources ? sources[t] : t;
    if (s < 0 || s >= n) {
      free(dist);
      free(queue);
      return -1;
    }
    for (int32_t v = 0; v < n; ++v) dist[v] = -1;
    int32_t head = 0, tail = 0;
    dist[s] = 0;
    queue[tail++] = s;
    while (head < tail) {
      const int32_t u = queue[head++];
      for (int32_t k = rowptr[u]; k < rowptr[u + 1]; ++k)
        if (dist[colidx[k]] < 0) {
          dist[colidx[k]] = dist[u] + 1;
          queue[tail++] = colidx[k];
        }
    }
    for (int32_t v = 0; v < n; ++v) {
      if (v == s) continue;
      if (dist[v] < 0) {
        ++U;
        continue;
      }
      const double dx = (double)xy[2 * v] - (double)xy[2 * s];
      const double dy = (double)xy[2 * v + 1] - (double)xy[2 * s + 1];
      const double l2 = dx * dx + dy * dy, d = (double)dist[v];
      A = A + sqrt(l2) / d;
      B = B + l2 / (d * d);
      ++N;
    }
  }
  free(dist);
  free(queue);
  const double sc = B > 0 ? A / B : 0.0;
  *scale = sc;
  *stress = sc * sc * B - 2.0 * sc * A + (double)N;
  *pairs = N;
  *unreachable = U;
  return 0;
}

/* M2 */
int oracle_edge_uniformity(int32_t n, const int32_t *rowptr, const int32_t *colidx,
                           const float *xy, double *eu) {
  if (n < 1) return -1;
  double sum = 0;
  long long m = 0;
  for (int32_t i = 0; i < n; ++i)
    for (int32_t k = rowptr[i]; k < rowptr[i + 1]; ++k) {
      const int32_t j = colidx[k];
      if (j <= i) continue;
      const double dx = (double)xy[2 * j] - (double)xy[2 * i];
      const double dy = (double)xy[2 * j + 1] - (double)xy[2 * i + 1];
      sum = sum + sqrt(dx * dx + dy * dy);
      ++m;
    }
  if (m == 0) {
    *eu = 0.0;
    return 0;
  }
  const double mu = sum / (double)m;
  double ss = 0;
  for (int32_t i = 0; i < n; ++i)
    for (int32_t k = rowptr[i]; k < rowptr[i + 1]; ++k) {
      const int32_t j = colidx[k];
      if (j <= i) continue;
      const double dx = (double)xy[2 * j] - (double)xy[2 * i];
      const double dy = (double)xy[2 * j + 1] - (double)xy[2 * i + 1];
      const double e = sqrt(dx * dx + dy * dy) - mu;
      ss = ss + e * e;
    }
  *eu = mu > 0 ? sqrt(ss / ((double)m * mu * mu)) : 0.0;
  return 0;
}

typedef struct {
  float d2;
  int32_t id;
} np_key;

static int np_cmp(const void *a, const void *b) {
  const np_key *x = (const np_key *)a, *y = (const np_key *)b;
  if (x->d2 != y->d2) return x->d2 < y->d2 ? -1 : 1;
  return (x->id > y->id) - (x->id < y->id);
}

/* M3: queries = NULL -> all vertices.  np_out: mean Jaccard; counted: the
 * number of vertices with deg > 0 among the queries.  jac (nullable): the
 * per-query Jaccard (-1 for deg 0). */
int oracle_neighborhood_preservation(int32_t n, const int32_t *rowptr, const int32_t *colidx,
                                     const float *xy, const int32_t *queries, int32_t nq,
                                     double *np_out, int32_t *counted, double *jac) {
  if (n < 1 || nq < 0) return -1;
  np_key *keys = (np_key *)malloc(sizeof(np_key) * (size_t)n);
  unsigned char *mark = (unsigned char *)calloc((size_t)n, 1);
  if (!keys || !mark) {
    free(keys);
    free(mark);
    return -1;
  }
  const int32_t nqq = queries ? nq : n;
  double sum = 0;
  int32_t cnt = 0;
  for (int32_t t = 0; t < nqq; ++t) {
    const int32_t i = queries ? queries[t] : t;
    const int32_t k = rowptr[i + 1] - rowptr[i];
    if (k == 0) {
      if (jac) jac[t] = -1;
      continue;
    }
    int32_t m = 0;
    for (int32_t l = 0; l < n; ++l) {
      if (l == i) continue;
      const float dx = xy[2 * l] - xy[2 * i], dy = xy[2 * l + 1] - xy[2 * i + 1];
      keys[m].d2 = dx * dx + dy * dy; /* fp32, separately rounded (M4) */
      keys[m].id = l;
      ++m;
    }
    qsort(keys, (size_t)m, sizeof(np_key), np_cmp);
    for (int32_t e = rowptr[i]; e < rowptr[i + 1]; ++e) mark[colidx[e]] = 1;
    int32_t inter = 0;
    for (int32_t r = 0; r < k && r < m; ++r) inter += mark[keys[r].id];
    for (int32_t e = rowptr[i]; e < rowptr[i + 1]; ++e) mark[colidx[e]] = 0;
    const double J = (double)inter / (double)(2 * k - inter);
    if (jac) jac[t] = J;
    sum = sum + J;
    ++cnt;
  }
  free(keys);
  free(mark);
  *np_out = cnt ? sum / cnt : 0.0;
  *counted = cnt;
  return 0;
}
