/*
 * bl_oracle_init.h -- oracle of the greedy initialisation (Alg. 3, PAPER.md
 * P:809-835, §3.6), included once by bl_oracle.c.  TEST
 * INFRASTRUCTURE ONLY.
 *
 * Readings (G1-G4):
 *   G1 V0 is a caller-chosen root (the paper draws it at random).
 *   G2 literal Alg. 3: stack (LIFO), U = pop, d = 360/deg(U) with the FULL
 *      degree (already visited neighbours leave angular gaps), neighbours in
 *      CSR order, D advances only for newly placed ones; V_u = U +
 *      (cos(PI*D/180), sin(PI*D/180)) with the paper's constant PI = 3.1416
 *      (P:806); fp64 coordinates, rounded to fp32 on output.
 *   G3 Alg. 3 covers only V0's component; every other component restarts
 *      from its smallest vertex id at an origin on a square grid: component k
 *      (k = 0: V0's, then by smallest id) at ((k mod g) s, (k div g) s),
 *      g = ceil(sqrt(#components)), s = 2 ceil(sqrt(largest component size))
 *      (SPEC.md's choice).
 *   G4 a vertex of degree 0 places nothing (no division by zero).
 */
#define BL_PAPER_PI 3.1416

/* Components in the G3 order: comp[v] = component rank; returns the count and
 * writes the largest size.  Iterative DFS (stack of size n). */
static int32_t init_components(int32_t n, const int32_t *rowptr, const int32_t *colidx,
                               int32_t root, int32_t *comp, int32_t *stack, int32_t *largest) {
  for (int32_t v = 0; v < n; ++v) comp[v] = -1;
  int32_t ncomp = 0, big = 0;
  for (int32_t s = -1; s < n; ++s) {
    const int32_t start = s < 0 ? root : s;
    if (comp[start] >= 0) continue;
    int32_t top = 0, size = 0;
    stack[top++] = start;
    comp[start] = ncomp;
    while (top > 0) {
      const int32_t u = stack[--top];
      ++size;
      for (int32_t k = rowptr[u]; k < rowptr[u + 1]; ++k)
        if (comp[colidx[k]] < 0) {
          comp[colidx[k]] = ncomp;
          stack[top++] = colidx[k];
        }
    }
    if (size > big) big = size;
    ++ncomp;
  }
  *largest = big;
  return ncomp;
}

int oracle_greedy_init(int32_t n, const int32_t *rowptr, const int32_t *colidx, int32_t root,
                       float *xy_out) {
  if (n < 1 || root < 0 || root >= n) return -1;
  int32_t *comp = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
  int32_t *stack = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
  unsigned char *visited = (unsigned char *)calloc((size_t)n, 1);
  double *V = (double *)malloc(sizeof(double) * 2 * (size_t)n);
  if (!comp || !stack || !visited || !V) {
    free(comp);
    free(stack);
    free(visited);
    free(V);
    return -1;
  }
  int32_t largest = 0;
  const int32_t ncomp = init_components(n, rowptr, colidx, root, comp, stack, &largest);
  int32_t g = 1;
  while ((int64_t)g * g < ncomp) ++g;
  int32_t sq = 1;
  while ((int64_t)sq * sq < largest) ++sq;
  const double spacing = 2.0 * sq;
  for (int32_t s = -1; s < n; ++s) {
    const int32_t v0 = s < 0 ? root : s;
    if (visited[v0]) continue;
    const int32_t k = comp[v0];
    /* Alg. 3 lines 1-5 (origin per G3) */
    int32_t top = 0;
    V[2 * v0] = (double)(k % g) * spacing;
    V[2 * v0 + 1] = (double)(k / g) * spacing;
    stack[top++] = v0;
    visited[v0] = 1;
    while (top > 0) { /* lines 6-17 */
      const int32_t U = stack[--top];
      const int32_t deg = rowptr[U + 1] - rowptr[U];
      if (deg == 0) continue; /* G4 */
      const double d = 360.0 / (double)deg;
      double D = 0.0;
      for (int32_t e = rowptr[U]; e < rowptr[U + 1]; ++e) {
        const int32_t u = colidx[e];
        if (!visited[u]) {
          V[2 * u] = V[2 * U] + cos(BL_PAPER_PI * D / 180.0);
          V[2 * u + 1] = V[2 * U + 1] + sin(BL_PAPER_PI * D / 180.0);
          visited[u] = 1;
          stack[top++] = u;
          D = D + d;
        }
      }
    }
  }
  for (int64_t i = 0; i < 2 * (int64_t)n; ++i) xy_out[i] = (float)V[i];
  free(comp);
  free(stack);
  free(visited);
  free(V);
  return 0;
}
