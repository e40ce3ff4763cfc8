/*
 * bl_oracle_impl.h -- body of the BatchLayout oracle, instantiated twice by
 * bl_oracle.c: once with REAL = double (the oracle proper) and once with
 * REAL = float (used only to measure the fp32 "chaos floor" of SURVEY.md
 * §8(c) (ii)).  TEST INFRASTRUCTURE ONLY -- see bl_oracle.c for the header.
 *
 * Requires: REAL, SFX(name), SQRT defined by the includer.
 */

/* f_a(i,j) = ||c_i - c_j||^a / K  (§2.2); a = 2 is the
 * paper's evaluated model (2,-1); other a: the (a,r)-energy model
 * family, exponent set by oracle_set_model (reading C15). */
static REAL SFX(f_attr)(REAL d, REAL K) {
  if (g_model_a == 2.0) return (d * d) / K;
  return POW(d, (REAL)g_model_a) / K;
}

/* f_r(i,j) = -R K^2 / ||c_i - c_j|| (§2.2, under the
 * reading C1 of DESIGN.md: the (2,-1) model's repulsive force magnitude is
 * R K^2 / d, i.e. the Fruchterman-Reingold repulsion P:872).  R is called
 * C here (Hu's notation). */
static REAL SFX(f_rep)(REAL d, REAL K, REAL C) {
  if (g_model_r == -1.0) return -(C * K * K) / d;
  return -(C * K * K) * POW(d, (REAL)g_model_r); /* magnitude C K^2 d^r (C15) */
}

/* Force of vertex i against the frozen coordinates c, exactly as the inner
 * loops of Alg. 1 / Alg. 2: for every j != i, if
 * (i,j) in E add f_a * (c_j - c_i)/||c_i - c_j||, else add
 * f_r * (c_j - c_i)/||c_i - c_j||.  j runs in ascending order.
 * `mark` is an n-byte scratch array, all zero on entry and on exit.
 * Reading C3: j = i is skipped (the sum of §2.2 is over i != j).
 * Reading C4: a coincident pair (d = 0) contributes nothing.
 * flags & 1 (REPULSE_NEIGHBORS, reading C2): adjacent pairs also repel. */
static void SFX(force_of)(int32_t n, const int32_t *rowptr, const int32_t *colidx,
                          const REAL *c, int32_t i, REAL K, REAL C, uint32_t flags,
                          unsigned char *mark, REAL *fx_out, REAL *fy_out) {
  for (int32_t k = rowptr[i]; k < rowptr[i + 1]; ++k) mark[colidx[k]] = 1;
  REAL fx = 0, fy = 0;
  const REAL xi = c[2 * i], yi = c[2 * i + 1];
  for (int32_t j = 0; j < n; ++j) {
    if (j == i) continue;
    const REAL dx = c[2 * j] - xi;       /* c_j - c_i */
    const REAL dy = c[2 * j + 1] - yi;
    const REAL d = SQRT(dx * dx + dy * dy); /* ||c_i - c_j|| */
    if (d == 0) continue;
    const REAL ux = dx / d, uy = dy / d;    /* unit vector towards j */
    if (mark[j]) {
      const REAL fa = SFX(f_attr)(d, K);
      fx = fx + fa * ux;
      fy = fy + fa * uy;
      if (flags & 1u) {
        const REAL fr = SFX(f_rep)(d, K, C);
        fx = fx + fr * ux;
        fy = fy + fr * uy;
      }
    } else {
      const REAL fr = SFX(f_rep)(d, K, C);
      fx = fx + fr * ux;
      fy = fy + fr * uy;
    }
  }
  for (int32_t k = rowptr[i]; k < rowptr[i + 1]; ++k) mark[colidx[k]] = 0;
  *fx_out = fx;
  *fy_out = fy;
}

/* c_i = c_i + Step * f / ||f|| (Alg. 1 line 12; Alg. 2).
 * Reading C5: no move when ||f|| = 0.  Returns ||f||^2 (the energy term,
 * P:560 / P:727). */
static REAL SFX(apply_update)(REAL *ci, REAL fx, REAL fy, REAL step) {
  const REAL q = fx * fx + fy * fy;
  if (q > 0) {
    const REAL nrm = SQRT(q);
    ci[0] = ci[0] + step * (fx / nrm);
    ci[1] = ci[1] + step * (fy / nrm);
  }
  return q;
}

int SFX(oracle_apply_update)(REAL *ci, REAL fx, REAL fy, REAL step, REAL *q_out) {
  REAL q = SFX(apply_update)(ci, fx, fy, step);
  if (q_out) *q_out = q;
  return 0;
}

/* Raw forces f(i, c) for i in [first, first+count) at the given state, no
 * update (the §2.2 combined force).  Used by the parity tests. */
int SFX(oracle_forces)(int32_t n, const int32_t *rowptr, const int32_t *colidx,
                       const REAL *c, int32_t first, int32_t count, REAL K, REAL C,
                       uint32_t flags, REAL *f_out, int threads) {
  if (n < 1 || first < 0 || count < 0 || first + count > n) return -1;
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel
#endif
  {
    unsigned char *mark = (unsigned char *)calloc((size_t)n, 1);
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
    for (int32_t t = 0; t < count; ++t) {
      REAL fx, fy;
      SFX(force_of)(n, rowptr, colidx, c, first + t, K, C, flags, mark, &fx, &fy);
      f_out[2 * t] = fx;
      f_out[2 * t + 1] = fy;
    }
    free(mark);
  }
  (void)threads;
  return 0;
}

/* Alg. 2 (Cache Blocking BatchLayout) without its blocking (the
 * blocking is a performance device that does not change the result):
 *
 *   Step = step0; for Loop < iters:
 *     Energy = 0
 *     for each minibatch [lo, hi) of consecutive ids       (ragged
 *                                                          tail P:690-691)
 *       ParFor i in batch: ct_i = f(i, c)   (c frozen)     (P:705-721,
 *                                                          P:626-627)
 *       for i in batch: c_i += Step ct_i/||ct_i||; Energy += ||ct_i||^2
 *
 *     Step = Step * cooling
 *
 * xy: in/out, 2n values.  energy: iters values (nullable).  max_batches > 0
 * stops after that many batch updates in total (the partial iteration's
 * energy so far is written to energy[it]).  batch > n is clamped to n.
 * tol > 0: stop after the first iteration t >= 1 with |E_t - E_{t-1}| < tol
 * (the convergence criterion of §4.5).
 * shuffle_seed != 0: batch randomisation (§4.3.3, readings R1-R2 in
 * bl_oracle.c): batch t of iteration it is pi_it(t b .. ); 0 = sequential.
 * Returns 0, or -1 on invalid arguments. */
int SFX(oracle_layout)(int32_t n, const int32_t *rowptr, const int32_t *colidx,
                       REAL *xy, int32_t iters, int32_t batch, REAL K, REAL C,
                       double step0, double cooling, int32_t max_batches,
                       double tol, uint32_t flags, double *energy,
                       int32_t *iters_done, int threads, uint64_t shuffle_seed) {
  if (n < 1 || iters < 0 || batch < 1) return -1;
  if (batch > n) batch = n;
  REAL *ct = (REAL *)malloc(sizeof(REAL) * 2 * (size_t)batch);
  int32_t *vid = (int32_t *)malloc(sizeof(int32_t) * (size_t)batch);
  if (!ct || !vid) {
    free(ct);
    free(vid);
    return -1;
  }
  double step = step0;
  int32_t batches_done = 0;
  int32_t it_done = 0;
  int stop = 0;
  double E_prev = 0;
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#endif
  for (int32_t it = 0; it < iters && !stop; ++it) {
    REAL E = 0;
    const REAL stepr = (REAL)step;
    for (int32_t lo = 0; lo < n; lo += batch) {
      const int32_t hi = (lo + batch < n) ? lo + batch : n;
      /* the batch's vertices: lo..hi-1, or pi_it(lo..hi-1) with batch
       * randomisation (readings R1-R2; pi = identity for seed 0) */
      for (int32_t k = lo; k < hi; ++k) vid[k - lo] = oracle_perm(shuffle_seed, it, n, k);
      /* forces of the whole batch against frozen coordinates */
#ifdef _OPENMP
#pragma omp parallel
#endif
      {
        unsigned char *mark = (unsigned char *)calloc((size_t)n, 1);
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
        for (int32_t k = lo; k < hi; ++k) {
          SFX(force_of)(n, rowptr, colidx, xy, vid[k - lo], K, C, flags, mark,
                        &ct[2 * (k - lo)], &ct[2 * (k - lo) + 1]);
        }
        free(mark);
      }
      /* then the batch update, in order */
      for (int32_t k = lo; k < hi; ++k) {
        E = E + SFX(apply_update)(&xy[2 * vid[k - lo]], ct[2 * (k - lo)], ct[2 * (k - lo) + 1],
                                  stepr);
      }
      ++batches_done;
      if (max_batches > 0 && batches_done >= max_batches) {
        stop = 1;
        if (energy) energy[it] = (double)E;
        break;
      }
    }
    if (!stop) {
      if (energy) energy[it] = (double)E;
      ++it_done;
      step = step * cooling;
      if (tol > 0 && it > 0 && fabs((double)E - E_prev) < tol) break;
      E_prev = (double)E;
    }
  }
  free(ct);
  free(vid);
  if (iters_done) *iters_done = it_done;
  (void)threads;
  return 0;
}
