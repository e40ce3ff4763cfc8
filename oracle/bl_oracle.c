/*
 * bl_oracle.c -- plain, slow, obviously-correct CPU oracle for the
 * BatchLayout exact path (Rahman, Sujon & Azad, arXiv:2002.08233).
 *
 * TEST INFRASTRUCTURE.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product
 * path (paper_2002_08233_b200/, libbl.so) never calls it and shares no code,
 * header, table or helper with it.
 *
 * What it computes: Alg. 2 of the paper with the force model of
 * §2.2, step by step in the paper's order, per pair if/else as
 * written (attract if (i,j) in E, else repel), fp64, no FMA contraction
 * (built with -O2 -ffp-contract=off, no fast-math).  The optional OpenMP
 * parallel-for over the vertices of a batch is Alg. 2's ParFor; each
 * per-vertex sum keeps the same j order, so the result is bitwise identical
 * for any thread count (the property the paper states at P:1102-1103).
 *
 * Readings of silent/garbled points are listed in DESIGN.md §3 (C1-C13 of
 * SURVEY.md §8(c)).  Pins: tests/test_oracle_*.py.  Parity of long
 * trajectories' absolute energies is unpinned (chaotic dynamics, DESIGN.md
 * §3 "parity unpinned").
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* (a, r)-energy model exponents (§2.2, reading C15 of
 * DESIGN.md §3): attraction magnitude d^a / K, repulsion magnitude C K^2 d^r
 * (Noack / ForceAtlas2 convention: (2,-1) = Fruchterman-Reingold).
 * Process-global, set by the Python face around each call. */
static double g_model_a = 2.0, g_model_r = -1.0;
void oracle_set_model(double a, double r) {
  g_model_a = a;
  g_model_r = r;
}

/* Batch randomisation (§4.3.3, Fig. S3; readings R1-R2
 * of DESIGN.md §3).  The paper reshuffles which vertices form each minibatch
 * ("randomization of batches which is a common practice in machine
 * learning") but fixes no generator.  R1: every iteration `it` draws
 * a fresh permutation pi_it of the vertex ids and batch t holds
 * pi_it(t b), ..., pi_it(min((t+1) b, n) - 1); seed 0 = no shuffle (the
 * paper's default sequential batches).  R2: pi_it is a counter-based keyed
 * bijection -- a 4-round Feistel network on [0, 2^M) (M the smallest even
 * bit count >= 2 with 2^M >= n) restricted to [0, n) by cycle walking, round
 * keys and round function from splitmix64 -- so that any implementation can
 * evaluate pi_it(x) for one x with integer arithmetic only. */
static uint64_t oracle_splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
uint64_t oracle_mix64(uint64_t z) { return oracle_splitmix64(z); }

static int32_t oracle_perm(uint64_t seed, int32_t it, int32_t n, int32_t x) {
  if (seed == 0) return x;
  int M = 2;
  while (((int64_t)1 << M) < (int64_t)n) M += 2;
  const int h = M / 2;
  const uint64_t mask = ((uint64_t)1 << h) - 1;
  uint64_t key[4];
  for (int r = 0; r < 4; ++r)
    key[r] = oracle_splitmix64(seed ^ oracle_splitmix64((uint64_t)it * 4u + (uint64_t)r));
  uint64_t y = (uint64_t)x;
  do { /* cycle walking: repeat the Feistel bijection until inside [0, n) */
    uint64_t L = y >> h, R = y & mask;
    for (int r = 0; r < 4; ++r) {
      const uint64_t F = oracle_splitmix64(key[r] ^ R) >> (64 - h);
      const uint64_t t = L ^ F;
      L = R;
      R = t;
    }
    y = (L << h) | R;
  } while (y >= (uint64_t)n);
  return (int32_t)y;
}

/* pi_it(0..n-1) into out (for the tests' brute force and pins) */
int oracle_permutation(int32_t n, uint64_t seed, int32_t it, int32_t *out) {
  if (n < 1 || it < 0) return -1;
  for (int32_t x = 0; x < n; ++x) out[x] = oracle_perm(seed, it, n, x);
  return 0;
}

#define REAL double
#define SFX(name) name##_f64
#define SQRT sqrt
#define POW pow
#include "bl_oracle_impl.h"
#undef REAL
#undef SFX
#undef SQRT
#undef POW

#define REAL float
#define SFX(name) name##_f32
#define SQRT sqrtf
#define POW powf
#include "bl_oracle_impl.h"
#undef REAL
#undef SFX
#undef SQRT
#undef POW

/* BatchLayoutBH (Alg. S1-S3), fp64 force terms, fp32 decisions */
#include "bl_oracle_bh.h"

/* Greedy initialisation (Alg. 3) */
#include "bl_oracle_init.h"

/* Quality metrics (§3.7) */
#include "bl_oracle_metrics.h"

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
