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
