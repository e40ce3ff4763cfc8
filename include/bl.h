/*
 * bl.h -- C-ABI of libbl, the B200 (sm_100a) BatchLayout exact-path library.
 *
 * Method: "BatchLayout" (Rahman, Sujon & Azad, arXiv:2002.08233), the exact
 * minibatch force-directed layout of Alg. 2 with the
 * spring-electrical (2,-1) force model of §2.2.  Citations
 * "P:n" are lines of the paper's text; readings of points the
 * paper leaves open are C1-C13 in DESIGN.md §3.
 *
 * All functions are extern "C"; no C++ exception crosses this boundary.
 * The library links the CUDA runtime only (no torch); callers may hand in
 * device pointers and a cudaStream_t obtained from any framework.
 *
 * Status codes: every call returns a bl_status; on failure
 * bl_last_error(h) holds a one-line message for calls that took a handle.
 */
#ifndef BL_H_
#define BL_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bl_ctx bl_ctx; /* opaque; owns the device CSR and all scratch */

typedef enum {
  BL_OK = 0,
  BL_EINVAL = -1, /* invalid argument (CSR, params, pointers, sizes)      */
  BL_ENOMEM = -2, /* host or device allocation failed                      */
  BL_ECUDA = -3,  /* a CUDA call or the cooperative launch failed          */
  BL_ESTATE = -4  /* call order: e.g. bl_energy before any layout          */
} bl_status;

/* flags */
enum {
  /* Reading C2: by default adjacent pairs ATTRACT ONLY, as in the if/else of
   * Alg. 1 / Alg. 2 and the (i,j) not-in-E second
   * sum of §2.2.  With this flag adjacent pairs also repel (the
   * classic Fruchterman-Reingold form, and the BH variant Alg. S3). */
  BL_REPULSE_NEIGHBORS = 1u << 0,
  /* bl_forces only (measurement / parity of step a5 alone): return the CSR
   * attraction + neighbour correction S_i = sum over j in N(i) of
   * (d^(a-1)/K + C K^2 d^(r-1)) Δ_ij (without the correction under
   * BL_REPULSE_NEIGHBORS), i.e. f(i, c) without the all-pairs repulsion term
   * -C K^2 R_i.  Rejected (BL_EINVAL) by bl_layout / bl_layout_device and
   * with BL_ALGO_BH. */
  BL_ATTRACTION_ONLY = 1u << 1
};

/* repulsion algorithm (bl_params.algo) */
enum {
  BL_ALGO_EXACT = 0, /* exact all-pairs repulsion: BatchLayout, Alg. 2          */
  BL_ALGO_BH = 1     /* Barnes-Hut quadtree repulsion: BatchLayoutBH, Alg. S1-S3
                        (§3.5).  Per Alg. S3 adjacent pairs attract
                        AND repel (BL_REPULSE_NEIGHBORS is implied; flags are ignored).
                        The tree is rebuilt from the coordinates at every iteration start;
                        readings B1-B9 in DESIGN.md §3.                                   */
};

typedef struct {
  int32_t iters;       /* >= 0; MaxIteration of Alg. 2. 0 = no-op      */
  int32_t batch;       /* >= 1; BS of Alg. 2. > n is clamped to n  */
  float K;             /* > 0; optimal spring length of §2.2. Unstated
                          in the paper (reading C6); default 1                  */
  float C;             /* >= 0; the paper's R, relative strength;
                          default 1 (reading C6)                               */
  double step0;        /* > 0; initial Step, Alg. 2 P:700 (1.0)                */
  double cooling;      /* (0, 1]; Step *= cooling per iteration, P:730 (0.999).
                          The schedule is kept in fp64 (step_t = step0·γ^t by
                          repeated multiplication), cast to fp32 per use      */
  double tol;          /* >= 0; stop when |E_t - E_{t-1}| < tol (P:1082,
                          §4.5).  0 disables.                                  */
  int32_t max_batches; /* > 0: stop after that many batch updates in total
                          (debug / one-batch parity); <= 0: no limit           */
  uint32_t flags;      /* BL_REPULSE_NEIGHBORS; BL_ATTRACTION_ONLY (bl_forces)   */
  int32_t algo;        /* BL_ALGO_EXACT (default) or BL_ALGO_BH                */
  float theta;         /* BL_ALGO_BH: MAC threshold, accept a cell when
                          theta > D_cell / d; >= 0, 0 = exact; the
                          paper's value 1.2 is the default             */
  float a;             /* (a, r)-energy model (§2.2, reading C15): the
                          attractive force is d^a / K, a in [0, 4]; 2 = the
                          paper's model, 1 = ForceAtlas2, 0 = LinLog  */
  float r;             /* the repulsive force magnitude is C K^2 d^r, r in
                          [-3, 1); -1 = the paper's (Fruchterman-Reingold).
                          r != -1 costs two SFU ops per pair instead of one    */
  uint64_t shuffle_seed; /* batch randomisation (§4.3.3, Fig. S3;
                          readings R1-R2 in DESIGN.md §3): 0 = the paper's
                          default sequential batches; otherwise iteration it
                          walks the batches of a fresh seeded permutation
                          pi_it of the vertex ids (batch t = pi_it(t b ..)),
                          a keyed Feistel bijection any implementation can
                          evaluate.  BL_ALGO_EXACT only (BL_EINVAL with BH).
                          Each iteration is relabelled into position space
                          (one extra launch) and runs on the sequential
                          drivers (tol > 0 is tested on the device between
                          the launches); where those do not apply the
                          two-barrier driver randomises in the kernel
                                                              */
} bl_params;

/* Fill p with the paper's defaults: iters 600 (the CLI default),
 * batch 256, K = 1, C = 1, step0 = 1.0, cooling = 0.999, tol = 0,
 * max_batches = 0, flags = 0, algo = BL_ALGO_EXACT, theta = 1.2,
 * a = 2, r = -1, shuffle_seed = 0 (sequential batches). */
void bl_params_default(bl_params *p);

/* Create a context on the current CUDA device for the undirected graph G
 * given in CSR: rowptr int32[n+1], colidx int32[rowptr[n]],
 * host memory, owned by the caller (copied; may be freed on return).
 * Validation (-> BL_EINVAL): n >= 1, rowptr[0] = 0, rowptr nondecreasing,
 * rowptr[n] = nnz, colidx in [0, n), no self loops, rows strictly
 * ascending, symmetric (undirected graphs only).  Also n must fit the
 * resident-coordinate design (n <= bl_max_vertices()).
 * *out receives the handle on success, NULL otherwise. */
bl_status bl_create(int32_t n, const int32_t *rowptr, const int32_t *colidx, bl_ctx **out);

/* Run the layout on HOST coordinates xy (2n floats x0,y0,x1,y1,..., the
 * initial layout c of Alg. 2 on entry, the final layout on success; left
 * untouched on failure).  Synchronous: copies xy host->device, runs, copies
 * back, and records the energy trace.  *iters_done (nullable) receives the
 * number of completed iterations. */
bl_status bl_layout(bl_ctx *h, float *xy, const bl_params *p, int32_t *iters_done);

/* Same on DEVICE coordinates d_xy (float2[n], 8-byte aligned, in/out),
 * enqueued on cuda_stream (a cudaStream_t; NULL = legacy default stream).
 * Asynchronous: returns after the launch; the energy trace and iteration
 * count are complete when the stream is.  One persistent cooperative kernel
 * walks all iters x ceil(n/batch) dependent batches. */
bl_status bl_layout_device(bl_ctx *h, float *d_xy, const bl_params *p, void *cuda_stream);

/* Energy (sum_i ||f_i||^2, §2.2; accumulated per batch at each
 * batch's own time, reset per iteration, Alg. 2 P:703/P:727 -- reading C8)
 * of the last layout call on h.  Synchronises h's last stream.
 * e_last (nullable): energy of the last completed iteration.
 * trace (nullable): up to trace_len per-iteration fp64 energies.
 * n_written (nullable): entries written to trace.
 * iters_done (nullable): completed iterations of the last call.
 * BL_ESTATE if no layout call has completed an iteration. */
bl_status bl_energy(bl_ctx *h, double *e_last, double *trace, int32_t trace_len,
                    int32_t *n_written, int32_t *iters_done);

/* Greedy initial layout, Alg. 3 (§3.6): host-only (needs
 * no GPU and no context), O(n + m).  rowptr/colidx: CSR of G as for
 * bl_create (only ranges are validated here); root: the start vertex V0
 * (the paper picks it at random), placed at (0, 0); xy_out: 2n floats
 * (caller-owned).  Components other than V0's restart from their smallest
 * vertex id at origins on a square grid (reading G3).
 * BL_EINVAL on bad arguments. */
bl_status bl_greedy_init(int32_t n, const int32_t *rowptr, const int32_t *colidx, int32_t root,
                         float *xy_out);

/* Debug / parity: the raw combined forces f(i, c) of §2.2 for
 * i in [first, first+count) at the device state d_xy (not modified), written
 * to d_f_out (float2[count], device).  Uses the same device code as the
 * layout kernel.  Only p->K, p->C, p->flags, p->algo and p->theta are read
 * (BL_ALGO_BH: the tree is built from d_xy itself). */
bl_status bl_forces(bl_ctx *h, const float *d_xy, int32_t first, int32_t count, float *d_f_out,
                    const bl_params *p, void *cuda_stream);

/* BL_ALGO_BH: number of quadtree nodes the last bl_layout_device /
 * bl_layout / bl_forces call visited in Alg. S2 traversals (summed over all
 * queries; leaves and accepted or opened cells each count once).  Layout
 * calls walk the tree for every vertex at the start of each iteration (the
 * walk depends only on the iteration-start tree and the vertex's own,
 * not yet moved, position -- reading B5), so an iteration stopped early by
 * max_batches still counts all n walks.  Synchronises h's last stream.
 * *visits = 0 after an exact-algorithm call. */
bl_status bl_last_visits(bl_ctx *h, unsigned long long *visits);

/* ---- layout quality metrics, §3.7; readings M1-M4 in DESIGN.md §3.
 * All take the device layout d_xy (float2[n] of h's graph), run on cuda_stream
 * and return synchronously; results are bitwise reproducible. */

/* Edge uniformity: sqrt(sum_e (l_e - l_mu)^2 / (|E| l_mu^2)), each
 * undirected edge once; 0 for a graph without edges. */
bl_status bl_edge_uniformity(bl_ctx *h, const float *d_xy, double *eu, void *cuda_stream);

/* Scale-optimised stress: sum over ORDERED pairs (i, j), i in the
 * source set, j != i reachable, of (s ||c_i - c_j|| - d_ij)^2 / d_ij^2 with
 * d_ij = BFS hop distance and s = s* minimising it (closed form).  With all
 * n sources every unordered pair {i, j} is therefore counted twice: stress,
 * pairs and unreachable are 2x the unordered-pair (i < j) values SPEC.md's
 * program reports; s* is the same (reading M1 of DESIGN.md §3: a source
 * subset has no i < j form, so the ordered sum is the one definition that
 * covers both).  sources:
 * host int32[nsrc] (NULL = all n vertices, nsrc ignored); scale (nullable) <-
 * s*; pairs (nullable) <- reachable pairs; unreachable (nullable) <- pairs
 * excluded because j is not reachable from i.  BL_EINVAL on a bad source. */
bl_status bl_stress(bl_ctx *h, const float *d_xy, const int32_t *sources, int32_t nsrc,
                    double *stress, double *scale, long long *pairs, long long *unreachable,
                    void *cuda_stream);

/* Neighbourhood preservation (reading M3): mean over the query
 * vertices i with deg(i) = k > 0 of the Jaccard similarity between N(i) and
 * the k layout-nearest other vertices (fp32 squared distances, ties by vertex
 * id).  queries: host int32[nq] (NULL = all vertices); counted (nullable) <-
 * the number of queries with k > 0. */
bl_status bl_neighborhood_preservation(bl_ctx *h, const float *d_xy, const int32_t *queries,
                                       int32_t nq, double *np, int32_t *counted,
                                       void *cuda_stream);

/* Largest n the resident design accepts on the current device. */
int32_t bl_max_vertices(void);

/* Number of kernel launches the last bl_layout_device / bl_layout /
 * bl_forces call enqueued (the persistent design launches exactly one). */
int32_t bl_last_launch_count(const bl_ctx *h);

/* Name of the kernel the last layout call on h launched -- the whole-GPU
 * "bl_layout_kernel<NT,T,TP>" (NT threads per CTA, T register-blocked targets
 * per thread, TP of them with paired reciprocals), the single-cluster
 * "bl_cluster_kernel<T,TP> xCS" used for small graphs, or "bl_bh_kernel<512>"
 * -- or, before any call, the whole-GPU variant.  Static
 * storage owned by h. */
const char *bl_kernel_name(const bl_ctx *h);

/* How the last layout call on h sequenced its dependent batches (DESIGN.md
 * §4): "async" (one grid barrier per batch, no CTA-wide barrier between
 * phases; b n >= 2^22), "pipelined" (one grid barrier per batch), "two-barrier"
 * (phase R; barrier; phase U; barrier), "cluster" (single thread-block cluster)
 * or "bh" (BatchLayoutBH); "" before any call.  Static storage owned by h. */
const char *bl_driver_name(const bl_ctx *h);

/* Microbenchmark of the roofline denominators on the current device:
 * sustained thread-op rates per SM per clock of (0) 3-register FFMA,
 * (1) MUFU.RCP (rcp.approx.ftz.f32), (2) MUFU.RSQ, (3) packed FFMA2
 * (fma.rn.f32x2, 2 ops per lane), measured with clock64 inside one kernel on
 * every SM.  rates[4] receives ops/clk/SM.  Blocking. */
bl_status bl_microbench(double rates[4]);

/* Debug aid: when the context was created with the environment variable
 * BL_PROFILE=1, the persistent kernel records per-phase SM-cycle sums of
 * CTA 0 (out[0..7]: attraction, repulsion sweep, in-CTA combine, barrier 1,
 * update, barrier 2, -, tail) and per-CTA busy cycles of phase R (out[8+c]).
 * Copies up to len values; returns how many (0 if profiling is off). */
int32_t bl_debug_profile(bl_ctx *h, unsigned long long *out, int32_t len);

/* Debug aid for the CHECKED build of the library (libbl_checked.so, built
 * with -DBL_CHECKED): every cross-CTA value of the exact
 * whole-GPU kernel carries the batch it comes from, and readers check it
 * (Alg. 2's frozen-batch semantics), plus bounds and protocol
 * invariants; BL_JITTER=<seed> adds seeded random sleeps at task boundaries.
 * Copies the violation record of the last launch on h into out[8]: out[0] =
 * violations, out[1] = first code, out[2..4] = its details.  Synchronises h's
 * last stream.  Returns 1 (checked build), 0 (production build: nothing is
 * recorded, out zeroed) or -1 (NULL argument / CUDA error). */
int32_t bl_debug_check(bl_ctx *h, uint32_t *out);

/* Measurement aid: out[0] = BFS levels summed over the 64-source groups and
 * out[1] = CSR entries examined (each level pulls the rows of the
 * not-yet-complete vertices) by the last bl_stress call on h; out[2] = GPU
 * time in ns of the kernels of the last metric call (bl_edge_uniformity,
 * bl_stress or bl_neighborhood_preservation; CUDA events on its stream, no
 * host synchronisation included); out[3] = 0.  Returns 4, or -1 on a NULL
 * argument. */
int32_t bl_debug_counters(const bl_ctx *h, int64_t *out);

void bl_destroy(bl_ctx *h);
const char *bl_status_string(bl_status s);
const char *bl_last_error(const bl_ctx *h);

#ifdef __cplusplus
}
#endif
#endif /* BL_H_ */
