// bl_kernel.cuh -- the persistent sm_100a BatchLayout kernel (device side).
//
// One cooperative launch walks every dependent minibatch of every iteration
// of Alg. 2.  Per batch t = [lo, hi):
//
//   phase R  (all CTAs)  -- a4 + a5 of SURVEY.md §8(a)
//     * attraction items: edge-parallel over the batch's contiguous CSR slice
//       [rowptr[lo], rowptr[hi]) in items of <= BL_ECH entries, each gathering
//       xy[colidx[k]] through L2 and summing (d/K)·Δ + C K^2·Δ/d^2 (the
//       spring term f_a·û of §2.2 with f_a = d^2/K, plus the removal of that
//       neighbour's repulsion, so adjacent pairs attract only: the if/else of
//       Alg. 2, reading C2).
//     * all-pairs repulsion: CTA c holds its owned sources {v : v ≡ c mod G}
//       resident in shared memory for the whole call; every warp sweeps a
//       sub-range of them against 32·T register-blocked batch targets,
//       R_i += Δ_ij / d_ij^2 (branch-free: d^2 = Δx^2 + Δy^2 + 2^-63 makes the
//       self pair and coincident pairs contribute exactly 0, reading C3/C4;
//       1/d^2 on the SFU via rcp.approx.ftz).  Per-CTA partials go to
//       part[target][c] after a fixed-order in-CTA combine.
//   grid barrier
//   phase U  (owner CTA of each target)  -- a6 + a7
//     * f_i = S_i - C K^2 · Σ_c part[i][c] in fixed order; c_i += Step·f/||f||
//       (no move if f = 0, reading C5); xy in HBM and the owner's
//       shared copy are updated; ||f||^2 accumulates in fp64 per warp.
//   grid barrier
//
// Coordinates are frozen within a batch because nobody writes xy
// during phase R; the next batch sees the update (Fig. 2 caption P:644)
// because phase U precedes the next barrier.  Every sum has a fixed order,
// so runs are bitwise reproducible.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

// threads per CTA: a template parameter of the kernel (NT, launch bounds);
// device code reads it as blockDim.x.  BL_NT / BL_NW: the runtime values.
#define BL_NT ((int)blockDim.x)
#define BL_NW ((int)(blockDim.x >> 5))
#define BL_NW_MAX 32
#define BL_ECH 128         // CSR entries per attraction item
// self/coincident-pair guard folded into d^2: 2^-63, so that
// eps2*eps2 = 2^-126 is still a normal float and the paired reciprocal
// 1/(d2a d2b) stays finite even when both pairs are coincident
#define BL_EPS2 1.0842021724855044e-19f
#define BL_TGT_CAP 2048       // batch targets staged in shared memory (else read from L2)
#define BL_RED_MAX 16384      // max float2 slots for per-(sub-range, target) repulsion partials
#define BL_RED_MIN 4096       // min (the host sizes red from the shared memory left)
#define BL_MIN_UNIT4 16       // minimum float4 (2 sources) per repulsion sub-range
#define BL_NSUB_MAX 32

// Partition of one batch's repulsion work inside a CTA: ntt target tiles of
// 32·T targets x nsub sub-ranges of the CTA's resident sources.  The clean
// sources are cut into nc sub-ranges of decreasing size ("guided", so that
// warps that start late -- update warps -- balance out on small units), and
// the sources this CTA is updating in the same phase (dirty) form the last
// sub-range.
struct BLUnits {
  int ntt, nc, nsub;
};
// Precondition with a dirty range: red_cap holds >= 2 sub-ranges of every
// tile (the host's driver eligibility checks; tests/cpp/test_units.cu).
__host__ __device__ inline BLUnits bl_units(int bt, int T, int clean4, bool dirty, int red_cap,
                                            int nsub_max = BL_NSUB_MAX,
                                            int min_unit4 = BL_MIN_UNIT4) {
  BLUnits u;
  u.ntt = (bt + 32 * T - 1) / (32 * T);
  int cap = red_cap / (u.ntt * 32 * T);
  if (cap > nsub_max) cap = nsub_max;
  int nc = clean4 / (min_unit4 > 0 ? min_unit4 : 1);
  if (nc > cap - (dirty ? 1 : 0)) nc = cap - (dirty ? 1 : 0);
  u.nc = nc < 1 ? 1 : nc;
  u.nsub = u.nc + (dirty ? 1 : 0);
  if (cap < 1) u.nsub = u.nc = 1;  // very large batches: red unused (nsub == 1)
  return u;
}
// start (in the concatenated clean domain of length L) of clean sub-range k
// of nc.  Sizes decrease so that the units grabbed last (the tail of a
// batch, when warps run out of work) are small:
//   profile 0: equal sizes
//   profile 1: weights nc, nc-1, ..., 1        (linear)
//   profile 2: weights nc^2, (nc-1)^2, ..., 1  (quadratic; the default)
__host__ __device__ inline long long bl_sq_sum(long long m) { return m * (m + 1) * (2 * m + 1) / 6; }
__host__ __device__ inline int bl_guided_start(int k, int nc, int L, int profile) {
  long long W, cum;
  if (profile == 0) return (int)(((long long)L * k) / nc);  // uniform
  if (profile == 2) {
    W = bl_sq_sum(nc);
    cum = W - bl_sq_sum(nc - k);
  } else {
    W = (long long)nc * (nc + 1) / 2;
    cum = (long long)k * nc - (long long)k * (k - 1) / 2;
  }
  return (int)((L * cum) / W);
}
// shared memory: [src4: chunk4 float4][tgt: 2 x BL_TGT_CAP float2][red: red_cap float2]
__host__ __device__ inline size_t bl_smem_bytes(int chunk4, int red_cap) {
  return (size_t)chunk4 * 16 + (size_t)2 * BL_TGT_CAP * 8 + (size_t)red_cap * 8;
}

struct BLKParams {
  int n, b, nb, iters, max_batches;
  unsigned flags;
  float ck2, invK;
  double step0, cooling, tol;
  int chunk4;            // float4 slots (2 sources each) per CTA chunk
  int red_cap;           // float2 slots of the shared partial buffer
  int guided;            // sub-range size profile (bl_guided_start)
  int nsub_max;          // async driver: sub-ranges per target tile (incl. the dirty one)
  int min_unit4;         // pipelined / async: minimum float4 slots per clean sub-range
  unsigned spin_max;     // async driver: longest back-off sleep of a waiting warp (ns)
  // (a, r)-energy model (reading C15): attraction d^a/K, repulsion C K^2 d^r;
  // amode 0..3: a = 2, 1, 0, 3 (no pow), 4: general; rmode 0: r = -1, 1: general
  int amode, rmode;
  float a_half, r_half;  // (a-1)/2, (r-1)/2: vector coefficients d^(a-1), d^(r-1)
  int forces_mode, first, count;
  // batch randomisation (readings R1-R2): 0 = sequential; else
  // iteration it walks the batches of pi_it inside the two-barrier driver
  // (relabelled iterations, bl_relabel.cu, launch with shuf_seed = 0)
  unsigned long long shuf_seed;
  int shuf_h;            // Feistel half width: 2^(2h) >= n
  int attr_only;         // forces_mode + BL_ATTRACTION_ONLY: a5 alone (no sweep, R = 0)
  float2 *xy;
  const int *rowptr, *colidx;
  const int *item_ptr, *item_v, *item_k0;
  float2 *part;          // [2][b][G] (pipelined path double-buffers by batch parity)
  float2 *pend;          // [2][b]   new coordinates of the last two batches (pipelined)
  int pipelined;         // 1: one grid barrier per batch (needs nb >= 4); 2: the same
                         // without CTA-wide barriers between phases (bl_run_async)
  int part_nbuf;         // part buffers (2: pipelined, 3: async)
  int afence_gpu;        // async: GPU-scope fences in every task (debug, BL_AFENCE=1)
  const int *stop_in;    // relabelled iterations with tol > 0: the launch is a no-op once a
                         // previous iteration's convergence test set it (bl_relabel.cu)
  int lcoop;             // latency driver: rows of > BL_LCOOP entries walked by all updater
                         // warps of the CTA together (bl_long_row_part)
  int long8;             // update tasks walk long CSR rows 256 entries per round (8 gathers
                         // in flight per lane): the async driver always; the others when
                         // every batch holds hub rows (relabelled randomised batches)
  float2 *attr;          // [max items per batch]
  double *e_cta;         // [2][G]
  double *energy;        // [iters]
  int *iters_done;
  unsigned *bar;
  float2 *f_out;
  // checked builds (-DBL_CHECKED, libbl_checked.so): violation
  // record chk[0] = count, chk[1] = first code, chk[2..4] = its details;
  // phase stamps of every cross-CTA value (part, pend, committed xy);
  // jitter != 0 inserts seeded random sleeps at task boundaries
  unsigned *chk, *part_st, *pend_st, *xy_st;
  unsigned jitter;
  int chk_break;         // checked builds: 1 = skip the barrier wait of the control
                         // task (fault injection proving the checks are live)
  // optional phase profile (nullptr = off): [0..7] CTA-0 phase cycle sums,
  // [8 + c] CTA c's cycles from phase-R start to barrier-1 arrival
  unsigned long long *prof;
};

__device__ __forceinline__ float bl_rcp(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float bl_ex2(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float bl_lg2(float x) {
  float r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
// d^(2h) from d^2 on the SFU (two MUFU): the general (a, r)-model powers
__device__ __forceinline__ float bl_pow_d2(float d2, float h) { return bl_ex2(h * bl_lg2(d2)); }
__device__ __forceinline__ float bl_rsqrt(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
// ---- checked builds: invariant and phase-stamp checks (compiled out otherwise)
#ifdef BL_CHECKED
static __device__ __noinline__ void bl_chk_fail(const BLKParams &p, unsigned code, unsigned a, unsigned b) {
  atomicAdd(p.chk, 1u);
  if (atomicCAS(p.chk + 1, 0u, code) == 0u) {
    p.chk[2] = a;
    p.chk[3] = b;
    p.chk[4] = blockIdx.x;
  }
}
#define BL_CHK(cond, code, a, b)                                 \
  do {                                                           \
    if (!(cond)) bl_chk_fail(p, (code), (unsigned)(a), (unsigned)(b)); \
  } while (0)
#define BL_CHK_ON 1
// seeded random sleep (0..2 us, probability 1/4) at a task boundary: shakes
// the interleaving of warps and CTAs; results must stay bitwise identical
__device__ __forceinline__ void bl_jitter(const BLKParams &p, unsigned salt) {
  if (!p.jitter) return;
  unsigned long long t = clock64();
  unsigned long long z = ((unsigned long long)p.jitter << 32) ^ (t * 0x9E3779B97F4A7C15ull) ^
                         ((unsigned long long)blockIdx.x << 20) ^ (threadIdx.x >> 5) ^ salt;
  z ^= z >> 29;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 32;
  if ((z & 3ull) == 0ull) __nanosleep((unsigned)((z >> 8) & 2047ull));
}
#else
#define BL_CHK(cond, code, a, b) \
  do {                           \
  } while (0)
#define BL_CHK_ON 0
__device__ __forceinline__ void bl_jitter(const BLKParams &, unsigned) {}
#endif
// violation codes
enum {
  BLC_PART_STAMP = 1,   // an update read a partial not from its batch
  BLC_PEND_STAMP = 2,   // a neighbour coordinate from pend not from batch q-1
  BLC_XY_STAMP = 3,     // a neighbour coordinate from xy not the last committed one
  BLC_TGT_STAMP = 4,    // a staged target not the last committed coordinate
  BLC_DIRTY_EARLY = 5,  // a dirty unit started before this CTA's updates
  BLC_TOKENS = 6,       // more completion tokens than the phase needs
  BLC_BOUNDS = 7,       // index out of range (part / pend / red / src)
  BLC_PHASEU_STAMP = 8, // two-barrier phase U read a partial not from its batch
  BLC_SLOT_GEN = 9,     // async: a phase entered a slot not released for it
  BLC_LAT_TGT = 10,     // latency driver: a staged target not the committed coordinate
  BLC_LAT_CLEAN = 11    // latency driver: a clean partial not the sum over the clean sources
};

// ---- batch randomisation (§4.3.3; readings R1-R2 of DESIGN.md §3):
// pi_it is a 4-round Feistel bijection of [0, 2^(2h)) keyed from splitmix64,
// restricted to [0, n) by cycle walking -- integer arithmetic only, so any
// thread evaluates pi_it(x) for its own x, no permutation array.
__host__ __device__ __forceinline__ unsigned long long bl_mix64(unsigned long long z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
struct BLPerm {
  const unsigned long long *key;  // 4 round keys of pi_it, in shared memory
  int h, n, on;
};
// round keys of pi_it into key[4] (shared; every thread computes the same
// values, so no barrier is needed before use by the writing threads' CTA
// beyond the one at the caller)
__device__ __forceinline__ BLPerm bl_perm_make(unsigned long long seed, int h, int n, int it,
                                               unsigned long long *key) {
  BLPerm P;
  P.on = seed != 0ull;
  P.h = h;
  P.n = n;
  P.key = key;
  if (P.on && threadIdx.x < 4)
    key[threadIdx.x] =
        bl_mix64(seed ^ bl_mix64((unsigned long long)it * 4ull + (unsigned long long)threadIdx.x));
  return P;
}
__device__ __forceinline__ int bl_perm(const BLPerm &P, int x) {
  if (!P.on) return x;
  const unsigned long long mask = (1ull << P.h) - 1ull;
  unsigned long long y = (unsigned long long)x;
  do {
    unsigned long long L = y >> P.h, R = y & mask;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const unsigned long long t = L ^ (bl_mix64(P.key[r] ^ R) >> (64 - P.h));
      L = R;
      R = t;
    }
    y = (L << P.h) | R;
  } while (y >= (unsigned long long)P.n);
  return (int)y;
}

// ---- packed fp32x2 (sm_100a FADD2/FFMA2/FMUL2): two pair evaluations per
// issue slot.  Operand (a, b) lives in one 64-bit register pair.
typedef unsigned long long bl_f2;
__device__ __forceinline__ bl_f2 f2pack(float a, float b) {
  bl_f2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2unpack(bl_f2 v, float &a, float &b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ bl_f2 f2sub(bl_f2 a, bl_f2 b) {
  bl_f2 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ bl_f2 f2fma(bl_f2 a, bl_f2 b, bl_f2 c) {
  bl_f2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ bl_f2 f2mul(bl_f2 a, bl_f2 b) {
  bl_f2 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

// Shared-memory source chunk, two sources per float4 in (x_a, x_b, y_a, y_b)
// order so that one LDS.128 yields the packed X = (x_a, x_b), Y = (y_a, y_b).
__device__ __forceinline__ void bl_src_set(float4 *src4, int k, float2 v) {
  float *f = reinterpret_cast<float *>(src4 + (k >> 1));
  f[k & 1] = v.x;
  f[2 + (k & 1)] = v.y;
}
__device__ __forceinline__ float2 bl_src_get(const float4 *src4, int k) {
  const float *f = reinterpret_cast<const float *>(src4 + (k >> 1));
  return make_float2(f[k & 1], f[2 + (k & 1)]);
}

// The repulsion inner loop: for T register-blocked targets and the sources
// of src4[s0, s1): R_t += Δ / d^2.  Per (target, float4) = 2 pairs:
//   DX = X - tx, DY = Y - ty (FADD2 x2), D2 = DX^2 + DY^2 + eps (FFMA2 x2),
//   INV = 1/D2, R += (DX, DY) * INV (FFMA2 x2).
// INV: for the first TP targets the two reciprocals share ONE MUFU.RCP:
//   r = 1/(d2a d2b), INV = (d2b r, d2a r) (FMUL + MUFU + FMUL2), otherwise
//   two MUFU.RCP.  TP trades SFU work for FP32 work.
// Requires every D2 lane finite and d2a·d2b a normal float when paired: true
// for real sources (d^2 >= 2^-63 by the eps fold, so d2a d2b >= 2^-126;
// d^2 < 1.8e19); dummy (far)
// sources are only ever swept with TP = 0.
// TP < 0: the general repulsion exponent r: INV = d^(r-1) = 2^(rh lg2 d^2)
// (two MUFU per pair: the roofline halves).
// unroll of the source loop by tile width (measured same box, with a single
// call site per unit so that one copy of the loop is hot): T = 8 -> 4 (C5
// -1.6 % time vs 2), T = 16 -> 8 (C6 -3.6 %), small tiles 2
#ifndef BL_SWEEP_UNROLL
#define BL_SWEEP_UNROLL 4
#endif
template <int T, int TP, int UN = (T >= 16 ? 2 * BL_SWEEP_UNROLL : T >= 8 ? BL_SWEEP_UNROLL : 2)>
__device__ __forceinline__ void bl_sweep(const float4 *__restrict__ src4, int s0, int s1,
                                         const float (&tx)[T], const float (&ty)[T], bl_f2 (&AX)[T],
                                         bl_f2 (&AY)[T], float rh = 0.f) {
  const bl_f2 EPS = f2pack(BL_EPS2, BL_EPS2);
  bl_f2 TX[T], TY[T];
#pragma unroll
  for (int k = 0; k < T; ++k) {
    TX[k] = f2pack(tx[k], tx[k]);
    TY[k] = f2pack(ty[k], ty[k]);
  }
#pragma unroll UN
  for (int s = s0; s < s1; ++s) {
    const float4 q = src4[s];  // two sources, broadcast to the warp
    const bl_f2 X = f2pack(q.x, q.y), Y = f2pack(q.z, q.w);
#pragma unroll
    for (int k = 0; k < T; ++k) {
      const bl_f2 DX = f2sub(X, TX[k]);
      const bl_f2 DY = f2sub(Y, TY[k]);
      const bl_f2 D2 = f2fma(DX, DX, f2fma(DY, DY, EPS));
      float a, b;
      f2unpack(D2, a, b);
      bl_f2 INV;
      if (TP < 0) {
        INV = f2pack(bl_pow_d2(a, rh), bl_pow_d2(b, rh));
      } else if (k < TP) {
        const float r = bl_rcp(a * b);
        INV = f2mul(f2pack(b, a), f2pack(r, r));
      } else {
        INV = f2pack(bl_rcp(a), bl_rcp(b));
      }
      AX[k] = f2fma(DX, INV, AX[k]);
      AY[k] = f2fma(DY, INV, AY[k]);
    }
  }
}

// Coefficient of Δ for one CSR neighbour (reading C15): attraction
// f_a(d)/d = d^(a-1)/K plus, in the if/else model, the removal of the
// all-pairs repulsion rep * d^(r-1) (rep = C K^2, or 0 with
// BL_REPULSE_NEIGHBORS).  rs = 1/d.
template <bool FAST, class P>
__device__ __forceinline__ float bl_model_coef(const P &p, float d2, float rs, float rep) {
  if (FAST) return fmaf(rep * rs, rs, d2 * rs * p.invK);  // (a, r) = (2, -1)
  float at;
  switch (p.amode) {
    case 0: at = d2 * rs; break;  // a = 2 (the paper's FR model)
    case 1: at = 1.f; break;      // a = 1
    case 2: at = rs; break;       // a = 0
    case 3: at = d2; break;       // a = 3
    default: at = bl_pow_d2(d2, p.a_half);
  }
  const float rv = p.rmode == 0 ? rs * rs : bl_pow_d2(d2, p.r_half);
  return fmaf(rep, rv, at * p.invK);
}

// CTA-scope release/acquire fence for the task-queue handshakes in shared
// memory (a flag written after data / read before data): fence.acq_rel.cta,
// not the sequentially consistent MEMBAR.SC.CTA of __threadfence_block().
#ifndef BL_FENCE_ACQREL_CTA
#define BL_FENCE_ACQREL_CTA 0
#endif
#ifndef BL_EARLY_TGT
#define BL_EARLY_TGT 1
#endif
#ifndef BL_POLL_RELAXED
#define BL_POLL_RELAXED 0
#endif
__device__ __forceinline__ void bl_fence_cta() {
#if BL_FENCE_ACQREL_CTA
  asm volatile("fence.acq_rel.cta;" ::: "memory");
#else
  __threadfence_block();  // measured faster here than fence.acq_rel.cta
#endif
}
__device__ __forceinline__ unsigned bl_ld_relaxed(const unsigned *p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned bl_ld_acquire(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Sense-free monotone grid barrier: the counter only grows; barrier k of a
// launch completes when it reaches k·G.  Requires co-residency (cooperative
// launch).  After the CTA barrier, thread 0 publishes the CTA's writes with a
// gpu-scope acq_rel fence + relaxed reduction, then spins with acquire loads
// (the arrive/wait pattern of CUTLASS's GenericBarrier).  Thread 0 also
// resets the CTA's dynamic work counter for the next phase.
__device__ __forceinline__ void bl_grid_sync(unsigned *bar, unsigned &target, int *unit_ctr,
                                             int *u_done = nullptr) {
  __syncthreads();
  if (threadIdx.x == 0) {
    target += gridDim.x;
    asm volatile("fence.acq_rel.gpu;\n\tred.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(bar)
                 : "memory");
    *unit_ctr = 0;
    if (u_done) *u_done = 0;
    while ((int)(bl_ld_acquire(bar) - target) < 0) {
    }
  }
  __syncthreads();
}

__device__ __forceinline__ float bl_warp_sum0(float v) {
  // fixed butterfly; lane 0's value is deterministic run to run
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Phase profiler: thread 0 of each CTA marks phase boundaries (clock64).
struct BLProf {
  unsigned long long acc[8];
  long long last;
  bool on;
  __device__ void init(const BLKParams &p) {
    on = p.prof != nullptr && threadIdx.x == 0;
    for (int i = 0; i < 8; ++i) acc[i] = 0;
    last = on ? clock64() : 0;
  }
  __device__ __forceinline__ void mark(int slot) {
    if (on) {
      const long long t = clock64();
      acc[slot] += (unsigned long long)(t - last);
      last = t;
    }
  }
  __device__ void flush(const BLKParams &p) {
    if (!on) return;
    if (blockIdx.x == 0)
      for (int i = 0; i < 8; ++i) p.prof[i] = acc[i];
    p.prof[8 + blockIdx.x] = acc[0] + acc[1] + acc[2];
  }
};

// Sweep resident float4 slots [s0, s1) for T targets: paired reciprocals on
// float4s of two real sources; the (at most one) float4 at index full4 that
// holds a real source and a far dummy is swept unpaired.
template <int T, int TP, int UN = (T >= 16 ? 2 * BL_SWEEP_UNROLL : T >= 8 ? BL_SWEEP_UNROLL : 2)>
__device__ __forceinline__ void bl_sweep_range(const float4 *src4, int s0, int s1, int full4,
                                               const float (&tx)[T], const float (&ty)[T],
                                               bl_f2 (&AX)[T], bl_f2 (&AY)[T], float rh) {
  constexpr int TP1 = TP < 0 ? TP : 0;  // the dummy-holding slot is never paired
  const int e = s1 < full4 ? s1 : full4;
  if (s0 < e) bl_sweep<T, TP, UN>(src4, s0, e, tx, ty, AX, AY, rh);
  if (s1 > full4 && s0 <= full4) bl_sweep<T, TP1, 1>(src4, full4, full4 + 1, tx, ty, AX, AY, rh);
}

// Geometry of CTA c's resident sources: m_c = ceil((n - c)/G) owned
// sources in float4 slots [0, last4); slots [0, full4) hold two real
// sources, slot full4 (if m_c is odd) one real source and a far dummy.
// [d_lo, d_hi): slots holding the `owned` sources k_lo.. being updated by
// this CTA in the current phase ("dirty"); clean4 = slots outside them.
struct BLGeom {
  int full4, last4, d_lo, d_hi, clean4;
};
__host__ __device__ inline BLGeom bl_geom(int c, int G, int n, int k_lo, int owned) {
  BLGeom g;
  const int m_c = c < n ? (n - 1 - c) / G + 1 : 0;
  g.full4 = m_c >> 1;
  g.last4 = g.full4 + (m_c & 1);
  g.d_lo = g.d_hi = 0;
  if (owned > 0) {
    g.d_lo = k_lo >> 1;
    g.d_hi = ((k_lo + owned - 1) >> 1) + 1;
    if (g.d_hi > g.last4) g.d_hi = g.last4;
    if (g.d_lo > g.d_hi) g.d_lo = g.d_hi;
  }
  g.clean4 = g.last4 - (g.d_hi - g.d_lo);
  return g;
}

// Source-slot segments of sub-range `sub` (< nc: a clean sub-range, guided
// cut of [0, d_lo) ++ [d_hi, last4); else the dirty slots [d_lo, d_hi)).
__device__ __forceinline__ void bl_unit_segments(const BLGeom &geo, int nc, int sub, int guided,
                                                 int (&lo)[2], int (&hi)[2], int &nseg) {
  nseg = 0;
  if (sub < nc) {
    const int dw = geo.d_hi - geo.d_lo;
    const int a = bl_guided_start(sub, nc, geo.clean4, guided);
    const int e = bl_guided_start(sub + 1, nc, geo.clean4, guided);
    if (a < geo.d_lo) {
      lo[nseg] = a;
      hi[nseg++] = min(e, geo.d_lo);
    }
    if (e > geo.d_lo) {
      lo[nseg] = max(a, geo.d_lo) + dw;
      hi[nseg++] = e + dw;
    }
  } else {
    lo[0] = geo.d_lo;
    hi[0] = geo.d_hi;
    nseg = 1;
  }
}

// One repulsion work unit g = (target tile g % ntt, sub-range g / ntt):
// clean sub-ranges are guided cuts of [0, d_lo) ++ [d_hi, last4); the last
// sub-range (if any) is the dirty slots.  The result goes to its own slot
// (red, or part directly when there is a single sub-range).
// tgt: staged targets in shared memory, or nullptr to read them from L2.
template <int T, int TP>
__device__ __forceinline__ void bl_do_unit(const BLKParams &p, int lo, int bt, const float4 *src4,
                                           const float2 *tgt, float2 *red, float2 *part, int g,
                                           const BLUnits &U, const BLGeom &geo, int tag = 0) {
  const int G = gridDim.x, c = blockIdx.x;
  const int lane = threadIdx.x & 31;
  const int tile = g % U.ntt, sub = g / U.ntt;
  BL_CHK(geo.last4 <= p.chunk4, BLC_BOUNDS, 10, geo.last4);
  float tx[T], ty[T];
  bl_f2 AX[T], AY[T];
#pragma unroll
  for (int k = 0; k < T; ++k) {
    const int idx = tile * 32 * T + k * 32 + lane;
    float2 t = make_float2(0.f, 0.f);
    if (idx < bt) t = tgt ? tgt[idx] : __ldcg(p.xy + lo + idx);
    tx[k] = t.x;
    ty[k] = t.y;
    AX[k] = f2pack(0.f, 0.f);
    AY[k] = f2pack(0.f, 0.f);
  }
  // the unit's source slots as <= 2 segments, swept by ONE call site (a
  // single copy of the unrolled loop in the binary: warps running different
  // segments share the instruction cache)
  int seg_lo[2], seg_hi[2], nseg = 0;
  bl_unit_segments(geo, U.nc, sub, p.guided, seg_lo, seg_hi, nseg);
#pragma unroll 1
  for (int q = 0; q < nseg; ++q)
    bl_sweep_range<T, TP>(src4, seg_lo[q], seg_hi[q], geo.full4, tx, ty, AX, AY, p.r_half);
#pragma unroll
  for (int k = 0; k < T; ++k) {
    const int idx = tile * 32 * T + k * 32 + lane;
    float ax0, ax1, ay0, ay1;
    f2unpack(AX[k], ax0, ax1);
    f2unpack(AY[k], ay0, ay1);
    const float2 r = make_float2(ax0 + ax1, ay0 + ay1);
    if (idx < bt) {
      if (U.nsub == 1) {
        part[(size_t)idx * G + c] = r;
        if (BL_CHK_ON) {
          const size_t o = (size_t)(part - p.part) + (size_t)idx * G + c;
          BL_CHK(o < (size_t)p.part_nbuf * p.b * G, BLC_BOUNDS, 1, o);
          p.part_st[o] = (unsigned)tag + 1u;
        }
      } else {
        BL_CHK(sub * (U.ntt * 32 * T) + idx < p.red_cap, BLC_BOUNDS, 2, sub);
        red[sub * (U.ntt * 32 * T) + idx] = r;
      }
    }
  }
}

// Fixed-order combine of the sub-range slots into part[target][c] (after a
// CTA barrier).
template <int T>
__device__ __forceinline__ void bl_combine(const BLKParams &p, int bt, const float2 *red,
                                           float2 *part, const BLUnits &U, int tag = 0) {
  if (U.nsub <= 1) return;
  const int G = gridDim.x, c = blockIdx.x;
  for (int idx = threadIdx.x; idx < bt; idx += BL_NT) {
    float2 acc = red[idx];
    for (int sb = 1; sb < U.nsub; ++sb) {
      const float2 v = red[sb * (U.ntt * 32 * T) + idx];
      acc.x += v.x;
      acc.y += v.y;
    }
    part[(size_t)idx * G + c] = acc;
    if (BL_CHK_ON) p.part_st[(size_t)(part - p.part) + (size_t)idx * G + c] = (unsigned)tag + 1u;
  }
}

// The repulsion work of one batch inside a CTA (two-barrier driver), as
// dynamically grabbed units: warps that did attraction items first take
// fewer.  Each unit's result has its own slot and the slots are combined in
// a fixed order, so the result does not depend on which warp ran which unit.
template <int T, int TP>
__device__ __forceinline__ void bl_sweep_units(const BLKParams &p, int lo, int bt,
                                               const float4 *src4, const float2 *tgt, float2 *red,
                                               int *unit_ctr, float2 *part, BLProf &pf,
                                               int tag = 0) {
  const int G = gridDim.x, c = blockIdx.x;
  const int lane = threadIdx.x & 31;
  const BLGeom geo = bl_geom(c, G, p.n, 0, 0);
  const BLUnits U = bl_units(bt, T, geo.clean4, false, p.red_cap);
  const int nunits = U.ntt * U.nsub;
  for (;;) {
    int g = 0;
    if (lane == 0) g = atomicAdd(unit_ctr, 1);
    g = __shfl_sync(0xffffffffu, g, 0);
    if (g >= nunits) break;
    bl_do_unit<T, TP>(p, lo, bt, src4, tgt, red, part, g, U, geo, tag);
  }
  pf.mark(1);
  __syncthreads();
  bl_combine<T>(p, bt, red, part, U, tag);
}

// ---------------------------------------------------------------- phase R
__device__ __forceinline__ unsigned bl_exp_stamp(const BLKParams &p, int j, int qmax) {
  // stamp of the latest batch index L <= qmax containing j (sequential
  // batches: batch of j = j / b), + 1; 0 if none
  const int tj = j / p.b;
  const int L = qmax - (((qmax - tj) % p.nb) + p.nb) % p.nb;
  return L >= 0 ? (unsigned)L + 1u : 0u;
}
// Attraction items of a RANDOMISED batch (readings R1-R2): batch position k
// holds vertex pi(lo + k), whose items are item_ptr[v] .. item_ptr[v+1]; the
// batch's items are numbered through ioff[k] = sum_{k' < k} items(pi(lo+k'))
// (a block-wide scan, identical in every CTA), so all warps of the grid
// share them as in the sequential case.  Requires bt <= BL_TGT_CAP.
__device__ __forceinline__ void bl_batch_item_offsets(const BLKParams &p, const BLPerm &P, int lo,
                                                      int bt, int *ioff) {
  // per-thread contiguous chunks, then a scan of the chunk totals
  const int per = (bt + BL_NT - 1) / BL_NT;
  const int a = threadIdx.x * per, e = min(a + per, bt);
  int tot = 0;
  for (int k = a; k < e; ++k) {
    const int v = bl_perm(P, lo + k);
    const int m = __ldg(p.item_ptr + v + 1) - __ldg(p.item_ptr + v);
    ioff[k + 1] = m;
    tot += m;
  }
  // inclusive scan of the per-thread totals (warp shuffles + warp totals)
  __shared__ int wsum[BL_NW_MAX];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  int base = 0;
  for (int w = 0; w < warp; ++w) base += wsum[w];
  int run = base + x - tot;  // exclusive prefix of this thread's chunk
  if (threadIdx.x == 0) ioff[0] = 0;
  for (int k = a; k < e; ++k) {
    run += ioff[k + 1];
    ioff[k + 1] = run;
  }
  __syncthreads();
}

template <int T, int TP>
__device__ __forceinline__ void bl_phase_R(const BLKParams &p, int lo, int bt, const float4 *src4,
                                           float2 *tgt, float2 *red, int *unit_ctr, BLProf &pf,
                                           const BLPerm &P, int *ioff, int tag = 0) {
  const int G = gridDim.x, c = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool tgt_smem = bt <= BL_TGT_CAP;

  // (0) stage the batch's targets (frozen coordinates)
  if (tgt_smem && !p.attr_only)
    for (int i = threadIdx.x; i < bt; i += BL_NT) {
      tgt[i] = __ldcg(p.xy + bl_perm(P, lo + i));
      if (BL_CHK_ON && !P.on && !p.forces_mode)
        BL_CHK(__ldcg(p.xy_st + lo + i) == bl_exp_stamp(p, lo + i, tag - 1), BLC_TGT_STAMP, tag,
               lo + i);
    }

  // (1r) randomised batch: items through pi and the batch item offsets
  if (P.on) {
    bl_batch_item_offsets(p, P, lo, bt, ioff);
    const int GW = G * BL_NW, ni = ioff[bt];
    const float rep = (p.flags & 1u) ? 0.f : p.ck2;
    for (int it = c * BL_NW + warp; it < ni; it += GW) {
      int l = 0, h = bt;  // the position k with ioff[k] <= it < ioff[k+1]
      while (h - l > 1) {
        const int m = (l + h) >> 1;
        if (ioff[m] <= it) l = m;
        else h = m;
      }
      const int v = bl_perm(P, lo + l);
      const int ag = __ldg(p.item_ptr + v) + (it - ioff[l]);
      const int k0 = __ldg(p.item_k0 + ag), k1 = __ldg(p.item_k0 + ag + 1);
      const float2 ci = __ldcg(p.xy + v);
      float sx = 0.f, sy = 0.f;
      int jj[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = k0 + lane + 32 * u;
        jj[u] = k < k1 ? __ldg(p.colidx + k) : -1;
      }
      float2 cj[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) cj[u] = jj[u] >= 0 ? __ldcg(p.xy + jj[u]) : ci;
      auto scan_row = [&](auto fast) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (jj[u] < 0) continue;
          const float dx = cj[u].x - ci.x, dy = cj[u].y - ci.y;
          const float d2 = fmaf(dx, dx, fmaf(dy, dy, BL_EPS2));
          const float rs = bl_rsqrt(d2);
          const float coef = bl_model_coef<decltype(fast)::value>(p, d2, rs, rep);
          sx = fmaf(coef, dx, sx);
          sy = fmaf(coef, dy, sy);
        }
      };
      if (p.amode == 0 && p.rmode == 0) scan_row(std::true_type{});
      else scan_row(std::false_type{});
      sx = bl_warp_sum0(sx);
      sy = bl_warp_sum0(sy);
      if (lane == 0) p.attr[it] = make_float2(sx, sy);
    }
  }

  // (1) attraction items of this batch, spread over all warps of the grid
  if (!P.on) {
    const int ib = __ldg(p.item_ptr + lo), ie = __ldg(p.item_ptr + lo + bt);
    const int GW = G * BL_NW;
    // the next item's (v, k0, k1) is loaded while the current one is
    // processed; k1 = item_k0[it + 1] (items tile the CSR in order, sentinel
    // nnz); the <= 4 entries per lane are loaded before any is consumed
    static_assert(BL_ECH == 4 * 32, "4 CSR entries per lane per item");
    int it = ib + c * BL_NW + warp;
    int v_n = 0, k0_n = 0, k1_n = 0;
    if (it < ie) {
      v_n = __ldg(p.item_v + it);
      k0_n = __ldg(p.item_k0 + it);
      k1_n = __ldg(p.item_k0 + it + 1);
    }
    for (; it < ie; it += GW) {
      const int v = v_n, k0 = k0_n, k1 = k1_n;
      if (it + GW < ie) {
        v_n = __ldg(p.item_v + it + GW);
        k0_n = __ldg(p.item_k0 + it + GW);
        k1_n = __ldg(p.item_k0 + it + GW + 1);
      }
      const float2 ci = __ldcg(p.xy + v);
      float sx = 0.f, sy = 0.f;
      const float rep = (p.flags & 1u) ? 0.f : p.ck2;
      int jj[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = k0 + lane + 32 * u;
        jj[u] = k < k1 ? __ldg(p.colidx + k) : -1;
      }
      float2 cj[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        cj[u] = jj[u] >= 0 ? __ldcg(p.xy + jj[u]) : ci;
        if (BL_CHK_ON && jj[u] >= 0 && !p.forces_mode)
          BL_CHK(__ldcg(p.xy_st + jj[u]) == bl_exp_stamp(p, jj[u], tag - 1), BLC_XY_STAMP, tag,
                 jj[u]);
      }
      auto scan_row = [&](auto fast) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (jj[u] < 0) continue;
          const float dx = cj[u].x - ci.x, dy = cj[u].y - ci.y;
          const float d2 = fmaf(dx, dx, fmaf(dy, dy, BL_EPS2));
          const float rs = bl_rsqrt(d2);
          const float coef = bl_model_coef<decltype(fast)::value>(p, d2, rs, rep);
          sx = fmaf(coef, dx, sx);
          sy = fmaf(coef, dy, sy);
        }
      };
      if (p.amode == 0 && p.rmode == 0) scan_row(std::true_type{});  // branch hoisted out of the loop
      else scan_row(std::false_type{});
      sx = bl_warp_sum0(sx);
      sy = bl_warp_sum0(sy);
      if (lane == 0) p.attr[it - ib] = make_float2(sx, sy);
    }
  }
  pf.mark(0);
  __syncthreads();  // targets staged

  // (2) repulsion sweep over the CTA's resident sources
  if (!p.attr_only)
    bl_sweep_units<T, TP>(p, lo, bt, src4, tgt_smem ? tgt : nullptr, red, unit_ctr, p.part, pf,
                          tag);
  pf.mark(2);
}

// ---------------------------------------------------------------- phase U
// Owner CTA c handles v in [lo, lo+bt) with v ≡ c (mod G); warp w takes the
// w-th, (w+NW)-th, ... of them.  All loads of one vertex are issued before
// any is consumed (one L2 round trip for the partials + item bounds, one for
// the attraction items).  Accumulates ||f||^2 into e_acc (lane 0).
// Randomised batches (P.on): CTA c takes the batch POSITIONS k = c (mod G),
// vertex pi(lo + k), reading its old coordinate from xy (not the owner's
// resident copy, which another CTA holds) and its attraction items through
// ioff; the owners refresh their resident copies after the next grid
// barrier (bl_refresh_resident).
__device__ __forceinline__ void bl_phase_U(const BLKParams &p, int lo, int bt, double stepd,
                                           float4 *src4, double &e_acc, const BLPerm &P,
                                           const int *ioff, int tag = 0) {
  const int G = gridDim.x, c = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int v0 = P.on ? c : lo + ((c - lo % G) + G) % G;
  const int vend = P.on ? bt : lo + bt;
  const int ib = __ldg(p.item_ptr + lo);
  for (int w = v0 + warp * G; w < vend; w += BL_NW * G) {
    const int local = P.on ? w : w - lo;
    const int v = P.on ? bl_perm(P, lo + w) : w;
    const int a0 = P.on ? ioff[w] : __ldg(p.item_ptr + v) - ib;
    const int a1 = P.on ? ioff[w + 1] : __ldg(p.item_ptr + v + 1) - ib;
    const float2 *row = p.part + (size_t)local * G;
    float rx = 0.f, ry = 0.f;
    if (!p.attr_only) {
#pragma unroll 8
      for (int cc = lane; cc < G; cc += 32) {
        const float2 q = __ldcg(row + cc);
        rx += q.x;
        ry += q.y;
      }
      if (BL_CHK_ON)
        for (int cc = lane; cc < G; cc += 32)
          BL_CHK(__ldcg(p.part_st + (size_t)local * G + cc) == (unsigned)tag + 1u,
                 BLC_PHASEU_STAMP, tag, cc);
    }
    float sx = 0.f, sy = 0.f;
    for (int a = a0 + lane; a < a1; a += 32) {
      const float2 q = __ldcg(p.attr + a);
      sx += q.x;
      sy += q.y;
    }
    rx = bl_warp_sum0(rx);
    ry = bl_warp_sum0(ry);
    sx = bl_warp_sum0(sx);
    sy = bl_warp_sum0(sy);
    if (lane == 0) {
      const float fx = fmaf(-p.ck2, rx, sx);
      const float fy = fmaf(-p.ck2, ry, sy);
      if (p.forces_mode) {
        p.f_out[v - p.first] = make_float2(fx, fy);
      } else {
        const double q = (double)fx * fx + (double)fy * fy;
        if (q > 0.0) {
          const double s = stepd / sqrt(q);
          // the owner's resident copy of xy[v] (randomised: xy itself, frozen
          // until this store -- no other warp reads xy[v] in this phase)
          float2 cv = P.on ? __ldcg(p.xy + v) : bl_src_get(src4, (v - c) / G);
          cv.x = (float)((double)cv.x + s * fx);
          cv.y = (float)((double)cv.y + s * fy);
          p.xy[v] = cv;
          if (!P.on) bl_src_set(src4, (v - c) / G, cv);
        }
        if (BL_CHK_ON) p.xy_st[v] = (unsigned)tag + 1u;
        e_acc += q;
      }
    }
  }
}

// After the grid barrier that follows a randomised batch's phase U: every
// CTA copies the new coordinates of the batch members it owns (v = c mod G)
// from xy into its resident source chunk.
__device__ __forceinline__ void bl_refresh_resident(const BLKParams &p, const BLPerm &P, int lo,
                                                    int bt, float4 *src4) {
  const int G = gridDim.x, c = blockIdx.x;
  for (int k = threadIdx.x; k < bt; k += BL_NT) {
    const int v = bl_perm(P, lo + k);
    if (v % G == c) bl_src_set(src4, (v - c) / G, __ldcg(p.xy + v));
  }
  __syncthreads();
}

// ------------------------------------------------- pipelined driver (nb >= 4)
// One SPLIT grid barrier per batch and a per-CTA task queue.  A CTA arrives
// at barrier ph as soon as its partials for batch ph are written; the work
// of phase ph+1 that depends on other CTAs (control, updates) is picked up
// by whichever warp notices that the barrier has completed, while the
// other warps keep sweeping -- the barrier latency and the latency-bound
// updates hide behind the FP32/SFU-bound sweep.  Tasks of phase ph:
//   control (one warp, once the barrier ph-1 has completed):
//       (a) if batch ph-2 closed an iteration: that iteration's energy,
//           summed in the same order in every CTA (identical tol decision,
//           P:1082);
//       (b) commit: the CTA's owned vertices of batch ph-2 are copied from
//           its shared copy to xy;
//       (c) cp.async prefetch of batch ph+1's targets;
//   update tasks (after control), one per owned vertex v of batch ph-1:
//       S_v (attraction + neighbour correction over v's CSR row) and
//       R_v = Σ_c part[v][c] give f_v; c_v += Step f/||f|| goes to the shared
//       copy and to pend -- NOT to xy, whose batch-(ph-1) entries other CTAs'
//       update tasks may still be reading as frozen coordinates;
//   sweep units of R(ph): clean ones any time; the "dirty" sub-range (this
//       CTA's sources updated in this phase) after the update tasks.
// Then: in-CTA combine -> part[ph&1]; arrive at barrier ph.
// Coordinates seen by batch ph: the vertices of batch ph-1 live in pend
// until committed in phase ph+1, so a neighbour j of a batch-ph vertex is
// read from pend when j is in batch ph-1 and from xy otherwise.  This is
// exactly the frozen-batch semantics of Alg. 2.
#define BL_ETASK_MAX 64  // owned vertices per CTA per batch (b <= 64·G)
#define BL_RSTAGE 32     // owned vertices per CTA per batch whose CSR rows are staged
#define BL_NTT_MAX 32    // target tiles per batch (BL_TGT_CAP / (32 T), T >= 2)

struct BLShared {
  int unit_ctr;   // next sweep unit
  int u_next;     // next update task
  int u_done;     // update tasks finished
  int stop_flag;  // tol convergence reached
  int ready;      // last phase whose control work is done
  int ctrl_claim; // last phase whose control work was claimed
  int seen;       // last phase whose barrier ph-1 was observed complete: the
                  // update tasks only need that (they read pend, not the
                  // commits of the control task), so they run alongside it
  int done_iters;
  double e_prev;  // energy of the previous completed iteration
  double e_acc;   // this CTA's energy of the running iteration
  double e_task[BL_ETASK_MAX];
  double e_warp[BL_NW_MAX];
  int ioff[BL_TGT_CAP + 1];  // randomised batches: item offsets per position
#ifdef BL_CHECKED
  int chk_upd[BL_ETASK_MAX];   // batch (+1) whose update task t last finished
#endif
  unsigned long long pkey[4];  // randomised batches: round keys of pi_it
  // CSR rows (<= 32 entries) of this CTA's owned vertices of a batch, staged
  // by the control task of the phase that sweeps the batch, used by the
  // update tasks one phase later (two fewer dependent L2 round trips on the
  // per-batch critical path); rowq = the batch they belong to
  // three buffers (batch q -> q % 3): the async driver stages batch ph+1 in
  // the control task of phase ph, after publishing `ready`, a phase before
  // its update tasks need it; only the first BL_RSTAGE owned vertices
  int rows[3][BL_RSTAGE][32];
  int rdeg[3][BL_RSTAGE];
  int rowq[3];
  // asynchronous-phase driver (bl_run_async): per phase parity s = ph & 1
  int a_unit[2];               // next sweep unit
  int a_tdone[2][BL_NTT_MAX];  // finished units per target tile
  int a_tok[2];                // completion tokens (tiles, control, updates)
  int a_unext[2], a_udone[2];  // update tasks taken / finished
  int a_exit[2];               // warps that left the phase
  int a_gen[2];                // the phase allowed to use slot s next
  int a_updph;                 // last phase whose update tasks all finished
  // latency driver (bl_run_lat): monotone phase stamps + per-parity counters
  int l_applied;               // last batch whose owned updates are in src4
  int l_cleanp[2];             // phase whose clean partials are combined, per parity
  int l_dec;                   // last phase whose stop decision is taken
  int l_join[2];               // updater warps that finished phase q's update
  int l_unit[2], l_exit[2], l_gen[2], l_tiles[2];
  int l_tdone[2][BL_NTT_MAX];
  // long rows (> BL_LCOOP entries) of the CTA's members, walked by all updater
  // warps together: row start / degree per member, one partial per (member, warp)
  int l_k0[BL_NW_MAX / 2], l_deg[BL_NW_MAX / 2];
  float2 l_lpart[BL_NW_MAX / 2][BL_NW_MAX / 2];
#ifdef BL_PHASE_TS
  // critical-path timestamps (profiling builds, -DBL_PHASE_TS; they cost ~3 %
  // at C5 even when disabled at run time, so they are compiled out by
  // default): phase start, control claimed / published, last update done
  long long ts_start, ts_claim, ts_ready, ts_upd;
  long long ts_upd_a, ts_arr_prev;  // async driver: updates done, previous arrival
#endif
};

__device__ __forceinline__ void bl_grid_arrive(unsigned *bar, unsigned &target, BLShared &sh,
                                               bool prof = false) {
  __syncthreads();
  target += gridDim.x;  // every thread tracks the barrier target
  if (threadIdx.x == 0) {
#ifdef BL_PHASE_TS
    if (prof) sh.ts_start = clock64();
#endif
    sh.unit_ctr = 0;
    sh.u_next = 0;
    sh.u_done = 0;
    asm volatile("fence.acq_rel.gpu;\n\tred.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(bar)
                 : "memory");
  }
  __syncthreads();
}

// cp.async of batch targets [lo, lo+bt) into dst by the calling warp (pairs
// of targets, 16 bytes each; an odd tail is copied directly).
__device__ __forceinline__ void bl_prefetch_targets_warp(const BLKParams &p, int lo, int bt,
                                                         float2 *dst) {
  const int lane = threadIdx.x & 31;
  const int npairs = bt >> 1;
  for (int i = lane; i < npairs; i += 32) {
    const unsigned saddr = (unsigned)__cvta_generic_to_shared(dst + 2 * i);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(p.xy + lo + 2 * i)
                 : "memory");
  }
  if ((bt & 1) && lane == 0) dst[bt - 1] = __ldcg(p.xy + lo + bt - 1);
  asm volatile("cp.async.commit_group;" ::: "memory");
}

__device__ __forceinline__ void bl_commit_warp(const BLKParams &p, int q, const float4 *src4) {
  const int G = gridDim.x, c = blockIdx.x, lane = threadIdx.x & 31;
  const int lo = (q % p.nb) * p.b, hi = min(lo + p.b, p.n);
  const int v0 = lo + ((c - lo % G) + G) % G;
  for (int v = v0 + lane * G; v < hi; v += 32 * G) {
    p.xy[v] = bl_src_get(src4, (v - c) / G);
    if (BL_CHK_ON) p.xy_st[v] = (unsigned)q + 1u;
  }
}

// Energy of iteration `it` from the per-CTA sums, warp-cooperative, in a
// fixed order (identical in every CTA).
__device__ __forceinline__ double bl_energy_sum_warp(const BLKParams &p, int it) {
  const int G = gridDim.x, lane = threadIdx.x & 31;
  double e = 0.0;
  for (int cc = lane; cc < G; cc += 32) e += __ldcg(p.e_cta + (it & 1) * G + cc);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
  return __shfl_sync(0xffffffffu, e, 0);
}

// Checked builds: the coordinate of neighbour j read by the update of batch q
// must be exactly the one Alg. 2 prescribes (frozen batches):
// batch q-1's new value from pend, else the last COMMITTED update of j --
// batch L = the latest index <= q-2 of j's batch (sequential batches) -- or
// none (stamp 0).  Not older (a lost commit) and not newer.
__device__ __forceinline__ void bl_chk_nb(const BLKParams &p, int q, int j, int plo, int phi) {
#ifdef BL_CHECKED
  if (j >= plo && j < phi) {
    BL_CHK(__ldcg(p.pend_st + (size_t)((q - 1) & 1) * p.b + (j - plo)) == (unsigned)q,
           BLC_PEND_STAMP, q, j);
  } else {
    BL_CHK(__ldcg(p.xy_st + j) == bl_exp_stamp(p, j, q - 2), BLC_XY_STAMP, q, j);
  }
#endif
}

// Update of one owned vertex v of batch q (warp-cooperative); ||f||^2 -> *eq.
// apart != nullptr: the row's attraction was computed by napart warps
// (bl_long_row_part), summed here in warp order.
__device__ __forceinline__ void bl_update_one(const BLKParams &p, int q, int v, double stepd,
                                              float4 *src4, double *eq, const int *srow,
                                              int sdeg, const float2 *apart = nullptr,
                                              int napart = 0) {
  const int G = gridDim.x, c = blockIdx.x, lane = threadIdx.x & 31;
  const int lo = (q % p.nb) * p.b;
  const int local = v - lo;
  // neighbours in batch q-1 are read from pend (committed only next phase)
  int plo = 0, phi = 0;
  const float2 *pend_prev = p.pend + (size_t)((q - 1) & 1) * p.b;
  if (q >= 1) {
    plo = ((q - 1) % p.nb) * p.b;
    phi = min(plo + p.b, p.n);
  }
  const float2 ci = bl_src_get(src4, (v - c) / G);
  const float2 *row = p.part + (size_t)(q % p.part_nbuf) * p.b * G + (size_t)local * G;
  // latency: the staged row's neighbour gather (one entry per lane) and the
  // row bounds of a long row are issued BEFORE the partial-row loads are
  // consumed, so the two dependent L2 trips of an update overlap
  int j_st = -1;
  float2 cj_st = ci;
  if (srow && lane < sdeg) {
    j_st = srow[lane];
    cj_st = (j_st >= plo && j_st < phi) ? __ldcg(pend_prev + (j_st - plo)) : __ldcg(p.xy + j_st);
  }
  int k0 = 0, k1 = 0;
  if (!srow && !apart) {
    k0 = __ldg(p.rowptr + v);
    k1 = __ldg(p.rowptr + v + 1);
  }
  float rx = 0.f, ry = 0.f;
  {
    float2 pr[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int cc = lane + 32 * u;
      pr[u] = cc < G ? __ldcg(row + cc) : make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (lane + 32 * u < G) {
        rx += pr[u].x;
        ry += pr[u].y;
      }
    for (int cc = lane + 256; cc < G; cc += 32) {  // G > 256 (not on B200's 148 SMs)
      const float2 t = __ldcg(row + cc);
      rx += t.x;
      ry += t.y;
    }
  }
  if (BL_CHK_ON)
    for (int cc = lane; cc < G; cc += 32)
      BL_CHK(__ldcg(p.part_st + (size_t)(row - p.part) + cc) == (unsigned)q + 1u, BLC_PART_STAMP,
             q, cc);
  const float rep = (p.flags & 1u) ? 0.f : p.ck2;
  float sx = 0.f, sy = 0.f;
  auto scan_row = [&](auto fast) {
    if (srow) {  // staged row: one entry per lane (gathered above)
      if (lane < sdeg) {
        const int j = j_st;
        const float2 cj = cj_st;
        if (BL_CHK_ON) bl_chk_nb(p, q, j, plo, phi);
        const float dx = cj.x - ci.x, dy = cj.y - ci.y;
        const float d2 = fmaf(dx, dx, fmaf(dy, dy, BL_EPS2));
        const float rs = bl_rsqrt(d2);
        const float coef = bl_model_coef<decltype(fast)::value>(p, d2, rs, rep);
        sx = fmaf(coef, dx, sx);
        sy = fmaf(coef, dy, sy);
      }
      return;
    }
    // long rows: a lane's next 8 entries are loaded before any is used (two
    // dependent L2 round trips per 256 entries; per-lane order unchanged).
    // Measured: +1.4 % at C5 (async driver: shorter updates, less waiting on
    // other CTAs), -1..2 % on the latency-bound configs, which keep the
    // unrolled loop below.
    if (!p.long8) {
#pragma unroll 4
      for (int k = k0 + lane; k < k1; k += 32) {
        const int j = __ldg(p.colidx + k);
        const float2 cj = (j >= plo && j < phi) ? __ldcg(pend_prev + (j - plo)) : __ldcg(p.xy + j);
        if (BL_CHK_ON) bl_chk_nb(p, q, j, plo, phi);
        const float dx = cj.x - ci.x, dy = cj.y - ci.y;
        const float d2 = fmaf(dx, dx, fmaf(dy, dy, BL_EPS2));
        const float rs = bl_rsqrt(d2);
        const float coef = bl_model_coef<decltype(fast)::value>(p, d2, rs, rep);
        sx = fmaf(coef, dx, sx);
        sy = fmaf(coef, dy, sy);
      }
      return;
    }
    for (int base = k0; base < k1; base += 256) {
      int jj[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int k = base + lane + 32 * u;
        jj[u] = k < k1 ? __ldg(p.colidx + k) : -1;
      }
      float2 cj[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int j = jj[u];
        cj[u] = j < 0 ? ci : (j >= plo && j < phi) ? __ldcg(pend_prev + (j - plo)) : __ldcg(p.xy + j);
        if (BL_CHK_ON && j >= 0) bl_chk_nb(p, q, j, plo, phi);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (jj[u] < 0) continue;
        const float dx = cj[u].x - ci.x, dy = cj[u].y - ci.y;
        const float d2 = fmaf(dx, dx, fmaf(dy, dy, BL_EPS2));
        const float rs = bl_rsqrt(d2);
        const float coef = bl_model_coef<decltype(fast)::value>(p, d2, rs, rep);
        sx = fmaf(coef, dx, sx);
        sy = fmaf(coef, dy, sy);
      }
    }
  };
  if (apart) {
    if (lane == 0)
      for (int w = 0; w < napart; ++w) {
        sx += apart[w].x;
        sy += apart[w].y;
      }
  } else if (p.amode == 0 && p.rmode == 0) scan_row(std::true_type{});  // branch hoisted out of the loop
  else scan_row(std::false_type{});
  rx = bl_warp_sum0(rx);
  ry = bl_warp_sum0(ry);
  sx = bl_warp_sum0(sx);
  sy = bl_warp_sum0(sy);
  if (lane == 0) {
    const float fx = fmaf(-p.ck2, rx, sx);
    const float fy = fmaf(-p.ck2, ry, sy);
    const double qq = (double)fx * fx + (double)fy * fy;
    float2 cv = ci;
    if (qq > 0.0) {
      const double sc = stepd / sqrt(qq);
      cv.x = (float)((double)cv.x + sc * fx);
      cv.y = (float)((double)cv.y + sc * fy);
      bl_src_set(src4, (v - c) / G, cv);
    }
    p.pend[(size_t)(q & 1) * p.b + local] = cv;
    if (BL_CHK_ON) {
      BL_CHK(local >= 0 && local < p.b, BLC_BOUNDS, 3, local);
      p.pend_st[(size_t)(q & 1) * p.b + local] = (unsigned)q + 1u;
    }
    *eq = qq;
  }
}

// Latency driver: a member's long CSR row [k0, k0 + deg) walked by the CTA's U
// updater warps together -- warp w takes the 256-entry chunks w, w + U, ...
// (8 gathers in flight per lane), its partial attraction (+ neighbour
// correction) sum goes to lane 0.  Same terms as bl_update_one's row scan;
// the owner adds the U partials in warp order.
#define BL_LCOOP 256
__device__ __forceinline__ float2 bl_long_row_part(const BLKParams &p, int q, int k0, int deg,
                                                   float2 ci, int w, int U) {
  const int lane = threadIdx.x & 31;
  int plo = 0, phi = 0;
  const float2 *pend_prev = p.pend + (size_t)((q - 1) & 1) * p.b;
  if (q >= 1) {
    plo = ((q - 1) % p.nb) * p.b;
    phi = min(plo + p.b, p.n);
  }
  const float rep = (p.flags & 1u) ? 0.f : p.ck2;
  const int k1 = k0 + deg;
  float sx = 0.f, sy = 0.f;
  auto walk = [&](auto fast) {
    for (int base = k0 + w * 256; base < k1; base += U * 256) {
      int jj[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int k = base + lane + 32 * u;
        jj[u] = k < k1 ? __ldg(p.colidx + k) : -1;
      }
      float2 cj[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int j = jj[u];
        cj[u] = j < 0 ? ci : (j >= plo && j < phi) ? __ldcg(pend_prev + (j - plo)) : __ldcg(p.xy + j);
        if (BL_CHK_ON && j >= 0) bl_chk_nb(p, q, j, plo, phi);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (jj[u] < 0) continue;
        const float dx = cj[u].x - ci.x, dy = cj[u].y - ci.y;
        const float d2 = fmaf(dx, dx, fmaf(dy, dy, BL_EPS2));
        const float rs = bl_rsqrt(d2);
        const float coef = bl_model_coef<decltype(fast)::value>(p, d2, rs, rep);
        sx = fmaf(coef, dx, sx);
        sy = fmaf(coef, dy, sy);
      }
    }
  };
  if (p.amode == 0 && p.rmode == 0) walk(std::true_type{});
  else walk(std::false_type{});
  sx = bl_warp_sum0(sx);
  sy = bl_warp_sum0(sy);
  return make_float2(sx, sy);
}

// Phase geometry shared by all warps of a CTA.
struct BLPhase {
  int ph, P, q1, q2;
  int owned, v0;      // owned vertices of batch q1: v0, v0+G, ...
  double step_u;      // Step of batch q1 (fp64 schedule)
  float2 *tgt_next;   // staging buffer for batch ph+1's targets
};

__device__ __forceinline__ bool bl_closes_iteration(int q, int nb, int P) {
  return q % nb == nb - 1 || q == P - 1;
}

// Stage the CSR rows of this CTA's owned vertices of batch q (swept in this
// phase, updated in the next) into shared memory: rows of <= 32 entries,
// rdeg = -1 marks longer rows (they take the global path).
__device__ __forceinline__ void bl_stage_rows_warp(const BLKParams &p, int q, BLShared &sh) {
  const int G = gridDim.x, c = blockIdx.x, lane = threadIdx.x & 31;
  const int lo = (q % p.nb) * p.b, hi = min(lo + p.b, p.n);
  const int v0 = lo + ((c - lo % G) + G) % G;
  const int owned = min(BL_RSTAGE, v0 < hi ? (hi - 1 - v0) / G + 1 : 0);
  const int buf = q % 3;
  // two L2 round trips in all (latency is the cost here: this runs on the
  // per-batch critical path): the row bounds of up to 32 owned vertices in
  // one load per lane, then the rows of 8 vertices at a time, every load
  // issued before the first store
  for (int t0 = 0; t0 < owned; t0 += 32) {
    int k0 = 0, deg = 0;
    if (t0 + lane < owned) {
      const int v = v0 + (t0 + lane) * G;
      k0 = __ldg(p.rowptr + v);
      deg = __ldg(p.rowptr + v + 1) - k0;
    }
    const int m = min(32, owned - t0);
    for (int t1 = 0; t1 < m; t1 += 8) {
      int col[8], dg[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int kk = __shfl_sync(0xffffffffu, k0, (t1 + u) & 31);
        dg[u] = __shfl_sync(0xffffffffu, deg, (t1 + u) & 31);
        col[u] = (t1 + u < m && dg[u] <= 32 && lane < dg[u]) ? __ldg(p.colidx + kk + lane) : 0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (t1 + u < m) {
          const int t = t0 + t1 + u;
          if (dg[u] <= 32 && lane < dg[u]) sh.rows[buf][t][lane] = col[u];
          if (lane == 0) sh.rdeg[buf][t] = dg[u] <= 32 ? dg[u] : -1;
        }
      }
    }
  }
  __syncwarp();
  if (lane == 0) {
    bl_fence_cta();  // rows before rowq (the async driver stages after `ready`)
    *(volatile int *)&sh.rowq[buf] = q;
  }
}

// Writes that other CTAs read after barrier ph (part, pend, xy commits) are
// released to the phase's completer at CTA scope; the completer's
// fence.acq_rel.gpu before its arrival is cumulative, so it publishes them
// at GPU scope (the same argument as a CTA barrier followed by one thread's
// GPU fence).  BL_AFENCE=1 (debug) fences at GPU scope in every task instead.
__device__ __forceinline__ void bl_fence_to_completer(const BLKParams &p) {
  if (p.afence_gpu) __threadfence();
  else bl_fence_cta();
}

__device__ __forceinline__ void bl_token(const BLKParams &p, BLShared &sh, const BLPhase &f,
                                         int need) {
  // lane 0 of the caller, after its writes were fenced
  bl_jitter(p, 11);
  const int tok = atomicAdd(&sh.a_tok[f.ph & 1], 1);
  BL_CHK(tok < need, BLC_TOKENS, f.ph, tok);
  if (tok != need - 1) return;
  bl_fence_cta();
  const int G = gridDim.x, c = blockIdx.x;
  if (f.owned > 0) {
    double e = sh.e_acc;
    for (int i = 0; i < f.owned; ++i) e += sh.e_task[i];  // task order
    sh.e_acc = e;
  }
  if (f.q1 >= 0 && f.ph <= f.P && bl_closes_iteration(f.q1, p.nb, f.P)) {
    p.e_cta[((f.q1 / p.nb) & 1) * G + c] = sh.e_acc;
    sh.e_acc = 0.0;
  }
#ifdef BL_PHASE_TS
  const long long t_tok = clock64();
#endif
  if (f.ph <= f.P)
    asm volatile("fence.acq_rel.gpu;\n\tred.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(p.bar)
                 : "memory");
#ifdef BL_PHASE_TS
  // async critical-path timeline of CTA 0: per phase, barrier
  // ph-1 + its detection, control, updates, tail (dirty units + tile
  // combines after the later of control and updates), arrival
  if (p.prof && c == 0) {
    const long long t_arr = clock64();
    unsigned long long *hp = p.prof + 8 + G;
    if (f.ph > 0) {
      long long last = sh.ts_ready > sh.ts_claim ? sh.ts_ready : sh.ts_claim;
      if (f.owned > 0 && sh.ts_upd_a > last) last = sh.ts_upd_a;
      hp[0] += (unsigned long long)(sh.ts_claim - sh.ts_arr_prev);
      hp[1] += (unsigned long long)(sh.ts_ready - sh.ts_claim);
      if (f.owned > 0) hp[2] += (unsigned long long)(sh.ts_upd_a - sh.ts_claim);
      hp[3] += (unsigned long long)(t_tok > last ? t_tok - last : 0);
      hp[4] += (unsigned long long)(t_arr - t_tok);
      hp[5] += 1ull;
      if (f.owned > 0) hp[6] += 1ull;
    }
    sh.ts_arr_prev = t_arr;
  }
#endif
}

// Control work of phase ph, attempted by a warp between tasks: if barrier
// ph-1 has completed and no other warp claimed it, do (a)-(c) and publish.
__device__ __forceinline__ bool bl_try_control(const BLKParams &p, const BLPhase &f,
                                               const float4 *src4, BLShared &sh,
                                               unsigned bar_target, int need = -1) {
  const int lane = threadIdx.x & 31;
  int go = 0;
  // BL_POLL_RELAXED=1: poll with a relaxed load, the claimant alone then
  // acquires with a GPU-scope fence (measured slower than acquire polls,
  // DESIGN.md §13)
#if BL_POLL_RELAXED
  if (lane == 0 && ((int)(bl_ld_relaxed(p.bar) - bar_target) >= 0 || (BL_CHK_ON && p.chk_break))) {
    go = atomicCAS(&sh.ctrl_claim, f.ph - 1, f.ph) == f.ph - 1;
    if (go) asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
#else
  if (lane == 0 && ((int)(bl_ld_acquire(p.bar) - bar_target) >= 0 || (BL_CHK_ON && p.chk_break)))
    go = atomicCAS(&sh.ctrl_claim, f.ph - 1, f.ph) == f.ph - 1;
#endif
#ifdef BL_PHASE_TS
  if (go && p.prof) sh.ts_claim = clock64();
#endif
  if (go) {
    *(volatile int *)&sh.seen = f.ph;  // release the update tasks now
    bl_fence_cta();
  }
  go = __shfl_sync(0xffffffffu, go, 0);
  if (!go) return false;
  __syncwarp();  // order the lanes' reads after lane 0's acquire
  bool stop = false;
  const int nb = p.nb;
  // async driver: the next batch's targets were last written by batch
  // ph+1-nb, committed by the control task of phase ph+3-nb <= ph-1 when
  // nb >= 4, so their copy can be in flight while this task commits (one L2
  // round trip for both); the staging buffer's last readers (phase ph-1's
  // units) finished before barrier ph-1
  const bool early_tgt = BL_EARLY_TGT && need >= 0 && nb >= 4 && f.ph + 1 < f.P;
  if (early_tgt) {
    const int lo_n = ((f.ph + 1) % nb) * p.b;
    bl_prefetch_targets_warp(p, lo_n, min(p.b, p.n - lo_n), f.tgt_next);
  }
  if (f.q2 >= 0 && bl_closes_iteration(f.q2, nb, f.P)) {
    const int it = f.q2 / nb;
    const double E = bl_energy_sum_warp(p, it);
    if (blockIdx.x == 0 && lane == 0) p.energy[it] = E;
    if (f.q2 % nb == nb - 1 && f.q2 < f.P - 1 && p.tol > 0.0 && it > 0 &&
        fabs(E - sh.e_prev) < p.tol) {
      stop = true;
      if (lane == 0) sh.done_iters = it + 1;
    }
    __syncwarp();
    if (lane == 0) sh.e_prev = E;
  }
  if (f.q2 >= 0) bl_commit_warp(p, f.q2, src4);
  if (need >= 0) {  // async driver: the control task's completion token (the
                    // staging below is for the next phase, not this one)
    __syncwarp();
    if (lane == 0) {
      bl_fence_to_completer(p);  // commits to xy
      bl_token(p, sh, f, need);
    }
  }
  if (!stop && f.ph + 1 < f.P && !early_tgt) {
    const int lo_n = ((f.ph + 1) % nb) * p.b;
    bl_prefetch_targets_warp(p, lo_n, min(p.b, p.n - lo_n), f.tgt_next);
  }
  // (measured: staging the rows after `ready` -- even a phase ahead -- costs
  // ~1 us per batch at C2 / C3: the control warp is the awake warp that
  // picks up the next task)
  if (!stop && f.ph < f.P) bl_stage_rows_warp(p, f.ph, sh);
  // async driver: the targets must have landed before `ready` lets warps
  // into phase ph+1 (the pipelined driver waits at its phase-end barrier)
  if (need >= 0) asm volatile("cp.async.wait_all;" ::: "memory");
  if (BL_CHK_ON && !stop && f.ph + 1 < f.P) {
    // the staged targets of batch ph+1 are its last committed coordinates
    // (from the previous iteration; batch ph+1-nb <= ph-2 was committed by
    // an earlier control task) -- checked on the bytes that landed
    const int lo_n = ((f.ph + 1) % nb) * p.b, bt_n = min(p.b, p.n - lo_n);
    for (int i = lane; i < bt_n; i += 32) {
      if (need >= 0) {
        const float2 a = f.tgt_next[i], b = __ldcg(p.xy + lo_n + i);
        BL_CHK(a.x == b.x && a.y == b.y, BLC_TGT_STAMP, f.ph, lo_n + i);
      }
      BL_CHK(__ldcg(p.xy_st + lo_n + i) == bl_exp_stamp(p, lo_n + i, f.ph - 2), BLC_TGT_STAMP,
             f.ph, lo_n + i);
    }
  }
  __syncwarp();
  if (lane == 0) {
    if (stop) *(volatile int *)&sh.stop_flag = 1;
    bl_fence_cta();
#ifdef BL_PHASE_TS
    if (p.prof) sh.ts_ready = clock64();
#endif
    *(volatile int *)&sh.ready = f.ph;
  }
  __syncwarp();
  return true;
}

// Try to take and run one update task; returns true if one was run.
__device__ __forceinline__ bool bl_try_update(const BLKParams &p, const BLPhase &f, float4 *src4,
                                              BLShared &sh) {
  const int lane = threadIdx.x & 31;
  const volatile BLShared &vs = sh;
  if (vs.seen != f.ph || vs.stop_flag || vs.u_next >= f.owned) return false;
  int t = f.owned;
  if (lane == 0) t = atomicAdd(&sh.u_next, 1);
  t = __shfl_sync(0xffffffffu, t, 0);
  if (t >= f.owned) return false;
  bl_fence_cta();  // acquire the control warp's publication
  const int buf = f.q1 % 3;
  const volatile BLShared &vsh = sh;
  const bool staged = t < BL_RSTAGE && vsh.rowq[buf] == f.q1 && vsh.rdeg[buf][t] >= 0;
  bl_jitter(p, 21);
  bl_update_one(p, f.q1, f.v0 + t * gridDim.x, f.step_u, src4, &sh.e_task[t],
                staged ? sh.rows[buf][t] : nullptr, staged ? vsh.rdeg[buf][t] : 0);
  __syncwarp();
  if (lane == 0) {
#ifdef BL_CHECKED
    sh.chk_upd[t] = f.q1 + 1;
#endif
    bl_fence_cta();
#ifdef BL_PHASE_TS
    if (atomicAdd(&sh.u_done, 1) == f.owned - 1 && p.prof) sh.ts_upd = clock64();
#else
    atomicAdd(&sh.u_done, 1);
#endif
  }
  return true;
}

template <int T, int TP>
__device__ __forceinline__ void bl_phase_tasks(const BLKParams &p, const BLPhase &f,
                                               float4 *src4, const float2 *tgt, float2 *red,
                                               BLShared &sh, unsigned bar_target) {
  const int G = gridDim.x, c = blockIdx.x;
  const int lane = threadIdx.x & 31;
  const volatile BLShared &vs = sh;
  const bool has_R = f.ph < f.P;
  const int lo = has_R ? (f.ph % p.nb) * p.b : 0;
  const int bt = has_R ? min(p.b, p.n - lo) : 0;
  const BLGeom geo = bl_geom(c, G, p.n, f.owned > 0 ? (f.v0 - c) / G : 0, f.owned);
  BLUnits U = {1, 0, 0};
  if (has_R) U = bl_units(bt, T, geo.clean4, geo.d_lo < geo.d_hi, p.red_cap, BL_NSUB_MAX, p.min_unit4);
  const int n_all = has_R ? U.ntt * U.nsub : 0;
  const int n_clean = has_R ? U.ntt * U.nc : 0;
  float2 *part = p.part + (size_t)(f.ph & 1) * p.b * G;
  for (;;) {
    bl_jitter(p, 27);
    if (f.ph > 0 && vs.ready != f.ph) bl_try_control(p, f, src4, sh, bar_target);
    if (bl_try_update(p, f, src4, sh)) continue;
    int g = n_all;
    if (vs.unit_ctr < n_all) {
      if (lane == 0) g = atomicAdd(&sh.unit_ctr, 1);
      g = __shfl_sync(0xffffffffu, g, 0);
    }
    if (g < n_all) {
      if (g >= n_clean) {
        // dirty sub-range: needs this CTA's updates of batch q1; help until done
        for (;;) {
          if (f.ph > 0 && vs.ready != f.ph) bl_try_control(p, f, src4, sh, bar_target);
          if (bl_try_update(p, f, src4, sh)) continue;
          if ((f.ph == 0 || vs.seen == f.ph) && (vs.stop_flag || vs.u_done >= f.owned)) break;
          __nanosleep(64);
        }
        bl_fence_cta();
#ifdef BL_CHECKED
        if (!vs.stop_flag)
          for (int t = 0; t < f.owned; ++t)
            BL_CHK(((volatile int *)sh.chk_upd)[t] == f.q1 + 1, BLC_DIRTY_EARLY, f.ph, t);
#endif
      }
      bl_jitter(p, 24);
      bl_do_unit<T, TP>(p, lo, bt, src4, tgt, red, part, g, U, geo, f.ph);
      continue;
    }
    // nothing left to grab: done once control ran and every update is taken
    if ((f.ph == 0 || vs.ready == f.ph) && (vs.stop_flag || vs.u_next >= f.owned)) break;
    __nanosleep(32);
  }
}

template <int T, int TP>
__device__ __forceinline__ void bl_run_pipelined(const BLKParams &p, float4 *src4, float2 *tgt,
                                                 float2 *red, BLShared &sh, BLProf &pf,
                                                 unsigned &bar_target) {
  const int G = gridDim.x, c = blockIdx.x;
  const int nb = p.nb;
  const long long ptot = (long long)p.iters * nb;
  const bool mb_stop = p.max_batches > 0 && p.max_batches <= ptot;  // == ptot: as the oracle, iters - 1 done
  const int P = mb_stop ? p.max_batches : (int)ptot;
  double step_u = p.step0;
  if (threadIdx.x == 0) {
    sh.done_iters = mb_stop ? (P - 1) / nb : p.iters;
    sh.e_prev = 0.0;
    sh.e_acc = 0.0;
  }
  if (threadIdx.x < 32) {
    bl_prefetch_targets_warp(p, 0, min(p.b, p.n), tgt);
    if (P > 1) {
      bl_prefetch_targets_warp(p, (1 % nb) * p.b, min(p.b, p.n - (1 % nb) * p.b),
                               tgt + BL_TGT_CAP);
      asm volatile("cp.async.wait_group 1;" ::: "memory");  // batch 0's group landed
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");  // only batch 0 was issued
    }
  }
  __syncthreads();

  for (int ph = 0; ph <= P + 1; ++ph) {
    BLPhase f;
    f.ph = ph;
    f.P = P;
    f.q1 = ph - 1;
    f.q2 = ph - 2;
    f.owned = 0;
    f.v0 = 0;
    if (f.q1 >= 0 && ph <= P) {
      const int lo1 = (f.q1 % nb) * p.b, hi1 = min(lo1 + p.b, p.n);
      f.v0 = lo1 + ((c - lo1 % G) + G) % G;
      f.owned = f.v0 < hi1 ? (hi1 - 1 - f.v0) / G + 1 : 0;
      if (f.q1 > 0 && f.q1 % nb == 0) step_u = step_u * p.cooling;
    }
    f.step_u = step_u;
    f.tgt_next = tgt + ((ph + 1) & 1) * BL_TGT_CAP;
    pf.mark(3);
    bl_phase_tasks<T, TP>(p, f, src4, tgt + (ph & 1) * BL_TGT_CAP, red, sh, bar_target);
    pf.mark(1);
    __syncthreads();
#ifdef BL_PHASE_TS
    if (pf.on && ph > 0) {
      // critical-path split of this phase (CTA 0 reported): barrier ph-1 +
      // its detection, control task, update tasks after control
      pf.acc[0] += (unsigned long long)(sh.ts_claim - sh.ts_start);
      pf.acc[4] += (unsigned long long)(sh.ts_ready - sh.ts_claim);
      if (f.owned > 0) pf.acc[7] += (unsigned long long)(sh.ts_upd - sh.ts_ready);
    }
#endif
    if (sh.stop_flag) {
      if (c == 0 && threadIdx.x == 0) *p.iters_done = sh.done_iters;
      pf.flush(p);
      return;
    }
    if (ph < P) {
      const int lo = (ph % nb) * p.b, bt = min(p.b, p.n - lo);
      const BLGeom geo = bl_geom(c, G, p.n, f.owned > 0 ? (f.v0 - c) / G : 0, f.owned);
      const BLUnits U = bl_units(bt, T, geo.clean4, geo.d_lo < geo.d_hi, p.red_cap, BL_NSUB_MAX,
                                 p.min_unit4);
      bl_combine<T>(p, bt, red, p.part + (size_t)(ph & 1) * p.b * G, U, ph);
    }
    if (threadIdx.x == 0 && f.owned > 0) {
      double e = sh.e_acc;
      for (int i = 0; i < f.owned; ++i) e += sh.e_task[i];
      sh.e_acc = e;
    }
    if (f.q1 >= 0 && ph <= P && bl_closes_iteration(f.q1, nb, P) && threadIdx.x == 0) {
      p.e_cta[((f.q1 / nb) & 1) * G + c] = sh.e_acc;
      sh.e_acc = 0.0;
    }
    pf.mark(2);
    asm volatile("cp.async.wait_all;" ::: "memory");
    bl_jitter(p, 28);
    if (ph <= P) bl_grid_arrive(p.bar, bar_target, sh, p.prof != nullptr);
    pf.mark(5);
  }
  if (c == 0 && threadIdx.x == 0) *p.iters_done = sh.done_iters;
  pf.mark(6);
  pf.flush(p);
}

// ------------------------------------------- asynchronous-phase driver
// The tasks and the arithmetic of bl_run_pipelined, without the CTA-wide
// barrier (and the combine that follows it) at the end of each phase: every
// warp walks the phases on its own.  A warp leaves phase ph when it finds
// nothing left to grab there and enters phase ph+1 at once, so the tail of a
// phase (its last units, the combine, the grid-barrier arrival) overlaps the
// next phase's sweep.  Per phase (parity slot s = ph & 1):
//   * the warp that finishes the last unit of a target tile combines that
//     tile's sub-range partials (red slot s, fixed order) into part[ph % 3];
//   * completion tokens: one per tile, one for the control task, one per
//     update task; whoever adds the last token closes the phase (energy
//     bookkeeping) and arrives at grid barrier ph;
//   * entering phase ph+1 needs: the control task of phase ph done (targets
//     of ph+1 staged), the update tasks of phase ph done (their sources are
//     clean in ph+1), and slot (ph+1)&1 released by every warp of phase ph-1
//     (the last warp to leave a phase resets its slot).
// At most two phases are live in a CTA.  part has three buffers: a CTA
// enters phase ph once barrier ph-2 has completed, so its tile combines of
// phase ph (into part[ph % 3]) can run while slower CTAs' update tasks of
// phase ph-1 still read the partials of batch ph-2 (part[(ph-2) % 3]) and
// after barrier ph-1 everyone reads part[(ph-1) % 3]: three distinct
// buffers.  Results are independent of which warp ran which task (fixed
// summation orders), as in the pipelined driver.
__device__ __forceinline__ bool bl_try_update_a(const BLKParams &p, const BLPhase &f,
                                                float4 *src4, BLShared &sh, int need) {
  const int lane = threadIdx.x & 31, s = f.ph & 1;
  const volatile BLShared &vs = sh;
  if (vs.seen < f.ph || vs.stop_flag || vs.a_unext[s] >= f.owned) return false;
  int t = f.owned;
  if (lane == 0) t = atomicAdd(&sh.a_unext[s], 1);
  t = __shfl_sync(0xffffffffu, t, 0);
  if (t >= f.owned) return false;
  bl_fence_cta();  // acquire the control warp's publication
  const int buf = f.q1 % 3;
  bool staged = t < BL_RSTAGE && vs.rowq[buf] == f.q1;
  if (staged) {
    bl_fence_cta();  // rowq before the rows (the async driver stages them after `ready`)
    staged = vs.rdeg[buf][t] >= 0;
  }
  bl_jitter(p, 22);
  bl_update_one(p, f.q1, f.v0 + t * gridDim.x, f.step_u, src4, &sh.e_task[t],
                staged ? sh.rows[buf][t] : nullptr, staged ? vs.rdeg[buf][t] : 0);
  __syncwarp();
  if (lane == 0) {
#ifdef BL_CHECKED
    sh.chk_upd[t] = f.q1 + 1;
#endif
    bl_jitter(p, 23);
    bl_fence_to_completer(p);  // pend (read by other CTAs after barrier ph)
    if (atomicAdd(&sh.a_udone[s], 1) == f.owned - 1) {
#ifdef BL_PHASE_TS
      sh.ts_upd_a = clock64();
#endif
      bl_fence_cta();
      *(volatile int *)&sh.a_updph = f.ph;
    }
    bl_token(p, sh, f, need);
  }
  __syncwarp();
  return true;
}

template <int T, int TP>
__device__ __forceinline__ void bl_run_async(const BLKParams &p, float4 *src4, float2 *tgt,
                                             float2 *red, BLShared &sh) {
  const int G = gridDim.x, c = blockIdx.x, lane = threadIdx.x & 31;
  const int nb = p.nb;
  const long long ptot = (long long)p.iters * nb;
  const bool mb_stop = p.max_batches > 0 && p.max_batches <= ptot;  // == ptot: as the oracle, iters - 1 done
  const int P = mb_stop ? p.max_batches : (int)ptot;
  const int half = p.red_cap / 2;  // red slots per phase parity
  const volatile BLShared &vs = sh;
  if (threadIdx.x == 0) {
    sh.done_iters = mb_stop ? (P - 1) / nb : p.iters;
    sh.e_prev = 0.0;
    sh.e_acc = 0.0;
    sh.a_updph = -1;
    for (int k = 0; k < 2; ++k) {
      sh.a_unit[k] = sh.a_tok[k] = sh.a_unext[k] = sh.a_udone[k] = sh.a_exit[k] = 0;
      sh.a_gen[k] = k;
      for (int t = 0; t < BL_NTT_MAX; ++t) sh.a_tdone[k][t] = 0;
    }
  }
  if (threadIdx.x < 32) {
    bl_prefetch_targets_warp(p, 0, min(p.b, p.n), tgt);
    if (P > 1) {
      bl_prefetch_targets_warp(p, (1 % nb) * p.b, min(p.b, p.n - (1 % nb) * p.b),
                               tgt + BL_TGT_CAP);
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  }
  __syncthreads();

  double step_u = p.step0;
  int prev_owned = 0;
  bool stop = false;
  unsigned gate_ns = 32, idle_ns = 32;  // spin back-off (ns), capped at p.spin_max
#ifdef BL_PHASE_TS
  // warp-time accounting (profiling builds): 0 entry gate, 1 idle (nothing to
  // grab), 2 dirty wait, 3 units, 4 tile combine, 5 update tasks, 6 control,
  // 7 total; summed over all warps into p.prof[0..7]
  unsigned long long wt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long w0 = clock64(), wl = w0;
#define BL_WT(slot)                      \
  do {                                   \
    const long long t_ = clock64();      \
    wt[slot] += (unsigned long long)(t_ - wl); \
    wl = t_;                             \
  } while (0)
#else
#define BL_WT(slot) \
  do {              \
  } while (0)
#endif
  for (int ph = 0; ph <= P + 1 && !stop; ++ph) {
    const int s = ph & 1;
    BLPhase f;
    f.ph = ph;
    f.P = P;
    f.q1 = ph - 1;
    f.q2 = ph - 2;
    f.owned = 0;
    f.v0 = 0;
    if (f.q1 >= 0 && ph <= P) {
      const int lo1 = (f.q1 % nb) * p.b, hi1 = min(lo1 + p.b, p.n);
      f.v0 = lo1 + ((c - lo1 % G) + G) % G;
      f.owned = f.v0 < hi1 ? (hi1 - 1 - f.v0) / G + 1 : 0;
      if (f.q1 > 0 && f.q1 % nb == 0) step_u = step_u * p.cooling;
    }
    f.step_u = step_u;
    f.tgt_next = tgt + ((ph + 1) & 1) * BL_TGT_CAP;
    // entry gate
    if (ph >= 1) {
      for (;;) {
        if (vs.stop_flag) {
          stop = true;
          break;
        }
        if (vs.a_gen[s] == ph && (ph == 1 || vs.ready >= ph - 1) &&
            (prev_owned == 0 || vs.a_updph >= ph - 1))
          break;
        __nanosleep(gate_ns);
        gate_ns = min(2 * gate_ns, p.spin_max);
      }
      gate_ns = 32;
      BL_WT(0);
      if (stop) break;
      bl_fence_cta();
      BL_CHK(vs.a_gen[s] == ph, BLC_SLOT_GEN, ph, vs.a_gen[s]);
    }
    prev_owned = f.owned;

    const bool has_R = ph < P;
    const int lo = has_R ? (ph % nb) * p.b : 0;
    const int bt = has_R ? min(p.b, p.n - lo) : 0;
    const BLGeom geo = bl_geom(c, G, p.n, f.owned > 0 ? (f.v0 - c) / G : 0, f.owned);
    BLUnits U = {1, 0, 0};
    if (has_R) U = bl_units(bt, T, geo.clean4, geo.d_lo < geo.d_hi, half, p.nsub_max, p.min_unit4);
    const int n_all = has_R ? U.ntt * U.nsub : 0;
    const int n_clean = has_R ? U.ntt * U.nc : 0;
    const int need = (has_R ? U.ntt : 0) + (ph > 0 ? 1 : 0) + f.owned;
    float2 *red_s = red + s * half;
    float2 *part = p.part + (size_t)(ph % 3) * p.b * G;
    const float2 *tgt_s = tgt + s * BL_TGT_CAP;
    const unsigned bar_prev = (unsigned)ph * (unsigned)G;  // barrier ph-1 complete
    auto control = [&]() {
      return ph > 0 && vs.ctrl_claim < ph && bl_try_control(p, f, src4, sh, bar_prev, need);
    };
    for (;;) {
      if (vs.stop_flag) {
        stop = true;
        break;
      }
      BL_WT(1);
      bl_jitter(p, 26);
      if (control()) {
        BL_WT(6);
        idle_ns = 32;
        continue;
      }
      if (bl_try_update_a(p, f, src4, sh, need)) {
        BL_WT(5);
        idle_ns = 32;
        continue;
      }
      int g = n_all;
      if (vs.a_unit[s] < n_all) {
        if (lane == 0) g = atomicAdd(&sh.a_unit[s], 1);
        g = __shfl_sync(0xffffffffu, g, 0);
      }
      if (g < n_all) {
        idle_ns = 32;
        if (g >= n_clean) {
          // dirty sub-range: needs this CTA's updates of batch q1; help until done
          for (;;) {
            if (vs.stop_flag) {
              stop = true;
              break;
            }
            BL_WT(2);
            if (control()) {
              BL_WT(6);
              continue;
            }
            if (bl_try_update_a(p, f, src4, sh, need)) {
              BL_WT(5);
              continue;
            }
            if (vs.a_updph >= ph) break;
            __nanosleep(64);
          }
          BL_WT(2);
          if (stop) break;
          bl_fence_cta();
#ifdef BL_CHECKED
          for (int t = 0; t < f.owned; ++t)
            BL_CHK(((volatile int *)sh.chk_upd)[t] == f.q1 + 1, BLC_DIRTY_EARLY, ph, t);
#endif
        }
        BL_WT(1);
        bl_jitter(p, 25);
        bl_do_unit<T, TP>(p, lo, bt, src4, tgt_s, red_s, part, g, U, geo, ph);
        BL_WT(3);
        const int tile = g % U.ntt;
        __syncwarp();
        int last = 0;
        if (lane == 0) {
          bl_fence_cta();
          last = atomicAdd(&sh.a_tdone[s][tile], 1) == U.nsub - 1;
        }
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last) {
          bl_fence_cta();
          if (U.nsub > 1) {
            const int stride = U.ntt * 32 * T;
#pragma unroll
            for (int k = 0; k < T; ++k) {
              const int idx = tile * 32 * T + k * 32 + lane;
              if (idx < bt) {
                float2 acc = red_s[idx];
                for (int sb = 1; sb < U.nsub; ++sb) {
                  const float2 v = red_s[sb * stride + idx];
                  acc.x += v.x;
                  acc.y += v.y;
                }
                part[(size_t)idx * G + c] = acc;
                if (BL_CHK_ON)
                  p.part_st[(size_t)(part - p.part) + (size_t)idx * G + c] = (unsigned)ph + 1u;
              }
            }
          }
          __syncwarp();
          if (lane == 0) {
            bl_fence_to_completer(p);  // part (read by other CTAs after barrier ph)
            bl_token(p, sh, f, need);
          }
          __syncwarp();
          BL_WT(4);
        }
        continue;
      }
      // nothing left to grab: leave once control is claimed and every update
      // taken; back off exponentially (spinning warps issue integer work on
      // the FMA pipe that the sweeping warps need)
      if ((ph == 0 || vs.ctrl_claim >= ph) && vs.a_unext[s] >= f.owned) break;
      __nanosleep(idle_ns);
      idle_ns = min(2 * idle_ns, p.spin_max);
    }
    idle_ns = 32;
    if (stop) break;
    // leave the phase; the last warp out releases slot s for phase ph+2
    if (lane == 0 && atomicAdd(&sh.a_exit[s], 1) == BL_NW - 1) {
      bl_fence_cta();
      sh.a_unit[s] = sh.a_tok[s] = sh.a_unext[s] = sh.a_udone[s] = 0;
      for (int t = 0; t < BL_NTT_MAX; ++t) sh.a_tdone[s][t] = 0;
      sh.a_exit[s] = 0;
      bl_fence_cta();
      *(volatile int *)&sh.a_gen[s] = ph + 2;
    }
    __syncwarp();
  }
#ifdef BL_PHASE_TS
  BL_WT(1);
  wt[7] = (unsigned long long)(clock64() - w0);
  if (p.prof && lane == 0) {
    for (int k = 0; k < 8; ++k) atomicAdd(p.prof + k, wt[k]);
    atomicAdd(p.prof + 8 + c, wt[3] + wt[4] + wt[5] + wt[6]);  // this CTA's busy warp time
  }
#endif
#undef BL_WT
  __syncthreads();
  if (c == 0 && threadIdx.x == 0) *p.iters_done = sh.done_iters;
}

// ---------------------------------------------------------------------------
// Latency driver (bl_run_lat, BLKParams::pipelined == 3): the per-batch chain
// of small batches (C2-C4: 0.3-2 us of pair work per batch against a grid
// barrier + dependent L2 round trips) with no task queues and no hand-offs
// on it.  Warps 0..U-1 (U = max owned vertices per batch per CTA) are
// updaters, the others sweepers.  Phase q (targets = batch q):
//   sweepers  sweep the CTA's resident sources EXCEPT its owned members of
//             batch q-1, M(q-1), against batch q's targets (read from xy,
//             where batch q is committed: its last update, batch q-nb, was
//             committed in phase q-nb+2 <= q-2), as soon as M(q-2) is
//             applied -- one phase ahead of the chain; tile partials are
//             combined in sub-range order into the clean partial C_q (red,
//             parity q & 1), the targets kept in tgt[q & 1] for D(q);
//   updaters  each loads its next member's CSR row, spins on barrier q-1
//             itself, updates that member of M(q-1) (Alg. 2 for one vertex:
//             partial row, CSR attraction, fp64 step) and joins; the LAST
//             updater to join continues the chain: publishes M(q-1), books
//             the energy, commits M(q-2) to xy, adds the sweep of the dirty
//             float4s (M(q-1)'s slots at their new coordinates) to C_q for
//             every target in fixed order -> part, arrives at barrier q.
// Same values and summation order as the asynchronous driver's (the clean
// sub-ranges in order, then the dirty one).  Needs nb >= 4.
template <int T, int TP, bool LCOOP>
__device__ __forceinline__ void bl_run_lat(const BLKParams &p, float4 *src4, float2 *tgt,
                                           float2 *red, BLShared &sh) {
  const int G = gridDim.x, c = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nb = p.nb;
  const long long ptot = (long long)p.iters * nb;
  const bool mb_stop = p.max_batches > 0 && p.max_batches <= ptot;
  const int P = mb_stop ? p.max_batches : (int)ptot;
  const int half = p.red_cap / 2;
  // updater warps: >= the owned vertices per batch per CTA, >= 4 (D(q)'s
  // target chunks are shared), <= half the warps (host checks the first)
  const int U = min(BL_NW / 2, max(4, (p.b + G - 1) / G));
  const volatile BLShared &vs = sh;
  if (threadIdx.x == 0) {
    sh.done_iters = mb_stop ? (P - 1) / nb : p.iters;
    sh.e_prev = 0.0;
    sh.e_acc = 0.0;
    sh.l_applied = -1;
    sh.l_cleanp[0] = sh.l_cleanp[1] = -1;
    sh.l_dec = -1;
    for (int k = 0; k < 2; ++k) {
      sh.l_join[k] = sh.l_unit[k] = sh.l_exit[k] = sh.l_tiles[k] = 0;
      sh.l_gen[k] = k;
      for (int t = 0; t < BL_NTT_MAX; ++t) sh.l_tdone[k][t] = 0;
    }
  }
  __syncthreads();

  // owned members of batch q in this CTA: v0(q), v0 + G, ... (count m(q))
  auto members = [&](int q, int &v0, int &m) {
    const int lo = (q % nb) * p.b, hi = min(lo + p.b, p.n);
    v0 = lo + ((c - lo % G) + G) % G;
    m = v0 < hi ? (hi - 1 - v0) / G + 1 : 0;
  };

  if (warp >= U) {
    // ---------------- sweepers ----------------
    unsigned ns = 32;
    for (int r = 0; r < P; ++r) {
      const int s = r & 1;
      for (;;) {  // gate: M(r-2) applied, parity slot free
        if (vs.stop_flag) return;
        if (vs.l_applied >= r - 2 && vs.l_gen[s] == r) break;
        __nanosleep(ns);
        ns = min(2 * ns, 256u);
      }
      ns = 32;
      bl_fence_cta();
      int v0 = 0, m = 0;
      if (r >= 1) members(r - 1, v0, m);
      const int lo = (r % nb) * p.b, bt = min(p.b, p.n - lo);
      const BLGeom geo = bl_geom(c, G, p.n, m > 0 ? (v0 - c) / G : 0, m);
      const BLUnits Un = bl_units(bt, T, geo.clean4, true, half, p.nsub_max, p.min_unit4);
      const int n_clean = Un.ntt * Un.nc, stride = Un.ntt * 32 * T;
      float2 *red_s = red + s * half;
      float2 *tgt_s = tgt + s * BL_TGT_CAP;
      for (;;) {
        int g = n_clean;
        if (lane == 0) g = atomicAdd(&sh.l_unit[s], 1);
        g = __shfl_sync(0xffffffffu, g, 0);
        if (g >= n_clean) break;
        bl_jitter(p, 31);
        const int tile = g % Un.ntt, sub = g / Un.ntt;
        float tx[T], ty[T];
        bl_f2 AX[T], AY[T];
#pragma unroll
        for (int k = 0; k < T; ++k) {
          const int idx = tile * 32 * T + k * 32 + lane;
          const float2 t = idx < bt ? __ldcg(p.xy + lo + idx) : make_float2(0.f, 0.f);
          if (sub == 0 && idx < bt) tgt_s[idx] = t;  // for D(r)
          tx[k] = t.x;
          ty[k] = t.y;
          AX[k] = AY[k] = f2pack(0.f, 0.f);
        }
        // (two call sites here: measured 1.6 % faster at C4 than one)
        int seg_lo[2], seg_hi[2], nseg = 0;
        bl_unit_segments(geo, Un.nc, sub, p.guided, seg_lo, seg_hi, nseg);
        // (unroll 2: the small per-phase sweeps of this driver lose with 4)
        if (nseg > 0) bl_sweep_range<T, TP, 2>(src4, seg_lo[0], seg_hi[0], geo.full4, tx, ty, AX, AY, p.r_half);
        if (nseg > 1) bl_sweep_range<T, TP, 2>(src4, seg_lo[1], seg_hi[1], geo.full4, tx, ty, AX, AY, p.r_half);
#pragma unroll
        for (int k = 0; k < T; ++k) {
          const int idx = tile * 32 * T + k * 32 + lane;
          float ax0, ax1, ay0, ay1;
          f2unpack(AX[k], ax0, ax1);
          f2unpack(AY[k], ay0, ay1);
          if (idx < bt) red_s[sub * stride + idx] = make_float2(ax0 + ax1, ay0 + ay1);
        }
        __syncwarp();
        int last = 0;
        if (lane == 0) {
          bl_fence_cta();
          last = atomicAdd(&sh.l_tdone[s][tile], 1) == Un.nc - 1;
        }
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last) {  // combine the tile's clean sub-ranges in order into slot 0
          bl_fence_cta();
          if (Un.nc > 1) {
#pragma unroll
            for (int k = 0; k < T; ++k) {
              const int idx = tile * 32 * T + k * 32 + lane;
              if (idx < bt) {
                float2 acc = red_s[idx];
                for (int sb = 1; sb < Un.nc; ++sb) {
                  const float2 v = red_s[sb * stride + idx];
                  acc.x += v.x;
                  acc.y += v.y;
                }
                red_s[idx] = acc;
              }
            }
          }
          __syncwarp();
          if (lane == 0) {
            bl_fence_cta();
            if (atomicAdd(&sh.l_tiles[s], 1) == Un.ntt - 1) {
              bl_fence_cta();
              *(volatile int *)&sh.l_cleanp[s] = r;
            }
          }
          __syncwarp();
        }
      }
      // leave phase r; the last sweeper out resets parity s for phase r+2
      if (lane == 0 && atomicAdd(&sh.l_exit[s], 1) == BL_NW - U - 1) {
        bl_fence_cta();
        sh.l_unit[s] = sh.l_exit[s] = sh.l_tiles[s] = 0;
        for (int t = 0; t < BL_NTT_MAX; ++t) sh.l_tdone[s][t] = 0;
        bl_fence_cta();
        *(volatile int *)&sh.l_gen[s] = r + 2;
      }
      __syncwarp();
    }
    return;
  }

  // ---------------- updaters ----------------
  // U warps synchronised by the hardware named barrier 1 (bar.sync 1, 32 U):
  // warp 0 alone polls the grid barrier; every updater warp updates at most
  // one member and takes a share of D(q)'s target chunks; warp 0 arrives.
  double step_u = p.step0;
  int *myrow = sh.rows[0][warp];  // this warp's staged CSR row (<= 32 entries)
  const unsigned nthr = 32u * (unsigned)U;
  auto ubar = [&]() { asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory"); };
  for (int q = 0; q <= P; ++q) {
    const int s = q & 1;
    int v0 = 0, m = 0;
    if (q >= 1) {
      members(q - 1, v0, m);
      if (q - 1 > 0 && (q - 1) % nb == 0) step_u = step_u * p.cooling;
    }
#ifdef BL_PHASE_TS
    long long t_det = 0;
#endif
    if (q >= 1) {
      // this warp's member: its CSR row (constant) before the barrier
      int deg = -1;
      if (warp < m) {
        const int v = v0 + warp * G;
        const int k0 = __ldg(p.rowptr + v);
        deg = __ldg(p.rowptr + v + 1) - k0;
        if (deg <= 32 && lane < deg) myrow[lane] = __ldg(p.colidx + k0 + lane);
        if (LCOOP && lane == 0) {  // for the cooperative walk of long rows (read after ubar)
          sh.l_k0[warp] = k0;
          sh.l_deg[warp] = deg;
        }
        __syncwarp();
      }
      if (warp == 0) {
        // barrier q-1 (every CTA's partials of batch q-1)
        const unsigned target = (unsigned)q * (unsigned)G;
        if (lane == 0)
          while ((int)(bl_ld_acquire(p.bar) - target) < 0) {
          }
        __syncwarp();
        // iteration energy of batch q-2's iteration (booked before barrier
        // q-1) and the tol decision, identical in every CTA
        const int q2 = q - 2;
        if (q2 >= 0 && bl_closes_iteration(q2, nb, P)) {
          const int it = q2 / nb;
          const double E = bl_energy_sum_warp(p, it);
          if (c == 0 && lane == 0) p.energy[it] = E;
          if (lane == 0) {
            if (q2 % nb == nb - 1 && q2 < P - 1 && p.tol > 0.0 && it > 0 &&
                fabs(E - sh.e_prev) < p.tol) {
              sh.done_iters = it + 1;
              sh.stop_flag = 1;
            }
            sh.e_prev = E;
          }
        }
      }
      ubar();  // barrier q-1 seen (bar.sync orders warp 0's acquire before the reads below)
#ifdef BL_PHASE_TS
      t_det = clock64();
#endif
      bl_jitter(p, 32);
      // long rows of this CTA's members: all U updater warps walk them
      // together (p.lcoop; a hub's update is the batch's critical path)
      bool coop = false;
      if (LCOOP && vs.stop_flag == 0) {
        for (int t = 0; t < m; ++t) {
          const int dt = vs.l_deg[t];
          if (dt <= BL_LCOOP) continue;
          coop = true;
          const float2 ci = bl_src_get(src4, (v0 + t * G - c) / G);
          const float2 f = bl_long_row_part(p, q - 1, vs.l_k0[t], dt, ci, warp, U);
          if (lane == 0) sh.l_lpart[t][warp] = f;
        }
        if (coop) ubar();  // uniform: every updater warp sees the same degrees
      }
      if (vs.stop_flag == 0 && warp < m) {
        if (LCOOP && coop && deg > BL_LCOOP)
          bl_update_one(p, q - 1, v0 + warp * G, step_u, src4, &sh.e_task[warp], nullptr, 0,
                        sh.l_lpart[warp], U);
        else
          bl_update_one(p, q - 1, v0 + warp * G, step_u, src4, &sh.e_task[warp],
                        deg <= 32 ? myrow : nullptr, deg <= 32 ? deg : 0);
      }
    }
    ubar();  // every member of M(q-1) updated (src4, pend, e_task)
#ifdef BL_PHASE_TS
    const long long t_join = clock64();
#endif
    const bool stop = vs.stop_flag != 0;
    if (stop || q == P) {
      if (warp == 0) {
        if (!stop && q == P) {
          // the last batch's energy: book it, arrive at barrier P, wait for
          // every CTA's, sum (CTA 0 writes the trace)
          if (lane == 0) {
            double e = sh.e_acc;
            for (int i = 0; i < m; ++i) e += sh.e_task[i];
            p.e_cta[(((P - 1) / nb) & 1) * G + c] = e;
            asm volatile("fence.acq_rel.gpu;\n\tred.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(p.bar) : "memory");
            const unsigned target = (unsigned)(P + 1) * (unsigned)G;
            while ((int)(bl_ld_acquire(p.bar) - target) < 0) {
            }
          }
          __syncwarp();
          const double E = bl_energy_sum_warp(p, (P - 1) / nb);
          if (c == 0 && lane == 0) p.energy[(P - 1) / nb] = E;
        }
        // final positions: every owned source (all updates are done: after
        // barrier P, or a stop decided identically everywhere after barrier q-1)
        const int mc = c < p.n ? (p.n - 1 - c) / G + 1 : 0;
        for (int k = lane; k < mc; k += 32) p.xy[c + (size_t)k * G] = bl_src_get(src4, k);
        if (lane == 0) {
          *(volatile int *)&sh.stop_flag = 1;  // release the sweepers
          if (c == 0) *p.iters_done = sh.done_iters;
        }
      }
      break;
    }
    if (warp == 0) {
      // (a) publish M(q-1): sweepers of phase q+1 may start; (b) energy
      if (lane == 0 && q >= 1) {
        *(volatile int *)&sh.l_applied = q - 1;
        double e = sh.e_acc;
        for (int i = 0; i < m; ++i) e += sh.e_task[i];  // task order
        sh.e_acc = e;
        if (bl_closes_iteration(q - 1, nb, P)) {
          p.e_cta[(((q - 1) / nb) & 1) * G + c] = e;
          sh.e_acc = 0.0;
        }
      }
    }
    // (c) commit M(q-2) to xy (read as committed after barrier q)
    if (q >= 2 && warp == U - 1) bl_commit_warp(p, q - 2, src4);
    // (d) D(q): clean partial + the dirty float4s, per target, into part;
    // target chunks of 32 T split over the updater warps
    bl_jitter(p, 33);
    while (vs.l_cleanp[s] != q) {
    }
    bl_fence_cta();
#ifdef BL_PHASE_TS
    const long long t_clean = clock64();
#endif
    {
      const int lo = (q % nb) * p.b, bt = min(p.b, p.n - lo);
      const BLGeom geo = bl_geom(c, G, p.n, m > 0 ? (v0 - c) / G : 0, m);
      const float2 *red_s = red + s * half;
      const float2 *tgt_s = tgt + s * BL_TGT_CAP;
      float2 *part = p.part + (size_t)(q % p.part_nbuf) * p.b * G;
      for (int base = warp * 32 * T; base < bt; base += U * 32 * T) {
        float tx[T], ty[T];
        bl_f2 AX[T], AY[T];
#pragma unroll
        for (int k = 0; k < T; ++k) {
          const int idx = base + k * 32 + lane;
          const float2 t = idx < bt ? tgt_s[idx] : make_float2(0.f, 0.f);
          if (BL_CHK_ON && idx < bt) {  // the sweepers' copy is batch q's committed coordinate
            const float2 w = __ldcg(p.xy + lo + idx);
            BL_CHK(w.x == t.x && w.y == t.y, BLC_LAT_TGT, q, lo + idx);
          }
          tx[k] = t.x;
          ty[k] = t.y;
          AX[k] = AY[k] = f2pack(0.f, 0.f);
        }
        if (geo.d_lo < geo.d_hi)
          bl_sweep_range<T, TP>(src4, geo.d_lo, geo.d_hi, geo.full4, tx, ty, AX, AY, p.r_half);
#pragma unroll
        for (int k = 0; k < T; ++k) {
          const int idx = base + k * 32 + lane;
          if (idx < bt) {
            float ax0, ax1, ay0, ay1;
            f2unpack(AX[k], ax0, ax1);
            f2unpack(AY[k], ay0, ay1);
            float2 acc = red_s[idx];
            if (BL_CHK_ON) {  // the clean partial, recomputed in one pass over the clean slots
              float cx = 0.f, cy = 0.f;
              const float2 tt = tgt_s[idx];
              for (int k4 = 0; k4 < geo.last4; ++k4) {
                if (k4 >= geo.d_lo && k4 < geo.d_hi) continue;
                const float4 q4 = src4[k4];
                const float xs[2] = {q4.x, q4.y}, ys[2] = {q4.z, q4.w};
                for (int h2 = 0; h2 < 2; ++h2) {
                  if (k4 == geo.full4 && h2 == 1) continue;
                  const float dx = xs[h2] - tt.x, dy = ys[h2] - tt.y;
                  const float d2 = fmaf(dx, dx, fmaf(dy, dy, BL_EPS2));
                  cx += dx / d2;
                  cy += dy / d2;
                }
              }
              const float tol = 1e-3f * (fabsf(cx) + fabsf(cy)) + 1e-2f;
              BL_CHK(fabsf(cx - acc.x) + fabsf(cy - acc.y) <= tol, BLC_LAT_CLEAN, q, idx);
            }
            if (geo.d_lo < geo.d_hi) {
              acc.x += ax0 + ax1;
              acc.y += ay0 + ay1;
            }
            part[(size_t)idx * G + c] = acc;
            if (BL_CHK_ON) p.part_st[(size_t)(part - p.part) + (size_t)idx * G + c] = (unsigned)q + 1u;
          }
        }
      }
    }
    bl_jitter(p, 34);
    ubar();  // D(q), the commit and the energy booking are done
    // (e) arrive at barrier q
    if (warp == 0 && lane == 0) {
#ifdef BL_PHASE_TS
      const long long t_d = clock64();
#endif
      asm volatile("fence.acq_rel.gpu;\n\tred.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(p.bar) : "memory");
#ifdef BL_PHASE_TS
      // CTA-0 timeline (async_profile.py, latency driver): previous arrival ->
      // barrier seen -> updates done -> clean partial ready -> D done -> arrival
      const long long t_arr = clock64();
      if (p.prof && c == 0) {
        unsigned long long *hp = p.prof + 8 + G;
        if (q >= 1) {
          hp[0] += (unsigned long long)(t_det - sh.ts_arr_prev);
          hp[1] += (unsigned long long)(t_join - t_det);
          hp[2] += (unsigned long long)(t_clean - t_join);
          hp[3] += (unsigned long long)(t_d - t_clean);
          hp[4] += (unsigned long long)(t_arr - t_d);
          hp[5] += 1ull;
          hp[6] += 1ull;
        }
        sh.ts_arr_prev = t_arr;
      }
#endif
    }
  }
}

template <int NT, int T, int TP>
__global__ void __launch_bounds__(NT, 1) bl_layout_kernel(BLKParams p) {
  extern __shared__ float4 bl_smem[];
  if (p.stop_in && *(const volatile int *)p.stop_in) return;  // uniform: set by an earlier launch
  float4 *src4 = bl_smem;
  float2 *tgt = reinterpret_cast<float2 *>(bl_smem + p.chunk4);
  float2 *red = tgt + 2 * BL_TGT_CAP;
  __shared__ BLShared sh;
  if (threadIdx.x == 0) {
    sh.unit_ctr = 0;
    sh.u_next = 0;
    sh.u_done = 0;
    sh.stop_flag = 0;
    sh.ready = 0;
    sh.ctrl_claim = 0;
    sh.seen = 0;
    sh.rowq[0] = sh.rowq[1] = sh.rowq[2] = -1;
  }
  int *unit_ctr = &sh.unit_ctr;
  double *e_warp = sh.e_warp;

  const int G = gridDim.x, c = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned bar_target = 0;
  BLProf pf;
  pf.init(p);

  // resident source chunk: owned vertices c, c+G, ...; pad with far dummies
  // (Δ ~ 1e30 -> d^2 = inf -> 1/d^2 = 0 -> contributes exactly 0)
  for (int k = threadIdx.x; k < 2 * p.chunk4 && !p.attr_only; k += BL_NT) {
    const long long v = (long long)c + (long long)k * G;
    bl_src_set(src4, k, v < p.n ? __ldcg(p.xy + v) : make_float2(1e30f, 1e30f));
  }
  __syncthreads();

  if (p.forces_mode) {
    double e_dummy = 0.0;
    const BLPerm P0 = bl_perm_make(0ull, 1, p.n, 0, sh.pkey);  // identity
    bl_phase_R<T, TP>(p, p.first, p.count, src4, tgt, red, unit_ctr, pf, P0, sh.ioff);
    bl_grid_sync(p.bar, bar_target, unit_ctr);
    if (p.attr_only) {
      // a5 alone over a range of any size: one thread per vertex sums its
      // items in order (phase U's warp per vertex is built for one batch)
      const int ib = __ldg(p.item_ptr + p.first);
      for (int v = p.first + c * BL_NT + threadIdx.x; v < p.first + p.count; v += G * BL_NT) {
        const int a0 = __ldg(p.item_ptr + v) - ib, a1 = __ldg(p.item_ptr + v + 1) - ib;
        float sx = 0.f, sy = 0.f;
        for (int a = a0; a < a1; ++a) {
          const float2 q = __ldcg(p.attr + a);
          sx += q.x;
          sy += q.y;
        }
        p.f_out[v - p.first] = make_float2(sx, sy);
      }
      return;
    }
    bl_phase_U(p, p.first, p.count, 0.0, src4, e_dummy, P0, sh.ioff);
    return;
  }

  if (p.pipelined == 2) {
    bl_run_async<T, TP>(p, src4, tgt, red, sh);
    return;
  }
  if (p.pipelined == 3) {
    // two instances: the cooperative long-row walk costs the hub-free configs
    // 6 % when merely compiled into their loop (measured at C2 / C3)
    // (only in the small-tile variants, which the latency driver runs by
    // default: the host never sets lcoop for the others)
    if constexpr (T <= 2) {
      if (p.lcoop) {
        bl_run_lat<T, TP, true>(p, src4, tgt, red, sh);
        return;
      }
    }
    bl_run_lat<T, TP, false>(p, src4, tgt, red, sh);
    return;
  }
  if (p.pipelined) {
    bl_run_pipelined<T, TP>(p, src4, tgt, red, sh, pf, bar_target);
    return;
  }

  double step = p.step0;
  double e_acc = 0.0;
  double e_prev = 0.0;
  int batches = 0;
  int it = 0;
  bool stop = false;
  for (; it < p.iters && !stop; ++it) {
    e_acc = 0.0;
    __syncthreads();  // every thread is past the previous iteration's uses of pkey
    const BLPerm P = bl_perm_make(p.shuf_seed, p.shuf_h, p.n, it, sh.pkey);  // pi_it (R1)
    __syncthreads();
    for (int t = 0; t < p.nb; ++t) {
      const int lo = t * p.b;
      const int bt = min(p.b, p.n - lo);
      bl_phase_R<T, TP>(p, lo, bt, src4, tgt, red, unit_ctr, pf, P, sh.ioff, batches);
      bl_grid_sync(p.bar, bar_target, unit_ctr);
      pf.mark(3);
      bl_phase_U(p, lo, bt, step, src4, e_acc, P, sh.ioff, batches);
      pf.mark(4);
      ++batches;
      const bool last = (t == p.nb - 1);
      if (p.max_batches > 0 && batches >= p.max_batches) stop = true;
      if (last || stop) {
        if (lane == 0) e_warp[warp] = e_acc;
        __syncthreads();
        if (threadIdx.x == 0) {
          double e = 0.0;
          for (int w = 0; w < BL_NW; ++w) e += e_warp[w];
          p.e_cta[(it & 1) * G + c] = e;
        }
      }
      bl_grid_sync(p.bar, bar_target, unit_ctr);
      if (P.on) bl_refresh_resident(p, P, lo, bt, src4);
      pf.mark(5);
      if (last || stop) {
        // every CTA reduces the per-CTA energies in the same order, so the
        // convergence decision is identical everywhere
        double E = 0.0;
        for (int cc = 0; cc < G; ++cc) E += __ldcg(p.e_cta + (it & 1) * G + cc);
        if (c == 0 && threadIdx.x == 0) p.energy[it] = E;
        if (!stop && p.tol > 0.0 && it > 0 && fabs(E - e_prev) < p.tol) {
          if (c == 0 && threadIdx.x == 0) *p.iters_done = it + 1;
          pf.flush(p);
          return;
        }
        e_prev = E;
      }
      if (stop) break;
    }
    if (!stop) step = step * p.cooling;
  }
  if (c == 0 && threadIdx.x == 0) *p.iters_done = stop ? it - 1 : it;
  pf.mark(6);
  pf.flush(p);
}
