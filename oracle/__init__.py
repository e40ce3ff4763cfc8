"""Python face of the C oracle (oracle/bl_oracle.c).

TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` legs are the only callers.  The product
package `paper_2002_08233_b200` never imports this module, and this module
never imports the product package.

Functions mirror the paper's operations (§2.2, Alg. 1
P:542-569, Alg. 2); see bl_oracle.c for the header and DESIGN.md
§3 for the readings.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bl_oracle.c")
_IMPL = os.path.join(_HERE, "bl_oracle_impl.h")
_BH = os.path.join(_HERE, "bl_oracle_bh.h")
_INIT = os.path.join(_HERE, "bl_oracle_init.h")
_METRICS = os.path.join(_HERE, "bl_oracle_metrics.h")
_SO = os.path.join(_HERE, "libbl_oracle.so")
_lock = threading.Lock()
_lib = None

REPULSE_NEIGHBORS = 1


def build(force: bool = False) -> str:
    """Compile the oracle with gcc: -O2 -ffp-contract=off, no fast-math."""
    newest = max(os.path.getmtime(_SRC), os.path.getmtime(_IMPL), os.path.getmtime(_BH),
                 os.path.getmtime(_INIT), os.path.getmtime(_METRICS))
    if not force and os.path.exists(_SO) and os.path.getmtime(_SO) >= newest:
        return _SO
    tmp = _SO + f".tmp{os.getpid()}"
    cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC",
           "-shared", "-std=c11", "-o", tmp, _SRC, "-lm"]
    subprocess.run(cmd, check=True)
    os.replace(tmp, _SO)
    return _SO


def _load():
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        lib = ctypes.CDLL(build())
        i32, u32, dbl, flt = ctypes.c_int32, ctypes.c_uint32, ctypes.c_double, ctypes.c_float
        vp = ctypes.c_void_p
        for sfx, R in (("f64", dbl), ("f32", flt)):
            f = getattr(lib, f"oracle_layout_{sfx}")
            f.argtypes = [i32, vp, vp, vp, i32, i32, R, R, dbl, dbl, i32, dbl, u32, vp, vp, ctypes.c_int,
                          ctypes.c_uint64]
            f.restype = ctypes.c_int
            f = getattr(lib, f"oracle_forces_{sfx}")
            f.argtypes = [i32, vp, vp, vp, i32, i32, R, R, u32, vp, ctypes.c_int]
            f.restype = ctypes.c_int
            f = getattr(lib, f"oracle_apply_update_{sfx}")
            f.argtypes = [vp, R, R, R, vp]
            f.restype = ctypes.c_int
        lib.oracle_max_threads.restype = ctypes.c_int
        lib.oracle_permutation.argtypes = [i32, ctypes.c_uint64, i32, vp]
        lib.oracle_permutation.restype = ctypes.c_int
        lib.oracle_mix64.argtypes = [ctypes.c_uint64]
        lib.oracle_mix64.restype = ctypes.c_uint64
        ll = ctypes.c_longlong
        lib.oracle_bh_forces.argtypes = [i32, vp, vp, vp, vp, i32, i32, dbl, dbl, dbl, vp, vp]
        lib.oracle_bh_forces.restype = ctypes.c_int
        lib.oracle_bh_layout.argtypes = [i32, vp, vp, vp, i32, i32, dbl, dbl, dbl, dbl, dbl, i32,
                                         dbl, vp, vp, vp]
        lib.oracle_bh_layout.restype = ctypes.c_int
        lib.oracle_bh_tree.argtypes = [i32, vp, i32] + [vp] * 10
        lib.oracle_bh_tree.restype = ctypes.c_int
        lib.oracle_set_model.argtypes = [dbl, dbl]
        lib.oracle_set_model.restype = None
        lib.oracle_stress.argtypes = [i32, vp, vp, vp, vp, i32, vp, vp, vp, vp]
        lib.oracle_stress.restype = ctypes.c_int
        lib.oracle_edge_uniformity.argtypes = [i32, vp, vp, vp, vp]
        lib.oracle_edge_uniformity.restype = ctypes.c_int
        lib.oracle_neighborhood_preservation.argtypes = [i32, vp, vp, vp, vp, i32, vp, vp, vp]
        lib.oracle_neighborhood_preservation.restype = ctypes.c_int
        lib.oracle_greedy_init.argtypes = [i32, vp, vp, i32, vp]
        lib.oracle_greedy_init.restype = ctypes.c_int
        del ll
        _lib = lib
        return lib


class _model:
    """Set the (a, r)-energy model exponents for one call (reading C15)."""

    def __init__(self, a, r):
        self.a, self.r = float(a), float(r)

    def __enter__(self):
        _lock.acquire()
        _lib.oracle_set_model(self.a, self.r)

    def __exit__(self, *exc):
        _lib.oracle_set_model(2.0, -1.0)
        _lock.release()


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _csr(rowptr, colidx):
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int32)
    colidx = np.ascontiguousarray(colidx, dtype=np.int32)
    if colidx.size == 0:
        colidx = np.zeros(1, dtype=np.int32)  # valid pointer, never read
    return rowptr, colidx


def max_threads() -> int:
    return int(_load().oracle_max_threads())


def layout(n, rowptr, colidx, xy0, *, iters, batch, K=1.0, C=1.0, step0=1.0,
           cooling=0.999, max_batches=0, tol=0.0, flags=0, threads=0, precision="f64",
           a=2.0, r=-1.0, shuffle_seed=0):
    """Run Alg. 2 from xy0 ((n,2) any float dtype; converted to the oracle's
    precision).  shuffle_seed != 0: batch randomisation (readings R1-R2).
    Returns (xy (n,2), energy[iters] fp64, iters_done)."""
    lib = _load()
    dt = np.float64 if precision == "f64" else np.float32
    xy = np.ascontiguousarray(np.asarray(xy0, dtype=dt).reshape(n, 2)).copy()
    rowptr, colidx = _csr(rowptr, colidx)
    energy = np.zeros(max(iters, 1), dtype=np.float64)
    done = ctypes.c_int32(0)
    fn = getattr(lib, f"oracle_layout_{precision}")
    with _model(a, r):
        rc = fn(n, _ptr(rowptr), _ptr(colidx), _ptr(xy), iters, batch, K, C, step0, cooling,
                max_batches, tol, flags, _ptr(energy), ctypes.byref(done), threads,
                int(shuffle_seed) & 0xFFFFFFFFFFFFFFFF)
    if rc != 0:
        raise ValueError("oracle_layout: invalid arguments")
    return xy, energy[:int(done.value) if tol > 0 else iters], int(done.value)


def permutation(n, seed, it):
    """pi_it of batch randomisation (readings R1-R2): int32 (n,)."""
    lib = _load()
    out = np.zeros(max(int(n), 1), np.int32)
    if lib.oracle_permutation(int(n), int(seed) & 0xFFFFFFFFFFFFFFFF, int(it), _ptr(out)) != 0:
        raise ValueError("oracle_permutation: invalid arguments")
    return out[:int(n)]


def mix64(z):
    """The splitmix64 finaliser behind pi_it (for its known-answer pin)."""
    return int(_load().oracle_mix64(int(z) & 0xFFFFFFFFFFFFFFFF))


def forces(n, rowptr, colidx, xy, first=0, count=None, *, K=1.0, C=1.0, flags=0,
           threads=0, precision="f64", a=2.0, r=-1.0):
    """f(i, c) of §2.2 for i in [first, first+count) at state xy; (count, 2)."""
    lib = _load()
    if count is None:
        count = n - first
    dt = np.float64 if precision == "f64" else np.float32
    c = np.ascontiguousarray(np.asarray(xy, dtype=dt).reshape(n, 2))
    rowptr, colidx = _csr(rowptr, colidx)
    out = np.zeros((max(count, 1), 2), dtype=dt)
    fn = getattr(lib, f"oracle_forces_{precision}")
    with _model(a, r):
        rc = fn(n, _ptr(rowptr), _ptr(colidx), _ptr(c), first, count, K, C, flags, _ptr(out),
                threads)
    if rc != 0:
        raise ValueError("oracle_forces: invalid arguments")
    return out[:count]


def apply_update(ci, f, step, precision="f64"):
    """c_i + step * f/||f|| (Alg. 1 line 12); returns (new c_i, ||f||^2)."""
    lib = _load()
    dt = np.float64 if precision == "f64" else np.float32
    c = np.ascontiguousarray(np.asarray(ci, dtype=dt).reshape(2)).copy()
    q = np.zeros(1, dtype=dt)
    getattr(lib, f"oracle_apply_update_{precision}")(_ptr(c), float(f[0]), float(f[1]), float(step), _ptr(q))
    return c, float(q[0])


# ------------------------------------------------------------ BatchLayoutBH
THETA_PAPER = 1.2  # MAC threshold


def bh_layout(n, rowptr, colidx, xy0, *, iters, batch, K=1.0, C=1.0, step0=1.0, cooling=0.999,
              theta=THETA_PAPER, max_batches=0, tol=0.0, a=2.0, r=-1.0):
    """Alg. S3 (BatchLayoutBH) from xy0.  Returns (xy (n,2) fp64, energy,
    iters_done, node visits)."""
    lib = _load()
    xy = np.ascontiguousarray(np.asarray(xy0, dtype=np.float64).reshape(n, 2)).copy()
    rowptr, colidx = _csr(rowptr, colidx)
    energy = np.zeros(max(iters, 1), dtype=np.float64)
    done = ctypes.c_int32(0)
    visits = ctypes.c_longlong(0)
    with _model(a, r):
        rc = lib.oracle_bh_layout(n, _ptr(rowptr), _ptr(colidx), _ptr(xy), iters, batch, K, C,
                                  step0, cooling, theta, max_batches, tol, _ptr(energy),
                                  ctypes.byref(done), ctypes.byref(visits))
    if rc != 0:
        raise ValueError("oracle_bh_layout: invalid arguments")
    return xy, energy[:int(done.value) if tol > 0 else iters], int(done.value), int(visits.value)


def bh_forces(n, rowptr, colidx, snap, live, first=0, count=None, *, K=1.0, C=1.0,
              theta=THETA_PAPER, a=2.0, r=-1.0):
    """Forces of Alg. S3 lines 13-19 for [first, first+count): tree built from
    `snap` (rounded to fp32), live coordinates `live`.  Returns ((count,2)
    fp64, node visits)."""
    lib = _load()
    if count is None:
        count = n - first
    s = np.ascontiguousarray(np.asarray(snap, dtype=np.float32).reshape(n, 2))
    c = np.ascontiguousarray(np.asarray(live, dtype=np.float64).reshape(n, 2))
    rowptr, colidx = _csr(rowptr, colidx)
    out = np.zeros((max(count, 1), 2), dtype=np.float64)
    visits = ctypes.c_longlong(0)
    with _model(a, r):
        rc = lib.oracle_bh_forces(n, _ptr(rowptr), _ptr(colidx), _ptr(s), _ptr(c), first, count,
                                  K, C, theta, _ptr(out), ctypes.byref(visits))
    if rc != 0:
        raise ValueError("oracle_bh_forces: invalid arguments")
    return out[:count], int(visits.value)


def bh_tree(xy):
    """The quadtree of Alg. S1 for fp32 coordinates xy (n,2), pre-order.
    Returns a dict of node arrays plus the sorted codes, permutation and D."""
    lib = _load()
    xy = np.ascontiguousarray(np.asarray(xy, dtype=np.float32))
    n = xy.shape[0]
    cap = 17 * n + 1
    a = {k: np.zeros(cap, np.int32) for k in ("level", "start", "count", "nchild")}
    child = np.zeros(4 * cap, np.int32)
    cx = np.zeros(cap, np.float32)
    cy = np.zeros(cap, np.float32)
    codes = np.zeros(n, np.uint32)
    perm = np.zeros(n, np.int32)
    D = ctypes.c_float(0)
    nn = lib.oracle_bh_tree(n, _ptr(xy), cap, _ptr(a["level"]), _ptr(a["start"]), _ptr(a["count"]),
                            _ptr(a["nchild"]), _ptr(child), _ptr(cx), _ptr(cy), _ptr(codes),
                            _ptr(perm), ctypes.byref(D))
    if nn < 0:
        raise ValueError("oracle_bh_tree failed")
    out = {k: v[:nn] for k, v in a.items()}
    out.update(child=child[:4 * nn].reshape(nn, 4), cx=cx[:nn], cy=cy[:nn], codes=codes,
               perm=perm, D=float(D.value))
    return out


# ------------------------------------------------------------ greedy init
def greedy_init(n, rowptr, colidx, root=0):
    """Alg. 3 (greedy initialisation) with readings G1-G4; (n, 2) float32."""
    lib = _load()
    rowptr, colidx = _csr(rowptr, colidx)
    out = np.zeros((n, 2), np.float32)
    if lib.oracle_greedy_init(n, _ptr(rowptr), _ptr(colidx), int(root), _ptr(out)) != 0:
        raise ValueError("oracle_greedy_init: invalid arguments")
    return out


# ------------------------------------------------------------ quality metrics (§3.7)
def stress(n, rowptr, colidx, xy, sources=None):
    """M1: (scale-optimised stress, optimal scale s*, reachable ordered pairs,
    unreachable pairs) over sources (all vertices if None)."""
    lib = _load()
    rowptr, colidx = _csr(rowptr, colidx)
    c = np.ascontiguousarray(np.asarray(xy, np.float32).reshape(n, 2))
    src = None if sources is None else np.ascontiguousarray(sources, np.int32)
    st, sc = ctypes.c_double(0), ctypes.c_double(0)
    pr, un = ctypes.c_longlong(0), ctypes.c_longlong(0)
    rc = lib.oracle_stress(n, _ptr(rowptr), _ptr(colidx), _ptr(c),
                           None if src is None else _ptr(src), 0 if src is None else src.size,
                           ctypes.byref(st), ctypes.byref(sc), ctypes.byref(pr), ctypes.byref(un))
    if rc != 0:
        raise ValueError("oracle_stress: invalid arguments")
    return st.value, sc.value, pr.value, un.value


def edge_uniformity(n, rowptr, colidx, xy):
    """M2."""
    lib = _load()
    rowptr, colidx = _csr(rowptr, colidx)
    c = np.ascontiguousarray(np.asarray(xy, np.float32).reshape(n, 2))
    eu = ctypes.c_double(0)
    if lib.oracle_edge_uniformity(n, _ptr(rowptr), _ptr(colidx), _ptr(c), ctypes.byref(eu)) != 0:
        raise ValueError("oracle_edge_uniformity: invalid arguments")
    return eu.value


def neighborhood_preservation(n, rowptr, colidx, xy, queries=None, per_vertex=False):
    """M3: (NP, vertices counted[, per-query Jaccard])."""
    lib = _load()
    rowptr, colidx = _csr(rowptr, colidx)
    c = np.ascontiguousarray(np.asarray(xy, np.float32).reshape(n, 2))
    q = None if queries is None else np.ascontiguousarray(queries, np.int32)
    nq = n if q is None else q.size
    jac = np.zeros(max(nq, 1), np.float64)
    npv = ctypes.c_double(0)
    cnt = ctypes.c_int32(0)
    rc = lib.oracle_neighborhood_preservation(n, _ptr(rowptr), _ptr(colidx), _ptr(c),
                                              None if q is None else _ptr(q),
                                              0 if q is None else q.size, ctypes.byref(npv),
                                              ctypes.byref(cnt), _ptr(jac))
    if rc != 0:
        raise ValueError("oracle_neighborhood_preservation: invalid arguments")
    if per_vertex:
        return npv.value, cnt.value, jac[:nq]
    return npv.value, cnt.value
