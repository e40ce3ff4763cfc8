"""ctypes binding of libbl (include/bl.h).  Argument marshalling only: every
step of the layout runs in the CUDA kernels of csrc/.  There is no CPU
fallback -- if libbl.so is missing or cannot load, import fails loudly.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# BL_LIBRARY: another build of the same ABI (same-box A/B measurements only)
_SO = os.environ.get("BL_LIBRARY") or os.path.join(_HERE, "libbl.so")

BL_OK, BL_EINVAL, BL_ENOMEM, BL_ECUDA, BL_ESTATE = 0, -1, -2, -3, -4
BL_REPULSE_NEIGHBORS = 1
BL_ATTRACTION_ONLY = 2
BL_ALGO_EXACT, BL_ALGO_BH = 0, 1


class bl_params(ctypes.Structure):
    _fields_ = [
        ("iters", ctypes.c_int32),
        ("batch", ctypes.c_int32),
        ("K", ctypes.c_float),
        ("C", ctypes.c_float),
        ("step0", ctypes.c_double),
        ("cooling", ctypes.c_double),
        ("tol", ctypes.c_double),
        ("max_batches", ctypes.c_int32),
        ("flags", ctypes.c_uint32),
        ("algo", ctypes.c_int32),
        ("theta", ctypes.c_float),
        ("a", ctypes.c_float),
        ("r", ctypes.c_float),
        ("shuffle_seed", ctypes.c_uint64),
    ]


class BLError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{msg} [status {status}]")
        self.status = status


def _load() -> ctypes.CDLL:
    if not os.path.exists(_SO):
        raise ImportError(
            f"libbl.so not found at {_SO}; build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
    lib = ctypes.CDLL(_SO)
    vp, i32, P = ctypes.c_void_p, ctypes.c_int32, ctypes.POINTER
    lib.bl_params_default.argtypes = [P(bl_params)]
    lib.bl_params_default.restype = None
    lib.bl_create.argtypes = [i32, vp, vp, P(vp)]
    lib.bl_create.restype = ctypes.c_int
    lib.bl_layout.argtypes = [vp, vp, P(bl_params), P(i32)]
    lib.bl_layout.restype = ctypes.c_int
    lib.bl_layout_device.argtypes = [vp, vp, P(bl_params), vp]
    lib.bl_layout_device.restype = ctypes.c_int
    lib.bl_energy.argtypes = [vp, P(ctypes.c_double), vp, i32, P(i32), P(i32)]
    lib.bl_energy.restype = ctypes.c_int
    lib.bl_forces.argtypes = [vp, vp, i32, i32, vp, P(bl_params), vp]
    lib.bl_forces.restype = ctypes.c_int
    lib.bl_max_vertices.argtypes = []
    lib.bl_max_vertices.restype = i32
    lib.bl_last_launch_count.argtypes = [vp]
    lib.bl_last_launch_count.restype = i32
    lib.bl_greedy_init.argtypes = [i32, vp, vp, i32, vp]
    lib.bl_greedy_init.restype = ctypes.c_int
    lib.bl_edge_uniformity.argtypes = [vp, vp, P(ctypes.c_double), vp]
    lib.bl_edge_uniformity.restype = ctypes.c_int
    lib.bl_stress.argtypes = [vp, vp, vp, i32, P(ctypes.c_double), P(ctypes.c_double),
                              P(ctypes.c_longlong), P(ctypes.c_longlong), vp]
    lib.bl_stress.restype = ctypes.c_int
    lib.bl_neighborhood_preservation.argtypes = [vp, vp, vp, i32, P(ctypes.c_double), P(i32), vp]
    lib.bl_neighborhood_preservation.restype = ctypes.c_int
    lib.bl_last_visits.argtypes = [vp, P(ctypes.c_ulonglong)]
    lib.bl_last_visits.restype = ctypes.c_int
    lib.bl_kernel_name.argtypes = [vp]
    lib.bl_kernel_name.restype = ctypes.c_char_p
    lib.bl_driver_name.argtypes = [vp]
    lib.bl_driver_name.restype = ctypes.c_char_p
    lib.bl_microbench.argtypes = [P(ctypes.c_double)]
    lib.bl_microbench.restype = ctypes.c_int
    # debug aids: absent from older builds loaded through BL_LIBRARY (A/B runs)
    if hasattr(lib, "bl_debug_counters"):
        lib.bl_debug_counters.argtypes = [vp, vp]
        lib.bl_debug_counters.restype = i32
    if hasattr(lib, "bl_debug_check"):
        lib.bl_debug_check.argtypes = [vp, vp]
        lib.bl_debug_check.restype = i32
    lib.bl_debug_profile.argtypes = [vp, vp, i32]
    lib.bl_debug_profile.restype = i32
    lib.bl_destroy.argtypes = [vp]
    lib.bl_destroy.restype = None
    lib.bl_status_string.argtypes = [ctypes.c_int]
    lib.bl_status_string.restype = ctypes.c_char_p
    lib.bl_last_error.argtypes = [vp]
    lib.bl_last_error.restype = ctypes.c_char_p
    return lib


lib = _load()

# symbols include/bl.h declares (checked by tests/test_abi.py)
EXPORTS = ("bl_params_default", "bl_greedy_init", "bl_create", "bl_layout", "bl_layout_device", "bl_energy",
           "bl_forces", "bl_max_vertices", "bl_last_launch_count", "bl_last_visits", "bl_kernel_name", "bl_driver_name", "bl_edge_uniformity",
           "bl_stress", "bl_neighborhood_preservation", "bl_microbench",
           "bl_debug_profile", "bl_debug_check", "bl_debug_counters", "bl_destroy", "bl_status_string", "bl_last_error")


def _check(rc: int, h=None):
    if rc != BL_OK:
        msg = lib.bl_last_error(h).decode()
        raise BLError(rc, f"{lib.bl_status_string(rc).decode()}: {msg}")


def _ptr(x) -> int:
    """Raw address of a numpy array, a torch tensor, or an int."""
    if x is None:
        return 0
    if isinstance(x, int):
        return x
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    raise TypeError(f"cannot take the address of {type(x)}")


def bl_params_default(**overrides) -> bl_params:
    p = bl_params()
    lib.bl_params_default(ctypes.byref(p))
    for k, v in overrides.items():
        if not hasattr(p, k):
            raise TypeError(f"unknown parameter {k}")
        setattr(p, k, v)
    return p


def bl_create(n: int, rowptr, colidx) -> int:
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int32).reshape(-1)
    colidx = np.ascontiguousarray(colidx, dtype=np.int32).reshape(-1)
    # the C side reads rowptr[0..n] and colidx[0..rowptr[n]) unconditionally
    if int(n) < 1 or rowptr.size != int(n) + 1:
        raise BLError(BL_EINVAL, f"rowptr must have n+1 = {int(n) + 1} entries (got {rowptr.size})")
    if int(rowptr[-1]) != colidx.size:
        raise BLError(BL_EINVAL, f"colidx must have rowptr[n] = {int(rowptr[-1])} entries "
                                 f"(got {colidx.size})")
    h = ctypes.c_void_p()
    rc = lib.bl_create(int(n), rowptr.ctypes.data, colidx.ctypes.data if colidx.size else 0,
                       ctypes.byref(h))
    if rc != BL_OK:
        raise BLError(rc, f"{lib.bl_status_string(rc).decode()}: {lib.bl_last_error(None).decode()}")
    return h.value


def bl_layout(h: int, xy: np.ndarray, p: bl_params) -> int:
    """Host path: xy is a C-contiguous float32 (n, 2) numpy array, updated in
    place.  Returns the number of completed iterations."""
    if not (isinstance(xy, np.ndarray) and xy.dtype == np.float32 and xy.flags.c_contiguous):
        raise TypeError("xy must be a C-contiguous float32 numpy array")
    done = ctypes.c_int32(0)
    _check(lib.bl_layout(h, xy.ctypes.data, ctypes.byref(p), ctypes.byref(done)), h)
    return done.value


def bl_layout_device(h: int, d_xy, p: bl_params, stream=0) -> None:
    """Device path: d_xy is a device float32 buffer of 2n values (torch tensor
    or raw pointer); stream is a cudaStream_t handle (int) or a torch stream."""
    s = getattr(stream, "cuda_stream", stream)
    _check(lib.bl_layout_device(h, _ptr(d_xy), ctypes.byref(p), s or None), h)


def bl_energy(h: int, trace_len: int = 0):
    """(e_last, trace ndarray[n_written], iters_done)."""
    e = ctypes.c_double(0.0)
    trace = np.zeros(max(trace_len, 1), dtype=np.float64)
    nw = ctypes.c_int32(0)
    done = ctypes.c_int32(0)
    _check(lib.bl_energy(h, ctypes.byref(e), trace.ctypes.data if trace_len else None,
                         int(trace_len), ctypes.byref(nw), ctypes.byref(done)), h)
    return e.value, trace[: nw.value], done.value


def bl_forces(h: int, d_xy, first: int, count: int, d_f_out, p: bl_params, stream=0) -> None:
    s = getattr(stream, "cuda_stream", stream)
    _check(lib.bl_forces(h, _ptr(d_xy), int(first), int(count), _ptr(d_f_out), ctypes.byref(p),
                         s or None), h)


def bl_max_vertices() -> int:
    return int(lib.bl_max_vertices())


def bl_last_launch_count(h: int) -> int:
    return int(lib.bl_last_launch_count(h))


def bl_greedy_init(n: int, rowptr, colidx, root: int = 0) -> np.ndarray:
    """Alg. 3 greedy initial layout (host C++ in libbl); (n, 2) float32."""
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int32)
    colidx = np.ascontiguousarray(colidx, dtype=np.int32)
    out = np.zeros((int(n), 2), dtype=np.float32)
    rc = lib.bl_greedy_init(int(n), rowptr.ctypes.data, colidx.ctypes.data if colidx.size else 0,
                            int(root), out.ctypes.data)
    if rc != BL_OK:
        raise BLError(rc, f"{lib.bl_status_string(rc).decode()}: bl_greedy_init")
    return out


def bl_edge_uniformity(h: int, d_xy, stream=0) -> float:
    s = getattr(stream, "cuda_stream", stream)
    eu = ctypes.c_double(0)
    _check(lib.bl_edge_uniformity(h, _ptr(d_xy), ctypes.byref(eu), s or None), h)
    return eu.value


def bl_stress(h: int, d_xy, sources=None, stream=0):
    """(stress, s*, reachable pairs, unreachable pairs)."""
    s = getattr(stream, "cuda_stream", stream)
    src = None if sources is None else np.ascontiguousarray(sources, dtype=np.int32)
    st, sc = ctypes.c_double(0), ctypes.c_double(0)
    pr, un = ctypes.c_longlong(0), ctypes.c_longlong(0)
    _check(lib.bl_stress(h, _ptr(d_xy), None if src is None else src.ctypes.data,
                         0 if src is None else src.size, ctypes.byref(st), ctypes.byref(sc),
                         ctypes.byref(pr), ctypes.byref(un), s or None), h)
    return st.value, sc.value, pr.value, un.value


def bl_neighborhood_preservation(h: int, d_xy, queries=None, stream=0):
    """(NP, vertices counted)."""
    s = getattr(stream, "cuda_stream", stream)
    q = None if queries is None else np.ascontiguousarray(queries, dtype=np.int32)
    npv = ctypes.c_double(0)
    cnt = ctypes.c_int32(0)
    _check(lib.bl_neighborhood_preservation(h, _ptr(d_xy), None if q is None else q.ctypes.data,
                                            0 if q is None else q.size, ctypes.byref(npv),
                                            ctypes.byref(cnt), s or None), h)
    return npv.value, cnt.value


def bl_last_visits(h: int) -> int:
    v = ctypes.c_ulonglong(0)
    _check(lib.bl_last_visits(h, ctypes.byref(v)), h)
    return int(v.value)


def bl_kernel_name(h: int) -> str:
    return lib.bl_kernel_name(h).decode()


def bl_driver_name(h: int) -> str:
    return lib.bl_driver_name(h).decode()


def bl_microbench():
    r = (ctypes.c_double * 4)()
    _check(lib.bl_microbench(r))
    return {"ffma_per_clk_sm": r[0], "mufu_rcp_per_clk_sm": r[1], "mufu_rsq_per_clk_sm": r[2],
            "ffma2_lane_ops_per_clk_sm": r[3]}


def bl_debug_counters(h: int):
    """(BFS levels, CSR entries examined) of the last bl_stress call, GPU ns of
    the last metric call's kernels."""
    out = np.zeros(4, dtype=np.int64)
    lib.bl_debug_counters(h, out.ctypes.data)
    return int(out[0]), int(out[1]), int(out[2])


def bl_debug_check(h: int):
    """(build kind: 1 checked / 0 production, violation record uint32[8])."""
    out = np.zeros(8, dtype=np.uint32)
    rc = lib.bl_debug_check(h, out.ctypes.data)
    if rc < 0:
        raise BLError(BL_ECUDA, "bl_debug_check failed")
    return rc, out


def bl_debug_profile(h: int, length: int = 8 + 1024):
    out = np.zeros(length, dtype=np.uint64)
    m = lib.bl_debug_profile(h, out.ctypes.data, length)
    return out[:m]


def bl_destroy(h: int) -> None:
    if h:
        lib.bl_destroy(h)
