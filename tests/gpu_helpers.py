"""Shared helpers for the -m gpu tests: run the CUDA path through the C-ABI
and compare with the oracle.  Tolerances are derived in DESIGN.md §6.

BL_PARITY_LOG=<file>: every comparison appends one JSON line (what, the
measured error, the gate) -- the margins behind DESIGN.md §6's table."""
import json
import os

import numpy as np

# north star: "max position error <= 1e-4 x layout extent (fp32)" -- one full
# iteration and shadowed iterations (chaotic amplification inside the
# iteration)
POS_TOL = 1e-4
# one batch update: no propagation, error = Step x the direction error of
# fp32 forces
POS_TOL_BATCH = 1e-5
# energy of one batch / one iteration / one shadowed iteration, relative
# (fp32 chunked sums, fp64 energy accumulation)
E_TOL = 1e-6
# the same with (a, r)-model powers through lg2/ex2.approx
E_TOL_POW = 1e-5
U32 = 2.0 ** -24  # fp32 unit roundoff


def _log(what, kind, value, gate):
    path = os.environ.get("BL_PARITY_LOG")
    if path:
        with open(path, "a") as fh:
            fh.write(json.dumps({"test": os.environ.get("PYTEST_CURRENT_TEST", "").split(" ")[0],
                                 "what": what, "kind": kind, "value": float(value),
                                 "gate": float(gate)}) + "\n")


def energy_gate(g, state, params, oracle_layout=None):
    """Energy gate of ONE iteration from `state`: E_TOL, or
    twice the fp32 arithmetic floor of that very iteration when larger --
    |E_f32 - E_f64| / E_f64 of the oracle run in fp32 (sequential sums,
    longer chains than the kernel's) -- because inside an iteration every
    batch sees the rounding of the batches before it, amplified by close
    encounters (1/d^2 force gradients); with many dependent batches (b = 1 on
    a small graph) that floor reaches 1e-4.  Skipped above 20,000 vertices
    (the large configs' floors are < 3e-7)."""
    import oracle
    if g.n > 20000:
        return E_TOL
    q = dict(params)
    kw = dict(iters=1, batch=q["batch"], K=q.get("K", 1.0), C=q.get("C", 1.0),
              step0=q.get("step0", 1.0), cooling=q.get("cooling", 0.999),
              flags=q.get("flags", 0), a=q.get("a", 2.0), r=q.get("r", -1.0),
              shuffle_seed=q.get("shuffle_seed", 0))
    _, e64, _ = oracle.layout(g.n, g.rowptr, g.colidx, state, **kw)
    _, e32, _ = oracle.layout(g.n, g.rowptr, g.colidx, state, precision="f32", **kw)
    floor = abs(e32[0] - e64[0]) / e64[0] if e64[0] > 0 else 0.0
    _log("fp32 floor of the iteration", "energy_fp32_floor", floor, E_TOL)
    return max(E_TOL, 2.0 * floor)


def assert_energy_close(got, ref, tol=E_TOL, what=""):
    """|E_gpu - E_oracle| <= tol x E_oracle for every entry (E = 0 exactly
    when every force is 0, compared exactly)."""
    got = np.atleast_1d(np.asarray(got, np.float64))
    ref = np.atleast_1d(np.asarray(ref, np.float64))
    assert got.shape == ref.shape, (got.shape, ref.shape)
    rel = np.where(ref > 0, np.abs(got - ref) / np.where(ref > 0, ref, 1.0), np.abs(got - ref))
    worst = float(rel.max()) if rel.size else 0.0
    _log(what, "energy_rel", worst, tol)
    assert worst <= tol, f"{what}: energy rel. diff {worst:.3e} > {tol:g} ({got} vs {ref})"
    return worst


def extent(xy):
    """Reading C13: max(max x - min x, max y - min y) of the reference layout."""
    xy = np.asarray(xy, dtype=np.float64)
    return float(np.ptp(xy, axis=0).max())


def gpu_layout(g, xy0, *, device_path=True, **params):
    """Run the layout on the GPU; returns (xy fp32 (n,2), energy trace, iters_done)."""
    import torch

    import paper_2002_08233_b200 as bl
    iters = int(params.get("iters", 1))
    with bl.BatchLayout(g.n, g.rowptr, g.colidx) as lay:
        if device_path:
            d = torch.from_numpy(np.ascontiguousarray(xy0, dtype=np.float32).copy()).cuda()
            lay.layout_device(d, **params)
            torch.cuda.synchronize()
            xy = d.cpu().numpy()
        else:
            xy, _ = lay.layout(xy0, **params)
        if iters == 0:
            return xy, np.zeros(0), 0
        try:
            _, trace, done = lay.energy(trace_len=iters)
        except bl.BLError:
            trace, done = np.zeros(0), 0
    return xy, trace, done


def gpu_forces(g, xy, first=0, count=None, with_visits=False, **params):
    import torch

    import paper_2002_08233_b200 as bl
    with bl.BatchLayout(g.n, g.rowptr, g.colidx) as lay:
        d = torch.from_numpy(np.ascontiguousarray(xy, dtype=np.float32).copy()).cuda()
        f = lay.forces(d, first, count, **params)
        torch.cuda.synchronize()
        out = f.cpu().numpy().astype(np.float64)
        if with_visits:
            return out, bl.bl_last_visits(lay.h)
        return out


def assert_positions_close(got, ref, tol=POS_TOL, what="", ext=None):
    """max |got - ref| <= tol x extent (reading C13: the extent of the
    reference layout, or of the whole layout `ext` when comparing a part)."""
    ext = extent(ref) if ext is None else ext
    err = float(np.abs(np.asarray(got, np.float64) - ref).max())
    _log(what, "pos_over_extent", err / ext if ext > 0 else err, tol)
    assert err <= tol * ext, f"{what}: max |dxy| = {err:.3e} > {tol:g} x extent {ext:.4g}"
    return err / ext


def shadow_check(g, xy0, iters, oracle_layout, tol=POS_TOL, **params):
    """Per-iteration shadowing: from the GPU's own state
    x_t (fp32 bytes), one GPU iteration with step0 = step_t is compared with
    one oracle iteration from the same bytes.  Chaos-immune, so it can run
    for many iterations.  Returns the worst err/extent."""
    step = float(params.pop("step0", 1.0))
    cooling = float(params.get("cooling", 0.999))
    state = np.ascontiguousarray(xy0, dtype=np.float32)
    worst = 0.0
    for t in range(iters):
        p = dict(params, iters=1, step0=step)
        got, tr, _ = gpu_layout(g, state, **p)
        ref, E, _ = oracle_layout(g, state, p)
        worst = max(worst, assert_positions_close(got, ref, tol, what=f"shadowed iteration {t}"))
        assert_energy_close(tr[:1], E[:1], tol=energy_gate(g, state, p),
                            what=f"shadowed iteration {t}")
        state = got
        step = step * cooling
    return worst
