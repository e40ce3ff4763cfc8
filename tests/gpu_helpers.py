"""Shared helpers for the -m gpu tests: run the CUDA path through the C-ABI
and compare with the oracle.  Tolerances are derived in DESIGN.md §6."""
import numpy as np

# north star: "max position error <= 1e-4 x layout extent (fp32)"
POS_TOL = 1e-4


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


def assert_positions_close(got, ref, tol=POS_TOL, what=""):
    ext = extent(ref)
    err = float(np.abs(np.asarray(got, np.float64) - ref).max())
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
        worst = max(worst, assert_positions_close(got, ref, tol, what=f"iteration {t}"))
        assert abs(tr[0] - E[0]) <= 1e-3 * E[0] + 1e-30, (t, tr[0], E[0])
        state = got
        step = step * cooling
    return worst
