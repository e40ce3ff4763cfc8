"""(a, r)-energy models on the GPU (reading C15; §2.2): the exact
kernel (r = -1 keeps the packed paired-reciprocal sweep, other r run the
two-MUFU sweep variant) and the BH kernel against the oracle.  Marked gpu."""
import numpy as np
import pytest

import oracle
from blgen import build_config, cycle_graph
from tests.gpu_helpers import (E_TOL, E_TOL_POW, assert_energy_close, assert_positions_close,
                               gpu_forces, gpu_layout)

pytestmark = pytest.mark.gpu

MODELS = [(1.0, -1.0), (0.0, -1.0), (3.0, -1.0), (2.0, -2.0), (1.5, -0.5), (2.0, -3.0)]


@pytest.mark.parametrize("ar", MODELS)
@pytest.mark.parametrize("name", ["C1", "C3b256", "C4"])
def test_exact_batches_shadowed(ar, name):
    """One batch from the seeded state, then batches t of the first iteration
    from the GPU's own state after t batches (shadowing).  Free-running whole
    iterations are not compared for the steep models: with r <= -2 a vertex
    between two very close neighbours has a force that is a small difference
    of huge terms, so fp32-vs-fp64 state rounding after the first batch can
    turn its direction (the chaos of DESIGN.md §6, at batch scale)."""
    a, r = ar
    g, xy0, cfg = build_config(name)
    b = cfg.batch
    nb = -(-g.n // b)
    for t in sorted({0, 1, nb // 2, nb - 1}):
        s_t = xy0 if t == 0 else gpu_layout(g, xy0, iters=1, batch=b, max_batches=t, a=a, r=r)[0]
        s_t1 = gpu_layout(g, xy0, iters=1, batch=b, max_batches=t + 1, a=a, r=r)[0]
        lo, hi = t * b, min((t + 1) * b, g.n)
        f = oracle.forces(g.n, g.rowptr, g.colidx, s_t, lo, hi - lo, a=a, r=r)
        ref = s_t.astype(np.float64).copy()
        ref[lo:hi] += f / np.hypot(f[:, 0], f[:, 1])[:, None]
        assert_positions_close(s_t1, ref, what=f"{name} (a,r)={ar} batch {t}")


@pytest.mark.parametrize("ar", [(1.0, -1.0), (0.0, -1.0), (3.0, -1.0), (1.5, -0.5)])
@pytest.mark.parametrize("name", ["C1", "C3b256"])
def test_exact_one_iteration_free_running(ar, name):
    a, r = ar
    g, xy0, cfg = build_config(name)
    got, tr, _ = gpu_layout(g, xy0, iters=1, batch=cfg.batch, a=a, r=r)
    ref, E, _ = oracle.layout(g.n, g.rowptr, g.colidx, xy0, iters=1, batch=cfg.batch, a=a, r=r)
    assert_positions_close(got, ref, what=f"{name} (a,r)={ar} one iteration")
    # r != -1 / non-integer a: pair weights through lg2/ex2.approx (abs. error
    # ~2^-22 in the exponent, x |h| <= 2: ~2^-21 relative per term)
    tol = E_TOL if (r == -1.0 and a in (0.0, 1.0, 2.0, 3.0)) else E_TOL_POW
    assert_energy_close(tr[:1], E[:1], tol=tol, what=f"{name} (a,r)={ar} one iteration")


@pytest.mark.parametrize("ar", [(1.0, -1.0), (2.0, -2.0)])
def test_forces(ar):
    a, r = ar
    g, xy0, cfg = build_config("C4")
    got = gpu_forces(g, xy0, 700, 256, a=a, r=r)
    ref = oracle.forces(g.n, g.rowptr, g.colidx, xy0, 700, 256, a=a, r=r)
    scale = np.abs(ref).max()
    assert np.abs(got - ref).max() <= 2e-4 * scale


@pytest.mark.parametrize("ar", [(1.0, -1.0), (2.0, -2.0), (0.0, -1.0)])
@pytest.mark.parametrize("name", ["C1", "C4"])
def test_bh_one_batch(ar, name):
    a, r = ar
    g, xy0, cfg = build_config(name)
    p = dict(iters=1, batch=cfg.batch, max_batches=1)
    got, _, _ = gpu_layout(g, xy0, algo=1, theta=1.2, a=a, r=r, **p)
    ref, _, _, _ = oracle.bh_layout(g.n, g.rowptr, g.colidx, xy0, theta=1.2, a=a, r=r, **p)
    assert_positions_close(got, ref, what=f"BH {name} (a,r)={ar}")


def test_cycle_closed_form_general_model_on_gpu():
    a, r, n, K, C = 1.0, -2.0, 6, 1.2, 0.8
    ks = np.arange(2, n - 1)
    S = np.sum((np.sin(np.pi * ks / n) / np.sin(np.pi / n)) ** (r + 1))
    ell = (C * K ** 3 / 2 * S) ** (1 / (a - r))
    g = cycle_graph(n)
    th = 2 * np.pi * np.arange(n) / n + 0.03 * np.sin(np.arange(n))
    xy0 = (ell / (2 * np.sin(np.pi / n)) * np.stack([np.cos(th), np.sin(th)], 1)).astype(np.float32)
    got, _, _ = gpu_layout(g, xy0, iters=3000, batch=1, K=K, C=C, cooling=0.99, a=a, r=r)
    edge = np.hypot(*(got - np.roll(got, -1, 0)).T)
    np.testing.assert_allclose(edge, ell, rtol=1e-4)


def test_model_parameter_validation():
    import paper_2002_08233_b200 as bl
    g, xy0, cfg = build_config("C1")
    with bl.BatchLayout(g.n, g.rowptr, g.colidx) as lay:
        for bad in (dict(a=-0.5), dict(a=5.0), dict(r=1.0), dict(r=-3.5)):
            with pytest.raises(bl.BLError):
                lay.layout(xy0, iters=1, **bad)
