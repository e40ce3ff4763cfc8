"""BatchLayoutBH on the GPU (bl_bh_kernel through the C-ABI, algo = BL_ALGO_BH)
against the BH oracle (oracle/bl_oracle_bh.h).  Marked gpu.

Both sides take the structural decisions -- box, Morton codes, the tree, the
MAC -- in fp32 with the same operations (reading B7), so from the same fp32
state they build the same tree and visit the same nodes: the visit count
must match EXACTLY, forces and positions to the north-star tolerance.
Within an iteration the GPU's fp32 state and the oracle's fp64 state drift
apart by rounding, which can flip a later MAC decision, so iteration-level
parity is checked per batch from the GPU's own state (shadowing), as for
the C5 exact test.  DESIGN.md §6.
"""
import numpy as np
import pytest

import oracle
from blgen import build_config, edges_to_csr, grid_graph, rmat_graph, uniform_coords
from tests.gpu_helpers import (assert_energy_close, assert_positions_close, extent, gpu_forces,
                               gpu_layout)

pytestmark = pytest.mark.gpu

BH = 1  # BL_ALGO_BH


def _bh(**kw):
    d = dict(algo=BH, theta=1.2)
    d.update(kw)
    return d


def _force_bound(g, xy, first, count, f_ref):
    """1e-4 x the sum of term magnitudes (sum_j 1/d_ij + sum_nbr d) + 1e-5 |f|."""
    x = xy.astype(np.float64)
    b = np.empty(count)
    for t in range(count):
        i = first + t
        d = np.hypot(x[:, 0] - x[i, 0], x[:, 1] - x[i, 1])
        d[i] = np.inf
        nb = g.colidx[g.rowptr[i]:g.rowptr[i + 1]]
        b[t] = 1e-4 * (np.sum(1.0 / d) + np.sum(d[nb] ** 2)) + 1e-5 * np.hypot(*f_ref[t])
    return b


@pytest.mark.parametrize("name,theta", [("C1", 1.2), ("C1", 0.0), ("C4", 1.2), ("C4", 0.5),
                                        ("C5", 1.2)])
def test_forces_and_visits_match_oracle(name, theta):
    g, xy0, cfg = build_config(name)
    first, count = (0, g.n) if g.n <= 2048 else (g.n // 3, 512)
    got, visits = gpu_forces(g, xy0, first, count, with_visits=True, **_bh(theta=theta))
    ref, ref_visits = oracle.bh_forces(g.n, g.rowptr, g.colidx, xy0, xy0, first, count,
                                       theta=theta)
    assert visits == ref_visits                      # same tree, same MAC decisions
    err = np.hypot(*(got - ref).T)
    bound = _force_bound(g, xy0, first, count, ref)
    bad = np.nonzero(err > bound)[0]
    assert bad.size == 0, (bad[:5], err[bad[:5]], bound[bad[:5]])


@pytest.mark.parametrize("name", ["C1", "C2", "C3b256", "C4", "C5"])
def test_one_batch_parity(name):
    g, xy0, cfg = build_config(name)
    p = dict(iters=1, batch=cfg.batch, max_batches=1)
    got, _, _ = gpu_layout(g, xy0, **p, **_bh())
    ref, _, _, _ = oracle.bh_layout(g.n, g.rowptr, g.colidx, xy0, iters=1, batch=cfg.batch,
                                    max_batches=1)
    assert_positions_close(got, ref, what=f"BH {name} one batch")
    b = min(cfg.batch, g.n)
    assert np.array_equal(got[b:], xy0[b:])


@pytest.mark.parametrize("name,sample", [("C1", None), ("C3b1024", None),
                                         ("C4", (0, 1, 64, 127)), ("C5", (0, 1, 130, 255))])
def test_one_iteration_shadowed_per_batch(name, sample):
    """Iteration parity, batch by batch: the GPU's state after t batches (and
    the iteration-start state the tree is built from) goes to the oracle,
    which computes batch t; compared with the GPU's state after t+1."""
    g, xy0, cfg = build_config(name)
    b = min(cfg.batch, g.n)
    nb = -(-g.n // b)
    for t in (sample or range(nb)):
        s_t = xy0 if t == 0 else gpu_layout(g, xy0, iters=1, batch=b, max_batches=t, **_bh())[0]
        s_t1 = gpu_layout(g, xy0, iters=1, batch=b, max_batches=t + 1, **_bh())[0]
        lo, hi = t * b, min((t + 1) * b, g.n)
        assert np.array_equal(s_t1[:lo], s_t[:lo]) and np.array_equal(s_t1[hi:], s_t[hi:])
        f, _ = oracle.bh_forces(g.n, g.rowptr, g.colidx, xy0, s_t, lo, hi - lo)
        ref = s_t.astype(np.float64).copy()
        ref[lo:hi] += f / np.hypot(f[:, 0], f[:, 1])[:, None]
        assert_positions_close(s_t1, ref, what=f"BH {name} batch {t}")


@pytest.mark.parametrize("name", ["C1", "C3b256"])
def test_theta_zero_is_the_exact_method(name):
    """theta = 0 (reading B5): GPU BatchLayoutBH == the exact oracle with
    neighbour repulsion, one full iteration (no MAC decision to flip)."""
    g, xy0, cfg = build_config(name)
    got, tr, _ = gpu_layout(g, xy0, iters=1, batch=cfg.batch, **_bh(theta=0.0))
    ref, E, _ = oracle.layout(g.n, g.rowptr, g.colidx, xy0, iters=1, batch=cfg.batch,
                              flags=oracle.REPULSE_NEIGHBORS)
    assert_positions_close(got, ref, what=f"BH theta=0 {name}")
    assert_energy_close(tr[:1], E[:1], what=f"BH theta=0 {name}")


def test_small_graph_free_running_iterations():
    """A small graph where no decision flips over a few iterations: the free
    run matches the oracle's own BH run (positions and energies)."""
    g = grid_graph(12, 12)
    xy0 = uniform_coords(g.n, 21)
    got, tr, done = gpu_layout(g, xy0, iters=3, batch=50, **_bh())
    ref, E, _, _ = oracle.bh_layout(g.n, g.rowptr, g.colidx, xy0, iters=3, batch=50)
    assert done == 3
    assert_positions_close(got, ref, what="BH 12x12 x3")
    assert_energy_close(tr[:1], E[:1], what="BH 12x12 iteration 0")
    np.testing.assert_allclose(tr, E, rtol=1e-3)  # iterations 1-2: free-running


def test_determinism_bitwise():
    g, xy0, cfg = build_config("C4")
    a, ea, _ = gpu_layout(g, xy0, iters=2, batch=cfg.batch, **_bh())
    b, eb, _ = gpu_layout(g, xy0, iters=2, batch=cfg.batch, **_bh())
    assert np.array_equal(a, b) and np.array_equal(ea, eb)


def test_degenerate_and_edge_cases():
    # n = 1
    g1 = edges_to_csr(1, np.array([], np.int64), np.array([], np.int64))
    got, tr, done = gpu_layout(g1, np.array([[0.5, 0.25]], np.float32), iters=2, batch=3, **_bh())
    assert np.array_equal(got, [[0.5, 0.25]]) and done == 2 and np.all(tr == 0)
    # all coincident: one multi-vertex leaf; no force, no move
    g = grid_graph(8, 9)
    xy0 = np.full((g.n, 2), 0.5, np.float32)
    got, tr, _ = gpu_layout(g, xy0, iters=2, batch=16, **_bh())
    assert np.array_equal(got, xy0) and np.all(tr == 0)
    # duplicated points + ragged batches + b > n
    g = rmat_graph(10, 6, 0.57, 0.19, 0.19, seed=8)
    xy0 = uniform_coords(g.n, 8)
    xy0[1::7] = xy0[0:-1:7][: xy0[1::7].shape[0]]
    for b in (100, 5000):
        p = dict(iters=1, batch=b, max_batches=1)
        got, _, _ = gpu_layout(g, xy0, **p, **_bh())
        ref, _, _, _ = oracle.bh_layout(g.n, g.rowptr, g.colidx, xy0, iters=1, batch=b,
                                        max_batches=1)
        assert_positions_close(got, ref, what=f"BH dup b={b}")


def test_stops_iters_done_and_energy_trace():
    g = grid_graph(10, 10)
    xy0 = uniform_coords(g.n, 2)
    _, _, done = gpu_layout(g, xy0, iters=3, batch=30, max_batches=6, **_bh())
    _, _, rdone, _ = oracle.bh_layout(g.n, g.rowptr, g.colidx, xy0, iters=3, batch=30,
                                      max_batches=6)
    assert done == rdone == 1
    _, full, _ = gpu_layout(g, xy0, iters=60, batch=100, cooling=0.95, **_bh())
    tol = float(np.abs(np.diff(full)).min()) * 1.0001
    stop = next(t for t in range(1, 60) if abs(full[t] - full[t - 1]) < tol) + 1
    _, tr, done = gpu_layout(g, xy0, iters=60, batch=100, cooling=0.95, tol=tol, **_bh())
    assert done == stop and np.array_equal(tr, full[:stop])
    got, _, _ = gpu_layout(g, xy0, iters=0, batch=10, **_bh())
    assert np.array_equal(got, xy0)


def test_exact_path_unchanged_by_algo_field():
    """algo = BL_ALGO_EXACT still runs the exact kernel (0 visits)."""
    import torch

    import paper_2002_08233_b200 as bl
    g, xy0, cfg = build_config("C1")
    with bl.BatchLayout(g.n, g.rowptr, g.colidx) as lay:
        d = torch.from_numpy(xy0.copy()).cuda()
        lay.layout_device(d, iters=1, batch=256, algo=0)
        torch.cuda.synchronize()
        assert bl.bl_last_visits(lay.h) == 0
        lay.layout_device(d, iters=1, batch=256, algo=BH)
        torch.cuda.synchronize()
        assert bl.bl_last_visits(lay.h) > 0
        with pytest.raises(bl.BLError):
            lay.layout_device(d, iters=1, batch=256, algo=7)
        with pytest.raises(bl.BLError):
            lay.layout_device(d, iters=1, batch=256, algo=BH, theta=-1.0)


def test_C6_million_vertices_shadowed():
    """2^20 vertices (C6), the size class where the paper runs only
    BatchLayoutBH: batches 0, 1 and 700 of the first iteration from the GPU's
    own state against the oracle, and the exact visit count of batch 0."""
    g, xy0, cfg = build_config("C6")
    b = cfg.batch
    for t in (0, 1, 700):
        s_t = xy0 if t == 0 else gpu_layout(g, xy0, iters=1, batch=b, max_batches=t, **_bh())[0]
        s_t1 = gpu_layout(g, xy0, iters=1, batch=b, max_batches=t + 1, **_bh())[0]
        lo, hi = t * b, (t + 1) * b
        assert np.array_equal(s_t1[:lo], s_t[:lo]) and np.array_equal(s_t1[hi:], s_t[hi:])
        f, _ = oracle.bh_forces(g.n, g.rowptr, g.colidx, xy0, s_t, lo, hi - lo)
        ref = s_t.astype(np.float64).copy()
        ref[lo:hi] += f / np.hypot(f[:, 0], f[:, 1])[:, None]
        assert_positions_close(s_t1, ref, what=f"BH C6 batch {t}")
    got, visits = gpu_forces(g, xy0, 0, b, with_visits=True, **_bh())
    _, ref_visits = oracle.bh_forces(g.n, g.rowptr, g.colidx, xy0, xy0, 0, b)
    assert visits == ref_visits


@pytest.mark.parametrize("name,theta", [("C3b256", 1.2), ("C4", 1.2), ("C4", 0.5)])
def test_layout_visits_one_iteration(name, theta):
    """Layout mode precomputes every vertex's walk at the iteration start
    (accepted cells fixed per iteration, leaves later at live coordinates,
    reading B5); vertices whose leaf list overflows walk the tree in their
    batch.  Either way each vertex's Alg. S2 walk of iteration 0 is the
    oracle's: the node-visit totals match exactly, and the positions after
    the iteration's first batch too."""
    import torch

    import paper_2002_08233_b200 as bl
    g, xy0, cfg = build_config(name)
    with bl.BatchLayout(g.n, g.rowptr, g.colidx) as lay:
        d = torch.from_numpy(xy0.copy()).cuda()
        lay.layout_device(d, iters=1, batch=cfg.batch, **_bh(theta=theta))
        torch.cuda.synchronize()
        visits = bl.bl_last_visits(lay.h)
    _, _, _, ref_visits = oracle.bh_layout(g.n, g.rowptr, g.colidx, xy0, iters=1,
                                           batch=cfg.batch, theta=theta)
    assert visits == ref_visits
    got, _, _ = gpu_layout(g, xy0, iters=1, batch=cfg.batch, max_batches=1, **_bh(theta=theta))
    ref, _, _, _ = oracle.bh_layout(g.n, g.rowptr, g.colidx, xy0, iters=1, batch=cfg.batch,
                                    max_batches=1, theta=theta)
    assert_positions_close(got, ref, what=f"BH {name} theta {theta} one batch")


def test_precompute_off_matches(monkeypatch):
    """BL_BH_PRE=0 (every vertex walks the tree in its batch) and the default
    precomputation agree on one batch to the tolerance (summation order
    differs) and on the iteration's visit total exactly."""
    import torch

    import paper_2002_08233_b200 as bl
    g, xy0, cfg = build_config("C4")
    out = {}
    for pre in ("1", "0"):
        monkeypatch.setenv("BL_BH_PRE", pre)
        with bl.BatchLayout(g.n, g.rowptr, g.colidx) as lay:
            d = torch.from_numpy(xy0.copy()).cuda()
            lay.layout_device(d, iters=1, batch=cfg.batch, max_batches=1, **_bh())
            torch.cuda.synchronize()
            out[pre] = d.cpu().numpy()
    assert_positions_close(out["1"], out["0"].astype(np.float64), what="precompute on/off")


@pytest.mark.parametrize("name,iters", [("C4", 2), ("C2", 3), ("C5", 1)])
def test_prefetch_across_the_barrier_is_bitwise_neutral(name, iters, monkeypatch):
    """BL_BH_PRE2 (default on): a batch vertex's iteration-constant inputs are
    loaded between the arrival at the grid barrier and the wait, and batches
    without split rows skip the item pass -- the same terms in the same order,
    so positions, energy trace and visit count are bitwise those of the
    unprefetched loop (BL_BH_PRE2=0).  C4 / C2 have split (hub) rows in their
    first batches and none later."""
    import torch

    import paper_2002_08233_b200 as bl
    g, xy0, cfg = build_config(name)
    out = {}
    for pre2 in ("1", "0"):
        monkeypatch.setenv("BL_BH_PRE2", pre2)
        with bl.BatchLayout(g.n, g.rowptr, g.colidx) as lay:
            d = torch.from_numpy(xy0.copy()).cuda()
            lay.layout_device(d, iters=iters, batch=cfg.batch, **_bh())
            torch.cuda.synchronize()
            _, tr, done = lay.energy(trace_len=iters)
            out[pre2] = (d.cpu().numpy(), tr, done, bl.bl_last_visits(lay.h))
    assert out["1"][2] == out["0"][2] == iters
    assert np.array_equal(out["1"][0], out["0"][0])
    assert np.array_equal(out["1"][1], out["0"][1])
    assert out["1"][3] == out["0"][3]
