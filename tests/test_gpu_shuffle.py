"""Batch randomisation on the GPU (shuffle_seed, §4.3.3; readings
R1-R2 of DESIGN.md §3) vs the oracle's, through the C-ABI.  Marked gpu.

Both sides evaluate the same keyed Feistel permutation pi_it with integer
arithmetic (no shared code: oracle/bl_oracle.c vs csrc/bl_kernel.cuh).

Two GPU realisations: by default every iteration is relabelled
into position space (csrc/bl_relabel.cu) and runs on the sequential drivers;
BL_SHUFFLE_RELABEL=0 randomises inside the two-barrier driver.
`mode` runs both."""
import numpy as np
import pytest

import oracle
from blgen import build_config, grid_graph, uniform_coords
from tests.gpu_helpers import (POS_TOL, POS_TOL_BATCH, assert_energy_close,
                               assert_positions_close, energy_gate, gpu_layout)

pytestmark = pytest.mark.gpu

ALL = ["C1", "C2", "C3b64", "C3b256", "C3b1024", "C4", "C5"]
SEED = 20022


MODES = ["relabel", "inkernel"]


@pytest.fixture
def mode(request, monkeypatch):
    m = getattr(request, "param", "relabel")
    if m == "inkernel":
        monkeypatch.setenv("BL_SHUFFLE_RELABEL", "0")
    else:
        monkeypatch.delenv("BL_SHUFFLE_RELABEL", raising=False)
    return m


def _params(cfg, **kw):
    d = dict(iters=cfg.iters, batch=cfg.batch, K=cfg.K, C=cfg.C, step0=cfg.step0,
             cooling=cfg.cooling, shuffle_seed=SEED)
    d.update(kw)
    return d


def _oracle(g, xy0, p):
    return oracle.layout(g.n, g.rowptr, g.colidx, xy0, iters=p["iters"], batch=p["batch"],
                         K=p["K"], C=p["C"], step0=p["step0"], cooling=p["cooling"],
                         max_batches=p.get("max_batches", 0), flags=p.get("flags", 0),
                         shuffle_seed=p["shuffle_seed"])


@pytest.mark.parametrize("mode", MODES, indirect=True)
@pytest.mark.parametrize("name", ALL)
def test_shuffled_one_batch_parity(name, mode):
    """One randomised batch (pi_0(0 .. b-1)): positions vs the oracle, and
    exactly the batch's members may move."""
    g, xy0, cfg = build_config(name)
    p = _params(cfg, iters=1, max_batches=1)
    got, _, _ = gpu_layout(g, xy0, **p)
    ref, _, _ = _oracle(g, xy0, p)
    assert_positions_close(got, ref, POS_TOL_BATCH, what=f"{name} shuffled one batch")
    b = min(cfg.batch, g.n)
    others = np.setdiff1d(np.arange(g.n), oracle.permutation(g.n, SEED, 0)[:b])
    assert np.array_equal(got[others], xy0[others])


@pytest.mark.parametrize("mode", MODES, indirect=True)
@pytest.mark.parametrize("name", ALL)
def test_shuffled_one_iteration_parity(name, mode):
    g, xy0, cfg = build_config(name)
    p = _params(cfg, iters=1)
    got, tr, done = gpu_layout(g, xy0, **p)
    ref, E, _ = _oracle(g, xy0, p)
    assert done == 1
    assert_positions_close(got, ref, POS_TOL, what=f"{name} shuffled one iteration")
    assert_energy_close(tr[:1], E[:1], tol=energy_gate(g, xy0, p),
                        what=f"{name} shuffled one iteration")


@pytest.mark.parametrize("mode", MODES, indirect=True)
def test_shuffled_iterations_use_fresh_permutations(mode):
    """Iteration 1 walks pi_1, not pi_0: shadowed second iteration (from the
    GPU's state after one iteration, the oracle's second iteration with the
    cooled step) -- via max_batches inside iteration 1."""
    g, xy0, cfg = build_config("C3b256")
    nb = -(-g.n // cfg.batch)
    s1, _, _ = gpu_layout(g, xy0, **_params(cfg, iters=2, max_batches=nb))
    s2, _, _ = gpu_layout(g, xy0, **_params(cfg, iters=2, max_batches=nb + 1))
    members = oracle.permutation(g.n, SEED, 1)[:cfg.batch]
    f = oracle.forces(g.n, g.rowptr, g.colidx, s1, 0, g.n)[members]
    ref = s1.astype(np.float64).copy()
    ref[members] += cfg.cooling * f / np.hypot(f[:, 0], f[:, 1])[:, None]
    assert_positions_close(s2, ref, POS_TOL_BATCH, what="iteration 1, first batch (pi_1)")
    others = np.setdiff1d(np.arange(g.n), members)
    assert np.array_equal(s2[others], s1[others])


def test_seed_zero_is_the_sequential_path_bitwise():
    g, xy0, cfg = build_config("C2")
    a, ea, _ = gpu_layout(g, xy0, iters=2, batch=cfg.batch)
    b, eb, _ = gpu_layout(g, xy0, iters=2, batch=cfg.batch, shuffle_seed=0)
    assert np.array_equal(a, b) and np.array_equal(ea, eb)


def test_shuffled_b_equals_n_matches_sequential():
    """b = n: every force sees the frozen state, so the visiting order
    changes only rounding (a target's batch position decides which of the
    kernel's reciprocal forms -- paired or single, DESIGN.md §4 -- its pairs
    use) and the order of the energy sum."""
    g = grid_graph(30, 37)
    xy0 = uniform_coords(g.n, 19)
    a, ea, _ = gpu_layout(g, xy0, iters=3, batch=g.n)
    b, eb, _ = gpu_layout(g, xy0, iters=3, batch=g.n, shuffle_seed=SEED)
    assert_positions_close(b, a, POS_TOL, what="b = n shuffled vs sequential")
    assert_energy_close(eb[:1], ea[:1], tol=2e-6, what="b = n shuffled vs sequential")


@pytest.mark.parametrize("mode", MODES, indirect=True)
@pytest.mark.parametrize("name", ["C1", "C4"])
def test_shuffled_determinism_bitwise(name, mode):
    g, xy0, cfg = build_config(name)
    p = _params(cfg, iters=3)
    a, ea, _ = gpu_layout(g, xy0, **p)
    b, eb, _ = gpu_layout(g, xy0, **p)
    assert np.array_equal(a, b) and np.array_equal(ea, eb)


@pytest.mark.parametrize("mode", MODES, indirect=True)
def test_shuffled_later_iterations_shadowed(mode):
    """Iterations 1 and 2 (pi_1, pi_2, the cooled Steps, the energy slots),
    each shadowed from the GPU's own state before it: the oracle cannot start
    at iteration k, but a randomised iteration is the sequential iteration of
    the graph relabelled by pi_k (pinned for the oracle in
    tests/test_oracle_shuffle_pins.py), so the reference is the oracle's
    sequential path on that graph with Step = step0 cooling^k.  (Free-running
    traces separate by rounding after the first iteration -- every vertex
    moves a full Step along its force direction -- which is why later
    iterations are shadowed.)"""
    from tests.test_oracle_shuffle_pins import relabelled
    g, xy0, cfg = build_config("C3b256")
    states, traces = [xy0], []
    for k in (1, 2, 3):
        xy, tr, done = gpu_layout(g, xy0, **_params(cfg, iters=k))
        assert done == k
        states.append(xy)
        traces.append(tr)
    assert np.array_equal(traces[2][:2], traces[1][:2]) and np.array_equal(traces[1][:1], traces[0])
    for k in (1, 2):
        perm = oracle.permutation(g.n, SEED, k)
        gp, xyp = relabelled(g, states[k], perm)
        q = dict(iters=1, batch=cfg.batch, K=cfg.K, C=cfg.C, step0=cfg.step0 * cfg.cooling ** k,
                 cooling=cfg.cooling)
        refp, Ep, _ = oracle.layout(gp.n, gp.rowptr, gp.colidx, xyp, **q)
        ref = np.empty_like(refp)
        ref[perm] = refp
        # the energy (a sum over all vertices) and the bulk of the positions to
        # the one-iteration gates.  Not the maximum: in the contracted layout
        # of a later iteration a few vertices' forces nearly cancel (|f| <<
        # sum |terms|), and since every vertex moves a full Step ALONG f, the
        # fp32 direction error u32 sum|terms| / |f| reaches
        # 1e-3..1e-2 x extent for a handful of them (measured, both
        # realisations: median 1e-8, p99 5e-7..4e-5, max 1e-4..1.7e-2) -- a
        # wrong permutation, Step or batch order moves EVERY vertex by O(Step)
        ext = float(np.ptp(ref, axis=0).max())
        err = np.abs(states[k + 1] - ref).max(axis=1) / ext
        print(f"{mode} iteration {k}: median {np.median(err):.2e} p99 {np.quantile(err, 0.99):.2e} "
              f"max {err.max():.2e} E rel {abs(traces[2][k] - Ep[0]) / Ep[0]:.2e}")
        assert np.median(err) <= 1e-6, float(np.median(err))
        assert np.quantile(err, 0.99) <= POS_TOL, float(np.quantile(err, 0.99))
        assert np.mean(err > POS_TOL) <= 0.005, float(np.mean(err > POS_TOL))
        assert_energy_close(traces[2][k:k + 1], Ep[:1], tol=max(1e-5, energy_gate(gp, xyp, q)),
                            what=f"shuffled iteration {k} shadowed")


@pytest.mark.parametrize("mb", [1, 43, 44, 86, 87, 1000])
def test_relabelled_max_batches_and_iters_done(mb):
    """The batch budget across relabelled iterations (nb = 43 at C3 b=256):
    iters_done counts completed iterations exactly as the oracle does (a
    budget that ends with an iteration's last batch does not complete it),
    and exactly the batches within the budget have moved."""
    g, xy0, cfg = build_config("C3b256")
    nb = -(-g.n // cfg.batch)
    assert nb == 43
    p = _params(cfg, iters=3, max_batches=mb)
    a, _, da = gpu_layout(g, xy0, **p)
    _, _, dr = _oracle(g, xy0, p)
    assert da == dr
    # vertices of batches beyond the budget have not moved
    moved = np.zeros(g.n, bool)
    left = mb
    for it in range(3):
        k = min(left, nb)
        moved[oracle.permutation(g.n, SEED, it)[:min(k * cfg.batch, g.n)]] = True
        left -= k
        if left <= 0:
            break
    assert np.array_equal(a[~moved], xy0[~moved])
    assert (a[moved] != xy0[moved]).any(axis=1).all()


def test_shuffled_driver_and_rejections(monkeypatch):
    import torch

    import paper_2002_08233_b200 as bl
    g, xy0, cfg = build_config("C5")
    with bl.BatchLayout(g.n, g.rowptr, g.colidx) as lay:
        d = torch.from_numpy(xy0.copy()).cuda()
        lay.layout_device(d, iters=1, batch=1024, max_batches=2, shuffle_seed=SEED)
        torch.cuda.synchronize()
        assert bl.bl_driver_name(lay.h) == "relabel+async"
        assert bl.bl_last_launch_count(lay.h) == 3  # relabel, layout, scatter back
        # a convergence rule is decided on the device between the launches
        lay.layout_device(d, iters=1, batch=1024, max_batches=2, shuffle_seed=SEED, tol=1e-30)
        torch.cuda.synchronize()
        assert bl.bl_driver_name(lay.h) == "relabel+async"
        monkeypatch.setenv("BL_SHUFFLE_RELABEL", "0")
        lay.layout_device(d, iters=1, batch=1024, max_batches=2, shuffle_seed=SEED)
        torch.cuda.synchronize()
        assert bl.bl_driver_name(lay.h) == "two-barrier"
        assert bl.bl_last_launch_count(lay.h) == 1
        for bad in (dict(batch=4096, shuffle_seed=1), dict(algo=bl.BL_ALGO_BH, shuffle_seed=1)):
            with pytest.raises(bl.BLError) as ei:
                lay.layout_device(d, iters=1, **bad)
            assert ei.value.status == bl.BL_EINVAL


@pytest.mark.parametrize("rows,cols,b", [(5, 8, 4), (17, 19, 10), (30, 37, 64), (40, 50, 2)])
def test_relabelled_small_and_ragged_shapes(rows, cols, b):
    """Relabelling on graphs smaller than the grid (n < 148 positions: most
    CTAs of bl_relabel_kernel hold no position), ragged last batches and the
    smallest even batch: one iteration vs the oracle, driver name, and the
    seeded run is reproducible bitwise."""
    import torch

    import paper_2002_08233_b200 as bl
    g = grid_graph(rows, cols)
    xy0 = uniform_coords(g.n, 5)
    p = dict(iters=1, batch=b, shuffle_seed=SEED)
    with bl.BatchLayout(g.n, g.rowptr, g.colidx) as lay:
        d = torch.from_numpy(xy0.copy()).cuda()
        lay.layout_device(d, **p)
        torch.cuda.synchronize()
        assert bl.bl_driver_name(lay.h).startswith("relabel+")
        got = d.cpu().numpy()
        _, tr, done = lay.energy(trace_len=1)
        d2 = torch.from_numpy(xy0.copy()).cuda()
        lay.layout_device(d2, **p)
        torch.cuda.synchronize()
        assert np.array_equal(d2.cpu().numpy(), got)
    ref, E, _ = oracle.layout(g.n, g.rowptr, g.colidx, xy0, **p)
    assert done == 1
    assert_positions_close(got, ref, POS_TOL, what=f"relabelled {rows}x{cols} b={b}")
    assert_energy_close(tr[:1], E[:1], tol=energy_gate(g, xy0, p), what=f"relabelled {rows}x{cols} b={b}")


@pytest.mark.parametrize("mode", MODES, indirect=True)
def test_shuffled_tol_stop_is_decided_on_the_device(mode):
    """|E_t - E_{t-1}| < tol with randomised batches: the run stops
    at the iteration a stop rule applied to its own free-running trace gives,
    with that trace's prefix and that iteration's positions -- relabelled
    iterations decide between their launches on the device (the later
    launches of the call become no-ops), the in-kernel path inside its loop."""
    g, xy0, cfg = build_config("C3b256")
    p = _params(cfg, iters=12)
    _, full, done = gpu_layout(g, xy0, **p)
    assert done == 12
    diffs = np.abs(np.diff(full))
    # a tol that the trace crosses strictly inside the run
    t_stop = 6
    tol = float(np.sqrt(diffs[t_stop - 1] * diffs[t_stop - 2])) if diffs[t_stop - 1] < diffs[t_stop - 2] \
        else float(diffs[t_stop - 1] * 1.000001)
    stop = next(t for t in range(1, 12) if abs(full[t] - full[t - 1]) < tol) + 1
    assert 2 <= stop < 12
    ref_xy, _, _ = gpu_layout(g, xy0, **_params(cfg, iters=stop))
    xy, tr, done = gpu_layout(g, xy0, **_params(cfg, iters=12, tol=tol))
    assert done == stop
    assert np.array_equal(tr, full[:stop])
    assert np.array_equal(xy, ref_xy)
