"""The single-cluster exact kernel (csrc/bl_cluster.cuh, chosen for small
graphs: b n <= BL_CLUSTER_PAIRS) and the whole-GPU kernel on the same small
cases: both against the oracle, and the dispatch itself.  Marked gpu."""
import numpy as np
import pytest

import oracle
from blgen import (build_config, cycle_graph, edges_to_csr, grid_graph, rmat_graph,
                   uniform_coords)
from tests.gpu_helpers import assert_energy_close, assert_positions_close, gpu_layout

pytestmark = pytest.mark.gpu


def _kernel_used(g, xy0, **p):
    import torch

    import paper_2002_08233_b200 as bl
    with bl.BatchLayout(g.n, g.rowptr, g.colidx) as lay:
        d = torch.from_numpy(np.ascontiguousarray(xy0, np.float32).copy()).cuda()
        lay.layout_device(d, **p)
        torch.cuda.synchronize()
        return bl.bl_kernel_name(lay.h)


@pytest.mark.parametrize("driver", ["cluster", "grid"])
@pytest.mark.parametrize("name", ["C1", "C2", "C3b64"])
def test_small_configs_both_kernels(name, driver, monkeypatch):
    monkeypatch.setenv("BL_CLUSTER", "1" if driver == "cluster" else "0")
    monkeypatch.setenv("BL_CLUSTER_PAIRS", "100000000")   # force it regardless of the size rule
    g, xy0, cfg = build_config(name)
    p = dict(iters=1, batch=cfg.batch)
    assert _kernel_used(g, xy0, **p).startswith(
        "bl_cluster_kernel" if driver == "cluster" else "bl_layout_kernel")
    for q in (dict(p, max_batches=1), p):
        got, tr, _ = gpu_layout(g, xy0, **q)
        ref, E, _ = oracle.layout(g.n, g.rowptr, g.colidx, xy0, **q)
        assert_positions_close(got, ref, what=f"{name} {driver} {q}")
        if "max_batches" not in q:
            assert_energy_close(tr[:1], E[:1], what=f"{name} {driver} one iteration")


CASES = [  # (graph, batch, extra params)
    ("grid_odd", 7, {}),                     # odd n: padded slot; ragged batches
    ("grid_odd", 1, {}),                     # one target per batch
    ("grid_odd", 1000, {}),                  # b > n
    ("rmat", 96, {"flags": 1}),
    ("rmat", 200, {"K": 1.7, "C": 0.4, "step0": 0.3, "cooling": 0.9}),
    ("rmat", 64, {"a": 1.0, "r": -2.0, "max_batches": 1}),  # general-r sweep (one batch:
                                             # steep models are ill-conditioned)
    ("rmat", 1024, {}),                      # slice 64: two targets per lane
]


def _graph(kind):
    if kind == "grid_odd":
        return grid_graph(9, 13)              # 117 vertices
    return rmat_graph(10, 6, 0.57, 0.19, 0.19, seed=11)


@pytest.mark.parametrize("case", CASES)
def test_cluster_edge_cases(case, monkeypatch):
    monkeypatch.setenv("BL_CLUSTER", "1")
    monkeypatch.setenv("BL_CLUSTER_PAIRS", "100000000")
    kind, b, extra = case
    g = _graph(kind)
    xy0 = uniform_coords(g.n, 17)
    p = dict(iters=1, batch=b, **extra)
    assert _kernel_used(g, xy0, **p).startswith("bl_cluster_kernel")
    got, tr, _ = gpu_layout(g, xy0, **p)
    ref, E, _ = oracle.layout(g.n, g.rowptr, g.colidx, xy0, **p)
    assert_positions_close(got, ref, what=f"cluster {case}")
    if "max_batches" not in extra:
        assert_energy_close(tr[:1], E[:1], what=f"cluster {case}")


def test_cluster_stops_determinism_and_degenerate(monkeypatch):
    monkeypatch.setenv("BL_CLUSTER", "1")
    g = grid_graph(10, 10)
    xy0 = uniform_coords(g.n, 2)
    a, ea, _ = gpu_layout(g, xy0, iters=5, batch=30)
    b, eb, _ = gpu_layout(g, xy0, iters=5, batch=30)
    assert np.array_equal(a, b) and np.array_equal(ea, eb)
    _, _, done = gpu_layout(g, xy0, iters=3, batch=30, max_batches=6)
    _, _, rdone = oracle.layout(g.n, g.rowptr, g.colidx, xy0, iters=3, batch=30, max_batches=6)
    assert done == rdone == 1
    got, _, _ = gpu_layout(g, xy0, iters=3, batch=30, max_batches=6)
    ref, _, _ = oracle.layout(g.n, g.rowptr, g.colidx, xy0, iters=3, batch=30, max_batches=6)
    assert_positions_close(got, ref, what="cluster max_batches")
    c = cycle_graph(8)
    th = 2 * np.pi * np.arange(8) / 8
    x8 = np.stack([np.cos(th), 1.1 * np.sin(th)], 1).astype(np.float32)
    _, full, _ = gpu_layout(c, x8, iters=400, batch=8, cooling=0.98)
    stop = next(t for t in range(1, 400) if abs(full[t] - full[t - 1]) < 1e-3) + 1
    _, tr, done = gpu_layout(c, x8, iters=400, batch=8, cooling=0.98, tol=1e-3)
    assert done == stop and np.array_equal(tr, full[:stop])
    g1 = edges_to_csr(1, np.array([], np.int64), np.array([], np.int64))
    got, tr, done = gpu_layout(g1, np.array([[0.5, 0.5]], np.float32), iters=2, batch=3)
    assert np.array_equal(got, [[0.5, 0.5]]) and done == 2 and np.all(tr == 0)
    xs = np.full((g.n, 2), 0.3, np.float32)
    got, tr, _ = gpu_layout(g, xs, iters=2, batch=16)
    assert np.array_equal(got, xs) and np.all(tr == 0)


def test_cluster_and_grid_agree(monkeypatch):
    g, xy0, cfg = build_config("C1")
    monkeypatch.setenv("BL_CLUSTER", "1")
    a, ea, _ = gpu_layout(g, xy0, iters=1, batch=cfg.batch)
    monkeypatch.setenv("BL_CLUSTER", "0")
    b, eb, _ = gpu_layout(g, xy0, iters=1, batch=cfg.batch)
    assert_positions_close(a, b, what="cluster vs grid")
    assert_energy_close(ea, eb, tol=2 * 1e-6, what="cluster vs grid")


def test_dispatch_rule():
    """Default rule: the cluster kernel when b n <= 1e6 pairs per batch."""
    g, xy0, cfg = build_config("C1")                  # 256 x 1024
    assert _kernel_used(g, xy0, iters=1, batch=cfg.batch).startswith("bl_cluster_kernel")
    g, xy0, cfg = build_config("C3b256")              # 256 x 11000
    assert _kernel_used(g, xy0, iters=1, batch=cfg.batch).startswith("bl_layout_kernel")
