"""Quality metrics on the GPU (bl_edge_uniformity / bl_stress /
bl_neighborhood_preservation, csrc/bl_metrics.cuh) against the metric oracle
(readings M1-M4).  The nearest-neighbour sets and BFS distances are integer
decisions taken identically, so pair counts and NP agree exactly; the fp64
sums agree to rounding.  Marked gpu."""
import numpy as np
import pytest

import oracle
from blgen import build_config, edges_to_csr, grid_graph, uniform_coords
from tests.gpu_helpers import gpu_layout

pytestmark = pytest.mark.gpu


def _dev(xy):
    import torch
    return torch.from_numpy(np.ascontiguousarray(xy, dtype=np.float32).copy()).cuda()


def _metrics(g, xy, sources=None, queries=None):
    import paper_2002_08233_b200 as bl
    with bl.BatchLayout(g.n, g.rowptr, g.colidx) as lay:
        d = _dev(xy)
        eu = bl.bl_edge_uniformity(lay.h, d)
        st = bl.bl_stress(lay.h, d, sources)
        npv = bl.bl_neighborhood_preservation(lay.h, d, queries)
        again = bl.bl_stress(lay.h, d, sources), bl.bl_neighborhood_preservation(lay.h, d, queries)
    assert again == (st, npv)                                 # bitwise reproducible
    return eu, st, npv


@pytest.mark.parametrize("name,ns,nq", [("C1", None, None), ("C2", 128, 600),
                                        ("C3b256", 64, 500), ("C4", 64, 300), ("C5", 64, 100)])
def test_metrics_match_oracle(name, ns, nq):
    g, xy0, cfg = build_config(name)
    rng = np.random.default_rng(1)
    src = None if ns is None else rng.choice(g.n, ns, replace=False).astype(np.int32)
    qry = None if nq is None else rng.choice(g.n, nq, replace=False).astype(np.int32)
    for xy in (xy0, gpu_layout(g, xy0, iters=2, batch=cfg.batch)[0] if g.n < 100_000 else xy0):
        eu, (st, sc, pr, un), (npv, cnt) = _metrics(g, xy, src, qry)
        r_eu = oracle.edge_uniformity(g.n, g.rowptr, g.colidx, xy)
        r_st, r_sc, r_pr, r_un = oracle.stress(g.n, g.rowptr, g.colidx, xy, src)
        r_np, r_cnt = oracle.neighborhood_preservation(g.n, g.rowptr, g.colidx, xy, qry)
        assert eu == pytest.approx(r_eu, rel=1e-12)
        assert (pr, un) == (r_pr, r_un)
        assert st == pytest.approx(r_st, rel=1e-9, abs=1e-9) and sc == pytest.approx(r_sc, rel=1e-12)
        assert cnt == r_cnt and npv == pytest.approx(r_np, rel=1e-14, abs=1e-15)


def test_metric_edge_cases():
    # ties in the nearest-neighbour selection (duplicated positions), a vertex
    # whose degree exceeds the other vertices' count is impossible, isolated
    # vertices are skipped, a disconnected graph has unreachable pairs
    g = edges_to_csr(7, np.array([0, 0, 1, 4]), np.array([1, 2, 2, 5]))
    xy = np.array([[0, 0], [1, 0], [1, 0], [1, 0], [5, 5], [6, 5], [0, 0]], np.float32)
    eu, (st, sc, pr, un), (npv, cnt) = _metrics(g, xy)
    assert eu == pytest.approx(oracle.edge_uniformity(7, g.rowptr, g.colidx, xy), rel=1e-12)
    r = oracle.stress(7, g.rowptr, g.colidx, xy)
    assert (pr, un) == (r[2], r[3]) and st == pytest.approx(r[0], rel=1e-9, abs=1e-12)
    assert (npv, cnt) == pytest.approx(oracle.neighborhood_preservation(7, g.rowptr, g.colidx, xy), rel=1e-15)


def test_layout_improves_quality():
    """Layout-quality smoke test (SPEC acceptance 9's analogue of Table 4):
    on a 20x20 grid, 500 iterations of the exact GPU layout from the greedy
    initialisation cut the scale-optimised stress of the random initial
    layout by >= 50 %."""
    import paper_2002_08233_b200 as bl
    g = grid_graph(20, 20)
    xr = uniform_coords(g.n, 3) * 20
    xg = bl.bl_greedy_init(g.n, g.rowptr, g.colidx, 0)
    out, _, _ = gpu_layout(g, xg, iters=500, batch=64)
    st0 = oracle.stress(g.n, g.rowptr, g.colidx, xr)[0]
    st1 = _metrics(g, out)[1][0]
    assert st1 <= 0.5 * st0, (st1, st0)


def _mixed_degree_graph(n, seed):
    """A hub joined to every other vertex, a band of vertices of degree ~40-120
    and a sparse remainder: the queries of all three NP kernels (kk <= 32,
    kk <= 256, radix select) in one graph."""
    rng = np.random.default_rng(seed)
    src, dst = [np.zeros(n - 1, np.int64)], [np.arange(1, n)]
    for v in range(1, 40):
        nb = rng.choice(np.arange(1, n), rng.integers(40, 120), replace=False)
        src.append(np.full(nb.size, v))
        dst.append(nb)
    src.append(rng.integers(1, n, 3 * n))
    dst.append(rng.integers(1, n, 3 * n))
    s, d = np.concatenate(src), np.concatenate(dst)
    keep = s != d
    return edges_to_csr(n, s[keep], d[keep])


@pytest.mark.parametrize("lattice", [None, 4, 16])
def test_np_three_paths_with_ties(lattice):
    """NP routed through the one-scan threshold kernels and the radix select
    (kk <= 32 / <= 256 / above), on continuous positions and on coarse integer
    lattices where most squared distances tie (ties by vertex id, M3): the
    counted queries and the NP value agree with the oracle exactly."""
    import paper_2002_08233_b200 as bl
    n = 1500
    g = _mixed_degree_graph(n, 5)
    deg = np.diff(g.rowptr)
    assert deg.max() > 256 and ((deg > 32) & (deg <= 256)).any() and (deg <= 32).any()
    xy = uniform_coords(n, 9)
    if lattice is not None:
        xy = np.floor(xy * lattice).astype(np.float32)
    with bl.BatchLayout(g.n, g.rowptr, g.colidx) as lay:
        d = _dev(xy)
        got = bl.bl_neighborhood_preservation(lay.h, d, None)
        q = np.arange(n - 1, -1, -3, dtype=np.int32)        # an unordered subset
        got_q = bl.bl_neighborhood_preservation(lay.h, d, q)
    ref = oracle.neighborhood_preservation(g.n, g.rowptr, g.colidx, xy)
    ref_q = oracle.neighborhood_preservation(g.n, g.rowptr, g.colidx, xy, q)
    assert got[1] == ref[1] and got[0] == pytest.approx(ref[0], rel=1e-14, abs=1e-15)
    assert got_q[1] == ref_q[1] and got_q[0] == pytest.approx(ref_q[0], rel=1e-14, abs=1e-15)
