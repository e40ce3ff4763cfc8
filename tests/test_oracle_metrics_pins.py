"""Pins of the quality-metric oracle (§3.7; readings
M1-M4 of DESIGN.md §3): hand-derived cases, an
independent implementation on random graphs (scipy's shortest paths and
numpy sorting instead of the oracle's BFS and qsort), and the invariances
the definitions imply."""
import numpy as np
import pytest
from scipy.sparse import csr_matrix
from scipy.sparse.csgraph import shortest_path

import oracle
from blgen import cycle_graph, edges_to_csr, grid_graph, uniform_coords


def _g(n, edges):
    e = np.array(edges, np.int64).reshape(-1, 2)
    return edges_to_csr(n, e[:, 0], e[:, 1])


def test_stress_single_pair_scales_perfectly():
    """one edge at layout distance 1 -> stress 0, s* = 1; at
    distance 2 -> s* = 0.5, stress 0 (both ordered pairs counted, M1)."""
    g = _g(2, [(0, 1)])
    st, sc, pairs, un = oracle.stress(2, g.rowptr, g.colidx, [[0, 0], [1, 0]])
    assert (st, sc, pairs, un) == (0.0, 1.0, 2, 0)
    st, sc, _, _ = oracle.stress(2, g.rowptr, g.colidx, [[0, 0], [2, 0]])
    assert st == pytest.approx(0.0, abs=1e-15) and sc == 0.5


def test_stress_path_matches_scale_scan():
    """path 0-1-2 at (0,0), (1,0), (1.5,0): the closed-form minimum
    equals a brute-force scan over s (step 1e-5 around the optimum)."""
    g = _g(3, [(0, 1), (1, 2)])
    xy = np.array([[0, 0], [1, 0], [1.5, 0]], np.float64)
    st, sc, _, _ = oracle.stress(3, g.rowptr, g.colidx, xy)
    d = np.array([[0, 1, 2], [1, 0, 1], [2, 1, 0]], float)
    L = np.abs(xy[:, None, 0] - xy[None, :, 0])
    off = ~np.eye(3, dtype=bool)
    s = np.arange(0.5, 2.0, 1e-5)
    vals = [np.sum((si * L[off] - d[off]) ** 2 / d[off] ** 2) for si in s]
    assert st > 0 and st == pytest.approx(min(vals), rel=1e-6)
    assert sc == pytest.approx(s[int(np.argmin(vals))], abs=2e-5)


def test_stress_optimum_beats_perturbed_scales():
    g = grid_graph(6, 7)
    xy = uniform_coords(g.n, 3).astype(np.float64) * 5
    st, sc, pairs, _ = oracle.stress(g.n, g.rowptr, g.colidx, xy)
    D = shortest_path(csr_matrix((np.ones(g.nnz), g.colidx, g.rowptr), shape=(g.n, g.n)),
                      unweighted=True)
    L = np.hypot(*(xy[:, None, :] - xy[None, :, :]).transpose(2, 0, 1))
    off = ~np.eye(g.n, dtype=bool)
    for f in (0.99, 1.01):
        assert np.sum((f * sc * L[off] - D[off]) ** 2 / D[off] ** 2) > st


def test_edge_uniformity_of_equal_edges_is_zero():
    """EU of a layout with all edges of equal length = 0 exactly:
    the 4-cycle on the unit square's corners."""
    g = cycle_graph(4)
    assert oracle.edge_uniformity(4, g.rowptr, g.colidx, [[0, 0], [1, 0], [1, 1], [0, 1]]) == 0.0


def test_np_two_clusters_and_violated_cycle():
    """two well-separated tight cliques -> NP = 1; a 4-cycle laid
    out so that each vertex's nearest vertices are its non-neighbour and one
    neighbour -> Jaccard 1/3 everywhere."""
    edges = [(i, j) for i in range(4) for j in range(i + 1, 4)]
    edges += [(i + 4, j + 4) for i, j in edges]
    g = _g(8, edges)
    rng = np.random.default_rng(0)
    xy = np.concatenate([rng.random((4, 2)) * 0.1, 10 + rng.random((4, 2)) * 0.1])
    npv, cnt = oracle.neighborhood_preservation(8, g.rowptr, g.colidx, xy)
    assert npv == 1.0 and cnt == 8
    g = cycle_graph(4)                      # 0-1-2-3-0; put 0,2 and 1,3 close together
    xy = np.array([[0, 0], [5, 0], [0.1, 0], [5.1, 0]], np.float32)
    npv, _, jac = oracle.neighborhood_preservation(4, g.rowptr, g.colidx, xy, per_vertex=True)
    np.testing.assert_allclose(jac, 1 / 3)


def _np_numpy(g, xy):
    xy = np.asarray(xy, np.float32)
    out = []
    for i in range(g.n):
        k = g.rowptr[i + 1] - g.rowptr[i]
        if k == 0:
            continue
        dx = (xy[:, 0] - xy[i, 0]).astype(np.float32)
        dy = (xy[:, 1] - xy[i, 1]).astype(np.float32)
        d2 = (dx * dx + dy * dy).astype(np.float32)
        ids = np.delete(np.arange(g.n), i)
        order = np.lexsort((ids, np.delete(d2, i)))
        near = set(ids[order[:k]].tolist())
        nb = set(g.colidx[g.rowptr[i]:g.rowptr[i + 1]].tolist())
        out.append(len(near & nb) / len(near | nb))
    return float(np.mean(out)) if out else 0.0


@pytest.mark.parametrize("seed", range(8))
def test_metrics_vs_independent_implementation(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(8, 50))
    u, v = np.triu_indices(n, 1)
    keep = rng.random(u.size) < rng.uniform(0.05, 0.4)
    g = edges_to_csr(n, u[keep], v[keep])
    xy = (rng.random((n, 2)) * 4).astype(np.float32)
    xy[rng.integers(0, n)] = xy[0]                          # a coincident pair: ties by id
    A = csr_matrix((np.ones(g.nnz), g.colidx, g.rowptr), shape=(n, n))
    D = shortest_path(A, unweighted=True)
    X = xy.astype(np.float64)
    L = np.hypot(*(X[:, None, :] - X[None, :, :]).transpose(2, 0, 1))
    ok = np.isfinite(D) & ~np.eye(n, dtype=bool)
    a_ = np.sum(L[ok] / D[ok])
    b_ = np.sum(L[ok] ** 2 / D[ok] ** 2)
    s_ = a_ / b_ if b_ > 0 else 0.0
    st_ref = np.sum((s_ * L[ok] - D[ok]) ** 2 / D[ok] ** 2)
    st, sc, pairs, un = oracle.stress(n, g.rowptr, g.colidx, xy)
    assert pairs == ok.sum() and un == (~np.isfinite(D)).sum()
    assert st == pytest.approx(st_ref, rel=1e-9, abs=1e-9) and sc == pytest.approx(s_, rel=1e-12)
    # edge uniformity
    i, j = np.nonzero(np.triu(A.toarray()) > 0)
    le = L[i, j]
    eu_ref = np.sqrt(np.sum((le - le.mean()) ** 2) / (le.size * le.mean() ** 2)) if le.size else 0.0
    assert oracle.edge_uniformity(n, g.rowptr, g.colidx, xy) == pytest.approx(eu_ref, rel=1e-12)
    # neighbourhood preservation
    assert oracle.neighborhood_preservation(n, g.rowptr, g.colidx, xy)[0] == pytest.approx(
        _np_numpy(g, xy), rel=1e-15)


def test_metric_invariances():
    """Rigid motions (90-degree rotation, reflection) and scaling by 2 are
    exact in fp32: stress and NP unchanged, s* halves, EU unchanged."""
    g = grid_graph(8, 9)
    xy = uniform_coords(g.n, 5)
    base = (oracle.stress(g.n, g.rowptr, g.colidx, xy), oracle.edge_uniformity(g.n, g.rowptr, g.colidx, xy),
            oracle.neighborhood_preservation(g.n, g.rowptr, g.colidx, xy)[0])
    for T in (lambda p: np.stack([-p[:, 1], p[:, 0]], 1), lambda p: np.stack([-p[:, 0], p[:, 1]], 1)):
        p = T(xy).astype(np.float32)
        st = oracle.stress(g.n, g.rowptr, g.colidx, p)
        assert st[0] == pytest.approx(base[0][0], rel=1e-12) and st[1] == pytest.approx(base[0][1], rel=1e-12)
        assert oracle.edge_uniformity(g.n, g.rowptr, g.colidx, p) == pytest.approx(base[1], rel=1e-12)
        assert oracle.neighborhood_preservation(g.n, g.rowptr, g.colidx, p)[0] == base[2]
    p = (xy * 2).astype(np.float32)
    st = oracle.stress(g.n, g.rowptr, g.colidx, p)
    assert st[0] == pytest.approx(base[0][0], rel=1e-12) and st[1] == pytest.approx(base[0][1] / 2, rel=1e-12)
    assert oracle.neighborhood_preservation(g.n, g.rowptr, g.colidx, p)[0] == base[2]


def test_sampled_sources_and_disconnected():
    g = _g(5, [(0, 1), (1, 2), (3, 4)])
    xy = np.array([[0, 0], [1, 0], [2, 0], [5, 5], [6, 5]], np.float32)
    st, sc, pairs, un = oracle.stress(5, g.rowptr, g.colidx, xy)
    assert pairs == 2 * (3 + 1) and un == 20 - 8 and st == pytest.approx(0, abs=1e-12) and sc == pytest.approx(1.0)
    st, sc, pairs, un = oracle.stress(5, g.rowptr, g.colidx, xy, sources=[0, 4])
    assert pairs == 2 + 1 and un == 2 + 3
