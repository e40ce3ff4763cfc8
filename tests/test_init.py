"""Greedy initialisation (Alg. 3, §3.6): the
oracle against hand-derived layouts and DFS invariants, the product's host
C++ (bl_greedy_init in libbl, no GPU needed) against the oracle bitwise,
and the paper's claim that greedy initialisation converges faster
(Fig. 6(a)).  Readings G1-G4: DESIGN.md §3."""
import os

import numpy as np
import pytest

import oracle
from blgen import build_config, edges_to_csr, grid_graph, rmat_graph, tri_mesh_graph
from tests.test_oracle_pins import GOLDEN


def _golden():
    rows = []
    with open(GOLDEN) as fh:
        for line in fh:
            line = line.split("#")[0].strip()
            if not line.startswith("greedy "):
                continue
            lhs, rhs = line[len("greedy "):].split("->")
            n, edges, root = lhs.split()
            e = [tuple(int(t) for t in pair.split("-")) for pair in edges.split(",")]
            rows.append((int(n), e, int(root), np.array([float(t) for t in rhs.split()]).reshape(-1, 2)))
    assert rows
    return rows


@pytest.mark.parametrize("row", _golden())
def test_oracle_matches_hand_derived_layouts(row):
    n, edges, root, want = row
    g = edges_to_csr(n, np.array([a for a, _ in edges]), np.array([b for _, b in edges]))
    got = oracle.greedy_init(n, g.rowptr, g.colidx, root)
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-7)


def _random_graph(n, p, seed):
    rng = np.random.default_rng(seed)
    u, v = np.triu_indices(n, 1)
    keep = rng.random(u.size) < p
    return edges_to_csr(n, u[keep], v[keep])


@pytest.mark.parametrize("seed", range(5))
def test_dfs_invariants(seed):
    """Every vertex is placed; every vertex but a component root is at
    distance 1 from a neighbour (its DFS parent, Alg. 3 line 12); the
    component roots sit on the grid of reading G3 with V0 at the origin."""
    n = 60
    g = _random_graph(n, 0.04, seed)
    root = seed % n
    xy = oracle.greedy_init(n, g.rowptr, g.colidx, root).astype(np.float64)
    assert np.all(np.isfinite(xy)) and np.array_equal(xy[root], [0.0, 0.0])
    comp = _components(g)
    sizes = np.bincount(comp)
    s = 2 * int(np.ceil(np.sqrt(sizes.max()) - 1e-12))
    comp_roots = {comp[root]: root}
    for v in range(n):
        comp_roots.setdefault(comp[v], v)            # smallest id of the other components
    for v in range(n):
        if comp_roots[comp[v]] == v:
            assert np.allclose(xy[v] / s, np.round(xy[v] / s))   # origin on the grid (G3)
            continue
        nb = g.colidx[g.rowptr[v]:g.rowptr[v + 1]]
        dist = np.hypot(*(xy[nb] - xy[v]).T)
        assert np.any(np.abs(dist - 1.0) < 1e-5)     # placed on a unit circle (line 12)


def _components(g):
    n = g.n
    comp = -np.ones(n, int)
    c = 0
    for s in range(n):
        if comp[s] >= 0:
            continue
        stack = [s]
        comp[s] = c
        while stack:
            u = stack.pop()
            for w in g.colidx[g.rowptr[u]:g.rowptr[u + 1]]:
                if comp[w] < 0:
                    comp[w] = c
                    stack.append(w)
        c += 1
    return comp


@pytest.mark.parametrize("name", ["C1", "C2", "C3b256", "C4", "C5"])
def test_product_host_init_matches_oracle_bitwise(name):
    """libbl's bl_greedy_init (host C++, its own BFS/DFS code) == the oracle."""
    import paper_2002_08233_b200 as bl
    g, _, _ = build_config(name)
    for root in (0, g.n // 2):
        a = bl.bl_greedy_init(g.n, g.rowptr, g.colidx, root)
        b = oracle.greedy_init(g.n, g.rowptr, g.colidx, root)
        assert np.array_equal(a, b)


def test_product_host_init_errors_and_determinism():
    import paper_2002_08233_b200 as bl
    g = grid_graph(5, 5)
    with pytest.raises(bl.BLError):
        bl.bl_greedy_init(g.n, g.rowptr, g.colidx, g.n)
    a = bl.bl_greedy_init(g.n, g.rowptr, g.colidx, 3)
    b = bl.bl_greedy_init(g.n, g.rowptr, g.colidx, 3)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("graph,checkpoints", [("tri", (5, 10, 20)),
                                              ("grid", (5, 10, 20, 50, 100, 199))])
def test_greedy_init_converges_faster_than_random(graph, checkpoints):
    """P:916-923 / Fig. 6(a): 'in the i-th iteration, the greedy-initialized
    layout has lower energy than the randomly-initialized layout'.  Random
    init is uniform over the same box as the greedy layout (both
    'within a given range'; MAXMIN itself is unstated).  What holds with our
    readings (G-readings): greedy wins the early iterations on
    a triangulated mesh and every checkpoint on a square grid, for >= 4 of 5
    seeds; on the mesh the random run catches up after ~50 iterations (the
    paper's 'every iteration' is not reproduced there)."""
    g = tri_mesh_graph(24, 25) if graph == "tri" else grid_graph(30, 30)
    xg = oracle.greedy_init(g.n, g.rowptr, g.colidx, 0)
    lo, hi = xg.min(0), xg.max(0)
    T = max(checkpoints) + 1
    _, Eg, _ = oracle.layout(g.n, g.rowptr, g.colidx, xg, iters=T, batch=64)
    wins = 0
    for seed in range(5):
        rng = np.random.default_rng(seed)
        xr = (lo + (hi - lo) * rng.random((g.n, 2))).astype(np.float32)
        _, Er, _ = oracle.layout(g.n, g.rowptr, g.colidx, xr, iters=T, batch=64)
        wins += int(all(Eg[t] < Er[t] for t in checkpoints))
    assert wins >= 4, wins
