"""Pins of the C oracle against things other than itself (no GPU needed):
worked examples, closed forms, exact invariants, paper special cases and
brute force on tiny graphs.  Citations are PAPER.md lines (P:n) and SPEC.md
lines (S:n); readings C1-C13 are listed in DESIGN.md §3.
"""
import itertools
import math
import os

import numpy as np
import pytest

import oracle
from blgen import cycle_graph, star_graph, edges_to_csr, grid_graph, rmat_graph, uniform_coords
from tests import bruteforce

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "spec_examples.txt")


def _golden(kind):
    rows = []
    with open(GOLDEN) as fh:
        for line in fh:
            line = line.split("#")[0].strip()
            if not line or not line.startswith(kind + " "):
                continue
            lhs, rhs = line[len(kind):].split("->")
            rows.append(([float(t) for t in lhs.split()], [float(t) for t in rhs.split()]))
    assert rows
    return rows


def _edge_csr(n, edges):
    u = np.array([e[0] for e in edges], dtype=np.int64)
    v = np.array([e[1] for e in edges], dtype=np.int64)
    g = edges_to_csr(n, u, v)
    return g.rowptr, g.colidx


# ------------------------------------------------------------ worked examples

@pytest.mark.parametrize("row", _golden("pair"))
def test_pair_force_worked_examples(row):
    """§2.2; SPEC S:131-146 (golden fixture)."""
    (adj, K, C, xi, yi, xj, yj), (fx, fy) = row
    edges = [(0, 1)] if adj else []
    rp, ci = _edge_csr(2, edges)
    f = oracle.forces(2, rp, ci, np.array([[xi, yi], [xj, yj]]), 0, 1, K=K, C=C)
    assert f[0, 0] == pytest.approx(fx, abs=1e-15)
    assert f[0, 1] == pytest.approx(fy, abs=1e-15)


@pytest.mark.parametrize("row", _golden("update"))
def test_update_worked_examples(row):
    """Alg. 1 line 12 and the energy term."""
    (cx, cy, fx, fy, step), (ex, ey, eq) = row
    c, q = oracle.apply_update((cx, cy), (fx, fy), step)
    assert c[0] == pytest.approx(ex, abs=1e-15)
    assert c[1] == pytest.approx(ey, abs=1e-15)
    assert q == pytest.approx(eq, abs=1e-15)


def test_update_moves_exactly_step():
    """|c' - c| = Step whenever f != 0 (Alg. 1 line 12)."""
    rng = np.random.default_rng(0)
    for _ in range(200):
        c = rng.normal(size=2) * 10
        f = rng.normal(size=2) * 10 ** rng.uniform(-5, 5)
        step = rng.uniform(0.01, 3)
        c2, q = oracle.apply_update(c, f, step)
        assert np.hypot(*(c2 - c)) == pytest.approx(step, rel=1e-12)
        assert q == pytest.approx(f @ f, rel=1e-15)
        # the move is along f
        d = c2 - c
        assert d[0] * f[1] - d[1] * f[0] == pytest.approx(0, abs=1e-9 * step * np.hypot(*f))


def test_force_is_sum_of_pairs_and_antisymmetric():
    """§2.2 sum structure on 3 vertices against a hand sum of the two
    closed-form pair terms; f(i) from j is minus f(j) from i."""
    # path 0-1, 2 isolated; K=1.5, C=0.7
    K, C = 1.5, 0.7
    rp, ci = _edge_csr(3, [(0, 1)])
    c = np.array([[0.0, 0.0], [3.0, 4.0], [-1.0, 0.0]])
    f = oracle.forces(3, rp, ci, c, K=K, C=C)
    # on 0: attraction to 1 (d=5): (d/K) * delta = (5/1.5)*(3,4); repulsion from 2 (d=1): -(C K^2/d^2)*delta
    exp0 = (5 / 1.5) * np.array([3.0, 4.0]) - (C * K * K / 1.0) * np.array([-1.0, 0.0])
    np.testing.assert_allclose(f[0], exp0, rtol=1e-14)
    # on 2: repulsion from 0 (d=1) and from 1 (d=sqrt(32))
    d12 = np.array([4.0, 4.0])
    exp2 = -(C * K * K) * np.array([1.0, 0.0]) - (C * K * K / 32.0) * d12
    np.testing.assert_allclose(f[2], exp2, rtol=1e-14)


def test_coincident_pair_contributes_nothing():
    """Reading C4: d = 0 between distinct vertices contributes 0."""
    rp, ci = _edge_csr(3, [(0, 1)])
    c = np.array([[1.0, 1.0], [1.0, 1.0], [2.0, 1.0]])
    f = oracle.forces(3, rp, ci, c)
    assert np.all(np.isfinite(f))
    np.testing.assert_allclose(f[0], [-1.0, 0.0])   # only 2 repels 0
    np.testing.assert_allclose(f[1], [-1.0, 0.0])


# ------------------------------------------------------------ closed forms

@pytest.mark.parametrize("b", [1, 2])
def test_two_vertices_separation_and_energy(b):
    """Two vertices, no edge: each iteration both move apart by Step, so
    d_T = d0 + 2 sum_{t<T} step0 gamma^t.  Energy timing
    (reading C8): b=2 -> E_t = 2 (CK^2/d_t)^2; b=1 -> the second vertex
    sees the first one already moved: (CK^2/d_t)^2 + (CK^2/(d_t+step_t))^2."""
    K, C, step0, gamma, T = 1.25, 0.8, 0.5, 0.95, 20
    rp, ci = _edge_csr(2, [])
    xy0 = np.array([[0.1, 0.2], [0.4, 0.6]])  # d0 = 0.5
    xy, E, done = oracle.layout(2, rp, ci, xy0, iters=T, batch=b, K=K, C=C, step0=step0,
                                cooling=gamma)
    assert done == T
    steps = step0 * gamma ** np.arange(T)
    d = 0.5 + 2 * np.concatenate([[0.0], np.cumsum(steps)])
    assert np.hypot(*(xy[1] - xy[0])) == pytest.approx(d[T], rel=1e-13)
    s = C * K * K
    if b == 2:
        expE = 2 * (s / d[:T]) ** 2
    else:
        expE = (s / d[:T]) ** 2 + (s / (d[:T] + steps)) ** 2
    np.testing.assert_allclose(E, expE, rtol=1e-12)
    # direction: they separate along the initial line
    u = (xy[1] - xy[0]) / np.hypot(*(xy[1] - xy[0]))
    np.testing.assert_allclose(u, [0.6, 0.8], atol=1e-12)


def test_tol_stop_two_vertices():
    """|E_t - E_{t-1}| < tol stops the run (§4.5).  Two vertices, b=2:
    E_t = 2 (CK^2/d_t)^2 with d_t = d0 + 2 sum_{s<t} step_s (closed form above),
    so the stopping iteration is known in advance."""
    rp, ci = _edge_csr(2, [])
    xy0 = np.array([[0.0, 0.0], [0.3, 0.4]])
    gamma, T, tol = 0.9, 200, 1e-4
    steps = gamma ** np.arange(T)
    d = 0.5 + 2 * np.concatenate([[0.0], np.cumsum(steps)])
    E = 2 * (1.0 / d[:T]) ** 2
    stop = next(t for t in range(1, T) if abs(E[t] - E[t - 1]) < tol) + 1
    xy, Eo, done = oracle.layout(2, rp, ci, xy0, iters=T, batch=2, cooling=gamma, tol=tol)
    assert done == stop and len(Eo) == stop
    np.testing.assert_allclose(Eo, E[:stop], rtol=1e-12)
    assert np.hypot(*(xy[1] - xy[0])) == pytest.approx(d[stop], rel=1e-13)


def _circle(n, jitter, seed):
    rng = np.random.default_rng(seed)
    th = 2 * np.pi * np.arange(n) / n + rng.uniform(-jitter, jitter, n)
    r = 1.0 + rng.uniform(-jitter, jitter, n)
    return np.stack([r * np.cos(th), r * np.sin(th)], axis=1)


@pytest.mark.parametrize("n", [4, 5, 6, 8])
@pytest.mark.parametrize("bmode", ["b1", "bn"])
@pytest.mark.parametrize("KC", [(1.0, 1.0), (2.0, 0.5)])
@pytest.mark.parametrize("flags", [0, oracle.REPULSE_NEIGHBORS])
def test_cycle_relaxes_to_regular_polygon(n, bmode, KC, flags):
    """Cycle C_n relaxes to a regular polygon with edge length
    l = K ((n-3) C / 2)^(1/3) under the paper's if/else rule (Alg. 1
    P:553-557), or K ((n-1) C / 2)^(1/3) when neighbours also repel.  Each
    non-neighbour pushes exactly C K^2/(2 rho) radially; the two springs pull
    l^3/(rho K); balance gives the closed form (pin P1)."""
    K, C = KC
    g = cycle_graph(n)
    xy0 = _circle(n, 0.05, seed=n)
    b = 1 if bmode == "b1" else n
    xy, E, _ = oracle.layout(n, g.rowptr, g.colidx, xy0, iters=3000, batch=b, K=K, C=C,
                             cooling=0.99, flags=flags)
    m = (n - 1) if flags else (n - 3)
    ell = K * (m * C / 2) ** (1 / 3)
    edge = np.hypot(*(xy - np.roll(xy, -1, axis=0)).T)
    np.testing.assert_allclose(edge, ell, rtol=1e-9)
    cen = xy.mean(axis=0)
    rad = np.hypot(*(xy - cen).T)
    np.testing.assert_allclose(rad, ell / (2 * np.sin(np.pi / n)), rtol=1e-9)
    assert E[-1] < 1e-12 * max(1.0, E[0])


@pytest.mark.parametrize("k", [3, 5])
def test_star_relaxes_to_circle(k):
    """Star with k leaves: leaves at radius K ((k-1) C / 2)^(1/3) from the
    centre (attraction rho^2/K = (k-1) C K^2 / (2 rho))."""
    K, C = 1.0, 1.0
    g = star_graph(k)
    xy0 = np.vstack([[0.0, 0.0], _circle(k, 0.05, seed=k) * 0.7])
    xy, _, _ = oracle.layout(k + 1, g.rowptr, g.colidx, xy0, iters=3000, batch=1, K=K, C=C,
                             cooling=0.99)
    rho = K * ((k - 1) * C / 2) ** (1 / 3)
    r = np.hypot(*(xy[1:] - xy[0]).T)
    np.testing.assert_allclose(r, rho, rtol=1e-9)


# ------------------------------------------------------------ invariants

def _rand_graph(n, p, seed):
    rng = np.random.default_rng(seed)
    edges = [(i, j) for i in range(n) for j in range(i + 1, n) if rng.random() < p]
    return _edge_csr(n, edges)


def test_forces_sum_to_zero_with_b_eq_n():
    """With b = n, both parts are pairwise antisymmetric, so sum_i f_i = 0
    (north star)."""
    g = grid_graph(8, 9)
    xy = uniform_coords(g.n, 7).astype(np.float64)
    f = oracle.forces(g.n, g.rowptr, g.colidx, xy)
    scale = np.abs(f).sum()
    assert np.abs(f.sum(axis=0)).max() < 1e-13 * scale


def test_translation_invariance():
    """Shifting xy0 by t shifts the output by t."""
    rp, ci = _rand_graph(30, 0.15, 1)
    xy0 = uniform_coords(30, 3).astype(np.float64)
    t = np.array([5.0, -3.0])
    a, Ea, _ = oracle.layout(30, rp, ci, xy0, iters=5, batch=7)
    b, Eb, _ = oracle.layout(30, rp, ci, xy0 + t, iters=5, batch=7)
    np.testing.assert_allclose(b - t, a, atol=1e-11 * np.abs(t).max())
    np.testing.assert_allclose(Eb, Ea, rtol=1e-7)


def test_rotation_and_reflection_bitwise():
    """(x,y) -> (-y,x) and x -> -x commute with the method exactly (the
    oracle is built without contraction)."""
    rp, ci = _rand_graph(25, 0.2, 2)
    xy0 = uniform_coords(25, 4).astype(np.float64)
    a, Ea, _ = oracle.layout(25, rp, ci, xy0, iters=6, batch=4)
    rot = np.stack([-xy0[:, 1], xy0[:, 0]], axis=1)
    b, Eb, _ = oracle.layout(25, rp, ci, rot, iters=6, batch=4)
    assert np.array_equal(b, np.stack([-a[:, 1], a[:, 0]], axis=1))
    assert np.array_equal(Ea, Eb)
    ref = xy0 * np.array([-1.0, 1.0])
    c, Ec, _ = oracle.layout(25, rp, ci, ref, iters=6, batch=4)
    assert np.array_equal(c, a * np.array([-1.0, 1.0]))
    assert np.array_equal(Ec, Ea)


def test_K_C_scaling_bitwise():
    """(K, C) -> (lam K, C / lam^3), lam a power of two: identical trajectory
    bitwise, energy x lam^-2 (f_a and f_r both scale by 1/lam)."""
    rp, ci = _rand_graph(20, 0.25, 3)
    xy0 = uniform_coords(20, 5).astype(np.float64)
    a, Ea, _ = oracle.layout(20, rp, ci, xy0, iters=8, batch=6, K=1.0, C=1.0)
    b, Eb, _ = oracle.layout(20, rp, ci, xy0, iters=8, batch=6, K=2.0, C=1.0 / 8.0)
    assert np.array_equal(a, b)
    assert np.array_equal(Ea / Eb, np.full_like(Ea, 4.0))


def test_coordinate_scale_bitwise():
    """(xy0, K, step0) x s, s a power of two: output x s, energy x s^2."""
    rp, ci = _rand_graph(20, 0.25, 4)
    xy0 = uniform_coords(20, 6).astype(np.float64)
    a, Ea, _ = oracle.layout(20, rp, ci, xy0, iters=8, batch=5, K=1.0, step0=1.0)
    b, Eb, _ = oracle.layout(20, rp, ci, xy0 * 4.0, iters=8, batch=5, K=4.0, step0=4.0)
    assert np.array_equal(b, a * 4.0)
    assert np.array_equal(Eb, Ea * 16.0)


def test_permutation_equivariance_b_eq_n():
    """With b = n (all frozen together) relabelling permutes the output."""
    n = 15
    rng = np.random.default_rng(9)
    edges = [(i, j) for i in range(n) for j in range(i + 1, n) if rng.random() < 0.3]
    perm = rng.permutation(n)
    rp, ci = _edge_csr(n, edges)
    rp2, ci2 = _edge_csr(n, [(perm[i], perm[j]) for i, j in edges])
    xy0 = uniform_coords(n, 8).astype(np.float64)
    xy0p = np.empty_like(xy0)
    xy0p[perm] = xy0
    a, Ea, _ = oracle.layout(n, rp, ci, xy0, iters=5, batch=n)
    b, Eb, _ = oracle.layout(n, rp2, ci2, xy0p, iters=5, batch=n)
    np.testing.assert_allclose(b[perm], a, rtol=1e-11, atol=1e-11)
    np.testing.assert_allclose(Eb, Ea, rtol=1e-11)


def test_one_batch_leaves_other_vertices_bitwise_unchanged():
    """Only the batch's vertices move in a batch update (Alg. 2)."""
    g = grid_graph(6, 7)
    xy0 = uniform_coords(g.n, 11).astype(np.float64)
    for b in (1, 5, 16):
        xy, _, done = oracle.layout(g.n, g.rowptr, g.colidx, xy0, iters=3, batch=b, max_batches=1)
        assert done == 0
        assert np.array_equal(xy[b:], xy0[b:])
        assert np.all(np.hypot(*(xy[:b] - xy0[:b]).T) == pytest.approx(1.0, rel=1e-12))


def test_second_batch_sees_first_batch_update():
    """Fig. 2 caption: the next minibatch uses updated coordinates.
    Two batches of a path: the result after 2 batches equals running batch 0,
    then computing batch 1's forces at that state."""
    g = grid_graph(1, 6)
    xy0 = uniform_coords(6, 12).astype(np.float64)
    one, _, _ = oracle.layout(6, g.rowptr, g.colidx, xy0, iters=1, batch=3, max_batches=1)
    two, _, _ = oracle.layout(6, g.rowptr, g.colidx, xy0, iters=1, batch=3, max_batches=2)
    f = oracle.forces(6, g.rowptr, g.colidx, one, 3, 3)
    exp = one[3:] + f / np.hypot(f[:, 0], f[:, 1])[:, None]
    np.testing.assert_allclose(two[3:], exp, rtol=1e-15, atol=1e-15)
    assert np.array_equal(two[:3], one[:3])


def test_thread_count_invariance_bitwise():
    """Same layout irrespective of the number of threads."""
    g = rmat_graph(9, 8, 0.57, 0.19, 0.19, seed=5)
    xy0 = uniform_coords(g.n, 13)
    a, Ea, _ = oracle.layout(g.n, g.rowptr, g.colidx, xy0, iters=2, batch=64, threads=1)
    b, Eb, _ = oracle.layout(g.n, g.rowptr, g.colidx, xy0, iters=2, batch=64, threads=4)
    assert np.array_equal(a, b) and np.array_equal(Ea, Eb)


def test_degenerate_cases():
    # n = 1: no pairs, force 0, no move (reading C5), energy 0
    xy, E, done = oracle.layout(1, np.array([0, 0]), np.array([], np.int32),
                                np.array([[0.3, 0.4]]), iters=3, batch=1)
    assert np.array_equal(xy, [[0.3, 0.4]]) and np.all(E == 0) and done == 3
    # iters = 0 is a no-op
    g = grid_graph(3, 3)
    xy0 = uniform_coords(9, 1).astype(np.float64)
    xy, E, done = oracle.layout(9, g.rowptr, g.colidx, xy0, iters=0, batch=4)
    assert np.array_equal(xy, xy0) and done == 0
    # b > n is clamped to n
    a, Ea, _ = oracle.layout(9, g.rowptr, g.colidx, xy0, iters=3, batch=100)
    b, Eb, _ = oracle.layout(9, g.rowptr, g.colidx, xy0, iters=3, batch=9)
    assert np.array_equal(a, b) and np.array_equal(Ea, Eb)
    # invalid arguments are rejected
    with pytest.raises(ValueError):
        oracle.layout(9, g.rowptr, g.colidx, xy0, iters=1, batch=0)


# ------------------------------------------------------------ brute force

def test_b1_equals_algorithm_1():
    """'Algorithm 1 is a special case of Algorithm 2 when the size of the
    minibatch is 1': oracle at b=1 vs a literal Alg. 1."""
    for seed in range(6):
        n = 6 + seed % 3
        rng = np.random.default_rng(seed)
        edges = [(i, j) for i in range(n) for j in range(i + 1, n) if rng.random() < 0.4]
        rp, ci = _edge_csr(n, edges)
        xy0 = rng.random((n, 2))
        A = bruteforce.dense_adj(n, rp, ci)
        c_bf, E_bf = bruteforce.alg1(n, A, xy0, 4, K=1.0, R=1.0)
        c_or, E_or, _ = oracle.layout(n, rp, ci, xy0, iters=4, batch=1)
        np.testing.assert_allclose(c_or, np.array(c_bf), rtol=1e-10, atol=1e-10)
        np.testing.assert_allclose(E_or, E_bf, rtol=1e-10)


def _all_graphs(n):
    pairs = list(itertools.combinations(range(n), 2))
    for mask in range(1 << len(pairs)):
        yield [p for k, p in enumerate(pairs) if mask >> k & 1]


@pytest.mark.parametrize("n", [3, 4, 5])
def test_exhaustive_small_graphs_vs_bruteforce(n):
    """Every labelled graph on n <= 5 vertices, b in {1, 2, 3, n}, 3
    iterations, random coordinates: oracle == literal dense Alg. 2."""
    rng = np.random.default_rng(100 + n)
    for edges in _all_graphs(n):
        rp, ci = _edge_csr(n, edges)
        A = bruteforce.dense_adj(n, rp, ci)
        xy0 = rng.random((n, 2))
        K, R = rng.uniform(0.5, 2.0), rng.uniform(0.5, 2.0)
        for b in sorted({1, 2, 3, n}):
            c_bf, E_bf = bruteforce.alg2(n, A, xy0, 3, b, K=K, R=R)
            c_or, E_or, _ = oracle.layout(n, rp, ci, xy0, iters=3, batch=b, K=K, C=R)
            np.testing.assert_allclose(c_or, np.array(c_bf), rtol=1e-9, atol=1e-9)
            np.testing.assert_allclose(E_or, E_bf, rtol=1e-9)


@pytest.mark.parametrize("n", [6, 7, 8])
@pytest.mark.parametrize("flags", [0, oracle.REPULSE_NEIGHBORS])
def test_random_graphs_vs_bruteforce(n, flags):
    rng = np.random.default_rng(200 + n)
    for trial in range(20):
        p = rng.uniform(0.1, 0.9)
        edges = [(i, j) for i in range(n) for j in range(i + 1, n) if rng.random() < p]
        rp, ci = _edge_csr(n, edges)
        A = bruteforce.dense_adj(n, rp, ci)
        xy0 = rng.random((n, 2)) * 3
        iters = int(rng.integers(1, 6))
        for b in (1, 2, 3, n):
            c_bf, E_bf = bruteforce.alg2(n, A, xy0, iters, b, K=1.3, R=0.7,
                                         repulse_neighbors=bool(flags))
            c_or, E_or, _ = oracle.layout(n, rp, ci, xy0, iters=iters, batch=b, K=1.3, C=0.7,
                                          flags=flags)
            np.testing.assert_allclose(c_or, np.array(c_bf), rtol=1e-9, atol=1e-9)
            np.testing.assert_allclose(E_or, E_bf, rtol=1e-9)


def test_f32_variant_tracks_f64_for_one_iteration():
    """The fp32 instantiation (chaos-floor tool) follows the fp64 one closely
    over one iteration of a C1-shaped case."""
    g = grid_graph(16, 16)
    xy0 = uniform_coords(g.n, 42)
    a, Ea, _ = oracle.layout(g.n, g.rowptr, g.colidx, xy0, iters=1, batch=64)
    b, Eb, _ = oracle.layout(g.n, g.rowptr, g.colidx, xy0, iters=1, batch=64, precision="f32")
    ext = np.ptp(a, axis=0).max()
    assert np.abs(a - b).max() < 1e-4 * ext
    assert abs(Ea[0] - Eb[0]) < 1e-3 * Ea[0]


# ------------------------------------------------------------ (a, r)-energy models (C15)

@pytest.mark.parametrize("row", _golden("pairm"))
def test_model_pair_force_worked_examples(row):
    """(a, r)-energy model (§2.2): hand-derived pair forces."""
    (adj, a, r, K, C, xi, yi, xj, yj), (fx, fy) = row
    rp, ci = _edge_csr(2, [(0, 1)] if adj else [])
    f = oracle.forces(2, rp, ci, np.array([[xi, yi], [xj, yj]]), 0, 1, K=K, C=C, a=a, r=r)
    assert f[0, 0] == pytest.approx(fx, abs=1e-14)
    assert f[0, 1] == pytest.approx(fy, abs=1e-14)


@pytest.mark.parametrize("ar", [(1.0, -1.0), (0.0, -1.0), (3.0, -1.0), (2.0, -2.0),
                                (1.5, -0.5)])
@pytest.mark.parametrize("flags", [0, oracle.REPULSE_NEIGHBORS])
def test_models_vs_bruteforce(ar, flags):
    a, r = ar
    rng = np.random.default_rng(int(10 * a - 7 * r) + flags)
    for trial in range(6):
        n = int(rng.integers(4, 8))
        edges = [(i, j) for i in range(n) for j in range(i + 1, n) if rng.random() < 0.4]
        rp, ci = _edge_csr(n, edges)
        A = bruteforce.dense_adj(n, rp, ci)
        xy0 = rng.random((n, 2)) * 3
        for b in (1, 3, n):
            c_bf, E_bf = bruteforce.alg2(n, A, xy0, 3, b, K=1.3, R=0.7,
                                         repulse_neighbors=bool(flags), a=a, r=r)
            c_or, E_or, _ = oracle.layout(n, rp, ci, xy0, iters=3, batch=b, K=1.3, C=0.7,
                                          flags=flags, a=a, r=r)
            np.testing.assert_allclose(c_or, np.array(c_bf), rtol=1e-9, atol=1e-9)
            np.testing.assert_allclose(E_or, E_bf, rtol=1e-9)


@pytest.mark.parametrize("ar", [(1.0, -1.0), (3.0, -1.0), (2.0, -2.0), (1.5, -0.5)])
@pytest.mark.parametrize("flags", [0, oracle.REPULSE_NEIGHBORS])
def test_cycle_closed_form_general_model(ar, flags):
    """Regular n-gon equilibrium of the (a, r) model.  With edge l and the
    other vertices at d_k = l s_k, s_k = sin(pi k/n)/sin(pi/n): each vertex
    feels an inward pull l^(a+1)/(K rho) from its two springs and an outward
    push C K^2 d_k^(r+1)/(2 rho) from each repelling vertex, so
    l^(a-r) = (C K^3 / 2) sum_k s_k^(r+1) (k = 2..n-2, or 1..n-1 when
    neighbours repel).  For (2, -1) this is pin P1."""
    a, r = ar
    n, K, C = 6, 1.2, 0.8
    ks = np.arange(1, n) if flags else np.arange(2, n - 1)
    S = np.sum((np.sin(np.pi * ks / n) / np.sin(np.pi / n)) ** (r + 1))
    ell = (C * K ** 3 / 2 * S) ** (1 / (a - r))
    g = cycle_graph(n)
    xy0 = _circle(n, 0.05, seed=n) * ell
    xy, E, _ = oracle.layout(n, g.rowptr, g.colidx, xy0, iters=4000, batch=1, K=K, C=C,
                             cooling=0.99, flags=flags, a=a, r=r)
    edge = np.hypot(*(xy - np.roll(xy, -1, axis=0)).T)
    np.testing.assert_allclose(edge, ell, rtol=1e-7)
