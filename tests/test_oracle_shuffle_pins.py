"""Pins of the oracle's batch randomisation (§4.3.3, Fig. S3
P:278-284; readings R1-R2 of DESIGN.md §3).  -m "not gpu".

R1: iteration it uses a fresh permutation pi_it of the vertex ids, batch t =
pi_it(t b .. min((t+1) b, n) - 1); seed 0 = the paper's sequential batches.
R2: pi_it = 4-round Feistel network on [0, 2^M) keyed from splitmix64,
restricted to [0, n) by cycle walking.

Pins: splitmix64 known answers (the published first outputs of splitmix64
seeded with 0); bijection and determinism; the written spec of R2 evaluated
by an independent pure-Python implementation; the layout with shuffling vs
the dense literal Alg. 2 (tests/bruteforce.py) given the same orders;
b = n is order-independent (Jacobi); b = 1 is Alg. 1 in the permuted visiting
order; one batch moves exactly pi_0(0..b-1); thread-count invariance."""
import numpy as np
import pytest

import oracle
from blgen import edges_to_csr, grid_graph, rmat_graph, uniform_coords
from tests import bruteforce

GAMMA = 0x9E3779B97F4A7C15
MASK64 = (1 << 64) - 1


def test_splitmix64_known_answers():
    """splitmix64 seeded with 0 yields e220a8397b1dcdaf, 6e789e6aa1b965f4,
    06c45d188009454f (Vigna's reference generator); oracle_mix64(z) is the
    output for state z + gamma, i.e. the k-th output is mix64((k-1) gamma)."""
    assert oracle.mix64(0) == 0xE220A8397B1DCDAF
    assert oracle.mix64(GAMMA) == 0x6E789E6AA1B965F4
    assert oracle.mix64((2 * GAMMA) & MASK64) == 0x06C45D188009454F


def _py_perm(n, seed, it):
    """Reading R2 as written in DESIGN.md §3, in Python integers."""
    if seed == 0:
        return list(range(n))

    def mix(z):
        z = (z + GAMMA) & MASK64
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)

    M = 2
    while (1 << M) < n:
        M += 2
    h = M // 2
    keys = [mix(seed ^ mix(4 * it + r)) for r in range(4)]
    out = []
    for x in range(n):
        y = x
        while True:
            L, R = y >> h, y & ((1 << h) - 1)
            for r in range(4):
                L, R = R, L ^ (mix(keys[r] ^ R) >> (64 - h))
            y = (L << h) | R
            if y < n:
                break
        out.append(y)
    return out


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 16, 17, 100, 1023, 1025, 4096])
@pytest.mark.parametrize("seed", [1, 12345, 2 ** 63 + 11])
def test_permutation_is_a_bijection_and_follows_the_spec(n, seed):
    for it in (0, 1, 599):
        p = oracle.permutation(n, seed, it)
        assert sorted(p.tolist()) == list(range(n))
        assert p.tolist() == _py_perm(n, seed, it)
        assert np.array_equal(p, oracle.permutation(n, seed, it))  # deterministic


def test_seed_zero_is_identity_and_seeds_iterations_differ():
    n = 1000
    assert np.array_equal(oracle.permutation(n, 0, 5), np.arange(n))
    a, b, c = (oracle.permutation(n, 7, 0), oracle.permutation(n, 7, 1),
               oracle.permutation(n, 8, 0))
    assert not np.array_equal(a, b) and not np.array_equal(a, c)
    # not the identity and not a rotation: a genuine reshuffle
    assert np.mean(a == np.arange(n)) < 0.05
    assert abs(np.corrcoef(a, np.arange(n))[0, 1]) < 0.2


def test_seed_zero_layout_is_the_sequential_layout_bitwise():
    g = grid_graph(9, 11)
    xy0 = uniform_coords(g.n, 3)
    a, Ea, _ = oracle.layout(g.n, g.rowptr, g.colidx, xy0, iters=3, batch=16)
    b, Eb, _ = oracle.layout(g.n, g.rowptr, g.colidx, xy0, iters=3, batch=16, shuffle_seed=0)
    assert np.array_equal(a, b) and np.array_equal(Ea, Eb)


def _edge_csr(n, edges):
    u = np.array([e[0] for e in edges], np.int64)
    v = np.array([e[1] for e in edges], np.int64)
    g = edges_to_csr(n, u, v)
    return g.rowptr, g.colidx


@pytest.mark.parametrize("n", [3, 5, 6, 8])
@pytest.mark.parametrize("flags", [0, oracle.REPULSE_NEIGHBORS])
def test_shuffled_layout_vs_bruteforce(n, flags):
    """Random graphs on n <= 8 vertices, b in {1, 2, 3, n}, 4 iterations:
    the oracle with a seed == the dense literal Alg. 2 walking the batches in
    the orders pi_0 .. pi_3 (taken from the oracle's permutation, which the
    tests above pin to the written spec)."""
    rng = np.random.default_rng(300 + n)
    for trial in range(6):
        edges = [(i, j) for i in range(n) for j in range(i + 1, n) if rng.random() < 0.4]
        rp, ci = _edge_csr(n, edges)
        A = bruteforce.dense_adj(n, rp, ci)
        xy0 = rng.random((n, 2))
        seed = int(rng.integers(1, 2 ** 62))
        perms = [oracle.permutation(n, seed, it) for it in range(4)]
        for b in sorted({1, 2, 3, n}):
            c_bf, E_bf = bruteforce.alg2(n, A, xy0, 4, b, K=1.1, R=0.8, perms=perms,
                                         repulse_neighbors=bool(flags))
            c_or, E_or, _ = oracle.layout(n, rp, ci, xy0, iters=4, batch=b, K=1.1, C=0.8,
                                          flags=flags, shuffle_seed=seed)
            np.testing.assert_allclose(c_or, np.array(c_bf), rtol=1e-9, atol=1e-9)
            np.testing.assert_allclose(E_or, E_bf, rtol=1e-9)


def test_b_equals_n_is_order_independent():
    """b = n (the Jacobi variant): every force uses the frozen state, so the
    visiting order changes nothing but the order of the energy sum."""
    g = rmat_graph(9, 8, 0.57, 0.19, 0.19, seed=5)
    xy0 = uniform_coords(g.n, 13)
    a, Ea, _ = oracle.layout(g.n, g.rowptr, g.colidx, xy0, iters=3, batch=g.n)
    b, Eb, _ = oracle.layout(g.n, g.rowptr, g.colidx, xy0, iters=3, batch=g.n, shuffle_seed=99)
    assert np.array_equal(a, b)
    np.testing.assert_allclose(Ea, Eb, rtol=1e-13)


def test_b1_is_alg1_in_the_permuted_order():
    """b = 1 is Alg. 1 whatever the order: shuffled, it equals Alg. 1
    visiting the vertices in the order pi_it (brute force over a dense
    matrix)."""
    g = grid_graph(3, 3)
    xy0 = uniform_coords(g.n, 2).astype(np.float64)
    A = bruteforce.dense_adj(g.n, g.rowptr, g.colidx)
    perms = [oracle.permutation(g.n, 5, it) for it in range(3)]
    c_bf, E_bf = bruteforce.alg2(g.n, A, xy0, 3, 1, perms=perms)
    c_or, E_or, _ = oracle.layout(g.n, g.rowptr, g.colidx, xy0, iters=3, batch=1, shuffle_seed=5)
    np.testing.assert_allclose(c_or, np.array(c_bf), rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(E_or, E_bf, rtol=1e-12)


def test_one_batch_moves_exactly_its_permuted_members():
    g = rmat_graph(10, 8, 0.57, 0.19, 0.19, seed=2)
    xy0 = uniform_coords(g.n, 4)
    b = 100
    got, _, _ = oracle.layout(g.n, g.rowptr, g.colidx, xy0, iters=1, batch=b, max_batches=1,
                              shuffle_seed=42)
    members = oracle.permutation(g.n, 42, 0)[:b]
    moved = np.nonzero(np.any(got != xy0.astype(np.float64), axis=1))[0]
    assert set(moved.tolist()) <= set(members.tolist())
    assert len(moved) >= b - 2          # f = 0 is the only way not to move
    others = np.setdiff1d(np.arange(g.n), members)
    assert np.array_equal(got[others], xy0[others].astype(np.float64))


def test_shuffled_thread_count_invariance_bitwise():
    g = rmat_graph(10, 8, 0.57, 0.19, 0.19, seed=6)
    xy0 = uniform_coords(g.n, 8)
    a, Ea, _ = oracle.layout(g.n, g.rowptr, g.colidx, xy0, iters=2, batch=64, threads=1,
                             shuffle_seed=3)
    b, Eb, _ = oracle.layout(g.n, g.rowptr, g.colidx, xy0, iters=2, batch=64, threads=4,
                             shuffle_seed=3)
    assert np.array_equal(a, b) and np.array_equal(Ea, Eb)


def relabelled(g, xy, perm):
    """The graph and state in POSITION space of `perm` (position i holds
    vertex perm[i]): numpy only -- the identity behind the GPU's relabelled
    iterations (csrc/bl_relabel.cu), restated here for the oracle."""
    n = g.n
    inv = np.empty(n, np.int64)
    inv[perm] = np.arange(n)
    rows = np.repeat(np.arange(n), np.diff(g.rowptr))
    gp = edges_to_csr(n, inv[rows], inv[np.asarray(g.colidx)])
    return gp, np.asarray(xy)[perm]


@pytest.mark.parametrize("b", [1, 7, 64])
def test_shuffled_iteration_is_sequential_on_the_relabelled_graph(b):
    """Reading R1: the batches of pi_it are the CONTIGUOUS batches of the
    graph relabelled by pi_it, so a randomised iteration equals a sequential
    iteration (seed 0) of the relabelled problem, scattered back -- up to the
    order of the fp64 sums over the other vertices (1e-12).  Pins the
    oracle's batch membership, its per-batch freezing and the energy against
    its own sequential path on a different graph."""
    g = rmat_graph(8, 4, 0.57, 0.19, 0.19, 1)
    xy0 = uniform_coords(g.n, 3)
    seed = 77
    got, E, _ = oracle.layout(g.n, g.rowptr, g.colidx, xy0, iters=1, batch=b, shuffle_seed=seed)
    perm = oracle.permutation(g.n, seed, 0)
    gp, xyp = relabelled(g, xy0, perm)
    refp, Ep, _ = oracle.layout(gp.n, gp.rowptr, gp.colidx, xyp, iters=1, batch=b)
    ref = np.empty_like(refp)
    ref[perm] = refp
    assert np.abs(got - ref).max() <= 1e-11 * np.ptp(ref, axis=0).max()
    assert abs(E[0] - Ep[0]) <= 1e-11 * Ep[0]
