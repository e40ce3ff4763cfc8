"""Graph generators, CSR construction/validation and seeded coordinates.

No layout arithmetic lives here (see package docstring).  Every generator is
deterministic given its seed (numpy PCG64).

CSR conventions follow PAPER.md §2.1 (`rowptr` of length n+1,
`colids` of length m) with the invariants of SPEC.md S:31-35: rowptr[0]=0,
nondecreasing, rowptr[n]=nnz, ids in range, no self loops, rows strictly
ascending, symmetric (the paper treats graphs as undirected).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class CSRGraph:
    n: int
    rowptr: np.ndarray  # int32[n+1]
    colidx: np.ndarray  # int32[nnz]

    @property
    def nnz(self) -> int:
        return int(self.rowptr[-1])


def edges_to_csr(n: int, u: np.ndarray, v: np.ndarray) -> CSRGraph:
    """Symmetrise an undirected edge list, drop self loops and duplicates,
    keep isolated vertices, and return sorted int32 CSR."""
    u = np.asarray(u, dtype=np.int64)
    v = np.asarray(v, dtype=np.int64)
    if u.size:
        if u.min() < 0 or v.min() < 0 or u.max() >= n or v.max() >= n:
            raise ValueError("edge endpoint out of range")
    keep = u != v
    u, v = u[keep], v[keep]
    src = np.concatenate([u, v])
    dst = np.concatenate([v, u])
    key = np.unique(src * n + dst)  # sorted by (src, dst), deduplicated
    src = key // n
    dst = key % n
    counts = np.bincount(src, minlength=n)
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=rowptr[1:])
    if rowptr[-1] >= 2**31:
        raise ValueError("nnz does not fit int32")
    return CSRGraph(n, rowptr.astype(np.int32), dst.astype(np.int32))


def validate_csr(n: int, rowptr: np.ndarray, colidx: np.ndarray) -> None:
    """Raise ValueError unless (rowptr, colidx) is a valid symmetric,
    loop-free, strictly-row-sorted CSR on n vertices."""
    rowptr = np.asarray(rowptr)
    colidx = np.asarray(colidx)
    if n < 1:
        raise ValueError("n must be >= 1")
    if rowptr.shape != (n + 1,):
        raise ValueError("rowptr must have n+1 entries")
    if rowptr[0] != 0:
        raise ValueError("rowptr[0] != 0")
    if np.any(np.diff(rowptr.astype(np.int64)) < 0):
        raise ValueError("rowptr not nondecreasing")
    nnz = int(rowptr[-1])
    if colidx.shape != (nnz,):
        raise ValueError("colidx length != rowptr[n]")
    if nnz == 0:
        return
    if colidx.min() < 0 or colidx.max() >= n:
        raise ValueError("column index out of range")
    row = np.repeat(np.arange(n, dtype=np.int64), np.diff(rowptr.astype(np.int64)))
    col = colidx.astype(np.int64)
    if np.any(row == col):
        raise ValueError("self loop")
    same_row = row[1:] == row[:-1]
    if np.any(same_row & (col[1:] <= col[:-1])):
        raise ValueError("row not strictly ascending")
    fwd = np.sort(row * n + col)
    bwd = np.sort(col * n + row)
    if not np.array_equal(fwd, bwd):
        raise ValueError("not symmetric")


def csr_stats(g: CSRGraph) -> dict:
    deg = np.diff(g.rowptr.astype(np.int64))
    return {
        "n": g.n,
        "nnz": g.nnz,
        "undirected_edges": g.nnz // 2,
        "isolated": int(np.sum(deg == 0)),
        "max_degree": int(deg.max()) if g.n else 0,
    }


# ---------------------------------------------------------------- generators

def grid_graph(rows: int, cols: int) -> CSRGraph:
    """rows x cols grid; vertex (r, c) -> r*cols + c; edges right and down
    (32x32 -> 1,984 edges)."""
    r, c = np.meshgrid(np.arange(rows), np.arange(cols), indexing="ij")
    vid = r * cols + c
    u = [vid[:, :-1].ravel(), vid[:-1, :].ravel()]
    v = [vid[:, 1:].ravel(), vid[1:, :].ravel()]
    return edges_to_csr(rows * cols, np.concatenate(u), np.concatenate(v))


def tri_mesh_graph(rows: int, cols: int) -> CSRGraph:
    """rows x cols grid plus the down-right diagonal of every square
    (100x110 -> 32,581 edges)."""
    r, c = np.meshgrid(np.arange(rows), np.arange(cols), indexing="ij")
    vid = r * cols + c
    u = [vid[:, :-1].ravel(), vid[:-1, :].ravel(), vid[:-1, :-1].ravel()]
    v = [vid[:, 1:].ravel(), vid[1:, :].ravel(), vid[1:, 1:].ravel()]
    return edges_to_csr(rows * cols, np.concatenate(u), np.concatenate(v))


def ba_graph(n: int, m: int, seed: int) -> CSRGraph:
    """Barabasi-Albert preferential attachment.

    Seed graph: the single edge {0, 1}.  Each new vertex v = 2..n-1 attaches
    to min(m, v) *distinct* existing vertices drawn with probability
    proportional to degree, by sampling uniformly from the endpoint list and
    rejecting repeats.  n=6000, m=2 gives exactly 1 + 2*5998 = 11,997 edges.
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    endpoints = np.empty(2 + 2 * m * n, dtype=np.int64)
    endpoints[0], endpoints[1] = 0, 1
    ne = 2
    us, vs = [0], [1]
    for v in range(2, n):
        k = min(m, v)
        chosen: list[int] = []
        while len(chosen) < k:
            t = int(endpoints[int(rng.integers(0, ne))])
            if t not in chosen:
                chosen.append(t)
        for t in chosen:
            us.append(v)
            vs.append(t)
            endpoints[ne] = v
            endpoints[ne + 1] = t
            ne += 2
    return edges_to_csr(n, np.array(us), np.array(vs))


def rmat_graph(scale: int, edge_factor: int, a: float, b: float, c: float,
               seed: int) -> CSRGraph:
    """R-MAT: edge_factor * 2^scale sampled (u, v);
    per level the quadrant is a/b/c/d with no noise; symmetrised, self loops
    and duplicates removed, isolated vertices kept, no relabelling."""
    n = 1 << scale
    ne = edge_factor * n
    rng = np.random.Generator(np.random.PCG64(seed))
    u = np.zeros(ne, dtype=np.int64)
    v = np.zeros(ne, dtype=np.int64)
    ab = a + b
    abc = a + b + c
    for _level in range(scale):
        r = rng.random(ne)
        ubit = r >= ab                       # quadrants c, d -> lower half (row bit 1)
        vbit = ((r >= a) & (r < ab)) | (r >= abc)  # quadrants b, d -> right half
        u = (u << 1) | ubit
        v = (v << 1) | vbit
    return edges_to_csr(n, u, v)


def cycle_graph(n: int) -> CSRGraph:
    i = np.arange(n)
    return edges_to_csr(n, i, (i + 1) % n)


def star_graph(k: int) -> CSRGraph:
    """Vertex 0 is the centre, 1..k the leaves."""
    return edges_to_csr(k + 1, np.zeros(k, dtype=np.int64), np.arange(1, k + 1))


# ---------------------------------------------------------------- coordinates

def uniform_coords(n: int, seed: int) -> np.ndarray:
    """fp32 coordinates i.i.d. U[0,1)^2 (BASELINE.json configs), shape (n, 2),
    C-contiguous: x0, y0, x1, y1, ... (the float2 layout of the C-ABI)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return np.ascontiguousarray(rng.random((n, 2), dtype=np.float32))


def assert_no_coincident(xy: np.ndarray) -> None:
    """The reading C4 of SURVEY.md §8(c) makes coincident pairs contribute 0;
    the generators assert the inputs contain none (probability ~1e-4 at C5)."""
    keys = np.ascontiguousarray(xy, dtype=np.float32).view(np.int64).ravel()
    if np.unique(keys).size != keys.size:
        raise ValueError("coincident vertices in generated coordinates")
