"""The five BASELINE.json configurations.

C3 has a batch sweep (64/256/1024); each batch size is its own entry.
Parameters the paper leaves unstated use the readings of SURVEY.md §8(c):
K = 1, C (the paper's R) = 1 (C6); step0 = 1.0 and cooling 0.999 are the
paper's (Alg. 2).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from functools import lru_cache

import numpy as np

from . import graphs


@dataclass(frozen=True)
class LayoutConfig:
    name: str
    desc: str
    batch: int
    iters: int
    graph_seed: int = 1
    coord_seed: int = 42
    K: float = 1.0
    C: float = 1.0
    step0: float = 1.0
    cooling: float = 0.999
    extra: dict = field(default_factory=dict, hash=False, compare=False)


CONFIGS: dict[str, LayoutConfig] = {
    "C1": LayoutConfig("C1", "2-D grid 32x32 (1,024 vertices, 1,984 edges)", 256, 100),
    "C2": LayoutConfig("C2", "Barabasi-Albert n=6,000 m=2 (11,997 edges)", 256, 600),
    "C3b64": LayoutConfig("C3b64", "triangulated mesh 100x110 (11,000 vertices), batch 64", 64, 600),
    "C3b256": LayoutConfig("C3b256", "triangulated mesh 100x110 (11,000 vertices), batch 256", 256, 600),
    "C3b1024": LayoutConfig("C3b1024", "triangulated mesh 100x110 (11,000 vertices), batch 1024", 1024, 600),
    "C4": LayoutConfig("C4", "R-MAT scale 15, edge factor 16 (32,768 vertices)", 256, 600),
    "C5": LayoutConfig("C5", "R-MAT scale 18, edge factor 8 (262,144 vertices)", 1024, 50),
    # beyond BASELINE.json: a 2^20-vertex graph, the size class where the paper
    # runs only BatchLayoutBH; used for the BH measurements
    "C6": LayoutConfig("C6", "R-MAT scale 20, edge factor 8 (1,048,576 vertices)", 1024, 20),
}

RMAT_ABCD = (0.57, 0.19, 0.19)


def get_config(name: str) -> LayoutConfig:
    return CONFIGS[name]


@lru_cache(maxsize=None)
def _graph(name: str) -> graphs.CSRGraph:
    base = name[:2]
    cfg = CONFIGS[name]
    if base == "C1":
        return graphs.grid_graph(32, 32)
    if base == "C2":
        return graphs.ba_graph(6000, 2, cfg.graph_seed)
    if base == "C3":
        return graphs.tri_mesh_graph(100, 110)
    if base == "C4":
        return graphs.rmat_graph(15, 16, *RMAT_ABCD, seed=cfg.graph_seed)
    if base == "C5":
        return graphs.rmat_graph(18, 8, *RMAT_ABCD, seed=cfg.graph_seed)
    if base == "C6":
        return graphs.rmat_graph(20, 8, *RMAT_ABCD, seed=cfg.graph_seed)
    raise KeyError(name)


def build_config(name: str) -> tuple[graphs.CSRGraph, np.ndarray, LayoutConfig]:
    """(graph, xy0 fp32 (n,2), cfg) for a named config; validated."""
    cfg = CONFIGS[name]
    g = _graph(name)
    graphs.validate_csr(g.n, g.rowptr, g.colidx)
    xy = graphs.uniform_coords(g.n, cfg.coord_seed)
    graphs.assert_no_coincident(xy)
    return g, xy, cfg
