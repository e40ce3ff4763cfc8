"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic (no forces, no updates,
no energies).  It only builds graphs (as validated int32 CSR) and initial
fp32 coordinates, so that the oracle (`oracle/`) and the CUDA library
(`paper_2002_08233_b200/`) are fed identical bytes.

Stand-ins: the paper measures on SuiteSparse graphs and LFR graphs
(Table 1) that are not available here; the configs in
BASELINE.json (C1-C5) are synthetic graphs shaped like those workloads
(SURVEY.md §8(d)).
"""
from .graphs import (  # noqa: F401
    grid_graph, ba_graph, tri_mesh_graph, rmat_graph, cycle_graph, star_graph,
    edges_to_csr, validate_csr, csr_stats, uniform_coords, assert_no_coincident,
    CSRGraph,
)
from .configs import CONFIGS, LayoutConfig, get_config, build_config  # noqa: F401
