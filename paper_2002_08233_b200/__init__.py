"""paper_2002_08233_b200 -- B200-native BatchLayout exact path.

BatchLayout (Rahman, Sujon & Azad, arXiv:2002.08233) minibatch force-directed
layout, Alg. 2, as one persistent sm_100a kernel behind
the C-ABI of include/bl.h.  This package is the thin Python binding: it loads
the in-tree libbl.so (built by __graft_entry__.build()) and marshals
arguments.  PyTorch is used only for device memory and streams.
"""
from ._bl import (  # noqa: F401
    BL_OK, BL_EINVAL, BL_ENOMEM, BL_ECUDA, BL_ESTATE, BL_REPULSE_NEIGHBORS, BL_ATTRACTION_ONLY, BL_ALGO_EXACT,
    BL_ALGO_BH, EXPORTS,
    BLError, bl_params, bl_params_default, bl_greedy_init, bl_create, bl_layout, bl_layout_device,
    bl_energy, bl_forces, bl_max_vertices, bl_last_launch_count, bl_last_visits, bl_kernel_name, bl_driver_name, bl_edge_uniformity,
    bl_stress, bl_neighborhood_preservation, bl_microbench,
    bl_destroy, bl_debug_profile, bl_debug_check, bl_debug_counters, lib, _SO,
)
from .layout import BatchLayout  # noqa: F401
