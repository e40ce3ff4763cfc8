"""Step a5 alone and the §3.7 metrics once each on C5 (for ncu captures).
  python scripts/metrics_run.py [--config C5] [--what attr,eu,stress,np]"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2002_08233_b200 as bl  # noqa: E402
from blgen import build_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--what", default="attr,eu")
a = ap.parse_args()
g, xy0, cfg = build_config(a.config)
with bl.BatchLayout(g.n, g.rowptr, g.colidx) as lay:
    d = torch.from_numpy(xy0.copy()).cuda()
    for w in a.what.split(","):
        if w == "attr":
            lay.forces(d, 0, g.n, flags=bl.BL_ATTRACTION_ONLY)
        elif w == "eu":
            bl.bl_edge_uniformity(lay.h, d)
        elif w == "stress":
            bl.bl_stress(lay.h, d, np.arange(64, dtype=np.int32))
        elif w == "np":
            bl.bl_neighborhood_preservation(lay.h, d, np.arange(256, dtype=np.int32))
    torch.cuda.synchronize()
print("ok")
