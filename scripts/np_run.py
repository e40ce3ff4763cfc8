"""Neighbourhood preservation over all vertices of a config's seeded layout,
once (for ncu launch lists of the three NP kernels).
  python scripts/np_run.py [--config C5]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2002_08233_b200 as bl  # noqa: E402
from blgen import build_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
a = ap.parse_args()
g, xy0, cfg = build_config(a.config)
with bl.BatchLayout(g.n, g.rowptr, g.colidx) as lay:
    d = torch.from_numpy(xy0.copy()).cuda()
    print(bl.bl_neighborhood_preservation(lay.h, d, None))
