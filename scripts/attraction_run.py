"""Step a5 alone on a named config (bl_forces with BL_ATTRACTION_ONLY over all
n vertices), for ncu: one warm-up launch, then --reps launches.

  python scripts/attraction_run.py --config C5 --reps 1
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2002_08233_b200 as bl  # noqa: E402
from blgen import build_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
g, xy0, cfg = build_config(a.config)
with bl.BatchLayout(g.n, g.rowptr, g.colidx) as lay:
    d = torch.from_numpy(xy0.copy()).cuda()
    for _ in range(1 + a.reps):
        f = lay.forces(d, 0, g.n, K=cfg.K, C=cfg.C, flags=bl.BL_ATTRACTION_ONLY)
    torch.cuda.synchronize()
    print("sum |S|", float(f.abs().sum()))
