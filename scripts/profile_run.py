"""One layout call of a named config (for ncu / compute-sanitizer runs).

  python scripts/profile_run.py [--config C5] [--iters 2] [--reps 1]
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
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--algo", type=int, default=0)
ap.add_argument("--theta", type=float, default=1.2)
a = ap.parse_args()
g, xy0, cfg = build_config(a.config)
with bl.BatchLayout(g.n, g.rowptr, g.colidx) as lay:
    for _ in range(a.reps):
        d = torch.from_numpy(xy0.copy()).cuda()
        lay.layout_device(d, iters=a.iters, batch=cfg.batch, K=cfg.K, C=cfg.C, step0=cfg.step0,
                          cooling=cfg.cooling, algo=a.algo, theta=a.theta)
        torch.cuda.synchronize()
    print("energy", lay.energy(a.iters)[0])
    import paper_2002_08233_b200 as _b
    print("visits", _b.bl_last_visits(lay.h))
