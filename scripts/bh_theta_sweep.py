"""BatchLayoutBH speed/accuracy trade-off over theta on one config: per theta,
iterations/s of the full layout (CUDA events) and the mean / max relative
error of the BH forces against the exact forces (both from the GPU, bl_forces)
on the first 2,048 vertices of the seeded layout.
  python scripts/bh_theta_sweep.py [--config C5] [--iters 10]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2002_08233_b200 as bl  # noqa: E402
from blgen import build_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--iters", type=int, default=10)
a = ap.parse_args()
g, xy0, cfg = build_config(a.config)
out = {"config": a.config, "n": g.n, "iters": a.iters, "rows": []}
with bl.BatchLayout(g.n, g.rowptr, g.colidx) as lay:
    d0 = torch.from_numpy(xy0.copy()).cuda()
    fe = lay.forces(d0, 0, 2048, flags=1).cpu().numpy().astype(np.float64)  # exact, neighbours repel
    for theta in (0.0, 0.3, 0.6, 0.9, 1.2, 1.6, 2.0):
        fb = lay.forces(d0, 0, 2048, algo=1, theta=theta).cpu().numpy().astype(np.float64)
        rel = np.hypot(*(fb - fe).T) / np.hypot(*fe.T)
        d = torch.empty_like(d0)
        for rep in range(2):
            d.copy_(d0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            lay.layout_device(d, iters=a.iters, batch=cfg.batch, algo=1, theta=theta)
            e1.record()
            e1.synchronize()
        ms = e0.elapsed_time(e1)
        out["rows"].append({"theta": theta, "iters_per_sec": a.iters / (ms / 1e3),
                            "visits_per_iter": bl.bl_last_visits(lay.h) / a.iters,
                            "force_rel_err_mean": float(rel.mean()),
                            "force_rel_err_max": float(rel.max())})
print(json.dumps(out))
