"""BatchLayoutBH phase profile (BL_PROFILE=1, CTA 0 thread 0 clock64 marks).

  python scripts/profile_bh.py [--config C5] [--iters 3] [--theta 1.2]
Slots (us per iteration): bbox, sort, nodes, centroids, iteration glue,
forces (F, per batch summed), barrier waits.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["BL_PROFILE"] = "1"

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2002_08233_b200 as bl  # noqa: E402
from blgen import build_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--theta", type=float, default=1.2)
ap.add_argument("--noedges", action="store_true", help="same n and coordinates, no edges")
a = ap.parse_args()
g, xy0, cfg = build_config(a.config)
if a.noedges:
    from blgen import edges_to_csr
    g = edges_to_csr(g.n, np.array([], np.int64), np.array([], np.int64))
mhz = 1965.0
with bl.BatchLayout(g.n, g.rowptr, g.colidx) as lay:
    d = torch.from_numpy(xy0.copy()).cuda()
    for rep in range(2):
        d.copy_(torch.from_numpy(xy0))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        lay.layout_device(d, iters=a.iters, batch=cfg.batch, algo=1, theta=a.theta)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    pr = bl.bl_debug_profile(lay.h).astype(np.float64) / mhz
    names = ["bbox", "sort", "nodes", "centroids", "iter_glue", "forces", "barrier", "precompute"]
    nb = -(-g.n // cfg.batch)
    out = {"config": a.config, "theta": a.theta, "noedges": a.noedges, "iters": a.iters, "wall_ms": dt * 1e3,
           "us_per_iter": {k: round(v / a.iters, 1) for k, v in zip(names, pr[:8])},
           "us_per_batch_forces": round(pr[5] / (a.iters * nb), 2),
           "us_per_batch_barrier": round(pr[6] / (a.iters * nb), 2),
           "visits": bl.bl_last_visits(lay.h)}
    print(json.dumps(out))
