"""Time the quality metrics on the GPU (CUDA events) for a config's seeded
layout.  python scripts/bench_metrics.py [--config C5] [--sources 1024] [--queries 0]"""
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
ap.add_argument("--sources", type=int, default=1024)
ap.add_argument("--queries", type=int, default=0, help="0 = all vertices")
a = ap.parse_args()
g, xy0, cfg = build_config(a.config)
rng = np.random.default_rng(0)
src = rng.choice(g.n, min(a.sources, g.n), replace=False).astype(np.int32)
qry = None if a.queries <= 0 else rng.choice(g.n, a.queries, replace=False).astype(np.int32)
out = {"config": a.config, "n": g.n, "nnz": int(g.nnz)}
with bl.BatchLayout(g.n, g.rowptr, g.colidx) as lay:
    d = torch.from_numpy(xy0.copy()).cuda()
    for name, fn in (("eu", lambda: bl.bl_edge_uniformity(lay.h, d)),
                     ("stress", lambda: bl.bl_stress(lay.h, d, src)),
                     ("np", lambda: bl.bl_neighborhood_preservation(lay.h, d, qry))):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = fn()
        e1.record()
        e1.synchronize()
        out[name] = {"value": r, "ms": e0.elapsed_time(e1)}
out["stress"]["sources"] = int(src.size)
out["np"]["queries"] = g.n if qry is None else int(qry.size)
out["stress"]["pairs_per_s"] = out["stress"]["value"][2] / (out["stress"]["ms"] / 1e3)
out["eu"]["bytes_per_s_algorithmic"] = (12.0 * g.nnz + 4.0 * (g.n + 1)) / (out["eu"]["ms"] / 1e3) * 2
print(json.dumps(out))
