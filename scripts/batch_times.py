"""Per-batch cost of the first batches of an iteration vs the average: launch
the layout with max_batches = k for several k (median of reps, CUDA events)
and difference consecutive k.  Shows whether hub-heavy early batches (R-MAT:
low ids have the highest degrees) dominate the dependent chain.

  python scripts/batch_times.py --config C4 [--ks 1,2,3,4,5,6,8,16,64,128]
"""
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
ap.add_argument("--config", default="C4")
ap.add_argument("--ks", default="1,2,3,4,5,6,7,8,12,16,32,64,128")
ap.add_argument("--reps", type=int, default=7)
a = ap.parse_args()
g, xy0, cfg = build_config(a.config)
ks = [int(x) for x in a.ks.split(",")]
res = {}
with bl.BatchLayout(g.n, g.rowptr, g.colidx) as lay:
    d0 = torch.from_numpy(xy0.copy()).cuda()
    d = torch.empty_like(d0)
    for k in ks:
        ms = []
        for r in range(a.reps + 1):
            d.copy_(d0)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            lay.layout_device(d, iters=2, batch=cfg.batch, K=cfg.K, C=cfg.C, max_batches=k)
            e.record()
            e.synchronize()
            if r:
                ms.append(s.elapsed_time(e))
        res[k] = float(np.median(ms)) * 1e3
    drv = bl.bl_driver_name(lay.h)
deg = np.diff(g.rowptr)
nb = -(-g.n // cfg.batch)
out = {"config": a.config, "driver": drv, "us_at_max_batches": res,
       "us_per_batch_between": {f"{ks[i]}->{ks[i+1]}": (res[ks[i + 1]] - res[ks[i]]) / (ks[i + 1] - ks[i])
                                for i in range(len(ks) - 1)},
       "max_degree_in_batch": [int(deg[t * cfg.batch:(t + 1) * cfg.batch].max()) for t in range(min(nb, 8))]}
print(json.dumps(out, indent=1))
