"""Single-cluster kernel vs the whole-GPU latency driver on small graphs
(us per dependent batch): where is the crossover now that the latency driver
exists?  BL_CLUSTER=1 forces nothing -- it lets launch_cluster decide by
BL_CLUSTER_PAIRS (set huge here); BL_CLUSTER=0 turns it off.  GPU box only."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2002_08233_b200 as bl  # noqa: E402
from blgen import grid_graph, uniform_coords  # noqa: E402


def timed(lay, d0, params, steps=5, warm=2):
    d = torch.empty_like(d0)
    ms = []
    for i in range(warm + steps):
        d.copy_(d0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        lay.layout_device(d, **params)
        b.record()
        b.synchronize()
        if i >= warm:
            ms.append(a.elapsed_time(b))
    return float(np.median(ms)), bl.bl_driver_name(lay.h)


CASES = [(32, 32, 256), (32, 32, 64), (50, 40, 128), (50, 40, 256), (64, 64, 64), (64, 64, 128),
         (64, 64, 256), (100, 110, 64), (100, 110, 32), (100, 80, 128), (128, 128, 64)]
os.environ["BL_CLUSTER_PAIRS"] = "2000000000"
for (r, c, b) in CASES:
    g = grid_graph(r, c)
    xy0 = uniform_coords(g.n, 42)
    nb = -(-g.n // b)
    iters = max(4, 4000 // nb)
    p = dict(iters=iters, batch=b)
    out = {"n": g.n, "b": b, "bn": g.n * b, "nb": nb}
    with bl.BatchLayout(g.n, g.rowptr, g.colidx) as lay:
        d0 = torch.from_numpy(xy0.copy()).cuda()
        for mode in ("1", "0"):
            os.environ["BL_CLUSTER"] = mode
            t, drv = timed(lay, d0, p)
            out[drv] = 1e3 * t / (iters * nb)
    print(json.dumps(out), flush=True)
