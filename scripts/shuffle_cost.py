"""Cost of batch randomisation per config, both realisations:
relabelled iterations (default) vs the in-kernel randomisation of the
two-barrier driver (BL_SHUFFLE_RELABEL=0), against the sequential default.
One JSON line per config.  GPU box only."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2002_08233_b200 as bl  # noqa: E402
from blgen import build_config  # noqa: E402


def timed(lay, d0, params, steps=3, warm=1):
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


def main():
    for name in (sys.argv[1:] or ["C1", "C2", "C3b64", "C3b256", "C3b1024", "C4", "C5"]):
        g, xy0, cfg = build_config(name)
        iters = min(cfg.iters, 50 if name != "C5" else 10)
        p = dict(iters=iters, batch=cfg.batch, K=cfg.K, C=cfg.C, step0=cfg.step0, cooling=cfg.cooling)
        with bl.BatchLayout(g.n, g.rowptr, g.colidx) as lay:
            d0 = torch.from_numpy(xy0.copy()).cuda()
            t_seq, d_seq = timed(lay, d0, p)
            os.environ.pop("BL_SHUFFLE_RELABEL", None)
            t_rl, d_rl = timed(lay, d0, dict(p, shuffle_seed=1))
            os.environ["BL_SHUFFLE_RELABEL"] = "0"
            t_ik, d_ik = timed(lay, d0, dict(p, shuffle_seed=1))
            os.environ.pop("BL_SHUFFLE_RELABEL", None)
        print(json.dumps({"config": name, "iters": iters, "ms_per_iter_sequential": t_seq / iters,
                          "driver_sequential": d_seq, "ms_per_iter_relabel": t_rl / iters,
                          "driver_relabel": d_rl, "ms_per_iter_inkernel": t_ik / iters,
                          "driver_inkernel": d_ik, "cost_relabel": t_rl / t_seq,
                          "cost_inkernel": t_ik / t_seq}), flush=True)


if __name__ == "__main__":
    main()
