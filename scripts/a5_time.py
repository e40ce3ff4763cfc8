"""Step a5 alone (bl_forces with BL_ATTRACTION_ONLY over all n vertices):
mean device time of --reps back-to-back launches after warm-up (L2-warm), for
same-box A/B runs.  python scripts/a5_time.py [--config C5] [--reps 50]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2002_08233_b200 as bl  # noqa: E402
from blgen import build_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--reps", type=int, default=50)
a = ap.parse_args()
g, xy0, cfg = build_config(a.config)
with bl.BatchLayout(g.n, g.rowptr, g.colidx) as lay:
    d = torch.from_numpy(xy0.copy()).cuda()
    out = torch.empty((g.n, 2), dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream()
    prm = bl._bl.bl_params_default(K=cfg.K, C=cfg.C, flags=bl.BL_ATTRACTION_ONLY)
    for _ in range(5):
        bl._bl.bl_forces(lay.h, d, 0, g.n, out, prm, st)
    torch.cuda.synchronize()
    ref = out.clone()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(a.reps):
        bl._bl.bl_forces(lay.h, d, 0, g.n, out, prm, st)
    e1.record(st)
    e1.synchronize()
    us = 1e3 * e0.elapsed_time(e1) / a.reps
    byts = 12 * g.nnz + 4 * (g.n + 1) + 16 * g.n
    print(json.dumps({"config": a.config, "env": {k: v for k, v in os.environ.items() if k.startswith("BLA_")},
                      "us": us, "GB_per_s": byts / us / 1e3, "bitwise_same": bool(torch.equal(out, ref))}))
