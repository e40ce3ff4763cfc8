"""One layout through the CHECKED library (libbl_checked.so, -DBL_CHECKED;
DESIGN.md §14) in a fresh process (the library is chosen at import via
BL_LIBRARY): prints the violation record as JSON and saves the final
positions and energy trace for a bitwise comparison with the production
library.

  BL_LIBRARY=paper_2002_08233_b200/libbl_checked.so BL_JITTER=3 \\
      python scripts/checked_run.py C3b256 2 out.npz [key=value ...]
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2002_08233_b200 as bl  # noqa: E402
from blgen import build_config  # noqa: E402


def main():
    name, iters, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    extra = {}
    for kv in sys.argv[4:]:
        k, v = kv.split("=")
        extra[k] = int(v) if v.lstrip("-").isdigit() else float(v)
    g, xy0, cfg = build_config(name)
    p = dict(iters=iters, batch=cfg.batch, K=cfg.K, C=cfg.C, step0=cfg.step0,
             cooling=cfg.cooling)
    p.update(extra)
    with bl.BatchLayout(g.n, g.rowptr, g.colidx) as lay:
        d = torch.from_numpy(xy0.copy()).cuda()
        lay.layout_device(d, **p)
        torch.cuda.synchronize()
        kind, rec = bl.bl_debug_check(lay.h)
        try:
            _, tr, done = lay.energy(trace_len=iters)
        except bl.BLError:
            tr, done = np.zeros(0), 0
        np.savez(out, xy=d.cpu().numpy(), trace=tr)
        print(json.dumps({"config": name, "params": p, "library": os.path.basename(bl._SO),
                          "kind": kind, "violations": int(rec[0]), "first_code": int(rec[1]),
                          "detail": [int(x) for x in rec[2:5]], "driver": bl.bl_driver_name(lay.h),
                          "kernel": bl.bl_kernel_name(lay.h), "iters_done": int(done),
                          "jitter": os.environ.get("BL_JITTER", "0")}))


if __name__ == "__main__":
    main()
