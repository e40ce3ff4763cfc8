"""Debug aid: latency driver vs the asynchronous driver after k batches."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2002_08233_b200 as bl
from blgen import build_config
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
g, xy0, cfg = build_config(name)
nb = -(-g.n // cfg.batch)
with bl.BatchLayout(g.n, g.rowptr, g.colidx) as lay:
    for mb in [1, 2, 3, 4, 5, 6, 8, nb, nb + 3]:
        res = {}
        for lat in ("0", "1"):
            os.environ["BL_LAT"] = lat
            d = torch.from_numpy(xy0.copy()).cuda()
            lay.layout_device(d, iters=2, batch=cfg.batch, max_batches=mb)
            torch.cuda.synchronize()
            kind, chk = bl.bl_debug_check(lay.h)
            res[lat] = (d.cpu().numpy(), bl.bl_driver_name(lay.h))
            if kind and chk[0]:
                print("  checked:", lat, list(chk))
        a, b = res["0"][0], res["1"][0]
        diff = np.abs(a - b).max(axis=1)
        bad = np.nonzero(diff > 1e-6)[0]
        print(mb, res["0"][1], res["1"][1], "maxdiff", diff.max(), "nbad", bad.size,
              "first bad", bad[:8], "batches", sorted(set((bad // cfg.batch).tolist()))[:10])
