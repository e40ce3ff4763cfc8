"""Debug aid: repeatability of each driver after k batches, and which CTAs differ."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2002_08233_b200 as bl
from blgen import build_config
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
g, xy0, cfg = build_config(name)
G = torch.cuda.get_device_properties(0).multi_processor_count
with bl.BatchLayout(g.n, g.rowptr, g.colidx) as lay:
    for mb in [4, 5]:
        res = {}
        for lat in ("0", "0", "1", "1"):
            os.environ["BL_LAT"] = lat
            d = torch.from_numpy(xy0.copy()).cuda()
            lay.layout_device(d, iters=2, batch=cfg.batch, max_batches=mb)
            torch.cuda.synchronize()
            res.setdefault(lat, []).append(d.cpu().numpy())
        for lat in ("0", "1"):
            a, b = res[lat]
            print(mb, "driver", lat, "repeat maxdiff", np.abs(a - b).max())
        a, b = res["0"][0], res["1"][0]
        diff = np.abs(a - b).max(axis=1)
        bad = np.nonzero(diff > 0)[0]
        print(mb, "lat vs async: nbad", bad.size, "batches", np.bincount(bad // cfg.batch),
              "ctas", np.unique(bad % G).size, "of", G)
        # vertices changed from the start by each driver
        for lat in ("0", "1"):
            ch = np.nonzero(np.abs(res[lat][0] - xy0).max(axis=1) > 0)[0]
            print("   driver", lat, "moved vertices:", ch.size, "max id", ch.max() if ch.size else -1)
