"""Debug: one-batch / one-iteration parity errors per config, repeated."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import oracle
from blgen import build_config
from tests.gpu_helpers import gpu_layout, extent

names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["C3b1024"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
for name in names:
    g, xy0, cfg = build_config(name)
    for mb in (1, 0):
        p = dict(iters=1, batch=cfg.batch, max_batches=mb)
        ref, _, _ = oracle.layout(g.n, g.rowptr, g.colidx, xy0, iters=1, batch=cfg.batch, max_batches=mb)
        ext = extent(ref)
        outs = []
        for r in range(reps):
            got, _, _ = gpu_layout(g, xy0, **p)
            err = np.abs(got - ref).max(axis=1)
            bad = np.nonzero(err > 1e-4 * ext)[0]
            outs.append(got)
            print(name, "mb", mb, "rep", r, "pipe", os.environ.get("BL_PIPELINE", "1"),
                  "err/ext %.2e" % (err.max() / ext), "nbad", bad.size, bad[:10], flush=True)
        print("  deterministic:", all(np.array_equal(outs[0], o) for o in outs[1:]))
