"""Full-run energy check of the north star ("after a full run, the final
energy must match within 1% relative") with the chaos floor beside it, on one
config: the GPU's energy trace vs the fp64 oracle's, and the oracle from
1-ulp-perturbed inputs.  Slow on purpose (the C5 oracle is ~3.4e12 fp64 pair
evaluations per run).
  python tests/tools/full_run_energy.py --config C5 [--no-perturbed]"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from blgen import build_config  # noqa: E402
from tests.gpu_helpers import extent, gpu_layout  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--no-perturbed", action="store_true")
a = ap.parse_args()
g, xy0, cfg = build_config(a.config)
p = dict(iters=cfg.iters, batch=cfg.batch)
t0 = time.time()
got, trg, _ = gpu_layout(g, xy0, **p)
tg = time.time() - t0
t0 = time.time()
ref, E, _ = oracle.layout(g.n, g.rowptr, g.colidx, xy0, **p)
to = time.time() - t0
out = {"config": a.config, "iters": cfg.iters, "gpu_seconds": tg, "oracle_seconds": to,
       "oracle_threads": oracle.max_threads(),
       "energy_gpu": trg.tolist(), "energy_oracle": E.tolist(),
       "final_rel_diff": float(abs(trg[-1] - E[-1]) / E[-1]),
       "rel_diff_per_iteration": (np.abs(trg - E) / E).tolist(),
       "final_position_diff_over_extent": float(np.abs(got - ref).max() / extent(ref))}
if not a.no_perturbed:
    rng = np.random.default_rng(0)
    direction = np.where(rng.random(xy0.shape) < 0.5, -np.inf, np.inf).astype(np.float32)
    _, Ep, _ = oracle.layout(g.n, g.rowptr, g.colidx, np.nextafter(xy0, direction), **p)
    out["chaos_floor_final_1ulp"] = float(abs(Ep[-1] - E[-1]) / E[-1])
    out["chaos_floor_per_iteration"] = (np.abs(Ep - E) / E).tolist()
print(json.dumps(out))
