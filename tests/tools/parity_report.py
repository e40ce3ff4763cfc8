"""Parity report of SURVEY.md §8(c)'s acceptance protocol, per config (GPU vs
the fp64 oracle on the same seeded bytes), written as one JSON document:

  one_batch      max |xy_gpu - xy_oracle| / extent after max_batches = 1
  one_iteration  the same after one full iteration (C5: max over the sampled
                 batches 0, 1, 128, 255, each recomputed by the oracle from the
                 GPU's own state -- shadowing)
  energy         |E_gpu - E_oracle| / E_oracle at the last compared iteration
                 (full run for C1-C3, the first `horizon` iterations for C4)
  chaos_floor    the oracle's own spread at that iteration: the same run from
                 1-ulp-perturbed inputs, and the fp32 oracle vs the fp64 one

  python tests/tools/parity_report.py [--configs C1,C2,...] > report.json
"""
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

HORIZON = {"C1": None, "C2": None, "C3b64": None, "C3b256": None, "C3b1024": None, "C4": 20,
           "C5": 0}


def err_over_extent(got, ref):
    return float(np.abs(np.asarray(got, np.float64) - ref).max() / extent(ref))


def report(name):
    g, xy0, cfg = build_config(name)
    b = cfg.batch
    out = {"config": name, "n": g.n, "nnz": int(g.nnz), "batch": b, "iters": cfg.iters}
    t0 = time.time()
    # one batch
    got, _, _ = gpu_layout(g, xy0, iters=1, batch=b, max_batches=1)
    ref, _, _ = oracle.layout(g.n, g.rowptr, g.colidx, xy0, iters=1, batch=b, max_batches=1)
    out["one_batch"] = err_over_extent(got, ref)
    # one iteration
    nb = -(-g.n // b)
    if name == "C5":
        worst = 0.0
        for t in (0, 1, 128, 255):
            s_t = xy0 if t == 0 else gpu_layout(g, xy0, iters=1, batch=b, max_batches=t)[0]
            s_t1 = gpu_layout(g, xy0, iters=1, batch=b, max_batches=t + 1)[0]
            lo, hi = t * b, min((t + 1) * b, g.n)
            f = oracle.forces(g.n, g.rowptr, g.colidx, s_t, lo, hi - lo)
            r = s_t.astype(np.float64).copy()
            r[lo:hi] += f / np.hypot(f[:, 0], f[:, 1])[:, None]
            worst = max(worst, err_over_extent(s_t1, r))
        out["one_iteration"] = worst
        out["one_iteration_note"] = "max over shadowed batches 0, 1, 128, 255"
    else:
        got, tr, _ = gpu_layout(g, xy0, iters=1, batch=b)
        ref, E, _ = oracle.layout(g.n, g.rowptr, g.colidx, xy0, iters=1, batch=b)
        out["one_iteration"] = err_over_extent(got, ref)
        out["one_iteration_energy_rel"] = float(abs(tr[0] - E[0]) / E[0])
    # energy over the horizon + chaos floor
    T = HORIZON[name]
    T = cfg.iters if T is None else T
    if T > 0:
        _, trg, _ = gpu_layout(g, xy0, iters=T, batch=b)
        _, E, _ = oracle.layout(g.n, g.rowptr, g.colidx, xy0, iters=T, batch=b)
        rng = np.random.default_rng(0)
        direction = np.where(rng.random(xy0.shape) < 0.5, -np.inf, np.inf).astype(np.float32)
        pert = np.nextafter(xy0, direction)
        _, Ep, _ = oracle.layout(g.n, g.rowptr, g.colidx, pert, iters=T, batch=b)
        _, E32, _ = oracle.layout(g.n, g.rowptr, g.colidx, xy0, iters=T, batch=b,
                                  precision="f32")
        out["energy"] = {"iteration": T, "gpu": float(trg[-1]), "oracle": float(E[-1]),
                         "rel_diff": float(abs(trg[-1] - E[-1]) / E[-1]),
                         "chaos_floor_1ulp": float(abs(Ep[-1] - E[-1]) / E[-1]),
                         "chaos_floor_fp32_oracle": float(abs(E32[-1] - E[-1]) / E[-1]),
                         "rel_diff_per_iteration_max_first10": float(
                             np.max(np.abs(trg[:10] - E[:10]) / E[:10]))}
    out["seconds"] = round(time.time() - t0, 1)
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C2,C3b64,C3b256,C3b1024,C4,C5")
    a = ap.parse_args()
    res = [report(c) for c in a.configs.split(",")]
    print(json.dumps({"report": "SURVEY.md §8(c) acceptance protocol, round 1, B200",
                      "tolerance": "positions 1e-4 x extent (north star)", "configs": res},
                     indent=1))
