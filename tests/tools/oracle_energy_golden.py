"""Write tests/golden/energy_<cfg>.json: the ORACLE's full-run energy traces
for a config -- the unperturbed fp64 run, an ensemble of fp64 runs from
1-ulp-perturbed inputs (the chaos floor of SURVEY.md §8(c) (ii)/(iv)) and the
fp32 oracle -- for the -m gpu full-run energy tests, which are too long to
recompute on the GPU box's host at test time.

Calls only oracle/ and blgen/ (test infrastructure; no CUDA path).
Usage: python tests/tools/oracle_energy_golden.py C4 [--members 12] [--threads 0]
"""
import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from blgen import build_config  # noqa: E402


def input_digest(g, xy0):
    h = hashlib.sha256()
    for a in (np.int32(g.n), g.rowptr.astype(np.int32), g.colidx.astype(np.int32),
              np.ascontiguousarray(xy0, np.float32)):
        h.update(np.asarray(a).tobytes())
    return h.hexdigest()


def perturbed_inputs(xy0, members, seed=0):
    """1-ulp perturbations of every coordinate, each up or down at random
    (the same recipe as tests/test_gpu_parity.py's C1 ensemble)."""
    rng = np.random.default_rng(seed)
    up, down = np.float32(np.inf), np.float32(-np.inf)
    out = []
    for _ in range(members):
        direction = np.where(rng.random(xy0.shape) < 0.5, down, up).astype(np.float32)
        out.append(np.nextafter(xy0, direction))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--members", type=int, default=12)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--iters", type=int, default=0, help="0: the config's")
    ap.add_argument("--out", default="", help="output directory (default tests/golden)")
    args = ap.parse_args()
    g, xy0, cfg = build_config(args.config)
    iters = args.iters or cfg.iters
    kw = dict(iters=iters, batch=cfg.batch, K=cfg.K, C=cfg.C, step0=cfg.step0,
              cooling=cfg.cooling, threads=args.threads)
    t0 = time.time()
    _, E, _ = oracle.layout(g.n, g.rowptr, g.colidx, xy0, **kw)
    print(f"{args.config}: unperturbed done in {time.time() - t0:.0f} s, E_final {E[-1]:.9e}",
          flush=True)
    ens = []
    for k, xp in enumerate(perturbed_inputs(xy0, args.members)):
        _, Ek, _ = oracle.layout(g.n, g.rowptr, g.colidx, xp, **kw)
        ens.append(Ek.tolist())
        print(f"  member {k}: E_final {Ek[-1]:.9e} ({time.time() - t0:.0f} s)", flush=True)
    _, E32, _ = oracle.layout(g.n, g.rowptr, g.colidx, xy0, precision="f32", **kw)
    out = {
        "what": f"oracle energy traces for {args.config} (fp64 unperturbed, {args.members} "
                "fp64 runs from 1-ulp-perturbed xy0, fp32 oracle); written by "
                "tests/tools/oracle_energy_golden.py (calls only oracle/)",
        "config": args.config, "n": g.n, "nnz": int(g.nnz), "batch": cfg.batch, "iters": iters,
        "input_sha256": input_digest(g, xy0), "perturbation_seed": 0,
        "oracle_f64": E.tolist(), "ensemble_f64": ens, "oracle_f32": E32.tolist(),
        "seconds": time.time() - t0, "threads": oracle.max_threads() if not args.threads else args.threads,
    }
    path = os.path.join(args.out or os.path.join(ROOT, "tests", "golden"),
                        f"energy_{args.config}.json")
    with open(path, "w") as fh:
        json.dump(out, fh)
    print("wrote", path, flush=True)


if __name__ == "__main__":
    main()
