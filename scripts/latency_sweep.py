"""Sweep kernel variants / driver knobs on the latency-bound configurations
 and print microseconds per dependent batch.

  python scripts/latency_sweep.py --configs C2,C3b256,C4 \
      --variants "T=8,TP=2;T=2,TP=1;T=2,TP=1,MU=4" [--iters 100]

A variant is a ';'-separated list of comma-separated knobs: T, TP, NT (kernel
variant, read at bl_create), MU (BL_MIN_UNIT4), ASYNC (BL_ASYNC), NSUB, SPIN,
CLUSTER.  Timing: CUDA events around bl_layout_device on the launching
stream, L2 flushed, median of --steps after 2 warm-ups.  Each variant's
result is also checked against the default variant's positions after one
iteration (max |dxy| / extent) as a sanity check (the parity proper is the
-m gpu suite)."""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2002_08233_b200 as bl  # noqa: E402
from blgen import build_config  # noqa: E402

KNOBS = {"T": "BL_T", "TP": "BL_TP", "NT": "BL_NT", "MU": "BL_MIN_UNIT4", "ASYNC": "BL_ASYNC",
         "NSUB": "BL_NSUB", "SPIN": "BL_SPIN", "CLUSTER": "BL_CLUSTER", "PIPE": "BL_PIPELINE", "LAT": "BL_LAT", "GUIDED": "BL_GUIDED"}


def parse(v):
    env = {}
    for kv in filter(None, v.split(",")):
        k, x = kv.split("=")
        env[KNOBS[k.strip()]] = x.strip()
    return env


def run(name, env, iters, steps, ref=None):
    for k in KNOBS.values():
        os.environ.pop(k, None)
    os.environ.update(env)
    g, xy0, cfg = build_config(name)
    it = iters or cfg.iters
    p = dict(iters=it, batch=cfg.batch, K=cfg.K, C=cfg.C, step0=cfg.step0, cooling=cfg.cooling)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    with bl.BatchLayout(g.n, g.rowptr, g.colidx) as lay:
        d0 = torch.from_numpy(xy0.copy()).cuda()
        d = torch.empty_like(d0)
        one = d0.clone()
        lay.layout_device(one, **dict(p, iters=1))
        torch.cuda.synchronize()
        one = one.cpu().numpy()
        for _ in range(2):
            d.copy_(d0)
            lay.layout_device(d, **p)
        torch.cuda.synchronize()
        ms = []
        for i in range(steps):
            d.copy_(d0)
            flush.fill_(float(i))
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            lay.layout_device(d, **p)
            b.record()
            b.synchronize()
            ms.append(a.elapsed_time(b))
        t = float(np.median(ms)) / 1e3
        nb = -(-g.n // cfg.batch)
        out = {"config": name, "env": env, "kernel": bl.bl_kernel_name(lay.h),
               "driver": bl.bl_driver_name(lay.h), "iters": it,
               "us_per_batch": 1e6 * t / (it * nb), "iters_per_sec": it / t}
        if ref is not None:
            out["vs_default_1it"] = float(np.abs(one - ref).max() / np.ptp(ref, 0).max())
    for k in KNOBS.values():
        os.environ.pop(k, None)
    return out, one


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C2,C3b256,C4")
    ap.add_argument("--variants", default="")
    ap.add_argument("--iters", type=int, default=100)
    ap.add_argument("--steps", type=int, default=3)
    a = ap.parse_args()
    for name in a.configs.split(","):
        base, ref = run(name, {}, a.iters, a.steps)
        print(json.dumps(base), flush=True)
        for v in filter(None, a.variants.split(";")):
            try:
                r, _ = run(name, parse(v), a.iters, a.steps, ref)
            except Exception as e:  # a variant the library rejects
                r = {"config": name, "env": parse(v), "error": str(e)}
            print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
