"""Warp-time breakdown of the asynchronous-phase driver (profiling build:
BL_NVCC_EXTRA=-DBL_PHASE_TS, run with BL_PROFILE=1): the fraction of all
warps' time spent in the entry gate, idle (nothing to grab), dirty waits,
sweep units, tile combines, update tasks and control tasks.

  BL_NVCC_EXTRA=-DBL_PHASE_TS python paper_2002_08233_b200/_build.py --force
  BL_PROFILE=1 python scripts/async_profile.py --config C5 --iters 5
"""
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
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--mhz", type=float, default=1965.0, help="SM clock for cycles -> us")
a = ap.parse_args()
g, xy0, cfg = build_config(a.config)
names = ["entry_gate", "idle", "dirty_wait", "units", "tile_combine", "updates", "control"]
with bl.BatchLayout(g.n, g.rowptr, g.colidx) as lay:
    d = torch.from_numpy(xy0.copy()).cuda()
    st = torch.cuda.Event(enable_timing=True)
    en = torch.cuda.Event(enable_timing=True)
    st.record()
    lay.layout_device(d, iters=a.iters, batch=cfg.batch, K=cfg.K, C=cfg.C, step0=cfg.step0,
                      cooling=cfg.cooling)
    en.record()
    torch.cuda.synchronize()
    pr = bl.bl_debug_profile(lay.h, 16 + 1024).astype(float)
    tot = pr[7]
    out = {"config": a.config, "iters": a.iters, "driver": bl.bl_driver_name(lay.h),
           "kernel": bl.bl_kernel_name(lay.h), "ms": st.elapsed_time(en),
           "warp_time_fraction": {n: pr[i] / tot for i, n in enumerate(names)}}
    busy = pr[8:8 + torch.cuda.get_device_properties(0).multi_processor_count]
    busy = busy / busy.mean()
    out["cta_busy_rel"] = {"min": float(busy.min()), "max": float(busy.max()),
                           "std": float(busy.std()),
                           "slowest_ctas": [int(i) for i in busy.argsort()[-8:][::-1]],
                           "fastest_ctas": [int(i) for i in busy.argsort()[:8]]}
    G = torch.cuda.get_device_properties(0).multi_processor_count
    hp = pr[8 + G:8 + G + 8]
    mhz = float(a.mhz)
    if hp.size >= 7 and hp[5] > 0 and bl.bl_driver_name(lay.h) == "latency":
        nph = hp[5]
        out["cta0_timeline_us_per_batch"] = {
            "barrier_and_detection": hp[0] / nph / mhz, "updates_to_join": hp[1] / nph / mhz,
            "wait_clean_partial": hp[2] / nph / mhz, "dirty_sweep_D": hp[3] / nph / mhz,
            "arrival_fence_red": hp[4] / nph / mhz, "phases": int(nph),
            "total_batch_us": out["ms"] * 1e3 / (a.iters * -(-g.n // cfg.batch))}
    elif hp.size >= 7 and hp[5] > 0:
        nph, nown = hp[5], max(hp[6], 1.0)
        out["cta0_timeline_us_per_batch"] = {
            "barrier_and_detection": hp[0] / nph / mhz, "control": hp[1] / nph / mhz,
            "updates_after_claim": hp[2] / nown / mhz, "tail_dirty_and_tiles": hp[3] / nph / mhz,
            "arrival_fence_red": hp[4] / nph / mhz, "phases": int(nph),
            "phases_with_updates": int(hp[6]),
            "total_batch_us": out["ms"] * 1e3 / (a.iters * -(-g.n // cfg.batch))}
    print(json.dumps(out, indent=1))
