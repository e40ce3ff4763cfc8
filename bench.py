#!/usr/bin/env python
"""bench.py -- BatchLayout exact path on B200 (one JSON line on rank 0).

A "step" is one whole C-ABI layout call over the workload (default C5:
R-MAT scale 18, n = 262,144, b = 1024, 50 iterations = 12,800 dependent
batches, exact all-pairs repulsion), i.e. one pass of every §8(a) row.
Metric (BASELINE.json): pair interactions/s = iters * n(n-1) / T, plus
iterations/s and the fraction of the FP32/SFU issue roofline.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5]
  python bench.py --impl reference ...   # the oracle (CPU) as reference arm

Multi-GPU (torchrun): replicas only -- each rank lays out its own copy of
the workload (independent problems, no data-path collective); value = all
ranks' pairs / max-over-ranks device time ("scaling": "weak").
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "pair interactions/sec"
UNIT = "pair/s"
MUFU_PER_CLK_SM = 16  # SFU lanes per SM per clock


# ------------------------------------------------------------------ helpers
def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def max_over_ranks(value: float, world: int, device=None) -> float:
    """Max of a per-rank scalar over all ranks (identity at world 1)."""
    if world <= 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_value(units_per_rank: float, world: int, t_max: float) -> float:
    """Whole-job throughput: the units all ranks processed / the slowest
    rank's time (replicas: every rank processes the same units)."""
    return world * units_per_rank / t_max


def load_traffic(workload: str, kernel: str):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum)
    from the committed `ncu --set full` capture of this workload's launch
    (profiles/traffic.json), or None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None, None
    with open(p) as fh:
        d = json.load(fh)
    e = d.get(workload)
    if not e or e.get("kernel") != kernel:
        return None, None
    return float(e["bytes_per_launch"]), e.get("source")


def load_pipes(workload: str, kernel: str):
    """Pipe utilisation of the timed kernel from the committed ncu capture
    (profiles/pipes.json: XU = MUFU, FMA, issue-active, % of peak sustained),
    or None."""
    p = os.path.join(ROOT, "profiles", "pipes.json")
    if not os.path.exists(p):
        return None
    with open(p) as fh:
        e = json.load(fh).get(workload)
    if not e or e.get("kernel") != kernel:
        return None
    return e


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            return json.load(fh), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    def __init__(self, index: int, period: float = 0.1):
        self.index, self.period = index, period
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        self.ok = False

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            return self
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def _run(self):
        nv = self._nv
        names = {
            "sw_power_cap": getattr(nv, "nvmlClocksThrottleReasonSwPowerCap", 0x4),
            "hw_slowdown": getattr(nv, "nvmlClocksThrottleReasonHwSlowdown", 0x8),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksThrottleReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksThrottleReasonHwThermalSlowdown", 0x40),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksThrottleReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            self._stop.wait(self.period)

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def workload_desc(name, g, cfg, args=None, world=1):
    """The `config` object of the JSON line -- identical for both arms."""
    a = getattr(args, "a", 2.0) if args is not None else 2.0
    r = getattr(args, "r", -1.0) if args is not None else -1.0
    return {
        "workload": f"{name}: {cfg.desc}, batch {cfg.batch}, {cfg.iters} iterations, exact all-pairs "
                    "repulsion, fp32 coords U[0,1)^2 seed 42",
        "n": g.n, "nnz": int(g.nnz), "batch": cfg.batch, "iters": cfg.iters,
        "K": cfg.K, "C": cfg.C, "step0": cfg.step0, "cooling": cfg.cooling,
        "energy_model": {"a": a, "r": r},
        "l2": "flushed (512 MiB write) before every timed step (GPU arm)",
        "parallelism": f"replicas x{world}" if world > 1 else "1 GPU",
    }


# ------------------------------------------------------------------ oracle leg
def oracle_sample(g, xy0, cfg, seconds: float, threads: int = 0):
    """Time the oracle (as it stands) on a bounded prefix of the workload:
    the first k batches of iteration 0, k calibrated to ~`seconds`."""
    import oracle
    b = min(cfg.batch, g.n)
    t0 = time.perf_counter()
    oracle.layout(g.n, g.rowptr, g.colidx, xy0, iters=1, batch=b, max_batches=1, threads=threads)
    t1 = time.perf_counter() - t0
    nb = (g.n + b - 1) // b
    k = int(max(1, min(nb * cfg.iters, seconds / max(t1, 1e-6))))
    return k, t1


def run_oracle(g, xy0, cfg, k, threads=0):
    import oracle
    b = min(cfg.batch, g.n)
    t0 = time.perf_counter()
    oracle.layout(g.n, g.rowptr, g.colidx, xy0, iters=cfg.iters, batch=b, max_batches=k,
                  threads=threads)
    dt = time.perf_counter() - t0
    nb = (g.n + b - 1) // b
    pairs = 0
    for t in range(k):
        lo = (t % nb) * b
        pairs += min(b, g.n - lo) * (g.n - 1)
    return pairs, dt


def cpu_cores():
    import oracle
    return int(oracle.max_threads())


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


# ------------------------------------------------------------------ main arms
def bench_reference(args, name, g, xy0, cfg, rank, world):
    if rank != 0:
        return 0
    k, t1 = oracle_sample(g, xy0, cfg, args.ref_seconds)
    for _ in range(args.warmup):
        run_oracle(g, xy0, cfg, max(1, k // 4))
    tot_pairs, tot_t = 0, 0.0
    for _ in range(args.steps):
        p, dt = run_oracle(g, xy0, cfg, k)
        tot_pairs += p
        tot_t += dt
    value = tot_pairs / tot_t
    b = min(cfg.batch, g.n)
    sample = (f"first {k} batch update(s) of iteration 0 of {name} (b={b}, each {b}x{g.n - 1} "
              f"pairs) per step; oracle fp64, OpenMP over batch vertices")
    cores = cpu_cores()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": workload_desc(name, g, cfg, args, world),
        "iters_per_sec": value / (g.n * (g.n - 1.0)),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def bench_ours(args, name, g, xy0, cfg, rank, world, local_rank):
    import torch

    import paper_2002_08233_b200 as bl

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream(dev)
    params = dict(iters=cfg.iters, batch=cfg.batch, K=cfg.K, C=cfg.C, step0=cfg.step0,
                  cooling=cfg.cooling, a=args.a, r=args.r)
    lay = bl.BatchLayout(g.n, g.rowptr, g.colidx)
    d_xy0 = torch.from_numpy(xy0.copy()).to(dev)
    d_xy = torch.empty_like(d_xy0)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2

    def step():
        d_xy.copy_(d_xy0)
        lay.layout_device(d_xy, stream=stream, **params)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    launches = 0
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(dev.index if dev.index is not None else 0) as clk:
        for i in range(args.steps):
            flush.fill_(float(i))                 # evict L2 between timed steps
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
            launches += bl.bl_last_launch_count(lay.h)
        torch.cuda.synchronize()
    barrier(world)
    ms = [a.elapsed_time(b) for a, b in ev]
    # per-step device time: the MEDIAN of the K timed steps,
    # max over ranks; the mean is reported beside it
    t_step = float(np.median(ms)) / 1e3
    t_max = max_over_ranks(t_step, world, dev if world > 1 and args.backend == "nccl" else None)
    t_mean = max_over_ranks(sum(ms) / 1e3 / args.steps, world,
                            dev if world > 1 and args.backend == "nccl" else None)
    pairs_per_step = cfg.iters * g.n * (g.n - 1.0)
    value = aggregate_value(pairs_per_step, world, t_max)
    e_last, trace, done = lay.energy(trace_len=cfg.iters)
    assert done == cfg.iters

    # ---- e2e through the host C-ABI call (H2D + kernel + D2H inside bl_layout)
    e2e_steps = max(1, min(args.steps, 3))
    pinned = torch.empty(xy0.shape, dtype=torch.float32).pin_memory()   # page-locked inputs
    buf = pinned.numpy()
    tot = 0.0
    for _ in range(e2e_steps):
        np.copyto(buf, xy0)                                        # fresh inputs, untimed
        flush.fill_(0.0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        bl.bl_layout(lay.h, buf, bl.bl_params_default(**params))   # includes H2D/D2H of xy
        e_l, _, _ = lay.energy(trace_len=cfg.iters)                # D2H of the energy trace
        tot += time.perf_counter() - t0
    e2e_t = max_over_ranks(tot, world, dev if world > 1 and args.backend == "nccl" else None)
    e2e_value = aggregate_value(e2e_steps * pairs_per_step, world, e2e_t)

    peaks, peak_src = load_peaks()
    clocks = clk.summary()
    sm_max = float(clocks.get("sm_max_mhz") or peaks.get("sm_max_mhz", 1965.0))
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    mufu_per_pair = 1 if args.r == -1.0 else 2   # r != -1: lg2 + ex2
    # SFU rate per SM per clock measured on this box (bl_microbench: MUFU.RCP
    # with clock64 on every SM), rounded to the lane count it resolves
    mb = bl.bl_microbench()
    mb_rates = [float(mb[k]) for k in ("ffma_per_clk_sm", "mufu_rcp_per_clk_sm",
                                        "mufu_rsq_per_clk_sm", "ffma2_lane_ops_per_clk_sm")]
    mufu_clk = float(round(mb_rates[1])) if 8 <= mb_rates[1] <= 32 else float(MUFU_PER_CLK_SM)
    peak = nsm * mufu_clk * sm_max * 1e6 / mufu_per_pair
    achieved = pairs_per_step / t_step
    kname = bl.bl_kernel_name(lay.h)
    traffic, traffic_src = load_traffic(name, kname)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * t_max, "ms_per_step_mean": 1e3 * t_mean,
        "ms_per_step_all": [round(x, 4) for x in ms], "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": workload_desc(name, g, cfg, args, world),
        "iters_per_sec": world * cfg.iters / t_max,
        "roofline": {
            "bound": "alu", "achieved": achieved, "peak": peak, "unit": UNIT,
            "frac": achieved / peak, "traffic": traffic,
            "traffic_source": traffic_src,
            "kernel": kname + " (persistent, cooperative; NT threads, T targets/thread, TP of them "
                              "paired-reciprocal)",
            "driver": bl.bl_driver_name(lay.h),
            "peak_basis": f"{nsm} SMs x {mufu_clk:g} MUFU/clk (bl_microbench on this box: "
                          f"{mb_rates[1]:.2f}) x {sm_max:.0f} MHz (sm_max_mhz, {peak_src}) / "
                          f"{mufu_per_pair} MUFU per pair",
            "microbench_ops_per_clk_sm": {"ffma": mb_rates[0], "mufu_rcp": mb_rates[1],
                                          "mufu_rsq": mb_rates[2], "ffma2": mb_rates[3]},
            "frac_at_median_clock": (achieved * mufu_per_pair
                                     / (nsm * mufu_clk * clocks["sm_mhz"] * 1e6)
                                     if clocks.get("sm_mhz") else None),
            "pipes": load_pipes(name, kname),
        },
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 8 * g.n,
                "d2h_bytes_per_step": 8 * g.n + 8 * cfg.iters},
        "gpu_launches": launches,
        "clocks": clocks,
        "energy_final": e_last,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        k, _ = oracle_sample(g, xy0, cfg, args.cpu_seconds)
        pairs, dt = run_oracle(g, xy0, cfg, k)
        b = min(cfg.batch, g.n)
        line["cpu_baseline"] = {
            "value": pairs / dt, "unit": UNIT, "cores": cpu_cores(), "kind": "oracle",
            "cpu_model": cpu_model(), "per_core": pairs / dt / max(1, cpu_cores()),
            "sample": f"first {k} batch update(s) of iteration 0 of {name} (b={b}), {dt:.1f} s",
        }
    if not args.no_bh:
        line["bh"] = bench_bh(args, lay, d_xy0, params, stream, flush, g, cfg, t_step)
    line["attraction"] = bench_attraction(lay, d_xy0, params, stream, flush, g, peaks)
    if not args.no_metrics:
        line["metrics"] = bench_metrics(lay, d_xy, g, peaks, clocks.get("sm_mhz") or sm_max, nsm,
                                        stream)
    if not args.no_shuffle and cfg.batch <= 2048:
        line["shuffle"] = bench_shuffle(args, lay, d_xy0, params, stream, flush, cfg, t_step)
    if args.latency_configs and args.r == -1.0:
        line["latency"] = bench_latency(args, dev, stream, flush, peak)
    lay.close()
    if args.prof and rank == 0:
        line["phase_profile"] = phase_profile(g, xy0, params, dev, clocks.get("sm_mhz") or sm_max)
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def bench_bh(args, lay, d_xy0, params, stream, flush, g, cfg, exact_s):
    """Secondary line: BatchLayoutBH (algo = BL_ALGO_BH, Alg. S1-S3, theta =
    1.2 of P:869) on the same workload, same timing rules (L2 flushed, CUDA
    events on the launching stream, >= 1 warm-up)."""
    import torch

    import paper_2002_08233_b200 as bl
    p = dict(params, algo=bl.BL_ALGO_BH, theta=args.theta)
    d_xy = torch.empty_like(d_xy0)
    steps = max(2, args.steps)
    for _ in range(max(1, min(args.warmup, 2))):
        d_xy.copy_(d_xy0)
        lay.layout_device(d_xy, stream=stream, **p)
    torch.cuda.synchronize()
    ms = []
    for i in range(steps):
        d_xy.copy_(d_xy0)
        flush.fill_(float(i))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        lay.layout_device(d_xy, stream=stream, **p)
        b.record(stream)
        b.synchronize()
        ms.append(a.elapsed_time(b))
    visits = bl.bl_last_visits(lay.h)
    t = sum(ms) / 1e3 / steps
    return {"algo": f"BatchLayoutBH (Alg. S3), theta {args.theta}", "kernel": "bl_bh_kernel<512>",
            "iters_per_sec": cfg.iters / t, "ms_per_step": 1e3 * t, "steps": steps,
            "visits_per_step": visits, "visits_per_sec": visits / t,
            "speedup_vs_exact": exact_s / t, "gpu_launches_per_step": bl.bl_last_launch_count(lay.h)}


def bench_latency(args, dev, stream, flush, peak_per_sm_clk):
    """Secondary objects: the latency-bound configurations (SURVEY.md §8(a)
    a9: C2, C3 b=256, C4 -- 0.3-1.8 us of roofline work per dependent batch
    against a grid barrier of ~1.3 us), same timing rules as the headline
    (L2 flushed, CUDA events on the launching stream, median of the timed
    steps after warm-ups)."""
    import torch

    import paper_2002_08233_b200 as bl
    from blgen import build_config
    out = {}
    for name in args.latency_configs.split(","):
        if not name:
            continue
        g, xy0, cfg = build_config(name)
        params = dict(iters=cfg.iters, batch=cfg.batch, K=cfg.K, C=cfg.C, step0=cfg.step0,
                      cooling=cfg.cooling)
        with bl.BatchLayout(g.n, g.rowptr, g.colidx) as lay:
            d0 = torch.from_numpy(xy0.copy()).to(dev)
            d = torch.empty_like(d0)
            for _ in range(3):
                d.copy_(d0)
                lay.layout_device(d, stream=stream, **params)
            torch.cuda.synchronize()
            ms = []
            for i in range(max(3, min(args.steps, 5))):
                d.copy_(d0)
                flush.fill_(float(i))
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                lay.layout_device(d, stream=stream, **params)
                b.record(stream)
                b.synchronize()
                ms.append(a.elapsed_time(b))
            t = float(np.median(ms)) / 1e3
            nb = -(-g.n // cfg.batch)
            pairs = cfg.iters * g.n * (g.n - 1.0)
            out[name] = {
                "iters_per_sec": cfg.iters / t, "ms_per_step": 1e3 * t,
                "us_per_dependent_batch": 1e6 * t / (cfg.iters * nb),
                "pair_per_s": pairs / t, "roofline_frac": pairs / t / peak_per_sm_clk,
                "driver": bl.bl_driver_name(lay.h), "kernel": bl.bl_kernel_name(lay.h),
                "steps": len(ms), "gpu_launches_per_step": bl.bl_last_launch_count(lay.h)}
    return out


def _time_layout(lay, d_xy0, params, stream, flush, steps, warmup=2):
    import torch
    d = torch.empty_like(d_xy0)
    for _ in range(warmup):
        d.copy_(d_xy0)
        lay.layout_device(d, stream=stream, **params)
    torch.cuda.synchronize()
    ms = []
    for i in range(steps):
        d.copy_(d_xy0)
        flush.fill_(float(i))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        lay.layout_device(d, stream=stream, **params)
        b.record(stream)
        b.synchronize()
        ms.append(a.elapsed_time(b))
    return float(np.median(ms)) / 1e3


def bench_shuffle(args, lay, d_xy0, params, stream, flush, cfg, t_default):
    """Secondary object: batch randomisation (shuffle_seed, §4.3.3)
    on the same workload ("Randomization also introduces overhead").
    Default: every iteration relabelled into position space (one extra launch,
    csrc/bl_relabel.cu) and run by the sequential driver; `inkernel` is the
    round-2 first version, randomised inside the two-barrier driver
    (BL_SHUFFLE_RELABEL=0)."""
    import paper_2002_08233_b200 as bl
    steps = max(2, min(args.steps, 3))
    t_shuf = _time_layout(lay, d_xy0, dict(params, shuffle_seed=1), stream, flush, steps)
    drv = bl.bl_driver_name(lay.h)
    launches = bl.bl_last_launch_count(lay.h)
    os.environ["BL_SHUFFLE_RELABEL"] = "0"
    try:
        t_ik = _time_layout(lay, d_xy0, dict(params, shuffle_seed=1), stream, flush, 2, warmup=1)
        drv_ik = bl.bl_driver_name(lay.h)
    finally:
        os.environ.pop("BL_SHUFFLE_RELABEL", None)
    return {"shuffle_seed": 1, "driver": drv, "iters_per_sec": cfg.iters / t_shuf,
            "ms_per_step": 1e3 * t_shuf, "gpu_launches_per_step": launches,
            "default_iters_per_sec": cfg.iters / t_default,
            "cost_vs_default": t_shuf / t_default,
            "inkernel": {"driver": drv_ik, "iters_per_sec": cfg.iters / t_ik,
                         "cost_vs_default": t_ik / t_default}}


def bench_metrics(lay, d_xy, g, peaks, sm_mhz, nsm, stream, sources=1024):
    """Secondary object: the §3.7 quality metrics on the bench's
    final layout, each with a stated roofline fraction:
      EU: 2 passes x (4 nnz + 4 (n+1) + 8 n) algorithmic bytes vs HBM;
      stress: bit-parallel BFS (256 sources per 256-bit mask) -- bytes =
        36 B per CSR entry examined (index + mask gather) + 72 B per vertex
        per level (visited, next, rowptr) vs HBM, and TEPS (sources x nnz /
        t, the Graph500 convention);
      NP: the brute-force definition's n - 1 squared-distance evaluations per
        query (the one-scan threshold kernels do exactly that for deg <= 256;
        the radix select of the few larger queries does ~5 scans), 5 FP32
        lane-ops each, vs the FP32 lane peak.
    Timed with CUDA events around the (synchronous) C-ABI calls, after one
    warm-up call (the scratch is allocated once per context)."""
    import torch

    import paper_2002_08233_b200 as bl
    hbm = float(peaks.get("hbm_gbs", 6540.2)) * 1e9
    rng = np.random.default_rng(0)
    src = rng.choice(g.n, min(sources, g.n), replace=False).astype(np.int32)

    def timed(fn, reps):
        """median GPU time of the call's kernels (CUDA events recorded by the
        library on the call's stream around its kernels, bl_debug_counters)
        and the median wall time of the synchronous C-ABI call"""
        fn()
        gpu, wall = [], []
        for _ in range(reps):
            t0 = time.perf_counter()
            r = fn()
            wall.append(time.perf_counter() - t0)
            gpu.append(bl.bl_debug_counters(lay.h)[2] * 1e-9)
        return r, float(np.median(gpu)), float(np.median(wall))

    eu, t_eu, w_eu = timed(lambda: bl.bl_edge_uniformity(lay.h, d_xy, stream), 5)
    eu_bytes = 2.0 * (4 * g.nnz + 4 * (g.n + 1) + 8 * g.n)
    st, t_st, w_st = timed(lambda: bl.bl_stress(lay.h, d_xy, src, stream), 2)
    levels, examined, _ = bl.bl_debug_counters(lay.h)
    st_bytes = 36.0 * examined + 72.0 * g.n * levels
    npv, t_np, w_np = timed(lambda: bl.bl_neighborhood_preservation(lay.h, d_xy, None, stream), 2)
    evals = float(g.n - 1) * g.n
    fp32_evals = nsm * 128 * sm_mhz * 1e6 / 5.0
    return {
        "layout": "the bench's final layout",
        "timing": "GPU time of each call's kernels (CUDA events around them, inside the "
                  "library); call_us/call_ms = wall time of the synchronous C-ABI call",
        "edge_uniformity": {"value": eu, "us": 1e6 * t_eu, "call_us": 1e6 * w_eu,
                            "algorithmic_bytes": eu_bytes,
                            "GB_per_s": eu_bytes / t_eu / 1e9, "frac_of_hbm_peak": eu_bytes / t_eu / hbm},
        "stress": {"value": st[0], "sources": int(src.size), "ms": 1e3 * t_st, "call_ms": 1e3 * w_st,
                   "pairs": int(st[2]), "pairs_per_s": st[2] / t_st, "bfs_levels": levels,
                   "csr_entries_examined": examined, "teps": src.size * g.nnz / t_st,
                   "algorithmic_bytes": st_bytes, "frac_of_hbm_peak": st_bytes / t_st / hbm},
        "neighborhood_preservation": {
            "value": npv[0], "queries": g.n, "ms": 1e3 * t_np, "call_ms": 1e3 * w_np,
            "distance_evals": evals,
            "evals_per_s": evals / t_np, "frac_of_fp32_peak": evals / t_np / fp32_evals},
    }


def bench_attraction(lay, d_xy0, params, stream, flush, g, peaks):
    """Step a5 alone (bl_forces with BL_ATTRACTION_ONLY over all n vertices:
    the CSR attraction + neighbour correction of one whole iteration, one
    launch: 8 lanes per short row, 256-entry chunks of long rows).  Algorithmic bytes: 4 B
    colidx + 8 B gathered coordinate per CSR entry, rowptr, own coordinate
    read + S_i write.  In the layout these gathers hit L2 (CSR + xy = 19 MB
    at C5 stay resident), so `l2_warm` is the in-situ condition; `hbm_cold`
    flushes L2 first."""
    import torch

    import paper_2002_08233_b200 as bl
    p = dict(params, flags=int(params.get("flags", 0)) | bl.BL_ATTRACTION_ONLY)
    nbytes = 12 * g.nnz + 4 * (g.n + 1) + 16 * g.n
    out = {}
    # l2_warm: the average launch duration over 20 back-to-back launches
    # (CUDA events around all of them on the launching stream, queued behind
    # a sleep kernel so the host's per-call overhead is not timed)
    lay.forces(d_xy0, 0, g.n, stream=stream, **p)
    torch.cuda.synchronize()
    reps = 20
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(4_000_000)  # ~2 ms: the host enqueues all launches before the first runs
    a.record(stream)
    for _ in range(reps):
        lay.forces(d_xy0, 0, g.n, stream=stream, **p)
    b.record(stream)
    b.synchronize()
    t = a.elapsed_time(b) / reps / 1e3
    out["l2_warm"] = {"us": 1e6 * t, "GB_per_s": nbytes / t / 1e9, "launches_timed": reps,
                      "frac_of_hbm_peak": nbytes / t / 1e9 / float(peaks.get("hbm_gbs", 6540.2))}
    # hbm_cold: L2 flushed before each launch, the median of 5 single launches
    for mode in ("hbm_cold",):
        lay.forces(d_xy0, 0, g.n, stream=stream, **p)
        torch.cuda.synchronize()
        ms = []
        for i in range(5):
            flush.fill_(float(i))
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            lay.forces(d_xy0, 0, g.n, stream=stream, **p)
            b.record(stream)
            b.synchronize()
            ms.append(a.elapsed_time(b))
        t = float(np.median(ms)) / 1e3
        out[mode] = {"us": 1e6 * t, "GB_per_s": nbytes / t / 1e9,
                     "frac_of_hbm_peak": nbytes / t / 1e9 / float(peaks.get("hbm_gbs", 6540.2))}
    out.update({"step": "a5 (CSR attraction + neighbour correction), all n vertices, one launch",
                "algorithmic_bytes": nbytes, "csr_entries": int(g.nnz),
                "kernel": bl.bl_kernel_name(lay.h),
                "gpu_launches": bl.bl_last_launch_count(lay.h),
                "note": "standalone row-parallel kernel (bl_attr.cuh: 8 lanes per row of <= 64 "
                        "entries, 256-entry warp chunks of longer rows, 8 gathers in flight per "
                        "lane); in the layout the same arithmetic runs inside the update tasks"})
    return out


def phase_profile(g, xy0, params, dev, mhz):
    """One extra (untimed) run with BL_PROFILE=1: CTA-0 phase breakdown (us)
    and the spread of per-CTA phase-R busy time."""
    import torch

    import paper_2002_08233_b200 as bl
    os.environ["BL_PROFILE"] = "1"
    try:
        lay = bl.BatchLayout(g.n, g.rowptr, g.colidx)
    finally:
        os.environ.pop("BL_PROFILE", None)
    d = torch.from_numpy(xy0.copy()).to(dev)
    lay.layout_device(d, **params)
    torch.cuda.synchronize()
    pr = bl.bl_debug_profile(lay.h).astype(np.float64) / mhz  # cycles -> us
    lay.close()
    # pipelined driver: 1 = warp 0's task loop, 2 = in-CTA tail + combine,
    # 3 = loop glue, 5 = arrive; 0, 4, 7 (barrier-to-control, control, updates
    # after control) only in a -DBL_PHASE_TS build
    names = ["barrier_to_control", "tasks_warp0", "cta_tail_combine", "glue", "control",
             "arrive", "end", "updates_after_control"]
    busy = pr[8:]
    return {"cta0_us": {k: round(float(v), 1) for k, v in zip(names, pr[:8])},
            "phaseR_busy_us": {"min": float(busy.min()), "median": float(np.median(busy)),
                               "max": float(busy.max())}}


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-seconds", type=float, default=8.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--backend", default="nccl")
    ap.add_argument("--prof", action="store_true", help="add a phase profile (extra untimed run)")
    ap.add_argument("--no-bh", action="store_true", help="skip the secondary BatchLayoutBH line")
    ap.add_argument("--no-shuffle", action="store_true", help="skip the batch-randomisation object")
    ap.add_argument("--no-metrics", action="store_true", help="skip the quality-metrics object")
    ap.add_argument("--theta", type=float, default=1.2, help="BatchLayoutBH MAC threshold (P:869)")
    ap.add_argument("--latency-configs", default="C2,C3b256,C4",
                    help="secondary latency-bound configs ('' to skip)")
    ap.add_argument("--a", type=float, default=2.0, help="(a, r)-model attraction exponent (P:531)")
    ap.add_argument("--r", type=float, default=-1.0, help="(a, r)-model repulsion exponent")
    args = ap.parse_args(argv)
    if args.warmup < 3 and args.impl == "ours":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)

    rank, world, local_rank = dist_env()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group(backend=args.backend, init_method="env://")

    from blgen import build_config
    g, xy0, cfg = build_config(args.config)
    if args.impl == "reference":
        rc = bench_reference(args, args.config, g, xy0, cfg, rank, world)
    else:
        rc = bench_ours(args, args.config, g, xy0, cfg, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return rc


if __name__ == "__main__":
    sys.exit(main())
