"""Memory-ordering evidence for the exact kernel's hand-rolled protocols
(the pool closes compute-sanitizer): the CHECKED build of the
same sources (libbl_checked.so, -DBL_CHECKED) stamps every value one CTA
hands another -- the per-CTA repulsion partials, the new coordinates in
pend, the committed coordinates in xy -- with the batch it comes from, and
every reader verifies that it got EXACTLY the batch Alg. 2 prescribes
(frozen coordinates within a batch, the previous batch's update visible to
the next: P:626-627), plus bounds, completion-token and slot
invariants.  BL_JITTER=<seed> adds seeded random sleeps (0-2 us) at every
task boundary to shake the interleavings.  Every run must record zero
violations and produce results BITWISE equal to the production library
(fixed summation orders; P:1102-1103's thread-count independence).
Marked gpu."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from blgen import build_config
from tests.gpu_helpers import gpu_layout

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_2002_08233_b200", "libbl_checked.so")

# (config, iterations, driver environment, extra params)
CASES = [
    ("C3b256", 2, {"BL_ASYNC": "0"}, {}),                  # pipelined driver
    ("C3b256", 2, {"BL_ASYNC": "1"}, {}),                  # asynchronous phases
    ("C3b256", 1, {"BL_PIPELINE": "0"}, {}),               # two-barrier driver
    ("C4", 2, {"BL_ASYNC": "1"}, {}),                      # async, hub rows
    ("C4", 2, {}, {}),                                      # latency driver (default), hub rows
    ("C2", 3, {"BL_ASYNC": "0"}, {}),                      # pipelined
    ("C3b1024", 1, {"BL_LAT": "1"}, {"max_batches": 17}),  # latency driver, stop mid-iteration
    ("C3b1024", 1, {"BL_ASYNC": "1"}, {"max_batches": 17}),  # stop mid-iteration
    ("C3b256", 2, {}, {"shuffle_seed": 7}),                # randomised batches, relabelled (latency driver)
    ("C3b256", 1, {"BL_SHUFFLE_RELABEL": "0"}, {"shuffle_seed": 7}),  # randomised in the two-barrier driver
    ("C2", 2, {"BL_ASYNC": "1", "BL_T": "2", "BL_TP": "1"}, {}),  # small-tile variant
]


def _checked(name, iters, env, extra, jitter, tmp_path):
    out = str(tmp_path / f"{name}_{jitter}.npz")
    e = dict(os.environ, BL_LIBRARY=CHECKED, BL_JITTER=str(jitter), BL_CLUSTER="0", **env)
    args = [sys.executable, os.path.join(ROOT, "scripts", "checked_run.py"), name, str(iters), out]
    args += [f"{k}={v}" for k, v in extra.items()]
    r = subprocess.run(args, env=e, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    rec = json.loads(r.stdout.strip().splitlines()[-1])
    z = np.load(out)
    return rec, z["xy"], z["trace"]


@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}-{'-'.join(f'{k}{v}' for k, v in c[2].items()) or 'default'}-{'-'.join(c[3]) or 'plain'}" for c in CASES])
def test_checked_build_no_violations_and_bitwise_equal(case, tmp_path, monkeypatch):
    if not os.path.exists(CHECKED):
        pytest.fail("libbl_checked.so missing: __graft_entry__.build() builds it")
    name, iters, env, extra = case
    for k, v in dict(env, BL_CLUSTER="0").items():
        monkeypatch.setenv(k, v)
    g, xy0, cfg = build_config(name)
    ref, rtr, _ = gpu_layout(g, xy0, iters=iters, batch=cfg.batch, K=cfg.K, C=cfg.C,
                             step0=cfg.step0, cooling=cfg.cooling, **extra)
    for jitter in (0, 1, 2):
        rec, xy, tr = _checked(name, iters, env, extra, jitter, tmp_path)
        assert rec["kind"] == 1 and rec["library"] == "libbl_checked.so", rec
        assert rec["violations"] == 0, rec
        assert np.array_equal(xy, ref), (rec, float(np.abs(xy - ref).max()))
        assert np.array_equal(tr, rtr), rec


def test_checked_build_detects_a_broken_protocol(tmp_path):
    """The checks are live (mutation test): BL_CHK_BREAK=1 makes the checked
    build's control task skip its wait for the grid barrier, so update tasks
    read partial rows and coordinates before every CTA has written them --
    the stamps must report it."""
    # whether a skipped wait reads stale data depends on the interleaving: the
    # seeded jitter (0-2 us sleeps at task boundaries) makes it near certain,
    # several seeds make the test independent of one box's timing
    recs = []
    for jitter in (1, 2, 3, 0):
        rec, _, _ = _checked("C3b256", 1, {"BL_ASYNC": "0", "BL_CHK_BREAK": "1"}, {}, jitter, tmp_path)
        assert rec["kind"] == 1, rec
        recs.append(rec)
        if rec["violations"] > 0:
            break
    assert any(r["violations"] > 0 for r in recs), recs
