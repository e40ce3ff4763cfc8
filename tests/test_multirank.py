"""The N > 1 host path of bench.py on CPU (gloo, world size 2).

DESIGN.md §9: the layout does not shard across GPUs ("replicas only"), so
the multi-rank logic is the timing aggregation (max over ranks of the device
time, value = all ranks' units / that time) and the reference arm's
"rank 0 runs and prints, other ranks exit 0" rule.  Both are exercised here
without a GPU.
"""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, ROOT)
    import bench
    t_max = bench.max_over_ranks(1.5 + rank, world)          # per-rank device time
    value = bench.aggregate_value(units_per_rank=100.0, world=world, t_max=t_max)
    bench.barrier(world)
    q.put((rank, t_max, value))
    dist.destroy_process_group()


def test_max_over_ranks_and_aggregate_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    # both ranks see the slowest rank's time; value = 2 x 100 units / 2.5 s
    assert [g[1] for g in got] == [2.5, 2.5]
    assert [g[2] for g in got] == [80.0, 80.0]


def test_reference_arm_under_torchrun_gloo():
    """`bench.py --impl reference` launched like the driver's N = 2 run: rank 0
    alone times the oracle and prints ONE JSON line; rank 1 exits 0."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2", "--config",
           "C1", "--steps", "1", "--warmup", "0", "--ref-seconds", "0.3", "--backend", "gloo"]
    env = dict(os.environ, OMP_NUM_THREADS="2")
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.parametrize("world", [1, 2])
def test_aggregate_value_is_whole_job(world):
    sys.path.insert(0, ROOT)
    import bench
    assert bench.aggregate_value(units_per_rank=10.0, world=world, t_max=2.0) == 5.0 * world
