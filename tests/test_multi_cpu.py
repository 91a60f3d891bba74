"""The N>1 path of bench.py on CPU (gloo, world size 2).

A single Markov chain does not shard: N GPUs run N independent
chains — replicas of the state point or the mu isotherm sweep of
BASELINE configs[4] — and the only collective is the max over ranks of the
timed region. These tests cover that host logic without a GPU.
"""
from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_state_points_replicas_and_sweep():
    a = bench.parse_args([])
    assert a.n0 == 1 << 20 and not a.sweep
    assert [bench.state_point(a, r) for r in range(3)] == [(1.0, 1), (1.0, 2), (1.0, 3)]
    s = bench.parse_args(["--sweep"])
    assert s.n0 == 1 << 16  # BASELINE configs[4]: 64k chains
    assert [bench.state_point(s, g)[0] for g in range(8)] == [-3.0 + g for g in range(8)]
    assert len({bench.state_point(s, g)[1] for g in range(8)}) == 8  # distinct seeds
    cfg = bench.config_dict(s, 4)
    assert cfg["mu"] == [-3.0, -2.0, -1.0, 0.0] and "configs[4]" in cfg["workload"]


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = bench.reduce_max(dist, [float(rank + 1), 10.0 - rank], "cpu")
    q.put((rank, out))
    dist.destroy_process_group()


def test_max_over_ranks_gloo_world2():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res[0] == res[1] == [2.0, 10.0]


def test_reference_arm_world2_prints_one_line():
    """`bench.py --impl reference` launched like the driver's N=2 run:
    rank 0 times the reference CPU loop, rank 1 exits without work."""
    import oracle as O

    if not os.path.exists(O.REF_SO):
        pytest.skip("oracle/_ref not built")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py",
           "--impl", "reference", "--gpus", "2", "--n0", "2048", "--moves-per-step", "4000",
           "--steps", "2", "--warmup", "1"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["n_gpus"] == 2
    assert d["cpu_baseline"]["kind"] == "reference"
