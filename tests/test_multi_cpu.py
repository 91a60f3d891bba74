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


def test_chains_per_gpu_state_points():
    """--chains-per-gpu K: chain c of rank g is state point g * K + c: sweep
    mu = -3 + g + c / K, distinct seeds over the whole job."""
    s = bench.parse_args(["--sweep", "--chains-per-gpu", "4"])
    pts = [bench.state_point(s, g, c) for g in range(2) for c in range(4)]
    assert [p[0] for p in pts] == [-3.0 + g + c / 4 for g in range(2) for c in range(4)]
    assert len({p[1] for p in pts}) == 8
    cfg = bench.config_dict(s, 2)
    assert cfg["chains"] == 8 and len(cfg["mu"]) == 8 and "4 concurrent chains" in cfg["workload"]
    r = bench.parse_args(["--chains-per-gpu", "3"])
    assert {bench.state_point(r, 0, c)[0] for c in range(3)} == {1.0}


def test_latency_floor_from_measured_latencies(tmp_path, monkeypatch):
    """The latency block's floor: 2 one-way visibilities (half a ping-pong) +
    2 L2 hops + one pair term + 7 shuffle-add levels, in ns at the SM clock."""
    ub = {"source": "test", "sm_ghz": 2.0, "l2_relaxed_chase_cycles": 400, "pingpong_cycles": 1400,
          "pair_term_cycles": 300, "shfl_dadd_cycles": 40}
    (tmp_path / "ubench.json").write_text(json.dumps(ub))
    monkeypatch.setattr(bench, "PROFILE_DIR", str(tmp_path))
    lat = bench.latency_block({"issue_active_pct": 7.0, "source": "x"}, 20000.0, 350.0)
    floor = (1400 + 2 * 400 + 300 + 7 * 40) / 2.0
    assert abs(lat["floor_ns_per_round"] - floor) < 1e-9
    assert abs(lat["floor_frac"] - floor / 20000.0) < 1e-12
    assert lat["issue_active_pct"] == 7.0 and abs(lat["ns_per_move"] - 20000.0 / 350.0) < 1e-9


def test_profiles_summaries_are_consistent():
    """The committed bench-window ncu summaries bench.py reads exist and are
    self-consistent (traffic per move = traffic per launch / moves)."""
    e = json.load(open(os.path.join(ROOT, "profiles", "engine_ncu.json")))
    assert abs(e["dram_bytes_per_move"] * e["moves_per_launch"] - e["dram_bytes_per_launch"]) < 1.0
    assert 0 < e["issue_active_pct"] < 100 and 0 < e["fp64_pipe_pct"] < 100
    en = json.load(open(os.path.join(ROOT, "profiles", "energy_ncu.json")))
    assert en["duration_us"] > 0 and en["dram_bytes"] > 0
    u = json.load(open(os.path.join(ROOT, "profiles", "ubench.json")))
    assert u["pingpong_cycles"] > 0 and u["l2_relaxed_chase_cycles"] > 0
