"""Benchmark: MC trial moves/s of the GCMC per-move energy path on B200.

Workload (BASELINE.json configs[3], "LJ fluid GCMC ~1M particles on 1 B200"):
N0 = 1,048,576 LJ particles, rho0 = 0.67 (L = 116.10 sigma), T = 2, mu = +1,
r_cut = 2.5 sigma, microcell strategy, 30/35/35 displace/insert/delete mix,
seed 1 (+ rank), random sequential start (init_config.hpp:19-64, 0.85 sigma).
One "step" = one gcmc_run_moves() batch of --moves-per-step Simulation::step()s
on the device (proposal generation + persistent engine). Synthetic data: the
reference's own random initial configuration.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Multi-GPU (torchrun, one process per GPU): every rank runs an independent
chain (seed 1 + rank) — "replicas only", no collective on the hot path; the
only NCCL call is the max-over-ranks of the timed region.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MC trial moves/sec"
PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
# microcell, reference layout, rho ~ 0.67: per window ~220
# occupancy words (4 B) + ~147 candidates x (4 B slot id + 24 B xyz) ~ 5.0 KB;
# 1.3 windows per move (0.3 x 2 + 0.7 x 1) -> 6.5 KB per move.
ALG_BYTES_PER_MOVE = 6.5e3


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n0", type=int, default=1 << 20)
    ap.add_argument("--density", type=float, default=0.67)
    ap.add_argument("--mu", type=float, default=1.0)
    ap.add_argument("--temperature", type=float, default=2.0)
    ap.add_argument("--strategy", default="microcell")
    ap.add_argument("--moves-per-step", type=int, default=None,
                    help="moves per chain per step (default 2^22; 2^20 with >= 12 chains per GPU)")
    ap.add_argument("--cpu-moves", type=int, default=100000,
                    help="(--impl reference) unused; kept for compatibility")
    ap.add_argument("--cpu-steps", type=int, default=1,
                    help="timed steps of the CPU baseline (the first timed GPU steps; "
                         "bounded to ~20 s of CPU work)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--chains-per-gpu", type=int, default=1,
                    help="independent chains sharing each GPU (gcmc_run_chains); "
                         "value = moves/s summed over all chains")
    ap.add_argument("--no-energy", action="store_true",
                    help="skip the full-system energy timing (full_system_energy block)")
    ap.add_argument("--sweep", action="store_true",
                    help="BASELINE configs[4]: mu isotherm sweep, one 64k chain per GPU "
                         "(rank g runs mu = -3 + g, seed 1 + g)")
    a = ap.parse_args(argv)
    if a.moves_per_step is None:
        a.moves_per_step = 1 << 20 if a.chains_per_gpu >= 12 else 1 << 22
    if a.sweep:
        if a.n0 == 1 << 20:
            a.n0 = 1 << 16
    return a


def state_point(a, rank, chain=0):
    """(mu, seed) of chain c of rank g: replicas of the same state point, or
    the isotherm sweep mu = -3 + g + c / K (K = 1: mu_g = -3 + g).
    No collective is needed on the hot path: chains are independent."""
    k = a.chains_per_gpu
    seed = 1 + rank * k + chain
    if a.sweep:
        return -3.0 + rank + chain / k, seed
    return a.mu, seed


def reduce_max(pg, values, device):
    """Max over ranks of the timed quantities (the only collective)."""
    if pg is None:
        return values
    import torch

    t = torch.tensor(values, dtype=torch.float64, device=device)
    pg.all_reduce(t, op=pg.ReduceOp.MAX)
    return [float(x) for x in t.tolist()]


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}",
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 3:
                try:
                    self.samples.append((float(parts[0]), float(parts[1]), int(parts[2], 16)))
                except ValueError:
                    pass

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        names = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
                 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
                 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}
        mask = 0
        for _, _, r in self.samples:
            mask |= r
        reasons = [v for k, v in names.items() if mask & k and k != 0x1]
        return {"sm_mhz": statistics.median(s[0] for s in self.samples),
                "sm_max_mhz": max(s[1] for s in self.samples), "reasons": reasons}


def hbm_peak():
    try:
        with open(PEAKS_FILE) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def config_dict(a, world):
    if a.sweep:
        wl = (f"mu/T isotherm sweep of {a.n0}-particle GCMC chains, 1 chain per GPU "
              f"(BASELINE configs[4]); rank g: mu = -3 + g")
    elif a.n0 == 1 << 20:
        wl = "LJ fluid GCMC ~1M particles on 1 B200 (BASELINE configs[3])"
    else:
        wl = f"LJ fluid GCMC N0={a.n0}"
    if a.chains_per_gpu > 1:
        wl += f", {a.chains_per_gpu} concurrent chains per GPU (gcmc_run_chains"
        wl += ", chain-per-SM engine: one CTA per chain, one launch)" if a.chains_per_gpu >= 12 else ")"
    k = a.chains_per_gpu
    mus = ([-3.0 + g + c / k for g in range(world) for c in range(k)] if a.sweep else a.mu)
    return {"workload": wl,
            "n0": a.n0, "density": a.density, "temperature": a.temperature,
            "mu": mus,
            "r_cut": 2.5, "strategy": a.strategy, "move_mix": "30/35/35",
            "moves_per_step": a.moves_per_step, "chains": world * k,
            "start": "random sequential insertion, 0.85 sigma (init_config.hpp:19-64)",
            "l2": "state (~70 MB at 1M) stays L2/HBM resident; inputs > L2 flush not needed: "
                  "each step reads a fresh 12 MB proposal stream and random cells",
            "parallelism": f"replicas x{world * k} ({k} independent chain(s) per GPU, "
                           f"seed 1 + rank * {k} + chain)"}


PROFILE_DIR = os.path.join(ROOT, "profiles")


def _load_json(name):
    try:
        with open(os.path.join(PROFILE_DIR, name)) as f:
            return json.load(f)
    except (OSError, ValueError):
        return None


def engine_profile():
    """ncu figures of one k_engine2 launch captured in the bench window
    (profiles/engine_ncu.json, written by tools/ncu_engine.py from
    `ncu --set full` of `bench.py` after its warm-up steps)."""
    return _load_json("engine_ncu.json")


def latency_block(eprof, ns_round, moves_round):
    """The roof that binds a serial chain: ns per round against a floor built
    from the round's dependent steps, each at its measured latency
    (profiles/ubench.json, tools/ubench/ubench.cu on the same B200 type):
    decision store -> evaluators see it (one-way cross-SM visibility), window
    positions + x_pid / e_pid (one L2 hop, issued together), the window's pair
    terms and a 128-thread reduction (dependent FP64 chain), slot result ->
    sequencer sees it (one-way), read / write sets (one L2 hop), then the
    next decision. Everything else in a round (walk, verify, commits) is
    overhead above this floor."""
    ub = _load_json("ubench.json")
    out = {"ns_per_round": ns_round, "moves_per_round": moves_round,
           "ns_per_move": ns_round / max(moves_round, 1e-9)}
    if eprof:
        for k in ("issue_active_pct", "fp64_pipe_pct", "warps_active_pct", "l2_hit_pct",
                  "dram_bytes_per_move"):
            if k in eprof:
                out[k] = eprof[k]
        out["ncu_source"] = eprof.get("source")
    if ub:
        ghz = ub["sm_ghz"]
        oneway = ub["pingpong_cycles"] / 2.0
        hop = ub["l2_relaxed_chase_cycles"]
        pair = ub["pair_term_cycles"]
        floor_cyc = 2 * oneway + 2 * hop + pair + 7 * ub.get("shfl_dadd_cycles", 40)
        floor_ns = floor_cyc / ghz
        out.update({"floor_ns_per_round": floor_ns, "floor_frac": floor_ns / ns_round,
                    "floor_model": "2 x one-way cross-SM visibility (half the measured ping-pong) + 2 x dependent L2 hop (ld.relaxed.gpu chase) + "
                                   "one pair term + 7-level shuffle reduction, "
                                   f"{ub['source']}"})
    return out


def energy_block(sim, peak):
    """Full-system energy (SURVEY §8a row c, gcmc_total_energy) on the chain's
    final state: device time of the pass and of the pair kernel (CUDA events),
    achieved HBM bytes (N x 24 B of coordinates: the pass's algorithmic
    input) per second against the HBM peak, and pair evaluations per second."""
    n = sim.dev.get_state().n
    passes, kern = [], []
    for _ in range(6):
        sim.dev.total_energy()
        p_ms, k_ms = sim.dev.energy_timing()
        passes.append(p_ms)
        kern.append(k_ms)
    p_ms = statistics.median(passes[1:])
    k_ms = statistics.median(kern[1:])
    rho = n / sim.cfg.volume()
    pairs = 0.5 * n * rho * 4.0 / 3.0 * math.pi * sim.cfg.r_cut ** 3  # within r_c
    ach = 24.0 * n / (p_ms * 1e-3) / 1e9
    ep = _load_json("energy_ncu.json") or {}
    return {"n": n, "pass_us": 1e3 * p_ms, "kernel_us": 1e3 * k_ms,
            "alg_bytes": 24 * n, "achieved_gbs": ach, "hbm_frac": ach / peak,
            "pairs_in_cutoff": pairs, "pairs_per_s": pairs / (p_ms * 1e-3),
            "issue_active_pct": ep.get("issue_active_pct"), "fp64_pipe_pct": ep.get("fp64_pipe_pct"),
            "dram_bytes_ncu": ep.get("dram_bytes"), "ncu_source": ep.get("source"),
            "kernel": "k_energy (energy.cu: warp per cell >= r_cut, 14-cell half shell, FP32 prefilter, compensated sums)"}


def host_cpu():
    """(model name, logical cores) of this host (lscpu / os.cpu_count)."""
    model = "unknown"
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:  # pragma: no cover
        pass
    return model, os.cpu_count()


def snapshot(sim):
    """Full chain state for the same-trajectory check (outside device timing)."""
    st = sim.dev.get_state()
    return {"xyz": sim.dev.positions(), "rng": sim.dev.get_rng().serialize_hex(),
            "step": st.step, "n": st.n, "u": st.energy, "w": st.virial,
            "attempted": list(st.attempted), "accepted": list(st.accepted)}


def cpu_chain(s0, s1, a, box, mu):
    """One chain of the CPU baseline: the reference's own Simulation::step
    loop (oracle/_ref, g++ -O3 with the reference's Release flags) resumed
    (engine.hpp:244-252) from the GPU chain's state s0 at the start of the
    timed steps and run on exactly the moves of the first --cpu-steps timed
    GPU steps. The run doubles as a parity check against the GPU chain's
    state s1 after those steps: positions and RNG state bitwise, step / N /
    per-kind attempted and accepted counts exact, U and W within 1e-10
    relative. Returns (seconds, checks or None, kind)."""
    import numpy as np

    import oracle as O

    timed = a.cpu_steps * a.moves_per_step
    if not os.path.exists(O.REF_SO):
        p = O.port_params(temperature=a.temperature, chemical_potential=mu, box_length=box,
                          strategy=a.strategy)
        sim = O.PortSim(p, s0["xyz"], O.rng_from_hex(s0["rng"]), energy=s0["u"], virial=s0["w"])
        t0 = time.perf_counter()
        sim.run(timed)
        return time.perf_counter() - t0, None, "port"
    cfg = O.ref_config(temperature=a.temperature, chemical_potential=mu, box_length=box,
                       strategy=a.strategy)
    sim = O.RefSim(cfg, mode=2, xyz=s0["xyz"], rng_hex=s0["rng"], step=s0["step"],
                   energy=s0["u"], virial=s0["w"])
    secs, _ = sim.run(timed)
    same = None
    if s1 is not None:
        st = sim.state()
        tol = lambda x, y: abs(x - y) <= 1e-10 * max(1.0, abs(y))  # noqa: E731
        checks = {
            "positions_bitwise": bool(np.array_equal(sim.positions(), s1["xyz"])),
            "rng_bitwise": sim.rng_hex() == s1["rng"],
            "step_n": st.step == s1["step"] and st.n == s1["n"],
            "counts": all(st.attempted[k] == s1["attempted"][k] - s0["attempted"][k] and
                          st.accepted[k] == s1["accepted"][k] - s0["accepted"][k]
                          for k in range(3)),
            "energy_1e-10": tol(s1["u"], st.energy) and tol(s1["w"], st.virial),
        }
        same = {"all": all(checks.values()), **checks}
    return secs, same, "reference"


def cpu_baseline(s0s, s1s, a, box, mus):
    """The CPU baseline on this host: one reference chain per GPU chain of
    rank 0 (sweep chains run one per core, concurrently), each
    on its own chain's moves; value = all chains' moves / wall time."""
    from concurrent.futures import ThreadPoolExecutor

    timed = a.cpu_steps * a.moves_per_step
    model, ncpu = host_cpu()
    # one reference chain per host core: with more GPU chains than cores, the
    # first ncpu chains (the host's full throughput, bounded CPU time)
    k = min(len(s0s), ncpu or 1)
    s0s, s1s, mus = s0s[:k], (s1s[:k] if s1s is not None else None), mus[:k]
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=min(k, ncpu or 1)) as ex:  # ctypes calls drop the GIL
        res = list(ex.map(lambda c: cpu_chain(s0s[c], s1s[c], a, box, mus[c]), range(k)))
    wall = time.perf_counter() - t0
    kind = res[0][2]
    same = None
    if all(r[1] is not None for r in res):
        same = dict(res[0][1]) if k == 1 else {"all": all(r[1]["all"] for r in res),
                                               "chains": [r[1] for r in res]}
    s0 = s0s[0]
    return ({"value": k * timed / wall, "unit": "moves/s", "cores": min(k, ncpu or 1),
             "kind": kind,
             "sample": f"moves {s0['step']}..{s0['step'] + timed} of each of the first {k} chain(s) (the "
                       f"first {a.cpu_steps} of the {a.steps} timed GPU steps), reference "
                       f"Simulation::step loop resumed from each GPU chain's state there, "
                       f"{wall:.2f} s wall, {min(k, ncpu or 1)} thread(s) on host '{model}' "
                       f"({ncpu} logical cores)"}, same)


def run_reference(a, rank, world):
    """--impl reference: the reference CPU implementation on this host."""
    if rank != 0:
        return
    import oracle as O

    box = (a.n0 / a.density) ** (1.0 / 3.0)
    mu, seed = state_point(a, 0)  # the GPU arm's chain 0 of rank 0
    xyz, hexs = O.ref_initial_configuration(a.n0, box, seed)  # the reference's own init
    cfg = O.ref_config(temperature=a.temperature, chemical_potential=mu, box_length=box,
                       strategy=a.strategy)
    # U/W only matter for reported observables, not for the trajectory; the
    # resume ctor avoids the O(N^2) total energy (hours at 1M on one core).
    sim = O.RefSim(cfg, mode=2, xyz=xyz, rng_hex=hexs, step=0, energy=0.0, virial=0.0)
    # warm-up: the same moves as the GPU arm's warm-up steps; then each timed
    # step is a bounded sample of 2^20 consecutive moves of the same chain
    # (the run stays within a few minutes on one core)
    for _ in range(a.warmup):
        sim.run(a.moves_per_step)

    per_step = min(a.moves_per_step, 1 << 20)
    secs = 0.0
    for _ in range(a.steps):
        s, _ = sim.run(per_step)
        secs += s
    moves = per_step * a.steps
    v = moves / secs
    line = {"metric": METRIC, "value": v, "unit": "moves/s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": 1e3 * secs / a.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(a, 1), "impl": "reference",
            "cpu_baseline": {"value": v, "unit": "moves/s", "cores": 1,
                             "kind": "reference" if os.path.exists(O.REF_SO) else "port",
                             "sample": f"{a.warmup} warm-up steps of {a.moves_per_step} moves, then "
                                       f"{a.steps} timed steps of {per_step} consecutive moves, "
                                       "reference Simulation::step loop (oracle/_ref, g++ -O3, "
                                       "proj/CMakeLists Release flags), same start state as the GPU arm"},
            "e2e": {"value": v, "unit": "moves/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def make_chains(a, rank, local, E, RunConfig):
    """This rank's chains: K = --chains-per-gpu sharing the device
    (engine_share = K); chain c is state point j = rank * K + c."""
    box = (a.n0 / a.density) ** (1.0 / 3.0)
    sims = []
    for c in range(a.chains_per_gpu):
        mu, seed = state_point(a, rank, c)
        xyz, rng = E.random_initial_configuration(a.n0, box, 0.85, seed, device=local)
        cfg = RunConfig(temperature=a.temperature, chemical_potential=mu, box_length=box,
                        strategy=a.strategy, seed=seed)
        kw = {"engine_share": a.chains_per_gpu} if a.chains_per_gpu > 1 else {}
        sims.append(E.Simulation(cfg, xyz, rng, device=local, **kw))
    return sims, box


def main():
    a = parse_args()
    rank, world, local = dist_env()
    if a.impl == "reference":
        run_reference(a, rank, world)
        return
    import torch

    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device")
    torch.cuda.set_device(local)
    pg = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = dist
    from paper_1408_3764_b200 import engine as E
    from paper_1408_3764_b200.config import RunConfig

    sims, box = make_chains(a, rank, local, E, RunConfig)
    sim = sims[0]
    K = len(sims)

    engine_used = [0]

    def step():
        """One step: --moves-per-step moves on every chain of this rank.
        Returns (device ms of the step, engine ms, rounds). One chain: the
        library's CUDA events (proposal generation + engine). K chains:
        CUDA events bracketing gcmc_run_chains (all K chains, concurrent)."""
        if K == 1:
            sim.run(a.moves_per_step)
            r = sim.last_run
            engine_used[0] = r.engine
            return r.device_ms + r.gen_ms, r.device_ms, r.rounds, r.pair_evals
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        res = E.run_chains(sims, a.moves_per_step)
        engine_used[0] = res[0].engine
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        return (ms, max(r.device_ms for r in res), sum(r.rounds for r in res),
                sum(r.pair_evals for r in res))

    for _ in range(a.warmup):
        step()

    # CPU baseline (rank 0, N=1 only): the reference resumed from chain 0's
    # exact state, timed on the same moves after the GPU's timed region
    if not a.cpu_steps or a.cpu_steps > a.steps:
        a.cpu_steps = a.steps
    want_cpu = rank == 0 and world == 1 and not a.no_cpu_baseline
    s0 = [snapshot(s_) for s_ in sims] if want_cpu else None
    s1 = None

    def barrier():
        torch.cuda.synchronize()
        if pg:
            pg.barrier()

    def accepted():
        return sum(sum(s.dev.get_state().accepted) for s in sims)

    # ---- device-resident timing (value)
    barrier()
    dev_ms = eng_ms = 0.0
    rounds = pairs = 0
    acc0 = accepted()
    with ClockSampler(local) as clk:
        for k in range(a.steps):
            d, e, r, pe = step()
            dev_ms += d
            eng_ms += e
            rounds += r
            pairs += pe
            if want_cpu and k + 1 == a.cpu_steps:
                s1 = [snapshot(s_) for s_ in sims]  # host read-back: not in the device timing
    barrier()
    acc1 = accepted()
    # ---- end-to-end through the C ABI (run + checkpoint read-back of state,
    #      RNG and positions to host memory), wall clock
    barrier()
    t0 = time.perf_counter()
    for _ in range(a.steps):
        if K == 1:
            sim.run(a.moves_per_step)
        else:
            E.run_chains(sims, a.moves_per_step)
        for s_ in sims:
            s_.dev.get_state()
            s_.dev.get_rng()
            s_.dev.positions()
    barrier()
    e2e_s = time.perf_counter() - t0

    cpu, same = None, None
    if want_cpu:
        try:
            cpu, same = cpu_baseline(s0, s1, a, box, [s_.cfg.chemical_potential for s_ in sims])
        except Exception as e:  # pragma: no cover
            cpu = {"value": None, "unit": "moves/s", "cores": 1, "kind": "reference",
                   "sample": f"failed: {e}"}

    moves_rank = a.moves_per_step * a.steps * K
    t_dev = dev_ms / 1e3
    t_dev, e2e_s = reduce_max(pg, [t_dev, e2e_s], "cuda")
    value = moves_rank * world / t_dev
    e2e = moves_rank * world / e2e_s
    peak, peak_kind = hbm_peak()
    launches = (a.moves_per_step + (1 << 21) - 1) >> 21  # engine launches per step and chain
    moves_per_launch = a.moves_per_step / launches
    eng_launch_s = eng_ms / 1e3 / (a.steps * launches)
    achieved = ALG_BYTES_PER_MOVE * moves_per_launch / eng_launch_s / 1e9
    sm_engine = engine_used[0] == 3
    eprof = None if sm_engine else engine_profile()
    traffic = eprof["dram_bytes_per_move"] * moves_per_launch if eprof else None
    n_final = [s_.dev.get_state().n for s_ in sims]
    ns_round = 1e9 * (eng_ms / 1e3) / max(rounds / K, 1)
    latency = (latency_block(eprof, ns_round, a.moves_per_step * a.steps * K / max(rounds, 1))
               if not sm_engine else
               {"ns_per_round": ns_round, "moves_per_round": a.moves_per_step * a.steps * K / max(rounds, 1),
                "note": "chain-per-SM engine: every hand-off of a round is a CTA barrier; "
                        "per-phase cycles in profiles/r02sm (GCMC_SM_PHASES=1)"})
    energy = energy_block(sim, peak) if rank == 0 and not a.no_energy else None
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "moves/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * t_dev / a.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config_dict(a, world),
            "e2e": {"value": e2e, "unit": "moves/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": sum(256 + 314 * 8 + 24 * x for x in n_final)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "peak_source": peak_kind,
                         "kernel": ("k_engine_sm (one CTA per chain, all chains of the GPU in one launch)"
                                    if sm_engine else
                                    "k_engine2 (persistent whole-GPU Metropolis loop, maintained per-particle energies)"),
                         "alg_bytes_per_move": ALG_BYTES_PER_MOVE,
                         "traffic_source": eprof["source"] if eprof else None,
                         "note": "serial Markov chain: latency-bound, not HBM-bound; the "
                                 "latency block is the roof that binds"},
            "latency": latency,
            "full_system_energy": energy,
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
            # per step, chain and 2^21-move chunk (gcmc_run_moves): the engine
            # plus the look-ahead proposal generation (k_gen2, k_annotate)
            # per step and 2^21-move chunk: K > 1 chain-per-SM chains go out as one
            # generator, one annotate and one engine launch for all chains
            "gpu_launches": (3 * a.steps * launches if sm_engine and K > 1
                             else 3 * a.steps * K * launches),
            "engine": {1: "per-window (engine.cu)", 2: "multi-SM maintained-energy (engine2.cu)",
                       3: "chain-per-SM (engine_sm.cu)"}.get(engine_used[0], "?"),
            "pair_evals_per_s": pairs * world / t_dev,
            "pair_evals_per_move": pairs / moves_rank,
            "pair_evals_note": "counted on the device (gcmc_run_result.pair_evals): FP64 "
                               "minimum-image + cutoff evaluations in move windows and "
                               "neighbour-energy updates; the engine scans one window per "
                               "move (maintained per-particle energies)",
            "ns_per_move": 1e9 * t_dev / moves_rank,
            "ns_per_round": ns_round,
            "moves_per_round": a.moves_per_step * a.steps * K / max(rounds, 1),
            "acceptance": (acc1 - acc0) / moves_rank,
            "n_final": n_final[0] if K == 1 else n_final,
        }
        if cpu and cpu.get("value"):
            line["speedup_vs_cpu_e2e"] = e2e / cpu["value"]
            line["speedup_vs_cpu_device"] = value / cpu["value"]
        if same is not None:
            # the CPU reference ran the identical moves: the full state agrees
            line["cpu_gpu_same_trajectory"] = same
        print(json.dumps(line), flush=True)
    for s_ in sims:
        s_.close()
    if pg:
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
