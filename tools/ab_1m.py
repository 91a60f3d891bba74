"""A/B of engine shapes at the 1M bench state: warm 2^24 moves, then time
2^23 (device ms of gcmc_run_moves). Prints moves/s, moves per round, us per
round and a hash of the final positions (the chain must not change).
    GCMC_LIB=... python tools/ab_1m.py --group 64"""
import argparse, hashlib, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1408_3764_b200 import engine as E
from paper_1408_3764_b200.config import RunConfig

ap = argparse.ArgumentParser()
ap.add_argument("--group", type=int, default=0)
ap.add_argument("--n0", type=int, default=1 << 20)
ap.add_argument("--warm", type=int, default=1 << 24)
ap.add_argument("--moves", type=int, default=1 << 23)
ap.add_argument("--mu", type=float, default=1.0)
a = ap.parse_args()
box = (a.n0 / 0.67) ** (1 / 3)
xyz, rng = E.random_initial_configuration(a.n0, box, 0.85, 1, device=0)
cfg = RunConfig(temperature=2.0, chemical_potential=a.mu, box_length=box, strategy="microcell")
sim = E.Simulation(cfg, xyz, rng, engine_group=a.group)
sim.run(a.warm)
sim.run(a.moves)
r = sim.last_run
h = hashlib.sha1(sim.particles().tobytes()).hexdigest()[:16]
print(json.dumps({"lib": os.path.basename(os.environ.get("GCMC_LIB", "default")), "group": a.group,
                  "moves_per_s": a.moves / (r.device_ms / 1e3), "moves_per_round": a.moves / max(1, r.rounds),
                  "us_per_round": 1e3 * r.device_ms / max(1, r.rounds), "engine": r.engine, "hash": h,
                  "n": sim.particle_count()}), flush=True)
