"""Small end-to-end run for compute-sanitizer (memcheck / racecheck /
synccheck): 2k particles, both grid strategies, engine moves, ΔE batch,
total energy, device initial configuration.
    compute-sanitizer --tool racecheck python tools/sanitize_run.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1408_3764_b200 import engine as E
from paper_1408_3764_b200.config import RunConfig

moves = int(os.environ.get("MOVES", "4000"))
n0 = 2048
box = (n0 / 0.67) ** (1 / 3)
xyz, rng = E.random_initial_configuration(n0, box, 0.85, 1, device=0)
for strategy in ("microcell", "cell_list"):
    cfg = RunConfig(temperature=2.0, chemical_potential=-2.0, box_length=box, strategy=strategy)
    sim = E.Simulation(cfg, xyz, rng)
    tr = sim.run(moves, trace=True)
    print(strategy, "moves", moves, "accepted", int(tr["accepted"].sum()), "N", sim.particle_count(),
          "audit", sim.audit().passed(), flush=True)
    sim.close()
# the chain-per-SM engine (engine_mode = 2), alone and two chains in one launch
for strategy in ("microcell", "cell_list"):
    cfg = RunConfig(temperature=2.0, chemical_potential=-2.0, box_length=box, strategy=strategy)
    sims = [E.Simulation(cfg, xyz, rng, engine_mode=2) for _ in range(2)]
    tr = sims[0].run(moves, trace=True)
    res = E.run_chains(sims, [moves // 2, moves // 2])
    print(strategy, "engine_sm moves", moves, "accepted", int(tr["accepted"].sum()), "engines",
          [r.engine for r in res], "audit", sims[0].audit().passed(), flush=True)
    for s_ in sims:
        s_.close()
g = E.GpuNeighborStrategy("microcell", xyz, box)
du, dw = g.delta_batch(np.full(64, 1, np.int32), np.zeros(64, np.uint64), np.random.default_rng(1).random((64, 3)) * box)
print("delta batch ok", float(du.sum()), "energy", g.total_energy(), flush=True)
