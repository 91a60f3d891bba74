"""Engine timing / profiling driver.

python tools/prof_engine.py --n0 32768 --mu -2 --moves 100000 [--sweep] [--ctas 8 --warps 8]
"""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1408_3764_b200 import engine as E
from paper_1408_3764_b200.config import RunConfig

ap = argparse.ArgumentParser()
ap.add_argument("--n0", type=int, default=32768)
ap.add_argument("--mu", type=float, default=-2.0)
ap.add_argument("--moves", type=int, default=100000)
ap.add_argument("--strategy", default="microcell")
ap.add_argument("--ctas", type=int, default=0)
ap.add_argument("--warps", type=int, default=0)
ap.add_argument("--variants", type=int, default=0)
ap.add_argument("--sweep", action="store_true")
ap.add_argument("--warm", type=int, default=20000)
a = ap.parse_args()

box = (a.n0 / 0.67) ** (1 / 3)
t = time.time()
xyz, rng = E.random_initial_configuration(a.n0, box, 0.85, 1)
print(f"init {time.time()-t:.1f}s", flush=True)
cfg = RunConfig(temperature=2.0, chemical_potential=a.mu, box_length=box, strategy=a.strategy)

def one(ctas, warps):
    sim = E.Simulation(cfg, xyz, rng, engine_ctas=ctas, engine_group=warps, engine_variants=a.variants)
    sim.run(a.warm)
    sim.run(a.moves)
    r = sim.last_run
    st = sim.dev.get_state()
    acc = sum(st.accepted)
    print(f"ctas={ctas} warps={warps} moves={a.moves} rounds={r.rounds} dev_ms={r.device_ms:.2f} "
          f"gen_ms={r.gen_ms:.2f} us/round={1e3*r.device_ms/max(r.rounds,1):.2f} "
          f"moves/s={a.moves/(r.device_ms/1e3):.4e} N={st.n}", flush=True)
    sim.close()

if a.sweep:
    for c, m in ((1, 1), (1, 4), (4, 4), (8, 4), (16, 1), (16, 2), (16, 4)):
        try:
            one(c, m)
        except Exception as e:
            print(f"ctas={c} moves/cta={m} failed: {e}", flush=True)
else:
    one(a.ctas, a.warps)
