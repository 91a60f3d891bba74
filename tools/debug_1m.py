import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1408_3764_b200 import engine as E
from paper_1408_3764_b200.config import RunConfig
import oracle as O
n0 = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
moves = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
box = (n0 / 0.67) ** (1 / 3)
xyz, rng = E.random_initial_configuration(n0, box, 0.85, 1)
cfg = RunConfig(temperature=2.0, chemical_potential=1.0, box_length=box, strategy="microcell")
sim = E.Simulation(cfg, xyz, rng)
st = sim.dev.get_state()
for k in range(4):
    tr = sim.run(moves // 4, trace=True)
    print("chunk", k, "acc", tr["accepted"].mean(), "drift", sim.dev.energy_drift(), flush=True)
