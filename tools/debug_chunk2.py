import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1408_3764_b200 import engine as E
from paper_1408_3764_b200.config import RunConfig
n0, seed, mu = 2048, 5, -1.0
box = (n0 / 0.67) ** (1 / 3)
xyz, rng = E.random_initial_configuration(n0, box, 0.85, seed)
cfg = RunConfig(temperature=2.0, chemical_potential=mu, box_length=box, strategy="microcell", seed=seed)
b = E.Simulation(cfg, xyz, rng)
for k in (1, 2, 997, 12000):
    b.run(k, trace=True)
os.environ["GCMC_ENGINE_PROFILE"] = "1"
os.environ["GCMC_ROUND_LOG"] = "1"
t = b.run(17000, trace=True)
print(t[:8])
