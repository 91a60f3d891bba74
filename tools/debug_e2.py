import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
os.environ["GCMC_ENGINE_PROFILE"] = "1"; os.environ["GCMC_PROF_MASK"] = "16"; os.environ["GCMC_ROUND_LOG"] = "1"
from paper_1408_3764_b200 import engine as E
from paper_1408_3764_b200.config import RunConfig
n0 = 32768
box = (n0 / 0.67) ** (1 / 3)
xyz, rng = E.random_initial_configuration(n0, box, 0.85, 1)
cfg = RunConfig(temperature=2.0, chemical_potential=1.0, box_length=box, strategy="microcell")
sim = E.Simulation(cfg, xyz, rng)
t = sim.run(1024, trace=True)
print("drift", sim.dev.energy_drift())
