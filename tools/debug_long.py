import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1408_3764_b200 import engine as E
from paper_1408_3764_b200.config import RunConfig
n0 = int(sys.argv[1]); steps = int(sys.argv[2]); per = int(sys.argv[3])
box = (n0 / 0.67) ** (1 / 3)
xyz, rng = E.random_initial_configuration(n0, box, 0.85, 1)
cfg = RunConfig(temperature=2.0, chemical_potential=1.0, box_length=box, strategy="microcell")
sim = E.Simulation(cfg, xyz, rng)
for k in range(steps):
    st0 = sim.dev.get_state()
    t = time.time()
    try:
        sim.run(per)
    except Exception as e:
        print("step", k, "FAILED", e, flush=True)
        break
    st = sim.dev.get_state()
    acc = (sum(st.accepted) - sum(st0.accepted)) / per
    print("step", k, "n", st.n, "acc", round(acc, 4), "drift", sim.dev.energy_drift(), "peak", st.peak_occupancy, round(time.time() - t, 2), flush=True)
