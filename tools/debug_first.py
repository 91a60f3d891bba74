import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1408_3764_b200 import engine as E
from paper_1408_3764_b200.config import RunConfig
n0 = int(sys.argv[1]); chunk = int(sys.argv[2]); total = int(sys.argv[3])
box = (n0 / 0.67) ** (1 / 3)
xyz, rng = E.random_initial_configuration(n0, box, 0.85, 1)
cfg = RunConfig(temperature=2.0, chemical_potential=1.0, box_length=box, strategy="microcell")
sim = E.Simulation(cfg, xyz, rng)
done = 0
while done < total:
    tr = sim.run(chunk, trace=True)
    d = sim.dev.energy_drift()
    if d[0] > 1e-9:
        print("first drift after", done + chunk, d, "accepted in chunk", int(tr["accepted"].sum()), flush=True)
        acc = np.nonzero(tr["accepted"])[0]
        print("accepted moves", (done + acc).tolist()[:40], "kinds", tr["kind"][acc].tolist()[:40])
        break
    done += chunk
else:
    print("no drift", done)
