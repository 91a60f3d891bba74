import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1408_3764_b200 import engine as E
from paper_1408_3764_b200.config import RunConfig
import oracle as O
n0 = int(sys.argv[1]); chunk = int(sys.argv[2]); total = int(sys.argv[3])
box = (n0 / 0.67) ** (1 / 3)
xyz, rng = E.random_initial_configuration(n0, box, 0.85, 1)
cfg = RunConfig(temperature=2.0, chemical_potential=1.0, box_length=box, strategy="microcell")
sim = E.Simulation(cfg, xyz, rng)
st = sim.dev.get_state()
o = O.PortSim(O.port_params(box_length=box, strategy="microcell", chemical_potential=1.0), xyz,
              O.rng_from_hex(rng.serialize_hex()), energy=st.energy, virial=st.virial)
trs = []
done = 0
while done < total:
    trs.append(sim.run(chunk, trace=True)); done += chunk
tr = np.concatenate(trs)
tp = o.run(total, trace=True)
rel = np.abs(tr["delta_u"] - tp["delta_u"]) / np.maximum(1, np.abs(tp["delta_u"]))
bad = np.nonzero(rel > 1e-9)[0]
print("du mismatches", bad.size, bad[:10].tolist())
dec = np.nonzero(tr["accepted"] != tp["accepted"])[0]
print("decision mismatches", dec.size, dec[:10].tolist())
for i in bad[:3]:
    print(i, tr[i], tp[i], "diff", tr["delta_u"][i] - tp["delta_u"][i])
    acc = np.nonzero(tr["accepted"][max(0, i - 600):i])[0] + max(0, i - 600)
    print("  accepted before:", [(int(k), int(tr["kind"][k])) for k in acc[-12:]])
print("drift", sim.dev.energy_drift())
