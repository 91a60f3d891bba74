"""Debug: chunked vs single run of the same chain; first differing move and
which one matches the reference oracle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1408_3764_b200 import engine as E
from paper_1408_3764_b200.config import RunConfig
import oracle as O

n0, seed, mu = 2048, 5, -1.0
box = (n0 / 0.67) ** (1 / 3)
xyz, rng = E.random_initial_configuration(n0, box, 0.85, seed)
cfg = RunConfig(temperature=2.0, chemical_potential=mu, box_length=box, strategy="microcell", seed=seed)
a = E.Simulation(cfg, xyz, rng)
b = E.Simulation(cfg, xyz, rng)
st = a.dev.get_state()
ta = a.run(30000, trace=True)
tb = np.concatenate([b.run(k, trace=True) for k in (1, 2, 997, 12000, 17000)])
o = O.PortSim(O.port_params(box_length=box, strategy="microcell", chemical_potential=mu), xyz,
              O.rng_from_hex(rng.serialize_hex()), energy=st.energy, virial=st.virial)
tp = o.run(30000, trace=True)
for name, t in (("single", ta), ("chunked", tb)):
    bad = np.nonzero(t["accepted"] != tp["accepted"])[0]
    du = np.abs(t["delta_u"] - tp["delta_u"]) / np.maximum(1, np.abs(tp["delta_u"]))
    print(name, "decision mismatches", bad.size, bad[:5], "max rel du", du.max(), "argmax", du.argmax())
for f in ta.dtype.names:
    d = np.nonzero(ta[f] != tb[f])[0]
    if d.size:
        i = d[0]
        print(f, "first diff at", i, ta[i], tb[i], "ref", tp[i])
print("drift single", a.dev.energy_drift(), "chunked", b.dev.energy_drift())
d = np.nonzero(np.abs(ta["delta_u"] - tb["delta_u"]) > 1e-9 * np.maximum(1, np.abs(ta["delta_u"])))[0]
print("all du diffs:", d[:40], d.size)
for i in range(12996, 13006):
    print(i, "single", ta[i], "chunked", tb[i])
