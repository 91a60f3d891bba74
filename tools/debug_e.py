import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1408_3764_b200 import engine as E
from paper_1408_3764_b200.config import RunConfig
n0 = int(sys.argv[1]); chunk = int(sys.argv[2]); total = int(sys.argv[3])
box = (n0 / 0.67) ** (1 / 3)
xyz, rng = E.random_initial_configuration(n0, box, 0.85, 1)
cfg = RunConfig(temperature=2.0, chemical_potential=1.0, box_length=box, strategy="microcell")
sim = E.Simulation(cfg, xyz, rng)
lib = sim.dev.lib
lib.gcmc_debug_energies.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
trs, done = [], 0
while done < total:
    before = sim.particles().copy()
    t = sim.run(chunk, trace=True); trs.append(t); done += chunk
    n = sim.dev.get_state().n
    m = np.zeros((n, 2)); f = np.zeros((n, 2))
    lib.gcmc_debug_energies(sim.dev.h, m.ctypes.data, f.ctypes.data)
    d = np.abs(m - f).max(axis=1)
    bad = np.nonzero(d > 1e-9)[0]
    if bad.size:
        print("after", done, "bad particles", bad[:10].tolist(), "diff", (m - f)[bad[:5]].tolist())
        pos = sim.particles()
        for p in bad[:3]:
            dx = pos - pos[p]; dx -= box * np.round(dx / box); r2 = (dx * dx).sum(1)
            nb = np.nonzero((r2 <= 6.25) & (r2 > 0))[0]
            s2 = 1.0 / r2[nb]; s6 = s2 ** 3; u = 4 * (s6 * s6 - s6)
            print(" particle", p, "pos", pos[p].tolist(), "diff u", (m - f)[p, 0], "neighbours", len(nb),
                  "matching pair:", [(int(j), float(uu)) for j, uu in zip(nb, u) if abs(abs(uu) - abs((m - f)[p, 0])) < 1e-6])
        tr = np.concatenate(trs)
        acc = np.nonzero(tr["accepted"])[0]
        print("last accepted:", [(int(k), int(tr["kind"][k]), int(tr["n_after"][k])) for k in acc[-16:]])
        break
else:
    print("no drift")
