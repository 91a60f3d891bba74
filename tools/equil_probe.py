"""How the engine behaves along the relaxation from the random start at 1M
(mu = +1): moves/s, acceptance and N per segment."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1408_3764_b200 import engine as E
from paper_1408_3764_b200.config import RunConfig
n0 = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
segs = int(sys.argv[2]) if len(sys.argv) > 2 else 12
seg = int(sys.argv[3]) if len(sys.argv) > 3 else 1 << 22
box = (n0 / 0.67) ** (1 / 3)
xyz, rng = E.random_initial_configuration(n0, box, 0.85, 1)
cfg = RunConfig(temperature=2.0, chemical_potential=1.0, box_length=box, strategy="microcell")
sim = E.Simulation(cfg, xyz, rng)
done = 0
for k in range(segs):
    a0 = sum(sim.dev.get_state().accepted)
    sim.run(seg)
    r = sim.last_run
    st = sim.dev.get_state()
    done += seg
    print(f"moves {done/1e6:6.1f}M  N={st.n}  acc={(sum(st.accepted)-a0)/seg:.4f}  "
          f"{seg/(r.device_ms/1e3):.3e} moves/s  {seg/max(r.rounds,1):.1f} moves/round  "
          f"{r.device_ms*1e3/max(r.rounds,1):.2f} us/round", flush=True)
