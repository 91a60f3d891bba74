"""Many chains per GPU: K independent GCMC chains of a mu
isotherm run concurrently on one B200, each engine on its own subset of SMs
(engine_ctas = SMs // K) and its own stream; one host thread per chain
(ctypes releases the GIL inside gcmc_run_moves).

    python tools/sweep_multichain.py --n0 65536 --chains 8 --moves 262144

Reports per-chain and aggregate moves/s. The aggregate is taken over the
concurrent region (all chains synchronised before and after; wall clock of
that region, which is all device work) and compared with one chain alone.
"""
import argparse
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1408_3764_b200 import engine as E  # noqa: E402
from paper_1408_3764_b200.config import RunConfig  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n0", type=int, default=1 << 16)
ap.add_argument("--chains", type=int, default=8)
ap.add_argument("--moves", type=int, default=1 << 18)
ap.add_argument("--warm", type=int, default=1 << 17)
ap.add_argument("--sms", type=int, default=148)
a = ap.parse_args()

box = (a.n0 / 0.67) ** (1.0 / 3.0)
ctas = max(2, a.sms // a.chains)
sims = []
for g in range(a.chains):
    mu = -3.0 + g
    xyz, rng = E.random_initial_configuration(a.n0, box, 0.85, 1 + g)
    cfg = RunConfig(temperature=2.0, chemical_potential=mu, box_length=box, seed=1 + g,
                    strategy="microcell")
    sims.append(E.Simulation(cfg, xyz, rng, engine_ctas=ctas))


def run_all(n):
    ts = [threading.Thread(target=s.run, args=(n,)) for s in sims]
    t0 = time.perf_counter()
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    return time.perf_counter() - t0


run_all(a.warm)
dt = run_all(a.moves)
agg = a.chains * a.moves / dt
per = [a.moves / (s.last_run.device_ms / 1e3) for s in sims]
print(f"{a.chains} chains x {a.n0} particles, {ctas} CTAs each: aggregate {agg:.4e} moves/s "
      f"over {dt*1e3:.1f} ms; per chain (device) " + " ".join(f"{p:.3e}" for p in per))
for g, s in enumerate(sims):
    st = s.dev.get_state()
    print(f"  mu={-3.0 + g:+.0f}: N={st.n} acc={sum(st.accepted)}/{sum(st.attempted)}")
# one chain alone with the whole GPU, for comparison
solo = sims[0]
solo_dev = E.Simulation(solo.cfg, solo.dev.positions(), solo.dev.get_rng())
t0 = time.perf_counter()
solo_dev.run(a.moves)
print(f"1 chain, whole GPU: {a.moves / (time.perf_counter() - t0):.4e} moves/s (wall), "
      f"{a.moves / (solo_dev.last_run.device_ms / 1e3):.4e} (device)")
